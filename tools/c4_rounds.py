"""C4 wall / device time vs the number of pipelined rounds (tools/config_bench.run).
    python tools/c4_rounds.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402
import workloads as W  # noqa: E402
from paper_1304_0878_b200 import btask as B  # noqa: E402
from config_bench import run  # noqa: E402
torch.cuda.set_device(0)
p = W.c4_fine()
for rounds in (4, 6, 8):
    for name, flags in (("unfused", B.BT_FLAG_NO_FUSION), ("fused", 0)):
        run(f"C4 {name} rounds={rounds}", p, 7, flags=flags, pipeline_rounds=rounds)
