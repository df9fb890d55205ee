"""C2 fused (direct launch) device time vs the direct kernel's chunk, L2 flushed
before each rep.   BT_DIRECT_CHUNK=<floats> python tools/c2_direct.py"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402
import workloads as W  # noqa: E402
from paper_1304_0878_b200 import btask as B  # noqa: E402
import bench_configs as bc  # noqa: E402
torch.cuda.set_device(0)
p = W.c2_chain()
fl = bc._L2Flush(torch, 0)
r, _ = bc._run(torch, B, p, 15, flush=fl)
print(json.dumps({"chunk": os.environ.get("BT_DIRECT_CHUNK", "16384"), "device_us": r["device_span_ms"] * 1e3,
                  "kernel_us": r["kernel_ms"] * 1e3, "wall_us": r["wall_ms"] * 1e3}), flush=True)
