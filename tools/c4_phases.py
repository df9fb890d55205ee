"""C4 (1,000,000 dependent 4 KiB tasks) end-to-end phase breakdown:
run with BT_DEBUG_TIMING=1 to get the builder's per-phase timings on stderr.

    BT_DEBUG_TIMING=1 python tools/c4_phases.py [--fused]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1304_0878_b200 import btask as B  # noqa: E402
from config_bench import run  # noqa: E402

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--fused", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    p = W.c4_fine()
    run("C4 " + ("fused" if args.fused else "unfused"), p, args.reps,
        flags=0 if args.fused else B.BT_FLAG_NO_FUSION)
