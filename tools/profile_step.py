"""Minimal driver for ncu: build the context for a config and run W+K hot-path steps."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--nel", type=int, default=0)
ap.add_argument("--tile-sparse", action="store_true")
args = ap.parse_args()

import torch  # noqa: E402

from paper_2312_12771_b200 import workloads as W  # noqa: E402
from paper_2312_12771_b200.hom import Homogenizer  # noqa: E402

wl = W.make(args.config, **({"nel": args.nel} if args.nel else {}))
h = Homogenizer.from_workload(wl, tile_sparse=args.tile_sparse)
for _ in range(args.steps):
    C = h.condense()
    u, info = h.macro_solve(C)
    w = h.recover(u)
torch.cuda.synchronize()
print("ok", info.iterations)
