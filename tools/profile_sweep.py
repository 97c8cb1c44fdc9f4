"""Small driver for ncu captures: builds a workload's page pools and runs a
few fused sweeps (and one flat accumulate) so the kernels can be profiled.

    python tools/profile_sweep.py --config c2 --steps 3
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2303_02868_b200 import lockfree as LF  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--page-mib", type=int, default=0)
    ap.add_argument("--bucket-pages", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    specs, page, layout, buf, ms = bench.build_state(args, dev)
    grads = torch.cat(bench.synthetic_grads(layout.numels, args.dtype, dev, 7))
    hyper = LF.AdamHyper(lr=1e-3)
    for i in range(args.steps):
        buf.accumulate_flat(grads, i)
        LF.sweep(buf, ms, hyper)
    torch.cuda.synchronize()
    print("ok", sum(layout.numels), "params")


if __name__ == "__main__":
    main()
