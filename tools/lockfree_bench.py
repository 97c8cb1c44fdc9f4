"""Lock-free delayed update vs synchronous update on one B200 (Algorithm 2,
PAPER.md:541-612; the reference's scripts/lockfree_speedup.py measures the
same ratio on a simulated clock).

The fp32 master state lives in pinned host memory (swap tier), so every
update moves 24 B/param over PCIe; the GPU actor runs a wide tanh-MLP
forward/backward.  delay=0 waits for each update before the next forward;
delay=1 overlaps the update of step k with the compute of step k+1.

    python tools/lockfree_bench.py [--layers 8] [--dim 8192] [--batch 4096] [--iters 20]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2303_02868_b200 import lockfree as LF  # noqa: E402
from paper_2303_02868_b200.actors import LockFreeRunner  # noqa: E402
from paper_2303_02868_b200.swap import HostMasterState  # noqa: E402
from paper_2303_02868_b200.toy import ToyMLP  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--dim", type=int, default=8192)
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--state", default="host", choices=["host", "hbm"])
    ap.add_argument("--tf32", action="store_true", help="TF32 tensor-core matmuls in the GPU actor")
    args = ap.parse_args()
    torch.backends.cuda.matmul.allow_tf32 = args.tf32
    out = {"layers": args.layers, "dim": args.dim, "batch": args.batch, "iters": args.iters, "tf32": args.tf32,
           "params": args.layers * args.dim * args.dim, "state": args.state}
    hyper = LF.AdamHyper(lr=1e-4)
    for delay in (0, 1):
        toy = ToyMLP(num_layers=args.layers, dim=args.dim, batch_size=args.batch, seed=3)
        buf = LF.ParamBuffer(toy.student, dtype="bf16")
        ms = (HostMasterState(toy.student, group_pages=32) if args.state == "host"
              else LF.MasterState(toy.student))
        runner = LockFreeRunner(buf, ms, hyper, delay=delay)
        runner.run(3, toy.grads_fn)  # warm-up
        rep = runner.run(args.iters, toy.grads_fn, mode="lockfree" if delay else "sync")
        out[f"delay{delay}"] = {"iter_ms": rep.iter_ms, "final_loss": rep.loss_curve[-1],
                                "max_staleness": rep.max_staleness,
                                "val_loss": toy.val_loss([buf.layer_view(l) for l in range(args.layers)])}
        del buf, ms, runner, toy
        torch.cuda.empty_cache()
    out["speedup"] = out["delay0"]["iter_ms"] / out["delay1"]["iter_ms"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
