"""K3 (accumulate) probe: time ParamBuffer.accumulate_flat over the C2
gradient pages (first-message mode, 4 B/param), in add mode (6 B/param) and with mixed
per-layer modes, with and without the fused ledger sums.  Prints one JSON line per variant.

    python tools/k3_probe.py [--config c2] [--reps 20]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2303_02868_b200 import lockfree as LF  # noqa: E402
from paper_2303_02868_b200 import workloads as W  # noqa: E402
from paper_2303_02868_b200.layout import PageLayout  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="", help="ledger,mode (e.g. 0,first): one variant")
    args = ap.parse_args()
    only = tuple(args.only.split(",")) if args.only else None
    dev = torch.device("cuda", 0)
    specs = W.config_specs(args.config)
    numels = [s.bytes // 2 for s in specs]
    lay = PageLayout(numels, W.config_page_bytes(args.config))
    P = sum(numels)
    params = [torch.zeros(n, device=dev) for n in numels]
    g = torch.randn(P, device=dev).mul_(1e-2).to(torch.bfloat16)
    for ledger in (False, True):
        buf = LF.ParamBuffer(params, dtype="bf16", layout=lay, device=dev, ledger=ledger)
        for per_cta in (1,):
            for mode in ("first", "add", "mixed"):
                if only and only != (str(int(ledger)), mode):
                    continue

                def once():
                    for l in range(len(numels)):
                        buf._pending[l] = 0 if mode == "first" else 1 if mode == "add" else l % 2
                    buf._ring_pos = 0   # probe only: recycle the ledger row without resolving
                    buf.ledger._unresolved.clear()
                    buf.accumulate_flat(g, 0)
                for _ in range(50):          # clocks up, caches warm
                    once()
                torch.cuda.synchronize()
                best = float("inf")
                for _ in range(3):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(args.reps):
                        once()
                    b.record()
                    torch.cuda.synchronize()
                    best = min(best, a.elapsed_time(b) / args.reps)
                ms = best
                bpp = 4 if mode == "first" else 6 if mode == "add" else 5
                print(json.dumps({"ledger": ledger, "mode": mode, "ms": ms,
                                  "gbs": bpp * P / ms / 1e6, "bytes_per_param": bpp}), flush=True)
        del buf
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
