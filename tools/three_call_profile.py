"""Host-side profile (cProfile) of the reference's per-layer loop through the
drop-in (take -> update_layer -> publish, torch tensors) on C2: where the
~190 us per layer of launch overhead goes.  python tools/three_call_profile.py"""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2303_02868_b200 import lockfree as LF  # noqa: E402
from paper_2303_02868_b200 import workloads as W  # noqa: E402
from paper_2303_02868_b200.layout import PageLayout  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    specs = W.config_specs("c2")
    numels = [s.bytes // 2 for s in specs]
    lay = PageLayout(numels, W.config_page_bytes("c2"))
    params = [torch.zeros(n, device=dev) for n in numels]
    buf = LF.ParamBuffer(params, dtype="bf16", layout=lay, device=dev)
    ms = LF.MasterState(params, layout=lay, device=dev)
    del params
    g = torch.randn(sum(numels), device=dev).mul_(1e-2).to(torch.bfloat16)
    hyper = LF.AdamHyper(lr=1e-3)

    def step():
        buf.accumulate_flat(g, 0)
        for l in reversed(range(len(numels))):
            gr, _c, newest = buf.take(l)
            ms.update_layer(l, gr, hyper)
            buf.publish(l, ms.p32[l], applied_iter=newest, clear=False)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
