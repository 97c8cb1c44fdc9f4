"""K3 (accumulate) probe: time hm_accumulate over the C2 gradient pages with
and without the fused statistics, in overwrite and add mode, to locate the
cost of the flag/norm epilogue.  python tools/k3_probe.py"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_02868_b200 import _device as D  # noqa: E402
from paper_2303_02868_b200 import _native as N  # noqa: E402
from paper_2303_02868_b200 import workloads as W  # noqa: E402
from paper_2303_02868_b200.layout import PageLayout  # noqa: E402


def main():
    specs = W.config_specs("c2")
    lay = PageLayout([s.bytes // 2 for s in specs], 4 << 20)
    L = len(specs)
    parts, base = [], 0
    for l, n in enumerate(lay.numels):
        c = lay.seg_chunks(l, "16").copy()
        c["src_off"] += base
        c["slot"] = l
        parts.append(c)
        base += n
    ch = np.concatenate(parts)
    dev = torch.device("cuda", 0)
    dch = torch.from_numpy(ch.view(np.uint8).copy()).to(dev)
    src = torch.randn(base, device=dev).to(torch.bfloat16)
    dst = torch.zeros(lay.elems16, dtype=torch.bfloat16, device=dev)
    flags = torch.zeros(L, dtype=torch.int32, device=dev)
    sumsq = torch.zeros(L, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev)
    lib = N.lib()
    out = {"params": base, "chunks": len(ch)}
    for name, mode, f, s in [("overwrite+stats", 0, flags, sumsq), ("overwrite+flag", 0, flags, None),
                             ("overwrite-nostats", 0, None, None), ("add+stats", 1, flags, sumsq)]:
        def run():
            D.check(lib.hm_accumulate(D.ptr(src), N.DT_BF16, D.ptr(dst), N.DT_BF16, D.ptr(dch), len(ch),
                                      mode, None, D.ptr(f) if f is not None else None,
                                      D.ptr(s) if s is not None else None, D.sptr(st)))
        run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(20):
            run()
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 20
        nbytes = (6 if mode else 4) * base
        out[name] = {"ms": ms, "gbs": nbytes / (ms / 1e3) / 1e9}
    # the cast kernel over the same chunks (same geometry, no statistics)
    def cast():
        D.check(lib.hm_cast(D.ptr(src), N.DT_BF16, D.ptr(dst), N.DT_BF16, D.ptr(dch), len(ch), D.sptr(st)))
    cast()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(20):
        cast()
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    out["cast_bf16"] = {"ms": ms, "gbs": 4 * base / (ms / 1e3) / 1e9}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
