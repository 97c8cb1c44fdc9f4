"""Probe: CUDA green contexts (SM partitions) through torch, with our C-ABI
kernels launched on their streams.  Two HBM-streaming copies on two
partitions should overlap (concurrent time ~ max, not sum) and each should
slow down in proportion to its SM share only if it is SM-bound.

    python tools/green_probe.py
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2303_02868_b200 import _device as D  # noqa: E402
from paper_2303_02868_b200 import _native as N  # noqa: E402


def handle(s):
    for a in ("cuda_stream", "native_handle", "stream_id"):
        if hasattr(s, a):
            v = getattr(s, a)
            return int(v() if callable(v) else v), a
    raise RuntimeError(f"no raw handle on {type(s)}: {dir(s)}")


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    out = {"supported": torch.cuda.green_contexts.SUPPORTED}
    nbytes = 1 << 30
    a = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    b = torch.empty_like(a)
    c = torch.empty_like(a)
    d = torch.empty_like(a)
    piece = 64 * 1024
    desc = np.array([(i * piece, i * piece, piece) for i in range(nbytes // piece)], dtype=N.COPY_DESC)
    dd = torch.from_numpy(desc.view(np.uint8).copy()).to(dev)
    lib = N.lib()

    def copy(src, dst, sh):
        D.check(lib.hm_copy_runs(D.ptr(src), D.ptr(dst), D.ptr(dd), len(desc), sh))

    def timed(fn, reps=5):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    cur = torch.cuda.current_stream(dev)
    out["one_copy_full_gpu_ms"] = timed(lambda: copy(a, b, D.sptr(cur)))
    G = torch.cuda.green_contexts.GreenContext
    g1, g2 = G.create(32, 0), G.create(112, 0)
    s1, s2 = g1.Stream(), g2.Stream()
    h1, attr = handle(s1)
    h2, _ = handle(s2)
    out["handle_attr"] = attr
    import ctypes as C
    p1, p2 = C.c_void_p(h1), C.c_void_p(h2)
    out["copy_on_32sm_ms"] = timed(lambda: copy(a, b, p1))
    out["copy_on_112sm_ms"] = timed(lambda: copy(c, d, p2))

    def both():
        copy(a, b, p1)
        copy(c, d, p2)
    out["both_concurrent_ms"] = timed(both)
    out["both_serial_ms"] = out["copy_on_32sm_ms"] + out["copy_on_112sm_ms"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
