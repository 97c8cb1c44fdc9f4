"""One GPU: the owned-page update of rank 0 of a 2-way layout launched as
(a) hm_adam_main (local publish) and (b) hm_adam_main_ag with the local pool
as its only "peer" — same chunks, same bytes — to tell whether the HBM write
surplus seen for the peer-publish kernel (profiles/r1_nvlink_ncu.md) comes
from the kernel variant or from the remote stores.

    ncu -k regex:adam_main --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        python tools/publish_probe.py
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import build_state  # noqa: E402
from paper_2303_02868_b200 import _device as D  # noqa: E402
from paper_2303_02868_b200 import _native as N  # noqa: E402
from paper_2303_02868_b200 import lockfree as LF  # noqa: E402
from paper_2303_02868_b200.dp_bench import owned_grad_flat  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    bargs = SimpleNamespace(config="c2", dtype="bf16", page_mib=None, bucket_pages=32)
    specs, page, lay, buf, ms = build_state(bargs, dev, 2, 0)
    buf.accumulate_flat(owned_grad_flat(lay, "bf16", dev, 7), 0)
    L = len(specs)
    g = np.zeros(L, dtype=N.GROUP_LAUNCH)
    for l in range(L):
        g[l] = (0, lay.elems16, l, l)
    eng, lib = ms._eng, N.lib()
    adam = lay.adam_chunks(range(L), "pool", owned_only=True)
    st = torch.cuda.current_stream(dev)
    dgroups, rt = eng.desc.table(g), eng.rt_scratch(L, st)
    hyper = LF.AdamHyper(lr=1e-3)
    hc = D.hyper_c(hyper)
    bc, bc_len = ms._bias(hyper, range(L))
    flags = torch.zeros(L, dtype=torch.int32, device=dev)
    own = (C.c_uint64 * 1)(D.ptr(buf.p16_pool))
    times = {}
    for name in ("local", "peer_self", "local", "peer_self"):
        D.check(lib.hm_adam_prologue(D.ptr(dgroups), L, D.ptr(rt), hc, D.ptr(bc), bc_len, 0,
                                     D.ptr(ms._steps), D.ptr(ms._applied), D.ptr(flags), None, 1,
                                     None, None, D.sptr(st)))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        if name == "local":
            D.check(lib.hm_adam_main(D.ptr(eng.desc.static(adam)), len(adam), D.ptr(dgroups), D.ptr(rt),
                                     D.ptr(buf.g16_pool), buf._dt, D.ptr(ms.p32_pool), D.ptr(ms.m32_pool),
                                     D.ptr(ms.v32_pool), D.ptr(buf.p16_pool), buf._dt, hc, None, D.sptr(st)))
        else:
            D.check(lib.hm_adam_main_ag(D.ptr(eng.desc.static(adam)), len(adam), D.ptr(dgroups), D.ptr(rt),
                                        D.ptr(buf.g16_pool), buf._dt, D.ptr(ms.p32_pool),
                                        D.ptr(ms.m32_pool), D.ptr(ms.v32_pool), own, 1, None, buf._dt,
                                        hc, None, D.sptr(st)))
        b.record(st)
        torch.cuda.synchronize()
        times[name] = a.elapsed_time(b)
    owned = lay.owned_numel()
    print(json.dumps({"probe": "publish", "owned_params": owned, "algorithmic_bytes": 28 * owned,
                      "ms": times, "gbs": {k: 28 * owned / (v / 1e3) / 1e9 for k, v in times.items()}}))


if __name__ == "__main__":
    main()
