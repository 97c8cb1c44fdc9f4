"""NVLink evidence for the fused DP kernels, in ONE process (so ncu can
profile GPU 0 alone while its peers are plain mapped memory):

    python tools/nvlink_probe.py [--gpus 2] [--config c2] [--reps 5]
    ncu --devices 0 -k regex:"reduce_check|adam_main" --metrics \
        gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        python tools/nvlink_probe.py --reps 1

Every GPU holds the rank-r state of the C2 page layout (world = --gpus) with
peer access enabled between all pairs; a step is the fused DP step of
sharding.FusedShardedPageStep.step through the same C-ABI entry points
(hm_dp_reduce_check reading the owned pages from every peer, then prologue
+ hm_adam_main_ag storing the published pages into every peer), with host
synchronisation standing in for the cross-process signal barriers.
Timings are CUDA events per device, max over devices; busbw = pool bytes
x (N-1)/N / t.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from bench import build_state  # noqa: E402
from paper_2303_02868_b200 import _device as D  # noqa: E402
from paper_2303_02868_b200 import _native as N  # noqa: E402
from paper_2303_02868_b200 import lockfree as LF  # noqa: E402
from paper_2303_02868_b200.dp_bench import owned_grad_flat  # noqa: E402


def arr(ptrs):
    import ctypes as C
    return (C.c_uint64 * len(ptrs))(*ptrs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--reduce-ctas", type=int, nargs="*", default=[])
    ap.add_argument("--ag-publish", type=int, nargs="*", default=[])
    ap.add_argument("--onepass", action="store_true",
                    help="time the one-pass DP kernel (hm_dp_onepass_update) over double-buffered state")
    ap.add_argument("--solo", action="store_true",
                    help="only GPU 0 launches (clean ncu counters: no peer traffic into GPU 0)")
    args = ap.parse_args()
    n = min(args.gpus, torch.cuda.device_count())
    if n < 2:
        print(json.dumps({"probe": "nvlink", "skipped": "needs >= 2 GPUs in one process"}))
        return
    for a in range(n):
        for b in range(n):
            if a != b and not torch.cuda.can_device_access_peer(a, b):
                raise SystemExit(f"GPU {a} cannot access GPU {b}")
    # a cross-device copy makes torch enable peer access for that pair
    for a in range(n):
        for b in range(n):
            if a != b:
                torch.ones(4, device=f"cuda:{a}").copy_(torch.ones(4, device=f"cuda:{b}"))
    bargs = SimpleNamespace(config=args.config, dtype=args.dtype, page_mib=None, bucket_pages=32)
    ranks = []
    for r in range(n):
        dev = torch.device("cuda", r)
        with torch.cuda.device(dev):
            specs, page, lay, buf, ms = build_state(bargs, dev, n, r, double_buffered=args.onepass)
            buf.accumulate_flat(owned_grad_flat(lay, args.dtype, dev, 7 + r), 0)
            L = len(specs)
            span = lay.elems16
            g = np.zeros(L, dtype=N.GROUP_LAUNCH)
            for l in range(L):
                g[l] = (0, span, l, l)
            ranks.append(dict(dev=dev, lay=lay, buf=buf, ms=ms, L=L, groups=g,
                              check=lay.pool_chunks(range(L), "16", owned_only=True),
                              adam=lay.adam_chunks(range(L), "pool", owned_only=True),
                              flags=torch.zeros(L, dtype=torch.int32, device=dev),
                              sumsq=torch.zeros(L, dtype=torch.float64, device=dev),
                              stream=torch.cuda.Stream(dev)))
    g_ptrs = [D.ptr(x["buf"].g16_pool[0]) for x in ranks]
    p_ptrs = [D.ptr(x["buf"].p16_pool) for x in ranks]
    hyper = LF.AdamHyper(lr=1e-3, inv_scale=1.0 / n)
    hc = D.hyper_c(hyper)
    lib = N.lib()

    def sync_all():
        for x in ranks:
            torch.cuda.synchronize(x["dev"])

    def phase(fn):
        evs = []
        for x in (ranks[:1] if args.solo else ranks):
            with torch.cuda.device(x["dev"]), torch.cuda.stream(x["stream"]):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(x["stream"])
                fn(x)
                b.record(x["stream"])
                evs.append((a, b))
        sync_all()
        return max(a.elapsed_time(b) for a, b in evs)

    def rs(x):
        eng, buf = x["ms"]._eng, x["buf"]
        x["flags"].zero_()
        D.check(lib.hm_dp_reduce_check(arr(g_ptrs), n, None, D.ptr(buf.g16_pool[0]), buf._dt,
                                       D.ptr(eng.desc.static(x["check"])), len(x["check"]),
                                       D.ptr(x["flags"]), D.ptr(x["sumsq"]), None, D.sptr(x["stream"])))

    def upd(x):
        eng, buf, ms = x["ms"]._eng, x["buf"], x["ms"]
        dgroups = eng.desc.table(x["groups"])
        rt = eng.rt_scratch(x["L"], x["stream"])
        bc, bc_len = ms._bias(hyper, range(x["L"]))
        D.check(lib.hm_adam_prologue(D.ptr(dgroups), x["L"], D.ptr(rt), hc, D.ptr(bc), bc_len, 0,
                                     D.ptr(ms._steps), D.ptr(ms._applied), D.ptr(x["flags"]),
                                     None, 1, None, None, D.sptr(x["stream"])))
        D.check(lib.hm_adam_main_ag(D.ptr(eng.desc.static(x["adam"])), len(x["adam"]), D.ptr(dgroups),
                                    D.ptr(rt), D.ptr(buf.g16_pool), buf._dt, D.ptr(ms.p32_pool),
                                    D.ptr(ms.m32_pool), D.ptr(ms.v32_pool), arr(p_ptrs), n, None,
                                    buf._dt, hc, None, D.sptr(x["stream"])))

    def onepass(x):
        eng, buf, ms = x["ms"]._eng, x["buf"], x["ms"]
        dgroups = eng.desc.table(x["groups"])
        rt = eng.rt_scratch(x["L"], x["stream"])
        bc, bc_len = ms._bias(hyper, range(x["L"]))
        x["flags"].zero_()
        D.check(lib.hm_adam_prologue(D.ptr(dgroups), x["L"], D.ptr(rt), hc, D.ptr(bc), bc_len, 0,
                                     D.ptr(ms._steps_spec), None, None, None, 1, None, None,
                                     D.sptr(x["stream"])))
        D.check(lib.hm_dp_onepass_update(D.ptr(eng.desc.static(x["adam"])), len(x["adam"]), D.ptr(dgroups),
                                         D.ptr(rt), D.ptr(ms._state_sel), x["lay"].elems_state,
                                         arr([D.ptr(y["buf"].g16_pool) for y in ranks]), arr(p_ptrs), n,
                                         buf._dt, D.ptr(ms.p32_pool), D.ptr(ms.m32_pool), D.ptr(ms.v32_pool),
                                         D.ptr(x["flags"]), hc, None, D.sptr(x["stream"])))

    if args.onepass:
        sync_all()
        phase(onepass)
        t = float(np.median([phase(onepass) for _ in range(max(1, args.reps))]))
        lay = ranks[0]["lay"]
        S = 2 * sum(lay.numels)
        print(json.dumps({"probe": "nvlink_onepass", "gpus": n, "config": args.config, "onepass_ms": t,
                          "link_bytes_per_direction": 2 * S * (n - 1) / n,
                          "link_gbs": 2 * S * (n - 1) / n / (t / 1e3) / 1e9,
                          "hbm_algorithmic_bytes_per_gpu": (2 + 24 + 2) * lay.owned_numel()}))
        return
    sync_all()
    rs_ms, up_ms = [], []
    for _ in range(args.reps):
        rs_ms.append(phase(rs))
        up_ms.append(phase(upd))
    lay = ranks[0]["lay"]
    S = 2 * sum(lay.numels)   # algorithmic bytes: the padding of the pool never moves
    # reduce with 256-bit peer loads
    D.check(lib.hm_set_dp_reduce_wide(1))
    phase(rs)
    rs_wide_ms = float(np.median([phase(rs) for _ in range(max(3, args.reps))]))
    D.check(lib.hm_set_dp_reduce_wide(0))
    # update + AG with the bulk-copy publish epilogues
    upd_by_publish = {}
    for mode in args.ag_publish:
        D.check(lib.hm_set_ag_publish(mode))
        phase(upd)
        upd_by_publish[mode] = float(np.median([phase(upd) for _ in range(3)]))
    D.check(lib.hm_set_ag_publish(0))
    # reduce alone on a persistent grid of C CTAs (the pipelined step's knob)
    rs_by_ctas = {}
    for ctas in args.reduce_ctas:
        D.check(lib.hm_set_dp_reduce_ctas(ctas))
        phase(rs)
        rs_by_ctas[ctas] = float(np.median([phase(rs) for _ in range(3)]))
    D.check(lib.hm_set_dp_reduce_ctas(0))

    # Copy-engine reference for the same exchange: every GPU pulls S/N bytes
    # from every peer at once (cudaMemcpyAsync peer copies, one stream per peer).
    part = S // n // 2
    bufs = [torch.empty(part, dtype=torch.int16, device=x["dev"]) for x in ranks]
    dsts = [[torch.empty(part, dtype=torch.int16, device=x["dev"]) for _ in range(n)] for x in ranks]
    cstreams = [[torch.cuda.Stream(x["dev"]) for _ in range(n)] for x in ranks]

    def ce_round():
        evs = []
        for r, x in enumerate(ranks):
            with torch.cuda.device(x["dev"]):
                a = torch.cuda.Event(enable_timing=True)
                a.record(x["stream"])
                ends = []
                for q in range(n):
                    if q == r:
                        continue
                    s = cstreams[r][q]
                    s.wait_event(a)
                    with torch.cuda.stream(s):
                        dsts[r][q].copy_(bufs[q], non_blocking=True)
                        e = torch.cuda.Event(enable_timing=True)
                        e.record(s)
                        ends.append(e)
                evs.append((a, ends))
        sync_all()
        return max(max(a.elapsed_time(e) for e in ends) for a, ends in evs)

    ce_round()
    ce_ms = float(np.median([ce_round() for _ in range(max(3, args.reps))]))
    owned = lay.owned_numel()
    t_rs, t_up = float(np.median(rs_ms)), float(np.median(up_ms))
    bus = lambda t: S * (n - 1) / n / (t / 1e3) / 1e9
    print(json.dumps({
        "probe": "nvlink", "gpus": n, "config": args.config, "pool_bytes": S, "reps": args.reps,
        "reduce_check_ms": t_rs, "rs_busbw_gbs": bus(t_rs), "rs_frac_770": bus(t_rs) / 770.0,
        "adam_ag_ms": t_up, "ag_busbw_gbs": bus(t_up), "ag_frac_770": bus(t_up) / 770.0,
        "adam_hbm_gbs": 28 * owned / (t_up / 1e3) / 1e9,
        "ce_pull_ms": ce_ms, "ce_pull_busbw_gbs": bus(ce_ms),
        "reduce_ms_by_persistent_ctas": rs_by_ctas, "reduce_256bit_ms": rs_wide_ms, "adam_ag_ms_by_publish_mode": upd_by_publish,
        "rs_nvlink_bytes_in_per_gpu": S * (n - 1) / n, "ag_nvlink_bytes_out_per_gpu": S * (n - 1) / n,
    }))


if __name__ == "__main__":
    main()
