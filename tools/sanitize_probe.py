"""Every kernel of libhm_page.so at small sizes in ONE process, for
compute-sanitizer (memcheck / racecheck / synccheck — one tool per run):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_probe.py

Covers: K3 accumulate in its three forms (+ ledger), hm_stats_take, hm_cast,
hm_reduce_stats, the fused sweep (prologue + page-Adam, 256 and 512 threads,
LDG and TMA bulk-copy variants), apply_update, update_layer (both paths),
take/publish, hm_copy_runs, ingest_sweep with results, the swap tier, and
the DP kernels with the local pool standing in for every peer (the reduce
in both load widths and as a persistent grid, the flag merge, the update
with the per-thread and the staged bulk-copy all-gather epilogue, the
persistent update grid).  Each result is checked against the plain path so
a sanitizer-clean run is also a correct one.
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_02868_b200 import _device as D  # noqa: E402
from paper_2303_02868_b200 import _native as N  # noqa: E402
from paper_2303_02868_b200 import lockfree as LF  # noqa: E402
from paper_2303_02868_b200.pages import DevicePageManager  # noqa: E402

SIZES = [70001, 1, 5, 32768, 40000, 25003, 777, 12, 33333]
PAGE = 64 * 1024


def main():
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    params = [torch.from_numpy(rng.normal(0, 0.02, n).astype(np.float32)).to(dev) for n in SIZES]
    hyper = LF.AdamHyper(lr=1e-3)
    done = []
    for dtype in ("bf16", "fp16"):
        buf = LF.ParamBuffer(params, dtype=dtype, page_bytes=PAGE)
        ms = LF.MasterState(params, page_bytes=PAGE)
        tdt = D.TORCH16[dtype]
        flat = torch.from_numpy(rng.normal(0, 1e-2, sum(SIZES)).astype(np.float32)).to(dev).to(tdt)
        buf.accumulate_flat(flat, 0)                       # K3 first-message form
        buf.accumulate_flat(flat, 1)                       # K3 add form
        buf.take(2)
        buf.accumulate_flat(flat, 2)                       # K3 mixed form (+ hm_stats_take above)
        for threads, variant in ((256, 0), (512, 0), (256, 1)):
            LF.sweep(buf, ms, hyper, opts=D.opts(adam_threads=threads, adam_variant=variant))
            buf.accumulate_flat(flat, 3)
        g, _, newest = buf.take(4)                         # three-call fast path
        ms.update_layer(4, g, hyper)
        buf.publish(4, ms.p32[4], applied_iter=newest, clear=False)
        ms.update_layer(5, torch.zeros(SIZES[5], device=dev), hyper)   # generic path
        buf.publish(6, params[6], clear=True)
        LF.apply_update(params[0], params[0] * 0, params[0] * 0, params[0] * 1e-3, hyper, 3)
        host = flat.cpu().pin_memory()
        out = torch.empty_like(host).pin_memory()
        LF.ingest_sweep(buf, ms, host, hyper, 5, groups=3, results_to=out)
        torch.cuda.synchronize()
        assert buf.ledger.summary() is not None
        done.append(f"{dtype}: accumulate x3, sweep x3 variants, take/update/publish, apply_update, ingest")
        dp_kernels(buf, ms, hyper)
        done.append(f"{dtype}: DP kernels with self-peers")
    # swap tier
    from paper_2303_02868_b200.swap import HostMasterState, swap_sweep
    buf = LF.ParamBuffer(params, dtype="bf16", page_bytes=PAGE)
    hm = HostMasterState(params, page_bytes=PAGE, group_pages=2)
    buf.accumulate_flat(torch.ones(sum(SIZES), device=dev, dtype=torch.bfloat16), 0)
    swap_sweep(buf, hm, hyper)
    torch.cuda.synchronize()
    done.append("swap tier")
    # page pack / unpack / relocation
    dm = DevicePageManager([("GPU", 64 * PAGE, PAGE), ("CPU", 64 * PAGE, PAGE)], device=dev)
    from paper_2303_02868_b200.workloads import TensorSpec
    t = dm.allocate(TensorSpec("x", "param16", 3 * PAGE + 1234, 0), "GPU")
    data = torch.arange((3 * PAGE + 1234) // 2, device=dev, dtype=torch.int16).view(torch.float16)
    dm.write(t.tensor_id, data)
    assert torch.equal(dm.read(t.tensor_id).view(torch.int16), data.view(torch.int16))
    done.append("page pack/unpack")
    print("sanitize probe ok:", "; ".join(done), flush=True)


def dp_kernels(buf, ms, hyper):
    """The fused DP kernels with n_peers = 1 and the local pools as the
    'peer' (world-1 layout: every page is owned), compared with the sweep."""
    lib, eng = N.lib(), ms._eng
    lay = buf.layout
    L = buf.num_layers
    st = torch.cuda.current_stream()
    arr = lambda ptrs: (C.c_uint64 * len(ptrs))(*ptrs)
    check = lay.pool_chunks(range(L), "16", owned_only=True)
    adam = lay.adam_chunks(range(L), "pool", owned_only=True)
    flags = torch.zeros(L, dtype=torch.int32, device=buf.device)
    sumsq = torch.zeros(L, dtype=torch.float64, device=buf.device)
    merged = torch.zeros(L, dtype=torch.int32, device=buf.device)
    gpool = buf.g16_pool[0]
    for o in (D.opts(reduce_wide=1), D.opts(reduce_wide=0), D.opts(grid_ctas=5), D.opts(reduce_width=8)):
        D.check(lib.hm_dp_reduce_check(arr([D.ptr(gpool)]), 1, None, D.ptr(gpool), buf._dt,
                                       D.ptr(eng.desc.static(check)), len(check), D.ptr(flags),
                                       D.ptr(sumsq), o, D.sptr(st)))
    D.check(lib.hm_dp_flags_merge(arr([D.ptr(flags)]), arr([D.ptr(sumsq)]), 1, L, D.ptr(merged),
                                  D.ptr(sumsq), D.sptr(st)))
    rows = np.zeros(L, dtype=N.GROUP_LAUNCH)
    span = lay.elems16
    for l in range(L):
        rows[l] = (0, span, l, l)
    dgroups = eng.desc.table(rows, st)
    rt = eng.rt_scratch(L, st)
    bc, bc_len = ms._bias(hyper, range(L))
    hc = D.hyper_c(hyper)
    for o in (D.opts(ag_publish=0), D.opts(ag_publish=1), D.opts(grid_ctas=7)):
        D.check(lib.hm_adam_prologue(D.ptr(dgroups), L, D.ptr(rt), hc, D.ptr(bc), bc_len, 0, D.ptr(ms._steps),
                                     D.ptr(ms._applied), D.ptr(merged), None, 1, None, None, D.sptr(st)))
        D.check(lib.hm_adam_main_ag(D.ptr(eng.desc.static(adam)), len(adam), D.ptr(dgroups), D.ptr(rt),
                                    D.ptr(buf.g16_pool), buf._dt, D.ptr(ms.p32_pool), D.ptr(ms.m32_pool),
                                    D.ptr(ms.v32_pool), arr([D.ptr(buf.p16_pool)]), 1, None, buf._dt, hc,
                                    o, D.sptr(st)))
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
