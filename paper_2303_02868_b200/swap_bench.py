"""bench.py --config c3: GPT-3 13B page pools with the fp32 master state
off the GPU — pinned host memory (swap tier, ``--state-tier host``) or a
file on the SSD (``--state-tier ssd``) — lock-free update order preserved.

Host memory of the GPU box bounds the host-tier slice: the full 13B model
needs 154 GB of pinned fp32 state (12 B/param), so the default run takes the
first ``--c3-layers`` transformer layers plus the embeddings (every layer
has the same shape, so params/s is size-independent and the full-model step
time is the per-param time x 12.85e9, stated in the output).  Rooflines:
PCIe for the host tier (12 B/param fetched + 12 B/param stored, against
pinned cudaMemcpyAsync bandwidth measured in the same run); the drive for
the SSD tier (24 B/param of I/O against sequential O_DIRECT read/write
bandwidth measured on the same file system).
"""
from __future__ import annotations

import json
import os
import time
from collections.abc import Sequence

import torch


def measure_pcie(device, nbytes=1 << 30, reps=5):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=device)
    s1, s2 = torch.cuda.Stream(device), torch.cuda.Stream(device)

    def timed(fn):
        best = float("inf")
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    def h2d():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h.copy_(d, non_blocking=True)

    d2 = torch.empty_like(d)
    h2 = torch.empty_like(h).pin_memory()

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    t_h2d, t_d2h, t_both = timed(h2d), timed(d2h), timed(both)
    return {"h2d_gbs": nbytes / t_h2d / 1e9, "d2h_gbs": nbytes / t_d2h / 1e9,
            "bidir_gbs": 2 * nbytes / t_both / 1e9}


def measure_drive(path: str, nbytes: int = 2 << 30, block: int = 64 << 20):
    """Sequential write then read of ``nbytes`` with O_DIRECT (when allowed)
    from pinned memory, 4 threads, like the tier's own I/O."""
    from concurrent.futures import ThreadPoolExecutor
    from .ssd import _open
    fd, direct = _open(path, True)
    os.ftruncate(fd, nbytes)
    bufs = [torch.zeros(block, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
    views = [memoryview(b.numpy()) for b in bufs]

    def run(write):
        def one(i):
            mv = views[i % 4]
            (os.pwritev if write else os.preadv)(fd, [mv], i * block)
        t0 = time.perf_counter()
        with ThreadPoolExecutor(4) as ex:
            list(ex.map(one, range(nbytes // block)))
        if write:
            os.fsync(fd)
        return nbytes / (time.perf_counter() - t0) / 1e9

    w = run(True)
    r = run(False)
    os.close(fd)
    os.unlink(path)
    return {"write_gbs": w, "read_gbs": r, "o_direct": direct,
            "path": os.path.dirname(os.path.abspath(path))}


class LazyParams(Sequence):
    """Per-layer random f32 parameters generated on the device on demand (one
    layer alive at a time): the 13B model's 51 GB of initial fp32 values
    never sit in host memory next to its 154 GB of pinned state."""

    def __init__(self, numels, device, seed: int = 1234):
        self.numels, self.device, self.seed = list(numels), device, seed

    def __len__(self):
        return len(self.numels)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        g = torch.Generator(device=self.device)
        g.manual_seed(self.seed * 1_000_003 + i)
        return torch.empty(self.numels[i], dtype=torch.float32, device=self.device).normal_(0, 0.02, generator=g)


def fit_layers(requested: int, world: int) -> tuple[int, dict]:
    """Transformer layers of C3 whose pinned fp32 state (12 B/param, split over
    the ranks of this box) fits the box's host memory, at most 40."""
    from . import workloads as W
    per_layer = W.total_elems(W.gpt_param16(W.GPTShape(2048, 5120, 20480, 1), embeddings=False))
    emb = W.total_elems(W.gpt_param16(W.GPTShape(2048, 5120, 20480, 0), embeddings=True))
    avail = 0
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    avail = int(line.split()[1]) * 1024
    except OSError:
        pass
    budget = avail - (12 << 30) - world * (6 << 30)   # OS + per-rank process, CUDA context, transients
    fit = max(1, min(40, int((budget - 12 * emb) // (12 * per_layer)))) if avail else 8
    layers = fit if requested <= 0 else min(requested, 40)
    return layers, {"mem_available_gb": avail / 1e9, "state_budget_gb": budget / 1e9, "layers_that_fit": fit}


def run(args, metric, bytes_per_param, ClockSampler, load_peaks):
    from . import lockfree as LF
    from . import workloads as W
    from .layout import PageLayout
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        from .dp_bench import _init, _max_over_ranks
        rank, world, device = _init()
    else:
        rank, device = 0, torch.device("cuda", 0)
        torch.cuda.set_device(device)
    from . import _device as Dv
    numa = Dv.bind_to_gpu_numa(device.index)
    layers, mem = fit_layers(args.c3_layers, world)
    shape = W.GPTShape(2048, 5120, 20480, layers)
    specs = W.gpt_param16(shape)
    full_params = W.total_elems(W.config_specs("c3"))
    page = args.page_mib * 2**20 if args.page_mib else W.config_page_bytes("c3")
    numels = [s.bytes // 2 for s in specs]
    layout = PageLayout(numels, page, world_size=world, rank=rank, names=[s.name for s in specs])
    params = LazyParams(numels, device)
    pool_alloc = None
    if world > 1:
        from .sharding import symmetric_alloc
        pool_alloc = symmetric_alloc
    buf = LF.ParamBuffer(params, dtype=args.dtype, page_bytes=page, device=device, layout=layout,
                         pool_alloc=pool_alloc)
    t0 = time.perf_counter()
    ssd_path = None
    if args.state_tier == "ssd":
        from .ssd import SSDMasterState, ssd_sweep as sweep_fn
        ssd_path = os.path.join(args.ssd_dir, f"hm_state_{os.getpid()}.bin")
        hm = SSDMasterState(params, ssd_path, page_bytes=page, device=device, layout=layout,
                            group_pages=args.swap_group_pages, slots=max(3, args.swap_slots),
                            world_size=world, rank=rank)
    else:
        from .swap import HostMasterState, swap_sweep as sweep_fn
        hm = HostMasterState(params, page_bytes=page, device=device, layout=layout,
                             group_pages=args.swap_group_pages, slots=args.swap_slots,
                             world_size=world, rank=rank)
    init_s = time.perf_counter() - t0
    del params
    torch.cuda.empty_cache()
    P = sum(numels)
    owned = layout.owned_numel()
    hyper = LF.AdamHyper(lr=1e-3, inv_scale=1.0 / world)
    if world > 1:
        from .dp_bench import owned_grad_flat
        from .sharding import FusedShardedPageStep
        grads = owned_grad_flat(layout, args.dtype, device, 7 + rank)
        dp = FusedShardedPageStep(buf, hm)
        step = lambda: dp.step(hyper)
    else:
        gen = torch.Generator(device=device)
        gen.manual_seed(7)
        tdt = torch.bfloat16 if args.dtype == "bf16" else torch.float16
        grads = torch.empty(P, dtype=tdt, device=device)
        for a in range(0, P, 1 << 28):   # in slices: no 51 GB f32 temporary
            b = min(P, a + (1 << 28))
            grads[a:b] = torch.empty(b - a, device=device).normal_(0, 1e-2, generator=gen).to(tdt)
        step = lambda: sweep_fn(buf, hm, hyper)
    for rnd in range(2):
        buf.accumulate_flat(grads, rnd)
        if rnd == 0:
            step()
    L = len(specs)

    def rearm():
        for l in range(L):
            buf._pending[l] = 1

    for _ in range(args.warmup):
        rearm()
        step()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    stream = torch.cuda.current_stream(device)
    with ClockSampler(device.index) as clk:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t_wall = time.perf_counter()
        a.record(stream)
        for _ in range(args.steps):
            rearm()
            step()
        b.record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    # the SSD sweep blocks on host I/O, so its step time is the wall clock
    ms_step = (t_wall * 1e3 if args.state_tier == "ssd" else a.elapsed_time(b)) / args.steps
    if world > 1:
        ms_step = _max_over_ranks(ms_step)
    moved = 24 * owned  # 12 B fetched + 12 B stored per owned param, per rank
    achieved = moved / (ms_step / 1e3) / 1e9
    if args.state_tier == "ssd":
        hm.close()
        os.unlink(ssd_path)
        drive = measure_drive(os.path.join(args.ssd_dir, f"hm_probe_{os.getpid()}.bin"))
        peak = 1.0 / (0.5 / drive["read_gbs"] + 0.5 / drive["write_gbs"])  # 12 B read + 12 B write
        roof = {"bound": "ssd", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_kind": "measured sequential pread/pwrite (harmonic mean of read and write) "
                             "on the same file system", "bytes_per_param": 24, "drive": drive}
    else:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()   # every rank measures at once: the host memory is shared
        pcie = measure_pcie(device)
        peak = pcie["bidir_gbs"] if world == 1 else _min_over_ranks(pcie["bidir_gbs"])
        roof = {"bound": "pcie", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_kind": "measured pinned cudaMemcpyAsync H2D||D2H on this box" +
                (", all ranks at once, slowest rank" if world > 1 else ""),
                "bytes_per_param": 24, "per": "rank (its owned pages over its own PCIe link)", "pcie": pcie}
    lockfree = None
    if args.state_tier == "host" and args.c3_lockfree_iters > 0:
        upd = (lambda b, m, h, stream: dp.step(h, stream=stream)) if world > 1 else None
        lockfree = _lockfree(args, buf, hm, hyper, grads, P, device, update=upd)
        if world > 1:
            for k in ("sync_iter_ms", "lockfree_iter_ms"):
                lockfree[k] = _max_over_ranks(lockfree[k])
            lockfree["speedup"] = lockfree["sync_iter_ms"] / lockfree["lockfree_iter_ms"]
    line = {
        "metric": metric, "value": P / (ms_step / 1e3), "unit": "params/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": f"c3: GPT-3 13B page pools, {layers} of 40 layers + embeddings; fp32 state "
                               f"on the {args.state_tier} tier" + (", page-sharded over ranks" if world > 1 else ""),
                   "params": P, "full_model_params": full_params, "layers": L, "page_bytes": page,
                   "pages": layout.used_pages, "group_pages": args.swap_group_pages,
                   "staging_slots": args.swap_slots, "state_gb": 12 * P / 1e9,
                   "state_gb_per_rank": 12 * owned / 1e9, "parallelism": f"dp{world}" if world > 1 else "single GPU",
                   "host_memory": mem, "init_s": init_s,
                   "full_model_step_ms_extrapolated": ms_step * full_params / P,
                   "step": "swap sweep: per page group H2D -> page-Adam -> D2H" if world == 1 else
                           "DP step: fused reduce-scatter -> prologue -> per owned page group H2D -> "
                           "page-Adam with all-gather epilogue -> D2H"},
        "roofline": roof,
        "clocks": clk.summary(),
        # prologue + one page-Adam per page group (+ reduce-scatter and flag merge at N > 1)
        "gpu_launches": args.steps * (1 + hm.num_groups + (2 if world > 1 else 0)),
    }
    if lockfree:
        line["lockfree"] = lockfree
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def _min_over_ranks(x: float) -> float:
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return float(t.item())


def _lockfree(args, buf, hm, hyper, grads, P, device, update=None):
    """C3's "lock-free delayed update" (Algorithm 2) on the
    same pools: actors.LockFreeRunner with the host-tier sweep (or, at N > 1,
    the DP page step over the sharded host tier) as the updating actor and,
    as the GPU actor, the slice's forward+backward
    modelled as a spin of 6 x params x tokens / (measured bf16 peak x MFU) —
    the update path is the product here, not the model.  delay=0 is the
    synchronous loop (update, then the next compute); delay=1 overlaps the
    update of step k with the compute of step k+1 (staleness <= 1)."""
    from pathlib import Path
    from . import _device as Dv
    from . import _native as Nn
    from .actors import LockFreeRunner
    peaks = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    bf16 = json.loads(peaks.read_text()).get("bf16_tflops_sustained", 1369.5) if peaks.exists() else 1369.5
    tokens, mfu = args.c3_tokens, 0.5
    tc_ms = 6.0 * P * tokens / (bf16 * 1e12 * mfu) * 1e3
    zero = torch.zeros((), device=device)

    def grads_fn(params, it):
        Dv.check(Nn.lib().hm_spin(int(tc_ms * 1e6), Dv.sptr(torch.cuda.current_stream(device))))
        return zero, grads

    out = {"gpu_actor": f"spin of 6 x {P} params x {tokens} tokens / ({bf16} TF/s x MFU {mfu})",
           "compute_ms": tc_ms, "iters": args.c3_lockfree_iters,
           "updating_actor": "swap sweep" if update is None else "DP page step with the host-tier state"}
    for delay, name in ((0, "sync"), (1, "lockfree")):
        runner = LockFreeRunner(buf, hm, hyper, delay=delay, update=update)
        runner.run(1, grads_fn, mode=name)                     # warm-up iteration
        rep = runner.run(args.c3_lockfree_iters, grads_fn, mode=name)
        out[f"{name}_iter_ms"] = rep.iter_ms
        out[f"{name}_max_staleness"] = rep.max_staleness
    out["speedup"] = out["sync_iter_ms"] / out["lockfree_iter_ms"]
    return out
