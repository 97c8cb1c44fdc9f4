"""bench.py's N>1 arm: the data-parallel page step under torchrun (one
process per GPU over NVLink/NVSwitch).

Default (``--dp-mode p2p``): sharding.FusedShardedPageStep — reduce-scatter
of the 16-bit gradient pages fused with the finite/norm check over peer
memory -> flag merge -> prologue -> page-Adam whose publish epilogue writes
every peer's pool (the all-gather); at N=2 pipelined over layer groups
(``--dp-groups -1`` = the measured policy).  ``--dp-mode nccl``:
sharding.ShardedPageStep (NCCL RS, check, flag all-reduce, page-Adam per
bucket with the AG of bucket b overlapped with Adam of bucket b+1).
``value`` = params of the whole model updated per second (strong scaling:
the model is fixed, each rank updates 1/N of its pages); RS/AG bus
bandwidths are reported beside it, busbw = (S/t)(N-1)/N with S = 2 B x
params (the algorithmic payload).

Synthetic gradients: each rank holds non-zero gradients only in the pages it
owns, so the in-place reduce-scatter returns every owner its own values and
re-offering the same pages every step keeps them bounded (no growth across
timed steps); the collective still moves the whole pool.
"""
from __future__ import annotations

import json
import os
import sys
import time

import torch
import torch.distributed as dist


def _init():
    if not dist.is_initialized():
        from datetime import timedelta
        # a mismatched collective fails in minutes instead of hanging the box
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))),
                                timeout=timedelta(seconds=int(os.environ.get("HM_DIST_TIMEOUT_S", "300"))))
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    return rank, world, torch.device("cuda", local)


def owned_grad_flat(layout, dtype, device, seed):
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float16
    total = sum(layout.numels)
    flat = torch.zeros(total, dtype=tdt, device=device)
    base = 0
    for l, n in enumerate(layout.numels):
        for s in layout.segments[l]:
            if layout.owned(s):
                flat[base + s.pos: base + s.pos + s.n] = torch.empty(
                    s.n, device=device).normal_(0, 1e-2, generator=gen).to(tdt)
        base += n
    return flat


def _max_over_ranks(x: float) -> float:
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run(args, metric, bytes_per_param, ClockSampler, load_peaks, build_state):
    from . import lockfree as LF
    from . import workloads as W
    from .sharding import FusedShardedPageStep, ShardedPageStep, symmetric_alloc
    rank, world, device = _init()
    from . import _device as Dv
    numa = Dv.bind_to_gpu_numa(device.index)   # this rank's pinned buffers next to its GPU
    fused = args.dp_mode != "nccl"
    fallback = None
    if fused:
        try:   # symmetric (peer-mapped) pools; every rank must agree on the outcome
            if args.dp_onepass < 0:   # auto: measured policy (profiles/r2_bench.md)
                # N=2: one kernel beats the layer-group pipeline (4.04 vs 4.87 ms, C2);
                # N>=4 the step is link-bound and the two-phase kernels move the
                # bytes more efficiently (5.80 vs 5.98 ms)
                args.dp_onepass = 1 if world == 2 and args.dp_mode == "p2p" else 0
            specs, page, layout, buf, ms = build_state(args, device, world, rank,
                                                       pool_alloc=symmetric_alloc,
                                                       double_buffered=bool(args.dp_onepass))
            if args.dp_push < 0:
                args.dp_push = 0
            dp = FusedShardedPageStep(buf, ms, mode=args.dp_mode,
                                      push=bool(args.dp_push) and bool(args.dp_onepass))
            ok = torch.ones(1, device=device)
        except Exception as e:  # e.g. no peer mapping / multicast on this system
            fallback = f"{type(e).__name__}: {e}"[:200]
            ok = torch.zeros(1, device=device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 0:
            fallback = fallback or "a peer rank could not map symmetric memory"
            fused = False
            buf = ms = dp = None
            torch.cuda.empty_cache()
            if rank == 0:
                print(f"[bench] fused DP path unavailable ({fallback}); using NCCL", file=sys.stderr)
    if not fused:
        specs, page, layout, buf, ms = build_state(args, device, world, rank)
        dp = ShardedPageStep(buf, ms)
    L = len(specs)
    P = sum(layout.numels)
    hyper = LF.AdamHyper(lr=1e-3, inv_scale=1.0 / world)
    knobs = {"ag_publish": args.ag_publish, "reduce_wide": args.dp_reduce_wide} if fused else {}
    if args.dp_groups < 0:   # auto: measured policy (profiles/r1_dp_c2.md)
        # pipelining pays at N=2 once the per-group barriers are small next to
        # the transfer (C2/C4/C5, >= 1 GB of 16-bit pages), not for C1 (0.25 GB)
        big = 2 * P >= 1e9
        args.dp_groups, args.dp_reduce_ctas = (8, 128) if world == 2 and big else (1, 0)
    if fused and dp.one_pass:
        args.dp_groups = 1      # the one-pass kernel overlaps the exchange with the update itself
        knobs = {}
    pipelined = fused and args.dp_groups > 1

    def do_step(**kw):   # launch settings travel with each launch (hm_launch_opts)
        if pipelined:
            return dp.step_pipelined(hyper, args.dp_groups, reduce_ctas=args.dp_reduce_ctas,
                                     update_ctas=args.dp_update_ctas, reduce_sms=args.dp_reduce_sms,
                                     **knobs, **kw)
        return dp.step(hyper, **knobs, **kw)
    flat = owned_grad_flat(layout, args.dtype, device, 7 + rank)
    for rnd in range(2):  # fill both gradient page buffers (K3)
        buf.accumulate_flat(flat, rnd)
        if rnd == 0:
            do_step()

    def rearm():
        for l in range(L):
            buf._pending[l] = 1

    stream = torch.cuda.current_stream(device)
    for _ in range(args.warmup):
        rearm()
        do_step()
    torch.cuda.synchronize()
    dist.barrier()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", rank))) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            rearm()
            do_step()
        t1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    step_ms = _max_over_ranks(t0.elapsed_time(t1) / args.steps)

    # Phase timings from ONE unpipelined instrumented step (the pipelined
    # headline overlaps the phases, so its marks cannot be split honestly).
    rearm()
    dp.step(hyper, **knobs)    # first use of the unpipelined plan uploads its descriptors
    rearm()
    tm = {}
    dp.step(hyper, timings=tm, **knobs)
    torch.cuda.synchronize()
    mk = tm["_marks"]
    if fused:
        parts = {"barrier_ms": mk["start"].elapsed_time(mk["rs_start"]),
                 "rs_ms": mk["rs_start"].elapsed_time(mk["rs"]),
                 "check_ms": mk["rs"].elapsed_time(mk["check"]),
                 "update_ag_ms": mk["check"].elapsed_time(mk["adam"]),
                 "ag_tail_ms": mk["adam"].elapsed_time(mk["ag"]),
                 "step_ms": mk["start"].elapsed_time(mk["ag"])}
    else:
        parts = {"rs_ms": mk["start"].elapsed_time(mk["rs"]), "check_ms": mk["rs"].elapsed_time(mk["check"]),
                 "update_ms": mk["check"].elapsed_time(mk["adam"]), "ag_tail_ms": mk["adam"].elapsed_time(mk["ag"]),
                 "step_ms": mk["start"].elapsed_time(mk["ag"])}
    parts = {k: _max_over_ranks(v) for k, v in parts.items()}
    gpool = buf.g16_pool[buf._gsel[0] ^ 1]
    ppool = buf.p16_pool[buf._psel[0]]
    reps = 10

    def timed(fn):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return _max_over_ranks(a.elapsed_time(b) / reps)

    S = 2 * P                                  # the algorithmic 16-bit payload
    busbw = lambda ms_: S / (ms_ / 1e3) * (world - 1) / world / 1e9
    if fused and dp.one_pass:
        phases = {"onepass_ms": parts["update_ag_ms"], "rs_and_ag_busbw_gbs": 2 * busbw(parts["update_ag_ms"]),
                  "note": "one unpipelined instrumented step: the reduce-scatter, the update and the "
                          "all-gather are ONE kernel (plus the flag merge / commit); the busbw counts both "
                          "exchanges over its time"}
    elif fused:
        phases = {"rs_ms": parts["rs_ms"], "rs_busbw_gbs": busbw(parts["rs_ms"]),
                  "update_ag_ms": parts["update_ag_ms"],
                  "ag_busbw_gbs": busbw(parts["update_ag_ms"]),
                  "note": "one unpipelined instrumented step: rs = the reduce-scatter+check kernel; "
                          "ag = the page-Adam kernel whose epilogue stores into every peer (the update's "
                          "HBM time is inside it)"}
    else:
        rs_ms = timed(lambda: dp.coll.reduce_scatter(gpool))
        ag_ms = timed(lambda: dp.coll.all_gather(ppool))
        phases = {"rs_ms": rs_ms, "rs_busbw_gbs": busbw(rs_ms), "ag_ms": ag_ms, "ag_busbw_gbs": busbw(ag_ms),
                  "note": "NCCL collectives timed alone"}
    link = measure_nvlink(device, world, rank)
    pipe = None
    if fused and dp.one_pass:   # the one-pass kernel group by group as the gradient lands
        pipe = lambda ready, res: dp.step(hyper, ready=ready)
    elif fused:
        pipe = lambda ready, res: dp.step_pipelined(hyper, args.e2e_groups, reduce_ctas=args.dp_reduce_ctas,
                                                    ready=ready, results_to=res, **knobs)
    e2e = run_e2e(args, buf, ms, do_step, flat, layout, pipe,
                  with_results=not (fused and dp.one_pass)) if args.e2e_steps > 0 else None
    # Link-level bytes per direction per GPU for the step: P2P (and NCCL)
    # move (N-1)/N*S in for the reduce-scatter and (N-1)/N*S in for the
    # all-gather (the same out); NVLS reads the reduced S/N from the switch
    # and receives the multicast (N-1)/N*S, so S per direction.
    nvls = fused and args.dp_mode == "nvls"
    link_bytes = S if nvls else 2 * S * (world - 1) / world
    peak = link["ingress_gbs"]
    achieved = link_bytes / (step_ms / 1e3) / 1e9
    owned = layout.owned_numel()
    peak_hbm, peak_kind = load_peaks()
    upd_ms = parts["update_ag_ms"] if fused else parts["update_ms"]
    line = {
        "metric": metric, "value": P / (step_ms / 1e3), "unit": "params/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {W.CONFIGS[args.config][2]}", "params": P, "layers": L,
                   "page_bytes": page, "pages": layout.used_pages, "grad_dtype": args.dtype,
                   "parallelism": f"dp{world}", "l2": "inputs larger than L2 (28 B/param x params >> 126 MB)",
                   "step": "take -> update -> publish of every layer's pages (one updating-actor sweep)"},
        "run": {"bucket_pages_per_rank": layout.K, "buckets": layout.num_buckets,
                "sharding": "page-sharded ZeRO-3 (owner = page % N)",
                "numa_bind": {k: v for k, v in numa.items() if k != "_before"} if numa else None,
                "dp_mode": (args.dp_mode + (" one-pass" if fused and dp.one_pass else "")
                            + (" push" if fused and getattr(dp, "push", False) else "")) if fallback is None
                           else f"nccl (fallback: {fallback})",
                "dp_groups": args.dp_groups if pipelined else 1,
                "dp_reduce_ctas": args.dp_reduce_ctas if pipelined else 0,
                "dp_update_ctas": args.dp_update_ctas if pipelined else 0,
                "dp_reduce_sms": args.dp_reduce_sms if pipelined else 0,
                "ag_publish": ["per-thread stores", "bulk", "bulk"][args.ag_publish],
                "kernels": ("RS(grad pages) -> check -> flag all-reduce -> prologue -> "
                            "page-Adam(bucket) || AG(bucket)") if not fused else
                           ("barrier -> speculative prologue -> ONE kernel: pull every rank's gradient "
                            "page + f32 reduce + page-Adam into the other state copy + store to every "
                            "rank -> barrier -> flag merge/commit -> republish rejected -> barrier")
                           if dp.one_pass else
                           ("barrier -> fused reduce-scatter+check over peer memory -> barrier -> "
                            "flag merge -> prologue -> page-Adam with all-gather epilogue -> barrier")},
        "roofline": {"bound": "nvlink", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "peak_kind": "measured on this box: " + link["how"],
                     "bytes_per_step": link_bytes,
                     "bytes_rule": ("S per direction per GPU (NVLS: reduced S/N from the switch + the "
                                    "multicast (N-1)/N*S)") if nvls else
                                   "2(N-1)/N * S per direction per GPU (RS in + AG in), S = 2 B x params",
                     "link_bound_ms": link_bytes / peak / 1e6,
                     "kernel": "whole DP step (reduce-scatter, update, all-gather)"},
        "hbm": {"update_kernel_ms": upd_ms, "owned_params": owned,
                "gbs": 28 * owned / (upd_ms / 1e3) / 1e9 if upd_ms > 0 else None, "peak": peak_hbm,
                "peak_kind": peak_kind, "note": "owned-page update of the unpipelined instrumented step (the "
                                                "fused kernel also pushes the all-gather over NVLink)"},
        "nvlink": dict(phases, peak_gbs=peak, nominal_gbs=900.0, link=link, algorithmic_bytes=S,
                       pool_bytes_padded=layout.elems16 * 2),
        "components_ms": parts,
        "reference_model": _reference_model(layout, page, world),
        "clocks": clk.summary(),
        "gpu_launches": args.steps * ((2 + layout.num_buckets) if not fused else
                                     4 * (args.dp_groups if pipelined else 1)),
    }
    if e2e:
        line["e2e"] = e2e
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def measure_nvlink(device, world, rank, nbytes: int = 1 << 29, reps: int = 5) -> dict:
    """Per-GPU NVLink ingress measured on this box: every rank pulls a
    ``nbytes`` block from each peer in turn (copy-engine peer reads of a
    symmetric buffer, peers visited in rank-rotated order), all ranks at
    once — the traffic pattern of the reduce-scatter / all-gather.  Also the
    one-pair, one-direction copy for context."""
    import torch.distributed._symmetric_memory as symm
    buf = symm.empty(nbytes, dtype=torch.uint8, device=device)
    h = symm.rendezvous(buf, dist.group.WORLD.group_name)
    dst = torch.empty(nbytes, dtype=torch.uint8, device=device)
    peers = [h.get_buffer((rank + k) % world, (nbytes,), torch.uint8) for k in range(1, world)]
    st = torch.cuda.current_stream(device)

    def pull(which, active=True):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps if active else 0):
            for pv in which:
                dst.copy_(pv)
        b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps
    pull(peers)   # warm
    t_all = _max_over_ranks(pull(peers))
    # one pair, one direction: rank 0 pulls from rank 1 while the others idle
    # (every rank still takes part in the barrier and the reduction)
    t_pair = _max_over_ranks(pull(peers[:1], active=(rank == 0)))
    pair = nbytes / (t_pair / 1e3) / 1e9
    ingress = (world - 1) * nbytes / (t_all / 1e3) / 1e9
    return {"ingress_gbs": ingress, "pair_gbs": pair,
            "how": f"copy-engine peer reads, every rank pulling {nbytes >> 20} MiB from each peer at once, "
                   "slowest rank"}


def run_e2e(args, buf, ms, do_step, flat, layout, pipe=None, with_results=True):
    """The DP step through the public API with host buffers, per rank: H2D of
    this rank's whole 16-bit gradient from pinned memory + K3 accumulate, the
    sharded page step, and a D2H read of the per-layer applied flags.  Time =
    max over ranks of the wall time between synchronised barriers.

    serial:    ``ParamBuffer.accumulate_flat(host)`` then the step;
    pipelined: ``lockfree.ingest`` (per layer group: H2D -> K3, one event per
               group) feeding ``step_pipelined(ready=...)``, so the reduce,
               update and all-gather of group k run while group k+1 is still
               crossing PCIe (fused mode only).  The headline is the faster."""
    from . import lockfree as LF
    host = flat.cpu().pin_memory()
    out = torch.empty_like(host).pin_memory()
    h2d = host.numel() * host.element_size()
    d2h = 2 * layout.owned_numel()      # this rank's published pages

    def serial(it):
        buf.accumulate_flat(host, it)      # H2D (non_blocking from pinned) + K3
        do_step()
        return ms._applied.cpu()           # D2H of the step's result

    def pipelined(it, results=False):
        ready = LF.ingest(buf, host, it, groups=args.e2e_groups)
        pipe(ready, out if results else None)
        return ms._applied.cpu()

    def timed(step):
        for it in range(2):
            step(it)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for it in range(args.e2e_steps):
            step(it)
        torch.cuda.synchronize()
        return _max_over_ranks((time.perf_counter() - t0) / args.e2e_steps)

    dt_serial = timed(serial)
    dt_pipe = timed(pipelined) if pipe is not None else None
    dt_res = timed(lambda it: pipelined(it, True)) if pipe is not None and with_results else None
    dt = min(dt_serial, dt_pipe) if dt_pipe else dt_serial
    piped = bool(dt_pipe and dt_pipe <= dt_serial)
    P = sum(layout.numels)
    return {"value": P / dt, "unit": "params/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": 4 * len(layout.numels), "ms_per_step": dt * 1e3,
            "steps": args.e2e_steps, "h2d_gbs_per_rank": h2d / dt / 1e9,
            "serial_ms_per_step": dt_serial * 1e3,
            "pipelined_ms_per_step": dt_pipe * 1e3 if dt_pipe else None,
            "with_results": None if dt_res is None else {
                "ms_per_step": dt_res * 1e3, "params_per_s": P / dt_res, "d2h_bytes_per_step": d2h,
                "note": "step_pipelined(results_to=...): every rank also returns its owned published pages "
                        "(per rank, disjoint: the whole model once per step); the ranks share the host's "
                        "PCIe/memory bandwidth"},
            "api": ("lockfree.ingest(pinned host gradient, %d layer groups) -> FusedShardedPageStep.%s"
                    "(ready=...) -> applied flags to host, every rank"
                    % (args.e2e_groups, "step" if not with_results else "step_pipelined")) if piped else
                   "ParamBuffer.accumulate_flat(pinned host gradient) + sharded page step + "
                   "applied flags to host, every rank"}


def _reference_model(layout, page, world):
    """The reference simulator's view of the same exchange (per-page gather
    tasks on one interconnect resource, hiermem/simengine.py:255-257) with the
    measured B200 link of presets/b200-server.json — printed next to the
    measured step so the model can be checked."""
    from pathlib import Path
    from .sharding import modeled_gather_s
    preset = Path(__file__).resolve().parent.parent / "presets" / "b200-server.json"
    try:
        link = json.loads(preset.read_text())["links"]["gpu_interconnect"]
    except (OSError, KeyError, ValueError):
        return None
    ag = modeled_gather_s(page, layout.used_pages, world, link["bandwidth_bytes_per_s"], link["latency_s"])
    return {"preset": "presets/b200-server.json", "ag_ms": ag * 1e3, "rs_ms": ag * 1e3,
            "comm_ms": 2 * ag * 1e3, "formula": "pages x (lat + page (N-1)/N / bw) per collective"}
