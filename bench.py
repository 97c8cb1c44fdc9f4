"""Benchmark of the page-granular update hot path (BASELINE.json metric:
"page-Adam params/s + HBM GB/s; page RS/AG bus GB/s at 1/2/4/8 B200").

One *step* = one fused page sweep of the updating actor over every layer of
the workload (hiermem/lockfree.py:624-639: take -> update_layer ->
publish), i.e. prologue + page-Adam over all param pages: 28 B/param of HBM
traffic.  At N>1 a step is the data-parallel page step: gradient
reduce-scatter over the page pool, the sharded sweep, parameter all-gather.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--dtype bf16]
    python bench.py --impl reference ...     # the reference CPU path (oracle port)

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BYTES_PER_PARAM = 28  # read g16 2 + p/m/v 12; write p/m/v 12 + p16 2
METRIC = "page-Adam params/s + HBM GB/s; page RS/AG bus GB/s at 1/2/4/8 B200"


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


# ---- clocks sampling during the timed region -------------------------------------
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index: int = 0, period_ms: int = 20):
        self.index, self.period_ms = index, period_ms
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", f"-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.15)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                bits = int(parts[2], 16) if parts[2].startswith("0x") else int(parts[2])
            except ValueError:
                continue
            sm.append(s)
            mx = m
            for b, name in REASON_BITS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---- CPU baseline: the reference itself (baseline/_ref) or its oracle port --------

def import_reference():
    """hiermem from baseline/_ref (the unmodified reference, pip-installed
    there; git-ignored, shipped to the GPU box with the snapshot), or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "hiermem").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import hiermem.lockfree as lf
        return lf
    except Exception:
        return None


class CpuReferenceSample:
    """The reference's update chain over the first ``sample_pages`` pages'
    worth of parameters of the workload, cut into ``threads`` layers that
    ``threads`` host threads update concurrently (numpy ufuncs release the
    GIL).  With the reference installed (baseline/_ref) each layer runs the
    reference's OWN public calls — ``ParamBuffer.take`` -> ``MasterState.
    update_layer`` -> ``ParamBuffer.publish(clear=False)`` (hiermem/lockfree.py:
    624-639), fp16 gradients (its only 16-bit type), one ``accumulate`` per
    layer before each timed pass (the producer, untimed like the GPU arm's
    resident gradients); otherwise the same chain restated op for op in numpy
    (oracle/page_adam.py, pinned bit-exact to it).  ``run()`` times one pass."""

    def __init__(self, page_bytes: int, sample_pages: int, threads: int, dtype: str):
        from concurrent.futures import ThreadPoolExecutor
        self.n = sample_pages * (page_bytes // 2)
        pieces = np.array_split(np.arange(self.n), threads)
        self.bounds = [(int(a[0]), int(a[-1]) + 1) for a in pieces if len(a)]
        self.pool = ThreadPoolExecutor(max_workers=threads)
        self.lf = import_reference()
        rng = np.random.default_rng(0)
        if self.lf is not None:
            self.kind, self.dtype = "reference", "fp16"
            params = [rng.normal(0, 0.02, hi - lo).astype(np.float32) for lo, hi in self.bounds]
            self.grads = [rng.normal(0, 1e-2, hi - lo).astype(np.float16) for lo, hi in self.bounds]
            self.buf, self.ms = self.lf.ParamBuffer(params), self.lf.MasterState(params)
            self.hyper = self.lf.AdamHyper(lr=1e-3)
            self.it = 0
        else:
            from oracle import page_adam as O
            self.O, self.kind, self.dtype = O, "port", dtype
            self.p, self.m, self.v, self.g16 = O.synthetic_layer(0, 0, self.n, dtype, outliers=False)

    def describe(self) -> str:
        if self.kind == "reference":
            return (f"{self.n} params (first pages of the pool) as {len(self.bounds)} layers, one host thread "
                    "each, running hiermem's own ParamBuffer.take -> MasterState.update_layer -> "
                    "ParamBuffer.publish(clear=False) (baseline/_ref, hiermem/lockfree.py:624-639), fp16 "
                    "gradients; the accumulate before each pass is untimed")
        return (f"{self.n} params (first pages of the pool), {len(self.bounds)} threads; "
                "take->apply_update->publish restated op-for-op in numpy (oracle/page_adam.py, bit-exact "
                "to hiermem/lockfree.py:127-263)")

    def _arm(self, l):
        self.buf.accumulate(self.lf.GradMessage(l, self.grads[l], self.it))

    def _chain(self, l):
        g, _count, newest = self.buf.take(l)
        self.ms.update_layer(l, g, self.hyper)
        self.buf.publish(l, self.ms.p32[l], applied_iter=newest, clear=False)

    def _port(self, b):
        O, lo, hi = self.O, b[0], b[1]
        g = O.from16(self.g16[lo:hi], self.dtype)                                    # take (widen)
        pp, mm, vv, ok = O.adam_update(self.p[lo:hi], self.m[lo:hi], self.v[lo:hi], g,
                                       1e-3, 0.9, 0.999, 1e-8, 10)                   # apply_update
        O.publish16(pp, self.dtype)                                                  # publish cast
        return ok

    def run(self) -> float:
        if self.kind == "reference":
            L = range(len(self.bounds))
            list(self.pool.map(self._arm, L))
            self.it += 1
            t0 = time.perf_counter()
            list(self.pool.map(self._chain, L))
            return time.perf_counter() - t0
        t0 = time.perf_counter()
        list(self.pool.map(self._port, self.bounds))
        return time.perf_counter() - t0

    def close(self):
        self.pool.shutdown()


def cpu_reference_sample(page_bytes, sample_pages: int, threads: int, dtype: str,
                         min_seconds: float = 10.0, min_reps: int = 2):
    """Passes over the bounded sample until ``min_seconds`` of CPU work (and
    at least ``min_reps`` passes) have run; returns (sample, median pass time,
    passes)."""
    s = CpuReferenceSample(page_bytes, sample_pages, threads, dtype)
    s.run()  # warm
    times = []
    while len(times) < min_reps or sum(times) < min_seconds:
        times.append(s.run())
    s.close()
    return s, statistics.median(times), len(times)


def gpu_config(args, specs, page, layout):
    """The config dict both arms print: the same keys and values (the driver
    compares them); arm-specific settings go to the line's "run" key."""
    from paper_2303_02868_b200 import workloads as W
    return {"workload": f"{args.config}: {W.CONFIGS[args.config][2]}", "params": W.total_elems(specs),
            "layers": len(specs), "page_bytes": page, "pages": layout.used_pages,
            "grad_dtype": args.dtype, "parallelism": f"dp{args.gpus}" if args.gpus > 1 else "single GPU",
            "l2": "inputs larger than L2 (28 B/param x params >> 126 MB)",
            "step": "take -> update -> publish of every layer's pages (one updating-actor sweep)"}


def run_reference(args):
    """--impl reference: the reference's CPU update path on the host cores."""
    from paper_2303_02868_b200 import workloads as W
    from paper_2303_02868_b200.layout import PageLayout
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    specs = W.config_specs(args.config)
    page = args.page_mib * 2**20 if args.page_mib else W.config_page_bytes(args.config)
    threads = os.cpu_count() or 1
    sample_pages = max(1, min(args.cpu_sample_pages, sum(s.bytes for s in specs) // page))
    sample = CpuReferenceSample(page, sample_pages, threads, args.dtype)
    for _ in range(args.warmup):
        sample.run()
    times = [sample.run() for _ in range(args.steps)]
    sample.close()
    t = statistics.median(times)
    value = sample.n / t
    layout = PageLayout([s.bytes // 2 for s in specs], page)
    cfg = gpu_config(args, specs, page, layout)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "params/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": "params/s", "cores": threads, "kind": sample.kind,
                         "sample": sample.describe() + f"; median of {args.steps} passes"},
        "e2e": {"value": value, "unit": "params/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "run": {"reference_grad_dtype": sample.dtype, "sample_params": sample.n, "threads": threads},
    }
    print(json.dumps(line), flush=True)


# ---- the GPU arm ----------------------------------------------------------------------

def build_state(args, device, world=1, rank=0, pool_alloc=None, double_buffered=False):
    import torch
    from paper_2303_02868_b200 import lockfree as LF
    from paper_2303_02868_b200 import workloads as W
    from paper_2303_02868_b200.layout import PageLayout
    specs = W.config_specs(args.config)
    page = args.page_mib * 2**20 if args.page_mib else W.config_page_bytes(args.config)
    numels = [s.bytes // 2 for s in specs]
    layout = PageLayout(numels, page, world_size=world, rank=rank,
                        bucket_pages=args.bucket_pages if world > 1 else None,
                        names=[s.name for s in specs])
    gen = torch.Generator(device=device)
    gen.manual_seed(1234)
    params = [torch.empty(n, dtype=torch.float32, device=device).normal_(0, 0.02, generator=gen)
              for n in numels]
    buf = LF.ParamBuffer(params, dtype=args.dtype, page_bytes=page, device=device, layout=layout,
                         pool_alloc=pool_alloc)
    ms = LF.MasterState(params, page_bytes=page, device=device, layout=layout,
                        double_buffered=double_buffered)
    del params
    torch.cuda.empty_cache()
    return specs, page, layout, buf, ms


def synthetic_grads(numels, dtype, device, seed):
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float16
    return [torch.empty(n, dtype=torch.float32, device=device).normal_(0, 1e-2, generator=gen).to(tdt)
            for n in numels]


def _events(stream, fn, reps: int) -> float:
    """ms per call of ``fn`` over ``reps`` back-to-back calls (CUDA events)."""
    import torch
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def run_ours_single(args):
    import torch
    from paper_2303_02868_b200 import _device as Dv
    from paper_2303_02868_b200 import lockfree as LF
    device = torch.device("cuda", 0)
    numa = Dv.bind_to_gpu_numa(0)   # pinned host buffers next to the GPU's PCIe root
    torch.cuda.set_device(device)
    specs, page, layout, buf, ms = build_state(args, device)
    L = len(specs)
    numels = layout.numels
    P = sum(numels)
    hyper = LF.AdamHyper(lr=1e-3)
    opts = Dv.opts(adam_threads=args.adam_threads, adam_variant=args.adam_variant)
    # Fill BOTH gradient page buffers through accumulate (K3, which also
    # computes each layer's finite flag, norm and ledger sum); every step
    # re-offers them, so the timed region reads gradients already in HBM.
    grads = torch.cat(synthetic_grads(numels, args.dtype, device, 7))  # flat, layer order
    for rnd in range(2):
        buf.accumulate_flat(grads, rnd)
        if rnd == 0:
            LF.sweep(buf, ms, hyper, opts=opts)

    def rearm():
        for l in range(L):
            buf._pending[l] = 1

    stream = torch.cuda.current_stream(device)
    for _ in range(args.warmup):
        rearm()
        LF.sweep(buf, ms, hyper, opts=opts)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    with ClockSampler(0) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record(stream)
        for i in range(args.steps):
            rearm()
            ev[2 * i].record(stream)
            LF.sweep(buf, ms, hyper, opts=opts)
            ev[2 * i + 1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    total_ms = t0.elapsed_time(t1)
    kern_ms = statistics.mean(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(args.steps))
    ms_per_step = total_ms / args.steps
    value = P / (ms_per_step / 1e3)
    peak, peak_kind = load_peaks()
    achieved = BYTES_PER_PARAM * P / (kern_ms / 1e3) / 1e9

    # K3 producer alone (first message of one flat gradient into every layer's
    # pages, fused flag + norm + ledger sum), back to back.
    def first_message():
        for l in range(L):
            buf._pending[l] = 0
        buf.accumulate_flat(grads, 0)
    for _ in range(3):
        first_message()
    acc_ms = _events(stream, first_message, 10)
    buf._ledger_flush()

    # The whole device step of the updating path: K3 (gradient into pages)
    # then the fused sweep — 32 B/param (4 B K3 + 28 B update).
    def device_step():
        buf.accumulate_flat(grads, 0)
        LF.sweep(buf, ms, hyper, opts=opts)
    for _ in range(3):
        device_step()
    dev_ms = _events(stream, device_step, 10)
    buf._ledger_flush()

    three = run_three_call(args, buf, ms, hyper, grads) if args.three_call_steps > 0 else None
    e2e = run_e2e(args, buf, ms, hyper, grads, device) if args.e2e_steps > 0 else None
    traffic = load_traffic(args)
    cpu = None
    Dv.restore_affinity(numa)   # the CPU baseline gets every host core
    if not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        smp, t, passes = cpu_reference_sample(page, args.cpu_sample_pages, threads, args.dtype,
                                              min_seconds=args.cpu_seconds)
        cpu = {"value": smp.n / t, "unit": "params/s", "cores": threads, "kind": smp.kind,
               "sample": smp.describe() + f"; median of {passes} passes (>= {args.cpu_seconds:g} s of CPU work)"}
        # the reference itself is single-threaded numpy: one thread, for context
        one, t1s, _ = cpu_reference_sample(page, max(1, args.cpu_sample_pages // 8), 1, args.dtype,
                                           min_seconds=min(2.0, args.cpu_seconds))
        cpu["single_thread_value"] = one.n / t1s
    line = {
        "metric": METRIC, "value": value, "unit": "params/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": gpu_config(args, specs, page, layout),
        "run": {"adam_threads": args.adam_threads, "adam_variant": ["ldg", "tma"][args.adam_variant],
                "numa_bind": {k: v for k, v in numa.items() if k != "_before"} if numa else None,
                "kernels": "fused sweep: prologue + page-Adam over all pages"},
        "hbm_gbs": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic,
                     "bytes_per_param": BYTES_PER_PARAM, "kernel": "adam_main (+ prologue)",
                     "kernel_ms": kern_ms},
        "accumulate": {"params_per_s": P / (acc_ms / 1e3), "ms": acc_ms,
                       "gbs": 4 * P / (acc_ms / 1e3) / 1e9, "frac": 4 * P / (acc_ms / 1e3) / 1e9 / peak,
                       "bytes_per_param": 4,
                       "note": "K3: first-message accumulate of one flat gradient into all layers' "
                               "pages (read payload, write page) with fused finite flag + squared norm + "
                               "conservation-ledger sum, one launch"},
        "device_step": {"params_per_s": P / (dev_ms / 1e3), "ms": dev_ms,
                        "gbs": 32 * P / (dev_ms / 1e3) / 1e9, "frac": 32 * P / (dev_ms / 1e3) / 1e9 / peak,
                        "bytes_per_param": 32,
                        "note": "K3 accumulate + fused sweep, back to back (gradient into pages, then "
                                "take->update->publish)"},
        "clocks": clk.summary(),
        "gpu_launches": 2 * args.steps,
    }
    if three:
        line["three_call"] = three
    if e2e:
        line["e2e"] = e2e
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def run_three_call(args, buf, ms, hyper, grads):
    """The reference's own per-layer loop through the drop-in with torch
    tensors (hiermem/lockfree.py:755-769: take -> update_layer ->
    publish(clear=False), layers reversed), after the K3 accumulate — to set
    beside ``device_step`` (K3 + the fused sweep of the same work).  take
    widens (6 B/param); update_layer reads the taken 16-bit pages in place,
    pre-publishes and writes the new p32 as a tensor in ONE launch (28 + 4 B);
    p32[l] hands that tensor out; publish only flips: 38 B/param + one K3
    (4 B), two launches per layer (+ one batched ledger snapshot)."""
    import torch
    L = buf.num_layers
    P = sum(buf.layout.numels)

    def step():
        buf.accumulate_flat(grads, 0)
        for l in reversed(range(L)):
            g, _c, newest = buf.take(l)
            ms.update_layer(l, g, hyper)
            buf.publish(l, ms.p32[l], applied_iter=newest, clear=False)
    for _ in range(2):
        step()
    stream = torch.cuda.current_stream()
    t = _events(stream, step, args.three_call_steps)
    buf._ledger_flush()
    return {"params_per_s": P / (t / 1e3), "ms": t, "bytes_per_param": 42,
            "gbs": 42 * P / (t / 1e3) / 1e9,
            "api": "accumulate_flat + per layer (reversed): ParamBuffer.take -> MasterState.update_layer -> "
                   "ParamBuffer.publish(MasterState.p32[l], clear=False), torch tensors"}


def run_e2e(args, buf, ms, hyper, grads, device):
    """Public API with host buffers: per step H2D of every layer's gradient
    from pinned memory + accumulate (K3) + fused sweep (K2) + D2H of the
    step's result — the freshly published 16-bit parameters of every layer
    (and the per-layer applied flags)."""
    import torch
    from paper_2303_02868_b200 import lockfree as LF
    host = grads.cpu().pin_memory()
    out = torch.empty_like(host).pin_memory()
    h2d = host.numel() * host.element_size()
    L = buf.num_layers

    def serial_step():
        buf.accumulate_flat(host, 0)       # H2D from pinned memory + K3
        res = LF.sweep(buf, ms, hyper)     # fused take -> update -> publish (K2)
        return res.applied()               # D2H of the per-layer applied flags

    def pipelined_step(results):
        # per layer group: H2D on a copy stream -> K3 -> fused sweep -> D2H of
        # the group's published pages on a second copy stream; the transfer
        # of group k+1 overlaps the update of group k and the return of k-1
        res = LF.ingest_sweep(buf, ms, host, hyper, 0, groups=args.e2e_groups,
                              results_to=out if results else None)
        return res.applied()

    def timed(step):
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            step()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / args.e2e_steps

    dt_serial = timed(serial_step)
    dt_nores = timed(lambda: pipelined_step(False))
    dt = timed(lambda: pipelined_step(True))
    buf._ledger_flush()
    P = sum(buf.layout.numels)
    d2h = out.numel() * out.element_size() + 4 * L
    return {"value": P / dt, "unit": "params/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3, "steps": args.e2e_steps,
            "api": f"lockfree.ingest_sweep(pinned host gradient, {args.e2e_groups} layer groups, "
                   "results_to=pinned host params)",
            "pcie_gbs": (h2d + d2h) / dt / 1e9,
            "no_results_ms_per_step": dt_nores * 1e3,
            "serial_ms_per_step": dt_serial * 1e3,
            "serial_api": "accumulate_flat(host) + sweep (applied flags only)"}


def load_traffic(args):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get(f"{args.config}:{args.dtype}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp16"])
    ap.add_argument("--page-mib", type=int, default=0)
    ap.add_argument("--bucket-pages", type=int, default=32)
    ap.add_argument("--dp-groups", type=int, default=-1,
                    help="fused DP step: >1 pipelines the reduce-scatter of layer group k+1 with the "
                         "update + all-gather of group k; -1 = auto (8 groups with a 128-CTA reduce "
                         "grid at N=2 for >= 1 GB of 16-bit pages, where the update is HBM-bound; "
                         "1 otherwise and at N>=4, where the whole "
                         "step is NVLink-bound — profiles/r1_dp_c2.md)")
    ap.add_argument("--ag-publish", type=int, default=0, choices=[0, 1, 2],
                    help="fused DP all-gather epilogue: 0 per-thread peer stores, 1 per-CTA bulk "
                         "copies (cp.async.bulk, waiting for the remote writes); 2 = 1")
    ap.add_argument("--dp-reduce-wide", type=int, default=1, choices=[0, 1],
                    help="fused DP reduce with 256-bit peer loads (hm_set_dp_reduce_wide; 0 = 16 B loads)")
    ap.add_argument("--dp-reduce-sms", type=int, default=0,
                    help="pipelined DP step: run the reduce and the update in two CUDA green "
                         "contexts, this many SMs for the reduce (0 = shared SMs)")
    ap.add_argument("--dp-update-ctas", type=int, default=0,
                    help="pipelined DP step: persistent grid of the update+all-gather kernel (0 = one "
                         "CTA per chunk)")
    ap.add_argument("--dp-reduce-ctas", type=int, default=0,
                    help="pipelined DP step: persistent grid of the reduce kernel (0 = one CTA per "
                         "chunk) so it shares the SMs with the previous group's update")
    ap.add_argument("--dp-onepass", type=int, default=-1, choices=[-1, 0, 1],
                    help="fused P2P DP step as ONE kernel over a double-buffered fp32 state "
                         "(reduce-scatter + update + all-gather, commit after a flag merge); "
                         "-1 = auto (on at N=2, where it wins; profiles/r2_bench.md)")
    ap.add_argument("--dp-push", type=int, default=-1, choices=[-1, 0, 1],
                    help="one-pass DP step: 1 = push form (every rank stores the non-owned gradient into the "
                         "owner's receive pool), 0 = pull form, -1 = the measured policy")
    ap.add_argument("--dp-mode", default="p2p", choices=["nccl", "p2p", "nvls"],
                    help="N>1 collectives: NCCL RS/AG, or fused kernels over NVLink peer memory "
                         "(p2p) / NVSwitch multicast (nvls)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--three-call-steps", type=int, default=5,
                    help="N=1: also time the reference's per-layer take->update_layer->publish loop")
    ap.add_argument("--e2e-groups", type=int, default=8)
    ap.add_argument("--cpu-sample-pages", type=int, default=32)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="GPU arm's cpu_baseline: repeat the sample for at least this much CPU work")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--c3-layers", type=int, default=0,
                    help="C3 transformer layers (0 = as many of the 40 as the box's host memory holds)")
    ap.add_argument("--c3-lockfree-iters", type=int, default=4,
                    help="C3 host tier: also time sync vs lock-free delayed update (0 = skip)")
    ap.add_argument("--c3-tokens", type=int, default=16384,
                    help="tokens per step of the modelled GPU actor (C3 lock-free line)")
    ap.add_argument("--adam-threads", type=int, default=256, choices=[256, 512])
    ap.add_argument("--adam-variant", type=int, default=0, choices=[0, 1],
                    help="page-Adam data movement: 0 LDG/STG streaming, 1 TMA bulk-copy pipeline")
    ap.add_argument("--swap-group-pages", type=int, default=64)
    ap.add_argument("--swap-slots", type=int, default=2)
    ap.add_argument("--state-tier", default="host", choices=["host", "ssd"],
                    help="C3: fp32 state in pinned host memory or in a file on the SSD")
    ap.add_argument("--ssd-dir", default="/tmp", help="directory of the SSD tier's state file")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # plain `python bench.py --gpus N`: relaunch as N ranks, one per GPU
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.execvp(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                   f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
                                   f"--master-port={port}", str(ROOT / "bench.py"), *sys.argv[1:]])
    if args.config == "c3":
        from paper_2303_02868_b200 import swap_bench
        return swap_bench.run(args, METRIC, BYTES_PER_PARAM, ClockSampler, load_peaks)
    if world > 1 or args.gpus > 1:
        from paper_2303_02868_b200 import dp_bench
        return dp_bench.run(args, METRIC, BYTES_PER_PARAM, ClockSampler, load_peaks, build_state)
    return run_ours_single(args)


if __name__ == "__main__":
    main()
