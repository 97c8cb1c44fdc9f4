"""Executor for the reference's Algorithm-1 page schedules on real hardware.

The reference plans page motion ahead of time — ``schedule()`` emits
``move_to_gpu`` / ``all_gather`` / ``compute`` / ``evict_to_cpu`` tasks with
trigger slots (hiermem/scheduler.py:264-403) — and then
only *replays* them on a model of the hardware (hiermem/simengine.py:190-355).
The paper's Executor runs them.  This one runs a
``Schedule.to_dict()`` of one rank with real bytes on a B200:

* host tier: every parameter page (LayerModel numbering, scheduler.py:93-102)
  in pinned memory;
* GPU tier: a page pool of ``gpu_budget // page_bytes`` pages managed by the
  native page table — the allocator itself refuses a schedule that would
  exceed the budget on parameters;
* ``move_to_gpu``: cudaMemcpyAsync H2D on a copy stream into a claimed page
  (waits for the previous store out of that page and into that host page);
* ``evict_to_cpu``: D2H on a second copy stream once the computes that read
  the page have run, then the page is released;
* ``all_gather``: at world size 1 every page is owned, so the gather is the
  dependency "compute waits for the page's arrival" (the reference charges
  it on the interconnect; no bytes need to move);
* ``compute``: the slot's modelled duration (the simulator's own timing model,
  or a given list) as a spin of one warp — it moves no bytes, so the measured
  makespan isolates how the schedule's transfers overlap compute.

Tasks whose trigger is t are issued when slot t starts, in schedule order,
exactly the eligibility rule of simengine.py:1-10.  The report compares the
measured makespan with the simulated one and checks every page's bytes
after the round trip.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import ConfigError
from .pagemem import PageManager
from .workloads import TensorSpec


class ScheduleExecutor:
    def __init__(self, schedule: dict, *, device=None, slot_seconds=None, compute_scale: float = 1.0,
                 seed: int = 0):
        self.device = D.require_device(device)
        model = schedule["model"]
        if schedule.get("world_size", 1) != 1:
            raise ConfigError("this executor runs one rank of world size 1 (every page owned)")
        self.L = model["num_layers"]
        self.page = model["page_bytes"]
        self.budget = schedule["gpu_budget"]
        self.layer_pages, pid = [], 0
        for nbytes in model["layer_param_bytes"]:
            count = max(1, math.ceil(nbytes / self.page))
            self.layer_pages.append(list(range(pid, pid + count)))
            pid += count
        self.P = pid
        self.page_layer = {p: l for l, ps in enumerate(self.layer_pages) for p in ps}
        self.tasks = schedule["tasks"]
        self.slot_seconds = list(slot_seconds) if slot_seconds is not None else [0.0] * (2 * self.L)
        self.compute_scale = compute_scale
        cap_pages = self.budget // self.page
        if cap_pages < 1:
            raise ConfigError("budget smaller than one page")
        self.pm = PageManager([("GPU", cap_pages * self.page, self.page)])
        self.gpu = torch.empty(cap_pages * self.page, dtype=torch.uint8, device=self.device)
        g = torch.Generator().manual_seed(seed)
        self.ref = torch.randint(0, 256, (self.P * self.page,), dtype=torch.uint8, generator=g)
        self.host = self.ref.clone().pin_memory()
        self.h2d = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)
        self.cs = torch.cuda.Stream(self.device)

    def _copy(self, kind: int, src_off: int, dst_off: int, stream) -> None:
        d = np.array([(src_off, dst_off, self.page)], dtype=N.COPY_DESC)
        src, dst = (self.host, self.gpu) if kind == 1 else (self.gpu, self.host)
        D.check(N.lib().hm_memcpy_runs(D.ptr(src), D.ptr(dst), d.ctypes.data, 1, kind, D.sptr(stream)))

    def run(self) -> dict:
        by_trigger: dict[int, list] = {}
        for t in self.tasks:
            by_trigger.setdefault(t["trigger_id"], []).append(t)
        resident: dict[int, tuple] = {}          # page -> (tensor id, gpu page, arrival event)
        slot_free: dict[int, torch.cuda.Event] = {}
        host_ready: dict[int, torch.cuda.Event] = {}
        waits: dict[int, list] = {}              # layer -> arrival events its compute needs
        last_compute = None
        counts = {"move_to_gpu": 0, "evict_to_cpu": 0, "all_gather": 0, "compute": 0}
        torch.cuda.synchronize(self.device)
        start = torch.cuda.Event(enable_timing=True)
        start.record(self.cs)
        self.h2d.wait_event(start)
        self.d2h.wait_event(start)
        # triggers run 0..2n: the last backward slot's evictions fire at 2n
        for slot in range(max(max(by_trigger, default=0), 2 * self.L - 1) + 1):
            for task in by_trigger.get(slot, ()):
                op, target = task["operation"], task["target"]
                counts[op] += 1
                if op == "move_to_gpu":
                    spec = TensorSpec(f"page{target}", "param16", self.page, self.page_layer[target])
                    tid = self.pm.allocate(spec, "GPU").tensor_id
                    gpage = self.pm.tensors[tid].page_list[0]
                    if gpage in slot_free:
                        self.h2d.wait_event(slot_free[gpage])
                    if target in host_ready:
                        self.h2d.wait_event(host_ready[target])
                    self._copy(1, target * self.page, gpage * self.page, self.h2d)
                    ev = torch.cuda.Event()
                    ev.record(self.h2d)
                    resident[target] = (tid, gpage, ev)
                elif op == "all_gather":
                    if target not in resident:
                        raise ConfigError(f"all_gather of page {target} before its move_to_gpu")
                    waits.setdefault(self.page_layer[target], []).append(resident[target][2])
                elif op == "compute":
                    for ev in waits.pop(target, ()):
                        self.cs.wait_event(ev)
                    ns = int(self.slot_seconds[task["slot"]] * self.compute_scale * 1e9)
                    D.check(N.lib().hm_spin(ns, D.sptr(self.cs)))
                    last_compute = torch.cuda.Event()
                    last_compute.record(self.cs)
                elif op == "evict_to_cpu":
                    tid, gpage, ev = resident.pop(target)
                    self.d2h.wait_event(ev)
                    if last_compute is not None:
                        self.d2h.wait_event(last_compute)
                    self._copy(2, gpage * self.page, target * self.page, self.d2h)
                    fe = torch.cuda.Event()
                    fe.record(self.d2h)
                    slot_free[gpage] = fe
                    host_ready[target] = fe
                    self.pm.release(tid)
                else:
                    raise ConfigError(f"unknown task operation {op!r}")
        for s in (self.h2d, self.d2h):
            self.cs.wait_stream(s)
        end = torch.cuda.Event(enable_timing=True)
        end.record(self.cs)
        torch.cuda.synchronize(self.device)
        makespan = start.elapsed_time(end) / 1e3
        # integrity: evicted pages are back in host memory, resident ones on the GPU
        ok = True
        for p in range(self.P):
            lo = p * self.page
            if p in resident:
                gp = resident[p][1]
                got = self.gpu[gp * self.page:(gp + 1) * self.page].cpu()
            else:
                got = self.host[lo:lo + self.page]
            ok &= bool(torch.equal(got, self.ref[lo:lo + self.page]))
        pool = next(iter(self.pm.pools.values()))
        moved = counts["move_to_gpu"] * self.page
        evicted = counts["evict_to_cpu"] * self.page
        return {"makespan_s": makespan, "tasks": counts, "pages": self.P,
                "gpu_pages_budget": pool.num_pages, "gpu_pages_peak": pool.stats.peak_allocated_pages,
                "h2d_bytes": moved, "d2h_bytes": evicted,
                "pcie_gbs": (moved + evicted) / makespan / 1e9 if makespan > 0 else None,
                "bytes_intact": ok, "compute_s": sum(self.slot_seconds) * self.compute_scale}
