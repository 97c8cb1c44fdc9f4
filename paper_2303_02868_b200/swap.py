"""Pinned-host page swap tier (K8): fp32 master state in CPU memory, streamed
through HBM staging page by page in the updating actor's order.

The reference keeps master state "SSD-resident in spirit" (hiermem/lockfree.py:
8, MasterState tier="SSD" :148) and charges state fetch/store as sleeps of
``state_bytes32 / rate`` (DelayModel, :90-103; 12 B/param each way).  The
updating actor's per-layer order is: take -> state fetch -> update ->
publish -> state store, sweeping layers in reverse (:624-639).  Here those
bytes really move: p32/m32/v32 pages live in pinned host pools, and a sweep
walks page groups from the last page to the first (the reverse layer order
of a page table allocated layer by layer):

    copy stream H2D : host p/m/v pages of group k       -> staging slot k%S
    compute stream  : page-Adam on the staged pages (reads g16, writes p16)
    copy stream D2H : staging slot                      -> host pages

with S staging slots (double buffering by default): the fetch of group k+1
and the store of group k-1 overlap the update of group k, and a slot is only
re-filled after its previous store finished (event-gated), so every page is
fetched, updated, published and stored exactly once per sweep, in order.
Each page belongs to one group (groups are page ranges), so a page shared by
two layers' tails is never fetched twice in flight.  Takes and the per-layer
reject/step decision happen once, in the prologue at the start of the sweep.
Transfers are one cudaMemcpyAsync per contiguous run on dedicated copy
streams (copy engines, no SMs); PCIe is the roofline (12 B in + 12 B out
per param).  SSD (GDS/cuFile) is out of scope.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import ConfigError
from .layout import PageLayout
from .lockfree import MasterState, ParamBuffer, SweepResult, _Paged
from .pagemem import PAGE_BYTES_DEFAULT


class HostMasterState(_Paged):
    """MasterState with p32/m32/v32 in pinned host page pools."""

    def __init__(self, params, tier: str = "CPU", *, page_bytes: int = PAGE_BYTES_DEFAULT,
                 device=None, layout: PageLayout | None = None, group_pages: int = 64,
                 slots: int = 2):
        self._init_paged(params, page_bytes, device, layout)
        if self.layout.world_size != 1:
            raise ConfigError("the host swap tier is per process; shard with one layout per rank")
        self.tier = tier
        lay = self.layout
        E = lay.E
        self.group_pages = max(1, int(group_pages))
        self.num_groups = -(-lay.P_local // self.group_pages)
        n = lay.elems_state
        self.host_p = torch.zeros(n, dtype=torch.float32, pin_memory=True)
        self.host_m = torch.zeros(n, dtype=torch.float32, pin_memory=True)
        self.host_v = torch.zeros(n, dtype=torch.float32, pin_memory=True)
        for l, p in enumerate(params):
            flat = (p.detach().reshape(-1).float().cpu() if isinstance(p, torch.Tensor)
                    else torch.from_numpy(np.asarray(p, dtype=np.float32).reshape(-1)))
            for s in lay.segments[l]:
                o = lay.slot_state(s.page) * E + s.off
                self.host_p[o:o + s.n] = flat[s.pos:s.pos + s.n]
        gE = self.group_pages * E
        self.slots = max(2, int(slots))
        self.stage = [torch.empty(3, gE, dtype=torch.float32, device=self.device) for _ in range(self.slots)]
        self.h2d = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)
        with torch.cuda.stream(self._stream()):
            self._steps = torch.zeros(self.num_layers, dtype=torch.int32, device=self.device)
            self._applied = torch.zeros(self.num_layers, dtype=torch.int32, device=self.device)
        self._step_bound = [0] * self.num_layers
        self._stored = [None] * self.slots   # event: slot's last store finished
        self._plans: dict = {}

    # reference attributes (host reads: synchronise the copy streams first) ----
    def _host_layer(self, pool, layer):
        torch.cuda.current_stream(self.device).wait_stream(self.d2h)
        torch.cuda.synchronize(self.device)
        out = torch.empty(self.layout.numels[layer], dtype=torch.float32)
        E = self.layout.E
        for s in self.layout.segments[layer]:
            o = self.layout.slot_state(s.page) * E + s.off
            out[s.pos:s.pos + s.n] = pool[o:o + s.n]
        return out.numpy().reshape(self._shapes[layer]) if self._numpy else out.view(self._shapes[layer])

    @property
    def p32(self):
        from .lockfree import _LayerView
        return _LayerView(self, lambda l: self._host_layer(self.host_p, l))

    @property
    def m32(self):
        from .lockfree import _LayerView
        return _LayerView(self, lambda l: self._host_layer(self.host_m, l))

    @property
    def v32(self):
        from .lockfree import _LayerView
        return _LayerView(self, lambda l: self._host_layer(self.host_v, l))

    @property
    def steps(self) -> list[int]:
        return [int(x) for x in self._steps.cpu().tolist()]

    _bias = MasterState._bias

    # plan: per page group, the adam chunks re-based onto a staging slot ----------
    def _group_plan(self, layers: tuple):
        if layers in self._plans:
            return self._plans[layers]
        lay, E, G = self.layout, self.layout.E, self.group_pages
        full = lay.adam_chunks(layers, "pool", owned_only=True)
        page = full["s_off"] // E
        plan = []
        for k in reversed(range(self.num_groups)):   # last pages first: reverse layer order
            sel = (page >= k * G) & (page < (k + 1) * G)
            if not sel.any():
                continue
            c = full[sel].copy()
            c["s_off"] -= k * G * E
            first, last = k * G, min((k + 1) * G, lay.P_local)
            plan.append((k, first, last, c))
        self._plans[layers] = plan
        return plan


def _runs(hosts, stage, host_off: int, n: int, fetch: bool):
    """Three copy runs (p, m, v) with absolute addresses (bases are NULL)."""
    d = np.zeros(3, dtype=N.COPY_DESC)
    for a in range(3):
        h = hosts[a].data_ptr() + 4 * host_off
        g = stage[a].data_ptr()
        d[a] = (h, g, 4 * n) if fetch else (g, h, 4 * n)
    return d


def swap_sweep(buffer: ParamBuffer, masters: HostMasterState, hyper, layers=None, *,
               stream=None, timings: dict | None = None) -> SweepResult:
    """``sweep`` (lockfree.py) with the state in pinned host memory: one
    prologue, then per page group H2D -> page-Adam -> D2H, pipelined."""
    lay = buffer.layout
    if masters.layout.numels != lay.numels or masters.layout.page_bytes != lay.page_bytes:
        raise ConfigError("buffer and masters were built on different page tables")
    st = buffer._stream(stream)
    order = list(reversed(range(buffer.num_layers))) if layers is None else list(layers)
    sel = tuple(l for l in order if buffer._pending[l] > 0)
    if not sel:
        return SweepResult(masters, [], [], [])
    L, span = buffer.num_layers, lay.elems16
    rows, counts, newest = [], [], []
    for l in sel:
        gbuf, count, new = buffer._hand_over(l, st)
        rows.append((gbuf * span, (buffer._psel[l] ^ 1) * span, l, gbuf * L + l))
        counts.append(count)
        newest.append(new)
    groups = np.zeros(len(rows), dtype=N.GROUP_LAUNCH)
    for i, r in enumerate(rows):
        groups[i] = r
    eng = masters._eng
    dgroups = eng.desc.table(groups)
    rt = eng.rt_scratch(len(rows))
    bc, bc_len = masters._bias(hyper, sel)
    hc = D.hyper_c(hyper)
    lib = N.lib()
    D.check(lib.hm_adam_prologue(D.ptr(dgroups), len(rows), D.ptr(rt), hc, D.ptr(bc), bc_len, 0,
                                 D.ptr(masters._steps), D.ptr(masters._applied), D.ptr(buffer._flags),
                                 D.ptr(buffer._sumsq), 1, D.sptr(st)))
    E = lay.E
    hosts = (masters.host_p, masters.host_m, masters.host_v)
    ev = (lambda: torch.cuda.Event(enable_timing=True)) if timings is not None else torch.cuda.Event
    first_ev = last_ev = None
    for i, (k, first, last, chunks) in enumerate(masters._group_plan(sel)):
        slot = i % masters.slots
        stage = masters.stage[slot]
        n = (last - first) * E
        # fetch: wait until this slot's previous store has drained
        if masters._stored[slot] is not None:
            masters.h2d.wait_event(masters._stored[slot])
        runs = _runs(hosts, stage, first * E, n, fetch=True)
        D.check(lib.hm_memcpy_runs(None, None, runs.ctypes.data, 3, 1, D.sptr(masters.h2d)))
        with torch.cuda.stream(masters.h2d):
            fetched = ev()
            fetched.record(masters.h2d)
            if first_ev is None and timings is not None:
                first_ev = fetched
        st.wait_event(fetched)
        D.check(lib.hm_adam_main(D.ptr(eng.desc.static(chunks)), len(chunks), D.ptr(dgroups), D.ptr(rt),
                                 D.ptr(buffer.g16_pool), buffer._dt, D.ptr(stage[0]), D.ptr(stage[1]),
                                 D.ptr(stage[2]), D.ptr(buffer.p16_pool), buffer._dt, hc, D.sptr(st)))
        updated = torch.cuda.Event()
        updated.record(st)
        masters.d2h.wait_event(updated)
        runs = _runs(hosts, stage, first * E, n, fetch=False)
        D.check(lib.hm_memcpy_runs(None, None, runs.ctypes.data, 3, 2, D.sptr(masters.d2h)))
        with torch.cuda.stream(masters.d2h):
            stored = ev()
            stored.record(masters.d2h)
        masters._stored[slot] = stored
        last_ev = stored
    st.wait_stream(masters.d2h)
    for l, new in zip(sel, newest):
        buffer._psel[l] ^= 1
        buffer._version[l] += 1
        buffer._applied_iter[l] = new
    if timings is not None:
        timings["first_fetch"], timings["last_store"] = first_ev, last_ev
    return SweepResult(masters, sel, counts, newest)
