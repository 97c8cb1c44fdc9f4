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
per param).  The SSD tier (POSIX I/O, no GDS in the image) is ssd.py.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import ConfigError
from .layout import PageLayout
from .lockfree import MasterState, ParamBuffer, SweepResult, UpdateTicket, _Paged, update_prologue
from .pagemem import PAGE_BYTES_DEFAULT


class HostMasterState(_Paged):
    """MasterState with p32/m32/v32 in pinned host page pools.

    Data parallel: built on a world-sharded layout, a rank pins only the
    state pages it owns (``owner(page) = page % N``, hiermem/scheduler.py:
    72-76) — 12 B x params / N of host memory per rank — and the DP step
    (``sharding.FusedShardedPageStep``) streams them through the same
    pipeline between its reduce-scatter and its all-gather."""

    def __init__(self, params, tier: str = "CPU", *, page_bytes: int = PAGE_BYTES_DEFAULT,
                 device=None, layout: PageLayout | None = None, group_pages: int = 64,
                 slots: int = 2, world_size: int = 1, rank: int = 0):
        self._init_paged(params, page_bytes, device, layout, world_size, rank)
        self.tier = tier
        lay = self.layout
        E = lay.E
        self.group_pages = max(1, int(group_pages))
        self.num_groups = -(-lay.P_local // self.group_pages)
        n = lay.elems_state
        # exact-size page-locked pools (torch's pinned allocator would round
        # each up to a power of two: 64 GB for C3's 51.4 GB p32 pool)
        self.host_p = D.pinned_zeros(n)
        self.host_m = D.pinned_zeros(n)
        self.host_v = D.pinned_zeros(n)
        for l, p in enumerate(params):
            if p is None:   # caller fills host_p itself (e.g. a bench writing synthetic pages)
                continue
            flat = (p.detach().reshape(-1).float().cpu() if isinstance(p, torch.Tensor)
                    else torch.from_numpy(np.asarray(p, dtype=np.float32).reshape(-1)))
            for s in lay.segments[l]:
                if lay.owned(s):
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
        self._group_stored: dict = {}        # page group -> event: its last store finished
        self._plans: dict = {}

    # reference attributes (host reads: synchronise the copy streams first) ----
    def _host_layer(self, pool, layer):
        torch.cuda.current_stream(self.device).wait_stream(self.d2h)
        torch.cuda.synchronize(self.device)
        out = torch.zeros(self.layout.numels[layer], dtype=torch.float32)
        E = self.layout.E
        for s in self.layout.segments[layer]:
            if self.layout.owned(s):
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

    def planes(self, stage) -> tuple[int, int, int]:
        return stage_planes(stage)

    def stream_update(self, layers, st, launch, timings=None) -> None:
        swap_pipeline(self, layers, st, launch, timings)

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


def stage_planes(stage) -> tuple[int, int, int]:
    """Device addresses of the p / m / v planes of a staging slot."""
    return D.ptr(stage[0]), D.ptr(stage[1]), D.ptr(stage[2])


def _runs(hosts, stage, host_off: int, n: int, fetch: bool):
    """Three copy runs (p, m, v) with absolute addresses (bases are NULL)."""
    d = np.zeros(3, dtype=N.COPY_DESC)
    for a in range(3):
        h = hosts[a].data_ptr() + 4 * host_off
        g = stage[a].data_ptr()
        d[a] = (h, g, 4 * n) if fetch else (g, h, 4 * n)
    return d


def swap_pipeline(masters: HostMasterState, layers: tuple, st, launch, timings: dict | None = None):
    """Stream the state pages of ``layers`` through HBM staging: per page
    group (last first), H2D fetch on the copy stream -> ``launch(chunks,
    stage)`` (the main pass on ``st``, chunks re-based onto the stage) ->
    D2H store on the second copy stream.  A slot is refilled only after its
    previous store drained, and a group's fetch waits for the group's own
    last store (whichever slot it went through in an earlier sweep), so a
    page is never fetched before its last update reached the host."""
    lib = N.lib()
    E = masters.layout.E
    hosts = (masters.host_p, masters.host_m, masters.host_v)
    ev = (lambda: torch.cuda.Event(enable_timing=True)) if timings is not None else torch.cuda.Event
    first_ev = last_ev = None
    for i, (k, first, last, chunks) in enumerate(masters._group_plan(tuple(layers))):
        slot = i % masters.slots
        stage = masters.stage[slot]
        n = (last - first) * E
        if masters._stored[slot] is not None:    # this slot's previous store has drained
            masters.h2d.wait_event(masters._stored[slot])
        prev = masters._group_stored.get(k)
        if prev is not None:                     # the group's last update is back on the host
            masters.h2d.wait_event(prev)
        runs = _runs(hosts, stage, first * E, n, fetch=True)
        D.check(lib.hm_memcpy_runs(None, None, runs.ctypes.data, 3, 1, D.sptr(masters.h2d)))
        with torch.cuda.stream(masters.h2d):
            fetched = ev()
            fetched.record(masters.h2d)
            if first_ev is None and timings is not None:
                first_ev = fetched
        st.wait_event(fetched)
        launch(chunks, stage)
        updated = torch.cuda.Event()
        updated.record(st)
        masters.d2h.wait_event(updated)
        runs = _runs(hosts, stage, first * E, n, fetch=False)
        D.check(lib.hm_memcpy_runs(None, None, runs.ctypes.data, 3, 2, D.sptr(masters.d2h)))
        with torch.cuda.stream(masters.d2h):
            stored = ev()
            stored.record(masters.d2h)
        masters._stored[slot] = stored
        masters._group_stored[k] = stored
        last_ev = stored
    st.wait_stream(masters.d2h)
    if timings is not None:
        timings["first_fetch"], timings["last_store"] = first_ev, last_ev


def swap_sweep(buffer: ParamBuffer, masters: HostMasterState, hyper, layers=None, *,
               stream=None, timings: dict | None = None) -> SweepResult:
    """``sweep`` (lockfree.py) with the state in pinned host memory: one
    prologue, then per page group H2D -> page-Adam -> D2H, pipelined."""
    lay = buffer.layout
    if masters.layout.numels != lay.numels or masters.layout.page_bytes != lay.page_bytes:
        raise ConfigError("buffer and masters were built on different page tables")
    if lay.world_size != 1:
        raise ConfigError("a world-sharded host tier is updated by the DP step "
                          "(sharding.FusedShardedPageStep), which all-gathers the published pages")
    st = buffer._stream(stream)
    order = list(reversed(range(buffer.num_layers))) if layers is None else list(layers)
    sel = tuple(l for l in order if buffer._pending[l] > 0)
    if not sel:
        return SweepResult(masters, [], [], [])
    t = UpdateTicket(buffer, sel)
    dgroups, rt, hc = update_prologue(t, masters, hyper, st)
    lib = N.lib()

    def launch(chunks, stage):
        D.check(lib.hm_adam_main(D.ptr(masters._eng.desc.static(chunks)), len(chunks), D.ptr(dgroups),
                                 D.ptr(rt), D.ptr(buffer.g16_pool), buffer._dt, *masters.planes(stage),
                                 D.ptr(buffer.p16_pool), buffer._dt, hc, None, D.sptr(st)))

    swap_pipeline(masters, sel, st, launch, timings)
    t.finish()
    return SweepResult(masters, sel, t.counts, t.newest)
