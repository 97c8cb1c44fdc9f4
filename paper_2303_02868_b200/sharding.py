"""Data-parallel page sharding: gradient reduce-scatter and parameter
all-gather over the 16-bit page pools, one process per GPU.

Ownership is the reference's ``ShardingModel``: ``owner(page) = page % N``
(hiermem/scheduler.py:59-76), ZeRO-3 style at page granularity (PAPER.md:305,
685).  The reference only *models* the collectives — an all_gather task per
page costed as ``lat + page*(N-1)/N / bw`` (hiermem/simengine.py:255-257) and
no gradient reduce-scatter at all (SPEC.md:348 lists it as future work).
Here they move real bytes over NVLink/NVSwitch, two ways:

* ``FusedShardedPageStep`` (the default): the pools are symmetric memory
  mapped into every rank; the reduce-scatter is a kernel that pulls each
  owned page from every peer and fuses the finite flag / norm
  (hm_dp_reduce_check), and the all-gather is the page-Adam's publish
  epilogue storing into every peer (hm_adam_main_ag) — no NCCL on the data
  path; optionally pipelined over layer groups (``step_pipelined``), or,
  over a double-buffered fp32 state, ONE kernel for the reduce-scatter, the
  update and the all-gather (the one-pass step);
* ``ShardedPageStep`` (NCCL baseline): the 16-bit pools are laid out
  bucket-major, rank-major inside a bucket (layout.py), so bucket b is ONE
  contiguous buffer and rank r's owned pages are its r-th block:
  ``reduce_scatter_tensor`` / ``all_gather_into_tensor`` run in place; the
  step is RS(all buckets) -> finite/norm check -> all-reduce of the
  per-layer flags -> ONE prologue -> page-Adam(b) || AG(b) per bucket.

``PageCollectives`` is device-agnostic (it runs on CPU tensors under gloo in
the tests); the two step classes drive the CUDA kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _device as D
from . import _native as N
from .errors import ConfigError
from .layout import PageLayout
from .lockfree import UpdateTicket, update_prologue


@dataclass(frozen=True)
class ShardingModel:
    """Even page-level partitioning across data-parallel ranks
    (hiermem/scheduler.py:59-76)."""

    world_size: int = 1
    rank: int = 0

    def __post_init__(self):
        if self.world_size < 1 or not (0 <= self.rank < self.world_size):
            raise ConfigError(f"bad sharding: world_size={self.world_size} rank={self.rank}")

    def owner(self, page_id: int) -> int:
        return page_id % self.world_size

    def owns(self, page_id: int) -> bool:
        return self.owner(page_id) == self.rank


def modeled_gather_s(page_bytes: int, pages: int, world_size: int, bandwidth_bytes_per_s: float,
                     latency_s: float) -> float:
    """The reference's cost of gathering ``pages`` pages: one
    ``latency + page·(N−1)/N / bw`` task per page, serialised on the single
    ``gpu_interconnect`` resource (hiermem/simengine.py:255-257; a
    reduce-scatter moves the same bytes the other way).  bench.py prints it
    beside the measured fused step so the model can be checked against B200."""
    if world_size < 1 or pages < 0 or bandwidth_bytes_per_s <= 0:
        raise ConfigError("modeled_gather_s: bad arguments")
    frac = (world_size - 1) / world_size
    return pages * (latency_s + page_bytes * frac / bandwidth_bytes_per_s)


class PageCollectives:
    """In-place bucketed reduce-scatter / all-gather of a 16-bit page pool."""

    def __init__(self, layout: PageLayout, group=None):
        self.layout = layout
        self.group = group
        ws = dist.get_world_size(group)
        if ws != layout.world_size or dist.get_rank(group) != layout.rank:
            raise ConfigError(f"layout built for world {layout.world_size} rank {layout.rank}, "
                              f"process group is world {ws} rank {dist.get_rank(group)}")

    def bucket_views(self, pool: torch.Tensor, b: int):
        lay = self.layout
        lo, hi = lay.bucket_slots(b)
        whole = pool[lo * lay.E:hi * lay.E]
        blk = lay.K * lay.E
        mine = whole[lay.rank * blk:(lay.rank + 1) * blk]
        return whole, mine

    def reduce_scatter(self, pool: torch.Tensor, buckets=None, op=dist.ReduceOp.SUM, async_op=False,
                       coalesce: bool | None = None):
        """In-place RS of each bucket.  With ``coalesce`` (default on NCCL) all
        buckets go into ONE ncclGroupStart/End, i.e. one fused launch instead
        of a per-bucket latency each."""
        buckets = list(range(self.layout.num_buckets) if buckets is None else buckets)
        if coalesce is None:
            coalesce = pool.is_cuda and len(buckets) > 1
        if coalesce:
            with dist._coalescing_manager(group=self.group, device=pool.device, async_ops=True) as cm:
                for b in buckets:
                    whole, mine = self.bucket_views(pool, b)
                    dist.reduce_scatter_tensor(mine, whole, op=op, group=self.group)
            if async_op:
                return [cm]
            cm.wait()
            return []
        works = []
        for b in buckets:
            whole, mine = self.bucket_views(pool, b)
            works.append(dist.reduce_scatter_tensor(mine, whole, op=op, group=self.group,
                                                    async_op=async_op))
        return works

    def all_gather(self, pool: torch.Tensor, buckets=None, async_op=False):
        works = []
        for b in (range(self.layout.num_buckets) if buckets is None else buckets):
            whole, mine = self.bucket_views(pool, b)
            works.append(dist.all_gather_into_tensor(whole, mine, group=self.group, async_op=async_op))
        return works


class ShardedPageStep:
    """One data-parallel page step for a ParamBuffer/MasterState pair built on
    the same world-sharded PageLayout (MasterState holds owned pages only)."""

    def __init__(self, buffer, masters, group=None, comm_stream=None):
        if getattr(masters, "_db", False):
            raise ConfigError("a double-buffered state is updated by FusedShardedPageStep's one-pass step")
        lay = buffer.layout
        if masters.layout is not lay and (masters.layout.numels != lay.numels
                                          or masters.layout.world_size != lay.world_size):
            raise ConfigError("buffer and masters must share the sharded page layout")
        self.buffer, self.masters, self.layout = buffer, masters, lay
        self.coll = PageCollectives(lay, group)
        self.group = group
        self.device = buffer.device
        self.comm = comm_stream or torch.cuda.Stream(self.device)
        L = buffer.num_layers
        self.flags = torch.zeros(L, dtype=torch.int32, device=self.device)
        self.sumsq = torch.zeros(L, dtype=torch.float64, device=self.device)
        self._check_chunks = lay.pool_chunks(range(L), "16", owned_only=True)
        self._layers = tuple(range(L))

    def step(self, hyper, *, stream=None, timings: dict | None = None):
        """RS -> check -> flag all-reduce -> prologue -> [Adam(b) || AG(b)].
        Returns the list of layers updated (all layers with pending grads)."""
        buf, ms, lay = self.buffer, self.masters, self.layout
        st = buf._stream(stream)
        L = buf.num_layers
        if any(p == 0 for p in buf._pending):
            raise ConfigError("a DP page step needs a gradient for every layer on every rank")
        gsel = buf._gsel[0]
        if any(x != gsel for x in buf._gsel):
            raise ConfigError("DP page step expects all layers in the same gradient buffer")
        gpool = buf.g16_pool[gsel]
        ev = (lambda: torch.cuda.Event(enable_timing=True)) if timings is not None else None
        marks = {}

        def mark(name):
            if timings is not None:
                e = ev()
                e.record(torch.cuda.current_stream(self.device))
                marks[name] = e

        with torch.cuda.stream(st):
            mark("start")
            self.coll.reduce_scatter(gpool)                      # K6 (in place)
            mark("rs")
            self.flags.zero_()
            self.sumsq.zero_()
            ch = self._check_chunks
            D.check(N.lib().hm_reduce_stats(
                D.ptr(gpool), buf._dt, D.ptr(buf._eng.desc.static(ch)), len(ch),
                D.ptr(self.flags), None, D.ptr(self.sumsq), D.sptr(st)))
            dist.all_reduce(self.flags, op=dist.ReduceOp.MAX, group=self.group)
            if getattr(hyper, "max_norm", 0.0) > 0:
                dist.all_reduce(self.sumsq, op=dist.ReduceOp.SUM, group=self.group)
            mark("check")
        t = UpdateTicket(buf, range(L), flag_of=lambda l: l)
        dgroups, rt, hc = update_prologue(t, ms, hyper, st, flags=self.flags, sumsq=self.sumsq,
                                          lsum=t.lsum(gsel * L))
        eng, lib = ms._eng, N.lib()
        new_p = (buf._psel[0] ^ 1)
        ppool = buf.p16_pool[new_p]
        works = []
        for b in range(lay.num_buckets):
            chunks = lay.adam_chunks(self._layers, "pool", owned_only=True, bucket=b)
            D.check(lib.hm_adam_main(D.ptr(eng.desc.static(chunks)), len(chunks), D.ptr(dgroups),
                                     D.ptr(rt), D.ptr(buf.g16_pool), buf._dt, D.ptr(ms.p32_pool),
                                     D.ptr(ms.m32_pool), D.ptr(ms.v32_pool), D.ptr(buf.p16_pool),
                                     buf._dt, hc, None, D.sptr(st)))
            done = torch.cuda.Event()
            done.record(st)
            self.comm.wait_event(done)
            with torch.cuda.stream(self.comm):
                works += self.coll.all_gather(ppool, buckets=[b], async_op=True)   # K7 (in place)
        with torch.cuda.stream(st):
            mark("adam")
        for w in works:
            w.wait()
        st.wait_stream(self.comm)
        with torch.cuda.stream(st):
            mark("ag")
        t.finish(consumed_flags=False)
        if timings is not None:
            timings["_marks"] = marks
        return list(range(L))


# ---- fused path over symmetric (peer-mapped) page pools ------------------------------

def symmetric_alloc(shape, dtype, device):
    """Allocator for ParamBuffer pools that every rank can map (torch symmetric
    memory: cuMem handles exchanged at rendezvous, optional NVLS multicast)."""
    import torch.distributed._symmetric_memory as symm
    return symm.empty(*shape, dtype=dtype, device=device)


class FusedShardedPageStep:
    """The DP page step with the collectives fused into the page kernels:

        barrier -> hm_dp_reduce_check (owned pages read from every peer's
        gradient pool, f32 sum in rank order, rounded once; flags + norm)
        -> barrier -> hm_dp_flags_merge -> prologue ->
        hm_adam_main_ag (update + publish into every peer's p16 pool)
        -> barrier

    ``mode="p2p"`` moves the bytes with NVLink peer loads/stores;
    ``mode="nvls"`` uses the NVSwitch multicast address: the reduction
    happens in the switch (multimem.ld_reduce) and one store reaches every
    GPU (multimem.st).  The buffer's pools must come from ``symmetric_alloc``.

    With a double-buffered MasterState (``double_buffered=True``) ``step``
    is the ONE-PASS form: a single kernel pulls every rank's gradient of the
    owned pages, reduces, updates into the other state copy and publishes
    into every rank, speculatively; a flag merge then commits the applied
    layers (hm_dp_onepass_update / _finalize / hm_dp_republish_rejected).
    """

    def __init__(self, buffer, masters, group=None, mode: str = "p2p", push: bool = False):
        import torch.distributed._symmetric_memory as symm
        lay = buffer.layout
        if masters.layout.numels != lay.numels or masters.layout.world_size != lay.world_size:
            raise ConfigError("buffer and masters must share the sharded page layout")
        if mode not in ("p2p", "nvls"):
            raise ConfigError(f"unknown fused DP mode {mode!r}")
        self.buffer, self.masters, self.layout = buffer, masters, lay
        self.group = group if group is not None else dist.group.WORLD
        gname = self.group.group_name
        self.device = buffer.device
        L = buffer.num_layers
        self.h_g = symm.rendezvous(buffer.g16_pool, gname)
        self.h_p = symm.rendezvous(buffer.p16_pool, gname)
        self.flags_local = symm.empty(L, dtype=torch.int32, device=self.device)
        self.sumsq_local = symm.empty(L, dtype=torch.float64, device=self.device)
        self.h_f = symm.rendezvous(self.flags_local, gname)
        self.h_s = symm.rendezvous(self.sumsq_local, gname)
        self.flags = torch.zeros(L, dtype=torch.int32, device=self.device)
        self.sumsq = torch.zeros(L, dtype=torch.float64, device=self.device)
        self.n = lay.world_size
        mc_g = int(getattr(self.h_g, "multicast_ptr", 0) or 0)
        mc_p = int(getattr(self.h_p, "multicast_ptr", 0) or 0)
        if mode == "nvls" and (not mc_g or not mc_p):
            raise ConfigError("NVLS multicast is not available on this system (multicast_ptr is 0)")
        self.mode = mode
        self.mc_g, self.mc_p = (mc_g, mc_p) if mode == "nvls" else (0, 0)
        self.g_ptrs = [int(p) for p in self.h_g.buffer_ptrs]
        self.p_ptrs = [int(p) for p in self.h_p.buffer_ptrs]
        self.f_ptrs = [int(p) for p in self.h_f.buffer_ptrs]
        self.s_ptrs = [int(p) for p in self.h_s.buffer_ptrs]
        self._check_chunks = lay.pool_chunks(range(L), "16", owned_only=True)
        self._adam_chunks = lay.adam_chunks(range(L), "pool", owned_only=True)
        # pinned-host / SSD state tier: the state is streamed in step()
        self.host_tier = hasattr(masters, "stream_update")
        # double-buffered state: step() is ONE speculative pass (reduce-scatter
        # + update + all-gather in one kernel, commit after a flag merge)
        self.one_pass = bool(getattr(masters, "_db", False))
        if self.one_pass and mode != "p2p":
            raise ConfigError("the one-pass DP step pulls the gradient with P2P loads (mode='p2p')")
        # push form of the one-pass step: every rank stores the gradient of the
        # pages it does not own into the owner's receive pool (N x the owned
        # 16-bit pages per rank), then the update reads them from local HBM
        self.push = bool(push)
        if self.push:
            if not self.one_pass:
                raise ConfigError("push=True is a form of the one-pass step (double-buffered MasterState)")
            self.recv_pool = symm.empty(lay.world_size * lay.elems_state, dtype=buffer._t16, device=self.device)
            self.h_r = symm.rendezvous(self.recv_pool, gname)
            self.recv_ptrs = torch.tensor([int(p) for p in self.h_r.buffer_ptrs], dtype=torch.int64,
                                          device=self.device)
            self._push_chunks = lay.push_chunks()

    @staticmethod
    def _arr(ptrs):
        import ctypes as C
        return (C.c_uint64 * len(ptrs))(*ptrs)

    def _green_streams(self, reduce_sms: int):
        """Two CUDA green contexts (disjoint SM partitions): ``reduce_sms`` SMs
        for the link-bound reduce, the rest for the HBM-bound update, so the
        two kernels share the GPU by construction.  Streams wrapped as
        torch.cuda streams; cached per partition size."""
        cache = self.__dict__.setdefault("_green", {})
        if reduce_sms not in cache:
            G = torch.cuda.green_contexts
            if not G.SUPPORTED:
                raise ConfigError("this torch build has no CUDA green context support")
            total = torch.cuda.get_device_properties(self.device).multi_processor_count
            rest = (total - reduce_sms) // 8 * 8
            if reduce_sms <= 0 or rest <= 0:
                raise ConfigError(f"bad SM split {reduce_sms}/{total}")
            g_rs = G.GreenContext.create(reduce_sms, self.device.index)
            g_up = G.GreenContext.create(rest, self.device.index)
            rs = torch.cuda.ExternalStream(g_rs.Stream().cuda_stream, device=self.device)
            up = torch.cuda.ExternalStream(g_up.Stream().cuda_stream, device=self.device)
            cache[reduce_sms] = (g_rs, g_up, rs, up)   # keep the contexts alive
        return cache[reduce_sms][2], cache[reduce_sms][3]

    def _group_plan(self, groups: int):
        """Contiguous layer groups with their owned check / adam chunks."""
        cache = self.__dict__.setdefault("_gplans", {})
        if groups not in cache:
            from .lockfree import layer_groups
            lay = self.layout
            plan = []
            for grp in layer_groups(lay.numels, groups):
                t = tuple(grp)
                check = lay.pool_chunks(t, "16", owned_only=True).copy()
                check["slot"] += grp[0]          # flags/sumsq are indexed by global layer
                plan.append((t, check, lay.adam_chunks(t, "pool", owned_only=True)))
            # the reduce stream gets the higher priority: its CTAs are placed
            # first whenever the update kernel of the previous group frees a slot
            cache[groups] = (plan, torch.cuda.Stream(self.device, priority=-1),
                             torch.cuda.Stream(self.device))
        return cache[groups]

    def step_pipelined(self, hyper, groups: int = 4, *, reduce_ctas: int = 0, update_ctas: int = 0,
                       reduce_sms: int = 0, ready=None, stream=None, ag_publish: int = -1,
                       reduce_wide: int = -1, reduce_width: int = -1, results_to=None,
                       timings: dict | None = None):
        """``step`` with the layers cut into contiguous groups and two streams:
        the reduce-scatter + check of group k+1 runs while group k is updated
        and all-gathered.  Every group's flags are merged after its own
        cross-rank barrier, so the whole-layer reject semantics are unchanged.
        Two kernels filling every SM run back to back even on separate
        streams, so ``reduce_ctas > 0`` launches the reduce as a persistent
        grid of that many CTAs on a high-priority stream: the link-bound
        reduce then runs from a few SMs beside the HBM-bound update of the
        previous group; ``update_ctas > 0`` likewise gives the update a
        persistent grid of its own; ``reduce_sms > 0`` instead runs the reduce
        and the update in two CUDA green contexts (disjoint SM partitions).
        ``ready`` (one event per layer group,
        from ``lockfree.ingest``) lets the step start while the gradient is
        still arriving from the host: group k is reduced once its own K3 has
        run on every rank.  With NVLS the RS leg is outbound-heavy (S out, S/N
        in per GPU) and the AG leg inbound-heavy (S/N out, S in), so
        overlapping them moves (1 + 1/N)·S per link direction instead of
        2·(N−1)/N·S.  Launch settings travel with each launch (hm_launch_opts),
        nothing process-wide is changed.  ``results_to`` (pinned host, every
        layer's elements in layer order): right after each group's update,
        this rank's OWNED published pages of the group go back to the host on
        a copy stream — the ranks return disjoint pieces, the whole model
        once per step."""
        buf, ms, lay = self.buffer, self.masters, self.layout
        if self.host_tier:
            raise ConfigError("the layer-group pipeline keeps the state in HBM; a host/SSD-tier "
                              "DP step streams the state in step()")
        if self.one_pass:
            raise ConfigError("a double-buffered state is updated by the one-pass step(): "
                              "its reduce already overlaps the update inside one kernel")
        st = buf._stream(stream)
        L = buf.num_layers
        if any(p == 0 for p in buf._pending):
            raise ConfigError("a DP page step needs a gradient for every layer on every rank")
        gsel, psel = buf._gsel[0], buf._psel[0]
        if any(x != gsel for x in buf._gsel) or any(x != psel for x in buf._psel):
            raise ConfigError("DP page step expects all layers in the same page buffers")
        plan, rs, up = self._group_plan(groups)
        if reduce_sms > 0:   # SM partitions instead of block-scheduler priority
            rs, up = self._green_streams(reduce_sms)
        span_b = lay.elems16 * buf.g16_pool.element_size()
        span = lay.elems16
        lib, eng = N.lib(), ms._eng
        clip = getattr(hyper, "max_norm", 0.0) > 0
        if clip:
            raise ConfigError("global grad-norm clipping needs every group's norm first: use step()")
        rs_opts = D.opts(grid_ctas=int(reduce_ctas), reduce_wide=reduce_wide, reduce_width=reduce_width)
        up_opts = D.opts(grid_ctas=int(update_ctas), ag_publish=ag_publish)
        marks = {}

        def mark(name, s):
            if timings is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(s)
                marks[name] = e

        if ready is None:
            with torch.cuda.stream(st):
                mark("start", st)
                self.flags_local.zero_()
                self.h_g.barrier(channel=0)                      # every rank's gradients are complete
            rs.wait_stream(st)
            up.wait_stream(st)
        else:
            # Gradients still arriving (lockfree.ingest): group k is reduced as
            # soon as its own K3 is done here and on every peer (per-group
            # barrier below); the reduce stream only has to follow the end of
            # the previous step, not the K3s queued behind it on ``st``.
            if len(ready) != len(plan):
                raise ConfigError(f"{len(ready)} ready events for {len(plan)} layer groups")
            last = self.__dict__.get("_last_done")
            if last is not None:
                rs.wait_event(last)
                up.wait_event(last)
            with torch.cuda.stream(rs):
                mark("start", rs)
                self.flags_local.zero_()
        gp = self._arr([p + gsel * span_b for p in self.g_ptrs])
        mc = self.mc_g + gsel * span_b if self.mc_g else None
        t = UpdateTicket(buf, range(L), flag_of=lambda l: l)
        bc, bc_len = ms._bias(hyper, range(L))
        hc = D.hyper_c(hyper)
        rts = self.__dict__.setdefault("_rts", {})
        d2h = starts = None
        if results_to is not None:
            from .lockfree import _publish_to_host
            d2h = self.__dict__.setdefault("_d2h", torch.cuda.Stream(self.device))
            starts = self.__dict__.setdefault("_starts", np.cumsum([0] + lay.numels[:-1]))
        gmarks = []

        def gmark(s):
            if timings is None:
                return None
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            return e

        for k, (grp, check, adam) in enumerate(plan):
            first, n = grp[0], len(grp)
            with torch.cuda.stream(rs):
                if ready is not None:
                    rs.wait_event(ready[k])
                    self.h_g.barrier(channel=0)                  # group k landed on every rank
                r0 = gmark(rs)
                D.check(lib.hm_dp_reduce_check(gp, self.n, mc, D.ptr(buf.g16_pool[gsel]), buf._dt,
                                               D.ptr(eng.desc.static(check)), len(check),
                                               D.ptr(self.flags_local), None, rs_opts, D.sptr(rs)))
                r1 = gmark(rs)
                self.h_f.barrier(channel=1)                      # group k's flags visible everywhere
                done = torch.cuda.Event()
                done.record(rs)
            up.wait_event(done)
            with torch.cuda.stream(up):
                u0 = gmark(up)
                D.check(lib.hm_dp_flags_merge(self._arr([p + 4 * first for p in self.f_ptrs]), None,
                                              self.n, n, D.ptr(self.flags) + 4 * first, None, D.sptr(up)))
                rows = t.groups[first:first + n].copy()
                rows["flag"] -= first                            # the merged flags of this group start at 0
                rows["group"] = grp
                dgroups = eng.desc.table(rows, up)
                if (k, n) not in rts:
                    rts[(k, n)] = torch.empty(n * N.GROUP_RT_BYTES, dtype=torch.uint8, device=self.device)
                rt = rts[(k, n)]
                ledger_out = t.ledger_out + 16 * first if t.ledger_out else None
                D.check(lib.hm_adam_prologue(D.ptr(dgroups), n, D.ptr(rt), hc, D.ptr(bc), bc_len, 0,
                                             D.ptr(ms._steps), D.ptr(ms._applied),
                                             D.ptr(self.flags) + 4 * first, None, 1,
                                             t.lsum(gsel * L + first) or None, ledger_out, D.sptr(up)))
                D.check(lib.hm_adam_main_ag(D.ptr(eng.desc.static(adam)), len(adam), D.ptr(dgroups),
                                            D.ptr(rt), D.ptr(buf.g16_pool), buf._dt, D.ptr(ms.p32_pool),
                                            D.ptr(ms.m32_pool), D.ptr(ms.v32_pool), self._arr(self.p_ptrs),
                                            self.n, self.mc_p if self.mc_p else None, buf._dt, hc, up_opts,
                                            D.sptr(up)))
                gmarks.append((r0, r1, u0, gmark(up)))
                if d2h is not None:
                    _publish_to_host(buf, grp, results_to, starts, up, d2h, owned_only=True, pbuf=psel ^ 1)
        mark("rs", rs)
        st.wait_stream(rs)
        st.wait_stream(up)
        if d2h is not None:
            st.wait_stream(d2h)
        with torch.cuda.stream(st):
            mark("adam", st)
            self.h_p.barrier(channel=2)                          # published pages landed everywhere
            mark("ag", st)
            done = torch.cuda.Event()
            done.record(st)
            self._last_done = done
        t.finish(consumed_flags=False)
        if timings is not None:
            timings["_marks"] = marks
            timings["_groups"] = gmarks     # per group: reduce start/end, update start/end
        return list(range(L))

    def step(self, hyper, *, stream=None, ag_publish: int = -1, reduce_wide: int = -1,
             reduce_width: int = -1, ready=None, timings: dict | None = None):
        """barrier -> reduce-scatter + check -> barrier -> flag merge ->
        prologue -> update with the all-gather epilogue -> barrier.  With a
        host (or SSD) state tier the update streams the owned state pages
        through HBM staging (the tier's pipeline) between the reduce and the
        all-gather: each rank moves 24 B x its owned params over its own PCIe
        link, the 16-bit pages travel over NVLink as usual.  ``ready`` (one-pass
        step only; one event per layer group from ``lockfree.ingest``): the
        one-pass kernel runs group by group as each group's gradient lands on
        every rank — the commit waits for all of them anyway."""
        buf, ms, lay = self.buffer, self.masters, self.layout
        st = buf._stream(stream)
        if ready is not None and not self.one_pass:
            raise ConfigError("step(ready=...) streams the one-pass step; use step_pipelined(ready=...)")
        L = buf.num_layers
        if any(p == 0 for p in buf._pending):
            raise ConfigError("a DP page step needs a gradient for every layer on every rank")
        gsel, psel = buf._gsel[0], buf._psel[0]
        if any(x != gsel for x in buf._gsel) or any(x != psel for x in buf._psel):
            raise ConfigError("DP page step expects all layers in the same page buffers")
        span_b = lay.elems16 * buf.g16_pool.element_size()
        marks = {}

        def mark(name):
            if timings is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                marks[name] = e

        lib, eng = N.lib(), ms._eng
        clip = getattr(hyper, "max_norm", 0.0) > 0
        if self.one_pass:
            if clip:
                raise ConfigError("global grad-norm clipping needs the norm before the update: "
                                  "the one-pass step cannot clip (use a single-buffered state)")
            return self._step_one_pass(hyper, st, mark, marks, timings, reduce_width, ready)
        with torch.cuda.stream(st):
            mark("start")
            self.flags_local.zero_()
            if clip:
                self.sumsq_local.zero_()
            self.h_g.barrier(channel=0)                          # every rank's gradients are complete
            mark("rs_start")
            gp = self._arr([p + gsel * span_b for p in self.g_ptrs])
            mc = self.mc_g + gsel * span_b if self.mc_g else None
            ch = self._check_chunks
            D.check(lib.hm_dp_reduce_check(gp, self.n, mc, D.ptr(buf.g16_pool[gsel]), buf._dt,
                                           D.ptr(eng.desc.static(ch)), len(ch), D.ptr(self.flags_local),
                                           D.ptr(self.sumsq_local) if clip else None,
                                           D.opts(reduce_wide=reduce_wide, reduce_width=reduce_width),
                                           D.sptr(st)))
            mark("rs")
            self.h_f.barrier(channel=0)                          # flags / norms visible to all
            D.check(lib.hm_dp_flags_merge(self._arr(self.f_ptrs), self._arr(self.s_ptrs) if clip else None,
                                          self.n, L, D.ptr(self.flags), D.ptr(self.sumsq) if clip else None,
                                          D.sptr(st)))
            mark("check")
        t = UpdateTicket(buf, range(L), flag_of=lambda l: l)
        for l in range(L):
            if not self.host_tier:
                ms._prepub[l] = None
        dgroups, rt, hc = update_prologue(t, ms, hyper, st, flags=self.flags, sumsq=self.sumsq,
                                          lsum=t.lsum(gsel * L))
        peers = self._arr(self.p_ptrs)
        mcp = self.mc_p if self.mc_p else None
        up_opts = D.opts(ag_publish=ag_publish)

        def launch(chunks, planes):
            D.check(lib.hm_adam_main_ag(D.ptr(eng.desc.static(chunks)), len(chunks), D.ptr(dgroups),
                                        D.ptr(rt), D.ptr(buf.g16_pool), buf._dt, *planes, peers, self.n,
                                        mcp, buf._dt, hc, up_opts, D.sptr(st)))

        if self.host_tier:
            ms.stream_update(range(L), st, lambda chunks, stage: launch(chunks, ms.planes(stage)))
        else:
            launch(self._adam_chunks, (D.ptr(ms.p32_pool), D.ptr(ms.m32_pool), D.ptr(ms.v32_pool)))
        with torch.cuda.stream(st):
            mark("adam")
            self.h_p.barrier(channel=0)                          # published pages landed everywhere
            mark("ag")
            done = torch.cuda.Event()
            done.record(st)
            self._last_done = done
        t.finish(consumed_flags=False)
        if timings is not None:
            timings["_marks"] = marks
        return list(range(L))

    def _step_one_pass(self, hyper, st, mark, marks, timings, reduce_width=-1, ready=None):
        """barrier -> speculative prologue (on a copy of the step counters) ->
        hm_dp_onepass_update (pull every rank's gradient of the owned pages,
        reduce, update into the other state copy, publish to every rank) ->
        barrier -> hm_dp_onepass_finalize (merge the flags, commit steps and
        state copies of applied layers) -> republish rejected layers ->
        barrier.  One data-path kernel; the reduced gradient is never written."""
        buf, ms, lay = self.buffer, self.masters, self.layout
        L = buf.num_layers
        gsel = buf._gsel[0]
        lib, eng = N.lib(), ms._eng
        with torch.cuda.stream(st):
            mark("start")
            self.flags_local.zero_()
            ms._steps_spec.copy_(ms._steps)
            if ready is None:
                self.h_g.barrier(channel=0)                      # every rank's gradients are complete
            mark("rs_start")
            mark("rs")
            mark("check")
        t = UpdateTicket(buf, range(L), flag_of=lambda l: l)
        for l in range(L):
            ms._prepub[l] = None
        dgroups = eng.desc.table(t.groups, st)
        rt = eng.rt_scratch(L, st)
        bc, bc_len = ms._bias(hyper, range(L))
        hc = D.hyper_c(hyper)
        # speculative: every layer assumed finite, steps advanced in the copy;
        # the take record of the ledger is written here, its applied column
        # by the finalize
        D.check(lib.hm_adam_prologue(D.ptr(dgroups), L, D.ptr(rt), hc, D.ptr(bc), bc_len, 0,
                                     D.ptr(ms._steps_spec), None, None, None, 1,
                                     t.lsum(gsel * L) or None, t.ledger_out or None, D.sptr(st)))
        ac = self._adam_chunks
        gp, pp = self._arr(self.g_ptrs), self._arr(self.p_ptrs)
        es = lay.elems_state
        if ready is None:
            parts = [(None, ac)]
        else:   # one launch per layer group, each once its gradient landed on every rank
            cache = self.__dict__.setdefault("_onepass_parts", {})
            if len(ready) not in cache:
                from .lockfree import layer_groups
                slots = ac["slot"]
                cache[len(ready)] = [ac[(slots >= grp[0]) & (slots <= grp[-1])].copy()
                                     for grp in layer_groups(lay.numels, len(ready))]
            parts = list(zip(ready, cache[len(ready)]))
        if self.push:
            # the push form exchanges the whole gradient before any update:
            # every group must have landed (one wait per group, then one barrier)
            for ev, _chunks in parts:
                if ev is not None:
                    st.wait_event(ev)
            with torch.cuda.stream(st):
                if ready is not None:
                    self.h_g.barrier(channel=0)
                D.check(lib.hm_dp_push_grad(D.ptr(eng.desc.static(self._push_chunks)), len(self._push_chunks),
                                            D.ptr(buf.g16_pool[gsel]), D.ptr(self.recv_ptrs),
                                            lay.rank * es, D.sptr(st)))
                self.h_r.barrier(channel=0)                      # every rank's shares landed
            D.check(lib.hm_dp_onepass_recv_update(
                D.ptr(eng.desc.static(ac)), len(ac), D.ptr(dgroups), D.ptr(rt), D.ptr(ms._state_sel), es,
                D.ptr(buf.g16_pool), D.ptr(self.recv_pool), es, lay.rank, self.n, pp, self.n, buf._dt,
                D.ptr(ms.p32_pool), D.ptr(ms.m32_pool), D.ptr(ms.v32_pool), D.ptr(self.flags_local), hc,
                D.sptr(st)))
            parts = []
        for ev, chunks in parts:
            if ev is not None:
                st.wait_event(ev)
                with torch.cuda.stream(st):
                    self.h_g.barrier(channel=0)                  # this group landed on every rank
            D.check(lib.hm_dp_onepass_update(D.ptr(eng.desc.static(chunks)), len(chunks), D.ptr(dgroups),
                                             D.ptr(rt), D.ptr(ms._state_sel), es, gp, pp, self.n, buf._dt,
                                             D.ptr(ms.p32_pool), D.ptr(ms.m32_pool), D.ptr(ms.v32_pool),
                                             D.ptr(self.flags_local), hc, D.opts(reduce_width=reduce_width),
                                             D.sptr(st)))
        with torch.cuda.stream(st):
            self.h_f.barrier(channel=0)                          # every rank's flags are final
            D.check(lib.hm_dp_onepass_finalize(self._arr(self.f_ptrs), self.n, L, D.ptr(ms._steps),
                                               D.ptr(ms._steps_spec), D.ptr(ms._state_sel),
                                               D.ptr(ms._applied), t.ledger_out or None, D.sptr(st)))
            D.check(lib.hm_dp_republish_rejected(D.ptr(eng.desc.static(ac)), len(ac), D.ptr(dgroups),
                                                 D.ptr(ms._applied), D.ptr(ms._state_sel), es,
                                                 D.ptr(ms.p32_pool), pp, self.n, buf._dt, D.sptr(st)))
            mark("adam")
            self.h_p.barrier(channel=0)                          # published pages landed everywhere
            mark("ag")
            done = torch.cuda.Event()
            done.record(st)
            self._last_done = done
        t.finish(consumed_flags=False)
        if timings is not None:
            timings["_marks"] = marks
        return list(range(L))
