"""Data-parallel page sharding: gradient reduce-scatter and parameter
all-gather over the 16-bit page pools, one process per GPU.

Ownership is the reference's ``ShardingModel``: ``owner(page) = page % N``
(hiermem/scheduler.py:59-76), ZeRO-3 style at page granularity (PAPER.md:305,
685).  The reference only *models* the collectives — an all_gather task per
page costed as ``lat + page*(N-1)/N / bw`` (hiermem/simengine.py:255-257) and
no gradient reduce-scatter at all (SPEC.md:348 lists it as future work).
Here they are real NCCL collectives over NVLink/NVSwitch on the page pools:

* the 16-bit pools are laid out bucket-major, rank-major inside a bucket
  (layout.py), so bucket b is ONE contiguous buffer and rank r's owned pages
  are its r-th block: ``reduce_scatter_tensor`` / ``all_gather_into_tensor``
  run in place with no packing copies;
* the DP step is  RS(all buckets) -> finite/norm check of the owned reduced
  pages -> all-reduce of the per-layer flags (tiny) -> ONE prologue ->
  for each bucket: page-Adam(b) on the compute stream || AG(b) on the comm
  stream once Adam(b) is done — the transfer of bucket b overlaps the
  update of bucket b+1.

``PageCollectives`` is device-agnostic (it runs on CPU tensors under gloo in
the tests); ``ShardedPageStep`` drives the CUDA kernels.
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
        counts, newest = [], []
        for l in range(L):
            _, c, n = buf._hand_over(l, st)
            counts.append(c)
            newest.append(n)
        span = lay.elems16
        rows = [(gsel * span, (buf._psel[l] ^ 1) * span, l, l) for l in range(L)]
        groups = np.zeros(L, dtype=N.GROUP_LAUNCH)
        for i, r in enumerate(rows):
            groups[i] = r
        eng = ms._eng
        dgroups = eng.desc.table(groups)
        rt = eng.rt_scratch(L)
        bc, bc_len = ms._bias(hyper, range(L))
        hc = D.hyper_c(hyper)
        lib = N.lib()
        D.check(lib.hm_adam_prologue(D.ptr(dgroups), L, D.ptr(rt), hc, D.ptr(bc), bc_len, 0,
                                     D.ptr(ms._steps), D.ptr(ms._applied), D.ptr(self.flags),
                                     D.ptr(self.sumsq), 1, D.sptr(st)))
        new_p = (buf._psel[0] ^ 1)
        ppool = buf.p16_pool[new_p]
        works = []
        for b in range(lay.num_buckets):
            chunks = lay.adam_chunks(self._layers, "pool", owned_only=True, bucket=b)
            D.check(lib.hm_adam_main(D.ptr(eng.desc.static(chunks)), len(chunks), D.ptr(dgroups),
                                     D.ptr(rt), D.ptr(buf.g16_pool), buf._dt, D.ptr(ms.p32_pool),
                                     D.ptr(ms.m32_pool), D.ptr(ms.v32_pool), D.ptr(buf.p16_pool),
                                     buf._dt, hc, D.sptr(st)))
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
        for l in range(L):
            buf._psel[l] ^= 1
            buf._version[l] += 1
            buf._applied_iter[l] = newest[l]
        if timings is not None:
            timings["_marks"] = marks
        return list(range(L))
