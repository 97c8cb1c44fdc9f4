"""Page layout: from the page table to device pool addresses and kernel
descriptors.

One ``PageLayout`` places a list of tensors ("layers" in the sense of
hiermem/lockfree.py's MasterState/ParamBuffer lists) as ``param16`` specs
into a GPU page pool with the reference packing policy (PageManager.allocate,
hiermem/pagemem.py:233-283), then serves every pool that shares that
element-indexed page table:

* 16-bit pools (gradient g16, published p16): ``P`` pages of ``E`` elements;
* fp32 state pools (p32, m32, v32): only the pages this rank owns.

Data-parallel ownership is the reference's round robin ``owner(p) = p % N``
(hiermem/scheduler.py:72-76).  The 16-bit pools use a bucketed rank-major
slot order so that one bucket of ``N*K`` pages is one contiguous buffer in
which rank r's ``K`` owned pages are the r-th contiguous block — exactly the
in-place layout of ncclReduceScatter / ncclAllGather:

    bucket b = p // (N*K);  j = (p % (N*K)) // N;  r = p % N
    slot16(p) = b*N*K + r*K + j            local state slot = p // N

With N = 1 both maps are the identity.
"""
from __future__ import annotations

from dataclasses import dataclass
import numpy as np

from . import _native as N
from .pagemem import PAGE_BYTES_DEFAULT, PageManager
from .workloads import TensorSpec

CHUNK = 4096  # HM_ADAM_CHUNK
VEC = 8


def _split(off: int, n: int):
    """Split [off, off+n) into kernel units: an unaligned head (< 8), full
    4096-element aligned chunks, an aligned remainder that is a multiple of 8,
    and a ragged tail (< 8).  Yields (start_delta, count)."""
    pos = 0
    head = (-off) % VEC
    if head:
        h = min(head, n)
        yield 0, h
        pos = h
    while n - pos >= CHUNK:
        yield pos, CHUNK
        pos += CHUNK
    rest = n - pos
    body = rest - rest % VEC
    if body:
        yield pos, body
        pos += body
    if n - pos:
        yield pos, n - pos


@dataclass(frozen=True)
class Segment:
    layer: int
    page: int        # page id
    off: int         # element offset inside the page
    n: int           # elements
    pos: int         # element offset inside the tensor


class PageLayout:
    def __init__(self, numels, page_bytes: int = PAGE_BYTES_DEFAULT, world_size: int = 1,
                 rank: int = 0, bucket_pages: int | None = None, names=None):
        numels = [int(n) for n in numels]
        if not numels or min(numels) <= 0:
            from .errors import ConfigError
            raise ConfigError("PageLayout needs at least one non-empty tensor")
        self.numels = numels
        self.page_bytes = int(page_bytes)
        self.E = self.page_bytes // 2  # elements per page (16-bit page)
        self.world_size = int(world_size)
        self.rank = int(rank)
        need = sum(-(-2 * n // self.page_bytes) for n in numels)
        self.manager = PageManager([("GPU", need * self.page_bytes, self.page_bytes)])
        self.tensors = []
        for i, n in enumerate(numels):
            name = names[i] if names else f"layer{i}"
            self.tensors.append(self.manager.allocate(TensorSpec(name, "param16", 2 * n, i), "GPU"))
        used = max(max(t.page_list) for t in self.tensors) + 1
        Nw = self.world_size
        if bucket_pages is None:
            bucket_pages = -(-used // Nw)  # one bucket: fully rank-major
        self.K = max(1, int(bucket_pages))
        span = Nw * self.K
        self.num_buckets = -(-used // span)
        self.P = self.num_buckets * span          # padded page count of 16-bit pools
        self.P_local = self.P // Nw               # pages of the state pools on this rank
        self.used_pages = used
        self.segments: list[list[Segment]] = []
        for i, t in enumerate(self.tensors):
            segs, pos = [], 0
            for pid, boff, nbytes in t.segments():
                segs.append(Segment(i, pid, boff // 2, nbytes // 2, pos))
                pos += nbytes // 2
            self.segments.append(segs)

    # -- address maps ------------------------------------------------------
    @property
    def elems16(self) -> int:
        return self.P * self.E

    @property
    def elems_state(self) -> int:
        return self.P_local * self.E

    def owner(self, pid: int) -> int:
        return pid % self.world_size

    def slot16(self, pid: int) -> int:
        Nw, K = self.world_size, self.K
        b, q = divmod(pid, Nw * K)
        return b * Nw * K + (pid % Nw) * K + q // Nw

    def slot_state(self, pid: int) -> int:
        return pid // self.world_size

    def owned(self, seg: Segment) -> bool:
        return self.owner(seg.page) == self.rank

    def owned_numel(self, layers=None) -> int:
        layers = range(len(self.numels)) if layers is None else layers
        return sum(s.n for l in layers for s in self.segments[l] if self.owned(s))

    def bucket_slots(self, b: int) -> tuple[int, int]:
        """[first, end) 16-bit pool slots of bucket b."""
        span = self.world_size * self.K
        return b * span, (b + 1) * span

    # -- kernel descriptors --------------------------------------------------
    def bucket_of(self, pid: int) -> int:
        return pid // (self.world_size * self.K)

    def adam_chunks(self, layers, g_source: str = "pool", owned_only: bool = True,
                    bucket: int | None = None) -> np.ndarray:
        """hm_adam_chunk array for the given layers (slot = index in ``layers``).
        g_source="pool": gradient read from the 16-bit pool (fused sweep);
        "tensor": from a contiguous per-layer gradient tensor (update_layer).
        bucket: restrict to the pages of one all-gather bucket."""
        return _adam_chunks(self, tuple(layers), g_source, owned_only, bucket)

    def seg_chunks(self, layer: int, pool: str, owned_only: bool = False, slot: int = 0,
                   reverse: bool = False) -> np.ndarray:
        """hm_seg_chunk array mapping a contiguous tensor to pool pages.
        pool="16": the 16-bit pools; "state": the fp32 state pools.
        reverse=False: src = tensor, dst = pool (pack); True: unpack."""
        return _seg_chunks(self, layer, pool, owned_only, slot, reverse)

    def push_chunks(self) -> np.ndarray:
        """Units of every page another rank owns, routed to its owner's
        receive pool (the push form of the one-pass DP step)."""
        return _push_chunks(self)

    def adam_tensor_pos(self, layer: int) -> np.ndarray:
        """uint64 tensor offset of every unit of ``adam_chunks([layer])``
        (owned units, same order): where hm_adam_layer stores the new p32."""
        cache = self.__dict__.setdefault("_tpos_cache", {})
        if layer not in cache:
            cache[layer] = _unit_arrays(self, layer, True)[2].astype(np.uint64)
        return cache[layer]

    def pool_chunks(self, layers, pool: str = "16", owned_only: bool = True) -> np.ndarray:
        """hm_seg_chunk over pool segments with src == dst == pool offsets and
        slot = index in ``layers`` (reductions / casts done in place)."""
        return _pool_chunks(self, tuple(layers), pool, owned_only)


def _unit_arrays(lay: PageLayout, layer: int, owned_only: bool, bucket: int | None = None):
    """Per layer: (off16, off_state, tensor_pos, n) int64 arrays of kernel units,
    vectorised per segment (few segments, many 4096-element chunks)."""
    cache = lay.__dict__.setdefault("_unit_cache", {})
    key = (layer, owned_only, bucket)
    if key in cache:
        return cache[key]
    o16s, osts, poss, ns = [], [], [], []
    for s in lay.segments[layer]:
        if owned_only and not lay.owned(s):
            continue
        if bucket is not None and lay.bucket_of(s.page) != bucket:
            continue
        base16 = lay.slot16(s.page) * lay.E + s.off
        basest = lay.slot_state(s.page) * lay.E + s.off
        d_list, n_list = [], []
        head = (-s.off) % VEC
        pos = 0
        if head:
            h = min(head, s.n)
            d_list.append(np.array([0]))
            n_list.append(np.array([h]))
            pos = h
        nfull = (s.n - pos) // CHUNK
        if nfull:
            d_list.append(pos + CHUNK * np.arange(nfull))
            n_list.append(np.full(nfull, CHUNK))
            pos += nfull * CHUNK
        rest = s.n - pos
        body = rest - rest % VEC
        if body:
            d_list.append(np.array([pos]))
            n_list.append(np.array([body]))
            pos += body
        if s.n - pos:
            d_list.append(np.array([pos]))
            n_list.append(np.array([s.n - pos]))
        d = np.concatenate(d_list).astype(np.int64)
        n = np.concatenate(n_list).astype(np.int64)
        o16s.append(base16 + d)
        osts.append(basest + d)
        poss.append(s.pos + d)
        ns.append(n)
    if ns:
        out = tuple(np.concatenate(a) for a in (o16s, osts, poss, ns))
    else:
        out = tuple(np.zeros(0, np.int64) for _ in range(4))
    cache[key] = out
    return out


def _push_chunks(lay: PageLayout) -> np.ndarray:
    """hm_seg_chunk array of every page this rank does NOT own: src_off =
    16-bit pool offset here, dst_off = state-slot offset on the owner,
    slot = owner (hm_dp_push_grad)."""
    cache = lay.__dict__.setdefault("_push_cache", {})
    if "all" in cache:
        return cache["all"]
    parts = []
    for l in range(len(lay.numels)):
        for s in lay.segments[l]:
            if lay.owned(s):
                continue
            base16 = lay.slot16(s.page) * lay.E + s.off
            basest = lay.slot_state(s.page) * lay.E + s.off
            for d, n in _split(s.off, s.n):
                parts.append((base16 + d, basest + d, n, lay.owner(s.page)))
    arr = np.zeros(len(parts), dtype=N.SEG_CHUNK)
    if parts:
        a = np.asarray(parts, dtype=np.int64)
        arr["src_off"], arr["dst_off"], arr["n"], arr["slot"] = a[:, 0], a[:, 1], a[:, 2], a[:, 3]
    cache["all"] = arr
    return arr


def _adam_chunks(lay: PageLayout, layers: tuple, g_source: str, owned_only: bool,
                 bucket: int | None = None) -> np.ndarray:
    cache = lay.__dict__.setdefault("_adam_cache", {})
    key = (layers, g_source, owned_only, bucket)
    if key in cache:
        return cache[key]
    parts = []
    for slot, l in enumerate(layers):
        o16, ost, pos, n = _unit_arrays(lay, l, owned_only, bucket)
        a = np.empty(len(n), dtype=N.ADAM_CHUNK)
        a["g_off"] = pos if g_source == "tensor" else o16
        a["s_off"] = ost
        a["p_off"] = o16
        a["n"] = n
        a["slot"] = slot
        parts.append(a)
    arr = np.concatenate(parts) if parts else np.zeros(0, dtype=N.ADAM_CHUNK)
    cache[key] = arr
    return arr


def _seg_chunks(lay: PageLayout, layer: int, pool: str, owned_only: bool, slot: int,
                reverse: bool) -> np.ndarray:
    cache = lay.__dict__.setdefault("_seg_cache", {})
    key = (layer, pool, owned_only, slot, reverse)
    if key in cache:
        return cache[key]
    o16, ost, pos, n = _unit_arrays(lay, layer, owned_only)
    p = o16 if pool == "16" else ost
    arr = np.empty(len(n), dtype=N.SEG_CHUNK)
    arr["src_off"], arr["dst_off"] = (p, pos) if reverse else (pos, p)
    arr["n"] = n
    arr["slot"] = slot
    cache[key] = arr
    return arr


def _pool_chunks(lay: PageLayout, layers: tuple, pool: str, owned_only: bool) -> np.ndarray:
    cache = lay.__dict__.setdefault("_pool_cache", {})
    key = (layers, pool, owned_only)
    if key in cache:
        return cache[key]
    parts = []
    for slot, l in enumerate(layers):
        o16, ost, pos, n = _unit_arrays(lay, l, owned_only)
        p = o16 if pool == "16" else ost
        a = np.empty(len(n), dtype=N.SEG_CHUNK)
        a["src_off"] = p
        a["dst_off"] = p
        a["n"] = n
        a["slot"] = slot
        parts.append(a)
    arr = np.concatenate(parts) if parts else np.zeros(0, dtype=N.SEG_CHUNK)
    cache[key] = arr
    return arr
