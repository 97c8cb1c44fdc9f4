"""Drop-in page pools: the API of hiermem/pagemem.py backed by the native
page table of libhm_page.so (csrc/pagetable.cpp).

Names, arguments, return values, exceptions and ``state_dict`` output are
those of the reference (hiermem/pagemem.py:23-464); tests/test_pagetable.py
compares ``state_dict`` byte-for-byte against the reference on its own
randomized operation sequences.  Differences are additive only:

* allocation and tail sharing are O(log P) in C++ instead of O(P) scans;
* every occupant also has a byte ``offset`` inside its page, and
  ``ManagedTensor.segments()`` returns (page_id, offset, bytes) triples — the
  physical placement the device page pools (``layout.py``) are built from.
"""
from __future__ import annotations

import ctypes as C
from collections.abc import Mapping
from dataclasses import dataclass
from enum import Enum

from . import _native as N
from .errors import ConfigError

PAGE_BYTES_DEFAULT = 4 * 2**20
MIN_PAGE_BYTES = 64 * 2**10
NOT_READY = "NOT_READY"


class Tier(Enum):
    GPU = 0
    CPU = 1
    SSD = 2

    @classmethod
    def parse(cls, value: "Tier | str | int") -> "Tier":
        if isinstance(value, Tier):
            return value
        if isinstance(value, str):
            try:
                return cls[value.upper()]
            except KeyError:
                raise ConfigError(f"unknown tier {value!r}") from None
        return cls(value)


@dataclass
class Occupant:
    tensor_id: int
    bytes: int
    shareable: bool
    offset: int = 0  # byte offset inside the page (not modeled by the reference)


@dataclass
class PoolStats:
    allocations: int = 0
    releases: int = 0
    moves_in: int = 0
    moves_out: int = 0
    peak_allocated_pages: int = 0


@dataclass(frozen=True)
class TransferDescriptor:
    bytes: int
    src_tier: Tier
    dst_tier: Tier
    page_id: int
    new_page_id: int


class _Table:
    """Owner of one native hm_pagetable handle."""

    def __init__(self):
        h = C.c_void_p()
        N.check(N.lib().hm_pt_create(C.byref(h)))
        self.h = h
        self._lib = N.lib()

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self._lib.hm_pt_destroy(h)
            self.h = None

    def call(self, name, *args):
        N.check(getattr(self._lib, name)(self.h, *args))


class Page:
    """Live view of one page (hiermem/pagemem.py:55-68)."""

    __slots__ = ("_t", "page_id")

    def __init__(self, table: _Table, page_id: int):
        self._t = table
        self.page_id = page_id

    def _info(self):
        out = (C.c_int64 * 11)()
        self._t.call("hm_pt_page_info", C.c_int64(self.page_id), out)
        return list(out)

    @property
    def tier(self) -> Tier:
        return Tier(self._info()[0])

    @property
    def total_bytes(self) -> int:
        return self._info()[1]

    @property
    def occupants(self) -> list[Occupant]:
        v = self._info()
        return [Occupant(v[3 + 4 * i], v[4 + 4 * i], bool(v[5 + 4 * i]), v[6 + 4 * i])
                for i in range(v[2])]

    @property
    def occupied_bytes(self) -> int:
        v = self._info()
        return sum(v[4 + 4 * i] for i in range(v[2]))

    @property
    def available_bytes(self) -> int:
        v = self._info()
        return v[1] - sum(v[4 + 4 * i] for i in range(v[2]))

    def __eq__(self, other):
        return isinstance(other, Page) and other._t is self._t and other.page_id == self.page_id

    def __hash__(self):
        return hash((id(self._t), self.page_id))

    def __repr__(self):
        return f"Page(page_id={self.page_id}, tier={self.tier}, occupants={self.occupants})"


class _PagesView(Mapping):
    def __init__(self, pool: "TierPool"):
        self._pool = pool

    def __getitem__(self, pid):
        p = self._pool
        if not isinstance(pid, int) or not (p.first_page_id <= pid < p.first_page_id + p.num_pages):
            raise KeyError(pid)
        return Page(p._t, pid)

    def __iter__(self):
        p = self._pool
        return iter(range(p.first_page_id, p.first_page_id + p.num_pages))

    def __len__(self):
        return self._pool.num_pages

    def __contains__(self, pid):
        p = self._pool
        return isinstance(pid, int) and p.first_page_id <= pid < p.first_page_id + p.num_pages


class TierPool:
    """Pre-allocated pool of fixed-size pages for one memory tier
    (hiermem/pagemem.py:111-165)."""

    def __init__(self, tier, capacity_bytes: int, page_bytes: int, first_page_id: int = 0,
                 *, _table: _Table | None = None):
        tier = Tier.parse(tier)
        if _table is None:
            _table = _Table()
            _table.call("hm_pt_add_pool", int(tier.value), C.c_int64(capacity_bytes),
                        C.c_int64(page_bytes), C.c_int64(first_page_id))
        self._t = _table
        self.tier = tier
        info = self._info()
        self.capacity_bytes = info[1]
        self.page_bytes = info[2]
        self.first_page_id = info[3]
        self._num = info[4]
        self._manager = None

    def _index(self) -> int:
        lib = self._t._lib
        for i in range(lib.hm_pt_num_pools(self._t.h)):
            out = (C.c_int64 * 12)()
            N.check(lib.hm_pt_pool_info(self._t.h, i, out))
            if out[0] == self.tier.value:
                return i
        raise ConfigError(f"no pool configured for tier {self.tier.name}")

    def _info(self):
        out = (C.c_int64 * 12)()
        N.check(self._t._lib.hm_pt_pool_info(self._t.h, self._index(), out))
        return list(out)

    @property
    def num_pages(self) -> int:
        return self._num

    @property
    def free_page_count(self) -> int:
        return self._info()[5]

    @property
    def allocated_page_count(self) -> int:
        return self._num - self.free_page_count

    @property
    def pages(self) -> Mapping:
        return _PagesView(self)

    @property
    def stats(self) -> PoolStats:
        v = self._info()
        return PoolStats(v[6], v[7], v[8], v[9], v[10])

    def occupied_bytes(self) -> int:
        return self._info()[11]

    def allocated_page_ids(self) -> list[int]:
        lib = self._t._lib
        n = lib.hm_pt_allocated_pages(self._t.h, self.tier.value, None, 0)
        buf = N.i64_buf(n)
        lib.hm_pt_allocated_pages(self._t.h, self.tier.value, buf, n)
        return list(buf[:n])

    def allocated_pages(self) -> list[Page]:
        return [Page(self._t, pid) for pid in self.allocated_page_ids()]

    def free_page_ids(self) -> list[int]:
        lib = self._t._lib
        n = lib.hm_pt_free_pages(self._t.h, self.tier.value, None, 0)
        buf = N.i64_buf(n)
        lib.hm_pt_free_pages(self._t.h, self.tier.value, buf, n)
        return list(buf[:n])


def pool_init(tier, capacity_bytes: int, page_bytes: int = PAGE_BYTES_DEFAULT,
              first_page_id: int = 0) -> TierPool:
    """Create a tier pool with all pages free and deterministic page ids
    (hiermem/pagemem.py:168-171)."""
    return TierPool(Tier.parse(tier), capacity_bytes, page_bytes, first_page_id)


def fragmentation(pool: TierPool) -> float:
    """1 - occupied/allocated-page bytes; 0.0 for an empty pool
    (hiermem/pagemem.py:174-181)."""
    info = pool._info()
    allocated = info[4] - info[5]
    if not allocated:
        return 0.0
    total = allocated * pool.page_bytes
    return 1.0 - info[11] / total


def _dtype_for(kind: str) -> str:
    return "fp32" if kind == "optim32" else "fp16"


class ManagedTensor:
    """Tensor record (hiermem/pagemem.py:71-90); ``page_list`` and ``tier``
    are live views of the native table."""

    def __init__(self, tensor_id: int, dtype: str, shape: tuple, spec, manager: "PageManager"):
        self.tensor_id = tensor_id
        self.dtype = dtype
        self.shape = shape
        self.spec = spec
        self._manager = manager

    @property
    def bytes(self) -> int:
        return self.spec.bytes

    @property
    def page_list(self) -> list[int]:
        t = self._manager._t
        n = t._lib.hm_pt_tensor_pages(t.h, self.tensor_id, None, 0)
        if n < 0:
            raise KeyError(f"unknown tensor {self.tensor_id}")
        buf = N.i64_buf(n)
        t._lib.hm_pt_tensor_pages(t.h, self.tensor_id, buf, n)
        return list(buf[:n])

    def segments(self) -> list[tuple[int, int, int]]:
        """(page_id, byte_offset, bytes) per page, in tensor order."""
        t = self._manager._t
        n = t._lib.hm_pt_tensor_segments(t.h, self.tensor_id, None, 0)
        if n < 0:
            raise KeyError(f"unknown tensor {self.tensor_id}")
        buf = N.i64_buf(3 * n)
        t._lib.hm_pt_tensor_segments(t.h, self.tensor_id, buf, n)
        return [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n)]

    @property
    def tier(self):
        """Tier holding every page, or NOT_READY while pages span tiers."""
        out = (C.c_int64 * 4)()
        self._manager._t.call("hm_pt_tensor_info", C.c_int64(self.tensor_id), out)
        return Tier(out[2]) if out[2] >= 0 else NOT_READY

    def __repr__(self):
        return (f"ManagedTensor(tensor_id={self.tensor_id}, dtype={self.dtype!r}, "
                f"shape={self.shape}, page_list={self.page_list})")


class PageManager:
    """Owns one pool per tier plus the tensor registry spanning them
    (hiermem/pagemem.py:188-446)."""

    def __init__(self, pool_specs):
        """``pool_specs``: ``(tier, capacity)`` or ``(tier, capacity, page_bytes)`` entries;
        page ids are handed out pool after pool in this order."""
        self._t = _Table()
        self.pools: dict[Tier, TierPool] = {}
        for entry in pool_specs:
            tier = Tier.parse(entry[0])
            capacity = entry[1]
            page_bytes = entry[2] if len(entry) > 2 else PAGE_BYTES_DEFAULT
            self._t.call("hm_pt_add_pool", int(tier.value), C.c_int64(capacity),
                         C.c_int64(page_bytes), C.c_int64(-1))
            self.pools[tier] = TierPool(tier, capacity, page_bytes, _table=self._t)
        self.tensors: dict[int, ManagedTensor] = {}

    @classmethod
    def adopt(cls, pool: TierPool) -> "PageManager":
        mgr = cls([])
        mgr._t = pool._t
        mgr.pools[pool.tier] = pool
        return mgr

    def pool(self, tier) -> TierPool:
        tier = Tier.parse(tier)
        if tier not in self.pools:
            raise ConfigError(f"this manager has no {tier.name} pool")
        return self.pools[tier]

    def page(self, page_id: int) -> Page:
        for pool in self.pools.values():
            if page_id in pool.pages:
                return pool.pages[page_id]
        raise KeyError(f"page {page_id} belongs to no pool")

    # allocate / release

    def allocate(self, spec, tier) -> ManagedTensor:
        pool = self.pool(tier)
        tid = C.c_int64()
        self._t.call("hm_pt_allocate", int(pool.tier.value), N.KIND_CODES[spec.kind],
                     C.c_int64(spec.bytes), C.byref(tid))
        itemsize = 4 if spec.kind == "optim32" else 2
        tensor = ManagedTensor(tid.value, _dtype_for(spec.kind), (spec.bytes // itemsize,), spec, self)
        self.tensors[tid.value] = tensor
        return tensor

    def release(self, tensor_id: int) -> int:
        if tensor_id not in self.tensors:
            raise KeyError(f"tensor {tensor_id} is not live")
        freed = C.c_int64()
        self._t.call("hm_pt_release", C.c_int64(tensor_id), C.byref(freed))
        del self.tensors[tensor_id]
        return freed.value

    # page motion between tiers

    def page_move(self, page_id: int, target_tier) -> TransferDescriptor:
        target = Tier.parse(target_tier)
        out = (C.c_int64 * 5)()
        self._t.call("hm_pt_page_move", C.c_int64(page_id), int(target.value), out)
        return TransferDescriptor(out[0], Tier(out[1]), Tier(out[2]), out[3], out[4])

    # merge

    def tensor_merge(self, tensor_id: int) -> dict:
        """Defragment: move the tensor onto consecutive page ids of its tier
        (the native table picks the run; the reference's rules and report)."""
        if tensor_id not in self.tensors:
            raise KeyError(f"tensor {tensor_id} is not live")
        out = (C.c_int64 * 2)()
        self._t.call("hm_pt_tensor_merge", C.c_int64(tensor_id), out)
        n = len(self.tensors[tensor_id].page_list)
        return {"tensor_id": tensor_id, "contiguous": True,
                "page_ids": list(range(out[1], out[1] + n)), "moved_chunks": out[0]}

    # state dump (the parity artefact)

    def state_dict(self) -> dict:
        pools = {}
        for tier, pool in self.pools.items():
            info = pool._info()
            pools[tier.name] = {
                "capacity_bytes": info[1],
                "page_bytes": info[2],
                "free_pages": info[5],
                "allocated_pages": info[4] - info[5],
                "fragmentation": fragmentation(pool),
                "stats": vars(PoolStats(info[6], info[7], info[8], info[9], info[10])),
            }
        pages = []
        for pool in self.pools.values():
            for page in pool.allocated_pages():
                v = page._info()
                occ = [{"tensor_id": v[3 + 4 * i], "bytes": v[4 + 4 * i]} for i in range(v[2])]
                pages.append({
                    "page_id": page.page_id,
                    "tier": Tier(v[0]).name,
                    "total_bytes": v[1],
                    "available_bytes": v[1] - sum(o["bytes"] for o in occ),
                    "occupants": occ,
                })
        tensors = []
        for tid in sorted(self.tensors):
            t = self.tensors[tid]
            tier = t.tier
            tensors.append({
                "tensor_id": tid,
                "name": t.spec.name,
                "dtype": t.dtype,
                "bytes": t.bytes,
                "tier": tier.name if isinstance(tier, Tier) else tier,
                "page_list": list(t.page_list),
            })
        return {"pools": pools, "pages": pages, "tensors": tensors}


def _manager_of(pool: TierPool) -> PageManager:
    mgr = getattr(pool, "_manager", None)
    if mgr is None:
        mgr = PageManager.adopt(pool)
        pool._manager = mgr
    return mgr


def tensor_allocate(pool: TierPool, spec) -> ManagedTensor:
    """``PageManager.allocate`` on a pool used on its own (one implicit manager per pool)."""
    return _manager_of(pool).allocate(spec, pool.tier)


def tensor_release(pool: TierPool, tensor_id: int) -> int:
    """``PageManager.release`` on a pool used on its own; the occupant bytes freed."""
    return _manager_of(pool).release(tensor_id)
