"""Page pools with bytes behind them (K1 pack/unpack + K8 page motion).

The reference page manager is metadata-only: ``page_move`` frees at the
source and claims at the destination, ``tensor_merge`` reassigns ids, and no
byte ever moves (hiermem/pagemem.py:7-9, 323-326, 386-405).  The paper's
Allocator/Executor do move them (pre-allocated pools,
``cudaMemcpyAsync`` between tiers).  ``DevicePageManager`` is the drop-in
``PageManager`` (same table, same results, same errors) whose GPU pool is an
HBM byte buffer and whose CPU pool is a pinned host byte buffer:

* ``write(tid, data)`` / ``read(tid)`` pack / unpack a tensor into / out of
  its pages along the (page, offset, bytes) segments of the table —
  ``hm_copy_runs`` (16-byte vector copies) on the device, copy engines across
  the PCIe boundary;
* ``page_move`` copies the page to its new tier with one cudaMemcpyAsync on
  a copy stream before returning the reference's TransferDescriptor;
* ``tensor_merge`` copies every relocated chunk (keeping its in-page offset)
  through a staging buffer, so chains like page 5 -> 3 while 3 -> 4 are safe.

An SSD pool is backed by a file when ``ssd_path`` is given (no GPUDirect
Storage in the image: POSIX I/O from the host, ``O_DIRECT`` when the
filesystem allows it, through a pinned page-sized bounce buffer for the GPU
side); page moves to and from it and pack/unpack of SSD-resident pages move
real bytes.  Without ``ssd_path`` the SSD pool stays metadata-only, as in
the reference, and touching its bytes raises ConfigError.
"""
from __future__ import annotations

import os

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import ConfigError
from .pagemem import PageManager, Tier, TransferDescriptor

COPY_PIECE = 64 * 1024  # bytes per CTA work unit of hm_copy_runs


def _descs(rows) -> np.ndarray:
    """Split (src_off, dst_off, bytes) runs into <= COPY_PIECE pieces."""
    out = []
    for s, d, n in rows:
        k = 0
        while k < n:
            m = min(COPY_PIECE, n - k)
            out.append((s + k, d + k, m))
            k += m
    return np.array(out, dtype=N.COPY_DESC) if out else np.zeros(0, dtype=N.COPY_DESC)


class DevicePageManager(PageManager):
    def __init__(self, pool_specs, device=None, *, ssd_path: str | None = None):
        super().__init__(pool_specs)
        self.device = D.require_device(device)
        self.copy_stream = torch.cuda.Stream(self.device)
        self.storage: dict[Tier, torch.Tensor | None] = {}
        self._fd = None
        for tier, pool in self.pools.items():
            if tier is Tier.GPU:
                self.storage[tier] = torch.zeros(pool.capacity_bytes, dtype=torch.uint8, device=self.device)
            elif tier is Tier.CPU:
                self.storage[tier] = torch.zeros(pool.capacity_bytes, dtype=torch.uint8, pin_memory=True)
            elif tier is Tier.SSD and ssd_path is not None:
                from .ssd import _open
                self._fd, self.ssd_direct = _open(ssd_path, direct=True)
                os.ftruncate(self._fd, pool.capacity_bytes)
                self._ssd_page = pool.page_bytes
                self._bounce = torch.empty(pool.page_bytes, dtype=torch.uint8, pin_memory=True)
                self.storage[tier] = None          # backed by the file, not a tensor

    def close(self) -> None:
        if self._fd is not None:
            os.close(self._fd)
            self._fd = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- the SSD file (whole pages: O_DIRECT needs aligned offsets and sizes) ----
    def _pread(self, off: int, buf: torch.Tensor) -> None:
        mv = memoryview(buf.numpy()).cast("B")
        done = 0
        while done < len(mv):
            n = os.preadv(self._fd, [mv[done:]], off + done)
            if n <= 0:
                raise OSError(f"short read from the SSD pool at {off + done}")
            done += n

    def _pwrite(self, off: int, buf: torch.Tensor) -> None:
        mv = memoryview(buf.numpy()).cast("B")
        done = 0
        while done < len(mv):
            n = os.pwritev(self._fd, [mv[done:]], off + done)
            if n <= 0:
                raise OSError(f"short write to the SSD pool at {off + done}")
            done += n

    def _ssd_read_bytes(self, addr: int, n: int) -> np.ndarray:
        """Bytes [addr, addr+n) of the SSD pool (read page by page)."""
        P = self._ssd_page
        out = np.empty(n, dtype=np.uint8)
        pos = 0
        while pos < n:
            base = (addr + pos) // P * P
            k = min(n - pos, base + P - (addr + pos))
            self._pread(base, self._bounce)
            lo = addr + pos - base
            out[pos:pos + k] = self._bounce.numpy()[lo:lo + k]
            pos += k
        return out

    def _ssd_write_bytes(self, addr: int, data: np.ndarray) -> None:
        """Read-modify-write of whole pages (partial runs keep their neighbours)."""
        P, n, pos = self._ssd_page, len(data), 0
        while pos < n:
            base = (addr + pos) // P * P
            k = min(n - pos, base + P - (addr + pos))
            lo = addr + pos - base
            if k < P:
                self._pread(base, self._bounce)
            self._bounce.numpy()[lo:lo + k] = data[pos:pos + k]
            self._pwrite(base, self._bounce)
            pos += k

    # -- addressing -----------------------------------------------------------
    def _loc(self, pid: int):
        for tier, pool in self.pools.items():
            if pid in pool.pages:
                if tier not in self.storage:
                    raise ConfigError(f"{tier.name} pages have no backing store (pass ssd_path= to back the SSD pool)")
                return tier, (pid - pool.first_page_id) * pool.page_bytes
        raise KeyError(f"unknown page id {pid}")

    def _runs_by_tier(self, tensor_id: int):
        runs: dict[Tier, list] = {}
        pos = 0
        for pid, off, nbytes in self.tensors[tensor_id].segments():
            tier, base = self._loc(pid)
            runs.setdefault(tier, []).append((pos, base + off, nbytes))
            pos += nbytes
        return runs

    # -- pack / unpack ----------------------------------------------------------
    def write(self, tensor_id: int, data, *, stream=None) -> None:
        """Pack a tensor's bytes into its pages (K1)."""
        t = self.tensors[tensor_id]
        st = D.cur_stream(self.device, stream)
        src = data.detach().reshape(-1) if isinstance(data, torch.Tensor) else \
            torch.from_numpy(np.ascontiguousarray(data).reshape(-1))
        raw = src.contiguous().view(torch.uint8)
        if raw.numel() != t.bytes:
            raise ConfigError(f"tensor {tensor_id} holds {t.bytes} bytes, got {raw.numel()}")
        lib = N.lib()
        for tier, rows in self._runs_by_tier(tensor_id).items():
            store = self.storage[tier]
            if tier is Tier.GPU:
                with torch.cuda.stream(st):
                    dev = raw.to(self.device, non_blocking=raw.is_pinned()) if not raw.is_cuda else raw
                d = _descs(rows)
                D.check(lib.hm_copy_runs(D.ptr(dev), D.ptr(store), D.ptr(self._up(d, st)), len(d), D.sptr(st)))
                if dev is not raw:
                    dev.record_stream(st)
            elif tier is Tier.SSD:
                st.synchronize()
                host = raw.cpu().numpy()
                for sp, dpos, n in rows:
                    self._ssd_write_bytes(dpos, host[sp:sp + n])
            else:
                kind = 2 if raw.is_cuda else 0
                if kind == 0:
                    st.synchronize()
                    for s, dpos, n in rows:
                        store[dpos:dpos + n].copy_(raw[s:s + n].cpu())
                else:
                    d = np.array(rows, dtype=N.COPY_DESC)
                    D.check(lib.hm_memcpy_runs(D.ptr(raw), D.ptr(store), d.ctypes.data, len(d), 2,
                                               D.sptr(st)))

    def read(self, tensor_id: int, *, stream=None) -> torch.Tensor:
        """Unpack a tensor's pages into a contiguous CUDA tensor (K1)."""
        t = self.tensors[tensor_id]
        st = D.cur_stream(self.device, stream)
        with torch.cuda.stream(st):
            out = torch.empty(t.bytes, dtype=torch.uint8, device=self.device)
        lib = N.lib()
        for tier, rows in self._runs_by_tier(tensor_id).items():
            store = self.storage[tier]
            inv = [(dpos, s, n) for s, dpos, n in rows]
            if tier is Tier.GPU:
                d = _descs(inv)
                D.check(lib.hm_copy_runs(D.ptr(store), D.ptr(out), D.ptr(self._up(d, st)), len(d), D.sptr(st)))
            elif tier is Tier.SSD:
                for src, dst, n in inv:
                    chunk = torch.from_numpy(self._ssd_read_bytes(src, n))
                    with torch.cuda.stream(st):
                        out[dst:dst + n].copy_(chunk)
            else:
                d = np.array(inv, dtype=N.COPY_DESC)
                D.check(lib.hm_memcpy_runs(D.ptr(store), D.ptr(out), d.ctypes.data, len(d), 1, D.sptr(st)))
        dt = torch.float32 if t.dtype == "fp32" else torch.float16
        return out.view(dt)

    def _up(self, d: np.ndarray, stream=None) -> torch.Tensor:
        """Upload copy descriptors for a launch on ``stream``: allocated and
        copied on that stream, so the block cannot be handed to another
        upload before the kernel that reads it has run."""
        st = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.stream(st):
            return torch.from_numpy(d.view(np.uint8).copy()).to(self.device) if len(d) else \
                torch.empty(8, dtype=torch.uint8, device=self.device)

    # -- movement with data -----------------------------------------------------------
    def _tier_of(self, pid: int) -> Tier:
        for tier, pool in self.pools.items():
            if pid in pool.pages:
                return tier
        raise KeyError(f"unknown page id {pid}")

    def page_move(self, page_id: int, target_tier, *, stream=None) -> TransferDescriptor:
        src_tier = self._tier_of(page_id)
        backed_src = src_tier in self.storage
        src_off = self._loc(page_id)[1] if backed_src else None
        desc = super().page_move(page_id, target_tier)
        if not backed_src or desc.dst_tier not in self.storage:
            return desc  # an unbacked SSD side is metadata-only, as in the reference
        dst_tier, dst_off = self._loc(desc.new_page_id)
        st = D.cur_stream(self.device, stream)
        self.copy_stream.wait_stream(st)
        n = desc.bytes
        if Tier.SSD in (src_tier, dst_tier):
            self._move_ssd(src_tier, src_off, dst_tier, dst_off, n)
            return desc
        kind = {(Tier.GPU, Tier.CPU): 2, (Tier.CPU, Tier.GPU): 1}[(src_tier, dst_tier)]
        d = np.array([(src_off, dst_off, n)], dtype=N.COPY_DESC)
        D.check(N.lib().hm_memcpy_runs(D.ptr(self.storage[src_tier]), D.ptr(self.storage[dst_tier]),
                                       d.ctypes.data, 1, kind, D.sptr(self.copy_stream)))
        st.wait_stream(self.copy_stream)
        return desc

    def _move_ssd(self, src_tier, src_off, dst_tier, dst_off, n) -> None:
        """Whole-page moves to / from the SSD file (synchronous: the bounce
        buffer and the CPU pool are host memory the I/O reads directly)."""
        cs = self.copy_stream
        if src_tier is Tier.GPU:        # GPU -> SSD: D2H into the bounce, then write
            d = np.array([(src_off, 0, n)], dtype=N.COPY_DESC)
            D.check(N.lib().hm_memcpy_runs(D.ptr(self.storage[Tier.GPU]), D.ptr(self._bounce),
                                           d.ctypes.data, 1, 2, D.sptr(cs)))
            cs.synchronize()
            self._pwrite(dst_off, self._bounce[:n])
        elif dst_tier is Tier.GPU:      # SSD -> GPU: read into the bounce, then H2D
            self._pread(src_off, self._bounce[:n])
            d = np.array([(0, dst_off, n)], dtype=N.COPY_DESC)
            D.check(N.lib().hm_memcpy_runs(D.ptr(self._bounce), D.ptr(self.storage[Tier.GPU]),
                                           d.ctypes.data, 1, 1, D.sptr(cs)))
            cs.synchronize()
        elif src_tier is Tier.CPU:      # CPU -> SSD straight from the pinned pool
            cs.synchronize()
            self._pwrite(dst_off, self.storage[Tier.CPU][src_off:src_off + n])
        else:                           # SSD -> CPU straight into the pinned pool
            cs.synchronize()
            self._pread(src_off, self.storage[Tier.CPU][dst_off:dst_off + n])

    def tensor_merge(self, tensor_id: int, *, stream=None) -> dict:
        t = self.tensors.get(tensor_id)
        before = t.segments() if t is not None else None
        report = super().tensor_merge(tensor_id)
        if report["moved_chunks"] == 0:
            return report
        after = self.tensors[tensor_id].segments()
        moves = []
        for (p0, o0, n0), (p1, o1, n1) in zip(before, after):
            if p0 != p1:
                (t0, a0), (t1, a1) = self._loc(p0), self._loc(p1)
                if t0 is not t1:
                    raise ConfigError("merge stays within one tier")
                moves.append((a0 + o0, a1 + o1, n0))
        tier = self._loc(after[0][0])[0]
        store = self.storage[tier]
        st = D.cur_stream(self.device, stream)
        total = sum(n for _, _, n in moves)
        if tier is Tier.GPU:
            with torch.cuda.stream(st):
                tmp = torch.empty(total, dtype=torch.uint8, device=self.device)
            gather, scatter, pos = [], [], 0
            for a0, a1, n in moves:
                gather.append((a0, pos, n))
                scatter.append((pos, a1, n))
                pos += n
            g, s = _descs(gather), _descs(scatter)
            D.check(N.lib().hm_copy_runs(D.ptr(store), D.ptr(tmp), D.ptr(self._up(g, st)), len(g), D.sptr(st)))
            D.check(N.lib().hm_copy_runs(D.ptr(tmp), D.ptr(store), D.ptr(self._up(s, st)), len(s), D.sptr(st)))
        elif tier is Tier.SSD:
            tmp = [self._ssd_read_bytes(a0, n) for a0, _, n in moves]   # gather first: chains
            for (a0, a1, n), buf in zip(moves, tmp):
                self._ssd_write_bytes(a1, buf)
        else:
            st.synchronize()
            tmp = [store[a0:a0 + n].clone() for a0, _, n in moves]
            for (a0, a1, n), buf in zip(moves, tmp):
                store[a1:a1 + n].copy_(buf)
        return report


def _flat_runs(dm: "DevicePageManager", tensor_ids, reverse: bool):
    """All GPU-tier runs of many tensors against one flat buffer (tensor order)."""
    rows, base = [], 0
    for tid in tensor_ids:
        t = dm.tensors[tid]
        pos = 0
        for pid, off, nbytes in t.segments():
            tier, addr = dm._loc(pid)
            if tier is not Tier.GPU:
                raise ConfigError("batched pack/unpack covers GPU pages; move CPU pages first")
            rows.append((addr + off, base + pos, nbytes) if reverse else (base + pos, addr + off, nbytes))
            pos += nbytes
        base += t.bytes
    return rows, base


def pack_many(dm: "DevicePageManager", tensor_ids, flat: torch.Tensor, *, stream=None) -> None:
    """Pack many tensors, stored back to back in ``flat``, with ONE launch (K1)."""
    key = ("pack", tuple(tensor_ids))
    cache = dm.__dict__.setdefault("_batch_cache", {})
    if key not in cache:
        rows, total = _flat_runs(dm, tensor_ids, reverse=False)
        d = _descs(rows)
        cache[key] = (dm._up(d), len(d), total)
    dd, n, total = cache[key]
    raw = flat.reshape(-1).view(torch.uint8)
    if raw.numel() != total:
        raise ConfigError(f"flat buffer holds {raw.numel()} bytes, tensors need {total}")
    st = D.cur_stream(dm.device, stream)
    D.check(N.lib().hm_copy_runs(D.ptr(raw), D.ptr(dm.storage[Tier.GPU]), D.ptr(dd), n, D.sptr(st)))


def unpack_many(dm: "DevicePageManager", tensor_ids, *, stream=None) -> torch.Tensor:
    """Unpack many tensors back to back into one flat uint8 CUDA tensor (K1)."""
    key = ("unpack", tuple(tensor_ids))
    cache = dm.__dict__.setdefault("_batch_cache", {})
    if key not in cache:
        rows, total = _flat_runs(dm, tensor_ids, reverse=True)
        d = _descs(rows)
        cache[key] = (dm._up(d), len(d), total)
    dd, n, total = cache[key]
    st = D.cur_stream(dm.device, stream)
    with torch.cuda.stream(st):
        out = torch.empty(total, dtype=torch.uint8, device=dm.device)
    D.check(N.lib().hm_copy_runs(D.ptr(dm.storage[Tier.GPU]), D.ptr(out), D.ptr(dd), n, D.sptr(st)))
    return out
