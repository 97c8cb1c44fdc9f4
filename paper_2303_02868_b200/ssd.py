"""SSD page tier: fp32 master state in a file, streamed through pinned and
HBM staging in the updating actor's order (the bottom of the paper's
GPU/CPU/SSD hierarchy; the reference only
charges SSD time as DelayModel sleeps at 3.5 GB/s, hiermem/lockfree.py:
85-100, and models an ``ssd_io`` link, hiermem/simengine.py:298-309).

The image has no GPUDirect Storage, so the SSD leg is POSIX I/O from host
threads into pinned staging buffers (``O_DIRECT`` when the filesystem allows
it, so the page cache does not stand in for the drive), and the PCIe leg is
the swap tier's cudaMemcpyAsync.  Per page group, last page first:

    I/O thread  : pread  group k  -> pinned slot (k mod S)
    copy stream : H2D    pinned slot -> HBM stage
    compute     : page-Adam on the staged pages (reads g16, writes p16)
    copy stream : D2H    HBM stage -> pinned slot
    I/O thread  : pwrite pinned slot -> group k (after the D2H event)

Reads run up to S-1 groups ahead; a slot is re-read only after its write
drained, so every page is fetched, updated, published and stored exactly
once per sweep.  File layout is group-major: group k holds its p, m and v
planes back to back, so each leg is ONE sequential I/O of 12 B/param.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import ConfigError
from .layout import PageLayout
from .lockfree import (MasterState, ParamBuffer, SweepResult, UpdateTicket, _LayerView, _Paged,
                       update_prologue)
from .pagemem import PAGE_BYTES_DEFAULT


def _open(path: str, direct: bool):
    flags = os.O_RDWR | os.O_CREAT
    if direct and hasattr(os, "O_DIRECT"):
        try:
            return os.open(path, flags | os.O_DIRECT, 0o600), True
        except OSError:
            pass
    return os.open(path, flags, 0o600), False


class SSDMasterState(_Paged):
    """MasterState whose p32/m32/v32 pages live in a file on an SSD."""

    def __init__(self, params, path: str, tier: str = "SSD", *, page_bytes: int = PAGE_BYTES_DEFAULT,
                 device=None, layout: PageLayout | None = None, group_pages: int = 64,
                 slots: int = 3, direct: bool = True, io_threads: int = 4, world_size: int = 1,
                 rank: int = 0):
        # world-sharded: this rank's file holds only the pages it owns (page % N)
        self._init_paged(params, page_bytes, device, layout, world_size, rank)
        self.tier = tier
        lay = self.layout
        E = lay.E
        self.group_pages = max(1, int(group_pages))
        self.num_groups = -(-lay.P_local // self.group_pages)
        self.gE = self.group_pages * E                        # elements per plane per group
        self.group_bytes = 3 * 4 * self.gE
        self.path = path
        self.fd, self.direct = _open(path, direct)
        os.ftruncate(self.fd, self.num_groups * self.group_bytes)
        self.slots = max(2, int(slots))
        self.pinned = [torch.zeros(3 * self.gE, dtype=torch.float32, pin_memory=True)
                       for _ in range(self.slots)]
        self.stage = [torch.empty(3 * self.gE, dtype=torch.float32, device=self.device) for _ in range(2)]
        self.h2d = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)
        self.io = ThreadPoolExecutor(max_workers=max(2, io_threads))
        with torch.cuda.stream(self._stream()):
            self._steps = torch.zeros(self.num_layers, dtype=torch.int32, device=self.device)
            self._applied = torch.zeros(self.num_layers, dtype=torch.int32, device=self.device)
        self._step_bound = [0] * self.num_layers
        self._plans: dict = {}
        self._write_initial(params)

    # file I/O ------------------------------------------------------------------
    def _view(self, slot: int) -> memoryview:
        return memoryview(self.pinned[slot].numpy()).cast("B")

    def _pread(self, k: int, slot: int) -> None:
        mv, off, done = self._view(slot), k * self.group_bytes, 0
        while done < len(mv):
            n = os.preadv(self.fd, [mv[done:]], off + done)
            if n <= 0:
                raise OSError(f"short read of group {k} from {self.path}")
            done += n

    def _pwrite(self, k: int, slot: int, wait_event=None) -> None:
        if wait_event is not None:
            wait_event.synchronize()
        mv, off, done = self._view(slot), k * self.group_bytes, 0
        while done < len(mv):
            n = os.pwritev(self.fd, [mv[done:]], off + done)
            if n <= 0:
                raise OSError(f"short write of group {k} to {self.path}")
            done += n

    def _loc(self, pid_local: int, off: int):
        """(group, element offset inside the group's p plane) of a state slot."""
        k, r = divmod(pid_local, self.group_pages)
        return k, r * self.layout.E + off

    def _write_initial(self, params) -> None:
        lay = self.layout
        by_group: dict[int, list] = {}
        for l, p in enumerate(params):
            flat = (p.detach().reshape(-1).float().cpu().numpy() if isinstance(p, torch.Tensor)
                    else np.asarray(p, dtype=np.float32).reshape(-1))
            for s in lay.segments[l]:
                if not lay.owned(s):
                    continue
                k, o = self._loc(lay.slot_state(s.page), s.off)
                by_group.setdefault(k, []).append((o, flat[s.pos:s.pos + s.n]))
        buf = self.pinned[0].numpy()
        for k in range(self.num_groups):
            buf[:] = 0.0
            for o, vals in by_group.get(k, ()):
                buf[o:o + len(vals)] = vals
            self._pwrite(k, 0)
        os.fsync(self.fd)

    def close(self) -> None:
        if getattr(self, "fd", None) is not None:
            self.io.shutdown(wait=True)
            os.close(self.fd)
            self.fd = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # reference attributes (reads from the file) --------------------------------
    def _file_layer(self, plane: int, layer: int):
        torch.cuda.synchronize(self.device)
        lay = self.layout
        out = np.zeros(lay.numels[layer], dtype=np.float32)
        tmp = np.empty(3 * self.gE, dtype=np.float32)
        cache = {}
        for s in lay.segments[layer]:
            if not lay.owned(s):
                continue
            k, o = self._loc(lay.slot_state(s.page), s.off)
            if k not in cache:
                fd = os.open(self.path, os.O_RDONLY)
                try:
                    os.preadv(fd, [memoryview(tmp).cast("B")], k * self.group_bytes)
                finally:
                    os.close(fd)
                cache[k] = tmp.copy()
            out[s.pos:s.pos + s.n] = cache[k][plane * self.gE + o: plane * self.gE + o + s.n]
        out = out.reshape(self._shapes[layer])
        return out if self._numpy else torch.from_numpy(out)

    @property
    def p32(self):
        return _LayerView(self, lambda l: self._file_layer(0, l))

    @property
    def m32(self):
        return _LayerView(self, lambda l: self._file_layer(1, l))

    @property
    def v32(self):
        return _LayerView(self, lambda l: self._file_layer(2, l))

    @property
    def steps(self) -> list[int]:
        return [int(x) for x in self._steps.cpu().tolist()]

    _bias = MasterState._bias

    def planes(self, stage) -> tuple[int, int, int]:
        """Device addresses of the p / m / v planes of an HBM stage."""
        return D.ptr(stage), D.ptr(stage) + 4 * self.gE, D.ptr(stage) + 8 * self.gE

    def stream_update(self, layers, st, launch, timings=None) -> None:
        """Stream the state of ``layers`` through the tier: per page group
        (last first) pread -> H2D -> ``launch(chunks, stage)`` on ``st`` ->
        D2H -> pwrite, reads running up to S-1 groups ahead; blocks until
        every group is back in the file.  ``stage`` is laid out [p|m|v]."""
        plan = self._group_plan(tuple(layers))
        S, io = self.slots, self.io
        reads, writes = {}, {}

        def start_read(i):
            k = plan[i][0]
            slot = i % S
            if slot in writes:
                writes.pop(slot).result()            # slot drained to the drive
            reads[i] = io.submit(self._pread, k, slot)

        for i in range(min(S - 1, len(plan))):
            start_read(i)
        for i, (k, chunks) in enumerate(plan):
            if i + S - 1 < len(plan):
                start_read(i + S - 1)
            reads.pop(i).result()
            slot, stage = i % S, self.stage[i % 2]
            self.h2d.wait_stream(self.d2h)     # the HBM stage's previous store finished
            with torch.cuda.stream(self.h2d):
                stage.copy_(self.pinned[slot], non_blocking=True)
                fetched = torch.cuda.Event()
                fetched.record(self.h2d)
            st.wait_event(fetched)
            launch(chunks, stage)
            updated = torch.cuda.Event()
            updated.record(st)
            self.d2h.wait_event(updated)
            with torch.cuda.stream(self.d2h):
                self.pinned[slot].copy_(stage, non_blocking=True)
                stored = torch.cuda.Event()
                stored.record(self.d2h)
            writes[slot] = io.submit(self._pwrite, k, slot, stored)
        for f in writes.values():
            f.result()
        st.wait_stream(self.d2h)

    def _group_plan(self, layers: tuple):
        """Per group (reverse order): adam chunks with s_off rebased into a
        stage laid out as [p | m | v] planes of gE elements each."""
        if layers in self._plans:
            return self._plans[layers]
        lay, E, G = self.layout, self.layout.E, self.group_pages
        full = lay.adam_chunks(layers, "pool", owned_only=True)
        page = full["s_off"] // E
        plan = []
        for k in reversed(range(self.num_groups)):
            sel = (page >= k * G) & (page < (k + 1) * G)
            if not sel.any():
                continue
            c = full[sel].copy()
            c["s_off"] -= k * G * E
            plan.append((k, c))
        self._plans[layers] = plan
        return plan


def ssd_sweep(buffer: ParamBuffer, masters: SSDMasterState, hyper, layers=None, *,
              stream=None) -> SweepResult:
    """``sweep`` with the state on the SSD tier (blocking: returns when every
    group is back on the drive, like the reference's synchronous updater)."""
    lay = buffer.layout
    if masters.layout.numels != lay.numels or masters.layout.page_bytes != lay.page_bytes:
        raise ConfigError("buffer and masters were built on different page tables")
    if lay.world_size != 1:
        raise ConfigError("a world-sharded SSD tier is updated by the DP step "
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

    masters.stream_update(sel, st, launch)
    t.finish()
    return SweepResult(masters, sel, t.counts, t.newest)
