"""Drop-in optimizer-update path of hiermem/lockfree.py on B200 page pools.

Reference surface kept (hiermem/lockfree.py): ``AdamHyper`` (:37-42),
``GradMessage`` (:120-124), ``apply_update`` (:127-142), ``MasterState``
(:145-165), ``ParamBuffer`` (:174-263), ``publish_params`` /
``accumulate_gradient`` (:266-272), ``ConservationLedger`` (:275-326).

Data lives in device page pools that share one page table (``layout.py``):
ParamBuffer owns two 16-bit gradient buffers and two 16-bit published
buffers; MasterState owns the fp32 p/m/v pools and per-layer step counters.
All arithmetic runs in libhm_page.so kernels on the caller's current CUDA
stream; this module only keeps the reference's host-side bookkeeping
(pending counts, newest iteration, versions, ledger).

Two ways to drive an update:

* the reference's three calls per layer — ``buffer.take`` →
  ``masters.update_layer`` → ``buffer.publish`` — each one kernel over the
  layer's page segments, with the reference's synchronous return values;
* ``sweep(buffer, masters, hyper)`` — the same take → update → publish for
  every pending layer fused into one prologue + one page-Adam launch
  (28 B/param), asynchronous: this is the hot path.

Return types follow the inputs: numpy in → numpy out (drop-in for numpy
callers), torch in → CUDA tensors out.
"""
from __future__ import annotations

import math
import weakref
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import ConfigError, ProtocolError
from .layout import PageLayout
from .pagemem import PAGE_BYTES_DEFAULT


@dataclass(frozen=True)
class AdamHyper:
    """hiermem/lockfree.py:37-42, plus two B200 additions that are exact
    identities at their defaults: ``inv_scale`` (loss-scale unscale, x*1.0f)
    and ``max_norm`` (grad-norm clip, <= 0 disables; the norm is over the
    layers of one update: a sweep's or DP step's layers, the one layer of an
    ``update_layer``, the tensor of an ``apply_update``)."""

    lr: float = 0.01
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    inv_scale: float = 1.0
    max_norm: float = 0.0


@dataclass(frozen=True)
class DelayModel:
    """The reference's transfer/compute cost model (hiermem/lockfree.py:81-117),
    same fields, methods and presets, plus ``"b200"``: the rates this build
    measured on the GPU box (profiles/r1_raw) — pinned PCIe 55.5 GB/s per
    direction, the SSD tier's O_DIRECT 4.5 GB/s, and the update itself on
    the GPU at 28 B/param x 2.41e11 params/s (so ``update_compute_s`` is the
    page-Adam time instead of a CPU sweep)."""

    pcie_bytes_per_s: float = 32e9
    ssd_bytes_per_s: float | None = 3.5e9
    cpu_mem_bytes_per_s: float = 100e9
    gpu_flops_per_s: float = 1e11

    def fetch_s(self, nbytes: int) -> float:
        return nbytes / self.pcie_bytes_per_s

    def offload_s(self, nbytes: int) -> float:
        return nbytes / self.pcie_bytes_per_s

    def state_fetch_s(self, nbytes: int) -> float:
        rate = self.ssd_bytes_per_s or self.cpu_mem_bytes_per_s
        return nbytes / rate

    state_store_s = state_fetch_s

    def update_compute_s(self, nbytes_touched: int) -> float:
        return nbytes_touched / self.cpu_mem_bytes_per_s

    def compute_s(self, flops: float) -> float:
        return flops / self.gpu_flops_per_s

    @classmethod
    def preset(cls, name: str) -> "DelayModel":
        if name == "ssd":
            return cls()
        if name == "cpu":
            return cls(ssd_bytes_per_s=None)
        if name == "zero":
            return cls(pcie_bytes_per_s=math.inf, ssd_bytes_per_s=math.inf,
                       cpu_mem_bytes_per_s=math.inf, gpu_flops_per_s=math.inf)
        if name == "b200":
            return cls(pcie_bytes_per_s=55.5e9, ssd_bytes_per_s=4.5e9,
                       cpu_mem_bytes_per_s=28 * 2.41e11, gpu_flops_per_s=1.37e15)
        raise ConfigError(f"unknown delay preset {name!r}")


@dataclass(frozen=True)
class GradMessage:
    layer: int
    payload: object  # 16-bit (or f32) gradient, numpy or torch
    iteration: int


class _Pending:
    """A ledger entry still sitting in a device ledger row (resolved lazily)."""

    __slots__ = ("row", "col")

    def __init__(self, row: int, col: int):
        self.row, self.col = row, col


class ConservationLedger:
    """Gradient conservation bookkeeping (hiermem/lockfree.py:275-326):
    per-layer f64 produced deltas, consumed and applied sums and message
    counts; balanced iff fsum(produced) == fsum(consumed) == fsum(applied +
    rejected) and the counts agree.

    Always on, like the reference's.  The sums are not separate passes: the
    accumulate kernel (K3) folds the f64 sum of (new - old) of every message
    into the same HBM pass, into a per-slot running sum (the buffer's total)
    and into the message's row of a device ledger ring; the take (prologue of
    the fused update, or hm_stats_take) snapshots and resets the running sum.
    Entries stay on the device until someone reads the ledger (``summary()``
    or the list attributes), so the update path never synchronises for it."""

    def __init__(self, num_layers: int):
        self._produced = [[] for _ in range(num_layers)]
        self._consumed = [[] for _ in range(num_layers)]
        self._applied = [[] for _ in range(num_layers)]
        self._rejected = [[] for _ in range(num_layers)]
        self._apply_pending: list[tuple[int, int, int, int]] = []   # (layer, row, sum col, flag col)
        self._unresolved: list[tuple[list, int, int, int]] = []     # (entries, index, row, col)
        self.messages_sent = [0] * num_layers
        self.messages_accumulated = [0] * num_layers
        self.messages_consumed = [0] * num_layers
        self._resolver = None   # ParamBuffer._ledger_flush: device rows -> floats

    def _sync(self):
        if self._resolver is not None:
            self._resolver()

    def _pend(self, entries: list, row: int, col: int) -> None:
        """Append an entry that a device ledger row will fill in."""
        self._unresolved.append((entries, len(entries), row, col))
        entries.append(_Pending(row, col))

    def _resolve(self, host: np.ndarray) -> None:
        for entries, i, row, col in self._unresolved:
            entries[i] = float(host[row, col])
        self._unresolved.clear()
        for layer, row, cs, cf in self._apply_pending:
            (self._applied if host[row, cf] != 0.0 else self._rejected)[layer].append(float(host[row, cs]))
        self._apply_pending.clear()

    @property
    def produced_deltas(self):
        self._sync()
        return self._produced

    @property
    def consumed_sums(self):
        self._sync()
        return self._consumed

    @property
    def applied_sums(self):
        self._sync()
        return self._applied

    @property
    def rejected_sums(self):
        self._sync()
        return self._rejected

    def record_accumulate(self, layer: int, delta: float) -> None:
        self._sync()
        self._produced[layer].append(delta)
        self.messages_accumulated[layer] += 1

    def record_take(self, layer: int, total: float, count: int) -> None:
        self._sync()
        self._consumed[layer].append(total)
        self.messages_consumed[layer] += count

    def record_apply(self, layer: int, total: float, rejected: bool) -> None:
        self._sync()
        (self._rejected if rejected else self._applied)[layer].append(total)

    def summary(self) -> dict:
        self._sync()
        out, balanced = [], True
        for l in range(len(self._produced)):
            sums = [math.fsum(x) for x in (self._produced[l], self._consumed[l],
                                            self._applied[l], self._rejected[l])]
            ok = (sums[0] == sums[1] == sums[2] + sums[3]
                  and self.messages_accumulated[l] == self.messages_consumed[l] == self.messages_sent[l])
            balanced &= ok
            out.append({"layer": l, "produced": sums[0], "consumed": sums[1], "applied": sums[2],
                        "rejected": sums[3], "messages_sent": self.messages_sent[l],
                        "messages_accumulated": self.messages_accumulated[l],
                        "messages_consumed": self.messages_consumed[l], "balanced": ok})
        return {"balanced": balanced, "layers": out}


# ---- shared helpers -------------------------------------------------------------

def _is_numpy(seq) -> bool:
    return len(seq) > 0 and not isinstance(seq[0], torch.Tensor)


def _shape(x):
    return tuple(x.shape) if hasattr(x, "shape") else tuple(np.shape(x))


class _StreamScratch:
    """Device scratch of ONE stream: the prologue's per-group runtime table
    and the reject flag of update_layer.  Allocated on that stream, so the
    caching allocator orders any reuse behind the stream's own kernels, and
    launches on other streams never share it."""

    def __init__(self, device, stream):
        self.device, self.stream = device, stream
        with torch.cuda.stream(stream):
            self.rt = torch.empty(64 * N.GROUP_RT_BYTES, dtype=torch.uint8, device=device)
            self.flag = torch.zeros(1, dtype=torch.int32, device=device)
            self.done = torch.zeros(1, dtype=torch.int32, device=device)   # hm_adam_layer's arrival count
            self.sumsq = torch.zeros(1, dtype=torch.float64, device=device)  # update_layer's clip norm

    def rt_for(self, n_groups: int) -> torch.Tensor:
        need = max(1, n_groups) * N.GROUP_RT_BYTES
        if self.rt.numel() < need:
            with torch.cuda.stream(self.stream):
                self.rt = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self.rt


class _Engine:
    """Per-device descriptor cache and bias tables (read-only after build),
    plus per-stream scratch."""

    _per_device: dict = {}

    def __init__(self, device):
        self.device = device
        self.desc = D.DescCache(device)
        self.bias: dict[tuple[float, float], D.BiasTable] = {}
        self._scratch: dict[int, _StreamScratch] = {}

    @classmethod
    def of(cls, device) -> "_Engine":
        key = str(device)
        if key not in cls._per_device:
            cls._per_device[key] = cls(device)
        return cls._per_device[key]

    def scratch(self, stream) -> _StreamScratch:
        key = int(stream.cuda_stream)
        sc = self._scratch.get(key)
        if sc is None or sc.stream != stream:
            sc = self._scratch[key] = _StreamScratch(self.device, stream)
        return sc

    def rt_scratch(self, n_groups: int, stream) -> torch.Tensor:
        return self.scratch(stream).rt_for(n_groups)

    def bias_table(self, hyper, max_step: int):
        key = (float(hyper.beta1), float(hyper.beta2))
        if key not in self.bias:
            self.bias[key] = D.BiasTable(key[0], key[1], self.device)
        return self.bias[key].ensure(max_step)


def adam_launch(engine: _Engine, chunks: np.ndarray, groups: np.ndarray, g, g_dt: int,
                p32, m32, v32, p16, p16_dt: int, hyper, bc_dev, bc_len: int,
                explicit_step: int, steps, applied, nonfinite, sumsq, consume: bool, stream,
                static_chunks: bool = True, lsum: int = 0, ledger_out: int = 0, opts=None) -> None:
    """One fused page-Adam step (prologue + main kernel) on ``stream``.
    ``steps`` / ``applied`` / ``nonfinite`` / ``sumsq`` are tensors or raw
    device addresses (int); ``lsum`` / ``ledger_out`` raw addresses."""
    dchunks = engine.desc.static(chunks) if static_chunks else engine.desc.table(chunks, stream)
    dgroups = engine.desc.table(groups, stream)
    rt = engine.rt_scratch(len(groups), stream)
    hc = D.hyper_c(hyper)
    a = D.addr
    D.check(N.lib().hm_adam_step(
        D.ptr(dchunks), len(chunks), D.ptr(dgroups), len(groups), D.ptr(rt),
        D.ptr(g), g_dt, D.ptr(p32), D.ptr(m32), D.ptr(v32), D.ptr(p16), p16_dt,
        hc, D.ptr(bc_dev), bc_len, explicit_step, a(steps), a(applied),
        a(nonfinite), a(sumsq), 1 if consume else 0, lsum or None, ledger_out or None, opts,
        D.sptr(stream)))


_ROWS: dict = {}


def _group_rows(rows) -> np.ndarray:
    """hm_group_launch table of (g_shift, p_shift, group, flag) rows (cached:
    the per-layer calls of the three-call path repeat the same few rows)."""
    key = tuple(rows)
    a = _ROWS.get(key)
    if a is None:
        a = np.zeros(len(rows), dtype=N.GROUP_LAUNCH)
        for i, (gs, ps, grp, flag) in enumerate(rows):
            a[i] = (gs, ps, grp, flag)
        if len(_ROWS) > 4096:
            _ROWS.clear()
        _ROWS[key] = a
    return a


class Applied:
    """Lazy result of ``MasterState.update_layer`` for torch callers: the
    update is queued on the stream; the bool is read (one synchronisation)
    only when the caller asks for it — ``bool(x)``, ``x == True``."""

    __slots__ = ("_t", "_stream", "_v")

    def __init__(self, t: torch.Tensor, stream):
        self._t, self._stream, self._v = t, stream, None

    def __bool__(self) -> bool:
        if self._v is None:
            with D.on(self._stream):
                self._v = bool(self._t.item())
        return self._v

    def __eq__(self, other):
        return bool(self) == other

    def __hash__(self):
        return hash(bool(self))

    def __repr__(self):
        return repr(bool(self))


# ---- functional update (hiermem/lockfree.py:127-142) ------------------------------

def apply_update(p32, m32, v32, grad, hyper: AdamHyper, step: int, *, stream=None):
    """One bias-corrected Adam step on fp32 masters; rejects non-finite grads.

    Returns (p32, m32, v32, applied).  Functional like the reference: the
    inputs are never modified; on reject the input objects are returned."""
    numpy_io = not isinstance(p32, torch.Tensor)
    device = D.require_device(p32.device if (not numpy_io and p32.is_cuda) else None)
    eng = _Engine.of(device)
    st = D.cur_stream(device, stream)
    shape = _shape(p32)
    with D.on(st):
        p = D.to_device_flat(p32, device).to(torch.float32).clone()
        m = D.to_device_flat(m32, device).to(torch.float32).clone()
        v = D.to_device_flat(v32, device).to(torch.float32).clone()
        g = D.to_device_flat(grad, device)
    n = p.numel()
    if m.numel() != n or v.numel() != n or g.numel() != n:
        raise ProtocolError(f"apply_update: size mismatch p={n} m={m.numel()} v={v.numel()} g={g.numel()}")
    if n == 0:
        return p32, m32, v32, True
    with D.on(st):
        bc = torch.tensor([float(np.float32(1.0 - hyper.beta1 ** step)),
                           float(np.float32(1.0 - hyper.beta2 ** step))], dtype=torch.float32, device=device)
        flag = torch.zeros(1, dtype=torch.int32, device=device)
        applied = torch.zeros(1, dtype=torch.int32, device=device)
        sumsq = torch.zeros(1, dtype=torch.float64, device=device) if hyper.max_norm > 0 else None
    cc = D.contiguous_chunks_cached(n)
    D.check(N.lib().hm_reduce_stats(D.ptr(g), D.DT_OF_TORCH[g.dtype], D.ptr(eng.desc.static(cc)), len(cc),
                                     D.ptr(flag), None, D.addr(sumsq), D.sptr(st)))
    adam_launch(eng, D.contiguous_adam_chunks(n), _group_rows([(0, 0, 0, 0)]), g, D.DT_OF_TORCH[g.dtype],
                p, m, v, None, 0, hyper, bc, 1, int(step), None, applied, flag, sumsq, True, st,
                static_chunks=False)
    with D.on(st):
        if not bool(applied.item()):
            return p32, m32, v32, False
        if numpy_io:
            return D.to_host(p, shape), D.to_host(m, shape), D.to_host(v, shape), True
    return p.view(shape), m.view(shape), v.view(shape), True


# ---- layer views ----------------------------------------------------------------------

class _LayerView(Sequence):
    """List-like per-layer access that unpacks pages on read and packs on write."""

    def __init__(self, owner, getter, setter=None):
        self._owner, self._get, self._set = owner, getter, setter

    def __len__(self):
        return self._owner.num_layers

    def __getitem__(self, layer):
        if isinstance(layer, slice):
            return [self._get(i) for i in range(*layer.indices(len(self)))]
        if not (-len(self) <= layer < len(self)):
            raise IndexError(layer)
        return self._get(layer % len(self))

    def __setitem__(self, layer, value):
        if self._set is None:
            raise TypeError("read-only view")
        self._set(layer, value)


class _Paged:
    """Common state of ParamBuffer and MasterState: layout, device, IO mode."""

    def _init_paged(self, params, page_bytes, device, layout, world_size=1, rank=0):
        if len(params) == 0:
            raise ConfigError("need at least one layer")
        self.device = D.require_device(device if device is not None else
                                       (params[0].device if isinstance(params[0], torch.Tensor)
                                        and params[0].is_cuda else None))
        self._numpy = _is_numpy(params)
        self._shapes = [_shape(p) for p in params]
        numels = [int(np.prod(s)) if len(s) else 1 for s in self._shapes]
        if layout is None:
            layout = PageLayout(numels, page_bytes, world_size=world_size, rank=rank)
        elif list(layout.numels) != numels:
            raise ConfigError("layout does not match the parameter shapes")
        self.layout = layout
        self._eng = _Engine.of(self.device)

    @property
    def num_layers(self) -> int:
        return len(self._shapes)

    def _stream(self, stream=None):
        return D.cur_stream(self.device, stream)

    def _check_layer(self, layer: int):
        if not (0 <= layer < self.num_layers):
            raise ProtocolError(f"unknown layer {layer}")

    def _cast(self, src, src_dt, dst, dst_dt, chunks: np.ndarray, stream):
        if len(chunks) == 0:
            return
        D.check(N.lib().hm_cast(D.ptr(src), src_dt, D.ptr(dst), dst_dt,
                                D.ptr(self._eng.desc.static(chunks)), len(chunks), D.sptr(stream)))

    def _out(self, t: torch.Tensor, layer: int, readonly=False):
        shape = self._shapes[layer]
        return D.to_host(t, shape, readonly) if self._numpy else t.view(shape)


# ---- MasterState (hiermem/lockfree.py:145-165) ---------------------------------------

class _Taken:
    """Tag on the f32 tensor ``ParamBuffer.take`` returns to a torch caller:
    where its 16-bit source pages are, so ``update_layer`` can read them in
    place (2 B/param) and reuse the reject flag K3 already computed, as long
    as the tensor is unmodified (``_version``) and its pages were not taken
    again."""

    __slots__ = ("buffer", "layer", "gbuf", "version")

    def __init__(self, buffer, layer, gbuf, version):
        self.buffer, self.layer, self.gbuf, self.version = weakref.ref(buffer), layer, gbuf, version


class MasterState(_Paged):
    """FP32 masters (params, moments) per layer in fp32 page pools; mutated
    only by the updater.  ``tier`` is the reference's label (:148); the
    physical placement is HBM here (the pinned-host tier is swap.py)."""

    def __init__(self, params, tier: str = "SSD", *, page_bytes: int = PAGE_BYTES_DEFAULT,
                 device=None, layout: PageLayout | None = None, world_size: int = 1, rank: int = 0,
                 double_buffered: bool = False):
        """``double_buffered``: two copies of every state pool, the current
        one per layer selected on the device (``_state_sel``) — what the
        one-pass DP step (sharding.FusedShardedPageStep) updates
        speculatively: it writes the other copy and flips the layer only if
        the layer was applied.  Such a state is updated by that step only."""
        self._init_paged(params, page_bytes, device, layout, world_size, rank)
        self.tier = tier
        lay = self.layout
        self._db = bool(double_buffered)
        st = self._stream()
        with D.on(st):
            n = lay.elems_state * (2 if self._db else 1)
            self.p32_pool = torch.zeros(n, dtype=torch.float32, device=self.device)
            self.m32_pool = torch.zeros_like(self.p32_pool)
            self.v32_pool = torch.zeros_like(self.p32_pool)
            self._steps = torch.zeros(self.num_layers, dtype=torch.int32, device=self.device)
            self._applied = torch.zeros(self.num_layers, dtype=torch.int32, device=self.device)
            if self._db:
                self._state_sel = torch.zeros(self.num_layers, dtype=torch.int32, device=self.device)
                self._steps_spec = torch.zeros_like(self._steps)
        self._step_bound = [0] * self.num_layers
        # per layer, after a fast update_layer: (buffer ref, token of the
        # pre-published p16, the new p32 as a tensor or None, its stream)
        self._prepub = [None] * self.num_layers
        self._pout_layer = None
        for l, p in enumerate(params):
            self._pack_p32(l, p, st)

    def _current(self, pool, layer):
        """The layer's current copy of a state pool (double-buffered: the
        device's selection, read back)."""
        if not self._db:
            return pool
        es = self.layout.elems_state
        sel = int(self._state_sel[layer].item())
        return pool[sel * es:(sel + 1) * es]

    def _single_buffered(self, what: str):
        if self._db:
            raise ConfigError(f"{what}: a double-buffered MasterState is updated by the one-pass "
                              "DP step only")

    # reference attributes ------------------------------------------------------
    @property
    def p32(self):
        return _LayerView(self, self._p32_of, self._pack_p32)

    @property
    def m32(self):
        return _LayerView(self, lambda l: self._unpack(self._current(self.m32_pool, l), l))

    @property
    def v32(self):
        return _LayerView(self, lambda l: self._unpack(self._current(self.v32_pool, l), l))

    @property
    def steps(self) -> list[int]:
        return [int(x) for x in self._steps.cpu().tolist()]

    def _p32_of(self, layer):
        pre = self._prepub[layer]
        if pre is not None and pre[2] is not None and pre[3].cuda_stream == self._stream().cuda_stream:
            # the fast update_layer also wrote the new masters as a
            # contiguous tensor: handed out once, later reads unpack
            out = self._out(pre[2], layer)
            self._prepub[layer] = pre = (pre[0], pre[1], None, None)
        else:
            out = self._unpack(self._current(self.p32_pool, layer), layer)
        if isinstance(out, torch.Tensor) and pre is not None:
            # the fast update_layer already cast these values into the
            # buffer's inactive publish pages: publish() of this unmodified
            # tensor only has to flip the record
            out._hm_prepub = (pre[0], pre[1], layer, out._version)
        return out

    def _pack_p32(self, layer, value, stream=None):
        self._prepub[layer] = None
        st = self._stream(stream)
        with D.on(st):
            src = D.to_device_flat(value, self.device)
            if src.dtype != torch.float32:
                src = src.float()
        self._cast(src, N.DT_F32, self._current(self.p32_pool, layer), N.DT_F32,
                   self.layout.seg_chunks(layer, "state", owned_only=True), st)

    def _unpack(self, pool, layer, stream=None):
        st = self._stream(stream)
        with D.on(st):
            # world 1: every element is written by the unpack; sharded: the
            # pages other ranks own read as zeros
            alloc = torch.empty if self.layout.world_size == 1 else torch.zeros
            out = alloc(self.layout.numels[layer], dtype=torch.float32, device=self.device)
        self._cast(pool, N.DT_F32, out, N.DT_F32,
                   self.layout.seg_chunks(layer, "state", owned_only=True, reverse=True), st)
        return self._out(out, layer)

    def _bias(self, hyper, layers):
        for l in layers:
            self._step_bound[l] += 1
        return self._eng.bias_table(hyper, max(self._step_bound))

    def _same_pages(self, lay: PageLayout) -> bool:
        a = self.layout
        return a is lay or (a.numels == lay.numels and a.page_bytes == lay.page_bytes
                            and a.world_size == lay.world_size and a.rank == lay.rank and a.K == lay.K)

    def update_layer(self, layer: int, grad, hyper: AdamHyper, *, stream=None):
        """steps += 1; Adam over the layer's pages; on reject steps -= 1
        (lockfree.py:155-165).  numpy callers get the reference's synchronous
        bool; torch callers an ``Applied`` that synchronises only when read.

        A gradient tensor fresh from ``ParamBuffer.take`` is not re-read: the
        update streams its 16-bit source pages (g 2 B instead of 4 B/param),
        reuses the reject flag and norm its accumulate computed (no extra
        isfinite pass), and casts the new masters into the buffer's inactive
        publish pages, so the ``publish`` that follows is a record flip."""
        self._check_layer(layer)
        self._single_buffered("update_layer")
        st = self._stream(stream)
        self._prepub[layer] = None
        h = getattr(grad, "_hm_taken", None) if isinstance(grad, torch.Tensor) else None
        if h is not None:
            buf = h.buffer()
            if (buf is not None and h.layer == layer and grad._version == h.version
                    and buf._gsel[layer] != h.gbuf and self._same_pages(buf.layout)
                    and buf.device == self.device):
                return self._update_from_pages(buf, h.gbuf, layer, hyper, st)
        with D.on(st):
            g = D.to_device_flat(grad, self.device)
        n = self.layout.numels[layer]
        if g.numel() != n:
            raise ProtocolError(f"gradient has {g.numel()} elements, layer {layer} has {n}")
        eng = self._eng
        sc = eng.scratch(st)
        flag, sumsq = sc.flag, (sc.sumsq if hyper.max_norm > 0 else None)   # clip: the layer's own norm
        with D.on(st):
            flag.zero_()
            if sumsq is not None:
                sumsq.zero_()
        cc = D.contiguous_chunks_cached(n)
        D.check(N.lib().hm_reduce_stats(D.ptr(g), D.DT_OF_TORCH[g.dtype], D.ptr(eng.desc.static(cc)),
                                         len(cc), D.ptr(flag), None, D.addr(sumsq), D.sptr(st)))
        bc, bc_len = self._bias(hyper, [layer])
        with D.on(st):
            out = torch.empty(1, dtype=torch.int32, device=self.device)
        adam_launch(eng, self.layout.adam_chunks([layer], "tensor"), _group_rows([(0, 0, 0, 0)]),
                    g, D.DT_OF_TORCH[g.dtype], self.p32_pool, self.m32_pool, self.v32_pool, None, 0,
                    hyper, bc, bc_len, 0, D.ptr(self._steps) + 4 * layer, out, flag, sumsq, True, st)
        return self._applied_result(out, st)

    def _update_from_pages(self, buf, gbuf: int, layer: int, hyper, st):
        L, span = buf.num_layers, buf.layout.elems16
        lay, eng = self.layout, self._eng
        nxt = buf._psel[layer] ^ 1
        fidx = gbuf * L + layer
        chunks = lay.adam_chunks([layer], "pool")
        bc, bc_len = self._bias(hyper, [layer])
        # group 0 of the launch = this layer: steps[] is addressed at the
        # layer's counter, applied[] is the per-call result word
        rows = _group_rows([(gbuf * span, nxt * span, 0, fidx)])
        p_out = None
        with D.on(st):
            out = torch.empty(1, dtype=torch.int32, device=self.device)
            if lay.world_size == 1:
                p_out = torch.empty(lay.numels[layer], dtype=torch.float32, device=self.device)
        if len(chunks):
            # ONE launch (prologue fused); the new masters also land in p_out
            # for the p32[layer] read that follows in the reference loop
            D.check(N.lib().hm_adam_layer(
                D.ptr(eng.desc.static(chunks)), len(chunks), D.ptr(eng.desc.table(rows, st)),
                D.ptr(buf.g16_pool), buf._dt, D.ptr(self.p32_pool), D.ptr(self.m32_pool),
                D.ptr(self.v32_pool), D.ptr(buf.p16_pool), D.hyper_c(hyper), D.ptr(bc), bc_len,
                D.ptr(self._steps) + 4 * layer, D.ptr(out), D.ptr(buf._flags), D.ptr(buf._sumsq),
                D.ptr(eng.scratch(st).done), D.ptr(p_out) if p_out is not None else None,
                D.ptr(eng.desc.static(lay.adam_tensor_pos(layer))) if p_out is not None else None,
                D.sptr(st)))
        else:   # no owned page of this layer on this rank: the step bookkeeping only
            p_out = None
            adam_launch(eng, chunks, rows, buf.g16_pool, buf._dt, self.p32_pool, self.m32_pool,
                        self.v32_pool, buf.p16_pool, buf._dt, hyper, bc, bc_len, 0,
                        D.ptr(self._steps) + 4 * layer, out, buf._flags, buf._sumsq, False, st)
        # the flag is read, not consumed: a second update_layer of the same
        # tensor must see the same verdict (the reference re-checks, :133);
        # the slot stays marked for a reset before its next first message
        token = object()
        buf._prepub[layer] = (token, nxt)
        # at most one unclaimed p_out is kept (memory: one layer)
        if self._pout_layer is not None and self._prepub[self._pout_layer] is not None:
            q = self._prepub[self._pout_layer]
            self._prepub[self._pout_layer] = (q[0], q[1], None, None)
        self._prepub[layer] = (weakref.ref(buf), token, p_out, st if p_out is not None else None)
        self._pout_layer = layer if p_out is not None else None
        return self._applied_result(out, st)

    def _applied_result(self, out: torch.Tensor, st):
        if self._numpy:
            with D.on(st):
                return bool(out.item())
        return Applied(out, st)


# ---- ParamBuffer (hiermem/lockfree.py:174-263) ---------------------------------------

_RING_ROWS = 4096   # ledger rows between host resolutions (one per accumulate launch or take)


class ParamBuffer(_Paged):
    """16-bit parameter/gradient page buffers owned by the buffering actor.

    Gradients: two page buffers per layer.  ``take`` hands the active buffer
    over and switches accumulation to the other one, whose first message
    overwrites instead of adding — the reference's clear-at-take
    (lockfree.py:239) with zero clearing traffic.  Parameters: two page
    buffers per layer; a publish writes the inactive one and flips, and the
    (version, buffer, applied_iter) record swap keeps readers on the same
    stream tear-free (lockfree.py:258-262).

    Per gradient slot (buffer x layer) the producers keep three fused
    statistics next to the pages: the non-finite flag (the whole-layer
    reject), the squared norm (clipping) and the ledger's running f64 sum.
    ``ledger=False`` drops the ledger sums from the accumulate kernel (counts
    are still kept)."""

    def __init__(self, initial_params, *, dtype: str = "fp16", page_bytes: int = PAGE_BYTES_DEFAULT,
                 device=None, layout: PageLayout | None = None, ledger: bool = True,
                 world_size: int = 1, rank: int = 0, pool_alloc=None):
        if dtype not in D.TORCH16:
            raise ConfigError(f"dtype must be one of {sorted(D.TORCH16)}, got {dtype!r}")
        self._init_paged(initial_params, page_bytes, device, layout, world_size, rank)
        self.dtype = dtype
        self._t16 = D.TORCH16[dtype]
        self._dt = N.DTYPE_CODES[dtype]
        L, lay = self.num_layers, self.layout
        st = self._stream()
        with D.on(st):
            if pool_alloc is None:
                self.g16_pool = torch.zeros(2, lay.elems16, dtype=self._t16, device=self.device)
                self.p16_pool = torch.zeros(2, lay.elems16, dtype=self._t16, device=self.device)
            else:  # e.g. sharding.symmetric_alloc: peer-mapped pools for the fused DP step
                self.g16_pool = pool_alloc((2, lay.elems16), self._t16, self.device)
                self.p16_pool = pool_alloc((2, lay.elems16), self._t16, self.device)
                self.g16_pool.zero_()
                self.p16_pool.zero_()
            self._flags = torch.zeros(2 * L, dtype=torch.int32, device=self.device)
            self._sumsq = torch.zeros(2 * L, dtype=torch.float64, device=self.device)
            self._lsum = torch.zeros(2 * L, dtype=torch.float64, device=self.device) if ledger else None
            self._ring = torch.zeros(_RING_ROWS, 2 * L, dtype=torch.float64, device=self.device) \
                if ledger else None
        self._ring_pos = 0
        self._gsel = [0] * L
        self._psel = [0] * L
        self._pending = [0] * L
        self._max_iter = [-1] * L
        self._version = [0] * L
        self._applied_iter = [-1] * L
        self._prepub = [None] * L          # (token, buffer) of p16 pre-published by update_layer
        self._dirty: set[int] = set()      # slots handed over with their flag/norm not consumed
        self._snaps: list[int] = []        # taken slots whose ledger sum is still to be read
        self._snap_row = None              # (ring row, its address, stream) of those reads
        self._ledger_on = ledger
        self.ledger = ConservationLedger(L)
        if ledger:
            self.ledger._resolver = self._ledger_flush
        for l, p in enumerate(initial_params):
            with D.on(st):
                src = D.to_device_flat(p, self.device)
                if src.dtype != torch.float32:
                    src = src.float()
            self._cast(src, N.DT_F32, self.p16_pool[0], self._dt, lay.seg_chunks(l, "16"), st)

    # -- ledger ring ------------------------------------------------------------
    def _ledger_row(self) -> tuple[int, int]:
        """(row, device address) of a fresh ledger row (2L doubles, zeroed)."""
        if self._ring_pos == _RING_ROWS:
            self._ledger_flush()
        r = self._ring_pos
        self._ring_pos += 1
        return r, D.ptr(self._ring) + r * self._ring.shape[1] * 8

    def _ledger_flush(self) -> None:
        """Resolve every pending ledger entry from the device rows (one
        synchronisation), then recycle the rows."""
        self._flush_snaps()
        if not self._ring_pos:
            return
        torch.cuda.synchronize(self.device)
        host = self._ring[:self._ring_pos].cpu().numpy()
        self.ledger._resolve(host)
        self._ring[:self._ring_pos].zero_()
        torch.cuda.synchronize(self.device)   # rows are zero before any stream reuses them
        self._ring_pos = 0

    def _defer_snap(self, fidx: int, layer: int, stream) -> None:
        """record_take of a three-call ``take`` (lockfree.py:237): the slot's
        running ledger sum is read later, by one launch for every take since
        the last flush.  A handed-over slot's sum cannot change before the
        flush: the flush runs before any accumulate launch (the only writer)
        and before any ledger read."""
        if self._snap_row is not None and self._snap_row[2].cuda_stream != stream.cuda_stream:
            self._flush_snaps()
        if self._snap_row is None:
            row, rptr = self._ledger_row()
            self._snap_row = (row, rptr, stream)
        self.ledger._pend(self.ledger._consumed[layer], self._snap_row[0], 2 * len(self._snaps))
        self._snaps.append(fidx)
        if len(self._snaps) == self.num_layers:     # one ring row holds L (sum, flag) pairs
            self._flush_snaps()

    def _flush_snaps(self, stream=None) -> None:
        """Launch the deferred take snapshots (snapshot + reset of each slot's
        ledger sum); ``stream``, when it differs, waits for them."""
        if not self._snaps:
            return
        _row, rptr, st = self._snap_row
        slots = np.asarray(self._snaps, np.uint32)
        self._snaps, self._snap_row = [], None
        D.check(N.lib().hm_stats_take(D.ptr(self._eng.desc.table(slots, st)), len(slots), None, None,
                                      D.ptr(self._lsum), rptr, D.sptr(st)))
        if stream is not None and stream.cuda_stream != st.cuda_stream:
            ev = torch.cuda.Event()
            ev.record(st)
            stream.wait_event(ev)

    def _reset_dirty(self, slots, stream) -> None:
        """Reset the flag / norm / ledger sum of slots about to take a first
        message, if a hand-over left them unconsumed (one launch)."""
        hit = [f for f in slots if f in self._dirty]
        if not hit:
            return
        D.check(N.lib().hm_stats_take(D.ptr(self._eng.desc.table(np.asarray(hit, np.uint32), stream)),
                                      len(hit), D.ptr(self._flags), D.ptr(self._sumsq),
                                      D.ptr(self._lsum), None, D.sptr(stream)))
        self._dirty.difference_update(hit)

    def _record_consumed(self, layers, row: int) -> None:
        """The take of ``layers`` wrote (sum, flag) pairs to ledger row ``row``."""
        for i, l in enumerate(layers):
            self.ledger._pend(self.ledger._consumed[l], row, 2 * i)

    def _record_applies(self, layers, row: int) -> None:
        for i, l in enumerate(layers):
            self.ledger._apply_pending.append((l, row, 2 * i, 2 * i + 1))

    # -- reads ------------------------------------------------------------------
    def read(self, layer: int):
        """Snapshot (version, 16-bit params, applied_iter) (lockfree.py:194-196)."""
        self._check_layer(layer)
        return (self._version[layer], self._unpack16(self.p16_pool[self._psel[layer]], layer, True),
                self._applied_iter[layer])

    def version(self, layer: int) -> int:
        return self._version[layer]

    def applied_iter(self, layer: int) -> int:
        return self._applied_iter[layer]

    def min_applied_iter(self) -> int:
        return min(self._applied_iter)

    def total_pending(self) -> int:
        return sum(self._pending)

    @property
    def g16(self):
        return _LayerView(self, self._g16_of)

    def _g16_of(self, layer):
        if self._pending[layer] == 0:  # logically cleared (taken or published)
            t = torch.zeros(self.layout.numels[layer], dtype=self._t16, device=self.device)
            return self._out(t, layer)
        return self._unpack16(self.g16_pool[self._gsel[layer]], layer)

    def layer_view(self, layer: int, buf: int | None = None, *, stream=None) -> torch.Tensor:
        """The layer's 16-bit parameters in published buffer ``buf`` (default:
        the current record) as a CUDA tensor of the layer's shape: a zero-copy
        view when its page segments are contiguous in the pool (tensors
        allocated in order usually are), otherwise an unpacked copy."""
        buf = self._psel[layer] if buf is None else buf
        lay = self.layout
        segs = lay.segments[layer]
        base = lay.slot16(segs[0].page) * lay.E + segs[0].off
        pos = base
        for s in segs:
            if lay.slot16(s.page) * lay.E + s.off != pos:
                return self._unpack16(self.p16_pool[buf], layer, stream=stream, raw=True).view(
                    self._shapes[layer])
            pos += s.n
        return self.p16_pool[buf][base:pos].view(self._shapes[layer])

    def _unpack16(self, pool, layer, readonly=False, stream=None, raw=False):
        st = self._stream(stream)
        with D.on(st):
            out = torch.empty(self.layout.numels[layer], dtype=self._t16, device=self.device)
        self._cast(pool, self._dt, out, self._dt, self.layout.seg_chunks(layer, "16", reverse=True), st)
        return out if raw else self._out(out, layer, readonly)

    # -- writes -----------------------------------------------------------------
    def _k3(self, src, src_dt, chunks, modes, slots, layers, stream, iteration) -> None:
        """One accumulate launch (K3) + the host bookkeeping of its messages."""
        self._flush_snaps(stream)
        self._reset_dirty([f for f, m in zip(slots, modes) if not m], stream)
        row = None
        if self._ledger_on:
            row, rptr = self._ledger_row()
        dmodes = None
        if len(set(modes)) > 1:
            m = np.zeros(2 * self.num_layers, dtype=np.uint8)
            m[list(slots)] = modes
            dmodes = self._eng.desc.table(m, stream)
        D.check(N.lib().hm_accumulate(
            D.ptr(src), src_dt, D.ptr(self.g16_pool), self._dt,
            D.ptr(self._eng.desc.static(chunks)), len(chunks), modes[0] if dmodes is None else 0,
            D.ptr(dmodes), D.ptr(self._flags), D.ptr(self._sumsq),
            D.ptr(self._lsum) if self._ledger_on else None, rptr if self._ledger_on else None,
            None, D.sptr(stream)))
        for l, f in zip(layers, slots):
            if row is not None:
                self.ledger._pend(self.ledger._produced[l], row, f)
            self.ledger.messages_accumulated[l] += 1
            self._pending[l] += 1
            self._max_iter[l] = max(self._max_iter[l], iteration)

    def _acc_plan(self, layers, base_of) -> np.ndarray:
        """hm_seg_chunk plan accumulating a flat source into the CURRENT
        gradient buffers of ``layers`` (cached per buffer selection)."""
        L, lay = self.num_layers, self.layout
        sel = tuple(self._gsel[l] for l in layers)
        cache = self.__dict__.setdefault("_acc_plans", {})
        key = (tuple(layers), sel, base_of is None)
        if key not in cache:
            parts = []
            for l, b in zip(layers, sel):
                c = lay.seg_chunks(l, "16").copy()
                if base_of is not None:
                    c["src_off"] += base_of(l)
                c["dst_off"] += b * lay.elems16
                c["slot"] = b * L + l
                parts.append(c)
            cache[key] = np.concatenate(parts)
        return cache[key]

    def accumulate(self, msg: GradMessage, *, stream=None) -> None:
        """g16 = rn16(f32(g16) + f32(payload)) over the layer's pages, with the
        layer's non-finite flag, squared norm and ledger sum fused in
        (lockfree.py:210-224)."""
        layer = msg.layer
        if not (0 <= layer < self.num_layers):
            raise ProtocolError(f"gradient for unknown layer {layer}")
        if _shape(msg.payload) != self._shapes[layer]:
            raise ProtocolError(f"gradient shape {_shape(msg.payload)} != buffer shape "
                                f"{self._shapes[layer]} for layer {layer}")
        st = self._stream(stream)
        with D.on(st):
            src = D.to_device_flat(msg.payload, self.device)
        f = self._gsel[layer] * self.num_layers + layer
        self._k3(src, D.DT_OF_TORCH[src.dtype], self._acc_plan([layer], None),
                 [1 if self._pending[layer] > 0 else 0], [f], [layer], st, msg.iteration)

    def accumulate_flat(self, flat, iteration: int, *, stream=None) -> None:
        """Accumulate one flat gradient covering every layer in order (the
        layout a backward pass writes) with ONE K3 launch: the same arithmetic,
        flags and ledger entries as one ``accumulate`` per layer."""
        L, lay = self.num_layers, self.layout
        st = self._stream(stream)
        with D.on(st):
            src = D.to_device_flat(flat, self.device)
        if src.numel() != sum(lay.numels):
            raise ProtocolError(f"flat gradient has {src.numel()} elements, layers hold "
                                f"{sum(lay.numels)}")
        starts = self.__dict__.setdefault("_starts", np.cumsum([0] + lay.numels[:-1]))
        layers = list(range(L))
        self._k3(src, D.DT_OF_TORCH[src.dtype], self._acc_plan(layers, lambda l: int(starts[l])),
                 [1 if self._pending[l] > 0 else 0 for l in layers],
                 [self._gsel[l] * L + l for l in layers], layers, st, iteration)

    def _hand_over(self, layer: int):
        """Clear-at-take bookkeeping shared by every update path: the active
        gradient buffer is handed over and accumulation flips to the other."""
        buf = self._gsel[layer]
        count, newest = self._pending[layer], self._max_iter[layer]
        self.ledger.messages_consumed[layer] += count
        self._gsel[layer] = buf ^ 1
        self._pending[layer] = 0
        return buf, count, newest

    def _published(self, layer: int, applied_iter=None) -> int:
        """Flip the record to the inactive buffer just written (lockfree.py:258-262)."""
        self._psel[layer] ^= 1
        self._version[layer] += 1
        self._prepub[layer] = None
        if applied_iter is not None:
            self._applied_iter[layer] = applied_iter
        return self._version[layer]

    def take(self, layer: int, *, stream=None):
        """Atomically hand over and clear the accumulated gradient: returns
        (grad fp32, message_count, newest_iteration) or None (lockfree.py:226-241)."""
        self._check_layer(layer)
        if self._pending[layer] == 0:
            return None
        st = self._stream(stream)
        buf, count, newest = self._hand_over(layer)
        with D.on(st):
            g = torch.empty(self.layout.numels[layer], dtype=torch.float32, device=self.device)
        self._cast(self.g16_pool[buf], self._dt, g, N.DT_F32,
                   self.layout.seg_chunks(layer, "16", reverse=True), st)
        fidx = buf * self.num_layers + layer
        if self._ledger_on:   # record_take: snapshot + reset of the running sum, deferred
            self._defer_snap(fidx, layer, st)
        # the reject flag and norm stay for an update_layer of this tensor;
        # otherwise they are reset before the slot's next first message
        self._dirty.add(fidx)
        out = self._out(g, layer)
        if isinstance(out, torch.Tensor):
            out._hm_taken = _Taken(self, layer, buf, out._version)
        return out, count, newest

    def publish(self, layer: int, p32, applied_iter: int | None = None, clear: bool = True,
                *, stream=None) -> int:
        """Install fresh 16-bit params (RNE cast into the inactive page buffer,
        then flip); with ``clear`` also drop pending gradients (lockfree.py:243-263)."""
        self._check_layer(layer)
        st = self._stream(stream)
        if clear:
            self._flush_snaps(st)
            if self._pending[layer]:
                fidx = self._gsel[layer] * self.num_layers + layer
                row = rptr = None
                if self._ledger_on:
                    row, rptr = self._ledger_row()
                D.check(N.lib().hm_stats_take(D.ptr(self._eng.desc.table(np.array([fidx], np.uint32), st)),
                                              1, D.ptr(self._flags), D.ptr(self._sumsq),
                                              D.ptr(self._lsum), rptr, D.sptr(st)))
                if row is not None:
                    self._record_consumed([layer], row)
                self._dirty.discard(fidx)
                self.ledger.messages_consumed[layer] += self._pending[layer]
            elif self._ledger_on:
                self.ledger._consumed[layer].append(0.0)
            self._pending[layer] = 0
        tag = getattr(p32, "_hm_prepub", None) if isinstance(p32, torch.Tensor) else None
        pre = self._prepub[layer]
        if (tag is not None and pre is not None and tag[0]() is self and tag[1] is pre[0]
                and tag[2] == layer and p32._version == tag[3] and pre[1] == self._psel[layer] ^ 1):
            return self._published(layer, applied_iter)   # update_layer already cast these values
        with D.on(st):
            src = D.to_device_flat(p32, self.device)
            if src.dtype != torch.float32:
                src = src.float()
        if src.numel() != self.layout.numels[layer]:
            raise ProtocolError(f"publish: {src.numel()} elements for layer {layer} of "
                                f"{self.layout.numels[layer]}")
        nxt = self._psel[layer] ^ 1
        self._cast(src, N.DT_F32, self.p16_pool[nxt], self._dt, self.layout.seg_chunks(layer, "16"), st)
        return self._published(layer, applied_iter)


def publish_params(buffer: ParamBuffer, layer: int, p32) -> None:
    """Clear buffered gradients, then publish 16-bit params (version += 1)."""
    buffer.publish(layer, p32, clear=True)


def accumulate_gradient(buffer: ParamBuffer, msg: GradMessage) -> None:
    buffer.accumulate(msg)


# ---- the fused hot path ---------------------------------------------------------

class SweepResult:
    """Outcome of one fused sweep; ``applied()`` synchronises lazily."""

    def __init__(self, masters: MasterState, layers, counts, newest):
        self._m = masters
        self.layers = tuple(layers)
        self.counts = tuple(counts)
        self.newest = tuple(newest)

    def applied(self) -> dict[int, bool]:
        a = self._m._applied.cpu().tolist()
        return {l: bool(a[l]) for l in self.layers}


class UpdateTicket:
    """One update of a set of layers over a ParamBuffer, shared by every
    update path (fused sweep, pinned-host / SSD swap sweeps, DP steps): the
    hand-over (take), the prologue's group rows, the ledger row that records
    what was consumed and applied, and the publish flip at the end."""

    def __init__(self, buffer: ParamBuffer, layers, flag_of=None):
        self.buffer = buffer
        self.layers = list(layers)
        L, span = buffer.num_layers, buffer.layout.elems16
        buffer._flush_snaps(buffer._stream())
        rows, self.counts, self.newest = [], [], []
        for l in self.layers:
            gbuf, count, new = buffer._hand_over(l)
            rows.append((gbuf * span, (buffer._psel[l] ^ 1) * span, l,
                         gbuf * L + l if flag_of is None else flag_of(l)))
            self.counts.append(count)
            self.newest.append(new)
        self.groups = _group_rows(rows)
        self.row = None
        self.ledger_out = 0
        if buffer._ledger_on:
            self.row, self.ledger_out = buffer._ledger_row()

    def lsum(self, base_slot: int = 0) -> int:
        """Address of the ledger running sums as the prologue indexes them
        (``base_slot`` shifts it when the prologue's flags are not the buffer's)."""
        b = self.buffer
        return D.ptr(b._lsum) + 8 * base_slot if b._ledger_on else 0

    def finish(self, consumed_flags: bool = True) -> None:
        """Record the ledger entries and flip every layer's published record.
        ``consumed_flags=False``: the prologue consumed other flags (DP steps),
        so the buffer's own slots are reset before their next first message."""
        b = self.buffer
        L = b.num_layers
        for l, new in zip(self.layers, self.newest):
            b._published(l, new)
        slots = [int(r["flag"]) for r in self.groups]
        if consumed_flags:
            b._dirty.difference_update(slots)
        else:
            b._dirty.update(int(r["g_shift"]) // b.layout.elems16 * L + l
                            for r, l in zip(self.groups, self.layers))
        if self.row is not None:
            b._record_consumed(self.layers, self.row)
            b._record_applies(self.layers, self.row)


def update_prologue(ticket: UpdateTicket, masters, hyper, stream, *, flags=None, sumsq=None,
                    lsum: int | None = None):
    """The ticket's prologue (reject / step / bias lookup, ledger record) for
    callers that run the main pass themselves (swap tiers, DP steps).
    ``flags`` / ``sumsq`` default to the buffer's own fused statistics.
    Returns (device group table, rt scratch, hyper struct) for the main pass,
    which must run on ``stream`` (the rt scratch is the stream's)."""
    b = ticket.buffer
    eng = masters._eng
    pre = getattr(masters, "_prepub", None)
    if pre is not None:    # a fast update_layer's pre-published results are stale now
        for l in ticket.layers:
            pre[l] = None
    dgroups = eng.desc.table(ticket.groups, stream)
    rt = eng.rt_scratch(len(ticket.groups), stream)
    bc, bc_len = masters._bias(hyper, ticket.layers)
    hc = D.hyper_c(hyper)
    D.check(N.lib().hm_adam_prologue(
        D.ptr(dgroups), len(ticket.groups), D.ptr(rt), hc, D.ptr(bc), bc_len, 0, D.ptr(masters._steps),
        D.ptr(masters._applied), D.addr(b._flags if flags is None else flags),
        D.addr(b._sumsq if sumsq is None else sumsq), 1, (ticket.lsum() if lsum is None else lsum) or None,
        ticket.ledger_out or None, D.sptr(stream)))
    return dgroups, rt, hc


def sweep(buffer: ParamBuffer, masters: MasterState, hyper: AdamHyper, layers=None, *,
          stream=None, opts=None) -> SweepResult:
    """The updating actor's per-layer loop body (hiermem/lockfree.py:624-639):
    for every layer with pending gradients, take (clear) -> update_layer ->
    publish(clear=False, applied_iter=newest), fused into ONE prologue and
    ONE page-Adam launch over all their page segments: reads g16 + p/m/v
    (14 B/param), writes p/m/v + p16 (14 B/param).  Asynchronous; the
    whole-layer reject and step rollback happen on the device.  With
    ``hyper.max_norm > 0`` the clip norm is that of the swept layers."""
    lay = buffer.layout
    if masters.layout.numels != lay.numels or masters.layout.page_bytes != lay.page_bytes \
            or masters.layout.world_size != lay.world_size:
        raise ConfigError("buffer and masters were built on different page tables")
    masters._single_buffered("sweep")
    st = buffer._stream(stream)
    order = list(reversed(range(buffer.num_layers))) if layers is None else list(layers)
    sel = [l for l in order if buffer._pending[l] > 0]
    if not sel:
        return SweepResult(masters, [], [], [])
    t = UpdateTicket(buffer, sel)
    bc, bc_len = masters._bias(hyper, sel)
    for l in sel:
        masters._prepub[l] = None
    adam_launch(masters._eng, lay.adam_chunks(sel, "pool"), t.groups,
                buffer.g16_pool, buffer._dt, masters.p32_pool, masters.m32_pool, masters.v32_pool,
                buffer.p16_pool, buffer._dt, hyper, bc, bc_len, 0, masters._steps, masters._applied,
                buffer._flags, buffer._sumsq, True, st, lsum=t.lsum(), ledger_out=t.ledger_out, opts=opts)
    t.finish()
    return SweepResult(masters, sel, t.counts, t.newest)


class _MultiResult(SweepResult):
    def __init__(self, masters, parts):
        super().__init__(masters, [l for p in parts for l in p.layers],
                         [c for p in parts for c in p.counts], [n for p in parts for n in p.newest])


def layer_groups(numels, groups: int) -> list[list[int]]:
    """Contiguous layer ranges of about equal element count."""
    total = sum(numels)
    out, cur, acc = [], [], 0
    for l, n in enumerate(numels):
        cur.append(l)
        acc += n
        if acc >= total * (len(out) + 1) / groups and len(out) < groups - 1:
            out.append(cur)
            cur = []
    if cur:
        out.append(cur)
    return out


def ingest(buffer: ParamBuffer, host_grad, iteration: int = 0, *, groups: int = 8, stream=None,
           copy_stream=None, after_group=None) -> list:
    """Accumulate a flat gradient that sits in (pinned) host memory, one
    contiguous layer group at a time: cudaMemcpyAsync of the group's slice on
    a copy stream -> K3 into its pages on ``stream`` when it lands, so the
    PCIe transfer of group k+1 overlaps whatever runs after group k
    (``after_group(layers)`` is called right after the group's K3 is queued).
    Returns one event per group, recorded after its K3: a consumer on another
    stream (the pipelined DP step) waits on it."""
    lay = buffer.layout
    st = buffer._stream(stream)
    cache = buffer.__dict__.setdefault("_ingest", {})
    key = ("plan", groups)
    if key not in cache:
        cache[key] = layer_groups(lay.numels, groups)
    if "staging" not in cache:
        cache["staging"] = torch.empty(sum(lay.numels), dtype=buffer._t16, device=buffer.device)
        cache["copy"] = copy_stream or torch.cuda.Stream(buffer.device)
        cache["starts"] = np.cumsum([0] + lay.numels[:-1])
    plan, staging, cs, starts = cache[key], cache["staging"], cache["copy"], cache["starts"]
    src = host_grad.reshape(-1)
    if src.dtype != buffer._t16 or src.numel() != staging.numel():
        raise ProtocolError(f"host gradient must be {buffer._t16} with {staging.numel()} elements")
    L = buffer.num_layers
    done = []
    cs.wait_stream(st)   # the staging slice is free once the previous step consumed it
    for grp in plan:
        a, b = int(starts[grp[0]]), int(starts[grp[-1]] + lay.numels[grp[-1]])
        with torch.cuda.stream(cs):
            staging[a:b].copy_(src[a:b], non_blocking=True)
            landed = torch.cuda.Event()
            landed.record(cs)
        st.wait_event(landed)
        buffer._k3(staging, buffer._dt, buffer._acc_plan(grp, lambda l: int(starts[l])),
                   [1 if buffer._pending[l] > 0 else 0 for l in grp],
                   [buffer._gsel[l] * L + l for l in grp], grp, st, iteration)
        ev = torch.cuda.Event()
        ev.record(st)
        done.append(ev)
        if after_group is not None:
            after_group(grp)
    return done


def ingest_sweep(buffer: ParamBuffer, masters: MasterState, host_grad, hyper: AdamHyper,
                 iteration: int = 0, *, groups: int = 8, stream=None, copy_stream=None,
                 results_to=None) -> SweepResult:
    """One update step fed by a flat gradient in (pinned) host memory — what a
    host-side producer hands the updating actor.  Per contiguous layer group:
    cudaMemcpyAsync of the group's slice on a copy stream -> K3 accumulate
    into its pages when it lands -> fused sweep of the group, so the PCIe
    transfer of group k+1 overlaps the update of group k and the step costs
    about one transfer of the gradient (the reference's fetch/offload are
    DelayModel sleeps, hiermem/lockfree.py:90-94, 562-569).

    ``results_to`` (a pinned host 16-bit tensor of every layer's elements in
    layer order): each group's freshly published parameters are copied back
    to the host on a second copy stream right after the group's update, so
    the D2H of group k overlaps the H2D of group k+1 (PCIe is full duplex) —
    the step returns its result, not just the applied flags.

    Global grad-norm clipping needs every group's norm before the first
    update, so it is refused here (use accumulate + ``sweep``)."""
    if getattr(hyper, "max_norm", 0.0) > 0:
        raise ConfigError("ingest_sweep updates group by group: global grad-norm clipping "
                          "(max_norm > 0) needs the whole gradient first; use accumulate_flat + sweep")
    st = buffer._stream(stream)
    parts = []
    d2h = None
    if results_to is not None:
        lay = buffer.layout
        if results_to.dtype != buffer._t16 or results_to.numel() != sum(lay.numels):
            raise ProtocolError(f"results_to must be {buffer._t16} with {sum(lay.numels)} elements")
        cache = buffer.__dict__.setdefault("_ingest", {})
        d2h = cache.setdefault("d2h", torch.cuda.Stream(buffer.device))
        starts = cache.setdefault("starts", np.cumsum([0] + lay.numels[:-1]))

    def after(grp):
        parts.append(sweep(buffer, masters, hyper, layers=list(reversed(grp)), stream=st))
        if d2h is not None:
            _publish_to_host(buffer, grp, results_to, starts, st, d2h)

    ingest(buffer, host_grad, iteration, groups=groups, stream=st, copy_stream=copy_stream,
           after_group=after)
    if d2h is not None:
        st.wait_stream(d2h)
    return _MultiResult(masters, parts)


def _publish_to_host(buffer: ParamBuffer, grp, host, starts, st, d2h, *, owned_only: bool = False,
                     pbuf=None) -> None:
    """D2H of the published pages of layer group ``grp`` into the flat host
    tensor: one cudaMemcpyAsync per contiguous run of the pool (layers
    allocated in order are one run), queued on ``d2h`` behind the group's
    update on ``st``.  ``owned_only``: only this rank's pages (a DP step's
    ranks return disjoint pieces); ``pbuf``: the publish buffer to read
    (default: each layer's current record)."""
    lay = buffer.layout
    cache = buffer.__dict__.setdefault("_d2h_runs", {})
    sel = tuple(buffer._psel[l] if pbuf is None else pbuf for l in grp)
    key = (tuple(grp), sel, owned_only)
    if key not in cache:
        runs = []
        E, esz = lay.E, 2
        for l, b in zip(grp, sel):
            base = int(starts[l])
            for s in lay.segments[l]:
                if owned_only and not lay.owned(s):
                    continue
                src = (b * lay.elems16 + lay.slot16(s.page) * E + s.off) * esz
                dst = (base + s.pos) * esz
                if runs and runs[-1][0] + runs[-1][2] == src and runs[-1][1] + runs[-1][2] == dst:
                    runs[-1][2] += s.n * esz
                else:
                    runs.append([src, dst, s.n * esz])
        cache[key] = np.array([tuple(r) for r in runs], dtype=N.COPY_DESC)
    runs = cache[key]
    if not len(runs):
        return
    ev = torch.cuda.Event()
    ev.record(st)
    d2h.wait_event(ev)
    D.check(N.lib().hm_memcpy_runs(D.ptr(buffer.p16_pool), D.ptr(host), runs.ctypes.data, len(runs), 2,
                                   D.sptr(d2h)))
