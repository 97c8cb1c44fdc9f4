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
    and ``max_norm`` (global grad-norm clip, <= 0 disables)."""

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


class ConservationLedger:
    """Gradient conservation bookkeeping (hiermem/lockfree.py:275-326):
    per-layer f64 produced deltas, consumed and applied sums and message
    counts; balanced iff fsum(produced) == fsum(consumed) == fsum(applied +
    rejected) and the counts agree.  Sums are device f64 reductions, so they
    are recorded only when the owning buffer was built with ``ledger=True``."""

    def __init__(self, num_layers: int):
        self.produced_deltas = [[] for _ in range(num_layers)]
        self.consumed_sums = [[] for _ in range(num_layers)]
        self.applied_sums = [[] for _ in range(num_layers)]
        self.rejected_sums = [[] for _ in range(num_layers)]
        self.messages_sent = [0] * num_layers
        self.messages_accumulated = [0] * num_layers
        self.messages_consumed = [0] * num_layers

    def record_accumulate(self, layer: int, delta: float) -> None:
        self.produced_deltas[layer].append(delta)
        self.messages_accumulated[layer] += 1

    def record_take(self, layer: int, total: float, count: int) -> None:
        self.consumed_sums[layer].append(total)
        self.messages_consumed[layer] += count

    def record_apply(self, layer: int, total: float, rejected: bool) -> None:
        (self.rejected_sums if rejected else self.applied_sums)[layer].append(total)

    def summary(self) -> dict:
        out, balanced = [], True
        for l in range(len(self.produced_deltas)):
            sums = [math.fsum(x) for x in (self.produced_deltas[l], self.consumed_sums[l],
                                            self.applied_sums[l], self.rejected_sums[l])]
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


class _Engine:
    """Per-device descriptor cache, rt scratch and bias tables."""

    _per_device: dict = {}

    def __init__(self, device):
        self.device = device
        self.desc = D.DescCache(device)
        self.bias: dict[tuple[float, float], D.BiasTable] = {}
        self.rt = torch.empty(0, dtype=torch.uint8, device=device)
        self.flag = torch.zeros(1, dtype=torch.int32, device=device)
        self.sumsq = torch.zeros(1, dtype=torch.float64, device=device)

    @classmethod
    def of(cls, device) -> "_Engine":
        key = str(device)
        if key not in cls._per_device:
            cls._per_device[key] = cls(device)
        return cls._per_device[key]

    def rt_scratch(self, n_groups: int) -> torch.Tensor:
        need = max(1, n_groups) * N.GROUP_RT_BYTES
        if self.rt.numel() < need:
            self.rt = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self.rt

    def bias_table(self, hyper, max_step: int):
        key = (float(hyper.beta1), float(hyper.beta2))
        if key not in self.bias:
            self.bias[key] = D.BiasTable(key[0], key[1], self.device)
        return self.bias[key].ensure(max_step)


def adam_launch(engine: _Engine, chunks: np.ndarray, groups: np.ndarray, g, g_dt: int,
                p32, m32, v32, p16, p16_dt: int, hyper, bc_dev, bc_len: int,
                explicit_step: int, steps, applied, nonfinite, sumsq, consume: bool, stream,
                static_chunks: bool = True) -> None:
    """One fused page-Adam step (prologue + main kernel) on ``stream``."""
    dchunks = engine.desc.static(chunks) if static_chunks else engine.desc.table(chunks)
    dgroups = engine.desc.table(groups)
    rt = engine.rt_scratch(len(groups))
    hc = D.hyper_c(hyper)
    D.check(N.lib().hm_adam_step(
        D.ptr(dchunks), len(chunks), D.ptr(dgroups), len(groups), D.ptr(rt),
        D.ptr(g), g_dt, D.ptr(p32), D.ptr(m32), D.ptr(v32), D.ptr(p16), p16_dt,
        hc, D.ptr(bc_dev), bc_len, explicit_step, D.ptr(steps), D.ptr(applied),
        D.ptr(nonfinite), D.ptr(sumsq), 1 if consume else 0, D.sptr(stream)))


def _group_rows(rows) -> np.ndarray:
    a = np.zeros(len(rows), dtype=N.GROUP_LAUNCH)
    for i, (gs, ps, grp, flag) in enumerate(rows):
        a[i] = (gs, ps, grp, flag)
    return a


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
    with torch.cuda.stream(st):
        p = D.to_device_flat(p32, device).to(torch.float32).clone()
        m = D.to_device_flat(m32, device).to(torch.float32).clone()
        v = D.to_device_flat(v32, device).to(torch.float32).clone()
        g = D.to_device_flat(grad, device)
    n = p.numel()
    if m.numel() != n or v.numel() != n or g.numel() != n:
        raise ProtocolError(f"apply_update: size mismatch p={n} m={m.numel()} v={v.numel()} g={g.numel()}")
    if n == 0:
        return p32, m32, v32, True
    with torch.cuda.stream(st):
        bc = torch.tensor([float(np.float32(1.0 - hyper.beta1 ** step)),
                           float(np.float32(1.0 - hyper.beta2 ** step))], dtype=torch.float32, device=device)
        flag = torch.zeros(1, dtype=torch.int32, device=device)
        applied = torch.zeros(1, dtype=torch.int32, device=device)
    D.check(N.lib().hm_reduce_stats(D.ptr(g), D.DT_OF_TORCH[g.dtype],
                                     D.ptr(eng.desc.static(D.contiguous_chunks_cached(n))), len(D.contiguous_chunks_cached(n)),
                                     D.ptr(flag), None, None, D.sptr(st)))
    adam_launch(eng, D.contiguous_adam_chunks(n), _group_rows([(0, 0, 0, 0)]), g, D.DT_OF_TORCH[g.dtype],
                p, m, v, None, 0, hyper, bc, 1, int(step), None, applied, flag, None, True, st,
                static_chunks=False)
    with torch.cuda.stream(st):
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

class MasterState(_Paged):
    """FP32 masters (params, moments) per layer in fp32 page pools; mutated
    only by the updater.  ``tier`` is the reference's label (:148); the
    physical placement is HBM here (the pinned-host tier is swap.py)."""

    def __init__(self, params, tier: str = "SSD", *, page_bytes: int = PAGE_BYTES_DEFAULT,
                 device=None, layout: PageLayout | None = None, world_size: int = 1, rank: int = 0):
        self._init_paged(params, page_bytes, device, layout, world_size, rank)
        self.tier = tier
        lay = self.layout
        st = self._stream()
        with torch.cuda.stream(st):
            self.p32_pool = torch.zeros(lay.elems_state, dtype=torch.float32, device=self.device)
            self.m32_pool = torch.zeros_like(self.p32_pool)
            self.v32_pool = torch.zeros_like(self.p32_pool)
            self._steps = torch.zeros(self.num_layers, dtype=torch.int32, device=self.device)
            self._applied = torch.zeros(self.num_layers, dtype=torch.int32, device=self.device)
        self._step_bound = [0] * self.num_layers
        for l, p in enumerate(params):
            self._pack_p32(l, p, st)

    # reference attributes ------------------------------------------------------
    @property
    def p32(self):
        return _LayerView(self, lambda l: self._unpack(self.p32_pool, l), self._pack_p32)

    @property
    def m32(self):
        return _LayerView(self, lambda l: self._unpack(self.m32_pool, l))

    @property
    def v32(self):
        return _LayerView(self, lambda l: self._unpack(self.v32_pool, l))

    @property
    def steps(self) -> list[int]:
        return [int(x) for x in self._steps.cpu().tolist()]

    def _pack_p32(self, layer, value, stream=None):
        st = self._stream(stream)
        with torch.cuda.stream(st):
            src = D.to_device_flat(value, self.device)
            if src.dtype != torch.float32:
                src = src.float()
        self._cast(src, N.DT_F32, self.p32_pool, N.DT_F32,
                   self.layout.seg_chunks(layer, "state", owned_only=True), st)

    def _unpack(self, pool, layer, stream=None):
        st = self._stream(stream)
        with torch.cuda.stream(st):
            out = torch.zeros(self.layout.numels[layer], dtype=torch.float32, device=self.device)
        self._cast(pool, N.DT_F32, out, N.DT_F32,
                   self.layout.seg_chunks(layer, "state", owned_only=True, reverse=True), st)
        return self._out(out, layer)

    def _bias(self, hyper, layers):
        for l in layers:
            self._step_bound[l] += 1
        return self._eng.bias_table(hyper, max(self._step_bound))

    def update_layer(self, layer: int, grad, hyper: AdamHyper, *, stream=None) -> bool:
        """steps += 1; Adam over the layer's pages; on reject steps -= 1
        (lockfree.py:155-165).  Synchronous bool result like the reference."""
        self._check_layer(layer)
        st = self._stream(stream)
        with torch.cuda.stream(st):
            g = D.to_device_flat(grad, self.device)
        n = self.layout.numels[layer]
        if g.numel() != n:
            raise ProtocolError(f"gradient has {g.numel()} elements, layer {layer} has {n}")
        eng = self._eng
        with torch.cuda.stream(st):
            eng.flag.zero_()
        cc = D.contiguous_chunks_cached(n)
        D.check(N.lib().hm_reduce_stats(D.ptr(g), D.DT_OF_TORCH[g.dtype], D.ptr(eng.desc.static(cc)),
                                         len(cc), D.ptr(eng.flag), None, None, D.sptr(st)))
        bc, bc_len = self._bias(hyper, [layer])
        adam_launch(eng, self.layout.adam_chunks([layer], "tensor"), _group_rows([(0, 0, layer, 0)]),
                    g, D.DT_OF_TORCH[g.dtype], self.p32_pool, self.m32_pool, self.v32_pool, None, 0,
                    hyper, bc, bc_len, 0, self._steps, self._applied, eng.flag, None, True, st)
        with torch.cuda.stream(st):
            return bool(self._applied[layer].item())


# ---- ParamBuffer (hiermem/lockfree.py:174-263) ---------------------------------------

class ParamBuffer(_Paged):
    """16-bit parameter/gradient page buffers owned by the buffering actor.

    Gradients: two page buffers per layer.  ``take`` hands the active buffer
    over and switches accumulation to the other one, whose first message
    overwrites instead of adding — the reference's clear-at-take
    (lockfree.py:239) with zero clearing traffic.  Parameters: two page
    buffers per layer; a publish writes the inactive one and flips, and the
    (version, buffer, applied_iter) record swap keeps readers on the same
    stream tear-free (lockfree.py:258-262)."""

    def __init__(self, initial_params, *, dtype: str = "fp16", page_bytes: int = PAGE_BYTES_DEFAULT,
                 device=None, layout: PageLayout | None = None, ledger: bool = False,
                 world_size: int = 1, rank: int = 0, pool_alloc=None):
        if dtype not in D.TORCH16:
            raise ConfigError(f"dtype must be one of {sorted(D.TORCH16)}, got {dtype!r}")
        self._init_paged(initial_params, page_bytes, device, layout, world_size, rank)
        self.dtype = dtype
        self._t16 = D.TORCH16[dtype]
        self._dt = N.DTYPE_CODES[dtype]
        L, lay = self.num_layers, self.layout
        st = self._stream()
        with torch.cuda.stream(st):
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
        self._gsel = [0] * L
        self._psel = [0] * L
        self._pending = [0] * L
        self._max_iter = [-1] * L
        self._version = [0] * L
        self._applied_iter = [-1] * L
        self._ledger_on = ledger
        self.ledger = ConservationLedger(L)
        for l, p in enumerate(initial_params):
            with torch.cuda.stream(st):
                src = D.to_device_flat(p, self.device)
                if src.dtype != torch.float32:
                    src = src.float()
            self._cast(src, N.DT_F32, self.p16_pool[0], self._dt, lay.seg_chunks(l, "16"), st)

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
        with torch.cuda.stream(st):
            out = torch.empty(self.layout.numels[layer], dtype=self._t16, device=self.device)
        self._cast(pool, self._dt, out, self._dt, self.layout.seg_chunks(layer, "16", reverse=True), st)
        return out if raw else self._out(out, layer, readonly)

    def _pool_sum(self, buf, layer, stream) -> float:
        """f64 sum of the layer's gradient pages — ConservationLedger only
        (check-only bookkeeping, never on the update path).  The pages are
        unpacked by the page kernel and summed with torch's fixed-order
        reduction so that the same data always yields the same float (the
        ledger compares sums for equality, lockfree.py:311)."""
        g = self._unpack16(self.g16_pool[buf], layer, stream=stream, raw=True)
        with torch.cuda.stream(stream):
            return float(g.double().sum().item())

    # -- writes -----------------------------------------------------------------
    def accumulate(self, msg: GradMessage, *, stream=None) -> None:
        """g16 = rn16(f32(g16) + f32(payload)) over the layer's pages, with the
        layer's non-finite flag and squared norm fused in (lockfree.py:210-224)."""
        layer = msg.layer
        if not (0 <= layer < self.num_layers):
            raise ProtocolError(f"gradient for unknown layer {layer}")
        if _shape(msg.payload) != self._shapes[layer]:
            raise ProtocolError(f"gradient shape {_shape(msg.payload)} != buffer shape "
                                f"{self._shapes[layer]} for layer {layer}")
        st = self._stream(stream)
        with torch.cuda.stream(st):
            src = D.to_device_flat(msg.payload, self.device)
        buf = self._gsel[layer]
        add = self._pending[layer] > 0
        old = self._pool_sum(buf, layer, st) if (self._ledger_on and add) else 0.0
        if not add:  # first message into this buffer: reset its flag and norm
            with torch.cuda.stream(st):
                self._flags[buf * self.num_layers + layer] = 0
                self._sumsq[buf * self.num_layers + layer] = 0
        ch = self.layout.seg_chunks(layer, "16")
        fidx = buf * self.num_layers + layer
        D.check(N.lib().hm_accumulate(
            D.ptr(src), D.DT_OF_TORCH[src.dtype], D.ptr(self.g16_pool[buf]), self._dt,
            D.ptr(self._eng.desc.static(ch)), len(ch), 1 if add else 0, None,
            D.ptr(self._flags) + 4 * fidx, D.ptr(self._sumsq) + 8 * fidx, D.sptr(st)))
        if self._ledger_on:
            self.ledger.record_accumulate(layer, self._pool_sum(buf, layer, st) - old)
        else:
            self.ledger.messages_accumulated[layer] += 1
        self._pending[layer] += 1
        self._max_iter[layer] = max(self._max_iter[layer], msg.iteration)

    def accumulate_flat(self, flat, iteration: int, *, stream=None) -> None:
        """Accumulate one flat gradient covering every layer in order (the
        layout a backward pass writes) with ONE K3 launch: the same arithmetic
        and flags as one ``accumulate`` per layer.  Ledger sums need per-layer
        reductions, so a ledger-enabled buffer falls back to per-layer calls."""
        L, lay = self.num_layers, self.layout
        st = self._stream(stream)
        with torch.cuda.stream(st):
            src = D.to_device_flat(flat, self.device)
        if src.numel() != sum(lay.numels):
            raise ProtocolError(f"flat gradient has {src.numel()} elements, layers hold "
                                f"{sum(lay.numels)}")
        if self._ledger_on:
            pos = 0
            for l, n in enumerate(lay.numels):
                self.accumulate(GradMessage(l, src[pos:pos + n].view(self._shapes[l]), iteration),
                                stream=st)
                pos += n
            return
        key = tuple(self._gsel)
        cache = self.__dict__.setdefault("_flat_cache", {})
        if key not in cache:
            parts, base = [], 0
            for l, n in enumerate(lay.numels):
                c = lay.seg_chunks(l, "16").copy()
                c["src_off"] += base
                c["dst_off"] += key[l] * lay.elems16
                c["slot"] = key[l] * L + l
                parts.append(c)
                base += n
            cache[key] = np.concatenate(parts)
        chunks = cache[key]
        modes = np.zeros(2 * L, dtype=np.uint8)
        reset = []
        for l in range(L):
            f = self._gsel[l] * L + l
            if self._pending[l] > 0:
                modes[f] = 1
            else:
                reset.append(f)
        with torch.cuda.stream(st):
            if reset:
                if reset == list(range(reset[0], reset[0] + len(reset))):
                    self._flags[reset[0]:reset[0] + len(reset)].zero_()
                    self._sumsq[reset[0]:reset[0] + len(reset)].zero_()
                else:
                    idx = torch.tensor(reset, dtype=torch.int64, device=self.device)
                    self._flags.index_fill_(0, idx, 0)
                    self._sumsq.index_fill_(0, idx, 0)
        dmodes = self._eng.desc.table(modes)
        D.check(N.lib().hm_accumulate(
            D.ptr(src), D.DT_OF_TORCH[src.dtype], D.ptr(self.g16_pool), self._dt,
            D.ptr(self._eng.desc.static(chunks)), len(chunks), 0, D.ptr(dmodes),
            D.ptr(self._flags), D.ptr(self._sumsq), D.sptr(st)))
        for l in range(L):
            self.ledger.messages_accumulated[l] += 1
            self._pending[l] += 1
            self._max_iter[l] = max(self._max_iter[l], iteration)

    def _hand_over(self, layer: int, stream):
        """Clear-at-take bookkeeping shared by take() and sweep()."""
        buf = self._gsel[layer]
        count, newest = self._pending[layer], self._max_iter[layer]
        if self._ledger_on:
            self.ledger.record_take(layer, self._pool_sum(buf, layer, stream), count)
        else:
            self.ledger.messages_consumed[layer] += count
        self._gsel[layer] = buf ^ 1
        self._pending[layer] = 0
        return buf, count, newest

    def take(self, layer: int, *, stream=None):
        """Atomically hand over and clear the accumulated gradient: returns
        (grad fp32, message_count, newest_iteration) or None (lockfree.py:226-241)."""
        self._check_layer(layer)
        if self._pending[layer] == 0:
            return None
        st = self._stream(stream)
        buf, count, newest = self._hand_over(layer, st)
        with torch.cuda.stream(st):
            g = torch.empty(self.layout.numels[layer], dtype=torch.float32, device=self.device)
        self._cast(self.g16_pool[buf], self._dt, g, N.DT_F32,
                   self.layout.seg_chunks(layer, "16", reverse=True), st)
        fidx = buf * self.num_layers + layer
        with torch.cuda.stream(st):
            self._flags[fidx] = 0
            self._sumsq[fidx] = 0
        return self._out(g, layer), count, newest

    def publish(self, layer: int, p32, applied_iter: int | None = None, clear: bool = True,
                *, stream=None) -> int:
        """Install fresh 16-bit params (RNE cast into the inactive page buffer,
        then flip); with ``clear`` also drop pending gradients (lockfree.py:243-263)."""
        self._check_layer(layer)
        st = self._stream(stream)
        if clear:
            if self._ledger_on:
                total = self._pool_sum(self._gsel[layer], layer, st) if self._pending[layer] else 0.0
                self.ledger.record_take(layer, total, self._pending[layer])
            else:
                self.ledger.messages_consumed[layer] += self._pending[layer]
            self._pending[layer] = 0
        with torch.cuda.stream(st):
            src = D.to_device_flat(p32, self.device)
            if src.dtype != torch.float32:
                src = src.float()
        if src.numel() != self.layout.numels[layer]:
            raise ProtocolError(f"publish: {src.numel()} elements for layer {layer} of "
                                f"{self.layout.numels[layer]}")
        nxt = self._psel[layer] ^ 1
        self._cast(src, N.DT_F32, self.p16_pool[nxt], self._dt, self.layout.seg_chunks(layer, "16"), st)
        self._psel[layer] = nxt
        self._version[layer] += 1
        if applied_iter is not None:
            self._applied_iter[layer] = applied_iter
        return self._version[layer]


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


def sweep(buffer: ParamBuffer, masters: MasterState, hyper: AdamHyper, layers=None, *,
          stream=None, record_ledger: bool = True) -> SweepResult:
    """The updating actor's per-layer loop body (hiermem/lockfree.py:624-639):
    for every layer with pending gradients, take (clear) -> update_layer ->
    publish(clear=False, applied_iter=newest), fused into ONE prologue and
    ONE page-Adam launch over all their page segments: reads g16 + p/m/v
    (14 B/param), writes p/m/v + p16 (14 B/param).  Asynchronous; the
    whole-layer reject and step rollback happen on the device."""
    lay = buffer.layout
    if masters.layout.numels != lay.numels or masters.layout.page_bytes != lay.page_bytes \
            or masters.layout.world_size != lay.world_size:
        raise ConfigError("buffer and masters were built on different page tables")
    st = buffer._stream(stream)
    order = list(reversed(range(buffer.num_layers))) if layers is None else list(layers)
    sel = [l for l in order if buffer._pending[l] > 0]
    if not sel:
        return SweepResult(masters, [], [], [])
    L, span = buffer.num_layers, lay.elems16
    rows, counts, newest = [], [], []
    for l in sel:
        gbuf, count, new = buffer._hand_over(l, st)
        rows.append((gbuf * span, (buffer._psel[l] ^ 1) * span, l, gbuf * L + l))
        counts.append(count)
        newest.append(new)
    bc, bc_len = masters._bias(hyper, sel)
    adam_launch(masters._eng, lay.adam_chunks(sel, "pool"), _group_rows(rows),
                buffer.g16_pool, buffer._dt, masters.p32_pool, masters.m32_pool, masters.v32_pool,
                buffer.p16_pool, buffer._dt, hyper, bc, bc_len, 0, masters._steps, masters._applied,
                buffer._flags, buffer._sumsq, True, st)
    for l, new in zip(sel, newest):
        buffer._psel[l] ^= 1
        buffer._version[l] += 1
        buffer._applied_iter[l] = new
    if buffer._ledger_on and record_ledger:
        with torch.cuda.stream(st):
            ok = masters._applied.cpu().tolist()
        for l in sel:
            buffer.ledger.record_apply(l, buffer.ledger.consumed_sums[l][-1], rejected=not ok[l])
    return SweepResult(masters, sel, counts, newest)


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
        gkey = ("acc", tuple(grp), tuple(buffer._gsel[l] for l in grp))
        if gkey not in cache:
            rows = []
            for l in grp:
                c = lay.seg_chunks(l, "16").copy()
                c["src_off"] += int(starts[l])
                c["dst_off"] += buffer._gsel[l] * lay.elems16
                c["slot"] = buffer._gsel[l] * L + l
                rows.append(c)
            cache[gkey] = np.concatenate(rows)
        chunks = cache[gkey]
        modes = np.zeros(2 * L, dtype=np.uint8)
        reset = []
        for l in grp:
            f = buffer._gsel[l] * L + l
            if buffer._pending[l] > 0:
                modes[f] = 1
            else:
                reset.append(f)
        if reset:
            idx = buffer._eng.desc.table(np.array(reset, dtype=np.int64)).view(torch.int64)
            with torch.cuda.stream(st):
                buffer._flags.index_fill_(0, idx, 0)
                buffer._sumsq.index_fill_(0, idx, 0)
        D.check(N.lib().hm_accumulate(
            D.ptr(staging), buffer._dt, D.ptr(buffer.g16_pool), buffer._dt,
            D.ptr(buffer._eng.desc.static(chunks)), len(chunks), 0,
            D.ptr(buffer._eng.desc.table(modes)), D.ptr(buffer._flags), D.ptr(buffer._sumsq),
            D.sptr(st)))
        ev = torch.cuda.Event()
        ev.record(st)
        done.append(ev)
        for l in grp:
            buffer.ledger.messages_accumulated[l] += 1
            buffer._pending[l] += 1
            buffer._max_iter[l] = max(buffer._max_iter[l], iteration)
        if after_group is not None:
            after_group(grp)
    return done


def ingest_sweep(buffer: ParamBuffer, masters: MasterState, host_grad, hyper: AdamHyper,
                 iteration: int = 0, *, groups: int = 8, stream=None, copy_stream=None) -> SweepResult:
    """One update step fed by a flat gradient in (pinned) host memory — what a
    host-side producer hands the updating actor.  Per contiguous layer group:
    cudaMemcpyAsync of the group's slice on a copy stream -> K3 accumulate
    into its pages when it lands -> fused sweep of the group, so the PCIe
    transfer of group k+1 overlaps the update of group k and the step costs
    about one transfer of the gradient (the reference's fetch/offload are
    DelayModel sleeps, hiermem/lockfree.py:90-94, 562-569)."""
    st = buffer._stream(stream)
    parts = []
    ingest(buffer, host_grad, iteration, groups=groups, stream=st, copy_stream=copy_stream,
           after_group=lambda grp: parts.append(
               sweep(buffer, masters, hyper, layers=list(reversed(grp)), stream=st)))
    return _MultiResult(masters, parts)
