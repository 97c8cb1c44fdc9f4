"""Device plumbing: torch owns device memory and streams; this module turns
tensors into raw pointers for the C-ABI, caches descriptor uploads, and
holds the exact bias-correction tables.  No compute happens here."""
from __future__ import annotations

import contextlib
import ctypes as C
import weakref
from collections import OrderedDict

import numpy as np
import torch

from . import _native as N
from .errors import NativeError

TORCH16 = {"fp16": torch.float16, "bf16": torch.bfloat16}
DT_OF_TORCH = {torch.float16: N.DT_F16, torch.bfloat16: N.DT_BF16, torch.float32: N.DT_F32}
F32 = np.float32


def require_device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise NativeError("a CUDA device is required: the page-update path has no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise NativeError(f"device {d} is not a CUDA device (no CPU fallback)")
    return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def addr(x) -> int:
    """Device address of a tensor, or a raw address passed through."""
    return x if isinstance(x, int) else ptr(x)


_STREAMS: dict = {}
# torch's own binding behind torch.cuda.current_stream (private: fall back to
# the public call if a torch build does not have it)
_GET_CURRENT = getattr(torch._C, "_cuda_getCurrentStream", None)


def cur_stream(device, stream=None):
    """``stream`` or the device's current stream.  Same object as
    torch.cuda.current_stream(device), without its per-call device-index
    resolution (the three-call path asks ~7 times per layer)."""
    if stream is not None:
        return stream
    if _GET_CURRENT is None:
        return torch.cuda.current_stream(device)
    sid, didx, dtype = _GET_CURRENT(device.index)
    s = _STREAMS.get((sid, didx))
    if s is None:
        s = _STREAMS[(sid, didx)] = torch.cuda.Stream(stream_id=sid, device_index=didx, device_type=dtype)
    return s


def on(stream):
    """``torch.cuda.stream(stream)``, or a no-op when it already is the
    current stream (allocations then land on it either way)."""
    if _GET_CURRENT is not None and _GET_CURRENT(stream.device_index)[0] == stream.stream_id:
        return contextlib.nullcontext()
    return torch.cuda.stream(stream)


def sptr(stream) -> C.c_void_p:
    return C.c_void_p(int(stream.cuda_stream))


class DescCache:
    """Device copies of host descriptor arrays.  Static plans are keyed by the
    identity of the (cached, immortal) numpy array; per-launch tables by their
    bytes in an LRU sized for every layer's rows of both page buffers (the
    three-call path looks up a few hundred small tables per step), so steady
    state uploads nothing.

    Uploads are allocated on the caller's current stream.  A table used by a
    launch on another stream names that stream (``table(arr, stream)``):
    when the LRU evicts the table, it is ``record_stream``-ed on every stream
    that used it, so the caching allocator cannot hand the block to a new
    upload while a queued kernel may still read it."""

    def __init__(self, device, lru: int = 8192):
        self.device = device
        self._static: dict[int, tuple[np.ndarray, torch.Tensor]] = {}
        self._lru: OrderedDict[bytes, tuple[torch.Tensor, set]] = OrderedDict()
        self._lru_cap = lru

    def static(self, arr: np.ndarray) -> torch.Tensor:
        key = id(arr)
        hit = self._static.get(key)
        if hit is not None and hit[0]() is arr:
            return hit[1]
        dev = self._upload(arr)
        # the device copy lives exactly as long as the host plan it mirrors
        self._static[key] = (weakref.ref(arr), dev)
        weakref.finalize(arr, self._static.pop, key, None)
        return dev

    def table(self, arr: np.ndarray, stream=None) -> torch.Tensor:
        key = arr.tobytes()
        hit = self._lru.get(key)
        if hit is not None:
            self._lru.move_to_end(key)
            dev, users = hit
        else:
            dev, users = self._upload(arr), set()
            self._lru[key] = (dev, users)
            if len(self._lru) > self._lru_cap:
                old, old_users = self._lru.popitem(last=False)[1]
                for st in old_users:
                    old.record_stream(st)
        if stream is not None:
            users.add(stream)
        return dev

    def _upload(self, arr: np.ndarray) -> torch.Tensor:
        raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
        if raw.size == 0:
            return torch.empty(8, dtype=torch.uint8, device=self.device)
        return torch.from_numpy(raw.copy()).to(self.device)


class BiasTable:
    """f32(1 - beta**step) for step = 0..len-1, computed in Python double
    exactly as hiermem/lockfree.py:137-140 does (never a device pow).  The
    sequence is monotone and reaches 1.0f; the table grows lazily to the
    largest reachable step and stops growing once both columns saturate
    (the prologue clamps to the last row)."""

    def __init__(self, beta1: float, beta2: float, device):
        self.beta1, self.beta2 = float(beta1), float(beta2)
        self.device = device
        self.rows: list[tuple[float, float]] = [(0.0, 0.0)]
        self.saturated = False
        self.dev = None

    def ensure(self, max_step: int) -> tuple[torch.Tensor, int]:
        target = max_step + 1
        if (len(self.rows) < target and not self.saturated) or self.dev is None:
            grow = max(target, 2 * len(self.rows), 64)
            s = len(self.rows)
            while s < grow:
                a, b = F32(1.0 - self.beta1 ** s), F32(1.0 - self.beta2 ** s)
                self.rows.append((a, b))
                s += 1
                if a == F32(1.0) and b == F32(1.0) and s > 1:
                    self.saturated = True
                    break
            self.dev = torch.tensor(np.array(self.rows, dtype=F32).reshape(-1), device=self.device)
        return self.dev, len(self.rows)


def opts(**kw):
    """ctypes pointer to an hm_launch_opts with the given fields (others -1 =
    the process default); None when nothing is set."""
    if not kw:
        return None
    return C.byref(N.LaunchOpts(**kw))


_HYPER_C: dict = {}


def hyper_c(h) -> N.AdamHyperC:
    """AdamHyper -> f32 scalars with numpy's weak-scalar rounding
    (lockfree.py:135-141: python float -> f32 per operation).  Cached per
    (frozen, hashable) hyper: the struct is only ever read by the library."""
    try:
        hit = _HYPER_C.get(h)
    except TypeError:   # an unhashable stand-in
        return _hyper_c(h)
    if hit is None:
        hit = _HYPER_C[h] = _hyper_c(h)
    return hit


def _hyper_c(h) -> N.AdamHyperC:
    return N.AdamHyperC(
        float(F32(h.lr)), float(F32(h.beta1)), float(F32(1.0 - h.beta1)),
        float(F32(h.beta2)), float(F32(1.0 - h.beta2)), float(F32(h.eps)),
        float(F32(getattr(h, "inv_scale", 1.0))), float(F32(getattr(h, "max_norm", 0.0))))


def contiguous_chunks(n: int, slot: int = 0) -> np.ndarray:
    """hm_seg_chunk units covering [0, n) of a contiguous buffer (src == dst)."""
    full = n // 4096
    rest = n - full * 4096
    body = rest - rest % 8
    offs = [np.arange(full, dtype=np.int64) * 4096]
    ns = [np.full(full, 4096, dtype=np.int64)]
    if body:
        offs.append(np.array([full * 4096]))
        ns.append(np.array([body]))
    if rest - body:
        offs.append(np.array([full * 4096 + body]))
        ns.append(np.array([rest - body]))
    o = np.concatenate(offs)
    a = np.empty(len(o), dtype=N.SEG_CHUNK)
    a["src_off"] = o
    a["dst_off"] = o
    a["n"] = np.concatenate(ns)
    a["slot"] = slot
    return a


_CONTIG: dict[tuple[int, int], np.ndarray] = {}


def contiguous_chunks_cached(n: int, slot: int = 0) -> np.ndarray:
    key = (n, slot)
    if key not in _CONTIG:
        _CONTIG[key] = contiguous_chunks(n, slot)
    return _CONTIG[key]


def contiguous_adam_chunks(n: int) -> np.ndarray:
    seg = contiguous_chunks_cached(n)
    a = np.empty(len(seg), dtype=N.ADAM_CHUNK)
    a["g_off"] = seg["src_off"]
    a["s_off"] = seg["src_off"]
    a["p_off"] = seg["src_off"]
    a["n"] = seg["n"]
    a["slot"] = 0
    return a


# ---- host <-> device conversion ------------------------------------------------

def _np_bf16():
    try:
        import ml_dtypes
        return ml_dtypes.bfloat16
    except Exception:  # pragma: no cover
        return None


def to_device_flat(x, device, float_dtype=None) -> torch.Tensor:
    """Any array-like -> contiguous 1-D CUDA tensor (f16/bf16/f32 kept; f64 and
    ints rounded to f32 on the host, as numpy's astype(float32) would)."""
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if t.dtype not in DT_OF_TORCH:
            t = t.to(torch.float32)
        t = t.reshape(-1)
        if t.device.type == "cpu":
            return t.to(device, non_blocking=t.is_pinned()).contiguous()
        return t.to(device).contiguous()
    a = np.asarray(x)
    bf = _np_bf16()
    if bf is not None and a.dtype == bf:
        t = torch.from_numpy(np.ascontiguousarray(a).view(np.int16).reshape(-1).copy())
        return t.view(torch.bfloat16).to(device)
    if a.dtype not in (np.float16, np.float32):
        a = a.astype(np.float32)
    return torch.from_numpy(np.ascontiguousarray(a).reshape(-1).copy()).to(device)


def to_host(t: torch.Tensor, shape, readonly: bool = False) -> np.ndarray:
    if t.dtype == torch.bfloat16:
        bits = t.view(torch.int16).cpu().numpy().view(np.uint16)
        bf = _np_bf16()
        a = bits.view(bf) if bf is not None else bits
    else:
        a = t.cpu().numpy()
    a = a.reshape(shape)
    if readonly:
        a.flags.writeable = False
    return a


def check(rc: int) -> None:
    N.check(rc)


def pinned_zeros(n: int, dtype=torch.float32) -> torch.Tensor:
    """Page-locked host tensor of EXACTLY n zeros.  torch's pinned allocator
    rounds every block up to a power of two (the 13B model's 51.4 GB p32 pool
    would take 64 GB, and the three state pools 192 GB of a 196 GB box), so
    large pools come from the library's hm_host_alloc (cudaHostAlloc of the
    exact size), wrapped zero-copy and freed with the tensor."""
    esz = torch.empty(0, dtype=dtype).element_size()
    nbytes = n * esz
    if nbytes < (1 << 30):
        return torch.zeros(n, dtype=dtype).pin_memory()
    out = C.c_void_p()
    check(N.lib().hm_host_alloc(nbytes, C.byref(out)))
    raw = (C.c_char * nbytes).from_address(out.value)
    # freed when the last tensor or view over the block goes away (the
    # storage keeps the buffer object alive)
    weakref.finalize(raw, N.lib().hm_host_free, C.c_void_p(out.value))
    return torch.frombuffer(raw, dtype=dtype, count=n)


def _parse_cpulist(text: str) -> set[int]:
    cpus = set()
    for part in text.strip().split(","):
        if not part:
            continue
        lo, _, hi = part.partition("-")
        cpus.update(range(int(lo), int(hi or lo) + 1))
    return cpus


def bind_to_gpu_numa(device_index: int) -> dict | None:
    """Pin the calling process to the CPUs of the NUMA node that hosts the
    GPU's PCIe root, so pinned host buffers allocated afterwards (first touch)
    live next to that GPU's link — with one rank per GPU, every rank's
    host->device stream then stays on its own socket.  No-op (None) when the
    topology is not visible, the node is unknown, or HM_NO_NUMA_BIND=1."""
    import os
    if os.environ.get("HM_NO_NUMA_BIND") == "1" or not hasattr(os, "sched_setaffinity"):
        return None
    try:
        p = torch.cuda.get_device_properties(device_index)
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            node = int(f.read().strip())
        if node < 0:
            return None
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            cpus = _parse_cpulist(f.read()) & os.sched_getaffinity(0)
        if not cpus:
            return None
        before = os.sched_getaffinity(0)
        os.sched_setaffinity(0, cpus)
        return {"numa_node": node, "cpus": len(cpus), "pci": bus, "_before": sorted(before)}
    except (OSError, ValueError, AttributeError, RuntimeError):
        return None


def restore_affinity(info: dict | None) -> None:
    """Undo bind_to_gpu_numa (e.g. before a CPU-side measurement that should
    use every host core)."""
    import os
    if info and info.get("_before"):
        os.sched_setaffinity(0, set(info["_before"]))
