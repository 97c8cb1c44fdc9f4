"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

numpy restatement of the reference update chain, one numpy ufunc per
operator in the reference's order, so every intermediate is a correctly
rounded binary32 value exactly as in the reference:

  apply_update        hiermem/lockfree.py:127-142
  update_layer        hiermem/lockfree.py:155-165
  accumulate          hiermem/lockfree.py:210-224
  take                hiermem/lockfree.py:226-241
  publish (_published) hiermem/lockfree.py:168-171, 243-263

The reference's 16-bit type is IEEE fp16 (np.float16); the north star's is
bfloat16, produced here by an explicit round-to-nearest-even on the f32
bit pattern (checked against ml_dtypes in tests/test_oracle.py).
"""
from __future__ import annotations

import numpy as np

F32 = np.float32


# ---- 16-bit formats --------------------------------------------------------

def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even binary32 -> bfloat16, returned as uint16 bits."""
    u = np.ascontiguousarray(x, dtype=F32).view(np.uint32)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    rounded = ((u.astype(np.uint64) + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    quiet = ((u >> 16) | 0x0040).astype(np.uint16)
    return np.where(nan, quiet, rounded)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(F32)


def to16(x: np.ndarray, dtype: str) -> np.ndarray:
    """f32 -> 16-bit storage (np.float16 array, or uint16 bf16 bits)."""
    if dtype == "fp16":
        return np.asarray(x, dtype=F32).astype(np.float16)
    if dtype == "bf16":
        return f32_to_bf16_bits(np.asarray(x, dtype=F32))
    raise ValueError(dtype)


def from16(x: np.ndarray, dtype: str) -> np.ndarray:
    """16-bit storage -> f32 (exact widening)."""
    if dtype == "fp16":
        return np.asarray(x, dtype=np.float16).astype(F32)
    if dtype == "bf16":
        return bf16_bits_to_f32(x)
    raise ValueError(dtype)


# ---- Adam (hiermem/lockfree.py:127-142) --------------------------------------

def bias_corrections(beta1: float, beta2: float, step: int) -> tuple[np.float32, np.float32]:
    """f32(1 - beta**step) from Python-double arithmetic (lockfree.py:137-140)."""
    return F32(1.0 - beta1 ** step), F32(1.0 - beta2 ** step)


def adam_update(p32, m32, v32, grad, lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8, step=1):
    """Returns (p, m, v, applied); inputs untouched.  Restates lockfree.py:127-142."""
    g = np.asarray(grad).astype(F32, copy=False)
    if not np.isfinite(g).all():                               # :133-134
        return p32, m32, v32, False
    b1, ob1 = F32(beta1), F32(1.0 - beta1)
    b2, ob2 = F32(beta2), F32(1.0 - beta2)
    m = np.add(np.multiply(b1, m32), np.multiply(ob1, g))       # :135
    v = np.add(np.multiply(b2, v32), np.multiply(ob2, np.multiply(g, g)))  # :136
    bc1, bc2 = bias_corrections(beta1, beta2, step)             # :137-138
    mh = np.divide(m, bc1)                                      # :139
    vh = np.divide(v, bc2)                                      # :140
    den = np.add(np.sqrt(vh), F32(eps))                         # :141
    p = np.subtract(p32, np.divide(np.multiply(F32(lr), mh), den))
    return p.astype(F32), m.astype(F32), v.astype(F32), True


class OracleMasters:
    """MasterState restated (lockfree.py:145-165)."""

    def __init__(self, params):
        self.p32 = [np.asarray(p).astype(F32) for p in params]
        self.m32 = [np.zeros_like(p, dtype=F32) for p in self.p32]
        self.v32 = [np.zeros_like(p, dtype=F32) for p in self.p32]
        self.steps = [0] * len(self.p32)

    def update_layer(self, layer, grad, lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8) -> bool:
        self.steps[layer] += 1
        p, m, v, ok = adam_update(self.p32[layer], self.m32[layer], self.v32[layer], grad,
                                  lr, beta1, beta2, eps, self.steps[layer])
        if ok:
            self.p32[layer], self.m32[layer], self.v32[layer] = p, m, v
        else:
            self.steps[layer] -= 1
        return ok


# ---- gradient buffer ops (lockfree.py:210-263) -------------------------------

def accumulate16(g16: np.ndarray, payload: np.ndarray, dtype: str) -> np.ndarray:
    """rn16(f32(g16) + f32(payload)) — lockfree.py:219-220."""
    return to16(np.add(from16(g16, dtype), from16(payload, dtype)), dtype)


def publish16(p32: np.ndarray, dtype: str) -> np.ndarray:
    """p16 = rn16(p32) — lockfree.py:169."""
    return to16(p32, dtype)


# ---- page pack / unpack over segments --------------------------------------

def pack(pool: np.ndarray, tensor: np.ndarray, segments, page_elems: int, itemsize: int,
         slot_of=lambda pid: pid) -> None:
    """Scatter a flat tensor into pool pages along (page_id, byte_off, bytes)."""
    pos = 0
    for pid, off, nbytes in segments:
        n = nbytes // itemsize
        base = slot_of(pid) * page_elems + off // itemsize
        pool[base:base + n] = tensor[pos:pos + n]
        pos += n


def unpack(pool: np.ndarray, segments, page_elems: int, itemsize: int,
           slot_of=lambda pid: pid) -> np.ndarray:
    parts = []
    for pid, off, nbytes in segments:
        n = nbytes // itemsize
        base = slot_of(pid) * page_elems + off // itemsize
        parts.append(pool[base:base + n])
    return np.concatenate(parts) if parts else pool[:0].copy()


# ---- seeded synthetic inputs ---------------------------------

def synthetic_layer(seed: int, tensor_id: int, n: int, dtype: str = "bf16", outliers: bool = True):
    """p ~ N(0, .02), m ~ N(0, 1e-3), v = N(0, 1e-3)^2, g ~ N(0, 1e-2) with
    1% x10 outliers, rounded to the 16-bit type; rng idiom of lockfree.py:332."""
    rng = np.random.default_rng([seed, tensor_id, 7])
    p = rng.normal(0, 0.02, n).astype(F32)
    m = rng.normal(0, 1e-3, n).astype(F32)
    v = np.square(rng.normal(0, 1e-3, n)).astype(F32)
    g = rng.normal(0, 1e-2, n).astype(F32)
    if outliers:
        k = max(1, n // 100)
        idx = rng.choice(n, size=k, replace=False)
        g[idx] *= F32(10.0)
    return p, m, v, to16(g, dtype)
