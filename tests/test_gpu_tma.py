"""The TMA bulk-copy variant of the page-Adam main pass (page_adam_tma.cu,
hm_set_adam_variant(1)) — and the 512-thread form of the LDG kernel — produce
the same bits as the oracle on every path:
aligned chunks through the shared-memory pipeline, unaligned heads/tails from
global memory, rejected layers (publish only), f32 gradients (apply_update)."""
import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import page_adam as O
from paper_2303_02868_b200 import _native as N
from paper_2303_02868_b200 import lockfree as LF

pytestmark = pytest.mark.gpu
SIZES = [70001, 1, 5, 32768, 40000, 25003, 777, 65539, 12, 33333, 200000, 4096 * 40 + 8]


@pytest.fixture()
def tma_variant():
    N.check(N.lib().hm_set_adam_variant(1))
    yield
    N.check(N.lib().hm_set_adam_variant(0))


@pytest.fixture()
def threads512():
    N.check(N.lib().hm_set_adam_threads(512))
    yield
    N.check(N.lib().hm_set_adam_threads(256))


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_tma_sweep_bit_exact(cuda, tma_variant, dtype):
    _sweep_bit_exact(dtype)


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_512_thread_variant_bit_exact(cuda, threads512, dtype):
    """hm_set_adam_threads(512): one granule per thread instead of two."""
    _sweep_bit_exact(dtype)


def _sweep_bit_exact(dtype):
    rng = np.random.default_rng(17)
    params = [rng.normal(0, 0.02, n).astype(np.float32) for n in SIZES]
    buf = LF.ParamBuffer(params, dtype=dtype, page_bytes=64 * 1024)
    ms = LF.MasterState(params, page_bytes=64 * 1024)
    om = O.OracleMasters(params)
    for it in range(4):
        grads = []
        for l, n in enumerate(SIZES):
            g = rng.normal(0, 1e-2, n).astype(np.float32)
            if it == 2 and l == 10:
                g[5] = np.nan
            g16 = O.to16(g, dtype)
            grads.append(g16)
            payload = g16 if dtype == "fp16" else torch.from_numpy(g16.view(np.int16)).view(torch.bfloat16)
            buf.accumulate(LF.GradMessage(l, payload, it))
        applied = LF.sweep(buf, ms, LF.AdamHyper(lr=1e-3)).applied()
        for l in range(len(SIZES)):
            assert applied[l] == om.update_layer(l, O.from16(grads[l], dtype), lr=1e-3)
    assert ms.steps == om.steps
    for l in range(len(SIZES)):
        np.testing.assert_array_equal(np.asarray(ms.p32[l]).view(np.uint32), om.p32[l].view(np.uint32))
        np.testing.assert_array_equal(np.asarray(ms.v32[l]).view(np.uint32), om.v32[l].view(np.uint32))
        np.testing.assert_array_equal(np.asarray(buf.read(l)[1]).view(np.uint16),
                                      O.to16(om.p32[l], dtype).view(np.uint16))


def test_tma_apply_update_f32_grad(cuda, tma_variant):
    gold = np.load(GOLDEN / "adam_golden.npz")
    for c in range(int(gold["n_cases"][0])):
        k = f"c{c}"
        n, step, lr, b1, b2, eps, is_bf16 = gold[f"{k}.meta"]
        g16 = gold[f"{k}.g16"]
        g32 = O.from16(g16 if is_bf16 else g16.view(np.float16), "bf16" if is_bf16 else "fp16")
        p, m, v, ok = LF.apply_update(gold[f"{k}.p"], gold[f"{k}.m"], gold[f"{k}.v"], g32,
                                      LF.AdamHyper(lr=lr, beta1=b1, beta2=b2, eps=eps), int(step))
        assert ok
        np.testing.assert_array_equal(p.view(np.uint32), gold[f"{k}.rp"].view(np.uint32))
        np.testing.assert_array_equal(v.view(np.uint32), gold[f"{k}.rv"].view(np.uint32))
