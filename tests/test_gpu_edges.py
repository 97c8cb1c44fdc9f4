"""Edge cases of the update path on the GPU, bit-exact vs the oracle:

* subnormal gradients, moments and parameters (no flush-to-zero anywhere),
  signed zeros, values at the 16-bit overflow edge (publish -> +/-inf as
  numpy's astype does, hiermem/lockfree.py:169);
* lr = 0 (exact identity on p), beta = 0 / 1-ish hyper-parameters, step
  counts past the point where f32(1 - beta**step) saturates at 1.0f;
* a single layer of more than 2**31 elements (64-bit element offsets);
* empty / mismatched inputs raise the reference's exceptions.
"""
import numpy as np
import pytest
import torch

from oracle import page_adam as O
from paper_2303_02868_b200 import lockfree as LF
from paper_2303_02868_b200.errors import ConfigError, ProtocolError

pytestmark = pytest.mark.gpu
PAGE = 64 * 1024


def _run(params, grads_per_step, dtype, hyper_kw):
    buf = LF.ParamBuffer(params, dtype=dtype, page_bytes=PAGE)
    ms = LF.MasterState(params, page_bytes=PAGE)
    om = O.OracleMasters(params)
    for it, grads in enumerate(grads_per_step):
        for l, g16 in enumerate(grads):
            payload = g16 if dtype == "fp16" else torch.from_numpy(g16.view(np.int16)).view(torch.bfloat16)
            buf.accumulate(LF.GradMessage(l, payload, it))
        applied = LF.sweep(buf, ms, LF.AdamHyper(**hyper_kw)).applied()
        for l, g16 in enumerate(grads):
            assert applied[l] == om.update_layer(l, O.from16(g16, dtype), **hyper_kw)
    assert ms.steps == om.steps
    for l in range(len(params)):
        np.testing.assert_array_equal(np.asarray(ms.p32[l]).view(np.uint32), om.p32[l].view(np.uint32))
        np.testing.assert_array_equal(np.asarray(ms.m32[l]).view(np.uint32), om.m32[l].view(np.uint32))
        np.testing.assert_array_equal(np.asarray(ms.v32[l]).view(np.uint32), om.v32[l].view(np.uint32))
        pub = np.asarray(buf.read(l)[1]).view(np.uint16)
        np.testing.assert_array_equal(pub, O.to16(om.p32[l], dtype).view(np.uint16))


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_subnormals_zeros_and_overflow(cuda, dtype):
    rng = np.random.default_rng(1)
    n = 9000
    tiny = np.float32(1e-41)                                   # f32 subnormal
    p = np.concatenate([rng.normal(0, 0.02, n - 8).astype(np.float32),
                        np.array([tiny, -tiny, 0.0, -0.0, 65504.0, -65520.0, 3.0e38, 1e-45], np.float32)])
    grads = []
    for it in range(3):
        g = (rng.normal(0, 1, n) * np.float32(1e-38)).astype(np.float32)     # bf16/f32 subnormal range
        g[:10] = [0.0, -0.0, 1e-40, -1e-40, 6e-8, -6e-8, 1e-30, 5.9e-8, 1e4, -1e4]
        grads.append([O.to16(g, dtype)])
    _run([p], grads, dtype, dict(lr=1e-3))


def test_lr_zero_and_extreme_betas(cuda):
    rng = np.random.default_rng(2)
    params = [rng.normal(0, 0.02, n).astype(np.float32) for n in (4097, 33)]
    grads = [[O.to16(rng.normal(0, 1e-2, p.size).astype(np.float32), "bf16") for p in params]
             for _ in range(3)]
    _run(params, grads, "bf16", dict(lr=0.0))
    _run(params, grads, "bf16", dict(lr=0.1, beta1=0.0, beta2=0.0, eps=0.0))
    _run(params, grads, "bf16", dict(lr=1e-3, beta1=0.5, beta2=0.75, eps=1e-3))


def test_steps_past_bias_saturation(cuda):
    """beta2=0.5: f32(1-0.5**s) reaches 1.0f at s=25; run 40 steps."""
    rng = np.random.default_rng(3)
    params = [rng.normal(0, 0.02, 1000).astype(np.float32)]
    grads = [[O.to16(rng.normal(0, 1e-2, 1000).astype(np.float32), "bf16")] for _ in range(40)]
    _run(params, grads, "bf16", dict(lr=1e-3, beta1=0.25, beta2=0.5))


def test_layer_larger_than_2_pow_31(cuda):
    """64-bit element offsets: one layer of 2**31 + 4099 elements (4 MiB pages)."""
    n = 2 ** 31 + 4099
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    p = torch.empty(n, device=dev).normal_(0, 0.02, generator=gen)
    buf = LF.ParamBuffer([p], dtype="bf16", device=dev)
    ms = LF.MasterState([p], device=dev)
    g = torch.empty(n, device=dev).normal_(0, 1e-2, generator=gen).to(torch.bfloat16)
    buf.accumulate(LF.GradMessage(0, g, 0))
    assert LF.sweep(buf, ms, LF.AdamHyper(lr=1e-3)).applied() == {0: True}
    lay = ms.layout

    def state_range(pos, cnt):   # tensor elements [pos, pos+cnt) gathered along the segments
        out = []
        for s in lay.segments[0]:
            lo, hi = max(pos, s.pos), min(pos + cnt, s.pos + s.n)
            if lo < hi:
                o = lay.slot_state(s.page) * lay.E + s.off + (lo - s.pos)
                out.append(ms.p32_pool[o:o + (hi - lo)].cpu().numpy())
        return np.concatenate(out)

    for pos in (0, 2 ** 31 - 2048, 2 ** 31 + 3, n - 4099):   # across the 2**31 boundary and the tail
        cnt = min(4099, n - pos)
        pe = p[pos:pos + cnt].cpu().numpy()
        ge = O.from16(g[pos:pos + cnt].view(torch.int16).cpu().numpy().view(np.uint16), "bf16")
        want, _, _, _ = O.adam_update(pe, np.zeros_like(pe), np.zeros_like(pe), ge, lr=1e-3, step=1)
        np.testing.assert_array_equal(state_range(pos, cnt).view(np.uint32), want.view(np.uint32))
    del buf, ms, p, g
    torch.cuda.empty_cache()


def test_api_errors(cuda):
    with pytest.raises(ConfigError):
        LF.ParamBuffer([])
    with pytest.raises(ConfigError):
        LF.ParamBuffer([np.zeros(4, np.float32)], dtype="fp8")
    buf = LF.ParamBuffer([np.zeros(4, np.float32)], page_bytes=PAGE)
    ms = LF.MasterState([np.zeros(4, np.float32)], page_bytes=PAGE)
    with pytest.raises(ProtocolError):
        buf.accumulate_flat(torch.zeros(5, dtype=torch.float16, device="cuda"), 0)
    with pytest.raises(ProtocolError):
        ms.update_layer(0, np.zeros(3, np.float32), LF.AdamHyper())
    with pytest.raises(ProtocolError):
        buf.read(3)
    assert LF.sweep(buf, ms, LF.AdamHyper()).layers == ()      # nothing pending: no launch
    other = LF.MasterState([np.zeros(5, np.float32)], page_bytes=PAGE)
    buf.accumulate(LF.GradMessage(0, np.ones(4, np.float16), 0))
    with pytest.raises(ConfigError):
        LF.sweep(buf, other, LF.AdamHyper())
