"""GPU parity of the drop-in update path against the reference.

Every test calls the CUDA kernels through the C-ABI (libhm_page.so) and
compares bit-for-bit with (a) golden outputs of the reference itself
(tests/golden/adam_golden.npz) or (b) the oracle restatement (oracle/page_adam.py,
itself pinned to the reference by tests/test_oracle.py).  Tolerance: none —
p32/m32/v32 and the 16-bit published params are compared as bit patterns
(stronger than the north star's 1e-6 relative / 1 ULP).
"""
import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import page_adam as O
from paper_2303_02868_b200 import lockfree as LF
from paper_2303_02868_b200.errors import ProtocolError

pytestmark = pytest.mark.gpu


def bits(x):
    x = np.asarray(x)
    return x.view(np.uint32) if x.dtype == np.float32 else x.view(np.uint16)


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN / "adam_golden.npz")


# ---- apply_update: reference known answers (tests/test_lockfree.py:36-62) ----------

def test_zero_gradient_is_identity(cuda):
    p = np.ones(4, np.float32)
    p2, m2, v2, ok = LF.apply_update(p, np.zeros(4, np.float32), np.zeros(4, np.float32),
                                     np.zeros(4, np.float32), LF.AdamHyper(), step=1)
    assert ok
    np.testing.assert_array_equal(p2, p)
    np.testing.assert_array_equal(m2, 0)
    np.testing.assert_array_equal(v2, 0)


def test_degenerate_scalar_case(cuda):
    hyper = LF.AdamHyper(lr=0.1, beta1=0.0, beta2=0.0, eps=0.0)
    p, m, v, ok = LF.apply_update(np.array([1.0], np.float32), np.zeros(1, np.float32),
                                  np.zeros(1, np.float32), np.array([1.0], np.float32), hyper, step=1)
    assert ok and p[0] == pytest.approx(0.9)


def test_nonfinite_gradient_rejected(cuda):
    p = np.ones(2, np.float32)
    for bad in (np.nan, np.inf, -np.inf):
        g = np.array([1.0, bad], np.float32)
        p2, _, _, ok = LF.apply_update(p, np.zeros(2, np.float32), np.zeros(2, np.float32), g,
                                       LF.AdamHyper(), 1)
        assert not ok and p2 is p


def test_apply_update_golden_bit_exact(cuda, gold):
    for c in range(int(gold["n_cases"][0])):
        k = f"c{c}"
        n, step, lr, b1, b2, eps, is_bf16 = gold[f"{k}.meta"]
        hyper = LF.AdamHyper(lr=lr, beta1=b1, beta2=b2, eps=eps)
        g16 = gold[f"{k}.g16"]
        g = (torch.from_numpy(g16.view(np.int16).copy()).view(torch.bfloat16) if is_bf16
             else torch.from_numpy(g16.view(np.float16).copy()))
        p, m, v, ok = LF.apply_update(torch.from_numpy(gold[f"{k}.p"]).cuda(),
                                      torch.from_numpy(gold[f"{k}.m"]).cuda(),
                                      torch.from_numpy(gold[f"{k}.v"]).cuda(), g.cuda(), hyper, int(step))
        assert ok
        np.testing.assert_array_equal(bits(p.cpu().numpy()), bits(gold[f"{k}.rp"]), err_msg=k)
        np.testing.assert_array_equal(bits(m.cpu().numpy()), bits(gold[f"{k}.rm"]), err_msg=k)
        np.testing.assert_array_equal(bits(v.cpu().numpy()), bits(gold[f"{k}.rv"]), err_msg=k)


# ---- MasterState with rollback (lockfree.py:145-165) -------------------------------

def test_master_state_golden_sequence(cuda, gold):
    params = [gold[f"ms.init{l}"] for l in range(3)]
    ms = LF.MasterState(params, page_bytes=64 * 1024)
    grads = gold["ms.grads"].view(np.float16)
    pos = 0
    results = []
    for it in range(4):
        for layer in reversed(range(3)):
            n = params[layer].size
            results.append(ms.update_layer(layer, grads[pos:pos + n].astype(np.float32), LF.AdamHyper()))
            pos += n
    assert results.count(False) == 1
    assert ms.steps == list(gold["ms.steps"])
    for l in range(3):
        np.testing.assert_array_equal(bits(ms.p32[l]), bits(gold[f"ms.p{l}"]))
        np.testing.assert_array_equal(bits(ms.m32[l]), bits(gold[f"ms.m{l}"]))
        np.testing.assert_array_equal(bits(ms.v32[l]), bits(gold[f"ms.v{l}"]))


# ---- ParamBuffer (lockfree.py:174-263; reference tests :65-106) -------------------

class TestBuffers:
    def make(self, layers=2, dim=4):
        return LF.ParamBuffer([np.zeros((dim, dim), np.float32) for _ in range(layers)],
                              page_bytes=64 * 1024)

    def test_accumulate_two_unit_gradients(self, cuda):
        buf = self.make()
        g = np.ones((4, 4), np.float16)
        LF.accumulate_gradient(buf, LF.GradMessage(0, g, 0))
        LF.accumulate_gradient(buf, LF.GradMessage(0, g, 1))
        np.testing.assert_array_equal(buf.g16[0], np.full((4, 4), 2.0, np.float16))

    def test_publish_clears_gradients(self, cuda):
        buf = self.make()
        LF.accumulate_gradient(buf, LF.GradMessage(0, np.ones((4, 4), np.float16), 0))
        LF.publish_params(buf, 0, np.full((4, 4), 7.0, np.float32))
        np.testing.assert_array_equal(buf.g16[0], 0)
        assert buf.read(0)[1][0, 0] == np.float16(7.0)

    def test_publish_twice_bumps_version_only(self, cuda):
        buf = self.make()
        p = np.full((4, 4), 3.0, np.float32)
        v0 = buf.version(0)
        LF.publish_params(buf, 0, p)
        LF.publish_params(buf, 0, p)
        assert buf.version(0) == v0 + 2
        np.testing.assert_array_equal(buf.read(0)[1], p.astype(np.float16))

    def test_shape_mismatch_rejected(self, cuda):
        buf = self.make()
        with pytest.raises(ProtocolError):
            LF.accumulate_gradient(buf, LF.GradMessage(0, np.ones((2, 2), np.float16), 0))
        with pytest.raises(ProtocolError):
            LF.accumulate_gradient(buf, LF.GradMessage(9, np.ones((4, 4), np.float16), 0))

    def test_take_clears_and_counts(self, cuda):
        buf = self.make()
        LF.accumulate_gradient(buf, LF.GradMessage(1, np.ones((4, 4), np.float16), 3))
        grad, count, newest = buf.take(1)
        assert count == 1 and newest == 3
        assert buf.take(1) is None
        np.testing.assert_array_equal(buf.g16[1], 0)
        np.testing.assert_array_equal(grad, np.ones((4, 4), np.float32))

    def test_golden_accumulate_take_publish(self, cuda, gold):
        buf = LF.ParamBuffer([np.zeros(513, np.float32), np.zeros(64, np.float32)], page_bytes=64 * 1024)
        for it, msg in enumerate(gold["pb.msgs"]):
            buf.accumulate(LF.GradMessage(0, msg.view(np.float16), it))
        np.testing.assert_array_equal(bits(buf.g16[0]), gold["pb.g16"])
        g32, count, newest = buf.take(0)
        np.testing.assert_array_equal(bits(g32), bits(gold["pb.take"]))
        assert [count, newest] == list(gold["pb.take_meta"])
        ver = buf.publish(0, gold["pb.pub_in"], applied_iter=4, clear=False)
        np.testing.assert_array_equal(bits(buf.read(0)[1]), gold["pb.pub_out"])
        assert [ver, buf.read(0)[2]] == list(gold["pb.pub_meta"])

    def test_accumulate_after_take_starts_from_zero(self, cuda):
        buf = self.make(layers=1, dim=8)
        one = np.ones((8, 8), np.float16)
        buf.accumulate(LF.GradMessage(0, one * 3, 0))
        buf.take(0)
        buf.accumulate(LF.GradMessage(0, one, 1))
        buf.accumulate(LF.GradMessage(0, one, 2))
        np.testing.assert_array_equal(buf.g16[0], np.full((8, 8), 2.0, np.float16))
        buf.take(0)
        buf.accumulate(LF.GradMessage(0, -0.0 * one, 3))  # -0 + 0 -> +0 as in the reference
        assert (bits(buf.g16[0]) == 0).all()


# ---- the fused sweep over shared pages ---------------------------------------------

def _layer_sizes():
    # page = 64 KiB = 32768 elements: multi-page tensors with tails that share
    # pages (end-aligned, odd offsets), small own-page tensors, ragged sizes.
    return [70001, 1, 5, 32768, 40000, 25003, 777, 65536 + 3, 12, 33333]


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_sweep_matches_oracle_bit_exact(cuda, dtype):
    sizes = _layer_sizes()
    rng = np.random.default_rng(5)
    params = [rng.normal(0, 0.02, n).astype(np.float32) for n in sizes]
    buf = LF.ParamBuffer(params, dtype=dtype, page_bytes=64 * 1024)   # the ledger is on by default
    ms = LF.MasterState(params, page_bytes=64 * 1024)
    om = O.OracleMasters(params)
    hyper = LF.AdamHyper(lr=1e-3)
    for it in range(5):
        grads = []
        for l, n in enumerate(sizes):
            g = rng.normal(0, 1e-2, n).astype(np.float32) * np.float32(10.0 ** rng.integers(-2, 2))
            if it == 3 and l == 4:
                g[n // 2] = np.nan  # whole-layer reject + step rollback
            g16 = O.to16(g, dtype)
            grads.append(g16)
            payload = g16 if dtype == "fp16" else torch.from_numpy(g16.view(np.int16)).view(torch.bfloat16)
            buf.accumulate(LF.GradMessage(l, payload, it))
            buf.ledger.messages_sent[l] += 1
        res = LF.sweep(buf, ms, hyper)
        applied = res.applied()
        for l in range(len(sizes)):
            ok = om.update_layer(l, O.from16(grads[l], dtype), lr=1e-3)
            assert applied[l] == ok, (it, l)
    assert ms.steps == om.steps
    for l in range(len(sizes)):
        np.testing.assert_array_equal(bits(ms.p32[l]), bits(om.p32[l]), err_msg=f"p32 layer {l}")
        np.testing.assert_array_equal(bits(ms.m32[l]), bits(om.m32[l]), err_msg=f"m32 layer {l}")
        np.testing.assert_array_equal(bits(ms.v32[l]), bits(om.v32[l]), err_msg=f"v32 layer {l}")
        pub = buf.read(l)[1]
        pub = bits(pub) if dtype == "fp16" else np.asarray(pub).view(np.uint16)
        np.testing.assert_array_equal(pub, bits(O.publish16(om.p32[l], dtype)), err_msg=f"p16 {l}")
        assert buf.version(l) == 5 and buf.applied_iter(l) == 4
    # Conservation (lockfree.py:275-326): every layer balances except the one
    # that received a NaN gradient, whose f64 sums are NaN exactly as in the
    # reference ledger.
    summary = buf.ledger.summary()["layers"]
    assert [l["layer"] for l in summary if not l["balanced"]] == [4]
    assert all(l["messages_sent"] == l["messages_accumulated"] == l["messages_consumed"] == 5
               for l in summary)


def test_three_call_path_equals_sweep(cuda):
    sizes = _layer_sizes()
    rng = np.random.default_rng(9)
    params = [rng.normal(0, 0.02, n).astype(np.float32) for n in sizes]
    a_buf, a_ms = LF.ParamBuffer(params, page_bytes=64 * 1024), LF.MasterState(params, page_bytes=64 * 1024)
    b_buf, b_ms = LF.ParamBuffer(params, page_bytes=64 * 1024), LF.MasterState(params, page_bytes=64 * 1024)
    hyper = LF.AdamHyper()
    for it in range(3):
        for l, n in enumerate(sizes):
            g = rng.normal(0, 1e-2, n).astype(np.float16)
            a_buf.accumulate(LF.GradMessage(l, g, it))
            b_buf.accumulate(LF.GradMessage(l, g, it))
        LF.sweep(a_buf, a_ms, hyper)
        for l in reversed(range(len(sizes))):  # the reference actor loop, lockfree.py:624-639
            grad, _, newest = b_buf.take(l)
            b_ms.update_layer(l, grad, hyper)
            b_buf.publish(l, b_ms.p32[l], applied_iter=newest, clear=False)
    for l in range(len(sizes)):
        np.testing.assert_array_equal(bits(a_ms.p32[l]), bits(b_ms.p32[l]))
        np.testing.assert_array_equal(bits(a_buf.read(l)[1]), bits(b_buf.read(l)[1]))


@pytest.mark.parametrize("groups", [1, 3, 8])
def test_ingest_sweep_equals_accumulate_then_sweep(cuda, groups):
    """The pipelined host-gradient step (per layer group: H2D -> K3 -> sweep)
    is bit-identical to accumulate_flat + one sweep, including a rejected layer."""
    sizes = _layer_sizes()
    rng = np.random.default_rng(21)
    params = [rng.normal(0, 0.02, n).astype(np.float32) for n in sizes]
    tp = [torch.from_numpy(p) for p in params]
    a_buf, a_ms = LF.ParamBuffer(tp, dtype="bf16", page_bytes=64 * 1024), LF.MasterState(tp, page_bytes=64 * 1024)
    b_buf, b_ms = LF.ParamBuffer(tp, dtype="bf16", page_bytes=64 * 1024), LF.MasterState(tp, page_bytes=64 * 1024)
    hyper = LF.AdamHyper(lr=1e-3)
    for it in range(3):
        g = rng.normal(0, 1e-2, sum(sizes)).astype(np.float32)
        if it == 1:
            g[sizes[0] + sizes[1] + 3] = np.inf   # an element of layer 2: rejected this step
        host = torch.from_numpy(O.to16(g, "bf16").view(np.int16)).view(torch.bfloat16).pin_memory()
        ra = LF.ingest_sweep(a_buf, a_ms, host, hyper, it, groups=groups).applied()
        b_buf.accumulate_flat(host.cuda(), it)
        rb = LF.sweep(b_buf, b_ms, hyper).applied()
        assert ra == rb and ra[2] == (it != 1)
    assert a_ms.steps == b_ms.steps
    for l in range(len(sizes)):
        assert torch.equal(a_ms.p32[l].view(torch.int32), b_ms.p32[l].view(torch.int32))
        assert torch.equal(a_buf.layer_view(l).view(torch.int16), b_buf.layer_view(l).view(torch.int16))
