"""Host-glue concurrency and the accumulate kernel's launch shapes.

* update_layer / sweep on two streams at once: every launch carries its own
  stream's scratch (prologue runtime table, reject flag) and its own launch
  settings, so interleaved updates of two MasterStates on two streams are
  bit-identical to running them one after the other.
* K3 (hm_accumulate) in its three forms (first messages, adds, per-slot
  mixed), fp16 and bf16: bit-exact against the oracle's accumulate, with
  the same reject flags and ledger sums.
* ingest_sweep(results_to=...): the published pages land in host memory,
  equal to the device record.
"""
import numpy as np
import pytest
import torch

from oracle import page_adam as O
from paper_2303_02868_b200 import lockfree as LF

pytestmark = pytest.mark.gpu
SIZES = [70001, 1, 5, 32768, 40000, 25003, 777, 65539, 12, 33333]
PAGE = 64 * 1024


def _params(seed):
    rng = np.random.default_rng(seed)
    return [torch.from_numpy(rng.normal(0, 0.02, n).astype(np.float32)).cuda() for n in SIZES]


def test_update_layer_two_streams_bit_exact(cuda):
    hyper = LF.AdamHyper(lr=1e-3)
    rng = np.random.default_rng(3)
    grads = [[torch.from_numpy(rng.normal(0, 1e-2, n).astype(np.float32)).cuda() for n in SIZES]
             for _ in range(2)]
    grads[1][4][7] = float("nan")   # one rejected layer on the second state
    ref = [LF.MasterState(_params(s), page_bytes=PAGE) for s in (1, 2)]
    for k in range(2):                               # sequential reference
        for _ in range(3):
            for l in reversed(range(len(SIZES))):
                bool(ref[k].update_layer(l, grads[k][l], hyper))
    got = [LF.MasterState(_params(s), page_bytes=PAGE) for s in (1, 2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    res = [[], []]
    torch.cuda.synchronize()
    for _ in range(3):
        for l in reversed(range(len(SIZES))):        # interleaved launches on two streams
            for k in range(2):
                res[k].append(got[k].update_layer(l, grads[k][l], hyper, stream=streams[k]))
    torch.cuda.synchronize()
    assert [bool(r) for r in res[1]].count(False) == 3
    for k in range(2):
        assert got[k].steps == ref[k].steps
        for l in range(len(SIZES)):
            assert torch.equal(got[k].p32[l].view(torch.int32), ref[k].p32[l].view(torch.int32))
            assert torch.equal(got[k].v32[l].view(torch.int32), ref[k].v32[l].view(torch.int32))


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_accumulate_kinds_bit_exact(cuda, dtype):
    """The three K3 forms — all first messages, all adds, per-slot mixed —
    against the oracle's accumulate (lockfree.py:219-220), with the reject
    flags and the ledger's running sums."""
    rng = np.random.default_rng(11)
    L = len(SIZES)
    buf = LF.ParamBuffer([np.zeros(n, np.float32) for n in SIZES], dtype=dtype, page_bytes=PAGE)
    acc = [None] * L   # the oracle's 16-bit gradient buffer per layer
    taken = {2, 5}
    for it in range(3):
        if it == 2:                      # mixed: two layers start over after a take
            for l in taken:
                buf.take(l)
                acc[l] = None
        flat = []
        for l, n in enumerate(SIZES):
            g = O.to16((rng.normal(0, 1, n) * 10.0 ** rng.integers(-3, 3, n)).astype(np.float32), dtype)
            if it == 2 and l == 6:
                g[9] = O.to16(np.array([np.inf], np.float32), dtype)[0]
            flat.append(g)
            base = acc[l] if acc[l] is not None else O.to16(np.zeros(n, np.float32), dtype)
            acc[l] = O.accumulate16(base, g, dtype)
        f = np.concatenate(flat)
        t = torch.from_numpy(f.view(np.int16)).view(torch.bfloat16) if dtype == "bf16" else torch.from_numpy(f)
        buf.accumulate_flat(t.cuda(), it)
    want = [O.from16(a, dtype) for a in acc]
    for l in range(L):
        got = buf.g16[l]
        got = O.from16(np.asarray(got).view(np.uint16) if dtype == "bf16" else got, dtype)
        assert np.array_equal(got.view(np.uint32), want[l].view(np.uint32)), l
    slot = [buf._gsel[l] * L + l for l in range(L)]
    flags = buf._flags.cpu().numpy()
    assert [int(flags[slot[l]]) for l in range(L)] == [int(l == 6) for l in range(L)]
    sums = buf._lsum.cpu().numpy()
    for l in range(L):
        if l != 6:
            assert sums[slot[l]] == pytest.approx(float(np.sum(want[l].astype(np.float64))),
                                                  rel=1e-12, abs=1e-12), l


def test_ingest_sweep_returns_published_pages(cuda):
    params = _params(4)
    buf, ms = LF.ParamBuffer(params, dtype="bf16", page_bytes=PAGE), LF.MasterState(params, page_bytes=PAGE)
    rng = np.random.default_rng(8)
    host_out = torch.empty(sum(SIZES), dtype=torch.bfloat16).pin_memory()
    for it in range(2):
        g = torch.from_numpy(rng.normal(0, 1e-2, sum(SIZES)).astype(np.float32)).to(torch.bfloat16).pin_memory()
        LF.ingest_sweep(buf, ms, g, LF.AdamHyper(lr=1e-3), it, groups=3, results_to=host_out)
        torch.cuda.synchronize()
        pos = 0
        for l, n in enumerate(SIZES):
            assert torch.equal(host_out[pos:pos + n].view(torch.int16),
                               buf.layer_view(l).cpu().view(torch.int16)), (it, l)
            pos += n


def test_three_call_fast_path_rejects_every_time(cuda):
    """update_layer on a taken tensor re-uses the reject flag the accumulate
    computed; calling it twice with a NaN gradient must reject twice, like
    the reference's apply_update (hiermem/lockfree.py:133-134)."""
    params = [torch.zeros(4096, device="cuda"), torch.zeros(100, device="cuda")]
    buf, ms = LF.ParamBuffer(params, page_bytes=PAGE), LF.MasterState(params, page_bytes=PAGE)
    g = torch.ones(4096, dtype=torch.float16, device="cuda")
    g[17] = float("nan")
    buf.accumulate(LF.GradMessage(0, g, 0))
    gr, _, _ = buf.take(0)
    assert not bool(ms.update_layer(0, gr, LF.AdamHyper()))
    assert not bool(ms.update_layer(0, gr, LF.AdamHyper()))
    assert ms.steps == [0, 0]
    # the slot starts clean for the next first message
    buf.accumulate(LF.GradMessage(0, torch.ones(4096, dtype=torch.float16, device="cuda"), 1))
    gr, _, _ = buf.take(0)
    buf.accumulate(LF.GradMessage(0, torch.ones(4096, dtype=torch.float16, device="cuda"), 2))
    assert bool(ms.update_layer(0, gr, LF.AdamHyper()))
    assert ms.steps == [1, 0]


def test_deferred_take_snapshots_across_streams(cuda):
    """``take`` records the ledger's take sum (hiermem/lockfree.py:237) by a
    deferred launch shared by every take since the last flush.  Takes on one
    stream, accumulates on another (whose first message resets the slot the
    snapshot reads), and a publish(clear=True) in between: every consumed
    sum equals the f64 sum of the gradient the take returned, the counts
    match and the ledger balances."""
    rng = np.random.default_rng(11)
    params = _params(3)
    buf = LF.ParamBuffer(params, dtype="fp16", page_bytes=PAGE)
    s_take, s_acc = torch.cuda.Stream(), torch.cuda.Stream()
    want = [[] for _ in SIZES]
    for it in range(5):
        s_acc.wait_stream(s_take)          # the data dependency a caller owns (pages reused)
        with torch.cuda.stream(s_acc):
            for l, n in enumerate(SIZES):
                for _ in range(1 + (l + it) % 2):
                    g = torch.from_numpy(rng.normal(0, 1e-2, n).astype(np.float16)).cuda()
                    buf.accumulate(LF.GradMessage(l, g, it))
        s_take.wait_stream(s_acc)
        for l in reversed(range(len(SIZES))):
            if it == 2 and l == 3:
                with torch.cuda.stream(s_take):
                    got = buf.read(l)[1].float().sum(dtype=torch.float64)   # keep the stream busy
                buf.publish(l, params[l], clear=True, stream=s_take)        # a clear-consume instead of a take
                want[l].append(None)
                continue
            g, _c, _n = buf.take(l, stream=s_take)
            with torch.cuda.stream(s_take):
                want[l].append(g.double().sum())
    torch.cuda.synchronize()
    import math
    consumed, produced = buf.ledger.consumed_sums, buf.ledger.produced_deltas
    for l in range(len(SIZES)):
        assert len(consumed[l]) == len(want[l])
        for c, w in zip(consumed[l], want[l]):
            if w is not None:
                assert c == pytest.approx(float(w), rel=1e-6, abs=1e-9)
        # conservation (lockfree.py:300-326): what was produced was consumed
        assert math.fsum(produced[l]) == math.fsum(consumed[l]), l
    assert buf.ledger.messages_consumed == buf.ledger.messages_accumulated


def _bits(t):
    return t.detach().contiguous().view(torch.int32).cpu().numpy()


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("max_norm", [0.0, 0.05])
def test_fused_layer_update_matches_generic_path(cuda, dtype, max_norm):
    """The three-call update_layer on a taken tensor is ONE hm_adam_layer
    launch (prologue fused; the new masters also written as the contiguous
    tensor p32[l] hands out once).  It must equal the generic update_layer
    (prologue + main kernel over the f32 tensor, unpack on read): bit-exact
    without clipping, within f32 rounding of the clip coefficient with it
    (the two paths sum the squared norm in different orders).  Covers
    layers whose tensor offsets are not 8-aligned (SIZES), a rejected
    layer, a second p32 read (unpacked), and a sweep after an unclaimed
    fused update (the stale tensor must not be handed out)."""
    rng = np.random.default_rng(21)
    params = _params(5)
    hyper = LF.AdamHyper(lr=1e-3, max_norm=max_norm)
    buf = LF.ParamBuffer(params, dtype=dtype, page_bytes=PAGE)
    fast, slow = LF.MasterState(params, page_bytes=PAGE), LF.MasterState(params, page_bytes=PAGE)
    t16 = torch.float16 if dtype == "fp16" else torch.bfloat16
    same = (lambda a, b: np.array_equal(_bits(a), _bits(b))) if max_norm == 0 else \
        (lambda a, b: torch.allclose(a, b, rtol=2e-6, atol=1e-9))
    for it in range(4):
        for l, n in enumerate(SIZES):
            g = torch.from_numpy(rng.normal(0, 1e-2, n).astype(np.float32)).cuda()
            if it == 2 and l == 3:
                g[n // 3] = float("inf")
            buf.accumulate(LF.GradMessage(l, g.to(t16), it))
        for l in reversed(range(len(SIZES))):
            gr, _c, newest = buf.take(l)
            ok_f = fast.update_layer(l, gr, hyper)
            ok_s = slow.update_layer(l, gr.clone(), hyper)
            assert bool(ok_f) == bool(ok_s) == (not (it == 2 and l == 3)), (it, l)
            pf, pf2, ps = fast.p32[l], fast.p32[l], slow.p32[l]
            assert same(pf, ps) and np.array_equal(_bits(pf), _bits(pf2)), (it, l)
            buf.publish(l, pf, applied_iter=newest, clear=False)
    assert fast.steps == slow.steps
    for l in range(len(SIZES)):
        assert same(fast.m32[l], slow.m32[l]) and same(fast.v32[l], slow.v32[l]), l
    # an unclaimed fused result, then a sweep of the same layer: p32 reads the new state
    buf.accumulate(LF.GradMessage(0, torch.ones(SIZES[0], dtype=t16, device="cuda") * 1e-2, 9))
    gr, _c, _n = buf.take(0)
    fast.update_layer(0, gr, hyper)
    buf.accumulate(LF.GradMessage(0, torch.ones(SIZES[0], dtype=t16, device="cuda") * 1e-2, 10))
    LF.sweep(buf, fast, hyper, layers=[0])
    p = fast.p32[0]
    assert np.array_equal(_bits(p), _bits(fast._unpack(fast.p32_pool, 0)))
