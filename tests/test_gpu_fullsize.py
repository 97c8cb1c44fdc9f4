"""Parity at the BASELINE.json sizes, through the C-ABI.

* C1 (GPT-2 small, 124.3M params, 103 pages of 4 MiB, 13 shared tails):
  every element of every layer, two fused sweeps, bit-exact vs the oracle.
* C2 (GPT-3 1.3B), C4 (T5-MoE, 9,552 pages of 256 KiB), C5 (175B layer
  slice at 1 MiB and 64 MiB pages), C3 (13B slice through the pinned-host
  swap tier): a seeded sample of pages is checked bit-exact.  A page's new
  contents depend only on its own bytes and its layer's step, so a sample
  is a size-independent check of the whole pass.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from oracle import page_adam as O
from paper_2303_02868_b200 import lockfree as LF
from paper_2303_02868_b200 import workloads as W
from paper_2303_02868_b200.layout import PageLayout

pytestmark = pytest.mark.gpu
HYPER = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8)


def _bits16(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def _make(config, page=None, device="cuda:0", swap=False, layers=None):
    specs = W.config_specs(config) if layers is None else W.gpt_param16(
        W.GPTShape(2048, 5120, 20480, layers))
    page = page or W.config_page_bytes(config)
    numels = [s.bytes // 2 for s in specs]
    lay = PageLayout(numels, page)
    gen = torch.Generator(device=device)
    gen.manual_seed(11)
    params = [torch.empty(n, device=device).normal_(0, 0.02, generator=gen) for n in numels]
    buf = LF.ParamBuffer(params, dtype="bf16", page_bytes=page, device=device, layout=lay)
    if swap:
        from paper_2303_02868_b200.swap import HostMasterState
        ms = HostMasterState(params, page_bytes=page, device=device, layout=lay, group_pages=16)
    else:
        ms = LF.MasterState(params, page_bytes=page, device=device, layout=lay)
    return lay, buf, ms, params


def _grads(lay, seed, device="cuda:0"):
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    return torch.empty(sum(lay.numels), device=device).normal_(0, 1e-2, generator=gen).to(torch.bfloat16)


def _run(lay, buf, ms, params, steps, sample_pages, swap=False):
    """Run `steps` fused sweeps; return per-sampled-segment oracle comparison."""
    # host copies of the inputs of the sampled segments
    rng = np.random.default_rng(0)
    pages = sorted(set(rng.choice(lay.used_pages, size=min(sample_pages, lay.used_pages), replace=False).tolist())) \
        if sample_pages else list(range(lay.used_pages))
    segs = [s for l in range(len(lay.numels)) for s in lay.segments[l] if s.page in pages]
    state = {}
    for s in segs:
        p = params[s.layer][s.pos:s.pos + s.n].cpu().numpy()
        state[(s.layer, s.pos)] = [p, np.zeros_like(p), np.zeros_like(p)]
    starts = np.cumsum([0] + lay.numels[:-1])
    sweep = LF.sweep
    if swap:
        from paper_2303_02868_b200.swap import swap_sweep as sweep
    for step in range(1, steps + 1):
        g = _grads(lay, 100 + step)
        buf.accumulate_flat(g, step)
        res = sweep(buf, ms, LF.AdamHyper(**HYPER))
        assert all(res.applied().values())
        gh = _bits16(g)

        def upd(s):
            key = (s.layer, s.pos)
            a = int(starts[s.layer]) + s.pos
            gg = O.from16(gh[a:a + s.n], "bf16")
            p, m, v, ok = O.adam_update(*state[key], gg, step=step, **HYPER)
            state[key] = [p, m, v]

        with ThreadPoolExecutor(16) as ex:
            list(ex.map(upd, segs))
    torch.cuda.synchronize()
    p16 = _bits16(buf.p16_pool[buf._psel[0]])
    bad = []
    for s in segs:
        p, m, v = state[(s.layer, s.pos)]
        o = lay.slot_state(s.page) * lay.E + s.off
        if swap:
            got_p = ms.host_p[o:o + s.n].numpy()
            got_v = ms.host_v[o:o + s.n].numpy()
        else:
            got_p = ms.p32_pool[o:o + s.n].cpu().numpy()
            got_v = ms.v32_pool[o:o + s.n].cpu().numpy()
        if not np.array_equal(got_p.view(np.uint32), p.view(np.uint32)):
            bad.append(("p32", s))
        if not np.array_equal(got_v.view(np.uint32), v.view(np.uint32)):
            bad.append(("v32", s))
        o16 = lay.slot16(s.page) * lay.E + s.off
        if not np.array_equal(p16[o16:o16 + s.n], O.to16(p, "bf16")):
            bad.append(("p16", s))
    return segs, bad


def test_c1_full_bit_exact(cuda):
    lay, buf, ms, params = _make("c1")
    assert lay.used_pages == 103
    segs, bad = _run(lay, buf, ms, params, steps=2, sample_pages=0)
    assert sum(s.n for s in segs) == 124_336_896
    assert not bad, bad[:5]


@pytest.mark.parametrize("config,page", [("c2", None), ("c4", None), ("c5", 2**20), ("c5", 64 * 2**20)])
def test_sampled_pages_bit_exact(cuda, config, page):
    lay, buf, ms, params = _make(config, page)
    segs, bad = _run(lay, buf, ms, params, steps=2, sample_pages=24)
    assert segs and not bad, bad[:5]
    del buf, ms, params
    torch.cuda.empty_cache()


def test_c3_swap_slice_sampled(cuda):
    lay, buf, ms, params = _make("c3", swap=True, layers=2)
    segs, bad = _run(lay, buf, ms, params, steps=2, sample_pages=24, swap=True)
    assert segs and not bad, bad[:5]
