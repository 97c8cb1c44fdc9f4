"""Pinned-host swap tier (swap.py): state in host pages, fetched/updated/
stored group by group in reverse page order — bit-exact vs the oracle, with
small groups so that slots are reused many times within one sweep."""
import numpy as np
import pytest
import torch

from oracle import page_adam as O
from paper_2303_02868_b200 import lockfree as LF
from paper_2303_02868_b200.swap import HostMasterState, swap_sweep

pytestmark = pytest.mark.gpu

SIZES = [70001, 1, 5, 32768, 40000, 25003, 777, 65539, 12, 33333, 200000]


@pytest.mark.parametrize("group_pages,slots", [(1, 2), (2, 3), (64, 2)])
def test_swap_sweep_matches_oracle(cuda, group_pages, slots):
    rng = np.random.default_rng(3)
    params = [rng.normal(0, 0.02, n).astype(np.float32) for n in SIZES]
    buf = LF.ParamBuffer(params, dtype="bf16", page_bytes=64 * 1024)
    hm = HostMasterState(params, page_bytes=64 * 1024, group_pages=group_pages, slots=slots)
    om = O.OracleMasters(params)
    for it in range(4):
        grads = []
        for l, n in enumerate(SIZES):
            g = rng.normal(0, 1e-2, n).astype(np.float32)
            if it == 2 and l == 9:
                g[0] = np.nan
            g16 = O.to16(g, "bf16")
            grads.append(g16)
            buf.accumulate(LF.GradMessage(l, torch.from_numpy(g16.view(np.int16)).view(torch.bfloat16), it))
        applied = swap_sweep(buf, hm, LF.AdamHyper(lr=1e-3)).applied()
        for l in range(len(SIZES)):
            assert applied[l] == om.update_layer(l, O.from16(grads[l], "bf16"), lr=1e-3)
    assert hm.steps == om.steps
    for l in range(len(SIZES)):
        np.testing.assert_array_equal(hm.p32[l].view(np.uint32), om.p32[l].view(np.uint32))
        np.testing.assert_array_equal(hm.m32[l].view(np.uint32), om.m32[l].view(np.uint32))
        np.testing.assert_array_equal(hm.v32[l].view(np.uint32), om.v32[l].view(np.uint32))
        pub = np.asarray(buf.read(l)[1]).view(np.uint16)
        np.testing.assert_array_equal(pub, O.to16(om.p32[l], "bf16"))
