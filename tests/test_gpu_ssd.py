"""SSD page tier (ssd.py): fp32 state in a file, pread -> H2D -> page-Adam ->
D2H -> pwrite per page group, pipelined — bit-exact vs the oracle, with
small groups so pinned slots and HBM stages are reused many times."""
import numpy as np
import pytest
import torch

from oracle import page_adam as O
from paper_2303_02868_b200 import lockfree as LF
from paper_2303_02868_b200.ssd import SSDMasterState, ssd_sweep

pytestmark = pytest.mark.gpu
SIZES = [70001, 1, 5, 32768, 40000, 25003, 777, 65539, 12, 33333, 200000]


@pytest.mark.parametrize("group_pages,slots", [(1, 3), (2, 2), (64, 4)])
def test_ssd_sweep_matches_oracle(cuda, tmp_path, group_pages, slots):
    rng = np.random.default_rng(8)
    params = [rng.normal(0, 0.02, n).astype(np.float32) for n in SIZES]
    buf = LF.ParamBuffer(params, dtype="bf16", page_bytes=64 * 1024)
    sm = SSDMasterState(params, str(tmp_path / "state.bin"), page_bytes=64 * 1024,
                        group_pages=group_pages, slots=slots)
    om = O.OracleMasters(params)
    for it in range(3):
        grads = []
        for l, n in enumerate(SIZES):
            g = rng.normal(0, 1e-2, n).astype(np.float32)
            if it == 1 and l == 3:
                g[7] = np.inf
            g16 = O.to16(g, "bf16")
            grads.append(g16)
            buf.accumulate(LF.GradMessage(l, torch.from_numpy(g16.view(np.int16)).view(torch.bfloat16), it))
        applied = ssd_sweep(buf, sm, LF.AdamHyper(lr=1e-3)).applied()
        for l in range(len(SIZES)):
            assert applied[l] == om.update_layer(l, O.from16(grads[l], "bf16"), lr=1e-3)
    assert sm.steps == om.steps
    for l in range(len(SIZES)):
        np.testing.assert_array_equal(sm.p32[l].view(np.uint32), om.p32[l].view(np.uint32))
        np.testing.assert_array_equal(sm.m32[l].view(np.uint32), om.m32[l].view(np.uint32))
        np.testing.assert_array_equal(sm.v32[l].view(np.uint32), om.v32[l].view(np.uint32))
        np.testing.assert_array_equal(np.asarray(buf.read(l)[1]).view(np.uint16), O.to16(om.p32[l], "bf16"))
    sm.close()
