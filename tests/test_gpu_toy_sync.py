"""Whole-chain equivalence through the drop-in (reference tests/
test_lockfree.py:137-141 and :110-117): the reference's synchronous
training loop (hiermem/lockfree.py:731-769, restated in tests/toy_ref.py and
pinned against the reference classes by tests/test_toy_sync.py) driven by
THIS package's ParamBuffer / MasterState must reproduce the reference's loss
curve (tests/golden/toy_sync.json) bit for bit, and the always-on
conservation ledger must balance exactly as the reference's does.

Two IO forms: numpy in/out (the reference's own types, every call crosses
PCIe), and torch tensors (the take -> update_layer -> publish fast path:
update_layer reads the taken gradient's 16-bit pages in place and publish
only flips the record)."""
import json

import pytest
import torch

from conftest import GOLDEN
import toy_ref as T
from paper_2303_02868_b200 import lockfree as LF

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("torch_io", [False, True])
def test_run_sync_through_dropin_matches_reference(cuda, torch_io):
    gold = json.loads((GOLDEN / "toy_sync.json").read_text())
    c = gold["cfg"]
    cfg = T.ToyCfg(c["num_layers"], c["dim"], c["batch_size"], c["seed"], c["noise_std"])
    cfg.hyper = LF.AdamHyper()
    teacher, student, readout, _ = T.problem(cfg)
    params = [torch.from_numpy(p).cuda() for p in student] if torch_io else student
    buf = LF.ParamBuffer(params, dtype="fp16", page_bytes=64 * 1024)
    ms = LF.MasterState(params, page_bytes=64 * 1024)
    curve = T.run_sync_loop(buf, ms, cfg, gold["iterations"], cfg.hyper, teacher, readout,
                            LF.GradMessage, torch_io=torch_io)
    assert curve == gold["loss_curve"]            # bitwise float equality
    s = buf.ledger.summary()
    assert s["balanced"]
    for layer in s["layers"]:
        assert layer["produced"] == layer["consumed"] == layer["applied"]
        assert layer["messages_sent"] == layer["messages_accumulated"] == layer["messages_consumed"] \
            == gold["iterations"]


def test_ledger_flags_nan_layer_by_default(cuda):
    """A NaN gradient makes the reference ledger unbalanced for that layer
    (its f64 sums are NaN, hiermem/lockfree.py:218-222, 311): the drop-in's
    default ParamBuffer reports the same."""
    import numpy as np
    params = [np.zeros(300, np.float32), np.zeros(70, np.float32)]
    buf, ms = LF.ParamBuffer(params), LF.MasterState(params)
    g0 = np.ones(300, np.float16)
    g0[5] = np.nan
    for l, g in enumerate((g0, np.ones(70, np.float16))):
        buf.ledger.messages_sent[l] += 1
        buf.accumulate(LF.GradMessage(l, g, 0))
    res = LF.sweep(buf, ms, LF.AdamHyper()).applied()
    assert res == {0: False, 1: True}
    s = buf.ledger.summary()
    assert [l["balanced"] for l in s["layers"]] == [False, True]
    assert s["layers"][1]["produced"] == s["layers"][1]["consumed"] == s["layers"][1]["applied"] == 70.0
    assert s["layers"][0]["applied"] == 0.0 and s["layers"][0]["rejected"] != s["layers"][0]["rejected"]
