"""CPU side of the whole-chain equivalence (reference tests/test_lockfree.py:
137-141): the restated toy problem (tests/toy_ref.py) equals the
reference's, and the restated synchronous loop driven by the REFERENCE's
own ParamBuffer / MasterState reproduces tests/golden/toy_sync.json bit for
bit — so the same loop driven by the drop-in (tests/test_gpu_toy_sync.py)
is a test of the drop-in alone.  Skipped where /root/reference is absent."""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN
import toy_ref as T

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="needs the reference package (build container)")


@pytest.fixture(scope="module")
def hm():
    sys.path.insert(0, str(REF))
    import hiermem.lockfree as lf
    return lf


def _cfg(gold):
    c = gold["cfg"]
    return T.ToyCfg(c["num_layers"], c["dim"], c["batch_size"], c["seed"], c["noise_std"])


def test_restated_problem_matches_reference(hm):
    gold = json.loads((GOLDEN / "toy_sync.json").read_text())
    cfg = _cfg(gold)
    rcfg = hm.ToyTrainConfig(num_layers=cfg.num_layers, dim=cfg.dim, batch_size=cfg.batch_size,
                             seed=cfg.seed, noise_std=cfg.noise_std)
    a, b = T.problem(cfg), hm.init_problem(rcfg)
    for x, y in zip(a[0] + a[1] + [a[2], *a[3]], b[0] + b[1] + [b[2], *b[3]]):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    for it in (0, 7):
        xa, ya = T.batch(cfg, a[0], a[2], it)
        xb, yb = hm.batch_for(rcfg, b[0], b[2], it)
        assert np.array_equal(xa, xb) and np.array_equal(ya, yb)
        la, ga = T.loss_and_grads(a[1], a[2], xa, ya)
        lb, gb = hm.forward_backward(b[1], b[2], xb, yb)
        assert la == lb and all(np.array_equal(u.view(np.uint32), v.view(np.uint32)) for u, v in zip(ga, gb))


def test_loop_with_reference_classes_reproduces_golden(hm):
    gold = json.loads((GOLDEN / "toy_sync.json").read_text())
    cfg = _cfg(gold)
    cfg.hyper = hm.AdamHyper()
    teacher, student, readout, _ = T.problem(cfg)
    buf, ms = hm.ParamBuffer(student), hm.MasterState(student)
    curve = T.run_sync_loop(buf, ms, cfg, gold["iterations"], cfg.hyper, teacher, readout, hm.GradMessage)
    assert curve == gold["loss_curve"]
    s = buf.ledger.summary()
    assert s["balanced"]
