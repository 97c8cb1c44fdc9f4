"""The synthetic BASELINE workloads (paper_2303_02868_b200/workloads.py)
against the reference's own tensor inventory (hiermem/footprint.py:184-219):
for every GPT config the param16 specs — name, kind, bytes, layer index, in
emission order — equal the reference's, before the embeddings this build
appends (the reference excludes them, footprint.py:8).  Pinned by
tests/golden/inventory_param16.json (written by oracle/gen_golden.py from the
reference itself) so it also runs where /root/reference is absent, and
re-checked live against the reference when it is importable."""
import json
import sys
from pathlib import Path

import pytest

from conftest import GOLDEN
from paper_2303_02868_b200 import workloads as W

GPT = {"c1": 12, "c2": 24, "c3": 40, "c5": 1}
PARAMS = {"c1": 124_336_896, "c2": 1_315_178_496, "c3": 12_851_123_200, "c5": 1_811_963_904}


def _ours(name):
    specs = W.config_specs(name)
    body = [s for s in specs if not s.name.startswith(("wte.", "wpe."))]
    return [[s.name, s.kind, s.bytes, s.layer_index] for s in body], specs


@pytest.mark.parametrize("name", sorted(GPT))
def test_param16_inventory_matches_reference_golden(name):
    gold = json.loads((GOLDEN / "inventory_param16.json").read_text())[name]
    body, specs = _ours(name)
    assert body == gold
    assert len(gold) == 6 * GPT[name]
    # SURVEY.md §8(d) sizes (embeddings included for the GPT-2/3 model configs)
    assert W.total_elems(specs) == PARAMS[name]


def test_live_reference_inventory():
    ref = Path("/root/reference/pkg/src")
    if not ref.exists():
        pytest.skip("reference checkout absent (GPU box)")
    sys.path.insert(0, str(ref))
    from hiermem import footprint
    shapes = {"c1": (1024, 768, 3072, 12, 12), "c2": (2048, 2048, 8192, 24, 16),
              "c3": (2048, 5120, 20480, 40, 40), "c5": (2048, 12288, 49152, 1, 96)}
    for name, (seq, d, f, layers, heads) in shapes.items():
        cfg = footprint.TransformerConfig(1, seq, d, f, layers, heads)
        want = [[s.name, s.kind, s.bytes, s.layer_index] for s in footprint.tensor_inventory(cfg)
                if s.kind == "param16"]
        assert _ours(name)[0] == want, name
