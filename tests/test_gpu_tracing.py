"""Tracer hooks (tracing.LayerTracer): measured per-op times become a
TimingModel(kind="table") covering every tensor name of the reference
inventory (hiermem/footprint.py:184-219) with non-negative times."""
import pytest

from paper_2303_02868_b200 import workloads as W
from paper_2303_02868_b200.tracing import ROWS, LayerTracer

pytestmark = pytest.mark.gpu


def test_timing_table_covers_inventory(cuda):
    tr = LayerTracer(seq_len=128, d_model=256, d_ffn=1024, num_heads=4)
    d = tr.timing_table(num_layers=2, update_params_per_s=2.4e11, reps=3)
    assert d["kind"] == "table"
    table = d["table"]
    # the param16 names of the reference inventory for this shape
    names = {s.name for s in W.gpt_param16(W.GPTShape(128, 256, 1024, 2), embeddings=False)}
    assert names <= set(table)
    for name, (cpu, gpu) in table.items():
        assert cpu >= 0.0 and gpu >= 0.0, name
    # every name the reference's build_trace looks up (all but optim32,
    # hiermem/tracer.py:102-107) — pinned by a golden of the reference
    # inventory; tests/test_tracer_presets.py feeds tables of this format to
    # the reference itself
    import json
    from conftest import GOLDEN
    need = json.loads((GOLDEN / "tracer_inventory.json").read_text())["names"]
    missing = [n for n in need if n not in table]
    assert not missing, missing[:5]
    rows = d["_measured_rows"]
    assert set(rows) == set(ROWS)
    assert rows["ffn.linear_in"]["forward_s"] > 0
