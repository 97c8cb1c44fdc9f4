"""The tracer's measured timing tables (presets/b200-timing-*.json, emitted
by tracing.LayerTracer on a B200 via tools/calibrate_timing.py) are accepted
by the reference's own planning stack: TimingModel.from_dict, build_trace
(hiermem/tracer.py:138-170, a table entry for every non-optimizer tensor),
validate_trace, and Algorithm 1's schedule() + validate_schedule over the
traced lifetimes (hiermem/scheduler.py:388-457).  Skipped where
/root/reference is absent (the GPU box)."""
import json
import sys
from pathlib import Path

import pytest

from conftest import ROOT

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="needs the reference package (build container)")


@pytest.mark.parametrize("preset,model,budget_gib", [("b200-timing-tiny-2layer.json", "tiny-2layer", 0.012),
                                                     ("b200-timing-gpt3-1.7b.json", "gpt3-1.7b", 8)])
def test_reference_plans_with_measured_tables(preset, model, budget_gib):
    sys.path.insert(0, str(REF))
    from hiermem import footprint, presets
    from hiermem.scheduler import LayerModel, ShardingModel, schedule, validate_schedule
    from hiermem.tracer import LogicalTimeline, TimingModel, build_trace, validate_trace
    raw = json.loads((ROOT / "presets" / preset).read_text())
    timing = TimingModel.from_dict({"kind": raw["kind"], "table": raw["table"]})
    cfg = presets.model_preset(model)
    inv = footprint.tensor_inventory(cfg)
    traces = build_trace(inv, timing)                         # raises if any name is missing
    assert not validate_trace(traces, LogicalTimeline.build(cfg.num_layers, traces))
    assert any(t.gpu_time > 0 for t in traces) and any(t.cpu_time > 0 for t in traces)
    lm = LayerModel.from_inventory(inv, 4 << 20, cfg.batch_size)
    sched = schedule(lm, traces, int(budget_gib * 2**30), ShardingModel(1, 0))
    assert not validate_schedule(sched, traces, int(budget_gib * 2**30))
