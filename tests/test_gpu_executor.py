"""Algorithm-1 schedules of the reference executed with real bytes
(executor.ScheduleExecutor): the native allocator never exceeds the
schedule's GPU budget, every page survives its H2D/D2H round trips bit for
bit, and every task runs.  The schedules and their simulated makespans on the
measured B200 profile come from the reference itself
(tests/golden/schedules.json.gz, oracle/gen_golden.py)."""
import gzip
import json

import pytest

from conftest import GOLDEN
from paper_2303_02868_b200.executor import ScheduleExecutor

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def schedules():
    with gzip.open(GOLDEN / "schedules.json.gz", "rt") as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["tiny-2layer", "gpt3-1.7b"])
def test_schedule_runs_within_budget_and_preserves_pages(cuda, schedules, name):
    entry = schedules[name]
    sched = entry["schedule"]
    ex = ScheduleExecutor(sched, slot_seconds=entry["simulated"]["compute_s_by_slot"])
    rep = ex.run()
    ops = {}
    for t in sched["tasks"]:
        ops[t["operation"]] = ops.get(t["operation"], 0) + 1
    assert rep["tasks"] == {k: ops.get(k, 0) for k in rep["tasks"]}
    assert rep["bytes_intact"]
    assert rep["gpu_pages_peak"] <= sched["gpu_budget"] // sched["model"]["page_bytes"]
    assert rep["makespan_s"] > 0
    print(name, rep, "simulated", entry["simulated"]["makespan_s"])
