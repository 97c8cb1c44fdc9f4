"""Run the reference's Algorithm-1 schedules (tests/golden/schedules.json.gz)
with real bytes and compare the measured makespan with the reference
simulator's replay on the measured B200 profile (presets/b200-server.json).

    python tools/executor_bench.py [--reps 3]
"""
import argparse
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2303_02868_b200.executor import ScheduleExecutor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    with gzip.open(ROOT / "tests" / "golden" / "schedules.json.gz", "rt") as f:
        data = json.load(f)
    out = {}
    for name, entry in data.items():
        best = None
        for _ in range(args.reps):
            rep = ScheduleExecutor(entry["schedule"],
                                   slot_seconds=entry["simulated"]["compute_s_by_slot"]).run()
            if best is None or rep["makespan_s"] < best["makespan_s"]:
                best = rep
        sim = entry["simulated"]["makespan_s"]
        best["simulated_makespan_s"] = sim
        best["measured_over_simulated"] = best["makespan_s"] / sim
        out[name] = best
    print(json.dumps(out))


if __name__ == "__main__":
    main()
