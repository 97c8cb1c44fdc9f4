"""bench.py's GPU arm keeps the driver's contract (one JSON line with the
roofline / cpu_baseline / e2e / clocks / gpu_launches keys), on the small C1
workload so it stays quick."""
import json
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_line_keys(cuda):
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", "c1", "--steps", "5",
                          "--warmup", "3", "--e2e-steps", "1", "--cpu-sample-pages", "1", "--cpu-seconds", "1"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "clocks", "gpu_launches"):
        assert k in d, k
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["gpu_launches"] >= d["steps"] and d["n_gpus"] == 1 and d["warmup"] >= 3
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
