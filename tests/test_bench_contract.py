"""bench.py's JSON contract on the CPU-runnable arm (--impl reference): one
line with every key the driver reads, the reference arm's own keys, and the
W >= 3 warm-up rule."""
import json
import subprocess
import sys

from conftest import ROOT

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_line():
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--cpu-sample-pages", "1", "--config", "c1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "params/s" and d["value"] > 0
    assert d["warmup"] >= 3 and d["steps"] == 1
    assert d["metric"] == json.loads((ROOT / "BASELINE.json").read_text())["metric"]
    cb = d["cpu_baseline"]
    # the reference itself when baseline/_ref holds it, else the oracle port
    want = "reference" if (ROOT / "baseline" / "_ref" / "hiermem").exists() else "port"
    assert cb["kind"] == want and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("c1")


def test_both_arms_print_the_same_config():
    """The GPU arm's config is built by the same function (bench.gpu_config),
    so the driver's same-config check compares like with like."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", ROOT / "bench.py")
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    src = (ROOT / "bench.py").read_text()
    assert src.count('"config": gpu_config(args, specs, page, layout)') == 1   # the GPU arm
    assert "cfg = gpu_config(args, specs, page, layout)" in src               # the reference arm
