"""Reference simulator (hiermem.simengine.simulate) on the gpt3-1.7b Algorithm-1
schedule with the measured B200 op-time table, swept over the PCIe rate it
assumes per direction — to explain the executor's measured makespan
(profiles/r1_executor.md).  Needs the reference checkout (build container
only): python tools/sim_pcie_sensitivity.py
"""
import json, os, sys
sys.path.insert(0, "/root/reference/pkg/src")   # reference: analysis only, never shipped
os.environ["HIERMEM_PRESET_DIR"] = "/root/repo/presets"
from hiermem import presets, footprint
from hiermem.scheduler import LayerModel, ShardingModel, schedule
from hiermem.simengine import simulate
from hiermem.tracer import TimingModel, build_trace
import dataclasses
prof = presets.hardware_preset("b200-server")
cfg = presets.model_preset("gpt3-1.7b")
inv = footprint.tensor_inventory(cfg)
raw = json.load(open("/root/repo/presets/b200-timing-gpt3-1.7b.json"))
timing = TimingModel.from_dict({"kind": raw["kind"], "table": raw["table"]})
traces = build_trace(inv, timing)
lm = LayerModel.from_inventory(inv, 4 * 2**20, cfg.batch_size)
sched = schedule(lm, traces, 8 * 2**30, ShardingModel(1, 0))
for bw in (55.5e9, 48e9, 40.8e9, 35e9):
    d = prof.to_dict()
    d["links"]["pcie_h2d"]["bandwidth_bytes_per_s"] = bw
    d["links"]["pcie_d2h"]["bandwidth_bytes_per_s"] = bw
    p2 = type(prof).from_dict(d) if hasattr(type(prof), "from_dict") else None
    sim = simulate(sched, traces, p2)
    print(bw/1e9, round(sim.makespan_s*1e3, 1), {k: round(v*1e3,1) for k, v in sim.busy_s.items()})
