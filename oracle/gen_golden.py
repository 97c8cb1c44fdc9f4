"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Generates tests/golden/* by running the REFERENCE package itself
(/root/reference/pkg/src/hiermem, importable in the build container only;
the GPU box never reads /root/reference).  Run:

    python oracle/gen_golden.py

Outputs
  adam_golden.npz          reference apply_update / MasterState / ParamBuffer
                           outputs on seeded inputs (fp16 = reference-native;
                           bf16 = reference math on exactly widened bf16 grads,
                           published through ml_dtypes.bfloat16)
  pagetable_random.json.gz reference state_dict + op log of oracle/pt_ops.py
                           scripts (seeds 0..39)
  pagetable_configs.json.gz reference page tables of the BASELINE configs
                           C1..C5 (param16 specs in a GPU pool)
  toy_sync.json            reference run_sync(ZERO) / reference_train loss
                           curves for the whole-chain equivalence test
  inventory_param16.json   param16 specs of the reference's tensor_inventory
                           for C1, C2, C3, C5
  tracer_inventory.json    the names a TimingModel table must cover for the
                           traced test shape
"""
from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/pkg/src")
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

import ml_dtypes  # noqa: E402
from hiermem import footprint, lockfree, pagemem  # noqa: E402
from hiermem.errors import AllocationError, MoveError  # noqa: E402

from oracle import pt_ops  # noqa: E402
from oracle.page_adam import synthetic_layer  # noqa: E402

MIB = 2 ** 20


def adam_cases():
    out = {}
    hypers = {"default": lockfree.AdamHyper(), "lr1e-3": lockfree.AdamHyper(lr=1e-3)}
    case = 0
    for dtype in ("fp16", "bf16"):
        for hname, hyper in hypers.items():
            for step in (1, 10, 1000):
                n = 4099 + 8 * case  # ragged lengths
                p, m, v, g16 = synthetic_layer(case, 0, n, dtype)
                if dtype == "fp16":
                    grad = g16  # reference-native fp16 gradient
                else:
                    grad = (g16.astype(np.uint32) << 16).view(np.float32)  # exact bf16 widen
                rp, rm, rv, ok = lockfree.apply_update(p, m, v, grad, hyper, step)
                assert ok
                p16 = rp.astype(np.float16).view(np.uint16) if dtype == "fp16" else \
                    rp.astype(ml_dtypes.bfloat16).view(np.uint16)
                key = f"c{case}"
                out[f"{key}.meta"] = np.array([n, step, hyper.lr, hyper.beta1, hyper.beta2, hyper.eps,
                                               1.0 if dtype == "bf16" else 0.0])
                out[f"{key}.p"], out[f"{key}.m"], out[f"{key}.v"] = p, m, v
                out[f"{key}.g16"] = g16.view(np.uint16)
                out[f"{key}.rp"], out[f"{key}.rm"], out[f"{key}.rv"] = rp, rm, rv
                out[f"{key}.rp16"] = p16
                case += 1
    out["n_cases"] = np.array([case])
    # Non-finite rejection (lockfree.py:133-134): inputs returned untouched.
    p = np.ones(5, np.float32)
    g = np.array([1, 2, np.nan, 4, 5], np.float32)
    rp, _, _, ok = lockfree.apply_update(p, np.zeros(5, np.float32), np.zeros(5, np.float32), g,
                                         lockfree.AdamHyper(), 1)
    out["reject.ok"] = np.array([ok])
    # MasterState sequence with a rejected update in layer 1 (steps rollback).
    rng = np.random.default_rng(123)
    params = [rng.normal(0, 0.02, s).astype(np.float32) for s in (300, 1000, 77)]
    ms = lockfree.MasterState(params)
    grads = []
    for it in range(4):
        for layer in reversed(range(3)):
            gg = rng.normal(0, 1e-2, params[layer].shape).astype(np.float16)
            if it == 2 and layer == 1:
                gg[17] = np.float16(np.inf)
            grads.append(gg)
            ms.update_layer(layer, gg.astype(np.float32), lockfree.AdamHyper())
    for layer in range(3):
        out[f"ms.init{layer}"] = params[layer]
        out[f"ms.p{layer}"], out[f"ms.m{layer}"], out[f"ms.v{layer}"] = ms.p32[layer], ms.m32[layer], ms.v32[layer]
    out["ms.steps"] = np.array(ms.steps)
    out["ms.grads"] = np.concatenate([g.view(np.uint16) for g in grads])
    # ParamBuffer accumulate / take / publish (fp16, lockfree.py:210-263).
    buf = lockfree.ParamBuffer([np.zeros(513, np.float32), np.zeros(64, np.float32)])
    msgs = []
    for it in range(5):
        gg = (rng.normal(0, 3.0, 513) * (10.0 ** rng.integers(-3, 3, 513))).astype(np.float16)
        msgs.append(gg)
        buf.accumulate(lockfree.GradMessage(0, gg, it))
    out["pb.msgs"] = np.stack([g.view(np.uint16) for g in msgs])
    out["pb.g16"] = buf.g16[0].view(np.uint16).copy()
    g32, count, newest = buf.take(0)
    out["pb.take"] = g32
    out["pb.take_meta"] = np.array([count, newest])
    pub = rng.normal(0, 100.0, 513).astype(np.float32) * np.float32(1000.0)
    ver = buf.publish(0, pub, applied_iter=4, clear=False)
    out["pb.pub_in"] = pub
    out["pb.pub_out"] = buf.read(0)[1].view(np.uint16).copy()
    out["pb.pub_meta"] = np.array([ver, buf.read(0)[2]])
    np.savez_compressed(GOLDEN / "adam_golden.npz", **out)


def pagetable_random():
    spec = footprint.TensorSpec
    seeds = {}
    for seed in range(40):
        sd, log = pt_ops.replay(pagemem, spec, (AllocationError, MoveError), seed)
        seeds[str(seed)] = {"state": sd, "log": log}
    with gzip.open(GOLDEN / "pagetable_random.json.gz", "wt") as f:
        json.dump(seeds, f)


def pagetable_configs():
    from paper_2303_02868_b200 import workloads as W
    configs = {}
    for name in ("c1", "c2", "c3", "c4", "c5"):
        for page in ([W.config_page_bytes(name)] if name != "c5" else [MIB, 4 * MIB, 16 * MIB, 64 * MIB]):
            specs = [footprint.TensorSpec(s.name, s.kind, s.bytes, s.layer_index)
                     for s in W.config_specs(name)]
            pages_needed = sum(-(-s.bytes // page) for s in specs)
            mgr = pagemem.PageManager([("GPU", pages_needed * page, page)])
            for s in specs:
                mgr.allocate(s, "GPU")
            sd = mgr.state_dict()
            configs[f"{name}@{page}"] = {
                "pools": sd["pools"],
                "tensors": [[t["tensor_id"], t["bytes"], t["page_list"]] for t in sd["tensors"]],
                "pages": [[p["page_id"], [[o["tensor_id"], o["bytes"]] for o in p["occupants"]]]
                          for p in sd["pages"]],
            }
            print(name, page, len(sd["pages"]), "pages")
    with gzip.open(GOLDEN / "pagetable_configs.json.gz", "wt") as f:
        json.dump(configs, f)


def inventories():
    """param16 lists of the reference's tensor_inventory (hiermem/footprint.py:
    184-219) for the GPT configs of BASELINE.json (C1, C2, C3, C5): the
    fixture tests/test_workloads.py pins workloads.config_specs against."""
    shapes = {"c1": (1024, 768, 3072, 12, 12), "c2": (2048, 2048, 8192, 24, 16),
              "c3": (2048, 5120, 20480, 40, 40), "c5": (2048, 12288, 49152, 1, 96)}
    out = {}
    for name, (seq, d, f, layers, heads) in shapes.items():
        cfg = footprint.TransformerConfig(1, seq, d, f, layers, heads)
        out[name] = [[s.name, s.kind, s.bytes, s.layer_index] for s in footprint.tensor_inventory(cfg)
                     if s.kind == "param16"]
    with open(GOLDEN / "inventory_param16.json", "w") as fh:
        json.dump(out, fh)


def tracer_inventory():
    """Every tensor name the reference's build_trace needs a TimingModel table
    entry for (hiermem/tracer.py:102-107, 138-170: all but optim32), for the
    shape tests/test_gpu_tracing.py traces (seq 128, d 256, ffn 1024, 4 heads,
    2 layers)."""
    cfg = footprint.TransformerConfig(1, 128, 256, 1024, 2, 4)
    names = [s.name for s in footprint.tensor_inventory(cfg) if s.kind != "optim32"]
    with open(GOLDEN / "tracer_inventory.json", "w") as fh:
        json.dump({"shape": [1, 128, 256, 1024, 2, 4], "names": names}, fh)


def toy_sync():
    cfg = lockfree.ToyTrainConfig(num_layers=3, dim=16, batch_size=32, seed=5, noise_std=1.0)
    ref = lockfree.reference_train(cfg, 25)
    sync = lockfree.run_sync(cfg, lockfree.DelayModel.preset("zero"), 25)
    assert list(sync.loss_curve) == ref
    with open(GOLDEN / "toy_sync.json", "w") as f:
        json.dump({"cfg": {"num_layers": 3, "dim": 16, "batch_size": 32, "seed": 5, "noise_std": 1.0},
                   "iterations": 25, "loss_curve": ref, "val_loss": sync.val_loss}, f)


def schedules():
    """Algorithm-1 schedules of the reference (scheduler.schedule, phase 2) and
    their simulate() replay on the measured B200 profile (presets/b200-server.json),
    for the executor (paper_2303_02868_b200/executor.py) to run with real bytes."""
    import os
    os.environ["HIERMEM_PRESET_DIR"] = str(ROOT / "presets")
    from hiermem import presets
    from hiermem.scheduler import LayerModel, ShardingModel, peak_memory, schedule
    from hiermem.simengine import simulate
    from hiermem.tracer import TimingModel, build_trace
    prof = presets.hardware_preset("b200-server")
    out = {}
    cases = [("tiny-2layer", "tiny-2layer", int(0.012 * 2**30), None),
             ("gpt3-1.7b", "gpt3-1.7b", 8 * 2**30, None)]
    measured = ROOT / "presets" / "b200-timing-gpt3-1.7b.json"
    if measured.exists():   # tracer-measured B200 op times (tools/calibrate_timing.py)
        cases.append(("gpt3-1.7b-measured", "gpt3-1.7b", 8 * 2**30, measured))
    for key, name, budget, timing_file in cases:
        cfg = presets.model_preset(name)
        inv = footprint.tensor_inventory(cfg)
        if timing_file is not None:
            raw = json.loads(timing_file.read_text())
            timing = TimingModel.from_dict({"kind": raw["kind"], "table": raw["table"]})
        else:
            timing = TimingModel(gpu_sec_per_byte=1 / prof.gpu_bytes_per_s,
                                 cpu_sec_per_byte=1 / prof.cpu_bytes_per_s)
        traces = build_trace(inv, timing)
        lm = LayerModel.from_inventory(inv, 4 * MIB, cfg.batch_size)
        sched = schedule(lm, traces, budget, ShardingModel(1, 0))
        sim = simulate(sched, traces, prof)
        slot_s = [0.0] * sched.num_slots
        for e in sim.timeline:
            if e.operation == "compute":          # task id "it0.compute.s{slot}.l{layer}"
                slot = int(e.task_id.split(".s")[1].split(".")[0])
                slot_s[slot] = e.end_s - e.start_s
        d = sched.to_dict()
        d["model"].pop("tensors")  # the executor only needs the page numbering
        out[key] = {"schedule": d, "peak_bytes": peak_memory(sched, traces),
                    "timing": "measured B200 table" if timing_file else "proportional (bytes / B200 rates)",
                     "simulated": {"makespan_s": sim.makespan_s, "busy_s": sim.busy_s,
                                   "gpu_idle_fraction": sim.gpu_idle_fraction,
                                   "compute_s_by_slot": slot_s,
                                   "timeline_compute": [[e.task_id, e.start_s, e.end_s]
                                                        for e in sim.timeline if e.operation == "compute"]},
                     "hardware": prof.to_dict()}
        print(key, len(sched.tasks), "tasks, simulated makespan", sim.makespan_s)
    with gzip.open(GOLDEN / "schedules.json.gz", "wt") as f:
        json.dump(out, f)


if __name__ == "__main__":
    GOLDEN.mkdir(parents=True, exist_ok=True)
    adam_cases()
    pagetable_random()
    pagetable_configs()
    inventories()
    tracer_inventory()
    toy_sync()
    schedules()
    print("golden fixtures written to", GOLDEN)
