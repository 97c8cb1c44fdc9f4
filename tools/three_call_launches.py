"""GPU-side anatomy of the reference's per-layer loop through the drop-in
(take -> update_layer -> publish, torch tensors, C2, + K3): one step timed
with CUDA events, then (under ncu with --profile-from-start off) exactly one
step's launch list, so the sum of kernel durations can be set beside the
step time — the difference is launch gaps.

    python tools/three_call_launches.py                    # timing line
    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
        --log-file gpurun_out/tc_launches.csv python tools/three_call_launches.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2303_02868_b200 import lockfree as LF  # noqa: E402
from paper_2303_02868_b200 import workloads as W  # noqa: E402
from paper_2303_02868_b200.layout import PageLayout  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    specs = W.config_specs("c2")
    numels = [s.bytes // 2 for s in specs]
    lay = PageLayout(numels, W.config_page_bytes("c2"))
    params = [torch.zeros(n, device=dev) for n in numels]
    buf = LF.ParamBuffer(params, dtype="bf16", layout=lay, device=dev)
    ms = LF.MasterState(params, layout=lay, device=dev)
    del params
    g = torch.randn(sum(numels), device=dev).mul_(1e-2).to(torch.bfloat16)
    hyper = LF.AdamHyper(lr=1e-3)

    def step():
        buf.accumulate_flat(g, 0)
        for l in reversed(range(len(numels))):
            gr, _c, newest = buf.take(l)
            ms.update_layer(l, gr, hyper)
            buf.publish(l, ms.p32[l], applied_iter=newest, clear=False)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    times = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    import time
    t0 = time.perf_counter()
    step()
    host_ms = (time.perf_counter() - t0) * 1e3     # host time to enqueue one step
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(json.dumps({"probe": "three_call", "layers": len(numels), "step_ms": sorted(times)[len(times) // 2],
                      "host_enqueue_ms": host_ms}), flush=True)


if __name__ == "__main__":
    main()
