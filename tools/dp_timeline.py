"""Per-layer-group timeline of the pipelined DP step (torchrun, C2): when
each group's reduce-scatter and update+all-gather start and end on rank 0,
relative to the step start — to see how much of the reduce of group k+1
actually overlaps the update of group k.

    torchrun --nproc-per-node 2 tools/dp_timeline.py [--groups 8] [--reduce-ctas 128]
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2303_02868_b200 import lockfree as LF  # noqa: E402
from paper_2303_02868_b200 import workloads as W  # noqa: E402
from paper_2303_02868_b200.dp_bench import owned_grad_flat  # noqa: E402
from paper_2303_02868_b200.layout import PageLayout  # noqa: E402
from paper_2303_02868_b200.sharding import FusedShardedPageStep, symmetric_alloc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", type=int, default=8)
    ap.add_argument("--reduce-ctas", type=int, default=128)
    ap.add_argument("--update-ctas", type=int, default=0)
    ap.add_argument("--reduce-sms", type=int, default=0)
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", local)
    specs = W.config_specs("c2")
    numels = [s.bytes // 2 for s in specs]
    lay = PageLayout(numels, 4 << 20, world_size=world, rank=rank, bucket_pages=32)
    params = [torch.zeros(n, device=dev) for n in numels]
    buf = LF.ParamBuffer(params, dtype="bf16", layout=lay, device=dev, pool_alloc=symmetric_alloc)
    ms = LF.MasterState(params, layout=lay, device=dev)
    del params
    dp = FusedShardedPageStep(buf, ms)
    buf.accumulate_flat(owned_grad_flat(lay, "bf16", dev, 7 + rank), 0)
    hyper = LF.AdamHyper(lr=1e-3, inv_scale=1.0 / world)
    kw = dict(reduce_ctas=args.reduce_ctas, update_ctas=args.update_ctas, reduce_sms=args.reduce_sms)
    for _ in range(5):
        for l in range(len(numels)):
            buf._pending[l] = 1
        dp.step_pipelined(hyper, args.groups, **kw)
    for l in range(len(numels)):
        buf._pending[l] = 1
    tm = {}
    dp.step_pipelined(hyper, args.groups, timings=tm, **kw)
    torch.cuda.synchronize()
    if rank == 0:
        t0 = tm["_marks"]["start"]
        print(f"groups={args.groups} reduce_ctas={args.reduce_ctas} update_ctas={args.update_ctas} "
              f"reduce_sms={args.reduce_sms} step={t0.elapsed_time(tm['_marks']['ag']):.3f} ms")
        for k, (r0, r1, u0, u1) in enumerate(tm["_groups"]):
            print(f"  group {k}: reduce {t0.elapsed_time(r0):7.3f} -> {t0.elapsed_time(r1):7.3f}"
                  f"   update {t0.elapsed_time(u0):7.3f} -> {t0.elapsed_time(u1):7.3f}")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
