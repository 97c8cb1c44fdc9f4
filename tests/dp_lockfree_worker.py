"""torchrun worker: the lock-free delayed update (Algorithm 2, actors.
LockFreeRunner) with the data-parallel page step as its updating actor and
the fp32 state on the sharded pinned-host tier.  Every iteration each rank
offers the same seeded gradient, so whatever the staleness, every iteration's
gradient must be applied exactly once: after n iterations the sharded
masters equal the oracle applying the rank-order f32 sum n times, and every
rank's published pages equal its cast."""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import page_adam as O  # noqa: E402
from paper_2303_02868_b200 import lockfree as LF  # noqa: E402
from paper_2303_02868_b200.actors import LockFreeRunner  # noqa: E402
from paper_2303_02868_b200.layout import PageLayout  # noqa: E402
from paper_2303_02868_b200.sharding import FusedShardedPageStep, symmetric_alloc  # noqa: E402
from paper_2303_02868_b200.swap import HostMasterState  # noqa: E402

SIZES = [70001, 1, 5, 32768, 40000, 25003, 777, 12, 33333]
PAGE = 64 * 1024


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", local)
    lay = PageLayout(SIZES, PAGE, world_size=world, rank=rank, bucket_pages=2)
    rng = np.random.default_rng(3)
    params = [rng.normal(0, 0.02, n).astype(np.float32) for n in SIZES]
    tp = [torch.from_numpy(p) for p in params]
    buf = LF.ParamBuffer(tp, dtype="bf16", page_bytes=PAGE, device=dev, layout=lay, pool_alloc=symmetric_alloc)
    ms = HostMasterState(tp, page_bytes=PAGE, device=dev, layout=lay, group_pages=2, world_size=world, rank=rank)
    dp = FusedShardedPageStep(buf, ms)
    grads = [[O.to16(np.random.default_rng([r, l]).normal(0, 1e-2, n).astype(np.float32), "bf16")
              for l, n in enumerate(SIZES)] for r in range(world)]
    mine = torch.from_numpy(np.concatenate(grads[rank]).view(np.int16)).view(torch.bfloat16).to(dev)
    zero = torch.zeros((), device=dev)
    hyper = LF.AdamHyper(lr=1e-3)
    iters = 4
    runner = LockFreeRunner(buf, ms, hyper, delay=int(os.environ.get("DP_DELAY", "1")),
                            update=lambda b, m, h, stream: dp.step(h, stream=stream))
    rep = runner.run(iters, lambda params_, it: (zero, mine))
    torch.cuda.synchronize()
    failures = []
    om = O.OracleMasters(params)
    for l, n in enumerate(SIZES):
        acc = O.from16(grads[0][l], "bf16").copy()
        for r in range(1, world):
            acc = np.add(acc, O.from16(grads[r][l], "bf16"))
        red = O.from16(O.to16(acc, "bf16"), "bf16")
        for _ in range(iters):
            om.update_layer(l, red, lr=1e-3)
    if ms.steps != om.steps:
        failures.append(f"steps {ms.steps} != {om.steps}")
    p16 = buf.p16_pool[buf._psel[0]].view(torch.int16).cpu().numpy().view(np.uint16)
    for l in range(len(SIZES)):
        mp = ms.p32[l]
        mp = mp.numpy() if isinstance(mp, torch.Tensor) else mp
        want16 = O.to16(om.p32[l], "bf16").view(np.uint16)
        for s in lay.segments[l]:
            off = lay.slot16(s.page) * lay.E + s.off
            if not np.array_equal(p16[off:off + s.n], want16[s.pos:s.pos + s.n]):
                failures.append(f"layer{l} page{s.page}: published p16 differs")
            if lay.owned(s) and not np.array_equal(mp.reshape(-1)[s.pos:s.pos + s.n].view(np.uint32),
                                                   om.p32[l][s.pos:s.pos + s.n].view(np.uint32)):
                failures.append(f"layer{l} page{s.page}: owned p32 differs")
    if rep.max_staleness > 1:
        failures.append(f"staleness {rep.max_staleness} > 1")
    ok = torch.tensor([0 if failures else 1], device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if failures:
        print(f"rank {rank} FAIL:", *failures[:10], sep="\n  ")
    dist.destroy_process_group()
    sys.exit(0 if ok.item() == 1 else 1)


if __name__ == "__main__":
    main()
