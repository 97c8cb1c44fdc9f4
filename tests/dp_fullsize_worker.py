"""torchrun worker: the fused DP page step at the BASELINE C2 size (GPT-3
1.3B param set, 676 pages of 4 MiB) — the size bench.py measures — checked
on a seeded sample of pages.  A page's reduced gradient depends only on the
ranks' gradients of that page, and its update only on that and its layer's
step, so the sample is a size-independent check of the whole step:
  * the reduced gradient pages (owner): bit-exact vs the rank-order f32 sum
    rounded once;
  * the owner's p32/m32/v32 of the page: bit-exact vs the oracle Adam;
  * every rank's published 16-bit page: the cast of the oracle's p32.
DP_PIPE=1 runs the layer-group pipelined two-phase step; DP_PIPE=2 the
one-pass kernel over a double-buffered state (bench.py's N=2 default),
which never writes the reduced gradient back, so that check is skipped and
the state is read from each layer's current copy."""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import page_adam as O  # noqa: E402
from paper_2303_02868_b200 import lockfree as LF  # noqa: E402
from paper_2303_02868_b200 import workloads as W  # noqa: E402
from paper_2303_02868_b200.layout import PageLayout  # noqa: E402
from paper_2303_02868_b200.sharding import FusedShardedPageStep, symmetric_alloc  # noqa: E402


def grad_flat(total, seed, dev):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    return torch.empty(total, device=dev).normal_(0, 1e-2, generator=g).to(torch.bfloat16)


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", local)
    specs = W.config_specs("c2")
    numels = [s.bytes // 2 for s in specs]
    page = W.config_page_bytes("c2")
    lay = PageLayout(numels, page, world_size=world, rank=rank, bucket_pages=32)
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    params = [torch.empty(n, device=dev).normal_(0, 0.02, generator=gen) for n in numels]
    buf = LF.ParamBuffer(params, dtype="bf16", page_bytes=page, device=dev, layout=lay,
                         pool_alloc=symmetric_alloc)
    mode = os.environ.get("DP_PIPE", "0")
    ms = LF.MasterState(params, page_bytes=page, device=dev, layout=lay, double_buffered=mode == "2")
    dp = FusedShardedPageStep(buf, ms)
    total = sum(numels)
    buf.accumulate_flat(grad_flat(total, 100 + rank, dev), 0)
    gsel = buf._gsel[0]
    hyper = LF.AdamHyper(lr=1e-3)
    if mode == "1":
        dp.step_pipelined(hyper, 8, reduce_ctas=128)
    else:
        dp.step(hyper)
    torch.cuda.synchronize()
    # sample: (layer, segment) pairs over the whole model, seeded
    rng = np.random.default_rng(7)
    starts = np.cumsum([0] + numels[:-1])
    picks = []
    for _ in range(24):
        l = int(rng.integers(len(numels)))
        segs = lay.segments[l]
        picks.append((l, segs[int(rng.integers(len(segs)))]))
    all_g = [grad_flat(total, 100 + r, dev) for r in range(world)]
    failures = []
    p16 = buf.p16_pool[buf._psel[0]]
    for l, s in picks:
        a = int(starts[l]) + s.pos
        acc = np.zeros(s.n, np.float32)
        for r in range(world):
            acc = np.add(acc, O.from16(all_g[r][a:a + s.n].view(torch.int16).cpu().numpy().view(np.uint16), "bf16"))
        red16 = O.to16(acc, "bf16")
        p0 = params[l][s.pos:s.pos + s.n].cpu().numpy()
        rp, rm, rv, ok = O.adam_update(p0, np.zeros(s.n, np.float32), np.zeros(s.n, np.float32),
                                       O.from16(red16, "bf16"), 1e-3, 0.9, 0.999, 1e-8, 1)
        off16 = lay.slot16(s.page) * lay.E + s.off
        if not np.array_equal(p16[off16:off16 + s.n].view(torch.int16).cpu().numpy().view(np.uint16),
                              O.to16(rp, "bf16").view(np.uint16)):
            failures.append(f"layer{l} page{s.page}: published page differs")
        if lay.owned(s) and mode != "2":
            got = buf.g16_pool[gsel][off16:off16 + s.n].view(torch.int16).cpu().numpy().view(np.uint16)
            if not np.array_equal(got, red16.view(np.uint16)):
                failures.append(f"layer{l} page{s.page}: reduced gradient differs")
        if lay.owned(s):
            so = lay.slot_state(s.page) * lay.E + s.off
            for name, pool, want in (("p32", ms._current(ms.p32_pool, l), rp), ("m32", ms._current(ms.m32_pool, l), rm),
                                     ("v32", ms._current(ms.v32_pool, l), rv)):
                if not np.array_equal(pool[so:so + s.n].cpu().numpy().view(np.uint32), want.view(np.uint32)):
                    failures.append(f"layer{l} page{s.page}: owned {name} differs")
    if ms.steps != [1] * len(numels):
        failures.append(f"steps after one applied step: {sorted(set(ms.steps))}")
    ok = torch.tensor([0 if failures else 1], device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if failures:
        print(f"rank {rank} FAIL:", *failures[:10], sep="\n  ")
    else:
        print(f"rank {rank}: {len(picks)} sampled segments bit-exact", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok.item() == 1 else 1)


if __name__ == "__main__":
    main()
