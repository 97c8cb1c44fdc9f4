"""torchrun worker for tests/test_gpu_dp.py (one process per GPU, NCCL).

Every rank regenerates every rank's seeded gradients, so each can compute the
oracle independently: reduced gradient = rn16 sum over ranks (bit-exact at
N=2, where NCCL performs one bf16 add; within one bf16 ulp of the f32 sum
otherwise), then the oracle Adam on the CAPTURED post-reduce-scatter pages
must match the sharded masters bit for bit, and the all-gathered p16 pool
must equal the cast of the updated masters on every page.
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import page_adam as O  # noqa: E402
from paper_2303_02868_b200 import lockfree as LF  # noqa: E402
from paper_2303_02868_b200.layout import PageLayout  # noqa: E402
from paper_2303_02868_b200.sharding import (FusedShardedPageStep, ShardedPageStep,  # noqa: E402
                                            symmetric_alloc)

SIZES = [70001, 1, 5, 32768, 40000, 25003, 777, 65539, 12, 33333, 200000]
PAGE = 64 * 1024


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    K = int(os.environ.get("DP_BUCKET", "2"))
    dtype = os.environ.get("DP_DTYPE", "bf16")
    lay = PageLayout(SIZES, PAGE, world_size=world, rank=rank, bucket_pages=K)
    rng0 = np.random.default_rng(11)
    params = [rng0.normal(0, 0.02, n).astype(np.float32) for n in SIZES]
    dev = torch.device("cuda", local)
    mode = os.environ.get("DP_MODE", "nccl")
    buf = LF.ParamBuffer([torch.from_numpy(p) for p in params], dtype=dtype, page_bytes=PAGE,
                         device=dev, layout=lay, pool_alloc=None if mode == "nccl" else symmetric_alloc)
    host_tier = os.environ.get("DP_HOST", "0")
    if host_tier == "1":   # fp32 state in pinned host memory, owned pages only
        from paper_2303_02868_b200.swap import HostMasterState
        ms = HostMasterState([torch.from_numpy(p) for p in params], page_bytes=PAGE, device=dev, layout=lay,
                             group_pages=2, world_size=world, rank=rank)
    elif host_tier == "ssd":   # fp32 state in a per-rank file (owned pages only)
        import tempfile
        from paper_2303_02868_b200.ssd import SSDMasterState
        path = os.path.join(tempfile.gettempdir(), f"hm_dp_state_{os.getpid()}_{rank}.bin")
        ms = SSDMasterState([torch.from_numpy(p) for p in params], path, page_bytes=PAGE, device=dev,
                            layout=lay, group_pages=2, world_size=world, rank=rank)
    else:   # DP_ONEPASS=1: double-buffered state, the one-pass fused step
        ms = LF.MasterState([torch.from_numpy(p) for p in params], page_bytes=PAGE, device=dev, layout=lay,
                            double_buffered=os.environ.get("DP_ONEPASS", "0") == "1")
    onepass = getattr(ms, "_db", False)
    step = ShardedPageStep(buf, ms) if mode == "nccl" else \
        FusedShardedPageStep(buf, ms, mode=mode, push=os.environ.get("DP_PUSH", "0") == "1")
    from paper_2303_02868_b200 import _native as NL
    NL.check(NL.lib().hm_set_ag_publish(int(os.environ.get("DP_AG_PUBLISH", "0"))))
    NL.check(NL.lib().hm_set_dp_reduce_width(int(os.environ.get("DP_REDUCE_WIDTH", "0"))))
    if "DP_REDUCE_WIDE" in os.environ:
        NL.check(NL.lib().hm_set_dp_reduce_wide(int(os.environ["DP_REDUCE_WIDE"])))
    if mode == "nvls" and step is None:
        sys.exit(0)
    from paper_2303_02868_b200.sharding import PageCollectives
    coll = PageCollectives(lay)
    om = O.OracleMasters(params)
    clip = float(os.environ.get("DP_CLIP", "0"))   # global grad-norm clip over every rank's layers
    hyper = LF.AdamHyper(lr=1e-3, max_norm=clip)
    failures = []
    stats = {}
    if mode != "nccl":
        print(f"rank {rank}: fused mode {mode}, mc={getattr(step, 'mc_g', 0)}", flush=True)
    for it in range(3):
        per_rank = []
        for r in range(world):
            rr = np.random.default_rng([it, r])
            gs = []
            for l, n in enumerate(SIZES):
                g = rr.normal(0, 1e-2, n).astype(np.float32)
                if it == 1 and l == 6 and r == world - 1:
                    g[3] = np.inf   # one rank's non-finite gradient rejects the layer everywhere
                if it == 2 and l == 3 and r in (0, 1):
                    # finite on every rank, but the reduced sum overflows the
                    # 16-bit type: the rounded sum is inf and the layer is rejected
                    g[7] = 60000.0 if dtype == "fp16" else 3.0e38
                gs.append(O.to16(g, dtype))
            per_rank.append(gs)
        mine = per_rank[rank]
        flat = np.concatenate(mine)
        t = torch.from_numpy(flat.view(np.int16) if dtype == "bf16" else flat)
        if dtype == "bf16":
            t = t.view(torch.bfloat16)
        groups = int(os.environ.get("DP_GROUPS", "1"))
        ingest = os.environ.get("DP_INGEST", "0") == "1"
        if ingest:   # from pinned host memory, group by group; the step starts early
            ready = LF.ingest(buf, t.pin_memory(), it, groups=groups)
        else:
            buf.accumulate_flat(t.to(dev), it)
        gsel = buf._gsel[0]
        if ingest and onepass:   # the one-pass kernel group by group as the gradient lands
            step.step(hyper, ready=ready)
        elif ingest:   # ... and this rank's owned published pages come back to the host
            out_host = torch.empty(sum(SIZES), dtype=buf._t16).pin_memory()
            step.step_pipelined(hyper, groups, ready=ready, results_to=out_host)
        elif groups > 1 and mode != "nccl":
            step.step_pipelined(hyper, groups, reduce_ctas=int(os.environ.get("DP_REDUCE_CTAS", "0")),
                                update_ctas=int(os.environ.get("DP_UPDATE_CTAS", "0")),
                                reduce_sms=int(os.environ.get("DP_REDUCE_SMS", "0")))
        elif onepass:
            step.step(hyper, reduce_width=int(os.environ.get("DP_REDUCE_WIDTH", "0")) or -1)
        else:
            step.step(hyper)
        if ingest and not onepass:
            torch.cuda.synchronize()
            pub = buf.p16_pool[buf._psel[0]].view(torch.int16).cpu()
            host16 = out_host.view(torch.int16)
            base = 0
            for l, n in enumerate(SIZES):
                for s_ in lay.segments[l]:
                    if lay.owned(s_):
                        off = lay.slot16(s_.page) * lay.E + s_.off
                        if not torch.equal(host16[base + s_.pos: base + s_.pos + s_.n], pub[off:off + s_.n]):
                            failures.append(f"it{it} layer{l}: results_to differs from the published page")
                base += n
        # every owner's reduced (post reduce-scatter) pages, gathered so each
        # rank can run the oracle on the exact captured gradient of ALL pages
        gathered = buf.g16_pool[gsel].clone()
        coll.all_gather(gathered)
        torch.cuda.synchronize()
        gpool = gathered.view(torch.int16).cpu().numpy().view(np.uint16 if dtype == "bf16" else np.float16)
        caps = []
        for l, n in enumerate(SIZES):
            if mode == "nccl":   # NCCL ring: each hop adds into a 16-bit buffer
                red = per_rank[0][l]
                for r in range(1, world):
                    red = O.accumulate16(red, per_rank[r][l], dtype)
            else:                # fused kernel: f32 sum in rank order, rounded once
                acc = O.from16(per_rank[0][l], dtype).copy()
                for r in range(1, world):
                    acc = np.add(acc, O.from16(per_rank[r][l], dtype))
                red = O.to16(acc, dtype)
            captured = red.copy()
            for s in lay.segments[l]:
                if onepass:   # the one-pass step never writes the reduced gradient back
                    continue
                off = lay.slot16(s.page) * lay.E + s.off
                got = gpool[off:off + s.n]
                want = red[s.pos:s.pos + s.n]
                if mode == "p2p" or (mode == "nccl" and world == 2):   # one rounding: exact
                    if not np.array_equal(got.view(np.uint16), want.view(np.uint16)):
                        failures.append(f"it{it} layer{l}: reduced grad differs from oracle sum")
                else:   # NCCL ring at N>2 / NVLS in-switch reduction: 16-bit rounding bound
                    # Each of the N-1 additions may round by half an ulp of a partial
                    # sum, and every partial sum is bounded by sum_r |g_r|.
                    # compared with the EXACT (f64) sum: N roundings of at most half an
                    # ulp of a partial sum bounded by sum_r |g_r|
                    gf, wf = O.from16(got, dtype), O.from16(want, dtype)
                    fin = np.isfinite(wf)
                    u = 2.0 ** -8 if dtype == "bf16" else 2.0 ** -11
                    if fin.any():
                        absum = np.zeros(s.n, np.float64)
                        exact = np.zeros(s.n, np.float64)
                        for r in range(world):
                            x = O.from16(per_rank[r][l][s.pos:s.pos + s.n], dtype).astype(np.float64)
                            absum += np.abs(x)
                            exact += x
                        bound = world * u * absum[fin] + 1e-38
                        err = np.abs(gf[fin].astype(np.float64) - exact[fin])
                        worst = float((err / bound).max())
                        stats["max_err_over_bound"] = max(stats.get("max_err_over_bound", 0.0), worst)
                        stats["mismatch"] = stats.get("mismatch", 0) + int((gf[fin] != wf[fin]).sum())
                        stats["n"] = stats.get("n", 0) + int(fin.sum())
                        if worst > 1.0:
                            failures.append(f"it{it} layer{l}: reduced grad error {worst:.3g}x the rounding bound")
                    if np.isfinite(gf).sum() != fin.sum():
                        failures.append(f"it{it} layer{l}: non-finite pattern differs")
                captured[s.pos:s.pos + s.n] = got
            caps.append(captured)
        # oracle Adam on the captured reduced gradient (clip: the global norm
        # of the layers that will be applied, the device's coefficient rule)
        gscale = None
        if clip > 0:
            tot = 0.0
            for c in caps:
                g = O.from16(c, dtype).astype(np.float64)
                if np.isfinite(g).all():
                    tot += float(np.sum(g * g))
            norm = np.sqrt(tot)
            coef = clip / (norm + 1e-6) if norm > clip else 1.0
            gscale = np.float32(np.float32(1.0) * np.float32(coef))
        for l, c in enumerate(caps):
            g = O.from16(c, dtype)
            if gscale is not None:
                g = (g * gscale).astype(np.float32)
            om.update_layer(l, g, lr=1e-3)
    steps = ms.steps
    if steps != om.steps:
        failures.append(f"steps {steps} != oracle {om.steps}")
    p16 = buf.p16_pool[buf._psel[0]].view(torch.int16).cpu().numpy().view(np.uint16)
    for l, n in enumerate(SIZES):
        mp = ms.p32[l].cpu().numpy() if isinstance(ms.p32[l], torch.Tensor) else ms.p32[l]
        want16 = O.to16(om.p32[l], dtype).view(np.uint16)
        for s in lay.segments[l]:
            off = lay.slot16(s.page) * lay.E + s.off
            if clip > 0:   # the device's f32-partial norm may move the coefficient by a last bit
                d16 = np.abs(p16[off:off + s.n].astype(np.int32) - want16[s.pos:s.pos + s.n].astype(np.int32))
                if d16.max(initial=0) > 1:
                    failures.append(f"layer{l} page{s.page}: all-gathered p16 off by {d16.max()} ulp")
                # 1e-6 relative, or 1e-6 of the step size lr near zero, where the
                # masters are a difference of nearly equal terms (after three
                # updates of ~lr some elements sit at ~1e-7)
                if lay.owned(s) and not np.allclose(mp[s.pos:s.pos + s.n], om.p32[l][s.pos:s.pos + s.n],
                                                    rtol=1e-6, atol=1e-6 * 1e-3):
                    a, b = mp[s.pos:s.pos + s.n], om.p32[l][s.pos:s.pos + s.n]
                    rel = np.abs(a - b) / np.maximum(np.abs(b), 1e-30)
                    i = int(np.argmax(rel))
                    failures.append(f"layer{l} page{s.page}: owned p32 beyond 1e-6 relative "
                                    f"(max {rel[i]:.3g} at {i}: {a[i]!r} vs {b[i]!r}; "
                                    f"{int((rel > 1e-6).sum())} of {s.n})")
                continue
            if not np.array_equal(p16[off:off + s.n], want16[s.pos:s.pos + s.n]):
                failures.append(f"layer{l} page{s.page}: all-gathered p16 differs")
            if lay.owned(s) and not np.array_equal(mp[s.pos:s.pos + s.n].view(np.uint32),
                                                   om.p32[l][s.pos:s.pos + s.n].view(np.uint32)):
                failures.append(f"layer{l} page{s.page}: owned p32 differs")
    if host_tier == "ssd":
        ms.close()
        os.unlink(path)
    ok = torch.tensor([0 if failures else 1], device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if stats:
        print(f"rank {rank}: reduced-gradient deviation vs f32-sum oracle: {stats}", flush=True)
    if failures:
        print(f"rank {rank} FAIL:", *failures[:10], sep="\n  ")
    dist.destroy_process_group()
    sys.exit(0 if ok.item() == 1 else 1)


if __name__ == "__main__":
    main()
