"""Data-parallel page sharding host logic on CPU (no GPU):
* ShardingModel equals the reference's (hiermem/scheduler.py:59-76);
* the bucketed rank-major slot map is a bijection whose rank-r block of
  every bucket holds exactly the pages owner(p) = p % N assigns to r;
* PageCollectives' in-place bucketed reduce-scatter / all-gather, run with
  world_size 2, 4 and 8 over gloo, hands every owner the sum of its pages and
  reassembles the pool (the same calls run over NCCL on the GPU box);
* the push form's routing table delivers every non-owned element to its
  owner's receive pool where the owner's update reads it (world 2/4/8).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2303_02868_b200.errors import ConfigError
from paper_2303_02868_b200.layout import PageLayout
from paper_2303_02868_b200.sharding import PageCollectives, ShardingModel

SIZES = [70001, 1, 5, 32768, 40000, 25003, 777, 65539, 12, 33333, 200000]
PAGE = 64 * 1024


def test_sharding_model_matches_reference():
    sm = ShardingModel(4, 1)
    assert [sm.owner(p) for p in range(9)] == [p % 4 for p in range(9)]
    assert sm.owns(5) and not sm.owns(6)
    for bad in ((0, 0), (2, 2), (2, -1)):
        with pytest.raises(ConfigError):
            ShardingModel(*bad)


@pytest.mark.parametrize("world,K", [(1, None), (2, None), (2, 1), (4, 2), (8, 3)])
def test_slot_map_is_rank_major_bijection(world, K):
    lays = [PageLayout(SIZES, PAGE, world_size=world, rank=r, bucket_pages=K) for r in range(world)]
    lay = lays[0]
    slots = [lay.slot16(p) for p in range(lay.P)]
    assert sorted(slots) == list(range(lay.P))
    for p in range(lay.P):
        b = lay.bucket_of(p)
        lo, hi = lay.bucket_slots(b)
        r = p % world
        assert lo + r * lay.K <= lay.slot16(p) < lo + (r + 1) * lay.K
        assert lay.slot_state(p) == p // world
    # every element of every tensor is updated by exactly one rank
    total = sum(l.owned_numel() for l in lays)
    assert total == sum(SIZES)
    for r, l in enumerate(lays):
        c = l.adam_chunks(range(len(SIZES)))
        assert c["n"].sum() == l.owned_numel()
        assert (c["s_off"] + c["n"] <= l.elems_state).all()
        per_bucket = sum(l.adam_chunks(range(len(SIZES)), bucket=b)["n"].sum() for b in range(l.num_buckets))
        assert per_bucket == l.owned_numel()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, K, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lay = PageLayout(SIZES, PAGE, world_size=world, rank=rank, bucket_pages=K)
        coll = PageCollectives(lay)
        E = lay.E
        # gradient pool: value = f(page, elem, rank) at the page's slot
        pool = torch.zeros(lay.elems16, dtype=torch.float32)
        for p in range(lay.P):
            s = lay.slot16(p)
            pool[s * E:(s + 1) * E] = torch.arange(E, dtype=torch.float32) * 0.5 + p * 3 + rank
        coll.reduce_scatter(pool)
        ok = True
        for p in range(lay.P):
            if p % world != rank:
                continue
            s = lay.slot16(p)
            want = sum(torch.arange(E, dtype=torch.float32) * 0.5 + p * 3 + r for r in range(world))
            ok &= bool(torch.equal(pool[s * E:(s + 1) * E], want))
        # all-gather: each owner writes p*7 into its owned pages, everyone sees all
        out = torch.full((lay.elems16,), -1.0)
        for p in range(lay.P):
            if p % world == rank:
                s = lay.slot16(p)
                out[s * E:(s + 1) * E] = p * 7.0
        coll.all_gather(out)
        for p in range(lay.P):
            s = lay.slot16(p)
            ok &= bool((out[s * E:(s + 1) * E] == p * 7.0).all())
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,K", [(2, None), (2, 1), (2, 3), (4, None), (4, 2), (8, None), (8, 1)])
def test_bucketed_rs_ag_gloo(world, K):
    """The reference sweeps world in {1, 2, 4, 8} (tests/test_acceptance.py:188);
    world 8 is the north star's one-box DP width: same bucket layout,
    rendezvous and in-place collective plumbing as the NCCL run."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}


def test_modeled_gather_matches_reference_formula():
    """hiermem/simengine.py:255-257: one lat + page*(N-1)/N/bw task per page."""
    from paper_2303_02868_b200.sharding import modeled_gather_s
    page, pages, lat, bw = 4 << 20, 676, 10e-6, 770e9
    for n in (1, 2, 4, 8):
        want = sum(lat + page * ((n - 1) / n) / bw for _ in range(pages))
        assert abs(modeled_gather_s(page, pages, n, bw, lat) - want) < 1e-12
    with pytest.raises(ConfigError):
        modeled_gather_s(page, pages, 0, bw, lat)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_push_routes_every_non_owned_element_to_its_owner(world):
    """The push form's routing table (layout.push_chunks): simulated with
    numpy, every rank's non-owned gradient lands in its owner's receive
    pool at the slot of the sender and the state offset the owner's update
    reads; together with the owned pages this covers every element once."""
    lays = [PageLayout(SIZES, PAGE, world_size=world, rank=r, bucket_pages=2) for r in range(world)]
    es = lays[0].elems_state
    rng = np.random.default_rng(world)
    pools = [rng.integers(0, 2 ** 16, lays[0].elems16, dtype=np.uint16) for _ in range(world)]
    recv = [np.zeros(world * es, np.uint16) for _ in range(world)]
    for r, lay in enumerate(lays):
        pc = lay.push_chunks()
        assert (pc["slot"] != r).all() and (pc["n"] <= 4096).all()
        for c in pc:
            dst = r * es + int(c["dst_off"])
            recv[int(c["slot"])][dst:dst + int(c["n"])] = pools[r][int(c["src_off"]):int(c["src_off"]) + int(c["n"])]
    covered = 0
    for r, lay in enumerate(lays):
        ac = lay.adam_chunks(range(len(SIZES)), "pool", owned_only=True)
        for c in ac:
            g, so, n = int(c["g_off"]), int(c["s_off"]), int(c["n"])
            for q in range(world):
                share = pools[q][g:g + n] if q == r else recv[r][q * es + so:q * es + so + n]
                assert np.array_equal(share, pools[q][g:g + n]), (r, q)
            covered += n
    assert covered == sum(SIZES)
