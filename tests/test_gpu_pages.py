"""K1 pack/unpack and K8 page motion with real bytes (pages.DevicePageManager):
a randomized allocate / write / page_move / tensor_merge / release script in
which every live tensor must read back bit-identical after every operation,
plus the reference's own move/merge cases with data, and equality of the
page table with the metadata-only manager on the same script."""
import random

import numpy as np
import pytest
import torch

from oracle import page_adam as O
from paper_2303_02868_b200 import TensorSpec
from paper_2303_02868_b200.errors import AllocationError, MoveError
from paper_2303_02868_b200.pagemem import PageManager
from paper_2303_02868_b200.pages import DevicePageManager

pytestmark = pytest.mark.gpu
MIB = 2 ** 20
PAGE = 64 * 1024


def _data(rng, nbytes, kind):
    if kind == "optim32":
        return rng.normal(0, 1, nbytes // 4).astype(np.float32)
    return rng.normal(0, 1, nbytes // 2).astype(np.float16)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_script_preserves_bytes(cuda, seed):
    rng = random.Random(seed)
    nrng = np.random.default_rng(seed)
    specs = [("GPU", 64 * PAGE, PAGE), ("CPU", 64 * PAGE, PAGE)]
    dm = DevicePageManager(specs)
    meta = PageManager(specs)
    live: dict[int, np.ndarray] = {}
    for i in range(300):
        op = rng.random()
        if op < 0.45:
            kind = rng.choice(["param16", "optim32"])
            nbytes = rng.choice([4, 1000, 4096, PAGE, PAGE + 8, 3 * PAGE - 12, 5 * PAGE])
            nbytes -= nbytes % 4
            spec = TensorSpec(f"t{i}", kind, nbytes, 0)
            tier = rng.choice(["GPU", "CPU"])
            try:
                t = dm.allocate(spec, tier)
            except AllocationError:
                with pytest.raises(AllocationError):
                    meta.allocate(spec, tier)
                continue
            meta.allocate(spec, tier)
            data = _data(nrng, nbytes, kind)
            dm.write(t.tensor_id, data)
            live[t.tensor_id] = data
        elif op < 0.6 and live:
            tid = rng.choice(sorted(live))
            dm.release(tid)
            meta.release(tid)
            del live[tid]
        elif op < 0.85 and live:
            tid = rng.choice(sorted(live))
            pid = rng.choice(dm.tensors[tid].page_list)
            tgt = rng.choice(["GPU", "CPU"])
            try:
                dm.page_move(pid, tgt)
            except MoveError:
                with pytest.raises(MoveError):
                    meta.page_move(pid, tgt)
                continue
            meta.page_move(pid, tgt)
        elif live:
            tid = rng.choice(sorted(live))
            try:
                r = dm.tensor_merge(tid)
            except (AllocationError, MoveError) as e:
                with pytest.raises(type(e)):
                    meta.tensor_merge(tid)
                continue
            assert r == meta.tensor_merge(tid)
        if i % 10 == 0 or op >= 0.6:
            for tid, data in live.items():
                got = dm.read(tid).view(torch.uint8).cpu().numpy()
                assert np.array_equal(got, data.view(np.uint8)), f"tensor {tid} corrupted at op {i}"
    assert dm.state_dict() == meta.state_dict()


def test_merge_chain_with_data(cuda):
    # reference tests/test_pagemem.py:159-174 with bytes: pages [0, 2] -> [2, 3]
    dm = DevicePageManager([("GPU", 16 * PAGE, PAGE)])
    a = dm.allocate(TensorSpec("a", "param16", PAGE, 0), "GPU")
    b = dm.allocate(TensorSpec("b", "param16", PAGE, 0), "GPU")
    c = dm.allocate(TensorSpec("c", "param16", PAGE, 0), "GPU")
    bd = np.arange(PAGE // 2, dtype=np.float16)
    dm.write(b.tensor_id, bd)
    dm.release(a.tensor_id)
    dm.release(c.tensor_id)
    t = dm.allocate(TensorSpec("t", "param16", 2 * PAGE, 0), "GPU")
    td = np.random.default_rng(0).normal(0, 1, PAGE).astype(np.float16)
    dm.write(t.tensor_id, td)
    assert t.page_list == [0, 2]
    assert dm.tensor_merge(t.tensor_id)["page_ids"] == [2, 3]
    assert np.array_equal(dm.read(t.tensor_id).cpu().numpy().view(np.uint16), td.view(np.uint16))
    assert np.array_equal(dm.read(b.tensor_id).cpu().numpy().view(np.uint16), bd.view(np.uint16))


def test_pack_matches_oracle_layout(cuda):
    """Bytes land at (slot * page + offset) exactly as the oracle's pack()."""
    dm = DevicePageManager([("GPU", 32 * PAGE, PAGE)])
    rng = np.random.default_rng(4)
    pool = np.zeros(32 * PAGE // 2, dtype=np.uint16)
    for i, n in enumerate([40000, 5, 32768, 25003, 777]):
        t = dm.allocate(TensorSpec(f"x{i}", "param16", 2 * n, 0), "GPU")
        d = rng.integers(0, 65535, n, dtype=np.uint16)
        dm.write(t.tensor_id, d)
        O.pack(pool, d, t.segments(), PAGE // 2, 2)
    got = dm.storage[next(iter(dm.storage))].cpu().numpy().view(np.uint16)
    assert np.array_equal(got, pool)


def test_ssd_tier_moves_bytes(cuda, tmp_path):
    """An SSD pool backed by a file: page_move GPU/CPU <-> SSD (fp32 pages
    only, the reference's rule), pack/unpack of SSD-resident pages and a merge
    inside the SSD tier all move real bytes; the page table stays identical
    to the metadata-only manager."""
    specs = [("GPU", 16 * PAGE, PAGE), ("CPU", 16 * PAGE, PAGE), ("SSD", 16 * PAGE, PAGE)]
    dm = DevicePageManager(specs, ssd_path=str(tmp_path / "ssd.pool"))
    meta = PageManager(specs)
    nrng = np.random.default_rng(7)
    nbytes = 3 * PAGE + 4096
    spec = TensorSpec("opt", "optim32", nbytes, 0)
    t = dm.allocate(spec, "GPU")
    meta.allocate(spec, "GPU")
    data = nrng.normal(0, 1, nbytes // 4).astype(np.float32)
    dm.write(t.tensor_id, data)

    def check(want):
        got = dm.read(t.tensor_id).cpu().numpy()
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))

    for pid in list(dm.tensors[t.tensor_id].page_list):          # GPU -> SSD
        assert dm.page_move(pid, "SSD") == meta.page_move(pid, "SSD")
        check(data)
    data2 = nrng.normal(0, 1, nbytes // 4).astype(np.float32)     # pack into SSD pages
    dm.write(t.tensor_id, torch.from_numpy(data2).cuda())
    check(data2)
    for hop in ("CPU", "SSD", "GPU"):                             # SSD -> CPU -> SSD -> GPU
        for pid in list(dm.tensors[t.tensor_id].page_list):
            assert dm.page_move(pid, hop) == meta.page_move(pid, hop)
        check(data2)
    # a 16-bit tensor may not go to SSD (hiermem/pagemem.py page_move rules)
    h = dm.allocate(TensorSpec("p16", "param16", PAGE, 0), "GPU")
    meta.allocate(TensorSpec("p16", "param16", PAGE, 0), "GPU")
    with pytest.raises(MoveError):
        dm.page_move(dm.tensors[h.tensor_id].page_list[0], "SSD")
    with pytest.raises(MoveError):
        meta.page_move(meta.tensors[h.tensor_id].page_list[0], "SSD")
    # merge inside the SSD tier: fragment, then defragment with data
    for pid in list(dm.tensors[t.tensor_id].page_list):
        dm.page_move(pid, "SSD")
        meta.page_move(pid, "SSD")
    a = dm.allocate(TensorSpec("gap", "optim32", PAGE, 0), "SSD")
    meta.allocate(TensorSpec("gap", "optim32", PAGE, 0), "SSD")
    dm.release(a.tensor_id)
    meta.release(a.tensor_id)
    assert dm.tensor_merge(t.tensor_id) == meta.tensor_merge(t.tensor_id)
    check(data2)
    assert dm.state_dict() == meta.state_dict()
    dm.close()
