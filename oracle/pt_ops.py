"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Seeded page-table operation script, a superset of the reference's own
randomized generator (tests/test_pagemem.py:241-273 of the reference):
allocate / release / page_move as there, plus occasional tensor_merge.
It is replayed against any module exposing the hiermem.pagemem API, so the
same script runs on the reference (to make golden dumps) and on the native
page table (to check them).
"""
from __future__ import annotations

import copy
import random

MIB = 2 ** 20


def replay(mod, spec_cls, errors, seed: int, steps: int = 600, merge_rate: float = 0.05):
    """Returns (state_dict, op_log).  ``errors`` = (AllocationError, MoveError)."""
    alloc_err, move_err = errors
    rng = random.Random(seed)
    mgr = mod.PageManager([("GPU", 256 * MIB, 4 * MIB), ("CPU", 256 * MIB, 4 * MIB),
                           ("SSD", 128 * MIB, 4 * MIB)])
    live: list[int] = []
    counter = 0
    log = []
    for _ in range(steps):
        op = rng.random()
        if op < 0.5:
            kind = rng.choice(["param16", "grad16", "optim32", "activation16"])
            tier = "SSD" if (kind == "optim32" and rng.random() < 0.3) else rng.choice(["GPU", "CPU"])
            nbytes = rng.choice([1024, MIB, 2 * MIB, 4 * MIB, 7 * MIB, 12 * MIB])
            counter += 1
            try:
                t = mgr.allocate(spec_cls(f"t{counter}", kind, nbytes, 0), tier)
                live.append(t.tensor_id)
                log.append(["alloc", t.tensor_id, list(t.page_list)])
            except alloc_err as e:
                log.append(["alloc_err", e.requested_bytes, e.available_bytes])
        elif op < 0.8 and live:
            tid = live.pop(rng.randrange(len(live)))
            log.append(["release", tid, mgr.release(tid)])
        elif live:
            tid = rng.choice(live)
            pid = rng.choice(mgr.tensors[tid].page_list)
            target = rng.choice(["GPU", "CPU"])
            try:
                d = mgr.page_move(pid, target)
                log.append(["move", d.bytes, d.src_tier.name, d.dst_tier.name, d.page_id, d.new_page_id])
            except move_err:
                log.append(["move_err", pid, target])
        if live and rng.random() < merge_rate:
            tid = rng.choice(live)
            try:
                r = copy.deepcopy(mgr.tensor_merge(tid))
                log.append(["merge", r["tensor_id"], r["moved_chunks"], list(r["page_ids"])])
            except (alloc_err, move_err) as e:
                log.append(["merge_err", type(e).__name__])
    return mgr.state_dict(), log
