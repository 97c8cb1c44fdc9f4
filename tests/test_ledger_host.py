"""Host side of the always-on ConservationLedger (no GPU): entries that sit
in device ledger rows are resolved in place, in order, from one host copy of
the rows; the reference's summary rules (hiermem/lockfree.py:303-326) then
apply unchanged — balanced only when fsum(produced) == fsum(consumed) ==
fsum(applied + rejected) and the three message counts agree, and a NaN sum
makes its layer unbalanced."""
import math

import numpy as np

from paper_2303_02868_b200.lockfree import ConservationLedger


def _rows(*vals):
    a = np.zeros((len(vals), 8))
    for r, row in enumerate(vals):
        for c, v in row.items():
            a[r, c] = v
    return a


def test_pending_entries_resolve_in_order_and_balance():
    led = ConservationLedger(2)
    host = _rows({0: 1.5, 1: 0.25}, {0: 3.0}, {0: 4.75, 1: 1.0, 2: 3.0, 3: 1.0})
    # layer 0: two messages (rows 0 and 1, column = the slot), one take + apply (row 2)
    led._pend(led._produced[0], 0, 0)
    led._pend(led._produced[0], 1, 0)
    led.messages_accumulated[0] += 2
    led.messages_sent[0] += 2
    led._pend(led._consumed[0], 2, 0)
    led.messages_consumed[0] += 2
    led._apply_pending.append((0, 2, 0, 1))
    # layer 1: one message, taken and applied
    led._pend(led._produced[1], 0, 1)
    led.messages_accumulated[1] += 1
    led.messages_sent[1] += 1
    led._pend(led._consumed[1], 2, 2)
    led.messages_consumed[1] += 1
    led._apply_pending.append((1, 2, 2, 3))
    calls = []
    led._resolver = lambda: (calls.append(1), led._resolve(host)) if led._unresolved else None
    s = led.summary()
    assert calls == [1] and not led._unresolved and not led._apply_pending
    assert led.produced_deltas == [[1.5, 3.0], [0.25]]
    assert s["layers"][0]["produced"] == 4.5 and s["layers"][0]["consumed"] == 4.75
    assert not s["layers"][0]["balanced"]                 # 1.5 + 3.0 != 4.75
    assert s["layers"][1]["balanced"] is False            # 0.25 produced vs 3.0 consumed
    # host-side records (the reference's own calls) go through the same lists
    led2 = ConservationLedger(1)
    led2.messages_sent[0] = 1
    led2.record_accumulate(0, 2.0)
    led2.record_take(0, 2.0, 1)
    led2.record_apply(0, 2.0, rejected=False)
    assert led2.summary()["balanced"]


def test_rejected_and_nan_layers():
    led = ConservationLedger(2)
    host = _rows({0: 2.0, 1: float("nan")}, {0: 2.0, 1: 0.0, 2: float("nan"), 3: 0.0})
    for l in range(2):
        led.messages_sent[l] = led.messages_accumulated[l] = led.messages_consumed[l] = 1
        led._pend(led._produced[l], 0, l)
        led._pend(led._consumed[l], 1, 2 * l)
        led._apply_pending.append((l, 1, 2 * l, 2 * l + 1))
    led._resolve(host)
    s = led.summary()
    assert s["layers"][0]["rejected"] == 2.0 and s["layers"][0]["applied"] == 0.0
    assert s["layers"][0]["balanced"]                     # a rejected update still balances
    assert math.isnan(s["layers"][1]["produced"]) and not s["layers"][1]["balanced"]
    assert not s["balanced"]
