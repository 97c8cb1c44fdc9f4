"""DelayModel (hiermem/lockfree.py:81-117) mirrored: identical numbers for the
reference presets, plus the measured-B200 preset."""
import math

import pytest

from paper_2303_02868_b200.errors import ConfigError
from paper_2303_02868_b200.lockfree import DelayModel


def test_reference_presets():
    ssd, cpu, zero = (DelayModel.preset(n) for n in ("ssd", "cpu", "zero"))
    assert ssd.state_fetch_s(3.5e9) == pytest.approx(1.0)
    assert cpu.state_fetch_s(100e9) == pytest.approx(1.0)
    assert ssd.fetch_s(32e9) == ssd.offload_s(32e9) == pytest.approx(1.0)
    assert zero.compute_s(1e18) == 0.0 and zero.state_store_s(1) == 0.0
    assert math.isinf(zero.pcie_bytes_per_s)
    with pytest.raises(ConfigError):
        DelayModel.preset("tape")


def test_b200_preset_is_faster_everywhere():
    a, b = DelayModel.preset("ssd"), DelayModel.preset("b200")
    nbytes = 12 * 10**9
    assert b.fetch_s(nbytes) < a.fetch_s(nbytes)
    assert b.state_fetch_s(nbytes) < a.state_fetch_s(nbytes)
    assert b.update_compute_s(nbytes) < a.update_compute_s(nbytes) / 50
