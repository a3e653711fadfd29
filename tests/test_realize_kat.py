"""Known-answer tests of the realize module's helpers (the
reference declares them in realize.hpp:30-54 without an implementation, so
the SPEC examples and invariants are the pinning), and SPEC acceptance 7:
requantize relative error <= 2^-30 over 10^5 ratios in [2^-20, 2^20]."""
import numpy as np
import pytest

from paper_2103_14949_b200 import quantc as Q


def test_requantize_params_examples(b200):
    assert b200.requantize_params(0.5, 1.0) == (1 << 30, 31)       # ratio 0.5
    assert b200.requantize_params(1.0, 1.0) == (1 << 30, 30)       # ratio 1
    assert b200.requantize_params(0.75, 1.0) == (1610612736, 31)   # ratio 0.75
    assert b200.requantize_params(3.0, 4.0) == (1610612736, 31)
    with pytest.raises(Q.QuantcError):
        b200.requantize_params(0.0, 1.0)
    with pytest.raises(Q.QuantcError):
        b200.requantize_params(1.0, -2.0)


def test_requantize_params_acceptance_7(b200):
    """10^5 random ratios in [2^-20, 2^20]: multiplier in [2^30, 2^31) and
    |multiplier * 2^-shift - ratio| / ratio <= 2^-30."""
    rng = np.random.default_rng(7)
    ratios = np.exp2(rng.uniform(-20, 20, 100_000))
    worst = 0.0
    for r in ratios:
        m, sh = b200.requantize_params(float(r), 1.0)
        assert (1 << 30) <= m < (1 << 31)
        approx = m * 2.0 ** -sh
        worst = max(worst, abs(approx - r) / r)
    assert worst <= 2.0 ** -30, worst
    # rounding up to 2^31 halves the multiplier and decrements the shift
    r = 1.0 - 2.0 ** -40
    assert b200.requantize_params(r, 1.0) == (1 << 30, 30)


def test_requantize_params_pow2_is_shift_only(b200):
    """Power-of-two mode: every power-of-two ratio gives multiplier 2^30."""
    for e in range(-20, 21):
        m, sh = b200.requantize_params(2.0 ** e, 1.0)
        assert m == 1 << 30 and sh == 30 - e


def test_choose_storage_dtype_examples(b200):
    assert b200.choose_storage_dtype(6, ["int8", "int16"]) == "int8"
    assert b200.choose_storage_dtype(12, ["int8", "int16"]) == "int16"
    assert b200.choose_storage_dtype(8, ["int16", "int8"]) == "int8"   # narrowest wins
    assert b200.choose_storage_dtype(8, ["uint8", "int8"], sign=0) == "uint8"
    assert b200.choose_storage_dtype(7, ["uint8", "int8"], sign=1) == "int8"
    with pytest.raises(Q.QuantcError):
        b200.choose_storage_dtype(9, ["int8"])
    with pytest.raises(Q.QuantcError):
        b200.choose_storage_dtype(8, ["uint8"], sign=1)  # signed code needs a signed dtype


def test_rewrite_clip_examples(b200):
    assert b200.rewrite_clip(0.0, 6.0, 0.05, 0, "int8") == (0, 120)     # ReLU6
    assert b200.rewrite_clip(0.0, 6.0, 0.05, 10, "int8") == (10, 127)   # dtype intersection
    assert b200.rewrite_clip(-1.0, 1.0, 1.0, 0, "int8") == (-1, 1)
    assert b200.rewrite_clip(-100.0, 100.0, 0.5, 0, "int16") == (-200, 200)
    assert b200.rewrite_clip(0.0, 6.0, 0.01, 0, "uint8") == (0, 255)
