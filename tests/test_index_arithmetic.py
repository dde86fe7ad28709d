"""Host-side checks of the integer identities the raster flush relies on (raster.cu, the flush
after each batch): for a divisor d that is not a power of two, __umulhi(i, ceil(2^32 / d)) equals
i // d for every flush index i < MAX_SLOTS * BATCH * d when d <= 2048, and for every level
index ls < nlev * S when dividing by S.  Pure integer arithmetic, no GPU."""
import numpy as np
import pytest

MAX_SLOTS, BATCH, MAX_LEVELS, MAX_L = 16, 32, 4, 1024


def umulhi(i, m):
    return (i.astype(np.uint64) * np.uint64(m)) >> np.uint64(32)


def magic(d):
    return 0xFFFFFFFF // d + 1  # ceil(2^32 / d) for d not a power of two


@pytest.mark.parametrize("d", [3, 5, 6, 7, 12, 24, 48, 96, 1000, 1536, 2047, 2048 - 24])
def test_flush_index_division_exact(d):
    """i // LS for every flush index of a full slot table (the sweep's u = i / LS)."""
    n = MAX_SLOTS * BATCH * d
    i = np.arange(n, dtype=np.uint64)
    assert np.array_equal(umulhi(i, magic(d)), i // np.uint64(d))


def test_flush_index_division_all_small_divisors():
    """Every non-power-of-two LS up to 2048 (the bound the kernel checks), at the edges of the
    index range where the rounding error of the magic number is largest."""
    for d in range(3, 2049):
        if d & (d - 1) == 0:
            continue
        n = MAX_SLOTS * BATCH * d
        i = np.concatenate([np.arange(min(n, 2048)), np.arange(max(0, n - 2048), n)]).astype(np.uint64)
        assert np.array_equal(umulhi(i, magic(d)), i // np.uint64(d)), d


def test_level_index_division_exact():
    """l = ls // S for every ls < nlev * S, S up to SCOUP_MAX_L (dense features: S == L)."""
    for S in list(range(3, 70)) + [96, 100, 127, 500, 513, 1000, 1023]:
        if S & (S - 1) == 0:
            continue
        ls = np.arange(MAX_LEVELS * S, dtype=np.uint64)
        assert np.array_equal(umulhi(ls, magic(S)), ls // np.uint64(S)), S
    assert MAX_LEVELS * MAX_L * MAX_L < 2 ** 32
