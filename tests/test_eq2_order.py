"""Reading A9: ranking censuses by Eq. 2 in double precision is exact.

For every edge count m <= 120 (C(16,2): the deep path's cliques) the censuses (x, y, z) with x+y+z = m have
pairwise-distinct exact Eq. 2 values, separated by far more than double
rounding error, so any double evaluation (the C oracle, the library's host
rank table) orders them exactly as the rational values do.  CPU only."""
from fractions import Fraction

import pytest

from oracle import mapa_oracle as mo


@pytest.mark.parametrize("m", list(range(0, 121)))
def test_no_ties_and_wide_gaps(m):
    vals = sorted(mo.eq2_exact(x, y, m - x - y) for x in range(m + 1) for y in range(m + 1 - x))
    gaps = [b - a for a, b in zip(vals, vals[1:])]
    assert all(g > 0 for g in gaps)
    if gaps:
        # relative gap: the smallest is 4.7e-9 (m = 84), ~1e6 x double rounding
        assert min(g / max(abs(b), 1) for g, b in zip(gaps, vals[1:])) > Fraction(1, 10 ** 9)
    dbl = sorted((mo.eq2(x, y, m - x - y), (x, y)) for x in range(m + 1) for y in range(m + 1 - x))
    ex = sorted((mo.eq2_exact(x, y, m - x - y), (x, y)) for x in range(m + 1) for y in range(m + 1 - x))
    assert [c for _, c in dbl] == [c for _, c in ex]
