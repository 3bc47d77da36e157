"""Eq. 2 regression (§3.4.3; SPEC
fit_effbw_model S:286-294) — CPU only.  Pins: the synthetic round trip
recovers Table 4 within 1e-6, 13 samples are rejected, noisy
samples (sigma 0.5) fit with relative error <= 0.1; the library's QR
solve equals the oracle's numpy lstsq; a rank-deficient census set is named."""
import random

import pytest

from oracle import mapa_oracle as mo

import paper_2110_03214_b200 as mp

TABLE4 = [16.396, 4.536, 1.556, -20.694, -9.467, 7.615, -7.973, 12.733, -4.195, -8.413, 62.851, 27.418, -5.114,
          -46.973]


def _censuses(n):
    cs = [(x, y, z) for s in range(0, 8) for x in range(s + 1) for y in range(s + 1 - x) for z in [s - x - y]]
    return cs[:n]


def test_round_trip_recovers_table4():
    samples = [(x, y, z, mo.eq2(x, y, z)) for x, y, z in _censuses(31)]
    th, dg = mp.fit_effbw(samples)
    assert max(abs(a - b) for a, b in zip(th, TABLE4)) < 1e-6
    assert dg["rel_err"] < 1e-9
    th2, rel2 = mo.fit_effbw(samples)
    assert max(abs(a - b) for a, b in zip(th2, TABLE4)) < 1e-6


def test_underdetermined_and_rank_deficient():
    samples = [(x, y, z, mo.eq2(x, y, z)) for x, y, z in _censuses(13)]
    with pytest.raises(mp.MapaError):
        mp.fit_effbw(samples)
    with pytest.raises(ValueError):
        mo.fit_effbw(samples)
    flat = [(x, 0, 0, 10.0 + x) for x in range(20)]  # y = z = 0: y, z, yz, ... features collapse
    with pytest.raises(mp.MapaError) as e:
        mp.fit_effbw(flat)
    assert "rank-deficient" in str(e.value)


def test_noisy_fit_relative_error():
    rng = random.Random(614)
    for trial in range(5):
        samples = [(x, y, z, mo.eq2(x, y, z) + rng.gauss(0.0, 0.5)) for x, y, z in _censuses(31)]
        th, dg = mp.fit_effbw(samples)
        assert dg["rel_err"] <= 0.1
        th2, rel2 = mo.fit_effbw(samples)
        assert max(abs(a - b) / max(1.0, abs(b)) for a, b in zip(th, th2)) < 1e-7
        assert abs(dg["rel_err"] - rel2) < 1e-9
        # the fitted model evaluates as Eq. 2 with those coefficients
        for x, y, z in _censuses(40)[::7]:
            exp = sum(t * f for t, f in zip(th, mo.eq2_features(x, y, z)))
            assert abs(mp.pred_effbw_theta(th, x, y, z) - exp) < 1e-9 * max(1.0, abs(exp))
