"""GPU parity with a fitted Eq. 2 model: a pattern
whose coefficients come from mapa_fit_effbw (noisy synthetic samples) ranks
censuses by those coefficients on the device; the Preserve-sensitive decision
equals the Python oracle's with the same theta (exact rationals)."""
import random

import pytest

from oracle import mapa_oracle as mo

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2110_03214_b200 as mp  # noqa: E402


def test_fitted_model_decisions_vs_oracle():
    rng = random.Random(615)
    cens = [(x, y, z) for s in range(8) for x in range(s + 1) for y in range(s + 1 - x) for z in [s - x - y]][:31]
    theta, _dg = mp.fit_effbw([(x, y, z, mo.eq2(x, y, z) + rng.gauss(0, 3.0)) for x, y, z in cens])
    for name in ("dgx1v", "summit", "cubemesh16"):
        o = mo.builtin(name)
        t = mp.Topology(name)
        for trial in range(20):
            shape = rng.choice(["ring", "tree", "ringtree", "full"])
            k = rng.randint(2, 5 if o.n <= 8 else 4)
            busy = rng.randrange(0, 1 << o.n) & ~((1 << k) - 1) if o.n <= 8 else rng.randrange(0, 1 << o.n) | 0xFF
            if o.n - bin(busy).count("1") < k:
                busy = 0
            p = mp.Pattern.make(shape, k)
            p.set_effbw_model(theta)
            t.set_busy(busy)
            for deep in (False, True):
                g = mp.allocate(t, p, 1, True, deep=deep)
                kk, e = mo.make_pattern(shape, k)
                ex = mo.allocate(o, busy, kk, e, 1, True, theta=theta)
                for f in ("devices", "mapping", "used_edges", "x", "y", "z"):
                    assert g[f] == ex[f], (name, trial, shape, k, hex(busy), deep, f)
                assert abs(g["pred_effbw"] - float(ex["pred_effbw_exact"])) < 1e-6 * max(1, abs(g["pred_effbw"]))
