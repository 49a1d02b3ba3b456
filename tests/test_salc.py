"""SALC (Algorithm 2), the NEXT row f1 of SURVEY §8(f): oracle pins
from the paper's §5.4 parameters and product-vs-oracle parity."""
import random

import pytest

from oracle import salc_oracle as SO
from paper_2507_17133_b200.salc import SALC

# §5.4: warning factor 0.8, shrink ratio 0.8, increment 0.1; prefill SLO 0.25 s
P = dict(slo=0.25, warning_factor=0.8, increment=0.1, shrink_ratio=0.8)


@pytest.mark.parametrize("thr,lat,want", [
    (0.5, 0.26, 0.40),    # above the SLO: x 0.8
    (0.5, 0.15, 0.60),    # below the warning line 0.20: + 0.1
    (0.5, 0.22, 0.50),    # dead band [0.20, 0.25]
    (0.95, 0.10, 1.00),   # clamp to 1
    (0.5, None, 0.50),    # empty window: hold
])
def test_oracle_pins_alg2_arithmetic(thr, lat, want):
    assert SO.salc_update(thr, latency=lat, **P) == pytest.approx(want, abs=1e-12)


def test_oracle_p90_nearest_rank():
    s = [(i, 0.01 * (i + 1)) for i in range(10)]          # 0.01 .. 0.10
    assert SO.p90_nearest_rank(s, now=9, tw=100) == pytest.approx(0.09)
    assert SO.p90_nearest_rank([(0, 0.2)], now=0, tw=1) == 0.2
    assert SO.p90_nearest_rank([], now=0, tw=1) is None


def test_controller_matches_oracle_on_random_traces():
    rng = random.Random(0)
    for trial in range(50):
        tw = rng.choice([0.5, 1.0, 2.0])
        c = SALC(tw=tw, threshold=rng.random(), **P)
        thr = c.threshold
        samples = []
        t = 0.0
        for it in range(200):
            t += rng.random() * 0.05
            lat = rng.choice([0.1, 0.21, 0.3]) * (0.8 + 0.4 * rng.random())
            c.record(t, lat)
            samples.append((t, lat))
            got = c.update(t)
            thr = SO.salc_update(thr, latency=SO.p90_nearest_rank(samples, t, tw), **P)
            assert got == pytest.approx(thr, abs=1e-12)
            assert 0.0 <= got <= 1.0
            assert c.ratio == pytest.approx(1.0 - got)


def test_controller_rejects_time_regression():
    c = SALC(slo=0.25)
    c.record(1.0, 0.1)
    with pytest.raises(ValueError):
        c.record(0.5, 0.1)
