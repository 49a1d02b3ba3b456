"""Oracle of Algorithm 2, SLO-Aware Latency Control.

TEST INFRASTRUCTURE ONLY (see oracle/brownout_oracle.py header).  Written
literally from Alg. 2 with the readings of DESIGN.md (nearest-rank P90 over
the window (now - tw, now]; empty window holds; clamp to [0, 1]).
"""
import math


def p90_nearest_rank(samples, now, tw):
    """Alg. 2 line 4 get_recent_P90_latency: samples = [(t, latency)]."""
    window = sorted(v for (t, v) in samples if now - tw < t <= now)
    if not window:
        return None
    return window[math.ceil(0.9 * len(window)) - 1]


def salc_update(threshold, slo, warning_factor, increment, shrink_ratio, latency):
    """Alg. 2 lines 3-9 for a given recent P90 latency (None: hold)."""
    warning_line = slo * warning_factor
    if latency is None:
        return threshold
    if latency < warning_line:
        threshold = threshold + increment
    elif latency > slo:
        threshold = threshold * shrink_ratio
    return min(1.0, max(0.0, threshold))
