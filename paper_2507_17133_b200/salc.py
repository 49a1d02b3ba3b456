"""SLO-Aware Latency Control (SALC), Algorithm 2 of the paper.

Host-side controller of the brownout knob: after each forward the caller
records the measured latency; ``update`` computes the P90 latency over the
recent window ``tw`` and moves the threshold additively up (latency below the
warning line ``slo * warning_factor``) or multiplicatively down (latency above
the SLO), leaving it alone in the dead band between them.  The brownout ratio
handed to ``bo_set_brownout`` is ``1 - threshold`` (reading D2).

Readings: P90 is nearest-rank over the samples with timestamp in
(now - tw, now]; an empty window holds the threshold; the threshold is clamped
to [floor, cap] = [0, 1] (a proportion).  Defaults are the paper's §5.4
parameters (warning factor 0.8, shrink ratio 0.8, increment 0.1).
"""
from __future__ import annotations

import math
from collections import deque


class SALC:
    def __init__(self, slo: float, warning_factor: float = 0.8, tw: float = 1.0, increment: float = 0.1,
                 shrink_ratio: float = 0.8, threshold: float = 1.0, floor: float = 0.0, cap: float = 1.0):
        if not (0.0 < warning_factor < 1.0) or not (0.0 < shrink_ratio < 1.0) or slo <= 0 or tw <= 0:
            raise ValueError("invalid SALC parameters")
        if not (0.0 <= floor <= cap <= 1.0):
            raise ValueError("invalid threshold bounds")
        self.slo, self.warning_factor, self.tw = slo, warning_factor, tw
        self.increment, self.shrink_ratio = increment, shrink_ratio
        self.floor, self.cap = floor, cap
        self.threshold = min(cap, max(floor, threshold))
        self._t = deque()
        self._v = deque()

    @property
    def ratio(self) -> float:
        """Brownout ratio for bo_set_brownout (reading D2: ratio = 1 - threshold)."""
        return 1.0 - self.threshold

    def record(self, t: float, latency: float):
        if self._t and t < self._t[-1]:
            raise ValueError("latency samples must be recorded in time order")
        self._t.append(t)
        self._v.append(latency)

    def p90(self, now: float):
        """Nearest-rank 90th percentile of the samples in (now - tw, now]; None if empty."""
        while self._t and self._t[0] <= now - self.tw:   # evict samples that left the window
            self._t.popleft()
            self._v.popleft()
        vals = sorted(v for t, v in zip(self._t, self._v) if t <= now)
        if not vals:
            return None
        rank = math.ceil(0.9 * len(vals))                 # nearest rank, 1-based
        return vals[rank - 1]

    def update(self, now: float) -> float:
        """Algorithm 2 lines 3-9; returns the new threshold."""
        warning_line = self.slo * self.warning_factor        # line 3
        latency = self.p90(now)                              # line 4
        if latency is None:
            return self.threshold
        if latency < warning_line:                           # lines 5-6
            self.threshold = min(self.cap, self.threshold + self.increment)
        elif latency > self.slo:                             # lines 7-8
            self.threshold = max(self.floor, self.threshold * self.shrink_ratio)
        return self.threshold

