"""Oracle test infrastructure: small CPU restatements of the reference's primitives.

Checker only -- imported by tests/, never by the product.  Each function cites the reference
lines it restates.  Python floats are IEEE-754 binary64 and every expression below is evaluated
in the reference's operation order, so results are bit-identical to the C++ (which is built
without FMA contraction).  Pinned by tests/test_oracle_kats.py against the reference's own
known-answer tests and against the compiled reference in oracle/_ref.
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence, Tuple

M64 = (1 << 64) - 1


def fnv1a(s: str) -> int:
    """workload.cpp:24-31"""
    h = 1469598103934665603
    for c in s.encode():
        h ^= c
        h = (h * 1099511628211) & M64
    return h


def splitmix64(x: int) -> int:
    """workload.cpp:33-38"""
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def substream_seed(seed: int, name: str, purpose: int) -> int:
    """make_substream, workload.cpp:42-47"""
    m = splitmix64(seed)
    m = splitmix64(m ^ fnv1a(name))
    return splitmix64(m ^ purpose)


class MT19937_64:
    """std::mt19937_64 (libstdc++ random.tcc _M_gen_rand / operator())."""

    N, M = 312, 156
    A = 0xB5026F5AA96619E9
    UPPER, LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int):
        self.x = [0] * self.N
        self.x[0] = seed & M64
        for i in range(1, self.N):
            p = self.x[i - 1]
            self.x[i] = (6364136223846793005 * (p ^ (p >> 62)) + i) & M64
        self.p = self.N

    def _twist(self):
        x, N, M = self.x, self.N, self.M
        for k in range(N):
            y = (x[k] & self.UPPER) | (x[(k + 1) % N] & self.LOWER)
            x[k] = x[(k + M) % N] ^ (y >> 1) ^ (self.A if y & 1 else 0)
        self.p = 0

    def __call__(self) -> int:
        if self.p >= self.N:
            self._twist()
        z = self.x[self.p]
        self.p += 1
        z ^= (z >> 29) & 0x5555555555555555
        z ^= (z << 17) & 0x71D67FFFEDA60000 & M64
        z ^= (z << 37) & 0xFFF7EEE000000000 & M64
        z ^= z >> 43
        return z


def canonical(v: int) -> float:
    """generate_canonical<double,53> with a 64-bit engine (random.tcc:3346-3381)."""
    d = float(v) / 18446744073709551616.0
    return d if d < 1.0 else math.nextafter(1.0, 0.0)


def allocate_bandwidth(flows: Sequence[Tuple[float, Optional[float]]], capacity: float,
                       water_filling: bool = False) -> Tuple[List[float], float]:
    """fabric::allocate_bandwidth (fabric.cpp:31-87). flows = [(weight, cap or None)]."""
    if capacity <= 0.0:
        raise ValueError("fabric capacity must be > 0")
    if not flows:
        return [], capacity
    wsum = 0.0
    for w, c in flows:
        if w <= 0.0:
            raise ValueError("PS weights must be > 0")
        wsum += w
    grants = []
    granted = 0.0
    for w, c in flows:
        share = capacity * w / wsum
        b = min(share, c) if c is not None else share
        grants.append(b)
        granted += b
    if water_filling:
        residual = capacity - granted
        it = 0
        while it < 64 and residual > 1e-9 * capacity:
            open_w = 0.0
            for (w, c), g in zip(flows, grants):
                if c is None or g < c - 1e-12:
                    open_w += w
            if open_w <= 0.0:
                break
            moved = 0.0
            for i, (w, c) in enumerate(flows):
                g = grants[i]
                if c is not None and g >= c - 1e-12:
                    continue
                add = residual * w / open_w
                if c is not None:
                    add = min(add, c - g)
                grants[i] = g + add
                moved += add
            residual -= moved
            if moved <= 1e-12 * capacity:
                break
            it += 1
        granted = 0.0
        for g in grants:
            granted += g
    return grants, capacity - granted


def nearest_rank(values: Sequence[float], q: float) -> float:
    """TailWindow::quantile / Sim::finish rank (telemetry.cpp:38-56, engine.cpp:800-816)."""
    v = sorted(values)
    n = len(v)
    r = int(math.ceil(q * float(n)))
    r = max(1, min(r, n))
    return v[r - 1]


def ema_run(alpha: float, trigger: float, clear: float, xs: Sequence[float]):
    """SmoothedSignal::update (telemetry.cpp:81-95): returns [(ema, triggered)]."""
    ema, trig, out = None, False, []
    for x in xs:
        ema = x if ema is None else alpha * x + (1.0 - alpha) * ema
        if not trig and ema > trigger:
            trig = True
        elif trig and ema < clear:
            trig = False
        out.append((ema, trig))
    return out


def confidence_interval(values: Sequence[float]) -> Tuple[float, float]:
    """harness::confidence_interval (harness.cpp:32-43), population sigma, seed order."""
    if not values:
        return 0.0, 0.0
    n = float(len(values))
    s = 0.0
    for v in values:
        s += v
    mean = s / n
    ss = 0.0
    for v in values:
        ss += (v - mean) * (v - mean)
    return mean, 1.96 * math.sqrt(ss / n) / math.sqrt(n)


HIST_BINS = 2048
_HIST_SHIFT = 46
_HIST_BASE = ((1 << 63) | ((1023 - 10) << 52)) >> _HIST_SHIFT


def lat_bins(values):
    """Latency-histogram bin of each FP64 value (the engine's fixed log-spaced bins: the top 18 bits
    of the order-preserving key, 64 bins per octave from 2^-10 ms, clamped at both ends) -- a
    numpy restatement used to bin the reference's own completion records for the histogram tests."""
    import numpy as np

    b = np.ascontiguousarray(np.asarray(values, np.float64)).view(np.uint64)
    neg = (b >> np.uint64(63)) != 0
    key = np.where(neg, ~b, b | np.uint64(1 << 63))
    v = (key >> np.uint64(_HIST_SHIFT)).astype(np.int64)
    return np.clip(v - _HIST_BASE, 0, HIST_BINS - 1)
