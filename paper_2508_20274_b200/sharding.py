"""Seed sharding across GPUs and the end-of-run reduction.

Replicas (variant x seed) share nothing (/root/reference/proj/src/harness.cpp:156-176), so ranks
take contiguous seed blocks and run with no data-path communication.  At the end only two small
collectives run (torch.distributed: NCCL over NVLink on the GPU box, gloo in the CPU tests):
  * all-reduce (sum, int64) of the per-variant SLO-miss-rate histogram (1e-3 bins on [0, 1]);
  * all-gather of the per-seed focus rows (p99, miss rate, summed throughput) so rank 0 can
    build harness-identical confidence intervals by summing in seed order
    (harness.cpp:32-43, 178-204);
  * all-reduce (sum, int64) of the per-(variant, tenant) window-latency histograms (lat_hist.h
    bins, summed over seeds on the device) and the per-(variant, tenant) completion / window /
    SLO-miss counters (engine.cpp:497-501, 797-798).  Integer, so exact and order-independent.
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

import numpy as np

N_BINS = 1000


def seed_block(rank: int, world: int, seeds_per_rank: int, seed_base: int = 1) -> List[int]:
    """Contiguous block of seeds for `rank` (weak scaling: fixed seeds per rank)."""
    start = seed_base + rank * seeds_per_rank
    return list(range(start, start + seeds_per_rank))


def split_seeds(seeds: Sequence[int], rank: int, world: int) -> List[int]:
    """Contiguous block [r*N/P, (r+1)*N/P) of a fixed seed list (strong scaling)."""
    n = len(seeds)
    return list(seeds[rank * n // world:(rank + 1) * n // world])


def miss_histogram(miss_rates: np.ndarray) -> np.ndarray:
    """Exact integer histogram of per-seed miss rates, 1e-3 wide bins over [0, 1]."""
    idx = np.minimum((np.asarray(miss_rates, np.float64) * N_BINS).astype(np.int64), N_BINS - 1)
    return np.bincount(idx, minlength=N_BINS).astype(np.int64)


def confidence_interval(values: Sequence[float]) -> Tuple[float, float]:
    """harness::confidence_interval (harness.cpp:32-43): population sigma, summed in order."""
    if len(values) == 0:
        return 0.0, 0.0
    n = float(len(values))
    s = 0.0
    for v in values:
        s += float(v)
    mean = s / n
    ss = 0.0
    for v in values:
        ss += (float(v) - mean) * (float(v) - mean)
    return mean, 1.96 * math.sqrt(ss / n) / math.sqrt(n)


def gather_rows(local, dist):
    """All-gather of per-rank row blocks whose lengths may differ (uneven seed splits, empty
    ranks): all_gather needs equal shapes, so the counts go first, every block is padded to the
    largest, and each part is trimmed back to its real length, in rank order."""
    import torch

    world = dist.get_world_size()
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    width = max(counts)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], 0)


def reduce_rows(rows: np.ndarray, dist=None, device: str = "cpu"):
    """rows: float64 [n_local_seeds, 3] = (p99_ms, miss_rate, throughput_hz) in seed order.

    Returns (all_rows in global seed order, summed miss histogram, CIs) on every rank.
    """
    import torch

    rows = np.asarray(rows, np.float64).reshape(-1, 3)
    hist = torch.tensor(miss_histogram(rows[:, 1]), dtype=torch.int64, device=device)
    local = torch.tensor(np.ascontiguousarray(rows), device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(hist)
        local = gather_rows(local, dist)
    all_rows = local.cpu().numpy()
    cis = [confidence_interval(all_rows[:, k]) for k in range(3)]
    return all_rows, hist.cpu().numpy(), cis


def reduce_tenant_hists(lat_hist: np.ndarray, counts: np.ndarray, dist=None, device: str = "cpu"):
    """lat_hist: int64 [n_variants, n_tenants, bins]; counts: int64 [n_variants, n_tenants, 3]
    (completed_total, completed_window, window_misses), this rank's sums over its seeds.

    One all-reduce (sum) of both, packed into a single int64 buffer; returns the global sums on
    every rank.  Every rank must pass the same shapes (same scenario and variants)."""
    import torch

    lat_hist = np.ascontiguousarray(lat_hist, np.int64)
    counts = np.ascontiguousarray(counts, np.int64)
    if dist is None or not dist.is_initialized() or dist.get_world_size() <= 1:
        return lat_hist.copy(), counts.copy()
    buf = torch.from_numpy(np.concatenate([lat_hist.ravel(), counts.ravel()])).to(device)
    dist.all_reduce(buf)
    out = buf.cpu().numpy()
    return out[: lat_hist.size].reshape(lat_hist.shape), out[lat_hist.size:].reshape(counts.shape)


def pooled_quantiles(hist_row: np.ndarray, edges: np.ndarray, qs: Sequence[float] = (0.5, 0.95, 0.99, 0.999)
                     ) -> List[Tuple[float, float]]:
    """Pooled tail of one (variant, tenant) over every seed and rank: for each q, the latency bin
    [lo, hi) that holds the nearest-rank q-quantile (rank = clamp(ceil(q * N), 1, N), the reference's
    rule, telemetry.cpp:52-55) of ALL measurement-window latencies summed into `hist_row` (the
    reduced lat_hist.h histogram, 64 bins per octave).  The SURVEY 8(f)3 p999 / TTFT extension for
    C3 / C4: exact to the bin, from integer counts, so identical on any number of ranks.  `edges`:
    api.hist_bin_edges() (bin lower edges); the first bin is open below, the last open above."""
    h = np.asarray(hist_row, np.int64)
    n = int(h.sum())
    if n == 0:
        return [(math.nan, math.nan) for _ in qs]
    cum = np.cumsum(h)
    out = []
    for q in qs:
        rank = min(max(int(math.ceil(q * n)), 1), n)
        b = int(np.searchsorted(cum, rank))  # first bin whose cumulative count reaches the rank
        lo = -math.inf if b == 0 else float(edges[b])
        hi = math.inf if b + 1 >= len(edges) else float(edges[b + 1])
        out.append((lo, hi))
    return out
