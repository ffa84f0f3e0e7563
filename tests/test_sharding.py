"""Multi-rank (world_size 2, gloo on CPU) coverage of the seed sharding + end-of-run reduction
used by bench.py for N>1 GPUs."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import restate
from paper_2508_20274_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, rows_all, out, uneven=False):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if uneven:  # strong-scaling split of a seed list that does not divide evenly (sweep.py)
        seeds = sharding.split_seeds(list(range(1, len(rows_all) + 1)), rank, world)
    else:
        seeds = sharding.seed_block(rank, world, len(rows_all) // world)
    local = rows_all[np.array(seeds, dtype=np.int64) - 1] if seeds else np.zeros((0, 3))
    all_rows, hist, cis = sharding.reduce_rows(local, dist)
    out[rank] = (all_rows, hist, cis)
    dist.destroy_process_group()


def test_seed_blocks_partition():
    blocks = [sharding.seed_block(r, 4, 256) for r in range(4)]
    assert sum(blocks, []) == list(range(1, 1025))
    assert sum([sharding.split_seeds(list(range(10)), r, 3) for r in range(3)], []) == list(range(10))


def test_two_rank_reduction_matches_single_process():
    rng = np.random.default_rng(5)
    rows = np.stack([rng.lognormal(2, 0.5, 64), rng.uniform(0, 0.2, 64), rng.uniform(100, 200, 64)], 1)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rows, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    single_rows, single_hist, single_cis = sharding.reduce_rows(rows, None)
    for r in range(2):
        all_rows, hist, cis = out[r]
        assert (all_rows == rows).all()
        assert (hist == single_hist).all() and hist.sum() == 64
        assert cis == single_cis
        # CIs are harness-identical (population sigma, seed order)
        assert cis[0] == restate.confidence_interval(rows[:, 0].tolist())


def _run_ranks(rows, world, uneven):
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, rows, out, uneven)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    return dict(out)


@pytest.mark.parametrize("n,world", [(7, 2), (1, 2), (10, 3)])
def test_uneven_split_reduction(n, world):
    """all_gather of unequal per-rank blocks (7 seeds on 2 ranks, 1 seed on 2 ranks so one rank is
    empty, 10 on 3): counts first, pad, trim -- every rank sees all rows in seed order."""
    rng = np.random.default_rng(n)
    rows = np.stack([rng.lognormal(2, 0.5, n), rng.uniform(0, 0.2, n), rng.uniform(100, 200, n)], 1)
    out = _run_ranks(rows, world, True)
    single_rows, single_hist, single_cis = sharding.reduce_rows(rows, None)
    for r in range(world):
        all_rows, hist, cis = out[r]
        assert all_rows.shape == rows.shape and (all_rows == rows).all()
        assert (hist == single_hist).all() and cis == single_cis


def _hist_worker(rank, world, port, lat_all, cnt_all, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seeds = sharding.split_seeds(list(range(lat_all.shape[0])), rank, world)
    lat = lat_all[seeds].sum(0) if seeds else np.zeros(lat_all.shape[1:], np.int64)
    cnt = cnt_all[seeds].sum(0) if seeds else np.zeros(cnt_all.shape[1:], np.int64)
    out[rank] = sharding.reduce_tenant_hists(lat, cnt, dist)
    dist.destroy_process_group()


@pytest.mark.parametrize("n_seeds", [7, 1])
def test_two_rank_tenant_hists_equal_single_rank(n_seeds):
    """Per-(variant, tenant) latency histograms + completion/miss counters: the 2-rank all-reduce of
    per-seed-block sums equals the 1-rank sum (uneven and empty seed blocks included)."""
    rng = np.random.default_rng(11)
    lat_all = rng.integers(0, 1 << 40, size=(n_seeds, 3, 4, 2048), dtype=np.int64)
    cnt_all = rng.integers(0, 1 << 40, size=(n_seeds, 3, 4, 3), dtype=np.int64)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_hist_worker, args=(r, 2, port, lat_all, cnt_all, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    one = sharding.reduce_tenant_hists(lat_all.sum(0), cnt_all.sum(0), None)
    for r in range(2):
        lat, cnt = out[r]
        assert lat.dtype == np.int64 and (lat == one[0]).all() and (cnt == one[1]).all()


def test_pooled_quantiles_bracket_nearest_rank():
    """sharding.pooled_quantiles: the bin it returns for q holds the exact pooled nearest-rank
    q-quantile of the samples that were binned (telemetry.cpp:52-55 rule), incl. clamped end bins."""
    from oracle import restate
    from paper_2508_20274_b200.api import hist_bin_edges

    edges = hist_bin_edges()
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 1000, 54321):
        x = np.concatenate([rng.lognormal(1.5, 1.2, n), [1e-9, 5e7][: min(2, n // 500)]])
        hist = np.bincount(restate.lat_bins(x), minlength=restate.HIST_BINS)
        srt = np.sort(x)
        qs = (0.5, 0.95, 0.99, 0.999)
        for q, (lo, hi) in zip(qs, sharding.pooled_quantiles(hist, edges, qs)):
            k = min(max(int(np.ceil(q * len(x))), 1), len(x))
            v = srt[k - 1]
            assert lo <= v < hi, (n, q, v, lo, hi)
    assert all(np.isnan(a) for a in sharding.pooled_quantiles(np.zeros(restate.HIST_BINS, np.int64), edges)[0])
