"""GPU: the per-(variant, tenant) latency histograms and completion/miss counters the multi-GPU
reduction carries against the reference's own per-completion records.

The reference keeps every completion with keep_completions (engine.cpp:504); its measurement
window is `now >= measure_start_s` (engine.cpp:498-501).  Binning those window latencies with the
restated bins (oracle/restate.lat_bins) and summing over seeds per (variant, tenant) must give the
device histogram exactly; completed_total / completed_window / window_misses must equal the sums
of the reference's per-tenant summaries (engine.cpp:797-798)."""
import numpy as np
import pytest

from oracle import restate
from tests._libs import CONFIG_SCENARIOS, GOLDEN_SCENARIOS, ref_run
from tests.test_gpu_parity_wide import C4, _variants

pytestmark = pytest.mark.gpu


def _ref_hist(path, seeds, overrides, tids):
    T = len(tids)
    hist = np.zeros((T, restate.HIST_BINS), np.int64)
    counts = np.zeros((T, 3), np.int64)
    for seed in seeds:
        res, rc = ref_run(path, seed, overrides, keep_completions=True)
        summ = res["summary"]
        win = rc["done"] >= summ["measure_start_s"]
        for ti in range(T):
            s = summ["tenants"][tids[ti]]
            sel = win & (rc["tenant"] == ti)
            hist[ti] += np.bincount(restate.lat_bins(rc["total"][sel]), minlength=restate.HIST_BINS)
            misses = int((rc["total"][sel] > s["slo_tail_ms"]).sum())
            assert int(sel.sum()) == s["completed_window"]
            counts[ti] += (s["completed_total"], s["completed_window"], misses)
    return hist, counts


@pytest.mark.parametrize("path,variants", [(GOLDEN_SCENARIOS[0], C4), (CONFIG_SCENARIOS[1], C4[-1:])])
def test_latency_hist_matches_reference_completions(engine, path, variants):
    sid = engine.load_scenario(path)
    tids = engine.tenant_ids(sid)
    seeds = [3, 4, 5]
    res = engine.run_batch(sid, seeds, _variants(variants))
    try:
        lat, cnt = res.latency_hist(), res.tenant_counts()
    finally:
        res.close()
    assert lat.shape == (len(variants), len(tids), restate.HIST_BINS)
    for v, (_, ov) in enumerate(variants):
        h, c = _ref_hist(path, seeds, ov, tids)
        assert (lat[v] == h).all(), f"variant {variants[v][0]}: histogram differs"
        assert (cnt[v] == c).all(), f"variant {variants[v][0]}: counters differ {cnt[v]} vs {c}"
        # every window completion is in exactly one bin
        assert (lat[v].sum(1) == cnt[v][:, 1]).all()
    # the pooled tail (SURVEY 8(f)3 p999 extension) brackets the exact pooled nearest rank of the
    # reference's own window completions over all seeds
    from paper_2508_20274_b200 import sharding
    from paper_2508_20274_b200.api import hist_bin_edges

    edges = hist_bin_edges()
    for v, (_, ov) in enumerate(variants):
        pooled = {ti: [] for ti in range(len(tids))}
        for seed in seeds:
            r, rc = ref_run(path, seed, ov, keep_completions=True)
            win = rc["done"] >= r["summary"]["measure_start_s"]
            for ti in range(len(tids)):
                pooled[ti].append(rc["total"][win & (rc["tenant"] == ti)])
        for ti in range(len(tids)):
            vals = np.sort(np.concatenate(pooled[ti]))
            if len(vals) == 0:
                continue
            for q, (lo, hi) in zip((0.5, 0.99, 0.999), sharding.pooled_quantiles(lat[v, ti], edges, (0.5, 0.99, 0.999))):
                k = min(max(int(np.ceil(q * len(vals))), 1), len(vals))
                assert lo <= vals[k - 1] < hi, (variants[v][0], tids[ti], q)
