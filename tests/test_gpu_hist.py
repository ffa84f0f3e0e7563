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
