"""Batched admission control: Controller::admit (controller.cpp:637-692) as a
GPU kernel over many independent cases, bit-exact against the reference's own Controller::admit
(oracle/_ref) on the same states and snapshots -- outcomes, chosen (host, gpu, first), reason and
the chosen slot's placement_score."""
import ctypes
import os

import numpy as np
import pytest

from tests._libs import CONFIG_DIR, GOLDEN_SCENARIOS, oracle, scenario_json

C5 = os.path.join(CONFIG_DIR, "c5_mc64.yaml")
C2 = os.path.join(CONFIG_DIR, "c2_cluster16.yaml")


def _topology(path):
    """(tenant ids canonical, [(host, gpu id, total_slices)] in topology order, n_hosts)."""
    import json

    spec = json.loads(scenario_json(path))
    ids = sorted(t["id"] for t in spec["tenants"])
    gpus = []
    for h, host in enumerate(spec["topology"]["hosts"]):
        for g in host["gpus"]:
            gpus.append((h, int(g["id"]), int(g.get("total_slices", 7))))
    return ids, gpus, len(spec["topology"]["hosts"])


def random_cases(path, n, seed):
    """Random TenantStates + snapshots + requests over the scenario's topology."""
    ids, gpus, H = _topology(path)
    T = len(ids)
    rng = np.random.default_rng(seed)
    slices = np.array([1, 2, 3, 4, 7])
    c = {}
    c["tenant"] = rng.integers(0, T, n)
    c["profile"] = rng.integers(0, 5, n)
    c["admitted"] = (rng.random((n, T)) < rng.choice([0.3, 0.7, 0.95], (n, 1))).astype(np.int32)
    gi = rng.integers(0, len(gpus), (n, T))
    c["host"] = np.array([[gpus[k][0] for k in row] for row in gi], np.int32)
    c["gpu"] = np.array([[gpus[k][1] for k in row] for row in gi], np.int32)
    c["count"] = slices[rng.integers(0, 5, (n, T))].astype(np.int32)
    c["first"] = rng.integers(0, 7, (n, T)).astype(np.int32)
    pcie = rng.lognormal(20.0, 2.0, (n, T)) * (rng.random((n, T)) < 0.6)
    hio = rng.lognormal(17.0, 2.0, (n, T)) * (rng.random((n, T)) < 0.6)
    c["pcie"] = np.where(rng.random((n, T)) < 0.05, 0.0, pcie)
    c["hio"] = hio
    c["irq"] = (rng.random((n, H)) < 0.3).astype(np.uint32) * rng.integers(1, 4, (n, H)).astype(np.uint32)
    # a slice of easy cases: nobody admitted, or the request's own rate far below service
    c["admitted"][: n // 20] = 0
    return c


def ref_admit(path, c):
    n = len(c["tenant"])
    arrs = [np.ascontiguousarray(c[k], dt) for k, dt in
            (("tenant", np.int32), ("profile", np.int32), ("admitted", np.int32), ("host", np.int32),
             ("gpu", np.int32), ("first", np.int32), ("count", np.int32), ("pcie", np.float64),
             ("hio", np.float64), ("irq", np.uint32))]
    out = np.zeros((n, 6), np.int32)
    score = np.zeros(n, np.float64)
    lib = oracle()
    assert lib.ref_admit(scenario_json(path), n, *[a.ctypes.data for a in arrs], out.ctypes.data,
                         score.ctypes.data) == 0, lib.ref_last_error()
    return out, score


def test_reference_admission_oracle_sane():
    """The oracle wrapper around the reference's Controller::admit: empty clusters admit at the
    leftmost slot of the best-scoring GPU; overloaded requests are rejected for the service rate."""
    c = random_cases(C2, 400, 3)
    out, score = ref_admit(C2, c)
    assert set(np.unique(out[:, 0])) <= {0, 1, 2}
    assert (out[:, 0] == 0).sum() > 50 and (out[:, 0] != 0).sum() > 5
    empty = c["admitted"].sum(1) == 0
    ok = empty & (out[:, 0] == 0)
    assert ok.any() and (out[ok, 3] == 0).all()
    assert (out[out[:, 0] == 2, 5] != 0).all()


@pytest.mark.gpu
@pytest.mark.parametrize("path,n,seed", [(C2, 20000, 1), (C5, 20000, 2), (GOLDEN_SCENARIOS[0], 5000, 3)])
def test_gpu_admission_bit_exact(engine, path, n, seed):
    c = random_cases(path, n, seed)
    ref, rscore = ref_admit(path, c)
    sid = engine.load_scenario(path)
    mine, ms = engine.admit(sid, c["tenant"], c["profile"], c["admitted"], c["host"], c["gpu"], c["first"],
                            c["count"], c["pcie"], c["hio"], c["irq"])
    assert ms > 0
    assert (mine["outcome"] == ref[:, 0]).all()
    adm = ref[:, 0] == 0
    assert (mine["host"][adm] == ref[adm, 1]).all()
    assert (mine["gpu"][adm] == ref[adm, 2]).all()
    assert (mine["first"][adm] == ref[adm, 3]).all()
    assert (mine["count"][adm] == ref[adm, 4]).all()
    assert (mine["reason"] == ref[:, 5]).all()
    assert (mine["score"][adm].view(np.uint64) == rscore[adm].view(np.uint64)).all()
    assert adm.sum() > n // 10 and (~adm).sum() > 0


def ref_admit_repeat(path, c, repeat):
    n = len(c["tenant"])
    arrs = [np.ascontiguousarray(c[k], dt) for k, dt in
            (("tenant", np.int32), ("profile", np.int32), ("admitted", np.int32), ("host", np.int32),
             ("gpu", np.int32), ("first", np.int32), ("count", np.int32), ("pcie", np.float64),
             ("hio", np.float64), ("irq", np.uint32))]
    out = np.zeros((n, repeat, 6), np.int32)
    score = np.zeros((n, repeat), np.float64)
    lib = oracle()
    lib.ref_admit_repeat.argtypes = [ctypes.c_char_p, ctypes.c_int] + [ctypes.c_void_p] * 10 + [
        ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    assert lib.ref_admit_repeat(scenario_json(path), n, *[a.ctypes.data for a in arrs], repeat, out.ctypes.data,
                                score.ctypes.data) == 0, lib.ref_last_error()
    return out, score


def crowded_cases(path, n, seed):
    """Every GPU holds an admitted tenant (T >= G), so a 7g request has no free run and queues;
    a quarter of the cases ask for 1g and are admitted."""
    ids, gpus, H = _topology(path)
    T = len(ids)
    c = random_cases(path, n, seed)
    rng = np.random.default_rng(seed + 100)
    gi = np.tile(np.arange(T) % len(gpus), (n, 1))
    c["host"] = np.array([[gpus[k][0] for k in row] for row in gi], np.int32)
    c["gpu"] = np.array([[gpus[k][1] for k in row] for row in gi], np.int32)
    c["count"] = np.ones((n, T), np.int32)
    c["first"] = np.where(np.arange(T) < len(gpus), 0, 1).astype(np.int32)[None, :].repeat(n, 0)
    c["admitted"] = np.ones((n, T), np.int32)
    c["profile"] = np.where(rng.random(n) < 0.25, 0, 4).astype(np.int32)
    return c


def test_reference_queue_timeout_semantics():
    """Oracle: with no feasible slot the same request is queued for admission_queue_timeout_epochs
    retries, rejected on the next (reason: timeout), then the queue restarts (controller.cpp:677-691)."""
    c = crowded_cases(C5, 600, 7)
    out, _ = ref_admit_repeat(C5, c, 13)
    queued_first = out[:, 0, 0] == 1
    assert queued_first.sum() > 20
    q = out[queued_first]
    assert (q[:, :10, 0] == 1).all() and (q[:, 10, 0] == 2).all() and (q[:, 10, 5] == 3).all()
    assert (q[:, 11, 0] == 1).all()


@pytest.mark.gpu
@pytest.mark.parametrize("path,n,seed,crowded", [(C2, 4000, 11, False), (C5, 3000, 12, True), (C5, 3000, 13, False)])
def test_gpu_admission_stateful_retries(engine, path, n, seed, crowded):
    """Retry epochs carried across GPU calls in queue_epochs (in/out) give the reference's decision
    sequence for the same request repeated on one controller, bit-exact: queued x timeout, the
    timeout rejection, the queue restarting; admitted requests clear the entry."""
    repeat = 13
    c = crowded_cases(path, n, seed) if crowded else random_cases(path, n, seed)
    ref, rscore = ref_admit_repeat(path, c, repeat)
    sid = engine.load_scenario(path)
    qe = np.zeros(n, np.int32)
    for r in range(repeat):
        mine, _ = engine.admit(sid, c["tenant"], c["profile"], c["admitted"], c["host"], c["gpu"], c["first"],
                               c["count"], c["pcie"], c["hio"], c["irq"], queue_epochs=qe)
        assert (mine["outcome"] == ref[:, r, 0]).all(), r
        assert (mine["reason"] == ref[:, r, 5]).all(), r
        adm = ref[:, r, 0] == 0
        assert (mine["first"][adm] == ref[adm, r, 3]).all()
        assert (mine["score"][adm].view(np.uint64) == rscore[adm, r].view(np.uint64)).all()
        # the carried state itself: 0 after admission/rejection, the retry count while queued
        want = np.where(ref[:, r, 0] == 1, (r % 11) + 1, 0)
        assert (qe[ref[:, r, 5] != 1] == want[ref[:, r, 5] != 1]).all(), r
    if crowded:
        assert (ref[:, 10, 5] == 3).sum() > n // 2
