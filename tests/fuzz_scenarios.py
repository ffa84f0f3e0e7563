"""Randomised scenario-v1 generator for differential fuzzing of the engine against the reference.

Each seed yields a valid scenario that stresses paths the four shipped scenarios leave cold:
deterministic clocks (cv = 0), zero-byte and empty transfer mixes, phase / square-wave thinning,
uncapped and capped flows with and without water filling, non-MIG (MPS) devices, IRQ bursts,
aggressive controller settings (short dwell, low thresholds, tiny validation windows) so that
guardrails, moves, MIG up/down, rollbacks, expiries and drain timeouts all fire.
"""
from __future__ import annotations

import random

PRESETS = ["t1-inference", "t2-etl", "t3-train", "llm-ttft"]
PROFILES = [("1g.10gb", 1), ("2g.20gb", 2), ("3g.40gb", 3), ("4g.40gb", 4), ("7g.80gb", 7)]


def _sched(rng: random.Random) -> str:
    k = rng.random()
    if k < 0.55:
        return ""
    if k < 0.8:
        return (f"    schedule: {{ kind: square_wave, period_s: {rng.choice([20, 37.5, 60, 90])}, "
                f"duty: {rng.choice([0.0, 0.3, 0.5, 1.0])}, offset_s: {rng.choice([0, 5, 12.5])} }}\n")
    a = rng.uniform(0, 60)
    b = a + rng.uniform(5, 80)
    c = b + rng.uniform(5, 40)
    return (f"    schedule:\n      kind: phases\n      phases:\n        - {{ start_s: {a:.3f}, end_s: {b:.3f} }}\n"
            f"        - {{ start_s: {c:.3f}, end_s: {c + rng.uniform(10, 90):.3f} }}\n")


def make_scenario(seed: int, wide: bool = False, xwide: bool = False) -> str:
    """One random scenario-v1 document.  wide=True: 11-40 tenants on up to 4 hosts x 8 GPUs (the
    engine's T > 10 code path: event slots in shared memory).  xwide=True: 41-64 tenants on 4-5
    hosts x 8 GPUs (up to the engine's 64-tenant limit: 64-bit tenant masks, controller rings in
    global memory)."""
    rng = random.Random(seed)
    wide = wide or xwide
    n_hosts = rng.choice([4, 5]) if xwide else rng.choice([2, 3, 4]) if wide else rng.choice([1, 1, 2])
    hosts, gpus_of = [], []
    for h in range(n_hosts):
        n_roots = rng.choice([1, 2, 3])
        n_gpus = 8 if xwide else rng.choice([6, 8]) if wide else rng.choice([2, 3, 4])
        roots = "\n".join(f"        - {{ id: {r * 3 + 1}, capacity_Bps: {rng.choice(['8e9', '12e9', '16e9', '24e9'])} }}"
                          for r in range(n_roots))
        gl = []
        for g in range(n_gpus):
            mig = "" if rng.random() < 0.75 else ", mig_enabled: false"
            gl.append(f"        - {{ id: {g * 2}, pcie_root_id: {rng.randrange(n_roots) * 3 + 1}, numa_id: {g % 2}, "
                      f"core_group: {rng.randrange(3)}{mig} }}")
            gpus_of.append((h, g * 2, mig != ""))
        hosts.append(f"    - numa_domains: 2\n      io_capacity_Bps: {rng.choice(['3e8', '6e8', '1e9'])}\n"
                     f"      pcie_roots:\n{roots}\n      gpus:\n" + "\n".join(gl))
    # tenants: pack slices per GPU without overlap
    used = {}
    tenants = []
    n_t = rng.randint(41, 64) if xwide else rng.randint(11, 40) if wide else rng.randint(2, 7)
    for t in range(n_t):
        for _ in range(20):
            h, g, nomig = rng.choice(gpus_of)
            pname, pslices = rng.choice(PROFILES[:2] if xwide else PROFILES[:4])
            first = rng.randrange(0, 7 - pslices + 1)
            occ = used.setdefault((h, g), set())
            rngs = set(range(first, first + pslices))
            if nomig or not (occ & rngs):
                occ |= rngs
                break
        else:
            continue
        preset = rng.choice(PRESETS)
        tid = rng.choice(["a", "b", "c", "t", "x", "z", "llm", "etl"]) + str(t) + rng.choice(["", "0", "_1"])
        extra = []
        if rng.random() < 0.5:
            extra.append(f"    arrival_rate_hz: {rng.choice([2, 5, 12.5, 30, 60])}")
        if rng.random() < 0.25:
            extra.append(f"    arrival_cv: {rng.choice([0, 0.5, 1.0, 1.5])}")
        if rng.random() < 0.25:
            mix = rng.choice(["[]", "[{ bytes: 0 }]", "[{ bytes: 0, weight: 1 }, { bytes: 3e6, weight: 2 }]",
                              "[{ bytes: 5e8 }, { bytes: 1e6, weight: 3 }]"])
            extra.append(f"    transfer_mix: {mix}")
        if rng.random() < 0.3:
            extra.append(f"    service_cv: {rng.choice([0, 0.2, 0.6])}")
        if rng.random() < 0.3:
            extra.append(f"    noise_mean_ms: {rng.choice([0, 0.3, 2])}")
        if rng.random() < 0.4:
            extra.append(f"    slo_tail_ms: {rng.choice([5, 10, 20, 80, 400])}")
        if rng.random() < 0.3:
            extra.append(f"    pcie_cap_Bps: {rng.choice([0, 1e9, 4e9])}")
        if rng.random() < 0.2:
            extra.append(f"    weight: {rng.choice([0.5, 1, 2, 4])}")
        if rng.random() < 0.2:
            extra.append(f"    class: {rng.choice(['latency_sensitive', 'bandwidth_heavy', 'compute_heavy'])}")
        body = "\n".join(extra) + ("\n" if extra else "")
        tenants.append(f"  - preset: {preset}\n    id: {tid}\n{body}"
                       f"    placement: {{ host: {h}, gpu: {g}, profile: {pname}, first_slice: {first} }}\n{_sched(rng)}")
    # unique ids
    seen = set()
    out_t = []
    for t in tenants:
        tid = t.split("id: ")[1].split("\n")[0]
        if tid in seen:
            continue
        seen.add(tid)
        out_t.append(t)
    irq = ""
    if rng.random() < 0.6:
        irq = "irq_bursts:\n" + "".join(
            f"  - host: {rng.randrange(n_hosts)}\n    core_group: {rng.randrange(3)}\n"
            f"    extra_noise_ms: {rng.choice([0, 1.5, 4])}\n"
            f"    schedule: {{ kind: square_wave, period_s: {rng.choice([30, 45])}, duty: 0.4 }}\n"
            for _ in range(rng.randint(1, 2)))
    duration = rng.choice([120, 200, 300])
    ctrl = [f"  sample_interval_s: {rng.choice([1, 2, 3.5])}", f"  warmup_s: {rng.choice([5, 20])}",
            f"  dwell_obs: {rng.choice([16, 32, 64, 256])}", f"  cooldown_obs: {rng.choice([0, 8, 64])}",
            f"  validation_obs: {rng.choice([4, 16, 64])}", f"  persistence_windows: {rng.choice([1, 2, 3])}",
            f"  relax_stability_ratio: {rng.choice([0.5, 0.8, 0.95])}",
            f"  relax_score_threshold: {rng.choice([0.3, 2.5])}", f"  move_margin: {rng.choice([0.0, 0.25])}",
            f"  diag_pcie_util_threshold: {rng.choice([0.1, 0.8])}",
            f"  diag_host_io_threshold: {rng.choice([0.05, 0.8])}",
            f"  diag_sm_util_threshold: {rng.choice([0.05, 0.7])}",
            f"  throttle_duration_s: {rng.choice([5, 30])}", f"  quota_duration_s: {rng.choice([5, 30])}"]
    if rng.random() < 0.2:
        ctrl.append("  enabled: false")
    return (f"version: scenario-v1\nname: fuzz-{seed}\nduration_s: {duration}\nmeasure_start_s: {duration // 3}\n"
            f"fabric:\n  redistribute: {rng.choice(['true', 'false'])}\n"
            f"topology:\n  hosts:\n" + "\n".join(hosts) + "\n"
            "tenants:\n" + "".join(out_t) + irq + "controller:\n" + "\n".join(ctrl) + "\n")
