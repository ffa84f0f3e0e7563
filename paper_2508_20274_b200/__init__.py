"""migsim-b200: a B200-native batched engine for the arXiv 2508.20274 reference's replica hot path
(batched evaluation of the MIG/PCIe-aware multi-tenancy controller over scenarios x seeds).

Public API mirrors the reference (engine::run_scenario, harness::run_plan); execution is the
sm_100a CUDA engine behind the C-ABI in include/migsim_b200.h.
"""
from .api import (  # noqa: F401
    BatchResult,
    ConfigError,
    Engine,
    ParityGuardError,
    Variant,
    ablation_variants,
    load_library,
    main_variants,
    render_report,
    run_plan,
    run_scenario,
)

__all__ = [
    "BatchResult",
    "ConfigError",
    "Engine",
    "ParityGuardError",
    "Variant",
    "ablation_variants",
    "load_library",
    "main_variants",
    "render_report",
    "run_plan",
    "run_scenario",
]
