"""Oracle test infrastructure: a scenarios directory for the compiled reference binaries
(oracle/_ref/acceptance_cpu, acceptance_gpu, shim_parity).  Their scenario loader is the restated
oracle/scenario_json.cpp (the reference's scenario.cpp needs yaml-cpp, absent here), which reads
the JSON form produced by oracle/yaml_to_json.py; each scenario-v1 file is written under its own
name so the reference's tests/acceptance.cpp finds default.yaml, llm.yaml, stability.yaml and
unstable.yaml unchanged.

  python -m oracle.json_scenarios <out_dir> <scenario.yaml>...
"""
from __future__ import annotations

import os
import sys

from oracle.yaml_to_json import yaml_file_to_json


def write_dir(out_dir: str, paths) -> str:
    os.makedirs(out_dir, exist_ok=True)
    for p in paths:
        with open(os.path.join(out_dir, os.path.basename(p)), "w") as f:
            f.write(yaml_file_to_json(p))
    return out_dir


if __name__ == "__main__":
    write_dir(sys.argv[1], sys.argv[2:])
