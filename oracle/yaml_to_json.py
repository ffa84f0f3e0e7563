"""Oracle test infrastructure: scenario-v1 YAML -> JSON bridge for the compiled reference.

The reference loads scenarios with yaml-cpp (`/root/reference/proj/src/scenario.cpp:322-374`),
which is absent from this image.  The oracle therefore parses YAML with PyYAML's
`BaseLoader` -- every scalar stays a *string*, exactly as yaml-cpp hands scalars to
`as<T>()` -- and `oracle/scenario_json.cpp` performs the typed conversion with
yaml-cpp's rules (`12e9` is a double for yaml-cpp even though YAML 1.1 would call it a
string).  Line numbers of every mapping key are kept under `"__line__"` so the
restated loader can report `file:line` like `scenario.cpp:100-106`.

This file is only used by tests/, bench.py's reference arm and smoke(): it is the
checker, never the product path.
"""
from __future__ import annotations

import json
import sys

import yaml


def _to_plain(node):
    """Convert a composed yaml node into JSON-able data with string scalars and line marks."""
    if isinstance(node, yaml.MappingNode):
        out = {"__line__": node.start_mark.line + 1, "__keys__": {}}
        for k, v in node.value:
            key = k.value
            out[key] = _to_plain(v)
            out["__keys__"][key] = k.start_mark.line + 1
        return out
    if isinstance(node, yaml.SequenceNode):
        return [_to_plain(v) for v in node.value]
    # ScalarNode: keep the raw text; yaml-cpp's as<T>() decides the type.
    return node.value


def yaml_text_to_json(text: str) -> str:
    node = yaml.compose(text, Loader=yaml.BaseLoader)
    if node is None:
        return json.dumps(None)
    return json.dumps(_to_plain(node))


def yaml_file_to_json(path: str) -> str:
    with open(path, "r", encoding="utf-8") as f:
        return yaml_text_to_json(f.read())


if __name__ == "__main__":
    sys.stdout.write(yaml_file_to_json(sys.argv[1]))
