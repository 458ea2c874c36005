"""Load the flattened golden fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def _insert(root, parts, value):
    node = root
    for p in parts[:-1]:
        node = node.setdefault(p, {})
    node[parts[-1]] = value


def _listify(node):
    if not isinstance(node, dict):
        return node
    if "__len__" in node:
        n = int(node["__len__"])
        return [_listify(node[str(i)]) for i in range(n)]
    if "__none__" in node and len(node) == 1:
        return None
    return {k: _listify(v) for k, v in node.items()}


def load(name):
    z = np.load(GOLDEN / f"golden_{name}.npz")
    root = {}
    for key in z.files:
        _insert(root, key.split("."), z[key])
    return _listify(root)
