"""Decode tests/golden/golden.json (written by tools/make_golden.py from the
reference permkit). Floats are hex strings, ints decimal strings."""

from __future__ import annotations

import json
import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.json")


def load():
    with open(PATH) as f:
        return json.load(f)


def dec(v, kind):
    if kind == "integer":
        return int(v)
    if kind == "complex128":
        return complex(float.fromhex(v[0]), float.fromhex(v[1]))
    return float.fromhex(v)


def dec_dd(v):
    return (float.fromhex(v[0]), float.fromhex(v[1]))


def dense_array(case):
    m = case["matrix"]
    n, kind = m["n"], m["kind"]
    vals = [dec(v, kind) for v in m["data"]]
    if kind == "integer":
        return [vals[i * n:(i + 1) * n] for i in range(n)]
    dt = np.complex128 if kind == "complex128" else np.float64
    return np.array(vals, dtype=dt).reshape(n, n)


def triplets(case):
    m = case["matrix"]
    kind = m["kind"]
    if m["container"] == "sparse":
        return [(i, j, dec(v, kind)) for (i, j, v) in m["triplets"]]
    a = dense_array(case)
    n = m["n"]
    return [(i, j, a[i][j]) for i in range(n) for j in range(n) if a[i][j] != 0]


def cases(g, container=None, kind=None):
    out = []
    for c in g["cases"]:
        m = c["matrix"]
        if container and m["container"] != container:
            continue
        if kind and m["kind"] != kind:
            continue
        out.append(c)
    return out
