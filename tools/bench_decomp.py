"""Time the decomposition path end to end: this
package's decomp_run (host worklist + batched GPU leaves) against the
reference's own decomp_run (pure-Python worklist + one numba kernel call per
leaf) on the same matrices, on the same box.

    python tools/bench_decomp.py [--reference]

Matrices: random sparse matrices of the kind/size/density below (the
generator of tools/make_golden_preprocess.py, seeds fixed). Prints one JSON
line per case. The reference leg imports permkit from baseline/_ref (the
offline install) and is skipped when it is absent.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [("real20_d30", 20, 0.30, "real64", 20261017 + 9),
         ("int20_d30", 20, 0.30, "integer", 20261017 + 11),
         ("cplx18_d30", 18, 0.30, "complex128", 20261017 + 12),
         ("real24_d28", 24, 0.28, "real64", 7)]


def triplets(n, density, seed, kind):
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    out = []
    for i in range(n):
        for j in range(n):
            if j == perm[i] or rng.random() < density:
                if kind == "integer":
                    v = int(rng.integers(1, 4))
                elif kind == "complex128":
                    v = complex(rng.uniform(-1, 1), rng.uniform(-1, 1))
                else:
                    v = float(rng.uniform(0.0, 1.0))
                out.append((i, j, v))
    return out


def ours(trip, n, kind, policy):
    import paper_2502_16577_b200 as pk
    s = pk.sparse_from_triplets(n, trip, kind)
    pk.perm_nw(pk.random_real(16, 1), "kahan")  # device context + kernels warm
    pk.decomp_run(pk.sparse_from_triplets(4, [(i, i, 1) for i in range(4)], "integer"))
    t0 = time.perf_counter()
    val, st = pk.decomp_run(s, policy)
    dt = time.perf_counter() - t0
    return val, dt, st


def reference(trip, n, kind, policy):
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_pk")
    import permkit.preprocess as pp
    from permkit.matrix import sparse_from_triplets
    from permkit.precision import AccumulatorPolicy
    s = sparse_from_triplets(n, trip, kind=kind)
    # warm the numba kernels on a tiny matrix of the same kind
    pp.decomp_run(sparse_from_triplets(12, [(i, j, trip[0][2]) for i in range(12)
                                            for j in range(12)], kind=kind),
                  AccumulatorPolicy.parse(policy))
    t0 = time.perf_counter()
    val, st = pp.decomp_run(s, AccumulatorPolicy.parse(policy))
    return val, time.perf_counter() - t0, st


def enc(v):
    if isinstance(v, complex):
        return [v.real.hex(), v.imag.hex()]
    if isinstance(v, int):
        return str(v)
    return float(v).hex()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference", action="store_true", help="also time permkit's decomp_run")
    a = ap.parse_args()
    for name, n, d, kind, seed in CASES:
        trip = triplets(n, d, seed, kind)
        pol = "dd" if kind == "complex128" else "kahan"
        v, dt, st = ours(trip, n, kind, pol)
        line = {"case": name, "n": n, "kind": kind, "policy": pol, "tasks": st.tasks_created,
                "kernel_leaves": st.kernel_leaves, "leaf_launches": st.leaf_launches,
                "b200_s": dt, "value": enc(v)}
        if a.reference and os.path.isdir(os.path.join(ROOT, "baseline", "_ref")):
            rv, rdt, rst = reference(trip, n, kind, pol)
            line.update({"reference_s": rdt, "reference_value": enc(rv), "speedup": rdt / dt,
                         "reference_tasks": rst.tasks_created,
                         "agree": (rv == v) if kind == "integer"
                         else abs(rv - v) <= 1e-10 * abs(rv) + 1e-300})
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
