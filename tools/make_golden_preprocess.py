"""Generate tests/golden/preprocess.json by running the REFERENCE's
structural preprocessing (permkit.preprocess) on small sparse matrices.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=baseline/_ref \
        python tools/make_golden_preprocess.py

Recorded per case (all from permkit's public functions):
  * dm_filter: the filtered triplets (or the singular verdict), nnz before/after
  * min_nnz_row_col and d1/d2/d34 compressions of the sparsest row/column
  * decomp_run: every kernel leaf in evaluation order (n, triplets, multiplier,
    task id -- recorded by wrapping permkit's leaf kernels), the statistics and
    the final value under the KAHAN policy
Floats are hex strings, integers decimal strings, complex [re, im] hex pairs.
The GPU box never reads /root/reference; tests only read this JSON.
"""

from __future__ import annotations

import json
import os

import numpy as np

import permkit
import permkit.preprocess as pp
from permkit.matrix import sparse_from_triplets
from permkit.precision import AccumulatorPolicy

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden", "preprocess.json")
SEED = 20261017


def enc(v):
    if isinstance(v, bool):
        raise TypeError
    if isinstance(v, int):
        return str(v)
    if isinstance(v, complex):
        return [v.real.hex(), v.imag.hex()]
    return float(v).hex()


def enc_trips(trips):
    return [[int(i), int(j), enc(v)] for (i, j, v) in trips]


def rand_sparse(n, density, seed, kind):
    rng = np.random.default_rng(seed)
    trips = []
    # a permuted diagonal keeps most cases non-singular
    perm = rng.permutation(n)
    for i in range(n):
        for j in range(n):
            if j == perm[i] or rng.random() < density:
                if kind == "integer":
                    v = int(rng.integers(1, 4))
                elif kind == "complex128":
                    v = complex(rng.uniform(-1, 1), rng.uniform(-1, 1))
                else:
                    v = float(rng.uniform(0.0, 1.0))
                trips.append((i, j, v))
    return sparse_from_triplets(n, trips, kind=kind)


def singular_case(n):
    # two rows supported on the same single column: no perfect matching
    trips = [(0, 0, 1), (1, 0, 1)] + [(i, i, 1) for i in range(2, n)] + [(i, (i + 1) % n, 2)
                                                                         for i in range(2, n)]
    return sparse_from_triplets(n, trips, kind="integer")


def block_case():
    # block upper-triangular: the off-diagonal block lies on no permutation
    n = 10
    rng = np.random.default_rng(7)
    trips = []
    for i in range(n):
        for j in range(n):
            same = (i < 5) == (j < 5)
            upper = i < 5 <= j
            if (same and rng.random() < 0.6) or i == j or (upper and rng.random() < 0.5):
                trips.append((i, j, float(rng.uniform(0.1, 1.0))))
    return sparse_from_triplets(n, trips, kind="real64")


def record_leaves():
    leaves = []
    orig_nw, orig_spa = pp.perm_nw, pp.perm_spa

    def nw(m, policy=AccumulatorPolicy.DD):
        v = orig_nw(m, policy)
        leaves.append({"via": "nw", "n": m.n,
                       "triplets": enc_trips([(i, j, m.entry(i, j)) for i in range(m.n)
                                              for j in range(m.n) if m.entry(i, j) != 0]),
                       "value": enc(v)})
        return v

    def spa(s, policy=AccumulatorPolicy.DD):
        v = orig_spa(s, policy)
        leaves.append({"via": "spa", "n": s.n, "triplets": enc_trips(s.crs.triplets()),
                       "value": enc(v)})
        return v

    pp.perm_nw, pp.perm_spa = nw, spa
    return leaves, (orig_nw, orig_spa)


def case_record(name, s, policy="kahan"):
    rec = {"name": name, "n": s.n, "kind": s.kind, "triplets": enc_trips(s.crs.triplets())}
    res = pp.dm_filter(s)
    if isinstance(res, pp.SingularVerdict):
        rec["dm_filter"] = {"singular": True}
    else:
        rec["dm_filter"] = {"singular": False, "nnz_after": res.crs.nnz,
                            "triplets": enc_trips(res.crs.triplets())}
    pick = pp.min_nnz_row_col(s)
    rec["min_nnz"] = [pick.axis, pick.index, pick.count]
    comp = {}
    for axis in ("row", "col"):
        for idx in range(s.n):
            cnt = (s.crs.rptrs[idx + 1] - s.crs.rptrs[idx] if axis == "row"
                   else s.ccs.cptrs[idx + 1] - s.ccs.cptrs[idx])
            key = f"{axis}{idx}"
            if cnt == 1 and "d1" not in comp:
                a, minor = pp.d1compress(s, axis, idx)
                comp["d1"] = {"axis": axis, "index": idx, "alpha": enc(a),
                              "triplets": enc_trips(minor.crs.triplets())}
            elif cnt == 2 and "d2" not in comp:
                f = pp.d2compress(s, axis, idx)
                comp["d2"] = {"axis": axis, "index": idx, "triplets": enc_trips(f.crs.triplets())}
            elif cnt >= 3 and "d34_" + axis not in comp:
                z, f = pp.d34compress(s, axis, idx)
                comp["d34_" + axis] = {"axis": axis, "index": idx,
                                       "zeroed": enc_trips(z.crs.triplets()),
                                       "folded": enc_trips(f.crs.triplets())}
    rec["compress"] = comp
    leaves, orig = record_leaves()
    try:
        val, st = pp.decomp_run(s, AccumulatorPolicy.parse(policy))
    finally:
        pp.perm_nw, pp.perm_spa = orig
    # full leaf matrices for the first leaves, values for all (evaluation order)
    for lf in leaves[40:]:
        lf.pop("triplets")
    rec["decomp"] = {"policy": policy, "value": enc(val), "leaves": leaves,
                     "stats": {k: getattr(st, k) for k in
                               ("tasks_created", "d1_applied", "d2_applied", "d34_applied",
                                "trivial_leaves", "kernel_leaves", "dense_kernel_leaves",
                                "max_depth")}}
    return rec


def main():
    cases = []
    specs = [("int14_d15", 14, 0.15, "integer"), ("int18_d12", 18, 0.12, "integer"),
             ("int22_d10", 22, 0.10, "integer"), ("real16_d20", 16, 0.20, "real64"),
             ("real20_d12", 20, 0.12, "real64"), ("real24_d15", 24, 0.15, "real64"),
             ("cplx14_d20", 14, 0.20, "complex128"), ("int26_d35", 26, 0.35, "integer"),
             ("real28_d30", 28, 0.30, "real64"), ("real18_d33", 18, 0.33, "real64"),
             ("int20_d30", 20, 0.30, "integer"), ("cplx18_d30", 18, 0.30, "complex128"),
             ("real17_d40", 17, 0.40, "real64")]
    for k, (name, n, d, kind) in enumerate(specs):
        s = rand_sparse(n, d, SEED + k, kind)
        cases.append(case_record(name, s, "dd" if kind == "complex128" else "kahan"))
        print(name, cases[-1]["decomp"]["stats"], len(cases[-1]["decomp"]["leaves"]), flush=True)
    cases.append(case_record("singular12", singular_case(12)))
    cases.append(case_record("block10", block_case()))
    with open(OUT, "w") as f:
        json.dump({"generator": "tools/make_golden_preprocess.py", "reference": "permkit " +
                   getattr(permkit, "__version__", "?"), "cases": cases}, f, separators=(",", ":"))
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
