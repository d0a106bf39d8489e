"""Generate tests/golden/golden.json by running the REFERENCE (permkit).

Run here, where the reference is importable (baseline/_ref is the pip
--target install of /root/reference/pkg):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=baseline/_ref \
        python tools/make_golden.py

Every value comes from permkit's own public API (perm_nw, perm_spa,
run_range, permanent_chunked, initial_product). Floats are stored as hex so
comparisons are bit exact; integers as decimal strings. The GPU box never
reads /root/reference -- the tests only read this JSON.
"""

from __future__ import annotations

import json
import os
import random
import sys
import time

import numpy as np

import permkit
from permkit.kernels import perm_nw, perm_spa, total_iterates
from permkit.matrix import DenseMatrix, dense_to_sparse, sparse_from_triplets
from permkit.parallel import initial_product, permanent_chunked, run_range
from permkit.precision import AccumulatorPolicy

SEED = 20261017
POL = {p.value: p for p in AccumulatorPolicy}
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden", "golden.json")

TERNARY12 = (
    (-1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1),
    (0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, -1),
    (-1, 0, -1, 1, 0, 0, 0, 1, 0, 1, 1, 0),
    (1, 0, 0, 1, 0, -1, 0, -1, 0, -1, 1, 0),
    (0, 1, 1, 0, -1, 0, 0, 0, 0, 0, 0, 0),
    (0, 0, 0, 1, 0, 1, 0, 0, 0, 1, 0, -1),
    (0, 1, 0, 0, 0, 0, 1, 1, 0, 0, -1, 0),
    (0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, -1),
    (0, 0, 0, 1, 0, 1, 0, -1, 0, 1, 1, 0),
    (0, 0, 0, 1, 0, 0, 0, 1, 1, 0, 0, -1),
    (1, 0, 1, 0, 0, -1, -1, 0, 0, 0, 0, 0),
    (-1, 0, 1, 0, 0, 0, 1, 0, 1, 0, 1, -1),
)
DEMO6 = ((0, 0), (0, 2), (1, 0), (1, 1), (2, 1), (2, 2), (3, 0), (3, 3), (3, 5), (4, 2),
         (4, 4), (5, 1), (5, 5))


def enc(v):
    if isinstance(v, bool):
        raise TypeError
    if isinstance(v, int):
        return str(v)
    if isinstance(v, complex):
        return [v.real.hex(), v.imag.hex()]
    if isinstance(v, float):
        return v.hex()
    if hasattr(v, "hi"):
        return [v.hi.hex(), v.lo.hex()]
    raise TypeError(type(v))


def enc_matrix(m):
    if isinstance(m, DenseMatrix):
        return {"container": "dense", "n": m.n, "kind": m.kind, "data": [enc(v) for v in m.data]}
    trips = m.crs.triplets()
    return {"container": "sparse", "n": m.n, "kind": m.kind,
            "triplets": [[i, j, enc(v)] for (i, j, v) in trips]}


def haar_block(n, seed):
    """U(M)[:n,:n] with M = n^2, Mezzadri's QR recipe."""
    M = n * n
    rng = np.random.default_rng(seed)
    z = (rng.standard_normal((M, M)) + 1j * rng.standard_normal((M, M))) / np.sqrt(2.0)
    q, r = np.linalg.qr(z)
    d = np.diagonal(r)
    u = q * (d / np.abs(d))
    return DenseMatrix.from_rows([[complex(v) for v in row] for row in u[:n, :n]])


def rand_dense(n, seed, kind):
    rng = random.Random(seed)
    if kind == "integer":
        rows = [[rng.randint(-9, 9) for _ in range(n)] for _ in range(n)]
    elif kind == "complex128":
        rows = [[complex(rng.uniform(-3, 3), rng.uniform(-3, 3)) for _ in range(n)] for _ in range(n)]
    else:
        rows = [[rng.uniform(-4.0, 4.0) for _ in range(n)] for _ in range(n)]
    return DenseMatrix.from_rows(rows)


def sample_ranges(n, seed):
    T = total_iterates(n)
    rng = random.Random(seed)
    rs = {(1, T), (1, 1), (T, T)}
    if T >= 4:
        rs.add((2, T - 1))
    for k in (2, 5, 9, 12):
        size = 1 << k
        if size * 2 <= T:
            for c in (0, 1, (T // size) - 1):
                s = 1 + c * size
                rs.add((s, min(T, s + size - 1)))
    for _ in range(4):
        a = rng.randint(1, T)
        b = rng.randint(a, min(T, a + 5000))
        rs.add((a, b))
    return sorted(rs)


def case(name, m, policies, taus, ranges_seed, serial=True):
    t0 = time.time()
    n = m.n
    d = {"name": name, "matrix": enc_matrix(m)}
    sparse = not isinstance(m, DenseMatrix)
    if serial:
        d["serial"] = {}
        for p in policies:
            d["serial"][p] = enc(perm_spa(m, POL[p]) if sparse else perm_nw(m, POL[p]))
    d["p0"] = {p: enc(initial_product(m, POL[p])) for p in policies}
    d["chunked"] = []
    for p in policies:
        for tau in taus:
            for aligned in ((True, False) if tau in (3, 7) else (True,)):
                v = permanent_chunked(m, POL[p], tau=tau, aligned=aligned)
                d["chunked"].append({"policy": p, "tau": tau, "aligned": aligned, "value": enc(v)})
    d["ranges"] = []
    if total_iterates(n) >= 1:
        rr = sample_ranges(n, ranges_seed)
        T = total_iterates(n)
        # whole-walk ranges are already covered by "serial" for big n
        for p in policies:
            for (s, e) in rr:
                if e - s > 3_000_000 and m.kind == "integer":
                    continue
                pr = run_range(m, s, e, POL[p], worker_id=0)
                d["ranges"].append({"policy": p, "start": s, "end": e, "value": enc(pr.value)})
    print(f"{name}: n={n} {time.time() - t0:.1f}s", file=sys.stderr, flush=True)
    return d


def main():
    allp = ["dd", "kahan", "dq", "qq"]
    cases = []
    # dense real
    cases.append(case("real_rand8", rand_dense(8, 108, "real64"), allp, [1, 3, 7, 16], 1))
    cases.append(case("real_unit12", permkit.random_real(12, 7, -1.0, 1.0), allp, [1, 3, 64], 2))
    cases.append(case("config1_real20", permkit.random_real(20, SEED, 0.0, 1.0), allp, [1, 7, 64], 3))
    # n >= 24: long reference chunks let the per-row state drift (tau=64 at
    # n=28 is off by 3.6e-10); tau=65536 (short chunks) is the accurate anchor
    cases.append(case("real24", permkit.random_real(24, SEED, 0.0, 1.0), allp, [64, 65536], 4,
                      serial=False))
    cases.append(case("real28", permkit.random_real(28, SEED, 0.0, 1.0), ["kahan", "dq"],
                      [64, 65536], 5, serial=False))
    cases.append(case("ternary12_real",
                      DenseMatrix.from_rows([[float(v) for v in r] for r in TERNARY12]), allp,
                      [1, 2, 7, 32], 6))
    cases.append(case("uniform16_091", permkit.uniform(16, 0.91), allp, [1, 64], 7))
    # dense complex (DD only in the reference)
    cases.append(case("cplx_rand6", rand_dense(6, 206, "complex128"), ["dd"], [1, 3], 8))
    cases.append(case("cplx_rand12", rand_dense(12, 212, "complex128"), ["dd"], [1, 7, 64], 9))
    cases.append(case("haar16", haar_block(16, SEED), ["dd"], [1, 64, 4096], 10))
    cases.append(case("haar24", haar_block(24, SEED), ["dd"], [4096], 11, serial=False))
    # dense integer
    cases.append(case("int_rand8", rand_dense(8, 308, "integer"), ["dd"], [1, 3, 7], 12))
    cases.append(case("int_rand12", rand_dense(12, 312, "integer"), ["dd"], [1, 16], 13))
    cases.append(case("ternary12_int", DenseMatrix.from_rows([list(r) for r in TERNARY12]), ["dd"],
                      [1, 7], 14))
    cases.append(case("binary16", permkit.random_binary(16, SEED, 0.3), ["dd"], [1, 8], 15))
    cases.append(case("binary20_dense", permkit.random_binary(20, SEED, 0.5), ["dd"], [8], 16,
                      serial=False))
    # sparse
    demo6 = sparse_from_triplets(6, [(i, j, k + 1) for k, (i, j) in enumerate(DEMO6)], "integer")
    cases.append(case("demo6", demo6, ["dd"], [1, 3], 17))
    cases.append(case("sparse_real12", permkit.random_sparse_real(12, 0.3, SEED), allp, [1, 7], 18))
    cases.append(case("sparse_real18", permkit.random_sparse_real(18, 0.4, SEED), allp, [64], 19))
    zc = rand_dense(10, 410, "complex128")
    rng = random.Random(411)
    sparse_c = sparse_from_triplets(10, [(i, j, zc.entry(i, j)) for i in range(10) for j in range(10)
                                         if rng.random() < 0.4], "complex128")
    cases.append(case("sparse_cplx10", sparse_c, ["dd"], [1, 7], 20))
    cases.append(case("sparse_int12", permkit.random_sparse_int(12, 0.4, SEED), ["dd"], [1, 5], 21))
    cases.append(case("sparse_binary20", dense_to_sparse(permkit.random_binary(20, SEED, 0.3)),
                      ["dd"], [1, 8], 22))
    cases.append(case("sparse_binary22", dense_to_sparse(permkit.random_binary(22, SEED, 0.3)),
                      ["dd"], [1], 23))
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump({"generator": "tools/make_golden.py", "reference": "permkit 0.1.0 "
                   "(/root/reference/pkg)", "seed": SEED, "cases": cases}, f, indent=0)
    print("wrote", OUT, file=sys.stderr)


if __name__ == "__main__":
    main()
