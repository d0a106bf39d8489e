"""Accuracy of the dense real walk vs chunk size (the x-state drift of the
incremental Gray updates): permanent of random [0,1) matrices and of the
closed-form uniform(n, 0.91) for several log2 chunk sizes k and policies.

    python tools/accuracy_probe.py > profiles/r01_accuracy_probe.txt
"""
import math
import sys
from fractions import Fraction

import numpy as np

sys.path.insert(0, ".")
import paper_2502_16577_b200 as pk  # noqa: E402
from paper_2502_16577_b200.kernels import DenseF64Problem, _sign_factor, policy_product  # noqa: E402
from paper_2502_16577_b200.precision import AccumulatorPolicy, DoubleDouble, dd_add  # noqa: E402

SEED = 20261017


def perm(m, pol, k):
    prob = DenseF64Problem(m)
    n = m.n
    p0 = policy_product(prob.x0, pol)
    acc = p0 if isinstance(p0, DoubleDouble) else DoubleDouble(float(p0), 0.0)
    acc = dd_add(acc, prob.walk(1, (1 << (n - 1)) - 1, pol, log2_chunk=k))
    return acc.hi * _sign_factor(n)


for n in (32, 36, 40):
    g = np.random.default_rng(SEED).uniform(0.0, 1.0, size=(n, n))
    m = pk.DenseMatrix.from_rows([[float(v) for v in r] for r in g])
    u = pk.uniform(n, 0.91)
    exact_u = Fraction(math.factorial(n)) * Fraction(0.91) ** n
    ks = [k for k in (6, 8, 10, 12, 14, 16, 18) if k <= n - 6]
    res = {}
    for k in ks:
        for pol in ("kahan", "qq"):
            P = AccumulatorPolicy.parse(pol)
            v = perm(m, P, k)
            vu = perm(u, P, k)
            eu = float(abs(Fraction(vu) - exact_u) / exact_u)
            res[(k, pol)] = v
            print(f"n={n} k={k:2d} {pol:5s} random={v!r} uniform_relerr={eu:.3e}", flush=True)
    best = res[(ks[0], "qq")]
    for (k, pol), v in res.items():
        print(f"n={n} k={k:2d} {pol:5s} rel_to_k{ks[0]}_qq={(v - best) / best:+.3e}", flush=True)
