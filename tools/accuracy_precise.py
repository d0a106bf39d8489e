"""Fast walk vs the precise mode (exact fixed-point row sums, double-double
products and sums) on the bench matrices, plus uniform(n, 0.91) against its
closed form n! a^n.

    python tools/accuracy_precise.py 36 40
"""
import math
import os
import sys
import time
from fractions import Fraction

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_16577_b200 as pk  # noqa: E402

SEED = 20261017
for n in [int(v) for v in sys.argv[1:]] or [36, 40]:
    g = np.random.default_rng(SEED).uniform(0.0, 1.0, size=(n, n))
    m = pk.DenseMatrix.from_rows([[float(v) for v in r] for r in g])
    u = pk.uniform(n, 0.91)
    exact_u = Fraction(math.factorial(n)) * Fraction(0.91) ** n
    t0 = time.time()
    pr = pk.perm_nw(m, precise=True)
    tp = time.time() - t0
    pu = pk.perm_nw(u, precise=True)
    print(f"n={n} precise random={pr.hex()} ({pr!r}) t={tp:.2f}s  precise uniform "
          f"relerr={float((Fraction(pu) - exact_u) / exact_u):+.3e}", flush=True)
    for pol in ("kahan", "dq", "qq"):
        v = pk.perm_nw(m, pol)
        vu = pk.perm_nw(u, pol)
        print(f"n={n} fast {pol:5s} random relerr_vs_precise={(v - pr) / pr:+.3e}  uniform "
              f"relerr={float((Fraction(vu) - exact_u) / exact_u):+.3e}", flush=True)
