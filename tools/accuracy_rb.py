"""[historical (round 1 / early round 2): the x rebuild and PK_REBUILD_LOG2 were removed when the fast walks moved to exact grid-rounded states; kept to document profiles/r02_accuracy_*_rb*.txt]

Accuracy of the fast dense real walk vs the state rebuild period
(PK_REBUILD_LOG2): relative error of uniform(n, 0.91) against the closed form
n! a^n, and the random [0,1) value, per policy. One process per setting
(the period is read once per process).

    for rb in 4 6 8; do PK_REBUILD_LOG2=$rb python tools/accuracy_rb.py 36 40; done
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
rb = os.environ.get("PK_REBUILD_LOG2", "default")
for n in [int(v) for v in sys.argv[1:]] or [36, 40]:
    u = pk.uniform(n, 0.91)
    exact_u = Fraction(math.factorial(n)) * Fraction(0.91) ** n
    g = np.random.default_rng(SEED).uniform(0.0, 1.0, size=(n, n))
    m = pk.DenseMatrix.from_rows([[float(v) for v in r] for r in g])
    for pol in ("kahan", "qq"):
        t0 = time.time()
        vu = pk.perm_nw(u, pol)
        dt = time.time() - t0
        vr = pk.perm_nw(m, pol)
        eu = float((Fraction(vu) - exact_u) / exact_u)
        print(f"rb={rb} n={n} {pol:5s} uniform_relerr={eu:+.3e} random={vr.hex()} "
              f"({vr!r}) t={dt:.2f}s", flush=True)
