"""n = 48 accuracy (BASELINE config 5's order): uniform(48, 0.91) against its
closed form 48! a^48 under KAHAN and QQ (the paper's Table 3 probe: Kahan
5.68e-10, QQ 4.87e-10 at n = 48), and config 5's matrix
random_real(48, 20261017) under KAHAN. Each walk is 2^47 - 1 updates on one
B200 (~14 min KAHAN, ~45 min QQ).

    python tools/accuracy_n48.py > profiles/r02_accuracy_n48.txt
"""
import math
import os
import sys
import time
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_16577_b200 as pk  # noqa: E402

n = 48
u = pk.uniform(n, 0.91)
exact = Fraction(math.factorial(n)) * Fraction(0.91) ** n
for pol in ("kahan", "qq"):
    t0 = time.time()
    v = pk.perm_nw(u, pol)
    dt = time.time() - t0
    print(f"uniform(48, 0.91) {pol}: {v!r} relerr={float((Fraction(v) - exact) / exact):+.3e} "
          f"({dt:.0f} s, {((1 << 47) - 1) / dt:.3e} updates/s)", flush=True)
m = pk.random_real(n, 20261017, 0.0, 1.0)
t0 = time.time()
v = pk.perm_nw(m, "kahan")
dt = time.time() - t0
print(f"random_real(48, 20261017) kahan: {v.hex()} ({v!r}) ({dt:.0f} s, "
      f"{((1 << 47) - 1) / dt:.3e} updates/s)", flush=True)
