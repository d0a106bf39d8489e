"""One full n = 48 dense real permanent (config 5's matrix) on one B200:
2^47 - 1 Gray updates through the public API, timed end to end, plus the
same walk's first 1/8 (one rank's share of the 8-GPU configuration).

    python tools/run_n48.py > profiles/r01_n48_full_walk.json
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2502_16577_b200 as pk  # noqa: E402
from paper_2502_16577_b200 import _native  # noqa: E402
from paper_2502_16577_b200.distributed import rank_span  # noqa: E402
from paper_2502_16577_b200.kernels import DenseF64Problem  # noqa: E402
from paper_2502_16577_b200.precision import AccumulatorPolicy  # noqa: E402

SEED = 20261017
n = 48
g = np.random.default_rng(SEED).uniform(0.0, 1.0, size=(n, n))
rows = [[float(v) for v in r] for r in g]
pk.perm_nw(pk.random_real(20, 1), "kahan")  # context + kernels warm
prob = DenseF64Problem(pk.DenseMatrix.from_rows(rows))
lo, hi = rank_span(n, 0, 8)
st = _native.RunStats()
t0 = time.perf_counter()
prob.walk(lo, hi, AccumulatorPolicy.KAHAN, stats=st)
share_s = time.perf_counter() - t0
t0 = time.perf_counter()
perm = pk.permanent(rows, "kahan")
wall = time.perf_counter() - t0
T = (1 << (n - 1)) - 1
print(json.dumps({"n": n, "policy": "kahan", "matrix": f"random [0,1) seed {SEED}",
                  "permanent": perm.hex(), "permanent_float": perm,
                  "updates": T, "wall_s": wall, "updates_per_s": T / wall,
                  "rank0_of_8_share": {"iterates": hi - lo + 1, "kernel_ms": st.kernel_ms,
                                       "wall_s": share_s,
                                       "updates_per_s": (hi - lo + 1) / (st.kernel_ms * 1e-3)},
                  "projected_8gpu_s": share_s,
                  "paper_gv100_s": 4326.23}))
