"""Dense integer kernel K5 (template, int32 groups) vs the generated
float-group kernel (K6 codegen) on the same matrices."""
import sys
import time

sys.path.insert(0, ".")
import paper_2502_16577_b200 as pk  # noqa: E402
from paper_2502_16577_b200 import _native  # noqa: E402
from paper_2502_16577_b200.integer import IntProblem  # noqa: E402

for n, d in ((30, 0.5), (32, 0.3), (34, 0.5)):
    m = pk.random_binary(n, 20261017, d)
    prob = IntProblem(m)
    T = (1 << (n - 1)) - 1
    res = {}
    for sparse in (False, True):
        prob.walk(1, T, sparse=sparse)  # warm / compile
        st = _native.RunStats()
        words, _ = prob.walk(1, T, sparse=sparse, stats=st)
        res[sparse] = (words, T / (st.kernel_ms * 1e-3))
    print(f"n={n} d={d} K5 {res[False][1]:.4g} upd/s  generated {res[True][1]:.4g} upd/s  "
          f"same={res[False][0] == res[True][0]}", flush=True)
