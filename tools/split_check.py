import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2502_16577_b200 as pk
from paper_2502_16577_b200.kernels import DenseF64Problem
from paper_2502_16577_b200.precision import AccumulatorPolicy, dd_add, DoubleDouble
SEED = 20261017
for n in (30, 34, 40):
    g = np.random.default_rng(SEED).uniform(0.0, 1.0, size=(n, n))
    m = pk.DenseMatrix.from_rows([[float(v) for v in r] for r in g])
    prob = DenseF64Problem(m)
    T = (1 << (n - 1)) - 1
    K = AccumulatorPolicy.KAHAN
    whole = prob.walk(1, T, K)
    h = 1 << (n - 2)
    a = prob.walk(1, h, K); b = prob.walk(h + 1, T, K)
    s = dd_add(a, b)
    st = pk._native.RunStats(); prob.walk(h + 1, T, K, stats=st)
    print(n, whole, s, (whole.hi - s.hi) / whole.hi, 'k(rank1)=', st.log2_chunk, st.walker_ranges, st.chunks)
    # rank1 alone with forced k equal to rank0's
    b2 = prob.walk(h + 1, T, K, log2_chunk=st.log2_chunk + 1)
    print('   rank1 k vs k+1:', b, b2, (b.hi - b2.hi) / b2.hi)
