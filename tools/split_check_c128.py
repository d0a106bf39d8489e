import sys
sys.path.insert(0, '.')
import paper_2502_16577_b200 as pk
from paper_2502_16577_b200.complex_walk import DenseC128Problem
from paper_2502_16577_b200.distributed import rank_span
from paper_2502_16577_b200.precision import dd_pairwise
n = 32
h = pk.haar_unitary_block(n, 20261017)
prob = DenseC128Problem(h)
T = (1 << (n - 1)) - 1
st = pk._native.RunStats()
whole = prob.walk(1, T, log2_chunk=12, stats=st)
print('whole', whole, st.log2_chunk, st.chunks, st.walker_ranges)
parts = []
for r in range(4):
    lo, hi = rank_span(n, r, 4)
    st = pk._native.RunStats()
    parts.append(prob.walk(lo, hi, log2_chunk=12, stats=st))
    print(r, lo, hi, parts[-1], st.log2_chunk, st.chunks, st.walker_ranges)
print('re', dd_pairwise([tuple(p[0]) for p in parts]), 'im', dd_pairwise([tuple(p[1]) for p in parts]))
print('inproc4', prob.walk(1, T, log2_chunk=12, devices=[0, 0, 0, 0]))
