"""Small calls through every device path, for compute-sanitizer memcheck."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2502_16577_b200 as pk  # noqa: E402
from paper_2502_16577_b200.integer import IntProblem, int_batch_totals  # noqa: E402

m = pk.random_real(22, 3, 0.0, 1.0)
print(pk.perm_nw(m, "kahan"), pk.perm_nw(m, "qq"), pk.run_range(m, 3, 70001, "dq").value)
print(pk.perm_nw(pk.random_real(9, 1)))
s = pk.random_sparse_real(20, 0.4, 7, 0.0, 1.0)
print(pk.perm_spa(s, "kahan"))
h = pk.haar_unitary_block(18, 2)
print(pk.perm_nw(h), pk.perm_spa(pk.dense_to_sparse(h)))
b = pk.random_binary(24, 5, 0.4)
print(pk.permanent(b), pk.perm_spa(pk.dense_to_sparse(b)))
prob = IntProblem(b)
T = pk.total_iterates(24)
print(pk.run_range(b, 5, T - 7).value)
print(prob.ranges([(1, 1000), (5000, 90000)])[0][0])
print(int_batch_totals([pk.random_binary(16, k, 0.5) for k in range(5)]))
print(int_batch_totals([pk.random_binary(8, k, 0.5) for k in range(5)]))
print(pk.permanent_batch([pk.random_real(14, k) for k in range(4)] + [pk.haar_unitary_block(12, 1)]))
big = pk.random_binary(38, 9, 0.3)
print(IntProblem(big).walk(1, 1 << 24)[0])
print(pk.decomp_run(pk.random_sparse_real(16, 0.35, 3, 0.0, 1.0), "kahan")[0])
# round 2: the large-order block shapes, the precise mode, the lane-pair
# complex kernel and the grid-rounded fast inputs
from paper_2502_16577_b200.complex_walk import DenseC128Problem  # noqa: E402
from paper_2502_16577_b200.kernels import DenseF64Problem, SparseF64Problem  # noqa: E402
K = pk.AccumulatorPolicy.KAHAN
for n in (34, 40, 52):
    prob = DenseF64Problem(pk.random_real(n, 4, 0.0, 1.0))
    print(n, prob.walk(1, 1 << 22, K), prob.walk(1 << 30, (1 << 30) + (1 << 21) + 77, pk.AccumulatorPolicy.QQ))
print(DenseF64Problem(pk.random_real(36, 4, 0.0, 1.0)).walk(1, 1 << 20, K, precise=True))
print(SparseF64Problem(pk.random_sparse_real(36, 0.3, 5, 0.0, 1.0)).walk(1, 1 << 22, K))
for n in (32, 41, 63):
    hp = DenseC128Problem(pk.haar_unitary_block(n, 3, m=2 * n))
    print(n, hp.walk(1, 1 << 21), hp.chunks(7, 32, 32, exact=True)[1])
print(IntProblem(pk.dense_to_sparse(pk.random_binary(40, 5, 0.3))).walk(1, 1 << 22)[0])
print(DenseF64Problem(pk.random_real(40, 4, 0.0, 1.0)).chunks(8, 64, 32, pk.AccumulatorPolicy.QQ, exact=True)[1])
hp36 = DenseC128Problem(pk.haar_unitary_block(36, 3, m=72))
print(hp36.walk(1, 1 << 21), hp36.walk(1, 1 << 16, precise=True))
print(DenseF64Problem(pk.random_real(48, 4, 0.0, 1.0)).walk(1, 1 << 22, pk.AccumulatorPolicy.QQ))
print("memcheck paths done")
