"""A few small launches of each kernel family for compute-sanitizer racecheck."""
import sys

sys.path.insert(0, ".")
import paper_2502_16577_b200 as pk  # noqa: E402
from paper_2502_16577_b200.integer import int_batch_totals  # noqa: E402

print(pk.perm_nw(pk.random_real(16, 3, 0.0, 1.0), "kahan"))
print(pk.perm_nw(pk.haar_unitary_block(14, 2)))
print(pk.permanent(pk.random_binary(16, 5, 0.4)))
print(pk.permanent_batch([pk.random_real(13, k) for k in range(3)]))
print(pk.permanent_batch([pk.haar_unitary_block(12, k) for k in range(3)]))
print(int_batch_totals([pk.random_binary(13, k, 0.5) for k in range(3)]))
print(pk.perm_spa(pk.random_sparse_real(16, 0.4, 7, 0.0, 1.0), "kahan"))
from paper_2502_16577_b200.complex_walk import DenseC128Problem  # noqa: E402
from paper_2502_16577_b200.kernels import DenseF64Problem  # noqa: E402
print(DenseF64Problem(pk.random_real(40, 4, 0.0, 1.0)).walk(1, 1 << 18, pk.AccumulatorPolicy.KAHAN))
print(DenseF64Problem(pk.random_real(34, 4, 0.0, 1.0)).walk(1, 1 << 18, pk.AccumulatorPolicy.KAHAN, precise=True))
print(DenseC128Problem(pk.haar_unitary_block(44, 3, m=88)).walk(1, 1 << 18))
print("racecheck paths done")
