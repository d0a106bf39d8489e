"""Small calls through the lane-pair complex kernel K3p (single walks, exact
chunks, batches) for compute-sanitizer: PK_C128_PAIR=1 routes every complex
order through it, so small orders exercise the same code as n = 41..63."""
import os
import sys

os.environ["PK_C128_PAIR"] = "1"
sys.path.insert(0, ".")
import paper_2502_16577_b200 as pk  # noqa: E402
from paper_2502_16577_b200.complex_walk import DenseC128Problem  # noqa: E402

for n in (15, 20):
    h = pk.haar_unitary_block(n, 2, m=2 * n)
    print(n, pk.perm_nw(h), DenseC128Problem(h).chunks(6, 0, 32, exact=True)[1])
print(pk.permanent_batch([pk.haar_unitary_block(17, k, m=34) for k in range(3)]))
print(pk.permanent_batch([pk.haar_unitary_block(17, k, m=34) for k in range(3)], exact=True))
print("memcheck pair paths done")
