"""Complex walk accuracy vs chunk size (x-state drift), Haar blocks."""
import sys

sys.path.insert(0, ".")
import paper_2502_16577_b200 as pk  # noqa: E402
from paper_2502_16577_b200.complex_walk import DenseC128Problem  # noqa: E402
from paper_2502_16577_b200.kernels import _sign_factor  # noqa: E402
from paper_2502_16577_b200.precision import DoubleDouble, dd_add  # noqa: E402

for n in (28, 32):
    h = pk.haar_unitary_block(n, 20261017)
    prob = DenseC128Problem(h)
    p0 = prob.p0()
    vals = {}
    for k in (6, 8, 10, 12, 14, 16):
        if k > n - 6:
            continue
        wr, wi = prob.walk(1, (1 << (n - 1)) - 1, log2_chunk=k)
        re = dd_add(DoubleDouble(p0.real, 0.0), wr)
        im = dd_add(DoubleDouble(p0.imag, 0.0), wi)
        s = _sign_factor(n)
        vals[k] = complex(re.hi * s, im.hi * s)
    ref = vals[6]
    for k, v in vals.items():
        print(f"n={n} k={k:2d} perm={v!r} rel_to_k6={abs(v - ref) / abs(ref):.3e}", flush=True)
