"""How much of the fast walk's difference from the precise mode is the
one-off grid rounding of the input (pk_quantize_walk): the precise mode run
on the grid-rounded input vs on the original input, and the fast QQ walk.

    python tools/quantization_effect.py 36 40
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_16577_b200 as pk  # noqa: E402
from paper_2502_16577_b200 import _native as nat  # noqa: E402
from paper_2502_16577_b200.kernels import DenseF64Problem, _sign_factor, policy_product  # noqa: E402
from paper_2502_16577_b200.precision import AccumulatorPolicy, DoubleDouble, dd_add  # noqa: E402

QQ = AccumulatorPolicy.QQ
for n in [int(v) for v in sys.argv[1:]] or [36, 40]:
    g = np.random.default_rng(20261017).uniform(0.0, 1.0, size=(n, n))
    prob = DenseF64Problem(pk.DenseMatrix.from_rows([[float(v) for v in r] for r in g]))
    T = (1 << (n - 1)) - 1

    def total(cols, x0, flags):
        out = np.zeros(2)
        st = nat.RunStats()
        rc = nat.load().pk_dense_f64(nat.dptr(cols), nat.dptr(x0), n, 1, T, QQ.code, flags, 0,
                                     None, 0, nat.dptr(out), st)
        nat.check(rc, "pk_dense_f64")
        p0 = policy_product(x0, QQ)
        acc = dd_add(p0, DoubleDouble(out[0], out[1]))
        return acc.hi * _sign_factor(n)

    qc = np.zeros_like(prob.cols)
    qx = np.zeros_like(prob.x0)
    nat.check(nat.load().pk_quantize_walk(nat.dptr(prob.cols), nat.dptr(prob.x0), n, 1,
                                          nat.dptr(qc), nat.dptr(qx)), "quantize")
    p_orig = total(prob.cols, prob.x0, nat.PK_FLAG_PRECISE)
    p_quant = total(qc, qx, nat.PK_FLAG_PRECISE)
    f_qq = total(prob.cols, prob.x0, 0)
    print(f"n={n}: precise(rounded input) vs precise(input) {(p_quant - p_orig) / p_orig:+.3e}; "
          f"fast QQ vs precise(rounded input) {(f_qq - p_quant) / p_quant:+.3e}; "
          f"fast QQ vs precise(input) {(f_qq - p_orig) / p_orig:+.3e}", flush=True)
