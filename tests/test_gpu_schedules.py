"""Body schedules of the fast kernels give the same bits (DESIGN.md §3
"Row-major bodies"): the row-major body of K1 performs the same
additions and multiplications in the same order per row and per term as the
step-major body, only interleaved differently. Each schedule is selected per
process (PK_DENSE_VARIANT / PK_C128_VARIANT, read once), so the alternative
runs in a subprocess."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
import paper_2502_16577_b200 as pk
from paper_2502_16577_b200.complex_walk import DenseC128Problem
out = {}
for n in (24, 34, 40):
    m = pk.DenseMatrix.from_array(np.random.default_rng(n).uniform(0.0, 1.0, size=(n, n)))
    T = (1 << (n - 1)) - 1
    for pol in ("dd", "kahan", "dq"):
        p = pk.kernels.DenseF64Problem(m).walk(1, min(T, (1 << 34) - 5),
                                               pk.AccumulatorPolicy.parse(pol))
        out["real%%d_%%s" %% (n, pol)] = [p.hi.hex(), p.lo.hex()]
for n in (20, 30, 44):
    h = pk.haar_unitary_block(n, 3, m=2 * n)
    T = (1 << (n - 1)) - 1
    r, i = DenseC128Problem(h).walk(1, min(T, (1 << 33) - 9))
    out["cplx%%d" %% n] = [r.hi.hex(), r.lo.hex(), i.hi.hex(), i.lo.hex()]
print(json.dumps(out))
""" % ROOT


def run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", PROBE], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_row_major_and_step_major_bodies_agree_bitwise():
    # K1: same body length, step-major vs row-major -- same bits (K3 / K3p
    # change their body length or term-sum order with the schedule)
    a = run({"PK_DENSE_VARIANT": "2", "PK_C128_VARIANT": "2"})
    b = run({"PK_DENSE_VARIANT": "1", "PK_C128_VARIANT": "4"})
    for key in a:
        if key.startswith("real"):
            assert a[key] == b[key], key
