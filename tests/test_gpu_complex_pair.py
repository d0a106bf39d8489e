"""The lane-pair complex kernel K3p (csrc/pk_c128_pair.cuh): register walks of
complex matrices of order 41..63, where one thread's 4n registers of state no
longer fit. Exact mode keeps the reference's sequential
product across the two lanes and must reproduce run_range over every chunk
bit for bit (the C oracle restates chunk_dense_c128, _loops.py:186-209);
fast mode (exact grid-rounded states, fma products, compensated body sums)
must agree with it."""

import numpy as np
import pytest

import oracle
import paper_2502_16577_b200 as pk
from paper_2502_16577_b200.complex_walk import DenseC128Problem
from paper_2502_16577_b200.precision import dd_pairwise

pytestmark = pytest.mark.gpu


def _haar(n, seed):
    m = pk.haar_unitary_block(n, seed, m=2 * n)  # a smaller unitary: larger entries
    return m, np.array(m.data, dtype=np.complex128).reshape(n, n)


@pytest.mark.parametrize("n", [41, 44, 48, 55, 63])
def test_pair_exact_chunks_bitwise_vs_oracle(n):
    m, a = _haar(n, 900 + n)
    prob = DenseC128Problem(m)
    k = 7
    total_chunks = 1 << (n - 1 - k)
    for lo in (0, 1 << 20, total_chunks - 32):  # walk start, middle, last (clipped) chunks
        parts, (tr, ti) = prob.chunks(k, lo, 32, exact=True)
        T = (1 << (n - 1)) - 1
        for i in range(0, 32, 5):
            c = lo + i
            s, e = 1 + c * (1 << k), min((c + 1) << k, T)
            want = oracle.dense_c128_range(a, s, e)
            assert (parts[i][0].hex(), parts[i][1].hex()) == (want.real.hex(), want.imag.hex()), (n, c)
        # the launch total is the fixed tree over the chunk partials
        re = dd_pairwise([(float(p[0]), 0.0) for p in parts])
        im = dd_pairwise([(float(p[1]), 0.0) for p in parts])
        assert (re.hi, re.lo, im.hi, im.lo) == (tr.hi, tr.lo, ti.hi, ti.lo)


@pytest.mark.parametrize("n", [41, 52])
def test_pair_fast_chunks_close_to_exact(n):
    m, _ = _haar(n, 700 + n)
    prob = DenseC128Problem(m)
    k = 9
    lo = 3 << 12
    fe, _ = prob.chunks(k, lo, 64, exact=True)
    ff, _ = prob.chunks(k, lo, 64, exact=False)
    for e, f in zip(fe, ff):
        ze, zf = complex(e[0], e[1]), complex(f[0], f[1])
        assert abs(zf - ze) <= 1e-10 * max(abs(ze), 1e-300), (n, ze, zf)


def test_pair_whole_walk_n41_fast_vs_exact():
    # the whole 2^40-iterate walk both ways: fast (exact states) and exact
    # mode, the reference's incrementally updated states, over 2^10-step
    # chunks so that its row-sum drift stays small (over the default 2^21-step
    # chunks the two differ by 3.8e-9: the reference's drift)
    m, _ = _haar(41, 5)
    fast = pk.perm_nw(m)
    prob = DenseC128Problem(m)
    wr, wi = prob.walk(1, (1 << 40) - 1, exact=True, log2_chunk=10)
    p0 = prob.p0()
    from paper_2502_16577_b200.precision import DoubleDouble, dd_add
    re = dd_add(DoubleDouble(p0.real, 0.0), wr)
    im = dd_add(DoubleDouble(p0.imag, 0.0), wi)
    exact = complex(re.hi, im.hi) * pk.kernels._sign_factor(41)
    assert abs(fast - exact) <= 1e-10 * abs(exact), (fast, exact, abs(fast - exact) / abs(exact))


PAIR_BATCH_PROBE = r"""
import json, sys
sys.path.insert(0, %r)
import paper_2502_16577_b200 as pk
from paper_2502_16577_b200.complex_walk import DenseC128Problem
from paper_2502_16577_b200.csrc_params import c128_pair_fast_logu, c128_pair_logu
from paper_2502_16577_b200.kernels import _sign_factor
from paper_2502_16577_b200.precision import DoubleDouble, dd_add
n = int(sys.argv[1])
out = []
for exact in (False, True):
    ms = [pk.haar_unitary_block(n, 60 + s, m=2 * n) for s in range(3)]
    got = pk.permanent_batch(ms, exact=exact)
    k = max(n - 1 - 10, (c128_pair_logu(n) if exact else c128_pair_fast_logu(n)) + 1)
    for m, g in zip(ms, got):
        prob = DenseC128Problem(m)
        wr, wi = prob.walk(1, (1 << (n - 1)) - 1, exact=exact, log2_chunk=k)
        if exact:
            p0 = prob.p0()
            r0, i0 = DoubleDouble(p0.real, 0.0), DoubleDouble(p0.imag, 0.0)
        else:
            from paper_2502_16577_b200.complex_walk import fast_p0
            r0, i0 = fast_p0(prob)
        re = dd_add(r0, wr)
        im = dd_add(i0, wi)
        s = _sign_factor(n)
        out.append([g.real.hex(), g.imag.hex(), (re.hi * s).hex(), (im.hi * s).hex()])
print(json.dumps(out))
"""


def test_pair_batch_equals_single_launch_bitwise():
    # batched complex walks above n = 40 run the lane-pair layout, whose
    # entries must equal the single walk with the batch's chunk exponent bit
    # for bit. PK_C128_PAIR=1 (read once per process) routes n = 24 through
    # the same kernels, so the check runs in seconds in a subprocess.
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PK_C128_PAIR="1")
    r = subprocess.run([sys.executable, "-c", PAIR_BATCH_PROBE % root, "24"], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    for row in json.loads(r.stdout.strip().splitlines()[-1]):
        assert row[0:2] == row[2:4], row
