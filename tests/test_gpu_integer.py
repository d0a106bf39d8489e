"""GPU exactness of the integer path (K5/K6): every partial and permanent
must equal the reference's big-int result exactly."""

import math
import random

import numpy as np
import pytest

import golden_io as gio
import paper_2502_16577_b200 as pk
from paper_2502_16577_b200.integer import IntProblem

pytestmark = pytest.mark.gpu

INTS = [c["name"] for c in gio.cases(gio.load(), kind="integer")]


def _case(golden, name):
    return next(c for c in golden["cases"] if c["name"] == name)


def _matrix(case):
    m = case["matrix"]
    if m["container"] == "dense":
        return pk.DenseMatrix.from_rows(gio.dense_array(case), kind="integer")
    return pk.sparse_from_triplets(m["n"], gio.triplets(case), "integer")


def matching_count(rows):
    """perfect matchings of a 0/1 matrix: DP over used-column masks"""
    dp = {0: 1}
    for r in rows:
        nxt = {}
        for used, ways in dp.items():
            for j, v in enumerate(r):
                if v and not (used >> j) & 1:
                    nxt[used | 1 << j] = nxt.get(used | 1 << j, 0) + ways
        dp = nxt
    return dp.get((1 << len(rows)) - 1, 0)


@pytest.mark.parametrize("name", INTS)
def test_int_ranges_exact_vs_reference(golden, name):
    case = _case(golden, name)
    m = _matrix(case)
    for r in case["ranges"]:
        p = pk.run_range(m, r["start"], r["end"])
        assert p.value == int(r["value"]), (name, r)
        assert p.kind == "integer"


@pytest.mark.parametrize("name", INTS)
def test_int_permanents_exact_vs_reference(golden, name):
    case = _case(golden, name)
    m = _matrix(case)
    for ch in case["chunked"]:
        got = pk.permanent_chunked(m, "dd", tau=ch["tau"], aligned=ch["aligned"])
        assert got == int(ch["value"]), (name, ch)
    want = int(case["chunked"][0]["value"])
    got = pk.perm_spa(m) if isinstance(m, pk.SparsePair) else pk.perm_nw(m)
    assert got == want and isinstance(got, int)


def test_demo6_and_ternary12(golden):
    assert pk.perm_spa(_matrix(_case(golden, "demo6"))) == 61776
    assert pk.perm_nw(_matrix(_case(golden, "ternary12_int"))) == 2


@pytest.mark.parametrize("n", [12, 16, 18, 20])
def test_binary_matching_counts(n):
    rng = random.Random(n)
    for _ in range(3):
        rows = [[1 if rng.random() < 0.45 else 0 for _ in range(n)] for _ in range(n)]
        want = matching_count(rows)
        m = pk.DenseMatrix.from_rows(rows)
        assert pk.perm_nw(m) == want
        assert pk.perm_spa(pk.dense_to_sparse(m)) == want


def test_register_kernel_equals_walkers_on_random_ranges():
    # a 30x30 0/1 matrix: register kernels (aligned middle) + walkers (head
    # and tail) against one-thread-per-range walkers on the same ranges
    m = pk.random_binary(30, 3, 0.35)
    rng = np.random.default_rng(5)
    T = pk.total_iterates(30)
    prob = IntProblem(m)
    for _ in range(4):
        s = int(rng.integers(1, T // 2))
        e = s + int(rng.integers(1 << 20, 1 << 22))
        fast = pk.run_range(m, s, e).value
        pieces = [(a, min(a + (1 << 16) - 1, e)) for a in range(s, e + 1, 1 << 16)]
        words, info = prob.ranges(pieces)
        from paper_2502_16577_b200.integer import _signed
        slow = sum(_signed(w, 192) for w in words) << info.even_rows
        assert fast == slow


def test_device_split_is_exact():
    m = pk.random_binary(32, 11, 0.3)
    one = pk.perm_nw(m)
    two = pk.perm_nw(m, devices=[0, 0])
    three = pk.perm_nw(m, devices=[0, 0, 0])
    assert one == two == three


def test_large_terms_refuse_instead_of_rounding():
    # entries up to 9e4: the per-row bound product passes 2^127, so neither a
    # partial nor (with the row-sum permanent bound) the total is provably
    # exact in 128-bit arithmetic -- the path must refuse, never round
    rng = random.Random(2)
    n = 12
    rows = [[rng.randint(0, 90000) for _ in range(n)] for _ in range(n)]
    m = pk.DenseMatrix.from_rows(rows)
    info = IntProblem(m).walk(1, 2)[1]
    assert not info.exact_terms
    with pytest.raises(OverflowError):
        pk.run_range(m, 1, 100)
    with pytest.raises(OverflowError):
        pk.perm_nw(m)


@pytest.mark.parametrize("n,density", [(14, 0.3), (20, 0.25), (24, 0.4), (26, 0.15)])
def test_generated_spa_kernel_is_exact(n, density):
    # per-matrix NVRTC SpaRyser kernel vs the template register kernel vs the
    # walkers, on whole walks and on an unaligned range
    for seed in (1, 2):
        m = pk.random_binary(n, seed, density)
        prob = IntProblem(m)
        T = pk.total_iterates(n)
        a, info = prob.walk(1, T, sparse=True)
        b, _ = prob.walk(1, T, sparse=False)
        assert a == b
        s, e = 3 + T // 5, T - 7
        a, _ = prob.walk(s, e, sparse=True)
        w, _ = prob.ranges([(s, e)])
        assert a == w[0]


def test_sparse_general_integers():
    m = pk.random_sparse_int(22, 0.3, 4)
    prob = IntProblem(m)
    T = pk.total_iterates(22)
    assert prob.walk(1, T, sparse=True)[0] == prob.walk(1, T, sparse=False)[0]
