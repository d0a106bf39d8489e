"""Pin the C oracle (oracle/permref.c) to the reference's own outputs.

Every range partial recorded in tests/golden/golden.json by
tools/make_golden.py (permkit.parallel.run_range) must be reproduced bit for
bit; whole permanents via the oracle's chunked path must match permkit's
permanent_chunked bit for bit for the same tau.
"""

import pytest

import golden_io as gio
import oracle


def _hex_dd(v):
    return (v[0].hex(), v[1].hex())


@pytest.mark.parametrize("name", [c["name"] for c in gio.load()["cases"]])
def test_oracle_ranges_bitwise(golden, name):
    case = next(c for c in golden["cases"] if c["name"] == name)
    m = case["matrix"]
    n, kind, cont = m["n"], m["kind"], m["container"]
    checked = 0
    for r in case["ranges"]:
        s, e, pol = r["start"], r["end"], r["policy"]
        if kind == "real64":
            if cont == "dense":
                got = oracle.dense_f64_range(gio.dense_array(case), s, e, pol)
            else:
                got = oracle.sparse_f64_range(n, gio.triplets(case), s, e, pol)
            assert _hex_dd(got) == tuple(r["value"]), (name, s, e, pol)
        elif kind == "complex128":
            if cont == "dense":
                got = oracle.dense_c128_range(gio.dense_array(case), s, e)
            else:
                got = oracle.sparse_c128_range(n, gio.triplets(case), s, e)
            assert [got.real.hex(), got.imag.hex()] == r["value"], (name, s, e)
        else:
            if cont == "dense":
                got = oracle.dense_int_range(gio.dense_array(case), s, e)
            else:
                got = oracle.sparse_int_range(n, gio.triplets(case), s, e)
            assert got == int(r["value"]), (name, s, e)
        checked += 1
    assert checked == len(case["ranges"])


@pytest.mark.parametrize("name", [c["name"] for c in gio.cases(gio.load(), "dense", "real64")])
def test_oracle_chunked_bitwise(golden, name):
    case = next(c for c in golden["cases"] if c["name"] == name)
    a = gio.dense_array(case)
    for ch in case["chunked"]:
        if not ch["aligned"]:
            continue
        got = oracle.dense_f64_permanent(a, ch["policy"], ch["tau"], threads=4)
        assert got.hex() == ch["value"], (name, ch)


def test_oracle_p0_matches_initial_product(golden):
    for case in gio.cases(golden, "dense", "real64"):
        a = gio.dense_array(case)
        for pol, v in case["p0"].items():
            hi, lo = oracle.dense_f64_p0(a, pol)
            if pol == "qq":
                assert [hi.hex(), lo.hex()] == v
            else:
                assert hi.hex() == v
