"""Host-side logic that needs no GPU: the C-ABI library loads and exports
every symbol the public header declares; plans, containers, precision and
the partial-result reduction behave like the reference's
(/root/reference/pkg/tests/test_parallel.py, test_matrix.py,
test_precision.py)."""

import ctypes
import os
import re

import numpy as np

import pytest

import paper_2502_16577_b200 as pk
from paper_2502_16577_b200 import _native
from paper_2502_16577_b200.parallel import PartialResult
from paper_2502_16577_b200.precision import AccumulatorPolicy, DoubleDouble, dd_pairwise

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "permkit_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(pk_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _native.load()
    syms = header_symbols()
    assert "pk_dense_f64" in syms and len(syms) >= 6
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _native.SIGNATURES, f"{s} lacks a ctypes signature"
    assert lib.pk_abi_version() == 1


def test_no_device_is_a_loud_error():
    # CPU container: the call must fail with DeviceError, never compute on the host
    try:
        if _native.device_count() > 0:
            pytest.skip("a GPU is visible")
    except pk.DeviceError:
        pass
    with pytest.raises(pk.DeviceError):
        pk.perm_nw(pk.random_real(12, 1))


def test_plan_tiling_and_alignment():
    for n in range(2, 21):
        for tau in (1, 2, 3, 7, 16, 64):
            for aligned in (True, False):
                plan = pk.plan_chunks(n, tau, aligned)
                spans = list(plan.ranges) + ([plan.residual] if plan.residual else [])
                pos = 1
                for (s, e) in spans:
                    assert s == pos and e >= s
                    pos = e + 1
                assert pos == pk.total_iterates(n) + 1
                if aligned and plan.chunk_size:
                    assert plan.chunk_size & (plan.chunk_size - 1) == 0
    assert pk.plan_chunks(3, 100).tau_clamped
    with pytest.raises(ValueError):
        pk.plan_chunks(64, 4)
    with pytest.raises(ValueError):
        pk.plan_chunks(8, 0)


def test_alignment_report():
    for n in (10, 12, 14):
        for tau in (2, 4, 8):
            counts = pk.cbl_alignment_report(pk.plan_chunks(n, tau, aligned=True))
            assert all(c == 1 for c in counts[:-1])
    assert max(pk.cbl_alignment_report(pk.fixed_chunk_plan(12, 17, 4))) >= 3


def test_hierarchy_flattens_like_reference():
    for n in range(6, 15):
        for p in range(1, 5):
            for w in range(1, 4):
                h = pk.plan_hierarchy(n, p, w, aligned=False)
                flat = h.flatten()
                assert [x[0] for x in flat] == list(range(len(flat)))
                got = []
                for pi in range(h.processes):
                    got.extend(h.jobs_for(pi))
                assert got == flat
    with pytest.raises(ValueError):
        pk.plan_hierarchy(3, 4, 4)


def test_graycode():
    assert pk.cbl_sequence(3) == [0, 1, 0, 2, 0, 1, 0]
    for g in range(1, 1 << 12):
        st = pk.changed_bit(g)
        assert pk.gray_of(g) ^ pk.gray_of(g - 1) == 1 << st.j
        assert st.s == (1 if (pk.gray_of(g) >> st.j) & 1 else -1)


def test_containers_and_kinds():
    m = pk.DenseMatrix.from_rows([[1, 2], [3, 4]])
    assert m.kind == "integer"
    assert pk.DenseMatrix.from_rows([[1.0, 2], [3, 4]]).kind == "real64"
    assert pk.DenseMatrix.from_rows([[1j, 2], [3, 4]]).kind == "complex128"
    with pytest.raises(pk.ImpossibleError):
        pk.DenseMatrix.from_rows([[1] * 64 for _ in range(64)])
    with pytest.raises(pk.StructureError):
        pk.DenseMatrix.from_rows([[1, 2]])
    with pytest.raises(pk.StructureError):
        pk.DenseMatrix.from_rows([[float("nan")]])
    s = pk.dense_to_sparse(pk.DenseMatrix.from_rows([[0, 2], [3, 0]]))
    assert s.nnz == 2 and s.ccs.cptrs == (0, 1, 2) and s.ccs.rids == (1, 0)
    s.validate()
    assert pk.sparse_to_dense(s).rows() == [[0, 2], [3, 0]]
    with pytest.raises(pk.StructureError):
        pk.sparse_from_triplets(2, [(0, 0, 1), (0, 0, 2)], "integer")


def test_reference_objects_are_accepted():
    class Fake:
        n = 2
        kind = "real64"
        data = (1.0, 2.0, 3.0, 4.0)
    m = pk.coerce_matrix(Fake())
    assert isinstance(m, pk.DenseMatrix) and m.entry(1, 0) == 3.0


def test_policy_parse_and_codes():
    assert AccumulatorPolicy.parse("KAHAN") is AccumulatorPolicy.KAHAN
    assert [p.code for p in AccumulatorPolicy] == [0, 1, 2, 3]
    with pytest.raises(ValueError):
        AccumulatorPolicy.parse("fast")


def test_dd_pairwise_is_balanced_tree():
    vals = [DoubleDouble(float(i) * 1e-3 + 1.0, 0.0) for i in range(8)]
    t = dd_pairwise(vals)
    l = pk.dd_add(pk.dd_add(vals[0], vals[1]), pk.dd_add(vals[2], vals[3]))
    r = pk.dd_add(pk.dd_add(vals[4], vals[5]), pk.dd_add(vals[6], vals[7]))
    assert t == pk.dd_add(l, r)


def test_reduce_partials_validation():
    n = 6
    parts = [PartialResult(0, 1, 16, 16, "real64", DoubleDouble(1.0, 0.0)),
             PartialResult(1, 17, 31, 15, "real64", DoubleDouble(2.0, 0.0))]
    assert pk.reduce_partials(parts, 0.5, n) == -7.0
    assert pk.reduce_partials(list(reversed(parts)), 0.5, n) == -7.0
    with pytest.raises(pk.StructureError):
        pk.reduce_partials(parts[1:], 0.5, n)
    with pytest.raises(pk.StructureError):
        pk.reduce_partials(parts + [parts[0]], 0.5, n)


def test_partials_file_round_trip(tmp_path):
    m = pk.random_real(6, 3)
    parts = [PartialResult(0, 1, 16, 16, "real64", DoubleDouble(1.25, 2.0 ** -60)),
             PartialResult(1, 17, 31, 15, "real64", DoubleDouble(-2.0, 0.0))]
    path = tmp_path / "p.txt"
    pk.write_partials_file(path, m, "dd", parts)
    header, got = pk.read_partials_file(path)
    assert header["n"] == 6 and got == parts
    assert header["matrix_sha256"] == pk.matrix_content_hash(m)
    assert pk.matrix_content_hash(m) == pk.matrix_content_hash(pk.dense_to_sparse(m))
    bad = tmp_path / "bad.txt"
    bad.write_text("# nope\n" + path.read_text())
    with pytest.raises(pk.ParseError):
        pk.read_partials_file(bad)


def test_csrc_params_mirror():
    import re
    from paper_2502_16577_b200 import csrc_params as cp
    text = open(os.path.join(ROOT, "paper_2502_16577_b200", "csrc", "pk_launch.h")).read()
    assert "constexpr int dense_logu(int N) { return N <= 50 ? 4 : 3; }" in text
    assert "constexpr int dense_minb(int N) { return N <= 36 ? 3 : 2; }" in text
    assert "(N - 1 - 10) > (logu + 1) ? (N - 1 - 10) : (logu + 1)" in text
    assert "constexpr int c128_logu(int N) { return N <= 32 ? 2 : 1; }" in text
    assert cp.c128_logu(32) == 2 and cp.c128_logu(33) == 1
    assert "constexpr int kC128NMax = 40;" in text and cp.C128_N_MAX == 40
    assert "constexpr int c128_pair_logu(int N) { return N <= 48 ? 2 : 1; }" in text
    assert "constexpr int c128_fast_logu(int N) { return 3; }" in text
    assert cp.c128_register_logu(40) == 3 and cp.c128_register_logu(41) == 4
    assert "constexpr int c128_pair_fast_logu(int N) { return N <= 42 ? 4 : 3; }" in text
    assert cp.c128_pair_fast_logu(42) == 4 and cp.c128_pair_fast_logu(43) == 3
    assert cp.dense_logu(50) == 4 and cp.dense_logu(51) == 3
    assert cp.batch_log2_chunk(20, 4) == 9 and cp.batch_log2_chunk(12, 4) == 5


def test_generated_spa_source_compiles_for_sm100a(tmp_path):
    # the per-matrix SpaRyser kernel source is valid CUDA for sm_100a and
    # updates only the nonzeros of each statically known column
    import subprocess
    from paper_2502_16577_b200.integer import spa_source
    m = pk.random_binary(24, 3, 0.2)
    src = spa_source(m)
    assert "spa_int" in src and "switch (j)" in src
    nnz_col0 = sum(1 for i in range(24) if m.entry(i, 0))
    # float-group kernel (default): step 1 adds literal 2*a_i0 to z_i, nonzeros only
    body = src.split("const float smid")[1].split("{", 1)[1].split("const float f0")[0]
    assert body.count(".0f;") == nnz_col0
    assert "addsub128" in src and "__umul64hi" in src
    f = tmp_path / "spa.cu"
    f.write_text(src)
    r = subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++17", "-gencode",
                        "arch=compute_100a,code=sm_100a", "-cubin", "-o", str(tmp_path / "spa.cubin"),
                        str(f)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.parametrize("n,exact", [(40, False), (40, True), (24, False)])
def test_generated_spa_f64_source_compiles_without_spills(tmp_path, n, exact):
    # the per-pattern sparse real kernel is valid sm_100a CUDA against the
    # same device headers the nvcc-built kernels use, touches only the
    # nonzeros of each static column, and keeps x[n] in registers (no spills)
    import subprocess
    from paper_2502_16577_b200 import kernels as K
    from paper_2502_16577_b200.precision import AccumulatorPolicy
    rng = np.random.default_rng(n)
    a = rng.uniform(size=(n, n)) * (rng.uniform(size=(n, n)) < 0.3)
    trip = [(i, j, float(a[i, j])) for i in range(n) for j in range(n) if a[i, j] != 0.0]
    prob = K.SparseF64Problem(pk.sparse_from_triplets(n, trip, "real64"))
    src = prob.source(AccumulatorPolicy.KAHAN, exact=exact)
    assert "spa_f64" in src and "switch (j)" in src
    step1 = src.split("// step 1: column 0")[1].split("// step 2")[0]
    assert step1.count("__dadd_rn(x") + step1.count("__dsub_rn(x") == int((a[:, 0] != 0).sum())
    f = tmp_path / "spa_f64.cu"
    f.write_text(src)
    csrc = os.path.join(ROOT, "paper_2502_16577_b200", "csrc")
    r = subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++17", "-gencode",
                        "arch=compute_100a,code=sm_100a", "-cubin", "-I", csrc, "-Xptxas", "-v",
                        "-o", str(tmp_path / "spa.cubin"), str(f)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "0 bytes spill stores" in r.stderr and "0 bytes spill loads" in r.stderr, r.stderr


@pytest.mark.parametrize("n,exact", [(32, False), (40, True)])
def test_generated_spa_c128_source_compiles_without_spills(tmp_path, n, exact):
    import subprocess
    from paper_2502_16577_b200.complex_walk import DenseC128Problem
    rng = np.random.default_rng(n)
    a = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))) * (rng.uniform(size=(n, n)) < 0.3)
    trip = [(i, j, complex(a[i, j])) for i in range(n) for j in range(n) if a[i, j] != 0]
    src = DenseC128Problem(pk.sparse_from_triplets(n, trip, "complex128")).source(exact)
    step1 = src.split("// step 1: column 0")[1].split("// step 2")[0].split("const u64 g = gb")[0]
    assert step1.count("const double2 v = sv2[") == int((a[:, 0] != 0).sum())
    f = tmp_path / "spa_c128.cu"
    f.write_text(src)
    csrc = os.path.join(ROOT, "paper_2502_16577_b200", "csrc")
    r = subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++17", "-gencode",
                        "arch=compute_100a,code=sm_100a", "-cubin", "-I", csrc, "-Xptxas", "-v",
                        "-o", str(tmp_path / "spa.cubin"), str(f)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "0 bytes spill stores" in r.stderr, r.stderr


def test_haar_block_is_independent_of_blas_threads():
    # every rank of a multi-GPU run must rebuild the same matrix whatever
    # its BLAS thread count (torchrun sets OMP_NUM_THREADS=1 per rank)
    from threadpoolctl import threadpool_limits
    a = pk.haar_unitary_block(12, 99).data
    with threadpool_limits(limits=4):
        b = pk.haar_unitary_block(12, 99).data
    assert a == b
