"""The drop-in boundary from plain C: tests/c/abi_smoke.c is compiled with
gcc against include/permkit_b200.h and linked to libpk_b200.so. Without a
device it must get the loud PK_ERR_CUDA (no CPU fallback); on the GPU box it
walks a 12 x 12 permanent and matches the Python API."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2502_16577_b200")


def _build(tmp_path):
    exe = tmp_path / "abi_smoke"
    r = subprocess.run(["gcc", "-std=c11", "-O1", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-L", PKG, "-lpk_b200",
                        "-Wl,-rpath," + PKG, "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_client_links_and_fails_loudly_without_a_device(tmp_path):
    from paper_2502_16577_b200 import _native
    if _native.load().pk_device_count() > 0:
        pytest.skip("a device is present (covered by the gpu variant)")
    r = subprocess.run([str(_build(tmp_path))], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "no-device rc=5" in r.stdout


@pytest.mark.gpu
def test_c_client_walks_on_the_device(tmp_path):
    import paper_2502_16577_b200 as pk
    r = subprocess.run([str(_build(tmp_path))], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    perm = float(r.stdout.split("perm=")[1].split()[0])
    # same matrix through the Python API
    n, s, a = 12, 12345, []
    for _ in range(n * n):
        s = (s * 1103515245 + 12345) & 0xFFFFFFFF
        a.append((s >> 8) / 16777216.0)
    want = pk.perm_nw(pk.DenseMatrix.from_rows([a[i * n:(i + 1) * n] for i in range(n)]), "kahan")
    assert abs(perm - want) <= 1e-12 * abs(want)
    assert "updates=2047" in r.stdout
