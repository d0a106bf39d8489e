"""Multi-GPU readiness of the public API: permanent(m,
workers=N) splits the walk into N contiguous power-of-two iterate ranges, one
host thread per device, and combines the device trees in fixed order -- the
single-device bits for every kind. The round's boxes have one GPU: the
distinct-device tests skip there; the same split on one device repeated
(devices=[0, 0, ...]) runs everywhere and exercises the identical host path
(per-device contexts, attributes and workspaces)."""

import numpy as np
import pytest

import paper_2502_16577_b200 as pk
from paper_2502_16577_b200 import _native

pytestmark = pytest.mark.gpu


def _mats():
    rng = np.random.default_rng(5)
    real = pk.DenseMatrix.from_array(rng.uniform(0.0, 1.0, size=(34, 34)))
    cplx = pk.haar_unitary_block(26, 5)
    binary = pk.dense_to_sparse(pk.random_binary(30, 5, 0.3))
    return [("real", real, "kahan"), ("complex", cplx, "dd"), ("binary", binary, "dd")]


def two_devices():
    try:  # evaluated at collection, also on CPU-only hosts
        return _native.device_count() >= 2
    except Exception:
        return False


@pytest.mark.parametrize("kind,m,policy", _mats())
def test_repeated_device_split_reproduces_single_device(kind, m, policy):
    one = pk.permanent(m, policy, devices=[0])
    for devs in ([0, 0], [0, 0, 0, 0]):
        assert pk.permanent(m, policy, devices=devs) == one, (kind, devs)


@pytest.mark.skipif(not two_devices(), reason="needs two GPUs")
@pytest.mark.parametrize("kind,m,policy", _mats())
def test_workers_two_gpus_reproduces_single_device(kind, m, policy):
    one = pk.permanent(m, policy, devices=[0])
    assert pk.permanent(m, policy, workers=2) == one
    assert pk.permanent(m, policy, devices=[1, 0]) == one


@pytest.mark.skipif(not two_devices(), reason="needs two GPUs")
def test_second_device_alone_after_first():
    # kernel attributes (the >48 KB shared-memory opt-in) are per device:
    # a launch on device 1 after device 0 must not reuse device 0's state
    m = pk.random_real(40, 3, 0.0, 1.0)
    prob = pk.kernels.DenseF64Problem(m)
    T = pk.total_iterates(40)
    a = prob.walk(1, T >> 6, pk.AccumulatorPolicy.KAHAN, devices=[0])
    b = prob.walk(1, T >> 6, pk.AccumulatorPolicy.KAHAN, devices=[1])
    assert (a.hi, a.lo) == (b.hi, b.lo)
