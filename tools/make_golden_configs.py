"""Reference anchors for the BASELINE configurations (tests/golden/configs/).

Runs the REFERENCE (permkit, offline install under baseline/_ref) here, in
the container that has it; the GPU box only reads the JSON it writes.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=baseline/_ref \
        python tools/make_golden_configs.py JOB [JOB ...]

Jobs (each writes tests/golden/configs/JOB.json; values as hex / decimal):

  real36_kahan, real36_dq   config 2: permanent_chunked(random_real(36, SEED),
                            policy, tau=65536) -- whole-walk reference results
  real40_kahan              the metric's matrix: permanent_chunked(random_real(40,
                            SEED), KAHAN, tau=65536), ~50 min on 8 cores
  haar32_dd                 config 4: permanent_chunked(Haar U(1024)[:32,:32], DD,
                            tau=4096)
  binary40_ranges           config 3: run_range partials of dense_to_sparse(
                            random_binary(40, SEED, 0.3)) on 2^20..2^22-iterate
                            ranges (aligned and unaligned, near both ends)
  real_ranges               run_range partials of random_real(n, SEED) for
                            n = 36, 40, 48, 63 on 2^20-iterate ranges, every policy
  complex_ranges            run_range partials of complex matrices of order 41..63

Every value comes from permkit's public API (parallel.plan_chunks /
execute_plan / reduce_partials / initial_product / run_range); per-chunk
partials of the whole-walk jobs are recorded on a sample of worker ids so a
mismatch can be localised.
"""

from __future__ import annotations

import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

import permkit
from permkit.kernels import total_iterates
from permkit.matrix import DenseMatrix, dense_to_sparse
from permkit.parallel import (execute_plan, initial_product, plan_chunks, reduce_partials,
                              run_range)
from permkit.precision import AccumulatorPolicy

SEED = 20261017
POL = {p.value: p for p in AccumulatorPolicy}
HERE = os.path.dirname(os.path.abspath(__file__))
OUTDIR = os.path.join(HERE, "..", "tests", "golden", "configs")


def enc(v):
    if isinstance(v, bool):
        raise TypeError
    if isinstance(v, int):
        return str(v)
    if isinstance(v, complex):
        return [v.real.hex(), v.imag.hex()]
    if isinstance(v, float):
        return v.hex()
    if hasattr(v, "hi"):
        return [v.hi.hex(), v.lo.hex()]
    raise TypeError(type(v))


def haar_block(n, seed):
    """U(M)[:n,:n] with M = n^2 (Mezzadri's QR recipe);
    the same construction as paper_2502_16577_b200.generate.haar_unitary_block."""
    M = n * n
    rng = np.random.default_rng(seed)
    z = (rng.standard_normal((M, M)) + 1j * rng.standard_normal((M, M))) / np.sqrt(2.0)
    q, r = np.linalg.qr(z)
    d = np.diagonal(r)
    u = q * (d / np.abs(d))
    return DenseMatrix.from_rows([[complex(v) for v in row] for row in u[:n, :n]])


def random_complex(n, seed):
    rng = np.random.default_rng(seed)
    z = rng.uniform(-1.0, 1.0, size=(n, n)) + 1j * rng.uniform(-1.0, 1.0, size=(n, n))
    return DenseMatrix.from_rows([[complex(v) for v in row] for row in z])


def matrix_desc(m):
    if isinstance(m, DenseMatrix):
        return {"container": "dense", "n": m.n, "kind": m.kind,
                "data": [enc(v) for v in m.data]}
    return {"container": "sparse", "n": m.n, "kind": m.kind,
            "triplets": [[i, j, enc(v)] for (i, j, v) in m.crs.triplets()]}


def write(job, d):
    os.makedirs(OUTDIR, exist_ok=True)
    d = {"job": job, "generator": "tools/make_golden_configs.py",
         "reference": "permkit 0.1.0 (/root/reference/pkg, numba %s)" % _numba_version(),
         "seed": SEED, **d}
    path = os.path.join(OUTDIR, job + ".json")
    with open(path, "w") as f:
        json.dump(d, f, indent=0)
    print("wrote", path, file=sys.stderr, flush=True)


def _numba_version():
    try:
        import numba
        return numba.__version__
    except Exception:
        return "absent"


def whole(job, m, policy, tau, samples=64):
    t0 = time.time()
    pol = POL[policy]
    plan = plan_chunks(m.n, tau, True)
    parts = execute_plan(m, plan, pol)
    p0 = initial_product(m, pol)
    val = reduce_partials(parts, p0, m.n)
    step = max(1, len(parts) // samples)
    write(job, {
        "matrix": matrix_desc(m), "policy": policy, "tau": tau, "aligned": True,
        "chunk_size": plan.chunk_size, "num_partials": len(parts),
        "residual": list(plan.residual) if plan.residual else None,
        "p0": enc(p0), "value": enc(val),
        "sampled_partials": [{"worker_id": p.worker_id, "start": p.start, "end": p.end,
                              "value": enc(p.value)} for p in parts[::step]] +
                            [{"worker_id": parts[-1].worker_id, "start": parts[-1].start,
                              "end": parts[-1].end, "value": enc(parts[-1].value)}],
        "seconds": time.time() - t0, "cores": os.cpu_count()})


def _range_job(args):
    m, s, e, policy = args
    t0 = time.time()
    v = run_range(m, s, e, POL[policy]).value
    return {"start": s, "end": e, "policy": policy, "value": enc(v),
            "seconds": time.time() - t0}


def ranges_for(n, sizes_log2, seed):
    T = total_iterates(n)
    rng = np.random.default_rng(seed)
    out = []
    for lg in sizes_log2:
        size = 1 << lg
        out.append((1, size))                                      # walk start
        c = int(rng.integers(1, (T // size) - 1))
        out.append((1 + c * size, (c + 1) * size))                 # aligned middle
        out.append((T - size + 1, T))                              # walk end (unaligned)
        a = int(rng.integers(1, T - 2 * size))
        out.append((a, a + size + int(rng.integers(1, 4096))))     # unaligned middle
    return out


def run_ranges(job, mats, policies, sizes_log2, workers=None):
    tasks = []
    for name, m in mats:
        for k, (s, e) in enumerate(ranges_for(m.n, sizes_log2, m.n * 1000 + len(name))):
            for p in policies:
                tasks.append((name, m, s, e, p))
    with ProcessPoolExecutor(max_workers=workers or os.cpu_count()) as ex:
        res = list(ex.map(_range_job, [(m, s, e, p) for (_, m, s, e, p) in tasks]))
    cases = {}
    for (name, m, *_), r in zip(tasks, res):
        c = cases.setdefault(name, {"name": name, "matrix": matrix_desc(m), "ranges": []})
        c["ranges"].append(r)
    write(job, {"cases": list(cases.values())})


def main(jobs):
    for job in jobs:
        print("job", job, file=sys.stderr, flush=True)
        if job == "real36_kahan":
            whole(job, permkit.random_real(36, SEED, 0.0, 1.0), "kahan", 65536)
        elif job == "real36_dq":
            whole(job, permkit.random_real(36, SEED, 0.0, 1.0), "dq", 65536)
        elif job == "real40_kahan":
            whole(job, permkit.random_real(40, SEED, 0.0, 1.0), "kahan", 65536)
        elif job == "haar32_dd":
            whole(job, haar_block(32, SEED), "dd", 4096)
        elif job == "binary40_ranges":
            m = dense_to_sparse(permkit.random_binary(40, SEED, 0.3))
            run_ranges(job, [("binary40", m)], ["dd"], [20, 21])
        elif job == "real_ranges":
            mats = [(f"real{n}", permkit.random_real(n, SEED, 0.0, 1.0)) for n in (36, 40, 48, 63)]
            run_ranges(job, mats, ["dd", "kahan", "dq", "qq"], [16, 20])
        elif job == "complex_ranges":
            mats = [("haar48", haar_block(48, SEED))] + \
                   [(f"cplx{n}", random_complex(n, SEED + n)) for n in (41, 44, 52, 56, 63)]
            run_ranges(job, mats, ["dd"], [14, 18])
        else:
            raise SystemExit(f"unknown job {job}")


if __name__ == "__main__":
    main(sys.argv[1:])
