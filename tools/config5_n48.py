"""Config 5's matrix, random_real(48, 20261017): whole 2^47 - 1 walks on one
B200 under KAHAN and QQ (both fast, exact states). The two policies differ
only in the product / accumulator rounding, so their agreement bounds that
part of the error at n = 48; the precise mode anchors n <= 40 and the first
2^38 iterates of this matrix (tests/test_gpu_configs.py).

    python tools/config5_n48.py > profiles/r02_config5_n48.txt
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_16577_b200 as pk  # noqa: E402

m = pk.random_real(48, 20261017, 0.0, 1.0)
vals = {}
for pol in ("kahan", "qq"):
    t0 = time.time()
    v = pk.perm_nw(m, pol)
    dt = time.time() - t0
    vals[pol] = v
    print(f"random_real(48, 20261017) {pol}: {v.hex()} ({v!r}) {dt:.0f} s "
          f"({((1 << 47) - 1) / dt:.3e} updates/s)", flush=True)
print(f"kahan vs qq: {(vals['kahan'] - vals['qq']) / vals['qq']:+.3e}", flush=True)
