"""Complex accuracy against the precise mode: config 4 (Haar U(1024)[:32,
:32]) fast walk and the reference's permanent_chunked(DD, tau=4096) value
(tests/golden/configs/haar32_dd.json), and a complex n = 36 block.

    python tools/accuracy_c128_precise.py > profiles/r02_accuracy_c128_precise.txt
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_16577_b200 as pk  # noqa: E402

d = json.load(open(os.path.join(ROOT, "tests", "golden", "configs", "haar32_dd.json")))
n = d["matrix"]["n"]
vals = [complex(float.fromhex(v[0]), float.fromhex(v[1])) for v in d["matrix"]["data"]]
m = pk.DenseMatrix.from_rows([vals[i * n:(i + 1) * n] for i in range(n)])
ref = complex(float.fromhex(d["value"][0]), float.fromhex(d["value"][1]))
t0 = time.time()
truth = pk.perm_nw(m, precise=True)
dt = time.time() - t0
fast = pk.perm_nw(m)
print(f"config 4 Haar32: precise {truth!r} ({dt:.2f} s); fast rel {abs(fast - truth) / abs(truth):.3e}; "
      f"reference DD tau=4096 rel {abs(ref - truth) / abs(truth):.3e}", flush=True)
h = pk.haar_unitary_block(36, 20261017, m=72)
t0 = time.time()
truth = pk.perm_nw(h, precise=True)
dt = time.time() - t0
fast = pk.perm_nw(h)
print(f"Haar U(72)[:36,:36]: precise {truth!r} ({dt:.1f} s); fast rel "
      f"{abs(fast - truth) / abs(truth):.3e}", flush=True)
