"""int8 fused seed debugging: one gradient per (shape, R) in a subprocess with a
timeout; prints the relative Frobenius error per mode against the oracle."""
import subprocess
import sys

CASES = [((16, 16, 16), 20), ((60, 60, 60), 20), ((60, 60, 60, 60), 16), ((30, 30, 30, 30), 20),
         ((60, 60, 60, 60), 20), ((200, 200, 200), 10), ((14,) * 7, 10)]

CHILD = r'''
import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_1204_1586_b200 as cpd
from oracle import oracle
dims, R = eval(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(1)
y = rng.standard_normal(int(np.prod(dims)))
fac = [rng.standard_normal((d, R)) for d in dims]
ctx = cpd.default_context()
t = cpd.DenseTensor.from_values(y, dims, ctx=ctx)
t0 = time.time()
for _ in range(int(sys.argv[3])):
    g = cpd.cp_gradient_all(t, fac)
ctx.synchronize()
dt = time.time() - t0
want = oracle.cp_gradient_all(y, dims, fac)[0] if np.prod(dims) <= 2e7 else None
errs = [float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(g, want)] if want is not None else []
print(dims, R, "ok %.3fs" % dt, " ".join("%.2e" % e for e in errs))
'''

for dims, R in CASES:
    try:
        r = subprocess.run([sys.executable, "-c", CHILD, repr(dims), str(R), sys.argv[2] if len(sys.argv) > 2 else "1"], capture_output=True, text=True,
                           timeout=int(sys.argv[1]) if len(sys.argv) > 1 else 60)
        print(r.stdout.strip() or r.stderr.strip()[-500:], flush=True)
    except subprocess.TimeoutExpired:
        print(dims, R, "TIMEOUT", flush=True)
