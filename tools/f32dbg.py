import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import paper_1204_1586_b200 as cpd, oracle as O
ctx = cpd.Context(0)
for dims, R in [([16,16,16,16],5), ([40,40,40,40],64), ([7,9,11,13],8), ([300,300,20],16), ([12,10,14,9,8],70)]:
    y = cpd.DenseTensor.generate(dims, cpd.DIST_UNIFORM_PM1, seed=11, ctx=ctx, dtype=cpd.F32)
    yv = y.values().astype(np.float64)
    f = [O.fill_normal(110 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
    try:
        g = cpd.cp_gradient_all(y, f)
    except Exception as e:
        print(dims, R, "ERR", e); continue
    w, _, _ = O.cp_gradient_all(yv, dims, f)
    print(dims, R, ["%.2e" % (np.linalg.norm(a-b)/np.linalg.norm(b)) for a, b in zip(g, w)], flush=True)
