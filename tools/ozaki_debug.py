import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1806_01430_b200 import capi
n = int(sys.argv[1])
rs = np.random.RandomState(1)
a, bt = rs.uniform(-1, 1, (n, n)), rs.uniform(-1, 1, (n, n))
c0 = np.zeros((n, n))
with capi.Context(n=n, dtype=capi.F64, matmul_variant=40) as ctx:
    ctx.upload(capi.ARRAY_A, a); ctx.upload(capi.ARRAY_BT, bt); ctx.upload(capi.ARRAY_C, c0)
    ctx.run_loop(8)
    got = ctx.fetch(capi.ARRAY_C)
exact = a @ bt.T
err = np.abs(got - exact)
bad = err > 1e-9
print("bad fraction", bad.mean())
print("bad rows (by 32):", [int(bad[r:r+32].mean()*100) for r in range(0, n, 32)])
print("bad cols (by 32):", [int(bad[:, c:c+32].mean()*100) for c in range(0, n, 32)])
# which k-range contributes the error? compare with partial products
for k0 in range(0, n, 64):
    part = a[:, k0:k0+64] @ bt[:, k0:k0+64].T
    # correlation of the error with this k block's contribution
    d = (got - exact)
    print(k0, float(np.abs(d + part).mean()), float(np.abs(d).mean()))
    if k0 >= 192: break
