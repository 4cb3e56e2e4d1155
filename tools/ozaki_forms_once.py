"""One auto-mode launch of gene 8 per digit-pair form on synthetic integer operands (N = 1024; 96-wide tiles leave a ragged last
column tile), for compute-sanitizer: python tools/ozaki_forms_once.py [forms as "da,db" ...]   default: 2,2 3,2 2,3 3,3 4,4 5,1"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1806_01430_b200 import capi

n = 1024
pairs = [tuple(int(x) for x in p.split(",")) for p in sys.argv[1:]] or [(2, 2), (3, 2), (2, 3), (3, 3), (4, 4), (5, 1)]
rs = np.random.RandomState(1)


def ints(digits):
    top = 2 ** (7 * digits - 1)
    x = rs.randint(-top + 1, top, (n, n)).astype(np.float64)
    x[:, 0] = top - 1
    return x


for da, db in pairs:
    a, bt = ints(da), ints(db)
    with capi.Context(n=n, dtype=capi.F64, launch_batching=0) as ctx:
        ctx.upload(capi.ARRAY_A, a)
        ctx.upload(capi.ARRAY_BT, bt)
        ctx.run_loop(4)
        ctx.run_loop(8)
        got = ctx.fetch(capi.ARRAY_C)
        exact = (a.astype(np.int64) @ bt.astype(np.int64).T).astype(np.float64)
        print(f"digits {da} x {db}: form {ctx.gene8_form()}, max |error| / |exact| = {np.abs(got - exact).max() / np.abs(exact).max():.2e}", flush=True)
