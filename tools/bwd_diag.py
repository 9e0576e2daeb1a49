import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_bwd import run_bwd
from paper_2603_22300_b200 import sfa as lib
for shape in [(1, 2, 1, 256, 128, 128, 16), (1, 4, 2, 300, 128, 128, 16), (2, 2, 2, 200, 64, 64, 8)]:
    gpu, ref = run_bwd(lib, 91 + shape[3], *shape)
    rq, rk, rv, bq, bk, bv = ref
    for name, g, r, b, c in (("dq", gpu[0], rq, bq, 2**-7), ("dk", gpu[1], rk, bk, 2**-7), ("dv", gpu[2], rv, bv, 2**-8)):
        err = np.abs(g - r)
        print(shape, name, "max|r| %.3g  max err %.3g  rel-L2 %.3g  max err/tol %.3g  max |r|/b %.3g  median |r|/b %.3g" % (
            np.abs(r).max(), err.max(), np.linalg.norm(g - r) / np.linalg.norm(r), (err / (c * b + 1e-6)).max(),
            (np.abs(r) / (b + 1e-30)).max(), np.median(np.abs(r) / (b + 1e-30))))
