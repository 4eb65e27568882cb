"""Developer tool: run the device eigensolver on a dumped k x k Gram (PEPSB_DUMP_EIG)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_15234_b200.api as A
g = np.fromfile(sys.argv[1], dtype=np.complex128)
n = int(round(np.sqrt(g.size)))
g = g.reshape(n, n)
w = np.linalg.eigvalsh(g)[::-1]
print("n", n, "lam max %.3e min %.3e" % (w[0], w[-1]), "count < 1e-12 lmax:", int((w < 1e-12 * w[0]).sum()), flush=True)
ctx = A.default_context()
if len(sys.argv) > 2:
    ctx.set_option("eig_solver", int(sys.argv[2]))
r = A.gram_factors(g)
print("ok", [x.shape if hasattr(x, "shape") else x for x in r], flush=True)
