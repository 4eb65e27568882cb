"""Developer tool: k x k eigensolver timing per solver and size (CUDA events, warm)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_15234_b200.api as A
from oracle import peps_oracle as O
ctx = A.default_context()
for n in (4, 8, 12, 16, 24, 32, 41, 48, 64, 72):
    a = O.random_tensor((3 * n, n), n)
    g = a.conj().T @ a  # Gram-like, positive definite
    res = []
    for solver in (0, 2, 1):
        ctx.set_option("eig_solver", solver)
        for _ in range(3):
            A.gram_factors(g)
        ctx.profile(True)
        for _ in range(10):
            A.gram_factors(g)
        rep = ctx.profile_report()
        ctx.profile(False)
        res.append(rep["small"]["ms"] / max(1, rep["small"]["launches"]))
    print(n, "auto %.4f ms  dc %.4f ms  jacobi %.4f ms" % tuple(res), flush=True)
ctx.set_option("eig_solver", 0)
