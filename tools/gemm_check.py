"""Developer tool: GEMM correctness sweep over shapes / layouts for each algorithm."""
import sys
sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import paper_2006_15234_b200.api as A  # noqa: E402
from oracle import peps_oracle as O  # noqa: E402

ctx = A.default_context()
algos = [int(a) for a in sys.argv[1].split(',')] if len(sys.argv) > 1 else [0, 1, 2]
shapes = [(70, 90, 300), (64, 64, 64), (72, 72, 72), (128, 300, 64), (65, 70, 17), (5, 7, 3), (200, 72, 130),
          (72, 200, 33), (64, 72, 64), (72, 64, 48), (33, 65, 129), (1, 1, 1), (8, 300, 256), (300, 8, 256)]
specs = ["ik,kj->ij", "ki,kj->ij", "ik,jk->ij", "ki,jk->ij"]
bad = 0
for algo in algos:
    ctx.set_option("gemm_algo", algo)
    for (m, n, k) in shapes:
        for sp in specs:
            a_shape = (m, k) if sp[:2] == "ik" else (k, m)
            b_shape = (k, n) if sp[3:5] == "kj" else (n, k)
            a = O.random_tensor(a_shape, m * 7 + k)
            b = O.random_tensor(b_shape, n * 5 + k)
            got = A.contract(sp, a, b).numpy()
            ref = np.einsum(sp, a, b)
            err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300)
            if err > 1e-12:
                bad += 1
                print(f"FAIL algo={algo} {sp} M={m} N={n} K={k} err={err:.2e}", flush=True)
print("failures:", bad)
