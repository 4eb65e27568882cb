"""Developer tool: one n x n eigh (for ncu)."""
import sys
sys.path.insert(0, '.')
import paper_2006_15234_b200.api as A  # noqa: E402
from oracle import peps_oracle as O  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 72
ctx = A.default_context()
ctx.set_option("eig_solver", int(sys.argv[2]) if len(sys.argv) > 2 else 0)
a = O.random_tensor((n, n), n)
for _ in range(2):
    A.eigh(0.5 * (a + a.conj().T))
ctx.sync()
print("ok")
