"""One k x k gram_factors call (k = K env, default 72) for an ncu --set full capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_15234_b200.api as A  # noqa: E402
from oracle import peps_oracle as O  # noqa: E402
n = int(os.environ.get("K", "72"))
a = O.random_tensor((3 * n, n), n)
g = a.conj().T @ a
for _ in range(3):
    A.gram_factors(g)
A.default_context().sync()
