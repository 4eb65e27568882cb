"""Config 1 (4x4 r=2 norm, m=4) latency anatomy: wall per norm, then NORMS norms for an ncu launch list."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_15234_b200.api as A  # noqa: E402
from paper_2006_15234_b200 import inputs  # noqa: E402
c = inputs.config1()
ctx = A.default_context()
st = A.PepsState(4, 4, 2, c["sites"], ctx=ctx)
opt = A.ContractOption.two_layer_opt(4, c["seed"], 1, 4)
for _ in range(3):
    A.contract_two_layer(st, st, opt)
n = int(os.environ.get("NORMS", "20"))
t0 = time.perf_counter()
for _ in range(n):
    A.contract_two_layer(st, st, opt)
print("wall ms/norm %.3f" % (1e3 * (time.perf_counter() - t0) / n), flush=True)
