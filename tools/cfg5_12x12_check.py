"""Developer tool: device vs reference on the 12x12 lattice with the config-5 parameters (norm by
contract_two_layer; tests/golden/fullsize_cfg5_12x12_norm.npz), both complex-GEMM schemes, with timing."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2006_15234_b200.api as A
from fullsize_common import cfg5_small
g = np.load(os.path.join(ROOT, "tests", "golden", "fullsize_cfg5_12x12_norm.npz"))
c = cfg5_small(12)
ctx = A.default_context()
for algo in (1, 2):
    ctx.set_option("gemm_algo", algo)
    st = A.PepsState(12, 12, 2, c["sites"])
    opt = A.ContractOption.two_layer_opt(c["m"], c["seed"], c["power_iters"], c["oversample"])
    A.contract_two_layer(st, st, opt); ctx.sync()
    t0 = time.perf_counter(); norm = A.contract_two_layer(st, st, opt); ctx.sync()
    print("gemm_algo", algo, "seconds", round(time.perf_counter() - t0, 3), "norm rel err",
          abs(norm - g["norm"][0]) / abs(g["norm"][0]), "(reference:", float(g["seconds"][0]), "s)", flush=True)
ctx.set_option("gemm_algo", 1)
