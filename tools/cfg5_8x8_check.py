"""Developer tool: device vs reference golden on the 8x8 lattice with the config-5 parameters
(tests/golden/fullsize_cfg5_8x8.npz), for both complex-GEMM schemes."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2006_15234_b200.api as A
from fullsize_common import cfg5_small, cfg5_terms, device_local_expectations
g = np.load(os.path.join(ROOT, "tests", "golden", "fullsize_cfg5_8x8.npz"))
pp = os.path.join(ROOT, "tests", "golden", "fullsize_cfg5_8x8_pert.npz")
gp = np.load(pp) if os.path.exists(pp) else None
c = cfg5_small()
ctx = A.default_context()
for algo in (1, 2):
    ctx.set_option("gemm_algo", algo)
    st = A.PepsState(8, 8, 2, c["sites"])
    opt = A.ContractOption.two_layer_opt(c["m"], c["seed"], c["power_iters"], c["oversample"])
    terms = [tuple(t) for t in g["terms"]]
    ctx.sync()
    t0 = time.perf_counter()
    norm, vals = device_local_expectations(A, st, opt, terms)
    ctx.sync()
    print("gemm_algo", algo, "seconds (cache + 57 terms)", round(time.perf_counter() - t0, 3), "norm rel err", abs(norm - g["norm"][0]) / abs(g["norm"][0]), "max value err",
          float(np.max(np.abs(vals - g["values"]))), flush=True)
if gp is not None:
    print("reference spread: norm", abs(gp["norm"][0] - g["norm"][0]) / abs(g["norm"][0]), "values",
          float(np.max(np.abs(gp["values"] - g["values"]))))
ctx.set_option("gemm_algo", 1)
