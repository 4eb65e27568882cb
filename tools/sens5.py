"""Developer tool: rounding sensitivity of the config-5 norm (overlap off/on, input perturbed 1e-14)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_15234_b200.api as A
from paper_2006_15234_b200 import inputs
ctx = A.default_context()
c = inputs.config5()
n = int(os.environ.get("N", "32"))
sites = c["sites"] if n == 32 else inputs.random_peps(n, n, 8, 5, scale=1 / np.sqrt(128))
rs = np.random.default_rng(3)
pert = [x * (1.0 + 1e-14 * rs.standard_normal()) for x in sites]
opt = A.ContractOption.two_layer_opt(64, c["seed"], 2, 8)
out = {}
for ov in (0, 1):
    ctx.set_option("overlap", ov)
    for name, ss in (("base", sites), ("pert", pert)):
        st = A.PepsState(n, n, 2, ss, ctx=ctx)
        v = A.contract_two_layer(st, st, opt)
        out[f"ov{ov}_{name}"] = [v.real, v.imag]
        del st
b = complex(*out["ov0_base"])
for k, v in out.items():
    print(k, v, abs(complex(*v) - b) / abs(b))
