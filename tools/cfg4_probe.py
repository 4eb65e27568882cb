"""Config 4: how accurate is a boundary contraction of the final ITE state?

Runs the reference ITE (oracle/_ref) on |+> and on a 1e-14-perturbed |+>, the
device ITE, and contracts all three final states with the device's two-layer
BMPS at several m (sites rescaled by their max |entry|, log scale carried).
Prints one JSON line per (state, m).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2006_15234_b200.api as A  # noqa: E402
from fullsize_common import perturb  # noqa: E402
from oracle import ref  # noqa: E402

ms = [int(x) for x in (sys.argv[1:] or ["16", "32", "64", "96", "128"])]
ref.set_threads(os.cpu_count() or 1)
plus = [np.array([1, 1], dtype=complex).reshape(2, 1, 1, 1, 1) / np.sqrt(2) for _ in range(64)]
states = {}
t0 = time.time()
states["ref"], _ = ref.ite_tfim(plus, 8, 8, 1.0, 3.0, 0.01, 100, 8)
states["ref_pert"], _ = ref.ite_tfim(perturb(plus, 1e-14), 8, 8, 1.0, 3.0, 0.01, 100, 8)
print("ref ITE", time.time() - t0, flush=True)
dev = A.ite_tfim(A.PepsState(8, 8, 2, plus), 1.0, 3.0, 0.01, 100, 8)
states["dev"] = [s.numpy() for s in dev.sites]
for name, sites in states.items():
    mx = [float(np.abs(s).max()) for s in sites]
    scaled = [s / m for s, m in zip(sites, mx)]
    st = A.PepsState(8, 8, 2, scaled)
    for m in ms:
        t0 = time.time()
        opt = A.ContractOption.two_layer_opt(m, 7, 2, 8)
        try:
            e = A.expectation(st, A.tfim_terms(8, 8, 1.0, 3.0), A.ExpectationOptions(opt, True, True, True))
            ln = float(np.log(abs(e.norm_sq)) + 2 * np.log(mx).sum())
            print(json.dumps({"state": name, "m": m, "log_norm": ln, "energy": e.value, "energy_imag": e.complex_value.imag if hasattr(e, "complex_value") else None, "s": time.time() - t0}),
                  flush=True)
        except Exception as ex:  # noqa: BLE001
            print(json.dumps({"state": name, "m": m, "error": str(ex)}), flush=True)
