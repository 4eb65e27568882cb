"""Config 5 on the reference CPU path (oracle/_ref, all host cores): one L=32
interior row absorb (r=8, m=64, k=72, q=2; contraction.cpp:269-311) and one
cached 1-row band environment (contraction.cpp:572-624) between m=64
boundaries, timed once each; prints one JSON line.  A full sweep is 31 such
row absorbs; a cached expectation adds the bottom sweep and one
band environment per row."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2006_15234_b200 import inputs as I  # noqa: E402

cores = os.cpu_count() or 1
ref.set_threads(cores)
L, r, m = 32, 8, 64
scale = 1.0 / np.sqrt(r * r * 2)
sites = I.random_peps(3, L, r, 5, scale=scale)
top, phys = I.random_boundary(L, (r, r), m, I.derive_seed(5, 0x70), scale=0.1)
t0 = time.perf_counter()
_, _, info = ref.two_layer_apply_row(top, phys, sites, 3, L, 1, m, 5, 2, 8, True, 0x20)
row = time.perf_counter() - t0
bot, bphys = I.random_boundary(L, (r, r), m, I.derive_seed(5, 0x71), scale=0.1)
band = ref.band_environment_time(top, phys, bot, bphys, sites, 3, L, 1, 1)
print(json.dumps({"config": 5, "cores": cores, "kind": "reference (oracle/_ref, OpenBLAS 0.3.15)",
                  "s_per_row_absorb_L32": row, "reference_counter_flops_row": info["flops"],
                  "s_per_band_environment_1row_L32": band,
                  "s_per_norm_extrapolated": 31 * row,
                  "s_per_cached_expectation_extrapolated": 2 * 31 * row + 32 * band}), flush=True)
