"""Generates tests/golden/golden.npz from the REFERENCE ITSELF (oracle/_ref).

Run in the build container (needs /root/reference compiled by `make -C oracle`):
    python tests/golden/make_golden.py
The reference ships no stored golden vectors; these fixtures are
outputs of its own public API on seeded inputs, so the GPU tests can pin parity
without the oracle library.  Inputs are regenerated from the seeds by
paper_2006_15234_b200/inputs.py and oracle/peps_oracle.py (SplitMix64).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2006_15234_b200 import inputs as I  # noqa: E402

out = {}

# --- SplitMix64 / derive_seed / random_tensor (rng.hpp:12-44, tensor.cpp:192-208)
seeds = np.array([0, 1, 12345, 2 ** 63 + 7], dtype=np.uint64)
out["rng_seeds"] = seeds
out["rng_complex"] = np.stack([ref.random_tensor((3, 5), int(s)) for s in seeds])
out["rng_real"] = np.stack([ref.random_tensor((3, 5), int(s), real=True) for s in seeds])
out["rng_derived"] = np.array([ref.derive_seed(int(s), 0x20, 3, 4) for s in seeds], dtype=np.uint64)


def two_layer_net(r, m, seed):
    v = ref.random_tensor((m, r, r, m, r, r), seed)
    s = ref.random_tensor((r, r, m, m), seed + 1)
    b = ref.random_tensor((2, r, r, r, r), seed + 2)
    return [v, s, b.conj(), b], ["apqsmn", "uvst", "dumbe", "dvncf"]


# --- einsumsvd on a two-layer-shaped network (decomposition.cpp:308-352)
ts, labs = two_layer_net(3, 6, 100)
for absorb in ("split", "left", "right"):
    r = ref.einsumsvd(ts, labs, "apq", "bctef", 6, 1e-14, "implicit_rsvd", absorb, 2, -1, 11)
    out[f"es_tl_{absorb}_s"] = r["s"]
    out[f"es_tl_{absorb}_t1"] = r["t1"]
    out[f"es_tl_{absorb}_t2"] = r["t2"]
r = ref.einsumsvd(ts, labs, "apq", "bctef", 6, 1e-14, "exact", "split", 2, -1, 11)
out["es_tl_exact_s"] = r["s"]

# --- reference test networks (test_decomposition.cpp:209-230, 166-172, 134-145)
chain = [ref.random_tensor(s, sd) for s, sd in (((2, 3), 81), ((3, 2, 4), 82), ((4, 5), 83), ((5, 3, 2), 84),
                                                  ((2, 3), 85))]
chain_l = ["ab", "bcd", "de", "efg", "gh"]
out["es_chain_exact_s"] = ref.einsumsvd(chain, chain_l, "ac", "fh", 4, 1e-14, "exact")["s"]
out["es_chain_rsvd_s"] = ref.einsumsvd(chain, chain_l, "ac", "fh", 4, 1e-14, "implicit_rsvd", "split", 2, -1, 3)["s"]
lmat = ref.random_tensor((8, 5), 41)
rmat = ref.random_tensor((5, 8), 42)
out["rank5_s"] = ref.randomized_svd([lmat @ rmat], ["rc"], "r", "c", 5, 1e-14, 2, -1, 7)["s"]
d = np.zeros((4, 4), dtype=np.complex128)
d[0, 0], d[1, 1], d[2, 2] = 3, 2, 1
out["diag321_s"] = ref.randomized_svd([d], ["rc"], "r", "c", 3, 1e-14, 2, -1, 7)["s"]

# --- gram_orthogonalize (decomposition.cpp:160-193)
a = ref.random_tensor((64, 4), 17)
q, rr = ref.gram_orthogonalize(a, 1)
out["gram_q"], out["gram_r"] = q, rr
base = ref.random_tensor((32, 3), 23)
a2 = np.stack([base[:, 0], base[:, 1], base[:, 0], base[:, 2]], axis=1)
q2, r2 = ref.gram_orthogonalize(a2, 1)
out["gram_def_q"], out["gram_def_r"] = q2, r2

# --- config 1 (4x4, r=2, m=4, oversample 4, q=1) norm and the exact value
c1 = I.config1()
v, _ = ref.contract_two_layer(c1["sites"], 4, 4, 4, c1["seed"], 1, 4)
out["cfg1_norm"] = np.array([v])
out["cfg1_exact"] = np.array([ref.inner_exact(c1["sites"], 4, 4)])

# --- small two-layer row absorb (contraction.cpp:269-311): L=5, r=3, m=9, q=2, oversample -1
sites = I.random_peps(3, 5, 3, 71)
top, phys = I.random_boundary(5, (3, 3), 9, 72)
t, ph, _ = ref.two_layer_apply_row(top, phys, sites, 3, 5, 1, 9, 5, 2, -1, True, 0x20)
for i, s in enumerate(t):
    out[f"row_site{i}"] = s
t, ph, _ = ref.two_layer_apply_row(top, phys, sites, 3, 5, 1, 9, 5, 2, -1, False, 0x20)
for i, s in enumerate(t):
    out[f"row_split_site{i}"] = s

# --- cached environments + bands (observables.cpp:325-333, contraction.cpp:572-650)
c = dict(rows=4, cols=4, sites=I.random_peps(4, 4, 2, 91, scale=1 / np.sqrt(8)))
terms = [(0, i // 4, i % 4, i // 4, i % 4) for i in range(16)]
terms += [(1, 1, 1, 1, 2), (1, 0, 2, 1, 2), (1, 2, 3, 3, 3), (1, 3, 0, 3, 1)]
norm, vals, _ = ref.local_expectations(c["sites"], 4, 4, 4, 13, terms, 2, -1)
out["bands_terms"] = np.array(terms, dtype=np.int64)
out["bands_norm"] = np.array([norm])
out["bands_values"] = vals

np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
print("wrote", os.path.join(HERE, "golden.npz"), sum(v.nbytes for v in out.values()), "bytes")
