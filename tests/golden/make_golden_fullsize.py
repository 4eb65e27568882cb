"""Full-size golden values from the REFERENCE ITSELF (oracle/_ref), per BASELINE config.

TEST INFRASTRUCTURE ONLY.  Run in the build container (needs /root/reference
compiled by `make -C oracle`); each section is written to its own small .npz
under tests/golden/ as soon as it finishes (the whole run is hours of CPU):

    python tests/golden/make_golden_fullsize.py [section ...] [--threads N]

Sections (inputs regenerated from seeds by paper_2006_15234_b200/inputs.py):
  cfg2_row   two_layer_apply_row (contraction.cpp:269-311) on config 2 (L=8, m=64,
             r=8, k=72, q=2): gauge-invariant overlaps <b|b>, <x|b> of the emitted
             boundary with a fixed seeded MPS x, plus the site shapes.  ~6 min/8 cores.
  cfg2_col   one interior-column einsumsvd of config 2 (decomposition.cpp:308-352):
             singular values.  ~40 s.
  cfg3       config 3 (16x16, r=6, m=36, q=2, os=-1): cached norm + all 256 <Z_i>
             (observables.cpp:325-422).  ~25 min.
  cfg3_pert  config 3 with every site multiplied by (1 + 1e-14 xi): the
             reference's own rounding sensitivity of the 256 <Z_i>.  ~25 min.
  cfg5_8x8   config-5 parameters (r=8, m=64, q=2, os=8, N(0,1/128)) on an 8x8
             lattice: cached norm, <ZZ> on all 56 horizontal bonds and <Z> at
             the centre (one-row bands only: the reference's two-row band zipper
             for a vertical bond exceeds 62 GB here).  ~80 min.
  cfg5_12x12_norm  config-5 parameters on a 12x12 lattice: the norm by contract_two_layer.  ~65 min.
  cfg5_8x8_pert  the same lattice with every site multiplied by (1 + 1e-14 xi):
             the reference's own rounding sensitivity at this size.  ~80 min.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))  # tests/ (as pytest sees it)

from oracle import ref  # noqa: E402
from paper_2006_15234_b200 import inputs as I  # noqa: E402
from fullsize_common import (CFG2_COL_SEED, boundary_overlaps, cfg2_column_net, cfg5_small,  # noqa: E402
                             cfg5_terms, perturb)


def save(name, **kw):
    p = os.path.join(os.environ.get("GOLDEN_OUT", HERE), f"fullsize_{name}.npz")
    np.savez_compressed(p, **kw)
    print(f"wrote {p}", flush=True)


def sec_cfg2_col():
    ts, labels, seed = cfg2_column_net(CFG2_COL_SEED)
    t0 = time.time()
    r = ref.einsumsvd(ts, labels, "apq", "bctef", 64, 1e-14, "implicit_rsvd", "right", 2, 8, seed)
    save("cfg2_col", s=r["s"], seconds=np.array([time.time() - t0]))


def sec_cfg2_row():
    c2 = I.config2()
    t0 = time.time()
    t, phys, info = ref.two_layer_apply_row(c2["top"], c2["phys"], c2["sites"], 3, 8, 1, 64, c2["seed"], 2, 8,
                                            True, 0x20)
    bb, xb = boundary_overlaps(t)
    save("cfg2_row", bb=np.array([bb]), xb=np.array([xb]),
         shapes=np.array([s.shape for s in t], dtype=np.int64), seconds=np.array([time.time() - t0]))


def sec_cfg3(eps=0.0, name="cfg3"):
    c = I.config3()
    if eps:
        c["sites"] = perturb(c["sites"], eps)
    n = c["rows"]
    terms = [(0, i // n, i % n, i // n, i % n) for i in range(n * n)]
    t0 = time.time()
    norm, vals, info = ref.local_expectations(c["sites"], n, n, c["m"], c["seed"], terms, c["power_iters"],
                                              c["oversample"])
    save(name, norm=np.array([norm]), z=vals, terms=np.array(terms, dtype=np.int64), eps=np.array([eps]),
         t_cache=np.array([info["t_cache"]]), t_bands=np.array([info["t_bands"]]),
         seconds=np.array([time.time() - t0]))


def _cfg5(name, eps):
    c = cfg5_small()
    sites = perturb(c["sites"], eps) if eps else c["sites"]
    n = c["rows"]
    terms = cfg5_terms(n)
    t0 = time.time()
    norm, vals, info = ref.local_expectations(sites, n, n, c["m"], c["seed"], terms, c["power_iters"],
                                              c["oversample"])
    save(name, norm=np.array([norm]), values=vals, terms=np.array(terms, dtype=np.int64),
         t_cache=np.array([info["t_cache"]]), seconds=np.array([time.time() - t0]), eps=np.array([eps]))


def sec_cfg5_12x12_norm_pert():
    """The same 12x12 norm with every site multiplied by (1 + 1e-14 xi): the reference's own
    rounding sensitivity at this size.  ~65 min."""
    c = cfg5_small(12)
    t0 = time.time()
    val = ref.contract_two_layer(perturb(c["sites"], 1e-14), 12, 12, c["m"], c["seed"], c["power_iters"],
                                 c["oversample"])
    save("cfg5_12x12_norm_pert", norm=np.array([val[0] if isinstance(val, tuple) else val]),
         seconds=np.array([time.time() - t0]), eps=np.array([1e-14]))


def sec_cfg5_12x12_norm():
    """<psi|psi> of a 12x12 lattice with the config-5 parameters by contract_two_layer
    (contraction.cpp:313-338): 11 row absorbs of 12 columns at m = 64, r = 8.  ~65 min."""
    c = cfg5_small(12)
    t0 = time.time()
    val = ref.contract_two_layer(c["sites"], 12, 12, c["m"], c["seed"], c["power_iters"], c["oversample"])
    save("cfg5_12x12_norm", norm=np.array([val[0] if isinstance(val, tuple) else val]),
         seconds=np.array([time.time() - t0]))


SECTIONS = {"cfg2_col": sec_cfg2_col, "cfg2_row": sec_cfg2_row, "cfg3": sec_cfg3,
            "cfg3_pert": lambda: sec_cfg3(1e-14, "cfg3_pert"),
            "cfg5_8x8": lambda: _cfg5("cfg5_8x8", 0.0), "cfg5_8x8_pert": lambda: _cfg5("cfg5_8x8_pert", 1e-14),
            "cfg5_12x12_norm": sec_cfg5_12x12_norm, "cfg5_12x12_norm_pert": sec_cfg5_12x12_norm_pert}

if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    threads = os.cpu_count() or 1
    if "--threads" in sys.argv:
        threads = int(sys.argv[sys.argv.index("--threads") + 1])
        args = [a for a in args if a != str(threads)]
    ref.set_threads(threads)
    for name in args or list(SECTIONS):
        t0 = time.time()
        SECTIONS[name]()
        print(f"{name}: {time.time() - t0:.1f} s", flush=True)
