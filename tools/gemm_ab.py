"""A/B of a GEMM-kernel option on the config-2 shapes and on one whole row absorb.

  python tools/gemm_ab.py [option] [value_a] [value_b]     (default: gemm_stream 0 1)

For each representative contraction of the operator chain (GEMMs (1)/(2) with
the real bra/ket operand, a complex K=64 product) and for one config-2 row
absorb: device time per call (CUDA events on the library stream, median of 5)
under both settings, and whether the results are bitwise identical.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2006_15234_b200.api as A  # noqa: E402
from paper_2006_15234_b200 import inputs  # noqa: E402

opt_name = sys.argv[1] if len(sys.argv) > 1 else "gemm_stream"
va, vb = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 1)
ctx = A.default_context()
stream = torch.cuda.ExternalStream(ctx.stream)


def timed(fn, reps=5):
    fn()
    ctx.sync()
    ts = []
    out = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = fn()
        e1.record(stream)
        ctx.sync()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2], out


bra = A.to_device(inputs.gaussian((2, 8, 8, 8, 8), 3))
omega = A.random_tensor((8, 8, 64, 8, 8, 72), 5)
w1c = A.random_tensor((2, 8, 64, 8, 64, 8, 72), 6)  # (d,u,m,c,t,f,X) complex
zbig = A.random_tensor((262144, 72), 21)
cases = {
    "Gram Z^H Z 262144 x 72": lambda: A.gram(zbig),
    "G1 bra*(dum|be).Omega(be|ctfX) 128x64x294912 cxr": lambda: A.contract("dumbe,bctefX->dumctfX", bra.conj(), omega),
    "G2 ket(vn|dcf).W1(dcf|umtX) 64x128x294912 cxr": lambda: A.contract("dvncf,dumctfX->vnumtX", bra,
                                                                          A.contract("dumbe,bctefX->dumctfX",
                                                                                     bra.conj(), omega)),
    "C64 complex (ab|k).(k|n) 128x64x294912": lambda: A.contract("uvst,vnumtX->snmX",
                                                                   A.random_tensor((8, 8, 64, 8), 9),
                                                                   A.random_tensor((8, 8, 8, 64, 8, 72), 10)),
}
res = {"option": opt_name, "values": [va, vb], "cases": {}}
for name, fn in cases.items():
    outs, times = [], []
    for v in (va, vb):
        ctx.set_option(opt_name, v)
        t, o = timed(fn)
        times.append(t)
        outs.append(o.numpy())
    res["cases"][name] = {"ms": times, "bitwise_equal": bool(np.array_equal(outs[0], outs[1]))}

c2 = inputs.config2()
st = A.PepsState(3, 8, 2, c2["sites"])
tb = A.TwoLayerBoundary.from_sites(c2["top"], c2["phys"])
opt = A.ContractOption.two_layer_opt(64, c2["seed"], 2, 8)
rows = []
for v in (va, vb):
    ctx.set_option(opt_name, v)
    t, o = timed(lambda: A.two_layer_apply_row(tb, st, st, 1, opt, 0x20))
    rows.append((t, [s.numpy() for s in o.sites]))
res["row_absorb_ms"] = [rows[0][0], rows[1][0]]
res["row_bitwise_equal"] = all(np.array_equal(a, b) for a, b in zip(rows[0][1], rows[1][1]))

# config-5 shapes (L = 32, m = 64, r = 8) with a COMPLEX top boundary (as every
# boundary after the first row is): the chain then runs 3M products
L5 = 32
sites5 = inputs.random_peps(3, L5, 8, 11, scale=1 / np.sqrt(128))
top5, phys5 = inputs.random_boundary(L5, (8, 8), 64, 12, scale=0.1)
top5 = [t * np.exp(1j * inputs.gaussian(t.shape, 13 + i).real) for i, t in enumerate(top5)]
st5 = A.PepsState(3, L5, 2, sites5)
tb5 = A.TwoLayerBoundary.from_sites(top5, phys5)
rows5 = []
for v in (va, vb):
    ctx.set_option(opt_name, v)
    t, o = timed(lambda: A.two_layer_apply_row(tb5, st5, st5, 1, opt, 0x20), reps=3)
    rows5.append((t, [s.numpy() for s in o.sites]))
res["row_cfg5_complex_ms"] = [rows5[0][0], rows5[1][0]]
res["row_cfg5_bitwise_equal"] = all(np.array_equal(a, b) for a, b in zip(rows5[0][1], rows5[1][1]))
ctx.set_option(opt_name, vb)
print(json.dumps(res, indent=1))
