"""Scratch GPU sanity run (developer tool): library vs oracle on small cases + cfg2 timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import ref
import paper_2006_15234_b200.api as A
from paper_2006_15234_b200 import inputs as I

def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(1e-300, np.linalg.norm(np.asarray(b)))

ctx = A.default_context()
t = A.random_tensor((3, 4, 5), 77).numpy()
print("random bitwise:", np.array_equal(t, ref.random_tensor((3, 4, 5), 77)))
a = ref.random_tensor((6, 7, 8), 1); b = ref.random_tensor((8, 9), 2)
print("contract:", rel(A.contract("abc,cd->abd", a, b).numpy(), np.einsum("abc,cd->abd", a, b)))
c = ref.random_tensor((6, 8, 5), 3)
print("contract T:", rel(A.contract("abc,acd->bd", a, c).numpy(), np.einsum("abc,acd->bd", a, c)))
big = ref.random_tensor((70, 300), 4); b2 = ref.random_tensor((300, 90), 5)
print("gemm:", rel(A.contract("ik,kj->ij", big, b2).numpy(), big @ b2))
# implicit two-layer network r=2, m=4
r, m = 3, 5
v = ref.random_tensor((m, r, r, m, r, r), 11); S = ref.random_tensor((r, r, m, m), 12)
B = ref.random_tensor((2, r, r, r, r), 13); K = ref.random_tensor((2, r, r, r, r), 14)
ts = [v, S, B.conj(), K]; labs = ["apqsmn", "uvst", "dumbe", "dvncf"]
op = A.ImplicitOperator(ts, labs, "apq", "bctef")
q = ref.random_tensor((r, r, m, r, r, 7), 15)
print("apply:", rel(op.apply(q).numpy(), ref.implicit_apply(ts, labs, "apq", "bctef", q)))
p = ref.random_tensor((m, r, r, 7), 16)
print("adjoint:", rel(op.adjoint_apply(p).numpy(), ref.implicit_apply(ts, labs, "apq", "bctef", p, adjoint=True)))
print("materialize:", rel(op.materialize().numpy(), ref.materialize(ts, labs, "apq", "bctef")))
# gram
y = ref.random_tensor((40, 3, 6), 21)
qg, rg = A.gram_orthogonalize(y, 1)
qr_, rr_ = ref.gram_orthogonalize(y, 1)
print("gram Q:", rel(qg.numpy(), qr_), "R:", rel(rg.numpy(), rr_))
us, ss, vs = A.svd(y, 1); ur, sr, vr = ref.svd(y, 1)
print("svd s:", rel(ss, sr), "u:", rel(us.numpy(), ur), "v:", rel(vs.numpy(), vr))
# einsumsvd implicit
for strat in ("implicit_rsvd", "exact"):
    res = A.einsumsvd(op, A.TruncationPolicy(6, 1e-14), A.SvdStrategy[strat], A.Absorb.left, A.RsvdConfig(2, -1, 99))
    rr = ref.einsumsvd(ts, labs, "apq", "bctef", 6, 1e-14, strat, "left", 2, -1, 99)
    print(strat, "s:", rel(res.s, rr["s"]), "t1:", rel(res.t1.numpy(), rr["t1"]), "t2:", rel(res.t2.numpy(), rr["t2"]))
# cfg1
c1 = I.config1()
st = A.PepsState(4, 4, 2, c1["sites"])
opt = A.ContractOption.two_layer_opt(4, c1["seed"], 1, 4)
g = A.contract_two_layer(st, st, opt)
o, _ = ref.contract_two_layer(c1["sites"], 4, 4, 4, c1["seed"], 1, 4)
print("cfg1 norm gpu", g, "ref", o, "rel", abs(g - o) / abs(o))
# cfg2 row absorb
c2 = I.config2()
st2 = A.PepsState(3, 8, 2, c2["sites"])
top = A.TwoLayerBoundary.from_sites(c2["top"], c2["phys"])
opt2 = A.ContractOption.two_layer_opt(64, c2["seed"], 2, 8)
for it in range(3):
    ctx.sync(); t0 = time.time()
    outb = A.two_layer_apply_row(top, st2, st2, 1, opt2, 0x20)
    ctx.sync(); dt = time.time() - t0
    print("cfg2 row absorb s:", dt, ctx.counters())
sites = [s.numpy() for s in outb.sites]
print([s.shape for s in sites])
np.save("gpurun_out/cfg2_gpu_sites.npy", np.array(sites, dtype=object), allow_pickle=True)
