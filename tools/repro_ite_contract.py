"""Developer repro: contract an ITE-evolved 8x8 r=8 state (edge bonds 1) at m=64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_15234_b200.api as A
ctx = A.default_context()
if len(sys.argv) > 1:
    ctx.set_option("gemm_ws", int(sys.argv[1]))
plus = [np.array([1, 1], dtype=complex).reshape(2, 1, 1, 1, 1) / np.sqrt(2) for _ in range(64)]
st = A.PepsState(8, 8, 2, plus)
out = A.ite_tfim(st, 1.0, 3.0, 0.01, int(os.environ.get("STEPS", "5")), 8)
print([s.shape for s in out.sites[:9]], flush=True)
os.environ["PEPSB_TRACE_GEMM"] = "1"
opt = A.ContractOption.two_layer_opt(64, 7, 2, 8)
print(A.contract_two_layer(out, out, opt), flush=True)
