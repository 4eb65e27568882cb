"""Developer repro: contract an ITE-evolved 8x8 r=8 state (edge bonds 1) at m=64.

  python tools/repro_ite_contract.py WS [save.npz | load.npz]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_15234_b200.api as A
ctx = A.default_context()
if len(sys.argv) > 1:
    ctx.set_option("gemm_ws", int(sys.argv[1]))
path = sys.argv[2] if len(sys.argv) > 2 else None
if path and os.path.exists(path):
    z = np.load(path)
    out = A.PepsState(8, 8, 2, [z[f"s{i}"] for i in range(64)])
else:
    plus = [np.array([1, 1], dtype=complex).reshape(2, 1, 1, 1, 1) / np.sqrt(2) for _ in range(64)]
    st = A.PepsState(8, 8, 2, plus)
    out = A.ite_tfim(st, 1.0, 3.0, 0.01, int(os.environ.get("STEPS", "5")), 8)
    if path:
        np.savez(path, **{f"s{i}": s.numpy() for i, s in enumerate(out.sites)})
        print("saved", flush=True)
        sys.exit(0)
if os.environ.get("TRACE"):
    os.environ["PEPSB_TRACE"] = "1"
opt = A.ContractOption.two_layer_opt(64, 7, 2, 8)
print(A.contract_two_layer(out, out, opt), flush=True)
