"""One config-3 row absorb (row 8 of the 16x16 lattice, after a warm-up absorb) for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_15234_b200.api as A  # noqa: E402
from paper_2006_15234_b200 import inputs  # noqa: E402
c = inputs.config3()
st = A.PepsState(16, 16, 2, c["sites"])
opt = A.ContractOption.two_layer_opt(36, c["seed"], 2, -1)
b = A.two_layer_first_row(st, st)
for r in range(1, 8):
    b = A.two_layer_apply_row(b, st, st, r, opt, 0x20)
A.default_context().sync()
print("ready", flush=True)
for i in range(2):
    out = A.two_layer_apply_row(b, st, st, 8, opt, 0x20)
    A.default_context().sync()
print("done", flush=True)
