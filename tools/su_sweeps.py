import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2006_15234_b200.api as A
from paper_2006_15234_b200._lib import lib
ctx = A.default_context()
plus = [np.array([1, 1], dtype=complex).reshape(2, 1, 1, 1, 1) / np.sqrt(2) for _ in range(64)]
s = A.ite_tfim(A.PepsState(8, 8, 2, plus), 1.0, 3.0, 0.01, 20, 8)
ctx.sync()
for w in range(40): lib().pepsb_ctx_debug_word(ctx.h, w, 1)
s2 = A.ite_tfim(s, 1.0, 3.0, 0.01, 1, 8)
ctx.sync()
print([lib().pepsb_ctx_debug_word(ctx.h, w, 0) for w in range(40)])
