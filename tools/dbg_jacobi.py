"""Developer tool: time gram_orthogonalize (k x k Jacobi) on the device; sweeps used."""
import sys, time; sys.path.insert(0,'.')
import numpy as np
import paper_2006_15234_b200.api as A
from paper_2006_15234_b200._lib import lib
from oracle import peps_oracle as O
ctx = A.default_context()
for k in (16, 41, 64, 72):
    y = O.random_tensor((4096, k), 3) @ np.diag(np.logspace(0, -5, k))
    for it in range(3):
        lib().pepsb_ctx_debug_word(ctx.h, 7, 1)
        ctx.profile(True)
        q, r = A.gram_orthogonalize(y, 1)
        rep = ctx.profile_report(); ctx.profile(False)
        sw = lib().pepsb_ctx_debug_word(ctx.h, 7, 1)
    u, s, v = A.svd(y, 1)
    sw2 = lib().pepsb_ctx_debug_word(ctx.h, 7, 1)
    qq = q.numpy()
    print(k, "small ms", rep["small"]["ms"], "sweeps", sw, "svd sweeps", sw2, "orth err", np.abs(qq.conj().T @ qq - np.eye(k)).max(), flush=True)
for w in (8, 9, 10):
    print("stage word", w, lib().pepsb_ctx_debug_word(ctx.h, w, 1), "kcycles (cumulative)")
