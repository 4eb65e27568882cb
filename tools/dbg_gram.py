"""Developer tool: Jacobi sweep counts on dumped Gram matrices (PEPSB_DUMP_GRAM)."""
import glob
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_2006_15234_b200.api as A  # noqa: E402
from paper_2006_15234_b200._lib import lib  # noqa: E402

ctx = A.default_context()
for f in sorted(glob.glob(sys.argv[1] + "*.bin")):
    g = np.fromfile(f, dtype=np.complex128)
    k = int(round(len(g) ** 0.5))
    G = g.reshape(k, k)
    G = 0.5 * (G + G.conj().T)
    s = np.sqrt(np.real(np.diag(G)).max())
    y = np.linalg.cholesky(G / s**2).conj().T  # y^H y = G / s^2
    lib().pepsb_ctx_debug_word(ctx.h, 7, 1)
    q, r = A.gram_orthogonalize(y, 1)
    sw = lib().pepsb_ctx_debug_word(ctx.h, 7, 1)
    qq = q.numpy()
    print(f, "sweeps", sw, "orth err %.2e" % np.abs(qq.conj().T @ qq - np.eye(k)).max(), flush=True)
