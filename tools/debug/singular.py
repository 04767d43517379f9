"""Debug: exactly singular small-integer case, GPU vs oracle rotations/pivots."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from conftest import golden  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2101_05063_b200 import _lib, solver  # noqa: E402

O.build()
g = golden("singular")
t = str(g["tags"][0])
h, lam = g[f"{t}_h"], g[f"{t}_lam"]
n = h.shape[0]
print("h=\n", h, "\nlam", lam)
k = n
hdiag = np.ascontiguousarray(h[0:k, 0:k - 1])
rr = np.ascontiguousarray(np.repeat(h[0:k, k - 1:k], lam.size, 1))
rr[k - 1] -= lam
st, c, s = O.reduce_diag(hdiag, np.zeros(k), 0, lam, rr)
print("oracle reduce st", st)
x = np.ones((k, lam.size))
st2, xo, be = O.solve_rsolve(hdiag, np.zeros(k), 0, lam, rr, c, s, x, np.zeros(lam.size), True,
                             np.finfo(float).max / 2 / 8)
print("oracle solve st", hex(st2))
out, _ = solver.solve_group(h, None, lam, np.ones((n, lam.size)), 8, mode="solve")
print("gpu nfail", out.nfail, [hex(int(v)) for v in out.fail.cpu().numpy()])
cg = out.c_re.cpu().numpy()
sg = out.s.cpu().numpy()
print("c shape", cg.shape)
cg = cg.reshape(-1, cg.shape[-1]) if cg.ndim > 1 else cg
for q in range(lam.size):
    print("shift", q, "c eq", np.array_equal(cg[q][:n], c[:, q]), "s eq", np.array_equal(sg[q][:n], s[:, q]))
    print("  gpu c", cg[q][:n].tolist())
    print("  orc c", c[:, q].tolist())
    print("  gpu s", sg[q][:n].tolist())
    print("  orc s", s[:, q].tolist())
print("X gpu", out.X.cpu().numpy()[:, :n])
