"""Config 2 shift 904 (singular in the reference's instance): what the GPU does.

Prints the oracle's verdict and the GPU's fail code / represented norm for
shifts 903-905 solved alone and for the whole config-2 selection.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]
import instances  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2101_05063_b200 import solver  # noqa: E402

O.build()
O.use_reference_blas(True)
h = instances.make_h(2)
lam = instances.shifts(2)
n = h.shape[0]
rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
start = rho * np.ones(n)
for idx in (903, 904, 905):
    try:
        r = O.solve(h, lam[idx:idx + 1], start[:, None], 128, b_c=1, mode="eigvec")
        ov = f"ok log2norm={r.log2norm[0]:.3f}"
    except O.OracleError as e:
        ov = f"ERR {e}"
    out, _ = solver.solve_group(h, None, lam[idx:idx + 1], start, 128)
    print(idx, "oracle:", ov, "| gpu: fail", hex(int(out.fail.cpu()[0])), "log2norm",
          float(out.log2norm.cpu()[0]), flush=True)
out, _ = solver.solve_group(h, None, lam, start, 128)
f = out.fail.cpu().numpy()
print("whole selection: nfail", out.nfail, "failing", np.nonzero(f)[0].tolist(),
      [hex(int(c)) for c in f[f != 0]])
