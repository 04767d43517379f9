"""Where do two race_fuzz.py dumps differ (diagnostics)."""
import sys

import numpy as np

a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
for k in a.files:
    x, y = np.atleast_1d(a[k]), np.atleast_1d(b[k])
    if np.array_equal(x.view(np.uint8), y.view(np.uint8)):
        continue
    if x.dtype == np.float64:
        d = np.nonzero(x.view(np.int64) != y.view(np.int64))
        rel = np.abs(x - y).max() / max(np.abs(x).max(), 1e-300)
        print(f"{k} {x.shape}: {d[0].size} elems, rows {np.unique(d[0])[:12]}, "
              f"cols {np.unique(d[-1])[:12]} maxrel {rel:.3e}")
    else:
        d = np.nonzero(x != y)
        print(f"{k} {x.shape}: {d[0].size} elems at {[tuple(int(t[i]) for t in d) for i in range(min(6, d[0].size))]}"
              f" prod {x[d][:6]} other {y[d][:6]}")
