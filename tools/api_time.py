"""Wall time of the drop-in API at config 5: hsrq3in(H, eigenvalues) with a
numpy H and numpy eigenvalues in, numpy eigenvectors out (inviter.py:186-254)
-- everything a caller of the reference's entry point pays, one attempt
(max_restarts=0, every config-5 shift converges on the first attempt)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    import torch

    import instances
    from paper_2101_05063_b200 import InviterConfig, hsrq3in

    h = instances.make_h(5)
    sel = instances.shifts(5)
    rng = np.random.default_rng(0)
    sel = sel[rng.permutation(sel.size)]  # caller order: mixed kinds
    cfg = InviterConfig(b_r=128, max_restarts=0)
    for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = hsrq3in(h, sel, cfg)
        t1 = time.perf_counter()
        print(f"hsrq3in call {i}: {1e3 * (t1 - t0):.1f} ms, converged {int(r.converged.sum())}/{sel.size}",
              {k: round(v, 1) for k, v in r.extras.get("host_ms", {}).items()}, flush=True)
        del r


if __name__ == "__main__":
    main()
