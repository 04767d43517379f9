import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import numpy as np, torch
import instances
from oracle import oracle
from paper_2101_05063_b200 import solver
n = 1000
h = instances.random_hessenberg(n, 0)
ev = np.linalg.eigvals(h)
er = ev[ev.imag == 0].real[:4]; ec = ev[ev.imag > 0][:4]
rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
start = rho * np.ones(n)
for b_r in (128, 112, 100, 64):
    out, gs = solver.solve_group(h, ec, er, start, b_r)
    seg = out.seg_exp.cpu().numpy()
    X = out.X.cpu().numpy()
    o = oracle.solve(h, er, np.repeat(start[:, None], er.size, 1), b_r, mode="eigvec")
    print(b_r, "seg min", seg.min(), "oracle seg min", o.segment_exp.min(), "finite", np.isfinite(X).all(),
          "real vec err", np.max(np.abs(np.abs(X[2*ec.size:].T) - np.abs(o.x))))
