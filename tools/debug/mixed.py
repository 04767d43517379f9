import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import oracle
from paper_2101_05063_b200 import solver
n, b_r = 96, 32
rng = np.random.default_rng(0)
h = np.triu(rng.standard_normal((n, n)))
h[np.arange(1, n), np.arange(n - 1)] = np.abs(rng.standard_normal(n - 1)) + 0.1
ev = np.linalg.eigvals(h)
er = ev[ev.imag == 0][:6].real
ec = ev[ev.imag > 0][:6]
rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
start = rho * np.ones(n)
o_r = oracle.solve(h, er, np.repeat(start[:, None], er.size, 1), b_r, mode="eigvec")
o_c = oracle.solve(h, ec, np.repeat(start[:, None], ec.size, 1).astype(complex), b_r, mode="eigvec")
def run(ecs, ers, bvec):
    out, gs = solver.solve_group(h, ecs, ers, bvec, b_r)
    X = out.X.cpu().numpy(); mc = len(ecs) if ecs is not None else 0
    xc = (X[0:2*mc:2] + 1j*X[1:2*mc:2]).T
    xr = X[2*mc:].T
    return xc, xr, out
for label, ecs, ers in (("real only", None, er), ("cplx only", ec, None), ("mixed", ec, er)):
    for bl, b in (("bcast", start), ("full", None)):
        if b is None:
            mc = len(ecs) if ecs is not None else 0; mr = len(ers) if ers is not None else 0
            b = np.repeat(start[None, :], 2*mc+mr, 0).copy()
            b[1:2*mc:2] = 0
            b = b.T
        xc, xr, out = run(ecs, ers, b)
        e1 = np.max(np.abs(xr - o_r.x)) if ers is not None else 0
        e2 = np.max(np.abs(xc - o_c.x)) if ecs is not None else 0
        print(label, bl, "real err %.2e cplx err %.2e" % (e1, e2), "nfail", out.nfail)
hf = np.linalg.norm(h, 'fro')
xc, xr, out = run(ec, er, start)
for l in range(len(ec)):
    xg = xc[:, l]; xo = o_c.x[:, l]
    rg = np.linalg.norm(h @ xg - ec[l]*xg)/(hf*np.linalg.norm(xg)); ro = np.linalg.norm(h @ xo - ec[l]*xo)/(hf*np.linalg.norm(xo))
    ip = np.vdot(xg, xo); xa = xg * ip/abs(ip)
    print("cplx", l, "res gpu %.2e oracle %.2e |diff| %.2e aligned %.2e normgpu %.3e normor %.3e" % (rg, ro, np.max(np.abs(xg-xo)), np.linalg.norm(xa-xo), out.norms.cpu().numpy()[l], o_c.norms[l]))
oracle.use_reference_blas(True)
o_c2 = oracle.solve(h, ec, np.repeat(start[:, None], ec.size, 1).astype(complex), b_r, mode="eigvec")
print("oracle naive vs blas", np.max(np.abs(o_c2.x - o_c.x)))
