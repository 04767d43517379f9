"""Flop accounting for the measurement (the TFLOP/s numerator).

``reference_flops`` sums the reference's exact per-task counts (hessrq
flops.py:15-70) over the tasks one solve performs (one ReduceDiag and one
Solve per tile column, ReduceOffdiag and Update per above-diagonal tile, one
Backtransform), which is what the reference's RunStats accumulates.
``executed_flops`` counts what the B200 kernels actually issue, dominated by
the fused panel GEMM (2 * rows * k per output entry, two outputs -- W and Z --
per real column), so a reformulation never inflates TFLOP/s silently.
"""

from __future__ import annotations


def _reduce_diag(k, cplx):
    per = 0
    for kp in range(k - 1, 0, -1):
        per += (6 * (kp - 1) + 12 + 7) if cplx else (3 * (kp - 1) + 4 + 5)
    return per + 5


def _reduce_offdiag(k, w, cplx):
    return (w - 1) * 6 * k + 6 * k + 10 if cplx else (w - 1) * 3 * k + 3 * k + 2


def _solve(k, cplx):
    if not cplx:
        per = 0
        for kp in range(k - 1, 0, -1):
            per += 3 + 1 + 2 + 4 * (kp - 1) + 5 + 3 * (kp - 1) + 4
        return per + 4
    per = 0
    for kp in range(k - 1, 0, -1):
        per += 10 * (kp + 1) + 10 * kp + 2
    per += 8
    for j in range(k - 1, -1, -1):
        per += 9 + 8 * j
    return per


def _update(m, k, cplx):
    if not cplx:
        return (2 * m + 2) + (1 + 6 * (k - 1)) + 2 * m * (k - 1) + 2 * m
    return (4 * m + 6) + (6 + 20 * (k - 1)) + 4 * m * (k - 1) + 8 * m


def _backtransform(n, cplx):
    return (20 if cplx else 6) * (n - 1)


def per_shift_flops(n, b_r, cplx):
    """Reference flop-model count for one shift (exact task sums)."""
    ranges = [(s, min(s + b_r, n)) for s in range(0, n, b_r)]
    N = len(ranges)
    tot = 0
    for jt in range(N):
        k = ranges[jt][1] - ranges[jt][0]
        tot += _reduce_diag(k, cplx) + _solve(k, cplx)
        for i in range(jt):
            ki = ranges[i][1] - ranges[i][0]
            tot += _reduce_offdiag(ki, k, cplx) + _update(ki, k, cplx)
    return tot + _backtransform(n, cplx)


def reference_flops(n, b_r, m_real, m_cplx):
    """Total reference-model flops for m_real real and m_cplx complex shifts."""
    return m_real * per_shift_flops(n, b_r, False) + m_cplx * per_shift_flops(n, b_r, True)


def paper_flops(n, m_real, m_cplx):
    """The paper's 3.5 n^2 per real column convention."""
    return 3.5 * n * n * (m_real + 2 * m_cplx)


def panel_gemm_flops(n, b_r, ncol, jt):
    """DMMA flops one k_panel launch executes at tile column jt (ncol real columns)."""
    js = jt * b_r
    k = min(js + b_r, n) - js
    return 2.0 * js * k * 2 * ncol


def executed_flops(n, b_r, m_real, m_cplx):
    """Flops the B200 path issues: the panel GEMMs (dominant) over all tile columns."""
    ncol = m_real + 2 * m_cplx
    N = (n + b_r - 1) // b_r
    return sum(panel_gemm_flops(n, b_r, ncol, jt) for jt in range(1, N))


TASK_TYPES = ("ReduceDiag", "ReduceOffdiag", "Solve", "Update", "Backtransform")


def _formula(task, dims, cplx):
    """Leading-order per-shift counts (hessrq flops.py:79-96)."""
    if task == "ReduceDiag":
        return (3.0 if cplx else 1.5) * dims[0] ** 2
    if task == "ReduceOffdiag":
        return (6.0 if cplx else 3.0) * dims[0] * dims[1]
    if task == "Solve":
        return (15.0 if cplx else 3.5) * dims[0] ** 2
    if task == "Update":
        return (4.0 if cplx else 2.0) * dims[0] * dims[1]
    return (20.0 if cplx else 6.0) * (dims[0] - 1)


def task_flops(n, b_r, m, cplx):
    """Per task type: (exact counts, Table-1 formula counts) for m shifts --
    what the reference's RunStats accumulates over one solve (reduce.py:132,
    166; backsolve.py:168, 229, 299)."""
    ranges = [(s, min(s + b_r, n)) for s in range(0, n, b_r)]
    ex = dict.fromkeys(TASK_TYPES, 0)
    fo = dict.fromkeys(TASK_TYPES, 0.0)
    for jt, (js, je) in enumerate(ranges):
        k = je - js
        ex["ReduceDiag"] += _reduce_diag(k, cplx)
        ex["Solve"] += _solve(k, cplx)
        fo["ReduceDiag"] += _formula("ReduceDiag", (k,), cplx)
        fo["Solve"] += _formula("Solve", (k,), cplx)
        for i in range(jt):
            ki = ranges[i][1] - ranges[i][0]
            ex["ReduceOffdiag"] += _reduce_offdiag(ki, k, cplx)
            ex["Update"] += _update(ki, k, cplx)
            fo["ReduceOffdiag"] += _formula("ReduceOffdiag", (ki, k), cplx)
            fo["Update"] += _formula("Update", (ki, k), cplx)
    ex["Backtransform"] += _backtransform(n, cplx)
    fo["Backtransform"] += _formula("Backtransform", (n,), cplx)
    return ({t: float(v) * m for t, v in ex.items()}, {t: float(v) * m for t, v in fo.items()})
