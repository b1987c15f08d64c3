"""Plain fp64 L-BFGS of the paper's optimizer setting (liblbfgs, 5 Hessian
corrections, "backtracking line search with a Wolfe condition", stop when the metric
is stable within the last 20 steps or at the maximal iteration count), spelled out as
DESIGN.md reading c20 states it.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py):
the reference the F1 driver ``srwcr_register`` is compared with, iterate by iterate.

Textbook L-BFGS (Nocedal & Wright, Alg. 7.4 / 7.5), no blocking or reordering:
  d_0 = -g_0, first trial step 1/||g_0||, then step 1 with H_0 = (y.s / y.y) I of the
  newest stored pair; backtracking: trial x + step d, step *= 0.5 when the Armijo test
  f(x + step d) <= f(x) + ftol step g.d fails (or the cost is not finite / undefined),
  step *= 2.1 when the regular Wolfe curvature test g(x + step d).d >= wolfe g.d fails,
  at most max_linesearch trials; a pair (s, y) with y.s <= 0 is not stored; a
  direction with g.d >= 0 restarts from steepest descent (memory cleared, step 1/||g||).
Stops: ||g|| <= epsilon max(1, ||x||) (off by default), max - min of the cost over the
last stable_window accepted iterates (the start included) < stable_tol max(|f|, 1e-12),
max_iter iterations, or a failed line search.
"""
from __future__ import annotations

import numpy as np

STATUS = {0: "converged", 1: "stable", 2: "max_iter", 3: "line_search_failed"}


class Infeasible(Exception):
    """Raised by a cost function at a point where the cost is undefined (a trial the
    line search shortens, like a non-finite value)."""


def lbfgs(fun, x0, m=5, max_iter=200, max_linesearch=20, ftol=1e-4, wolfe=0.9, stable_window=20,
          stable_tol=1e-5, epsilon=0.0):
    """Minimise ``fun(x) -> (f, g)``.  Returns (x, report, iterates) with iterates the list
    of accepted (x_k, f_k, step_k, cost evaluations so far) for k = 1.. (x_0 excluded)."""
    shape = np.shape(x0)
    fun0 = fun

    def fun(v):   # flat fp64 vectors inside; the caller's shape outside
        f, g = fun0(v.reshape(shape))
        return f, np.asarray(g, dtype=np.float64).ravel()
    x = np.array(x0, dtype=np.float64, copy=True).ravel()
    f, g = fun(x)
    f0 = f
    evals = 1
    S, Y, rho = [], [], []          # newest last
    hscale = 1.0
    hist = [f]
    its = []
    d = -g
    step = 1.0 / np.sqrt(max(g @ g, 1e-300))
    status, it = 2, 0
    if np.sqrt(g @ g) <= epsilon * max(1.0, np.sqrt(x @ x)):
        status = 0
    while status == 2 and it < max_iter:
        it += 1
        gd = g @ d
        if not gd < 0:
            d = -g
            S, Y, rho = [], [], []
            gd = -(g @ g)
            step = 1.0 / np.sqrt(max(g @ g, 1e-300))
        ok = False
        for _ in range(max_linesearch):
            xp = x + step * d
            try:
                fp, gp = fun(xp)
                evals += 1
            except Infeasible:
                evals += 1
                step *= 0.5
                continue
            if not np.isfinite(fp) or fp > f + ftol * step * gd:
                step *= 0.5
                continue
            if gp @ d < wolfe * gd:
                step *= 2.1
                continue
            ok = True
            break
        if not ok:
            status = 3
            break
        s, y = xp - x, gp - g
        x, g, f = xp, gp, fp
        hist.append(f)
        its.append((x.reshape(shape).copy(), f, step, evals))
        if np.sqrt(g @ g) <= epsilon * max(1.0, np.sqrt(x @ x)):
            status = 0
            break
        if len(hist) >= stable_window:
            w = hist[-stable_window:]
            if max(w) - min(w) < stable_tol * max(abs(f), 1e-12):
                status = 1
                break
        ys = y @ s
        if ys > 0:
            S.append(s)
            Y.append(y)
            rho.append(1.0 / ys)
            hscale = ys / (y @ y)
            if len(S) > m:
                S.pop(0), Y.pop(0), rho.pop(0)
        # two-loop recursion: d = -H g
        q = -g
        alpha = [0.0] * len(S)
        for i in range(len(S) - 1, -1, -1):
            alpha[i] = rho[i] * (S[i] @ q)
            q = q - alpha[i] * Y[i]
        if S:
            q = hscale * q
        for i in range(len(S)):
            b = rho[i] * (Y[i] @ q)
            q = q + (alpha[i] - b) * S[i]
        d = q
        step = 1.0
    rep = {"iterations": it, "evaluations": evals, "status": status, "status_name": STATUS[status],
           "initial_cost": f0, "final_cost": f, "grad_norm": float(np.sqrt(g @ g))}
    return x.reshape(shape), rep, its
