"""Oracle restatement of the reference 1D bases (test infrastructure only).

Follows ``sdmefem/quadrature.py:31-58`` (rules), ``sdmefem/basis1d.py:128-198``
(Jacobi / modal / Lagrange evaluation), ``basis1d.py:234-351`` (SDME
construction) and ``sdmefem/densela.py:43-140`` (cyclic Jacobi eigen-solver and
Cholesky solve).  Written loop-first for clarity, not speed.
"""

from __future__ import annotations

import numpy as np

TAGS = ("LagrangeGLL", "ModalJacobi", "SDME_M", "SDME_K", "SDME_H")


def gauss(n):
    """quadrature.py:31-37."""
    return np.polynomial.legendre.leggauss(n)


def gll(n):
    """quadrature.py:40-58 (roots of P'_{n-1} via Jacobi(1,1))."""
    from scipy.special import roots_jacobi

    if n == 2:
        x = np.array([-1.0, 1.0])
    else:
        r, _ = roots_jacobi(n - 2, 1.0, 1.0)
        x = np.r_[-1.0, np.sort(r), 1.0]
    pl = np.polynomial.legendre.legval(x, [0.0] * (n - 1) + [1.0])
    return x, 2.0 / (n * (n - 1) * pl ** 2)


def jacobi(n, a, b, x):
    """basis1d.py:128-146: three-term recurrence."""
    x = np.asarray(x, dtype=float)
    p_prev, p = np.ones_like(x), None
    if n == 0:
        return p_prev
    p = 0.5 * (a + b + 2.0) * x + 0.5 * (a - b)
    for m in range(1, n):
        s = 2 * m + a + b
        num = ((s + 1) * (a * a - b * b) + s * (s + 1) * (s + 2) * x) * p \
            - 2.0 * (m + a) * (m + b) * (s + 2) * p_prev
        p_prev, p = p, num / (2.0 * (m + 1) * (m + a + b + 1) * s)
    return p


def modal(P, a, b, x):
    """basis1d.py:157-170: vertex ramps + (1-x)(1+x)/4 * P^{a,b}_{p-2}."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    v = np.zeros((P + 1, x.size))
    d = np.zeros((P + 1, x.size))
    v[0], d[0] = 0.5 * (1 - x), -0.5
    v[1], d[1] = 0.5 * (1 + x), 0.5
    bub = 0.25 * (1 - x) * (1 + x)
    for p in range(2, P + 1):
        j = jacobi(p - 2, a, b, x)
        dj = 0.0 if p == 2 else 0.5 * (p - 2 + a + b + 1) * jacobi(p - 3, a + 1, b + 1, x)
        v[p] = bub * j
        d[p] = -0.5 * x * j + bub * dj
    return v, d


def lagrange(nodes, x):
    """basis1d.py:173-198: product-formula cardinal functions, node order."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    n = len(nodes)
    v = np.ones((n, x.size))
    d = np.zeros((n, x.size))
    for a in range(n):
        for b in range(n):
            if b != a:
                v[a] *= (x - nodes[b]) / (nodes[a] - nodes[b])
        for c in range(n):
            if c == a:
                continue
            t = np.ones_like(x) / (nodes[a] - nodes[c])
            for b in range(n):
                if b not in (a, c):
                    t *= (x - nodes[b]) / (nodes[a] - nodes[b])
            d[a] += t
    return v, d


def _reorder(rows):
    n = rows.shape[0]
    return rows[[0, n - 1] + list(range(1, n - 1))]


def sym_eig(a):
    """densela.py:43-105: cyclic Jacobi, eigenvalues ascending."""
    a = 0.5 * (np.array(a, dtype=float) + np.array(a, dtype=float).T)
    n = a.shape[0]
    if n == 1:
        return a[0].copy(), np.ones((1, 1))
    v = np.eye(n)
    thr = 1e-14 * np.linalg.norm(a)
    for _ in range(100):
        if np.linalg.norm(a - np.diag(np.diag(a))) <= thr:
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                if abs(a[p, q]) <= thr / n:
                    continue
                tau = (a[q, q] - a[p, p]) / (2.0 * a[p, q])
                t = (1.0 / (tau + np.hypot(1.0, tau)) if tau >= 0
                     else -1.0 / (-tau + np.hypot(1.0, tau)))
                c = 1.0 / np.hypot(1.0, t)
                s = t * c
                apq = a[p, q]
                app, aqq = a[p, p] - t * apq, a[q, q] + t * apq
                for r in range(n):
                    if r in (p, q):
                        continue
                    arp, arq = a[r, p], a[r, q]
                    a[r, p] = a[p, r] = c * arp - s * arq
                    a[r, q] = a[q, r] = s * arp + c * arq
                a[p, p], a[q, q] = app, aqq
                a[p, q] = a[q, p] = 0.0
                vp = v[:, p].copy()
                v[:, p] = c * vp - s * v[:, q]
                v[:, q] = s * vp + c * v[:, q]
    w = np.diag(a).copy()
    o = np.argsort(w, kind="stable")
    return w[o], v[:, o]


def chol_solve(a, b):
    """densela.py:108-140."""
    n = a.shape[0]
    l = np.zeros_like(a)
    for j in range(n):
        l[j, j] = np.sqrt(a[j, j] - l[j, :j] @ l[j, :j])
        for i in range(j + 1, n):
            l[i, j] = (a[i, j] - l[i, :j] @ l[j, :j]) / l[j, j]
    y = np.array(b, dtype=float).reshape(n, -1)
    for j in range(n):
        y[j] /= l[j, j]
        y[j + 1:] -= np.outer(l[j + 1:, j], y[j])
    for j in range(n - 1, -1, -1):
        y[j] /= l[j, j]
        y[:j] -= np.outer(l[j, :j], y[j])
    return y


def _sd(m, k, kexp):
    """basis1d.py:234-253."""
    lm, x = sym_eig(m)
    xs = x / np.sqrt(lm)
    l = xs.T @ k @ xs
    ls, z = sym_eig(0.5 * (l + l.T))
    return (xs @ z @ np.diag(ls ** (-0.5 * kexp))).T, ls


def _sd_parity(m, k, kexp, with_parity=False):
    """basis1d.py:263-287 (symmetric weights: even/odd blocks; internal slot i
    holds mode p = i + 2 of parity (-1)^i, so a block's rows share its parity)."""
    n = m.shape[0]
    if n <= 1:
        y = _sd(m, k, kexp)[0]
        return (y, np.ones(n)) if with_parity else y
    rows = []
    for par in (0, 1):
        idx = list(range(par, n, 2))
        yb, lb = _sd(m[np.ix_(idx, idx)], k[np.ix_(idx, idx)], kexp)
        for j in range(len(idx)):
            r = np.zeros(n)
            r[idx] = yb[j]
            rows.append((lb[j], r, (-1.0) ** par))
    rows.sort(key=lambda t: t[0])
    y = np.array([r for _, r, _ in rows])
    return (y, np.array([s for _, _, s in rows])) if with_parity else y


class Basis:
    """Order-P basis, function order [left, right, internal] (basis1d.py:79-125)."""

    def __init__(self, tag, P, alpha=1.0, beta=1.0, k=0.5, lam=100.0):
        assert tag in TAGS
        self.tag, self.P, self.alpha, self.beta = tag, P, alpha, beta
        self.nodes = None
        # reflection parity of the internal functions (basis1d.py:85-89, 326-328):
        # None for the nodal basis (orientation by index reversal) and for
        # non-symmetric Jacobi weights
        self.internal_parity = (np.array([(-1.0) ** p for p in range(2, P + 1)])
                                if tag != "LagrangeGLL" and alpha == beta and P >= 2 else None)
        t = np.eye(P + 1)
        if tag == "LagrangeGLL":  # basis1d.py:317-323
            self.nodes = gll(P + 1)[0]
        elif tag.startswith("SDME"):  # basis1d.py:331-348
            xq, wq = gauss(P + 2)
            v, d = modal(P, alpha, beta, xq)
            mm = (v * wq) @ v.T
            kk = (d * wq) @ d.T
            if alpha == beta:
                y, self.internal_parity = _sd_parity(mm[2:, 2:], kk[2:, 2:], k, with_parity=True)
            else:
                y = _sd(mm[2:, 2:], kk[2:, 2:], k)[0]
            g = {"SDME_M": mm, "SDME_K": kk, "SDME_H": kk + lam * mm}[tag]
            avi = g[:2, 2:] @ y.T
            aii = y @ g[2:, 2:] @ y.T
            me = chol_solve(aii, avi.T).T
            t[2:, 2:] = y
            t[:2, 2:] = -me @ y
        self.T = t

    def eval(self, x):
        if self.nodes is not None:
            v, d = lagrange(self.nodes, x)
            return _reorder(v), _reorder(d)
        v, d = modal(self.P, self.alpha, self.beta, x)
        return self.T @ v, self.T @ d
