"""Host-side 1D expansion bases: the only part of the path that stays on the CPU.

The GPU kernels never see a basis *kind*; they only see three small tables per
(basis, P, m): the values ``B[a, t]`` and derivatives ``D[a, t]`` of the P+1
1D functions at the m quadrature points, and the weights ``w[a]``.  This module
builds those tables with the same construction as the reference
(``sdmefem/basis1d.py:301-351`` ``build_basis``) so that coefficient vectors
mean the same thing on both sides of the drop-in boundary:

* nodal Lagrange on the P+1 Gauss-Lobatto-Legendre points
  (``basis1d.py:317-323``),
* the standard Jacobi modal basis -- vertex ramps plus weighted bubbles
  (``basis1d.py:157-170``),
* SDME_M / SDME_K / SDME_H: simultaneous diagonalisation of the internal
  mass/stiffness blocks per reflection parity (``basis1d.py:234-287``) followed
  by the minimum-energy re-orthogonalisation of the two vertex functions
  (``basis1d.py:256-260, 331-348``).

Function order is the reference's: [left vertex, right vertex, internal 2..P]
(``basis1d.py:83``).  The eigen-solver is the same cyclic Jacobi sweep as
``densela.py:43-105`` so eigenvector signs -- and therefore the sign of every
SDME internal mode -- agree with the reference.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

__all__ = [
    "BasisKind",
    "Rule",
    "gauss_rule",
    "gll_rule",
    "Basis1D",
    "build_basis",
    "jacobi_poly",
    "modal_tables",
    "lagrange_tables",
    "constant_coeffs",
]

ALL_TAGS = ("LagrangeGLL", "ModalJacobi", "SDME_M", "SDME_K", "SDME_H")


# --------------------------------------------------------------------------- rules

@dataclass(frozen=True)
class Rule:
    """1D quadrature rule on [-1, 1] (``quadrature.py:21-35``)."""

    kind: str
    points: np.ndarray
    weights: np.ndarray

    @property
    def n(self) -> int:
        return int(self.points.size)


@lru_cache(maxsize=None)
def gauss_rule(n: int) -> Rule:
    """n-point Gauss-Legendre (``quadrature.py:31-37``)."""
    if n < 1:
        raise ValueError(f"Gauss-Legendre rule needs n >= 1, got {n}")
    x, w = np.polynomial.legendre.leggauss(n)
    return Rule("GaussLegendre", x, w)


@lru_cache(maxsize=None)
def gll_rule(n: int) -> Rule:
    """n-point Gauss-Lobatto-Legendre (``quadrature.py:40-58``).

    Interior nodes are the roots of P'_{n-1} (Jacobi(1,1) of degree n-2);
    weights 2 / (n (n-1) P_{n-1}(x)^2).
    """
    if n < 2:
        raise ValueError(f"Gauss-Lobatto-Legendre rule needs n >= 2, got {n}")
    if n == 2:
        x = np.array([-1.0, 1.0])
    else:
        from scipy.special import roots_jacobi

        inner, _ = roots_jacobi(n - 2, 1.0, 1.0)
        x = np.concatenate(([-1.0], np.sort(inner), [1.0]))
    leg = np.polynomial.legendre.legval(x, np.eye(n)[n - 1])
    return Rule("GaussLobattoLegendre", x, 2.0 / (n * (n - 1) * leg * leg))


# ---------------------------------------------------------------- 1D polynomials

def jacobi_poly(deg: int, a: float, b: float, x) -> np.ndarray:
    """P_deg^{(a,b)}(x) by the three-term recurrence (``basis1d.py:128-146``)."""
    x = np.asarray(x, dtype=float)
    prev = np.ones_like(x)
    if deg == 0:
        return prev
    cur = 0.5 * (a + b + 2.0) * x + 0.5 * (a - b)
    for k in range(1, deg):
        s = 2 * k + a + b
        c1 = 2.0 * (k + 1) * (k + a + b + 1) * s
        c2 = (s + 1) * (a * a - b * b)
        c3 = s * (s + 1) * (s + 2)
        c4 = 2.0 * (k + a) * (k + b) * (s + 2)
        prev, cur = cur, ((c2 + c3 * x) * cur - c4 * prev) / c1
    return cur


def _jacobi_dpoly(deg: int, a: float, b: float, x) -> np.ndarray:
    if deg == 0:
        return np.zeros_like(np.asarray(x, dtype=float))
    return 0.5 * (deg + a + b + 1) * jacobi_poly(deg - 1, a + 1, b + 1, x)


def modal_tables(P: int, a: float, b: float, x) -> tuple[np.ndarray, np.ndarray]:
    """Standard modal functions and derivatives, rows = functions
    (``basis1d.py:157-170``)."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    val = np.empty((P + 1, x.size))
    der = np.empty((P + 1, x.size))
    val[0] = 0.5 * (1.0 - x)
    der[0] = -0.5
    if P >= 1:
        val[1] = 0.5 * (1.0 + x)
        der[1] = 0.5
    bub = 0.25 * (1.0 - x) * (1.0 + x)
    for t in range(2, P + 1):
        j = jacobi_poly(t - 2, a, b, x)
        val[t] = bub * j
        der[t] = -0.5 * x * j + bub * _jacobi_dpoly(t - 2, a, b, x)
    return val, der


def lagrange_tables(nodes, x) -> tuple[np.ndarray, np.ndarray]:
    """Lagrange cardinal functions on ``nodes`` and their derivatives, node
    order (``basis1d.py:173-198``; direct product formulas)."""
    nodes = np.asarray(nodes, dtype=float)
    if np.unique(nodes).size != nodes.size:
        raise ValueError("Lagrange nodes must be distinct")
    x = np.atleast_1d(np.asarray(x, dtype=float))
    k = nodes.size
    val = np.ones((k, x.size))
    der = np.zeros((k, x.size))
    for i in range(k):
        others = [j for j in range(k) if j != i]
        for j in others:
            val[i] *= (x - nodes[j]) / (nodes[i] - nodes[j])
        for c in others:
            term = np.full(x.shape, 1.0 / (nodes[i] - nodes[c]))
            for j in others:
                if j != c:
                    term = term * ((x - nodes[j]) / (nodes[i] - nodes[j]))
            der[i] += term
    return val, der


def _nodal_to_function_order(rows: np.ndarray) -> np.ndarray:
    k = rows.shape[0]
    return rows[[0, k - 1] + list(range(1, k - 1))]


# ------------------------------------------------------------ small dense algebra

def _cyclic_jacobi_eig(a: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Symmetric eigen-decomposition by cyclic Jacobi rotations.

    Same sweep order, threshold (1e-14 ||A||_F, skip |a_pq| <= thr/n) and
    rotation root as ``densela.py:43-105`` so the eigenvector signs match.
    Returns eigenvalues ascending (stable sort) and eigenvectors as columns.
    """
    a = np.asarray(a, dtype=float)
    a = 0.5 * (a + a.T)
    n = a.shape[0]
    if n == 1:
        return a[0].copy(), np.ones((1, 1))
    vec = np.eye(n)
    fro = np.linalg.norm(a)
    if fro == 0.0:
        return np.zeros(n), vec
    thr = 1e-14 * fro
    for _sweep in range(100):
        if np.linalg.norm(a - np.diag(np.diag(a))) <= thr:
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = a[p, q]
                if abs(apq) <= thr / n:
                    continue
                theta = (a[q, q] - a[p, p]) / (2.0 * apq)
                if theta >= 0.0:
                    t = 1.0 / (theta + np.hypot(1.0, theta))
                else:
                    t = -1.0 / (-theta + np.hypot(1.0, theta))
                c = 1.0 / np.hypot(1.0, t)
                s = t * c
                d_p = a[p, p] - t * apq
                d_q = a[q, q] + t * apq
                rest = [r for r in range(n) if r != p and r != q]
                col_p = a[rest, p].copy()
                col_q = a[rest, q].copy()
                a[rest, p] = c * col_p - s * col_q
                a[rest, q] = s * col_p + c * col_q
                a[p, rest] = a[rest, p]
                a[q, rest] = a[rest, q]
                a[p, p], a[q, q] = d_p, d_q
                a[p, q] = a[q, p] = 0.0
                vp = vec[:, p].copy()
                vec[:, p] = c * vp - s * vec[:, q]
                vec[:, q] = s * vp + c * vec[:, q]
    else:
        raise RuntimeError("cyclic Jacobi did not converge")
    lam = np.diag(a).copy()
    order = np.argsort(lam, kind="stable")
    return lam[order], vec[:, order]


def _chol_solve(a: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """SPD solve by an explicit lower Cholesky factor (``densela.py:108-140``)."""
    a = 0.5 * (a + a.T)
    n = a.shape[0]
    low = np.zeros_like(a)
    floor = 1e-14 * max(np.abs(np.diag(a)).max(), 1.0)
    for j in range(n):
        piv = a[j, j] - low[j, :j] @ low[j, :j]
        if piv <= floor:
            raise ValueError("matrix is not SPD")
        low[j, j] = np.sqrt(piv)
        low[j + 1:, j] = (a[j + 1:, j] - low[j + 1:, :j] @ low[j, :j]) / low[j, j]
    y = np.array(rhs, dtype=float).reshape(n, -1)
    for j in range(n):
        y[j] /= low[j, j]
        y[j + 1:] -= np.outer(low[j + 1:, j], y[j])
    for j in range(n - 1, -1, -1):
        y[j] /= low[j, j]
        y[:j] -= np.outer(low[j, :j], y[j])
    return y


def _sd_block(m_ii: np.ndarray, k_ii: np.ndarray, kexp: float):
    """Whiten M, diagonalise whitened K, rescale by L^(-k/2)
    (``basis1d.py:234-253``).  Returns (Y rows = new modes, L ascending)."""
    lm, xm = _cyclic_jacobi_eig(m_ii)
    if lm[0] <= 0.0:
        raise ValueError("internal mass block is not SPD")
    xs = xm / np.sqrt(lm)
    kw = xs.T @ k_ii @ xs
    ls, zs = _cyclic_jacobi_eig(0.5 * (kw + kw.T))
    if ls[0] <= 0.0:
        raise ValueError("internal stiffness block is not SPD")
    return (xs @ zs @ np.diag(ls ** (-0.5 * kexp))).T, ls


def _sd_by_parity(m_ii, k_ii, kexp, split):
    """SD per reflection-parity block, modes re-sorted by eigenvalue
    (``basis1d.py:263-287``)."""
    n = m_ii.shape[0]
    if not split or n <= 1:
        y, lam = _sd_block(m_ii, k_ii, kexp)
        return y, lam, None
    recs = []
    for par in (0, 1):
        idx = np.arange(par, n, 2)
        yb, lb = _sd_block(m_ii[np.ix_(idx, idx)], k_ii[np.ix_(idx, idx)], kexp)
        for j in range(idx.size):
            row = np.zeros(n)
            row[idx] = yb[j]
            recs.append((lb[j], 1.0 - 2.0 * par, row))
    recs.sort(key=lambda r: r[0])
    return (np.array([r[2] for r in recs]), np.array([r[0] for r in recs]),
            np.array([r[1] for r in recs]))


# ------------------------------------------------------------------------ basis

@dataclass(frozen=True)
class BasisKind:
    """Basis family tag and shape parameters (``basis1d.py:46-76``)."""

    tag: str
    jacobi_alpha: float = 1.0
    jacobi_beta: float = 1.0
    k: float = 0.5
    lam: float = 100.0

    def __post_init__(self):
        if self.tag not in ALL_TAGS:
            raise ValueError(f"unknown basis tag {self.tag!r}; expected one of {ALL_TAGS}")
        if not 0.0 <= self.k <= 1.0:
            raise ValueError(f"k must lie in [0, 1], got {self.k}")
        if self.lam < 0.0:
            raise ValueError(f"lambda must be >= 0, got {self.lam}")

    @property
    def is_nodal(self) -> bool:
        return self.tag == "LagrangeGLL"


@dataclass(frozen=True)
class Basis1D:
    """Order-P 1D basis: ``transform`` expresses each function in the standard
    modal basis (rows), function order [left, right, internal]."""

    P: int
    kind: BasisKind
    transform: np.ndarray
    gll_nodes: np.ndarray | None = None

    @property
    def n(self) -> int:
        return self.P + 1

    def eval(self, x) -> tuple[np.ndarray, np.ndarray]:
        """Values/derivatives (P+1, len(x)) at arbitrary points
        (``basis1d.py:113-120``)."""
        if self.kind.is_nodal:
            v, d = lagrange_tables(self.gll_nodes, x)
            return _nodal_to_function_order(v), _nodal_to_function_order(d)
        v, d = modal_tables(self.P, self.kind.jacobi_alpha, self.kind.jacobi_beta, x)
        return self.transform @ v, self.transform @ d

    def tables(self, rule: Rule) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """Kernel inputs at ``rule``: B (m, n), D (m, n), w (m)."""
        v, d = self.eval(rule.points)
        return np.ascontiguousarray(v.T), np.ascontiguousarray(d.T), rule.weights.copy()


def build_basis(P: int, kind: BasisKind) -> Basis1D:
    """Any of the five kinds at order P (``basis1d.py:301-351``)."""
    if P < 1:
        raise ValueError("polynomial order must be >= 1")
    sdme = kind.tag.startswith("SDME")
    if sdme and P < 2:
        raise ValueError(f"{kind.tag} needs P >= 2 (no internal modes at P={P})")
    a, b = kind.jacobi_alpha, kind.jacobi_beta
    if kind.is_nodal:
        nodes = gll_rule(P + 1).points
        psi, _ = modal_tables(P, a, b, nodes)
        t = _nodal_to_function_order(np.eye(P + 1)) @ np.linalg.inv(psi.T)
        return Basis1D(P, kind, t, nodes)
    t = np.eye(P + 1)
    if sdme:
        q = gauss_rule(P + 2)
        v, d = modal_tables(P, a, b, q.points)
        mass = (v * q.weights) @ v.T
        stiff = (d * q.weights) @ d.T
        y, _, _ = _sd_by_parity(mass[2:, 2:], stiff[2:, 2:], kind.k, a == b)
        if kind.tag == "SDME_M":
            gram = mass
        elif kind.tag == "SDME_K":
            gram = stiff
        else:
            gram = stiff + kind.lam * mass
        a_vi = gram[:2, 2:] @ y.T
        a_ii = y @ gram[2:, 2:] @ y.T
        coeff = _chol_solve(a_ii, a_vi.T).T
        t[2:, 2:] = y
        t[:2, 2:] = -coeff @ y
    return Basis1D(P, kind, t)


def constant_coeffs(basis: Basis1D) -> np.ndarray:
    """1D coefficients c with sum_t c_t phi_t == 1 (SURVEY §8a notes).

    phi = T psi with psi the standard modal functions; 1 = psi_0 + psi_1, so
    c^T T = (1, 1, 0, ...), i.e. c = T^-T e.
    """
    e = np.zeros(basis.n)
    e[:2] = 1.0
    if basis.kind.is_nodal:
        return np.ones(basis.n)
    return np.linalg.solve(basis.transform.T, e)
