"""Oracle restatement of the reference solvers and time stepping (test
infrastructure only).

``pcg``: ``sdmefem/solver.py:102-170`` (diagonal / none preconditioners, same
order of checks: pAp <= 0 -> error, recursive-residual stop, maxit error with the
true residual).  ``newmark``: ``dynamics.py:173-257`` with
``SolverConfig(precond="diagonal", condense=False)``.
``explicit_lumped``: the D6 restatement -- ``explicit_run``'s central-difference
formulas (``dynamics.py:152-164``) with the row-sum lumped mass and penalty
contact forces (``contact.py:103-128``).
"""

from __future__ import annotations

import numpy as np


class PCGError(RuntimeError):
    def __init__(self, msg, iterations, residual):
        super().__init__(msg)
        self.iterations, self.residual = iterations, residual


def pcg(a, b, precond="diagonal", tol=1e-8, maxit=10000):
    """solver.py:129-170; returns (x, iterations, final relative residual)."""
    if not 0.0 < tol < 1.0:
        raise ValueError("tolerance must lie in (0, 1)")
    if precond == "diagonal":
        d = a.diagonal()
        if np.any(d <= 0):
            raise ValueError("diagonal preconditioner needs positive diagonal entries")
        inv = 1.0 / d
    else:
        inv = np.ones(a.shape[0])
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return np.zeros_like(b), 0, 0.0
    x = np.zeros_like(b)
    r = b.copy()
    z = inv * r
    p = z.copy()
    rz = r @ z
    for it in range(1, maxit + 1):
        ap = a @ p
        pap = p @ ap
        if pap <= 0:
            raise PCGError("indefinite", it, np.linalg.norm(r) / nb)
        al = rz / pap
        x += al * p
        r -= al * ap
        rel = np.linalg.norm(r) / nb
        if rel <= tol:
            return x, it, rel
        z = inv * r
        rzn = r @ z
        p = z + (rzn / rz) * p
        rz = rzn
    raise PCGError("maxit", maxit, np.linalg.norm(b - a @ x) / nb)


def newmark(problem, load, dt, n_steps, newton_tol=1e-8, newton_maxit=25, pcg_tol=1e-10,
            gamma=0.5, beta=0.25, u0=None, v0=None, maxit=200000, contact=None, track_energy=False):
    """dynamics.py:173-257, condense=False, Jacobi-PCG, optional penalty
    contact (residual + fc, Newton waits for settled pressures, operator
    + K_c of the iteration's active set, accept_step per step).

    Returns dict(u, v, a, newton_iters, pcg_iters) with pcg_iters a list of
    (step, newton_iter, iterations)."""
    b1 = 1.0 / (beta * dt * dt)
    b2 = 1.0 / (beta * dt)
    b3 = (1.0 - 2.0 * beta) / (2.0 * beta)
    n = problem.n_free
    u = np.zeros(n) if u0 is None else np.array(u0, float)
    v = np.zeros(n) if v0 is None else np.array(v0, float)
    mass = problem.mass()

    def residual(uk, atr, tt):
        psi = load(tt) - problem.internal_force(uk) - mass @ atr
        if contact is None:
            return psi, True, None
        fc, _ = contact.force(uk)
        ok = contact.settled(contact.pressures(uk))
        return psi + fc, ok, contact.stiffness(uk)

    psi0, _, _ = residual(u, np.zeros(n), 0.0)
    a, _, _ = pcg(mass, psi0, "diagonal", pcg_tol, maxit)
    t = 0.0
    newton_iters, pcg_iters, energy = [], [], []

    def energy_row(tt):  # dynamics.py:260-265
        pen = contact.penalty_energy(u) if contact is not None else 0.0
        energy.append((tt, 0.5 * float(v @ (mass @ v)), problem.total_strain_energy(u), pen))

    if track_energy:
        energy_row(t)
    for step in range(n_steps):
        tn = t + dt
        uk = u.copy()
        ref = None
        cnt = 0
        for k in range(newton_maxit):
            atr = b1 * (uk - u) - b2 * v - b3 * a
            psi, ok, kc = residual(uk, atr, tn)
            rn = np.linalg.norm(psi)
            if ref is None:
                ref = rn
            if ref == 0.0 or (rn <= newton_tol * ref and ok):
                break
            if k == newton_maxit - 1:
                raise RuntimeError("Newton did not converge")
            eff = problem.assemble(uk, 1.0, b1)
            if kc is not None:
                eff = (eff + kc).tocsr()
            du, its, _ = pcg(eff, psi, "diagonal", pcg_tol, maxit)
            pcg_iters.append((step, k, its))
            uk = uk + du
            cnt += 1
        newton_iters.append(cnt)
        an = b1 * (uk - u) - b2 * v - b3 * a
        v = v + dt * ((1.0 - gamma) * a + gamma * an)
        u, a, t = uk, an, tn
        if contact is not None:
            contact.accept_step(u)
        if track_energy:
            energy_row(t)
    return dict(u=u, v=v, a=a, newton_iters=newton_iters, pcg_iters=pcg_iters, energy=energy)


def explicit_lumped(problem, load, dt, n_steps, u0=None, v0=None, contact=None):
    """Central difference with row-sum lumped mass and penalty contact (D6).

    Startup a0 = M_L^-1 psi0, u_{-1} = u0 - dt v0 + dt^2/2 a0
    (dynamics.py:152-155); step w = dt^2 psi / M_L, u+ = 2u - u_prev + w,
    v = (u+ - u_prev)/(2 dt) (dynamics.py:158-164)."""
    n = problem.n_free
    u = np.zeros(n) if u0 is None else np.array(u0, float)
    v = np.zeros(n) if v0 is None else np.array(v0, float)
    ml = problem.lumped_mass()

    def psi_of(t, uu):
        p = load(t) - problem.internal_force(uu)
        if contact is not None:
            p = p + contact.force(uu)[0]
        return p

    a = psi_of(0.0, u) / ml
    u_prev = u - dt * v + 0.5 * dt * dt * a
    t = 0.0
    pen = []
    for _ in range(n_steps):
        w = dt * dt * psi_of(t, u) / ml
        un = 2.0 * u - u_prev + w
        v = (un - u_prev) / (2.0 * dt)
        u_prev, u = u, un
        t += dt
        if contact is not None:
            pen.append(contact.penetration(u))
    return dict(u=u, v=v, u_prev=u_prev, penetration=pen, m_lumped=ml)
