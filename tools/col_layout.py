"""Shared-memory layout search for the collocated element kernel (element_col.cuh, P = 4).

Every 1D stage of one element is 25 pencils on 25 lanes; each pencil reads or
writes 5 doubles of a 5x5x5 array.  The arrays (x-stage output X, y-stage
output Y, point values U, point slots Q) are laid out as
    addr = alpha * outer + beta * middle + inner
and each stage chooses which of its two pencil indices is the fast lane index.
This script evaluates the half-warp 64-bit bank model (tools/bank_model.py;
validated against ncu) for every access of the forward u and p passes and the
backward pass, and searches strides and lane orders for the minimum number of
shared wavefronts per element.

    python tools/col_layout.py          # current layout, then the best found
"""
import itertools
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from bank_model import wavefronts  # noqa: E402

N = 5
R5 = range(N)


def lanes(order):
    """items of a stage in lane order: order 0 -> (p, q) with q fastest."""
    return [(p, q) if order == 0 else (q, p) for p in R5 for q in R5] if True else None


def items(order):
    out = []
    for s in R5:
        for f in R5:
            out.append((s, f) if order == 0 else (f, s))
    return out


class Lay:
    def __init__(self, al, be):
        self.al, self.be = al, be

    def __call__(self, o, m, i):
        return self.al * o + self.be * m + i

    def ok(self):
        return len({self(o, m, i) for o in R5 for m in R5 for i in R5}) == N ** 3

    def span(self):
        return max(self(o, m, i) for o in R5 for m in R5 for i in R5) + 1


def cost_access(its, addr):
    """its: the 25 lane items; addr(item, t) for t in 0..4 -> total wavefronts."""
    return sum(wavefronts([addr(it, t) for it in its]) for t in R5)


def total(X, Y, U, Q, o):
    """o: lane orders of the stages (dict).  Returns (X, Y, U, Q) wavefronts per element."""
    cx = cy = cu = cq = 0
    F = 6  # forward passes: 2 fields x 3 components
    B = 3  # backward: 3 components
    # forward x stage: items (k, j); X write (k, j, a)
    its = items(o["x"])
    cx += F * cost_access(its, lambda it, a: X(it[0], it[1], a))
    # y stage: items (k, a); X read (k, j, a) over j; Y write (k, b, a) over b
    its = items(o["y"])
    cx += F * cost_access(its, lambda it, j: X(it[0], j, it[1]))
    cy += F * cost_access(its, lambda it, b: Y(it[0], b, it[1]))
    # z stage: items (b, a); Y read (k, b, a) over k; U write and Q2 write (c, b, a) over c
    its = items(o["z"])
    cy += F * cost_access(its, lambda it, k: Y(k, it[0], it[1]))
    cu += F * cost_access(its, lambda it, c: U(c, it[0], it[1]))
    cq += F * cost_access(its, lambda it, c: Q(c, it[0], it[1]))
    # x pencils: items (c, b); U read / Q0 write (c, b, a) over a
    its = items(o["px"])
    cu += F * cost_access(its, lambda it, a: U(it[0], it[1], a))
    cq += F * cost_access(its, lambda it, a: Q(it[0], it[1], a))
    # y pencils: items (c, a); U read / Q1 write (c, b, a) over b
    its = items(o["py"])
    cu += F * cost_access(its, lambda it, b: U(it[0], b, it[1]))
    cq += F * cost_access(its, lambda it, b: Q(it[0], b, it[1]))
    # point phase: thread t, point q = t + 32 r; 9 (u) + 9 (p) reads + 9 writes per point
    pts = [(q // 25, (q // 5) % 5, q % 5) for q in range(125)]
    for r in range(4):
        grp = pts[32 * r:32 * r + 32]
        cq += 27 * wavefronts([Q(*p) for p in grp])
    # backward x' pencils: items (c, b): Q0 read, U write over a
    its = items(o["bx"])
    cq += B * cost_access(its, lambda it, a: Q(it[0], it[1], a))
    cu += B * cost_access(its, lambda it, a: U(it[0], it[1], a))
    # y' pencils: items (c, a): Q1 read, U read + write over b
    its = items(o["by"])
    cq += B * cost_access(its, lambda it, b: Q(it[0], b, it[1]))
    cu += 2 * B * cost_access(its, lambda it, b: U(it[0], b, it[1]))
    # z': items (b, a): U read, Q2 read over c; Y write over k
    its = items(o["bz"])
    cu += B * cost_access(its, lambda it, c: U(c, it[0], it[1]))
    cq += B * cost_access(its, lambda it, c: Q(c, it[0], it[1]))
    cy += B * cost_access(its, lambda it, k: Y(k, it[0], it[1]))
    # y': items (k, a): Y read over b, X write over j
    its = items(o["byy"])
    cy += B * cost_access(its, lambda it, b: Y(it[0], b, it[1]))
    cx += B * cost_access(its, lambda it, j: X(it[0], j, it[1]))
    # x': items (k, j): X read over a
    its = items(o["bxx"])
    cx += B * cost_access(its, lambda it, a: X(it[0], it[1], a))
    return cx, cy, cu, cq


CUR = dict(X=(25, 5), Y=(37, 5), U=(25, 5), Q=(25, 5))
CUR_O = dict(x=0, y=0, z=0, px=0, py=0, bx=0, by=0, bz=0, byy=0, bxx=0)


CANDS = [L for L in (Lay(a, b) for a in range(25, 44) for b in range(5, 9)) if L.ok()]


def best_for(orders):
    """arrays are independent given the lane orders: minimise each alone"""
    o = dict(zip(CUR_O, orders))
    lay = {k: Lay(*v) for k, v in CUR.items()}
    parts = []
    for idx in range(4):
        bestL = None
        for L in CANDS:
            args = [lay["X"], lay["Y"], lay["U"], lay["Q"]]
            args[idx] = L
            v = total(*args, o)[idx] * 1000 + L.span()
            if bestL is None or v < bestL[0]:
                bestL = (v, L)
        parts.append(bestL)
    return sum(p[0] // 1000 for p in parts), o, [(p[1].al, p[1].be, p[0] // 1000) for p in parts]


def main():
    from multiprocessing import Pool
    lay = {k: Lay(*v) for k, v in CUR.items()}
    c = total(lay["X"], lay["Y"], lay["U"], lay["Q"], CUR_O)
    print("current", c, sum(c))
    with Pool() as pool:
        res = pool.map(best_for, itertools.product((0, 1), repeat=len(CUR_O)), chunksize=8)
    res.sort(key=lambda r: r[0])
    for r in res[:5]:
        print(r)


if __name__ == "__main__":
    main()
