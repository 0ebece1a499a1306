"""Shared-memory bank-conflict model for the v2/v3 element-kernel layouts.

A warp-wide 64-bit LDS/STS touches two 4-byte banks per lane and is served
per half-warp; see wavefronts().
Used to choose padded strides / item orders ("shared layouts").
"""
import itertools
import sys


def wavefronts(addrs):
    """64-bit accesses are served per half-warp (16 lanes x 8 B = 128 B); the
    cost of each half is the max number of distinct words in one bank.  This
    model reproduces the measured v2/v3 LDS/STS wavefront ratios (1.33-1.49)."""
    total = 0
    for half in (addrs[:16], addrs[16:]):
        banks = {}
        for d in half:
            for w in (2 * d, 2 * d + 1):
                banks.setdefault(w % 32, set()).add(w)
        total += max(len(s) for s in banks.values()) if banks else 0
    return total


def stage(items, order, access, T=32):
    """items: list of item tuples; order: permutation index of items -> lane slot;
    access(item, inner) -> double index, inner loops over the per-item accesses."""
    seq = [items[i] for i in order]
    total = 0
    ideal = 0
    rounds = (len(seq) + T - 1) // T
    for r in range(rounds):
        lanes = seq[r * T:(r + 1) * T]
        for inner in access.inners:
            addrs = [access(it, inner) for it in lanes]
            total += wavefronts(addrs)
            ideal += (len(addrs) * 8 + 127) // 128
    return total, ideal


class Acc:
    def __init__(self, fn, inners):
        self.fn, self.inners = fn, inners

    def __call__(self, it, inner):
        return self.fn(it, inner)


def evaluate(N, M, sck_x, sck_y, sq, orders, NC=3):
    """Total / ideal wavefronts of all shared accesses of one element (apply mode)."""
    NX = [(c, k, j) for c in range(NC) for k in range(N) for j in range(N)]
    NY = [(c, k, a) for c in range(NC) for k in range(N) for a in range(M)]
    NZ = [(c, b, a) for c in range(NC) for b in range(M) for a in range(M)]
    X = lambda c, k, j, a, s: s * NC * N * sck_x + (c * N + k) * sck_x + j * M + a
    Y = lambda c, s, k, b, a: (c * 3 + s) * N * sck_y + k * sck_y + b * M + a
    Qi = lambda c, d, q: (d * 3 + c) * sq + q
    tot = ideal = 0
    def add(x):
        nonlocal tot, ideal
        tot += x[0]; ideal += x[1]
    ox, oy, oz = orders
    reps = 3 // NC
    # forward x2 (u and p): X writes (B, D), Y reads X (2) writes Y (3), Z reads Y (3) writes Q (3)
    for _ in range(2 * reps):
        add(stage(NX, ox, Acc(lambda it, i: X(it[0], it[1], it[2], i[0], i[1]), [(a, s) for a in range(M) for s in range(2)])))
        add(stage(NY, oy, Acc(lambda it, i: X(it[0], it[1], i[0], it[2], i[1]), [(j, s) for j in range(N) for s in range(2)])))
        add(stage(NY, oy, Acc(lambda it, i: Y(it[0], i[1], it[1], i[0], it[2]), [(b, s) for b in range(M) for s in range(3)])))
        add(stage(NZ, oz, Acc(lambda it, i: Y(it[0], i[1], i[0], it[1], it[2]), [(k, s) for k in range(N) for s in range(3)])))
        add(stage(NZ, oz, Acc(lambda it, i: Qi(it[0], i[1], i[0] * M * M + it[1] * M + it[2]), [(c, d) for c in range(M) for d in range(3)])))
    # backward: Z' reads Q (3) writes Y-layout (3); Y' reads (3) writes X-layout (2); X' reads (2)
    for _ in range(reps):
        _backward(N, M, NX, NY, NZ, X, Y, Qi, ox, oy, oz, add)
    return tot, ideal


def _backward(N, M, NX, NY, NZ, X, Y, Qi, ox, oy, oz, add):
    if True:
        add(stage(NZ, oz, Acc(lambda it, i: Qi(it[0], i[1], i[0] * M * M + it[1] * M + it[2]), [(c, d) for c in range(M) for d in range(3)])))
        add(stage(NZ, oz, Acc(lambda it, i: Y(it[0], i[1], i[0], it[1], it[2]), [(k, s) for k in range(N) for s in range(3)])))
        add(stage(NY, oy, Acc(lambda it, i: Y(it[0], i[1], it[1], i[0], it[2]), [(b, s) for b in range(M) for s in range(3)])))
        add(stage(NY, oy, Acc(lambda it, i: X(it[0], it[1], i[0], it[2], i[1]), [(j, s) for j in range(N) for s in range(2)])))
        add(stage(NX, ox, Acc(lambda it, i: X(it[0], it[1], it[2], i[0], i[1]), [(a, s) for a in range(M) for s in range(2)])))


if __name__ == "__main__":
    N, M = int(sys.argv[1]), int(sys.argv[2])
    nat = lambda n: list(range(n))
    base = evaluate(N, M, N * M, M * M, M ** 3, (nat(3 * N * N), nat(3 * N * M), nat(3 * M * M)))
    print("natural", base)
    best = None
    for sx in range(N * M, N * M + 16):
        for sy in range(M * M, M * M + 16):
            for sq in range(M ** 3, M ** 3 + 16):
                r = evaluate(N, M, sx, sy, sq, (nat(3 * N * N), nat(3 * N * M), nat(3 * M * M)))
                if best is None or r[0] < best[0][0]:
                    best = (r, sx, sy, sq)
    print("best padded", best)


def orders_for(N, M, NC=3):
    """Candidate lane->item orders per stage (natural, transposed)."""
    NX = [(c, k, j) for c in range(NC) for k in range(N) for j in range(N)]
    NY = [(c, k, a) for c in range(NC) for k in range(N) for a in range(M)]
    NZ = [(c, b, a) for c in range(NC) for b in range(M) for a in range(M)]
    def perm(items, key):
        return sorted(range(len(items)), key=lambda i: key(items[i]))
    ox = {"nat": list(range(len(NX))), "jfirst": perm(NX, lambda t: (t[2], t[0], t[1]))}
    oy = {"nat": list(range(len(NY))), "ckfirst": perm(NY, lambda t: (t[2], t[0], t[1])),
          "kfirst": perm(NY, lambda t: (t[0], t[2], t[1]))}
    oz = {"nat": list(range(len(NZ)))}
    return ox, oy, oz


def search(N, M, NC=3):
    ox, oy, oz = orders_for(N, M, NC)
    best = None
    for (nx_, o1), (ny_, o2), (nz_, o3) in itertools.product(ox.items(), oy.items(), oz.items()):
        for sx in range(N * M, N * M + 16):
            for sy in range(M * M, M * M + 16):
                sq = M ** 3 + ((M * M - M ** 3) % 16)
                r = evaluate(N, M, sx, sy, sq, (o1, o2, o3), NC)
                if best is None or r[0] < best[0][0]:
                    best = (r, nx_, ny_, nz_, sx, sy, sq)
    return best
