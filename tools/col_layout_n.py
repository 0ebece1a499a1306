"""Bank-model search of the collocated kernel's shared layouts for any N (P = N - 1),
component-serial, item w on thread w (tools/col_layout.py generalised; half-warp
64-bit model of tools/bank_model.py).  Prints the current layout's wavefronts per
element and the best 3-stride layouts found for the X, Y and U arrays.

    python tools/col_layout_n.py 7
"""
import itertools
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from bank_model import wavefronts  # noqa: E402


def run(N):
    R = range(N)

    def cost(items, addr):
        """items: lane -> item (lane order); per inner index a set of accesses by all lanes,
        split into warps of 32 (wavefronts per warp-instruction)."""
        tot = 0
        for t in R:
            addrs = [addr(it, t) for it in items]
            for w0 in range(0, len(addrs), 32):
                tot += wavefronts(addrs[w0:w0 + 32])
        return tot

    pairs = [(s, f) for s in R for f in R]  # item w = s*N + f on lane w
    F, B = 6, 3

    def costX(L):
        c = F * cost(pairs, lambda it, a: L(it[0], it[1], a))          # x write (k, j) over a
        c += F * cost(pairs, lambda it, j: L(it[0], j, it[1]))         # y read (k, a) over j
        c += B * cost(pairs, lambda it, j: L(it[0], j, it[1]))         # y' write
        c += B * cost(pairs, lambda it, a: L(it[0], it[1], a))         # x' read
        return c

    def costY(L):
        c = F * cost(pairs, lambda it, b: L(it[0], b, it[1]))          # y write (k, a) over b
        c += F * cost(pairs, lambda it, k: L(k, it[0], it[1]))         # z read (b, a) over k
        c += B * cost(pairs, lambda it, k: L(k, it[0], it[1]))         # z' write
        c += B * cost(pairs, lambda it, b: L(it[0], b, it[1]))         # y' read
        return c

    def costU(L):
        c = F * cost(pairs, lambda it, cc: L(cc, it[0], it[1]))        # z write (b, a) over c
        c += F * cost(pairs, lambda it, a: L(it[0], it[1], a))         # x pencils (c, b) over a
        c += F * cost(pairs, lambda it, b: L(it[0], b, it[1]))         # y pencils (c, a) over b
        c += B * cost(pairs, lambda it, a: L(it[0], it[1], a))         # x' pencils write
        c += 2 * B * cost(pairs, lambda it, b: L(it[0], b, it[1]))     # y' pencils read + write
        c += B * cost(pairs, lambda it, cc: L(cc, it[0], it[1]))       # z' read
        return c

    def lay(a, b, g):
        return lambda o, m, i: a * o + b * m + g * i

    def ok(a, b, g):
        return len({a * o + b * m + g * i for o in R for m in R for i in R}) == N ** 3

    nn = N * N
    XA = (nn + 14) // 16 * 16 + 1
    sy_cur = {7: 49, 9: 81, 5: 37}.get(N, nn)
    cur = {"X": (N, 1, XA), "Y": (sy_cur, N, 1), "U": (nn, N, 1)}
    print("N", N, "current", {k: f(lay(*cur[k])) for k, f in (("X", costX), ("Y", costY), ("U", costU))})
    cands = [(a, b, g) for a in range(1, 3 * nn) for b in range(1, 2 * N + 8) for g in (1, 2, 3, N, N + 1, XA)
             if ok(a, b, g) and (N - 1) * (a + b + g) < 2 * N ** 3]
    for name, f in (("X", costX), ("Y", costY), ("U", costU)):
        best = min(cands, key=lambda c: (f(lay(*c)), (N - 1) * (c[0] + c[1] + c[2])))
        print(" best", name, best, f(lay(*best)), "span", (N - 1) * sum(best) + 1)


if __name__ == "__main__":
    run(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
