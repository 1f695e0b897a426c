"""Padding search for the slice buffers of the 3-D N >= 7 predictors (adg_predictor_stream.cu, adg_predictor_phased.cu):
Q node-major [i][j][k][v] with strides (SI, SJ, M); B x-line-major
[j][k][i][v] with strides (TJ, TK, M).  Lanes of each owner role map to
(a0, b0) = (rr // P, rr % P).  Prints the wavefronts per access pattern
(sum over a role's warps, all l / v) for the unpadded and the best layout."""
import sys
from bankcheck import wavefronts

M = 5


def role_warps(P):
    PP = P * P
    for w0 in range(0, PP, 32):
        yield [(rr // P, rr % P) if rr < PP else None for rr in range(w0, w0 + 32)]


def cost(P, fn):
    tot = 0
    for warp in role_warps(P):
        for l in range(P):
            for v in range(M):
                tot += wavefronts([None if x is None else 8 * fn(x[0], x[1], l, v)
                                   for x in warp], 8)
    return tot


def q_costs(P, SI, SJ):
    q = lambda i, j, k, v: i * SI + j * SJ + k * M + v
    return (cost(P, lambda a, b, l, v: q(l, a, b, v)), cost(P, lambda a, b, l, v: q(a, l, b, v)),
            cost(P, lambda a, b, l, v: q(a, b, l, v)))


def b_costs(P, TJ, TK):
    B = lambda j, k, i, v: j * TJ + k * TK + i * M + v
    return (cost(P, lambda a, b, o, v: B(o, b, a, v)), cost(P, lambda a, b, o, v: B(b, o, a, v)),
            cost(P, lambda a, b, i, v: B(a, b, i, v)))


for P in map(int, sys.argv[1:] or ["8", "9", "10"]):
    base_q = q_costs(P, P * P * M, P * M)
    best = None
    for pj in range(0, 16):
        for pi in range(0, 16):
            SJ = P * M + pj
            SI = P * SJ + pi
            c = q_costs(P, SI, SJ)
            if best is None or sum(c) < best[0]:
                best = (sum(c), pj, pi, c)
    base_b = b_costs(P, P * P * M, P * M)
    bestb = None
    for pk in range(0, 16):
        for pj in range(0, 16):
            TK = P * M + pk
            TJ = P * TK + pj
            c = b_costs(P, TJ, TK)
            if bestb is None or sum(c) < bestb[0]:
                bestb = (sum(c), pk, pj, c)
    print(f"P={P}: Q unpadded x/y/z {base_q} -> pad j {best[1]} i {best[2]}: {best[3]};"
          f" B unpadded ypub/zpub/xread {base_b} -> pad k {bestb[1]} j {bestb[2]}: {bestb[3]}")
