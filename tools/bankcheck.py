"""Shared-memory wavefront estimator for the predictor layouts (sm_100:
32 banks x 4 B; 64-bit accesses are served per half-warp, 128-bit per
quarter-warp; identical words broadcast)."""
import itertools


def wavefronts(addrs_bytes, width):
    lanes_per_phase = {4: 32, 8: 16, 16: 8}[width]
    total = 0
    for ph in range(0, 32, lanes_per_phase):
        banks = {}
        for a in addrs_bytes[ph:ph + lanes_per_phase]:
            if a is None:
                continue
            for w in range(a // 4, (a + width) // 4):
                banks.setdefault(w % 32, set()).add(w)
        total += max((len(s) for s in banks.values()), default=0)
    return total


def lanes(P, D, order):
    """thread items of one element in lane order -> list of (la, lb, lt)"""
    items = []
    for it in range(P ** D):
        if order == "la":
            la, lb, lt = it % P, (it // P) % P, it // (P * P)
        else:
            lt, lb, la = it % P, (it // P) % P, it // (P * P)
        items.append((la, lb, lt))
    return items


def avg_wf(P, fn, width, order="la", n=125):
    its = lanes(P, 3, order)
    tot = 0
    cnt = 0
    for w0 in range(0, n, 32):
        warp = its[w0:w0 + 32] + [None] * max(0, 32 - len(its[w0:w0 + 32]))
        for var in fn.variants:
            addrs = [None if x is None else 8 * fn(x, *var) for x in warp]
            tot += wavefronts(addrs, width)
            cnt += 1
    return tot / cnt
