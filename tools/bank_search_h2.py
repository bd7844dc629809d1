"""Shared-memory bank search for the plane kernel with split planes at N = 4 (H = 2, dev helper).

Thread order (jp, e, ih, f), f fastest; thread (e, jp, ih, f) owns xi rows I0 = 3 ih .. I0 + 3 (row 5 is a
dummy) and eta-line zeta levels K0 = 3 ih .. K0 + 3.  Counts wavefronts per tile-layer of every shared access
pattern (same bank model as tools/bank_search.py) for candidate padded strides of s_q [f][u][v][k] and the
scratch s_s [f][e][a][b][c]; prints the best layouts.
"""
import itertools
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from bank_search import wavefronts  # noqa: E402

n, N, TX, TY, F, H = 5, 4, 2, 2, 4, 2
NR = (n + H - 1) // H
U, V = TX * N + 1, TY * N + 1
NE = TX * TY
NP = NE * n * F * H
NT = (NP + 31) & ~31


def lanes():
    for warp in range(NT // 32):
        out = []
        for ln in range(32):
            tid = warp * 32 + ln
            if tid >= NP:
                out.append(None)
                continue
            f = tid % F
            ih = (tid // F) % H
            e = (tid // (F * H)) % NE
            jp = tid // (F * H * NE)
            out.append((e, jp, ih, f))
        yield out


def node_uvk(node):
    uv, k = divmod(node, n)
    u, v = divmod(uv, V)
    return u, v, k


def cost_q(QP, KS, US):
    qa = lambda f, u, v, k: f * QP + u * US + v * KS + k
    t = 0
    for lw in lanes():
        for r in range(NR):
            for k in range(n):
                t += wavefronts([None if x is None or x[2] * NR + r >= n else
                                 qa(x[3], (x[0] // TY) * N + x[2] * NR + r, (x[0] % TY) * N + x[1], k) for x in lw])
        for kk in range(NR):
            for a in range(n):
                t += wavefronts([None if x is None or x[2] * NR + kk >= n else
                                 qa(x[3], (x[0] // TY) * N + x[1], (x[0] % TY) * N + a, x[2] * NR + kk) for x in lw])
    PN = (U * V * n + NT - 1) // NT
    for warp in range(NT // 32):
        for it in range(PN):
            nodes = [warp * 32 + ln + it * NT for ln in range(32)]
            nodes = [x if x < U * V * n else None for x in nodes]
            for f in range(F):
                t += wavefronts([None if x is None else qa(f, *node_uvk(x)) for x in nodes])
    return t


def cost_s(SP, ES, AS, BS):
    sa = lambda f, e, a, b, c: f * SP + e * ES + a * AS + b * BS + c
    t = 0
    for lw in lanes():
        for r in range(NR):        # c: d1 load + flux store; e: load + store -> 4 per (row, k)
            for k in range(n):
                t += 4 * wavefronts([None if x is None or x[2] * NR + r >= n else
                                     sa(x[3], x[0], x[2] * NR + r, x[1], k) for x in lw])
        for kk in range(NR):       # b: eta strong store; d: load + store -> 3 per (level, a)
            for a in range(n):
                t += 3 * wavefronts([None if x is None or x[2] * NR + kk >= n else
                                     sa(x[3], x[0], x[1], a, x[2] * NR + kk) for x in lw])
    return t


if __name__ == "__main__":
    qs = []
    for KS in (5, 6, 7):
        for usp in range(8):
            US = V * KS + usp
            for qpad in range(16):
                QP = U * US + qpad
                qs.append((cost_q(QP, KS, US), QP, KS, US))
    qs.sort()
    print("s_q best (cost, QP, KS, US):", qs[:5], " plain:", [x for x in qs if x[1:] == (U * V * n + ((4 - (U * V * n) % 16) + 16) % 16, n, V * n)][:1])
    ss = []
    for BS in (5, 6, 7):
        for asp in range(4):
            AS = n * BS + asp
            for esp in range(8):
                ES = n * AS + esp
                for spp in range(16):
                    SP = NE * ES + spp
                    ss.append((cost_s(SP, ES, AS, BS), SP, ES, AS, BS))
    ss.sort()
    print("s_s best (cost, SP, ES, AS, BS):", ss[:5])
