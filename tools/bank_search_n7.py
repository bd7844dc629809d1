"""Shared-memory bank search for the N = 7 split-plane sweep (1x1 tiles, H = 4, F = 4; dev helper).

Thread order (jp, e, ih, f), f fastest; thread (jp, ih, f) owns xi rows 2 ih, 2 ih + 1 of plane jp and the
eta lines (i = 2 ih, 2 ih + 1; level jp) of the single element.  Counts wavefronts per layer (bank model of tools/bank_search.py)
for candidate strides of s_q [f][u][v][k] (QP, US, KS), the scratch s_s [f][a][b][c] (SP, AS, BS) and the
isotropic metric [i][k][j] (row stride MIS), and prints the best ones next to the plain padded layout.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from bank_search import wavefronts as _wf_full  # noqa: E402


def wavefronts(addrs):
    """64-bit accesses are served per half-warp (ncu-confirmed on the N = 4 and N = 7 sweeps): the
    wavefronts of a warp instruction are those of its two 16-lane halves."""
    return _wf_full(addrs[:16]) + _wf_full(addrs[16:])

n, N, F, H = 8, 7, 4, 4
NR = n // H
U = V = n
NT = n * F * H          # 128 plane threads, no helpers


def lanes():
    for warp in range(NT // 32):
        out = []
        for ln in range(32):
            tid = warp * 32 + ln
            f = tid % F
            ih = (tid // F) % H
            jp = tid // (F * H)
            out.append((jp, ih, f))
        yield out


def cost_q(QP, KS, US):
    qa = lambda f, u, v, k: f * QP + u * US + v * KS + k
    t = 0
    for lw in lanes():
        for r in range(NR):
            for k in range(n):
                t += wavefronts([qa(f, ih * NR + r, jp, k) for jp, ih, f in lw])
        for kk in range(NR):   # eta lines (i = 2 ih + kk, level jp)
            for a in range(n):
                t += wavefronts([qa(f, ih * NR + kk, a, jp) for jp, ih, f in lw])
    for warp in range(NT // 32):   # gather (node-granular, all F fields per node)
        for it in range((U * V * n) // NT):
            nodes = [warp * 32 + ln + it * NT for ln in range(32)]
            for f in range(F):
                t += wavefronts([qa(f, x // (V * n), (x // n) % V, x % n) for x in nodes])
    return t


def cost_s(SP, AS, BS):
    sa = lambda f, a, b, c: f * SP + a * AS + b * BS + c
    t = 0
    for lw in lanes():
        for kk in range(NR):   # eta lines (i = 2 ih + kk, level jp)
            for a2 in range(n):
                t += 3 * wavefronts([sa(f, ih * NR + kk, a2, jp) for jp, ih, f in lw])
        for r in range(NR):
            for k in range(n):
                t += 4 * wavefronts([sa(f, ih * NR + r, jp, k) for jp, ih, f in lw])
    for warp in range(NT // 32):   # node-owner step: items (column, k < N), one copy per node at 1x1 tiles
        for it in range((U * V * N + NT - 1) // NT):
            items = [warp * 32 + ln + it * NT for ln in range(32)]
            items = [x if x < U * V * N else None for x in items]
            for f in range(F):
                t += wavefronts([None if x is None else sa(f, (x // N) // V, (x // N) % V, x % N) for x in items])
    return t


def cost_m(MIS):
    ma = lambda i, k, j: i * MIS + k * n + j
    t = 0
    for lw in lanes():
        for r in range(NR):
            for k in range(n):
                t += wavefronts([ma(ih * NR + r, k, jp) for jp, ih, f in lw])
    return t


if __name__ == "__main__":
    pad16 = lambda x: x + ((4 - (x % 16)) + 16) % 16
    qs = sorted((cost_q(U * (V * KS + usp) + qp, KS, V * KS + usp), U * (V * KS + usp) + qp, KS, V * KS + usp)
                for KS in (8, 9, 10, 11) for usp in range(8) for qp in range(16))
    print("s_q best (cost, QP, KS, US):", qs[:4], "plain:", cost_q(pad16(U * V * n), n, V * n))
    ss = sorted((cost_s(n * (n * BS + asp) + spp, n * BS + asp, BS), n * (n * BS + asp) + spp, n * BS + asp, BS)
                for BS in (8, 9, 10, 11) for asp in range(8) for spp in range(16))
    print("s_s best (cost, SP, AS, BS):", ss[:4], "plain:", cost_s(pad16(n ** 3), n * n, n))
    ms = sorted((cost_m(n * n + p), n * n + p) for p in range(17))
    print("metric best (cost, MIS):", ms[:4], "plain:", cost_m(n * n))
