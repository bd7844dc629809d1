"""Shared-memory bank model for the tile-ordered intermediate (IO 2 reads of lap_plane.cu; dev helper,
DESIGN.md §4.2): half-warp wavefronts of the step-b q reads (plane and eta-line loads) for candidate
block layouts.  A block holds the k < N levels of one tile-layer; the top level k = N is level 0 of
the next block (other ring slot, same layout).

split layout: tile-interior columns (1 <= u, v <= N*TX - 1) field-major [f][u-1][k][v-1] with strides
(QP, US, KS, 1); perimeter columns (shared with other tiles; the slot fix-up writes them as 128-byte
runs) [pidx][k][f] with strides (PS, 4, 1) after the interior part (offset PB).
"""
import itertools
import sys
from collections import defaultdict

n, N, TX, TY, F = 5, 4, 2, 2, 4
U, V = TX * N + 1, TY * N + 1
NE = TX * TY
NT = 96


def wavefronts(addrs):
    per_bank = defaultdict(set)
    for a in addrs:
        if a is None:
            continue
        per_bank[a % 16].add(a)
    return max((len(s) for s in per_bank.values()), default=0)


def wf_half(addrs):
    return wavefronts(addrs[:16]) + wavefronts(addrs[16:])


def lanes():
    for warp in range((NT + 31) // 32):
        out = []
        for ln in range(32):
            tid = warp * 32 + ln
            if tid >= NE * n * F:
                out.append(None)
            else:
                f = tid % F
                e = (tid // F) % NE
                jp = tid // (F * NE)
                out.append((e, jp, f))
        yield out


def perim_order():
    p = [(0, v) for v in range(V)] + [(U - 1, v) for v in range(V)]
    p += [(u, 0) for u in range(1, U - 1)] + [(u, V - 1) for u in range(1, U - 1)]
    return {c: i for i, c in enumerate(p)}


PIDX = perim_order()


def cost(addr):
    tot = 0
    for lw in lanes():
        for i in range(n):
            for k in range(n):
                tot += wf_half([None if x is None else addr(x[2], (x[0] // TY) * N + i, (x[0] % TY) * N + x[1], k)
                                for x in lw])
                tot += wf_half([None if x is None else addr(x[2], (x[0] // TY) * N + x[1], (x[0] % TY) * N + i, k)
                                for x in lw])
    return tot


def full(QP=345, US=38, KS=9):
    def a(f, u, v, k):
        kk = k if k < N else 0
        return f * QP + u * US + kk * KS + v
    return a


def split(QP, US, KS, PB, PS):
    def a(f, u, v, k):
        kk = k if k < N else 0
        if 1 <= u <= U - 2 and 1 <= v <= V - 2:
            return f * QP + (u - 1) * US + kk * KS + (v - 1)
        return PB + PIDX[(u, v)] * PS + kk * 4 + f
    return a


if __name__ == "__main__":
    base = cost(full())
    print("full grid [f][u][k][v] (345, 38, 9):", base, "wavefronts / tile-layer")
    best = []
    ni = (U - 2)
    for KS in (7, 8, 9):
        for US in range(ni * 0 + 4 * KS, 4 * KS + 6):
            for QP in range(ni * US, ni * US + 8):
                interior = F * QP
                for PBo in range(0, 16, 4):
                    PB = ((interior + 3) // 4) * 4 + PBo
                    for PS in (16, 20, 24):
                        c = cost(split(QP, US, KS, PB, PS))
                        size = PB + len(PIDX) * PS
                        best.append((c, size, QP, US, KS, PB, PS))
        print("KS", KS, "done", min(best), flush=True)
    best.sort()
    for b in best[:15]:
        print(b)
