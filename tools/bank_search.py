"""Shared-memory bank model for the plane kernel (dev helper) (n=5, 2x2 tile, F=4, NT=80): count wavefronts
per tile-layer for the access patterns of each step under candidate padded layouts."""
import itertools
from collections import defaultdict

n, N, TX, TY, F = 5, 4, 2, 2, 4
U, V = TX * N + 1, TY * N + 1
NE = TX * TY
NT = NE * n * F


def wavefronts(addrs, width=1):
    """addrs: list of double addresses (None = inactive), width in doubles (1 or 2).
    4-byte banks: word d covers banks 2d, 2d+1 (mod 32).  Wavefronts = max distinct words per bank."""
    per_bank = defaultdict(set)
    for a in addrs:
        if a is None:
            continue
        for w in range(width):
            d = a + w
            per_bank[(2 * d) % 32].add(d)
            per_bank[(2 * d + 1) % 32].add(d)
    return max((len(s) for s in per_bank.values()), default=0)


def lanes():
    for warp in range((NT + 31) // 32):
        out = []
        for ln in range(32):
            tid = warp * 32 + ln
            if tid >= NT:
                out.append(None)
            else:
                # the kernel's thread order (jp, e, f), f fastest (lap_plane.cu); the tuned layout
                # (QP, US) = (415, 46), (SP, ES, AS) = (588, 147, 28) is optimal under it
                f = tid % F
                e = (tid // F) % NE
                jp = tid // (F * NE)
                out.append((e, jp, f))
        yield out


def cost(L):
    QP, KS, US, SP, ES, AS, BS = L
    qa = lambda f, u, v, k: f * QP + u * US + v * KS + k
    sa = lambda f, e, a, b, c: f * SP + e * ES + a * AS + b * BS + c
    tot = defaultdict(int)
    for lw in lanes():
        for i in range(n):
            for k in range(n):
                # P1 plane load q(px*N+i, py*N+jp, k)
                tot["b_plane"] += wavefronts([None if x is None else qa(x[2], (x[0] // TY) * N + i, (x[0] % TY) * N + x[1], k) for x in lw])
                # P2 eta-line q(px*N+jp, py*N+i(a), k)
                tot["b_etaq"] += wavefronts([None if x is None else qa(x[2], (x[0] // TY) * N + x[1], (x[0] % TY) * N + i, k) for x in lw])
                # P3 / P5 s_s(e, jp, a, k)
                w = wavefronts([None if x is None else sa(x[2], x[0], x[1], i, k) for x in lw])
                tot["b_etaw"] += w
                tot["d_rw"] += 2 * w
                # P4 / P6 s_s(e, i, jp, k): c read+write, e read+write
                w = wavefronts([None if x is None else sa(x[2], x[0], i, x[1], k) for x in lw])
                tot["c_rw"] += 2 * w
                tot["e_rw"] += 2 * w
    return tot


def layout_ok(L):
    QP, KS, US, SP, ES, AS, BS = L
    return KS >= n and US >= V * KS and QP >= U * US and BS >= n and AS >= n * BS and ES >= n * AS and SP >= NE * ES





def wf_half(addrs, width=1):
    return wavefronts(addrs[:16], width) + wavefronts(addrs[16:], width)


def node_uvk(node):
    uv, k = divmod(node, n)
    u, v = divmod(uv, V)
    return u, v, k


PN = (U * V * n + NT - 1) // NT


def cost_q(QP, KS, US, wf=wavefronts):
    qa = lambda f, u, v, k: f * QP + u * US + v * KS + k
    t = defaultdict(int)
    for lw in lanes():
        for i in range(n):
            for k in range(n):
                t["b_plane"] += wf([None if x is None else qa(x[2], (x[0] // TY) * N + i, (x[0] % TY) * N + x[1], k) for x in lw])
                t["b_etaq"] += wf([None if x is None else qa(x[2], (x[0] // TY) * N + x[1], (x[0] % TY) * N + i, k) for x in lw])
    for warp in range((NT + 31) // 32):
        for it in range(PN):
            nodes = [warp * 32 + ln + it * NT for ln in range(32)]
            nodes = [x if (warp * 32 + ln) < NT and x < U * V * n else None for ln, x in enumerate(nodes)]
            for f in range(F):
                t["gather"] += wf([None if x is None else qa(f, *node_uvk(x)) for x in nodes])
    return t


def elem_copies(u, v):
    pu1, pv1 = min(u // N, TX - 1), min(v // N, TY - 1)
    pu0 = u // N - 1 if (u % N == 0 and u > 0) else pu1
    pv0 = v // N - 1 if (v % N == 0 and v > 0) else pv1
    return [(a * TY + b, u - a * N, v - b * N) for a in range(pu0, pu1 + 1) for b in range(pv0, pv1 + 1)]


def cost_s(SP, ES, AS, BS, wf=wavefronts):
    sa = lambda f, e, a, b, c: f * SP + e * ES + a * AS + b * BS + c
    t = defaultdict(int)
    for lw in lanes():
        for i in range(n):
            for k in range(n):
                w = wf([None if x is None else sa(x[2], x[0], x[1], i, k) for x in lw])
                t["b_etaw"] += w
                t["d_rw"] += 2 * w
                w = wf([None if x is None else sa(x[2], x[0], i, x[1], k) for x in lw])
                t["c_rw"] += 2 * w
                t["e_rw"] += 2 * w
    for warp in range((NT + 31) // 32):
        for it in range(PN):
            nodes = [warp * 32 + ln + it * NT for ln in range(32)]
            nodes = [x if (warp * 32 + ln) < NT and x < U * V * n and x % n < N else None for ln, x in enumerate(nodes)]
            for f in range(F):
                for c in range(4):
                    addrs = []
                    for x in nodes:
                        if x is None:
                            addrs.append(None)
                            continue
                        u, v, k = node_uvk(x)
                        cp = elem_copies(u, v)
                        addrs.append(sa(f, cp[c][0], cp[c][1], cp[c][2], k) if c < len(cp) else None)
                    if any(a is not None for a in addrs):
                        t["f_read"] += wf(addrs)
    return t


def _enumerate_layouts():
    """The candidate layouts of the original search (dev record)."""
    cur = (420, 5, 45, 500, 125, 25, 5)
    c = cost(cur)
    print("current", dict(c), sum(c.values()))
    best = []
    for KS in (5, 6, 7):
        for usp in range(0, 8):
            US = V * KS + usp
            base_q = U * US
            for qpad in range(0, 16):
                QP = base_q + qpad
                for BS in (5, 6, 7):
                    for asp in range(0, 4):
                        AS = n * BS + asp
                        for esp in range(0, 8):
                            ES = n * AS + esp
                            for spp in range(0, 16):
                                SP = NE * ES + spp
                                L = (QP, KS, US, SP, ES, AS, BS)
                                best.append(L)
    print(len(best), "candidates")
    return best


if __name__ == "__main__":
    _enumerate_layouts()
    import sys
    for name, wf in (("full", wavefronts), ("half", wf_half)):
        cq = cost_q(420, 5, 45, wf); cs = cost_s(500, 125, 25, 5, wf)
        print(name, "current q", dict(cq), sum(cq.values()), "s", dict(cs), sum(cs.values()))
