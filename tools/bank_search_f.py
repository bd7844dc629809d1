"""Bank model for the plane kernel's element scratch s_s (dev helper): the step b-e
plane / eta-line accesses plus step f's element-copy sums in the item orders of the tile-ordered passes
(pass 1: (k, u, v) block order; pass 2: s_perm order, tile-owned columns first), half-warp model.

python tools/bank_search_f.py        -> the current layout's cost and the best candidates
"""
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from bank_search import NE, N, NT, TX, TY, U, V, elem_copies, F, lanes, n, wf_half  # noqa: E402


def items_kuv():
    return [(u, v, k) for k in range(N) for u in range(U) for v in range(V)]


def items_perm(owned=lambda u, v: 0 < u < U - 1 and 0 < v < V - 1):
    cols = [(u, v) for u in range(U) for v in range(V) if owned(u, v)]
    cols += [(u, v) for u in range(U) for v in range(V) if not owned(u, v)]
    return [(u, v, k) for (u, v) in cols for k in range(N)]


def cost(SP, ES, AS, BS, wf=wf_half):
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
    NTH = 96
    for name, items in (("f_kuv", items_kuv()), ("f_perm", items_perm())):
        nit = len(items)
        for warp in range(NTH // 32):
            for it in range((nit + NTH - 1) // NTH):
                idx = [warp * 32 + ln + it * NTH for ln in range(32)]
                sel = [items[x] if x < nit else None for x in idx]
                for f in range(F):
                    for c in range(4):
                        addrs = []
                        for x in sel:
                            if x is None:
                                addrs.append(None)
                                continue
                            u, v, k = x
                            cp = elem_copies(u, v)
                            addrs.append(sa(f, cp[c][0], cp[c][1], cp[c][2], k) if c < len(cp) else None)
                        if any(a is not None for a in addrs):
                            t[name] += wf(addrs)
    return t


if __name__ == "__main__":
    cur = cost(588, 147, 28, 5)
    print("current (588,147,28,5)", dict(cur), sum(cur.values()))
    res = []
    for BS in (5, 6, 7):
        for AS in range(n * BS, n * BS + 6):
            for ES in range(n * AS, n * AS + 8):
                for SP in range(NE * ES, NE * ES + 8):
                    if SP > 660:
                        continue
                    c = cost(SP, ES, AS, BS)
                    res.append((sum(c.values()), c["f_kuv"], c["f_perm"], SP, ES, AS, BS))
    res.sort()
    for r in res[:12]:
        print(r)


def items_perm_colfast(owned=lambda u, v: 0 < u < U - 1 and 0 < v < V - 1):
    cols = [(u, v) for u in range(U) for v in range(V) if owned(u, v)]
    cols += [(u, v) for u in range(U) for v in range(V) if not owned(u, v)]
    return [(u, v, k) for k in range(N) for (u, v) in cols]


def cost_items(items, SP=588, ES=147, AS=28, BS=5, wf=wf_half):
    sa = lambda f, e, a, b, c: f * SP + e * ES + a * AS + b * BS + c
    NTH, tot = 96, 0
    nit = len(items)
    for warp in range(NTH // 32):
        for it in range((nit + NTH - 1) // NTH):
            idx = [warp * 32 + ln + it * NTH for ln in range(32)]
            sel = [items[x] if x < nit else None for x in idx]
            for f in range(F):
                for c in range(4):
                    addrs = []
                    for x in sel:
                        if x is None:
                            addrs.append(None)
                            continue
                        u, v, k = x
                        cp = elem_copies(u, v)
                        addrs.append(sa(f, cp[c][0], cp[c][1], cp[c][2], k) if c < len(cp) else None)
                    if any(a is not None for a in addrs):
                        tot += wf(addrs)
    return tot
