"""Lane-remap model for NEXT-3 pass A (k_mana_rowS, N = 12: 243 thread groups, 5 shifted digits).

Thread group g loads the 9-blocks at rowA[9 shift(g, c) + k] and rowB[9 neg(g, c) + k] and stores
its 9 results at tile[9 g + i]; 9 = 1 (mod 8), so a quarter-warp (8 lanes) is conflict-free on all
three accesses iff g, shift(g, c) and neg(g, c) are each injective mod 8 over its lanes.
    python tools/mana_remap_model.py [shifts]
prints, for random shifts c: the identity order's wavefronts (ideal 9 x 3 x 31 = 837), a greedy
partition into conflict-free octets (how many octets it needs; a 256-thread CTA has 32), and
annealing into 31 full octets (residual key collisions).  DESIGN.md section 17 quotes the result."""
import itertools
import math
import random
import sys

D = 5
NT = 3 ** D


def digits(x):
    return [(x // 3 ** j) % 3 for j in range(D)]


def shift(g, c, neg):
    gd = digits(g)
    return sum((((6 - gd[j] - c[j]) % 3) if neg else ((gd[j] - c[j] + 3) % 3)) * 3 ** j for j in range(D))


def keys(c):
    return [(g % 8, shift(g, c, 0) % 8, shift(g, c, 1) % 8) for g in range(NT)]


def cost(octets, c):
    """Wavefronts of the 9 + 9 loads and 9 stores per quarter-warp (distinct addresses per bank group)."""
    tot = 0
    for o in octets:
        for f in (lambda g: shift(g, c, 0), lambda g: shift(g, c, 1), lambda g: g):
            groups = {}
            for g in o:
                groups.setdefault(f(g) % 8, set()).add(f(g))
            tot += 9 * max(len(s) for s in groups.values())
    return tot


def greedy(c, tries=30, rnd=random):
    k = keys(c)
    best = None
    for _ in range(tries):
        rem = list(range(NT))
        rnd.shuffle(rem)
        octs = []
        while rem:
            o, used = [], [set(), set(), set()]
            for g in list(rem):
                if len(o) == 8:
                    break
                if all(k[g][i] not in used[i] for i in range(3)):
                    o.append(g)
                    for i in range(3):
                        used[i].add(k[g][i])
                    rem.remove(g)
            octs.append(o)
        if best is None or len(octs) < len(best):
            best = octs
    return best


def anneal(c, nb=31, iters=200000, seed=0):
    rnd = random.Random(seed)
    k = keys(c)
    slots = list(range(NT)) + [None] * (nb * 8 - NT)
    rnd.shuffle(slots)
    cnt = [[[0] * 8 for _ in range(3)] for _ in range(nb)]

    def upd(b, g, s):
        if g is None:
            return 0
        d = 0
        for i in range(3):
            if s > 0:
                d += cnt[b][i][k[g][i]]
                cnt[b][i][k[g][i]] += 1
            else:
                cnt[b][i][k[g][i]] -= 1
                d += cnt[b][i][k[g][i]]
        return d

    col = sum(upd(p // 8, g, 1) for p, g in enumerate(slots))
    temp = 2.0
    for _ in range(iters):
        p, q = rnd.randrange(nb * 8), rnd.randrange(nb * 8)
        if p // 8 == q // 8 or (slots[p] is None and slots[q] is None):
            continue
        bp, bq, gp, gq = p // 8, q // 8, slots[p], slots[q]
        d = -upd(bp, gp, -1) - upd(bq, gq, -1) + upd(bp, gq, 1) + upd(bq, gp, 1)
        if d <= 0 or rnd.random() < math.exp(-d / temp):
            slots[p], slots[q] = gq, gp
            col += d
        else:
            upd(bp, gq, -1), upd(bq, gp, -1), upd(bp, gp, 1), upd(bq, gq, 1)
        temp = max(0.05, temp * 0.99997)
        if col == 0:
            break
    return col


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    rnd = random.Random(1)
    shifts = rnd.sample([list(c) for c in itertools.product(range(3), repeat=D)], n)
    for c in shifts:
        ident = cost([list(range(q, min(q + 8, NT))) for q in range(0, NT, 8)], c)
        octs = greedy(c, rnd=rnd)
        print(f"c={c}: identity {ident} ({ident / 837:.2f}x ideal); greedy {len(octs)} octets, "
              f"{cost(octs, c)} wavefronts; annealed 31 octets: {anneal(c)} collisions", flush=True)
