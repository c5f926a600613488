"""Bank-group model of k_legs04_tma's four shared-memory legs on the 81 x 81 tile (element R + 81 C,
16-B double2 slots): for each leg J, score every order of the six free ternary digits as the fiber ->
thread map (fastest first).  An LDS.128/STS.128 runs as 4 phases of 8 threads; a phase costs as
many wavefronts as its most-shared 16-B bank group (slot mod 8) has distinct addresses.

    python tools/mana_tile_order.py        # prints the best order per leg and the tile total
The same model gives 9126 for leg_stage's generic order (ncu: 9717 per tile)."""
import itertools

NT = 256


def wavefronts(addrs):
    tot = 0
    for ph in range(4):
        groups = {}
        for a in addrs[8 * ph:8 * ph + 8]:
            if a is not None:
                groups.setdefault(a % 8, set()).add(a)
        if groups:
            tot += max(len(s) for s in groups.values())
    return tot


def leg_cost(J, order, P=81):
    """order: digit codes fastest first, 0..3 row digit k, 4..7 column digit k - 4."""
    tot, PJ = 0, 3 ** J
    for base in range(0, 729, NT):
        for w in range(0, NT, 32):
            if base + w >= 729:
                continue
            fib = []
            for lane in range(32):
                f = base + w + lane
                if f >= 729:
                    fib.append(None)
                    continue
                tb = 0
                for k in order:
                    tb += (f % 3) * (3 ** k if k < 4 else P * 3 ** (k - 4))
                    f //= 3
                fib.append(tb)
            for r in range(3):
                for c in range(3):
                    tot += 2 * wavefronts([None if b is None else b + r * PJ + c * P * PJ for b in fib])
    return tot


if __name__ == "__main__":
    total = 0
    for J in range(4):
        free = [k for k in range(4) if k != J] + [4 + k for k in range(4) if k != J]
        cost, order = min((leg_cost(J, o), o) for o in itertools.permutations(free))
        total += cost
        print(f"leg {J}: {cost} wavefronts, order {order}")
    print("tile total", total)
