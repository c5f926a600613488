"""Index algebra of the sm_100a kernels, checked on the CPU (no GPU): the TMEM transpose trips of
k_passA10s, the XOR swizzles of the radix-64 transposes, and their shared-memory bank behaviour.
The GPU tests (element-wise chi through the production kernels) check the same maps on hardware."""


def trip(state):
    """tcgen05.st 32x32b (thread l -> lane l, double column r) then two tcgen05.ld 16x256b.x8 at lane
    bases 0/16: thread t = t0 + 4 t1 gets lane 16b + 8s + t1, column 4c + t0 into register
    r = s + 2c + 16b (CUTLASS Copy_Traits<SM100_TMEM_LOAD_16dp256b1x>::DstLayout)."""
    new = [[None] * 32 for _ in range(32)]
    for t in range(32):
        t0, t1 = t & 3, t >> 2
        for b in range(2):
            for c in range(8):
                for s in range(2):
                    new[t][s + 2 * c + 16 * b] = state[16 * b + 8 * s + t1][4 * c + t0]
    return new


def pa10_freq(pos):          # csrc/sre_kernels.cuh, written out again
    t, r = pos & 31, pos >> 5
    bits = [(t & 1, 1), ((t >> 1) & 1, 8), ((t >> 2) & 1, 3), ((t >> 3) & 1, 7), ((t >> 4) & 1, 5),
            (r & 1, 6), ((r >> 1) & 1, 9), ((r >> 2) & 1, 4), ((r >> 3) & 1, 2), ((r >> 4) & 1, 0)]
    return sum(v << k for v, k in bits)


def test_tmem_trips_cover_every_bit_and_match_pa10_freq():
    state = [[l + 32 * j for j in range(32)] for l in range(32)]   # element e = lane + 32 j
    butterflied = {5, 6, 7, 8, 9}                                     # round 0: register bits
    schedule = [(0, 4), (0, 4), (4,)]                                 # register bits butterflied per trip
    for regbits in schedule:
        state = trip(state)
        for rb in regbits:   # the register bit rb must flip exactly one element bit, not yet done
            diff = state[0][1 << rb] ^ state[0][0]
            assert diff & (diff - 1) == 0
            k = diff.bit_length() - 1
            assert k not in butterflied
            butterflied.add(k)
            assert all((state[t][r] ^ state[t][r ^ (1 << rb)]) == diff for t in range(32) for r in range(32))
    assert butterflied == set(range(10))
    for t in range(32):
        for r in range(32):
            assert state[t][r] == pa10_freq(t + 32 * r)
    assert sorted(pa10_freq(p) for p in range(1024)) == list(range(1024))


def xsw12(e):
    return e ^ ((e >> 6) & 15)


def xsw13(e):
    return e ^ (((e >> 7) & 7) << 1)


def _half_warp_conflict_free(addrs):          # 8-B accesses: 16 lanes of a half-warp, 16 double banks
    return all(len({a % 16 for a in addrs[h:h + 16]}) == 16 for h in (0, 16))


def test_radix64_swizzles_bijective_and_conflict_free():
    assert sorted(map(xsw12, range(4096))) == list(range(4096))
    assert sorted(map(xsw13, range(8192))) == list(range(8192))
    # k_passAq / k_passAw: unit of 64 threads, thread t = 32 w + lane; round 0 STS at t + 64 j,
    # round 1 LDS at 64 t + j
    for w in range(2):
        for j in range(64):
            assert _half_warp_conflict_free([xsw12(32 * w + l + 64 * j) for l in range(32)])
            assert _half_warp_conflict_free([xsw12(64 * (32 * w + l) + j) for l in range(32)])
    # k_passBr / k_passBw: 128 threads; round 0 STS at t + 128 j, round 1 LDS at tb | (j << 1) with
    # tb = (t & 1) | ((t >> 1) << 7)
    for w in range(4):
        for j in range(64):
            ts = [32 * w + l for l in range(32)]
            assert _half_warp_conflict_free([xsw13(t + 128 * j) for t in ts])
            assert _half_warp_conflict_free([xsw13((t & 1) | ((t >> 1) << 7) | (j << 1)) for t in ts])


def test_row_staging_reads_pairs():
    """k_passAw stages a row at xsw12(pos) and reads 16-B chunks C = t + 64 i as the pair (2C, 2C+1):
    both sit in one aligned 16-B slot (swapped when the XOR key is odd), and a quarter-warp's 8
    chunks hit 8 distinct 16-B bank groups."""
    for c in range(2048):
        e = 2 * c
        key = (e >> 6) & 15
        base = (e ^ key) & ~1
        got = (base, base + 1) if key % 2 == 0 else (base + 1, base)
        assert (xsw12(e), xsw12(e + 1)) == got
    for q in range(0, 2048, 8):
        assert len({((2 * c) ^ ((2 * c >> 6) & 15)) // 2 % 8 for c in range(q, q + 8)}) == 8


def test_rowmajor_store_order_is_a_permutation():
    """k_passA10s<ROWM> writes (lane t, register r) at position 2 t + (r & 1) + 64 (r >> 1); the chi
    decode (pa10_freq_rowm) inverts it."""
    seen = set()
    for t in range(32):
        for r in range(32):
            pos = 2 * t + (r & 1) + 64 * (r >> 1)
            tt, rr = (pos >> 1) & 31, (pos & 1) | ((pos >> 6) << 1)
            assert (tt, rr) == (t, r)
            seen.add(pos)
    assert seen == set(range(1024))


def test_mixed_81_tile_fiber_orders():
    """k_legs04 (mana_mixed.cu ord81): each leg's fiber order is a permutation of its six free tile
    digits (so the 729 fibers cover the 81 x 81 tile once), and the bank-group model of
    tools/mana_tile_order.py rates the four orders at 6768 wavefronts per tile (ideal 6624)."""
    import os
    import re
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = open(os.path.join(root, "paper_2601_07824_b200", "csrc", "mana_mixed.cu")).read()
    body = re.search(r"constexpr int o\[4\]\[6\] = \{(.*?)\};", src).group(1)
    orders = [[int(x) for x in grp.split(",")] for grp in re.findall(r"\{([^{}]*)\}", body)]
    assert len(orders) == 4
    for J, o in enumerate(orders):
        assert sorted(o) == sorted([k for k in range(4) if k != J] + [4 + k for k in range(4) if k != J])
        covered = set()
        for f in range(729):
            tb, q = 0, f
            for k in o:
                tb += (q % 3) * (3 ** k if k < 4 else 81 * 3 ** (k - 4))
                q //= 3
            for r in range(3):
                for c in range(3):
                    covered.add(tb + r * 3 ** J + 81 * c * 3 ** J)
        assert covered == set(range(6561))
    sys.path.insert(0, os.path.join(root, "tools"))
    from mana_tile_order import leg_cost
    assert sum(leg_cost(J, orders[J]) for J in range(4)) == 6768


def test_passaw_tma_store_staging():
    """k_passAw<TS>: after round 1 thread t holds v[j] = position 64 t + j of the row-plane.  It writes
    the pair (v[j], v[j+1]) as the 16-B chunk at byte 8192 (j >> 4) + 128 t + 16 (((j & 15) >> 1) ^ (t & 7)).
    The TMA tensor store (box {16 doubles, 64 rows}, SWIZZLE_128B: 16-B chunk bits [4:6] ^= bits [7:9]
    of the box offset) must read position 64 t + 16 b + jj there, and each quarter-warp STS.128 must hit
    8 distinct 16-B bank groups."""
    def tma_image(b, row, jj):                  # where the TMA engine expects box b's element (jj, row)
        off = 128 * row + 8 * jj
        return 8192 * b + (off ^ (((off >> 7) & 7) << 4))

    seen = set()
    for t in range(64):
        for j in range(0, 64, 2):
            addr = 8192 * (j >> 4) + 128 * t + 16 * ((((j & 15) >> 1)) ^ (t & 7))
            assert addr == tma_image(j >> 4, t, j & 15)
            assert addr + 8 == tma_image(j >> 4, t, (j & 15) + 1)
            seen.add(addr)
    assert len(seen) == 64 * 32
    for j in range(0, 64, 2):
        for q in range(0, 64, 8):
            groups = {((8192 * (j >> 4) + 128 * t + 16 * ((((j & 15) >> 1)) ^ (t & 7))) // 16) % 8
                      for t in range(q, q + 8)}
            assert len(groups) == 8


def test_mana_remap_table():
    """csrc/mana_remap_tab.h (tools/mana_remap_gen.c): for every shift c, kManaRemap[c] is a
    permutation of the 243 thread groups, and the quarter-warp key collisions of the three
    bank-group maps (g, shift(g, c), neg(g, c), mod 8) total what the header states."""
    import os
    import re
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = open(os.path.join(root, "paper_2601_07824_b200", "csrc", "mana_remap_tab.h")).read()
    stated = int(re.search(r"collisions: total (\d+)", src).group(1))
    rows = [[int(x) for x in r.split(",")] for r in re.findall(r"\{([0-9,]+)\}", src)]
    assert len(rows) == 243

    def shift(g, c, neg):
        r, p = 0, 1
        for _ in range(5):
            gd, cd = g % 3, c % 3
            g, c = g // 3, c // 3
            r += ((6 - gd - cd) % 3 if neg else (gd - cd + 3) % 3) * p
            p *= 3
        return r

    total = 0
    for c, row in enumerate(rows):
        assert sorted(row) == list(range(243))
        for q in range(0, 243, 8):
            octet = row[q:q + 8]
            for f in (lambda g: g, lambda g: shift(g, c, 0), lambda g: shift(g, c, 1)):
                ks = [f(g) % 8 for g in octet]
                total += sum(ks.count(k) * (ks.count(k) - 1) // 2 for k in set(ks))
    assert total == stated
