"""Model check of the Switch Executor's device barrier (csrc/copy.cu barrier_kernel_v), CPU only.

Every interleaving of N ranks running K consecutive barriers is explored; a rank's arrival
signals its peers one at a time (as the kernel's loop does) and its pass is one atomic check.
Safety: no rank passes barrier k before every rank has reached barrier k (sent a signal).
Liveness: every interleaving ends with all ranks past barrier K.

Protocols: round 1's shared counter (each arrival adds 1 to every peer's counter; pass when the
own counter >= k (N-1)) and the epoch slots used now (arrival stores k into the rank's slot of
every peer; pass when every peer slot >= k).

`late_zero`: the signal memory of rank 0 is zero-filled by a stream-ordered kernel that may run
after peers have already signalled it -- what round 1's lazily created barrier counter did
(`torch.zeros` queued behind the rank's decode work, its address already shared with peers
whose devices were idle). The counter form then loses the early adds and hangs -- the
multi-process stall seen this round (counters stuck at 5, 4, 3 of 6 while peers had passed); the
slot form heals at the next epoch. The backend now also creates and shares the barrier memory
before the stage (B200Backend._init_barrier), so the zero-fill completes before any peer signal.
"""


def explore(n: int, k: int, protocol: str, late_zero: bool = False, duplicate: bool = False):
    """(safe, live) over all interleavings."""
    zero_row = 0 if protocol == "counter" else tuple([0] * n)
    zero = tuple([zero_row] * n)
    # pc per rank: (barrier b, step); step 0..n-2 = peers signalled so far, n-1 = waiting;
    # rank 0 starts at b = 0 (its memory's zero-fill still queued) when late_zero
    pcs0 = tuple(((0 if (late_zero and r == 0) else 1), 0) for r in range(n))
    start = (pcs0, zero, duplicate)
    seen, stack = {start}, [start]
    safe = live = True
    while stack:
        pcs, mem, dup = stack.pop()
        moved = False
        for r in range(n):
            b, step = pcs[r]
            if b > k:
                continue
            peers = [q for q in range(n) if q != r]
            if b == 0:  # the late zero-fill of rank 0's signal memory runs now
                nmem = (zero_row,) + mem[1:]
                npc, ndup = (1, 0), dup
            elif step < len(peers):  # signal the next peer
                q = peers[step]
                times = 2 if (dup and r == 1) else 1
                if protocol == "counter":
                    m = list(mem)
                    m[q] += times
                    nmem = tuple(m)
                else:
                    m = [list(row) for row in mem]
                    m[q][r] = max(m[q][r], b)
                    nmem = tuple(tuple(row) for row in m)
                npc = (b, step + 1)
                ndup = dup and r != 1
            else:  # waiting: pass when the condition holds
                ok = mem[r] >= b * (n - 1) if protocol == "counter" else \
                    all(mem[r][q] >= b for q in peers)
                if not ok:
                    continue
                if any(pcs[q][0] < b or (pcs[q][0] == b and pcs[q][1] == 0) for q in range(n)):
                    safe = False
                nmem, npc, ndup = mem, (b + 1, 0), dup
            moved = True
            st = (pcs[:r] + (npc,) + pcs[r + 1:], nmem, ndup)
            if st not in seen:
                seen.add(st)
                stack.append(st)
        if not moved and any(pc[0] <= k for pc in pcs):
            live = False
    return safe, live


def test_both_barrier_protocols_are_safe_and_live():
    for n, k in ((2, 3), (3, 3), (4, 2)):
        for proto in ("counter", "slots"):
            assert explore(n, k, proto) == (True, True), (proto, n, k)


def test_late_zero_fill_hangs_the_counter_barrier_not_the_slots():
    for n, k in ((3, 2), (4, 2)):
        assert explore(n, k, "counter", late_zero=True)[1] is False, n  # an early add is wiped: stuck
        assert explore(n, k, "slots", late_zero=True) == (True, True), n  # healed by the next epoch


def test_only_epoch_slots_tolerate_a_duplicated_signal():
    assert explore(3, 2, "slots", duplicate=True) == (True, True)
    assert explore(3, 2, "counter", duplicate=True)[0] is False
