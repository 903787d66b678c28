"""Model check of the Switch Executor's device barrier (csrc/copy.cu barrier_kernel_v), CPU only.

Every interleaving of N ranks running K consecutive barriers is explored; a rank's arrival
signals its peers one at a time (as the kernel's loop does) and its pass is one atomic check.
Safety: no rank passes barrier k before every rank has reached barrier k (started signalling). Liveness: every
interleaving ends with all ranks past barrier K.

Both protocols are checked: round 1's shared counter (each arrival adds 1 to every peer's
counter; pass when the own counter >= k (N-1)) and the epoch slots used now (arrival stores k
into the rank's slot of every peer; pass when every peer slot >= k). Both are safe and live in
isolation -- a rank can only run ahead to barrier k+1 after every rank arrived at k -- so the
multi-process hang seen with the counter form (counters stuck below target while peers had
passed: adds that never reached the waiting rank) was not a protocol race; see DESIGN section 6.
The slot form additionally tolerates a duplicated or replayed signal (a store of the same epoch
is idempotent, a duplicated add is not), which the counter form cannot.
"""


def explore(n: int, k: int, protocol: str, duplicate: bool = False):
    """(safe, live) over all interleavings; `duplicate`: one rank's first signal is delivered twice."""
    zero = tuple([0] * n) if protocol == "counter" else tuple(tuple([0] * n) for _ in range(n))
    # pc per rank: (barrier b, step) with step 0..n-1 = peers signalled so far, n = waiting
    start = (tuple((1, 0) for _ in range(n)), zero, duplicate)
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
            if step < len(peers):  # signal the next peer
                q = peers[step]
                times = 2 if (dup and r == 0) else 1
                if protocol == "counter":
                    m = list(mem)
                    m[q] += times
                    nmem = tuple(m)
                else:
                    m = [list(row) for row in mem]
                    m[q][r] = max(m[q][r], b)
                    nmem = tuple(tuple(row) for row in m)
                npc = (b, step + 1)
                ndup = dup and r != 0
            else:  # waiting: pass when the condition holds
                ok = mem[r] >= b * (n - 1) if protocol == "counter" else \
                    all(mem[r][q] >= b for q in peers)
                if not ok:
                    continue
                if any(pcs[q][0] < b or (pcs[q][0] == b and pcs[q][1] == 0) for q in range(n)):
                    safe = False  # some rank has not reached barrier b (not a single signal sent)
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


def test_only_epoch_slots_tolerate_a_duplicated_signal():
    assert explore(3, 2, "slots", duplicate=True) == (True, True)
    safe, _ = explore(3, 2, "counter", duplicate=True)
    assert not safe  # one extra add releases a rank before the last one arrives
