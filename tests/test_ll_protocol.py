"""Model check of the tail step's TP allreduce exchange (the LL protocol), CPU only.

What runs on the GPU: every row-parallel projection (O, down) of a TP rank stores each output
element as ONE 8-byte {fp32 value, tag} pair into its slot of every peer's receive area
(`tps_linear_push_ll_cluster`, `tps_linear_push_ll`, `tps_reduce_push_ll`, `tps_gemv_push_ll`),
tag = epoch * n_phases + phase, n_phases = 2L + 1 (csrc/gemm_tcgen05.cu, csrc/gemv.cu); the
consumer (`tps_add_norm_ll`) polls every source's pair until its tag equals the expected one and uses the
value of that same load. Receive areas are double-buffered by phase parity
(GroupComm.ll_slot; a step has 2L LL phases -- O and down of every layer -- so parities keep
alternating across the step boundary); epochs start at 1 and the slots at 0
(GroupComm.__init__); a bucket's split count S (slots per source) may differ from the previous
step's.

The model: tp ranks each run `steps` steps of `phases` exchanges; a push is tp separate atomic
stores (one per destination, in order), a consume is tp atomic {value, tag} loads that each
succeed only on the expected tag. A rank's push of phase g+1 follows its consume of phase g in
program order (the next projection reads the normed activations). Every interleaving is
explored. Safety: every accepted value is the one the source pushed for that phase (no stale
or overwritten data). Liveness: no reachable state where some rank is stuck and none can move.

Results pinned below: the shipped protocol (2 parities, an even number of LL phases per step,
epochs from 1) is safe and live for tp 2-3 over changing split counts; one parity deadlocks (a
fast rank's phase g+1 push overwrites the phase-g pair a slow peer has not read yet); epochs starting at 0 accept a zeroed
slot as data (tag 0 == epoch 0, phase 0); an odd number of LL phases per step would put the
last phase of step e and the first of step e+1 on one parity and deadlock the same way.
"""

import pytest


def explore(tp: int, steps: int, phases: int, parities: int = 2, epoch0: int = 1, splits=(1,)):
    """(safe, live, states) over all interleavings. `splits[e % len(splits)]` = S of step e:
    a source's S pairs go to slots src*S .. src*S+S-1 of the parity's area."""
    smax = max(splits)
    nslot = tp * smax
    program = []  # per global phase g: (parity, tag, S)
    for e in range(steps):
        for p in range(phases):
            program.append((p % parities, (epoch0 + e) * (phases + 1) + p, splits[e % len(splits)]))
    G = len(program)

    def val(g, src, s):
        return 1000 * (g + 1) + 10 * src + s  # nonzero, unique per (phase, source, split)

    # per rank pc = (g, stage, i): stage 0 = pushing (i = next destination), 1 = consuming
    # (i = next source); g == G: done. mem[dst][parity][slot] = (tag, value)
    zero = tuple(tuple(tuple((0, 0) for _ in range(nslot)) for _ in range(parities)) for _ in range(tp))
    start = (tuple((0, 0, 0) for _ in range(tp)), zero)
    seen, stack = {start}, [start]
    safe = live = True
    while stack:
        pcs, mem = stack.pop()
        moved = False
        for r in range(tp):
            g, stage, i = pcs[r]
            if g == G:
                continue
            par, tag, S = program[g]
            if stage == 0:  # store this rank's S pairs into destination i
                m = [list(list(a) for a in d) for d in mem]
                for s in range(S):
                    m[i][par][r * S + s] = (tag, val(g, r, s))
                nmem = tuple(tuple(tuple(a) for a in d) for d in m)
                npc = (g, 0, i + 1) if i + 1 < tp else (g, 1, 0)
            else:  # load source i's S pairs from this rank's own area
                pairs = [mem[r][par][i * S + s] for s in range(S)]
                if any(t != tag for t, _ in pairs):
                    continue  # still polling
                if any(v != val(g, i, s) for s, (_, v) in enumerate(pairs)):
                    safe = False
                nmem = mem
                npc = (g, 1, i + 1) if i + 1 < tp else (g + 1, 0, 0)
            moved = True
            nxt = (pcs[:r] + (npc,) + pcs[r + 1:], nmem)
            if nxt not in seen:
                seen.add(nxt)
                stack.append(nxt)
        if not moved and any(pc[0] < G for pc in pcs):
            live = False
    return safe, live, len(seen)


@pytest.mark.parametrize("tp,steps,phases", [(2, 2, 2), (2, 3, 4), (3, 2, 2), (2, 2, 6)])
def test_shipped_protocol_is_safe_and_live(tp, steps, phases):
    safe, live, n = explore(tp, steps, phases)
    assert safe and live, (safe, live)
    assert n > 10


@pytest.mark.parametrize("splits", [(2, 1), (1, 2), (3, 1, 2)])
def test_changing_split_counts_between_steps(splits):
    """A bucket change between steps (cluster form S = 1 <-> per-partial form S > 1 <-> GEMV
    S = 1) leaves the previous step's pairs in the slots: their older tags never match."""
    safe, live, _ = explore(2, len(splits), 2, splits=splits)
    assert safe and live


def test_one_parity_deadlocks():
    """Why the receive areas alternate by phase parity: with one area, a rank that has consumed
    phase g pushes phase g+1 over the phase-g pair a slower peer has not loaded yet; the peer
    then polls for a tag that never comes back."""
    safe, live, _ = explore(2, 2, 2, parities=1)
    assert safe and not live


def test_epoch_zero_accepts_a_zeroed_slot():
    """Why epochs start at 1: at epoch 0 phase 0 expects tag 0, which every zeroed slot holds."""
    safe, live, _ = explore(2, 1, 2, epoch0=0)
    assert not safe


def test_odd_phase_count_per_step_deadlocks():
    """The executor's LL phases per step are 2L (phase 2l: O, 2l+1: down), so the parity
    alternates across steps; three phases per step would not."""
    assert explore(2, 2, 4)[1]
    safe, live, _ = explore(2, 2, 3)
    assert safe and not live
