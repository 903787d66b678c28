"""Global Coordinator on B200: the reference's generation-stage loop driving real execution.

`GlobalCoordinator.run()` runs tpshift's loop (engine._run_node: lock-step
rounds, completions, Algorithm 1 evaluations, committed switches) with the
B200 backend behind its two seams:

* decode seam: each local DP group's Infer Executor replays its CUDA graph
  for the block's n rounds; a CUDA event is recorded after every round;
* switch seam: the Switch Executor plans and executes the weight / KV /
  history pulls into the new layout between two device barriers, and the
  groups resume on the new layout (graphs captured for its buckets).

The host never waits for the GPU: stop points are per-request lengths known
on the host and Algorithm 1 needs no device data, so the coordinator runs
ahead and each decision (and any switch planning / graph capture) overlaps
queued GPU work. After the stage, the recorded events become per-round
latencies and the *same* engine loop is replayed with them (RecordedBackend),
producing a SimReport whose clocks are measured B200 time.

One process per GPU runs the loop SPMD (identical decisions everywhere, no
control-plane messages except the switch-time handle/placement exchange); a
virtual world runs all ranks in one process on one device.
"""

from __future__ import annotations

import gc
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .cache_manager import CacheManager, World
from .engine import GroupState, NodeState, ScenarioSpec, SimReport, run
from .executor import GroupRunner, InferExecutor
from .group import RankState, admit, h2d, n_phases
from .kvcache import KVPool, SlotTable, pages_for
from .models import DecoderGeometry, rank_shard
from .shards import RankWeights
from .switch_executor import (KVSource, KVTarget, Layout, cached_weight_pulls, check, kv_move_bytes, nvlink_bytes,
                              pack_kv_moves, plan_history_pulls, plan_kv_moves, to_items, verify_kv_moves)
from .switchcost import MIGRATE, RECOMPUTE, SwitchCostBreakdown
from .errors import PlanVerificationError
from .workload import as_int64, sampler_seed


PREFILL_ROWS = 512  # (sample, prompt position) rows per chunked-prefill step


def _event(stream) -> torch.cuda.Event:
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


@dataclass
class GroupTimeline:
    rank: int
    prefill_end: object = None
    rounds: list = field(default_factory=list)


@dataclass
class SwitchTiming:
    # rank -> [arrive, released, weights_done, kv_done, resumed] events: arrive = the rank reached
    # the opening device barrier, released = every rank had (barrier passed), resumed = the
    # closing barrier passed (decode on the new layout may start)
    marks: dict
    nvlink_bytes: int    # summed over this process's ranks (bytes pulled from other ranks)
    local_bytes: int     # summed over this process's ranks (copies inside a rank's own HBM)
    kv_bytes: int
    weight_bytes: int
    host_plan_s: float
    host_capture_s: float
    state_method: str = MIGRATE
    host_build_s: float = 0.0
    per_rank: dict = field(default_factory=dict)  # rank -> {"nvlink": bytes, "local": bytes}
    host_s: float = 0.0  # host seconds from the switch call to the last launch


class B200Backend:
    """Real execution behind the engine's seams (prefill, decode blocks, switches)."""

    exact_pool_cost = False

    def __init__(self, spec: ScenarioSpec, geom: DecoderGeometry, world: World, seed: int = 0,
                 use_graphs: bool = True, copy_mode: int = 1, prompts: np.ndarray | None = None,
                 host_io: bool = False, state_method: str | None = None, temperature: float = 0.0,
                 prebuild: bool | None = None, mem_headroom_gb: float = 6.0, alias_replicas: bool = False):
        self.spec, self.geom, self.world = spec, geom, world
        self.alias_replicas = alias_replicas and not world.distributed
        self._alias: dict = {}
        self.temperature = temperature  # 0: greedy; > 0: Gumbel-max with per-sample Philox keys
        # None: each switch handles KV state as Algorithm 1 priced it (migrate or
        # recompute); MIGRATE / RECOMPUTE force one method (measurement, tests)
        self.state_method = state_method
        self.use_graphs = use_graphs
        self.copy_mode = copy_mode
        self.host_io = host_io
        self.max_len = spec.prompt_len + spec.l_max
        self.layout = Layout(spec.initial_tp, world.gpus)
        per_node = spec.global_batch // spec.cluster.num_nodes
        self.max_batch = max(1, -(-per_node // self.layout.dp))
        if prompts is None:
            prompts = np.random.default_rng(spec.seed).integers(0, geom.vocab, (spec.global_batch, spec.prompt_len),
                                                                dtype=np.int32)
        host = torch.from_numpy(np.ascontiguousarray(prompts, dtype=np.int32))
        dev0 = world.devices[world.local_ranks[0]]
        self.prompts_host = host.pin_memory()
        # device-timed runs start with the prompts already resident in HBM; host_io
        # runs (the e2e measurement) copy each prompt from pinned host memory
        self.prompts_dev = self.prompts_host.to(dev0)
        self.out_host = torch.zeros((spec.global_batch, spec.l_max), dtype=torch.int32).pin_memory()
        # receive slots must hold any group's batch after merges (size them for the whole
        # node) and a chunked-prefill step's rows
        self.cache = CacheManager(world, max(per_node, PREFILL_ROWS + self.max_batch), geom.hidden,
                                  n_phases(geom))
        self.epoch = 0
        self.ranks: dict[int, RankState] = {}
        self.runners: dict[int, GroupRunner] = {}
        self.slot_of: dict[int, int] = {}
        self.timeline: dict[tuple[int, int], GroupTimeline] = {}
        self.switches: list[SwitchTiming] = []
        self.kernels_launched = 0
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.retired_here: list[int] = []  # samples whose tokens this process wrote to out_host
        self.copy_events: list | None = None  # (start event, bytes, end event) per copy launch (probes)
        self.start: dict[int, torch.cuda.Event] = {}
        self._keep: list = []
        self._barrier_epoch = 0
        self._bar = None
        # built layouts (ranks + runners with their captured graphs) per TP degree, kept for the
        # life of the backend like the communicator pool: a later switch to the same degree,
        # or the next stage, reuses the buffers and graphs instead of allocating and capturing
        self._layouts: dict[int, dict] = {}
        self._witems: dict = {}  # device copy-item tables per (transition, rank, arena pointers)
        self._shared: dict = {}  # peer pointers / pool geometry of a built layout (per tp + buffers)
        self._items_ws: dict[int, torch.Tensor] = {}  # per rank: KV copy items expanded on the device
        self._bad: dict[int, torch.Tensor] = {}       # per rank: out-of-range pages seen by the expander
        self._staging: dict[int, tuple] = {}          # per rank: pinned + device staging area of a switch
        self.mem_headroom = int(mem_headroom_gb * 2 ** 30)
        self.ranks, self.runners = self._build_layout(self.layout, weights_seed=seed)
        self._layouts[self.layout.tp] = {"ranks": self.ranks, "runners": self.runners, "cap": self.max_batch}
        self.preplan_s = self.preplan()
        # every candidate layout is built (buffers, executors, communicators; graphs are
        # captured with the initial layout's) before the stage, within an HBM budget, so a
        # switch only moves bytes (recapture is the switch's largest fixed cost)
        self._init_barrier()
        if prebuild is None:
            prebuild = os.environ.get("TPS_PREBUILD", "1") == "1"
        # a static stage (or a disabled controller) never switches: nothing to prepare
        prebuild = prebuild and spec.mode != "static" and spec.controller.enabled
        self.prebuilt: dict[int, int] = self.prebuild() if prebuild else {}

    def preplan(self) -> float:
        """Plan (and verify) this process's weight pulls for every switch between candidate
        degrees before the stage starts, so a switch's critical path only plans its KV moves
        (Qwen2.5-7B TP1 -> TP2: ~0.15 s of host planning per rank moved off the switch). Plans
        are memoised per (geometry, layouts, rank) for the process."""
        t0 = time.perf_counter()
        tps = sorted({self.spec.initial_tp} | {t for t in self.spec.controller.tp_list if self.world.gpus % t == 0})
        if self.spec.mode == "static" or not self.spec.controller.enabled:
            tps = []
        for a in tps:
            for b in tps:
                if a != b:
                    for r in self.world.local_ranks:
                        cached_weight_pulls(self.geom, Layout(a, self.world.gpus), Layout(b, self.world.gpus), r)
        return time.perf_counter() - t0

    def layout_bytes(self, lay: Layout, slots: int) -> int:
        """HBM the local ranks of `lay` need with `slots` sample slots per group: weight shards +
        KV pools + slot tables + decode/prefill activations (estimate of the executor's
        workspaces)."""
        nloc = len(self.world.local_ranks)
        w, rest = self._rank_bytes(lay, slots)
        nw = min(nloc, lay.tp) if self.alias_replicas else nloc
        return nw * w + nloc * rest

    def _rank_bytes(self, lay: Layout, slots: int) -> tuple[int, int]:
        from .shards import arena_layout
        g = self.geom
        sh = rank_shard(g, lay.tp, 0)
        w = arena_layout(g, sh).total_bytes
        pages = slots * pages_for(self.max_len)
        kv = g.num_layers * 2 * pages * sh.n_kv * 64 * g.head_dim * 2
        tables = slots * (self.max_len * 4 + pages_for(self.max_len) * 4 + 32)
        rows = max(slots, PREFILL_ROWS + slots)
        act = rows * (g.hidden * 6 + (g.ffn // lay.tp) * 2 + g.n_q * g.head_dim * 4) + (g.vocab // lay.tp) * 64 * 4
        return int(w), int(kv + tables + 4 * act + (64 << 20))

    def prebuild(self) -> dict[int, int]:
        """Build every other candidate degree's layout now (slot capacity per group: the whole
        node's batch over its dp, reduced to fit the HBM left after a headroom): {tp: slots}."""
        out = {}
        per_node = self.spec.global_batch // self.spec.cluster.num_nodes
        for tp in self.spec.controller.tp_list:
            if tp == self.layout.tp or self.world.gpus % tp or tp in self._layouts:
                continue
            lay = Layout(tp, self.world.gpus)
            want = max(1, -(-per_node // lay.dp))
            dev = self.world.devices[self.world.local_ranks[0]]
            free = torch.cuda.mem_get_info(dev)[0] + torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
            if self.world.distributed and os.environ.get("TPS_SHARE_DEVICE") == "1":
                free //= self.world.gpus  # every rank's process allocates on this one device
            cap = want  # (a virtual world holds every rank on one device)
            while cap > 0 and self.layout_bytes(lay, cap) > free - self.mem_headroom:
                cap = cap * 3 // 4 if cap > 4 else cap - 1
            # one capacity on every process (each builds, shares and rebuilds the same layouts:
            # the peer-pointer exchanges are collectives)
            cap = min(self.world.allgather(cap))
            if cap <= 0:
                continue  # built at the switch instead (host time on the critical path)
            ranks, runners = self._build_layout(lay, weights_seed=None,
                                                per_group={g: cap for g in self.local_groups(lay)})
            self._layouts[tp] = {"ranks": ranks, "runners": runners, "cap": cap}
            out[tp] = cap
        return out

    # ------------------------------------------------------------- layout ---
    def stream(self, r: int):
        return torch.cuda.current_stream(self.world.devices[r])

    def local_groups(self, lay: Layout | None = None) -> list[int]:
        lay = lay or self.layout
        return sorted({lay.group_of(r) for r in self.world.local_ranks})

    def _build_layout(self, lay: Layout, weights_seed: int | None, per_group: dict[int, int] | None = None,
                      prefill: bool = True):
        """(ranks, runners) of layout `lay` on this process (new buffers)."""
        comms = self.cache.get(lay.tp)
        ranks = {}
        for r in self.world.local_ranks:
            n = self.max_batch if per_group is None else per_group.get(lay.group_of(r), 0)
            ranks[r] = self._make_rank(lay, r, max(1, n), weights_seed, comms[r], prefill)
        runners = {}
        for g in self.local_groups(lay):
            exs = [ranks[r].executor for r in lay.ranks_of_group(g) if r in ranks]
            runners[g] = GroupRunner(exs, use_graphs=self.use_graphs)
        return ranks, runners

    def _make_rank(self, lay: Layout, r: int, slots: int, weights_seed, comm, prefill: bool) -> RankState:
        dev = self.world.devices[r]
        nat.init_device(dev.index or 0)
        sh = rank_shard(self.geom, lay.tp, lay.tp_rank(r))
        key = (lay.tp, lay.tp_rank(r))
        if self.alias_replicas and key in self._alias:
            # microbench option (virtual world): DP replicas of one TP rank hold identical canonical
            # shards, so they may share one arena (reads are identical; pulls write equal bytes)
            w = self._alias[key]
        else:
            w = RankWeights(self.geom, sh, dev)
            if weights_seed is not None:
                w.fill_random(weights_seed)
            if self.alias_replicas:
                self._alias[key] = w
        kv = KVPool(self.geom.num_layers, sh.n_kv, self.geom.head_dim, slots * pages_for(self.max_len), dev)
        st = SlotTable(slots, self.max_len, dev)
        pf = slots * max(1, PREFILL_ROWS // slots) if prefill else 0
        ex = InferExecutor(self.geom, sh, w, kv, st, slots, dev, comm=comm, prefill_rows=pf)
        ex.temperature = self.temperature
        return RankState(w, kv, st, ex, comm)

    def _use_layout(self, lay: Layout, per_group: dict[int, int] | None) -> bool:
        """Make `lay` current: reuse the cached ranks/runners of this TP degree when its slot
        capacity (one per layout, the same for every group) holds the largest group of the
        placement (slot tables and page pools reset), else build it (new buffers, weights
        filled by the switch's pulls) and cache it. The placement covers every group and is the
        same on every process, so every process rebuilds the same layouts. True if built."""
        need = max(1, self.max_batch) if per_group is None else max([1] + list(per_group.values()))
        c = self._layouts.get(lay.tp)
        if c is not None and c["cap"] >= need:
            for rs in c["ranks"].values():
                rs.slots.reset()
                rs.kv.reset()
            self.ranks, self.runners = c["ranks"], c["runners"]
            return False
        cap = max(need, c["cap"] if c else 0)
        if c is not None and lay.tp != self.spec.initial_tp:
            # grown: the smaller cached layout of this degree is dropped first (bounded HBM:
            # at most one layout per candidate degree is ever held)
            del self._layouts[lay.tp]
            c = None
            self._shared = {k: v for k, v in self._shared.items() if k[0] != lay.tp}
            self._witems = {k: v for k, v in self._witems.items() if lay not in (k[0], k[1])}
            gc.collect()
        self.ranks, self.runners = self._build_layout(lay, weights_seed=None,
                                                      per_group={g: cap for g in self.local_groups(lay)})
        self._layouts[lay.tp] = {"ranks": self.ranks, "runners": self.runners, "cap": cap}
        return True

    def reset(self, seed: int) -> None:
        """Return to the initial layout with no samples (between repeated stages)."""
        init = Layout(self.spec.initial_tp, self.world.gpus)
        rebuild = bool(self.epoch) or self.layout != init
        self.epoch = 0
        if rebuild:
            # the cached initial layout holds the canonical shards (a switch back to it pulls
            # bit-identical bytes), so only its slot tables and pages are reset
            self.layout = init
            self._use_layout(init, None)
            self.capture_all()
        self.timeline = {}
        self.switches = []
        self.slot_of = {}
        self.retired_here = []
        self.kernels_launched = 0
        self.h2d_bytes = self.d2h_bytes = 0
        self.start = {}
        self._keep.clear()

    def capture_all(self, every_layout: bool = False) -> float:
        """Capture the decode graph of every bucket of every local group of the current layout
        (or of every built layout): host seconds. Already-captured buckets are skipped."""
        t0 = time.perf_counter()
        if self.use_graphs:
            runners = [ru for c in self._layouts.values() for ru in c["runners"].values()] if every_layout \
                else list(self.runners.values())
            for runner in runners:
                for b in runner.ex[0].buckets():
                    runner.capture(b)
                R = runner.ex[0].prefill_rows
                if R and ("prefill", R) not in runner.graphs:
                    runner._capture_key(("prefill", R), lambda st, rr=runner, n=R: rr._issue_prefill(n, st))
        return time.perf_counter() - t0

    def group_ranks(self, g: int) -> list[RankState]:
        return [self.ranks[r] for r in self.layout.ranks_of_group(g) if r in self.ranks]

    def first_local(self, g: int) -> int:
        return next(r for r in self.layout.ranks_of_group(g) if r in self.ranks)

    # ---------------------------------------------------------------- seams ---
    def begin(self) -> None:
        """Stage start event on every local device, after an all-rank barrier."""
        for r in self.world.local_ranks:
            torch.cuda.synchronize(self.world.devices[r])
        self.world.barrier()
        for r in self.world.local_ranks:
            self.start[r] = _event(self.stream(r))

    def prefill(self, node: NodeState, g: int, members, tp: int) -> float:
        if g not in self.runners:
            return 0.0
        grp = self.group_ranks(g)
        slots = []
        for s in members:
            if not self.host_io:
                prompt = self.prompts_dev[s.id]
            else:
                prompt = self.prompts_host[s.id].to(grp[0].slots.device, non_blocking=True)
                self.h2d_bytes += prompt.numel() * 4
            slots.append(admit(grp, s.id, prompt, max_ctx=self.max_len, seed=sampler_seed(self.spec.seed, s.id)))
            self.slot_of[s.id] = slots[-1]
        runner = self.runners[g]
        r = self.first_local(g)
        tl = self.timeline.setdefault((self.epoch, g), GroupTimeline(rank=r))
        # chunked prefill through the decode kernels: prompt positions 0..L-2 of every
        # sample, several positions per launch; position L-1 is decode round 1
        self.kernels_launched += runner.prefill(slots, self.spec.prompt_len)
        tl.prefill_end = _event(self.stream(r))
        return 0.0

    def decode_block(self, node: NodeState, group: GroupState, n: int) -> np.ndarray:
        g = group.index
        if g in self.runners:
            runner = self.runners[g]
            slots = [self.slot_of[s.id] for s in group.samples]
            B = runner.ex[0].bucket(len(slots))
            runner.set_rows(B, slots)
            r = self.first_local(g)
            tl = self.timeline.setdefault((self.epoch, g), GroupTimeline(rank=r))
            if self.use_graphs and B not in runner.graphs:
                runner.capture(B)
            st = self.stream(r)
            for _ in range(n):
                runner.step(B, 1)
                tl.rounds.append(_event(st))
            self.kernels_launched += n * runner.kernels_per_step(B)
        return np.zeros(n)

    def retire(self, node: NodeState, group: GroupState, done) -> None:
        """Stream finished samples' generated tokens to the host; free their slots/pages."""
        g = group.index
        if g not in self.runners:
            return
        grp = self.group_ranks(g)
        lead = self.layout.ranks_of_group(g)[0] in self.ranks  # TP rank 0 writes the output
        lo = self.spec.prompt_len
        for s in done:
            slot = self.slot_of.pop(s.id)
            if lead:
                n = min(s.target_response_len, self.spec.l_max)
                self.out_host[s.id, :n].copy_(grp[0].slots.history[slot, lo:lo + n], non_blocking=True)
                self.retired_here.append(s.id)
                self.d2h_bytes += 4 * n
            for r in grp:
                r.kv.release(r.slots.pages.get(slot, []))
                r.slots.release(slot)

    def planned_state_method(self, decision, naive_mode: bool) -> str:
        return self.state_method or decision.breakdown.state_method

    def realize_switch(self, node: NodeState, decision, statuses, merged, naive_mode: bool):
        quote = decision.breakdown
        method = self.planned_state_method(decision, naive_mode)
        self._execute_switch(decision.target.tp, merged, recompute=method == RECOMPUTE)
        # host-side placeholder with the realised method; the reported clocks come from
        # the recorded events (RecordedBackend)
        return SwitchCostBreakdown.build(quote.t_state_handling, method, quote.t_weight_reshard,
                                         quote.t_graph_recapture, quote.t_comm_group_init, quote.t_fixed_control)

    def switch_record_extra(self, node: NodeState) -> dict:
        t = self.switches[-1]
        return {"nvlink_bytes_local_ranks": t.nvlink_bytes, "local_copy_bytes": t.local_bytes,
                "host_plan_s": t.host_plan_s, "host_capture_s": t.host_capture_s}

    def after_switch(self, node: NodeState) -> None:
        pass

    def finish(self, node: NodeState) -> None:
        pass

    # -------------------------------------------------------------- switch ---
    def _execute_switch(self, tp_new: int, merged: list[list], recompute: bool = False) -> None:
        """Weights are always pulled (canonical slices of the new layout). KV state is
        either migrated (page pulls, tpshift/reshard.py:113-151) or recomputed: only
        the token histories move, and every sample's KV is rebuilt by a chunked
        prefill over its prompt + generated tokens under the new TP
        (tpshift/switchcost.py:203-219, engine.py:187-203).

        Host work on the critical path is O(samples): the target layout, its graphs and the
        weight copy-item tables (device-resident) are prepared before the stage; KV pages
        are described by one move per (sample, kv-head run) that the device expands from
        the source and target page tables (tps_kv_move_items)."""
        th = time.perf_counter()
        old, new = self.layout, Layout(tp_new, self.world.gpus)
        old_ranks = self.ranks
        # where every live sample sits now: {id: (old group, slot)}, gathered across processes
        here = {}
        for g in self.local_groups(old):
            lead = self.ranks[self.first_local(g)]
            for slot, sid in lead.slots.sample_of.items():
                here[sid] = (g, slot)
        where = {}
        for part in self.world.allgather(here):
            where.update(part)
        src = self._shared_layout(old, old_ranks)
        marks = {r: [_event(self.stream(r))] for r in self.world.local_ranks}
        self._device_barrier()  # every rank has finished decoding on the old layout
        for r in self.world.local_ranks:
            marks[r].append(_event(self.stream(r)))
        tb = time.perf_counter()
        self.epoch += 1
        self.layout = new
        self._use_layout(new, {g: len(m) for g, m in enumerate(merged)})
        t_build = time.perf_counter() - tb
        stats = dict(nv=0, loc=0, kv=0, w=0)
        per_rank = {}
        t_plan = 0.0
        L = self.geom.num_layers
        for r in self.world.local_ranks:
            rs, st = self.ranks[r], self.stream(r)
            t0 = time.perf_counter()
            w_parts, (wnv, wloc) = self._weight_items(old, new, r, src, rs)
            mine = merged[new.group_of(r)] if new.group_of(r) < len(merged) else []
            n = len(mine)
            slot_list, pages_of = [], []
            for s in mine:
                slot = rs.slots.alloc(s.id)
                pages = rs.kv.alloc(pages_for(self.max_len))
                rs.slots.pages[slot] = pages
                slot_list.append(slot)
                pages_of.append(pages)
            ids = np.fromiter((s.id for s in mine), dtype=np.int64, count=n)
            ctx = np.fromiter((s.context_len for s in mine), dtype=np.int64, count=n)
            plen = np.fromiter((s.prompt_len for s in mine), dtype=np.int64, count=n)
            og = np.fromiter((where[int(i)][0] for i in ids), dtype=np.int64, count=n)
            oslot = np.fromiter((where[int(i)][1] for i in ids), dtype=np.int64, count=n)
            nslot = np.asarray(slot_list, dtype=np.int64)
            kv_nv = kv_loc = 0
            n_items, hist = 0, np.zeros((0, 4), dtype=np.int64)
            if n:
                P = rs.slots.max_pages
                seeds = np.fromiter((as_int64(sampler_seed(self.spec.seed, int(i))) for i in ids), dtype=np.int64,
                                    count=n)
                if not recompute:
                    moves = plan_kv_moves(self.geom, old, new, r, og, oslot, nslot, ctx - 1)
                    check(verify_kv_moves(moves, rs.kv.n_kv, rs.slots.num_slots, nslot[ctx - 1 > 0]), "kv move plan")
                    kv_nv, kv_loc = kv_move_bytes(self.geom, moves, r)
                    packed, n_items = pack_kv_moves(self.geom, moves, src, rs.slots.page_table.data_ptr(),
                                                    rs.slots.page_table.stride(0) * 4)
                else:
                    packed = np.zeros(0, dtype=np.uint8)
                srcs = [KVSource(old_group=int(a), slot=int(b), pages=()) for a, b in zip(og, oslot)]
                tgts = [KVTarget(slot=int(x), pages=()) for x in nslot]
                hp = plan_history_pulls(old, r, srcs, tgts, ctx.tolist(), self.max_len, self.max_len)
                hist = to_items(hp, {k: v["hist"] for k, v in src.items()}, rs.slots.history.data_ptr())
                a, b = nvlink_bytes(hp, r)
                kv_nv, kv_loc = kv_nv + a, kv_loc + b
                # one pinned staging area, one host->device copy: per-slot state (page-table
                # rows, next position -- KV holds positions < pos --, prompt length, sampler
                # key), slot indices, KV moves, history copy items
                blob = np.zeros((n, P + 4), dtype=np.int32)
                blob[:, :P] = np.asarray(pages_of, dtype=np.int32)
                blob[:, P] = ctx - 1
                blob[:, P + 1] = plen
                blob[:, P + 2:P + 4] = seeds.view(np.int32).reshape(n, 2)
                dev = self._stage(r, [blob, nslot, packed.view(np.uint8) if len(packed) else packed,
                                      np.ascontiguousarray(hist, dtype=np.int64)], st)
                dblob = dev[0].view(torch.int32).view(n, P + 4)
                idx = dev[1].view(torch.int64)
                rs.slots.page_table.index_copy_(0, idx, dblob[:, :P])
                rs.slots.pos.index_copy_(0, idx, dblob[:, P])
                rs.executor.prompt_len.index_copy_(0, idx, dblob[:, P + 1])
                rs.slots.seed.index_copy_(0, idx, dblob[:, P + 2:P + 4].contiguous().view(torch.int64).view(-1))
                dmoves, dhist = dev[2], dev[3]
            t_plan += time.perf_counter() - t0
            for dev, cnt, mode, nb in w_parts:
                self._launch_items(dev, cnt, mode, st, nb)
            marks[r].append(_event(st))
            if n_items:
                ws = self._item_ws(r, n_items)
                nat.check(nat.lib().tps_kv_move_items(dmoves.data_ptr(), len(packed), n_items, rs.kv.buf.data_ptr(),
                                                      rs.kv.num_pages, rs.kv.n_kv, rs.kv.chunk_bytes, ws.data_ptr(),
                                                      self._bad[r].data_ptr(), st.cuda_stream), "tps_kv_move_items")
                self.kernels_launched += 1
                self._launch_items(ws, n_items, self.copy_mode, st, kv_nv + kv_loc - int(hist[:, 2].sum()))
            if len(hist):
                # history rows: 4-B multiples, through the LSU engine (no per-switch re-staging)
                self._launch_items(dhist, len(hist), 0, st, int(hist[:, 2].sum()))
            if not recompute:
                marks[r].append(_event(st))
            stats["nv"] += wnv + kv_nv
            stats["loc"] += wloc + kv_loc
            stats["w"] += wnv + wloc
            stats["kv"] += kv_nv + kv_loc
            per_rank[r] = {"nvlink": wnv + kv_nv, "local": wloc + kv_loc}
            for s, slot in zip(mine, slot_list):
                self.slot_of[s.id] = slot
        if recompute:
            # rebuild each new group's KV from the pulled histories: positions < pos
            for g in self.local_groups(new):
                mine = merged[g] if g < len(merged) else []
                if mine:
                    self.kernels_launched += self.runners[g].prefill(
                        [self.slot_of[s.id] for s in mine], [s.context_len - 1 for s in mine])
            for r in self.world.local_ranks:
                marks[r].append(_event(self.stream(r)))
        self._device_barrier()  # every rank has finished pulling: old buffers may be released
        for r in self.world.local_ranks:
            marks[r].append(_event(self.stream(r)))
        host_s = time.perf_counter() - th
        tc = time.perf_counter()
        self.capture_all()  # (a no-op for prebuilt layouts: their graphs exist)
        self.switches.append(SwitchTiming(marks=marks, nvlink_bytes=stats["nv"], local_bytes=stats["loc"],
                                          kv_bytes=stats["kv"], weight_bytes=stats["w"], host_plan_s=t_plan,
                                          host_capture_s=time.perf_counter() - tc,
                                          state_method=RECOMPUTE if recompute else MIGRATE,
                                          host_build_s=t_build, per_rank=per_rank, host_s=host_s))
        self._keep.append(old_ranks)  # (cached layouts are reused, never freed mid-stage)

    def _shared_layout(self, lay: Layout, ranks: dict) -> dict[int, dict]:
        """Pointers (valid in this process) to every rank's weight arena, KV pool, token history
        and page table under `lay`, plus its pool geometry: exchanged once per built layout."""
        key = (lay.tp, tuple(sorted((r, rs.kv.buf.data_ptr()) for r, rs in ranks.items())))
        out = self._shared.get(key)
        if out is None:
            ptrs = self.world.share({r: {"w": rs.weights.arena, "kv": rs.kv.buf, "hist": rs.slots.history,
                                         "pt": rs.slots.page_table} for r, rs in ranks.items()})
            geo = {}
            for part in self.world.allgather({r: (rs.kv.num_pages, rs.kv.n_kv) for r, rs in ranks.items()}):
                geo.update(part)
            out = {r: dict(ptrs[r], np=geo[r][0], nkv=geo[r][1]) for r in ptrs}
            self._shared[key] = out
        return out

    def _weight_items(self, old: Layout, new: Layout, r: int, src: dict, rs: RankState):
        """Device-resident copy-item tables of rank r's weight pulls for old -> new (memoised per
        transition and buffer set; arena pointers of cached layouts do not change) and the
        (peer, local) byte counts."""
        w_src = tuple(sorted((k, v["w"]) for k, v in src.items()))
        ikey = (old, new, r, rs.weights.arena.data_ptr(), w_src)
        hit = self._witems.get(ikey)
        if hit is None:
            wp = cached_weight_pulls(self.geom, old, new, r)  # verified once when first planned
            items = to_items(wp, dict(w_src), rs.weights.arena.data_ptr())
            hit = self._witems[ikey] = (self._stage_items(items, rs.slots.device), nvlink_bytes(wp, r))
        return hit

    def prepare_switch_items(self) -> float:
        """Stage the weight copy-item tables of every switch between built layouts -- the initial
        one and every prebuilt candidate, both directions -- before the stage (host seconds), so
        a multi-stage run (TP1 -> 2 -> 4 -> 8 and back) plans no weight pull at a switch."""
        t0 = time.perf_counter()
        if self.spec.initial_tp not in self._layouts:
            return 0.0
        built = [self.spec.initial_tp] + sorted(self.prebuilt)
        shared = {tp: self._shared_layout(Layout(tp, self.world.gpus), self._layouts[tp]["ranks"]) for tp in built}
        for a in built:
            for b in built:
                if a == b:
                    continue
                old, new = Layout(a, self.world.gpus), Layout(b, self.world.gpus)
                for r in self.world.local_ranks:
                    self._weight_items(old, new, r, shared[a], self._layouts[b]["ranks"][r])
        if self.prebuilt:
            self._warm_switch_path()
        return time.perf_counter() - t0

    def _warm_switch_path(self) -> None:
        """Load (lazy CUDA module loading) and allocate what a switch launches before the stage:
        staging areas, the slot-state scatter kernels, the KV-move expander and both copy engines
        (a cold first switch paid ~17 ms of host time for them)."""
        for r in self.world.local_ranks:
            st = self.stream(r)
            dev = self.world.devices[r]
            one = np.zeros(1, dtype=np.int64)
            v = self._stage(r, [np.zeros((1, 4), dtype=np.int32), one], st)
            idx = v[1].view(torch.int64)
            for c in self._layouts.values():  # (rewrites slot 0 with its own values)
                rs = c["ranks"][r]
                rs.slots.pos.index_copy_(0, idx, rs.slots.pos[:1].clone())
                rs.slots.page_table.index_copy_(0, idx, rs.slots.page_table[:1].clone())
                rs.slots.seed.index_copy_(0, idx, rs.slots.seed[:1].clone())
            ws = self._item_ws(r, 1)
            zero = torch.zeros(64, dtype=torch.int32, device=dev)
            scratch = torch.zeros(1 << 16, dtype=torch.uint8, device=dev)
            from .switch_executor import KV_MOVE_DTYPE
            mv = np.zeros(1, dtype=KV_MOVE_DTYPE)
            mv["src_kv"], mv["src_pages"], mv["dst_pages"] = scratch.data_ptr(), zero.data_ptr(), zero.data_ptr()
            mv["src_num_pages"] = mv["src_nkv"] = mv["n_heads"] = mv["n_pages"] = 1
            dm = torch.from_numpy(mv.view(np.uint8).copy()).to(dev)
            nat.check(nat.lib().tps_kv_move_items(dm.data_ptr(), 1, 2, scratch.data_ptr(), 1, 1, 1 << 14,
                                                  ws.data_ptr(), None, st.cuda_stream), "tps_kv_move_items")
            items = torch.tensor([[scratch.data_ptr(), scratch.data_ptr() + 32768, 16384, 0]], dtype=torch.int64,
                                 device=dev)
            for mode in (0, 1):
                nat.check(nat.lib().tps_copy_items(items.data_ptr(), 1, mode, 0, st.cuda_stream), "tps_copy_items")
            torch.cuda.synchronize(dev)

    def _stage_items(self, items: np.ndarray, device) -> list:
        """[(device item table, count, copy mode, bytes)]: 16-B aligned items go to the bulk-copy
        engine (mode 1), the rest to the LSU engine."""
        if len(items) == 0:
            return []
        items = np.ascontiguousarray(items, dtype=np.int64)
        parts = [(items, self.copy_mode)]
        if self.copy_mode == 1:
            ok = ((items[:, 0] | items[:, 1] | items[:, 2]) & 15) == 0
            parts = [(p, m) for p, m in ((items[ok], 1), (items[~ok], 0)) if len(p)]
        return [(torch.from_numpy(np.ascontiguousarray(p)).to(device), len(p), m, int(p[:, 2].sum()))
                for p, m in parts]

    def _stage(self, r: int, arrays: list[np.ndarray], st) -> list[torch.Tensor]:
        """Pack host arrays into this rank's pinned staging area (16-B aligned), copy them to the
        device in one transfer and return uint8 device views, one per array. The area is reused:
        the previous switch's transfer is waited for (long complete) before it is overwritten."""
        offs, o = [], 0
        for a in arrays:
            offs.append(o)
            o += (a.nbytes + 15) // 16 * 16
        host, devbuf, ev = self._staging.get(r, (None, None, None))
        if host is None or host.numel() < o:
            size = max(o, 2 << 20)
            host = torch.empty(size, dtype=torch.uint8).pin_memory()
            devbuf = torch.empty(size, dtype=torch.uint8, device=self.world.devices[r])
            ev = None
        if ev is not None:
            ev.synchronize()
        hn = host.numpy()
        for a, off in zip(arrays, offs):
            if a.nbytes:
                hn[off:off + a.nbytes] = np.ascontiguousarray(a).view(np.uint8).ravel()
        devbuf[:o].copy_(host[:o], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(st)
        self._staging[r] = (host, devbuf, ev)
        return [devbuf[off:off + a.nbytes] for a, off in zip(arrays, offs)]

    def _item_ws(self, r: int, n_items: int) -> torch.Tensor:
        ws = self._items_ws.get(r)
        if ws is None or ws.shape[0] < n_items:
            dev = self.world.devices[r]
            ws = self._items_ws[r] = torch.empty((max(n_items, 1 << 16), 4), dtype=torch.int64, device=dev)
        if r not in self._bad:
            self._bad[r] = torch.zeros(1, dtype=torch.int32, device=self.world.devices[r])
        return ws

    def _launch_items(self, dev: torch.Tensor, n: int, mode: int, st, nbytes: int = 0) -> None:
        if n == 0:
            return
        if self.copy_events is not None:
            self.copy_events.append((_event(st), int(nbytes)))
        nat.check(nat.lib().tps_copy_items(dev.data_ptr(), n, mode, 0, st.cuda_stream), "tps_copy_items")
        if self.copy_events is not None:
            self.copy_events[-1] += (_event(st),)
        self.kernels_launched += 1

    def _copy(self, items: np.ndarray, st) -> None:
        """Copy host-planned items (staged to the device, then executed)."""
        for dev, n, mode, nb in self._stage_items(items, st.device):
            self._launch_items(dev, n, mode, st, nb)
            self._keep.append(dev)

    def _init_barrier(self) -> None:
        """The device barrier's slot array, zeroed and exchanged before the stage: its zero-fill
        is stream-ordered, so created lazily at the first switch it could run after an idle
        peer had already signalled it and wipe the signal (tests/test_barrier_protocol.py)."""
        if not self.world.distributed or self._bar is not None:
            return
        r = self.world.local_ranks[0]
        mine = torch.zeros(self.world.gpus, dtype=torch.int64, device=self.world.devices[r])
        torch.cuda.synchronize(self.world.devices[r])  # zeroed before any peer can see the address
        ptrs = self.world.share({r: {"bar": mine}})
        self._bar = (mine, [ptrs[x]["bar"] + 8 * r for x in range(self.world.gpus) if x != r])

    def _device_barrier(self) -> None:
        """Node-wide device barrier (a virtual world is already ordered by its single stream):
        one epoch slot per source rank in every rank's slot array (tps_barrier)."""
        if not self.world.distributed:
            return
        r = self.world.local_ranks[0]
        self._init_barrier()
        mine, peers = self._bar
        self._barrier_epoch += 1
        nat.check(nat.lib().tps_barrier(nat.ptr_array(peers), len(peers), mine.data_ptr(), self.world.gpus, r,
                                        self._barrier_epoch, self.stream(r).cuda_stream), "tps_barrier")
        self.kernels_launched += 1

    # -------------------------------------------------------------- timing ---
    def measurements(self) -> dict:
        """Synchronise; seconds since each device's stage-start event."""
        for r in self.world.local_ranks:
            torch.cuda.synchronize(self.world.devices[r])
        out = {"groups": {}, "switches": []}
        for (ep, g), tl in self.timeline.items():
            s = self.start[tl.rank]
            out["groups"][f"{ep}:{g}"] = {
                "prefill": s.elapsed_time(tl.prefill_end) / 1e3 if tl.prefill_end is not None else None,
                "rounds": [s.elapsed_time(e) / 1e3 for e in tl.rounds]}
        nat.check_abort("generation stage")
        for r, bad in self._bad.items():
            if int(bad.item()):
                raise PlanVerificationError(f"rank {r}: {int(bad.item())} KV copy items pointed outside a pool")
        for t in self.switches:
            out["switches"].append({
                "ranks": {r: [self.start[r].elapsed_time(e) / 1e3 for e in ev] for r, ev in t.marks.items()},
                "nvlink_bytes": t.nvlink_bytes, "local_bytes": t.local_bytes, "kv_bytes": t.kv_bytes,
                "weight_bytes": t.weight_bytes, "host_plan_s": t.host_plan_s, "host_capture_s": t.host_capture_s,
                "host_build_s": t.host_build_s, "host_s": t.host_s, "state_method": t.state_method,
                "per_rank": {r: dict(v) for r, v in t.per_rank.items()}})
        self._keep.clear()
        return out


class RecordedBackend:
    """Replays measured B200 clocks through the engine loop (same events, real times)."""

    exact_pool_cost = False

    def __init__(self, meas: list[dict]):
        self.groups: dict[str, dict] = {}
        for m in meas:
            self.groups.update(m["groups"])
        self.switch_meas = []
        for i in range(max((len(m["switches"]) for m in meas), default=0)):
            agg = dict(ranks={}, per_rank={}, nv=0, loc=0, kv=0, w=0, plan=0.0, cap=0.0, build=0.0, host=0.0,
                       method=MIGRATE)
            for m in meas:
                if i < len(m["switches"]):
                    s = m["switches"][i]
                    agg["ranks"].update(s["ranks"])
                    agg["per_rank"].update(s.get("per_rank", {}))
                    agg["nv"] += s["nvlink_bytes"]
                    agg["loc"] += s["local_bytes"]
                    agg["kv"] += s["kv_bytes"]
                    agg["w"] += s["weight_bytes"]
                    agg["plan"] = max(agg["plan"], s["host_plan_s"])
                    agg["cap"] = max(agg["cap"], s["host_capture_s"])
                    agg["build"] = max(agg["build"], s.get("host_build_s", 0.0))
                    agg["host"] = max(agg["host"], s.get("host_s", 0.0))
                    agg["method"] = s.get("state_method", MIGRATE)
            self.switch_meas.append(agg)
        self.epoch = 0
        self.cursor: dict[str, int] = {}
        self.nswitch = 0

    def prefill(self, node, g, members, tp) -> float:
        return self.groups[f"0:{g}"]["prefill"]

    def decode_block(self, node, group, n) -> np.ndarray:
        key = f"{self.epoch}:{group.index}"
        i = self.cursor.get(key, 0)
        ends = np.asarray(self.groups[key]["rounds"][i:i + n], dtype=float)
        self.cursor[key] = i + n
        return np.diff(np.concatenate([[group.clock], ends]))

    def planned_state_method(self, decision, naive_mode) -> str:
        return self.switch_meas[self.nswitch]["method"]

    def realize_switch(self, node, decision, statuses, merged, naive_mode):
        """Measured components: marks per rank = [arrive, released, weights done, KV done, resumed]
        (device clock since the stage start). The switch ends when the last rank resumes."""
        m = self.switch_meas[self.nswitch]
        barrier = max(g.clock for g in node.live_groups())
        marks = list(m["ranks"].values())
        end = max(v[4] for v in marks)
        w = max(v[2] - v[1] for v in marks)
        kv = max(v[3] - v[2] for v in marks)
        total = max(end - barrier, 0.0)
        w = min(w, total)
        kv = min(kv, total - w)
        self.nswitch += 1
        return SwitchCostBreakdown.build(kv, m["method"], w, 0.0, 0.0, total - w - kv)

    def switch_record_extra(self, node) -> dict:
        """SURVEY 8(d) switch units: bytes each GPU pulled from peers (NVLink when the ranks are
        GPUs of one node; local copies reported separately) over that GPU's barrier-release ->
        resume window; the switch rate is the max over GPUs."""
        m = self.switch_meas[self.nswitch - 1]
        win = {r: v[4] - v[1] for r, v in m["ranks"].items()}
        copy = {r: v[3] - v[1] for r, v in m["ranks"].items()}
        per = m["per_rank"]
        peer = max((per[r]["nvlink"] for r in per), default=0)
        local = max((per[r]["local"] for r in per), default=0)
        wall = max(win.values()) if win else 0.0
        rate = {r: per[r]["nvlink"] / win[r] / 1e9 for r in per if r in win and win[r] > 0}
        return {"measured": True, "state_method": m["method"], "nvlink_bytes_total": m["nv"],
                "local_copy_bytes": m["loc"], "kv_bytes": m["kv"], "weight_bytes": m["w"],
                "max_gpu_peer_bytes": peer, "max_gpu_local_bytes": local,
                "release_to_resume_s": wall, "copy_seconds": max(copy.values()) if copy else 0.0,
                "peer_gbps_per_gpu": max(rate.values()) if rate else None,
                "copy_gbps_per_gpu": (max(per[r]["nvlink"] + per[r]["local"] for r in per) / max(copy.values()) / 1e9)
                if per and copy and max(copy.values()) > 0 else None,
                "host_plan_s": m["plan"], "host_capture_s": m["cap"], "host_build_s": m["build"],
                "host_switch_s": m["host"]}

    def after_switch(self, node) -> None:
        self.epoch += 1

    def finish(self, node) -> None:
        pass


class GlobalCoordinator:
    """Run one generation stage on B200 and report it in the reference's SimReport schema."""

    def __init__(self, spec: ScenarioSpec, geom: DecoderGeometry, world: World | None = None, seed: int = 0,
                 table=None, use_graphs: bool = True, copy_mode: int = 1, host_io: bool = False,
                 state_method: str | None = None, temperature: float = 0.0, **backend_opts):
        self.spec = spec
        self.geom = geom
        self.world = world or World.virtual(spec.cluster.gpus_per_node)
        self.table = table
        self.seed = seed
        self.backend = B200Backend(spec, geom, self.world, seed=seed, use_graphs=use_graphs,
                                   copy_mode=copy_mode, host_io=host_io, state_method=state_method,
                                   temperature=temperature, **backend_opts)
        self.setup_capture_s = self.backend.capture_all(every_layout=True)
        self.setup_items_s = self.backend.prepare_switch_items()
        self.runs = 0
        self.last_wall_s = 0.0

    def run(self) -> tuple[SimReport, dict]:
        """One generation stage: real execution, then the measured-clock report."""
        be = self.backend
        if self.runs:
            be.reset(self.seed)
        self.runs += 1
        be.begin()
        t0 = time.perf_counter()
        run(self.spec, self.table, backend=be)
        meas = be.measurements()  # synchronises: includes the final device->host token copies
        self.last_wall_s = time.perf_counter() - t0
        report = run(self.spec, self.table, backend=RecordedBackend(self.world.allgather(meas)))
        return report, meas

    def outputs(self) -> torch.Tensor:
        """Generated tokens per sample (host, after run): [global_batch, l_max] int32."""
        return self.backend.out_host
