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
from .switch_executor import (KVSource, KVTarget, Layout, Pieces, cached_weight_pulls, check, nvlink_bytes,
                              plan_history_pulls, plan_kv_pulls, to_items, verify_cover)
from .switchcost import MIGRATE, RECOMPUTE, SwitchCostBreakdown
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
    marks: dict          # rank -> [start, weights_done, kv_done, end] events
    nvlink_bytes: int
    local_bytes: int
    kv_bytes: int
    weight_bytes: int
    host_plan_s: float
    host_capture_s: float
    state_method: str = MIGRATE
    host_build_s: float = 0.0


class B200Backend:
    """Real execution behind the engine's seams (prefill, decode blocks, switches)."""

    exact_pool_cost = False

    def __init__(self, spec: ScenarioSpec, geom: DecoderGeometry, world: World, seed: int = 0,
                 use_graphs: bool = True, copy_mode: int = 1, prompts: np.ndarray | None = None,
                 host_io: bool = False, state_method: str | None = None, temperature: float = 0.0):
        self.spec, self.geom, self.world = spec, geom, world
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
        self._witems: dict = {}  # weight copy items per (transition, rank, arena pointers)
        self._build_layout(self.layout, weights_seed=seed)
        self._layouts[self.layout.tp] = {"ranks": self.ranks, "runners": self.runners,
                                         "cap": {g: self.max_batch for g in self.local_groups()}}
        self.preplan_s = self.preplan()

    def preplan(self) -> float:
        """Plan (and verify) this process's weight pulls for every switch from the initial layout
        to a wider candidate degree before the stage starts, so a switch's critical path only
        plans its KV pages (Qwen2.5-7B TP1 -> TP2: ~0.15 s of host planning per rank moved off the
        switch). Plans are memoised per (geometry, layouts, rank) for the process."""
        t0 = time.perf_counter()
        init = Layout(self.spec.initial_tp, self.world.gpus)
        for tp in self.spec.controller.tp_list:
            if tp > init.tp and self.world.gpus % tp == 0:
                new = Layout(tp, self.world.gpus)
                for r in self.world.local_ranks:
                    cached_weight_pulls(self.geom, init, new, r)
        return time.perf_counter() - t0

    # ------------------------------------------------------------- layout ---
    def stream(self, r: int):
        return torch.cuda.current_stream(self.world.devices[r])

    def local_groups(self, lay: Layout | None = None) -> list[int]:
        lay = lay or self.layout
        return sorted({lay.group_of(r) for r in self.world.local_ranks})

    def _build_layout(self, lay: Layout, weights_seed: int | None, per_group: dict[int, int] | None = None,
                      prefill: bool = True):
        comms = self.cache.get(lay.tp)
        ranks = {}
        for r in self.world.local_ranks:
            n = self.max_batch if per_group is None else per_group.get(lay.group_of(r), 0)
            ranks[r] = self._make_rank(lay, r, max(1, n), weights_seed, comms[r], prefill)
        self.ranks = ranks
        self.runners = {}
        for g in self.local_groups(lay):
            exs = [ranks[r].executor for r in lay.ranks_of_group(g) if r in ranks]
            self.runners[g] = GroupRunner(exs, use_graphs=self.use_graphs)

    def _make_rank(self, lay: Layout, r: int, slots: int, weights_seed, comm, prefill: bool) -> RankState:
        dev = self.world.devices[r]
        nat.init_device(dev.index or 0)
        sh = rank_shard(self.geom, lay.tp, lay.tp_rank(r))
        w = RankWeights(self.geom, sh, dev)
        if weights_seed is not None:
            w.fill_random(weights_seed)
        kv = KVPool(self.geom.num_layers, sh.n_kv, self.geom.head_dim, slots * pages_for(self.max_len), dev)
        st = SlotTable(slots, self.max_len, dev)
        pf = slots * max(1, PREFILL_ROWS // slots) if prefill else 0
        ex = InferExecutor(self.geom, sh, w, kv, st, slots, dev, comm=comm, prefill_rows=pf)
        ex.temperature = self.temperature
        return RankState(w, kv, st, ex, comm)

    def _use_layout(self, lay: Layout, per_group: dict[int, int] | None) -> bool:
        """Make `lay` current: reuse the cached ranks/runners of this TP degree when every
        local group's slot capacity suffices (slot tables and page pools reset), else build
        it (new buffers, weights filled by the switch's pulls) and cache it. True if built."""
        need = {g: max(1, self.max_batch if per_group is None else per_group.get(g, 0))
                for g in self.local_groups(lay)}
        c = self._layouts.get(lay.tp)
        if c is not None and all(c["cap"].get(g, 0) >= n for g, n in need.items()):
            for rs in c["ranks"].values():
                rs.slots.reset()
                rs.kv.reset()
            self.ranks, self.runners = c["ranks"], c["runners"]
            return False
        cap = {g: max(n, c["cap"].get(g, 0) if c else 0) for g, n in need.items()}
        self._build_layout(lay, weights_seed=None, per_group=cap)
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

    def capture_all(self) -> float:
        """Capture the decode graph of every bucket of every local group (host seconds)."""
        t0 = time.perf_counter()
        if self.use_graphs:
            for runner in self.runners.values():
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
        (tpshift/switchcost.py:203-219, engine.py:187-203)."""
        old, new = self.layout, Layout(tp_new, self.world.gpus)
        old_ranks = self.ranks
        # where every live sample sits now: {id: (old group, slot, pages)}, gathered across processes
        here = {}
        for g in self.local_groups(old):
            lead = self.ranks[self.first_local(g)]
            for slot, sid in lead.slots.sample_of.items():
                here[sid] = (g, slot, tuple(lead.slots.pages[slot]))
        where = {}
        for part in self.world.allgather(here):
            where.update(part)
        ptrs = self.world.share({r: {"w": rs.weights.arena, "kv": rs.kv.buf, "hist": rs.slots.history}
                                 for r, rs in old_ranks.items()})
        npg = {}
        for part in self.world.allgather({r: rs.kv.num_pages for r, rs in old_ranks.items()}):
            npg.update(part)
        marks = {r: [_event(self.stream(r))] for r in self.world.local_ranks}
        self._device_barrier()  # every rank has finished decoding on the old layout
        tb = time.perf_counter()
        self.epoch += 1
        self.layout = new
        self._use_layout(new, {g: len(m) for g, m in enumerate(merged)})
        stats = dict(nv=0, loc=0, kv=0, w=0)
        t_build = time.perf_counter() - tb
        t_plan = 0.0
        for r in self.world.local_ranks:
            rs, st = self.ranks[r], self.stream(r)
            t0 = time.perf_counter()
            wp = cached_weight_pulls(self.geom, old, new, r)  # verified once when first planned
            w_src = {k: v["w"] for k, v in ptrs.items()}
            # layouts (and so arena pointers) are cached: the items of a repeated transition too
            ikey = (old, new, r, rs.weights.arena.data_ptr(), tuple(sorted(w_src.items())))
            w_items = self._witems.get(ikey)
            if w_items is None:
                w_items = self._witems[ikey] = to_items(wp, w_src, rs.weights.arena.data_ptr())
            nv, loc = nvlink_bytes(wp, r)
            stats["nv"] += nv
            stats["loc"] += loc
            stats["w"] += nv + loc
            mine = merged[new.group_of(r)] if new.group_of(r) < len(merged) else []
            tgts, srcs, kvlen, hlen, pos_vals, plen, slot_list, seeds = [], [], [], [], [], [], [], []
            for s in mine:
                slot = rs.slots.alloc(s.id)
                pages = rs.kv.alloc(pages_for(self.max_len))
                rs.slots.pages[slot] = pages
                og, oslot, opages = where[s.id]
                tgts.append(KVTarget(slot=slot, pages=tuple(pages)))
                srcs.append(KVSource(old_group=og, slot=oslot, pages=opages))
                pos = s.context_len - 1          # next token to process; KV holds positions < pos
                kvlen.append(pos)
                hlen.append(s.context_len)
                pos_vals.append(pos)
                plen.append(s.prompt_len)
                seeds.append(as_int64(sampler_seed(self.spec.seed, s.id)))  # the sampler state's key
                slot_list.append(slot)
                h2d(rs.slots.page_table[slot, :len(pages)], pages)
            if slot_list:
                idx = torch.tensor(slot_list, dtype=torch.long).pin_memory().to(rs.slots.device, non_blocking=True)
                rs.slots.pos.index_copy_(0, idx, torch.tensor(pos_vals, dtype=torch.int32).pin_memory()
                                         .to(rs.slots.device, non_blocking=True))
                rs.executor.prompt_len.index_copy_(0, idx, torch.tensor(plen, dtype=torch.int32).pin_memory()
                                                   .to(rs.slots.device, non_blocking=True))
                rs.slots.seed.index_copy_(0, idx, torch.tensor(seeds, dtype=torch.int64).pin_memory()
                                          .to(rs.slots.device, non_blocking=True))
            kp = Pieces()
            by_pool: dict[int, list[int]] = {}
            for i, s in enumerate(srcs):
                by_pool.setdefault(npg[s.old_group * old.tp], []).append(i)
            for n_old, idxs in (by_pool.items() if not recompute else ()):
                p = plan_kv_pulls(self.geom, old, new, r, [srcs[i] for i in idxs], [tgts[i] for i in idxs],
                                  [kvlen[i] for i in idxs], n_old, rs.kv.num_pages)
                kp.add(*p.arrays())
            hp = plan_history_pulls(old, r, srcs, tgts, hlen, self.max_len, self.max_len)
            items = np.concatenate([to_items(kp, {k: v["kv"] for k, v in ptrs.items()}, rs.kv.buf.data_ptr()),
                                    to_items(hp, {k: v["hist"] for k, v in ptrs.items()},
                                             rs.slots.history.data_ptr())])
            for p in (kp, hp):
                a, b = nvlink_bytes(p, r)
                stats["nv"] += a
                stats["loc"] += b
                stats["kv"] += a + b
            t_plan += time.perf_counter() - t0
            self._copy(w_items, st)
            marks[r].append(_event(st))
            self._copy(items, st)
            if not recompute:
                marks[r].append(_event(st))
            for s, t in zip(mine, tgts):
                self.slot_of[s.id] = t.slot
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
        tc = time.perf_counter()
        self.capture_all()
        self.switches.append(SwitchTiming(marks=marks, nvlink_bytes=stats["nv"], local_bytes=stats["loc"],
                                          kv_bytes=stats["kv"], weight_bytes=stats["w"], host_plan_s=t_plan,
                                          host_capture_s=time.perf_counter() - tc,
                                          state_method=RECOMPUTE if recompute else MIGRATE,
                                          host_build_s=t_build))
        self._keep.append(old_ranks)  # (cached layouts are reused, never freed mid-stage)

    def _copy(self, items: np.ndarray, st) -> None:
        if len(items) == 0:
            return
        items = np.ascontiguousarray(items, dtype=np.int64)
        parts = [(items, self.copy_mode)]
        if self.copy_mode == 1:
            # the bulk-copy engine needs 16-B aligned addresses and sizes; the rest go through LSU
            ok = ((items[:, 0] | items[:, 1] | items[:, 2]) & 15) == 0
            parts = [(p, m) for p, m in ((items[ok], 1), (items[~ok], 0)) if len(p)]
        devs = []
        for part, mode in parts:  # item tables staged before the timed copy kernels
            host = torch.from_numpy(np.ascontiguousarray(part)).pin_memory()
            devs.append((host.to(st.device, non_blocking=True), len(part), mode))
        if self.copy_events is not None:
            self.copy_events.append((_event(st), int(items[:, 2].sum())))
        for dev, n, mode in devs:
            nat.check(nat.lib().tps_copy_items(dev.data_ptr(), n, mode, 0, st.cuda_stream), "tps_copy_items")
            self._keep.append(dev)
        if self.copy_events is not None:
            self.copy_events[-1] += (_event(st),)
        self.kernels_launched += len(parts)

    def _device_barrier(self) -> None:
        """Node-wide device barrier (a virtual world is already ordered by its single stream)."""
        if not self.world.distributed:
            return
        if self._bar is None:
            r = self.world.local_ranks[0]
            mine = torch.zeros(1, dtype=torch.int64, device=self.world.devices[r])
            ptrs = self.world.share({r: {"bar": mine}})
            self._bar = (mine, {k: v["bar"] for k, v in ptrs.items()})
        mine, ptrs = self._bar
        self._barrier_epoch += 1
        r = self.world.local_ranks[0]
        peers = [ptrs[x] for x in range(self.world.gpus) if x != r]
        nat.check(nat.lib().tps_barrier(nat.ptr_array(peers), len(peers), mine.data_ptr(),
                                        self._barrier_epoch * (self.world.gpus - 1), self.stream(r).cuda_stream),
                  "tps_barrier")
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
        for t in self.switches:
            out["switches"].append({
                "ranks": {r: [self.start[r].elapsed_time(e) / 1e3 for e in ev] for r, ev in t.marks.items()},
                "nvlink_bytes": t.nvlink_bytes, "local_bytes": t.local_bytes, "kv_bytes": t.kv_bytes,
                "weight_bytes": t.weight_bytes, "host_plan_s": t.host_plan_s, "host_capture_s": t.host_capture_s,
                "state_method": t.state_method})
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
            agg = dict(ranks={}, nv=0, loc=0, kv=0, w=0, plan=0.0, cap=0.0, method=MIGRATE)
            for m in meas:
                if i < len(m["switches"]):
                    s = m["switches"][i]
                    agg["ranks"].update(s["ranks"])
                    agg["nv"] += s["nvlink_bytes"]
                    agg["loc"] += s["local_bytes"]
                    agg["kv"] += s["kv_bytes"]
                    agg["w"] += s["weight_bytes"]
                    agg["plan"] = max(agg["plan"], s["host_plan_s"])
                    agg["cap"] = max(agg["cap"], s["host_capture_s"])
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
        m = self.switch_meas[self.nswitch]
        barrier = max(g.clock for g in node.live_groups())
        marks = list(m["ranks"].values())
        end = max(v[3] for v in marks)
        w = max(v[1] - v[0] for v in marks)
        kv = max(v[2] - v[1] for v in marks)
        total = max(end - barrier, 0.0)
        w = min(w, total)
        kv = min(kv, total - w)
        self.nswitch += 1
        return SwitchCostBreakdown.build(kv, m["method"], w, 0.0, 0.0, total - w - kv)

    def switch_record_extra(self, node) -> dict:
        m = self.switch_meas[self.nswitch - 1]
        marks = list(m["ranks"].values())
        copy_s = max(v[2] for v in marks) - min(v[0] for v in marks)
        moved = m["nv"] + m["loc"]
        return {"measured": True, "state_method": m["method"], "nvlink_bytes_total": m["nv"], "local_copy_bytes": m["loc"],
                "kv_bytes": m["kv"], "weight_bytes": m["w"], "copy_seconds": copy_s,
                "copy_gbps_per_gpu": (moved / max(1, len(marks))) / copy_s / 1e9 if copy_s > 0 else None,
                "host_plan_s": m["plan"], "host_capture_s": m["cap"]}

    def after_switch(self, node) -> None:
        self.epoch += 1

    def finish(self, node) -> None:
        pass


class GlobalCoordinator:
    """Run one generation stage on B200 and report it in the reference's SimReport schema."""

    def __init__(self, spec: ScenarioSpec, geom: DecoderGeometry, world: World | None = None, seed: int = 0,
                 table=None, use_graphs: bool = True, copy_mode: int = 1, host_io: bool = False,
                 state_method: str | None = None, temperature: float = 0.0):
        self.spec = spec
        self.geom = geom
        self.world = world or World.virtual(spec.cluster.gpus_per_node)
        self.table = table
        self.seed = seed
        self.backend = B200Backend(spec, geom, self.world, seed=seed, use_graphs=use_graphs,
                                   copy_mode=copy_mode, host_io=host_io, state_method=state_method,
                                   temperature=temperature)
        self.setup_capture_s = self.backend.capture_all()
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
