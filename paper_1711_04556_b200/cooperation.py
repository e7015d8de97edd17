"""Working set, exchange protocol and the orchestrator (reference cooperation.py).

`orchestrate` / `orchestrate_batch` are the B200 path: the instance(s), the
pool of |F| solutions per instance, every worker's order, tabu list and rng
live in HBM / shared memory for the whole run (the paper's homogeneous
model).  One CTA is one worker; the exchange transaction is the reference's
(write back an improvement, round-robin adoption, Eq. 8 grant) executed by
the CTA under a per-instance lock in global memory.  The host uploads the
packed instances once and reads back only the final results.

The host-side `WorkingSet` / `exchange` / `Worker` objects remain for code
written against the reference's cooperation API (they drive device chunks).
"""

from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import device, moves
from .evaluator import Schedule, check_schedule_feasible, evaluate
from .instance import ProjectInstance, critical_path_length, extract_features
from .search import SearchParams, Worker, run_worker  # noqa: F401
from .selector import DEFAULT_RULES, EvalMode, decide_dynamic, decide_static


@dataclass
class WorkingSetEntry:
    order: np.ndarray
    cmax: int
    tabu_entries: np.ndarray
    tabu_head: int
    iter_count: int = 0
    reads_without_improvement: int = 0
    mode: EvalMode = EvalMode.TIME


def assigned_iterations(entry: WorkingSetEntry, block_iters: int, best_cmax: int) -> int:
    """Eq. 8 with the quantity term read as block_iters/5 (cooperation.py:39-49).

    The device evaluates the same expression in double precision
    (csrc/kernels.cu:eq8); tests/test_gpu_parity.py pins the two together."""
    quality = 0.8 * math.exp(-100.0 * (entry.cmax / best_cmax - 1.0))
    intactness = 0.2 * math.exp(-4.0 * (entry.iter_count / block_iters))
    return math.floor((block_iters / 5.0) * (quality + intactness))


class WorkingSet:
    """|F| entries plus the global best behind one lock (host mirror)."""

    def __init__(self, entries: list[WorkingSetEntry], total_iters: int, floor_cmax: int):
        if not entries:
            raise ValueError("working set needs at least one entry")
        self.entries = entries
        self.lock = threading.Lock()
        self.cursor = 0
        self.total_iters = total_iters
        self.floor_cmax = floor_cmax
        self.planned = 0
        self.consumed = 0
        self.stop = False
        self.grant_cap = 0
        self.mode_controller = None
        best = min(range(len(entries)), key=lambda i: entries[i].cmax)
        self.best_cmax = entries[best].cmax
        self.best_order = entries[best].order.copy()
        self.best_mode = entries[best].mode
        if self.best_cmax <= floor_cmax:
            self.stop = True

    def _assert_pool_min(self) -> None:
        pool_min = min(e.cmax for e in self.entries)
        assert self.best_cmax <= pool_min, (
            f"global best {self.best_cmax} above pool minimum {pool_min}")


def exchange(worker: Worker, ws: WorkingSet):
    """Write back, then adopt the next entry round-robin (cooperation.py:82-135).
    Returns (order copy, grant, best-known cmax, diversify flag) or None."""
    with ws.lock:
        if worker.entry_index >= 0:
            ws.planned -= max(0, worker.granted - worker.used_iterations)
            ws.consumed += worker.used_iterations
            entry = ws.entries[worker.entry_index]
            entry.iter_count += worker.used_iterations
            if worker.improved:
                entry.order = worker.best_order.copy()
                entry.cmax = worker.local_best_cmax
                entry.tabu_entries, entry.tabu_head = worker.tabu.snapshot()
                entry.reads_without_improvement = 0
                entry.mode = worker.mode
                if worker.local_best_cmax < ws.best_cmax:
                    ws.best_cmax = worker.local_best_cmax
                    ws.best_order = worker.best_order.copy()
                    ws.best_mode = worker.mode
            worker.improved = False
            worker.entry_index = -1
        ws._assert_pool_min()
        if ws.best_cmax <= ws.floor_cmax:
            ws.stop = True
        if ws.stop or ws.planned >= ws.total_iters:
            return None
        index = ws.cursor % len(ws.entries)
        ws.cursor += 1
        entry = ws.entries[index]
        entry.reads_without_improvement += 1
        needs_diversify = entry.reads_without_improvement > worker.params.phi_max
        grant = max(1, assigned_iterations(entry, worker.params.block_iters, ws.best_cmax))
        if ws.grant_cap > 0:
            grant = min(grant, ws.grant_cap)
        grant = min(grant, ws.total_iters - ws.planned)
        ws.planned += grant
        worker.entry_index = index
        worker.adopted_cmax = entry.cmax
        worker.granted = grant
        worker.used_iterations = 0
        worker.tabu.load(entry.tabu_entries, entry.tabu_head)
        if ws.mode_controller is not None:
            worker.mode = ws.mode_controller.mode_for(ws.consumed)
        return entry.order.copy(), grant, ws.best_cmax, needs_diversify


def _solve_config(params: SearchParams, collect_trace: bool | None = None,
                  grant_cap: int = 0, **kw) -> device.SolveConfig:
    return device.SolveConfig(
        total_iters=params.total_iters, workers=params.workers, pool_size=params.pool_size,
        tabu_size=params.tabu_size, delta=params.delta, phi_steps=params.phi_steps,
        phi_max=params.phi_max, seed=params.seed,
        collect_trace=params.collect_trace if collect_trace is None else collect_trace,
        grant_cap=grant_cap, **kw)


def initialize_working_set(instance: ProjectInstance, params: SearchParams,
                           rng: np.random.Generator, mode: EvalMode, floor_cmax: int,
                           counters: dict | None = None) -> WorkingSet:
    """Pool initialisation on the GPU (k_pool_orders + k_pool_entry: shuffled
    levels, FBI on even entries, evaluation), read back as a host WorkingSet.
    `rng` supplies the PCG64 state and is advanced past the draws made."""
    st = rng.bit_generator.state
    m64 = (1 << 64) - 1
    words = np.array([st["state"]["state"] >> 64, st["state"]["state"] & m64,
                      st["state"]["inc"] >> 64, st["state"]["inc"] & m64, st["has_uint32"],
                      st["uinteger"]], np.uint64)
    solver = device.BatchSolver([instance], [int(mode)], _solve_config(params, False))
    solver.pool_rng_host[0] = words
    solver.upload()
    solver.pool_init()
    import torch
    torch.cuda.synchronize()
    device._raise_dev_err(solver.err)
    n = instance.n_activities
    orders = solver.ent_order.cpu().numpy()[0, :, :n]
    cmax = solver.ent_cmax.cpu().numpy()[0]
    pool_evals = int(solver.ws_hdr.cpu().numpy()[0, device.WS_FIELDS["pool_evals"]])
    # advance the caller's rng past the permutation draws (replayed on the host)
    for _ in range(params.pool_size):
        moves.initial_order(instance, shuffle=True, rng=rng)
    entries = [WorkingSetEntry(order=orders[i].astype(np.int32).copy(), cmax=int(cmax[i]),
                               tabu_entries=np.zeros((params.tabu_size, 2), np.int32),
                               tabu_head=0, mode=mode)
               for i in range(params.pool_size)]
    if counters is not None:
        counters["evaluations"] = counters.get("evaluations", 0) + pool_evals
    return WorkingSet(entries, params.total_iters, floor_cmax)


class DynamicModeController:
    """Re-times both modes every `window` consumed iterations (GPU timing)."""

    def __init__(self, instance: ProjectInstance, order: np.ndarray, delta: int, window: int):
        self.instance = instance
        self.order = np.asarray(order, dtype=np.int32)
        self.delta = delta
        self.window = max(1, window)
        self.next_measure_at = 0
        self.mode = EvalMode.TIME
        self.lock = threading.Lock()
        self.measurements = 0

    def mode_for(self, consumed: int) -> EvalMode:
        with self.lock:
            if consumed >= self.next_measure_at:
                self.mode = decide_dynamic(self.instance, self.order, self.delta)
                self.next_measure_at = consumed + self.window
                self.measurements += 1
            return self.mode


@dataclass
class RunStats:
    best_cmax: int
    schedule: Schedule
    feasible: bool
    iterations: int
    evaluations: int
    wall_time: float
    exchanges: int
    diversifications: int
    forced_tabu_picks: int
    workers: int
    mode: str
    stop_reason: str
    critical_path: int
    traces: list[np.ndarray] = field(default_factory=list)
    # device time (CUDA events) of pool init + search; wall_time is the host
    # perf_counter span as in the reference (cooperation.py:254, 273)
    device_ms: float = 0.0


def choose_mode(instance: ProjectInstance, params: SearchParams, requested: str,
                rules=DEFAULT_RULES) -> tuple[EvalMode, DynamicModeController | None]:
    """Resolve an --eval request (cooperation.py:204-225)."""
    if requested == "capacity":
        return EvalMode.CAPACITY, None
    if requested == "time":
        return EvalMode.TIME, None
    if requested == "auto-rule":
        return decide_static(extract_features(instance), rules), None
    if requested == "auto-measure":
        probe = moves.initial_order(instance, shuffle=False)
        if params.workers == 1:
            ctl = DynamicModeController(instance, probe, params.delta, params.measure_window)
            return ctl.mode_for(0), ctl
        return decide_dynamic(instance, probe, params.delta), None
    raise ValueError(f"unknown evaluator request {requested!r}")


def _finish(instance: ProjectInstance, res: device.BatchResult, i: int, params: SearchParams,
            mode_name: str, wall: float, device_ms: float | None = None) -> RunStats:
    n = instance.n_activities
    best_order = res.best_order[i, :n].astype(np.int32)
    schedule = evaluate(best_order, instance, int(res.best_mode[i]))
    feasible, problems = check_schedule_feasible(instance, schedule)
    if schedule.cmax != int(res.best_cmax[i]):
        raise AssertionError(f"stored best {int(res.best_cmax[i])} != re-evaluated "
                             f"{schedule.cmax}")
    if problems:
        raise AssertionError(f"best schedule failed the feasibility check: {problems}")
    floor = int(res.critical_path[i])
    return RunStats(
        best_cmax=int(res.best_cmax[i]), schedule=schedule, feasible=feasible,
        iterations=int(res.iterations[i]), evaluations=int(res.evaluations[i]), wall_time=wall,
        exchanges=int(res.exchanges[i]), diversifications=int(res.diversifications[i]),
        forced_tabu_picks=int(res.forced[i]), workers=params.workers, mode=mode_name,
        stop_reason="critical_path" if int(res.best_cmax[i]) <= floor else "budget",
        critical_path=floor, traces=res.traces[i] if res.traces else [],
        device_ms=res.device_ms if device_ms is None else device_ms)


def orchestrate(instance: ProjectInstance, params: SearchParams, mode: EvalMode | None = None,
                mode_controller: DynamicModeController | None = None,
                time_limit_s: float | None = None) -> RunStats:
    """Solve one instance on the GPU with `params.workers` CTAs (cooperation.py:237-302).

    With B = 1 and a pinned mode the trajectory (trace, evaluations,
    exchanges, best) is identical to the reference.  A dynamic controller
    (B = 1, 'auto-measure') re-measures the modes on the GPU between search
    epochs of `measure_window` granted iterations, the grant cap the
    reference applies in that mode.

    time_limit_s (an extension; the reference has no time stop): the search
    also stops when this much device time has passed (%globaltimer), like a
    solver's wall-clock limit."""
    if mode is None:
        mode = params.mode
    if mode_controller is not None and params.workers == 1:
        return _orchestrate_dynamic(instance, params, mode_controller)
    solver = device.BatchSolver([instance], [int(mode)],
                                _solve_config(params, time_limit_s=time_limit_s))
    res = solver.run()
    return _finish(instance, res, 0, params, EvalMode(mode).name, res.wall_s)


def _orchestrate_dynamic(instance: ProjectInstance, params: SearchParams,
                         ctl: DynamicModeController) -> RunStats:
    import torch
    window = max(1, params.measure_window)
    mode = ctl.mode_for(0)
    cfg = _solve_config(params, grant_cap=window)
    solver = device.BatchSolver([instance], [int(mode)], cfg)
    tick = time.perf_counter()
    solver.upload()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    solver.pool_init()
    limit = 0
    ms = 0.0
    while limit < params.total_iters:
        limit = min(params.total_iters, limit + window)
        solver.search(epoch_limit=limit)
        ev1.record()
        ev1.synchronize()
        ms += ev0.elapsed_time(ev1)
        hdr = solver.ws_hdr.cpu().numpy()[0]
        if hdr[device.WS_FIELDS["stop"]]:
            break
        new_mode = ctl.mode_for(int(hdr[device.WS_FIELDS["consumed"]]))
        if new_mode != mode:
            mode = new_mode
            solver.groups = {(int(mode), k[1]): v for k, v in solver.groups.items()}
            solver.d_ids = {k: solver.d_ids[old] for k, old in
                            zip(solver.groups, list(solver.d_ids))}
        ev0.record()
    wall = time.perf_counter() - tick
    res = solver.collect(ms, ms)
    return _finish(instance, res, 0, params, "dynamic", wall)


@dataclass
class BatchStats:
    """Aggregate of one orchestrate_batch call."""

    runs: list[RunStats]
    evaluations: int
    device_seconds: float
    wall_seconds: float
    launches: int
    solve_wall_seconds: float = 0.0   # host: upload + pool init + search (synced)

    @property
    def schedules_per_second(self) -> float:
        return self.evaluations / self.device_seconds if self.device_seconds > 0 else 0.0

    @property
    def cpm_dev(self) -> float:
        devs = [100.0 * (r.best_cmax - r.critical_path) / r.critical_path
                for r in self.runs if r.critical_path]
        return sum(devs) / len(devs) if devs else float("nan")


def orchestrate_batch(instances: list[ProjectInstance], params: SearchParams,
                      modes: list[EvalMode] | None = None, rules=DEFAULT_RULES,
                      group: int | None = None, threads: int = 0,
                      time_limit_s: float | None = None) -> BatchStats:
    """Solve many instances at once: each gets its own working set and
    `params.workers` CTAs; all run concurrently on the GPU.  Modes default
    to the static rules per instance (BASELINE config: heuristic selection)."""
    if modes is None:
        modes = [decide_static(extract_features(x), rules) for x in instances]
    tick = time.perf_counter()
    solver = device.BatchSolver(instances, [int(m) for m in modes],
                                _solve_config(params, group=group, threads=threads,
                                              time_limit_s=time_limit_s))
    res = solver.run()
    wall = time.perf_counter() - tick
    dev_s = res.device_ms * 1e-3
    # every instance ran concurrently over the same host wall span
    runs = [_finish(x, res, i, params, EvalMode(int(modes[i])).name, res.wall_s)
            for i, x in enumerate(instances)]
    return BatchStats(runs=runs, evaluations=int(res.evaluations.sum()), device_seconds=dev_s,
                      wall_seconds=wall, launches=res.n_launches, solve_wall_seconds=res.wall_s)


def _critical_path(instance: ProjectInstance) -> int:
    return critical_path_length(instance)
