"""CPU oracle for the rcpsp_tabu hot path -- TEST INFRASTRUCTURE ONLY.

This package restates the reference's numba kernels and search loop in plain C
(`oracle/oracle.c`, built to `oracle/liboracle.so` by `oracle/Makefile`) plus a
pure-Python PCG64 replica (`oracle/pcg64.py`).  Only `tests/`,
`__graft_entry__.smoke()` and the CPU legs of `bench.py` may import it; the
product package (`paper_1711_04556_b200`) never does, and fails loudly when
its CUDA library is missing instead of falling back to anything here.

Parity of this oracle with the reference is pinned by `tests/test_oracle.py`
against golden vectors produced by the reference itself
(`tests/golden/make_golden.py`, run in the build container where
`/root/reference` is importable).

Instances are duck-typed: any object with `durations`, `capacities`,
`demands` (N x M) and `successors` (tuple of tuples) works -- the reference's
`ProjectInstance` and the product's mirror alike.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"
_lib = None

MODE_CAPACITY = 0
MODE_TIME = 1

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_c_int = ctypes.c_int
_c_long = ctypes.c_long


def build() -> Path:
    """Compile liboracle.so (gcc) if it is missing or stale."""
    src = _HERE / "oracle.c"
    if not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        inst = [_c_int, _c_int, _c_int, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p]
        L.oracle_evaluate_batch.argtypes = inst + [_i32p, _c_int, _c_int, _c_int, _i32p,
                                                   ctypes.c_void_p]
        L.oracle_touches.argtypes = [_c_int, _c_int, _c_int, _i32p, _i32p, _i32p, _i32p, _i32p,
                                     _i32p, _c_int, _c_int, ctypes.POINTER(_c_long)]
        L.oracle_touches.restype = _c_long
        L.oracle_filter_moves.argtypes = [_u8p, _c_int, _i32p, _i32p, _c_int, _i32p]
        L.oracle_tabu_add.argtypes = [_i32p, _c_int, _i32p, _c_int, _c_int, _c_int, _c_int]
        L.oracle_select_move.argtypes = [_i32p, _c_int, _i32p, _i32p, _c_int, _c_int]
        L.oracle_select_min.argtypes = [_c_int, _i32p]
        L.oracle_run_chunk.argtypes = inst + [_c_int, _c_int, _i32p, _i32p, _c_int, _i32p,
                                              _c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                                              _i32p, _i32p, _i64p]
        L.oracle_fbi.argtypes = inst + [_i32p, _c_int, _i32p, _i32p, ctypes.POINTER(_c_long)]
        L.oracle_critical_path.argtypes = [_c_int, _i32p, _i32p, _i32p, _i32p, _i32p]
        L.oracle_assigned_iterations.argtypes = [_c_int, _c_long, _c_long, _c_int]
        L.oracle_assigned_iterations.restype = _c_long
        L.oracle_orchestrate.argtypes = inst + [_i64p, _c_int, _u64p, _i32p, _i64p,
                                                ctypes.POINTER(ctypes.c_double),
                                                ctypes.c_void_p, _c_long, ctypes.c_void_p, _c_long]
        L.oracle_diversify.argtypes = [_c_int, _i32p, _i32p, _i32p, _c_int, _u64p]
        L.oracle_pcg_integers.argtypes = [_u64p, ctypes.c_int64]
        L.oracle_pcg_integers.restype = ctypes.c_int64
        L.oracle_pcg_permute.argtypes = [_u64p, _i32p, _c_int]
        L.oracle_cap_earliest_start.argtypes = [_i32p, _c_int, _i32p, _c_int, _i32p, _c_int]
        L.oracle_cap_update.argtypes = [_i32p, _c_int, _i32p, _c_int, _i32p, _i32p, _c_int,
                                        _c_int, _c_int]
        L.oracle_time_earliest_start.argtypes = [_i32p, _c_int, _c_int, _i32p, _c_int, _c_int,
                                                 _c_int, _c_int]
        L.oracle_time_update.argtypes = [_i32p, _c_int, _c_int, _i32p, _c_int, _c_int, _c_int]
        _lib = L
    return _lib


class OInst:
    """Flat int32 arrays of one instance, in the reference's kernel layout
    (instance.py:53-80): CSR pred/succ with sorted ids, dense adjacency,
    horizon = sum of durations."""

    def __init__(self, inst):
        self.durations = np.ascontiguousarray(inst.durations, dtype=np.int32)
        self.capacities = np.ascontiguousarray(inst.capacities, dtype=np.int32)
        self.demands = np.ascontiguousarray(inst.demands, dtype=np.int32)
        n = len(self.durations)
        succ = [sorted(int(j) for j in s) for s in inst.successors]
        preds = [[] for _ in range(n)]
        for i, ss in enumerate(succ):
            for j in ss:
                preds[j].append(i)
        preds = [sorted(p) for p in preds]
        self.n = n
        self.m = len(self.capacities)
        self.horizon = int(self.durations.sum())
        self.succ_ptr = np.zeros(n + 1, np.int32)
        self.pred_ptr = np.zeros(n + 1, np.int32)
        for i in range(n):
            self.succ_ptr[i + 1] = self.succ_ptr[i] + len(succ[i])
            self.pred_ptr[i + 1] = self.pred_ptr[i] + len(preds[i])
        self.succ_dat = np.array([j for s in succ for j in s] or [0], np.int32)
        self.pred_dat = np.array([j for p in preds for j in p] or [0], np.int32)
        self.adj = np.zeros((n, n), np.uint8)
        for i, ss in enumerate(succ):
            for j in ss:
                self.adj[i, j] = 1
        self.successors = tuple(tuple(s) for s in succ)
        self.predecessors = tuple(tuple(p) for p in preds)

    def args(self):
        return (self.n, self.m, self.horizon, self.durations, self.demands.reshape(-1),
                self.capacities, self.pred_ptr, self.pred_dat, self.succ_ptr, self.succ_dat)


def _oi(inst) -> OInst:
    return inst if isinstance(inst, OInst) else OInst(inst)


def rng_state(seed: int) -> np.ndarray:
    """numpy default_rng(seed) PCG64 state as 6 uint64 (state hi/lo, inc hi/lo,
    has_uint32, uinteger) -- the layout oracle.c and the device kernels use."""
    st = np.random.default_rng(seed).bit_generator.state
    return state_words(st)


def state_words(st: dict) -> np.ndarray:
    s, inc = st["state"]["state"], st["state"]["inc"]
    m64 = (1 << 64) - 1
    return np.array([s >> 64, s & m64, inc >> 64, inc & m64, st["has_uint32"],
                     st["uinteger"]], dtype=np.uint64)


def evaluate_batch(inst, orders, mode: int, reverse: bool = False):
    """kernels.evaluate_order (kernels.py:152-194) over a batch of orders.
    Returns (cmax[B], starts[B, N])."""
    oi = _oi(inst)
    orders = np.ascontiguousarray(np.atleast_2d(orders), dtype=np.int32)
    B = orders.shape[0]
    cmax = np.zeros(B, np.int32)
    starts = np.zeros((B, oi.n), np.int32)
    rc = lib().oracle_evaluate_batch(*oi.args(), orders.reshape(-1), B, int(mode), int(reverse),
                                     cmax, starts.ctypes.data)
    assert rc == 0
    return cmax, starts


def touches(inst, order, mode: int, reset_upto: int | None = None):
    """Element touches W of one evaluation and scan steps."""
    oi = _oi(inst)
    steps = _c_long(0)
    w = lib().oracle_touches(oi.n, oi.m, oi.horizon, oi.durations, oi.demands.reshape(-1),
                             oi.capacities, oi.pred_ptr, oi.pred_dat,
                             np.ascontiguousarray(order, np.int32), int(mode),
                             oi.horizon if reset_upto is None else int(reset_upto),
                             ctypes.byref(steps))
    return int(w), int(steps.value)


def neighborhood(n: int, delta: int) -> np.ndarray:
    """moves.py:60-72."""
    pairs = [(u, v) for u in range(1, n - 2) for v in range(u + 1, min(u + delta, n - 2) + 1)]
    return np.asarray(pairs, dtype=np.int32).reshape(len(pairs), 2)


def filter_moves(inst, order, moves) -> np.ndarray:
    """kernels.filter_moves (kernels.py:218-255)."""
    oi = _oi(inst)
    moves = np.ascontiguousarray(moves, np.int32).reshape(-1, 2)
    out = np.zeros_like(moves)
    k = lib().oracle_filter_moves(oi.adj.reshape(-1), oi.n, np.ascontiguousarray(order, np.int32),
                                  moves.reshape(-1), len(moves), out.reshape(-1))
    return out[:k].copy()


def select_move(moves, cmax, counts, aspiration: int) -> int:
    moves = np.ascontiguousarray(moves, np.int32).reshape(-1, 2)
    counts = np.ascontiguousarray(counts, np.int32)
    return int(lib().oracle_select_move(moves.reshape(-1), len(moves),
                                        np.ascontiguousarray(cmax, np.int32), counts.reshape(-1),
                                        counts.shape[0], int(aspiration)))


def select_min(cmax) -> int:
    cmax = np.ascontiguousarray(cmax, np.int32)
    return int(lib().oracle_select_min(len(cmax), cmax))


def run_chunk(inst, order, tabu_list, tabu_head, budget, adopted_cmax, start_cmax,
              best_known_cmax, floor_cmax, delta, mode):
    """kernels.run_chunk (kernels.py:316-385) on copies; counts are rebuilt from
    the list (tabu.py:52-60).  Returns dict(order, best_order, trace, stats7,
    tabu_list)."""
    oi = _oi(inst)
    order = np.ascontiguousarray(order, np.int32).copy()
    tl = np.ascontiguousarray(tabu_list, np.int32).reshape(-1, 2).copy()
    counts = np.zeros((oi.n, oi.n), np.int32)
    for u, v in tl:
        if u or v:
            counts[u, v] += 1
    best = order.copy()
    trace = np.zeros(max(1, budget), np.int32)
    out7 = np.zeros(7, np.int64)
    lib().oracle_run_chunk(*oi.args(), int(delta), int(mode), order, tl.reshape(-1), len(tl),
                           counts.reshape(-1), int(tabu_head), int(budget), int(adopted_cmax),
                           int(start_cmax), int(best_known_cmax), int(floor_cmax), best, trace,
                           out7)
    iters = int(out7[0])
    return dict(order=order, best_order=best, trace=trace[:iters].copy(),
                stats=tuple(int(x) for x in out7), tabu_list=tl, counts=counts)


def fbi(inst, order, mode: int):
    """forward_backward_improve (evaluator.py:207-266): (order, starts, cmax, evals)."""
    oi = _oi(inst)
    fo = np.zeros(oi.n, np.int32)
    fs = np.zeros(oi.n, np.int32)
    ev = _c_long(0)
    c = lib().oracle_fbi(*oi.args(), np.ascontiguousarray(order, np.int32), int(mode), fo, fs,
                         ctypes.byref(ev))
    return fo, fs, int(c), int(ev.value)


def critical_path(inst) -> int:
    oi = _oi(inst)
    return int(lib().oracle_critical_path(oi.n, oi.durations, oi.pred_ptr, oi.pred_dat,
                                          oi.succ_ptr, oi.succ_dat))


def assigned_iterations(cmax: int, iter_count: int, block_iters: int, best_cmax: int) -> int:
    return int(lib().oracle_assigned_iterations(int(cmax), int(iter_count), int(block_iters),
                                                int(best_cmax)))


def diversify(inst, order, phi_steps: int, state: np.ndarray):
    """search.diversify (search.py:77-94); `state` (6 uint64) advances in place."""
    oi = _oi(inst)
    work = np.ascontiguousarray(order, np.int32).copy()
    lib().oracle_diversify(oi.n, oi.succ_ptr, oi.succ_dat, work, int(phi_steps), state)
    return work


def size_defaults(n: int):
    """SearchParams.defaults_for size classes (search.py:44-57)."""
    if n <= 32:
        return 30, 60
    if n <= 62:
        return 60, 250
    if n <= 92:
        return 60, 600
    return 60, 800


def orchestrate(inst, total_iters: int, workers: int = 1, seed: int = 0, mode: int = MODE_TIME,
                delta: int | None = None, tabu_size: int | None = None, phi_steps: int = 20,
                phi_max: int = 3, pool_size: int = 16, collect_trace: bool = False) -> dict:
    """cooperation.orchestrate (cooperation.py:237-302) with a pinned mode."""
    oi = _oi(inst)
    d0, t0 = size_defaults(oi.n)
    delta = d0 if delta is None else delta
    tabu_size = t0 if tabu_size is None else tabu_size
    params = np.array([total_iters, workers, delta, tabu_size, phi_steps, phi_max, pool_size],
                      np.int64)
    seeds = np.concatenate([rng_state(seed)] + [rng_state(seed ^ w) for w in range(workers)])
    best = np.zeros(oi.n, np.int32)
    out = np.zeros(16, np.int64)
    wall = ctypes.c_double(0.0)
    tcap = max(1, total_iters + workers) if collect_trace else 0
    trace = np.zeros(max(tcap, 1), np.int32)
    chunks = np.zeros(max(tcap, 1), np.int64)
    lib().oracle_orchestrate(*oi.args(), params, int(mode), seeds, best, out, ctypes.byref(wall),
                             trace.ctypes.data if collect_trace else None, tcap,
                             chunks.ctypes.data if collect_trace else None, tcap)
    res = dict(best_cmax=int(out[0]), iterations=int(out[1]), evaluations=int(out[2]),
               exchanges=int(out[3]), diversifications=int(out[4]), forced_tabu_picks=int(out[5]),
               stop_reason="critical_path" if out[6] else "budget", critical_path=int(out[7]),
               best_mode=int(out[8]), pool_evaluations=int(out[9]), wall_time=wall.value,
               best_order=best)
    if collect_trace:
        lens = chunks[:int(out[11])]
        flat = trace[:int(out[10])]
        pieces, p = [], 0
        for ln in lens:
            pieces.append(flat[p:p + int(ln)].copy())
            p += int(ln)
        res["traces"] = pieces
    return res


def cap_earliest_start(inst, levels: np.ndarray, act: int) -> int:
    """kernels.cap_earliest_start (kernels.py:68-78) on levels [m][R_max]."""
    oi = _oi(inst)
    return int(lib().oracle_cap_earliest_start(np.ascontiguousarray(levels, np.int32).reshape(-1),
                                               levels.shape[1], oi.capacities, oi.m,
                                               oi.demands.reshape(-1), int(act)))


def cap_update(inst, levels: np.ndarray, act: int, start: int) -> None:
    """kernels.cap_update (kernels.py:81-110); levels updated in place."""
    oi = _oi(inst)
    flat = np.ascontiguousarray(levels, np.int32).reshape(-1)
    buf = np.zeros(levels.shape[1], np.int32)
    lib().oracle_cap_update(flat, levels.shape[1], oi.capacities, oi.m, oi.demands.reshape(-1),
                            buf, int(act), int(start), int(oi.durations[act]))
    levels[...] = flat.reshape(levels.shape)


def time_earliest_start(inst, free: np.ndarray, act: int, es_prec: int) -> int:
    """kernels.time_earliest_start (kernels.py:117-136) on free [m][H+1]."""
    oi = _oi(inst)
    return int(lib().oracle_time_earliest_start(
        np.ascontiguousarray(free, np.int32).reshape(-1), free.shape[1], oi.m,
        oi.demands.reshape(-1), int(act), int(es_prec), int(oi.durations[act]), oi.horizon))


def time_update(inst, free: np.ndarray, act: int, start: int) -> None:
    """kernels.time_update (kernels.py:139-146); free updated in place."""
    oi = _oi(inst)
    flat = np.ascontiguousarray(free, np.int32).reshape(-1)
    lib().oracle_time_update(flat, free.shape[1], oi.m, oi.demands.reshape(-1), int(act),
                             int(start), int(oi.durations[act]))
    free[...] = flat.reshape(free.shape)


def pcg_integers(state: np.ndarray, n: int) -> int:
    return int(lib().oracle_pcg_integers(state, int(n)))


def pcg_permute(state: np.ndarray, arr) -> np.ndarray:
    a = np.ascontiguousarray(arr, np.int32).copy()
    lib().oracle_pcg_permute(state, a, len(a))
    return a


def cpu_count() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
