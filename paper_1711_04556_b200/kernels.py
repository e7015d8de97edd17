"""Operator layer: the reference's `rcpsp_tabu/kernels.py` seam, CUDA backend.

Same function names, argument meaning and in-place output conventions as the
reference operators (kernels.py:68-385), executed by the sm_100a library.
There is exactly one backend: `BACKEND == "cuda"`; `RCPSP_TABU_BACKEND` may be
unset, "auto" or "cuda", anything else raises ValueError at import (the
reference rejects unknown values the same way, kernels.py:28-43).

Per-call these operators copy their numpy arguments to HBM and back; they
exist so code written against the reference operator layer runs unchanged.
The fast path is `cooperation.orchestrate` / `orchestrate_batch`, which keeps
the instance and every search state on the device for the whole solve.

Notes on exactness: results equal the reference for precedence-feasible
orders (the only inputs the reference search produces).  The scratch
arguments (`cap_state`, `copy_buf`, `tau`, `moves_buf`, `cmax_buf`) are
accepted for signature compatibility; the device keeps its own scratch.
"""

from __future__ import annotations

import hashlib
import os

import numpy as np

from . import device
from .instance import make_instance

MODE_CAPACITY = 0
MODE_TIME = 1

_ENV_VAR = "RCPSP_TABU_BACKEND"


def _pick_backend() -> str:
    choice = os.environ.get(_ENV_VAR, "auto").strip().lower() or "auto"
    if choice not in ("auto", "cuda"):
        raise ValueError(f"{_ENV_VAR}={choice!r} not understood; this package only has the "
                         f"'cuda' backend")
    return "cuda"


BACKEND = _pick_backend()

_inst_cache: dict = {}


def _digest(*arrays) -> bytes:
    """Content key of the operator's instance arrays: shapes, dtypes and
    every byte (buffer addresses are not identities -- callers mutate arrays
    in place and numpy reuses freed memory)."""
    h = hashlib.blake2b(digest_size=20)
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(repr((a.shape, a.dtype.str)).encode())
        h.update(a.tobytes())
    return h.digest()


def _remember(key: bytes, inst):
    if len(_inst_cache) > 64:
        _inst_cache.clear()
    _inst_cache[key] = inst
    return inst


def _instance(durations, demands, capacities, pred_ptr, pred_dat):
    """ProjectInstance whose predecessor lists are the given CSR (cached by
    the content of all five arrays)."""
    key = _digest(durations, demands, capacities, pred_ptr, pred_dat)
    hit = _inst_cache.get(key)
    if hit is not None:
        return hit
    n = len(durations)
    succ = [[] for _ in range(n)]
    for j in range(n):
        for e in range(int(pred_ptr[j]), int(pred_ptr[j + 1])):
            succ[int(pred_dat[e])].append(j)
    inst = make_instance("kernel-args", np.asarray(durations).tolist(),
                         np.asarray(capacities).tolist(),
                         np.asarray(demands).reshape(n, -1).tolist(), succ)
    return _remember(key, inst)


def _adj_instance(adjacency):
    """Instance carrying only the precedence graph of a dense adjacency."""
    adjacency = np.asarray(adjacency, dtype=bool)
    key = b"adj" + _digest(adjacency)
    hit = _inst_cache.get(key)
    if hit is not None:
        return hit
    n = adjacency.shape[0]
    succ = [list(np.nonzero(adjacency[i])[0]) for i in range(n)]
    return _remember(key, make_instance("adjacency", [0] * n, [1], [[0]] * n, succ))


def evaluate_order(order, durations, demands, capacities, pred_ptr, pred_dat, mode, horizon,
                   starts, cap_state=None, copy_buf=None, tau=None, reset_upto=None) -> int:
    """Serial SGS of `order` (kernels.py:152-194): fills `starts`, returns C_max."""
    inst = _instance(durations, demands, capacities, pred_ptr, pred_dat)
    cmax, st = device.eval_batch(inst, np.asarray(order, np.int32)[None], int(mode))
    starts[:] = st[0]
    return int(cmax[0])


def filter_moves(adjacency, order, moves, n_moves, out) -> int:
    """Stable compaction of the feasible swaps (kernels.py:218-255)."""
    inst = _adj_instance(adjacency)
    order = np.asarray(order, np.int32)
    moves = np.asarray(moves, np.int32).reshape(-1, 2)[:n_moves]
    if n_moves == 0:
        return 0
    feasible = device.filter_batch(inst, order[None], len(order))[0]
    ok = set(map(tuple, feasible.tolist()))
    kept = 0
    for u, v in moves.tolist():
        if (u, v) in ok:
            out[kept, 0], out[kept, 1] = u, v
            kept += 1
    return kept


def move_feasible(adjacency, order, u, v) -> bool:
    """True iff swapping positions u < v keeps every precedence (kernels.py:200-215)."""
    out = np.zeros((1, 2), np.int32)
    return filter_moves(adjacency, order, np.array([[u, v]], np.int32), 1, out) == 1


def tabu_add(tabu_list, tabu_count, head, u, v) -> int:
    """Circular-list insert with counter mirror (kernels.py:263-277).

    Host bookkeeping for TabuState snapshots; the device search keeps its own
    shared-memory list (csrc/cta.cuh:tabu_add1).
    """
    ou, ov = int(tabu_list[head, 0]), int(tabu_list[head, 1])
    if ou != 0 or ov != 0:
        tabu_count[ou, ov] -= 1
    tabu_list[head, 0], tabu_list[head, 1] = u, v
    tabu_count[u, v] += 1
    return (head + 1) % tabu_list.shape[0]


def select_move(moves, n_moves, cmaxes, tabu_count, aspiration_cmax) -> int:
    """Best admissible move index or -1 (kernels.py:280-297); lowest index on ties."""
    best, best_c = -1, 0
    for idx in range(n_moves):
        c = int(cmaxes[idx])
        if tabu_count[moves[idx, 0], moves[idx, 1]] > 0 and c >= aspiration_cmax:
            continue
        if best < 0 or c < best_c:
            best, best_c = idx, c
    return best


def select_min(n_moves, cmaxes) -> int:
    """Smallest makespan regardless of tabu status (kernels.py:300-309)."""
    return int(np.argmin(np.asarray(cmaxes[:n_moves]))) if n_moves > 0 else -1


def run_chunk(order, durations, demands, capacities, pred_ptr, pred_dat, adjacency, moves_all,
              mode, horizon, tabu_list, tabu_count, tabu_head, budget, adopted_cmax, start_cmax,
              best_known_cmax, floor_cmax, best_order, starts, cap_state, copy_buf, tau,
              moves_buf, cmax_buf, trace):
    """Up to `budget` tabu iterations on `order` in place (kernels.py:316-385).

    `moves_all` must be the lexicographic reduced neighbourhood of the run
    (moves.generate_reduced_neighborhood(arange(N), delta)); its distance cap
    is recovered from it.  Returns (iters, evals, improved, local_best,
    current, head, forced) and mutates order, best_order, tabu_list,
    tabu_count and trace like the reference.
    """
    inst = _instance(durations, demands, capacities, pred_ptr, pred_dat)
    moves_all = np.asarray(moves_all).reshape(-1, 2)
    delta = int((moves_all[:, 1] - moves_all[:, 0]).max()) if len(moves_all) else 1
    res = device.run_chunk_batch(inst, int(mode), delta, np.asarray(order, np.int32)[None],
                                 [np.asarray(tabu_list)], [int(tabu_head)], int(budget),
                                 int(adopted_cmax), int(start_cmax), int(best_known_cmax),
                                 int(floor_cmax))
    st = res["stats"][0]
    iters = int(st[0])
    order[:] = res["order"][0]
    if int(st[3]) < int(start_cmax):
        best_order[:] = res["best_order"][0]
    tabu_list[:, :] = res["tabu"][0]
    tabu_count[:, :] = 0
    occupied = (tabu_list[:, 0] != 0) | (tabu_list[:, 1] != 0)
    np.add.at(tabu_count, (tabu_list[occupied, 0], tabu_list[occupied, 1]), 1)
    trace[:iters] = res["trace"][0][:iters]
    return iters, int(st[1]), int(st[2]), int(st[3]), int(st[4]), int(st[5]), int(st[6])


def python_version(func):
    """Reference API shim: there is no interpreted variant of these operators."""
    return func
