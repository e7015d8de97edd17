"""The operator-level drop-in (paper_1711_04556_b200.kernels, the reference's
rcpsp_tabu/kernels.py seam) called exactly as the reference's callers call
it -- positional numpy arguments, caller-owned scratch, in-place outputs,
tuple returns (kernels.py:68-385; evaluator.py:128-144; moves.py:83-94;
search.py:60-75; make_golden.py reproduces the reference's own calls) --
against the golden vectors the reference produced."""

import numpy as np
import pytest

import oracle
from conftest import random_topological_order

pytestmark = pytest.mark.gpu

from paper_1711_04556_b200 import kernels, synth  # noqa: E402
from paper_1711_04556_b200.tabu import TabuState  # noqa: E402


def _scratch(inst):
    ka = inst.kernel_arrays
    r_max = int(ka.capacities.max())
    m = inst.n_resources
    return (np.zeros(inst.n_activities, np.int32), np.zeros((m, r_max), np.int32),
            np.zeros(r_max, np.int32), np.zeros((m, ka.horizon + 1), np.int32))


def test_evaluate_order_signature(golden, ginst):
    for rec in golden["evaluate"]:
        inst = ginst[rec["instance"]]
        ka = inst.kernel_arrays
        starts, cap_state, copy_buf, tau = _scratch(inst)
        order = np.array(rec["order"], np.int32)
        for mode in (0, 1):
            cm = kernels.evaluate_order(order, ka.durations, ka.demands, ka.capacities,
                                        ka.pred_ptr, ka.pred_dat, mode, ka.horizon, starts,
                                        cap_state, copy_buf, tau, ka.horizon)
            assert cm == rec[f"cmax{mode}"], (rec["instance"], mode)
            assert starts.tolist() == rec[f"starts{mode}"], (rec["instance"], mode)


def test_filter_moves_and_move_feasible(golden, ginst):
    for rec in golden["filter"]:
        inst = ginst[rec["instance"]]
        ka = inst.kernel_arrays
        order = np.array(rec["order"], np.int32)
        moves = oracle.neighborhood(inst.n_activities, rec["delta"])
        out = np.empty_like(moves)
        kept = kernels.filter_moves(ka.adjacency, order, moves, len(moves), out)
        assert out[:kept].tolist() == rec["kept"], (rec["instance"], rec["delta"])
        ok = {tuple(x) for x in rec["kept"]}
        for u, v in moves[:: max(1, len(moves) // 25)].tolist():
            assert kernels.move_feasible(ka.adjacency, order, u, v) == ((u, v) in ok)


def test_run_chunk_signature(golden, ginst):
    """kernels.run_chunk with the reference's 26 positional arguments: order,
    best_order, tabu list/counts and trace mutated in place, the 7-tuple
    returned -- equal to the reference's outputs (make_golden.py:175-179)."""
    for rec in golden["run_chunk"]:
        inst = ginst[rec["instance"]]
        ka = inst.kernel_arrays
        n = inst.n_activities
        moves_all = oracle.neighborhood(n, rec["delta"])
        tabu = TabuState(n, rec["tabu_size"])
        tabu.load(np.array(rec["tabu_list"], np.int32), rec["tabu_head"])
        tl, tc = tabu.entries, tabu.counts
        order_io = np.array(rec["order"], np.int32)
        best = order_io.copy()
        trace = np.zeros(rec["budget"], np.int32)
        starts, cap_state, copy_buf, tau = _scratch(inst)
        cmax_buf = np.empty(max(1, len(moves_all)), np.int32)
        moves_buf = np.empty_like(moves_all)
        out = kernels.run_chunk(order_io, ka.durations, ka.demands, ka.capacities, ka.pred_ptr,
                                ka.pred_dat, ka.adjacency, moves_all, rec["mode"], ka.horizon,
                                tl, tc, rec["tabu_head"], rec["budget"], rec["adopted_cmax"],
                                rec["start_cmax"], rec["best_known_cmax"], rec["floor_cmax"],
                                best, starts, cap_state, copy_buf, tau, moves_buf, cmax_buf,
                                trace)
        iters = int(out[0])
        key = (rec["instance"], rec["mode"])
        assert [int(x) for x in out] == rec["out_stats"], key
        assert order_io.tolist() == rec["out_order"], key
        assert best.tolist() == rec["out_best_order"], key
        assert trace[:iters].tolist() == rec["out_trace"], key
        assert tl.tolist() == rec["out_tabu_list"], key
        # the counter table mirrors the list (tabu.py:1-10)
        want = np.zeros_like(tc)
        for u, v in tl.tolist():
            if u or v:
                want[u, v] += 1
        assert (tc == want).all(), key


def test_select_and_tabu_add_semantics():
    """select_move / select_min / tabu_add (kernels.py:263-309) against the
    oracle's C restatement on random neighbourhoods and tabu states."""
    rng = np.random.default_rng(7)
    for trial in range(200):
        n = int(rng.integers(6, 40))
        k = int(rng.integers(0, 30))
        moves = np.stack([rng.integers(1, n - 2, k), rng.integers(1, n - 2, k)], 1).astype(np.int32)
        cm = rng.integers(10, 20, k).astype(np.int32)
        counts = (rng.random((n, n)) < 0.3).astype(np.int32)
        asp = int(rng.integers(9, 21))
        got = kernels.select_move(moves, k, cm, counts, asp)
        want = oracle.select_move(moves, cm, counts, asp)
        assert got == want, trial
        assert kernels.select_min(k, cm) == oracle.select_min(cm)
    tl = np.zeros((5, 2), np.int32)
    tc = np.zeros((8, 8), np.int32)
    head = 0
    seq = [(1, 2), (3, 4), (1, 2), (5, 6), (2, 3), (1, 2), (4, 5)]
    for u, v in seq:
        head = kernels.tabu_add(tl, tc, head, u, v)
    assert head == len(seq) % 5
    assert tl.tolist() == [[1, 2], [4, 5], [1, 2], [5, 6], [2, 3]]
    assert tc[1, 2] == 2 and tc[3, 4] == 0 and tc[4, 5] == 1


def test_operator_layer_on_genp(ginst):
    """The seam on the benchmarked Gen-P shape: evaluate_order on random
    orders (both modes) equals the oracle, start times included."""
    inst = synth.benchmark_batch("j120p", 1, first_seed=311)[0]
    ka = inst.kernel_arrays
    rng = np.random.default_rng(4)
    starts, cap_state, copy_buf, tau = _scratch(inst)
    for _ in range(6):
        order = random_topological_order(inst, rng)
        for mode in (0, 1):
            cm = kernels.evaluate_order(order, ka.durations, ka.demands, ka.capacities,
                                        ka.pred_ptr, ka.pred_dat, mode, ka.horizon, starts,
                                        cap_state, copy_buf, tau, ka.horizon)
            wc, ws = oracle.evaluate_batch(inst, order[None], mode)
            assert cm == int(wc[0]) and starts.tolist() == ws[0].tolist()
