"""The CPU oracle (oracle/) against the reference's golden vectors.

Pins the oracle before it is trusted as the checker of the GPU path: every
vector in tests/golden/golden.json was produced by the reference package
itself (numba backend) -- see tests/golden/make_golden.py.
"""

import numpy as np
import pytest

import oracle
from conftest import instance_from


def test_evaluate_matches_reference(golden, ginst):
    for rec in golden["evaluate"]:
        inst = ginst[rec["instance"]]
        for mode in (0, 1):
            c, s = oracle.evaluate_batch(inst, np.array([rec["order"]]), mode)
            assert int(c[0]) == rec[f"cmax{mode}"], (rec["instance"], mode)
            assert s[0].tolist() == rec[f"starts{mode}"]


def test_worked_example_and_gap(ginst):
    ex = ginst["example12"]
    order = [0, 1, 2, 3, 4, 6, 5, 7, 9, 10, 8, 11]
    c, s = oracle.evaluate_batch(ex, np.array([order]), oracle.MODE_TIME)
    assert c[0] == 22 and s[0].tolist() == [0, 0, 4, 4, 7, 12, 9, 12, 20, 15, 16, 22]
    gap = ginst["gap"]
    assert oracle.evaluate_batch(gap, np.array([[0, 1, 2, 3, 4]]), 1)[0][0] == 10
    assert oracle.evaluate_batch(gap, np.array([[0, 1, 2, 3, 4]]), 0)[0][0] == 13
    assert oracle.critical_path(ex) == 16


def test_fbi_matches_reference(golden, ginst):
    for rec in golden["fbi"]:
        fo, fs, fc, fe = oracle.fbi(ginst[rec["instance"]], rec["order"], rec["mode"])
        assert fo.tolist() == rec["final_order"]
        assert fs.tolist() == rec["starts"]
        assert fc == rec["cmax"] and fe == rec["evaluations"]


def test_filter_matches_reference(golden, ginst):
    for rec in golden["filter"]:
        inst = ginst[rec["instance"]]
        moves = oracle.neighborhood(inst.n_activities, rec["delta"])
        assert len(moves) == rec["n_moves"]
        kept = oracle.filter_moves(inst, rec["order"], moves)
        assert kept.tolist() == rec["kept"]


def test_run_chunk_matches_reference(golden, ginst):
    for rec in golden["run_chunk"]:
        inst = ginst[rec["instance"]]
        out = oracle.run_chunk(inst, rec["order"], rec["tabu_list"], rec["tabu_head"],
                               rec["budget"], rec["adopted_cmax"], rec["start_cmax"],
                               rec["best_known_cmax"], rec["floor_cmax"], rec["delta"],
                               rec["mode"])
        assert list(out["stats"]) == rec["out_stats"], rec["instance"]
        assert out["trace"].tolist() == rec["out_trace"]
        assert out["order"].tolist() == rec["out_order"]
        assert out["best_order"].tolist() == rec["out_best_order"]
        assert out["tabu_list"].tolist() == rec["out_tabu_list"]


def test_orchestrate_matches_reference(golden, ginst):
    for rec in golden["orchestrate"]:
        inst = ginst[rec["instance"]]
        ex = rec["extra"]
        got = oracle.orchestrate(inst, rec["total_iters"], 1, rec["seed"], rec["mode"],
                                 collect_trace=True, **ex)
        key = (rec["instance"], rec["total_iters"], rec["mode"])
        assert got["best_cmax"] == rec["best_cmax"], key
        assert got["evaluations"] == rec["evaluations"], key
        assert got["exchanges"] == rec["exchanges"], key
        assert got["diversifications"] == rec["diversifications"], key
        assert got["forced_tabu_picks"] == rec["forced_tabu_picks"], key
        assert got["iterations"] == rec["iterations"], key
        assert got["stop_reason"] == rec["stop_reason"], key
        assert [t.tolist() for t in got["traces"]] == rec["traces"], key


def test_diversify_matches_reference(golden, ginst):
    for rec in golden["diversify"]:
        st = oracle.rng_state(rec["seed"])
        out = oracle.diversify(ginst[rec["instance"]], rec["order"], rec["phi_steps"], st)
        assert out.tolist() == rec["out"]


def test_rng_matches_numpy(golden):
    for rec in golden["rng"]:
        st = oracle.rng_state(rec["seed"])
        for kind, n, want in rec["seq"]:
            if kind == "int":
                assert oracle.pcg_integers(st, n) == want
            else:
                assert oracle.pcg_permute(st, np.arange(n)).tolist() == want


def test_assigned_iterations_matches_reference(golden):
    for cmax, ic, bi, best, want in golden["assigned_iterations"]:
        assert oracle.assigned_iterations(cmax, ic, bi, best) == want
    # reference test_cooperation.py:28-48 goldens
    assert oracle.assigned_iterations(100, 0, 1000, 100) == 200
    assert oracle.assigned_iterations(101, 1000, 1000, 100) == 59
    assert oracle.assigned_iterations(100, 10**9, 1000, 100) == 160


def test_single_step_goldens():
    """Fig. 4 and the gap cases (reference test_evaluator.py:49-160)."""
    from paper_1711_04556_b200 import make_instance
    inst = make_instance("fig4", [0, 3, 0], [7], [[0], [3], [0]], [[1], [2], []])
    lv = np.array([[7, 7, 5, 5, 5, 5, 4]], np.int32)
    assert oracle.cap_earliest_start(inst, lv, 1) == 5
    oracle.cap_update(inst, lv, 1, 5)
    assert lv[0].tolist() == [8, 8, 8, 7, 7, 5, 4]
    gap = make_instance("g", [0, 5, 3, 5, 0], [2], [[0], [2], [2], [0], [0]],
                        [[1, 2, 3], [4], [4], [4], []])
    free = np.full((1, 14), 2, np.int32)
    oracle.time_update(gap, free, 1, 5)
    assert oracle.time_earliest_start(gap, free, 2, 0) == 0
    assert oracle.time_earliest_start(gap, free, 2, 4) == 10


def test_touch_counter_positive(ginst):
    inst = ginst["genr120s0"]
    order = np.arange(inst.n_activities)
    from conftest import random_topological_order
    order = random_topological_order(inst, np.random.default_rng(0))
    w_time, steps = oracle.touches(inst, order, 1)
    w_cap, _ = oracle.touches(inst, order, 0)
    assert w_time > w_cap > 0 and steps > 0


@pytest.mark.slow
def test_multiworker_oracle_feasible(ginst):
    got = oracle.orchestrate(ginst["genr60s0"], 400, 4, 3, 1)
    assert got["iterations"] == 400
    assert got["best_cmax"] >= got["critical_path"]
