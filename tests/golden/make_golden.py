#!/usr/bin/env python3
"""Generate golden vectors from the REFERENCE implementation (rcpsp_tabu).

Run in the build container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden.py

Writes tests/golden/golden.json.  Everything in it is produced by the
reference's own public API (evaluate, forward_backward_improve,
filter_infeasible, kernels.run_chunk, orchestrate, numpy's Generator) on
inputs built with the reference's own test helpers (helpers.random_instance,
random_topological_order) and fixtures (conftest.py example12/dummy2).  The
GPU box has no /root/reference, so tests there compare against this file.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]

import rcpsp_tabu as R  # noqa: E402
from rcpsp_tabu import kernels  # noqa: E402
from rcpsp_tabu.cooperation import assigned_iterations, WorkingSetEntry  # noqa: E402
from helpers import random_instance, random_topological_order  # noqa: E402
import conftest as C  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden.json"


def inst_dict(inst, recipe=None):
    return {
        "name": inst.name,
        "durations": inst.durations.tolist(),
        "capacities": inst.capacities.tolist(),
        "demands": inst.demands.tolist(),
        "successors": [list(s) for s in inst.successors],
        "recipe": recipe,
    }


def main() -> None:
    assert kernels.BACKEND == "numba", kernels.BACKEND
    g: dict = {"reference_backend": kernels.BACKEND, "numpy": np.__version__}
    instances: dict = {}

    # --- fixtures from conftest.py:17-55 and test_evaluator.py ------------
    instances["example12"] = inst_dict(R.make_instance(
        "example12", C.EXAMPLE_DURATIONS, C.EXAMPLE_CAPACITIES, C.EXAMPLE_DEMANDS,
        C.EXAMPLE_SUCCESSORS))
    instances["dummy2"] = inst_dict(R.make_instance("dummy2", [0, 0], [1], [[0], [0]],
                                                    [[1], []]))
    instances["gap"] = inst_dict(R.make_instance(
        "gap", [0, 5, 5, 3, 0], [2], [[0], [0], [2], [2], [0]], [[1, 3], [2], [4], [4], []]))
    ex = R.make_instance("e", C.EXAMPLE_DURATIONS, C.EXAMPLE_CAPACITIES, C.EXAMPLE_DEMANDS,
                         C.EXAMPLE_SUCCESSORS)
    instances["roomy"] = inst_dict(R.make_instance(
        "roomy", ex.durations.tolist(), [999, 999], ex.demands.tolist(),
        [list(s) for s in ex.successors]))
    instances["lowcap"] = inst_dict(R.make_instance(
        "low-cap", [0] + [25] * 24 + [0], [1], [[0]] + [[1]] * 24 + [[0]],
        [list(range(1, 25))] + [[25]] * 24 + [[]]))

    # --- Gen-R instances (benchmarks/compare_backends.py:31 recipe) -------
    genr = [(30, 0), (30, 1), (60, 0), (120, 0), (120, 1), (300, 0)]
    for n_real, seed in genr:
        kw = dict(demand_density=0.5, cap_lo=10, cap_hi=16)
        if n_real == 300:
            kw.update(cap_lo=40, cap_hi=80)
        inst = random_instance(n_real, 4, seed=seed, **kw)
        instances[f"genr{n_real}s{seed}"] = inst_dict(inst, dict(n_real=n_real, m=4, seed=seed,
                                                                 **kw))
    # small fuzz family with varied shapes (helpers.random_instance defaults)
    rng = np.random.default_rng(2024)
    for i in range(12):
        n_real = int(rng.integers(3, 25))
        m = int(rng.integers(1, 6))
        kw = dict(cap_lo=int(rng.integers(1, 8)), cap_hi=int(rng.integers(8, 20)),
                  demand_density=float(rng.choice([0.3, 0.5, 1.0])))
        inst = random_instance(n_real, m, seed=100 + i, **kw)
        instances[f"fuzz{i}"] = inst_dict(inst, dict(n_real=n_real, m=m, seed=100 + i, **kw))
    g["instances"] = instances

    def load(name):
        d = instances[name]
        return R.make_instance(d["name"], d["durations"], d["capacities"], d["demands"],
                               d["successors"])

    # --- evaluate_order: both modes, starts included ----------------------
    ev = []
    orng = np.random.default_rng(7)
    for name in instances:
        inst = load(name)
        k = 3 if inst.n_activities > 200 else 6
        orders = [R.initial_order(inst, shuffle=False).tolist()]
        orders += [random_topological_order(inst, orng).tolist() for _ in range(k)]
        if name == "example12":
            orders.append(C.EXAMPLE_ORDER.tolist())
        for order in orders:
            rec = {"instance": name, "order": order}
            for mode in (0, 1):
                s = R.evaluate(np.array(order, np.int32), inst, mode)
                rec[f"cmax{mode}"] = s.cmax
                rec[f"starts{mode}"] = s.starts.tolist()
            ev.append(rec)
    g["evaluate"] = ev

    # --- forward-backward improvement --------------------------------------
    fb = []
    for name in ("example12", "genr30s0", "genr60s0", "genr120s0", "fuzz3", "fuzz7"):
        inst = load(name)
        for mode in (0, 1):
            order = random_topological_order(inst, orng)
            from rcpsp_tabu.evaluator import EvalScratch
            scratch = EvalScratch(inst)
            fo, sched = R.forward_backward_improve(inst, order, mode, scratch)
            fb.append({"instance": name, "mode": mode, "order": order.tolist(),
                       "final_order": fo.tolist(), "starts": sched.starts.tolist(),
                       "cmax": sched.cmax, "evaluations": scratch.evaluations})
    g["fbi"] = fb

    # --- filter_moves ------------------------------------------------------
    fl = []
    for name in ("example12", "genr30s0", "genr120s0", "fuzz1", "fuzz5"):
        inst = load(name)
        for delta in (1, 5, 30, 60, inst.n_activities):
            order = random_topological_order(inst, orng)
            moves = R.generate_reduced_neighborhood(order, delta)
            kept = R.filter_infeasible(moves, order, inst)
            fl.append({"instance": name, "delta": delta, "order": order.tolist(),
                       "kept": kept.tolist(), "n_moves": len(moves)})
    g["filter"] = fl

    # --- run_chunk (kernels.py:316-385) ------------------------------------
    rc = []
    # (instance, mode, budget, tabu size, delta, adopted: "zero" = no improvement
    # exit, "start" = exit on first improvement)
    cases = [("example12", 1, 150, 20, 30, "zero"), ("genr30s0", 1, 60, 60, 30, "zero"),
             ("genr30s1", 0, 60, 60, 30, "zero"), ("genr60s0", 1, 25, 250, 60, "zero"),
             ("genr120s0", 1, 6, 800, 60, "zero"), ("genr120s1", 0, 8, 800, 60, "zero"),
             ("fuzz2", 1, 80, 7, 10, "zero"), ("fuzz4", 0, 80, 7, 10, "zero"),
             ("genr30s0", 0, 60, 60, 30, "start"), ("genr60s0", 1, 40, 250, 60, "start"),
             ("genr300s0", 1, 2, 800, 60, "zero"), ("genr300s0", 0, 2, 800, 60, "zero")]
    for name, mode, budget, tsize, delta, adopt in cases:
        inst = load(name)
        ka = inst.kernel_arrays
        n = inst.n_activities
        order = random_topological_order(inst, orng)
        moves_all = R.generate_reduced_neighborhood(np.arange(n, dtype=np.int32), delta)
        tabu = R.TabuState(n, tsize)
        # seed the tabu list with some moves from the neighbourhood (some repeated)
        for _ in range(min(tsize + 3, 40)):
            if len(moves_all):
                u, v = moves_all[int(orng.integers(len(moves_all)))]
                tabu.add(int(u), int(v))
        list0, head0 = tabu.snapshot()
        starts = np.zeros(n, np.int32)
        from rcpsp_tabu.evaluator import EvalScratch
        sc = EvalScratch(inst)
        start_cmax = R.evaluate(order, inst, mode).cmax
        order_io = order.copy()
        best = order.copy()
        trace = np.zeros(budget, np.int32)
        cmax_buf = np.empty(max(1, len(moves_all)), np.int32)
        moves_buf = np.empty_like(moves_all)
        floor = R.critical_path_length(inst)
        adopted = start_cmax if adopt == "start" else 0
        best_known = start_cmax + 2
        out = kernels.run_chunk(order_io, ka.durations, ka.demands, ka.capacities, ka.pred_ptr,
                                ka.pred_dat, ka.adjacency, moves_all, mode, ka.horizon,
                                tabu.entries, tabu.counts, tabu.head, budget, adopted, start_cmax,
                                best_known, floor, best, sc.starts, sc.cap_state, sc.copy_buf,
                                sc.tau, moves_buf, cmax_buf, trace)
        iters = int(out[0])
        rc.append({"instance": name, "mode": mode, "budget": budget, "tabu_size": tsize,
                   "delta": delta, "order": order.tolist(), "tabu_list": list0.tolist(),
                   "tabu_head": int(head0), "adopted_cmax": int(adopted),
                   "start_cmax": int(start_cmax), "best_known_cmax": int(best_known),
                   "floor_cmax": int(floor), "out_order": order_io.tolist(),
                   "out_best_order": best.tolist(), "out_trace": trace[:iters].tolist(),
                   "out_stats": [int(x) for x in out], "out_tabu_list": tabu.entries.tolist()})
    g["run_chunk"] = rc

    # --- orchestrate, B = 1, pinned mode (cooperation.py:237-302) -----------
    orch = []
    runs = [("genr30s0", 1000, 0, 1, {}), ("genr30s0", 1000, 0, 0, {}),
            ("example12", 300, 21, 1, {}), ("example12", 2000, 3, 1, {}),
            ("genr60s0", 200, 0, 1, {}), ("genr120s0", 30, 0, 1, {}),
            ("genr120s0", 30, 0, 0, {}),
            ("fuzz3", 400, 5, 1, {"pool_size": 2, "phi_max": 1}),
            ("fuzz6", 400, 9, 0, {"pool_size": 1, "phi_max": 0, "phi_steps": 7}),
            ("genr30s1", 600, 4, 1, {"pool_size": 3, "phi_max": 1}),
            ("roomy", 5000, 2, 1, {}), ("dummy2", 50, 0, 1, {}), ("example12", 0, 1, 1, {})]
    for name, iters, seed, mode, extra in runs:
        inst = load(name)
        p = R.SearchParams.defaults_for(inst.n_activities, total_iters=iters, workers=1,
                                        seed=seed, mode=R.EvalMode(mode), collect_trace=True,
                                        **extra)
        st = R.orchestrate(inst, p)
        orch.append({"instance": name, "total_iters": iters, "seed": seed, "mode": mode,
                     "extra": extra, "best_cmax": st.best_cmax,
                     "starts": st.schedule.starts.tolist(), "iterations": st.iterations,
                     "evaluations": st.evaluations, "exchanges": st.exchanges,
                     "diversifications": st.diversifications,
                     "forced_tabu_picks": st.forced_tabu_picks, "stop_reason": st.stop_reason,
                     "critical_path": st.critical_path,
                     "traces": [t.tolist() for t in st.traces]})
    g["orchestrate"] = orch

    # --- diversify (search.py:77-94) ----------------------------------------
    dv = []
    for name in ("example12", "genr30s0", "fuzz3"):
        inst = load(name)
        for seed in (0, 77, 123):
            order = R.initial_order(inst, shuffle=False)
            out = R.diversify(order, 20, inst, np.random.default_rng(seed))
            dv.append({"instance": name, "seed": seed, "phi_steps": 20, "order": order.tolist(),
                       "out": out.tolist()})
    g["diversify"] = dv

    # --- initial_order with shuffle (moves.py:42-57) -------------------------
    io = []
    for name in ("example12", "genr30s0", "genr120s0"):
        inst = load(name)
        r = np.random.default_rng(5)
        io.append({"instance": name, "seed": 5,
                   "orders": [R.initial_order(inst, True, r).tolist() for _ in range(4)]})
    g["initial_order"] = io

    # --- Eq. 8 (cooperation.py:39-49) --------------------------------------
    ai = []
    grid_rng = np.random.default_rng(11)
    for _ in range(400):
        best = int(grid_rng.integers(10, 800))
        cmax = best + int(grid_rng.integers(0, 40))
        ic = int(grid_rng.integers(0, 20000))
        bi = int(grid_rng.integers(1, 12000))
        e = WorkingSetEntry(order=np.zeros(2, np.int32), cmax=cmax,
                            tabu_entries=np.zeros((1, 2), np.int32), tabu_head=0, iter_count=ic)
        ai.append([cmax, ic, bi, best, assigned_iterations(e, bi, best)])
    g["assigned_iterations"] = ai

    # --- numpy PCG64 draws ---------------------------------------------------
    rg = []
    for seed in (0, 1, 5, 2**31 + 7):
        gen = np.random.default_rng(seed)
        seq = []
        drng = np.random.default_rng(seed + 1)
        for _ in range(60):
            if drng.random() < 0.5:
                n = int(drng.integers(1, 5000))
                seq.append(["int", n, int(gen.integers(n))])
            else:
                k = int(drng.integers(2, 30))
                seq.append(["perm", k, gen.permutation(np.arange(k, dtype=np.int32)).tolist()])
        rg.append({"seed": seed, "seq": seq})
    g["rng"] = rg

    OUT.write_text(json.dumps(g, separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size / 1024:.0f} KiB)")


if __name__ == "__main__":
    main()
