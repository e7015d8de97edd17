#!/usr/bin/env python3
"""Small launches of every search-path kernel for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck), run on the GPU box:

    compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize.py

K1 k_eval_batch (TIME groups 32/16/8, CAPACITY 32/1, reversed), K2 k_run_chunk
(single CTA and 2-CTA cluster), K0 k_pool_orders/k_pool_entry/k_pool_finalize,
K3 k_solve (TIME and CAPACITY, one CTA per worker and clusters, B = 1 and
B = 3 with steals, a B_BIG instance), K4 k_export_elites/k_merge_elites,
filter, diversify, state ops.  Sizes are tiny so the instrumented run stays
within minutes; results are checked against the CPU oracle so a sanitizer
run also fails on a wrong answer."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import oracle  # noqa: E402
from conftest import random_topological_order  # noqa: E402
from paper_1711_04556_b200 import synth  # noqa: E402
from paper_1711_04556_b200 import device  # noqa: E402
from paper_1711_04556_b200.device import BatchSolver, SolveConfig  # noqa: E402


def main(sections: set[str]) -> None:
    import torch
    rng = np.random.default_rng(0)
    j30 = synth.benchmark_batch("j30p", 2, first_seed=3)
    j60 = synth.benchmark_batch("j60", 1, first_seed=2)[0]
    big = synth.random_instance(20, 3, seed=77, cap_lo=4, cap_hi=9, max_dur=45,
                                demand_density=0.8)          # durations > 32 (B_BIG)
    # K1
    for inst in ((j30[0], j60, big) if "K1" in sections else ()):
        orders = np.stack([random_topological_order(inst, rng) for _ in range(9)])
        for mode, groups in ((1, (32, 16, 8)), (0, (32, 1))):
            want, _ = oracle.evaluate_batch(inst, orders, mode)
            for g in groups:
                got, _ = device.eval_batch(inst, orders, mode, group=g)
                assert got.tolist() == want.tolist(), (inst.name, mode, g)
            rev = orders[:, ::-1].copy()
            want_r, _ = oracle.evaluate_batch(inst, rev, mode, reverse=True)
            assert device.eval_batch(inst, rev, mode, reverse=True)[0].tolist() == want_r.tolist()
    print("K1 ok", flush=True)
    # filter / diversify / state ops
    if "misc" not in sections:
        return _rest(sections, rng, j30, j60, big)
    o = random_topological_order(j60, rng)
    got = device.filter_batch(j60, o[None], 7)[0]
    assert got.tolist() == oracle.filter_moves(j60, o, oracle.neighborhood(j60.n_activities, 7)).tolist()
    st = np.stack([device.rng_words(5)])
    device.diversify_batch(j60, o[None], 20, st)
    state = np.zeros((j60.n_resources, int(j60.capacities.max())), np.int32)
    device.state_op(j60, "cap_update", state, 3, 0)
    print("filter/diversify/state ok", flush=True)
    _rest(sections, rng, j30, j60, big)


def _rest(sections, rng, j30, j60, big) -> None:
    import torch
    # K2 (the operator's cluster choice spreads a batch of 1 over 8 CTAs)
    for inst in ((j30[0], big) if "K2" in sections else ()):
        orders = np.stack([random_topological_order(inst, rng) for _ in range(2)])
        cm, _ = oracle.evaluate_batch(inst, orders, 1)
        for mode, group in ((1, 32), (0, 32), (0, 1)):
            cmm, _ = oracle.evaluate_batch(inst, orders, mode)
            for b in (1, 2):
                res = device.run_chunk_batch(inst, mode, 10, orders[:b],
                                             [np.zeros((20, 2), np.int32)] * b, [0] * b, 5, 0,
                                             cmm[:b], cmm[:b], 0, group=group)
                for k in range(b):
                    want = oracle.run_chunk(inst, orders[k], np.zeros((20, 2), np.int32), 0, 5,
                                            0, int(cmm[k]), int(cmm[k]), 0, 10, mode)
                    assert res["stats"][k][:7].tolist() == list(want["stats"]), (inst.name, mode)
    print("K2 ok", flush=True)
    # K0 + K3 + K4
    insts = j30 + [j60, big]
    for mode, cap_group in ((1, None), (0, 32), (0, 1)) if "K3" in sections else ():
        for workers, cluster in ((1, 1), (1, 2), (3, 1), (2, 4)):
            cfg = SolveConfig(total_iters=30, workers=workers, pool_size=4, tabu_size=30,
                              delta=20, phi_steps=5, phi_max=1, seed=1, cluster=cluster,
                              cap_group=cap_group, collect_trace=workers == 1)
            r = BatchSolver(insts, [mode] * len(insts), cfg).run()
            if workers == 1:
                for i, inst in enumerate(insts):
                    want = oracle.orchestrate(inst, 30, 1, 1, mode, delta=20, tabu_size=30,
                                              phi_steps=5, phi_max=1, pool_size=4)
                    assert int(r.best_cmax[i]) == want["best_cmax"], (i, mode, cluster)
                    assert int(r.evaluations[i]) == want["evaluations"], (i, mode, cluster)
            else:
                assert ((r.iterations == 30) | (r.best_cmax == r.critical_path)).all()
    # the large-project search kernel (TIME, > 64 activities: 20-warp CTAs,
    # long-suffix loop) and CAPACITY on the same instances
    big_insts = synth.benchmark_batch("j120p", 2, first_seed=3)
    for mode in ((1, 0) if "K3L" in sections else ()):
        for workers in (1, 2):
            cfg = SolveConfig(total_iters=12, workers=workers, pool_size=4, tabu_size=60,
                              delta=30, phi_steps=5, phi_max=1, seed=1, cluster=1)
            r = BatchSolver(big_insts, [mode] * 2, cfg).run()
            if workers == 1:
                for i, inst in enumerate(big_insts):
                    want = oracle.orchestrate(inst, 12, 1, 1, mode, delta=30, tabu_size=60,
                                              phi_steps=5, phi_max=1, pool_size=4)
                    assert int(r.best_cmax[i]) == want["best_cmax"], ("K3L", mode, i)
                    assert int(r.evaluations[i]) == want["evaluations"], ("K3L", mode, i)
    if "K3L" in sections:
        print("K3L ok", flush=True)
    # TIME with makespan-bounded per-warp profiles forced tight (fallback path)
    j60 = synth.benchmark_batch("j60p", 2, first_seed=0)
    for slots in (160, 96) if "sized" in sections else ():
        cfg = SolveConfig(total_iters=15, workers=1, pool_size=4, tabu_size=60, delta=20,
                          phi_steps=5, phi_max=1, seed=1, cluster=1, profile_slots=slots)
        r = BatchSolver(j60, [1, 1], cfg).run()
        for i, inst in enumerate(j60):
            want = oracle.orchestrate(inst, 15, 1, 1, 1, delta=20, tabu_size=60, phi_steps=5,
                                      phi_max=1, pool_size=4)
            assert int(r.best_cmax[i]) == want["best_cmax"], ("sized", slots, i)
            assert int(r.evaluations[i]) == want["evaluations"], ("sized", slots, i)
    print("sized profiles ok", flush=True)
    if "K4" not in sections:
        return
    s = BatchSolver(insts, [1] * len(insts), SolveConfig(total_iters=10, workers=1, pool_size=4,
                                                         tabu_size=30, delta=20, phi_steps=5,
                                                         phi_max=1, seed=2))
    s.upload()
    s.pool_init()
    el = torch.zeros((len(insts), s.n_max), dtype=torch.int32, device="cuda")
    ec = torch.zeros(len(insts), dtype=torch.int32, device="cuda")
    s.export_elites(el, ec)
    s.merge_elites(el, ec - 1, 1)
    torch.cuda.synchronize()
    print("K0/K3/K4 ok", flush=True)


ALL = {"K1", "misc", "K2", "K3", "K3L", "sized", "K4"}

if __name__ == "__main__":
    main(set(sys.argv[1:]) or ALL)
