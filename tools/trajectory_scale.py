#!/usr/bin/env python3
"""Trajectory parity at scale (GPU box): B = 1 searches of many instances in
one batched solve (k_solve, one CTA per instance, every instance's own seed)
against the oracle's orchestrate (cooperation.py:237-302) with the same pinned
mode and parameters -- traces, evaluations, exchanges, diversifications,
forced picks and best makespans compared.  Prints one JSON line per config
and mode.  usage: python tools/trajectory_scale.py [scale]"""
from __future__ import annotations

import json
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import oracle  # noqa: E402
from paper_1711_04556_b200 import SearchParams, synth  # noqa: E402
from paper_1711_04556_b200.device import BatchSolver, SolveConfig  # noqa: E402


def run(cfg, n_inst, iters, mode, seed):
    insts = synth.benchmark_batch(cfg, n_inst, first_seed=900)
    p = SearchParams.defaults_for(insts[0].n_activities, total_iters=iters, workers=1, seed=seed)
    sc = SolveConfig(total_iters=iters, workers=1, pool_size=p.pool_size, tabu_size=p.tabu_size,
                     delta=p.delta, phi_steps=p.phi_steps, phi_max=p.phi_max, seed=seed,
                     collect_trace=True)
    t0 = time.time()
    r = BatchSolver(insts, [mode] * len(insts), sc).run()
    t_gpu = time.time() - t0

    def want(inst):
        return oracle.orchestrate(inst, iters, 1, seed, mode, delta=p.delta, tabu_size=p.tabu_size,
                                  phi_steps=p.phi_steps, phi_max=p.phi_max,
                                  pool_size=p.pool_size, collect_trace=True)
    t0 = time.time()
    with ThreadPoolExecutor(max_workers=16) as ex:
        ws = list(ex.map(want, insts))
    t_cpu = time.time() - t0
    bad, iters_cmp, divs = [], 0, 0
    for i, w in enumerate(ws):
        got = (int(r.best_cmax[i]), int(r.evaluations[i]), int(r.exchanges[i]),
               int(r.diversifications[i]), int(r.forced[i]),
               [t.tolist() for t in r.traces[i]])
        exp = (w["best_cmax"], w["evaluations"], w["exchanges"], w["diversifications"],
               w["forced_tabu_picks"], [t.tolist() for t in w["traces"]])
        iters_cmp += sum(len(t) for t in w["traces"])
        divs += w["diversifications"]
        if got != exp:
            bad.append(i)
    return {"config": cfg, "mode": "TIME" if mode == 1 else "CAPACITY", "instances": len(insts),
            "iterations_per_instance": iters, "trace_points_compared": iters_cmp,
            "diversifications": divs, "mismatching_instances": bad,
            "gpu_s": round(t_gpu, 1), "oracle_s": round(t_cpu, 1)}


def main() -> None:
    k = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    plan = [("j30p", 128, 600), ("j60p", 96, 400), ("j120p", 48, 250), ("act300", 16, 40)]
    for cfg, n_inst, iters in plan:
        for mode in (1, 0):
            print(json.dumps(run(cfg, max(1, int(n_inst * k)), iters, mode, seed=7)), flush=True)


if __name__ == "__main__":
    main()
