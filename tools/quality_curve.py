#!/usr/bin/env python3
"""Mean % deviation from the critical-path bound at fixed wall-clock budgets:
K Gen-P j120 instances (spread over the PSPLIB grid); the reference algorithm
(C port, all host threads) gets T seconds per instance (iterations calibrated
from a short timed run), the B200 solves all K at once within K*T seconds on
the device clock.  usage: quality_curve.py [K] [T1 T2 ...]"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    budgets = [float(x) for x in sys.argv[2:]] or [0.25, 1.0, 4.0]
    import torch
    import oracle
    from paper_1711_04556_b200 import SearchParams, synth
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    insts = [synth.benchmark_batch("j120p", 1, first_seed=(k * 157) % 600)[0] for k in range(K)]
    cpm = np.array([oracle.critical_path(x) for x in insts], dtype=float)
    cores = oracle.cpu_count()
    # iterations per second of the port on each instance (all host threads)
    rates = []
    for x in insts:
        t = time.perf_counter()
        oracle.orchestrate(x, 200, cores, 0, 1)
        rates.append(200 / (time.perf_counter() - t))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    workers = max(1, (2 * sms) // K)
    print(f"K={K} instances, {cores} host threads, GPU {workers} workers per instance")
    print(f"{'T/instance':>10} {'CPU dev %':>10} {'CPU iters':>10} {'GPU dev %':>10} {'GPU iters':>10}")
    for T in budgets:
        devs, its = [], []
        for x, r, c in zip(insts, rates, cpm):
            it = max(10, int(r * T))
            o = oracle.orchestrate(x, it, cores, 0, 1)
            devs.append(100 * (o["best_cmax"] - c) / c)
            its.append(it)
        p = SearchParams.defaults_for(122, total_iters=10 ** 7, workers=workers, seed=0)
        cfg = SolveConfig(total_iters=10 ** 7, workers=workers, pool_size=p.pool_size,
                          tabu_size=p.tabu_size, delta=p.delta, phi_steps=p.phi_steps,
                          phi_max=p.phi_max, seed=0, time_limit_s=K * T)
        res = BatchSolver(insts, [1] * K, cfg).run()
        torch.cuda.synchronize()
        gdev = 100 * (res.best_cmax - cpm) / cpm
        print(f"{T:10.2f} {np.mean(devs):10.2f} {np.mean(its):10.0f} {np.mean(gdev):10.2f} "
              f"{np.mean(res.iterations):10.0f}", flush=True)


if __name__ == "__main__":
    main()
