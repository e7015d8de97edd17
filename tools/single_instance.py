#!/usr/bin/env python3
"""Single-instance solve latency (the orchestrate() drop-in): one j120 Gen-P
instance, B workers, I_total iterations; one CTA per worker vs a thread-block
cluster per worker (auto: up to 8 CTAs), against the reference algorithm (C
port) with B host threads.  usage: single_instance.py [iters] [seed]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 305
    import torch
    import oracle
    from paper_1711_04556_b200 import SearchParams, synth
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    inst = synth.benchmark_batch("j120p", 1, first_seed=seed)[0]
    for B in (1, 16):
        p = SearchParams.defaults_for(inst.n_activities, total_iters=iters, workers=B, seed=0)
        for cl in (1, None):
            cfg = SolveConfig(total_iters=iters, workers=B, pool_size=p.pool_size,
                              tabu_size=p.tabu_size, delta=p.delta, phi_steps=p.phi_steps,
                              phi_max=p.phi_max, seed=0, cluster=cl)
            s = BatchSolver([inst], [1], cfg)
            s.run()
            s.reset()
            r = s.run()
            torch.cuda.synchronize()
            print(f"B={B:2d} cluster={'auto' if cl is None else cl:>4}: {r.device_ms:8.1f} ms "
                  f"device, best {int(r.best_cmax[0])}, {int(r.evaluations[0]) / (r.device_ms * 1e-3) / 1e6:7.2f} M sched/s",
                  flush=True)
        t = time.perf_counter()
        o = oracle.orchestrate(inst, iters, B, 0, 1)
        w = time.perf_counter() - t
        print(f"B={B:2d} reference algorithm (C port, {B} threads): {1e3 * w:8.1f} ms, best "
              f"{o['best_cmax']}, {o['evaluations'] / w / 1e6:7.2f} M sched/s", flush=True)


if __name__ == "__main__":
    main()
