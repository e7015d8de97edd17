#!/usr/bin/env python3
"""Per-step times of bench.py's per-config measurement (GPU box), to find a
slow step after the warm-up: j120p solve first (as the headline), then the
j60p TIME per-config solver stepped 6 times."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def steps(cfg, n_inst, workers, iters, k):
    import torch
    from paper_1711_04556_b200 import SearchParams, synth
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    insts = synth.benchmark_batch(cfg, n_inst)
    p = SearchParams.defaults_for(insts[0].n_activities, total_iters=iters, workers=workers, seed=0)
    s = BatchSolver(insts, [1] * n_inst, SolveConfig(total_iters=iters, workers=workers,
                                                     pool_size=p.pool_size, tabu_size=p.tabu_size,
                                                     delta=p.delta, phi_steps=p.phi_steps,
                                                     phi_max=p.phi_max, seed=0))
    s.upload()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    out = []
    for _ in range(k):
        s.reset()
        flush.fill_(1)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(st)
        s.pool_init(st)
        e[1].record(st)
        s.search(stream=st)
        e[2].record(st)
        torch.cuda.synchronize()
        out.append((round(e[0].elapsed_time(e[1]), 1), round(e[1].elapsed_time(e[2]), 1)))
    return out


def main() -> None:
    print("j120p", steps("j120p", 600, 2, 200, 2), flush=True)
    for rep in range(3):
        print("j60p", steps("j60p", 148, 8, 1000, 6), flush=True)


if __name__ == "__main__":
    main()
