#!/usr/bin/env python3
"""Step times of a j60p batch solve right after the GPU sat idle for a few
seconds (GPU box): does the first step after an idle period run slow?"""
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    import torch
    from paper_1711_04556_b200 import SearchParams, synth
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    insts = synth.benchmark_batch("j60p", 148)
    p = SearchParams.defaults_for(insts[0].n_activities, total_iters=1000, workers=8, seed=0)
    s = BatchSolver(insts, [1] * 148, SolveConfig(total_iters=1000, workers=8, pool_size=p.pool_size,
                                                  tabu_size=p.tabu_size, delta=p.delta,
                                                  phi_steps=p.phi_steps, phi_max=p.phi_max, seed=0))
    s.upload()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    for idle in (0, 0, 2, 5, 0, 5, 10, 0):
        time.sleep(idle)
        clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu",
                              "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
        row = []
        for _ in range(4):
            s.reset()
            flush.fill_(1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            s.pool_init(st)
            s.search(None, st)
            e1.record(st)
            torch.cuda.synchronize()
            row.append(round(e0.elapsed_time(e1), 1))
        print(f"idle {idle:2d}s before: clocks {clk:30s} steps ms {row}", flush=True)


if __name__ == "__main__":
    main()
