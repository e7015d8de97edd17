#!/usr/bin/env python3
"""Per-step device times of one batch solve repeated K times (GPU box):
pool init and search timed separately with CUDA events, plus the work done,
to find bimodal step times.  usage: tools/step_jitter.py [config] [instances]
[workers] [iters] [steps]"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    import torch
    from paper_1711_04556_b200 import SearchParams, synth
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "j30p"
    ni, wk, it, K = (int(x) for x in (sys.argv[2:6] + ["148", "8", "1000", "40"][len(sys.argv[2:6]):]))
    insts = synth.benchmark_batch(cfgname, ni)
    p = SearchParams.defaults_for(insts[0].n_activities, total_iters=it, workers=wk, seed=0)
    cfg = SolveConfig(total_iters=it, workers=wk, pool_size=p.pool_size, tabu_size=p.tabu_size,
                      delta=p.delta, phi_steps=p.phi_steps, phi_max=p.phi_max, seed=0)
    s = BatchSolver(insts, [1] * len(insts), cfg)
    s.upload()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    rows = []
    for k in range(K + 2):
        s.reset()
        flush.fill_(1)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(st)
        s.pool_init(st)
        e[1].record(st)
        s.search(None, st)
        e[2].record(st)
        torch.cuda.synchronize()
        r = s.collect()
        rows.append({"pool_ms": e[0].elapsed_time(e[1]), "search_ms": e[1].elapsed_time(e[2]),
                     "evals": int(r.evaluations.sum()), "iters": int(r.iterations.sum())})
    rows = rows[2:]
    sm = np.array([x["search_ms"] for x in rows])
    print(json.dumps({"config": cfgname, "search_ms_sorted": sorted(np.round(sm, 2).tolist()),
                      "pool_ms_max": max(x["pool_ms"] for x in rows),
                      "evals": sorted({x["evals"] for x in rows})[:5]}))
    for x in rows:
        if x["search_ms"] > 1.5 * np.median(sm):
            print("outlier", x)


if __name__ == "__main__":
    main()
