#!/usr/bin/env python3
"""Independent search populations sharing the work of one solve (GPU box).

Launched with torchrun (gloo plumbing; every rank on the same GPU when the
box has one):

    python -m torch.distributed.run --nproc-per-node K --master-addr 127.0.0.1 \
        --master-port 29511 tools/populations.py --exchange peer --iters 1000

Each of the K ranks solves the same Gen-P batch with I_total / K iterations
per instance and its own seeds; the exchange is "peer" (live, peer memory),
"epochs" (all_gather between E search epochs: the GPU drains E-1 times) or
"none".  The answer per instance is the best over the ranks.  Prints one JSON
line (rank 0): mean CPM deviation of that answer, the wall time (max over
ranks, host clock around pool init + search), evaluations, exchange counters.
With K = 1 and --exchange epochs --epochs E it measures the cost of E-1
epoch drains on one population.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="j120p")
    ap.add_argument("--instances", type=int, default=148)
    ap.add_argument("--workers", type=int, default=2)
    ap.add_argument("--iters", type=int, default=1000, help="I_total of the whole solve")
    ap.add_argument("--exchange", default="peer", choices=["peer", "epochs", "none"])
    ap.add_argument("--epochs", type=int, default=4)
    ap.add_argument("--poll-every", type=int, default=4)
    ap.add_argument("--repeats", type=int, default=2)
    args = ap.parse_args()

    import torch
    import torch.distributed as dist
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    if ws > 1:
        dist.init_process_group("gloo")
    from paper_1711_04556_b200 import SearchParams, decide_static, extract_features, synth
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    from paper_1711_04556_b200.population import EliteExchange, PeerExchange, run_epochs

    insts = synth.benchmark_batch(args.config, args.instances)
    modes = [int(decide_static(extract_features(x))) for x in insts]
    per_rank = max(1, args.iters // ws)
    p = SearchParams.defaults_for(insts[0].n_activities, total_iters=per_rank,
                                  workers=args.workers, seed=1000 * rank)
    cfg = SolveConfig(total_iters=per_rank, workers=p.workers, pool_size=p.pool_size,
                      tabu_size=p.tabu_size, delta=p.delta, phi_steps=p.phi_steps,
                      phi_max=p.phi_max, seed=p.seed)
    solver = BatchSolver(insts, modes, cfg)
    exchange, peer = None, None
    if args.exchange == "peer" and ws > 1:
        peer = PeerExchange(solver, poll_every=args.poll_every)
        solver.peer = peer
    elif args.exchange == "epochs" and ws > 1:
        exchange = EliteExchange(solver, len(insts), solver.n_max)
    epochs = args.epochs if args.exchange == "epochs" else 1
    solver.upload()
    walls, devs, evals = [], [], []
    for rep in range(args.repeats + 1):          # the first run warms up
        solver.reset()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        solver.pool_init()
        run_epochs(solver, per_rank, epochs, exchange)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        res = solver.collect()
        best = torch.tensor(res.best_cmax, dtype=torch.int64)
        ev = torch.tensor([int(res.evaluations.sum())], dtype=torch.int64)
        wt = torch.tensor([wall], dtype=torch.float64)
        if ws > 1:
            dist.all_reduce(best, op=dist.ReduceOp.MIN)
            dist.all_reduce(ev, op=dist.ReduceOp.SUM)
            dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        if rep:
            walls.append(float(wt.item()))
            evals.append(int(ev.item()))
            devs.append(float(np.mean(100.0 * (best.numpy() - res.critical_path)
                                      / res.critical_path)))
    if rank == 0:
        print(json.dumps({"populations": ws, "exchange": args.exchange, "epochs": epochs,
                          "config": args.config, "instances": len(insts),
                          "iters_total": args.iters, "iters_per_population": per_rank,
                          "workers_per_instance": args.workers,
                          "wall_s": float(np.mean(walls)), "cpm_dev": float(np.mean(devs)),
                          "schedules_per_s": float(np.sum(evals) / np.sum(walls)),
                          **({"peer": peer.counters()} if peer else {})}), flush=True)
    if peer is not None:
        dist.barrier()
        peer.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
