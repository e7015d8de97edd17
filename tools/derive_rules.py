#!/usr/bin/env python3
"""Re-derive the static evaluation-mode rules for the B200 (SURVEY.md sec. 8f
item 3; the paper's method): time the search kernel in both
modes on instance families that vary the two features the reference's rules
test (max capacity, average duration) and report which mode evaluates more
schedules per second.  Writes profiles/r2/mode_rules_b200.json (round 1:
profiles/r1/).

usage: python tools/derive_rules.py [--instances 148] [--iters 100]"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", type=int, default=148)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--n", type=int, default=120)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r2" / "mode_rules_b200.json"))
    args = ap.parse_args()
    import torch
    from paper_1711_04556_b200 import SearchParams, extract_features, synth
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    rows = []
    for cap_lo, cap_hi in ((2, 6), (4, 10), (10, 16), (16, 32), (40, 80)):
        for max_dur in (10, 20, 40):
            insts = [synth.random_instance(args.n, 4, seed=s, cap_lo=cap_lo, cap_hi=cap_hi,
                                           max_dur=max_dur, demand_density=0.5)
                     for s in range(args.instances)]
            feats = [extract_features(x) for x in insts]
            rec = {"cap": [cap_lo, cap_hi], "max_dur": max_dur,
                   "avg_duration": float(np.mean([f.avg_duration for f in feats])),
                   "max_capacity": float(np.mean([f.max_capacity for f in feats]))}
            for mode, name in ((1, "time"), (0, "capacity")):
                p = SearchParams.defaults_for(insts[0].n_activities, total_iters=args.iters,
                                              workers=2, seed=0)
                cfg = SolveConfig(total_iters=args.iters, workers=2, pool_size=p.pool_size,
                                  tabu_size=p.tabu_size, delta=p.delta, phi_steps=p.phi_steps,
                                  phi_max=p.phi_max, seed=0)
                s = BatchSolver(insts, [mode] * len(insts), cfg)
                s.run()                      # warm-up
                s.reset()
                r = s.run()
                torch.cuda.synchronize()
                rec[name] = {"sched_per_s": float(r.evaluations.sum() / (r.device_ms * 1e-3)),
                             "cpm_dev": float(np.mean(100.0 * (r.best_cmax - r.critical_path)
                                                      / r.critical_path))}
            rec["faster"] = "capacity" if rec["capacity"]["sched_per_s"] > rec["time"]["sched_per_s"] else "time"
            rows.append(rec)
            print(f"cap {cap_lo}-{cap_hi} dur<= {max_dur}: TIME {rec['time']['sched_per_s']/1e6:8.2f} M/s "
                  f"(dev {rec['time']['cpm_dev']:6.1f}%)  CAP {rec['capacity']['sched_per_s']/1e6:8.2f} M/s "
                  f"(dev {rec['capacity']['cpm_dev']:6.1f}%)  -> {rec['faster']}", flush=True)
    out = Path(args.out)
    out.write_text(json.dumps({"n": args.n, "instances": args.instances, "iters": args.iters,
                               "rows": rows}, indent=1))
    print("wrote", out)


if __name__ == "__main__":
    main()
