#!/usr/bin/env python3
"""Long B = 1 trajectories on the headline workload (Gen-P j120), pinned.

Run in the build container:

    python tests/golden/make_long_trajectories.py

For each case below the CPU oracle (oracle/, the C restatement) runs the whole
`orchestrate` (pool of 16, B = 1, seeded, pinned mode) and, when the reference
package is importable (/root/reference), the REFERENCE itself (rcpsp_tabu,
numba backend) runs the same solve; the two must agree on every field and on
the full per-iteration trace, else this script fails.  The fixture keeps the
trace as a sha256 of its int32 bytes plus its length and the chunk lengths
(the exchange structure), the counters and the best schedule's starts, so
tests/test_gpu_long.py can compare the device trajectory without the
reference on the GPU box.  The cases were chosen (probe, this script's git
history) so that diversification and forced tabu picks both occur:
1000-1500 iterations, default parameters or a small swap distance delta.
"""

from __future__ import annotations

import hashlib
import json
import sys
from multiprocessing import Pool
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import oracle  # noqa: E402
from paper_1711_04556_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent / "long_trajectories.json"
REF = Path("/root/reference/pkg/src")

# (config, batch index, I_total, seed, mode, delta, tabu_size, phi_max)
CASES = [
    ("j120p", 157, 1500, 0, 1, 60, 800, 3),   # default parameters, diversifies
    ("j120p", 471, 1200, 0, 1, 2, 800, 1),    # forced picks + diversification
    ("j120p", 157, 1200, 0, 1, 2, 800, 1),
    ("j120p", 471, 1000, 0, 0, 2, 800, 1),    # CAPACITY mode
    ("j120p", 28, 1200, 0, 1, 2, 800, 1),
]


def digest(chunks) -> tuple[str, int]:
    flat = np.concatenate([np.asarray(c, np.int32) for c in chunks]) if chunks else \
        np.zeros(0, np.int32)
    return hashlib.sha256(flat.astype("<i4").tobytes()).hexdigest(), int(len(flat))


def run_oracle(case):
    cfg, idx, iters, seed, mode, delta, tabu, phi_max = case
    inst = synth.benchmark_batch(cfg, 1, first_seed=idx)[0]
    r = oracle.orchestrate(inst, iters, 1, seed, mode, delta=delta, tabu_size=tabu,
                           phi_max=phi_max, pool_size=16, collect_trace=True)
    sha, ln = digest(r["traces"])
    return {"config": cfg, "index": idx, "total_iters": iters, "seed": seed, "mode": mode,
            "delta": delta, "tabu_size": tabu, "phi_max": phi_max, "pool_size": 16,
            "best_cmax": r["best_cmax"], "evaluations": r["evaluations"],
            "exchanges": r["exchanges"], "diversifications": r["diversifications"],
            "forced_tabu_picks": r["forced_tabu_picks"], "iterations": r["iterations"],
            "critical_path": r["critical_path"], "trace_sha256": sha, "trace_len": ln,
            "chunk_lens": [len(c) for c in r["traces"]],
            "best_order": [int(x) for x in r["best_order"]]}


def run_reference(rec) -> dict:
    sys.path.insert(0, str(REF))
    import rcpsp_tabu as R
    from rcpsp_tabu import kernels
    assert kernels.BACKEND == "numba", kernels.BACKEND
    ours = synth.benchmark_batch(rec["config"], 1, first_seed=rec["index"])[0]
    inst = R.make_instance(ours.name, ours.durations.tolist(), ours.capacities.tolist(),
                           ours.demands.tolist(), [list(s) for s in ours.successors])
    p = R.SearchParams.defaults_for(inst.n_activities, total_iters=rec["total_iters"],
                                    workers=1, seed=rec["seed"], mode=R.EvalMode(rec["mode"]),
                                    collect_trace=True, delta=rec["delta"],
                                    tabu_size=rec["tabu_size"], phi_max=rec["phi_max"],
                                    pool_size=rec["pool_size"])
    st = R.orchestrate(inst, p)
    sha, ln = digest(st.traces)
    return {"best_cmax": st.best_cmax, "evaluations": st.evaluations,
            "exchanges": st.exchanges, "diversifications": st.diversifications,
            "forced_tabu_picks": st.forced_tabu_picks, "iterations": st.iterations,
            "critical_path": st.critical_path, "trace_sha256": sha, "trace_len": ln,
            "chunk_lens": [len(c) for c in st.traces], "starts": st.schedule.starts.tolist()}


def main() -> None:
    with Pool(min(8, len(CASES))) as pool:
        recs = pool.map(run_oracle, CASES)
    have_ref = (REF / "rcpsp_tabu").is_dir()
    for rec in recs:
        if have_ref:
            ref = run_reference(rec)
            for k, v in ref.items():
                if k != "starts":
                    assert rec[k] == v, (rec["index"], k, rec[k], v)
            rec["starts"] = ref["starts"]
        rec["verified_by_reference"] = have_ref
        print({k: rec[k] for k in ("index", "mode", "delta", "best_cmax", "evaluations",
                                   "exchanges", "diversifications", "forced_tabu_picks")},
              flush=True)
    OUT.write_text(json.dumps({"_doc": __doc__.strip().splitlines()[0], "cases": recs}) + "\n")


if __name__ == "__main__":
    main()
