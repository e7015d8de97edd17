#!/usr/bin/env python3
"""Benchmark: evaluated schedules/sec of the B200 tabu search (BASELINE.json).

One "step" = one full on-device solve of a batch of synthetic j120-shape
instances: by default "Gen-P", 600 PSPLIB-shape instances over PSPLIB j120's
(NC, RF, RS) parameter grid (synth.progen_instance; PSPLIB itself is offline),
or "Gen-R", the reference's own benchmark recipe (--config j120).  Pool
initialisation (FBI), then the persistent search with the working set in HBM,
per-instance evaluation mode picked by the paper's static rules (TIME for
these configs).  value = evaluated schedules (the reference's counting rule: pool +
per-adoption + every neighbourhood evaluation) / device time of the step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 (torchrun, one rank per GPU): every rank runs an independent search
population on the same instances (seed offset by rank); between search
epochs the populations exchange their elites with one NCCL all_gather over
NVLink and merge them into their working sets (weak scaling).

--impl reference times the reference algorithm on the host cores: the C port
of the reference's numba path (oracle/, bit-exact with the reference), all
host threads, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIG = "j120p"
METRIC = "evaluated schedules/sec at 1/2/4/8 B200, j120-shape; mean % dev from CPM bound"


def parse():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=CONFIG,
                    choices=["j30", "j60", "j120", "act300", "j30p", "j60p", "j120p"],
                    help="Gen-R (reference benchmark recipe) or Gen-P (*p: PSPLIB grid)")
    ap.add_argument("--instances", type=int, default=600,
                    help="instances per batch (step); 600 = the size of PSPLIB's j120 set "
                         "(PAPER.md:772)")
    ap.add_argument("--workers", type=int, default=2, help="CTAs (search workers) per instance")
    ap.add_argument("--iters", type=int, default=1000, help="I_total per instance")
    ap.add_argument("--epochs", type=int, default=2,
                    help="search epochs with an elite exchange between them (N > 1); every "
                         "epoch boundary drains the GPU once")
    ap.add_argument("--group", type=int, default=None, help="TIME lanes per schedule")
    ap.add_argument("--threads", type=int, default=0, help="threads per CTA (0 = auto)")
    ap.add_argument("--mode", default="rule", choices=["rule", "time", "capacity"],
                    help="evaluation mode: the static rules (default) or forced")
    ap.add_argument("--cap-group", type=int, default=None, choices=[32, 1],
                    help="CAPACITY evaluator: 32 = warp, 1 = thread per schedule (default auto)")
    ap.add_argument("--full-sgs", action="store_true",
                    help="evaluate every swap by a full SGS (no prefix reuse)")
    ap.add_argument("--no-steal", action="store_true",
                    help="fixed worker-to-instance mapping (no tail balancing)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target CPU time of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-quality", action="store_true",
                    help="skip the fixed-wall-clock CPM-deviation comparison")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# helpers

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        if self.path and os.path.exists(self.path):
            for line in Path(self.path).read_text().splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) == 6 and parts[0].isdigit():
                    rows.append(parts)
            os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(int(r[0]) for r in rows),
                "sm_max_mhz": max(int(r[1]) for r in rows), "reasons": reasons,
                "samples": len(rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def work_per_schedule(cfg: str) -> dict:
    path = ROOT / "profiles" / "work_per_schedule.json"
    return json.loads(path.read_text())[cfg]


# ---------------------------------------------------------------------------
# reference arm / cpu baseline (the C port of the reference, oracle/)

def workload_name(cfg: str) -> str:
    if cfg.endswith("p"):
        return (f"{cfg[:-1]}-shape Gen-P batch (PSPLIB {cfg[:-1]} NC/RF/RS grid, "
                f"ProGen-style synthetic)")
    return f"{cfg}-shape Gen-R batch (reference benchmark recipe)"


SAMPLE_STRIDE = 157  # coprime with the batch sizes used: the sample spreads over the batch


def sample_index(k: int, batch: int) -> int:
    """Batch index of the k-th CPU-sample instance (spread over Gen-P's grid cells)."""
    return (k * SAMPLE_STRIDE) % batch


def cpu_sample(cfg: str, iters: int, target_s: float, threads: int, batch: int,
               seed: int = 0) -> dict:
    """Time the reference algorithm (C port, `threads` workers per instance,
    instances one after another like `rcpsp-tabu bench`) on a bounded sample
    of the workload: instances sample_index(0..) of the step's batch.  Returns
    schedules/sec, the sample and the CPM deviation."""
    import oracle
    from paper_1711_04556_b200 import extract_features, decide_static, synth
    evals = 0
    wall = 0.0
    devs = []
    k = 0
    while True:
        inst = synth.benchmark_batch(cfg, 1, first_seed=sample_index(k, batch))[0]
        mode = int(decide_static(extract_features(inst)))
        r = oracle.orchestrate(inst, iters, threads, seed, mode)
        evals += r["evaluations"]
        wall += r["wall_time"]
        devs.append(100.0 * (r["best_cmax"] - r["critical_path"]) / r["critical_path"])
        k += 1
        if wall >= target_s or k >= 64:
            break
    return {"value": evals / wall, "evaluations": evals, "wall": wall, "instances": k,
            "cpm_dev": float(np.mean(devs)), "iters": iters, "threads": threads}


def run_reference(args, ws: int, rank: int) -> None:
    if rank != 0:
        return
    import oracle
    cores = oracle.cpu_count()
    iters = args.iters
    per_step = max(2.0, args.cpu_seconds / max(1, args.steps))
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_sample(args.config, min(iters, 50), 0.5, cores, args.instances)
    vals, evals, walls, devs = [], 0, 0.0, []
    for _ in range(args.steps):
        r = cpu_sample(args.config, iters, per_step, cores, args.instances)
        vals.append(r["value"])
        evals += r["evaluations"]
        walls += r["wall"]
        devs.append(r["cpm_dev"])
    value = evals / walls
    sample = (f"{r['instances']} {args.config} instances of the {args.instances}-instance batch "
              f"(indices k*{SAMPLE_STRIDE} mod {args.instances}), I_total={iters}, "
              f"{cores} worker threads per instance, instances solved one after another "
              f"(~{per_step:.0f} s per step)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "schedules/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * walls / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"{workload_name(args.config)}, reference C port on host",
                   "iters_per_instance": iters, "cpm_dev": float(np.mean(devs))},
        "cpu_baseline": {"value": value, "unit": "schedules/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "schedules/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm

def quality_leg(args, insts, modes, cb: dict) -> dict:
    """Mean % deviation from the CPM bound at a fixed wall-clock budget: the
    CPU sample's instances solved on the GPU within the wall time the
    reference algorithm took for them on all host cores.  The search stops on
    the device clock (SolveConfig.time_limit_s -> %globaltimer): no new grant
    and no further iteration once the budget is spent."""
    import torch
    from paper_1711_04556_b200 import SearchParams
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    K = int(cb["instances"])
    pick = [sample_index(k, len(insts)) for k in range(K)]  # the CPU sample's instances
    qi, qm = [insts[i] for i in pick], [modes[i] for i in pick]
    # every CTA must be resident from the start (2 per SM): a wave that starts
    # after the clock stopped the search would never run
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    workers = max(1, (2 * sms) // K)
    budget_iters = 10 ** 7                                  # never reached: the clock stops it
    p = SearchParams.defaults_for(qi[0].n_activities, total_iters=budget_iters, workers=workers,
                                  seed=0)
    cfg = SolveConfig(total_iters=budget_iters, workers=workers, pool_size=p.pool_size,
                      tabu_size=p.tabu_size, delta=p.delta, phi_steps=p.phi_steps,
                      phi_max=p.phi_max, seed=0, group=args.group, threads=args.threads,
                      time_limit_s=0.97 * cb["wall"])
    res = BatchSolver(qi, qm, cfg).run()
    torch.cuda.synchronize()
    dev = float(np.mean(100.0 * (res.best_cmax - res.critical_path) / res.critical_path))
    return {"wall_budget_s": cb["wall"], "instances": K,
            "cpu": {"cpm_dev": cb["cpm_dev"], "iters_per_instance": cb["iters"],
                    "kind": "port", "workers_per_instance": cb.get("threads")},
            "gpu": {"cpm_dev": dev, "iters_per_instance": float(np.mean(res.iterations)),
                    "workers_per_instance": workers, "device_s": res.device_ms * 1e-3,
                    "stop": "device clock (%globaltimer), 97 % of the budget"}}


def main() -> None:
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return

    import torch
    import torch.distributed as dist

    # one rank per GPU; BENCH_DIST_BACKEND=gloo (testing only) lets several
    # ranks share one GPU to exercise the N > 1 path on a single-GPU box
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    dev_index = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    from paper_1711_04556_b200 import SearchParams, decide_static, extract_features, synth
    from paper_1711_04556_b200.device import (BatchSolver, SolveConfig, smem_bandwidth)
    from paper_1711_04556_b200.population import EliteExchange, run_epochs

    insts = synth.benchmark_batch(args.config, args.instances)
    if args.mode == "rule":
        modes = [int(decide_static(extract_features(x))) for x in insts]
    else:
        modes = [1 if args.mode == "time" else 0] * len(insts)
    p = SearchParams.defaults_for(insts[0].n_activities, total_iters=args.iters,
                                  workers=args.workers, seed=1000 * rank)
    cfg = SolveConfig(total_iters=p.total_iters, workers=p.workers, pool_size=p.pool_size,
                      tabu_size=p.tabu_size, delta=p.delta, phi_steps=p.phi_steps,
                      phi_max=p.phi_max, seed=p.seed, group=args.group, threads=args.threads,
                      steal=not args.no_steal, full_sgs=args.full_sgs,
                      cap_group=args.cap_group)
    solver = BatchSolver(insts, modes, cfg)
    solver.upload()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")  # > L2
    epochs = args.epochs if ws > 1 else 1
    n_max = solver.n_max
    I = len(insts)
    exchange = EliteExchange(solver, I, n_max) if ws > 1 else None

    def one_step(timed_search: list | None = None) -> None:
        solver.pool_init(stream)
        marks: list = []

        def mark(begin: bool) -> None:
            if timed_search is None:
                return
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            marks.append(ev)
            if not begin:
                timed_search.append((marks[-2], marks[-1]))

        run_epochs(solver, args.iters, epochs, exchange, stream, on_search=mark)

    for _ in range(args.warmup):
        solver.reset()
        one_step()
    torch.cuda.synchronize()

    launches0 = solver.launches
    step_ms, search_ms, evals, search_evals, devs = [], [], 0, 0, []
    sgs_steps, iters_done = 0, 0
    with ClockSampler(dev_index) as clocks:
        for _ in range(args.steps):
            solver.reset()
            flush.fill_(1)                       # L2 flush between timed steps
            torch.cuda.synchronize()
            if ws > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            spans: list = []
            e0.record(stream)
            one_step(spans)
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            search_ms.append(sum(a.elapsed_time(b) for a, b in spans))
            res = solver.collect()
            evals += int(res.evaluations.sum())
            search_evals += int((res.evaluations - res.pool_evaluations).sum())
            sgs_steps += res.sgs_steps
            iters_done += int(res.iterations.sum())
            devs.append(float(np.mean(100.0 * (res.best_cmax - res.critical_path)
                                      / res.critical_path)))
    launches = solver.launches - launches0
    clk = clocks.summary()

    # whole-job aggregation: evaluations summed over ranks, time = max over ranks
    tot_ms = sum(step_ms)
    if ws > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        ev = torch.tensor([evals], dtype=torch.float64, device="cuda")
        dist.all_reduce(ev, op=dist.ReduceOp.SUM)
        evals_all = int(ev.item())
    else:
        evals_all = evals
    value = evals_all / (tot_ms * 1e-3)

    # e2e through the public batch API: pinned H2D of the inputs + solve + D2H
    e2e_vals, h2d, d2h = [], 0, 0
    for _ in range(args.e2e_steps):
        solver.reset()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        h2d = solver.upload(pinned=True)
        one_step()
        res = solver.collect()
        t1 = time.perf_counter()
        d2h = (res.best_cmax.nbytes + res.best_order.nbytes + solver.ws_hdr.numel() * 8
               + solver.w_stats.numel() * 8)
        e2e_vals.append((int(res.evaluations.sum()), t1 - t0))
    e_ev = sum(v for v, _ in e2e_vals)
    e_t = sum(t for _, t in e2e_vals)
    if ws > 1:
        tt = torch.tensor([e_t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e_t = float(tt.item())
        ee = torch.tensor([e_ev], dtype=torch.float64, device="cuda")
        dist.all_reduce(ee, op=dist.ReduceOp.SUM)
        e_ev = int(ee.item())
    e2e = e_ev / e_t if e_t > 0 else 0.0

    if rank != 0:
        dist.destroy_process_group()
        return

    # roofline of the dominant kernel (k_solve): algorithmic bytes of the
    # schedules it evaluated / its measured duration, vs measured SMEM bandwidth
    W = work_per_schedule(args.config)
    n_act = insts[0].n_activities
    mode_key = "time" if modes.count(1) >= modes.count(0) else "cap"
    bytes_per_sched = W[mode_key]["bytes"]
    s_ms = sum(search_ms)
    achieved = search_evals * bytes_per_sched / (s_ms * 1e-3) / 1e9
    peak = smem_bandwidth()
    peaks = {}
    pk = ROOT / "MEASURED_PEAKS.json"
    if pk.exists():
        peaks = json.loads(pk.read_text())
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    # DRAM traffic of the dominant kernel: ncu bytes per evaluated schedule
    # (profiles/ncu_traffic.json) x the schedules one timed k_solve launch evaluated
    traffic = None
    tr = ROOT / "profiles" / "ncu_traffic.json"
    if tr.exists():
        rec = json.loads(tr.read_text()).get(args.config)
        if rec:
            traffic = rec["dram_bytes_per_schedule"] * search_evals / (args.steps * epochs)

    line = {
        "metric": METRIC, "value": value, "unit": "schedules/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": {"workload": f"{workload_name(args.config)}, static-rule mode selection",
                   "instances": I,
                   "workers_per_instance": args.workers, "iters_per_instance": args.iters,
                   "pool_size": p.pool_size, "delta": p.delta, "tabu_size": p.tabu_size,
                   "modes": {"TIME": modes.count(1), "CAPACITY": modes.count(0)},
                   "epochs": epochs, "cpm_dev": float(np.mean(devs)),
                   "evaluations_per_step": evals // args.steps,
                   "iterations_per_step": iters_done // args.steps,
                   "l2": "256 MiB buffer written between timed steps",
                   "parallelism": f"{ws} independent populations" + (
                       ", NCCL all_gather elite exchange" if ws > 1 else "")},
        "roofline": {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "kernel": "k_solve", "bytes_per_schedule": bytes_per_sched,
                     "bytes_basis": "reference full-SGS element touches x 4 B per evaluated "
                                    "schedule (profiles/work_per_schedule.json)",
                     "sgs_steps_per_schedule": sgs_steps / max(1, search_evals),
                     "executed_step_fraction": sgs_steps / max(1, search_evals * n_act),
                     "peak_source": "measured in this run: rcpsp_smem_probe (LDS.128 stream)",
                     "hbm_peak_gbs": hbm_peak,
                     "hbm_achieved_gbs": (traffic * args.steps * epochs / (s_ms * 1e-3) / 1e9
                                          if traffic is not None else None)},
        "clocks": clk,
        "gpu_launches": launches,
        "e2e": {"value": e2e, "unit": "schedules/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
    }
    if ws == 1 and not args.no_cpu_baseline:
        import oracle
        cores = oracle.cpu_count()
        cb = cpu_sample(args.config, args.iters, args.cpu_seconds, cores, args.instances)
        line["cpu_baseline"] = {
            "value": cb["value"], "unit": "schedules/s", "cores": cores, "kind": "port",
            "sample": f"{cb['instances']} {args.config} instances of the batch "
                      f"(indices k*{SAMPLE_STRIDE} mod {args.instances}), "
                      f"I_total={cb['iters']}, {cores} worker threads each, "
                      f"{cb['wall']:.1f} s; cpm_dev {cb['cpm_dev']:.2f}%"}
        if not args.no_quality:
            line["quality"] = quality_leg(args, insts, modes, cb)
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
