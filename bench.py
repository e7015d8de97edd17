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
    ap.add_argument("--exchange", default="peer", choices=["peer", "epochs"],
                    help="N > 1 elite exchange: 'peer' = live, the search kernels read each "
                         "other's outboxes over peer memory (CUDA IPC / NVLink), no pause; "
                         "'epochs' = all_gather between search epochs (drains the GPU)")
    ap.add_argument("--epochs", type=int, default=2,
                    help="search epochs with an elite exchange between them (--exchange "
                         "epochs, N > 1)")
    ap.add_argument("--poll-every", type=int, default=4,
                    help="--exchange peer: exchanges of a worker between outbox polls")
    ap.add_argument("--group", type=int, default=None, help="TIME lanes per schedule")
    ap.add_argument("--threads", type=int, default=0, help="threads per CTA (0 = auto)")
    ap.add_argument("--mode", default="rule", choices=["rule", "time", "capacity"],
                    help="evaluation mode: the static rules (default) or forced")
    ap.add_argument("--cap-group", type=int, default=None, choices=[32, 1],
                    help="CAPACITY evaluator: 32 = warp, 1 = thread per schedule (default auto)")
    ap.add_argument("--full-sgs", action="store_true",
                    help="evaluate every swap by a full SGS (no prefix reuse)")
    ap.add_argument("--profile-slots", type=int, default=None,
                    help="TIME per-warp profile slots: default sized by a makespan bound when "
                         "that keeps more warps resident; 0 = always the horizon")
    ap.add_argument("--no-steal", action="store_true",
                    help="fixed worker-to-instance mapping (no tail balancing)")
    ap.add_argument("--cpu-sample", type=int, default=None,
                    help="instances in the CPU sample (default synth.CPU_SAMPLE = 30): "
                         "cpu_baseline and the reference arm time the same ones")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true",
                    help="skip the j60p / act300 (TIME and CAPACITY) entries")
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


def host_cpu() -> dict:
    """Host CPU model (lscpu 'Model name') and the cores this process may use."""
    import oracle
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.split(":")[0].strip() == "Model name":
                model = line.split(":", 1)[1].strip()
                break
    except (OSError, subprocess.SubprocessError):
        pass
    if model is None and Path("/proc/cpuinfo").exists():
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    return {"model": model, "cores": oracle.cpu_count(), "nproc": os.cpu_count()}


def workload_config(cfg: str, insts, modes, params, iters: int) -> dict:
    """The workload both arms run (identical dict in both JSON lines)."""
    return {"workload": f"{workload_name(cfg)}, static-rule mode selection",
            "instances": len(insts), "iters_per_instance": iters,
            "pool_size": params.pool_size, "delta": params.delta, "tabu_size": params.tabu_size,
            "modes": {"TIME": modes.count(1), "CAPACITY": modes.count(0)}}


def solve_cpu(insts, modes, indices, iters: int, threads: int, seed: int = 0) -> dict:
    """The reference algorithm (C port, `threads` workers per instance) on the
    given batch indices, one instance after another like `rcpsp-tabu bench`;
    schedules/sec = evaluations / wall summed over the instances
    (cooperation.py:254-293, cli.py:236)."""
    import oracle
    evals, wall, devs = 0, 0.0, []
    for i in indices:
        r = oracle.orchestrate(insts[i], iters, threads, seed, modes[i])
        evals += r["evaluations"]
        wall += r["wall_time"]
        devs.append(100.0 * (r["best_cmax"] - r["critical_path"]) / r["critical_path"])
    return {"evaluations": evals, "wall": wall, "instances": len(indices),
            "value": evals / wall if wall > 0 else 0.0,
            "cpm_dev": float(np.mean(devs)) if devs else None, "iters": iters,
            "threads": threads, "indices": list(indices)}


def batch_and_modes(cfg: str, count: int, mode: str = "rule"):
    from paper_1711_04556_b200 import decide_static, extract_features, synth
    insts = synth.benchmark_batch(cfg, count)
    if mode == "rule":
        modes = [int(decide_static(extract_features(x))) for x in insts]
    else:
        modes = [1 if mode == "time" else 0] * len(insts)
    return insts, modes


def cpu_baseline(cfg: str, insts, modes, iters: int, count: int, w1: bool = True) -> dict:
    """cpu_baseline object: the CPU sample on all host cores, plus a W = 1
    number (one worker thread) on the sample's first two instances at a
    fifth of the iterations."""
    from paper_1711_04556_b200 import synth
    hc = host_cpu()
    idx = synth.sample_indices(cfg, count, len(insts))
    cb = solve_cpu(insts, modes, idx, iters, hc["cores"])
    out = {"value": cb["value"], "unit": "schedules/s", "cores": hc["cores"], "kind": "port",
           "cpu_model": hc["model"], "nproc": hc["nproc"],
           "sample": (f"{cb['instances']} {cfg} instances of the {len(insts)}-instance batch "
                      f"(indices k*{synth.SAMPLE_STRIDE} mod {len(insts)}), I_total={iters}, "
                      f"{hc['cores']} worker threads each, instances one after another, "
                      f"{cb['wall']:.1f} s; cpm_dev {cb['cpm_dev']:.2f}%"),
           "cpm_dev": cb["cpm_dev"], "wall_s": cb["wall"]}
    if w1:
        one = solve_cpu(insts, modes, idx[:2], max(50, iters // 5), 1)
        out["w1"] = {"value": one["value"], "unit": "schedules/s", "cores": 1,
                     "sample": f"first 2 sample instances, I_total={one['iters']}, 1 worker",
                     "wall_s": one["wall"]}
    return out, cb


def run_reference(args, ws: int, rank: int) -> None:
    """--impl reference: the reference algorithm (C port) on all host cores
    over the SAME instance sample as the b200 arm's cpu_baseline, split over
    the timed steps (step i solves sample instances [i*S/K, (i+1)*S/K), the
    whole sample once over K steps; K > S cycles).  Rank 0 only."""
    if rank != 0:
        return
    from paper_1711_04556_b200 import SearchParams, synth
    insts, modes = batch_and_modes(args.config, args.instances, args.mode)
    hc = host_cpu()
    S = args.cpu_sample or synth.CPU_SAMPLE
    idx = synth.sample_indices(args.config, S, len(insts))
    K = max(1, args.steps)
    for w in range(args.warmup):            # warm-up: short solves on the sample
        solve_cpu(insts, modes, [idx[w % S]], min(args.iters, 50), hc["cores"])
    evals, wall, devs, step_ms = 0, 0.0, [], []
    for i in range(K):
        part = idx[i * S // K:(i + 1) * S // K] if K <= S else [idx[i % S]]
        r = solve_cpu(insts, modes, part, args.iters, hc["cores"])
        evals += r["evaluations"]
        wall += r["wall"]
        step_ms.append(1e3 * r["wall"])
        if r["cpm_dev"] is not None:
            devs.append((r["cpm_dev"], r["instances"]))
    value = evals / wall if wall > 0 else 0.0
    p = SearchParams.defaults_for(insts[0].n_activities, total_iters=args.iters)
    cpm = sum(d * k for d, k in devs) / max(1, sum(k for _, k in devs))
    sample = (f"{S} {args.config} instances of the {len(insts)}-instance batch (indices "
              f"k*{synth.SAMPLE_STRIDE} mod {len(insts)}, the b200 arm's cpu_baseline sample), "
              f"split over {K} steps, I_total={args.iters}, {hc['cores']} worker threads per "
              f"instance, instances one after another")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "schedules/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(step_ms)), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": workload_config(args.config, insts, modes, p, args.iters),
        "run": {"cpm_dev": cpm, "evaluations": evals, "wall_s": wall,
                "executor": "reference algorithm, C port of the numba path (oracle/), host"},
        "cpu_baseline": {"value": value, "unit": "schedules/s", "cores": hc["cores"],
                         "kind": "port", "cpu_model": hc["model"], "sample": sample},
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
    pick = cb["indices"]                       # the CPU sample's instances
    K = len(pick)
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
                    "host_wall_s": res.wall_s,
                    "stop": "device clock (%globaltimer), 97 % of the budget"}}


#: compact entries beside the headline (BASELINE.json configs[1] and [4]):
#: (config, mode, workers per instance, I_total per instance)
PER_CONFIG = (("j60p", "time", 8, 1000), ("j60p", "capacity", 8, 1000),
              ("act300", "time", 2, 100), ("act300", "capacity", 2, 100))


def per_config_entry(args, cfg: str, mode: str, workers: int, iters: int, smem_peak: float,
                     cpu_count: int) -> dict:
    """One compact measurement of another BASELINE config: the synth batch of
    DEFAULT_BATCH instances, mode forced, warm-up steps for >= 0.5 s of device
    time, then 1 more + 2 timed steps (CUDA events around pool init + search,
    L2 flushed), its roofline fraction with
    the same SMEM peak, and its own cpu_baseline on the config's CPU sample
    (as many sample instances as fit ~4 s on all host cores, >= 2)."""
    import torch
    from paper_1711_04556_b200 import SearchParams, synth
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    insts, modes = batch_and_modes(cfg, synth.DEFAULT_BATCH[cfg], mode)
    p = SearchParams.defaults_for(insts[0].n_activities, total_iters=iters, workers=workers,
                                  seed=0)
    scfg = SolveConfig(total_iters=iters, workers=workers, pool_size=p.pool_size,
                       tabu_size=p.tabu_size, delta=p.delta, phi_steps=p.phi_steps,
                       phi_max=p.phi_max, seed=0)
    solver = BatchSolver(insts, modes, scfg)
    solver.upload()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()
    ms, sms, evals, sevals, steps, devs = 0.0, 0.0, 0, 0, 0, []
    # warm-up until >= 0.5 s of device time (at least one step): short steps
    # otherwise meet the clocks still ramping after the CPU legs left the GPU
    # idle (one j60p step is ~44 ms)
    warm_ms, k = 0.0, 0
    while k == 0 or warm_ms < 500.0:
        solver.reset()
        torch.cuda.synchronize()
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0.record(stream)
        solver.pool_init(stream)
        solver.search(stream=stream)
        w1.record(stream)
        torch.cuda.synchronize()
        warm_ms += w0.elapsed_time(w1)
        k += 1
    for k in range(3):
        solver.reset()
        flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        solver.pool_init(stream)
        e1.record(stream)
        solver.search(stream=stream)
        e2.record(stream)
        torch.cuda.synchronize()
        if k == 0:
            continue
        res = solver.collect()
        ms += e0.elapsed_time(e2)
        sms += e1.elapsed_time(e2)
        evals += int(res.evaluations.sum())
        sevals += int((res.evaluations - res.pool_evaluations).sum())
        steps += res.sgs_steps
        devs.append(float(np.mean(100.0 * (res.best_cmax - res.critical_path)
                                  / res.critical_path)))
    W = work_per_schedule(cfg)["time" if mode == "time" else "cap"]
    achieved = sevals * W["bytes"] / (sms * 1e-3) / 1e9
    # CPU sample: sample instances one by one until ~4 s
    idx = synth.sample_indices(cfg, synth.CPU_SAMPLE, len(insts))
    done, ev, wall = [], 0, 0.0
    for i in idx:
        r = solve_cpu(insts, modes, [i], iters, cpu_count)
        ev += r["evaluations"]
        wall += r["wall"]
        done.append(r["cpm_dev"])
        if wall >= 4.0 and len(done) >= 2:
            break
    return {"config": cfg, "mode": mode.upper(), "instances": len(insts),
            "workers_per_instance": workers, "iters_per_instance": iters,
            "value": evals / (ms * 1e-3), "unit": "schedules/s", "ms_per_step": ms / 2,
            "cpm_dev": float(np.mean(devs)),
            "roofline": {"achieved": achieved, "peak": smem_peak, "unit": "GB/s",
                         "frac": achieved / smem_peak if smem_peak else None,
                         "bytes_per_schedule": W["bytes"],
                         "sgs_steps_per_schedule": steps / max(1, sevals)},
            "cpu_baseline": {"value": ev / wall if wall else 0.0, "unit": "schedules/s",
                             "cores": cpu_count, "kind": "port",
                             "sample": f"{len(done)} sample instances, I_total={iters}, "
                                       f"{wall:.1f} s", "cpm_dev": float(np.mean(done))}}


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
    from paper_1711_04556_b200 import SearchParams, synth
    from paper_1711_04556_b200.device import (BatchSolver, SolveConfig, smem_bandwidth)
    from paper_1711_04556_b200.population import EliteExchange, run_epochs

    insts, modes = batch_and_modes(args.config, args.instances, args.mode)
    p = SearchParams.defaults_for(insts[0].n_activities, total_iters=args.iters,
                                  workers=args.workers, seed=1000 * rank)
    cfg = SolveConfig(total_iters=p.total_iters, workers=p.workers, pool_size=p.pool_size,
                      tabu_size=p.tabu_size, delta=p.delta, phi_steps=p.phi_steps,
                      phi_max=p.phi_max, seed=p.seed, group=args.group, threads=args.threads,
                      steal=not args.no_steal, full_sgs=args.full_sgs,
                      cap_group=args.cap_group, profile_slots=args.profile_slots)
    solver = BatchSolver(insts, modes, cfg)
    solver.upload()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")  # > L2
    n_max = solver.n_max
    I = len(insts)
    exchange, peer, xmode, xnote = None, None, "none", None
    if ws > 1 and args.exchange == "peer":
        try:
            from paper_1711_04556_b200.population import PeerExchange
            peer = PeerExchange(solver, poll_every=args.poll_every)
            solver.peer = peer
            xmode = "peer"
        except Exception as exc:  # e.g. no CUDA IPC between the ranks' devices
            xnote = f"peer exchange unavailable ({type(exc).__name__}: {exc}); epochs used"
    if ws > 1 and peer is None:
        exchange = EliteExchange(solver, I, n_max)
        xmode = "epochs"
    epochs = args.epochs if xmode == "epochs" else 1

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
    peer_counters = peer.counters() if peer is not None else None

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

    if peer is not None:
        dist.barrier()          # nobody unmaps an outbox a peer may still read
        peer.close()
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

    if xmode == "peer":
        par = (f"{ws} independent search populations (one per GPU), live elite exchange: "
               f"search kernels read each other's outboxes over peer memory (CUDA IPC), "
               f"poll every {args.poll_every} exchanges; {backend} for the host plumbing")
    elif xmode == "epochs":
        par = (f"{ws} independent search populations (one per GPU), elite exchange "
               f"between {epochs} epochs by all_gather over {backend}")
    else:
        par = "1 search population on 1 GPU (no exchange)"
    line = {
        "metric": METRIC, "value": value, "unit": "schedules/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": workload_config(args.config, insts, modes, p, args.iters),
        "run": {"workers_per_instance": args.workers, "epochs": epochs,
                "cpm_dev": float(np.mean(devs)), "evaluations_per_step": evals // args.steps,
                "iterations_per_step": iters_done // args.steps,
                "l2": "256 MiB buffer written between timed steps", "parallelism": par,
                "exchange": xmode, **({"exchange_note": xnote} if xnote else {}),
                **({"peer_counters_last_step": peer_counters} if peer is not None else {})},
        "roofline": {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "kernel": "k_solve", "bytes_per_schedule": bytes_per_sched,
                     "bytes_basis": "reference full-SGS element touches x 4 B per evaluated "
                                    "schedule (profiles/work_per_schedule.json, pinned over "
                                    "the CPU sample's instances)",
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
        cb_line, cb = cpu_baseline(args.config, insts, modes, args.iters,
                                   args.cpu_sample or synth.CPU_SAMPLE)
        line["cpu_baseline"] = cb_line
        if not args.no_quality:
            line["quality"] = quality_leg(args, insts, modes, cb)
    if ws == 1 and not args.no_per_config:
        cores = host_cpu()["cores"]
        line["per_config"] = [per_config_entry(args, c, m, w, it, peak, cores)
                              for c, m, w, it in PER_CONFIG]
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
