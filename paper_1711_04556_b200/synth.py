"""Synthetic PSPLIB-shape instances (PSPLIB itself is not available offline).

`random_instance` is "Gen-R", the reference's own benchmark workload recipe
(pkg/tests/helpers.py:15-42, used by pkg/benchmarks/compare_backends.py:31):
the same numpy Generator draws in the same order, so a (n_real, m, seed, ...)
tuple names the same instance on both sides.  `progen_instance` is "Gen-P",
PSPLIB-shape instances after the ProGen parameters (NC, RF, RS) of PSPLIB's
sets.  `benchmark_batch` builds the instance batches named in BASELINE.json's
configs.
"""

from __future__ import annotations

import numpy as np

from .instance import ProjectInstance, make_instance


def random_instance(n_real: int, m: int, seed: int, cap_lo: int = 8, cap_hi: int = 14,
                    max_dur: int = 10, demand_density: float = 1.0) -> ProjectInstance:
    """Connected random DAG with dummy source/sink (Gen-R)."""
    gen = np.random.default_rng(seed)
    n = n_real + 2
    durations = [0, *(int(d) for d in gen.integers(1, max_dur + 1, n_real)), 0]
    capacities = [int(c) for c in gen.integers(cap_lo, cap_hi + 1, m)]
    demands = np.zeros((n, m), dtype=int)
    for act in range(1, n - 1):
        for k in range(m):
            if gen.random() < demand_density:
                demands[act, k] = int(gen.integers(1, capacities[k] + 1))
    succ: list[set[int]] = [set() for _ in range(n)]
    for j in range(2, n - 1):
        want = int(gen.integers(1, 3))
        for p in gen.choice(np.arange(1, j), size=min(j - 1, want), replace=False):
            succ[int(p)].add(j)
    has_pred = set().union(*succ)
    for act in range(1, n - 1):
        if act not in has_pred:
            succ[0].add(act)
        if not succ[act]:
            succ[act].add(n - 1)
    if not succ[0]:
        succ[0].add(1)
    return make_instance(f"rand{n_real}x{m}s{seed}", durations, capacities, demands.tolist(),
                         [sorted(s) for s in succ])


#: BASELINE.json configs -> Gen-R parameters
CONFIGS = {
    "j30": dict(n_real=30, m=4, demand_density=0.5, cap_lo=10, cap_hi=16),
    "j60": dict(n_real=60, m=4, demand_density=0.5, cap_lo=10, cap_hi=16),
    "j120": dict(n_real=120, m=4, demand_density=0.5, cap_lo=10, cap_hi=16),
    "act300": dict(n_real=300, m=4, demand_density=0.5, cap_lo=40, cap_hi=80),
}


def progen_instance(n_real: int, seed: int, nc: float, rf: float, rs: float, m: int = 4,
                    max_dur: int = 10, max_dem: int = 10, max_fan: int = 3,
                    n_start: int = 3) -> ProjectInstance:
    """"Gen-P": a PSPLIB-shape instance after the ProGen parameters PSPLIB's
    j30/j60/j120 sets were generated with (Kolisch, Sprecher & Drexl 1995;
    SURVEY.md sec. 8d).  PSPLIB itself is not available offline.

    * network: `n_start` start activities (successors of the source); every
      other activity gets one earlier predecessor, then non-redundant arcs
      (no transitive shortcut, at most `max_fan` successors / predecessors per
      activity) are added until the network complexity -- arcs per node,
      dummy arcs included -- reaches `nc`; activities without successors
      precede the sink;
    * resource factor `rf`: each activity requests round(rf * m) (at least
      one) resources chosen at random; demands U{1..max_dem}, durations
      U{1..max_dur};
    * resource strength `rs`: R_k = K_min + round(rs * (K_max - K_min)) with
      K_min the largest single demand and K_max the peak demand of the
      earliest-start (precedence-only) schedule.
    """
    gen = np.random.default_rng(seed)
    n = n_real + 2
    sink = n - 1
    succ: list[set[int]] = [set() for _ in range(n)]
    pred: list[set[int]] = [set() for _ in range(n)]
    reach = [0] * n                      # bitset of activities reachable from i

    def add(i: int, j: int) -> None:
        succ[i].add(j)
        pred[j].add(i)

    starts = list(range(1, 1 + min(n_start, n_real)))
    for j in range(1, n - 1):
        if j in starts:
            add(0, j)
            continue
        cands = [i for i in range(1, j) if len(succ[i]) < max_fan]
        if not cands:
            cands = list(range(1, j))
        add(int(gen.choice(cands)), j)
    # reachability over real activities (arcs only go from lower to higher ids)
    def rebuild() -> None:
        for i in range(n - 2, 0, -1):
            r = 0
            for j in succ[i]:
                r |= (1 << j) | reach[j]
            reach[i] = r
    rebuild()
    target = int(round(nc * n))
    arcs = sum(len(x) for x in succ) + sum(1 for i in range(1, n - 1) if not succ[i])
    tries = 0
    while arcs < target and tries < 50 * n:
        tries += 1
        i = int(gen.integers(1, n - 2))
        j = int(gen.integers(i + 1, n - 1))
        if j in succ[i] or len(succ[i]) >= max_fan or len(pred[j]) >= max_fan:
            continue
        # no transitive shortcut: j must not already be reachable from i
        if (reach[i] >> j) & 1:
            continue
        had_no_succ = not succ[i]
        add(i, j)
        arcs += 0 if had_no_succ else 1
        rebuild()
    for i in range(1, n - 1):
        if not succ[i]:
            add(i, sink)
    durations = [0, *(int(d) for d in gen.integers(1, max_dur + 1, n_real)), 0]
    demands = np.zeros((n, m), dtype=np.int64)
    for a in range(1, n - 1):
        k_used = max(1, int(round(rf * m)))
        use = gen.permutation(m)[:k_used]
        demands[a, use] = gen.integers(1, max_dem + 1, k_used)
    # earliest-start schedule (precedence only) -> peak demand per resource
    es = [0] * n
    for a in range(n):
        for j in succ[a]:
            es[j] = max(es[j], es[a] + durations[a])
    horizon = max(es[a] + durations[a] for a in range(n))
    prof = np.zeros((horizon + 1, m), dtype=np.int64)
    for a in range(1, n - 1):
        prof[es[a]:es[a] + durations[a]] += demands[a]
    kmin = demands.max(axis=0)
    kmax = prof.max(axis=0)
    caps = [int(max(1, kmin[k] + round(rs * (kmax[k] - kmin[k])))) for k in range(m)]
    name = f"progen{n_real}nc{nc}rf{rf}rs{rs}s{seed}"
    return make_instance(name, durations, caps, demands.tolist(), [sorted(x) for x in succ])


#: PSPLIB's full-factorial parameter grids (Kolisch & Sprecher 1996):
#: 10 instances per (NC, RF, RS) cell -> j30/j60: 480, j120: 600 instances
PSPLIB_GRID = {
    "j30p": dict(n_real=30, rs=(0.2, 0.5, 0.7, 1.0)),
    "j60p": dict(n_real=60, rs=(0.2, 0.5, 0.7, 1.0)),
    "j120p": dict(n_real=120, rs=(0.1, 0.2, 0.3, 0.4, 0.5)),
}
PSPLIB_NC = (1.5, 1.8, 2.1)
PSPLIB_RF = (0.25, 0.5, 0.75, 1.0)


def progen_cell(config: str, k: int) -> tuple[float, float, float]:
    """(NC, RF, RS) of the k-th instance of a Gen-P set (10 per cell, PSPLIB order)."""
    g = PSPLIB_GRID[config]
    cells = [(nc, rf, rs) for nc in PSPLIB_NC for rf in PSPLIB_RF for rs in g["rs"]]
    return cells[(k // 10) % len(cells)]


def benchmark_batch(config: str, count: int, first_seed: int = 0) -> list[ProjectInstance]:
    """`count` instances of a BASELINE config, seeds first_seed.. : Gen-R
    ("j30", "j60", "j120", "act300") or Gen-P over PSPLIB's parameter grid
    ("j30p", "j60p", "j120p")."""
    if config in PSPLIB_GRID:
        n_real = PSPLIB_GRID[config]["n_real"]
        return [progen_instance(n_real, seed=k, nc=c[0], rf=c[1], rs=c[2])
                for k in range(first_seed, first_seed + count)
                for c in [progen_cell(config, k)]]
    kw = dict(CONFIGS[config])
    n_real, m = kw.pop("n_real"), kw.pop("m")
    return [random_instance(n_real, m, seed=s, **kw)
            for s in range(first_seed, first_seed + count)]


#: instances per benchmark step (bench.py): the size of PSPLIB's j120 set
#: (600) for the j120 configs, one instance per SM otherwise
DEFAULT_BATCH = {"j30": 148, "j60": 148, "j120": 600, "act300": 148, "j30p": 148,
                 "j60p": 148, "j120p": 600}
#: the CPU sample: instances k * SAMPLE_STRIDE mod batch, k < CPU_SAMPLE -- the
#: stride is coprime with every batch size, so the sample spreads over the
#: batch (and over Gen-P's parameter-grid cells, 10 consecutive per cell)
SAMPLE_STRIDE = 157
CPU_SAMPLE = 30


def sample_indices(config: str, count: int = CPU_SAMPLE, batch: int | None = None) -> list[int]:
    """Batch indices of the CPU-sample instances of a benchmark config (bench.py's
    cpu_baseline, its reference arm and quality leg, and the pinned W of
    profiles/work_per_schedule.json all use this sample)."""
    batch = DEFAULT_BATCH[config] if batch is None else batch
    return [(k * SAMPLE_STRIDE) % batch for k in range(count)]
