"""Synthetic PSPLIB-shape instances (PSPLIB itself is not available offline).

`random_instance` is "Gen-R", the reference's own benchmark workload recipe
(pkg/tests/helpers.py:15-42, used by pkg/benchmarks/compare_backends.py:31):
the same numpy Generator draws in the same order, so a (n_real, m, seed, ...)
tuple names the same instance on both sides.  `benchmark_batch` builds the
instance batches named in BASELINE.json's configs.
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


def benchmark_batch(config: str, count: int, first_seed: int = 0) -> list[ProjectInstance]:
    """`count` Gen-R instances of a BASELINE config, seeds first_seed.. ."""
    kw = dict(CONFIGS[config])
    n_real, m = kw.pop("n_real"), kw.pop("m")
    return [random_instance(n_real, m, seed=s, **kw)
            for s in range(first_seed, first_seed + count)]
