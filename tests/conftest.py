"""Shared fixtures: golden vectors (tests/golden/golden.json, produced by the
reference via tests/golden/make_golden.py) and instance builders."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLDEN_PATH = ROOT / "tests" / "golden" / "golden.json"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and the sm_100a library")
    config.addinivalue_line("markers", "slow: long-running")


def _built_oracle():
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)


_built_oracle()


@pytest.fixture(scope="session")
def golden() -> dict:
    return json.loads(GOLDEN_PATH.read_text())


def instance_from(d: dict):
    from paper_1711_04556_b200 import make_instance
    return make_instance(d["name"], d["durations"], d["capacities"], d["demands"],
                         d["successors"])


@pytest.fixture(scope="session")
def ginst(golden):
    """name -> ProjectInstance for every golden instance."""
    return {k: instance_from(v) for k, v in golden["instances"].items()}


def random_topological_order(instance, rng: np.random.Generator) -> np.ndarray:
    """Random linear extension (restates the reference's helpers.py:54-69)."""
    n = instance.n_activities
    indeg = [len(instance.predecessors[i]) for i in range(n)]
    ready = [i for i in range(n) if indeg[i] == 0]
    out = np.empty(n, dtype=np.int32)
    for pos in range(n):
        act = ready.pop(int(rng.integers(len(ready))))
        out[pos] = act
        for j in instance.successors[act]:
            indeg[j] -= 1
            if indeg[j] == 0:
                ready.append(j)
    return out


def random_topological_orders(instance, rng: np.random.Generator, count: int) -> np.ndarray:
    """`count` random precedence-feasible orders at once (vectorised over the
    batch): every activity draws a uniform key, keys are raised along the
    edges (key_j >= key_p + eps for every predecessor p, in topological
    order) and each row is sorted by key.  Not the uniform distribution over
    linear extensions, but every order is feasible and rows vary; the fuzz
    tests use it for 10^4-10^5 orders per config."""
    n = instance.n_activities
    preds = instance.predecessors
    topo = np.asarray(random_topological_order(instance, np.random.default_rng(0)))
    key = rng.random((count, n))
    eps = 1.0 / (4 * n)
    for j in topo:
        p = list(preds[j])
        if p:
            key[:, j] = np.maximum(key[:, j], key[:, p].max(axis=1) + eps)
    return np.argsort(key, axis=1, kind="stable").astype(np.int32)


def chain_instance(durations_mid, cap=3):
    from paper_1711_04556_b200 import make_instance
    n = len(durations_mid) + 2
    return make_instance("chain", [0, *durations_mid, 0], [cap],
                         [[0]] + [[1]] * len(durations_mid) + [[0]],
                         [[i + 1] for i in range(n - 1)] + [[]])


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
