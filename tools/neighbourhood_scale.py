#!/usr/bin/env python3
"""Parity at scale for the search kernels' neighbourhood evaluators (GPU box):
every evaluated swap's makespan of whole neighbourhoods of many random
precedence-feasible orders, computed by the prefix-reusing / closed-form
evaluators inside k_run_chunk (group 32, as the search runs them), against the
oracle's full SGS of the swapped order (kernels.py:350-362).  Prints one JSON
line per config and mode with the number of moves checked and mismatches.

usage: python tools/neighbourhood_scale.py [moves_per_config]"""
from __future__ import annotations

import json
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import oracle  # noqa: E402
from conftest import random_topological_order  # noqa: E402
from paper_1711_04556_b200 import device, synth  # noqa: E402


def oracle_cmax(inst, orders, mode):
    parts = np.array_split(orders, min(32, max(1, len(orders))))
    with ThreadPoolExecutor(max_workers=16) as ex:
        res = list(ex.map(lambda o: oracle.evaluate_batch(inst, o, mode)[0], parts))
    return np.concatenate(res)


def swap_rows(order, moves):
    out = np.repeat(order[None], len(moves), 0)
    r = np.arange(len(moves))
    out[r, moves[:, 0]] = order[moves[:, 1]]
    out[r, moves[:, 1]] = order[moves[:, 0]]
    return out


def run(cfg, mode, target, delta=60, batch=64):
    rng = np.random.default_rng(1000 + mode)
    insts = synth.benchmark_batch(cfg, 8, first_seed=500)
    checked = bad = orders_done = 0
    t0 = time.time()
    k = 0
    while checked < target:
        inst = insts[k % len(insts)]
        k += 1
        orders = np.stack([random_topological_order(inst, rng) for _ in range(batch)])
        cm, _ = oracle.evaluate_batch(inst, orders, mode)
        tl = [np.zeros((8, 2), np.int32) for _ in range(batch)]
        res = device.run_chunk_batch(inst, mode, delta, orders, tl, [0] * batch, 1, 0, cm, cm,
                                     0, group=32)
        allrows, allgot = [], []
        for b in range(batch):
            moves, got = res["neighbourhood"][b]
            if len(moves):
                allrows.append(swap_rows(orders[b], moves))
                allgot.append(got)
        if allrows:
            want = oracle_cmax(inst, np.concatenate(allrows), mode)
            got = np.concatenate(allgot)
            bad += int((want != got).sum())
            checked += len(got)
        orders_done += batch
    return {"config": cfg, "mode": "TIME" if mode == 1 else "CAPACITY", "moves_checked": checked,
            "mismatches": bad, "orders": orders_done, "delta": delta,
            "seconds": round(time.time() - t0, 1)}


def main() -> None:
    target = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
    for cfg in ("j120p", "j60p", "j30p", "j120", "act300"):
        for mode in (1, 0):
            print(json.dumps(run(cfg, mode, target)), flush=True)


if __name__ == "__main__":
    main()
