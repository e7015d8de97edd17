"""Multi-GPU population plumbing, world size 2 over gloo on CPU.

The device kernels cannot run here, so the ranks drive a host stand-in
solver whose export/merge follow the documented semantics of
k_export_elites / k_merge_elites (a foreign elite replaces the worst pool
entry when it is strictly better and its makespan is not already in the
pool; the global best follows).  tests/test_gpu_parity.py::test_merge_elites_model
pins the device kernels to this same model on a GPU.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1711_04556_b200.population import EliteExchange, epoch_limits, run_epochs


def merge_model(pool_cmax, pool_orders, best, best_order, elites, elite_cmax):
    """Host model of k_merge_elites for one instance (sources in rank order)."""
    pool_cmax = list(pool_cmax)
    pool_orders = [list(o) for o in pool_orders]
    for src_order, cm in zip(elites, elite_cmax):
        worst = max(range(len(pool_cmax)), key=lambda i: (pool_cmax[i], -i))
        if cm in pool_cmax or cm >= pool_cmax[worst]:
            continue
        pool_cmax[worst] = cm
        pool_orders[worst] = list(src_order)
        if cm < best:
            best, best_order = cm, list(src_order)
    return pool_cmax, pool_orders, best, best_order


class HostPopulation:
    """Stand-in for device.BatchSolver: per instance a pool of (cmax, order)."""

    def __init__(self, rank: int, n_inst: int, n: int, F: int):
        rng = np.random.default_rng(100 + rank)
        self.n = n
        self.cmax = rng.integers(50, 90, size=(n_inst, F)).astype(np.int32)
        self.orders = np.stack([[rng.permutation(n) for _ in range(F)] for _ in range(n_inst)])
        self.best = self.cmax.min(1)
        self.best_order = np.stack([self.orders[i, int(np.argmin(self.cmax[i]))]
                                    for i in range(n_inst)])
        self.searched = []

    def search(self, epoch_limit=None, stream=None):
        self.searched.append(epoch_limit)
        self.cmax -= 1          # "improve" every entry a little
        self.best -= 1

    def export_elites(self, elites, elite_cmax, stream=None):
        elites.copy_(torch.from_numpy(self.best_order.astype(np.int32)))
        elite_cmax.copy_(torch.from_numpy(self.best.astype(np.int32)))

    def merge_elites(self, all_orders, all_cmax, n_src, stream=None):
        n_inst = self.cmax.shape[0]
        ao = all_orders.numpy().reshape(n_src, n_inst, -1)
        ac = all_cmax.numpy().reshape(n_src, n_inst)
        for i in range(self.cmax.shape[0]):
            pc, po, b, bo = merge_model(self.cmax[i], self.orders[i], int(self.best[i]),
                                        self.best_order[i], ao[:, i], ac[:, i])
            self.cmax[i], self.orders[i], self.best[i], self.best_order[i] = pc, po, b, bo


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pop = HostPopulation(rank, n_inst=3, n=7, F=4)
    ex = EliteExchange(pop, n_inst=3, n_max=7, device="cpu")
    before = pop.best.copy()
    run_epochs(pop, total_iters=100, epochs=4, exchange=ex)
    # after the last exchange every rank holds the best elite of all ranks
    allb = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allb, torch.from_numpy(pop.best.astype(np.int64)))
    out[rank] = dict(searched=pop.searched, rounds=ex.rounds, before=before.tolist(),
                     after=pop.best.tolist(), all_after=[b.tolist() for b in allb],
                     bytes=ex.bytes_per_round)
    dist.destroy_process_group()


def test_epoch_limits():
    assert epoch_limits(100, 4) == [25, 50, 75, 100]
    assert epoch_limits(10, 1) == [10]
    assert epoch_limits(7, 3) == [2, 4, 7]


def test_two_rank_elite_exchange():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    r0, r1 = out[0], out[1]
    assert r0["searched"] == [25, 50, 75, 100] and r1["searched"] == [25, 50, 75, 100]
    assert r0["rounds"] == 3 and r1["rounds"] == 3          # no exchange after the last epoch
    # both ranks end with the same per-instance best: the min over ranks
    assert r0["all_after"][0] == r0["all_after"][1]
    for i in range(3):
        assert r0["after"][i] <= min(r0["before"][i], r1["before"][i]) - 1
    assert r0["bytes"] == (3 * 7 + 3) * 4 * world


def test_merge_model_semantics():
    pool_c = [10, 12, 15]
    pool_o = [[0, 1], [0, 1], [0, 1]]
    # 12 already present -> skipped; 11 replaces 15 (worst); 9 replaces 12, becomes best
    pc, po, b, bo = merge_model(pool_c, pool_o, 10, [0, 1], [[1, 0], [2, 0], [3, 0]], [12, 11, 9])
    assert pc == [10, 9, 11] and b == 9 and bo == [3, 0]


# ---------------------------------------------------------------------------
# the same plumbing with device.BatchSolver: two ranks sharing one GPU (gloo)

def _gpu_worker(rank: int, world: int, port: int, kind: str, out):
    import sys
    from conftest import ROOT
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1711_04556_b200 import evaluate, synth
    from paper_1711_04556_b200.device import BatchSolver, SolveConfig
    from paper_1711_04556_b200.population import PeerExchange
    # the hardest grid cell (RS 0.1): the pools do not start at the critical path
    insts = synth.benchmark_batch("j120p", 6, first_seed=0)
    res = {}
    if kind == "epochs":
        cfg = SolveConfig(total_iters=200, workers=2, pool_size=8, tabu_size=800, delta=60,
                          phi_steps=20, phi_max=3, seed=1000 * rank)
        s = BatchSolver(insts, [1] * 6, cfg)
        s.upload()
        s.pool_init()
        ex = EliteExchange(s, len(insts), s.n_max)
        run_epochs(s, 200, 4, ex)
        r = s.collect()
        res["rounds"] = ex.rounds
    else:
        iters = 2000 if rank == 1 else 5
        cfg = SolveConfig(total_iters=iters, workers=1, pool_size=8, tabu_size=800, delta=60,
                          phi_steps=20, phi_max=3, seed=1000 * rank)
        s = BatchSolver(insts, [1] * 6, cfg)
        peer = PeerExchange(s, poll_every=1)
        s.peer = peer
        s.upload()
        s.pool_init()
        torch.cuda.synchronize()
        res["pool_worst"] = s.ent_cmax.cpu().numpy().max(1).tolist()
        res["pool_all"] = s.ent_cmax.cpu().numpy().tolist()
        if rank == 1:
            s.search()                 # publishes its improvements
            torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            s.search()                 # polls rank 1's outbox at its exchanges
            torch.cuda.synchronize()
        dist.barrier()
        r = s.collect()
        res["counters"] = peer.counters()
        res["pool_after"] = s.ent_cmax.cpu().numpy().tolist()
        dist.barrier()                 # nobody unmaps before everyone is done
        peer.close()
    res["best"] = r.best_cmax.tolist()
    res["iters_ok"] = bool(((r.iterations == cfg.total_iters)
                            | (r.best_cmax == r.critical_path)).all())
    res["valid"] = [evaluate(r.best_order[i, :x.n_activities], x, 1).cmax == int(r.best_cmax[i])
                    for i, x in enumerate(insts)]
    out[rank] = res
    dist.destroy_process_group()


def _spawn_gpu(kind: str):
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gpu_worker, args=(world, port, kind, out), nprocs=world, join=True)
    return out[0], out[1]


@pytest.mark.gpu
def test_two_rank_epoch_exchange_batchsolver():
    """Epoch exchange (export -> all_gather -> merge) driving device.BatchSolver:
    every epoch boundary merges, budgets are kept, bests are valid schedules,
    and every instance spends its budget (or stops at the critical path)."""
    r0, r1 = _spawn_gpu("epochs")
    for r in (r0, r1):
        assert r["rounds"] == 3
        assert all(r["valid"])
        assert r["iters_ok"]


@pytest.mark.gpu
def test_two_rank_peer_exchange():
    """Live exchange over peer memory (CUDA IPC; two processes on one GPU):
    rank 1 searches and publishes, rank 0 then polls at its first exchange and
    imports every foreign elite that beats its pool's worst entry; imported
    orders are consistent (their evaluation equals the claimed makespan)."""
    r0, r1 = _spawn_gpu("peer")
    improved = sum(b < min(p) for b, p in zip(r1["best"], r1["pool_all"]))
    # every improvement of a global best is published (at least once)
    assert r1["counters"]["publishes"] >= improved > 0, (r1["counters"], improved)
    assert r0["counters"]["polls"] > 0 and r0["counters"]["imports"] > 0
    assert r0["counters"]["torn_reads"] == 0
    for i, b1 in enumerate(r1["best"]):
        if b1 < r0["pool_worst"][i] and b1 not in r0["pool_all"][i]:
            assert b1 in r0["pool_after"][i] or min(r0["pool_after"][i]) < b1, i
        assert r0["best"][i] <= min(b1, min(r0["pool_all"][i])), i
    assert all(r0["valid"]) and all(r1["valid"])
    assert r0["iters_ok"] and r1["iters_ok"]
