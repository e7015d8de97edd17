"""Independent search populations across GPUs with elite exchange.

The tabu search shards naturally: every rank (one process per GPU) runs its
own population -- its own working sets, workers and seeds -- on the same
instances.  The only collective is the
periodic elite exchange: between search epochs each rank exports every
instance's global best (order + makespan) from HBM, one NCCL all_gather moves
them over NVLink, and each rank merges the foreign elites into its working
sets on the device (csrc/kernels.cu:k_merge_elites).  The host only sequences
launches; the data never leaves device memory.

`run_epochs` is the driver used by bench.py and by `solve_populations`; it
works with any solver object exposing search / export_elites / merge_elites
(device.BatchSolver on GPUs; the multi-process CPU test substitutes a host
stand-in to check the plumbing).
"""

from __future__ import annotations


class EliteExchange:
    """all_gather of per-instance elites between the ranks of a process group."""

    def __init__(self, solver, n_inst: int, n_max: int, device: str = "cuda", group=None):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.solver = solver
        self.mine = torch.zeros((n_inst, n_max), dtype=torch.int32, device=device)
        self.mine_c = torch.zeros(n_inst, dtype=torch.int32, device=device)
        # gathered layout [source rank][instance][n_max], as k_merge_elites reads it
        self.all = torch.zeros((self.world * n_inst, n_max), dtype=torch.int32, device=device)
        self.all_c = torch.zeros(self.world * n_inst, dtype=torch.int32, device=device)
        self.n_inst = n_inst
        self.rounds = 0

    @property
    def bytes_per_round(self) -> int:
        return (self.mine.numel() + self.mine_c.numel()) * 4 * self.world

    def __call__(self, stream=None) -> None:
        self.solver.export_elites(self.mine, self.mine_c, stream)
        self.dist.all_gather_into_tensor(self.all, self.mine, group=self.group)
        self.dist.all_gather_into_tensor(self.all_c, self.mine_c, group=self.group)
        self.solver.merge_elites(self.all, self.all_c, self.world, stream)
        self.rounds += 1


def epoch_limits(total_iters: int, epochs: int) -> list[int]:
    """Planned-iteration limit of each epoch (the last one is the budget)."""
    epochs = max(1, epochs)
    return [total_iters * (e + 1) // epochs for e in range(epochs)]


def run_epochs(solver, total_iters: int, epochs: int, exchange=None, stream=None,
               on_search=None) -> None:
    """Search in `epochs` slices of the iteration budget; exchange elites
    between slices when `exchange` is given.  `on_search(begin)` (optional)
    is called around every search launch (begin=True/False) for timing."""
    limits = epoch_limits(total_iters, epochs)
    for e, limit in enumerate(limits):
        if on_search:
            on_search(True)
        solver.search(epoch_limit=limit, stream=stream)
        if on_search:
            on_search(False)
        if exchange is not None and e + 1 < len(limits):
            exchange(stream)
