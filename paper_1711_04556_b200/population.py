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


class PeerExchange:
    """Live elite exchange over peer memory (no epochs, no host round trip).

    Every rank's search kernel publishes each instance's new global best in a
    device outbox (a seqlock record: sequence number, makespan, order) and,
    every `poll_every` exchanges of a worker, reads the other ranks' outboxes
    directly -- CUDA IPC mappings, so the loads go over NVLink/NVSwitch --
    importing the best new foreign elite into its worst pool entry
    (csrc/kernels.cu: publish_best / import_peer_elite).  The search never
    stops for it.  The host's part is one-time setup: allocate the outbox,
    all-gather the 64-byte IPC handles over the process group, map the peers'.
    """

    def __init__(self, solver, poll_every: int = 4, group=None):
        import ctypes
        import torch
        import torch.distributed as dist
        from . import _native
        self.L = _native.lib()
        self.solver = solver
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world - 1 > 32:
            raise ValueError("at most 32 peer populations")
        I, n_max = len(solver.instances), solver.n_max
        self.words = 4 + n_max
        nbytes = I * self.words * 4
        self.outbox = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        _native.check(self.L.rcpsp_outbox_alloc(nbytes, ctypes.byref(self.outbox), handle),
                      "rcpsp_outbox_alloc")
        handles: list = [None] * self.world
        dist.all_gather_object(handles, bytes(handle), group=group)
        self.mapped = []
        for r, h in enumerate(handles):
            if r == self.rank:
                continue
            ptr_r = ctypes.c_void_p()
            buf = (ctypes.c_char * 64).from_buffer_copy(h)
            _native.check(self.L.rcpsp_outbox_open(buf, ctypes.byref(ptr_r)), "rcpsp_outbox_open")
            self.mapped.append(ptr_r)
        self.n_peers = len(self.mapped)
        self.peers = torch.tensor([p.value for p in self.mapped] or [0], dtype=torch.int64,
                                  device="cuda")
        self.seen = torch.zeros((I, max(1, self.n_peers)), dtype=torch.int32, device="cuda")
        self.stats = torch.zeros(4, dtype=torch.int64, device="cuda")
        self.poll_every = max(1, int(poll_every))
        self.I = I
        self.nbytes = nbytes

    def fill_args(self, a) -> None:
        a.outbox = self.outbox.value
        a.peers = self.peers.data_ptr()
        a.n_peers = self.n_peers
        a.peer_seen = self.seen.data_ptr()
        a.poll_every = self.poll_every
        a.peer_stats = self.stats.data_ptr()

    def reset(self, stream=None) -> None:
        """Between independent solves of the same batch: forget what was
        imported and zero the own outbox (the callers separate solves with a
        barrier, so the peers reset in step)."""
        from . import _native
        self.seen.zero_()
        self.stats.zero_()
        _native.check(self.L.rcpsp_outbox_reset(self.outbox, self.nbytes,
                                                _native.stream_handle(stream)),
                      "rcpsp_outbox_reset")

    def counters(self) -> dict:
        s = self.stats.cpu().tolist()
        return {"imports": s[0], "publishes": s[1], "polls": s[2], "torn_reads": s[3]}

    def close(self) -> None:
        for p in self.mapped:
            self.L.rcpsp_outbox_close(p)
        self.mapped = []
        if self.outbox.value:
            self.L.rcpsp_outbox_free(self.outbox)
            self.outbox = None
