"""Device side of the host: instance packing, HBM buffers and the launches.

PyTorch is plumbing only here (device memory, streams); every computation
happens in the sm_100a library through the C ABI (`_native`).  Layout of a
packed instance ("blob", int32, see csrc/common.cuh):

    header[32] | dur[n] | dem[n*m] | cap[m] | pred_ptr[n+1] | pred_dat[e]
    | succ_ptr[n+1] | succ_dat[e] | req[n*W] | capw[W] | lvl_ptr[L+1] | lvl_dat[n]

`req` packs an activity's demands on all resources into W 32-bit words of
8-bit (capacities <= 127) or 16-bit (<= 32767) lanes -- the TIME profile
slot uses the same packing, so the per-slot window test is one word op.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import RcpspShape, RcpspSolveArgs, check, ptr, stream_handle
from .instance import ProjectInstance

MODE_CAPACITY = 0
MODE_TIME = 1
BLOB_MAGIC = 0x52435053
HDR = 32
(B_MAGIC, B_N, B_M, B_H, B_E, B_W, B_LB, B_RMAX, B_CPM, B_LEN, B_NLVL, B_BIG,
 B_SUMCAP, B_LBRES) = range(14)
(B_OFF_DUR, B_OFF_DEM, B_OFF_CAP, B_OFF_PPTR, B_OFF_PDAT, B_OFF_SPTR, B_OFF_SDAT, B_OFF_REQ,
 B_OFF_CAPW, B_OFF_LPTR, B_OFF_LDAT) = range(16, 27)

WS_FIELDS = dict(cursor=0, total=1, planned=2, consumed=3, stop=4, best=5, best_mode=6, floor=7,
                 pool_evals=8, t0=9, t1=10, iterations=11, evaluations=12, exchanges=13,
                 diversifications=14, forced=15)
WK_FIELDS = dict(iterations=0, evaluations=1, exchanges=2, diversifications=3, forced=4,
                 chunks=5, trace_len=6, t0=7, t1=8, sgs_steps=9)

KEY_LIMIT = 1 << 16   # selection key packs (C_max << 16 | rank)


class UnsupportedInstance(ValueError):
    """The instance shape is outside what the packed device encoding handles."""


def packing_for(capacities: np.ndarray) -> tuple[int, int]:
    """(lane_bits, words per slot) of the TIME profile for these capacities,
    (0, 0) when they do not pack into <= 2 words (CAPACITY mode only) --
    the rule rcpsp_pack_instance applies (csrc/pack.cpp)."""
    cmax = int(np.max(capacities)) if len(capacities) else 0
    if not len(capacities):
        return 8, 1
    if cmax > 32767:
        return 0, 0
    lb = 8 if cmax <= 127 else 16
    words = math.ceil(len(capacities) / (32 // lb))
    return (lb, words) if words <= 2 else (0, 0)


def _c_arrays(inst: ProjectInstance):
    ka = inst.kernel_arrays
    n, m = inst.n_activities, inst.n_resources
    arrs = [np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))
            for a in (ka.durations, ka.demands, ka.capacities, ka.pred_ptr, ka.pred_dat,
                      ka.succ_ptr, ka.succ_dat)]
    return n, m, arrs, int(ka.horizon)


def pack_instance(inst: ProjectInstance) -> np.ndarray:
    """int32 blob of one instance, built by the C ABI's host packer
    (rcpsp_blob_words + rcpsp_pack_instance, csrc/pack.cpp; layout in the
    module docstring).  Needs the built library but no GPU."""
    L = _native.host_lib()
    n, m, arrs, horizon = _c_arrays(inst)
    if n >= KEY_LIMIT:
        raise UnsupportedInstance(f"{n} activities >= {KEY_LIMIT}")
    if horizon >= KEY_LIMIT - 1:
        raise UnsupportedInstance(f"horizon {horizon} >= {KEY_LIMIT - 1}")
    dur, dem, cap, pp, pd, sp, sd = (a.ctypes.data for a in arrs)
    words = L.rcpsp_blob_words(dur, dem, cap, n, m, pp, pd, sp, sd, horizon)
    if words < 0:
        raise ValueError(L.rcpsp_pack_last_error().decode(errors="replace"))
    blob = np.zeros(int(words), dtype=np.int32)
    if L.rcpsp_pack_instance(dur, dem, cap, n, m, pp, pd, sp, sd, horizon, blob.ctypes.data,
                             int(words)) != 0:
        raise ValueError(L.rcpsp_pack_last_error().decode(errors="replace"))
    return blob


def blob_shape(blob: np.ndarray) -> RcpspShape:
    """RcpspShape of a packed host blob (rcpsp_blob_shape)."""
    shape = RcpspShape()
    blob = np.ascontiguousarray(blob, dtype=np.int32)
    if _native.host_lib().rcpsp_blob_shape(blob.ctypes.data, ctypes.byref(shape)) != 0:
        raise ValueError(_native.host_lib().rcpsp_pack_last_error().decode(errors="replace"))
    return shape


def require_time_packing(blob: np.ndarray, mode: int) -> None:
    if int(mode) == MODE_TIME and int(blob[B_W]) == 0:
        raise UnsupportedInstance(
            "capacities / resource count do not fit the packed TIME profile (<= 8 resources "
            "with capacities <= 127, <= 4 with <= 32767): use CAPACITY mode")


def neighborhood_size(n: int, delta: int) -> int:
    return sum(min(delta, n - 2 - u) for u in range(1, n - 2))


def rng_words(seed: int) -> np.ndarray:
    """numpy default_rng(seed) PCG64 state as 6 uint64 words."""
    st = np.random.default_rng(seed).bit_generator.state
    s, inc = st["state"]["state"], st["state"]["inc"]
    m64 = (1 << 64) - 1
    return np.array([s >> 64, s & m64, inc >> 64, inc & m64, st["has_uint32"], st["uinteger"]],
                    dtype=np.uint64)


def words_state(words: np.ndarray) -> dict:
    w = [int(x) for x in words]
    return {"bit_generator": "PCG64", "state": {"state": (w[0] << 64) | w[1],
                                                "inc": (w[2] << 64) | w[3]},
            "has_uint32": w[4], "uinteger": w[5]}


def _torch():
    import torch
    return torch


def to_dev(arr: np.ndarray, stream=None):
    torch = _torch()
    t = torch.from_numpy(np.ascontiguousarray(arr))
    return t.to("cuda", non_blocking=False)


@dataclass
class DeviceInstance:
    """One packed instance resident in HBM."""

    inst: ProjectInstance
    blob_host: np.ndarray
    blob: object  # torch int32 cuda tensor
    shape: RcpspShape = None

    @property
    def n(self) -> int:
        return int(self.blob_host[B_N])

    @property
    def words(self) -> int:
        return int(self.blob_host[B_W])


_cache: dict[int, DeviceInstance] = {}


def device_instance(inst: ProjectInstance) -> DeviceInstance:
    """Pack and upload once per instance object (cached by identity)."""
    _native.lib()
    key = id(inst)
    hit = _cache.get(key)
    if hit is not None and hit.inst is inst:
        return hit
    host = pack_instance(inst)
    dev = DeviceInstance(inst, host, to_dev(host), blob_shape(host))
    if len(_cache) > 256:
        _cache.clear()
    _cache[key] = dev
    return dev


def pick_group(n: int) -> int:
    """TIME lanes per schedule for the search kernel (tuned on B200)."""
    return 32


def sm_count() -> int:
    return int(_torch().cuda.get_device_properties(0).multi_processor_count)


def pick_cluster(workers_total: int) -> int:
    """CTAs per worker: a small launch (a single instance, a few workers)
    leaves most SMs idle, so each worker becomes a thread-block cluster whose
    CTAs share its neighbourhood evaluation (up to 8; about two CTAs per SM in
    total).  Batches that fill the GPU run one CTA per worker."""
    if workers_total <= 0:
        return 1
    return max(1, min(8, (2 * sm_count()) // workers_total))


def pick_cap_group(n: int, m: int, rmax: int) -> int:
    """CAPACITY evaluator for the search kernel: one warp per schedule.
    Measured on B200 (profiles/r2/cap_group.txt) once rows of up to 32
    entries are updated in registers: the warp evaluator beats one thread per
    schedule on every config where the thread's state is small enough to
    compete -- Gen-R j120 99 vs 89 M schedules/s, j60 184 vs 164 M, j30 295 vs
    236 M, Gen-P j30 169 vs 41 M (round 1 picked one thread per schedule for
    states of <= 256 words).  `SolveConfig.cap_group = 1` still selects it."""
    del n, m, rmax
    return 32


# ---------------------------------------------------------------------------
# single-purpose batches (the operator layer and the parity tests use these)

def eval_batch(inst: ProjectInstance, orders: np.ndarray, mode: int, reverse: bool = False,
               want_starts: bool = True, group: int = 32):
    """evaluate_order for every row of `orders` on the GPU -> (cmax, starts|None)."""
    torch = _torch()
    L = _native.lib()
    di = device_instance(inst)
    require_time_packing(di.blob_host, mode)
    orders = np.ascontiguousarray(np.atleast_2d(orders), dtype=np.int32)
    B, n = orders.shape
    if n != di.n:
        raise ValueError(f"orders have {n} columns, instance has {di.n} activities")
    d_ord = to_dev(orders)
    cmax = torch.zeros(B, dtype=torch.int32, device="cuda")
    starts = torch.zeros((B, n), dtype=torch.int32, device="cuda") if want_starts else None
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    check(L.rcpsp_eval_batch(ptr(di.blob), ctypes.byref(di.shape), int(mode), ptr(d_ord), B, int(bool(reverse)),
                             ptr(cmax), ptr(starts), int(group), ptr(err), stream_handle()),
          "rcpsp_eval_batch")
    _raise_dev_err(err)
    return cmax.cpu().numpy(), (starts.cpu().numpy() if want_starts else None)


def filter_batch(inst: ProjectInstance, orders: np.ndarray, delta: int) -> list[np.ndarray]:
    """filter_moves for every row of `orders` -> list of (k, 2) move arrays."""
    torch = _torch()
    L = _native.lib()
    di = device_instance(inst)
    orders = np.ascontiguousarray(np.atleast_2d(orders), dtype=np.int32)
    B = orders.shape[0]
    cap = max(1, neighborhood_size(di.n, delta))
    out = torch.zeros((B, cap), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(B, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    check(L.rcpsp_filter_batch(ptr(di.blob), ctypes.byref(di.shape), ptr(to_dev(orders)), B,
                               int(delta), ptr(out), cap, ptr(cnt), ptr(err), stream_handle()),
          "rcpsp_filter_batch")
    _raise_dev_err(err)
    packed = out.cpu().numpy().view(np.uint32)
    res = []
    for b, k in enumerate(cnt.cpu().numpy()):
        mv = packed[b, :k]
        res.append(np.stack([(mv >> 16).astype(np.int32), (mv & 0xFFFF).astype(np.int32)], 1)
                   .reshape(-1, 2))
    return res


def pack_moves(moves: np.ndarray) -> np.ndarray:
    moves = np.asarray(moves, np.int64).reshape(-1, 2)
    return ((moves[:, 0] << 16) | moves[:, 1]).astype(np.uint32)


def run_chunk_batch(inst: ProjectInstance, mode: int, delta: int, orders, tabu_lists, heads,
                    budget, adopted, start_cmax, best_known, floor_cmax: int,
                    collect_trace: bool = True, group: int | None = None, threads: int = 512):
    """run_chunk for independent searches (one CTA each) -> dict of arrays."""
    torch = _torch()
    L = _native.lib()
    di = device_instance(inst)
    require_time_packing(di.blob_host, mode)
    orders = np.ascontiguousarray(np.atleast_2d(orders), np.int32)
    S, n = orders.shape
    tl = np.stack([pack_moves(t) for t in tabu_lists]).astype(np.uint32)
    T = tl.shape[1]
    nb = max(1, neighborhood_size(n, delta))
    budget = np.broadcast_to(np.asarray(budget, np.int32), (S,)).copy()
    tcap = max(1, int(budget.max())) if collect_trace else 1
    d_ord = to_dev(orders)
    d_tabu = to_dev(tl.view(np.int32))
    d_head = to_dev(np.asarray(heads, np.int32).reshape(S))
    vecs = [to_dev(np.broadcast_to(np.asarray(x, np.int32), (S,)).copy())
            for x in (budget, adopted, start_cmax, best_known)]
    best = torch.zeros((S, n), dtype=torch.int32, device="cuda")
    trace = torch.zeros((S, tcap), dtype=torch.int32, device="cuda") if collect_trace else None
    stats = torch.zeros((S, 8), dtype=torch.int64, device="cuda")
    mbuf = torch.zeros((S, nb), dtype=torch.int32, device="cuda")
    cbuf = torch.zeros((S, nb), dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    if group is not None:
        g = group
    elif mode == MODE_CAPACITY:
        g = pick_cap_group(n, len(inst.capacities), max(int(c) for c in inst.capacities))
    else:
        g = pick_group(n)
    check(L.rcpsp_run_chunk_batch(ptr(di.blob), ctypes.byref(di.shape), int(mode), int(delta), T, S, ptr(d_ord),
                                  ptr(d_tabu), ptr(d_head), *(ptr(v) for v in vecs),
                                  int(floor_cmax), ptr(best), ptr(trace), tcap, ptr(stats),
                                  ptr(mbuf), ptr(cbuf), nb, int(g), int(threads), ptr(err),
                                  stream_handle()), "rcpsp_run_chunk_batch")
    _raise_dev_err(err)
    st = stats.cpu().numpy()
    tl_out = d_tabu.cpu().numpy().view(np.uint32)
    # the last iteration's compacted neighbourhood and its makespans
    n_last = st[:, 1] if int(budget.max()) == 1 else None
    mv = mbuf.cpu().numpy().view(np.uint32)
    cm = cbuf.cpu().numpy() & 0xFFFF   # high bits: evaluator flags (CONV_FLAG)
    last = None
    if n_last is not None:
        last = [(np.stack([(mv[b, :k] >> 16).astype(np.int32),
                           (mv[b, :k] & 0xFFFF).astype(np.int32)], 1).reshape(-1, 2),
                 cm[b, :k].copy()) for b, k in enumerate(n_last)]
    return dict(order=d_ord.cpu().numpy(), best_order=best.cpu().numpy(), stats=st,
                neighbourhood=last,
                trace=(trace.cpu().numpy() if collect_trace else None),
                tabu=np.stack([(tl_out >> 16).astype(np.int32),
                               (tl_out & 0xFFFF).astype(np.int32)], -1),
                heads=d_head.cpu().numpy())


def diversify_batch(inst: ProjectInstance, orders, phi_steps: int, rng_states: np.ndarray):
    """search.diversify on the GPU; rng_states (B, 6) uint64 advance in place."""
    L = _native.lib()
    di = device_instance(inst)
    orders = np.ascontiguousarray(np.atleast_2d(orders), np.int32)
    d_ord = to_dev(orders)
    d_rng = to_dev(np.ascontiguousarray(rng_states, np.uint64).view(np.int64))
    err = _torch().zeros(1, dtype=_torch().int32, device="cuda")
    check(L.rcpsp_diversify_batch(ptr(di.blob), ctypes.byref(di.shape), ptr(d_ord),
                                  orders.shape[0], int(phi_steps), ptr(d_rng), ptr(err),
                                  stream_handle()), "rcpsp_diversify_batch")
    _raise_dev_err(err)
    rng_states[...] = d_rng.cpu().numpy().view(np.uint64).reshape(rng_states.shape)
    return d_ord.cpu().numpy()


def rng_probe(seed_words: np.ndarray, ops: list[tuple[int, int]]) -> tuple[np.ndarray, np.ndarray]:
    """Run a sequence of (0, n) integers(n) / (1, k) permutation(k) draws on the GPU."""
    torch = _torch()
    L = _native.lib()
    st = to_dev(np.ascontiguousarray(seed_words, np.uint64).view(np.int64))
    o = np.asarray(ops, np.int32).reshape(-1, 2)
    total = int(sum(1 if kind == 0 else k for kind, k in o))
    out = torch.zeros(max(1, total), dtype=torch.int32, device="cuda")
    check(L.rcpsp_rng_probe(ptr(st), ptr(to_dev(o)), len(o), ptr(out), stream_handle()),
          "rcpsp_rng_probe")
    return out.cpu().numpy()[:total], st.cpu().numpy().view(np.uint64)


def eq8_probe(quads: np.ndarray) -> np.ndarray:
    torch = _torch()
    L = _native.lib()
    q = np.ascontiguousarray(quads, np.int64).reshape(-1, 4)
    out = torch.zeros(len(q), dtype=torch.int64, device="cuda")
    check(L.rcpsp_eq8_probe(ptr(to_dev(q)), len(q), ptr(out), stream_handle()),
          "rcpsp_eq8_probe")
    return out.cpu().numpy()


STATE_OPS = {"cap_es": 0, "cap_update": 1, "time_es": 2, "time_update": 3}


def state_op(inst: ProjectInstance, op: str, state: np.ndarray, act: int, arg: int = 0) -> int:
    """One resource-state step on the GPU (rcpsp_state_op); `state` (the
    reference's CAP [m][R_max] or TIME [m][H+1] int32 layout) is updated in
    place for the *_update ops.  Returns the earliest start for the *_es ops."""
    torch = _torch()
    L = _native.lib()
    di = device_instance(inst)
    d_state = to_dev(np.ascontiguousarray(state, np.int32))
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    check(L.rcpsp_state_op(ptr(di.blob), ctypes.byref(di.shape), STATE_OPS[op], ptr(d_state), int(act), int(arg),
                           ptr(out), ptr(err), stream_handle()), "rcpsp_state_op")
    code = int(err.cpu()[0])
    if code == 8:
        raise ValueError(f"cap_update start {arg} below the capacity bound (Eq. 7) of "
                         f"activity {act}: the closed-form update needs a start an SGS "
                         "could produce")
    if code:
        raise ValueError("resource state holds values outside the packed lane range")
    if op.endswith("update"):
        state[...] = d_state.cpu().numpy().reshape(state.shape)
    return int(out.cpu()[0])


def smem_bandwidth(iters: int = 4096, reps: int = 5) -> float:
    """Measured shared-memory load bandwidth of this GPU in GB/s (best of reps)."""
    torch = _torch()
    L = _native.lib()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, threads = sms * 2, 1024
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    best = 0.0
    for r in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        check(L.rcpsp_smem_probe(blocks, threads, iters, ptr(sink), stream_handle()),
              "rcpsp_smem_probe")
        e1.record()
        e1.synchronize()
        if r:
            best = max(best, blocks * threads * iters * 64 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


DEV_ERRORS = {1: "bad instance blob", 2: "no resource window before the horizon "
              "(demand above capacity?)", 3: "shared memory plan", 4: "tabu move outside the "
              "delta band", 5: "precedence cycle", 6: "bad move",
              7: "pool-min invariant violated: global best above a pool entry",
              8: "cap_update start below the capacity bound (Eq. 7)"}


def _raise_dev_err(err) -> None:
    code = int(err.cpu()[0])
    if code:
        raise RuntimeError(f"device error {code}: {DEV_ERRORS.get(code, '?')}")


# ---------------------------------------------------------------------------
# the full on-device orchestrate for a batch of instances

@dataclass
class SolveConfig:
    """Everything one batch solve needs (the reference's SearchParams plus the
    device choices).  Every device choice is result-neutral: evaluator groups,
    prefix reuse, clusters and CTA sizes give the same makespans and, for one
    worker per instance, the same trajectories."""

    total_iters: int
    workers: int
    pool_size: int
    tabu_size: int
    delta: int
    phi_steps: int
    phi_max: int
    seed: int
    collect_trace: bool = False
    grant_cap: int = 0
    group: int | None = None
    threads: int = 0          # 0 = auto (two CTAs per SM when they fit)
    steal: bool = True        # B > 1: idle workers help instances with budget left
    full_sgs: bool = False    # True: no prefix reuse in the group-32 evaluators
    cap_group: int | None = None  # CAPACITY: 32 = warp, 1 = thread per schedule, None = auto
    cluster: int | None = None    # CTAs per worker (1..8, prefix-reusing evaluators), None = auto
    time_limit_s: float | None = None  # wall-clock budget of the search on the device clock
    # TIME: per-warp profile slots; None = sized by a makespan bound when that
    # keeps more warps resident, 0 = always the horizon, > 0 = forced (tests)
    profile_slots: int | None = None

    @property
    def block_iters(self) -> int:
        return max(1, -(-self.total_iters // self.workers))


@dataclass
class BatchResult:
    best_cmax: np.ndarray            # [I]
    best_order: np.ndarray           # [I, n_max]
    best_mode: np.ndarray            # [I]
    critical_path: np.ndarray        # [I]
    iterations: np.ndarray           # [I] consumed
    evaluations: np.ndarray          # [I] pool + worker evaluations
    pool_evaluations: np.ndarray     # [I]
    exchanges: np.ndarray            # [I]
    diversifications: np.ndarray     # [I]
    forced: np.ndarray               # [I]
    stopped: np.ndarray              # [I] global best hit the critical path
    device_ms: float                 # pool init + search, CUDA events
    search_ms: float
    inst_wall_s: np.ndarray          # [I] per-instance search span (globaltimer)
    traces: list = field(default_factory=list)   # per instance: list of chunk arrays
    n_launches: int = 0
    sgs_steps: int = 0               # activity steps the workers' neighbourhood SGS ran
    wall_s: float = 0.0              # host perf_counter: upload + pool init + search (synced)


class BatchSolver:
    """All device buffers of one batch solve (instances x workers CTAs).

    Instances are grouped by (mode, packing words); each group is one
    pool-init and one search launch.  The working set of every instance stays
    in HBM for the whole solve; only final results are read back.
    """

    def __init__(self, instances: list[ProjectInstance], modes: list[int], cfg: SolveConfig,
                 pool_seeds: list[int] | None = None):
        torch = _torch()
        _native.lib()
        self.instances = instances
        self.modes = [int(m) for m in modes]
        self.cfg = cfg
        I = len(instances)
        blobs = [pack_instance(x) for x in instances]
        for b, md in zip(blobs, self.modes):
            require_time_packing(b, md)
        self.blobs_host = blobs
        offs = np.zeros(I, np.int64)
        offs[1:] = np.cumsum([len(b) for b in blobs[:-1]])
        self.blob_cat = np.concatenate(blobs)
        self.offs = offs
        self.n_max = max(int(b[B_N]) for b in blobs)
        self.h_max = max(int(b[B_H]) for b in blobs)
        self.e_max = max(int(b[B_E]) for b in blobs)
        self.m_max = max(int(b[B_M]) for b in blobs)
        self.rmax_max = max(int(b[B_RMAX]) for b in blobs)
        self.no_big = int(not any(int(b[B_BIG]) for b in blobs))
        self.sumcap_max = max(int(b[B_SUMCAP]) for b in blobs)
        # TIME: per-warp profile slots sized by a makespan bound -- twice the
        # larger of the energy and critical-path bounds plus the 64 slots a
        # booking keeps free, plus the scan pad (the kernel uses it only when
        # it keeps more warps resident; longer schedules fall back exactly)
        lb = max(max(int(b[B_LBRES]), int(b[B_CPM])) for b in blobs)
        self.prof_slots = 2 * lb + 64 + 32 + 32
        self.nbhd_max = max(1, max(neighborhood_size(int(b[B_N]), cfg.delta) for b in blobs))
        if self.nbhd_max >= KEY_LIMIT:
            raise UnsupportedInstance(f"neighbourhood of {self.nbhd_max} moves >= {KEY_LIMIT}")
        groups: dict[tuple[int, int], list[int]] = {}
        for i, b in enumerate(blobs):
            # the packing words size every kernel's instance staging, in both modes
            key = (self.modes[i], int(b[B_W]))
            groups.setdefault(key, []).append(i)
        self.groups = groups
        seeds = pool_seeds if pool_seeds is not None else [cfg.seed] * I
        self.pool_rng_host = np.stack([rng_words(s) for s in seeds])
        wr = np.stack([rng_words(cfg.seed ^ w) for w in range(cfg.workers)])
        self.w_rng_host = np.tile(wr[None], (I, 1, 1))
        F, T, B, n_max = cfg.pool_size, cfg.tabu_size, cfg.workers, self.n_max
        z = lambda shape, dt: torch.zeros(shape, dtype=dt, device="cuda")  # noqa: E731
        i32, i64 = torch.int32, torch.int64
        self.d_blob = z(len(self.blob_cat), i32)
        self.d_offs = z(I, i64)
        self.ws_lock = z(I, i32)
        self.ent_lock = z((I, F), i32)
        self.ws_hdr = z((I, 16), i64)
        self.ent_order = z((I, F, n_max), i32)
        self.ent_cmax = z((I, F), i32)
        self.ent_tabu = z((I, F, T), i32)
        self.ent_head = z((I, F), i32)
        self.ent_ic = z((I, F), i64)
        self.ent_reads = z((I, F), i64)
        self.best_order = z((I, n_max), i32)
        self.w_rng = z((I, B, 6), i64)
        self.w_stats = z((I, B, 16), i64)
        tcap = cfg.total_iters + 1 if cfg.collect_trace else 0
        self.trace_cap = tcap
        self.w_trace = z((I, B, max(1, tcap)), i32) if cfg.collect_trace else None
        self.w_chunks = z((I, B, max(1, tcap)), i32) if cfg.collect_trace else None
        grid_max = I * B
        self.moves_buf = z((grid_max, self.nbhd_max), i32)
        self.cmax_buf = z((grid_max, self.nbhd_max), i32)
        self.err = z(1, i32)
        self.t0 = torch.full((1,), np.iinfo(np.int64).max, dtype=torch.int64, device="cuda")
        self.d_pool_rng = z((I, 6), i64)
        self.d_ids = {k: z(len(v), i32) for k, v in groups.items()}
        self.launches = 0
        self.peer = None          # population.PeerExchange (live elite exchange), or None

    # -- host -> device inputs (the e2e measurement times this too)
    def upload(self, pinned: bool = False) -> int:
        """Copy the inputs to HBM; returns the bytes moved."""
        torch = _torch()
        pairs = [(self.d_blob, self.blob_cat), (self.d_offs, self.offs),
                 (self.d_pool_rng, self.pool_rng_host.view(np.int64)),
                 (self.w_rng, self.w_rng_host.view(np.int64))]
        pairs += [(self.d_ids[k], np.asarray(v, np.int32)) for k, v in self.groups.items()]
        moved = 0
        for dst, src in pairs:
            t = torch.from_numpy(np.ascontiguousarray(src))
            if pinned:
                t = t.pin_memory()
            dst.copy_(t.reshape(dst.shape), non_blocking=pinned)
            moved += t.numel() * t.element_size()
        return moved

    def reset(self) -> None:
        """Zero the working set and worker state (re-running the same batch)."""
        for t in (self.ws_lock, self.ent_lock, self.ws_hdr, self.ent_order, self.ent_cmax, self.ent_tabu,
                  self.ent_head, self.ent_ic, self.ent_reads, self.best_order, self.w_stats,
                  self.err):
            t.zero_()
        self.w_rng.copy_(_torch().from_numpy(self.w_rng_host.view(np.int64)).cuda())
        self.t0.fill_(np.iinfo(np.int64).max)
        if self.peer is not None:
            self.peer.reset()
        if self.w_trace is not None:
            self.w_trace.zero_()
            self.w_chunks.zero_()

    def args(self, epoch_limit: int | None = None, group_key=None) -> RcpspSolveArgs:
        cfg = self.cfg
        a = RcpspSolveArgs()
        a.blob, a.blob_off = ptr(self.d_blob), ptr(self.d_offs)
        a.n_inst, a.n_max = len(self.instances), self.n_max
        a.workers, a.pool_size, a.tabu_size = cfg.workers, cfg.pool_size, cfg.tabu_size
        a.delta, a.phi_steps, a.phi_max = cfg.delta, cfg.phi_steps, cfg.phi_max
        a.total_iters, a.block_iters = cfg.total_iters, cfg.block_iters
        a.epoch_limit = cfg.total_iters if epoch_limit is None else epoch_limit
        a.grant_cap, a.collect_trace = cfg.grant_cap, int(cfg.collect_trace)
        a.ws_lock, a.ws_hdr = ptr(self.ws_lock), ptr(self.ws_hdr)
        a.ent_lock = ptr(self.ent_lock)
        a.ent_order, a.ent_cmax, a.ent_tabu = ptr(self.ent_order), ptr(self.ent_cmax), ptr(self.ent_tabu)
        a.ent_head, a.ent_ic, a.ent_reads = ptr(self.ent_head), ptr(self.ent_ic), ptr(self.ent_reads)
        a.ws_best_order = ptr(self.best_order)
        a.w_rng, a.w_stats = ptr(self.w_rng), ptr(self.w_stats)
        a.w_trace, a.trace_cap = ptr(self.w_trace), self.trace_cap
        a.w_chunks, a.chunk_cap = ptr(self.w_chunks), self.trace_cap
        a.moves_buf, a.cmax_buf, a.nbhd_max = ptr(self.moves_buf), ptr(self.cmax_buf), self.nbhd_max
        a.err = ptr(self.err)
        a.h_max, a.e_max, a.m_max, a.rmax_max = self.h_max, self.e_max, self.m_max, self.rmax_max
        mode, words = group_key if group_key is not None else (MODE_TIME, 1)
        a.words = words
        if mode == MODE_CAPACITY:
            a.group = cfg.cap_group if cfg.cap_group is not None else pick_cap_group(
                self.n_max, self.m_max, self.rmax_max)
        else:
            a.group = cfg.group if cfg.group is not None else pick_group(self.n_max)
        a.threads = cfg.threads
        a.steal = int(cfg.steal and cfg.workers > 1 and not cfg.collect_trace)
        a.full_sgs = int(cfg.full_sgs)
        n_group = len(self.groups.get(group_key, [])) if group_key is not None else len(
            self.instances)
        a.cluster = (cfg.cluster if cfg.cluster is not None
                     else pick_cluster(n_group * cfg.workers))
        a.time_budget_ns = int(cfg.time_limit_s * 1e9) if cfg.time_limit_s else 0
        a.no_big = self.no_big
        a.sumcap_max = self.sumcap_max
        if cfg.profile_slots is None:
            a.prof_slots = self.prof_slots          # auto: used when it helps
        else:
            a.prof_slots = -int(cfg.profile_slots)  # forced (tests), 0 = off
        a.t0_ns = ptr(self.t0)
        if self.peer is not None:
            self.peer.fill_args(a)
        return a

    def pool_init(self, stream=None) -> None:
        L = _native.lib()
        for key, ids in self.groups.items():
            a = self.args(group_key=key)
            check(L.rcpsp_pool_init(a, ptr(self.d_ids[key]), len(ids), key[0],
                                    ptr(self.d_pool_rng), stream_handle(stream)),
                  "rcpsp_pool_init")
            self.launches += 3

    def search(self, epoch_limit: int | None = None, stream=None) -> None:
        L = _native.lib()
        for key, ids in self.groups.items():
            a = self.args(epoch_limit, group_key=key)
            check(L.rcpsp_solve(a, ptr(self.d_ids[key]), len(ids), key[0], stream_handle(stream)),
                  "rcpsp_solve")
            self.launches += 1

    def export_elites(self, elites, elite_cmax, stream=None) -> None:
        L = _native.lib()
        check(L.rcpsp_export_elites(self.args(), ptr(elites), ptr(elite_cmax),
                                    stream_handle(stream)), "rcpsp_export_elites")
        self.launches += 1

    def merge_elites(self, elites, elite_cmax, n_src: int, stream=None) -> None:
        L = _native.lib()
        check(L.rcpsp_merge_elites(self.args(), ptr(elites), ptr(elite_cmax), int(n_src),
                                   stream_handle(stream)), "rcpsp_merge_elites")
        self.launches += 1

    def collect(self, device_ms: float = 0.0, search_ms: float = 0.0) -> BatchResult:
        _raise_dev_err(self.err)
        hdr = self.ws_hdr.cpu().numpy()
        ws = self.w_stats.cpu().numpy()
        I = len(self.instances)
        pool = hdr[:, WS_FIELDS["pool_evals"]]
        evals = pool + hdr[:, WS_FIELDS["evaluations"]]
        t0 = hdr[:, WS_FIELDS["t0"]].astype(np.float64)
        t1 = hdr[:, WS_FIELDS["t1"]].astype(np.float64)
        span = np.where(t1 > 0, (t1 - t0) * 1e-9, 0.0)
        traces = []
        if self.w_trace is not None:
            tr = self.w_trace.cpu().numpy()
            ch = self.w_chunks.cpu().numpy()
            for i in range(I):
                pieces = []
                for w in range(self.cfg.workers):
                    nchunk = int(ws[i, w, WK_FIELDS["chunks"]])
                    p = 0
                    for c in ch[i, w, :nchunk]:
                        pieces.append(tr[i, w, p:p + int(c)].copy())
                        p += int(c)
                traces.append(pieces)
        return BatchResult(
            best_cmax=hdr[:, WS_FIELDS["best"]].astype(np.int64),
            best_order=self.best_order.cpu().numpy(),
            best_mode=hdr[:, WS_FIELDS["best_mode"]].astype(np.int64),
            critical_path=hdr[:, WS_FIELDS["floor"]].astype(np.int64),
            iterations=hdr[:, WS_FIELDS["consumed"]].astype(np.int64),
            evaluations=evals.astype(np.int64),
            pool_evaluations=pool.astype(np.int64),
            exchanges=hdr[:, WS_FIELDS["exchanges"]].astype(np.int64),
            diversifications=hdr[:, WS_FIELDS["diversifications"]].astype(np.int64),
            forced=hdr[:, WS_FIELDS["forced"]].astype(np.int64),
            stopped=hdr[:, WS_FIELDS["stop"]].astype(bool),
            device_ms=device_ms, search_ms=search_ms, inst_wall_s=span, traces=traces,
            n_launches=self.launches, sgs_steps=int(ws[:, :, WK_FIELDS["sgs_steps"]].sum()))

    def run(self, stream=None) -> BatchResult:
        """upload -> pool init -> search -> collect.  Device time from CUDA
        events around pool init + search; host wall time (perf_counter, the
        reference's clock, cooperation.py:254/273) around upload + pool init
        + search up to the stream synchronisation."""
        torch = _torch()
        s = stream or torch.cuda.current_stream()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        tick = time.perf_counter()
        self.upload()
        e0.record(s)
        self.pool_init(s)
        e1.record(s)
        self.search(stream=s)
        e2.record(s)
        e2.synchronize()
        wall = time.perf_counter() - tick
        res = self.collect(e0.elapsed_time(e2), e1.elapsed_time(e2))
        res.wall_s = wall
        return res
