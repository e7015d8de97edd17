// kernels.cu -- sm_100a kernels and the C ABI (include/rcpsp_tabu_b200.h).
//
// K1 k_eval_batch   evaluate_order over a batch of orders (kernels.py:152-194)
// K2 k_run_chunk    run_chunk, one CTA per independent search (kernels.py:316-385)
// K0 k_pool_*       initialize_working_set + FBI (cooperation.py:138-160,
//                   evaluator.py:187-266), one warp per pool entry
// K3 k_solve        persistent search: exchange (cooperation.py:82-135) +
//                   diversify (search.py:77-94) + run_adopted (search.py:144-173)
//                   per CTA, the working set in HBM behind a per-instance lock
// K4 k_merge_elites elite exchange between independent populations (multi-GPU)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <string>

#include "../../include/rcpsp_tabu_b200.h"
#include "common.cuh"
#include "pcg64.cuh"
#include "search.cuh"
#include "sgs.cuh"

using namespace rt;
static_assert(rt::DE_BAD_BLOB == RCPSP_DE_BAD_BLOB && rt::DE_NO_WINDOW == RCPSP_DE_NO_WINDOW &&
                  rt::DE_SMEM == RCPSP_DE_SMEM && rt::DE_TABU_BAND == RCPSP_DE_TABU_BAND &&
                  rt::DE_CYCLE == RCPSP_DE_CYCLE && rt::DE_BAD_MOVE == RCPSP_DE_BAD_MOVE &&
                  rt::DE_POOL_MIN == RCPSP_DE_POOL_MIN && rt::DE_CAP_START == RCPSP_DE_CAP_START,
              "device error codes: common.cuh and the public header agree");

namespace {

enum WsField {
  WS_CURSOR = 0, WS_TOTAL = 1, WS_PLANNED = 2, WS_CONSUMED = 3, WS_STOP = 4, WS_BEST = 5,
  WS_BEST_MODE = 6, WS_FLOOR = 7, WS_POOL_EVALS = 8, WS_T0 = 9, WS_T1 = 10, WS_ITERS = 11,
  WS_EVALS = 12, WS_EXCH = 13, WS_DIV = 14, WS_FORCED = 15
};
enum WkField {
  WK_ITERS = 0, WK_EVALS = 1, WK_EXCH = 2, WK_DIV = 3, WK_FORCED = 4, WK_CHUNKS = 5,
  WK_TRACE = 6, WK_T0 = 7, WK_T1 = 8, WK_STEPS = 9
};

thread_local std::string g_err;

int fail(const std::string& msg) {
  g_err = msg;
  return -1;
}

int cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}

struct Hdr {
  int n, m, H, e, W, lb, rmax, cpm;
};

}  // namespace

// The launch was sized from the caller's RcpspShape: the device blob must
// carry the same header (else DE_BAD_BLOB and the CTA leaves before staging).
__device__ __forceinline__ bool shape_ok(const int* __restrict__ blob, const RcpspShape& s,
                                         int* err) {
  const bool ok = blob[B_MAGIC] == BLOB_MAGIC && blob[B_N] == s.n && blob[B_M] == s.m &&
                  blob[B_H] == s.horizon && blob[B_E] == s.edges && blob[B_W] == s.words &&
                  blob[B_RMAX] == s.rmax && blob[B_SUMCAP] == s.sumcap;
  if (!ok && threadIdx.x == 0) set_err(err, DE_BAD_BLOB);
  return ok;
}

// k_solve's launch bound (2 CTAs per SM): the prefix-reusing TIME evaluator
// runs 18 warps per CTA at 56 registers (+4 % over 16 warps at 64 on j120;
// 20 warps at 48: +1.2…1.6 % on j120p/j120 but -1…-4 % on j30p/j60p, so the
// 20-warp instantiation, TIME_THREADS_LARGE, serves projects above 64
// activities only; profiles/r2/ab_launch_bounds.txt), so does the CAPACITY
// warp evaluator (+2.5…3.4 % on
// j60p/j120p/j120 over 16 warps, -3 % j30p); the thread-per-schedule one keeps
// 16 warps at 64 registers (at 56 it spills: -16 % on j120)
#ifndef CAP_THREADS
#define CAP_THREADS 576
#endif
#ifndef TIME_THREADS
#define TIME_THREADS 576
#endif
#ifndef TIME_THREADS_LARGE
#define TIME_THREADS_LARGE 640
#endif
__host__ __device__ constexpr int ksolve_threads(int mode, int G) {
  return mode == MODE_TIME && G == 32 ? TIME_THREADS
                                      : (mode == MODE_CAPACITY && G == 32 ? CAP_THREADS : 512);
}
constexpr int KSOLVE_THREADS_MAX = TIME_THREADS > CAP_THREADS ? (TIME_THREADS > 512 ? TIME_THREADS : 512)
                                                              : (CAP_THREADS > 512 ? CAP_THREADS : 512);

// =========================================================================
// K1: batch evaluation

template <int MODE, int G, int W>
__global__ void __launch_bounds__(256) k_eval_batch(const int* __restrict__ blob, RcpspShape sh,
                                                    const int* __restrict__ orders, int batch,
                                                    int reverse, int* __restrict__ cmax,
                                                    int* __restrict__ starts, int cap_lanes,
                                                    int* err) {
  if (!shape_ok(blob, sh, err)) return;
  int* smem = dsm;
  SInst I;
  const int used = align4(stage_instance(blob, smem, I));
  __syncthreads();
  const int n = I.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int* pp = reverse ? I.pptr : I.sptr;  // push graph (see sgs.cuh)
  const int* pd = reverse ? I.pdat : I.sdat;
  int* scratch = smem + used;
  if constexpr (MODE == MODE_TIME) {
    constexpr int S = 32 / G;
    const int grp = lane / G, lane_g = lane & (G - 1);
    const int gwords = (I.H + 1) * W + 2 * n;
    uint32_t* tau = reinterpret_cast<uint32_t*>(scratch + (warp * S + grp) * gwords);
    int* es = reinterpret_cast<int*>(tau) + (I.H + 1) * W;
    int* ord = es + n;
    const int b = (blockIdx.x * nw + warp) * S + grp;
    const bool active = b < batch;
    if (active)
      for (int p = lane_g; p < n; p += G) ord[p] = orders[static_cast<size_t>(b) * n + p];
    __syncwarp();
    if (!__any_sync(FULL_MASK, active)) return;
    int cm;
    if constexpr (G == 32) {
      if (!active) return;
      cm = sgs_time_warp<W>(sa(reverse ? I.info_r : I.info_f), sa(reverse ? I.pdat : I.sdat), sa(I.req), I.capw[0],
                            W == 2 ? I.capw[1] : 0u, I.hi, n, I.H, sa(tau), sa(es), sa(ord),
                            starts ? starts + static_cast<size_t>(b) * n : nullptr, err);
    } else {
      cm = sgs_time_split<G, W>(sa(reverse ? I.info_r : I.info_f), sa(reverse ? I.pdat : I.sdat), sa(I.req), I.capw[0],
                                W == 2 ? I.capw[1] : 0u, I.hi, n, I.H, sa(tau), sa(es), sa(ord),
                                active, starts ? starts + static_cast<size_t>(b) * n : nullptr,
                                err);
    }
    if (active && lane_g == 0) cmax[b] = cm;
  } else if constexpr (G == 32) {
    const int words = cap_warp_words(n, I.m, I.rmax) + n;
    int* scr = scratch + warp * words;
    int* ord = scr + cap_warp_words(n, I.m, I.rmax);
    const int b = blockIdx.x * nw + warp;
    if (b >= batch) return;
    for (int p = lane; p < n; p += 32) ord[p] = orders[static_cast<size_t>(b) * n + p];
    __syncwarp();
    const int cm = sgs_cap_warp(sa(reverse ? I.info_r : I.info_f), sa(pd), sa(I.dem), I.cap, n,
                                I.m, cap_row_stride(I.rmax), sa(scr), sa(ord),
                                starts ? starts + static_cast<size_t>(b) * n : nullptr);
    if (lane == 0) cmax[b] = cm;
  } else {
    const int L = cap_lanes;
    const int words = cap_thread_words(n, I.m, I.rmax) + n;
    int* st = scratch + warp * L * words;
    int* ord = st + cap_thread_words(n, I.m, I.rmax) * L;
    const int b = (blockIdx.x * nw + warp) * L + lane;
    if (lane >= L || b >= batch) return;
    for (int p = 0; p < n; ++p) ord[p * L + lane] = orders[static_cast<size_t>(b) * n + p];
    cmax[b] = sgs_cap_thread(I, st, L, lane, [&](int p) { return ord[p * L + lane]; }, pp, pd,
                             starts ? starts + static_cast<size_t>(b) * n : nullptr);
  }
}

// =========================================================================
// K2: stand-alone run_chunk (parity / kernels.run_chunk drop-in)

template <int MODE, int G, int W>
__global__ void __launch_bounds__(512, 2) k_run_chunk(
    const int* __restrict__ blob, RcpspShape sh, int delta, int T, int* orders, uint32_t* tabu, int* heads,
    const int* budget, const int* adopted, const int* start_cmax, const int* best_known,
    int floor_cmax, int* best_orders, int* trace, int trace_cap, long long* stats,
    uint32_t* moves_buf, int* cmax_buf, int nbhd_max, SmemPlan plan, int* err, int C) {
  if (!shape_ok(blob, sh, err)) return;
  int* smem = dsm;
  const int b = blockIdx.x / C;  // search index; C > 1: a cluster of CTAs per search
  CtaCtx c;
  cta_setup(c, blob, smem, plan, delta, T, moves_buf + static_cast<size_t>(b) * nbhd_max,
            cmax_buf + static_cast<size_t>(b) * nbhd_max, err);
  if constexpr ((MODE == MODE_TIME && G == 32) || MODE == MODE_CAPACITY) {
    if (C > 1) {
      if (cluster_rank() != 0) {
        cta_follow<MODE, G, W>(c, blob, nullptr, 0, smem, plan.inst, C);
        return;
      }
      c.csize = C;
      if (threadIdx.x == 0) c.scal[SC_IID] = 0;
    }
  }
  const int n = c.I.n;
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    c.base[p] = orders[static_cast<size_t>(b) * n + p];
    c.best[p] = c.base[p];
  }
  for (int i = threadIdx.x; i < T; i += blockDim.x) c.tabu_list[i] = tabu[static_cast<size_t>(b) * T + i];
  if (threadIdx.x == 0) c.scal[SC_HEAD] = heads[b] % T;
  __syncthreads();
  cta_tabu_rebuild(c);
  ChunkOut o = run_chunk_cta<MODE, G, W>(c, budget[b], adopted[b], start_cmax[b], best_known[b],
                                         floor_cmax,
                                         trace ? trace + static_cast<size_t>(b) * trace_cap : nullptr);
  if (c.csize > 1) {  // release the followers; keep this CTA alive until they are out
    if (threadIdx.x == 0) c.scal[SC_CMD] = CMD_DONE;
    __syncthreads();
    cluster_sync_all();
    cluster_sync_all();
  }
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    orders[static_cast<size_t>(b) * n + p] = c.base[p];
    best_orders[static_cast<size_t>(b) * n + p] = c.best[p];
  }
  for (int i = threadIdx.x; i < T; i += blockDim.x) tabu[static_cast<size_t>(b) * T + i] = c.tabu_list[i];
  if (threadIdx.x == 0) {
    heads[b] = c.scal[SC_HEAD];
    long long* s = stats + static_cast<size_t>(b) * 8;
    s[0] = o.iters; s[1] = o.evals; s[2] = o.improved; s[3] = o.local_best; s[4] = o.cur;
    s[5] = c.scal[SC_HEAD]; s[6] = o.forced; s[7] = 0;
  }
}

// =========================================================================
// filter / diversify / probes

__global__ void __launch_bounds__(256) k_filter_batch(const int* __restrict__ blob, RcpspShape sh,
                                                      const int* orders, int delta,
                                                      uint32_t* out_moves, int nbhd_cap,
                                                      int* out_count, SmemPlan plan, int* err) {
  if (!shape_ok(blob, sh, err)) return;
  int* smem = dsm;
  const int b = blockIdx.x;
  CtaCtx c;
  cta_setup(c, blob, smem, plan, delta, 1, out_moves + static_cast<size_t>(b) * nbhd_cap, nullptr,
            nullptr);
  for (int p = threadIdx.x; p < c.I.n; p += blockDim.x)
    c.base[p] = orders[static_cast<size_t>(b) * c.I.n + p];
  __syncthreads();
  const int k = cta_filter(c);
  if (threadIdx.x == 0) out_count[b] = k;
}

__global__ void __launch_bounds__(256) k_diversify(const int* __restrict__ blob, RcpspShape sh,
                                                   int* orders, int steps, uint64_t* rng_words,
                                                   SmemPlan plan, int* err) {
  if (!shape_ok(blob, sh, err)) return;
  int* smem = dsm;
  const int b = blockIdx.x;
  CtaCtx c;
  cta_setup(c, blob, smem, plan, 1, 1, nullptr, nullptr, nullptr);
  const int n = c.I.n;
  for (int p = threadIdx.x; p < n; p += blockDim.x) c.base[p] = orders[static_cast<size_t>(b) * n + p];
  Pcg64 rng;
  if (threadIdx.x == 0) rng.load(rng_words + static_cast<size_t>(b) * 6);
  __syncthreads();
  cta_diversify(c, c.base, steps, rng);
  for (int p = threadIdx.x; p < n; p += blockDim.x) orders[static_cast<size_t>(b) * n + p] = c.base[p];
  if (threadIdx.x == 0) rng.store(rng_words + static_cast<size_t>(b) * 6);
}

__global__ void k_rng_probe(uint64_t* state, const int* ops, int k, int* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Pcg64 g;
  g.load(state);
  int o = 0;
  for (int i = 0; i < k; ++i) {
    const int kind = ops[2 * i], n = ops[2 * i + 1];
    if (kind == 0) {
      out[o++] = static_cast<int>(g.integers(static_cast<uint32_t>(n)));
    } else {
      for (int j = 0; j < n; ++j) out[o + j] = j;
      g.permute(out + o, n);
      o += n;
    }
  }
  g.store(state);
}

// Eq. 8, cooperation.py:39-49 (same double-precision operation order)
__device__ __forceinline__ long long eq8(long long cmax, long long ic, long long block_iters,
                                         long long best) {
  const double quality = 0.8 * exp(-100.0 * (static_cast<double>(cmax) / static_cast<double>(best) - 1.0));
  const double intact = 0.2 * exp(-4.0 * (static_cast<double>(ic) / static_cast<double>(block_iters)));
  return static_cast<long long>(floor((static_cast<double>(block_iters) / 5.0) * (quality + intact)));
}

__global__ void k_eq8_probe(const long long* quad, int k, long long* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) out[i] = eq8(quad[4 * i], quad[4 * i + 1], quad[4 * i + 2], quad[4 * i + 3]);
}

// Shared-memory bandwidth probe (roofline denominator): every thread streams
// 128-bit loads over a 32 KB shared array; bytes = threads * iters * 64.
__global__ void __launch_bounds__(1024) k_smem_probe(int iters, int* sink) {
  __shared__ __align__(16) int4 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_int4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  int4 acc = make_int4(0, 0, 0, 0);
  int idx = threadIdx.x & 2047;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int4 v = buf[(idx + j * 32) & 2047];
      acc.x ^= v.x; acc.y += v.y; acc.z ^= v.z; acc.w += v.w;
    }
    idx = (idx + 128 + (acc.x & 1)) & 2047;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x7fffffff) sink[0] = 1;
}

// Single-step resource-state operations on the reference's state layouts
// (evaluator.py:30-107 wrappers of kernels.py:68-146), executed with the
// same device functions the SGS uses.  state: CAP -> int32 [m][R_max];
// TIME -> int32 [m][H+1] free units (packed into lane words in shared
// memory for the warp window search, unpacked back after an update).
enum StateOp { OP_CAP_ES = 0, OP_CAP_UPDATE = 1, OP_TIME_ES = 2, OP_TIME_UPDATE = 3 };

template <int W>
__global__ void __launch_bounds__(32) k_state_op(const int* __restrict__ blob, RcpspShape sh, int op,
                                                 int* state, int act, int arg, int* out, int* err) {
  if (!shape_ok(blob, sh, err)) return;
  int* smem = dsm;
  SInst I;
  const int used = align4(stage_instance(blob, smem, I));
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int m = I.m, R = I.rmax, H = I.H, dur = I.dur[act];
  const int* dem = I.dem + act * m;
  if (op == OP_CAP_ES) {
    if (lane == 0) out[0] = cap_es(state, 1, dem, I.cap, m, R);
    return;
  }
  if (op == OP_CAP_UPDATE) {  // the SGS's warp-wide closed form of Alg. 4
    // the closed form holds for starts at or above Eq. 7's bound -- the only
    // ones an SGS produces; a start below it is refused, state untouched
    if (dur > 0 && arg < cap_es(state, 1, dem, I.cap, m, R)) {
      if (lane == 0) set_err(err, DE_CAP_START);
      return;
    }
    int* st = smem + used;
    for (int j = lane; j < m * R; j += 32) st[j] = state[j];
    __syncwarp();
    const int capk = lane < m ? I.cap[lane] : 0, req = lane < m ? dem[lane] : 0;
    if (dur > 0) cap_update_all(sa(st), lane * R, m, capk, req, arg, dur);
    __syncwarp();
    for (int j = lane; j < m * R; j += 32) state[j] = st[j];
    if (lane == 0) out[0] = 0;
    return;
  }
  // TIME: pack [m][H+1] into lane words
  const int lb = blob[B_LB], lanes = 32 / lb;
  const uint32_t lmask = lb == 8 ? 0xffu : 0xffffu;
  uint32_t* tau = reinterpret_cast<uint32_t*>(smem + used);
  for (int t = lane; t <= H; t += 32)
    for (int w = 0; w < W; ++w) {
      uint32_t word = 0;
      for (int k = w * lanes; k < min(m, (w + 1) * lanes); ++k) {
        const int v = state[k * (H + 1) + t];
        if (v < 0 || static_cast<uint32_t>(v) > (lmask >> 1)) set_err(err, DE_BAD_BLOB);
        word |= (static_cast<uint32_t>(v) & lmask) << (lb * (k - w * lanes));
      }
      tau[t * W + w] = word;
    }
  __syncwarp();
  const uint32_t r0 = I.req[act * W], r1 = W == 2 ? I.req[act * W + 1] : 0u;
  const uint32_t cap0 = I.capw[0], cap1 = W == 2 ? I.capw[1] : 0u;
  if (op == OP_TIME_ES) {
    int start = arg;  // dur == 0 or es_prec >= H: the reference returns es_prec
    if (dur > 0 && arg < H)
      start = warp_window<W, true, true>(sa(tau), H + 1, H, r0, r1, cap0, cap1, I.hi, arg, dur,
                             window_mask(dur), nullptr);
    if (lane == 0) out[0] = start;
    return;
  }
  int hw = H + 1;
  if (dur > 0) warp_commit<W>(sa(tau), hw, arg, dur, r0, r1, cap0, cap1);
  __syncwarp();
  for (int t = lane; t <= H; t += 32)
    for (int k = 0; k < m; ++k) {
      const int w = k / lanes;
      state[k * (H + 1) + t] = static_cast<int>((tau[t * W + w] >> (lb * (k % lanes))) & lmask);
    }
  if (lane == 0) out[0] = 0;
}

// =========================================================================
// K0: working-set initialisation

// initial_order(shuffle=True) per pool entry (moves.py:42-57); one thread per
// instance consumes that instance's pool rng sequentially, as the reference.
__global__ void k_pool_orders(RcpspSolveArgs A, const int* ids, int n_ids,
                              const uint64_t* pool_rng) {
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= n_ids) return;
  const int iid = ids[slot];
  const int* blob = A.blob + A.blob_off[iid];
  const int n = blob[B_N], nl = blob[B_NLVL];
  const int* lptr = blob + blob[B_OFF_LPTR];
  const int* ldat = blob + blob[B_OFF_LDAT];
  Pcg64 g;
  g.load(pool_rng + static_cast<size_t>(iid) * 6);
  for (int f = 0; f < A.pool_size; ++f) {
    int* ord = A.ent_order + (static_cast<size_t>(iid) * A.pool_size + f) * A.n_max;
    for (int l = 0; l < nl; ++l) {
      const int a = lptr[l], b = lptr[l + 1];
      for (int i = a; i < b; ++i) ord[i] = ldat[i];
      if (b - a > 1) g.permute(ord + a, b - a);
    }
  }
}

// one warp evaluates `ord` (TIME: 32-lane group; CAP: lane 0); starts -> smem
template <int MODE, int W>
__device__ __forceinline__ int warp_eval(const SInst& I, int* scr, const int* ord, bool reverse,
                                         int* starts, int* err) {
  const int* pp = reverse ? I.pptr : I.sptr;
  const int* pd = reverse ? I.pdat : I.sdat;
  int cm;
  if constexpr (MODE == MODE_TIME) {
    cm = sgs_time_warp<W>(sa(reverse ? I.info_r : I.info_f), sa(reverse ? I.pdat : I.sdat), sa(I.req), I.capw[0],
                          W == 2 ? I.capw[1] : 0u, I.hi, I.n, I.H, sa(scr),
                          sa(scr + (I.H + 1) * W), sa(ord), starts, err);
  } else {
    (void)pp;
    cm = sgs_cap_warp(sa(reverse ? I.info_r : I.info_f), sa(pd), sa(I.dem), I.cap, I.n, I.m,
                      cap_row_stride(I.rmax), sa(scr), sa(ord), starts);
  }
  __syncwarp();
  return cm;
}

// _priority_topo (evaluator.py:187-205) by one warp: repeatedly emit the
// ready activity with the smallest (key, id).  deg_ptr gives the in-degree.
__device__ bool warp_ptopo(int n, const int* nxt_ptr, const int* nxt_dat, const int* deg_ptr,
                           const int* key, int* out, int* indeg, int* ready) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < n; i += 32) {
    indeg[i] = deg_ptr[i + 1] - deg_ptr[i];
    ready[i] = indeg[i] == 0;
  }
  __syncwarp();
  for (int k = 0; k < n; ++k) {
    unsigned long long best = ~0ull;
    for (int i = lane; i < n; i += 32)
      if (ready[i]) {
        const unsigned long long kk =
            (static_cast<unsigned long long>(static_cast<unsigned>(key[i]) ^ 0x80000000u) << 32) |
            static_cast<unsigned>(i);
        best = kk < best ? kk : best;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long y = __shfl_xor_sync(FULL_MASK, best, o);
      best = y < best ? y : best;
    }
    if (best == ~0ull) return false;
    const int sel = static_cast<int>(best & 0xffffffffu);
    __syncwarp();
    if (lane == 0) {
      out[k] = sel;
      ready[sel] = 0;
    }
    for (int e = nxt_ptr[sel] + lane; e < nxt_ptr[sel + 1]; e += 32) {
      const int j = nxt_dat[e];
      if (--indeg[j] == 0) ready[j] = 1;
    }
    __syncwarp();
  }
  return true;
}

__host__ __device__ inline int pool_entry_words(int mode, int n, int m, int H, int e, int W,
                                                int rmax) {
  const int inst = (inst_smem_words(n, m, e, W) + 3) & ~3;
  const int arrays = 8 * n;  // ord, s1, s2, key, indeg, ready, border/forder, final
  const int ev = mode == MODE_TIME ? (H + 1) * W + n : cap_warp_words(n, m, rmax);
  return inst + arrays + ev + 8;
}

// forward_backward_improve (evaluator.py:207-266) for even entries, then the
// evaluation of every entry (cooperation.py:146-157); one warp per entry.
template <int MODE, int W>
__global__ void __launch_bounds__(32) k_pool_entry(RcpspSolveArgs A, const int* ids) {
  int* smem = dsm;
  const int slot = blockIdx.x / static_cast<int>(A.pool_size);
  const int f = blockIdx.x % static_cast<int>(A.pool_size);
  const int iid = ids[slot];
  const int lane = threadIdx.x;
  SInst I;
  const int used = align4(stage_instance(A.blob + A.blob_off[iid], smem, I));
  __syncthreads();
  const int n = I.n;
  int* ord = smem + used;
  int* s1 = ord + n;
  int* s2 = s1 + n;
  int* key = s2 + n;
  int* indeg = key + n;
  int* ready = indeg + n;
  int* tmp = ready + n;
  int* fin = tmp + n;
  int* scr = fin + n;
  int* gord = A.ent_order + (static_cast<size_t>(iid) * A.pool_size + f) * A.n_max;
  for (int p = lane; p < n; p += 32) ord[p] = gord[p];
  __syncwarp();
  long long evals = 0;
  if (f % 2 == 0) {
    int cm = warp_eval<MODE, W>(I, scr, ord, false, s1, A.err);
    ++evals;
    for (;;) {
      for (int i = lane; i < n; i += 32) key[i] = -(s1[i] + I.dur[i]);
      __syncwarp();
      if (!warp_ptopo(n, I.pptr, I.pdat, I.sptr, key, tmp, indeg, ready)) set_err(A.err, DE_CYCLE);
      warp_eval<MODE, W>(I, scr, tmp, true, s2, A.err);
      ++evals;
      for (int i = lane; i < n; i += 32) key[i] = -(s2[i] + I.dur[i]);
      __syncwarp();
      if (!warp_ptopo(n, I.sptr, I.sdat, I.pptr, key, tmp, indeg, ready)) set_err(A.err, DE_CYCLE);
      const int ncm = warp_eval<MODE, W>(I, scr, tmp, false, s2, A.err);
      ++evals;
      if (ncm < cm) {
        for (int i = lane; i < n; i += 32) s1[i] = s2[i];
        cm = ncm;
        __syncwarp();
      } else {
        break;
      }
    }
    for (int i = lane; i < n; i += 32) key[i] = s1[i];
    __syncwarp();
    if (!warp_ptopo(n, I.sptr, I.sdat, I.pptr, key, fin, indeg, ready)) set_err(A.err, DE_CYCLE);
    for (int p = lane; p < n; p += 32) ord[p] = fin[p];
    __syncwarp();
  }
  const int cm = warp_eval<MODE, W>(I, scr, ord, false, s2, A.err);
  ++evals;
  for (int p = lane; p < n; p += 32) gord[p] = ord[p];
  if (lane == 0) {
    A.ent_cmax[static_cast<size_t>(iid) * A.pool_size + f] = cm;
    atomicAdd(reinterpret_cast<unsigned long long*>(&A.ws_hdr[static_cast<size_t>(iid) * 16 + WS_POOL_EVALS]),
              static_cast<unsigned long long>(evals));
  }
}

// WorkingSet.__init__ (cooperation.py:55-74)
__global__ void k_pool_finalize(RcpspSolveArgs A, const int* ids, int n_ids, int mode) {
  const int slot = blockIdx.x;
  if (slot >= n_ids) return;
  const int iid = ids[slot];
  const int* blob = A.blob + A.blob_off[iid];
  const int n = blob[B_N];
  __shared__ int s_best;
  if (threadIdx.x == 0) {
    int best = 0;
    const int* cm = A.ent_cmax + static_cast<size_t>(iid) * A.pool_size;
    for (int i = 1; i < A.pool_size; ++i)
      if (cm[i] < cm[best]) best = i;
    s_best = best;
    int64_t* H = A.ws_hdr + static_cast<size_t>(iid) * 16;
    H[WS_CURSOR] = 0;
    H[WS_TOTAL] = A.total_iters;
    H[WS_PLANNED] = 0;
    H[WS_CONSUMED] = 0;
    H[WS_BEST] = cm[best];
    H[WS_BEST_MODE] = mode;
    H[WS_FLOOR] = blob[B_CPM];
    H[WS_STOP] = cm[best] <= blob[B_CPM] ? 1 : 0;
    H[WS_T0] = 0x7fffffffffffffffll;
    H[WS_T1] = 0;
  }
  __syncthreads();
  const int* src = A.ent_order + (static_cast<size_t>(iid) * A.pool_size + s_best) * A.n_max;
  for (int p = threadIdx.x; p < n; p += blockDim.x)
    A.ws_best_order[static_cast<size_t>(iid) * A.n_max + p] = src[p];
}

// =========================================================================
// K3: the persistent search (run_worker loop, search.py:176-194)

__device__ __forceinline__ int64_t ldcg64(const int64_t* p) {
  return static_cast<int64_t>(__ldcg(reinterpret_cast<const unsigned long long*>(p)));
}

__device__ __forceinline__ void add64(int64_t* p, long long v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(v));
}

// ---- CTA-wide spin locks in global memory (thread 0 acquires, the CTA waits)
__device__ __forceinline__ void cta_lock(int* lk) {
  if (threadIdx.x == 0) {
    while (atomicCAS(lk, 0, 1) != 0) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}
__device__ __forceinline__ void cta_unlock(int* lk) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) atomicExch(lk, 0);
}

// ---- live elite exchange over peer memory (RcpspSolveArgs.outbox / peers)
__device__ __forceinline__ int ld_acquire_sys(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_volatile_g(const int32_t* p) {
  int v;
  asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Publish this population's new global best of instance iid (all threads;
// caller holds the instance lock, so there is one writer per outbox).
// Seqlock: seq odd while the order is being written, even once complete.
__device__ void publish_best(const RcpspSolveArgs& A, int iid, const int* best, int n, int cmax) {
  volatile int32_t* ob = A.outbox + static_cast<size_t>(iid) * RCPSP_OUTBOX_WORDS(A.n_max);
  const int tid = threadIdx.x;
  if (tid == 0) ob[0] = ob[0] + 1;
  __threadfence_system();
  __syncthreads();
  for (int p = tid; p < n; p += blockDim.x) ob[4 + p] = best[p];
  __threadfence_system();
  __syncthreads();
  if (tid == 0) {
    ob[1] = cmax;
    __threadfence_system();
    ob[0] = ob[0] + 1;
    __threadfence_system();
    if (A.peer_stats) atomicAdd(reinterpret_cast<unsigned long long*>(&A.peer_stats[1]), 1ull);
  }
  __syncthreads();
}

// Import the best new foreign elite of instance iid, if it beats the pool's
// worst entry and its makespan is not in the pool yet (k_merge_elites' rule):
// the entry takes the order, its tabu list is cleared, IC and reads reset,
// and the global best follows.  Warp 0 reads the peers (one per lane,
// n_peers <= 32) into `stage` (free shared scratch of n words); the writes
// take the instance's best lock, then the entry's lock, like a write-back.
template <int MODE>
__device__ void import_peer_elite(const RcpspSolveArgs& A, CtaCtx& c, int iid, int* stage,
                                  int64_t* Hd) {
  const int tid = threadIdx.x, lane = tid & 31, n = c.I.n;
  const int np = static_cast<int>(A.n_peers), F = static_cast<int>(A.pool_size),
            T = static_cast<int>(A.tabu_size);
  const size_t W = RCPSP_OUTBOX_WORDS(A.n_max);
  if (tid < 32) {
    int seq = 0;
    unsigned key = 0xffffffffu;
    const int32_t* pob = nullptr;
    if (lane < np) {
      pob = reinterpret_cast<const int32_t*>(A.peers[lane]) + static_cast<size_t>(iid) * W;
      seq = ld_acquire_sys(pob);
      const int cm = ld_volatile_g(pob + 1);
      const int seen = A.peer_seen[static_cast<size_t>(iid) * np + lane];
      if (seq != 0 && !(seq & 1) && seq != seen) key = (static_cast<unsigned>(cm) << 5) | lane;
    }
    const unsigned best = __reduce_min_sync(FULL_MASK, key);
    int go = 0, ccm = 0, worst = 0;
    if (best != 0xffffffffu) {
      const int src = static_cast<int>(best & 31u);
      ccm = static_cast<int>(best >> 5);
      const int sseq = __shfl_sync(FULL_MASK, seq, src);
      const int32_t* sob = reinterpret_cast<const int32_t*>(
          __shfl_sync(FULL_MASK, reinterpret_cast<unsigned long long>(pob), src));
      // the pool's worst entry (lowest index on ties) and the duplicate test
      unsigned wkey = 0;
      bool dup = false;
      for (int i = lane; i < F; i += 32) {
        const int v = __ldcg(&A.ent_cmax[static_cast<size_t>(iid) * F + i]);
        dup |= v == ccm;
        const unsigned k = (static_cast<unsigned>(v) << 16) | static_cast<unsigned>(0xffff - i);
        wkey = k > wkey ? k : wkey;
      }
      dup = __any_sync(FULL_MASK, dup);
      wkey = __reduce_max_sync(FULL_MASK, wkey);
      worst = 0xffff - static_cast<int>(wkey & 0xffffu);
      if (!dup && ccm < static_cast<int>(wkey >> 16)) {
        for (int p = lane; p < n; p += 32) stage[p] = ld_volatile_g(sob + 4 + p);
        __threadfence_system();
        __syncwarp();
        const int seq2 = __shfl_sync(FULL_MASK, lane == 0 ? ld_acquire_sys(sob) : 0, 0);
        go = seq2 == sseq;  // not overwritten meanwhile: a consistent order
        if (!go && lane == 0 && A.peer_stats)
          atomicAdd(reinterpret_cast<unsigned long long*>(&A.peer_stats[3]), 1ull);
      }
      // a consistent elite is consumed whether or not it enters the pool
      if (lane == 0 && (go || dup || ccm >= static_cast<int>(wkey >> 16)))
        A.peer_seen[static_cast<size_t>(iid) * np + src] = sseq;
    }
    if (lane == 0) {
      c.scal[SC_FLAG] = go;
      c.scal[SC_PEERC] = ccm;
      c.scal[SC_PEERW] = worst;
      if (A.peer_stats) atomicAdd(reinterpret_cast<unsigned long long*>(&A.peer_stats[2]), 1ull);
    }
  }
  __syncthreads();
  if (!c.scal[SC_FLAG]) return;
  const int ccm = c.scal[SC_PEERC], worst = c.scal[SC_PEERW];
  // the global best first (pool-min), then the entry
  cta_lock(&A.ws_lock[iid]);
  if (tid == 0) c.scal[SC_FLAG] = ccm < ldcg64(&Hd[WS_BEST]);
  __syncthreads();
  if (c.scal[SC_FLAG]) {
    for (int p = tid; p < n; p += blockDim.x)
      A.ws_best_order[static_cast<size_t>(iid) * A.n_max + p] = stage[p];
    if (tid == 0) {
      Hd[WS_BEST] = ccm;
      Hd[WS_BEST_MODE] = MODE;
    }
  }
  cta_unlock(&A.ws_lock[iid]);
  const size_t eo = static_cast<size_t>(iid) * F + worst;
  cta_lock(&A.ent_lock[eo]);
  if (tid == 0) c.scal[SC_FLAG] = ccm < __ldcg(&A.ent_cmax[eo]);  // still worse than the elite?
  __syncthreads();
  if (c.scal[SC_FLAG]) {
    for (int p = tid; p < n; p += blockDim.x) A.ent_order[eo * A.n_max + p] = stage[p];
    for (int i = tid; i < T; i += blockDim.x) A.ent_tabu[eo * T + i] = 0u;
    if (tid == 0) {
      A.ent_cmax[eo] = ccm;
      A.ent_head[eo] = 0;
      A.ent_ic[eo] = 0;
      A.ent_reads[eo] = 0;
      if (A.peer_stats) atomicAdd(reinterpret_cast<unsigned long long*>(&A.peer_stats[0]), 1ull);
    }
  }
  cta_unlock(&A.ent_lock[eo]);
}

// One CTA = one search worker.  Worker loop (search.run_worker): exchange
// with its instance's working set under the instance lock (cooperation.py:
// 276-329) -> optional diversify (search.py:77-94) -> evaluate the adopted
// order (search.py:134-142) -> run_chunk (kernels.py:316-385).  With
// A.steal, a worker whose instance has no budget left (or hit the critical
// path) moves on to the next instance of the launch that still has budget,
// so the batch finishes together; without it (the reference's fixed
// worker-to-pool mapping, and exact B = 1 trajectories) it exits.
template <int MODE, int G, int W, bool LONG = false>
__device__ __forceinline__ void solve_body(RcpspSolveArgs A, const int* __restrict__ ids, int n_ids,
                                           const SmemPlan& plan) {
  int* smem = dsm;
  const int B = static_cast<int>(A.workers);
  // with clusters (A.cluster > 1, TIME group 32 only) a worker is a cluster
  // of CTAs: rank 0 runs the search, the others only evaluate moves
  const int C = A.cluster > 1 ? static_cast<int>(A.cluster) : 1;
  const int wkr = blockIdx.x / C;  // worker index in the launch
  const int slot0 = wkr / B, wk = wkr % B;
  int slot = slot0;
  int iid = ids[slot];
  const int tid = threadIdx.x;
  const int F = static_cast<int>(A.pool_size), T = static_cast<int>(A.tabu_size);
  CtaCtx c;
  cta_setup(c, A.blob + A.blob_off[iid], smem, plan, static_cast<int>(A.delta), T,
            A.moves_buf + static_cast<size_t>(wkr) * A.nbhd_max,
            A.cmax_buf + static_cast<size_t>(wkr) * A.nbhd_max, A.err);
  c.inc = A.full_sgs == 0;
  // the shared-memory plan leaves out the TIME undo log only on the caller's
  // no_big guarantee: an instance that needs it stops the launch loudly
  if (A.no_big && c.I.big) {
    if (tid == 0) set_err(A.err, DE_SMEM);
    return;
  }
  if (A.time_budget_ns > 0) {
    c.budget_ns = A.time_budget_ns;
    c.t0_ns = reinterpret_cast<const long long*>(A.t0_ns);
    if (tid == 0)
      atomicMin(reinterpret_cast<unsigned long long*>(A.t0_ns),
                static_cast<unsigned long long>(globaltimer()));
  }
  if constexpr ((MODE == MODE_TIME && G == 32) || MODE == MODE_CAPACITY) {
    if (C > 1) {
      if (cluster_rank() != 0) {
        cta_follow<MODE, G, W, LONG>(c, A.blob, A.blob_off, iid, smem, plan.inst, C);
        return;
      }
      c.csize = C;
      if (tid == 0) c.scal[SC_IID] = iid;
    }
  }
  const size_t wid = static_cast<size_t>(iid) * B + wk;  // this worker's rng / stats slot
  int64_t* st = A.w_stats + wid * 16;
  int* wtrace = A.collect_trace ? A.w_trace + wid * A.trace_cap : nullptr;
  int* wchunks = A.collect_trace ? A.w_chunks + wid * A.chunk_cap : nullptr;
  const bool steal = A.steal != 0 && !A.collect_trace;
  Pcg64 rng;
  long long chunks = st[WK_CHUNKS], tlen = st[WK_TRACE];
  if (tid == 0) {
    rng.load(A.w_rng + wid * 6);
    if (st[WK_T0] == 0) st[WK_T0] = static_cast<long long>(globaltimer());
  }
  int64_t* Hd = A.ws_hdr + static_cast<size_t>(iid) * 16;
  if (tid == 0) atomicMin(reinterpret_cast<unsigned long long*>(&Hd[WS_T0]), globaltimer());
  int entry = -1, improved = 0, local_best = 0;
  long long granted = 0, used = 0, polls = 0;
  int hops = 0;
  for (;;) {
    // ---------------- exchange (cooperation.py:82-135), fine-grained: the
    // instance lock ws_lock[iid] guards only the global best (taken by a
    // worker that improves it), every pool entry has its own lock
    // (ent_lock), the budget counters are atomics.  A single worker (B = 1)
    // performs the reference's sequence of updates exactly; with B > 1 the
    // workers of an instance no longer queue behind one another.
    if (entry >= 0) {
      const size_t eo = static_cast<size_t>(iid) * F + entry;
      // 1. the global best first: it stays <= every pool entry (pool-min)
      if (tid == 0) c.scal[SC_FLAG] = improved && local_best < ldcg64(&Hd[WS_BEST]);
      __syncthreads();
      if (c.scal[SC_FLAG]) {
        cta_lock(&A.ws_lock[iid]);
        if (tid == 0) c.scal[SC_FLAG] = local_best < ldcg64(&Hd[WS_BEST]);
        __syncthreads();
        if (c.scal[SC_FLAG]) {
          int* bo = A.ws_best_order + static_cast<size_t>(iid) * A.n_max;
          for (int p = tid; p < c.I.n; p += blockDim.x) bo[p] = c.best[p];
          if (A.outbox) publish_best(A, iid, c.best, c.I.n, local_best);
          if (tid == 0) {
            Hd[WS_BEST] = local_best;
            Hd[WS_BEST_MODE] = MODE;
          }
        }
        cta_unlock(&A.ws_lock[iid]);
      }
      // 2. the entry (write back an improvement) and the budget counters
      if (improved) {
        cta_lock(&A.ent_lock[eo]);
        int* dst = A.ent_order + eo * A.n_max;
        for (int p = tid; p < c.I.n; p += blockDim.x) dst[p] = c.best[p];
        uint32_t* tl = A.ent_tabu + eo * T;
        for (int i = tid; i < T; i += blockDim.x) tl[i] = c.tabu_list[i];
        if (tid == 0) {
          A.ent_cmax[eo] = local_best;
          A.ent_head[eo] = c.scal[SC_HEAD];
          A.ent_reads[eo] = 0;
          A.ent_ic[eo] = ldcg64(&A.ent_ic[eo]) + used;
        }
        cta_unlock(&A.ent_lock[eo]);
      } else if (tid == 0) {
        add64(&A.ent_ic[eo], used);
      }
      if (tid == 0) {
        const long long unused = granted - used;
        if (unused > 0) add64(&Hd[WS_PLANNED], -unused);
        add64(&Hd[WS_CONSUMED], used);
      }
      entry = -1;
      improved = 0;
      // the reference's pool-min invariant after every write-back
      // (WorkingSet._assert_pool_min, cooperation.py:76-79, called by exchange):
      // entries read before the best, which only ever decreases
      __syncthreads();
      bool above = false;
      for (int i = tid; i < F; i += blockDim.x) {
        const long long v = __ldcg(&A.ent_cmax[static_cast<size_t>(iid) * F + i]);
        __threadfence();
        above |= v < ldcg64(&Hd[WS_BEST]);
      }
      if (__syncthreads_or(above) && tid == 0) set_err(A.err, DE_POOL_MIN);
    }
    // live elite exchange: poll the other populations' outboxes (c.best is
    // free here: the write-back above has consumed it)
    if (A.n_peers > 0 && ++polls % A.poll_every == 0)
      import_peer_elite<MODE>(A, c, iid, c.best, Hd);
    // ---------------- stop test, then the next entry round robin
    if (tid == 0) {
      const long long best = ldcg64(&Hd[WS_BEST]);
      if (best <= ldcg64(&Hd[WS_FLOOR])) Hd[WS_STOP] = 1;
      if (budget_spent(c.budget_ns, c.t0_ns)) Hd[WS_STOP] = 1;
      const bool none = ldcg64(&Hd[WS_STOP]) || ldcg64(&Hd[WS_PLANNED]) >= A.epoch_limit;
      c.scal[SC_NONE] = none ? 1 : 0;
      c.scal[SC_BESTK] = static_cast<int>(best);
      if (!none)
        c.scal[SC_ENTRY] = static_cast<int>(
            atomicAdd(reinterpret_cast<unsigned long long*>(&Hd[WS_CURSOR]), 1ull) %
            static_cast<unsigned long long>(F));
    }
    __syncthreads();
    if (!c.scal[SC_NONE]) {
      // adopt the entry under its lock: order, tabu list, Eq. 8 grant
      const size_t eo = static_cast<size_t>(iid) * F + c.scal[SC_ENTRY];
      cta_lock(&A.ent_lock[eo]);
      const int* src = A.ent_order + eo * A.n_max;
      for (int p = tid; p < c.I.n; p += blockDim.x) c.base[p] = __ldcg(&src[p]);
      const uint32_t* tl = A.ent_tabu + eo * T;
      for (int i = tid; i < T; i += blockDim.x) c.tabu_list[i] = __ldcg(&tl[i]);
      if (tid == 0) {
        const long long reads = ldcg64(&A.ent_reads[eo]) + 1;
        A.ent_reads[eo] = reads;
        const int ecm = __ldcg(&A.ent_cmax[eo]);
        long long grant = eq8(ecm, ldcg64(&A.ent_ic[eo]), A.block_iters, c.scal[SC_BESTK]);
        if (grant < 1) grant = 1;
        if (A.grant_cap > 0 && grant > A.grant_cap) grant = A.grant_cap;
        // claim the grant from the budget (another worker may have moved it)
        long long p = ldcg64(&Hd[WS_PLANNED]), g = 0;
        for (;;) {
          if (p >= A.epoch_limit) {
            g = 0;
            break;
          }
          g = grant;
          if (g > A.total_iters - p) g = A.total_iters - p;
          if (g > A.epoch_limit - p) g = A.epoch_limit - p;
          const long long q = static_cast<long long>(atomicCAS(
              reinterpret_cast<unsigned long long*>(&Hd[WS_PLANNED]),
              static_cast<unsigned long long>(p), static_cast<unsigned long long>(p + g)));
          if (q == p) break;
          p = q;
        }
        c.scal[SC_GRANT] = static_cast<int>(g);
        c.scal[SC_ADOPT] = ecm;
        c.scal[SC_DIV] = reads > A.phi_max ? 1 : 0;
        c.scal[SC_HEAD] = __ldcg(&A.ent_head[eo]) % T;
        if (g == 0) c.scal[SC_NONE] = 1;  // the budget ran out meanwhile (B > 1)
      }
      cta_unlock(&A.ent_lock[eo]);
    }
    if (c.scal[SC_NONE]) {
      if (tid == 0) atomicMax(reinterpret_cast<unsigned long long*>(&Hd[WS_T1]), globaltimer());
      if (!steal) break;
      // ---------------- move on to an instance that still has budget
      if (tid == 0) {
        int next = -1;
        for (int k = 1; k <= n_ids && next < 0; ++k) {
          const int s2 = (slot + k) % n_ids;
          const int64_t* H2 = A.ws_hdr + static_cast<size_t>(ids[s2]) * 16;
          if (!ldcg64(&H2[WS_STOP]) && ldcg64(&H2[WS_PLANNED]) < A.epoch_limit) next = s2;
        }
        c.scal[SC_FLAG] = next;
      }
      __syncthreads();
      const int next = c.scal[SC_FLAG];
      if (next < 0 || ++hops > 4 * n_ids) break;
      slot = next;
      iid = ids[slot];
      Hd = A.ws_hdr + static_cast<size_t>(iid) * 16;
      __syncthreads();
      stage_instance(A.blob + A.blob_off[iid], smem + plan.inst, c.I);
      if (tid == 0) c.scal[SC_IID] = iid;
      __syncthreads();
      if (A.no_big && c.I.big) {  // see the launch-entry check
        if (tid == 0) set_err(A.err, DE_SMEM);
        break;
      }
      if (c.snap) cta_snap_stride(c);
      cta_init_rows(c);
      continue;
    }
    entry = c.scal[SC_ENTRY];
    granted = c.scal[SC_GRANT];
    const int adopted = c.scal[SC_ADOPT];
    const int best_known = c.scal[SC_BESTK];
    const bool needs_div = c.scal[SC_DIV] != 0;
    cta_tabu_rebuild(c);
    // ---------------- run_worker body (search.py:189-194)
    if (needs_div) cta_diversify(c, c.base, static_cast<int>(A.phi_steps), rng);
    // ---------------- Worker.run_adopted (search.py:144-173)
    const int start_cmax = cta_eval_one<MODE, G, W>(c, c.base);
    for (int p = tid; p < c.I.n; p += blockDim.x) c.best[p] = c.base[p];
    __syncthreads();
    ChunkOut o = run_chunk_cta<MODE, G, W, LONG>(c, static_cast<int>(granted), adopted, start_cmax,
                                           best_known, c.I.cpm,
                                           wtrace ? wtrace + tlen : nullptr);
    used = o.iters;
    improved = o.improved;
    local_best = o.local_best;
    if (tid == 0) {
      // per-instance counters (RunStats) and per-worker ones (WorkerStats)
      add64(&Hd[WS_ITERS], o.iters);
      add64(&Hd[WS_EVALS], o.evals + 1);
      add64(&Hd[WS_EXCH], 1);
      add64(&Hd[WS_DIV], needs_div ? 1 : 0);
      add64(&Hd[WS_FORCED], o.forced);
      st[WK_ITERS] += o.iters;
      st[WK_EVALS] += o.evals + 1;
      st[WK_EXCH] += 1;
      st[WK_DIV] += needs_div ? 1 : 0;
      st[WK_FORCED] += o.forced;
      st[WK_STEPS] += o.steps;
    }
    if (wtrace) {
      if (tid == 0 && chunks < A.chunk_cap) wchunks[chunks] = o.iters;
      ++chunks;
      tlen += o.iters;
    }
  }
  if (c.csize > 1) {  // release the followers, then keep this CTA alive until they are out
    if (tid == 0) c.scal[SC_CMD] = CMD_DONE;
    __syncthreads();
    cluster_sync_all();
    cluster_sync_all();
  }
  if (tid == 0) {
    st[WK_CHUNKS] = chunks;
    st[WK_TRACE] = tlen;
    st[WK_T1] = static_cast<long long>(globaltimer());
    rng.store(A.w_rng + wid * 6);
  }
}

template <int MODE, int G, int W, int LB = ksolve_threads(MODE, G)>
__global__ void __launch_bounds__(LB, 2) k_solve(RcpspSolveArgs A, const int* __restrict__ ids,
                                                 int n_ids, SmemPlan plan) {
  // the large-project instantiation also takes the long-suffix evaluator
  solve_body<MODE, G, W, (LB != ksolve_threads(MODE, G))>(A, ids, n_ids, plan);
}

// One CTA per SM with up to 32 warps (64 registers), for launches whose
// shared memory leaves two CTAs per SM fewer warps -- 300 activities: TIME
// ran 16 warps per SM in one 512-thread CTA (the per-warp resource profile
// spans the horizon), CAPACITY 2 x 13.
template <int MODE, int G, int W>
__global__ void __launch_bounds__(1024, 1) k_solve_wide(RcpspSolveArgs A, const int* __restrict__ ids,
                                                        int n_ids, SmemPlan plan) {
  solve_body<MODE, G, W>(A, ids, n_ids, plan);
}

// =========================================================================
// K4: elite exchange between populations (multi-GPU)

__global__ void k_export_elites(RcpspSolveArgs A, int* elites, int* elite_cmax) {
  const int iid = blockIdx.x;
  const int n = A.blob[A.blob_off[iid] + B_N];
  for (int p = threadIdx.x; p < A.n_max; p += blockDim.x)
    elites[static_cast<size_t>(iid) * A.n_max + p] =
        p < n ? A.ws_best_order[static_cast<size_t>(iid) * A.n_max + p] : 0;
  if (threadIdx.x == 0) elite_cmax[iid] = static_cast<int>(A.ws_hdr[static_cast<size_t>(iid) * 16 + WS_BEST]);
}

__global__ void k_merge_elites(RcpspSolveArgs A, const int* elites, const int* elite_cmax, int n_src) {
  const int iid = blockIdx.x;
  const int n = A.blob[A.blob_off[iid] + B_N];
  const int F = static_cast<int>(A.pool_size), T = static_cast<int>(A.tabu_size);
  int64_t* Hd = A.ws_hdr + static_cast<size_t>(iid) * 16;
  __shared__ int s_slot, s_src;
  for (int s = 0; s < n_src; ++s) {
    if (threadIdx.x == 0) {
      s_slot = -1;
      const int cm = elite_cmax[static_cast<size_t>(s) * A.n_inst + iid];
      int worst = 0;
      const int* ec = A.ent_cmax + static_cast<size_t>(iid) * F;
      bool dup = false;
      for (int i = 0; i < F; ++i) {
        if (ec[i] > ec[worst]) worst = i;
        if (ec[i] == cm) dup = true;  // keep diversity: one entry per makespan value
      }
      if (!dup && cm < ec[worst]) {
        s_slot = worst;
        s_src = s;
        const size_t eo = static_cast<size_t>(iid) * F + worst;
        A.ent_cmax[eo] = cm;
        A.ent_head[eo] = 0;
        A.ent_ic[eo] = 0;
        A.ent_reads[eo] = 0;
        if (cm < Hd[WS_BEST]) {
          Hd[WS_BEST] = cm;
          s_slot = -(worst + 2);  // also copy into the global best
        }
      }
    }
    __syncthreads();
    if (s_slot != -1) {
      const int slot = s_slot >= 0 ? s_slot : -(s_slot + 2);
      const size_t eo = static_cast<size_t>(iid) * F + slot;
      const int* src = elites + (static_cast<size_t>(s_src) * A.n_inst + iid) * A.n_max;
      for (int p = threadIdx.x; p < n; p += blockDim.x) {
        A.ent_order[eo * A.n_max + p] = src[p];
        if (s_slot < -1) A.ws_best_order[static_cast<size_t>(iid) * A.n_max + p] = src[p];
      }
      for (int i = threadIdx.x; i < T; i += blockDim.x) A.ent_tabu[eo * T + i] = 0;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && Hd[WS_BEST] <= Hd[WS_FLOOR]) Hd[WS_STOP] = 1;
  __syncthreads();
  bool above = false;
  for (int i = threadIdx.x; i < F; i += blockDim.x)
    above |= A.ent_cmax[static_cast<size_t>(iid) * F + i] < Hd[WS_BEST];
  if (__syncthreads_or(above) && threadIdx.x == 0) set_err(A.err, DE_POOL_MIN);
}

// =========================================================================
// host side

namespace {

// launch shape from the caller's RcpspShape (no device read: every entry
// point stays asynchronous on its stream)
int shape_hdr(const RcpspShape* s, Hdr& h) {
  if (s == nullptr) return fail("null RcpspShape");
  if (s->n < 1 || s->m < 0 || s->horizon < 0 || s->edges < 0 || s->words < 0 || s->words > 2 ||
      s->rmax < 1)
    return fail("RcpspShape out of range (use rcpsp_blob_shape on the packed blob)");
  h.n = s->n; h.m = s->m; h.H = s->horizon; h.e = s->edges; h.W = s->words; h.lb = s->lane_bits;
  h.rmax = s->rmax; h.cpm = s->cpm;
  if (s->sumcap < 0 || s->sumcap > s->m * s->rmax) return fail("RcpspShape.sumcap out of range");
  return 0;
}

size_t smem_optin() {
  static int optin = -1;
  if (optin < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return static_cast<size_t>(optin);
}

size_t smem_per_sm() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  }
  return static_cast<size_t>(v);
}

// search-kernel plan: the most warps (<= want) and CAP lanes whose shared
// memory fits `limit` bytes
bool fit_plan_limit(int mode, int G, int W, int n, int m, int H, int e, int rmax, int delta,
                    int T, int want_threads, size_t limit, int min_threads, SmemPlan& p,
                    int& threads, int big = 1, int sumcap = 0, int slots = 0) {
  for (threads = want_threads; threads >= min_threads; threads -= 32) {
    for (int lanes = 32; lanes >= (mode == MODE_CAPACITY && G == 1 ? 1 : 32); --lanes) {
      p = plan_smem(mode, G, W, n, m, H, e, rmax, delta, T, threads / 32, lanes, big, sumcap,
                    slots);
      if (static_cast<size_t>(p.total) * 4 <= limit) return true;
    }
  }
  return false;
}

// want_threads == 0: prefer two resident CTAs per SM (>= 256 threads each),
// else one CTA with as many warps as fit
int sm_count() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  }
  return v;
}

// want_threads == 0 with a grid of `grid` CTAs: small projects (<= 64
// activities: short SGS, few moves per iteration) run more, smaller CTAs per
// SM when the grid fills them -- per-iteration barriers cost less and more
// searches progress at once (j30: 563 M vs ~400 M schedules/s with 8 x 128
// threads per SM, j60: 354 M vs 311 M; j120: 2 x 512 stays best)
bool fit_search_plan(int mode, int G, int W, int n, int m, int H, int e, int rmax, int delta,
                     int T, int want_threads, SmemPlan& p, int& threads, long long grid = 0,
                     int big = 1, int sumcap = 0, int slots = 0) {
  if (want_threads == 0 && n <= 64 && grid > 0) {
    const long long sms = sm_count();
    for (int per_sm : {8, 4}) {
      if (grid < per_sm * sms) continue;
      const int nt = 1024 / per_sm;
      const size_t lim = smem_per_sm() / per_sm - 1024;
      if (fit_plan_limit(mode, G, W, n, m, H, e, rmax, delta, T, nt, lim, nt, p, threads, big,
                         sumcap, slots))
        return true;
    }
  }
  if (want_threads == 0) {
    const size_t half = smem_per_sm() / 2 - 1024;
    if (fit_plan_limit(mode, G, W, n, m, H, e, rmax, delta, T, ksolve_threads(mode, G), half,
                       256, p, threads, big, sumcap, slots))
      return true;
    want_threads = 512;
  }
  return fit_plan_limit(mode, G, W, n, m, H, e, rmax, delta, T, want_threads, smem_optin(), 32, p,
                        threads, big, sumcap, slots);
}

template <class Kern>
int set_smem(Kern k, size_t bytes) {
  const size_t optin = smem_optin();
  if (bytes > optin)
    return fail("shared memory plan of " + std::to_string(bytes) + " B exceeds the " +
                std::to_string(optin) + " B per-CTA limit");
  return cuda_check(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bytes)),
                    "cudaFuncSetAttribute");
}

int launch_check(const char* what) { return cuda_check(cudaGetLastError(), what); }

// dispatch helper: calls f.template operator()<MODE,G,W>()
template <class Fn>
int dispatch(int mode, int group, int words, int m, Fn&& f) {
  if (mode == MODE_CAPACITY) {
    // group 1: one thread per schedule; otherwise one warp per schedule (lane = resource)
    if (group == 1) return f.template operator()<MODE_CAPACITY, 1, 1>();
    if (m > 32) return fail("CAPACITY group 32 supports at most 32 resources (use group 1)");
    return f.template operator()<MODE_CAPACITY, 32, 1>();
  }
  if (mode != MODE_TIME) return fail("mode must be 0 (CAPACITY) or 1 (TIME)");
  if (words != 1 && words != 2) return fail("TIME packing needs 1 or 2 words per slot");
  if (group == 32) return words == 1 ? f.template operator()<MODE_TIME, 32, 1>() : f.template operator()<MODE_TIME, 32, 2>();
  if (group == 16) return words == 1 ? f.template operator()<MODE_TIME, 16, 1>() : f.template operator()<MODE_TIME, 16, 2>();
  if (group == 8) return words == 1 ? f.template operator()<MODE_TIME, 8, 1>() : f.template operator()<MODE_TIME, 8, 2>();
  return fail("group must be 32, 16 or 8");
}

}  // namespace

extern "C" {

int rcpsp_abi_version(void) { return RCPSP_ABI_VERSION; }

const char* rcpsp_last_error(void) { return g_err.c_str(); }

int rcpsp_device_info(int* sm_count, int* smem_optin, int* cc_major, int* cc_minor) {
  int dev = 0;
  if (cuda_check(cudaGetDevice(&dev), "cudaGetDevice")) return -1;
  cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
  return 0;
}

int rcpsp_eval_batch(const int32_t* blob, const RcpspShape* shape, int mode, const int32_t* orders,
                     int batch, int reverse, int32_t* cmax, int32_t* starts, int group,
                     int32_t* err, void* stream) {
  if (batch <= 0) return 0;
  Hdr h;
  if (shape_hdr(shape, h)) return -1;
  const RcpspShape sh = *shape;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t limit = smem_optin();
  const size_t inst = (inst_smem_words(h.n, h.m, h.e, h.W) + 3) & ~3;
  return dispatch(mode, group, h.W, h.m, [&]<int MODE, int G, int W>() -> int {
    // largest warp count (<= 8) and CAP lane count (<= 32) whose scratch fits
    int nw = 8, lanes = 32;
    size_t words = 0;
    for (;;) {
      if (MODE == MODE_TIME)
        words = inst + static_cast<size_t>(nw) * (32 / G) * ((h.H + 1) * W + 2 * h.n);
      else if (G == 32)
        words = inst + static_cast<size_t>(nw) * (cap_warp_words(h.n, h.m, h.rmax) + h.n);
      else
        words = inst + static_cast<size_t>(nw) * lanes * (cap_thread_words(h.n, h.m, h.rmax) + h.n);
      if (words * 4 <= limit) break;
      if (nw > 1) nw >>= 1;
      else if (MODE == MODE_CAPACITY && lanes > 1) --lanes;
      else return fail("evaluation scratch does not fit in shared memory");
    }
    const int per_block = MODE == MODE_TIME ? nw * (32 / G) : (G == 32 ? nw : nw * lanes);
    const int blocks = (batch + per_block - 1) / per_block;
    auto k = k_eval_batch<MODE, G, W>;
    if (set_smem(k, words * 4)) return -1;
    k<<<blocks, nw * 32, words * 4, s>>>(blob, sh, orders, batch, reverse, cmax, starts, lanes, err);
    return launch_check("k_eval_batch");
  });
}

int rcpsp_filter_batch(const int32_t* blob, const RcpspShape* shape, const int32_t* orders,
                       int batch, int delta, uint32_t* out_moves, int nbhd_cap,
                       int32_t* out_count, int32_t* err, void* stream) {
  if (batch <= 0) return 0;
  Hdr h;
  if (shape_hdr(shape, h)) return -1;
  const int threads = 256;
  SmemPlan p = plan_smem(MODE_TIME, 32, h.W, h.n, h.m, 0, h.e, h.rmax, delta, 1, 0);
  if (set_smem(k_filter_batch, p.total * 4)) return -1;
  k_filter_batch<<<batch, threads, p.total * 4, static_cast<cudaStream_t>(stream)>>>(
      blob, *shape, orders, delta, out_moves, nbhd_cap, out_count, p, err);
  return launch_check("k_filter_batch");
}

int rcpsp_run_chunk_batch(const int32_t* blob, const RcpspShape* shape, int mode, int delta, int tabu_size, int batch,
                          int32_t* orders, uint32_t* tabu, int32_t* heads, const int32_t* budget,
                          const int32_t* adopted, const int32_t* start_cmax,
                          const int32_t* best_known, int floor_cmax, int32_t* best_orders,
                          int32_t* trace, int trace_cap, int64_t* stats, uint32_t* moves_buf,
                          int32_t* cmax_buf, int nbhd_max, int group, int threads, int32_t* err,
                          void* stream) {
  if (batch <= 0) return 0;
  if (tabu_size < 1) return fail("tabu_size must be >= 1");
  Hdr h;
  if (shape_hdr(shape, h)) return -1;
  const RcpspShape sh = *shape;
  if (threads % 32 || threads < 32 || threads > 512) return fail("threads must be 32..512, x32");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return dispatch(mode, group, h.W, h.m, [&]<int MODE, int G, int W>() -> int {
    SmemPlan p;
    int nt;
    if (!fit_search_plan(MODE, G, h.W, h.n, h.m, h.H, h.e, h.rmax, delta, tabu_size, threads, p, nt,
                         0, 1, shape->sumcap))
      return fail("search state does not fit in shared memory");
    auto k = k_run_chunk<MODE, G, W>;
    if (set_smem(k, p.total * 4)) return -1;
    // a small batch leaves SMs idle: spread each search over a cluster of up
    // to 8 CTAs when its evaluator deals moves from a shared counter
    const bool shared_counter = MODE == MODE_TIME ? G == 32 : (G == 32 || h.n >= 48);
    int C = shared_counter ? std::min(8, std::max(1, 2 * sm_count() / batch)) : 1;
    if (C == 1) {
      k<<<batch, nt, p.total * 4, s>>>(blob, sh, delta, tabu_size, orders, tabu, heads, budget,
                                            adopted, start_cmax, best_known, floor_cmax,
                                            best_orders, trace, trace_cap,
                                            reinterpret_cast<long long*>(stats), moves_buf,
                                            cmax_buf, nbhd_max, p, err, 1);
      return launch_check("k_run_chunk");
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(batch * C);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = p.total * 4;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cuda_check(cudaLaunchKernelEx(&cfg, k, blob, sh, delta, tabu_size, orders, tabu, heads, budget,
                                      adopted, start_cmax, best_known, floor_cmax, best_orders,
                                      trace, trace_cap, reinterpret_cast<long long*>(stats),
                                      moves_buf, cmax_buf, nbhd_max, p, err, C),
                   "k_run_chunk (cluster)"))
      return -1;
    return launch_check("k_run_chunk");
  });
}

int rcpsp_pool_init(const RcpspSolveArgs* args, const int32_t* inst_ids, int n_ids, int mode,
                    const uint64_t* pool_rng, void* stream) {
  if (n_ids <= 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  RcpspSolveArgs A = *args;
  k_pool_orders<<<(n_ids + 63) / 64, 64, 0, s>>>(A, inst_ids, n_ids,
                                                 pool_rng);
  if (launch_check("k_pool_orders")) return -1;
  const int words = pool_entry_words(mode, static_cast<int>(A.n_max), static_cast<int>(A.m_max),
                                     static_cast<int>(A.h_max), static_cast<int>(A.e_max),
                                     static_cast<int>(A.words), static_cast<int>(A.rmax_max));
  const int grid = n_ids * static_cast<int>(A.pool_size);
  int rc;
  if (mode == MODE_CAPACITY) {
    auto k = k_pool_entry<MODE_CAPACITY, 1>;
    if (set_smem(k, words * 4)) return -1;
    k<<<grid, 32, words * 4, s>>>(A, inst_ids);
    rc = launch_check("k_pool_entry");
  } else if (A.words == 1) {
    auto k = k_pool_entry<MODE_TIME, 1>;
    if (set_smem(k, words * 4)) return -1;
    k<<<grid, 32, words * 4, s>>>(A, inst_ids);
    rc = launch_check("k_pool_entry");
  } else {
    auto k = k_pool_entry<MODE_TIME, 2>;
    if (set_smem(k, words * 4)) return -1;
    k<<<grid, 32, words * 4, s>>>(A, inst_ids);
    rc = launch_check("k_pool_entry");
  }
  if (rc) return rc;
  k_pool_finalize<<<n_ids, 128, 0, s>>>(A, inst_ids, n_ids, mode);
  return launch_check("k_pool_finalize");
}

int rcpsp_solve(const RcpspSolveArgs* args, const int32_t* inst_ids, int n_ids, int mode,
                void* stream) {
  if (n_ids <= 0) return 0;
  RcpspSolveArgs A = *args;
  const int threads = static_cast<int>(A.threads);
  if (threads % 32 || threads < 0 || threads > KSOLVE_THREADS_MAX)
    return fail("threads must be 0 (auto) or 32.." + std::to_string(KSOLVE_THREADS_MAX) + ", x32");
  if (A.tabu_size < 1) return fail("tabu_size must be >= 1");
  if (A.ent_lock == nullptr) return fail("RcpspSolveArgs.ent_lock is required (ABI 8)");
  if (A.n_peers < 0 || A.n_peers > 32) return fail("n_peers must be 0..32");
  if (A.n_peers > 0 && (A.peers == nullptr || A.peer_seen == nullptr || A.poll_every < 1))
    return fail("peer exchange needs peers, peer_seen and poll_every >= 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return dispatch(mode, static_cast<int>(A.group), static_cast<int>(A.words), static_cast<int>(A.m_max),
                  [&]<int MODE, int G, int W>() -> int {
    if (threads > ksolve_threads(MODE, G))
      return fail("threads must be <= " + std::to_string(ksolve_threads(MODE, G)) +
                  " for this evaluator");
    SmemPlan p;
    int nt;
    if (!fit_search_plan(MODE, G, static_cast<int>(A.words), static_cast<int>(A.n_max), static_cast<int>(A.m_max),
                         static_cast<int>(A.h_max), static_cast<int>(A.e_max),
                         static_cast<int>(A.rmax_max), static_cast<int>(A.delta),
                         static_cast<int>(A.tabu_size), threads, p, nt,
                         static_cast<long long>(n_ids) * A.workers, A.no_big ? 0 : 1,
                         static_cast<int>(A.sumcap_max)))
      return fail("search state does not fit in shared memory");
    auto k = k_solve<MODE, G, W>;
#if TIME_THREADS_LARGE > 0
    // TIME on projects above 64 activities: 20 warps per CTA at 48 registers
    // when two such CTAs fit per SM (A/B on B200: +1.4 % on j120p; projects of
    // <= 64 activities run smaller CTAs at 56 registers, where 48 cost 1-4 %,
    // profiles/r2/ab_launch_bounds.txt)
    if constexpr (MODE == MODE_TIME && G == 32) {
      SmemPlan q;
      int tq;
      if (threads == 0 && A.n_max > 64 &&
          fit_plan_limit(MODE, G, static_cast<int>(A.words), static_cast<int>(A.n_max),
                         static_cast<int>(A.m_max), static_cast<int>(A.h_max),
                         static_cast<int>(A.e_max), static_cast<int>(A.rmax_max),
                         static_cast<int>(A.delta), static_cast<int>(A.tabu_size),
                         TIME_THREADS_LARGE, smem_per_sm() / 2 - 1024, TIME_THREADS_LARGE, q, tq,
                         A.no_big ? 0 : 1, static_cast<int>(A.sumcap_max))) {
        p = q;
        nt = tq;
        k = k_solve<MODE, G, W, TIME_THREADS_LARGE>;
      }
    }
#endif
    // Alternatives when the plan above is shared-memory-limited, the one that
    // keeps the most threads resident per SM wins (ties: the plan above):
    //  * the wide variant (one CTA per SM, up to 32 warps at 64 registers);
    //  * TIME: per-warp profiles sized by a makespan bound (A.prof_slots, no
    //    duration above 32; see eval_moves_time32_inc SIZED), two CTAs or wide.
    if constexpr (G == 32) {
      auto resident_of = [&](const SmemPlan& q, int t) {
        return static_cast<size_t>(q.total) * 4 > smem_per_sm() / 2 - 1024 ? t : 2 * t;
      };
      int best = resident_of(p, nt);
      SmemPlan q_forced;
      int tf;
      const int W_ = static_cast<int>(A.words), n_ = static_cast<int>(A.n_max),
                m_ = static_cast<int>(A.m_max), H_ = static_cast<int>(A.h_max),
                e_ = static_cast<int>(A.e_max), r_ = static_cast<int>(A.rmax_max),
                d_ = static_cast<int>(A.delta), T_ = static_cast<int>(A.tabu_size),
                big_ = A.no_big ? 0 : 1, sc_ = static_cast<int>(A.sumcap_max);
#ifndef NO_WIDE_CTA
      const bool try_alt = threads == 0 && A.n_max > 64 && best < 1024 && A.prof_slots >= 0;
#else
      const bool try_alt = false;
#endif
      const bool try_sized = try_alt && MODE == MODE_TIME && A.no_big && A.prof_slots > 0 &&
                             A.prof_slots < A.h_max + 1 + TAU_PAD;
      // prof_slots < 0: sized profiles of -prof_slots slots forced (tests)
      if (MODE == MODE_TIME && A.no_big && A.prof_slots < 0) {
        if (!fit_search_plan(MODE, G, W_, n_, m_, H_, e_, r_, d_, T_, threads, q_forced, tf,
                             static_cast<long long>(n_ids) * A.workers, big_, sc_,
                             static_cast<int>(-A.prof_slots)))
          return fail("search state does not fit in shared memory (forced profile slots)");
        p = q_forced;
        nt = tf;
      }
      SmemPlan q;
      int tq;
      if (try_alt && fit_plan_limit(MODE, G, W_, n_, m_, H_, e_, r_, d_, T_, 1024, smem_optin(),
                                    32, q, tq, big_, sc_) &&
          tq > best) {
        p = q; nt = tq; best = tq; k = k_solve_wide<MODE, G, W>;
      }
      const int sl = static_cast<int>(A.prof_slots);
      if (try_sized &&
          fit_search_plan(MODE, G, W_, n_, m_, H_, e_, r_, d_, T_, 0, q, tq,
                          static_cast<long long>(n_ids) * A.workers, big_, sc_, sl) &&
          resident_of(q, tq) > best) {
        p = q; nt = tq; best = resident_of(q, tq); k = k_solve<MODE, G, W>;
      }
      if (try_sized && fit_plan_limit(MODE, G, W_, n_, m_, H_, e_, r_, d_, T_, 1024,
                                      smem_optin(), 32, q, tq, big_, sc_, sl) &&
          tq > best) {
        p = q; nt = tq; best = tq; k = k_solve_wide<MODE, G, W>;
      }
    }
    if (set_smem(k, p.total * 4)) return -1;
    // clusters need a move counter to share: the prefix-reusing evaluators
    // (TIME group 32, CAPACITY group 32, CAPACITY group 1 from 48 activities)
    const bool shared_counter = MODE == MODE_TIME ? G == 32 : (G == 32 || A.n_max >= 48);
    int C = (shared_counter && A.full_sgs == 0) ? static_cast<int>(A.cluster) : 1;
    if (C < 1) C = 1;
    if (C > 8) return fail("cluster must be 1..8 CTAs");
    A.cluster = C;
    const int grid = n_ids * static_cast<int>(A.workers) * C;
    if (C == 1) {
      k<<<grid, nt, p.total * 4, s>>>(A, inst_ids, n_ids, p);
      return launch_check("k_solve");
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = p.total * 4;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cuda_check(cudaLaunchKernelEx(&cfg, k, A, inst_ids, n_ids, p), "k_solve (cluster)"))
      return -1;
    return launch_check("k_solve");
  });
}

int rcpsp_outbox_alloc(int64_t bytes, void** dev_ptr, void* handle) {
  if (bytes <= 0 || dev_ptr == nullptr || handle == nullptr) return fail("bad outbox request");
  if (cuda_check(cudaMalloc(dev_ptr, static_cast<size_t>(bytes)), "cudaMalloc(outbox)")) return -1;
  if (cuda_check(cudaMemset(*dev_ptr, 0, static_cast<size_t>(bytes)), "cudaMemset(outbox)"))
    return -1;
  cudaIpcMemHandle_t h;
  if (cuda_check(cudaIpcGetMemHandle(&h, *dev_ptr), "cudaIpcGetMemHandle")) return -1;
  std::memcpy(handle, &h, sizeof(h));
  return 0;
}

int rcpsp_outbox_open(const void* handle, void** dev_ptr) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return cuda_check(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess),
                    "cudaIpcOpenMemHandle");
}

int rcpsp_outbox_close(void* dev_ptr) {
  return cuda_check(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
}

int rcpsp_outbox_free(void* dev_ptr) { return cuda_check(cudaFree(dev_ptr), "cudaFree(outbox)"); }

int rcpsp_outbox_reset(void* dev_ptr, int64_t bytes, void* stream) {
  return cuda_check(cudaMemsetAsync(dev_ptr, 0, static_cast<size_t>(bytes),
                                    static_cast<cudaStream_t>(stream)),
                    "cudaMemsetAsync(outbox)");
}

int rcpsp_export_elites(const RcpspSolveArgs* args, int32_t* elites, int32_t* elite_cmax,
                        void* stream) {
  RcpspSolveArgs A = *args;
  k_export_elites<<<static_cast<int>(A.n_inst), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      A, elites, elite_cmax);
  return launch_check("k_export_elites");
}

int rcpsp_merge_elites(const RcpspSolveArgs* args, const int32_t* elites,
                       const int32_t* elite_cmax, int n_src, void* stream) {
  RcpspSolveArgs A = *args;
  k_merge_elites<<<static_cast<int>(A.n_inst), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      A, elites, elite_cmax, n_src);
  return launch_check("k_merge_elites");
}

int rcpsp_diversify_batch(const int32_t* blob, const RcpspShape* shape, int32_t* orders,
                          int batch, int phi_steps, uint64_t* rng, int32_t* err, void* stream) {
  if (batch <= 0) return 0;
  Hdr h;
  if (shape_hdr(shape, h)) return -1;
  SmemPlan p = plan_smem(MODE_TIME, 32, h.W, h.n, h.m, 0, h.e, h.rmax, 1, 1, 0);
  if (set_smem(k_diversify, p.total * 4)) return -1;
  k_diversify<<<batch, 256, p.total * 4, static_cast<cudaStream_t>(stream)>>>(
      blob, *shape, orders, phi_steps, rng, p, err);
  return launch_check("k_diversify");
}

int rcpsp_smem_probe(int blocks, int threads, int iters, int32_t* sink, void* stream) {
  k_smem_probe<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(iters, sink);
  return launch_check("k_smem_probe");
}

int rcpsp_state_op(const int32_t* blob, const RcpspShape* shape, int op, int32_t* state, int act,
                   int arg, int32_t* out, int32_t* err, void* stream) {
  Hdr h;
  if (shape_hdr(shape, h)) return -1;
  if (op < OP_CAP_ES || op > OP_TIME_UPDATE) return fail("unknown state op");
  if (op >= OP_TIME_ES && h.W == 0) return fail("instance has no TIME packing (CAPACITY only)");
  if (act < 0 || act >= h.n) return fail("activity out of range");
  const size_t words = ((inst_smem_words(h.n, h.m, h.e, h.W) + 3) & ~3) +
                       static_cast<size_t>(std::max((h.H + 1) * h.W, h.m * h.rmax)) + 4;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (h.W == 2) {
    if (set_smem(k_state_op<2>, words * 4)) return -1;
    k_state_op<2><<<1, 32, words * 4, s>>>(blob, *shape, op, state, act, arg, out, err);
  } else {
    if (set_smem(k_state_op<1>, words * 4)) return -1;
    k_state_op<1><<<1, 32, words * 4, s>>>(blob, *shape, op, state, act, arg, out, err);
  }
  return launch_check("k_state_op");
}

int rcpsp_rng_probe(uint64_t* state, const int32_t* ops, int k, int32_t* out, void* stream) {
  k_rng_probe<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      state, ops, k, out);
  return launch_check("k_rng_probe");
}

int rcpsp_eq8_probe(const int64_t* quad, int k, int64_t* out, void* stream) {
  if (k <= 0) return 0;
  k_eq8_probe<<<(k + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const long long*>(quad), k, reinterpret_cast<long long*>(out));
  return launch_check("k_eq8_probe");
}

}  // extern "C"
