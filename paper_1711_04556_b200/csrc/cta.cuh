// cta.cuh -- per-CTA search context and the building blocks of one tabu
// iteration: block reductions, the shared-memory tabu list, the neighbourhood
// filter (kernels.py:200-255, 263-277), shared-memory / cluster helpers.
#pragma once
#include "common.cuh"
#include "sgs.cuh"

namespace rt {

enum Scal {
  SC_NFEAS = 0, SC_KEYA, SC_KEYL, SC_CUR, SC_LBEST, SC_HEAD, SC_START, SC_FLAG, SC_TOTAL,
  SC_PICKU, SC_PICKV, SC_GRANT, SC_BESTK, SC_ADOPT, SC_ENTRY, SC_DIV, SC_NONE, SC_BASEC,
  SC_CTR, SC_STEPS, SC_BSTOK, SC_CMD, SC_NF, SC_IID, SC_PEERC, SC_PEERW, SC_FBLOCK, SC_WORDS = 32
};

struct CtaCtx {
  SInst I;
  int delta, T, nbhd;
  int* base;       // [n] current order
  int* pos;        // [n] position of each activity
  int* msp;        // [n] min successor position
  int* mpp;        // [n] max predecessor position
  int* rs;         // [n] row start of the flat neighbourhood (rows 1..n-2)
  int* best;       // [n] best order of the chunk
  int* rowc;       // [n] diversify row counts
  int* bst;        // [n] start of each activity in the current order's schedule
  uint32_t* tabu_list;  // [T] packed (u << 16) | v, 0 = empty slot
  uint32_t* tabu_cnt;   // [ceil(n*(delta+1)/32)] one bit per band move: in the list
  int* red;        // [72] reduction scratch
  int* scal;       // [SC_WORDS]
  int* evs;        // evaluation scratch (per warp)
  int* snap;       // CAPACITY group 32: uint16 [n/k][S] state after every k-th
                   // position of the current schedule (move starts, convergence)
  int snap_words;  // its capacity (32-bit words)
  int* fb;         // TIME group 32 with sized per-warp profiles: the full-horizon
                   // region for whole schedules (base pass, abandoned moves), or null
  int slots;       // TIME group 32: profile slots per warp
  int snap_k, snap_S;  // this instance's stride k and state size S
  int warp_words;  // evaluation scratch words per warp
  int cap_lanes;   // CAP: lanes per warp that evaluate (scratch stride)
  bool inc;        // TIME G = 32: reuse the current order's schedule prefix
  int csize;       // CTAs of this worker's cluster (1: no cluster); this CTA is the leader
  long long budget_ns;         // > 0: wall-clock budget of the launch (device clock)
  const long long* t0_ns;      // launch start
  uint32_t* moves_buf;  // global [nbhd] compacted moves
  int* cmax_buf;        // global [nbhd] makespans
  int* err;
};

// the snapshot stride of the staged instance: k = 1 unless n*S uint16 exceed
// the plan's snapshot capacity (all threads call; no barrier needed)
__device__ __forceinline__ void cta_snap_stride(CtaCtx& c) {
  int S = 0;
  for (int k = 0; k < c.I.m; ++k) S += c.I.cap[k];
  const int cap16 = 2 * c.snap_words;
  int k = 1;
  while (k < c.I.n && (c.I.n / k) * S > cap16) ++k;
  c.snap_S = S;
  c.snap_k = k;
}

// ---------------------------------------------------------------- block ops

__device__ __forceinline__ unsigned block_min_u32(unsigned v, int* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = __reduce_min_sync(FULL_MASK, v);
  if (lane == 0) red[warp] = static_cast<int>(v);
  __syncthreads();
  if (warp == 0) {
    unsigned x = lane < nw ? static_cast<unsigned>(red[lane]) : 0xffffffffu;
    x = __reduce_min_sync(FULL_MASK, x);
    if (lane == 0) red[64] = static_cast<int>(x);
  }
  __syncthreads();
  const unsigned r = static_cast<unsigned>(red[64]);
  __syncthreads();
  return r;
}

// exclusive scan of one int per thread; *total receives the block sum
__device__ __forceinline__ int block_excl_scan(int v, int* red, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL_MASK, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) red[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int x = lane < nw ? red[lane] : 0;
    int xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL_MASK, xi, o);
      if (lane >= o) xi += y;
    }
    red[32 + lane] = xi - x;
    if (lane == 31) red[64] = xi;
  }
  __syncthreads();
  const int r = red[32 + warp] + incl - v;
  *total = red[64];
  __syncthreads();
  return r;
}

// -------------------------------------------------------------- tabu (SMEM)
//
// The reference keeps an N x N counter table mirroring the circular list
// (tabu.py:21-63; counters so that a move held in two slots stays tabu until
// both are evicted).  Only moves with v - u <= delta ever enter the list, so a
// band of n*(delta+1) moves suffices, and one bit per move ("in the list")
// answers every query the search makes: on eviction the warp checks whether
// the evicted move still sits in another slot (one pass over the T slots, 32
// at a time) before clearing its bit.  n*(delta+1)/32 words instead of 16-bit
// counters: 300 activities, delta 60 -> 2.3 KB instead of 37 KB.

__device__ __forceinline__ int tabu_idx(const CtaCtx& c, int u, int v) {
  return u * (c.delta + 1) + (v - u);
}
__device__ __forceinline__ int tabu_get(const CtaCtx& c, int u, int v) {
  const int i = tabu_idx(c, u, v);
  return (c.tabu_cnt[i >> 5] >> (i & 31)) & 1u;
}

// tabu.py:52-60 (load: rebuild the membership bits); all threads call
__device__ __forceinline__ void cta_tabu_rebuild(const CtaCtx& c) {
  const int words = (c.I.n * (c.delta + 1) + 31) / 32;
  for (int i = threadIdx.x; i < words; i += blockDim.x) c.tabu_cnt[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < c.T; i += blockDim.x) {
    const uint32_t mv = c.tabu_list[i];
    if (mv != 0) {
      const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
      if (v - u < 0 || v - u > c.delta || u >= c.I.n) {
        set_err(c.err, DE_TABU_BAND);
      } else {
        const int k = tabu_idx(c, u, v);
        atomicOr(&c.tabu_cnt[k >> 5], 1u << (k & 31));
      }
    }
  }
  __syncthreads();
}

// kernels.py:263-277, by one warp: the slot at head takes (u, v); the move it
// held leaves the tabu set unless another slot still holds it.
__device__ __forceinline__ int tabu_add_warp(const CtaCtx& c, int head, int u, int v) {
  const int lane = threadIdx.x & 31;
  const uint32_t old = c.tabu_list[head];
  const uint32_t mv = (static_cast<uint32_t>(u) << 16) | static_cast<uint32_t>(v);
  bool again = false;
  if (old != 0u && old != mv)
    for (int j = lane; j < c.T; j += 32) again |= j != head && c.tabu_list[j] == old;
  again = __any_sync(FULL_MASK, again);
  if (lane == 0) {
    if (old != 0u && old != mv && !again) {
      const int k = tabu_idx(c, static_cast<int>(old >> 16), static_cast<int>(old & 0xffff));
      c.tabu_cnt[k >> 5] &= ~(1u << (k & 31));
    }
    c.tabu_list[head] = mv;
    const int k = tabu_idx(c, u, v);
    c.tabu_cnt[k >> 5] |= 1u << (k & 31);
  }
  __syncwarp();
  return (head + 1) % c.T;
}

// ----------------------------------------------------------- neighbourhood

// moves.py:60-72 rows: u = 1..n-3, v = u+1..min(u+delta, n-2)
__device__ __forceinline__ void cta_init_rows(CtaCtx& c) {
  const int n = c.I.n;
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int u = 1; u <= n - 2; ++u) {
      c.rs[u] = acc;
      if (u <= n - 3) acc += min(c.delta, n - 2 - u);
    }
    c.rs[0] = 0;
    c.nbhd = n >= 4 ? acc : 0;
    c.scal[SC_TOTAL] = c.nbhd;
  }
  __syncthreads();
  c.nbhd = c.scal[SC_TOTAL];
}

__device__ __forceinline__ void decode_move(const CtaCtx& c, int idx, int& u, int& v) {
  int lo = 1, hi = c.I.n - 3;  // largest u with rs[u] <= idx
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (c.rs[mid] <= idx) lo = mid; else hi = mid - 1;
  }
  u = lo;
  v = u + 1 + (idx - c.rs[u]);
}

// positions and precedence bounds of `ord`; all threads call
__device__ __forceinline__ void cta_bounds(const CtaCtx& c, const int* ord) {
  const int n = c.I.n;
  for (int p = threadIdx.x; p < n; p += blockDim.x) c.pos[ord[p]] = p;
  __syncthreads();
  for (int a = threadIdx.x; a < n; a += blockDim.x) {
    int lo = 0x7fffffff, hi = -1;
    for (int e = c.I.sptr[a]; e < c.I.sptr[a + 1]; ++e) lo = min(lo, c.pos[c.I.sdat[e]]);
    for (int e = c.I.pptr[a]; e < c.I.pptr[a + 1]; ++e) hi = max(hi, c.pos[c.I.pdat[e]]);
    c.msp[a] = lo;
    c.mpp[a] = hi;
  }
  __syncthreads();
}

// kernels.py:218-255 -> compacted lexicographic list in moves_buf; returns n_feas
__device__ __forceinline__ int cta_filter(CtaCtx& c) {
  cta_bounds(c, c.base);
  const int nb = c.nbhd, NT = blockDim.x, n = c.I.n;
  int K = (nb + NT - 1) / NT;
  K = K < 1 ? 1 : (K > 32 ? 32 : K);
  int total = 0;
  for (int tile = 0; tile < nb; tile += NT * K) {
    const int first = tile + threadIdx.x * K;
    uint32_t bits = 0;
    int u0 = 0, v0 = 0;
    if (first < nb) {
      decode_move(c, first, u0, v0);
      int u = u0, v = v0;
      for (int j = 0; j < K && first + j < nb; ++j) {
        if (v < c.msp[c.base[u]] && u > c.mpp[c.base[v]]) bits |= 1u << j;
        if (++v > min(u + c.delta, n - 2)) {
          ++u;
          v = u + 1;
        }
      }
    }
    int tot;
    int off = block_excl_scan(__popc(bits), c.red, &tot);
    if (bits) {
      int u = u0, v = v0;
      for (int j = 0; j < K && first + j < nb; ++j) {
        if (bits & (1u << j))
          c.moves_buf[total + off++] = (static_cast<uint32_t>(u) << 16) | static_cast<uint32_t>(v);
        if (++v > min(u + c.delta, n - 2)) {
          ++u;
          v = u + 1;
        }
      }
    }
    total += tot;
  }
  __syncthreads();
  return total;
}

// ------------------------------------------------------------- evaluation
//
// The evaluation phases are __noinline__ with scalar arguments (shared
// arrays as word offsets into the dynamic shared memory `dsm`), so the hot
// loops get their own register allocation, independent of the exchange /
// selection code around them, and every shared access stays an LDS/STS.

extern __shared__ __align__(16) int dsm[];

__device__ __forceinline__ int soff(const void* p) {
  return static_cast<int>(reinterpret_cast<const int*>(p) - dsm);
}

// cmax_buf entries of moves whose schedule converged to the current one carry
// this flag (makespans are < 2^16): when such a move is picked, the next
// iteration's current schedule has the same starts and needs no new pass
constexpr int CONV_FLAG = 1 << 30;

__device__ __forceinline__ int atom_inc_shared(uint32_t a) {
  int old;
  asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(a) : "memory");
  return old;
}

// ---- thread-block clusters: distributed shared memory of the leader (rank 0)
enum ClusterCmd { CMD_EVAL = 1, CMD_DONE = 2 };

__device__ __forceinline__ uint32_t cluster_map(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t ld_cluster(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int atom_add_cluster(uint32_t a, int v) {
  int old;
  asm volatile("atom.shared::cluster.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
// all threads of all CTAs of the cluster; release/acquire at cluster scope
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
// the launch's wall-clock budget is spent (device clock, %globaltimer)
__device__ __forceinline__ bool budget_spent(long long budget_ns, const long long* t0_ns) {
  if (budget_ns <= 0) return false;
  const long long t0 = *reinterpret_cast<const volatile long long*>(t0_ns);
  return static_cast<long long>(globaltimer()) - t0 >= budget_ns;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

}  // namespace rt
