// search.cuh -- one CTA runs one tabu search (run_chunk, kernels.py:316-385).
//
// Per iteration, all in one CTA, nothing leaves the SM except the compacted
// move list / makespans (L2-resident per-CTA scratch):
//   filter   Alg. 1 two-phase filter (kernels.py:218-255) as the equivalent
//            position test  v < minSuccPos(order[u]) && u > maxPredPos(order[v])
//            over the flat lexicographic neighbourhood, stable block-wide
//            compaction (ballot bits + block exclusive scan)
//   evaluate every surviving swap: TIME -> one G-lane group per schedule,
//            CAP -> one thread per schedule (sgs.cuh)
//   select   admissible = not tabu or C < aspiration; argmin over the packed
//            key (C << 16 | rank) = lexicographic tie break (kernels.py:280-309)
//   apply    swap + tabu_add on the shared-memory circular list with banded
//            16-bit counters (kernels.py:263-277)
#pragma once
#include "common.cuh"
#include "pcg64.cuh"
#include "sgs.cuh"

namespace rt {

enum Scal {
  SC_NFEAS = 0, SC_KEYA, SC_KEYL, SC_CUR, SC_LBEST, SC_HEAD, SC_START, SC_FLAG, SC_TOTAL,
  SC_PICKU, SC_PICKV, SC_GRANT, SC_BESTK, SC_ADOPT, SC_ENTRY, SC_DIV, SC_NONE, SC_BASEC,
  SC_CTR, SC_STEPS, SC_BSTOK, SC_CMD, SC_NF, SC_IID, SC_WORDS = 32
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
  uint32_t* tabu_cnt;   // [(n*(delta+1)+1)/2] two 16-bit counters per word
  int* red;        // [72] reduction scratch
  int* scal;       // [SC_WORDS]
  int* evs;        // evaluation scratch (per warp)
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

__device__ __forceinline__ int tabu_idx(const CtaCtx& c, int u, int v) {
  return u * (c.delta + 1) + (v - u);
}
__device__ __forceinline__ int tabu_get(const CtaCtx& c, int u, int v) {
  const int i = tabu_idx(c, u, v);
  return (c.tabu_cnt[i >> 1] >> ((i & 1) * 16)) & 0xffff;
}
__device__ __forceinline__ void tabu_bump(const CtaCtx& c, uint32_t mv, int d) {
  const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
  const int i = tabu_idx(c, u, v);
  atomicAdd(&c.tabu_cnt[i >> 1], static_cast<uint32_t>(d) << ((i & 1) * 16));
}

// tabu.py:52-60 (load: rebuild the counter mirror); all threads call
__device__ __forceinline__ void cta_tabu_rebuild(const CtaCtx& c) {
  const int words = (c.I.n * (c.delta + 1) + 1) / 2;
  for (int i = threadIdx.x; i < words; i += blockDim.x) c.tabu_cnt[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < c.T; i += blockDim.x) {
    const uint32_t mv = c.tabu_list[i];
    if (mv != 0) {
      const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
      if (v - u < 0 || v - u > c.delta || u >= c.I.n)
        set_err(c.err, DE_TABU_BAND);
      else
        tabu_bump(c, mv, 1);
    }
  }
  __syncthreads();
}

// kernels.py:263-277 (single thread)
__device__ __forceinline__ int tabu_add1(const CtaCtx& c, int head, int u, int v) {
  const uint32_t old = c.tabu_list[head];
  if (old != 0) {
    const int ou = static_cast<int>(old >> 16), ov = static_cast<int>(old & 0xffff);
    const int i = tabu_idx(c, ou, ov);
    c.tabu_cnt[i >> 1] -= 1u << ((i & 1) * 16);
  }
  const uint32_t mv = (static_cast<uint32_t>(u) << 16) | static_cast<uint32_t>(v);
  c.tabu_list[head] = mv;
  const int i = tabu_idx(c, u, v);
  c.tabu_cnt[i >> 1] += 1u << ((i & 1) * 16);
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

// TIME, one warp per schedule
template <int W>
__device__ __noinline__ void eval_moves_time32(int o_info, int o_pull, int o_req, int o_base,
                                               int o_evs, uint32_t cap0, uint32_t cap1,
                                               uint32_t hi, int n, int H,
                                               const uint32_t* __restrict__ moves,
                                               int* __restrict__ cmax_out, int n_feas,
                                               int warp_words, int* err) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int4* info = reinterpret_cast<const int4*>(dsm + o_info);
  const int* pull = dsm + o_pull;
  const uint32_t* req = reinterpret_cast<const uint32_t*>(dsm + o_req);
  const int* base = dsm + o_base;
  uint32_t* tau = reinterpret_cast<uint32_t*>(dsm + o_evs + warp * warp_words);
  int* es = dsm + o_evs + warp * warp_words + (H + 1) * W;
  int* ord = es + n;
  const uint32_t a_info = sa(info), a_push = sa(pull), a_req = sa(req), a_tau = sa(tau),
                 a_es = sa(es), a_ord = sa(ord);
  for (int idx = warp; idx < n_feas; idx += nw) {
    const uint32_t mv = moves[idx];
    const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
    for (int p = lane; p < n; p += 32) ord[p] = base[p == u ? v : (p == v ? u : p)];
    __syncwarp();
    const int cm = sgs_time_warp<W>(a_info, a_push, a_req, cap0, cap1, hi, n, H, a_tau, a_es,
                                    a_ord, nullptr, err);
    if (lane == 0) cmax_out[idx] = cm;
  }
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

// TIME, one warp per schedule, reusing the current order's schedule.
//
// For the swap (u, v) (u < v) the swapped order equals the current one on
// positions < u, so the serial SGS state after those positions is the
// current schedule's.  Each warp keeps that prefix state -- profile below
// the mark hw_pre, the finish times of the prefix activities, its makespan --
// and extends it with the known starts `bst` as its u grows: moves are
// handed out in increasing (lexicographic) index order by a shared counter,
// so a warp's u never decreases.  A move then schedules positions u.. only
// (precedence pulled: es = max over the predecessors' finish times, which
// the suffix overwrites for its own activities before any successor reads
// them), and undoes its bookings below hw_pre afterwards.
//
// Convergence: the SGS state after position p is a function of the starts
// of the activities at positions <= p.  If every activity at positions
// u..v starts where it does in the current schedule (the activities there
// are the same set), the state after v equals the current one and the rest
// of the schedule -- hence the makespan -- is the current schedule's.
//
// Every makespan equals the full SGS's (kernels.py:152-194); the work per
// move shrinks from n activity steps to the suffix.
//   o_bst: [n] starts of the current schedule; base_cmax: its makespan
//   o_ctr: shared move counter (zeroed by the caller)
//   per-warp scratch: tau (H+1)*W | fin [n] | log [2n] | ord [n + 1] (ord[n]: a
//   valid pad the unrolled loop's prefetch may read)
// The log lists the suffix bookings below hw_pre -- (start | dur << 16,
// packed demand (W = 1) or activity (W = 2)) -- the only ones the undo has to
// give back (a zero demand gives back nothing).
//   ctr_cl: != 0 -> the move counter (and the step counter after it) live in
//   the cluster leader's shared memory at this shared::cluster address
template <int W, bool BIG>
__device__ __noinline__ void eval_moves_time32_inc(int o_info, int o_pull, int o_req, int o_base,
                                                   int o_bst, int o_ctr, int o_evs, uint32_t cap0,
                                                   uint32_t cap1, uint32_t hi, int n, int H,
                                                   const uint32_t* __restrict__ moves,
                                                   int* __restrict__ cmax_out, int n_feas,
                                                   int warp_words, int base_cmax, int* err,
                                                   uint32_t ctr_cl) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* ws = dsm + o_evs + warp * warp_words;
  // o_info: pull records (info_r: duration, demand, predecessor span, mask);
  // o_pull: predecessor lists (pdat)
  const uint32_t a_info = sa(dsm + o_info), a_pdat = sa(dsm + o_pull), a_req = sa(dsm + o_req),
                 a_base = sa(dsm + o_base), a_bst = sa(dsm + o_bst), a_ctr = sa(dsm + o_ctr),
                 a_tau = sa(ws), a_fin = sa(ws + (H + 1) * W),
                 a_log = (a_fin + 4 * n + 7) & ~7u, a_ord = a_log + 8 * n;
  if (lane == 0) sts32(a_ord + 4 * n, 0u);
  int up = 0, hw_pre = 0, cm_pre = 0, steps = 0;
  // the last position holds the sink (every activity precedes it, and moves
  // never reach it): with zero duration it starts at max(es) <= cm, so it
  // cannot change the makespan and is not scheduled
  const int pend = lds128(a_info + 16 * static_cast<int>(lds32(a_base + 4 * (n - 1)))).x == 0
                       ? n - 1 : n;
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = ctr_cl ? atom_add_cluster(ctr_cl, 1) : atom_inc_shared(a_ctr);
    idx = __shfl_sync(FULL_MASK, idx, 0);
    if (idx >= n_feas) break;
    const uint32_t mv = moves[idx];
    const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
    // ---- extend the prefix to positions < u with the known starts
    for (; up < u; ++up) {
      const int act = static_cast<int>(lds32(a_base + 4 * up));
      const int4 rec = lds128(a_info + 16 * act);
      const int s = static_cast<int>(lds32(a_bst + 4 * act));
      const uint32_t r0 = static_cast<uint32_t>(rec.y);
      const uint32_t r1 = W == 2 ? lds32(a_req + 8 * act + 4) : 0u;
      if (rec.x > 0 && (r0 | r1) != 0) warp_commit<W, BIG>(a_tau, hw_pre, s, rec.x, r0, r1, cap0, cap1);
      const int fin = s + rec.x;
      cm_pre = max(cm_pre, fin);
      sts32_if(lane == 0, a_fin + 4 * act, static_cast<uint32_t>(fin));
      __syncwarp();
    }
    // ---- the swapped order's suffix u.. (materialised); fin of the prefix
    // activities holds their current finish times, the suffix overwrites its
    // own entries before any successor pulls them
    for (int q = u + lane; q < n; q += 32)
      sts32(a_ord + 4 * q, lds32(a_base + 4 * (q == u ? v : (q == v ? u : q))));
    __syncwarp();
    int hw = hw_pre, cm = cm_pre, p = u, nlog = 0;
    bool div = false;
    // log the bookings below hw_pre for the undo
    // (entry: start << 16 | activity; horizons are < 2^16, see KEY_LIMIT)
    auto log_below = [&](int act, const int4& rec, int st) {
      if (st < hw_pre && rec.x > 0) {
        if (lane == 0) sts64(a_log + 8 * nlog, (static_cast<uint32_t>(rec.x) << 16) | st,
                             W == 1 ? static_cast<uint32_t>(rec.y) : static_cast<uint32_t>(act));
        ++nlog;
      }
    };
    // phase A, positions u..v: until a start differs from the current
    // schedule's (then phase B) or v is reached with none differing
    // (converged: the rest is the current schedule)
    int act = static_cast<int>(lds32(a_ord + 4 * u));
    int4 rec = lds128(a_info + 16 * act);
    for (;;) {
      const int act_n = static_cast<int>(lds32(a_ord + 4 * (p + 1)));  // p + 1 <= v + 1 < n
      const int4 rec_n = lds128(a_info + 16 * act_n);
      const int st = time_step_pull<W, BIG>(act, rec, a_pdat, a_req, cap0, cap1, hi, H, a_tau,
                                            a_fin, hw, cm, err);
      log_below(act, rec, st);
      div = st != static_cast<int>(lds32(a_bst + 4 * act));
      if (div || p == v) {
        ++p;
        act = act_n;
        rec = rec_n;
        break;
      }
      ++p;
      act = act_n;
      rec = rec_n;
    }
    // phase B, positions p..pend-1 after a divergence; unrolled by two so the
    // prefetched next activity needs no register copies
    if (div && p < pend) {
      int act_a = act;
      int4 rec_a = rec;
      for (;;) {
        const int act_b = static_cast<int>(lds32(a_ord + 4 * (p + 1)));  // ord[n]: pad
        const int4 rec_b = lds128(a_info + 16 * act_b);
        int st = time_step_pull<W, BIG>(act_a, rec_a, a_pdat, a_req, cap0, cap1, hi, H,
                                          a_tau, a_fin, hw, cm, err);
        log_below(act_a, rec_a, st);
        if (++p >= pend) break;
        act_a = static_cast<int>(lds32(a_ord + 4 * (p + 1)));
        rec_a = lds128(a_info + 16 * act_a);
        st = time_step_pull<W, BIG>(act_b, rec_b, a_pdat, a_req, cap0, cap1, hi, H, a_tau,
                                      a_fin, hw, cm, err);
        log_below(act_b, rec_b, st);
        if (++p >= pend) break;
      }
    }
    if (lane == 0) cmax_out[idx] = div ? cm : (base_cmax | CONV_FLAG);
    steps += p - u;  // converged: p = v + 1; else pend
    // ---- undo the suffix's bookings below hw_pre
    __syncwarp();
    for (int k = 0; k < nlog; ++k) {
      const uint2 ent = lds64(a_log + 8 * k);
      uint32_t r0 = ent.y, r1 = 0u;
      if (W == 2) {
        r0 = lds32(a_req + 8 * ent.y);
        r1 = lds32(a_req + 8 * ent.y + 4);
      }
      warp_uncommit<W>(a_tau, hw_pre, static_cast<int>(ent.x & 0xffffu),
                       static_cast<int>(ent.x >> 16), r0, r1);
    }
    __syncwarp();
  }
  // SGS activity steps of this warp: suffixes + prefix extension
  if (lane == 0) {
    if (ctr_cl)
      atom_add_cluster(ctr_cl + 4, steps + up);
    else
      atomicAdd(&dsm[o_ctr + 1], steps + up);
  }
}

// TIME, G = 16 / 8 lanes per schedule (S = 32/G schedules per warp)
template <int G, int W>
__device__ __noinline__ void eval_moves_split(int o_info, int o_pull, int o_req, int o_base,
                                              int o_evs, uint32_t cap0, uint32_t cap1,
                                              uint32_t hi, int n, int H,
                                              const uint32_t* __restrict__ moves,
                                              int* __restrict__ cmax_out, int n_feas,
                                              int warp_words, int* err) {
  constexpr int S = 32 / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int grp = lane / G, lg = lane & (G - 1);
  const int gwords = (H + 1) * W + 2 * n;
  const int* base = dsm + o_base;
  int* tau = dsm + o_evs + warp * warp_words + grp * gwords;
  int* es = tau + (H + 1) * W;
  int* ord = es + n;
  const uint32_t a_info = sa(dsm + o_info), a_push = sa(dsm + o_pull), a_req = sa(dsm + o_req),
                 a_tau = sa(tau), a_es = sa(es), a_ord = sa(ord);
  for (int b = 0; b < n_feas; b += nw * S) {
    const int idx = b + warp * S + grp;
    const bool active = idx < n_feas;
    if (!__any_sync(FULL_MASK, active)) break;
    if (active) {
      const uint32_t mv = moves[idx];
      const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
      for (int p = lg; p < n; p += G) ord[p] = base[p == u ? v : (p == v ? u : p)];
    }
    __syncwarp();
    const int cm = sgs_time_split<G, W>(a_info, a_push, a_req, cap0, cap1, hi, n, H, a_tau, a_es,
                                        a_ord, active, nullptr, err);
    if (active && lg == 0) cmax_out[idx] = cm;
  }
}

// CAP, one warp per schedule (sgs.cuh: cap_step_warp), reusing the current
// order's schedule prefix like eval_moves_time32_inc.  Alg. 4 is not
// invertible and its state depends on the update order (not only on the set
// of starts), so there is no undo and no convergence exit: each move copies
// the prefix state (c_pre, es_pre) and schedules positions u..n-1.  With
// reuse == false the prefix stays empty (full SGS of every swapped order).
//   per-warp scratch: c [m*rs] | cb [m*rs] | es [n] | c_pre [m*rs] | es_pre [n]
__device__ __noinline__ void eval_moves_cap_warp(int o_info, int o_pull, int o_dem, int o_cap,
                                                 int o_base, int o_bst, int o_ctr, int o_evs,
                                                 int n, int m, int rs,
                                                 const uint32_t* __restrict__ moves,
                                                 int* __restrict__ cmax_out, int n_feas,
                                                 int warp_words, bool reuse, uint32_t ctr_cl) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mr = m * rs;
  const uint32_t a_scr = sa(dsm + o_evs + warp * warp_words);
  const uint32_t a_c = a_scr, a_cb = a_c + 4 * mr, a_es = a_cb + 4 * mr, a_cp = a_es + 4 * n,
                 a_esp = a_cp + 4 * mr;
  const uint32_t a_info = sa(dsm + o_info), a_push = sa(dsm + o_pull), a_dem = sa(dsm + o_dem),
                 a_base = sa(dsm + o_base), a_bst = sa(dsm + o_bst), a_ctr = sa(dsm + o_ctr);
  const int capk = lane < m ? dsm[o_cap + lane] : 0;
  for (int j = lane; j < mr; j += 32) sts32(a_cp + 4 * j, 0);
  for (int a = lane; a < n; a += 32) sts32(a_esp + 4 * a, 0);
  __syncwarp();
  int up = 0, cm_pre = 0, steps = 0;
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = ctr_cl ? atom_add_cluster(ctr_cl, 1) : atom_inc_shared(a_ctr);
    idx = __shfl_sync(FULL_MASK, idx, 0);
    if (idx >= n_feas) break;
    const uint32_t mv = moves[idx];
    const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
    const int u0 = reuse ? u : 0;
    // ---- extend the prefix state to positions < u0 with the known starts
    for (; up < u0; ++up) {
      const int act = static_cast<int>(lds32(a_base + 4 * up));
      const int4 rec = lds128(a_info + 16 * act);
      const int st = static_cast<int>(lds32(a_bst + 4 * act));
      if (rec.x > 0) {
        const int req = lane < m ? static_cast<int>(lds32(a_dem + 4 * (act * m + lane))) : 0;
        cap_commit_all(a_cp, a_cb, rs, m, capk, req, st, rec.x);
      }
      const int fin = st + rec.x;
      cm_pre = max(cm_pre, fin);
      const int e0 = rec.z & 0xffff, ecnt = rec.z >> 16;
      for (int e = lane; e < ecnt; e += 32) {
        const uint32_t adr = a_esp + 4 * lds32(a_push + 4 * (e0 + e));
        if (static_cast<int>(lds32(adr)) < fin) sts32(adr, static_cast<uint32_t>(fin));
      }
      __syncwarp();
    }
    for (int j = lane; j < mr; j += 32) sts32(a_c + 4 * j, lds32(a_cp + 4 * j));
    for (int a = lane; a < n; a += 32) sts32(a_es + 4 * a, lds32(a_esp + 4 * a));
    __syncwarp();
    // ---- positions u0.. of the swapped order
    int cm = cm_pre;
    for (int p = u0; p < n; ++p) {
      const int q = p == u ? v : (p == v ? u : p);
      const int act = static_cast<int>(lds32(a_base + 4 * q));
      const int4 rec = lds128(a_info + 16 * act);
      const int esv = static_cast<int>(lds32(a_es + 4 * act));
      cap_step_warp(act, rec.x, esv, a_dem, m, capk, rs, a_c, a_cb, a_push, rec.z & 0xffff,
                    rec.z >> 16, a_es, cm);
    }
    if (lane == 0) cmax_out[idx] = cm;
    steps += n - u0;
  }
  if (lane == 0) {
    if (ctr_cl)
      atom_add_cluster(ctr_cl + 4, steps + up);
    else
      atomicAdd(&dsm[o_ctr + 1], steps + up);
  }
}

// CAP, one thread per schedule
__device__ __noinline__ void eval_moves_cap(const SInst& I, int o_base, int o_evs,
                                            const uint32_t* __restrict__ moves,
                                            int* __restrict__ cmax_out, int n_feas,
                                            int warp_words, int lanes) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int* base = dsm + o_base;
  int* st = dsm + o_evs + warp * warp_words;
  if (lane >= lanes) return;
  for (int idx = warp * lanes + lane; idx < n_feas; idx += nw * lanes) {
    const uint32_t mv = moves[idx];
    const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
    const int au = base[v], av = base[u];
    cmax_out[idx] = sgs_cap_thread(
        I, st, lanes, lane, [&](int p) { return p == u ? au : (p == v ? av : base[p]); }, I.sptr,
        I.sdat, nullptr);
  }
}

// CAP, one thread per schedule, reusing the current schedule's prefix.  A
// warp takes L consecutive moves at once (lane l: move base + l); moves are
// dealt in increasing index order, so lane 0 has the smallest u of the batch,
// u_min, and the warp keeps one shared prefix state for positions < u_min
// (extended with the known starts `bst`, whole warp per resource row).  Every
// lane copies it into its own state and schedules positions u_min.. of its
// swapped order; positions u_min..u-1 are the current order's, booked at their
// known starts.
//   per-warp scratch: L lanes x (c [m*R] | cb [R] | es [n]) interleaved by lane
//                     | c_pre [m*rs] | cb_w [m*rs] | es_pre [n]
__device__ __noinline__ void eval_moves_cap_thread_inc(const SInst& I, int o_base, int o_bst,
                                                       int o_ctr, int o_evs,
                                                       const uint32_t* __restrict__ moves,
                                                       int* __restrict__ cmax_out, int n_feas,
                                                       int warp_words, int lanes,
                                                       uint32_t ctr_cl, int nw_total) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = I.n, m = I.m, R = I.rmax, rs = cap_row_stride(R), L = lanes;
  const int* base = dsm + o_base;
  const int* bst = dsm + o_bst;
  int* st = dsm + o_evs + warp * warp_words;
  int* cpre = st + L * cap_thread_words(n, m, R);
  int* esp = cpre + 2 * m * rs;
  const uint32_t a_cpre = sa(cpre), a_cbw = sa(cpre + m * rs), a_dem = sa(I.dem),
                 a_ctr = sa(dsm + o_ctr);
  const int capk = lane < m ? I.cap[lane] : 0;
  int* c = st + lane;                     // c[(k*R + i)*L]
  int* cb = st + (m * R) * L + lane;      // cb[i*L]
  int* es = cb + R * L;                   // es[a*L]
  for (int j = lane; j < m * rs; j += 32) cpre[j] = 0;
  for (int a = lane; a < n; a += 32) esp[a] = 0;
  __syncwarp();
  // batch size: all warps busy on small neighbourhoods (j30: ~90 moves)
  const int nw = nw_total;  // warps sharing the phase (the cluster's)
  const int bsz = min(L, max(1, (n_feas + nw - 1) / nw));
  int up = 0, cm_pre = 0, steps = 0;
  for (;;) {
    int b0 = 0;
    if (lane == 0)
      b0 = ctr_cl ? atom_add_cluster(ctr_cl, bsz) : atomicAdd(reinterpret_cast<int*>(dsm + o_ctr), bsz);
    b0 = __shfl_sync(FULL_MASK, b0, 0);
    if (b0 >= n_feas) break;
    const int idx = b0 + lane;
    const bool active = lane < bsz && idx < n_feas;
    const uint32_t mv = moves[active ? idx : b0];
    const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
    const int u0 = __shfl_sync(FULL_MASK, u, 0);
    // ---- extend the shared prefix to positions < u0 (known starts)
    for (; up < u0; ++up) {
      const int act = base[up];
      const int dur = I.dur[act], s0 = bst[act];
      if (dur > 0) {
        const int req = lane < m ? static_cast<int>(lds32(a_dem + 4 * (act * m + lane))) : 0;
        cap_commit_all(a_cpre, a_cbw, rs, m, capk, req, s0, dur);
      }
      const int fin = s0 + dur;
      cm_pre = max(cm_pre, fin);
      for (int e = I.sptr[act] + lane; e < I.sptr[act + 1]; e += 32) atomicMax(&esp[I.sdat[e]], fin);
      __syncwarp();
    }
    if (active) {
      for (int k = 0; k < m; ++k)
        for (int i = 0; i < R; ++i) c[(k * R + i) * L] = cpre[k * rs + i];
      for (int a = 0; a < n; ++a) es[a * L] = esp[a];
      const int au = base[v], av = base[u];
      int cm = cm_pre;
      for (int p = u0; p < n; ++p) {
        const int act = p == u ? au : (p == v ? av : base[p]);
        const int dur = I.dur[act];
        const int* dem = I.dem + act * m;
        const int start = p < u ? bst[act] : max(es[act * L], cap_es(c, L, dem, I.cap, m, R));
        cap_commit(c, cb, L, dem, I.cap, m, R, start, dur);
        const int fin = start + dur;
        cm = max(cm, fin);
        for (int e = I.sptr[act]; e < I.sptr[act + 1]; ++e) {
          const int sc = I.sdat[e];
          if (es[sc * L] < fin) es[sc * L] = fin;
        }
      }
      cmax_out[idx] = cm;
      steps += n - u0;
    }
    __syncwarp();
  }
  steps = __reduce_add_sync(FULL_MASK, steps);
  if (lane == 0) {
    if (ctr_cl)
      atom_add_cluster(ctr_cl + 4, steps + up);
    else
      atomicAdd(&dsm[o_ctr + 1], steps + up);
  }
}

// Leader side of a cluster neighbourhood phase (no-ops without a cluster):
// publish the phase and meet the followers at B1; B2 once every move is done.
__device__ __forceinline__ void cluster_phase_begin(CtaCtx& c, int n_feas) {
  if (c.csize <= 1) return;
  if (threadIdx.x == 0) {
    c.scal[SC_NF] = n_feas;
    c.scal[SC_CMD] = CMD_EVAL;
  }
  __syncthreads();
  cluster_sync_all();  // B1: followers read the leader's state
}
__device__ __forceinline__ void cluster_phase_end(const CtaCtx& c) {
  if (c.csize <= 1) return;
  __syncthreads();
  cluster_sync_all();  // B2: every move of the phase is evaluated
}
// the move counter the phase deals from: the leader's, as a cluster address
__device__ __forceinline__ uint32_t cluster_counter(const CtaCtx& c) {
  return c.csize > 1 ? cluster_map(sa(c.scal + SC_CTR), 0) : 0u;
}

// the prefix-reusing TIME evaluator on this CTA's copy of the current order
template <int W>
__device__ __forceinline__ void eval_moves_time32_dispatch(const CtaCtx& c, int n_feas,
                                                           int base_cmax, uint32_t ctr_cl) {
  if (c.I.big)
    eval_moves_time32_inc<W, true>(soff(c.I.info_r), soff(c.I.pdat), soff(c.I.req),
                                   soff(c.base), soff(c.bst), soff(c.scal + SC_CTR), soff(c.evs),
                                   c.I.capw[0], W == 2 ? c.I.capw[1] : 0u, c.I.hi, c.I.n, c.I.H,
                                   c.moves_buf, c.cmax_buf, n_feas, c.warp_words, base_cmax,
                                   c.err, ctr_cl);
  else
    eval_moves_time32_inc<W, false>(soff(c.I.info_r), soff(c.I.pdat), soff(c.I.req),
                                    soff(c.base), soff(c.bst), soff(c.scal + SC_CTR),
                                    soff(c.evs), c.I.capw[0], W == 2 ? c.I.capw[1] : 0u, c.I.hi,
                                    c.I.n, c.I.H, c.moves_buf, c.cmax_buf, n_feas, c.warp_words,
                                    base_cmax, c.err, ctr_cl);
}

// Cluster follower (rank > 0): evaluates moves of the leader's neighbourhood
// phases until the leader is done.  Per phase: B1 (leader published the
// phase), copy the current order and its starts from the leader's shared
// memory, deal moves from the leader's counter, write makespans into the
// leader's global buffer, B2.  The instance follows the leader's (steals).
template <int MODE, int G, int W>
//   blob/blob_off: the launch's instances (blob_off null: one instance)
__device__ void cta_follow(CtaCtx& c, const int* blob, const int64_t* blob_off, int iid, int* smem,
                           int plan_inst, int csize) {
  const int tid = threadIdx.x;
  const uint32_t l_scal = cluster_map(sa(c.scal), 0);
  const uint32_t l_base = cluster_map(sa(c.base), 0), l_bst = cluster_map(sa(c.bst), 0);
  for (;;) {
    cluster_sync_all();  // B1
    const int cmd = static_cast<int>(ld_cluster(l_scal + 4 * SC_CMD));
    if (cmd == CMD_DONE) break;
    const int liid = static_cast<int>(ld_cluster(l_scal + 4 * SC_IID));
    if (blob_off != nullptr && liid != iid) {
      iid = liid;
      stage_instance(blob + blob_off[iid], smem + plan_inst, c.I);
    }
    const int n_feas = static_cast<int>(ld_cluster(l_scal + 4 * SC_NF));
    const int base_cmax = static_cast<int>(ld_cluster(l_scal + 4 * SC_BASEC));
    for (int p = tid; p < c.I.n; p += blockDim.x) {
      c.base[p] = static_cast<int>(ld_cluster(l_base + 4 * p));
      c.bst[p] = static_cast<int>(ld_cluster(l_bst + 4 * p));
    }
    __syncthreads();
    const uint32_t ctr = l_scal + 4 * SC_CTR;
    if constexpr (MODE == MODE_TIME) {
      eval_moves_time32_dispatch<W>(c, n_feas, base_cmax, ctr);
    } else if constexpr (G == 32) {
      eval_moves_cap_warp(soff(c.I.info_f), soff(c.I.sdat), soff(c.I.dem), soff(c.I.cap),
                          soff(c.base), soff(c.bst), soff(c.scal + SC_CTR), soff(c.evs), c.I.n,
                          c.I.m, cap_row_stride(c.I.rmax), c.moves_buf, c.cmax_buf, n_feas,
                          c.warp_words, true, ctr);
    } else {
      eval_moves_cap_thread_inc(c.I, soff(c.base), soff(c.bst), soff(c.scal + SC_CTR),
                                soff(c.evs), c.moves_buf, c.cmax_buf, n_feas, c.warp_words,
                                c.cap_lanes, ctr, static_cast<int>(blockDim.x >> 5) * csize);
    }
    (void)base_cmax;
    __syncthreads();
    cluster_sync_all();  // B2
  }
  cluster_sync_all();  // the leader's shared memory stays valid until every follower is out
}

// every compacted move -> cmax_buf (full SGS of the swapped order)
template <int MODE, int G, int W>
__device__ __forceinline__ void cta_eval_moves(CtaCtx& c, int n_feas) {
  if constexpr (MODE == MODE_TIME) {
    if constexpr (G == 32) {
      if (c.inc) {
        // the current order's schedule (starts -> bst), then prefix-reusing moves
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (warp == 0) {
          const bool keep = c.scal[SC_BSTOK] != 0;  // picked move had converged
          if (!keep) {
            uint32_t* tau = reinterpret_cast<uint32_t*>(c.evs);
            int* es = c.evs + (c.I.H + 1) * W;
            const int cm = sgs_time_warp<W>(sa(c.I.info_f), sa(c.I.sdat), sa(c.I.req),
                                            c.I.capw[0], W == 2 ? c.I.capw[1] : 0u, c.I.hi,
                                            c.I.n, c.I.H, sa(tau), sa(es), sa(c.base), c.bst,
                                            c.err);
            if (lane == 0) c.scal[SC_BASEC] = cm;
          }
          if (lane == 0) {
            c.scal[SC_CTR] = 0;
            c.scal[SC_STEPS] = keep ? 0 : c.I.n;  // the current order's schedule
          }
        }
        __syncthreads();
        cluster_phase_begin(c, n_feas);
        eval_moves_time32_dispatch<W>(c, n_feas, c.scal[SC_BASEC], cluster_counter(c));
        cluster_phase_end(c);
      } else {
        eval_moves_time32<W>(soff(c.I.info_f), soff(c.I.sdat), soff(c.I.req), soff(c.base),
                             soff(c.evs), c.I.capw[0], W == 2 ? c.I.capw[1] : 0u, c.I.hi, c.I.n,
                             c.I.H, c.moves_buf, c.cmax_buf, n_feas, c.warp_words, c.err);
      }
    } else {
      eval_moves_split<G, W>(soff(c.I.info_f), soff(c.I.sdat), soff(c.I.req), soff(c.base),
                             soff(c.evs), c.I.capw[0], W == 2 ? c.I.capw[1] : 0u, c.I.hi, c.I.n,
                             c.I.H, c.moves_buf, c.cmax_buf, n_feas, c.warp_words, c.err);
    }
  } else if constexpr (G == 32) {
    // the current order's schedule (starts -> bst), then one warp per move
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
      if (c.inc)
        sgs_cap_warp(sa(c.I.info_f), sa(c.I.sdat), sa(c.I.dem), c.I.cap, c.I.n, c.I.m,
                     cap_row_stride(c.I.rmax), sa(c.evs), sa(c.base), c.bst);
      if (lane == 0) {
        c.scal[SC_CTR] = 0;
        c.scal[SC_STEPS] = c.inc ? c.I.n : 0;
      }
    }
    __syncthreads();
    cluster_phase_begin(c, n_feas);
    eval_moves_cap_warp(soff(c.I.info_f), soff(c.I.sdat), soff(c.I.dem), soff(c.I.cap),
                        soff(c.base), soff(c.bst), soff(c.scal + SC_CTR), soff(c.evs), c.I.n,
                        c.I.m, cap_row_stride(c.I.rmax), c.moves_buf, c.cmax_buf, n_feas,
                        c.warp_words, c.inc, cluster_counter(c));
    cluster_phase_end(c);
  } else {
    // prefix reuse pays from j60 on; on j30-size projects the per-batch state
    // copy and the current-schedule pass outweigh the shorter suffixes
    // (131.9 M vs 163 M schedules/s on j30, 147.4 M vs 123 M on j60)
    if (c.inc && c.I.n >= 48) {
      // the current order's schedule (starts -> bst) on warp 0's prefix scratch
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      if (warp == 0) {
        int* scr = c.evs + c.cap_lanes * cap_thread_words(c.I.n, c.I.m, c.I.rmax);
        sgs_cap_warp(sa(c.I.info_f), sa(c.I.sdat), sa(c.I.dem), c.I.cap, c.I.n, c.I.m,
                     cap_row_stride(c.I.rmax), sa(scr), sa(c.base), c.bst);
        if (lane == 0) {
          c.scal[SC_CTR] = 0;
          c.scal[SC_STEPS] = c.I.n;
        }
      }
      __syncthreads();
      cluster_phase_begin(c, n_feas);
      eval_moves_cap_thread_inc(c.I, soff(c.base), soff(c.bst), soff(c.scal + SC_CTR),
                                soff(c.evs), c.moves_buf, c.cmax_buf, n_feas, c.warp_words,
                                c.cap_lanes, cluster_counter(c),
                                static_cast<int>(blockDim.x >> 5) * c.csize);
      cluster_phase_end(c);
    } else {
      eval_moves_cap(c.I, soff(c.base), soff(c.evs), c.moves_buf, c.cmax_buf, n_feas,
                     c.warp_words, c.cap_lanes);
    }
  }
  __syncthreads();
}

// makespan of one order held in shared memory (evaluate_current, search.py:134)
template <int MODE, int G, int W>
__device__ __forceinline__ int cta_eval_one(CtaCtx& c, const int* ord) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    int cm;
    if constexpr (MODE == MODE_TIME) {
      uint32_t* tau = reinterpret_cast<uint32_t*>(c.evs);
      int* es = reinterpret_cast<int*>(tau) + (c.I.H + 1) * W;
      cm = sgs_time_warp<W>(sa(c.I.info_f), sa(c.I.sdat), sa(c.I.req), c.I.capw[0],
                            W == 2 ? c.I.capw[1] : 0u, c.I.hi, c.I.n, c.I.H, sa(tau), sa(es),
                            sa(ord), nullptr, c.err);
    } else if constexpr (G == 32) {
      cm = sgs_cap_warp(sa(c.I.info_f), sa(c.I.sdat), sa(c.I.dem), c.I.cap, c.I.n, c.I.m,
                        cap_row_stride(c.I.rmax), sa(c.evs), sa(ord), nullptr);
    } else {
      cm = 0;
      if (lane == 0)
        cm = sgs_cap_thread(c.I, c.evs, c.cap_lanes, 0, [&](int p) { return ord[p]; }, c.I.sptr,
                            c.I.sdat, nullptr);
    }
    if (lane == 0) c.scal[SC_START] = cm;
  }
  __syncthreads();
  return c.scal[SC_START];
}

// ---------------------------------------------------------------- the chunk

struct ChunkOut {
  int iters, improved, local_best, cur, forced;
  long long evals;
  long long steps;  // SGS activity steps spent on the neighbourhoods
};

// kernels.py:316-385.  c.base holds the order (mutated in place), the tabu
// list/counters/head are in shared memory.  trace may be null.
template <int MODE, int G, int W>
__device__ ChunkOut run_chunk_cta(CtaCtx& c, int budget, int adopted_cmax, int start_cmax,
                                  int best_known_cmax, int floor_cmax, int* trace) {
  const int tid = threadIdx.x, n = c.I.n;
  int local_best = start_cmax, cur = start_cmax, iters = 0, forced = 0;
  long long evals = 0, steps = 0;
  if (tid == 0) c.scal[SC_BSTOK] = 0;  // a new order: no current-schedule starts yet
  for (int it = 0; it < budget; ++it) {
    const int n_feas = cta_filter(c);
    ++iters;
    if (n_feas == 0) {
      if (tid == 0 && trace) trace[iters - 1] = cur;
      break;
    }
    cta_eval_moves<MODE, G, W>(c, n_feas);
    evals += n_feas;
    const bool counted =
        MODE == MODE_CAPACITY ? (G == 32 || (c.inc && n >= 48)) : (G == 32 && c.inc);
    steps += counted ? c.scal[SC_STEPS] : static_cast<long long>(n_feas) * n;
    const int asp = best_known_cmax < local_best ? best_known_cmax : local_best;
    unsigned ka = 0xffffffffu, kl = 0xffffffffu;
    for (int idx = tid; idx < n_feas; idx += blockDim.x) {
      const unsigned cm = static_cast<unsigned>(c.cmax_buf[idx]) & 0xffffu;
      const unsigned key = (cm << 16) | static_cast<unsigned>(idx);
      kl = min(kl, key);
      const uint32_t mv = c.moves_buf[idx];
      const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
      if (tabu_get(c, u, v) == 0 || static_cast<int>(cm) < asp) ka = min(ka, key);
    }
    ka = block_min_u32(ka, c.red);
    kl = block_min_u32(kl, c.red);
    const bool forced_pick = ka == 0xffffffffu;
    const unsigned key = forced_pick ? kl : ka;
    forced += forced_pick ? 1 : 0;
    const int pick = static_cast<int>(key & 0xffff);
    cur = static_cast<int>(key >> 16);
    if (tid == 0) {
      const uint32_t mv = c.moves_buf[pick];
      const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
      const int t = c.base[u];
      c.base[u] = c.base[v];
      c.base[v] = t;
      c.scal[SC_HEAD] = tabu_add1(c, c.scal[SC_HEAD], u, v);
      if (trace) trace[iters - 1] = cur;
      c.scal[SC_BSTOK] = (c.cmax_buf[pick] & CONV_FLAG) ? 1 : 0;
      c.scal[SC_FLAG] = budget_spent(c.budget_ns, c.t0_ns) ? 1 : 0;
    }
    __syncthreads();
    if (cur < local_best) {
      local_best = cur;
      for (int p = tid; p < n; p += blockDim.x) c.best[p] = c.base[p];
    }
    if (local_best < adopted_cmax) break;
    if (local_best <= floor_cmax) break;
    if (c.scal[SC_FLAG]) break;  // wall-clock budget spent (only with a budget)
  }
  __syncthreads();
  ChunkOut o;
  o.iters = iters;
  o.evals = evals;
  o.steps = steps;
  o.improved = local_best < adopted_cmax ? 1 : 0;
  o.local_best = local_best;
  o.cur = cur;
  o.forced = forced;
  return o;
}

// ------------------------------------------------------------- diversify

// search.py:77-94: phi_steps uniform feasible swaps over ALL pairs (delta = N),
// skipped without an RNG draw when nothing is feasible.  rng is thread 0's.
__device__ void cta_diversify(CtaCtx& c, int* work, int steps, Pcg64& rng) {
  const int n = c.I.n;
  for (int s = 0; s < steps; ++s) {
    cta_bounds(c, work);
    for (int u = 1 + threadIdx.x; u <= n - 3; u += blockDim.x) {
      const int lim = c.msp[work[u]];
      int cnt = 0;
      for (int v = u + 1; v <= n - 2 && v < lim; ++v) cnt += (u > c.mpp[work[v]]) ? 1 : 0;
      c.rowc[u] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int total = 0;
      for (int u = 1; u <= n - 3; ++u) total += c.rowc[u];
      if (total > 0) {
        int k = static_cast<int>(rng.integers(static_cast<uint32_t>(total)));
        int u = 1;
        while (k >= c.rowc[u]) {
          k -= c.rowc[u];
          ++u;
        }
        int v = u + 1;
        for (;; ++v) {
          if (u > c.mpp[work[v]]) {
            if (k == 0) break;
            --k;
          }
        }
        const int t = work[u];
        work[u] = work[v];
        work[v] = t;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------ shared-memory plan

struct SmemPlan {
  int inst, base, pos, msp, mpp, rs, best, rowc, bst, tabu_list, tabu_cnt, red, scal, evs;
  int warp_words, total, cap_lanes;
};

__host__ __device__ inline int eval_warp_words(int mode, int G, int W, int n, int m, int H,
                                               int rmax, int cap_lanes) {
  if (mode == MODE_TIME) return G == 32 ? (H + 1) * W + 4 * n + 3 : (32 / G) * ((H + 1) * W + 2 * n);
  if (G == 32) return cap_warp_words(n, m, rmax) + m * cap_row_stride(rmax) + n;
  return cap_lanes * cap_thread_words(n, m, rmax) + cap_warp_words(n, m, rmax);
}

__host__ __device__ inline SmemPlan plan_smem(int mode, int G, int W, int n, int m, int H, int e,
                                              int rmax, int delta, int T, int nwarps,
                                              int cap_lanes = 32) {
  SmemPlan p;
  auto a4 = [](int x) { return (x + 3) & ~3; };
  int off = 0;
  p.inst = off; off += a4(inst_smem_words(n, m, e, W));
  p.base = off; off += a4(n);
  p.pos = off; off += a4(n);
  p.msp = off; off += a4(n);
  p.mpp = off; off += a4(n);
  p.rs = off; off += a4(n);
  p.best = off; off += a4(n);
  p.rowc = off; off += a4(n);
  p.bst = off; off += a4(n);
  p.tabu_list = off; off += a4(T > 0 ? T : 1);
  p.tabu_cnt = off; off += a4((n * (delta + 1) + 1) / 2);
  p.red = off; off += 72;
  p.scal = off; off += SC_WORDS;
  p.cap_lanes = cap_lanes;
  p.warp_words = a4(eval_warp_words(mode, G, W, n, m, H, rmax, cap_lanes));
  p.evs = off; off += p.warp_words * nwarps;
  p.total = off;
  return p;
}

__device__ __forceinline__ void cta_setup(CtaCtx& c, const int* blob, int* smem, const SmemPlan& p,
                                          int delta, int T, uint32_t* moves_buf, int* cmax_buf,
                                          int* err) {
  stage_instance(blob, smem + p.inst, c.I);
  c.delta = delta;
  c.T = T;
  c.base = smem + p.base;
  c.pos = smem + p.pos;
  c.msp = smem + p.msp;
  c.mpp = smem + p.mpp;
  c.rs = smem + p.rs;
  c.best = smem + p.best;
  c.rowc = smem + p.rowc;
  c.bst = smem + p.bst;
  c.inc = true;
  c.csize = 1;
  c.budget_ns = 0;
  c.t0_ns = nullptr;
  c.tabu_list = reinterpret_cast<uint32_t*>(smem + p.tabu_list);
  c.tabu_cnt = reinterpret_cast<uint32_t*>(smem + p.tabu_cnt);
  c.red = smem + p.red;
  c.scal = smem + p.scal;
  c.evs = smem + p.evs;
  c.warp_words = p.warp_words;
  c.cap_lanes = p.cap_lanes;
  c.moves_buf = moves_buf;
  c.cmax_buf = cmax_buf;
  c.err = err;
  __syncthreads();
  cta_init_rows(c);
}

}  // namespace rt
