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
//   apply    swap + tabu_add on the shared-memory circular list with a banded
//            membership bitmap (kernels.py:263-277)
#pragma once
#include "common.cuh"
#include "pcg64.cuh"
#include "cta.cuh"
#include "eval_moves.cuh"

namespace rt {
// ---------------------------------------------------------------- the chunk

struct ChunkOut {
  int iters, improved, local_best, cur, forced;
  long long evals;
  long long steps;  // SGS activity steps spent on the neighbourhoods
};

// kernels.py:316-385.  c.base holds the order (mutated in place), the tabu
// list/counters/head are in shared memory.  trace may be null.
template <int MODE, int G, int W, bool LONG = false>
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
    cta_eval_moves<MODE, G, W, LONG>(c, n_feas);
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
    if (tid < 32) {  // warp 0: apply the move, tabu_add (kernels.py:263-277)
      const uint32_t mv = c.moves_buf[pick];
      const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
      const int head = tabu_add_warp(c, c.scal[SC_HEAD], u, v);
      if (tid == 0) {
        const int t = c.base[u];
        c.base[u] = c.base[v];
        c.base[v] = t;
        c.scal[SC_HEAD] = head;
        if (trace) trace[iters - 1] = cur;
        c.scal[SC_BSTOK] = (c.cmax_buf[pick] & CONV_FLAG) ? 1 : 0;
        c.scal[SC_FLAG] = budget_spent(c.budget_ns, c.t0_ns) ? 1 : 0;
      }
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
  int snap, snap_words;  // CAPACITY group 32: state snapshots (uint16), -1 / 0 = none
  int slots;             // TIME group 32: profile slots per warp
  int fb;                // TIME group 32 with sized profiles: full-horizon region, -1 = none
};

// shared-memory budget of the CAPACITY evaluator's state snapshots: an
// instance whose n*S uint16 exceed it keeps every k-th position's state
// (j120-shape projects: k = 1; 300 activities with capacities ~80: k = 3)
constexpr int SNAP_MAX_BYTES = 40 * 1024;

// big: some instance of the launch has a duration or fan-out above 32 -- only
// then does the prefix-reusing TIME evaluator keep an undo log (2n words)
__host__ __device__ inline int eval_warp_words(int mode, int G, int W, int n, int m, int H,
                                               int rmax, int cap_lanes, int big = 1,
                                               bool snap = false, int slots = 0) {
  if (mode == MODE_TIME)
    return G == 32 ? (slots > 0 ? slots : H + 1 + TAU_PAD) * W + (big ? 4 : 2) * n + 3
                   : (32 / G) * ((H + 1) * W + 2 * n);
  if (G == 32) return m * cap_row_stride(rmax) + n;  // c | fin (snapshots: CTA-wide)
  return max(cap_lanes * cap_thread_words(n, m, rmax) + cap_prefix_words(n, m, rmax),
             cap_warp_words(n, m, rmax));
}

// slots > 0 (TIME group 32, no duration above 32): per-warp profiles of
// that many slots plus one full-horizon region per CTA (see
// eval_moves_time32_inc, SIZED)
__host__ __device__ inline SmemPlan plan_smem(int mode, int G, int W, int n, int m, int H, int e,
                                              int rmax, int delta, int T, int nwarps,
                                              int cap_lanes = 32, int big = 1, int sumcap = 0,
                                              int slots = 0) {
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
  p.tabu_cnt = off; off += a4((n * (delta + 1) + 31) / 32);  // membership bits
  p.red = off; off += 72;
  p.scal = off; off += SC_WORDS;
  p.cap_lanes = cap_lanes;
  const bool snap = mode == MODE_CAPACITY && G == 32;
  p.snap = -1;
  p.snap_words = 0;
  if (snap) {
    long long need = (static_cast<long long>(n) * (sumcap > 0 ? sumcap : m * rmax) + 1) / 2;
    if (need > SNAP_MAX_BYTES / 4) need = SNAP_MAX_BYTES / 4;
    p.snap = off;
    p.snap_words = a4(static_cast<int>(need));
    off += p.snap_words;
  }
  const bool sized = mode == MODE_TIME && G == 32 && slots > 0 && slots < H + 1 + TAU_PAD;
  p.slots = mode == MODE_TIME && G == 32 ? (sized ? slots : H + 1 + TAU_PAD) : 0;
  p.fb = -1;
  if (sized) {  // whole schedules: profile (H+1)*W | es [n] | ord [n]
    p.fb = off;
    off += a4((H + 1) * W + 2 * n);
  }
  p.warp_words = a4(eval_warp_words(mode, G, W, n, m, H, rmax, cap_lanes, big, snap,
                                    sized ? slots : 0));
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
  c.snap = p.snap >= 0 ? smem + p.snap : nullptr;
  c.snap_words = p.snap_words;
  c.snap_k = 1;
  c.snap_S = 0;
  c.fb = p.fb >= 0 ? smem + p.fb : nullptr;
  c.slots = p.slots;
  c.warp_words = p.warp_words;
  c.cap_lanes = p.cap_lanes;
  c.moves_buf = moves_buf;
  c.cmax_buf = cmax_buf;
  c.err = err;
  if (threadIdx.x == 0) c.scal[SC_FBLOCK] = 0;
  __syncthreads();
  if (c.snap) cta_snap_stride(c);
  cta_init_rows(c);
}

}  // namespace rt
