// eval_moves.cuh -- evaluation of every compacted move of an iteration
// (kernels.py:350-362): the prefix-reusing TIME and CAPACITY evaluators, the
// full-SGS alternatives, and the cluster leader/follower protocol that
// spreads a phase over several CTAs.
#pragma once
#include "cta.cuh"

namespace rt {
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
//   per-warp scratch: tau (H+1+TAU_PAD)*W | fin [n] | log [2n] (BIG only) |
//   ord [n + 1] (ord[n]: a valid pad the unrolled loop's prefetch may read)
// The undo gives back the suffix bookings below hw_pre (a zero demand gives
// back nothing): with durations <= 32 every suffix step's booking is found
// from ord, the records and fin, 32 at once; with longer ones (BIG) a log
// lists them -- (start | dur << 16, packed demand (W = 1) or activity
// (W = 2)) -- and the warp gives them back one by one.
//   ctr_cl: != 0 -> the move counter (and the step counter after it) live in
//   the cluster leader's shared memory at this shared::cluster address
//   SIZED: the profile holds P slots (< H + 1 + TAU_PAD, sized by a makespan
//   bound; no duration above 32): a move whose schedule would book past
//   P - 64 is abandoned (time_step_pull sets ovf), the profile is rebuilt from
//   the prefix, and the move is evaluated exactly by the full-horizon SGS on
//   the CTA's fallback region o_fb (one warp at a time, lock at o_fblock);
//   o_info_f / o_push: the push records and successor lists it needs.
//   LONG: phase B tests its loop once per eight positions instead of four --
//   used by the large-project search kernel only (k_solve at
//   TIME_THREADS_LARGE; A/B on B200: +1.6 % j120p, +1.4 % Gen-R j120; in
//   every kernel it cost j60p 1.8 %, profiles/r2/ab_phaseb8.txt)
template <int W, bool BIG, bool SIZED, bool LONG = false>
__device__ __noinline__ void eval_moves_time32_inc(int o_info, int o_pull, int o_req, int o_base,
                                                   int o_bst, int o_ctr, int o_evs, uint32_t cap0,
                                                   uint32_t cap1, uint32_t hi, int n, int H,
                                                   const uint32_t* __restrict__ moves,
                                                   int* __restrict__ cmax_out, int n_feas,
                                                   int warp_words, int base_cmax, int* err,
                                                   uint32_t ctr_cl, int P, int o_fb, int o_fblock,
                                                   int o_info_f, int o_push) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* ws = dsm + o_evs + warp * warp_words;
  // o_info: pull records (info_r: duration, demand, predecessor span, mask);
  // o_pull: predecessor lists (pdat)
  const uint32_t a_info = sa(dsm + o_info), a_pdat = sa(dsm + o_pull), a_req = sa(dsm + o_req),
                 a_base = sa(dsm + o_base), a_bst = sa(dsm + o_bst), a_ctr = sa(dsm + o_ctr),
                 a_tau = sa(ws), a_fin = sa(ws + P * W),
                 a_log = (a_fin + 4 * n + 7) & ~7u, a_ord = a_log + (BIG ? 8 * n : 0);
  // the lane's base addresses of the profile and the predecessor lists
  const uint32_t a_tau_l = opaque(a_tau + 4 * W * lane), a_pdat_l = opaque(a_pdat + 4 * lane);
  if (lane == 0) sts32(a_ord + 4 * n, 0u);
  // the profile is kept materialised: every slot from the high-water mark on
  // (and the 32-slot pad past the horizon the scan may read) holds the capacity
  // (capacity with every packed lane's guard bit set, see window_fits_ballot)
  const uint32_t capg0 = cap0 | hi, capg1 = cap1 | hi;
  auto materialise = [&]() {
    for (int t = lane; t < P; t += 32) {
      sts32(a_tau + 4 * W * t, capg0);
      if (W == 2) sts32(a_tau + 4 * W * t + 4, capg1);
    }
  };
  materialise();
  __syncwarp();
  int up = 0, hw_pre = 0, cm_pre = 0, steps = 0;
  // the last position holds the sink (every activity precedes it, and moves
  // never reach it): with zero duration it starts at max(es) <= cm, so it
  // cannot change the makespan and is not scheduled
  const int pend = lds128(a_info + 16 * static_cast<int>(lds32(a_base + 4 * (n - 1)))).x == 0
                       ? n - 1 : n;
  // SIZED: the exact makespan of the swapped order by the full-horizon SGS
  // on the CTA's fallback region (one warp at a time)
  auto full_eval = [&](int u, int v) -> int {
    const uint32_t a_fb = sa(dsm + o_fb), a_fbes = a_fb + 4 * (H + 1) * W, a_fbord = a_fbes + 4 * n;
    // (acquire: the fence orders the previous holder's accesses, released by
    // its fence + exchange below, before this warp's; compute-sanitizer
    // racecheck does not model such a lock and reports the region's reuse by
    // the next warp as a race -- profiles/r2/sanitizer3/README.md)
    if (lane == 0) {
      while (atomicCAS(&dsm[o_fblock], 0, 1) != 0) __nanosleep(32);
      __threadfence_block();
    }
    __syncwarp();
    for (int q = lane; q < n; q += 32)
      sts32(a_fbord + 4 * q, lds32(a_base + 4 * (q == u ? v : (q == v ? u : q))));
    __syncwarp();
    const int cmf = sgs_time_warp<W>(sa(dsm + o_info_f), sa(dsm + o_push), a_req, cap0, cap1, hi,
                                      n, H, a_fb, a_fbes, a_fbord, nullptr, err);
    __syncwarp();
    __threadfence_block();
    if (lane == 0) atomicExch(&dsm[o_fblock], 0);
    return cmf;
  };
  // SIZED: the current schedule itself books past the profile (rare): every
  // move of this phase is evaluated on the fallback region
  const bool all_full = SIZED && base_cmax + 64 > P;
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = ctr_cl ? atom_add_cluster(ctr_cl, 1) : atom_inc_shared(a_ctr);
    idx = __shfl_sync(FULL_MASK, idx, 0);
    if (idx >= n_feas) break;
    const uint32_t mv = moves[idx];
    const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
    if (SIZED && all_full) {
      const int cmf = full_eval(u, v);
      if (lane == 0) cmax_out[idx] = cmf;
      steps += n;
      continue;
    }
    // ---- extend the prefix to positions < u with the known starts
    for (; up < u; ++up) {
      const int act = static_cast<int>(lds32(a_base + 4 * up));
      const int4 rec = lds128(a_info + 16 * act);
      const int s = static_cast<int>(lds32(a_bst + 4 * act));
      const uint32_t r0 = static_cast<uint32_t>(rec.y);
      const uint32_t r1 = W == 2 ? lds32(a_req + 8 * act + 4) : 0u;
      if (rec.x > 0 && (r0 | r1) != 0) warp_commit_mat<W, BIG>(a_tau_l, hw_pre, s, rec.x, r0, r1);
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
    bool div = false, ovf = false;
    // BIG: log the bookings below hw_pre for the undo (entry: dur << 16 |
    // start, demand or activity; horizons are < 2^16, see KEY_LIMIT).  !BIG
    // logs nothing: the undo finds every suffix step's booking from the
    // order (ord[u..p)), the records and the finish times (fin).
    auto log_below = [&](int act, const int4& rec, int st) {
      if (BIG && st < hw_pre && rec.x > 0) {  // (a zero duration gives back nothing)
        if (lane == 0)
          sts64(a_log + 8 * nlog, (static_cast<uint32_t>(rec.x) << 16) | static_cast<uint32_t>(st),
                W == 1 ? static_cast<uint32_t>(rec.y) : static_cast<uint32_t>(act));
        ++nlog;
      }
    };
    // phase A, positions u..v: until a start differs from the current
    // schedule's (then phase B) or v is reached with none differing
    // (converged: the rest is the current schedule)
    // (unrolled by two like phase B, so the prefetched activity needs no
    // register copies; p + 1 <= v + 1 < n)
    int act = static_cast<int>(lds32(a_ord + 4 * u));
    int4 rec = lds128(a_info + 16 * act);
    {
      int act_a = act;
      int4 rec_a = rec;
      for (;;) {
        const int act_b = static_cast<int>(lds32(a_ord + 4 * (p + 1)));
        const int4 rec_b = lds128(a_info + 16 * act_b);
        int st = time_step_pull<W, BIG, false, true, SIZED>(act_a, rec_a, a_pdat_l, a_req, cap0, cap1,
                                                     hi, H, a_tau_l, a_fin, hw, cm, err, P, &ovf);
        log_below(act_a, rec_a, st);
        div = st != static_cast<int>(lds32(a_bst + 4 * act_a));
        ++p;
        if (div || p > v) {
          act = act_b;
          rec = rec_b;
          break;
        }
        __syncwarp();  // after the loop test: the next REDUX follows it branch-free
        act_a = static_cast<int>(lds32(a_ord + 4 * (p + 1)));
        rec_a = lds128(a_info + 16 * act_a);
        st = time_step_pull<W, BIG, false, true, SIZED>(act_b, rec_b, a_pdat_l, a_req, cap0, cap1, hi, H,
                                                 a_tau_l, a_fin, hw, cm, err, P, &ovf);
        log_below(act_b, rec_b, st);
        div = st != static_cast<int>(lds32(a_bst + 4 * act_b));
        ++p;
        if (div || p > v) {
          act = act_a;
          rec = rec_a;
          break;
        }
        __syncwarp();
      }
    }
    __syncwarp();
    // phase B, positions p..pend-1 after a divergence; unrolled by two so the
    // prefetched next activity needs no register copies
    if (div && p < pend) {
      int act_a = act;
      int4 rec_a = rec;
      // two steps (positions p, p + 1), the next activity prefetched
      auto pair = [&]() {
        const int act_b = static_cast<int>(lds32(a_ord + 4 * (p + 1)));
        const int4 rec_b = lds128(a_info + 16 * act_b);
        int st = time_step_pull<W, BIG, false, true, SIZED>(act_a, rec_a, a_pdat_l, a_req, cap0, cap1,
                                                     hi, H, a_tau_l, a_fin, hw, cm, err, P, &ovf);
        log_below(act_a, rec_a, st);
        __syncwarp();
        act_a = static_cast<int>(lds32(a_ord + 4 * (p + 2)));  // ord[n]: pad
        rec_a = lds128(a_info + 16 * act_a);
        st = time_step_pull<W, BIG, false, true, SIZED>(act_b, rec_b, a_pdat_l, a_req, cap0, cap1, hi, H,
                                                 a_tau_l, a_fin, hw, cm, err, P, &ovf);
        log_below(act_b, rec_b, st);
        __syncwarp();
        p += 2;
      };
      // one loop test per four positions (branches cost more than their
      // instructions here), then a pair and a single step for the rest
      if constexpr (LONG) {  // one test per eight positions on long suffixes
        while (p + 7 < pend && !(SIZED && ovf)) {
          pair();
          pair();
          pair();
          pair();
        }
        if (p + 3 < pend && !(SIZED && ovf)) {
          pair();
          pair();
        }
      } else {
        while (p + 3 < pend && !(SIZED && ovf)) {
          pair();
          pair();
        }
      }
      if (p + 1 < pend && !(SIZED && ovf)) pair();
      if (p < pend && !(SIZED && ovf)) {
        const int st = time_step_pull<W, BIG, false, true, SIZED>(
            act_a, rec_a, a_pdat_l, a_req, cap0, cap1, hi, H, a_tau_l, a_fin, hw, cm, err, P, &ovf);
        log_below(act_a, rec_a, st);
        ++p;
      }
    }
    if (SIZED && ovf) {
      // abandoned: rebuild the profile from the prefix (whatever the suffix
      // booked is gone with it), then the exact evaluation on the fallback
      __syncwarp();
      materialise();
      __syncwarp();
      hw_pre = 0;
      for (int q = 0; q < up; ++q) {
        const int act = static_cast<int>(lds32(a_base + 4 * q));
        const int4 rec = lds128(a_info + 16 * act);
        const uint32_t r0 = static_cast<uint32_t>(rec.y);
        const uint32_t r1 = W == 2 ? lds32(a_req + 8 * act + 4) : 0u;
        warp_commit_mat<W, BIG>(a_tau_l, hw_pre, static_cast<int>(lds32(a_bst + 4 * act)), rec.x,
                                r0, r1);
        __syncwarp();
      }
      const int cmf = full_eval(u, v);
      if (lane == 0) cmax_out[idx] = cmf;
      steps += p - u + n;
      continue;
    }
    if (lane == 0) cmax_out[idx] = div ? cm : (base_cmax | CONV_FLAG);
    steps += p - u;  // converged: p = v + 1; else pend
    if (!BIG) nlog = p - u;
    // ---- undo the suffix's bookings below hw_pre
    __syncwarp();
    if (!BIG) {
      // one entry per lane (durations <= 32, a short serial loop each): the
      // demand goes back by shared-memory additions, as entries may overlap
      // in time -- no packed lane over- or underflows, since every partial
      // sum lies between the booked and the restored value
      // (position u + k's booking: start = fin - dur of its activity)
      for (int k0 = 0; k0 < nlog; k0 += 32) {
        const int k = k0 + lane;
        const int a = static_cast<int>(lds32(a_ord + 4 * (u + min(k, nlog - 1))));
        const int4 r = lds128(a_info + 16 * a);
        const int f = static_cast<int>(lds32(a_fin + 4 * a));
        uint32_t r0 = static_cast<uint32_t>(r.y), r1 = 0u;
        if (W == 2) r1 = lds32(a_req + 8 * a + 4);
        const int s = f - r.x;
        const int e = k < nlog ? min(f, hw_pre) : s;
        for (int t = s; t < e; ++t) {
          red_add_shared(a_tau + 4 * W * t, r0);
          if (W == 2) red_add_shared(a_tau + 4 * W * t + 4, r1);
        }
      }
    } else
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
    // ... and give [hw_pre, hw) back its capacity (!BIG: every step raises hw
    // to its finish time, so cm >= hw bounds the range and hw is not kept)
    for (int t = hw_pre + lane, e = BIG ? hw : cm; t < e; t += 32) {
      sts32(a_tau + 4 * W * t, capg0);
      if (W == 2) sts32(a_tau + 4 * W * t + 4, capg1);
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

// CAP, one warp per schedule, reusing the current order's schedule prefix
// like eval_moves_time32_inc.  Alg. 4 runs in closed form with the whole warp
// (sgs.cuh: cap_update_row); the state is compact (row k at the sum of the
// capacities before it, S words).  Precedence is pulled as in the TIME
// evaluator: es = max over the predecessors' finish times fin[] (the prefix
// activities hold the current schedule's, the suffix overwrites its own
// before a successor reads them).  The zero-duration sink is not scheduled
// (its start, max(es, Eq. 7), is bounded by the finish times already in the
// makespan).
//
// The current schedule's state after every k-th position (positions k-1,
// 2k-1, ...; k = 1 unless n*S exceeds the snapshot budget) is in shared
// memory (uint16 [n/k][S], written by the base pass, o_snap).  A move starts
// from the latest snapshot before u and replays the few positions up to u-1
// with their known starts.  If every activity at positions u..p (p >= v, a
// snapshot position) starts where it does in the current schedule AND the
// state after p equals the snapshot, the rest of the schedule is the current
// one: C_max = base_cmax (convergence exit).  Capacity-indexed states depend
// on the order of the updates, so the state is compared, not implied by the
// starts as in TIME -- and it may only agree a few positions after v, once
// the differing entries have been overwritten.
//   per-warp scratch: c [S] | fin [n]  (S <= m*rs)
//   o_info: pull records (info_r); o_pull: padded predecessor lists (pdat)
template <bool BIG>
__device__ __noinline__ void eval_moves_cap_warp(int o_info, int o_pull, int o_dem, int o_cap,
                                                 int o_base, int o_bst, int o_ctr, int o_evs,
                                                 int o_snap, int snap_k, int n, int m, int rs,
                                                 const uint32_t* __restrict__ moves,
                                                 int* __restrict__ cmax_out, int n_feas,
                                                 int warp_words, bool reuse, uint32_t ctr_cl,
                                                 bool packed, int base_cmax) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int capk = lane < m ? dsm[o_cap + lane] : 0;
  const int off = cap_row_offset(capk);
  const int S = __shfl_sync(FULL_MASK, off + capk, 31);
  const uint32_t a_scr = sa(dsm + o_evs + warp * warp_words);
  const uint32_t a_c = a_scr, a_fin = a_c + 4 * m * rs;
  const uint32_t a_info = sa(dsm + o_info), a_pdat = sa(dsm + o_pull), a_dem = sa(dsm + o_dem),
                 a_base = sa(dsm + o_base), a_bst = sa(dsm + o_bst), a_ctr = sa(dsm + o_ctr),
                 a_snap = sa(dsm + o_snap);
  const uint32_t a_pdat_l = opaque(a_pdat + 4 * lane);
  const int pend = lds128(a_info + 16 * static_cast<int>(lds32(a_base + 4 * (n - 1)))).x == 0
                       ? n - 1 : n;
  auto demand = [&](int act, const int4& rec) {  // lane k < m: resource k's demand
    if (lane >= m) return 0;
    return packed ? static_cast<int>((static_cast<uint32_t>(rec.y) >> (8 * lane)) & 0xffu)
                  : static_cast<int>(lds32(a_dem + 4 * (act * m + lane)));
  };
  int up = 0, cm_pre = 0, steps = 0;
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = ctr_cl ? atom_add_cluster(ctr_cl, 1) : atom_inc_shared(a_ctr);
    idx = __shfl_sync(FULL_MASK, idx, 0);
    if (idx >= n_feas) break;
    const uint32_t mv = moves[idx];
    const int u = static_cast<int>(mv >> 16), v = static_cast<int>(mv & 0xffff);
    const int u0 = reuse ? u : 0;
    // ---- positions < u0: the current schedule's finish times
    for (; up < u0; ++up) {
      const int act = static_cast<int>(lds32(a_base + 4 * up));
      const int fin = static_cast<int>(lds32(a_bst + 4 * act)) + lds128(a_info + 16 * act).x;
      cm_pre = max(cm_pre, fin);
      sts32_if(lane == 0, a_fin + 4 * act, static_cast<uint32_t>(fin));
    }
    // ---- the state after u0 - 1: the latest snapshot, then the positions
    // after it replayed with their known starts
    const int q = u0 / snap_k;  // snapshots 0..q-1 cover positions < q*k
    if (q > 0)
      for (int j = lane; j < S; j += 32) sts32(a_c + 4 * j, lds16(a_snap + 2 * ((q - 1) * S + j)));
    else
      for (int j = lane; j < S; j += 32) sts32(a_c + 4 * j, 0u);
    __syncwarp();
    for (int p = q * snap_k; p < u0; ++p) {
      const int act = static_cast<int>(lds32(a_base + 4 * p));
      const int4 rec = lds128(a_info + 16 * act);
      if (rec.x > 0)
        cap_update_all(a_c, off, m, capk, demand(act, rec),
                       static_cast<int>(lds32(a_bst + 4 * act)), rec.x);
    }
    steps += u0 - q * snap_k;
    // ---- positions u0.. of the swapped order
    int cm = cm_pre, p = u0;
    bool div = !reuse;
    for (; p < pend; ++p) {
      const int qq = p == u ? v : (p == v ? u : p);
      const int act = static_cast<int>(lds32(a_base + 4 * qq));
      const int4 rec = lds128(a_info + 16 * act);
      const int p0 = rec.z & 0xffff, pc = rec.z >> 16;
      int f = static_cast<int>(lds32(a_fin + 4 * lds32(a_pdat_l + 4 * p0)));
      f = lane < pc ? f : 0;
      if (BIG && pc > 32)
        for (int e = lane + 32; e < pc; e += 32)
          f = max(f, static_cast<int>(lds32(a_fin + 4 * lds32(a_pdat + 4 * (p0 + e)))));
      const int esv = __reduce_max_sync(FULL_MASK, f);
      int req;
      const int start = cap_start_warp(act, esv, a_dem, m, capk, off, a_c, req, packed,
                                       static_cast<uint32_t>(rec.y));
      if (rec.x > 0) cap_update_all(a_c, off, m, capk, req, start, rec.x);
      const int fin = start + rec.x;
      cm = max(cm, fin);
      sts32_if(lane == 0, a_fin + 4 * act, static_cast<uint32_t>(fin));
      if (!div) {
        div = start != static_cast<int>(lds32(a_bst + 4 * act));
        if (!div && p >= v && p % snap_k == snap_k - 1) {  // compare with the snapshot
          __syncwarp();
          bool diff = false;
          for (int j = lane; j < S; j += 32)
            diff |= lds32(a_c + 4 * j) != lds16(a_snap + 2 * ((p / snap_k) * S + j));
          if (!__any_sync(FULL_MASK, diff)) {
            ++p;
            break;  // converged: the rest is the current schedule
          }
        }
      }
      __syncwarp();
    }
    if (lane == 0) cmax_out[idx] = div || p >= pend ? cm : base_cmax;
    steps += p - u0;
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
//                     | c_pre [m*rs] | es_pre [n]   (cap_prefix_words)
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
  int* esp = cpre + m * rs;
  const uint32_t a_cpre = sa(cpre), a_dem = sa(I.dem), a_ctr = sa(dsm + o_ctr);
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
        cap_update_all(a_cpre, lane * rs, m, capk, req, s0, dur);
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
template <int W, bool LONG = false>
// (noinline: keeps the evaluators' argument set out of the search loop's
// register allocation -- A/B on B200, profiles/r2/ab_dispatch_noinline.txt:
// j30 +10 %, j30p +6 %, j60p +2 %, j120p +0.5 %, j120p CAPACITY +1.3 %)
__device__ __noinline__ void eval_moves_time32_dispatch(const CtaCtx& c, int n_feas,
                                                           int base_cmax, uint32_t ctr_cl) {
  const int full = c.I.H + 1 + TAU_PAD;
  if (c.I.big)
    eval_moves_time32_inc<W, true, false>(
        soff(c.I.info_r), soff(c.I.pdat), soff(c.I.req), soff(c.base), soff(c.bst),
        soff(c.scal + SC_CTR), soff(c.evs), c.I.capw[0], W == 2 ? c.I.capw[1] : 0u, c.I.hi,
        c.I.n, c.I.H, c.moves_buf, c.cmax_buf, n_feas, c.warp_words, base_cmax, c.err, ctr_cl,
        full, 0, 0, 0, 0);
  else if (c.fb && c.slots < full)
    eval_moves_time32_inc<W, false, true>(
        soff(c.I.info_r), soff(c.I.pdat), soff(c.I.req), soff(c.base), soff(c.bst),
        soff(c.scal + SC_CTR), soff(c.evs), c.I.capw[0], W == 2 ? c.I.capw[1] : 0u, c.I.hi,
        c.I.n, c.I.H, c.moves_buf, c.cmax_buf, n_feas, c.warp_words, base_cmax, c.err, ctr_cl,
        c.slots, soff(c.fb), soff(c.scal + SC_FBLOCK), soff(c.I.info_f), soff(c.I.sdat));
  else if (LONG)
    eval_moves_time32_inc<W, false, false, true>(
        soff(c.I.info_r), soff(c.I.pdat), soff(c.I.req), soff(c.base), soff(c.bst),
        soff(c.scal + SC_CTR), soff(c.evs), c.I.capw[0], W == 2 ? c.I.capw[1] : 0u, c.I.hi,
        c.I.n, c.I.H, c.moves_buf, c.cmax_buf, n_feas, c.warp_words, base_cmax, c.err, ctr_cl,
        full, 0, 0, 0, 0);
  else
    eval_moves_time32_inc<W, false, false>(
        soff(c.I.info_r), soff(c.I.pdat), soff(c.I.req), soff(c.base), soff(c.bst),
        soff(c.scal + SC_CTR), soff(c.evs), c.I.capw[0], W == 2 ? c.I.capw[1] : 0u, c.I.hi,
        c.I.n, c.I.H, c.moves_buf, c.cmax_buf, n_feas, c.warp_words, base_cmax, c.err, ctr_cl,
        full, 0, 0, 0, 0);
}

// the prefix-reusing CAPACITY warp evaluator on this CTA's copy of the current order
__device__ __noinline__ void eval_moves_cap_warp_dispatch(const CtaCtx& c, int n_feas,
                                                             bool reuse, uint32_t ctr_cl,
                                                             int base_cmax) {
  if (c.I.big)
    eval_moves_cap_warp<true>(soff(c.I.info_r), soff(c.I.pdat), soff(c.I.dem), soff(c.I.cap),
                              soff(c.base), soff(c.bst), soff(c.scal + SC_CTR), soff(c.evs),
                              soff(c.snap), c.snap_k, c.I.n, c.I.m, cap_row_stride(c.I.rmax),
                              c.moves_buf, c.cmax_buf, n_feas, c.warp_words, reuse, ctr_cl,
                              cap_demand_packed(c.I), base_cmax);
  else
    eval_moves_cap_warp<false>(soff(c.I.info_r), soff(c.I.pdat), soff(c.I.dem), soff(c.I.cap),
                               soff(c.base), soff(c.bst), soff(c.scal + SC_CTR), soff(c.evs),
                               soff(c.snap), c.snap_k, c.I.n, c.I.m, cap_row_stride(c.I.rmax),
                               c.moves_buf, c.cmax_buf, n_feas, c.warp_words, reuse, ctr_cl,
                               cap_demand_packed(c.I), base_cmax);
}

// Cluster follower (rank > 0): evaluates moves of the leader's neighbourhood
// phases until the leader is done.  Per phase: B1 (leader published the
// phase), copy the current order and its starts from the leader's shared
// memory, deal moves from the leader's counter, write makespans into the
// leader's global buffer, B2.  The instance follows the leader's (steals).
template <int MODE, int G, int W, bool LONG = false>
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
    if (MODE == MODE_CAPACITY && G == 32) {  // the current schedule's state snapshots
      __syncthreads();  // a re-staged instance's capacities are in place
      cta_snap_stride(c);
      const uint32_t l_snap = cluster_map(sa(c.snap), 0);
      for (int w = tid; w < ((c.I.n / c.snap_k) * c.snap_S + 1) / 2; w += blockDim.x)
        c.snap[w] = static_cast<int>(ld_cluster(l_snap + 4 * w));
    }
    __syncthreads();
    const uint32_t ctr = l_scal + 4 * SC_CTR;
    if constexpr (MODE == MODE_TIME) {
      eval_moves_time32_dispatch<W, LONG>(c, n_feas, base_cmax, ctr);
    } else if constexpr (G == 32) {
      eval_moves_cap_warp_dispatch(c, n_feas, true, ctr, base_cmax);
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
template <int MODE, int G, int W, bool LONG = false>
__device__ __forceinline__ void cta_eval_moves(CtaCtx& c, int n_feas) {
  if constexpr (MODE == MODE_TIME) {
    if constexpr (G == 32) {
      if (c.inc) {
        // the current order's schedule (starts -> bst), then prefix-reusing moves
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (warp == 0) {
          const bool keep = c.scal[SC_BSTOK] != 0;  // picked move had converged
          if (!keep) {
            // (a sized per-warp profile cannot hold a whole schedule: the
            // fallback region can)
            uint32_t* tau = reinterpret_cast<uint32_t*>(c.fb ? c.fb : c.evs);
            int* es = reinterpret_cast<int*>(tau) + (c.I.H + 1) * W;
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
        eval_moves_time32_dispatch<W, LONG>(c, n_feas, c.scal[SC_BASEC], cluster_counter(c));
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
      int cm = 0;
      if (c.inc)
        cm = sgs_cap_warp(sa(c.I.info_f), sa(c.I.sdat), sa(c.I.dem), c.I.cap, c.I.n, c.I.m,
                          cap_row_stride(c.I.rmax), sa(c.evs), sa(c.base), c.bst, sa(c.snap),
                          c.snap_k);
      if (lane == 0) {
        c.scal[SC_CTR] = 0;
        c.scal[SC_STEPS] = c.inc ? c.I.n : 0;
        c.scal[SC_BASEC] = cm;
      }
    }
    __syncthreads();
    cluster_phase_begin(c, n_feas);
    eval_moves_cap_warp_dispatch(c, n_feas, c.inc, cluster_counter(c), c.scal[SC_BASEC]);
    cluster_phase_end(c);
  } else {
    // prefix reuse pays from j60 on; on j30-size projects the per-batch state
    // copy and the current-schedule pass outweigh the shorter suffixes
    // (131.9 M vs 163 M schedules/s on j30, 147.4 M vs 123 M on j60)
    if (c.inc && c.I.n >= 48) {
      // the current order's schedule (starts -> bst) on warp 0's prefix scratch
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      if (warp == 0) {
        // (warp 0's whole scratch: the per-lane states are free between phases;
        // eval_warp_words reserves cap_warp_words there)
        int* scr = c.evs;
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
      uint32_t* tau = reinterpret_cast<uint32_t*>(c.fb ? c.fb : c.evs);
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

}  // namespace rt
