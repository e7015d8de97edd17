// sgs.cuh -- serial schedule generation (kernels.py:152-194) on the device.
//
// Two evaluators, bit-exact with the reference for precedence-feasible
// orders:
//
//  * TIME (time-indexed resource profile, kernels.py:117-146): a group of G
//    lanes (G = 32 / 16 / 8, S = 32/G schedules per warp) owns one schedule.
//    The profile is one packed word per time slot per W (all resources of the
//    slot as 8- or 16-bit lanes), so the window test for a slot is one
//    OR/SUB/AND on the word.  The group tests G consecutive slots per round,
//    ballots the verdicts and finds the first run of `dur` fitting slots with
//    bit tricks (carry of the run across rounds).  Slots at or beyond the
//    profile's high-water mark `hw` are implicitly at full capacity, so no
//    per-schedule reset of the profile is needed (the reference bounds its
//    reset by `touched` for the same reason, kernels.py:343/359/170-172).
//
//  * CAP (capacity-indexed state, kernels.py:68-110, Alg. 4): one thread per
//    schedule; per-resource descending arrays c_k[R_k] and the copy buffer
//    live in shared memory interleaved by lane (word j of lane l at
//    j*32 + l), so the data-dependent indexing is bank-conflict free.
//
// Both use push-based precedence: when an activity finishes at f, every
// successor's earliest start es[s] = max(es[s], f).  For a topological order
// es[act] equals max over preds of (start + dur) exactly (kernels.py:177-182).
#pragma once
#include "common.cuh"

namespace rt {

// one packed slot test: every lane of `w` holds >= the matching lane of `r`
__device__ __forceinline__ bool fits1(uint32_t w, uint32_t r, uint32_t hi) {
  return (((w | hi) - r) & hi) == hi;
}

// Time-indexed SGS for one schedule per G-lane group.
//   tau:   the group's profile, (H+1)*W words, slot t at tau[t*W + w]
//   es:    the group's [n] earliest-start scratch
//   act_at(pos) -> activity at position pos (group-uniform)
//   info / push_dat: per-activity records (common.cuh) and the edge targets
//     finish times propagate to (I.info_f + I.sdat forward; I.info_r +
//     I.pdat for the reversed project)
//   starts_out: optional [n] (lane 0 of the group writes)
// Returns the makespan (group-uniform).  `active` false: the group only
// joins the warp-collective votes.
//
// Per activity: record + es in two LDS; no scan when the activity needs no
// resource, or when es is at/after the materialised profile (everything there
// is free).  Otherwise each round tests G slots (one LDS each lane), ballots,
// and resolves the earliest window branch-free: the carried run from the
// previous round, else the first run of `dur` ones inside the round (five
// precomputed doubling shifts).
template <int G, int W, class ActFn>
__device__ __forceinline__ int sgs_time_group(const SInst& I, uint32_t* __restrict__ tau,
                                              int* __restrict__ es, ActFn act_at,
                                              const int4* __restrict__ info,
                                              const int* __restrict__ push_dat,
                                              int* __restrict__ starts_out, bool active,
                                              int* err) {
  const int lane = threadIdx.x & 31;
  const int lane_g = lane & (G - 1);
  const int gshift = lane & ~(G - 1) & 31;
  constexpr uint32_t GM = (G == 32) ? 0xffffffffu : ((1u << G) - 1u);
  const int n = I.n, H = I.H;
  const uint32_t hi = I.hi;
  const uint32_t cap0 = I.capw[0];
  const uint32_t cap1 = W == 2 ? I.capw[1] : 0u;

  if (active)
    for (int a = lane_g; a < n; a += G) es[a] = 0;
  __syncwarp();

  int cmax = 0;
  int hw = 0;  // profile slots [0, hw) are materialised; >= hw are at capacity
  for (int pos = 0; pos < n; ++pos) {
    int4 rec = make_int4(0, 0, 0, 0);
    int act = 0, esv = 0;
    uint32_t r1 = 0;
    if (active) {
      act = act_at(pos);
      rec = info[act];
      esv = es[act];
      if (W == 2) r1 = I.req[act * 2 + 1];
    }
    const int dur = rec.x;
    const uint32_t r0 = static_cast<uint32_t>(rec.y);
    const bool need = dur > 0 && (r0 | r1) != 0;
    int start = esv;
    bool done = !(need && esv < hw);
    int t0 = esv, carry = 0;
    while (__any_sync(FULL_MASK, !done)) {
      bool ok = false;
      if (!done) {
        const int t = t0 + lane_g;
        uint32_t w0 = cap0, w1 = cap1;
        if (t < hw) {
          w0 = tau[t * W];
          if (W == 2) w1 = tau[t * W + 1];
        }
        ok = t < H && fits1(w0, r0, hi) && (W == 1 || fits1(w1, r1, hi));
      }
      const uint32_t m = (__ballot_sync(FULL_MASK, ok) >> gshift) & GM;
      if (!done) {
        const uint32_t zm = ~m & GM;
        const int z = zm ? __ffs(zm) - 1 : G;
        uint32_t y = 0;
        if (dur <= G) {
          const int sh = rec.w;
          y = m;
          y &= y >> (sh & 63);
          y &= y >> ((sh >> 6) & 63);
          y &= y >> ((sh >> 12) & 63);
          y &= y >> ((sh >> 18) & 63);
          y &= y >> ((sh >> 24) & 63);
        }
        if (carry + z >= dur) {
          start = t0 - carry;
          done = true;
        } else if (y) {
          start = t0 + __ffs(y) - 1;
          done = true;
        } else {
          carry = zm ? __clz(~(m << (32 - G))) : carry + G;
          t0 += G;
          if (t0 >= H) {  // cannot happen for valid instances
            start = H;
            done = true;
            if (lane_g == 0) set_err(err, DE_NO_WINDOW);
          }
        }
      }
    }
    if (active) {
      const int fin = start + dur;
      if (need) {
        // materialise [hw, start) at capacity, subtract the demand on [start, fin)
        for (int t = hw + lane_g; t < start; t += G) {
          tau[t * W] = cap0;
          if (W == 2) tau[t * W + 1] = cap1;
        }
        for (int t = start + lane_g; t < fin; t += G) {
          const bool old = t < hw;
          tau[t * W] = (old ? tau[t * W] : cap0) - r0;
          if (W == 2) tau[t * W + 1] = (old ? tau[t * W + 1] : cap1) - r1;
        }
        hw = max(hw, fin);
      }
      cmax = max(cmax, fin);
      const int e0 = rec.z & 0xffff, ecnt = rec.z >> 16;
      for (int e = lane_g; e < ecnt; e += G) {
        const int s = push_dat[e0 + e];
        if (es[s] < fin) es[s] = fin;
      }
      if (starts_out && lane_g == 0) starts_out[act] = start;
    }
    __syncwarp();
  }
  return cmax;
}

// ---- explicit shared-memory access (32-bit shared addresses)
__device__ __forceinline__ uint32_t sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int4 lds128(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Warp-uniform time-indexed SGS (G = 32, one schedule per warp).  Same
// results as sgs_time_group; every branch is warp-uniform and every shared
// access goes through a precomputed 32-bit shared address.
//   a_ord:  the warp's order [n] (already swapped)      a_info: records [n]
//   a_push: edge targets of the push graph               a_req:  packed demand
//   a_tau:  profile (H+1)*W words                        a_es:   [n] scratch
template <int W>
__device__ __forceinline__ int sgs_time_warp(uint32_t a_info, uint32_t a_push, uint32_t a_req,
                                             uint32_t cap0, uint32_t cap1, uint32_t hi, int n,
                                             int H, uint32_t a_tau, uint32_t a_es,
                                             uint32_t a_ord, int* __restrict__ starts_out,
                                             int* err) {
  const int lane = threadIdx.x & 31;
  for (int a = lane; a < n; a += 32) sts32(a_es + 4 * a, 0);
  __syncwarp();
  int cmax = 0, hw = 0;
  for (int pos = 0; pos < n; ++pos) {
    const int act = static_cast<int>(lds32(a_ord + 4 * pos));
    const int4 rec = lds128(a_info + 16 * act);
    const int esv = static_cast<int>(lds32(a_es + 4 * act));
    const int dur = rec.x;
    const uint32_t r0 = static_cast<uint32_t>(rec.y);
    const uint32_t r1 = W == 2 ? lds32(a_req + 8 * act + 4) : 0u;
    int start = esv;
    if (dur > 0 && (r0 | r1) != 0) {
      if (esv < hw) {
        const int sh = rec.w;
        const int s0 = sh & 63, s1 = (sh >> 6) & 63, s2 = (sh >> 12) & 63,
                  s3 = (sh >> 18) & 63, s4 = (sh >> 24) & 63;
        int t0 = esv, carry = 0;
        for (;;) {
          const int t = t0 + lane;
          uint32_t w0 = cap0, w1 = cap1;
          if (t < hw) {
            w0 = lds32(a_tau + 4 * W * t);
            if (W == 2) w1 = lds32(a_tau + 4 * W * t + 4);
          }
          const bool ok = t < H && fits1(w0, r0, hi) && (W == 1 || fits1(w1, r1, hi));
          const uint32_t m = __ballot_sync(FULL_MASK, ok);
          const int z = __ffs(~m) - 1;              // -1 when all 32 slots fit
          if (carry + (z < 0 ? 32 : z) >= dur) {
            start = t0 - carry;
            break;
          }
          if (dur <= 32) {
            uint32_t y = m;
            y &= y >> s0;
            y &= y >> s1;
            y &= y >> s2;
            y &= y >> s3;
            y &= y >> s4;
            if (y) {
              start = t0 + __ffs(y) - 1;
              break;
            }
          }
          carry = z < 0 ? carry + 32 : __clz(~m);
          t0 += 32;
          if (t0 >= H) {  // cannot happen for valid instances
            start = H;
            if (lane == 0) set_err(err, DE_NO_WINDOW);
            break;
          }
        }
      }
      const int fin = start + dur;
      if (start > hw)
        for (int t = hw + lane; t < start; t += 32) {
          sts32(a_tau + 4 * W * t, cap0);
          if (W == 2) sts32(a_tau + 4 * W * t + 4, cap1);
        }
      for (int t = start + lane; t < fin; t += 32) {
        const uint32_t adr = a_tau + 4 * W * t;
        const bool old = t < hw;
        sts32(adr, (old ? lds32(adr) : cap0) - r0);
        if (W == 2) sts32(adr + 4, (old ? lds32(adr + 4) : cap1) - r1);
      }
      hw = max(hw, fin);
    }
    const int fin = start + dur;
    cmax = max(cmax, fin);
    const int e0 = rec.z & 0xffff, ecnt = rec.z >> 16;
    for (int e = lane; e < ecnt; e += 32) {
      const uint32_t adr = a_es + 4 * lds32(a_push + 4 * (e0 + e));
      if (static_cast<int>(lds32(adr)) < fin) sts32(adr, static_cast<uint32_t>(fin));
    }
    if (starts_out && lane == 0) starts_out[act] = start;
    __syncwarp();
  }
  return cmax;
}

// Capacity-indexed SGS, one thread per schedule.
//   st: the warp's interleaved scratch; word j of slot `slot` at st[j*SK + slot]
//       (SK = lanes sharing the scratch, 32 normally: conflict-free)
//       layout: c[m*rmax] | copy_buf[rmax] | es[n]
template <class ActFn>
__device__ __forceinline__ int sgs_cap_thread(const SInst& I, int* __restrict__ st, int SK,
                                              int slot, ActFn act_at,
                                              const int* __restrict__ push_ptr,
                                              const int* __restrict__ push_dat,
                                              int* __restrict__ starts_out) {
  const int n = I.n, m = I.m, R = I.rmax;
  int* c = st + slot;                 // c[(k*R + i)*SK]
  int* cb = st + (m * R) * SK + slot;  // cb[i*SK]
  int* es = cb + R * SK;              // es[a*SK]
  for (int j = 0; j < m * R; ++j) c[j * SK] = 0;
  for (int a = 0; a < n; ++a) es[a * SK] = 0;
  int cmax = 0;
  for (int pos = 0; pos < n; ++pos) {
    const int act = act_at(pos);
    const int dur = I.dur[act];
    const int* dem = I.dem + act * m;
    // Eq. 7 (kernels.py:68-78)
    int es_res = 0;
    for (int k = 0; k < m; ++k) {
      const int req = dem[k];
      if (req > 0) es_res = max(es_res, c[(k * R + I.cap[k] - req) * SK]);
    }
    const int start = max(es[act * SK], es_res);
    // Alg. 4 (kernels.py:81-110), quirks preserved
    for (int k = 0; k < m; ++k) {
      const int req = dem[k];
      int effort = req * dur;
      if (effort <= 0) continue;
      int* ck = c + (k * R) * SK;
      const int capk = I.cap[k];
      int copy_idx = 0;
      int new_time = start + dur;
      for (int res_idx = 0; effort > 0 && res_idx < capk; ++res_idx) {
        const int cv = ck[res_idx * SK];
        if (cv < new_time) {
          if (copy_idx >= req) new_time = cb[(copy_idx - req) * SK];
          const int fl = cv < start ? start : cv;
          const int diff = new_time - fl;
          if (effort - diff > 0) {
            effort -= diff;
            cb[copy_idx * SK] = cv;
            ++copy_idx;
            ck[res_idx * SK] = new_time;
          } else {
            ck[res_idx * SK] = fl + effort;
            effort = 0;
          }
        }
      }
    }
    const int fin = start + dur;
    cmax = max(cmax, fin);
    for (int e = push_ptr[act]; e < push_ptr[act + 1]; ++e) {
      const int s = push_dat[e];
      if (es[s * SK] < fin) es[s * SK] = fin;
    }
    if (starts_out) starts_out[act] = start;
  }
  return cmax;
}

__host__ __device__ __forceinline__ int cap_thread_words(int n, int m, int rmax) {
  return m * rmax + rmax + n;  // per lane
}

}  // namespace rt
