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

template <int W>
struct Req {
  uint32_t r[W];
};

// Time-indexed SGS for one schedule per G-lane group.
//   tau:   group's profile, (H+1)*W words, slot t at tau[t*W + w]
//   es:    group's [n] earliest-start scratch
//   act_at(pos) -> activity at position pos (group-uniform)
//   push_ptr/push_dat: graph along which finish times propagate (successors
//     for a forward pass; predecessors for the reversed project)
//   starts_out: optional [n] (lane 0 of the group writes)
// Returns the makespan (group-uniform).  `active` false: the group only
// joins the warp-collective ballots.
template <int G, int W, class ActFn>
__device__ __forceinline__ int sgs_time_group(const SInst& I, uint32_t* __restrict__ tau,
                                              int* __restrict__ es, ActFn act_at,
                                              const int* __restrict__ push_ptr,
                                              const int* __restrict__ push_dat,
                                              int* __restrict__ starts_out, bool active,
                                              int* err) {
  const int lane = threadIdx.x & 31;
  const int lane_g = lane & (G - 1);
  const int gshift = lane & ~(G - 1) & 31;
  const uint32_t GM = (G == 32) ? 0xffffffffu : ((1u << G) - 1u);
  const int n = I.n, H = I.H;
  const uint32_t hi = I.hi;

  if (active)
    for (int a = lane_g; a < n; a += G) es[a] = 0;
  __syncwarp();

  uint32_t capw[W];
#pragma unroll
  for (int w = 0; w < W; ++w) capw[w] = I.capw[w];

  int cmax = 0;
  int hw = 0;  // profile slots [0, hw) are materialised; >= hw are full
  for (int pos = 0; pos < n; ++pos) {
    int act = 0, dur = 0, esv = 0;
    bool need = false;
    Req<W> rq;
#pragma unroll
    for (int w = 0; w < W; ++w) rq.r[w] = 0;
    if (active) {
      act = act_at(pos);
      dur = I.dur[act];
      esv = es[act];
      uint32_t any = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        rq.r[w] = I.req[act * W + w];
        any |= rq.r[w];
      }
      need = dur > 0 && any != 0;
    }
    int start = esv;
    // window scan (kernels.py:117-136): first t >= es with [t, t+dur) fitting
    bool done = !need;
    int t0 = esv, carry = 0;
    while (__any_sync(FULL_MASK, !done)) {
      bool ok = false;
      if (!done) {
        const int t = t0 + lane_g;
        if (t < H) {
          if (t >= hw) {
            ok = true;
          } else {
            ok = true;
#pragma unroll
            for (int w = 0; w < W; ++w) ok = ok && fits1(tau[t * W + w], rq.r[w], hi);
          }
        }
      }
      const uint32_t bal = __ballot_sync(FULL_MASK, ok);
      if (!done) {
        const uint32_t m = (bal >> gshift) & GM;
        const int z = (m == GM) ? G : (__ffs(~m) - 1);
        if (carry + z >= dur) {
          start = t0 - carry;
          done = true;
        } else if (z == G) {
          carry += G;
        } else {
          uint32_t y = 0;
          if (dur <= G) {
            y = m;
            int k = 1;
            while (2 * k <= dur) {
              y &= y >> k;
              k <<= 1;
            }
            if (k < dur) y &= y >> (dur - k);
          }
          if (y) {
            start = t0 + __ffs(y) - 1;
            done = true;
          } else {
            carry = __clz(~(m << (32 - G)));
          }
        }
        t0 += G;
        if (!done && t0 >= H) {  // cannot happen for valid instances
          start = H;
          done = true;
          if (lane_g == 0) set_err(err, DE_NO_WINDOW);
        }
      }
    }
    if (active) {
      const int fin = start + dur;
      if (need) {
        // materialise [hw, start) at full capacity, subtract on [start, fin)
        for (int t = hw + lane_g; t < start; t += G) {
#pragma unroll
          for (int w = 0; w < W; ++w) tau[t * W + w] = capw[w];
        }
        for (int t = start + lane_g; t < fin; t += G) {
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const uint32_t v = (t >= hw) ? capw[w] : tau[t * W + w];
            tau[t * W + w] = v - rq.r[w];
          }
        }
        hw = max(hw, fin);
      }
      cmax = max(cmax, fin);
      const int e0 = push_ptr[act], e1 = push_ptr[act + 1];
      for (int e = e0 + lane_g; e < e1; e += G) {
        const int s = push_dat[e];
        if (es[s] < fin) es[s] = fin;
      }
      if (starts_out && lane_g == 0) starts_out[act] = start;
    }
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
