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
// predicated forms: straight-line code instead of a (potentially divergent)
// branch with a reconvergence point around it
__device__ __forceinline__ uint32_t lds32_if(bool p, uint32_t a, uint32_t dflt) {
  uint32_t v = dflt;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q ld.shared.u32 %0, [%2];\n\t}"
               : "+r"(v) : "r"(static_cast<uint32_t>(p)), "r"(a));
  return v;
}
__device__ __forceinline__ void sts32_if(bool p, uint32_t a, uint32_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.u32 [%1], %2;\n\t}"
               ::"r"(static_cast<uint32_t>(p)), "r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_max_shared_if(bool p, uint32_t a, int v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q red.shared.max.s32 [%1], %2;\n\t}"
               ::"r"(static_cast<uint32_t>(p)), "r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void sts64_if(bool p, uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.v2.u32 [%1], {%2, %3};\n\t}"
               ::"r"(static_cast<uint32_t>(p)), "r"(a), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(static_cast<unsigned short>(v)) : "memory");
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
// *a += v as one shared-memory reduction (no return value)
__device__ __forceinline__ void red_add_shared(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// es[s] = max(es[s], v) as one shared-memory reduction (no return value)
__device__ __forceinline__ void red_max_shared(uint32_t a, int v) {
  asm volatile("red.shared.max.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// a - b kept as one subtraction (the guard-bit test below then folds the
// complement into its LOP3 instead of being rewritten as ~a + b)
__device__ __forceinline__ uint32_t sub_opaque(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// v through an opaque move: keeps a precomputed base address (e.g. profile +
// 4 W lane) a single register the slot offsets are added to, instead of the
// compiler re-distributing it into (t + lane) * 4 + profile
__device__ __forceinline__ uint32_t opaque(uint32_t v) {
  uint32_t r;
  asm("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// wrap-mode funnel shift: y >> (s & 31) (the window shift fields are 5 bits)
__device__ __forceinline__ uint32_t shr_wrap(uint32_t y, int s) {
  return __funnelshift_r(y, 0u, static_cast<uint32_t>(s));
}

// run of `dur` ones: y &= y >> s_i for the five packed fields of `sh`
__device__ __forceinline__ uint32_t window_runs(uint32_t m, int sh) {
  uint32_t y = m;
  y &= shr_wrap(y, sh);
  y &= shr_wrap(y, sh >> 5);
  y &= shr_wrap(y, sh >> 10);
  y &= shr_wrap(y, sh >> 15);
  y &= shr_wrap(y, sh >> 20);
  return y;
}

// Earliest window (kernels.py:117-136) for one activity, whole warp:
// first t >= esv with [t, t+dur) fitting, slots >= hw at capacity, t+dur <= H.
// Each round tests 32 slots and resolves the window branch-free: the run
// carried from the previous round, else the first run of `dur` ones.
// MAT: the profile is materialised at capacity from hw on (and 32 slots past
// the horizon), so the load needs no test, and every packed lane carries its
// guard bit (hi) set -- a fitting demand leaves it set, so the test is one
// subtraction
// Lane i tests slot t0 + i.  With MAT, a_tau is the lane's base address
// (profile + 4 W lane), so a slot address is one multiply-add.
template <int W, bool HCHK, bool MAT = false>
__device__ __forceinline__ uint32_t window_fits_ballot(uint32_t a_tau, int t0, int hw, int H,
                                                       uint32_t r0, uint32_t r1, uint32_t cap0,
                                                       uint32_t cap1, uint32_t hi) {
  const int t = t0 + static_cast<int>(threadIdx.x & 31);
  const bool in = MAT || t < hw;
  const uint32_t adr = MAT ? a_tau + 4 * W * t0 : a_tau + 4 * W * t;
  const uint32_t w0 = MAT ? lds32(adr) : lds32_if(in, adr, cap0);
  const uint32_t w1 = W == 2 ? (MAT ? lds32(adr + 4) : lds32_if(in, adr + 4, cap1)) : cap1;
  // HCHK = false (the SGS): no t < H test -- packing rejects demands above
  // capacity, so every activity fits from hw on (slots >= hw are free) and no
  // window reaches past hw + dur <= H; the scan loop keeps its t0 >= H guard.
  // The single-step state operation (arbitrary states) keeps the test, as the
  // reference's scan stops at the horizon (kernels.py:127).
  if (MAT)  // the materialised profile keeps every lane's guard bit set
    return __ballot_sync(FULL_MASK, (!HCHK || t < H) && (~sub_opaque(w0, r0) & hi) == 0u &&
                                        (W == 1 || (~sub_opaque(w1, r1) & hi) == 0u));
  return __ballot_sync(FULL_MASK, (!HCHK || t < H) && fits1(w0, r0, hi) &&
                                      (W == 1 || fits1(w1, r1, hi)));
}

// BIG = false (every duration <= 32): a lane whose window would end past the
// round cannot hit -- m >> lane brings in zeros, and dmask covers them -- so
// the candidate test is implied.
template <int W, bool BIG = true, bool HCHK = false, bool MAT = false>
__device__ __forceinline__ int warp_window(uint32_t a_tau, int hw, int H, uint32_t r0,
                                           uint32_t r1, uint32_t cap0, uint32_t cap1,
                                           uint32_t hi, int esv, int dur, uint32_t dmask,
                                           int* err) {
  const int lane = threadIdx.x & 31;
  // lane i tests the window [t0+i, t0+i+dur) inside the round: a candidate
  // iff it ends in the round, a hit iff dur fitting slots start at bit i
  const bool cand = !BIG || lane + dur <= 32;
  // first round, peeled: nothing is carried in, so lane 0's test covers the
  // window starting at esv
  uint32_t m = window_fits_ballot<W, HCHK, MAT>(a_tau, esv, hw, H, r0, r1, cap0, cap1, hi);
  uint32_t y = __ballot_sync(FULL_MASK, cand && (~(m >> lane) & dmask) == 0u);
  int start = esv + __ffs(y) - 1;  // (one branch on the first-round path)
  if (y == 0u) {
    int t0 = esv, carry = m == FULL_MASK ? 32 : __clz(~m);
    for (;;) {
      t0 += 32;
      if (t0 >= H) {  // cannot happen for valid instances
        if (lane == 0) set_err(err, DE_NO_WINDOW);
        start = H;
        break;
      }
      m = window_fits_ballot<W, HCHK, MAT>(a_tau, t0, hw, H, r0, r1, cap0, cap1, hi);
      const int tz = __popc(m & ~(m + 1u));  // fitting slots from t0 on (32: all)
      if (carry + tz >= dur) {
        start = t0 - carry;
        break;
      }
      y = __ballot_sync(FULL_MASK, cand && (~(m >> lane) & dmask) == 0u);
      if (y) {
        start = t0 + __ffs(y) - 1;
        break;
      }
      carry = tz == 32 ? carry + 32 : __clz(~m);
    }
  }
  return start;
}

// Book an activity on [start, start+dur) (kernels.py:139-146): materialise
// [hw, start) at capacity, subtract the packed demand, advance hw.
template <int W, bool BIG = true>
__device__ __forceinline__ void warp_commit(uint32_t a_tau, int& hw, int start, int dur,
                                            uint32_t r0, uint32_t r1, uint32_t cap0,
                                            uint32_t cap1) {
  const int lane = threadIdx.x & 31;
  const int fin = start + dur;
  const int gap = start - hw;
  if (gap > 0) {  // materialise [hw, start): one predicated store per lane, a loop past 32
    const uint32_t adr = a_tau + 4 * W * (hw + lane);
    sts32_if(lane < gap, adr, cap0);
    if (W == 2) sts32_if(lane < gap, adr + 4, cap1);
    for (int t = hw + 32 + lane; t < start; t += 32) {
      sts32(a_tau + 4 * W * t, cap0);
      if (W == 2) sts32(a_tau + 4 * W * t + 4, cap1);
    }
  }
  const int t = start + lane;  // one slot per lane (a loop only for dur > 32)
  {
    const uint32_t adr = a_tau + 4 * W * t;
    const bool in = lane < dur, old = in && t < hw;
    sts32_if(in, adr, lds32_if(old, adr, cap0) - r0);
    if (W == 2) sts32_if(in, adr + 4, lds32_if(old, adr + 4, cap1) - r1);
  }
  if (BIG && dur > 32)
    for (int tt = t + 32; tt < fin; tt += 32) {
      const uint32_t adr = a_tau + 4 * W * tt;
      const bool old = tt < hw;
      sts32(adr, (old ? lds32(adr) : cap0) - r0);
      if (W == 2) sts32(adr + 4, (old ? lds32(adr + 4) : cap1) - r1);
    }
  hw = max(hw, fin);
}

// warp_commit on a materialised profile (slots >= hw hold the capacity):
// no gap to fill, every booked slot is a read-modify-write.  a_tau_l: the
// lane's base address (profile + 4 W lane).
template <int W, bool BIG = true>
__device__ __forceinline__ void warp_commit_mat(uint32_t a_tau_l, int& hw, int start, int dur,
                                                uint32_t r0, uint32_t r1) {
  const int lane = threadIdx.x & 31;
  {
    const uint32_t adr = a_tau_l + 4 * W * start;  // start + lane < H + 32: inside the pad
    const bool in = lane < dur;
    sts32_if(in, adr, lds32(adr) - r0);
    if (W == 2) sts32_if(in, adr + 4, lds32(adr + 4) - r1);
  }
  if (BIG && dur > 32)
    for (int k = 32; k < dur - lane; k += 32) {
      const uint32_t adr = a_tau_l + 4 * W * (start + k);
      sts32(adr, lds32(adr) - r0);
      if (W == 2) sts32(adr + 4, lds32(adr + 4) - r1);
    }
  hw = max(hw, start + dur);
}

// Inverse of warp_commit below the mark `hw_keep`: give the demand on
// [start, min(start+dur, hw_keep)) back.  Slots at or above hw_keep need no
// undo -- resetting the high-water mark to hw_keep makes them implicit
// capacity again.
template <int W>
__device__ __forceinline__ void warp_uncommit(uint32_t a_tau, int hw_keep, int start, int dur,
                                              uint32_t r0, uint32_t r1) {
  const int lane = threadIdx.x & 31;
  const int e = min(start + dur, hw_keep);
  for (int t = start + lane; t < e; t += 32) {
    const uint32_t adr = a_tau + 4 * W * t;
    sts32(adr, lds32(adr) + r0);
    if (W == 2) sts32(adr + 4, lds32(adr + 4) + r1);
  }
}

// One activity of the warp-uniform time-indexed SGS (see sgs_time_warp), push
// form: the finish time goes to the successors' es.  Returns the start.
// BIG = false: the instance has no duration and no fan-out above 32 (I.big).
template <int W, bool BIG = true>
__device__ __forceinline__ int time_step_warp(int act, const int4& rec, uint32_t a_push,
                                               uint32_t a_req, uint32_t cap0, uint32_t cap1,
                                               uint32_t hi, int H, uint32_t a_tau,
                                               uint32_t a_es, int& hw, int& cmax,
                                               int* __restrict__ starts_out, int* err) {
  const int lane = threadIdx.x & 31;
  const int esv = static_cast<int>(lds32(a_es + 4 * act));
  const int dur = rec.x;
  const uint32_t r0 = static_cast<uint32_t>(rec.y);
  const uint32_t r1 = W == 2 ? lds32(a_req + 8 * act + 4) : 0u;
  int start = esv;
  if (dur > 0 && (r0 | r1) != 0) {
    if (esv < hw)
      start = warp_window<W, BIG>(a_tau, hw, H, r0, r1, cap0, cap1, hi, esv, dur,
                                     static_cast<uint32_t>(rec.w), err);
    warp_commit<W, BIG>(a_tau, hw, start, dur, r0, r1, cap0, cap1);
  }
  const int fin = start + dur;
  cmax = max(cmax, fin);
  const int e0 = rec.z & 0xffff, ecnt = rec.z >> 16;
  {  // push the finish time to the successors' es
    const bool pe = lane < ecnt;
    red_max_shared_if(pe, a_es + 4 * lds32_if(pe, a_push + 4 * (e0 + lane), 0u), fin);
  }
  if (BIG && ecnt > 32)
    for (int e = lane + 32; e < ecnt; e += 32)
      red_max_shared(a_es + 4 * lds32(a_push + 4 * (e0 + e)), fin);
  if (starts_out && lane == 0) starts_out[act] = start;
  __syncwarp();
  return start;
}

// One activity with pulled precedence: es = max over the predecessors of
// fin[pred] (kernels.py:177-182 computes es_prec exactly so), then the window
// and the booking as time_step_warp; fin[act] is recorded.  rec is the
// activity's pull record (info_r: duration, demand, predecessor span, mask).
// MAT: materialised profile (see window_fits_ballot); a_tau and a_pdat are
// then the lane's base addresses (+ 4 W lane, + 4 lane).
// SIZED (the search evaluator's profile of P < H + 1 + TAU_PAD slots; no
// duration above 32): a booking must end at least 64 slots before P -- every
// window read then stays inside the profile (a window is found in the round
// holding max(es, hw) or the next one) -- else the step books nothing and
// sets ovf (the caller abandons the move to an exact full-horizon
// evaluation); with ovf already set the step touches no profile slot.
template <int W, bool BIG, bool SYNC = true, bool MAT = false, bool SIZED = false>
__device__ __forceinline__ int time_step_pull(int act, const int4& rec, uint32_t a_pdat,
                                              uint32_t a_req, uint32_t cap0, uint32_t cap1,
                                              uint32_t hi, int H, uint32_t a_tau, uint32_t a_fin,
                                              int& hw, int& cmax, int* err, int P = 0,
                                              bool* ovf = nullptr) {
  static_assert(!SIZED || !BIG, "sized profiles are for durations <= 32");
  const int lane = threadIdx.x & 31;
  const int p0 = rec.z & 0xffff, pc = rec.z >> 16;
  // the predecessor lists are padded by 32 entries (common.cuh): every lane
  // loads, lanes past the span are masked (MAT: a_pdat is the lane's base)
  // (MAT: the span's start as one PRMT, then one multiply-add for the address)
  const uint32_t p0b = MAT ? __byte_perm(static_cast<uint32_t>(rec.z), 0u, 0x4410) : 0u;
  int f = static_cast<int>(lds32(a_fin + 4 * lds32(MAT ? a_pdat + 4 * p0b : a_pdat + 4 * (p0 + lane))));
  // lane < pc, as one compare of the record word with (lane + 1) << 16
  f = (MAT ? static_cast<uint32_t>(rec.z) >= ((lane + 1u) << 16) : lane < pc) ? f : 0;
  if (BIG && pc > 32)
    for (int e = lane + 32; e < pc; e += 32)
      f = max(f, static_cast<int>(lds32(a_fin + 4 * lds32(MAT ? a_pdat + 4 * (p0 + e - lane)
                                                              : a_pdat + 4 * (p0 + e)))));
  const int esv = __reduce_max_sync(FULL_MASK, f);
  const int dur = rec.x;
  const uint32_t r0 = static_cast<uint32_t>(rec.y);
  const uint32_t r1 = W == 2 ? lds32(a_req + 8 * act + 4) : 0u;
  int start = esv;
  if constexpr (SIZED) {
    if (!*ovf) {
      start = warp_window<W, BIG, false, MAT>(a_tau, hw, H, r0, r1, cap0, cap1, hi, esv, dur,
                                              static_cast<uint32_t>(rec.w), err);
      if (start + dur + 64 > P)
        *ovf = true;
      else
        warp_commit_mat<W, BIG>(a_tau, hw, start, dur, r0, r1);
    }
  } else if constexpr (!BIG) {
    // no branch on es < hw or on the demand: from hw on every slot is free, so
    // the first round returns es; a zero demand or duration books nothing
    start = warp_window<W, BIG, false, MAT>(a_tau, hw, H, r0, r1, cap0, cap1, hi, esv, dur,
                                            static_cast<uint32_t>(rec.w), err);
    if (MAT)
      warp_commit_mat<W, BIG>(a_tau, hw, start, dur, r0, r1);
    else
      warp_commit<W, BIG>(a_tau, hw, start, dur, r0, r1, cap0, cap1);
  } else if (dur > 0 && (r0 | r1) != 0) {
    if (esv < hw)
      start = warp_window<W, BIG, false, MAT>(a_tau, hw, H, r0, r1, cap0, cap1, hi, esv, dur,
                                              static_cast<uint32_t>(rec.w), err);
    if (MAT)
      warp_commit_mat<W, BIG>(a_tau, hw, start, dur, r0, r1);
    else
      warp_commit<W, BIG>(a_tau, hw, start, dur, r0, r1, cap0, cap1);
  }
  const int fin = start + dur;
  if (!SIZED || !*ovf) cmax = max(cmax, fin);
  sts32_if(lane == 0, a_fin + 4 * act, static_cast<uint32_t>(fin));
  // SYNC = false: the caller synchronises after its own bookkeeping, so the
  // next step's REDUX needs no divergence check
  if (SYNC) __syncwarp();
  return start;
}

// Warp-uniform time-indexed SGS (G = 32, one schedule per warp).  Same
// results as the reference's time-indexed SGS; every branch is warp-uniform
// and every shared access goes through a precomputed 32-bit shared address.
// The next activity's order entry and record depend only on the order, so
// they are loaded one activity ahead (loop unrolled by two so the prefetch
// needs no register copies); precedence is pushed (finish time ->
// successors' es) so an activity's es is a single load.
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
  int act_a = static_cast<int>(lds32(a_ord));
  int4 rec_a = lds128(a_info + 16 * act_a);
  int pos = 0;
  for (; pos + 1 < n; pos += 2) {
    const int act_b = static_cast<int>(lds32(a_ord + 4 * (pos + 1)));
    const int4 rec_b = lds128(a_info + 16 * act_b);
    time_step_warp<W>(act_a, rec_a, a_push, a_req, cap0, cap1, hi, H, a_tau, a_es, hw, cmax,
                      starts_out, err);
    act_a = static_cast<int>(lds32(a_ord + 4 * min(pos + 2, n - 1)));
    rec_a = lds128(a_info + 16 * act_a);
    time_step_warp<W>(act_b, rec_b, a_push, a_req, cap0, cap1, hi, H, a_tau, a_es, hw, cmax,
                      starts_out, err);
  }
  if (pos < n)
    time_step_warp<W>(act_a, rec_a, a_push, a_req, cap0, cap1, hi, H, a_tau, a_es, hw, cmax,
                      starts_out, err);
  return cmax;
}

// Split-warp time-indexed SGS: S = 32/G schedules per warp (G = 16 or 8
// lanes each), same results as sgs_time_warp.  Group state is predicated
// instead of branched (the warp runs the scan rounds until every group has
// found its window), so per-activity work -- record loads, update, push -- is
// shared by S schedules in one instruction stream.
//   a_ord/a_es/a_tau: this lane's group arrays (32-bit shared addresses)
//   active: this group has a schedule (false: it only joins the votes)
template <int G, int W>
__device__ __forceinline__ int sgs_time_split(uint32_t a_info, uint32_t a_push, uint32_t a_req,
                                              uint32_t cap0, uint32_t cap1, uint32_t hi, int n,
                                              int H, uint32_t a_tau, uint32_t a_es,
                                              uint32_t a_ord, bool active,
                                              int* __restrict__ starts_out, int* err) {
  static_assert(G == 16 || G == 8, "split evaluator is for 16 or 8 lanes per schedule");
  constexpr uint32_t GM = (1u << G) - 1u;
  const int lane = threadIdx.x & 31;
  const int lg = lane & (G - 1);
  const int gshift = lane & ~(G - 1);
  if (active)
    for (int a = lg; a < n; a += G) sts32(a_es + 4 * a, 0);
  __syncwarp();
  int cmax = 0, hw = 0;
  int act = 0;
  int4 rec = make_int4(0, 0, 0, 0);
  if (active) {
    act = static_cast<int>(lds32(a_ord));
    rec = lds128(a_info + 16 * act);
  }
  for (int pos = 0; pos < n; ++pos) {
    int esv = 0, act_n = 0;
    int4 rec_n = make_int4(0, 0, 0, 0);
    uint32_t r1 = 0;
    if (active) {
      esv = static_cast<int>(lds32(a_es + 4 * act));
      act_n = static_cast<int>(lds32(a_ord + 4 * min(pos + 1, n - 1)));
      rec_n = lds128(a_info + 16 * act_n);
      if (W == 2) r1 = lds32(a_req + 8 * act + 4);
    }
    const int dur = rec.x;
    const uint32_t r0 = static_cast<uint32_t>(rec.y);
    const bool need = dur > 0 && (r0 | r1) != 0;
    bool scanning = need && esv < hw;
    int start = esv;
    if (__any_sync(FULL_MASK, scanning)) {
      const int sh = window_shifts(dur);
      int t0 = esv, carry = 0;
      do {
        const int t = t0 + lg;
        uint32_t w0 = cap0, w1 = cap1;
        if (scanning && t < hw) {
          w0 = lds32(a_tau + 4 * W * t);
          if (W == 2) w1 = lds32(a_tau + 4 * W * t + 4);
        }
        const bool ok = scanning && t < H && fits1(w0, r0, hi) && (W == 1 || fits1(w1, r1, hi));
        const uint32_t m = (__ballot_sync(FULL_MASK, ok) >> gshift) & GM;
        const int z = __ffs(~m) - 1;  // first blocked slot, G when none
        const uint32_t y = window_runs(m, sh);
        const bool fc = carry + z >= dur;
        const int cand = fc ? t0 - carry : t0 + __ffs(y) - 1;
        if (scanning && (fc || y != 0)) {
          start = cand;
          scanning = false;
        } else if (scanning) {
          carry = z == G ? carry + G : __clz(~(m << (32 - G)));
          t0 += G;
          if (t0 >= H) {  // cannot happen for valid instances
            start = H;
            scanning = false;
            if (lg == 0) set_err(err, DE_NO_WINDOW);
          }
        }
      } while (__any_sync(FULL_MASK, scanning));
    }
    if (active) {
      const int fin = start + dur;
      if (need) {
        for (int t = hw + lg; t < start; t += G) {
          sts32(a_tau + 4 * W * t, cap0);
          if (W == 2) sts32(a_tau + 4 * W * t + 4, cap1);
        }
        for (int t = start + lg; t < fin; t += G) {
          const uint32_t adr = a_tau + 4 * W * t;
          const bool old = t < hw;
          sts32(adr, (old ? lds32(adr) : cap0) - r0);
          if (W == 2) sts32(adr + 4, (old ? lds32(adr + 4) : cap1) - r1);
        }
        hw = max(hw, fin);
      }
      cmax = max(cmax, fin);
      const int e0 = rec.z & 0xffff, ecnt = rec.z >> 16;
      for (int e = lg; e < ecnt; e += G) {
        const uint32_t adr = a_es + 4 * lds32(a_push + 4 * (e0 + e));
        if (static_cast<int>(lds32(adr)) < fin) sts32(adr, static_cast<uint32_t>(fin));
      }
      if (starts_out && lg == 0) starts_out[act] = start;
    }
    act = act_n;
    rec = rec_n;
    __syncwarp();
  }
  return cmax;
}

// Eq. 7 (kernels.py:68-78): earliest start the capacity-indexed state allows.
// c: the state, element (k, i) at c[(k*R + i)*SK]
__device__ __forceinline__ int cap_es(const int* c, int SK, const int* dem, const int* cap, int m,
                                      int R) {
  int es_res = 0;
  for (int k = 0; k < m; ++k) {
    const int req = dem[k];
    if (req > 0) es_res = max(es_res, c[(k * R + cap[k] - req) * SK]);
  }
  return es_res;
}

// Alg. 4 (kernels.py:81-110), quirks preserved: consume req*dur effort per
// resource with the shifted-copy buffer cb[i*SK].
__device__ __forceinline__ void cap_commit(int* c, int* cb, int SK, const int* dem,
                                           const int* cap, int m, int R, int start, int dur) {
  for (int k = 0; k < m; ++k) {
    const int req = dem[k];
    int effort = req * dur;
    if (effort <= 0) continue;
    int* ck = c + (k * R) * SK;
    const int capk = cap[k];
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
    const int start = max(es[act * SK], cap_es(c, SK, dem, I.cap, m, R));
    cap_commit(c, cb, SK, dem, I.cap, m, R, start, dur);
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

// ---------------------------------------------------------------------------
// Warp-cooperative capacity-indexed SGS (group 32): one warp per schedule.
// Lane k < m holds resource k's capacity and demand, so Eq. 7's max over the
// resources is one REDUX; Alg. 4 then runs per demanded resource with the
// whole warp in closed form (cap_update_row).  Rows are `rs` words apart
// (rmax rounded up to odd: the m rows fall in distinct banks).
//   scratch: c [m*rs] | es [n]

__host__ __device__ __forceinline__ int cap_row_stride(int rmax) { return rmax | 1; }

__host__ __device__ __forceinline__ int cap_warp_words(int n, int m, int rmax) {
  return m * cap_row_stride(rmax) + n;  // c rows | es (or fin)
}
// the thread-per-schedule evaluator's shared prefix: c rows | es
__host__ __device__ __forceinline__ int cap_prefix_words(int n, int m, int rmax) {
  return m * cap_row_stride(rmax) + n;
}

// Alg. 4 (kernels.py:81-110) on one resource row c[0..capk) (descending),
// whole warp, in closed form -- the same result as the reference's loop for
// every descending row with c[capk - r] <= s (Eq. 7), its quirks included
// (exhaustively fuzzed against the loop: tests/test_gpu_state.py through
// rcpsp_state_op, and the SGS parity tests).  With T = s + d and i0 the first
// entry below T (the leading entries >= T are skipped):
//  * c[i0] <= s: every entry from i0 on is free at s; the loop spends the
//    effort r*d on exactly the r entries i0..i0+r-1, which become T;
//  * else entries i0..i0+r-1 become T with a surplus E = sum (max(c,s) - s)
//    > 0, and the loop then moves the row right by r (entry i takes the old
//    c[i-r]; a run of equal entries it skips keeps the same value), spending
//    c[i-r] - max(c[i], s) per entry while the surplus lasts.  With
//    g(i) = s - max(c_i, s) for i < i0 + r, c_{i-r} - max(c_i, s) after, and
//    S(i) = sum_{j=i0..i} g(j): it stops at the first t >= i0 + r with
//    S(t) >= 0, setting c[t] = max(c_t, s) - S(t-1); the entries after t keep
//    their values (no stop: the shift runs to the end of the row).
// One warp-wide inclusive scan per 32 entries finds t; the reference's loop
// walks the row entry by entry on one thread.
//
// Alg. 4 on a row of at most 32 entries (most rows: capacities <= 32): the
// row is loaded once, one entry per lane, and everything else is register
// work -- i0 is the first lane below T; the fast case (c[i0] <= s) holds iff
// no entry lies in (s, T) (entries before i0 are >= T, the row descends);
// c[i - r] is a shuffle; one warp-wide scan finds the stop t; one predicated
// store per lane writes the row.
__device__ __forceinline__ void cap_update_short(uint32_t a_row, int capk, int r, int s, int d) {
  const int lane = threadIdx.x & 31;
  const int T = s + d;
  const bool in = lane < capk;
  const int w = in ? static_cast<int>(lds32(a_row + 4 * lane)) : 0;
  const int i0 = __ffs(__ballot_sync(FULL_MASK, in && w < T)) - 1;  // >= 0 by Eq. 7
  const bool mid = __any_sync(FULL_MASK, in && w > s && w < T);
  const bool pre = lane >= i0 && lane < i0 + r;
  if (!mid) {  // entries i0..i0+r-1 become T (i0 + r <= capk by Eq. 7)
    __syncwarp();
    sts32_if(pre, a_row + 4 * lane, static_cast<uint32_t>(T));
    __syncwarp();
    return;
  }
  const int o = __shfl_sync(FULL_MASK, w, (lane - r) & 31);  // c[lane - r]
  const bool sh = in && lane >= i0 + r;
  const int f = max(w, s);
  const int g = pre ? s - f : (sh ? o - f : 0);
  int S = g;
#pragma unroll
  for (int q = 1; q < 32; q <<= 1) {
    const int y = __shfl_up_sync(FULL_MASK, S, q);
    if (lane >= q) S += y;
  }
  const unsigned term = __ballot_sync(FULL_MASK, sh && S >= 0);
  const int l = __ffs(term) - 1;  // -1: no stop, the shift runs to the row's end
  const int newt = __shfl_sync(FULL_MASK, f - (S - g), l & 31);
  const int end = term ? l : capk;
  __syncwarp();
  sts32_if(lane >= i0 && (lane < end || lane == l), a_row + 4 * lane,
           static_cast<uint32_t>(lane == l ? newt : (pre ? T : o)));
  __syncwarp();
}

// Alg. 4 on one row in windows of 32 entries aligned at i0 (entry i0 + 32k +
// lane in lane `lane` of window k): window 0 is held in registers, its
// shifted value c[i - r] a shuffle for demands below 32; one warp-wide scan
// per window finds the stop t, carrying the surplus into the next window
// (rows longer than a warp); the writes follow once every read is done --
// the later windows backward (each reads its c[i - r] before its lanes
// write, and no lower window has been written yet), window 0 from registers.
// A/B on B200 (tools/ab_args.sh, profiles/r2/cap_ab.txt): three windows held
// in registers cost spills on the common path; 384 threads per CTA to avoid
// them: -13 %.
__device__ __forceinline__ void cap_update_row(uint32_t a_row, int capk, int r, int s, int d) {
  if (capk <= 32) {
    cap_update_short(a_row, capk, r, s, d);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int T = s + d;
  int i0 = capk, c0 = 0;
  for (int b = 0; b < capk; b += 32) {
    const int i = b + lane;
    const int v = i < capk ? static_cast<int>(lds32(a_row + 4 * i)) : 0;
    const unsigned msk = __ballot_sync(FULL_MASK, i < capk && v < T);
    if (msk) {
      const int l = __ffs(msk) - 1;
      i0 = b + l;
      c0 = __shfl_sync(FULL_MASK, v, l);
      break;
    }
  }
  if (i0 >= capk) return;  // cannot happen: Eq. 7 gives c[capk - r] <= s < T
  if (c0 <= s) {
    __syncwarp();  // every lane's read of the row precedes the writes
    sts32_if(lane < r, a_row + 4 * (i0 + lane), static_cast<uint32_t>(T));
    if (r > 32) {  // (uniform; keeps the loop's trip-count set-up off the common path)
#pragma unroll 1
      for (int j = lane + 32; j < r; j += 32) sts32(a_row + 4 * (i0 + j), static_cast<uint32_t>(T));
    }
    __syncwarp();
    return;
  }
  int t = capk, newt = 0, ov0, b = i0;
  {  // window 0
    const int i = i0 + lane;
    const bool in = i < capk, sh = i >= i0 + r;
    const int w = in ? static_cast<int>(lds32(a_row + 4 * i)) : 0;
    int o;
    if (r < 32)
      o = __shfl_sync(FULL_MASK, w, (lane - r) & 31);
    else
      o = (in && sh) ? static_cast<int>(lds32(a_row + 4 * (i - r))) : 0;
    ov0 = o;
    const int f = max(w, s);
    const int g = in ? (sh ? o - f : s - f) : 0;
    int S = g;
#pragma unroll
    for (int q = 1; q < 32; q <<= 1) {
      const int y = __shfl_up_sync(FULL_MASK, S, q);
      if (lane >= q) S += y;
    }
    const unsigned term = __ballot_sync(FULL_MASK, in && sh && S >= 0);
    if (term) {
      const int l = __ffs(term) - 1;
      t = i0 + l;
      newt = __shfl_sync(FULL_MASK, f - (S - g), l);
    } else if (i0 + 32 < capk) {
      // the surplus outlasts window 0: the next windows, carrying it
      int carry = __shfl_sync(FULL_MASK, S, 31);
      for (b = i0 + 32;; b += 32) {
        const int i = b + lane;
        const bool in = i < capk, sh = i >= i0 + r;
        const int w = in ? static_cast<int>(lds32(a_row + 4 * i)) : 0;
        const int o = (in && sh) ? static_cast<int>(lds32(a_row + 4 * (i - r))) : 0;
        const int f = max(w, s);
        const int g = in ? (sh ? o - f : s - f) : 0;
        int S = g;
#pragma unroll
        for (int q = 1; q < 32; q <<= 1) {
          const int y = __shfl_up_sync(FULL_MASK, S, q);
          if (lane >= q) S += y;
        }
        S += carry;
        const unsigned term = __ballot_sync(FULL_MASK, in && sh && S >= 0);
        if (term) {
          const int l = __ffs(term) - 1;
          t = b + l;
          newt = __shfl_sync(FULL_MASK, f - (S - g), l);
          break;
        }
        if (b + 32 >= capk) break;  // no stop: the shift runs to the row's end
        carry = __shfl_sync(FULL_MASK, S, 31);
      }
    }
  }
  const int end = t < capk ? t : capk;  // [i0, end): T / shifted; t: newt
  __syncwarp();
  for (int bb = b; bb > i0; bb -= 32) {  // the later windows, backward
    const int i = bb + lane;
    const int v = (i < end && i >= i0 + r) ? static_cast<int>(lds32(a_row + 4 * (i - r))) : T;
    __syncwarp();
    if (i < end) sts32(a_row + 4 * i, static_cast<uint32_t>(v));
    if (i == t) sts32(a_row + 4 * i, static_cast<uint32_t>(newt));
    __syncwarp();
  }
  const int i = i0 + lane;
  if (i < end) sts32(a_row + 4 * i, static_cast<uint32_t>(i < i0 + r ? T : ov0));
  if (i == t) sts32(a_row + 4 * i, static_cast<uint32_t>(newt));
  __syncwarp();
}

// Alg. 4 for every resource the activity demands (lane k < m: capacity,
// demand and row offset -- in words from a_c -- of resource k), one after
// another with the whole warp (capacity and demand travel in one shuffle:
// both are below 2^16, a row fits in shared memory).
__device__ __forceinline__ void cap_update_all(uint32_t a_c, int off, int m, int capk, int req,
                                               int start, int dur) {
  const int lane = threadIdx.x & 31;
  unsigned used = __ballot_sync(FULL_MASK, lane < m && req > 0);
  const int cr = capk | (req << 16);
  const uint32_t a_row = a_c + 4 * off;
  while (used) {
    const int k = __ffs(used) - 1;
    used &= used - 1;
    const int x = __shfl_sync(FULL_MASK, cr, k);
    cap_update_row(__shfl_sync(FULL_MASK, a_row, k), x & 0xffff, x >> 16, start, dur);
  }
}

// compact state layout: row k starts at the sum of the capacities before it
// (lane k < m gets its row's offset; S = the sum of all capacities)
__device__ __forceinline__ int cap_row_offset(int capk) {
  const int lane = threadIdx.x & 31;
  int x = capk;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL_MASK, x, o);
    if (lane >= o) x += y;
  }
  return x - capk;
}

// Eq. 7 start (kernels.py:68-78, also for zero durations, as kernels.py:
// 182-186) of an activity whose precedence bound is esv; req: lane k < m gets
// resource k's demand.
// packed: the record's demand word holds every demand as an 8-bit lane (one
// packing word, 8-bit lanes: m <= 4), so no demand load is needed.
__device__ __forceinline__ int cap_start_warp(int act, int esv, uint32_t a_dem, int m, int capk,
                                              int off, uint32_t a_c, int& req,
                                              bool packed = false, uint32_t dword = 0u) {
  const int lane = threadIdx.x & 31;
  int t = 0;
  req = 0;
  if (lane < m) {
    req = packed ? static_cast<int>((dword >> (8 * lane)) & 0xffu)
                 : static_cast<int>(lds32(a_dem + 4 * (act * m + lane)));
    if (req > 0) t = static_cast<int>(lds32(a_c + 4 * (off + capk - req)));
  }
  return max(esv, __reduce_max_sync(FULL_MASK, t));
}

// One activity, push form: start = max(es_prec, Eq. 7), Alg. 4 per resource,
// the finish time pushed to the successors' es.
//   capk: lane k < m holds resource k's capacity (lanes >= m: 0)
__device__ __forceinline__ int cap_step_warp(int act, int dur, int esv, uint32_t a_dem, int m,
                                             int capk, int off, uint32_t a_c, uint32_t a_push,
                                             int e0, int ecnt, uint32_t a_es, int& cmax) {
  const int lane = threadIdx.x & 31;
  int req;
  const int start = cap_start_warp(act, esv, a_dem, m, capk, off, a_c, req);
  if (dur > 0) cap_update_all(a_c, off, m, capk, req, start, dur);
  const int fin = start + dur;
  cmax = max(cmax, fin);
  for (int e = lane; e < ecnt; e += 32) red_max_shared(a_es + 4 * lds32(a_push + 4 * (e0 + e)), fin);
  __syncwarp();
  return start;
}

// Whole schedule of the order at a_ord (one warp); starts_out may be null.
//   a_info: per-activity records (dur, -, push span, -); a_push: push targets
//   scratch: c (compact rows, S = sum of capacities <= m * rs words) | es [n]
//   snap (optional): the state after every k-th position (positions k-1,
//   2k-1, ...), uint16 [n/k][S] at this shared address -- the CAPACITY
//   evaluator starts its moves from them and tests convergence against them
__device__ __forceinline__ int sgs_cap_warp(uint32_t a_info, uint32_t a_push, uint32_t a_dem,
                                            const int* cap, int n, int m, int rs, uint32_t a_scr,
                                            uint32_t a_ord, int* __restrict__ starts_out,
                                            uint32_t a_snap = 0u, int snap_k = 1) {
  const int lane = threadIdx.x & 31;
  const int capk = lane < m ? cap[lane] : 0;
  const int off = cap_row_offset(capk);
  const int S = __shfl_sync(FULL_MASK, off + capk, 31);  // lanes >= m: capk 0
  const uint32_t a_c = a_scr, a_es = a_scr + 4 * m * rs;
  for (int j = lane; j < S; j += 32) sts32(a_c + 4 * j, 0);
  for (int a = lane; a < n; a += 32) sts32(a_es + 4 * a, 0);
  __syncwarp();
  int cmax = 0;
  for (int pos = 0; pos < n; ++pos) {
    const int act = static_cast<int>(lds32(a_ord + 4 * pos));
    const int4 rec = lds128(a_info + 16 * act);
    const int esv = static_cast<int>(lds32(a_es + 4 * act));
    const int s = cap_step_warp(act, rec.x, esv, a_dem, m, capk, off, a_c, a_push,
                                rec.z & 0xffff, rec.z >> 16, a_es, cmax);
    if (starts_out && lane == 0) starts_out[act] = s;
    if (a_snap && pos % snap_k == snap_k - 1)
      for (int j = lane; j < S; j += 32)
        sts16(a_snap + 2 * ((pos / snap_k) * S + j), lds32(a_c + 4 * j));
  }
  __syncwarp();
  return cmax;
}

}  // namespace rt
