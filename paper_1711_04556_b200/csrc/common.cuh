// common.cuh -- shared definitions for the B200 tabu-search kernels.
//
// Device instance encoding ("blob"): one contiguous int32 array per instance,
// produced on the host by paper_1711_04556_b200/device.py:pack_instance from
// the reference's KernelArrays (instance.py:53-80).  The header is 32 words;
// the arrays follow at the recorded offsets.  The kernels stage the arrays a
// CTA needs into shared memory once per launch.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#define FULL_MASK 0xffffffffu

namespace rt {

enum { MODE_CAPACITY = 0, MODE_TIME = 1 };  // kernels.py:22-23

enum BlobField {
  B_MAGIC = 0, B_N = 1, B_M = 2, B_H = 3, B_E = 4, B_W = 5, B_LB = 6, B_RMAX = 7, B_CPM = 8,
  B_LEN = 9, B_NLVL = 10, B_BIG = 11, B_SUMCAP = 12, B_LBRES = 13,
  B_OFF_DUR = 16, B_OFF_DEM = 17, B_OFF_CAP = 18, B_OFF_PPTR = 19, B_OFF_PDAT = 20,
  B_OFF_SPTR = 21, B_OFF_SDAT = 22, B_OFF_REQ = 23, B_OFF_CAPW = 24, B_OFF_LPTR = 25,
  B_OFF_LDAT = 26,
  B_HDR = 32
};
constexpr int BLOB_MAGIC = 0x52435053;  // "RCPS"
// slots past the horizon H + 1 of the prefix-reusing TIME evaluator's profile:
// a scan round starting at t <= H reads up to t + 31
constexpr int TAU_PAD = 32;

// error codes written to the device error word (first error wins)
enum DevErr {
  DE_OK = 0, DE_BAD_BLOB = 1, DE_NO_WINDOW = 2, DE_SMEM = 3, DE_TABU_BAND = 4, DE_CYCLE = 5,
  DE_BAD_MOVE = 6,
  DE_POOL_MIN = 7,  // global best above a pool entry (cooperation.py:76-79 invariant)
  DE_CAP_START = 8  // rcpsp_state_op cap_update below the Eq. 7 bound (see k_state_op)
};

__device__ __forceinline__ void set_err(int* err, int code) {
  if (err) atomicCAS(err, 0, code);
}

// Shared-memory view of one instance.  All arrays are int32 / uint32.
// Per-activity record of the TIME evaluator (one LDS.128 per activity):
//   x = duration, y = packed demand word 0,
//   z = push span: first edge | (edge count << 16) of the activities whose
//       earliest start this one's finish time bounds (successors forward,
//       predecessors for the reversed project),
//   w = window_mask(dur): the low `dur` bits, the run the warp evaluator's
//       window test looks for (the split evaluators derive window_shifts).
struct SInst {
  int n, m, H, e, W, rmax, cpm;
  int big;               // a duration or fan-out > 32 (multi-round paths needed)
  uint32_t hi;           // high bit of every packed resource lane (TIME fits test)
  const int4* info_f;    // [n] forward records
  const int4* info_r;    // [n] reversed-project records
  const int* dur;        // [n]
  const uint32_t* req;   // [n*W] packed per-resource demands (TIME)
  const int* dem;        // [n*m] row-major demands (CAP)
  const int* cap;        // [m]
  const uint32_t* capw;  // [W] packed capacities (TIME "full" slot)
  const int* pptr;       // [n+1]
  const int* pdat;       // [e]
  const int* sptr;       // [n+1]
  const int* sdat;       // [e]
};

__host__ __device__ __forceinline__ int inst_smem_words(int n, int m, int e, int W) {
  return 8 * n + n + n * W + n * m + m + W + 2 * (n + 1) + 2 * e + 32;  // + pdat padding
}

// y &= y >> s_i (i = 1..5) turns a slot mask into "a run of d ones starts
// here" (d <= 32): s_i = min(acc, d - acc), acc += s_i, acc starting at 1.
// Fields are 5 bits wide at bit 5*i (every s_i <= 16); a wrap-mode funnel
// shift uses only the low 5 bits of its amount, so field i is applied as
// shf.r.wrap(y, 0, packed >> 5*i) without masking.
// low `d` bits set (all 32 for d >= 32): the window test of the warp evaluator
__host__ __device__ __forceinline__ uint32_t window_mask(int d) {
  return d >= 32 ? 0xffffffffu : (1u << d) - 1u;
}

__host__ __device__ __forceinline__ int window_shifts(int d) {
  int packed = 0, acc = 1;
  for (int i = 0; i < 5; ++i) {
    const int s = d > acc ? (acc < d - acc ? acc : d - acc) : 0;
    packed |= s << (5 * i);
    acc += s;
  }
  return packed;
}

// Stage a blob into shared memory (all threads of the CTA call this; the
// caller must __syncthreads() afterwards).  Returns the number of words used.
__device__ __forceinline__ int stage_instance(const int* __restrict__ blob, int* smem, SInst& I) {
  I.n = blob[B_N];
  I.m = blob[B_M];
  I.H = blob[B_H];
  I.e = blob[B_E];
  I.W = blob[B_W];
  I.rmax = blob[B_RMAX];
  I.cpm = blob[B_CPM];
  I.big = blob[B_BIG];
  I.hi = blob[B_LB] == 8 ? 0x80808080u : 0x80008000u;
  const int n = I.n, m = I.m, e = I.e, W = I.W;
  int4* inf = reinterpret_cast<int4*>(smem);  // smem base is 16-byte aligned
  {
    const int* bd = blob + blob[B_OFF_DUR];
    const int* br = blob + blob[B_OFF_REQ];
    const int* sp = blob + blob[B_OFF_SPTR];
    const int* pp = blob + blob[B_OFF_PPTR];
    for (int a = threadIdx.x; a < n; a += blockDim.x) {
      const int d = bd[a], r = W ? br[a * W] : 0, sh = static_cast<int>(window_mask(d));
      inf[a] = make_int4(d, r, sp[a] | ((sp[a + 1] - sp[a]) << 16), sh);
      inf[n + a] = make_int4(d, r, pp[a] | ((pp[a + 1] - pp[a]) << 16), sh);
    }
  }
  I.info_f = inf;
  I.info_r = inf + n;
  int* p = smem + 8 * n;
  auto copy = [&](int off, int cnt) -> int* {
    int* dst = p;
    const int* src = blob + off;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) dst[i] = src[i];
    p += cnt;
    return dst;
  };
  I.dur = copy(blob[B_OFF_DUR], n);
  I.req = reinterpret_cast<const uint32_t*>(copy(blob[B_OFF_REQ], n * W));
  I.dem = copy(blob[B_OFF_DEM], n * m);
  I.cap = copy(blob[B_OFF_CAP], m);
  I.capw = reinterpret_cast<const uint32_t*>(copy(blob[B_OFF_CAPW], W));
  I.pptr = copy(blob[B_OFF_PPTR], n + 1);
  I.pdat = copy(blob[B_OFF_PDAT], e);
  // 32 zero entries after the predecessor lists: a warp may read a whole
  // 32-lane window from any span start (lanes past the span read activity 0)
  for (int i = threadIdx.x; i < 32; i += blockDim.x) p[i] = 0;
  p += 32;
  I.sptr = copy(blob[B_OFF_SPTR], n + 1);
  I.sdat = copy(blob[B_OFF_SDAT], e);
  return static_cast<int>(p - smem);
}

__device__ __forceinline__ int align4(int words) { return (words + 3) & ~3; }

// every demand of an activity sits in its record's demand word as an 8-bit
// lane (one packing word of 8-bit lanes, so m <= 4)
__device__ __forceinline__ bool cap_demand_packed(const SInst& I) {
  return I.W == 1 && I.hi == 0x80808080u;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace rt
