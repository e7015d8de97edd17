// pack.cpp -- host-side instance packer of the C ABI (rcpsp_blob_words,
// rcpsp_pack_instance, rcpsp_blob_shape).  Plain C++, no CUDA: it turns the
// reference's KernelArrays fields (instance.py:53-80 -- durations, demands
// [N x M] row-major, capacities, predecessor / successor CSR with sorted ids,
// horizon = sum of durations) into the int32 blob every kernel stages
// (layout: csrc/common.cuh, BlobField):
//
//   header[32] | dur[n] | dem[n*m] | cap[m] | pred_ptr[n+1] | pred_dat[e]
//   | succ_ptr[n+1] | succ_dat[e] | req[n*W] | capw[W] | lvl_ptr[L+1] | lvl_dat[n]
//
// Derived fields computed here: the TIME packing (W words of 8- or 16-bit
// lanes per slot; W = 0 when the capacities do not pack -- such blobs run in
// CAPACITY mode only), the critical-path length (instance.py:374-388, the
// sink's longest duration-weighted distance), the precedence levels
// (instance.py:396-415: longest unit-weight distance from any root, ids
// ascending inside a level), the B_BIG flag (a duration, fan-out or --
// except into a zero-duration sink -- fan-in above 32) and B_SUMCAP (the sum
// of the capacities: the compact capacity-indexed state's size), B_LBRES (the
// energy bound max_k ceil(sum_i d_i r_ik / R_k) of the makespan).
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rcpsp_tabu_b200.h"

namespace {

constexpr int kHdr = 32;
constexpr int kMagic = 0x52435053;   // "RCPS"
constexpr int kKeyLimit = 1 << 16;   // selection key packs (C_max << 16) | rank

enum {
  B_MAGIC = 0, B_N = 1, B_M = 2, B_H = 3, B_E = 4, B_W = 5, B_LB = 6, B_RMAX = 7, B_CPM = 8,
  B_LEN = 9, B_NLVL = 10, B_BIG = 11, B_SUMCAP = 12, B_LBRES = 13,
  B_OFF_DUR = 16, B_OFF_DEM, B_OFF_CAP, B_OFF_PPTR, B_OFF_PDAT, B_OFF_SPTR, B_OFF_SDAT,
  B_OFF_REQ, B_OFF_CAPW, B_OFF_LPTR, B_OFF_LDAT
};

thread_local std::string g_pack_err;

int pack_fail(const std::string& msg) {
  g_pack_err = msg;
  return -1;
}

struct Derived {
  int lane_bits = 8, words = 1, rmax = 1, cpm = 0, big = 0;
  std::vector<int32_t> depth;  // level of each activity
  int n_levels = 0;
};

// Validates the arrays and computes everything the header needs.
int derive(const int32_t* dur, const int32_t* dem, const int32_t* cap, int n, int m,
           const int32_t* pred_ptr, const int32_t* pred_dat, const int32_t* succ_ptr,
           const int32_t* succ_dat, int32_t horizon, Derived& d) {
  if (n < 1) return pack_fail("an instance needs at least one activity");
  if (m < 0) return pack_fail("negative resource count");
  if (n >= kKeyLimit) return pack_fail(std::to_string(n) + " activities >= 65536");
  if (horizon < 0 || horizon >= kKeyLimit - 1)
    return pack_fail("horizon " + std::to_string(horizon) + " outside [0, 65535)");
  if (pred_ptr[0] != 0 || succ_ptr[0] != 0) return pack_fail("CSR pointers must start at 0");
  const int e = pred_ptr[n];
  if (succ_ptr[n] != e) return pack_fail("predecessor and successor lists differ in size");
  for (int i = 0; i < n; ++i) {
    if (dur[i] < 0) return pack_fail("negative duration");
    if (pred_ptr[i + 1] < pred_ptr[i] || succ_ptr[i + 1] < succ_ptr[i])
      return pack_fail("CSR pointers must not decrease");
  }
  for (int k = 0; k < e; ++k)
    if (pred_dat[k] < 0 || pred_dat[k] >= n || succ_dat[k] < 0 || succ_dat[k] >= n)
      return pack_fail("edge endpoint out of range");
  int cmax = 0;
  for (int k = 0; k < m; ++k) {
    if (cap[k] < 0) return pack_fail("negative capacity");
    cmax = cap[k] > cmax ? cap[k] : cmax;
  }
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < m; ++k) {
      const int r = dem[static_cast<size_t>(i) * m + k];
      if (r < 0) return pack_fail("negative demand");
      if (r > cap[k])
        return pack_fail("activity " + std::to_string(i) + " demands " + std::to_string(r) +
                         " of resource " + std::to_string(k) + " with capacity " +
                         std::to_string(cap[k]));
    }
  // TIME packing: every resource of a slot in one (or two) words
  if (m == 0) {
    d.lane_bits = 8;
    d.words = 1;
  } else if (cmax <= 32767) {
    d.lane_bits = cmax <= 127 ? 8 : 16;
    const int lanes = 32 / d.lane_bits;
    d.words = (m + lanes - 1) / lanes;
    if (d.words > 2) d.words = 0;  // no TIME packing: CAPACITY mode only
  } else {
    d.words = 0;
  }
  if (d.words == 0) d.lane_bits = 0;
  d.rmax = m && cmax > 0 ? cmax : 1;
  // Kahn over the successor lists: critical path and unit-weight levels
  std::vector<int> indeg(n), stack, dist(n, 0);
  d.depth.assign(n, 0);
  for (int i = 0; i < n; ++i) indeg[i] = pred_ptr[i + 1] - pred_ptr[i];
  for (int i = 0; i < n; ++i)
    if (indeg[i] == 0) stack.push_back(i);
  int seen = 0;
  while (!stack.empty()) {
    const int i = stack.back();
    stack.pop_back();
    ++seen;
    for (int k = succ_ptr[i]; k < succ_ptr[i + 1]; ++k) {
      const int j = succ_dat[k];
      if (dist[i] + dur[i] > dist[j]) dist[j] = dist[i] + dur[i];
      if (d.depth[i] + 1 > d.depth[j]) d.depth[j] = d.depth[i] + 1;
      if (--indeg[j] == 0) stack.push_back(j);
    }
  }
  if (seen != n) return pack_fail("precedence graph has a cycle");
  d.cpm = dist[n - 1];
  int maxd = 0;
  for (int i = 0; i < n; ++i) maxd = d.depth[i] > maxd ? d.depth[i] : maxd;
  d.n_levels = maxd + 1;
  // multi-round device paths are needed only past one warp (32)
  const bool sink_free = dur[n - 1] == 0;
  int fan = 0, dmax = 0;
  for (int i = 0; i < n; ++i) {
    const int fo = succ_ptr[i + 1] - succ_ptr[i];
    const int fi = (sink_free && i == n - 1) ? 0 : pred_ptr[i + 1] - pred_ptr[i];
    fan = fo > fan ? fo : fan;
    fan = fi > fan ? fi : fan;
    dmax = dur[i] > dmax ? dur[i] : dmax;
  }
  d.big = (dmax > 32 || fan > 32) ? 1 : 0;
  return 0;
}

int64_t words_for(int n, int m, int e, int W, int n_levels) {
  return static_cast<int64_t>(kHdr) + n + static_cast<int64_t>(n) * m + m + 2 * (n + 1) + 2 * e +
         static_cast<int64_t>(n) * W + W + (n_levels + 1) + n;
}

}  // namespace

extern "C" {

const char* rcpsp_pack_last_error(void) { return g_pack_err.c_str(); }

int64_t rcpsp_blob_words(const int32_t* dur, const int32_t* dem, const int32_t* cap, int n, int m,
                         const int32_t* pred_ptr, const int32_t* pred_dat,
                         const int32_t* succ_ptr, const int32_t* succ_dat, int32_t horizon) {
  Derived d;
  if (derive(dur, dem, cap, n, m, pred_ptr, pred_dat, succ_ptr, succ_dat, horizon, d)) return -1;
  return words_for(n, m, pred_ptr[n], d.words, d.n_levels);
}

int rcpsp_pack_instance(const int32_t* dur, const int32_t* dem, const int32_t* cap, int n, int m,
                        const int32_t* pred_ptr, const int32_t* pred_dat, const int32_t* succ_ptr,
                        const int32_t* succ_dat, int32_t horizon, int32_t* blob,
                        int64_t blob_words) {
  Derived d;
  if (derive(dur, dem, cap, n, m, pred_ptr, pred_dat, succ_ptr, succ_dat, horizon, d)) return -1;
  const int e = pred_ptr[n], W = d.words;
  const int64_t need = words_for(n, m, e, W, d.n_levels);
  if (blob_words < need)
    return pack_fail("blob buffer of " + std::to_string(blob_words) + " words < " +
                     std::to_string(need));
  std::memset(blob, 0, sizeof(int32_t) * kHdr);
  int64_t off = kHdr;
  auto put = [&](int slot, const int32_t* src, int64_t cnt) {
    blob[slot] = static_cast<int32_t>(off);
    if (src) std::memcpy(blob + off, src, sizeof(int32_t) * cnt);
    const int64_t at = off;
    off += cnt;
    return blob + at;
  };
  put(B_OFF_DUR, dur, n);
  put(B_OFF_DEM, dem, static_cast<int64_t>(n) * m);
  put(B_OFF_CAP, cap, m);
  put(B_OFF_PPTR, pred_ptr, n + 1);
  put(B_OFF_PDAT, pred_dat, e);
  put(B_OFF_SPTR, succ_ptr, n + 1);
  put(B_OFF_SDAT, succ_dat, e);
  uint32_t* req = reinterpret_cast<uint32_t*>(put(B_OFF_REQ, nullptr, static_cast<int64_t>(n) * W));
  uint32_t* capw = reinterpret_cast<uint32_t*>(put(B_OFF_CAPW, nullptr, W));
  if (W > 0) {
    const int lb = d.lane_bits, lanes = 32 / lb;
    std::memset(req, 0, sizeof(uint32_t) * n * W);
    std::memset(capw, 0, sizeof(uint32_t) * W);
    for (int k = 0; k < m; ++k) {
      const int w = k / lanes, sh = (k % lanes) * lb;
      capw[w] |= static_cast<uint32_t>(cap[k]) << sh;
      for (int i = 0; i < n; ++i)
        req[static_cast<size_t>(i) * W + w] |= static_cast<uint32_t>(dem[static_cast<size_t>(i) * m + k]) << sh;
    }
  }
  // levels: counting sort by depth, ids ascending inside a level
  int32_t* lptr = put(B_OFF_LPTR, nullptr, d.n_levels + 1);
  int32_t* ldat = put(B_OFF_LDAT, nullptr, n);
  std::vector<int> fill(d.n_levels + 1, 0);
  for (int i = 0; i < n; ++i) ++fill[d.depth[i] + 1];
  for (int l = 0; l < d.n_levels; ++l) fill[l + 1] += fill[l];
  for (int l = 0; l <= d.n_levels; ++l) lptr[l] = fill[l];
  for (int i = 0; i < n; ++i) ldat[fill[d.depth[i]]++] = i;
  blob[B_MAGIC] = kMagic;
  blob[B_N] = n;
  blob[B_M] = m;
  blob[B_H] = horizon;
  blob[B_E] = e;
  blob[B_W] = W;
  blob[B_LB] = d.lane_bits;
  blob[B_RMAX] = d.rmax;
  blob[B_CPM] = d.cpm;
  blob[B_LEN] = static_cast<int32_t>(off);
  blob[B_NLVL] = d.n_levels;
  blob[B_BIG] = d.big;
  int sumcap = 0;
  for (int k = 0; k < m; ++k) sumcap += cap[k];
  blob[B_SUMCAP] = sumcap;
  // resource (energy) lower bound of the makespan: max_k ceil(sum_i d_i r_ik / R_k)
  long long lbres = 0;
  for (int k = 0; k < m; ++k) {
    if (cap[k] <= 0) continue;
    long long e = 0;
    for (int i = 0; i < n; ++i) e += static_cast<long long>(dur[i]) * dem[static_cast<size_t>(i) * m + k];
    const long long b = (e + cap[k] - 1) / cap[k];
    lbres = b > lbres ? b : lbres;
  }
  blob[B_LBRES] = static_cast<int32_t>(lbres);
  return 0;
}

int rcpsp_blob_shape(const int32_t* blob, RcpspShape* shape) {
  if (blob == nullptr || shape == nullptr) return pack_fail("null blob or shape");
  if (blob[B_MAGIC] != kMagic) return pack_fail("bad instance blob (magic)");
  shape->n = blob[B_N];
  shape->m = blob[B_M];
  shape->horizon = blob[B_H];
  shape->edges = blob[B_E];
  shape->words = blob[B_W];
  shape->lane_bits = blob[B_LB];
  shape->rmax = blob[B_RMAX];
  shape->cpm = blob[B_CPM];
  shape->len = blob[B_LEN];
  shape->big = blob[B_BIG];
  shape->sumcap = blob[B_SUMCAP];
  return 0;
}

}  // extern "C"
