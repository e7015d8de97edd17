/* c_abi_eval.c -- the C ABI without the Python package: pack an instance on
 * the host (rcpsp_pack_instance), copy it to the GPU, evaluate orders
 * (rcpsp_eval_batch) and run one tabu chunk (rcpsp_run_chunk_batch).
 *
 * The instance is the reference's 12-activity worked example
 * (pkg/tests/conftest.py:17-55): the order below has makespan 22 in TIME
 * mode with starts {0,0,4,4,7,12,9,12,20,15,16,22} (test_evaluator.py:196-201).
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_abi_eval.c -o /tmp/c_abi_eval \
 *       -L paper_1711_04556_b200/_lib -lb200tabu -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1711_04556_b200/_lib -Wl,-rpath,/usr/local/cuda/lib64
 *   /tmp/c_abi_eval          # prints "cmax 22 ..." and exits 0 on success
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "rcpsp_tabu_b200.h"

#define N 12
#define M 2

static int check(int rc, const char* what) {
  if (rc != 0) {
    fprintf(stderr, "%s failed: %s\n", what, rcpsp_last_error());
    exit(1);
  }
  return 0;
}

int main(void) {
  /* example12: durations, two resources of capacity 6, demands, successors */
  const int32_t dur[N] = {0, 4, 3, 5, 5, 3, 2, 4, 2, 3, 4, 0};
  const int32_t dem[N * M] = {0, 0, 5, 3, 2, 1, 3, 2, 2, 3, 3, 4,
                              4, 1, 2, 2, 4, 5, 1, 2, 2, 2, 0, 0};
  const int32_t cap[M] = {6, 6};
  const int succ[N][3] = {{1, 2, -1}, {3, 6, -1}, {4, 5, -1}, {5, 10, -1}, {7, -1, -1},
                          {8, 9, -1}, {7, 9, -1}, {8, 10, -1}, {11, -1, -1},
                          {11, -1, -1}, {11, -1, -1}, {-1, -1, -1}};
  int32_t sptr[N + 1] = {0}, sdat[32], pptr[N + 1] = {0}, pdat[32], cnt[N] = {0};
  int e = 0, horizon = 0;
  for (int i = 0; i < N; ++i) {
    horizon += dur[i];
    for (int k = 0; k < 3 && succ[i][k] >= 0; ++k) {
      sdat[e++] = succ[i][k];
      cnt[succ[i][k]]++;
    }
    sptr[i + 1] = e;
  }
  for (int i = 0; i < N; ++i) pptr[i + 1] = pptr[i] + cnt[i];
  {
    int fill[N];
    memcpy(fill, pptr, sizeof(fill));
    for (int i = 0; i < N; ++i)  /* predecessor ids ascending: scan tails in order */
      for (int k = sptr[i]; k < sptr[i + 1]; ++k) pdat[fill[sdat[k]]++] = i;
  }
  const int64_t words = rcpsp_blob_words(dur, dem, cap, N, M, pptr, pdat, sptr, sdat, horizon);
  if (words < 0) {
    fprintf(stderr, "pack: %s\n", rcpsp_pack_last_error());
    return 1;
  }
  int32_t* blob = (int32_t*)malloc(sizeof(int32_t) * words);
  if (rcpsp_pack_instance(dur, dem, cap, N, M, pptr, pdat, sptr, sdat, horizon, blob, words)) {
    fprintf(stderr, "pack: %s\n", rcpsp_pack_last_error());
    return 1;
  }
  RcpspShape shape;
  if (rcpsp_blob_shape(blob, &shape)) return 1;
  printf("packed %lld words: n %d m %d horizon %d cpm %d words/slot %d\n", (long long)words,
         shape.n, shape.m, shape.horizon, shape.cpm, shape.words);

  const int32_t order[N] = {0, 1, 2, 3, 4, 6, 5, 7, 9, 10, 8, 11};
  const int32_t want_starts[N] = {0, 0, 4, 4, 7, 12, 9, 12, 20, 15, 16, 22};
  int32_t *d_blob, *d_order, *d_cmax, *d_starts, *d_err;
  cudaMalloc((void**)&d_blob, sizeof(int32_t) * words);
  cudaMalloc((void**)&d_order, sizeof(order));
  cudaMalloc((void**)&d_cmax, sizeof(int32_t));
  cudaMalloc((void**)&d_starts, sizeof(int32_t) * N);
  cudaMalloc((void**)&d_err, sizeof(int32_t));
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaMemcpyAsync(d_blob, blob, sizeof(int32_t) * words, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_order, order, sizeof(order), cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(d_err, 0, sizeof(int32_t), s);
  check(rcpsp_eval_batch(d_blob, &shape, 1 /* TIME */, d_order, 1, 0, d_cmax, d_starts, 32,
                         d_err, s), "rcpsp_eval_batch");
  int32_t cmax = 0, starts[N], err = 0;
  cudaMemcpyAsync(&cmax, d_cmax, sizeof(cmax), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(starts, d_starts, sizeof(starts), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&err, d_err, sizeof(err), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  int ok = cmax == 22 && err == 0 && memcmp(starts, want_starts, sizeof(starts)) == 0;
  printf("cmax %d err %d starts", cmax, err);
  for (int i = 0; i < N; ++i) printf(" %d", starts[i]);
  printf(" -> %s\n", ok ? "ok" : "MISMATCH");

  /* one run_chunk of 20 iterations from the same order (kernels.py:316-385) */
  const int T = 8, budget = 20;
  uint32_t *d_tabu, *d_moves;
  int32_t *d_head, *d_vec, *d_best, *d_trace, *d_cbuf;
  int64_t* d_stats;
  const int nb = 45;  /* neighbourhood size for N = 12, delta = 30 */
  cudaMalloc((void**)&d_tabu, sizeof(uint32_t) * T);
  cudaMalloc((void**)&d_head, sizeof(int32_t));
  cudaMalloc((void**)&d_vec, sizeof(int32_t) * 4);
  cudaMalloc((void**)&d_best, sizeof(int32_t) * N);
  cudaMalloc((void**)&d_trace, sizeof(int32_t) * budget);
  cudaMalloc((void**)&d_stats, sizeof(int64_t) * 8);
  cudaMalloc((void**)&d_moves, sizeof(uint32_t) * nb);
  cudaMalloc((void**)&d_cbuf, sizeof(int32_t) * nb);
  const int32_t vec[4] = {budget, 22, 22, 22};  /* budget, adopted, start, best-known */
  cudaMemsetAsync(d_tabu, 0, sizeof(uint32_t) * T, s);
  cudaMemsetAsync(d_head, 0, sizeof(int32_t), s);
  cudaMemcpyAsync(d_vec, vec, sizeof(vec), cudaMemcpyHostToDevice, s);
  check(rcpsp_run_chunk_batch(d_blob, &shape, 1, 30, T, 1, d_order, d_tabu, d_head, d_vec,
                              d_vec + 1, d_vec + 2, d_vec + 3, shape.cpm, d_best, d_trace,
                              budget, d_stats, d_moves, d_cbuf, nb, 32, 256, d_err, s),
        "rcpsp_run_chunk_batch");
  int64_t stats[8];
  cudaMemcpyAsync(stats, d_stats, sizeof(stats), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&err, d_err, sizeof(err), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  printf("run_chunk: iters %lld evals %lld local_best %lld err %d\n", (long long)stats[0],
         (long long)stats[1], (long long)stats[3], err);
  ok = ok && err == 0 && stats[3] >= shape.cpm && stats[3] <= 22;
  free(blob);
  return ok ? 0 : 2;
}
