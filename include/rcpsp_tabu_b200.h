/*
 * rcpsp_tabu_b200.h -- C ABI of the B200-native parallel tabu search for the
 * RCPSP (drop-in for the hot path of the reference package rcpsp_tabu).
 *
 * The reference's plugin seam is its operator layer `rcpsp_tabu/kernels.py`
 * (backend picked by RCPSP_TABU_BACKEND, kernels.py:25-55): plain functions
 * over caller-owned int32 arrays, mutating outputs in place.  Each entry point
 * below replaces one of those operators (or, for rcpsp_solve, the whole
 * worker/working-set loop of cooperation.orchestrate) with a CUDA launch for
 * sm_100a.  Conventions:
 *   - every pointer is caller-owned DEVICE memory unless stated otherwise;
 *   - every device call is asynchronous on `stream` (a cudaStream_t, NULL =
 *     legacy) and never synchronises: launch sizing uses the instance shape
 *     the caller passes in (RcpspShape, from rcpsp_pack_instance's host blob
 *     via rcpsp_blob_shape), and the kernels check it against the device
 *     blob's header (mismatch -> DE_BAD_BLOB in the err word);
 *   - return 0 on success, <0 on a host-side error; rcpsp_last_error()
 *     returns a thread-local message.  Device-side invariant violations are
 *     written to the caller's `err` word (first error wins, see DevErr in
 *     csrc/common.cuh) and read back only when the caller syncs;
 *   - an instance is a packed int32 "blob" built by rcpsp_pack_instance (host
 *     code, below) from the reference's KernelArrays fields (instance.py:53-80);
 *     the caller copies it to device memory; batches are blobs concatenated
 *     with an int64 offset table.
 * No torch types appear here; the Python host passes tensor data_ptr()s.
 */
#ifndef RCPSP_TABU_B200_H
#define RCPSP_TABU_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RCPSP_ABI_VERSION 8

/* Values of the device error word (the `err` argument / RcpspSolveArgs.err):
 * the first error a kernel hits is kept. */
enum {
    RCPSP_DE_OK = 0,
    RCPSP_DE_BAD_BLOB = 1,    /* blob header does not match RcpspShape           */
    RCPSP_DE_NO_WINDOW = 2,   /* no resource window before the horizon           */
    RCPSP_DE_SMEM = 3,        /* shared-memory plan broken (e.g. no_big violated) */
    RCPSP_DE_TABU_BAND = 4,   /* tabu move outside the delta band                */
    RCPSP_DE_CYCLE = 5,       /* precedence cycle                                */
    RCPSP_DE_BAD_MOVE = 6,    /* malformed move                                  */
    RCPSP_DE_POOL_MIN = 7,    /* global best above a pool entry (cooperation.py:76-79) */
    RCPSP_DE_CAP_START = 8    /* rcpsp_state_op cap_update below the Eq. 7 bound */
};

/* Everything the on-device orchestrate needs (all fields 64-bit so the ctypes
 * mirror in device.py is a flat array).  Sizes: I = instances in the batch,
 * B = workers (CTAs) per instance, F = pool_size, T = tabu_size,
 * n_max = max activities over the batch. */
typedef struct RcpspSolveArgs {
    const int32_t *blob;        /* concatenated instance blobs            */
    const int64_t *blob_off;    /* [I] word offset of each blob           */
    int64_t n_inst;             /* I                                      */
    int64_t n_max;              /* max activities                         */
    int64_t workers;            /* B                                      */
    int64_t pool_size;          /* F                                      */
    int64_t tabu_size;          /* T                                      */
    int64_t delta;              /* swap distance cap                      */
    int64_t phi_steps;          /* diversification swaps                  */
    int64_t phi_max;            /* unimproved reads before diversify      */
    int64_t total_iters;        /* I_total per instance                   */
    int64_t block_iters;        /* ceil(I_total / B) (search.py:39-42)    */
    int64_t epoch_limit;        /* planned-iteration limit of this launch */
    int64_t grant_cap;          /* 0 = uncapped (cooperation.py:123-124)      */
    int64_t collect_trace;      /* 1 = write per-iteration traces         */
    /* working set (cooperation.py:52-80, 253-273), per instance */
    int32_t *ws_lock;           /* [I]                                    */
    int64_t *ws_hdr;            /* [I*16] see WS_* in kernels.cu          */
    int32_t *ent_order;         /* [I*F*n_max]                            */
    int32_t *ent_cmax;          /* [I*F]                                  */
    uint32_t *ent_tabu;         /* [I*F*T] packed (u<<16)|v, 0 = empty    */
    int32_t *ent_head;          /* [I*F]                                  */
    int64_t *ent_ic;            /* [I*F] iterations invested              */
    int64_t *ent_reads;         /* [I*F] reads without improvement        */
    int32_t *ws_best_order;     /* [I*n_max]                              */
    /* workers (search.py:107-132), per instance x worker */
    uint64_t *w_rng;            /* [I*B*6] PCG64 state words              */
    int64_t *w_stats;           /* [I*B*16] see WK_* in kernels.cu        */
    int32_t *w_trace;           /* [I*B*trace_cap] or NULL                */
    int64_t trace_cap;
    int32_t *w_chunks;          /* [I*B*chunk_cap] chunk lengths or NULL  */
    int64_t chunk_cap;
    /* per-CTA scratch */
    uint32_t *moves_buf;        /* [grid*nbhd_max]                        */
    int32_t *cmax_buf;          /* [grid*nbhd_max]                        */
    int64_t nbhd_max;
    int32_t *err;               /* device error word                      */
    /* shape maxima of the launch group (shared-memory sizing) */
    int64_t h_max, e_max, m_max, rmax_max, words;
    int64_t group;              /* TIME lanes per schedule: 32, 16 or 8   */
    int64_t threads;            /* threads per CTA (0 = auto: 2 CTAs/SM)  */
    int64_t steal;              /* 1 = a worker whose instance has spent its
                                 * budget moves on to instances with budget
                                 * left (balances the batch tail; B > 1) */
    int64_t full_sgs;           /* 1 = evaluate every swap by a full SGS;
                                 * 0 (default) = group 32 reuses the base
                                 * order's schedule prefix (same makespans) */
    int64_t cluster;            /* CTAs per worker (thread-block cluster,
                                 * 1..8): the leader CTA runs the search, the
                                 * others evaluate neighbourhood moves over
                                 * distributed shared memory (prefix-reusing
                                 * evaluators; others run with 1) */
    int64_t time_budget_ns;     /* > 0: wall-clock budget of the launch on the
                                 * device clock (%globaltimer): no new grants
                                 * and no further iterations once it is spent */
    int64_t *t0_ns;             /* [1] launch start (atomicMin of every CTA's
                                 * first clock read); host sets INT64_MAX */
    int64_t no_big;             /* 1 = the caller guarantees that no instance
                                 * of the launch has a duration or a fan-out/
                                 * -in above 32 (RcpspShape.big == 0): the
                                 * TIME evaluator's shared-memory plan then
                                 * leaves out its undo log.  0 (the zero-
                                 * initialised default) is always safe.  A
                                 * violated guarantee is caught on the device
                                 * (DE_SMEM) instead of corrupting memory. */
    int64_t sumcap_max;         /* max over the instances of the sum of the
                                 * capacities (RcpspShape.sumcap): sizes the
                                 * CAPACITY evaluator's state snapshots (0 =
                                 * no snapshots, no convergence exit) */
    int64_t prof_slots;         /* TIME: per-warp profile slots sized by a
                                 * makespan bound (0 = the horizon); used when
                                 * it keeps more warps resident and no_big
                                 * holds (< 0: -prof_slots slots, always --
                                 * tests) -- a move that books past it is
                                 * evaluated exactly on a full-horizon
                                 * region instead */
    int32_t *ent_lock;          /* [I*F] per-entry locks (zeroed; ABI 8): the
                                 * exchange locks one entry at a time, and
                                 * ws_lock guards only the global best */
    /* live elite exchange between independent populations over peer memory
     * (ABI 8; all NULL / 0 = off).  Each population publishes its
     * per-instance global best in its outbox (seqlock: seq odd while being
     * written) and, every poll_every exchanges of a worker, reads the other
     * populations' outboxes directly (CUDA IPC mappings: P2P loads over
     * NVLink/NVSwitch), importing the best new foreign elite into the worst
     * pool entry -- no host round trip, no pause of the search. */
    int32_t *outbox;            /* [I * RCPSP_OUTBOX_WORDS(n_max)] own, or NULL */
    const int64_t *peers;       /* [n_peers] device addresses of peer outboxes */
    int64_t n_peers;            /* <= 32 */
    int32_t *peer_seen;         /* [I * n_peers] last sequence imported per peer */
    int64_t poll_every;         /* exchanges between polls (>= 1) */
    int64_t *peer_stats;        /* [4]: imports, publishes, polls, torn reads */
} RcpspSolveArgs;

/* words of one instance's outbox: seq, cmax, 2 reserved, order[n_max] */
#define RCPSP_OUTBOX_WORDS(n_max) (4 + (n_max))

/* Shape of one packed instance (the blob header), what the host needs to size
 * a launch without reading device memory. */
typedef struct RcpspShape {
    int32_t n;          /* activities incl. the two dummies                  */
    int32_t m;          /* renewable resources                               */
    int32_t horizon;    /* sum of durations (TIME profile length - 1)        */
    int32_t edges;      /* precedence edges                                  */
    int32_t words;      /* TIME packing: words per slot (0 = CAPACITY only)  */
    int32_t lane_bits;  /* 8 or 16 (0 with words == 0)                       */
    int32_t rmax;       /* max capacity (>= 1)                               */
    int32_t cpm;        /* critical-path length (the search's floor)         */
    int32_t len;        /* blob length in int32 words                        */
    int32_t big;        /* a duration or fan-out/-in above 32                */
    int32_t sumcap;     /* sum of the capacities (CAPACITY state words)      */
} RcpspShape;

int rcpsp_abi_version(void);
const char *rcpsp_last_error(void);

/* ---- host-side instance packing (no CUDA calls; usable without a GPU) ----
 * Inputs are the reference's KernelArrays fields (instance.py:53-80):
 * durations [n], demands [n*m] row-major, capacities [m], predecessor and
 * successor CSR (ptr [n+1], dat [e], ids ascending per activity), horizon =
 * sum of durations.  Every pointer is HOST memory.
 * rcpsp_blob_words: validated size of the blob in int32 words, or -1.
 * rcpsp_pack_instance: writes the blob (csrc/common.cuh layout) into `blob`
 *   (blob_words >= rcpsp_blob_words); 0 or -1 (rcpsp_pack_last_error()).
 *   Replaces the reference's ProjectInstance -> KernelArrays step
 *   (instance.py:95-120) as the input of every device entry point below;
 *   the levels (instance.py:396-415) and the critical path (instance.py:
 *   374-388) are computed here.
 * rcpsp_blob_shape: the shape of a packed (host) blob, for the entry points. */
int64_t rcpsp_blob_words(const int32_t *dur, const int32_t *dem, const int32_t *cap, int n, int m,
                         const int32_t *pred_ptr, const int32_t *pred_dat,
                         const int32_t *succ_ptr, const int32_t *succ_dat, int32_t horizon);
int rcpsp_pack_instance(const int32_t *dur, const int32_t *dem, const int32_t *cap, int n, int m,
                        const int32_t *pred_ptr, const int32_t *pred_dat,
                        const int32_t *succ_ptr, const int32_t *succ_dat, int32_t horizon,
                        int32_t *blob, int64_t blob_words);
int rcpsp_blob_shape(const int32_t *blob, RcpspShape *shape);
const char *rcpsp_pack_last_error(void);

/* Device properties used for launch sizing: SM count, opt-in smem/CTA. */
int rcpsp_device_info(int *sm_count, int *smem_optin, int *cc_major, int *cc_minor);

/* Batch of evaluate_order calls (kernels.py:152-194; evaluator.evaluate
 * evaluator.py:128-144).  orders: [B*n] precedence-feasible permutations.
 * reverse != 0 evaluates the time-reversed project (successor lists used as
 * predecessor lists, evaluator.py:234-242).  cmax: [B]; starts: [B*n] or
 * NULL.  group: TIME lanes per schedule (32/16/8). */
int rcpsp_eval_batch(const int32_t *blob, const RcpspShape *shape, int mode, const int32_t *orders, int batch,
                     int reverse, int32_t *cmax, int32_t *starts, int group, int32_t *err,
                     void *stream);

/* filter_moves (kernels.py:218-255) over the reduced neighbourhood with
 * distance cap `delta` for a batch of orders: out_moves [batch*nbhd_cap]
 * packed (u<<16)|v in lexicographic order, out_count [batch]. */
int rcpsp_filter_batch(const int32_t *blob, const RcpspShape *shape, const int32_t *orders,
                       int batch, int delta, uint32_t *out_moves, int nbhd_cap,
                       int32_t *out_count, int32_t *err, void *stream);

/* run_chunk (kernels.py:316-385) for `batch` independent searches on one
 * instance; one CTA each.  In/out: orders [batch*n], tabu [batch*T] packed,
 * heads [batch].  In: per-search budget/adopted/start/best_known [batch],
 * floor.  Out: best_orders [batch*n], trace [batch*trace_cap] (or NULL),
 * stats [batch*8] = (iters, evals, improved, local_best, cur, head, forced, 0)
 * -- the reference's 7-tuple.  Tabu counters are rebuilt from the list
 * (tabu.py:52-60); list entries must satisfy v-u <= delta. */
int rcpsp_run_chunk_batch(const int32_t *blob, const RcpspShape *shape, int mode, int delta, int tabu_size, int batch,
                          int32_t *orders, uint32_t *tabu, int32_t *heads, const int32_t *budget,
                          const int32_t *adopted, const int32_t *start_cmax,
                          const int32_t *best_known, int floor_cmax, int32_t *best_orders,
                          int32_t *trace, int trace_cap, int64_t *stats, uint32_t *moves_buf,
                          int32_t *cmax_buf, int nbhd_max, int group, int threads, int32_t *err,
                          void *stream);

/* initialize_working_set (cooperation.py:138-160) for the instances listed in
 * inst_ids: level-shuffled orders from the pool PCG64 state (one state per
 * instance, 6 words each: default_rng(seed)), forward-backward improvement
 * of even entries (evaluator.py:207-266), evaluation, global best. */
int rcpsp_pool_init(const RcpspSolveArgs *args, const int32_t *inst_ids, int n_ids, int mode,
                    const uint64_t *pool_rng, void *stream);

/* The search proper (search.run_worker + cooperation.exchange +
 * Worker.run_adopted): one persistent CTA per (instance, worker), the working
 * set in HBM behind a per-instance lock, until the planned iterations reach
 * args->epoch_limit or the global best hits the critical path. */
int rcpsp_solve(const RcpspSolveArgs *args, const int32_t *inst_ids, int n_ids, int mode,
                void *stream);

/* Elite exchange between independent populations (multi-GPU, host passes the
 * all-gathered elites): for every instance, each received elite order whose
 * makespan beats the worst pool entry replaces it (tabu list cleared, IC and
 * reads reset); the global best follows.  elites: [n_src*I*n_max] orders,
 * elite_cmax [n_src*I]. */
int rcpsp_merge_elites(const RcpspSolveArgs *args, const int32_t *elites,
                       const int32_t *elite_cmax, int n_src, void *stream);

/* Outboxes of the live exchange: cudaMalloc'd (the IPC handle of an
 * allocation names its base), zeroed; handle: 64 bytes (cudaIpcMemHandle_t)
 * for the peers, which map it with rcpsp_outbox_open (P2P enabled lazily). */
int rcpsp_outbox_alloc(int64_t bytes, void **dev_ptr, void *handle);
int rcpsp_outbox_open(const void *handle, void **dev_ptr);
int rcpsp_outbox_close(void *dev_ptr);
int rcpsp_outbox_free(void *dev_ptr);
int rcpsp_outbox_reset(void *dev_ptr, int64_t bytes, void *stream);  /* zero, async */

/* Export each instance's global best (order, cmax) into [I*n_max] / [I]. */
int rcpsp_export_elites(const RcpspSolveArgs *args, int32_t *elites, int32_t *elite_cmax,
                        void *stream);

/* diversify (search.py:77-94) for a batch of orders with per-order PCG64
 * states (advanced in place). */
int rcpsp_diversify_batch(const int32_t *blob, const RcpspShape *shape, int32_t *orders,
                          int batch, int phi_steps, uint64_t *rng, int32_t *err, void *stream);

/* Single-step resource-state operations on the reference's state layouts
 * (kernels.py:68-146 via evaluator.py:69-107): op 0 = cap_earliest_start,
 * 1 = cap_update (arg = start), 2 = time_earliest_start (arg = es_prec),
 * 3 = time_update (arg = start).  state: CAP int32 [m][R_max], TIME int32
 * [m][H+1] (updated in place); out[0] receives the earliest start.  A
 * cap_update start below the activity's Eq. 7 bound (cap_earliest_start) is
 * refused with error word 8 and the state left as it was. */
int rcpsp_state_op(const int32_t *blob, const RcpspShape *shape, int op, int32_t *state, int act, int arg, int32_t *out,
                   int32_t *err, void *stream);

/* Parity probes of the device RNG and Eq. 8 (assigned_iterations,
 * cooperation.py:39-49). ops: [k*2] (kind, n) with kind 0 = integers(n),
 * 1 = permutation(arange(n)); out receives the draws back to back. */
int rcpsp_rng_probe(uint64_t *state, const int32_t *ops, int k, int32_t *out, void *stream);
/* Shared-memory bandwidth microbenchmark (the roofline denominator of the
 * on-chip-bound search kernel): blocks x threads stream iters x 64 bytes each
 * out of a 32 KB shared array; the caller times it with CUDA events. */
int rcpsp_smem_probe(int blocks, int threads, int iters, int32_t *sink, void *stream);
int rcpsp_eq8_probe(const int64_t *quad /*[k*4] cmax, ic, block_iters, best*/, int k,
                    int64_t *out, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* RCPSP_TABU_B200_H */
