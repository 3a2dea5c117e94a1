/*
 * include/acs_gpu.h -- the drop-in C-ABI of the B200 ACS hot path.
 *
 * The reference (arXiv 1605.02669 artifact, /root/reference) exposes its path
 * as a C++ library API: the instance layer in proj/include/acs/tsp_instance.hpp
 * (TspInstance, build_candidates, nn_tour_length, tour_length) and the
 * SPEC-defined solver surface run(inst, AcsParams) -> RunReport
 * (SPEC.md:276-311).  The C++ drop-in (include/acs/solver.hpp) is a thin layer
 * over the plain-C entry points below, which are also what a cgo/JNI/ctypes
 * binding would bind.  Every function returns 0 on success
 * and a negative ACS_E_* code on failure; acs_gpu_last_error() then returns a
 * thread-local message.  There is no CPU fallback: without a CUDA device every
 * compute entry point fails with ACS_E_CUDA.
 *
 * Ownership: the caller owns every host buffer; a context owns every device
 * allocation until acs_gpu_destroy.  One context = one device + one stream;
 * calls on a context must be externally serialised; distinct contexts may be
 * driven from distinct host threads (island model).
 */
#ifndef ACS_GPU_H
#define ACS_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACS_GPU_ABI_VERSION 5  /* 2: acs_counters.fallback_full, acs_random_instance; 3: ACS_VARIANT_SPM_SYNC;
                                  4: acs_gpu_island_exchange_local, acs_gpu_l2_latency, 16-bit island ranks;
                                  5: acs_counters.relaxed_writes / lost_updates / fallback_grid */

/* status codes */
#define ACS_OK 0
#define ACS_E_ARG (-1)     /* invalid argument / unsupported parameter combination */
#define ACS_E_CUDA (-2)    /* CUDA runtime error or no device */
#define ACS_E_NOMEM (-3)   /* device allocation failed */
#define ACS_E_NCCL (-4)    /* NCCL unavailable or failed (island exchange) */
#define ACS_E_PARSE (-5)   /* TSPLIB parse error (message names the field) */

/* TSPLIB edge weight types, tsp_instance.hpp:16 */
enum acs_edge_weight { ACS_EUC_2D = 0, ACS_CEIL_2D = 1, ACS_ATT = 2 };

/* Pheromone-memory variants (SURVEY.md section 8(a) variant mapping). */
enum acs_variant {
    ACS_VARIANT_ATOMIC = 0,   /* dense matrix, whole tour per launch, CAS local updates (CONSISTENT) */
    ACS_VARIANT_DEFERRED = 1, /* dense matrix, SPEC SYNC: select on step snapshot, ordered apply */
    ACS_VARIANT_RELAXED = 2,  /* dense matrix, plain relaxed ld/st, lost updates allowed (ACS-GPU-Alt) */
    ACS_VARIANT_SPM = 3,      /* selective pheromone memory, relaxed (ACS-GPU-SPM) */
    ACS_VARIANT_SEQ = 4,      /* dense, SPEC SEQ (ant-major, immediate updates) on one warp */
    ACS_VARIANT_SPM_SEQ = 5,  /* selective memory, SPEC SEQ on one warp */
    ACS_VARIANT_SPM_SYNC = 6  /* selective memory, SPEC SYNC: step snapshot, ordered apply (parity mode, m <= 8192) */
};

enum acs_rng_kind { ACS_RNG_XOSHIRO = 0, ACS_RNG_PHILOX = 1 };

typedef struct {
    uint32_t n;                /* node count, >= 3 */
    uint32_t edge_weight_type; /* enum acs_edge_weight */
    const double *xs;          /* host, n entries */
    const double *ys;          /* host, n entries */
} acs_instance_desc;

/* AcsParams.  alpha = GLOBAL evaporation, rho = LOCAL
 * evaporation, as in the paper/SPEC (north_star's "phi" = rho here). */
typedef struct {
    double beta;             /* heuristic exponent, paper 3 */
    double alpha;            /* global evaporation, paper 0.2 */
    double rho;              /* local evaporation, paper 0.01 */
    double q0;               /* exploitation prob.; < 0 -> max(0,(n-20)/n) */
    uint32_t cl;             /* candidate list length, 1..32 (paper 32) */
    uint32_t ants;           /* m; 0 -> n */
    uint32_t slots;          /* selective memory slots s: 1,2,4,8,16 (paper 8) */
    uint32_t update_period;  /* local update every k-th edge, >= 1 */
    uint32_t variant;        /* enum acs_variant */
    uint32_t rng;            /* enum acs_rng_kind */
    uint64_t seed;
} acs_params;

typedef struct {
    int64_t iter_best_len;   /* best tour length constructed in this iteration */
    uint32_t iter_best_ant;  /* ties -> lowest ant */
    uint32_t improved;       /* 1 if the global best strictly improved */
    int64_t global_best_len; /* L_gb after this iteration */
} acs_iter_stats;

typedef struct {
    uint64_t local_updates;  /* local-update invocations */
    uint64_t hits, misses;   /* selective memory record updates (local + global) */
    uint64_t fallback_steps; /* steps with every candidate visited */
    uint64_t greedy_steps, roulette_steps;
    uint64_t cas_retries;    /* always 0: the atomic variant's updates are contention-free counters (red.add), no CAS */
    uint64_t iterations;     /* iterations run on this context */
    uint64_t fallback_elems; /* unvisited nodes a full fallback scan covers (algorithmic) */
    uint64_t fallback_full;  /* fallback steps the pruned pass could not settle (full scan run) */
    /* RELAXED lost-update instrumentation (library built with -DACS_COUNT_LOST, else 0):
     * candidate-copy pheromone writes of the relaxed construction, and those that
     * replaced a value other than the one their update read (another ant's update
     * of that trail landed in between and was lost) */
    uint64_t relaxed_writes, lost_updates;
    uint64_t fallback_grid;  /* fallback steps settled by the grid-ring walk past the ext rows (n > 4096) */
} acs_counters;

typedef struct {
    uint32_t n, ants, list_len, slots;
    double q0, tau0;
    int64_t nn_len;          /* L_nn from node 0 (tau0 = 1/(n*L_nn)) */
    uint64_t device_bytes;   /* device memory held by the context */
} acs_ctx_info;

typedef struct acs_gpu_ctx acs_gpu_ctx;

const char *acs_gpu_last_error(void);
int acs_gpu_abi_version(void);
int acs_gpu_device_count(int *count);

/* ---- TSPLIB text (replaces parse_tsplib, tsp_instance.cpp:111-189) ----
 * Parses into caller storage: *n receives DIMENSION; xs/ys may be NULL to
 * query the size first (then cap is ignored).  name may be NULL.  Errors
 * return ACS_E_PARSE with the reference's field-naming message. */
int acs_parse_tsplib(const char *text, size_t len, uint32_t *n, uint32_t *edge_weight_type,
                     double *xs, double *ys, uint32_t cap, char *name, size_t name_cap);

/* synthetic uniform instance: coordinates drawn by the
 * reference RngStream(seed).uniform_int(side) (rng.hpp:16-84), x then y per node */
int acs_random_instance(uint32_t n, uint64_t seed, uint32_t side, double *xs, double *ys);

/* host-only: two-sided Wilcoxon rank-sum p-value (SPEC stats.rank_sum_test,
 * SPEC.md:416-424): exact enumeration when nx + ny <= 12, else normal
 * approximation with tie and continuity correction; nx, ny >= 3 */
int acs_rank_sum_test(const double *xs, uint32_t nx, const double *ys, uint32_t ny, double *p);

/* diagnostic: L2 read bandwidth (GB/s) streaming over an L2-resident buffer of
 * `bytes` (the roofline denominator of the L2-resident construction working set) */
int acs_gpu_l2_read_bandwidth(int device, uint64_t bytes, double *gbs);
/* diagnostic: absolute per-step floors of the construction chain over an
 * L2-resident buffer of `bytes` (>= 4 MiB; 48 MiB is L2- but not L1-resident):
 *   *load_ns  L2 load-to-use latency (one-thread pointer chase, ld.global.cg)
 *   *step_ns  one warp's minimal selection step: 512 B row + 256 B trail load,
 *             visited test, score, exact warp argmax, next row = the winner's */
int acs_gpu_l2_latency(int device, uint64_t bytes, double *load_ns, double *step_ns);

/* ---- stateless device ops (setup path) ----
 * replaces TspInstance ctor's dist_table_ (tsp_instance.cpp:23-47) */
int acs_gpu_distance_table(const acs_instance_desc *inst, int device, int32_t *out /* n*n */);
/* replaces build_candidates (tsp_instance.cpp:219-252); identical flat_ layout */
int acs_gpu_build_candidates(const acs_instance_desc *inst, uint32_t cl, int device,
                             uint32_t *out_flat /* n*min(cl,n-1) */, uint32_t *list_len);
/* replaces nn_tour_length (tsp_instance.cpp:254-280) */
int acs_gpu_nn_tour_length(const acs_instance_desc *inst, uint32_t start, int device, int64_t *out);
/* replaces TspInstance::tour_length (tsp_instance.cpp:67-78) for m routes of n nodes */
int acs_gpu_tour_lengths(const acs_instance_desc *inst, const uint32_t *routes, uint32_t m,
                         int device, int64_t *out);
/* device RngStream (rng.hpp:16-84) script: op 0 next_u64, 1 uniform01 bits,
 * 2 uniform_int(args[i]); kind = enum acs_rng_kind; derive=0 -> RngStream(seed) */
int acs_gpu_rng_script(uint32_t kind, uint64_t seed, uint64_t iteration, uint64_t ant, int derive,
                       const int32_t *ops, const uint64_t *args, uint64_t *out, uint32_t count,
                       int device);
/* selective-store op script on the device, single-threaded semantics
 * (SPEC.md:119-163): op (u,v,rule) rule 0 = local update, 1 = global update
 * with l_gb, 2 = read; out[i] = value read / stored.  Final records dumped. */
int acs_gpu_spm_script(uint32_t n, uint32_t slots, double tau_min, double rho, double tau0,
                       double alpha, const uint32_t *ops /* 3*count */, const int64_t *l_gb,
                       uint32_t count, int device, double *out, uint32_t *ids, double *vals,
                       uint32_t *tail, uint64_t *hits, uint64_t *misses);

/* ---- solver context (replaces SPEC run()) ---- */
int acs_gpu_create(const acs_instance_desc *inst, const acs_params *params, int device,
                   acs_gpu_ctx **out);
int acs_gpu_info(const acs_gpu_ctx *ctx, acs_ctx_info *info);
/* runs n_iter ACS iterations (construct + eval + select_best + global update);
 * out may be NULL, else n_iter entries.  Synchronises once at the end. */
int acs_gpu_iterate(acs_gpu_ctx *ctx, uint32_t n_iter, acs_iter_stats *out);
/* device time (CUDA events on the context stream) of the last iterate call:
 * total and the construction kernels alone, in milliseconds */
int acs_gpu_last_timing(const acs_gpu_ctx *ctx, float *total_ms, float *construct_ms);
int acs_gpu_get_best(const acs_gpu_ctx *ctx, uint32_t *order /* n */, int64_t *len);
/* island import: adopts (order, len) if strictly better than the current best */
int acs_gpu_set_best(acs_gpu_ctx *ctx, const uint32_t *order, int64_t len);
int acs_gpu_get_routes(const acs_gpu_ctx *ctx, uint32_t *routes /* m*n */, int64_t *lengths /* m */);
int acs_gpu_get_pheromone(const acs_gpu_ctx *ctx, double *tau /* n*n, dense variants */);
int acs_gpu_get_selective(const acs_gpu_ctx *ctx, uint32_t *ids, double *vals, uint32_t *tail);
int acs_gpu_get_candidates(const acs_gpu_ctx *ctx, uint32_t *flat /* n*list_len */);
int acs_gpu_get_counters(const acs_gpu_ctx *ctx, acs_counters *out);
void acs_gpu_destroy(acs_gpu_ctx *ctx);

/* one-call solve: create + iterations + best + destroy (host buffers in/out) */
int acs_gpu_run(const acs_instance_desc *inst, const acs_params *params, uint64_t iterations,
                int device, uint32_t *best_order /* n */, int64_t *best_len,
                int64_t *trace /* iterations, may be NULL */);

/* ---- island model ----
 * NCCL is loaded lazily (dlopen libnccl.so.2) so the library has no hard
 * NCCL dependency.  unique_id is NCCL's 128-byte ncclUniqueId. */
int acs_gpu_nccl_unique_id(void *unique_id /* 128 bytes */);
int acs_gpu_island_init(acs_gpu_ctx *ctx, const void *unique_id, int nranks, int rank);
/* min-allreduce of (L_gb, rank) then broadcast of the winner's tour; every
 * colony adopts it if strictly better.  Device-side, no host round trip. */
int acs_gpu_island_exchange(acs_gpu_ctx *ctx, int64_t *global_best_len);
/* islands within one GPU: the same exchange (same pack / mask / adopt kernels,
 * ties to the lowest index, strictly-better adoption) among `count` colonies
 * of this process on one device, with the two all-reduces done as device
 * reductions; ctxs[i] plays rank i.  *global_best_len = INT64_MAX when no
 * colony has a tour yet. */
int acs_gpu_island_exchange_local(acs_gpu_ctx *const *ctxs, int count, int64_t *global_best_len);

#ifdef __cplusplus
}
#endif
#endif /* ACS_GPU_H */
