// acs_kernels.cuh -- device-side data layout of one colony and the host
// launchers of every sm_100a kernel (implemented in acs_kernels.cu).
//
// HBM / L2 layout:
//   rows   n x 32 uint4   per candidate slot: {id | mirror<<24, dist, eta^beta (f64)}
//                         -- immutable, one coalesced 512 B row per step
//   tauc   n x 32 f64     pheromone of the candidate edges, candidate order
//   tau    n x n  f64     dense pheromone matrix (fallback + non-candidate edges)
//   spm    n records {vals[S] f64 | ids[S] u32 | tail u32}, 128 B aligned (SpmMem)
//   dist   n x n  i32     distance table (n <= 4096, as tsp_instance.hpp:31)
//   routes m x n  u32, lens m i64
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace acs_dev {

// island exchange key (k_island_pack): L_gb << 16 | rank; at most 65536 ranks
// and tour lengths below 2^47 (n < 2^24 cities at < 2^23 per edge)
constexpr int kIslandRankBits = 16;
constexpr int64_t kIslandRankMask = (int64_t{1} << kIslandRankBits) - 1;
constexpr int kIslandMaxRanks = 1 << kIslandRankBits;
constexpr int64_t kIslandMaxLen = (int64_t{1} << (63 - kIslandRankBits)) - 1;
constexpr int64_t kNoIslandKey = INT64_MAX;

// Selective memory, record-major: record u is one 128 B-aligned block
// {vals[S] f64 | ids[S] u32 | tail u32} (S = 8: 100 B in one line), so reading
// a record is one line instead of three, and two records never share a line
// (a store to record u never sits behind a pending load of record v).
struct SpmMem {
    unsigned char *base = nullptr;
    uint32_t stride = 0;  // bytes per record, multiple of 128
    uint32_t S = 0;
    __host__ __device__ static uint32_t stride_for(uint32_t S) { return (12u * S + 4u + 127u) / 128u * 128u; }
    __device__ __forceinline__ double *vals(uint32_t u) const {
        return reinterpret_cast<double *>(base + static_cast<size_t>(u) * stride);
    }
    __device__ __forceinline__ uint32_t *ids(uint32_t u) const {
        return reinterpret_cast<uint32_t *>(base + static_cast<size_t>(u) * stride + 8u * S);
    }
    __device__ __forceinline__ uint32_t *tail(uint32_t u) const {
        return reinterpret_cast<uint32_t *>(base + static_cast<size_t>(u) * stride + 12u * S);
    }
};


struct DevInstance {
    uint32_t n, words;   // words = ceil(n/32) visited-bitmask words
    int type;            // acs_edge_weight
    const double *xs, *ys;
    const int32_t *dist; // n*n or nullptr (on-the-fly above 4096 nodes)
    const double *etab;  // n*n eta^beta (fallback scan operand) or nullptr
    // non-integral beta: eta^beta by integer distance d (0..eta_dmax), built on
    // the host with the C library's pow -- the value the oracle computes -- so
    // every eta^beta on the device is bit-identical to it; nullptr otherwise
    const double *eta_d;
    uint32_t eta_dmax;
};

constexpr uint32_t kHot = 32;  // hot-list entries per row (one per lane)

struct DevColony {
    uint32_t m, L, k, S;   // ants, list length, update period, spm slots
    double q0, beta;
    uint64_t q0_k;         // floor(q0 * 2^53): q <= q0 as a 53-bit integer compare
    int beta_int;          // >=0: integral beta (repeated multiply), -1: pow
    double c_l, c_0;       // local update tau' = c_l*tau + c_0
    double tau_min;
    uint64_t seed;
    const uint4 *rows;     // n*32 packed candidate rows
    const uint4 *ext;      // n*ext_len next-nearest rows {id, d, eta^beta} for the pruned fallback
    uint32_t ext_len;      // multiple of 32, or 0
    double tau_bound;      // tau0 * (1 + 2^-29): bound on every trail outside the hot lists
    uint32_t *hot;         // n*kHot: non-candidate neighbours the global update deposited on
    uint32_t *hot_cnt;     // n: entries used (> kHot: overflowed, full scan)
    double *tau;           // n*n dense, or nullptr
    double *tauc;          // n*32, or nullptr
    uint32_t *cnt;         // ATOMIC: n*n pending local updates of tau (tau = f^cnt(base))
    uint32_t *cntc;        // ATOMIC: n*32 pending local updates of tauc
    const double *pw_lo;   // ATOMIC: c_l^j, j < 512
    const double *pw_hi;   // ATOMIC: c_l^(512 k), k < pw_hi_n
    uint32_t pw_hi_n;
    SpmMem spm;            // selective memory (record-major), SPM variants only
    uint32_t *routes;      // m*n
    int64_t *lens;         // m
    unsigned long long *counters;  // [8], see Counter
    const uint64_t *iter;  // device iteration counter (RNG derivation index)
    // uniform grid over the bounding box (n > 4096, EUC_2D / CEIL_2D): the
    // pruned fallback continues past the ext rows ring by ring of cells
    const uint32_t *cell_start;  // g*g + 1 (CSR), or nullptr
    const uint32_t *cell_nodes;  // n node ids, by cell then id
    uint32_t grid_g;
    double grid_x0, grid_y0, grid_h;
};

enum Counter {
    kCntUpdates = 0, kCntHits, kCntMisses, kCntFallback, kCntGreedy, kCntRoulette,
    kCntCasRetry, kCntIters, kCntFallbackElems, kCntFallbackFull, kCntRelaxedWrites, kCntLost,
    kCntFallbackGrid, kNumCounters = 16
};

struct DevBest {
    uint32_t *tour;        // n
    int64_t *len;          // 1 (INT64_MAX = none yet)
    double alpha, c_g;     // global update: tau' = c_g*tau + alpha*(1/L_gb)
    uint64_t *iter;        // incremented by the epilogue
    void *stats;           // acs_iter_stats[capacity]
};

// deferred variant: grid-barrier words (arrive count, generation); the per-ant
// state lives in shared memory of the persistent kernel
// SYNC x SELECTIVE (parity mode): per-ant state, visited bitmasks, step ops
struct DevSpmSync {
    void *ants;            // m x SyncAnt<RNG>
    uint32_t *vis;         // m x words
    uint4 *ops;            // 2m {key lo, key hi, neighbour, 0}
    // colonies above one CTA's sort (m > 8192): device-wide radix sort of the keys
    unsigned long long *keys_in, *keys_out;  // 2m
    uint32_t *idx_in, *idx_out;              // 2m
    void *sort_tmp;
    size_t sort_tmp_bytes;
};

struct DevDeferred {
    uint32_t ants_per_warp;    // set by the launcher (grid barrier: cooperative groups)
};

// ---- setup launchers (stream-ordered, async) ----
void launch_distance_table(const DevInstance &I, int32_t *out, cudaStream_t s);
void launch_topk(const DevInstance &I, uint32_t L, uint32_t *out, cudaStream_t s);
void launch_build_rows(const DevInstance &I, const uint32_t *cand, uint32_t L, double beta,
                       int beta_int, uint4 *rows, cudaStream_t s);
void launch_nn_tour_cand(const DevInstance &I, const uint32_t *cand, uint32_t L, uint32_t start, int64_t *out,
                         cudaStream_t s, const uint4 *ext = nullptr, uint32_t ext_len = 0);
void launch_tour_lengths(const DevInstance &I, const uint32_t *routes, uint32_t m, int64_t *out,
                         cudaStream_t s);
void launch_eta_table(const DevInstance &I, double beta, int beta_int, double *out,
                      cudaStream_t s);
// extended neighbour rows (positions L .. L+ext_len-1 of each node's distance
// order), ext_len a multiple of 32; scratch: n*32 keys + n lower bounds
void launch_ext_rows(const DevInstance &I, const uint32_t *cand, uint32_t L, uint32_t ext_len,
                     double beta, int beta_int, uint64_t *scratch_keys, uint64_t *scratch_lower,
                     uint4 *ext, cudaStream_t s);
void launch_fill(double *p, size_t count, double value, cudaStream_t s);
void launch_l2_read(const uint4 *p, size_t count, uint32_t reps, uint32_t *sink, int sms, cudaStream_t s);
void launch_spm_init(const SpmMem &M, uint32_t n, double tau_min, cudaStream_t s);
void launch_rng_script(uint32_t kind, uint64_t seed, uint64_t it, uint64_t ant, int derive,
                       const int32_t *ops, const uint64_t *args, uint64_t *out, uint32_t count,
                       cudaStream_t s);
void launch_spm_script(const SpmMem &M, double tau_min, double c_l, double c_0, double alpha, double c_g,
                       const uint32_t *ops, const int64_t *lgb, uint32_t count, double *out,
                       unsigned long long *hits_misses, cudaStream_t s);

// ---- per-iteration launchers ----
// variant: 0 atomic, 2 relaxed, 3 spm, 4 seq (dense, 1 warp), 5 spm seq (1 warp)
void launch_construct(int variant, int rng, const DevInstance &I, const DevColony &C,
                      cudaStream_t s);
// deferred (SYNC) variant: one cooperative persistent launch per iteration;
// returns 0, or -1 if the colony cannot be made co-resident
int launch_deferred(int rng, const DevInstance &I, const DevColony &C, const DevDeferred &D,
                    cudaStream_t s);
// eval-free epilogue: iteration best (ties lowest ant), strict global best,
// global update on the best tour, stats[slot], iter++
int launch_spm_sync(int rng, const DevInstance &I, const DevColony &C, const DevSpmSync &Y, cudaStream_t s);
size_t spm_sync_ant_bytes();
size_t spm_sync_sort_tmp_bytes(uint32_t count);  // cub::DeviceRadixSort temp storage for 2m keys
void launch_epilogue(bool spm, bool fold, const DevInstance &I, const DevColony &C,
                     const DevBest &B, uint32_t slot, cudaStream_t s);
// island import: adopt (tour,len) from device buffers if strictly better
void launch_adopt_best(const uint32_t *tour, const int64_t *len, const DevInstance &I,
                       const DevBest &B, cudaStream_t s);

// island exchange helpers
void launch_l2_chase(const uint32_t *next, uint32_t steps, uint32_t start, uint32_t *sink, cudaStream_t s);
void launch_step_floor(const uint4 *rows, const double *tau, uint32_t nrows, uint32_t steps, uint32_t tour,
                       uint32_t *sink, cudaStream_t s);
void launch_island_pack(const int64_t *best_len, int rank, int64_t *key, cudaStream_t s);
void launch_island_min(const int64_t *keys, int count, int64_t *out, cudaStream_t s);
void launch_island_sum(const uint32_t *const *tours, int count, uint32_t n, uint32_t *out, cudaStream_t s);
void launch_island_mask(const int64_t *key, int rank, const uint32_t *best_tour, uint32_t n,
                        uint32_t *x_tour, int64_t *x_len, cudaStream_t s);

}  // namespace acs_dev
