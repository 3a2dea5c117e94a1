// acs_kernels.cu -- sm_100a kernels of the ACS hot path (arXiv 1605.02669).
//
// Kernel map:
//   K1 k_distance_table      tsp_instance.cpp:23-47 dist_table_
//   K2 k_topk                tsp_instance.cpp:219-252 build_candidates (bit-exact)
//      k_build_rows          eta^beta + mirror positions of the candidate rows
//      k_nn_tour             tsp_instance.cpp:254-280 nn_tour_length
//   K4 k_construct_dense     whole tour per launch, warp per ant: ATOMIC (CAS) /
//                            RELAXED (plain ld/st, ACS-GPU-Alt) / SEQ (1 warp)
//   K4 k_construct_spm       selective memory (ACS-GPU-SPM) / SPM SEQ (1 warp)
//   K3 k_def_select/apply    step-synchronous deferred variant (SPEC SYNC)
//   K6 k_tour_lengths        tsp_instance.cpp:67-78 tour_length (validation path;
//                            the construction kernels accumulate lengths in int64)
//   K7 k_epilogue            select_best + is_better + global update
//
// The selection loop is latency-bound (one dependent L2 round trip per step);
// every per-step read of a candidate row is ONE coalesced 512 B load of
// immutable data plus one coalesced 256 B load of candidate-ordered pheromone.
#include <algorithm>
#include <climits>
#include <cstdio>

#include "acs_device.cuh"
#include "acs_kernels.cuh"
#include "../../include/acs_gpu.h"

namespace acs_dev {

constexpr int kBlock = 128;           // 4 ants per CTA
constexpr int kMinBlocks = 5;         // >= 20 resident ants per SM (regs <= 102)
constexpr int kWarpsPerBlock = kBlock / 32;
constexpr uint32_t kIdMask = 0x00FFFFFFu;
constexpr uint32_t kNoMirror = 0xFFu;

__device__ __forceinline__ int32_t dist_of(const DevInstance &I, uint32_t u, uint32_t v,
                                           double xu, double yu) {
    if (I.dist) return __ldg(I.dist + static_cast<size_t>(u) * I.n + v);
    return tsplib_distance(I.type, xu, yu, __ldg(I.xs + v), __ldg(I.ys + v));
}

__device__ __forceinline__ bool visited(const uint32_t *vis, uint32_t v) {
    return (vis[v >> 5] >> (v & 31)) & 1u;
}

// ============================================================ setup kernels

__global__ void k_distance_table(DevInstance I, int32_t *out) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t u = blockIdx.y;
    if (v >= I.n) return;
    out[static_cast<size_t>(u) * I.n + v] =
        tsplib_distance(I.type, __ldg(I.xs + u), __ldg(I.ys + u), __ldg(I.xs + v), __ldg(I.ys + v));
}

__device__ __forceinline__ uint64_t shfl_u64(uint64_t x, int src) {
    const uint32_t lo = __shfl_sync(kFull, static_cast<uint32_t>(x), src);
    const uint32_t hi = __shfl_sync(kFull, static_cast<uint32_t>(x >> 32), src);
    return (static_cast<uint64_t>(hi) << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t x, int m) {
    const uint32_t lo = __shfl_xor_sync(kFull, static_cast<uint32_t>(x), m);
    const uint32_t hi = __shfl_xor_sync(kFull, static_cast<uint32_t>(x >> 32), m);
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

// bitonic sort of one key per lane, ascending by lane
__device__ __forceinline__ uint64_t warp_sort_u64(uint64_t x, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const uint64_t p = shfl_xor_u64(x, j);
            const bool up = (lane & k) == 0;
            const bool lower = (lane & j) == 0;
            x = (lower == up) ? (x < p ? x : p) : (x > p ? x : p);
        }
    }
    return x;
}
// sort a bitonic sequence ascending
__device__ __forceinline__ uint64_t warp_merge_u64(uint64_t x, int lane) {
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const uint64_t p = shfl_xor_u64(x, j);
        x = ((lane & j) == 0) ? (x < p ? x : p) : (x > p ? x : p);
    }
    return x;
}

// K2: warp per city keeps the 32 smallest (d<<32 | id) keys of its row as a
// lane-sorted register list; a 32-key chunk is merged only when one of its
// keys beats the current 32nd (ballot), so most chunks cost one distance
// evaluation per lane.  Key order == the reference comparator (cpp:241-245).
__global__ void __launch_bounds__(kBlock) k_topk(DevInstance I, uint32_t L, uint32_t *out) {
    const int lane = threadIdx.x & 31;
    const uint32_t u = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (u >= I.n) return;
    const double xu = __ldg(I.xs + u), yu = __ldg(I.ys + u);
    uint64_t top = ~0ull;
    for (uint32_t base = 0; base < I.n; base += 32) {
        const uint32_t v = base + lane;
        uint64_t key = ~0ull;
        if (v < I.n && v != u) {
            const int32_t d = tsplib_distance(I.type, xu, yu, __ldg(I.xs + v), __ldg(I.ys + v));
            key = (static_cast<uint64_t>(static_cast<uint32_t>(d)) << 32) | v;
        }
        const uint64_t thr = shfl_u64(top, 31);
        if (!__any_sync(kFull, key < thr)) continue;
        key = warp_sort_u64(key, lane);
        const uint64_t rev = shfl_u64(key, 31 - lane);
        top = top < rev ? top : rev;
        top = warp_merge_u64(top, lane);
    }
    if (static_cast<uint32_t>(lane) < L) out[static_cast<size_t>(u) * L + lane] = static_cast<uint32_t>(top);
}

// packed candidate rows: {id | mirror<<24, d, eta^beta lo, eta^beta hi}
__global__ void k_build_rows(DevInstance I, const uint32_t *cand, uint32_t L, double beta,
                             int beta_int, uint4 *rows) {
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<size_t>(I.n) * 32) return;
    const uint32_t u = static_cast<uint32_t>(idx >> 5), p = static_cast<uint32_t>(idx & 31);
    uint4 el = make_uint4(0xFFFFFFFFu, 0u, 0u, 0u);
    if (p < L) {
        const uint32_t c = cand[static_cast<size_t>(u) * L + p];
        const int32_t d = tsplib_distance(I.type, I.xs[u], I.ys[u], I.xs[c], I.ys[c]);
        const double eb = eta_beta(d, beta, beta_int);
        uint32_t mirror = kNoMirror;
        for (uint32_t q = 0; q < L; ++q)
            if (cand[static_cast<size_t>(c) * L + q] == u) { mirror = q; break; }
        const uint64_t b = dbits(eb);
        el = make_uint4(c | (mirror << 24), static_cast<uint32_t>(d), static_cast<uint32_t>(b),
                        static_cast<uint32_t>(b >> 32));
    }
    rows[idx] = el;
}

// nn_tour_length: one CTA, per step a block argmin of (d<<32 | v) over the
// unvisited nodes (strict < in ascending v == min key), cpp:254-280.
__global__ void __launch_bounds__(1024) k_nn_tour(DevInstance I, uint32_t start, int64_t *out) {
    extern __shared__ uint32_t vis[];
    __shared__ uint64_t red[32];
    __shared__ uint64_t pick;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (uint32_t i = tid; i < I.words; i += blockDim.x) vis[i] = 0;
    __syncthreads();
    if (tid == 0) vis[start >> 5] |= 1u << (start & 31);
    __syncthreads();
    uint32_t cur = start;
    int64_t total = 0;
    for (uint32_t step = 1; step < I.n; ++step) {
        const double xc = __ldg(I.xs + cur), yc = __ldg(I.ys + cur);
        uint64_t best = ~0ull;
        for (uint32_t v = tid; v < I.n; v += blockDim.x) {
            if (visited(vis, v)) continue;
            const int32_t d = dist_of(I, cur, v, xc, yc);
            const uint64_t key = (static_cast<uint64_t>(static_cast<uint32_t>(d)) << 32) | v;
            best = key < best ? key : best;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t p = shfl_xor_u64(best, o);
            best = p < best ? p : best;
        }
        if (lane == 0) red[wid] = best;
        __syncthreads();
        if (wid == 0) {
            uint64_t b = lane < static_cast<int>(blockDim.x >> 5) ? red[lane] : ~0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const uint64_t p = shfl_xor_u64(b, o);
                b = p < b ? p : b;
            }
            if (lane == 0) {
                pick = b;
                const uint32_t v = static_cast<uint32_t>(b);
                vis[v >> 5] |= 1u << (v & 31);
            }
        }
        __syncthreads();
        total += static_cast<int64_t>(pick >> 32);
        cur = static_cast<uint32_t>(pick);
    }
    if (tid == 0) *out = total + dist_of(I, cur, start, __ldg(I.xs + cur), __ldg(I.ys + cur));
}

// K6: warp per route, int64 closed-tour sum (cpp:67-78)
__global__ void k_tour_lengths(DevInstance I, const uint32_t *routes, uint32_t m, int64_t *out) {
    const int lane = threadIdx.x & 31;
    const uint32_t a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (a >= m) return;
    const uint32_t *r = routes + static_cast<size_t>(a) * I.n;
    long long acc = 0;
    for (uint32_t i = lane; i < I.n; i += 32) {
        const uint32_t u = r[i == 0 ? I.n - 1 : i - 1], v = r[i];
        acc += dist_of(I, u, v, __ldg(I.xs + u), __ldg(I.ys + u));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (lane == 0) out[a] = acc;
}

__global__ void k_fill(double *p, size_t count, double v) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

__global__ void k_spm_init(uint32_t *ids, double *vals, uint32_t *tail, uint32_t n, uint32_t S,
                           double tau_min) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
         i < static_cast<size_t>(n) * S; i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        ids[i] = kEmpty;
        vals[i] = tau_min;
        if (i < n) tail[i] = S - 1;  // D5: first insertion lands in slot 0
    }
}

template <class E>
__device__ void rng_script_body(E &e, const int32_t *ops, const uint64_t *args, uint64_t *out,
                                uint32_t count) {
    for (uint32_t i = 0; i < count; ++i) {
        if (ops[i] == 0) out[i] = e.next();
        else if (ops[i] == 1) out[i] = dbits(uniform01(e));
        else out[i] = uniform_int(e, args[i]);
    }
}

__global__ void k_rng_script(uint32_t kind, uint64_t seed, uint64_t it, uint64_t ant, int derive,
                             const int32_t *ops, const uint64_t *args, uint64_t *out,
                             uint32_t count) {
    if (kind == ACS_RNG_PHILOX) {
        Philox e;
        e.derive(seed, it, ant);
        rng_script_body(e, ops, args, out, count);
    } else {
        Xoshiro e;
        if (derive) e.derive(seed, it, ant);
        else e.seed(seed);
        rng_script_body(e, ops, args, out, count);
    }
}

// ============================================================ selective memory

// Single-thread record update on global memory (Fig. alg:3):
// hit -> in place, tail untouched; miss -> value from tau_min inserted at
// (tail+1) % S evicting the least-recently inserted.  Relaxed accesses keep
// the RELAXED contract's range invariants under races.
__device__ __forceinline__ bool spm_update_mem(uint32_t *ids, double *vals, uint32_t *tail,
                                               uint32_t S, uint32_t u, uint32_t v, double c_mul,
                                               double c_add, double tau_min, double *stored) {
    const size_t base = static_cast<size_t>(u) * S;
    for (uint32_t j = 0; j < S; ++j) {
        if (ld_relaxed_u32(ids + base + j) == v) {
            const double y = affine(ld_relaxed(vals + base + j), c_mul, c_add);
            st_relaxed(vals + base + j, y);
            if (stored) *stored = y;
            return true;
        }
    }
    const double y = affine(tau_min, c_mul, c_add);
    const uint32_t t = (ld_relaxed_u32(tail + u) + 1) % S;
    st_relaxed_u32(ids + base + t, v);
    st_relaxed(vals + base + t, y);
    st_relaxed_u32(tail + u, t);
    if (stored) *stored = y;
    return false;
}

__device__ __forceinline__ double spm_read_mem(const uint32_t *ids, const double *vals, uint32_t S,
                                               uint32_t u, uint32_t v, double tau_min) {
    const size_t base = static_cast<size_t>(u) * S;
    for (uint32_t j = 0; j < S; ++j)
        if (ld_relaxed_u32(ids + base + j) == v) return ld_relaxed(vals + base + j);
    return tau_min;
}

__global__ void k_spm_script(uint32_t *ids, double *vals, uint32_t *tail, uint32_t S,
                             double tau_min, double c_l, double c_0, double alpha, double c_g,
                             const uint32_t *ops, const int64_t *lgb, uint32_t count, double *out,
                             unsigned long long *hm) {
    for (uint32_t i = 0; i < count; ++i) {
        const uint32_t u = ops[3 * i], v = ops[3 * i + 1], rule = ops[3 * i + 2];
        if (rule == 2) {
            out[i] = spm_read_mem(ids, vals, S, u, v, tau_min);
            continue;
        }
        double cm = c_l, ca = c_0;
        if (rule == 1) {
            cm = c_g;
            ca = __dmul_rn(alpha, __ddiv_rn(1.0, static_cast<double>(lgb[i])));
        }
        const bool hit = spm_update_mem(ids, vals, tail, S, u, v, cm, ca, tau_min, &out[i]);
        hm[hit ? 0 : 1] += 1;
    }
}

// Register copy of one record: every lane holds all S slots (broadcast loads).
template <int S>
struct SpmRec {
    uint32_t id[S];
    double val[S];
    uint32_t tail;

    __device__ __forceinline__ void load(const DevColony &C, uint32_t u) {
        const size_t base = static_cast<size_t>(u) * S;
        if constexpr (S >= 4) {
#pragma unroll
            for (int j = 0; j < S; j += 4) {
                const uint4 q = __ldcg(reinterpret_cast<const uint4 *>(C.spm_ids + base + j));
                id[j] = q.x; id[j + 1] = q.y; id[j + 2] = q.z; id[j + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < S; ++j) id[j] = __ldcg(C.spm_ids + base + j);
        }
        if constexpr (S >= 2) {
#pragma unroll
            for (int j = 0; j < S; j += 2) {
                const double2 q = __ldcg(reinterpret_cast<const double2 *>(C.spm_vals + base + j));
                val[j] = q.x; val[j + 1] = q.y;
            }
        } else {
            val[0] = __ldcg(C.spm_vals + base);
        }
        tail = __ldcg(C.spm_tail + u);
    }
    __device__ __forceinline__ double lookup(uint32_t v, double tau_min) const {
        double r = tau_min;
        bool found = false;
#pragma unroll
        for (int j = 0; j < S; ++j)
            if (!found && id[j] == v) { r = val[j]; found = true; }
        return r;
    }
    // update record u with neighbour v; lane 0 writes through. Returns hit.
    __device__ __forceinline__ bool update(const DevColony &C, uint32_t u, uint32_t v, double c_mul,
                                           double c_add, int lane) {
        int hit = -1;
#pragma unroll
        for (int j = 0; j < S; ++j)
            if (hit < 0 && id[j] == v) hit = j;
        const size_t base = static_cast<size_t>(u) * S;
        if (hit >= 0) {
            double y = 0.0;
#pragma unroll
            for (int j = 0; j < S; ++j)
                if (j == hit) { y = affine(val[j], c_mul, c_add); val[j] = y; }
            if (lane == 0) st_relaxed(C.spm_vals + base + hit, y);
            return true;
        }
        const double y = affine(C.tau_min, c_mul, c_add);
        const uint32_t t = (tail + 1) % S;
#pragma unroll
        for (int j = 0; j < S; ++j)
            if (j == static_cast<int>(t)) { id[j] = v; val[j] = y; }
        tail = t;
        if (lane == 0) {
            st_relaxed_u32(C.spm_ids + base + t, v);
            st_relaxed(C.spm_vals + base + t, y);
            st_relaxed_u32(C.spm_tail + u, t);
        }
        return false;
    }
};

// ============================================================ selection

struct Step {
    uint32_t v;        // chosen node
    int pos;           // candidate position, -1 for fallback
    uint32_t mirror;   // position of cur in v's list, kNoMirror if absent
    double tau_old;    // trail value the selection read for (cur, v)
    int32_t d;         // distance(cur, v)
    int kind;          // 0 greedy, 1 roulette, 2 fallback
};

// full-scan fallback (Alg.2 l.18): argmax tau*eta^beta over all
// unvisited nodes, ties -> lowest id, no RNG draw (P1).  Lane-strided over
// the visited bitmask words so only unvisited nodes are touched.
template <class TauFn>
__device__ __forceinline__ void fallback_scan(const DevInstance &I, const DevColony &C,
                                              const uint32_t *vis, uint32_t cur, double xc,
                                              double yc, TauFn tau_of, int lane, Step &o) {
    double bs = 0.0, bt = 0.0;
    uint32_t bv = 0xffffffffu;
    int32_t bd = 0;
    bool have = false;
    for (uint32_t w0 = 0; w0 < I.words; w0 += 32) {
        const uint32_t w = w0 + lane;
        uint32_t bits = 0;
        if (w < I.words) {
            bits = ~vis[w];
            if (w == I.words - 1 && (I.n & 31)) bits &= (1u << (I.n & 31)) - 1u;
        }
        while (__any_sync(kFull, bits != 0)) {
            if (bits) {
                const uint32_t v = w * 32 + (__ffs(bits) - 1);
                bits &= bits - 1;
                const double tv = tau_of(v);
                const int32_t d = dist_of(I, cur, v, xc, yc);
                const double s = __dmul_rn(tv, eta_beta(d, C.beta, C.beta_int));
                if (!have || s > bs) { have = true; bs = s; bv = v; bt = tv; bd = d; }
            }
        }
    }
    double s = bs;
    uint32_t node = have ? bv : 0xffffffffu;
    warp_argmax_node(s, node, have);
    const unsigned owner = __ballot_sync(kFull, have && bv == node);
    const int src = __ffs(owner) - 1;
    o.v = node;
    o.tau_old = __shfl_sync(kFull, bt, src);
    o.d = __shfl_sync(kFull, bd, src);
    o.pos = -1;
    o.kind = 2;
    // mirror: where does cur sit in v's candidate row?
    const uint32_t id = __ldg(&C.rows[static_cast<size_t>(node) * 32 + lane].x) & kIdMask;
    const unsigned mm = __ballot_sync(kFull, static_cast<uint32_t>(lane) < C.L && id == cur);
    o.mirror = mm ? static_cast<uint32_t>(__ffs(mm) - 1) : kNoMirror;
}

// candidate branch (Eq.1 / Eq.2 over the filtered list, Alg.2 l.5-16) with
// the P1 draw protocol; falls through to fallback_scan when all are visited.
template <class RNG, class TauFn>
__device__ __forceinline__ void select_step(const DevInstance &I, const DevColony &C,
                                            const uint32_t *vis, uint32_t cur, double xc,
                                            double yc, uint4 el, double tau_lane, RNG &rng,
                                            double *scratch, int lane, TauFn tau_of, Step &o) {
    const uint32_t c = el.x & kIdMask;
    const bool valid = static_cast<uint32_t>(lane) < C.L;
    const bool unv = valid && !visited(vis, c);
    const unsigned um = __ballot_sync(kFull, unv);
    if (um) {
        const double eb = __hiloint2double(static_cast<int>(el.w), static_cast<int>(el.z));
        const double score = unv ? __dmul_rn(tau_lane, eb) : 0.0;
        const double q = uniform01(rng);
        int pos;
        if (q <= C.q0) {
            pos = warp_argmax_pos(score, unv);
            o.kind = 0;
        } else {
            const double r = uniform01(rng);
            pos = warp_roulette_pos(score, um, r, scratch, lane);
            o.kind = 1;
        }
        o.pos = pos;
        o.v = __shfl_sync(kFull, c, pos);
        o.mirror = __shfl_sync(kFull, el.x >> 24, pos);
        o.d = static_cast<int32_t>(__shfl_sync(kFull, el.y, pos));
        o.tau_old = __shfl_sync(kFull, tau_lane, pos);
        return;
    }
    fallback_scan(I, C, vis, cur, xc, yc, tau_of, lane, o);
}

struct WarpCounters {
    unsigned long long fallback = 0, greedy = 0, roulette = 0, updates = 0, retry = 0, hits = 0,
                       misses = 0, fb_elems = 0;
    // unvisited = n - t at step t: the elements a fallback scan touches
    __device__ __forceinline__ void count(int kind, uint32_t unvisited) {
        if (kind == 0) ++greedy;
        else if (kind == 1) ++roulette;
        else { ++fallback; fb_elems += unvisited; }
    }
    __device__ __forceinline__ void flush(unsigned long long *c, int lane) {
        if (lane != 0) return;
        if (updates) atomicAdd(c + kCntUpdates, updates);
        if (hits) atomicAdd(c + kCntHits, hits);
        if (misses) atomicAdd(c + kCntMisses, misses);
        if (fallback) atomicAdd(c + kCntFallback, fallback);
        if (greedy) atomicAdd(c + kCntGreedy, greedy);
        if (roulette) atomicAdd(c + kCntRoulette, roulette);
        if (retry) atomicAdd(c + kCntCasRetry, retry);
        if (fb_elems) atomicAdd(c + kCntFallbackElems, fb_elems);
    }
};

// route buffered in registers: lane (t & 31) holds route[t]; one coalesced
// 128 B store per 32 steps.
__device__ __forceinline__ void route_put(uint32_t *route, uint32_t &rbuf, uint32_t t, uint32_t v,
                                          int lane) {
    if (static_cast<uint32_t>(lane) == (t & 31)) rbuf = v;
    if ((t & 31) == 31) route[(t & ~31u) + lane] = rbuf;
}
__device__ __forceinline__ void route_flush(uint32_t *route, uint32_t rbuf, uint32_t last,
                                            int lane) {
    if ((last & 31) != 31 && static_cast<uint32_t>(lane) <= (last & 31))
        route[(last & ~31u) + lane] = rbuf;
}

// ============================================================ dense whole tour

// dense local update of (u,v) on its (up to) four copies, one lane each:
// lane 0 tau[u][v], lane 1 tau[v][u], lane 2 tauc[u][pos], lane 3 tauc[v][mirror].
__device__ __forceinline__ double *dense_copy_addr(const DevColony &C, uint32_t n, uint32_t u,
                                                   uint32_t v, int pos, uint32_t mirror,
                                                   int lane) {
    if (lane == 0) return C.tau + static_cast<size_t>(u) * n + v;
    if (lane == 1) return C.tau + static_cast<size_t>(v) * n + u;
    if (lane == 2 && pos >= 0) return C.tauc + static_cast<size_t>(u) * 32 + pos;
    if (lane == 3 && mirror != kNoMirror) return C.tauc + static_cast<size_t>(v) * 32 + mirror;
    return nullptr;
}

// In-flight CAS of one lane (ATOMIC variant): issued at step t, verified at
// step t+1 after that step's row loads are in flight, so the atomic round
// trip overlaps the next dependent load instead of adding to it.
struct PendingCas {
    unsigned long long *addr = nullptr;
    unsigned long long expect = 0, got = 0;

    __device__ __forceinline__ void issue(double *p, double old, const DevColony &C) {
        addr = reinterpret_cast<unsigned long long *>(p);
        expect = dbits(old);
        got = atomicCAS(addr, expect, dbits(affine(old, C.c_l, C.c_0)));
    }
    __device__ __forceinline__ void settle(const DevColony &C, WarpCounters &wc) {
        if (addr == nullptr) return;
        while (got != expect) {
            ++wc.retry;
            expect = got;
            got = atomicCAS(addr, expect, dbits(affine(bitsd(expect), C.c_l, C.c_0)));
        }
        addr = nullptr;
    }
};

template <bool kAtomic, class RNG>
__global__ void __launch_bounds__(kBlock, kMinBlocks) k_construct_dense(DevInstance I, DevColony C) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    double *scratch = reinterpret_cast<double *>(smem) + wib * 32;
    uint32_t *vis = reinterpret_cast<uint32_t *>(smem + wpb * 32 * sizeof(double)) +
                    static_cast<size_t>(wib) * I.words;
    const uint64_t it = *C.iter;
    const uint32_t n = I.n;
    WarpCounters wc;
    PendingCas pc;

    for (uint32_t a = blockIdx.x * wpb + wib; a < C.m; a += gridDim.x * wpb) {
        for (uint32_t i = lane; i < I.words; i += 32) vis[i] = 0;
        RNG rng;
        rng.derive(C.seed, it, a);
        const uint32_t start = static_cast<uint32_t>(uniform_int(rng, n));  // P1.1
        __syncwarp();
        if (lane == 0) vis[start >> 5] |= 1u << (start & 31);
        __syncwarp();
        uint32_t *route = C.routes + static_cast<size_t>(a) * n;
        uint32_t rbuf = start, cur = start;
        long long len = 0;
        double xc = __ldg(I.xs + cur), yc = __ldg(I.ys + cur);
        auto tau_row = [&](uint32_t v) { return ld_relaxed(C.tau + static_cast<size_t>(cur) * n + v); };

        for (uint32_t t = 1; t < n; ++t) {
            const size_t ri = static_cast<size_t>(cur) * 32 + lane;
            const uint4 el = __ldg(C.rows + ri);
            const double tau_lane = ld_relaxed(C.tauc + ri);
            if constexpr (kAtomic) pc.settle(C, wc);
            Step st;
            select_step(I, C, vis, cur, xc, yc, el, tau_lane, rng, scratch, lane, tau_row, st);
            wc.count(st.kind, n - t);
            if (t % C.k == 0) {  // D9 per-ant edge counter
                ++wc.updates;
                double *p = dense_copy_addr(C, n, cur, st.v, st.pos, st.mirror, lane);
                if (p) {
                    if constexpr (kAtomic) pc.issue(p, st.tau_old, C);
                    else st_relaxed(p, affine(st.tau_old, C.c_l, C.c_0));
                }
            }
            if (lane == 0) {
                vis[st.v >> 5] |= 1u << (st.v & 31);
                len += st.d;
            }
            route_put(route, rbuf, t, st.v, lane);
            cur = st.v;
            xc = __ldg(I.xs + cur);
            yc = __ldg(I.ys + cur);
            __syncwarp();
        }
        route_flush(route, rbuf, n - 1, lane);
        if constexpr (kAtomic) pc.settle(C, wc);

        // closing edge (cur -> start): counted as edge n (D9)
        const uint32_t id = __ldg(&C.rows[static_cast<size_t>(cur) * 32 + lane].x);
        const unsigned hit = __ballot_sync(kFull, static_cast<uint32_t>(lane) < C.L && (id & kIdMask) == start);
        int32_t dclose;
        if (hit) {
            const int p = __ffs(hit) - 1;
            dclose = static_cast<int32_t>(__ldg(&C.rows[static_cast<size_t>(cur) * 32 + p].y));
        } else {
            dclose = dist_of(I, cur, start, xc, yc);
        }
        if (n % C.k == 0) {
            ++wc.updates;
            const int pos = hit ? __ffs(hit) - 1 : -1;
            uint32_t mirror = kNoMirror;
            if (hit) {
                mirror = __shfl_sync(kFull, id >> 24, pos);
            } else {
                const uint32_t id2 = __ldg(&C.rows[static_cast<size_t>(start) * 32 + lane].x) & kIdMask;
                const unsigned mm = __ballot_sync(kFull, static_cast<uint32_t>(lane) < C.L && id2 == cur);
                if (mm) mirror = static_cast<uint32_t>(__ffs(mm) - 1);
            }
            const double told = ld_relaxed(C.tau + static_cast<size_t>(cur) * n + start);
            double *p = dense_copy_addr(C, n, cur, start, pos, mirror, lane);
            if (p) {
                if constexpr (kAtomic) wc.retry += cas_affine(p, told, C.c_l, C.c_0);
                else st_relaxed(p, affine(told, C.c_l, C.c_0));
            }
        }
        if (lane == 0) C.lens[a] = len + dclose;
        __syncwarp();
    }
    wc.flush(C.counters, lane);
}

// ============================================================ selective whole tour

template <int S, class RNG>
__global__ void __launch_bounds__(kBlock, kMinBlocks) k_construct_spm(DevInstance I, DevColony C) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    double *scratch = reinterpret_cast<double *>(smem) + wib * 32;
    uint32_t *vis = reinterpret_cast<uint32_t *>(smem + wpb * 32 * sizeof(double)) +
                    static_cast<size_t>(wib) * I.words;
    const uint64_t it = *C.iter;
    const uint32_t n = I.n;
    WarpCounters wc;

    for (uint32_t a = blockIdx.x * wpb + wib; a < C.m; a += gridDim.x * wpb) {
        for (uint32_t i = lane; i < I.words; i += 32) vis[i] = 0;
        RNG rng;
        rng.derive(C.seed, it, a);
        const uint32_t start = static_cast<uint32_t>(uniform_int(rng, n));
        __syncwarp();
        if (lane == 0) vis[start >> 5] |= 1u << (start & 31);
        __syncwarp();
        uint32_t *route = C.routes + static_cast<size_t>(a) * n;
        uint32_t rbuf = start, cur = start, prev = 0;
        bool pending = false;  // record `cur` still owes the update with `prev` (D4)
        long long len = 0;
        double xc = __ldg(I.xs + cur), yc = __ldg(I.ys + cur);
        SpmRec<S> rec;

        for (uint32_t t = 1; t < n; ++t) {
            const uint4 el = __ldg(C.rows + static_cast<size_t>(cur) * 32 + lane);
            rec.load(C, cur);
            if (pending) {
                if (rec.update(C, cur, prev, C.c_l, C.c_0, lane)) ++wc.hits; else ++wc.misses;
            }
            const uint32_t c = el.x & kIdMask;
            const double tau_lane = rec.lookup(c, C.tau_min);
            Step st;
            select_step(I, C, vis, cur, xc, yc, el, tau_lane, rng, scratch, lane,
                        [&](uint32_t v) { return rec.lookup(v, C.tau_min); }, st);
            wc.count(st.kind, n - t);
            pending = (t % C.k == 0);
            if (pending) {
                ++wc.updates;
                if (rec.update(C, cur, st.v, C.c_l, C.c_0, lane)) ++wc.hits; else ++wc.misses;
                prev = cur;
            }
            if (lane == 0) {
                vis[st.v >> 5] |= 1u << (st.v & 31);
                len += st.d;
            }
            route_put(route, rbuf, t, st.v, lane);
            cur = st.v;
            xc = __ldg(I.xs + cur);
            yc = __ldg(I.ys + cur);
            __syncwarp();
        }
        route_flush(route, rbuf, n - 1, lane);
        rec.load(C, cur);
        if (pending) {
            if (rec.update(C, cur, prev, C.c_l, C.c_0, lane)) ++wc.hits; else ++wc.misses;
        }
        const int32_t dclose = dist_of(I, cur, start, xc, yc);
        if (n % C.k == 0) {  // closing edge: record last, then record start
            ++wc.updates;
            if (rec.update(C, cur, start, C.c_l, C.c_0, lane)) ++wc.hits; else ++wc.misses;
            __syncwarp();
            SpmRec<S> r2;
            r2.load(C, start);
            if (r2.update(C, start, cur, C.c_l, C.c_0, lane)) ++wc.hits; else ++wc.misses;
        }
        if (lane == 0) C.lens[a] = len + dclose;
        __syncwarp();
    }
    wc.flush(C.counters, lane);
}

// ============================================================ deferred (SYNC)

template <class RNG>
__global__ void k_def_init(DevInstance I, DevColony C, DevDeferred D) {
    const int lane = threadIdx.x & 31;
    const uint32_t a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (a >= C.m) return;
    uint32_t *vis = D.vis + static_cast<size_t>(a) * I.words;
    for (uint32_t i = lane; i < I.words; i += 32) vis[i] = 0;
    RNG rng;
    rng.derive(C.seed, *C.iter, a);
    const uint32_t start = static_cast<uint32_t>(uniform_int(rng, I.n));
    __syncwarp();
    if (lane == 0) {
        vis[start >> 5] |= 1u << (start & 31);
        D.cur[a] = start;
        D.start[a] = start;
        reinterpret_cast<RNG *>(D.rng)[a] = rng;
        C.routes[static_cast<size_t>(a) * I.n] = start;
        C.lens[a] = 0;
    }
}

// one step for every ant against the step-start pheromone (no writes to tau)
template <class RNG>
__global__ void __launch_bounds__(kBlock) k_def_select(DevInstance I, DevColony C, DevDeferred D,
                                                       uint32_t t) {
    __shared__ double scratch_all[kWarpsPerBlock * 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t a = blockIdx.x * kWarpsPerBlock + wib;
    if (a >= C.m) return;
    double *scratch = scratch_all + wib * 32;
    uint32_t *vis = D.vis + static_cast<size_t>(a) * I.words;
    const uint32_t cur = D.cur[a];
    RNG rng = reinterpret_cast<RNG *>(D.rng)[a];
    const size_t ri = static_cast<size_t>(cur) * 32 + lane;
    const uint4 el = __ldg(C.rows + ri);
    const double tau_lane = C.tauc[ri];
    const double xc = __ldg(I.xs + cur), yc = __ldg(I.ys + cur);
    Step st;
    select_step(I, C, vis, cur, xc, yc, el, tau_lane, rng, scratch, lane,
                [&](uint32_t v) { return C.tau[static_cast<size_t>(cur) * I.n + v]; }, st);
    WarpCounters wc;
    wc.count(st.kind, I.n - t);
    const bool due = (t % C.k == 0);
    if (due) ++wc.updates;
    if (lane == 0) {
        vis[st.v >> 5] |= 1u << (st.v & 31);
        C.routes[static_cast<size_t>(a) * I.n + t] = st.v;
        C.lens[a] += st.d;
        D.cur[a] = st.v;
        reinterpret_cast<RNG *>(D.rng)[a] = rng;
        D.pend[a] = make_uint4(cur, st.v, (static_cast<uint32_t>(st.pos) & 0xFFu) | (st.mirror << 8),
                               due ? 1u : 0u);
    }
    wc.flush(C.counters, lane);
}

// apply the step's local updates: CAS on each copy (the affine maps commute,
// so any interleaving yields f^c(tau) bit-exactly -- P7)
__global__ void k_def_apply(DevInstance I, DevColony C, DevDeferred D) {
    const int lane = threadIdx.x & 31;
    const uint32_t a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (a >= C.m) return;
    const uint4 p = D.pend[a];
    if (!p.w) return;
    const uint32_t u = p.x, v = p.y;
    const int pos = (p.z & 0xFFu) == 0xFFu ? -1 : static_cast<int>(p.z & 0xFFu);
    const uint32_t mirror = (p.z >> 8) & 0xFFu;
    double *addr = dense_copy_addr(C, I.n, u, v, pos, mirror, lane);
    if (addr) cas_affine(addr, *addr, C.c_l, C.c_0);
}

// closing edges in a separate pass after step n-1 (PAPER Alg.1 l.13-14)
__global__ void k_def_close(DevInstance I, DevColony C, DevDeferred D) {
    const int lane = threadIdx.x & 31;
    const uint32_t a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (a >= C.m) return;
    const uint32_t last = D.cur[a], start = D.start[a];
    const uint32_t id = __ldg(&C.rows[static_cast<size_t>(last) * 32 + lane].x);
    const unsigned hit = __ballot_sync(kFull, static_cast<uint32_t>(lane) < C.L && (id & kIdMask) == start);
    const int pos = hit ? __ffs(hit) - 1 : -1;
    uint32_t mirror = kNoMirror;
    if (hit) {
        mirror = __shfl_sync(kFull, id >> 24, pos);
    } else {
        const uint32_t id2 = __ldg(&C.rows[static_cast<size_t>(start) * 32 + lane].x) & kIdMask;
        const unsigned mm = __ballot_sync(kFull, static_cast<uint32_t>(lane) < C.L && id2 == last);
        if (mm) mirror = static_cast<uint32_t>(__ffs(mm) - 1);
    }
    if (I.n % C.k == 0) {
        double *addr = dense_copy_addr(C, I.n, last, start, pos, mirror, lane);
        if (addr) cas_affine(addr, *addr, C.c_l, C.c_0);
        if (lane == 0) atomicAdd(C.counters + kCntUpdates, 1ull);
    }
    if (lane == 0)
        C.lens[a] += dist_of(I, last, start, __ldg(I.xs + last), __ldg(I.ys + last));
}

// ============================================================ epilogue

// select_best (ties -> lowest ant), strict is_better, global update on the
// global-best edges only (D3), per-iteration stats; one CTA.
template <bool kSpm>
__global__ void __launch_bounds__(1024) k_epilogue(DevInstance I, DevColony C, DevBest B,
                                                   uint32_t slot) {
    __shared__ unsigned long long red_len[32];
    __shared__ uint32_t red_ant[32];
    __shared__ int improved;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    long long bl = LLONG_MAX;
    uint32_t ba = 0xffffffffu;
    for (uint32_t a = tid; a < C.m; a += blockDim.x) {
        const long long l = C.lens[a];
        if (l < bl) { bl = l; ba = a; }  // ascending a per thread: strict keeps lowest
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long ol = __shfl_xor_sync(kFull, bl, o);
        const uint32_t oa = __shfl_xor_sync(kFull, ba, o);
        if (ol < bl || (ol == bl && oa < ba)) { bl = ol; ba = oa; }
    }
    if (lane == 0) { red_len[wid] = static_cast<unsigned long long>(bl); red_ant[wid] = ba; }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        bl = lane < nw ? static_cast<long long>(red_len[lane]) : LLONG_MAX;
        ba = lane < nw ? red_ant[lane] : 0xffffffffu;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long ol = __shfl_xor_sync(kFull, bl, o);
            const uint32_t oa = __shfl_xor_sync(kFull, ba, o);
            if (ol < bl || (ol == bl && oa < ba)) { bl = ol; ba = oa; }
        }
        if (lane == 0) {
            red_len[0] = static_cast<unsigned long long>(bl);
            red_ant[0] = ba;
            improved = bl < *B.len;  // strict
        }
    }
    __syncthreads();
    const long long ib_len = static_cast<long long>(red_len[0]);
    const uint32_t ib_ant = red_ant[0];
    const uint32_t n = I.n;
    if (improved) {
        const uint32_t *r = C.routes + static_cast<size_t>(ib_ant) * n;
        for (uint32_t i = tid; i < n; i += blockDim.x) B.tour[i] = r[i];
    }
    __syncthreads();
    const long long gb = improved ? ib_len : *B.len;
    const double c_d = __dmul_rn(B.alpha, __ddiv_rn(1.0, static_cast<double>(gb)));
    if constexpr (kSpm) {
        // record r = tour[j]: edge j-1 (b-side, neighbour tour[j-1]) precedes
        // edge j (a-side, neighbour tour[j+1]); record tour[0] goes a-side first.
        unsigned long long hits = 0, misses = 0;
        for (uint32_t j = tid; j < n; j += blockDim.x) {
            const uint32_t r = B.tour[j];
            const uint32_t nb_prev = B.tour[j == 0 ? n - 1 : j - 1];
            const uint32_t nb_next = B.tour[j + 1 == n ? 0 : j + 1];
            const uint32_t first = j == 0 ? nb_next : nb_prev;
            const uint32_t second = j == 0 ? nb_prev : nb_next;
            if (spm_update_mem(C.spm_ids, C.spm_vals, C.spm_tail, C.S, r, first, B.c_g, c_d, C.tau_min, nullptr)) ++hits; else ++misses;
            if (spm_update_mem(C.spm_ids, C.spm_vals, C.spm_tail, C.S, r, second, B.c_g, c_d, C.tau_min, nullptr)) ++hits; else ++misses;
        }
        if (hits) atomicAdd(C.counters + kCntHits, hits);
        if (misses) atomicAdd(C.counters + kCntMisses, misses);
    } else {
        for (uint32_t i = tid; i < n; i += blockDim.x) {
            const uint32_t a = B.tour[i], b = B.tour[i + 1 == n ? 0 : i + 1];
            double *p = C.tau + static_cast<size_t>(a) * n + b;
            *p = affine(*p, B.c_g, c_d);
            p = C.tau + static_cast<size_t>(b) * n + a;
            *p = affine(*p, B.c_g, c_d);
            for (uint32_t q = 0; q < C.L; ++q) {
                if ((C.rows[static_cast<size_t>(a) * 32 + q].x & kIdMask) == b) {
                    double *t = C.tauc + static_cast<size_t>(a) * 32 + q;
                    *t = affine(*t, B.c_g, c_d);
                }
                if ((C.rows[static_cast<size_t>(b) * 32 + q].x & kIdMask) == a) {
                    double *t = C.tauc + static_cast<size_t>(b) * 32 + q;
                    *t = affine(*t, B.c_g, c_d);
                }
            }
        }
    }
    if (tid == 0) {
        if (improved) *B.len = ib_len;
        acs_iter_stats *s = reinterpret_cast<acs_iter_stats *>(B.stats) + slot;
        s->iter_best_len = ib_len;
        s->iter_best_ant = ib_ant;
        s->improved = improved ? 1u : 0u;
        s->global_best_len = gb;
        *B.iter += 1;
        atomicAdd(C.counters + kCntIters, 1ull);
    }
}

__global__ void k_adopt_best(const uint32_t *tour, const int64_t *len, uint32_t n, DevBest B) {
    __shared__ int take;
    if (threadIdx.x == 0) take = *len < *B.len;
    __syncthreads();
    if (!take) return;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) B.tour[i] = tour[i];
    __syncthreads();
    if (threadIdx.x == 0) *B.len = *len;
}

// ============================================================ launchers

static unsigned blocks_for(size_t work, unsigned per) {
    return static_cast<unsigned>((work + per - 1) / per);
}

void launch_distance_table(const DevInstance &I, int32_t *out, cudaStream_t s) {
    dim3 grid(blocks_for(I.n, 256), I.n);
    k_distance_table<<<grid, 256, 0, s>>>(I, out);
}

void launch_topk(const DevInstance &I, uint32_t L, uint32_t *out, cudaStream_t s) {
    k_topk<<<blocks_for(I.n, kWarpsPerBlock), kBlock, 0, s>>>(I, L, out);
}

void launch_build_rows(const DevInstance &I, const uint32_t *cand, uint32_t L, double beta,
                       int beta_int, uint4 *rows, cudaStream_t s) {
    k_build_rows<<<blocks_for(static_cast<size_t>(I.n) * 32, 256), 256, 0, s>>>(I, cand, L, beta,
                                                                                beta_int, rows);
}

void launch_nn_tour(const DevInstance &I, uint32_t start, int64_t *out, cudaStream_t s) {
    k_nn_tour<<<1, 1024, I.words * sizeof(uint32_t), s>>>(I, start, out);
}

void launch_tour_lengths(const DevInstance &I, const uint32_t *routes, uint32_t m, int64_t *out,
                         cudaStream_t s) {
    k_tour_lengths<<<blocks_for(m, 8), 256, 0, s>>>(I, routes, m, out);
}

void launch_fill(double *p, size_t count, double value, cudaStream_t s) {
    k_fill<<<std::min<size_t>(blocks_for(count, 256), 148 * 16), 256, 0, s>>>(p, count, value);
}

void launch_spm_init(uint32_t *ids, double *vals, uint32_t *tail, uint32_t n, uint32_t S,
                     double tau_min, cudaStream_t s) {
    const size_t work = std::max<size_t>(static_cast<size_t>(n) * S, n);
    k_spm_init<<<std::min<size_t>(blocks_for(work, 256), 148 * 16), 256, 0, s>>>(ids, vals, tail, n, S, tau_min);
}

void launch_rng_script(uint32_t kind, uint64_t seed, uint64_t it, uint64_t ant, int derive,
                       const int32_t *ops, const uint64_t *args, uint64_t *out, uint32_t count,
                       cudaStream_t s) {
    k_rng_script<<<1, 1, 0, s>>>(kind, seed, it, ant, derive, ops, args, out, count);
}

void launch_spm_script(uint32_t *ids, double *vals, uint32_t *tail, uint32_t S, double tau_min,
                       double c_l, double c_0, double alpha, double c_g, const uint32_t *ops,
                       const int64_t *lgb, uint32_t count, double *out,
                       unsigned long long *hits_misses, cudaStream_t s) {
    k_spm_script<<<1, 1, 0, s>>>(ids, vals, tail, S, tau_min, c_l, c_0, alpha, c_g, ops, lgb,
                                 count, out, hits_misses);
}

static size_t construct_smem(const DevInstance &I, int wpb) {
    return static_cast<size_t>(wpb) * (32 * sizeof(double) + I.words * sizeof(uint32_t));
}

template <class K>
static void launch_tour_kernel(K kernel, const DevInstance &I, const DevColony &C, bool one_warp,
                               cudaStream_t s) {
    const int threads = one_warp ? 32 : kBlock;
    const int wpb = threads / 32;
    const unsigned grid = one_warp ? 1u : blocks_for(C.m, wpb);
    const size_t smem = construct_smem(I, wpb);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kernel<<<grid, threads, smem, s>>>(I, C);
}

template <class RNG>
static void launch_spm_rng(const DevInstance &I, const DevColony &C, bool one_warp, cudaStream_t s) {
    switch (C.S) {
        case 1: launch_tour_kernel(k_construct_spm<1, RNG>, I, C, one_warp, s); break;
        case 2: launch_tour_kernel(k_construct_spm<2, RNG>, I, C, one_warp, s); break;
        case 4: launch_tour_kernel(k_construct_spm<4, RNG>, I, C, one_warp, s); break;
        case 8: launch_tour_kernel(k_construct_spm<8, RNG>, I, C, one_warp, s); break;
        default: launch_tour_kernel(k_construct_spm<16, RNG>, I, C, one_warp, s); break;
    }
}

void launch_construct(int variant, int rng, const DevInstance &I, const DevColony &C,
                      cudaStream_t s) {
    const bool philox = rng == ACS_RNG_PHILOX;
    switch (variant) {
        case ACS_VARIANT_ATOMIC:
            if (philox) launch_tour_kernel(k_construct_dense<true, Philox>, I, C, false, s);
            else launch_tour_kernel(k_construct_dense<true, Xoshiro>, I, C, false, s);
            break;
        case ACS_VARIANT_RELAXED:
            if (philox) launch_tour_kernel(k_construct_dense<false, Philox>, I, C, false, s);
            else launch_tour_kernel(k_construct_dense<false, Xoshiro>, I, C, false, s);
            break;
        case ACS_VARIANT_SEQ:
            if (philox) launch_tour_kernel(k_construct_dense<false, Philox>, I, C, true, s);
            else launch_tour_kernel(k_construct_dense<false, Xoshiro>, I, C, true, s);
            break;
        case ACS_VARIANT_SPM:
        case ACS_VARIANT_SPM_SEQ:
            if (philox) launch_spm_rng<Philox>(I, C, variant == ACS_VARIANT_SPM_SEQ, s);
            else launch_spm_rng<Xoshiro>(I, C, variant == ACS_VARIANT_SPM_SEQ, s);
            break;
        default: break;
    }
}

size_t deferred_rng_bytes(int rng) {
    return rng == ACS_RNG_PHILOX ? sizeof(Philox) : sizeof(Xoshiro);
}

void launch_deferred_init(int rng, const DevInstance &I, const DevColony &C, const DevDeferred &D,
                          cudaStream_t s) {
    const unsigned grid = blocks_for(C.m, kWarpsPerBlock);
    if (rng == ACS_RNG_PHILOX) k_def_init<Philox><<<grid, kBlock, 0, s>>>(I, C, D);
    else k_def_init<Xoshiro><<<grid, kBlock, 0, s>>>(I, C, D);
}

void launch_deferred_select(int rng, const DevInstance &I, const DevColony &C,
                            const DevDeferred &D, uint32_t step, cudaStream_t s) {
    const unsigned grid = blocks_for(C.m, kWarpsPerBlock);
    if (rng == ACS_RNG_PHILOX) k_def_select<Philox><<<grid, kBlock, 0, s>>>(I, C, D, step);
    else k_def_select<Xoshiro><<<grid, kBlock, 0, s>>>(I, C, D, step);
}

void launch_deferred_apply(const DevInstance &I, const DevColony &C, const DevDeferred &D,
                           cudaStream_t s) {
    k_def_apply<<<blocks_for(C.m, kWarpsPerBlock), kBlock, 0, s>>>(I, C, D);
}

void launch_deferred_close(const DevInstance &I, const DevColony &C, const DevDeferred &D,
                           cudaStream_t s) {
    k_def_close<<<blocks_for(C.m, kWarpsPerBlock), kBlock, 0, s>>>(I, C, D);
}

void launch_epilogue(bool spm, const DevInstance &I, const DevColony &C, const DevBest &B,
                     uint32_t slot, cudaStream_t s) {
    if (spm) k_epilogue<true><<<1, 1024, 0, s>>>(I, C, B, slot);
    else k_epilogue<false><<<1, 1024, 0, s>>>(I, C, B, slot);
}

void launch_adopt_best(const uint32_t *tour, const int64_t *len, const DevInstance &I,
                       const DevBest &B, cudaStream_t s) {
    k_adopt_best<<<1, 256, 0, s>>>(tour, len, I.n, B);
}

__global__ void k_island_pack(const int64_t *best_len, int rank, int64_t *key) {
    *key = (*best_len << 8) | rank;
}
__global__ void k_island_mask(const int64_t *key, int rank, const uint32_t *tour, uint32_t n,
                              uint32_t *x_tour, int64_t *x_len) {
    const bool mine = static_cast<int>(*key & 0xFF) == rank;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        x_tour[i] = mine ? tour[i] : 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) *x_len = *key >> 8;
}

void launch_island_pack(const int64_t *best_len, int rank, int64_t *key, cudaStream_t s) {
    k_island_pack<<<1, 1, 0, s>>>(best_len, rank, key);
}
void launch_island_mask(const int64_t *key, int rank, const uint32_t *best_tour, uint32_t n,
                        uint32_t *x_tour, int64_t *x_len, cudaStream_t s) {
    k_island_mask<<<std::min<unsigned>(blocks_for(n, 256), 64), 256, 0, s>>>(key, rank, best_tour, n, x_tour, x_len);
}

}  // namespace acs_dev
