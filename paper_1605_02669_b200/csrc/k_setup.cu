// k_setup.cu -- setup-path kernels of the ACS hot path (sm_100a):
//   K1 k_distance_table   tsp_instance.cpp:23-47 dist_table_ (n <= 4096)
//   K2 k_topk             tsp_instance.cpp:219-252 build_candidates (bit-exact)
//      k_build_rows       packed candidate rows: id | mirror, distance, eta^beta
//      k_eta_table        eta^beta of every edge (fallback scan operand, n <= 4096)
//      k_nn_tour_cand     tsp_instance.cpp:254-280 nn_tour_length -> tau0 (candidate-list probe + full scan)
//   K6 k_tour_lengths     tsp_instance.cpp:67-78 tour_length (validation / eval)
//   plus device RNG and selective-store op scripts used by the parity tests.
#include <algorithm>
#include <cstdlib>
#include <climits>

#include "../../include/acs_gpu.h"
#include "acs_common.cuh"

namespace acs_dev {

// ============================================================ setup kernels

__global__ void k_distance_table(DevInstance I, int32_t *out) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t u = blockIdx.y;
    if (v >= I.n) return;
    out[static_cast<size_t>(u) * I.n + v] =
        tsplib_distance(I.type, __ldg(I.xs + u), __ldg(I.ys + u), __ldg(I.xs + v), __ldg(I.ys + v));
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

// K2': the 32 smallest keys of node u STRICTLY above lower[u] -- successive
// 32-slices of u's distance order (the extended neighbour list of the exact
// pruned fallback scan).  Same warp merge as k_topk.
__global__ void __launch_bounds__(kBlock) k_topk_after(DevInstance I, const uint64_t *lower,
                                                      uint64_t *keys_out) {
    const int lane = threadIdx.x & 31;
    const uint32_t u = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (u >= I.n) return;
    const double xu = __ldg(I.xs + u), yu = __ldg(I.ys + u);
    const uint64_t lo = lower[u];
    uint64_t top = ~0ull;
    for (uint32_t base = 0; base < I.n; base += 32) {
        const uint32_t v = base + lane;
        uint64_t key = ~0ull;
        if (v < I.n && v != u) {
            const int32_t d = tsplib_distance(I.type, xu, yu, __ldg(I.xs + v), __ldg(I.ys + v));
            key = (static_cast<uint64_t>(static_cast<uint32_t>(d)) << 32) | v;
            if (key <= lo) key = ~0ull;
        }
        const uint64_t thr = shfl_u64(top, 31);
        if (!__any_sync(kFull, key < thr)) continue;
        key = warp_sort_u64(key, lane);
        const uint64_t rev = shfl_u64(key, 31 - lane);
        top = top < rev ? top : rev;
        top = warp_merge_u64(top, lane);
    }
    keys_out[static_cast<size_t>(u) * 32 + lane] = top;
}

// key of the last candidate of every node: the lower bound of the first slice
__global__ void k_last_cand_key(DevInstance I, const uint32_t *cand, uint32_t L, uint64_t *lower) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= I.n) return;
    const uint32_t c = cand[static_cast<size_t>(u) * L + L - 1];
    const int32_t d = tsplib_distance(I.type, I.xs[u], I.ys[u], I.xs[c], I.ys[c]);
    lower[u] = (static_cast<uint64_t>(static_cast<uint32_t>(d)) << 32) | c;
}

// slice j of the extended rows {id | mirror<<24, d, eta^beta lo, hi} (kEmpty
// past the end; mirror = u's slot in v's candidate list, as in the packed
// rows, so a fallback settled here needs no extra row load); also advances
// lower[u] to the slice's last key
__global__ void k_ext_rows(DevInstance I, const uint32_t *cand, uint32_t L, const uint64_t *keys, uint32_t j,
                           uint32_t ext_len, double beta, int beta_int, uint4 *ext, uint64_t *lower) {
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<size_t>(I.n) * 32) return;
    const uint32_t u = static_cast<uint32_t>(idx >> 5), p = static_cast<uint32_t>(idx & 31);
    const uint64_t key = keys[idx];
    uint4 el = make_uint4(kEmpty, 0u, 0u, 0u);
    if (key != ~0ull) {
        const int32_t d = static_cast<int32_t>(key >> 32);
        const uint64_t b = dbits(eta_beta_i(I, d, beta, beta_int));
        const uint32_t v = static_cast<uint32_t>(key);
        uint32_t mirror = kNoMirror;
        for (uint32_t q = 0; q < L; ++q)
            if (cand[static_cast<size_t>(v) * L + q] == u) { mirror = q; break; }
        el = make_uint4(v | (mirror << 24), static_cast<uint32_t>(d), static_cast<uint32_t>(b),
                        static_cast<uint32_t>(b >> 32));
    }
    ext[static_cast<size_t>(u) * ext_len + j * 32 + p] = el;
    if (p == 31) lower[u] = key;
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
        const double eb = eta_beta_i(I, d, beta, beta_int);
        uint32_t mirror = kNoMirror;
        for (uint32_t q = 0; q < L; ++q)
            if (cand[static_cast<size_t>(c) * L + q] == u) { mirror = q; break; }
        const uint64_t b = dbits(eb);
        el = make_uint4(c | (mirror << 24), static_cast<uint32_t>(d), static_cast<uint32_t>(b),
                        static_cast<uint32_t>(b >> 32));
    }
    rows[idx] = el;
}

// nn_tour_length with the candidate lists at hand (colony setup): one warp.
// The lists are sorted by (d, id) (cpp:241-245), so the first unvisited entry
// of cur's list is the nearest unvisited node with ties -> lowest id, exactly
// the reference's full-scan pick (cpp:254-280); only when the whole list is
// visited does the warp scan all n nodes.  ~2% of steps scan, so the setup
// drops from n block-wide scans to n list probes.
__global__ void __launch_bounds__(32) k_nn_tour_cand(DevInstance I, const uint32_t *cand, uint32_t L,
                                                     uint32_t start, int64_t *out, const uint4 *ext,
                                                     uint32_t ext_len) {
    extern __shared__ uint32_t vis[];
    const int lane = threadIdx.x & 31;
    for (uint32_t i = lane; i < I.words; i += 32) vis[i] = 0;
    __syncwarp();
    if (lane == 0) vis[start >> 5] |= 1u << (start & 31);
    __syncwarp();
    uint32_t cur = start;
    long long total = 0;
    for (uint32_t step = 1; step < I.n; ++step) {
        const double xc = __ldg(I.xs + cur), yc = __ldg(I.ys + cur);
        const bool in = static_cast<uint32_t>(lane) < L;
        const uint32_t c = in ? __ldg(cand + static_cast<size_t>(cur) * L + lane) : 0u;
        const unsigned um = __ballot_sync(kFull, in && !visited(vis, c));
        uint32_t next;
        int32_t d;
        bool found = um != 0u;
        if (found) {
            next = __shfl_sync(kFull, c, __ffs(um) - 1);
            d = dist_of(I, cur, next, xc, yc);
        }
        // every candidate visited: the next-nearest rows (sorted by (d, id),
        // like the full scan's key) hold the answer when any of them is unvisited
        for (uint32_t base = 0; !found && base < ext_len; base += 32) {
            const uint4 q = __ldg(ext + static_cast<size_t>(cur) * ext_len + base + lane);
            const bool ok = q.x != kEmpty;
            const uint32_t id = q.x & kIdMask;
            const unsigned ue = __ballot_sync(kFull, ok && !visited(vis, id));
            if (ue) {
                const int src = __ffs(ue) - 1;
                next = __shfl_sync(kFull, id, src);
                d = static_cast<int32_t>(__shfl_sync(kFull, q.y, src));
                found = true;
            } else if (__any_sync(kFull, !ok)) {
                break;  // the list ended
            }
        }
        if (!found) {
            uint64_t best = ~0ull;
            for (uint32_t v = lane; v < I.n; v += 32) {
                if (visited(vis, v)) continue;
                const int32_t dv = dist_of(I, cur, v, xc, yc);
                const uint64_t key = (static_cast<uint64_t>(static_cast<uint32_t>(dv)) << 32) | v;
                best = key < best ? key : best;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const uint64_t p = shfl_xor_u64(best, o);
                best = p < best ? p : best;
            }
            next = static_cast<uint32_t>(best);
            d = static_cast<int32_t>(best >> 32);
        }
        __syncwarp();
        if (lane == 0) vis[next >> 5] |= 1u << (next & 31);
        __syncwarp();
        total += d;
        cur = next;
    }
    if (lane == 0) *out = total + dist_of(I, cur, start, __ldg(I.xs + cur), __ldg(I.ys + cur));
}

// The same NN tour with the candidate lists staged in shared memory as 16-bit
// ids (n < 65536, n*L*2 B within the CTA's shared memory): the walk's
// dependent load per step is then an LDS instead of an L2 round trip.  The
// route is kept in shared memory and the length summed afterwards by the
// whole CTA, so no distance load sits in the walk either.  Same answer as
// k_nn_tour_cand (candidates first, then the next-nearest rows, then the full
// scan; ties -> lowest id).
__global__ void __launch_bounds__(1024) k_nn_tour_smem(DevInstance I, const uint32_t *cand, uint32_t L,
                                                      uint32_t start, int64_t *out, const uint4 *ext,
                                                      uint32_t ext_len) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t n = I.n;
    uint32_t *vis = reinterpret_cast<uint32_t *>(smem);
    uint32_t *route = vis + I.words;
    uint16_t *c16 = reinterpret_cast<uint16_t *>(route + n);
    __shared__ long long part[32];
    for (uint32_t i = threadIdx.x; i < I.words; i += blockDim.x) vis[i] = 0;
    for (size_t i = threadIdx.x; i < static_cast<size_t>(n) * L; i += blockDim.x) c16[i] = static_cast<uint16_t>(cand[i]);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        if (lane == 0) {
            vis[start >> 5] |= 1u << (start & 31);
            route[0] = start;
        }
        __syncwarp();
        uint32_t cur = start;
        for (uint32_t step = 1; step < n; ++step) {
            const bool in = static_cast<uint32_t>(lane) < L;
            const uint32_t c = in ? c16[static_cast<size_t>(cur) * L + lane] : 0u;
            const unsigned um = __ballot_sync(kFull, in && !visited(vis, c));
            uint32_t next = 0;
            bool found = um != 0u;
            if (found) next = __shfl_sync(kFull, c, __ffs(um) - 1);
            for (uint32_t base = 0; !found && base < ext_len; base += 32) {
                const uint4 q = __ldg(ext + static_cast<size_t>(cur) * ext_len + base + lane);
                const bool ok = q.x != kEmpty;
                const uint32_t id = q.x & kIdMask;
                const unsigned ue = __ballot_sync(kFull, ok && !visited(vis, id));
                if (ue) {
                    next = __shfl_sync(kFull, id, __ffs(ue) - 1);
                    found = true;
                } else if (__any_sync(kFull, !ok)) {
                    break;
                }
            }
            if (!found) {
                const double xc = __ldg(I.xs + cur), yc = __ldg(I.ys + cur);
                uint64_t best = ~0ull;
                for (uint32_t v = lane; v < n; v += 32) {
                    if (visited(vis, v)) continue;
                    const int32_t dv = dist_of(I, cur, v, xc, yc);
                    const uint64_t key = (static_cast<uint64_t>(static_cast<uint32_t>(dv)) << 32) | v;
                    best = key < best ? key : best;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const uint64_t p = shfl_xor_u64(best, o);
                    best = p < best ? p : best;
                }
                next = static_cast<uint32_t>(best);
            }
            __syncwarp();
            if (lane == 0) {
                vis[next >> 5] |= 1u << (next & 31);
                route[step] = next;
            }
            __syncwarp();
            cur = next;
        }
    }
    __syncthreads();
    // closed-tour length, every thread a share of the edges
    long long acc = 0;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t u = route[i], v = route[i + 1 == n ? 0 : i + 1];
        acc += dist_of(I, u, v, __ldg(I.xs + u), __ldg(I.ys + u));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += static_cast<long long>(shfl_xor_u64(static_cast<uint64_t>(acc), o));
    if (lane == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) t += part[w];
        *out = t;
    }
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

__global__ void k_spm_init(SpmMem M, uint32_t n, double tau_min) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
         i < static_cast<size_t>(n) * M.S; i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint32_t u = static_cast<uint32_t>(i / M.S), j = static_cast<uint32_t>(i % M.S);
        M.ids(u)[j] = kEmpty;
        M.vals(u)[j] = tau_min;
        if (j == 0) *M.tail(u) = M.S - 1;  // D5: first insertion lands in slot 0
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


__global__ void k_eta_table(DevInstance I, double beta, int beta_int, double *out) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t u = blockIdx.y;
    if (v >= I.n) return;
    const int32_t d = tsplib_distance(I.type, __ldg(I.xs + u), __ldg(I.ys + u), __ldg(I.xs + v),
                                      __ldg(I.ys + v));
    out[static_cast<size_t>(u) * I.n + v] = eta_beta_i(I, d, beta, beta_int);
}

__global__ void k_spm_script(SpmMem M, double tau_min, double c_l, double c_0, double alpha, double c_g,
                             const uint32_t *ops, const int64_t *lgb, uint32_t count, double *out,
                             unsigned long long *hm) {
    for (uint32_t i = 0; i < count; ++i) {
        const uint32_t u = ops[3 * i], v = ops[3 * i + 1], rule = ops[3 * i + 2];
        if (rule == 2) {
            out[i] = spm_read_mem(M, u, v, tau_min);
            continue;
        }
        double cm = c_l, ca = c_0;
        if (rule == 1) {
            cm = c_g;
            ca = __dmul_rn(alpha, __ddiv_rn(1.0, static_cast<double>(lgb[i])));
        }
        const bool hit = spm_update_mem(M, u, v, cm, ca, tau_min, &out[i]);
        hm[hit ? 0 : 1] += 1;
    }
}


// ============================================================ launchers

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


void launch_nn_tour_cand(const DevInstance &I, const uint32_t *cand, uint32_t L, uint32_t start, int64_t *out,
                         cudaStream_t s, const uint4 *ext, uint32_t ext_len) {
    const size_t smem = static_cast<size_t>(I.words) * 4 + static_cast<size_t>(I.n) * 4 +
                        static_cast<size_t>(I.n) * L * sizeof(uint16_t);
    if (I.n < 65536 && smem <= 200 * 1024 && !std::getenv("ACS_NN_GLOBAL")) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_nn_tour_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        k_nn_tour_smem<<<1, 1024, smem, s>>>(I, cand, L, start, out, ext, ext_len);
        return;
    }
    k_nn_tour_cand<<<1, 32, I.words * sizeof(uint32_t), s>>>(I, cand, L, start, out, ext, ext_len);
}

void launch_tour_lengths(const DevInstance &I, const uint32_t *routes, uint32_t m, int64_t *out,
                         cudaStream_t s) {
    k_tour_lengths<<<blocks_for(m, 8), 256, 0, s>>>(I, routes, m, out);
}

void launch_fill(double *p, size_t count, double value, cudaStream_t s) {
    k_fill<<<std::min<size_t>(blocks_for(count, 256), static_cast<size_t>(device_sms()) * 16), 256, 0, s>>>(p, count, value);
}

void launch_spm_init(const SpmMem &M, uint32_t n, double tau_min, cudaStream_t s) {
    const size_t work = static_cast<size_t>(n) * M.S;
    k_spm_init<<<std::min<size_t>(blocks_for(work, 256), static_cast<size_t>(device_sms()) * 16), 256, 0, s>>>(M, n, tau_min);
}

void launch_rng_script(uint32_t kind, uint64_t seed, uint64_t it, uint64_t ant, int derive,
                       const int32_t *ops, const uint64_t *args, uint64_t *out, uint32_t count,
                       cudaStream_t s) {
    k_rng_script<<<1, 1, 0, s>>>(kind, seed, it, ant, derive, ops, args, out, count);
}

void launch_spm_script(const SpmMem &M, double tau_min, double c_l, double c_0, double alpha, double c_g,
                       const uint32_t *ops, const int64_t *lgb, uint32_t count, double *out,
                       unsigned long long *hits_misses, cudaStream_t s) {
    k_spm_script<<<1, 1, 0, s>>>(M, tau_min, c_l, c_0, alpha, c_g, ops, lgb, count, out, hits_misses);
}

void launch_ext_rows(const DevInstance &I, const uint32_t *cand, uint32_t L, uint32_t ext_len,
                     double beta, int beta_int, uint64_t *scratch_keys, uint64_t *scratch_lower,
                     uint4 *ext, cudaStream_t s) {
    k_last_cand_key<<<blocks_for(I.n, 256), 256, 0, s>>>(I, cand, L, scratch_lower);
    for (uint32_t j = 0; j * 32 < ext_len; ++j) {
        k_topk_after<<<blocks_for(I.n, kWarpsPerBlock), kBlock, 0, s>>>(I, scratch_lower, scratch_keys);
        k_ext_rows<<<blocks_for(static_cast<size_t>(I.n) * 32, 256), 256, 0, s>>>(
            I, cand, L, scratch_keys, j, ext_len, beta, beta_int, ext, scratch_lower);
    }
}

void launch_eta_table(const DevInstance &I, double beta, int beta_int, double *out,
                      cudaStream_t s) {
    dim3 grid(blocks_for(I.n, 256), I.n);
    k_eta_table<<<grid, 256, 0, s>>>(I, beta, beta_int, out);
}


// ------------------------------------------------------------ L2 read probe
// Streaming 16-byte reads (ld.global.cg: L2, not L1) over an L2-resident
// buffer, grid-stride, persistent grid; the xor keeps the loads alive.
__global__ void k_l2_read(const uint4 *__restrict__ p, size_t count, uint32_t reps, uint32_t *sink) {
    uint32_t acc = 0;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (uint32_t r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count; i += stride) {
            const uint4 v = __ldcg(p + i);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x9E3779B9u) *sink = acc;  // practically never taken
}

void launch_l2_read(const uint4 *p, size_t count, uint32_t reps, uint32_t *sink, int sms, cudaStream_t s) {
    k_l2_read<<<sms * 4, 512, 0, s>>>(p, count, reps, sink);
}

}  // namespace acs_dev
