// acs_common.cuh -- constants and small device helpers shared by the setup
// (k_setup.cu) and colony (k_colony.cu) translation units.
#pragma once

#include <cstdint>

#include "acs_device.cuh"
#include "acs_kernels.cuh"

namespace acs_dev {


#ifndef ACS_BLOCK
#define ACS_BLOCK 64
#endif
constexpr int kBlock = ACS_BLOCK;     // 2 ants per CTA: fine-grained spread over 148 SMs
#ifndef ACS_MAXREGS
#define ACS_MAXREGS 96
#endif
constexpr int kMaxRegs = ACS_MAXREGS;  // 96: 5 warps per SM sub-partition (16K regs each), 20 ants per SM
constexpr int kWarpsPerBlock = kBlock / 32;
constexpr int kDefBlock = 640;        // deferred persistent kernel: 20 warps, one CTA per SM
constexpr uint32_t kIdMask = 0x00FFFFFFu;
constexpr uint32_t kNoMirror = 0xFFu;

__device__ __forceinline__ int32_t dist_of(const DevInstance &I, uint32_t u, uint32_t v,
                                           double xu, double yu) {
    if (I.dist) return __ldg(I.dist + static_cast<size_t>(u) * I.n + v);
    return tsplib_distance(I.type, xu, yu, __ldg(I.xs + v), __ldg(I.ys + v));
}

// eta^beta of distance d: repeated multiply for integral beta (P2), the
// host-built distance table otherwise (DevInstance::eta_d)
__device__ __forceinline__ double eta_beta_i(const DevInstance &I, int32_t d, double beta, int beta_int) {
    if (beta_int >= 0 || !I.eta_d) return eta_beta(d, beta, beta_int);
    const uint32_t k = static_cast<uint32_t>(d > 0 ? d : 0);
    return __ldg(I.eta_d + (k < I.eta_dmax ? k : I.eta_dmax));
}

__device__ __forceinline__ bool visited(const uint32_t *vis, uint32_t v) {
    return (vis[v >> 5] >> (v & 31)) & 1u;
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

// Single-thread record update on global memory (Fig. alg:3):
// hit -> in place, tail untouched; miss -> value from tau_min inserted at
// (tail+1) % S evicting the least-recently inserted.  Relaxed accesses keep
// the RELAXED contract's range invariants under races.
// SPEC selective update of record u with neighbour v (D4-D6):
// hit -> update in place, miss -> insert f(tau_min) at (tail+1) % S
__device__ __forceinline__ bool spm_update_mem(const SpmMem &M, uint32_t u, uint32_t v, double c_mul,
                                               double c_add, double tau_min, double *stored) {
    uint32_t *ids = M.ids(u);
    double *vals = M.vals(u);
    for (uint32_t j = 0; j < M.S; ++j) {
        if (ld_relaxed_u32(ids + j) == v) {
            const double y = affine(ld_relaxed(vals + j), c_mul, c_add);
            st_relaxed(vals + j, y);
            if (stored) *stored = y;
            return true;
        }
    }
    const double y = affine(tau_min, c_mul, c_add);
    const uint32_t t = (ld_relaxed_u32(M.tail(u)) + 1) % M.S;
    st_relaxed_u32(ids + t, v);
    st_relaxed(vals + t, y);
    st_relaxed_u32(M.tail(u), t);
    if (stored) *stored = y;
    return false;
}

__device__ __forceinline__ double spm_read_mem(const SpmMem &M, uint32_t u, uint32_t v, double tau_min) {
    const uint32_t *ids = M.ids(u);
    for (uint32_t j = 0; j < M.S; ++j)
        if (ld_relaxed_u32(ids + j) == v) return ld_relaxed(M.vals(u) + j);
    return tau_min;
}


// SM count of the current device (grid sizing of the grid-stride kernels)
static inline unsigned device_sms() {
    static thread_local int cached_dev = -1;
    static thread_local unsigned cached_sms = 1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != cached_dev) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cached_dev = dev;
        cached_sms = sms > 0 ? static_cast<unsigned>(sms) : 1u;
    }
    return cached_sms;
}

static inline unsigned blocks_for(size_t work, unsigned per) {
    return static_cast<unsigned>((work + per - 1) / per);
}

}  // namespace acs_dev
