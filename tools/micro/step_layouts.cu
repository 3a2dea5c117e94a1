// Minimal construction step (as acs k_step_floor) over different row layouts:
// one warp, dependent chain row(cur) -> visited test -> score -> REDUX argmax
// -> next row; rows L2-resident (the whole region is warmed first).
//   mode 0: 512 B {id,0,eta} row (ld.global.nc.v4) + 256 B trail (ld.relaxed.gpu)   [k_tour_lean]
//   mode 1: 128 B ids (nc) + 256 B fused score (ld.relaxed.gpu)
//   mode 2: 128 B ids (nc) + 256 B fused score (ld.global weak, L1-cacheable)
//   mode 3: 128 B ids (nc) + 256 B fused score (nc)
//   mode 4: 256 B {id, score f32} packed 8 B per lane (ld.relaxed.gpu.v2.u32)
//   mode 5: 512 B row only (nc), score from the row
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/step_layouts tools/micro/step_layouts.cu
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ bool argmax_id(double score, bool valid, uint32_t id, int lane, uint32_t &v) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(score));
    const uint32_t hk = valid ? static_cast<uint32_t>(b >> 32) + 1u : 0u;
    const uint32_t mh = __reduce_max_sync(0xffffffffu, hk);
    const bool t1 = valid && hk == mh;
    const uint32_t ml = __reduce_max_sync(0xffffffffu, t1 ? static_cast<uint32_t>(b) : 0u);
    const bool t2 = t1 && static_cast<uint32_t>(b) == ml;
    const uint32_t key = __reduce_max_sync(0xffffffffu, t2 ? ((31u - lane) << 24) | id : 0u);
    v = key & 0xFFFFFFu;
    return mh != 0;
}
__device__ __forceinline__ double ld_rel(const double *p) {
    uint64_t r;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return __longlong_as_double(static_cast<long long>(r));
}
__device__ __forceinline__ double ld_weak(const double *p) {
    uint64_t r;
    asm volatile("ld.global.b64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return __longlong_as_double(static_cast<long long>(r));
}

template <int M>
__global__ void k(const uint4 *rows, const double *tau, const uint32_t *ids, const double *sc, const uint2 *pk,
                  uint32_t nrows, uint32_t steps, uint32_t *sink) {
    __shared__ uint32_t vis[1 << 11];
    const int lane = threadIdx.x;
    const uint32_t words = (nrows + 31) / 32;
    uint32_t cur = 0;
    for (uint32_t s = 0; s < steps; ++s) {
        if (s % 2048 == 0) {
            __syncwarp();
            for (uint32_t w = lane; w < words; w += 32) vis[w] = 0;
            __syncwarp();
        }
        const size_t ri = static_cast<size_t>(cur) * 32 + lane;
        uint32_t c = 0;
        double score = 0.0;
        if (M == 0) {
            const uint4 e = __ldg(rows + ri);
            const double t = ld_rel(tau + ri);
            c = e.x;
            score = __dmul_rn(t, __hiloint2double(e.w, e.z));
        }
        if (M == 1) { c = __ldg(ids + ri); score = ld_rel(sc + ri); }
        if (M == 2) { c = __ldg(ids + ri); score = ld_weak(sc + ri); }
        if (M == 3) { c = __ldg(ids + ri); score = __ldg(sc + ri); }
        if (M == 4) {
            uint32_t a, b;
            asm volatile("ld.relaxed.gpu.global.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "l"(pk + ri) : "memory");
            c = a;
            score = static_cast<double>(__uint_as_float(b));
        }
        if (M == 5) {
            const uint4 e = __ldg(rows + ri);
            c = e.x;
            score = __hiloint2double(e.w, e.z);
        }
        const bool unv = !((vis[c >> 5] >> (c & 31)) & 1u);
        uint32_t v;
        if (!argmax_id(score, unv, c, lane, v)) v = (cur + 1) % nrows;
        vis[v >> 5] |= 1u << (v & 31);
        cur = v;
        __syncwarp();
    }
    if (lane == 0) *sink = cur;
}

__global__ void warm(const uint4 *p, size_t n, uint32_t *sink) {
    uint32_t a = 0;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint4 v = __ldcg(p + i);
        a ^= v.x ^ v.w;
    }
    if (a == 0x12345u) *sink = a;
}

int main() {
    const uint32_t nrows = 65536, steps = 100000;
    const size_t E = static_cast<size_t>(nrows) * 32;
    std::vector<uint4> rows(E);
    std::vector<double> tau(E, 1.0), sc(E);
    std::vector<uint32_t> ids(E);
    std::vector<uint2> pk(E);
    uint64_t x = 88172645463325252ull;
    for (size_t i = 0; i < E; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        const uint32_t r = static_cast<uint32_t>(i / 32), id = static_cast<uint32_t>((r + 1 + x % (nrows - 1)) % nrows);
        const double eta = 1.0 / static_cast<double>(1 + (x >> 20) % 1000);
        uint64_t b;
        std::memcpy(&b, &eta, 8);
        rows[i] = make_uint4(id, 0, static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32));
        ids[i] = id;
        sc[i] = eta;
        const float f = static_cast<float>(eta);
        uint32_t fb;
        std::memcpy(&fb, &f, 4);
        pk[i] = make_uint2(id, fb);
    }
    uint4 *dr; double *dt, *ds; uint32_t *di, *sink; uint2 *dp;
    cudaMalloc(&dr, E * 16); cudaMalloc(&dt, E * 8); cudaMalloc(&ds, E * 8); cudaMalloc(&di, E * 4);
    cudaMalloc(&dp, E * 8); cudaMalloc(&sink, 4);
    cudaMemcpy(dr, rows.data(), E * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, tau.data(), E * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(ds, sc.data(), E * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(di, ids.data(), E * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, pk.data(), E * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[] = {"512B row(nc)+256B tau(relaxed) [lean]", "128B ids(nc)+256B score(relaxed)",
                           "128B ids(nc)+256B score(weak/L1)", "128B ids(nc)+256B score(nc)",
                           "256B {id,f32}(relaxed.v2)", "512B row only (nc)"};
    for (int m = 0; m < 6; ++m) {
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            warm<<<592, 512>>>(dr, E, sink);
            warm<<<592, 512>>>(reinterpret_cast<uint4 *>(dt), E / 2, sink);
            warm<<<592, 512>>>(reinterpret_cast<uint4 *>(ds), E / 2, sink);
            warm<<<592, 512>>>(reinterpret_cast<uint4 *>(di), E / 4, sink);
            warm<<<592, 512>>>(reinterpret_cast<uint4 *>(dp), E / 2, sink);
            cudaEventRecord(e0);
            switch (m) {
                case 0: k<0><<<1, 32>>>(dr, dt, di, ds, dp, nrows, steps, sink); break;
                case 1: k<1><<<1, 32>>>(dr, dt, di, ds, dp, nrows, steps, sink); break;
                case 2: k<2><<<1, 32>>>(dr, dt, di, ds, dp, nrows, steps, sink); break;
                case 3: k<3><<<1, 32>>>(dr, dt, di, ds, dp, nrows, steps, sink); break;
                case 4: k<4><<<1, 32>>>(dr, dt, di, ds, dp, nrows, steps, sink); break;
                default: k<5><<<1, 32>>>(dr, dt, di, ds, dp, nrows, steps, sink); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("%-42s %7.1f ns/step\n", names[m], best * 1e6 / steps);
    }
    return 0;
}
