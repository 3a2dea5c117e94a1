// Dependent-chain latency (cycles) of the warp ops on the construction
// chain: SHFL, VOTE (ballot), REDUX.MAX, DMUL, DADD, LDS, FLO (ffs), and a
// uniform branch.  One warp, clock64 around 1024 dependent repetitions.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/warp_op_latency tools/micro/warp_op_latency.cu
#include <cstdio>
#include <cstdint>

#define REPS 1024

__global__ void k(unsigned long long *out, uint32_t seed, double dseed) {
    __shared__ uint32_t sm[64];
    const int lane = threadIdx.x;
    sm[lane] = lane ^ seed;
    sm[lane + 32] = lane;
    __syncwarp();
    unsigned long long t0, t1;
    uint32_t x = seed + lane;
    double d = dseed;
    int i = 0;
#define CHAIN(name, stmt)                                        \
    t0 = clock64();                                               \
    for (i = 0; i < REPS; ++i) { stmt; }                          \
    t1 = clock64();                                               \
    if (lane == 0) out[name] = t1 - t0;
    CHAIN(0, x = __shfl_sync(0xffffffffu, x, x & 31))
    CHAIN(1, x = __ballot_sync(0xffffffffu, x & 1) + lane)
    CHAIN(2, x = __reduce_max_sync(0xffffffffu, x) + lane)
    CHAIN(3, d = __dmul_rn(d, 1.0000001))
    CHAIN(4, d = __dadd_rn(d, 1.0000001))
    CHAIN(5, x = sm[x & 63])
    CHAIN(6, x = __ffs(x) + lane)
    CHAIN(7, x = (x + 1) & 63)
    CHAIN(8, { unsigned m = __ballot_sync(0xffffffffu, x & 1); x = __ffs(m) + lane; x = __shfl_sync(0xffffffffu, x, x & 31); })
    CHAIN(9, { x = __reduce_max_sync(0xffffffffu, x); unsigned m = __ballot_sync(0xffffffffu, x == (uint32_t)lane); x = (m & (m - 1)) ? x + 1 : x + 2; })
    if (x == 12345 && d == 1.0) out[15] = x;
}

int main() {
    unsigned long long *d, h[16] = {};
    cudaMalloc(&d, sizeof(h));
    cudaMemset(d, 0, sizeof(h));
    for (int r = 0; r < 2; ++r) k<<<1, 32>>>(d, 7u, 1.5);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const char *names[] = {"SHFL.IDX", "VOTE.ANY+IADD", "REDUX.MAX+IADD", "DMUL", "DADD", "LDS",
                           "FLO(ffs)+IADD", "IADD+LOP", "VOTE+FLO+SHFL", "REDUX+VOTE+branchy"};
    for (int i = 0; i < 10; ++i) printf("%-22s %6.1f cycles/iter\n", names[i], (double)h[i] / REPS);
    return 0;
}
