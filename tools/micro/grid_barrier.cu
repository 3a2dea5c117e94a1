// Micro-benchmark: cost of one grid-wide barrier in a cooperative persistent
// kernel on B200 (148 CTAs x 640 threads, the deferred variant's shape).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/grid_barrier tools/micro/grid_barrier.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
namespace cg = cooperative_groups;

constexpr unsigned kGroups = 8;

__device__ __forceinline__ void sync_two_level(unsigned *bar, unsigned nblocks, int sleep_ns) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar;
        const unsigned g = *gen;
        const unsigned grp = blockIdx.x % kGroups;
        const unsigned members = nblocks / kGroups + (grp < nblocks % kGroups ? 1u : 0u);
        const unsigned groups = nblocks < kGroups ? nblocks : kGroups;
        unsigned *gcount = bar + 32 * (1 + grp);
        unsigned *root = bar + 32 * (1 + kGroups);
        __threadfence();
        bool release = false;
        if (atomicAdd(gcount, 1u) == members - 1) {
            *gcount = 0;
            if (atomicAdd(root, 1u) == groups - 1) { *root = 0; release = true; }
        }
        if (release) { __threadfence(); atomicAdd(bar, 1u); }
        else { while (*gen == g) { if (sleep_ns) __nanosleep(sleep_ns); } }
        __threadfence();
    }
    __syncthreads();
}

// flat: one counter, generation bit flip (sense reversal)
__device__ __forceinline__ void sync_flat(unsigned *bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar + 32, 1u) == nblocks - 1) { bar[32] = 0; __threadfence(); atomicAdd(bar, 1u); }
        else { while (*gen == g) {} }
        __threadfence();
    }
    __syncthreads();
}

// acquire/release flavoured: red.release on arrival, ld.acquire polling
__device__ __forceinline__ void sync_acqrel(unsigned *bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar));
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar + 32) : "memory");
        if (old == nblocks - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar + 32) : "memory");
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        } else {
            unsigned cur;
            do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory"); } while (cur == g);
        }
    }
    __syncthreads();
}

// monotonic counter: arrival is a non-returning red.release (no round trip),
// every CTA polls with ld.acquire until the count reaches this generation's
// target (the counter is never reset: target = (generation + 1) * nblocks)
__device__ __forceinline__ void sync_mono(unsigned *bar, unsigned nblocks, unsigned &target) {
    __syncthreads();
    target += nblocks;
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 64) : "memory");
        unsigned cur, spins = 0;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 64) : "memory"); }
        while (static_cast<int>(cur - target) < 0 && ++spins < (1u << 24));
        if (spins >= (1u << 24)) bar[96] = 1;  // watchdog: report instead of hanging
    }
    __syncthreads();
}

__global__ void k_bar(unsigned *bar, int mode, int iters, int sleep_ns) {
    cg::grid_group grid = cg::this_grid();
    unsigned target = 0;
    if (mode == 4) {  // resume from the counter's current generation
        target = *reinterpret_cast<volatile unsigned *>(bar + 64);
        target -= target % gridDim.x;
        grid.sync();
    }
    for (int i = 0; i < iters; ++i) {
        if (mode == 4) { sync_mono(bar, gridDim.x, target); continue; }
        if (mode == 0) sync_two_level(bar, gridDim.x, sleep_ns);
        else if (mode == 1) sync_flat(bar, gridDim.x);
        else if (mode == 2) sync_acqrel(bar, gridDim.x);
        else grid.sync();
    }
}

int main(int argc, char **argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int mode_lo = argc > 1 ? atoi(argv[1]) : 0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *bar;
    cudaMalloc(&bar, 4096);
    cudaMemset(bar, 0, 4096);
    const int iters = 4784;
    const char *names[] = {"two-level nanosleep(8)", "flat spin", "flat acq_rel", "cg::grid.sync", "mono red+poll"};
    for (int blk : {640, 128}) {
        for (int mode = mode_lo; mode < 5; ++mode) {
            for (int sl : {8, 0}) {
                if (mode != 0 && sl == 0) continue;
                int grid = sms;
                void *args[] = {&bar, &mode, (void *)&iters, &sl};
                cudaEvent_t a, b;
                cudaEventCreate(&a); cudaEventCreate(&b);
                cudaLaunchCooperativeKernel((void *)k_bar, grid, blk, args, 0, 0);  // warm
                cudaEventRecord(a);
                cudaLaunchCooperativeKernel((void *)k_bar, grid, blk, args, 0, 0);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                unsigned wd = 0;
                cudaMemcpy(&wd, bar + 96, 4, cudaMemcpyDeviceToHost);
                if (wd) printf("watchdog fired\n");
                printf("block %4d %-24s sleep %d: %.3f us per barrier (%s)\n", blk, names[mode], mode ? -1 : sl,
                       ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}
