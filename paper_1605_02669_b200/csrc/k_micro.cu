// k_micro.cu -- hardware floors for the construction roofline (sm_100a).
//
// The construction kernels are a dependent chain per ant: row(cur) -> 32
// scores -> argmax -> row(v).  Two microbenchmarks give the absolute floor of
// one such step on this GPU, independent of the ACS kernels themselves:
//
//   k_l2_chase    one thread, pointer chase through a random cycle of 128 B
//                 lines of an L2-resident (not L1-resident) buffer,
//                 ld.global.cg: L2 load-to-use latency.
//   k_step_floor  one warp, the minimal selection step: one coalesced 512 B
//                 row load {id, eta^beta} + one 256 B trail load (the two
//                 loads every construction step issues), the shared-memory
//                 visited test, the score multiply, the exact warp argmax
//                 with the winner's id (warp_argmax_id: three REDUX), the visited
//                 update -- and the next row is the winner's.  No RNG, no
//                 bookkeeping, no pheromone update: what no implementation of
//                 a warp-per-ant step over L2-resident rows can undercut.
#include <cstdint>

#include "acs_common.cuh"

namespace acs_dev {

__global__ void k_l2_chase(const uint32_t *__restrict__ next, uint32_t steps, uint32_t start, uint32_t *sink) {
    uint32_t i = start;
    for (uint32_t s = 0; s < steps; ++s) i = __ldcg(next + static_cast<size_t>(i) * 32);
    *sink = i;
}

// rows: nrows x 32 uint4 {id, 0, eta lo, eta hi}; tau: nrows x 32 f64
__global__ void k_step_floor(const uint4 *__restrict__ rows, const double *tau, uint32_t nrows, uint32_t steps,
                             uint32_t tour, uint32_t *sink) {
    extern __shared__ uint32_t vis[];
    const int lane = threadIdx.x & 31;
    const uint32_t words = (nrows + 31) / 32;
    uint32_t cur = 0;
    for (uint32_t s = 0; s < steps; ++s) {
        if (s % tour == 0) {  // a new "tour": clear the visited set
            __syncwarp();
            for (uint32_t w = lane; w < words; w += 32) vis[w] = 0;
            __syncwarp();
        }
        const size_t ri = static_cast<size_t>(cur) * 32 + lane;
        const uint4 el = __ldg(rows + ri);
        const double t = ld_relaxed(tau + ri);
        const uint32_t c = el.x;
        const bool unv = !visited(vis, c);
        const double score = unv ? __dmul_rn(t, __hiloint2double(static_cast<int>(el.w), static_cast<int>(el.z))) : 0.0;
        int pos;
        uint32_t v;
        if (!warp_argmax_id(score, unv, c, lane, pos, v)) v = (cur + 1) % nrows;  // all visited (rare)
        vis[v >> 5] |= 1u << (v & 31);
        cur = v;
        __syncwarp();
    }
    if (lane == 0) *sink = cur;
}

void launch_l2_chase(const uint32_t *next, uint32_t steps, uint32_t start, uint32_t *sink, cudaStream_t s) {
    k_l2_chase<<<1, 1, 0, s>>>(next, steps, start, sink);
}

void launch_step_floor(const uint4 *rows, const double *tau, uint32_t nrows, uint32_t steps, uint32_t tour,
                       uint32_t *sink, cudaStream_t s) {
    k_step_floor<<<1, 32, ((nrows + 31) / 32) * sizeof(uint32_t), s>>>(rows, tau, nrows, steps, tour, sink);
}

}  // namespace acs_dev
