// acs_device.cuh -- device building blocks shared by every ACS kernel.
//
// Bit-exactness rules: every double op
// that must match the CPU oracle is spelled with an explicit IEEE intrinsic
// (__dmul_rn/__dadd_rn/__dsub_rn/__ddiv_rn/__dsqrt_rn) so nvcc never contracts
// it into a DFMA, regardless of -fmad.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace acs_dev {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kEmpty = 0xffffffffu;  // empty selective slot
constexpr int kLanes = 32;                // candidate slots per row (cl <= 32)

// ---------------------------------------------------------------- distance
// tsp_instance.cpp:49-65 (EUC_2D nint, CEIL_2D, ATT pseudo-Euclidean)
__device__ __forceinline__ int32_t tsplib_distance(int type, double xu, double yu, double xv,
                                                   double yv) {
    const double xd = __dsub_rn(xu, xv);
    const double yd = __dsub_rn(yu, yv);
    const double sq = __dadd_rn(__dmul_rn(xd, xd), __dmul_rn(yd, yd));
    if (type == 0) return static_cast<int32_t>(__dadd_rn(__dsqrt_rn(sq), 0.5));
    if (type == 1) return static_cast<int32_t>(ceil(__dsqrt_rn(sq)));
    const double r = __dsqrt_rn(__ddiv_rn(sq, 10.0));
    const int32_t t = static_cast<int32_t>(__dadd_rn(r, 0.5));
    return (static_cast<double>(t) < r) ? t + 1 : t;
}

// D1 / P2: eta = 1/max(d,1); integral beta by left-to-right repeated multiply
__device__ __forceinline__ double eta_beta(int32_t d, double beta, int beta_int) {
    const double eta = __ddiv_rn(1.0, static_cast<double>(d > 0 ? d : 1));
    if (beta_int >= 0) {
        double e = 1.0;
        for (int i = 0; i < beta_int; ++i) e = __dmul_rn(e, eta);
        return e;
    }
    return pow(eta, beta);
}

// ---------------------------------------------------------------- rng
// xoshiro256** seeded by splitmix64, bit-identical to rng.hpp:16-84.
__host__ __device__ __forceinline__ uint64_t splitmix_next(uint64_t &z) {
    z += 0x9e3779b97f4a7c15ull;
    uint64_t x = z;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

struct Xoshiro {
    uint64_t s0, s1, s2, s3;

    __host__ __device__ __forceinline__ void seed(uint64_t seed) {
        uint64_t z = seed;
        s0 = splitmix_next(z);
        s1 = splitmix_next(z);
        s2 = splitmix_next(z);
        s3 = splitmix_next(z);
        if ((s0 | s1 | s2 | s3) == 0) s0 = 0x9e3779b97f4a7c15ull;
    }
    __host__ __device__ __forceinline__ void derive(uint64_t seed_, uint64_t it, uint64_t ant) {
        uint64_t h = seed_ ^ (it * 0xbf58476d1ce4e5b9ull);
        h = splitmix_next(h);
        h ^= ant * 0x94d049bb133111ebull;
        h = splitmix_next(h);
        seed(h);
    }
    // the next output depends on s1 only: it can be read before the state
    // transition is committed (speculative draws without a state copy)
    __host__ __device__ __forceinline__ uint64_t peek() const {
        const uint64_t x = s1 * 5;
        return ((x << 7) | (x >> 57)) * 9;
    }
    __host__ __device__ __forceinline__ void advance() {
        const uint64_t t = s1 << 17;
        s2 ^= s0;
        s3 ^= s1;
        s1 ^= s2;
        s0 ^= s3;
        s2 ^= t;
        s3 = (s3 << 45) | (s3 >> 19);
    }
    __host__ __device__ __forceinline__ uint64_t next() {
        const uint64_t result = peek();
        advance();
        return result;
    }
};

// Philox4x32-10 (Salmon et al., SC'11): key = seed, counter = (draw, ant, iteration)
struct Philox {
    uint32_t k0, k1, ant, it_lo, it_hi, draw;

    __host__ __device__ __forceinline__ void derive(uint64_t seed_, uint64_t it, uint64_t a) {
        k0 = static_cast<uint32_t>(seed_);
        k1 = static_cast<uint32_t>(seed_ >> 32);
        ant = static_cast<uint32_t>(a);
        it_lo = static_cast<uint32_t>(it);
        it_hi = static_cast<uint32_t>(it >> 32);
        draw = 0;
    }
    __host__ __device__ __forceinline__ uint64_t next() {
        const uint64_t r = peek();
        advance();
        return r;
    }
    __host__ __device__ __forceinline__ void advance() { ++draw; }
    __host__ __device__ __forceinline__ uint64_t peek() const {
        uint32_t c0 = draw, c1 = ant, c2 = it_lo, c3 = it_hi, a = k0, b = k1;
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            if (r) { a += 0x9E3779B9u; b += 0xBB67AE85u; }
            const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
            const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
            const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ a;
            const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ b;
            c1 = static_cast<uint32_t>(p1);
            c3 = static_cast<uint32_t>(p0);
            c0 = n0;
            c2 = n2;
        }
        return static_cast<uint64_t>(c0) | (static_cast<uint64_t>(c1) << 32);
    }
};

// rng.hpp:50-52 and 55-68 on top of either engine
template <class E>
__host__ __device__ __forceinline__ double uniform01(E &e) {
    return static_cast<double>(e.next() >> 11) * 0x1.0p-53;
}
template <class E>
__host__ __device__ __forceinline__ uint64_t uniform_int(E &e, uint64_t bound) {
    uint64_t x = e.next();
    uint64_t lo = x * bound;
    uint64_t hi = mulhi64(x, bound);
    if (lo < bound) {
        const uint64_t threshold = (0 - bound) % bound;
        while (lo < threshold) {
            x = e.next();
            lo = x * bound;
            hi = mulhi64(x, bound);
        }
    }
    return hi;
}

// ---------------------------------------------------------------- memory
// RELAXED contract: torn-free 64-bit accesses at gpu scope.
__device__ __forceinline__ double ld_relaxed(const double *p) {
    uint64_t r;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return __longlong_as_double(static_cast<long long>(r));
}
__device__ __forceinline__ void st_relaxed(double *p, double v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p),
                 "l"(static_cast<uint64_t>(__double_as_longlong(v)))
                 : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t *p) {
    uint32_t r;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t dbits(double x) {
    return static_cast<uint64_t>(__double_as_longlong(x));
}
__device__ __forceinline__ double bitsd(uint64_t x) {
    return __longlong_as_double(static_cast<long long>(x));
}
// affine pheromone rule tau' = c_mul*tau + c_add (P4), never contracted
__device__ __forceinline__ double affine(double tau, double c_mul, double c_add) {
    return __dadd_rn(__dmul_rn(c_mul, tau), c_add);
}

// ---------------------------------------------------------------- warp ops
// argmax over lanes with `valid`, exact on non-negative doubles (their bit
// patterns order like unsigned integers); ties -> lowest lane (D7).
// Returns -1 when no lane is valid.
__device__ __forceinline__ int warp_argmax_pos(double score, bool valid) {
    const uint64_t b = valid ? dbits(score) : 0ull;
    const uint32_t hi = static_cast<uint32_t>(b >> 32);
    const uint32_t lo = static_cast<uint32_t>(b);
    const uint32_t mh = __reduce_max_sync(kFull, hi);
    const bool top = valid && hi == mh;
    const unsigned th = __ballot_sync(kFull, top);
    if ((th & (th - 1)) == 0) return th ? __ffs(th) - 1 : -1;  // unique high word: done
    const uint32_t ml = __reduce_max_sync(kFull, top ? lo : 0u);
    const unsigned win = __ballot_sync(kFull, top && lo == ml);
    return __ffs(win) - 1;
}

// The same argmax (non-negative doubles, ties -> lowest lane) as three
// dependent REDUX ops and no VOTE / FLO / SHFL on the chain (measured on
// B200: REDUX 18 cycles, VOTE 23, BREV+FLO 36, SHFL 32): max of the high
// words, max of the low words among those lanes, then one max over the key
// (31 - lane) << 24 | id, which yields the lowest winning lane and its node
// id together.  `id` < 2^24.  Returns false when no lane is valid.
__device__ __forceinline__ bool warp_argmax_id(double score, bool valid, uint32_t id, int lane, int &pos,
                                               uint32_t &v) {
    const uint64_t b = dbits(score);
    const uint32_t hk = valid ? static_cast<uint32_t>(b >> 32) + 1u : 0u;  // finite: hi + 1 never wraps
    const uint32_t mh = __reduce_max_sync(kFull, hk);
    const bool t1 = valid && hk == mh;
    const uint32_t lo = static_cast<uint32_t>(b);
    const uint32_t ml = __reduce_max_sync(kFull, t1 ? lo : 0u);
    const bool t2 = t1 && lo == ml;
    const uint32_t key = __reduce_max_sync(kFull, t2 ? ((31u - static_cast<uint32_t>(lane)) << 24) | id : 0u);
    pos = 31 - static_cast<int>(key >> 24);
    v = key & 0x00FFFFFFu;
    return mh != 0u;
}

// Roulette (Eq.2, D8, P5): sequential prefix in candidate
// order computed by lane 0 in shared scratch, then one ballot.  Zero weights
// stand for filtered-out (visited) slots: x + 0.0 == x keeps it bit-exact.
__device__ __forceinline__ int warp_roulette_pos(double w, unsigned unvisited_mask, double r,
                                                 double *scratch, int lane) {
    scratch[lane] = w;
    __syncwarp();
    if (lane == 0) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < kLanes; ++i) {
            acc = __dadd_rn(acc, scratch[i]);
            scratch[i] = acc;
        }
    }
    __syncwarp();
    const double prefix = scratch[lane];
    const double total = scratch[kLanes - 1];
    __syncwarp();
    const double thr = __dmul_rn(r, total);
    const unsigned exceed = __ballot_sync(kFull, prefix > thr);
    if (exceed) return __ffs(exceed) - 1;
    const unsigned pos = __ballot_sync(kFull, w > 0.0);
    if (pos) return 31 - __clz(pos);           // rounding left none: last positive
    return __ffs(unvisited_mask) - 1;          // all-zero weights: greedy tie rule
}

// (score, node) argmax with ties -> lowest node id, for the full-scan fallback
__device__ __forceinline__ void warp_argmax_node(double &score, uint32_t &node, bool valid) {
    const uint64_t b = valid ? dbits(score) : 0ull;
    const uint32_t hi = static_cast<uint32_t>(b >> 32);
    const uint32_t lo = static_cast<uint32_t>(b);
    const uint32_t mh = __reduce_max_sync(kFull, hi);
    const uint32_t lo2 = (valid && hi == mh) ? lo : 0u;
    const uint32_t ml = __reduce_max_sync(kFull, lo2);
    const bool top = valid && hi == mh && lo == ml;
    const uint32_t vmin = __reduce_min_sync(kFull, top ? node : 0xffffffffu);
    node = vmin;
    score = bitsd((static_cast<uint64_t>(mh) << 32) | ml);
}

}  // namespace acs_dev
