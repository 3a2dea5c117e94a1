// include/acs/rng_stream.hpp -- acs::RngStream, the reproducible per-ant
// stream of the reference (rng.hpp:16-84: xoshiro256** seeded through
// splitmix64, derive(seed, iteration, ant), uniform01 on the top 53 bits,
// Lemire's unbiased uniform_int).  Header-only and usable from host code;
// the kernels use the identical engine in csrc/acs_device.cuh, and the two
// are checked bit-for-bit against the reference in tests/.
#pragma once

#include <cstdint>

namespace acs {

class RngStream {
public:
    RngStream() : RngStream(0) {}

    explicit RngStream(uint64_t seed) {
        uint64_t z = seed;
        for (uint64_t &w : s_) w = mix(z);
        if ((s_[0] | s_[1] | s_[2] | s_[3]) == 0) s_[0] = kGolden;
    }

    static RngStream derive(uint64_t seed, uint64_t iteration, uint64_t ant) {
        uint64_t h = seed ^ (iteration * kMulA);
        h = mix(h);
        h ^= ant * kMulB;
        return RngStream(mix(h));
    }

    uint64_t next_u64() {
        const uint64_t x = s_[1] * 5;
        const uint64_t out = ((x << 7) | (x >> 57)) * 9;
        const uint64_t t = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= t;
        s_[3] = (s_[3] << 45) | (s_[3] >> 19);
        return out;
    }

    // [0, 1), never 1.0
    double uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

    // unbiased [0, bound), bound >= 1
    uint64_t uniform_int(uint64_t bound) {
        unsigned __int128 prod = static_cast<unsigned __int128>(next_u64()) * bound;
        if (static_cast<uint64_t>(prod) < bound) {
            const uint64_t floor = (0 - bound) % bound;
            while (static_cast<uint64_t>(prod) < floor)
                prod = static_cast<unsigned __int128>(next_u64()) * bound;
        }
        return static_cast<uint64_t>(prod >> 64);
    }

private:
    static constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
    static constexpr uint64_t kMulA = 0xbf58476d1ce4e5b9ull;
    static constexpr uint64_t kMulB = 0x94d049bb133111ebull;

    static uint64_t mix(uint64_t &z) {
        z += kGolden;
        uint64_t x = z;
        x = (x ^ (x >> 30)) * kMulA;
        x = (x ^ (x >> 27)) * kMulB;
        return x ^ (x >> 31);
    }

    uint64_t s_[4];
};

}  // namespace acs
