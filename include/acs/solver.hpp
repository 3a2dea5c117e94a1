// include/acs/solver.hpp -- drop-in solver surface:
// AcsParams, RunReport, run(inst, params), plus the engine helpers
// default_q0 / select_best / is_better and stats::relative_error.
//
// run() executes on the GPU for every SPEC mode x memory combination:
//   DENSE     x SEQ     -> ACS_VARIANT_SEQ       (ant-major, one warp; deterministic)
//   DENSE     x SYNC    -> ACS_VARIANT_DEFERRED  (step snapshot + ordered apply; deterministic)
//   DENSE     x RELAXED -> ACS_VARIANT_ATOMIC    (CONSISTENT, CAS)  or
//                          ACS_VARIANT_RELAXED   (consistent=false: ACS-GPU-Alt lost updates)
//   SELECTIVE x SEQ     -> ACS_VARIANT_SPM_SEQ
//   SELECTIVE x SYNC    -> ACS_VARIANT_SPM_SYNC  (step snapshot + ordered record updates; deterministic)
//   SELECTIVE x RELAXED -> ACS_VARIANT_SPM       (ACS-GPU-SPM)
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "instance.hpp"

namespace acs {

enum class Mode { kSeq, kSync, kRelaxed };
enum class Memory { kDense, kSelective };
enum class Variant { kAuto, kAtomic, kDeferred, kRelaxed, kSpm, kSeq, kSpmSeq, kSpmSync };
enum class RngKind { kXoshiro, kPhilox };

struct AcsParams {
    double beta = 3.0;    // heuristic exponent
    double alpha = 0.2;   // GLOBAL evaporation (paper/SPEC naming)
    double rho = 0.01;    // LOCAL evaporation (north_star's "phi")
    double q0 = -1.0;     // < 0 -> default_q0(n)
    uint32_t cl = 32;     // candidate list length (GPU path: 1..32)
    uint32_t m = 0;       // ants; 0 -> n
    uint32_t s = 8;       // selective-memory slots
    uint32_t k = 1;       // local update period
    // exactly one budget form: iterations, budget (solutions), or time limit
    uint64_t iterations = 1000;
    uint64_t budget = 0;
    double time_limit_s = 0.0;
    Mode mode = Mode::kRelaxed;
    Memory memory = Memory::kDense;
    bool consistent = true;  // RELAXED dense: CAS (true) or plain ld/st (false)
    Variant variant = Variant::kAuto;
    RngKind rng = RngKind::kXoshiro;
    uint64_t seed = 0;
    uint32_t workers = 0;    // CPU-engine knob, accepted and ignored on the GPU
    int device = 0;
};

struct RunReport {
    std::vector<uint32_t> best_tour;
    int64_t best_length = 0;
    std::vector<int64_t> trace;      // L_gb after each iteration
    std::vector<double> trace_ms;    // wall-clock ms of each iteration (interpolated inside a host chunk)
    std::optional<double> error_pct; // vs the instance optimum when known
    double total_ms = 0, setup_ms = 0, construct_ms_per_iter = 0;
    uint64_t iterations = 0, solutions = 0;
    uint64_t local_updates = 0, hits = 0, misses = 0, fallback_steps = 0;
    uint64_t greedy_steps = 0, roulette_steps = 0, cas_retries = 0;
    double tau0 = 0, q0 = 0;
    AcsParams params;
    std::string mode, memory, variant;

    double hit_ratio() const;  // SPEC.md:155-163; throws if no selective update
};

double default_q0(uint32_t n);
uint32_t select_best(std::span<const int64_t> lengths);  // ties -> lowest ant
bool is_better(int64_t a, int64_t b);                     // strict
double relative_error(int64_t length, int64_t optimum);  // percent
int resolve_variant(const AcsParams &p);                  // -> enum acs_variant

RunReport run(const TspInstance &inst, const AcsParams &params);

namespace gpu {
RunReport run(const TspInstance &inst, const AcsParams &params);
CandidateLists build_candidates(const TspInstance &inst, uint32_t cl, int device = 0);
}  // namespace gpu

}  // namespace acs
