// solver.cpp -- the drop-in run(inst, params) -> RunReport
// over the C-ABI.  Budget handling (iterations / solution budget / coarse
// time limit checked between iteration chunks, D14) lives here; everything
// inside an iteration runs on the device.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>

#include "../../include/acs/solver.hpp"

namespace acs {

namespace {

[[noreturn]] void gpu_fail(const char *what) {
    throw GpuError(std::string(what) + ": " + acs_gpu_last_error());
}

const char *mode_name(Mode m) {
    switch (m) {
        case Mode::kSeq: return "seq";
        case Mode::kSync: return "sync";
        case Mode::kRelaxed: return "relaxed";
    }
    return "?";
}

const char *variant_name(int v) {
    switch (v) {
        case ACS_VARIANT_ATOMIC: return "atomic";
        case ACS_VARIANT_DEFERRED: return "deferred";
        case ACS_VARIANT_RELAXED: return "relaxed";
        case ACS_VARIANT_SPM: return "spm";
        case ACS_VARIANT_SEQ: return "seq";
        case ACS_VARIANT_SPM_SEQ: return "spm-seq";
        case ACS_VARIANT_SPM_SYNC: return "spm-sync";
    }
    return "?";
}

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

}  // namespace

double default_q0(uint32_t n) {  // SPEC.md:291-299 (clamped, D10)
    return n <= 20 ? 0.0 : static_cast<double>(n - 20) / static_cast<double>(n);
}

uint32_t select_best(std::span<const int64_t> lengths) {
    uint32_t best = 0;
    for (uint32_t a = 1; a < lengths.size(); ++a)
        if (lengths[a] < lengths[best]) best = a;
    return best;
}

bool is_better(int64_t a, int64_t b) { return a < b; }

double relative_error(int64_t length, int64_t optimum) {
    if (optimum <= 0) throw std::invalid_argument("relative_error: optimum must be > 0");
    return 100.0 * static_cast<double>(length - optimum) / static_cast<double>(optimum);
}

double RunReport::hit_ratio() const {
    if (hits + misses == 0) throw std::logic_error("hit_ratio: no selective-memory update yet");
    return static_cast<double>(hits) / static_cast<double>(hits + misses);
}

int resolve_variant(const AcsParams &p) {
    switch (p.variant) {
        case Variant::kAtomic: return ACS_VARIANT_ATOMIC;
        case Variant::kDeferred: return ACS_VARIANT_DEFERRED;
        case Variant::kRelaxed: return ACS_VARIANT_RELAXED;
        case Variant::kSpm: return ACS_VARIANT_SPM;
        case Variant::kSeq: return ACS_VARIANT_SEQ;
        case Variant::kSpmSeq: return ACS_VARIANT_SPM_SEQ;
        case Variant::kSpmSync: return ACS_VARIANT_SPM_SYNC;
        case Variant::kAuto: break;
    }
    if (p.memory == Memory::kDense) {
        if (p.mode == Mode::kSeq) return ACS_VARIANT_SEQ;
        if (p.mode == Mode::kSync) return ACS_VARIANT_DEFERRED;
        return p.consistent ? ACS_VARIANT_ATOMIC : ACS_VARIANT_RELAXED;
    }
    if (p.mode == Mode::kSeq) return ACS_VARIANT_SPM_SEQ;
    if (p.mode == Mode::kSync) return ACS_VARIANT_SPM_SYNC;
    return ACS_VARIANT_SPM;
}

namespace gpu {

CandidateLists build_candidates(const TspInstance &inst, uint32_t cl, int device) {
    return acs::build_candidates(inst, cl, device);
}

RunReport run(const TspInstance &inst, const AcsParams &p) {
    const int forms = (p.budget > 0) + (p.time_limit_s > 0.0) + (p.budget == 0 && p.time_limit_s <= 0.0);
    if (forms != 1) throw std::invalid_argument("exactly one budget form must be set");
    const uint32_t m = p.m ? p.m : inst.dimension_;
    uint64_t iterations = p.iterations;
    if (p.budget > 0) {
        if (p.budget % m) throw std::invalid_argument("budget must be a multiple of the ant count");
        iterations = p.budget / m;
    }
    if (iterations == 0 && p.time_limit_s <= 0.0) throw std::invalid_argument("budget of zero");

    const auto t0 = Clock::now();
    const acs_instance_desc d = inst.desc();
    acs_params ap{};
    ap.beta = p.beta;
    ap.alpha = p.alpha;
    ap.rho = p.rho;
    ap.q0 = p.q0;
    ap.cl = p.cl;
    ap.ants = m;
    ap.slots = p.s;
    ap.update_period = p.k;
    ap.variant = static_cast<uint32_t>(resolve_variant(p));
    ap.rng = p.rng == RngKind::kPhilox ? ACS_RNG_PHILOX : ACS_RNG_XOSHIRO;
    ap.seed = p.seed;
    acs_gpu_ctx *raw = nullptr;
    if (acs_gpu_create(&d, &ap, p.device, &raw) != ACS_OK) gpu_fail("acs_gpu_create");
    std::unique_ptr<acs_gpu_ctx, void (*)(acs_gpu_ctx *)> ctx(raw, acs_gpu_destroy);

    RunReport rep;
    rep.params = p;
    rep.mode = mode_name(p.mode);
    rep.memory = p.memory == Memory::kDense ? "dense" : "selective";
    rep.variant = variant_name(static_cast<int>(ap.variant));
    acs_ctx_info info{};
    acs_gpu_info(ctx.get(), &info);
    rep.tau0 = info.tau0;
    rep.q0 = info.q0;
    rep.setup_ms = ms_since(t0);

    const bool timed = p.time_limit_s > 0.0;
    double construct_ms = 0;
    std::vector<acs_iter_stats> st;
    uint64_t done = 0, chunk = 1;
    double last = ms_since(t0);
    while (timed ? ms_since(t0) < p.time_limit_s * 1e3 : done < iterations) {
        // chunks of iterations, one host sync each; the wall-clock limit is checked
        // between chunks (D14), which are sized to ~2 ms when timed
        const uint64_t want = timed ? chunk : std::min<uint64_t>(iterations - done, 256);
        st.resize(want);
        if (acs_gpu_iterate(ctx.get(), static_cast<uint32_t>(want), st.data()) != ACS_OK)
            gpu_fail("acs_gpu_iterate");
        float tot = 0, con = 0;
        acs_gpu_last_timing(ctx.get(), &tot, &con);
        construct_ms += con;
        const double now = ms_since(t0);
        for (uint64_t i = 0; i < want; ++i) {  // per-iteration timestamps, interpolated in a chunk
            rep.trace.push_back(st[i].global_best_len);
            rep.trace_ms.push_back(last + (now - last) * static_cast<double>(i + 1) / static_cast<double>(want));
        }
        if (timed)
            chunk = static_cast<uint64_t>(std::clamp(2.0 * static_cast<double>(want) / std::max(now - last, 1e-3), 1.0, 64.0));
        last = now;
        done += want;
    }
    rep.iterations = done;
    rep.solutions = done * m;
    rep.best_tour.resize(inst.dimension_);
    if (acs_gpu_get_best(ctx.get(), rep.best_tour.data(), &rep.best_length) != ACS_OK)
        gpu_fail("acs_gpu_get_best");
    acs_counters c{};
    acs_gpu_get_counters(ctx.get(), &c);
    rep.local_updates = c.local_updates;
    rep.hits = c.hits;
    rep.misses = c.misses;
    rep.fallback_steps = c.fallback_steps;
    rep.greedy_steps = c.greedy_steps;
    rep.roulette_steps = c.roulette_steps;
    rep.cas_retries = c.cas_retries;
    rep.construct_ms_per_iter = done ? construct_ms / static_cast<double>(done) : 0.0;
    if (inst.optimum_) rep.error_pct = relative_error(rep.best_length, *inst.optimum_);
    rep.total_ms = ms_since(t0);
    return rep;
}

}  // namespace gpu

RunReport run(const TspInstance &inst, const AcsParams &params) { return gpu::run(inst, params); }

}  // namespace acs
