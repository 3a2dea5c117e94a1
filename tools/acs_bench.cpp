// tools/acs_bench.cpp -- thin C++ CLI over the drop-in API:
//
//   acs-bench solve --instance data/tsplib/pr2392.tsp.gz [--mode seq|sync|relaxed]
//             [--memory dense|selective] [--variant atomic|deferred|relaxed|spm|seq|spm-seq]
//             [--ants M] [--iterations I | --budget B | --time-limit-ms T]
//             [--update-period K] [--slots S] [--beta B] [--alpha A] [--rho R] [--phi R]
//             [--q0 Q] [--cl CL] [--seed S] [--reps R] [--rng xoshiro|philox]
//             [--device D] [--optima FILE] [--format csv|json]
//
// One row per repetition with the SPEC CSV columns
// instance,n,mode,memory,ants,period,slots,rep,seed,best_len,err_pct,iters,
// total_ms,construct_ms_per_iter,hit_ratio (+ variant, tours_per_s).
// The optimum catalog comes from --optima or $ACS_OPTIMA.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <map>
#include <string>

#include "acs/solver.hpp"
#include "acs/tsp_instance.hpp"

namespace {

int usage() {
    std::fprintf(stderr, "usage: acs-bench solve --instance FILE [options]  (see tools/acs_bench.cpp)\n");
    return 2;
}

std::string basename_of(const std::string &path) {
    std::string b = path.substr(path.find_last_of('/') + 1);
    for (const char *ext : {".gz", ".tsp"}) {
        const size_t k = std::strlen(ext);
        if (b.size() > k && b.compare(b.size() - k, k, ext) == 0) b.resize(b.size() - k);
    }
    return b;
}

}  // namespace

int main(int argc, char **argv) {
    if (argc < 2 || std::string(argv[1]) != "solve") return usage();
    std::map<std::string, std::string> opt;
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0 || i + 1 >= argc) return usage();
        opt[k.substr(2)] = argv[++i];
    }
    if (!opt.count("instance")) return usage();
    try {
        acs::TspInstance inst = acs::load_tsplib_file(opt["instance"]);
        const std::string base = basename_of(opt["instance"]);
        std::string optima = opt.count("optima") ? opt["optima"] : (std::getenv("ACS_OPTIMA") ? std::getenv("ACS_OPTIMA") : "");
        if (!optima.empty()) {
            const auto cat = acs::load_optimum_catalog_file(optima);
            const auto it = cat.find(inst.name_.empty() ? base : inst.name_);
            if (it != cat.end()) inst.optimum_ = it->second;
            else std::fprintf(stderr, "warning: %s not in optimum catalog\n", inst.name_.c_str());
        }
        acs::AcsParams p;
        auto num = [&](const char *k, double d) { return opt.count(k) ? std::stod(opt[k]) : d; };
        p.beta = num("beta", p.beta);
        p.alpha = num("alpha", p.alpha);
        p.rho = num("rho", num("phi", p.rho));
        p.q0 = num("q0", p.q0);
        p.cl = static_cast<uint32_t>(num("cl", p.cl));
        p.m = static_cast<uint32_t>(num("ants", 0));
        p.s = static_cast<uint32_t>(num("slots", p.s));
        p.k = static_cast<uint32_t>(num("update-period", p.k));
        p.iterations = static_cast<uint64_t>(num("iterations", 1000));
        p.budget = static_cast<uint64_t>(num("budget", 0));
        p.time_limit_s = num("time-limit-ms", 0) / 1e3;
        p.seed = static_cast<uint64_t>(num("seed", 0));
        p.device = static_cast<int>(num("device", 0));
        const std::string mode = opt.count("mode") ? opt["mode"] : "relaxed";
        p.mode = mode == "seq" ? acs::Mode::kSeq : mode == "sync" ? acs::Mode::kSync : acs::Mode::kRelaxed;
        p.memory = opt.count("memory") && opt["memory"] == "selective" ? acs::Memory::kSelective : acs::Memory::kDense;
        if (opt.count("variant")) {
            const std::string v = opt["variant"];
            p.variant = v == "atomic" ? acs::Variant::kAtomic : v == "deferred" ? acs::Variant::kDeferred
                      : v == "relaxed" ? acs::Variant::kRelaxed : v == "spm" ? acs::Variant::kSpm
                      : v == "seq" ? acs::Variant::kSeq : v == "spm-seq" ? acs::Variant::kSpmSeq
                      : acs::Variant::kAuto;
        }
        p.rng = opt.count("rng") && opt["rng"] == "philox" ? acs::RngKind::kPhilox : acs::RngKind::kXoshiro;
        const int reps = static_cast<int>(num("reps", 1));
        const bool json = opt.count("format") && opt["format"] == "json";
        if (!json)
            std::printf("instance,n,mode,memory,variant,ants,period,slots,rep,seed,best_len,err_pct,iters,"
                        "total_ms,construct_ms_per_iter,hit_ratio,tours_per_s\n");
        for (int r = 0; r < reps; ++r) {
            acs::AcsParams pr = p;
            pr.seed = p.seed + static_cast<uint64_t>(r);
            const acs::RunReport rep = acs::run(inst, pr);
            const uint32_t m = pr.m ? pr.m : inst.dimension_;
            const double tps = rep.construct_ms_per_iter > 0 ? m / (rep.construct_ms_per_iter / 1e3) : 0.0;
            char err[32] = "", hr[32] = "";
            if (rep.error_pct) std::snprintf(err, sizeof(err), "%.4f", *rep.error_pct);
            if (rep.hits + rep.misses) std::snprintf(hr, sizeof(hr), "%.6f", rep.hit_ratio());
            if (json) {
                std::printf("{\"instance\":\"%s\",\"n\":%u,\"mode\":\"%s\",\"memory\":\"%s\",\"variant\":\"%s\","
                            "\"ants\":%u,\"period\":%u,\"slots\":%u,\"rep\":%d,\"seed\":%llu,\"best_len\":%lld,"
                            "\"err_pct\":%s,\"iters\":%llu,\"total_ms\":%.3f,\"construct_ms_per_iter\":%.4f,"
                            "\"hit_ratio\":%s,\"tours_per_s\":%.1f}\n",
                            base.c_str(), inst.dimension_, rep.mode.c_str(), rep.memory.c_str(), rep.variant.c_str(), m,
                            pr.k, pr.s, r, static_cast<unsigned long long>(pr.seed),
                            static_cast<long long>(rep.best_length), *err ? err : "null",
                            static_cast<unsigned long long>(rep.iterations), rep.total_ms, rep.construct_ms_per_iter,
                            *hr ? hr : "null", tps);
            } else {
                std::printf("%s,%u,%s,%s,%s,%u,%u,%u,%d,%llu,%lld,%s,%llu,%.3f,%.4f,%s,%.1f\n", base.c_str(),
                            inst.dimension_, rep.mode.c_str(), rep.memory.c_str(), rep.variant.c_str(), m, pr.k,
                            pr.s, r, static_cast<unsigned long long>(pr.seed), static_cast<long long>(rep.best_length),
                            err, static_cast<unsigned long long>(rep.iterations), rep.total_ms,
                            rep.construct_ms_per_iter, hr, tps);
            }
            std::fflush(stdout);
        }
    } catch (const acs::ParseError &e) {
        std::fprintf(stderr, "parse error: %s\n", e.what());
        return 1;
    } catch (const std::exception &e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
