// tools/acs_bench.cpp -- the bench-cli of the reference SPEC
// over the drop-in API:
//
//   acs-bench solve   --instance FILE [options]                    one report per repetition
//   acs-bench sweep   --instance FILE --sweep "k=1,2,4,8;m=256" [options] [--out PREFIX]
//   acs-bench compare --instance FILE --a "memory=dense" --b "memory=selective"
//                     --time-limit-ms T [options] [--out PREFIX]
//
// options: [--mode seq|sync|relaxed] [--memory dense|selective]
//          [--variant atomic|deferred|relaxed|spm|seq|spm-seq|spm-sync] [--ants M]
//          [--iterations I | --budget B | --time-limit-ms T] [--update-period K] [--slots S]
//          [--beta B] [--alpha A] [--rho R] [--phi R] [--q0 Q] [--cl CL] [--seed S] [--reps R]
//          [--workers W] [--rng xoshiro|philox] [--device D] [--optima FILE] [--format csv|json]
//
// CSV columns: instance,n,mode,memory,ants,period,slots,rep,seed,best_len,
// err_pct,iters,total_ms,construct_ms_per_iter,hit_ratio (+ variant, tours_per_s; sweep adds
// the point's mean/min error, mean construction time and the +/- mark vs the first point).
// The optimum catalog comes from --optima or $ACS_OPTIMA.  Exit code 0 on success,
// 1 on a run/IO error, 2 on a usage error.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "acs/solver.hpp"
#include "acs/stats.hpp"
#include "acs/tsp_instance.hpp"

namespace {

using Opts = std::map<std::string, std::string>;

int usage() {
    std::fprintf(stderr,
                 "usage: acs-bench solve|sweep|compare --instance FILE [options]  (see tools/acs_bench.cpp)\n");
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

std::vector<std::string> split(const std::string &s, char sep) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    for (std::string item; std::getline(ss, item, sep);)
        if (!item.empty()) out.push_back(item);
    return out;
}

// one AcsParams field from its CLI name (also used for sweep axes and compare configs)
void apply(acs::AcsParams &p, const std::string &k, const std::string &v) {
    auto num = [&] { return std::stod(v); };
    if (k == "beta") p.beta = num();
    else if (k == "alpha") p.alpha = num();
    else if (k == "rho" || k == "phi") p.rho = num();
    else if (k == "q0") p.q0 = num();
    else if (k == "cl") p.cl = static_cast<uint32_t>(num());
    else if (k == "ants" || k == "m") p.m = static_cast<uint32_t>(num());
    else if (k == "slots" || k == "s") p.s = static_cast<uint32_t>(num());
    else if (k == "update-period" || k == "k") p.k = static_cast<uint32_t>(num());
    else if (k == "iterations") p.iterations = static_cast<uint64_t>(num());
    else if (k == "budget") p.budget = static_cast<uint64_t>(num());
    else if (k == "time-limit-ms") p.time_limit_s = num() / 1e3;
    else if (k == "seed") p.seed = static_cast<uint64_t>(num());
    else if (k == "device") p.device = static_cast<int>(num());
    else if (k == "workers") p.workers = static_cast<uint32_t>(num());
    else if (k == "consistent") p.consistent = v != "0" && v != "false";
    else if (k == "mode") {
        if (v == "seq") p.mode = acs::Mode::kSeq;
        else if (v == "sync") p.mode = acs::Mode::kSync;
        else if (v == "relaxed") p.mode = acs::Mode::kRelaxed;
        else throw std::invalid_argument("unknown mode " + v);
    } else if (k == "memory") {
        if (v == "dense") p.memory = acs::Memory::kDense;
        else if (v == "selective") p.memory = acs::Memory::kSelective;
        else throw std::invalid_argument("unknown memory " + v);
    } else if (k == "variant") {
        p.variant = v == "atomic" ? acs::Variant::kAtomic : v == "deferred" ? acs::Variant::kDeferred
                  : v == "relaxed" ? acs::Variant::kRelaxed : v == "spm" ? acs::Variant::kSpm
                  : v == "seq" ? acs::Variant::kSeq : v == "spm-seq" ? acs::Variant::kSpmSeq
                  : v == "spm-sync" ? acs::Variant::kSpmSync
                  : v == "auto" ? acs::Variant::kAuto
                  : throw std::invalid_argument("unknown variant " + v);
    } else if (k == "rng") {
        p.rng = v == "philox" ? acs::RngKind::kPhilox : acs::RngKind::kXoshiro;
    } else {
        throw std::invalid_argument("unknown parameter " + k);
    }
}

// "k1=v1,k2=v2" applied in order
void apply_config(acs::AcsParams &p, const std::string &cfg) {
    for (const std::string &kv : split(cfg, ',')) {
        const size_t eq = kv.find('=');
        if (eq == std::string::npos) throw std::invalid_argument("expected key=value, got " + kv);
        apply(p, kv.substr(0, eq), kv.substr(eq + 1));
    }
}

struct Row {
    acs::AcsParams p;
    acs::RunReport rep;
    uint32_t m;
    int r;
};

const char *CSV_HEAD = "instance,n,mode,memory,variant,ants,period,slots,rep,seed,best_len,err_pct,iters,"
                       "total_ms,construct_ms_per_iter,hit_ratio,tours_per_s";

double tours_per_s(const Row &x) {
    return x.rep.construct_ms_per_iter > 0 ? x.m / (x.rep.construct_ms_per_iter / 1e3) : 0.0;
}

std::string csv_row(const std::string &base, uint32_t n, const Row &x) {
    char err[32] = "", hr[32] = "", buf[512];
    if (x.rep.error_pct) std::snprintf(err, sizeof(err), "%.4f", *x.rep.error_pct);
    if (x.rep.hits + x.rep.misses) std::snprintf(hr, sizeof(hr), "%.6f", x.rep.hit_ratio());
    std::snprintf(buf, sizeof(buf), "%s,%u,%s,%s,%s,%u,%u,%u,%d,%llu,%lld,%s,%llu,%.3f,%.4f,%s,%.1f", base.c_str(), n,
                  x.rep.mode.c_str(), x.rep.memory.c_str(), x.rep.variant.c_str(), x.m, x.p.k, x.p.s, x.r,
                  static_cast<unsigned long long>(x.p.seed), static_cast<long long>(x.rep.best_length), err,
                  static_cast<unsigned long long>(x.rep.iterations), x.rep.total_ms, x.rep.construct_ms_per_iter,
                  hr, tours_per_s(x));
    return buf;
}

// full report with parameter provenance (enough to re-run SEQ bit-identically)
std::string json_report(const std::string &base, uint32_t n, const Row &x, bool with_tour) {
    std::ostringstream o;
    o.precision(17);
    const acs::AcsParams &p = x.p;
    o << "{\"instance\":\"" << base << "\",\"n\":" << n << ",\"mode\":\"" << x.rep.mode << "\",\"memory\":\""
      << x.rep.memory << "\",\"variant\":\"" << x.rep.variant << "\",\"ants\":" << x.m << ",\"period\":" << p.k
      << ",\"slots\":" << p.s << ",\"rep\":" << x.r << ",\"seed\":" << p.seed
      << ",\"best_len\":" << x.rep.best_length << ",\"err_pct\":";
    if (x.rep.error_pct) o << *x.rep.error_pct;
    else o << "null";
    o << ",\"iters\":" << x.rep.iterations << ",\"solutions\":" << x.rep.solutions << ",\"total_ms\":"
      << x.rep.total_ms << ",\"setup_ms\":" << x.rep.setup_ms << ",\"construct_ms_per_iter\":"
      << x.rep.construct_ms_per_iter << ",\"hit_ratio\":";
    if (x.rep.hits + x.rep.misses) o << x.rep.hit_ratio();
    else o << "null";
    o << ",\"tours_per_s\":" << tours_per_s(x) << ",\"tau0\":" << x.rep.tau0 << ",\"q0\":" << x.rep.q0
      << ",\"counters\":{\"local_updates\":" << x.rep.local_updates << ",\"hits\":" << x.rep.hits
      << ",\"misses\":" << x.rep.misses << ",\"fallback_steps\":" << x.rep.fallback_steps
      << ",\"greedy_steps\":" << x.rep.greedy_steps << ",\"roulette_steps\":" << x.rep.roulette_steps << "}"
      << ",\"params\":{\"beta\":" << p.beta << ",\"alpha\":" << p.alpha << ",\"rho\":" << p.rho
      << ",\"q0\":" << p.q0 << ",\"cl\":" << p.cl << ",\"m\":" << p.m << ",\"s\":" << p.s << ",\"k\":" << p.k
      << ",\"iterations\":" << p.iterations << ",\"budget\":" << p.budget << ",\"time_limit_s\":" << p.time_limit_s
      << ",\"consistent\":" << (p.consistent ? "true" : "false") << ",\"rng\":\""
      << (p.rng == acs::RngKind::kPhilox ? "philox" : "xoshiro") << "\",\"seed\":" << p.seed << "}";
    o << ",\"trace\":[";
    for (size_t i = 0; i < x.rep.trace.size(); ++i) o << (i ? "," : "") << x.rep.trace[i];
    o << "],\"trace_ms\":[";
    for (size_t i = 0; i < x.rep.trace_ms.size(); ++i) o << (i ? "," : "") << x.rep.trace_ms[i];
    o << "]";
    if (with_tour) {
        o << ",\"best_tour\":[";
        for (size_t i = 0; i < x.rep.best_tour.size(); ++i) o << (i ? "," : "") << x.rep.best_tour[i];
        o << "]";
    }
    o << "}";
    return o.str();
}

std::vector<double> errors_of(const std::vector<Row> &rows) {  // % error, or raw length without optimum
    std::vector<double> e;
    for (const Row &x : rows)
        e.push_back(x.rep.error_pct ? *x.rep.error_pct : static_cast<double>(x.rep.best_length));
    return e;
}

std::string fmt(double v) {
    if (std::isnan(v)) return "";
    char b[32];
    std::snprintf(b, sizeof(b), "%.4f", v);
    return b;
}

std::string jnum(double v) { return std::isnan(v) ? "null" : fmt(v); }

acs::SampleSummary summary_of(const std::vector<Row> &rows, int64_t opt) {
    std::vector<int64_t> len;
    std::vector<double> tot, con;
    for (const Row &x : rows) {
        len.push_back(x.rep.best_length);
        tot.push_back(x.rep.total_ms);
        con.push_back(x.rep.construct_ms_per_iter);
    }
    return acs::summarize(len, opt, tot, con);
}

std::vector<Row> run_reps(const acs::TspInstance &inst, const acs::AcsParams &p, int reps) {
    std::vector<Row> rows;
    for (int r = 0; r < reps; ++r) {
        Row x{p, {}, p.m ? p.m : inst.dimension_, r};
        x.p.seed = p.seed + static_cast<uint64_t>(r);
        x.rep = acs::run(inst, x.p);
        rows.push_back(std::move(x));
    }
    return rows;
}

void write_file(const std::string &path, const std::string &text) {
    std::ofstream f(path);
    if (!f) throw std::runtime_error("cannot write " + path);
    f << text;
}

int cmd_solve(const acs::TspInstance &inst, const std::string &base, const acs::AcsParams &p, int reps,
              bool json) {
    if (!json) std::printf("%s\n", CSV_HEAD);
    for (int r = 0; r < reps; ++r) {
        const std::vector<Row> one = run_reps(inst, [&] {
            acs::AcsParams q = p;
            q.seed = p.seed + static_cast<uint64_t>(r);
            return q;
        }(), 1);
        Row x = one[0];
        x.r = r;
        std::printf("%s\n", json ? json_report(base, inst.dimension_, x, true).c_str()
                                 : csv_row(base, inst.dimension_, x).c_str());
        std::fflush(stdout);
    }
    return 0;
}

// cmd_sweep: cartesian product of the axes, reps per point,
// one row per (point, repetition) annotated with the point's summary and the
// significance mark vs the first (baseline) point
int cmd_sweep(const acs::TspInstance &inst, const std::string &base, const acs::AcsParams &p, int reps,
              const std::string &axes_spec, const std::string &out, bool json) {
    std::vector<std::pair<std::string, std::vector<std::string>>> axes;
    for (const std::string &ax : split(axes_spec, ';')) {
        const size_t eq = ax.find('=');
        if (eq == std::string::npos) throw std::invalid_argument("sweep axis must be key=v1,v2,...");
        axes.push_back({ax.substr(0, eq), split(ax.substr(eq + 1), ',')});
        if (axes.back().second.empty()) throw std::invalid_argument("empty sweep axis " + ax);
    }
    if (axes.empty()) throw std::invalid_argument("--sweep needs at least one axis");
    std::vector<std::vector<std::string>> points{{}};
    for (const auto &ax : axes) {
        std::vector<std::vector<std::string>> next;
        for (const auto &pt : points)
            for (const std::string &v : ax.second) {
                auto q = pt;
                q.push_back(v);
                next.push_back(q);
            }
        points = next;
    }
    const int64_t opt = inst.optimum_ ? *inst.optimum_ : 0;
    std::ostringstream csv, js;
    csv << CSV_HEAD << ",point,mean_err_pct,min_err_pct,mean_construct_ms,mark\n";
    js << "[";
    std::vector<double> baseline;
    for (size_t i = 0; i < points.size(); ++i) {
        acs::AcsParams q = p;
        std::string label;
        for (size_t a = 0; a < axes.size(); ++a) {
            apply(q, axes[a].first, points[i][a]);
            label += (a ? ";" : "") + axes[a].first + "=" + points[i][a];
        }
        const std::vector<Row> rows = run_reps(inst, q, reps);
        const acs::SampleSummary sm = summary_of(rows, opt);
        const std::vector<double> err = errors_of(rows);
        const char mark = i == 0 ? ' ' : acs::significance_mark(err, baseline);
        if (i == 0) baseline = err;
        for (const Row &x : rows)
            csv << csv_row(base, inst.dimension_, x) << "," << label << "," << fmt(sm.mean_error_pct) << ","
                << fmt(sm.min_error_pct) << "," << fmt(sm.mean_construct_ms_per_iter) << ","
                << (mark == ' ' ? "" : std::string(1, mark)) << "\n";
        js << (i ? "," : "") << "{\"point\":\"" << label << "\",\"runs\":" << sm.runs
           << ",\"mean_err_pct\":" << jnum(sm.mean_error_pct) << ",\"min_err_pct\":" << jnum(sm.min_error_pct)
           << ",\"best_len\":" << sm.best_length << ",\"mean_construct_ms_per_iter\":"
           << fmt(sm.mean_construct_ms_per_iter) << ",\"p_vs_baseline\":"
           << (i == 0 || reps < 3 ? std::string("null") : jnum(acs::rank_sum_test(err, baseline)))
           << ",\"mark\":\"" << (mark == ' ' ? "" : std::string(1, mark)) << "\",\"reports\":[";
        for (size_t r = 0; r < rows.size(); ++r)
            js << (r ? "," : "") << json_report(base, inst.dimension_, rows[r], false);
        js << "]}";
    }
    js << "]\n";
    if (!out.empty()) {
        write_file(out + ".csv", csv.str());
        write_file(out + ".json", js.str());
    }
    std::printf("%s", json ? js.str().c_str() : csv.str().c_str());
    return 0;
}

// cmd_compare: two configs on the same instance under the
// same wall-clock limit, reps each; means, best, two-sided p, flagged winner
int cmd_compare(const acs::TspInstance &inst, const std::string &base, const acs::AcsParams &p, int reps,
                const std::string &cfg_a, const std::string &cfg_b, const std::string &out) {
    if (p.time_limit_s <= 0) throw std::invalid_argument("compare needs --time-limit-ms");
    if (reps < 3) throw std::invalid_argument("compare needs --reps >= 3 for the rank-sum test");
    acs::AcsParams pa = p, pb = p;
    apply_config(pa, cfg_a);
    apply_config(pb, cfg_b);
    const int64_t opt = inst.optimum_ ? *inst.optimum_ : 0;
    const std::vector<Row> ra = run_reps(inst, pa, reps), rb = run_reps(inst, pb, reps);
    const std::vector<double> ea = errors_of(ra), eb = errors_of(rb);
    const acs::SampleSummary sa = summary_of(ra, opt), sb = summary_of(rb, opt);
    const double pv = acs::rank_sum_test(ea, eb);
    const char mark = acs::significance_mark(ea, eb);
    const std::string winner = mark == '+' ? "A" : mark == '-' ? "B" : "none";
    std::ostringstream o;
    o.precision(10);
    auto side = [&](const char *name, const std::string &cfg, const acs::SampleSummary &s, const std::vector<Row> &rows) {
        o << "\"" << name << "\":{\"config\":\"" << cfg << "\",\"runs\":" << s.runs << ",\"mean_err_pct\":"
          << jnum(s.mean_error_pct) << ",\"min_err_pct\":" << jnum(s.min_error_pct) << ",\"best_len\":"
          << s.best_length << ",\"mean_len\":" << s.mean_length << ",\"mean_iters\":";
        double it = 0;
        for (const Row &x : rows) it += static_cast<double>(x.rep.iterations);
        o << it / rows.size() << ",\"mean_construct_ms_per_iter\":" << fmt(s.mean_construct_ms_per_iter)
          << ",\"lengths\":[";
        for (size_t i = 0; i < rows.size(); ++i) o << (i ? "," : "") << rows[i].rep.best_length;
        o << "]}";
    };
    o << "{\"instance\":\"" << base << "\",\"n\":" << inst.dimension_ << ",\"time_limit_ms\":" << p.time_limit_s * 1e3
      << ",\"errors_are\":\"" << (opt > 0 ? "percent over optimum" : "raw lengths (no optimum)") << "\",";
    side("A", cfg_a, sa, ra);
    o << ",";
    side("B", cfg_b, sb, rb);
    o << ",\"p_value\":" << pv << ",\"significant\":" << (pv < 0.05 ? "true" : "false") << ",\"winner\":\""
      << winner << "\"}\n";
    if (!out.empty()) write_file(out + ".json", o.str());
    std::printf("%s", o.str().c_str());
    return 0;
}

}  // namespace

int main(int argc, char **argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    if (cmd != "solve" && cmd != "sweep" && cmd != "compare") return usage();
    Opts opt;
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0 || i + 1 >= argc) return usage();
        opt[k.substr(2)] = argv[++i];
    }
    if (!opt.count("instance")) return usage();
    try {
        acs::TspInstance inst = acs::load_tsplib_file(opt["instance"]);
        const std::string base = basename_of(opt["instance"]);
        const char *env = std::getenv("ACS_OPTIMA");
        const std::string optima = opt.count("optima") ? opt["optima"] : (env ? env : "");
        if (!optima.empty()) {
            const auto cat = acs::load_optimum_catalog_file(optima);
            const auto it = cat.find(inst.name_.empty() ? base : inst.name_);
            if (it != cat.end()) inst.optimum_ = it->second;
            else std::fprintf(stderr, "warning: %s not in optimum catalog\n", inst.name_.c_str());
        }
        acs::AcsParams p;
        for (const auto &[k, v] : opt) {
            if (k == "instance" || k == "optima" || k == "reps" || k == "format" || k == "out" || k == "sweep" ||
                k == "a" || k == "b")
                continue;
            apply(p, k, v);
        }
        const int reps = opt.count("reps") ? std::stoi(opt["reps"]) : 1;
        if (reps < 1) throw std::invalid_argument("--reps must be >= 1");
        const bool json = opt.count("format") && opt["format"] == "json";
        const std::string out = opt.count("out") ? opt["out"] : "";
        if (cmd == "solve") return cmd_solve(inst, base, p, reps, json);
        if (cmd == "sweep") {
            if (!opt.count("sweep")) return usage();
            return cmd_sweep(inst, base, p, reps, opt["sweep"], out, json);
        }
        if (!opt.count("a") || !opt.count("b")) return usage();
        return cmd_compare(inst, base, p, reps, opt["a"], opt["b"], out);
    } catch (const acs::ParseError &e) {
        std::fprintf(stderr, "parse error: %s\n", e.what());
        return 1;
    } catch (const std::invalid_argument &e) {
        std::fprintf(stderr, "usage error: %s\n", e.what());
        return 2;
    } catch (const std::exception &e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
