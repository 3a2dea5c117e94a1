// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim compiled TOGETHER WITH the unmodified reference sources
// where they lie (/root/reference/proj/src/tsp_instance.cpp and the headers
// under /root/reference/proj/include) into oracle/_ref/libacsref.so by
// oracle/Makefile.  Nothing from the reference is copied into this repo; this
// file only adapts the reference's C++ API (tsp_instance.hpp:14-96,
// rng.hpp:16-84) to plain C calls so pytest can drive it through ctypes and
// pin the oracle restatement (acs_oracle.c) and the product against it.
#include <cstring>
#include <sstream>
#include <string>

#include "acs/rng.hpp"
#include "acs/tsp_instance.hpp"

namespace {
void put_err(char *err, size_t cap, const std::string &msg) {
    if (!err || cap == 0) return;
    const size_t k = msg.size() < cap - 1 ? msg.size() : cap - 1;
    std::memcpy(err, msg.data(), k);
    err[k] = '\0';
}
}  // namespace

extern "C" {

void *ref_parse(const char *text, char *err, size_t cap) {
    try {
        return new acs::TspInstance(acs::parse_tsplib(std::string(text)));
    } catch (const acs::ParseError &e) {
        put_err(err, cap, e.what());
    } catch (const std::exception &e) {
        put_err(err, cap, std::string("other: ") + e.what());
    }
    return nullptr;
}

void *ref_make(const char *name, int type, const double *xs, const double *ys, uint32_t n,
               char *err, size_t cap) {
    try {
        return new acs::TspInstance(name, static_cast<acs::EdgeWeightType>(type),
                                    std::vector<double>(xs, xs + n),
                                    std::vector<double>(ys, ys + n));
    } catch (const std::exception &e) {
        put_err(err, cap, e.what());
    }
    return nullptr;
}

void ref_free(void *p) { delete static_cast<acs::TspInstance *>(p); }

uint32_t ref_n(void *p) { return static_cast<acs::TspInstance *>(p)->dimension_; }
int ref_type(void *p) { return static_cast<int>(static_cast<acs::TspInstance *>(p)->edge_weight_type_); }
size_t ref_name(void *p, char *out, size_t cap) {
    const std::string &s = static_cast<acs::TspInstance *>(p)->name_;
    put_err(out, cap, s);
    return s.size();
}
void ref_coords(void *p, double *xs, double *ys) {
    auto *I = static_cast<acs::TspInstance *>(p);
    std::memcpy(xs, I->xs_.data(), sizeof(double) * I->dimension_);
    std::memcpy(ys, I->ys_.data(), sizeof(double) * I->dimension_);
}
int32_t ref_distance(void *p, uint32_t u, uint32_t v) {
    return static_cast<acs::TspInstance *>(p)->distance(u, v);
}
void ref_distance_table(void *p, int32_t *out) {
    auto *I = static_cast<acs::TspInstance *>(p);
    const uint32_t n = I->dimension_;
    for (uint32_t u = 0; u < n; ++u)
        for (uint32_t v = 0; v < n; ++v) out[static_cast<size_t>(u) * n + v] = I->distance(u, v);
}
uint32_t ref_build_candidates(void *p, uint32_t cl, uint32_t *out) {
    const acs::CandidateLists c = acs::build_candidates(*static_cast<acs::TspInstance *>(p), cl);
    std::memcpy(out, c.flat_.data(), sizeof(uint32_t) * c.flat_.size());
    return c.list_len_;
}
int64_t ref_nn_tour_length(void *p, uint32_t start) {
    return acs::nn_tour_length(*static_cast<acs::TspInstance *>(p), start);
}
int64_t ref_tour_length(void *p, const uint32_t *order, uint32_t len) {
    return static_cast<acs::TspInstance *>(p)->tour_length(std::span<const uint32_t>(order, len));
}
size_t ref_serialize(void *p, char *out, size_t cap) {
    const std::string s = acs::serialize_tsplib(*static_cast<acs::TspInstance *>(p));
    if (out && cap > s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
    return s.size();
}

// Optimum catalog: returns the entry count; names are '\n'-joined.
int ref_catalog(const char *text, char *names, size_t cap, int64_t *values, int max_entries) {
    std::istringstream in{std::string(text)};
    const auto cat = acs::load_optimum_catalog(in);
    std::string joined;
    int i = 0;
    for (const auto &[k, v] : cat) {
        if (i < max_entries) values[i] = v;
        joined += k;
        joined += '\n';
        ++i;
    }
    put_err(names, cap, joined);
    return i;
}

// RNG script: op 0 = next_u64, 1 = uniform01 (bit pattern), 2 = uniform_int(arg).
// derive != 0 -> RngStream::derive(seed, it, ant) else RngStream(seed).
void ref_rng_script(uint64_t seed, uint64_t it, uint64_t ant, int derive, const int32_t *ops,
                    const uint64_t *args, uint64_t *out, int count) {
    acs::RngStream r = derive ? acs::RngStream::derive(seed, it, ant) : acs::RngStream(seed);
    for (int i = 0; i < count; ++i) {
        if (ops[i] == 0) {
            out[i] = r.next_u64();
        } else if (ops[i] == 1) {
            const double d = r.uniform01();
            std::memcpy(&out[i], &d, 8);
        } else {
            out[i] = r.uniform_int(args[i]);
        }
    }
}

}  // extern "C"
