// instance.cpp -- host side of the drop-in instance layer (include/acs/instance.hpp).
//
// TSPLIB95 parsing keeps the reference's observable behaviour
// (tsp_instance.cpp:80-217): the same accepted header forms, the same
// ParseError messages naming the offending field, exact coordinate round trip
// through serialize_tsplib.  Candidate lists and the NN tour are computed by
// the sm_100a kernels through the C-ABI.
#include <zlib.h>

#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>

#include "../../include/acs/instance.hpp"
#include "../../include/acs/rng_stream.hpp"

void acs_set_error(const char *msg);  // capi.cu: thread-local ABI error

namespace acs {

namespace {

constexpr const char *kWs = " \t\r\n";

std::string strip(const std::string &s) {
    const size_t b = s.find_first_not_of(kWs);
    if (b == std::string::npos) return {};
    return s.substr(b, s.find_last_not_of(kWs) - b + 1);
}

// "KEY : value", "KEY: value" or "KEY value"
bool header_kv(const std::string &line, std::string &key, std::string &value) {
    const size_t colon = line.find(':');
    if (colon != std::string::npos) {
        key = strip(line.substr(0, colon));
        value = strip(line.substr(colon + 1));
        return true;
    }
    const size_t b = line.find_first_not_of(kWs);
    if (b == std::string::npos) return false;
    const size_t e = line.find_first_of(kWs, b);
    key = line.substr(b, e == std::string::npos ? std::string::npos : e - b);
    value = e == std::string::npos ? std::string() : strip(line.substr(e));
    return true;
}

std::optional<EdgeWeightType> weight_type_of(const std::string &v) {
    if (v == "EUC_2D") return EdgeWeightType::kEuc2d;
    if (v == "CEIL_2D") return EdgeWeightType::kCeil2d;
    if (v == "ATT") return EdgeWeightType::kAtt;
    return std::nullopt;
}

[[noreturn]] void gpu_fail(const char *what) {
    throw GpuError(std::string(what) + ": " + acs_gpu_last_error());
}

}  // namespace

const char *to_string(EdgeWeightType type) {
    switch (type) {
        case EdgeWeightType::kEuc2d: return "EUC_2D";
        case EdgeWeightType::kCeil2d: return "CEIL_2D";
        case EdgeWeightType::kAtt: return "ATT";
    }
    return "?";
}

TspInstance::TspInstance(std::string name, EdgeWeightType type, std::vector<double> xs,
                         std::vector<double> ys)
    : name_(std::move(name)),
      dimension_(static_cast<uint32_t>(xs.size())),
      edge_weight_type_(type),
      xs_(std::move(xs)),
      ys_(std::move(ys)) {
    if (dimension_ < 3)
        throw ParseError("instance needs at least 3 nodes, got " + std::to_string(dimension_));
    if (xs_.size() != ys_.size()) throw ParseError("coordinate arrays differ in length");
}

// TSPLIB95 costs (EUC_2D nint, CEIL_2D, ATT); the kernels use the identical
// expression with explicit IEEE intrinsics (csrc/acs_device.cuh).
int32_t TspInstance::distance(uint32_t u, uint32_t v) const {
    volatile double xd = xs_[u] - xs_[v];  // volatile: no FMA contraction
    volatile double yd = ys_[u] - ys_[v];
    volatile double xx = xd * xd;
    volatile double yy = yd * yd;
    const double sq = xx + yy;
    switch (edge_weight_type_) {
        case EdgeWeightType::kEuc2d: return static_cast<int32_t>(std::sqrt(sq) + 0.5);
        case EdgeWeightType::kCeil2d: return static_cast<int32_t>(std::ceil(std::sqrt(sq)));
        case EdgeWeightType::kAtt: {
            const double r = std::sqrt(sq / 10.0);
            const int32_t t = static_cast<int32_t>(r + 0.5);
            return (static_cast<double>(t) < r) ? t + 1 : t;
        }
    }
    return 0;
}

int64_t TspInstance::tour_length(std::span<const uint32_t> order) const {
    int64_t sum = 0;
    for (size_t i = 0; i < order.size(); ++i)
        sum += distance(order[i == 0 ? order.size() - 1 : i - 1], order[i]);
    return sum;
}

acs_instance_desc TspInstance::desc() const {
    acs_instance_desc d{};
    d.n = dimension_;
    d.edge_weight_type = static_cast<uint32_t>(edge_weight_type_);
    d.xs = xs_.data();
    d.ys = ys_.data();
    return d;
}

TspInstance parse_tsplib(std::istream &in) {
    std::string name;
    std::optional<uint32_t> dim;
    std::optional<EdgeWeightType> type;
    std::vector<double> xs, ys;
    bool coords = false;
    std::string raw;
    while (std::getline(in, raw)) {
        const std::string line = strip(raw);
        if (line.empty()) continue;
        if (line == "EOF") break;
        if (coords) {
            std::istringstream f(line);
            long id;
            double x, y;
            if (!(f >> id >> x >> y))
                throw ParseError("NODE_COORD_SECTION: malformed line '" + line + "'");
            xs.push_back(x);
            ys.push_back(y);
            if (dim && xs.size() > *dim)
                throw ParseError("NODE_COORD_SECTION: more coordinates than DIMENSION=" +
                                 std::to_string(*dim));
            continue;
        }
        std::string key, value;
        if (!header_kv(line, key, value)) continue;
        if (key == "NAME") {
            name = value;
        } else if (key == "DIMENSION") {
            uint32_t d = 0;
            const auto r = std::from_chars(value.data(), value.data() + value.size(), d);
            if (r.ec != std::errc() || d == 0)
                throw ParseError("DIMENSION: cannot parse '" + value + "'");
            dim = d;
        } else if (key == "EDGE_WEIGHT_TYPE") {
            type = weight_type_of(value);
            if (!type) throw ParseError("EDGE_WEIGHT_TYPE: unsupported '" + value + "'");
        } else if (key == "NODE_COORD_SECTION") {
            if (!dim) throw ParseError("DIMENSION: missing before NODE_COORD_SECTION");
            if (!type) throw ParseError("EDGE_WEIGHT_TYPE: missing before NODE_COORD_SECTION");
            coords = true;
        }
        // TYPE, COMMENT and any other keyword: ignored
    }
    if (!dim) throw ParseError("DIMENSION: missing");
    if (!type) throw ParseError("EDGE_WEIGHT_TYPE: missing");
    if (xs.size() != *dim)
        throw ParseError("NODE_COORD_SECTION: expected " + std::to_string(*dim) +
                         " coordinates, got " + std::to_string(xs.size()));
    return TspInstance(name, *type, std::move(xs), std::move(ys));
}

TspInstance parse_tsplib(const std::string &text) {
    std::istringstream in(text);
    return parse_tsplib(in);
}

namespace {
// whole file, plain or gzip-compressed (zlib reads both transparently);
// false when it cannot be opened or read
bool read_maybe_gz(const std::string &path, std::string &text) {
    gzFile f = gzopen(path.c_str(), "rb");
    if (!f) return false;
    char buf[1 << 16];
    int got;
    while ((got = gzread(f, buf, sizeof(buf))) > 0) text.append(buf, static_cast<size_t>(got));
    gzclose(f);
    return got >= 0;
}
}  // namespace

TspInstance load_tsplib_file(const std::string &path) {
    std::string text;
    if (!read_maybe_gz(path, text)) throw ParseError("cannot open instance file: " + path);
    return parse_tsplib(text);
}

std::string serialize_tsplib(const TspInstance &inst) {
    std::ostringstream out;
    out.precision(17);  // 17 significant digits: exact double round trip
    out << "NAME : " << inst.name_ << '\n'
        << "TYPE : TSP\n"
        << "DIMENSION : " << inst.dimension_ << '\n'
        << "EDGE_WEIGHT_TYPE : " << to_string(inst.edge_weight_type_) << '\n'
        << "NODE_COORD_SECTION\n";
    for (uint32_t i = 0; i < inst.dimension_; ++i)
        out << i + 1 << ' ' << inst.xs_[i] << ' ' << inst.ys_[i] << '\n';
    out << "EOF\n";
    return out.str();
}

CandidateLists build_candidates(const TspInstance &inst, uint32_t cl, int device) {
    const acs_instance_desc d = inst.desc();
    CandidateLists c;
    c.cl_ = cl;
    c.n_ = inst.dimension_;
    if (acs_gpu_build_candidates(&d, cl, device, nullptr, &c.list_len_) != ACS_OK)
        gpu_fail("build_candidates");
    c.flat_.resize(static_cast<size_t>(c.n_) * c.list_len_);
    if (acs_gpu_build_candidates(&d, cl, device, c.flat_.data(), &c.list_len_) != ACS_OK)
        gpu_fail("build_candidates");
    return c;
}

int64_t nn_tour_length(const TspInstance &inst, uint32_t start, int device) {
    const acs_instance_desc d = inst.desc();
    int64_t out = 0;
    if (acs_gpu_nn_tour_length(&d, start, device, &out) != ACS_OK) gpu_fail("nn_tour_length");
    return out;
}

std::map<std::string, int64_t> load_optimum_catalog(std::istream &in) {
    std::map<std::string, int64_t> cat;
    std::string line;
    while (std::getline(in, line)) {
        line = line.substr(0, line.find('#'));
        std::istringstream f(line);
        std::string name;
        int64_t value = 0;
        if (f >> name >> value) cat[name] = value;
    }
    return cat;
}

std::map<std::string, int64_t> load_optimum_catalog_file(const std::string &path) {
    std::string text;  // plain or .gz, like the instance files
    if (!read_maybe_gz(path, text)) throw std::runtime_error("cannot open optimum catalog: " + path);
    std::istringstream in(text);
    return load_optimum_catalog(in);
}

TspInstance random_uniform_instance(uint32_t n, uint64_t seed, uint32_t side) {
    RngStream rng(seed);
    std::vector<double> xs(n), ys(n);
    for (uint32_t i = 0; i < n; ++i) {  // x then y per node, sequenced draws
        xs[i] = static_cast<double>(rng.uniform_int(side));
        ys[i] = static_cast<double>(rng.uniform_int(side));
    }
    std::string name = n % 1000 == 0 ? "rnd" + std::to_string(n / 1000) + "k" : "rnd" + std::to_string(n);
    return TspInstance(std::move(name), EdgeWeightType::kEuc2d, std::move(xs), std::move(ys));
}

}  // namespace acs

extern "C" int acs_random_instance(uint32_t n, uint64_t seed, uint32_t side, double *xs, double *ys) {
    if (n < 3 || side == 0 || !xs || !ys) {
        acs_set_error("acs_random_instance: need n >= 3, side >= 1 and output buffers");
        return ACS_E_ARG;
    }
    const acs::TspInstance inst = acs::random_uniform_instance(n, seed, side);
    std::memcpy(xs, inst.xs_.data(), sizeof(double) * n);
    std::memcpy(ys, inst.ys_.data(), sizeof(double) * n);
    return ACS_OK;
}

// ---- C-ABI: TSPLIB text -> caller storage ----
extern "C" int acs_parse_tsplib(const char *text, size_t len, uint32_t *n, uint32_t *type,
                                double *xs, double *ys, uint32_t cap, char *name,
                                size_t name_cap) {
    if (!text || !n) return ACS_E_ARG;
    try {
        const acs::TspInstance inst = acs::parse_tsplib(std::string(text, len));
        *n = inst.dimension_;
        if (type) *type = static_cast<uint32_t>(inst.edge_weight_type_);
        if (name && name_cap) {
            const size_t k = std::min(name_cap - 1, inst.name_.size());
            std::memcpy(name, inst.name_.data(), k);
            name[k] = '\0';
        }
        if (xs && ys) {
            if (cap < inst.dimension_) return ACS_E_ARG;
            std::memcpy(xs, inst.xs_.data(), sizeof(double) * inst.dimension_);
            std::memcpy(ys, inst.ys_.data(), sizeof(double) * inst.dimension_);
        }
        return ACS_OK;
    } catch (const acs::ParseError &e) {
        acs_set_error(e.what());
        return ACS_E_PARSE;
    }
}
