// capi.cu -- extern "C" entry points of include/acs_gpu.h: the drop-in
// boundary of the B200 ACS hot path.  Contexts own all device memory; every
// compute call is stream-ordered on the context stream and synchronises only
// where the ABI hands results back to the host.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <memory>
#include <mutex>

#ifndef ACS_EXT_MAX
#define ACS_EXT_MAX 192u // next-nearest entries per row for the pruned fallback (multiple of 32)
#endif
#include <string>
#include <vector>

#include "../../include/acs_gpu.h"
#include "acs_kernels.cuh"

using namespace acs_dev;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                  \
    do {                                                                                \
        const cudaError_t e_ = (expr);                                                  \
        if (e_ != cudaSuccess)                                                          \
            return fail(e_ == cudaErrorMemoryAllocation ? ACS_E_NOMEM : ACS_E_CUDA,      \
                        std::string(#expr) + ": " + cudaGetErrorString(e_));            \
    } while (0)

// device buffer with RAII.
// Context allocations are stream-ordered from the device's default memory
// pool (release threshold raised once per device, see PoolScope), so a
// context's ~150 MB of buffers are recycled by the next context instead of
// going through cudaMalloc / cudaFree each time (acs_gpu_run = create + K
// iterations + destroy).  Buffers of the stateless setup ops use cudaMalloc.
thread_local cudaStream_t t_alloc_stream = nullptr;

template <class T>
struct DBuf {
    T *p = nullptr;
    size_t count = 0;
    cudaStream_t s = nullptr;  // pool allocation ordered on this stream (nullptr: cudaMalloc)
    DBuf() = default;
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) {
            if (s) cudaFreeAsync(p, s);
            else cudaFree(p);
        }
        p = nullptr;
        count = 0;
    }
    cudaError_t alloc(size_t n) {
        release();
        count = n;
        s = t_alloc_stream;
        if (!n) return cudaSuccess;
        return s ? cudaMallocAsync(reinterpret_cast<void **>(&p), n * sizeof(T), s)
                 : cudaMalloc(reinterpret_cast<void **>(&p), n * sizeof(T));
    }
    size_t bytes() const { return count * sizeof(T); }
};

// While alive, DBuf::alloc on this thread draws from `device`'s default pool,
// ordered on `stream`; the pool keeps freed memory cached (threshold = max).
struct PoolScope {
    PoolScope(int device, cudaStream_t stream) {
        static std::mutex mu;  // contexts may be created from several host threads (islands)
        static bool configured[64] = {};
        {
            std::lock_guard<std::mutex> lock(mu);
            if (device >= 0 && device < 64 && !configured[device]) {
                cudaMemPool_t pool;
                if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
                    uint64_t keep = UINT64_MAX;
                    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
                }
                configured[device] = true;
            }
        }
        t_alloc_stream = stream;
    }
    ~PoolScope() { t_alloc_stream = nullptr; }
};

int check_instance(const acs_instance_desc *inst) {
    if (!inst || !inst->xs || !inst->ys) return fail(ACS_E_ARG, "instance: null pointer");
    if (inst->n < 3) return fail(ACS_E_ARG, "instance needs at least 3 nodes, got " + std::to_string(inst->n));
    if (inst->n > 0x00FFFFFEu) return fail(ACS_E_ARG, "instance: n exceeds 2^24-2 nodes");
    if (inst->edge_weight_type > ACS_ATT) return fail(ACS_E_ARG, "instance: unknown edge weight type");
    return ACS_OK;
}

int set_device(int device) {
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(ACS_E_CUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e));
    if (device < 0 || device >= count) return fail(ACS_E_ARG, "device index out of range");
    CUDA_TRY(cudaSetDevice(device));
    return ACS_OK;
}

// instance coordinates resident on the device (+ distance table when n <= 4096)
struct DevInst {
    DBuf<double> xs, ys;
    DBuf<int32_t> dist;
    DevInstance view{};

    int upload(const acs_instance_desc *inst, bool want_table, cudaStream_t s) {
        const uint32_t n = inst->n;
        CUDA_TRY(xs.alloc(n));
        CUDA_TRY(ys.alloc(n));
        CUDA_TRY(cudaMemcpyAsync(xs.p, inst->xs, n * sizeof(double), cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(ys.p, inst->ys, n * sizeof(double), cudaMemcpyHostToDevice, s));
        view.n = n;
        view.words = (n + 31) / 32;
        view.type = static_cast<int>(inst->edge_weight_type);
        view.xs = xs.p;
        view.ys = ys.p;
        view.dist = nullptr;
        view.etab = nullptr;
        view.eta_d = nullptr;
        view.eta_dmax = 0;
        if (want_table && n <= 4096) {  // tsp_instance.hpp:31 kDistTableMaxNodes
            CUDA_TRY(dist.alloc(static_cast<size_t>(n) * n));
            launch_distance_table(view, dist.p, s);
            CUDA_TRY(cudaGetLastError());
            view.dist = dist.p;
        }
        return ACS_OK;
    }
};

struct Stream {
    cudaStream_t s = nullptr;
    ~Stream() {
        if (s) cudaStreamDestroy(s);
    }
    int create() {
        CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        return ACS_OK;
    }
};

int beta_int_of(double beta) {
    return (beta >= 0.0 && beta <= 64.0 && beta == std::floor(beta)) ? static_cast<int>(beta) : -1;
}

double default_q0(uint32_t n) { return n <= 20 ? 0.0 : static_cast<double>(n - 20) / static_cast<double>(n); }

// ---- lazily loaded NCCL (island model) ----
typedef struct { char internal[128]; } nccl_uid;
typedef void *nccl_comm;
struct NcclApi {
    void *h = nullptr;
    int (*get_unique_id)(nccl_uid *) = nullptr;
    int (*comm_init_rank)(nccl_comm *, int, nccl_uid, int) = nullptr;
    int (*comm_destroy)(nccl_comm) = nullptr;
    int (*all_reduce)(const void *, void *, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    int (*broadcast)(const void *, void *, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    const char *(*error_string)(int) = nullptr;

    int load() {
        if (h) return ACS_OK;
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *nm : names) {
            h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) return fail(ACS_E_NCCL, "libnccl.so.2 not loadable");
        get_unique_id = reinterpret_cast<decltype(get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        comm_init_rank = reinterpret_cast<decltype(comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        comm_destroy = reinterpret_cast<decltype(comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        all_reduce = reinterpret_cast<decltype(all_reduce)>(dlsym(h, "ncclAllReduce"));
        broadcast = reinterpret_cast<decltype(broadcast)>(dlsym(h, "ncclBroadcast"));
        error_string = reinterpret_cast<decltype(error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!get_unique_id || !comm_init_rank || !comm_destroy || !all_reduce || !broadcast)
            return fail(ACS_E_NCCL, "libnccl: missing symbols");
        return ACS_OK;
    }
};
NcclApi g_nccl;
constexpr int kNcclInt64 = 4, kNcclUint32 = 3, kNcclMin = 3, kNcclSum = 0;

}  // namespace

void acs_set_error(const char *msg) { g_err = msg ? msg : ""; }

struct acs_gpu_ctx {
    int device = 0;
    Stream stream;
    acs_params params{};
    DevInst inst;
    uint32_t n = 0, m = 0, L = 0, S = 0;
    double q0 = 0, tau0 = 0;
    int64_t nn_len = 0;
    DBuf<uint4> rows, ext;     // candidate rows; next-nearest rows for the pruned fallback
    DBuf<uint32_t> hot, hot_cnt;  // per-row non-candidate edges the global update touched
    DBuf<uint32_t> cell_start, cell_nodes;  // uniform grid (CSR) for the fallback beyond the ext rows
    DBuf<uint32_t> cand;  // flat n*L (reference layout), kept for get_candidates
    DBuf<double> tau, tauc, etab, pw;
    DBuf<double> eta_d;  // non-integral beta: eta^beta by integer distance
    DBuf<unsigned char> spm;   // record-major selective memory (SpmMem)
    SpmMem spm_mem;
    DBuf<uint32_t> cnt, cntc;  // ATOMIC variant: pending local updates per copy
    DBuf<uint32_t> routes, best_tour;
    DBuf<int64_t> lens, best_len;
    DBuf<uint64_t> iter;
    DBuf<unsigned long long> counters;
    DBuf<acs_iter_stats> stats;
    // island exchange scratch
    DBuf<int64_t> x_key;
    DBuf<uint32_t> x_tour;
    DBuf<int64_t> x_len;
    DBuf<int64_t> xl_keys;            // in-process exchange (this ctx leads): one key per colony
    DBuf<const uint32_t *> xl_tours;  // the colonies' masked tours
    DBuf<uint32_t> xl_sum;            // their sum = the winner's tour
    nccl_comm comm = nullptr;
    int rank = 0, nranks = 1;
    // timing
    std::vector<cudaEvent_t> events;
    float last_total_ms = 0, last_construct_ms = 0;
    DevColony colony{};
    DevBest best{};
    DevDeferred deferred{};
    DBuf<unsigned char> sy_ants;  // SYNC x SELECTIVE: per-ant state, bitmasks, step ops
    DBuf<uint32_t> sy_vis;
    DBuf<uint4> sy_ops;
    DBuf<unsigned long long> sy_keys;  // m > 8192: radix-sort keys (in | out)
    DBuf<uint32_t> sy_idx;             // and their op indices
    DBuf<unsigned char> sy_tmp;        // cub temp storage
    DevSpmSync spm_sync{};

    ~acs_gpu_ctx() {
        if (comm && g_nccl.comm_destroy) g_nccl.comm_destroy(comm);
        for (cudaEvent_t e : events) cudaEventDestroy(e);
    }
    bool dense() const {
        return params.variant != ACS_VARIANT_SPM && params.variant != ACS_VARIANT_SPM_SEQ &&
               params.variant != ACS_VARIANT_SPM_SYNC;
    }
    int ensure_events(size_t count) {
        while (events.size() < count) {
            cudaEvent_t e;
            CUDA_TRY(cudaEventCreate(&e));
            events.push_back(e);
        }
        return ACS_OK;
    }
    size_t device_bytes() const {
        return inst.xs.bytes() + inst.ys.bytes() + inst.dist.bytes() + etab.bytes() + rows.bytes() + ext.bytes() + hot.bytes() + hot_cnt.bytes() + cell_start.bytes() + cell_nodes.bytes() + cand.bytes() +
               tau.bytes() + tauc.bytes() + spm.bytes() +
               routes.bytes() + best_tour.bytes() + lens.bytes() + cnt.bytes() + cntc.bytes();
    }
};

extern "C" {

const char *acs_gpu_last_error(void) { return g_err.c_str(); }
int acs_gpu_abi_version(void) { return ACS_GPU_ABI_VERSION; }

int acs_gpu_device_count(int *count) {
    if (!count) return fail(ACS_E_ARG, "null count");
    *count = 0;
    const cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        return fail(ACS_E_CUDA, cudaGetErrorString(e));
    }
    return ACS_OK;
}

int acs_gpu_distance_table(const acs_instance_desc *inst, int device, int32_t *out) {
    if (int rc = check_instance(inst)) return rc;
    if (!out) return fail(ACS_E_ARG, "null output");
    if (int rc = set_device(device)) return rc;
    Stream st;
    if (int rc = st.create()) return rc;
    DevInst di;
    if (int rc = di.upload(inst, false, st.s)) return rc;
    DBuf<int32_t> d;
    CUDA_TRY(d.alloc(static_cast<size_t>(inst->n) * inst->n));
    launch_distance_table(di.view, d.p, st.s);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out, d.p, d.bytes(), cudaMemcpyDeviceToHost, st.s));
    CUDA_TRY(cudaStreamSynchronize(st.s));
    return ACS_OK;
}

int acs_gpu_build_candidates(const acs_instance_desc *inst, uint32_t cl, int device,
                             uint32_t *out_flat, uint32_t *list_len) {
    if (int rc = check_instance(inst)) return rc;
    if (cl < 1 || cl > 32) return fail(ACS_E_ARG, "cl must be in [1, 32] on the GPU path");
    const uint32_t L = cl < inst->n - 1 ? cl : inst->n - 1;
    if (list_len) *list_len = L;
    if (!out_flat) return ACS_OK;
    if (int rc = set_device(device)) return rc;
    Stream st;
    if (int rc = st.create()) return rc;
    DevInst di;
    if (int rc = di.upload(inst, false, st.s)) return rc;
    DBuf<uint32_t> d;
    CUDA_TRY(d.alloc(static_cast<size_t>(inst->n) * L));
    launch_topk(di.view, L, d.p, st.s);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out_flat, d.p, d.bytes(), cudaMemcpyDeviceToHost, st.s));
    CUDA_TRY(cudaStreamSynchronize(st.s));
    return ACS_OK;
}

int acs_gpu_nn_tour_length(const acs_instance_desc *inst, uint32_t start, int device, int64_t *out) {
    if (int rc = check_instance(inst)) return rc;
    if (!out || start >= inst->n) return fail(ACS_E_ARG, "bad start / null output");
    if (int rc = set_device(device)) return rc;
    Stream st;
    if (int rc = st.create()) return rc;
    DevInst di;
    if (int rc = di.upload(inst, true, st.s)) return rc;
    DBuf<int64_t> d;
    CUDA_TRY(d.alloc(1));
    // candidate lists first (K2, tens of us): the NN walk then probes the
    // first unvisited list entry and scans all n only when a list is exhausted
    const uint32_t L = inst->n - 1 < 32u ? inst->n - 1 : 32u;
    DBuf<uint32_t> cand;
    CUDA_TRY(cand.alloc(static_cast<size_t>(inst->n) * L));
    launch_topk(di.view, L, cand.p, st.s);
    launch_nn_tour_cand(di.view, cand.p, L, start, d.p, st.s);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out, d.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st.s));
    CUDA_TRY(cudaStreamSynchronize(st.s));
    return ACS_OK;
}

int acs_gpu_tour_lengths(const acs_instance_desc *inst, const uint32_t *routes, uint32_t m,
                         int device, int64_t *out) {
    if (int rc = check_instance(inst)) return rc;
    if (!routes || !out || m == 0) return fail(ACS_E_ARG, "null routes/output or m == 0");
    if (int rc = set_device(device)) return rc;
    Stream st;
    if (int rc = st.create()) return rc;
    DevInst di;
    if (int rc = di.upload(inst, true, st.s)) return rc;
    DBuf<uint32_t> r;
    DBuf<int64_t> d;
    CUDA_TRY(r.alloc(static_cast<size_t>(m) * inst->n));
    CUDA_TRY(d.alloc(m));
    CUDA_TRY(cudaMemcpyAsync(r.p, routes, r.bytes(), cudaMemcpyHostToDevice, st.s));
    launch_tour_lengths(di.view, r.p, m, d.p, st.s);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out, d.p, d.bytes(), cudaMemcpyDeviceToHost, st.s));
    CUDA_TRY(cudaStreamSynchronize(st.s));
    return ACS_OK;
}

int acs_gpu_l2_read_bandwidth(int device, uint64_t bytes, double *gbs) {
    if (!gbs || bytes < (1u << 20)) return fail(ACS_E_ARG, "null output or buffer below 1 MiB");
    if (int rc = set_device(device)) return rc;
    Stream st;
    if (int rc = st.create()) return rc;
    int sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const size_t count = bytes / sizeof(uint4);
    DBuf<uint4> buf;
    DBuf<uint32_t> sink;
    CUDA_TRY(buf.alloc(count));
    CUDA_TRY(sink.alloc(1));
    CUDA_TRY(cudaMemsetAsync(buf.p, 1, buf.bytes(), st.s));
    const uint32_t reps = 20;
    launch_l2_read(buf.p, count, 2, sink.p, sms, st.s);  // warm: pull the buffer into L2
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int t = 0; t < 5; ++t) {
        CUDA_TRY(cudaEventRecord(e0, st.s));
        launch_l2_read(buf.p, count, reps, sink.p, sms, st.s);
        CUDA_TRY(cudaEventRecord(e1, st.s));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CUDA_TRY(cudaGetLastError());
    *gbs = static_cast<double>(count) * sizeof(uint4) * reps / (best * 1e-3) / 1e9;
    return ACS_OK;
}

int acs_gpu_l2_latency(int device, uint64_t bytes, double *load_ns, double *step_ns) {
    if (!load_ns || !step_ns || bytes < (4u << 20)) return fail(ACS_E_ARG, "null output or buffer below 4 MiB");
    if (int rc = set_device(device)) return rc;
    Stream st;
    if (int rc = st.create()) return rc;
    int sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    struct EvGuard {
        cudaEvent_t a, b;
        ~EvGuard() { cudaEventDestroy(a); cudaEventDestroy(b); }
    } eg{e0, e1};
    auto timed = [&](auto &&launch) -> float {
        float best = 1e30f;
        for (int t = 0; t < 3; ++t) {
            cudaEventRecord(e0, st.s);
            launch();
            cudaEventRecord(e1, st.s);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        return best;
    };
    DBuf<uint32_t> sink;
    CUDA_TRY(sink.alloc(1));
    uint64_t x = 0x2545F4914F6CDD1Dull;  // xorshift64 for the host-side layouts
    auto rnd = [&x](uint64_t bound) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        return x % bound;
    };
    // (1) pointer chase: a random cycle (Sattolo) over the 128 B lines
    {
        const size_t lines = bytes / 128;
        std::vector<uint32_t> perm(lines), h(lines * 32, 0u);
        for (size_t i = 0; i < lines; ++i) perm[i] = static_cast<uint32_t>(i);
        for (size_t i = lines - 1; i > 0; --i) std::swap(perm[i], perm[rnd(i)]);
        for (size_t i = 0; i < lines; ++i) h[i * 32] = perm[i];
        DBuf<uint32_t> buf;
        CUDA_TRY(buf.alloc(h.size()));
        CUDA_TRY(cudaMemcpyAsync(buf.p, h.data(), buf.bytes(), cudaMemcpyHostToDevice, st.s));
        launch_l2_chase(buf.p, static_cast<uint32_t>(lines), 0, sink.p, st.s);  // warm: every line into L2
        const uint32_t steps = 200000;
        const float ms = timed([&] { launch_l2_chase(buf.p, steps, 1, sink.p, st.s); });
        CUDA_TRY(cudaGetLastError());
        *load_ns = static_cast<double>(ms) * 1e6 / steps;
    }
    // (2) minimal selection step over L2-resident rows (nrows x 512 B + 256 B)
    {
        const uint32_t nrows = static_cast<uint32_t>(std::min<uint64_t>(bytes / 768, 1u << 20));
        std::vector<uint4> rows(static_cast<size_t>(nrows) * 32);
        for (uint32_t r = 0; r < nrows; ++r)
            for (int l = 0; l < 32; ++l) {
                const uint32_t id = static_cast<uint32_t>((r + 1 + rnd(nrows - 1)) % nrows);
                const double eta = 1.0 / static_cast<double>(1 + rnd(1000));
                uint64_t b;
                std::memcpy(&b, &eta, 8);
                rows[static_cast<size_t>(r) * 32 + l] = make_uint4(id, 0u, static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32));
            }
        std::vector<double> tau(static_cast<size_t>(nrows) * 32, 1.0);
        DBuf<uint4> drows;
        DBuf<double> dtau;
        CUDA_TRY(drows.alloc(rows.size()));
        CUDA_TRY(dtau.alloc(tau.size()));
        CUDA_TRY(cudaMemcpyAsync(drows.p, rows.data(), drows.bytes(), cudaMemcpyHostToDevice, st.s));
        CUDA_TRY(cudaMemcpyAsync(dtau.p, tau.data(), dtau.bytes(), cudaMemcpyHostToDevice, st.s));
        launch_l2_read(drows.p, drows.bytes() / sizeof(uint4), 2, sink.p, sms, st.s);  // warm into L2
        launch_l2_read(reinterpret_cast<const uint4 *>(dtau.p), dtau.bytes() / sizeof(uint4), 2, sink.p, sms, st.s);
        const uint32_t steps = 100000;
        const float ms = timed([&] { launch_step_floor(drows.p, dtau.p, nrows, steps, 2048, sink.p, st.s); });
        CUDA_TRY(cudaGetLastError());
        *step_ns = static_cast<double>(ms) * 1e6 / steps;
    }
    CUDA_TRY(cudaStreamSynchronize(st.s));
    return ACS_OK;
}

int acs_gpu_rng_script(uint32_t kind, uint64_t seed, uint64_t iteration, uint64_t ant, int derive,
                       const int32_t *ops, const uint64_t *args, uint64_t *out, uint32_t count,
                       int device) {
    if (!ops || !out || count == 0) return fail(ACS_E_ARG, "null ops/out or empty script");
    if (kind > ACS_RNG_PHILOX) return fail(ACS_E_ARG, "unknown rng kind");
    if (int rc = set_device(device)) return rc;
    Stream st;
    if (int rc = st.create()) return rc;
    DBuf<int32_t> o;
    DBuf<uint64_t> a, r;
    CUDA_TRY(o.alloc(count));
    CUDA_TRY(a.alloc(count));
    CUDA_TRY(r.alloc(count));
    CUDA_TRY(cudaMemcpyAsync(o.p, ops, o.bytes(), cudaMemcpyHostToDevice, st.s));
    if (args) CUDA_TRY(cudaMemcpyAsync(a.p, args, a.bytes(), cudaMemcpyHostToDevice, st.s));
    else CUDA_TRY(cudaMemsetAsync(a.p, 0, a.bytes(), st.s));
    launch_rng_script(kind, seed, iteration, ant, derive, o.p, a.p, r.p, count, st.s);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out, r.p, r.bytes(), cudaMemcpyDeviceToHost, st.s));
    CUDA_TRY(cudaStreamSynchronize(st.s));
    return ACS_OK;
}

// record-major device image -> the ABI's separate n*S ids, n*S vals, n tails
static void unpack_spm(const unsigned char *h, uint32_t stride, uint32_t S, uint32_t n, uint32_t *ids,
                       double *vals, uint32_t *tail) {
    for (uint32_t u = 0; u < n; ++u) {
        const unsigned char *r = h + static_cast<size_t>(u) * stride;
        if (vals) std::memcpy(vals + static_cast<size_t>(u) * S, r, 8u * S);
        if (ids) std::memcpy(ids + static_cast<size_t>(u) * S, r + 8u * S, 4u * S);
        if (tail) std::memcpy(tail + u, r + 12u * S, 4u);
    }
}

int acs_gpu_spm_script(uint32_t n, uint32_t slots, double tau_min, double rho, double tau0,
                       double alpha, const uint32_t *ops, const int64_t *l_gb, uint32_t count,
                       int device, double *out, uint32_t *ids, double *vals, uint32_t *tail,
                       uint64_t *hits, uint64_t *misses) {
    if (n == 0 || slots == 0 || !ops || count == 0) return fail(ACS_E_ARG, "bad spm script");
    for (uint32_t i = 0; i < count; ++i) {
        if (ops[3 * i] >= n || ops[3 * i + 1] >= n || ops[3 * i + 2] > 2)
            return fail(ACS_E_ARG, "spm script op out of range");
        if (ops[3 * i + 2] == 1 && (!l_gb || l_gb[i] <= 0)) return fail(ACS_E_ARG, "global op needs l_gb > 0");
    }
    if (int rc = set_device(device)) return rc;
    Stream st;
    if (int rc = st.create()) return rc;
    DBuf<unsigned char> dspm;
    DBuf<uint32_t> dops;
    DBuf<double> dout;
    DBuf<int64_t> dl;
    DBuf<unsigned long long> hm;
    const uint32_t stride = SpmMem::stride_for(slots);
    CUDA_TRY(dspm.alloc(static_cast<size_t>(n) * stride));
    const SpmMem M{dspm.p, stride, slots};
    CUDA_TRY(dops.alloc(3ull * count));
    CUDA_TRY(dout.alloc(count));
    CUDA_TRY(dl.alloc(count));
    CUDA_TRY(hm.alloc(2));
    launch_spm_init(M, n, tau_min, st.s);
    CUDA_TRY(cudaMemcpyAsync(dops.p, ops, dops.bytes(), cudaMemcpyHostToDevice, st.s));
    if (l_gb) CUDA_TRY(cudaMemcpyAsync(dl.p, l_gb, dl.bytes(), cudaMemcpyHostToDevice, st.s));
    else CUDA_TRY(cudaMemsetAsync(dl.p, 0, dl.bytes(), st.s));
    CUDA_TRY(cudaMemsetAsync(hm.p, 0, hm.bytes(), st.s));
    const double c_l = 1.0 - rho, c_0 = rho * tau0, c_g = 1.0 - alpha;
    launch_spm_script(M, tau_min, c_l, c_0, alpha, c_g, dops.p, dl.p, count, dout.p, hm.p, st.s);
    CUDA_TRY(cudaGetLastError());
    unsigned long long h[2] = {0, 0};
    std::vector<unsigned char> img(dspm.bytes());
    if (out) CUDA_TRY(cudaMemcpyAsync(out, dout.p, dout.bytes(), cudaMemcpyDeviceToHost, st.s));
    CUDA_TRY(cudaMemcpyAsync(img.data(), dspm.p, img.size(), cudaMemcpyDeviceToHost, st.s));
    CUDA_TRY(cudaMemcpyAsync(h, hm.p, sizeof(h), cudaMemcpyDeviceToHost, st.s));
    CUDA_TRY(cudaStreamSynchronize(st.s));
    unpack_spm(img.data(), stride, slots, n, ids, vals, tail);
    if (hits) *hits = h[0];
    if (misses) *misses = h[1];
    return ACS_OK;
}

int acs_gpu_create(const acs_instance_desc *inst, const acs_params *p, int device, acs_gpu_ctx **out) {
    if (!out) return fail(ACS_E_ARG, "null ctx output");
    *out = nullptr;
    if (int rc = check_instance(inst)) return rc;
    if (!p) return fail(ACS_E_ARG, "null params");
    if (p->cl < 1 || p->cl > 32) return fail(ACS_E_ARG, "cl must be in [1, 32] on the GPU path");
    if (p->update_period < 1) return fail(ACS_E_ARG, "update_period (k) must be >= 1");
    if (p->variant > ACS_VARIANT_SPM_SYNC) return fail(ACS_E_ARG, "unknown variant");
    if (p->rng > ACS_RNG_PHILOX) return fail(ACS_E_ARG, "unknown rng");
    if (!(p->rho > 0.0 && p->rho < 1.0)) return fail(ACS_E_ARG, "rho (local evaporation) must be in (0,1)");
    if (!(p->alpha > 0.0 && p->alpha < 1.0)) return fail(ACS_E_ARG, "alpha (global evaporation) must be in (0,1)");
    if (p->q0 > 1.0) return fail(ACS_E_ARG, "q0 must be <= 1");
    if (!(p->beta >= 0.0)) return fail(ACS_E_ARG, "beta must be >= 0");
    const bool spm = p->variant == ACS_VARIANT_SPM || p->variant == ACS_VARIANT_SPM_SEQ ||
                     p->variant == ACS_VARIANT_SPM_SYNC;
    if (spm && !(p->slots == 1 || p->slots == 2 || p->slots == 4 || p->slots == 8 || p->slots == 16))
        return fail(ACS_E_ARG, "slots must be one of 1,2,4,8,16");
    if (int rc = set_device(device)) return rc;

    auto *c = new acs_gpu_ctx();
    std::unique_ptr<acs_gpu_ctx> guard(c);
    c->device = device;
    c->params = *p;
    c->n = inst->n;
    c->m = p->ants ? p->ants : inst->n;
    c->L = p->cl < inst->n - 1 ? p->cl : inst->n - 1;
    c->S = spm ? p->slots : 0;
    if (int rc = c->stream.create()) return rc;
    cudaStream_t s = c->stream.s;
    const PoolScope pool_scope(device, s);
    if (int rc = c->inst.upload(inst, true, s)) return rc;
    const DevInstance &I = c->inst.view;
    const uint32_t n = c->n;
    const int bint = beta_int_of(p->beta);
    if (bint < 0) {
        // non-integral beta: eta^beta per integer distance, host pow (bit-identical
        // to the oracle's), bounded by the bounding-box diagonal
        double x0 = inst->xs[0], x1 = x0, y0 = inst->ys[0], y1 = y0;
        for (uint32_t i = 1; i < n; ++i) {
            x0 = std::min(x0, inst->xs[i]); x1 = std::max(x1, inst->xs[i]);
            y0 = std::min(y0, inst->ys[i]); y1 = std::max(y1, inst->ys[i]);
        }
        double diag = std::sqrt((x1 - x0) * (x1 - x0) + (y1 - y0) * (y1 - y0));
        if (inst->edge_weight_type == ACS_ATT) diag = diag / std::sqrt(10.0);
        if (!(diag < 1e9)) return fail(ACS_E_ARG, "non-integral beta: coordinate range too large for the eta^beta table");
        const uint32_t dmax = static_cast<uint32_t>(std::ceil(diag)) + 2;
        std::vector<double> tab(static_cast<size_t>(dmax) + 1);
        for (uint32_t d = 0; d <= dmax; ++d) tab[d] = std::pow(1.0 / static_cast<double>(d > 0 ? d : 1), p->beta);
        CUDA_TRY(c->eta_d.alloc(tab.size()));
        CUDA_TRY(cudaMemcpyAsync(c->eta_d.p, tab.data(), c->eta_d.bytes(), cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaStreamSynchronize(s));  // the host table dies with this scope
        c->inst.view.eta_d = c->eta_d.p;
        c->inst.view.eta_dmax = dmax;
    }

    // candidate lists (K2) + packed rows
    CUDA_TRY(c->cand.alloc(static_cast<size_t>(n) * c->L));
    CUDA_TRY(c->rows.alloc(static_cast<size_t>(n) * 32));
    launch_topk(I, c->L, c->cand.p, s);
    launch_build_rows(I, c->cand.p, c->L, p->beta, bint, c->rows.p, s);
    CUDA_TRY(cudaGetLastError());
    // next-nearest rows after the candidate list (pruned exact fallback scan)
    {
        const uint32_t rest = n - 1 - c->L;
        const uint32_t ext_len = std::min<uint32_t>(ACS_EXT_MAX, (rest + 31) / 32 * 32);
        if (ext_len) {
            DBuf<uint64_t> keys, lower;
            CUDA_TRY(keys.alloc(static_cast<size_t>(n) * 32));
            CUDA_TRY(lower.alloc(n));
            CUDA_TRY(c->ext.alloc(static_cast<size_t>(n) * ext_len));
            launch_ext_rows(I, c->cand.p, c->L, ext_len, p->beta, bint, keys.p, lower.p, c->ext.p, s);
            CUDA_TRY(cudaGetLastError());
            CUDA_TRY(cudaStreamSynchronize(s));
        }
    }
    // tau0 = 1/(n * L_nn) from the NN tour from node 0
    CUDA_TRY(c->best_len.alloc(1));
    launch_nn_tour_cand(I, c->cand.p, c->L, 0, c->best_len.p, s, c->ext.p,
                        c->ext.p ? static_cast<uint32_t>(c->ext.count / n) : 0u);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(&c->nn_len, c->best_len.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    c->tau0 = 1.0 / (static_cast<double>(n) * static_cast<double>(c->nn_len));
    c->q0 = p->q0 < 0 ? default_q0(n) : p->q0;
    // The colony never reads the integer table again: the fallback scan needs
    // eta^beta, which is tabulated instead (same n <= 4096 cut-off), and the
    // few distances it needs come from the coordinates.
    if (c->inst.dist.p) {
        CUDA_TRY(c->etab.alloc(static_cast<size_t>(n) * n));
        launch_eta_table(I, p->beta, bint, c->etab.p, s);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaStreamSynchronize(s));
        c->inst.dist.release();
        c->inst.view.dist = nullptr;
        c->inst.view.etab = c->etab.p;
    }

    if (!spm) {
        CUDA_TRY(c->tau.alloc(static_cast<size_t>(n) * n));
        CUDA_TRY(c->tauc.alloc(static_cast<size_t>(n) * 32));
        launch_fill(c->tau.p, c->tau.count, c->tau0, s);
        launch_fill(c->tauc.p, c->tauc.count, c->tau0, s);
        if (p->variant == ACS_VARIANT_ATOMIC || p->variant == ACS_VARIANT_DEFERRED) {
            CUDA_TRY(c->cnt.alloc(static_cast<size_t>(n) * n));
            CUDA_TRY(c->cntc.alloc(static_cast<size_t>(n) * 32));
            CUDA_TRY(cudaMemsetAsync(c->cnt.p, 0, c->cnt.bytes(), s));
            CUDA_TRY(cudaMemsetAsync(c->cntc.p, 0, c->cntc.bytes(), s));
            // c_l^j (j < 512) and c_l^(512k) (k <= m/512 + 1) by repeated multiplication:
            // one copy's count per iteration is at most m (one traversal per ant)
            const double c_l = 1.0 - p->rho;
            const size_t hi = c->m / 512 + 2;
            std::vector<double> pw(512 + hi);
            pw[0] = 1.0;
            for (size_t j = 1; j < 512; ++j) pw[j] = pw[j - 1] * c_l;
            const double c512 = pw[511] * c_l;
            pw[512] = 1.0;
            for (size_t k = 1; k < hi; ++k) pw[512 + k] = pw[512 + k - 1] * c512;
            CUDA_TRY(c->pw.alloc(pw.size()));
            CUDA_TRY(cudaMemcpyAsync(c->pw.p, pw.data(), c->pw.bytes(), cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaStreamSynchronize(s));
        }
    } else {
        const uint32_t stride = SpmMem::stride_for(c->S);
        CUDA_TRY(c->spm.alloc(static_cast<size_t>(n) * stride));
        c->spm_mem = SpmMem{c->spm.p, stride, c->S};
        launch_spm_init(c->spm_mem, n, c->tau0, s);
    }
    CUDA_TRY(c->routes.alloc(static_cast<size_t>(c->m) * n));
    CUDA_TRY(c->lens.alloc(c->m));
    CUDA_TRY(c->best_tour.alloc(n));
    CUDA_TRY(c->iter.alloc(1));
    CUDA_TRY(c->counters.alloc(kNumCounters));
    CUDA_TRY(c->stats.alloc(64));
    CUDA_TRY(cudaMemsetAsync(c->iter.p, 0, sizeof(uint64_t), s));
    CUDA_TRY(cudaMemsetAsync(c->counters.p, 0, c->counters.bytes(), s));
    CUDA_TRY(cudaMemsetAsync(c->best_tour.p, 0, c->best_tour.bytes(), s));
    const int64_t none = LLONG_MAX;
    CUDA_TRY(cudaMemcpyAsync(c->best_len.p, &none, sizeof(int64_t), cudaMemcpyHostToDevice, s));

    if (p->variant == ACS_VARIANT_DEFERRED) {
        c->deferred = DevDeferred{1};
    }
    if (p->variant == ACS_VARIANT_SPM_SYNC) {
        // the apply pass sorts the step's 2m ops in one CTA's shared memory
        // above 8192 ants the step's record operations are sorted device-wide (cub)
        CUDA_TRY(c->sy_ants.alloc(static_cast<size_t>(c->m) * spm_sync_ant_bytes()));
        CUDA_TRY(c->sy_vis.alloc(static_cast<size_t>(c->m) * I.words));
        CUDA_TRY(c->sy_ops.alloc(static_cast<size_t>(c->m) * 2));
        c->spm_sync = DevSpmSync{c->sy_ants.p, c->sy_vis.p, c->sy_ops.p, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
        if (c->m > 8192 || std::getenv("ACS_SSYNC_WIDE")) {
            const size_t count = static_cast<size_t>(c->m) * 2;
            CUDA_TRY(c->sy_keys.alloc(2 * count));
            CUDA_TRY(c->sy_idx.alloc(2 * count));
            const size_t tmp = spm_sync_sort_tmp_bytes(static_cast<uint32_t>(count));
            CUDA_TRY(c->sy_tmp.alloc(tmp));
            DevSpmSync &Y = c->spm_sync;
            Y.keys_in = c->sy_keys.p;
            Y.keys_out = c->sy_keys.p + count;
            Y.idx_in = c->sy_idx.p;
            Y.idx_out = c->sy_idx.p + count;
            Y.sort_tmp = c->sy_tmp.p;
            Y.sort_tmp_bytes = tmp;
        }
    }

    DevColony &C = c->colony;
    C.m = c->m;
    C.L = c->L;
    C.k = p->update_period;
    C.S = c->S;
    C.q0 = c->q0;
    C.q0_k = static_cast<uint64_t>(std::floor(c->q0 * 9007199254740992.0));  // exact: q0 * 2^53
    C.beta = p->beta;
    C.beta_int = bint;
    C.c_l = 1.0 - p->rho;
    C.c_0 = p->rho * c->tau0;
    C.tau_min = c->tau0;
    C.seed = p->seed;
    C.rows = c->rows.p;
    C.ext = c->ext.p;
    C.ext_len = c->ext.p ? static_cast<uint32_t>(c->ext.count / n) : 0;
    C.tau_bound = c->tau0 * (1.0 + 0x1.0p-29);
    if (C.ext_len) {
        CUDA_TRY(c->hot.alloc(static_cast<size_t>(n) * kHot));
        CUDA_TRY(c->hot_cnt.alloc(n));
        CUDA_TRY(cudaMemsetAsync(c->hot_cnt.p, 0, n * sizeof(uint32_t), s));
        C.hot = c->hot.p;
        C.hot_cnt = c->hot_cnt.p;
        // without an eta^beta table (n > 4096) a fallback the ext rows cannot
        // settle continues over a uniform grid, about two nodes per cell
        if (!I.etab && I.type != ACS_ATT && !std::getenv("ACS_NO_GRID")) {
            double x0 = inst->xs[0], x1 = x0, y0 = inst->ys[0], y1 = y0;
            for (uint32_t i = 1; i < n; ++i) {
                x0 = std::min(x0, inst->xs[i]); x1 = std::max(x1, inst->xs[i]);
                y0 = std::min(y0, inst->ys[i]); y1 = std::max(y1, inst->ys[i]);
            }
            const uint32_t g = std::max<uint32_t>(1, static_cast<uint32_t>(std::ceil(std::sqrt(n / 2.0))));
            const double w = std::max(x1 - x0, y1 - y0);
            const double h = w > 0 ? w / g : 1.0;
            auto cell_of = [&](uint32_t i) {
                const uint32_t cx = std::min<uint32_t>(g - 1, static_cast<uint32_t>((inst->xs[i] - x0) / h));
                const uint32_t cy = std::min<uint32_t>(g - 1, static_cast<uint32_t>((inst->ys[i] - y0) / h));
                return cy * g + cx;
            };
            std::vector<uint32_t> start(static_cast<size_t>(g) * g + 1, 0), nodes(n);
            for (uint32_t i = 0; i < n; ++i) ++start[cell_of(i) + 1];
            for (size_t k = 1; k < start.size(); ++k) start[k] += start[k - 1];
            std::vector<uint32_t> fill(start.begin(), start.end() - 1);
            for (uint32_t i = 0; i < n; ++i) nodes[fill[cell_of(i)]++] = i;  // ascending id within a cell
            CUDA_TRY(c->cell_start.alloc(start.size()));
            CUDA_TRY(c->cell_nodes.alloc(n));
            CUDA_TRY(cudaMemcpyAsync(c->cell_start.p, start.data(), c->cell_start.bytes(), cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaMemcpyAsync(c->cell_nodes.p, nodes.data(), c->cell_nodes.bytes(), cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            C.cell_start = c->cell_start.p;
            C.cell_nodes = c->cell_nodes.p;
            C.grid_g = g;
            C.grid_x0 = x0;
            C.grid_y0 = y0;
            C.grid_h = h;
        }
    }
    C.tau = c->tau.p;
    C.tauc = c->tauc.p;
    C.cnt = c->cnt.p;
    C.cntc = c->cntc.p;
    C.pw_lo = c->pw.p;
    C.pw_hi = c->pw.p ? c->pw.p + 512 : nullptr;
    C.pw_hi_n = c->pw.p ? static_cast<uint32_t>(c->pw.count - 512) : 0;
    C.spm = c->spm_mem;
    C.routes = c->routes.p;
    C.lens = c->lens.p;
    C.counters = c->counters.p;
    C.iter = c->iter.p;
    DevBest &B = c->best;
    B.tour = c->best_tour.p;
    B.len = c->best_len.p;
    B.alpha = p->alpha;
    B.c_g = 1.0 - p->alpha;
    B.iter = c->iter.p;
    B.stats = c->stats.p;
    CUDA_TRY(cudaStreamSynchronize(s));
    *out = guard.release();
    return ACS_OK;
}

int acs_gpu_info(const acs_gpu_ctx *c, acs_ctx_info *info) {
    if (!c || !info) return fail(ACS_E_ARG, "null ctx/info");
    info->n = c->n;
    info->ants = c->m;
    info->list_len = c->L;
    info->slots = c->S;
    info->q0 = c->q0;
    info->tau0 = c->tau0;
    info->nn_len = c->nn_len;
    info->device_bytes = c->device_bytes();
    return ACS_OK;
}

// Iterations are issued in chunks of at most kIterChunk: the per-iteration
// construct events and the device stats buffer are bounded by the chunk, not
// by n_iter (a single call with a huge n_iter holds kIterChunk of each).
constexpr uint32_t kIterChunk = 1024;

int acs_gpu_iterate(acs_gpu_ctx *c, uint32_t n_iter, acs_iter_stats *out) {
    if (!c) return fail(ACS_E_ARG, "null ctx");
    if (n_iter == 0) return ACS_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    const uint32_t cap = std::min(n_iter, kIterChunk);
    if (c->stats.count < cap) {
        CUDA_TRY(c->stats.alloc(cap));
        c->best.stats = c->stats.p;
    }
    if (int rc = c->ensure_events(2 + 2 * static_cast<size_t>(cap))) return rc;
    cudaStream_t s = c->stream.s;
    const DevInstance &I = c->inst.view;
    const int variant = static_cast<int>(c->params.variant);
    const int rng = static_cast<int>(c->params.rng);
    float total = 0, construct = 0;
    for (uint32_t done = 0; done < n_iter;) {
        const uint32_t chunk = std::min(n_iter - done, kIterChunk);
        CUDA_TRY(cudaEventRecord(c->events[0], s));
        for (uint32_t i = 0; i < chunk; ++i) {
            CUDA_TRY(cudaEventRecord(c->events[2 + 2 * i], s));
            if (variant == ACS_VARIANT_DEFERRED) {
                if (launch_deferred(rng, I, c->colony, c->deferred, s) != 0)
                    return fail(ACS_E_CUDA, std::string("deferred: cooperative launch failed (colony not co-resident): ") +
                                                cudaGetErrorString(cudaGetLastError()));
            } else if (variant == ACS_VARIANT_SPM_SYNC) {
                if (launch_spm_sync(rng, I, c->colony, c->spm_sync, s) != 0)
                    return fail(ACS_E_CUDA, std::string("spm-sync launch failed: ") + cudaGetErrorString(cudaGetLastError()));
            } else {
                launch_construct(variant, rng, I, c->colony, s);
            }
            CUDA_TRY(cudaEventRecord(c->events[3 + 2 * i], s));
            launch_epilogue(!c->dense(), variant == ACS_VARIANT_ATOMIC, I, c->colony, c->best, i, s);
            CUDA_TRY(cudaGetLastError());
        }
        CUDA_TRY(cudaEventRecord(c->events[1], s));
        if (out)
            CUDA_TRY(cudaMemcpyAsync(out + done, c->stats.p, sizeof(acs_iter_stats) * chunk,
                                     cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, c->events[0], c->events[1]));
        total += ms;
        for (uint32_t i = 0; i < chunk; ++i) {
            CUDA_TRY(cudaEventElapsedTime(&ms, c->events[2 + 2 * i], c->events[3 + 2 * i]));
            construct += ms;
        }
        done += chunk;
    }
    c->last_total_ms = total;
    c->last_construct_ms = construct;
    return ACS_OK;
}

int acs_gpu_last_timing(const acs_gpu_ctx *c, float *total_ms, float *construct_ms) {
    if (!c) return fail(ACS_E_ARG, "null ctx");
    if (total_ms) *total_ms = c->last_total_ms;
    if (construct_ms) *construct_ms = c->last_construct_ms;
    return ACS_OK;
}

int acs_gpu_get_best(const acs_gpu_ctx *c, uint32_t *order, int64_t *len) {
    if (!c) return fail(ACS_E_ARG, "null ctx");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream.s;
    if (order) CUDA_TRY(cudaMemcpyAsync(order, c->best_tour.p, c->best_tour.bytes(), cudaMemcpyDeviceToHost, s));
    if (len) CUDA_TRY(cudaMemcpyAsync(len, c->best_len.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return ACS_OK;
}

int acs_gpu_set_best(acs_gpu_ctx *c, const uint32_t *order, int64_t len) {
    if (!c || !order) return fail(ACS_E_ARG, "null ctx/order");
    if (len <= 0) return fail(ACS_E_ARG, "len must be > 0");
    std::vector<uint8_t> seen(c->n, 0);
    for (uint32_t i = 0; i < c->n; ++i) {
        if (order[i] >= c->n || seen[order[i]]) return fail(ACS_E_ARG, "order is not a permutation");
        seen[order[i]] = 1;
    }
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream.s;
    if (!c->x_tour.p) {
        CUDA_TRY(c->x_tour.alloc(c->n));
        CUDA_TRY(c->x_len.alloc(1));
        CUDA_TRY(c->x_key.alloc(1));
    }
    CUDA_TRY(cudaMemcpyAsync(c->x_tour.p, order, c->x_tour.bytes(), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->x_len.p, &len, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    launch_adopt_best(c->x_tour.p, c->x_len.p, c->inst.view, c->best, s);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(s));
    return ACS_OK;
}

int acs_gpu_get_routes(const acs_gpu_ctx *c, uint32_t *routes, int64_t *lengths) {
    if (!c) return fail(ACS_E_ARG, "null ctx");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream.s;
    if (routes) CUDA_TRY(cudaMemcpyAsync(routes, c->routes.p, c->routes.bytes(), cudaMemcpyDeviceToHost, s));
    if (lengths) CUDA_TRY(cudaMemcpyAsync(lengths, c->lens.p, c->lens.bytes(), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return ACS_OK;
}

int acs_gpu_get_pheromone(const acs_gpu_ctx *c, double *tau) {
    if (!c || !tau) return fail(ACS_E_ARG, "null ctx/tau");
    if (!c->dense()) return fail(ACS_E_ARG, "selective-memory context has no dense matrix");
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaMemcpyAsync(tau, c->tau.p, c->tau.bytes(), cudaMemcpyDeviceToHost, c->stream.s));
    CUDA_TRY(cudaStreamSynchronize(c->stream.s));
    return ACS_OK;
}

int acs_gpu_get_selective(const acs_gpu_ctx *c, uint32_t *ids, double *vals, uint32_t *tail) {
    if (!c) return fail(ACS_E_ARG, "null ctx");
    if (c->dense()) return fail(ACS_E_ARG, "dense context has no selective memory");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream.s;
    std::vector<unsigned char> h(c->spm.bytes());
    CUDA_TRY(cudaMemcpyAsync(h.data(), c->spm.p, h.size(), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    unpack_spm(h.data(), c->spm_mem.stride, c->S, c->n, ids, vals, tail);
    return ACS_OK;
}

int acs_gpu_get_candidates(const acs_gpu_ctx *c, uint32_t *flat) {
    if (!c || !flat) return fail(ACS_E_ARG, "null ctx/flat");
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaMemcpyAsync(flat, c->cand.p, c->cand.bytes(), cudaMemcpyDeviceToHost, c->stream.s));
    CUDA_TRY(cudaStreamSynchronize(c->stream.s));
    return ACS_OK;
}

int acs_gpu_get_counters(const acs_gpu_ctx *c, acs_counters *o) {
    if (!c || !o) return fail(ACS_E_ARG, "null ctx/out");
    unsigned long long h[kNumCounters];
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaMemcpyAsync(h, c->counters.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream.s));
    CUDA_TRY(cudaStreamSynchronize(c->stream.s));
    o->local_updates = h[kCntUpdates];
    o->hits = h[kCntHits];
    o->misses = h[kCntMisses];
    o->fallback_steps = h[kCntFallback];
    o->greedy_steps = h[kCntGreedy];
    o->roulette_steps = h[kCntRoulette];
    o->cas_retries = h[kCntCasRetry];
    o->iterations = h[kCntIters];
    o->fallback_elems = h[kCntFallbackElems];
    o->fallback_full = h[kCntFallbackFull];
    o->relaxed_writes = h[kCntRelaxedWrites];
    o->lost_updates = h[kCntLost];
    o->fallback_grid = h[kCntFallbackGrid];
    return ACS_OK;
}

void acs_gpu_destroy(acs_gpu_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream.s);
    delete c;
}

int acs_gpu_run(const acs_instance_desc *inst, const acs_params *params, uint64_t iterations,
                int device, uint32_t *best_order, int64_t *best_len, int64_t *trace) {
    if (iterations == 0) return fail(ACS_E_ARG, "iterations must be > 0");
    acs_gpu_ctx *c = nullptr;
    if (int rc = acs_gpu_create(inst, params, device, &c)) return rc;
    std::unique_ptr<acs_gpu_ctx, void (*)(acs_gpu_ctx *)> guard(c, acs_gpu_destroy);
    std::vector<acs_iter_stats> st;
    uint64_t done = 0;
    while (done < iterations) {
        const uint32_t chunk = static_cast<uint32_t>(std::min<uint64_t>(iterations - done, 1024));
        st.resize(chunk);
        if (int rc = acs_gpu_iterate(c, chunk, st.data())) return rc;
        if (trace)
            for (uint32_t i = 0; i < chunk; ++i) trace[done + i] = st[i].global_best_len;
        done += chunk;
    }
    return acs_gpu_get_best(c, best_order, best_len);
}

// ---------------------------------------------------------------- islands

int acs_gpu_nccl_unique_id(void *uid) {
    if (!uid) return fail(ACS_E_ARG, "null unique id buffer");
    if (int rc = g_nccl.load()) return rc;
    nccl_uid id;
    const int r = g_nccl.get_unique_id(&id);
    if (r != 0) return fail(ACS_E_NCCL, std::string("ncclGetUniqueId: ") + (g_nccl.error_string ? g_nccl.error_string(r) : "?"));
    std::memcpy(uid, &id, sizeof(id));
    return ACS_OK;
}

int acs_gpu_island_init(acs_gpu_ctx *c, const void *uid, int nranks, int rank) {
    if (!c || !uid || nranks < 1 || rank < 0 || rank >= nranks) return fail(ACS_E_ARG, "bad island init args");
    if (nranks > kIslandMaxRanks) return fail(ACS_E_ARG, "island model supports at most 65536 ranks");
    if (int rc = g_nccl.load()) return rc;
    CUDA_TRY(cudaSetDevice(c->device));
    nccl_uid id;
    std::memcpy(&id, uid, sizeof(id));
    const int r = g_nccl.comm_init_rank(&c->comm, nranks, id, rank);
    if (r != 0) return fail(ACS_E_NCCL, std::string("ncclCommInitRank: ") + (g_nccl.error_string ? g_nccl.error_string(r) : "?"));
    c->rank = rank;
    c->nranks = nranks;
    if (!c->x_tour.p) {
        CUDA_TRY(c->x_tour.alloc(c->n));
        CUDA_TRY(c->x_len.alloc(1));
        CUDA_TRY(c->x_key.alloc(1));
    }
    return ACS_OK;
}

int acs_gpu_island_exchange_local(acs_gpu_ctx *const *ctxs, int count, int64_t *global_best_len) {
    if (!ctxs || count < 1) return fail(ACS_E_ARG, "island_exchange_local: no colonies");
    if (count > kIslandMaxRanks) return fail(ACS_E_ARG, "island model supports at most 65536 ranks");
    acs_gpu_ctx *lead = ctxs[0];
    for (int i = 0; i < count; ++i) {
        if (!ctxs[i]) return fail(ACS_E_ARG, "island_exchange_local: null ctx");
        if (ctxs[i]->device != lead->device || ctxs[i]->n != lead->n)
            return fail(ACS_E_ARG, "island_exchange_local: colonies must share the device and the instance size");
        for (int j = 0; j < i; ++j)
            if (ctxs[j] == ctxs[i]) return fail(ACS_E_ARG, "island_exchange_local: duplicate ctx");
    }
    CUDA_TRY(cudaSetDevice(lead->device));
    cudaStream_t s = lead->stream.s;
    const uint32_t n = lead->n;
    for (int i = 0; i < count; ++i) {
        acs_gpu_ctx *c = ctxs[i];
        if (!c->x_tour.p) {
            CUDA_TRY(c->x_tour.alloc(n));
            CUDA_TRY(c->x_len.alloc(1));
            CUDA_TRY(c->x_key.alloc(1));
        }
    }
    if (lead->xl_keys.count < static_cast<size_t>(count)) {
        CUDA_TRY(lead->xl_keys.alloc(count));
        CUDA_TRY(lead->xl_tours.alloc(count));
    }
    if (!lead->xl_sum.p) CUDA_TRY(lead->xl_sum.alloc(n));
    // order: every colony's pending iterations before the exchange, the
    // exchange before any colony's next iteration
    std::vector<cudaEvent_t> ev(count);
    for (int i = 0; i < count; ++i) CUDA_TRY(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    struct EvGuard {
        std::vector<cudaEvent_t> &e;
        ~EvGuard() { for (cudaEvent_t x : e) cudaEventDestroy(x); }
    } eg{ev};
    for (int i = 1; i < count; ++i) {
        CUDA_TRY(cudaEventRecord(ev[i], ctxs[i]->stream.s));
        CUDA_TRY(cudaStreamWaitEvent(s, ev[i], 0));
    }
    std::vector<const uint32_t *> tours(count);
    for (int i = 0; i < count; ++i) {
        launch_island_pack(ctxs[i]->best_len.p, i, lead->xl_keys.p + i, s);
        tours[i] = ctxs[i]->x_tour.p;
    }
    CUDA_TRY(cudaMemcpyAsync(lead->xl_tours.p, tours.data(), sizeof(const uint32_t *) * count,
                             cudaMemcpyHostToDevice, s));
    launch_island_min(lead->xl_keys.p, count, lead->x_key.p, s);               // = min-allreduce
    for (int i = 0; i < count; ++i)
        launch_island_mask(lead->x_key.p, i, ctxs[i]->best_tour.p, n, ctxs[i]->x_tour.p, ctxs[i]->x_len.p, s);
    launch_island_sum(lead->xl_tours.p, count, n, lead->xl_sum.p, s);         // = sum-allreduce
    for (int i = 0; i < count; ++i)
        launch_adopt_best(lead->xl_sum.p, lead->x_len.p, ctxs[i]->inst.view, ctxs[i]->best, s);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(ev[0], s));
    for (int i = 1; i < count; ++i) CUDA_TRY(cudaStreamWaitEvent(ctxs[i]->stream.s, ev[0], 0));
    if (global_best_len)
        CUDA_TRY(cudaMemcpyAsync(global_best_len, lead->x_len.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    // the host pointer table is read by the copy above; events die with the guard
    CUDA_TRY(cudaStreamSynchronize(s));
    return ACS_OK;
}

}  // extern "C"

extern "C" int acs_gpu_island_exchange(acs_gpu_ctx *c, int64_t *global_best_len) {
    if (!c) return fail(ACS_E_ARG, "null ctx");
    if (!c->comm) return fail(ACS_E_NCCL, "island not initialised (acs_gpu_island_init)");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream.s;
    // 1. key = L_gb << 16 | rank (kNoIslandKey before the first tour); min over ranks -> best colony, ties to the lowest rank
    launch_island_pack(c->best_len.p, c->rank, c->x_key.p, s);
    CUDA_TRY(cudaGetLastError());
    int r = g_nccl.all_reduce(c->x_key.p, c->x_key.p, 1, kNcclInt64, kNcclMin, c->comm, s);
    if (r != 0) return fail(ACS_E_NCCL, "ncclAllReduce(min) failed");
    // 2. winner contributes its tour, everyone else zeros: a sum-allreduce is
    //    a broadcast whose root is only known on the device (no host round trip)
    launch_island_mask(c->x_key.p, c->rank, c->best_tour.p, c->n, c->x_tour.p, c->x_len.p, s);
    CUDA_TRY(cudaGetLastError());
    r = g_nccl.all_reduce(c->x_tour.p, c->x_tour.p, c->n, kNcclUint32, kNcclSum, c->comm, s);
    if (r != 0) return fail(ACS_E_NCCL, "ncclAllReduce(sum) failed");
    // 3. adopt if strictly better
    launch_adopt_best(c->x_tour.p, c->x_len.p, c->inst.view, c->best, s);
    CUDA_TRY(cudaGetLastError());
    if (global_best_len) {
        CUDA_TRY(cudaMemcpyAsync(global_best_len, c->x_len.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
    return ACS_OK;
}
