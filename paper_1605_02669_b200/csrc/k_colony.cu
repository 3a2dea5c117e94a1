// k_colony.cu -- per-iteration kernels of the ACS hot path (sm_100a).
//
//   K4 k_tour_lean         whole tour per launch, warp per ant, lane per candidate slot,
//                          the paper's configuration (k = 1, 32-slot lists):
//                          ATOMIC (red.add counters, CONSISTENT) / RELAXED (ACS-GPU-Alt)
//   K4 k_construct_dense   the same for any k and list length; SEQ (one warp, bit-exact)
//   K4 k_spm_lean          selective pheromone memory (ACS-GPU-SPM), k = 1, s = 8
//   K4 k_construct_spm     the same for any k / s; SPM SEQ
//   K3 k_deferred          step-synchronous deferred variant (SPEC SYNC, bit-exact)
//   K3 k_ssync_*           SYNC x SELECTIVE (spm-sync, bit-exact)
//   K7 k_best              select_best (ties -> lowest ant) + strict is_better + stats
//   K7 k_global_*          global update on the global-best edges only (D3)
//
// The selection loop is a dependent chain (row(cur) -> scores -> argmax -> row(v)).
// Each step issues ONE coalesced 512 B load of the immutable packed row and ONE
// coalesced 256 B load of candidate-ordered pheromone; the next row is prefetched
// as soon as v is known, so the CAS of the ATOMIC variant and the bookkeeping
// overlap the next dependent load instead of adding to it.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include <cooperative_groups.h>
#include <type_traits>
#include <cub/device/device_radix_sort.cuh>

#include "../../include/acs_gpu.h"
#include "acs_common.cuh"

namespace acs_dev {

namespace cg = cooperative_groups;

struct Step {
    uint32_t v;        // chosen node
    int pos;           // candidate position, -1 for fallback
    uint32_t mirror;   // position of cur in v's list, kNoMirror if absent
    double tau_old;    // trail value the selection read for (cur, v)
    int32_t d;         // distance(cur, v)
    int kind;          // 0 greedy, 1 roulette, 2 fallback
};

// Per-lane running best of a full-scan fallback (score, node, trail value).
struct ScanBest {
    double bs = 0.0, bt = 0.0;
    uint32_t bv = 0xffffffffu;
    bool have = false;
};

// Full scan (Alg.2 l.18) of the unvisited nodes in bitmask words
// [wb, we): per-lane argmax of tau*eta^beta, nodes ascending within a lane, so
// a strict > keeps the lowest id.  The whole fallback is this over [0, words)
// followed by finish_scan; the deferred kernel splits the range over the warps
// of a CTA and combines the per-warp results (argmax, ties -> lowest id).
template <class TauFn>
__device__ __forceinline__ void full_scan_range(const DevInstance &I, const DevColony &C,
                                                const uint32_t *vis, uint32_t cur, TauFn tau_of, int lane,
                                                uint32_t wb, uint32_t we, ScanBest &b) {
    const double xc = __ldg(I.xs + cur), yc = __ldg(I.ys + cur);
    const double *erow = I.etab ? I.etab + static_cast<size_t>(cur) * I.n : nullptr;
    auto eta_of = [&](uint32_t v) -> double {
        if (erow) return __ldg(erow + v);
        return eta_beta_i(I, tsplib_distance(I.type, xc, yc, __ldg(I.xs + v), __ldg(I.ys + v)), C.beta,
                          C.beta_int);
    };
    const uint32_t last = I.words - 1;
    const uint32_t tail_mask = (I.n & 31) ? ((1u << (I.n & 31)) - 1u) : 0xffffffffu;
#ifndef ACS_COMPACT_ALWAYS
#define ACS_COMPACT_ALWAYS 0
#endif
    if (erow && !ACS_COMPACT_ALWAYS) {
        // With an eta^beta table (n <= 4096): coalesced 32-node chunks, four in
        // flight, fully visited chunks skipped on the broadcast bitmask word.
        constexpr int kChunks = 4;  // 8 independent loads per lane (8 chunks spill at the cap)
        for (uint32_t w = wb; w < we; w += kChunks) {
            uint32_t f[kChunks];
            uint32_t any = 0;
#pragma unroll
            for (int j = 0; j < kChunks; ++j) {
                f[j] = (w + j < we) ? ~vis[w + j] : 0u;
                if (w + j == last) f[j] &= tail_mask;
                any |= f[j];
            }
            if (any == 0u) continue;  // warp-uniform: all visited
            double t[kChunks], e[kChunks];
#pragma unroll
            for (int j = 0; j < kChunks; ++j) {
                const uint32_t v = (w + j) * 32 + lane;
                const bool act = (f[j] >> lane) & 1u;
                t[j] = tau_of(v, act);  // called by every lane (the SPM lookup shuffles)
                e[j] = act ? __ldg(erow + v) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < kChunks; ++j) {
                if ((f[j] >> lane) & 1u) {  // ascending v within the lane: strict > keeps the lowest id
                    const double sc = __dmul_rn(t[j], e[j]);
                    if (!b.have || sc > b.bs) { b.have = true; b.bs = sc; b.bv = (w + j) * 32 + lane; b.bt = t[j]; }
                }
            }
        }
    } else {
        // Without the table (n > 4096) eta^beta costs a sqrt and a pow per node, so
        // only the unvisited ones are touched.  Compacted scan: the unvisited nodes of each group of 32 bitmask words are
        // enumerated 32 per round, one per lane -- a warp prefix sum of the words'
        // popcounts, a shuffle search for the owning word, __fns for the bit -- and
        // the tau / eta^beta loads of 4 rounds are in flight together.  The cost
        // follows the number of unvisited nodes, not n: late in a tour, where the
        // pruned pass gives up, that is a few rounds instead of n/128 chunk loads.
        constexpr int kRounds = 4;
        for (uint32_t g = wb; g < we; g += 32) {
            const uint32_t w = g + lane;
            uint32_t u = w < we ? ~vis[w] : 0u;
            if (w == last) u &= tail_mask;
            const uint32_t pc = __popc(u);
            uint32_t incl = pc;
    #pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += t;
            }
            const uint32_t total = __shfl_sync(kFull, incl, 31);
            const uint32_t excl = incl - pc;
            for (uint32_t b0 = 0; b0 < total; b0 += kRounds * 32) {
                uint32_t vv[kRounds];
                bool act[kRounds];
                double t[kRounds], e[kRounds];
    #pragma unroll
                for (int r = 0; r < kRounds; ++r) {
                    const uint32_t idx = b0 + r * 32 + lane;
                    act[r] = idx < total;
                    int src = 0;  // the last lane whose exclusive offset is <= idx owns it
    #pragma unroll
                    for (int step = 16; step > 0; step >>= 1)
                        if (__shfl_sync(kFull, excl, src + step) <= idx) src += step;
                    const uint32_t ul = __shfl_sync(kFull, u, src);
                    const uint32_t k = idx - __shfl_sync(kFull, excl, src);
                    vv[r] = act[r] ? (g + src) * 32 + __fns(ul, 0, static_cast<int>(k) + 1) : 0u;
                }
    #pragma unroll
                for (int r = 0; r < kRounds; ++r) {
                    t[r] = tau_of(vv[r], act[r]);  // called by every lane (the SPM lookup shuffles)
                    e[r] = act[r] ? eta_of(vv[r]) : 0.0;
                }
    #pragma unroll
                for (int r = 0; r < kRounds; ++r) {
                    if (act[r]) {
                        const double sc = __dmul_rn(t[r], e[r]);
                        if (!b.have || sc > b.bs || (sc == b.bs && vv[r] < b.bv)) {
                            b.have = true; b.bs = sc; b.bv = vv[r]; b.bt = t[r];
                        }
                    }
                }
            }
        }
    }
}

// The fallback's chosen node `node` (warp-uniform) with its trail value:
// distance and the mirror slot (where cur sits in node's candidate row) --
// from `mirror` when the caller knows it (next-nearest rows carry it), else
// by a search of node's row (kMirrorUnknown).
constexpr uint32_t kMirrorUnknown = 0x100u;
__device__ __forceinline__ void finish_scan(const DevInstance &I, const DevColony &C, uint32_t cur,
                                            uint32_t node, double tau_old, int lane, Step &o,
                                            uint32_t mirror = kMirrorUnknown) {
    o.v = node;
    o.tau_old = tau_old;
    o.d = tsplib_distance(I.type, __ldg(I.xs + cur), __ldg(I.ys + cur), __ldg(I.xs + node), __ldg(I.ys + node));
    o.pos = -1;
    o.kind = 2;
    if (mirror != kMirrorUnknown) {
        o.mirror = mirror;
        return;
    }
    const uint32_t id = __ldg(&C.rows[static_cast<size_t>(node) * 32 + lane].x) & kIdMask;
    const unsigned mm = __ballot_sync(kFull, static_cast<uint32_t>(lane) < C.L && id == cur);
    o.mirror = mm ? static_cast<uint32_t>(__ffs(mm) - 1) : kNoMirror;
}

// Fallback (Alg.2 l.18): argmax tau*eta^beta over all unvisited
// nodes, ties -> lowest id, no RNG draw (P1).  An exact pruned pass first; if
// it cannot decide, the full scan -- or, with kDefer (the deferred kernel),
// o.kind = 3: the caller's CTA runs the full scan cooperatively.
#ifndef ACS_EXT_BATCH
#define ACS_EXT_BATCH 1  // free-running kernels (2 and 3 measured within noise, +2 % instructions)
#endif
#ifndef ACS_EXT_BATCH_DEFER
#define ACS_EXT_BATCH_DEFER 3  // the lockstep kernel: its step waits for the slowest fallback
#endif
template <bool kDefer = false, class TauFn>
__device__ __forceinline__ void fallback_scan(const DevInstance &I, const DevColony &C,
                                              const uint32_t *vis, uint32_t cur, TauFn tau_of,
                                              int lane, Step &o) {
    const double xc = __ldg(I.xs + cur), yc = __ldg(I.ys + cur);
    // Exact pruned pass.  Only the global update raises a trail above tau0
    // (local updates move it towards tau0), and every non-candidate edge it
    // ever touched is in cur's hot list.  So: score the hot list exactly, then
    // walk the next-nearest neighbours in distance order; once
    // tau_bound * eta^beta(last scanned) < best, no unscanned node can win or
    // tie, and the result equals the full scan's (argmax, ties -> lowest id).
    // The hot count, the hot list and the first next-nearest slice are
    // independent loads: issued together, so the common case (decided in the
    // first slice) costs two dependent L2 trips (ids, then trails) instead of five.
    const uint32_t hcnt = C.ext_len ? __ldg(C.hot_cnt + cur) : kHot + 1;
    const uint32_t hv = C.ext_len ? __ldg(C.hot + static_cast<size_t>(cur) * kHot + lane) : 0u;
    const uint4 *xrow = C.ext + static_cast<size_t>(cur) * C.ext_len;
    uint4 q = C.ext_len ? __ldg(xrow + lane) : make_uint4(kEmpty, 0u, 0u, 0u);
    if (hcnt <= kHot) {
        double bs = 0.0, bt = 0.0;
        uint32_t bv = 0xffffffffu, bm = kMirrorUnknown;  // bm: the best entry's mirror slot
        bool have = false;
        {
            const bool in_list = static_cast<uint32_t>(lane) < hcnt;
            const uint32_t v = in_list ? hv : 0u;
            const bool act = in_list && !visited(vis, v);
            const double tv = tau_of(v, act);
            if (act) {
                const double e = I.etab ? __ldg(I.etab + static_cast<size_t>(cur) * I.n + v)
                                        : eta_beta_i(I, tsplib_distance(I.type, xc, yc, __ldg(I.xs + v), __ldg(I.ys + v)),
                                                     C.beta, C.beta_int);
                have = true; bs = __dmul_rn(tv, e); bv = v; bt = tv;
            }
        }
        // kExtBatch slices per round trip: their id loads, then their trail
        // loads, are issued together; the slices are still decided one by one
        // in distance order, so the result is the slice-at-a-time walk's (a
        // fallback that walks the whole list pays ceil(slices / kExtBatch)
        // pairs of dependent L2 trips instead of one pair per slice)
        constexpr uint32_t kExtBatch = kDefer ? ACS_EXT_BATCH_DEFER : ACS_EXT_BATCH;
        if constexpr (kExtBatch == 1) {  // one slice per trip (the free-running kernels)
        for (uint32_t base = 0; base < C.ext_len; base += 32) {
            if (base) q = __ldg(xrow + base + lane);
            const bool in_list = q.x != kEmpty;
            const uint32_t qid = q.x & kIdMask;
            const bool act = in_list && !visited(vis, qid);
            const double tv = tau_of(in_list ? qid : 0u, act);
            if (act) {
                const double sc = __dmul_rn(tv, __hiloint2double(static_cast<int>(q.w), static_cast<int>(q.z)));
                if (!have || sc > bs || (sc == bs && qid < bv)) {
                    have = true; bs = sc; bv = qid; bt = tv; bm = q.x >> 24;
                }
            }
            double sb = bs;
            uint32_t node = have ? bv : 0xffffffffu;
            warp_argmax_node(sb, node, have);
            // the list ends inside this slice: every non-candidate node was scanned
            const bool exhausted = __any_sync(kFull, !in_list);
            const uint32_t lw = __shfl_sync(kFull, q.w, 31), lz = __shfl_sync(kFull, q.z, 31);
            const double bound = __dmul_rn(C.tau_bound, __hiloint2double(static_cast<int>(lw), static_cast<int>(lz)));
            if (node != 0xffffffffu && (exhausted || bound < sb)) {
                const unsigned owner = __ballot_sync(kFull, have && bv == node);
                const int src = __ffs(owner) - 1;
                finish_scan(I, C, cur, node, __shfl_sync(kFull, bt, src), lane, o, __shfl_sync(kFull, bm, src));
                return;
            }
        }
        } else {
        for (uint32_t base = 0; base < C.ext_len; base += 32 * kExtBatch) {
            uint4 qs[kExtBatch];
            qs[0] = base ? __ldg(xrow + base + lane) : q;
#pragma unroll
            for (uint32_t j = 1; j < kExtBatch; ++j)
                qs[j] = base + 32 * j < C.ext_len ? __ldg(xrow + base + 32 * j + lane) : make_uint4(kEmpty, 0u, 0u, 0u);
            double tvs[kExtBatch];
            bool acts[kExtBatch];
#pragma unroll
            for (uint32_t j = 0; j < kExtBatch; ++j) {
                const bool in_list = qs[j].x != kEmpty;
                const uint32_t qid = qs[j].x & kIdMask;
                acts[j] = in_list && !visited(vis, qid);
                tvs[j] = tau_of(in_list ? qid : 0u, acts[j]);
            }
#pragma unroll
            for (uint32_t j = 0; j < kExtBatch; ++j) {
                const uint4 qj = qs[j];
                const bool in_list = qj.x != kEmpty;
                const uint32_t qid = qj.x & kIdMask;
                const double tv = tvs[j];
                if (acts[j]) {
                    const double sc = __dmul_rn(tv, __hiloint2double(static_cast<int>(qj.w), static_cast<int>(qj.z)));
                    if (!have || sc > bs || (sc == bs && qid < bv)) {
                        have = true; bs = sc; bv = qid; bt = tv; bm = qj.x >> 24;
                    }
                }
                double sb = bs;
                uint32_t node = have ? bv : 0xffffffffu;
                warp_argmax_node(sb, node, have);
                // the list ends inside this slice: every non-candidate node was scanned
                const bool exhausted = __any_sync(kFull, !in_list);
                const uint32_t lw = __shfl_sync(kFull, qj.w, 31), lz = __shfl_sync(kFull, qj.z, 31);
                const double bound = __dmul_rn(C.tau_bound, __hiloint2double(static_cast<int>(lw), static_cast<int>(lz)));
                if (node != 0xffffffffu && (exhausted || bound < sb)) {
                    const unsigned owner = __ballot_sync(kFull, have && bv == node);
                    const int src = __ffs(owner) - 1;
                    finish_scan(I, C, cur, node, __shfl_sync(kFull, bt, src), lane, o, __shfl_sync(kFull, bm, src));
                    return;
                }
                if (base + 32 * j < C.ext_len) q = qj;  // the ring stage starts past the last slice
            }
        }
        }
        // Past the ext rows: rings of grid cells around cur, nearest first.
        // Every node closer than the last ext entry is a candidate or an ext
        // entry (scanned), so the walk starts at the first ring that can hold a
        // farther node; before ring r every unscanned node is at Euclidean
        // distance >= (r - 1) h, so its TSPLIB distance is >= floor((r - 1) h
        // - 0.5) and its score <= tau_bound * eta^beta of that: once that bound
        // is below the best, the result equals the full scan's (ties -> lowest id).
        if (C.grid_g && C.ext_len) {
            const int g = static_cast<int>(C.grid_g);
            const double h = C.grid_h;
            const int ccx = min(g - 1, static_cast<int>((xc - C.grid_x0) / h));
            const int ccy = min(g - 1, static_cast<int>((yc - C.grid_y0) / h));
            const double dext = static_cast<double>(__shfl_sync(kFull, q.y, 31));
            int r = max(0, static_cast<int>(ceil((dext - 0.5) / (h * 1.4142135623730951))) - 1);
            for (;; ++r) {
                double sb = bs;
                uint32_t node = have ? bv : 0xffffffffu;
                warp_argmax_node(sb, node, have);
                const double dlo = r >= 1 ? (r - 1) * h - 0.5 : 0.0;
                const int32_t dl = max(1, static_cast<int32_t>(floor(dlo)));
                const double bound = __dmul_rn(C.tau_bound, eta_beta_i(I, dl, C.beta, C.beta_int));
                const bool outside = r > g;  // every cell scanned
                if (node != 0xffffffffu && (outside || bound < sb)) {
                    const unsigned owner = __ballot_sync(kFull, have && bv == node);
                    const int src = __ffs(owner) - 1;
                    finish_scan(I, C, cur, node, __shfl_sync(kFull, bt, src), lane, o);
                    if (lane == 0) atomicAdd(C.counters + kCntFallbackGrid, 1ull);
                    return;
                }
                if (outside) break;  // no unvisited node at all: not reachable in a fallback
                // ring r: 8r cells (1 for r = 0), 32 at a time one per lane; their
                // nodes enumerated 32 per round in lockstep (tau_of may shuffle)
                const int ncell = r ? 8 * r : 1;
                for (int c0 = 0; c0 < ncell; c0 += 32) {
                    const int k = c0 + lane;
                    int cx = ccx, cy = ccy;
                    if (r) {
                        const int side = 2 * r + 1;
                        if (k < side) { cx = ccx - r + k; cy = ccy - r; }
                        else if (k < 2 * side) { cx = ccx - r + (k - side); cy = ccy + r; }
                        else if (k < 2 * side + (side - 2)) { cx = ccx - r; cy = ccy - r + 1 + (k - 2 * side); }
                        else { cx = ccx + r; cy = ccy - r + 1 + (k - 2 * side - (side - 2)); }
                    }
                    const bool inside = k < ncell && cx >= 0 && cy >= 0 && cx < g && cy < g;
                    const uint32_t cell = inside ? static_cast<uint32_t>(cy) * C.grid_g + static_cast<uint32_t>(cx) : 0u;
                    const uint32_t cs = inside ? __ldg(C.cell_start + cell) : 0u;
                    const uint32_t cnt = inside ? __ldg(C.cell_start + cell + 1) - cs : 0u;
                    uint32_t incl = cnt;
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const uint32_t t = __shfl_up_sync(kFull, incl, off);
                        if (lane >= off) incl += t;
                    }
                    const uint32_t total = __shfl_sync(kFull, incl, 31);
                    const uint32_t excl = incl - cnt;
                    for (uint32_t b0 = 0; b0 < total; b0 += 32) {
                        const uint32_t idx = b0 + lane;
                        int src = 0;  // the last lane whose exclusive offset is <= idx owns it
#pragma unroll
                        for (int step = 16; step > 0; step >>= 1)
                            if (__shfl_sync(kFull, excl, src + step) <= idx) src += step;
                        const uint32_t sc = __shfl_sync(kFull, cs, src);
                        const uint32_t ex = __shfl_sync(kFull, excl, src);
                        const uint32_t x = idx < total ? __ldg(C.cell_nodes + sc + (idx - ex)) : 0u;
                        const bool act = idx < total && !visited(vis, x);
                        const double tv = tau_of(x, act);  // every lane calls
                        if (act) {
                            const int32_t d = tsplib_distance(I.type, xc, yc, __ldg(I.xs + x), __ldg(I.ys + x));
                            const double scv = __dmul_rn(tv, eta_beta_i(I, d, C.beta, C.beta_int));
                            if (!have || scv > bs || (scv == bs && x < bv)) {
                                have = true; bs = scv; bv = x; bt = tv; bm = kMirrorUnknown;
                            }
                        }
                    }
                }
            }
        }
    }
    if (lane == 0) atomicAdd(C.counters + kCntFallbackFull, 1ull);
    if constexpr (kDefer) {
        o.kind = 3;
        return;
    }
    ScanBest b;
    full_scan_range(I, C, vis, cur, tau_of, lane, 0u, I.words, b);
    double s = b.bs;
    uint32_t node = b.have ? b.bv : 0xffffffffu;
    warp_argmax_node(s, node, b.have);
    const unsigned owner = __ballot_sync(kFull, b.have && b.bv == node);
    finish_scan(I, C, cur, node, __shfl_sync(kFull, b.bt, __ffs(owner) - 1), lane, o);
}

// The q draw of the next step, computed speculatively on a copy of the stream
// while the next row is in flight (it does not depend on the row) and
// committed only when that step's filtered candidate set is non-empty (P1).
// q = (x >> 11) * 2^-53 is exact, so q <= q0  <=>  (x >> 11) <= floor(q0 * 2^53):
// the comparison is done on the 53-bit integer (C.q0_k) without a conversion.
// Both engines expose peek()/advance(), so no copy of the stream is needed.
template <class RNG>
struct Lookahead {
    uint64_t q53;
    __device__ __forceinline__ void prepare(const RNG &rng) {
        q53 = rng.peek() >> 11;
        asm volatile("" : "+l"(q53));  // keep it here: no rematerialisation on the chain
    }
    __device__ __forceinline__ bool greedy(const DevColony &C) const { return q53 <= C.q0_k; }
};

// Philox4x32-10 evaluated 32 draws at a time, one per lane, for a warp that
// owns one ant.  Draw j of (seed, iteration, ant) is Philox::peek() at draw
// j, so the stream is bit-identical to the scalar engine (and to the oracle's
// PHILOX mode); what changes is the cost: one Philox evaluation per 32 draws
// instead of one per draw, and the q <= q0 test of every draw of the batch is
// a single ballot (qmask), so a greedy step reads one bit.
struct PhiloxWarp {
    Philox key;         // (seed, iteration, ant); key.draw unused
    uint64_t q0_k;
    uint64_t mine;      // draw base + lane
    uint32_t base;      // first draw of the current block of 32
    uint32_t off;       // draws consumed in this block
    uint32_t qsh;       // the block's greedy-test ballot shifted by off: bit 0 = next draw's

    __device__ __forceinline__ void fill() {
        Philox p = key;
        p.draw = base + (threadIdx.x & 31u);
        mine = p.peek();
        qsh = __ballot_sync(kFull, (mine >> 11) <= q0_k);
    }
    __device__ __forceinline__ void derive(uint64_t seed, uint64_t it, uint64_t a, uint64_t q0k) {
        key.derive(seed, it, a);
        q0_k = q0k;
        base = off = 0;
        fill();
    }
    __device__ __forceinline__ uint64_t peek() const { return shfl_u64(mine, static_cast<int>(off)); }
    __device__ __forceinline__ void advance() {
        qsh >>= 1;
        if (++off == 32u) {  // warp-uniform, once per 32 draws
            base += 32u;
            off = 0;
            fill();
        }
    }
    __device__ __forceinline__ uint64_t next() {
        const uint64_t r = peek();
        advance();
        return r;
    }
    __device__ __forceinline__ bool greedy_bit() const { return qsh & 1u; }
};

template <>
struct Lookahead<PhiloxWarp> {
    bool g;
    __device__ __forceinline__ void prepare(const PhiloxWarp &rng) { g = rng.greedy_bit(); }
    __device__ __forceinline__ bool greedy(const DevColony &) const { return g; }
};

// per-ant stream of a construction warp
template <class RNG>
__device__ __forceinline__ void rng_init(RNG &rng, const DevColony &C, uint64_t it, uint64_t a) {
    rng.derive(C.seed, it, a);
}
template <>
__device__ __forceinline__ void rng_init(PhiloxWarp &rng, const DevColony &C, uint64_t it, uint64_t a) {
    rng.derive(C.seed, it, a, C.q0_k);
}

// PhiloxWarp with the round-1 bookkeeping (the ballot shifted by the draw
// offset at every test).  The pre-shifted form is faster in every 96-register
// build but 8 % slower in the 72-register RELAXED build of multi-wave colonies
// (rnd10k: 25.9 vs 28.1 ms, where it changes what ptxas spills), so that one
// instantiation keeps this form.  Identical draws.
struct PhiloxWarpU {  // the same stream with an unshifted ballot (see below)
    Philox key;         // (seed, iteration, ant); key.draw unused
    uint64_t q0_k;
    uint64_t mine;      // draw base + lane
    uint32_t base, draw, qmask;

    __device__ __forceinline__ void fill() {
        Philox p = key;
        p.draw = base + (threadIdx.x & 31u);
        mine = p.peek();
        qmask = __ballot_sync(kFull, (mine >> 11) <= q0_k);
    }
    __device__ __forceinline__ void derive(uint64_t seed, uint64_t it, uint64_t a, uint64_t q0k) {
        key.derive(seed, it, a);
        q0_k = q0k;
        base = draw = 0;
        fill();
    }
    __device__ __forceinline__ uint64_t peek() const { return shfl_u64(mine, static_cast<int>(draw - base)); }
    __device__ __forceinline__ void advance() {
        if (++draw - base == 32u) {  // warp-uniform, once per 32 draws
            base += 32u;
            fill();
        }
    }
    __device__ __forceinline__ uint64_t next() {
        const uint64_t r = peek();
        advance();
        return r;
    }
    __device__ __forceinline__ bool greedy_bit() const { return (qmask >> (draw - base)) & 1u; }
};
template <>
struct Lookahead<PhiloxWarpU> {
    bool g;
    __device__ __forceinline__ void prepare(const PhiloxWarpU &rng) { g = rng.greedy_bit(); }
    __device__ __forceinline__ bool greedy(const DevColony &) const { return g; }
};
template <>
__device__ __forceinline__ void rng_init(PhiloxWarpU &rng, const DevColony &C, uint64_t it, uint64_t a) {
    rng.derive(C.seed, it, a, C.q0_k);
}

// Candidate branch (Eq.1 / Eq.2 over the filtered list, Alg.2 l.5-16) with the
// P1 draw protocol; falls through to fallback_scan when all are visited.
// Stream commit: roulette commits q (and draws r) here; for a greedy step
// (o.kind == 0) the caller commits q with rng.advance() AFTER issuing the next
// row load, which keeps the state transition off the dependent chain.
template <bool kDefer = false, bool kL32 = false, class RNG, class TauFn>
__device__ __forceinline__ void select_step(const DevInstance &I, const DevColony &C,
                                            const uint32_t *vis, uint32_t cur, uint4 el,
                                            double tau_lane, RNG &rng, const Lookahead<RNG> &la,
                                            double *scratch, int lane, TauFn tau_of, Step &o) {
    const uint32_t c = el.x & kIdMask;
    const bool valid = kL32 || static_cast<uint32_t>(lane) < C.L;  // kL32: full 32-slot lists
    const bool unv = valid && !visited(vis, c);
    const unsigned um = __ballot_sync(kFull, unv);
    if (um) {
        const double eb = __hiloint2double(static_cast<int>(el.w), static_cast<int>(el.z));
        const double score = unv ? __dmul_rn(tau_lane, eb) : 0.0;
        int pos;
        if (la.greedy(C)) {
            uint32_t v;
            warp_argmax_id(score, unv, c, lane, pos, v);  // um != 0: a lane is valid
            o.v = v;
            o.kind = 0;
        } else {
            rng.advance();  // commit q
            const double r = uniform01(rng);
            pos = warp_roulette_pos(score, um, r, scratch, lane);
            o.v = __shfl_sync(kFull, c, pos);
            o.kind = 1;
        }
        o.pos = pos;
        o.mirror = __shfl_sync(kFull, el.x >> 24, pos);
        o.d = static_cast<int32_t>(__shfl_sync(kFull, el.y, pos));
        o.tau_old = __shfl_sync(kFull, tau_lane, pos);
        return;
    }
    fallback_scan<kDefer>(I, C, vis, cur, tau_of, lane, o);
}

// Per-ant event counters, 32-bit (one tour has < n^2/2 fallback elements and
// n < 2^24 steps), flushed and reset once per ant.  greedy is derived at flush
// time as (steps - roulette - fallback).
struct WarpCounters {
    uint32_t fallback = 0, roulette = 0, updates = 0, hits = 0, misses = 0, fb_elems = 0;
#ifdef ACS_COUNT_LOST
    uint32_t writes = 0, lost = 0;  // per lane (the writing lanes differ), summed at flush
#endif
    // unvisited = n - t at step t: the elements a fallback scan touches
    __device__ __forceinline__ void count(int kind, uint32_t unvisited) {
        roulette += kind == 1;
        fallback += kind == 2;
        fb_elems += kind == 2 ? unvisited : 0u;
    }
    __device__ __forceinline__ void flush(unsigned long long *c, int lane, uint32_t steps) {
        if (lane == 0) {
            using ull = unsigned long long;
            if (updates) atomicAdd(c + kCntUpdates, static_cast<ull>(updates));
            if (hits) atomicAdd(c + kCntHits, static_cast<ull>(hits));
            if (misses) atomicAdd(c + kCntMisses, static_cast<ull>(misses));
            if (fallback) atomicAdd(c + kCntFallback, static_cast<ull>(fallback));
            if (steps) atomicAdd(c + kCntGreedy, static_cast<ull>(steps - roulette - fallback));
            if (roulette) atomicAdd(c + kCntRoulette, static_cast<ull>(roulette));
            if (fb_elems) atomicAdd(c + kCntFallbackElems, static_cast<ull>(fb_elems));
        }
#ifdef ACS_COUNT_LOST
        if (writes) atomicAdd(c + kCntRelaxedWrites, static_cast<unsigned long long>(writes));
        if (lost) atomicAdd(c + kCntLost, static_cast<unsigned long long>(lost));
        writes = lost = 0;
#endif
        fallback = roulette = updates = hits = misses = fb_elems = 0;
    }
};

// route buffered in registers: lane (t & 31) holds route[t]; one coalesced
// 128 B store per 32 steps.
__device__ __forceinline__ void route_put(uint32_t *route, uint32_t &rbuf, uint32_t t, uint32_t v,
                                          int lane) {
    if (static_cast<uint32_t>(lane) == (t & 31)) rbuf = v;
    if ((t & 31) == 31) route[(t & ~31u) + lane] = rbuf;
}
__device__ __forceinline__ void route_flush(uint32_t *route, uint32_t rbuf, uint32_t last,
                                            int lane) {
    if ((last & 31) != 31 && static_cast<uint32_t>(lane) <= (last & 31))
        route[(last & ~31u) + lane] = rbuf;
}

// The (up to) four copies of trail (u,v), one lane each: lane 0 tau[u][v],
// lane 1 tau[v][u], lane 2 tauc[u][pos], lane 3 tauc[v][mirror].
__device__ __forceinline__ double *copy_addr(const DevColony &C, uint32_t n, uint32_t u, uint32_t v,
                                             int pos, uint32_t mirror, int lane) {
    const bool odd = lane & 1;
    const bool dense = lane < 2;
    const uint32_t row = odd ? v : u;
    const uint32_t col = dense ? (odd ? u : v) : (odd ? mirror : static_cast<uint32_t>(pos));
    const bool ok = lane < 4 && (dense || col < 32u);
    double *base = dense ? C.tau : C.tauc;
    const uint32_t stride = dense ? n : 32u;
    return ok ? base + (static_cast<size_t>(row) * stride + col) : nullptr;
}

// closing edge (last -> start): its candidate position / mirror by row search
__device__ __forceinline__ void closing_slots(const DevColony &C, uint32_t last, uint32_t start,
                                              int lane, int &pos, uint32_t &mirror, int32_t &d,
                                              bool &have_d) {
    const uint4 el = __ldg(&C.rows[static_cast<size_t>(last) * 32 + lane]);
    const unsigned hit =
        __ballot_sync(kFull, static_cast<uint32_t>(lane) < C.L && (el.x & kIdMask) == start);
    pos = hit ? __ffs(hit) - 1 : -1;
    mirror = kNoMirror;
    have_d = hit != 0;
    d = 0;
    if (hit) {
        mirror = __shfl_sync(kFull, el.x >> 24, pos);
        d = static_cast<int32_t>(__shfl_sync(kFull, el.y, pos));
    } else {
        const uint32_t id2 = __ldg(&C.rows[static_cast<size_t>(start) * 32 + lane].x) & kIdMask;
        const unsigned mm = __ballot_sync(kFull, static_cast<uint32_t>(lane) < C.L && id2 == last);
        if (mm) mirror = static_cast<uint32_t>(__ffs(mm) - 1);
    }
}

// ============================================================ dense whole tour

// Trail value of an ATOMIC-variant copy: base b with c pending local updates,
// tau = f^c(b).  c <= 1 is the exact affine rule (so a lone ant -- and the
// SEQ parity test -- is bit-identical to the CAS/sequential result); c >= 2
// uses the closed form tau0 + c_l^c (b - tau0) with c_l^c from two small
// power tables (lo: c & 511, hi: c >> 9).
__device__ __forceinline__ double trail_value(double b, uint32_t c, const DevColony &C,
                                              const double *pw_lo, const double *pw_hi) {
    const double one = affine(b, C.c_l, C.c_0);
    double p = 1.0;
    if (c >= 2u) p = __dmul_rn(pw_lo[c & 511u], pw_hi[c >> 9]);
    const double closed = __dadd_rn(C.tau_min, __dmul_rn(p, __dsub_rn(b, C.tau_min)));
    return c == 0u ? b : (c == 1u ? one : closed);
}

__device__ __forceinline__ void red_add1(uint32_t *p) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

// index of copy `lane` (0: tau[u][v], 1: tau[v][u], 2: tauc[u][pos], 3: tauc[v][mirror])
// into the dense (n*n) or candidate (n*32) array; returns false when absent
// ATOMIC: a dense counter cnt[a][b] is bumped only when b has no slot in a's
// candidate row (no candidate copy of the entry is counted): the fallback
// scans, the only readers of dense trails during construction, never look at
// a's candidates (all visited), and the fold takes the count of such an entry
// from its candidate copy (k_fold_counts).  One red per step instead of two.
#ifndef ACS_DENSE_CAND_SKIP
#define ACS_DENSE_CAND_SKIP 1
#endif
// skip predicate for the dense lanes of copy_index (lane 0: (u, v), lane 1:
// (v, u)): the entry's candidate copy is bumped instead
__device__ __forceinline__ bool dense_counted_by_cand(int lane, int pos, uint32_t mirror, uint32_t lmax) {
    return ACS_DENSE_CAND_SKIP && (lane == 0 ? (pos >= 0 && pos < 32) : mirror < lmax);
}
__device__ __forceinline__ bool copy_index(uint32_t n, uint32_t u, uint32_t v, int pos,
                                           uint32_t mirror, int lane, bool &dense, size_t &idx) {
    const bool odd = lane & 1;
    dense = lane < 2;
    const uint32_t row = odd ? v : u;
    const uint32_t col = dense ? (odd ? u : v) : (odd ? mirror : static_cast<uint32_t>(pos));
    idx = static_cast<size_t>(row) * (dense ? n : 32u) + col;
    return lane < 4 && (dense || col < 32u);
}


// kMode 0 = RELAXED (ACS-GPU-Alt): plain relaxed stores of f(tau_old), lost
//           updates allowed; also SEQ when launched on one warp.
// kMode 1 = ATOMIC (CONSISTENT): every local update is one contention-free
//           `red.add` on a per-copy counter -- no update can be lost and no
//           ant ever waits on an atomic -- and readers see f^c(base).  The
//           iteration epilogue folds the counters back into the bases.
// The general kernel (any update period k, lists of up to 32 slots, one warp
// for SEQ); the paper's configuration (k = 1, 32-slot lists) runs k_tour_lean.
template <int kMode, class RNG, int kRegs = kMaxRegs>
__global__ void __maxnreg__(kRegs) k_construct_dense(DevInstance I, DevColony C) {
    constexpr bool kAtomic = kMode == 1;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    double *scratch = reinterpret_cast<double *>(smem) + wib * 32;
    // ATOMIC: c_l^c power tables staged in shared memory (the L1 is thrashed by
    // the row stream, so a global-table lookup on the chain costs an L2 trip)
    double *pw_lo = reinterpret_cast<double *>(smem) + wpb * 32;
    double *pw_hi = pw_lo + 512;
    const uint32_t pw_n = kAtomic ? 512 + C.pw_hi_n : 0;
    uint32_t *vis = reinterpret_cast<uint32_t *>(smem + (wpb * 32 + pw_n) * sizeof(double)) +
                    static_cast<size_t>(wib) * I.words;
    if constexpr (kAtomic) {
        for (uint32_t i = threadIdx.x; i < pw_n; i += blockDim.x) pw_lo[i] = C.pw_lo[i];
        __syncthreads();
    }
    const uint64_t it = *C.iter;
    const uint32_t n = I.n;
    WarpCounters wc;

    for (uint32_t a = blockIdx.x * wpb + wib; a < C.m; a += gridDim.x * wpb) {
        for (uint32_t i = lane; i < I.words; i += 32) vis[i] = 0;
        RNG rng;
        rng_init(rng, C, it, a);
        const uint32_t start = static_cast<uint32_t>(uniform_int(rng, n));  // P1.1
        size_t ri = static_cast<size_t>(start) * 32 + lane;
        uint4 el = __ldg(C.rows + ri);
        double tl = ld_relaxed(C.tauc + ri);
        uint32_t cl = kAtomic ? ld_relaxed_u32(C.cntc + ri) : 0u;
        __syncwarp();
        if (lane == 0) vis[start >> 5] |= 1u << (start & 31);
        __syncwarp();
        uint32_t *route = C.routes + static_cast<size_t>(a) * n;
        uint32_t rbuf = start, cur = start, kc = 0;
        long long len = 0;
        Lookahead<RNG> la;
        la.prepare(rng);
        // The copy tauc[v][mirror] of edge (u,v) is written one step late, by
        // the lane of row v whose candidate is u (RELAXED: from the value it
        // just loaded) -- row v is never written while its own load is in
        // flight, and u is visited, so the delay is invisible to this ant.
        uint32_t mprev = kEmpty;

        for (uint32_t t = 1; t < n; ++t) {
            // The copy of the previous edge in THIS row (cur -> prev) is written
            // by the lane holding prev, after the row's own load has completed.
            // Its operands depend on the row only, so they are formed here, off
            // the selection chain, and the store is issued after the next
            // row's loads.
            const bool mw = static_cast<uint32_t>(lane) < C.L && (el.x & kIdMask) == mprev;
            const size_t mi = static_cast<size_t>(cur) * 32 + lane;
            const double mval = kAtomic ? 0.0 : affine(tl, C.c_l, C.c_0);
            Step st;
            if constexpr (kAtomic) {
                const double tv = trail_value(tl, cl, C, pw_lo, pw_hi);
                select_step<false>(I, C, vis, cur, el, tv, rng, la, scratch, lane,
                            [&](uint32_t v, bool act) {
                                if (!act) return 0.0;
                                const size_t k = static_cast<size_t>(cur) * n + v;
                                return trail_value(ld_relaxed(C.tau + k), ld_relaxed_u32(C.cnt + k), C, pw_lo,
                                                   pw_hi);
                            },
                            st);
            } else {
                select_step<false>(I, C, vis, cur, el, tl, rng, la, scratch, lane,
                            [&](uint32_t v, bool act) {
                                return act ? ld_relaxed(C.tau + static_cast<size_t>(cur) * n + v) : 0.0;
                            },
                            st);
            }
            // Next dependent row load, issued as soon as v is known: the writes
            // below touch rows u (tauc, tau) and v of the DENSE matrix only --
            // the one copy in tauc row v is written a step late (above), because
            // a write to the same line behind a pending load measured ~30%
            // slower per step (profiles/README.md, v6).
            ri = static_cast<size_t>(st.v) * 32 + lane;
            el = __ldg(C.rows + ri);
            tl = ld_relaxed(C.tauc + ri);
            if constexpr (kAtomic) cl = ld_relaxed_u32(C.cntc + ri);
            if (mw) {
                if constexpr (kAtomic) red_add1(C.cntc + mi);
                else st_relaxed(C.tauc + mi, mval);
            }
            mprev = kEmpty;
            if (st.kind) wc.count(st.kind, n - t);  // greedy steps are derived at flush
            if (++kc == C.k) {  // D9 per-ant edge counter (warp-uniform)
                kc = 0;
                ++wc.updates;
                bool dense;
                size_t k;
                // lanes 0-2 now; lane 3's copy (tauc[v][mirror]) one step late, above
                if (lane < 3 && copy_index(n, cur, st.v, st.pos, st.mirror, lane, dense, k)) {
                    if constexpr (kAtomic) {
                        // lane 1's candidate copy is the late mirror one: counted iff mirror < L
                        if (!(dense && dense_counted_by_cand(lane, st.pos, st.mirror, C.L)))
                            red_add1((dense ? C.cnt : C.cntc) + k);
                    } else {
                        st_relaxed((dense ? C.tau : C.tauc) + k, affine(st.tau_old, C.c_l, C.c_0));
                    }
                }
                mprev = cur;
            }
            // commit a greedy step's q draw and peek the next one, off the chain
            if (st.kind == 0) rng.advance();
            la.prepare(rng);
            // every lane writes the same word: no divergent branch on the chain
            vis[st.v >> 5] |= 1u << (st.v & 31);
            len += st.d;
            route_put(route, rbuf, t, st.v, lane);
            cur = st.v;
            __syncwarp();
        }
        route_flush(route, rbuf, n - 1, lane);
        // last step's deferred mirror copy (el/tl hold row `cur`)
        if (static_cast<uint32_t>(lane) < C.L && (el.x & kIdMask) == mprev) {
            if constexpr (kAtomic) red_add1(C.cntc + static_cast<size_t>(cur) * 32 + lane);
            else st_relaxed(C.tauc + static_cast<size_t>(cur) * 32 + lane, affine(tl, C.c_l, C.c_0));
        }
        __syncwarp();

        // closing edge (cur -> start) is edge n of the ant (D9)
        int pos;
        uint32_t mirror;
        int32_t dclose;
        bool have_d;
        closing_slots(C, cur, start, lane, pos, mirror, dclose, have_d);
        if (!have_d)
            dclose = tsplib_distance(I.type, __ldg(I.xs + cur), __ldg(I.ys + cur), __ldg(I.xs + start),
                                     __ldg(I.ys + start));
        if (++kc == C.k) {
            ++wc.updates;
            bool dense;
            size_t k;
            if (copy_index(n, cur, start, pos, mirror, lane, dense, k)) {
                if constexpr (kAtomic) {
                    if (!(dense && dense_counted_by_cand(lane, pos, mirror, 32u)))
                        red_add1((dense ? C.cnt : C.cntc) + k);
                } else {
                    const double told = ld_relaxed(C.tau + static_cast<size_t>(cur) * n + start);
                    st_relaxed((dense ? C.tau : C.tauc) + k, affine(told, C.c_l, C.c_0));
                }
            }
        }
        if (lane == 0) C.lens[a] = len + dclose;
        wc.flush(C.counters, lane, n - 1);
        __syncwarp();
    }
}

// ============================================================ lean whole tour

#ifdef ACS_COUNT_LOST
__device__ __forceinline__ uint32_t xchg_lost(double *p, double v, double expect) {
    const unsigned long long old = atomicExch(reinterpret_cast<unsigned long long *>(p), dbits(v));
    return old != dbits(expect) ? 1u : 0u;
}
#endif

// Predicated single-instruction stores (no branch, no BSSY/BSYNC around them).
__device__ __forceinline__ void st_relaxed_if(bool p, double *ptr, double v) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q st.relaxed.gpu.global.b64 [%1], %2; }" ::"r"(
                     static_cast<int>(p)),
                 "l"(ptr), "l"(dbits(v))
                 : "memory");
}
__device__ __forceinline__ void red_add_if(bool p, uint32_t *ptr, uint32_t one) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q red.relaxed.gpu.global.add.u32 [%1], %2; }" ::"r"(
                     static_cast<int>(p)),
                 "l"(ptr), "r"(one)
                 : "memory");
}
__device__ __forceinline__ void st_u32_if(bool p, uint32_t *ptr, uint32_t v) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q st.global.u32 [%1], %2; }" ::"r"(static_cast<int>(p)),
                 "l"(ptr), "r"(v)
                 : "memory");
}

// ATOMIC trail value f^c(b) (trail_value) for the lean kernel: c_l^c from the
// static shared tables, every operand formed unconditionally and the three
// cases (c = 0, 1, >= 2) picked by selects -- no branch on the chain.
constexpr uint32_t kLeanPwHi = 64;  // c < 512 * 64 pending updates (m <= 31744)
template <bool kPw1 = false>
__device__ __forceinline__ double trail_value_sel(double b, uint32_t c, const DevColony &C, const double *pw) {
    // c < 512 * kLeanPwHi: the launcher runs this kernel only for m <= that
    // (kPw1: pw is the one-table c_l^c, c <= m)
    const double p = kPw1 ? pw[c] : __dmul_rn(pw[c & 511u], pw[512u + (c >> 9)]);
    const double one = affine(b, C.c_l, C.c_0);
    const double closed = __dadd_rn(C.tau_min, __dmul_rn(p, __dsub_rn(b, C.tau_min)));
    const double x = c >= 2u ? closed : one;
    return c == 0u ? b : x;
}
__device__ __forceinline__ void sts_if(bool p, uint32_t *ptr, uint32_t v) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q st.shared.u32 [%1], %2; }" ::"r"(static_cast<int>(p)),
                 "r"(static_cast<uint32_t>(__cvta_generic_to_shared(ptr))), "r"(v)
                 : "memory");
}

// K4 for the paper's configuration (k = 1, 32-slot candidate lists), dense
// memory: ATOMIC (kMode 1) / RELAXED (kMode 0).  Same semantics and RNG
// protocol as k_construct_dense; the step is laid out for the shortest
// dependent chain and the fewest warp instructions:
//   * chain: row load -> visited word (LDS) -> score -> warp_argmax_id (three
//     REDUX, winner id included) -> next row address -> next loads;
//   * a greedy step needs no ballot (argmax validity = non-empty filtered set)
//     and no select of the masked score;
//   * everything else -- pheromone update stores, the late mirror copy, the
//     visited mark, RNG commit, route, length, counters -- is issued after the
//     next row's loads, as predicated stores without branches;
//   * the visited mark of a candidate step is the store of the word the
//     winning lane already loaded for its test (no second LDS).
// kPw1 (ATOMIC, m <= kPw1Max): c_l^c from ONE shared table of m + 1 entries,
// pw1[c] = c_l^(c mod 512) * c_l^(512 (c div 512)) -- the two-table product
// formed once per CTA, so the values are the same -- one LDS and no DMUL on
// the chain.  A copy's count never exceeds m within an iteration (each ant
// bumps each copy at most once per tour; the counts are folded every iteration).
constexpr uint32_t kPw1Max = 4096;
template <int kMode, class RNG, int kRegs, bool kPw1 = false>
__global__ void __maxnreg__(kRegs) k_tour_lean(DevInstance I, DevColony C) {
    constexpr bool kAtomic = kMode == 1;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double s_pw[kAtomic && !kPw1 ? 512 + kLeanPwHi : 1];  // ATOMIC: c_l^j | c_l^(512k)
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    double *scratch = reinterpret_cast<double *>(smem) + wib * 32;
    uint32_t *vis = reinterpret_cast<uint32_t *>(smem + wpb * 32 * sizeof(double)) + static_cast<size_t>(wib) * I.words;
    double *pw1 = reinterpret_cast<double *>(
        smem + ((wpb * (32 * sizeof(double) + I.words * sizeof(uint32_t)) + 15) & ~static_cast<size_t>(15)));
    if constexpr (kAtomic && kPw1) {
#pragma unroll 4
        for (uint32_t i = threadIdx.x; i <= C.m; i += blockDim.x)
            pw1[i] = __dmul_rn(__ldg(C.pw_lo + (i & 511u)), __ldg(C.pw_hi + (i >> 9)));
        __syncthreads();
    } else if constexpr (kAtomic) {
        for (uint32_t i = threadIdx.x; i < 512 + kLeanPwHi; i += blockDim.x)
            s_pw[i] = i < 512 + C.pw_hi_n ? C.pw_lo[i] : 0.0;
        __syncthreads();
    }
    const double *pwt = kPw1 ? pw1 : s_pw;
    const uint64_t it = *C.iter;
    const uint32_t n = I.n;
    const uint32_t one = 1u;
    WarpCounters wc;

    for (uint32_t a = blockIdx.x * wpb + wib; a < C.m; a += gridDim.x * wpb) {
        for (uint32_t i = lane; i < I.words; i += 32) vis[i] = 0;
        RNG rng;
        rng_init(rng, C, it, a);
        const uint32_t start = static_cast<uint32_t>(uniform_int(rng, n));  // P1.1
        size_t ri = static_cast<size_t>(start) * 32 + lane;
        uint4 el = __ldg(C.rows + ri);
        double tl = ld_relaxed(C.tauc + ri);
        uint32_t cl = kAtomic ? ld_relaxed_u32(C.cntc + ri) : 0u;
        __syncwarp();
        if (lane == 0) vis[start >> 5] |= 1u << (start & 31);
        __syncwarp();
        uint32_t *route = C.routes + static_cast<size_t>(a) * n;
        uint32_t rbuf = start, cur = start;
        long long lenl = 0;  // this lane's share of the tour length (edges chosen from its slot)
        Lookahead<RNG> la;
        la.prepare(rng);
        uint32_t mprev = kEmpty;  // row cur owes the late copy of edge (prev, cur)

        for (uint32_t t = 1; t < n; ++t) {
            const uint32_t c = el.x & kIdMask;
            uint32_t *vw = vis + (c >> 5);
            const uint32_t word = *vw, bit = 1u << (c & 31);
            const bool unv = !(word & bit);
            const double tv = kAtomic ? trail_value_sel<kPw1>(tl, cl, C, pwt) : tl;
            const double score = __dmul_rn(tv, __hiloint2double(static_cast<int>(el.w), static_cast<int>(el.z)));
            // off-chain: this lane's copy tauc[cur][lane] gets f(its trail) if it
            // holds the chosen slot or the late mirror copy (the slot of prev)
            const bool mw = c == mprev;
            // ATOMIC reuses the index row cur was loaded with (ri = cur * 32 + lane);
            // RELAXED recomputes it (reusing it there measured 3 % slower: spills)
            const size_t mi = kAtomic ? ri : static_cast<size_t>(cur) * 32 + lane;
            const double mval = kAtomic ? 0.0 : affine(tl, C.c_l, C.c_0);
#ifdef ACS_COUNT_LOST
            const double told = tl;  // the value this lane's update read (tl is reloaded below)
#endif
            const int32_t dl = static_cast<int32_t>(el.y);
            const bool nomir = (el.x >> 24) == kNoMirror;  // this slot's node has no slot for cur
            int pos;
            uint32_t v;
            bool cand;
            const bool greedy = la.greedy(C);
            if (greedy) {
                cand = warp_argmax_id(score, unv, c, lane, pos, v);
            } else {
                const unsigned um = __ballot_sync(kFull, unv);
                cand = um != 0u;
                if (cand) {
                    rng.advance();  // commit q (P1: only when the filtered set is non-empty)
                    const double r = uniform01(rng);
                    pos = warp_roulette_pos(unv ? score : 0.0, um, r, scratch, lane);
                    v = __shfl_sync(kFull, c, pos);
                    ++wc.roulette;
                }
            }
            if (!cand) {  // every candidate visited: fallback (no draw, P1)
                Step st;
                if constexpr (kAtomic) {
                    fallback_scan(I, C, vis, cur,
                                  [&](uint32_t x, bool act) {
                                      if (!act) return 0.0;
                                      const size_t k = static_cast<size_t>(cur) * n + x;
                                      return trail_value_sel<kPw1>(ld_relaxed(C.tau + k), ld_relaxed_u32(C.cnt + k), C, pwt);
                                  },
                                  lane, st);
                } else {
                    fallback_scan(I, C, vis, cur,
                                  [&](uint32_t x, bool act) {
                                      return act ? ld_relaxed(C.tau + static_cast<size_t>(cur) * n + x) : 0.0;
                                  },
                                  lane, st);
                }
                v = st.v;
                pos = -1;
                // the non-candidate edge's dense copies: lane 0 tau[u][v], lane 1 tau[v][u]
                if (lane < 2) {
                    const size_t di = lane ? static_cast<size_t>(v) * n + cur : static_cast<size_t>(cur) * n + v;
                    if constexpr (kAtomic) {
                        if (!(lane == 1 && dense_counted_by_cand(1, -1, st.mirror, 32u))) red_add1(C.cnt + di);
                    } else {
                        st_relaxed(C.tau + di, affine(st.tau_old, C.c_l, C.c_0));
                    }
                }
                if (lane == 0) {
                    vis[v >> 5] |= 1u << (v & 31);
                    lenl += st.d;
                }
                ++wc.fallback;
                wc.fb_elems += n - t;
            }
            // this edge's length share, formed before the next row's loads: the
            // row's d must not stay live across them (ptxas would copy the
            // reloaded register at the loop end and wait there for the load)
            const int32_t dme = lane == pos ? dl : 0;
            // ---- next row: issued as soon as v is known
            ri = static_cast<size_t>(v) * 32 + lane;
            el = __ldg(C.rows + ri);
            tl = ld_relaxed(C.tauc + ri);
            if constexpr (kAtomic) cl = ld_relaxed_u32(C.cntc + ri);
            // ---- off the chain: predicated stores, no shuffles.  The lane of
            // the chosen slot writes all three copies of (cur, v) with f of the
            // trail it scored (tau[u][v], tau[v][u], tauc[u][pos]); the lane of
            // prev writes the late mirror copy of the previous edge; the fourth
            // copy, tauc[v][mirror], is next step's late copy.
            const bool me = lane == pos;
            // the pheromone update stores; ATOMIC issues them after the RNG and
            // route work, RELAXED before it (each order measured ~1 % faster
            // for its mode)
            auto update_stores = [&]() {
                if constexpr (kAtomic) {
                    red_add_if(me || mw, C.cntc + mi, one);
#if ACS_DENSE_CAND_SKIP
                    // dense counters: (cur, v) has its candidate copy; (v, cur)
                    // only when cur is not in v's row (no late mirror copy)
                    red_add_if(me && nomir, C.cnt + (static_cast<size_t>(v) * n + cur), one);
#else
                    // the two dense counters in one instruction: lane pos bumps
                    // cnt[u][v], lane pos ^ 1 bumps cnt[v][u] (no value to move)
                    const bool mate = lane == (pos ^ 1);
                    const uint32_t row = me ? cur : v;
                    red_add_if(pos >= 0 && (me || mate), C.cnt + (static_cast<size_t>(row) * n + (cur ^ v ^ row)), one);
#endif
                } else {
                    const size_t d_uv = static_cast<size_t>(cur) * n + v, d_vu = static_cast<size_t>(v) * n + cur;
#ifdef ACS_COUNT_LOST
                    // instrumented build: the candidate-copy write (the copy this lane
                    // read as tl) is an exchange; an old value other than tl means
                    // another ant's update of that trail landed in between and is lost
                    if (me || mw) {
                        ++wc.writes;
                        wc.lost += xchg_lost(C.tauc + mi, mval, told);
                    }
                    st_relaxed_if(me, C.tau + d_uv, mval);
                    st_relaxed_if(me, C.tau + d_vu, mval);
#else
                    st_relaxed_if(me || mw, C.tauc + mi, mval);
                    st_relaxed_if(me, C.tau + d_uv, mval);
                    st_relaxed_if(me, C.tau + d_vu, mval);
#endif
                }
            };
            if constexpr (!kAtomic) update_stores();
            // visited mark: the winning lane stores the word it tested (pos = -1
            // after a fallback, which marked v itself)
            sts_if(me, vw, word | bit);
            lenl += dme;
            // RNG: commit a greedy step's q draw, peek the next one
            if (greedy && cand) rng.advance();
            la.prepare(rng);
            {   // route buffered in registers, one 128 B store per 32 steps
                const uint32_t tl5 = t & 31u;
                if (static_cast<uint32_t>(lane) == tl5) rbuf = v;
                if (tl5 == 31u) route[(t & ~31u) + lane] = rbuf;
            }
            if constexpr (kAtomic) update_stores();
            mprev = cur;
            cur = v;
            __syncwarp();
        }
        route_flush(route, rbuf, n - 1, lane);
        wc.updates += n - 1;
        long long len = lenl;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) len += static_cast<long long>(shfl_xor_u64(static_cast<uint64_t>(len), o));
        // last step's late mirror copy (el/tl hold row `cur`)
        if ((el.x & kIdMask) == mprev) {
            if constexpr (kAtomic) red_add1(C.cntc + static_cast<size_t>(cur) * 32 + lane);
            else st_relaxed(C.tauc + static_cast<size_t>(cur) * 32 + lane, affine(tl, C.c_l, C.c_0));
        }
        __syncwarp();
        // closing edge (cur -> start) is edge n of the ant (D9, k = 1: due)
        int pos;
        uint32_t mirror;
        int32_t dclose;
        bool have_d;
        closing_slots(C, cur, start, lane, pos, mirror, dclose, have_d);
        if (!have_d)
            dclose = tsplib_distance(I.type, __ldg(I.xs + cur), __ldg(I.ys + cur), __ldg(I.xs + start),
                                     __ldg(I.ys + start));
        ++wc.updates;
        bool dense;
        size_t k;
        if (copy_index(n, cur, start, pos, mirror, lane, dense, k)) {
            if constexpr (kAtomic) {
                if (!(dense && dense_counted_by_cand(lane, pos, mirror, 32u)))
                    red_add1((dense ? C.cnt : C.cntc) + k);
            } else {
                const double told = ld_relaxed(C.tau + static_cast<size_t>(cur) * n + start);
                st_relaxed((dense ? C.tau : C.tauc) + k, affine(told, C.c_l, C.c_0));
            }
        }
        if (lane == 0) C.lens[a] = len + dclose;
        wc.flush(C.counters, lane, n - 1);
        __syncwarp();
    }
}

// ATOMIC variant: fold the per-copy counters into the bases (tau = f^c(base),
// c = 0) before the global update.  Grid-stride over the dense and candidate
// arrays; 4 counters per thread step, skipping untouched words.
__global__ void k_fold_counts(DevColony C, size_t dense_count, size_t cand_count) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t t0 = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    // dense counters as 16-byte vectors (4 per load): the sweep is a pure
    // HBM/L2 read of n^2 x 4 B; tau is touched only where a count is pending
    const size_t q4 = dense_count / 4;
    const uint4 *cnt4 = reinterpret_cast<const uint4 *>(C.cnt);
    for (size_t q = t0; q < q4; q += stride) {
        const uint4 c = cnt4[q];
        if ((c.x | c.y | c.z | c.w) == 0u) continue;
        const uint32_t cs[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (cs[j]) {
                const size_t i = 4 * q + j;
                C.tau[i] = trail_value(C.tau[i], cs[j], C, C.pw_lo, C.pw_hi);
                C.cnt[i] = 0;
            }
        }
    }
    for (size_t i = 4 * q4 + t0; i < dense_count; i += stride) {
        const uint32_t c = C.cnt[i];
        if (c) {
            C.tau[i] = trail_value(C.tau[i], c, C, C.pw_lo, C.pw_hi);
            C.cnt[i] = 0;
        }
    }
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cand_count; i += stride) {
        const uint32_t c = C.cntc[i];
        if (c) {
            C.tauc[i] = trail_value(C.tauc[i], c, C, C.pw_lo, C.pw_hi);
            C.cntc[i] = 0;
#if ACS_DENSE_CAND_SKIP
            // the dense copy of the same entry was not counted: same count
            const uint32_t b = C.rows[i].x & kIdMask;
            const size_t di = (i / 32) * (cand_count / 32) + b;
            C.tau[di] = trail_value(C.tau[di], c, C, C.pw_lo, C.pw_hi);
#endif
        }
    }
}

// ============================================================ selective whole tour

// Register copy of one record.  The S ids are in every lane (broadcast loads,
// so the first-match search is local compares); the S values are spread one
// per lane (lane j < S holds slot j) and fetched with one shuffle -- this keeps
// the record at S + 3 registers per lane instead of 3S.
template <int S>
struct SpmRec {
    uint32_t id[S];
    uint32_t idl;   // slot `lane`'s id (lanes < S, kEmpty above): warp-uniform finds are one ballot
    double val;     // slot `lane` (lanes < S)
    uint32_t tail;

    __device__ __forceinline__ void load(const DevColony &C, uint32_t u, int lane) {
        const uint32_t *ids = C.spm.ids(u);
        if constexpr (S >= 4) {
#pragma unroll
            for (int j = 0; j < S; j += 4) {
                const uint4 q = __ldcg(reinterpret_cast<const uint4 *>(ids + j));
                id[j] = q.x; id[j + 1] = q.y; id[j + 2] = q.z; id[j + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < S; ++j) id[j] = __ldcg(ids + j);
        }
        val = lane < S ? __ldcg(C.spm.vals(u) + lane) : 0.0;
        idl = lane < S ? __ldcg(ids + lane) : kEmpty;
        tail = __ldcg(C.spm.tail(u));
    }
    // first slot holding the warp-uniform v, or -1
    __device__ __forceinline__ int find_uniform(uint32_t v) const {
        const unsigned m = __ballot_sync(kFull, idl == v);
        return m ? __ffs(m) - 1 : -1;
    }
    // record u gets neighbour v (warp-uniform) with this record's registers kept
    // current for later lookups in the same step; returns hit
    __device__ __forceinline__ bool update_keep(const DevColony &C, uint32_t u, uint32_t v, double c_mul,
                                                double c_add, int lane) {
        const int hit = find_uniform(v);
        if (hit >= 0) {
            const double y = affine(__shfl_sync(kFull, val, hit), c_mul, c_add);
            if (lane == hit) val = y;
            if (lane == 0) st_relaxed(C.spm.vals(u) + hit, y);
            return true;
        }
        const double y = affine(C.tau_min, c_mul, c_add);
        const uint32_t t = (tail + 1) % S;
#pragma unroll
        for (int j = 0; j < S; ++j)
            if (j == static_cast<int>(t)) id[j] = v;
        if (lane == static_cast<int>(t)) { idl = v; val = y; }
        tail = t;
        if (lane == 0) {
            st_relaxed_u32(C.spm.ids(u) + t, v);
            st_relaxed(C.spm.vals(u) + t, y);
            st_relaxed_u32(C.spm.tail(u), t);
        }
        return false;
    }
    // the same, write-only: the registers are dead afterwards (next record loads)
    __device__ __forceinline__ bool update_last(const DevColony &C, uint32_t u, uint32_t v, double tau_old,
                                                double c_mul, double c_add, int lane) const {
        const int hit = find_uniform(v);
        if (hit >= 0) {
            if (lane == 0) st_relaxed(C.spm.vals(u) + hit, affine(tau_old, c_mul, c_add));
            return true;
        }
        const uint32_t t = (tail + 1) % S;
        if (lane == 0) {
            st_relaxed_u32(C.spm.ids(u) + t, v);
            st_relaxed(C.spm.vals(u) + t, affine(C.tau_min, c_mul, c_add));
            st_relaxed_u32(C.spm.tail(u), t);
        }
        return false;
    }
    __device__ __forceinline__ int find(uint32_t v) const {
        int hit = -1;
#pragma unroll
        for (int j = S - 1; j >= 0; --j)
            if (id[j] == v) hit = j;  // first (lowest) matching slot
        return hit;
    }
    // tau of (u, v) for this lane's v; all lanes must call (warp shuffle)
    __device__ __forceinline__ double lookup(uint32_t v, double tau_min) const {
        const int hit = find(v);
        const double x = __shfl_sync(kFull, val, hit < 0 ? 0 : hit);
        return hit < 0 ? tau_min : x;
    }
    // update record u with neighbour v (warp-uniform); lane 0 writes through. Returns hit.
    __device__ __forceinline__ bool update(const DevColony &C, uint32_t u, uint32_t v, double c_mul,
                                           double c_add, int lane) {
        const int hit = find(v);
        if (hit >= 0) {
            const double y = affine(__shfl_sync(kFull, val, hit), c_mul, c_add);
            if (lane == hit) val = y;
            if (lane == 0) st_relaxed(C.spm.vals(u) + hit, y);
            return true;
        }
        const double y = affine(C.tau_min, c_mul, c_add);
        const uint32_t t = (tail + 1) % S;
#pragma unroll
        for (int j = 0; j < S; ++j)
            if (j == static_cast<int>(t)) id[j] = v;
        if (lane == static_cast<int>(t)) val = y;
        tail = t;
        if (lane == 0) {
            st_relaxed_u32(C.spm.ids(u) + t, v);
            st_relaxed(C.spm.vals(u) + t, y);
            st_relaxed_u32(C.spm.tail(u), t);
        }
        return false;
    }
};

// The general selective kernel (any k, s, list length; one warp for SPM SEQ);
// the paper's configuration (k = 1, 32-slot lists, s = 8) runs k_spm_lean.
template <int S, class RNG>
__global__ void __maxnreg__(kMaxRegs) k_construct_spm(DevInstance I, DevColony C) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    double *scratch = reinterpret_cast<double *>(smem) + wib * 32;
    uint32_t *vis = reinterpret_cast<uint32_t *>(smem + wpb * 32 * sizeof(double)) +
                    static_cast<size_t>(wib) * I.words;
    const uint64_t it = *C.iter;
    const uint32_t n = I.n;
    WarpCounters wc;

    for (uint32_t a = blockIdx.x * wpb + wib; a < C.m; a += gridDim.x * wpb) {
        for (uint32_t i = lane; i < I.words; i += 32) vis[i] = 0;
        RNG rng;
        rng_init(rng, C, it, a);
        const uint32_t start = static_cast<uint32_t>(uniform_int(rng, n));
        uint4 el = __ldg(C.rows + static_cast<size_t>(start) * 32 + lane);
        SpmRec<S> rec;
        rec.load(C, start, lane);
        __syncwarp();
        if (lane == 0) vis[start >> 5] |= 1u << (start & 31);
        __syncwarp();
        uint32_t *route = C.routes + static_cast<size_t>(a) * n;
        uint32_t rbuf = start, cur = start, prev = 0, kc = 0;
        bool pending = false;  // record `cur` still owes the update with `prev` (D4)
        long long len = 0;
        Lookahead<RNG> la;
        la.prepare(rng);

        for (uint32_t t = 1; t < n; ++t) {
            if (pending) {
                if (rec.update_keep(C, cur, prev, C.c_l, C.c_0, lane)) ++wc.hits; else ++wc.misses;
            }
            const double tau_lane = rec.lookup(el.x & kIdMask, C.tau_min);
            Step st;
            select_step<false>(I, C, vis, cur, el, tau_lane, rng, la, scratch, lane,
                        [&](uint32_t v, bool act) { return rec.lookup(act ? v : kEmpty, C.tau_min); }, st);
            wc.count(st.kind, n - t);
            el = __ldg(C.rows + static_cast<size_t>(st.v) * 32 + lane);  // next row first
            pending = ++kc == C.k;
            if (pending) {
                kc = 0;
                ++wc.updates;
                // tau_old is what the selection read for (cur, v): the record's
                // value on a hit
                if (rec.update_last(C, cur, st.v, st.tau_old, C.c_l, C.c_0, lane)) ++wc.hits; else ++wc.misses;
                prev = cur;
            }
            rec.load(C, st.v, lane);  // record of the next node
            if (st.kind == 0) rng.advance();
            la.prepare(rng);
            vis[st.v >> 5] |= 1u << (st.v & 31);
            len += st.d;
            route_put(route, rbuf, t, st.v, lane);
            cur = st.v;
            __syncwarp();
        }
        route_flush(route, rbuf, n - 1, lane);
        if (pending) {
            if (rec.update(C, cur, prev, C.c_l, C.c_0, lane)) ++wc.hits; else ++wc.misses;
        }
        const int32_t dclose = tsplib_distance(I.type, __ldg(I.xs + cur), __ldg(I.ys + cur),
                                               __ldg(I.xs + start), __ldg(I.ys + start));
        if (++kc == C.k) {  // closing edge: record last, then record start
            ++wc.updates;
            if (rec.update(C, cur, start, C.c_l, C.c_0, lane)) ++wc.hits; else ++wc.misses;
            __syncwarp();
            SpmRec<S> r2;
            r2.load(C, start, lane);
            if (r2.update(C, start, cur, C.c_l, C.c_0, lane)) ++wc.hits; else ++wc.misses;
        }
        if (lane == 0) C.lens[a] = len + dclose;
        wc.flush(C.counters, lane, n - 1);
        __syncwarp();
    }
}

// Lean SPM records (s = 8): one 128 B line per record {vals[8] f64 | ids[8]
// u32 | tail u32}, addressed as base + (u << 7) with constant field offsets.
constexpr uint32_t kRec8Ids = 64, kRec8Tail = 96;
__device__ __forceinline__ unsigned char *rec8(const DevColony &C, uint32_t u) {
    return C.spm.base + (static_cast<size_t>(u) << 7);
}
__device__ __forceinline__ void st_relaxed_u32_if(bool p, uint32_t *ptr, uint32_t v) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q st.relaxed.gpu.global.b32 [%1], %2; }" ::"r"(
                     static_cast<int>(p)),
                 "l"(ptr), "r"(v)
                 : "memory");
}

// One record update (D5) on the lane-distributed copy of the
// record (lane j < 8: slot j's id and value, tail in every lane), written
// through by lane 0 with predicated stores: hit -> the slot's value, miss ->
// f(tau_min) into slot (tail + 1) % 8 with its id, and the tail.  kKeep: the
// copy stays current for a following update; otherwise a hit's new value is
// f(tau_old), the value the selection read.  Returns hit.
// The same with the hit already known (hit: slot hslot holds nb): the lean
// step knows both from its lookup, so no ballot is spent on them.
template <bool kKeep>
__device__ __forceinline__ bool spm8_update_at(const DevColony &C, unsigned char *rb, uint32_t nb, double tau_old,
                                               bool hit, uint32_t hslot, uint32_t &idl, double &val, uint32_t &tail,
                                               int lane, uint32_t *stale = nullptr);

template <bool kKeep>
__device__ __forceinline__ bool spm8_update(const DevColony &C, unsigned char *rb, uint32_t nb, double tau_old,
                                            uint32_t &idl, double &val, uint32_t &tail, int lane,
                                            uint32_t *stale = nullptr) {
    const unsigned m = __ballot_sync(kFull, idl == nb);
    return spm8_update_at<kKeep>(C, rb, nb, tau_old, m != 0u, m ? static_cast<uint32_t>(__ffs(m) - 1) : 0u, idl, val,
                                 tail, lane, stale);
}

template <bool kKeep>
__device__ __forceinline__ bool spm8_update_at(const DevColony &C, unsigned char *rb, uint32_t nb, double tau_old,
                                               bool hit, uint32_t hslot, uint32_t &idl, double &val, uint32_t &tail,
                                               int lane, uint32_t *stale) {
    const uint32_t t = (tail + 1) & 7u;
    const uint32_t slot = hit ? hslot : t;
#ifdef ACS_COUNT_LOST
    // instrumented build: the update works from a copy of the record read at
    // the start of the step; stale if another ant changed its tail or the
    // updated slot's id since
    {
        const uint32_t cid = __shfl_sync(kFull, idl, static_cast<int>(slot));
        if (stale && lane == 0) {
            const uint32_t mt = ld_relaxed_u32(reinterpret_cast<const uint32_t *>(rb + kRec8Tail));
            const uint32_t mid = ld_relaxed_u32(reinterpret_cast<const uint32_t *>(rb + kRec8Ids) + slot);
            *stale += (mt != tail || mid != cid) ? 1u : 0u;
        }
    }
#endif
    const double hv = kKeep ? __shfl_sync(kFull, val, static_cast<int>(slot)) : tau_old;
    const double y = affine(hit ? hv : C.tau_min, C.c_l, C.c_0);
    const bool l0 = lane == 0;
    st_relaxed_if(l0, reinterpret_cast<double *>(rb) + slot, y);
    st_relaxed_u32_if(l0 && !hit, reinterpret_cast<uint32_t *>(rb + kRec8Ids) + slot, nb);
    st_relaxed_u32_if(l0 && !hit, reinterpret_cast<uint32_t *>(rb + kRec8Tail), t);
    if (kKeep) {
        if (static_cast<uint32_t>(lane) == slot) {
            val = y;
            if (!hit) idl = nb;
        }
        if (!hit) tail = t;
    }
    return hit;
}

// The lean kernel's register copy of record u: the ids in every lane
// (broadcast loads; a lane's lookup is eight compares), slot `lane`'s id and
// value in lanes 0-7, the tail.
struct Rec8 {
    uint32_t id[8];
    uint32_t idl, tail;
    double val;
    __device__ __forceinline__ void load(const unsigned char *rb, int lane) {
        const uint4 q0 = __ldcg(reinterpret_cast<const uint4 *>(rb + kRec8Ids));
        const uint4 q1 = __ldcg(reinterpret_cast<const uint4 *>(rb + kRec8Ids + 16));
        id[0] = q0.x; id[1] = q0.y; id[2] = q0.z; id[3] = q0.w;
        id[4] = q1.x; id[5] = q1.y; id[6] = q1.z; id[7] = q1.w;
        val = lane < 8 ? __ldcg(reinterpret_cast<const double *>(rb) + lane) : 0.0;
        idl = lane < 8 ? __ldcg(reinterpret_cast<const uint32_t *>(rb + kRec8Ids) + lane) : kEmpty;
        tail = __ldcg(reinterpret_cast<const uint32_t *>(rb + kRec8Tail));
    }
    // first slot holding v, or -1: a depth-3 select tree over the eight
    // (parallel) compares instead of a chain of eight selects
    __device__ __forceinline__ int find(uint32_t v) const {
        const int a = id[0] == v ? 0 : (id[1] == v ? 1 : -1);
        const int b = id[2] == v ? 2 : (id[3] == v ? 3 : -1);
        const int c = id[4] == v ? 4 : (id[5] == v ? 5 : -1);
        const int d = id[6] == v ? 6 : (id[7] == v ? 7 : -1);
        const int ab = a >= 0 ? a : b, cd = c >= 0 ? c : d;
        return ab >= 0 ? ab : cd;
    }
};

// SPM for the paper's configuration (k = 1, 32-slot lists, s = 8 slots): the
// lean step of k_tour_lean over the selective memory.  Record cur owes two
// ordered updates in a step (D4): the second half of the previous edge
// (neighbour prev), then the first half of this edge (neighbour v).  Both are
// applied after the next row's loads.  The selection reads the record as it
// will be after the first one: only an unvisited candidate's value matters,
// prev is visited, so the only effect is a miss evicting slot (tail + 1) % S.
#ifndef ACS_SPM_REGS
#define ACS_SPM_REGS 96
#endif
// 96 registers: 5 warps per SM sub-partition (16K registers each), so m = n = 2392 is one wave
template <class RNG>
__global__ void __maxnreg__(ACS_SPM_REGS) k_spm_lean(DevInstance I, DevColony C) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    double *scratch = reinterpret_cast<double *>(smem) + wib * 32;
    uint32_t *vis = reinterpret_cast<uint32_t *>(smem + wpb * 32 * sizeof(double)) + static_cast<size_t>(wib) * I.words;
    const uint64_t it = *C.iter;
    const uint32_t n = I.n;
    WarpCounters wc;

    for (uint32_t a = blockIdx.x * wpb + wib; a < C.m; a += gridDim.x * wpb) {
        for (uint32_t i = lane; i < I.words; i += 32) vis[i] = 0;
        RNG rng;
        rng_init(rng, C, it, a);
        const uint32_t start = static_cast<uint32_t>(uniform_int(rng, n));
        uint4 el = __ldg(C.rows + static_cast<size_t>(start) * 32 + lane);
        Rec8 rec;
        rec.load(rec8(C, start), lane);
        __syncwarp();
        if (lane == 0) vis[start >> 5] |= 1u << (start & 31);
        __syncwarp();
        uint32_t *route = C.routes + static_cast<size_t>(a) * n;
        uint32_t rbuf = start, cur = start, prev = kEmpty;  // kEmpty: no pending update yet
        long long lenl = 0;
        Lookahead<RNG> la;
        la.prepare(rng);

        for (uint32_t t = 1; t < n; ++t) {
            const uint32_t c = el.x & kIdMask;
            uint32_t *vw = vis + (c >> 5);
            const uint32_t word = *vw, bit = 1u << (c & 31);
            const bool unv = !(word & bit);
            // pending update of record cur with prev: a miss evicts slot (tail+1) % S
            const bool pend = prev != kEmpty;
            const unsigned pm = __ballot_sync(kFull, pend && rec.idl == prev);  // prev's slot, if any
            const bool pmiss = pend && pm == 0u;
            const int evict = pmiss ? static_cast<int>((rec.tail + 1) & 7u) : -1;
            int hit = rec.find(c);
            if (hit == evict) hit = -1;
            const double hv = __shfl_sync(kFull, rec.val, hit < 0 ? 0 : hit);
            const double tv = hit < 0 ? C.tau_min : hv;
            const double score = __dmul_rn(tv, __hiloint2double(static_cast<int>(el.w), static_cast<int>(el.z)));
            const int32_t dl = static_cast<int32_t>(el.y);
            int pos;
            uint32_t v;
            bool cand;
            const bool greedy = la.greedy(C);
            if (greedy) {
                cand = warp_argmax_id(score, unv, c, lane, pos, v);
            } else {
                const unsigned um = __ballot_sync(kFull, unv);
                cand = um != 0u;
                if (cand) {
                    rng.advance();  // commit q (P1)
                    const double r = uniform01(rng);
                    pos = warp_roulette_pos(unv ? score : 0.0, um, r, scratch, lane);
                    v = __shfl_sync(kFull, c, pos);
                    ++wc.roulette;
                }
            }
            double tau_old = 0.0;
            int vslot = -1;  // v's slot in record cur after the pending update (candidate steps)
            if (!cand) {  // fallback: the record after its pending update, then the scan
                if (pend) {
                    wc.misses += !spm8_update<true>(C, rec8(C, cur), prev, 0.0, rec.idl, rec.val, rec.tail, lane);
                    prev = kEmpty;
                }
                Step st;
                fallback_scan(I, C, vis, cur,
                              [&](uint32_t x, bool act) {  // all lanes call: the value comes by shuffle
                                  const int j = act ? rec.find(x) : -1;
                                  const double y = __shfl_sync(kFull, rec.val, j < 0 ? 0 : j);
                                  return j < 0 ? C.tau_min : y;
                              },
                              lane, st);
                v = st.v;
                pos = -1;
                tau_old = st.tau_old;
                if (lane == 0) {
                    vis[v >> 5] |= 1u << (v & 31);
                    lenl += st.d;
                }
                ++wc.fallback;
                wc.fb_elems += n - t;
            } else {
#ifdef ACS_COUNT_LOST
                tau_old = __shfl_sync(kFull, tv, pos);
#endif
                vslot = __shfl_sync(kFull, hit, pos);
            }
            // record cur's lane-distributed slots: all its two updates need
            uint32_t ridl = rec.idl, rtail = rec.tail;
            double rval = rec.val;
            const int32_t dme = lane == pos ? dl : 0;  // before the loads (as k_tour_lean)
            // ---- next row and record: issued as soon as v is known
            el = __ldg(C.rows + static_cast<size_t>(v) * 32 + lane);
            rec.load(rec8(C, v), lane);
            // ---- off the chain: record cur's two ordered updates
            // (hits are derived at the tour end: 2 record operations per update)
            unsigned char *rb = rec8(C, cur);
#ifdef ACS_COUNT_LOST
            uint32_t *stale = &wc.lost;  // counted by lane 0, as the updates
            if (lane == 0) wc.writes += (prev != kEmpty) ? 2 : 1;
#else
            uint32_t *stale = nullptr;
#endif
            // the step's other off-chain work first, then the record updates
            // (measured 1 % faster than the reverse order)
            sts_if(lane == pos, vw, word | bit);
            lenl += dme;
            if (greedy && cand) rng.advance();
            la.prepare(rng);
            route_put(route, rbuf, t, v, lane);
            // the lookup already located both neighbours: prev by the step's
            // first ballot, v (candidate step) by the winning lane's find
#ifndef ACS_COUNT_LOST
            if (cand) {
                // both updates at once, each by the lane owning its slot: the
                // owner holds the slot's value, so no shuffle; a slot written
                // twice (v's miss evicting prev's slot) is written by one lane
                // in program order, prev's update first (D4)
                const bool phit = pm != 0u, vhit = vslot >= 0;
                const uint32_t e1 = (rtail + 1) & 7u;
                const uint32_t s1 = !pend ? 32u : (phit ? static_cast<uint32_t>(__ffs(pm) - 1) : e1);
                const uint32_t tail1 = (pend && !phit) ? e1 : rtail;
                const uint32_t e2 = (tail1 + 1) & 7u;
                const uint32_t s2 = vhit ? static_cast<uint32_t>(vslot) : e2;
                const bool o1 = static_cast<uint32_t>(lane) == s1, o2 = static_cast<uint32_t>(lane) == s2;
                const double y1 = affine(phit ? rval : C.tau_min, C.c_l, C.c_0);
                const double y2 = affine(vhit ? rval : C.tau_min, C.c_l, C.c_0);
                double *vp = reinterpret_cast<double *>(rb) + lane;
                uint32_t *ip = reinterpret_cast<uint32_t *>(rb + kRec8Ids) + lane;
                st_relaxed_if(o1, vp, y1);
                st_relaxed_u32_if(o1 && !phit, ip, prev);
                st_relaxed_if(o2, vp, y2);
                st_relaxed_u32_if(o2 && !vhit, ip, v);
                st_relaxed_u32_if(lane == 0 && ((pend && !phit) || !vhit), reinterpret_cast<uint32_t *>(rb + kRec8Tail),
                                  vhit ? tail1 : e2);
                wc.misses += static_cast<uint32_t>(pend && !phit) + static_cast<uint32_t>(!vhit);
            } else
                wc.misses += !spm8_update<false>(C, rb, v, tau_old, ridl, rval, rtail, lane, stale);
#else
            if (prev != kEmpty)
                wc.misses += !spm8_update_at<true>(C, rb, prev, 0.0, pm != 0u, pm ? static_cast<uint32_t>(__ffs(pm) - 1) : 0u,
                                                   ridl, rval, rtail, lane, stale);
            if (cand) wc.misses += !spm8_update_at<false>(C, rb, v, tau_old, vslot >= 0, static_cast<uint32_t>(vslot), ridl,
                                                          rval, rtail, lane, stale);
            else wc.misses += !spm8_update<false>(C, rb, v, tau_old, ridl, rval, rtail, lane, stale);
#endif
            prev = cur;
            cur = v;
            __syncwarp();
        }
        route_flush(route, rbuf, n - 1, lane);
        wc.updates += n - 1;
        long long len = lenl;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) len += static_cast<long long>(shfl_xor_u64(static_cast<uint64_t>(len), o));
        // record cur's pending update, then the closing edge: record last, then record start
        unsigned char *rb = rec8(C, cur);
        if (prev != kEmpty) wc.misses += !spm8_update<true>(C, rb, prev, 0.0, rec.idl, rec.val, rec.tail, lane);
        const int32_t dclose = tsplib_distance(I.type, __ldg(I.xs + cur), __ldg(I.ys + cur), __ldg(I.xs + start),
                                               __ldg(I.ys + start));
        ++wc.updates;
        wc.misses += !spm8_update<true>(C, rb, start, 0.0, rec.idl, rec.val, rec.tail, lane);
        __syncwarp();
        Rec8 r2;
        r2.load(rec8(C, start), lane);
        wc.misses += !spm8_update<true>(C, rec8(C, start), cur, 0.0, r2.idl, r2.val, r2.tail, lane);
        wc.hits = 2 * n - wc.misses;  // n local updates (k = 1), two record operations each
        if (lane == 0) C.lens[a] = len + dclose;
        wc.flush(C.counters, lane, n - 1);
        __syncwarp();
    }
}

// ============================================================ deferred (SYNC)

// Grid-wide barrier of the cooperative (all-CTAs-resident) deferred kernel.
// cooperative_groups' grid sync measured 1.3 us per barrier on B200 at
// 148 x 640 threads, against 2.6 us for a two-level atomic-counter barrier
// and 1.9 us for a flat acquire/release one (tools/micro/grid_barrier.cu).
__device__ __forceinline__ void grid_sync() { cg::this_grid().sync(); }

template <class RNG>
struct DefAnt {             // per-ant state of the deferred variant, in shared memory
    RNG rng;
    long long len;
    uint32_t cur, start, v, slots;  // slots = pos | mirror << 8 of this step's edge
    int32_t d;                      // distance of this step's edge
    int kind;                       // 0 greedy, 1 roulette, 2 fallback, 3 full scan requested
};

// One warp's share of a cooperative full scan: (score, node, trail) of its
// word range, combined by the requesting warp (argmax, ties -> lowest id).
struct ScanPart {
    double s, t;
    uint32_t v;
};

// Shared-memory layout of the deferred kernel (wpb warps, A ants per warp).
struct DefSmem {
    size_t ants_off, vis_off, part_off, req_off, bytes;
    __host__ __device__ DefSmem(uint32_t wpb, uint32_t A, uint32_t words) {
        ants_off = static_cast<size_t>(wpb) * 32 * sizeof(double);  // roulette scratch
        vis_off = ants_off + static_cast<size_t>(wpb) * A * 64;      // DefAnt <= 64 B
        part_off = vis_off + static_cast<size_t>(wpb) * A * words * sizeof(uint32_t);
        part_off = (part_off + 15) & ~static_cast<size_t>(15);
        req_off = part_off + static_cast<size_t>(wpb) * A * wpb * sizeof(ScanPart);
        bytes = req_off + (static_cast<size_t>(wpb) * A + 1) * sizeof(uint32_t);
    }
};

// Fold the pending count of one copy into its base by applying f c times in
// sequence -- exactly what SYNC's ordered local updates do (P7) -- after an
// exchange that hands the whole count to exactly one of the ants that bumped it.
__device__ __forceinline__ void fold_copy(const DevColony &C, uint32_t n, uint32_t u, uint32_t v,
                                          uint32_t slots, int lane) {
    bool dense;
    size_t k;
    const int pos = (slots & 0xFFu) == 0xFFu ? -1 : static_cast<int>(slots & 0xFFu);
    if (!copy_index(n, u, v, pos, (slots >> 8) & 0xFFu, lane, dense, k)) return;
    uint32_t *cp = (dense ? C.cnt : C.cntc) + k;
    double *bp = (dense ? C.tau : C.tauc) + k;
    // the base is loaded alongside the exchange: only the ant that receives
    // the count writes it, so the value read here is current for that ant
    double x = ld_relaxed(bp);
    const uint32_t c = atomicExch(cp, 0u);
    if (c) {
        for (uint32_t i = 0; i < c; ++i) x = affine(x, C.c_l, C.c_0);
        st_relaxed(bp, x);
    }
}

__device__ __forceinline__ void bump_copy(const DevColony &C, uint32_t n, uint32_t u, uint32_t v,
                                          uint32_t slots, int lane) {
    bool dense;
    size_t k;
    const int pos = (slots & 0xFFu) == 0xFFu ? -1 : static_cast<int>(slots & 0xFFu);
    if (copy_index(n, u, v, pos, (slots >> 8) & 0xFFu, lane, dense, k))
        red_add1((dense ? C.cnt : C.cntc) + k);
}

// SPEC SYNC (deferred / ordered local updates) as ONE persistent cooperative
// launch per iteration.  Per step: every ant selects against the step-start
// pheromone and bumps the counters of its edge's copies (bases untouched);
// grid barrier; the count of every touched copy is exchanged to one ant that
// applies f that many times; grid barrier.  The affine updates commute, so the
// result is bit-identical to the oracle's ant-ordered application.  Closing
// edges are a separate pass after step n-1 (PAPER Alg.1 l.13-14).
//
// The lockstep makes a step as slow as its slowest ant, and the slowest ant is
// one whose fallback the pruned pass could not decide: a full scan of n nodes.
// Those scans are not run by the one warp: an ant that needs one posts a
// request, and ALL warps of the CTA (idle until the grid barrier otherwise)
// scan a slice of its bitmask words each; the requester combines the slices.
template <class RNG>
__global__ void __maxnreg__(kMaxRegs) k_deferred(DevInstance I, DevColony C, DevDeferred D) {
    static_assert(sizeof(DefAnt<RNG>) <= 64, "DefSmem reserves 64 B per ant");
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const uint32_t A = D.ants_per_warp;
    const uint32_t W = gridDim.x * wpb;
    // warp-major across CTAs: ant a runs in CTA a % grid, so a colony smaller
    // than the resident warps spreads evenly over every SM
    const uint32_t gw = wib * gridDim.x + blockIdx.x;
    const uint32_t n = I.n;
    const DefSmem L(wpb, A, I.words);
    double *scratch = reinterpret_cast<double *>(smem) + wib * 32;
    DefAnt<RNG> *ants_cta = reinterpret_cast<DefAnt<RNG> *>(smem + L.ants_off);
    DefAnt<RNG> *ants = ants_cta + wib * A;
    uint32_t *vis_cta = reinterpret_cast<uint32_t *>(smem + L.vis_off);
    uint32_t *vis_base = vis_cta + static_cast<size_t>(wib) * A * I.words;
    ScanPart *parts = reinterpret_cast<ScanPart *>(smem + L.part_off);  // [request][warp]
    uint32_t *nreq = reinterpret_cast<uint32_t *>(smem + L.req_off);
    uint32_t *reqs = nreq + 1;                                            // (warp << 16) | ant slot
    // slice of the bitmask words per warp in a cooperative scan (multiple of 4)
    const uint32_t slice = ((I.words + wpb - 1) / wpb + 3) & ~3u;
    const uint64_t it = *C.iter;
    WarpCounters wc;
    uint32_t my_ants = 0;
    if (threadIdx.x == 0) *nreq = 0;

    for (uint32_t j = 0; j < A; ++j) {
        const uint32_t a = gw + j * W;
        if (a >= C.m) break;
        ++my_ants;
        uint32_t *vis = vis_base + j * I.words;
        for (uint32_t i = lane; i < I.words; i += 32) vis[i] = 0;
        RNG rng;
        rng_init(rng, C, it, a);
        const uint32_t start = static_cast<uint32_t>(uniform_int(rng, n));
        __syncwarp();
        if (lane == 0) {
            vis[start >> 5] |= 1u << (start & 31);
            ants[j].rng = rng;
            ants[j].len = 0;
            ants[j].cur = start;
            ants[j].start = start;
            C.routes[static_cast<size_t>(a) * n] = start;
        }
        __syncwarp();
    }
    grid_sync();

    for (uint32_t t = 1; t < n; ++t) {
        const bool due = (t % C.k) == 0;
        // (1) selection against the step-start pheromone; undecided fallbacks post a request
        for (uint32_t j = 0; j < my_ants; ++j) {
            uint32_t *vis = vis_base + j * I.words;
            DefAnt<RNG> &s = ants[j];
            const uint32_t cur = s.cur;
            RNG rng = s.rng;
            const size_t ri = static_cast<size_t>(cur) * 32 + lane;
            const uint4 el = __ldg(C.rows + ri);
            const double tau_lane = ld_relaxed(C.tauc + ri);
            Lookahead<RNG> la;
            la.prepare(rng);
            Step st;
            select_step<true>(I, C, vis, cur, el, tau_lane, rng, la, scratch, lane,
                              [&](uint32_t v, bool act) {
                                  return act ? ld_relaxed(C.tau + static_cast<size_t>(cur) * n + v) : 0.0;
                              },
                              st);
            if (st.kind == 0) rng.advance();
            __syncwarp();
            if (lane == 0) {
                s.rng = rng;
                s.kind = st.kind;
                if (st.kind == 3) {
                    reqs[atomicAdd(nreq, 1u)] = (static_cast<uint32_t>(wib) << 16) | j;
                } else {
                    s.v = st.v;
                    s.d = st.d;
                    s.slots = (static_cast<uint32_t>(st.pos) & 0xFFu) | (st.mirror << 8);
                }
            }
            __syncwarp();
        }
        // (2) the CTA's full scans, every warp one slice of each
        __syncthreads();
        const uint32_t nr = *nreq;
        if (nr) {  // CTA-uniform
            for (uint32_t r = 0; r < nr; ++r) {
                const uint32_t q = reqs[r];
                const uint32_t ow = q >> 16, oj = q & 0xFFFFu;
                const uint32_t *vis = vis_cta + (static_cast<size_t>(ow) * A + oj) * I.words;
                const uint32_t cur = ants_cta[ow * A + oj].cur;
                const uint32_t wb = wib * slice, we = min(wb + slice, I.words);
                ScanBest b;
                if (wb < we)
                    full_scan_range(I, C, vis, cur,
                                    [&](uint32_t v, bool act) {
                                        return act ? ld_relaxed(C.tau + static_cast<size_t>(cur) * n + v) : 0.0;
                                    },
                                    lane, wb, we, b);
                double sc = b.bs;
                uint32_t node = b.have ? b.bv : 0xffffffffu;
                warp_argmax_node(sc, node, b.have);
                const unsigned owner = __ballot_sync(kFull, b.have && b.bv == node);
                const double tv = __shfl_sync(kFull, b.bt, owner ? __ffs(owner) - 1 : 0);
                if (lane == 0) parts[r * wpb + wib] = ScanPart{sc, tv, node};
            }
            __syncthreads();
            for (uint32_t r = 0; r < nr; ++r) {
                const uint32_t q = reqs[r];
                if ((q >> 16) != static_cast<uint32_t>(wib)) continue;  // warp-uniform
                DefAnt<RNG> &s = ants[q & 0xFFFFu];
                // combine the slices: argmax, ties -> lowest id (slices hold disjoint ids)
                const bool ok = lane < wpb && parts[r * wpb + lane].v != 0xffffffffu;
                const ScanPart pp = ok ? parts[r * wpb + lane] : ScanPart{0.0, 0.0, 0xffffffffu};
                double sc = pp.s;
                uint32_t node = pp.v;
                warp_argmax_node(sc, node, ok);
                const unsigned owner = __ballot_sync(kFull, ok && pp.v == node);
                Step st;
                finish_scan(I, C, s.cur, node, __shfl_sync(kFull, pp.t, __ffs(owner) - 1), lane, st);
                __syncwarp();
                if (lane == 0) {
                    s.kind = 2;
                    s.v = st.v;
                    s.d = st.d;
                    s.slots = 0xFFu | (st.mirror << 8);
                }
                __syncwarp();
            }
            __syncthreads();  // every warp has read *nreq and its parts
            if (threadIdx.x == 0) *nreq = 0;
        }
        // (3) bump the counters of this step's edges, record the step
        for (uint32_t j = 0; j < my_ants; ++j) {
            const uint32_t a = gw + j * W;
            uint32_t *vis = vis_base + j * I.words;
            DefAnt<RNG> &s = ants[j];
            const uint32_t v = s.v, slots = s.slots;
            wc.count(s.kind, n - t);
            if (due) {
                ++wc.updates;
                bump_copy(C, n, s.cur, v, slots, lane);
            }
            __syncwarp();
            if (lane == 0) {
                vis[v >> 5] |= 1u << (v & 31);
                C.routes[static_cast<size_t>(a) * n + t] = v;
                s.len += s.d;
            }
            __syncwarp();
        }
        grid_sync();
        for (uint32_t j = 0; j < my_ants; ++j) {
            DefAnt<RNG> &s = ants[j];
            if (due) fold_copy(C, n, s.cur, s.v, s.slots, lane);
            __syncwarp();
            if (lane == 0) s.cur = s.v;
            __syncwarp();
        }
        if (due) grid_sync();
    }

    // closing edges: a separate pass after step n-1
    const bool close_due = (n % C.k) == 0;
    for (uint32_t j = 0; j < my_ants; ++j) {
        const uint32_t a = gw + j * W;
        DefAnt<RNG> &s = ants[j];
        int pos;
        uint32_t mirror;
        int32_t d;
        bool have_d;
        closing_slots(C, s.cur, s.start, lane, pos, mirror, d, have_d);
        if (!have_d)
            d = tsplib_distance(I.type, __ldg(I.xs + s.cur), __ldg(I.ys + s.cur), __ldg(I.xs + s.start),
                                __ldg(I.ys + s.start));
        const uint32_t slots = (static_cast<uint32_t>(pos) & 0xFFu) | (mirror << 8);
        if (close_due) {
            ++wc.updates;
            bump_copy(C, n, s.cur, s.start, slots, lane);
        }
        __syncwarp();
        if (lane == 0) {
            C.lens[a] = s.len + d;
            s.slots = slots;
        }
        __syncwarp();
    }
    if (close_due) {
        grid_sync();
        for (uint32_t j = 0; j < my_ants; ++j) fold_copy(C, n, ants[j].cur, ants[j].start, ants[j].slots, lane);
    }
    wc.flush(C.counters, lane, my_ants * (n - 1));
}

// ============================================================ SYNC x SELECTIVE

// SPEC SYNC over the selective memory (the oracle's SYNC mode with SELECTIVE
// memory): every step all ants select against the step-start records, then
// the step's local updates are applied in ant order -- per ant record u then
// record v (D4).  Inserts into a record do not commute (FIFO eviction), so the
// apply pass sorts the step's 2m record operations by (record, ant, u/v) and
// one thread walks each record's operations in that order.  Deterministic,
// bit-exact with the oracle; a parity mode, launched per step.

template <class RNG>
struct SyncAnt {              // per-ant state between the per-step launches
    RNG rng;
    long long len;
    uint32_t cur, start;
    uint32_t roulette, fallback, fb_elems;
};

// op key: record << 32 | ant << 1 | (0: record u gets v, 1: record v gets u);
// payload: the neighbour
__device__ __forceinline__ void post_op(uint4 *ops, uint32_t i, uint32_t record, uint32_t ant, uint32_t sub,
                                        uint32_t nb) {
    const uint64_t key = (static_cast<uint64_t>(record) << 32) | (ant << 1) | sub;
    ops[i] = make_uint4(static_cast<uint32_t>(key), static_cast<uint32_t>(key >> 32), nb, 0u);
}

template <class RNG>
__global__ void k_ssync_init(DevInstance I, DevColony C, DevSpmSync Y) {
    const int lane = threadIdx.x & 31;
    const uint32_t a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (a >= C.m) return;
    uint32_t *vis = Y.vis + static_cast<size_t>(a) * I.words;
    for (uint32_t i = lane; i < I.words; i += 32) vis[i] = 0;
    RNG rng;
    rng_init(rng, C, *C.iter, a);
    const uint32_t start = static_cast<uint32_t>(uniform_int(rng, I.n));
    __syncwarp();
    if (lane == 0) {
        vis[start >> 5] |= 1u << (start & 31);
        SyncAnt<RNG> &s = reinterpret_cast<SyncAnt<RNG> *>(Y.ants)[a];
        s.rng = rng;
        s.len = 0;
        s.cur = s.start = start;
        s.roulette = s.fallback = s.fb_elems = 0;
        C.routes[static_cast<size_t>(a) * I.n] = start;
    }
}

template <class RNG>
__global__ void __maxnreg__(kMaxRegs) k_ssync_select(DevInstance I, DevColony C, DevSpmSync Y, uint32_t t,
                                                     int due) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double *scratch = reinterpret_cast<double *>(smem) + wib * 32;
    const uint32_t a = blockIdx.x * (blockDim.x >> 5) + wib;
    if (a >= C.m) return;
    SyncAnt<RNG> &s = reinterpret_cast<SyncAnt<RNG> *>(Y.ants)[a];
    const uint32_t *vis = Y.vis + static_cast<size_t>(a) * I.words;
    const uint32_t cur = s.cur;
    RNG rng = s.rng;
    const uint4 el = __ldg(C.rows + static_cast<size_t>(cur) * 32 + lane);
    // the step-start record of cur: slot j in lane j
    const bool mine = static_cast<uint32_t>(lane) < C.S;
    const double val = mine ? ld_relaxed(C.spm.vals(cur) + lane) : 0.0;
    const uint32_t idl = mine ? ld_relaxed_u32(C.spm.ids(cur) + lane) : kEmpty;
    auto lookup = [&](uint32_t v) {  // all lanes call; first matching slot
        int hit = -1;
        for (int j = static_cast<int>(C.S) - 1; j >= 0; --j)
            if (__shfl_sync(kFull, idl, j) == v) hit = j;
        const double x = __shfl_sync(kFull, val, hit < 0 ? 0 : hit);
        return hit < 0 ? C.tau_min : x;
    };
    const double tau_lane = lookup(el.x & kIdMask);
    Lookahead<RNG> la;
    la.prepare(rng);
    Step st;
    select_step(I, C, vis, cur, el, tau_lane, rng, la, scratch, lane,
                [&](uint32_t v, bool act) { return lookup(act ? v : kEmpty); }, st);
    if (st.kind == 0) rng.advance();
    __syncwarp();
    if (lane == 0) {
        Y.vis[static_cast<size_t>(a) * I.words + (st.v >> 5)] |= 1u << (st.v & 31);
        C.routes[static_cast<size_t>(a) * I.n + t] = st.v;
        s.rng = rng;
        s.len += st.d;
        s.cur = st.v;
        s.roulette += st.kind == 1;
        s.fallback += st.kind == 2;
        s.fb_elems += st.kind == 2 ? I.n - t : 0u;
        if (due) {
            post_op(Y.ops, 2 * a, cur, a, 0, st.v);
            post_op(Y.ops, 2 * a + 1, st.v, a, 1, cur);
        } else {
            Y.ops[2 * a] = Y.ops[2 * a + 1] = make_uint4(kEmpty, kEmpty, 0u, 0u);
        }
    }
}

// closing edges (after step n-1): lengths, counters, and the closing ops
template <class RNG>
__global__ void k_ssync_close(DevInstance I, DevColony C, DevSpmSync Y, int due) {
    const int lane = threadIdx.x & 31;
    const uint32_t a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (a >= C.m) return;
    SyncAnt<RNG> &s = reinterpret_cast<SyncAnt<RNG> *>(Y.ants)[a];
    (void)lane;
    const int32_t d = tsplib_distance(I.type, __ldg(I.xs + s.cur), __ldg(I.ys + s.cur), __ldg(I.xs + s.start),
                                      __ldg(I.ys + s.start));
    if (lane == 0) {
        C.lens[a] = s.len + d;
        if (due) {
            post_op(Y.ops, 2 * a, s.cur, a, 0, s.start);
            post_op(Y.ops, 2 * a + 1, s.start, a, 1, s.cur);
        } else {
            Y.ops[2 * a] = Y.ops[2 * a + 1] = make_uint4(kEmpty, kEmpty, 0u, 0u);
        }
        using ull = unsigned long long;
        const uint32_t steps = I.n - 1;
        const uint32_t updates = (steps / C.k) + (due ? 1u : 0u);
        atomicAdd(C.counters + kCntUpdates, static_cast<ull>(updates));
        atomicAdd(C.counters + kCntGreedy, static_cast<ull>(steps - s.roulette - s.fallback));
        if (s.roulette) atomicAdd(C.counters + kCntRoulette, static_cast<ull>(s.roulette));
        if (s.fallback) atomicAdd(C.counters + kCntFallback, static_cast<ull>(s.fallback));
        if (s.fb_elems) atomicAdd(C.counters + kCntFallbackElems, static_cast<ull>(s.fb_elems));
    }
}

// One CTA: bitonic sort of the step's 2m op keys (with their index), then
// every record's operations applied in (ant, u/v) order by one thread.
__global__ void __launch_bounds__(1024) k_ssync_apply(DevColony C, DevSpmSync Y, uint32_t count, uint32_t pow2) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t *key = reinterpret_cast<uint64_t *>(smem);
    uint32_t *idx = reinterpret_cast<uint32_t *>(key + pow2);
    for (uint32_t i = threadIdx.x; i < pow2; i += blockDim.x) {
        if (i < count) {
            const uint4 o = Y.ops[i];
            key[i] = (static_cast<uint64_t>(o.y) << 32) | o.x;
        } else {
            key[i] = ~0ull;
        }
        idx[i] = i;
    }
    __syncthreads();
    for (uint32_t k = 2; k <= pow2; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < pow2; i += blockDim.x) {
                const uint32_t l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    if ((key[i] > key[l]) == up) {
                        const uint64_t tk = key[i]; key[i] = key[l]; key[l] = tk;
                        const uint32_t ti = idx[i]; idx[i] = idx[l]; idx[l] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    unsigned long long hits = 0, misses = 0;
    for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) {
        if (key[i] == ~0ull) continue;
        const uint32_t r = static_cast<uint32_t>(key[i] >> 32);
        if (i > 0 && static_cast<uint32_t>(key[i - 1] >> 32) == r) continue;  // not a segment head
        for (uint32_t j = i; j < count && key[j] != ~0ull && static_cast<uint32_t>(key[j] >> 32) == r; ++j) {
            const uint4 o = Y.ops[idx[j]];
            if (spm_update_mem(C.spm, r, o.z, C.c_l, C.c_0, C.tau_min, nullptr)) ++hits; else ++misses;
        }
    }
    if (hits) atomicAdd(C.counters + kCntHits, hits);
    if (misses) atomicAdd(C.counters + kCntMisses, misses);
}

// Large colonies: the step's keys sorted device-wide (cub radix sort, stable,
// 56 key bits: record < 2^24 above (ant << 1 | u/v)), then a thread per
// record segment applies its operations in order -- the k_ssync_apply walk.
__global__ void k_ssync_keys(DevSpmSync Y, uint32_t count) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint4 o = Y.ops[i];
    Y.keys_in[i] = (static_cast<unsigned long long>(o.y) << 32) | o.x;
    Y.idx_in[i] = i;
}

__global__ void k_ssync_apply_sorted(DevColony C, DevSpmSync Y, uint32_t count) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long hits = 0, misses = 0;
    if (i < count) {
        const unsigned long long k = Y.keys_out[i];
        const uint32_t r = static_cast<uint32_t>(k >> 32);
        const bool head = k != ~0ull && (i == 0 || static_cast<uint32_t>(Y.keys_out[i - 1] >> 32) != r);
        if (head) {
            for (uint32_t j = i; j < count && Y.keys_out[j] != ~0ull && static_cast<uint32_t>(Y.keys_out[j] >> 32) == r;
                 ++j) {
                const uint4 o = Y.ops[Y.idx_out[j]];
                if (spm_update_mem(C.spm, r, o.z, C.c_l, C.c_0, C.tau_min, nullptr)) ++hits; else ++misses;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        hits += __shfl_xor_sync(kFull, hits, o);
        misses += __shfl_xor_sync(kFull, misses, o);
    }
    if ((threadIdx.x & 31) == 0 && (hits | misses)) {
        atomicAdd(C.counters + kCntHits, hits);
        atomicAdd(C.counters + kCntMisses, misses);
    }
}

size_t spm_sync_sort_tmp_bytes(uint32_t count) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const unsigned long long *>(nullptr),
                                    static_cast<unsigned long long *>(nullptr), static_cast<const uint32_t *>(nullptr),
                                    static_cast<uint32_t *>(nullptr), static_cast<int>(count), 0, 56);
    return bytes;
}

static void spm_sync_apply_wide(const DevColony &C, const DevSpmSync &Y, uint32_t count, cudaStream_t s) {
    k_ssync_keys<<<blocks_for(count, 256), 256, 0, s>>>(Y, count);
    size_t bytes = Y.sort_tmp_bytes;
    cub::DeviceRadixSort::SortPairs(Y.sort_tmp, bytes, Y.keys_in, Y.keys_out, Y.idx_in, Y.idx_out,
                                    static_cast<int>(count), 0, 56, s);
    k_ssync_apply_sorted<<<blocks_for(count, 256), 256, 0, s>>>(C, Y, count);
}

template <class RNG>
static int spm_sync_iteration(const DevInstance &I, const DevColony &C, const DevSpmSync &Y, cudaStream_t s) {
    const unsigned wpb = 4, grid = blocks_for(C.m, wpb);
    const uint32_t count = 2 * C.m;
    uint32_t pow2 = 1;
    while (pow2 < count) pow2 <<= 1;
    const size_t apply_smem = static_cast<size_t>(pow2) * (sizeof(uint64_t) + sizeof(uint32_t));
    // above one CTA's sort: device-wide radix sort (also when the context
    // allocated it for a smaller colony: ACS_SSYNC_WIDE, the test of that path)
    const bool wide = apply_smem > 200 * 1024 || Y.sort_tmp;
    if (wide && !Y.sort_tmp) return -1;
    if (!wide)
        cudaFuncSetAttribute(k_ssync_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(apply_smem));
    auto apply = [&] {
        if (wide) spm_sync_apply_wide(C, Y, count, s);
        else k_ssync_apply<<<1, 1024, apply_smem, s>>>(C, Y, count, pow2);
    };
    k_ssync_init<RNG><<<grid, wpb * 32, 0, s>>>(I, C, Y);
    for (uint32_t t = 1; t < I.n; ++t) {
        const int due = (t % C.k) == 0;
        k_ssync_select<RNG><<<grid, wpb * 32, wpb * 32 * sizeof(double), s>>>(I, C, Y, t, due);
        if (due) apply();
    }
    const int close_due = (I.n % C.k) == 0;
    k_ssync_close<RNG><<<grid, wpb * 32, 0, s>>>(I, C, Y, close_due);
    if (close_due) apply();
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_spm_sync(int rng, const DevInstance &I, const DevColony &C, const DevSpmSync &Y, cudaStream_t s) {
    return rng == ACS_RNG_PHILOX ? spm_sync_iteration<Philox>(I, C, Y, s) : spm_sync_iteration<Xoshiro>(I, C, Y, s);
}

size_t spm_sync_ant_bytes() { return std::max(sizeof(SyncAnt<Philox>), sizeof(SyncAnt<Xoshiro>)); }

// ============================================================ iteration end

// select_best (ties -> lowest ant), strict is_better, best
// tour copy, per-iteration stats; one CTA.
__global__ void __launch_bounds__(1024) k_best(DevColony C, DevBest B, uint32_t n, uint32_t slot) {
    __shared__ unsigned long long red_len[32];
    __shared__ uint32_t red_ant[32];
    __shared__ int improved;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    long long bl = LLONG_MAX;
    uint32_t ba = 0xffffffffu;
    for (uint32_t a = tid; a < C.m; a += blockDim.x) {
        const long long l = C.lens[a];
        if (l < bl) { bl = l; ba = a; }  // ascending a per thread: strict keeps lowest
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long ol = __shfl_xor_sync(kFull, bl, o);
        const uint32_t oa = __shfl_xor_sync(kFull, ba, o);
        if (ol < bl || (ol == bl && oa < ba)) { bl = ol; ba = oa; }
    }
    if (lane == 0) { red_len[wid] = static_cast<unsigned long long>(bl); red_ant[wid] = ba; }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        bl = lane < nw ? static_cast<long long>(red_len[lane]) : LLONG_MAX;
        ba = lane < nw ? red_ant[lane] : 0xffffffffu;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long ol = __shfl_xor_sync(kFull, bl, o);
            const uint32_t oa = __shfl_xor_sync(kFull, ba, o);
            if (ol < bl || (ol == bl && oa < ba)) { bl = ol; ba = oa; }
        }
        if (lane == 0) {
            red_len[0] = static_cast<unsigned long long>(bl);
            red_ant[0] = ba;
            improved = bl < *B.len;  // strict
        }
    }
    __syncthreads();
    const long long ib_len = static_cast<long long>(red_len[0]);
    const uint32_t ib_ant = red_ant[0];
    if (improved) {
        const uint4 *r = reinterpret_cast<const uint4 *>(C.routes + static_cast<size_t>(ib_ant) * n);
        if ((n & 3) == 0) {
            for (uint32_t i = tid; i < n / 4; i += blockDim.x) reinterpret_cast<uint4 *>(B.tour)[i] = r[i];
        } else {
            const uint32_t *rr = C.routes + static_cast<size_t>(ib_ant) * n;
            for (uint32_t i = tid; i < n; i += blockDim.x) B.tour[i] = rr[i];
        }
    }
    __syncthreads();
    if (tid == 0) {
        const long long gb = improved ? ib_len : *B.len;
        if (improved) *B.len = ib_len;
        acs_iter_stats *s = reinterpret_cast<acs_iter_stats *>(B.stats) + slot;
        s->iter_best_len = ib_len;
        s->iter_best_ant = ib_ant;
        s->improved = improved ? 1u : 0u;
        s->global_best_len = gb;
        *B.iter += 1;
        atomicAdd(C.counters + kCntIters, 1ull);
    }
}

// Record v in u's hot list (non-candidate neighbours whose trail the global
// update raised above tau0).  Tour edges are distinct, so no two threads insert
// the same (u, v) concurrently; an earlier iteration's insert is visible here.
// Past kHot entries the row is marked full and its fallback scans everything.
__device__ __forceinline__ void hot_insert(const DevColony &C, uint32_t u, uint32_t v) {
    const uint32_t have = C.hot_cnt[u];
    const uint32_t *h = C.hot + static_cast<size_t>(u) * kHot;
    for (uint32_t i = 0; i < min(have, kHot); ++i)
        if (h[i] == v) return;
    if (have > kHot) return;
    const uint32_t slot = atomicAdd(C.hot_cnt + u, 1u);
    if (slot < kHot) C.hot[static_cast<size_t>(u) * kHot + slot] = v;
}

// dense global update, warp per global-best edge (a,b): lanes 0-3 update the
// four copies of the trail; tour edges are distinct, so no two warps touch
// the same word.
__global__ void k_global_dense(DevInstance I, DevColony C, DevBest B) {
    const int lane = threadIdx.x & 31;
    const uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t n = I.n;
    if (i >= n) return;
    const uint32_t a = B.tour[i], b = B.tour[i + 1 == n ? 0 : i + 1];
    const double c_d = __dmul_rn(B.alpha, __ddiv_rn(1.0, static_cast<double>(*B.len)));
    const uint32_t ida = __ldg(&C.rows[static_cast<size_t>(a) * 32 + lane].x);
    const unsigned hit = __ballot_sync(kFull, static_cast<uint32_t>(lane) < C.L && (ida & kIdMask) == b);
    const int pos = hit ? __ffs(hit) - 1 : -1;
    uint32_t mirror = kNoMirror;
    if (hit) {
        mirror = __shfl_sync(kFull, ida >> 24, pos);
    } else {
        const uint32_t idb = __ldg(&C.rows[static_cast<size_t>(b) * 32 + lane].x) & kIdMask;
        const unsigned mm = __ballot_sync(kFull, static_cast<uint32_t>(lane) < C.L && idb == a);
        if (mm) mirror = static_cast<uint32_t>(__ffs(mm) - 1);
    }
    double *p = copy_addr(C, n, a, b, pos, mirror, lane);
    if (p) *p = affine(*p, B.c_g, c_d);
    if (C.hot && lane == 0) {
        if (pos < 0) hot_insert(C, a, b);
        if (mirror == kNoMirror) hot_insert(C, b, a);
    }
}

// selective global update, thread per record r = tour[j]: edge j-1 (b-side,
// neighbour tour[j-1]) precedes edge j (a-side, neighbour tour[j+1]); record
// tour[0] goes a-side first -- exactly the sequential tour-order semantics.
__global__ void k_global_spm(DevInstance I, DevColony C, DevBest B) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t n = I.n;
    unsigned long long hits = 0, misses = 0;
    if (j < n) {
        const double c_d = __dmul_rn(B.alpha, __ddiv_rn(1.0, static_cast<double>(*B.len)));
        const uint32_t r = B.tour[j];
        const uint32_t nb_prev = B.tour[j == 0 ? n - 1 : j - 1];
        const uint32_t nb_next = B.tour[j + 1 == n ? 0 : j + 1];
        const uint32_t first = j == 0 ? nb_next : nb_prev;
        const uint32_t second = j == 0 ? nb_prev : nb_next;
        if (spm_update_mem(C.spm, r, first, B.c_g, c_d, C.tau_min, nullptr)) ++hits; else ++misses;
        if (spm_update_mem(C.spm, r, second, B.c_g, c_d, C.tau_min, nullptr)) ++hits; else ++misses;
        if (C.hot) {
            bool in1 = false, in2 = false;
            for (uint32_t l = 0; l < C.L; ++l) {
                const uint32_t id = __ldg(&C.rows[static_cast<size_t>(r) * 32 + l].x) & kIdMask;
                in1 |= id == first;
                in2 |= id == second;
            }
            if (!in1) hot_insert(C, r, first);
            if (!in2) hot_insert(C, r, second);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        hits += __shfl_xor_sync(kFull, hits, o);
        misses += __shfl_xor_sync(kFull, misses, o);
    }
    if ((threadIdx.x & 31) == 0 && (hits | misses)) {
        atomicAdd(C.counters + kCntHits, hits);
        atomicAdd(C.counters + kCntMisses, misses);
    }
}

__global__ void k_adopt_best(const uint32_t *tour, const int64_t *len, uint32_t n, DevBest B) {
    __shared__ int take;
    if (threadIdx.x == 0) take = *len < *B.len;
    __syncthreads();
    if (!take) return;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) B.tour[i] = tour[i];
    __syncthreads();
    if (threadIdx.x == 0) *B.len = *len;
}

// Island key: L_gb << kIslandRankBits | rank, so a min-allreduce picks the best
// colony with ties to the lowest rank.  A colony with no tour yet (L_gb still
// the LLONG_MAX sentinel) -- or a length too large to shift -- packs the
// sentinel kNoIslandKey itself: it never wins against a real tour, and if
// every rank holds it the exchange adopts nothing.
__global__ void k_island_pack(const int64_t *best_len, int rank, int64_t *key) {
    const int64_t l = *best_len;
    *key = (l < 0 || l > kIslandMaxLen) ? kNoIslandKey : ((l << kIslandRankBits) | rank);
}

__global__ void k_island_mask(const int64_t *key, int rank, const uint32_t *tour, uint32_t n,
                              uint32_t *x_tour, int64_t *x_len) {
    const int64_t k = *key;
    const bool none = k == kNoIslandKey;
    const bool mine = !none && static_cast<int>(k & kIslandRankMask) == rank;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        x_tour[i] = mine ? tour[i] : 0u;
    // LLONG_MAX: k_adopt_best's strict < never takes it
    if (blockIdx.x == 0 && threadIdx.x == 0) *x_len = none ? LLONG_MAX : (k >> kIslandRankBits);
}

// In-process exchange (acs_gpu_island_exchange_local): the two NCCL
// all-reduces of the multi-GPU path, restated as device reductions over the
// colonies of one process on one GPU -- min over the packed keys, and the sum
// of the masked tours (only the winner's is non-zero).  The pack / mask /
// adopt kernels around them are the ones the NCCL path runs.
__global__ void k_island_min(const int64_t *keys, int count, int64_t *out) {
    int64_t k = kNoIslandKey;
    for (int i = threadIdx.x; i < count; i += blockDim.x) k = min(k, keys[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) k = min(k, static_cast<int64_t>(shfl_xor_u64(static_cast<uint64_t>(k), o)));
    __shared__ int64_t part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = k;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) k = min(k, part[w]);
        *out = k;
    }
}

__global__ void k_island_sum(const uint32_t *const *tours, int count, uint32_t n, uint32_t *out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t x = 0;
        for (int r = 0; r < count; ++r) x += tours[r][i];
        out[i] = x;
    }
}

// ============================================================ launchers

static size_t construct_smem(const DevInstance &I, const DevColony &C, int wpb, bool pw, size_t extra = 0) {
    const size_t base = static_cast<size_t>(wpb) * (32 * sizeof(double) + I.words * sizeof(uint32_t)) +
                        (pw ? (512 + C.pw_hi_n) * sizeof(double) : 0);
    return extra ? ((base + 15) & ~static_cast<size_t>(15)) + extra : base;
}

template <class K>
static void launch_tour_kernel(K kernel, const DevInstance &I, const DevColony &C, bool one_warp,
                               cudaStream_t s, bool pw = false, size_t extra_smem = 0) {
    const int threads = one_warp ? 32 : kBlock;
    const int wpb = threads / 32;
    unsigned grid = one_warp ? 1u : blocks_for(C.m, wpb);
    // Diagnostic: ACS_RESIDENT_ANTS=W caps the ants constructing at once (the
    // grid-stride loop runs the rest as later waves), to compare the relaxed
    // variants with the oracle's RELAXED mode at the same concurrency.
    static const unsigned cap = [] {
        const char *e = std::getenv("ACS_RESIDENT_ANTS");
        return e ? static_cast<unsigned>(std::strtoul(e, nullptr, 10)) : 0u;
    }();
    if (cap && !one_warp) grid = std::min(grid, std::max(1u, cap / wpb));
    const size_t smem = construct_smem(I, C, wpb, pw, extra_smem);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kernel<<<grid, threads, smem, s>>>(I, C);
}

// Register cap vs residency: at 96 registers 20 ants fit per SM (one wave for
// pr2392); a colony larger than that runs in waves, and a 72-register build
// (28 ants per SM, a few spills off the hot loop) finishes rnd10k in three
// waves instead of four (measured: relaxed 41.9 -> 38.2, atomic 57.9 -> 49.8 ms).
constexpr int kWideRegs = 72;

template <int kMode, class RNG, int kRegs, bool kLean, bool kPw1 = false>
constexpr auto dense_kernel() {
    if constexpr (kLean && kMode == 0 && kRegs == kWideRegs && std::is_same_v<RNG, PhiloxWarp>)
        return k_tour_lean<kMode, PhiloxWarpU, kRegs, kPw1>;  // see PhiloxWarpU
    else if constexpr (kLean) return k_tour_lean<kMode, RNG, kRegs, kPw1>;
    else return k_construct_dense<kMode, RNG, kRegs>;
}

template <int kMode, class RNG, bool kLean, bool kPw1 = false>
static void launch_dense_t(const DevInstance &I, const DevColony &C, bool one_warp, cudaStream_t s, bool pw) {
    auto narrow = dense_kernel<kMode, RNG, kMaxRegs, kLean, kPw1>();
    const size_t extra = kPw1 ? (static_cast<size_t>(C.m) + 1) * sizeof(double) : 0;
    if (!one_warp) {
        // The narrow-vs-wide decision (occupancy query) is made once per
        // (device, shared memory, m) and remembered per host thread: it costs
        // microseconds of host time between the step's start event and the
        // kernel, which small instances (d198: 0.17 ms per step) would see.
        struct Memo { int dev = -1; size_t smem = 0; uint32_t m = 0; bool wide = false; };
        static thread_local Memo memo;
        int dev = 0;
        cudaGetDevice(&dev);
        const size_t smem = construct_smem(I, C, kBlock / 32, pw, extra);
        if (memo.dev != dev || memo.smem != smem || memo.m != C.m) {
            int sms = 0, per_sm = 0;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(narrow, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, narrow, kBlock, smem);
            memo = Memo{dev, smem, C.m, static_cast<uint64_t>(per_sm) * sms * (kBlock / 32) < C.m};
        }
        if (memo.wide) {
            launch_tour_kernel(dense_kernel<kMode, RNG, kWideRegs, kLean, kPw1>(), I, C, false, s, pw, extra);
            return;
        }
    }
    launch_tour_kernel(narrow, I, C, one_warp, s, pw, extra);
}

template <int kMode, class RNG>
static void launch_dense(const DevInstance &I, const DevColony &C, bool one_warp, cudaStream_t s, bool pw = false) {
    if (C.k == 1 && C.L == 32 && !one_warp && (!pw || C.pw_hi_n <= kLeanPwHi)) {
#ifndef ACS_NO_PW1
        if constexpr (kMode == 1) {
            // k_tour_lean, ATOMIC: the one-table c_l^c in shared memory, when its
            // (m + 1) * 8 B per CTA still lets the whole colony be resident in
            // one wave (pr2392: 19 KB, 10 CTAs per SM as without it); else the
            // two-table build (measured: pr2392 atomic 1.554 -> 1.488 ms)
            struct Memo { int dev = -1; uint32_t m = 0, words = 0; bool fits = false; };
            static thread_local Memo memo;
            int dev = 0;
            cudaGetDevice(&dev);
            if (memo.dev != dev || memo.m != C.m || memo.words != I.words) {
                bool fits = false;
                if (C.m <= kPw1Max) {
                    auto k = dense_kernel<kMode, RNG, kMaxRegs, true, true>();
                    const size_t smem = construct_smem(I, C, kBlock / 32, false, (static_cast<size_t>(C.m) + 1) * sizeof(double));
                    int sms = 0, per_sm = 0;
                    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                    if (smem > 48 * 1024)
                        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kBlock, smem);
                    fits = static_cast<uint64_t>(per_sm) * sms * (kBlock / 32) >= C.m;
                }
                memo = Memo{dev, C.m, I.words, fits};
            }
            if (memo.fits) {
                launch_dense_t<kMode, RNG, true, true>(I, C, one_warp, s, false);
                return;
            }
        }
#endif
        launch_dense_t<kMode, RNG, true>(I, C, one_warp, s, false);  // k_tour_lean: static power tables
        return;
    }
    launch_dense_t<kMode, RNG, false>(I, C, one_warp, s, pw);
}

template <class RNG>
static void launch_spm_rng(const DevInstance &I, const DevColony &C, bool one_warp, cudaStream_t s) {
    switch (C.S) {
        case 1: launch_tour_kernel(k_construct_spm<1, RNG>, I, C, one_warp, s); break;
        case 2: launch_tour_kernel(k_construct_spm<2, RNG>, I, C, one_warp, s); break;
        case 4: launch_tour_kernel(k_construct_spm<4, RNG>, I, C, one_warp, s); break;
        case 8:
            if (C.k == 1 && C.L == 32 && !one_warp) launch_tour_kernel(k_spm_lean<RNG>, I, C, false, s);
            else launch_tour_kernel(k_construct_spm<8, RNG>, I, C, one_warp, s);
            break;
        default: launch_tour_kernel(k_construct_spm<16, RNG>, I, C, one_warp, s); break;
    }
}

void launch_construct(int variant, int rng, const DevInstance &I, const DevColony &C,
                      cudaStream_t s) {
    const bool philox = rng == ACS_RNG_PHILOX;
    switch (variant) {
        case ACS_VARIANT_ATOMIC:
            if (philox) launch_dense<1, PhiloxWarp>(I, C, false, s, true);
            else launch_dense<1, Xoshiro>(I, C, false, s, true);
            break;
        case ACS_VARIANT_RELAXED:
            if (philox) launch_dense<0, PhiloxWarp>(I, C, false, s);
            else launch_dense<0, Xoshiro>(I, C, false, s);
            break;
        case ACS_VARIANT_SEQ:
            if (philox) launch_dense<0, PhiloxWarp>(I, C, true, s);
            else launch_dense<0, Xoshiro>(I, C, true, s);
            break;
        case ACS_VARIANT_SPM:
        case ACS_VARIANT_SPM_SEQ:
            if (philox) launch_spm_rng<PhiloxWarp>(I, C, variant == ACS_VARIANT_SPM_SEQ, s);
            else launch_spm_rng<Xoshiro>(I, C, variant == ACS_VARIANT_SPM_SEQ, s);
            break;
        default: break;
    }
}

template <class RNG>
static int deferred_launch(const DevInstance &I, const DevColony &C, DevDeferred D, cudaStream_t s) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int wpb = kDefBlock / 32;
    auto kern = k_deferred<RNG>;
    auto smem_of = [&](uint32_t a) { return DefSmem(wpb, a, I.words).bytes; };
    uint32_t A = 1;
    size_t smem = 0;
    for (;; ++A) {
        smem = smem_of(A);
        if (smem > 220 * 1024 || A > 0xFFFFu) return -1;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDefBlock, smem);
        if (per_sm < 1) return -1;
        if (static_cast<uint64_t>(sms) * per_sm * wpb * A >= C.m) break;
    }
    const unsigned grid = std::min<unsigned>(sms * per_sm, blocks_for(C.m, A));
    D.ants_per_warp = A;
    void *args[] = {const_cast<DevInstance *>(&I), const_cast<DevColony *>(&C), &D};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void *>(kern), grid, kDefBlock, args, smem, s) == cudaSuccess
               ? 0
               : -1;
}

int launch_deferred(int rng, const DevInstance &I, const DevColony &C, const DevDeferred &D,
                    cudaStream_t s) {
    return rng == ACS_RNG_PHILOX ? deferred_launch<Philox>(I, C, D, s) : deferred_launch<Xoshiro>(I, C, D, s);
}

void launch_epilogue(bool spm, bool fold, const DevInstance &I, const DevColony &C,
                     const DevBest &B, uint32_t slot, cudaStream_t s) {
    k_best<<<1, 1024, 0, s>>>(C, B, I.n, slot);
    if (fold) {  // grid sized to the counters (4 per thread), at most 8 CTAs per SM
        const size_t dense = static_cast<size_t>(I.n) * I.n;
        k_fold_counts<<<std::min<size_t>(static_cast<size_t>(device_sms()) * 8, blocks_for(dense / 4 + 1, 256)), 256, 0, s>>>(
            C, dense, static_cast<size_t>(I.n) * 32);
    }
    if (spm) k_global_spm<<<blocks_for(I.n, 256), 256, 0, s>>>(I, C, B);
    else k_global_dense<<<blocks_for(I.n, 8), 256, 0, s>>>(I, C, B);
}

void launch_adopt_best(const uint32_t *tour, const int64_t *len, const DevInstance &I,
                       const DevBest &B, cudaStream_t s) {
    k_adopt_best<<<1, 256, 0, s>>>(tour, len, I.n, B);
}

void launch_island_pack(const int64_t *best_len, int rank, int64_t *key, cudaStream_t s) {
    k_island_pack<<<1, 1, 0, s>>>(best_len, rank, key);
}

void launch_island_mask(const int64_t *key, int rank, const uint32_t *best_tour, uint32_t n,
                        uint32_t *x_tour, int64_t *x_len, cudaStream_t s) {
    k_island_mask<<<std::min<unsigned>(blocks_for(n, 256), 64), 256, 0, s>>>(key, rank, best_tour, n,
                                                                            x_tour, x_len);
}

void launch_island_min(const int64_t *keys, int count, int64_t *out, cudaStream_t s) {
    k_island_min<<<1, 256, 0, s>>>(keys, count, out);
}

void launch_island_sum(const uint32_t *const *tours, int count, uint32_t n, uint32_t *out, cudaStream_t s) {
    k_island_sum<<<std::min<unsigned>(blocks_for(n, 256), 64), 256, 0, s>>>(tours, count, n, out);
}

}  // namespace acs_dev
