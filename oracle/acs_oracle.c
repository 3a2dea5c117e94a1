/*
 * oracle/acs_oracle.c -- TEST INFRASTRUCTURE ONLY (see acs_oracle.h).
 *
 * Plain C11 + OpenMP restatement of the reference ACS path.  Compiled with
 * -O2 -ffp-contract=off so every double operation is a single IEEE op in the
 * order written here; the sm_100a product follows the same order with
 * __dmul_rn/__dadd_rn, which is what makes bit-exact tour parity possible.
 *
 * Frozen semantic decisions are cited as Pn.
 */
#include "acs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EMPTY_ID 0xFFFFFFFFu

/* ========================= instance ========================= */

/* tsp_instance.cpp:49-65 -- TSPLIB95 EUC_2D nint, CEIL_2D, ATT pseudo-Euclid */
int32_t orc_distance(int type, const double *xs, const double *ys, uint32_t u, uint32_t v) {
    const double xd = xs[u] - xs[v];
    const double yd = ys[u] - ys[v];
    const double sq = xd * xd + yd * yd;
    switch (type) {
        case ORC_EUC_2D: return (int32_t)(sqrt(sq) + 0.5);
        case ORC_CEIL_2D: return (int32_t)ceil(sqrt(sq));
        case ORC_ATT: {
            const double r = sqrt(sq / 10.0);
            const int32_t t = (int32_t)(r + 0.5);
            return ((double)t < r) ? t + 1 : t;
        }
        default: return 0;
    }
}

/* tsp_instance.cpp:23-47 (table for n <= 4096 in the reference) */
void orc_distance_table(uint32_t n, int type, const double *xs, const double *ys, int32_t *out) {
    #pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < (int64_t)n; ++u)
        for (uint32_t v = 0; v < n; ++v)
            out[(size_t)u * n + v] = orc_distance(type, xs, ys, (uint32_t)u, v);
}

static int key_cmp(const void *a, const void *b) {
    const uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : (x > y);
}

/* tsp_instance.cpp:219-252: per node the min(cl, n-1) nearest, ordered by
 * (distance asc, id asc).  Restated as a full sort of (d<<32 | v) keys. */
uint32_t orc_build_candidates(uint32_t n, int type, const double *xs, const double *ys,
                              uint32_t cl, uint32_t *out) {
    const uint32_t len = cl < n - 1 ? cl : n - 1;
    #pragma omp parallel
    {
        uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * n);
        #pragma omp for schedule(static)
        for (int64_t u = 0; u < (int64_t)n; ++u) {
            uint32_t c = 0;
            for (uint32_t v = 0; v < n; ++v) {
                if (v == (uint32_t)u) continue;
                const int32_t d = orc_distance(type, xs, ys, (uint32_t)u, v);
                keys[c++] = ((uint64_t)(uint32_t)d << 32) | v;
            }
            qsort(keys, c, sizeof(uint64_t), key_cmp);
            for (uint32_t i = 0; i < len; ++i) out[(size_t)u * len + i] = (uint32_t)keys[i];
        }
        free(keys);
    }
    return len;
}

/* tsp_instance.cpp:254-280: greedy NN closed tour, ties -> lowest id */
int64_t orc_nn_tour_length(uint32_t n, int type, const double *xs, const double *ys, uint32_t start) {
    uint8_t *vis = (uint8_t *)calloc(n, 1);
    vis[start] = 1;
    uint32_t cur = start;
    int64_t total = 0;
    for (uint32_t step = 1; step < n; ++step) {
        int32_t bd = 0;
        uint32_t best = n;
        for (uint32_t v = 0; v < n; ++v) {
            if (vis[v]) continue;
            const int32_t d = orc_distance(type, xs, ys, cur, v);
            if (best == n || d < bd) { bd = d; best = v; }
        }
        vis[best] = 1;
        total += bd;
        cur = best;
    }
    total += orc_distance(type, xs, ys, cur, start);
    free(vis);
    return total;
}

/* tsp_instance.cpp:67-78: closed tour incl. the closing edge */
int64_t orc_tour_length(int type, const double *xs, const double *ys, const uint32_t *order, uint32_t len) {
    if (len == 0) return 0;
    int64_t total = 0;
    uint32_t prev = order[len - 1];
    for (uint32_t i = 0; i < len; ++i) {
        total += orc_distance(type, xs, ys, prev, order[i]);
        prev = order[i];
    }
    return total;
}

/* ========================= rng ========================= */

static uint64_t splitmix64(uint64_t *z) { /* rng.hpp:71-77 */
    *z += 0x9e3779b97f4a7c15ull;
    uint64_t x = *z;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void orc_rng_seed(orc_rng *r, uint64_t seed) { /* rng.hpp:20-28 */
    memset(r, 0, sizeof(*r));
    r->kind = ORC_RNG_XOSHIRO;
    uint64_t z = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&z);
    if ((r->s[0] | r->s[1] | r->s[2] | r->s[3]) == 0) r->s[0] = 0x9e3779b97f4a7c15ull;
}

void orc_rng_derive(orc_rng *r, int kind, uint64_t seed, uint64_t iteration, uint64_t ant) {
    if (kind == ORC_RNG_PHILOX) {
        /* counter-based stream: key = seed, counter = (draw, ant, iteration) */
        memset(r, 0, sizeof(*r));
        r->kind = ORC_RNG_PHILOX;
        r->key[0] = (uint32_t)seed;
        r->key[1] = (uint32_t)(seed >> 32);
        r->ctr_hi[0] = (uint32_t)ant;
        r->ctr_hi[1] = (uint32_t)iteration;
        r->ctr_hi[2] = (uint32_t)(iteration >> 32);
        r->draw = 0;
        return;
    }
    /* rng.hpp:30-35 */
    uint64_t h = seed;
    h ^= iteration * 0xbf58476d1ce4e5b9ull;
    h = splitmix64(&h);
    h ^= ant * 0x94d049bb133111ebull;
    h = splitmix64(&h);
    orc_rng_seed(r, h);
}

static uint64_t philox_draw(const uint32_t key_in[2], uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    return (uint64_t)c0 | ((uint64_t)c1 << 32);
}

uint64_t orc_rng_next_u64(orc_rng *r) {
    if (r->kind == ORC_RNG_PHILOX) {
        return philox_draw(r->key, r->draw++, r->ctr_hi[0], r->ctr_hi[1], r->ctr_hi[2]);
    }
    /* rng.hpp:37-47 xoshiro256** */
    uint64_t *s = r->s;
    const uint64_t result = rotl64(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

double orc_rng_uniform01(orc_rng *r) { /* rng.hpp:50-52 */
    return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

uint64_t orc_rng_uniform_int(orc_rng *r, uint64_t bound) { /* rng.hpp:55-68, Lemire */
    uint64_t x = orc_rng_next_u64(r);
    __uint128_t m = (__uint128_t)x * bound;
    uint64_t lo = (uint64_t)m;
    if (lo < bound) {
        const uint64_t threshold = (0 - bound) % bound;
        while (lo < threshold) {
            x = orc_rng_next_u64(r);
            m = (__uint128_t)x * bound;
            lo = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

/* ========================= op-level ========================= */

double orc_default_q0(uint32_t n) { /* SPEC.md:291-299, D10 */
    if (n <= 20) return 0.0;
    return (double)(n - 20) / (double)n;
}

double orc_tau0(uint32_t n, int64_t nn_len) { /* SPEC.md:171 D2 */
    return 1.0 / ((double)n * (double)nn_len);
}

/* P4: coefficients computed once, tau' = c_mul*tau + c_add */
double orc_local_update_value(double tau, double rho, double tau0) {
    const double c_l = 1.0 - rho, c_0 = rho * tau0;
    return c_l * tau + c_0;
}

double orc_global_update_value(double tau, double alpha, int64_t l_gb) {
    const double c_g = 1.0 - alpha, c_d = alpha * (1.0 / (double)l_gb);
    return c_g * tau + c_d;
}

/* P2 / D1: eta = 1/max(d,1); integral beta -> left-to-right repeated multiply */
static int beta_is_int(double beta) { return beta >= 0.0 && beta <= 64.0 && beta == floor(beta); }
static double eta_pow(double eta, double beta) {
    if (beta_is_int(beta)) {
        double e = 1.0;
        for (int i = 0; i < (int)beta; ++i) e = e * eta;
        return e;
    }
    return pow(eta, beta);
}
double orc_eta_beta(int32_t d, double beta) {
    const double eta = 1.0 / (double)(d > 0 ? d : 1);
    return eta_pow(eta, beta);
}
double orc_score(double tau, double eta, double beta) {
    return tau * eta_pow(eta, beta);
}

/* SPEC.md:220-228, D7: argmax, ties to earliest position */
uint32_t orc_greedy_pick(const double *scores, uint32_t len) {
    uint32_t best = 0;
    for (uint32_t i = 1; i < len; ++i)
        if (scores[i] > scores[best]) best = i;
    return best;
}

/* SPEC.md:229-237, D8, P5: sequential prefix in candidate order */
uint32_t orc_roulette_pick(const double *w, uint32_t len, double r) {
    double total = 0.0;
    for (uint32_t i = 0; i < len; ++i) total = total + w[i];
    if (total == 0.0) return 0; /* all-zero -> greedy tie rule (first) */
    const double thr = r * total;
    double prefix = 0.0;
    uint32_t last_pos = 0;
    for (uint32_t i = 0; i < len; ++i) {
        prefix = prefix + w[i];
        if (prefix > thr) return i;
        if (w[i] > 0.0) last_pos = i;
    }
    return last_pos; /* rounding left none: last positive weight */
}

uint32_t orc_select_best(const int64_t *lengths, uint32_t m) {
    uint32_t best = 0;
    for (uint32_t a = 1; a < m; ++a)
        if (lengths[a] < lengths[best]) best = a;
    return best;
}

/* ========================= selective store ========================= */

struct orc_spm {
    uint32_t n, s;
    double tau_min;
    uint32_t *ids;
    double *vals;
    uint32_t *tail;
    uint64_t hits, misses;
};

orc_spm *orc_spm_new(uint32_t n, uint32_t s, double tau_min) {
    orc_spm *p = (orc_spm *)calloc(1, sizeof(orc_spm));
    p->n = n; p->s = s; p->tau_min = tau_min;
    p->ids = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n * s);
    p->vals = (double *)malloc(sizeof(double) * (size_t)n * s);
    p->tail = (uint32_t *)malloc(sizeof(uint32_t) * n);
    for (size_t i = 0; i < (size_t)n * s; ++i) { p->ids[i] = EMPTY_ID; p->vals[i] = tau_min; }
    for (uint32_t u = 0; u < n; ++u) p->tail[u] = s - 1; /* D5 */
    return p;
}

void orc_spm_free(orc_spm *p) {
    if (!p) return;
    free(p->ids); free(p->vals); free(p->tail); free(p);
}

/* first slot of record u holding v, else tau_min */
static double spm_read_relaxed(const orc_spm *p, uint32_t u, uint32_t v) {
    const uint32_t *ids = p->ids + (size_t)u * p->s;
    for (uint32_t j = 0; j < p->s; ++j) {
        uint32_t id;
        __atomic_load(&ids[j], &id, __ATOMIC_RELAXED);
        if (id == v) {
            double x;
            __atomic_load(&p->vals[(size_t)u * p->s + j], &x, __ATOMIC_RELAXED);
            return x;
        }
    }
    return p->tau_min;
}
double orc_spm_read(const orc_spm *p, uint32_t u, uint32_t v) { return spm_read_relaxed(p, u, v); }

/* Fig. alg:3 / SPEC.md:128-154: hit -> update in place (tail untouched);
 * miss -> value from tau_min, insert at (tail+1) % s evicting the oldest. */
static int spm_update(orc_spm *p, uint32_t u, uint32_t v, double c_mul, double c_add, int count) {
    const size_t base = (size_t)u * p->s;
    for (uint32_t j = 0; j < p->s; ++j) {
        uint32_t id;
        __atomic_load(&p->ids[base + j], &id, __ATOMIC_RELAXED);
        if (id == v) {
            double x;
            __atomic_load(&p->vals[base + j], &x, __ATOMIC_RELAXED);
            const double y = c_mul * x + c_add;
            __atomic_store(&p->vals[base + j], &y, __ATOMIC_RELAXED);
            if (count) __atomic_fetch_add(&p->hits, 1, __ATOMIC_RELAXED);
            return 1;
        }
    }
    const double y = c_mul * p->tau_min + c_add;
    uint32_t t;
    __atomic_load(&p->tail[u], &t, __ATOMIC_RELAXED);
    t = (t + 1) % p->s; /* always in range, even under races */
    __atomic_store(&p->ids[base + t], &v, __ATOMIC_RELAXED);
    __atomic_store(&p->vals[base + t], &y, __ATOMIC_RELAXED);
    __atomic_store(&p->tail[u], &t, __ATOMIC_RELAXED);
    if (count) __atomic_fetch_add(&p->misses, 1, __ATOMIC_RELAXED);
    return 0;
}
int orc_spm_update_record(orc_spm *p, uint32_t u, uint32_t v, double c_mul, double c_add) {
    return spm_update(p, u, v, c_mul, c_add, 1);
}

void orc_spm_dump(const orc_spm *p, uint32_t *ids, double *vals, uint32_t *tail) {
    if (ids) memcpy(ids, p->ids, sizeof(uint32_t) * (size_t)p->n * p->s);
    if (vals) memcpy(vals, p->vals, sizeof(double) * (size_t)p->n * p->s);
    if (tail) memcpy(tail, p->tail, sizeof(uint32_t) * p->n);
}
void orc_spm_counts(const orc_spm *p, uint64_t *hits, uint64_t *misses) {
    *hits = p->hits; *misses = p->misses;
}

uint64_t orc_fnv1a64(const void *data, uint64_t len) {
    const unsigned char *b = (const unsigned char *)data;
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < len; ++i) { h ^= b[i]; h *= 0x100000001b3ull; }
    return h;
}

/* ========================= engine ========================= */

typedef struct {
    uint32_t n, L, m;
    int type;
    const double *xs, *ys;
    int32_t *dist;    /* n*n when n <= 4096 (hpp:31), else NULL */
    uint32_t *cand;   /* n*L */
    double *etab;     /* n*L, eta^beta of candidate edges */
    double beta, q0, tau0;
    double c_l, c_0;  /* local update coefficients (P4) */
    uint32_t k;
    int memory, consistent, atomic_access;
    double *tau;      /* dense n*n */
    orc_spm *spm;
} eng;

typedef struct {
    uint32_t *route;  /* n */
    uint8_t *vis;     /* n */
    uint32_t cur, start, step;
    orc_rng rng;
    uint64_t fallback, greedy, roulette, updates;
    double *buf;      /* L weights */
    uint32_t *fbuf;   /* L filtered ids */
} ant_t;

static inline int32_t eng_dist(const eng *E, uint32_t u, uint32_t v) {
    if (E->dist) return E->dist[(size_t)u * E->n + v];
    return orc_distance(E->type, E->xs, E->ys, u, v);
}

static inline double ld_tau(const eng *E, size_t i) {
    double x;
    if (E->atomic_access) __atomic_load(&E->tau[i], &x, __ATOMIC_RELAXED);
    else x = E->tau[i];
    return x;
}

static inline double read_tau(const eng *E, uint32_t u, uint32_t v) {
    if (E->memory == ORC_SELECTIVE) return spm_read_relaxed(E->spm, u, v);
    return ld_tau(E, (size_t)u * E->n + v);
}

/* dense write of one direction: plain / relaxed (lost updates allowed) /
 * CAS loop (CONSISTENT contract) */
static void dense_apply(eng *E, size_t i, double c_mul, double c_add) {
    if (!E->atomic_access) {
        E->tau[i] = c_mul * E->tau[i] + c_add;
        return;
    }
    if (E->consistent) {
        uint64_t *w = (uint64_t *)&E->tau[i];
        uint64_t old = __atomic_load_n(w, __ATOMIC_RELAXED);
        for (;;) {
            double x; memcpy(&x, &old, 8);
            const double y = c_mul * x + c_add;
            uint64_t nw; memcpy(&nw, &y, 8);
            if (__atomic_compare_exchange_n(w, &old, nw, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) break;
        }
        return;
    }
    double x;
    __atomic_load(&E->tau[i], &x, __ATOMIC_RELAXED);
    const double y = c_mul * x + c_add;
    __atomic_store(&E->tau[i], &y, __ATOMIC_RELAXED);
}

/* SPEC.md:128-136 (dense: both directions; selective: record u then v, D4) */
static void local_update(eng *E, uint32_t u, uint32_t v) {
    if (E->memory == ORC_SELECTIVE) {
        spm_update(E->spm, u, v, E->c_l, E->c_0, 1);
        spm_update(E->spm, v, u, E->c_l, E->c_0, 1);
        return;
    }
    dense_apply(E, (size_t)u * E->n + v, E->c_l, E->c_0);
    dense_apply(E, (size_t)v * E->n + u, E->c_l, E->c_0);
}

/* SPEC.md:238-246 + P1 draw protocol */
static uint32_t select_next(const eng *E, ant_t *A) {
    const uint32_t u = A->cur;
    const uint32_t *cl = E->cand + (size_t)u * E->L;
    const double *eb = E->etab + (size_t)u * E->L;
    uint32_t cnt = 0;
    for (uint32_t i = 0; i < E->L; ++i) { /* filter_candidates */
        const uint32_t c = cl[i];
        if (!A->vis[c]) {
            A->fbuf[cnt] = c;
            A->buf[cnt] = read_tau(E, u, c) * eb[i]; /* score, P3 */
            ++cnt;
        }
    }
    if (cnt) {
        const double q = orc_rng_uniform01(&A->rng);
        uint32_t pos;
        if (q <= E->q0) {
            pos = orc_greedy_pick(A->buf, cnt);
            A->greedy++;
        } else {
            const double r = orc_rng_uniform01(&A->rng);
            pos = orc_roulette_pick(A->buf, cnt, r);
            A->roulette++;
        }
        return A->fbuf[pos];
    }
    /* fallback: argmax over all unvisited, ties -> lowest id (no RNG, P1) */
    A->fallback++;
    uint32_t best = E->n;
    double bs = 0.0;
    for (uint32_t v = 0; v < E->n; ++v) {
        if (A->vis[v]) continue;
        const double s = read_tau(E, u, v) * orc_eta_beta(eng_dist(E, u, v), E->beta);
        if (best == E->n || s > bs) { bs = s; best = v; }
    }
    return best;
}

static void ant_begin(const eng *E, ant_t *A, int rng_kind, uint64_t seed, uint64_t it, uint64_t a) {
    memset(A->vis, 0, E->n);
    orc_rng_derive(&A->rng, rng_kind, seed, it, a);
    A->start = (uint32_t)orc_rng_uniform_int(&A->rng, E->n); /* P1.1, D11 */
    A->cur = A->start;
    A->vis[A->start] = 1;
    A->route[0] = A->start;
    A->step = 0;
}

/* one step; returns 1 when the step's edge is due for a local update (D9) */
static int ant_step(const eng *E, ant_t *A, uint32_t *u_out, uint32_t *v_out) {
    const uint32_t u = A->cur;
    const uint32_t v = select_next(E, A);
    A->step++;
    A->route[A->step] = v;
    A->vis[v] = 1;
    A->cur = v;
    *u_out = u; *v_out = v;
    return (A->step % E->k) == 0;
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

static void ant_alloc(ant_t *A, uint32_t n, uint32_t L, uint32_t *route) {
    memset(A, 0, sizeof(*A));
    A->route = route;
    A->vis = (uint8_t *)malloc(n);
    A->buf = (double *)malloc(sizeof(double) * (L ? L : 1));
    A->fbuf = (uint32_t *)malloc(sizeof(uint32_t) * (L ? L : 1));
}
static void ant_free(ant_t *A) { free(A->vis); free(A->buf); free(A->fbuf); }

/* whole tour with immediate updates (SEQ: one ant at a time, RELAXED: concurrent) */
static void construct_whole(eng *E, ant_t *A, int rng_kind, uint64_t seed, uint64_t it, uint64_t a) {
    ant_begin(E, A, rng_kind, seed, it, a);
    for (uint32_t t = 1; t < E->n; ++t) {
        uint32_t u, v;
        if (ant_step(E, A, &u, &v)) { local_update(E, u, v); A->updates++; }
    }
    if ((E->n % E->k) == 0) { local_update(E, A->cur, A->start); A->updates++; } /* closing edge, D9 */
}

int orc_run(uint32_t n, int type, const double *xs, const double *ys,
            const orc_params *p, orc_report *rep) {
    if (n < 3 || p->m == 0 || p->k == 0 || p->cl == 0 || p->iterations == 0) return -1;
    if (p->memory == ORC_SELECTIVE && p->s == 0) return -1;
    const double t_begin = now_ms();
    eng E;
    memset(&E, 0, sizeof(E));
    E.n = n; E.m = p->m; E.type = type; E.xs = xs; E.ys = ys; E.k = p->k;
    E.memory = p->memory; E.consistent = p->consistent;
    E.atomic_access = (p->mode == ORC_RELAXED);
    E.beta = p->beta;
    E.q0 = p->q0 < 0 ? orc_default_q0(n) : p->q0;
    if (n <= 4096) {
        E.dist = (int32_t *)malloc(sizeof(int32_t) * (size_t)n * n);
        orc_distance_table(n, type, xs, ys, E.dist);
    }
    E.L = p->cl < n - 1 ? p->cl : n - 1;
    E.cand = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n * E.L);
    orc_build_candidates(n, type, xs, ys, p->cl, E.cand);
    E.etab = (double *)malloc(sizeof(double) * (size_t)n * E.L);
    for (size_t i = 0; i < (size_t)n * E.L; ++i)
        E.etab[i] = orc_eta_beta(eng_dist(&E, (uint32_t)(i / E.L), E.cand[i]), E.beta);
    const int64_t nn = orc_nn_tour_length(n, type, xs, ys, 0);
    E.tau0 = orc_tau0(n, nn);
    E.c_l = 1.0 - p->rho;
    E.c_0 = p->rho * E.tau0;
    const double c_g = 1.0 - p->alpha;
    if (p->memory == ORC_SELECTIVE) {
        E.spm = orc_spm_new(n, p->s, E.tau0); /* tau_min = tau0, D2 */
    } else {
        E.tau = (double *)malloc(sizeof(double) * (size_t)n * n);
        for (size_t i = 0; i < (size_t)n * n; ++i) E.tau[i] = E.tau0;
    }

    const uint32_t m = p->m;
    uint32_t *routes = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)m * n);
    int64_t *lens = (int64_t *)malloc(sizeof(int64_t) * m);
    uint32_t *gb = (uint32_t *)malloc(sizeof(uint32_t) * n);
    int64_t gb_len = INT64_MAX;
    uint64_t updates = 0, fallback = 0, greedy = 0, roulette = 0;

    int threads = p->threads > 0 ? p->threads : 1;
#ifndef _OPENMP
    threads = 1;
#endif
    /* SEQ / SYNC keep one ant state per ant; RELAXED one per thread */
    const uint32_t n_states = (p->mode == ORC_SYNC) ? m : (p->mode == ORC_RELAXED ? (uint32_t)threads : 1);
    ant_t *ants = (ant_t *)malloc(sizeof(ant_t) * n_states);
    for (uint32_t i = 0; i < n_states; ++i) ant_alloc(&ants[i], n, E.L, routes);
    uint32_t *su = (uint32_t *)malloc(sizeof(uint32_t) * m);
    uint32_t *sv = (uint32_t *)malloc(sizeof(uint32_t) * m);
    uint8_t *sdue = (uint8_t *)malloc(m);

    const double t_loop = now_ms();
    for (uint64_t it = 0; it < p->iterations; ++it) {
        const double t_it = now_ms();
        if (p->mode == ORC_SEQ) { /* ant-major, immediate updates */
            ant_t *A = &ants[0];
            for (uint32_t a = 0; a < m; ++a) {
                A->route = routes + (size_t)a * n;
                construct_whole(&E, A, p->rng, p->seed, it, a);
            }
        } else if (p->mode == ORC_SYNC) {
            for (uint32_t a = 0; a < m; ++a) {
                ants[a].route = routes + (size_t)a * n;
                ant_begin(&E, &ants[a], p->rng, p->seed, it, a);
            }
            for (uint32_t t = 1; t < n; ++t) {
                for (uint32_t a = 0; a < m; ++a) sdue[a] = (uint8_t)ant_step(&E, &ants[a], &su[a], &sv[a]);
                for (uint32_t a = 0; a < m; ++a)
                    if (sdue[a]) { local_update(&E, su[a], sv[a]); ants[a].updates++; }
            }
            if ((n % E.k) == 0) /* closing edges in a separate pass, PAPER Alg.1 l.13-14 */
                for (uint32_t a = 0; a < m; ++a) { local_update(&E, ants[a].cur, ants[a].start); ants[a].updates++; }
        } else { /* RELAXED: task per ant */
            #pragma omp parallel num_threads(threads)
            {
                int tid = 0;
#ifdef _OPENMP
                tid = omp_get_thread_num();
#endif
                ant_t *A = &ants[tid];
                #pragma omp for schedule(dynamic, 1)
                for (int64_t a = 0; a < (int64_t)m; ++a) {
                    A->route = routes + (size_t)a * n;
                    construct_whole(&E, A, p->rng, p->seed, it, (uint64_t)a);
                }
            }
        }
        /* eval + select_best (ties lowest ant) + strict is_better */
        #pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t a = 0; a < (int64_t)m; ++a)
            lens[a] = orc_tour_length(type, xs, ys, routes + (size_t)a * n, n);
        const uint32_t ib = orc_select_best(lens, m);
        if (lens[ib] < gb_len) {
            gb_len = lens[ib];
            memcpy(gb, routes + (size_t)ib * n, sizeof(uint32_t) * n);
        }
        /* global update on the global-best edges only (D3), tour order */
        const double c_d = p->alpha * (1.0 / (double)gb_len);
        for (uint32_t i = 0; i < n; ++i) {
            const uint32_t a = gb[i], b = gb[(i + 1) % n];
            if (E.memory == ORC_SELECTIVE) {
                spm_update(E.spm, a, b, c_g, c_d, 1);
                spm_update(E.spm, b, a, c_g, c_d, 1);
            } else {
                E.tau[(size_t)a * n + b] = c_g * E.tau[(size_t)a * n + b] + c_d;
                E.tau[(size_t)b * n + a] = c_g * E.tau[(size_t)b * n + a] + c_d;
            }
        }
        if (rep->trace) rep->trace[it] = gb_len;
        if (rep->iter_best_len) rep->iter_best_len[it] = lens[ib];
        if (rep->iter_best_ant) rep->iter_best_ant[it] = ib;
        if (rep->iter_ms) rep->iter_ms[it] = now_ms() - t_it;
    }
    rep->loop_ms = now_ms() - t_loop;
    for (uint32_t i = 0; i < n_states; ++i) {
        updates += ants[i].updates; fallback += ants[i].fallback;
        greedy += ants[i].greedy; roulette += ants[i].roulette;
        ant_free(&ants[i]);
    }

    rep->best_len = gb_len;
    if (rep->best_tour) memcpy(rep->best_tour, gb, sizeof(uint32_t) * n);
    if (rep->routes) memcpy(rep->routes, routes, sizeof(uint32_t) * (size_t)m * n);
    if (rep->lengths) memcpy(rep->lengths, lens, sizeof(int64_t) * m);
    if (rep->tau && E.tau) memcpy(rep->tau, E.tau, sizeof(double) * (size_t)n * n);
    if (E.spm) {
        orc_spm_dump(E.spm, rep->spm_ids, rep->spm_vals, rep->spm_tail);
        rep->hits = E.spm->hits;
        rep->misses = E.spm->misses;
    } else {
        rep->hits = rep->misses = 0;
    }
    rep->local_updates = updates;
    rep->fallback_steps = fallback;
    rep->greedy_steps = greedy;
    rep->roulette_steps = roulette;
    rep->tau0 = E.tau0;
    rep->nn_len = nn;
    rep->elapsed_ms = now_ms() - t_begin;

    free(ants); free(su); free(sv); free(sdue);
    free(routes); free(lens); free(gb);
    free(E.dist); free(E.cand); free(E.etab); free(E.tau);
    orc_spm_free(E.spm);
    return 0;
}
