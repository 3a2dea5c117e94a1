/*
 * oracle/acs_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference path of arXiv 1605.02669 (Ant Colony
 * System for the symmetric TSP) used as the parity checker for the sm_100a
 * product in paper_1605_02669_b200/. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product never links, loads or calls it.
 *
 * What is pinned by reference CODE (bit-exact against oracle/_ref, which is
 * compiled from /root/reference/proj/src/tsp_instance.cpp and
 * /root/reference/proj/include/acs/rng.hpp -- see oracle/Makefile):
 *   distance, distance table, candidate lists, nn_tour_length, tour_length,
 *   RngStream (xoshiro256** / splitmix64 derive, uniform01, uniform_int).
 * What is pinned by reference SPEC known-answer tests only
 * (/root/reference/SPEC.md op examples + acceptance criteria):
 *   pheromone stores, construction, engine.  At the tour level the reference
 *   ships no code and no test, so tour parity is anchored on this
 *   restatement + the SPEC KATs ("parity unpinned at tour level by reference
 *   code").
 */
#ifndef ACS_ORACLE_H
#define ACS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_EUC_2D = 0, ORC_CEIL_2D = 1, ORC_ATT = 2 };
enum { ORC_SEQ = 0, ORC_SYNC = 1, ORC_RELAXED = 2 };
enum { ORC_DENSE = 0, ORC_SELECTIVE = 1 };
enum { ORC_RNG_XOSHIRO = 0, ORC_RNG_PHILOX = 1 };

/* ---- instance (tsp_instance.cpp:49-65, 67-78, 219-252, 254-280) ---- */
int32_t orc_distance(int type, const double *xs, const double *ys, uint32_t u, uint32_t v);
void orc_distance_table(uint32_t n, int type, const double *xs, const double *ys, int32_t *out);
uint32_t orc_build_candidates(uint32_t n, int type, const double *xs, const double *ys,
                              uint32_t cl, uint32_t *out /* n * min(cl,n-1) */);
int64_t orc_nn_tour_length(uint32_t n, int type, const double *xs, const double *ys, uint32_t start);
int64_t orc_tour_length(int type, const double *xs, const double *ys,
                        const uint32_t *order, uint32_t len);

/* ---- rng (rng.hpp:16-84; Philox4x32-10 per Salmon et al. SC'11) ---- */
typedef struct {
    int32_t kind;
    uint32_t key[2];     /* philox key = seed */
    uint32_t ctr_hi[3];  /* philox counter words 1..3 = ant, iter lo, iter hi */
    uint32_t draw;       /* philox counter word 0 */
    uint64_t s[4];       /* xoshiro state */
} orc_rng;

void orc_rng_seed(orc_rng *r, uint64_t seed); /* RngStream(seed), xoshiro */
void orc_rng_derive(orc_rng *r, int kind, uint64_t seed, uint64_t iteration, uint64_t ant);
uint64_t orc_rng_next_u64(orc_rng *r);
double orc_rng_uniform01(orc_rng *r);
uint64_t orc_rng_uniform_int(orc_rng *r, uint64_t bound);

/* ---- op-level restatements ---- */
double orc_default_q0(uint32_t n);
double orc_tau0(uint32_t n, int64_t nn_len);
double orc_local_update_value(double tau, double rho, double tau0);
double orc_global_update_value(double tau, double alpha, int64_t l_gb);
double orc_eta_beta(int32_t d, double beta);
double orc_score(double tau, double eta, double beta);
uint32_t orc_greedy_pick(const double *scores, uint32_t len);
uint32_t orc_roulette_pick(const double *weights, uint32_t len, double r);
uint32_t orc_select_best(const int64_t *lengths, uint32_t m);

/* selective store, single-threaded (Fig. alg:3) */
typedef struct orc_spm orc_spm;
orc_spm *orc_spm_new(uint32_t n, uint32_t s, double tau_min);
void orc_spm_free(orc_spm *p);
double orc_spm_read(const orc_spm *p, uint32_t u, uint32_t v);
/* rule 0: local (c_l, c_0), rule 1: global (c_g, c_d); returns 1 on hit */
int orc_spm_update_record(orc_spm *p, uint32_t u, uint32_t v, double c_mul, double c_add);
void orc_spm_dump(const orc_spm *p, uint32_t *ids, double *vals, uint32_t *tail);
void orc_spm_counts(const orc_spm *p, uint64_t *hits, uint64_t *misses);

/* FNV-1a-64 over bytes (SURVEY Appendix A golden hashes) */
uint64_t orc_fnv1a64(const void *data, uint64_t len);

/* ---- engine ---- */
typedef struct {
    double beta, alpha, rho, q0; /* q0 < 0 -> default_q0(n) */
    uint32_t cl, m, s, k;
    uint64_t iterations, seed;
    int32_t mode, memory, consistent, rng, threads;
} orc_params;

typedef struct {
    int64_t best_len;
    uint32_t *best_tour;      /* [n] or NULL */
    int64_t *trace;           /* [iterations] L_gb after each iteration, or NULL */
    int64_t *iter_best_len;   /* [iterations] or NULL */
    uint32_t *iter_best_ant;  /* [iterations] or NULL */
    uint32_t *routes;         /* [m*n] routes of the last iteration, or NULL */
    int64_t *lengths;         /* [m] lengths of the last iteration, or NULL */
    double *tau;              /* [n*n] final dense pheromone, or NULL */
    uint32_t *spm_ids;        /* [n*s] final selective ids, or NULL */
    double *spm_vals;         /* [n*s] */
    uint32_t *spm_tail;       /* [n] */
    uint64_t local_updates, hits, misses, fallback_steps, greedy_steps, roulette_steps;
    double tau0;
    int64_t nn_len;
    double elapsed_ms;        /* whole call incl. setup */
    double loop_ms;           /* iteration loop only (construct+eval+best+global) */
    double *iter_ms;          /* [iterations] wall time of each iteration, or NULL */
} orc_report;

int orc_run(uint32_t n, int type, const double *xs, const double *ys,
            const orc_params *p, orc_report *rep);

#ifdef __cplusplus
}
#endif
#endif
