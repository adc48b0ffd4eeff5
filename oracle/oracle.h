/*
 * oracle.h -- plain, slow, single-threaded CPU oracle for Pipette (arXiv 2405.18093).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call anything under oracle/.
 * The product path (paper_2405_18093_b200/, include/pipette.h) never does, and the
 * two share no code: no headers, helpers, tables or constant generators.
 *
 * Every function cites the passage of /root/reference/PAPER.md ("P:n" = line n) it
 * follows, plus the reading in DESIGN.md ("Rk") where the paper is silent or garbled.
 * Floating point: IEEE-754 binary64, round-to-nearest, built with -ffp-contract=off,
 * every + - * / written in the normative order of DESIGN.md section 3.
 */
#ifndef PIPETTE_ORACLE_H
#define PIPETTE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t n_nodes, gpus_per_node;
  uint64_t mem_capacity_bytes;
  int32_t mem_margin_permille;
} or_cluster;

typedef struct {
  int32_t n_layers, hidden, heads, seq_len, vocab, bytes_per_elem, bytes_per_param_state;
  uint64_t overhead_bytes;
} or_model;

typedef struct {
  int32_t tp, mb;
  double c_layer_s, tp_layer_s;
} or_profile;

/* One enumerated configuration (Alg.1 l.3-5). */
typedef struct {
  int32_t pp, tp, dp, mb, n_mb, e;
  uint64_t mem_bytes;   /* max over stages of the analytic per-GPU memory (R11) */
  int32_t feasible;     /* mem_bytes <= floor(cap*(1000-margin)/1000) (Alg.1 l.7) */
  int32_t has_profile;  /* (tp, mb) present in the profile table */
} or_config;

/* Per-config model constants. */
typedef struct {
  int32_t pp, dp, spn, N, n_nodes, n_mb;
  double S, m2, md, r, Sb, Ss;
} or_consts;

typedef struct {
  double T, t_pp, t_in, t_ex, t_dp, t_bubble, t_straggler;
  int32_t k;
} or_breakdown;

typedef struct {
  double best, best_t_pp, best_t_dp, L0;
  int32_t best_step;
  uint32_t accepted;
} or_chain_result;

typedef struct {
  uint32_t i;
  uint16_t p, q;
  uint32_t accept;
  double L;   /* latency of the proposal */
} or_trace_record;

typedef struct {
  int32_t status;          /* 0 ok, 1 no feasible, 2 invalid, 3 profile missing */
  int32_t E, F;
  or_config cfg;
  or_breakdown bd;
  int32_t cfg_index, chain, best_step, n_slots;
  uint64_t sa_steps, sa_accepted;
} or_plan;

/* --- enumeration and memory ----------------------------------------------- */
int32_t or_enumerate(const or_cluster* cl, const or_model* m, int64_t bs_global,
                     const or_profile* prof, int32_t n_prof, or_config* out, int32_t cap);
uint64_t or_stage_memory(const or_model* m, int32_t pp, int32_t tp, int32_t mb, int32_t n_mb, int32_t s);
uint64_t or_memory(const or_model* m, int32_t pp, int32_t tp, int32_t mb, int32_t n_mb);
int32_t  or_feasible(uint64_t mem, uint64_t cap, int32_t margin_permille);

/* --- constants and latency ------------------------------------------------ */
int32_t or_constants(const or_cluster* cl, const or_model* m, const or_config* c,
                     const or_profile* prof, int32_t n_prof, or_consts* out);
double or_qi(const or_consts* K, int32_t c);
double or_qe(const or_consts* K, int32_t k);
void   or_inverse_bandwidth(const double* B, int32_t n, double* R);
double or_latency(const or_consts* K, const double* R, const uint16_t* perm, or_breakdown* bd);
int32_t or_is_permutation(const uint16_t* perm, int32_t N);

/* --- randomness ------------------------------------------------------------ */
void   or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double or_exp_det(double x);
void   or_draw(uint32_t i, uint32_t c, uint32_t e, uint64_t seed, int32_t N,
               uint32_t* p, uint32_t* q, double* u);

/* --- simulated annealing and search --------------------------------------- */
void or_sa_chain(const or_consts* K, const double* R, int32_t iterations, uint64_t seed,
                 uint32_t chain, uint32_t e, double alpha, double tau, double t0,
                 or_chain_result* res, uint16_t* best_perm,
                 or_trace_record* trace, int32_t trace_cap);

/* NEXT-4: Eq.7's memory MLP, reading R23; or_set_memory_model(NULL)
 * restores the analytic estimator for or_enumerate (process-global, test use only). */
double or_log_det(double x);
int64_t or_mlp_param_count(void);
uint64_t or_mlp_memory(const double* params, const double feat[10]);
void or_set_memory_model(const double* params);

/* NEXT-2: Eq.1 and a 1F1B discrete-event simulation, reading R22. */
double or_des_1f1b(int32_t pp, int32_t n_mb, double f, double b, const double* hop_f, const double* hop_b);
void or_models(const or_consts* K, const double* R, const uint16_t* perm, double* t_pipette, double* t_prev,
               double* t_des);

/* NEXT-1: the paper's three SA movements, reading R21. */
/* R24: one Philox draw of counter (i, c, e, d) as (p, q, t), and the
 * calibrated inverse initial temperature of configuration e: ln(1.25) / median |Delta| of
 * 100 seeded moves of the identity mapping (fallback 1/(tau L0)).  or_sa_chain[_moves]
 * use it when t0 < 0. */
void or_draw_ctr(uint32_t i, uint32_t c, uint32_t e, uint32_t d, uint64_t seed, int32_t N,
                 uint32_t* p, uint32_t* q, uint32_t* t);
double or_calibrate_beta(const or_consts* K, const double* R, uint64_t seed, uint32_t e,
                         int32_t w_migrate, int32_t w_reverse, double tau);
void or_draw_move(uint32_t i, uint32_t c, uint32_t e, uint64_t seed, int32_t N,
                  uint32_t* p, uint32_t* q, double* u, uint32_t* t);
int32_t or_move_kind(uint32_t t, int32_t w_migrate, int32_t w_reverse);   /* 0 swap, 1 migrate, 2 reverse */
void or_apply_move(uint16_t* perm, int32_t kind, uint32_t p, uint32_t q);
void or_undo_move(uint16_t* perm, int32_t kind, uint32_t p, uint32_t q);
void or_sa_chain_moves(const or_consts* K, const double* R, int32_t iterations, uint64_t seed,
                       uint32_t chain, uint32_t e, double alpha, double tau, double t0,
                       int32_t w_migrate, int32_t w_reverse,
                       or_chain_result* res, uint16_t* best_perm,
                       or_trace_record* trace, int32_t trace_cap);
int32_t or_search_moves(const or_cluster* cl, const double* B, const or_profile* prof, int32_t n_prof,
                        const or_model* m, int64_t bs_global, int32_t chains, int32_t iterations,
                        uint64_t seed, double alpha, double tau, double t0, int32_t w_migrate, int32_t w_reverse,
                        int32_t world, or_plan* plan, uint16_t* perm_out, int32_t perm_cap,
                        double* per_config_best, int32_t* per_config_chain);

int32_t or_search(const or_cluster* cl, const double* B, const or_profile* prof, int32_t n_prof,
                  const or_model* m, int64_t bs_global, int32_t chains, int32_t iterations,
                  uint64_t seed, double alpha, double tau, double t0, int32_t world,
                  or_plan* plan, uint16_t* perm_out, int32_t perm_cap,
                  double* per_config_best /* F entries or NULL */,
                  int32_t* per_config_chain /* F entries or NULL */);

#ifdef __cplusplus
}
#endif
#endif
