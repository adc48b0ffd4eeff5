/*
 * oracle.c -- plain single-threaded CPU oracle for Pipette (arXiv 2405.18093).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Nothing here is blocked, fused or
 * incremental: every proposal of the simulated annealing is re-evaluated from the
 * definition.  Citations: "P:n" = /root/reference/PAPER.md line n; "Rk" = reading k
 * in DESIGN.md section 2 (where the paper is silent, ambiguous or garbled).
 *
 * Build: gcc -O2 -std=c99 -ffp-contract=off -fno-fast-math -fPIC -shared
 * (binary64 on SSE2, no FMA contraction, so every operation below is one IEEE op).
 *
 * Parity status: every function is pinned by a -m "not gpu" test in
 * tests/test_oracle_*.py (worked examples, closed forms, DES, brute force, KATs);
 * see DESIGN.md section 5 for the pin of each function.
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* Enumeration: Alg.1 lines 3-5.  R1: tp | gpus_per_node (TP groups  */
/* stay inside a server); R2: pp <= n_layers; dp must divide bs_global     */
/* (bs_mini = bs_global/dp, l.4); mb ranges over all divisors of bs_mini (l.5).   */
/* Canonical order: pp ascending, tp ascending, mb ascending.                      */
/* ------------------------------------------------------------------------- */
int32_t or_feasible(uint64_t mem, uint64_t cap, int32_t margin_permille) {
  /* Alg.1 l.7 "MemEstimator(Conf, bs_micro) > M_limit then continue"
     with the soft margin of P:370 (R12): runnable iff mem <= floor(cap*(1000-m)/1000). */
  uint64_t limit = cap / 1000u * (uint64_t)(1000 - margin_permille)
                 + (cap % 1000u) * (uint64_t)(1000 - margin_permille) / 1000u;
  return mem <= limit;
}

static int32_t has_profile(const or_profile* prof, int32_t n_prof, int32_t tp, int32_t mb) {
  for (int32_t i = 0; i < n_prof; ++i)
    if (prof[i].tp == tp && prof[i].mb == mb) return 1;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* NEXT-4: the memory estimator MLP of Eq.7, reading     */
/* R23.  Features (Eq.7's order): n_gpus, n_layers, n_hiddens, n_heads, tp, pp, dp,*/
/* bs_micro, bs_mini, bs_global, each as ln(x) by or_log_det, standardised as      */
/* (ln x - mean_i) / std_i; layers 10 -> 200 -> 200 -> 200 -> 200 -> 1 (ReLU        */
/* between); each neuron acc = b_j, then acc = acc + W_ji * in_i for i ascending;  */
/* z = y * y_std + y_mean = ln(M / 1 GB); M = exp(z) GB = exp_det(min(z,16) - 16) *  */
/* fl(e^16) * 1e9 bytes, truncated to an integer.                                 */
/* Parameters, flat: mean[10], std[10], then per layer W (out x in, row-major) and */
/* b[out], then y_std, y_mean (123023 doubles).                                    */
/* ------------------------------------------------------------------------- */
double or_log_det(double x) {   /* ln(x) for x >= 1, only IEEE + - * / on exact parts */
  uint64_t bits;
  memcpy(&bits, &x, sizeof bits);
  int64_t ex = (int64_t)((bits >> 52) & 0x7ff) - 1023;
  uint64_t mb = (bits & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
  double m;
  memcpy(&m, &mb, sizeof m);                    /* x = m * 2^ex, m in [1, 2) exactly */
  double s = (m - 1.0) / (m + 1.0);             /* ln(m) = 2 atanh(s), s in [0, 1/3) */
  double s2 = s * s;
  double p = 1.0 / 31.0;
  for (int k = 14; k >= 0; --k) p = p * s2 + 1.0 / (double)(2 * k + 1);
  double lnm = 2.0 * (s * p);
  double e = (double)ex;
  return (e * 6.93147180369123816490e-01 + lnm) + e * 1.90821492927058770002e-10;
}

#define MLP_H 200
int64_t or_mlp_param_count(void) {
  return 20 + (int64_t)MLP_H * 10 + MLP_H + 3 * ((int64_t)MLP_H * MLP_H + MLP_H) + MLP_H + 1 + 2;
}

uint64_t or_mlp_memory(const double* P, const double feat[10]) {
  double a[MLP_H], b[MLP_H];
  const double* mean = P;
  const double* sd = P + 10;
  const double* w = P + 20;
  double x[10];
  for (int i = 0; i < 10; ++i) x[i] = (or_log_det(feat[i]) - mean[i]) / sd[i];
  const double* in = x;
  int n_in = 10;
  double* bufs[2] = {a, b};
  for (int l = 0; l < 4; ++l) {
    double* out = bufs[l & 1];
    const double* W = w;
    const double* bias = w + (size_t)MLP_H * n_in;
    for (int j = 0; j < MLP_H; ++j) {
      double acc = bias[j];
      for (int i = 0; i < n_in; ++i) acc = acc + W[(size_t)j * n_in + i] * in[i];
      out[j] = acc > 0.0 ? acc : 0.0;
    }
    w = bias + MLP_H;
    in = out;
    n_in = MLP_H;
  }
  double y = w[MLP_H];                                           /* output bias */
  for (int i = 0; i < MLP_H; ++i) y = y + w[i] * in[i];
  const double y_std = w[MLP_H + 1], y_mean = w[MLP_H + 2];
  double z = y * y_std + y_mean;
  if (z > 16.0) z = 16.0;
  double gb = or_exp_det(z - 16.0) * 0x1.0f2ebd0a80020p+23;   /* fl(e^16) */
  double bytes = gb * 1e9;
  return bytes > 0.0 ? (uint64_t)bytes : 0u;
}

static const double* g_mlp = NULL;   /* NULL: analytic estimator (R11) */
void or_set_memory_model(const double* params) { g_mlp = params; }

static uint64_t config_memory(const or_model* m, int64_t G, int64_t bs_global, int32_t pp, int32_t tp, int32_t dp,
                              int32_t mb, int32_t n_mb) {
  if (!g_mlp) return or_memory(m, pp, tp, mb, n_mb);
  double f[10] = {(double)G, (double)m->n_layers, (double)m->hidden, (double)m->heads, (double)tp, (double)pp,
                  (double)dp, (double)mb, (double)(bs_global / dp), (double)bs_global};
  return or_mlp_memory(g_mlp, f);
}

int32_t or_enumerate(const or_cluster* cl, const or_model* m, int64_t bs_global,
                     const or_profile* prof, int32_t n_prof, or_config* out, int32_t cap) {
  int64_t G = (int64_t)cl->n_nodes * cl->gpus_per_node;
  int32_t E = 0;
  for (int64_t pp = 1; pp <= G; ++pp) {
    if (G % pp != 0 || pp > m->n_layers) continue;
    for (int64_t tp = 1; tp <= cl->gpus_per_node; ++tp) {
      if (cl->gpus_per_node % tp != 0) continue;
      if (G % (pp * tp) != 0) continue;
      int64_t dp = G / (pp * tp);
      if (bs_global % dp != 0) continue;
      int64_t bs_mini = bs_global / dp;
      for (int64_t mb = 1; mb <= bs_mini; ++mb) {
        if (bs_mini % mb != 0) continue;
        if (out && E < cap) {
          or_config* c = &out[E];
          c->pp = (int32_t)pp; c->tp = (int32_t)tp; c->dp = (int32_t)dp; c->mb = (int32_t)mb;
          c->n_mb = (int32_t)(bs_mini / mb);
          c->e = E;
          c->mem_bytes = config_memory(m, G, bs_global, c->pp, c->tp, c->dp, c->mb, c->n_mb);
          c->feasible = or_feasible(c->mem_bytes, cl->mem_capacity_bytes, cl->mem_margin_permille);
          c->has_profile = has_profile(prof, n_prof, c->tp, c->mb);
        }
        ++E;
      }
    }
  }
  return E;
}

/* ------------------------------------------------------------------------- */
/* Analytic memory estimator (R11; north_star "parameters, optimizer state, and   */
/* 1F1B in-flight activations per stage"; the paper's heuristic family).   */
/* Stage s is 1-based.  All integers, exact.                                      */
/* ------------------------------------------------------------------------- */
static uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

uint64_t or_stage_memory(const or_model* m, int32_t pp, int32_t tp, int32_t mb, int32_t n_mb, int32_t s) {
  uint64_t L = (uint64_t)m->n_layers, h = (uint64_t)m->hidden, a = (uint64_t)m->heads;
  uint64_t seq = (uint64_t)m->seq_len, V = (uint64_t)m->vocab;
  uint64_t Lps = ceil_div(L, (uint64_t)pp);                       /* layers per stage */
  uint64_t P = Lps * (12u * h * h + 13u * h);                     /* transformer layers */
  if (s == 1) P += V * h + seq * h;                               /* word + position embeddings */
  if (s == pp && pp > 1) P += V * h;                              /* tied LM head copy on last stage */
  uint64_t W = (uint64_t)m->bytes_per_param_state * ceil_div(P, (uint64_t)tp); /* params+grads+Adam */
  /* Korthikanti et al. per-layer activations, TP without SP, no recompute:        */
  /* seq*mb*h*(10 + 24/tp) + 5*a*seq^2*mb/tp bytes.                                  */
  uint64_t act_num = seq * (uint64_t)mb * h * (10u * (uint64_t)tp + 24u)
                   + 5u * a * seq * seq * (uint64_t)mb;
  uint64_t act = ceil_div(act_num, (uint64_t)tp);
  int64_t inflight = (int64_t)pp - s + 1;                         /* 1F1B bound */
  if (inflight > n_mb) inflight = n_mb;
  uint64_t A = (uint64_t)inflight * Lps * act;
  return W + A + m->overhead_bytes;
}

uint64_t or_memory(const or_model* m, int32_t pp, int32_t tp, int32_t mb, int32_t n_mb) {
  uint64_t best = 0;
  for (int32_t s = 1; s <= pp; ++s) {                            /* max over every stage */
    uint64_t v = or_stage_memory(m, pp, tp, mb, n_mb, s);
    if (v > best) best = v;
  }
  return best;
}

/* ------------------------------------------------------------------------- */
/* Per-config constants.  C = per-stage fwd+bwd compute for one   */
/* microbatch = Lps * c_layer (R3); T_TP likewise.                  */
/* msg_PP = mb*seq*h*bpe, msg_DP = floor(n_params/(pp*tp))*bpe (R4).              */
/* ------------------------------------------------------------------------- */
int32_t or_constants(const or_cluster* cl, const or_model* m, const or_config* c,
                     const or_profile* prof, int32_t n_prof, or_consts* K) {
  const or_profile* pe = NULL;
  for (int32_t i = 0; i < n_prof; ++i)
    if (prof[i].tp == c->tp && prof[i].mb == c->mb) { pe = &prof[i]; break; }
  if (!pe) return 3;
  uint64_t L = (uint64_t)m->n_layers, h = (uint64_t)m->hidden;
  uint64_t Lps = ceil_div(L, (uint64_t)c->pp);
  uint64_t msg_pp = (uint64_t)c->mb * (uint64_t)m->seq_len * h * (uint64_t)m->bytes_per_elem;
  uint64_t n_params = 12u * L * h * h + (uint64_t)m->vocab * h;
  uint64_t msg_dp = n_params / ((uint64_t)c->pp * (uint64_t)c->tp) * (uint64_t)m->bytes_per_elem;
  double Lf = (double)Lps;
  K->pp = c->pp; K->dp = c->dp; K->spn = cl->gpus_per_node / c->tp;
  K->N = c->pp * c->dp; K->n_nodes = cl->n_nodes; K->n_mb = c->n_mb;
  K->S  = (Lf * pe->c_layer_s) + (Lf * pe->tp_layer_s);         /* C + T_TP */
  K->m2 = 2.0 * (double)msg_pp;                                  /* Eq.5 "2*msg_PP" */
  K->md = (double)msg_dp;
  K->r  = (double)c->n_mb / (double)c->pp;                       /* n_mb/pp, real (R7) */
  K->Sb = (double)c->pp * K->S;                                  /* pp*(C+T_TP), Eq.4 */
  K->Ss = (double)(c->pp - 1) * K->S;                            /* (pp-1)*(C+T_TP), Eq.4 */
  return 0;
}

/* Eq.6 intra-node factor 4(|W|-1)msg/|W| and inter-node factor 2(|W|-1)msg/|W|. */
double or_qi(const or_consts* K, int32_t c) { return ((4.0 * (double)(c - 1)) * K->md) / (double)c; }
double or_qe(const or_consts* K, int32_t k) { return ((2.0 * (double)(k - 1)) * K->md) / (double)k; }

/* R = 1/B elementwise (R5: node-granular directed matrix, diagonal = intra-node). */
void or_inverse_bandwidth(const double* B, int32_t n, double* R) {
  for (int32_t i = 0; i < n * n; ++i) R[i] = 1.0 / B[i];
}

int32_t or_is_permutation(const uint16_t* perm, int32_t N) {
  char* seen = (char*)calloc((size_t)N + 1, 1);
  int32_t ok = 1;
  for (int32_t w = 0; w < N; ++w) {
    if (perm[w] >= N || seen[perm[w]]) { ok = 0; break; }
    seen[perm[w]] = 1;
  }
  free(seen);
  return ok;
}

/* ------------------------------------------------------------------------- */
/* Latency of a mapping, Eq.3-6, from the definition.                 */
/* Worker position w = z*pp + x (R9: pipeline-major string); slot perm[w] is a    */
/* TP block of tp GPUs inside node perm[w]/spn (R8, Eq.2).              */
/*   T_PP = max_z sum_{x<pp-1} m2 * R[node(z,x)][node(z,x+1)]       Eq.5  */
/*   T_DP = max_n qi(c_n) R[n][n] + qe(k) max_{a!=b in N1} R[a][b]  Eq.6  */
/*   T    = (pp*S + T_PP) * n_mb/pp + (pp-1)*S + T_DP               Eq.3-4, R6    */
/* ------------------------------------------------------------------------- */
double or_latency(const or_consts* K, const double* R, const uint16_t* perm, or_breakdown* bd) {
  const int32_t pp = K->pp, dp = K->dp, n = K->n_nodes, spn = K->spn;
  /* Eq.5: sum along each pipeline in stage order, then the slowest pipeline. */
  double t_pp = 0.0;
  for (int32_t z = 0; z < dp; ++z) {
    double Pz = 0.0;
    for (int32_t x = 0; x + 1 < pp; ++x) {
      int32_t a = perm[z * pp + x] / spn;
      int32_t b = perm[z * pp + x + 1] / spn;
      Pz = Pz + K->m2 * R[a * n + b];
    }
    if (Pz > t_pp) t_pp = Pz;
  }
  /* Eq.6, stage 1 only: occupancy of each node by stage-1 DP members. */
  int32_t* cnt = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  for (int32_t z = 0; z < dp; ++z) cnt[perm[z * pp] / spn] += 1;
  int32_t k = 0;
  double t_in = 0.0;
  for (int32_t a = 0; a < n; ++a) {
    if (cnt[a] > 0) ++k;
    if (cnt[a] >= 2) {                                  /* R10: per-node intra ring */
      double v = or_qi(K, cnt[a]) * R[a * n + a];
      if (v > t_in) t_in = v;
    }
  }
  double t_ex = 0.0;
  if (k >= 2) {                                         /* slowest link over all pairs (R10) */
    double maxR = 0.0;
    for (int32_t a = 0; a < n; ++a)
      for (int32_t b = 0; b < n; ++b)
        if (a != b && cnt[a] > 0 && cnt[b] > 0 && R[a * n + b] > maxR) maxR = R[a * n + b];
    t_ex = or_qe(K, k) * maxR;
  }
  free(cnt);
  double t_dp = t_in + t_ex;
  double T = (((K->Sb + t_pp) * K->r) + K->Ss) + t_dp;
  if (bd) {
    bd->T = T; bd->t_pp = t_pp; bd->t_in = t_in; bd->t_ex = t_ex; bd->t_dp = t_dp;
    bd->t_bubble = K->Sb + t_pp; bd->t_straggler = K->Ss; bd->k = k;
  }
  return T;
}

/* ------------------------------------------------------------------------- */
/* NEXT-2: the prior-work closed form Eq.1 and a       */
/* discrete-event simulation of the memory-efficient 1F1B schedule (P:107-111,   */
/* Fig.2b; the "hidden critical paths" of P:269-271), reading R22.     */
/*                                                                                */
/* or_des_1f1b: one pipeline of pp stages and n_mb microbatches.  Stage s         */
/* (0-based) runs Megatron's 1F1B op order: w = min(pp-s-1, n_mb) warm-up         */
/* forwards, then one forward / one backward until its forwards are exhausted,    */
/* then the remaining w backwards.  F(s,m) may start when F(s-1,m) has ended plus */
/* hop_f[s-1] (s-1 -> s); B(s,m) when B(s+1,m) has ended plus hop_b[s] (s+1 -> s);*/
/* B(pp-1,m) after F(pp-1,m).  A stage runs one op at a time, in its order;       */
/* start = max(stage free, dependency ready), end = start + f (or b).  Plain      */
/* event loop: every stage advances while its next op's dependency has ended.     */
/* Returns the makespan (the last end).                                           */
/* ------------------------------------------------------------------------- */
static void des_op(int32_t pp, int32_t n_mb, int32_t s, int32_t k, int32_t* is_f, int32_t* m) {
  int32_t w = pp - s - 1 < n_mb ? pp - s - 1 : n_mb;
  if (k < w) { *is_f = 1; *m = k; }
  else if (k < 2 * n_mb - w) { int32_t j = k - w; *is_f = (j % 2) == 0; *m = (j % 2) == 0 ? w + j / 2 : j / 2; }
  else { *is_f = 0; *m = k - n_mb; }
}

double or_des_1f1b(int32_t pp, int32_t n_mb, double f, double b, const double* hop_f, const double* hop_b) {
  double* fend = (double*)malloc(sizeof(double) * (size_t)pp * (size_t)n_mb);
  double* bend = (double*)malloc(sizeof(double) * (size_t)pp * (size_t)n_mb);
  char* fdone = (char*)calloc((size_t)pp * (size_t)n_mb, 1);
  char* bdone = (char*)calloc((size_t)pp * (size_t)n_mb, 1);
  int32_t* ptr = (int32_t*)calloc((size_t)pp, sizeof(int32_t));
  double* freet = (double*)calloc((size_t)pp, sizeof(double));
  int64_t remaining = 2 * (int64_t)pp * n_mb;
  double makespan = 0.0;
  while (remaining > 0) {
    int progressed = 0;
    for (int32_t s = 0; s < pp; ++s) {
      while (ptr[s] < 2 * n_mb) {
        int32_t is_f, m;
        des_op(pp, n_mb, s, ptr[s], &is_f, &m);
        double dep = 0.0, dur;
        if (is_f) {
          if (s > 0) {
            if (!fdone[(s - 1) * n_mb + m]) break;
            dep = fend[(s - 1) * n_mb + m] + hop_f[s - 1];
          }
          dur = f;
        } else {
          if (s < pp - 1) {
            if (!bdone[(s + 1) * n_mb + m]) break;
            dep = bend[(s + 1) * n_mb + m] + hop_b[s];
          } else {
            dep = fend[s * n_mb + m];
          }
          dur = b;
        }
        double start = freet[s] > dep ? freet[s] : dep;
        double end = start + dur;
        if (is_f) { fend[s * n_mb + m] = end; fdone[s * n_mb + m] = 1; }
        else      { bend[s * n_mb + m] = end; bdone[s * n_mb + m] = 1; }
        freet[s] = end;
        if (end > makespan) makespan = end;
        ++ptr[s];
        --remaining;
        progressed = 1;
      }
    }
    if (!progressed) break;   /* cannot happen for the 1F1B order (deadlock-free) */
  }
  free(fend); free(bend); free(fdone); free(bdone); free(ptr); free(freet);
  return makespan;
}

/* The three latency models of one plan (reading R22):
 *   T_Pipette  Eq.3-6 (or_latency);
 *   T_prev     Eq.1 with the same terms: (n_mb-1)(C+T_TP) + pp(C+T_TP) + T_PP + T_DP,
 *              where Eq.5's sum stands for (pp-1) T_com^PP (R6), evaluated as
 *              ((((n_mb-1) * S) + Sb) + T_PP) + (T_in + T_ex);
 *   T_DES      max over the dp pipelines of the 1F1B simulation + (T_in + T_ex), with
 *              per-stage f = S / 3, b = S - f (backward = 2 x forward), one-way hops
 *              msg_PP * R in the direction of the transfer (msg_PP = m2 / 2, exact). */
void or_models(const or_consts* K, const double* R, const uint16_t* perm, double* t_pipette, double* t_prev,
               double* t_des) {
  or_breakdown bd;
  *t_pipette = or_latency(K, R, perm, &bd);
  *t_prev = ((((double)(K->n_mb - 1) * K->S) + K->Sb) + bd.t_pp) + bd.t_dp;
  const int32_t pp = K->pp, n = K->n_nodes, spn = K->spn;
  const double f = K->S / 3.0, b = K->S - f, half = K->m2 * 0.5;
  double* hf = (double*)malloc(sizeof(double) * (size_t)(pp > 1 ? pp - 1 : 1));
  double* hb = (double*)malloc(sizeof(double) * (size_t)(pp > 1 ? pp - 1 : 1));
  double mk = 0.0;
  for (int32_t z = 0; z < K->dp; ++z) {
    for (int32_t x = 0; x + 1 < pp; ++x) {
      int32_t a = perm[z * pp + x] / spn, c = perm[z * pp + x + 1] / spn;
      hf[x] = half * R[a * n + c];
      hb[x] = half * R[c * n + a];
    }
    double v = or_des_1f1b(pp, K->n_mb, f, b, hf, hb);
    if (v > mk) mk = v;
  }
  free(hf); free(hb);
  *t_des = mk + bd.t_dp;
}

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon et al. SC'11), R14: counter (step, chain, cfg, 0),       */
/* key (seed lo32, seed hi32).  Round = Random123 / cuRAND definition.            */
/* ------------------------------------------------------------------------- */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* One SA proposal's randomness (R14): positions p != q in [0,N) by 64-bit          */
/* multiply-high, and a 53-bit uniform u in [0,1).                                   */
void or_draw(uint32_t i, uint32_t c, uint32_t e, uint64_t seed, int32_t N,
             uint32_t* p, uint32_t* q, double* u) {
  uint32_t ctr[4] = {i, c, e, 0u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t w[4];
  or_philox4x32_10(ctr, key, w);
  uint32_t pp_ = (uint32_t)(((uint64_t)w[0] * (uint64_t)N) >> 32);
  uint32_t off = (uint32_t)(((uint64_t)w[1] * (uint64_t)(N - 1)) >> 32);
  *p = pp_;
  *q = (pp_ + 1u + off) % (uint32_t)N;
  uint64_t bits = ((uint64_t)(w[2] >> 5) << 26) | (uint64_t)(w[3] >> 6);
  *u = (double)bits * 0x1p-53;
}

/* ------------------------------------------------------------------------- */
/* exp(x) for x <= 0 with only IEEE + - * and floor (R15), so that the Metropolis  */
/* decision is reproducible on any IEEE machine.  Cody-Waite reduction by ln 2,    */
/* degree-13 Taylor polynomial of e^r on |r| <= ln2/2, exact scaling by 2^k.       */
/* ------------------------------------------------------------------------- */
double or_exp_det(double x) {
  if (x < -708.0) return 0.0;
  double k = floor(x * 1.4426950408889634 + 0.5);
  double r = (x - k * 6.93147180369123816490e-01) - k * 1.90821492927058770002e-10;
  double fact = 1.0;
  double coef[14];
  for (int n = 0; n <= 13; ++n) {               /* coef[n] = fl(1/n!) ; n! exact for n<=13 */
    if (n > 0) fact = fact * (double)n;
    coef[n] = 1.0 / fact;
  }
  double poly = coef[13];
  for (int n = 12; n >= 0; --n) poly = poly * r + coef[n];
  int64_t ki = (int64_t)k;                      /* k in [-1022, 0] */
  uint64_t bits = (uint64_t)(ki + 1023) << 52;
  double scale;
  memcpy(&scale, &bits, sizeof scale);
  return poly * scale;
}

/* ------------------------------------------------------------------------- */
/* One simulated-annealing chain of worker dedication (Alg.1 l.9-15).  */
/* Swap move only (north_star); Metropolis acceptance (R13); beta <- beta/alpha    */
/* every iteration (R13); pi0 = identity "alphabetical" (R16); best updated */
/* on strict < (R17).  Every proposal is re-evaluated from the definition.         */
/* ------------------------------------------------------------------------- */
/* ------------------------------------------------------------------------- */
/* The three SA movements of P:252 ("Regarding f as a string, ... migration      */
/* (remove a single element to a random position), swap (exchange two elements),  */
/* and reverse (take a substring and reverse its order)"), reading R21: the move  */
/* kind comes from the 11 bits of the step's Philox block that u leaves unused,   */
/* t = ((w2 & 31) << 6) | (w3 & 63) in [0, 2048): swap if t < 2048 - wm - wr,     */
/* migrate if t < 2048 - wr, else reverse (weights wm, wr in 1/2048 units).       */
/* (p, q) are the draw's two distinct positions.                                  */
/*   swap:    exchange positions p and q                                          */
/*   migrate: remove the element at p and insert it at index q of the remaining   */
/*            string (element 0 to position 2 of abcd gives bcad)     */
/*   reverse: reverse positions min(p,q)..max(p,q) inclusive                      */
/* ------------------------------------------------------------------------- */
void or_draw_move(uint32_t i, uint32_t c, uint32_t e, uint64_t seed, int32_t N,
                  uint32_t* p, uint32_t* q, double* u, uint32_t* t) {
  uint32_t ctr[4] = {i, c, e, 0u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t w[4];
  or_philox4x32_10(ctr, key, w);
  or_draw(i, c, e, seed, N, p, q, u);
  *t = ((w[2] & 31u) << 6) | (w[3] & 63u);
}

int32_t or_move_kind(uint32_t t, int32_t w_migrate, int32_t w_reverse) {
  if ((int32_t)t < 2048 - w_migrate - w_reverse) return 0;   /* swap */
  if ((int32_t)t < 2048 - w_reverse) return 1;               /* migrate */
  return 2;                                                  /* reverse */
}

void or_apply_move(uint16_t* perm, int32_t kind, uint32_t p, uint32_t q) {
  if (kind == 0) {
    uint16_t t = perm[p]; perm[p] = perm[q]; perm[q] = t;
  } else if (kind == 1) {
    uint16_t x = perm[p];
    if (p < q) { for (uint32_t w = p; w < q; ++w) perm[w] = perm[w + 1]; }
    else       { for (uint32_t w = p; w > q; --w) perm[w] = perm[w - 1]; }
    perm[q] = x;
  } else {
    uint32_t lo = p < q ? p : q, hi = p < q ? q : p;
    while (lo < hi) { uint16_t t = perm[lo]; perm[lo] = perm[hi]; perm[hi] = t; ++lo; --hi; }
  }
}

/* The inverse move: swap and reverse are involutions; migrating p -> q is undone by q -> p. */
void or_undo_move(uint16_t* perm, int32_t kind, uint32_t p, uint32_t q) {
  if (kind == 1) or_apply_move(perm, 1, q, p);
  else or_apply_move(perm, kind, p, q);
}

/* ------------------------------------------------------------------------- */
/* Initial temperature by self-calibration (reading R24; NEXT-1): the  */
/* paper fixes only alpha.  T0 is chosen "so the median |Delta| of 100     */
/* seeded random moves is accepted with probability 0.8": exp(-median / T0) = 0.8, */
/* i.e. beta0 = 1/T0 = ln(1.25) / median.                                          */
/*   move i = 0..99: the Philox block of counter (i, 0, e, 1) -- fourth word 1, so  */
/*     the stream is disjoint from every SA proposal (fourth word 0) -- drawn and   */
/*     selected exactly like an SA proposal (R14, R21), applied to the identity     */
/*     mapping (the chains' start, R16);                                            */
/*   |Delta_i| = |L(move_i(identity)) - L0|, both from the definition (or_latency); */
/*   median = (s[49] + s[50]) * 0.5 of the |Delta| sorted ascending;                */
/*   beta0 = 0.22314355131420976 / median (the double nearest ln 1.25).            */
/* One value per configuration and seed (independent of the chain).  If median is  */
/* 0 (every move keeps the latency, e.g. pp = 1) or N < 2, beta0 = 1/(tau * L0).    */
/* ------------------------------------------------------------------------- */
void or_draw_ctr(uint32_t i, uint32_t c, uint32_t e, uint32_t d, uint64_t seed, int32_t N,
                 uint32_t* p, uint32_t* q, uint32_t* t) {
  uint32_t ctr[4] = {i, c, e, d};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t w[4];
  or_philox4x32_10(ctr, key, w);
  uint32_t pp_ = (uint32_t)(((uint64_t)w[0] * (uint64_t)N) >> 32);
  uint32_t off = (uint32_t)(((uint64_t)w[1] * (uint64_t)(N - 1)) >> 32);
  *p = pp_;
  *q = (pp_ + 1u + off) % (uint32_t)N;
  *t = ((w[2] & 31u) << 6) | (w[3] & 63u);
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

double or_calibrate_beta(const or_consts* K, const double* R, uint64_t seed, uint32_t e,
                         int32_t w_migrate, int32_t w_reverse, double tau) {
  const int32_t N = K->N;
  uint16_t* perm = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(N > 0 ? N : 1));
  for (int32_t w = 0; w < N; ++w) perm[w] = (uint16_t)w;
  or_breakdown bd;
  const double L0 = or_latency(K, R, perm, &bd);
  double beta = 1.0 / (tau * L0);
  if (N >= 2) {
    double d[100];
    for (int32_t i = 0; i < 100; ++i) {
      uint32_t p, q, t;
      or_draw_ctr((uint32_t)i, 0u, e, 1u, seed, N, &p, &q, &t);
      const int32_t kind = or_move_kind(t, w_migrate, w_reverse);
      for (int32_t w = 0; w < N; ++w) perm[w] = (uint16_t)w;
      or_apply_move(perm, kind, p, q);
      d[i] = fabs(or_latency(K, R, perm, &bd) - L0);
    }
    qsort(d, 100, sizeof(double), cmp_double);
    const double median = (d[49] + d[50]) * 0.5;
    if (median > 0.0) beta = 0.22314355131420976 / median;
  }
  free(perm);
  return beta;
}

/* ------------------------------------------------------------------------- */
/* One SA chain of fine-grained worker dedication (Alg.1 l.9-15) on   */
/* configuration e: Metropolis acceptance (R13, R16), every proposal evaluated   */
/* from scratch by or_latency.  w_migrate = w_reverse = 0 is the swap-only chain. */
/* ------------------------------------------------------------------------- */
void or_sa_chain_moves(const or_consts* K, const double* R, int32_t iterations, uint64_t seed,
                       uint32_t chain, uint32_t e, double alpha, double tau, double t0,
                       int32_t w_migrate, int32_t w_reverse,
                       or_chain_result* res, uint16_t* best_perm,
                       or_trace_record* trace, int32_t trace_cap) {
  const int32_t N = K->N;
  uint16_t* perm = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)N);
  for (int32_t w = 0; w < N; ++w) perm[w] = (uint16_t)w;
  or_breakdown bd;
  double L0 = or_latency(K, R, perm, &bd);
  double cur = L0, best = L0;
  double best_tpp = bd.t_pp, best_tdp = bd.t_dp;
  int32_t best_step = -1;
  uint32_t accepted = 0;
  if (best_perm) memcpy(best_perm, perm, sizeof(uint16_t) * (size_t)N);
  /* R13: beta0 = 1/t0 (t0 > 0), the self-calibration of R24 (t0 < 0), else 1/(tau L0) */
  double beta = (t0 > 0.0) ? 1.0 / t0
              : (t0 < 0.0 ? or_calibrate_beta(K, R, seed, e, w_migrate, w_reverse, tau) : 1.0 / (tau * L0));
  double ia = 1.0 / alpha;
  if (N >= 2) {
    for (int32_t i = 0; i < iterations; ++i) {
      uint32_t p, q, t; double u;
      or_draw_move((uint32_t)i, chain, e, seed, N, &p, &q, &u, &t);
      int32_t kind = or_move_kind(t, w_migrate, w_reverse);
      or_apply_move(perm, kind, p, q);
      double Lp = or_latency(K, R, perm, &bd);
      double d = Lp - cur;
      int acc = (d <= 0.0) || (u < or_exp_det(-(d * beta)));        /* Metropolis */
      if (acc) {
        cur = Lp; ++accepted;
        if (Lp < best) {
          best = Lp; best_step = i; best_tpp = bd.t_pp; best_tdp = bd.t_dp;
          if (best_perm) memcpy(best_perm, perm, sizeof(uint16_t) * (size_t)N);
        }
      } else {
        or_undo_move(perm, kind, p, q);
      }
      beta = beta * ia;
      if (trace && i < trace_cap) {
        trace[i].i = (uint32_t)i; trace[i].p = (uint16_t)p; trace[i].q = (uint16_t)q;
        trace[i].accept = (uint32_t)acc; trace[i].L = Lp;
      }
    }
  }
  res->best = best; res->best_t_pp = best_tpp; res->best_t_dp = best_tdp; res->L0 = L0;
  res->best_step = best_step; res->accepted = accepted;
  free(perm);
}

void or_sa_chain(const or_consts* K, const double* R, int32_t iterations, uint64_t seed,
                 uint32_t chain, uint32_t e, double alpha, double tau, double t0,
                 or_chain_result* res, uint16_t* best_perm,
                 or_trace_record* trace, int32_t trace_cap) {
  or_sa_chain_moves(K, R, iterations, seed, chain, e, alpha, tau, t0, 0, 0, res, best_perm, trace, trace_cap);
}

/* ------------------------------------------------------------------------- */
/* Alg.1: every feasible (Conf, bs_micro) runs `chains` SA chains;     */
/* winner = lexicographic min of (latency, config index e, chain c) (R17).         */
/* `world` simulates the W-rank sharding: item j = f*chains + c belongs to rank    */
/* j mod W; each rank takes its local argmin; the ranks are combined by a min over */
/* the latency bits, then a min over the item ids that attain it (R18).           */
/* ------------------------------------------------------------------------- */
int32_t or_search_moves(const or_cluster* cl, const double* B, const or_profile* prof, int32_t n_prof,
                        const or_model* m, int64_t bs_global, int32_t chains, int32_t iterations,
                        uint64_t seed, double alpha, double tau, double t0, int32_t w_migrate, int32_t w_reverse,
                        int32_t world, or_plan* plan, uint16_t* perm_out, int32_t perm_cap,
                        double* per_config_best, int32_t* per_config_chain) {
  memset(plan, 0, sizeof *plan);
  int32_t n = cl->n_nodes;
  int32_t E = or_enumerate(cl, m, bs_global, prof, n_prof, NULL, 0);
  or_config* cfgs = (or_config*)calloc((size_t)E + 1, sizeof(or_config));
  or_enumerate(cl, m, bs_global, prof, n_prof, cfgs, E);
  double* R = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
  or_inverse_bandwidth(B, n, R);
  int32_t F = 0;
  for (int32_t i = 0; i < E; ++i) {
    if (!cfgs[i].feasible) continue;
    if (!cfgs[i].has_profile) { plan->status = 3; plan->E = E; free(cfgs); free(R); return 3; }
    ++F;
  }
  plan->E = E; plan->F = F;
  if (F == 0) { plan->status = 1; free(cfgs); free(R); return 1; }

  /* per-rank local winners */
  double* rank_best = (double*)malloc(sizeof(double) * (size_t)world);
  int64_t* rank_item = (int64_t*)malloc(sizeof(int64_t) * (size_t)world);
  for (int32_t r = 0; r < world; ++r) { rank_best[r] = INFINITY; rank_item[r] = INT64_MAX; }
  int32_t maxN = 0;
  for (int32_t i = 0; i < E; ++i) if (cfgs[i].feasible && cfgs[i].pp * cfgs[i].dp > maxN) maxN = cfgs[i].pp * cfgs[i].dp;
  uint16_t* bp = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)maxN);
  uint64_t steps = 0, acc = 0;
  int32_t f = 0;
  for (int32_t i = 0; i < E; ++i) {
    if (!cfgs[i].feasible) continue;
    or_consts K;
    or_constants(cl, m, &cfgs[i], prof, n_prof, &K);
    if (per_config_best) per_config_best[f] = INFINITY;
    if (per_config_chain) per_config_chain[f] = -1;
    for (int32_t c = 0; c < chains; ++c) {
      or_chain_result res;
      or_sa_chain_moves(&K, R, iterations, seed, (uint32_t)c, (uint32_t)cfgs[i].e, alpha, tau, t0, w_migrate,
                        w_reverse, &res, NULL, NULL, 0);
      if (K.N >= 2) steps += (uint64_t)iterations;
      acc += res.accepted;
      int64_t j = (int64_t)f * chains + c;
      int32_t r = (int32_t)(j % world);
      if (res.best < rank_best[r] || (res.best == rank_best[r] && j < rank_item[r])) {
        rank_best[r] = res.best; rank_item[r] = j;
      }
      if (per_config_best && (res.best < per_config_best[f])) {
        per_config_best[f] = res.best;
        if (per_config_chain) per_config_chain[f] = c;
      }
    }
    ++f;
  }
  /* combine: min over latency, then min item id among ranks attaining it */
  double gbest = INFINITY;
  for (int32_t r = 0; r < world; ++r) if (rank_best[r] < gbest) gbest = rank_best[r];
  int64_t gitem = INT64_MAX;
  for (int32_t r = 0; r < world; ++r) if (rank_best[r] == gbest && rank_item[r] < gitem) gitem = rank_item[r];
  int32_t wf = (int32_t)(gitem / chains), wc = (int32_t)(gitem % chains);
  /* re-run the winning chain to recover its best mapping and breakdown */
  f = 0;
  for (int32_t i = 0; i < E; ++i) {
    if (!cfgs[i].feasible) continue;
    if (f == wf) {
      or_consts K;
      or_constants(cl, m, &cfgs[i], prof, n_prof, &K);
      or_chain_result res;
      or_sa_chain_moves(&K, R, iterations, seed, (uint32_t)wc, (uint32_t)cfgs[i].e, alpha, tau, t0, w_migrate,
                        w_reverse, &res, bp, NULL, 0);
      plan->cfg = cfgs[i];
      or_latency(&K, R, bp, &plan->bd);
      plan->cfg_index = cfgs[i].e; plan->chain = wc; plan->best_step = res.best_step;
      plan->n_slots = K.N;
      if (perm_out && perm_cap >= K.N) memcpy(perm_out, bp, sizeof(uint16_t) * (size_t)K.N);
      break;
    }
    ++f;
  }
  plan->sa_steps = steps; plan->sa_accepted = acc; plan->status = 0;
  free(bp); free(rank_best); free(rank_item); free(cfgs); free(R);
  return 0;
}

int32_t or_search(const or_cluster* cl, const double* B, const or_profile* prof, int32_t n_prof,
                  const or_model* m, int64_t bs_global, int32_t chains, int32_t iterations,
                  uint64_t seed, double alpha, double tau, double t0, int32_t world,
                  or_plan* plan, uint16_t* perm_out, int32_t perm_cap,
                  double* per_config_best, int32_t* per_config_chain) {
  return or_search_moves(cl, B, prof, n_prof, m, bs_global, chains, iterations, seed, alpha, tau, t0, 0, 0, world,
                         plan, perm_out, perm_cap, per_config_best, per_config_chain);
}
