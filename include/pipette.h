/*
 * pipette.h -- C ABI of the B200-native Pipette plan evaluator (arXiv 2405.18093).
 *
 * One shared library, libpipette.so (paper_2405_18093_b200/lib/), built for sm_100a.
 * Citations: "P:n" = line n of the paper's LaTeX source with the section,
 * equation or algorithm named; "Rk" = reading k of DESIGN.md section 2.
 *
 * Conventions for every entry point:
 *   - plain C99, no CUDA or torch types; streams are passed as void* (cudaStream_t);
 *   - functions return pipette_status and never throw or exit; a human-readable
 *     message for the last failure is available from pipette_last_error(ctx);
 *   - one context per device per process; a context is not thread-safe;
 *   - all floating point is IEEE binary64 evaluated in the fixed operation order of
 *     DESIGN.md section 3 (no FMA contraction), so results are bit-identical to the
 *     CPU oracle (oracle/), to which the tests compare them.
 */
#ifndef PIPETTE_H
#define PIPETTE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pipette_ctx pipette_ctx; /* opaque */

typedef enum {
  PIPETTE_OK = 0,
  PIPETTE_NO_FEASIBLE = 1,   /* every configuration fails the memory filter (Alg.1 l.7) */
  PIPETTE_E_INVALID = 2,     /* input validation failed; see pipette_last_error */
  PIPETTE_E_PROFILE = 3,     /* a feasible (tp, mb) has no profile entry (R3) */
  PIPETTE_E_CUDA = 4,        /* a CUDA runtime call failed */
  PIPETTE_E_NCCL = 5,        /* an NCCL call failed */
  PIPETTE_E_UNSUPPORTED = 6  /* outside v1 limits (G > 1024 GPUs, n_nodes > 128, gpus_per_node > 255) */
} pipette_status;

/* Cluster shape (Alg.1 inputs G and M_limit). G = n_nodes * gpus_per_node.
 * mem_margin_permille: the soft margin of P:370 in 1/1000 of capacity (R12), 0..500. */
typedef struct {
  int32_t n_nodes, gpus_per_node;
  uint64_t mem_capacity_bytes;
  int32_t mem_margin_permille;
} pipette_cluster;

/* Profile table entry ("we use the profiled values"): per-layer forward+backward
 * compute c_layer_s (> 0) and per-layer TP all-reduce time tp_layer_s (>= 0), in seconds,
 * for TP degree tp and micro-batch size mb (R3). */
typedef struct {
  int32_t tp, mb;
  double c_layer_s, tp_layer_s;
} pipette_profile_entry;

/* Host transport of the combine (optional, see pipette_dist): allreduce of `count` uint64
 * words in place on a HOST buffer, op 0 = element-wise min, 1 = element-wise sum (mod 2^64);
 * returns 0 on success, anything else fails the search with E_NCCL.  Called on the thread
 * that called pipette_search, three times per search, in the same order on every rank. */
typedef int (*pipette_host_allreduce_fn)(void* user, uint64_t* buf, int64_t count, int32_t op);

/* Multi-GPU description (one process per GPU).  world == 1 needs no NCCL id. For
 * world > 1 either
 *   - nccl_unique_id points to the 128-byte ncclUniqueId produced on rank 0 by
 *     pipette_nccl_unique_id() and broadcast by the caller (e.g. torch.distributed): the
 *     combine's reductions run as ncclAllReduce on the context's stream; or
 *   - nccl_unique_id == NULL and host_allreduce != NULL: the same three reductions (R18)
 *     run through the caller's host collective on D2H-staged buffers (e.g. a gloo process
 *     group, or several ranks sharing one GPU, which NCCL refuses).  Identical results.
 * host_allreduce / host_user may be NULL/unused otherwise. */
typedef struct {
  int32_t rank, world, device;
  const void* nccl_unique_id;
  pipette_host_allreduce_fn host_allreduce;
  void* host_user;
} pipette_dist;

/* GPT-style model shape (Eq.7 inputs; message sizes R4; memory R11).
 * hidden % heads == 0.  bytes_per_elem = 2 (bf16 activations/messages),
 * bytes_per_param_state = 16 (mixed-precision Adam), overhead_bytes added per GPU. */
typedef struct {
  int32_t n_layers, hidden, heads, seq_len, vocab, bytes_per_elem, bytes_per_param_state;
  uint64_t overhead_bytes;
} pipette_model;

/* One candidate configuration (pp, tp, dp, bs_micro), Alg.1 l.3-5. */
typedef struct {
  uint16_t pp, tp, dp, mb;
} pipette_config;

/* One SA proposal of a traced chain: step i, swapped positions p and q, the Metropolis
 * decision, and the proposal's latency (Alg.1 l.11). */
typedef struct {
  uint32_t i;
  uint16_t p, q;
  uint32_t accept;
  double latency;
} pipette_trace_record;

/* Per-chain result (for parity tests and diagnostics). */
typedef struct {
  double best, best_t_pp, best_t_dp, L0;
  int32_t best_step;        /* -1 if the identity mapping was never improved */
  uint32_t accepted;
  int32_t cfg_index;        /* e: index of the config in the full enumeration */
  int32_t chain;            /* c */
  int32_t rank;             /* rank that ran the chain; entries of other ranks are untouched */
  int32_t n_slots;          /* N = pp*dp */
} pipette_chain_result;

/* Simulated-annealing options (R13).  NULL means: alpha = 0.999, tau = 0.05,
 * t0 = 0 (T0 = tau * L(identity)), no diagnostics.  t0 < 0 selects SPEC's self-calibration
 * (reading R24): per feasible configuration, T0 such that the median |Delta| of 100
 * seeded moves of the identity mapping (Philox counter (i, 0, e, 1), i < 100, drawn and
 * selected like SA proposals) is accepted with probability 0.8, i.e. 1/T0 = ln(1.25) /
 * median; a zero median (e.g. pp = 1) falls back to tau * L(identity).  Note the defaults
 * differ from SPEC's CLI defaults: swap moves only (north_star) and T0 = tau * L0;
 * SPEC's behaviour is w_migrate = 683, w_reverse = 682 and t0 < 0.  Diagnostic outputs are HOST buffers
 * owned by the caller; items are numbered j = f*chains_per_config + c (f = index among
 * feasible configs), as in R18. */
typedef struct {
  double alpha;             /* temperature reduction per iteration, (0, 1] */
  double tau;               /* T0 = tau * L(identity) when t0 <= 0 */
  double t0;                /* explicit initial temperature (s) if > 0; < 0: self-calibrated (R24) */
  pipette_chain_result* chains;   /* chains_cap entries indexed by j, or NULL */
  uint16_t* chain_perms;          /* chains_cap x chain_perm_stride best mappings, or NULL */
  int32_t chain_perm_stride;
  int64_t chains_cap;
  const int64_t* trace_items;     /* global item ids j to trace, or NULL */
  int32_t n_trace;
  int32_t trace_cap;              /* records kept per traced item (first trace_cap steps) */
  pipette_trace_record* trace;    /* n_trace x trace_cap records (host) */
  /* The paper's full move set (reading R21): probabilities of the migration
   * and reverse movements in 1/2048 units (swap takes the rest, 2048 - w_migrate -
   * w_reverse).  Both 0 (the zero-initialised default) = swap only.  Requires
   * N = pp*dp <= 256 (else PIPETTE_E_UNSUPPORTED); every proposal is then evaluated in
   * full (O(N) per step). */
  int32_t w_migrate, w_reverse;
} pipette_sa_opts;

/* A plan (Alg.1 output "Conf, Map, T") plus counters and timings. */
typedef struct {
  pipette_config cfg;
  int32_t n_mb;
  double latency_s;         /* T_Pipette of the best mapping (Eq.3) */
  double t_bubble, t_straggler, t_pp, t_dp;   /* Eq.4-6 terms of that mapping (R6) */
  uint64_t mem_bytes;       /* analytic per-GPU memory of cfg (R11) */
  int32_t cfg_index;        /* e */
  int32_t chain;            /* c */
  int32_t best_step;
  int32_t n_slots;          /* N = pp*dp; perm[w] = TP-block slot of worker w = z*pp + x (R8, R9) */
  uint16_t* perm;           /* caller buffer of perm_cap entries (host) */
  int32_t perm_cap;
  uint64_t configs_enumerated, configs_rejected_oom, sa_steps, sa_accepted;
  double enumerate_ms, sa_ms, argmin_ms, combine_ms;   /* device time per phase on this rank */
} pipette_plan;

/* Create a context on device dist->device (or the current device if dist == NULL):
 * validates the inputs, computes R = 1/B (R5) and uploads it with the profile table,
 * and, for world > 1, creates the NCCL communicator (collective over all ranks).
 *   bw_bytes_per_s: n_nodes x n_nodes row-major directed bandwidths in bytes/s, the
 *     diagonal holding each node's intra-node bandwidth ("network_profile()",
 *     P:295 "B(g1,g2)"); finite and > 0.  Copied; the caller may free it on return.
 *   profile: n_profile entries, copied.
 * Errors: E_INVALID (shapes, non-finite or non-positive values, margin outside
 * [0,500], hidden % heads checked later), E_UNSUPPORTED (n_nodes > 128, G > 1024 or
 * gpus_per_node > 255: per-node stage-1 member counts are bytes on the device),
 * E_CUDA, E_NCCL.  On error *out is NULL. */
pipette_status pipette_init(pipette_ctx** out, const pipette_cluster* cluster,
                            const double* bw_bytes_per_s,
                            const pipette_profile_entry* profile, int32_t n_profile,
                            const pipette_dist* dist);

/* Replace the bandwidth matrix (host, same shape and rules as pipette_init); the
 * re-profiling step of Alg.1 l.1.  The host computes R = 1/B and the copy and the derived
 * tables are stream-ordered on the search stream: evals still in flight on any stream finish
 * with the old tables (the update waits for them on the device), every later
 * pipette_eval / pipette_search sees the new ones.  The caller's buffer may be reused on
 * return.  No device-wide synchronisation. */
pipette_status pipette_set_bandwidth(pipette_ctx* ctx, const double* bw_bytes_per_s);

/* Stream used by pipette_search (cudaStream_t as void*; NULL = legacy default stream). */
pipette_status pipette_set_stream(pipette_ctx* ctx, void* stream);

/* Alg.1 l.3-7 alone (K1 on the device, synchronous): enumerate every configuration in
 * canonical order (pp, tp, bs_micro ascending; R1, R2) with its analytic memory (R11)
 * and memory-filter verdict.  Host output arrays of `cap` entries (any
 * may be NULL): cfgs, n_mb, mem_bytes, feasible (1/0).  *E and *F receive the number of
 * enumerated and feasible configurations even when cap is smaller.
 * Errors: E_INVALID, E_UNSUPPORTED, E_CUDA. */
pipette_status pipette_enumerate(pipette_ctx* ctx, const pipette_model* model, int64_t bs_global,
                                 int32_t* E, int32_t* F, pipette_config* cfgs, int32_t* n_mb,
                                 uint64_t* mem_bytes, uint8_t* feasible, int32_t cap);

/* Evaluate n caller-supplied candidate plans (north_star "pipette_eval(candidates) ->
 * latencies and memory"): memory filter (Alg.1 l.7) and Eq.3-6 latency of each.
 * All array arguments are DEVICE pointers; the call is asynchronous on `stream` and
 * the buffers must stay alive until the stream is synchronised.
 *   d_cfg[i]        : configuration of candidate i
 *   d_perm          : candidate i's mapping at d_perm + i*perm_stride, N = pp*dp slots
 *                     (uint16, slot ids in [0,N)); perm_stride >= N of every candidate
 *                     (a shorter row gets status 3)
 *   d_latency[i]    : T_Pipette in seconds, NaN when status is 2, 3 or 4
 *   d_mem[i]        : per-GPU memory in bytes (0 when status is 2)
 *   d_status[i]     : 0 feasible, 1 over the memory limit (latency still computed),
 *                     2 configuration not in the enumeration of Alg.1 l.3-5,
 *                     3 mapping not a bijection on [0,N) (also when perm_stride < N: the
 *                       row is never read past perm_stride), 4 profile entry missing.
 * Errors: E_INVALID (n < 0, null pointers with n > 0, perm_stride < 1, bad model). */
pipette_status pipette_eval(pipette_ctx* ctx, const pipette_model* model, int64_t bs_global,
                            int64_t n, const pipette_config* d_cfg, const uint16_t* d_perm,
                            int32_t perm_stride, double* d_latency, uint64_t* d_mem,
                            uint8_t* d_status, void* stream);

/* Alg.1 on the device: enumerate and memory-filter all configurations,
 * run chains_per_config simulated-annealing chains of `iterations` swap proposals on
 * every feasible configuration (Alg.1 l.9-15), and return the best plan.
 * Synchronous and collective: every rank calls it with identical arguments; chains are
 * sharded by item j mod world (R18) and the per-rank winners are combined with NCCL;
 * every rank receives the identical plan, bit-identical for every world size.
 *   out->perm must hold at least N entries (else E_INVALID with out->n_slots = N).
 *   per_config (optional, per_config_cap entries, each with its own perm buffer):
 *     the best plan of each feasible configuration, sorted by (latency, e).
 * Errors: E_INVALID, E_PROFILE (R3), NO_FEASIBLE (configs_rejected_oom ==
 * configs_enumerated), E_CUDA, E_NCCL. */
pipette_status pipette_search(pipette_ctx* ctx, const pipette_model* model, int64_t bs_global,
                              int32_t chains_per_config, int32_t iterations, uint64_t seed,
                              const pipette_sa_opts* opts, pipette_plan* out,
                              pipette_plan* per_config, int32_t per_config_cap);

/* NEXT-4: use the memory estimator MLP of Eq.7 (reading
 * R23) instead of the analytic estimate (R11) for the memory filter of every later
 * enumeration, search and eval.  params (HOST, copied): 123023 doubles -- the 10 feature
 * means and 10 scales of ln(n_gpus, n_layers, hidden, heads, tp, pp, dp, bs_micro,
 * bs_mini, bs_global), then for each layer 10->200->200->200->200->1 the weights (out x in,
 * row-major) and biases, then the output's scale and mean (ln GB).  NULL restores the
 * analytic estimate.  Errors: E_INVALID (count, non-finite values, scale <= 0), E_CUDA. */
pipette_status pipette_set_memory_model(pipette_ctx* ctx, const double* params, int64_t n_params);

/* NEXT-2: three latency models of n caller candidates (same inputs,
 * layout, ownership and asynchrony as pipette_eval; reading R22 of DESIGN.md):
 *   d_t_pipette[i] : Eq.3-6, bit-identical to pipette_eval's latency
 *   d_t_prev[i]    : Eq.1, the prior-work model, with Eq.5's sum for
 *                    (pp-1) T_com^PP: ((((n_mb-1) C') + pp C') + T_PP) + T_DP, C' = C + T_TP
 *   d_t_des[i]     : a discrete-event simulation of the 1F1B schedule (P:107-111,
 *                    P:132-138) of every pipeline with f = C'/3, b = C' - f and directed
 *                    one-way hops msg_PP / B, max over pipelines, plus T_DP
 *   d_status[i]    : as pipette_eval, plus 5 = pp > 128 (not simulated); no memory output.
 * The three are NaN when status is 2..5.  Errors: as pipette_eval. */
pipette_status pipette_eval_models(pipette_ctx* ctx, const pipette_model* model, int64_t bs_global, int64_t n,
                                   const pipette_config* d_cfg, const uint16_t* d_perm, int32_t perm_stride,
                                   double* d_t_pipette, double* d_t_prev, double* d_t_des, uint8_t* d_status,
                                   void* stream);

/* NEXT-3: Alg.1 l.1 "network_profile()" (the paper's mpiGraph
 * profile of node pairs, Fig.3) on the GPUs of this box, from ONE process that
 * sees them all.  Every ordered pair (i, j) of devices[0..n_gpus) is timed with an
 * SM-driven copy kernel on GPU i that pushes `bytes` into GPU j's memory (peer stores over
 * NVLink / NVSwitch), the diagonal with the same copy inside GPU i; median of `reps`
 * launches after two warm-ups, CUDA events on GPU i.
 *   bw_out : n_gpus x n_gpus row-major bytes/s (HOST), directed, diagonal = intra -- the
 *            matrix pipette_init takes for a cluster of n_gpus one-GPU nodes (R5)
 *   ms_out : the median times (HOST, optional)
 *   err    : message buffer (optional)
 * Errors: E_INVALID, E_UNSUPPORTED (a pair without a peer path), E_CUDA. */
pipette_status pipette_profile_bandwidth(int32_t n_gpus, const int32_t* devices, uint64_t bytes, int32_t reps,
                                         double* bw_out, double* ms_out, char* err, int32_t err_cap);

/* Measured roofline denominators on `device`: sustained FP64 DADD+DMUL
 * instructions per second (counted per thread op) and 32-bit ALU (LOP3 + SHF) ops per
 * second, from independent chains at full occupancy.  Outputs HOST (either may be NULL).
 * Errors: E_CUDA. */
pipette_status pipette_measure_peaks(int32_t device, double* fp64_ops_per_s, double* alu_ops_per_s);

/* Measured shared-memory load bandwidth of this GPU in bytes per second (the SMEM
 * ceiling of SURVEY 8(d)'s min(FP64, INT, SMEM) roofline of the SA kernel): conflict-free
 * 64-bit loads from every warp at 64 warps per SM, CUDA-event timed, best of 3.
 * Output HOST (may be NULL).  Errors: E_CUDA. */
pipette_status pipette_measure_smem_bw(int32_t device, double* bytes_per_s);

/* Host-only helper (no GPU needed): the items j in [0, n_items) that `rank` of `world`
 * runs (R18), written to items (capacity cap).  Returns the count (may exceed cap). */
int64_t pipette_shard_items(int64_t n_items, int32_t rank, int32_t world, int64_t* items, int64_t cap);

/* Write a fresh 128-byte ncclUniqueId to id_out (rank 0, before pipette_init). */
pipette_status pipette_nccl_unique_id(void* id_out);

/* Diagnostics of the last pipette_search on this rank: per SA warp task (32 chains of one
 * configuration) [start ns, end ns, SM id, config index e] from the device globaltimer,
 * written to out (cap tasks x 4 uint64, host).  Returns the task count (-1 on error). */
int64_t pipette_last_task_profile(pipette_ctx* ctx, uint64_t* out, int64_t cap);

/* Work plan of the last pipette_search on this rank (diagnostics and tests): out[0] K3
 * variant (0: n <= 16 hop codes, 1: n <= 128 slot bytes, 2: wide positions), out[1] warp
 * tasks (32 chains of one configuration each), out[2] block chunks, out[3] grid (resident
 * blocks), out[4] warps per block, out[5] dynamic shared memory per block (bytes), out[6]
 * of it the block's shared tables.  Writes min(cap, 7) values, returns that count. */
int32_t pipette_last_search_stats(const pipette_ctx* ctx, int64_t* out, int32_t cap);

/* Number of kernel launches the last pipette_search / pipette_eval issued. */
int64_t pipette_last_launch_count(const pipette_ctx* ctx);

void pipette_destroy(pipette_ctx* ctx);
const char* pipette_last_error(const pipette_ctx* ctx);
const char* pipette_strerror(pipette_status status);

#ifdef __cplusplus
}
#endif
#endif /* PIPETTE_H */
