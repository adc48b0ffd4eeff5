// pipette_dev.cuh -- device data layout shared by the kernels and the host library.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/pipette.h"
#include "devmath.cuh"

namespace pip {

constexpr int kMaxNodes = 128;      // v1 limit (R table and node ids)
constexpr int kMaxGpus = 1024;      // v1 limit (G); N = G/tp <= 1024 slots
constexpr int kMaxGpusPerNode = 255;   // v1 limit: stage-1 counts c_n <= gpus_per_node are bytes

// One enumerated configuration (Alg.1 l.3-5) with its memory verdict (l.7) and the
// per-config model constants of DESIGN.md section 3.  Built on the device by
// k_enumerate_filter; read by k_eval_stream and k_sa_chains.
// K3 MODE 0 with n <= 8 nodes: hop codes a | b << 4 stay below 0x78, so the block's m2*R
// table has kSaCodesN8 codes (x 16 lane copies x 8 B = 15 KB instead of 32 KB).
constexpr int kSaCodesN8 = 120;
// Block shape of that variant: threads per block and resident blocks per SM (the
// __launch_bounds__ pair, hence the register cap); build-time knobs for A/B runs.
#ifndef PIPETTE_N8_THREADS
#define PIPETTE_N8_THREADS 128
#endif
#ifndef PIPETTE_N8_BLOCKS
#define PIPETTE_N8_BLOCKS 3   // (4 blocks of 128 = 128 registers: spills, measured 30% slower on C2)
#endif
constexpr int kSaThreadsN8 = PIPETTE_N8_THREADS;
constexpr int kSaBlocksN8 = PIPETTE_N8_BLOCKS;
// K3 MODE 1: warps per block (one block per SM; a chunk runs as many of them as its
// configuration's chain state fits); build-time knob for A/B runs.
#ifndef PIPETTE_M1_WARPS
#define PIPETTE_M1_WARPS 8
#endif
constexpr int kSaM1Warps = PIPETTE_M1_WARPS;
// entries of the global pair list kept in shared memory (list-mode witness scans start at
// the old witness's rank, expected (n/k)^2 <= 64 probes for |N1| >= 16 at n = 128)
constexpr int kSaM1PairPrefix = 1024;
// SaTask.pad of a MODE 1 task: warp-state stride / 16 in bits 0-15 and these flags
constexpr uint32_t kTfCache = 1u << 16;    // Eq.5 pipeline sums cached in shared memory
constexpr uint32_t kTfCounts = 1u << 17;   // stage-1 member counts kept (min(spn, dp) >= 2)
constexpr uint32_t kTfDirect = 1u << 18;   // T_ex by member pairs (min(dp, n) <= 8)

struct DevCfg {
  int32_t pp, tp, dp, mb;
  int32_t n_mb, e, N, spn;
  unsigned long long mem;            // bytes, exact (R11)
  int32_t feasible, has_profile;
  uint32_t pp_magic, spn_magic;      // ceil(2^32/pp), ceil(2^32/spn) for div_small
  int32_t qi_off, qe_off;            // qtab[qi_off + c] = qi(c), qtab[qe_off + k] = qe(k)
  double S, m2, md, r, Sb, Ss;
};

// Enumeration summary written by k_enumerate_filter.
struct EnumOut {
  int32_t E, F, qtab_used, overflow;
};

// One warp-task of the SA kernel: 32 chains (lanes) of one feasible configuration.
struct SaTask {
  int32_t cfg;        // index into the DevCfg table (= e)
  int32_t f;          // feasible index
  int32_t c_first;    // first local chain id of this config on this rank
  int32_t k0;         // first local ordinal of this task within the config
  int32_t count;      // active lanes (<= 32)
  int32_t slot0;      // first local chain slot (outputs) of this task
  int32_t perm_off;   // offset (uint16 units) of this task's best-perm block [N][32]
  int32_t pad;
};

// Per-chain outputs of k_sa_chains, indexed by local chain slot.
struct ChainOut {
  double best, best_tpp, best_tdp, L0;
  int32_t best_step;
  uint32_t accepted;
  int32_t f, c;
};

// Per-config winner of this rank (k_argmin).
struct CfgBest {
  double best, best_tpp, best_tdp;
  int32_t chain, slot, best_step, pad;
  unsigned long long accepted;
};

struct SaParams {
  const DevCfg* cfgs;
  const double* qtab;
  const double* R;           // n x n, R[a][b] = 1/B[a][b]
  const double* subset_max;  // 2^n subset maxima of R off-diagonal (n <= 16), or null
  const uint8_t* tin_rank;   // per feasible config: 256 ranks (k_tin_rank), MODE 0
  const double* tin_vs;      // per feasible config: 256 values in rank order, MODE 0
  const uint8_t* nl_node;    // S1Large cluster tables (k_node_lists, k_pair_list)
  const double* nl_val;
  const uint16_t* gl_ab;
  const double* gl_val;
  const uint16_t* tl_ac;     // S1Large per-config T_in lists (k_tin_list), row stride tl_stride
  const double* tl_val;
  const int* tl_len;
  int32_t tl_stride;
  int32_t psum_dp_cap;       // pipeline sums cached in shared memory when dp <= this
  const SaTask* tasks;
  int32_t n_tasks;
  const int2* chunks;        // block work units: (first task, task count <= warps per block), one config each
  int32_t n_chunks;
  int32_t* task_counter;
  int32_t* claimed;          // per chunk: taken (zeroed per launch)
  int32_t* sm_slot;          // per SM: blocks that made their first fetch (zeroed per launch)
  int32_t n_sms;
  int32_t n_nodes;
  int32_t iterations;
  uint2 key;                 // Philox key (seed lo, seed hi)
  RoundKeys rk;              // its ten round keys (philox_round_keys(key))
  int32_t world;             // chain ids c = c_first + k*world
  double alpha_inv, tau, t0;
  int32_t warps_per_block;
  int32_t warp_smem_bytes;   // per-warp chain-state region
  int32_t r_smem_bytes;
  ChainOut* out;
  uint16_t* best_perm;
  unsigned long long* task_prof;   // per task: [start ns, end ns, smid, cfg] (diagnostics)
  // trace (debug): trace_slot[local slot] = record row or -1
  const int32_t* trace_slot;
  int32_t trace_cap;
  pipette_trace_record* trace;
  int32_t w_migrate, w_reverse;   // full move set (R21); both 0: swap only
  int32_t s1_nib;                 // MODE 1 swap kernels: stage-1 counts as nibbles (all <= 15)
  // MODE 1: the block's R table has row stride 2^r_lg; pt = per-node pair rows in
  // global-list order (k_partner_lists), pt_stride entries each; plen = pair-list prefix
  // entries kept in shared memory
  int32_t r_lg;
  const uint32_t* pt;
  int32_t pt_stride;
  int32_t plen;
  // per feasible config: beta0 = 1/T0 by self-calibration (R24, k_t0_calibrate), or null
  const double* beta0;
};

// Inverse initial temperature of a chain (R13, R24): 1/t0 for an explicit t0 > 0, the
// configuration's self-calibrated value when requested (t0 < 0), else 1/(tau * L(identity)).
__device__ __forceinline__ double sa_beta0(const SaParams& P, int f, double L0) {
  if (P.t0 > 0.0) return __ddiv_rn(1.0, P.t0);
  if (P.beta0) return P.beta0[f];
  return __ddiv_rn(1.0, __dmul_rn(P.tau, L0));
}

struct EvalParams {
  const DevCfg* cfgs;
  const unsigned long long* keys;   // sorted (pp<<48 | tp<<32 | dp<<16 | mb) of every config
  int32_t E;
  const double* qtab;
  const double* R;
  const double* subset_max;  // 2^n table (MODE 0)
  const double* vin;         // [E][256] qi(c) R[a][a] values (MODE 0)
  const uint16_t* gl_ab;     // all ordered node pairs (a | b << 8) by R descending (MODE 1)
  const double* gl_val;      // their R values
  int32_t n_nodes;
  int64_t n;
  const pipette_config* cand;
  const uint16_t* perm;
  int32_t perm_stride;
  int32_t vec16;             // perm rows are 16-byte aligned
  int32_t staged;            // rows gathered into per-warp shared staging buffers (vec16, fits)
  int32_t bm_words;          // bitmap words per thread (ceil(maxN/32))
  int32_t rep;
  int32_t tma;               // single-configuration tiles staged by TMA (128-byte rows, tensor map)
  int32_t cnt_nib;           // per-thread stage-1 counts as nibbles (every count <= 15)
  int32_t plen;              // MODE 1: entries of the R-sorted pair list copied to shared memory
  double* latency;
  unsigned long long* mem;
  uint8_t* status;
};

}  // namespace pip
