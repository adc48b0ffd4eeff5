// host.cu -- the C ABI of include/pipette.h: validation, context, device tables,
// launch orchestration of K1-K6 and the NCCL combine across ranks.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "devmath.cuh"
#include "pipette_dev.cuh"

namespace pip {
// kernels (k_enumerate.cu, k_eval.cu, k_sa.cu)
__global__ void k_enumerate_filter(int, int, unsigned long long, int, pipette_model, long long,
                                   const pipette_profile_entry*, int, DevCfg*, unsigned long long*, int, int*,
                                   double*, int, EnumOut*);
const void* eval_kernel(int mode, int threads);
const void* eval_warp_kernel();
size_t eval_warp_smem_bytes(int n_nodes, int E);
int eval_warp_threads();
void launch_mlp_filter(const double* P, int G, int n_nodes, const pipette_model& m, long long bs, unsigned long long cap,
                       int margin, DevCfg* cfgs, int* feas, EnumOut* out, cudaStream_t s);
int eval_tile_size();
pipette_status netprof_run(int n, const int* devs, size_t bytes, int reps, double* bw, double* ms_out, char* err,
                           size_t err_cap);
pipette_status models_launch(const DevCfg* cfgs, const unsigned long long* keys, int E, const double* qtab,
                             const double* R, int n_nodes, long long n, const pipette_config* cand,
                             const uint16_t* perm, int stride, double* tp, double* tprev, double* tdes,
                             uint8_t* status, void* stream);
size_t eval_smem_bytes(int mode, int perm_stride, bool staged, int n_nodes, int E, int bm_words, int threads,
                       bool cnt_nib, int plen);
__global__ void k_tin_values(const DevCfg*, const double*, const double*, int, double*);
const void* sa_kernel(int mode, bool trace, int n_nodes, bool full);
int sa_warp_state_bytes(int mode, int N, int pp, int dp, int n, int dp_cap, bool nib);
int sa_m1_warp_state_bytes(int N, int dp, int n, bool counts, bool cache, bool nib, bool direct);
int sa_m1_count_bytes(int n, bool nib);
void launch_t0_calibrate(const DevCfg*, const int*, int, const double*, const double*, int, const RoundKeys&, int, int,
                         double, double*, cudaStream_t);
__global__ void k_partner_lists(const uint16_t*, int, uint32_t*, int);
__global__ void k_cfg_cost(const unsigned long long*, const SaTask*, int, unsigned long long*);
__global__ void k_node_lists(const double*, int, uint8_t*, double*);
__global__ void k_pair_list(const double*, int, uint16_t*, double*);
__global__ void k_tin_list(const DevCfg*, const int*, const double*, const double*, int, int, uint16_t*, double*, int*);
__global__ void k_subset_max(const double*, int, double*);
__global__ void k_tin_rank(const DevCfg*, const int*, const double*, const double*, int, uint8_t*, double*);
__global__ void k_argmin(const ChainOut*, const int*, int, CfgBest*);
constexpr int kEnumThreads = 1024, kSaThreads = 128;

// K5 (combine, phase 1): per-config local winner item id if it attains the global
// minimum latency, else UINT64_MAX (second allreduce(min) of R18).
__global__ void k_combine_items(const CfgBest* __restrict__ cb, const unsigned long long* __restrict__ gbits,
                                int F, long long chains, unsigned long long* __restrict__ items) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const CfgBest b = cb[f];
  const bool mine = b.chain >= 0 && (unsigned long long)__double_as_longlong(b.best) == gbits[f];
  items[f] = mine ? (unsigned long long)f * (unsigned long long)chains + (unsigned long long)b.chain : ~0ull;
}

// K6 (combine, phase 2): the owner of each config's winner packs its plan -- Eq.4-6
// breakdown, best step and the best mapping gathered from the lane-interleaved SA
// buffer -- and every other rank packs zeros, so one allreduce(sum) broadcasts all
// per-config plans at once.  Row layout (u64 words): [t_pp, t_dp, t_bubble, best_step+1,
// perm words (4 slots per word)...]; the last element carries this rank's accepted count.
__global__ void k_combine_pack(const CfgBest* __restrict__ cb, const unsigned long long* __restrict__ gitem,
                               const DevCfg* __restrict__ cfgs, const int* __restrict__ feas,
                               const int* __restrict__ slot_perm_off, const int* __restrict__ slot_lane,
                               const uint16_t* __restrict__ best_perm, int F, long long chains, int row_words,
                               unsigned long long* __restrict__ pack) {
  const int f = blockIdx.x;
  if (f >= F) return;
  const CfgBest b = cb[f];
  const bool owner = b.chain >= 0 && gitem[f] == (unsigned long long)f * (unsigned long long)chains + b.chain;
  unsigned long long* row = pack + (size_t)f * row_words;
  const DevCfg C = cfgs[feas[f]];
  for (int w = threadIdx.x; w < row_words; w += blockDim.x) {
    unsigned long long v = 0ull;
    if (owner) {
      if (w == 0) v = (unsigned long long)__double_as_longlong(b.best_tpp);
      else if (w == 1) v = (unsigned long long)__double_as_longlong(b.best_tdp);
      else if (w == 2) v = (unsigned long long)__double_as_longlong(__dadd_rn(C.Sb, b.best_tpp));
      else if (w == 3) v = (unsigned long long)(long long)(b.best_step + 1);
      else {
        const int s0 = (w - 4) * 4;
        const int off = slot_perm_off[b.slot], lane = slot_lane[b.slot];
        for (int j = 3; j >= 0; --j) {
          const int s = s0 + j;
          v = (v << 16) | (s < C.N ? (unsigned long long)best_perm[off + s * 32 + lane] : 0ull);
        }
      }
    }
    row[w] = v;
  }
}

__global__ void k_sum_accepted(const CfgBest* __restrict__ cb, int F, unsigned long long* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long s = 0;
    for (int f = 0; f < F; ++f) s += cb[f].accepted;
    *out = s;
  }
}
}  // namespace pip

using namespace pip;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct HostPlanKey {
  pipette_model model;
  long long bs;
  int chains, W, r, dp_cap_env, full_moves;
};
struct HostPlan {
  std::vector<SaTask> sorted;
  std::vector<int2> chunks;
  std::vector<int> cfg_slot, slot_perm_off, slot_lane;
  int slots = 0, perm_words = 0, maxN = 1, mode = 0, r_bytes = 0, dp_cap = 0, warp_bytes = 16, tl_stride = 1, wpb = 1;
  int r_lg = 0, plen = 0;   // MODE 1: R row stride 2^r_lg, pair-list prefix entries
  bool big = false, nib = false;
  bool measured = false;    // tasks ordered by measured per-configuration durations
  size_t smem = 0;
};

struct pipette_ctx {
  int device = 0, rank = 0, world = 1;
  int n_nodes = 0, g = 0, margin = 0;
  unsigned long long cap = 0;
  int n_sms = 148;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  pipette_host_allreduce_fn host_ar = nullptr;   // host transport of the combine (no NCCL)
  void* host_user = nullptr;
  unsigned long long* h_ar = nullptr;            // its pinned staging buffer
  size_t h_ar_words = 0;
  std::string err;
  int64_t launches = 0;
  // device tables
  double* dR = nullptr;
  double* dTab = nullptr;   // subset-max table (n <= 16)
  // sorted cluster tables for larger clusters (n > 16)
  uint8_t* dNlNode = nullptr;
  double* dNlVal = nullptr;
  uint16_t* dGlAb = nullptr;
  double* dGlVal = nullptr;
  uint32_t* dPt = nullptr;   // MODE 1 per-node pair rows (k_partner_lists)
  int pt_stride = 0;
  pipette_profile_entry* dProf = nullptr;
  int n_prof = 0;
  std::vector<pipette_profile_entry> prof;
  // enumeration cache (model, bs_global) -> device config table
  bool enum_valid = false;
  pipette_model enum_model{};
  long long enum_bs = 0;
  int E = 0, F = 0;
  std::vector<DevCfg> hcfg;
  std::vector<int> hfeas;
  DevBuf cfgs, keys, feas, qtab, eout, vin;
  bool vin_valid = false;   // K2 intra-node value table matches the config table and R
  // search buffers
  DevBuf mlp;   // Eq.7 MLP parameters (NEXT-4), empty = analytic memory (R11)
  DevBuf claimed;   // SA chunk claim flags + per-SM first-fetch slots
  DevBuf tasks, chunks, counter, chain_out, best_perm, cfg_slot, cfg_best, gbits, items, gitems, pack, accepted,
      slot_perm_off, slot_lane, trace_slot, trace, task_prof, tin_rank, tin_vs, tl_ac, tl_val, tl_len, beta0, cfg_cost;
  // measured mean task duration (ms) of each enumerated configuration from the last search's
  // task profile (k_cfg_cost), for the longest-first order of the next work plan; empty = none
  std::vector<double> cfg_cost_ms;
  int64_t n_tasks_last = 0;
  HostPlanKey plan_key{};
  HostPlan plan;
  bool plan_valid = false;
  // host copies of the last uploaded SA work lists (skip identical re-uploads)
  std::vector<unsigned char> up_tasks, up_chunks, up_cfg_slot, up_slot_perm_off, up_slot_lane;
  cudaEvent_t ev[6] = {};
  // stream ordering of the device tables (R, subset-max, sorted lists, K2's vin): a rewrite
  // on ctx->stream waits for the evals still in flight on their streams (one event per
  // stream an eval ran on), and every later eval/search waits for ev_tables
  cudaEvent_t ev_tables = nullptr;
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> eval_streams;
  double* hR = nullptr;   // pinned staging of R for the stream-ordered upload
  struct FnAttr { const void* fn; size_t smem; int threads; int occ; };
  std::vector<FnAttr> fn_cache;   // dynamic shared-memory limit set and occupancy, per kernel/shape
  int64_t stats[8] = {};          // last search: mode, tasks, chunks, grid, warps/block, smem, r_bytes, launches
};

namespace {

constexpr int64_t kMlpParams = 20 + 200 * 10 + 200 + 3 * (200 * 200 + 200) + 200 + 1 + 2;   // Eq.7 MLP (R23)

int align16(int x) { return (x + 15) & ~15; }
thread_local std::string g_init_err;

const char* kStatusText[] = {"ok", "no feasible configuration (every candidate exceeds the memory limit)",
                             "invalid argument", "profile entry missing for a feasible (tp, mb)",
                             "CUDA error", "NCCL error", "unsupported size (v1 limits)"};

pipette_status fail(pipette_ctx* c, pipette_status s, const char* fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
  }
  return s;
}

#define CU(call)                                                                                         \
  do {                                                                                                   \
    cudaError_t e_ = (call);                                                                             \
    if (e_ != cudaSuccess) return fail(ctx, PIPETTE_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
#define NC(call)                                                                                         \
  do {                                                                                                   \
    ncclResult_t r_ = (call);                                                                            \
    if (r_ != ncclSuccess) return fail(ctx, PIPETTE_E_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
  } while (0)

// One reduction of the combine (R18) over `count` uint64 words, op 0 = min, 1 = sum: NCCL
// on the stream, or the caller's host collective (pipette_dist.host_allreduce) on a pinned
// copy -- the stream is drained around the host call, the result copied back in order.
pipette_status allreduce_u64(pipette_ctx* ctx, const unsigned long long* src, unsigned long long* dst, size_t count,
                             int op, cudaStream_t s) {
  if (ctx->comm) {
    NC(ncclAllReduce(src, dst, count, ncclUint64, op == 0 ? ncclMin : ncclSum, ctx->comm, s));
    return PIPETTE_OK;
  }
  if (!ctx->host_ar) return fail(ctx, PIPETTE_E_NCCL, "world > 1 without a transport");
  if (ctx->h_ar_words < count) {
    if (ctx->h_ar) cudaFreeHost(ctx->h_ar);
    ctx->h_ar = nullptr;
    ctx->h_ar_words = 0;
    CU(cudaMallocHost(&ctx->h_ar, sizeof(unsigned long long) * count));
    ctx->h_ar_words = count;
  }
  CU(cudaMemcpyAsync(ctx->h_ar, src, sizeof(unsigned long long) * count, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (ctx->host_ar(ctx->host_user, reinterpret_cast<uint64_t*>(ctx->h_ar), (int64_t)count, op) != 0)
    return fail(ctx, PIPETTE_E_NCCL, "host allreduce (op %d, %zu words) failed", op, count);
  CU(cudaMemcpyAsync(dst, ctx->h_ar, sizeof(unsigned long long) * count, cudaMemcpyHostToDevice, s));
  return PIPETTE_OK;
}

cudaError_t ensure(DevBuf& b, size_t bytes) {
  if (b.bytes >= bytes && b.p) return cudaSuccess;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  cudaError_t e = cudaMalloc(&b.p, std::max<size_t>(bytes, 16));
  if (e == cudaSuccess) b.bytes = std::max<size_t>(bytes, 16);
  return e;
}

// ensure() for a buffer whose host copy of the last upload is kept: a reallocation drops
// the device contents, so it also forgets the copy
cudaError_t ensure_up(DevBuf& b, size_t bytes, std::vector<unsigned char>& up) {
  void* before = b.p;
  cudaError_t e = ensure(b, bytes);
  if (b.p != before) up.clear();
  return e;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link); null if
// the driver does not provide it
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// Blocks per SM of kern at (threads, smem); the kernel's dynamic shared-memory limit is
// raised once per size (cached: no attribute call or occupancy query per launch).
pipette_status kernel_occupancy(pipette_ctx* ctx, const void* kern, int threads, size_t smem, int* occ) {
  for (const auto& a : ctx->fn_cache)
    if (a.fn == kern && a.smem == smem && a.threads == threads) { *occ = a.occ; return PIPETTE_OK; }
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int o = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, smem));
  o = std::max(o, 1);
  ctx->fn_cache.push_back({kern, smem, threads, o});
  *occ = o;
  return PIPETTE_OK;
}

// Table updates happen on ctx->stream between tables_begin (wait for every eval in flight)
// and tables_end (record ev_tables); a launch on stream s first waits for ev_tables.
cudaError_t tables_begin(pipette_ctx* ctx) {
  for (const auto& se : ctx->eval_streams)
    if (se.first != ctx->stream) {
      cudaError_t e = cudaStreamWaitEvent(ctx->stream, se.second, 0);
      if (e != cudaSuccess) return e;
    }
  return cudaSuccess;
}
cudaError_t tables_end(pipette_ctx* ctx) { return cudaEventRecord(ctx->ev_tables, ctx->stream); }
cudaError_t wait_tables(pipette_ctx* ctx, cudaStream_t s) { return cudaStreamWaitEvent(s, ctx->ev_tables, 0); }
// an eval was launched on s: the next table rewrite waits for it
cudaError_t note_eval(pipette_ctx* ctx, cudaStream_t s) {
  for (auto& se : ctx->eval_streams)
    if (se.first == s) return cudaEventRecord(se.second, s);
  if (ctx->eval_streams.size() >= 16) {   // many streams: keep the table rewrites safe by a device sync
    for (auto& se : ctx->eval_streams) cudaEventDestroy(se.second);
    ctx->eval_streams.clear();
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return e;
  }
  cudaEvent_t ev;
  cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e != cudaSuccess) return e;
  ctx->eval_streams.push_back({s, ev});
  return cudaEventRecord(ev, s);
}

int n_div(long long n) {
  int c = 0;
  for (long long d = 1; d * d <= n; ++d)
    if (n % d == 0) c += (d * d == n) ? 1 : 2;
  return c;
}

pipette_status check_bw(pipette_ctx* ctx, const double* bw, int n) {
  if (!bw) return fail(ctx, PIPETTE_E_INVALID, "bandwidth matrix is NULL");
  for (int i = 0; i < n * n; ++i)
    if (!std::isfinite(bw[i]) || !(bw[i] > 0.0))
      return fail(ctx, PIPETTE_E_INVALID, "bandwidth[%d][%d] = %g must be finite and > 0", i / n, i % n, bw[i]);
  return PIPETTE_OK;
}

// R = 1/B (R5, IEEE division on the host) and the tables derived from it, uploaded in
// stream order on ctx->stream (pinned staging, no device-wide synchronisation): evals in
// flight finish with the old tables, every later call sees the new ones.
pipette_status upload_bw(pipette_ctx* ctx, const double* bw) {
  const int n = ctx->n_nodes;
  if (!ctx->hR) CU(cudaMallocHost(&ctx->hR, sizeof(double) * n * n));
  CU(cudaEventSynchronize(ctx->ev_tables));   // the previous upload has left the staging buffer
  for (int i = 0; i < n * n; ++i) ctx->hR[i] = 1.0 / bw[i];  // R5: IEEE division, never symmetrised
  if (n <= 16 && !ctx->dTab) CU(cudaMalloc(&ctx->dTab, sizeof(double) << n));
  const size_t L1 = (size_t)n * 2 * (n - 1), L2 = (size_t)n * (n - 1);
  if (n >= 2 && !ctx->dNlNode) {   // sorted partner / pair lists (MODE 1 and 2 stage-1 searches)
    CU(cudaMalloc(&ctx->dNlNode, L1));
    CU(cudaMalloc(&ctx->dNlVal, sizeof(double) * L1));
    CU(cudaMalloc(&ctx->dGlAb, sizeof(uint16_t) * L2));
    CU(cudaMalloc(&ctx->dGlVal, sizeof(double) * L2));
    ctx->pt_stride = ((2 * (n - 1)) + 3) & ~3;
    CU(cudaMalloc(&ctx->dPt, sizeof(uint32_t) * (size_t)n * ctx->pt_stride));
  }
  cudaStream_t s = ctx->stream;
  CU(tables_begin(ctx));
  CU(cudaMemcpyAsync(ctx->dR, ctx->hR, sizeof(double) * n * n, cudaMemcpyHostToDevice, s));
  if (n <= 16) k_subset_max<<<((1 << n) + 255) / 256, 256, 0, s>>>(ctx->dR, n, ctx->dTab);
  if (n >= 2) {
    k_node_lists<<<n, 256, 0, s>>>(ctx->dR, n, ctx->dNlNode, ctx->dNlVal);
    k_pair_list<<<(unsigned)((L2 + 255) / 256), 256, 0, s>>>(ctx->dR, n, ctx->dGlAb, ctx->dGlVal);
    k_partner_lists<<<n, 32, 0, s>>>(ctx->dGlAb, n, ctx->dPt, ctx->pt_stride);
  }
  CU(cudaGetLastError());
  CU(tables_end(ctx));
  ctx->vin_valid = false;
  return PIPETTE_OK;
}

pipette_status check_model(pipette_ctx* ctx, const pipette_model* m, long long bs) {
  if (!m) return fail(ctx, PIPETTE_E_INVALID, "model is NULL");
  if (m->n_layers < 1 || m->hidden < 1 || m->heads < 1 || m->seq_len < 1 || m->vocab < 1 ||
      m->bytes_per_elem < 1 || m->bytes_per_param_state < 0)
    return fail(ctx, PIPETTE_E_INVALID, "model fields must be positive");
  if (m->hidden % m->heads != 0) return fail(ctx, PIPETTE_E_INVALID, "hidden %% heads != 0");
  if (bs < 1 || bs > (1ll << 30)) return fail(ctx, PIPETTE_E_INVALID, "bs_global out of range");
  return PIPETTE_OK;
}

// K1 on ctx->stream; synchronous readback of the table (cached per (model, bs)).
// The host-side work plan of pipette_search (R18 sharding, warp tasks in longest-first
// order, block chunks of one configuration, kernel variant and shared-memory layout).
pipette_status build_plan(pipette_ctx* ctx, int chains, int W, int r, const char* cap_env, bool full_moves,
                          HostPlan& hp) {
  // ---- shard items j = f*chains + c by j mod world (R18); group 32 local chains per warp task
  const int F = ctx->F;
  std::vector<SaTask> tasks;
  std::vector<int>& cfg_slot = hp.cfg_slot;
  std::vector<int>& slot_perm_off = hp.slot_perm_off;
  std::vector<int>& slot_lane = hp.slot_lane;
  cfg_slot.assign(F + 1, 0);
  int slots = 0, perm_words = 0, maxN = 1, maxdp2 = 0;
  for (int f = 0; f < F; ++f) {
    const DevCfg& c = ctx->hcfg[ctx->hfeas[f]];
    const long long base = (long long)f * chains;
    const int c_first = (int)(((r - base) % W + W) % W);
    const int count = c_first < chains ? (chains - 1 - c_first) / W + 1 : 0;
    cfg_slot[f] = slots;
    maxN = std::max(maxN, c.N);
    if (c.pp >= 2) maxdp2 = std::max(maxdp2, c.dp);
    for (int k0 = 0; k0 < count; k0 += 32) {
      SaTask t{};
      t.cfg = c.e;
      t.f = f;
      t.c_first = c_first;
      t.k0 = k0;
      t.count = std::min(32, count - k0);
      t.slot0 = slots;
      t.perm_off = perm_words;
      for (int l = 0; l < t.count; ++l) { slot_perm_off.push_back(perm_words); slot_lane.push_back(l); }
      slots += t.count;
      perm_words += c.N * 32;
      tasks.push_back(t);
    }
  }
  cfg_slot[F] = slots;
  // longest-processing-time-first order of the warp tasks.  The cost of a task is its
  // expected duration, fitted (least squares) to the per-task timings of tools/task_profile.py
  // on B200 (profiles/r01i_task_profile_c*.log): MODE 0 with n <= 8 on C2; MODE 1 on C4/C5,
  // where the stage-1 updates (probability pchg = 2(1/pp)(1-1/pp)) dominate and grow with n;
  // MODE 0 with 8 < n <= 16 keeps the earlier pp-driven estimate (the C2 fit measured 6%
  // slower on the multi-wave C3).  PIPETTE_COST_FIT=0 selects the earlier estimate everywhere.
  std::vector<double> cost(tasks.size());
  const char* cf_env = getenv("PIPETTE_COST_FIT");
  const bool cost_fit = !(cf_env && atoi(cf_env) == 0);
  // measured durations of the previous search on this enumeration, when every configuration
  // has one (the plan is then rebuilt once: ordering never changes results, chains are
  // independent and their Philox streams are indexed by (step, chain, e))
  // (MODE 0 keeps its fitted model: ordering by measured means interleaves pipeline depths
  // on an SM and measured C3 165 vs 150 ms, C2 up to 17.9 vs 16.0 ms -- I-cache)
  const bool mode0_plan = ctx->n_nodes <= 16 && maxN <= 256 && ctx->g <= 15 && ctx->dTab;
  bool measured = cost_fit && !mode0_plan && !ctx->cfg_cost_ms.empty();
  for (size_t i = 0; measured && i < tasks.size(); ++i)
    measured = tasks[i].cfg < (int)ctx->cfg_cost_ms.size() && ctx->cfg_cost_ms[tasks[i].cfg] > 0.0;
  hp.measured = measured;
  const int n_nodes = ctx->n_nodes;
  const bool mode0 = n_nodes <= 16 && maxN <= 256 && ctx->g <= 15 && ctx->dTab;
  for (size_t i = 0; i < tasks.size(); ++i) {
    const DevCfg& c = ctx->hcfg[tasks[i].cfg];
    const double pchg = 2.0 * (1.0 / c.pp) * (1.0 - 1.0 / c.pp);
    double v = c.pp >= 2 ? 60.0 + 12.0 * (c.pp - 1) + pchg * (40.0 + 4.0 * n_nodes) : 10.0;
    if (cost_fit && mode0 && n_nodes <= 8)
      v = c.pp >= 2 ? 10.3 + 0.079 * c.pp + 0.037 * c.N + 0.067 * c.dp + 3.06 * pchg : 1.8;
    else if (cost_fit && !mode0)   // (fit to C5 task durations after the round-2 MODE 1 redesign)
      v = c.pp >= 2 ? 48.4 - 0.26 * (c.pp - 1) - 72.4 * pchg + 0.17 * c.dp - 5.3 * (c.spn > 1 ? 1.0 : 0.0) : 1.0;
    if (measured) v = ctx->cfg_cost_ms[tasks[i].cfg];
    cost[i] = c.N < 2 ? 0.0 : v;
  }
  std::vector<int> order(tasks.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  std::vector<SaTask>& sorted = hp.sorted;
  sorted.resize(tasks.size());
  for (size_t i = 0; i < order.size(); ++i) sorted[i] = tasks[order[i]];
  if (const char* only = getenv("PIPETTE_DIAG_ONLY_CFG")) {   // diagnostics (per-config profiles):
    const int e = atoi(only);                                // run only configuration e's tasks;
    std::vector<SaTask> keep;                                // the plan is then meaningless
    for (const SaTask& t : sorted)
      if (t.cfg == e) keep.push_back(t);
    sorted.swap(keep);
  }

  const int n = ctx->n_nodes;
  // MODE 0 (n <= 16): packed positions, register stage-1 state, lane-replicated R,
  // subset-max table.  MODE 1 (N <= 256): slot bytes, the block's shared R table, S1M
  // stage-1 state.  MODE 2: 32-bit positions (N > 256).
  // (the MODE 1 swap kernel maps slots to nodes by shifts: gpus_per_node a power of two)
  const bool g_pow2 = (ctx->g & (ctx->g - 1)) == 0;
  const int mode = (n <= 16 && maxN <= 256 && ctx->g <= 15 && ctx->dTab) ? 0
                 : ((maxN <= 256 && (g_pow2 || full_moves)) ? 1 : 2);
  if (mode == 2 && full_moves)
    return fail(ctx, PIPETTE_E_UNSUPPORTED, "the full move set needs N = pp*dp <= 256 (max N here %d)", maxN);
  if (mode == 1) {
    // MODE 1: one block of kSaM1Warps warps per SM; the block holds R (row stride 2^lg) and
    // the pair-list prefix; a chunk of a configuration runs as many warps as that
    // configuration's chain state fits in the rest of shared memory.  Per configuration:
    // stage-1 counts when some node can hold >= 2 members, T_ex by member pairs when N1
    // never exceeds 8 nodes, and the pipeline-sum cache when it saves re-summing long
    // pipelines (pp >= PIPETTE_M1_CACHE_PP, default 2; the old sums of the two touched
    // pipelines are otherwise re-summed) and costs at most one resident warp
    // (PIPETTE_M1_CACHE_MIN: the fewest warps the cache may leave).
    int lg = 0;
    while ((1 << lg) < n) ++lg;
    const int plen = std::min(n * (n - 1), kSaM1PairPrefix);
    const int r_bytes = align16(8 << (2 * lg)) + align16(plen * 2);
    const int avail = 227 * 1024 - 64 - r_bytes;
    bool nib = !full_moves;
    for (int f = 0; f < F; ++f) {
      const DevCfg& c = ctx->hcfg[ctx->hfeas[f]];
      nib = nib && std::min(c.spn, c.dp) <= 15;
    }
    const char* cm_env = getenv("PIPETTE_M1_CACHE_MIN");
    const int cache_min = cm_env ? atoi(cm_env) : kSaM1Warps - 1;
    const char* cp_env = getenv("PIPETTE_M1_CACHE_PP");
    const int cache_pp = cp_env ? atoi(cp_env) : 2;
    std::vector<int> fbytes(F), fwarps(F);
    std::vector<uint32_t> fflags(F);
    for (int f = 0; f < F; ++f) {
      const DevCfg& c = ctx->hcfg[ctx->hfeas[f]];
      const bool counts = full_moves || std::min(c.spn, c.dp) >= 2;
      const bool direct = std::min(c.dp, n) <= 8;
      const int base = full_moves ? align16(((c.N + 3) / 4) * 128) + sa_m1_count_bytes(n, false)
                                  : sa_m1_warp_state_bytes(c.N, c.dp, n, counts, false, nib, direct);
      const int with = sa_m1_warp_state_bytes(c.N, c.dp, n, counts, true, nib, direct);
      const int w_nc = std::min(kSaM1Warps, avail / base), w_c = std::min(kSaM1Warps, avail / with);
      // (measured on C5, 3 alternating reps: keeping the cache at the cost of at most one
      // resident warp, 770-775 ms per search, beats both no lost warp (822-826) and the earlier
      // pp >= 16 rule that let (16,4,16) drop to 6 warps (779-782))
      const int need = std::min(w_nc, cm_env ? cache_min : kSaM1Warps - 1);
      const bool cache = !full_moves && c.pp >= std::max(2, cache_pp) && w_c >= 1 && w_c >= need;
      fbytes[f] = cache ? with : base;
      fwarps[f] = cache ? w_c : w_nc;
      if (fwarps[f] < 1)
        return fail(ctx, PIPETTE_E_UNSUPPORTED, "SA state of config e=%d (%d B/warp) exceeds shared memory", c.e, base);
      fflags[f] = (uint32_t)(fbytes[f] / 16) | (cache ? kTfCache : 0u) | (counts ? kTfCounts : 0u) |
                  (direct ? kTfDirect : 0u);
    }
    for (SaTask& t : sorted) t.pad = (int32_t)fflags[t.f];
    // block work units: up to the configuration's warp count of consecutive tasks of one
    // configuration, and no more than an even share of the tasks per SM (a small search
    // spreads over every SM)
    const int share = std::max(1, (int)((sorted.size() + ctx->n_sms - 1) / ctx->n_sms));
    std::vector<int2>& chunks = hp.chunks;
    size_t smem = (size_t)r_bytes;
    for (size_t i = 0; i < sorted.size();) {
      const int f = sorted[i].f;
      const int cap = std::min(fwarps[f], share);
      size_t j = i + 1;
      while (j < sorted.size() && (int)(j - i) < cap && sorted[j].cfg == sorted[i].cfg) ++j;
      chunks.push_back(make_int2((int)i, (int)(j - i)));
      smem = std::max(smem, (size_t)r_bytes + (size_t)(j - i) * fbytes[f]);
      i = j;
    }
    int tls = 1;
    for (int f = 0; f < F; ++f) {
      const DevCfg& c = ctx->hcfg[ctx->hfeas[f]];
      tls = std::max(tls, n * (std::min(c.spn, c.dp) - 1));
    }
    hp.slots = slots; hp.perm_words = perm_words; hp.maxN = maxN; hp.mode = 1; hp.r_bytes = r_bytes;
    hp.big = false; hp.nib = nib; hp.dp_cap = 0; hp.warp_bytes = 0; hp.tl_stride = tls; hp.wpb = kSaM1Warps;
    hp.smem = smem; hp.r_lg = lg; hp.plen = plen;
    return PIPETTE_OK;
  }
  // MODE 0: the block's m2*R table, 256 hop codes x 16 lane copies (64-bit loads are served
  // per half-warp, so 16 copies make every lookup conflict free)
  // (+ MODE 0's shared stage-1 tables: vs 256, qe 32 and tab 256 doubles, rank 256 bytes)
  const int r_bytes = mode == 0 ? (n <= 8 ? kSaCodesN8 : 256) * 16 * 8 + (n <= 8 ? (256 + 32 + 256) * 8 + 256 : 0) : 0;
  const int threads = (mode == 0 && n <= 8) ? kSaThreadsN8 : kSaThreads;
  // psum (Eq.5 sums) cached in shared memory for configs with dp <= dp_cap: the largest cap
  // that still reaches the best achievable number of resident blocks per SM
  const bool nib = false;
  auto warp_bytes_for = [&](int cap, int& tls) {
    int wb = 16;
    tls = 1;
    for (int f = 0; f < F; ++f) {
      const DevCfg& c = ctx->hcfg[ctx->hfeas[f]];
      wb = std::max(wb, sa_warp_state_bytes(mode, c.N, c.pp, c.dp, n, cap, nib));
      tls = std::max(tls, n * (std::min(c.spn, c.dp) - 1));
    }
    return wb;
  };
  const int reg_blocks = mode == 0 ? (n <= 8 ? kSaBlocksN8 : 3) : 2;   // __launch_bounds__
  auto blocks_for = [&](int wb) {
    return std::min(reg_blocks, (227 * 1024) / std::max(1, r_bytes + (threads / 32) * wb));
  };
  int dp_cap = 0, warp_bytes = 16, tl_stride = 1, best_blocks = -1;
  for (int cap : {1024, 64, 32, 16, 8, 4, 2}) {
    int tls;
    const int wb = warp_bytes_for(cap, tls);
    const int b = blocks_for(wb);
    if (b > best_blocks) { best_blocks = b; dp_cap = cap; warp_bytes = wb; tl_stride = tls; }
  }
  if (cap_env) {   // tuning knob
    dp_cap = atoi(cap_env);
    warp_bytes = warp_bytes_for(dp_cap, tl_stride);
  }
  int wpb = threads / 32;
  const int smem_max = 227 * 1024;
  if (r_bytes + warp_bytes > smem_max)
    return fail(ctx, PIPETTE_E_UNSUPPORTED, "SA state (%d B/warp + %d B) exceeds shared memory", warp_bytes, r_bytes);
  while (wpb > 1 && r_bytes + wpb * warp_bytes > smem_max) --wpb;
  const size_t smem = (size_t)r_bytes + (size_t)wpb * warp_bytes;
  // block work units: up to wpb consecutive tasks of one configuration
  std::vector<int2>& chunks = hp.chunks;
  for (size_t i = 0; i < sorted.size();) {
    size_t j = i + 1;
    while (j < sorted.size() && (int)(j - i) < wpb && sorted[j].cfg == sorted[i].cfg) ++j;
    chunks.push_back(make_int2((int)i, (int)(j - i)));
    i = j;
  }

  hp.slots = slots; hp.perm_words = perm_words; hp.maxN = maxN; hp.mode = mode; hp.r_bytes = r_bytes;
  hp.big = false; hp.nib = nib; hp.dp_cap = dp_cap; hp.warp_bytes = warp_bytes; hp.tl_stride = tl_stride; hp.wpb = wpb;
  hp.smem = smem;
  (void)maxdp2;
  return PIPETTE_OK;
}

pipette_status enumerate(pipette_ctx* ctx, const pipette_model* m, long long bs, bool time_it) {
  const bool cached = ctx->enum_valid && std::memcmp(&ctx->enum_model, m, sizeof *m) == 0 && ctx->enum_bs == bs;
  if (cached && !time_it) return PIPETTE_OK;
  const int G = ctx->n_nodes * ctx->g;
  const long long E_cap = (long long)n_div(G) * n_div(ctx->g) * n_div(bs);
  const long long q_cap = E_cap * (G + ctx->n_nodes + 4);
  if (E_cap > (1 << 24) || q_cap > (1ll << 28)) return fail(ctx, PIPETTE_E_UNSUPPORTED, "enumeration too large");
  CU(ensure(ctx->cfgs, sizeof(DevCfg) * E_cap));
  CU(ensure(ctx->keys, sizeof(unsigned long long) * E_cap));
  CU(ensure(ctx->feas, sizeof(int) * E_cap));
  CU(ensure(ctx->qtab, sizeof(double) * q_cap));
  CU(ensure(ctx->eout, sizeof(EnumOut)));
  if (time_it) CU(cudaEventRecord(ctx->ev[0], ctx->stream));
  k_enumerate_filter<<<1, kEnumThreads, 0, ctx->stream>>>(
      ctx->n_nodes, ctx->g, ctx->cap, ctx->margin, *m, bs, ctx->dProf, ctx->n_prof, (DevCfg*)ctx->cfgs.p,
      (unsigned long long*)ctx->keys.p, (int)E_cap, (int*)ctx->feas.p, (double*)ctx->qtab.p, (int)q_cap,
      (EnumOut*)ctx->eout.p);
  ctx->launches++;
  CU(cudaGetLastError());
  if (ctx->mlp.p) {   // NEXT-4: Eq.7's MLP replaces the analytic memory and the verdicts
    launch_mlp_filter((const double*)ctx->mlp.p, G, ctx->n_nodes, *m, bs, ctx->cap, ctx->margin, (DevCfg*)ctx->cfgs.p,
                      (int*)ctx->feas.p, (EnumOut*)ctx->eout.p, ctx->stream);
    ctx->launches++;
    CU(cudaGetLastError());
  }
  if (time_it) CU(cudaEventRecord(ctx->ev[1], ctx->stream));
  // a search re-runs K1 every call (it is step a1-a3 of the path); with the same model and
  // batch its tables are identical, so the host keeps its copy and does not wait for them
  if (cached) return PIPETTE_OK;
  EnumOut eo;
  CU(cudaMemcpyAsync(&eo, ctx->eout.p, sizeof eo, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (eo.overflow) return fail(ctx, PIPETTE_E_UNSUPPORTED, "enumeration capacity exceeded (%d)", eo.overflow);
  ctx->E = eo.E;
  ctx->F = eo.F;
  ctx->hcfg.resize(eo.E);
  ctx->hfeas.resize(eo.F);
  if (eo.E) CU(cudaMemcpy(ctx->hcfg.data(), ctx->cfgs.p, sizeof(DevCfg) * eo.E, cudaMemcpyDeviceToHost));
  if (eo.F) CU(cudaMemcpy(ctx->hfeas.data(), ctx->feas.p, sizeof(int) * eo.F, cudaMemcpyDeviceToHost));
  ctx->enum_valid = true;
  ctx->vin_valid = false;
  ctx->cfg_cost_ms.clear();   // (measured task durations belong to the previous enumeration)
  ctx->plan_valid = false;   // the SA work plan is built from this enumeration
  ctx->enum_model = *m;
  ctx->enum_bs = bs;
  return PIPETTE_OK;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

}  // namespace

extern "C" {

const char* pipette_strerror(pipette_status s) {
  const int i = (int)s;
  return (i >= 0 && i <= 6) ? kStatusText[i] : "unknown status";
}

const char* pipette_last_error(const pipette_ctx* ctx) { return ctx ? ctx->err.c_str() : g_init_err.c_str(); }

int64_t pipette_last_launch_count(const pipette_ctx* ctx) { return ctx ? ctx->launches : 0; }

int32_t pipette_last_search_stats(const pipette_ctx* ctx, int64_t* out, int32_t cap) {
  if (!ctx || !out) return 0;
  const int32_t k = std::min<int32_t>(cap, 7);
  for (int32_t i = 0; i < k; ++i) out[i] = ctx->stats[i];
  return k;
}

int64_t pipette_last_task_profile(pipette_ctx* ctx, uint64_t* out, int64_t cap) {
  if (!ctx || ctx->n_tasks_last <= 0 || !ctx->task_prof.p) return 0;
  const int64_t n = ctx->n_tasks_last;
  if (out && cap > 0) {
    if (cudaMemcpy(out, ctx->task_prof.p, sizeof(uint64_t) * 4 * std::min(n, cap), cudaMemcpyDeviceToHost) != cudaSuccess)
      return -1;
  }
  return n;
}

int64_t pipette_shard_items(int64_t n_items, int32_t rank, int32_t world, int64_t* items, int64_t cap) {
  if (world < 1 || rank < 0 || rank >= world || n_items < 0) return 0;
  int64_t c = 0;
  for (int64_t j = rank; j < n_items; j += world) {  // R18: item j belongs to rank j mod W
    if (items && c < cap) items[c] = j;
    ++c;
  }
  return c;
}

pipette_status pipette_profile_bandwidth(int32_t n_gpus, const int32_t* devices, uint64_t bytes, int32_t reps,
                                         double* bw_out, double* ms_out, char* err, int32_t err_cap) {
  static char dummy[8];
  if (!err || err_cap <= 0) { err = dummy; err_cap = sizeof dummy; }
  err[0] = 0;
  if (n_gpus < 1 || !devices || !bw_out || bytes < 16 || reps < 1) {
    std::snprintf(err, (size_t)err_cap, "n_gpus >= 1, devices, bw_out, bytes >= 16 and reps >= 1 required");
    return PIPETTE_E_INVALID;
  }
  return pip::netprof_run(n_gpus, devices, (size_t)bytes, reps, bw_out, ms_out, err, (size_t)err_cap);
}

pipette_status pipette_set_memory_model(pipette_ctx* ctx, const double* params, int64_t n_params) {
  if (!ctx) return PIPETTE_E_INVALID;
  CU(cudaSetDevice(ctx->device));
  if (!params) {
    if (ctx->mlp.p) cudaFree(ctx->mlp.p);
    ctx->mlp.p = nullptr;
    ctx->mlp.bytes = 0;
  } else {
    if (n_params != kMlpParams)
      return fail(ctx, PIPETTE_E_INVALID, "memory model needs %lld parameters, got %lld", (long long)kMlpParams,
                  (long long)n_params);
    for (int64_t i = 0; i < n_params; ++i)
      if (!std::isfinite(params[i])) return fail(ctx, PIPETTE_E_INVALID, "memory model parameter %lld not finite", (long long)i);
    for (int i = 10; i < 20; ++i)
      if (!(params[i] > 0.0)) return fail(ctx, PIPETTE_E_INVALID, "feature scale %d must be > 0", i - 10);
    CU(ensure(ctx->mlp, sizeof(double) * (size_t)n_params));
    CU(cudaMemcpy(ctx->mlp.p, params, sizeof(double) * (size_t)n_params, cudaMemcpyHostToDevice));
  }
  ctx->enum_valid = false;   // the verdicts change
  ctx->vin_valid = false;
  return PIPETTE_OK;
}

pipette_status pipette_nccl_unique_id(void* id_out) {
  if (!id_out) return PIPETTE_E_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return PIPETTE_E_NCCL;
  std::memcpy(id_out, &id, sizeof id);
  return PIPETTE_OK;
}

pipette_status pipette_init(pipette_ctx** out, const pipette_cluster* cl, const double* bw,
                            const pipette_profile_entry* prof, int32_t n_prof, const pipette_dist* dist) {
  if (!out) return PIPETTE_E_INVALID;
  *out = nullptr;
  pipette_ctx* ctx = new pipette_ctx();
  auto bail = [&](pipette_status s) {
    g_init_err = ctx->err;  // reachable through pipette_last_error(NULL)
    pipette_destroy(ctx);
    return s;
  };
  if (!cl) { fail(ctx, PIPETTE_E_INVALID, "cluster is NULL"); return bail(PIPETTE_E_INVALID); }
  if (cl->n_nodes < 1 || cl->gpus_per_node < 1) { fail(ctx, PIPETTE_E_INVALID, "cluster shape must be >= 1"); return bail(PIPETTE_E_INVALID); }
  // per-node stage-1 member counts are bytes on the device (c_n <= gpus_per_node), so
  // gpus_per_node is limited to 255
  if (cl->n_nodes > kMaxNodes || (long long)cl->n_nodes * cl->gpus_per_node > kMaxGpus ||
      cl->gpus_per_node > kMaxGpusPerNode) {
    fail(ctx, PIPETTE_E_UNSUPPORTED, "v1 supports n_nodes <= %d, gpus_per_node <= %d and G <= %d", kMaxNodes,
         kMaxGpusPerNode, kMaxGpus);
    return bail(PIPETTE_E_UNSUPPORTED);
  }
  if (cl->mem_margin_permille < 0 || cl->mem_margin_permille > 500) { fail(ctx, PIPETTE_E_INVALID, "margin must be in [0, 500] permille"); return bail(PIPETTE_E_INVALID); }
  if (cl->mem_capacity_bytes == 0) { fail(ctx, PIPETTE_E_INVALID, "memory capacity must be > 0"); return bail(PIPETTE_E_INVALID); }
  if (check_bw(ctx, bw, cl->n_nodes) != PIPETTE_OK) return bail(PIPETTE_E_INVALID);
  if (n_prof < 0 || (n_prof > 0 && !prof)) { fail(ctx, PIPETTE_E_INVALID, "bad profile table"); return bail(PIPETTE_E_INVALID); }
  for (int i = 0; i < n_prof; ++i) {
    if (prof[i].tp < 1 || prof[i].mb < 1 || !std::isfinite(prof[i].c_layer_s) || !(prof[i].c_layer_s > 0.0) ||
        !std::isfinite(prof[i].tp_layer_s) || prof[i].tp_layer_s < 0.0) {
      fail(ctx, PIPETTE_E_INVALID, "profile entry %d invalid (tp, mb >= 1; c_layer > 0; tp_layer >= 0)", i);
      return bail(PIPETTE_E_INVALID);
    }
  }
  if (dist && (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world || (dist->world > 1 && !dist->nccl_unique_id && !dist->host_allreduce))) {
    fail(ctx, PIPETTE_E_INVALID, "bad dist description");
    return bail(PIPETTE_E_INVALID);
  }
  ctx->n_nodes = cl->n_nodes;
  ctx->g = cl->gpus_per_node;
  ctx->cap = cl->mem_capacity_bytes;
  ctx->margin = cl->mem_margin_permille;
  ctx->rank = dist ? dist->rank : 0;
  ctx->world = dist ? dist->world : 1;
  ctx->prof.assign(prof, prof + n_prof);
  ctx->n_prof = n_prof;
  pipette_status st;
  {
    int dev = 0;
    if (dist) {
      dev = dist->device;
      if (cudaSetDevice(dev) != cudaSuccess) { fail(ctx, PIPETTE_E_CUDA, "cudaSetDevice(%d) failed", dev); return bail(PIPETTE_E_CUDA); }
    } else if (cudaGetDevice(&dev) != cudaSuccess) {
      fail(ctx, PIPETTE_E_CUDA, "no CUDA device");
      return bail(PIPETTE_E_CUDA);
    }
    ctx->device = dev;
    cudaDeviceGetAttribute(&ctx->n_sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaMalloc(&ctx->dR, sizeof(double) * ctx->n_nodes * ctx->n_nodes) != cudaSuccess ||
        cudaMalloc(&ctx->dProf, sizeof(pipette_profile_entry) * std::max(1, n_prof)) != cudaSuccess) {
      fail(ctx, PIPETTE_E_CUDA, "cudaMalloc failed");
      return bail(PIPETTE_E_CUDA);
    }
    if (n_prof && cudaMemcpy(ctx->dProf, prof, sizeof(pipette_profile_entry) * n_prof, cudaMemcpyHostToDevice) != cudaSuccess) {
      fail(ctx, PIPETTE_E_CUDA, "profile upload failed");
      return bail(PIPETTE_E_CUDA);
    }
    for (auto& e : ctx->ev)
      if (cudaEventCreate(&e) != cudaSuccess) { fail(ctx, PIPETTE_E_CUDA, "event create failed"); return bail(PIPETTE_E_CUDA); }
    if (cudaEventCreateWithFlags(&ctx->ev_tables, cudaEventDisableTiming) != cudaSuccess) {
      fail(ctx, PIPETTE_E_CUDA, "event create failed");
      return bail(PIPETTE_E_CUDA);
    }
    if ((st = upload_bw(ctx, bw)) != PIPETTE_OK) return bail(st);
  }
  if (ctx->world > 1 && !dist->nccl_unique_id) {
    ctx->host_ar = dist->host_allreduce;
    ctx->host_user = dist->host_user;
  } else if (ctx->world > 1) {
    ncclUniqueId id;
    std::memcpy(&id, dist->nccl_unique_id, sizeof id);
    ncclResult_t r = ncclCommInitRank(&ctx->comm, ctx->world, id, ctx->rank);
    if (r != ncclSuccess) { fail(ctx, PIPETTE_E_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)); return bail(PIPETTE_E_NCCL); }
  }
  *out = ctx;
  return PIPETTE_OK;
}

pipette_status pipette_set_bandwidth(pipette_ctx* ctx, const double* bw) {
  if (!ctx) return PIPETTE_E_INVALID;
  pipette_status st = check_bw(ctx, bw, ctx->n_nodes);
  if (st != PIPETTE_OK) return st;
  CU(cudaSetDevice(ctx->device));
  return upload_bw(ctx, bw);   // stream-ordered (tables_begin / tables_end)
}

pipette_status pipette_set_stream(pipette_ctx* ctx, void* stream) {
  if (!ctx) return PIPETTE_E_INVALID;
  ctx->stream = (cudaStream_t)stream;
  return PIPETTE_OK;
}

void pipette_destroy(pipette_ctx* ctx) {
  if (!ctx) return;
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->h_ar) cudaFreeHost(ctx->h_ar);
  DevBuf* bufs[] = {&ctx->cfgs, &ctx->keys, &ctx->feas, &ctx->qtab, &ctx->eout, &ctx->vin, &ctx->mlp, &ctx->claimed, &ctx->tasks, &ctx->chunks, &ctx->counter,
                    &ctx->chain_out, &ctx->best_perm, &ctx->cfg_slot, &ctx->cfg_best, &ctx->gbits, &ctx->items,
                    &ctx->gitems, &ctx->pack, &ctx->accepted, &ctx->slot_perm_off, &ctx->slot_lane,
                    &ctx->trace_slot, &ctx->trace, &ctx->task_prof, &ctx->tin_rank, &ctx->tin_vs, &ctx->tl_ac,
                    &ctx->tl_val, &ctx->tl_len, &ctx->beta0, &ctx->cfg_cost};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  if (ctx->dR) cudaFree(ctx->dR);
  if (ctx->dTab) cudaFree(ctx->dTab);
  if (ctx->dNlNode) cudaFree(ctx->dNlNode);
  if (ctx->dNlVal) cudaFree(ctx->dNlVal);
  if (ctx->dGlAb) cudaFree(ctx->dGlAb);
  if (ctx->dGlVal) cudaFree(ctx->dGlVal);
  if (ctx->dPt) cudaFree(ctx->dPt);
  if (ctx->dProf) cudaFree(ctx->dProf);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->ev_tables) cudaEventDestroy(ctx->ev_tables);
  for (auto& se : ctx->eval_streams) cudaEventDestroy(se.second);
  if (ctx->hR) cudaFreeHost(ctx->hR);
  delete ctx;
}

pipette_status pipette_enumerate(pipette_ctx* ctx, const pipette_model* model, int64_t bs_global, int32_t* E,
                                 int32_t* F, pipette_config* cfgs, int32_t* n_mb, uint64_t* mem_bytes,
                                 uint8_t* feasible, int32_t cap) {
  if (!ctx) return PIPETTE_E_INVALID;
  ctx->launches = 0;
  pipette_status st = check_model(ctx, model, bs_global);
  if (st != PIPETTE_OK) return st;
  CU(cudaSetDevice(ctx->device));
  ctx->enum_valid = false;
  if ((st = enumerate(ctx, model, bs_global, false)) != PIPETTE_OK) return st;
  if (E) *E = ctx->E;
  if (F) *F = ctx->F;
  for (int e = 0; e < std::min(ctx->E, (int)std::max(cap, 0)); ++e) {
    const DevCfg& c = ctx->hcfg[e];
    if (cfgs) { cfgs[e].pp = (uint16_t)c.pp; cfgs[e].tp = (uint16_t)c.tp; cfgs[e].dp = (uint16_t)c.dp; cfgs[e].mb = (uint16_t)c.mb; }
    if (n_mb) n_mb[e] = c.n_mb;
    if (mem_bytes) mem_bytes[e] = c.mem;
    if (feasible) feasible[e] = (uint8_t)c.feasible;
  }
  return PIPETTE_OK;
}

pipette_status pipette_eval(pipette_ctx* ctx, const pipette_model* model, int64_t bs_global, int64_t n,
                            const pipette_config* d_cfg, const uint16_t* d_perm, int32_t perm_stride,
                            double* d_latency, uint64_t* d_mem, uint8_t* d_status, void* stream) {
  if (!ctx) return PIPETTE_E_INVALID;
  ctx->launches = 0;
  pipette_status st = check_model(ctx, model, bs_global);
  if (st != PIPETTE_OK) return st;
  if (n < 0 || perm_stride < 1) return fail(ctx, PIPETTE_E_INVALID, "n >= 0 and perm_stride >= 1 required");
  if (n == 0) return PIPETTE_OK;
  if (!d_cfg || !d_perm || !d_latency || !d_mem || !d_status) return fail(ctx, PIPETTE_E_INVALID, "null device pointer");
  CU(cudaSetDevice(ctx->device));
  if ((st = enumerate(ctx, model, bs_global, false)) != PIPETTE_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  int maxN = 1;
  for (const DevCfg& c : ctx->hcfg) maxN = std::max(maxN, c.N);
  const int mode = (ctx->n_nodes <= 16 && ctx->g <= 15 && ctx->dTab) ? 0 : 1;
  EvalParams P{};
  P.cfgs = (const DevCfg*)ctx->cfgs.p;
  P.keys = (const unsigned long long*)ctx->keys.p;
  P.E = ctx->E;
  P.qtab = (const double*)ctx->qtab.p;
  P.R = ctx->dR;
  P.subset_max = ctx->dTab;
  if (mode == 0 && !ctx->vin_valid) {   // a table rewrite: ordered on ctx->stream after evals in flight
    CU(ensure(ctx->vin, sizeof(double) * 256 * (size_t)std::max(1, ctx->E)));
    CU(tables_begin(ctx));
    k_tin_values<<<std::max(1, ctx->E), 256, 0, ctx->stream>>>((const DevCfg*)ctx->cfgs.p, (const double*)ctx->qtab.p,
                                                              ctx->dR, ctx->n_nodes, (double*)ctx->vin.p);
    ctx->launches++;
    CU(cudaGetLastError());
    CU(tables_end(ctx));
    ctx->vin_valid = true;
  }
  P.vin = (const double*)ctx->vin.p;
  P.gl_ab = ctx->dGlAb;
  P.gl_val = ctx->dGlVal;
  P.n_nodes = ctx->n_nodes;
  P.n = n;
  P.cand = d_cfg;
  P.perm = d_perm;
  P.perm_stride = perm_stride;
  P.vec16 = ((uintptr_t)d_perm % 16 == 0) && (perm_stride % 8 == 0);
  P.bm_words = (std::min(maxN, (int)perm_stride) + 31) / 32;   // (a row longer than perm_stride gets status 3)
  P.latency = d_latency;
  P.mem = (unsigned long long*)d_mem;
  P.status = d_status;
  if (ctx->E >= 32767) return fail(ctx, PIPETTE_E_UNSUPPORTED, "eval supports < 32767 enumerated configurations");
  const void* kern;
  size_t smem;
  int threads, grid, occ = 0;
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof tmap);
  P.tma = 0;
  // K2 path: one thread per candidate, in blocks of 768 for n >= 64 (the R table of up to
  // 128 KB leaves one block per SM; nibble counts, a bitmap sized by perm_stride and the
  // pair-list prefix in shared memory keep 24 warps resident) -- measured on C5 1.2e9 vs
  // 8.1e8 candidates/s for one warp per candidate (k_eval_warp) and 5.6e8 with 8 warps.
  // Knobs: PIPETTE_EVAL_THREAD=0 (warp path) / 1 (thread), PIPETTE_EVAL_THREADS=256/768.
  const char* thr_env = getenv("PIPETTE_EVAL_THREAD");
  const char* thn_env = getenv("PIPETTE_EVAL_THREADS");
  const bool warp_path = mode == 1 && thr_env && atoi(thr_env) == 0;
  P.cnt_nib = ctx->g <= 15 ? 1 : 0;   // (a stage-1 count never exceeds gpus_per_node)
  P.plen = mode == 1 ? std::min(ctx->n_nodes * (ctx->n_nodes - 1), kSaM1PairPrefix) : 0;
  int eval_threads = (mode == 1 && ctx->n_nodes >= 64) ? 768 : 256;
  if (thn_env && (atoi(thn_env) == 256 || (atoi(thn_env) == 768 && mode == 1))) eval_threads = atoi(thn_env);
  if (warp_path) {
    // large clusters: one warp per candidate (k_eval_warp)
    kern = eval_warp_kernel();
    threads = eval_warp_threads();
    smem = eval_warp_smem_bytes(ctx->n_nodes, ctx->E);
    if (smem > 227 * 1024) return fail(ctx, PIPETTE_E_UNSUPPORTED, "eval shared memory %zu B too large", smem);
    if ((st = kernel_occupancy(ctx, kern, threads, smem, &occ)) != PIPETTE_OK) return st;
    const long long need = (n + threads / 32 - 1) / (threads / 32);
    grid = (int)std::min<long long>(need, (long long)occ * ctx->n_sms);
  } else {
    // rows gathered into per-warp shared staging buffers when they are 16-byte aligned and
    // the buffers fit beside the tables (else read straight from global memory)
    smem = eval_smem_bytes(mode, perm_stride, P.vec16 != 0, ctx->n_nodes, ctx->E, P.bm_words, eval_threads,
                           P.cnt_nib != 0, P.plen);
    P.staged = P.vec16 && perm_stride <= 64 && smem <= 96 * 1024;   // long rows: direct 16-byte loads measured faster
    if (!P.staged)
      smem = eval_smem_bytes(mode, perm_stride, false, ctx->n_nodes, ctx->E, P.bm_words, eval_threads,
                             P.cnt_nib != 0, P.plen);
    if (eval_threads == 768 && smem > 227 * 1024) {   // (does not fit: the 256-thread block)
      eval_threads = 256;
      smem = eval_smem_bytes(mode, perm_stride, false, ctx->n_nodes, ctx->E, P.bm_words, eval_threads,
                             P.cnt_nib != 0, P.plen);
    }
    // single-configuration tiles of 128-byte rows: TMA tensor copies (SWIZZLE_128B) instead of
    // per-lane cp.async (PIPETTE_EVAL_TMA=0 disables)
    const char* tma_env = getenv("PIPETTE_EVAL_TMA");
    if (P.staged && perm_stride == 64 && !(tma_env && atoi(tma_env) == 0)) {
      if (PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder()) {
        cuuint64_t dims[2] = {64, (cuuint64_t)n};
        cuuint64_t strides[1] = {128};
        cuuint32_t box[2] = {64, 32}, estr[2] = {1, 1};
        if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, (void*)d_perm, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
          P.tma = 1;
          smem += 1024;   // (1024-byte alignment of the staging buffers)
        }
      }
    }
    if (smem > 227 * 1024) return fail(ctx, PIPETTE_E_UNSUPPORTED, "eval shared memory %zu B too large", smem);
    kern = eval_kernel(mode, eval_threads);
    threads = eval_threads;
    if ((st = kernel_occupancy(ctx, kern, threads, smem, &occ)) != PIPETTE_OK) return st;
    const long long need = (n + eval_tile_size() - 1) / eval_tile_size();   // candidate tiles
    grid = (int)std::min<long long>(need, (long long)occ * ctx->n_sms);
  }
  void* args_thread[] = {&P, &tmap};
  void* args_warp[] = {&P};
  void** args = warp_path ? args_warp : args_thread;
  nvtxRangePushA("pipette_eval K2");
  CU(wait_tables(ctx, s));
  CU(cudaLaunchKernel(kern, dim3(grid), dim3(threads), args, smem, s));
  ctx->launches++;
  CU(cudaGetLastError());
  CU(note_eval(ctx, s));
  nvtxRangePop();
  return PIPETTE_OK;
}

pipette_status pipette_eval_models(pipette_ctx* ctx, const pipette_model* model, int64_t bs_global, int64_t n,
                                   const pipette_config* d_cfg, const uint16_t* d_perm, int32_t perm_stride,
                                   double* d_t_pipette, double* d_t_prev, double* d_t_des, uint8_t* d_status,
                                   void* stream) {
  if (!ctx) return PIPETTE_E_INVALID;
  ctx->launches = 0;
  pipette_status st = check_model(ctx, model, bs_global);
  if (st != PIPETTE_OK) return st;
  if (n < 0 || perm_stride < 1) return fail(ctx, PIPETTE_E_INVALID, "n >= 0 and perm_stride >= 1 required");
  if (n == 0) return PIPETTE_OK;
  if (!d_cfg || !d_perm || !d_t_pipette || !d_t_prev || !d_t_des || !d_status)
    return fail(ctx, PIPETTE_E_INVALID, "null device pointer");
  CU(cudaSetDevice(ctx->device));
  if ((st = enumerate(ctx, model, bs_global, false)) != PIPETTE_OK) return st;
  CU(wait_tables(ctx, (cudaStream_t)stream));
  st = models_launch((const DevCfg*)ctx->cfgs.p, (const unsigned long long*)ctx->keys.p, ctx->E,
                     (const double*)ctx->qtab.p, ctx->dR, ctx->n_nodes, n, d_cfg, d_perm, perm_stride, d_t_pipette,
                     d_t_prev, d_t_des, d_status, stream);
  ctx->launches++;
  if (st != PIPETTE_OK) return fail(ctx, st, "k_models launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  CU(note_eval(ctx, (cudaStream_t)stream));
  return PIPETTE_OK;
}

pipette_status pipette_search(pipette_ctx* ctx, const pipette_model* model, int64_t bs_global,
                              int32_t chains, int32_t iterations, uint64_t seed, const pipette_sa_opts* opts,
                              pipette_plan* out, pipette_plan* per_config, int32_t per_config_cap) {
  if (!ctx) return PIPETTE_E_INVALID;
  ctx->launches = 0;
  pipette_status st = check_model(ctx, model, bs_global);
  if (st != PIPETTE_OK) return st;
  if (!out) return fail(ctx, PIPETTE_E_INVALID, "out is NULL");
  if (chains < 1 || iterations < 0) return fail(ctx, PIPETTE_E_INVALID, "chains >= 1 and iterations >= 0 required");
  pipette_sa_opts o{};
  o.alpha = 0.999;
  o.tau = 0.05;
  if (opts) o = *opts;
  if (!(o.alpha > 0.0 && o.alpha <= 1.0)) return fail(ctx, PIPETTE_E_INVALID, "alpha must be in (0, 1]");
  if (!(o.t0 > 0.0) && !(o.tau > 0.0)) return fail(ctx, PIPETTE_E_INVALID, "tau > 0 or t0 > 0 required");
  if (o.w_migrate < 0 || o.w_reverse < 0 || o.w_migrate + o.w_reverse > 2048)
    return fail(ctx, PIPETTE_E_INVALID, "move weights must satisfy 0 <= w_migrate, w_reverse and sum <= 2048");
  CU(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  nvtxRangePushA("pipette_search");
  struct NvtxPop { ~NvtxPop() { nvtxRangePop(); } } nvtx_pop_;   // (every return path)

  CU(wait_tables(ctx, s));   // (the stream may have changed since the last table update)
  nvtxRangeId_t nv = nvtxRangeStartA("K1 enumerate + memory filter");
  if ((st = enumerate(ctx, model, bs_global, true)) != PIPETTE_OK) return st;
  nvtxRangeEnd(nv);
  const int E = ctx->E, F = ctx->F;
  out->configs_enumerated = E;
  out->configs_rejected_oom = E - F;
  out->sa_steps = out->sa_accepted = 0;
  if (F == 0) return fail(ctx, PIPETTE_NO_FEASIBLE, "all %d configurations exceed the memory limit", E);
  for (int f = 0; f < F; ++f) {
    const DevCfg& c = ctx->hcfg[ctx->hfeas[f]];
    if (!c.has_profile)
      return fail(ctx, PIPETTE_E_PROFILE, "no profile entry for tp=%d mb=%d (feasible config e=%d)", c.tp, c.mb, c.e);
  }

  // ---- the host-side work plan (work items, warp tasks, block chunks, kernel variant and
  //      shared-memory layout) depends only on the enumeration and (chains, world, rank):
  //      it is rebuilt only when those change
  const int W = ctx->world, r = ctx->rank;
  const char* cap_env = getenv("PIPETTE_DP_CAP");
  HostPlanKey key{};
  key.model = *model; key.bs = bs_global; key.chains = chains; key.W = W; key.r = r;
  key.dp_cap_env = cap_env ? atoi(cap_env) : -1;
  key.full_moves = (o.w_migrate || o.w_reverse) ? 1 : 0;
  if (!(ctx->plan_valid && std::memcmp(&ctx->plan_key, &key, sizeof key) == 0)) {
    ctx->plan_valid = false;
    HostPlan& np_ = ctx->plan;
    np_ = HostPlan{};
    pipette_status pst = build_plan(ctx, chains, W, r, cap_env, key.full_moves != 0, np_);
    if (pst != PIPETTE_OK) return pst;
    ctx->plan_key = key;
    ctx->plan_valid = true;
  }
  const HostPlan& pl = ctx->plan;
  const std::vector<SaTask>& sorted = pl.sorted;
  const std::vector<int2>& chunks = pl.chunks;
  const std::vector<int>& cfg_slot = pl.cfg_slot;
  const std::vector<int>& slot_perm_off = pl.slot_perm_off;
  const std::vector<int>& slot_lane = pl.slot_lane;
  const int slots = pl.slots, perm_words = pl.perm_words, maxN = pl.maxN, mode = pl.mode, n = ctx->n_nodes;
  const int r_bytes = pl.r_bytes, dp_cap = pl.dp_cap, warp_bytes = pl.warp_bytes, tl_stride = pl.tl_stride;
  const int wpb = pl.wpb;
  const size_t smem = pl.smem;
  (void)maxN;
  uint64_t steps = 0;
  for (int f = 0; f < F; ++f)
    if (ctx->hcfg[ctx->hfeas[f]].N >= 2) steps += (uint64_t)chains * (uint64_t)iterations;
  out->sa_steps = steps;

  const bool tracing = o.trace && o.trace_items && o.n_trace > 0 && o.trace_cap > 0;
  std::vector<int> trace_slot;
  if (tracing) {
    trace_slot.assign(std::max(slots, 1), -1);
    for (int t = 0; t < o.n_trace; ++t) {
      const int64_t j = o.trace_items[t];
      if (j < 0 || j >= (int64_t)F * chains || j % W != r) continue;
      const int f = (int)(j / chains), c = (int)(j % chains);
      const long long base = (long long)f * chains;
      const int c_first = (int)(((r - base) % W + W) % W);
      trace_slot[cfg_slot[f] + (c - c_first) / W] = t;
    }
  }

  CU(ensure_up(ctx->tasks, sizeof(SaTask) * std::max<size_t>(1, sorted.size()), ctx->up_tasks));
  CU(ensure_up(ctx->chunks, sizeof(int2) * std::max<size_t>(1, chunks.size()), ctx->up_chunks));
  CU(ensure(ctx->counter, sizeof(int)));
  CU(ensure(ctx->task_prof, sizeof(unsigned long long) * 4 * std::max<size_t>(1, sorted.size())));
  ctx->n_tasks_last = (int64_t)sorted.size();
  CU(ensure(ctx->chain_out, sizeof(ChainOut) * std::max(1, slots)));
  CU(ensure(ctx->best_perm, sizeof(uint16_t) * std::max(1, perm_words)));
  CU(ensure_up(ctx->cfg_slot, sizeof(int) * (F + 1), ctx->up_cfg_slot));
  CU(ensure_up(ctx->slot_perm_off, sizeof(int) * std::max(1, slots), ctx->up_slot_perm_off));
  CU(ensure_up(ctx->slot_lane, sizeof(int) * std::max(1, slots), ctx->up_slot_lane));
  CU(ensure(ctx->cfg_best, sizeof(CfgBest) * F));
  CU(ensure(ctx->gbits, sizeof(unsigned long long) * F));
  CU(ensure(ctx->items, sizeof(unsigned long long) * F));
  CU(ensure(ctx->gitems, sizeof(unsigned long long) * F));
  const int row_words = 4 + (maxN + 3) / 4;
  CU(ensure(ctx->pack, sizeof(unsigned long long) * ((size_t)F * row_words + 1)));
  // the work lists of the previous call are still on the device: upload only what changed
  auto upload = [&](std::vector<unsigned char>& last, DevBuf& dst, const void* src, size_t bytes) -> cudaError_t {
    if (bytes == 0) return cudaSuccess;
    if (last.size() == bytes && std::memcmp(last.data(), src, bytes) == 0) return cudaSuccess;
    last.assign((const unsigned char*)src, (const unsigned char*)src + bytes);
    return cudaMemcpyAsync(dst.p, last.data(), bytes, cudaMemcpyHostToDevice, s);
  };
  CU(upload(ctx->up_tasks, ctx->tasks, sorted.data(), sizeof(SaTask) * sorted.size()));
  CU(upload(ctx->up_chunks, ctx->chunks, chunks.data(), sizeof(int2) * chunks.size()));
  CU(upload(ctx->up_cfg_slot, ctx->cfg_slot, cfg_slot.data(), sizeof(int) * (F + 1)));
  CU(upload(ctx->up_slot_perm_off, ctx->slot_perm_off, slot_perm_off.data(), sizeof(int) * slots));
  CU(upload(ctx->up_slot_lane, ctx->slot_lane, slot_lane.data(), sizeof(int) * slots));
  CU(cudaMemsetAsync(ctx->counter.p, 0, sizeof(int), s));
  CU(ensure(ctx->claimed, sizeof(int) * (std::max<size_t>(1, chunks.size()) + 1024)));
  CU(cudaMemsetAsync(ctx->claimed.p, 0, sizeof(int) * (std::max<size_t>(1, chunks.size()) + 1024), s));
  if (tracing) {
    CU(ensure(ctx->trace_slot, sizeof(int) * trace_slot.size()));
    CU(ensure(ctx->trace, sizeof(pipette_trace_record) * (size_t)o.n_trace * o.trace_cap));
    CU(cudaMemcpyAsync(ctx->trace_slot.p, trace_slot.data(), sizeof(int) * trace_slot.size(), cudaMemcpyHostToDevice, s));
    CU(cudaMemsetAsync(ctx->trace.p, 0, sizeof(pipette_trace_record) * (size_t)o.n_trace * o.trace_cap, s));
  }

  if (mode == 0) {   // T_in rank tables of every feasible config (S1Reg)
    CU(ensure(ctx->tin_rank, (size_t)F * 256));
    CU(ensure(ctx->tin_vs, sizeof(double) * (size_t)F * 256));
  } else {           // sorted T_in lists of every feasible config (S1Large)
    CU(ensure(ctx->tl_ac, sizeof(uint16_t) * (size_t)F * tl_stride));
    CU(ensure(ctx->tl_val, sizeof(double) * (size_t)F * tl_stride));
    CU(ensure(ctx->tl_len, sizeof(int) * (size_t)F));
  }
  SaParams P{};
  P.cfgs = (const DevCfg*)ctx->cfgs.p;
  P.qtab = (const double*)ctx->qtab.p;
  P.R = ctx->dR;
  P.subset_max = ctx->dTab;
  P.tin_rank = mode == 0 ? (const uint8_t*)ctx->tin_rank.p : nullptr;
  P.tin_vs = mode == 0 ? (const double*)ctx->tin_vs.p : nullptr;
  P.nl_node = ctx->dNlNode;
  P.nl_val = ctx->dNlVal;
  P.gl_ab = ctx->dGlAb;
  P.gl_val = ctx->dGlVal;
  P.tl_ac = mode != 0 ? (const uint16_t*)ctx->tl_ac.p : nullptr;
  P.tl_val = mode != 0 ? (const double*)ctx->tl_val.p : nullptr;
  P.tl_len = mode != 0 ? (const int*)ctx->tl_len.p : nullptr;
  P.tl_stride = tl_stride;
  P.psum_dp_cap = dp_cap;
  P.tasks = (const SaTask*)ctx->tasks.p;
  P.n_tasks = (int)sorted.size();
  P.chunks = (const int2*)ctx->chunks.p;
  P.n_chunks = (int)chunks.size();
  P.task_counter = (int*)ctx->counter.p;
  P.claimed = (int*)ctx->claimed.p;
  P.sm_slot = (int*)ctx->claimed.p + std::max<size_t>(1, chunks.size());   // 1024 per-SM slots after the flags
  P.n_sms = ctx->n_sms;
  P.n_nodes = n;
  P.iterations = iterations;
  P.key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  P.rk = philox_round_keys(P.key);
  P.world = W;
  P.alpha_inv = 1.0 / o.alpha;
  P.tau = o.tau;
  P.t0 = o.t0 > 0.0 ? o.t0 : 0.0;
  P.warps_per_block = wpb;
  P.warp_smem_bytes = warp_bytes;
  P.r_smem_bytes = r_bytes;
  P.out = (ChainOut*)ctx->chain_out.p;
  P.best_perm = (uint16_t*)ctx->best_perm.p;
  P.task_prof = (unsigned long long*)ctx->task_prof.p;
  P.trace_slot = tracing ? (const int*)ctx->trace_slot.p : nullptr;
  P.trace_cap = tracing ? o.trace_cap : 0;
  P.trace = tracing ? (pipette_trace_record*)ctx->trace.p : nullptr;
  P.w_migrate = o.w_migrate;
  P.w_reverse = o.w_reverse;
  P.s1_nib = pl.nib ? 1 : 0;
  P.r_lg = pl.r_lg;
  P.pt = ctx->dPt;
  P.pt_stride = ctx->pt_stride;
  P.plen = pl.plen;

  const void* kern = sa_kernel(mode, tracing, n, o.w_migrate || o.w_reverse);
  int occ = 0;
  if ((st = kernel_occupancy(ctx, kern, wpb * 32, smem, &occ)) != PIPETTE_OK) return st;
  const int grid = (int)std::max<long long>(1, std::min<long long>((long long)chunks.size(), (long long)occ * ctx->n_sms));
  ctx->stats[0] = mode; ctx->stats[1] = (int64_t)sorted.size(); ctx->stats[2] = (int64_t)chunks.size();
  ctx->stats[3] = grid; ctx->stats[4] = wpb; ctx->stats[5] = (int64_t)smem; ctx->stats[6] = r_bytes;
  nv = nvtxRangeStartA("K3 sa_chains (+ T_in lists, T0 calibration)");
  CU(cudaEventRecord(ctx->ev[2], s));
  if (mode == 0) {
    k_tin_rank<<<F, 256, 0, s>>>((const DevCfg*)ctx->cfgs.p, (const int*)ctx->feas.p, (const double*)ctx->qtab.p,
                                 ctx->dR, n, (uint8_t*)ctx->tin_rank.p, (double*)ctx->tin_vs.p);
  } else {
    k_tin_list<<<F, 256, 0, s>>>((const DevCfg*)ctx->cfgs.p, (const int*)ctx->feas.p, (const double*)ctx->qtab.p,
                                 ctx->dR, n, tl_stride, (uint16_t*)ctx->tl_ac.p, (double*)ctx->tl_val.p,
                                 (int*)ctx->tl_len.p);
  }
  ctx->launches++;
  CU(cudaGetLastError());
  if (o.t0 < 0.0) {   // R24: self-calibrated 1/T0 per feasible configuration
    CU(ensure(ctx->beta0, sizeof(double) * (size_t)F));
    launch_t0_calibrate((const DevCfg*)ctx->cfgs.p, (const int*)ctx->feas.p, F, (const double*)ctx->qtab.p, ctx->dR, n,
                        P.rk, o.w_migrate, o.w_reverse, o.tau, (double*)ctx->beta0.p, s);
    ctx->launches++;
    CU(cudaGetLastError());
    P.beta0 = (const double*)ctx->beta0.p;
  }
  if (!sorted.empty()) {
    void* args[] = {&P};
    CU(cudaLaunchKernel(kern, dim3(grid), dim3(wpb * 32), args, smem, s));
    ctx->launches++;
    CU(cudaGetLastError());
  }
  const bool learn_costs = !pl.measured && !sorted.empty() && mode != 0;   // (once per work plan)
  if (learn_costs) {
    CU(ensure(ctx->cfg_cost, sizeof(unsigned long long) * 2 * (size_t)E));
    CU(cudaMemsetAsync(ctx->cfg_cost.p, 0, sizeof(unsigned long long) * 2 * (size_t)E, s));
    k_cfg_cost<<<(unsigned)((sorted.size() + 255) / 256), 256, 0, s>>>(
        (const unsigned long long*)ctx->task_prof.p, (const SaTask*)ctx->tasks.p, (int)sorted.size(),
        (unsigned long long*)ctx->cfg_cost.p);
    ctx->launches++;
    CU(cudaGetLastError());
  }
  CU(cudaEventRecord(ctx->ev[3], s));
  nvtxRangeEnd(nv);
  nv = nvtxRangeStartA("K4 argmin");
  k_argmin<<<F, 256, 0, s>>>((const ChainOut*)ctx->chain_out.p, (const int*)ctx->cfg_slot.p, F,
                              (CfgBest*)ctx->cfg_best.p);
  ctx->launches++;
  CU(cudaGetLastError());
  CU(cudaEventRecord(ctx->ev[4], s));
  nvtxRangeEnd(nv);
  nv = nvtxRangeStartA("combine (NCCL allreduce min, min, sum)");

  // ---- combine (R18): min latency bits, then min item among ranks attaining it, then
  //      the owners' plans (one fused allreduce(sum) of owner-only rows)
  unsigned long long* gbits = (unsigned long long*)ctx->gbits.p;
  unsigned long long* items = (unsigned long long*)ctx->items.p;
  unsigned long long* gitems = (unsigned long long*)ctx->gitems.p;
  unsigned long long* pack = (unsigned long long*)ctx->pack.p;
  // local latency bits of each config (ChainOut.best is the first field of CfgBest)
  CU(cudaMemcpy2DAsync(gbits, sizeof(unsigned long long), ctx->cfg_best.p, sizeof(CfgBest),
                       sizeof(unsigned long long), F, cudaMemcpyDeviceToDevice, s));
  if (W > 1 && (st = allreduce_u64(ctx, gbits, gbits, F, 0, s)) != PIPETTE_OK) return st;
  k_combine_items<<<(F + 127) / 128, 128, 0, s>>>((const CfgBest*)ctx->cfg_best.p, gbits, F, chains, items);
  ctx->launches++;
  if (W > 1) {
    if ((st = allreduce_u64(ctx, items, gitems, F, 0, s)) != PIPETTE_OK) return st;
  } else CU(cudaMemcpyAsync(gitems, items, sizeof(unsigned long long) * F, cudaMemcpyDeviceToDevice, s));
  k_combine_pack<<<F, 128, 0, s>>>((const CfgBest*)ctx->cfg_best.p, gitems, (const DevCfg*)ctx->cfgs.p,
                                    (const int*)ctx->feas.p, (const int*)ctx->slot_perm_off.p,
                                    (const int*)ctx->slot_lane.p, (const uint16_t*)ctx->best_perm.p, F, chains,
                                    row_words, pack);
  ctx->launches++;
  k_sum_accepted<<<1, 32, 0, s>>>((const CfgBest*)ctx->cfg_best.p, F, pack + (size_t)F * row_words);
  ctx->launches++;
  CU(cudaGetLastError());
  if (W > 1 && (st = allreduce_u64(ctx, pack, pack, (size_t)F * row_words + 1, 1, s)) != PIPETTE_OK) return st;
  CU(cudaEventRecord(ctx->ev[5], s));
  nvtxRangeEnd(nv);

  std::vector<unsigned long long> hb(F), hi(F), hp((size_t)F * row_words + 1);
  CU(cudaMemcpyAsync(hb.data(), gbits, sizeof(unsigned long long) * F, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(hi.data(), gitems, sizeof(unsigned long long) * F, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(hp.data(), pack, sizeof(unsigned long long) * hp.size(), cudaMemcpyDeviceToHost, s));
  std::vector<ChainOut> hco;
  std::vector<uint16_t> hperm;
  if (o.chains && o.chains_cap > 0 && slots > 0) {
    hco.resize(slots);
    CU(cudaMemcpyAsync(hco.data(), ctx->chain_out.p, sizeof(ChainOut) * slots, cudaMemcpyDeviceToHost, s));
    if (o.chain_perms) {
      hperm.resize(perm_words);
      CU(cudaMemcpyAsync(hperm.data(), ctx->best_perm.p, sizeof(uint16_t) * perm_words, cudaMemcpyDeviceToHost, s));
    }
  }
  std::vector<unsigned long long> hcost;
  if (learn_costs) {
    hcost.resize(2 * (size_t)E);
    CU(cudaMemcpyAsync(hcost.data(), ctx->cfg_cost.p, sizeof(unsigned long long) * hcost.size(), cudaMemcpyDeviceToHost, s));
  }
  std::vector<pipette_trace_record> htr;
  if (tracing) {
    htr.resize((size_t)o.n_trace * o.trace_cap);
    CU(cudaMemcpyAsync(htr.data(), ctx->trace.p, sizeof(pipette_trace_record) * htr.size(), cudaMemcpyDeviceToHost, s));
  }
  CU(cudaStreamSynchronize(s));
  if (learn_costs) {   // the next call orders its tasks by these measured durations
    ctx->cfg_cost_ms.assign(E, 0.0);
    for (int e = 0; e < E; ++e)
      if (hcost[2 * e + 1]) ctx->cfg_cost_ms[e] = (double)hcost[2 * e] / (double)hcost[2 * e + 1] * 1e-6;
    ctx->plan_valid = false;
  }
  out->enumerate_ms = elapsed(ctx->ev[0], ctx->ev[1]);
  out->sa_ms = elapsed(ctx->ev[2], ctx->ev[3]);
  out->argmin_ms = elapsed(ctx->ev[3], ctx->ev[4]);
  out->combine_ms = elapsed(ctx->ev[4], ctx->ev[5]);
  out->sa_accepted = hp[(size_t)F * row_words];

  // ---- assemble plans on the host from the combined rows (identical on every rank)
  auto fill = [&](int f, pipette_plan* p) -> pipette_status {
    const DevCfg& c = ctx->hcfg[ctx->hfeas[f]];
    const unsigned long long* row = hp.data() + (size_t)f * row_words;
    p->cfg.pp = (uint16_t)c.pp; p->cfg.tp = (uint16_t)c.tp; p->cfg.dp = (uint16_t)c.dp; p->cfg.mb = (uint16_t)c.mb;
    p->n_mb = c.n_mb;
    double v;
    std::memcpy(&v, &hb[f], 8); p->latency_s = v;
    std::memcpy(&v, &row[0], 8); p->t_pp = v;
    std::memcpy(&v, &row[1], 8); p->t_dp = v;
    std::memcpy(&v, &row[2], 8); p->t_bubble = v;
    p->t_straggler = c.Ss;
    p->best_step = (int32_t)((long long)row[3] - 1);
    p->mem_bytes = c.mem;
    p->cfg_index = c.e;
    p->chain = (int32_t)(hi[f] % (unsigned long long)chains);
    p->n_slots = c.N;
    if (!p->perm || p->perm_cap < c.N) return fail(ctx, PIPETTE_E_INVALID, "plan perm buffer needs %d entries", c.N);
    for (int w = 0; w < c.N; ++w) p->perm[w] = (uint16_t)(row[4 + w / 4] >> (16 * (w % 4)));
    return PIPETTE_OK;
  };
  int fw = 0;
  for (int f = 1; f < F; ++f)
    if (hb[f] < hb[fw]) fw = f;  // lexicographic (T, e, c): ties keep the lower f (R17)
  const uint64_t keep_steps = out->sa_steps, keep_acc = out->sa_accepted;
  const double t_en = out->enumerate_ms, t_sa = out->sa_ms, t_am = out->argmin_ms, t_cb = out->combine_ms;
  out->n_slots = ctx->hcfg[ctx->hfeas[fw]].N;
  if ((st = fill(fw, out)) != PIPETTE_OK) return st;
  out->configs_enumerated = E; out->configs_rejected_oom = E - F;
  out->sa_steps = keep_steps; out->sa_accepted = keep_acc;
  out->enumerate_ms = t_en; out->sa_ms = t_sa; out->argmin_ms = t_am; out->combine_ms = t_cb;
  if (per_config && per_config_cap > 0) {
    std::vector<int> ord(F);
    for (int f = 0; f < F; ++f) ord[f] = f;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return hb[a] < hb[b]; });
    for (int i = 0; i < std::min(F, per_config_cap); ++i) {
      pipette_plan* p = &per_config[i];
      if ((st = fill(ord[i], p)) != PIPETTE_OK) return st;
      p->configs_enumerated = E; p->configs_rejected_oom = E - F; p->sa_steps = keep_steps; p->sa_accepted = keep_acc;
    }
  }
  // ---- diagnostics: per-chain results and traces of this rank's items
  if (!hco.empty()) {
    for (int sidx = 0; sidx < slots; ++sidx) {
      const ChainOut& co = hco[sidx];
      const int64_t j = (int64_t)co.f * chains + co.c;
      if (j >= o.chains_cap) continue;
      pipette_chain_result& cr = o.chains[j];
      const DevCfg& c = ctx->hcfg[ctx->hfeas[co.f]];
      cr.best = co.best; cr.best_t_pp = co.best_tpp; cr.best_t_dp = co.best_tdp; cr.L0 = co.L0;
      cr.best_step = co.best_step; cr.accepted = co.accepted; cr.cfg_index = c.e; cr.chain = co.c;
      cr.rank = r; cr.n_slots = c.N;
      if (o.chain_perms && o.chain_perm_stride >= c.N)
        for (int w = 0; w < c.N; ++w)
          o.chain_perms[j * o.chain_perm_stride + w] = hperm[slot_perm_off[sidx] + w * 32 + slot_lane[sidx]];
    }
  }
  if (tracing) {
    for (int t = 0; t < o.n_trace; ++t) {
      const int64_t j = o.trace_items[t];
      if (j < 0 || j >= (int64_t)F * chains || j % W != r) continue;
      std::memcpy(o.trace + (size_t)t * o.trace_cap, htr.data() + (size_t)t * o.trace_cap,
                  sizeof(pipette_trace_record) * o.trace_cap);
    }
  }
  return PIPETTE_OK;
}

}  // extern "C"
