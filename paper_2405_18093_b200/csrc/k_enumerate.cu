// k_enumerate.cu -- K1: device-side configuration enumerator + memory filter +
// per-config constants.
//
// Alg.1 l.3-5: all (pp, tp, dp, bs_micro) with pp*tp*dp = G, tp | g (R1),
// pp <= n_layers (R2), dp | bs_global (l.4), bs_micro | bs_mini (l.5), in canonical order
// pp ascending, tp ascending, bs_micro ascending.  Alg.1 l.7 with the soft
// margin of P:370 (R12) on the analytic memory estimate of R11.  One block; E is a few
// hundred at most, so this kernel is launch-latency bound.
#include "devmath.cuh"
#include "pipette_dev.cuh"

namespace pip {

constexpr int kEnumThreads = 1024;

// Exclusive block-wide scan of one int per thread; `total` = sum over the block.
__device__ int block_scan_excl(int v, int* sh, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < nw ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sh[lane] = s;
  }
  __syncthreads();
  const int excl = x - v + (wid > 0 ? sh[wid - 1] : 0);
  total = sh[nw - 1];
  __syncthreads();
  return excl;
}

__device__ __forceinline__ unsigned long long ceil_div_u64(unsigned long long a, unsigned long long b) {
  return (a + b - 1) / b;
}

// Per-GPU memory of stage 1 (R11): parameters + gradients + Adam state of the stage's
// layers and embeddings, plus min(pp, n_mb) in-flight micro-batches of activations
// (the 1F1B bound).  Stage 1 holds the maximum (M = M_1, R11),
// so it is the only stage evaluated here.
__device__ unsigned long long stage1_memory(const pipette_model& m, int pp, int tp, int mb, int n_mb) {
  const unsigned long long L = m.n_layers, h = m.hidden, a = m.heads, s = m.seq_len, V = m.vocab;
  const unsigned long long lps = ceil_div_u64(L, (unsigned long long)pp);
  const unsigned long long P1 = lps * (12ull * h * h + 13ull * h) + V * h + s * h;
  const unsigned long long W1 = (unsigned long long)m.bytes_per_param_state * ceil_div_u64(P1, (unsigned long long)tp);
  const unsigned long long act =
      ceil_div_u64(s * (unsigned long long)mb * h * (10ull * tp + 24ull) + 5ull * a * s * s * (unsigned long long)mb,
                   (unsigned long long)tp);
  const unsigned long long infl = (unsigned long long)min(pp, n_mb);
  return W1 + infl * lps * act + m.overhead_bytes;
}

__device__ __forceinline__ int n_divisors(long long n) {
  int c = 0;
  for (long long d = 1; d * d <= n; ++d)
    if (n % d == 0) c += (d * d == n) ? 1 : 2;
  return c;
}

__global__ void __launch_bounds__(kEnumThreads)
k_enumerate_filter(int n_nodes, int g, unsigned long long cap, int margin, pipette_model m,
                   long long bs_global, const pipette_profile_entry* __restrict__ prof, int n_prof,
                   DevCfg* __restrict__ cfgs, unsigned long long* __restrict__ keys, int E_cap,
                   int* __restrict__ feas, double* __restrict__ qtab, int qtab_cap,
                   EnumOut* __restrict__ out) {
  __shared__ int sh_scan[32];
  __shared__ int divG[kMaxGpus], divg[kMaxGpus];
  __shared__ int nG, ng;
  const int G = n_nodes * g;
  const int tid = threadIdx.x;

  // divisors of G and of g in ascending order (ordered stream compaction)
  {
    int tot;
    const int d = tid + 1;
    const int isG = (d <= G && G % d == 0);
    const int oG = block_scan_excl(isG, sh_scan, tot);
    if (isG) divG[oG] = d;
    if (tid == 0) nG = tot;
    const int isg = (d <= g && g % d == 0);
    const int og = block_scan_excl(isg, sh_scan, tot);
    if (isg) divg[og] = d;
    if (tid == 0) ng = tot;
    __syncthreads();
  }

  // (pp, tp) pairs in canonical order; each contributes divisors(bs_mini) configurations
  const int n_pairs = nG * ng;
  int carry = 0;
  for (int base = 0; base < n_pairs; base += blockDim.x) {
    const int i = base + tid;
    int pp = 0, tp = 0, dp = 0, cnt = 0;
    long long bs_mini = 0;
    if (i < n_pairs) {
      pp = divG[i / ng];
      tp = divg[i % ng];
      if (pp <= m.n_layers && G % (pp * tp) == 0) {
        dp = G / (pp * tp);
        if (bs_global % dp == 0) {
          bs_mini = bs_global / dp;
          cnt = n_divisors(bs_mini);
        }
      }
    }
    int tot;
    const int off = carry + block_scan_excl(cnt, sh_scan, tot);
    carry += tot;
    if (cnt > 0) {
      // ascending divisors: small ones d <= sqrt, then the cofactors in reverse
      int k = 0;
      long long d = 1;
      for (; d * d <= bs_mini; ++d) {
        if (bs_mini % d) continue;
        const int e = off + k++;
        if (e < E_cap) { cfgs[e].pp = pp; cfgs[e].tp = tp; cfgs[e].dp = dp; cfgs[e].mb = (int)d; }
      }
      for (--d; d >= 1; --d) {
        if (bs_mini % d || d * d == bs_mini) continue;
        const int e = off + k++;
        if (e < E_cap) { cfgs[e].pp = pp; cfgs[e].tp = tp; cfgs[e].dp = dp; cfgs[e].mb = (int)(bs_mini / d); }
      }
    }
  }
  const int E = carry;
  __syncthreads();
  if (E > E_cap) {
    if (tid == 0) { out->E = E; out->F = 0; out->qtab_used = 0; out->overflow = 1; }
    return;
  }

  // per configuration: memory verdict, profile lookup, constants
  int qcarry = 0, fcarry = 0;
  for (int base = 0; base < E; base += blockDim.x) {
    const int e = base + tid;
    int feasible = 0, qsize = 0;
    if (e < E) {
      DevCfg c = cfgs[e];
      c.e = e;
      c.n_mb = (int)(bs_global / ((long long)c.dp * c.mb));
      c.N = c.pp * c.dp;
      c.spn = g / c.tp;
      c.pp_magic = c.pp >= 2 ? (uint32_t)((0x100000000ull + c.pp - 1) / c.pp) : 0u;
      c.spn_magic = c.spn >= 2 ? (uint32_t)((0x100000000ull + c.spn - 1) / c.spn) : 0u;
      c.mem = stage1_memory(m, c.pp, c.tp, c.mb, c.n_mb);
      const unsigned long long keep = (unsigned long long)(1000 - margin);
      const unsigned long long limit = cap / 1000ull * keep + (cap % 1000ull) * keep / 1000ull;
      c.feasible = c.mem <= limit;
      feasible = c.feasible;
      int pe = -1;
      for (int j = 0; j < n_prof; ++j)
        if (prof[j].tp == c.tp && prof[j].mb == c.mb) { pe = j; break; }
      c.has_profile = pe >= 0;
      const unsigned long long L = m.n_layers, h = m.hidden;
      const unsigned long long lps = ceil_div_u64(L, (unsigned long long)c.pp);
      const unsigned long long msg_pp = (unsigned long long)c.mb * m.seq_len * h * m.bytes_per_elem;
      const unsigned long long n_params = 12ull * L * h * h + (unsigned long long)m.vocab * h;
      const unsigned long long msg_dp = n_params / ((unsigned long long)c.pp * c.tp) * m.bytes_per_elem;
      const double Lf = (double)lps;
      if (pe >= 0) {
        c.S = __dadd_rn(__dmul_rn(Lf, prof[pe].c_layer_s), __dmul_rn(Lf, prof[pe].tp_layer_s));
      } else {
        c.S = __longlong_as_double(0x7ff8000000000000ll);
      }
      c.m2 = __dmul_rn(2.0, (double)msg_pp);
      c.md = (double)msg_dp;
      c.r = __ddiv_rn((double)c.n_mb, (double)c.pp);
      c.Sb = __dmul_rn((double)c.pp, c.S);
      c.Ss = __dmul_rn((double)(c.pp - 1), c.S);
      qsize = (c.dp + 1) + (min(c.dp, n_nodes) + 1);
      cfgs[e] = c;
      keys[e] = ((unsigned long long)c.pp << 48) | ((unsigned long long)c.tp << 32) |
                ((unsigned long long)c.dp << 16) | (unsigned long long)c.mb;
    }
    int tot;
    const int qo = qcarry + block_scan_excl(qsize, sh_scan, tot);
    qcarry += tot;
    const int fo = fcarry + block_scan_excl(feasible, sh_scan, tot);
    fcarry += tot;
    if (e < E) {
      cfgs[e].qi_off = qo;
      cfgs[e].qe_off = qo + cfgs[e].dp + 1;
      if (feasible) feas[fo] = e;
    }
  }
  __syncthreads();
  if (qcarry > qtab_cap) {
    if (tid == 0) { out->E = E; out->F = fcarry; out->qtab_used = qcarry; out->overflow = 2; }
    return;
  }
  // Eq.6 ring factors: qi(c) = ((4(c-1)) md)/c, qe(k) = ((2(k-1)) md)/k; one warp per config
  const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  for (int e = wid; e < E; e += nw) {
    const DevCfg c = cfgs[e];
    for (int x = lane; x <= c.dp; x += 32)
      qtab[c.qi_off + x] = x < 1 ? 0.0 : __ddiv_rn(__dmul_rn(__dmul_rn(4.0, (double)(x - 1)), c.md), (double)x);
    const int kmax = min(c.dp, n_nodes);
    for (int x = lane; x <= kmax; x += 32)
      qtab[c.qe_off + x] = x < 1 ? 0.0 : __ddiv_rn(__dmul_rn(__dmul_rn(2.0, (double)(x - 1)), c.md), (double)x);
  }
  if (tid == 0) { out->E = E; out->F = fcarry; out->qtab_used = qcarry; out->overflow = 0; }
}

}  // namespace pip

namespace pip {

// ------------------------------------------------------------------ NEXT-4: Eq.7's MLP
// The memory estimator MLP of Eq.7 (reading R23) replacing the analytic
// estimate of K1 when the context has one (pipette_set_memory_model).  One block; warp w
// takes configurations w, w + 8, ...; a layer's 200 neurons are split over the lanes, each
// neuron accumulated in the oracle's order (acc = b, then acc + W_ji * in_i, i ascending),
// activations in shared memory; lane 0 forms the output sum.  Then the verdicts and the
// ordered feasible list are rebuilt with a block scan.
constexpr int kMlpH = 200, kMlpWarps = 8;

// ln(x), x >= 1: exact split x = m 2^e, ln m = 2 atanh((m-1)/(m+1)) by a degree-31 odd
// series in Horner form with fl(1/(2k+1)) -- the oracle's or_log_det, op for op
__device__ double log_det(double x) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  const long long ex = (long long)((bits >> 52) & 0x7ffull) - 1023;
  const double m = __longlong_as_double((long long)((bits & 0x000fffffffffffffull) | 0x3ff0000000000000ull));
  const double s = __ddiv_rn(__dadd_rn(m, -1.0), __dadd_rn(m, 1.0));
  const double s2 = __dmul_rn(s, s);
  double p = __ddiv_rn(1.0, 31.0);
  for (int k = 14; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, s2), __ddiv_rn(1.0, (double)(2 * k + 1)));
  const double lnm = __dmul_rn(2.0, __dmul_rn(s, p));
  const double e = (double)ex;
  return __dadd_rn(__dadd_rn(__dmul_rn(e, 6.93147180369123816490e-01), lnm), __dmul_rn(e, 1.90821492927058770002e-10));
}

__global__ void __launch_bounds__(kMlpWarps * 32)
k_mlp_filter(const double* __restrict__ P, int G, int n_nodes, pipette_model m, long long bs_global,
             unsigned long long cap, int margin, DevCfg* __restrict__ cfgs, int* __restrict__ feas,
             EnumOut* __restrict__ out) {
  __shared__ double act[kMlpWarps][2][kMlpH];
  __shared__ int sh_scan[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int E = out->E;
  if (out->overflow) return;
  const unsigned long long keep = (unsigned long long)(1000 - margin);
  const unsigned long long limit = cap / 1000ull * keep + (cap % 1000ull) * keep / 1000ull;
  for (int e = wid; e < E; e += kMlpWarps) {
    const DevCfg c = cfgs[e];
    const double f[10] = {(double)G, (double)m.n_layers, (double)m.hidden, (double)m.heads, (double)c.tp,
                          (double)c.pp, (double)c.dp, (double)c.mb, (double)(bs_global / c.dp), (double)bs_global};
    double x[10];
#pragma unroll
    for (int i = 0; i < 10; ++i) x[i] = __ddiv_rn(__dadd_rn(log_det(f[i]), -P[i]), P[10 + i]);
    const double* w = P + 20;
    // layer 1: 10 -> 200
    for (int j = lane; j < kMlpH; j += 32) {
      double acc = w[kMlpH * 10 + j];
#pragma unroll
      for (int i = 0; i < 10; ++i) acc = __dadd_rn(acc, __dmul_rn(w[j * 10 + i], x[i]));
      act[wid][0][j] = fmax(acc, 0.0);
    }
    w += kMlpH * 10 + kMlpH;
    __syncwarp();
    // layers 2..4: 200 -> 200
    for (int l = 1; l < 4; ++l) {
      const double* in = act[wid][(l - 1) & 1];
      double* o = act[wid][l & 1];
      for (int j = lane; j < kMlpH; j += 32) {
        double acc = w[kMlpH * kMlpH + j];
        const double* row = w + (size_t)j * kMlpH;
        for (int i = 0; i < kMlpH; ++i) acc = __dadd_rn(acc, __dmul_rn(row[i], in[i]));
        o[j] = fmax(acc, 0.0);
      }
      w += kMlpH * kMlpH + kMlpH;
      __syncwarp();
    }
    if (lane == 0) {
      const double* in = act[wid][1];
      double y = w[kMlpH];
      for (int i = 0; i < kMlpH; ++i) y = __dadd_rn(y, __dmul_rn(w[i], in[i]));
      double z = __dadd_rn(__dmul_rn(y, w[kMlpH + 1]), w[kMlpH + 2]);
      z = fmin(z, 16.0);
      const double gb = __dmul_rn(exp_det(__dadd_rn(z, -16.0)), 0x1.0f2ebd0a80020p+23);   // fl(e^16)
      const double bytes = __dmul_rn(gb, 1e9);
      const unsigned long long mem = bytes > 0.0 ? __double2ull_rz(bytes) : 0ull;
      cfgs[e].mem = mem;
      cfgs[e].feasible = mem <= limit;
    }
    __syncwarp();
  }
  __syncthreads();
  // ordered feasible list
  int carry = 0;
  for (int base = 0; base < E; base += blockDim.x) {
    const int e = base + tid;
    const int fe = e < E ? cfgs[e].feasible : 0;
    int tot;
    const int o = carry + block_scan_excl(fe, sh_scan, tot);
    carry += tot;
    if (fe) feas[o] = e;
  }
  if (tid == 0) out->F = carry;
}

void launch_mlp_filter(const double* P, int G, int n_nodes, const pipette_model& m, long long bs, unsigned long long cap,
                       int margin, DevCfg* cfgs, int* feas, EnumOut* out, cudaStream_t s) {
  k_mlp_filter<<<1, kMlpWarps * 32, 0, s>>>(P, G, n_nodes, m, bs, cap, margin, cfgs, feas, out);
}

}  // namespace pip
