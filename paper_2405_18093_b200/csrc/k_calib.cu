// k_calib.cu -- the SA's initial temperature by self-calibration (NEXT-1, reading
// R24 of DESIGN.md).  The paper fixes only the reduction coefficient alpha; SPEC's
// design decision picks T0 "so the median |Delta| of 100 seeded random moves is accepted
// with probability 0.8": exp(-median / T0) = 0.8, i.e. beta0 = 1/T0 = ln(1.25) / median.
//
// One block per feasible configuration; thread i < 100 draws move i from the Philox block
// of counter (i, 0, e, 1) (fourth word 1: disjoint from every SA proposal, whose fourth word
// is 0), selects its kind like an SA proposal (R14, R21), applies it to the identity mapping
// (the chains' start, R16) and evaluates Eq.3-6 from scratch in the normative operation
// order.  |Delta_i| = |L_i - L0|; the median of the 100 values is
// (s[49] + s[50]) * 0.5 of the ascending sort; beta0 = 0.22314355131420976 / median (the
// double nearest ln 1.25), or 1/(tau * L0) when the median is 0 or N < 2.  Every value is
// one IEEE round-to-nearest operation, so beta0 equals the oracle's or_calibrate_beta.
#include "devmath.cuh"
#include "pipette_dev.cuh"

namespace pip {

// Slot at position w of the identity mapping after move (kind, p, q) (R21): swap p <-> q;
// migration: the element at p removed and inserted at index q; reverse of [min, max].
__device__ __forceinline__ uint32_t moved_slot(uint32_t w, int kind, uint32_t p, uint32_t q) {
  if (kind == 0) return w == p ? q : (w == q ? p : w);
  if (kind == 1) {
    if (p < q) return (w < p || w > q) ? w : (w == q ? p : w + 1u);
    return (w < q || w > p) ? w : (w == q ? p : w - 1u);
  }
  const uint32_t lo = min(p, q), hi = max(p, q);
  return (w >= lo && w <= hi) ? lo + hi - w : w;
}

// Eq.3-6 of the moved identity mapping, from the definition (one thread; cnt: n counters).
__device__ double latency_moved(const DevCfg& C, const double* __restrict__ qtab, const double* __restrict__ R, int n,
                                int kind, uint32_t p, uint32_t q, uint16_t* cnt) {
  const int pp = C.pp, dp = C.dp;
  const uint32_t spn = (uint32_t)C.spn;
  double tpp = 0.0;
  for (int z = 0; z < dp; ++z) {   // Eq.5: sequential over stages, max over pipelines
    const uint32_t b = (uint32_t)(z * pp);
    uint32_t prev = moved_slot(b, kind, p, q) / spn;
    double s = 0.0;
    for (int x = 1; x < pp; ++x) {
      const uint32_t cur = moved_slot(b + (uint32_t)x, kind, p, q) / spn;
      s = __dadd_rn(s, __dmul_rn(C.m2, R[prev * (uint32_t)n + cur]));
      prev = cur;
    }
    tpp = fmax(tpp, s);
  }
  for (int a = 0; a < n; ++a) cnt[a] = 0;   // Eq.6: stage-1 occupancy of every node
  for (int z = 0; z < dp; ++z) ++cnt[moved_slot((uint32_t)(z * pp), kind, p, q) / spn];
  double tin = 0.0, mx = 0.0;
  int k = 0;
  for (int a = 0; a < n; ++a) {
    if (!cnt[a]) continue;
    ++k;
    if (cnt[a] >= 2) tin = fmax(tin, __dmul_rn(qtab[C.qi_off + cnt[a]], R[a * n + a]));
    for (int b = 0; b < n; ++b)
      if (b != a && cnt[b]) mx = fmax(mx, R[a * n + b]);
  }
  const double tex = k >= 2 ? __dmul_rn(qtab[C.qe_off + k], mx) : 0.0;
  return compose(C.Sb, C.r, C.Ss, tpp, tin, tex);
}

__global__ void __launch_bounds__(128) k_t0_calibrate(const DevCfg* __restrict__ cfgs, const int* __restrict__ feas,
                                                      const double* __restrict__ qtab, const double* __restrict__ R,
                                                      int n, RoundKeys rk, int w_migrate, int w_reverse, double tau,
                                                      double* __restrict__ beta0) {
  const int f = blockIdx.x, i = threadIdx.x;
  const DevCfg C = cfgs[feas[f]];
  __shared__ double d[100];
  __shared__ double L0s;
  uint16_t cnt[kMaxNodes];
  if (i == 0) L0s = latency_moved(C, qtab, R, n, 0, 0u, 0u, cnt);   // (swap 0 <-> 0: the identity)
  __syncthreads();
  const double L0 = L0s;
  const uint32_t N = (uint32_t)C.N;
  if (N >= 2 && i < 100) {
    const uint4 w = philox4x32_10_rk(make_uint4((uint32_t)i, 0u, (uint32_t)C.e, 1u), rk);
    const Draw dr = draw_from_words(w, N);
    const int t = (int)(((w.z & 31u) << 6) | (w.w & 63u));
    const int kind = t < 2048 - w_migrate - w_reverse ? 0 : (t < 2048 - w_reverse ? 1 : 2);
    d[i] = fabs(__dadd_rn(latency_moved(C, qtab, R, n, kind, dr.p, dr.q, cnt), -L0));
  }
  __syncthreads();
  if (i == 0) {
    double b = __ddiv_rn(1.0, __dmul_rn(tau, L0));
    if (N >= 2) {
      for (int a = 1; a < 100; ++a) {   // insertion sort, ascending
        const double v = d[a];
        int j = a - 1;
        while (j >= 0 && d[j] > v) { d[j + 1] = d[j]; --j; }
        d[j + 1] = v;
      }
      const double median = __dmul_rn(__dadd_rn(d[49], d[50]), 0.5);
      if (median > 0.0) b = __ddiv_rn(0.22314355131420976, median);
    }
    beta0[f] = b;
  }
}

void launch_t0_calibrate(const DevCfg* cfgs, const int* feas, int F, const double* qtab, const double* R, int n,
                         const RoundKeys& rk, int w_migrate, int w_reverse, double tau, double* beta0,
                         cudaStream_t s) {
  k_t0_calibrate<<<F, 128, 0, s>>>(cfgs, feas, qtab, R, n, rk, w_migrate, w_reverse, tau, beta0);
}

}  // namespace pip
