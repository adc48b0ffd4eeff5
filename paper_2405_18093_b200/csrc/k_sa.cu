// k_sa.cu -- K3: simulated-annealing chains of fine-grained worker dedication and
// K4: per-configuration argmin.
//
// Alg.1 l.9-15 with the SA of P:250-255: each proposal swaps two positions
// of the mapping string (Eq.2), re-evaluates Eq.3-6 and is
// accepted by Metropolis (R13) with Philox randomness (R14).
//
// Design: one chain per LANE; a warp runs 32 chains of one
// configuration, so every instruction advances 32 independent Markov chains.  Chain
// state lives in shared memory in a lane-interleaved layout ([element][lane], 4- or
// 8-byte words), which makes every per-lane random access bank-conflict free:
//   pos[w]   = slot | node << 16             (N words)
//   psum[z]  = Eq.5 sum of pipeline z        (dp doubles, pp >= 2)
//   cnt[a]   = stage-1 DP members on node a  (u8, packed 4 per word; c_a <= spn)
// R = 1/B is staged once per block, replicated per lane when small (conflict free).
// Re-evaluation is incremental but bit-exact: only the (at most two) touched pipelines
// are re-summed from scratch in stage order, and the max terms (T_PP, T_in, T_ex) are
// maintained with witnesses and rescanned when a witness could drop -- max is exact,
// so every latency equals the from-scratch definition bit for bit.
#include "devmath.cuh"
#include "pipette_dev.cuh"

namespace pip {

constexpr int kSaThreads = 128;

__device__ __forceinline__ int align16(int x) { return (x + 15) & ~15; }

template <bool REP>
struct RTab {
  const double* s;
  int n, lane;
  __device__ __forceinline__ double operator()(uint32_t a, uint32_t b) const {
    return REP ? s[((int)a * n + (int)b) * 32 + lane] : s[(int)a * n + (int)b];
  }
};


__device__ __forceinline__ uint32_t cnt_get(const uint32_t* cnt, uint32_t a, int lane) {
  return (cnt[(a >> 2) * 32 + lane] >> ((a & 3) * 8)) & 0xffu;
}
__device__ __forceinline__ void cnt_add(uint32_t* cnt, uint32_t a, int lane, int delta) {
  const uint32_t sh = (a & 3) * 8;
  uint32_t& w = cnt[(a >> 2) * 32 + lane];
  w = delta > 0 ? w + (1u << sh) : w - (1u << sh);
}

// Eq.6 intra term from scratch over the stage-1 node set: max_{c_a >= 2} qi(c_a) R[a][a].
template <int MW, bool REP>
__device__ __forceinline__ double tin_full(const Mask<MW>& m, const uint32_t* cnt, int lane, uint32_t dn,
                                           uint32_t c_dn, uint32_t up, uint32_t c_up, const double* qi,
                                           const RTab<REP>& R, int& win) {
  double t = 0.0;
  win = -1;
#pragma unroll
  for (int wd = 0; wd < MW; ++wd) {
    uint32_t bits = m.w[wd];
    while (bits) {
      const uint32_t a = wd * 32 + __ffs(bits) - 1;
      bits &= bits - 1;
      const uint32_t c = a == dn ? c_dn : (a == up ? c_up : cnt_get(cnt, a, lane));
      if (c >= 2) {
        const double v = __dmul_rn(__ldg(qi + c), R(a, a));
        if (v > t) { t = v; win = (int)a; }
      }
    }
  }
  return t;
}

// Eq.6 inter term's slowest link from scratch: max over ordered pairs a != b of R[a][b].
template <int MW, bool REP>
__device__ __forceinline__ double maxr_full(const Mask<MW>& m, const RTab<REP>& R, int& wa, int& wb) {
  double mx = 0.0;
  wa = wb = -1;
#pragma unroll
  for (int wd = 0; wd < MW; ++wd) {
    uint32_t bits = m.w[wd];
    while (bits) {
      const uint32_t a = wd * 32 + __ffs(bits) - 1;
      bits &= bits - 1;
#pragma unroll
      for (int wd2 = 0; wd2 < MW; ++wd2) {
        uint32_t bits2 = m.w[wd2];
        while (bits2) {
          const uint32_t b = wd2 * 32 + __ffs(bits2) - 1;
          bits2 &= bits2 - 1;
          if (a == b) continue;
          const double v = R(a, b);
          if (v > mx) { mx = v; wa = (int)a; wb = (int)b; }
        }
      }
    }
  }
  return mx;
}

// Eq.5 sum of pipeline z in stage order, with positions p and q holding nodes np and nq
// after the proposed swap (P_z = ((0 + m2 R[..]) + m2 R[..]) + ...).
// PP > 0: compile-time pipeline depth (fully unrolled); PP == 0: runtime depth pp.
template <bool REP, int PP>
__device__ __forceinline__ uint32_t node_at(uint32_t w, const uint32_t* pos, int lane, uint32_t p, uint32_t q,
                                            uint32_t np, uint32_t nq) {
  return w == p ? nq : (w == q ? np : (pos[w * 32 + lane] >> 16));
}

template <bool REP, int PP>
__device__ __forceinline__ double pipe_sum(int z, int pp_rt, const uint32_t* pos, int lane, uint32_t p, uint32_t q,
                                           uint32_t np, uint32_t nq, double m2, const RTab<REP>& R) {
  const int pp = PP > 0 ? PP : pp_rt;
  const uint32_t base = (uint32_t)(z * pp);
  uint32_t prev = node_at<REP, PP>(base, pos, lane, p, q, np, nq);
  double s = 0.0;
#pragma unroll
  for (int x = 1; x < (PP > 0 ? PP : pp); ++x) {
    const uint32_t nd = node_at<REP, PP>(base + x, pos, lane, p, q, np, nq);
    s = __dadd_rn(s, __dmul_rn(m2, R(prev, nd)));
    prev = nd;
  }
  return s;
}

// Two pipelines re-summed in one interleaved loop (independent dependency chains).
template <bool REP, int PP>
__device__ __forceinline__ void pipe_sum2(int za, int zb, int pp_rt, const uint32_t* pos, int lane, uint32_t p,
                                          uint32_t q, uint32_t np, uint32_t nq, double m2, const RTab<REP>& R,
                                          double& sa, double& sb) {
  const int pp = PP > 0 ? PP : pp_rt;
  const uint32_t ba = (uint32_t)(za * pp), bb = (uint32_t)(zb * pp);
  uint32_t pa = node_at<REP, PP>(ba, pos, lane, p, q, np, nq);
  uint32_t pb = node_at<REP, PP>(bb, pos, lane, p, q, np, nq);
  double a = 0.0, b = 0.0;
#pragma unroll
  for (int x = 1; x < (PP > 0 ? PP : pp); ++x) {
    const uint32_t na = node_at<REP, PP>(ba + x, pos, lane, p, q, np, nq);
    const uint32_t nb = node_at<REP, PP>(bb + x, pos, lane, p, q, np, nq);
    a = __dadd_rn(a, __dmul_rn(m2, R(pa, na)));
    b = __dadd_rn(b, __dmul_rn(m2, R(pb, nb)));
    pa = na;
    pb = nb;
  }
  sa = a;
  sb = b;
}

template <int MW, bool REP, bool TRACE, int PP>
__device__ void run_task(const SaParams& P, const SaTask& T, const DevCfg& C, const double* Rs, unsigned char* ws,
                         int lane) {
  if (lane >= T.count) return;
  const int N = C.N, pp = PP > 0 ? PP : C.pp, dp = C.dp, n = P.n_nodes;
  const uint32_t spn = (uint32_t)C.spn;
  const uint32_t chain = (uint32_t)(T.c_first + (T.k0 + lane) * P.world);
  const int slot = T.slot0 + lane;
  const double* qi = P.qtab + C.qi_off;
  const double* qe = P.qtab + C.qe_off;
  const RTab<REP> R{Rs, n, lane};

  uint32_t* pos = reinterpret_cast<uint32_t*>(ws);
  double* psum = reinterpret_cast<double*>(ws + align16(N * 128));
  uint32_t* cnt = reinterpret_cast<uint32_t*>(ws + align16(N * 128) + (pp >= 2 ? align16(dp * 256) : 0));
  uint16_t* bperm = P.best_perm + T.perm_off;

  // ---- initial state: identity mapping (R16) and its latency from scratch
  for (int w = 0; w < N; ++w) {
    pos[w * 32 + lane] = (uint32_t)w | (div_small((uint32_t)w, C.spn_magic, spn) << 16);
    bperm[w * 32 + lane] = (uint16_t)w;
  }
  for (int wd = 0; wd < (n + 3) / 4; ++wd) cnt[wd * 32 + lane] = 0u;
  Mask<MW> mask;
  mask.clear();
  double tpp = 0.0;
  for (int z = 0; z < dp; ++z) {
    const uint32_t n0 = pos[z * pp * 32 + lane] >> 16;
    cnt_add(cnt, n0, lane, +1);
    mask.set(n0);
    if (pp >= 2) {
      const double s = pipe_sum<REP, PP>(z, pp, pos, lane, 0xffffffffu, 0xffffffffu, 0u, 0u, C.m2, R);
      psum[z * 32 + lane] = s;
      tpp = fmax(tpp, s);
    }
  }
  int k = mask.count();
  int win, wa, wb;
  double t_in = tin_full<MW, REP>(mask, cnt, lane, 0xffffffffu, 0u, 0xffffffffu, 0u, qi, R, win);
  double maxR = 0.0;
  wa = wb = -1;
  if (k >= 2) maxR = maxr_full<MW, REP>(mask, R, wa, wb);
  double t_ex = k >= 2 ? __dmul_rn(__ldg(qe + k), maxR) : 0.0;

  const double L0 = compose(C.Sb, C.r, C.Ss, tpp, t_in, t_ex);
  double cur = L0, best = L0, best_tpp = tpp, best_tdp = __dadd_rn(t_in, t_ex);
  int best_step = -1;
  uint32_t accepted = 0;
  double beta = P.t0 > 0.0 ? __ddiv_rn(1.0, P.t0) : __ddiv_rn(1.0, __dmul_rn(P.tau, L0));
  const double ia = P.alpha_inv;
  const int trow = TRACE ? P.trace_slot[slot] : -1;

  if (N >= 2) {
    Draw dnext = draw_swap_rk(0u, chain, (uint32_t)C.e, P.rk, (uint32_t)N);
    for (int i = 0; i < P.iterations; ++i) {
      const Draw d = dnext;
      // the next proposal's Philox words do not depend on this step: issue them now (ILP)
      dnext = draw_swap_rk((uint32_t)(i + 1), chain, (uint32_t)C.e, P.rk, (uint32_t)N);
      const uint32_t wp = pos[d.p * 32 + lane], wq = pos[d.q * 32 + lane];
      const uint32_t np = wp >> 16, nq = wq >> 16;
      double Lp = cur;
      bool acc = true;
      bool improved = false;
      if (np != nq) {
        // ---- Eq.5: re-sum the (at most two) touched pipelines, maintain the max
        uint32_t xp = 0, xq = 0;
        int zp = 0, zq = 0;
        bool two = false;
        double sA = 0.0, sB = 0.0, tpp2 = tpp;
        if (pp >= 2) {
          zp = (int)div_small(d.p, C.pp_magic, (uint32_t)pp);
          zq = (int)div_small(d.q, C.pp_magic, (uint32_t)pp);
          xp = d.p - (uint32_t)(zp * pp);
          xq = d.q - (uint32_t)(zq * pp);
          two = zq != zp;
          if (two) pipe_sum2<REP, PP>(zp, zq, pp, pos, lane, d.p, d.q, np, nq, C.m2, R, sA, sB);
          else sA = pipe_sum<REP, PP>(zp, pp, pos, lane, d.p, d.q, np, nq, C.m2, R);
          const double oldA = psum[zp * 32 + lane];
          const double oldB = two ? psum[zq * 32 + lane] : oldA;
          const bool drop = (oldA == tpp && sA < tpp) || (two && oldB == tpp && sB < tpp);
          if (drop) {
            double mx = two ? fmax(sA, sB) : sA;
            for (int z = 0; z < dp; ++z)
              if (z != zp && z != zq) mx = fmax(mx, psum[z * 32 + lane]);
            tpp2 = mx;
          } else {
            tpp2 = fmax(tpp, two ? fmax(sA, sB) : sA);
          }
        }
        // ---- Eq.6: the stage-1 node multiset changes only if exactly one of p, q is stage 1
        const bool sp = xp == 0u, sq = xq == 0u;
        double tin2 = t_in, tex2 = t_ex, maxR2 = maxR;
        int win2 = win, wa2 = wa, wb2 = wb, k2 = k;
        uint32_t dn = 0, up = 0, c_dn = 0, c_up = 0;
        Mask<MW> mask2 = mask;
        const bool dpchg = sp != sq;
        if (dpchg) {
          dn = sp ? np : nq;   // node losing a stage-1 DP member
          up = sp ? nq : np;   // node gaining one
          c_dn = cnt_get(cnt, dn, lane) - 1u;
          c_up = cnt_get(cnt, up, lane) + 1u;
          const bool leave = c_dn == 0u, join = c_up == 1u;
          if (leave) mask2.reset(dn);
          if (join) mask2.set(up);
          k2 = k - (int)leave + (int)join;
          if ((int)dn == win) {
            tin2 = tin_full<MW, REP>(mask2, cnt, lane, dn, c_dn, up, c_up, qi, R, win2);
          } else if (c_up >= 2u) {
            const double v = __dmul_rn(__ldg(qi + c_up), R(up, up));
            if (v > tin2) { tin2 = v; win2 = (int)up; }
          }
          if (k2 < 2) {
            maxR2 = 0.0; wa2 = wb2 = -1;
          } else if (leave && ((int)dn == wa || (int)dn == wb)) {
            maxR2 = maxr_full<MW, REP>(mask2, R, wa2, wb2);
          } else if (join) {
#pragma unroll
            for (int wd = 0; wd < MW; ++wd) {
              uint32_t bits = mask2.w[wd];
              while (bits) {
                const uint32_t b = wd * 32 + __ffs(bits) - 1;
                bits &= bits - 1;
                if (b == up) continue;
                const double v1 = R(up, b), v2 = R(b, up);
                if (v1 > maxR2) { maxR2 = v1; wa2 = (int)up; wb2 = (int)b; }
                if (v2 > maxR2) { maxR2 = v2; wa2 = (int)b; wb2 = (int)up; }
              }
            }
          }
          tex2 = k2 >= 2 ? __dmul_rn(__ldg(qe + k2), maxR2) : 0.0;
        }
        Lp = compose(C.Sb, C.r, C.Ss, tpp2, tin2, tex2);
        acc = metropolis_fast(__dadd_rn(Lp, -cur), beta, d.u);
        if (acc) {
          if (pp >= 2) {
            psum[zp * 32 + lane] = sA;
            if (two) psum[zq * 32 + lane] = sB;
            tpp = tpp2;
          }
          if (dpchg) {
            cnt_add(cnt, dn, lane, -1);
            cnt_add(cnt, up, lane, +1);
            mask = mask2; k = k2;
            t_in = tin2; win = win2;
            t_ex = tex2; maxR = maxR2; wa = wa2; wb = wb2;
          }
          cur = Lp;
          if (Lp < best) {
            best = Lp; best_step = i; best_tpp = tpp; best_tdp = __dadd_rn(t_in, t_ex);
            improved = true;
          }
        }
      }
      if (acc) {
        pos[d.p * 32 + lane] = wq;
        pos[d.q * 32 + lane] = wp;
        ++accepted;
      }
      if (improved)
        for (int w = 0; w < N; ++w) bperm[w * 32 + lane] = (uint16_t)(pos[w * 32 + lane] & 0xffffu);
      if (TRACE && trow >= 0 && i < P.trace_cap) {
        pipette_trace_record rec;
        rec.i = (uint32_t)i; rec.p = (uint16_t)d.p; rec.q = (uint16_t)d.q;
        rec.accept = acc ? 1u : 0u; rec.latency = Lp;
        P.trace[(size_t)trow * P.trace_cap + i] = rec;
      }
      beta = __dmul_rn(beta, ia);
    }
  }
  ChainOut o;
  o.best = best; o.best_tpp = best_tpp; o.best_tdp = best_tdp; o.L0 = L0;
  o.best_step = best_step; o.accepted = accepted; o.f = T.f; o.c = (int32_t)chain;
  P.out[slot] = o;
}

template <int MW, bool REP, bool TRACE>
__global__ void __launch_bounds__(kSaThreads) k_sa_chains(SaParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* Rs = reinterpret_cast<double*>(smem);
  const int nn = P.n_nodes * P.n_nodes;
  if (REP) {
    for (int i = threadIdx.x; i < nn * 32; i += blockDim.x) Rs[i] = P.R[i >> 5];
  } else {
    for (int i = threadIdx.x; i < nn; i += blockDim.x) Rs[i] = P.R[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned char* ws = smem + P.r_smem_bytes + wid * P.warp_smem_bytes;
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(P.task_counter, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= P.n_tasks) break;
    const SaTask T = P.tasks[t];
    const DevCfg C = P.cfgs[T.cfg];
    unsigned long long t_start = 0;
    if (lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    switch (C.pp) {   // compile-time pipeline depth for the common power-of-two depths
      case 1: run_task<MW, REP, TRACE, 1>(P, T, C, Rs, ws, lane); break;
      case 2: run_task<MW, REP, TRACE, 2>(P, T, C, Rs, ws, lane); break;
      case 4: run_task<MW, REP, TRACE, 4>(P, T, C, Rs, ws, lane); break;
      case 8: run_task<MW, REP, TRACE, 8>(P, T, C, Rs, ws, lane); break;
      case 16: run_task<MW, REP, TRACE, 16>(P, T, C, Rs, ws, lane); break;
      default: run_task<MW, REP, TRACE, 0>(P, T, C, Rs, ws, lane); break;
    }
    __syncwarp();
    if (lane == 0) {
      unsigned long long t_end;
      uint32_t smid;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      ulonglong4* tp = reinterpret_cast<ulonglong4*>(P.task_prof) + t;
      *tp = make_ulonglong4(t_start, t_end, smid, (unsigned long long)T.cfg);
    }
  }
}

// K4: per-configuration lexicographic (latency, chain) minimum over this rank's chains,
// plus the sum of accepted proposals (Alg.1 l.13).  One block per feasible config.
__global__ void __launch_bounds__(256) k_argmin(const ChainOut* __restrict__ out, const int* __restrict__ cfg_slot,
                                                int F, CfgBest* __restrict__ res) {
  const int f = blockIdx.x;
  if (f >= F) return;
  const int s0 = cfg_slot[f], s1 = cfg_slot[f + 1];
  unsigned long long bk = ~0ull;
  int bc = 0x7fffffff, bs = -1;
  unsigned long long acc = 0;
  for (int s = s0 + threadIdx.x; s < s1; s += blockDim.x) {
    const ChainOut o = out[s];
    const unsigned long long k = (unsigned long long)__double_as_longlong(o.best);  // latency >= 0
    if (k < bk || (k == bk && o.c < bc)) { bk = k; bc = o.c; bs = s; }
    acc += o.accepted;
  }
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long k2 = __shfl_down_sync(0xffffffffu, bk, off);
    const int c2 = __shfl_down_sync(0xffffffffu, bc, off);
    const int s2 = __shfl_down_sync(0xffffffffu, bs, off);
    acc += __shfl_down_sync(0xffffffffu, acc, off);
    if (k2 < bk || (k2 == bk && c2 < bc)) { bk = k2; bc = c2; bs = s2; }
  }
  __shared__ unsigned long long sk[8], sa[8];
  __shared__ int sc[8], ss[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sk[wid] = bk; sc[wid] = bc; ss[wid] = bs; sa[wid] = acc; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      if (sk[w] < bk || (sk[w] == bk && sc[w] < bc)) { bk = sk[w]; bc = sc[w]; bs = ss[w]; }
      acc += sa[w];
    }
    CfgBest r;
    r.accepted = acc;
    r.slot = bs;
    if (bs >= 0) {
      const ChainOut o = out[bs];
      r.best = o.best; r.best_tpp = o.best_tpp; r.best_tdp = o.best_tdp;
      r.chain = o.c; r.best_step = o.best_step;
    } else {
      r.best = __longlong_as_double(0x7ff0000000000000ll);
      r.best_tpp = r.best_tdp = 0.0; r.chain = -1; r.best_step = -1;
    }
    r.pad = 0;
    res[f] = r;
  }
}

// Host-side handle of the K3 variant: MW = mask words (n <= 32 -> 1, else 4), REP = R
// replicated per lane, TRACE = debug trace records.
const void* sa_kernel(int mw, bool rep, bool trace) {
  if (mw == 1) {
    if (rep) return trace ? (const void*)k_sa_chains<1, true, true> : (const void*)k_sa_chains<1, true, false>;
    return trace ? (const void*)k_sa_chains<1, false, true> : (const void*)k_sa_chains<1, false, false>;
  }
  if (rep) return trace ? (const void*)k_sa_chains<4, true, true> : (const void*)k_sa_chains<4, true, false>;
  return trace ? (const void*)k_sa_chains<4, false, true> : (const void*)k_sa_chains<4, false, false>;
}

}  // namespace pip
