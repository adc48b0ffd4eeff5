// k_eval.cu -- K2: eval stream.  Memory verdict and Eq.3-6 latency of caller-supplied
// candidate plans (north_star "pipette_eval(candidates) ->
// latencies and memory").
//
// HBM-bound by design: 8 B of configuration + 2N B of mapping in, 17 B out per
// candidate.  One thread per candidate (DESIGN.md section 7 explains why not one warp:
// the per-candidate work is a sequential, fixed-order sum, and thread-per-candidate
// keeps all 32 lanes busy).  The mapping row is read with 16-byte vector loads; the
// config table keys and R = 1/B (lane-replicated when small) live in shared memory.
//   MODE 0 (n <= 16 nodes, <= 15 slots per node): stage-1 node counts are nibbles of a
//          64-bit register, the node set a 32-bit mask, the bijection bitmap two
//          registers (N <= 64), and the slowest inter-node link of Eq.6 one load from
//          the subset-max table.
//   MODE 1 (general): bitmap and counts in thread-interleaved shared memory (bank-
//          conflict free), pairwise scan of the stage-1 node set.
#include "devmath.cuh"
#include "pipette_dev.cuh"

namespace pip {

constexpr int kEvalThreads = 256;

template <int MODE>
__global__ void __launch_bounds__(kEvalThreads) k_eval_stream(EvalParams P) {
  constexpr bool REP = MODE == 0;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = P.n_nodes, nn = n * n;
  const int tid = threadIdx.x, lane = tid & 31;
  double* Rs = reinterpret_cast<double*>(smem);
  const int r_bytes = (REP ? nn * 32 : nn) * 8;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem + r_bytes);
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem + r_bytes + ((P.E * 8 + 15) & ~15));
  uint32_t* cnt = bm + P.bm_words * kEvalThreads;
  if (REP) {
    for (int i = tid; i < nn * 32; i += blockDim.x) Rs[i] = P.R[i >> 5];
  } else {
    for (int i = tid; i < nn; i += blockDim.x) Rs[i] = P.R[i];
  }
  for (int i = tid; i < P.E; i += blockDim.x) keys[i] = P.keys[i];
  __syncthreads();
  auto Rab = [&](uint32_t a, uint32_t b) -> double {
    return REP ? Rs[((int)a * n + (int)b) * 32 + lane] : Rs[(int)a * n + (int)b];
  };
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  const int cwords = (n + 3) / 4;

  for (long long i = (long long)blockIdx.x * blockDim.x + tid; i < P.n; i += (long long)gridDim.x * blockDim.x) {
    const pipette_config cf = P.cand[i];
    const unsigned long long key = ((unsigned long long)cf.pp << 48) | ((unsigned long long)cf.tp << 32) |
                                   ((unsigned long long)cf.dp << 16) | (unsigned long long)cf.mb;
    int lo = 0, hi = P.E;   // first index with keys[idx] >= key
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (keys[mid] < key) lo = mid + 1; else hi = mid;
    }
    if (lo >= P.E || keys[lo] != key) {      // not in the enumeration of Alg.1 l.3-5
      P.latency[i] = qnan; P.mem[i] = 0ull; P.status[i] = 2;
      continue;
    }
    const DevCfg C = P.cfgs[lo];
    const int N = C.N, pp = C.pp;
    const uint32_t spn = (uint32_t)C.spn;
    const uint16_t* row = P.perm + i * (long long)P.perm_stride;
    const bool regbm = MODE == 0 && N <= 64;
    if (!regbm)
      for (int w = 0; w < (N + 31) / 32; ++w) bm[w * kEvalThreads + tid] = 0u;
    if (MODE != 0)
      for (int w = 0; w < cwords; ++w) cnt[w * kEvalThreads + tid] = 0u;
    uint32_t b0 = 0u, b1 = 0u, dup = 0u;        // register bitmap (MODE 0, N <= 64)
    unsigned long long c64 = 0ull;              // nibble counts (MODE 0)
    Mask<MODE == 0 ? 1 : 4> mask;
    mask.clear();
    bool ok = true;
    double tpp = 0.0, s = 0.0;
    uint32_t prev = 0;
    int x = 0;
    auto visit = [&](uint32_t v) {
      uint32_t nd = 0;
      if (v >= (uint32_t)N) {
        ok = false;
      } else {
        if (regbm) {
          const uint32_t bit = 1u << (v & 31);
          const bool hi32 = v >= 32;
          dup |= (hi32 ? b1 : b0) & bit;
          b0 |= hi32 ? 0u : bit;
          b1 |= hi32 ? bit : 0u;
        } else {
          uint32_t& bw = bm[(v >> 5) * kEvalThreads + tid];
          const uint32_t bit = 1u << (v & 31);
          if (bw & bit) ok = false;
          bw |= bit;
        }
        nd = div_small(v, C.spn_magic, spn);
      }
      if (x == 0) {                                  // stage-1 worker of pipeline z (Eq.6)
        if (MODE == 0) c64 += 1ull << (4u * nd);
        else cnt[(nd >> 2) * kEvalThreads + tid] += 1u << ((nd & 3) * 8);
        mask.set(nd);
        s = 0.0;
      } else {                                       // Eq.5 hop x-1 -> x, stage order
        s = __dadd_rn(s, __dmul_rn(C.m2, Rab(prev, nd)));
      }
      prev = nd;
      if (++x == pp) {
        x = 0;
        if (pp >= 2) tpp = fmax(tpp, s);
      }
    };
    if (P.vec16) {
      const uint4* r4 = reinterpret_cast<const uint4*>(row);
      for (int w0 = 0; w0 < N; w0 += 8) {
        const uint4 v = __ldg(r4 + (w0 >> 3));
        const uint32_t pk[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (w0 + j < N) visit((pk[j >> 1] >> ((j & 1) * 16)) & 0xffffu);
      }
    } else {
      for (int w = 0; w < N; ++w) visit(__ldg(row + w));
    }
    if (dup) ok = false;
    P.mem[i] = C.mem;
    if (!ok) { P.latency[i] = qnan; P.status[i] = 3; continue; }
    if (!C.has_profile) { P.latency[i] = qnan; P.status[i] = 4; continue; }
    // Eq.6: per-node intra ring over nodes with >= 2 stage-1 members, slowest inter link
    const double* qi = P.qtab + C.qi_off;
    double t_in = 0.0, mx = 0.0;
    const int k = mask.count();
    if (MODE == 0) {
      uint32_t bits = mask.w[0];
      while (bits) {
        const uint32_t a = __ffs(bits) - 1;
        bits &= bits - 1;
        const uint32_t c = (uint32_t)(c64 >> (4u * a)) & 15u;
        if (c >= 2) t_in = fmax(t_in, __dmul_rn(__ldg(qi + c), Rab(a, a)));
      }
      if (k >= 2) mx = __ldg(P.subset_max + mask.w[0]);
    } else {
#pragma unroll
      for (int wd = 0; wd < 4; ++wd) {
        uint32_t bits = mask.w[wd];
        while (bits) {
          const uint32_t a = wd * 32 + __ffs(bits) - 1;
          bits &= bits - 1;
          const uint32_t c = (cnt[(a >> 2) * kEvalThreads + tid] >> ((a & 3) * 8)) & 0xffu;
          if (c >= 2) t_in = fmax(t_in, __dmul_rn(__ldg(qi + c), Rab(a, a)));
#pragma unroll
          for (int wd2 = 0; wd2 < 4; ++wd2) {
            uint32_t bits2 = mask.w[wd2];
            while (bits2) {
              const uint32_t b = wd2 * 32 + __ffs(bits2) - 1;
              bits2 &= bits2 - 1;
              if (a != b) mx = fmax(mx, Rab(a, b));
            }
          }
        }
      }
    }
    const double t_ex = k >= 2 ? __dmul_rn(__ldg(P.qtab + C.qe_off + k), mx) : 0.0;
    P.latency[i] = compose(C.Sb, C.r, C.Ss, tpp, t_in, t_ex);
    P.status[i] = C.feasible ? 0 : 1;
  }
}

// Host-side handle of the K2 variant (MODE 0 small clusters, 1 general).
const void* eval_kernel(int mode) {
  return mode == 0 ? (const void*)k_eval_stream<0> : (const void*)k_eval_stream<1>;
}

}  // namespace pip
