// k_eval.cu -- K2: eval stream.  Memory verdict and Eq.3-6 latency of caller-supplied
// candidate plans (north_star "pipette_eval(candidates) ->
// latencies and memory").
//
// HBM-bound by design: 8 B of configuration + 2N B of mapping in, 17 B out per
// candidate.  One thread per candidate (DESIGN.md section 7 explains why not one warp:
// the per-candidate work is a sequential, fixed-order sum, and thread-per-candidate
// keeps all 32 lanes busy).  A block works on tiles of TR candidates (TR = its thread
// count); the tile's mapping rows -- one contiguous range of HBM -- are staged into
// shared memory with coalesced 16-byte cp.async copies, double-buffered so the next
// tile streams in while this one is evaluated, and stored with the 128-byte XOR swizzle
// (16-byte chunk c of 128-byte line l at chunk c ^ (l & 7)) so that the per-thread row
// reads are bank-conflict free.  The config table keys and R = 1/B (16 lane copies when
// small) live in shared memory.
//   MODE 0 (n <= 16 nodes, <= 15 slots per node): the pipeline depth is a template
//          parameter (the stage of each mapping slot is static inside a 16-byte chunk),
//          stage-1 node counts are nibbles of a 64-bit register, the bijection bitmap is
//          a 64-bit register (N <= 64; shared memory above), and the slowest inter-node
//          link of Eq.6 is one load from the subset-max table.
//   MODE 1 (general): bitmap and counts in thread-interleaved shared memory (bank-
//          conflict free), pairwise scan of the stage-1 node set.
#include <cuda.h>

#include "devmath.cuh"
#include "pipette_dev.cuh"

namespace pip {


// Exclusive block-wide scan (one int per thread); total = block sum.
__device__ int block_scan_excl_eval(int v, int* sh, int& total) {
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

// 128-byte XOR swizzle of a byte offset inside a staging buffer (16-byte granules).
__device__ __forceinline__ uint32_t swz(uint32_t x) { return x ^ (((x >> 7) & 7u) << 4); }

// PTX shl.b64: shift amounts >= 64 give 0; two SASS funnel shifts (SHF.L.U32 for the low
// word, SHF.L.U64.HI for the high word), no range fix-up.
__device__ __forceinline__ unsigned long long shl64_clamp(uint32_t sh) {
  unsigned long long r;
  asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(1ull), "r"(sh));
  return r;
}

// PTX shl.b32: shift amounts >= 32 give 0 (C's << is undefined there).
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t sh) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(sh));
  return r;
}

// Where a candidate's mapping row is read from: the swizzled staging buffer (16-byte
// aligned rows) or global memory (any stride).
struct RowSrc {
  const unsigned char* sbuf;   // staging buffer of the warp (nullptr: global)
  uint32_t roff;               // byte offset of the row inside the buffer
  const uint16_t* g;           // global row
  bool vec;                    // 16-byte chunks (staged, or 16-byte aligned global rows)
  __device__ __forceinline__ uint4 chunk(int k) const {   // 8 slots [8k, 8k+8)
    if (sbuf) return *reinterpret_cast<const uint4*>(sbuf + swz(roff + (uint32_t)k * 16u));
    return __ldg(reinterpret_cast<const uint4*>(g) + k);
  }
  __device__ __forceinline__ uint32_t slot(int w) const { return __ldg(g + w); }
};

struct EvalShared {
  const double* Rs;
  uint32_t* bm;     // [bm_words][T]
  uint32_t* cnt;    // [ceil(n/4)][T] byte counts, or [ceil(n/8)][T] nibbles (cnt_nib)
  const uint16_t* pl;   // MODE 1: shared prefix of the R-sorted pair list (plen entries)
  int n, tid, lane, T;
  int plen;
  uint32_t cnt_nib;     // 1: stage-1 counts as nibbles (every count <= 15)
  uint32_t lgn;     // MODE 0: log2 of the padded table side
  const unsigned char* Rl;   // MODE 0: this lane's copy, &Rs[lane & 15]
  uint32_t row_bytes;        // MODE 0: 2^lgn * 16 copies * 8 B
};

// MODE 0: R padded to npad x npad (npad = 2^lgn >= n; zeros outside n x n) with 16 lane
// copies, so any masked node pair (a, b < npad) is in range and conflict free.
// (MODE 0 address: two integer multiply-adds, which issue on the FMA pipe and leave the
// ALU pipe -- K2's limiter -- to the bijection test)
template <bool REP>
__device__ __forceinline__ double r_at(const EvalShared& S, uint32_t a, uint32_t b) {
  return REP ? *reinterpret_cast<const double*>(S.Rl + a * S.row_bytes + b * 128u) : S.Rs[(int)a * S.n + (int)b];
}

// MODE 0 evaluation of one candidate with compile-time pipeline depth PP (0: runtime).
template <int PP, bool RB>
__device__ __forceinline__ void eval_small(const EvalParams& P, const EvalShared& S, const DevCfg& C,
                                           const RowSrc& row, long long i, int e) {
  const int N = C.N;
  const int pp = PP > 0 ? PP : C.pp;
  const uint32_t spn = (uint32_t)C.spn;
  const uint32_t nmask = (1u << S.lgn) - 1u;
  constexpr bool regbm = RB;   // N <= 64: bitmap in a register pair
  if (!regbm)
    for (int w = 0; w < (N + 31) / 32; ++w) S.bm[w * S.T + S.tid] = 0u;
  // Bijection test (Eq.2): OR the bit of every slot id into [0, 64) (a 2x32-bit register
  // pair; shl clamps, so ids >= 64 set nothing).  The row is a permutation of [0, N) iff
  // exactly the N low bits end up set: an id >= N sets a bit above N or none, and a
  // duplicate leaves one of the N bits unset.  Larger N: bitmap in shared memory.
  unsigned long long seen = 0ull;
  uint32_t c_lo = 0u, c_hi = 0u;        // stage-1 counts, nibble a of (c_hi:c_lo) = node a
  bool bad = false;
  double tpp = 0.0, s = 0.0;
  uint32_t prev = 0;
  int x = 0;   // runtime stage counter (PP == 0 only)
  auto visit = [&](uint32_t v, bool stage1, bool last) {
    if (regbm) {
      seen |= shl64_clamp(v);
    } else {
      bad |= v >= (uint32_t)N;
      const uint32_t vc = min(v, (uint32_t)N - 1u);
      uint32_t& bw = S.bm[(vc >> 5) * S.T + S.tid];
      bw |= 1u << (vc & 31);
    }
    // node of the slot; an id >= N (invalid row, flagged above) is masked into the padded
    // table instead of clamped
    const uint32_t nd = div_small(v, C.spn_magic, spn) & nmask;
    if (stage1) {                                    // stage-1 worker of pipeline z (Eq.6)
      c_lo += shl_clamp(1u, 4u * nd);
      c_hi += shl_clamp(1u, 4u * nd - 32u);
      s = 0.0;
    } else {                                         // Eq.5 hop x-1 -> x, stage order
      s = __dadd_rn(s, __dmul_rn(C.m2, r_at<true>(S, prev, nd)));
    }
    prev = nd;
    if (last && pp >= 2) tpp = dmax(tpp, s);
  };
  auto flags = [&](int w0, int j, bool& st, bool& la) {
    if constexpr (PP == 1) {
      st = true; la = true;
    } else if constexpr (PP == 2 || PP == 4 || PP == 8) {   // stage of slot j is static
      st = (j % PP) == 0; la = (j % PP) == PP - 1;
    } else if constexpr (PP >= 16) {                       // chunks never straddle pipelines
      st = j == 0 && (w0 & (PP - 1)) == 0;
      la = j == 7 && (w0 & (PP - 1)) == PP - 8;
    } else {
      st = x == 0; la = x == pp - 1;
      x = (x + 1 == pp) ? 0 : x + 1;
    }
  };
  if (row.vec) {
    const int full = N & ~7;                         // whole 8-slot chunks: no per-slot guard
    for (int w0 = 0; w0 < full; w0 += 8) {
      const uint4 v = row.chunk(w0 >> 3);
      const uint32_t pk[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        bool st, la;
        flags(w0, j, st, la);
        visit((pk[j >> 1] >> ((j & 1) * 16)) & 0xffffu, st, la);
      }
    }
    if (full < N) {
      const uint4 v = row.chunk(full >> 3);
      const uint32_t pk[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (full + j < N) {
          bool st, la;
          flags(full, j, st, la);
          visit((pk[j >> 1] >> ((j & 1) * 16)) & 0xffffu, st, la);
        }
      }
    }
  } else {
    for (int w = 0; w < N; ++w) {
      const bool st = (w % pp) == 0, la = (w % pp) == pp - 1;
      visit(row.slot(w), st, la);
    }
  }
  bool ok = !bad;
  if (regbm) {
    ok = seen == (N >= 64 ? ~0ull : ((1ull << N) - 1ull));
  } else {
    int c = 0;
    for (int w = 0; w < (N + 31) / 32; ++w) c += __popc(S.bm[w * S.T + S.tid]);
    ok = ok && c == N;
  }
  // stage-1 node set N1 from the nibble counts: bit a set iff nibble a is non-zero
  uint32_t lo = c_lo | (c_lo >> 1), hi = c_hi | (c_hi >> 1);
  lo = (lo | (lo >> 2)) & 0x11111111u; hi = (hi | (hi >> 2)) & 0x11111111u;
  lo = (lo | (lo >> 3)) & 0x03030303u; hi = (hi | (hi >> 3)) & 0x03030303u;
  lo = (lo | (lo >> 6)) & 0x000f000fu; hi = (hi | (hi >> 6)) & 0x000f000fu;
  lo = (lo | (lo >> 12)) & 0xffu;      hi = (hi | (hi >> 12)) & 0xffu;
  const uint32_t mask = lo | (hi << 8);
  P.mem[i] = C.mem;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  if (!ok) { P.latency[i] = qnan; P.status[i] = 3; return; }
  if (!C.has_profile) { P.latency[i] = qnan; P.status[i] = 4; return; }
  // Eq.6: per-node intra ring over nodes with >= 2 stage-1 members (value table
  // vin[e][a*16 + c] = qi(c) R[a][a], 0 for c < 2), slowest inter link
  const double* vin = P.vin + (size_t)e * 256;
  // only nodes with c >= 2 members contribute (a nibble with bit 1, 2 or 3 set)
  double t_in = 0.0;
#pragma unroll
  for (int hw = 0; hw < 2; ++hw) {
    const uint32_t h = hw ? c_hi : c_lo;
    uint32_t b = h & 0xeeeeeeeeu;
    while (b) {
      const uint32_t sh = (uint32_t)(__ffs(b) - 1) & ~3u;
      b &= ~(15u << sh);
      t_in = dmax(t_in, __ldg(vin + (hw * 8 + (sh >> 2)) * 16 + ((h >> sh) & 15u)));
    }
  }
  const int k = __popc(mask);
  const double t_ex = k >= 2 ? __dmul_rn(__ldg(P.qtab + C.qe_off + k), __ldg(P.subset_max + mask)) : 0.0;
  P.latency[i] = compose(C.Sb, C.r, C.Ss, tpp, t_in, t_ex);
  P.status[i] = C.feasible ? 0 : 1;
}

template <int PP>
__device__ __forceinline__ void dispatch_n(const EvalParams& P, const EvalShared& S, const DevCfg& C,
                                           const RowSrc& row, long long i, int e) {
  if (C.N <= 64) eval_small<PP, true>(P, S, C, row, i, e);    // bijection bitmap in registers
  else eval_small<PP, false>(P, S, C, row, i, e);
}

// MODE 1 (general) evaluation of one candidate.  PP > 0: compile-time pipeline depth for
// 16-byte rows with N % 8 == 0 (a power of two up to 32): the stage of a slot follows from
// its place in the 8-slot chunk, so the slot loop carries no stage counter or branches.
template <int PP>
__device__ __forceinline__ void eval_general(const EvalParams& P, const EvalShared& S, const DevCfg& C,
                                             const RowSrc& row, long long i) {
  const int N = C.N, pp = PP > 0 ? PP : C.pp;
  const uint32_t spn = (uint32_t)C.spn;
  for (int w = 0; w < (N + 31) / 32; ++w) S.bm[w * S.T + S.tid] = 0u;
  const uint32_t clg = 2u + S.cnt_nib, cbits = 8u >> S.cnt_nib, cmask = (1u << cbits) - 1u;   // count plane
  for (int w = 0; w < ((S.n - 1) >> clg) + 1; ++w) S.cnt[w * S.T + S.tid] = 0u;
  Mask<4> mask;
  mask.clear();
  bool ok = true;
  double tpp = 0.0, s = 0.0;
  uint32_t prev = 0;
  int x = 0;
  if constexpr (PP > 0) {
    // branch-free slots: an id >= N flags the row and is clamped to N - 1 for the (then
    // meaningless) bitmap and node updates
    const double m2 = C.m2;
    uint32_t* const bmt = S.bm + S.tid;   // this thread's bitmap column (word stride T)
    const uint32_t nm1 = (uint32_t)N - 1u;
    uint32_t bad = 0u;
    for (int w0 = 0; w0 < N; w0 += 8) {
      const uint4 v4 = row.chunk(w0 >> 3);
      const uint32_t pk[4] = {v4.x, v4.y, v4.z, v4.w};
      const bool head = PP >= 8 ? (w0 & (PP - 1)) == 0 : true;            // chunk starts a pipeline
      const bool tail = PP >= 8 ? ((w0 + 8) & (PP - 1)) == 0 : true;      // chunk ends one
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t v = (pk[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
        bad |= (uint32_t)(v > nm1);
        const uint32_t vc = min(v, nm1);
        uint32_t* const bw = bmt + (vc >> 5) * (uint32_t)S.T;
        const uint32_t bit = 1u << (vc & 31), old = *bw;
        bad |= old & bit;
        *bw = old | bit;
        const uint32_t nd = div_small(vc, C.spn_magic, spn);
        const bool st0 = PP >= 8 ? (j == 0 && head) : (j % PP) == 0;
        if (st0) {
          S.cnt[(nd >> clg) * S.T + S.tid] += 1u << ((nd & ((1u << clg) - 1u)) * cbits);
          s = 0.0;
        } else {
          s = __dadd_rn(s, __dmul_rn(m2, r_at<false>(S, prev, nd)));
        }
        prev = nd;
        const bool last = PP >= 8 ? (j == 7 && tail) : (j % PP) == PP - 1;
        if (PP >= 2 && last) tpp = dmax(tpp, s);
      }
    }
    ok = bad == 0u;
  } else {
  auto visit = [&](uint32_t v) {
    uint32_t nd = 0;
    if (v >= (uint32_t)N) {
      ok = false;
    } else {
      uint32_t& bw = S.bm[(v >> 5) * S.T + S.tid];
      const uint32_t bit = 1u << (v & 31);
      if (bw & bit) ok = false;
      bw |= bit;
      nd = div_small(v, C.spn_magic, spn);
    }
    if (x == 0) {
      S.cnt[(nd >> clg) * S.T + S.tid] += 1u << ((nd & ((1u << clg) - 1u)) * cbits);
      s = 0.0;
    } else {
      s = __dadd_rn(s, __dmul_rn(C.m2, r_at<false>(S, prev, nd)));
    }
    prev = nd;
    if (++x == pp) {
      x = 0;
      if (pp >= 2) tpp = dmax(tpp, s);
    }
  };
  if (row.vec) {
    for (int w0 = 0; w0 < N; w0 += 8) {
      const uint4 v = row.chunk(w0 >> 3);
      const uint32_t pk[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (w0 + j < N) visit((pk[j >> 1] >> ((j & 1) * 16)) & 0xffffu);
    }
  } else {
    for (int w = 0; w < N; ++w) visit(row.slot(w));
  }
  }
  P.mem[i] = C.mem;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  if (!ok) { P.latency[i] = qnan; P.status[i] = 3; return; }
  if (!C.has_profile) { P.latency[i] = qnan; P.status[i] = 4; return; }
  const double* qi = P.qtab + C.qi_off;
  double t_in = 0.0, mx = 0.0;
  // N1 (nodes with a stage-1 member) and T_in (Eq.6 intra term over nodes with >= 2) from
  // the count plane, one word of 8 nibbles (or 4 bytes) at a time: the non-zero fields
  // compressed to a byte of N1, the fields >= 2 visited for T_in (fmax: any order)
  for (int w = 0; w < ((S.n - 1) >> clg) + 1; ++w) {
    const uint32_t cw = S.cnt[w * S.T + S.tid];
    if (cw == 0u) continue;
    uint32_t nz, ge2, x = cw | (cw >> 1);
    if (S.cnt_nib) {
      x = (x | (x >> 2)) & 0x11111111u;
      x = (x | (x >> 3)) & 0x03030303u;
      x = (x | (x >> 6)) & 0x000f000fu;
      nz = ((x | (x >> 12)) & 0xffu) << ((w & 3) * 8);
      ge2 = cw & 0xeeeeeeeeu;
    } else {
      x |= x >> 2;
      x = (x | (x >> 4)) & 0x01010101u;
      x = (x | (x >> 7)) & 0x00030003u;
      nz = ((x | (x >> 14)) & 0xfu) << ((w & 7) * 4);
      ge2 = cw & 0xfefefefeu;
    }
    const uint32_t q = (uint32_t)w >> (S.cnt_nib ? 2 : 3);   // mask word
#pragma unroll
    for (int m = 0; m < 4; ++m) mask.w[m] |= q == (uint32_t)m ? nz : 0u;
    while (ge2) {
      const uint32_t sh = (uint32_t)(__ffs(ge2) - 1) & ~(cbits - 1u);
      ge2 &= ~(cmask << sh);
      const uint32_t a = ((uint32_t)w << clg) + sh / cbits, c = (cw >> sh) & cmask;
      t_in = dmax(t_in, __dmul_rn(__ldg(qi + c), r_at<false>(S, a, a)));
    }
  }
  const int k = mask.count();
  // slowest link of N1: the k(k-1) member pairs when k^2 <= n, else the first pair inside N1
  // of the R-descending pair list (expected ~(n/k)^2 probes; every thread scans the same
  // prefix, so it stays in L1).  Both give the exact max.
  // (a converged warp scans the list cooperatively, below: there the list beats the pairs
  // from k = 6 on; a lone lane probes ~(n/k)^2 pairs, so it takes the pairs while k^2 <= n)
  const bool coop = __activemask() == 0xffffffffu;
  const bool pairs = coop ? k <= 5 : k * k <= S.n;
  if (pairs) {
#pragma unroll
    for (int wd = 0; wd < 4; ++wd) {
      uint32_t bits = mask.w[wd];
      while (bits) {
        const uint32_t a = wd * 32 + __ffs(bits) - 1;
        bits &= bits - 1;
#pragma unroll
        for (int wd2 = 0; wd2 < 4; ++wd2) {
          uint32_t bits2 = mask.w[wd2];
          while (bits2) {
            const uint32_t b = wd2 * 32 + __ffs(bits2) - 1;
            bits2 &= bits2 - 1;
            if (a != b) mx = dmax(mx, r_at<false>(S, a, b));
          }
        }
      }
    }
  }
  // first pair of the R-sorted list inside N1; the value from the R table
  const bool want = !pairs && k >= 2;
  if (coop && __activemask() == 0xffffffffu) {
    // whole warp converged: one cooperative scan for all its lanes.  Every lane probes the
    // same list prefix, so the warp takes 32 consecutive pairs per round, one per lane, and
    // tests them against all 32 lanes' N1 at once through the transposed membership (lane t
    // holds, for node 32q + t, the bit set of the lanes whose N1 has it): a lane's witness
    // is its first hit in list order.  (A lane alone would probe ~(n/k)^2 pairs, the warp in
    // lockstep the max of 32 such runs.)
    const unsigned full = 0xffffffffu;
    unsigned pending = __ballot_sync(full, want);
    if (pending) {
      const int nq = (S.n + 31) >> 5;
      uint32_t mt[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {   // 32 x 32 bit transpose by five shuffle stages
        uint32_t x = mask.w[q];
        if (q < nq) {
#pragma unroll
          for (int jj = 16; jj >= 1; jj >>= 1) {
            const uint32_t m = jj == 16 ? 0x0000ffffu : (jj == 8 ? 0x00ff00ffu : (jj == 4 ? 0x0f0f0f0fu
                             : (jj == 2 ? 0x33333333u : 0x55555555u)));
            const uint32_t y = __shfl_xor_sync(full, x, jj);
            x = (S.lane & jj) ? ((x & ~m) | ((y & ~m) >> jj)) : ((x & m) | ((y & m) << jj));
          }
        }
        mt[q] = x;
      }
      const int len = S.n * (S.n - 1);
      for (int base = 0; pending != 0u && base < len; base += 32) {
        const int j = base + S.lane;
        const uint32_t ab = j < len ? (j < S.plen ? (uint32_t)S.pl[j] : (uint32_t)__ldg(P.gl_ab + j)) : 0u;
        const uint32_t a = ab & 0xffu, b = ab >> 8;
        uint32_t ma = 0u, mb = 0u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (q < nq) {
            const uint32_t xa = __shfl_sync(full, mt[q], (int)(a & 31u)), xb = __shfl_sync(full, mt[q], (int)(b & 31u));
            ma = (a >> 5) == (uint32_t)q ? xa : ma;
            mb = (b >> 5) == (uint32_t)q ? xb : mb;
          }
        }
        const uint32_t hit = j < len ? (ma & mb & pending) : 0u;
        const unsigned got = __reduce_or_sync(full, hit);   // lanes with a witness in this round
        for (unsigned todo = got; todo; todo &= todo - 1u) {
          const int l = __ffs(todo) - 1;
          const int t = __ffs(__ballot_sync(full, (hit >> l) & 1u)) - 1;
          const uint32_t abt = __shfl_sync(full, ab, t);
          if (S.lane == l) mx = r_at<false>(S, abt & 0xffu, abt >> 8);
        }
        pending &= ~got;
      }
    }
  } else if (want) {
    const int len = S.n * (S.n - 1);
    for (int j = 0; j < len; ++j) {
      const uint32_t ab = j < S.plen ? (uint32_t)S.pl[j] : (uint32_t)__ldg(P.gl_ab + j);
      if (mask.test(ab & 0xffu) && mask.test(ab >> 8)) { mx = r_at<false>(S, ab & 0xffu, ab >> 8); break; }
    }
  }
  const double t_ex = k >= 2 ? __dmul_rn(__ldg(P.qtab + C.qe_off + k), mx) : 0.0;
  P.latency[i] = compose(C.Sb, C.r, C.Ss, tpp, t_in, t_ex);
  P.status[i] = C.feasible ? 0 : 1;
}

constexpr int kEvalTile = 2048;   // candidates per block tile (bucketed by configuration)

// Gather the mapping rows of 32 candidates (tile positions ks[0..31], -1 = none) into a
// warp's staging buffer: 16-byte cp.async pieces, lanes 8r..8r+7 of a 128-byte row
// reading one whole line (coalesced), stored swizzled at row r * rb.
__device__ __forceinline__ void gather_rows(const EvalParams& P, unsigned char* wbuf, const short* ks, long long base,
                                            uint32_t rb, int lane) {
  const uint32_t pr = rb >> 4;   // pieces per row
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(wbuf);
  const unsigned char* src = reinterpret_cast<const unsigned char*>(P.perm);
  const bool pow2 = (pr & (pr - 1u)) == 0u;
  const uint32_t sh = 31u - __clz(pr);
  for (uint32_t pc = (uint32_t)lane; pc < 32u * pr; pc += 32u) {
    const uint32_t r = pow2 ? pc >> sh : pc / pr, c = pc - r * pr;
    const int k = ks[r];
    if (k >= 0)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + swz(r * rb + c * 16u)),
                   "l"(src + (size_t)(base + k) * rb + c * 16u)
                   : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// The same for 32 consecutive candidates (a tile of one configuration): their rows are one
// contiguous range of rows * rb bytes, so piece pc sits at byte pc * 16 on both sides.
__device__ __forceinline__ void gather_contig(const EvalParams& P, unsigned char* wbuf, long long first, int rows,
                                              uint32_t rb, int lane) {
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(wbuf);
  const unsigned char* src = reinterpret_cast<const unsigned char*>(P.perm) + (size_t)first * rb;
  const uint32_t bytes = (uint32_t)rows * rb;
  for (uint32_t b = (uint32_t)lane * 16u; b < bytes; b += 512u)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + swz(b)), "l"(src + b) : "memory");
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// TMA (cp.async.bulk.tensor) staging of a single-configuration tile's rows when a row is
// exactly 128 bytes (perm_stride = 64): the tensor map describes the candidate rows as a 2-D
// u16 tensor (64 x n) with SWIZZLE_128B, whose smem layout -- 16-byte chunk c of row r at
// chunk c ^ (r & 7) -- is the XOR swizzle the per-thread row reads use (swz), so one elected
// lane's copy replaces the warp's per-lane cp.async address and swizzle arithmetic.  The
// copy completes on a per-warp mbarrier (transaction bytes); rows past n are zero-filled.
__device__ __forceinline__ void tma_rows(const CUtensorMap* tmap, unsigned char* dst, uint32_t mbar, long long row0) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // (after the generic reads of the buffer)
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar), "r"(32u * 128u) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(d), "l"(reinterpret_cast<unsigned long long>(tmap)), "r"(0), "r"((int)row0), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\n"
                 : "=r"(done) : "r"(mbar), "r"(phase) : "memory");
}

template <int MODE, int THREADS>
__global__ void __launch_bounds__(THREADS, THREADS <= 256 ? 4 : 1)
    k_eval_stream(EvalParams P, const __grid_constant__ CUtensorMap tmap) {
  constexpr int kEvalThreads = THREADS;   // (block size: 256, or 768 for large clusters)
  constexpr bool REP = MODE == 0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // (TMA's 128-byte swizzle needs 1024-byte aligned destinations: the host adds 1 KB)
  unsigned char* smem = P.tma ? smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u)
                              : smem_raw;
  const int n = P.n_nodes, nn = n * n;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarps = kEvalThreads / 32;
  // layout: [warp staging buffers nwarps x 32 x rb][R][keys][per-thread scratch]
  //         [tile_e][hist][order]
  const uint32_t rb = (uint32_t)P.perm_stride * 2u;
  const bool staged = P.staged != 0;
  const uint32_t wb_bytes = staged ? 32u * rb : 0u;   // one buffer
  unsigned char* wbuf = smem + (size_t)wid * wb_bytes;
  __shared__ __align__(8) unsigned long long s_mbar[kEvalThreads / 32];
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&s_mbar[wid]);
  uint32_t mbar_phase = 0;
  if (P.tma && lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  size_t off = (size_t)nwarps * wb_bytes;
  double* Rs = reinterpret_cast<double*>(smem + off);
  const uint32_t lgn = n <= 1 ? 0u : 32u - __clz(n - 1);   // MODE 0 padded side 2^lgn >= n
  const int np = 1 << lgn;
  off += (size_t)(REP ? np * np * 16 : nn) * 8;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem + off);
  off += ((size_t)P.E * 8 + 15) & ~(size_t)15;
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem + off);
  const int cnt_words = P.cnt_nib ? (n + 7) / 8 : (n + 3) / 4;
  off += (size_t)(P.bm_words + cnt_words) * kEvalThreads * 4;
  uint16_t* pl = reinterpret_cast<uint16_t*>(smem + off);   // MODE 1: pair-list prefix
  off += ((size_t)P.plen * 2 + 15) & ~(size_t)15;
  short* tile_e = reinterpret_cast<short*>(smem + off);   // config index per candidate (E < 32767)
  int* hist = reinterpret_cast<int*>(tile_e + kEvalTile);
  short* order = reinterpret_cast<short*>(hist + ((P.E + 2 + 3) & ~3));
  __shared__ int sh_scan[32];

  if (REP) {
    for (int i = tid; i < np * np * 16; i += kEvalThreads) {
      const int a = i >> (4 + lgn), b = (i >> 4) & (np - 1);
      Rs[i] = (a < n && b < n) ? P.R[a * n + b] : 0.0;
    }
  } else {
    for (int i = tid; i < nn; i += kEvalThreads) Rs[i] = P.R[i];
  }
  for (int i = tid; i < P.E; i += kEvalThreads) keys[i] = P.keys[i];
  for (int i = tid; i < P.plen; i += kEvalThreads) pl[i] = P.gl_ab[i];
  __syncthreads();
  const EvalShared S{Rs, bm, bm + P.bm_words * kEvalThreads, pl, n, tid, lane, kEvalThreads, P.plen,
                     (uint32_t)P.cnt_nib, lgn, reinterpret_cast<const unsigned char*>(Rs + (lane & 15)),
                     (uint32_t)np * 128u};
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  const bool bucket_ok = true;   // (E < 32767 is checked by the host)
  unsigned long long last_raw = ~0ull;   // (pp = 0xffff is never a valid record)
  int last_e = -1;

  for (long long base = (long long)blockIdx.x * kEvalTile; base < P.n; base += (long long)gridDim.x * kEvalTile) {
    const int cnt_valid = (int)min((long long)kEvalTile, P.n - base);
    // configuration lookup (Alg.1 l.3-5 membership) of every candidate of the tile
    // (a thread's previous candidate usually has the same configuration: the binary search
    // runs only when the raw 8-byte record changes)
    bool mixed = false;
    for (int k = tid; k < cnt_valid; k += kEvalThreads) {
      const unsigned long long raw = __ldg(reinterpret_cast<const unsigned long long*>(P.cand) + base + k);
      if (raw != last_raw) {
        const pipette_config cf = *reinterpret_cast<const pipette_config*>(&raw);
        const unsigned long long key = ((unsigned long long)cf.pp << 48) | ((unsigned long long)cf.tp << 32) |
                                       ((unsigned long long)cf.dp << 16) | (unsigned long long)cf.mb;
        int lo = 0, hi = P.E;   // first index with keys[idx] >= key
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (keys[mid] < key) lo = mid + 1; else hi = mid;
        }
        last_e = (lo >= P.E || keys[lo] != key) ? -1 : lo;   // -1: not in the enumeration
        last_raw = raw;
      }
      tile_e[k] = (short)last_e;
    }
    __syncthreads();
    for (int k = tid; k < cnt_valid; k += kEvalThreads) mixed |= tile_e[k] != tile_e[0];
    // a tile of one configuration is evaluated in candidate order (coalesced rows and
    // outputs); a mixed tile is bucketed by configuration so a warp shares a code path
    mixed = __syncthreads_or(mixed) && bucket_ok;
    if (mixed) {
      for (int k = tid; k <= P.E; k += kEvalThreads) hist[k] = 0;
      __syncthreads();
      for (int k = tid; k < cnt_valid; k += kEvalThreads) atomicAdd(&hist[tile_e[k] + 1], 1);
      __syncthreads();
      int carry = 0;
      for (int b0 = 0; b0 <= P.E; b0 += kEvalThreads) {
        const int k = b0 + tid;
        const int v = k <= P.E ? hist[k] : 0;
        int tot;
        const int ex = carry + block_scan_excl_eval(v, sh_scan, tot);
        carry += tot;
        if (k <= P.E) hist[k] = ex;
      }
      __syncthreads();
      for (int k = tid; k < cnt_valid; k += kEvalThreads) order[atomicAdd(&hist[tile_e[k] + 1], 1)] = (short)k;
    } else {
      for (int k = tid; k < kEvalTile; k += kEvalThreads) order[k] = (short)k;
    }
    if (staged)   // sentinel past the tile: gathers of the last group skip missing rows
      for (int k = cnt_valid + tid; k < kEvalTile; k += kEvalThreads) order[k] = -1;
    __syncthreads();

    // warp w takes the groups of 32 sorted positions g = w, w + 8, ...; its rows stream
    // into one half of its staging buffer while the other half is evaluated
    const int groups = (cnt_valid + 31) >> 5;
    for (int g = wid; g < groups; g += nwarps) {
      unsigned char* cur = wbuf;
      if (staged) {   // (one buffer per warp: the other resident warps hide the gather)
        if (!mixed && P.tma) {   // one elected lane, the tensor engine does the copy
          if (lane == 0) tma_rows(&tmap, wbuf, mbar, base + (long long)g * 32);
          mbar_wait(mbar, mbar_phase);
          mbar_phase ^= 1u;
        } else {
          if (mixed) gather_rows(P, wbuf, order + g * 32, base, rb, lane);
          else gather_contig(P, wbuf, base + (long long)g * 32, min(32, cnt_valid - g * 32), rb, lane);
          asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncwarp();
      }
      const int sidx = g * 32 + lane;
      if (sidx < cnt_valid) {
        const int k = order[sidx];
        const long long i = base + k;
        const int e = tile_e[k];
        if (e < 0) {
          P.latency[i] = qnan; P.mem[i] = 0ull; P.status[i] = 2;
        } else {
          const DevCfg C = P.cfgs[e];
          if (C.N > P.perm_stride) {   // the row cannot hold a mapping of [0, N): never read past it
            P.latency[i] = qnan; P.mem[i] = C.mem; P.status[i] = 3;
          } else {
          RowSrc row;
          row.sbuf = staged ? cur : nullptr;
          row.roff = (uint32_t)lane * rb;
          row.g = P.perm + i * (long long)P.perm_stride;
          row.vec = P.vec16 != 0;
          if (MODE == 0) {
            switch (C.pp) {
              case 1: dispatch_n<1>(P, S, C, row, i, e); break;
              case 2: dispatch_n<2>(P, S, C, row, i, e); break;
              case 4: dispatch_n<4>(P, S, C, row, i, e); break;
              case 8: dispatch_n<8>(P, S, C, row, i, e); break;
              default: dispatch_n<0>(P, S, C, row, i, e); break;
            }
          } else if (!mixed && row.vec && (C.N & 7) == 0) {
            // single-configuration tile: compile-time depth (mixed tiles take the generic pass:
            // warps of several depths on one SM thrash the instruction cache -- measured C4
            // mixed 3.8e9 -> 2.2e9 candidates/s with per-depth code there)
            switch (C.pp) {
              case 1: eval_general<1>(P, S, C, row, i); break;
              case 2: eval_general<2>(P, S, C, row, i); break;
              case 4: eval_general<4>(P, S, C, row, i); break;
              case 8: eval_general<8>(P, S, C, row, i); break;
              case 16: eval_general<16>(P, S, C, row, i); break;
              case 32: eval_general<32>(P, S, C, row, i); break;
              default: eval_general<0>(P, S, C, row, i); break;
            }
          } else {
            eval_general<0>(P, S, C, row, i);
          }
          }
        }
      }
      __syncwarp();   // the buffer is refilled by the next group
    }
    __syncthreads();
  }
}

int eval_tile_size() { return kEvalTile; }

// Dynamic shared memory of k_eval_stream (staged: per-warp row staging; cnt_nib: nibble
// counts; plen: pair-list prefix entries; threads: block size).
size_t eval_smem_bytes(int mode, int perm_stride, bool staged, int n_nodes, int E, int bm_words, int threads,
                       bool cnt_nib, int plen) {
  const size_t nn = (size_t)n_nodes * n_nodes;
  const size_t wb = staged ? (size_t)32 * perm_stride * 2 : 0;
  size_t np = 1;
  while (np < (size_t)n_nodes) np <<= 1;
  const size_t cnt_words = cnt_nib ? (n_nodes + 7) / 8 : (n_nodes + 3) / 4;
  return (size_t)(threads / 32) * wb + (mode == 0 ? np * np * 16 : nn) * 8 + (((size_t)E * 8 + 15) & ~(size_t)15) +
         (size_t)(bm_words + cnt_words) * threads * 4 + (((size_t)plen * 2 + 15) & ~(size_t)15) +
         (size_t)kEvalTile * sizeof(short) + (size_t)((E + 2 + 3) & ~3) * sizeof(int) + (size_t)kEvalTile * sizeof(short);
}

// qi(c) R[a][a] for every enumerated config, node a < n <= 16 and c < 16 (0 for c < 2):
// the intra-node term of Eq.6 by lookup in K2 MODE 0.  One block per config.
__global__ void k_tin_values(const DevCfg* __restrict__ cfgs, const double* __restrict__ qtab,
                             const double* __restrict__ R, int n, double* __restrict__ vin) {
  const int e = blockIdx.x;
  const DevCfg C = cfgs[e];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    const int a = i >> 4, c = i & 15;
    vin[(size_t)e * 256 + i] = (a < n && c >= 2 && c <= C.dp) ? __dmul_rn(qtab[C.qi_off + c], R[a * n + a]) : 0.0;
  }
}

// Host-side handle of the K2 variant (MODE 0 small clusters, 1 general).
const void* eval_kernel(int mode, int threads) {
  if (mode == 0) return (const void*)k_eval_stream<0, 256>;
  return threads == 768 ? (const void*)k_eval_stream<1, 768> : (const void*)k_eval_stream<1, 256>;
}

}  // namespace pip

namespace pip {

// ------------------------------------------------------------------ K2 MODE 1: warp per candidate
// Large clusters (n > 16 nodes or more than 15 slots per node), where a candidate's mapping is
// long (N up to 1024) and Eq.6's stage-1 set has many nodes: one WARP per candidate
// (north_star: "one warp per candidate ... lane-parallel reductions over links and stages
// via warp shuffles").  The row is read coalesced across the lanes (slot p by lane p mod 32),
// the bijection is tested with a per-warp bitmap (atomicOr: a duplicate finds its bit set),
// node ids go to a per-warp byte array; lane z sums pipeline z of Eq.5 in stage order (the
// normative order), T_PP is a shuffle max; stage-1 counts are per-warp byte counters, N1 a
// 128-bit mask OR-reduced over the lanes; T_ex takes the k(k-1) member pairs split over the
// lanes (k <= 16) or the first pair inside N1 of the R-descending pair list, 32 probes per
// round.  R (n x n) lives in shared memory; one block of 16 warps per SM.
constexpr int kEvalWarpThreads = 512;
constexpr int kEvalWarpMaxN = 1024;   // (G <= 1024)

struct WarpScratch {
  uint32_t bm[kEvalWarpMaxN / 32];   // bijection bitmap
  uint32_t cnt[kMaxNodes / 4];       // stage-1 member counts, bytes (c_n <= gpus_per_node <= 255)
  uint8_t nd[kEvalWarpMaxN];         // node of every position
};

// Warp max of non-negative doubles: their bit patterns order like the values, so two 32-bit
// redux.sync on the halves (instead of a five-level shuffle butterfly of doubles).
__device__ __forceinline__ double warp_max(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const uint32_t hi = (uint32_t)(b >> 32);
  const uint32_t H = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t L = __reduce_max_sync(0xffffffffu, hi == H ? (uint32_t)b : 0u);
  return __longlong_as_double((long long)(((unsigned long long)H << 32) | L));
}

// One candidate, processed by the whole warp (raw = its 8-byte configuration record, ch =
// this lane's 16-byte chunk of the row when the row is read as one uint4 per lane).
__device__ __forceinline__ void eval_warp_one(const EvalParams& P, const double* Rs, const unsigned long long* keys,
                                              WarpScratch* ws, long long i, unsigned long long raw, const uint4& ch,
                                              bool vec, unsigned long long& last_raw, int& e, int lane) {
  const unsigned full = 0xffffffffu;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  const int n = P.n_nodes;
  // configuration lookup (Alg.1 l.3-5 membership), warp-uniform; repeated records skip it
  if (raw != last_raw) {
    const pipette_config cf = *reinterpret_cast<const pipette_config*>(&raw);
    const unsigned long long key = ((unsigned long long)cf.pp << 48) | ((unsigned long long)cf.tp << 32) |
                                   ((unsigned long long)cf.dp << 16) | (unsigned long long)cf.mb;
    int lo = 0, hi = P.E;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (keys[mid] < key) lo = mid + 1; else hi = mid;
    }
    e = (lo >= P.E || keys[lo] != key) ? -1 : lo;
    last_raw = raw;
  }
  if (e < 0) {
    if (lane == 0) { P.latency[i] = qnan; P.mem[i] = 0ull; P.status[i] = 2; }
    return;
  }
  const DevCfg C = P.cfgs[e];
  const int N = C.N, pp = C.pp, dp = C.dp;
  if (N > P.perm_stride || N > kEvalWarpMaxN) {   // the row cannot hold a mapping of [0, N)
    if (lane == 0) { P.latency[i] = qnan; P.mem[i] = C.mem; P.status[i] = 3; }
    return;
  }
  // ---- the row: bijection (Eq.2) and the node of every position
  for (int w = lane; w < (N + 31) / 32; w += 32) ws->bm[w] = 0u;
  for (int w = lane; w < (n + 3) / 4; w += 32) ws->cnt[w] = 0u;
  __syncwarp();
  // bijection: every id < N, and the union of the ids' bits (fire-and-forget atomicOr into
  // the warp's bitmap) has N bits -- a duplicate leaves one of them unset
  bool bad = false;
  if (vec) {   // slots 8 lane .. 8 lane + 7 from this lane's prefetched chunk; nodes stored as 8 bytes
    const uint32_t wv[4] = {ch.x, ch.y, ch.z, ch.w};
    uint32_t nw0 = 0u, nw1 = 0u;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int p = lane * 8 + j;
      const uint32_t v = (wv[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
      if (p < N) {
        if (v >= (uint32_t)N) bad = true;
        else atomicOr(&ws->bm[v >> 5], 1u << (v & 31));
        const uint32_t nd = div_small(min(v, (uint32_t)N - 1u), C.spn_magic, (uint32_t)C.spn);
        if (j < 4) nw0 |= nd << (8 * j); else nw1 |= nd << (8 * (j - 4));
      }
    }
    if (lane * 8 < N) *reinterpret_cast<uint2*>(ws->nd + lane * 8) = make_uint2(nw0, nw1);
  } else {
    const uint16_t* row = P.perm + i * (long long)P.perm_stride;
    for (int p = lane; p < N; p += 32) {
      const uint32_t v = __ldg(row + p);
      if (v >= (uint32_t)N) {
        bad = true;
      } else {
        atomicOr(&ws->bm[v >> 5], 1u << (v & 31));
        ws->nd[p] = (uint8_t)div_small(v, C.spn_magic, (uint32_t)C.spn);
      }
    }
  }
  __syncwarp();
  {
    int c = 0;
    for (int w = lane; w < (N + 31) / 32; w += 32) c += __popc(ws->bm[w]);
    bad |= (int)__reduce_add_sync(full, (uint32_t)c) != N;
  }
  if (__any_sync(full, bad) || !C.has_profile) {
    if (lane == 0) { P.latency[i] = qnan; P.mem[i] = C.mem; P.status[i] = C.has_profile ? 3 : 4; }
    __syncwarp();
    return;
  }
  __syncwarp();
  // ---- Eq.5: lane z sums pipeline z in stage order; T_PP = max over pipelines
  double tpp = 0.0;
  uint32_t m0 = 0u, m1 = 0u, m2w = 0u, m3 = 0u;   // N1 bits held by this lane
  for (int z = lane; z < dp; z += 32) {
    const int b = z * pp;
    uint32_t prev = ws->nd[b];
    double s = 0.0;
    if ((pp & 3) == 0) {   // the pipeline's node bytes as whole words
      const uint32_t* nw = reinterpret_cast<const uint32_t*>(ws->nd + b);
      uint32_t wd = nw[0];
      for (int x = 1; x < pp; ++x) {
        if ((x & 3) == 0) wd = nw[x >> 2];
        const uint32_t cur = __byte_perm(wd, 0u, 0x4440u | (uint32_t)(x & 3));
        s = __dadd_rn(s, __dmul_rn(C.m2, Rs[prev * (uint32_t)n + cur]));
        prev = cur;
      }
    } else {
      for (int x = 1; x < pp; ++x) {
        const uint32_t cur = ws->nd[b + x];
        s = __dadd_rn(s, __dmul_rn(C.m2, Rs[prev * (uint32_t)n + cur]));
        prev = cur;
      }
    }
    tpp = dmax(tpp, s);
    const uint32_t a = ws->nd[b];           // stage-1 worker of pipeline z (Eq.6)
    atomicAdd(&ws->cnt[a >> 2], 1u << ((a & 3) * 8));
    const uint32_t bit = 1u << (a & 31), q = a >> 5;
    m0 |= q == 0u ? bit : 0u; m1 |= q == 1u ? bit : 0u; m2w |= q == 2u ? bit : 0u; m3 |= q == 3u ? bit : 0u;
  }
  tpp = warp_max(tpp);
  Mask4 m;
  m.w0 = __reduce_or_sync(full, m0); m.w1 = __reduce_or_sync(full, m1);
  m.w2 = __reduce_or_sync(full, m2w); m.w3 = __reduce_or_sync(full, m3);
  __syncwarp();
  // ---- Eq.6, intra: nodes with c >= 2 stage-1 members (each counted by its pipelines' lanes)
  double tin = 0.0;
  for (int z = lane; z < dp; z += 32) {
    const uint32_t a = ws->nd[z * pp];
    const uint32_t c = (ws->cnt[a >> 2] >> ((a & 3) * 8)) & 0xffu;
    if (c >= 2u) tin = dmax(tin, __dmul_rn(__ldg(P.qtab + C.qi_off + c), Rs[a * (uint32_t)n + a]));
  }
  tin = warp_max(tin);
  // ---- Eq.6, inter: the slowest link among the k stage-1 nodes
  const int k = m.count();
  double mx = 0.0;
  if (k >= 2) {
    if (k <= 16) {   // the k(k-1) member pairs over the lanes; lane t holds member t
      uint32_t memv = 0u;
      {
        const uint32_t c0 = __popc(m.w0), c1 = c0 + __popc(m.w1), c2 = c1 + __popc(m.w2);
        const uint32_t t = (uint32_t)lane;
        const uint32_t wd = t < c0 ? 0u : (t < c1 ? 1u : (t < c2 ? 2u : 3u));
        const uint32_t r = t - (wd == 0u ? 0u : (wd == 1u ? c0 : (wd == 2u ? c1 : c2)));
        if (t < (uint32_t)k) memv = wd * 32u + (uint32_t)__fns(m.word((int)wd), 0u, (int)r + 1);
      }
      const uint32_t kk = (uint32_t)k, npair = kk * kk;
      const uint32_t mg = (uint32_t)((0x100000000ull + kk - 1u) / kk);
      for (uint32_t base = 0; base < npair; base += 32u) {
        const uint32_t j = base + (uint32_t)lane;
        const uint32_t ia = __umulhi(j, mg), ib = j - ia * kk;
        const uint32_t a = __shfl_sync(full, memv, (int)(ia & 31u)), b = __shfl_sync(full, memv, (int)(ib & 31u));
        if (j < npair && ia != ib) mx = dmax(mx, Rs[a * (uint32_t)n + b]);
      }
      mx = warp_max(mx);
    } else {         // first pair of the R-descending list inside N1 (expected (n/k)^2 probes)
      const int len = n * (n - 1);
      for (int base = 0; base < len; base += 32) {
        const int j = base + lane;
        uint32_t ab = 0u;
        bool h = false;
        if (j < len) {
          ab = __ldg(P.gl_ab + j);
          h = m.test(ab & 0xffu) && m.test(ab >> 8);
        }
        const unsigned bal = __ballot_sync(full, h);
        if (bal) {
          ab = __shfl_sync(full, ab, __ffs(bal) - 1);
          mx = Rs[(ab & 0xffu) * (uint32_t)n + (ab >> 8)];
          break;
        }
      }
    }
  }
  if (lane == 0) {
    const double tex = k >= 2 ? __dmul_rn(__ldg(P.qtab + C.qe_off + k), mx) : 0.0;
    P.latency[i] = compose(C.Sb, C.r, C.Ss, tpp, tin, tex);
    P.mem[i] = C.mem;
    P.status[i] = C.feasible ? 0 : 1;
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kEvalWarpThreads, 1) k_eval_warp(EvalParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int n = P.n_nodes, nn = n * n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = kEvalWarpThreads / 32;
  double* Rs = reinterpret_cast<double*>(smem);
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem + (size_t)nn * 8);
  WarpScratch* ws = reinterpret_cast<WarpScratch*>(smem + (size_t)nn * 8 + (((size_t)P.E * 8 + 15) & ~(size_t)15)) + wid;
  for (int i = threadIdx.x; i < nn; i += blockDim.x) Rs[i] = P.R[i];
  for (int i = threadIdx.x; i < P.E; i += blockDim.x) keys[i] = P.keys[i];
  __syncthreads();
  // rows of up to 256 slots in 16-byte aligned rows: one uint4 per lane, prefetched two
  // candidates ahead (the loads of the next rows are in flight while this one is evaluated)
  const bool vec = P.vec16 != 0 && P.perm_stride <= 256;
  const long long step = (long long)gridDim.x * nwarps;
  const unsigned long long* cand = reinterpret_cast<const unsigned long long*>(P.cand);
  auto fetch = [&](long long j, unsigned long long& raw, uint4& ch) {
    raw = ~0ull;
    ch = make_uint4(0u, 0u, 0u, 0u);
    if (j < P.n) {
      raw = __ldg(cand + j);
      if (vec && lane * 8 < P.perm_stride)
        ch = __ldg(reinterpret_cast<const uint4*>(P.perm + j * (long long)P.perm_stride) + lane);
    }
  };
  unsigned long long last_raw = ~0ull;
  int e = -1;
  long long i = (long long)blockIdx.x * nwarps + wid;
  unsigned long long r0, r1, r2;
  uint4 c0, c1, c2;
  fetch(i, r0, c0);
  fetch(i + step, r1, c1);
  for (; i < P.n; i += step) {
    fetch(i + 2 * step, r2, c2);
    eval_warp_one(P, Rs, keys, ws, i, r0, c0, vec, last_raw, e, lane);
    r0 = r1; c0 = c1; r1 = r2; c1 = c2;
  }
}

const void* eval_warp_kernel() { return (const void*)k_eval_warp; }
size_t eval_warp_smem_bytes(int n_nodes, int E) {
  return (size_t)n_nodes * n_nodes * 8 + (((size_t)E * 8 + 15) & ~(size_t)15) +
         (size_t)(kEvalWarpThreads / 32) * sizeof(WarpScratch);
}
int eval_warp_threads() { return kEvalWarpThreads; }

}  // namespace pip
