// sa_mode1.cuh -- K3 MODE 1 (n <= 128 nodes, N <= 256 positions): one warp task of SA
// chains with slot-byte chain state, Eq.5 sums from the block's shared R table, and the
// stage-1 (Eq.6) state S1M.  Included by k_sa.cu inside namespace pip, after the pieces it
// shares with MODE 0 and 2 (HcState, S1Ctx, Mask4, compose, metropolis_fast, draws); it is
// not a standalone header.
//
// Design ("K3 MODE 1"):
//   - the block holds the cluster's R = 1/B in shared memory, row stride 2^lg >= n, loaded
//     once per block (every configuration shares it).  A hop of Eq.5 is fl(m2 * R[a][b]),
//     the product the oracle forms, and Eq.6's pair maxima read exact R values from the
//     same table, so no search needs a round trip to L2 for a value;
//   - T_ex (the slowest inter-node pair of the stage-1 node set N1, R10) keeps a canonical
//     witness: the first pair of the global R-descending pair list (ties by index) that
//     lies inside N1.  A node joining N1 can only move the witness to one of its own pairs
//     ranked before it: a per-lane scan of the node's pair row (global-list order) stops at
//     the witness's rank, so it is a probe or two.  Only when the witness pair itself
//     leaves N1 is the global list scanned, from the old witness's rank on, by the whole
//     warp (32 probes per round, the list prefix in shared memory).  Configurations whose
//     N1 never exceeds 8 nodes use the member pairs directly instead (<= 56 loads);
//   - T_in (nodes with >= 2 stage-1 members, R10) keeps a witness node and the per-config
//     sorted (node, count) list (S1Large's scheme); spn = 1 configurations have no counts;
//   - the per-warp region (slot plane, count plane, pipeline-sum cache) has a
//     per-configuration size, so blocks run as many warps as their configuration's state
//     fits (task flags, built by the host).
#pragma once

constexpr int kNoWit = 0x7fffffff;         // no T_ex witness (|N1| < 2)

// Block context of MODE 1 (also used by the full move set of MODE 0 with its hop-code table).
// P2 (the swap kernel; the host routes clusters whose gpus_per_node is not a power of two to
// MODE 2): spn is a power of two, node(slot) = slot >> sh, and the four nodes of a slot word
// are (word >> sh) & bmask in one shift and one AND.
template <bool P2 = false>
struct SbCtxT {
  static constexpr bool kP2 = P2;
  const double* T;   // MODE 1: R = 1/B, row stride 2^lg; MODE 0: the 16-copy m2*R hop-code table
  double m2;
  uint32_t lg;
  int n;
  uint32_t spn, spn_magic, spn_sh;
  uint32_t m16;      // ceil(2^16 / spn)
  uint32_t sh, bmask, rowmul, tbase;   // P2: log2(spn), per-byte node mask, 8 << lg, shared address of T
  // node = floor(slot / spn): a shift (P2), else (slot * m16) >> 16, exact for slot < 256 and
  // spn < 256 (the error slot * (m16 - 2^16/spn) / 2^16 < 1/256 never crosses an integer)
  __device__ __forceinline__ uint32_t node(uint32_t slot) const { return P2 ? slot >> sh : (slot * m16) >> 16; }
  __device__ __forceinline__ double r(uint32_t a, uint32_t b) const { return T[(a << lg) + b]; }
  // the Eq.5 hop term fl(m2 * R[a][b]) (MODE 1)
  __device__ __forceinline__ double hop(uint32_t a, uint32_t b) const { return __dmul_rn(m2, r(a, b)); }
  // R at a shared-memory byte address (P2 sums: row address + 8 * column, one LEA)
  __device__ __forceinline__ double ld(uint32_t addr) const {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));   // (the table is read-only here)
    return v;
  }
};
using SbCtx = SbCtxT<false>;

template <int PP, class KT>
__device__ __forceinline__ double sb_sum(const HcState& st, uint32_t z, int pp_rt, const KT& K) {
  double s = 0.0;
  if constexpr (PP >= 4 && KT::kP2) {   // node words, row addresses: ~6 instructions per hop
    constexpr int NW = PP / 4;
    uint32_t wd[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) wd[k] = (st.hw[(z * (uint32_t)NW + (uint32_t)k) * 32u] >> K.sh) & K.bmask;
    uint32_t row = K.tbase + (wd[0] & 0xffu) * K.rowmul;
#pragma unroll
    for (int x = 1; x < PP; ++x) {
      const uint32_t cur = __byte_perm(wd[x >> 2], 0u, 0x4440u | (uint32_t)(x & 3));
      s = __dadd_rn(s, __dmul_rn(K.m2, K.ld(row + cur * 8u)));
      row = K.tbase + cur * K.rowmul;
    }
  } else if constexpr (PP >= 4) {
    constexpr int NW = PP / 4;
    uint32_t wd[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) wd[k] = st.hw[(z * (uint32_t)NW + (uint32_t)k) * 32u];
    uint32_t prev = K.node(wd[0] & 0xffu);
#pragma unroll
    for (int x = 1; x < PP; ++x) {
      const uint32_t cur = K.node(__byte_perm(wd[x >> 2], 0u, 0x4440u | (uint32_t)(x & 3)));
      s = __dadd_rn(s, K.hop(prev, cur));
      prev = cur;
    }
  } else {
    const int pp = PP > 0 ? PP : pp_rt;
    const uint32_t b = z * (uint32_t)pp;
    uint32_t prev = K.node(st.hb[HcState::off(b)]);
    for (int x = 1; x < pp; ++x) {
      const uint32_t cur = K.node(st.hb[HcState::off(b + (uint32_t)x)]);
      s = __dadd_rn(s, K.hop(prev, cur));
      prev = cur;
    }
  }
  return s;
}

// Two pipelines in one interleaved loop (two independent DMUL/DADD chains); za == zb allowed.
template <int PP, class KT>
__device__ __forceinline__ void sb_sum2(const HcState& st, uint32_t za, uint32_t zb, int pp_rt, const KT& K,
                                        double& sa, double& sb) {
  double a = 0.0, b = 0.0;
  if constexpr (PP >= 4 && KT::kP2) {   // node words, row addresses: ~6 instructions per hop
    constexpr int NW = PP / 4;
    uint32_t wa[NW], wb[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      wa[k] = (st.hw[(za * (uint32_t)NW + (uint32_t)k) * 32u] >> K.sh) & K.bmask;
      wb[k] = (st.hw[(zb * (uint32_t)NW + (uint32_t)k) * 32u] >> K.sh) & K.bmask;
    }
    uint32_t ra = K.tbase + (wa[0] & 0xffu) * K.rowmul, rb = K.tbase + (wb[0] & 0xffu) * K.rowmul;
#pragma unroll
    for (int x = 1; x < PP; ++x) {
      const uint32_t ca = __byte_perm(wa[x >> 2], 0u, 0x4440u | (uint32_t)(x & 3));
      const uint32_t cb = __byte_perm(wb[x >> 2], 0u, 0x4440u | (uint32_t)(x & 3));
      a = __dadd_rn(a, __dmul_rn(K.m2, K.ld(ra + ca * 8u)));
      b = __dadd_rn(b, __dmul_rn(K.m2, K.ld(rb + cb * 8u)));
      ra = K.tbase + ca * K.rowmul;
      rb = K.tbase + cb * K.rowmul;
    }
  } else if constexpr (PP >= 4) {
    constexpr int NW = PP / 4;
    uint32_t wa[NW], wb[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      wa[k] = st.hw[(za * (uint32_t)NW + (uint32_t)k) * 32u];
      wb[k] = st.hw[(zb * (uint32_t)NW + (uint32_t)k) * 32u];
    }
    uint32_t pa = K.node(wa[0] & 0xffu), pb = K.node(wb[0] & 0xffu);
#pragma unroll
    for (int x = 1; x < PP; ++x) {
      const uint32_t ca = K.node(__byte_perm(wa[x >> 2], 0u, 0x4440u | (uint32_t)(x & 3)));
      const uint32_t cb = K.node(__byte_perm(wb[x >> 2], 0u, 0x4440u | (uint32_t)(x & 3)));
      a = __dadd_rn(a, K.hop(pa, ca));
      b = __dadd_rn(b, K.hop(pb, cb));
      pa = ca;
      pb = cb;
    }
  } else {
    const int pp = PP > 0 ? PP : pp_rt;
    const uint32_t ba = za * (uint32_t)pp, bb = zb * (uint32_t)pp;
    uint32_t pa = K.node(st.hb[HcState::off(ba)]), pb = K.node(st.hb[HcState::off(bb)]);
    for (int x = 1; x < pp; ++x) {
      const uint32_t ca = K.node(st.hb[HcState::off(ba + (uint32_t)x)]);
      const uint32_t cb = K.node(st.hb[HcState::off(bb + (uint32_t)x)]);
      a = __dadd_rn(a, K.hop(pa, ca));
      b = __dadd_rn(b, K.hop(pb, cb));
      pa = ca;
      pb = cb;
    }
  }
  sa = a;
  sb = b;
}

// T_PP of a lane's tentative mapping when its unique max pipeline decreased: the max over
// all dp Eq.5 sums and its multiplicity, computed by the whole warp (called converged).
// For each flagged lane L, lane j takes pipelines j, j + 32, ... -- lane L's cached sums,
// which already hold the two touched pipelines' new sums (cache), or re-summed in stage order
// from lane L's slot plane, which already holds the tentative swap.  The reads hit one bank (lane L's
// column), so they cost shared-memory wavefronts, not the divergent per-lane loop over all
// dp pipelines that one lane's rescan would make its warp execute.
template <int PP, class KT>
__device__ __forceinline__ void coop_tpp(bool need, unsigned char* ws, const double* psum, bool cache, int dp, int pp,
                                         uint32_t zp, uint32_t zb, double sA, double sB, const KT& K, int lane,
                                         double& tpp2, int& nmax2) {
  const unsigned full = 0xffffffffu;
  __syncwarp();   // (flagged lanes' tentative cache writes are visible to the warp)
  for (unsigned todo = __ballot_sync(full, need); todo; todo &= todo - 1u) {
    const int L = __ffs(todo) - 1;
    HcState stL;
    stL.hb = ws + L * 4;
    stL.sb = stL.hb;
    stL.hw = reinterpret_cast<const uint32_t*>(ws) + L;
    double m = 0.0;
    int c = 0;
    for (int z = lane; z < dp; z += 32) {
      const double v = cache ? psum[z * 32 + L]
                             : sb_sum<PP, KT>(stL, (uint32_t)z, pp, K);
      c = v > m ? 1 : c + (v == m ? 1 : 0);
      m = dmax(m, v);
    }
    uint32_t cnt;
    m = warp_max_nonneg(m, (uint32_t)c, cnt);   // (max, count at max) over the lanes
    if (lane == L) { tpp2 = m; nmax2 = (int)cnt; }
  }
}

// [slot plane][stage-1 counts: bytes, or nibbles when nib][psum]
__host__ __device__ inline int sb_count_bytes(int n, bool nib) { return align16((nib ? (n + 7) / 8 : (n + 3) / 4) * 128); }
// [slot plane][stage-1 counts][psum cache][direct mode: N1 member bytes, 2 words per lane]
__host__ __device__ inline int m1_warp_state_bytes(int N, int dp, int n, bool counts, bool cache, bool nib,
                                                   bool direct) {
  return align16(((N + 3) / 4) * 128) + (counts ? sb_count_bytes(n, nib) : 0) + (cache ? align16(dp * 256) : 0) +
         (direct ? 256 : 0);
}

// ------------------------------------------------------------------ stage-1 state (Eq.6)
// Direct-mode joins of one step go through the warp when at most this many lanes have one,
// else per lane: measured on B200, always cooperative on C5 (128 nodes, N <= 256: 847 vs
// 871 ms per search at 0), at most 2 on C4 (32 nodes, N = 32: a stage-1 move in ~3x more
// proposals; 40.2 ms vs 63.7 always cooperative).  Build-time override for A/B runs.
#ifndef PIPETTE_JOIN_COOP_MAX
#define PIPETTE_JOIN_COOP_MAX -1
#endif
__device__ __forceinline__ int join_coop_max(int n) {
  return PIPETTE_JOIN_COOP_MAX >= 0 ? PIPETTE_JOIN_COOP_MAX : (n >= 64 ? 32 : 2);
}

struct S1M {
  uint32_t* c;   // count plane [ceil(n / per-word)][32] (counts configurations only)
  uint32_t* ml;  // direct mode: N1's member nodes as bytes, any order, [2][32] (k bytes valid)
  int lane;
  uint32_t lgw = 2u, bw = 8u, cm = 0xffu;   // log2 counts per word, bits per count, count mask
  bool counts, direct;
  Mask4 mask, mask2;                         // N1 and its tentative successor
  int k, k2, win, win2, jw, jw2;             // |N1|; T_in witness node; T_ex witness rank
  uint32_t wab, wab2;                        // T_ex witness pair a | b << 8 (0xffff: none)
  uint32_t dn_, up_, c_dn_, c_up_;
  bool need_tin, need_scan, need_join;
  double tin, tin2, tex, tex2, maxR, maxR2;

  __device__ __forceinline__ void set_nibbles(bool nib) {   // (nibbles: every count <= 15)
    lgw = nib ? 3u : 2u; bw = nib ? 4u : 8u; cm = nib ? 0xfu : 0xffu;
  }
  __device__ __forceinline__ uint32_t get_of(uint32_t a, int L) const {
    return (c[(a >> lgw) * 32 + L] >> ((a & ((1u << lgw) - 1u)) * bw)) & cm;
  }
  __device__ __forceinline__ uint32_t get(uint32_t a) const { return counts ? get_of(a, lane) : (uint32_t)mask.test(a); }
  __device__ __forceinline__ void add(uint32_t a, int delta) {
    uint32_t& w = c[(a >> lgw) * 32 + lane];
    const uint32_t sh = (a & ((1u << lgw) - 1u)) * bw;
    w = delta > 0 ? w + (1u << sh) : w - (1u << sh);
  }
  static __device__ __forceinline__ uint32_t pair_at(const S1Ctx& X, int j) {
    return j < X.plen ? (uint32_t)X.pl[j] : (uint32_t)__ldg(X.gl_ab + j);
  }

  // max over ordered member pairs a != b of m of R[a][b], with a witness pair
  template <class KT>
  static __device__ __forceinline__ double pairs_max(const Mask4& m, const KT& K, uint32_t& wab_o) {
    double mx = 0.0;
    uint32_t w = 0xffffu;
#pragma unroll
    for (int wd = 0; wd < 4; ++wd) {
      uint32_t ba = m.word(wd);
      while (ba) {
        const uint32_t a = (uint32_t)(wd * 32 + __ffs(ba) - 1);
        ba &= ba - 1;
#pragma unroll
        for (int wd2 = 0; wd2 < 4; ++wd2) {
          uint32_t bb = m.word(wd2);
          while (bb) {
            const uint32_t b = (uint32_t)(wd2 * 32 + __ffs(bb) - 1);
            bb &= bb - 1;
            if (b == a) continue;
            const double v = K.r(a, b);
            if (v > mx) { mx = v; w = a | (b << 8); }
          }
        }
      }
    }
    wab_o = w;
    return mx;
  }
  // max over members b != u of m of R[u][b] and R[b][u] (per lane)
  template <class KT>
  static __device__ __forceinline__ double join_max(const Mask4& m, uint32_t u, const KT& K, uint32_t& wab_o) {
    double mx = 0.0;
    uint32_t w = 0xffffu;
#pragma unroll
    for (int wd = 0; wd < 4; ++wd) {
      uint32_t bb = m.word(wd);
      while (bb) {
        const uint32_t b = (uint32_t)(wd * 32 + __ffs(bb) - 1);
        bb &= bb - 1;
        if (b == u) continue;
        const double v1 = K.r(u, b), v2 = K.r(b, u);
        if (v1 > mx) { mx = v1; w = u | (b << 8); }
        if (v2 > mx) { mx = v2; w = b | (u << 8); }
      }
    }
    wab_o = w;
    return mx;
  }
  // first pair of node u's row (global-list order) with list rank < lim whose other node is
  // in m: the only pairs a joining node can put ahead of the current witness
  static __device__ __forceinline__ bool partner_scan(uint32_t u, const Mask4& m, int lim, const S1Ctx& X, int& j_o,
                                                      uint32_t& ab_o) {
    const uint4* row = reinterpret_cast<const uint4*>(X.pt + (size_t)u * (size_t)X.pt_stride);
    for (int i = 0; i < X.nl_len; i += 4) {   // (the padding's rank 0xffff ends a partial last chunk)
      const uint4 e4 = __ldg(row + (i >> 2));
      const uint32_t e[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int g = (int)(e[t] & 0xffffu);
        if (g >= lim) return false;
        const uint32_t o = (e[t] >> 16) & 0xffu;
        if (m.test(o)) { j_o = g; ab_o = (e[t] >> 24) ? (u | (o << 8)) : (o | (u << 8)); return true; }
      }
    }
    return false;
  }

  __device__ __forceinline__ void clear(int n) {
    if (counts)
      for (int wd = 0; wd < ((n - 1) >> lgw) + 1; ++wd) c[wd * 32 + lane] = 0u;
    mask.clear();
  }
  __device__ __forceinline__ void add_init(uint32_t a) {
    if (counts) add(a, +1);
    mask.set(a);
  }
  template <class KT>
  __device__ __forceinline__ void finish_init(const S1Ctx& X, const KT& K) {
    k = mask.count();
    tin = 0.0;
    win = -1;
    if (counts) {   // per-lane scan of the config's (node, count) list, once per task
      for (int i = 0; i < X.tl_len; ++i) {
        const uint32_t ac = X.tl_ac[i];
        if (get(ac & 0xffu) == (ac >> 8)) { win = (int)(ac & 0xffu); tin = X.tl_val[i]; break; }
      }
    }
    wab = 0xffffu;
    jw = kNoWit;
    maxR = 0.0;
    if (k >= 2) {
      if (direct) {
        maxR = pairs_max(mask, K, wab);
      } else {   // canonical witness: the first list pair inside N1 (per lane, once per task)
        for (int j = 0; j < X.gl_len; ++j) {
          const uint32_t p = pair_at(X, j);
          if (mask.test(p & 0xffu) && mask.test(p >> 8)) { jw = j; wab = p; maxR = K.r(p & 0xffu, p >> 8); break; }
        }
      }
    }
    tex = k >= 2 ? __dmul_rn(__ldg(X.qe + k), maxR) : 0.0;
    need_tin = need_scan = need_join = false;
    if (direct) {   // member bytes in ascending node order (k <= 8)
      unsigned long long l = 0ull;
      int t = 0;
#pragma unroll
      for (int wd = 0; wd < 4; ++wd)
        for (uint32_t bb = mask.word(wd); bb; bb &= bb - 1u, ++t)
          l |= (unsigned long long)(wd * 32 + __ffs(bb) - 1) << (8 * t);
      ml[lane] = (uint32_t)l;
      ml[32 + lane] = (uint32_t)(l >> 32);
    }
  }

  // a stage-1 member moves from node dn to node up (tentative); long searches are flagged
  template <class KT>
  __device__ __forceinline__ void propose(uint32_t dn, uint32_t up, const S1Ctx& X, const KT& K) {
    dn_ = dn; up_ = up;
    const uint32_t cd = counts ? get_of(dn, lane) : 1u, cu = counts ? get_of(up, lane) : 0u;
    c_dn_ = cd - 1u; c_up_ = cu + 1u;
    const bool leave = c_dn_ == 0u, join = c_up_ == 1u;
    mask2 = mask;
    if (leave) mask2.reset(dn);
    if (join) mask2.set(up);
    k2 = k - (int)leave + (int)join;
    // T_in: the witness node lost a member -> cooperative search; else the gaining node may
    // take over
    tin2 = tin; win2 = win;
    if (counts) {
      if ((int)dn == win) {
        need_tin = true;
      } else if (c_up_ >= 2u) {
        const double v = __dmul_rn(__ldg(X.qi + c_up_), K.r(up, up));
        if (v > tin2) { tin2 = v; win2 = (int)up; }
      }
    }
    // T_ex
    maxR2 = maxR; wab2 = wab; jw2 = jw;
    if (k2 < 2) { maxR2 = 0.0; wab2 = 0xffffu; jw2 = kNoWit; return; }
    const bool wit_left = leave && (dn == (wab & 0xffu) || dn == (wab >> 8));
    if (direct) {
      if (wit_left || k < 2) {
        need_scan = true;   // recompute over the member pairs, split over the warp (coop)
      } else if (join) {
        need_join = true;   // the new pairs (up, b), (b, up): one cooperative round
      }
    } else {
      bool found = false;
      if (join) {   // a pair of up ranked before the witness becomes the witness
        int j;
        uint32_t p;
        if (partner_scan(up, mask2, jw, X, j, p)) {
          jw2 = j; wab2 = p; maxR2 = K.r(p & 0xffu, p >> 8);
          found = true;
        }
      }
      // the witness pair left N1 (and up brought no earlier pair): every pair ranked before
      // it was outside N1, so the new witness is the first pair inside N1' after it
      if (!found && wit_left) need_scan = true;
    }
  }

  // warp-cooperative searches (called by all 32 lanes, converged).  JC: direct-mode joins
  // always through the warp (no per-lane join code in the kernel: large clusters)
  template <bool JC = false, class KT>
  __device__ __forceinline__ void coop(const S1Ctx& X, const KT& K) {
    const unsigned full = 0xffffffffu;
    if (!__any_sync(full, need_tin | need_scan | need_join)) return;   // (the common case: one vote)
    if (counts) {   // T_in: first (a, c) entry (by value) whose node has c members after the move
      unsigned todo = __ballot_sync(full, need_tin);
      while (todo) {
        const int L = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint32_t dnL = __shfl_sync(full, dn_, L), upL = __shfl_sync(full, up_, L);
        const uint32_t cdL = __shfl_sync(full, c_dn_, L), cuL = __shfl_sync(full, c_up_, L);
        int hit = -1;
        uint32_t acv = 0u;
        double v = 0.0;
        for (int base = 0; base < X.tl_len; base += 32) {
          const int i = base + lane;
          uint32_t ac = 0u;
          bool h = false;
          if (i < X.tl_len) {
            ac = X.tl_ac[i];
            const uint32_t a = ac & 0xffu;
            const uint32_t cnt = a == dnL ? cdL : (a == upL ? cuL : get_of(a, L));
            h = cnt == (ac >> 8);
          }
          const unsigned b = __ballot_sync(full, h);
          if (b) {
            const int f = __ffs(b) - 1;
            hit = base + f;
            acv = __shfl_sync(full, ac, f);
            break;
          }
        }
        if (hit >= 0) v = __dmul_rn(__ldg(X.qi + (acv >> 8)), K.r(acv & 0xffu, acv & 0xffu));
        if (lane == L) {
          need_tin = false;
          if (hit >= 0) { tin2 = v; win2 = (int)(acv & 0xffu); } else { tin2 = 0.0; win2 = -1; }
        }
      }
    }
    // T_ex, direct mode: many joins in one step go per lane (in parallel, each over the k'
    // members), a few through the warp (one round each, below)
    if (!JC && direct && __popc(__ballot_sync(full, need_join && !need_scan)) > join_coop_max(X.n)) {
      if (need_join && !need_scan) {
        uint32_t w;
        const double v = join_max(mask2, up_, K, w);
        if (v > maxR2) { maxR2 = v; wab2 = w; }
      }
      need_join = false;
    }
    // T_ex: the witness pair left N1 -- first pair inside N1' after the old witness's rank
    // (list mode), or the max over N1's member pairs split over the lanes (direct mode)
    unsigned todo = __ballot_sync(full, need_scan | need_join);
    while (todo) {
      const int L = __ffs(todo) - 1;
      todo &= todo - 1;
      if (direct) {
        // lane t (mod 8) holds member slot t of lane L's N1' = N1 - dn (+ up): slots 0..k-1
        // are N1's member bytes (dn's slot taken by up, or empty, when dn leaves), slot k is
        // up when it joins without a leave.  A join pairs up with every member (lanes 0-15,
        // one round); a recompute takes the ordered slot pairs (lane j of round r: slots
        // (4r + j / 8, j % 8)).
        const uint32_t info = __shfl_sync(full, dn_ | (up_ << 8) | ((uint32_t)k << 16) | ((c_dn_ == 0u) ? 1u << 20 : 0u) |
                                                    ((c_up_ == 1u) ? 1u << 21 : 0u) |
                                                    ((need_join && !need_scan) ? 1u << 22 : 0u), L);
        const uint32_t dnL = info & 0xffu, upL = (info >> 8) & 0xffu, kL = (info >> 16) & 0xfu;
        const bool lv = (info >> 20) & 1u, jn = (info >> 21) & 1u, jo = (info >> 22) & 1u;
        const uint32_t t = (uint32_t)lane & 7u;
        uint32_t memv = __byte_perm(t < 4u ? ml[L] : ml[32 + L], 0u, 0x4440u | (t & 3u));
        bool val = t < kL;
        if (val && lv && memv == dnL) { memv = upL; val = jn; }
        if (!lv && jn && t == kL) { memv = upL; val = true; }
        memv = val ? memv : 0xffffffffu;
        const uint32_t slots = kL + ((!lv && jn) ? 1u : 0u);
        double mx = 0.0;
        uint32_t wbest = 0xffffu;
        if (jo) {
          if (lane < 16 && memv != 0xffffffffu && memv != upL) {
            const uint32_t a = lane < 8 ? upL : memv, b = lane < 8 ? memv : upL;
            mx = K.r(a, b);
            wbest = a | (b << 8);
          }
        } else {
          for (uint32_t base = 0; base < slots * 8u; base += 32u) {
            const uint32_t ia = (base + (uint32_t)lane) >> 3;
            const uint32_t a = __shfl_sync(full, memv, (int)(ia & 7u)), b = __shfl_sync(full, memv, (int)t);
            if (ia != t && a != 0xffffffffu && b != 0xffffffffu) {
              const double v = K.r(a, b);
              if (v > mx) { mx = v; wbest = a | (b << 8); }
            }
          }
        }
        uint32_t cnt;   // max-reduce; the witness of the lowest lane holding it (any equal max is fine)
        const double gmx = warp_max_nonneg(mx, 1u, cnt);
        const unsigned holders = __ballot_sync(full, mx == gmx);
        wbest = __shfl_sync(full, wbest, __ffs(holders) - 1);
        if (lane == L) {
          if (!jo || gmx > maxR2) { maxR2 = gmx; wab2 = wbest; }
          need_scan = need_join = false;
        }
        continue;
      }
      Mask4 m;
      m.w0 = __shfl_sync(full, mask2.w0, L); m.w1 = __shfl_sync(full, mask2.w1, L);
      m.w2 = __shfl_sync(full, mask2.w2, L); m.w3 = __shfl_sync(full, mask2.w3, L);
      const int start = __shfl_sync(full, jw, L) + 1;
      int hit = -1;
      uint32_t pab = 0u;
      for (int base = start; base < X.gl_len; base += 32) {
        const int j = base + lane;
        uint32_t p = 0u;
        bool h = false;
        if (j < X.gl_len) {
          p = pair_at(X, j);
          h = m.test(p & 0xffu) & m.test(p >> 8);   // (both tests, no branch: 747 vs 750.5 ms on C5)
        }
        const unsigned b = __ballot_sync(full, h);
        if (b) {
          const int f = __ffs(b) - 1;
          hit = base + f;
          pab = __shfl_sync(full, p, f);
          break;
        }
      }
      if (lane == L) {
        need_scan = false;
        if (hit >= 0) { jw2 = hit; wab2 = pab; maxR2 = K.r(pab & 0xffu, pab >> 8); }
        else { jw2 = kNoWit; wab2 = 0xffffu; maxR2 = 0.0; }   // (unreachable: |N1'| >= 2)
      }
    }
  }
  __device__ __forceinline__ void finish(const S1Ctx& X) { tex2 = k2 >= 2 ? __dmul_rn(__ldg(X.qe + k2), maxR2) : 0.0; }
  __device__ __forceinline__ void commit() {
    if (counts) { add(dn_, -1); add(up_, +1); }
    if (direct && (c_dn_ == 0u || c_up_ == 1u)) {   // member bytes: dn's byte <- the last one; up appended
      unsigned long long l = (unsigned long long)ml[lane] | ((unsigned long long)ml[32 + lane] << 32);
      int kk = k;
      if (c_dn_ == 0u) {
        const uint32_t d4 = dn_ * 0x01010101u;
        unsigned long long e = (unsigned long long)__vcmpeq4(ml[lane], d4) |
                               ((unsigned long long)__vcmpeq4(ml[32 + lane], d4) << 32);
        e &= kk >= 8 ? ~0ull : (1ull << (8 * kk)) - 1ull;
        const int pos = (__ffsll((long long)e) - 1) >> 3;
        const unsigned long long last = (l >> (8 * (kk - 1))) & 0xffull;
        l = (l & ~(0xffull << (8 * pos))) | (last << (8 * pos));
        l &= ~(0xffull << (8 * (kk - 1)));
        --kk;
      }
      if (c_up_ == 1u) l |= (unsigned long long)up_ << (8 * kk);
      ml[lane] = (uint32_t)l;
      ml[32 + lane] = (uint32_t)(l >> 32);
    }
    mask = mask2; k = k2; tin = tin2; win = win2; tex = tex2; maxR = maxR2; wab = wab2; jw = jw2;
  }
};

// ------------------------------------------------------------------ one warp task of MODE 1
// Same step structure as run_task_hc: the swap is applied tentatively, the touched
// pipelines are re-summed in stage order, T_PP keeps the count of pipelines at its max.
template <bool TRACE, int PP, bool ID, bool JC>
__device__ __forceinline__ void run_task_sb(const SaParams& P, const SaTask T, const DevCfg C, const double* Rt,
                                            const uint16_t* pl, unsigned char* ws, int lane) {
  const bool active = lane < T.count;
  const int N = C.N, pp = PP > 0 ? PP : C.pp, dp = C.dp, n = P.n_nodes;
  const uint32_t flags = (uint32_t)T.pad;
  const uint32_t chain = (uint32_t)(T.c_first + (T.k0 + lane) * P.world);
  const int slot = T.slot0 + lane;
  S1Ctx X;
  X.qi = P.qtab + C.qi_off; X.qe = P.qtab + C.qe_off;
  X.gl_ab = P.gl_ab; X.gl_len = n * (n - 1);
  X.tl_ac = P.tl_ac + (size_t)T.f * P.tl_stride;
  X.tl_val = P.tl_val + (size_t)T.f * P.tl_stride;
  X.tl_len = P.tl_len[T.f];
  X.nl_len = 2 * (n - 1);
  X.n = n;
  X.pt = P.pt; X.pt_stride = P.pt_stride; X.pl = pl; X.plen = P.plen;
  SbCtxT<ID> K;
  K.T = Rt; K.m2 = C.m2; K.lg = (uint32_t)P.r_lg; K.n = n;
  K.spn = (uint32_t)C.spn; K.spn_magic = C.spn_magic;
  K.spn_sh = (C.spn & (C.spn - 1)) == 0 ? (uint32_t)(31 - __clz(C.spn)) : 32u;
  K.m16 = (uint32_t)((65536u + (uint32_t)C.spn - 1u) / (uint32_t)C.spn);
  K.sh = (uint32_t)(31 - __clz(C.spn));   // (P2: spn is a power of two)
  K.bmask = (0xffu >> K.sh) * 0x01010101u;
  K.rowmul = 8u << K.lg;
  K.tbase = (uint32_t)__cvta_generic_to_shared(Rt);

  const bool cache = (flags & kTfCache) != 0;
  const int plane = align16(((N + 3) / 4) * 128);
  HcState st;
  st.hb = ws + lane * 4;   // slot bytes (st.hb doubles as the slot plane)
  st.sb = st.hb;
  st.hw = reinterpret_cast<const uint32_t*>(ws) + lane;
  S1M s1;
  s1.counts = (flags & kTfCounts) != 0;
  s1.direct = (flags & kTfDirect) != 0;
  s1.lane = lane;
  s1.c = reinterpret_cast<uint32_t*>(ws + plane);
  s1.set_nibbles(P.s1_nib != 0);
  double* psum = reinterpret_cast<double*>(ws + plane + (s1.counts ? sb_count_bytes(n, P.s1_nib != 0) : 0));
  s1.ml = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(psum) + (cache ? align16(dp * 256) : 0));
  uint16_t* bperm = P.best_perm + T.perm_off;
  s1.clear(n);

  for (int w = 0; w < N; ++w) {
    st.hb[HcState::off((uint32_t)w)] = (uint8_t)w;
    bperm[w * 32 + lane] = (uint16_t)w;
  }
  __syncwarp();
  double tpp = 0.0;
  int nmax = 0;
  for (int z = 0; z < dp; ++z) {
    s1.add_init(K.node((uint32_t)(z * pp)));
    if (pp >= 2) {
      const double s = sb_sum<PP, SbCtxT<ID>>(st, (uint32_t)z, pp, K);
      if (cache) psum[z * 32 + lane] = s;
      if (s > tpp) { tpp = s; nmax = 1; } else if (s == tpp) { ++nmax; }
    }
  }
  s1.finish_init(X, K);

  const double L0 = compose(C.Sb, C.r, C.Ss, tpp, s1.tin, s1.tex);
  // the best point's breakdown and step go straight to the chain's output record (rarely
  // written; kept out of the registers of the step loop)
  ChainOut* const out = P.out + slot;
  if (active) { out->best_tpp = tpp; out->best_tdp = __dadd_rn(s1.tin, s1.tex); out->best_step = -1; out->L0 = L0; }
  double cur = L0, best = L0;
  uint32_t accepted = 0;
  double beta = sa_beta0(P, T.f, L0);
  const int trow = (TRACE && active) ? P.trace_slot[slot] : -1;

  if (N >= 2) {
    Draw dnext = draw_swap_rk(0u, chain, (uint32_t)C.e, P.rk, (uint32_t)N);
    for (int i = 0; i < P.iterations; ++i) {
      const Draw d = dnext;
      dnext = draw_swap_rk((uint32_t)(i + 1), chain, (uint32_t)C.e, P.rk, (uint32_t)N);
      const uint32_t p = d.p, q = d.q;
      uint8_t* const bp = st.hb + HcState::off(p);
      uint8_t* const bq = st.hb + HcState::off(q);
      const uint32_t sp = *bp, sq = *bq;
      bool dpchg = false;
      const uint32_t np = K.node(sp), nq = K.node(sq);
      double Lp = cur;
      bool acc = true, improved = false;
      if (pp >= 2) {
        const uint32_t zp = PP > 0 ? p / (uint32_t)PP : div_small(p, C.pp_magic, (uint32_t)pp);
        const uint32_t zq = PP > 0 ? q / (uint32_t)PP : div_small(q, C.pp_magic, (uint32_t)pp);
        const uint32_t xp = p - zp * (uint32_t)pp, xq = q - zq * (uint32_t)pp;
        const bool two = zq != zp;
        const uint32_t zb = two ? zq : zp;
        double oldA, oldB;
        if (cache) {
          oldA = psum[zp * 32 + lane];
          oldB = psum[zb * 32 + lane];
        } else {
          sb_sum2<PP, SbCtxT<ID>>(st, zp, zb, pp, K, oldA, oldB);
        }
        *bp = (uint8_t)sq;   // tentative swap
        *bq = (uint8_t)sp;
        double sA, sB;
        sb_sum2<PP, SbCtxT<ID>>(st, zp, zb, pp, K, sA, sB);
        double tpp2 = tpp;
        int nmax2 = nmax;
        const double snew = dmax(sA, sB);
        const int keep = nmax - (oldA == tpp ? 1 : 0) - ((two && oldB == tpp) ? 1 : 0);
        const bool fast = keep > 0 || snew >= tpp;
        if (fast) {
          tpp2 = (keep > 0) ? dmax(tpp, snew) : snew;
          nmax2 = (keep > 0 && tpp2 == tpp ? keep : 0) + (sA == tpp2 ? 1 : 0) + ((two && sB == tpp2) ? 1 : 0);
        }
        // the unique max pipeline decreased: rescan over all pipelines -- up to 4 cached sums
        // per lane, else warp-cooperatively (measured per configuration: a dp = 16 per-lane
        // rescan ran at 3 active lanes and cost 400 warp instructions per step)
        if (!fast && cache) {   // the new sums enter the cache tentatively (restored if rejected)
          psum[zp * 32 + lane] = sA;
          psum[zb * 32 + lane] = sB;
        }
        if (cache && dp <= 8) {
          if (!fast) {   // (unrolled: independent loads and a max tree, then the tie count)
            double v[8];
#pragma unroll
            for (int z = 0; z < 8; ++z) v[z] = z < dp ? psum[z * 32 + lane] : 0.0;
            const double m = dmax(dmax(dmax(v[0], v[1]), dmax(v[2], v[3])), dmax(dmax(v[4], v[5]), dmax(v[6], v[7])));
            int c = 0;
#pragma unroll
            for (int z = 0; z < 8; ++z) c += (z < dp && v[z] == m) ? 1 : 0;
            tpp2 = m;
            nmax2 = c;
          }
        } else {
          coop_tpp<PP, SbCtxT<ID>>(!fast, ws, psum, cache, dp, pp, zp, zb, sA, sB, K, lane, tpp2, nmax2);
        }
        dpchg = ((xp == 0u) != (xq == 0u)) && np != nq;
        if (dpchg) {
          const uint32_t dn = xp == 0u ? np : nq;
          const uint32_t up = xp == 0u ? nq : np;
          s1.propose(dn, up, X, K);
        }
        s1.coop<JC>(X, K);   // converged: all lanes' flagged searches
        double tin2 = s1.tin, tex2 = s1.tex;
        if (dpchg) {
          s1.finish(X);
          tin2 = s1.tin2;
          tex2 = s1.tex2;
        }
        Lp = compose(C.Sb, C.r, C.Ss, tpp2, tin2, tex2);
        acc = metropolis_fast(__dadd_rn(Lp, -cur), beta, d.u);
        if (acc) {
          if (cache) {
            psum[zp * 32 + lane] = sA;
            psum[zb * 32 + lane] = sB;
          }
          tpp = tpp2;
          nmax = nmax2;
          if (dpchg) s1.commit();
          cur = Lp;
          if (Lp < best) {
            best = Lp;
            if (active) { out->best_tpp = tpp; out->best_tdp = __dadd_rn(s1.tin, s1.tex); out->best_step = i; }
            improved = true;
          }
        } else {
          if (!fast && cache) {   // restore the cached sums of the rejected proposal
            psum[zb * 32 + lane] = oldB;
            psum[zp * 32 + lane] = oldA;
          }
          *bq = (uint8_t)sq;   // revert
          *bp = (uint8_t)sp;
        }
      } else {
        *bp = (uint8_t)sq;   // pp = 1: L' = cur (no hops, stage-1 multiset unchanged)
        *bq = (uint8_t)sp;
      }
      if (acc) ++accepted;
      for (uint32_t imp = __ballot_sync(0xffffffffu, improved); imp; imp &= imp - 1u) {   // (as in MODE 0)
        const int L = __ffs(imp) - 1;
        const uint8_t* sbL = ws + L * 4;
        for (int w = lane; w < N; w += 32) bperm[w * 32 + L] = (uint16_t)sbL[HcState::off((uint32_t)w)];
      }
      if (TRACE && trow >= 0 && i < P.trace_cap) {
        pipette_trace_record rec;
        rec.i = (uint32_t)i; rec.p = (uint16_t)d.p; rec.q = (uint16_t)d.q;
        rec.accept = acc ? 1u : 0u; rec.latency = Lp;
        P.trace[(size_t)trow * P.trace_cap + i] = rec;
      }
      beta = __dmul_rn(beta, P.alpha_inv);
    }
  }
  if (active) { out->best = best; out->accepted = accepted; out->f = T.f; out->c = (int32_t)chain; }
}

// Compile-time pipeline depth for the common power-of-two depths (the Eq.5 sums unroll).
// ID: the context's node map (true: power-of-two spn, the only variant the swap kernel
// instantiates -- two variants in one kernel made ptxas spill in the hot loop).
template <bool TRACE, bool ID, bool JC>
__device__ __forceinline__ void run_task_sb_pp(const SaParams& P, const SaTask T, const DevCfg C, const double* Rt,
                                               const uint16_t* pl, unsigned char* ws, int lane) {
  switch (C.pp) {
    case 1: run_task_sb<TRACE, 1, ID, JC>(P, T, C, Rt, pl, ws, lane); break;
    case 2: run_task_sb<TRACE, 2, ID, JC>(P, T, C, Rt, pl, ws, lane); break;
    case 4: run_task_sb<TRACE, 4, ID, JC>(P, T, C, Rt, pl, ws, lane); break;
    case 8: run_task_sb<TRACE, 8, ID, JC>(P, T, C, Rt, pl, ws, lane); break;
    case 16: run_task_sb<TRACE, 16, ID, JC>(P, T, C, Rt, pl, ws, lane); break;
    case 32: run_task_sb<TRACE, 32, ID, JC>(P, T, C, Rt, pl, ws, lane); break;
    default: run_task_sb<TRACE, 0, ID, JC>(P, T, C, Rt, pl, ws, lane); break;
  }
}
