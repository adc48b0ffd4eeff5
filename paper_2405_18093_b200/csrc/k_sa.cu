// k_sa.cu -- K3: simulated-annealing chains of fine-grained worker dedication and
// K4: per-configuration argmin.
//
// Alg.1 l.9-15 with the SA of P:250-255: each proposal swaps two positions
// of the mapping string (Eq.2), re-evaluates Eq.3-6 and is
// accepted by Metropolis (R13) with Philox randomness (R14).
//
// Design: one chain per LANE; a warp runs 32 chains of one
// configuration, so every instruction advances 32 independent Markov chains.  Chain
// state lives in shared memory in lane-interleaved layouts ([element / 4][lane] words), so
// every per-lane access is bank-conflict free:
//   MODE 0 (n <= 16, N <= 256)   hop codes node(w-1) | node(w) << 4 and slot ids, one
//                                byte per position; the block's 16-copy m2*R table;
//                                stage-1 state in registers (S1Reg), subset-max T_ex
//   MODE 1 (n <= 128, N <= 256)  slot ids, one byte per position; the block's n x n m2*R
//                                table; member counts in shared memory with sorted-table
//                                witnesses and warp-cooperative searches (S1Large)
//   MODE 2 (general)             32-bit positions, R through L1 (PosWide, S1Large)
//   psum[z]                      Eq.5 sum of pipeline z (cached when pp >= 4, dp small)
// Re-evaluation is incremental but bit-exact: the (at most two) touched pipelines are
// re-summed from scratch in stage order, the max terms (T_PP, T_in, T_ex) are kept with
// counts, witnesses or tables and rescanned when a witness could drop.  max is exact, so
// every latency equals the from-scratch definition of the oracle bit for bit.
#include <type_traits>

#include "devmath.cuh"
#include "pipette_dev.cuh"

namespace pip {


__host__ __device__ __forceinline__ int align16(int x) { return (x + 15) & ~15; }

// R = 1/B through the read-only path (MODE 1 searches, MODE 2 hops).
struct RGlob {
  const double* s;
  int n, lane;
  __device__ __forceinline__ double operator()(uint32_t a, uint32_t b) const { return __ldg(s + (int)a * n + (int)b); }
};

// ------------------------------------------------------------------ position storage
struct PosWide {
  uint32_t* s;
  int lane;
  static __host__ __device__ int bytes(int N) { return N * 128; }
  __device__ __forceinline__ uint32_t raw(uint32_t w) const { return s[w * 32 + lane]; }
  __device__ __forceinline__ uint32_t node(uint32_t w) const { return raw(w) >> 16; }
  static __device__ __forceinline__ uint32_t node_of(uint32_t r) { return r >> 16; }
  static __device__ __forceinline__ uint32_t slot_of(uint32_t r) { return r & 0xffffu; }
  __device__ __forceinline__ void init(int N, uint32_t spn, uint32_t spn_magic) {
    for (int w = 0; w < N; ++w) s[w * 32 + lane] = (uint32_t)w | (div_small((uint32_t)w, spn_magic, spn) << 16);
  }
  __device__ __forceinline__ void swap(uint32_t p, uint32_t q, uint32_t rp, uint32_t rq) {
    s[p * 32 + lane] = rq;
    s[q * 32 + lane] = rp;
  }
};

constexpr uint32_t kNone = 0xffffffffu;

// Node of position w with positions p and q reading as nodes nq and np instead (kNone: no
// substitution -- the compiler then drops the compares).
template <class POS>
__device__ __forceinline__ uint32_t node_at(const POS& pos, uint32_t w, uint32_t p, uint32_t q, uint32_t np,
                                            uint32_t nq) {
  const uint32_t v = pos.node(w);
  if (p == kNone) return v;
  return w == p ? nq : (w == q ? np : v);
}

// Eq.5 sum of pipeline z in stage order (P_z = ((0 + m2 R[..]) + m2 R[..]) + ..., DESIGN.md
// 3).  PP > 0: compile-time pipeline depth (fully unrolled, loads hoisted); PP == 0: runtime.
template <class RT, int PP, class POS>
__device__ __forceinline__ double pipe_sum(int z, int pp_rt, const POS& pos, uint32_t p, uint32_t q, uint32_t np,
                                           uint32_t nq, double m2, const RT& R) {
  const int pp = PP > 0 ? PP : pp_rt;
  const uint32_t base = (uint32_t)(z * pp);
  uint32_t prev = node_at(pos, base, p, q, np, nq);
  double s = 0.0;
#pragma unroll (PP > 0 ? 32 : 4)
  for (int x = 1; x < (PP > 0 ? PP : pp); ++x) {
    const uint32_t nd = node_at(pos, base + x, p, q, np, nq);
    s = __dadd_rn(s, __dmul_rn(m2, R(prev, nd)));
    prev = nd;
  }
  return s;
}

// Two pipelines re-summed in one interleaved loop (two independent dependency chains).
template <class RT, int PP, class POS>
__device__ __forceinline__ void pipe_sum2(int za, int zb, int pp_rt, const POS& pos, uint32_t p, uint32_t q,
                                          uint32_t np, uint32_t nq, double m2, const RT& R, double& sa,
                                          double& sb) {
  const int pp = PP > 0 ? PP : pp_rt;
  const uint32_t ba = (uint32_t)(za * pp), bb = (uint32_t)(zb * pp);
  uint32_t pa = node_at(pos, ba, p, q, np, nq);
  uint32_t pb = node_at(pos, bb, p, q, np, nq);
  double a = 0.0, b = 0.0;
#pragma unroll (PP > 0 ? 32 : 4)
  for (int x = 1; x < (PP > 0 ? PP : pp); ++x) {
    const uint32_t na = node_at(pos, ba + x, p, q, np, nq);
    const uint32_t nb = node_at(pos, bb + x, p, q, np, nq);
    a = __dadd_rn(a, __dmul_rn(m2, R(pa, na)));
    b = __dadd_rn(b, __dmul_rn(m2, R(pb, nb)));
    pa = na;
    pb = nb;
  }
  sa = a;
  sb = b;
}

// ------------------------------------------------------------------ stage-1 (Eq.6) state
struct S1Ctx {
  const double* qi;      // qi(c), c = 0..dp
  const double* qe;      // qe(k), k = 0..min(dp, n)
  const double* tab;     // subset-max table (S1Reg only)
  const uint8_t* rank;   // [a*16 + c] rank of qi(c)*R[a][a], 255 if c < 2 (S1Reg only)
  const double* vs;      // values in rank order (S1Reg only)
  // S1Large tables
  const uint8_t* nl_node;   // [a][nl_len] other endpoints of pairs with a, by R descending
  const double* nl_val;     // their R values (both directions)
  const uint16_t* gl_ab;    // all ordered pairs (a | b << 8) by R descending
  const double* gl_val;
  const uint16_t* tl_ac;    // this config's (a | c << 8), c >= 2, by qi(c) R[a][a] descending
  const double* tl_val;
  int nl_len, gl_len, tl_len;
  int n;
  // MODE 1 (S1M): per node, its 2(n-1) ordered pairs in global-list order (entry = list
  // index | other node << 16 | node first << 24, rows of pt_stride entries padded with
  // 0xffffffff; k_partner_lists), and the
  // block's shared copy of the first plen entries of gl_ab
  const uint32_t* pt;
  int pt_stride;
  const uint16_t* pl;
  int plen;
};

// n <= 16 nodes and <= 15 stage-1 members per node.  T_in by ranks: for this config every
// value qi(c)*R[a][a] (c >= 2) has a precomputed position in descending order
// (k_tin_rank); a node's current rank is one byte of rk[], and T_in is the value at the
// smallest rank present (SIMD byte minimum) -- the max of Eq.6's intra term without a scan.
template <class RT, int NW = 4>
struct S1Reg {
  // NW = 4: n <= 16 nodes, counts in a 64-bit register, rank bytes in four words;
  // NW = 2: n <= 8 nodes, counts in a 32-bit register, rank bytes in two words
  using CT = typename std::conditional<NW == 2, uint32_t, uint64_t>::type;
  CT cnt, cnt2;
  uint32_t mask, mask2;
  uint32_t rk0, rk1, rk2_, rk3, nk0, nk1, nk2, nk3;   // current / tentative rank bytes
  uint32_t pend;   // NW = 4: the tentative move instead, dn | up << 8 | dn's new rank << 16 | up's << 24
  int k, k2;
  double tin, tex, tin2, tex2;

  static __device__ __forceinline__ uint32_t get(CT c, uint32_t a) { return (uint32_t)(c >> (4u * a)) & 15u; }
  // byte a of the rank vector (r0..r3) := v (scalars, never an indexed array)
  static __device__ __forceinline__ void set_byte(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t a,
                                                  uint32_t v) {
    const uint32_t sh = (a & 3u) * 8u, q = a >> 2;
    const uint32_t keep = ~(0xffu << sh), put = v << sh;
    r0 = q == 0u ? ((r0 & keep) | put) : r0;
    r1 = q == 1u ? ((r1 & keep) | put) : r1;
    if constexpr (NW == 4) {
      r2 = q == 2u ? ((r2 & keep) | put) : r2;
      r3 = q == 3u ? ((r3 & keep) | put) : r3;
    }
  }
  static __device__ __forceinline__ double tin_of(uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3, const S1Ctx& X) {
    uint32_t m = NW == 4 ? __vminu4(__vminu4(r0, r1), __vminu4(r2, r3)) : __vminu4(r0, r1);
    m = __vminu4(m, m >> 16);
    m = __vminu4(m, m >> 8) & 0xffu;
    return m == 0xffu ? 0.0 : X.vs[m];
  }
  // NW = 2: X.tab is the block's table of the whole term, tab[m] = fl(qe(|m|) * maxR(m))
  // (0 for |m| < 2), so T_ex is one load
  __device__ __forceinline__ double tex_of(uint32_t m, int kk, const S1Ctx& X) const {
    if constexpr (NW == 2) return X.tab[m];
    return kk >= 2 ? __dmul_rn(X.qe[kk], X.tab[m]) : 0.0;
  }
  __device__ __forceinline__ void clear() { cnt = 0; mask = 0u; }
  __device__ __forceinline__ void add_init(uint32_t a) { cnt += (CT)1 << (4u * a); mask |= 1u << a; }
  __device__ __forceinline__ void finish_init(const S1Ctx& X, const RT& R) {
    rk0 = rk1 = rk2_ = rk3 = 0xffffffffu;
    for (int a = 0; a < X.n; ++a) set_byte(rk0, rk1, rk2_, rk3, (uint32_t)a, X.rank[a * 16 + get(cnt, (uint32_t)a)]);
    k = __popc(mask);
    tin = tin_of(rk0, rk1, rk2_, rk3, X);
    tex = tex_of(mask, k, X);
  }
  // a stage-1 member moves from node dn to node up (tentative state)
  // NW = 4 keeps only the move and the two new ranks live until commit (C3 145.7 -> 121.3 ms:
  // the 16-node state spilled); NW = 2 keeps the whole tentative state (C2 14.9 vs 17.2 ms)
  __device__ __forceinline__ void propose(uint32_t dn, uint32_t up, const S1Ctx& X, const RT& R) {
    const uint32_t c_dn = get(cnt, dn) - 1u, c_up = get(cnt, up) + 1u;
    const uint32_t m2 = (mask & (c_dn == 0u ? ~(1u << dn) : 0xffffffffu)) | (1u << up);
    const uint32_t r_dn = X.rank[dn * 16 + c_dn], r_up = X.rank[up * 16 + c_up];
    uint32_t t0 = rk0, t1 = rk1, t2 = rk2_, t3 = rk3;
    set_byte(t0, t1, t2, t3, dn, r_dn);
    set_byte(t0, t1, t2, t3, up, r_up);
    tin2 = tin_of(t0, t1, t2, t3, X);
    tex2 = (m2 == mask) ? tex : tex_of(m2, __popc(m2), X);
    if constexpr (NW == 4) {
      pend = dn | (up << 8) | (r_dn << 16) | (r_up << 24);
    } else {
      cnt2 = cnt - ((CT)1 << (4u * dn)) + ((CT)1 << (4u * up));
      mask2 = m2; k2 = __popc(m2);
      nk0 = t0; nk1 = t1; nk2 = t2; nk3 = t3;
    }
  }
  __device__ __forceinline__ void coop(const S1Ctx&, const RT&) {}
  __device__ __forceinline__ void finish(const S1Ctx&) {}
  __device__ __forceinline__ void commit() {
    if constexpr (NW == 4) {
      const uint32_t dn = pend & 0xffu, up = (pend >> 8) & 0xffu;
      mask = (mask & (get(cnt, dn) == 1u ? ~(1u << dn) : 0xffffffffu)) | (1u << up);
      cnt = cnt - ((CT)1 << (4u * dn)) + ((CT)1 << (4u * up));
      k = __popc(mask);
      set_byte(rk0, rk1, rk2_, rk3, dn, (pend >> 16) & 0xffu);
      set_byte(rk0, rk1, rk2_, rk3, up, pend >> 24);
    } else {
      cnt = cnt2; mask = mask2; k = k2;
      rk0 = nk0; rk1 = nk1; rk2_ = nk2; rk3 = nk3;
    }
    tin = tin2; tex = tex2;
  }
};

// General stage-1 state (n <= 128): counts (u8, c_n <= spn <= 255) in shared memory, a
// 128-bit node mask N1 in registers, witnesses for both max terms of Eq.6 and sorted
// tables instead of scans:
//   T_in: witness node; when it loses a member, the config's (a, c) list sorted by
//         qi(c) R[a][a] is searched for the first entry whose node has exactly c members.
//   T_ex: witness pair {wa, wb}; a node joining N1 searches its own pair list (sorted by R)
//         for the first partner in N1 (expected n/k probes); the witness leaving
//         recomputes the max over member pairs (small k) or searches the global sorted
//         pair list for the first pair inside N1 (expected (n/k)^2 probes).
// The three searches are rare per chain but long, so they are done warp-cooperatively:
// propose() only flags them; coop() (all 32 lanes converged) serves each flagged lane
// with the whole warp probing 32 entries per round (ballot picks the first hit), or
// splitting the member rows over the lanes (shuffle max-reduction).
template <class RT>
struct S1Large {
  uint32_t* c;   // [ceil(n/4)][32] words of byte counts, or [ceil(n/8)][32] of nibbles
  int lane;
  uint32_t lgw = 2u, bw = 8u, cm = 0xffu;   // log2 counts per word, bits per count, count mask
  __device__ __forceinline__ void set_nibbles(bool nib) {   // (nibbles: every count <= 15)
    lgw = nib ? 3u : 2u; bw = nib ? 4u : 8u; cm = nib ? 0xfu : 0xffu;
  }
  Mask4 mask, mask2;
  int k, k2, win, win2, wa, wb, wa2, wb2;
  uint32_t dn_, up_, c_dn_, c_up_;
  bool need_tin, need_maxr, need_join;
  double tin, tex, maxR, tin2, tex2, maxR2;

  __device__ __forceinline__ uint32_t get(uint32_t a) const { return get_of(a, lane); }
  __device__ __forceinline__ uint32_t get_of(uint32_t a, int L) const {
    return (c[(a >> lgw) * 32 + L] >> ((a & ((1u << lgw) - 1u)) * bw)) & cm;
  }
  __device__ __forceinline__ void add(uint32_t a, int delta) {
    uint32_t& w = c[(a >> lgw) * 32 + lane];
    const uint32_t sh = (a & ((1u << lgw) - 1u)) * bw;
    w = delta > 0 ? w + (1u << sh) : w - (1u << sh);
  }
  static __device__ __forceinline__ bool in(const Mask4& m, uint32_t a) { return m.test(a); }

  // ---- per-lane versions (initial state only)
  __device__ __forceinline__ double tin_scan_own(const S1Ctx& X, int& w) const {
    for (int i = 0; i < X.tl_len; ++i) {
      const uint32_t ac = X.tl_ac[i];
      if (get(ac & 0xffu) == (ac >> 8)) { w = (int)(ac & 0xffu); return X.tl_val[i]; }
    }
    w = -1;
    return 0.0;
  }
  __device__ __forceinline__ double maxr_global_own(const Mask4& m, const S1Ctx& X, int& a_, int& b_) const {
    for (int i = 0; i < X.gl_len; ++i) {
      const uint32_t ab = X.gl_ab[i];
      if (in(m, ab & 0xffu) && in(m, ab >> 8)) { a_ = (int)(ab & 0xffu); b_ = (int)(ab >> 8); return X.gl_val[i]; }
    }
    a_ = b_ = -1;
    return 0.0;
  }

  __device__ __forceinline__ void clear(int n) {
    for (int wd = 0; wd < ((n - 1) >> lgw) + 1; ++wd) c[wd * 32 + lane] = 0u;
    mask.clear();
  }
  __device__ __forceinline__ void add_init(uint32_t a) { add(a, +1); mask.set(a); }
  __device__ __forceinline__ void finish_init(const S1Ctx& X, const RT& R) {
    k = mask.count();
    tin = tin_scan_own(X, win);
    maxR = k >= 2 ? maxr_global_own(mask, X, wa, wb) : 0.0;
    if (k < 2) wa = wb = -1;
    tex = k >= 2 ? __dmul_rn(__ldg(X.qe + k), maxR) : 0.0;
    need_tin = need_maxr = need_join = false;
  }
  // a stage-1 member moves from node dn to node up (tentative); long searches are flagged
  __device__ __forceinline__ void propose(uint32_t dn, uint32_t up, const S1Ctx& X, const RT& R) {
    dn_ = dn; up_ = up;
    c_dn_ = get(dn) - 1u; c_up_ = get(up) + 1u;
    const bool leave = c_dn_ == 0u, join = c_up_ == 1u;
    mask2 = mask;
    if (leave) mask2.reset(dn);
    if (join) mask2.set(up);
    k2 = k - (int)leave + (int)join;
    tin2 = tin; win2 = win;
    if ((int)dn == win) {
      need_tin = true;
    } else if (c_up_ >= 2u) {
      const double v = __dmul_rn(__ldg(X.qi + c_up_), R(up, up));
      if (v > tin2) { tin2 = v; win2 = (int)up; }
    }
    maxR2 = maxR; wa2 = wa; wb2 = wb;
    if (k2 < 2) {
      maxR2 = 0.0; wa2 = wb2 = -1;
    } else if (leave && ((int)dn == wa || (int)dn == wb)) {
      need_maxr = true;
    } else if (join) {
      need_join = true;
    }
  }

  // ---- warp-cooperative searches (called by all 32 lanes, converged)
  // first index >= 0 in [0, len) with hit(i); the warp probes 32 entries per round
  template <class F>
  static __device__ __forceinline__ int coop_first(int len, F hit) {
    const int ln = threadIdx.x & 31;
    for (int base = 0; base < len; base += 32) {
      const int i = base + ln;
      const unsigned b = __ballot_sync(0xffffffffu, i < len && hit(i));
      if (b) return base + __ffs(b) - 1;
    }
    return -1;
  }
  // PAIRS: the witness recompute for small k splits the member PAIRS over the lanes (the
  // BIG kernel, where R comes from L2 and a serial per-lane scan is latency-bound);
  // otherwise the member ROWS are split (fewer registers: the small-table kernel spills)
  // The same, also returning the hit entry's value and key: every probe loads its value
  // beside its key, and the hit lane's pair is shuffled out (no dependent round trip to L2
  // after the search).  hit(i, key) sets the key it read.
  template <class F, class G>
  static __device__ __forceinline__ int coop_first_v(int len, F hit, G val, double& v_out, uint32_t& key_out) {
    const int ln = threadIdx.x & 31;
    for (int base = 0; base < len; base += 32) {
      const int i = base + ln;
      const bool ok = i < len;
      const double v = ok ? val(i) : 0.0;
      uint32_t key = 0u;
      const unsigned b = __ballot_sync(0xffffffffu, ok && hit(i, key));
      if (b) {
        const int f = __ffs(b) - 1;
        v_out = __shfl_sync(0xffffffffu, v, f);
        key_out = __shfl_sync(0xffffffffu, key, f);
        return base + f;
      }
    }
    v_out = 0.0;
    key_out = 0u;
    return -1;
  }
  template <bool PAIRS = false>
  __device__ __forceinline__ void coop(const S1Ctx& X, const RT& R) {
    const unsigned full = 0xffffffffu;
    // T_in: first (a, c) entry (by value) whose node has c members after the move
    unsigned todo = __ballot_sync(full, need_tin);
    while (todo) {
      const int L = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t dnL = __shfl_sync(full, dn_, L), upL = __shfl_sync(full, up_, L);
      const uint32_t cdL = __shfl_sync(full, c_dn_, L), cuL = __shfl_sync(full, c_up_, L);
      double v;
      uint32_t acv;
      const int i = coop_first_v(X.tl_len, [&](int j, uint32_t& ac) {
        ac = X.tl_ac[j];
        const uint32_t a = ac & 0xffu;
        const uint32_t cnt = a == dnL ? cdL : (a == upL ? cuL : get_of(a, L));
        return cnt == (ac >> 8);
      }, [&](int j) { return X.tl_val[j]; }, v, acv);
      if (lane == L) {
        need_tin = false;
        if (i >= 0) { tin2 = v; win2 = (int)(acv & 0xffu); } else { tin2 = 0.0; win2 = -1; }
      }
    }
    // T_ex, join: first partner (by R) of the joining node inside N1
    todo = __ballot_sync(full, need_join);
    while (todo) {
      const int L = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t upL = __shfl_sync(full, up_, L);
      Mask4 m;
      m.w0 = __shfl_sync(full, mask2.w0, L); m.w1 = __shfl_sync(full, mask2.w1, L);
      m.w2 = __shfl_sync(full, mask2.w2, L); m.w3 = __shfl_sync(full, mask2.w3, L);
      const uint8_t* nl = X.nl_node + (size_t)upL * X.nl_len;
      const double* nv = X.nl_val + (size_t)upL * X.nl_len;
      double v;
      uint32_t bn;
      const int i = coop_first_v(X.nl_len, [&](int j, uint32_t& b) { b = nl[j]; return in(m, b); },
                                 [&](int j) { return nv[j]; }, v, bn);
      if (lane == L) {
        need_join = false;
        if (i >= 0 && v > maxR2) { maxR2 = v; wa2 = (int)upL; wb2 = (int)bn; }
      }
    }
    // T_ex, the witness left: recompute the slowest link of N1
    todo = __ballot_sync(full, need_maxr);
    while (todo) {
      const int L = __ffs(todo) - 1;
      todo &= todo - 1;
      Mask4 m;
      m.w0 = __shfl_sync(full, mask2.w0, L); m.w1 = __shfl_sync(full, mask2.w1, L);
      m.w2 = __shfl_sync(full, mask2.w2, L); m.w3 = __shfl_sync(full, mask2.w3, L);
      const int kL = __shfl_sync(full, k2, L);
      double mx = 0.0;
      int a_ = -1, b_ = -1;
      if (!PAIRS && kL * kL * kL * kL <= 4 * X.n * X.n) {
        // member rows split over the lanes: lane j takes nodes j, j+32, ... in N1
        for (int a = lane; a < X.n; a += 32) {
          if (!in(m, (uint32_t)a)) continue;
#pragma unroll
          for (int wd = 0; wd < 4; ++wd) {
            uint32_t bits = m.word(wd);
            while (bits) {
              const int b = wd * 32 + __ffs(bits) - 1;
              bits &= bits - 1;
              if (b == a) continue;
              const double v = R((uint32_t)a, (uint32_t)b);
              if (v > mx) { mx = v; a_ = a; b_ = b; }
            }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {   // max-reduce (any witness of an equal max is fine)
          const double v2 = __shfl_xor_sync(full, mx, o);
          const int a2 = __shfl_xor_sync(full, a_, o), b2 = __shfl_xor_sync(full, b_, o);
          if (v2 > mx) { mx = v2; a_ = a2; b_ = b2; }
        }
      } else if (PAIRS && kL * kL * kL * kL <= 4 * X.n * X.n) {
        // the k^2 ordered member pairs split over the lanes (k <= 16 here): lane i holds
        // the i-th member node, pair j = (j / k, j % k) is fetched by shuffles, and the R
        // loads of four pairs per lane are in flight together (independent, unrolled)
        uint32_t memv = 0u;
        {
          const uint32_t c0 = __popc(m.w0), c1 = c0 + __popc(m.w1), c2 = c1 + __popc(m.w2);
          const uint32_t i = (uint32_t)lane;
          const uint32_t wd = i < c0 ? 0u : (i < c1 ? 1u : (i < c2 ? 2u : 3u));
          const uint32_t r = i - (wd == 0u ? 0u : (wd == 1u ? c0 : (wd == 2u ? c1 : c2)));
          const uint32_t bits = m.word((int)wd);
          if (i < (uint32_t)kL) memv = wd * 32u + (uint32_t)__fns(bits, 0u, (int)r + 1);
        }
        const uint32_t kk = (uint32_t)kL, npair = kk * kk;
        const uint32_t mg = (uint32_t)((0x100000000ull + kk - 1u) / kk);   // j / k = umulhi(j, mg), j < 2^16
        for (uint32_t base = 0; base < npair; base += 128u) {
          double v[4];
          uint32_t ja[4], jb[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t j = base + (uint32_t)u * 32u + (uint32_t)lane;
            const uint32_t ia = __umulhi(j, mg), ib = j - ia * kk;
            ja[u] = __shfl_sync(full, memv, (int)(ia & 31u));
            jb[u] = __shfl_sync(full, memv, (int)(ib & 31u));
            v[u] = (j < npair && ia != ib) ? R(ja[u], jb[u]) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (v[u] > mx) { mx = v[u]; a_ = (int)ja[u]; b_ = (int)jb[u]; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {   // max-reduce (any witness of an equal max is fine)
          const double v2 = __shfl_xor_sync(full, mx, o);
          const int a2 = __shfl_xor_sync(full, a_, o), b2 = __shfl_xor_sync(full, b_, o);
          if (v2 > mx) { mx = v2; a_ = a2; b_ = b2; }
        }
      } else {
        uint32_t abv;
        double v;
        const int i = coop_first_v(X.gl_len, [&](int j, uint32_t& ab) {
          ab = X.gl_ab[j];
          return in(m, ab & 0xffu) && in(m, ab >> 8);
        }, [&](int j) { return X.gl_val[j]; }, v, abv);
        if (i >= 0) { mx = v; a_ = (int)(abv & 0xffu); b_ = (int)(abv >> 8); }
      }
      if (lane == L) { need_maxr = false; maxR2 = mx; wa2 = a_; wb2 = b_; }
    }
  }
  __device__ __forceinline__ void finish(const S1Ctx& X) { tex2 = k2 >= 2 ? __dmul_rn(__ldg(X.qe + k2), maxR2) : 0.0; }
  __device__ __forceinline__ void commit() {
    add(dn_, -1); add(up_, +1);
    mask = mask2; k = k2; tin = tin2; win = win2; tex = tex2; maxR = maxR2; wa = wa2; wb = wb2;
  }
};

// psum cached in shared memory when pp >= 2 and dp <= dp_cap.
template <class POS>
__host__ __device__ inline int warp_state_bytes(int N, int pp, int dp, int n, bool s1smem, int dp_cap) {
  return align16(POS::bytes(N)) + ((pp >= 2 && dp <= dp_cap) ? align16(dp * 256) : 0) +
         (s1smem ? align16((n + 3) / 4 * 128) : 0);
}

// ------------------------------------------------------------------ one warp task
template <class POS, class S1, class RT, bool TRACE, int PP>
__device__ __forceinline__ void run_task(const SaParams& P, const SaTask T, const DevCfg C, const RT R,
                                         unsigned char* ws, int lane) {
  // lanes past the task's chain count run a throw-away chain (their outputs are never
  // written) so that the warp stays converged for the cooperative searches
  const bool active = lane < T.count;
  constexpr bool kLargeS1 = !std::is_same<S1, S1Reg<RT>>::value;
  const int N = C.N, pp = PP > 0 ? PP : C.pp, dp = C.dp, n = P.n_nodes;
  const uint32_t chain = (uint32_t)(T.c_first + (T.k0 + lane) * P.world);
  const int slot = T.slot0 + lane;
  S1Ctx X;
  X.qi = P.qtab + C.qi_off; X.qe = P.qtab + C.qe_off; X.tab = P.subset_max;
  X.rank = P.tin_rank ? P.tin_rank + (size_t)T.f * 256 : nullptr;
  X.vs = P.tin_vs ? P.tin_vs + (size_t)T.f * 256 : nullptr;
  X.nl_node = P.nl_node; X.nl_val = P.nl_val; X.gl_ab = P.gl_ab; X.gl_val = P.gl_val;
  X.tl_ac = P.tl_ac ? P.tl_ac + (size_t)T.f * P.tl_stride : nullptr;
  X.tl_val = P.tl_val ? P.tl_val + (size_t)T.f * P.tl_stride : nullptr;
  X.nl_len = 2 * (n - 1); X.gl_len = n * (n - 1); X.tl_len = P.tl_len ? P.tl_len[T.f] : 0;
  X.n = n;

  // psum (Eq.5 sum of every pipeline) cached in shared memory unless dp is large; then the
  // old sums of the touched pipelines are re-summed before the tentative swap instead
  const bool cache = pp >= 2 && dp <= P.psum_dp_cap;
  POS pos{reinterpret_cast<uint32_t*>(ws), lane};
  double* psum = reinterpret_cast<double*>(ws + align16(POS::bytes(N)));
  uint16_t* bperm = P.best_perm + T.perm_off;
  S1 s1;
  if constexpr (kLargeS1) {
    s1.c = reinterpret_cast<uint32_t*>(ws + align16(POS::bytes(N)) + (cache ? align16(dp * 256) : 0));
    s1.lane = lane;
    s1.clear(n);
  } else {
    s1.clear();
  }

  // ---- initial state: identity mapping (R16) and its latency from scratch
  pos.init(N, (uint32_t)C.spn, C.spn_magic);
  for (int w = 0; w < N; ++w) bperm[w * 32 + lane] = (uint16_t)w;
  double tpp = 0.0;
  int nmax = 0;   // pipelines whose sum equals tpp
  for (int z = 0; z < dp; ++z) {
    s1.add_init(pos.node((uint32_t)(z * pp)));
    if (pp >= 2) {
      const double s = pipe_sum<RT, PP>(z, pp, pos, kNone, kNone, 0u, 0u, C.m2, R);
      if (cache) psum[z * 32 + lane] = s;
      if (s > tpp) { tpp = s; nmax = 1; } else if (s == tpp) { ++nmax; }
    }
  }
  s1.finish_init(X, R);

  const double L0 = compose(C.Sb, C.r, C.Ss, tpp, s1.tin, s1.tex);
  double cur = L0, best = L0, best_tpp = tpp, best_tdp = __dadd_rn(s1.tin, s1.tex);
  int best_step = -1;
  uint32_t accepted = 0;
  double beta = sa_beta0(P, T.f, L0);
  const double ia = P.alpha_inv;
  const int trow = (TRACE && active) ? P.trace_slot[slot] : -1;

  if (N >= 2) {
    Draw dnext = draw_swap_rk(0u, chain, (uint32_t)C.e, P.rk, (uint32_t)N);
    for (int i = 0; i < P.iterations; ++i) {
      const Draw d = dnext;
      // the next proposal's Philox words do not depend on this step: issue them now (ILP)
      dnext = draw_swap_rk((uint32_t)(i + 1), chain, (uint32_t)C.e, P.rk, (uint32_t)N);
      const uint32_t rp = pos.raw(d.p), rq = pos.raw(d.q);
      const uint32_t np = POS::node_of(rp), nq = POS::node_of(rq);
      double Lp = cur;
      bool acc = true;
      bool improved = false;
      const bool evald = np != nq;
      uint32_t xp = 0, xq = 0;
      int zp = 0, zq = 0;
      bool two = false, dpchg = false;
      double sA = 0.0, sB = 0.0, tpp2 = tpp;
      int nmax2 = nmax;
      if (evald) {
        // ---- Eq.5: re-sum the (at most two) touched pipelines, maintain the max
        if (pp >= 2) {
          zp = (int)div_small(d.p, C.pp_magic, (uint32_t)pp);
          zq = (int)div_small(d.q, C.pp_magic, (uint32_t)pp);
          xp = d.p - (uint32_t)(zp * pp);
          xq = d.q - (uint32_t)(zq * pp);
          two = zq != zp;
          double oldA, oldB;
          if (cache) {
            oldA = psum[zp * 32 + lane];
            oldB = two ? psum[zq * 32 + lane] : oldA;
          } else {
            if (two) pipe_sum2<RT, PP>(zp, zq, pp, pos, kNone, kNone, 0u, 0u, C.m2, R, oldA, oldB);
            else oldB = oldA = pipe_sum<RT, PP>(zp, pp, pos, kNone, kNone, 0u, 0u, C.m2, R);
          }
          // apply the swap tentatively (reverted below if rejected): the re-sum then reads
          // plain positions, with no per-hop substitution
          pos.swap(d.p, d.q, rp, rq);
          if (two) pipe_sum2<RT, PP>(zp, zq, pp, pos, kNone, kNone, 0u, 0u, C.m2, R, sA, sB);
          else sA = pipe_sum<RT, PP>(zp, pp, pos, kNone, kNone, 0u, 0u, C.m2, R);
          const double snew = two ? dmax(sA, sB) : sA;
          const int keep = nmax - (oldA == tpp ? 1 : 0) - ((two && oldB == tpp) ? 1 : 0);  // untouched at max
          if (keep > 0 || snew >= tpp) {
            // the max is max(tpp if an untouched pipeline still holds it, new sums)
            tpp2 = (keep > 0) ? dmax(tpp, snew) : snew;
            nmax2 = (keep > 0 && tpp2 == tpp ? keep : 0) + (sA == tpp2 ? 1 : 0) + ((two && sB == tpp2) ? 1 : 0);
          } else if (cache) {
            // the unique max pipeline decreased: rescan for the max and its multiplicity in
            // one pass (two independent (max, count) accumulators)
            double m0 = sA, m1 = two ? sB : 0.0;
            int c0 = 1, c1 = two ? 1 : 0;
            int z = 0;
            for (; z + 2 <= dp; z += 2) {
              const double v0 = (z == zp || z == zq) ? 0.0 : psum[z * 32 + lane];
              const double v1 = (z + 1 == zp || z + 1 == zq) ? 0.0 : psum[(z + 1) * 32 + lane];
              c0 = v0 > m0 ? 1 : c0 + (v0 == m0 ? 1 : 0);
              m0 = dmax(m0, v0);
              c1 = v1 > m1 ? 1 : c1 + (v1 == m1 ? 1 : 0);
              m1 = dmax(m1, v1);
            }
            if (z < dp) {
              const double v0 = (z == zp || z == zq) ? 0.0 : psum[z * 32 + lane];
              c0 = v0 > m0 ? 1 : c0 + (v0 == m0 ? 1 : 0);
              m0 = dmax(m0, v0);
            }
            tpp2 = dmax(m0, m1);
            nmax2 = (m0 == tpp2 ? c0 : 0) + (m1 == tpp2 ? c1 : 0);
          } else {
            // no cache: re-sum every pipeline of the tentative mapping
            tpp2 = 0.0;
            nmax2 = 0;
            for (int z = 0; z < dp; ++z) {
              const double v = (z == zp) ? sA : ((z == zq) ? sB : pipe_sum<RT, PP>(z, pp, pos, kNone, kNone, 0u, 0u, C.m2, R));
              if (v > tpp2) { tpp2 = v; nmax2 = 1; } else if (v == tpp2) { ++nmax2; }
            }
          }
        }
        // ---- Eq.6: the stage-1 node multiset changes only if exactly one of p, q is stage 1
        dpchg = (xp == 0u) != (xq == 0u);
        if (dpchg) {
          const uint32_t dn = xp == 0u ? np : nq;   // node losing a stage-1 DP member
          const uint32_t up = xp == 0u ? nq : np;   // node gaining one
          s1.propose(dn, up, X, R);
        }
      }
      s1.coop(X, R);   // warp-converged: long stage-1 searches of any lane, done cooperatively
      if (evald) {
        double tin2 = s1.tin, tex2 = s1.tex;
        if (dpchg) {
          s1.finish(X);
          tin2 = s1.tin2;
          tex2 = s1.tex2;
        }
        Lp = compose(C.Sb, C.r, C.Ss, tpp2, tin2, tex2);
        acc = metropolis_fast(__dadd_rn(Lp, -cur), beta, d.u);
        if (acc) {
          if (pp >= 2) {
            if (cache) {
              psum[zp * 32 + lane] = sA;
              if (two) psum[zq * 32 + lane] = sB;
            }
            tpp = tpp2;
            nmax = nmax2;
          }
          if (dpchg) s1.commit();
          cur = Lp;
          if (Lp < best) {
            best = Lp; best_step = i; best_tpp = tpp; best_tdp = __dadd_rn(s1.tin, s1.tex);
            improved = true;
          }
        }
      }
      if (acc) {
        if (pp < 2 || np == nq) pos.swap(d.p, d.q, rp, rq);   // (already applied when re-summed)
        ++accepted;
      } else if (pp >= 2) {
        pos.swap(d.p, d.q, rq, rp);                             // revert the tentative swap
      }
      if (improved)
        for (int w = 0; w < N; ++w) bperm[w * 32 + lane] = (uint16_t)POS::slot_of(pos.raw((uint32_t)w));
      if (TRACE && trow >= 0 && i < P.trace_cap) {
        pipette_trace_record rec;
        rec.i = (uint32_t)i; rec.p = (uint16_t)d.p; rec.q = (uint16_t)d.q;
        rec.accept = acc ? 1u : 0u; rec.latency = Lp;
        P.trace[(size_t)trow * P.trace_cap + i] = rec;
      }
      beta = __dmul_rn(beta, ia);
    }
  }
  if (active) {
    ChainOut o;
    o.best = best; o.best_tpp = best_tpp; o.best_tdp = best_tdp; o.L0 = L0;
    o.best_step = best_step; o.accepted = accepted; o.f = T.f; o.c = (int32_t)chain;
    P.out[slot] = o;
  }
}

// ------------------------------------------------------------------ MODE 0: hop codes
// Chain state of MODE 0 (n <= 16 nodes, N <= 256 positions), lane-interleaved bytes
// ([w/4][lane] words, so every per-lane byte access hits the lane's own bank):
//   H[w]  hop code of position w = z*pp + x: node(w-1) | node(w) << 4 for x >= 1 (the
//         Eq.5 hop x-1 -> x of pipeline z), node(w) * 17 for x = 0 (the stage-1 worker).
//         node(w) = H[w] >> 4 in both cases.
//   S[w]  slot id of position w (the mapping string of Eq.2; slot < N <= 256)
// The block's table Tt[code][16 copies] = fl(m2 * R[a][b]), a = code & 15, b = code >> 4,
// of the block's configuration: a hop of Eq.5 is one byte extraction, one address, one
// 64-bit shared load and one DADD -- the same product the oracle forms, so the sums are
// bit-identical.  A pipeline's codes are read as whole words.
struct HcState {
  uint8_t* hb;   // byte view of H for this lane: position w at hb + ((w >> 2) << 7) + (w & 3)
  uint8_t* sb;   // same for S
  const uint32_t* hw;   // word view of H for this lane: word j at hw[j * 32]
  __device__ __forceinline__ static uint32_t off(uint32_t w) { return ((w >> 2) << 7) | (w & 3u); }
};

// Eq.5 sum of pipeline z (bytes z*PP .. z*PP+PP-1), stage order.  Tl = this lane's copy
// of the block table (Tt + (lane & 15)); the entry of code c is Tl[c * 16].
template <int PP>
__device__ __forceinline__ double hc_sum(const HcState& st, uint32_t z, int pp_rt, const double* Tl) {
  double s = 0.0;
  if constexpr (PP == 2) {
    s = __dadd_rn(s, Tl[(uint32_t)st.hb[HcState::off(z * 2u + 1u)] * 16u]);
  } else if constexpr (PP >= 4) {
    constexpr int NW = PP / 4;
    uint32_t wd[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) wd[k] = st.hw[(z * (uint32_t)NW + (uint32_t)k) * 32u];
#pragma unroll
    for (int x = 1; x < PP; ++x) {
      const uint32_t code = __byte_perm(wd[x >> 2], 0u, 0x4440u | (uint32_t)(x & 3));
      s = __dadd_rn(s, Tl[code * 16u]);
    }
  } else {
    const uint32_t b = z * (uint32_t)pp_rt;
    for (int x = 1; x < pp_rt; ++x) s = __dadd_rn(s, Tl[(uint32_t)st.hb[HcState::off(b + (uint32_t)x)] * 16u]);
  }
  return s;
}

// Two pipelines in one interleaved loop (two independent DADD chains); za == zb is allowed.
template <int PP>
__device__ __forceinline__ void hc_sum2(const HcState& st, uint32_t za, uint32_t zb, int pp_rt, const double* Tl,
                                        double& sa, double& sb) {
  double a = 0.0, b = 0.0;
  if constexpr (PP == 2) {
    a = __dadd_rn(a, Tl[(uint32_t)st.hb[HcState::off(za * 2u + 1u)] * 16u]);
    b = __dadd_rn(b, Tl[(uint32_t)st.hb[HcState::off(zb * 2u + 1u)] * 16u]);
  } else if constexpr (PP >= 4) {
    constexpr int NW = PP / 4;
    uint32_t wa[NW], wb[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      wa[k] = st.hw[(za * (uint32_t)NW + (uint32_t)k) * 32u];
      wb[k] = st.hw[(zb * (uint32_t)NW + (uint32_t)k) * 32u];
    }
#pragma unroll
    for (int x = 1; x < PP; ++x) {
      const uint32_t ca = __byte_perm(wa[x >> 2], 0u, 0x4440u | (uint32_t)(x & 3));
      const uint32_t cb = __byte_perm(wb[x >> 2], 0u, 0x4440u | (uint32_t)(x & 3));
      a = __dadd_rn(a, Tl[ca * 16u]);
      b = __dadd_rn(b, Tl[cb * 16u]);
    }
  } else {
    const uint32_t ba = za * (uint32_t)pp_rt, bb = zb * (uint32_t)pp_rt;
    for (int x = 1; x < pp_rt; ++x) {
      a = __dadd_rn(a, Tl[(uint32_t)st.hb[HcState::off(ba + (uint32_t)x)] * 16u]);
      b = __dadd_rn(b, Tl[(uint32_t)st.hb[HcState::off(bb + (uint32_t)x)] * 16u]);
    }
  }
  sa = a;
  sb = b;
}

// max over all dp pipelines of the Eq.5 sums and its multiplicity, from the hop codes.
// PP = 2: a pipeline's sum is its single hop term, two pipelines per code word.
template <int PP>
__device__ __forceinline__ void hc_rescan(const HcState& st, int dp, int pp_rt, const double* Tl, double& mx,
                                          int& cnt) {
  double m0 = 0.0, m1 = 0.0;
  int c0 = 0, c1 = 0;
  auto acc = [](double v, double& m, int& c) {
    c = v > m ? 1 : c + (v == m ? 1 : 0);
    m = dmax(m, v);
  };
  if constexpr (PP == 2) {
    const int full = dp >> 1;
    for (int j = 0; j < full; ++j) {
      const uint32_t w = st.hw[j * 32];
      acc(Tl[__byte_perm(w, 0u, 0x4441u) * 16u], m0, c0);
      acc(Tl[__byte_perm(w, 0u, 0x4443u) * 16u], m1, c1);
    }
    if (dp & 1) acc(Tl[__byte_perm(st.hw[full * 32], 0u, 0x4441u) * 16u], m0, c0);
  } else {
    int z = 0;
    for (; z + 2 <= dp; z += 2) {
      double a, b;
      hc_sum2<PP>(st, (uint32_t)z, (uint32_t)z + 1u, pp_rt, Tl, a, b);
      acc(a, m0, c0);
      acc(b, m1, c1);
    }
    if (z < dp) acc(hc_sum<PP>(st, (uint32_t)z, pp_rt, Tl), m0, c0);
  }
  mx = dmax(m0, m1);
  cnt = (m0 == mx ? c0 : 0) + (m1 == mx ? c1 : 0);
}

// MODE 0 counterpart of sa_mode1.cuh's coop_tpp: for each flagged lane L (its unique max
// pipeline decreased), lane j takes pipelines j, j + 32, ... -- L's cached sums (which hold
// the tentative new sums) or re-summed from L's hop codes (which hold the tentative swap) --
// and the (max, count) pair is reduced by redux.sync.  Called by all lanes, converged.
template <int PP>
__device__ __forceinline__ void hc_coop_tpp(bool need, unsigned char* ws, const double* psum, bool cache, int dp, int pp,
                                            const double* Tl, int lane, double& tpp2, int& nmax2) {
  __syncwarp();
  for (unsigned todo = __ballot_sync(0xffffffffu, need); todo; todo &= todo - 1u) {
    const int L = __ffs(todo) - 1;
    HcState stL;
    stL.hb = ws + L * 4;
    stL.sb = nullptr;
    stL.hw = reinterpret_cast<const uint32_t*>(ws) + L;
    double m = 0.0;
    int c = 0;
    for (int z = lane; z < dp; z += 32) {
      const double v = cache ? psum[z * 32 + L] : hc_sum<PP>(stL, (uint32_t)z, pp, Tl);
      c = v > m ? 1 : c + (v == m ? 1 : 0);
      m = dmax(m, v);
    }
    uint32_t cnt;
    m = warp_max_nonneg(m, (uint32_t)c, cnt);
    if (lane == L) { tpp2 = m; nmax2 = (int)cnt; }
  }
}

__host__ __device__ inline int hc_warp_state_bytes(int N, int pp, int dp, int dp_cap) {
  const int plane = align16(((N + 3) / 4) * 128);
  return 2 * plane + ((pp >= 4 && dp <= dp_cap) ? align16(dp * 256) : 0);
}

// One warp task of MODE 0.  Every lane runs the same instruction stream whatever its
// proposal (the swap is always applied tentatively, both touched pipelines are always
// re-summed), so the only divergent paths are the rare rescans and best-mapping writes.
// The block's shared copies of the configuration's stage-1 tables (MODE 0): ranks and
// values of T_in, qe(k), and the subset-max table when n <= 8 (2^n entries).
struct S1Shared {
  const uint8_t* rank;
  const double* vs;
  const double* qe;
  const double* tab;
};

template <bool TRACE, int PP, int NW>
__device__ __forceinline__ void run_task_hc(const SaParams& P, const SaTask T, const DevCfg C, const double* Tl,
                                            const S1Shared& SS, unsigned char* ws, int lane) {
  using RT = RGlob;   // (S1Reg takes no R)
  const bool active = lane < T.count;
  const int N = C.N, pp = PP > 0 ? PP : C.pp, dp = C.dp, n = P.n_nodes;
  const uint32_t chain = (uint32_t)(T.c_first + (T.k0 + lane) * P.world);
  const int slot = T.slot0 + lane;
  S1Ctx X;
  X.qi = P.qtab + C.qi_off;
  if (NW == 2) {   // the block's shared copies
    X.qe = SS.qe; X.tab = SS.tab; X.rank = SS.rank; X.vs = SS.vs;
  } else {
    X.qe = P.qtab + C.qe_off; X.tab = P.subset_max;
    X.rank = P.tin_rank + (size_t)T.f * 256;
    X.vs = P.tin_vs + (size_t)T.f * 256;
  }
  X.n = n;
  const RT Rdummy{nullptr, n, 0};

  const bool cache = pp >= 4 && dp <= P.psum_dp_cap;   // (pp = 2: re-summing one hop is as cheap)
  const int plane = align16(((N + 3) / 4) * 128);
  HcState st;
  st.hb = ws + lane * 4;
  st.sb = ws + plane + lane * 4;
  st.hw = reinterpret_cast<const uint32_t*>(ws) + lane;
  double* psum = reinterpret_cast<double*>(ws + 2 * plane);
  uint16_t* bperm = P.best_perm + T.perm_off;
  S1Reg<RT, NW> s1;
  s1.clear();

  // ---- initial state: identity mapping (R16) and its latency from scratch
  {
    uint32_t prevnd = 0;
    for (int w = 0; w < N; ++w) {
      const uint32_t nd = div_small((uint32_t)w, C.spn_magic, (uint32_t)C.spn);
      const int x = w % pp;
      st.hb[HcState::off((uint32_t)w)] = (uint8_t)(x == 0 ? nd * 17u : (prevnd | (nd << 4)));
      st.sb[HcState::off((uint32_t)w)] = (uint8_t)w;
      bperm[w * 32 + lane] = (uint16_t)w;
      prevnd = nd;
    }
  }
  __syncwarp();
  double tpp = 0.0;
  int nmax = 0;   // pipelines whose sum equals tpp
  for (int z = 0; z < dp; ++z) {
    s1.add_init((uint32_t)st.hb[HcState::off((uint32_t)(z * pp))] >> 4);
    if (pp >= 2) {
      const double s = hc_sum<PP>(st, (uint32_t)z, pp, Tl);
      if (cache) psum[z * 32 + lane] = s;
      if (s > tpp) { tpp = s; nmax = 1; } else if (s == tpp) { ++nmax; }
    }
  }
  s1.finish_init(X, Rdummy);

  const double L0 = compose(C.Sb, C.r, C.Ss, tpp, s1.tin, s1.tex);
  double cur = L0, best = L0, best_tpp = tpp, best_tdp = __dadd_rn(s1.tin, s1.tex);
  int best_step = -1;
  uint32_t accepted = 0;
  double beta = sa_beta0(P, T.f, L0);
  const double ia = P.alpha_inv;
  const int trow = (TRACE && active) ? P.trace_slot[slot] : -1;

  if (N >= 2) {
    Draw dnext = draw_swap_rk(0u, chain, (uint32_t)C.e, P.rk, (uint32_t)N);
    for (int i = 0; i < P.iterations; ++i) {
      const Draw d = dnext;
      dnext = draw_swap_rk((uint32_t)(i + 1), chain, (uint32_t)C.e, P.rk, (uint32_t)N);
      const uint32_t p = d.p, q = d.q;
      uint8_t* const bp = st.hb + HcState::off(p);
      uint8_t* const bq = st.hb + HcState::off(q);
      uint8_t* const sp_ = st.sb + HcState::off(p);
      uint8_t* const sq_ = st.sb + HcState::off(q);
      const uint32_t hp = *bp, hq = *bq, sp = *sp_, sq = *sq_;
      const uint32_t np = hp >> 4, nq = hq >> 4;
      double Lp = cur;
      bool acc = true, improved = false;
      if (pp >= 2) {
        const uint32_t zp = PP > 0 ? p / (uint32_t)PP : div_small(p, C.pp_magic, (uint32_t)pp);
        const uint32_t zq = PP > 0 ? q / (uint32_t)PP : div_small(q, C.pp_magic, (uint32_t)pp);
        const uint32_t xp = p - zp * (uint32_t)pp, xq = q - zq * (uint32_t)pp;
        const bool two = zq != zp;
        const uint32_t zb = two ? zq : zp;
        const bool pn = xp + 1u < (uint32_t)pp, qn = xq + 1u < (uint32_t)pp;   // p+1 / q+1 in the same pipeline
        uint8_t* const bp1 = st.hb + HcState::off(p + 1u);
        uint8_t* const bq1 = st.hb + HcState::off(q + 1u);
        const uint32_t hp1 = pn ? *bp1 : 0u, hq1 = qn ? *bq1 : 0u;
        double oldA, oldB;
        if (cache) {
          oldA = psum[zp * 32 + lane];
          oldB = psum[zb * 32 + lane];
        } else {
          hc_sum2<PP>(st, zp, zb, pp, Tl, oldA, oldB);
        }
        // the hop codes after swapping the nodes of positions p and q (node'(p) = nq,
        // node'(q) = np); when p and q are adjacent both formulas give the shared byte
        const uint32_t vp = xp == 0u ? nq * 17u : (((p - 1u == q) ? np : (hp & 15u)) | (nq << 4));
        const uint32_t vp1 = nq | (((p + 1u == q) ? np : (hp1 >> 4)) << 4);
        const uint32_t vq = xq == 0u ? np * 17u : (((q - 1u == p) ? nq : (hq & 15u)) | (np << 4));
        const uint32_t vq1 = np | (((q + 1u == p) ? nq : (hq1 >> 4)) << 4);
        *bp = (uint8_t)vp;
        if (pn) *bp1 = (uint8_t)vp1;
        *bq = (uint8_t)vq;
        if (qn) *bq1 = (uint8_t)vq1;
        double sA, sB;
        hc_sum2<PP>(st, zp, zb, pp, Tl, sA, sB);
        // ---- T_PP (Eq.5): max over pipelines with its multiplicity
        double tpp2 = tpp;
        int nmax2 = nmax;
        const double snew = dmax(sA, sB);
        const int keep = nmax - (oldA == tpp ? 1 : 0) - ((two && oldB == tpp) ? 1 : 0);  // untouched at max
        const bool fast = keep > 0 || snew >= tpp;
        if (fast) {
          tpp2 = (keep > 0) ? dmax(tpp, snew) : snew;
          nmax2 = (keep > 0 && tpp2 == tpp ? keep : 0) + (sA == tpp2 ? 1 : 0) + ((two && sB == tpp2) ? 1 : 0);
        }
        // the unique max pipeline decreased: rescan over all pipelines (the new sums enter the
        // cache tentatively, restored if rejected) -- up to 8 cached sums per lane, else the
        // whole warp (as MODE 1's coop_tpp: a per-lane rescan runs at a few active lanes)
        if (!fast && cache) {
          psum[zp * 32 + lane] = sA;
          psum[zb * 32 + lane] = sB;
        }
        if (dp <= 8) {   // (few pipelines: per lane; uncached pp = 2 C2 configs measured 19 vs 16 ms coop)
          if (!fast) {
            if (cache) {
              double m = 0.0;
              int c = 0;
              for (int z = 0; z < dp; ++z) {
                const double v = psum[z * 32 + lane];
                c = v > m ? 1 : c + (v == m ? 1 : 0);
                m = dmax(m, v);
              }
              tpp2 = m;
              nmax2 = c;
            } else {
              hc_rescan<PP>(st, dp, pp, Tl, tpp2, nmax2);   // (H already holds the tentative swap)
            }
          }
        } else {
          hc_coop_tpp<PP>(!fast, ws, psum, cache, dp, pp, Tl, lane, tpp2, nmax2);
        }
        // ---- Eq.6: the stage-1 node multiset changes only if exactly one of p, q is a
        //      stage-1 position and the two nodes differ
        const bool dpchg = ((xp == 0u) != (xq == 0u)) && np != nq;
        double tin2 = s1.tin, tex2 = s1.tex;
        if (dpchg) {
          const uint32_t dn = xp == 0u ? np : nq;   // node losing a stage-1 DP member
          const uint32_t up = xp == 0u ? nq : np;   // node gaining one
          s1.propose(dn, up, X, Rdummy);
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
            best = Lp; best_step = i; best_tpp = tpp; best_tdp = __dadd_rn(s1.tin, s1.tex);
            improved = true;
          }
        } else {   // revert the tentative hop codes (reverse order: adjacent bytes end right)
          if (!fast && cache) {
            psum[zb * 32 + lane] = oldB;
            psum[zp * 32 + lane] = oldA;
          }
          if (qn) *bq1 = (uint8_t)hq1;
          *bq = (uint8_t)hq;
          if (pn) *bp1 = (uint8_t)hp1;
          *bp = (uint8_t)hp;
        }
      } else {
        // pp = 1: every position is a stage-1 position, the multiset never changes (Eq.6)
        // and there are no hops (Eq.5): L' = cur, accepted
        *bp = (uint8_t)hq;
        *bq = (uint8_t)hp;
      }
      if (acc) {
        *sp_ = (uint8_t)sq;
        *sq_ = (uint8_t)sp;
        ++accepted;
      }
      // best-mapping copy, warp-cooperative (the warp is converged here): the lanes copy
      // the slot plane of each improved lane together, 32 positions per instruction
      for (uint32_t imp = __ballot_sync(0xffffffffu, improved); imp; imp &= imp - 1u) {
        const int L = __ffs(imp) - 1;
        const uint8_t* sbL = ws + plane + L * 4;
        for (int w = lane; w < N; w += 32) bperm[w * 32 + L] = (uint16_t)sbL[HcState::off((uint32_t)w)];
      }
      if (TRACE && trow >= 0 && i < P.trace_cap) {
        pipette_trace_record rec;
        rec.i = (uint32_t)i; rec.p = (uint16_t)d.p; rec.q = (uint16_t)d.q;
        rec.accept = acc ? 1u : 0u; rec.latency = Lp;
        P.trace[(size_t)trow * P.trace_cap + i] = rec;
      }
      beta = __dmul_rn(beta, ia);
    }
  }
  if (active) {
    ChainOut o;
    o.best = best; o.best_tpp = best_tpp; o.best_tdp = best_tdp; o.L0 = L0;
    o.best_step = best_step; o.accepted = accepted; o.f = T.f; o.c = (int32_t)chain;
    P.out[slot] = o;
  }
}

// ------------------------------------------------------------------ MODE 1 (sa_mode1.cuh)
// n <= 128 nodes, N <= 256 positions: slot-byte chain state, the block's shared R table,
// stage-1 state S1M (canonical list witnesses), per-configuration warp regions.
#include "sa_mode1.cuh"

// ------------------------------------------------------------------ full move set (NEXT-1)
// The paper's three movements (R21): swap, migration (remove the element at p,
// insert it at index q) and reverse (positions min(p,q)..max(p,q)).  A migration or a
// reverse changes up to N positions at once, and a warp almost always holds one, so
// every proposal is evaluated in full from the slot bytes (the oracle's definition in
// the kernel's fixed order, O(N) per step) and rejected moves are undone in place.
__device__ __forceinline__ void move_bytes(uint8_t* sb, int kind, uint32_t p, uint32_t q) {
  if (kind == 0) {
    const uint8_t a = sb[HcState::off(p)], b = sb[HcState::off(q)];
    sb[HcState::off(p)] = b;
    sb[HcState::off(q)] = a;
  } else if (kind == 1) {
    const uint8_t x = sb[HcState::off(p)];
    if (p < q) {
      for (uint32_t w = p; w < q; ++w) sb[HcState::off(w)] = sb[HcState::off(w + 1u)];
    } else {
      for (uint32_t w = p; w > q; --w) sb[HcState::off(w)] = sb[HcState::off(w - 1u)];
    }
    sb[HcState::off(q)] = x;
  } else {
    uint32_t lo = min(p, q), hi = max(p, q);
    for (; lo < hi; ++lo, --hi) {
      const uint8_t a = sb[HcState::off(lo)], b = sb[HcState::off(hi)];
      sb[HcState::off(lo)] = b;
      sb[HcState::off(hi)] = a;
    }
  }
}
__device__ __forceinline__ void unmove_bytes(uint8_t* sb, int kind, uint32_t p, uint32_t q) {
  if (kind == 1) move_bytes(sb, 1, q, p);
  else move_bytes(sb, kind, p, q);
}

// max over ordered pairs a != b of the node set m (|m| = kk >= 2) of R[a][b]: the member
// rows (k^2 loads) or the first pair of the global R-sorted list inside m (about (n/k)^2)
__device__ __forceinline__ double pair_max_lane(const Mask4& m, int kk, const S1Ctx& X, const double* R) {
  const int n = X.n;
  double mx = 0.0;
  if (kk * kk <= max(n, 64)) {   // (k^2 pair loads against ~(n/k)^2 list probes; measured on C4, C5)
#pragma unroll
    for (int wd = 0; wd < 4; ++wd) {
      uint32_t ba = m.word(wd);
      while (ba) {
        const int a = wd * 32 + __ffs(ba) - 1;
        ba &= ba - 1;
#pragma unroll
        for (int wd2 = 0; wd2 < 4; ++wd2) {
          uint32_t bb = m.word(wd2);
          while (bb) {
            const int b = wd2 * 32 + __ffs(bb) - 1;
            bb &= bb - 1;
            if (b != a) mx = dmax(mx, __ldg(R + a * n + b));
          }
        }
      }
    }
    return mx;
  }
  // every lane scans the same list prefix (L1-resident); four probes per round in flight
  int i = 0;
  for (; i + 4 <= X.gl_len; i += 4) {
    const uint2 ab4 = __ldg(reinterpret_cast<const uint2*>(X.gl_ab + i));   // (i is a multiple of 4)
    const uint32_t e0 = ab4.x & 0xffffu, e1 = ab4.x >> 16, e2 = ab4.y & 0xffffu, e3 = ab4.y >> 16;
    const bool h0 = m.test(e0 & 0xffu) && m.test(e0 >> 8), h1 = m.test(e1 & 0xffu) && m.test(e1 >> 8);
    const bool h2 = m.test(e2 & 0xffu) && m.test(e2 >> 8), h3 = m.test(e3 & 0xffu) && m.test(e3 >> 8);
    if (h0 | h1 | h2 | h3) return __ldg(X.gl_val + i + (h0 ? 0 : (h1 ? 1 : (h2 ? 2 : 3))));
  }
  for (; i < X.gl_len; ++i) {
    const uint32_t ab = __ldg(X.gl_ab + i);
    if (m.test(ab & 0xffu) && m.test(ab >> 8)) return __ldg(X.gl_val + i);
  }
  return 0.0;
}

// Eq.3-6 of the mapping in the slot plane, from scratch.  MODE 0: nibble-coded table
// (16 lane copies), stage-1 counts as register nibbles, T_in by ranks, T_ex by the
// subset-max table.  MODE 1: n x n table, counts in shared memory, T_in over the member
// nodes, T_ex by pair_max_lane.
template <int MODE, int PP, int NW>
__device__ __forceinline__ double full_eval(const uint8_t* sb, const uint32_t* sw, uint8_t* cb, const DevCfg& C,
                                            const SbCtx& K, const S1Ctx& X, const double* R, double& tpp_o,
                                            double& tdp_o) {
  using CT = typename std::conditional<NW == 2, uint32_t, uint64_t>::type;
  const int pp = PP > 0 ? PP : C.pp, dp = C.dp, n = K.n;
  CT cnt = 0;
  Mask4 mask;
  mask.clear();
  if constexpr (MODE == 1)
    for (int a = 0; a < n; a += 4) *reinterpret_cast<uint32_t*>(cb + HcState::off((uint32_t)a)) = 0u;
  auto stage1 = [&](uint32_t nd) {
    if constexpr (MODE == 0) {
      cnt += (CT)1 << (4u * nd);
    } else {
      cb[HcState::off(nd)] = (uint8_t)(cb[HcState::off(nd)] + 1u);
      mask.set(nd);
    }
  };
  auto term = [&](uint32_t a, uint32_t b) -> double {
    return MODE == 0 ? K.T[(a | (b << 4)) * 16u] : K.hop(a, b);
  };
  double tpp = 0.0;
  for (int z = 0; z < dp; ++z) {
    double s = 0.0;
    if constexpr (PP >= 4) {
      constexpr int NWD = PP / 4;
      uint32_t wd[NWD];
#pragma unroll
      for (int k = 0; k < NWD; ++k) wd[k] = sw[((uint32_t)z * NWD + (uint32_t)k) * 32u];
      uint32_t prev = K.node(wd[0] & 0xffu);
      stage1(prev);
#pragma unroll
      for (int x = 1; x < PP; ++x) {
        const uint32_t cur = K.node(__byte_perm(wd[x >> 2], 0u, 0x4440u | (uint32_t)(x & 3)));
        s = __dadd_rn(s, term(prev, cur));
        prev = cur;
      }
    } else {
      const uint32_t b = (uint32_t)(z * pp);
      uint32_t prev = K.node(sb[HcState::off(b)]);
      stage1(prev);
      for (int x = 1; x < pp; ++x) {
        const uint32_t cur = K.node(sb[HcState::off(b + (uint32_t)x)]);
        s = __dadd_rn(s, term(prev, cur));
        prev = cur;
      }
    }
    tpp = dmax(tpp, s);
  }
  double tin = 0.0, tex = 0.0;
  if constexpr (MODE == 0) {
    uint32_t m = 0u, rmin = 0xffu;
    for (int a = 0; a < n; ++a) {
      const uint32_t c = (uint32_t)(cnt >> (4u * (uint32_t)a)) & 15u;
      if (c) {
        m |= 1u << a;
        rmin = min(rmin, (uint32_t)__ldg(X.rank + a * 16 + c));
      }
    }
    tin = rmin == 0xffu ? 0.0 : __ldg(X.vs + rmin);
    const int k = __popc(m);
    tex = k >= 2 ? __dmul_rn(__ldg(X.qe + k), __ldg(X.tab + m)) : 0.0;
  } else {
#pragma unroll
    for (int wd = 0; wd < 4; ++wd) {
      uint32_t bits = mask.word(wd);
      while (bits) {
        const uint32_t a = (uint32_t)(wd * 32 + __ffs(bits) - 1);
        bits &= bits - 1;
        const uint32_t c = cb[HcState::off(a)];
        if (c >= 2u) tin = dmax(tin, __dmul_rn(__ldg(X.qi + c), __ldg(R + a * (uint32_t)n + a)));
      }
    }
    const int k = mask.count();
    tex = k >= 2 ? __dmul_rn(__ldg(X.qe + k), pair_max_lane(mask, k, X, R)) : 0.0;
  }
  tpp_o = tpp;
  tdp_o = __dadd_rn(tin, tex);
  return compose(C.Sb, C.r, C.Ss, tpp, tin, tex);
}

// One warp task with the full move set (MODE 0 or 1 state layout, slot plane only).
template <int MODE, bool TRACE, int PP, int NW>
__device__ __forceinline__ void run_task_full(const SaParams& P, const SaTask T, const DevCfg C, const double* Tt,
                                              unsigned char* ws, int lane) {
  const bool active = lane < T.count;
  const int N = C.N, n = P.n_nodes;
  const uint32_t chain = (uint32_t)(T.c_first + (T.k0 + lane) * P.world);
  const int slot = T.slot0 + lane;
  S1Ctx X;
  X.qi = P.qtab + C.qi_off; X.qe = P.qtab + C.qe_off; X.tab = P.subset_max;
  X.rank = MODE == 0 ? P.tin_rank + (size_t)T.f * 256 : nullptr;
  X.vs = MODE == 0 ? P.tin_vs + (size_t)T.f * 256 : nullptr;
  X.gl_ab = P.gl_ab; X.gl_val = P.gl_val; X.gl_len = n * (n - 1);
  X.n = n;
  SbCtx K;
  K.T = MODE == 0 ? Tt + (lane & 15) : Tt; K.m2 = C.m2; K.lg = (uint32_t)P.r_lg;
  K.n = n; K.spn = (uint32_t)C.spn; K.spn_magic = C.spn_magic;
  K.spn_sh = (C.spn & (C.spn - 1)) == 0 ? (uint32_t)(31 - __clz(C.spn)) : 32u;
  K.m16 = (uint32_t)((65536u + (uint32_t)C.spn - 1u) / (uint32_t)C.spn);
  const int plane = align16(((N + 3) / 4) * 128);
  // MODE 0 layout: [hop-code plane (unused)][slot plane]; MODE 1: [slot plane][counts]
  unsigned char* splane = MODE == 0 ? ws + plane : ws;
  uint8_t* sb = splane + lane * 4;
  const uint32_t* sw = reinterpret_cast<const uint32_t*>(splane) + lane;
  uint8_t* cb = MODE == 1 ? ws + plane + lane * 4 : nullptr;
  uint16_t* bperm = P.best_perm + T.perm_off;
  for (int w = 0; w < N; ++w) {
    sb[HcState::off((uint32_t)w)] = (uint8_t)w;
    bperm[w * 32 + lane] = (uint16_t)w;
  }
  __syncwarp();
  double tpp, tdp;
  const double L0 = full_eval<MODE, PP, NW>(sb, sw, cb, C, K, X, P.R, tpp, tdp);
  double cur = L0, best = L0, best_tpp = tpp, best_tdp = tdp;
  int best_step = -1;
  uint32_t accepted = 0;
  double beta = sa_beta0(P, T.f, L0);
  const double ia = P.alpha_inv;
  const int trow = (TRACE && active) ? P.trace_slot[slot] : -1;
  const int th_swap = 2048 - P.w_migrate - P.w_reverse, th_mig = 2048 - P.w_reverse;
  if (N >= 2) {
    DrawM next = draw_move_rk(0u, chain, (uint32_t)C.e, P.rk, (uint32_t)N);
    for (int i = 0; i < P.iterations; ++i) {
      const DrawM m = next;
      next = draw_move_rk((uint32_t)(i + 1), chain, (uint32_t)C.e, P.rk, (uint32_t)N);
      const int kind = (int)m.t < th_swap ? 0 : ((int)m.t < th_mig ? 1 : 2);
      move_bytes(sb, kind, m.d.p, m.d.q);
      double tpp2, tdp2;
      const double Lp = full_eval<MODE, PP, NW>(sb, sw, cb, C, K, X, P.R, tpp2, tdp2);
      const bool acc = metropolis_fast(__dadd_rn(Lp, -cur), beta, m.d.u);
      bool improved = false;
      if (acc) {
        cur = Lp;
        ++accepted;
        if (Lp < best) {
          best = Lp; best_step = i; best_tpp = tpp2; best_tdp = tdp2;
          improved = true;
        }
      } else {
        unmove_bytes(sb, kind, m.d.p, m.d.q);
      }
      __syncwarp();
      for (uint32_t imp = __ballot_sync(0xffffffffu, improved); imp; imp &= imp - 1u) {   // (as in run_task_hc)
        const int L = __ffs(imp) - 1;
        const uint8_t* sbL = splane + L * 4;
        for (int w = lane; w < N; w += 32) bperm[w * 32 + L] = (uint16_t)sbL[HcState::off((uint32_t)w)];
      }
      if (TRACE && trow >= 0 && i < P.trace_cap) {
        pipette_trace_record rec;
        rec.i = (uint32_t)i; rec.p = (uint16_t)m.d.p; rec.q = (uint16_t)m.d.q;
        rec.accept = acc ? 1u : 0u; rec.latency = Lp;
        P.trace[(size_t)trow * P.trace_cap + i] = rec;
      }
      beta = __dmul_rn(beta, ia);
    }
  }
  if (active) {
    ChainOut o;
    o.best = best; o.best_tpp = best_tpp; o.best_tdp = best_tdp; o.L0 = L0;
    o.best_step = best_step; o.accepted = accepted; o.f = T.f; o.c = (int32_t)chain;
    P.out[slot] = o;
  }
}

// MODE 0: n <= 16 nodes, N <= 256, spn <= 15: hop-code chain state (run_task_hc), register
//         stage-1 state, the block's m2*R table in shared memory, subset-max table.
// MODE 1: n <= 128, N <= 256: packed positions, S1Large, R through L1.
// MODE 2: general (N <= 1024): 32-bit positions, S1Large, R through L1.
// launch bounds per mode: MODE 0 4 warps x 3 blocks; MODE 1 4 warps x 3 blocks (small
// table) or 8 warps x 1 block (BIG: a table of up to 128 KB shared by more warps); MODE 2.
// MODE 0 with n <= 8 (NW = 2): the m2*R table has 120 codes (15 KB), so 4 blocks fit.
template <int MODE, bool BIG, int NW = 4>
struct SaLB {
  static constexpr int threads = MODE == 1 ? kSaM1Warps * 32 : ((MODE == 0 && NW == 2) ? kSaThreadsN8 : 128);
  static constexpr int blocks = MODE == 0 ? (NW == 2 ? kSaBlocksN8 : 3) : (MODE == 1 ? 1 : 2);
};

// FULL: the full move set (run_task_full) -- a separate instantiation, so the swap kernel's
// instruction footprint stays small (its cold start after an L2 flush refetches the code).
template <int MODE, bool TRACE, int NW = 4, bool BIG = false, bool FULL = false>
__global__ void __launch_bounds__(SaLB<MODE, BIG, NW>::threads, SaLB<MODE, BIG, NW>::blocks) k_sa_chains(SaParams P) {
  using POS = PosWide;
  using RT = RGlob;
  using S1 = S1Large<RT>;
  extern __shared__ __align__(16) unsigned char smem[];
  double* Rs = reinterpret_cast<double*>(smem);
  const int n = P.n_nodes;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  RT R{P.R, n, lane};
  const double* Tl = Rs + (lane & 15);   // MODE 0: this lane's copy of the block's m2*R table
  // MODE 0: the block's stage-1 tables after the m2*R table (kS1SharedBytes)
  constexpr int kCodes = NW == 2 ? kSaCodesN8 : 256;   // hop codes a | b << 4 in the table
  double* s1_vs = Rs + kCodes * 16;
  double* s1_qe = s1_vs + 256;
  double* s1_tab = s1_qe + 32;
  uint8_t* s1_rank = reinterpret_cast<uint8_t*>(s1_tab + 256);
  // (n <= 8 only: at n <= 16 the extra shared memory costs more than the loads save)
  const S1Shared SS{s1_rank, s1_vs, s1_qe, s1_tab};
  // MODE 1: the cluster's R (row stride 2^r_lg) and the first plen entries of the global
  // pair list, loaded once; every configuration shares them
  const uint16_t* pl_s = reinterpret_cast<const uint16_t*>(smem + align16((8 << (2 * P.r_lg))));
  if constexpr (MODE == 1) {
    const int np = 1 << P.r_lg;
    for (int i = threadIdx.x; i < np * np; i += blockDim.x) {
      const int a = i >> P.r_lg, b = i & (np - 1);
      Rs[i] = (a < n && b < n) ? P.R[a * n + b] : 0.0;
    }
    uint16_t* pw = const_cast<uint16_t*>(pl_s);
    for (int i = threadIdx.x; i < P.plen; i += blockDim.x) pw[i] = P.gl_ab[i];
  }
  unsigned char* ws = smem + P.r_smem_bytes + wid * P.warp_smem_bytes;
  __shared__ int s_chunk;
  int table_cfg = -1;
  bool first_fetch = true;
  for (;;) {
    // a block takes one chunk: up to warps-per-block consecutive tasks of ONE configuration
    // (host-built), so the block runs one code path (I-cache locality), shares the
    // configuration's m2*R table (MODE 0/1), and its warps finish together
    // The first chunk of a block is the one its SM slot points at (chunk slot*SMs + smid,
    // snaking: reversed on odd slots): the chunk list is longest first, so the first wave
    // puts one of the heaviest chunks on every SM with the lightest of the next group beside
    // it, whatever order the blocks start in.
    // Later chunks come from the global counter; a claim flag per chunk makes every chunk
    // run exactly once either way.
    __syncthreads();
    if (threadIdx.x == 0) {
      int c = -1;
      if (first_fetch) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        const int slot = atomicAdd(P.sm_slot + (smid % (uint32_t)P.n_sms), 1);
        const int sm = (int)(smid % (uint32_t)P.n_sms);
        const int pref = slot * P.n_sms + ((slot & 1) ? P.n_sms - 1 - sm : sm);   // snake: heavy beside light
        if (pref < P.n_chunks && atomicExch(P.claimed + pref, 1) == 0) c = pref;
      }
      while (c < 0) {
        const int g = atomicAdd(P.task_counter, 1);
        if (g >= P.n_chunks) { c = P.n_chunks; break; }
        if (atomicExch(P.claimed + g, 1) == 0) c = g;
      }
      s_chunk = c;
    }
    first_fetch = false;
    __syncthreads();
    const int ch = s_chunk;
    if (ch >= P.n_chunks) break;
    const int2 chunk = P.chunks[ch];
    if constexpr (MODE == 0) {
      const int cfg0 = P.tasks[chunk.x].cfg;
      if (cfg0 != table_cfg) {   // block-uniform: rebuild the table for this configuration
        const double m2 = P.cfgs[cfg0].m2;
        if constexpr (MODE == 0) {
          for (int i = threadIdx.x; i < kCodes * 16; i += blockDim.x) {
            const int code = i >> 4, a = code & 15, b = code >> 4;
            Rs[i] = (a < n && b < n) ? __dmul_rn(m2, P.R[a * n + b]) : 0.0;
          }
          // the configuration's stage-1 tables (all chunks of a configuration share f)
          if (NW == 2) {
          const int f0 = P.tasks[chunk.x].f;
          const DevCfg& C0 = P.cfgs[cfg0];
          for (int i = threadIdx.x; i < 256; i += blockDim.x) {
            s1_rank[i] = P.tin_rank[(size_t)f0 * 256 + i];
            s1_vs[i] = P.tin_vs[(size_t)f0 * 256 + i];
          }
          for (int i = threadIdx.x; i < 32; i += blockDim.x) s1_qe[i] = i <= min(C0.dp, n) ? P.qtab[C0.qe_off + i] : 0.0;
          for (int i = threadIdx.x; i < (1 << n); i += blockDim.x) {
            const int k = __popc(i);
            s1_tab[i] = (k >= 2 && k <= min(C0.dp, n)) ? __dmul_rn(P.qtab[C0.qe_off + k], P.subset_max[i]) : 0.0;
          }
          }
        }
        table_cfg = cfg0;
      }
    }
    __syncthreads();
    if (wid >= chunk.y) continue;
    const int t = chunk.x + wid;
    const SaTask T = P.tasks[t];
    const DevCfg C = P.cfgs[T.cfg];
    // MODE 1: the warp's region has its configuration's size (task flags, bits 0-15)
    if constexpr (MODE == 1) ws = smem + P.r_smem_bytes + wid * (int)(((uint32_t)T.pad & 0xffffu) * 16u);
    unsigned long long t_start = 0;
    if (lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    if constexpr (FULL && (MODE == 0 || MODE == 1)) {   // the full move set
      switch (C.pp) {
        case 4: run_task_full<MODE, TRACE, 4, NW>(P, T, C, Rs, ws, lane); break;
        case 8: run_task_full<MODE, TRACE, 8, NW>(P, T, C, Rs, ws, lane); break;
        case 16: run_task_full<MODE, TRACE, 16, NW>(P, T, C, Rs, ws, lane); break;
        default: run_task_full<MODE, TRACE, 0, NW>(P, T, C, Rs, ws, lane); break;
      }
    } else if constexpr (MODE == 0) {
      switch (C.pp) {   // compile-time pipeline depth for the common power-of-two depths
        case 1: run_task_hc<TRACE, 1, NW>(P, T, C, Tl, SS, ws, lane); break;
        case 2: run_task_hc<TRACE, 2, NW>(P, T, C, Tl, SS, ws, lane); break;
        case 4: run_task_hc<TRACE, 4, NW>(P, T, C, Tl, SS, ws, lane); break;
        case 8: run_task_hc<TRACE, 8, NW>(P, T, C, Tl, SS, ws, lane); break;
        case 16: run_task_hc<TRACE, 16, NW>(P, T, C, Tl, SS, ws, lane); break;
        case 32: run_task_hc<TRACE, 32, NW>(P, T, C, Tl, SS, ws, lane); break;
        default: run_task_hc<TRACE, 0, NW>(P, T, C, Tl, SS, ws, lane); break;
      }
    } else if constexpr (MODE == 1) {
      run_task_sb_pp<TRACE, true, BIG>(P, T, C, Rs, pl_s, ws, lane);   // (power-of-two spn: the host's MODE 1 rule)
    } else {
      switch (C.pp) {
        case 1: run_task<POS, S1, RT, TRACE, 1>(P, T, C, R, ws, lane); break;
        case 2: run_task<POS, S1, RT, TRACE, 2>(P, T, C, R, ws, lane); break;
        case 4: run_task<POS, S1, RT, TRACE, 4>(P, T, C, R, ws, lane); break;
        case 8: run_task<POS, S1, RT, TRACE, 8>(P, T, C, R, ws, lane); break;
        case 16: run_task<POS, S1, RT, TRACE, 16>(P, T, C, R, ws, lane); break;
        case 32: run_task<POS, S1, RT, TRACE, 32>(P, T, C, R, ws, lane); break;
        default: run_task<POS, S1, RT, TRACE, 0>(P, T, C, R, ws, lane); break;
      }
    }
    __syncwarp();
    if (lane == 0) {
      unsigned long long t_end;
      uint32_t smid;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      reinterpret_cast<ulonglong4*>(P.task_prof)[t] = make_ulonglong4(t_start, t_end, smid, (unsigned long long)T.cfg);
    }
  }
}

// Sorted tables of the cluster for S1Large (n <= 256).  Node lists: for each node a, the
// 2(n-1) values R[a][b] and R[b][a] (b != a) in descending order with their partner b.
// Ties are broken by index, so the order is total.  One block per node.
__global__ void k_node_lists(const double* __restrict__ R, int n, uint8_t* __restrict__ nl_node,
                             double* __restrict__ nl_val) {
  const int a = blockIdx.x, L = 2 * (n - 1);
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    const int bi = i >> 1, b = bi < a ? bi : bi + 1;
    const double v = (i & 1) ? R[b * n + a] : R[a * n + b];
    int r = 0;
    for (int j = 0; j < L; ++j) {
      const int bj = j >> 1, b2 = bj < a ? bj : bj + 1;
      const double u = (j & 1) ? R[b2 * n + a] : R[a * n + b2];
      r += (u > v || (u == v && j < i)) ? 1 : 0;
    }
    nl_node[(size_t)a * L + r] = (uint8_t)b;
    nl_val[(size_t)a * L + r] = v;
  }
}

// Global list: all ordered pairs a != b by R[a][b] descending (one thread per pair).
__global__ void k_pair_list(const double* __restrict__ R, int n, uint16_t* __restrict__ gl_ab,
                            double* __restrict__ gl_val) {
  const int L = n * (n - 1);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L) return;
  const int a = i / (n - 1), bi = i % (n - 1), b = bi < a ? bi : bi + 1;
  const double v = R[a * n + b];
  int r = 0;
  for (int j = 0; j < L; ++j) {
    const int a2 = j / (n - 1), bj = j % (n - 1), b2 = bj < a2 ? bj : bj + 1;
    const double u = R[a2 * n + b2];
    r += (u > v || (u == v && j < i)) ? 1 : 0;
  }
  gl_ab[r] = (uint16_t)(a | (b << 8));
  gl_val[r] = v;
}

// Per feasible config (block f): the (a, c) entries, 2 <= c <= min(spn, dp), sorted by
// qi(c) R[a][a] descending (ties by index); tl_len[f] entries, row stride `stride`.
__global__ void k_tin_list(const DevCfg* __restrict__ cfgs, const int* __restrict__ feas,
                           const double* __restrict__ qtab, const double* __restrict__ R, int n, int stride,
                           uint16_t* __restrict__ tl_ac, double* __restrict__ tl_val, int* __restrict__ tl_len) {
  const int f = blockIdx.x;
  const DevCfg C = cfgs[feas[f]];
  const int cmax = min(min(C.spn, C.dp), 255);
  const int per = cmax >= 2 ? cmax - 1 : 0;
  const int L = min(n * per, stride);
  if (threadIdx.x == 0) tl_len[f] = L;
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    const int a = i / per, c = 2 + i % per;
    const double v = __dmul_rn(qtab[C.qi_off + c], R[a * n + a]);
    int r = 0;
    for (int j = 0; j < L; ++j) {
      const int a2 = j / per, c2 = 2 + j % per;
      const double u = __dmul_rn(qtab[C.qi_off + c2], R[a2 * n + a2]);
      r += (u > v || (u == v && j < i)) ? 1 : 0;
    }
    tl_ac[(size_t)f * stride + r] = (uint16_t)(a | (c << 8));
    tl_val[(size_t)f * stride + r] = v;
  }
}

// Subset-max table for the inter-node term of Eq.6 (R10): tab[m] = max over ordered pairs
// a != b of nodes in bit set m of R[a][b] (0 for |m| < 2).  max is exact, so the value
// is the one a pairwise scan gives.  One thread per subset, n <= 16.
__global__ void k_subset_max(const double* __restrict__ R, int n, double* __restrict__ tab) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= (1u << n)) return;
  double mx = 0.0;
  for (int a = 0; a < n; ++a) {
    if (!((m >> a) & 1u)) continue;
    for (int b = 0; b < n; ++b)
      if (b != a && ((m >> b) & 1u)) mx = dmax(mx, R[a * n + b]);
  }
  tab[m] = mx;
}

// Per feasible config (block f): rank every value qi(c)*R[a][a], a < n, 2 <= c <= min(spn,
// dp), in descending order (ties by index), so that T_in = the value of the smallest rank
// present.  rank[f][a*16 + c] (255 when c < 2 or out of range), vs[f][rank] = value.
__global__ void k_tin_rank(const DevCfg* __restrict__ cfgs, const int* __restrict__ feas, const double* __restrict__ qtab,
                           const double* __restrict__ R, int n, uint8_t* __restrict__ rank, double* __restrict__ vs) {
  const int f = blockIdx.x;
  const DevCfg C = cfgs[feas[f]];
  const int cmax = min(min(C.spn, C.dp), 15);
  const int per = cmax >= 2 ? cmax - 1 : 0;      // values c = 2..cmax per node
  const int P = n * per;
  __shared__ double v[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) rank[(size_t)f * 256 + i] = 0xff;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    const int a = i / per, c = 2 + i % per;
    v[i] = __dmul_rn(qtab[C.qi_off + c], R[a * n + a]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    int r = 0;
    for (int j = 0; j < P; ++j) r += (v[j] > v[i] || (v[j] == v[i] && j < i)) ? 1 : 0;
    const int a = i / per, c = 2 + i % per;
    rank[(size_t)f * 256 + a * 16 + c] = (uint8_t)r;
    vs[(size_t)f * 256 + r] = v[i];
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

// Host-side handles of the K3 variants (MODE 0/1/2 as above; TRACE records).
// Per-node pair rows for S1M (MODE 1): for node u (one warp per node), every ordered pair
// with u as an endpoint, in global-list order (so by R descending, ties by index), entry =
// list rank | other endpoint << 16 | (u is the first endpoint) << 24; rows of `stride`
// entries (a multiple of 4), padded with 0xffffffff (rank 0xffff: beyond any witness).
__global__ void k_partner_lists(const uint16_t* __restrict__ gl, int n, uint32_t* __restrict__ pt, int stride) {
  const int u = blockIdx.x, lane = threadIdx.x & 31, L = n * (n - 1);
  int base = 0;
  for (int j0 = 0; j0 < L; j0 += 32) {
    const int j = j0 + lane;
    const uint32_t p = j < L ? (uint32_t)gl[j] : 0u;
    const bool hit = j < L && ((int)(p & 0xffu) == u || (int)(p >> 8) == u);
    const unsigned b = __ballot_sync(0xffffffffu, hit);
    const uint32_t first = (p & 0xffu) == (uint32_t)u ? 1u : 0u, other = first ? (p >> 8) : (p & 0xffu);
    if (hit) pt[(size_t)u * stride + base + __popc(b & ((1u << lane) - 1u))] = (uint32_t)j | (other << 16) | (first << 24);
    base += __popc(b);
  }
  for (int i = base + lane; i < stride; i += 32) pt[(size_t)u * stride + i] = 0xffffffffu;
}

// Host-side handles of the K3 variants (MODE 0/1/2 as above; TRACE records).
const void* sa_kernel(int mode, bool trace, int n_nodes, bool full) {
  if (full) {
    if (mode == 0 && n_nodes <= 8)
      return trace ? (const void*)k_sa_chains<0, true, 2, false, true> : (const void*)k_sa_chains<0, false, 2, false, true>;
    if (mode == 0)
      return trace ? (const void*)k_sa_chains<0, true, 4, false, true> : (const void*)k_sa_chains<0, false, 4, false, true>;
    if (mode == 1)
      return trace ? (const void*)k_sa_chains<1, true, 4, false, true> : (const void*)k_sa_chains<1, false, 4, false, true>;
    return nullptr;   // (MODE 2: rejected by the host)
  }
  if (mode == 0 && n_nodes <= 8) return trace ? (const void*)k_sa_chains<0, true, 2> : (const void*)k_sa_chains<0, false, 2>;
  if (mode == 0) return trace ? (const void*)k_sa_chains<0, true, 4> : (const void*)k_sa_chains<0, false, 4>;
  if (mode == 1 && n_nodes >= 64)   // (BIG: large clusters, direct-mode joins always cooperative)
    return trace ? (const void*)k_sa_chains<1, true, 4, true> : (const void*)k_sa_chains<1, false, 4, true>;
  if (mode == 1) return trace ? (const void*)k_sa_chains<1, true> : (const void*)k_sa_chains<1, false>;
  return trace ? (const void*)k_sa_chains<2, true> : (const void*)k_sa_chains<2, false>;
}

// Per-warp chain-state bytes: MODE 0 and 2 (psum cached when dp <= dp_cap); MODE 1 with the
// per-configuration flags of its tasks (counts, cache)
int sa_warp_state_bytes(int mode, int N, int pp, int dp, int n, int dp_cap, bool nib) {
  if (mode == 0) return hc_warp_state_bytes(N, pp, dp, dp_cap);
  return warp_state_bytes<PosWide>(N, pp, dp, n, true, dp_cap);
}
int sa_m1_warp_state_bytes(int N, int dp, int n, bool counts, bool cache, bool nib, bool direct) {
  return m1_warp_state_bytes(N, dp, n, counts, cache, nib, direct);
}
int sa_m1_count_bytes(int n, bool nib) { return sb_count_bytes(n, nib); }

}  // namespace pip

namespace pip {
// Per enumerated configuration e: the sum of its warp tasks' durations (ns, globaltimer
// stamps of the task profile) and their count -- the longest-first order of the next
// search's work plan uses the means (host.cu, build_plan).
__global__ void k_cfg_cost(const unsigned long long* __restrict__ prof, const SaTask* __restrict__ tasks, int n_tasks,
                           unsigned long long* __restrict__ acc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tasks) return;
  const ulonglong4 p = reinterpret_cast<const ulonglong4*>(prof)[t];
  const int e = tasks[t].cfg;
  atomicAdd(acc + 2 * e, p.y > p.x ? p.y - p.x : 0ull);
  atomicAdd(acc + 2 * e + 1, 1ull);
}
}  // namespace pip
