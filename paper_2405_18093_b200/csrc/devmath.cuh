// devmath.cuh -- device arithmetic primitives of the Pipette hot path (sm_100a).
//
// Every floating-point operation is an explicit round-to-nearest intrinsic
// (__dadd_rn / __dmul_rn / __ddiv_rn), so ptxas can never contract a multiply and an
// add into a DFMA: the results are the IEEE binary64 values DESIGN.md section 3 fixes.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pip {

// Philox4x32-10 (Salmon et al., SC'11), the counter-based generator of R14: counter
// (step, chain, e, 0), key (seed lo, seed hi).  Ten rounds of two 32x32->64 multiplies
// (Weyl key schedule between rounds).
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// Same generator with the ten round keys precomputed (they depend only on the seed, so the
// SA kernel receives them as kernel parameters, i.e. constant-bank operands), and each
// 32x32 multiply as one 64-bit IMAD.WIDE giving both halves.
struct RoundKeys {
  uint32_t x[10], y[10];
};

__host__ __device__ inline RoundKeys philox_round_keys(uint2 k) {
  RoundKeys r;
  for (int i = 0; i < 10; ++i) {
    r.x[i] = k.x;
    r.y[i] = k.y;
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return r;
}

__device__ __forceinline__ uint4 philox4x32_10_rk(uint4 c, const RoundKeys& rk) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long p0 = (unsigned long long)0xD2511F53u * c.x;
    const unsigned long long p1 = (unsigned long long)0xCD9E8D57u * c.z;
    c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ rk.x[r], (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ rk.y[r],
                   (uint32_t)p0);
  }
  return c;
}

// One proposal's randomness (R14): p uniform in [0,N), q uniform in [0,N)\{p}, u in [0,1).
struct Draw {
  uint32_t p, q;
  double u;
};

__device__ __forceinline__ Draw draw_from_words(uint4 w, uint32_t N) {
  Draw d;
  d.p = __umulhi(w.x, N);
  uint32_t q = d.p + 1u + __umulhi(w.y, N - 1u);
  d.q = (q >= N) ? q - N : q;
  const unsigned long long bits = ((unsigned long long)(w.z >> 5) << 26) | (unsigned long long)(w.w >> 6);
  d.u = __dmul_rn(__ull2double_rn(bits), 0x1p-53);
  return d;
}

// A proposal of the full move set (R21): the same (p, q, u) plus the move selector
// t = ((w2 & 31) << 6) | (w3 & 63) in [0, 2048), the 11 bits u leaves unused.
struct DrawM {
  Draw d;
  uint32_t t;
};

__device__ __forceinline__ DrawM draw_move_rk(uint32_t step, uint32_t chain, uint32_t e, const RoundKeys& rk,
                                              uint32_t N);

__device__ __forceinline__ Draw draw_swap(uint32_t step, uint32_t chain, uint32_t e, uint2 key, uint32_t N) {
  return draw_from_words(philox4x32_10(make_uint4(step, chain, e, 0u), key), N);
}

__device__ __forceinline__ Draw draw_swap_rk(uint32_t step, uint32_t chain, uint32_t e, const RoundKeys& rk,
                                             uint32_t N) {
  return draw_from_words(philox4x32_10_rk(make_uint4(step, chain, e, 0u), rk), N);
}

__device__ __forceinline__ DrawM draw_move_rk(uint32_t step, uint32_t chain, uint32_t e, const RoundKeys& rk,
                                              uint32_t N) {
  const uint4 w = philox4x32_10_rk(make_uint4(step, chain, e, 0u), rk);
  DrawM m;
  m.d = draw_from_words(w, N);
  m.t = ((w.z & 31u) << 6) | (w.w & 63u);
  return m;
}

// e^x for x <= 0 from IEEE + - * and floor only (R15): Cody-Waite reduction by ln 2
// (hi/lo split), Horner evaluation of the degree-13 Taylor polynomial with coefficients
// fl(1/n!) (hex literals below), exact scaling by 2^k built from the exponent bits.
__device__ __forceinline__ double exp_det(double x) {
  if (x < -708.0) return 0.0;
  const double k = floor(__dadd_rn(__dmul_rn(x, 1.4426950408889634), 0.5));
  const double r = __dadd_rn(__dadd_rn(x, -__dmul_rn(k, 6.93147180369123816490e-01)),
                             -__dmul_rn(k, 1.90821492927058770002e-10));
  double p = 0x1.6124613a86d09p-33;                       // 1/13!
  p = __dadd_rn(__dmul_rn(p, r), 0x1.1eed8eff8d898p-29);  // 1/12!
  p = __dadd_rn(__dmul_rn(p, r), 0x1.ae64567f544e4p-26);  // 1/11!
  p = __dadd_rn(__dmul_rn(p, r), 0x1.27e4fb7789f5cp-22);  // 1/10!
  p = __dadd_rn(__dmul_rn(p, r), 0x1.71de3a556c734p-19);  // 1/9!
  p = __dadd_rn(__dmul_rn(p, r), 0x1.a01a01a01a01ap-16);  // 1/8!
  p = __dadd_rn(__dmul_rn(p, r), 0x1.a01a01a01a01ap-13);  // 1/7!
  p = __dadd_rn(__dmul_rn(p, r), 0x1.6c16c16c16c17p-10);  // 1/6!
  p = __dadd_rn(__dmul_rn(p, r), 0x1.1111111111111p-7);   // 1/5!
  p = __dadd_rn(__dmul_rn(p, r), 0x1.5555555555555p-5);   // 1/4!
  p = __dadd_rn(__dmul_rn(p, r), 0x1.5555555555555p-3);   // 1/3!
  p = __dadd_rn(__dmul_rn(p, r), 0x1.0000000000000p-1);   // 1/2!
  p = __dadd_rn(__dmul_rn(p, r), 1.0);                    // 1/1!
  p = __dadd_rn(__dmul_rn(p, r), 1.0);                    // 1/0!
  const long long ki = (long long)k;                      // in [-1022, 0]
  return __dmul_rn(p, __longlong_as_double((ki + 1023LL) << 52));
}

// Metropolis decision (R13): accept iff d <= 0 or u < exp_det(-(d*beta)).
__device__ __forceinline__ bool metropolis(double d, double beta, double u) {
  if (d <= 0.0) return true;
  return u < exp_det(-__dmul_rn(d, beta));
}

// Out-of-line exact tail of metropolis_fast (rare: keeps the hot loop's code small).
static __device__ __noinline__ bool metropolis_exact(double x, double u) { return u < exp_det(x); }

// The same decision with a cheap screen: e^x is first approximated in fp32 (relative
// error < 2e-5 for -87 <= x <= 0: argument rounding 5.2e-6, ex2.approx scaling 5.2e-6,
// ex2.approx 2e-7), and exp_det (< 1 ulp from e^x) is evaluated only when u falls within
// +-0.1% of the approximation.  Outside that band both give the same answer, so the
// decision is bit-identical to metropolis().
__device__ __forceinline__ bool metropolis_fast(double d, double beta, double u) {
  if (d <= 0.0) return true;
  const double x = -__dmul_rn(d, beta);
  if (x < -708.0) return false;                       // exp_det(x) == 0 and u >= 0
  if (x < -87.0) return u == 0.0;                     // e^x < 1.7e-38 < 2^-53 <= any u > 0
  const double y = (double)__expf(__double2float_rn(x));
  if (u < __dmul_rn(y, 0.999)) return true;
  if (u > __dmul_rn(y, 1.001)) return false;
  return metropolis_exact(x, u);
}

// max of two non-NaN doubles: DSETP + two selects (fmax adds NaN handling, ~5 SASS
// instructions).  Every latency term, sum and table value here is finite and >= +0, where it
// returns the same value as fmax.
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }

// Warp max of non-negative doubles (their bit patterns order like the values) by two 32-bit
// redux.sync, and the sum of c over the lanes holding it: three REDUX instead of a five-level
// shuffle butterfly on (double, int) pairs.
__device__ __forceinline__ double warp_max_nonneg(double m, uint32_t c, uint32_t& count) {
  const unsigned full = 0xffffffffu;
  const unsigned long long b = (unsigned long long)__double_as_longlong(m);
  const uint32_t hi = (uint32_t)(b >> 32), lo = (uint32_t)b;
  const uint32_t H = __reduce_max_sync(full, hi);
  const uint32_t Lo = __reduce_max_sync(full, hi == H ? lo : 0u);
  const unsigned long long B = ((unsigned long long)H << 32) | Lo;
  count = __reduce_add_sync(full, b == B ? c : 0u);
  return __longlong_as_double((long long)B);
}

// Eq.3-4 composition with the Eq.5 value inside T_bubble (R6):
// T = (((Sb + T_PP) * r) + Ss) + (T_in + T_ex).
__device__ __forceinline__ double compose(double Sb, double r, double Ss, double tpp, double tin, double tex) {
  return __dadd_rn(__dadd_rn(__dmul_rn(__dadd_rn(Sb, tpp), r), Ss), __dadd_rn(tin, tex));
}

// x / d for x < 2^16 via a 32-bit multiply-high with m = ceil(2^32 / d), d >= 2
// (error < x/2^32 < 1/d, so the floor is exact).
__device__ __forceinline__ uint32_t div_small(uint32_t x, uint32_t m, uint32_t d) {
  return d == 1u ? x : __umulhi(x, m);
}

// Bit set of node ids (< 32*MW) held in registers.  MW == 4 is spelled out as four scalar
// words: with an array member the compiler may place the set in local memory and index it.
template <int MW>
struct Mask {
  uint32_t w[MW];
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int i = 0; i < MW; ++i) w[i] = 0u;
  }
  __device__ __forceinline__ void set(uint32_t a) {
#pragma unroll
    for (int i = 0; i < MW; ++i) w[i] |= ((a >> 5) == (uint32_t)i) ? (1u << (a & 31)) : 0u;
  }
  __device__ __forceinline__ void reset(uint32_t a) {
#pragma unroll
    for (int i = 0; i < MW; ++i) w[i] &= ((a >> 5) == (uint32_t)i) ? ~(1u << (a & 31)) : 0xffffffffu;
  }
  __device__ __forceinline__ bool test(uint32_t a) const {
    uint32_t x = 0u;
#pragma unroll
    for (int i = 0; i < MW; ++i) x |= ((a >> 5) == (uint32_t)i) ? w[i] : 0u;
    return (x >> (a & 31)) & 1u;
  }
  __device__ __forceinline__ int count() const {
    int c = 0;
#pragma unroll
    for (int i = 0; i < MW; ++i) c += __popc(w[i]);
    return c;
  }
};

struct Mask4 {
  uint32_t w0, w1, w2, w3;
  __device__ __forceinline__ void clear() { w0 = w1 = w2 = w3 = 0u; }
  __device__ __forceinline__ uint32_t word(int i) const { return i == 0 ? w0 : (i == 1 ? w1 : (i == 2 ? w2 : w3)); }
  __device__ __forceinline__ void set(uint32_t a) {
    const uint32_t b = 1u << (a & 31), q = a >> 5;
    w0 |= q == 0u ? b : 0u; w1 |= q == 1u ? b : 0u; w2 |= q == 2u ? b : 0u; w3 |= q == 3u ? b : 0u;
  }
  __device__ __forceinline__ void reset(uint32_t a) {
    const uint32_t b = ~(1u << (a & 31)), q = a >> 5;
    w0 &= q == 0u ? b : ~0u; w1 &= q == 1u ? b : ~0u; w2 &= q == 2u ? b : ~0u; w3 &= q == 3u ? b : ~0u;
  }
  __device__ __forceinline__ bool test(uint32_t a) const {   // a < 128: two select levels, a wrapping funnel shift
    const uint32_t lo = (a & 32u) ? w1 : w0, hi = (a & 32u) ? w3 : w2;
    const uint32_t x = (a & 64u) ? hi : lo;
    return (__funnelshift_r(x, x, a) & 1u) != 0u;
  }
  __device__ __forceinline__ int count() const { return __popc(w0) + __popc(w1) + __popc(w2) + __popc(w3); }
};

}  // namespace pip
