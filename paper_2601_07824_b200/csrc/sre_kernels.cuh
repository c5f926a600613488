// sre_kernels.cuh -- sm_100a kernels for the exact stabilizer Renyi entropy (Alg. 2 of
// arXiv:2601.07824).
//
// Half-length reformulation (reading C3):
//   For an X-string a != 0 with pivot p = highest set bit of a, pair x with x^a (x_p = 0).
//   v_x = conj(psi_{x^a}) psi_x satisfies v_{x^a} = conj(v_x), hence
//     chi_b(a) = 2 Re-hat(b')      if a.b even,   chi_b(a) = 2i Im-hat(b')   if a.b odd,
//   where b' is b with bit p removed and Re-hat / Im-hat are the unnormalised Walsh-Hadamard
//   transforms over the N-1 remaining bits of A_y = Re v_{x(y)}, B_y = Im v_{x(y)},
//   x(y) = y with a 0 inserted at bit p.  Every |chi_b| is 2|y| for exactly one output y of the
//   two real (N-1)-bit transforms.  For a = 0 (v real), the pivot butterfly is applied at
//   generation: A_y = (|psi_x0|^2 + |psi_x1|^2)/2, B_y = (|psi_x0|^2 - |psi_x1|^2)/2, x1 = x0 + 2^{N-1},
//   so again |chi| = 2|y|.  Kernels accumulate t' = y^2; the reduce kernel rescales t = 4 t'.
//
// Transform engine: a "unit" of NT = 2^(T-5) threads holds a 2^T-point real vector, 32 values
// per thread.  Round k puts 5 index bits [s_k, s_k+5) in the register index j (radix-32
// butterflies in registers); between rounds the unit transposes through shared memory with
// one pad double per 32 (swz(e) = e + (e >> 5): additive addressing, conflict-free for every
// round layout).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <type_traits>


namespace sre {

constexpr int MAXA = 4;          // Renyi indices per sweep (more are done in extra sweeps)
constexpr int NACC = MAXA + 2;   // [0,MAXA) alpha sums, [MAXA] purity, [MAXA+1] t ln t

struct Alphas {
  int n;                // alphas in this sweep
  int need_log;         // any alpha == 1
  int any_real;         // any kind == 2 (non-integer alpha)
  unsigned long long* hist;   // spectrum epilogue (two-pass kernels; nullptr = off)
  double* chi;          // sre_chi through the production pass-B kernels: chi_b(a) element-wise (nullptr = off)
  unsigned long long chi_a0;  // first X-string of the launch (chi mode)
  int kind[MAXA];       // 0: integer exponent iexp[i] >= 1, 2: general real power
  int iexp[MAXA];
  double alpha[MAXA];
};

// value type of a precision: FP64 (default) or FP32 mode (transform/workspace in FP32,
// accumulators FP64; north-star "optional FP32 mode", tolerance 1e-4)
template <class R> struct Cx;
template <> struct Cx<double> { using T = double2; };
template <> struct Cx<float> { using T = float2; };

// ------------------------------------------------------------------------------------------
// small helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t ins0(uint64_t y, int p) {  // insert a 0 bit at position p
  const uint64_t lo = y & ((1ull << p) - 1ull);
  return lo | ((y >> p) << (p + 1));
}
__device__ __forceinline__ uint32_t lay(uint32_t t, uint32_t j, int s) {
  return (t & ((1u << s) - 1u)) | (j << s) | ((t >> s) << (s + 5));
}
// shared-memory index of element e: one pad double per 32 (additive, conflict-free for every
// round layout because the half-warp's lanes always span 4 distinct bits of e)
__device__ __forceinline__ uint32_t swz(uint32_t e) { return e + (e >> 5); }
__host__ __device__ constexpr int padded(int n) { return n + n / 32; }

struct Round { int s, rlo, rhi; };
__host__ __device__ constexpr int nrounds(int T, int LO) {
  int hi = T, n = 0;
  while (hi > LO) { hi = (hi - LO >= 5) ? hi - 5 : LO; ++n; }
  return n;
}
__host__ __device__ constexpr Round round_k(int T, int LO, int k) {
  int hi = T;
  for (int i = 0;; ++i) {
    Round r{0, 0, 0};
    if (hi - LO >= 5) { r.s = hi - 5; r.rlo = 0; r.rhi = 5; }
    else { r.s = hi - 5 > 0 ? hi - 5 : 0; r.rlo = LO - r.s; r.rhi = hi - r.s; }
    if (i == k) return r;
    hi = (hi - LO >= 5) ? hi - 5 : LO;
  }
}

template <int RLO, int RHI, class R>
__device__ __forceinline__ void bfly32(R (&v)[32]) {
#pragma unroll
  for (int b = RLO; b < RHI; ++b) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if ((i >> b) & 1) continue;
      const int k = i | (1 << b);
      const R u = v[i], w = v[k];
      v[i] = u + w;
      v[k] = u - w;
    }
  }
}

struct BarWarp { __device__ __forceinline__ void sync() const { __syncwarp(); } };
struct BarNamed {
  int id, n;
  __device__ __forceinline__ void sync() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
  }
};
struct BarCta { __device__ __forceinline__ void sync() const { __syncthreads(); } };

// Rounds K..end of the transform of NP planes (each a 2^T vector in its own 2^T smem slice).
// On entry the registers hold round K-1's layout (or round 0's with butterflies pending if
// K == 0); on exit the final round's layout with all butterflies done.
template <int T, int LO, int K, int NP, class Bar, bool SEQ = false, class R = double>
struct Rounds {
  // SEQ: the NP planes share one 2^T smem slice and are exchanged one after the other.
  __device__ __forceinline__ static void run(R (&v)[NP][32], R* sm, uint32_t t, const Bar& bar) {
    constexpr int NR = nrounds(T, LO);
    if constexpr (K < NR) {
      constexpr Round r = round_k(T, LO, K);
      if constexpr (K > 0) {
        constexpr Round q = round_k(T, LO, K - 1);
        if constexpr (SEQ) {
#pragma unroll
          for (int pl = 0; pl < NP; ++pl) {
            bar.sync();
#pragma unroll
            for (int j = 0; j < 32; ++j) sm[swz(lay(t, j, q.s))] = v[pl][j];
            bar.sync();
#pragma unroll
            for (int j = 0; j < 32; ++j) v[pl][j] = sm[swz(lay(t, j, r.s))];
          }
        } else {
          bar.sync();
#pragma unroll
          for (int pl = 0; pl < NP; ++pl)
#pragma unroll
            for (int j = 0; j < 32; ++j) sm[pl * padded(1 << T) + swz(lay(t, j, q.s))] = v[pl][j];
          bar.sync();
#pragma unroll
          for (int pl = 0; pl < NP; ++pl)
#pragma unroll
            for (int j = 0; j < 32; ++j) v[pl][j] = sm[pl * padded(1 << T) + swz(lay(t, j, r.s))];
        }
      }
#pragma unroll
      for (int pl = 0; pl < NP; ++pl) bfly32<r.rlo, r.rhi>(v[pl]);
      Rounds<T, LO, K + 1, NP, Bar, SEQ, R>::run(v, sm, t, bar);
    }
  }
};
template <int T, int LO>
__host__ __device__ constexpr int final_s() { return round_k(T, LO, nrounds(T, LO) - 1).s; }

// ------------------------------------------------------------------------------------------
// epilogue: power sums of t' = y^2 (DESIGN "Epilogue"); A2 = compile-time single alpha == 2
// ------------------------------------------------------------------------------------------
template <bool A2, class R = double>
struct Epi {
  __device__ __forceinline__ static void add(R (&acc)[NACC], R y, const Alphas& al) {
    const R t = y * y;
    acc[MAXA] += t;
    if constexpr (A2) {
      acc[0] = fma(t, t, acc[0]);
    } else {
#pragma unroll
      for (int i = 0; i < MAXA; ++i) {
        if (i >= al.n) break;            // uniform: stop after the requested alphas
        if (al.kind[i] == 0) {
          R pw = t;
          for (int k = 1; k < al.iexp[i]; ++k) pw *= t;
          acc[i] += pw;
        } else {
          acc[i] += (t > R(0)) ? exp(R(al.alpha[i]) * log(t)) : R(0);
        }
      }
      if (al.need_log) acc[MAXA + 1] += (t > R(0)) ? t * log(t) : R(0);
    }
  }
};

// Natural logarithm for the general-alpha epilogue (t > 0 normal):
// t = 2^e m with m in [sqrt(1/2), sqrt(2)), ln t = e ln 2 + 2 atanh(s), s = (m - 1)/(m + 1), |s| <= 0.1716,
// 2 atanh(s) = 2 s (1 + s^2/3 + ... + s^18/19): truncation s^20/21 < 1e-17 relative, so the result is
// within a few ulp (the CUDA log() spends ~4x the instructions on correct rounding we do not need:
// every term of sum t ln t has the same sign, so 1e-15 relative per term is far inside the 1e-10 bar).
__device__ __forceinline__ double ln_fast(double t) {
  long long b = __double_as_longlong(t);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  double m = __longlong_as_double((b & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);   // [1, 2)
  const bool hi = m > 1.4142135623730951;
  m = hi ? 0.5 * m : m;
  e += hi ? 1 : 0;
  // s = (m - 1) / (m + 1) with a reciprocal: MUFU approximation + two Newton steps (2^-23 -> 2^-92),
  // shorter and branch-free compared with the IEEE division sequence
  const double y = m + 1.0;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  r = fma(r, fma(-y, r, 1.0), r);
  r = fma(r, fma(-y, r, 1.0), r);
  const double s = (m - 1.0) * r;
  const double z = s * s, z2 = z * z, z4 = z2 * z2;
  // 1/3 + z/5 + ... + z^8/19 by Estrin's scheme (dependency depth 4 instead of 8)
  const double p01 = fma(1.0 / 5, z, 1.0 / 3), p23 = fma(1.0 / 9, z, 1.0 / 7);
  const double p45 = fma(1.0 / 13, z, 1.0 / 11), p67 = fma(1.0 / 17, z, 1.0 / 15);
  const double p03 = fma(p23, z2, p01), p47 = fma(p67, z2, p45);
  const double p = fma(fma(1.0 / 19, z4, p47), z4, p03);
  const double ls = fma(2.0 * s * z, p, 2.0 * s);                                         // 2 atanh(s)
  return fma((double)e, 0.6931471805599453, fma((double)e, 2.3190468138462996e-17, ls)); // e ln2 (hi + lo)
}
// Table-driven ln for the t ln t pass (t = y^2 <= 1/4, so ln t <= -1.38 and nothing cancels): m in
// [1, 2) split at its top 7 mantissa bits i; r_i = RN(1 / m_i), m_i = 1 + (i + 1/2)/128, L_i = -ln r_i;
// ln m = L_i + ln(1 + d), d = m r_i - 1 (one FMA, |d| < 2^-8), ln(1 + d) to d^7 by Estrin (truncation
// d^8/8 < 2e-20).  11 FP64 ops against ln_fast's ~25; 1.7e-16 relative on t <= 1/4 (host check against
// logl).  The 2 KB table lives in each CTA's shared memory, built once per launch (ln_table_init).
__device__ __forceinline__ double2* ln_table() {
  __shared__ double2 tab[128];
  return tab;
}
__device__ __forceinline__ void ln_table_init(bool need) {   // every thread of the CTA, before any use
  if (need) {
    double2* tab = ln_table();
    for (int i = threadIdx.x; i < 128; i += blockDim.x) {
      const double r = 1.0 / (1.0 + (i + 0.5) / 128.0);
      tab[i] = make_double2(r, -log(r));
    }
    __syncthreads();
  }
}
__device__ __forceinline__ double ln_tab(double t) {
  const long long b = __double_as_longlong(t);
  const int e = (int)((b >> 52) & 0x7ff) - 1023;
  const double2 T = ln_table()[(b >> 45) & 127];
  const double m = __longlong_as_double((b & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  const double d = fma(m, T.x, -1.0), d2 = d * d;
  const double q = fma(fma(1.0 / 7, d, -1.0 / 6), d2, fma(1.0 / 5, d, -1.0 / 4));
  const double poly = fma(fma(q, d2, fma(1.0 / 3, d, -0.5)), d2, d);
  return fma((double)e, 0.6931471805599453, fma((double)e, 2.3190468138462996e-17, T.y + poly));
}
__device__ __forceinline__ float ln_tab(float t) { return logf(t); }

// e^z for z <= 0 (t^alpha = e^(alpha ln t)): z = k ln 2 + r, |r| <= ln2/2, Taylor to r^13
// (truncation r^14/14! < 2e-17 relative); 2^k applied in two exponent steps; z < -745 -> 0.
__device__ __forceinline__ double exp_fast(double z) {
  if (!(z > -745.0)) return 0.0;
  const double k = rint(z * 1.4426950408889634);
  const double r = fma(-k, 2.3190468138462996e-17, fma(-k, 0.6931471805599453, z));
  double p = 1.0 / 6227020800.0;
  p = fma(p, r, 1.0 / 479001600.0); p = fma(p, r, 1.0 / 39916800.0); p = fma(p, r, 1.0 / 3628800.0);
  p = fma(p, r, 1.0 / 362880.0); p = fma(p, r, 1.0 / 40320.0); p = fma(p, r, 1.0 / 5040.0);
  p = fma(p, r, 1.0 / 720.0); p = fma(p, r, 1.0 / 120.0); p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0); p = fma(p, r, 0.5); p = fma(p, r, 1.0); p = fma(p, r, 1.0);
  const int ki = (int)k;                                                                // in [-1075, 1]
  const int k1 = ki / 2, k2 = ki - k1;
  return p * __longlong_as_double((long long)(k1 + 1023) << 52) * __longlong_as_double((long long)(k2 + 1023) << 52);
}
__device__ __forceinline__ float ln_fast(float t) { return logf(t); }
__device__ __forceinline__ float exp_fast(float z) { return expf(z); }

// Epilogue of one tile's values per thread into a fresh local sum, then one add into the long-lived
// accumulators: keeps the running-sum chains short (DESIGN "Summation").  The general-alpha body is
// compact (ln_fast ~30 SASS instead of the ~120 of log(), which made a full unroll I-cache bound in
// round 1).  Terms with t below 1e-300 add 0 (t ln t > -1e-297); in FP32 mode the cut is t > 0.
template <bool A2, class R, int M>
__device__ __forceinline__ void tile_accumulate(double (&acc)[NACC], const R (&v)[M], const Alphas& al) {
  constexpr R kTiny = std::is_same<R, double>::value ? R(1e-300) : R(0);
  R loc[NACC];          // FP32 mode: local sums in FP32, one conversion per tile
#pragma unroll
  for (int i = 0; i < NACC; ++i) loc[i] = R(0);
  if constexpr (A2) {
#pragma unroll
    for (int j = 0; j < M; ++j) Epi<true, R>::add(loc, v[j], al);
  } else if (!al.any_real) {
    // Integer alphas (+ t ln t when some alpha = 1): registers only, unrolled passes over the tile.  The round-1 compact loop
    // staged t through a per-thread local array, which misses L1 beside a ~200 KB smem ring (LDL
    // long-scoreboard stalls: config 2 pass B 3.2x slower, measured); one fused per-value body over all
    // slots grows the kernel past the instruction cache; several partial sums per pass spill at M = 64.
    // one pass for the purity and the powers t^1..t^4 (independent sums), exponents > 4 in their own pass
    R s1 = R(0), s2 = R(0), s3 = R(0), s4 = R(0);
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const R t = v[j] * v[j], t2 = t * t;
      s1 += t;
      s2 += t2;
      s3 = fma(t2, t, s3);
      s4 = fma(t2, t2, s4);
    }
    loc[MAXA] += s1;
#pragma unroll
    for (int i = 0; i < MAXA; ++i) {
      if (i >= al.n) break;
      const int e = al.iexp[i];
      R sum = e == 1 ? s1 : e == 2 ? s2 : e == 3 ? s3 : s4;
      if (e > 4) {
        sum = R(0);
#pragma unroll
        for (int j = 0; j < M; ++j) {
          const R t = v[j] * v[j];
          R pw = t;
          for (int k = 1; k < e; ++k) pw *= t;
          sum += pw;
        }
      }
      loc[i] += sum;
    }
    if (al.need_log) {                          // two interleaved sums (more spill at M = 64)
      R l0 = R(0), l1 = R(0);
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const R t = v[j] * v[j];
        const R x = t > kTiny ? t * ln_tab(t) : R(0);
        if (j & 1) l1 += x; else l0 += x;
      }
      loc[MAXA + 1] += l0 + l1;
    }
  } else {
    // some non-integer alpha (rare): a compact rolled loop over a per-thread local copy of t (unrolled
    // exp(alpha ln t) bodies spill at M = 64)
    R tv[M];
#pragma unroll
    for (int j = 0; j < M; ++j) tv[j] = v[j] * v[j];
#pragma unroll 1
    for (int j = 0; j < M; ++j) {
      const R t = tv[j];
      loc[MAXA] += t;
      const bool pos = t > kTiny;
      const R lt = ln_fast(pos ? t : R(1));
      if (al.need_log) loc[MAXA + 1] = fma(t, pos ? lt : R(0), loc[MAXA + 1]);
#pragma unroll
      for (int i = 0; i < MAXA; ++i) {
        if (i >= al.n) break;
        if (al.kind[i] == 0) {
          R pw = t;
          for (int k = 1; k < al.iexp[i]; ++k) pw *= t;
          loc[i] += pw;
        } else {
          loc[i] += pos ? exp_fast(R(al.alpha[i]) * lt) : R(0);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] += (double)loc[i];
}

// Block reduction of the NACC accumulators; thread 0 adds them to partial[slot].
__device__ __forceinline__ void block_flush(double (&acc)[NACC], double* partial, int slot) {
  __shared__ double red[32][NACC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    double x = acc[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    acc[i] = x;
  }
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NACC; ++i) red[w][i] = acc[i];
  __syncthreads();
  if (threadIdx.x < NACC) {
    double s = 0.0;
    for (int k = 0; k < nw; ++k) s += red[k][threadIdx.x];
    partial[(size_t)slot * NACC + threadIdx.x] += s;
  }
}

// Generation of (A_y, B_y) for the half-index y of X-string a (pivot p; a == 0 special).
template <class R>
__device__ __forceinline__ void gen_pair(const typename Cx<R>::T* __restrict__ psi, uint64_t y, uint64_t a, int p,
                                         int N, R& A, R& B) {
  using C2 = typename Cx<R>::T;
  if (a != 0) {
    const uint64_t x = ins0(y, p);
    const C2 q = __ldg(psi + x);             // alpha_x = psi_x
    const C2 r = __ldg(psi + (x ^ a));       // beta_x = psi_{x^a}
    A = fma(r.x, q.x, r.y * q.y);            // Re conj(beta) alpha
    B = fma(r.x, q.y, -(r.y * q.x));         // Im conj(beta) alpha
  } else {
    const uint64_t x0 = y, x1 = y | (1ull << (N - 1));
    const C2 q0 = __ldg(psi + x0), q1 = __ldg(psi + x1);
    const R n0 = fma(q0.x, q0.x, q0.y * q0.y), n1 = fma(q1.x, q1.x, q1.y * q1.y);
    A = (n0 + n1) * R(0.5);
    B = (n0 - n1) * R(0.5);
  }
}
__device__ __forceinline__ int pivot_of(uint64_t a, int N) { return a ? 63 - __clzll((long long)a) : N - 1; }

// chi_b from an output y of plane pl at half-index bq (debug path, natural b order).
__device__ __forceinline__ void chi_store(double* chi, uint64_t a, int p, int pl, uint64_t bq, double y) {
  uint64_t b0 = ins0(bq, p), b;
  double re = 2.0 * y, im = 0.0;
  if (a == 0) {
    b = b0 | ((uint64_t)pl << p);
  } else {
    const uint64_t arest = a & ~(1ull << p);
    const int par = __popcll(arest & b0) & 1;  // parity of a.b with b_p = 0
    const int bp = pl == 0 ? par : (par ^ 1);  // plane A <-> a.b even, plane B <-> odd
    b = b0 | ((uint64_t)bp << p);
    if (pl == 1) { im = re; re = 0.0; }
  }
  chi[2 * b] = re;
  chi[2 * b + 1] = im;
}

// ------------------------------------------------------------------------------------------
// k_small: T = N-1 <= 10.  Group of G = min(32, 2^T) lanes per X-string, R = 2^T/G values
// per plane per lane; register bits then shuffle bits.  One pass, no workspace.
// ------------------------------------------------------------------------------------------
// Spectrum epilogue (NEXT-2, DESIGN C22): bin k = round(-log2 t) for t = |<P>|^2, k <= 62; bin 63
// holds t < 2^-62.5 and exact zeros.  Decided from the FP64 exponent and mantissa bits.
constexpr int SPEC_BINS = 64;
__device__ __forceinline__ int spec_bin(double t) {
  if (!(t > 0.0)) return SPEC_BINS - 1;
  const long long b = __double_as_longlong(t);
  const int e = (int)((b >> 52) & 0x7ff) - 1023;
  const long long mant = b & 0xfffffffffffffLL;
  const int k = -e - (mant > 0x6a09e667f3bcdLL ? 1 : 0);   // mantissa of sqrt(2)
  return k < 0 ? 0 : (k > SPEC_BINS - 1 ? SPEC_BINS - 1 : k);
}
// Warp-aggregated: lanes holding the same bin elect one leader that adds the popcount (values
// crowd into a few bins, so per-lane shared atomics serialised: 10x slower than the sums).
template <class V, int M>
__device__ __forceinline__ void spec_add(unsigned long long* sh, const V (&v)[M]) {
  const unsigned mask = __activemask();
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const double y = (double)v[j];
    const int bin = spec_bin(4.0 * y * y);                   // t = 4 y^2 (half-length transform)
    const unsigned peers = __match_any_sync(mask, bin);
    if (lane == __ffs(peers) - 1) atomicAdd(sh + bin, (unsigned long long)__popc(peers));
  }
}

template <int T, bool A2, bool DEBUG, class V = double>
__global__ void __launch_bounds__(256) k_small(const typename Cx<V>::T* __restrict__ psi_all, int N, uint64_t a0,
                                               uint64_t count, Alphas al, double* partial, double* chi,
                                               const uint64_t* __restrict__ alist, unsigned long long* hist) {
  ln_table_init(!A2 && al.need_log && std::is_same<V, double>::value);   // t ln t pass (tile_accumulate)
  __shared__ unsigned long long shist[SPEC_BINS];   // hist != nullptr: spectrum epilogue
  if (hist) {
    for (int i = threadIdx.x; i < SPEC_BINS; i += blockDim.x) shist[i] = 0ull;
    __syncthreads();
  }
  // alist != nullptr: list mode (sre_x_string_sums) -- item i is X-string alist[i] and its sums
  // go to partial[i * NACC] (reduced over its G lanes) instead of the CTA's running slot.
  constexpr int G = T >= 5 ? 32 : (1 << T);
  constexpr int LG = T >= 5 ? 5 : T;
  constexpr int R = (1 << T) / G;
  constexpr int PER_CTA = 256 / G;
  const typename Cx<V>::T* psi = psi_all + ((size_t)blockIdx.y << N);
  const int g = threadIdx.x & (G - 1);
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * PER_CTA;
  const uint64_t warp_first = (uint64_t)blockIdx.x * PER_CTA + (threadIdx.x >> 5) * (32 / G);
  for (uint64_t base = warp_first; base < count; base += stride) {
    const uint64_t item = base + ((threadIdx.x & 31) >> LG);
    const bool valid = item < count;
    const uint64_t a = alist ? (valid ? alist[item] : 0) : a0 + item;
    const int p = pivot_of(a, N);
    V A[R], B[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      A[j] = V(0); B[j] = V(0);
      if (valid) gen_pair<V>(psi, (uint64_t)g + (uint64_t)G * j, a, p, N, A[j], B[j]);
    }
#pragma unroll
    for (int h = 1; h < R; h <<= 1)
#pragma unroll
      for (int i = 0; i < R; ++i) {
        if (i & h) continue;
        V u = A[i], w = A[i + h]; A[i] = u + w; A[i + h] = u - w;
        u = B[i]; w = B[i + h]; B[i] = u + w; B[i + h] = u - w;
      }
#pragma unroll
    for (int m = 1; m < G; m <<= 1) {
      const bool up = (g & m) != 0;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const V pa = __shfl_xor_sync(0xffffffffu, A[i], m, G);
        const V pb = __shfl_xor_sync(0xffffffffu, B[i], m, G);
        A[i] = up ? pa - A[i] : A[i] + pa;
        B[i] = up ? pb - B[i] : B[i] + pb;
      }
    }
    if (valid) {
      if constexpr (DEBUG) {
#pragma unroll
        for (int j = 0; j < R; ++j) {
          chi_store(chi, a, p, 0, (uint64_t)g + (uint64_t)G * j, A[j]);
          chi_store(chi, a, p, 1, (uint64_t)g + (uint64_t)G * j, B[j]);
        }
      } else {
        {
          tile_accumulate<A2>(acc, A, al);
          tile_accumulate<A2>(acc, B, al);
          if (hist) {
            spec_add(shist, A);
            spec_add(shist, B);
          }
        }
      }
    }
    if constexpr (!DEBUG) {
      if (alist) {                     // per-item reduction over the G lanes (all lanes take part)
#pragma unroll
        for (int i = 0; i < NACC; ++i) {
          double x = acc[i];
#pragma unroll
          for (int m = 1; m < G; m <<= 1) x += __shfl_xor_sync(0xffffffffu, x, m, G);
          if (valid && g == 0) partial[(size_t)item * NACC + i] = x;
          acc[i] = 0.0;
        }
      }
    }
  }
  if constexpr (!DEBUG) {
    if (!alist) block_flush(acc, partial, blockIdx.y * gridDim.x + blockIdx.x);
  }
  if (hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < SPEC_BINS; i += blockDim.x)
      if (shist[i]) atomicAdd(hist + i, shist[i]);
  }
}

// ------------------------------------------------------------------------------------------
// k_mid: 11 <= T = N-1 <= 13.  A unit of NT = 2^(T-5) threads owns one X-string: 32 values of
// each plane per thread, smem 2 * 2^T doubles per unit.  CTA = 256 threads.
// ------------------------------------------------------------------------------------------
template <int T, class V>
__device__ __forceinline__ void unit_gen(const typename Cx<V>::T* __restrict__ psi, uint64_t ybase, uint64_t a, int p,
                                         int N, uint32_t t, V (&v)[2][32]) {
  constexpr int NT = 1 << (T - 5);
#pragma unroll
  for (int j = 0; j < 32; ++j) gen_pair<V>(psi, ybase + t + (uint64_t)NT * j, a, p, N, v[0][j], v[1][j]);
}

template <int T, class F>
__device__ __forceinline__ void with_unit_bar(F&& f) {
  constexpr int NT = 1 << (T - 5);
  if constexpr (NT == 32) f(BarWarp{});
  else f(BarNamed{1 + (int)(threadIdx.x / NT), NT});
}

template <int T, bool A2, bool DEBUG, class V = double>
__global__ void __launch_bounds__(256, 1) k_mid(const typename Cx<V>::T* __restrict__ psi_all, int N, uint64_t a0,
                                                uint64_t count, Alphas al, double* partial, double* chi,
                                                const uint64_t* __restrict__ alist, unsigned long long* hist) {
  ln_table_init(!A2 && al.need_log && std::is_same<V, double>::value);   // t ln t pass (tile_accumulate)
  __shared__ unsigned long long shist[SPEC_BINS];   // hist != nullptr: spectrum epilogue
  if (hist) {
    for (int i = threadIdx.x; i < SPEC_BINS; i += blockDim.x) shist[i] = 0ull;
    __syncthreads();
  }
  // alist != nullptr: list mode, as in k_small (per-item sums reduced over the unit).
  constexpr int NT = 1 << (T - 5);
  constexpr int UPC = 256 / NT;
  extern __shared__ double smem[];
  const typename Cx<V>::T* psi = psi_all + ((size_t)blockIdx.y << N);
  const uint32_t t = threadIdx.x & (NT - 1);
  const int unit = threadIdx.x / NT;
  V* sm = reinterpret_cast<V*>(smem + (size_t)unit * 2 * padded(1 << T));
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
  __shared__ double lred[8][NACC];   // list mode: per-warp partials of the unit's reduction
  for (uint64_t item = (uint64_t)blockIdx.x * UPC + unit; item < count; item += (uint64_t)gridDim.x * UPC) {
    const uint64_t a = alist ? alist[item] : a0 + item;
    const int p = pivot_of(a, N);
    V v[2][32];
    unit_gen<T, V>(psi, 0, a, p, N, t, v);
    with_unit_bar<T>([&](const auto& bar) { Rounds<T, 0, 0, 2, std::decay_t<decltype(bar)>, false, V>::run(v, sm, t, bar); });
    if constexpr (DEBUG) {
      constexpr int sf = final_s<T, 0>();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        chi_store(chi, a, p, 0, lay(t, j, sf), v[0][j]);
        chi_store(chi, a, p, 1, lay(t, j, sf), v[1][j]);
      }
    } else {
      tile_accumulate<A2>(acc, v[0], al);
      tile_accumulate<A2>(acc, v[1], al);
      if (hist) {
        spec_add(shist, v[0]);
        spec_add(shist, v[1]);
      }
      if (alist) {                     // per-item reduction over the unit's NT / 32 warps
        const int w = threadIdx.x >> 5;
#pragma unroll
        for (int i = 0; i < NACC; ++i) {
          double x = acc[i];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
          if ((threadIdx.x & 31) == 0) lred[w][i] = x;
          acc[i] = 0.0;
        }
        with_unit_bar<T>([&](const auto& bar) { bar.sync(); });
        if (t == 0) {
          const int w0 = unit * (NT / 32);
#pragma unroll
          for (int i = 0; i < NACC; ++i) {
            double x = 0.0;
            for (int k = 0; k < NT / 32; ++k) x += lred[w0 + k][i];
            partial[(size_t)item * NACC + i] = x;
          }
        }
      }
    }
  }
  if constexpr (!DEBUG) {
    if (!alist) block_flush(acc, partial, blockIdx.y * gridDim.x + blockIdx.x);
  }
  if (hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < SPEC_BINS; i += blockDim.x)
      if (shist[i]) atomicAdd(hist + i, shist[i]);
  }
}

// ------------------------------------------------------------------------------------------
// Two-pass path, T = N-1 >= 14 = L + H.  Workspace per X-string: planes [2][2^H][2^L] doubles.
// Pass A: a unit (NT = 2^(L-5) threads) generates one row y_h of both planes and transforms
// the L low bits; writes row positions pos = t + NT*j (position pos holds b_l = lay(t,j,sL)).
// ------------------------------------------------------------------------------------------
template <int L, class V = double>
__global__ void __launch_bounds__(256, 1) k_passA(const typename Cx<V>::T* __restrict__ psi, int N, uint64_t a0,
                                                  int kcount, V* __restrict__ ws) {
  constexpr int NT = 1 << (L - 5);
  constexpr int UPC = 256 / NT;
  extern __shared__ double smem[];
  const int H = N - 1 - L;
  const uint32_t t = threadIdx.x & (NT - 1);
  const int unit = threadIdx.x / NT;
  V* sm = reinterpret_cast<V*>(smem + (size_t)unit * 2 * padded(1 << L));
  // item = y_h * kcount + k: the X-strings of the batch (which share a_h) take the same psi rows
  // at the same time, so each row pair comes from HBM once per batch and from L2 otherwise
  const uint64_t item = (uint64_t)blockIdx.x * UPC + unit;
  const uint64_t rows = 1ull << H;
  if (item >= (uint64_t)kcount * rows) return;  // whole units only; bars are per unit
  const int k = (int)(item % (uint64_t)kcount);
  const uint64_t yh = item / (uint64_t)kcount;
  const uint64_t a = a0 + (uint64_t)k;
  const int p = pivot_of(a, N);
  V v[2][32];
  unit_gen<L, V>(psi, yh << L, a, p, N, t, v);
  with_unit_bar<L>([&](const auto& bar) { Rounds<L, 0, 0, 2, std::decay_t<decltype(bar)>, false, V>::run(v, sm, t, bar); });
  const size_t plane = (size_t)1 << (N - 1);
  V* w0 = ws + (size_t)k * 2 * plane + (yh << L) + t;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    __stcg(w0 + (size_t)NT * j, v[0][j]);
    __stcg(w0 + plane + (size_t)NT * j, v[1][j]);
  }
}

// Pass B: a unit (NT = 2^(TP-5) threads, TP = CB + H) reads a slab of C = 2^CB columns x 2^H
// rows of one plane, transforms the H row bits, and accumulates the epilogue.
template <int TP, int CB, bool A2, bool DEBUG, class V = double>
__global__ void __launch_bounds__(TP >= 14 ? 512 : 256, 1) k_passB(int N, int L, uint64_t a0, int kcount,
                                                                   const V* __restrict__ ws, Alphas al,
                                                                   double* partial, double* chi) {
  ln_table_init(!A2 && al.need_log && std::is_same<V, double>::value);   // t ln t pass (tile_accumulate)
  __shared__ unsigned long long shist[SPEC_BINS];
  if (al.hist) {
    for (int i = threadIdx.x; i < SPEC_BINS; i += blockDim.x) shist[i] = 0ull;
    __syncthreads();
  }
  constexpr int NT = 1 << (TP - 5);
  constexpr int BLK = TP >= 14 ? 512 : 256;
  constexpr int UPC = BLK / NT;
  constexpr int H = TP - CB;
  extern __shared__ double smem[];
  const uint32_t t = threadIdx.x & (NT - 1);
  const int unit = threadIdx.x / NT;
  V* sm = reinterpret_cast<V*>(smem + (size_t)unit * padded(1 << TP));
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
  const uint64_t slabs = 1ull << (L - CB);  // per plane
  const uint64_t item = (uint64_t)blockIdx.x * UPC + unit;  // item = (k*2 + plane) * slabs + slab
  if (item < (uint64_t)kcount * 2 * slabs) {
    const uint64_t kp = item / slabs, slab = item % slabs;
    const size_t plane_sz = (size_t)1 << (N - 1);
    const V* src = ws + kp * plane_sz + (slab << CB);
    V v[1][32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint32_t e = t + (uint32_t)NT * j;  // round-0 layout
      v[0][j] = __ldcg(src + ((size_t)(e >> CB) << L) + (e & ((1u << CB) - 1u)));
    }
    with_unit_bar<TP>([&](const auto& bar) { Rounds<TP, CB, 0, 1, std::decay_t<decltype(bar)>, false, V>::run(v, sm, t, bar); });
    if constexpr (DEBUG) {
      const uint64_t a = a0 + kp / 2;
      const int p = pivot_of(a, N);
      const int pl = (int)(kp & 1);
      constexpr int sf = final_s<TP, CB>();
      const int ntA = 1 << (L - 5);
      const int sA = L == 10 ? final_s<10, 0>() : L == 11 ? final_s<11, 0>() : L == 12 ? final_s<12, 0>() : final_s<13, 0>();
      for (int j = 0; j < 32; ++j) {
        const uint32_t e = lay(t, j, sf);
        const uint64_t bh = e >> CB;
        const uint32_t pos = (uint32_t)(slab << CB) + (e & ((1u << CB) - 1u));
        const uint64_t bl = lay(pos & (ntA - 1), pos / ntA, sA);
        chi_store(chi, a, p, pl, (bh << L) | bl, v[0][j]);
      }
    } else {
      tile_accumulate<A2>(acc, v[0], al);
      if constexpr (!DEBUG && std::is_same<V, double>::value) {
        if (al.hist) spec_add(shist, v[0]);
      }
    }
  }
  (void)H;
  if constexpr (!DEBUG) block_flush(acc, partial, blockIdx.x);
  if (al.hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < SPEC_BINS; i += blockDim.x)
      if (shist[i]) atomicAdd(al.hist + i, shist[i]);
  }
}

// ------------------------------------------------------------------------------------------
// Staged pass A for L = 10 (N = 15..20): a persistent CTA of 8 warps walks the rows y_h of a
// group of up to 8 X-strings that share a_h = a >> 10 (hence the pivot p >= 10 and the two
// psi rows x_h = ins0(y_h, p-10), x_h ^ a_h).  The two rows (2 x 16 KB) are staged in shared
// memory with cp.async, double-buffered one row ahead; warp w generates X-string a0 + w from
// the staged rows (q = row[y_l], r = partner_row[y_l ^ a_l]), transforms 10 bits with one
// warp-local exchange, and writes its row of both planes.  Items = (group, row).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory"); }

// mbarrier / bulk-copy (TMA) helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred P;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}

// k_midr: k_mid for T = 13 (N = 14; one 256-thread unit per CTA) with the generation fed by a
// bulk-copy ring instead of L1/L2 gathers (k_mid is latency-bound on them: long_scoreboard).  For
// a >= 512 the pivot p >= 9, so the 512 positions y of stage s map to the contiguous x block
// ins0(512 s, p) + [0, 512), and x ^ a to the block (x_0 ^ (a & ~511)) + (i ^ (a & 511)): one
// 2 x 512-complex stage per 512 positions, 16 stages per X-string, in an MR_NS-deep ring refilled
// by the last of the 8 warps to leave a slot.  Thread t takes positions t + 256 e (e = 0, 1) of each
// stage, i.e. k_mid's register j = 2 s + e.  The CTA's X-strings with a < 512 (a prefix, since a
// grows with the item index) keep k_mid's global-load generation.
constexpr int MR_NS = 4;
template <int T, bool A2, class V = double>
__global__ void __launch_bounds__(256, 1) k_midr(const typename Cx<V>::T* __restrict__ psi_all, int N, uint64_t a0,
                                                 uint64_t count, Alphas al, double* partial, unsigned long long* hist) {
  static_assert(T == 13, "k_midr: one 256-thread unit per CTA");
  using C2 = typename Cx<V>::T;
  ln_table_init(!A2 && al.need_log && std::is_same<V, double>::value);   // t ln t pass (tile_accumulate)
  __shared__ unsigned long long shist[SPEC_BINS];
  __shared__ __align__(8) uint64_t full[MR_NS];
  __shared__ int used[MR_NS];
  if (hist)
    for (int i = threadIdx.x; i < SPEC_BINS; i += blockDim.x) shist[i] = 0ull;
  constexpr int SPI = (1 << T) / 512;                                  // stages per X-string
  extern __shared__ __align__(128) double smem[];
  V* sm = reinterpret_cast<V*>(smem);
  C2* ring = reinterpret_cast<C2*>(smem + 2 * padded(1 << T));        // [NS][q 512 | r 512]
  const typename Cx<V>::T* psi = psi_all + ((size_t)blockIdx.y << N);
  const uint32_t t = threadIdx.x, lane = t & 31;
  const uint64_t gx = gridDim.x;
  const uint64_t my_items = count > blockIdx.x ? (count - 1 - blockIdx.x) / gx + 1 : 0;
  const uint64_t first = a0 + blockIdx.x;                             // a of item n = first + n gx
  const uint64_t n0 = first >= 512 ? 0 : (512 - first + gx - 1) / gx;
  const uint64_t stages = my_items > n0 ? (my_items - n0) * SPI : 0;
  auto produce = [&](uint64_t s, int slot) {                          // one thread
    const uint64_t a = first + (n0 + s / SPI) * gx;
    const int p = 63 - __clzll((long long)a);
    const uint64_t x0 = ins0(512 * (s % SPI), p);
    C2* dst = ring + (size_t)slot * 1024;
    mbar_expect_tx(&full[slot], 2 * 512 * sizeof(C2));
    bulk_g2s(dst, psi + x0, 512 * sizeof(C2), &full[slot]);
    bulk_g2s(dst + 512, psi + (x0 ^ (a & ~511ull)), 512 * sizeof(C2), &full[slot]);
  };
  if (t == 0) {
    for (int i = 0; i < MR_NS; ++i) { mbar_init(&full[i], 1); used[i] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int i = 0; i < MR_NS; ++i)
      if ((uint64_t)i < stages) produce(i, i);
  }
  __syncthreads();
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
  uint64_t s = 0;
  for (uint64_t n = 0; n < my_items; ++n) {
    const uint64_t a = first + n * gx;
    const int p = pivot_of(a, N);
    V v[2][32];
    if (n < n0) {
      unit_gen<T, V>(psi, 0, a, p, N, t, v);
    } else {
      const uint32_t alo = (uint32_t)(a & 511u);
#pragma unroll
      for (int c = 0; c < SPI; ++c, ++s) {
        const int slot = (int)(s % MR_NS);
        mbar_wait(&full[slot], (uint32_t)(s / MR_NS) & 1u);
        const C2* cq = ring + (size_t)slot * 1024;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint32_t i = t + 256u * e;
          const C2 q = cq[i];
          const C2 r = cq[512 + (i ^ alo)];
          v[0][2 * c + e] = fma(r.x, q.x, r.y * q.y);                  // Re conj(psi_{x^a}) psi_x
          v[1][2 * c + e] = fma(r.x, q.y, -(r.y * q.x));               // Im
        }
        __syncwarp();
        if (lane == 0 && atomicAdd(&used[slot], 1) == 7) {             // the last warp refills the slot
          atomicExch(&used[slot], 0);
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          if (s + MR_NS < stages) produce(s + MR_NS, slot);
        }
      }
    }
    Rounds<T, 0, 0, 2, BarNamed, false, V>::run(v, sm, t, BarNamed{1, 256});
    tile_accumulate<A2>(acc, v[0], al);
    tile_accumulate<A2>(acc, v[1], al);
    if (hist) {
      spec_add(shist, v[0]);
      spec_add(shist, v[1]);
    }
  }
  block_flush(acc, partial, blockIdx.y * gridDim.x + blockIdx.x);
  if (hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < SPEC_BINS; i += blockDim.x)
      if (shist[i]) atomicAdd(hist + i, shist[i]);
  }
}

// ------------------------------------------------------------------------------------------
// Tensor memory (TMEM) as a per-thread register extension.  Thread lane of warp w owns TMEM
// lane 32 (w % 4) + lane; a double occupies two consecutive 32-bit columns.  tcgen05.ld/st
// run on the tensor-memory datapath, not on the L1TEX data pipe the transposes saturate.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {   // one full warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
               ::"r"(smem_u32(dst_smem)), "r"(ncols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {      // same warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
// 8 doubles -> columns [ta, ta + 16) of this thread's lane
__device__ __forceinline__ void tmem_st8d(uint32_t ta, const double (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%16], {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15};\n"
               ::"r"(__double2loint(v[0])), "r"(__double2hiint(v[0])), "r"(__double2loint(v[1])), "r"(__double2hiint(v[1])),
                 "r"(__double2loint(v[2])), "r"(__double2hiint(v[2])), "r"(__double2loint(v[3])), "r"(__double2hiint(v[3])),
                 "r"(__double2loint(v[4])), "r"(__double2hiint(v[4])), "r"(__double2loint(v[5])), "r"(__double2hiint(v[5])),
                 "r"(__double2loint(v[6])), "r"(__double2hiint(v[6])), "r"(__double2loint(v[7])), "r"(__double2hiint(v[7])),
                 "r"(ta) : "memory");
}
// columns [ta, ta + 16) -> 8 doubles (no wait: the caller issues tmem_wait_ld before use)
__device__ __forceinline__ void tmem_ld8d(uint32_t ta, uint32_t (&u)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
                 "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
               : "r"(ta) : "memory");
}
__device__ __forceinline__ void stg_v4(double* p, double a, double b, double c, double d) {   // one 32-B sector
  asm volatile("st.global.cg.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// ------------------------------------------------------------------------------------------
// Warp-local 10-bit transform of two 1024-point planes with the transposes in TMEM (k_passA10s, FP64).
// Start: lane l, register j holds element e = l + 32 j.  Round 0 butterflies e bits 5..9.  A "trip"
// stores the 32 doubles with tcgen05.st 32x32b (lane l, double column j) and reads them back with two
// tcgen05.ld 16x256b.x8 (lane bases 0, 16): thread t = t0 + 4 t1 receives lane 16b + 8s + t1, double
// column 4c + t0 into register r = s + 2c + 16b (CUTLASS Copy_Traits<SM100_TMEM_LOAD_16dp256b1x>).
// Each trip brings two new element bits into the register index (tools/microbench_tmem_transpose.cu
// verifies the map on B200): trip 1 -> e3 (r0), e4 (r4); trip 2 -> e1 (r0), e2 (r4); trip 3 -> e0 (r4).
// After trip 3, (lane t, register r) holds frequency pa10_freq(t + 32 r).  The TMEM datapath runs
// beside the L1TEX pipe the generation loads and stores saturate (microbenchmark: a transpose split
// between the two costs 0.075 clk/value vs 0.126 for shared memory alone).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pa10_freq(uint32_t pos) {
  const uint32_t t = pos & 31u, r = pos >> 5;
  return ((t & 1u) << 1) | (((t >> 1) & 1u) << 8) | (((t >> 2) & 1u) << 3) | (((t >> 3) & 1u) << 7) |
         (((t >> 4) & 1u) << 5) | ((r & 1u) << 6) | (((r >> 1) & 1u) << 9) | (((r >> 2) & 1u) << 4) |
         (((r >> 3) & 1u) << 2) | ((r >> 4) & 1u);
}
// k_passA10s<ROWM> stores (lane t, register r) at position 2 t + (r & 1) + 64 (r >> 1)
__device__ __forceinline__ uint32_t pa10_freq_rowm(uint32_t pos) {
  const uint32_t t = (pos >> 1) & 31u, r = (pos & 1u) | ((pos >> 6) << 1);
  return pa10_freq(t + 32u * r);
}
__device__ __forceinline__ void tmem_st32d(uint32_t ta, const double (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x64.b32 [%64], {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63};\n"
               ::"r"(__double2loint(v[0])), "r"(__double2hiint(v[0])), "r"(__double2loint(v[1])), "r"(__double2hiint(v[1])), "r"(__double2loint(v[2])), "r"(__double2hiint(v[2])), "r"(__double2loint(v[3])), "r"(__double2hiint(v[3])),
                 "r"(__double2loint(v[4])), "r"(__double2hiint(v[4])), "r"(__double2loint(v[5])), "r"(__double2hiint(v[5])), "r"(__double2loint(v[6])), "r"(__double2hiint(v[6])), "r"(__double2loint(v[7])), "r"(__double2hiint(v[7])),
                 "r"(__double2loint(v[8])), "r"(__double2hiint(v[8])), "r"(__double2loint(v[9])), "r"(__double2hiint(v[9])), "r"(__double2loint(v[10])), "r"(__double2hiint(v[10])), "r"(__double2loint(v[11])), "r"(__double2hiint(v[11])),
                 "r"(__double2loint(v[12])), "r"(__double2hiint(v[12])), "r"(__double2loint(v[13])), "r"(__double2hiint(v[13])), "r"(__double2loint(v[14])), "r"(__double2hiint(v[14])), "r"(__double2loint(v[15])), "r"(__double2hiint(v[15])),
                 "r"(__double2loint(v[16])), "r"(__double2hiint(v[16])), "r"(__double2loint(v[17])), "r"(__double2hiint(v[17])), "r"(__double2loint(v[18])), "r"(__double2hiint(v[18])), "r"(__double2loint(v[19])), "r"(__double2hiint(v[19])),
                 "r"(__double2loint(v[20])), "r"(__double2hiint(v[20])), "r"(__double2loint(v[21])), "r"(__double2hiint(v[21])), "r"(__double2loint(v[22])), "r"(__double2hiint(v[22])), "r"(__double2loint(v[23])), "r"(__double2hiint(v[23])),
                 "r"(__double2loint(v[24])), "r"(__double2hiint(v[24])), "r"(__double2loint(v[25])), "r"(__double2hiint(v[25])), "r"(__double2loint(v[26])), "r"(__double2hiint(v[26])), "r"(__double2loint(v[27])), "r"(__double2hiint(v[27])),
                 "r"(__double2loint(v[28])), "r"(__double2hiint(v[28])), "r"(__double2loint(v[29])), "r"(__double2hiint(v[29])), "r"(__double2loint(v[30])), "r"(__double2hiint(v[30])), "r"(__double2loint(v[31])), "r"(__double2hiint(v[31])),
                 "r"(ta) : "memory");
}
__device__ __forceinline__ void tmem_ld16x256(uint32_t ta, double* v) {     // 16 doubles, no wait
  uint32_t u[32];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15]),
                 "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
               : "r"(ta) : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __hiloint2double(u[2 * i + 1], u[2 * i]);
}
template <int B>
__device__ __forceinline__ void bfly_bit(double (&v)[32]) { bfly32<B, B + 1>(v); }
__device__ __forceinline__ void tmem_ld_plane(uint32_t ta, double (&v)[32]) {
  tmem_ld16x256(ta, v);
  tmem_ld16x256(ta + (16u << 16), v + 16);
}
// The two planes' trips are interleaved so that one plane's butterflies run while the other plane's
// tcgen05.st/ld are in flight (the waits cover every outstanding op of the thread):
//   st A1 st B1 | wait.st | ld A1 ld B1 | wait.ld | bfly A, st A2 | bfly B, st B2 | wait.st | ...
__device__ __forceinline__ void transform10_tmem(uint32_t tm, double (&v)[2][32]) {
  bfly32<0, 5>(v[0]);                                     // e bits 5..9
  tmem_st32d(tm, v[0]);
  bfly32<0, 5>(v[1]);
  tmem_st32d(tm + 64u, v[1]);
  tmem_wait_st();
  tmem_ld_plane(tm, v[0]);
  tmem_ld_plane(tm + 64u, v[1]);
  tmem_wait_ld();
  bfly_bit<0>(v[0]); bfly_bit<4>(v[0]);                   // e3, e4
  tmem_st32d(tm, v[0]);
  bfly_bit<0>(v[1]); bfly_bit<4>(v[1]);
  tmem_st32d(tm + 64u, v[1]);
  tmem_wait_st();
  tmem_ld_plane(tm, v[0]);
  tmem_ld_plane(tm + 64u, v[1]);
  tmem_wait_ld();
  bfly_bit<0>(v[0]); bfly_bit<4>(v[0]);                   // e1, e2
  tmem_st32d(tm, v[0]);
  bfly_bit<0>(v[1]); bfly_bit<4>(v[1]);
  tmem_st32d(tm + 64u, v[1]);
  tmem_wait_st();
  tmem_ld_plane(tm, v[0]);
  tmem_ld_plane(tm + 64u, v[1]);
  tmem_wait_ld();
  bfly_bit<4>(v[0]); bfly_bit<4>(v[1]);                   // e0
}

constexpr int PA10_NS = 4;                                   // staging ring depth (6 measured no better at N = 20)
constexpr int PA10_SMEM = PA10_NS * 2 * 1024 * 16 + 8 * padded(1024) * 8;  // 128 KB ring + 66 KB exchange

// Staged pass A for L = 10 (N = 15..20).  A persistent CTA of 8 warps walks items
// (group g of 8 X-strings sharing a_h != 0, row y_h).  The two psi rows an item needs
// (x_h = ins0(y_h, p-10) and x_h ^ a_h, 16 KB each) arrive by two bulk copies into a 4-deep
// ring completed on an mbarrier; warps run free (no CTA barrier): the last of the 8 warps to
// finish with a ring slot refills it with the item NS positions ahead.  Warp w generates
// X-string 8g + w from the staged rows, transforms 10 bits (one warp-local exchange per
// plane) and writes its row of both planes.
// ROWM: row-major planes [2^H][1024] (FP64, k_passBw)
template <int N, class V = double, bool ROWM = false>
__global__ void __launch_bounds__(256, 1) k_passA10s(const typename Cx<V>::T* __restrict__ psi, uint64_t a_first,
                                                     int kcount, int groups, V* __restrict__ ws) {
  using C2 = typename Cx<V>::T;
  // slab-major pass-B tiles of 2^12 values for k_passBt (N = 15, 16 and the FP32 mode); FP64 N >= 17
  // writes row-major planes (ROWM) for the TMA-gather k_passBw
  constexpr int cb = 12 - (N - 11);
  extern __shared__ __align__(128) double smem[];
  C2* ring = reinterpret_cast<C2*>(smem);                       // [NS][q row | r row][1024]
  V* exch = reinterpret_cast<V*>(smem + PA10_NS * 2 * 1024 * 2);   // [warp][padded 1024]
  __shared__ __align__(8) uint64_t full[PA10_NS];
  __shared__ int used[PA10_NS];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int H = N - 11;
  constexpr uint64_t rows = 1ull << H;
  const uint64_t items = rows * (uint64_t)groups;
  constexpr size_t plane = (size_t)1 << (N - 1);
  auto issue = [&](uint64_t item, int slot) {                  // one thread
    const uint64_t g = item >> H, yh = item & (rows - 1);
    const uint64_t ag = a_first + 8 * g;
    const int p = 63 - __clzll((long long)ag);
    const uint64_t xh = ins0(yh, p - 10);
    C2* dst = ring + (size_t)slot * 2048;
    mbar_expect_tx(&full[slot], 2 * 1024 * sizeof(C2));
    bulk_g2s(dst, psi + (xh << 10), 1024 * sizeof(C2), &full[slot]);
    bulk_g2s(dst + 1024, psi + ((xh ^ (ag >> 10)) << 10), 1024 * sizeof(C2), &full[slot]);
  };
  constexpr bool TM = std::is_same<V, double>::value;           // FP64: transposes through TMEM
  __shared__ uint32_t tmem_s;
  if (TM && w == 0) tmem_alloc(&tmem_s, 256);
  if (threadIdx.x == 32) {
    for (int i = 0; i < PA10_NS; ++i) { mbar_init(&full[i], 1); used[i] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (TM) tmem_fence_before();
  __syncthreads();
  if (TM) tmem_fence_after();
  // this warp's TMEM slice: its lane quadrant, double columns [0, 64) for w < 4, [64, 128) for w >= 4
  const uint32_t tm = TM ? tmem_s + ((uint32_t)(32 * (w & 3)) << 16) + 128u * (uint32_t)(w >> 2) : 0u;
  if (threadIdx.x == 0)
    for (int i = 0; i < PA10_NS; ++i)
      if (blockIdx.x + (uint64_t)i * gridDim.x < items) issue(blockIdx.x + (uint64_t)i * gridDim.x, i);
  V* xw = exch + (size_t)w * padded(1024);
  uint32_t n = 0;
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x, ++n) {
    const int slot = (int)(n % PA10_NS);
    mbar_wait(&full[slot], (n / PA10_NS) & 1u);
    const uint64_t g = item >> H, yh = item & (rows - 1);
    const int k = 8 * (int)g + w;
    const C2* sq = ring + (size_t)slot * 2048;
    V v[2][32];
    const bool active = k < kcount;
    if (active) {
      const uint32_t al = (uint32_t)((a_first + (uint64_t)k) & 1023u);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const uint32_t yl = lane + 32 * j;
        const C2 q = sq[yl];
        const C2 r = sq[1024 + (yl ^ al)];
        v[0][j] = fma(r.x, q.x, r.y * q.y);
        v[1][j] = fma(r.x, q.y, -(r.y * q.x));
      }
    }
    __syncwarp();
    if (lane == 0) {                                             // release the slot; last warp refills
      const int prev = atomicAdd(&used[slot], 1);
      if (prev == 7) {
        atomicExch(&used[slot], 0);
        const uint64_t nx = item + (uint64_t)PA10_NS * gridDim.x;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        if (nx < items) issue(nx, slot);
      }
    }
    if (active) {
      if constexpr (TM) transform10_tmem(tm, v);              // position lane + 32 j <- pa10_freq
      else Rounds<10, 0, 0, 2, BarWarp, true, V>::run(v, xw, lane, BarWarp{});
      if constexpr (ROWM) {   // row-major: 8 KB per row; registers (2 i, 2 i + 1) of lane l go to positions
        // 64 i + 2 l + {0, 1} as one 16-B store (512 contiguous bytes per warp instruction)
        V* w0 = ws + (size_t)k * 2 * plane + (yh << 10) + 2 * lane;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          __stcg(reinterpret_cast<double2*>(w0 + 64 * i), make_double2(v[0][2 * i], v[0][2 * i + 1]));
          __stcg(reinterpret_cast<double2*>(w0 + plane + 64 * i), make_double2(v[1][2 * i], v[1][2 * i + 1]));
        }
        continue;
      }
      // slab-major workspace: (y_h, pos) -> ((pos >> cb) << (H + cb)) | (y_h << cb) | (pos & (C-1))
      V* w0 = ws + (size_t)k * 2 * plane + (yh << cb);
      constexpr uint32_t cm = (1u << cb) - 1u;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const uint32_t pos = lane + 32 * j;
        const size_t off = ((size_t)(pos >> cb) << (H + cb)) + (pos & cm);   // compile-time in j
        __stcg(w0 + off, v[0][j]);
        __stcg(w0 + plane + off, v[1][j]);
      }
    }
  }
  if constexpr (TM) {
    tmem_fence_before();
    __syncthreads();
    if (w == 0) tmem_dealloc(tmem_s, 256);
  }
}

// Pass B over the slab-major workspace written by k_passA10s: a tile (X-string k, plane, slab)
// is one contiguous block of 2^TP doubles (2^H rows x C = 2^CB columns).  A CTA holds two
// independent 128-thread units (TP = 12); each streams its tiles through a 3-deep ring of bulk
// copies completed on mbarriers, reads the tile in the round-0 layout, and uses the same slot
// for its shared-memory exchange before handing it back to the copy engine.
constexpr int PBT_NS = 3;
__host__ __device__ constexpr int pbt_slot(int TP) { return padded(1 << TP); }         // tile + exchange padding
__host__ __device__ constexpr int pbt_smem(int TP) { return PBT_NS * 256 / (1 << (TP - 5)) * pbt_slot(TP) * 8; }

template <int TP, int CB, bool A2, class V = double>   // TP = 12: two 128-thread units; 13: one 256-thread unit
__global__ void __launch_bounds__(256, 1) k_passBt(int N, int kcount, const V* __restrict__ ws, Alphas al,
                                                   double* partial) {
  ln_table_init(!A2 && al.need_log && std::is_same<V, double>::value);   // t ln t pass (tile_accumulate)
  constexpr int NT = 1 << (TP - 5), UNITS = 256 / NT, TILE = 1 << TP, SLOT = pbt_slot(TP);
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[UNITS][PBT_NS];
  const int unit = threadIdx.x / NT;
  const uint32_t t = threadIdx.x % NT;
  const int L = N - 1 - (TP - CB);
  const uint64_t slabs = 1ull << (L - CB);
  const uint64_t tiles = (uint64_t)kcount * 2 * slabs;   // tile = kp * slabs + slab, contiguous blocks
  V* ring = reinterpret_cast<V*>(smem + (size_t)unit * PBT_NS * SLOT);   // slots of SLOT doubles
  const BarNamed bar{1 + unit, NT};
  if (threadIdx.x == 0) {
    for (int u = 0; u < UNITS; ++u)
      for (int i = 0; i < PBT_NS; ++i) mbar_init(&full[u][i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const uint64_t first = (uint64_t)blockIdx.x * UNITS + unit, step = (uint64_t)gridDim.x * UNITS;
  constexpr int SLOT_V = SLOT * (int)(sizeof(double) / sizeof(V));      // slot stride in V elements
  auto issue = [&](uint64_t tile, int slot) {
    mbar_expect_tx(&full[unit][slot], TILE * sizeof(V));
    bulk_g2s(ring + (size_t)slot * SLOT_V, ws + tile * TILE, TILE * sizeof(V), &full[unit][slot]);
  };
  if (t == 0)
    for (int i = 0; i < PBT_NS; ++i)
      if (first + i * step < tiles) issue(first + i * step, i);
  __shared__ unsigned long long shist[SPEC_BINS];   // al.hist: spectrum epilogue
  if (al.hist) {
    for (int i = threadIdx.x; i < SPEC_BINS; i += blockDim.x) shist[i] = 0ull;
    __syncthreads();
  }
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
  uint32_t n = 0;
  for (uint64_t tile = first; tile < tiles; tile += step, ++n) {
    const int slot = (int)(n % PBT_NS);
    V* buf = ring + (size_t)slot * SLOT_V;
    mbar_wait(&full[unit][slot], (n / PBT_NS) & 1u);
    V v[1][32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[0][j] = buf[t + NT * j];   // round-0 layout e = t + NT j
    Rounds<TP, CB, 0, 1, BarNamed, false, V>::run(v, buf, t, bar);
    bar.sync();                                                  // slot free: refill it
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      const uint64_t nx = tile + (uint64_t)PBT_NS * step;
      if (nx < tiles) issue(nx, slot);
    }
    tile_accumulate<A2>(acc, v[0], al);
    if constexpr (std::is_same<V, double>::value) {
      if (al.hist) spec_add(shist, v[0]);
      if (al.chi) {   // sre_chi: element (row, col) of tile (k, plane, slab) is the output b' = (row << L) | b_l
        constexpr int sf = final_s<TP, CB>();
        const int L = N - 1 - (TP - CB);
        const uint64_t kp = tile / slabs, slab = tile % slabs;
        const uint64_t a = al.chi_a0 + (kp >> 1);
        const int p = pivot_of(a, N);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const uint32_t e = lay(t, j, sf);
          const uint64_t pos = (slab << CB) | (e & ((1u << CB) - 1u));
          // k_passA10s (FP64, TMEM transposes) stores frequency pa10_freq(pos) at pos = lane + 32 j (N <= 20)
          const uint64_t bl = L == 10 ? pa10_freq((uint32_t)pos) : pos;
          chi_store(al.chi, a, p, (int)(kp & 1), ((uint64_t)(e >> CB) << L) | bl, v[0][j]);
        }
      }
    }
  }
  block_flush(acc, partial, blockIdx.x);
  if (al.hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < SPEC_BINS; i += blockDim.x)
      if (shist[i]) atomicAdd(al.hist + i, shist[i]);
  }
}

// ------------------------------------------------------------------------------------------
// Streamed pass A for L = 12, 13 (N = 21..25): persistent units of 2^(L-5) threads walk items
// (row y_h, X-string k) in row-major order, so the K X-strings of a launch read the same psi
// rows back to back (HBM once, L2 for the rest).  Generation operands stream as 32 chunks of
// 2^(L-5) y values (q chunk + r chunk, the r chunk index permuted by a_l >> (L-5)) through an
// 8-deep bulk-copy ring per unit; then three rounds (two unit-wide exchanges, one plane at a
// time) and a slab-major store for the TMA-fed pass B (tile = 2^13 doubles, CB = 13 - H).
// L = 12 runs two independent 128-thread units per CTA so one unit's exchange barriers overlap
// the other's arithmetic (L = 13's single CTA-wide unit measured barrier-bound).
// ------------------------------------------------------------------------------------------
constexpr int PAS_NS = 2;   // ring stages per unit
constexpr int PAS_JS = 8;   // j-blocks per stage: copies of 8 x 2^(L-5) complex (16 KB at L = 12)
__host__ __device__ constexpr int pas_smem(int L) {
  // per unit: ring of NS stages x (q | r) x JS*NT complex  +  one padded plane of 2^L doubles
  return (256 >> (L - 5)) * (PAS_NS * 2 * PAS_JS * (1 << (L - 5)) * 16 + padded(1 << L) * 8);
}

template <int N, int L, class V = double>
__global__ void __launch_bounds__(256, 1) k_passAs(const typename Cx<V>::T* __restrict__ psi, uint64_t a_first,
                                                   int kcount, V* __restrict__ ws) {
  using C2 = typename Cx<V>::T;
  constexpr int NT = 1 << (L - 5), UNITS = 256 / NT, WPU = NT / 32;   // threads, units, warps per unit
  constexpr int H = N - 1 - L, CB = 13 - H;                            // pass-B tile = 2^13 doubles
  constexpr int SPI = 32 / PAS_JS;                                     // stages per item
  constexpr int SD = PAS_JS * NT;                                      // complex per half-stage
  constexpr uint64_t ROWS = 1ull << H;
  constexpr size_t PLANE = (size_t)1 << (N - 1);
  constexpr int UNIT_D = PAS_NS * 2 * SD * 2 + padded(1 << L);        // doubles of smem per unit
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[UNITS][PAS_NS];
  __shared__ int used[UNITS][PAS_NS];
  const int u = threadIdx.x / NT;
  const uint32_t t = threadIdx.x % NT;
  const int lane = threadIdx.x & 31;
  C2* ring = reinterpret_cast<C2*>(smem + (size_t)u * UNIT_D);   // [NS][q | r][SD]
  V* exch = reinterpret_cast<V*>(smem + (size_t)u * UNIT_D + PAS_NS * 2 * SD * 2);
  const BarNamed bar{1 + u, NT};
  const uint64_t items = ROWS * (uint64_t)kcount;
  const uint64_t first = (uint64_t)blockIdx.x * UNITS + u, step = (uint64_t)gridDim.x * UNITS;
  const uint64_t my_items = items > first ? (items - 1 - first) / step + 1 : 0;
  const uint64_t stages = my_items * SPI;
  if (threadIdx.x == 0) {
    for (int x = 0; x < UNITS; ++x)
      for (int i = 0; i < PAS_NS; ++i) { mbar_init(&full[x][i], 1); used[x][i] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto produce = [&](uint64_t st, int slot) {                   // one thread of the unit
    const uint64_t item = first + (st / SPI) * step;
    const uint32_t g = (uint32_t)(st % SPI);                    // j-blocks [JS g, JS g + JS)
    const uint64_t yh = item / (uint64_t)kcount;
    const uint64_t a = a_first + item % (uint64_t)kcount;
    const int p = 63 - __clzll((long long)a);                   // >= L (a >= 2^L)
    const uint64_t xh = ins0(yh, p - L);
    const uint32_t ahi = (uint32_t)((a & ((1u << L) - 1u)) >> (L - 5));   // r block of block j is j ^ ahi
    C2* dst = ring + (size_t)slot * 2 * SD;
    mbar_expect_tx(&full[u][slot], 2 * SD * sizeof(C2));
    bulk_g2s(dst, psi + (xh << L) + (size_t)SD * g, SD * sizeof(C2), &full[u][slot]);
    // blocks {JS g + i} ^ ahi form the aligned group (g ^ (ahi / JS)) permuted by ahi % JS
    bulk_g2s(dst + SD, psi + ((xh ^ (a >> L)) << L) + (size_t)SD * (g ^ (ahi / PAS_JS)), SD * sizeof(C2), &full[u][slot]);
  };
  if (t == 0)
    for (int i = 0; i < PAS_NS; ++i)
      if ((uint64_t)i < stages) produce(i, i);
  uint64_t st = 0;
  for (uint64_t li = 0; li < my_items; ++li) {
    const uint64_t item = first + li * step;
    const uint64_t yh = item / (uint64_t)kcount;
    const int k = (int)(item % (uint64_t)kcount);
    const uint32_t al = (uint32_t)((a_first + (uint64_t)k) & ((1u << L) - 1u));
    const uint32_t alo = al & (NT - 1), ahl = (al >> (L - 5)) % PAS_JS;
    V v[2][32];
#pragma unroll
    for (int gi = 0; gi < SPI; ++gi, ++st) {
      const int slot = (int)(st % PAS_NS);
      mbar_wait(&full[u][slot], (uint32_t)(st / PAS_NS) & 1u);
      const C2* c = ring + (size_t)slot * 2 * SD;
#pragma unroll
      for (int i = 0; i < PAS_JS; ++i) {
        const int j = PAS_JS * gi + i;
        const C2 q = c[NT * i + t];
        const C2 r = c[SD + NT * (i ^ ahl) + (t ^ alo)];
        v[0][j] = fma(r.x, q.x, r.y * q.y);
        v[1][j] = fma(r.x, q.y, -(r.y * q.x));
      }
      __syncwarp();
      int last = 0;
      if (lane == 0) last = atomicAdd(&used[u][slot], 1) == WPU - 1;
      if (__shfl_sync(0xffffffffu, last, 0) && lane == 0) {
        atomicExch(&used[u][slot], 0);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        if (st + PAS_NS < stages) produce(st + PAS_NS, slot);
      }
    }
    Rounds<L, 0, 0, 2, BarNamed, true, V>::run(v, exch, t, bar);
    // position pos = t + NT j (round-0 layout) -> slab-major ((pos >> CB) << (H+CB)) + (y_h << CB) + (pos & (C-1))
    V* w0 = ws + (size_t)k * 2 * PLANE + (yh << CB);
    constexpr uint32_t cm = (1u << CB) - 1u;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint32_t pos = t + NT * j;
      const size_t off = ((size_t)(pos >> CB) << (H + CB)) + (pos & cm);
      __stcg(w0 + off, v[0][j]);
      __stcg(w0 + PLANE + off, v[1][j]);
    }
  }
}

// 64-point radix-2 butterflies over the register index (6 stages, pure DADD)
__device__ __forceinline__ void bfly64(double (&v)[64]) {
#pragma unroll
  for (int h = 1; h < 64; h <<= 1)
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      if (i & h) continue;
      const double a = v[i], b = v[i + h];
      v[i] = a + b;
      v[i + h] = a - b;
    }
}

__device__ __forceinline__ uint32_t xsw12(uint32_t e) { return e ^ ((e >> 6) & 15u); }   // radix-64 transpose swizzle

// Radix-64 pass B transpose (k_passBw): tile element e = row * 2^CB + col, 2^13 per tile; round-0
// registers e bits 7..12, round-1 registers e bits 1..6; physical e ^ (((e >> 7) & 7) << 1) is
// conflict-free for both layouts (tests/test_layouts.py)
constexpr int PBR_SMEM = 3 * 8192 * 8;
__device__ __forceinline__ uint32_t xsw13(uint32_t e) { return e ^ (((e >> 7) & 7u) << 1); }

// ------------------------------------------------------------------------------------------
// Row-major streamed path for N = 21..24 (FP64): k_passAw + k_passBw.
// Workspace plane (X-string k, plane p) is row-major [2^H rows][4096 positions]: pass A writes each
// 32 KB row contiguously (coalesced 16-B stores: HBM takes contiguous writes at ~6.3 TB/s against
// 3.3-3.7 TB/s for the 32-B runs a slab-major layout forces, tools/microbench_wr.cu), and pass B
// gathers a tile of 2^H rows x 2^CB columns with TMA tensor copies (32-B pieces at a 32 KB stride
// read at 5.2 TB/s vs 7.3 for contiguous tiles) into the smem layout of the radix-64 transform.
// ------------------------------------------------------------------------------------------
// k_passAw: CTA = 4 units x 64 threads; an item is (row y_h, group of 4 consecutive X-strings);
// unit u takes X-string 4g + u.  The 4 X-strings share a_h and a_l >> 9, hence both psi rows and
// every chunk: one ring of 16 KB stages (q chunk c, r chunk c ^ (a_l >> 9), 512 complex each) is
// read by all 8 warps.  Radix-64: a 4096-point row-plane is 64 threads x 64 values, two register
// rounds around ONE XOR-swizzled transpose (round 0: pos = t + 64 j, bits 6..11 in registers; round 1:
// pos = 64 t + j); plane B parked in TMEM (128 columns per thread).  After round 1 the
// unit stores its row with TMA (TS): the row-plane is the 64 x 64 matrix [t][j] (pos = 64 t + j), four
// tensor boxes of {16 doubles, 64 rows} with SWIZZLE_128B; thread t writes its pairs (v[j], v[j+1])
// as 16-B chunks at row t, chunk ((j & 15) >> 1) ^ (t & 7) of box j >> 4 (conflict-free per
// quarter-warp), and the TMA engine reads the 32 KB back from shared memory and writes whole 128-B
// lines -- no LDS/STG wavefronts on the L1TEX pipe.  !TS: natural-order staging in the XOR-swizzled
// buffer and coalesced 16-B stores (A/B measurements, SRE_PAW_TMA=0).
constexpr int PAW_NS = 6;                                             // ring stages (16 KB each)
constexpr int PAW_SMEM = PAW_NS * 2 * 512 * 16 + 4 * 4096 * 8 + 1024; // 96 KB ring + 4 x 32 KB buffers + alignment

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tmap, int c0, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n"
               ::"l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src)) : "memory");
}

template <int N, bool TS>
__global__ void __launch_bounds__(256, 1) k_passAw(const double2* __restrict__ psi, uint64_t a_first, int kcount,
                                                   uint64_t gmagic, double* __restrict__ ws,
                                                   const __grid_constant__ CUtensorMap tmw) {
  constexpr int L = 12, H = N - 1 - L;
  static_assert(H >= 8 && H <= 11, "k_passAw covers N = 21..24");
  constexpr uint64_t ROWS = 1ull << H;
  constexpr size_t PLANE = (size_t)1 << (N - 1);
  extern __shared__ __align__(128) double smem_raw[];
  double* smem = smem_raw + (((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) >> 3);   // SWIZZLE_128B: 1024-B aligned
  double2* ring = reinterpret_cast<double2*>(smem);                 // [NS][q 512 | r 512]
  double* exch = smem + PAW_NS * 2 * 512 * 2;                        // [unit][4096]
  __shared__ __align__(8) uint64_t full[PAW_NS];
  __shared__ int used[PAW_NS];
  __shared__ uint32_t tmem_s;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = w >> 1;
  const uint32_t t = threadIdx.x & 63;
  const uint64_t groups = (uint64_t)(kcount + 3) / 4;
  const uint64_t items = ROWS * groups;
  const uint64_t my_items = items > blockIdx.x ? (items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint64_t stages = my_items * 8;
  auto split = [&](uint64_t item, uint64_t& yh, uint64_t& g) {       // gmagic = ceil(2^40 / groups)
    yh = (item * gmagic) >> 40;
    g = item - yh * groups;
  };
  if (w == 0) tmem_alloc(&tmem_s, 256);
  if (threadIdx.x == 32) {
    for (int i = 0; i < PAW_NS; ++i) { mbar_init(&full[i], 1); used[i] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tm = tmem_s + ((uint32_t)(32 * (w & 3)) << 16) + 128u * (uint32_t)(w >> 2);
  auto produce = [&](uint64_t s, int slot) {                       // one thread
    uint64_t yh, g;
    split(blockIdx.x + (s >> 3) * gridDim.x, yh, g);
    const uint32_t c = (uint32_t)(s & 7);
    const uint64_t a = a_first + 4 * g;
    const int p = 63 - __clzll((long long)a);                       // >= 12
    const uint64_t xh = ins0(yh, p - L);
    const uint32_t ahi = (uint32_t)((a >> 9) & 7u);
    double2* dst = ring + (size_t)slot * 1024;
    mbar_expect_tx(&full[slot], 2 * 512 * sizeof(double2));
    bulk_g2s(dst, psi + (xh << L) + 512 * c, 512 * sizeof(double2), &full[slot]);
    bulk_g2s(dst + 512, psi + ((xh ^ (a >> L)) << L) + 512 * (c ^ ahi), 512 * sizeof(double2), &full[slot]);
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < PAW_NS; ++i)
      if ((uint64_t)i < stages) produce(i, i);
  double* xb = exch + (size_t)u * 4096;
  const BarNamed bar{1 + u, 64};
  uint64_t s = 0;
  for (uint64_t li = 0; li < my_items; ++li) {
    uint64_t yh, g;
    split(blockIdx.x + li * gridDim.x, yh, g);
    const int k = 4 * (int)g + u;
    const bool active = k < kcount;
    const uint32_t al = (uint32_t)((a_first + (uint64_t)k) & 4095u);
    const uint32_t alo = al & 63u, ajh = (al >> 6) & 7u;
    double v[64];
#pragma unroll
    for (int c = 0; c < 8; ++c, ++s) {
      const int slot = (int)(s % PAW_NS);
      mbar_wait(&full[slot], (uint32_t)(s / PAW_NS) & 1u);
      const double2* cq = ring + (size_t)slot * 1024;
      double b8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double2 q = cq[t + 64 * i];
        const double2 r = cq[512 + (t ^ alo) + 64 * (i ^ ajh)];
        v[8 * c + i] = fma(r.x, q.x, r.y * q.y);        // Re conj(psi_{x^a}) psi_x
        b8[i] = fma(r.x, q.y, -(r.y * q.x));            // Im
      }
      if (active) tmem_st8d(tm + 16u * c, b8);
      __syncwarp();
      if (lane == 0) {                                   // release the stage; the 8th warp refills it
        if (atomicAdd(&used[slot], 1) == 7) {
          atomicExch(&used[slot], 0);
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          if (s + PAW_NS < stages) produce(s + PAW_NS, slot);
        }
      }
    }
    if (!active) continue;
    tmem_wait_st();
    double* wrow = ws + ((size_t)k * 2 << (N - 1)) + (yh << L);
    auto transform_store = [&](double* wp, int p) {
      bfly64(v);                                         // round 0: pos bits 6..11
      if constexpr (TS)
        if (t == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");   // last TMA store read xb
      bar.sync();                                        // previous readers of xb are done
#pragma unroll
      for (int j = 0; j < 64; ++j) xb[xsw12(t + 64u * j)] = v[j];
      bar.sync();
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] = xb[xsw12(64u * t + j)];
      bar.sync();                                        // the transpose reads are done: reuse xb
      bfly64(v);                                         // round 1: pos bits 0..5 (pos = 64 t + j)
      if constexpr (TS) {
#pragma unroll
        for (int j = 0; j < 64; j += 2) {
          const uint32_t chunk = (((uint32_t)j & 15u) >> 1) ^ (t & 7u);
          *reinterpret_cast<double2*>(xb + 1024u * (uint32_t)(j >> 4) + 16u * t + 2u * chunk) = make_double2(v[j], v[j + 1]);
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic writes -> TMA reads
        bar.sync();
        if (t == 0) {
          const int row = (int)(((uint64_t)(2 * k + p) << H) + yh);
#pragma unroll
          for (int b = 0; b < 4; ++b) tma_store_3d(&tmw, 16 * b, 0, row, xb + 1024 * b);
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
      } else {
#pragma unroll
        for (int j = 0; j < 64; ++j) xb[xsw12(64u * t + j)] = v[j];
        bar.sync();
        // chunk C = t + 64 i holds positions 2C, 2C + 1: one 16-B load (halves swapped when the XOR key
        // flips bit 0) and one coalesced 16-B store -- each warp instruction writes 512 contiguous bytes
#pragma unroll 8
        for (int i = 0; i < 32; ++i) {
          const uint32_t e = 2u * (t + 64u * i);
          const uint32_t key = (e >> 6) & 15u;
          const double2 x = *reinterpret_cast<const double2*>(xb + ((e ^ key) & ~1u));
          const double2 y = (key & 1u) ? make_double2(x.y, x.x) : x;
          __stcg(reinterpret_cast<double2*>(wp + e), y);
        }
      }
    };
    transform_store(wrow, 0);                            // plane A
#pragma unroll
    for (int c = 0; c < 8; ++c) {                        // plane B back from TMEM
      uint32_t r32[16];
      tmem_ld8d(tm + 16u * c, r32);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 8; ++i) v[8 * c + i] = __hiloint2double(r32[2 * i + 1], r32[2 * i]);
    }
    transform_store(wrow + PLANE, 1);                    // plane B
  }
  if constexpr (TS)
    if (t == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  tmem_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tmem_s, 256);
}

// TMA tensor copy of one box into shared memory, completing on an mbarrier
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
               ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
               : "memory");
}

// k_passBw: radix-64 pass B over the row-major planes of k_passAw (L = 12) or k_passA10s<ROWM>
// (L = 10).  Tile (plane kp = 2k + p, column group s) = 2^H rows x 2^CB columns, gathered by 2^H / R
// TMA boxes of R = min(256, 2^H) rows x 2^CB columns (tensor map: dims {2^L, 2^H, 2K}) into the slot
// as e = row * 2^CB + col.
template <int CB, int L, bool A2>
__global__ void __launch_bounds__(256, 1) k_passBw(int kcount, const __grid_constant__ CUtensorMap tmap, Alphas al,
                                                   double* partial) {
  ln_table_init(!A2 && al.need_log);   // t ln t pass (tile_accumulate)
  constexpr int H = 13 - CB;
  static_assert(H >= 6 && H <= 11, "k_passBw: N = 17..20 (L = 10) and 21..24 (L = 12)");
  constexpr int R = H >= 8 ? 256 : (1 << H), NBOX = (1 << H) / R;
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[3];
  __shared__ volatile unsigned long long issued[3];
  __shared__ unsigned long long shist[SPEC_BINS];
  const int u = threadIdx.x >> 7;
  const uint32_t t = threadIdx.x & 127;
  const uint64_t slabs = 1ull << (L - CB);
  const uint64_t tiles = (uint64_t)kcount * 2 * slabs;
  const uint64_t my_tiles = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const BarNamed bar{1 + u, 128};
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) { mbar_init(&full[i], 1); issued[i] = ~0ull; }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (al.hist)
    for (int i = threadIdx.x; i < SPEC_BINS; i += blockDim.x) shist[i] = 0ull;
  __syncthreads();
  // issued[slot] = the CTA tile whose copy targets the slot.  The two units share three slots, so a
  // unit may only wait on a slot's mbarrier once its own tile has been issued there (tile n - 3, the
  // previous occupant, belongs to the other unit: testing the parity early could read a phase two
  // completions ahead and let a second copy land in the slot).
  auto issue = [&](uint64_t n) {                                   // one thread
    const int slot = (int)(n % 3);
    issued[slot] = n;
    const uint64_t tile = blockIdx.x + n * gridDim.x;
    const int kp = (int)(tile / slabs), col = (int)(tile % slabs) << CB;
    double* dst = smem + (size_t)slot * 8192;
    mbar_expect_tx(&full[slot], 8192 * sizeof(double));
#pragma unroll
    for (int b = 0; b < NBOX; ++b) tma_load_3d(dst + b * (R << CB), &tmap, col, b * R, kp, &full[slot]);
  };
  if (threadIdx.x == 0)
    for (uint64_t n = 0; n < 3 && n < my_tiles; ++n) issue(n);
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
  for (uint64_t n = (uint64_t)u; n < my_tiles; n += 2) {
    const int slot = (int)(n % 3);
    double* buf = smem + (size_t)slot * 8192;
    while (issued[slot] != n) __nanosleep(32);
    mbar_wait(&full[slot], (uint32_t)(n / 3) & 1u);
    double v[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = buf[t + 128u * j];      // round-0 layout, natural order
    bfly64(v);                                                   // 6 high row bits
    bar.sync();
#pragma unroll
    for (int j = 0; j < 64; ++j) buf[xsw13(t + 128u * j)] = v[j];
    bar.sync();
    const uint32_t tb = (t & 1u) | ((t >> 1) << 7);
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = buf[xsw13(tb | ((uint32_t)j << 1))];
    bar.sync();                                                  // slot free
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      if (n + 3 < my_tiles) issue(n + 3);
    }
    constexpr int CLO = CB - 1;
#pragma unroll
    for (int h = 1 << CLO; h < 64; h <<= 1)
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        if (i & h) continue;
        const double a = v[i], b = v[i + h];
        v[i] = a + b;
        v[i + h] = a - b;
      }
    tile_accumulate<A2>(acc, v, al);
    if (al.hist) spec_add(shist, v);
    if (al.chi) {     // sre_chi: tile element e = (row, col) of column group slab -> b' = (row << L) | position
      const uint64_t tile = blockIdx.x + n * gridDim.x;
      const uint64_t kp = tile / slabs, slab = tile % slabs;
      const uint64_t a = al.chi_a0 + (kp >> 1);
      const int p = pivot_of(a, L + H + 1);
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const uint32_t e = tb | ((uint32_t)j << 1);
        const uint64_t pos = (slab << CB) | (e & ((1u << CB) - 1u));
        const uint64_t bl = L == 10 ? pa10_freq_rowm((uint32_t)pos) : pos;   // k_passA10s<ROWM> store order
        chi_store(al.chi, a, p, (int)(kp & 1), ((uint64_t)(e >> CB) << L) | bl, v[j]);
      }
    }
  }
  block_flush(acc, partial, blockIdx.x);
  if (al.hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < SPEC_BINS; i += blockDim.x)
      if (shist[i]) atomicAdd(al.hist + i, shist[i]);
  }
}

// Per-call control block in the workspace (zeroed by the host before each range): a nonzero
// error makes k_reduce write NaN sums.
struct Ctl {
  int error;
};
// ------------------------------------------------------------------------------------------
// reduction of per-CTA partials (fixed order) + rescale t = 4 t' (DESIGN "Half-length").
//   out[s*(n+2)+i] = scale_i * sum_slot partial[s][slot][i]
// ------------------------------------------------------------------------------------------
struct ReduceArgs {
  int nslots;       // partial slots per state
  int n_alpha;      // total alphas of the call (row stride n_alpha + 2)
  int first;        // index of this sweep's first alpha
  int n_this;       // alphas in this sweep
  int write_common; // 1: also write purity and t ln t (sweep 0)
  double scale4[MAXA];  // 4^alpha_i
  const int* err;   // nonzero => a persistent kernel's watchdog fired: results are NaN
};

#ifdef SRE_API_TU   // non-template kernels: defined once, in sre_api.cu

__global__ void __launch_bounds__(256) k_reduce(const double* __restrict__ partial, ReduceArgs r, double* out) {
  // one block per state; thread i sums slots i, i+256, ... in order, then a fixed binary tree
  // over the 256 thread sums: deterministic for a given nslots
  const int s = blockIdx.x;
  const double* base = partial + (size_t)s * r.nslots * NACC;
  __shared__ double red[NACC][256];
  __shared__ double col[NACC];
  const int i = threadIdx.x;
  double acc[NACC];
#pragma unroll
  for (int c = 0; c < NACC; ++c) acc[c] = 0.0;
  for (int k = i; k < r.nslots; k += 256)
#pragma unroll
    for (int c = 0; c < NACC; ++c) acc[c] += base[(size_t)k * NACC + c];
#pragma unroll
  for (int c = 0; c < NACC; ++c) red[c][i] = acc[c];
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (i < h)
#pragma unroll
      for (int c = 0; c < NACC; ++c) red[c][i] += red[c][i + h];
    __syncthreads();
  }
  if (i < NACC) col[i] = red[i][0];
  __syncthreads();
  if (i == 0) {
    double* o = out + (size_t)s * (r.n_alpha + 2);
    if (r.err && *r.err) {
      for (int k = 0; k < r.n_alpha + 2; ++k) o[k] = __longlong_as_double(0x7ff8000000000000ll);
      return;
    }
    for (int k = 0; k < r.n_this; ++k) o[r.first + k] = col[k] * r.scale4[k];
    if (r.write_common) {
      o[r.n_alpha] = 4.0 * col[MAXA];
      // t = 4 t':  sum t ln t = 4 sum t' ln t' + 4 ln(4) sum t'
      o[r.n_alpha + 1] = 4.0 * col[MAXA + 1] + 4.0 * 1.3862943611198906 * col[MAXA];
    }
  }
}

// FP32 mode: psi (complex128) -> complex64 copy used by the FP32 kernels
__global__ void k_to_f32(const double2* __restrict__ src, float2* __restrict__ dst, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const double2 v = __ldg(src + i);
    dst[i] = make_float2((float)v.x, (float)v.y);
  }
}

// sum_x |psi_x|^2 per state (for the norm check), fixed-order block reduce then host/tiny sum
__global__ void k_norm2_partial(const double2* __restrict__ psi, int N, double* part) {
  const double2* ps = psi + ((size_t)blockIdx.y << N);
  const uint64_t n = 1ull << N;
  double acc = 0.0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const double2 q = __ldg(ps + i);
    acc = fma(q.x, q.x, fma(q.y, q.y, acc));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
    part[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}
__global__ void k_norm2_final(const double* __restrict__ part, int nb, double* out) {
  const int s = blockIdx.x;
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int k = 0; k < nb; ++k) acc += part[(size_t)s * nb + k];
    out[s] = acc;
  }
}

#endif  // SRE_API_TU

}  // namespace sre
