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
#include <cuda_runtime.h>
#include <type_traits>

#include "tmem.cuh"

namespace sre {

constexpr int MAXA = 4;          // Renyi indices per sweep (more are done in extra sweeps)
constexpr int NACC = MAXA + 2;   // [0,MAXA) alpha sums, [MAXA] purity, [MAXA+1] t ln t

struct Alphas {
  int n;                // alphas in this sweep
  int need_log;         // any alpha == 1
  int any_real;         // any kind == 2 (non-integer alpha)
  unsigned long long* hist;   // spectrum epilogue (two-pass kernels; nullptr = off)
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

// Epilogue of one tile's 32 values per thread into a fresh local sum, then one add into the
// long-lived accumulators: keeps the running-sum chains ~32x shorter (DESIGN "Summation").
// General alphas run in three compact phases (integer powers + purity; t ln t if some alpha = 1;
// real powers if some alpha is non-integer): interleaving the rarely-taken exp/log blocks with
// the common path made the executed code sparse in a ~200 KB body (10x slower, I-cache bound).
template <bool A2, class R, int M>
__device__ __forceinline__ void tile_accumulate(double (&acc)[NACC], const R (&v)[M], const Alphas& al) {
  R loc[NACC];          // FP32 mode: 32-term local sums in FP32, one conversion per tile
#pragma unroll
  for (int i = 0; i < NACC; ++i) loc[i] = R(0);
  if constexpr (A2) {
#pragma unroll
    for (int j = 0; j < M; ++j) Epi<true, R>::add(loc, v[j], al);
  } else {
    // General alphas: one compact (not unrolled) loop over the tile, t values staged through a
    // per-thread local array (L1).  Unrolling 32 copies of log / exp(a log t) made the kernel
    // instruction-cache bound (ncu: "no_instruction" the top stall).
    R tv[M];
#pragma unroll
    for (int j = 0; j < M; ++j) tv[j] = v[j] * v[j];
#pragma unroll 1
    for (int j = 0; j < M; ++j) {
      const R t = tv[j];
      loc[MAXA] += t;
#pragma unroll
      for (int i = 0; i < MAXA; ++i) {
        if (i >= al.n) break;
        if (al.kind[i] == 0) {
          R pw = t;
          for (int k = 1; k < al.iexp[i]; ++k) pw *= t;
          loc[i] += pw;
        } else {
          loc[i] += (t > R(0)) ? exp(R(al.alpha[i]) * log(t)) : R(0);
        }
      }
      if (al.need_log) loc[MAXA + 1] += (t > R(0)) ? t * log(t) : R(0);
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
// Chunk-major workspace for the TMEM pass B (H = 8): within a plane, position group
// g = pos >> 7 (128 positions), then chunk c = y_h & 7, then m = y_h >> 3, then pos & 127.
// A pass-B chunk (rows {c + 8m}, one 128-position group) is one contiguous 32 KB block.
__device__ __forceinline__ size_t cm_row_off(uint64_t yh) { return (size_t)(((yh & 7) << 5) | (yh >> 3)) << 7; }
template <int J>   // offset of position lane + 32 J (+ 1024 h) minus the lane: compile time
__device__ __forceinline__ constexpr size_t cm_pos_off(int h) {
  return ((size_t)((J >> 2) + 8 * h) << 15) + 32 * (J & 3);
}

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

constexpr int PA10_NS = 4;                                   // staging ring depth
constexpr int PA10_SMEM = PA10_NS * 2 * 1024 * 16 + 8 * padded(1024) * 8;  // 128 KB ring + 66 KB exchange

// Staged pass A for L = 10 (N = 15..20).  A persistent CTA of 8 warps walks items
// (group g of 8 X-strings sharing a_h != 0, row y_h).  The two psi rows an item needs
// (x_h = ins0(y_h, p-10) and x_h ^ a_h, 16 KB each) arrive by two bulk copies into a 4-deep
// ring completed on an mbarrier; warps run free (no CTA barrier): the last of the 8 warps to
// finish with a ring slot refills it with the item NS positions ahead.  Warp w generates
// X-string 8g + w from the staged rows, transforms 10 bits (one warp-local exchange per
// plane) and writes its row of both planes.
template <int N, bool RM = false, class V = double>   // RM: chunk-major workspace for the TMEM pass B
__global__ void __launch_bounds__(256, 1) k_passA10s(const typename Cx<V>::T* __restrict__ psi, uint64_t a_first,
                                                     int kcount, int groups, V* __restrict__ ws) {
  using C2 = typename Cx<V>::T;
  constexpr int cb = RM ? 10 : 12 - (N - 11);                   // pass B tile = 2^12 values
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
  if (threadIdx.x == 0) {
    for (int i = 0; i < PA10_NS; ++i) { mbar_init(&full[i], 1); used[i] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
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
      Rounds<10, 0, 0, 2, BarWarp, true, V>::run(v, xw, lane, BarWarp{});
      // slab-major workspace: (y_h, pos) -> ((pos >> cb) << (H + cb)) | (y_h << cb) | (pos & (C-1));
      // RM (TMEM pass B, H = 8): chunk-major ((pos >> 7) << 15) + row_off(y_h) + (pos & 127)
      if constexpr (RM) {
        static_assert(H == 8, "chunk-major layout assumes H = 8");
        V* w1 = ws + (size_t)k * 2 * plane + cm_row_off(yh) + lane;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const size_t o = ((size_t)(j >> 2) << 15) + 32 * (j & 3);
          __stcg(w1 + o, v[0][j]);
          __stcg(w1 + plane + o, v[1][j]);
        }
        continue;
      }
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

// ------------------------------------------------------------------------------------------
// k_fused: the whole two-pass sweep for N = 15..20 in ONE persistent launch (grid = #SMs,
// cooperative so every CTA is resident).  Each CTA runs two roles concurrently:
//   warps 0-3 ("A"): items (batch b, row y_h); a batch is 4 consecutive X-strings sharing a_h;
//                    the two psi rows arrive by bulk copy in a ring shared by the 4 warps;
//                    warp w generates X-string 4b + w and transforms the 10 low bits
//                    (same arithmetic as k_passA10s), writing the slab-major workspace slot b%S.
//   warps 4-7 ("B"): one 128-thread unit; tiles (batch b, plane, slab) of 2^12 doubles arrive by
//                    bulk copy (same arithmetic as k_passBt) and go through the H row bits and
//                    the epilogue.
// Work comes from two global tickets (in order), and the only waits are on earlier work:
//   A-item of batch b waits until every B-tile of batch b - S has been copied in (slot reuse);
//   B-tile of batch b waits until every A-item of batch b has been written.
// Waits spin on L2 counters with acquire loads and a 10 s watchdog that records an error.
// ------------------------------------------------------------------------------------------
struct FusedCtl {              // zeroed by the host before each launch
  unsigned long long a_next, b_next;
  unsigned long long a_done[4], b_done[4];
  int error;
};
constexpr int FZ_S = 2;                      // workspace slots (batches in flight)
constexpr int FZ_KB = 4;                     // X-strings per batch (= A warps)
constexpr int FZ_NSA = 3;                    // A staging ring depth (32 KB each)
constexpr int FZ_NSB = 2;                    // B tile ring depth (33 KB each)
constexpr int FZ_SMEM = FZ_NSA * 2048 * 16 + FZ_KB * padded(1024) * 8 + FZ_NSB * padded(4096) * 8;

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;\n" : "=l"(t));
  return t;
}
// spin until *p >= target; false (and ctl->error set) on a 10 s timeout
__device__ __forceinline__ bool wait_geq(const unsigned long long* p, unsigned long long target, FusedCtl* ctl) {
  if (ld_acquire(p) >= target) return true;
  const uint64_t t0 = gtimer();
  while (ld_acquire(p) < target) {
    __nanosleep(200);
    if (gtimer() - t0 > 10000000000ull || *(volatile int*)&ctl->error) { atomicExch(&ctl->error, 1); return false; }
  }
  return true;
}

template <int N, bool A2>
__global__ void __launch_bounds__(256, 1) k_fused(const double2* __restrict__ psi, uint64_t a_first, uint64_t count,
                                                  double* __restrict__ ws, FusedCtl* ctl, Alphas al, double* partial) {
  constexpr int H = N - 11, CB = 12 - H, TP = 12, TILE = 1 << TP;
  constexpr uint64_t ROWS = 1ull << H;
  constexpr uint64_t SLABS = 1ull << (10 - CB);
  constexpr uint64_t TPB = (uint64_t)FZ_KB * 2 * SLABS;   // B tiles per full batch
  constexpr size_t PLANE = (size_t)1 << (N - 1);
  constexpr size_t SLOT = (size_t)FZ_KB * 2 * PLANE;     // doubles per workspace slot
  constexpr uint64_t END = ~0ull;
  extern __shared__ __align__(128) double smem[];
  double2* ringA = reinterpret_cast<double2*>(smem);                          // [NSA][2048]
  double* exA = smem + FZ_NSA * 2048 * 2;                                     // [4][padded 1024]
  double* ringB = exA + FZ_KB * padded(1024);                                 // [NSB][padded 4096]
  __shared__ __align__(8) uint64_t fullA[FZ_NSA], fullB[FZ_NSB];
  __shared__ uint64_t itemA[FZ_NSA], itemB[FZ_NSB];
  __shared__ int usedA[FZ_NSA];
  __shared__ double redB[4][NACC];
  const uint64_t nbatch = (count + FZ_KB - 1) / FZ_KB;
  const uint64_t totA = nbatch * ROWS;
  const uint64_t totB = (count / FZ_KB) * TPB + (count % FZ_KB) * 2 * SLABS;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < FZ_NSA; ++i) { mbar_init(&fullA[i], 1); usedA[i] = 0; }
    for (int i = 0; i < FZ_NSB; ++i) mbar_init(&fullB[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // A producer (one thread, never waits): next A ticket into ring slot s, stage its psi rows
  auto produceA = [&](int s) {
    const uint64_t t = atomicAdd(&ctl->a_next, 1ull);
    if (t >= totA) {
      itemA[s] = END;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&fullA[s])) : "memory");
      return;
    }
    const uint64_t b = t >> H, yh = t & (ROWS - 1);
    const uint64_t ag = a_first + FZ_KB * b;
    const int p = 63 - __clzll((long long)ag);
    const uint64_t xh = ins0(yh, p - 10);
    itemA[s] = t;
    double2* dst = ringA + (size_t)s * 2048;
    mbar_expect_tx(&fullA[s], 2 * 1024 * 16);
    bulk_g2s(dst, psi + (xh << 10), 1024 * 16, &fullA[s]);
    bulk_g2s(dst + 1024, psi + ((xh ^ (ag >> 10)) << 10), 1024 * 16, &fullA[s]);
  };

  if (w < 4) {
    // ======================= A role =======================
    if (threadIdx.x == 0)
      for (int s = 0; s < FZ_NSA; ++s) produceA(s);
    double* xw = exA + (size_t)w * padded(1024);
    for (uint32_t n = 0;; ++n) {
      const int s = (int)(n % FZ_NSA);
      mbar_wait(&fullA[s], (n / FZ_NSA) & 1u);
      const uint64_t t = itemA[s];
      if (t == END) break;
      const uint64_t b = t >> H, yh = t & (ROWS - 1);
      const uint64_t kglob = FZ_KB * b + w;
      const bool active = kglob < count;
      double v[2][32];
      if (active) {
        const uint32_t alow = (uint32_t)((a_first + kglob) & 1023u);
        const double2* sq = ringA + (size_t)s * 2048;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const uint32_t yl = lane + 32 * j;
          const double2 q = sq[yl];
          const double2 r = sq[1024 + (yl ^ alow)];
          v[0][j] = fma(r.x, q.x, r.y * q.y);
          v[1][j] = fma(r.x, q.y, -(r.y * q.x));
        }
        Rounds<10, 0, 0, 2, BarWarp, true>::run(v, xw, lane, BarWarp{});
        // workspace slot b%S is free once every B tile of batch b - S has been copied out
        if (b >= FZ_S && lane == 0) wait_geq(&ctl->b_done[b % FZ_S], (b / FZ_S) * TPB, ctl);
        __syncwarp();
        double* w0 = ws + (b % FZ_S) * SLOT + (size_t)w * 2 * PLANE + (yh << CB);
        constexpr uint32_t cm = (1u << CB) - 1u;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const uint32_t pos = lane + 32 * j;
          const size_t off = ((size_t)(pos >> CB) << (H + CB)) + (pos & cm);
          __stcg(w0 + off, v[0][j]);
          __stcg(w0 + PLANE + off, v[1][j]);
        }
        __threadfence();
      }
      __syncwarp();
      if (lane == 0) {
        // the last of the 4 warps to finish this item publishes it and refills the ring slot
        if (atomicAdd(&usedA[s], 1) == FZ_KB - 1) {
          atomicExch(&usedA[s], 0);
          __threadfence();
          red_release_add(&ctl->a_done[b % FZ_S], 1ull);
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          produceA(s);
        }
      }
    }
  } else {
    // ======================= B role =======================
    const uint32_t tb = threadIdx.x - 128;
    const BarNamed bar{1, 128};
    double acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
    // Leader-only producer state.  positions [0, issued) are staged; [0, credited) have been
    // credited to b_done (their copy has landed, so the workspace slot no longer needs them).
    // A claimed tile may have to wait for its batch; before the leader waits it credits every
    // staged position, so nothing another warp waits on is ever held back by that wait.
    uint32_t issued = 0, credited = 0;
    bool ended = false;
    auto credit_upto = [&](uint32_t upto) {
      for (; credited < upto; ++credited) {
        const int cs = (int)(credited % FZ_NSB);
        mbar_wait(&fullB[cs], (credited / FZ_NSB) & 1u);
        const uint64_t ct = itemB[cs];
        if (ct != END) red_release_add(&ctl->b_done[(ct / TPB) % FZ_S], 1ull);
      }
    };
    auto produce_upto = [&](uint32_t upto) {     // fill positions [issued, upto)
      while (issued < upto && !ended) {
        const int ps = (int)(issued % FZ_NSB);
        const uint64_t t = atomicAdd(&ctl->b_next, 1ull);
        if (t >= totB) {
          itemB[ps] = END;
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&fullB[ps])) : "memory");
          ++issued;
          ended = true;
          return;
        }
        const uint64_t b = t / TPB;
        const unsigned long long need = (b / FZ_S + 1) * ROWS;
        if (ld_acquire(&ctl->a_done[b % FZ_S]) < need) {
          credit_upto(issued);
          if (!wait_geq(&ctl->a_done[b % FZ_S], need, ctl)) {
            itemB[ps] = END;
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&fullB[ps])) : "memory");
            ++issued;
            ended = true;
            return;
          }
        }
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        itemB[ps] = t;
        mbar_expect_tx(&fullB[ps], TILE * 8);
        bulk_g2s(ringB + (size_t)ps * padded(TILE), ws + (b % FZ_S) * SLOT + (t % TPB) * TILE, TILE * 8, &fullB[ps]);
        ++issued;
      }
    };
    for (uint32_t n = 0;; ++n) {
      const int s = (int)(n % FZ_NSB);
      if (tb == 0) {
        produce_upto(n + FZ_NSB);
        credit_upto(n + 1);                      // this position's copy has landed
      }
      mbar_wait(&fullB[s], (n / FZ_NSB) & 1u);
      const uint64_t t = itemB[s];
      if (t == END) break;
      double* buf = ringB + (size_t)s * padded(TILE);
      double v[1][32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[0][j] = buf[tb + 128 * j];
      Rounds<TP, CB, 0, 1, BarNamed>::run(v, buf, tb, bar);
      bar.sync();                                // the slot's smem is free for the next copy
      if (tb == 0) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      tile_accumulate<A2>(acc, v[0], al);
    }
    // B-role accumulators -> partial[blockIdx.x]
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      double x = acc[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) redB[w - 4][i] = x;
    }
    bar.sync();
    if (tb < NACC) {
      double sacc = 0.0;
      for (int k = 0; k < 4; ++k) sacc += redB[k][tb];
      partial[(size_t)blockIdx.x * NACC + tb] += sacc;
    }
  }
}

// ==========================================================================================
// TMEM path for N = 19, 20 (T = N-1 = L + 8).  Pass B gives every thread one workspace column of
// 2^8 rows held in tensor memory, so the 8 row bits are transformed inside the thread with no
// shared-memory exchange; pass A (L = 11 at N = 20) parks one plane in TMEM so a warp can own
// 64 values per plane per lane (6 in-thread bits).  L1TEX data-pipe traffic per output value:
// 16 B generation + 16 B exchange + 8 B store (A) + 8 B load (B) = 48 B.
// Workspace: row-major planes [k][plane][y_h][pos], 2^L positions per row; pos low 5 bits are
// y_l bits 5..9 (the lane index of pass A's final layout), so both passes access it coalesced.
// ==========================================================================================
// 32x32 transpose of one value per (lane, j) through a warp-private padded buffer:
// element e = lane + 32 j is read back as e = j + 32 lane (conflict-free both ways)
__device__ __forceinline__ void warp_transpose32(double (&v)[32], double* xw, int lane) {
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 32; ++j) xw[swz(lane + 32 * j)] = v[j];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = xw[swz(j + 32 * lane)];
}

constexpr int PA11_NS = 2;                                                   // staging ring depth
constexpr int PA11_SMEM = PA11_NS * 2 * 2048 * 16 + 8 * padded(1024) * 8;   // 128 KB ring + 66 KB exchange

template <int N>
__global__ void __launch_bounds__(256, 1) k_passA11t(const double2* __restrict__ psi, uint64_t a_first, int kcount,
                                                     int groups, double* __restrict__ ws) {
  constexpr int L = 11, H = N - 1 - L;
  constexpr uint64_t ROWS = 1ull << H;
  constexpr size_t PLANE = (size_t)1 << (N - 1);
  extern __shared__ __align__(128) double smem[];
  double2* ring = reinterpret_cast<double2*>(smem);             // [NS][q row | r row][2048]
  double* exch = smem + PA11_NS * 2 * 2048 * 2;                 // [warp][padded 1024]
  __shared__ __align__(8) uint64_t full[PA11_NS];
  __shared__ int used[PA11_NS];
  __shared__ uint32_t tbase;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t items = ROWS * (uint64_t)groups;
  if (w == 0) tmem_alloc_warp(&tbase, 512);
  if (threadIdx.x == 0) {
    for (int i = 0; i < PA11_NS; ++i) { mbar_init(&full[i], 1); used[i] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  // this warp's TMEM: lanes 32*(w%4).., columns (w/4)*256 ..; chunks A0 @0, B0 @64, B1 @128
  const uint32_t tw = tbase + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)(w >> 2) * 256;
  auto issue = [&](uint64_t item, int slot) {
    const uint64_t g = item >> H, yh = item & (ROWS - 1);
    const uint64_t ag = a_first + 8 * g;
    const int p = 63 - __clzll((long long)ag);                  // >= 11 (a >= 2048)
    const uint64_t xh = ins0(yh, p - L);
    double2* dst = ring + (size_t)slot * 4096;
    mbar_expect_tx(&full[slot], 2 * 2048 * 16);
    bulk_g2s(dst, psi + (xh << L), 2048 * 16, &full[slot]);
    bulk_g2s(dst + 2048, psi + ((xh ^ (ag >> L)) << L), 2048 * 16, &full[slot]);
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < PA11_NS; ++i)
      if (blockIdx.x + (uint64_t)i * gridDim.x < items) issue(blockIdx.x + (uint64_t)i * gridDim.x, i);
  double* xw = exch + (size_t)w * padded(1024);
  uint32_t n = 0;
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x, ++n) {
    const int slot = (int)(n % PA11_NS);
    mbar_wait(&full[slot], (n / PA11_NS) & 1u);
    const uint64_t g = item >> H, yh = item & (ROWS - 1);
    const int k = 8 * (int)g + w;
    const bool active = k < kcount;
    double lo[32], hi[32];
    if (active) {
      const uint32_t al = (uint32_t)((a_first + (uint64_t)k) & 2047u);
      const double2* sq = ring + (size_t)slot * 4096;
      // chunk c: y_l = lane + 32 j + 1024 c; registers j <-> y bits 5..9
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        double A[32], B[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const uint32_t yl = lane + 32 * j + 1024 * c;
          const double2 q = sq[yl];
          const double2 r = sq[2048 + (yl ^ al)];
          A[j] = fma(r.x, q.x, r.y * q.y);
          B[j] = fma(r.x, q.y, -(r.y * q.x));
        }
        bfly32<0, 5>(A);
        bfly32<0, 5>(B);
        if (c == 0) {
          tmem_st32(tw + 0, A);
          tmem_st32(tw + 64, B);
        } else {
          tmem_st32(tw + 128, B);
#pragma unroll
          for (int j = 0; j < 32; ++j) hi[j] = A[j];
        }
      }
    }
    __syncwarp();
    if (lane == 0 && atomicAdd(&used[slot], 1) == 7) {          // ring slot read out by all 8 warps
      atomicExch(&used[slot], 0);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      const uint64_t nx = item + (uint64_t)PA11_NS * gridDim.x;
      if (nx < items) issue(nx, slot);
    }
    if (active) {
      tmem_wait_st();
#pragma unroll
      for (int pl = 0; pl < 2; ++pl) {
        if (pl == 0) tmem_ld32(tw + 0, lo);                     // A0; A1 is already in hi
        else { tmem_ld32(tw + 64, lo); tmem_ld32(tw + 128, hi); }
#pragma unroll
        for (int j = 0; j < 32; ++j) {                          // y bit 10
          const double u = lo[j], v2 = hi[j];
          lo[j] = u + v2;
          hi[j] = u - v2;
        }
        // exchange each half: (lane <-> y bits 0-4, j <-> 5-9) -> (lane <-> 5-9, j <-> 0-4)
        warp_transpose32(lo, xw, lane);
        warp_transpose32(hi, xw, lane);
        bfly32<0, 5>(lo);
        bfly32<0, 5>(hi);
        // position pos = lane + 32 j + 1024 h  (pos bits 0-4 = b_l bits 5-9, contiguous over lanes),
        // stored chunk-major: ((pos >> 7) << 15) + row_off(y_h) + (pos & 127)
        double* dst = ws + (size_t)k * 2 * PLANE + (size_t)pl * PLANE + cm_row_off(yh) + lane;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const size_t o = ((size_t)(j >> 2) << 15) + 32 * (j & 3);
          __stcg(dst + o, lo[j]);
          __stcg(dst + (8ull << 15) + o, hi[j]);
        }
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc_warp(tbase, 512);
}

// Pass B with the 8 row bits in TMEM: a CTA of 4 warps walks tiles (k, plane, 128-position
// group); thread = one position (column), its 256 rows live in its TMEM lane (512 columns).
// The tile streams in as 8 chunks (chunk c = rows {c + 8m}, m = 0..31) through a 4-deep ring of
// 32 KB shared-memory buffers filled by bulk copies (one 1 KB row segment per lane), so global
// latency is off the critical path.  Round 1: chunk c (row bits 3-7 in registers) is read from
// shared memory, transformed and parked at TMEM columns 64c.  Round 2: groups of 4 m's across
// the 8 chunks (row bits 0-2) come back from TMEM and feed the epilogue directly.
constexpr int PB8_NS = 4;
constexpr int PB8_SMEM = PB8_NS * 32 * 128 * 8;   // 4 x 32 KB

template <int N, bool A2>
__global__ void __launch_bounds__(128, 1) k_passBt8(int kcount, const double* __restrict__ ws, Alphas al,
                                                    double* partial) {
  constexpr int H = 8, L = N - 1 - H;
  constexpr size_t PLANE = (size_t)1 << (N - 1);
  constexpr uint64_t GROUPS = 1ull << (L - 7);                  // 128-position groups per plane
  extern __shared__ __align__(128) double smem[];               // [NS][32 rows][128 positions]
  __shared__ __align__(8) uint64_t full[PB8_NS];
  __shared__ int used[PB8_NS];
  __shared__ uint32_t tbase;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 0) tmem_alloc_warp(&tbase, 512);
  if (threadIdx.x == 0) {
    for (int i = 0; i < PB8_NS; ++i) { mbar_init(&full[i], 1); used[i] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tw = tbase + ((uint32_t)(32 * w) << 16);
  const uint64_t tiles = (uint64_t)kcount * 2 * GROUPS;
  const uint64_t my_tiles = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint64_t nchunks = my_tiles * 8;                        // chunk n: tile blockIdx + (n/8) grid, c = n%8
  // a chunk (rows {c + 8m} of one 128-position group) is one contiguous 32 KB block (chunk-major)
  auto issue = [&](uint64_t nch, int slot) {
    if (lane != 0) return;
    const uint64_t tile = blockIdx.x + (nch >> 3) * gridDim.x;
    const int c = (int)(nch & 7);
    const uint64_t kp = tile / GROUPS, grp = tile % GROUPS;
    mbar_expect_tx(&full[slot], 32 * 128 * 8);
    bulk_g2s(smem + (size_t)slot * 4096, ws + kp * PLANE + (grp << 15) + ((size_t)c << 12), 32 * 128 * 8, &full[slot]);
  };
  if (w == 0)
    for (int i = 0; i < PB8_NS; ++i)
      if ((uint64_t)i < nchunks) issue(i, i);
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
  uint64_t n = 0;
  for (uint64_t t = 0; t < my_tiles; ++t) {
#pragma unroll 1
    for (int c = 0; c < 8; ++c, ++n) {
      const int slot = (int)(n % PB8_NS);
      mbar_wait(&full[slot], (uint32_t)(n / PB8_NS) & 1u);
      double v[32];
      const double* buf = smem + (size_t)slot * 4096 + 32 * w + lane;
#pragma unroll
      for (int m = 0; m < 32; ++m) v[m] = buf[128 * m];
      __syncwarp();
      int last = 0;
      if (lane == 0) last = atomicAdd(&used[slot], 1) == 3;     // last of the 4 warps to read it
      if (__shfl_sync(0xffffffffu, last, 0)) {
        if (lane == 0) atomicExch(&used[slot], 0);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        if (n + PB8_NS < nchunks) issue(n + PB8_NS, slot);
      }
      bfly32<0, 5>(v);
      tmem_st32(tw + 64 * c, v);
    }
    tmem_wait_st();
    double loc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) loc[i] = 0.0;
#pragma unroll 1
    for (int q = 0; q < 8; ++q) {
      double u[32];                                             // u[4c + i] = row c + 8 (4q + i)
      tmem_ld4x8(tw + 8 * q, u);
#pragma unroll
      for (int b = 2; b < 5; ++b) {                             // register bits 2-4 <-> row bits 0-2
        const int hh = 1 << b;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (i & hh) continue;
          const double x = u[i], y = u[i + hh];
          u[i] = x + y;
          u[i + hh] = x - y;
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) Epi<A2>::add(loc, u[j], al);
    }
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] += loc[i];
  }
  tmem_fence_before();
  block_flush(acc, partial, blockIdx.x);
  if (w == 0) tmem_dealloc_warp(tbase, 512);
}

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
