// mana.cu -- pure-state qutrit mana (NEXT-3): Algorithm 5 of PAPER.md on sm_100a.
//
// For every X-string a in Z_3^N: alpha = X_a psi (alpha_x = psi_{x-a}), v_x = conj(alpha_x) alpha_{-x}
// (Eq. (32)), chi(a) = F_3^{(x)N} v with (F_3)_{jk} = omega^{2jk} (Eqs. (35)-(36),
// P:836-868), and the sums  S_abs = sum_{a,b} |chi_b(a)|,  S_sum = sum_{a,b} chi_b(a).
// mana = log2(S_abs / 3^N) (Eq. (10), reading C18); S_sum = 3^N ||psi||^2 (sum_u A_u = 3^N I).
//
// B200 design:
//  * Hermitian packing.  v_{-x} = conj(v_x), so chi(a) is real.  Two X-strings a1, a2
//    share one complex transform: F(v1 + i v2) = chi(a1) + i chi(a2), read back as |Re| + |Im|.
//    This halves the transform work and the workspace traffic against one transform per a.
//  * Index split x = h 3^L + l (high digits h, low digits l).  The digit-wise shifts x - a and
//    -x - a split the same way, so a CTA that owns row h reads two contiguous rows of psi per a.
//  * Pass A (k_mana_row): per (pair, h): gather + conj-product of 3^G consecutive l per thread,
//    radix-3^G in registers, the remaining L - G digits as radix-9/3 stages in shared memory,
//    then either the row is stored to the workspace (N > 8) or |Re| + |Im| is accumulated (N <= 8).
//  * Pass B (k_mana_col): per (pair, block of S columns): the 3^H x S tile of the workspace,
//    F_3 over the H high digits in shared memory, |Re| + |Im| accumulated in the last stage.
//  * Persistent grids; per-CTA FP64 accumulators added to per-CTA slots in launch order and a
//    fixed-order reduction: results are bitwise reproducible for a given device and N.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/sre.h"
#include "launch.cuh"
#include "mana_remap_tab.h"

namespace sre_host {
int fail(int code, const char* fmt, ...);
int get_dev(Dev& d);
int is_device_ptr(const void* ptr, bool& dev);
}  // namespace sre_host

namespace mana {

__host__ __device__ constexpr int p3(int k) {
  int r = 1;
  for (int i = 0; i < k; ++i) r *= 3;
  return r;
}

constexpr int kThreads = 256;
constexpr int kSlots = 4096;          // per-CTA accumulator slots (2 doubles each)

// Radix-3 butterfly, y_r = sum_c omega^{2rc} u_c (Eq. (35)):
//   y0 = u0 + s,  y1 = t - i c d,  y2 = t + i c d,  s = u1 + u2, d = u1 - u2, t = u0 - s/2, c = sqrt3/2.
__device__ __forceinline__ void bfly3(double2& u0, double2& u1, double2& u2) {
  const double c = 0.86602540378443864676;
  const double sr = u1.x + u2.x, si = u1.y + u2.y;
  const double dr = u1.x - u2.x, di = u1.y - u2.y;
  const double tr = fma(-0.5, sr, u0.x), ti = fma(-0.5, si, u0.y);
  u0.x += sr;
  u0.y += si;
  u1.x = fma(c, di, tr);
  u1.y = fma(-c, dr, ti);
  u2.x = fma(-c, di, tr);
  u2.y = fma(c, dr, ti);
}

// F_3 on the G ternary digits of a register array (digit g has stride 3^g).
template <int G>
__device__ __forceinline__ void reg_f3(double2* r) {
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int s = p3(g);
#pragma unroll
    for (int f = 0; f < p3(G - 1); ++f) {
      const int lo = f % s, hi = f / s;
      const int b = hi * 3 * s + lo;
      bfly3(r[b], r[b + s], r[b + 2 * s]);
    }
  }
}

// Digit-wise (x - a) mod 3 and (-x - a) mod 3 over n ternary digits.
template <int n>
__device__ __forceinline__ void tshift(int x, int a, int& sub, int& neg) {
  sub = 0;
  neg = 0;
  int p = 1;
#pragma unroll
  for (int j = 0; j < n; ++j) {
    const int xj = x % 3, aj = a % 3;
    x /= 3;
    a /= 3;
    sub += ((xj - aj + 3) % 3) * p;
    neg += ((6 - xj - aj) % 3) * p;
    p *= 3;
  }
}
__device__ __forceinline__ void tshift_rt(int x, int a, int n, int& sub, int& neg) {
  sub = 0;
  neg = 0;
  int p = 1;
  for (int j = 0; j < n; ++j) {
    const int xj = x % 3, aj = a % 3;
    x /= 3;
    a /= 3;
    sub += ((xj - aj + 3) % 3) * p;
    neg += ((6 - xj - aj) % 3) * p;
    p *= 3;
  }
}

// One shared-memory stage: F_3 on digits [J, J+g) of the row index of a 3^M x S tile
// (element (e, c) at tile[e*S + c]).  ACC: accumulate |Re| + |Im| and Re + Im instead of storing.
template <int M, int S, int J, int g, bool ACC>
__device__ __forceinline__ void stage(double2* tile, double& aa, double& as) {
  constexpr int R = p3(g);
  constexpr int st = p3(J);
  constexpr int fibers = p3(M - g) * S;
  for (int f = threadIdx.x; f < fibers; f += kThreads) {
    const int c = f % S, rest = f / S;
    const int lo = rest % st, hi = rest / st;
    const int base = (hi * st * R + lo) * S + c;
    double2 r[R];
#pragma unroll
    for (int k = 0; k < R; ++k) r[k] = tile[base + k * st * S];
    reg_f3<g>(r);
    if constexpr (ACC) {
#pragma unroll
      for (int k = 0; k < R; ++k) {
        aa += fabs(r[k].x) + fabs(r[k].y);
        as += r[k].x + r[k].y;
      }
    } else {
#pragma unroll
      for (int k = 0; k < R; ++k) tile[base + k * st * S] = r[k];
    }
  }
}

template <int M, int S, int J, bool ACC_LAST>
__device__ __forceinline__ void stages(double2* tile, double& aa, double& as) {
  if constexpr (J < M) {
    constexpr int g = (M - J >= 2) ? 2 : 1;
    constexpr bool last = (J + g == M);
    stage<M, S, J, g, ACC_LAST && last>(tile, aa, as);
    if constexpr (!(ACC_LAST && last)) __syncthreads();
    stages<M, S, J + g, ACC_LAST>(tile, aa, as);
  }
}

// Functor-driven stage: same fibers as stage(), element e read through ld(e) and written through
// st(e, v) -- lets the first stage read global memory and the last write it (or accumulate).
template <int M, int S, int J, int g, class Ld, class St>
__device__ __forceinline__ void stage_f(Ld ld, St st) {
  constexpr int R = p3(g);
  constexpr int sj = p3(J);
  constexpr int fibers = p3(M - g) * S;
  for (int f = threadIdx.x; f < fibers; f += kThreads) {
    const int c = f % S, rest = f / S;
    const int lo = rest % sj, hi = rest / sj;
    const int base = (hi * sj * R + lo) * S + c;
    double2 r[R];
#pragma unroll
    for (int k = 0; k < R; ++k) r[k] = ld(base + k * sj * S);
    reg_f3<g>(r);
#pragma unroll
    for (int k = 0; k < R; ++k) st(base + k * sj * S, r[k]);
  }
}

// Digits [J, M) of a 3^M x S tile; the first stage (if FIRST) loads through ldf, the last stores
// through stl, intermediate stages go through shared memory.
template <int M, int S, int J, bool FIRST, class LdF, class StL>
__device__ __forceinline__ void stages_f(double2* tile, LdF ldf, StL stl) {
  if constexpr (J < M) {
    constexpr int g = (M - J >= 2) ? 2 : 1;
    constexpr bool last = (J + g == M);
    auto lds = [&](int e) { return tile[e]; };
    auto sts = [&](int e, double2 v) { tile[e] = v; };
    if constexpr (FIRST && last) stage_f<M, S, J, g>(ldf, stl);
    else if constexpr (FIRST) stage_f<M, S, J, g>(ldf, sts);
    else if constexpr (last) stage_f<M, S, J, g>(lds, stl);
    else stage_f<M, S, J, g>(lds, sts);
    if constexpr (!last) __syncthreads();
    stages_f<M, S, J + g, false>(tile, ldf, stl);
  }
}

// Fixed-order block reduction of (aa, as); thread 0 adds the result to slots[2*blockIdx.x..].
__device__ __forceinline__ void flush(double aa, double as, double* slots) {
  __shared__ double red[2][kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    aa += __shfl_down_sync(0xffffffffu, aa, o);
    as += __shfl_down_sync(0xffffffffu, as, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = aa;
    red[1][w] = as;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ta = 0.0, ts = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) {
      ta += red[0][i];
      ts += red[1][i];
    }
    slots[2 * blockIdx.x] += ta;
    slots[2 * blockIdx.x + 1] += ts;
  }
}

struct RowArgs {
  const double2* psi;
  double2* ws;          // [pairs in launch][3^N]  (unused when FINAL)
  double* slots;
  uint64_t a_begin, a_end;
  uint64_t pair0;       // first pair of this launch (pair p covers a_begin + 2p, a_begin + 2p + 1)
  int npairs;           // pairs in this launch
  int H;                // high digits (N - L)
};

// Pass A / single pass.  Row h of pair p: w_l = v1_{h,l} + i v2_{h,l}, F_3 over the L low digits.
template <int L, bool FINAL, int G = (L > 5 ? L - 5 : 0)>
__global__ void __launch_bounds__(kThreads) k_mana_row(RowArgs A) {
  // G: low digits done in registers (3^G consecutive l per thread group)
  constexpr int RG = p3(G);
  constexpr int NT = p3(L - G);              // thread groups per row
  constexpr int NL = p3(L);
  extern __shared__ double2 tile[];
  const int nh = p3(A.H);
  const long items = (long)A.npairs * nh;
  double aa = 0.0, as = 0.0;
  for (long it = blockIdx.x; it < items; it += gridDim.x) {
    const int pl = (int)(it / nh), h = (int)(it % nh);
    const uint64_t a1 = A.a_begin + 2 * (A.pair0 + pl);
    const bool two = a1 + 1 < A.a_end;
    for (int t = threadIdx.x; t < NT; t += kThreads) {
      double2 r[RG];
      // X-string a1 (and a2 = a1 + 1): rows of psi and the shifted low-index bases
      int rs[2], rn[2], ls[2], ln[2], alo[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint64_t a = a1 + q;
        const int ah = (int)(a / NL), al = (int)(a % NL);
        int hs, hn;
        tshift_rt(h, ah, A.H, hs, hn);
        rs[q] = hs;
        rn[q] = hn;
        int us, un;
        tshift<L - G>(t, al / RG, us, un);
        ls[q] = us * RG;
        ln[q] = un * RG;
        alo[q] = al % RG;
      }
#pragma unroll
      for (int i = 0; i < RG; ++i) {
        double2 w = make_double2(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (q == 1 && !two) break;
          int ss, sn;
          tshift<G>(i, alo[q], ss, sn);
          const double2 x1 = __ldg(A.psi + (size_t)rs[q] * NL + ls[q] + ss);   // alpha_x
          const double2 x2 = __ldg(A.psi + (size_t)rn[q] * NL + ln[q] + sn);   // alpha_{-x}
          const double vr = x1.x * x2.x + x1.y * x2.y;                           // conj(alpha_x) alpha_{-x}
          const double vi = x1.x * x2.y - x1.y * x2.x;
          if (q == 0) {
            w.x += vr;
            w.y += vi;
          } else {
            w.x -= vi;                                                           // + i v2
            w.y += vr;
          }
        }
        r[i] = w;
      }
      reg_f3<G>(r);
#pragma unroll
      for (int i = 0; i < RG; ++i) tile[t * RG + i] = r[i];
    }
    __syncthreads();
    if constexpr (FINAL) {
      stages<L, 1, G, true>(tile, aa, as);
    } else {
      stages<L, 1, G, false>(tile, aa, as);
      double2* dst = A.ws + (size_t)pl * ((size_t)nh * NL) + (size_t)h * NL;
      for (int l = threadIdx.x; l < NL; l += kThreads) __stcg(dst + l, tile[l]);
    }
    __syncthreads();
  }
  if constexpr (FINAL) flush(aa, as, A.slots);
}


struct ColArgs {
  const double2* ws;    // [pairs in launch][3^H][3^L]
  double* slots;
  int npairs;
  int L;
};

// Pass B.  Columns [c0, c0 + S) of pair p: F_3 over the H high digits, |Re| + |Im| accumulated.
template <int H, int S>
__global__ void __launch_bounds__(kThreads) k_mana_col(ColArgs A) {
  extern __shared__ double2 tile[];
  constexpr int NH = p3(H);
  const int NL = p3(A.L);
  const int nblk = (NL + S - 1) / S;
  const long items = (long)A.npairs * nblk;
  double aa = 0.0, as = 0.0;
  for (long it = blockIdx.x; it < items; it += gridDim.x) {
    const int pl = (int)(it / nblk), cb = (int)(it % nblk);
    const int c0 = cb * S;
    const int ncol = min(S, NL - c0);
    const double2* src = A.ws + (size_t)pl * NH * NL + c0;
    for (int e = threadIdx.x; e < NH * S; e += kThreads) {
      const int row = e / S, c = e % S;
      tile[e] = c < ncol ? __ldcs(src + (size_t)row * NL + c) : make_double2(0.0, 0.0);
    }
    __syncthreads();
    stages<H, S, 0, true>(tile, aa, as);
    __syncthreads();
  }
  flush(aa, as, A.slots);
}

// ---------------------------------------------------------------------------------------------
// Staged two-pass (N = 9..14): rows of psi staged in shared memory and shared by the PP pairs of
// one item; the workspace is column-blocked, ws[pair][cb][h][c] (S columns per block), so that a
// pass-B tile is one contiguous 3^H x S chunk.
// ---------------------------------------------------------------------------------------------
struct RowSArgs {
  const double2* psi;
  double2* ws;
  uint64_t a_begin, a_end;
  uint64_t pair0;       // first pair of this launch
  int npairs;           // pairs in this launch
  int H;                // high digits
  int S;                // columns per workspace block
  int PP;               // pairs per item
  int remap;            // L - G = 5: per-shift lane remap (kManaRemap) of the thread groups
};

// Digit-shift tables of one X-string's low digits: for ternary digit j of an index k,
//   sub(k) = sum_j ds[j][k_j],  neg(k) = sum_j dn[j][k_j]   with
//   ds[j][d] = ((d - a_j) mod 3) 3^j,  dn[j][d] = ((-d - a_j) mod 3) 3^j.
// Built once per X-string; an unrolled loop over compile-time k then needs two adds per index.
template <int G>
struct ShiftTab {
  int ds[G > 0 ? G : 1][3], dn[G > 0 ? G : 1][3];
  __device__ __forceinline__ void build(int a) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int aj = a % 3, p = p3(j);
      a /= 3;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        ds[j][d] = ((d - aj + 3) % 3) * p;
        dn[j][d] = ((6 - d - aj) % 3) * p;
      }
    }
  }
};

// Two-digit (G = 2) generator with compile-time shifts: both X-strings of a pair whose low parts
// are C and C + 1 (mod 9, no carry into digit 2) read the same two 9-blocks bA (rowA) and bB
// (rowB); the digit shifts are then compile-time permutations of registers.
__host__ __device__ constexpr int sub2(int i, int c) {
  return ((i % 3 - c % 3 + 3) % 3) + 3 * ((i / 3 - c / 3 + 3) % 3);
}
__host__ __device__ constexpr int neg2(int i, int c) {
  return ((6 - i % 3 - c % 3) % 3) + 3 * ((6 - i / 3 - c / 3) % 3);
}
template <int C>
__device__ __forceinline__ void gen9(const double2 (&bA)[9], const double2 (&bB)[9], double2 (&r)[9], bool two) {
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const double2 x1 = bA[sub2(i, C)], x2 = bB[neg2(i, C)];
    double2 w;
    w.x = x1.x * x2.x + x1.y * x2.y;
    w.y = x1.x * x2.y - x1.y * x2.x;
    if (two) {
      const double2 y1 = bA[sub2(i, C + 1)], y2 = bB[neg2(i, C + 1)];
      w.x -= y1.x * y2.y - y1.y * y2.x;
      w.y += y1.x * y2.x + y1.y * y2.y;
    }
    r[i] = w;
  }
}

// Staged pass A.  Template S = workspace column-block width (compile-time: the store index
// l -> (l / S, l % S) is a shift).  Per thread: the 3^G consecutive l of group t; per pair the
// shift tables of the two X-strings' low digits, and the shifted upper digits of t.
template <int L, int G, int S>
__global__ void __launch_bounds__(kThreads) k_mana_rowS(RowSArgs A) {
  constexpr int RG = p3(G);
  constexpr int NT = p3(L - G);
  constexpr int NL = p3(L);
  constexpr int NBLK = (NL + S - 1) / S;
  static_assert(NT <= kThreads, "one thread group per thread");
  extern __shared__ double2 smem[];
  double2* rowA = smem;            // psi row (h - a_hi)
  double2* rowB = smem + NL;       // psi row (-h - a_hi)
  double2* tile = smem + 2 * NL;
  const int nh = p3(A.H);
  const int nchunk = (A.npairs + A.PP - 1) / A.PP;
  const long items = (long)nh * nchunk;
  const int t = threadIdx.x;
  // Lane remap (L - G = 5, 243 groups): thread t takes group g = kManaRemap[c][t] for the shift c
  // = a_l1 / 3^G of each pair, so that each quarter-warp's two 9-block loads (blocks shift(g, c),
  // neg(g, c)) and its tile store (9 g + i) hit distinct 16-B bank groups (tools/mana_remap_gen.c,
  // DESIGN.md section 17).  Without it g = t.
  constexpr bool RMP = (L - G == 5) && (G == 2);
  int td[L - G > 0 ? L - G : 1];     // ternary digits of this thread's group index
  auto set_group = [&](int g) {
    int x = g;
#pragma unroll
    for (int j = 0; j < L - G; ++j) {
      td[j] = x % 3;
      x /= 3;
    }
  };
  set_group(t);
  int grp = t;
  for (long it = blockIdx.x; it < items; it += gridDim.x) {
    const int h = (int)(it / nchunk), ch = (int)(it % nchunk);
    const int p_lo = ch * A.PP, p_hi = min(A.npairs, p_lo + A.PP);
    int cur = -1;
    for (int pl = p_lo; pl < p_hi; ++pl) {
      const uint64_t a1 = A.a_begin + 2 * (A.pair0 + pl);
      const bool two = a1 + 1 < A.a_end;
      const int ah1 = (int)(a1 / NL);
      if (ah1 != cur) {                       // (re)stage the two rows this a_hi needs
        __syncthreads();
        int hs, hn;
        tshift_rt(h, ah1, A.H, hs, hn);
        const double2* r1 = A.psi + (size_t)hs * NL;
        const double2* r2 = A.psi + (size_t)hn * NL;
        for (int l = threadIdx.x; l < NL; l += kThreads) {
          rowA[l] = __ldg(r1 + l);
          rowB[l] = __ldg(r2 + l);
        }
        __syncthreads();
        cur = ah1;
      }
      const int al1 = (int)(a1 % NL);
      const uint64_t a2 = a1 + 1;
      const int ah2 = (int)(a2 / NL), al2 = (int)(a2 % NL);
      const bool staged2 = (ah2 == ah1);
      int g2s = 0, g2n = 0;                   // rows for a2 when it crosses an a_hi boundary
      if (two && !staged2) tshift_rt(h, ah2, A.H, g2s, g2n);
      if (t < NT) {
        if constexpr (RMP) {
          if (A.remap) {
            grp = kManaRemap[al1 / RG][t];
            set_group(grp);
          }
        }
        // upper digits: (g - a_up) and (-g - a_up) digit-wise, from the digits of the group g
        int us1 = 0, un1 = 0, us2 = 0, un2 = 0;
        {
          int b1 = al1 / RG, b2 = al2 / RG;
#pragma unroll
          for (int j = 0; j < L - G; ++j) {
            const int c1 = b1 % 3, c2 = b2 % 3, p = p3(j);
            b1 /= 3;
            b2 /= 3;
            us1 += ((td[j] - c1 + 3) % 3) * p;
            un1 += ((6 - td[j] - c1) % 3) * p;
            us2 += ((td[j] - c2 + 3) % 3) * p;
            un2 += ((6 - td[j] - c2) % 3) * p;
          }
        }
        ShiftTab<G> T1, T2;
        T1.build(al1 % RG);
        T2.build(al2 % RG);
        const int oA1 = us1 * RG, oB1 = un1 * RG, oA2 = us2 * RG, oB2 = un2 * RG;
        double2 r[RG];
        bool done = false;
        if constexpr (G == 2) {
          const int c = al1 % 9;
          if (c != 8) {                        // a2's 9-blocks are a1's: one load per block element
            double2 bA[9], bB[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) {
              bA[k] = rowA[oA1 + k];
              bB[k] = rowB[oB1 + k];
            }
            switch (c) {
              case 0: gen9<0>(bA, bB, r, two); break;
              case 1: gen9<1>(bA, bB, r, two); break;
              case 2: gen9<2>(bA, bB, r, two); break;
              case 3: gen9<3>(bA, bB, r, two); break;
              case 4: gen9<4>(bA, bB, r, two); break;
              case 5: gen9<5>(bA, bB, r, two); break;
              case 6: gen9<6>(bA, bB, r, two); break;
              default: gen9<7>(bA, bB, r, two); break;
            }
            done = true;
          }
        }
#pragma unroll
        for (int i = 0; i < RG; ++i) {
          if (done) break;
          int ss1 = 0, sn1 = 0, ss2 = 0, sn2 = 0;
#pragma unroll
          for (int j = 0; j < G; ++j) {
            const int dj = (i / p3(j)) % 3;   // compile-time digit of i
            ss1 += T1.ds[j][dj];
            sn1 += T1.dn[j][dj];
            ss2 += T2.ds[j][dj];
            sn2 += T2.dn[j][dj];
          }
          double2 x1 = rowA[oA1 + ss1];
          double2 x2 = rowB[oB1 + sn1];
          double2 w;
          w.x = x1.x * x2.x + x1.y * x2.y;        // conj(alpha_x) alpha_{-x}
          w.y = x1.x * x2.y - x1.y * x2.x;
          if (two) {
            if (staged2) {
              x1 = rowA[oA2 + ss2];
              x2 = rowB[oB2 + sn2];
            } else {                               // a2 crosses an a_hi boundary (1 pair in 3^L / 2)
              x1 = __ldg(A.psi + (size_t)g2s * NL + oA2 + ss2);
              x2 = __ldg(A.psi + (size_t)g2n * NL + oB2 + sn2);
            }
            w.x -= x1.x * x2.y - x1.y * x2.x;      // + i v2
            w.y += x1.x * x2.x + x1.y * x2.y;
          }
          r[i] = w;
        }
        reg_f3<G>(r);
#pragma unroll
        for (int i = 0; i < RG; ++i) tile[grp * RG + i] = r[i];
      }
      __syncthreads();
      double2* dst = A.ws + (size_t)pl * ((size_t)NBLK * nh * S) + (size_t)h * S;
      const size_t bs = (size_t)nh * S;
      auto to_ws = [&](int l, double2 v) {     // last stage: straight to the column-blocked workspace
        __stcg(dst + (size_t)(l / S) * bs + (l % S), v);
      };
      auto from_tile = [&](int e) { return tile[e]; };
      stages_f<L, 1, G, false>(tile, from_tile, to_ws);
      __syncthreads();
    }
  }
}

struct ColCArgs {
  const double2* ws;    // [pairs][nblk][3^H][S]
  double* slots;
  int npairs;
  int L;
};

// Pass B on the column-blocked workspace: one contiguous 3^H x S tile per item.
template <int H, int S>
__global__ void __launch_bounds__(kThreads) k_mana_colC(ColCArgs A) {
  extern __shared__ double2 tile[];
  constexpr int NH = p3(H);
  constexpr int E = NH * S;
  const int NL = p3(A.L);
  const int nblk = (NL + S - 1) / S;
  const long items = (long)A.npairs * nblk;
  double aa = 0.0, as = 0.0;
  for (long it = blockIdx.x; it < items; it += gridDim.x) {
    const int cb = (int)(it % nblk);
    const int ncol = min(S, NL - cb * S);
    const double2* src = A.ws + (size_t)it * E;
    auto acc = [&](int, double2 v) {
      aa += fabs(v.x) + fabs(v.y);
      as += v.x + v.y;
    };
    if (ncol == S) {                          // first stage straight from the contiguous tile
      auto ld = [&](int e) { return __ldcs(src + e); };
      stages_f<H, S, 0, true>(tile, ld, acc);
    } else {
      auto ld = [&](int e) { return (e % S) < ncol ? __ldcs(src + e) : make_double2(0.0, 0.0); };
      stages_f<H, S, 0, true>(tile, ld, acc);
    }
    __syncthreads();
  }
  flush(aa, as, A.slots);
}

// Pass B with bulk-copy prefetch (H <= 7): each item's contiguous 3^H x S tile arrives by ONE
// cp.async.bulk (41-93 KB) into a 2-deep ring completed on mbarriers, so the next tile's HBM read
// overlaps the current tile's transform.  Ragged last column blocks are zero-filled in smem.
template <int H, int S>
__global__ void __launch_bounds__(kThreads, 1) k_mana_colT(ColCArgs A) {
  extern __shared__ __align__(128) double2 ring[];
  __shared__ __align__(8) uint64_t full[2];
  constexpr int NH = p3(H);
  constexpr int E = NH * S;
  const int NL = p3(A.L);
  const int nblk = (NL + S - 1) / S;
  const long items = (long)A.npairs * nblk;
  if (threadIdx.x == 0) {
    sre::mbar_init(&full[0], 1);
    sre::mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](long it, int slot) {
    sre::mbar_expect_tx(&full[slot], E * (unsigned)sizeof(double2));
    sre::bulk_g2s(ring + (size_t)slot * E, A.ws + (size_t)it * E, E * (unsigned)sizeof(double2), &full[slot]);
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < 2; ++i)
      if (blockIdx.x + (long)i * gridDim.x < items) issue(blockIdx.x + (long)i * gridDim.x, i);
  double aa = 0.0, as = 0.0;
  uint32_t n = 0;
  for (long it = blockIdx.x; it < items; it += gridDim.x, ++n) {
    const int slot = (int)(n & 1u);
    double2* tile = ring + (size_t)slot * E;
    sre::mbar_wait(&full[slot], (n >> 1) & 1u);
    const int cb = (int)(it % nblk);
    const int ncol = min(S, NL - cb * S);
    if (ncol < S) {                                   // columns pass A never wrote
      for (int e = threadIdx.x; e < E; e += kThreads)
        if (e % S >= ncol) tile[e] = make_double2(0.0, 0.0);
      __syncthreads();
    }
    stages<H, S, 0, true>(tile, aa, as);
    __syncthreads();                                  // everyone is done with this slot
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      const long nx = it + 2L * gridDim.x;
      if (nx < items) issue(nx, slot);
    }
  }
  flush(aa, as, A.slots);
}

// Fixed-order sum of the per-CTA slots: out = (S_abs, S_sum).
__global__ void __launch_bounds__(256) k_mana_reduce(const double* slots, int n, double* out) {
  __shared__ double sa[256], ss[256];
  double a = 0.0, s = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) {
    a += slots[2 * i];
    s += slots[2 * i + 1];
  }
  sa[threadIdx.x] = a;
  ss[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      sa[threadIdx.x] += sa[threadIdx.x + o];
      ss[threadIdx.x] += ss[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = sa[0];
    out[1] = ss[0];
  }
}

}  // namespace mana

// ==========================================================================================
// host: planning, launch schedule, C ABI
// ==========================================================================================
namespace {
using namespace sre_host;
using mana::p3;
using mana::kThreads;
using mana::kSlots;

#define MCK(x)                                                                                \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) return fail(SRE_ECUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                   \
  } while (0)

struct MPlan {
  int N = 0, L = 0, H = 0, S = 0;
  bool single = false;
  bool staged = false;    // N = 9..14: k_mana_rowS + k_mana_colC
  int PP = 1;             // pairs per pass-A item (staged)
  size_t row_smem = 0, col_smem = 0;
  size_t row_bytes = 0;   // workspace bytes per pair (3^N complex)
  uint64_t P = 0;         // preferred pairs per launch
};

constexpr size_t kSlotBytes = (size_t)kSlots * 2 * sizeof(double);

void make_mplan(int N, MPlan& m) {
  static const int tab[17][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0},
                                 {0, 0, 0}, {0, 0, 0}, {5, 4, 32}, {6, 4, 32}, {6, 5, 16}, {7, 5, 8},
                                 {7, 6, 4}, {7, 7, 2}, {7, 8, 2}, {8, 8, 2}};
  m.N = N;
  if (N <= 8) {
    m.single = true;
    m.L = N;
    m.H = 0;
  } else {
    m.L = tab[N][0];
    m.H = tab[N][1];
    m.S = tab[N][2];
  }
  if (!m.single) {  // SRE_MANA_PLAN="L,H,S" overrides the split (experiments; must match N)
    const char* e = std::getenv("SRE_MANA_PLAN");
    int l = 0, h = 0, c = 0;
    if (e && std::sscanf(e, "%d,%d,%d", &l, &h, &c) == 3 && l + h == N) {
      m.L = l;
      m.H = h;
      m.S = c;
    }
  }
  m.staged = !m.single && m.L <= 7 && std::getenv("SRE_MANA_UNSTAGED") == nullptr;
  m.row_smem = (size_t)p3(m.L) * sizeof(double2) * (m.staged ? 3 : 1);
  m.col_smem = m.single ? 0 : (size_t)p3(m.H) * m.S * sizeof(double2);
  m.row_bytes = (size_t)p3(N) * sizeof(double2);
  if (m.staged)  // column-blocked: the last block of columns is padded to S
    m.row_bytes = (size_t)((p3(m.L) + m.S - 1) / m.S) * m.S * p3(m.H) * sizeof(double2);
  if (m.single) {
    m.P = 0;
  } else {
    // ~2 GiB of pairs per launch pair (measured: an L2-resident 64 MiB batch
    // loses more to launch tails than it gains in L2 hits; HBM has room for the larger batch).
    uint64_t P = (2ull << 30) / m.row_bytes;
    if (P < 8) P = 8;
    if (const char* e = std::getenv("SRE_MANA_P")) P = (uint64_t)std::atoll(e);   // experiments
    m.P = P < 1 ? 1 : (P > 4096 ? 4096 : P);
    m.PP = m.staged ? 8 : 1;
    if (const char* e = std::getenv("SRE_MANA_PP")) m.PP = std::max(1, std::atoi(e));
  }
}

size_t ws_needed(const MPlan& m, uint64_t P) { return kSlotBytes + (m.single ? 0 : (size_t)P * m.row_bytes); }

using RowFn = void (*)(mana::RowArgs);
using ColFn = void (*)(mana::ColArgs);
using RowSFn = void (*)(mana::RowSArgs);
using ColCFn = void (*)(mana::ColCArgs);

RowSFn rows_fn(int L, int S) {
  switch (L * 100 + S) {
    case 532: return mana::k_mana_rowS<5, 0, 32>;
    case 516: return mana::k_mana_rowS<5, 0, 16>;
    case 632: return mana::k_mana_rowS<6, 1, 32>;
    case 616: return mana::k_mana_rowS<6, 1, 16>;
    case 608: return mana::k_mana_rowS<6, 1, 8>;
    case 716: return mana::k_mana_rowS<7, 2, 16>;
    case 708: return mana::k_mana_rowS<7, 2, 8>;
    case 704: return mana::k_mana_rowS<7, 2, 4>;
    case 702: return mana::k_mana_rowS<7, 2, 2>;
  }
  return nullptr;
}

ColCFn colt_fn(int H, int S) {
  if (H == 4 && S == 32) return mana::k_mana_colT<4, 32>;
  if (H == 5 && S == 16) return mana::k_mana_colT<5, 16>;
  if (H == 5 && S == 8) return mana::k_mana_colT<5, 8>;
  if (H == 6 && S == 8) return mana::k_mana_colT<6, 8>;
  if (H == 6 && S == 4) return mana::k_mana_colT<6, 4>;
  if (H == 7 && S == 4) return mana::k_mana_colT<7, 4>;
  if (H == 7 && S == 2) return mana::k_mana_colT<7, 2>;
  return nullptr;
}

ColCFn colc_fn(int H, int S) {
  if (H == 4 && S == 32) return mana::k_mana_colC<4, 32>;
  if (H == 5 && S == 16) return mana::k_mana_colC<5, 16>;
  if (H == 5 && S == 8) return mana::k_mana_colC<5, 8>;
  if (H == 6 && S == 8) return mana::k_mana_colC<6, 8>;
  if (H == 6 && S == 4) return mana::k_mana_colC<6, 4>;
  if (H == 7 && S == 4) return mana::k_mana_colC<7, 4>;
  if (H == 7 && S == 2) return mana::k_mana_colC<7, 2>;
  if (H == 8 && S == 2) return mana::k_mana_colC<8, 2>;
  return nullptr;
}

RowFn row_fn(int L, bool final_) {
  if (final_) {
    switch (L) {
      case 1: return mana::k_mana_row<1, true>;
      case 2: return mana::k_mana_row<2, true>;
      case 3: return mana::k_mana_row<3, true>;
      case 4: return mana::k_mana_row<4, true>;
      case 5: return mana::k_mana_row<5, true>;
      case 6: return mana::k_mana_row<6, true>;
      case 7: return mana::k_mana_row<7, true>;
      case 8: return mana::k_mana_row<8, true>;
    }
  } else {
    switch (L) {
      case 5: return mana::k_mana_row<5, false>;
      case 6: return mana::k_mana_row<6, false>;
      case 7: return mana::k_mana_row<7, false>;
      case 8: return std::getenv("SRE_MANA_G2") ? mana::k_mana_row<8, false, 2> : mana::k_mana_row<8, false>;
    }
  }
  return nullptr;
}

ColFn col_fn(int H, int S) {
  if (H == 4 && S == 32) return mana::k_mana_col<4, 32>;
  if (H == 4 && S == 16) return mana::k_mana_col<4, 16>;
  if (H == 5 && S == 16) return mana::k_mana_col<5, 16>;
  if (H == 5 && S == 8) return mana::k_mana_col<5, 8>;
  if (H == 6 && S == 8) return mana::k_mana_col<6, 8>;
  if (H == 6 && S == 4) return mana::k_mana_col<6, 4>;
  if (H == 7 && S == 4) return mana::k_mana_col<7, 4>;
  if (H == 7 && S == 2) return mana::k_mana_col<7, 2>;
  if (H == 8 && S == 2) return mana::k_mana_col<8, 2>;
  return nullptr;
}

// resident CTAs per SM for a kernel at its dynamic shared memory (sets the opt-in limit once)
int occupancy(const void* fn, size_t smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, int>> seen;   // (kernel, device) -> CTAs per SM
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0;
  cudaGetDevice(&dev);                          // the smem attribute is per device context
  for (auto& s : seen)
    if (s.first.first == fn && s.first.second == dev) return s.second;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, smem) != cudaSuccess || occ < 1) occ = 1;
  cudaGetLastError();
  seen.push_back({{fn, dev}, occ});
  return occ;
}

int grid_for(long items, int occ, int sms) {
  long g = (long)occ * sms;
  if (g > items) g = items;
  if (g > kSlots) g = kSlots;
  return (int)(g < 1 ? 1 : g);
}

int run_mana(const double2* psi, int N, uint64_t a_begin, uint64_t a_end, char* ws, size_t ws_bytes,
             double* sums_dev, cudaStream_t st) {
  Dev d;
  int rc = get_dev(d);
  if (rc) return rc;
  MPlan m;
  make_mplan(N, m);
  if (ws_bytes < ws_needed(m, 1)) return fail(SRE_EWORKSPACE, "workspace %zu < required %zu", ws_bytes, ws_needed(m, 1));
  double* slots = reinterpret_cast<double*>(ws);
  double2* rows = reinterpret_cast<double2*>(ws + kSlotBytes);
  MCK(cudaMemsetAsync(slots, 0, kSlotBytes, st));
  const uint64_t n_a = a_end - a_begin;
  const uint64_t pairs = (n_a + 1) / 2;
  int used = 0;  // slots touched
  if (pairs > 0) {
    if (m.single) {
      RowFn f = row_fn(m.L, true);
      const int g = grid_for((long)pairs, occupancy((const void*)f, m.row_smem), d.sms);
      used = g;
      for (uint64_t p0 = 0; p0 < pairs; p0 += (1u << 30)) {
        mana::RowArgs A{psi, nullptr, slots, a_begin, a_end, p0, (int)std::min<uint64_t>(pairs - p0, 1u << 30), 0};
        MCK(launch_counted(LK_SINGLE, st, [&] { f<<<g, kThreads, m.row_smem, st>>>(A); return cudaGetLastError(); }));
      }
    } else if (m.staged) {
      uint64_t P = (ws_bytes - kSlotBytes) / m.row_bytes;
      if (P > m.P) P = m.P;
      if (P > pairs) P = pairs;
      RowSFn fa = rows_fn(m.L, m.S);
      ColCFn fb = colc_fn(m.H, m.S);
      size_t smemB = m.col_smem;
      const char* ct = std::getenv("SRE_MANA_COLT");   // SRE_MANA_COLT=0: plain pass B (comparison)
      // measured: pass B 803 -> 628 us per launch at N = 14 (H = 7), neutral at H = 6, slower at H = 5
      if (m.H >= 6 && m.H <= 7 && 2 * m.col_smem <= (size_t)220 * 1024 && !(ct && ct[0] == '0')) {
        ColCFn ft = colt_fn(m.H, m.S);
        if (ft) {
          fb = ft;
          smemB = 2 * m.col_smem;
        }
      }
      if (!fa || !fb) return fail(SRE_EINTERNAL, "no staged mana kernels for N=%d (L=%d H=%d S=%d)", N, m.L, m.H, m.S);
      const int occA = occupancy((const void*)fa, m.row_smem), occB = occupancy((const void*)fb, smemB);
      const int nblk = (p3(m.L) + m.S - 1) / m.S;
      for (uint64_t p0 = 0; p0 < pairs; p0 += P) {
        const int np = (int)std::min<uint64_t>(P, pairs - p0);
        const int PP = std::min(m.PP, np);
        const int gA = grid_for((long)p3(m.H) * ((np + PP - 1) / PP), occA, d.sms);
        const int gB = grid_for((long)np * nblk, occB, d.sms);
        static const int remap = [] { const char* e = std::getenv("SRE_MANA_REMAP"); return (e && e[0] == '0') ? 0 : 1; }();
        mana::RowSArgs A{psi, rows, a_begin, a_end, p0, np, m.H, m.S, PP, remap};
        mana::ColCArgs B{rows, slots, np, m.L};
        MCK(launch_counted(LK_PASSA, st, [&] { fa<<<gA, kThreads, m.row_smem, st>>>(A); return cudaGetLastError(); }));
        MCK(launch_counted(LK_PASSB, st, [&] { fb<<<gB, kThreads, smemB, st>>>(B); return cudaGetLastError(); }));
      }
    } else {
      uint64_t P = (ws_bytes - kSlotBytes) / m.row_bytes;
      if (P > m.P) P = m.P;
      if (P > pairs) P = pairs;
      RowFn fa = row_fn(m.L, false);
      ColFn fb = col_fn(m.H, m.S);
      if (!fa || !fb) return fail(SRE_EINTERNAL, "no mana kernels for N=%d", N);
      const int occA = occupancy((const void*)fa, m.row_smem), occB = occupancy((const void*)fb, m.col_smem);
      const int nblk = (p3(m.L) + m.S - 1) / m.S;
      for (uint64_t p0 = 0; p0 < pairs; p0 += P) {
        const int np = (int)std::min<uint64_t>(P, pairs - p0);
        const int gA = grid_for((long)np * p3(m.H), occA, d.sms);
        const int gB = grid_for((long)np * nblk, occB, d.sms);
        if (gB > used) used = gB;
        mana::RowArgs A{psi, rows, slots, a_begin, a_end, p0, np, m.H};
        mana::ColArgs B{rows, slots, np, m.L};
        MCK(launch_counted(LK_PASSA, st, [&] { fa<<<gA, kThreads, m.row_smem, st>>>(A); return cudaGetLastError(); }));
        MCK(launch_counted(LK_PASSB, st, [&] { fb<<<gB, kThreads, m.col_smem, st>>>(B); return cudaGetLastError(); }));
      }
    }
  }
  MCK(launch_counted(LK_AUX, st, [&] { mana::k_mana_reduce<<<1, 256, 0, st>>>(slots, kSlots, sums_dev); return cudaGetLastError(); }));
  (void)used;
  return SRE_OK;
}

struct MCache {
  std::mutex mu;
  char* ws = nullptr;
  size_t ws_bytes = 0;
  char* in = nullptr;
  size_t in_bytes = 0;
  int dev = -1;
};
MCache g_mcache;

int mcache_get(char** buf, size_t* have, size_t need) {
  if (*have >= need) return SRE_OK;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  *have = 0;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(buf), need);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(SRE_ENOMEM, "cudaMalloc(%zu): %s", need, cudaGetErrorString(e));
  }
  *have = need;
  return SRE_OK;
}

uint64_t pow3u(int n) {
  uint64_t r = 1;
  for (int i = 0; i < n; ++i) r *= 3;
  return r;
}

}  // namespace

extern "C" {

size_t sre_mana_workspace_size(int N) {
  if (N < 1 || N > SRE_MANA_MAX_N) return 0;
  MPlan m;
  make_mplan(N, m);
  return ws_needed(m, m.P);
}

int sre_mana_partial_sums(const void* psi, int N, uint64_t a_begin, uint64_t a_end, void* workspace,
                          size_t ws_bytes, double* sums_dev, void* stream) {
  if (!psi) return fail(SRE_EINVAL, "psi is NULL");
  if (N < 1 || N > SRE_MANA_MAX_N) return fail(SRE_ERANGE, "N=%d outside [1, %d]", N, SRE_MANA_MAX_N);
  if (a_begin > a_end || a_end > pow3u(N)) return fail(SRE_ERANGE, "X-string range [%llu, %llu) outside [0, 3^%d]",
                                                      (unsigned long long)a_begin, (unsigned long long)a_end, N);
  if (!workspace) return fail(SRE_EINVAL, "workspace is NULL");
  if (!sums_dev) return fail(SRE_EINVAL, "sums_dev is NULL");
  if (reinterpret_cast<uintptr_t>(psi) % 16) return fail(SRE_EINVAL, "psi not 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return fail(SRE_EINVAL, "workspace not 256-byte aligned");
  bool dv = false;
  int rc = is_device_ptr(psi, dv);
  if (rc) return rc;
  if (!dv) return fail(SRE_EINVAL, "psi must be a device pointer");
  return run_mana(reinterpret_cast<const double2*>(psi), N, a_begin, a_end, reinterpret_cast<char*>(workspace),
                  ws_bytes, sums_dev, reinterpret_cast<cudaStream_t>(stream));
}

int sre_mana_finalize(const double* sums_host, int N, double* out_mana, double* out_norm2) {
  if (!sums_host || !out_mana) return fail(SRE_EINVAL, "NULL argument");
  if (N < 1 || N > SRE_MANA_MAX_N) return fail(SRE_ERANGE, "N=%d outside [1, %d]", N, SRE_MANA_MAX_N);
  const double D = std::pow(3.0, N);                      // exact for N <= 16 (3^16 < 2^53)
  if (!(sums_host[0] > 0.0)) return fail(SRE_EINVAL, "S_abs = %.17g is not positive", sums_host[0]);
  *out_mana = std::log2(sums_host[0] / D);                // Eq. (10): log2(sum_u |W_u|) = log2(S_abs / 3^N)
  if (out_norm2) *out_norm2 = sums_host[1] / D;           // S_sum = 3^N ||psi||^2
  return SRE_OK;
}

int sre_mana(const void* psi, int N, double* out_mana, double* out_norm2) {
  if (!psi) return fail(SRE_EINVAL, "psi is NULL");
  if (N < 1 || N > SRE_MANA_MAX_N) return fail(SRE_ERANGE, "N=%d outside [1, %d]", N, SRE_MANA_MAX_N);
  if (!out_mana) return fail(SRE_EINVAL, "out_mana is NULL");
  if (reinterpret_cast<uintptr_t>(psi) % 16) return fail(SRE_EINVAL, "psi not 16-byte aligned");
  Dev d;
  int rc = get_dev(d);
  if (rc) return rc;
  bool dev_ptr = false;
  rc = is_device_ptr(psi, dev_ptr);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(g_mcache.mu);
  if (g_mcache.dev != d.id) {
    g_mcache.ws = nullptr; g_mcache.ws_bytes = 0; g_mcache.in = nullptr; g_mcache.in_bytes = 0; g_mcache.dev = d.id;
  }
  MPlan m;
  make_mplan(N, m);
  const uint64_t D = pow3u(N);
  const size_t need = ws_needed(m, m.P) + 256;
  rc = mcache_get(&g_mcache.ws, &g_mcache.ws_bytes, need);
  if (rc) return rc;
  cudaStream_t st = 0;
  const double2* dpsi = reinterpret_cast<const double2*>(psi);
  if (!dev_ptr) {
    rc = mcache_get(&g_mcache.in, &g_mcache.in_bytes, D * sizeof(double2));
    if (rc) return rc;
    MCK(cudaMemcpyAsync(g_mcache.in, psi, D * sizeof(double2), cudaMemcpyHostToDevice, st));
    dpsi = reinterpret_cast<const double2*>(g_mcache.in);
  }
  double* sums = reinterpret_cast<double*>(g_mcache.ws + ws_needed(m, m.P));
  rc = run_mana(dpsi, N, 0, D, g_mcache.ws, ws_needed(m, m.P), sums, st);
  if (rc) return rc;
  double hs[2];
  MCK(cudaMemcpyAsync(hs, sums, sizeof(hs), cudaMemcpyDeviceToHost, st));
  MCK(cudaStreamSynchronize(st));
  const double n2 = hs[1] / (double)D;   // sum_u <psi|A_u|psi> = 3^N ||psi||^2
  if (out_norm2) *out_norm2 = n2;
  if (!(std::fabs(n2 - 1.0) <= 1e-8)) return fail(SRE_ENOTNORM, "||psi||^2 = %.17g", n2);
  *out_mana = std::log2(hs[0] / (double)D);
  return SRE_OK;
}

}  // extern "C"
