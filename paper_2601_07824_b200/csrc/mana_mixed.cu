// mana_mixed.cu -- mixed-state qutrit mana (NEXT-4): Algorithm 6 of PAPER.md on sm_100a.
//
// w = M^{(x)N} Vec_N(rho) (Eq. (45)), w_u = Tr(rho A_u), mana = log2(sum_u |w_u| / 3^N) (DESIGN C18,
// C20).  The single-qutrit map M acts on the nine entries rho_{rc} of one leg as
//     w_{(a,b)} = omega^{2ab} sum_r omega^{a r} rho_{r, 2b-r}
// i.e. three 3-point DFTs on the lines r + c = 2b (the F_3 (+) F_3 (+) F_3 structure of P:971-982)
// and a unit phase.  B200 design:
//  * No Vec_N reorder: the leg sweep runs in place on the column-major rho the caller provides
//    (rho[r + c 3^N]); leg k is the ternary digit pair (k, N + k) of the flat index.
//  * HBM-bound (9^N complex128 = 56 GB at N = 10): several legs are fused per pass on a shared-
//    memory tile of <= 6561 elements: pass 1 covers legs 0..3 (contiguous 81-element runs), later
//    passes 3 legs each with 9 contiguous spectator elements (r digits 0, 1) per run.  N = 10
//    therefore costs 3 HBM round trips instead of the 10 of a leg-by-leg sweep; the last pass
//    accumulates sum |Re w| and sum Re w instead of storing w.
//  * Persistent grids, per-CTA FP64 slots in launch order, a fixed-order reduction (deterministic).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/sre.h"
#include "launch.cuh"

namespace sre_host {
int fail(int code, const char* fmt, ...);
int get_dev(Dev& d);
int is_device_ptr(const void* ptr, bool& dev);
}  // namespace sre_host

namespace mixed {
using sre::mbar_expect_tx;
using sre::mbar_init;
using sre::mbar_wait;
using sre::smem_u32;

__host__ __device__ constexpr long p3(int k) {
  long r = 1;
  for (int i = 0; i < k; ++i) r *= 3;
  return r;
}

constexpr int kThreads = 256;
constexpr int kSlots = 4096;
constexpr double kC = 0.86602540378443864676;   // sqrt(3)/2

__device__ __forceinline__ double2 mul_w(double2 v) {   // v * omega, omega = (-1/2, sqrt3/2)
  return make_double2(fma(-0.5, v.x, -kC * v.y), fma(kC, v.x, -0.5 * v.y));
}
__device__ __forceinline__ double2 mul_w2(double2 v) {  // v * omega^2 = v * (-1/2, -sqrt3/2)
  return make_double2(fma(-0.5, v.x, kC * v.y), fma(-kC, v.x, -0.5 * v.y));
}

// One leg: x[r][c] = rho_{rc} of the fiber -> x[a][b] = w_{(a,b)}.
__device__ __forceinline__ void leg9(double2 (&x)[3][3]) {
  double2 y[3][3];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const double2 x0 = x[0][(2 * b) % 3], x1 = x[1][(2 * b + 2) % 3], x2 = x[2][(2 * b + 1) % 3];
    const double sr = x1.x + x2.x, si = x1.y + x2.y;
    const double dr = x1.x - x2.x, di = x1.y - x2.y;
    const double tr = fma(-0.5, sr, x0.x), ti = fma(-0.5, si, x0.y);
    const double2 z0 = make_double2(x0.x + sr, x0.y + si);
    const double2 z1 = make_double2(fma(-kC, di, tr), fma(kC, dr, ti));   // t + i c d
    const double2 z2 = make_double2(fma(kC, di, tr), fma(-kC, dr, ti));   // t - i c d
    y[0][b] = z0;
    // a = 1: omega^{2b};  a = 2: omega^{4b} = omega^{b}
    y[1][b] = (b == 0) ? z1 : (b == 1 ? mul_w2(z1) : mul_w(z1));
    y[2][b] = (b == 0) ? z2 : (b == 1 ? mul_w(z2) : mul_w2(z2));
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) x[a][b] = y[a][b];
}

// Leg J of a tile with SP spectator digits and NL legs: tile element e = s + 3^SP (R + 3^NL C),
// global element base + s + R sR + C sC.  LDG: the fiber is read from global memory (first leg),
// STG: written to global memory (last leg of a non-final pass), ACC: accumulated (last leg of the
// final pass); otherwise shared memory.
template <int SP, int NL, int J, bool LDG, bool STG, bool ACC, int NT>
__device__ __forceinline__ void leg_stage(double2* tile, double2* g, long base, long sR, long sC, double& aa,
                                          double& as) {
  constexpr int S3 = (int)p3(SP), R3 = (int)p3(NL), PJ = (int)p3(J), PH = (int)p3(NL - 1 - J);
  constexpr int sr = S3 * PJ, sc = S3 * R3 * PJ;
  constexpr int fibers = S3 * (int)p3(NL - 1) * (int)p3(NL - 1);
  const long gr = PJ * sR, gc = PJ * sC;
#pragma unroll 2
  for (int f = threadIdx.x; f < fibers; f += NT) {
    int q = f;
    const int s = q % S3;
    q /= S3;
    int rlo, rhi;
    if constexpr (SP == 0 && J == 1) {   // stride-9 fibers first: 8 consecutive threads hit 8 banks
      rhi = q % PH;
      q /= PH;
      rlo = q % PJ;
      q /= PJ;
    } else {
      rlo = q % PJ;
      q /= PJ;
      rhi = q % PH;
      q /= PH;
    }
    const int clo = q % PJ;
    q /= PJ;
    const int chi = q;
    const int tb = s + S3 * (rlo + PJ * 3 * rhi + R3 * (clo + PJ * 3 * chi));
    const long gb = base + s + (long)(rlo + PJ * 3 * rhi) * sR + (long)(clo + PJ * 3 * chi) * sC;
    double2 x[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if constexpr (LDG) x[r][c] = __ldg(g + gb + r * gr + c * gc);
        else x[r][c] = tile[tb + r * sr + c * sc];
      }
    leg9(x);
    if constexpr (ACC) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          aa += fabs(x[a][b].x);
          as += x[a][b].x;
        }
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          if constexpr (STG) __stcs(g + gb + a * gr + b * gc, x[a][b]);
          else tile[tb + a * sr + b * sc] = x[a][b];
        }
    }
  }
}

// SMEM: the tile arrives in shared memory and (unless FINAL) leaves from it (k_legs_tma, TMA)
template <int SP, int NL, int J, bool FINAL, int NT, bool SMEM = false>
__device__ __forceinline__ void leg_stages(double2* tile, double2* g, long base, long sR, long sC, double& aa,
                                           double& as) {
  if constexpr (J < NL) {
    constexpr bool first = (J == 0) && !SMEM, last = (J == NL - 1);
    leg_stage<SP, NL, J, first, last && !FINAL && !SMEM, last && FINAL, NT>(tile, g, base, sR, sC, aa, as);
    __syncthreads();
    leg_stages<SP, NL, J + 1, FINAL, NT, SMEM>(tile, g, base, sR, sC, aa, as);
  }
}

__device__ __forceinline__ void flush(double aa, double as, double* slots) {
  __shared__ double red[2][16];
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
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      ta += red[0][i];
      ts += red[1][i];
    }
    slots[2 * blockIdx.x] += ta;
    slots[2 * blockIdx.x + 1] += ts;
  }
}

struct LegArgs {
  double2* rho;         // column-major 3^N x 3^N, transformed in place
  double* slots;
  int N;
  int k0;               // first leg of this pass
  long items;           // 9^N / (3^SP 9^NL)
};

// One pass: legs k0 .. k0+NL-1 on tiles of 3^SP x 9^NL elements.  Free digits (the item index,
// fastest first): r digits [SP, k0), r digits [k0+NL, N), c digits [0, k0), c digits [k0+NL, N).
template <int SP, int NL, bool FINAL, int NT = kThreads>
__global__ void __launch_bounds__(NT) k_legs(LegArgs A) {
  constexpr int S3 = (int)p3(SP);
  extern __shared__ double2 tile[];
  const int N = A.N, k0 = A.k0;
  const long nrl = p3(k0 - SP), nrh = p3(N - k0 - NL), ncl = p3(k0);
  const long sR = p3(k0), sC = p3(N + k0);
  const long pRH = p3(k0 + NL), pCL = p3(N), pCH = p3(N + k0 + NL);
  double aa = 0.0, as = 0.0;
  if constexpr (NL == 1) {       // one leg: no tile, every thread owns one fiber of some item
    const long nf = A.items * S3;
    for (long F = (long)blockIdx.x * NT + threadIdx.x; F < nf; F += (long)gridDim.x * NT) {
      const long s = F % S3;
      long x = F / S3;
      const long rl = x % nrl;
      x /= nrl;
      const long rh = x % nrh;
      x /= nrh;
      const long cl = x % ncl;
      x /= ncl;
      const long gb = s + rl * S3 + rh * pRH + cl * pCL + x * pCH;
      double2 v[3][3];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) v[r][c] = __ldcs(A.rho + gb + r * sR + c * sC);
      leg9(v);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          if constexpr (FINAL) {
            aa += fabs(v[a][b].x);
            as += v[a][b].x;
          } else {
            __stcs(A.rho + gb + a * sR + b * sC, v[a][b]);
          }
        }
    }
  } else {
    for (long it = blockIdx.x; it < A.items; it += gridDim.x) {
      long x = it;
      const long rl = x % nrl;
      x /= nrl;
      const long rh = x % nrh;
      x /= nrh;
      const long cl = x % ncl;
      x /= ncl;
      const long base = rl * S3 + rh * pRH + cl * pCL + x * pCH;
      leg_stages<SP, NL, 0, FINAL, NT>(tile, A.rho, base, sR, sC, aa, as);   // ends with __syncthreads
    }
  }
  if constexpr (FINAL) flush(aa, as, A.slots);
}

// Tile passes with TMA tiles (k_legs_tma).  The pass (SP, NL, k0) tile is one tensor box of the
// column-major rho viewed as a 5-D tensor (fastest first):
//     d0 = (r digits [0, SP), re/im)  extent 2 3^SP doubles         box 2 3^SP
//     d1 = r digits [SP, k0)           extent 3^(k0-SP)              box 1
//     d2 = r digits [k0, N)            extent 3^(N-k0)               box 3^NL (the row legs)
//     d3 = c digits [0, k0)            extent 3^k0                   box 1
//     d4 = c digits [k0, N)            extent 3^(N-k0)               box 3^NL (the column legs)
// whose shared-memory image is exactly tile[s + 3^SP (R + 3^NL C)] (R5); the first pass (k0 = 0,
// SP = 0) is the 2-D view {2 3^N doubles, 3^N columns}, box {2 3^NL, 3^NL} (contiguous 81-element
// runs).  Item it = rl + nrl (rh + nrh (cl + ncl ch)) as in k_legs.  Persistent CTAs double-buffer
// the tiles: item n + 1's box lands while item n runs its legs in shared memory; a non-final pass
// stores the tile with one TMA tensor store, and the buffer is reloaded once that store has read it.
__host__ __device__ constexpr int tile_elems(int SP, int NL) { return (int)p3(SP) * (int)p3(2 * NL); }
__host__ __device__ constexpr int tile_stride(int SP, int NL) { return (tile_elems(SP, NL) + 7) & ~7; }   // 128-B aligned

template <bool R5>
__device__ __forceinline__ void tma_tile_load(void* dst, const CUtensorMap* tm, const int (&c)[5], uint64_t* bar) {
  if constexpr (R5)
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n"
                 ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]),
                 "r"(c[4]), "r"(smem_u32(bar)) : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                 ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c[0]), "r"(c[1]), "r"(smem_u32(bar))
                 : "memory");
}
template <bool R5>
__device__ __forceinline__ void tma_tile_store(const CUtensorMap* tm, const int (&c)[5], const void* src) {
  if constexpr (R5)
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n"
                 ::"l"(reinterpret_cast<uint64_t>(tm)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]),
                 "r"(smem_u32(src)) : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n"
                 ::"l"(reinterpret_cast<uint64_t>(tm)), "r"(c[0]), "r"(c[1]), "r"(smem_u32(src)) : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}

__device__ __forceinline__ constexpr int ord81(int J, int i) {
  constexpr int o[4][6] = {{5, 6, 7, 2, 1, 3}, {4, 7, 6, 3, 0, 2}, {5, 4, 7, 0, 1, 3}, {4, 5, 6, 1, 0, 2}};
  return o[J][i];
}
template <int J, int NT>
__device__ __forceinline__ void leg81(double2* tile) {
  constexpr int PJ = (int)p3(J), sr = PJ, sc = 81 * PJ;
#pragma unroll 2
  for (int f = threadIdx.x; f < 729; f += NT) {
    int q = f, tb = 0;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const int d = q % 3, k = ord81(J, i);
      q /= 3;
      tb += d * (k < 4 ? (int)p3(k) : 81 * (int)p3(k - 4));
    }
    double2 x[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) x[r][c] = tile[tb + r * sr + c * sc];
    leg9(x);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) tile[tb + a * sr + b * sc] = x[a][b];
  }
  __syncthreads();
}

template <int SP, int NL, bool FINAL, bool R5, int NT>
__global__ void __launch_bounds__(NT) k_legs_tma(LegArgs A, const __grid_constant__ CUtensorMap tm) {
  constexpr int E = tile_elems(SP, NL), TS = tile_stride(SP, NL), B3 = (int)p3(NL);
  extern __shared__ __align__(128) double2 tbuf[];
  __shared__ __align__(8) uint64_t full[2];
  const int N = A.N, k0 = A.k0;
  const long nrl = p3(k0 - SP), nrh = p3(N - k0 - NL), ncl = p3(k0);
  const long items = A.items;
  auto coords = [&](long it, int (&c)[5]) {
    const long rl = it % nrl;
    long x = it / nrl;
    const long rh = x % nrh;
    x /= nrh;
    const long cl = x % ncl, ch = x / ncl;
    if constexpr (R5) {
      c[0] = 0;
      c[1] = (int)rl;
      c[2] = (int)(B3 * rh);
      c[3] = (int)cl;
      c[4] = (int)(B3 * ch);
    } else {
      c[0] = (int)(2 * B3 * rh);
      c[1] = (int)(B3 * ch);
      c[2] = c[3] = c[4] = 0;
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const long it = blockIdx.x + (long)b * gridDim.x;
      if (it < items) {
        int c[5];
        coords(it, c);
        mbar_expect_tx(&full[b], E * sizeof(double2));
        tma_tile_load<R5>(tbuf + b * TS, &tm, c, &full[b]);
      }
    }
  }
  __syncthreads();
  double aa = 0.0, as = 0.0;
  int n = 0;
  for (long it = blockIdx.x; it < items; it += gridDim.x, ++n) {
    const int b = n & 1;
    double2* tile = tbuf + b * TS;
    mbar_wait(&full[b], (n >> 1) & 1);
    if constexpr (SP == 0 && NL == 4 && !FINAL) {
      leg81<0, NT>(tile);
      leg81<1, NT>(tile);
      leg81<2, NT>(tile);
      leg81<3, NT>(tile);
    } else {
      leg_stages<SP, NL, 0, FINAL, NT, true>(tile, A.rho, 0, 0, 0, aa, as);
    }                                      // both end with __syncthreads: every thread is done with tile
    if (threadIdx.x == 0) {
      int c[5];
      if constexpr (!FINAL) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic writes -> TMA reads
        coords(it, c);
        tma_tile_store<R5>(&tm, c, tile);
      }
      const long nx = it + 2 * (long)gridDim.x;
      if (nx < items) {
        if constexpr (!FINAL) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");   // store read buffer b
        coords(nx, c);
        mbar_expect_tx(&full[b], E * sizeof(double2));
        tma_tile_load<R5>(tile, &tm, c, &full[b]);
      }
    }
  }
  if constexpr (FINAL) flush(aa, as, A.slots);
  else if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

__global__ void __launch_bounds__(256) k_mixed_reduce(const double* slots, int n, double* out) {
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

}  // namespace mixed

// ==========================================================================================
// host
// ==========================================================================================
namespace {
using namespace sre_host;
using mixed::kSlots;
using mixed::kThreads;

#define XCK(x)                                                                                \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) return fail(SRE_ECUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                   \
  } while (0)

constexpr size_t kSlotBytes = (size_t)kSlots * 2 * sizeof(double);

struct Pass {
  int SP, NL, k0;
};

// Default: legs 0..3 on contiguous 81 x 81 tiles, then 3 legs per pass with 9 spectators.
// SRE_MIXED_PLAN="SP:NL,SP:NL,..." overrides (experiments).
std::vector<Pass> make_passes(int N) {
  std::vector<Pass> v;
  const char* e = std::getenv("SRE_MIXED_PLAN");
  if (e) {
    int k0 = 0;
    const char* p = e;
    while (*p && k0 < N) {
      int sp = 0, nl = 0, used = 0;
      if (std::sscanf(p, "%d:%d%n", &sp, &nl, &used) != 2) break;
      const bool ok = nl >= 1 && nl <= 4 && sp >= 0 && sp <= 4 && sp <= k0 && mixed::p3(sp) * mixed::p3(2 * nl) <= 6561;
      if (!ok) break;
      v.push_back({sp, nl, k0});
      k0 += nl;
      p += used;
      if (*p == ',') ++p;
    }
    if (k0 == N) return v;
    v.clear();
  }
  // measured on B200: after the 81 x 81 pass, 3-leg passes with 9-element
  // runs; a remainder of 1, 2 or 4 legs goes to 27-element-run passes (a read-only final pass
  // with 27-element runs is 2x faster than one with 9-element runs).
  const int first = N < 4 ? N : 4;
  v.push_back({0, first, 0});
  int k0 = first;
  int rem = N - k0;
  while (rem > 0) {
    const int nl = (rem == 4 || rem == 2) ? 2 : (rem >= 3 ? 3 : 1);
    v.push_back({nl == 3 ? 2 : 3, nl, k0});
    k0 += nl;
    rem -= nl;
  }
  return v;
}

using LegFn = void (*)(mixed::LegArgs);

template <bool F>
LegFn leg_fn_t(int sp, int nl) {
  switch (sp * 10 + nl) {
    case 1: return mixed::k_legs<0, 1, F>;
    case 2: return mixed::k_legs<0, 2, F>;
    case 3: return mixed::k_legs<0, 3, F>;
    case 4: return mixed::k_legs<0, 4, F>;
    case 21: return mixed::k_legs<2, 1, F>;
    case 22: return mixed::k_legs<2, 2, F>;
    case 23: return mixed::k_legs<2, 3, F>;
    case 31: return mixed::k_legs<3, 1, F>;
    case 32: return mixed::k_legs<3, 2, F>;
    case 41: return mixed::k_legs<4, 1, F>;
    case 42: return mixed::k_legs<4, 2, F>;
  }
  return nullptr;
}
LegFn leg_fn(int sp, int nl, bool fin, int threads) {
  if (threads == 512 && sp == 0 && nl == 4) return fin ? mixed::k_legs<0, 4, true, 512> : mixed::k_legs<0, 4, false, 512>;
  return fin ? leg_fn_t<true>(sp, nl) : leg_fn_t<false>(sp, nl);
}

int occupancy(const void* fn, size_t smem, int threads) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, int>> seen;   // (kernel, device) -> CTAs per SM
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0;
  cudaGetDevice(&dev);                          // the smem attribute is per device context
  for (auto& s : seen)
    if (s.first.first == fn && s.first.second == dev) return s.second;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess || occ < 1) occ = 1;
  cudaGetLastError();
  seen.push_back({{fn, dev}, occ});
  return occ;
}

bool use_tma() {   // SRE_MIXED_TMA=0: the LDG/STG k_legs tile passes (A/B measurements)
  const char* e = std::getenv("SRE_MIXED_TMA");
  return !(e && std::atoi(e) == 0);
}

using TmaFn = void (*)(mixed::LegArgs, CUtensorMap);
template <bool F>
TmaFn tma_fn_t(int sp, int nl, bool r5) {
  if (!r5) {   // first pass: the 2-D view
    switch (sp * 10 + nl) {
      case 2: return mixed::k_legs_tma<0, 2, F, false, kThreads>;
      case 3: return mixed::k_legs_tma<0, 3, F, false, kThreads>;
      case 4: return mixed::k_legs_tma<0, 4, F, false, kThreads>;
    }
    return nullptr;
  }
  switch (sp * 10 + nl) {
    case 2: return mixed::k_legs_tma<0, 2, F, true, kThreads>;
    case 3: return mixed::k_legs_tma<0, 3, F, true, kThreads>;
    case 4: return mixed::k_legs_tma<0, 4, F, true, kThreads>;
    case 22: return mixed::k_legs_tma<2, 2, F, true, kThreads>;
    case 23: return mixed::k_legs_tma<2, 3, F, true, kThreads>;
    case 32: return mixed::k_legs_tma<3, 2, F, true, kThreads>;
    case 42: return mixed::k_legs_tma<4, 2, F, true, kThreads>;
  }
  return nullptr;
}
size_t tma_smem(int sp, int nl) { return 2 * (size_t)((mixed::p3(sp) * mixed::p3(2 * nl) + 7) & ~7L) * sizeof(double2); }

// One tile pass with TMA tiles (k_legs_tma); returns -1 when no instance covers (SP, NL).
int launch_legs_tma(const Pass& p, bool fin, double2* rho, int N, double* slots, const Dev& d, cudaStream_t st) {
  const bool r5 = p.k0 > 0;
  TmaFn f = fin ? tma_fn_t<true>(p.SP, p.NL, r5) : tma_fn_t<false>(p.SP, p.NL, r5);
  if (!f) return -1;
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SRE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t D = (cuuint64_t)mixed::p3(N), S3 = (cuuint64_t)mixed::p3(p.SP), B3 = (cuuint64_t)mixed::p3(p.NL);
  CUtensorMap tm;
  CUresult cr;
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUtensorMapL2promotion l2p = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;   // best of 0/64/128/256 on x10
  if (const char* e = std::getenv("SRE_MIXED_L2P")) {   // experiments: 0, 64, 128, 256
    const int v = std::atoi(e);
    l2p = v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
        : v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  }
  if (r5) {
    const cuuint64_t K0 = (cuuint64_t)mixed::p3(p.k0);
    const cuuint64_t dims[5] = {2 * S3, K0 / S3, D / K0, K0, D / K0};
    const cuuint64_t strides[4] = {S3 * 16, K0 * 16, D * 16, D * K0 * 16};   // bytes, dims 1..4
    const cuuint32_t box[5] = {(cuuint32_t)(2 * S3), 1, (cuuint32_t)B3, 1, (cuuint32_t)B3};
    cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, rho, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, l2p, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[2] = {2 * D, D};
    const cuuint64_t strides[1] = {D * 16};
    const cuuint32_t box[2] = {(cuuint32_t)(2 * B3), (cuuint32_t)B3};
    cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, rho, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, l2p, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (cr != CUDA_SUCCESS) return fail(SRE_ECUDA, "cuTensorMapEncodeTiled failed (N=%d SP=%d NL=%d k0=%d)", N, p.SP, p.NL, p.k0);
  const size_t smem = tma_smem(p.SP, p.NL);
  const long items = mixed::p3(2 * N) / (mixed::p3(p.SP) * mixed::p3(2 * p.NL));
  long g = (long)occupancy((const void*)f, smem, kThreads) * d.sms;
  if (g > items) g = items;
  if (g > kSlots) g = kSlots;
  const int grid = (int)g;
  mixed::LegArgs A{rho, slots, N, p.k0, items};
  XCK(launch_counted(fin ? LK_PASSB : LK_PASSA, st, [&] { f<<<grid, kThreads, smem, st>>>(A, tm); return cudaGetLastError(); }));
  return SRE_OK;
}

int run_mixed(double2* rho, int N, char* ws, size_t ws_bytes, double* sums_dev, cudaStream_t st) {
  Dev d;
  int rc = get_dev(d);
  if (rc) return rc;
  if (ws_bytes < kSlotBytes) return fail(SRE_EWORKSPACE, "workspace %zu < required %zu", ws_bytes, kSlotBytes);
  double* slots = reinterpret_cast<double*>(ws);
  XCK(cudaMemsetAsync(slots, 0, kSlotBytes, st));
  const std::vector<Pass> passes = make_passes(N);
  for (size_t i = 0; i < passes.size(); ++i) {
    const Pass& p = passes[i];
    const bool fin = (i + 1 == passes.size());
    if (p.NL > 1 && use_tma()) {
      rc = launch_legs_tma(p, fin, rho, N, slots, d, st);
      if (rc >= 0) {
        if (rc) return rc;
        continue;
      }
    }
    int threads = kThreads;
    if (p.SP == 0 && p.NL == 4) {
      const char* e = std::getenv("SRE_MIXED_T0");   // experiments: threads of the 81 x 81 pass
      if (e && std::atoi(e) == 512) threads = 512;
    }
    LegFn f = leg_fn(p.SP, p.NL, fin, threads);
    if (!f || p.k0 < p.SP) return fail(SRE_EINTERNAL, "no leg kernel for SP=%d NL=%d k0=%d", p.SP, p.NL, p.k0);
    const long E = mixed::p3(p.SP) * mixed::p3(2 * p.NL);
    const size_t smem = p.NL == 1 ? 0 : (size_t)E * sizeof(double2);
    const long items = mixed::p3(2 * N) / E;
    const long work = p.NL == 1 ? (items * mixed::p3(p.SP) + threads - 1) / threads : items;
    long g = (long)occupancy((const void*)f, smem, threads) * d.sms;
    if (g > work) g = work;
    if (g > kSlots) g = kSlots;
    mixed::LegArgs A{rho, slots, N, p.k0, items};
    const int grid = (int)g;
    XCK(launch_counted(fin ? LK_PASSB : LK_PASSA, st, [&] { f<<<grid, threads, smem, st>>>(A); return cudaGetLastError(); }));
  }
  XCK(launch_counted(LK_AUX, st, [&] { mixed::k_mixed_reduce<<<1, 256, 0, st>>>(slots, kSlots, sums_dev); return cudaGetLastError(); }));
  return SRE_OK;
}

struct XCache {
  std::mutex mu;
  char* buf = nullptr;
  size_t bytes = 0;
  int dev = -1;
};
XCache g_xcache;

uint64_t pow3u(int n) {
  uint64_t r = 1;
  for (int i = 0; i < n; ++i) r *= 3;
  return r;
}

}  // namespace

extern "C" {

size_t sre_mana_mixed_workspace_size(int N) {
  if (N < 1 || N > SRE_MANA_MIXED_MAX_N) return 0;
  return kSlotBytes;
}

int sre_mana_mixed_sums(void* rho, int N, void* workspace, size_t ws_bytes, double* sums_dev, void* stream) {
  if (!rho) return fail(SRE_EINVAL, "rho is NULL");
  if (N < 1 || N > SRE_MANA_MIXED_MAX_N) return fail(SRE_ERANGE, "N=%d outside [1, %d]", N, SRE_MANA_MIXED_MAX_N);
  if (!workspace) return fail(SRE_EINVAL, "workspace is NULL");
  if (!sums_dev) return fail(SRE_EINVAL, "sums_dev is NULL");
  if (reinterpret_cast<uintptr_t>(rho) % 16) return fail(SRE_EINVAL, "rho not 16-byte aligned");
  bool dv = false;
  int rc = is_device_ptr(rho, dv);
  if (rc) return rc;
  if (!dv) return fail(SRE_EINVAL, "rho must be a device pointer");
  return run_mixed(reinterpret_cast<double2*>(rho), N, reinterpret_cast<char*>(workspace), ws_bytes, sums_dev,
                   reinterpret_cast<cudaStream_t>(stream));
}

int sre_mana_mixed(const void* rho, int N, double* out_mana, double* out_trace) {
  if (!rho) return fail(SRE_EINVAL, "rho is NULL");
  if (N < 1 || N > SRE_MANA_MIXED_MAX_N) return fail(SRE_ERANGE, "N=%d outside [1, %d]", N, SRE_MANA_MIXED_MAX_N);
  if (!out_mana) return fail(SRE_EINVAL, "out_mana is NULL");
  if (reinterpret_cast<uintptr_t>(rho) % 16) return fail(SRE_EINVAL, "rho not 16-byte aligned");
  Dev d;
  int rc = get_dev(d);
  if (rc) return rc;
  bool dev_ptr = false;
  rc = is_device_ptr(rho, dev_ptr);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(g_xcache.mu);
  if (g_xcache.dev != d.id) {
    g_xcache.buf = nullptr;
    g_xcache.bytes = 0;
    g_xcache.dev = d.id;
  }
  const uint64_t D = pow3u(N);
  const size_t vbytes = (size_t)(D * D) * sizeof(double2);
  const size_t need = vbytes + kSlotBytes + 256;
  if (g_xcache.bytes < need) {
    if (g_xcache.buf) cudaFree(g_xcache.buf);
    g_xcache.buf = nullptr;
    g_xcache.bytes = 0;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&g_xcache.buf), need);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(SRE_ENOMEM, "cudaMalloc(%zu): %s", need, cudaGetErrorString(e));
    }
    g_xcache.bytes = need;
  }
  cudaStream_t st = 0;
  double2* v = reinterpret_cast<double2*>(g_xcache.buf);
  XCK(cudaMemcpyAsync(v, rho, vbytes, dev_ptr ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  char* ws = g_xcache.buf + vbytes;
  double* sums = reinterpret_cast<double*>(ws + kSlotBytes);
  rc = run_mixed(v, N, ws, kSlotBytes, sums, st);
  if (rc) return rc;
  double hs[2];
  XCK(cudaMemcpyAsync(hs, sums, sizeof(hs), cudaMemcpyDeviceToHost, st));
  XCK(cudaStreamSynchronize(st));
  const double tr = hs[1] / (double)D;   // sum_u Tr(rho A_u) = 3^N Tr(rho)
  if (out_trace) *out_trace = tr;
  if (!(std::fabs(tr - 1.0) <= 1e-8)) return fail(SRE_ENOTNORM, "Tr(rho) = %.17g", tr);
  *out_mana = std::log2(hs[0] / (double)D);
  return SRE_OK;
}

}  // extern "C"
