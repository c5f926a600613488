// Write-pattern microbenchmark for the pass-A workspace at N = 24 (H = 11 rows of 4096 positions per
// plane): how fast can HBM absorb the slab-major layout's 32-B runs, depending on which rows and
// X-strings a CTA's four 64-thread units write together?
//   mode 0: units = 4 X-strings of one row (k_passAr's item), items row-major over (row, group)
//   mode 1: units = 4 consecutive rows of one X-string (lines of 4 rows x 32 B complete in the CTA)
//   mode 2: row-major workspace (each row-plane contiguous 32 KB), units = 4 X-strings of one row
//   mode 3: CB = 4 layout (128-B runs per row), units = 4 X-strings of one row
// Each thread writes 64 consecutive positions as 16 x 32-B stores (k_passAr's round-1 layout).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_wr tools/microbench_wr.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void stg_v4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.cg.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_wr(double* ws, int K) {
  constexpr int H = 11;
  constexpr size_t PLANE = (size_t)1 << 23;
  const int u = threadIdx.x >> 6;
  const uint32_t t = threadIdx.x & 63;
  const uint64_t items = (uint64_t)(1 << H) * (K / 4);     // 4 row-planes (x2 planes) per item
  for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
    uint64_t yh, k;
    if (MODE == 6) {                                       // ceiling: fully coalesced contiguous writes
      double* wp = ws + it * 32768;
      for (int i = threadIdx.x; i < 8192; i += 256) {
        const double v = (double)i;
        stg_v4(wp + 4 * i, v, v + 1, v + 2, v + 3);
      }
      continue;
    }
    if (MODE == 4) {                                       // 4 rows per CTA, each instruction = 8 full lines
      const uint64_t rb = it / K, kk = it % K;
      for (int pl = 0; pl < 2; ++pl) {
        double* wp = ws + (size_t)kk * 2 * PLANE + (size_t)pl * PLANE + (rb << 4);
        // 4096 slabs-rows: lane -> (row = lane & 3, slab = 8 * warp-step + lane / 4)
        for (int i = threadIdx.x; i < 4096; i += 256) {
          const uint32_t row = i & 3, slab = i >> 2;
          const double v = (double)i;
          stg_v4(wp + ((size_t)slab << (H + 2)) + 4 * row, v, v + 1, v + 2, v + 3);
        }
      }
      continue;
    }
    if (MODE == 5) {                                       // 16 rows x 32 B runs (as a 4-CTA cluster would write)
      const uint64_t rb = it / K, kk = it % K;             // block of 4 rows; 4 consecutive CTAs = 16 rows
      const uint64_t r16 = rb >> 2, part = rb & 3;         // this CTA writes slabs [256 part, 256 part + 256)
      for (int pl = 0; pl < 2; ++pl) {
        double* wp = ws + (size_t)kk * 2 * PLANE + (size_t)pl * PLANE + (r16 << 6);
        for (int i = threadIdx.x; i < 4096; i += 256) {
          const uint32_t row = i & 15, slab = 256 * (uint32_t)part + (i >> 4);
          const double v = (double)i;
          stg_v4(wp + ((size_t)slab << (H + 2)) + 4 * row, v, v + 1, v + 2, v + 3);
        }
      }
      continue;
    }
    if (MODE == 9) {                                       // CB = 3 slabs (2^11 rows x 8 cols): 4 rows per CTA, 64-B row runs
      const uint64_t rb = it / K, kk = it % K;
      const uint64_t yh9 = rb * 4 + u;
      for (int pl = 0; pl < 2; ++pl) {
        double* wp = ws + (size_t)kk * 2 * PLANE + (size_t)pl * PLANE;
#pragma unroll
        for (int r4 = 0; r4 < 16; ++r4) {
          const uint32_t pos = 64u * t + 4u * r4;
          const size_t off = ((size_t)(pos >> 3) << (H + 3)) + (yh9 << 3) + (pos & 7u);
          const double v = (double)(pos + yh9);
          stg_v4(wp + off, v, v + 1, v + 2, v + 3);
        }
      }
      continue;
    }
    if (MODE == 1) {                                       // 4 consecutive rows of one X-string
      const uint64_t rb = it / K, kk = it % K;             // row block of 4, X-string
      yh = rb * 4 + u; k = kk;
    } else {
      const uint64_t g = it % (K / 4);
      yh = it / (K / 4); k = 4 * g + u;
    }
    for (int pl = 0; pl < 2; ++pl) {
      double* wp = ws + (size_t)k * 2 * PLANE + (size_t)pl * PLANE;
#pragma unroll
      for (int r4 = 0; r4 < 16; ++r4) {
        const uint32_t pos = 64u * t + 4u * r4;
        size_t off;
        if (MODE == 2) off = (yh << 12) + pos;
        else if (MODE == 3) off = ((size_t)(pos >> 4) << (H + 4)) + (yh << 4) + (pos & 15u);
        else off = ((size_t)(pos >> 2) << (H + 2)) + (yh << 2) + (pos & 3u);
        const double v = (double)(pos + yh);
        stg_v4(wp + off, v, v + 1, v + 2, v + 3);
      }
    }
  }
}

// Read side (pass B): a "tile" is 2^11 rows x 4 doubles.  RMODE 0: contiguous 64-KB tiles (slab-major
// CB = 2); RMODE 1: tiles are 32-B pieces at 128-B stride inside 2^11 x 16 slabs (CB = 4 layout), the
// four quarter tiles of a slab processed by neighbouring CTAs at the same time.
template <int RMODE>
__global__ void __launch_bounds__(256) k_rd(const double* __restrict__ ws, uint64_t tiles, double* out) {
  double acc = 0.0;
  for (uint64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const double* base;
    size_t stride;
    if (RMODE == 0) { base = ws + tile * 8192; stride = 4; }
    else if (RMODE == 1) { base = ws + (tile >> 2) * 32768 + 4 * (tile & 3); stride = 16; }
    else { base = ws + (tile >> 10) * (8192ull * 1024) + 4 * (tile & 1023); stride = 4096; }   // row-major [2048][4096] planes
    for (int r = threadIdx.x; r < 2048; r += 256) {
      double a, b, c, d;
      asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(base + r * stride));
      acc += a + b + c + d;
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

// mode 7: 4-CTA cluster; CTA rank c writes rows 16 m + 4 c .. + 3 as full 128-B lines (one instruction
// covers 8 lines), the four CTAs synchronised by a cluster barrier before each plane, so the four lines
// of every 512-B run leave four SMs at about the same time.  mode 8: 8-row (256-B) runs from one CTA.
template <int MODE>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(256, 1) k_wrc(double* ws, int K) {
  constexpr int H = 11;
  constexpr size_t PLANE = (size_t)1 << 23;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const uint64_t nclu = gridDim.x / 4, clu = blockIdx.x / 4;
  const uint64_t items = (uint64_t)(1 << H) / 16 * K;      // (16-row block, X-string)
  for (uint64_t it = clu; it < items; it += nclu) {
    const uint64_t r16 = it / K, kk = it % K;
    for (int pl = 0; pl < 2; ++pl) {
      asm volatile("barrier.cluster.arrive.aligned; barrier.cluster.wait.aligned;" ::: "memory");
      double* wp = ws + (size_t)kk * 2 * PLANE + (size_t)pl * PLANE + (r16 << 6) + 16 * rank;
      for (int i = threadIdx.x; i < 4096; i += 256) {
        const uint32_t row = i & 3, slab = i >> 2;
        const double v = (double)i;
        stg_v4(wp + ((size_t)slab << (H + 2)) + 4 * row, v, v + 1, v + 2, v + 3);
      }
    }
  }
}
__global__ void __launch_bounds__(256, 1) k_wr8(double* ws, int K) {   // 8 rows x 32 B = 256-B runs
  constexpr int H = 11;
  constexpr size_t PLANE = (size_t)1 << 23;
  const uint64_t items = (uint64_t)(1 << H) / 8 * K;
  for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const uint64_t r8 = it / K, kk = it % K;
    for (int pl = 0; pl < 2; ++pl) {
      double* wp = ws + (size_t)kk * 2 * PLANE + (size_t)pl * PLANE + (r8 << 5);
      for (int i = threadIdx.x; i < 8192; i += 256) {
        const uint32_t row = i & 7, slab = i >> 3;
        const double v = (double)i;
        stg_v4(wp + ((size_t)slab << (H + 2)) + 4 * row, v, v + 1, v + 2, v + 3);
      }
    }
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* ws;
  const int Kmax = 32;
  const size_t bytes = (size_t)Kmax * 2 * ((size_t)1 << 23) * 8;
  if (cudaMalloc(&ws, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name, int K) {
    const int g = sms / 4 * 4;
    kern<<<g, 256>>>(ws, K);
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) kern<<<g, 256>>>(ws, K);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double b = 3.0 * K * 2 * ((size_t)1 << 23) * 8;
    printf("{\"mode\": \"%s\", \"K\": %d, \"err\": \"%s\", \"ms_per_launch\": %.3f, \"GBps\": %.1f, \"us_per_xstring\": %.2f}\n",
           name, K, cudaGetErrorString(e), ms / 3, b / (ms * 1e-3) / 1e9, ms * 1e3 / 3 / K);
  };
  for (int K : {8, 32}) {
    run(k_wr<0>, "slab32B_4xstrings_per_row", K);
    run(k_wr<1>, "slab32B_4rows_per_cta", K);
    run(k_wr<2>, "row_major", K);
    run(k_wr<3>, "slab128B_4xstrings_per_row", K);
    run(k_wr<4>, "slab32B_4rows_full_line_instr", K);
    run(k_wr<5>, "slab32B_16rows_512B_runs", K);
    run(k_wr<6>, "coalesced_contiguous", K);
    run(k_wrc<7>, "cluster4_synced_4row_lines", K);
    run(k_wr<9>, "slab64B_4rows_per_cta", K);
    run(k_wr8, "slab32B_8rows_256B_runs", K);
  }
  for (int rm = 0; rm < 3; ++rm) {
    const uint64_t tiles = bytes / 8 / 8192;
    auto kern = rm == 0 ? k_rd<0> : rm == 1 ? k_rd<1> : k_rd<2>;
    kern<<<4 * sms, 256>>>(ws, tiles, ws);
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) kern<<<4 * sms, 256>>>(ws, tiles, ws);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"read_mode\": %d, \"err\": \"%s\", \"GBps\": %.1f}\n", rm, cudaGetErrorString(e), 3.0 * bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
