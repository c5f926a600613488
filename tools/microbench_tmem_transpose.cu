// Warp-local 32 x 32 transpose of doubles for the 10-bit pass-A transform: shared memory (padded
// STS/LDS, the k_passA10s exchange) versus three TMEM round trips (tcgen05.st 32x32b.x64, then two
// tcgen05.ld 16x256b.x8 at lane bases 0 and 16: thread t = t0 + 4 t1 receives lane 16b + 8s + t1,
// double column 4c + t0 into register r = s + 2c + 16b; CUTLASS Copy_Traits<SM100_TMEM_LOAD_16dp256b1x>).
// Checks the element ids after each trip against tools' Python simulation, then times 8 warps/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_tmem_transpose tools/microbench_tmem_transpose.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void st64(uint32_t ta, const double (&v)[32]) {
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
// 16 doubles: lanes (lane base) + t1 and + 8, double columns 4c + t0 of the 16 x 256-bit chunk c = 0..7
__device__ __forceinline__ void ld16(uint32_t ta, double* v) {
  uint32_t u[32];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15]),
                 "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
               : "r"(ta) : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __hiloint2double(u[2 * i + 1], u[2 * i]);
}
__device__ __forceinline__ void trip(uint32_t ta, double (&v)[32]) {
  st64(ta, v);
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  ld16(ta, v);                      // lanes 0..15 of the warp's quadrant
  ld16(ta + (16u << 16), v + 16);   // lanes 16..31
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// expected element id of (thread t, register r) after k trips (from the simulation's bit maps)
__device__ int expect(int k, int t, int r) {
  if (k == 0) return t + 32 * r;
  // generic: simulate on the fly by composing the trip map (cheap, per thread)
  // element held at (thread tt, reg rr) before trip k: recursive closed form via loops
  // (only used in the verification kernel)
  int tt = t, rr = r;
  for (int kk = k; kk > 0; --kk) {      // undo trips: (t, r) after <- (lane, dcol) before
    const int t0 = tt & 3, t1 = tt >> 2, s = rr & 1, c = (rr >> 1) & 7, b = rr >> 4;
    const int lane = 16 * b + 8 * s + t1, dcol = 4 * c + t0;
    tt = lane; rr = dcol;
  }
  return tt + 32 * rr;
}

__global__ void __launch_bounds__(256, 1) k_verify(int* bad) {
  __shared__ uint32_t taddr_s;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(su32(&taddr_s)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t ta = taddr_s + ((uint32_t)(32 * (w & 3)) << 16) + 128u * (uint32_t)(w >> 2);
  double v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = (double)(lane + 32 * r + 1024 * w);
  for (int k = 1; k <= 3; ++k) {
    trip(ta, v);
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (v[r] != (double)(expect(k, lane, r) + 1024 * w)) atomicAdd(bad + k, 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(taddr_s) : "memory");
}

// timing: MODE 0 = smem transpose (2 planes, padded, as k_passA10s), 1 = TMEM 3 trips x 2 planes
template <int MODE>
__global__ void __launch_bounds__(256, 1) k_time(double* out, int iters) {
  __shared__ uint32_t taddr_s;
  extern __shared__ double smx[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (MODE >= 1) {
    if (w == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(su32(&taddr_s)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  }
  __syncthreads();
  if (MODE >= 1) asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t ta = taddr_s + ((uint32_t)(32 * (w & 3)) << 16) + 128u * (uint32_t)(w >> 2);
  double a[32], b[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) { a[r] = lane + r; b[r] = lane - r; }
  double* x = smx + w * 32 * 33;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        double (&v)[32] = p ? b : a;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j * 33 + lane] = v[j];
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = x[lane * 33 + j];
      }
    } else if (MODE == 1) {
      trip(ta, a); trip(ta + 64, b);
      trip(ta, a); trip(ta + 64, b);
      trip(ta, a); trip(ta + 64, b);
    } else {                      // plane a through shared memory, plane b through TMEM, interleaved
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j * 33 + lane] = a[j];
      trip(ta + 64, b);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j) a[j] = x[lane * 33 + j];
      trip(ta + 64, b);
      trip(ta + 64, b);
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) { a[r] += 1.0; b[r] -= 1.0; }
  }
  double t = 0;
  for (int r = 0; r < 32; ++r) t += a[r] + b[r];
  if (t == 1.2345) out[0] = t;
  if (MODE >= 1) {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(taddr_s) : "memory");
  }
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int* bad;
  cudaMalloc(&bad, 16);
  cudaMemset(bad, 0, 16);
  k_verify<<<sms, 256>>>(bad);
  int hb[4];
  cudaError_t e = cudaMemcpy(hb, bad, 16, cudaMemcpyDeviceToHost);
  printf("{\"verify\": \"%s\", \"bad_trip1\": %d, \"bad_trip2\": %d, \"bad_trip3\": %d}\n", cudaGetErrorString(e), hb[1], hb[2], hb[3]);
  double* out;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  auto run = [&](auto kern, const char* name) {
    const int smb = 8 * 32 * 33 * 8;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smb);
    kern<<<sms, 256, smb>>>(out, 10);
    cudaEventRecord(e0);
    kern<<<sms, 256, smb>>>(out, iters);
    cudaEventRecord(e1);
    cudaError_t er = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    // per SM: 8 warps x 2 planes x 1024 values per iteration
    const double vals = (double)sms * 8 * 2 * 1024 * iters;
    printf("{\"mode\": \"%s\", \"err\": \"%s\", \"ms\": %.3f, \"sm_clk_per_value\": %.4f}\n", name, cudaGetErrorString(er), ms,
           ms * 1e-3 * clk * 1e3 * sms / vals);
  };
  run(k_time<0>, "smem_transpose_2planes");
  run(k_time<1>, "tmem_3trips_2planes");
  run(k_time<2>, "smem_plane_a_plus_tmem_plane_b");
  return 0;
}
