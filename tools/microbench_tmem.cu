// TMEM bandwidth microbenchmark: tcgen05.st / tcgen05.ld (32x32b.x64) per SM, alone and mixed
// with shared-memory transposes (is TMEM a separate datapath from the L1TEX data pipe?).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tst(uint32_t ta, uint32_t (&r)[64]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x64.b32 [%64], {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63};\n" :: "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]), "r"(r[32]), "r"(r[33]), "r"(r[34]), "r"(r[35]), "r"(r[36]), "r"(r[37]), "r"(r[38]), "r"(r[39]), "r"(r[40]), "r"(r[41]), "r"(r[42]), "r"(r[43]), "r"(r[44]), "r"(r[45]), "r"(r[46]), "r"(r[47]), "r"(r[48]), "r"(r[49]), "r"(r[50]), "r"(r[51]), "r"(r[52]), "r"(r[53]), "r"(r[54]), "r"(r[55]), "r"(r[56]), "r"(r[57]), "r"(r[58]), "r"(r[59]), "r"(r[60]), "r"(r[61]), "r"(r[62]), "r"(r[63]), "r"(ta) : "memory");
}
__device__ __forceinline__ void tld(uint32_t ta, uint32_t (&r)[64]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];\n" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63]) : "r"(ta) : "memory");
}
template <int MODE>
__global__ void __launch_bounds__(128, 1) k(double* out, int iters) {
  __shared__ uint32_t taddr_s;
  extern __shared__ double sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&taddr_s)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t ta = taddr_s + ((uint32_t)(w * 32) << 16);
  uint32_t r[64];
#pragma unroll
  for (int i = 0; i < 64; i++) r[i] = threadIdx.x * 7 + i;
  double q[32];
#pragma unroll
  for (int j = 0; j < 32; j++) q[j] = lane + j;
  double* b = sm + w * 1056;
  for (int it = 0; it < iters; it++) {
    if (MODE & 1) {
#pragma unroll
      for (int c = 0; c < 8; c++) tst(ta + c * 64, r);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int c = 0; c < 8; c++) {
        tld(ta + c * 64, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int i = 0; i < 64; i++) r[i] += 1;
      }
    }
    if (MODE & 2) {
#pragma unroll
      for (int rep = 0; rep < 4; rep++) {
#pragma unroll
        for (int j = 0; j < 32; j++) b[j * 33 + lane] = q[j];
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 32; j++) q[j] = b[lane * 33 + j];
        __syncwarp();
      }
    }
  }
  double t = 0;
  for (int i = 0; i < 64; i++) t += r[i];
  for (int j = 0; j < 32; j++) t += q[j];
  if (t == 1.2345) out[0] = t;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(taddr_s) : "memory");
}
int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smb = 4 * 1056 * 8, iters = 2000;
  auto run = [&](auto kern, const char* name, double tmem_b, double smem_b) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smb);
    kern<<<sms, 128, smb>>>(out, 10);
    cudaEventRecord(e0);
    kern<<<sms, 128, smb>>>(out, iters);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("{\"test\": \"%s\", \"err\": \"%s\", \"ms\": %.3f, \"tmem_B_per_clk_sm\": %.1f, \"smem_B_per_clk_sm\": %.1f}\n", name,
           cudaGetErrorString(e), ms, 128.0 * iters * tmem_b / cyc, 128.0 * iters * smem_b / cyc);
  };
  run(k<1>, "tmem", 8 * 256 * 2, 0);
  run(k<2>, "smem", 0, 4 * 32 * 16);
  run(k<3>, "both", 8 * 256 * 2, 4 * 32 * 16);
  return 0;
}
