// Do SHFL and LDS/STS share a datapath on B200?  And TMEM? (timing only; prints JSON lines)
//   smem : 32 LDS.64 + 32 STS.64 per iteration (transpose pattern, padded)
//   shfl : 32 SHFL.64 (two SHFL.32 each) per iteration
//   both : the two bodies interleaved in the same warps
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench2 microbench2.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, int iters) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* b = sm + w * 1056;
  double r[32], q[32];
#pragma unroll
  for (int j = 0; j < 32; j++) { r[j] = lane + j; q[j] = lane * 2 + j; }
  for (int it = 0; it < iters; it++) {
    if (MODE & 1) {
#pragma unroll
      for (int j = 0; j < 32; j++) b[j * 33 + lane] = r[j];
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; j++) r[j] = b[lane * 33 + j];
      __syncwarp();
    }
    if (MODE & 2) {
#pragma unroll
      for (int j = 0; j < 32; j++) q[j] = __shfl_xor_sync(0xffffffffu, q[j], (j & 31) | 1);
    }
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < 32; j++) t += r[j] + q[j];
  if (t == 1.2345) out[0] = t;
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
  const int th = 256, iters = 2000;
  const int smb = 8 * 1056 * 8;
  auto run = [&](auto kern, const char* name, double bytes_smem_per_it, double shfl_dbl_per_it) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smb);
    kern<<<sms * 2, th, smb>>>(out, 10);
    cudaEventRecord(e0);
    kern<<<sms * 2, th, smb>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double thr = (double)sms * 2 * th * iters;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("{\"test\": \"%s\", \"ms\": %.3f, \"smem_B_per_clk_sm\": %.1f, \"shfl_dbl_per_clk_sm\": %.2f}\n", name, ms,
           thr * bytes_smem_per_it / cyc / sms, thr * shfl_dbl_per_it / cyc / sms);
  };
  run(k<1>, "smem", 32 * 16, 0);
  run(k<2>, "shfl", 0, 32);
  run(k<3>, "both", 32 * 16, 32);
  return 0;
}
