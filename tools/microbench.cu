// Microbenchmarks that ground the roofline denominators for the SRE hot path on B200:
//   fp64   : DADD/DFMA issue rate (ops/clk/SM) with many independent chains
//   l2rd   : read bandwidth of an L2-resident buffer (LDG.128)
//   hbmrd  : read bandwidth of a 4 GiB buffer
//   hbmcp  : copy bandwidth (read+write) of a 2 GiB buffer
//   smem64 : shared-memory bandwidth with 64-bit lane accesses (transpose pattern, XOR swizzle)
//   shfl64 : warp-shuffle throughput for doubles
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void k_fp64(double* out, int iters, double s) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; i++) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) a[i] = a[i] + s;   // DADD
#pragma unroll
    for (int i = 0; i < 16; i++) a[i] = fma(a[i], s, a[(i + 1) & 15]);  // DFMA
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) t += a[i];
  if (t == 1.2345) out[0] = t;
}

__global__ void k_read(const double2* __restrict__ p, size_t n, int reps, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; r++)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      double2 v = __ldg(p + i);
      acc += v.x + v.y;
    }
  if (acc == 1.2345) out[0] = acc;
}

__global__ void k_copy(const double2* __restrict__ p, double2* __restrict__ q, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) q[i] = p[i];
}

__global__ void k_smem(double* out, int iters) {
  extern __shared__ double sm[];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* b = sm + w * 1024;
  double r[32];
#pragma unroll
  for (int j = 0; j < 32; j++) r[j] = lane + j;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 32; j++) b[j * 32 + (lane ^ j)] = r[j];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; j++) r[j] = b[lane * 32 + (j ^ lane)];
    __syncwarp();
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < 32; j++) t += r[j];
  if (t == 1.2345) out[0] = t;
}

__global__ void k_shfl(double* out, int iters) {
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = threadIdx.x + j;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = __shfl_xor_sync(0xffffffffu, r[j], (j + it) & 31 | 1);
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) t += r[j];
  if (t == 1.2345) out[0] = t;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  int l2 = 0; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  printf("{\"sms\": %d, \"clock_khz\": %d, \"l2_bytes\": %d}\n", sms, clk, l2);
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;
  // fp64
  for (int occ = 2; occ <= 8; occ *= 2) {
    int iters = 20000, th = 256;
    k_fp64<<<sms * occ, th>>>(out, 100, 1.0000001);
    CK(cudaEventRecord(e0));
    k_fp64<<<sms * occ, th>>>(out, iters, 1.0000001);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double ops = (double)sms * occ * th * iters * 32.0;
    printf("{\"test\": \"fp64\", \"ctas_per_sm\": %d, \"ms\": %.3f, \"fp64_ops_per_s\": %.4e, \"ops_per_clk_sm_at_max\": %.2f}\n",
           occ, ms, ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / (clk * 1e3));
  }
  // long fp64 run (~3 s) for clock sampling
  {
    int iters = 400000, th = 256, occ = 4;
    CK(cudaEventRecord(e0));
    k_fp64<<<sms * occ, th>>>(out, iters, 1.0000001);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double ops = (double)sms * occ * th * iters * 32.0;
    printf("{\"test\": \"fp64_long\", \"ms\": %.3f, \"fp64_ops_per_s\": %.4e}\n", ms, ops / (ms * 1e-3));
  }
  // reads
  size_t big = (size_t)4 << 30;
  double2* buf; CK(cudaMalloc(&buf, big));
  CK(cudaMemset(buf, 0, big));
  size_t sizes[] = {(size_t)8 << 20, (size_t)32 << 20, (size_t)64 << 20, (size_t)96 << 20, big};
  for (size_t sz : sizes) {
    size_t n = sz / 16;
    int reps = (int)(((size_t)16 << 30) / sz); if (reps < 1) reps = 1;
    for (int th : {256, 512}) {
      k_read<<<sms * 4, th>>>(buf, n, 1, out);
      CK(cudaEventRecord(e0));
      k_read<<<sms * 4, th>>>(buf, n, reps, out);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("{\"test\": \"read\", \"bytes\": %zu, \"threads\": %d, \"GBps\": %.1f}\n", sz, th, (double)sz * reps / (ms * 1e-3) / 1e9);
    }
  }
  {
    size_t n = ((size_t)1 << 30) / 16;
    k_copy<<<sms * 8, 256>>>(buf, buf + n, n);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; r++) k_copy<<<sms * 8, 256>>>(buf, buf + n, n);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("{\"test\": \"copy\", \"bytes_rw\": %zu, \"GBps\": %.1f}\n", n * 32 * 5, (double)n * 32 * 5 / (ms * 1e-3) / 1e9);
  }
  // smem
  {
    int th = 256, iters = 2000;
    size_t smb = th / 32 * 1024 * 8;
    CK(cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
    k_smem<<<sms * 2, th, smb>>>(out, 10);
    CK(cudaEventRecord(e0));
    k_smem<<<sms * 2, th, smb>>>(out, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double bytes = (double)sms * 2 * th * iters * 32 * 16;
    printf("{\"test\": \"smem64\", \"GBps\": %.1f, \"B_per_clk_sm_at_max\": %.1f}\n", bytes / (ms * 1e-3) / 1e9,
           bytes / (ms * 1e-3) / sms / (clk * 1e3));
  }
  {
    int th = 256, iters = 20000;
    k_shfl<<<sms * 4, th>>>(out, 10);
    CK(cudaEventRecord(e0));
    k_shfl<<<sms * 4, th>>>(out, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double sh = (double)sms * 4 * th * iters * 8;
    printf("{\"test\": \"shfl64\", \"doubles_per_clk_sm_at_max\": %.2f}\n", sh / (ms * 1e-3) / sms / (clk * 1e3));
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
