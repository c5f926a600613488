// Shared-memory wavefronts of pass A's access patterns (run under ncu with the
// l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld/st metrics; one kernel per pattern).
//   k_q128   : double2 loads, lane-contiguous (generation q operand)
//   k_r128   : double2 loads, index (lane ^ a5) + 32 (j ^ ah) (generation r operand)
//   k_r64x2  : the r pattern as two 8-byte loads
//   k_xld    : exchange read  swz(j + 32 lane) = j + 33 lane (8-byte)
//   k_xst    : exchange write swz(lane + 32 j) = lane + 32 j + j (8-byte)
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 64;
__global__ void k_q128(double* out, int a) {
  __shared__ double2 s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_double2(i, -i);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc = 0;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int j = 0; j < 32; ++j) { double2 q = s[lane + 32 * j]; acc += q.x * q.y; }
  if (acc == 1.5) out[0] = acc;
}
__global__ void k_r128(double* out, int a) {
  __shared__ double2 s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_double2(i, -i);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc = 0;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int j = 0; j < 32; ++j) { double2 r = s[1024 + ((lane + 32 * j) ^ (a & 1023))]; acc += r.x * r.y; }
  if (acc == 1.5) out[0] = acc;
}
__global__ void k_r64x2(double* out, int a) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc = 0;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int e = 1024 + ((lane + 32 * j) ^ (a & 1023));
      acc += s[2 * e] * s[2 * e + 1];
    }
  if (acc == 1.5) out[0] = acc;
}
__global__ void k_xld(double* out, int a) {
  __shared__ double s[4 * 1056];
  for (int i = threadIdx.x; i < 4 * 1056; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc = 0;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int j = 0; j < 32; ++j) acc += s[w * 1056 + j + 33 * lane];
  if (acc == 1.5) out[0] = acc;
}
__global__ void k_xst(double* out, int a) {
  __shared__ double s[4 * 1056];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 32; ++j) s[w * 1056 + lane + 33 * j] = it + j;
    __syncwarp();
  }
  __syncthreads();
  if (s[threadIdx.x] == 1.5) out[0] = 1;
}

int main() {
  double* out;
  cudaMalloc(&out, 64);
  for (int a : {0, 0x15, 0x2b5}) {
    k_q128<<<148, 256>>>(out, a);
    k_r128<<<148, 256>>>(out, a);
    k_r64x2<<<148, 256>>>(out, a);
  }
  k_xld<<<148, 128>>>(out, 0);
  k_xst<<<148, 128>>>(out, 0);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
