// Microbenchmark: does the FP64 tensor-core MMA (mma.sync m8n8k4 f64) run on
// a pipe separate from DFMA on this GPU? Three kernels with the same
// per-thread loop structure: DMMA only, DFMA only, and both interleaved. If
// the mixed kernel takes ~max(DMMA, DFMA) the pipes are separate; ~sum:
// shared. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_bench tools/dmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int NM, int NF>
__global__ void mix(double* out, int iters) {
  double acc[NM > 0 ? NM : 1][2];
  double f[NF > 0 ? NF : 1];
#pragma unroll
  for (int k = 0; k < (NM > 0 ? NM : 1); ++k) acc[k][0] = acc[k][1] = threadIdx.x + k;
#pragma unroll
  for (int k = 0; k < (NF > 0 ? NF : 1); ++k) f[k] = 2.0 + k;
  const double a = 1.0000001 + threadIdx.x * 1e-9, b = 0.999999;
  const double m = 1.0000001, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NM; ++k) dmma(acc[k], a, b);
#pragma unroll
    for (int k = 0; k < NF; ++k) f[k] = fma(f[k], m, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < (NM > 0 ? NM : 1); ++k) s += acc[k][0] + acc[k][1];
#pragma unroll
  for (int k = 0; k < (NF > 0 ? NF : 1); ++k) s += f[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
float timeit(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 20000;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  const double warps = double(blocks) * threads / 32;
  const float t_m = timeit([&] { mix<8, 0><<<blocks, threads>>>(out, iters); });
  const float t_f = timeit([&] { mix<0, 16><<<blocks, threads>>>(out, iters); });
  const float t_mf = timeit([&] { mix<8, 16><<<blocks, threads>>>(out, iters); });
  // flops: DMMA m8n8k4 = 2*8*8*4 = 512 per warp-instruction; DFMA 2 per thread
  const double fm = warps * iters * 8 * 512, ff = double(blocks) * threads * iters * 16 * 2;
  printf("DMMA only  : %8.3f ms  %7.2f TFLOP/s\n", t_m, fm / t_m * 1e-9);
  printf("DFMA only  : %8.3f ms  %7.2f TFLOP/s\n", t_f, ff / t_f * 1e-9);
  printf("both mixed : %8.3f ms  (separate pipes ~ %.3f, shared ~ %.3f)\n", t_mf, t_m > t_f ? t_m : t_f, t_m + t_f);
  return 0;
}
