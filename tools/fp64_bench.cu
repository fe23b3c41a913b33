// Microbenchmark: FP64 DFMA peak and Laplace kernel-evaluation throughput in
// the P2P pattern the matrix-free matvec uses (warp = 4..8 target rows, lanes
// stride over sources in global/L1). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_bench tools/fp64_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_peak(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  const double m = 1.0000001, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// MUFU.RSQ64H issue rate: 8 independent seeds per thread per iteration
__global__ void mufu_peak(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double y;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a[k]));
      a[k] = y + 1.0;  // DADD keeps the chain alive (1 DP op per seed)
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// RSQ64H and DFMA interleaved: NR seeds + NF independent FMAs per iteration
// (separate pipes: time ~ max of the two; shared: ~ sum)
template <int NR, int NF>
__global__ void mix_peak(double* out, int iters) {
  double a[8], f[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = 1.0 + threadIdx.x + k;
    f[k] = 2.0 + k;
  }
  const double m = 1.0000001, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      double y;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a[k & 7]));
      a[k & 7] = y;
    }
#pragma unroll
    for (int k = 0; k < NF; ++k) f[k & 7] = fma(f[k & 7], m, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k] + f[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ double rsqrt_nr1(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double p = x * y;
  const double e = fma(-p, y, 1.0);
  return fma(0.5 * y, e, y);
}

__device__ __forceinline__ double rsqrt_nr2(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double p = x * y;
  double e = fma(-p, y, 1.0);
  y = fma(0.5 * y, e, y);
  p = x * y;
  e = fma(-p, y, 1.0);
  return fma(0.5 * y, e, y);
}

template <int MODE, int ROWS>
__global__ void __launch_bounds__(256) p2p(const double* __restrict__ sx, const double* __restrict__ sy,
                                           const double* __restrict__ sz, const double* __restrict__ sq,
                                           int ns, const double* __restrict__ tx, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row0 = (blockIdx.x * 8 + warp) * ROWS;
  double px[ROWS], py[ROWS], pz[ROWS], acc[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    px[r] = tx[3 * (row0 + r)];
    py[r] = tx[3 * (row0 + r) + 1];
    pz[r] = tx[3 * (row0 + r) + 2];
    acc[r] = 0.0;
  }
  for (int j = lane; j < ns; j += 32) {
    const double x = sx[j], y = sy[j], z = sz[j], q = sq[j];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const double dx = px[r] - x, dy = py[r] - y, dz = pz[r] - z;
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      double k;
      if (MODE == 0) k = rsqrt(r2);
      else if (MODE == 1) k = rsqrt_nr1(r2);
      else if (MODE == 2) k = rsqrt_nr2(r2);
      else k = 1.0 / sqrt(r2);
      acc[r] = fma(k, q, acc[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    double v = acc[r];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) out[row0 + r] = v;
  }
}

template <int MODE, int ROWS>
float run_p2p(double* sx, double* sy, double* sz, double* sq, int ns, double* tx, double* out,
              int nt) {
  const int blocks = nt / (8 * ROWS);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  p2p<MODE, ROWS><<<blocks, 256>>>(sx, sy, sz, sq, ns, tx, out);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) p2p<MODE, ROWS><<<blocks, 256>>>(sx, sy, sz, sq, ns, tx, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * (1 << 24));
  {
    const int iters = 1 << 16, blocks = sms * 8, threads = 256;
    dfma_peak<<<blocks, threads>>>(out, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dfma_peak<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = double(blocks) * threads * iters * 8;
    printf("DFMA: %.2f T fma/s = %.1f TFLOP/s (fp64)\n", fmas / ms / 1e9, 2 * fmas / ms / 1e9);
  }
  {
    const int iters = 20000, blocks = 148 * 8, threads = 256;
    double* o;
    cudaMalloc(&o, sizeof(double) * blocks * threads);
    auto run = [&](auto kern, const char* name) {
      kern<<<blocks, threads>>>(o, 10);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      kern<<<blocks, threads>>>(o, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%s: %.3f ms\n", name, ms);
    };
    run(mix_peak<8, 0>, "8 RSQ64H        ");
    run(mix_peak<0, 32>, "32 DFMA         ");
    run(mix_peak<8, 32>, "8 RSQ64H+32 DFMA");
    cudaFree(o);
  }
  {
    const int iters = 20000, blocks = 148 * 8, threads = 256;
    double* o;
    cudaMalloc(&o, sizeof(double) * blocks * threads);
    mufu_peak<<<blocks, threads>>>(o, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mufu_peak<<<blocks, threads>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 8.0 * iters * blocks * threads;
    printf("MUFU.RSQ64H (+1 DADD each): %.3f T seeds/s = %.2f per SM per clock at 1.965 GHz\n",
           ops / ms / 1e9, ops / (ms * 1e-3) / 148 / 1.965e9);
    cudaFree(o);
  }
  const int ns = 1 << 16, nt = 1 << 20;
  double *sx, *sy, *sz, *sq, *tx;
  cudaMalloc(&sx, ns * 8);
  cudaMalloc(&sy, ns * 8);
  cudaMalloc(&sz, ns * 8);
  cudaMalloc(&sq, ns * 8);
  cudaMalloc(&tx, nt * 24);
  double* h = new double[3 * nt];
  for (int i = 0; i < 3 * nt; ++i) h[i] = (i * 0.6180339887) - (long)(i * 0.6180339887);
  cudaMemcpy(tx, h, nt * 24, cudaMemcpyHostToDevice);
  cudaMemcpy(sx, h + 7, ns * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(sy, h + 7 + ns, ns * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(sz, h + 7 + 2 * ns, ns * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(sq, h + 11, ns * 8, cudaMemcpyHostToDevice);
  const int ntp = nt / 16;  // 65536 targets
  const double ev = double(ntp) * ns;
  printf("P2P evals per launch: %.3g\n", ev);
#define RUN(M, R)                                                                     \
  {                                                                                   \
    float ms = run_p2p<M, R>(sx, sy, sz, sq, ns, tx, out, ntp);                       \
    printf("mode %d rows %d: %.3f ms  %.3f T evals/s\n", M, R, ms, ev / ms / 1e9);    \
  }
  RUN(0, 4) RUN(0, 8) RUN(1, 4) RUN(1, 8) RUN(2, 4) RUN(2, 8) RUN(3, 4)
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
