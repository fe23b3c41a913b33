// Microbenchmark for the proxy-level evaluation core (matvec.cu proxy_evalT):
// (1) does a non-FP64 instruction beside a DFMA cost an issue slot the FP64
//     pipe needs (DFMA + k IMAD / LDS per DFMA), and
// (2) variants of the Laplace admissible-path core: targets per thread,
//     sources per loop trip, and the 7-instruction form with the weight folded
//     into the staged source (r2' = r2 / w^2, signed).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/eval_bench tools/eval_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

// ---- (1) issue-slot probe ---------------------------------------------------
template <int NI, int NL>
__global__ void __launch_bounds__(128, 5) issue_probe(double* out, int iters) {
  __shared__ double2 sm[256];
  sm[threadIdx.x] = make_double2(threadIdx.x, 1.0);
  sm[threadIdx.x + 128] = make_double2(threadIdx.x, 2.0);
  __syncthreads();
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
  int q[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) q[k] = threadIdx.x * 3 + k;
  const double m = 1.0000001, c = 1e-9;
  double ls = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
#pragma unroll
    for (int k = 0; k < NI; ++k) asm volatile("mad.lo.s32 %0, %0, 3, 7;" : "+r"(q[k & 7]));
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const double2 v = sm[(i + k) & 255];
      ls += v.x;  // one DADD per load keeps it alive (counted in the table)
    }
  }
  double s = ls;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k] + q[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}


// ---- (1b) seed probes: NF DFMA + NR rsqrt seeds per trip (KIND 0: RSQ64H,
// 1: fp32 MUFU.RSQ, 2: MUFU.RCP64H)
template <int NF, int NR, int KIND>
__global__ void __launch_bounds__(128, 5) seed_probe(double* out, int iters) {
  double a[8], f[8];
  float g[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = 1.5 + threadIdx.x + k;
    g[k] = 1.5f + threadIdx.x + k;
    f[k] = 2.0 + k;
  }
  const double m = 1.0000001, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      if (KIND == 0) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(a[k & 7]));
      else if (KIND == 1) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(g[k & 7]));
      else asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a[k & 7]));
    }
#pragma unroll
    for (int k = 0; k < NF; ++k) f[k & 7] = fma(f[k & 7], m, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k] + f[k] + g[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}


// ---- (1c) register-operand probe: DFMAs with 1 / 2 / 3 distinct register
// operands per instruction (the rest repeat from the previous instruction)
template <int KIND>
__global__ void __launch_bounds__(128, 5) operand_probe(double* out, int iters) {
  double a[8], b[8], c[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = threadIdx.x + k;
    b[k] = 1.0 + 1e-9 * (threadIdx.x + k);
    c[k] = 1e-9 * (threadIdx.x + 2 * k);
  }
  const double m = b[3] + out[0];
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (KIND == 0) a[k] = fma(a[k], m, 1e-9);          // 1 register pair read + reuse
      else if (KIND == 1) a[k] = fma(b[k], m, a[k]);     // 2 distinct + 1 repeated
      else if (KIND == 2) a[k] = fma(b[k], c[k], a[k]);  // 3 distinct
      else if (KIND == 3) a[k] = fma(b[k], c[7 - k], a[k]);  // 3 distinct, other pairing
      else a[k] = fma(b[k], b[k], a[k]);                 // one register in two slots + 1 distinct
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x + 1] = s;
}

// ---- (2) evaluation cores ---------------------------------------------------
struct Tgt {
  double ax, ay, az, tt;
};
constexpr int kSrc = 128;

// FORM 0: the product's core (8 FP64: DADD + 3 DFMA, DMUL, DFMA, DMUL, DFMA)
// FORM 1: weight folded into the source (7 FP64: 4 DFMA, DMUL, DFMA, DFMA):
//   staged (x k, y k), (z k, ss k), (k, 3 sgn) with k = sgn(w) / w^2
template <int FORM, int NT>
__device__ __forceinline__ void one_src(const Tgt (&tg)[NT], double (&acc)[NT][2], const double2* src, int jj,
                                        int u) {
  const double2 s0 = src[3 * jj], s1 = src[3 * jj + 1], s2 = src[3 * jj + 2];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    if constexpr (FORM == 0) {
      const double r2 = fma(tg[t].ax, s0.x, fma(tg[t].ay, s0.y, fma(tg[t].az, s1.x, tg[t].tt + s1.y)));
      double y;
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
      const double tt = r2 * y;
      const double h = fma(tt, y, -3.0);
      acc[t][u] = fma(y * h, s2.x, acc[t][u]);
    } else if constexpr (FORM == 1) {  // signed r2', |.| on the high word (one LOP3)
      const double r2 = fma(tg[t].ax, s0.x, fma(tg[t].ay, s0.y, fma(tg[t].az, s1.x, fma(tg[t].tt, s2.x, s1.y))));
      double y;
      const double ar = __hiloint2double(__double2hiint(r2) & 0x7fffffff, 0);
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(ar));
      const double tt = r2 * y;
      const double h = fma(tt, y, -s2.y);
      acc[t][u] = fma(y, h, acc[t][u]);
    } else if constexpr (FORM == 4) {  // FORM 0 with the Newton step through y * y (exact: y has 21 bits)
      const double r2 = fma(tg[t].ax, s0.x, fma(tg[t].ay, s0.y, fma(tg[t].az, s1.x, tg[t].tt + s1.y)));
      double y;
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
      const double h = fma(r2, y * y, -3.0);
      acc[t][u] = fma(y * h, s2.x, acc[t][u]);
    } else if constexpr (FORM == 3) {  // FORM 0 with the seed from the fp32 MUFU.RSQ via bit moves
      const double r2 = fma(tg[t].ax, s0.x, fma(tg[t].ay, s0.y, fma(tg[t].az, s1.x, tg[t].tt + s1.y)));
      const int hi = __double2hiint(r2);
      const unsigned lo = static_cast<unsigned>(__double2loint(r2));
      const int fb = ((hi - 0x38000000) << 3) | static_cast<int>(lo >> 29);
      float yf;
      asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"(__int_as_float(fb)));
      const int yb = __float_as_int(yf);
      const double y = __hiloint2double((yb >> 3) + 0x38000000, yb << 29);
      const double tt = r2 * y;
      const double h = fma(tt, y, -3.0);
      acc[t][u] = fma(y * h, s2.x, acc[t][u]);
    } else {  // FORM 2: sources sorted by sign, r2' = r2 / w^2 > 0 (the caller subtracts the two sums)
      const double r2 = fma(tg[t].ax, s0.x, fma(tg[t].ay, s0.y, fma(tg[t].az, s1.x, fma(tg[t].tt, s2.x, s1.y))));
      double y;
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
      const double tt = r2 * y;
      const double h = fma(tt, y, -3.0);
      acc[t][u] = fma(y, h, acc[t][u]);
    }
  }
}

template <int FORM, int NT, int UN>
__global__ void __launch_bounds__(128, 5) core(const double4* __restrict__ pts, double* out, int reps) {
  __shared__ double2 src[3 * kSrc];
  {
    const double4 v = pts[threadIdx.x];
    const double ss = v.x * v.x + v.y * v.y + v.z * v.z;
    if (FORM == 0) {
      src[3 * threadIdx.x] = make_double2(v.x, v.y);
      src[3 * threadIdx.x + 1] = make_double2(v.z, ss);
      src[3 * threadIdx.x + 2] = make_double2(v.w, 0.0);
    } else {
      const double k = FORM == 1 ? copysign(1.0 / (v.w * v.w), v.w) : 1.0 / (v.w * v.w);
      src[3 * threadIdx.x] = make_double2(v.x * k, v.y * k);
      src[3 * threadIdx.x + 1] = make_double2(v.z * k, ss * k);
      src[3 * threadIdx.x + 2] = make_double2(k, copysign(3.0, v.w));
    }
  }
  Tgt tg[NT];
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const double4 q = pts[1024 + (blockIdx.x * NT + t) * 128 + threadIdx.x];
    const double x = q.x + 3.0, y = q.y, z = q.z;
    tg[t] = Tgt{-2.0 * x, -2.0 * y, -2.0 * z, x * x + y * y + z * z};
    acc[t][0] = acc[t][1] = 0.0;
  }
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int j = 0; j < kSrc; j += UN) {
#pragma unroll
      for (int u = 0; u < UN; ++u) one_src<FORM, NT>(tg, acc, src, j + u, u & 1);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < NT; ++t) s += acc[t][0] + acc[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (FORM == 0 ? -0.5 : -0.5) * s;
}


// Stage-ordered block: NT targets x NS sources, every stage issued for the
// whole block before the next one so that consecutive FP64 instructions share
// an operand (ORD 0: source-major, targets inner; ORD 1: target-major).
template <int NT, int NS, int ORD>
__device__ __forceinline__ void block_eval(const Tgt (&tg)[NT], double (&acc)[NT][2], const double2* src, int j0) {
  double sx[NS], sy[NS], sz[NS], ss[NS], w[NS];
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    const double2 s0 = src[3 * (j0 + j)], s1 = src[3 * (j0 + j) + 1], s2 = src[3 * (j0 + j) + 2];
    sx[j] = s0.x, sy[j] = s0.y, sz[j] = s1.x, ss[j] = s1.y, w[j] = s2.x;
  }
  double q[NT][NS], y[NT][NS];
#define FOR_TJ(body)                                       \
  if (ORD == 0) {                                          \
    _Pragma("unroll") for (int j = 0; j < NS; ++j)         \
        _Pragma("unroll") for (int t = 0; t < NT; ++t) body \
  } else {                                                 \
    _Pragma("unroll") for (int t = 0; t < NT; ++t)         \
        _Pragma("unroll") for (int j = 0; j < NS; ++j) body \
  }
  FOR_TJ({ q[t][j] = tg[t].tt + ss[j]; })
  FOR_TJ({ q[t][j] = fma(tg[t].az, sz[j], q[t][j]); })
  FOR_TJ({ q[t][j] = fma(tg[t].ay, sy[j], q[t][j]); })
  FOR_TJ({ q[t][j] = fma(tg[t].ax, sx[j], q[t][j]); })
  FOR_TJ({ asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y[t][j]) : "d"(q[t][j])); })
  FOR_TJ({ q[t][j] = q[t][j] * y[t][j]; })
  FOR_TJ({ q[t][j] = fma(q[t][j], y[t][j], -3.0); })
  FOR_TJ({ q[t][j] = q[t][j] * y[t][j]; })
  FOR_TJ({ acc[t][j & 1] = fma(q[t][j], w[j], acc[t][j & 1]); })
#undef FOR_TJ
}

template <int NT, int NS, int ORD>
__global__ void __launch_bounds__(128, 5) core_blk(const double4* __restrict__ pts, double* out, int reps) {
  __shared__ double2 src[3 * kSrc];
  {
    const double4 v = pts[threadIdx.x];
    const double ss = v.x * v.x + v.y * v.y + v.z * v.z;
    src[3 * threadIdx.x] = make_double2(v.x, v.y);
    src[3 * threadIdx.x + 1] = make_double2(v.z, ss);
    src[3 * threadIdx.x + 2] = make_double2(v.w, 0.0);
  }
  Tgt tg[NT];
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const double4 q = pts[1024 + (blockIdx.x * NT + t) * 128 + threadIdx.x];
    const double x = q.x + 3.0, y = q.y, z = q.z;
    tg[t] = Tgt{-2.0 * x, -2.0 * y, -2.0 * z, x * x + y * y + z * z};
    acc[t][0] = acc[t][1] = 0.0;
  }
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int j = 0; j < kSrc; j += NS) block_eval<NT, NS, ORD>(tg, acc, src, j);
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < NT; ++t) s += acc[t][0] + acc[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = -0.5 * s;
}


// ---- (3) r^2 on the FP64 tensor-core path: one DMMA m8n8k4 gives the 8 x 8
// block r2[t][j] = [-2t, 1] . [s, |s|^2] + |t|^2 (A: lane l = target l / 4,
// component l % 4; B: source l / 4, component l % 4; C / D: target l / 4,
// sources 2 (l % 4), +1), 4 register-pair reads per 64 values instead of 11
// per value; each lane then runs the Newton form on its 2 values.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
      : "=d"(d0), "=d"(d1)
      : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

template <int NF, int NACC>
__global__ void __launch_bounds__(128, 5) core_mma(const double4* __restrict__ pts, double* out, int reps) {
  __shared__ double sB[4 * kSrc];
  __shared__ double sW[kSrc];
  {
    const double4 v = pts[threadIdx.x];
    sB[4 * threadIdx.x] = v.x, sB[4 * threadIdx.x + 1] = v.y, sB[4 * threadIdx.x + 2] = v.z;
    sB[4 * threadIdx.x + 3] = v.x * v.x + v.y * v.y + v.z * v.z;
    sW[threadIdx.x] = v.w;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = lane >> 2, comp = lane & 3;
  double a[NF], c[NF], acc[NF][NACC];
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const double4 q = pts[1024 + ((blockIdx.x * 4 + warp) * NF + f) * 8 + row];
    const double x = q.x + 3.0, y = q.y, z = q.z;
    a[f] = comp == 0 ? -2.0 * x : comp == 1 ? -2.0 * y : comp == 2 ? -2.0 * z : 1.0;
    c[f] = x * x + y * y + z * z;
#pragma unroll
    for (int u = 0; u < NACC; ++u) acc[f][u] = 0.0;
  }
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int j = 0; j < kSrc; j += 8) {
      const double b = sB[4 * (j + row) + comp];
      const double2 w = *reinterpret_cast<const double2*>(&sW[j + 2 * comp]);
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        double d0, d1;
        dmma884(d0, d1, a[f], b, c[f], c[f]);
        double y0, y1;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(d0));
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y1) : "d"(d1));
        const double h0 = fma(d0 * y0, y0, -3.0), h1 = fma(d1 * y1, y1, -3.0);
        acc[f][0] = fma(y0 * h0, w.x, acc[f][0]);
        acc[f][NACC - 1] = fma(y1 * h1, w.y, acc[f][NACC - 1]);
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int u = 0; u < NACC; ++u) s += acc[f][u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = -0.5 * s;
}


// ---- (4) r^2 stages written as PTX blocks, one per stage and source, the
// targets adjacent (shared source operand in the same slot): does ptxas keep
// them together and set .reuse?
template <int NT>
__device__ __forceinline__ void stage_add(double (&q)[NT], const Tgt (&tg)[NT], double ss) {
  if constexpr (NT == 4)
    asm("add.f64 %0, %4, %8;\n\tadd.f64 %1, %5, %8;\n\tadd.f64 %2, %6, %8;\n\tadd.f64 %3, %7, %8;"
        : "=d"(q[0]), "=d"(q[1]), "=d"(q[2]), "=d"(q[3])
        : "d"(tg[0].tt), "d"(tg[1].tt), "d"(tg[2].tt), "d"(tg[3].tt), "d"(ss));
  else
    asm("add.f64 %0, %2, %4;\n\tadd.f64 %1, %3, %4;" : "=d"(q[0]), "=d"(q[1]) : "d"(tg[0].tt), "d"(tg[1].tt), "d"(ss));
}
template <int NT>
__device__ __forceinline__ void stage_fma(double (&q)[NT], double a0, double a1, double a2, double a3, double s) {
  if constexpr (NT == 4)
    asm("fma.rn.f64 %0, %4, %8, %0;\n\tfma.rn.f64 %1, %5, %8, %1;\n\tfma.rn.f64 %2, %6, %8, %2;\n\tfma.rn.f64 %3, %7, %8, %3;"
        : "+d"(q[0]), "+d"(q[1]), "+d"(q[2]), "+d"(q[3])
        : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(s));
  else
    asm("fma.rn.f64 %0, %2, %4, %0;\n\tfma.rn.f64 %1, %3, %4, %1;" : "+d"(q[0]), "+d"(q[1]) : "d"(a0), "d"(a1), "d"(s));
}

template <int NT, int NS>
__global__ void __launch_bounds__(128, 4) core_ptx(const double4* __restrict__ pts, double* out, int reps) {
  __shared__ double2 src[3 * kSrc];
  {
    const double4 v = pts[threadIdx.x];
    const double ss = v.x * v.x + v.y * v.y + v.z * v.z;
    src[3 * threadIdx.x] = make_double2(v.x, v.y);
    src[3 * threadIdx.x + 1] = make_double2(v.z, ss);
    src[3 * threadIdx.x + 2] = make_double2(v.w, 0.0);
  }
  Tgt tg[NT];
  double acc[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const double4 q = pts[1024 + (blockIdx.x * NT + t) * 128 + threadIdx.x];
    const double x = q.x + 3.0, y = q.y, z = q.z;
    tg[t] = Tgt{-2.0 * x, -2.0 * y, -2.0 * z, x * x + y * y + z * z};
    acc[t] = 0.0;
  }
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int j0 = 0; j0 < kSrc; j0 += NS) {
      double q[NS][NT], w[NS];
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        const double2 s0 = src[3 * (j0 + j)], s1 = src[3 * (j0 + j) + 1], s2 = src[3 * (j0 + j) + 2];
        w[j] = s2.x;
        stage_add<NT>(q[j], tg, s1.y);
        if constexpr (NT == 4) {
          stage_fma<NT>(q[j], tg[0].az, tg[1].az, tg[2].az, tg[3].az, s1.x);
          stage_fma<NT>(q[j], tg[0].ay, tg[1].ay, tg[2].ay, tg[3].ay, s0.y);
          stage_fma<NT>(q[j], tg[0].ax, tg[1].ax, tg[2].ax, tg[3].ax, s0.x);
        } else {
          stage_fma<NT>(q[j], tg[0].az, tg[1].az, 0.0, 0.0, s1.x);
          stage_fma<NT>(q[j], tg[0].ay, tg[1].ay, 0.0, 0.0, s0.y);
          stage_fma<NT>(q[j], tg[0].ax, tg[1].ax, 0.0, 0.0, s0.x);
        }
      }
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        double g[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          double y;
          asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q[j][t]));
          const double h = fma(q[j][t] * y, y, -3.0);
          g[t] = y * h;
        }
        stage_fma<NT>(acc, g[0], g[1], NT == 4 ? g[NT - 2] : 0.0, NT == 4 ? g[NT - 1] : 0.0, w[j]);
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < NT; ++t) s += acc[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = -0.5 * s;
}


// ---- (5) many targets per thread, one (or two) sources per trip, not unrolled
// over sources: the only independent work in a trip is the NT targets of the
// same source, so ptxas has little choice but to keep them adjacent
template <int NT, int NS>
__global__ void __launch_bounds__(128, 4) core_wide(const double4* __restrict__ pts, double* out, int reps) {
  __shared__ double2 src[3 * kSrc];
  {
    const double4 v = pts[threadIdx.x];
    const double ss = v.x * v.x + v.y * v.y + v.z * v.z;
    src[3 * threadIdx.x] = make_double2(v.x, v.y);
    src[3 * threadIdx.x + 1] = make_double2(v.z, ss);
    src[3 * threadIdx.x + 2] = make_double2(v.w, 0.0);
  }
  Tgt tg[NT];
  double acc[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const double4 q = pts[1024 + ((blockIdx.x * NT + t) * 128 + threadIdx.x) % (1 << 20)];
    const double x = q.x + 3.0, y = q.y, z = q.z;
    tg[t] = Tgt{-2.0 * x, -2.0 * y, -2.0 * z, x * x + y * y + z * z};
    acc[t] = 0.0;
  }
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int j0 = 0; j0 < kSrc; j0 += NS) {
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        const double2 s0 = src[3 * (j0 + j)], s1 = src[3 * (j0 + j) + 1], s2 = src[3 * (j0 + j) + 2];
        double q[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) q[t] = tg[t].tt + s1.y;
#pragma unroll
        for (int t = 0; t < NT; ++t) q[t] = fma(tg[t].az, s1.x, q[t]);
#pragma unroll
        for (int t = 0; t < NT; ++t) q[t] = fma(tg[t].ay, s0.y, q[t]);
#pragma unroll
        for (int t = 0; t < NT; ++t) q[t] = fma(tg[t].ax, s0.x, q[t]);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          double y;
          asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q[t]));
          const double h = fma(q[t] * y, y, -3.0);
          q[t] = y * h;
        }
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[t] = fma(q[t], s2.x, acc[t]);
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < NT; ++t) s += acc[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = -0.5 * s;
}

template <class F>
float timed(F launch) {
  launch();
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("kernel failed: %s\n", cudaGetErrorString(cudaGetLastError()));
    exit(1);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double) * (1 << 22)) != cudaSuccess) {
    printf("no device\n");
    return 1;
  }
  printf("start\n");
  const int blocks = 148 * 5 * 4;
  {
    const int iters = 1 << 15;
#define PROBE(NI, NL)                                                                      \
  {                                                                                        \
    const float ms = timed([&] { issue_probe<NI, NL><<<blocks, 128>>>(out, iters); });     \
    const double f = double(blocks) * 128 * iters * (8 + NL);                              \
    printf("8 DFMA + %d IMAD + %d (LDS.128 + DADD): %.3f ms, %.2f T FP64 instr/s\n", NI, NL, ms, \
           f / ms / 1e9);                                                                  \
  }
    PROBE(0, 0) PROBE(2, 0) PROBE(4, 0) PROBE(8, 0) PROBE(0, 2) PROBE(0, 4) PROBE(4, 2)
  }
  {
    const int iters = 1 << 14;
#define SEED(NF, NR, KIND)                                                                  \
  {                                                                                         \
    const float ms = timed([&] { seed_probe<NF, NR, KIND><<<blocks, 128>>>(out, iters); }); \
    printf("%d DFMA + %d seeds (kind %d): %.3f ms; DFMA alone would take %.3f ms; seeds %.2f per SM per clock\n", NF, NR, KIND, ms, \
           double(blocks) * 128 * iters * NF / 18.37e9, double(blocks) * 128 * iters * NR / (ms * 1e-3) / 148 / 1.965e9); \
  }
    SEED(0, 8, 0) SEED(0, 8, 1) SEED(0, 8, 2) SEED(8, 1, 0) SEED(8, 2, 0) SEED(8, 1, 1) SEED(8, 2, 1) SEED(16, 1, 0) SEED(16, 2, 0)
  }
  {
    const int iters = 1 << 15;
    cudaMemset(out, 0, 8);
#define OPER(KIND)                                                                        \
  {                                                                                       \
    const float ms = timed([&] { operand_probe<KIND><<<blocks, 128>>>(out, iters); });    \
    printf("operand probe kind %d: %.3f ms, %.2f T DFMA/s\n", KIND, ms, double(blocks) * 128 * iters * 8 / ms / 1e9); \
  }
    OPER(0) OPER(1) OPER(2) OPER(3) OPER(4)
  }
  const int npts = 1024 + blocks * 4 * 128 + 64;
  double4* h = new double4[npts];
  for (int i = 0; i < npts; ++i) {
    auto u = [&](int k) { const double v = (i * 4 + k) * 0.6180339887; return 2.0 * (v - (long long)v) - 1.0; };
    h[i] = make_double4(u(0), u(1), u(2), u(3));
  }
  double4* pts;
  cudaMalloc(&pts, sizeof(double4) * npts);
  cudaMemcpy(pts, h, sizeof(double4) * npts, cudaMemcpyHostToDevice);
  double* ho = new double[blocks * 128];
  const int reps = 400;
#define CORE(FORM, NT, UN)                                                                          \
  {                                                                                                 \
    const int bl = blocks * 2 / NT;                                                                 \
    const float ms = timed([&] { core<FORM, NT, UN><<<bl, 128>>>(pts, out, reps); });               \
    const double ev = double(bl) * 128 * NT * kSrc * reps;                                          \
    cudaMemcpy(ho, out, sizeof(double) * 128, cudaMemcpyDeviceToHost);                              \
    printf("core form %d, %d targets/thread, %d sources/trip: %.3f ms, %.3f T evals/s (out[5] %.15g)\n", \
           FORM, NT, UN, ms, ev / ms / 1e9, ho[5]);                                                 \
  }
  CORE(0, 2, 4) CORE(0, 2, 8) CORE(0, 4, 4) CORE(0, 4, 2) CORE(0, 1, 8)
  CORE(1, 2, 4) CORE(1, 2, 8) CORE(1, 4, 4) CORE(1, 4, 2) CORE(1, 1, 8)
  CORE(4, 2, 4) CORE(4, 4, 4) CORE(4, 2, 8)
  CORE(2, 2, 4) CORE(2, 2, 8) CORE(2, 4, 4) CORE(2, 4, 2) CORE(2, 1, 8) CORE(2, 2, 2)
#define BLK(NT, NS, ORD)                                                                            \
  {                                                                                                 \
    const int bl = blocks * 2 / NT;                                                                 \
    const float ms = timed([&] { core_blk<NT, NS, ORD><<<bl, 128>>>(pts, out, reps); });            \
    const double ev = double(bl) * 128 * NT * kSrc * reps;                                          \
    cudaMemcpy(ho, out, sizeof(double) * 128, cudaMemcpyDeviceToHost);                              \
    printf("block core %d targets x %d sources, order %d: %.3f ms, %.3f T evals/s (out[5] %.15g)\n", \
           NT, NS, ORD, ms, ev / ms / 1e9, ho[5]);                                                  \
  }
  BLK(2, 4, 0) BLK(2, 4, 1) BLK(4, 2, 0) BLK(4, 2, 1) BLK(4, 4, 0) BLK(4, 4, 1) BLK(2, 8, 1) BLK(2, 2, 0)
#define MMA(NF, NACC)                                                                               \
  {                                                                                                 \
    const int bl = blocks * 2 * 8 / NF;                                                             \
    const float ms = timed([&] { core_mma<NF, NACC><<<bl, 128>>>(pts, out, reps); });               \
    const double ev = double(bl) * 4 * NF * 8 * kSrc * reps;                                        \
    cudaMemcpy(ho, out, sizeof(double) * 128, cudaMemcpyDeviceToHost);                              \
    printf("dmma core %d fragments (%d targets) per warp, %d accumulators: %.3f ms, %.3f T evals/s (out[5] %.15g)\n", \
           NF, NF * 8, NACC, ms, ev / ms / 1e9, ho[5]);                                             \
  }
  MMA(8, 1) MMA(8, 2) MMA(4, 2) MMA(4, 1) MMA(2, 2)
#define PTXC(NT, NS)                                                                                \
  {                                                                                                 \
    const int bl = blocks * 2 / NT;                                                                 \
    const float ms = timed([&] { core_ptx<NT, NS><<<bl, 128>>>(pts, out, reps); });                 \
    const double ev = double(bl) * 128 * NT * kSrc * reps;                                          \
    cudaMemcpy(ho, out, sizeof(double) * 128, cudaMemcpyDeviceToHost);                              \
    printf("ptx-staged core %d targets x %d sources per trip: %.3f ms, %.3f T evals/s (out[5] %.15g)\n", \
           NT, NS, ms, ev / ms / 1e9, ho[5]);                                                       \
  }
  PTXC(2, 4) PTXC(4, 2) PTXC(4, 4) PTXC(2, 2) PTXC(4, 1)
#define WIDE(NT, NS)                                                                                \
  {                                                                                                 \
    const int bl = blocks * 2 / NT;                                                                 \
    const float ms = timed([&] { core_wide<NT, NS><<<bl, 128>>>(pts, out, reps); });                \
    const double ev = double(bl) * 128 * NT * kSrc * reps;                                          \
    printf("wide core %d targets/thread, %d sources per trip (no unroll): %.3f ms, %.3f T evals/s\n", NT, NS, ms, \
           ev / ms / 1e9);                                                                          \
  }
  WIDE(4, 1) WIDE(8, 1) WIDE(8, 2) WIDE(4, 2) WIDE(6, 1) WIDE(6, 2)
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
