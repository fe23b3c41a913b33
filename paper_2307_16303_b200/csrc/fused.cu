// Fused proxy pass for kModeFused levels (planner.h): every admissible pair
// (X, Y) is applied from the reference's own storage (pivots sigma in X, tau
// in Y and the packed pivot LU, lowrank.cpp:277-327), both orientations in
// one visit, with every regenerated kernel entry evaluated ONCE:
//
//   E_X[k][q] = K(tau_k, q)  (q in X),      E_Y[k][q] = K(sigma_k, q)  (q in Y)
//   v_X = E_X x_X = K(tau, X) x_X,          v_Y = E_Y x_Y = K(sigma, Y) x_Y
//   s_X = R^-1 L^-1 v_Y,                    s_Y = L^-T R^-T v_X      (lowrank.cpp:310-320)
//   b_X += E_X^T s_X,                       b_Y += E_Y^T s_Y
//
// K(X, tau) is the transpose of K(tau, X) (the kernels are symmetric,
// kernel.cpp:7-21), so the entries phase 1 evaluates for one orientation are
// the phase-2 entries of the other. The two-phase proxy path (matvec.cu)
// evaluates each of them twice; here they stay in shared memory between the
// phases (rows k < kc; rows above the cache are evaluated again).
//
// One 2-CTA cluster per pair at a time (static interleave over the clusters,
// deterministic): CTA 0 holds node X, CTA 1 node Y. Each evaluates its node's
// points against the partner's pivots, keeps the entries, and sums its v;
// the two v vectors cross over distributed shared memory (one cluster
// barrier per pair, double-buffered by pair parity); each CTA then solves
// its own side and applies the cached entries. Two clusters share an SM, so
// one CTA's solve and setup latency overlap another's evaluation. Thread t
// owns point t of its node; the products e x feed the v sums through
// a reduce-scatter over the warp (8 pivots per 9 shuffles) plus a fixed-order
// sum over warps. The LU inverses (lu_invert_kernel) are bulk-copied into
// shared memory when they fit beside the full entry cache, else read from L2
// (prefetched at pair start).
#include <algorithm>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace h3db {

namespace {

constexpr int kFThreads = 352;
constexpr int kFWarps = kFThreads / 32;
constexpr int kFMaxNode = kFThreads;      // points per node (one per thread)
constexpr int kFPool = 11776;             // 92 KB: [staged LU | entry cache]
constexpr double kFarCoord = 1e100;       // padding points: far away, weight 0
constexpr int kR = kFusedMaxRank;

struct FusedSmem {
  double pool[kFPool];
  double4 pv[kR];            // partner pivots, centred and scaled (-2 p', |p'|^2)
  double vw[kFWarps][kR];    // per-warp partial v sums / triangular-step partials
  double vout[2][kR];        // this node's v (read by the partner CTA), by pair parity
  double vin[kR], tmp[kR], s[kR];
  unsigned long long lu_bar;
};

// scaled admissible entry: far_acc<K>(r2, 1, 0) without the accumulate
template <int K>
__device__ __forceinline__ double fent(double r2) {
  if constexpr (K == kLaplace) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
    const double t = r2 * y;
    return y * fma(t, y, -3.0);
  } else if constexpr (K == kR4) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
    const double t = r2 * y;
    const double g = y * fma(t, y, -3.0);
    const double g2 = g * g;
    return g2 * g2;
  } else {
    return kernel_r2<K>(r2);
  }
}

// r^2 between pivot p (scaled: a = -2 p', tt = |p'|^2) and point q (q', qq),
// both relative to the pair centre; touching boxes use the difference form
template <bool TOUCH>
__device__ __forceinline__ double pr2(const double4& p, double qx, double qy, double qz, double qq) {
  if constexpr (TOUCH) return sq3(fma(-0.5, p.x, -qx), fma(-0.5, p.y, -qy), fma(-0.5, p.z, -qz));
  else return fma(p.x, qx, fma(p.y, qy, fma(p.z, qz, p.w + qq)));
}

// Sum of v[r] over the 32 lanes for 8 rows at once: returns, in every lane,
// the total of row (lane >> 2) & 7.
__device__ __forceinline__ double reduce8(const double (&v)[8], int lane) {
  const int b = (lane >> 4) & 1, c = (lane >> 3) & 1, d = (lane >> 2) & 1;
  double k4[4], k2[2];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double send = b ? v[q] : v[4 + q];
    const double keep = b ? v[4 + q] : v[q];
    k4[q] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const double send = c ? k4[q] : k4[2 + q];
    const double keep = c ? k4[2 + q] : k4[q];
    k2[q] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  double r = (d ? k2[1] : k2[0]) + __shfl_xor_sync(0xffffffffu, d ? k2[0] : k2[1], 4);
  r += __shfl_xor_sync(0xffffffffu, r, 2);
  r += __shfl_xor_sync(0xffffffffu, r, 1);
  return r;
}

// Evaluation of pivots [kb, kb + 8) for this thread's point: entries stored
// (E[k * stride + t]) when STORE, v partial to vw[warp][k].
template <int K, bool TOUCH, bool STORE, bool TAIL>
__device__ __forceinline__ void eval_block(FusedSmem& sm, double* E, int kb, int r, int stride, int tid,
                                           int warp, int lane, const double (&q)[4], double xq) {
  double prod[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int k = TAIL ? min(kb + u, r - 1) : kb + u;
    const double e = fent<K>(pr2<TOUCH>(sm.pv[k], q[0], q[1], q[2], q[3]));
    if (STORE && (!TAIL || kb + u < r)) E[(kb + u) * stride + tid] = e;
    prod[u] = (TAIL && kb + u >= r) ? 0.0 : e * xq;
  }
  const double v = reduce8(prod, lane);
  const int k = kb + ((lane >> 2) & 7);
  if ((lane & 3) == 0 && (!TAIL || k < r)) sm.vw[warp][k] = v;
}

// all pivots; kc (cached rows) is r or a multiple of 8
template <int K, bool TOUCH>
__device__ __forceinline__ void eval_pass(FusedSmem& sm, double* E2, int r, int kc, int half, int tid,
                                          int warp, int lane, const double (&q)[4], double xq) {
  const int r8 = r & ~7;
  int kb = 0;
  for (; kb < min(kc, r8); kb += 8)
    eval_block<K, TOUCH, true, false>(sm, E2, kb, r, half, tid, warp, lane, q, xq);
  for (; kb < r8; kb += 8)
    eval_block<K, TOUCH, false, false>(sm, E2, kb, r, half, tid, warp, lane, q, xq);
  if (kb < r) {
    if (kc == r) eval_block<K, TOUCH, true, true>(sm, E2, kb, r, half, tid, warp, lane, q, xq);
    else eval_block<K, TOUCH, false, true>(sm, E2, kb, r, half, tid, warp, lane, q, xq);
  }
}

// sum_k E[k][q] s[k] for this thread's point: cached rows, then rows k >= kc
// evaluated again
template <int K, bool TOUCH>
__device__ __forceinline__ double apply_pass(const FusedSmem& sm, const double* E, int r, int kc, int stride,
                                             int tid, const double (&q)[4]) {
  const double* s = sm.s;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int k = 0;
#pragma unroll 2
  for (; k + 3 < kc; k += 4) {
    a0 = fma(E[k * stride + tid], s[k], a0);
    a1 = fma(E[(k + 1) * stride + tid], s[k + 1], a1);
    a2 = fma(E[(k + 2) * stride + tid], s[k + 2], a2);
    a3 = fma(E[(k + 3) * stride + tid], s[k + 3], a3);
  }
  for (; k < kc; ++k) a0 = fma(E[k * stride + tid], s[k], a0);
  for (; k < r; ++k) a1 = fma(fent<K>(pr2<TOUCH>(sm.pv[k], q[0], q[1], q[2], q[3])), s[k], a1);
  return (a0 + a1) + (a2 + a3);
}

// One triangular GEMV step of this CTA's solve, spread over its 8 warps
// (lu_invert_kernel: P row-major, PT = the same matrix column-major):
//   X (side 0, M = PT):  step 0  w_i = v_i + sum_{j<i} PT[j][i] v_j,  step 1  s_i = sum_{j>=i} PT[j][i] w_j
//   Y (side 1, M = P):   step 0  u_i = sum_{j<=i} P[j][i] v_j,        step 1  s_i = u_i + sum_{j>i} P[j][i] u_j
// (the reference's forward / back substitution as two triangular GEMVs).
// Warp w sums rows j of its slice (lane = output i, loads of 4 rows issued
// together), partials to part[w][i].
template <int NK, int STEP>
__device__ __forceinline__ void tri_slice(int side, int r, int w, const double* __restrict__ M, const double* x,
                                          double (*part)[kR], int lane) {
  const int j0 = w * r / kFWarps, j1 = (w + 1) * r / kFWarps;
  double acc[NK];
#pragma unroll
  for (int t = 0; t < NK; ++t) acc[t] = 0.0;
  for (int jb = j0; jb < j1; jb += 4) {
    double f[4][NK], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = min(jb + u, j1 - 1);
      xv[u] = jb + u < j1 ? x[j] : 0.0;
      const double* row = M + static_cast<long long>(j) * r;
#pragma unroll
      for (int t = 0; t < NK; ++t) f[u][t] = row[min(lane + 32 * t, r - 1)];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = jb + u;
#pragma unroll
      for (int t = 0; t < NK; ++t) {
        const int i = lane + 32 * t;
        const bool on = STEP == 0 ? (side == 0 ? j < i : j <= i) : (side == 0 ? j >= i : j > i);
        acc[t] = fma(on ? f[u][t] : 0.0, xv[u], acc[t]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < NK; ++t) {
    const int i = lane + 32 * t;
    if (i < r) part[w][i] = acc[t];
  }
}

template <int STEP>
__device__ __forceinline__ void tri_step(int side, int r, int warp, int lane, const double* M, const double* x,
                                         double (*part)[kR]) {
  switch ((r + 31) >> 5) {
    case 1: tri_slice<1, STEP>(side, r, warp, M, x, part, lane); break;
    case 2: tri_slice<2, STEP>(side, r, warp, M, x, part, lane); break;
    case 3: tri_slice<3, STEP>(side, r, warp, M, x, part, lane); break;
    default: tri_slice<4, STEP>(side, r, warp, M, x, part, lane); break;
  }
}

template <int K>
__global__ void __launch_bounds__(kFThreads, 2) fused_kernel(const FusedArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  FusedSmem& sm = *reinterpret_cast<FusedSmem*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int side = static_cast<int>(cluster.block_rank());  // 0: node X, 1: node Y
  const long long ncl = gridDim.x / 2, cl = blockIdx.x / 2;
  FusedSmem* peer = cluster.map_shared_rank(&sm, side ^ 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double4* __restrict__ p4 = reinterpret_cast<const double4*>(a.p4);
  if (tid == 0) {
    mbar_init(&sm.lu_bar, 1);
    mbar_fence_init();
  }
  unsigned lu_phase = 0, parity = 0;
  // optional phase profile (thread 0): cycles from pair start to pivots
  // staged, evaluation done, v exchanged, solve done, apply done
  unsigned long long ph[kFusedProfSlots] = {0, 0, 0, 0, 0, 0}, tp = 0;
  auto mark = [&](int slot) {
    if (a.prof != nullptr && tid == 0) {
      const unsigned long long now = clock64();
      ph[slot] += now - tp;
      tp = now;
    }
  };
  for (long long pk = cl; pk < a.n; pk += ncl, parity ^= 1u) {
    if (a.prof != nullptr && tid == 0) {
      tp = clock64();
      ++ph[5];
    }
    const FusedDesc d = a.descs[pk];
    const int r = d.r;
    const int m = side == 0 ? d.m : d.n;                  // this node's points
    const long long row0 = side == 0 ? d.xrow : d.yrow;   // its first permuted row
    const long long prow0 = side == 0 ? d.yrow : d.xrow;  // partner node (pivots)
    const int wall = (m + 31) >> 5;                       // warps with points
    const int stride = 32 * wall;                         // E row stride (one per thread)
    // side 0 solves with PT, side 1 with P; staged when it fits beside the
    // full entry cache, else read from L2 (prefetched below)
    const double* Mg = a.lu + d.lu_off + (side == 0 ? a.lu_total : 0);
    const int lus = (r * r + 1) & ~1;
    const bool stage = lus + stride * r <= kFPool;
    const int lusz = stage ? lus : 0;
    int kc = min(r, (kFPool - lusz) / stride);
    if (kc < r) kc &= ~7;  // partial cache: whole blocks of 8 pivots
    double* E = sm.pool + lusz;
    __syncthreads();  // previous pair done with every shared buffer
    if (stage) {
      if (tid == 0) {
        const unsigned tb = static_cast<unsigned>(lus) * 8u;
        mbar_arrive_tx(&sm.lu_bar, tb);
        bulk_g2s(sm.pool, Mg, tb, &sm.lu_bar, l2_evict_first());
      }
    } else {
      const int lines = (r * r * 8 + 127) / 128;
      for (int l = tid; l < lines; l += kFThreads) asm volatile("prefetch.global.L2 [%0];" ::"l"(Mg + 16LL * l));
    }
    // partner pivots (X holds tau, the column pivots in Y; Y holds sigma)
    for (int k = tid; k < r; k += kFThreads) {
      const std::int32_t loc = a.piv[d.piv_off + (side == 0 ? r : 0) + k];
      const double4 v = p4[prow0 + loc];
      const double x = v.x - d.cx, y = v.y - d.cy, z = v.z - d.cz;
      sm.pv[k] = make_double4(-2.0 * x, -2.0 * y, -2.0 * z, fma(z, z, fma(y, y, x * x)));
    }
    // this thread's point
    double q[4], xq = 0.0;
    if (tid < m) {
      const double4 v = p4[row0 + tid];
      const double x = v.x - d.cx, y = v.y - d.cy, z = v.z - d.cz;
      q[0] = x;
      q[1] = y;
      q[2] = z;
      q[3] = fma(z, z, fma(y, y, x * x));
      xq = v.w;
    } else {
      q[0] = q[1] = q[2] = kFarCoord;
      q[3] = 3.0 * kFarCoord * kFarCoord;
    }
    __syncthreads();  // pivots staged
    mark(0);
    const bool active = warp < wall;  // warp-uniform
    if (active) {
      if (d.touch) eval_pass<K, true>(sm, E, r, kc, stride, tid, warp, lane, q, xq);
      else eval_pass<K, false>(sm, E, r, kc, stride, tid, warp, lane, q, xq);
    }
    __syncthreads();
    mark(1);
    for (int k = tid; k < r; k += kFThreads) {
      double acc = 0.0;
      for (int w = 0; w < wall; ++w) acc += sm.vw[w][k];
      sm.vout[parity][k] = far_scale<K>() * acc;
    }
    cluster.sync();  // both v ready (and the partner is past its previous pair)
    for (int k = tid; k < r; k += kFThreads) sm.vin[k] = peer->vout[parity][k];
    if (stage) {
      mbar_wait(&sm.lu_bar, lu_phase);
      lu_phase ^= 1u;
    }
    __syncthreads();
    mark(2);
    const double* M = stage ? sm.pool : Mg;
    tri_step<0>(side, r, warp, lane, M, sm.vin, sm.vw);
    __syncthreads();
    for (int i = tid; i < r; i += kFThreads) {
      double acc = 0.0;
#pragma unroll
      for (int w = 0; w < kFWarps; ++w) acc += sm.vw[w][i];
      sm.tmp[i] = side == 0 ? sm.vin[i] + acc : acc;  // w = L^-1 v  /  u = R^-T v
    }
    __syncthreads();
    tri_step<1>(side, r, warp, lane, M, sm.tmp, sm.vw);
    __syncthreads();
    for (int i = tid; i < r; i += kFThreads) {
      double acc = 0.0;
#pragma unroll
      for (int w = 0; w < kFWarps; ++w) acc += sm.vw[w][i];
      sm.s[i] = side == 0 ? acc : sm.tmp[i] + acc;  // s = R^-1 w  /  L^-T u
    }
    __syncthreads();
    mark(3);
    if (active && (d.own & (side == 0 ? 1 : 2))) {
      const double o = d.touch ? apply_pass<K, true>(sm, E, r, kc, stride, tid, q)
                               : apply_pass<K, false>(sm, E, r, kc, stride, tid, q);
      if (tid < m) a.out[d.out + (side == 0 ? 0 : d.m) + tid] = far_scale<K>() * o;
    }
    if (a.prof != nullptr) {
      __syncthreads();
      mark(4);
    }
  }
  if (a.prof != nullptr && tid == 0)
    for (int q = 0; q < kFusedProfSlots; ++q) a.prof[blockIdx.x * kFusedProfSlots + q] = ph[q];
  cluster.sync();  // the partner may still read this CTA's last v
}

template <int K>
void launch_fused_t(const FusedArgs& a, cudaStream_t s) {
  const void* f = reinterpret_cast<const void*>(fused_kernel<K>);
  static PerDeviceOnce attr;
  attr([f] {
    H3D_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sizeof(FusedSmem))));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kFThreads);
  cfg.dynamicSmemBytes = sizeof(FusedSmem);
  cfg.stream = s;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = 2;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  // co-resident clusters, per device (the occupancy query is device-specific)
  static int max_cl_dev[64] = {};
  int dev = 0;
  H3D_CUDA_CHECK(cudaGetDevice(&dev));
  int& max_cl = max_cl_dev[dev & 63];
  if (max_cl == 0) {
    cfg.gridDim = dim3(2);
    int m = 0;
    H3D_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&m, f, &cfg));
    max_cl = std::max(m, 1);
  }
  const std::int64_t ncl = std::max<std::int64_t>(1, std::min<std::int64_t>(max_cl, a.n));
  cfg.gridDim = dim3(static_cast<unsigned>(2 * ncl));
  void* args[] = {const_cast<FusedArgs*>(&a)};
  H3D_CUDA_CHECK(cudaLaunchKernelExC(&cfg, f, args));
}

}  // namespace

int fused_max_node() { return kFMaxNode; }

void launch_fused(const FusedArgs& a, int kernel, int sms, cudaStream_t s) {
  (void)sms;  // grid = the co-resident clusters (two CTAs per SM)
  if (a.n == 0) return;
  switch (kernel) {
    case kLaplace: launch_fused_t<kLaplace>(a, s); break;
    case kR4: launch_fused_t<kR4>(a, s); break;
    default: launch_fused_t<kHelmholtz>(a, s); break;
  }
}

}  // namespace h3db
