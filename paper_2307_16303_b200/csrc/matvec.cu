// HODLR3D matvec kernels (reference hmatrix.cpp:153-226, Algorithm 2).
//
// Every admissible block (Z,k) is F_Z F_k^T with F_Z = K(Z, P_Zk) M_Zk, where
// P_Zk are the ACA pivots of the pair that lie in k ("proxies") and M_Zk a
// triangular factor of the pivot LU (reference lowrank.cpp:291-327). Per node Z
// the partner segments share one column layout (rpad_Z columns):
//
//   stream levels : W_Z = [F_Z^(Z,k1) | ...] stored row-major and streamed (HBM);
//   proxy levels  : only proxy coordinates + pivots + LU are stored and the
//                   entries K(Z, P_Z) are regenerated (FP64 pipes);
//   direct (leaf) : leaf-level admissible blocks are evaluated exactly and
//                   join the near field.
//
// Two resources, two kernels per phase, run concurrently on two CUDA streams
// as persistent CTAs that co-reside on every SM:
//
//   phase 1  p1_stream_kernel : T_Z = W_Z^T x_Z           (HBM)
//            p1_proxy_kernel  : v_Z = K(P_Z, Z) x_Z         (FP64, lane = target)
//            -> scattered through spos into S (target-major t-vectors),
//               partial sums of tall nodes reduced in fixed order;
//   solve    proxy_solve_kernel: s = (LU)^-1 v or (U^T L^T)^-1 v in place;
//   phase 2  p2_stream_kernel : rows of W_A(l) . S_A(l) over stream levels (HBM)
//            p2_compute_kernel: near field + direct leaf blocks + K(X, P_A) s_A
//                               over proxy levels, one continuous source walk
//                               per warp, lane = target row (FP64)
//            combine_kernel   : b[perm[p]] = compute + stream (fused un-permute).
//
// Every output has one writer and a fixed accumulation order (no atomics), so
// matvecs are bitwise reproducible (reference hmatrix.hpp:68-69).
#include "common.cuh"
#include "kernels.h"

namespace h3db {

namespace {

constexpr double kFar = 1e100;  // coordinate of padding / inactive targets
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kP1Cols = 256;    // phase-1 columns per item
constexpr int kChunk = 256;     // phase-1 proxy: sources staged per round
constexpr int kMaxRanges = 256; // phase-2 compute: source ranges per tile

__global__ void gather_kernel(const double* __restrict__ x, const std::int32_t* __restrict__ perm,
                              std::int64_t n, double* __restrict__ xp) {
  const std::int64_t p = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (p < n) xp[p] = __ldg(x + perm[p]);
}

__device__ __forceinline__ void p1_write(const P1Item& it, std::int64_t g, int c, double v,
                                         const P1Args& a) {
  if (it.pslot < 0) {
    const std::int32_t dst = a.spos[a.nt.soff[g] + it.col0 + c];
    if (dst >= 0) a.S[dst] = v;
  } else {
    a.P[it.pslot + c] = v;
  }
}

// ---- phase 1, stream levels: T = W_Z^T x_Z over <= 2048 rows x 256 columns
__global__ void __launch_bounds__(kThreads, 2) p1_stream_kernel(const P1Args a) {
  __shared__ double red[kWarps][kP1Cols + 2];
  __shared__ long long s_k;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_k = static_cast<long long>(atomicAdd(a.counter, 1u));
    __syncthreads();
    const long long k = s_k;
    if (k >= a.nitems) break;
    const P1Item it = a.items[k];
    const std::int64_t g = it.node;
    const int rpad = a.nt.rpad[g];
    const double* __restrict__ Wn =
        a.W + a.nt.woff[g] + static_cast<std::int64_t>(it.row0) * rpad + it.col0;
    const double* __restrict__ xn = a.xp + a.nt.rowbeg[g] + it.row0;
    const int ng = (it.ncols + 63) >> 6;
    double acc[4][2];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = 0.0;
    int i = warp;
    for (; i + kWarps < it.nrows; i += 2 * kWarps) {
      const double x0 = xn[i], x1 = xn[i + kWarps];
      const double2* r0 = reinterpret_cast<const double2*>(Wn + static_cast<std::int64_t>(i) * rpad);
      const double2* r1 =
          reinterpret_cast<const double2*>(Wn + static_cast<std::int64_t>(i + kWarps) * rpad);
      double2 w0[4], w1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool ok = q < ng && (2 * lane + 64 * q) < it.ncols;
        w0[q] = ok ? ld_stream(r0 + lane + 32 * q) : make_double2(0.0, 0.0);
        w1[q] = ok ? ld_stream(r1 + lane + 32 * q) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[q][0] = fma(w0[q].x, x0, acc[q][0]);
        acc[q][1] = fma(w0[q].y, x0, acc[q][1]);
        acc[q][0] = fma(w1[q].x, x1, acc[q][0]);
        acc[q][1] = fma(w1[q].y, x1, acc[q][1]);
      }
    }
    for (; i < it.nrows; i += kWarps) {
      const double x0 = xn[i];
      const double2* r0 = reinterpret_cast<const double2*>(Wn + static_cast<std::int64_t>(i) * rpad);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q < ng && (2 * lane + 64 * q) < it.ncols) {
          const double2 w = ld_stream(r0 + lane + 32 * q);
          acc[q][0] = fma(w.x, x0, acc[q][0]);
          acc[q][1] = fma(w.y, x0, acc[q][1]);
        }
      }
    }
    __syncthreads();  // red reuse across items
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      red[warp][2 * lane + 64 * q] = acc[q][0];
      red[warp][2 * lane + 64 * q + 1] = acc[q][1];
    }
    __syncthreads();
    const int c = threadIdx.x;
    if (c < it.ncols) {
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) v += red[w][c];
      p1_write(it, g, c, v, a);
    }
  }
}

// ---- phase 1, proxy levels: v_c = sum_j K(P_c, z_j) x_j, thread = target,
// sources staged in shared memory and read as broadcasts.
template <int K>
__global__ void __launch_bounds__(kThreads, 2) p1_proxy_kernel(const P1Args a) {
  __shared__ double2 src[2 * kChunk];  // (x, y), (z, w)
  __shared__ long long s_k;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_k = static_cast<long long>(atomicAdd(a.counter, 1u));
    __syncthreads();
    const long long k = s_k;
    if (k >= a.nitems) break;
    const P1Item it = a.items[k];
    const std::int64_t g = it.node;
    const std::int64_t rb = a.nt.rowbeg[g] + it.row0;
    const int c = threadIdx.x;
    const std::int64_t qi = a.nt.soff[g] + it.col0 + c;
    const bool active = c < it.ncols;
    const double tx = active ? a.qx[qi] : kFar, ty = active ? a.qy[qi] : kFar,
                 tz = active ? a.qz[qi] : kFar;
    double acc0 = 0.0, acc1 = 0.0;
    for (int j0 = 0; j0 < it.nrows; j0 += kChunk) {
      const int nj = min(kChunk, it.nrows - j0);
      __syncthreads();
      if (threadIdx.x < nj) {
        const std::int64_t p = rb + j0 + threadIdx.x;
        src[2 * threadIdx.x] = make_double2(a.px[p], a.py[p]);
        src[2 * threadIdx.x + 1] = make_double2(a.pz[p], a.xp[p]);
      }
      __syncthreads();
      int j = 0;
      for (; j + 1 < nj; j += 2) {
        const double2 s0 = src[2 * j], s1 = src[2 * j + 1];
        const double2 u0 = src[2 * j + 2], u1 = src[2 * j + 3];
        acc0 = fma(kernel_r2_fast<K>(sq3(tx - s0.x, ty - s0.y, tz - s1.x)), s1.y, acc0);
        acc1 = fma(kernel_r2_fast<K>(sq3(tx - u0.x, ty - u0.y, tz - u1.x)), u1.y, acc1);
      }
      if (j < nj) {
        const double2 s0 = src[2 * j], s1 = src[2 * j + 1];
        acc0 = fma(kernel_r2_fast<K>(sq3(tx - s0.x, ty - s0.y, tz - s1.x)), s1.y, acc0);
      }
    }
    if (active) p1_write(it, g, c, acc0 + acc1, a);
  }
}

__global__ void phase1_reduce_kernel(const P1Reduce* __restrict__ red, NodeTable nt,
                                     const std::int32_t* __restrict__ spos,
                                     const double* __restrict__ P, double* __restrict__ S) {
  const P1Reduce r = red[blockIdx.x];
  const std::int64_t g = r.node;
  for (int c = threadIdx.x; c < r.ncols; c += blockDim.x) {
    double v = 0.0;
    for (int k = 0; k < r.nchunks; ++k) v += P[r.pbase + static_cast<std::int64_t>(k) * r.ncols + c];
    const std::int32_t dst = spos[nt.soff[g] + c];
    if (dst >= 0) S[dst] = v;
  }
}

// Proxy coordinates: for segment (Z, k) the pivots of the pair lying in k.
__global__ void proxy_gather_kernel(const ProxySeg* __restrict__ segs, std::int64_t nseg,
                                    const std::int32_t* __restrict__ piv,
                                    const double* __restrict__ px, const double* __restrict__ py,
                                    const double* __restrict__ pz, double* __restrict__ qx,
                                    double* __restrict__ qy, double* __restrict__ qz) {
  const std::int64_t s = blockIdx.x * static_cast<std::int64_t>(blockDim.y) + threadIdx.y;
  if (s >= nseg) return;
  const ProxySeg sg = segs[s];
  for (int q = threadIdx.x; q < sg.r; q += blockDim.x) {
    // side 0: Z = X, proxies = column pivots tau (in Y = k); side 1: row pivots sigma
    const std::int32_t loc = piv[sg.piv_off + (sg.side == 0 ? sg.r : 0) + q];
    const std::int64_t idx = sg.base + loc;
    qx[sg.so + q] = px[idx];
    qy[sg.so + q] = py[idx];
    qz[sg.so + q] = pz[idx];
  }
}

// Triangular inverses of the packed pivot LU, in place (build time; one thread
// per column): strict lower <- L^-1 (unit diagonal implied), upper incl.
// diagonal <- R^-1. Applying L^-1 and R^-1 as two GEMVs is as accurate as the
// reference's forward/backward substitution (lowrank.cpp:310-320) on these
// ill-conditioned pivot blocks (cond ~ 1e12 at eps 1e-10), unlike forming
// (L R)^-1, and turns the sequential solves into coalesced, parallel GEMVs.
__global__ void lu_invert_kernel(const ProxySeg* __restrict__ segs, std::int64_t nseg,
                                 double* __restrict__ lu, double* __restrict__ scratch,
                                 int max_r) {
  const std::int64_t s = blockIdx.x;
  if (s >= nseg) return;
  const ProxySeg sg = segs[s];
  if (sg.side != 0) return;  // each pair appears once with side 0 per owning shard
  const int r = sg.r;
  double* A = lu + sg.lu_off;
  double* Gs = scratch + static_cast<std::int64_t>(blockIdx.x) * max_r * max_r;  // column-major
  for (int c = threadIdx.x; c < r; c += blockDim.x) {
    double* g = Gs + static_cast<std::int64_t>(c) * max_r;
    // column c of L^-1 (entries q > c; the diagonal 1 is implicit)
    for (int q = c + 1; q < r; ++q) {
      double acc = -A[static_cast<std::int64_t>(q) * r + c];
      for (int b = c + 1; b < q; ++b) acc = fma(-A[static_cast<std::int64_t>(q) * r + b], g[b], acc);
      g[q] = acc;
    }
    // column c of R^-1 (entries q <= c)
    g[c] = 1.0 / A[static_cast<std::int64_t>(c) * r + c];
    for (int q = c - 1; q >= 0; --q) {
      double acc = 0.0;
      for (int b = q + 1; b <= c; ++b) acc = fma(-A[static_cast<std::int64_t>(q) * r + b], g[b], acc);
      g[q] = acc / A[static_cast<std::int64_t>(q) * r + q];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {  // row-major over the LU slot
    const int row = e / r, col = e % r;
    A[e] = Gs[static_cast<std::int64_t>(col) * max_r + row];
  }
}

// Per ordered proxy block (one warp), in place on S, with P the packed
// inverses (strict lower L^-1, upper R^-1):
//   side 0 (target = pair's row side X):  s = R^-1 (L^-1 v)       (lowrank.cpp:310-320)
//   side 1 (target = pair's col side Y):  s = L^-T (R^-T v)       (the transposed block)
__global__ void proxy_solve_kernel(const ProxySeg* __restrict__ segs, std::int64_t nseg,
                                   const double* __restrict__ lu, double* __restrict__ S) {
  extern __shared__ double sh[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::int64_t s = blockIdx.x * static_cast<std::int64_t>(blockDim.x >> 5) + warp;
  if (s >= nseg) return;
  const ProxySeg sg = segs[s];
  const int r = sg.r;
  double* v = sh + warp * 640;  // v and w, r <= 320 (enforced on the host)
  double* w = v + 320;
  double* Sg = S + sg.so;
  for (int q = lane; q < r; q += 32) v[q] = Sg[q];
  __syncwarp();
  const double* P = lu + sg.lu_off;
  if (sg.side == 0) {
    for (int i = 0; i < r; ++i) {  // w = L^-1 v: w_i = v_i + sum_{j<i} P[i][j] v_j
      const double* row = P + static_cast<std::int64_t>(i) * r;
      double acc = 0.0;
      for (int j = lane; j < i; j += 32) acc = fma(row[j], v[j], acc);
      acc = warp_sum(acc);
      if (lane == 0) w[i] = v[i] + acc;
    }
    __syncwarp();
    for (int i = 0; i < r; ++i) {  // s = R^-1 w: s_i = sum_{j>=i} P[i][j] w_j
      const double* row = P + static_cast<std::int64_t>(i) * r;
      double acc = 0.0;
      for (int j = i + lane; j < r; j += 32) acc = fma(row[j], w[j], acc);
      acc = warp_sum(acc);
      if (lane == 0) Sg[i] = acc;
    }
  } else {
    double acc[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) acc[k] = 0.0;
    for (int i = 0; i < r; ++i) {  // u = R^-T v: u_j = sum_{i<=j} P[i][j] v_i
      const double vi = v[i];
      const double* row = P + static_cast<std::int64_t>(i) * r;
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        const int j = lane + 32 * k;
        if (j >= i && j < r) acc[k] = fma(row[j], vi, acc[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < 10; ++k) {
      const int j = lane + 32 * k;
      if (j < r) w[j] = acc[k];
    }
    __syncwarp();
    for (int i = 0; i < r; ++i) {  // s = L^-T u: s_j = u_j + sum_{i>j} P[i][j] u_i
      const double ui = w[i];
      const double* row = P + static_cast<std::int64_t>(i) * r;
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        const int j = lane + 32 * k;
        if (j < i) acc[k] = fma(row[j], ui, acc[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < 10; ++k) {
      const int j = lane + 32 * k;
      if (j < r) Sg[j] = acc[k];
    }
  }
}

// ---- phase 2, compute part --------------------------------------------------
// One leaf tile per work unit. Lane = target row (two rows per lane above 32
// rows; below, the warp splits into G = 32/mp source groups). Sources: the
// self block (diagonal rule) read directly, then every other range (near and
// direct neighbour leaves, proxy lists of the ancestors at proxy levels)
// flattened into one virtual stream that the CTA stages through shared memory
// in chunks (many independent loads in flight), each warp evaluating its
// eighth of every chunk against all rows.
enum RangeKind : int { kRangeSelf = 0, kRangePoints = 1, kRangeProxy = 2 };
constexpr int kStage = 512;  // sources staged per chunk (16 KB)

struct TileRanges {
  std::int64_t start[kMaxRanges];  // first index in its array (points / S space)
  int pre[kMaxRanges + 1];         // prefix of lengths
  unsigned char kind[kMaxRanges];
  int n;
};

template <int K>
__device__ __forceinline__ void eval4(const double (&tx)[4], const double (&ty)[4],
                                      const double (&tz)[4], double (&acc)[4], double2 s0,
                                      double2 s1) {
#pragma unroll
  for (int r = 0; r < 4; ++r)
    acc[r] = fma(kernel_r2_fast<K>(sq3(tx[r] - s0.x, ty[r] - s0.y, tz[r] - s1.x)), s1.y, acc[r]);
}

// Rows [r0, r0 + nr) of the tile (nr <= 32): warps form ng row groups of 4
// rows (ng a power of two) x gs = 8 / ng source slices; lanes stride over the
// sources of the staged chunks; partial sums per (slice, row) are reduced in a
// fixed order. Returns after writing rowsum[r0 - r0 .. nr).
template <int K>
__device__ void compute_pass(const Phase2Args& a, const TileRanges& tr, double2* stage,
                             std::int64_t xb, int r0, int nr, double* part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int ng = 1;
  while (ng * 4 < nr) ng <<= 1;
  const int gs = kWarps / ng;
  const int group = warp / gs, slice = warp % gs;
  double tx[4], ty[4], tz[4], acc[4];
  int ti[4];
  bool any = false;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = 4 * group + r;
    const bool ok = i < nr;
    any |= ok;
    const std::int64_t gi = xb + r0 + i;
    tx[r] = ok ? a.px[gi] : kFar;
    ty[r] = ok ? a.py[gi] : kFar;
    tz[r] = ok ? a.pz[gi] : kFar;
    ti[r] = ok ? r0 + i : -1;
    acc[r] = 0.0;
  }
  const int step = 32 * gs;
  int vbeg = 0;
  if (tr.n > 0 && tr.kind[0] == kRangeSelf) {  // self block, diagonal rule
    const std::int64_t st = tr.start[0];
    const int len = tr.pre[1];
    if (any)
      for (int j = slice * 32 + lane; j < len; j += step) {
        const double x0 = a.px[st + j], y0 = a.py[st + j], z0 = a.pz[st + j], w0 = a.xp[st + j];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const double k0 = ti[r] == j ? a.diag
                                       : kernel_r2_fast<K>(sq3(tx[r] - x0, ty[r] - y0, tz[r] - z0));
          acc[r] = fma(k0, w0, acc[r]);
        }
      }
    vbeg = len;
  }
  const int T = tr.pre[tr.n];
  for (int base = vbeg; base < T; base += kStage) {
    const int cnt = min(kStage, T - base);
    __syncthreads();  // previous chunk consumed
    for (int q = threadIdx.x; q < cnt; q += kThreads) {
      const int v = base + q;
      int lo = 0, hi = tr.n - 1;  // range with pre[lo] <= v < pre[lo + 1]
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tr.pre[mid] <= v) lo = mid;
        else hi = mid - 1;
      }
      const std::int64_t idx = tr.start[lo] + (v - tr.pre[lo]);
      if (tr.kind[lo] == kRangeProxy) {
        stage[2 * q] = make_double2(a.qx[idx], a.qy[idx]);
        stage[2 * q + 1] = make_double2(a.qz[idx], a.S[idx]);
      } else {
        stage[2 * q] = make_double2(a.px[idx], a.py[idx]);
        stage[2 * q + 1] = make_double2(a.pz[idx], a.xp[idx]);
      }
    }
    __syncthreads();
    if (any) {
      int j = slice * 32 + lane;
#pragma unroll 1
      for (; j < cnt; j += step) eval4<K>(tx, ty, tz, acc, stage[2 * j], stage[2 * j + 1]);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double v = warp_sum(acc[r]);
    if (lane == 0) part[slice * 32 + 4 * group + r] = v;
  }
  __syncthreads();
  if (threadIdx.x < nr) {
    double v = 0.0;
    for (int s = 0; s < gs; ++s) v += part[s * 32 + threadIdx.x];
    part[kWarps * 32 + threadIdx.x] = v;  // pass result
  }
  __syncthreads();
}

// Persistent CTAs pull leaf tiles from a work counter (dynamic balance).
template <int K, bool STORED>
__global__ void __launch_bounds__(kThreads, 3) p2_compute_kernel(const Phase2Args a) {
  __shared__ TileRanges tr;
  __shared__ double cpart[kWarps * 32 + 32];
  __shared__ double2 stage[2 * kStage];
  __shared__ long long s_t;
  const int L = a.depth;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_t = static_cast<long long>(atomicAdd(a.counter, 1u));
    __syncthreads();
    const long long t = s_t;
    if (t >= a.nleaves) break;
    const std::int64_t X = a.leaf0 + t;
    const std::int64_t xb = a.leaf_off[X];
    const int mrows = static_cast<int>(a.leaf_off[X + 1] - xb);
    if (mrows == 0) continue;
    if (threadIdx.x == 0) {
      // source ranges: self, neighbours (stored mode: only the direct
      // partners), then the proxy ranges of the ancestors at proxy levels
      int n = 0, pre = 0;
      const std::int32_t nb = a.near_off[X], ne = a.near_off[X + 1];
      const std::int32_t nd = STORED ? a.near_dense[X] : 0;
      for (std::int32_t e = nb; e < ne && n < kMaxRanges; ++e) {
        if (STORED && e - nb < nd) continue;
        const std::int32_t Y = a.near_ids[e];
        const std::int64_t yb = a.leaf_off[Y];
        const int len = static_cast<int>(a.leaf_off[Y + 1] - yb);
        tr.start[n] = yb;
        tr.kind[n] = Y == X ? kRangeSelf : kRangePoints;
        tr.pre[n] = pre;
        pre += len;
        ++n;
      }
      for (int l = 1; l <= L && n < kMaxRanges; ++l) {
        if (a.mode[l] != 1 || a.p2_items != nullptr) continue;
        const std::int64_t g = a.lbase[l] + (X >> (3 * (L - l)));
        const int R = a.nt.rpad[g];
        if (R == 0) continue;
        tr.start[n] = a.nt.soff[g];
        tr.kind[n] = kRangeProxy;
        tr.pre[n] = pre;
        pre += R;
        ++n;
      }
      tr.pre[n] = pre;
      tr.n = n;
    }
    __syncthreads();
    for (int r0 = 0; r0 < mrows; r0 += 32) {
      const int m = min(32, mrows - r0);
      compute_pass<K>(a, tr, stage, xb, r0, m, cpart);
      if (threadIdx.x < m) {
        const int i = threadIdx.x;
        double v = cpart[kWarps * 32 + i];
        if (STORED) {  // stored dense near blocks, column-major per leaf
          const std::int32_t nb = a.near_off[X];
          const std::int32_t nd = a.near_dense[X];
          const double* nf = a.NF + a.nf_off[X];
          int c = 0;
          for (std::int32_t e = nb; e < nb + nd; ++e) {
            const std::int32_t Y = a.near_ids[e];
            const std::int64_t yb = a.leaf_off[Y];
            const int len = static_cast<int>(a.leaf_off[Y + 1] - yb);
            for (int j = 0; j < len; ++j, ++c)
              v = fma(nf[static_cast<std::int64_t>(c) * mrows + r0 + i], a.xp[yb + j], v);
          }
        }
        if (a.cpart_out) a.cpart_out[xb + r0 + i] = v;
        else a.b[a.perm[xb + r0 + i]] = v;
      }
      __syncthreads();
    }
  }
}

// ---- phase 2, stream part: rows of W_A . S_A over the stream levels
__global__ void __launch_bounds__(kThreads, 2) p2_stream_kernel(const Phase2Args a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int L = a.depth;
  __shared__ long long s_t;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_t = static_cast<long long>(atomicAdd(a.counter2, 1u));
    __syncthreads();
    const long long t = s_t;
    if (t >= a.nleaves) break;
    const std::int64_t X = a.leaf0 + t;
    const std::int64_t xb = a.leaf_off[X];
    const int m = static_cast<int>(a.leaf_off[X + 1] - xb);
    for (int i = warp; i < m; i += kWarps) {
      double s0 = 0.0, s1 = 0.0;
      for (int l = 1; l <= L; ++l) {
        if (a.mode[l] != 0) continue;
        const std::int64_t g = a.lbase[l] + (X >> (3 * (L - l)));
        const int R = a.nt.rpad[g];
        if (R == 0) continue;
        const double2* row = reinterpret_cast<const double2*>(
            a.W + a.nt.woff[g] + (xb + i - a.nt.rowbeg[g]) * R);
        const double2* S2 = reinterpret_cast<const double2*>(a.S + a.nt.soff[g]);
        const int R2 = R >> 1;
        int c = lane;
        for (; c + 224 < R2; c += 256) {
          double2 w[8], q[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) w[u] = ld_stream(row + c + 32 * u);
#pragma unroll
          for (int u = 0; u < 8; ++u) q[u] = __ldg(S2 + c + 32 * u);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            s0 = fma(w[u].x, q[u].x, s0);
            s1 = fma(w[u].y, q[u].y, s1);
          }
        }
        for (; c < R2; c += 32) {
          const double2 w0 = ld_stream(row + c);
          const double2 q0 = __ldg(S2 + c);
          s0 = fma(w0.x, q0.x, s0);
          s1 = fma(w0.y, q0.y, s1);
        }
      }
      const double v = warp_sum(s0 + s1);
      if (lane == 0) a.spart[xb + i] = v;
    }
  }
}

// ---- phase 2, proxy levels, node-major: b_X += K(X, P_A) s_A for the rows of
// node A, thread = target row, proxy sources staged in shared memory (the
// phase-1 proxy layout, which keeps the FP64 pipe ~80% busy).
template <int K>
__global__ void __launch_bounds__(kThreads, 2) p2_proxy_kernel(const Phase2Args a) {
  __shared__ double2 src[2 * kChunk];
  __shared__ long long s_k;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_k = static_cast<long long>(atomicAdd(a.counter3, 1u));
    __syncthreads();
    const long long k = s_k;
    if (k >= a.n_p2_items) break;
    const P2Item it = a.p2_items[k];
    const std::int64_t g = it.node;
    const std::int64_t so = a.nt.soff[g];
    const int R = a.nt.rpad[g];
    const int i = threadIdx.x;
    const bool active = i < it.nrows;
    const std::int64_t p = a.nt.rowbeg[g] + it.row0 + i;
    const double tx = active ? a.px[p] : kFar, ty = active ? a.py[p] : kFar,
                 tz = active ? a.pz[p] : kFar;
    double acc0 = 0.0, acc1 = 0.0;
    for (int j0 = 0; j0 < R; j0 += kChunk) {
      const int nj = min(kChunk, R - j0);
      __syncthreads();
      if (threadIdx.x < nj) {
        const std::int64_t q = so + j0 + threadIdx.x;
        src[2 * threadIdx.x] = make_double2(a.qx[q], a.qy[q]);
        src[2 * threadIdx.x + 1] = make_double2(a.qz[q], a.S[q]);
      }
      __syncthreads();
      int j = 0;
      for (; j + 1 < nj; j += 2) {
        const double2 s0 = src[2 * j], s1 = src[2 * j + 1];
        const double2 u0 = src[2 * j + 2], u1 = src[2 * j + 3];
        acc0 = fma(kernel_r2_fast<K>(sq3(tx - s0.x, ty - s0.y, tz - s1.x)), s1.y, acc0);
        acc1 = fma(kernel_r2_fast<K>(sq3(tx - u0.x, ty - u0.y, tz - u1.x)), u1.y, acc1);
      }
      if (j < nj) {
        const double2 s0 = src[2 * j], s1 = src[2 * j + 1];
        acc0 = fma(kernel_r2_fast<K>(sq3(tx - s0.x, ty - s0.y, tz - s1.x)), s1.y, acc0);
      }
    }
    if (active) a.lvl_part[static_cast<std::int64_t>(it.slot) * a.n_total + p] = acc0 + acc1;
  }
}

__global__ void combine_kernel(const double* __restrict__ cpart, const double* __restrict__ spart,
                               const double* __restrict__ lvl, int n_lvl, std::int64_t n_total,
                               const std::int32_t* __restrict__ perm, std::int64_t row0,
                               std::int64_t row1, double* __restrict__ b) {
  const std::int64_t p = row0 + blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (p >= row1) return;
  double v = cpart[p];
  for (int l = 0; l < n_lvl; ++l) v += lvl[static_cast<std::int64_t>(l) * n_total + p];
  if (spart) v += spart[p];
  b[perm[p]] = v;
}

// Build-time pass over every dense near-field pair: the reference forms all
// dense leaf blocks during initialize (hmatrix.cpp:124-147), so coincident
// points raise DegenerateGeometryError there; optionally stores the blocks
// (column-major per leaf: NF[nf_off[X] + c * m + i]).
template <int K>
__global__ void __launch_bounds__(kThreads) near_scan_kernel(const Phase2Args a,
                                                             double* __restrict__ NF,
                                                             unsigned* flags) {
  const std::int64_t X = a.leaf0 + blockIdx.x;
  const std::int64_t xb = a.leaf_off[X];
  const int m = static_cast<int>(a.leaf_off[X + 1] - xb);
  if (m == 0) return;
  const std::int32_t nb = a.near_off[X];
  const std::int32_t nd = a.near_dense[X];
  unsigned f = 0;
  std::int64_t coff = 0;
  for (std::int32_t e = nb; e < nb + nd; ++e) {
    const std::int32_t Y = a.near_ids[e];
    const std::int64_t yb = a.leaf_off[Y];
    const int n = static_cast<int>(a.leaf_off[Y + 1] - yb);
    for (int q = threadIdx.x; q < m * n; q += blockDim.x) {
      const int j = q / m, i = q % m;
      const std::int64_t gi = xb + i, gj = yb + j;
      double v;
      if (gi == gj) {
        v = a.diag;
      } else {
        const double r2 = sq3(a.px[gi] - a.px[gj], a.py[gi] - a.py[gj], a.pz[gi] - a.pz[gj]);
        if (r2 < kCoincidentTol2) f |= kFlagDegenGeom;
        v = kernel_r2_fast<K>(r2);
      }
      if (NF) NF[a.nf_off[X] + (coff + j) * m + i] = v;
    }
    coff += n;
  }
  if (f) atomicOr(flags, f);
}

template <class F>
int grid_for(F kernel, int sms, int per_sm, std::int64_t work) {
  int nb = 0;
  H3D_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kThreads, 0));
  const std::int64_t g = static_cast<std::int64_t>(sms) * std::max(1, std::min(nb, per_sm));
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(g, work)));
}

}  // namespace

void launch_gather(const double* x, const std::int32_t* perm, std::int64_t n, double* xp,
                   cudaStream_t s) {
  gather_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(x, perm, n, xp);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_p1_stream(const P1Args& a, int sms, int per_sm, cudaStream_t s) {
  if (a.nitems == 0) return;
  const int grid = grid_for(p1_stream_kernel, sms, per_sm, a.nitems);
  p1_stream_kernel<<<grid, kThreads, 0, s>>>(a);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_p1_proxy(const P1Args& a, int kernel, int sms, int per_sm, cudaStream_t s) {
  if (a.nitems == 0) return;
  switch (kernel) {
    case kLaplace: {
      const int grid = grid_for(p1_proxy_kernel<kLaplace>, sms, per_sm, a.nitems);
      p1_proxy_kernel<kLaplace><<<grid, kThreads, 0, s>>>(a);
      break;
    }
    case kR4: {
      const int grid = grid_for(p1_proxy_kernel<kR4>, sms, per_sm, a.nitems);
      p1_proxy_kernel<kR4><<<grid, kThreads, 0, s>>>(a);
      break;
    }
    default: {
      const int grid = grid_for(p1_proxy_kernel<kHelmholtz>, sms, per_sm, a.nitems);
      p1_proxy_kernel<kHelmholtz><<<grid, kThreads, 0, s>>>(a);
      break;
    }
  }
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_phase1_reduce(const P1Reduce* red, std::int64_t nred, NodeTable nt,
                          const std::int32_t* spos, const double* P, double* S,
                          cudaStream_t s) {
  if (nred == 0) return;
  phase1_reduce_kernel<<<static_cast<unsigned>(nred), 256, 0, s>>>(red, nt, spos, P, S);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_proxy_gather(const ProxySeg* segs, std::int64_t nseg, const std::int32_t* piv,
                         const double* px, const double* py, const double* pz, double* qx,
                         double* qy, double* qz, cudaStream_t s) {
  if (nseg == 0) return;
  const dim3 block(32, 8);
  proxy_gather_kernel<<<static_cast<unsigned>((nseg + 7) / 8), block, 0, s>>>(segs, nseg, piv, px, py,
                                                                            pz, qx, qy, qz);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_lu_invert(const ProxySeg* segs, std::int64_t nseg, double* lu, int max_r,
                      cudaStream_t s) {
  if (nseg == 0 || max_r == 0) return;
  // scratch for a batch of column-major inverses
  const std::int64_t batch = std::max<std::int64_t>(1, std::min<std::int64_t>(
      nseg, (std::int64_t(1) << 29) / (static_cast<std::int64_t>(max_r) * max_r * 8)));
  double* scratch = nullptr;
  H3D_CUDA_CHECK(cudaMallocAsync(&scratch, batch * max_r * max_r * 8, s));
  for (std::int64_t b0 = 0; b0 < nseg; b0 += batch) {
    const std::int64_t nb = std::min(batch, nseg - b0);
    lu_invert_kernel<<<static_cast<unsigned>(nb), 128, 0, s>>>(segs + b0, nb, lu, scratch, max_r);
    H3D_CUDA_CHECK(cudaGetLastError());
  }
  H3D_CUDA_CHECK(cudaFreeAsync(scratch, s));
}

void launch_proxy_solve(const ProxySeg* segs, std::int64_t nseg, const double* lu, double* S,
                        cudaStream_t s) {
  if (nseg == 0) return;
  constexpr int warps = 4;
  proxy_solve_kernel<<<static_cast<unsigned>((nseg + warps - 1) / warps), 32 * warps,
                       warps * 640 * sizeof(double), s>>>(segs, nseg, lu, S);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_p2_compute(const Phase2Args& a, int sms, int per_sm, cudaStream_t s) {
  if (a.nleaves == 0) return;
  const bool stored = a.NF != nullptr;
#define H3D_P2C(KK)                                                                      \
  if (stored) {                                                                          \
    const int grid = grid_for(p2_compute_kernel<KK, true>, sms, per_sm, a.nleaves);      \
    p2_compute_kernel<KK, true><<<grid, kThreads, 0, s>>>(a);                            \
  } else {                                                                               \
    const int grid = grid_for(p2_compute_kernel<KK, false>, sms, per_sm, a.nleaves);     \
    p2_compute_kernel<KK, false><<<grid, kThreads, 0, s>>>(a);                           \
  }
  switch (a.kernel) {
    case kLaplace: H3D_P2C(kLaplace); break;
    case kR4: H3D_P2C(kR4); break;
    default: H3D_P2C(kHelmholtz); break;
  }
#undef H3D_P2C
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_p2_stream(const Phase2Args& a, int sms, int per_sm, cudaStream_t s) {
  if (a.nleaves == 0) return;
  const int grid = grid_for(p2_stream_kernel, sms, per_sm, a.nleaves);
  p2_stream_kernel<<<grid, kThreads, 0, s>>>(a);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_p2_proxy(const Phase2Args& a, int sms, int per_sm, cudaStream_t s) {
  if (a.n_p2_items == 0) return;
  switch (a.kernel) {
    case kLaplace: {
      const int grid = grid_for(p2_proxy_kernel<kLaplace>, sms, per_sm, a.n_p2_items);
      p2_proxy_kernel<kLaplace><<<grid, kThreads, 0, s>>>(a);
      break;
    }
    case kR4: {
      const int grid = grid_for(p2_proxy_kernel<kR4>, sms, per_sm, a.n_p2_items);
      p2_proxy_kernel<kR4><<<grid, kThreads, 0, s>>>(a);
      break;
    }
    default: {
      const int grid = grid_for(p2_proxy_kernel<kHelmholtz>, sms, per_sm, a.n_p2_items);
      p2_proxy_kernel<kHelmholtz><<<grid, kThreads, 0, s>>>(a);
      break;
    }
  }
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_combine(const double* cpart, const double* spart, const double* lvl_part,
                    int n_lvl, std::int64_t n_total, const std::int32_t* perm,
                    std::int64_t row0, std::int64_t row1, double* b, cudaStream_t s) {
  if (row1 <= row0) return;
  combine_kernel<<<static_cast<unsigned>((row1 - row0 + 255) / 256), 256, 0, s>>>(
      cpart, spart, lvl_part, n_lvl, n_total, perm, row0, row1, b);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_near_scan(const Phase2Args& a, double* NF_out, unsigned* flags, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(a.nleaves);
  if (grid == 0) return;
  switch (a.kernel) {
    case kLaplace: near_scan_kernel<kLaplace><<<grid, kThreads, 0, s>>>(a, NF_out, flags); break;
    case kR4: near_scan_kernel<kR4><<<grid, kThreads, 0, s>>>(a, NF_out, flags); break;
    default: near_scan_kernel<kHelmholtz><<<grid, kThreads, 0, s>>>(a, NF_out, flags); break;
  }
  H3D_CUDA_CHECK(cudaGetLastError());
}

}  // namespace h3db
