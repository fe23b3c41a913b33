// HODLR3D matvec kernels (reference hmatrix.cpp:153-226, Algorithm 2).
//
// Every admissible block (Z,k) is F_Z F_k^T with F_Z = K(Z, P_Zk) M_Zk, where
// P_Zk are the ACA pivots of the pair that lie in k ("proxies") and M_Zk a
// triangular factor of the pivot LU (reference lowrank.cpp:291-327). Per node Z
// the partner segments share one column layout (rpad_Z columns):
//
//   stream levels : W_Z = [F_Z^(Z,k1) | ...] stored row-major, streamed;
//   proxy levels  : only the proxy coordinates (q*) + pivots + LU are stored,
//                   the entries K(Z, P_Z) are regenerated in FP64;
//   direct (leaf) : leaf-level admissible blocks are evaluated exactly and
//                   join the near field.
//
//   phase 1  per node: T_Z = W_Z^T x_Z (stream) or v_Z = K(P_Z, Z) x_Z (proxy),
//            scattered through spos into S (target-major t-vectors);
//   solve    per ordered proxy block: s = (LU)^-1 v or (U^T L^T)^-1 v in place;
//   phase 2  per leaf tile X (one CTA): b_X = near/direct P2P
//            + sum over ancestor levels of W_A[rows] S_A (stream) or
//              K(X, P_A) S_A (proxy); one writer per b entry, fused un-permute.
//
// Streaming uses 16-byte L1::no_allocate loads; P2P uses lanes over sources
// and 4 register-resident target rows per warp. No atomics anywhere: results
// are bitwise reproducible run to run (reference hmatrix.hpp:68-69).
#include "common.cuh"
#include "kernels.h"

namespace h3db {

namespace {

constexpr double kFar = 1e100;  // coordinate of padding / inactive targets

__global__ void gather_kernel(const double* __restrict__ x, const std::int32_t* __restrict__ perm,
                              std::int64_t n, double* __restrict__ xp) {
  const std::int64_t p = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (p < n) xp[p] = __ldg(x + perm[p]);
}

// acc[r] += sum_j K(t_r, s_j) w_j over sources [0, ns), lanes striding j.
template <int K, int R>
__device__ __forceinline__ void p2p_rows(const double (&tx)[R], const double (&ty)[R],
                                         const double (&tz)[R], double (&acc)[R],
                                         const double* __restrict__ sx,
                                         const double* __restrict__ sy,
                                         const double* __restrict__ sz,
                                         const double* __restrict__ sw, int ns, int lane) {
  int j = lane;
  for (; j + 32 < ns; j += 64) {
    const double x0 = __ldg(sx + j), y0 = __ldg(sy + j), z0 = __ldg(sz + j), w0 = __ldg(sw + j);
    const double x1 = __ldg(sx + j + 32), y1 = __ldg(sy + j + 32), z1 = __ldg(sz + j + 32),
                 w1 = __ldg(sw + j + 32);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double a0 = sq3(tx[r] - x0, ty[r] - y0, tz[r] - z0);
      const double a1 = sq3(tx[r] - x1, ty[r] - y1, tz[r] - z1);
      acc[r] = fma(kernel_r2_fast<K>(a0), w0, acc[r]);
      acc[r] = fma(kernel_r2_fast<K>(a1), w1, acc[r]);
    }
  }
  if (j < ns) {
    const double x0 = __ldg(sx + j), y0 = __ldg(sy + j), z0 = __ldg(sz + j), w0 = __ldg(sw + j);
#pragma unroll
    for (int r = 0; r < R; ++r)
      acc[r] = fma(kernel_r2_fast<K>(sq3(tx[r] - x0, ty[r] - y0, tz[r] - z0)), w0, acc[r]);
  }
}

// Self block: the diagonal entry is KernelSpec::diagonal (kernel.cpp:73-80).
template <int K, int R>
__device__ __forceinline__ void p2p_rows_self(const double (&tx)[R], const double (&ty)[R],
                                              const double (&tz)[R], const int (&ti)[R],
                                              double (&acc)[R], const double* __restrict__ sx,
                                              const double* __restrict__ sy,
                                              const double* __restrict__ sz,
                                              const double* __restrict__ sw, int ns, int lane,
                                              double diag) {
  for (int j = lane; j < ns; j += 32) {
    const double x0 = sx[j], y0 = sy[j], z0 = sz[j], w0 = sw[j];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double k = ti[r] == j ? diag : kernel_r2_fast<K>(sq3(tx[r] - x0, ty[r] - y0, tz[r] - z0));
      acc[r] = fma(k, w0, acc[r]);
    }
  }
}

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kP1Cols = 256;  // 32 lanes x 2 doubles x 4 groups
constexpr int kRows = 4;      // P2P target rows per warp

struct P1Args {
  const P1Item* items;
  NodeTable nt;
  const double* W;
  const double* xp;
  const std::int32_t* spos;
  double* S;
  double* P;
  const double *px, *py, *pz;  // permuted points
  const double *qx, *qy, *qz;  // proxy points (S-space)
};

template <int K>
__global__ void __launch_bounds__(kThreads) phase1_kernel(const P1Args a) {
  __shared__ double red[kWarps][kP1Cols + 2];
  __shared__ double outv[kP1Cols];
  const P1Item it = a.items[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::int64_t g = it.node;
  const std::int64_t rb = a.nt.rowbeg[g] + it.row0;
  if (it.kind == 0) {
    // ---- stream: T = W_Z^T x_Z over rows [row0, row0+nrows), 256 columns
    const int rpad = a.nt.rpad[g];
    const double* __restrict__ Wn =
        a.W + a.nt.woff[g] + static_cast<std::int64_t>(it.row0) * rpad + it.col0;
    const double* __restrict__ xn = a.xp + rb;
    const int ng = (it.ncols + 63) >> 6;
    double acc[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = 0.0;
    int i = warp;
    for (; i + kWarps < it.nrows; i += 2 * kWarps) {
      const double x0 = xn[i], x1 = xn[i + kWarps];
      const double2* r0 = reinterpret_cast<const double2*>(Wn + static_cast<std::int64_t>(i) * rpad);
      const double2* r1 =
          reinterpret_cast<const double2*>(Wn + static_cast<std::int64_t>(i + kWarps) * rpad);
      double2 w0[4], w1[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool ok = k < ng && (2 * lane + 64 * k) < it.ncols;
        w0[k] = ok ? ld_stream(r0 + lane + 32 * k) : make_double2(0.0, 0.0);
        w1[k] = ok ? ld_stream(r1 + lane + 32 * k) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[k][0] = fma(w0[k].x, x0, acc[k][0]);
        acc[k][1] = fma(w0[k].y, x0, acc[k][1]);
        acc[k][0] = fma(w1[k].x, x1, acc[k][0]);
        acc[k][1] = fma(w1[k].y, x1, acc[k][1]);
      }
    }
    for (; i < it.nrows; i += kWarps) {
      const double x0 = xn[i];
      const double2* r0 = reinterpret_cast<const double2*>(Wn + static_cast<std::int64_t>(i) * rpad);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k < ng && (2 * lane + 64 * k) < it.ncols) {
          const double2 w = ld_stream(r0 + lane + 32 * k);
          acc[k][0] = fma(w.x, x0, acc[k][0]);
          acc[k][1] = fma(w.y, x0, acc[k][1]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      red[warp][2 * lane + 64 * k] = acc[k][0];
      red[warp][2 * lane + 64 * k + 1] = acc[k][1];
    }
    __syncthreads();
    const int c = threadIdx.x;
    if (c < it.ncols) {
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) v += red[w][c];
      outv[c] = v;
    }
  } else {
    // ---- proxy: v_c = sum_j K(P_c, z_j) x_j, targets = proxy columns
    const std::int64_t qb = a.nt.soff[g] + it.col0;
    for (int t0 = warp * 32; t0 < it.ncols; t0 += kWarps * 32) {
      for (int grp = 0; grp < 32 && t0 + grp < it.ncols; grp += kRows) {
        double tx[kRows], ty[kRows], tz[kRows], acc[kRows];
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          const int c = t0 + grp + r;
          const bool ok = c < it.ncols;
          tx[r] = ok ? a.qx[qb + c] : kFar;
          ty[r] = ok ? a.qy[qb + c] : kFar;
          tz[r] = ok ? a.qz[qb + c] : kFar;
          acc[r] = 0.0;
        }
        p2p_rows<K, kRows>(tx, ty, tz, acc, a.px + rb, a.py + rb, a.pz + rb, a.xp + rb, it.nrows,
                           lane);
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          const double v = warp_sum(acc[r]);
          const int c = t0 + grp + r;
          if (lane == 0 && c < it.ncols) outv[c] = v;
        }
      }
    }
    __syncthreads();
  }
  const int c = threadIdx.x;
  if (c < it.ncols) {
    const double v = outv[c];
    if (it.pslot < 0) {
      const std::int32_t dst = a.spos[a.nt.soff[g] + it.col0 + c];
      if (dst >= 0) a.S[dst] = v;
    } else {
      a.P[it.pslot + c] = v;
    }
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
  for (int a = threadIdx.x; a < sg.r; a += blockDim.x) {
    // side 0: Z = X, proxies = column pivots tau (in Y = k); side 1: row pivots sigma
    const std::int32_t loc = piv[sg.piv_off + (sg.side == 0 ? sg.r : 0) + a];
    const std::int64_t idx = sg.base + loc;
    qx[sg.so + a] = px[idx];
    qy[sg.so + a] = py[idx];
    qz[sg.so + a] = pz[idx];
  }
}

// In-place triangular solves on S segments, one warp per ordered proxy block:
//   side 0 (target = row side X):  s = R^-1 L^-1 v        (lowrank.cpp:310-320)
//   side 1 (target = col side Y):  s = L^-T R^-T v        (the transposed block)
// LU packed row-major: strict lower = unit-lower L, upper incl. diagonal = R.
__global__ void proxy_solve_kernel(const ProxySeg* __restrict__ segs, std::int64_t nseg,
                                   const double* __restrict__ lu, double* __restrict__ S) {
  extern __shared__ double sh[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::int64_t s = blockIdx.x * static_cast<std::int64_t>(blockDim.x >> 5) + warp;
  if (s >= nseg) return;
  const ProxySeg sg = segs[s];
  const int r = sg.r;
  double* v = sh + warp * 320;  // r <= 320 (enforced on the host)
  double* Sg = S + sg.so;
  for (int a = lane; a < r; a += 32) v[a] = Sg[a];
  __syncwarp();
  const double* A = lu + sg.lu_off;
  if (sg.side == 0) {
    for (int a = 0; a < r; ++a) {  // L (unit lower): v_b -= L[b][a] v_a
      const double va = v[a];
      __syncwarp();
      for (int b = a + 1 + lane; b < r; b += 32) v[b] = fma(-A[static_cast<std::int64_t>(b) * r + a], va, v[b]);
      __syncwarp();
    }
    for (int a = r - 1; a >= 0; --a) {  // R (upper): s_a = v_a / R[a][a]; v_b -= R[b][a] s_a
      const double sa = v[a] / A[static_cast<std::int64_t>(a) * r + a];
      __syncwarp();
      if (lane == 0) v[a] = sa;
      for (int b = lane; b < a; b += 32) v[b] = fma(-A[static_cast<std::int64_t>(b) * r + a], sa, v[b]);
      __syncwarp();
    }
  } else {
    for (int a = 0; a < r; ++a) {  // R^T (lower): w_a = v_a / R[a][a]; v_b -= R[a][b] w_a
      const double wa = v[a] / A[static_cast<std::int64_t>(a) * r + a];
      __syncwarp();
      if (lane == 0) v[a] = wa;
      for (int b = a + 1 + lane; b < r; b += 32) v[b] = fma(-A[static_cast<std::int64_t>(a) * r + b], wa, v[b]);
      __syncwarp();
    }
    for (int a = r - 1; a >= 0; --a) {  // L^T (unit upper): v_b -= L[a][b] v_a
      const double va = v[a];
      __syncwarp();
      for (int b = lane; b < a; b += 32) v[b] = fma(-A[static_cast<std::int64_t>(a) * r + b], va, v[b]);
      __syncwarp();
    }
  }
  for (int a = lane; a < r; a += 32) Sg[a] = v[a];
}

// One CTA per leaf tile, rows in passes of 32 (8 warps x 4 rows).
template <int K, bool STORED>
__global__ void __launch_bounds__(kThreads) phase2_kernel(const Phase2Args a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::int64_t X = a.leaf0 + blockIdx.x;
  const std::int64_t xb = a.leaf_off[X];
  const int mrows = static_cast<int>(a.leaf_off[X + 1] - xb);
  if (mrows == 0) return;
  const int L = a.depth;
  const std::int32_t nb = a.near_off[X], ne = a.near_off[X + 1];

  for (int r0 = 0; r0 < mrows; r0 += kWarps * kRows) {
    double tx[kRows], ty[kRows], tz[kRows], acc[kRows];
    int ti[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int i = r0 + warp * kRows + r;
      const bool ok = i < mrows;
      tx[r] = ok ? a.px[xb + i] : kFar;
      ty[r] = ok ? a.py[xb + i] : kFar;
      tz[r] = ok ? a.pz[xb + i] : kFar;
      ti[r] = ok ? i : -1;
      acc[r] = 0.0;
    }

    // ---- near field (self, edge, face) + directly evaluated leaf partners
    if (STORED) {
      std::int64_t ntot = 0;
      for (std::int32_t e = nb; e < ne; ++e) {
        const std::int32_t Y = a.near_ids[e];
        ntot += a.leaf_off[Y + 1] - a.leaf_off[Y];
      }
      const double* nf = a.NF + a.nf_off[X];
      std::int64_t coff = 0;
      for (std::int32_t e = nb; e < ne; ++e) {
        const std::int32_t Y = a.near_ids[e];
        const std::int64_t yb = a.leaf_off[Y];
        const int n = static_cast<int>(a.leaf_off[Y + 1] - yb);
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          if (ti[r] < 0) continue;
          const double* row = nf + static_cast<std::int64_t>(ti[r]) * ntot + coff;
          for (int j = lane; j < n; j += 32) acc[r] = fma(ld_stream1(row + j), a.xp[yb + j], acc[r]);
        }
        coff += n;
      }
    } else {
      for (std::int32_t e = nb; e < ne; ++e) {
        const std::int32_t Y = a.near_ids[e];
        const std::int64_t yb = a.leaf_off[Y];
        const int n = static_cast<int>(a.leaf_off[Y + 1] - yb);
        if (Y == X)
          p2p_rows_self<K, kRows>(tx, ty, tz, ti, acc, a.px + yb, a.py + yb, a.pz + yb, a.xp + yb, n,
                                  lane, a.diag);
        else
          p2p_rows<K, kRows>(tx, ty, tz, acc, a.px + yb, a.py + yb, a.pz + yb, a.xp + yb, n, lane);
      }
    }

    // ---- low-rank levels 1..L
    for (int l = 1; l <= L; ++l) {
      const std::int64_t g = a.lbase[l] + (X >> (3 * (L - l)));
      const int R = a.nt.rpad[g];
      if (R == 0) continue;
      const std::int64_t so = a.nt.soff[g];
      if (a.mode[l] == 1) {  // proxy: K(X, P_A) s_A
        p2p_rows<K, kRows>(tx, ty, tz, acc, a.qx + so, a.qy + so, a.qz + so, a.S + so, R, lane);
        continue;
      }
      const std::int64_t rowoff = xb + r0 + warp * kRows - a.nt.rowbeg[g];
      const double* Wg = a.W + a.nt.woff[g] + rowoff * R;
      const double2* S2 = reinterpret_cast<const double2*>(a.S + so);
      const int R2 = R >> 1;
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        if (ti[r] < 0) continue;
        const double2* row = reinterpret_cast<const double2*>(Wg + static_cast<std::int64_t>(r) * R);
        double s0 = 0.0, s1 = 0.0;
        int c = lane;
        for (; c + 96 < R2; c += 128) {
          const double2 w0 = ld_stream(row + c), w1 = ld_stream(row + c + 32);
          const double2 w2 = ld_stream(row + c + 64), w3 = ld_stream(row + c + 96);
          const double2 q0 = __ldg(S2 + c), q1 = __ldg(S2 + c + 32);
          const double2 q2 = __ldg(S2 + c + 64), q3 = __ldg(S2 + c + 96);
          s0 = fma(w0.x, q0.x, s0);
          s1 = fma(w0.y, q0.y, s1);
          s0 = fma(w1.x, q1.x, s0);
          s1 = fma(w1.y, q1.y, s1);
          s0 = fma(w2.x, q2.x, s0);
          s1 = fma(w2.y, q2.y, s1);
          s0 = fma(w3.x, q3.x, s0);
          s1 = fma(w3.y, q3.y, s1);
        }
        for (; c < R2; c += 32) {
          const double2 w0 = ld_stream(row + c);
          const double2 q0 = __ldg(S2 + c);
          s0 = fma(w0.x, q0.x, s0);
          s1 = fma(w0.y, q0.y, s1);
        }
        acc[r] += s0 + s1;
      }
    }

#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const double v = warp_sum(acc[r]);
      if (lane == 0 && ti[r] >= 0) a.b[a.perm[xb + ti[r]]] = v;
    }
  }
}

// Build-time pass over every near-field pair: the reference forms all dense
// leaf blocks during initialize (hmatrix.cpp:124-147), so coincident points
// raise DegenerateGeometryError there; optionally stores the blocks.
template <int K>
__global__ void __launch_bounds__(kThreads) near_scan_kernel(const Phase2Args a,
                                                             double* __restrict__ NF,
                                                             unsigned* flags) {
  const std::int64_t X = a.leaf0 + blockIdx.x;
  const std::int64_t xb = a.leaf_off[X];
  const int m = static_cast<int>(a.leaf_off[X + 1] - xb);
  if (m == 0) return;
  const std::int32_t nb = a.near_off[X], ne = a.near_off[X + 1];
  std::int64_t ntot = 0;
  for (std::int32_t e = nb; e < ne; ++e) {
    const std::int32_t Y = a.near_ids[e];
    ntot += a.leaf_off[Y + 1] - a.leaf_off[Y];
  }
  unsigned f = 0;
  std::int64_t coff = 0;
  for (std::int32_t e = nb; e < ne; ++e) {
    const std::int32_t Y = a.near_ids[e];
    const std::int64_t yb = a.leaf_off[Y];
    const int n = static_cast<int>(a.leaf_off[Y + 1] - yb);
    for (int q = threadIdx.x; q < m * n; q += blockDim.x) {
      const int i = q / n, j = q % n;
      const std::int64_t gi = xb + i, gj = yb + j;
      double v;
      if (gi == gj) {
        v = a.diag;
      } else {
        const double r2 = sq3(a.px[gi] - a.px[gj], a.py[gi] - a.py[gj], a.pz[gi] - a.pz[gj]);
        if (r2 < kCoincidentTol2) f |= kFlagDegenGeom;
        v = kernel_r2_fast<K>(r2);
      }
      if (NF) NF[a.nf_off[X] + static_cast<std::int64_t>(i) * ntot + coff + j] = v;
    }
    coff += n;
  }
  if (f) atomicOr(flags, f);
}

}  // namespace

void launch_gather(const double* x, const std::int32_t* perm, std::int64_t n, double* xp,
                   cudaStream_t s) {
  gather_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(x, perm, n, xp);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_phase1(const P1Item* items, std::int64_t nitems, NodeTable nt, const double* W,
                   const double* xp, const std::int32_t* spos, double* S, double* P,
                   const double* px, const double* py, const double* pz, const double* qx,
                   const double* qy, const double* qz, int kernel, cudaStream_t s) {
  if (nitems == 0) return;
  const P1Args a{items, nt, W, xp, spos, S, P, px, py, pz, qx, qy, qz};
  const unsigned grid = static_cast<unsigned>(nitems);
  switch (kernel) {
    case kLaplace: phase1_kernel<kLaplace><<<grid, kThreads, 0, s>>>(a); break;
    case kR4: phase1_kernel<kR4><<<grid, kThreads, 0, s>>>(a); break;
    default: phase1_kernel<kHelmholtz><<<grid, kThreads, 0, s>>>(a); break;
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

void launch_proxy_solve(const ProxySeg* segs, std::int64_t nseg, const double* lu, double* S,
                        cudaStream_t s) {
  if (nseg == 0) return;
  constexpr int warps = 4;
  proxy_solve_kernel<<<static_cast<unsigned>((nseg + warps - 1) / warps), 32 * warps,
                       warps * 320 * sizeof(double), s>>>(segs, nseg, lu, S);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_phase2(const Phase2Args& a, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(a.nleaves);
  const bool stored = a.NF != nullptr;
#define H3D_P2(KK)                                                              \
  if (stored) phase2_kernel<KK, true><<<grid, kThreads, 0, s>>>(a);             \
  else phase2_kernel<KK, false><<<grid, kThreads, 0, s>>>(a);
  switch (a.kernel) {
    case kLaplace: H3D_P2(kLaplace); break;
    case kR4: H3D_P2(kR4); break;
    default: H3D_P2(kHelmholtz); break;
  }
#undef H3D_P2
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_near_scan(const Phase2Args& a, double* NF_out, unsigned* flags, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(a.nleaves);
  switch (a.kernel) {
    case kLaplace: near_scan_kernel<kLaplace><<<grid, kThreads, 0, s>>>(a, NF_out, flags); break;
    case kR4: near_scan_kernel<kR4><<<grid, kThreads, 0, s>>>(a, NF_out, flags); break;
    default: near_scan_kernel<kHelmholtz><<<grid, kThreads, 0, s>>>(a, NF_out, flags); break;
  }
  H3D_CUDA_CHECK(cudaGetLastError());
}

}  // namespace h3db
