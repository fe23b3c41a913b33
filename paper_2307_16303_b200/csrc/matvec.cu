// HODLR3D matvec kernels (reference hmatrix.cpp:153-226, Algorithm 2).
//
// The low-rank factors live in a node-major pool W: for every node Z the
// factors of all its admissible partners are concatenated column-wise into
// one row-major matrix W_Z (|Z| x rpad_Z). A block (Z,k) is F_Z^(Zk) F_k^(Zk)^T,
// so the whole matvec is two streaming passes over W:
//
//   phase 1  T_Z = W_Z^T x_Z   per node (items = row chunk x 256 columns);
//            each column's result is scattered (spos) into S, the
//            target-major "t-vector" pool: S_Z holds t for every partner of Z
//   phase 2  per leaf tile X (one CTA): b_X = near(X) x + sum_l W_A(l)[rows of X] S_A(l)
//            over the ancestors A(l) of X, written once, straight to original
//            order (fused un-permute; reference hmatrix.cpp:216-217).
//
// Both passes stream W with 16-byte L1::no_allocate loads; every b entry has
// exactly one writer and a fixed accumulation order (no atomics), so results
// are bitwise reproducible run to run (reference hmatrix.hpp:68-69).
#include "common.cuh"
#include "kernels.h"

namespace h3db {

namespace {

__global__ void gather_kernel(const double* __restrict__ x, const std::int32_t* __restrict__ perm,
                              std::int64_t n, double* __restrict__ xp) {
  const std::int64_t p = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (p < n) xp[p] = __ldg(x + perm[p]);
}

constexpr int kP1Threads = 256;
constexpr int kP1Warps = kP1Threads / 32;
constexpr int kP1Cols = 256;  // 32 lanes x 2 doubles x 4 groups

__global__ void __launch_bounds__(kP1Threads) phase1_kernel(const P1Item* __restrict__ items,
                                                            NodeTable nt,
                                                            const double* __restrict__ W,
                                                            const double* __restrict__ xp,
                                                            const std::int32_t* __restrict__ spos,
                                                            double* __restrict__ S,
                                                            double* __restrict__ P) {
  __shared__ double red[kP1Warps][kP1Cols + 2];
  const P1Item it = items[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::int64_t g = it.node;
  const int rpad = nt.rpad[g];
  const double* __restrict__ Wn =
      W + nt.woff[g] + static_cast<std::int64_t>(it.row0) * rpad + it.col0;
  const double* __restrict__ xn = xp + nt.rowbeg[g] + it.row0;
  const int ng = (it.ncols + 63) >> 6;  // active 64-column groups (<= 4)

  double acc[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = 0.0;

  int i = warp;
  for (; i + kP1Warps < it.nrows; i += 2 * kP1Warps) {
    const double x0 = xn[i], x1 = xn[i + kP1Warps];
    const double2* r0 = reinterpret_cast<const double2*>(Wn + static_cast<std::int64_t>(i) * rpad);
    const double2* r1 = reinterpret_cast<const double2*>(Wn + static_cast<std::int64_t>(i + kP1Warps) * rpad);
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
  for (; i < it.nrows; i += kP1Warps) {
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
    for (int w = 0; w < kP1Warps; ++w) v += red[w][c];
    if (it.pslot < 0) {
      const std::int32_t dst = spos[nt.soff[g] + it.col0 + c];
      if (dst >= 0) S[dst] = v;
    } else {
      P[it.pslot + c] = v;
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

constexpr int kP2Threads = 256;
constexpr int kP2Warps = kP2Threads / 32;
constexpr int kMaxLeafRows = 64;  // n_max <= 64 leaves; larger leaves loop in row blocks
constexpr int kRowsPerWarp = kMaxLeafRows / kP2Warps;

// One CTA per leaf tile: near field (stored or matrix-free) plus the
// low-rank contributions of every ancestor level, one writer per b entry.
template <int K, bool STORED>
__global__ void __launch_bounds__(kP2Threads) phase2_kernel(const Phase2Args a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::int64_t X = a.leaf0 + blockIdx.x;
  const std::int64_t xb = a.leaf_off[X];
  const int mrows = static_cast<int>(a.leaf_off[X + 1] - xb);
  if (mrows == 0) return;
  const int L = a.depth;

  for (int r0 = 0; r0 < mrows; r0 += kMaxLeafRows) {
    const int m = min(kMaxLeafRows, mrows - r0);
    double acc[kRowsPerWarp];
#pragma unroll
    for (int t = 0; t < kRowsPerWarp; ++t) acc[t] = 0.0;

    // ---- near field: self, near_edge, near_face (hmatrix.cpp:169-198)
    const std::int32_t nb = a.near_off[X], ne = a.near_off[X + 1];
    if (STORED) {
      const double* nf = a.NF + a.nf_off[X];
      std::int64_t ntot = 0;
      for (std::int32_t e = nb; e < ne; ++e) {
        const std::int32_t Y = a.near_ids[e];
        ntot += a.leaf_off[Y + 1] - a.leaf_off[Y];
      }
      std::int64_t coff = 0;
      for (std::int32_t e = nb; e < ne; ++e) {
        const std::int32_t Y = a.near_ids[e];
        const std::int64_t yb = a.leaf_off[Y];
        const int n = static_cast<int>(a.leaf_off[Y + 1] - yb);
#pragma unroll
        for (int t = 0; t < kRowsPerWarp; ++t) {
          const int i = warp + kP2Warps * t;
          if (i < m) {
            const double* row = nf + static_cast<std::int64_t>(r0 + i) * ntot + coff;
            for (int j = lane; j < n; j += 32) acc[t] = fma(ld_stream1(row + j), a.xp[yb + j], acc[t]);
          }
        }
        coff += n;
      }
    } else {
      for (std::int32_t e = nb; e < ne; ++e) {
        const std::int32_t Y = a.near_ids[e];
        const std::int64_t yb = a.leaf_off[Y];
        const int n = static_cast<int>(a.leaf_off[Y + 1] - yb);
        for (int j = lane; j < n; j += 32) {
          const double yx = a.px[yb + j], yy = a.py[yb + j], yz = a.pz[yb + j];
          const double xj = a.xp[yb + j];
          const std::int64_t gj = yb + j;
#pragma unroll
          for (int t = 0; t < kRowsPerWarp; ++t) {
            const int i = warp + kP2Warps * t;
            if (i < m) {
              const std::int64_t gi = xb + r0 + i;
              const double r2 = sq3(a.px[gi] - yx, a.py[gi] - yy, a.pz[gi] - yz);
              const double v = gi == gj ? a.diag : kernel_r2<K>(r2);
              acc[t] = fma(v, xj, acc[t]);
            }
          }
        }
      }
    }

    // ---- low-rank levels 1..L (hmatrix.cpp:200-214): rows of W_A times S_A
    for (int l = 1; l <= L; ++l) {
      const std::int64_t g = a.lbase[l] + (X >> (3 * (L - l)));
      const int R = a.nt.rpad[g];
      if (R == 0) continue;
      const std::int64_t rowoff = xb + r0 - a.nt.rowbeg[g];
      const double* Wg = a.W + a.nt.woff[g] + rowoff * R;
      const double2* S2 = reinterpret_cast<const double2*>(a.S + a.nt.soff[g]);
      const int R2 = R >> 1;
#pragma unroll
      for (int t = 0; t < kRowsPerWarp; ++t) {
        const int i = warp + kP2Warps * t;
        if (i < m) {
          const double2* row = reinterpret_cast<const double2*>(Wg + static_cast<std::int64_t>(i) * R);
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
          acc[t] += s0 + s1;
        }
      }
    }

#pragma unroll
    for (int t = 0; t < kRowsPerWarp; ++t) {
      const int i = warp + kP2Warps * t;
      const double v = warp_sum(acc[t]);
      if (lane == 0 && i < m) a.b[a.perm[xb + r0 + i]] = v;
    }
  }
}

// Build-time pass over every near-field pair: the reference forms all dense
// leaf blocks during initialize (hmatrix.cpp:124-147), so coincident points
// raise DegenerateGeometryError there; optionally stores the blocks.
template <int K>
__global__ void __launch_bounds__(kP2Threads) near_scan_kernel(const Phase2Args a,
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
        v = kernel_r2<K>(r2);
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
                   cudaStream_t s) {
  if (nitems == 0) return;
  phase1_kernel<<<static_cast<unsigned>(nitems), kP1Threads, 0, s>>>(items, nt, W, xp, spos, S, P);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_phase1_reduce(const P1Reduce* red, std::int64_t nred, NodeTable nt,
                          const std::int32_t* spos, const double* P, double* S,
                          cudaStream_t s) {
  if (nred == 0) return;
  phase1_reduce_kernel<<<static_cast<unsigned>(nred), 256, 0, s>>>(red, nt, spos, P, S);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_phase2(const Phase2Args& a, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(a.nleaves);
  const bool stored = a.NF != nullptr;
#define H3D_P2(KK)                                                              \
  if (stored) phase2_kernel<KK, true><<<grid, kP2Threads, 0, s>>>(a);           \
  else phase2_kernel<KK, false><<<grid, kP2Threads, 0, s>>>(a);
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
    case kLaplace: near_scan_kernel<kLaplace><<<grid, kP2Threads, 0, s>>>(a, NF_out, flags); break;
    case kR4: near_scan_kernel<kR4><<<grid, kP2Threads, 0, s>>>(a, NF_out, flags); break;
    default: near_scan_kernel<kHelmholtz><<<grid, kP2Threads, 0, s>>>(a, NF_out, flags); break;
  }
  H3D_CUDA_CHECK(cudaGetLastError());
}

}  // namespace h3db
