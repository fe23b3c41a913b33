// Batched partially pivoted ACA on the device. One pair per CTA (persistent
// CTAs pulling pairs from an atomic counter) or, for the few huge blocks of
// the top levels, one pair per thread-block cluster of up to 16 CTAs that
// split the rows/columns and reduce through distributed shared memory.
// u_k / v_k columns live in a per-slot global workspace (L1/L2 resident for
// leaf and mid levels).
//
// Algorithm (pivot rules, stop rules, running Frobenius estimate) follows
// reference proj/src/lowrank.cpp:157-289 (aca_compress) step for step:
//   * row pivot: `suggested` if unused else the first unused row;
//   * residual row = K(i,:) - sum_a v_a u_a(i); column pivot = argmax |.| over
//     unused columns (ties -> lowest index); rows whose residual max is below
//     pivot_floor = 1e-30 are retired;
//   * residual column, v = row / delta; stop if |u||v| <= 1e-12 |S|_F, or on
//     the second consecutive |u||v| <= eps |S|_F (candidate dropped);
//   * |S|_F^2 += |u|^2 |v|^2 + 2 (U^T u).(V^T v); next row = argmax |u|.
// Reductions are fixed-order (warp butterflies, ordered per-warp and per-CTA
// combines) so a launch configuration (CTA size, cluster size) is bitwise
// deterministic; the rank pass and the write pass use the same configuration
// and therefore produce identical factors.
//
// Output (write pass): U = [u_1..u_r] (m x r) and V = [v_1..v_r] (n x r) with
// U V^T ~= K(X,Y), written row-major into the node-major factor pool W at the
// pair's column offsets (stream levels), or the reference's own
// representation, pivots + packed LU (lowrank.cpp:277-287; proxy levels).
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace h3db {

namespace {

template <int NT, bool CLU>
struct Ctx {
  static constexpr int NW = NT / 32;
  double* rv;        // [NW] per-warp scratch
  long long* ri;     // [NW]
  double* cv;        // [1] cluster slot
  long long* ci;     // [1]
  int CL;

  __device__ __forceinline__ void bar() {
    if constexpr (CLU) cg::this_cluster().sync();
    else __syncthreads();
  }
  template <class T>
  __device__ __forceinline__ T remote(T* p, int rank) {
    if constexpr (CLU) return *cg::this_cluster().map_shared_rank(p, rank);
    else return *p;
  }

  __device__ double local_sum(double x) {
    x = warp_sum(x);
    if (NW > 1) {
      if ((threadIdx.x & 31) == 0) rv[threadIdx.x >> 5] = x;
      __syncthreads();
      x = 0.0;
#pragma unroll
      for (int k = 0; k < NW; ++k) x += rv[k];
      __syncthreads();
    }
    return x;
  }

  __device__ double sum(double x) {
    x = warp_sum(x);
    if (NW > 1) {
      if ((threadIdx.x & 31) == 0) rv[threadIdx.x >> 5] = x;
      __syncthreads();
      x = 0.0;
#pragma unroll
      for (int k = 0; k < NW; ++k) x += rv[k];
      __syncthreads();
    }
    if constexpr (CLU) {
      if (threadIdx.x == 0) cv[0] = x;
      bar();
      double t = 0.0;
      for (int c = 0; c < CL; ++c) t += remote(cv, c);
      bar();
      return t;
    }
    return x;
  }

  __device__ void argmax(double& x, long long& j) {
    warp_argmax(x, j);
    if (NW > 1) {
      if ((threadIdx.x & 31) == 0) {
        rv[threadIdx.x >> 5] = x;
        ri[threadIdx.x >> 5] = j;
      }
      __syncthreads();
      x = -1.0;
      j = -1;
#pragma unroll
      for (int k = 0; k < NW; ++k) argmax_combine(x, j, rv[k], ri[k]);
      __syncthreads();
    }
    if constexpr (CLU) {
      if (threadIdx.x == 0) {
        cv[0] = x;
        ci[0] = j;
      }
      bar();
      x = -1.0;
      j = -1;
      for (int c = 0; c < CL; ++c) argmax_combine(x, j, remote(cv, c), remote(ci, c));
      bar();
    }
  }

  __device__ long long min_ll(long long x) {
    x = warp_min_ll(x);
    if (NW > 1) {
      if ((threadIdx.x & 31) == 0) ri[threadIdx.x >> 5] = x;
      __syncthreads();
      x = ri[0];
#pragma unroll
      for (int k = 1; k < NW; ++k) x = ri[k] < x ? ri[k] : x;
      __syncthreads();
    }
    if constexpr (CLU) {
      if (threadIdx.x == 0) ci[0] = x;
      bar();
      long long t = remote(ci, 0);
      for (int c = 1; c < CL; ++c) {
        const long long v = remote(ci, c);
        t = v < t ? v : t;
      }
      bar();
      return t;
    }
    return x;
  }
};

template <int NT>
__device__ __forceinline__ void tbar() {
  if (NT == 32) __syncwarp();
  else __syncthreads();
}

// Transpose a column-major (rows x r, column stride ld) workspace matrix into
// the node's tile-major factor pool (planner.h: kTileRows x kTileCols tiles,
// nct column tiles per tile row): element (i, q) lands at node row row0 + i,
// node column col0 + q. Staged through a 32 x 33 shared tile.
template <int NT>
__device__ void write_rows(const double* __restrict__ src, int ld, int rows, int r,
                           double* __restrict__ Wn, int row0, int col0, int nct, double* tile,
                           bool row_major) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i0 = 0; i0 < rows; i0 += 32) {
    for (int a0 = 0; a0 < r; a0 += 32) {
      for (int al = w; al < 32; al += NW) {
        const int q = a0 + al, i = i0 + lane;
        tile[al * 33 + lane] = (q < r && i < rows) ? src[static_cast<std::int64_t>(q) * ld + i] : 0.0;
      }
      tbar<NT>();
      for (int il = w; il < 32; il += NW) {
        const int i = i0 + il, q = a0 + lane;
        if (i < rows && q < r) {
          // row_major (pair pools): nct is the row stride
          const std::int64_t at = row_major ? static_cast<std::int64_t>(row0 + i) * nct + col0 + q
                                            : tile_index(row0 + i, col0 + q, nct);
          Wn[at] = tile[lane * 33 + il];
        }
      }
      tbar<NT>();
    }
  }
}

template <int NT, int K, bool CLU>
__global__ void __launch_bounds__(NT) aca_kernel(const AcaArgs a) {
  constexpr int NW = NT / 32;
  extern __shared__ double smem[];
  const int cw = a.cap_ws;
  double* s_vec = smem;            // gathered U(i,:) / V(pj,:)   [cw]
  double* s_cu = s_vec + cw;       // U^T u (this CTA's rows)     [cw]
  double* s_cv = s_cu + cw;        // V^T v (this CTA's columns)  [cw]
  double* s_delta = s_cv + cw;     //                             [cw]
  double* s_tile = s_delta + cw;   // 32 x 33
  int* s_prow = reinterpret_cast<int*>(s_tile + 32 * 33);  // [cw]
  int* s_pcol = s_prow + cw;                               // [cw]
  __shared__ double s_rv[NW];
  __shared__ long long s_ri[NW];
  __shared__ double s_c1;
  __shared__ long long s_c2;
  __shared__ long long s_pair;
  __shared__ long long s_off;
  int CL = 1, crank = 0;
  if constexpr (CLU) {
    CL = static_cast<int>(cg::this_cluster().num_blocks());
    crank = static_cast<int>(cg::this_cluster().block_rank());
  }
  Ctx<NT, CLU> cx{s_rv, s_ri, &s_c1, &s_c2, CL};

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const std::int64_t slot = blockIdx.x / CL;
  double* U = a.ws + slot * a.slot_doubles;
  double* V = U + static_cast<std::int64_t>(cw + 1) * a.ms;
  unsigned char* row_used = reinterpret_cast<unsigned char*>(V + static_cast<std::int64_t>(cw + 1) * a.ns);
  unsigned char* col_used = row_used + a.ms;

  for (;;) {
    cx.bar();
    if (crank == 0 && tid == 0) {
      const long long c = static_cast<long long>(atomicAdd(a.counter, 1ULL));
      const long long nc = a.nclaims < 0 ? a.npairs : a.nclaims;
      s_pair = c >= nc ? a.npairs : a.order != nullptr ? a.order[c] : c;
    }
    cx.bar();
    const long long p = cx.remote(&s_pair, 0);
    cx.bar();  // no CTA may exit while a peer still reads its shared memory
    if (p >= a.npairs) break;

    const std::int64_t xb = a.xb[p], yb = a.yb[p];
    const int m = a.m[p], n = a.n[p];
    const int r0 = static_cast<int>(static_cast<long long>(m) * crank / CL);
    const int r1 = static_cast<int>(static_cast<long long>(m) * (crank + 1) / CL);
    const int c0 = static_cast<int>(static_cast<long long>(n) * crank / CL);
    const int c1 = static_cast<int>(static_cast<long long>(n) * (crank + 1) / CL);
    int cap = m < n ? m : n;
    if (a.max_rank > 0 && a.max_rank < cap) cap = static_cast<int>(a.max_rank);
    const double* __restrict__ rx = a.px + xb;
    const double* __restrict__ ry = a.py + xb;
    const double* __restrict__ rz = a.pz + xb;
    const double* __restrict__ cx_ = a.px + yb;
    const double* __restrict__ cy_ = a.py + yb;
    const double* __restrict__ cz_ = a.pz + yb;
    for (int i = r0 + tid; i < r1; i += NT) row_used[i] = 0;
    for (int j = c0 + tid; j < c1; j += NT) col_used[j] = 0;
    cx.bar();

    int rank = 0, hits = 0;
    long long suggested = 0;
    double fro2 = 0.0;
    bool overflow = false;
    unsigned local_flags = 0;

    while (rank < cap) {
      long long pi = -1, pj = -1;
      double* Vc = V + static_cast<std::int64_t>(rank) * a.ns;  // candidate v (residual row)
      double* Uc = U + static_cast<std::int64_t>(rank) * a.ms;  // candidate u (residual col)
      for (;;) {
        long long i = -1;
        if (suggested >= 0 && suggested < m && !row_used[suggested]) {
          i = suggested;
        } else {
          long long first = 0x7fffffffffffffffLL;
          for (int t = r0 + tid; t < r1; t += NT)
            if (!row_used[t]) {
              first = t;
              break;
            }
          first = cx.min_ll(first);
          i = first == 0x7fffffffffffffffLL ? -1 : first;
        }
        if (i < 0) break;
        for (int q = tid; q < rank; q += NT) s_vec[q] = U[static_cast<std::int64_t>(q) * a.ms + i];
        __syncthreads();
        const double xi = rx[i], yi = ry[i], zi = rz[i];
        double best = -1.0;
        long long bestj = -1;
        for (int j = c0 + tid; j < c1; j += NT) {
          double val;
          if (xb + i == yb + j) {
            val = a.diag;
          } else {
            const double r2 = sq3(xi - cx_[j], yi - cy_[j], zi - cz_[j]);
            if (r2 < kCoincidentTol2) local_flags |= kFlagDegenGeom;
            val = kernel_r2_fast<K>(r2);
          }
          if (rank > 0) {
            double acc = 0.0;
            for (int q = 0; q < rank; ++q)
              acc = fma(V[static_cast<std::int64_t>(q) * a.ns + j], s_vec[q], acc);
            val -= acc;
          }
          Vc[j] = val;
          if (!col_used[j]) argmax_combine(best, bestj, fabs(val), j);
        }
        cx.argmax(best, bestj);
        if (bestj < 0) break;
        if (best < 1e-30) {  // AcaOptions::pivot_floor (lowrank.hpp:99)
          cx.bar();
          if (crank == 0 && tid == 0) row_used[i] = 1;
          suggested = -1;
          cx.bar();
          continue;
        }
        pi = i;
        pj = bestj;
        break;
      }
      if (pi < 0) break;
      cx.bar();  // Vc complete across the cluster
      const double delta = Vc[pj];
      for (int q = tid; q < rank; q += NT) s_vec[q] = V[static_cast<std::int64_t>(q) * a.ns + pj];
      __syncthreads();
      const double xj = cx_[pj], yj = cy_[pj], zj = cz_[pj];
      double u2 = 0.0, v2 = 0.0;
      for (int i = r0 + tid; i < r1; i += NT) {
        double val;
        if (xb + i == yb + pj) {
          val = a.diag;
        } else {
          const double r2 = sq3(rx[i] - xj, ry[i] - yj, rz[i] - zj);
          if (r2 < kCoincidentTol2) local_flags |= kFlagDegenGeom;
          val = kernel_r2_fast<K>(r2);
        }
        if (rank > 0) {
          double acc = 0.0;
          for (int q = 0; q < rank; ++q)
            acc = fma(U[static_cast<std::int64_t>(q) * a.ms + i], s_vec[q], acc);
          val -= acc;
        }
        Uc[i] = val;
        u2 = fma(val, val, u2);
      }
      const double inv = 1.0 / delta;
      for (int j = c0 + tid; j < c1; j += NT) {
        const double v = Vc[j] * inv;
        Vc[j] = v;
        v2 = fma(v, v, v2);
      }
      u2 = cx.sum(u2);
      v2 = cx.sum(v2);
      const double uv = sqrt(u2 * v2);
      if (rank > 0) {  // two-hit stop rule (lowrank.cpp:225-239)
        const double ns = sqrt(fro2 > 0.0 ? fro2 : 0.0);
        if (uv <= 1e-12 * ns) break;
        if (uv <= a.eps * ns) {
          if (++hits >= 2) break;
        } else {
          hits = 0;
        }
      }
      if (rank >= cw) {  // workspace full: the host doubles cap_ws and retries
        overflow = true;
        break;
      }
      double cross = 0.0;
      if (rank > 0) {
        __syncthreads();  // Uc / Vc of this CTA complete
        for (int q = warp; q < rank; q += NW) {
          const double* uq = U + static_cast<std::int64_t>(q) * a.ms;
          const double* vq = V + static_cast<std::int64_t>(q) * a.ns;
          double su = 0.0, sv = 0.0;
          for (int i = r0 + lane; i < r1; i += 32) su = fma(uq[i], Uc[i], su);
          for (int j = c0 + lane; j < c1; j += 32) sv = fma(vq[j], Vc[j], sv);
          su = warp_sum(su);
          sv = warp_sum(sv);
          if (lane == 0) {
            s_cu[q] = su;
            s_cv[q] = sv;
          }
        }
        cx.bar();
        // combine the per-CTA partial vectors in rank order, then the dot
        // (block-local fixed-order reduction: identical in every CTA)
        double part = 0.0;
        for (int q = tid; q < rank; q += NT) {
          double fu = 0.0, fv = 0.0;
          for (int c = 0; c < CL; ++c) {
            fu += cx.remote(s_cu + q, c);
            fv += cx.remote(s_cv + q, c);
          }
          part = fma(fu, fv, part);
        }
        cross = cx.local_sum(part);
      }
      fro2 += u2 * v2 + 2.0 * cross;
      cx.bar();
      if (tid == 0) {
        s_delta[rank] = delta;
        s_prow[rank] = static_cast<int>(pi);
        s_pcol[rank] = static_cast<int>(pj);
        if (crank == 0) {
          row_used[pi] = 1;
          col_used[pj] = 1;
        }
      }
      ++rank;
      cx.bar();
      // next row pivot: argmax |u| over unused rows (lowrank.cpp:260-270)
      double best = -1.0;
      long long bi = -1;
      for (int i = r0 + tid; i < r1; i += NT)
        if (!row_used[i]) argmax_combine(best, bi, fabs(Uc[i]), i);
      cx.argmax(best, bi);
      suggested = bi;
    }

    if (local_flags) atomicOr(a.flags, local_flags);
    if (overflow) {
      if (crank == 0 && tid == 0) {
        a.rank_out[p] = -1;
        atomicOr(a.flags, kFlagAcaOverflow);
      }
      continue;
    }
    if (crank == 0 && tid == 0) a.rank_out[p] = rank;
    cx.bar();  // every CTA's u / v columns are complete
    if (a.pool != nullptr && crank == 0) {
      // single-pass build: the pair's pivots + packed LU into the pool
      if (tid == 0) {
        long long off = -2;
        if (rank > 0) {
          const long long need = static_cast<long long>(rank) * rank + rank;
          off = static_cast<long long>(atomicAdd(a.pool_ctr, static_cast<unsigned long long>(need)));
          if (off + need > a.pool_cap) {
            off = -1;
            atomicOr(a.flags, kFlagPoolFull);
          }
        }
        a.pool_off[p] = off;
        s_off = off;
      }
      __syncthreads();
      const long long off = s_off;
      if (off >= 0) {
        double* lu = a.pool + off;
        int* pv = reinterpret_cast<int*>(lu + static_cast<long long>(rank) * rank);
        for (int q = tid; q < rank; q += NT) {
          pv[q] = s_prow[q];
          pv[rank + q] = s_pcol[q];
        }
        for (int e = tid; e < rank * rank; e += NT) {
          const int row = e / rank, col = e % rank;
          double v;
          if (row > col) v = U[static_cast<std::int64_t>(col) * a.ms + s_prow[row]] / s_delta[col];
          else v = s_delta[row] * V[static_cast<std::int64_t>(row) * a.ns + s_pcol[col]];
          lu[e] = v;
        }
      }
    }
    if (a.W != nullptr && rank > 0) {
      write_rows<NT>(U + r0, a.ms, r1 - r0, rank, a.W + a.wx[p], r0, a.cx[p], a.rx[p], s_tile,
                     a.row_major != 0);
      write_rows<NT>(V + c0, a.ns, c1 - c0, rank, a.W + a.wy[p], c0, a.cy[p], a.ry[p], s_tile,
                     a.row_major != 0);
    }
    if (a.lu != nullptr && rank > 0 && crank == 0) {
      // packed LU (lowrank.cpp:277-287): strict lower u_a(i_b)/delta_a,
      // upper delta_a * v_a(j_b); row-major r x r.
      const std::int64_t po = a.piv_off[p], lo = a.lu_off[p];
      for (int q = tid; q < rank; q += NT) {
        a.piv[po + q] = s_prow[q];
        a.piv[po + rank + q] = s_pcol[q];
      }
      for (int e = tid; e < rank * rank; e += NT) {
        const int row = e / rank, col = e % rank;
        double v;
        if (row > col) v = U[static_cast<std::int64_t>(col) * a.ms + s_prow[row]] / s_delta[col];
        else v = s_delta[row] * V[static_cast<std::int64_t>(row) * a.ns + s_pcol[col]];
        a.lu[lo + e] = v;
      }
    }
  }
}

template <int NT, bool CLU>
const void* kernel_ptr(int kernel) {
  switch (kernel) {
    case kLaplace: return reinterpret_cast<const void*>(aca_kernel<NT, kLaplace, CLU>);
    case kR4: return reinterpret_cast<const void*>(aca_kernel<NT, kR4, CLU>);
    default: return reinterpret_cast<const void*>(aca_kernel<NT, kHelmholtz, CLU>);
  }
}

const void* kernel_for(int threads, int kernel, bool cluster) {
  if (cluster) return threads >= 512 ? kernel_ptr<512, true>(kernel) : kernel_ptr<256, true>(kernel);
  switch (threads) {
    case 32: return kernel_ptr<32, false>(kernel);
    case 128: return kernel_ptr<128, false>(kernel);
    case 256: return kernel_ptr<256, false>(kernel);
    default: return kernel_ptr<512, false>(kernel);
  }
}

// pool -> final pivot / LU arrays (single-pass build)
__global__ void aca_compact_kernel(const double* __restrict__ pool, const std::int64_t* __restrict__ pool_off,
                                   const std::int32_t* __restrict__ rank, std::int32_t* __restrict__ piv,
                                   const std::int64_t* __restrict__ piv_off, double* __restrict__ lu,
                                   const std::int64_t* __restrict__ lu_off) {
  const std::int64_t p = blockIdx.x;
  const int r = rank[p];
  const std::int64_t off = pool_off[p];
  if (r <= 0 || off < 0) return;
  const double* src = pool + off;
  const int* pv = reinterpret_cast<const int*>(src + static_cast<std::int64_t>(r) * r);
  for (int q = threadIdx.x; q < 2 * r; q += blockDim.x) piv[piv_off[p] + q] = pv[q];
  if (lu == nullptr) return;  // pivots only (half levels)
  double* dst = lu + lu_off[p];
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) dst[e] = src[e];
}

__device__ __forceinline__ std::int64_t w_index(int row, int col, int nct, bool row_major) {
  return row_major ? static_cast<std::int64_t>(row) * nct + col : tile_index(row, col, nct);
}

// One side of a pair's explicit factor (rc-row chunks): out[i][b] for the node's rows
// (points pts + base, count rows) against the partner's pivot points
// (pivot indices piv[a], local in the partner, base pbase):
//   upper (U side): out[i][b] = sum_{a <= b} E[i][a] C[b][a], C = column-major R^-1
//   lower (V side): out[i][b] = E[i][b] + sum_{a < b} E[i][a] C[b][a], C = row-major L^-1
// with E[i][a] = K(point i, pivot point a). 32-row chunks: E and the output
// tile staged in shared memory (rows padded to r + 1), the output written
// column-fastest into the node's pool (coalesced).
// full (half levels, U side): then out2[i][b] = out[i][b] + sum_{a > b}
// out[i][a] C[b][a] with the strictly lower part of the same column-major
// copy (L^-1), i.e. U' = K(X, tau) R^-1 L^-1.
template <int K>
__device__ void factor_side(const FactorGenArgs& a, std::int64_t base, int rows, std::int64_t pbase,
                            const std::int32_t* __restrict__ piv, int r, const double* __restrict__ C,
                            bool upper, double* __restrict__ Wn, int col0, int nct, double* sm, int rc,
                            bool full = false) {
  const int ld = r + 1;
  double* E = sm;            // [rc][ld]
  double* O = sm + rc * ld;  // [rc][ld]
  double* Q = O + rc * ld;   // [r][3] pivot points
  for (int q = threadIdx.x; q < r; q += blockDim.x) {
    const std::int64_t k = pbase + piv[q];
    Q[3 * q] = a.px[k];
    Q[3 * q + 1] = a.py[k];
    Q[3 * q + 2] = a.pz[k];
  }
  __syncthreads();
  for (int i0 = 0; i0 < rows; i0 += rc) {
    const int nr = min(rc, rows - i0);
    for (int e = threadIdx.x; e < nr * r; e += blockDim.x) {
      const int i = e / r, q = e % r;
      const std::int64_t k = base + i0 + i;
      E[i * ld + q] = kernel_r2_fast<K>(sq3(a.px[k] - Q[3 * q], a.py[k] - Q[3 * q + 1], a.pz[k] - Q[3 * q + 2]));
    }
    __syncthreads();
    // (b, i) with i fastest: a warp shares b, so its C row is one broadcast stream
    for (int e = threadIdx.x; e < nr * r; e += blockDim.x) {
      const int b = e / nr, i = e % nr;
      const double* cb = C + static_cast<std::int64_t>(b) * r;
      const double* ei = E + i * ld;
      double acc = 0.0;
      if (upper) {
        for (int q = 0; q <= b; ++q) acc = fma(ei[q], __ldg(cb + q), acc);
      } else {
        for (int q = 0; q < b; ++q) acc = fma(ei[q], __ldg(cb + q), acc);
        acc += ei[b];
      }
      O[i * ld + b] = acc;
    }
    __syncthreads();
    const double* R = O;
    if (full) {
      for (int e = threadIdx.x; e < nr * r; e += blockDim.x) {
        const int b = e / nr, i = e % nr;
        const double* cb = C + static_cast<std::int64_t>(b) * r;
        const double* oi = O + i * ld;
        double acc = oi[b];
        for (int q = b + 1; q < r; ++q) acc = fma(oi[q], __ldg(cb + q), acc);
        E[i * ld + b] = acc;
      }
      __syncthreads();
      R = E;
    }
    for (int e = threadIdx.x; e < nr * r; e += blockDim.x) {
      const int i = e / r, b = e % r;
      Wn[w_index(i0 + i, col0 + b, nct, a.row_major != 0)] = R[i * ld + b];
    }
    __syncthreads();
  }
}

template <int K>
__global__ void __launch_bounds__(256) factor_gen_kernel(const FactorGenArgs a) {
  extern __shared__ double fg_smem[];
  const std::int64_t p = blockIdx.x;
  const int r = a.rank[p];
  if (r <= 0) return;
  const std::int32_t* pv = a.piv + a.piv_off[p];
  const double* inv = a.inv + a.inv_off[p];
  // U = K(X, tau) R^-1: R^-1 column b = row b of the column-major copy
  factor_side<K>(a, a.xb[p], a.m[p], a.yb[p], pv + r, r, inv + a.inv_total, true, a.W + a.wx[p], a.cx[p],
                 a.rx[p], fg_smem, a.rc, a.full != 0);
  if (a.full) return;  // half levels: the Y side is regenerated
  // V = K(Y, sigma) L^-T: L^-1 row b (strict lower part of the row-major block)
  factor_side<K>(a, a.yb[p], a.n[p], a.xb[p], pv, r, inv, false, a.W + a.wy[p], a.cy[p], a.ry[p], fg_smem,
                 a.rc);
}

}  // namespace

void launch_aca_compact(const double* pool, const std::int64_t* pool_off, const std::int32_t* rank,
                        std::int64_t npairs, std::int32_t* piv, const std::int64_t* piv_off, double* lu,
                        const std::int64_t* lu_off, cudaStream_t s) {
  if (npairs == 0) return;
  aca_compact_kernel<<<static_cast<unsigned>(npairs), 256, 0, s>>>(pool, pool_off, rank, piv, piv_off, lu, lu_off);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_factor_gen(const FactorGenArgs& a0, cudaStream_t s) {
  if (a0.npairs == 0 || a0.max_r == 0) return;
  FactorGenArgs a = a0;
  // rows per staged chunk: 32, halved until E + out tiles fit 200 KB
  a.rc = 32;
  auto bytes = [&](int rc) { return sizeof(double) * (2 * rc * static_cast<std::size_t>(a.max_r + 1) + 3 * a.max_r); };
  while (a.rc > 1 && bytes(a.rc) > 200u * 1024u) a.rc >>= 1;
  const std::size_t smem = bytes(a.rc);
  const void* f = a.kernel == kLaplace ? reinterpret_cast<const void*>(factor_gen_kernel<kLaplace>)
                  : a.kernel == kR4    ? reinterpret_cast<const void*>(factor_gen_kernel<kR4>)
                                       : reinterpret_cast<const void*>(factor_gen_kernel<kHelmholtz>);
  H3D_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  void* args[] = {const_cast<FactorGenArgs*>(&a)};
  H3D_CUDA_CHECK(cudaLaunchKernel(f, dim3(static_cast<unsigned>(a.npairs)), dim3(256), args, smem, s));
}

std::size_t aca_smem_bytes(int /*threads*/, int cap_ws) {
  return sizeof(double) * (4 * static_cast<std::size_t>(cap_ws) + 32 * 33) +
         sizeof(int) * 2 * static_cast<std::size_t>(cap_ws);
}

int aca_blocks_per_sm(int threads, int kernel, std::size_t smem) {
  int nb = 0;
  const void* f = kernel_for(threads, kernel, false);
  H3D_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
  H3D_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, threads, smem));
  return nb < 1 ? 1 : nb;
}

void launch_aca(const AcaArgs& a, int threads, int grid, cudaStream_t s) {
  const std::size_t smem = aca_smem_bytes(threads, a.cap_ws);
  const void* f = kernel_for(threads, a.kernel, false);
  H3D_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
  void* args[] = {const_cast<AcaArgs*>(&a)};
  H3D_CUDA_CHECK(cudaLaunchKernel(f, dim3(grid), dim3(threads), args, smem, s));
}

int aca_max_clusters(int threads, int kernel, int cluster, std::size_t smem) {
  const void* f = kernel_for(threads, kernel, true);
  H3D_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
  if (cluster > 8)
    H3D_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster);
  cfg.blockDim = dim3(threads >= 512 ? 512 : 256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = cluster;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  H3D_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&n, f, &cfg));
  return n;
}

void launch_aca_cluster(const AcaArgs& a, int threads, int cluster, int nclusters, cudaStream_t s) {
  const std::size_t smem = aca_smem_bytes(threads, a.cap_ws);
  const void* f = kernel_for(threads, a.kernel, true);
  H3D_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
  if (cluster > 8)
    H3D_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster * nclusters);
  cfg.blockDim = dim3(threads >= 512 ? 512 : 256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = cluster;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  void* args[] = {const_cast<AcaArgs*>(&a)};
  H3D_CUDA_CHECK(cudaLaunchKernelExC(&cfg, f, args));
}

}  // namespace h3db
