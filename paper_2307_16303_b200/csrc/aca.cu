// Batched partially pivoted ACA on the device: one CTA per admissible pair,
// persistent CTAs pulling pairs from an atomic counter, u_k / v_k columns in
// a per-CTA global workspace slot (L1/L2 resident for leaf and mid levels).
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
// Reductions are fixed-order (warp butterflies + ordered per-warp combine) so
// a given launch configuration is bitwise deterministic; the rank pass and
// the write pass therefore produce identical factors.
//
// Output (write pass): U = [u_1..u_r] (m x r) and V = [v_1..v_r] (n x r) with
// U V^T ~= K(X,Y), written row-major into the node-major factor pool W at the
// pair's column offsets (see engine.cu: W layout). Optionally the reference's
// own representation (pivots + packed LU, lowrank.cpp:277-287).
#include "common.cuh"
#include "kernels.h"

namespace h3db {

namespace {

template <int NT>
struct Reduce {
  static constexpr int NW = NT / 32;
  double* v;     // [NW]
  long long* i;  // [NW]

  __device__ __forceinline__ double sum(double x) {
    x = warp_sum(x);
    if (NW == 1) return x;
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) v[w] = x;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < NW; ++k) t += v[k];
    __syncthreads();
    return t;
  }

  __device__ __forceinline__ void argmax(double& x, long long& j) {
    warp_argmax(x, j);
    if (NW == 1) return;
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
      v[w] = x;
      i[w] = j;
    }
    __syncthreads();
    x = -1.0;
    j = -1;
#pragma unroll
    for (int k = 0; k < NW; ++k) argmax_combine(x, j, v[k], i[k]);
    __syncthreads();
  }

  __device__ __forceinline__ long long min_ll(long long x) {
    x = warp_min_ll(x);
    if (NW == 1) return x;
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) i[w] = x;
    __syncthreads();
    long long t = i[0];
#pragma unroll
    for (int k = 1; k < NW; ++k) t = i[k] < t ? i[k] : t;
    __syncthreads();
    return t;
  }
};

template <int NT>
__device__ __forceinline__ void bar() {
  if (NT == 32) __syncwarp();
  else __syncthreads();
}

// Transpose a column-major (rows x r, column stride ld) workspace matrix into
// row-major W rows (row stride rs) through a 32 x 33 shared tile.
template <int NT>
__device__ void write_rows(const double* __restrict__ src, int ld, int rows, int r,
                           double* __restrict__ dst, int rs, double* tile) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i0 = 0; i0 < rows; i0 += 32) {
    for (int a0 = 0; a0 < r; a0 += 32) {
      for (int al = w; al < 32; al += NW) {
        const int a = a0 + al, i = i0 + lane;
        tile[al * 33 + lane] = (a < r && i < rows) ? src[static_cast<std::int64_t>(a) * ld + i] : 0.0;
      }
      bar<NT>();
      for (int il = w; il < 32; il += NW) {
        const int i = i0 + il, a = a0 + lane;
        if (i < rows && a < r) dst[static_cast<std::int64_t>(i) * rs + a] = tile[lane * 33 + il];
      }
      bar<NT>();
    }
  }
}

template <int NT, int K>
__global__ void __launch_bounds__(NT) aca_kernel(const AcaArgs a) {
  constexpr int NW = NT / 32;
  extern __shared__ double smem[];
  const int cw = a.cap_ws;
  double* s_vec = smem;            // gathered U(i,:) / V(pj,:)   [cw]
  double* s_cu = s_vec + cw;       // U^T u                       [cw]
  double* s_cv = s_cu + cw;        // V^T v                       [cw]
  double* s_delta = s_cv + cw;     //                             [cw]
  double* s_tile = s_delta + cw;   // 32 x 33
  int* s_prow = reinterpret_cast<int*>(s_tile + 32 * 33);  // [cw]
  int* s_pcol = s_prow + cw;                               // [cw]
  __shared__ double s_rv[NW];
  __shared__ long long s_ri[NW];
  __shared__ long long s_pair;
  Reduce<NT> red{s_rv, s_ri};

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* U = a.ws + static_cast<std::int64_t>(blockIdx.x) * a.slot_doubles;
  double* V = U + static_cast<std::int64_t>(cw + 1) * a.ms;
  unsigned char* row_used = reinterpret_cast<unsigned char*>(V + static_cast<std::int64_t>(cw + 1) * a.ns);
  unsigned char* col_used = row_used + a.ms;

  for (;;) {
    __syncthreads();
    if (tid == 0) s_pair = static_cast<long long>(atomicAdd(a.counter, 1ULL));
    __syncthreads();
    const long long p = s_pair;
    if (p >= a.npairs) break;

    const std::int64_t xb = a.xb[p], yb = a.yb[p];
    const int m = a.m[p], n = a.n[p];
    int cap = m < n ? m : n;
    if (a.max_rank > 0 && a.max_rank < cap) cap = static_cast<int>(a.max_rank);
    const double* __restrict__ rx = a.px + xb;
    const double* __restrict__ ry = a.py + xb;
    const double* __restrict__ rz = a.pz + xb;
    const double* __restrict__ cx = a.px + yb;
    const double* __restrict__ cy = a.py + yb;
    const double* __restrict__ cz = a.pz + yb;
    for (int i = tid; i < m; i += NT) row_used[i] = 0;
    for (int j = tid; j < n; j += NT) col_used[j] = 0;
    __syncthreads();

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
          for (int t = tid; t < m; t += NT)
            if (!row_used[t]) {
              first = t;
              break;
            }
          first = red.min_ll(first);
          i = first == 0x7fffffffffffffffLL ? -1 : first;
        }
        if (i < 0) break;
        for (int q = tid; q < rank; q += NT) s_vec[q] = U[static_cast<std::int64_t>(q) * a.ms + i];
        __syncthreads();
        const double xi = rx[i], yi = ry[i], zi = rz[i];
        double best = -1.0;
        long long bestj = -1;
        for (int j = tid; j < n; j += NT) {
          double val;
          if (xb + i == yb + j) {
            val = a.diag;
          } else {
            const double r2 = sq3(xi - cx[j], yi - cy[j], zi - cz[j]);
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
        red.argmax(best, bestj);
        if (bestj < 0) break;
        if (best < 1e-30) {  // AcaOptions::pivot_floor (lowrank.hpp:99)
          __syncthreads();
          if (tid == 0) row_used[i] = 1;
          suggested = -1;
          __syncthreads();
          continue;
        }
        pi = i;
        pj = bestj;
        break;
      }
      if (pi < 0) break;
      __syncthreads();  // Vc visible to all threads
      const double delta = Vc[pj];
      for (int q = tid; q < rank; q += NT) s_vec[q] = V[static_cast<std::int64_t>(q) * a.ns + pj];
      __syncthreads();
      const double xj = cx[pj], yj = cy[pj], zj = cz[pj];
      double u2 = 0.0, v2 = 0.0;
      for (int i = tid; i < m; i += NT) {
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
      for (int j = tid; j < n; j += NT) {
        const double v = Vc[j] * inv;
        Vc[j] = v;
        v2 = fma(v, v, v2);
      }
      u2 = red.sum(u2);
      v2 = red.sum(v2);
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
        __syncthreads();  // Uc / Vc complete
        for (int q = warp; q < rank; q += NW) {
          const double* uq = U + static_cast<std::int64_t>(q) * a.ms;
          const double* vq = V + static_cast<std::int64_t>(q) * a.ns;
          double su = 0.0, sv = 0.0;
          for (int i = lane; i < m; i += 32) su = fma(uq[i], Uc[i], su);
          for (int j = lane; j < n; j += 32) sv = fma(vq[j], Vc[j], sv);
          su = warp_sum(su);
          sv = warp_sum(sv);
          if (lane == 0) {
            s_cu[q] = su;
            s_cv[q] = sv;
          }
        }
        __syncthreads();
        for (int q = 0; q < rank; ++q) cross = fma(s_cu[q], s_cv[q], cross);
      }
      fro2 += u2 * v2 + 2.0 * cross;
      __syncthreads();
      if (tid == 0) {
        s_delta[rank] = delta;
        s_prow[rank] = static_cast<int>(pi);
        s_pcol[rank] = static_cast<int>(pj);
        row_used[pi] = 1;
        col_used[pj] = 1;
      }
      ++rank;
      __syncthreads();
      // next row pivot: argmax |u| over unused rows (lowrank.cpp:260-270)
      double best = -1.0;
      long long bi = -1;
      for (int i = tid; i < m; i += NT)
        if (!row_used[i]) argmax_combine(best, bi, fabs(Uc[i]), i);
      red.argmax(best, bi);
      suggested = bi;
    }

    if (local_flags) atomicOr(a.flags, local_flags);
    if (overflow) {
      if (tid == 0) {
        a.rank_out[p] = -1;
        atomicOr(a.flags, kFlagAcaOverflow);
      }
      continue;
    }
    if (tid == 0) a.rank_out[p] = rank;
    __syncthreads();
    if (a.W != nullptr && rank > 0) {
      write_rows<NT>(U, a.ms, m, rank, a.W + a.wx[p], a.rx[p], s_tile);
      write_rows<NT>(V, a.ns, n, rank, a.W + a.wy[p], a.ry[p], s_tile);
    }
    if (a.lu != nullptr && rank > 0) {
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

template <int NT>
void launch_nt(const AcaArgs& a, int grid, cudaStream_t s) {
  const std::size_t smem = aca_smem_bytes(NT, a.cap_ws);
  switch (a.kernel) {
    case kLaplace:
      H3D_CUDA_CHECK(cudaFuncSetAttribute(aca_kernel<NT, kLaplace>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      aca_kernel<NT, kLaplace><<<grid, NT, smem, s>>>(a);
      break;
    case kR4:
      H3D_CUDA_CHECK(cudaFuncSetAttribute(aca_kernel<NT, kR4>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      aca_kernel<NT, kR4><<<grid, NT, smem, s>>>(a);
      break;
    default:
      H3D_CUDA_CHECK(cudaFuncSetAttribute(aca_kernel<NT, kHelmholtz>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      aca_kernel<NT, kHelmholtz><<<grid, NT, smem, s>>>(a);
      break;
  }
  H3D_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

std::size_t aca_smem_bytes(int /*threads*/, int cap_ws) {
  return sizeof(double) * (4 * static_cast<std::size_t>(cap_ws) + 32 * 33) +
         sizeof(int) * 2 * static_cast<std::size_t>(cap_ws);
}

int aca_blocks_per_sm(int threads, int kernel, std::size_t smem) {
  int nb = 0;
  const void* f = nullptr;
#define H3D_F(NT)                                                                   \
  f = kernel == kLaplace ? reinterpret_cast<const void*>(aca_kernel<NT, kLaplace>)  \
      : kernel == kR4    ? reinterpret_cast<const void*>(aca_kernel<NT, kR4>)       \
                         : reinterpret_cast<const void*>(aca_kernel<NT, kHelmholtz>);
  switch (threads) {
    case 32: H3D_F(32); break;
    case 128: H3D_F(128); break;
    case 256: H3D_F(256); break;
    default: H3D_F(512); break;
  }
#undef H3D_F
  H3D_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
  H3D_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, threads, smem));
  return nb < 1 ? 1 : nb;
}

void launch_aca(const AcaArgs& a, int threads, int grid, cudaStream_t s) {
  switch (threads) {
    case 32: launch_nt<32>(a, grid, s); break;
    case 128: launch_nt<128>(a, grid, s); break;
    case 256: launch_nt<256>(a, grid, s); break;
    default: launch_nt<512>(a, grid, s); break;
  }
}

}  // namespace h3db
