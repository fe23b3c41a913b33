// Fused pair pass for kModePair levels (planner.h): every admissible pair
// (X, Y) is applied from its factors F = [U; V] ((m + n) x rp, row-major in
// the W pool), both orientations in one visit:
//
//   t_U = U^T x_X,  t_V = V^T x_Y        (pass 1: column sums over F's rows)
//   out_X = U t_V,  out_Y = V t_U        (pass 2: row dots, written per pair)
//
// The node-major pools of kModeStream are read twice from HBM (phase 1 and
// phase 2 are a whole matrix apart); here the two passes over a pair are
// adjacent in time, so the second one is served by L2: the producer copies
// the pair's rows with an evict-normal policy in pass 1 and evict-first in
// pass 2. Warp-specialised persistent CTA, the same bulk-copy ring as the
// stream kernels (matvec.cu): one producer warp claims pairs (kPairBatch per
// atomic) and issues cp.async.bulk row chunks into a kPStages-deep shared
// ring (mbarrier full/empty); four consumer warps accumulate. Outputs are
// summed per node in pair order by pair_gather (deterministic).
//
// Reference mapping: lr_apply (lowrank.cpp:291-327) for both orientations of
// the pair's block, with the explicit factors of the ACA (u_k, v_k).
#include "common.cuh"
#include "kernels.h"

namespace h3db {

namespace {

constexpr int kPStages = 4;
constexpr int kPC = 4;  // consumer warps
constexpr int kPThreads = 32 * (kPC + 1);
constexpr unsigned kPStageBytes = 32 * 1024;
constexpr int kPMaxRows = 128;  // rows per stage (one x value per lane per consumer warp)
constexpr int kPairBatch = 8;
constexpr int kPNK = kPairMaxRp / 32;

struct PairMeta {
  long long xrow, yrow, out;
  int k;            // pair (< 0: stop)
  int pass;         // 0: column sums, 1: row dots
  int r0, nr;       // rows [r0, r0 + nr) of F in this stage
  int m, n, rp, own;
  int last;         // last stage of the pass
  int pad;
};

struct PairSmem {
  double buf[kPStages][kPStageBytes / 8];
  unsigned long long full[kPStages], empty[kPStages];
  PairMeta meta[kPStages];
  double red[kPC][2][kPairMaxRp];  // per-warp partial t_U, t_V
  double t[2][kPairMaxRp];         // t_U, t_V of the current pair
};

__device__ __forceinline__ void pair_put(PairSmem& sm, unsigned t, const PairMeta& mt, const double* src,
                                         unsigned bytes, unsigned long long pol) {
  const int s = t % kPStages;
  if (t >= kPStages) mbar_wait(&sm.empty[s], ((t / kPStages) - 1) & 1);
  sm.meta[s] = mt;
  if (src) {
    mbar_arrive_tx(&sm.full[s], bytes);
    bulk_g2s(sm.buf[s], src, bytes, &sm.full[s], pol);
  } else {
    mbar_arrive(&sm.full[s]);
  }
}

__device__ __forceinline__ PairDesc shfl_pd(const PairDesc& d, int src) {
  PairDesc e;
  e.woff = __shfl_sync(0xffffffffu, d.woff, src);
  e.xrow = __shfl_sync(0xffffffffu, d.xrow, src);
  e.yrow = __shfl_sync(0xffffffffu, d.yrow, src);
  e.out = __shfl_sync(0xffffffffu, d.out, src);
  e.m = __shfl_sync(0xffffffffu, d.m, src);
  e.n = __shfl_sync(0xffffffffu, d.n, src);
  e.rp = __shfl_sync(0xffffffffu, d.rp, src);
  e.own = __shfl_sync(0xffffffffu, d.own, src);
  return e;
}

// Sum of v[r] over the 32 lanes for 8 rows at once (9 shuffles instead of
// 40): returns, in every lane, the total of row (lane >> 2) & 7.
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

template <int NK>
__device__ void pair_consume(PairSmem& sm, const PairArgs& a, unsigned& t, int cw, int lane) {
  // first stage of the pair is waited for by the caller
  double pu[NK], pv[NK];
#pragma unroll
  for (int k = 0; k < NK; ++k) pu[k] = pv[k] = 0.0;
  for (;;) {  // pass 1: this warp's rows of the stage are r0 + cw + 4 j
    const int s = t % kPStages;
    const PairMeta m = sm.meta[s];
    const int J = (m.nr - cw + kPC - 1) / kPC;  // rows of this warp
    const int i_lane = m.r0 + cw + kPC * lane;
    double xv = 0.0;
    if (lane < J)
      xv = i_lane < m.m ? __ldg(a.xp + m.xrow + i_lane) : __ldg(a.xp + m.yrow + (i_lane - m.m));
    const double* b = sm.buf[s] + static_cast<long long>(cw) * m.rp;
    const int ju = min(J, max(0, (m.m - m.r0 - cw + kPC - 1) / kPC));  // rows < m
#pragma unroll 4
    for (int j = 0; j < ju; ++j) {
      const double x = __shfl_sync(0xffffffffu, xv, j);
      const double* row = b + static_cast<long long>(kPC * j) * m.rp;
#pragma unroll
      for (int k = 0; k < NK; ++k)
        if (lane + 32 * k < m.rp) pu[k] = fma(row[lane + 32 * k], x, pu[k]);
    }
#pragma unroll 4
    for (int j = ju; j < J; ++j) {
      const double x = __shfl_sync(0xffffffffu, xv, j);
      const double* row = b + static_cast<long long>(kPC * j) * m.rp;
#pragma unroll
      for (int k = 0; k < NK; ++k)
        if (lane + 32 * k < m.rp) pv[k] = fma(row[lane + 32 * k], x, pv[k]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s]);
    ++t;
    if (m.last) break;
    mbar_wait(&sm.full[t % kPStages], (t / kPStages) & 1);
  }
  // t_U, t_V: warp partials summed in warp order
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    sm.red[cw][0][lane + 32 * k] = pu[k];
    sm.red[cw][1][lane + 32 * k] = pv[k];
  }
  named_bar(2, 32 * kPC);
  for (int q = cw * 32 + lane; q < 2 * NK * 32; q += 32 * kPC) {
    const int side = q / (NK * 32), c = q % (NK * 32);
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < kPC; ++w) v += sm.red[w][side][c];
    sm.t[side][c] = v;
  }
  named_bar(2, 32 * kPC);
  double tu[NK], tv[NK];
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    tu[k] = sm.t[0][lane + 32 * k];
    tv[k] = sm.t[1][lane + 32 * k];
  }
  for (;;) {  // pass 2: row dots, 8 rows of the warp at a time
    const int s = t % kPStages;
    mbar_wait(&sm.full[s], (t / kPStages) & 1);
    const PairMeta m = sm.meta[s];
    const double* b = sm.buf[s];
    const int J = (m.nr - cw + kPC - 1) / kPC;
    for (int j0 = 0; j0 < J; j0 += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[q] = 0.0;
        const int j = j0 + q;
        if (j < J) {
          const int i = m.r0 + cw + kPC * j;
          const double* row = b + static_cast<long long>(i - m.r0) * m.rp;
          const bool xs = i < m.m;
#pragma unroll
          for (int k = 0; k < NK; ++k)
            if (lane + 32 * k < m.rp) v[q] = fma(row[lane + 32 * k], xs ? tv[k] : tu[k], v[q]);
        }
      }
      const double sum = reduce8(v, lane);
      const int q = (lane >> 2) & 7, j = j0 + q;
      if ((lane & 3) == 0 && j < J) {
        const int i = m.r0 + cw + kPC * j;
        if (m.own & (i < m.m ? 1 : 2)) a.out[m.out + i] = sum;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s]);
    ++t;
    if (m.last) break;
  }
  // sm.t is rewritten by the next pair only after every warp passed the
  // first barrier of that pair's reduction
}

__global__ void __launch_bounds__(kPThreads, 1) pair_kernel(const PairArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PairSmem& sm = *reinterpret_cast<PairSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kPC);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kPC) {  // producer
    unsigned long long pol_keep, pol_drop;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_keep));
    pol_drop = l2_evict_first();
    unsigned t = 0;
    long long base = 0;
    if (lane == 0) base = atomicAdd(a.counter, static_cast<unsigned>(kPairBatch));
    base = __shfl_sync(0xffffffffu, base, 0);
    PairDesc d{};
    if (lane < kPairBatch && base + lane < a.n) d = a.descs[base + lane];
    while (base < a.n) {
      long long nb = 0;
      if (lane == 0) nb = atomicAdd(a.counter, static_cast<unsigned>(kPairBatch));
      const int cnt = static_cast<int>(min(static_cast<long long>(kPairBatch), a.n - base));
      for (int j = 0; j < cnt; ++j) {
        const PairDesc e = shfl_pd(d, j);
        if (lane == 0) {
          const int M = e.m + e.n;
          const int rows = max(2, min(kPMaxRows, static_cast<int>(kPStageBytes / (8u * e.rp))) & ~1);
          const double* F = a.W + e.woff;
          for (int pass = 0; pass < 2; ++pass)
            for (int r0 = 0; r0 < M; r0 += rows, ++t) {
              const int nr = min(rows, M - r0);
              pair_put(sm, t,
                       PairMeta{e.xrow, e.yrow, e.out, static_cast<int>(base + j), pass, r0, nr, e.m, e.n,
                                e.rp, e.own, r0 + nr == M ? 1 : 0, 0},
                       F + static_cast<long long>(r0) * e.rp, static_cast<unsigned>(nr) * e.rp * 8u,
                       pass == 0 ? pol_keep : pol_drop);
            }
        }
        __syncwarp();
      }
      base = __shfl_sync(0xffffffffu, nb, 0);
      if (lane < kPairBatch && base + lane < a.n) d = a.descs[base + lane];
    }
    if (lane == 0) {
      PairMeta stop{};
      stop.k = -1;
      pair_put(sm, t, stop, nullptr, 0, 0);
    }
    return;
  }
  unsigned t = 0;
  for (;;) {
    mbar_wait(&sm.full[t % kPStages], (t / kPStages) & 1);
    const PairMeta m = sm.meta[t % kPStages];
    if (m.k < 0) break;
    switch ((m.rp + 31) >> 5) {
      case 1: pair_consume<1>(sm, a, t, warp, lane); break;
      case 2: pair_consume<2>(sm, a, t, warp, lane); break;
      case 3: pair_consume<3>(sm, a, t, warp, lane); break;
      case 4: pair_consume<4>(sm, a, t, warp, lane); break;
      case 5: pair_consume<5>(sm, a, t, warp, lane); break;
      case 6: pair_consume<6>(sm, a, t, warp, lane); break;
      case 7: pair_consume<7>(sm, a, t, warp, lane); break;
      default: pair_consume<8>(sm, a, t, warp, lane); break;
    }
  }
}

// b-side gather: lvl_part[slot][row] = sum over the node's pairs (pair order)
// of their output run.
__global__ void pair_gather_kernel(const P2Item* __restrict__ items, std::int64_t nitems,
                                   const std::int64_t* __restrict__ rowbeg,
                                   const std::int32_t* __restrict__ pc_off,
                                   const std::int64_t* __restrict__ pc_pos,
                                   const double* __restrict__ out, double* __restrict__ lvl,
                                   std::int64_t n_total) {
  const std::int64_t k = blockIdx.x;
  if (k >= nitems) return;
  const P2Item it = items[k];
  const int e0 = pc_off[it.node], e1 = pc_off[it.node + 1];
  for (int i = threadIdx.x; i < it.nrows; i += blockDim.x) {
    const int row = it.row0 + i;
    double v = 0.0;
    for (int e = e0; e < e1; ++e) v += out[pc_pos[e] + row];
    lvl[static_cast<std::int64_t>(it.slot) * n_total + rowbeg[it.node] + row] = v;
  }
}

}  // namespace

std::size_t pair_smem_bytes() { return sizeof(PairSmem); }

void launch_pair(const PairArgs& a, int sms, int per_sm, cudaStream_t s) {
  if (a.n == 0) return;
  static bool attr = false;
  if (!attr) {
    H3D_CUDA_CHECK(cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sizeof(PairSmem))));
    H3D_CUDA_CHECK(cudaFuncSetAttribute(pair_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        cudaSharedmemCarveoutMaxShared));
    attr = true;
  }
  int nb = 0;
  H3D_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pair_kernel, kPThreads,
                                                               sizeof(PairSmem)));
  const std::int64_t g = static_cast<std::int64_t>(sms) * std::max(1, std::min(nb, per_sm));
  const int grid = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(g, a.n)));
  pair_kernel<<<grid, kPThreads, sizeof(PairSmem), s>>>(a);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_pair_gather(const P2Item* items, std::int64_t nitems, const std::int64_t* rowbeg,
                        const std::int32_t* pc_off, const std::int64_t* pc_pos, const double* out,
                        double* lvl, std::int64_t n_total, cudaStream_t s) {
  if (nitems == 0) return;
  pair_gather_kernel<<<static_cast<unsigned>(nitems), 256, 0, s>>>(items, nitems, rowbeg, pc_off, pc_pos,
                                                                   out, lvl, n_total);
  H3D_CUDA_CHECK(cudaGetLastError());
}

}  // namespace h3db
