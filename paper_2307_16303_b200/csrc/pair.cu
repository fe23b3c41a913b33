// Fused pair pass for kModePair levels (planner.h): every admissible pair
// (X, Y) is applied from its factors F = [U; V] ((m + n) x rp, row-major in
// the W pool), both orientations in one visit, in three passes over F:
//
//   A  (V rows)  t_V = V^T x_Y                           (only if X is owned)
//   B  (U rows)  out_X = U t_V,   t_U = U^T x_X           (one read serves both)
//   C  (V rows)  out_Y = V t_U                            (only if Y is owned)
//
// U is read once and V twice, the second time from L2 a few microseconds
// later (the node-major pools of kModeStream read every factor twice from
// HBM, a whole matrix apart). One CTA works on one pair at a time (static
// interleave: pair k on CTA k mod grid, deterministic; two CTAs per SM, so
// one CTA's t-vector reductions overlap the other's streaming). A producer
// warp streams the pair's rows pass by pass through a kPD-deep cp.async.bulk
// ring of 16 KB stages (the x values of a stage's rows copied with it),
// running ahead across pass and pair boundaries; each of the kPW consumer
// warps takes a contiguous share of every stage's rows, and the only CTA-wide
// syncs are the two t-vector reductions per pair. A lane group of G lanes owns a row, each
// lane two columns per double2 load (G = 8 / 16 / 32 by rank, <= 4 column
// pairs per lane). Outputs are summed per node in pair order by pair_gather
// (deterministic).
//
// Reference mapping: lr_apply (lowrank.cpp:291-327) for both orientations of
// the pair's block, with the explicit factors of the ACA (u_k, v_k).
#include <cstddef>

#include "common.cuh"
#include "kernels.h"

namespace h3db {

namespace {

#ifndef H3D_PAIR_WARPS
#define H3D_PAIR_WARPS 4
#endif
constexpr int kPW = H3D_PAIR_WARPS;  // consumer warps
constexpr int kPThreads = 32 * (kPW + 1);
#ifndef H3D_PAIR_STAGES
#define H3D_PAIR_STAGES 4
#endif
#ifndef H3D_PAIR_STAGE_KB
#define H3D_PAIR_STAGE_KB 16
#endif
constexpr int kPD = H3D_PAIR_STAGES;                       // ring depth
constexpr unsigned kPStageBytes = H3D_PAIR_STAGE_KB * 1024;  // F rows per stage
constexpr int kPMaxRows = 256;            // rows per stage cap (x slots)
constexpr int kPXSlots = kPMaxRows + 4;  // x run copied from a 16-B aligned start

struct PairMeta {
  int k;       // pair index (< 0: stop)
  int pass;    // 0 A, 1 B, 2 C
  int r0, nr;  // rows [r0, r0 + nr) of F
  int xo;      // x of stage row j at xst[xo + j]
  int pad;
};

struct PairSmem {
  double buf[kPD][kPStageBytes / 8];
  double xst[kPD][kPXSlots];
  double red[2][kPW][kPairMaxRp];  // per-warp partial t_V (0) and t_U (1)
  unsigned long long full[kPD], empty[kPD];
  PairMeta meta[kPD];
};

__device__ __forceinline__ int stage_rows(int rp) {
  const int fit = min(kPMaxRows, static_cast<int>(kPStageBytes / (8u * static_cast<unsigned>(rp))));
  return max(1, fit >= 8 * kPW ? fit / kPW * kPW : fit);
}

// rows of F in pass p (lo == hi: skipped)
__device__ __forceinline__ void pass_range(const PairDesc& d, int p, int& lo, int& hi) {
  if (p == 1) {
    lo = 0;
    hi = d.m;
  } else if (d.own & (p == 0 ? 1 : 2)) {
    lo = d.m;
    hi = d.m + d.n;
  } else {
    lo = hi = 0;
  }
}

__device__ __forceinline__ void pair_put(PairSmem& sm, unsigned t, const PairMeta& mt, const double* src,
                                         unsigned bytes, const double* xsrc, unsigned xbytes,
                                         unsigned long long pol) {
  const int s = t % kPD;
  if (t >= kPD) mbar_wait(&sm.empty[s], ((t / kPD) - 1) & 1);
  sm.meta[s] = mt;
  if (src) {
    mbar_arrive_tx(&sm.full[s], bytes + xbytes);
    bulk_g2s(sm.buf[s], src, bytes, &sm.full[s], pol);
    if (xbytes) bulk_g2s(sm.xst[s], xsrc, xbytes, &sm.full[s], l2_evict_first());
  } else {
    mbar_arrive(&sm.full[s]);
  }
}

template <int G, int Q>
__device__ __forceinline__ void red_store(PairSmem& sm, double2 (&acc)[Q], int side, int w, int lane, int rp) {
#pragma unroll
  for (int o = G; o < 32; o <<= 1)
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      acc[q].x += __shfl_xor_sync(0xffffffffu, acc[q].x, o);
      acc[q].y += __shfl_xor_sync(0xffffffffu, acc[q].y, o);
    }
  if (lane < G) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int c = 2 * (lane + G * q);
      if (c < rp) {
        sm.red[side][w][c] = acc[q].x;
        sm.red[side][w][c + 1] = acc[q].y;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = make_double2(0.0, 0.0);
}

template <int G, int Q>
__device__ __forceinline__ void red_load(const PairSmem& sm, double2 (&t)[Q], int side, int gl, int rp) {
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int c = 2 * (gl + G * q);
    double x = 0.0, y = 0.0;
    if (c < rp)
#pragma unroll
      for (int v = 0; v < kPW; ++v) {
        x += sm.red[side][v][c];
        y += sm.red[side][v][c + 1];
      }
    t[q] = make_double2(x, y);  // zero past rp: over-read column slots meet t = 0
  }
}

// Sum over the G lanes of a row group for 4 rows at once: on return, lane
// with (lane % G) & 3 == u holds the total of row u (reduce-scatter over lane
// bits 1 and 0, then a butterfly over the group's higher bits).
template <int G>
__device__ __forceinline__ double group_sum4(const double (&p)[4], int lane) {
  const bool b1 = lane & 2, b0 = lane & 1;
  double k[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const double send = b1 ? p[q] : p[2 + q];
    const double keep = b1 ? p[2 + q] : p[q];
    k[q] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  double r = (b0 ? k[1] : k[0]) + __shfl_xor_sync(0xffffffffu, b0 ? k[0] : k[1], 1);
#pragma unroll
  for (int o = 4; o < G; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}

// One stage of pass `pass` (rows [r0, r0 + nr) of F): this warp takes rows
// [w nr / kPW, (w + 1) nr / kPW) of it, a G-lane group per row, 4 rows per
// group per step (independent chains, one reduce-scatter for the 4 dots).
// SUM: acc += F_row^T x (column sums); DOT: out[row] = F_row . t. Column
// slots past rp read finite stale data (shared memory is zeroed at start and
// only ever holds factors and x) and meet t = 0, or are never stored.
template <int G, int Q, bool SUM, bool DOT>
__device__ __forceinline__ void stage_work(const PairSmem& sm, int s, const PairMeta& mt, int rp, int w,
                                           int lane, double2 (&acc)[Q], const double2 (&tv)[Q], double* out) {
  constexpr int R = 32 / G;
  const int rg = lane / G, gl = lane % G;
  const double* b = sm.buf[s] + 2 * gl;
  const double* xs = sm.xst[s] + mt.xo;
  const int lo = w * mt.nr / kPW, hi = (w + 1) * mt.nr / kPW;
  for (int jb = lo; jb < hi; jb += 4 * R) {  // warp-uniform trip count (shuffles inside)
    double2 f[4][Q];
    double x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = jb + rg + u * R;
      const bool ok = j < hi;
      const double2* row = reinterpret_cast<const double2*>(b + (ok ? j : lo) * rp);
#pragma unroll
      for (int q = 0; q < Q; ++q) f[u][q] = row[G * q];
      if constexpr (SUM) x[u] = ok ? xs[j] : 0.0;
    }
    if constexpr (SUM) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          acc[q].x = fma(f[u][q].x, x[u], acc[q].x);
          acc[q].y = fma(f[u][q].y, x[u], acc[q].y);
        }
    }
    if constexpr (DOT) {
      double p[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double e = f[u][0].x * tv[0].x, o = f[u][0].y * tv[0].y;
#pragma unroll
        for (int q = 1; q < Q; ++q) {
          e = fma(f[u][q].x, tv[q].x, e);
          o = fma(f[u][q].y, tv[q].y, o);
        }
        p[u] = e + o;
      }
      const double v = group_sum4<G>(p, lane);
      const int j = jb + rg + (gl & 3) * R;
      if (gl < 4 && j < hi) out[mt.r0 + j] = v;
    }
  }
}

// Consumer warps walk every pass of every pair of the CTA (two CTA barriers
// per pair), consuming the stages of each pass as they arrive.
template <int G, int Q>
__device__ unsigned pair_visit(PairSmem& sm, const PairArgs& a, const PairDesc& d, long long k, unsigned t,
                               int w, int lane) {
  const int gl = lane % G;
  const int rp = d.rp;
  double* out = a.out + d.out;
  double2 acc[Q], tv[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = tv[q] = make_double2(0.0, 0.0);
  for (int pass = 0; pass < 3; ++pass) {
    if (pass == 2 && !(d.own & 2)) break;
    for (;;) {
      const int s = t % kPD;
      mbar_wait(&sm.full[s], (t / kPD) & 1);
      const PairMeta mt = sm.meta[s];
      if (mt.k != k || mt.pass != pass) break;  // belongs to a later pass: keep it
      if (pass == 0) stage_work<G, Q, true, false>(sm, s, mt, rp, w, lane, acc, tv, out);
      else if (pass == 2) stage_work<G, Q, false, true>(sm, s, mt, rp, w, lane, acc, tv, out);
      else if ((d.own & 3) == 3) stage_work<G, Q, true, true>(sm, s, mt, rp, w, lane, acc, tv, out);
      else if (d.own & 1) stage_work<G, Q, false, true>(sm, s, mt, rp, w, lane, acc, tv, out);
      else stage_work<G, Q, true, false>(sm, s, mt, rp, w, lane, acc, tv, out);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
      ++t;
    }
    if (pass == 0) {
      if (d.own & 1) red_store<G, Q>(sm, acc, 0, w, lane, rp);
      named_bar(1, 32 * kPW);
      if (d.own & 1) red_load<G, Q>(sm, tv, 0, gl, rp);
    } else if (pass == 1) {
      if (d.own & 2) red_store<G, Q>(sm, acc, 1, w, lane, rp);
      named_bar(1, 32 * kPW);
      if (d.own & 2) red_load<G, Q>(sm, tv, 1, gl, rp);
    }
  }
  return t;
}

__global__ void __maxnreg__(128) pair_kernel(const PairArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PairSmem& sm = *reinterpret_cast<PairSmem*>(smem_raw);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // every slot a consumer may over-read must hold finite values (stage_work)
  for (unsigned i = threadIdx.x; i < offsetof(PairSmem, full) / 16; i += blockDim.x)
    reinterpret_cast<double2*>(smem_raw)[i] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPD; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kPW);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (w == kPW) {  // producer
    if (lane == 0) {
      unsigned long long pk, pd;
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pk));
      pd = l2_evict_first();
      unsigned t = 0;
      for (long long k = blockIdx.x; k < a.n; k += gridDim.x) {
        const PairDesc d = a.descs[k];
        const int rs = stage_rows(d.rp);
        for (int p = 0; p < 3; ++p) {
          int lo, hi;
          pass_range(d, p, lo, hi);
          for (int r = lo; r < hi; r += rs, ++t) {
            const int nr = min(rs, hi - r);
            PairMeta mt{static_cast<int>(k), p, r, nr, 0, 0};
            const double* xsrc = nullptr;
            unsigned xbytes = 0;
            if (p < 2) {  // passes A and B need x of their rows
              const long long i = p == 1 ? d.xrow + r : d.yrow + (r - d.m);
              const long long a0 = i & ~1LL;
              xsrc = a.xp + a0;
              xbytes = static_cast<unsigned>(((i + nr - a0 + 1) & ~1LL) * 8);
              mt.xo = static_cast<int>(i - a0);
            }
            pair_put(sm, t, mt, a.W + d.woff + static_cast<long long>(r) * d.rp,
                     static_cast<unsigned>(nr) * d.rp * 8u, xsrc, xbytes, p == 0 ? pk : pd);
          }
        }
      }
      pair_put(sm, t, PairMeta{-1, 0, 0, 0, 0, 0}, nullptr, 0, nullptr, 0, 0);  // stop marker
    }
    return;
  }
  unsigned t = 0;
  for (long long k = blockIdx.x; k < a.n; k += gridDim.x) {
    const PairDesc d = a.descs[k];
    const int rp = d.rp;
    if (rp <= 16) t = pair_visit<8, 1>(sm, a, d, k, t, w, lane);
    else if (rp <= 32) t = pair_visit<8, 2>(sm, a, d, k, t, w, lane);
    else if (rp <= 48) t = pair_visit<8, 3>(sm, a, d, k, t, w, lane);
    else if (rp <= 64) t = pair_visit<8, 4>(sm, a, d, k, t, w, lane);
    else if (rp <= 96) t = pair_visit<16, 3>(sm, a, d, k, t, w, lane);
    else t = pair_visit<16, 4>(sm, a, d, k, t, w, lane);
  }
  mbar_wait(&sm.full[t % kPD], (t / kPD) & 1);  // the stop marker
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
  static PerDeviceOnce attr;
  attr([] {
    H3D_CUDA_CHECK(cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sizeof(PairSmem))));
    H3D_CUDA_CHECK(cudaFuncSetAttribute(pair_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        cudaSharedmemCarveoutMaxShared));
  });
  int nb = 0;
  H3D_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pair_kernel, kPThreads,
                                                               sizeof(PairSmem)));
  // pairs are interleaved statically over the CTAs (deterministic)
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
