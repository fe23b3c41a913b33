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
//            p2_near_kernel   : near field (matrix-free, or the cached values)
//                               + direct leaf blocks, each owned pair once
//            p2_proxy_kernel  : K(X, P_A) s_A over proxy levels (FP64)
//            combine_kernel   : b[perm[p]] = compute + stream (fused un-permute).
//
// Every output has one writer and a fixed accumulation order (no atomics), so
// matvecs are bitwise reproducible (reference hmatrix.hpp:68-69).
#include "common.cuh"
#include "kernels.h"

#include <cstdio>
#include <cstdlib>
#include <mutex>

namespace h3db {

namespace {

constexpr double kFar = 1e100;  // coordinate of padding / inactive targets
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kP1Cols = 256;    // phase-1 columns per item
constexpr int kChunk = 256;     // phase-1 proxy: sources staged per round
constexpr int kHalfChunk = kChunk / 2;  // p1 / p2_proxy: two buffers of this many sources
static_assert(kHalfChunk == 128, "one staged source per thread of a 128-thread proxy CTA");
constexpr int kMaxRanges = 256; // phase-2 compute: source ranges per tile
// p2_stream's solves-done throttle gives up after this long (the solves take
// 0.3-2.5 ms; the flag orders nothing the kernel's results depend on)
constexpr unsigned long long kFlagWaitLimitNs = 20000000ULL;

// x in Morton order, into xp and the weight lane of the packed points
__global__ void gather_kernel(const double* __restrict__ x, const std::int32_t* __restrict__ perm,
                              std::int64_t n, double* __restrict__ xp, double* __restrict__ p4) {
  const std::int64_t p = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (p < n) {
    const double v = __ldg(x + perm[p]);
    xp[p] = v;
    p4[4 * p + 3] = v;
  }
}

__global__ void pack_w_kernel(const double* __restrict__ xp, std::int64_t n, double* __restrict__ p4) {
  const std::int64_t p = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (p < n) p4[4 * p + 3] = xp[p];
}

__global__ void pack_points_kernel(const double* __restrict__ px, const double* __restrict__ py,
                                   const double* __restrict__ pz, std::int64_t n,
                                   double4* __restrict__ p4) {
  const std::int64_t p = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (p < n) p4[p] = make_double4(px[p], py[p], pz[p], 0.0);
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

// ---- stream levels: tile pipeline --------------------------------------------
// Persistent CTA = one producer warp + kSC consumer warps. The producer
// claims work items (kBatch per atomic, descriptors prefetched) and streams
// their factor tiles (planner.h tile-major pools) into a kStages-deep
// shared-memory ring: one stage = up to kSC consecutive 8 KB tiles of one
// tile row, contiguous in the pool, moved by ONE cp.async.bulk (TMA engine,
// L2 evict-first) whose completion is counted in bytes on the stage's "full"
// mbarrier; consumer warp c takes tile c of every stage and releases the
// stage on its "empty" mbarrier. Few, large bulk copies keep the single
// issuing thread off the critical path; with the copies off the SM's load
// path one CTA (5 warps) per SM holds HBM near peak and leaves the rest of
// the SM to the FP64-bound kernels running beside it.
constexpr int kStages = 4;  // 4 x 32 KB in flight per SM (~19 MB device-wide)
constexpr int kSC = 4;      // consumer warps = tiles per stage
constexpr int kStreamThreads = 32 * (kSC + 1);
constexpr unsigned kTileBytes = kTileDoubles * sizeof(double);

struct StageMeta {
  int k;          // item (< 0: stop)
  int rt, ct;     // phase 1: tile row in the item; phase 2: first column tile of the stage
  int n;          // tiles in this stage
  long long aux;  // phase 1: first x row of the item; phase 2: output index of row 0
  int nrows;      // rows of the item
  int last;       // phase 1: column count; phase 2: 1 on the item's last stage
  long long sb;   // phase 2: S offset of the node's columns
};

struct StreamSmem {
  double tile[kStages][kSC * kTileDoubles];
  unsigned long long full[kStages], empty[kStages];
  StageMeta meta[kStages];
  double red[2][kSC][kTileRows];  // phase-2 cross-warp row sums (double-buffered)
};

__device__ __forceinline__ void stream_init(StreamSmem& sm) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kSC);
    }
    mbar_fence_init();
  }
  __syncthreads();
}

// Producer step: wait for stage t's slot, publish its metadata, start the
// copy of ntiles consecutive tiles (src == nullptr: the stop marker).
__device__ __forceinline__ void stream_put(StreamSmem& sm, unsigned t, const StageMeta& meta,
                                           const double* src, int ntiles, unsigned long long pol) {
  const int s = t % kStages;
  if (t >= kStages) mbar_wait(&sm.empty[s], ((t / kStages) - 1) & 1);
  sm.meta[s] = meta;
  if (src) {
    mbar_arrive_tx(&sm.full[s], kTileBytes * ntiles);
    bulk_g2s(sm.tile[s], src, kTileBytes * ntiles, &sm.full[s], pol);
  } else {
    mbar_arrive(&sm.full[s]);
  }
}

__device__ __forceinline__ StreamDesc shfl_desc(const StreamDesc& d, int src) {
  StreamDesc e;
  e.wbase = __shfl_sync(0xffffffffu, d.wbase, src);
  e.aux = __shfl_sync(0xffffffffu, d.aux, src);
  e.sbase = __shfl_sync(0xffffffffu, d.sbase, src);
  e.nrt = __shfl_sync(0xffffffffu, d.nrt, src);
  e.ncti = __shfl_sync(0xffffffffu, d.ncti, src);
  e.nct = __shfl_sync(0xffffffffu, d.nct, src);
  e.nrows = __shfl_sync(0xffffffffu, d.nrows, src);
  e.ncols = __shfl_sync(0xffffffffu, d.ncols, src);
  e.pad = 0;
  return e;
}

// Producer warp: claims kBatch items per atomic; the next claim and the next
// batch's descriptors are in flight while this batch's stages are issued, so
// the ring does not drain on a claim. Lane 0 issues the copies.
constexpr int kBatch = 8;
template <class Issue>
__device__ __forceinline__ void stream_producer(StreamSmem& sm, const StreamDesc* __restrict__ descs,
                                                long long nitems, unsigned* counter, Issue issue) {
  const int lane = threadIdx.x & 31;
  unsigned t = 0;
  long long base = 0;
  if (lane == 0) base = atomicAdd(counter, static_cast<unsigned>(kBatch));
  base = __shfl_sync(0xffffffffu, base, 0);
  StreamDesc d{};
  if (lane < kBatch && base + lane < nitems) d = descs[base + lane];
  while (base < nitems) {
    long long nb = 0;
    if (lane == 0) nb = atomicAdd(counter, static_cast<unsigned>(kBatch));
    const int cnt = static_cast<int>(min(static_cast<long long>(kBatch), nitems - base));
    for (int j = 0; j < cnt; ++j) {
      const StreamDesc e = shfl_desc(d, j);
      if (lane == 0) issue(t, static_cast<int>(base + j), e);
      __syncwarp();
    }
    base = __shfl_sync(0xffffffffu, nb, 0);
    if (lane < kBatch && base + lane < nitems) d = descs[base + lane];
  }
  if (lane == 0) stream_put(sm, t, StageMeta{-1, 0, 0, 0, 0, 0, 0, 0}, nullptr, 0, 0);
}

// ---- phase 1, stream levels: T = W_Z^T x_Z, item = <= 2048 rows x <= 256
// columns of W_Z; a stage is one tile row of the item (its <= kSC column
// tiles), consumer warp c owns the item's column tile c, lane = two columns,
// rows accumulated in order. x rows come from L2 through the read-only path,
// one row tile ahead.
__global__ void __maxnreg__(64) p1_stream_kernel(const P1Args a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  StreamSmem& sm = *reinterpret_cast<StreamSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  stream_init(sm);
  if (warp == 0) {
    const unsigned long long pol = l2_evict_first();
    stream_producer(sm, a.descs, a.nitems, a.counter, [&](unsigned& t, int k, const StreamDesc& e) {
      for (int rt = 0; rt < e.nrt; ++rt, ++t)
        stream_put(sm, t, StageMeta{k, rt, 0, e.ncti, e.aux, e.nrows, e.ncols, 0},
                   a.W + e.wbase + static_cast<long long>(rt) * e.nct * kTileDoubles, e.ncti, pol);
    });
    return;
  }
  const int cw = warp - 1;
  double acc0 = 0.0, acc1 = 0.0;
  long long pk = -1;
  int prt = -1;
  double xpre = 0.0;
  auto xload = [&](long long aux, int rt, int nrows) {
    const int r = rt * kTileRows + lane;
    return (lane < kTileRows && r < nrows) ? __ldg(a.xp + aux + r) : 0.0;
  };
  for (unsigned t = 0;; ++t) {
    const int s = t % kStages;
    mbar_wait(&sm.full[s], (t / kStages) & 1);
    const StageMeta m = sm.meta[s];
    if (m.k < 0) break;
    if (cw < m.n) {
      const double xv = (pk == m.k && prt == m.rt) ? xpre : xload(m.aux, m.rt, m.nrows);
      const int nrt = (m.nrows + kTileRows - 1) / kTileRows;
      if (m.rt + 1 < nrt) {
        xpre = xload(m.aux, m.rt + 1, m.nrows);
        pk = m.k;
        prt = m.rt + 1;
      }
      const double2* tl = reinterpret_cast<const double2*>(sm.tile[s] + cw * kTileDoubles);
#pragma unroll
      for (int i = 0; i < kTileRows; ++i) {
        const double xi = __shfl_sync(0xffffffffu, xv, i);
        const double2 w = tl[i * (kTileCols / 2) + lane];
        acc0 = fma(w.x, xi, acc0);
        acc1 = fma(w.y, xi, acc1);
      }
      if (m.rt == nrt - 1) {
        const P1Item it = a.items[m.k];
        const int c = cw * kTileCols + 2 * lane;
        if (c < m.last) p1_write(it, it.node, c, acc0, a);
        if (c + 1 < m.last) p1_write(it, it.node, c + 1, acc1, a);
        acc0 = acc1 = 0.0;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s]);
  }
}

// ---- proxy-level evaluation core (both phases): a 128-thread CTA owns up to
// 256 targets, two per thread (t and t + 128), and streams the sources
// through shared memory in chunks of kChunk, read as broadcasts; each staged
// source feeds two targets, two sources per step give four independent FP64
// chains per thread. Coordinates are centred on the node's box (planner.h
// `center`): a target is held as a = -2 t', tt = |t'|^2, a source as
// (s', ss = |s'|^2, w), and for partners at least one box apart
// r^2 = tt + ss - 2 t'.s' (1 DADD + 3 DFMA instead of 3 DADD + DMUL + 2 DFMA;
// rounding ~ eps (tt + ss) / r^2 < 50 eps there). Vertex-adjacent partners
// (whose points can nearly touch; their columns come first, vcols) use the
// difference form t' - s' = fma(-0.5, a, -s') exactly.
constexpr int kProxyThreads = 128;

struct Tgt {
  double ax, ay, az, tt;
};

template <int K, int NT, bool TRICK>
__device__ __forceinline__ void proxy_evalT(const Tgt (&tg)[2], double (&acc)[2][2],
                                            const double2* __restrict__ src, int j, int nj) {
  auto one = [&](int jj, int u) {
    const double2 s0 = src[3 * jj], s1 = src[3 * jj + 1], s2 = src[3 * jj + 2];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      double r2;
      if constexpr (TRICK) {
        r2 = fma(tg[t].ax, s0.x, fma(tg[t].ay, s0.y, fma(tg[t].az, s1.x, tg[t].tt + s1.y)));
      } else {
        r2 = sq3(fma(-0.5, tg[t].ax, -s0.x), fma(-0.5, tg[t].ay, -s0.y), fma(-0.5, tg[t].az, -s1.x));
      }
      acc[t][u] = far_acc<K>(r2, s2.x, acc[t][u]);
    }
  };
  for (; j + 3 < nj; j += 4) {  // four independent evaluations in flight per target
    one(j, 0);
    one(j + 1, 1);
    one(j + 2, 0);
    one(j + 3, 1);
  }
  for (; j < nj; ++j) one(j, 0);  // a runtime accumulator index would put acc in local memory
}

// nt = targets of this warp that exist (warp-uniform: 0, 1 or 2 per thread;
// warps without targets skip straight to the next barrier); sources [j0, jv)
// of the span are vertex-adjacent (difference form), [jv, j1) the rest
template <int K>
__device__ __forceinline__ void proxy_eval2(const Tgt (&tg)[2], double (&acc)[2][2],
                                            const double2* __restrict__ src, int j0, int jv, int j1,
                                            int nt, bool vertex_targets) {
  if (vertex_targets) jv = j1;  // a warp holding vertex-partner targets: all difference form
  if (nt == 2) {
    proxy_evalT<K, 2, false>(tg, acc, src, j0, jv);
    proxy_evalT<K, 2, true>(tg, acc, src, jv, j1);
  } else if (nt == 1) {
    proxy_evalT<K, 1, false>(tg, acc, src, j0, jv);
    proxy_evalT<K, 1, true>(tg, acc, src, jv, j1);
  }
}

__device__ __forceinline__ int warp_targets(int loc, int tpg, int n) {
  if (__any_sync(0xffffffffu, loc + tpg < n)) return 2;
  if (__any_sync(0xffffffffu, loc < n)) return 1;
  return 0;
}

__device__ __forceinline__ Tgt make_tgt(double x, double y, double z, const double4& c) {
  const double px = x - c.x, py = y - c.y, pz = z - c.z;
  return Tgt{-2.0 * px, -2.0 * py, -2.0 * pz, fma(pz, pz, fma(py, py, px * px))};
}

// ---- phase 1, proxy levels: v_c = sum_j K(P_c, z_j) x_j (targets = the
// item's proxies, sources = the node's points); items with <= 128 / <= 64
// proxies split the sources over 2 / 4 thread groups as in p2_proxy_kernel.
template <int K>
__global__ void __launch_bounds__(kProxyThreads, 5) p1_proxy_kernel(const P1Args a) {
  __shared__ double2 src[3 * kChunk];  // (x', y'), (z', ss), (w, -)
  __shared__ double red[2 * kProxyThreads];
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
    const double4 cen = reinterpret_cast<const double4*>(a.cen)[g];
    const int G = it.ncols <= 64 ? 4 : it.ncols <= 128 ? 2 : 1;
    const int tpg = kProxyThreads / G;
    const int grp = threadIdx.x / tpg, loc = threadIdx.x % tpg;
    const int nt = warp_targets(loc, tpg, it.ncols);
    const int vc = a.vcols[g] - it.col0;  // target columns < vc: vertex partners
    const bool vwarp = __any_sync(0xffffffffu, loc < vc);
    Tgt tg[2];
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int c = loc + t * tpg;
      const std::int64_t qi = a.nt.soff[g] + it.col0 + c;
      const double4 q = c < it.ncols ? reinterpret_cast<const double4*>(a.q4)[qi]
                                     : make_double4(kFar, kFar, kFar, 0.0);
      tg[t] = make_tgt(q.x, q.y, q.z, cen);
    }
    // sources (the node's points) in chunks of kHalfChunk, double-buffered
    // like p2_proxy_kernel: one barrier per chunk, the next chunk's loads in
    // flight during the current chunk's evaluations
    const double4* P4s = reinterpret_cast<const double4*>(a.p4) + rb;
    const int nrw = it.nrows;
    auto stage = [&](double2* d, const double4& v) {
      const double px = v.x - cen.x, py = v.y - cen.y, pz = v.z - cen.z;
      d[0] = make_double2(px, py);
      d[1] = make_double2(pz, fma(pz, pz, fma(py, py, px * px)));
      d[2] = make_double2(v.w, 0.0);
    };
    double4 nv = make_double4(0.0, 0.0, 0.0, 0.0);
    if (threadIdx.x < nrw) nv = P4s[threadIdx.x];
    __syncthreads();  // the previous item is done with both buffers
    stage(src + 3 * threadIdx.x, nv);
    __syncthreads();
    for (int j0 = 0, b = 0; j0 < nrw; j0 += kHalfChunk, b ^= 1) {
      const int nj = min(kHalfChunk, nrw - j0);
      const bool more = j0 + kHalfChunk < nrw;
      const int qn = j0 + kHalfChunk + threadIdx.x;
      if (more && qn < nrw) nv = P4s[qn];
      const int sub = (nj + G - 1) / G;
      const int lo = min(nj, grp * sub), hi = min(nj, lo + sub);
      proxy_eval2<K>(tg, acc, src + 3 * kHalfChunk * b, lo, lo, hi, nt, vwarp);
      if (more && qn < nrw) stage(src + 3 * kHalfChunk * (b ^ 1) + 3 * threadIdx.x, nv);
      __syncthreads();
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) red[grp * 2 * tpg + loc + t * tpg] = acc[t][0] + acc[t][1];
    __syncthreads();
    for (int c = threadIdx.x; c < it.ncols; c += kProxyThreads) {
      const int per = 2 * tpg;
      double v = 0.0;
      for (int q = 0; q < G; ++q) v += red[q * per + c];
      p1_write(it, g, c, far_scale<K>() * v, a);
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
                                    const double* __restrict__ pz, const double4* __restrict__ cen,
                                    double4* __restrict__ q4, double4* __restrict__ q4c) {
  const std::int64_t s = blockIdx.x * static_cast<std::int64_t>(blockDim.y) + threadIdx.y;
  if (s >= nseg) return;
  const ProxySeg sg = segs[s];
  const double4 c = cen[sg.node];
  for (int q = threadIdx.x; q < sg.r; q += blockDim.x) {
    // side 0: Z = X, proxies = column pivots tau (in Y = k); side 1: row pivots sigma
    const std::int32_t loc = piv[sg.piv_off + (sg.side == 0 ? sg.r : 0) + q];
    const std::int64_t idx = sg.base + loc;
    q4[sg.so + q] = make_double4(px[idx], py[idx], pz[idx], 0.0);
    const double x = px[idx] - c.x, y = py[idx] - c.y, z = pz[idx] - c.z;
    q4c[sg.so + q] = make_double4(x, y, z, fma(z, z, fma(y, y, x * x)));
  }
}

// Triangular inverses of the packed pivot LU, in place (build time; one thread
// per column): strict lower <- L^-1 (unit diagonal implied), upper incl.
// diagonal <- R^-1, and the same matrix column-major at lu + lu_total (the
// side-0 solve reads it by columns). Applying L^-1 and R^-1 as two GEMVs is as
// accurate as the reference's forward/backward substitution
// (lowrank.cpp:310-320) on these ill-conditioned pivot blocks (cond ~ 1e12 at
// eps 1e-10), unlike forming (L R)^-1, and turns the sequential solves into
// coalesced, parallel GEMVs.
__global__ void lu_invert_kernel(const ProxySeg* __restrict__ segs, std::int64_t nseg,
                                 double* __restrict__ lu, std::int64_t lu_total,
                                 double* __restrict__ scratch, int max_r) {
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
  double* AT = A + lu_total;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int hi = e / r, lo = e % r;
    A[e] = Gs[static_cast<std::int64_t>(lo) * max_r + hi];   // row-major: (row hi, col lo)
    AT[e] = Gs[static_cast<std::int64_t>(hi) * max_r + lo];  // column-major: (row lo, col hi)
  }
}

// ---- proxy solves: one ordered proxy block per warp, in place on S -------
// Lane owns outputs i = lane + 32 k (k < NK = ceil(r / 32)). Both triangular
// factors are applied in ONE pass over the rows of the r x r inverse block
// (column-major PT for side 0, row-major P for side 1), so every block is
// read from HBM once per orientation (2 x 8 r^2 bytes per pair):
//   side 0 (target = pair's row side X):  s = R^-1 (L^-1 v)       (lowrank.cpp:310-320)
//     row j of PT: w_j = v_j + (tail sums so far) is complete (rows < j added
//     their strictly-lower parts), then head i <= j: s_i += PT[j][i] w_j and
//     tail i > j: t_i += PT[j][i] v_j
//   side 1 (target = pair's col side Y):  s = L^-T (R^-T v)       (the transposed block)
//     row i of P: tail j >= i: u_j += P[i][j] v_i (u_i is then complete),
//     head j < i: s_j += P[i][j] u_i; finally s_j += u_j
// The completed value of row j lives in lane j % 32's register j / 32 and is
// broadcast with one shuffle. Fixed order per output: deterministic.
//
// The rows stream through shared memory: every warp runs its own bulk-copy
// ring (kSolveStages stages of up to kSolveStageD doubles, blocks of whole
// rows, lane 0 issues cp.async.bulk into the stage it just consumed), so the
// copies of the next blocks - across segment boundaries - are in flight while
// the warp works through the current rows from shared memory. Segments are
// assigned round-robin over all warps of the grid (host-sorted by
// decreasing rank for balance).
#ifndef H3D_SOLVE_STAGES
#define H3D_SOLVE_STAGES 2
#endif
constexpr int kSolveWarps = 4;
constexpr int kSolveStages = H3D_SOLVE_STAGES;
constexpr int kSolveStageD = 640;  // 5 KB per stage: two rows of the largest block (r <= 320)
constexpr int kSolveMaxR = 320;
static_assert(kSolveStageD >= 2 * kSolveMaxR, "a stage holds at least two rows");

constexpr int kSolveQ = 8;  // claimed segments queued per warp (issue runs <= kSolveStages ahead)

struct SolveSmem {
  double ring[kSolveWarps][kSolveStages][kSolveStageD];
  double v[kSolveWarps][kSolveMaxR];
  unsigned long long full[kSolveWarps][kSolveStages];
  long long queue[kSolveWarps][kSolveQ];  // segments in issue order (nseg: no more)
};

// rows per staged block (even, so every block starts 16-byte aligned)
__device__ __forceinline__ int solve_block_rows(int r) { return max(2, (kSolveStageD / r) & ~1); }

// Issue cursor of a warp (lane 0): segments are claimed dynamically (an
// atomic counter over the rank-sorted list, so the largest blocks go first
// and a CTA that starts late, beside other kernels, takes less), queued in
// claim order for the consuming side.
struct SolveIssue {
  long long seg;  // segment being issued (< 0: claim the next one)
  int row;        // next row of that segment to copy
  unsigned n;     // blocks issued so far
  unsigned q;     // segments queued so far
  bool done;      // the terminator is queued
};

struct SolveCtx {
  const ProxySeg* segs;
  std::int64_t nseg;
  unsigned* counter;
  const double* lu;
  std::int64_t lu_total;
  unsigned long long pol;
};

// lane 0: copy the next row block of this warp's segment stream (claiming a
// segment when the previous one is fully issued) into stage n % kSolveStages
__device__ __forceinline__ void solve_issue(SolveSmem& sm, int w, SolveIssue& is, const SolveCtx& cx) {
  if (is.done) return;
  if (is.seg < 0) {
    is.seg = static_cast<long long>(atomicAdd(cx.counter, 1u));
    if (is.seg >= cx.nseg) is.seg = cx.nseg;
    sm.queue[w][is.q++ % kSolveQ] = is.seg;
    if (is.seg >= cx.nseg) {
      is.done = true;
      return;
    }
  }
  const ProxySeg sg = cx.segs[is.seg];
  const int r = sg.r, rb = solve_block_rows(r);
  const int nrow = min(rb, r - is.row);
  long long nd = static_cast<long long>(nrow) * r;
  nd += nd & 1;  // 16-byte multiple (the packed slot has r^2 + (r & 1) doubles)
  const double* src = cx.lu + sg.lu_off + (sg.side == 0 ? cx.lu_total : 0) + static_cast<long long>(is.row) * r;
  const int st = is.n % kSolveStages;
  mbar_arrive_tx(&sm.full[w][st], static_cast<unsigned>(nd * 8));
  bulk_g2s(sm.ring[w][st], src, static_cast<unsigned>(nd * 8), &sm.full[w][st], cx.pol);
  ++is.n;
  is.row += nrow;
  if (is.row >= r) {
    is.row = 0;
    is.seg = -1;
  }
}

template <int NK, bool SIDE1>
__device__ __forceinline__ void solve_rows(SolveSmem& sm, int w, int lane, int r, const double* v,
                                           double* __restrict__ out, unsigned& c, SolveIssue& is,
                                           const SolveCtx& cx) {
  double t[NK], acc[NK];
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    t[k] = 0.0;
    acc[k] = 0.0;
  }
  const int rb = solve_block_rows(r);
  for (int j0 = 0; j0 < r; j0 += rb) {
    const int st = c % kSolveStages;
    mbar_wait(&sm.full[w][st], (c / kSolveStages) & 1);
    const double* blk = sm.ring[w][st];
    const int j1 = min(r, j0 + rb);
    for (int j = j0; j < j1; ++j) {
      const double* row = blk + (j - j0) * r;
      const double vj = v[j];
      const int kj = j >> 5, lj = j & 31;
      double cv[NK];
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        const int i = lane + 32 * k;
        cv[k] = i < r ? row[i] : 0.0;
      }
      if constexpr (!SIDE1) {
        double tj = t[0];
#pragma unroll
        for (int k = 1; k < NK; ++k) tj = k == kj ? t[k] : tj;
        const double wj = vj + __shfl_sync(0xffffffffu, tj, lj);
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          const int i = lane + 32 * k;
          if (i <= j) acc[k] = fma(cv[k], wj, acc[k]);
          else t[k] = fma(cv[k], vj, t[k]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          const int i = lane + 32 * k;
          if (i >= j) t[k] = fma(cv[k], vj, t[k]);
        }
        double tj = t[0];
#pragma unroll
        for (int k = 1; k < NK; ++k) tj = k == kj ? t[k] : tj;
        const double uj = __shfl_sync(0xffffffffu, tj, lj);
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          const int i = lane + 32 * k;
          if (i < j) acc[k] = fma(cv[k], uj, acc[k]);
        }
      }
    }
    __syncwarp();  // every lane is done with this stage
    ++c;
    if (lane == 0) solve_issue(sm, w, is, cx);
  }
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const int i = lane + 32 * k;
    if (i < r) out[i] = SIDE1 ? t[k] + acc[k] : acc[k];  // in place over v
  }
}

template <int NK>
__device__ __noinline__ void solve_seg(SolveSmem& sm, int w, int lane, const ProxySeg& sg, const double* v,
                                       double* out, unsigned& c, SolveIssue& is, const SolveCtx& cx) {
  if (sg.side == 0) solve_rows<NK, false>(sm, w, lane, sg.r, v, out, c, is, cx);
  else solve_rows<NK, true>(sm, w, lane, sg.r, v, out, c, is, cx);
}

__global__ void __launch_bounds__(32 * kSolveWarps) proxy_solve_kernel(const ProxySeg* __restrict__ segs,
                                                                        std::int64_t nseg,
                                                                        const double* __restrict__ lu,
                                                                        std::int64_t lu_total,
                                                                        double* __restrict__ S, unsigned* counter) {
  extern __shared__ __align__(128) unsigned char solve_smem[];
  SolveSmem& sm = *reinterpret_cast<SolveSmem*>(solve_smem);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  SolveCtx cx;
  cx.segs = segs;
  cx.nseg = nseg;
  cx.counter = counter;
  cx.lu = lu;
  cx.lu_total = lu_total;
  cx.pol = l2_evict_first();
  if (lane == 0) {
    for (int st = 0; st < kSolveStages; ++st) mbar_init(&sm.full[w][st], 1);
    mbar_fence_init();
  }
  __syncwarp();
  SolveIssue is{-1, 0, 0, 0, false};
  if (lane == 0)
    for (int st = 0; st < kSolveStages; ++st) solve_issue(sm, w, is, cx);
  __syncwarp();
  unsigned c = 0;
  double* v = sm.v[w];
  for (unsigned qh = 0;; ++qh) {
    const long long sidx = sm.queue[w][qh % kSolveQ];
    if (sidx >= nseg) break;
    const ProxySeg sg = segs[sidx];
    double* Sg = S + sg.so;
    for (int q = lane; q < sg.r; q += 32) v[q] = Sg[q];
    __syncwarp();
    switch ((sg.r + 31) >> 5) {
      case 0: break;
      case 1: solve_seg<1>(sm, w, lane, sg, v, Sg, c, is, cx); break;
      case 2: solve_seg<2>(sm, w, lane, sg, v, Sg, c, is, cx); break;
      case 3: solve_seg<3>(sm, w, lane, sg, v, Sg, c, is, cx); break;
      case 4: solve_seg<4>(sm, w, lane, sg, v, Sg, c, is, cx); break;
      case 5: solve_seg<5>(sm, w, lane, sg, v, Sg, c, is, cx); break;
      case 6: solve_seg<6>(sm, w, lane, sg, v, Sg, c, is, cx); break;
      case 7: solve_seg<7>(sm, w, lane, sg, v, Sg, c, is, cx); break;
      case 8: solve_seg<8>(sm, w, lane, sg, v, Sg, c, is, cx); break;
      case 9: solve_seg<9>(sm, w, lane, sg, v, Sg, c, is, cx); break;
      default: solve_seg<10>(sm, w, lane, sg, v, Sg, c, is, cx); break;
    }
    __syncwarp();  // v is reused by the next segment; the queue entry is read
  }
}

// ---- phase 2, near field + direct leaf blocks, matrix-free ------------------
// Warp-specialised persistent CTA: a producer warp claims owned leaves X,
// builds X's source range table (planner.h sym lists: self | dense one-way |
// direct one-way | dense sym | direct sym) and streams the flattened sources
// from the packed (x, y, z, w) points into a double-buffered shared stage
// with cp.async.bulk (one copy per range piece, byte-counted on the buffer's
// "full" mbarrier); seven consumer warps own the leaf's rows (warp w: rows
// [w RPW, (w + 1) RPW), RPW = ceil(m / 7) <= 7), lanes stride over the staged
// sources and evaluate each one against the warp's RPW rows (RPW independent
// FP64 chains per lane). Dense-near sources use the full-accuracy rsqrt (+ the
// diagonal rule on the self block), admissible ones the Newton form.
// Symmetry: an owned pair (X, Y), Y > X, is evaluated once - each entry feeds
// X's row sums and a column sum for Y's point (sum over the warp's rows, then
// over the warps through shared memory in warp order), written to the pair
// buffer; combine adds Y's incoming runs. Every output has one writer and a
// fixed order: bitwise reproducible.
constexpr int kNearStage = 256;            // sources per staged chunk (8 KB)
constexpr int kNearConsumers = kWarps - 1;  // 7 consumer warps + 1 producer = 256 threads
constexpr int kNearThreads = 32 * (kNearConsumers + 1);
constexpr int kNearRows = kNearPassRows;  // rows per pass (7 per consumer warp; larger leaves: 2+ passes)
static_assert(kNearRows == 7 * kNearConsumers, "near pass = 7 rows per consumer warp");
constexpr int kMaxNear = kMaxNearRanges;

struct NearMeta {
  long long xb;    // first permuted row of the leaf
  long long obase; // pair-buffer index of flattened source 0 (sym sources only)
  int r0, mr;      // row pass: rows [r0, r0 + mr) of the leaf (mr <= kNearRows)
  int base, cnt;   // flattened index of the chunk's first source, sources in the chunk (< 0: stop)
  int e0, e1, e2, e3;  // flattened ends: self, dense one-way, direct one-way, dense sym
  int last;        // last chunk of this row pass
  int nds;         // stored near field: dense columns of the leaf (row stride)
  long long nfb;   // stored near field: the leaf's block offset
};

struct NearSmem {
  double4 stage[2][kNearStage];
  double col[kNearConsumers][kNearStage];  // per-warp column partials of sym sources
  unsigned long long full[2], empty[2];
  NearMeta meta[2];
  long long rstart[kMaxNear];  // producer's range table (permuted index, length)
  int rlen[kMaxNear];
};

// Staged sources are 32-byte (x, y, z, w) records read one per lane: two
// 16-byte loads per lane, the half order swizzled by lane bit 2 so each
// group of 8 lanes covers all 32 banks (a plain stride-32 B read is 2-way
// bank-conflicted).
__device__ __forceinline__ double4 ld_src(const double4* __restrict__ st, int j, int h) {
  const double2* p = reinterpret_cast<const double2*>(st + j);
  const double2 a = p[h], b = p[h ^ 1];
  return h ? make_double4(b.x, b.y, a.x, a.y) : make_double4(a.x, a.y, b.x, b.y);
}

// One row accumulator per row in the admissible (Newton) scale: dense-near
// terms enter with weight w / far_scale (exact power-of-two scalings), the
// caller multiplies by far_scale once; column partials likewise.
template <int K, int RPW, bool DENSE, bool SYM, bool STORED>
__device__ __forceinline__ void near_seg(const double4* __restrict__ st, int lo, int hi,
                                         const double (&tx)[RPW], const double (&ty)[RPW],
                                         const double (&tz)[RPW], const double (&tw)[RPW],
                                         double (&acc)[RPW], double* __restrict__ col, int lane,
                                         const double* __restrict__ nf0, int nds, int nvalid, int dbias) {
  constexpr double inv = 1.0 / far_scale<K>();
  const int h = (lane >> 2) & 1;
  for (int j = lo + lane; j < hi; j += 32) {
    const double4 q = ld_src(st, j, h);
    double cp = 0.0;
    if constexpr (DENSE) {
      const double w = inv * q.w;
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        double k;
        if constexpr (STORED) k = r < nvalid ? ldg_stream(nf0 + r * nds + j + dbias) : 0.0;
        else k = kernel_r2_fast<K>(sq3(tx[r] - q.x, ty[r] - q.y, tz[r] - q.z));
        acc[r] = fma(k, w, acc[r]);
        if constexpr (SYM) cp = fma(k, tw[r], cp);
      }
      if constexpr (SYM) col[j] = inv * cp;
    } else {
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        if constexpr (STORED) {
          // the stored Newton-form value (near_store_kernel), both sums
          const double g = r < nvalid ? ldg_stream(nf0 + r * nds + j + dbias) : 0.0;
          acc[r] = fma(g, q.w, acc[r]);
          if constexpr (SYM) cp = fma(g, tw[r], cp);
        } else {
          const double r2 = sq3(tx[r] - q.x, ty[r] - q.y, tz[r] - q.z);
          if constexpr (SYM) {
            // the Newton-form value once, for both sums
            const double g = far_acc<K>(r2, 1.0, 0.0);
            acc[r] = fma(g, q.w, acc[r]);
            cp = fma(g, tw[r], cp);
          } else {
            acc[r] = far_acc<K>(r2, q.w, acc[r]);
          }
        }
      }
      if constexpr (SYM) col[j] = cp;
    }
  }
}

// The stored near field (STORED) replaces every dense kernel value by the one
// the build stored for it (near_store_kernel: the same function of the same
// operands), so cached and matrix-free matvecs agree bit for bit (reference
// test_hmatrix.cpp:138-152). Row r of the warp reads nfr[r] (null: padding
// row) at the source's dense column: flattened index f for f < e1, f - (e2 -
// e1) in the dense sym segment.
template <int K, int RPW, bool STORED>
__device__ __forceinline__ void near_chunk(const double4* __restrict__ st, const NearMeta& mt, int row0,
                                           const double (&tx)[RPW], const double (&ty)[RPW],
                                           const double (&tz)[RPW], const double (&tw)[RPW],
                                           double (&acc)[RPW], double* __restrict__ col, double diag,
                                           int lane, const double* __restrict__ nf0, int nvalid, int mask) {
  constexpr double inv = 1.0 / far_scale<K>();
  const int h = (lane >> 2) & 1;
  const int base = mt.base, cnt = mt.cnt;
  auto cut = [&](int e) { return max(0, min(cnt, e - base)); };
  const int c0 = cut(mt.e0), c1 = cut(mt.e1), c2 = cut(mt.e2), c3 = cut(mt.e3);
  // NF column of flattened source f (planner.h): the unstored categories
  // before it are skipped
  const bool sd = STORED && (mask & 1), sx = STORED && (mask & 2);
  const int bd1 = sd ? 0 : mt.e1;                            // direct one-way
  const int bs2 = sx ? 0 : mt.e2 - mt.e1;                    // dense sym
  const int bx2 = sd ? 0 : mt.e1 + (mt.e3 - mt.e2);           // direct sym
  // self block, diagonal rule
  for (int j = lane; j < c0; j += 32) {
    const double4 q = ld_src(st, j, h);
    const double w = inv * q.w;
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      double k;
      if (sd) k = r < nvalid ? ldg_stream(nf0 + r * mt.nds + base + j) : 0.0;
      else k = (row0 + r == base + j) ? diag : kernel_r2_fast<K>(sq3(tx[r] - q.x, ty[r] - q.y, tz[r] - q.z));
      acc[r] = fma(k, w, acc[r]);
    }
  }
  if (sd) near_seg<K, RPW, true, false, true>(st, c0, c1, tx, ty, tz, tw, acc, col, lane, nf0, mt.nds, nvalid, base);
  else near_seg<K, RPW, true, false, false>(st, c0, c1, tx, ty, tz, tw, acc, col, lane, nf0, 0, 0, 0);
  if (sx)
    near_seg<K, RPW, false, false, true>(st, c1, c2, tx, ty, tz, tw, acc, col, lane, nf0, mt.nds, nvalid, base - bd1);
  else near_seg<K, RPW, false, false, false>(st, c1, c2, tx, ty, tz, tw, acc, col, lane, nf0, 0, 0, 0);
  if (sd)
    near_seg<K, RPW, true, true, true>(st, c2, c3, tx, ty, tz, tw, acc, col, lane, nf0, mt.nds, nvalid, base - bs2);
  else near_seg<K, RPW, true, true, false>(st, c2, c3, tx, ty, tz, tw, acc, col, lane, nf0, 0, 0, 0);
  if (sx)
    near_seg<K, RPW, false, true, true>(st, c3, cnt, tx, ty, tz, tw, acc, col, lane, nf0, mt.nds, nvalid, base - bx2);
  else near_seg<K, RPW, false, true, false>(st, c3, cnt, tx, ty, tz, tw, acc, col, lane, nf0, 0, 0, 0);
}

// Consumer warp: one row pass of one leaf, starting at the (already waited)
// stage t; returns the next stage sequence number.
template <int K, int RPW, bool STORED>
__device__ unsigned near_consume(NearSmem& sm, const Phase2Args& a, unsigned t) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const NearMeta m0 = sm.meta[t % 2];
  const int row0 = m0.r0 + warp * RPW;
  const double4* P4 = reinterpret_cast<const double4*>(a.p4);
  double tx[RPW], ty[RPW], tz[RPW], tw[RPW], acc[RPW];
  // stored near field: this warp's first row, rows below nvalid are real
  const int nvalid = STORED ? max(0, min(RPW, m0.r0 + m0.mr - row0)) : 0;
  const double* nf0 = STORED ? a.NF + m0.nfb + static_cast<long long>(row0) * m0.nds : nullptr;
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const bool ok = row0 + r < m0.r0 + m0.mr;
    const double4 q = ok ? P4[m0.xb + row0 + r] : make_double4(kFar, kFar, kFar, 0.0);
    tx[r] = q.x;
    ty[r] = q.y;
    tz[r] = q.z;
    tw[r] = q.w;
    acc[r] = 0.0;
  }
  for (;;) {
    const int s = t % 2;
    const NearMeta mt = sm.meta[s];
    near_chunk<K, RPW, STORED>(sm.stage[s], mt, row0, tx, ty, tz, tw, acc, sm.col[warp], a.diag, lane, nf0,
                               nvalid, a.nf_mask);
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s]);
    if (mt.base + mt.cnt > mt.e2) {  // chunk holds sym sources: column sums in warp order
      named_bar(1, 32 * kNearConsumers);
      const int lo = max(0, mt.e2 - mt.base);
      for (int j = lo + threadIdx.x; j < mt.cnt; j += 32 * kNearConsumers) {
        double v = sm.col[0][j];
#pragma unroll
        for (int w = 1; w < kNearConsumers; ++w) v += sm.col[w][j];
        a.pairbuf[mt.obase + mt.base + j] = far_scale<K>() * v;
      }
      named_bar(1, 32 * kNearConsumers);
    }
    ++t;
    if (mt.last) break;
    mbar_wait(&sm.full[t % 2], (t / 2) & 1);
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const double v = far_scale<K>() * warp_sum(acc[r]);
    const int i = row0 + r;
    if (lane == r && i < m0.r0 + m0.mr) {
      if (a.cpart_out) a.cpart_out[m0.xb + i] = v;
      else a.b[a.perm[m0.xb + i]] = v;
    }
  }
  return t;
}

// Producer warp: wait for the stage's slot, copy the chunk's range pieces,
// publish its metadata: one cp.async.bulk per piece from lane 0, byte-counted
// on the buffer's mbarrier (H3D_NEAR_LDG: the warp's lanes copy the records
// with 16-byte loads instead - measured 1.4x slower, the producer then
// cannot stay a chunk ahead).
__device__ __forceinline__ void near_put(NearSmem& sm, unsigned t, NearMeta mt, const double4* p4,
                                         int& re, int& roff, int nrange, int lane) {
  const int s = t % 2;
  if (t >= 2) {
    if (lane == 0) mbar_wait(&sm.empty[s], ((t / 2) - 1) & 1);
    __syncwarp();
  }
  int filled = 0;
  if (mt.cnt >= 0) {
    while (re < nrange && filled < kNearStage) {
      const int len = sm.rlen[re];
      const int take = min(len - roff, kNearStage - filled);
      if (take > 0) {
        const double4* src = p4 + sm.rstart[re] + roff;
#ifndef H3D_NEAR_LDG
        if (lane == 0) {
          const unsigned bytes = static_cast<unsigned>(take) * 32u;
          mbar_expect_tx(&sm.full[s], bytes);
          bulk_g2s(&sm.stage[s][filled], src, bytes, &sm.full[s], 0);
        }
#else
        const double2* s2 = reinterpret_cast<const double2*>(src);
        double2* d2 = reinterpret_cast<double2*>(&sm.stage[s][filled]);
        for (int i = lane; i < 2 * take; i += 32) d2[i] = __ldg(s2 + i);
#endif
        filled += take;
        roff += take;
      }
      if (roff >= len) {
        ++re;
        roff = 0;
      }
    }
    mt.cnt = filled;
  }
  __syncwarp();
  if (lane == 0) {
    sm.meta[s] = mt;
    mbar_arrive(&sm.full[s]);
  }
}

template <int K, bool STORED>
__global__ void __launch_bounds__(kNearThreads, 2) p2_near_kernel(const Phase2Args a) {
  __shared__ __align__(128) NearSmem sm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.full[b], 1);
      mbar_init(&sm.empty[b], kNearConsumers);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kNearConsumers) {  // producer warp
    const double4* P4 = reinterpret_cast<const double4*>(a.p4);
    unsigned t = 0;
    for (;;) {
      long long k = 0;
      if (lane == 0) k = static_cast<long long>(atomicAdd(a.counter, 1u));
      k = __shfl_sync(0xffffffffu, k, 0);
      if (k >= a.nleaves) break;
      const std::int64_t X = a.leaf0 + k;
      const std::int64_t xb = a.leaf_off[X];
      const int m = static_cast<int>(a.leaf_off[X + 1] - xb);
      if (m == 0) continue;
      const std::int32_t nb = a.sym_off[X], ne = a.sym_off[X + 1];
      const int nrange = ne - nb;
      // range-count boundaries of the four categories after self
      const int b1 = 1 + a.sym_cnt[4 * X], b2 = b1 + a.sym_cnt[4 * X + 1];
      const int b3 = b2 + a.sym_cnt[4 * X + 2];
      int tot = 0, e1 = 0, e2 = 0, e3 = 0;  // per lane, then warp-reduced (integers: exact)
      for (int e = lane; e < nrange; e += 32) {
        const std::int32_t Y = a.sym_ids[nb + e];
        const std::int64_t yb = a.leaf_off[Y];
        const int len = static_cast<int>(a.leaf_off[Y + 1] - yb);
        sm.rstart[e] = yb;
        sm.rlen[e] = len;
        tot += len;
        if (e < b1) e1 += len;
        if (e < b2) e2 += len;
        if (e < b3) e3 += len;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        tot += __shfl_xor_sync(0xffffffffu, tot, o);
        e1 += __shfl_xor_sync(0xffffffffu, e1, o);
        e2 += __shfl_xor_sync(0xffffffffu, e2, o);
        e3 += __shfl_xor_sync(0xffffffffu, e3, o);
      }
      __syncwarp();
      // Ranges that follow one another in the packed point array (the
      // children of one parent cell are consecutive leaves) merge into one
      // copy: the flattened source order is unchanged, the producer issues
      // 3-5x fewer bulk copies per leaf (it is the bottleneck on small
      // leaves: one lane issues them). In place, 32 ranges per step.
      int nrun = 0;
      {
        long long carry_end = -1;
        for (int base = 0; base < nrange; base += 32) {
          const int e = base + lane;
          const bool valid = e < nrange;
          const long long rs = valid ? sm.rstart[e] : 0;
          const int rl = valid ? sm.rlen[e] : 0;
          const long long my_end = rs + rl;
          long long prev_end = __shfl_up_sync(0xffffffffu, my_end, 1);
          if (lane == 0) prev_end = carry_end;
          const bool head = valid && rs != prev_end;
          const unsigned heads = __ballot_sync(0xffffffffu, head);
          const int nv = __popc(__ballot_sync(0xffffffffu, valid));
          int cum = rl;  // inclusive prefix of the lengths
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int up = __shfl_up_sync(0xffffffffu, cum, o);
            if (lane >= o) cum += up;
          }
          // ranges before the block's first head continue the previous run
          const int first = heads ? __ffs(heads) - 1 : nv;
          const int lead = __shfl_sync(0xffffffffu, cum, max(first - 1, 0));
          // a head's run ends before the next head (or the block's end)
          const unsigned after = lane == 31 ? 0u : heads & ~((2u << lane) - 1u);
          const int nxt = after ? __ffs(after) - 1 : nv;
          const int cum_end = __shfl_sync(0xffffffffu, cum, max(nxt - 1, 0));
          const long long last_end = __shfl_sync(0xffffffffu, my_end, max(nv - 1, 0));
          __syncwarp();
          if (lane == 0 && first > 0) sm.rlen[nrun - 1] += lead;
          if (head) {
            const int w = nrun + __popc(heads & ((1u << lane) - 1u));
            sm.rstart[w] = rs;
            sm.rlen[w] = cum_end - cum + rl;
          }
          nrun += __popc(heads);
          carry_end = last_end;
          __syncwarp();
        }
      }
      const long long obase = a.out_off[X] - e2;
      const int nchunks = (tot + kNearStage - 1) / kNearStage;
      const long long nfb = STORED ? a.nf_off[X] : 0;
      const int nds = STORED ? a.nf_cols[X] : 0;
      for (int r0 = 0; r0 < m; r0 += kNearRows) {
        const int mr = min(kNearRows, m - r0);
        // leaves above one pass have no sym partners (planner.cpp), so the
        // column sums of a sym source are always complete after one sweep
        int re = 0, roff = 0;
        for (int c = 0; c < nchunks; ++c, ++t)
          near_put(sm, t,
                   NearMeta{xb, obase, r0, mr, c * kNearStage, 0, m, e1, e2, e3,
                            c + 1 == nchunks ? 1 : 0, nds, nfb},
                   P4, re, roff, nrun, lane);
      }
      __syncwarp();
    }
    {
      int re = 0, roff = 0;
      near_put(sm, t, NearMeta{0, 0, 0, 0, 0, -1, 0, 0, 0, 0, 1, 0, 0}, P4, re, roff, 0, lane);
    }
    return;
  }
  unsigned t = 0;
  for (;;) {
    mbar_wait(&sm.full[t % 2], (t / 2) & 1);
    const NearMeta mt = sm.meta[t % 2];
    if (mt.cnt < 0) break;
    switch ((mt.mr + kNearConsumers - 1) / kNearConsumers) {
      case 1: t = near_consume<K, 1, STORED>(sm, a, t); break;
      case 2: t = near_consume<K, 2, STORED>(sm, a, t); break;
      case 3: t = near_consume<K, 3, STORED>(sm, a, t); break;
      case 4: t = near_consume<K, 4, STORED>(sm, a, t); break;
      case 5: t = near_consume<K, 5, STORED>(sm, a, t); break;
      case 6: t = near_consume<K, 6, STORED>(sm, a, t); break;
      default: t = near_consume<K, 7, STORED>(sm, a, t); break;
    }
  }
}

// ---- phase 2, stream levels: rows of W_A . S_A, item = one row tile of an
// owned node A (all its column tiles, kSC per stage); consumer warp c owns
// column tiles c, c + kSC, ..., lane = two columns, sixteen row accumulators;
// S columns come through the read-only path one stage ahead. At the item's
// last stage the warps reduce (fixed butterfly, then warp order) and write
// the level's partial (combined in level order by combine_kernel).
__global__ void __maxnreg__(64) p2_stream_kernel(const Phase2Args a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  StreamSmem& sm = *reinterpret_cast<StreamSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  stream_init(sm);
  if (warp == 0) {
    const unsigned long long pol = l2_evict_first();
    // a throttle only (stream-level S columns are complete when this kernel
    // starts, by stream order): bounded, so the kernel never depends on the
    // FP64 lane being scheduled beside it
    if (a.wait_flag != nullptr && lane == 0) {
      const unsigned long long t0 = global_ns();
      for (;;) {
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.wait_flag) : "memory");
        if (static_cast<int>(v - a.wait_value) >= 0) break;
        if (global_ns() - t0 > kFlagWaitLimitNs) break;
        __nanosleep(256);
      }
    }
    __syncwarp();
    stream_producer(sm, a.p2s_descs, a.n_p2s_items, a.counter2,
                    [&](unsigned& t, int k, const StreamDesc& e) {
                      for (int c0 = 0; c0 < e.nct; c0 += kSC, ++t) {
                        const int nt = min(kSC, e.nct - c0);
                        stream_put(sm, t,
                                   StageMeta{k, 0, c0, nt, e.aux, e.nrows, c0 + nt == e.nct ? 1 : 0,
                                             e.sbase},
                                   a.W + e.wbase + static_cast<long long>(c0) * kTileDoubles, nt, pol);
                      }
                    });
    return;
  }
  const int cw = warp - 1;
  double acc[kTileRows];
#pragma unroll
  for (int i = 0; i < kTileRows; ++i) acc[i] = 0.0;
  int parity = 0;
  // S columns of this warp's tile, prefetched one stage ahead (S is padded
  // by kSC * kTileCols doubles, engine.cu)
  long long pk = -1;
  int pc = -1;
  double2 spre = make_double2(0.0, 0.0);
  auto sload = [&](long long sb, int c) {
    return __ldg(reinterpret_cast<const double2*>(a.S + sb + static_cast<long long>(c) * kTileCols) + lane);
  };
  for (unsigned t = 0;; ++t) {
    const int s = t % kStages;
    mbar_wait(&sm.full[s], (t / kStages) & 1);
    const StageMeta m = sm.meta[s];
    if (m.k < 0) break;
    if (cw < m.n) {
      const int c = m.ct + cw;
      const double2 sv = (pk == m.k && pc == c) ? spre : sload(m.sb, c);
      if (!m.last) {
        spre = sload(m.sb, c + kSC);
        pk = m.k;
        pc = c + kSC;
      }
      const double2* tl = reinterpret_cast<const double2*>(sm.tile[s] + cw * kTileDoubles);
#pragma unroll
      for (int i = 0; i < kTileRows; ++i) {
        const double2 w = tl[i * (kTileCols / 2) + lane];
        acc[i] = fma(w.y, sv.y, fma(w.x, sv.x, acc[i]));
      }
    }
    if (m.last) {
      double mine = 0.0;
#pragma unroll
      for (int i = 0; i < kTileRows; ++i) {
        const double v = warp_sum(acc[i]);
        if (lane == i) mine = v;
        acc[i] = 0.0;
      }
      if (lane < kTileRows) sm.red[parity][cw][lane] = mine;
      named_bar(1, 32 * kSC);
      if (cw == 0 && lane < m.nrows) {
        double v = sm.red[parity][0][lane];
#pragma unroll
        for (int w = 1; w < kSC; ++w) v += sm.red[parity][w][lane];
        a.lvl_part[m.aux + lane] = v;
      }
      parity ^= 1;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s]);
  }
}

// ---- phase 2, proxy levels, node-major: b_X += K(X, P_A) s_A for the rows of
// node A (up to 256 per item, two per thread), the node's proxy list staged
// in shared memory (proxy_eval2 above; the node's first vcols sources are
// vertex partners). Items of <= 128 / <= 64 rows split the CTA into 2 / 4
// groups that take disjoint parts of every staged chunk (all 256 target
// slots busy on small nodes), partials summed in group order.
template <int K>
__global__ void __launch_bounds__(kProxyThreads, 5) p2_proxy_kernel(const Phase2Args a) {
  __shared__ double2 src[3 * kChunk];
  __shared__ double red[2 * kProxyThreads];
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
    const int vc = a.vcols[g];
    const double4 cen = reinterpret_cast<const double4*>(a.cen)[g];
    const int G = it.nrows <= 64 ? 4 : it.nrows <= 128 ? 2 : 1;
    const int tpg = kProxyThreads / G;  // threads per group
    const int grp = threadIdx.x / tpg, loc = threadIdx.x % tpg;
    const int nt = warp_targets(loc, tpg, it.nrows);
    const double4* P4 = reinterpret_cast<const double4*>(a.p4);
    Tgt tg[2];
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int i = loc + t * tpg;
      const double4 q = i < it.nrows ? P4[a.nt.rowbeg[g] + it.row0 + i] : make_double4(kFar, kFar, kFar, 0.0);
      tg[t] = make_tgt(q.x, q.y, q.z, cen);
    }
    // sources in chunks of kHalfChunk, double-buffered: each thread loads one
    // source of the next chunk into registers before the current chunk's
    // evaluations and stores it after them, one barrier per chunk
    const double4* Q4 = reinterpret_cast<const double4*>(a.q4c) + so;
    const double* Sv = a.S + so;
    double4 nq = make_double4(0.0, 0.0, 0.0, 0.0);
    double nw = 0.0;
    if (threadIdx.x < R) {
      nq = Q4[threadIdx.x];
      nw = Sv[threadIdx.x];
    }
    __syncthreads();  // the previous item is done with both buffers
    if (threadIdx.x < kHalfChunk) {
      double2* d = src + 3 * threadIdx.x;
      d[0] = make_double2(nq.x, nq.y);
      d[1] = make_double2(nq.z, nq.w);
      d[2] = make_double2(nw, 0.0);
    }
    __syncthreads();
    for (int j0 = 0, b = 0; j0 < R; j0 += kHalfChunk, b ^= 1) {
      const int nj = min(kHalfChunk, R - j0);
      const bool more = j0 + kHalfChunk < R;
      const int qn = j0 + kHalfChunk + threadIdx.x;
      if (more && qn < R) {
        nq = Q4[qn];
        nw = Sv[qn];
      }
      const double2* cur = src + 3 * kHalfChunk * b;
      const int sub = (nj + G - 1) / G;
      const int lo = min(nj, grp * sub), hi = min(nj, lo + sub);
      const int jv = max(lo, min(hi, vc - j0));
      proxy_eval2<K>(tg, acc, cur, lo, jv, hi, nt, false);
      if (more && threadIdx.x < kHalfChunk && qn < R) {
        double2* d = src + 3 * kHalfChunk * (b ^ 1) + 3 * threadIdx.x;
        d[0] = make_double2(nq.x, nq.y);
        d[1] = make_double2(nq.z, nq.w);
        d[2] = make_double2(nw, 0.0);
      }
      __syncthreads();
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) red[grp * 2 * tpg + loc + t * tpg] = acc[t][0] + acc[t][1];
    __syncthreads();
    for (int i = threadIdx.x; i < it.nrows; i += kProxyThreads) {
      const int per = 2 * tpg;  // targets per group
      double v = 0.0;
      for (int q = 0; q < G; ++q) v += red[q * per + i];
      a.lvl_part[static_cast<std::int64_t>(it.slot) * a.n_total + a.nt.rowbeg[g] + it.row0 + i] =
          far_scale<K>() * v;
    }
  }
}

// ---- half levels, the regenerated side (planner.h H2Item): one pass per
// row chunk of a node's virtual group evaluates each entry e = K(row, proxy)
// once for both uses: b_row += e t_proxy (t = the partner's streamed
// U'^T x, in S) and v_proxy += e x_row (the partner's phase-2 weight). Same
// evaluation core as p2_proxy_kernel (two targets per thread, box-centred
// sources staged in shared memory); the v sums over the rows go through an
// 8-source warp reduce-scatter (9 shuffles per 8 sources per lane, 2 targets
// each) and a fixed-order sum over the 4 warps. Deterministic.
__device__ __forceinline__ double h2_reduce8(const double (&v)[8], int lane) {
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
  return r;  // the total of source (lane >> 2) & 7
}

constexpr int kH2Warps = kProxyThreads / 32;

template <int K, bool TRICK>
__device__ __forceinline__ void h2_block(const Tgt (&tg)[2], const double (&xw)[2], double (&bacc)[2],
                                         const double2* __restrict__ src, int j0, double* __restrict__ vw,
                                         int lane) {
  double prod[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int jj = j0 + u;
    const double2 s0 = src[3 * jj], s1 = src[3 * jj + 1], s2 = src[3 * jj + 2];
    double p = 0.0;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      double r2;
      if constexpr (TRICK) {
        r2 = fma(tg[t].ax, s0.x, fma(tg[t].ay, s0.y, fma(tg[t].az, s1.x, tg[t].tt + s1.y)));
      } else {
        r2 = sq3(fma(-0.5, tg[t].ax, -s0.x), fma(-0.5, tg[t].ay, -s0.y), fma(-0.5, tg[t].az, -s1.x));
      }
      const double e = far_val<K>(r2);
      bacc[t] = fma(e, s2.x, bacc[t]);
      p = fma(e, xw[t], p);
    }
    prod[u] = p;
  }
  const double v = h2_reduce8(prod, lane);
  if ((lane & 3) == 0) vw[j0 + ((lane >> 2) & 7)] = v;
}

template <int K>
__global__ void __launch_bounds__(kProxyThreads, 4) half2_kernel(const Phase2Args a) {
  __shared__ double2 src[3 * kChunk];
  __shared__ double vw[kH2Warps][kChunk];
  __shared__ double red[2 * kProxyThreads];
  __shared__ long long s_k;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_k = static_cast<long long>(atomicAdd(a.counter_h2, 1u));
    __syncthreads();
    const long long k = s_k;
    if (k >= a.n_h2_items) break;
    const H2Item it = a.h2_items[k];
    const std::int64_t g = it.node;
    const std::int64_t so = a.nt.soff[g];
    const int R = a.nt.rpad[g];
    const int vc = a.vcols[g];
    const double4 cen = reinterpret_cast<const double4*>(a.cen)[g];
    const double4* P4 = reinterpret_cast<const double4*>(a.p4);
    // items of <= 128 / <= 64 rows: G = 2 / 4 thread groups, each covering
    // every row and taking a disjoint share of every staged chunk
    const int G = it.nrows <= 64 ? 4 : it.nrows <= 128 ? 2 : 1;
    const int tpg = kProxyThreads / G, wpg = tpg / 32;
    const int grp = threadIdx.x / tpg, loc = threadIdx.x % tpg;
    Tgt tg[2];
    double xw[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int i = loc + t * tpg;
      const double4 q = i < it.nrows ? P4[a.nt.rowbeg[g] + it.row0 + i] : make_double4(kFar, kFar, kFar, 0.0);
      tg[t] = make_tgt(q.x, q.y, q.z, cen);
      xw[t] = q.w;
    }
    double bacc[2] = {0.0, 0.0};
    for (int j0 = 0; j0 < R; j0 += kChunk) {
      const int nj = min(kChunk, R - j0);
      const int sub = (((nj + G - 1) / G) + 7) & ~7;  // sources per group, whole blocks of 8
      const int lo = min(kChunk, grp * sub), hi = min(kChunk, lo + sub);
      const int nstage = min(kChunk, G * sub);
      __syncthreads();  // the previous chunk's sources and v partials are consumed
      for (int q = threadIdx.x; q < nstage; q += kProxyThreads) {
        if (q < nj) {
          const double4 c4 = reinterpret_cast<const double4*>(a.q4c)[so + j0 + q];
          src[3 * q] = make_double2(c4.x, c4.y);
          src[3 * q + 1] = make_double2(c4.z, c4.w);
          src[3 * q + 2] = make_double2(a.S[so + j0 + q], 0.0);
        } else {  // padding sources: far away (away from the padding rows too), weight 0
          src[3 * q] = make_double2(-kFar, -kFar);
          src[3 * q + 1] = make_double2(-kFar, 3.0 * kFar * kFar);
          src[3 * q + 2] = make_double2(0.0, 0.0);
        }
      }
      __syncthreads();
      // sources [0, vc) of the node (vertex-adjacent partners): difference form
      const int jv = vc - j0;
      for (int jb = lo; jb < hi; jb += 8) {
        if (jb < jv) h2_block<K, false>(tg, xw, bacc, src, jb, vw[warp], lane);
        else h2_block<K, true>(tg, xw, bacc, src, jb, vw[warp], lane);
      }
      __syncthreads();
      // v of the chunk's sources: fixed-order sum over the owning group's warps
      for (int c = threadIdx.x; c < nj; c += kProxyThreads) {
        const int og = c / sub;
        double v = 0.0;
        for (int w = og * wpg; w < (og + 1) * wpg; ++w) v += vw[w][c];
        v *= far_scale<K>();
        if (it.pslot >= 0) {
          a.P[it.pslot + j0 + c] = v;
        } else {
          const std::int32_t dst = a.spos[so + j0 + c];
          if (dst >= 0) a.Sw[dst] = v;
        }
      }
    }
    if (it.slot >= 0) {
#pragma unroll
      for (int t = 0; t < 2; ++t) red[grp * 2 * tpg + loc + t * tpg] = bacc[t];
      __syncthreads();
      for (int i = threadIdx.x; i < it.nrows; i += kProxyThreads) {
        const int per = 2 * tpg;
        double v = 0.0;
        for (int q = 0; q < G; ++q) v += red[q * per + i];
        a.lvl_part[static_cast<std::int64_t>(it.slot) * a.n_total + a.nt.rowbeg[g] + it.row0 + i] =
            far_scale<K>() * v;
      }
    }
  }
}

__global__ void combine_kernel(const double* __restrict__ cpart, const double* __restrict__ lvl,
                               int n_lvl, std::int64_t n_total, const std::int64_t* __restrict__ leaf_off,
                               std::int64_t leaf0, std::int64_t nleaves,
                               const std::int32_t* __restrict__ in_off,
                               const std::int64_t* __restrict__ in_pos,
                               const double* __restrict__ pairbuf,
                               const std::int32_t* __restrict__ perm, double* __restrict__ b,
                               double* __restrict__ bm) {
  const std::int64_t t = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nleaves) return;
  const std::int64_t X = leaf0 + t;
  const std::int64_t xb = leaf_off[X];
  const int m = static_cast<int>(leaf_off[X + 1] - xb);
  const int i0 = in_off ? in_off[X] : 0, i1 = in_off ? in_off[X + 1] : 0;
  for (int i = lane; i < m; i += 32) {
    const std::int64_t p = xb + i;
    double v = cpart[p];
    for (int e = i0; e < i1; ++e) v += pairbuf[in_pos[e] + i];
    for (int l = 0; l < n_lvl; ++l) v += lvl[static_cast<std::int64_t>(l) * n_total + p];
    b[perm[p]] = v;
    if (bm) bm[p] = v;  // Morton copy for the all-gather of b
  }
}

// Build-time pass over every owned leaf's dense sources in its symmetric
// list order (self | dense one-way | dense sym; planner.cpp): the reference
// forms all dense leaf blocks during initialize (hmatrix.cpp:124-147), so
// coincident points raise DegenerateGeometryError here. With NF set (stored
// near field, planner.h set_near_storage) it stores, row-major per leaf,
// exactly the value the matrix-free near pass computes for each (row,
// stored source) from the same packed points: diag on the self block's
// diagonal, kernel_r2_fast of the same sq3 operands for dense sources, the
// Newton-form far_acc value for direct (leaf-level admissible) ones.
template <int K>
__global__ void __launch_bounds__(kThreads) near_store_kernel(const Phase2Args a, double* __restrict__ NF,
                                                              unsigned* flags) {
  __shared__ long long rs[kMaxNearRanges];
  __shared__ int rpre[kMaxNearRanges + 1];   // visited-column prefix
  __shared__ int rsto[kMaxNearRanges];       // stored-column prefix (-1: not stored)
  __shared__ unsigned char rdir[kMaxNearRanges];
  __shared__ int nr;
  const std::int64_t X = a.leaf0 + blockIdx.x;
  const std::int64_t xb = a.leaf_off[X];
  const int m = static_cast<int>(a.leaf_off[X + 1] - xb);
  if (m == 0) return;
  const std::int32_t nb = a.sym_off[X];
  const int mask = NF ? a.nf_mask : 0;
  if (threadIdx.x == 0) {
    const int c[4] = {a.sym_cnt[4 * X], a.sym_cnt[4 * X + 1], a.sym_cnt[4 * X + 2], a.sym_cnt[4 * X + 3]};
    int n = 0, pre = 0, sto = 0;
    // every dense source (the coincident-point scan) and, when stored, the
    // direct ones, in symmetric-list order: self, dense one-way, direct
    // one-way, dense sym, direct sym
    auto add = [&](std::int32_t e, bool direct) {
      const bool stored = (mask & (direct ? 2 : 1)) != 0;
      if (direct && !stored) return;
      const std::int32_t Y = a.sym_ids[nb + e];
      const int len = static_cast<int>(a.leaf_off[Y + 1] - a.leaf_off[Y]);
      rs[n] = a.leaf_off[Y];
      rpre[n] = pre;
      rsto[n] = stored ? sto : -1;
      rdir[n] = direct ? 1 : 0;
      pre += len;
      if (stored) sto += len;
      ++n;
    };
    add(0, false);  // self
    int e = 1;
    for (int k = 0; k < 4; ++k)
      for (int q = 0; q < c[k]; ++q, ++e) add(e, (k & 1) != 0);
    rpre[n] = pre;
    nr = n;
  }
  __syncthreads();
  const int nvis = rpre[nr];
  const int nds = NF ? a.nf_cols[X] : 0;
  const double4* P4 = reinterpret_cast<const double4*>(a.p4);
  unsigned f = 0;
  for (long long q = threadIdx.x; q < static_cast<long long>(m) * nvis; q += blockDim.x) {
    const int i = static_cast<int>(q / nvis), d = static_cast<int>(q % nvis);
    int lo = 0;
    while (lo + 1 < nr && rpre[lo + 1] <= d) ++lo;
    const double4 t = P4[xb + i];
    const double4 sp = P4[rs[lo] + (d - rpre[lo])];
    double v;
    if (lo == 0 && d == i) {
      v = a.diag;
    } else {
      const double r2 = sq3(t.x - sp.x, t.y - sp.y, t.z - sp.z);
      if (r2 < kCoincidentTol2) f |= kFlagDegenGeom;
      // the values the matrix-free pass evaluates: full accuracy for the
      // dense blocks, the Newton form for the direct (admissible) ones
      v = rdir[lo] ? far_acc<K>(r2, 1.0, 0.0) : kernel_r2_fast<K>(r2);
    }
    if (NF && rsto[lo] >= 0) NF[a.nf_off[X] + static_cast<long long>(i) * nds + rsto[lo] + (d - rpre[lo])] = v;
  }
  if (f) atomicOr(flags, f);
}

template <class F>
int grid_for(F kernel, int sms, int per_sm, std::int64_t work, int threads = kThreads) {
  int nb = 0;
  H3D_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, 0));
  if (std::getenv("H3D_DEBUG_GRID")) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kernel);
    std::fprintf(stderr, "grid_for: threads %d regs %d smem %zu occ %d per_sm %d\n", threads, fa.numRegs,
                 fa.sharedSizeBytes, nb, per_sm);
  }
  const std::int64_t g = static_cast<std::int64_t>(sms) * std::max(1, std::min(nb, per_sm));
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(g, work)));
}

}  // namespace

void configure_kernels();

void launch_gather(const double* x, const std::int32_t* perm, std::int64_t n, double* xp, double* p4,
                   cudaStream_t s) {
  if (n <= 0) return;
  gather_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(x, perm, n, xp, p4);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_pack_w(const double* xp, std::int64_t n, double* p4, cudaStream_t s) {
  if (n <= 0) return;
  pack_w_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(xp, n, p4);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_pack_points(const double* px, const double* py, const double* pz, std::int64_t n,
                        double* p4, cudaStream_t s) {
  if (n <= 0) return;
  pack_points_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
      px, py, pz, n, reinterpret_cast<double4*>(p4));
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_p2_near(const Phase2Args& a, int sms, int per_sm, cudaStream_t s) {
  if (a.nleaves == 0) return;
  configure_kernels();
  const bool stored = a.NF != nullptr;
#define H3D_P2N(KK)                                                                          \
  if (stored) {                                                                              \
    const int grid = grid_for(p2_near_kernel<KK, true>, sms, per_sm, a.nleaves, kNearThreads); \
    p2_near_kernel<KK, true><<<grid, kNearThreads, 0, s>>>(a);                              \
  } else {                                                                                   \
    const int grid = grid_for(p2_near_kernel<KK, false>, sms, per_sm, a.nleaves, kNearThreads); \
    p2_near_kernel<KK, false><<<grid, kNearThreads, 0, s>>>(a);                             \
  }
  switch (a.kernel) {
    case kLaplace: H3D_P2N(kLaplace); break;
    case kR4: H3D_P2N(kR4); break;
    default: H3D_P2N(kHelmholtz); break;
  }
#undef H3D_P2N
  H3D_CUDA_CHECK(cudaGetLastError());
}

// Once per process: the bulk-copy kernels' dynamic shared memory, and one
// shared-heavy carveout for every matvec kernel - the HBM lane's CTA
// (~130 KB) and the FP64 kernels co-reside on each SM, so they must agree on
// the SM's L1/shared split.
void configure_kernels() {
  static PerDeviceOnce once;
  once([] {
    H3D_CUDA_CHECK(cudaFuncSetAttribute(p1_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sizeof(StreamSmem))));
    H3D_CUDA_CHECK(cudaFuncSetAttribute(p2_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sizeof(StreamSmem))));
    H3D_CUDA_CHECK(cudaFuncSetAttribute(proxy_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sizeof(SolveSmem))));
    const void* fs[] = {
        reinterpret_cast<const void*>(p1_stream_kernel),
        reinterpret_cast<const void*>(p2_stream_kernel),
        reinterpret_cast<const void*>(p1_proxy_kernel<kLaplace>),
        reinterpret_cast<const void*>(p1_proxy_kernel<kR4>),
        reinterpret_cast<const void*>(p1_proxy_kernel<kHelmholtz>),
        reinterpret_cast<const void*>(p2_proxy_kernel<kLaplace>),
        reinterpret_cast<const void*>(p2_proxy_kernel<kR4>),
        reinterpret_cast<const void*>(p2_proxy_kernel<kHelmholtz>),
        reinterpret_cast<const void*>(p2_near_kernel<kLaplace, false>),
        reinterpret_cast<const void*>(p2_near_kernel<kR4, false>),
        reinterpret_cast<const void*>(p2_near_kernel<kHelmholtz, false>),
        reinterpret_cast<const void*>(p2_near_kernel<kLaplace, true>),
        reinterpret_cast<const void*>(p2_near_kernel<kR4, true>),
        reinterpret_cast<const void*>(p2_near_kernel<kHelmholtz, true>),
        reinterpret_cast<const void*>(proxy_solve_kernel),
    };
    for (const void* f : fs)
      H3D_CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          cudaSharedmemCarveoutMaxShared));
  });
}

template <class F>
int stream_grid(F kernel, int sms, int per_sm, std::int64_t work) {
  configure_kernels();
  int nb = 0;
  H3D_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kStreamThreads,
                                                               sizeof(StreamSmem)));
  const std::int64_t g = static_cast<std::int64_t>(sms) * std::max(1, std::min(nb, per_sm));
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(g, work)));
}

void launch_p1_stream(const P1Args& a, int sms, int per_sm, cudaStream_t s) {
  if (a.nitems == 0) return;
  const int grid = stream_grid(p1_stream_kernel, sms, per_sm, a.nitems);
  p1_stream_kernel<<<grid, kStreamThreads, sizeof(StreamSmem), s>>>(a);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_p1_proxy(const P1Args& a, int kernel, int sms, int per_sm, cudaStream_t s) {
  if (a.nitems == 0) return;
  configure_kernels();
  switch (kernel) {
    case kLaplace: {
      const int grid = grid_for(p1_proxy_kernel<kLaplace>, sms, per_sm, a.nitems, kProxyThreads);
      p1_proxy_kernel<kLaplace><<<grid, kProxyThreads, 0, s>>>(a);
      break;
    }
    case kR4: {
      const int grid = grid_for(p1_proxy_kernel<kR4>, sms, per_sm, a.nitems, kProxyThreads);
      p1_proxy_kernel<kR4><<<grid, kProxyThreads, 0, s>>>(a);
      break;
    }
    default: {
      const int grid = grid_for(p1_proxy_kernel<kHelmholtz>, sms, per_sm, a.nitems, kProxyThreads);
      p1_proxy_kernel<kHelmholtz><<<grid, kProxyThreads, 0, s>>>(a);
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

__global__ void fill_far_kernel(double4* __restrict__ q4, std::int64_t n, double w) {
  const std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) q4[i] = make_double4(kFar, kFar, kFar, w);
}

void launch_fill_far(double* q4, std::int64_t n, bool centred, cudaStream_t s) {
  if (n <= 0) return;
  // centred records carry |s'|^2 in w: a padding slot must keep r^2 > 0 in
  // the tt + ss - 2 t'.s' form (its weight, in the other array, is 0)
  fill_far_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
      reinterpret_cast<double4*>(q4), n, centred ? 3.0 * kFar * kFar : 0.0);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_proxy_gather(const ProxySeg* segs, std::int64_t nseg, const std::int32_t* piv,
                         const double* px, const double* py, const double* pz, const double* cen,
                         double* q4, double* q4c, cudaStream_t s) {
  if (nseg == 0) return;
  const dim3 block(32, 8);
  proxy_gather_kernel<<<static_cast<unsigned>((nseg + 7) / 8), block, 0, s>>>(segs, nseg, piv, px, py,
                                                                            pz, reinterpret_cast<const double4*>(cen), reinterpret_cast<double4*>(q4),
      reinterpret_cast<double4*>(q4c));
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_lu_invert(const ProxySeg* segs, std::int64_t nseg, double* lu, std::int64_t lu_total,
                      int max_r, cudaStream_t s) {
  if (nseg == 0 || max_r == 0) return;
  // scratch for a batch of column-major inverses
  const std::int64_t batch = std::max<std::int64_t>(1, std::min<std::int64_t>(
      nseg, (std::int64_t(1) << 29) / (static_cast<std::int64_t>(max_r) * max_r * 8)));
  double* scratch = nullptr;
  H3D_CUDA_CHECK(cudaMallocAsync(&scratch, batch * max_r * max_r * 8, s));
  for (std::int64_t b0 = 0; b0 < nseg; b0 += batch) {
    const std::int64_t nb = std::min(batch, nseg - b0);
    lu_invert_kernel<<<static_cast<unsigned>(nb), 128, 0, s>>>(segs + b0, nb, lu, lu_total, scratch,
                                                              max_r);
    H3D_CUDA_CHECK(cudaGetLastError());
  }
  H3D_CUDA_CHECK(cudaFreeAsync(scratch, s));
}

void launch_proxy_solve(const ProxySeg* segs, std::int64_t nseg, const double* lu, std::int64_t lu_total,
                        double* S, int sms, int per_sm, unsigned* counter, cudaStream_t s) {
  if (nseg == 0) return;
  configure_kernels();
  int nb = 0;
  H3D_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, proxy_solve_kernel, 32 * kSolveWarps,
                                                               sizeof(SolveSmem)));
  const std::int64_t want = (nseg + kSolveWarps - 1) / kSolveWarps;
  const int grid = static_cast<int>(std::max<std::int64_t>(
      1, std::min<std::int64_t>(want, static_cast<std::int64_t>(sms) * std::max(1, std::min(nb, per_sm)))));
  proxy_solve_kernel<<<grid, 32 * kSolveWarps, sizeof(SolveSmem), s>>>(segs, nseg, lu, lu_total, S, counter);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_half2(const Phase2Args& a, int sms, int per_sm, cudaStream_t s) {
  if (a.n_h2_items == 0) return;
  configure_kernels();
  switch (a.kernel) {
    case kLaplace: {
      const int grid = grid_for(half2_kernel<kLaplace>, sms, per_sm, a.n_h2_items, kProxyThreads);
      half2_kernel<kLaplace><<<grid, kProxyThreads, 0, s>>>(a);
      break;
    }
    case kR4: {
      const int grid = grid_for(half2_kernel<kR4>, sms, per_sm, a.n_h2_items, kProxyThreads);
      half2_kernel<kR4><<<grid, kProxyThreads, 0, s>>>(a);
      break;
    }
    default: {
      const int grid = grid_for(half2_kernel<kHelmholtz>, sms, per_sm, a.n_h2_items, kProxyThreads);
      half2_kernel<kHelmholtz><<<grid, kProxyThreads, 0, s>>>(a);
      break;
    }
  }
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_p2_stream(const Phase2Args& a, int sms, int per_sm, cudaStream_t s) {
  if (a.n_p2s_items == 0) return;
  const int grid = stream_grid(p2_stream_kernel, sms, per_sm, a.n_p2s_items);
  p2_stream_kernel<<<grid, kStreamThreads, sizeof(StreamSmem), s>>>(a);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_p2_proxy(const Phase2Args& a, int sms, int per_sm, cudaStream_t s) {
  if (a.n_p2_items == 0) return;
  configure_kernels();
  switch (a.kernel) {
    case kLaplace: {
      const int grid = grid_for(p2_proxy_kernel<kLaplace>, sms, per_sm, a.n_p2_items, kProxyThreads);
      p2_proxy_kernel<kLaplace><<<grid, kProxyThreads, 0, s>>>(a);
      break;
    }
    case kR4: {
      const int grid = grid_for(p2_proxy_kernel<kR4>, sms, per_sm, a.n_p2_items, kProxyThreads);
      p2_proxy_kernel<kR4><<<grid, kProxyThreads, 0, s>>>(a);
      break;
    }
    default: {
      const int grid = grid_for(p2_proxy_kernel<kHelmholtz>, sms, per_sm, a.n_p2_items, kProxyThreads);
      p2_proxy_kernel<kHelmholtz><<<grid, kProxyThreads, 0, s>>>(a);
      break;
    }
  }
  H3D_CUDA_CHECK(cudaGetLastError());
}

__global__ void set_flag_kernel(unsigned* flag, unsigned value) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

void launch_set_flag(unsigned* flag, unsigned value, cudaStream_t s) {
  set_flag_kernel<<<1, 1, 0, s>>>(flag, value);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_combine(const double* cpart, const double* lvl_part, int n_lvl, std::int64_t n_total,
                    const std::int64_t* leaf_off, std::int64_t leaf0, std::int64_t nleaves,
                    const std::int32_t* in_off, const std::int64_t* in_pos, const double* pairbuf,
                    const std::int32_t* perm, double* b, double* bm, cudaStream_t s) {
  if (nleaves <= 0) return;
  const std::int64_t threads = nleaves * 32;
  combine_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(
      cpart, lvl_part, n_lvl, n_total, leaf_off, leaf0, nleaves, in_off, in_pos, pairbuf, perm, b, bm);
  H3D_CUDA_CHECK(cudaGetLastError());
}

// rows outside [row0, row1) of the all-gathered Morton-order b to the
// original order (the owned rows were written by combine)
__global__ void unpermute_rest_kernel(const double* __restrict__ bm, const std::int32_t* __restrict__ perm,
                                      std::int64_t n, std::int64_t row0, std::int64_t row1,
                                      double* __restrict__ b) {
  for (std::int64_t p = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    if (p < row0 || p >= row1) b[perm[p]] = bm[p];
}

void launch_unpermute_rest(const double* bm, const std::int32_t* perm, std::int64_t n, std::int64_t row0,
                           std::int64_t row1, double* b, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(std::min<std::int64_t>((n + 255) / 256, 148 * 8));
  unpermute_rest_kernel<<<grid, 256, 0, s>>>(bm, perm, n, row0, row1, b);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_near_scan(const Phase2Args& a, double* NF_out, unsigned* flags, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(a.nleaves);
  if (grid == 0) return;
  switch (a.kernel) {
    case kLaplace: near_store_kernel<kLaplace><<<grid, kThreads, 0, s>>>(a, NF_out, flags); break;
    case kR4: near_store_kernel<kR4><<<grid, kThreads, 0, s>>>(a, NF_out, flags); break;
    default: near_store_kernel<kHelmholtz><<<grid, kThreads, 0, s>>>(a, NF_out, flags); break;
  }
  H3D_CUDA_CHECK(cudaGetLastError());
}

}  // namespace h3db
