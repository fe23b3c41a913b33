// Interaction lists on the device, one thread per (level, node), for the
// three variants of the reference (octree.cpp:197-260).
//
// The reference's candidate set for node m at level l is the 7 siblings plus
// the children of parent.near_edge and parent.near_face (HODLR3D) or of
// parent.near_edge, near_face and near_vertex (H-strong), sorted ascending,
// then classified: well-separated -> inter; vertex -> inter (HODLR3D) or
// near_vertex (H-strong); edge -> near_edge; face -> near_face. HODLR puts
// every sibling in inter. By induction the parent's near lists are exactly
// its in-bounds same-level neighbours with 1..2 (HODLR3D) or 1..3 (H-strong)
// nonzero offset components, so the candidate set is generated here
// geometrically and in ascending Morton order: the parent neighbourhood
// (parent included: its children are the siblings) sorted by Morton id, then
// children 8q..8q+7 of each q. Output is bit-identical to the reference
// (tests/test_gpu_parity.py, golden lists per variant).
#include "common.cuh"
#include "kernels.h"

namespace h3db {

namespace {

__device__ __forceinline__ int interleave(int ix, int iy, int iz, int level) {
  int code = 0;
  for (int b = 0; b < level; ++b) {
    code |= ((ix >> b) & 1) << (3 * b);
    code |= ((iy >> b) & 1) << (3 * b + 1);
    code |= ((iz >> b) & 1) << (3 * b + 2);
  }
  return code;
}

__device__ __forceinline__ void deinterleave(int code, int level, int& ix, int& iy, int& iz) {
  ix = iy = iz = 0;
  for (int b = 0; b < level; ++b) {
    ix |= ((code >> (3 * b)) & 1) << b;
    iy |= ((code >> (3 * b + 1)) & 1) << b;
    iz |= ((code >> (3 * b + 2)) & 1) << b;
  }
}

// classify_offset (octree.hpp:27-37) folded to list kind per variant:
// -1 self, 0 inter, 1 near_edge, 2 near_face, 3 near_vertex (H-strong).
__device__ __forceinline__ int list_kind(int dx, int dy, int dz, int variant) {
  const int ax = abs(dx), ay = abs(dy), az = abs(dz);
  if ((ax | ay | az) == 0) return -1;
  if (variant == kVariantHodlr) return 0;
  if (ax >= 2 || ay >= 2 || az >= 2) return 0;
  const int nz = (ax != 0) + (ay != 0) + (az != 0);
  return nz == 1 ? 2 : nz == 2 ? 1 : variant == kVariantHStrong ? 3 : 0;
}

// Visit the ascending candidate list of node m at level l; f(cand, kind).
template <class F>
__device__ __forceinline__ void for_each_candidate(int level, int m, int variant, F&& f) {
  int mx, my, mz;
  deinterleave(m, level, mx, my, mz);
  const int par = m >> 3;
  const int pl = level - 1;
  const int pside = 1 << pl;
  int px, py, pz;
  deinterleave(par, pl, px, py, pz);
  // parent neighbourhood: offsets with at most this many nonzero components
  const int max_nz = variant == kVariantHodlr ? 0 : variant == kVariantHStrong ? 3 : 2;
  int q[27];
  int nq = 0;
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dz = -1; dz <= 1; ++dz) {
        const int nz = (dx != 0) + (dy != 0) + (dz != 0);
        if (nz > max_nz) continue;
        const int ax = px + dx, ay = py + dy, az = pz + dz;
        if (ax < 0 || ay < 0 || az < 0 || ax >= pside || ay >= pside || az >= pside) continue;
        q[nq++] = interleave(ax, ay, az, pl);
      }
  // insertion sort (<= 27 entries)
  for (int i = 1; i < nq; ++i) {
    const int v = q[i];
    int j = i - 1;
    while (j >= 0 && q[j] > v) {
      q[j + 1] = q[j];
      --j;
    }
    q[j + 1] = v;
  }
  for (int t = 0; t < nq; ++t) {
    int qx, qy, qz;
    deinterleave(q[t], pl, qx, qy, qz);
    for (int c = 0; c < 8; ++c) {
      const int cand = 8 * q[t] + c;
      const int cx = 2 * qx + (c & 1), cy = 2 * qy + ((c >> 1) & 1), cz = 2 * qz + ((c >> 2) & 1);
      const int k = list_kind(cx - mx, cy - my, cz - mz, variant);
      if (k >= 0) f(cand, k);
    }
  }
}

__global__ void list_count_kernel(int level, int count, int variant, std::int32_t* __restrict__ counts) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= count) return;
  int c[kListKinds] = {0, 0, 0, 0};
  for_each_candidate(level, m, variant, [&](int, int k) { ++c[k]; });
  for (int k = 0; k < kListKinds; ++k) counts[k * (count + 1) + m] = c[k];
}

struct ListIds {
  std::int32_t* p[kListKinds];
};

__global__ void list_fill_kernel(int level, int count, int variant, const std::int32_t* __restrict__ offsets,
                                 ListIds ids) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= count) return;
  std::int32_t pos[kListKinds];
  for (int k = 0; k < kListKinds; ++k) pos[k] = offsets[k * (count + 1) + m];
  for_each_candidate(level, m, variant, [&](int cand, int k) { ids.p[k][pos[k]++] = cand; });
}

}  // namespace

// counts layout: kListKinds consecutive arrays of (8^l + 1) int32 (last entry 0)
void launch_list_counts(int level, int variant, std::int32_t* counts, cudaStream_t s) {
  const int count = 1 << (3 * level);
  list_count_kernel<<<(count + 127) / 128, 128, 0, s>>>(level, count, variant, counts);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_list_fill(int level, int variant, const std::int32_t* offsets, std::int32_t* const* ids,
                      cudaStream_t s) {
  const int count = 1 << (3 * level);
  ListIds li;
  for (int k = 0; k < kListKinds; ++k) li.p[k] = ids[k];
  list_fill_kernel<<<(count + 127) / 128, 128, 0, s>>>(level, count, variant, offsets, li);
  H3D_CUDA_CHECK(cudaGetLastError());
}

}  // namespace h3db
