// Host planning (see planner.h). Reference mapping:
//   build_pairs  <- the per-level ACA job list of initialize (hmatrix.cpp:74-98),
//                   halved to unordered pairs X < Y (lists swap-symmetric,
//                   test_octree.cpp:167-181; kernels symmetric, kernel.cpp:7-21)
//   near lists   <- the dense leaf block list (hmatrix.cpp:105-120): self, edge,
//                   face, vertex (H-strong)
//   ownership    <- Morton-subtree analogue of plan_partition (parallel.cpp:34-74)
#include "planner.h"

#include <algorithm>

namespace h3db {

namespace {
// Morton ids at one level (bit b of ix / iy / iz -> bit 3b / 3b+1 / 3b+2,
// reference octree.cpp:30-38): Chebyshev distance 1 between distinct boxes
// every third bit (0, 3, 6, ...) of a 63-bit Morton id, compacted
inline std::int64_t compact3(std::uint64_t x) {
  x &= 0x1249249249249249ULL;
  x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ULL;
  x = (x ^ (x >> 4)) & 0x100f00f00f00f00fULL;
  x = (x ^ (x >> 8)) & 0x1f0000ff0000ffULL;
  x = (x ^ (x >> 16)) & 0x1f00000000ffffULL;
  x = (x ^ (x >> 32)) & 0x1fffffULL;
  return static_cast<std::int64_t>(x);
}
bool vertex_adjacent(std::int64_t a, std::int64_t b) {
  std::int64_t d = 0;
  for (int dim = 0; dim < 3; ++dim) {
    const std::int64_t ca = compact3(static_cast<std::uint64_t>(a) >> dim);
    const std::int64_t cb = compact3(static_cast<std::uint64_t>(b) >> dim);
    d = std::max<std::int64_t>(d, ca > cb ? ca - cb : cb - ca);
  }
  return d == 1;
}
}  // namespace

bool boxes_touch(std::int64_t a, std::int64_t b) { return vertex_adjacent(a, b); }

namespace {
constexpr std::int64_t kRowChunk = 2048;  // phase-1 stream: rows per item
static_assert(kRowChunk % kTileRows == 0, "phase-1 stream items start on a row tile");
constexpr int kColChunk = 256;            // phase-1: columns (targets) per item
constexpr std::int64_t kSrcChunk = 2048;  // phase-1 proxy: source points per item
}  // namespace

std::vector<int> default_modes(int depth, std::int64_t n, int policy) {
  std::vector<int> m(depth + 1, kModeStream);
  if (policy == 0 || depth == 0) return m;  // all streamed
  // policy 1 (hybrid): leaf level exact, then alternate compute/stream so the
  // FP64 pipes and HBM work concurrently (cost model: DESIGN.md section 4).
  m[depth] = kModeDirect;
  for (int l = 1; l < depth; ++l) m[l] = kModeProxy;
  (void)n;
  return m;
}

Planner::Planner(int depth, std::int64_t n, std::vector<std::vector<std::int64_t>> off,
                 std::vector<LevelLists> lists, int rank, int world, std::vector<int> modes)
    : L_(depth), n_(n), off_(std::move(off)), lists_(std::move(lists)), rank_(rank),
      world_(world), mode_(std::move(modes)) {
  if (static_cast<int>(off_.size()) != L_ + 1 || static_cast<int>(lists_.size()) != L_ + 1)
    throw std::invalid_argument("planner: offsets/lists do not match the depth");
  if (!(world_ == 1 || world_ == 2 || world_ == 4 || world_ == 8))
    throw std::invalid_argument("planner: shard_world must be 1, 2, 4 or 8");
  if (rank_ < 0 || rank_ >= world_) throw std::invalid_argument("planner: shard_rank out of range");
  if (static_cast<int>(mode_.size()) != L_ + 1) mode_.assign(L_ + 1, kModeStream);
  for (int l = 1; l <= L_; ++l) {
    if (mode_[l] < 0 || mode_[l] > kModeLast) throw std::invalid_argument("planner: bad level mode");
    if (mode_[l] == kModeDirect && l != L_)
      throw std::invalid_argument("planner: direct mode is only valid at the leaf level");
  }
  oct0_ = 8 * rank_ / world_;
  oct1_ = 8 * (rank_ + 1) / world_;
  node_base_.assign(L_ + 2, 0);
  for (int l = 0; l <= L_; ++l) node_base_[l + 1] = node_base_[l] + (1LL << (3 * l));
  if (L_ == 0) {
    row0 = 0;
    row1 = rank_ == 0 ? n_ : 0;
  } else {
    row0 = off_[1][oct0_];
    row1 = off_[1][oct1_];
  }
  if (L_ == 0) {
    leaf0 = 0;
    leaf1 = rank_ == 0 ? 1 : 0;
  } else {
    leaf0 = static_cast<std::int64_t>(oct0_) << (3 * (L_ - 1));
    leaf1 = static_cast<std::int64_t>(oct1_) << (3 * (L_ - 1));
  }
  rank_row0.resize(world_);
  rank_row1.resize(world_);
  for (int r = 0; r < world_; ++r) {
    if (L_ == 0) {
      rank_row0[r] = 0;
      rank_row1[r] = r == 0 ? n_ : 0;
    } else {
      rank_row0[r] = off_[1][8 * r / world_];
      rank_row1[r] = off_[1][8 * (r + 1) / world_];
    }
  }
  build_pairs();
}

bool Planner::owned(int level, std::int64_t m) const {
  if (level == 0) return rank_ == 0;
  const std::int64_t oct = m >> (3 * (level - 1));
  return oct >= oct0_ && oct < oct1_;
}

// Admissible blocks with both nodes non-empty (hmatrix.cpp:74-98); one ACA per
// unordered pair X < Y, on every shard that owns X or Y (cross pairs are
// compressed redundantly, like the reference's shared nodes, parallel.cpp:308-380).
void Planner::build_pairs() {
  pairs_.assign(L_ + 1, LevelPairs{});
  entry_pair_.assign(L_ + 1, {});
  entry_col_.assign(L_ + 1, {});
  sizes.nblocks_ordered = 0;
  for (int l = 1; l <= L_; ++l) {
    const std::int64_t cnt = 1LL << (3 * l);
    const auto& off = lists_[l].off[0];
    const auto& ids = lists_[l].ids[0];
    auto& ep = entry_pair_[l];
    ep.assign(ids.size(), -1);
    auto& P = pairs_[l];
    for (std::int64_t X = 0; X < cnt; ++X) {
      if (node_size(l, X) == 0) continue;
      for (std::int32_t e = off[X]; e < off[X + 1]; ++e) {
        const std::int32_t Y = ids[e];
        if (node_size(l, Y) == 0) continue;
        ++sizes.nblocks_ordered;
        if (mode_[l] == kModeDirect) continue;
        if (Y <= X || !(owned(l, X) || owned(l, Y))) continue;
        ep[e] = static_cast<std::int32_t>(P.X.size());
        P.X.push_back(static_cast<std::int32_t>(X));
        P.Y.push_back(Y);
        P.eX.push_back(e);
        const int m = static_cast<int>(node_size(l, X)), nn = static_cast<int>(node_size(l, Y));
        P.max_m = std::max(P.max_m, m);
        P.max_n = std::max(P.max_n, nn);
        P.max_mn = std::max(P.max_mn, std::min(m, nn));
      }
    }
    P.eY.assign(P.X.size(), -1);
    for (std::int64_t Z = 0; Z < cnt; ++Z) {
      if (node_size(l, Z) == 0) continue;
      for (std::int32_t e = off[Z]; e < off[Z + 1]; ++e) {
        const std::int32_t k = ids[e];
        if (k >= Z || node_size(l, k) == 0 || mode_[l] == kModeDirect ||
            !(owned(l, Z) || owned(l, k)))
          continue;
        const auto b = ids.begin() + off[k], en = ids.begin() + off[k + 1];
        const auto it = std::lower_bound(b, en, static_cast<std::int32_t>(Z));
        if (it == en || *it != Z) throw std::logic_error("interaction lists not swap-symmetric");
        const std::int32_t p = ep[static_cast<std::size_t>(it - ids.begin())];
        ep[e] = p;
        P.eY[p] = e;
      }
    }
    P.rank.assign(P.X.size(), 0);
    const double mbar = static_cast<double>(n_) / static_cast<double>(cnt);
    P.threads = mbar <= 64 ? 32 : mbar <= 2048 ? 128 : mbar <= 8192 ? 256 : 512;
  }
  sizes.npairs = 0;
  for (const auto& P : pairs_) sizes.npairs += static_cast<std::int64_t>(P.X.size());
}

void Planner::layout() {
  // half levels: a second (virtual) node id per node for its regenerated
  // column group
  std::int64_t T = total_nodes();
  vbase.assign(L_ + 1, -1);
  for (int l = 1; l <= L_; ++l)
    if (two_groups(mode_[l])) {
      vbase[l] = T;
      T += 1LL << (3 * l);
    }
  woff.assign(T, 0);
  soff.assign(T, 0);
  rowbeg.assign(T, 0);
  rpad.assign(T, 0);
  rows.assign(T, 0);
  vcols.assign(T, 0);
  p1a.assign(T, 0);
  p1b.assign(T, 0);
  p1c.assign(T, 0);
  center.assign(4 * T, 0.0);
  for (int l = 0; l <= L_; ++l) {
    const std::int64_t cnt = 1LL << (3 * l);
    const double w = 2.0 / static_cast<double>(1LL << l);
    for (std::int64_t z = 0; z < cnt; ++z) {
      std::int64_t c[3] = {0, 0, 0};
      for (int b = 0; b < l; ++b)
        for (int d = 0; d < 3; ++d) c[d] |= ((z >> (3 * b + d)) & 1) << b;
      for (int d = 0; d < 3; ++d) {
        center[4 * gid(l, z) + d] = -1.0 + (static_cast<double>(c[d]) + 0.5) * w;
        if (vbase[l] >= 0) center[4 * gv(l, z) + d] = center[4 * gid(l, z) + d];
      }
    }
  }
  for (int l = 0; l <= L_; ++l) {
    const std::int64_t cnt = 1LL << (3 * l);
    for (std::int64_t z = 0; z < cnt; ++z) {
      rowbeg[gid(l, z)] = off_[l][z];
      rows[gid(l, z)] = static_cast<std::int32_t>(node_size(l, z));
      if (vbase[l] >= 0) {
        rowbeg[gv(l, z)] = off_[l][z];
        rows[gv(l, z)] = static_cast<std::int32_t>(node_size(l, z));
      }
    }
  }
  PlanSizes& S = sizes;
  S.w_doubles = S.s_doubles = S.piv_total = S.lu_total = 0;
  S.factor_doubles = S.proxy_units = S.half_units = S.sum_rank = 0;
  S.max_rank = 0;
  S.ref_float_count = S.ref_int_count = 0;
  pair_wx.assign(L_ + 1, {});
  pair_wy.assign(L_ + 1, {});
  pair_rx.assign(L_ + 1, {});
  pair_ry.assign(L_ + 1, {});
  pair_cx.assign(L_ + 1, {});
  pair_cy.assign(L_ + 1, {});
  pair_piv.assign(L_ + 1, {});
  pair_lu.assign(L_ + 1, {});
  std::vector<std::int8_t> grp;
  for (int l = 1; l <= L_; ++l) {
    const auto& P = pairs_[l];
    const std::int64_t cnt = 1LL << (3 * l);
    for (std::size_t p = 0; p < P.X.size(); ++p) {
      const std::int64_t r = P.rank[p];
      const std::int64_t units = r * (node_size(l, P.X[p]) + node_size(l, P.Y[p]));
      S.sum_rank += r;
      if (mode_[l] == kModeStream || mode_[l] == kModePair) {
        S.factor_doubles += units;
      } else if (mode_[l] == kModeHalf) {  // U' streamed, the Y side regenerated
        S.factor_doubles += r * node_size(l, P.X[p]);
        S.proxy_units += r * node_size(l, P.Y[p]);
        S.half_units += r * node_size(l, P.Y[p]);
      } else if (mode_[l] == kModeSplit) {  // X side twice, Y side once (two-use pass)
        S.proxy_units += units;
        S.half_units += r * node_size(l, P.Y[p]);
      } else {
        S.proxy_units += units;
      }
      S.max_rank = std::max(S.max_rank, P.rank[p]);
      S.ref_float_count += 2ull * static_cast<std::uint64_t>(r * r);
      S.ref_int_count += 4ull * static_cast<std::uint64_t>(r);
    }
    if (mode_[l] == kModeProxy || mode_[l] == kModeFused || two_groups(mode_[l])) {
      pair_piv[l].resize(P.X.size());
      pair_lu[l].resize(P.X.size());
      for (std::size_t p = 0; p < P.X.size(); ++p) {
        const std::int64_t r = P.rank[p];
        pair_piv[l][p] = S.piv_total;
        pair_lu[l][p] = S.lu_total;
        S.piv_total += 2 * r;
        // half levels keep the pivots only (their LU lives in U')
        if (mode_[l] != kModeHalf) S.lu_total += r * r + (r & 1);  // even: 16-B aligned slots (fused.cu)
      }
    }
    const auto& off = lists_[l].off[0];
    const auto& ep = entry_pair_[l];
    auto& ec = entry_col_[l];
    ec.assign(ep.size(), -1);
    const auto& lid = lists_[l].ids[0];
    const bool half = two_groups(mode_[l]);  // two column groups per node
    for (std::int64_t z = 0; z < cnt; ++z)
      for (int side = 0; side < (half ? 2 : 1); ++side) {
        // half levels: side 0 = the pairs z is X of (explicit U', streamed,
        // node id gid), side 1 = the pairs z is Y of (regenerated, node id gv)
        std::int32_t cols = 0;
        bool any = false;
        const std::int64_t g = side == 0 ? gid(l, z) : gv(l, z);
        // column groups: touching partners (Chebyshev distance 1) first (the
        // proxy kernels' difference form covers the prefix [0, vcols)); within
        // each, partners whose phase-1 output is consumed on this shard first.
        // An owned node's columns against a remote partner feed only phase 2
        // (that partner's t-vector comes from its ghost pool here), so phase 1
        // runs over [0, p1a) and [p1b, p1c) only. One shard: one range.
        const bool oz = owned(l, z);
        std::int32_t grp_end[4] = {0, 0, 0, 0};
        // group of every entry (0: touching + consumed here, 1: touching,
        // 2: consumed here, 3: rest; -1: no pair / the other side), computed once
        grp.resize(static_cast<std::size_t>(off[z + 1] - off[z]));
        for (std::int32_t e = off[z]; e < off[z + 1]; ++e) {
          const bool mine = ep[e] >= 0 && (!half || (P.X[ep[e]] == z) == (side == 0));
          grp[e - off[z]] = !mine ? -1
                                  : (vertex_adjacent(z, lid[e]) ? 0 : 2) + ((!oz || owned(l, lid[e])) ? 0 : 1);
        }
        for (int pass = 0; pass < 4; ++pass) {
          for (std::int32_t e = off[z]; e < off[z + 1]; ++e) {
            if (grp[e - off[z]] != pass) continue;
            ec[e] = cols;
            cols += P.rank[ep[e]];
            any = true;
          }
          grp_end[pass] = cols;
        }
        vcols[g] = grp_end[1];
        p1a[g] = grp_end[0];
        p1b[g] = grp_end[1];
        p1c[g] = grp_end[2];
        const bool stream = mode_[l] == kModeStream || (mode_[l] == kModeHalf && side == 0);
        const std::int32_t rp = !any || mode_[l] == kModePair || mode_[l] == kModeFused
                                    ? 0
                                    : stream ? (cols + kTileCols - 1) / kTileCols * kTileCols
                                             : cols + (cols & 1);
        rpad[g] = rp;
        soff[g] = S.s_doubles;
        S.s_doubles += rp;
        if (stream) {
          woff[g] = S.w_doubles;
          S.w_doubles += (node_size(l, z) + kTileRows - 1) / kTileRows * kTileRows * rp;
        }
      }
    if (mode_[l] == kModePair) {
      // pair-major pool: F_p = [U_p; V_p], (m + n) x rp row-major
      pair_wx[l].resize(P.X.size());
      pair_wy[l].resize(P.X.size());
      pair_rx[l].resize(P.X.size());
      pair_ry[l].resize(P.X.size());
      pair_cx[l].assign(P.X.size(), 0);
      pair_cy[l].assign(P.X.size(), 0);
      for (std::size_t p = 0; p < P.X.size(); ++p) {
        const std::int64_t m = node_size(l, P.X[p]), nn = node_size(l, P.Y[p]);
        const std::int32_t rp = P.rank[p] + (P.rank[p] & 1);
        pair_wx[l][p] = S.w_doubles;
        pair_wy[l][p] = S.w_doubles + m * rp;
        pair_rx[l][p] = rp;
        pair_ry[l][p] = rp;
        S.w_doubles += (m + nn) * rp;
      }
    }
    if (mode_[l] == kModeHalf) {
      // explicit U' of the X side only: W node base, first column, column tiles
      pair_wx[l].resize(P.X.size());
      pair_cx[l].resize(P.X.size());
      pair_rx[l].resize(P.X.size());
      pair_wy[l].assign(P.X.size(), 0);
      pair_cy[l].assign(P.X.size(), 0);
      pair_ry[l].assign(P.X.size(), 0);
      for (std::size_t p = 0; p < P.X.size(); ++p) {
        const std::int64_t gx = gid(l, P.X[p]);
        pair_wx[l][p] = woff[gx];
        pair_cx[l][p] = ec[P.eX[p]];
        pair_rx[l][p] = rpad[gx] / kTileCols;
      }
    }
    if (mode_[l] == kModeStream) {
      pair_wx[l].resize(P.X.size());
      pair_wy[l].resize(P.X.size());
      pair_rx[l].resize(P.X.size());
      pair_ry[l].resize(P.X.size());
      pair_cx[l].resize(P.X.size());
      pair_cy[l].resize(P.X.size());
      for (std::size_t p = 0; p < P.X.size(); ++p) {
        const std::int64_t gx = gid(l, P.X[p]), gy = gid(l, P.Y[p]);
        pair_wx[l][p] = woff[gx];
        pair_cx[l][p] = ec[P.eX[p]];
        pair_rx[l][p] = rpad[gx] / kTileCols;
        pair_wy[l][p] = woff[gy];
        pair_cy[l][p] = ec[P.eY[p]];
        pair_ry[l][p] = rpad[gy] / kTileCols;
      }
    }
  }
  if (S.s_doubles > 0x7fffffffLL) throw std::invalid_argument("planner: t-vector pool exceeds int32");

  // spos: column c of node z's layout (partner k) -> S slot of the mirrored
  // block (target k, partner z). Only owned targets run phase 2.
  spos.assign(std::max<std::int64_t>(S.s_doubles, 1), -1);
  proxy_segs.clear();
  for (int l = 1; l <= L_; ++l) {
    // no column layout: t-vectors stay inside the pair-major passes
    if (mode_[l] == kModePair || mode_[l] == kModeFused) continue;
    const std::int64_t cnt = 1LL << (3 * l);
    const auto& off = lists_[l].off[0];
    const auto& ids = lists_[l].ids[0];
    const auto& ep = entry_pair_[l];
    const auto& ec = entry_col_[l];
    const auto& P = pairs_[l];
    for (std::int64_t z = 0; z < cnt; ++z) {
      for (std::int32_t e = off[z]; e < off[z + 1]; ++e) {
        const std::int32_t p = ep[e];
        if (p < 0) continue;
        const std::int32_t k = ids[e];
        const int r = P.rank[p];
        const bool zx = P.X[p] == z;
        // half levels: z's column for k sits in z's stream group when z is
        // the pair's X, in its regenerated (virtual) group when z is Y
        const bool half = two_groups(mode_[l]);
        const bool split = mode_[l] == kModeSplit;
        const std::int64_t gz = half && !zx ? gv(l, z) : gid(l, z);
        const std::int64_t so = soff[gz] + ec[e];
        if (mode_[l] == kModeProxy || split || (half && !zx)) {
          ProxySeg sg{};
          sg.so = so;
          sg.base = off_[l][k];
          sg.piv_off = pair_piv[l][p];
          sg.lu_off = pair_lu[l][p];
          sg.r = r;
          sg.side = zx ? 0 : 1;
          // half levels: the phase-1 output of a regenerated column is the
          // transposed block's weight as it is (U' carries (LR)^-1): no solve.
          // Split levels: the Y-role columns are solved before the two-use
          // pass (2), the X-role ones after it, with the proxy levels (1)
          sg.solve = !owned(l, z) ? 0 : split ? (zx ? 1 : 2) : half ? 0 : 1;
          sg.node = static_cast<std::int32_t>(gz);
          proxy_segs.push_back(sg);
        }
        if (!owned(l, k)) continue;
        const std::int32_t e2 = zx ? P.eY[p] : P.eX[p];
        const std::int64_t gk = half && zx ? gv(l, k) : gid(l, k);  // k is the pair's Y iff z is X
        const std::int64_t dst = soff[gk] + ec[e2];
        for (int a = 0; a < r; ++a) spos[so + a] = static_cast<std::int32_t>(dst + a);
      }
    }
  }

  // phase-1 items: stream levels (rows x 256 columns of W_Z), proxy levels
  // (256 proxy targets x <= 2048 source points of Z)
  items.clear();
  reds.clear();
  std::int64_t ptot = 0;
  for (int l = 1; l <= L_; ++l) {
    if (mode_[l] == kModeDirect || mode_[l] == kModePair || mode_[l] == kModeFused) continue;
    const std::int64_t cnt = 1LL << (3 * l);
    // half / split levels: the X-role groups (node ids gid) here - streamed
    // (half) or regenerated (split); the Y-role ones (node ids gv) run as
    // h2_items (both uses at once)
    for (int side = 0; side < 1; ++side) {
    const int kind = mode_[l] == kModeHalf ? kModeStream : mode_[l] == kModeSplit ? kModeProxy : mode_[l];
    const std::int64_t chunk = kind == kModeStream ? kRowChunk : kSrcChunk;
    for (std::int64_t z = 0; z < cnt; ++z) {
      const std::int64_t g = side == 0 ? gid(l, z) : gv(l, z);
      const int rp = rpad[g];
      if (rp == 0) continue;
      const std::int64_t nr = node_size(l, z);
      const std::int64_t nrc = (nr + chunk - 1) / chunk;
      const std::int64_t pbase = ptot;
      if (nrc > 1) {
        ptot += nrc * rp;
        reds.push_back(P1Reduce{static_cast<std::int32_t>(g), rp, static_cast<std::int32_t>(nrc), kind, pbase});
      }
      // column ranges whose t-vectors are consumed on this shard (see the
      // column groups above), tile-aligned on stream levels
      const int al = kind == kModeStream ? kTileCols : 1;
      auto down = [&](int v) { return v / al * al; };
      auto up = [&](int v) { return std::min(rp, (v + al - 1) / al * al); };
      int rng[2][2] = {{0, up(p1a[g])}, {down(p1b[g]), up(p1c[g])}};
      if (rng[1][0] <= rng[0][1]) {  // adjacent or overlapping after alignment: merge
        rng[0][1] = std::max(rng[0][1], rng[1][1]);
        rng[1][0] = rng[1][1] = 0;
      }
      for (std::int64_t k = 0; k < nrc; ++k)
        for (const auto& rg : rng)
          for (int c0 = rg[0]; c0 < rg[1]; c0 += kColChunk) {
            P1Item it{};
            it.node = static_cast<std::int32_t>(g);
            it.row0 = static_cast<std::int32_t>(k * chunk);
            it.nrows = static_cast<std::int32_t>(std::min<std::int64_t>(chunk, nr - k * chunk));
            it.col0 = c0;
            it.ncols = std::min(kColChunk, rg[1] - c0);
            it.kind = kind;
            it.pslot = nrc > 1 ? pbase + k * rp + c0 : -1;
            items.push_back(it);
          }
    }
    }
  }
  S.p_doubles = ptot;

  // phase-2 proxy items (node-major, thread = target row): b_X += K(X, P_A) s_A
  // for every owned node A of a proxy level, rows in chunks of 256
  p2_items.clear();
  p2s_items.clear();
  h2_items.clear();
  pg_items.clear();
  pair_descs.clear();
  pd_level.assign(L_ + 2, 0);
  fused_descs.clear();
  fd_level.assign(L_ + 2, 0);
  pg_level.assign(L_ + 2, 0);
  pc_off.assign(T + 1, 0);
  pc_pos.clear();
  pair_out_total = 0;
  n_proxy_levels = 0;
  {
    // pair levels: descriptors of the pairs with an owned side, output runs
    std::vector<std::vector<std::int64_t>> runs(T);
    for (int l = 1; l <= L_; ++l) {
      pd_level[l] = static_cast<std::int64_t>(pair_descs.size());
      fd_level[l] = static_cast<std::int64_t>(fused_descs.size());
      if (mode_[l] == kModeFused) {
        const auto& P = pairs_[l];
        for (std::size_t p = 0; p < P.X.size(); ++p) {
          const bool ox = owned(l, P.X[p]), oy = owned(l, P.Y[p]);
          if (!ox && !oy) continue;
          FusedDesc d{};
          d.piv_off = pair_piv[l][p];
          d.lu_off = pair_lu[l][p];
          d.xrow = off_[l][P.X[p]];
          d.yrow = off_[l][P.Y[p]];
          d.m = static_cast<std::int32_t>(node_size(l, P.X[p]));
          d.n = static_cast<std::int32_t>(node_size(l, P.Y[p]));
          d.r = P.rank[p];
          d.own = (ox ? 1 : 0) | (oy ? 2 : 0);
          d.touch = vertex_adjacent(P.X[p], P.Y[p]) ? 1 : 0;
          const std::int64_t gx = gid(l, P.X[p]), gy = gid(l, P.Y[p]);
          d.cx = 0.5 * (center[4 * gx] + center[4 * gy]);
          d.cy = 0.5 * (center[4 * gx + 1] + center[4 * gy + 1]);
          d.cz = 0.5 * (center[4 * gx + 2] + center[4 * gy + 2]);
          d.out = pair_out_total;
          if (ox) runs[gx].push_back(d.out);
          if (oy) runs[gy].push_back(d.out + d.m);
          pair_out_total += d.m + d.n;
          fused_descs.push_back(d);
        }
        continue;
      }
      if (mode_[l] != kModePair) continue;
      const auto& P = pairs_[l];
      for (std::size_t p = 0; p < P.X.size(); ++p) {
        const bool ox = owned(l, P.X[p]), oy = owned(l, P.Y[p]);
        if (!ox && !oy) continue;
        PairDesc d{};
        d.woff = pair_wx[l][p];
        d.xrow = off_[l][P.X[p]];
        d.yrow = off_[l][P.Y[p]];
        d.m = static_cast<std::int32_t>(node_size(l, P.X[p]));
        d.n = static_cast<std::int32_t>(node_size(l, P.Y[p]));
        d.rp = pair_rx[l][p];
        d.own = (ox ? 1 : 0) | (oy ? 2 : 0);
        d.out = pair_out_total;
        if (ox) runs[gid(l, P.X[p])].push_back(d.out);
        if (oy) runs[gid(l, P.Y[p])].push_back(d.out + d.m);
        pair_out_total += d.m + d.n;
        pair_descs.push_back(d);
      }
    }
    pd_level[L_ + 1] = static_cast<std::int64_t>(pair_descs.size());
    fd_level[L_ + 1] = static_cast<std::int64_t>(fused_descs.size());
    for (std::int64_t g = 0; g < T; ++g) {
      pc_off[g] = static_cast<std::int32_t>(pc_pos.size());
      pc_pos.insert(pc_pos.end(), runs[g].begin(), runs[g].end());
    }
    pc_off[T] = static_cast<std::int32_t>(pc_pos.size());
  }
  for (int l = 1; l <= L_; ++l) {
    pg_level[l] = static_cast<std::int64_t>(pg_items.size());
    if (mode_[l] == kModeDirect) continue;
    if (mode_[l] == kModePair || mode_[l] == kModeFused) {
      // gather the pair outputs of every owned node into the level's partial
      const std::int64_t cnt = 1LL << (3 * l);
      int slot = -1;
      for (std::int64_t z = 0; z < cnt; ++z) {
        const std::int64_t g = gid(l, z);
        if (pc_off[g + 1] == pc_off[g]) continue;
        if (slot < 0) slot = n_proxy_levels++;
        const std::int64_t nr = node_size(l, z);
        for (std::int64_t r0 = 0; r0 < nr; r0 += kColChunk)
          pg_items.push_back(P2Item{static_cast<std::int32_t>(g), static_cast<std::int32_t>(r0),
                                    static_cast<std::int32_t>(std::min<std::int64_t>(kColChunk, nr - r0)),
                                    slot});
      }
      continue;
    }
    const bool half = two_groups(mode_[l]);
    // half / split levels: the X-role groups and the Y-role groups write a
    // partial each (two output slots)
    for (int side = 0; side < (half ? 2 : 1); ++side) {
      const bool stream = mode_[l] == kModeHalf ? side == 0 : mode_[l] == kModeStream;
      const std::int64_t cnt = 1LL << (3 * l);
      const std::int64_t step = stream ? kTileRows : kColChunk;
      auto& dst = stream ? p2s_items : p2_items;
      int slot = -1;
      for (std::int64_t z = 0; z < cnt; ++z) {
        const std::int64_t g = side == 0 ? gid(l, z) : gv(l, z);
        // half levels' regenerated groups: every shard that holds the group
        // evaluates it (its v feeds the owned partners' streamed rows)
        if (rpad[g] == 0 || (!owned(l, z) && !(half && side == 1))) continue;
        if (slot < 0) slot = n_proxy_levels++;
        const std::int64_t nr = node_size(l, z);
        // proxy levels: even split into ceil(nr / 256) items (a 256 + small
        // remainder split leaves most of the second item's target slots idle)
        const std::int64_t per =
            stream ? step : (nr + (nr + step - 1) / step - 1) / ((nr + step - 1) / step);
        if (half && side == 1) {
          // both uses in one pass; the node's v partials per chunk when it
          // spans several. Chunks of 256 rows and the remainder (which runs
          // on 2 / 4 thread groups when it is <= 128 / <= 64 rows): an even
          // split of 257-320 rows would fill two 256-slot chunks half
          const std::int64_t per = step;
          const std::int64_t nch = (nr + per - 1) / per;
          const std::int64_t pbase = S.p_doubles;
          if (nch > 1) {
            S.p_doubles += nch * rpad[g];
            reds.push_back(P1Reduce{static_cast<std::int32_t>(g), rpad[g], static_cast<std::int32_t>(nch),
                                    kModeHalf, pbase});
          }
          std::int64_t k = 0;
          for (std::int64_t r0 = 0; r0 < nr; r0 += per, ++k)
            h2_items.push_back(H2Item{static_cast<std::int32_t>(g), static_cast<std::int32_t>(r0),
                                      static_cast<std::int32_t>(std::min<std::int64_t>(per, nr - r0)),
                                      owned(l, z) ? slot : -1, nch > 1 ? pbase + k * rpad[g] : -1});
          continue;
        }
        for (std::int64_t r0 = 0; r0 < nr; r0 += per)
          dst.push_back(P2Item{static_cast<std::int32_t>(g), static_cast<std::int32_t>(r0),
                               static_cast<std::int32_t>(std::min<std::int64_t>(per, nr - r0)), slot});
      }
    }
  }
  pg_level[L_ + 1] = static_cast<std::int64_t>(pg_items.size());

  if (!leaf_done_) layout_leaf();
}

// Leaf plan and the symmetric near-field lists. They depend on the tree, the
// lists and the (fixed) leaf mode only, not on ranks, so the engine runs this
// on a host thread while the ACA rank pass occupies the GPU.
void Planner::layout_leaf() {
  PlanSizes& S = sizes;
  // leaf plan: owned leaves; near lists = self, near_edge, near_face (the
  // reference's dense blocks), plus the leaf-level admissible partners when
  // that level is evaluated directly
  const std::int64_t nl = 1LL << (3 * L_);
  if (L_ == 0) {
    leaf0 = 0;
    leaf1 = rank_ == 0 ? 1 : 0;
  } else {
    leaf0 = static_cast<std::int64_t>(oct0_) << (3 * (L_ - 1));
    leaf1 = static_cast<std::int64_t>(oct1_) << (3 * (L_ - 1));
  }
  near_off.assign(nl + 1, 0);
  near_dense.assign(nl + 1, 0);
  near_ids.clear();
  S.near_blocks = S.near_entries = S.direct_evals = 0;
  for (std::int64_t x = 0; x < nl; ++x) {
    near_off[x] = static_cast<std::int32_t>(near_ids.size());
    const std::int64_t mx = node_size(L_, x);
    if (mx == 0 || x < leaf0 || x >= leaf1) continue;
    std::int64_t ndense_pts = 0;
    std::int32_t nd = 0;
    auto add = [&](std::int64_t y, bool dense) {
      const std::int64_t ny = node_size(L_, y);
      if (ny == 0) return;
      near_ids.push_back(static_cast<std::int32_t>(y));
      if (dense) {
        ++nd;
        ndense_pts += ny;
        ++S.near_blocks;
        S.near_entries += mx * ny;
      } else {
        S.direct_evals += mx * ny;
      }
    };
    add(x, true);
    if (L_ > 0) {
      for (int k = 1; k < kListKinds; ++k)
        for (std::int32_t e = lists_[L_].off[k][x]; e < lists_[L_].off[k][x + 1]; ++e)
          add(lists_[L_].ids[k][e], true);
      if (mode_[L_] == kModeDirect)
        for (std::int32_t e = lists_[L_].off[0][x]; e < lists_[L_].off[0][x + 1]; ++e)
          add(lists_[L_].ids[0][e], false);
    }
    near_dense[x] = nd;
    (void)ndense_pts;
  }
  near_off[nl] = static_cast<std::int32_t>(near_ids.size());

  // symmetric matrix-free lists (see planner.h)
  sym_off.assign(nl + 1, 0);
  sym_ids.clear();
  sym_cnt.assign(4 * nl, 0);
  out_off.assign(nl + 1, 0);
  nf_off.assign(nl + 1, 0);
  nf_cols.assign(nl + 1, 0);
  nf_total = 0;
  std::vector<std::pair<std::int32_t, std::int64_t>> incoming;  // (target leaf, pair-buffer run)
  std::vector<std::int32_t> cat[4];  // dense one-way, direct one-way, dense sym, direct sym
  std::int64_t otot = 0;
  auto own = [&](std::int64_t y) { return y >= leaf0 && y < leaf1; };
  // a pair is evaluated once iff both leaves are owned and fit one pass of
  // the near kernel (their column sums are then complete after one sweep)
  auto sym = [&](std::int64_t u) { return own(u) && node_size(L_, u) <= kNearPassRows; };
  for (std::int64_t x = 0; x < nl; ++x) {
    sym_off[x] = static_cast<std::int32_t>(sym_ids.size());
    out_off[x] = otot;
    nf_off[x] = nf_total;
    if (node_size(L_, x) == 0 || !own(x)) continue;
    for (auto& c : cat) c.clear();
    auto put = [&](std::int64_t y, bool dense) {
      if (node_size(L_, y) == 0) return;
      const bool pair = sym(x) && sym(y);
      if (pair && y < x) return;  // supplied by y's pass
      cat[(pair ? 2 : 0) + (dense ? 0 : 1)].push_back(static_cast<std::int32_t>(y));
    };
    if (L_ > 0) {
      for (int k = 1; k < kListKinds; ++k)
        for (std::int32_t e = lists_[L_].off[k][x]; e < lists_[L_].off[k][x + 1]; ++e)
          put(lists_[L_].ids[k][e], true);
      if (mode_[L_] == kModeDirect)
        for (std::int32_t e = lists_[L_].off[0][x]; e < lists_[L_].off[0][x + 1]; ++e)
          put(lists_[L_].ids[0][e], false);
    }
    sym_ids.push_back(static_cast<std::int32_t>(x));
    // stored columns: self + dense categories 0 and 2 (bit 0), direct
    // categories 1 and 3 (bit 1)
    std::int64_t ncols = (nf_mask_ & 1) ? node_size(L_, x) : 0;
    for (int c = 0; c < 4; ++c)
      if (nf_mask_ & ((c & 1) ? 2 : 1))
        for (std::int32_t y : cat[c]) ncols += node_size(L_, y);
    nf_cols[x] = static_cast<std::int32_t>(ncols);
    nf_total += node_size(L_, x) * ncols;
    for (int c = 0; c < 4; ++c) {
      sym_cnt[4 * x + c] = static_cast<std::int32_t>(cat[c].size());
      for (std::int32_t y : cat[c]) {
        sym_ids.push_back(y);
        if (c >= 2) {
          incoming.emplace_back(y, otot);
          otot += node_size(L_, y);
        }
      }
    }
  }
  sym_off[nl] = static_cast<std::int32_t>(sym_ids.size());
  out_off[nl] = otot;
  nf_off[nl] = nf_total;
  // incoming runs per leaf, in the order they were produced (counting sort)
  in_off.assign(nl + 1, 0);
  for (const auto& iv : incoming) ++in_off[iv.first + 1];
  for (std::int64_t y = 0; y < nl; ++y) in_off[y + 1] += in_off[y];
  in_pos.assign(incoming.size(), 0);
  {
    std::vector<std::int32_t> fill(in_off.begin(), in_off.end() - 1);
    for (const auto& iv : incoming) in_pos[fill[iv.first]++] = iv.second;
  }
  leaf_done_ = true;
}

}  // namespace h3db
