// schedule.cpp -- see schedule.hpp.
#include "schedule.hpp"

#include <array>
#include <climits>
#include <cstdint>

#include "fx_core.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <utility>

namespace igm {
namespace {

struct Grid {
  long long gx = 0, gy = 0, gz = 0;
};

// Fraction of (sampled) dependencies that are +-1 neighbours on the grid.
double neighbour_score(int n, const std::vector<int>& orp, const std::vector<int>& oci, long long gx,
                       long long gxy) {
  long long hit = 0, tot = 0;
  const int step = std::max(1, n / 200000);
  for (int i = 0; i < n; i += step) {
    const long long xi = i % gx, yi = (i / gx) % (gxy / gx), zi = i / gxy;
    for (int k = orp[i]; k < orp[i + 1]; ++k) {
      const long long j = oci[k];
      const long long xj = j % gx, yj = (j / gx) % (gxy / gx), zj = j / gxy;
      ++tot;
      if (std::llabs(xi - xj) <= 1 && std::llabs(yi - yj) <= 1 && std::llabs(zi - zj) <= 1) ++hit;
    }
  }
  return tot ? static_cast<double>(hit) / tot : 0.0;
}

// Infer a gx*gy*gz natural-order grid from the distinct dependency offsets.
Grid detect_grid(int n, const std::vector<int>& orp, const std::vector<int>& oci) {
  std::vector<long long> offs;
  for (int i = 0; i < n && offs.size() <= 64; i += std::max(1, n / 4096)) {
    for (int k = orp[i]; k < orp[i + 1]; ++k) {
      const long long d = std::llabs(static_cast<long long>(i) - oci[k]);
      if (std::find(offs.begin(), offs.end(), d) == offs.end()) offs.push_back(d);
    }
  }
  Grid best;
  if (offs.empty() || offs.size() > 64) return best;
  std::sort(offs.begin(), offs.end());
  long long dmin2 = 0;
  for (long long d : offs)
    if (d >= 2) {
      dmin2 = d;
      break;
    }
  if (dmin2 == 0) return best;
  double best_score = 0.0;
  const long long dmax = offs.back();
  for (long long gx = dmin2 - 1; gx <= dmin2 + 1; ++gx) {
    if (gx < 2 || n % gx) continue;
    std::vector<long long> cand{static_cast<long long>(n)};
    for (int a = -1; a <= 1; ++a)
      for (int b = -1; b <= 1; ++b) cand.push_back(dmax - a * gx - b);
    for (long long gxy : cand) {
      if (gxy < gx || gxy % gx || n % gxy) continue;
      const double sc = neighbour_score(n, orp, oci, gx, gxy);
      if (sc > best_score + 1e-12) {
        best_score = sc;
        best = Grid{gx, gxy / gx, n / gxy};
      }
    }
  }
  if (best_score < 0.99) return Grid{};
  return best;
}

long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

}  // namespace

TriSchedule build_tri_schedule(int n, const int* rp, const int* ci, const std::int64_t* vals,
                               const int* dpos, bool upper, int num_sms, int tile_cap_override) {
  TriSchedule S;
  S.n = n;
  // ---- strip: off-diagonal, structurally meaningful entries in CSR order (a
  // "lower" entry with j > i multiplies a zero-initialised slot in
  // ilu.cpp:126-135, an "upper" one with j < i likewise) and the diagonal
  std::vector<int> orp(static_cast<size_t>(n) + 1, 0), oci;
  std::vector<std::int64_t> ov, dg(static_cast<size_t>(n));
  oci.reserve(rp[n]);
  ov.reserve(rp[n]);
  for (int i = 0; i < n; ++i) {
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int j = ci[k];
      if (j < 0 || j >= n) throw std::invalid_argument("upload_ilu: column index out of range");
      if (j == i || (upper ? (j < i) : (j > i))) continue;
      oci.push_back(j);
      ov.push_back(vals[k]);
    }
    orp[i + 1] = static_cast<int>(oci.size());
    const int dp = dpos[i];
    if (dp < 0 || dp >= rp[n]) throw std::invalid_argument("upload_ilu: diagonal position out of range");
    dg[i] = vals[dp];
    if (dg[i] == 0) throw std::invalid_argument("upload_ilu: zero diagonal entry");
  }
  // ---- DAG levels
  std::vector<int> lev(static_cast<size_t>(n), 0);
  for (int q = 0; q < n; ++q) {
    const int i = upper ? n - 1 - q : q;
    int l = 0;
    for (int k = orp[i]; k < orp[i + 1]; ++k) l = std::max(l, lev[oci[k]] + 1);
    lev[i] = l;
    S.nlevels = std::max(S.nlevels, l + 1);
    S.maxd = std::max(S.maxd, orp[i + 1] - orp[i]);
  }
  S.stride = S.maxd <= 4 ? 4 : (S.maxd <= 8 ? 8 : 16);
  // ---- tiles
  const int cap = tile_cap_override > 0 ? std::min(tile_cap_override, tri_tile_cap(S.stride))
                                        : tri_tile_cap(S.stride);
  S.tile_cap = cap;
  const int nsm = std::max(1, num_sms);
  std::vector<int> tile_of(static_cast<size_t>(n));
  const Grid g = n > 0 ? detect_grid(n, orp, oci) : Grid{};
  if (g.gx > 0 && tile_cap_override <= 0) {
    const long long G[3] = {g.gx, g.gy, g.gz};
    // x-y cross-section <= 256 rows (one row per compute thread per level),
    // then as deep in z as the shared-memory tile allows
    long long B[3] = {g.gx, g.gy, g.gz};
    static const long long xsec = [] {
      const char* e = std::getenv("IGM_TRI_XSEC");
      return e ? std::max(1LL, std::atoll(e)) : 256LL;
    }();
    static const long long zcap = [] {
      const char* e = std::getenv("IGM_TRI_ZCAP");
      return e ? std::max(1LL, std::atoll(e)) : (1LL << 40);
    }();
    while (B[0] * B[1] > xsec && (B[0] > 1 || B[1] > 1)) {
      if (B[0] >= B[1]) B[0] = cdiv(B[0], 2);
      else B[1] = cdiv(B[1], 2);
    }
    while (B[0] * B[1] * B[2] > cap || B[2] > zcap) B[2] = cdiv(B[2], 2);
    auto assign = [&](const long long* b) {
      const long long nb0 = cdiv(G[0], b[0]), nb1 = cdiv(G[1], b[1]);
      for (int i = 0; i < n; ++i) {
        const long long x = i % G[0], y = (i / G[0]) % G[1], z = i / (G[0] * G[1]);
        tile_of[i] = static_cast<int>(((z / b[2]) * nb1 + y / b[1]) * nb0 + x / b[0]);
      }
    };
    // every dependency in an earlier-or-same tile (ticket order)?  Then the
    // tile graph is acyclic and any residency works; otherwise the tiles of
    // one z-layer (where back edges can occur) must fit on the GPU at once.
    auto acyclic = [&]() {
      for (int i = 0; i < n; ++i)
        for (int k = orp[i]; k < orp[i + 1]; ++k) {
          const int tj = tile_of[oci[k]];
          if (upper ? (tj < tile_of[i]) : (tj > tile_of[i])) return false;
        }
      return true;
    };
    assign(B);
    bool ok = acyclic();
    S.acyclic = ok;
    // Wavefront ticket order (stencils whose z-layer tile graph has cycles,
    // e.g. 27-point): tiles sorted by the DAG level of their first row in
    // ticket direction, tickets of equal level forming one layer.  Valid when
    // every cross-tile dependency points to a strictly earlier layer, or to
    // the same layer with each layer small enough to be co-resident; then
    // the wavefront flows through consecutive layers instead of serialising
    // the z-layers (which must each be fully resident).  Among candidate
    // bricks the one with the smallest max(critical path, tile-levels / SMs)
    // is taken.
    if (!ok) {
      struct Cand {
        long long b[3];
        double cost;
        bool cyclic = false;     // some dependency within a layer
        std::vector<int> perm;   // old tile id -> new (ticket-ordered) id
        std::vector<int> layer;  // per new tile id
      };
      auto try_wave = [&](const long long* b, Cand& c) {
        assign(b);
        const long long nb0 = cdiv(G[0], b[0]), nb1 = cdiv(G[1], b[1]), nb2 = cdiv(G[2], b[2]);
        const long long nt = nb0 * nb1 * nb2;
        if (b[0] * b[1] * b[2] > cap) return false;
        std::vector<int> lo(static_cast<size_t>(nt), INT32_MAX), hi(static_cast<size_t>(nt), -1);
        for (int i = 0; i < n; ++i) {
          lo[tile_of[i]] = std::min(lo[tile_of[i]], lev[i]);
          hi[tile_of[i]] = std::max(hi[tile_of[i]], lev[i]);
        }
        std::vector<int> ord(static_cast<size_t>(nt));
        std::iota(ord.begin(), ord.end(), 0);
        // ticket order = ascending first level; the backward factor's tickets
        // run from the last tile id down, so its ids are assigned reversed
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int bb) { return lo[a] < lo[bb]; });
        if (upper) std::reverse(ord.begin(), ord.end());
        c.perm.assign(static_cast<size_t>(nt), 0);
        for (long long q = 0; q < nt; ++q) c.perm[ord[q]] = static_cast<int>(q);
        c.layer.assign(static_cast<size_t>(nt), 0);
        std::vector<int> key(static_cast<size_t>(nt));
        for (long long t = 0; t < nt; ++t) key[c.perm[t]] = lo[t];
        // layers in ticket order
        long long max_layer = 0, run = 0;
        int lay = -1;
        for (long long q = 0; q < nt; ++q) {
          const int id = upper ? static_cast<int>(nt - 1 - q) : static_cast<int>(q);
          const int prev = upper ? static_cast<int>(nt - q) : static_cast<int>(q - 1);
          if (q == 0 || key[id] != key[prev]) {
            ++lay;
            run = 0;
          }
          c.layer[id] = lay;
          max_layer = std::max(max_layer, ++run);
        }
        bool same_layer_dep = false;
        for (int i = 0; i < n; ++i)
          for (int k = orp[i]; k < orp[i + 1]; ++k) {
            const int ti = c.perm[tile_of[i]], tj = c.perm[tile_of[oci[k]]];
            if (ti == tj) continue;
            if (c.layer[tj] > c.layer[ti]) return false;
            if (c.layer[tj] == c.layer[ti]) same_layer_dep = true;
          }
        if (same_layer_dep && max_layer > nsm) return false;
        c.cyclic = same_layer_dep;
        long long tl = 0;
        for (long long t = 0; t < nt; ++t)
          if (hi[t] >= 0) tl += hi[t] - lo[t] + 1;
        c.cost = std::max(static_cast<double>(S.nlevels), static_cast<double>(tl) / nsm) *
                 (same_layer_dep ? 1.1 : 1.0);
        for (int d = 0; d < 3; ++d) c.b[d] = b[d];
        return true;
      };
      std::vector<std::array<long long, 3>> cands;
      cands.push_back({B[0], B[1], B[2]});
      {  // the co-resident z-layer brick (below) as a candidate too
        long long b[3] = {B[0], B[1], B[2]};
        while (cdiv(G[0], b[0]) * cdiv(G[1], b[1]) > nsm && b[2] > 1) {
          b[2] = cdiv(b[2], 2);
          if (b[0] <= b[1]) b[0] = std::min(G[0], 2 * b[0]);
          else b[1] = std::min(G[1], 2 * b[1]);
          while (b[0] * b[1] * b[2] > cap && b[2] > 1) b[2] = cdiv(b[2], 2);
        }
        cands.push_back({b[0], b[1], b[2]});
      }
      Cand best;
      best.cost = -1;
      for (auto& cb : cands) {
        Cand c;
        if (try_wave(cb.data(), c) && (best.cost < 0 || c.cost < best.cost)) best = std::move(c);
      }
      if (best.cost >= 0 && !std::getenv("IGM_TRI_NO_WAVE")) {
        assign(best.b);
        for (int i = 0; i < n; ++i) tile_of[i] = best.perm[tile_of[i]];
        for (int d = 0; d < 3; ++d) B[d] = best.b[d];
        S.tile_layer = best.layer;
        S.acyclic = !best.cyclic;
        ok = true;
      } else {
        assign(B);
      }
    }
    if (!ok) {
      while (cdiv(G[0], B[0]) * cdiv(G[1], B[1]) > nsm && B[2] > 1) {
        B[2] = cdiv(B[2], 2);
        if (B[0] <= B[1]) B[0] = std::min(G[0], 2 * B[0]);
        else B[1] = std::min(G[1], 2 * B[1]);
        while (B[0] * B[1] * B[2] > cap && B[2] > 1) B[2] = cdiv(B[2], 2);
      }
      ok = B[0] * B[1] * B[2] <= cap && cdiv(G[0], B[0]) * cdiv(G[1], B[1]) <= nsm;
      if (ok) assign(B);
    }
    if (ok) {
      for (int d = 0; d < 3; ++d) {
        S.grid[d] = static_cast<int>(G[d]);
        S.brick[d] = static_cast<int>(B[d]);
      }
      S.ntiles = static_cast<int>(cdiv(G[0], B[0]) * cdiv(G[1], B[1]) * cdiv(G[2], B[2]));
    }
  }
  if (S.ntiles == 0) {  // contiguous row blocks (dependencies only to earlier blocks)
    S.acyclic = true;
    int T = std::min(cap, std::max(32, static_cast<int>(cdiv(std::max(n, 1), nsm))));
    if (tile_cap_override > 0) T = cap;
    S.ntiles = n > 0 ? static_cast<int>(cdiv(n, T)) : 1;
    for (int i = 0; i < n; ++i) tile_of[i] = i / T;
  }
  // ---- slots: tile-major, then level, then row
  std::vector<int> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    if (tile_of[a] != tile_of[b]) return tile_of[a] < tile_of[b];
    if (lev[a] != lev[b]) return lev[a] < lev[b];
    return a < b;
  });
  std::vector<int> slot(static_cast<size_t>(n));
  for (int p = 0; p < n; ++p) slot[order[p]] = p;
  S.tile_pbase.assign(static_cast<size_t>(S.ntiles) + 1, 0);
  for (int i = 0; i < n; ++i) S.tile_pbase[tile_of[i] + 1]++;
  for (int t = 0; t < S.ntiles; ++t) S.tile_pbase[t + 1] += S.tile_pbase[t];
  for (int t = 0; t < S.ntiles; ++t) {
    if (S.tile_pbase[t + 1] - S.tile_pbase[t] > cap)
      throw std::logic_error("upload_ilu: tile exceeds shared-memory capacity");
    S.max_tile_rows = std::max(S.max_tile_rows, S.tile_pbase[t + 1] - S.tile_pbase[t]);
  }
  // segments
  S.tile_seg.assign(static_cast<size_t>(S.ntiles) + 1, 0);
  S.seg_rows.push_back(0);
  for (int t = 0; t < S.ntiles; ++t) {
    int seg_start = S.tile_pbase[t];
    for (int p = S.tile_pbase[t]; p < S.tile_pbase[t + 1]; ++p) {
      // a new segment per level, and wide levels split into <= 256-row parts
      // (rows of one level are independent of each other)
      if (p == S.tile_pbase[t] || lev[order[p]] != lev[order[p - 1]] || p - seg_start >= kTriSegRows) {
        if (p != S.tile_pbase[t]) S.seg_rows.push_back(p);
        S.seg_level.push_back(lev[order[p]]);
        seg_start = p;
      }
    }
    if (S.tile_pbase[t + 1] > S.tile_pbase[t]) S.seg_rows.push_back(S.tile_pbase[t + 1]);
    S.tile_seg[t + 1] = static_cast<int>(S.seg_level.size());
  }
  if (S.seg_level.empty()) {  // n == 0: one empty segment keeps the arrays valid
    S.seg_level.push_back(0);
    S.seg_rows.push_back(0);
  }
  // ---- per segment: distinct cross-tile producer rows (schedule statistics
  // and validation)
  const int nseg_all = static_cast<int>(S.seg_level.size());
  S.seg_xptr.assign(static_cast<size_t>(nseg_all) + 1, 0);
  for (int sg = 0; sg < nseg_all; ++sg) {
    const size_t x0 = S.seg_xrow.size();
    for (int p = S.seg_rows[sg]; p < S.seg_rows[sg + 1] && p < n; ++p) {
      const int i = order[p];
      for (int k = orp[i]; k < orp[i + 1]; ++k) {
        const int j = oci[k];
        if (tile_of[j] == tile_of[i]) continue;
        if (std::find(S.seg_xrow.begin() + static_cast<std::ptrdiff_t>(x0), S.seg_xrow.end(), j) == S.seg_xrow.end())
          S.seg_xrow.push_back(j);
      }
    }
    S.seg_xptr[sg + 1] = static_cast<int>(S.seg_xrow.size());
    S.max_seg_ext = std::max(S.max_seg_ext, S.seg_xptr[sg + 1] - S.seg_xptr[sg]);
  }
  if (S.seg_xrow.empty()) S.seg_xrow.push_back(0);
  // ---- stripped factor in natural order (counting pass)
  S.c_rp = orp;
  S.c_ci = oci;
  S.c_val = ov;
  S.c_diag = dg;
  if (S.c_ci.empty()) {
    S.c_ci.push_back(0);
    S.c_val.push_back(0);
  }
  if (S.c_diag.empty()) S.c_diag.push_back(1);
  // ---- per-slot records
  const int W = S.stride;
  S.p_row.resize(static_cast<size_t>(std::max(n, 1)));
  S.p_nd.resize(static_cast<size_t>(std::max(n, 1)));
  // unused dependency slots: local slot 0 with factor 0 (an exact zero term)
  S.p_dep.assign(static_cast<size_t>(std::max(n, 1)) * W, 0);
  S.p_val.assign(static_cast<size_t>(std::max(n, 1)) * W, 0);
  S.p_xrp.assign(static_cast<size_t>(n) + 1, 0);
  S.p_mag.resize(static_cast<size_t>(std::max(n, 1)));
  S.p_info.resize(static_cast<size_t>(std::max(n, 1)));
  S.p_diag.resize(static_cast<size_t>(std::max(n, 1)));
  for (int p = 0; p < n; ++p) {
    const int i = order[p];
    const int t = tile_of[i];
    S.p_row[p] = i;
    S.p_nd[p] = orp[i + 1] - orp[i];
    for (int k = orp[i], d = 0; k < orp[i + 1]; ++k, ++d) {
      const int j = oci[k];
      const int enc = tile_of[j] == t ? slot[j] - S.tile_pbase[t] : ~j;  // tile-local slot or ~global row
      if (d < W) {
        S.p_dep[static_cast<size_t>(p) * W + d] = enc;
        S.p_val[static_cast<size_t>(p) * W + d] = ov[k];
      } else {
        S.p_xdep.push_back(enc);
        S.p_xval.push_back(ov[k]);
      }
    }
    S.p_xrp[p + 1] = static_cast<int>(S.p_xdep.size());
    const SDivMagic gm = make_sdiv(dg[i]);
    S.p_mag[p] = gm.u.m;
    S.p_info[p] = gm.u.sh1 | (gm.u.sh2 << 1) | (gm.den_neg << 8) | (gm.den_is_m1 << 9);
    S.p_diag[p] = dg[i];
  }
  if (S.p_xdep.empty()) {
    S.p_xdep.push_back(0);
    S.p_xval.push_back(0);
  }
  // rows read by another tile are published as tagged 128-bit words
  {
    std::vector<char> exported(static_cast<size_t>(std::max(n, 1)), 0);
    for (int i = 0; i < n; ++i)
      for (int k = orp[i]; k < orp[i + 1]; ++k)
        if (tile_of[oci[k]] != tile_of[i]) exported[oci[k]] = 1;
    for (int p = 0; p < n; ++p)
      if (exported[order[p]]) S.p_info[p] |= 1 << 10;
  }
  // packed records (compact when every factor value fits in int32)
  S.compact = !std::getenv("IGM_TRI_WIDE_REC");
  for (size_t q = 0; q < S.p_val.size() && S.compact; ++q)
    S.compact = S.p_val[q] >= INT32_MIN && S.p_val[q] <= INT32_MAX;
  for (int p = 0; p < n && S.compact; ++p) S.compact = S.p_nd[p] <= 255;
  S.rec_bytes = S.compact ? 16 + 8 * W : 32 + 12 * W;
  S.p_rec.assign(static_cast<size_t>(std::max(n, 1)) * S.rec_bytes, 0);
  for (int p = 0; p < n; ++p) {
    unsigned char* r = S.p_rec.data() + static_cast<size_t>(p) * S.rec_bytes;
    if (S.compact) {
      const int hdr[2] = {S.p_row[p], S.p_info[p] | (S.p_nd[p] << 16)};
      std::memcpy(r, hdr, 8);
      std::memcpy(r + 8, &S.p_mag[p], 8);
      std::memcpy(r + 16, &S.p_dep[static_cast<size_t>(p) * W], 4 * W);
      for (int d = 0; d < W; ++d) {
        const int32_t v = static_cast<int32_t>(S.p_val[static_cast<size_t>(p) * W + d]);
        std::memcpy(r + 16 + 4 * W + 4 * d, &v, 4);
      }
    } else {
      const int hdr[4] = {S.p_row[p], S.p_nd[p], S.p_info[p], S.p_xrp[p]};
      std::memcpy(r, hdr, 16);
      std::memcpy(r + 16, &S.p_mag[p], 8);
      std::memcpy(r + 24, &S.p_diag[p], 8);
      std::memcpy(r + 32, &S.p_dep[static_cast<size_t>(p) * W], 4 * W);
      std::memcpy(r + 32 + 4 * W, &S.p_val[static_cast<size_t>(p) * W], 8 * W);
    }
  }
  // ---- per segment: producer tiles of its cross-tile dependencies
  S.seg_wptr.push_back(0);
  const int nseg = static_cast<int>(S.seg_level.size());
  for (int sg = 0; sg < nseg; ++sg) {
    const size_t w0 = S.seg_wt.size();
    for (int p = S.seg_rows[sg]; p < S.seg_rows[sg + 1]; ++p) {
      const int i = order[p];
      for (int k = orp[i]; k < orp[i + 1]; ++k) {
        const int tj = tile_of[oci[k]];
        if (tj != tile_of[i] &&
            std::find(S.seg_wt.begin() + static_cast<std::ptrdiff_t>(w0), S.seg_wt.end(), tj) == S.seg_wt.end())
          S.seg_wt.push_back(tj);
      }
    }
    S.seg_wptr.push_back(static_cast<int>(S.seg_wt.size()));
  }
  if (S.seg_wt.empty()) S.seg_wt.push_back(0);
  return S;
}

int validate_tri_schedule(const TriSchedule& S, const int* rp, const int* ci, bool upper) {
  const int n = S.n;
  std::vector<int> slot_of(static_cast<size_t>(n), -1), tile_of(static_cast<size_t>(n), -1),
      lev_of(static_cast<size_t>(n), -1);
  for (int t = 0; t < S.ntiles; ++t)
    for (int sg = S.tile_seg[t]; sg < S.tile_seg[t + 1]; ++sg)
      for (int p = S.seg_rows[sg]; p < S.seg_rows[sg + 1]; ++p) {
        const int i = S.p_row[p];
        if (i < 0 || i >= n || slot_of[i] >= 0) return 1;  // each row exactly once
        slot_of[i] = p;
        tile_of[i] = t;
        lev_of[i] = S.seg_level[sg];
        if (p < S.tile_pbase[t] || p >= S.tile_pbase[t + 1]) return 2;
      }
  for (int i = 0; i < n; ++i)
    if (slot_of[i] < 0) return 1;
  for (int t = 0; t < S.ntiles; ++t)
    for (int sg = S.tile_seg[t] + 1; sg < S.tile_seg[t + 1]; ++sg)
      if (S.seg_level[sg] < S.seg_level[sg - 1] || S.seg_rows[sg + 1] - S.seg_rows[sg] > kTriSegRows)
        return 3;  // levels non-decreasing in a tile, segments <= 256 rows
  const int W = S.stride;
  for (int i = 0; i < n; ++i) {
    const int p = slot_of[i];
    int d = 0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int j = ci[k];
      if (j == i || (upper ? (j < i) : (j > i))) continue;
      const int enc = d < W ? S.p_dep[static_cast<size_t>(p) * W + d] : S.p_xdep[S.p_xrp[p] + d - W];
      ++d;
      if (lev_of[j] >= lev_of[i]) return 4;  // dependencies sit on lower levels
      if (tile_of[j] == tile_of[i]) {
        if (enc != slot_of[j] - S.tile_pbase[tile_of[i]]) return 5;
      } else {
        int sg = -1;
        for (int q = S.tile_seg[tile_of[i]]; q < S.tile_seg[tile_of[i] + 1]; ++q)
          if (p >= S.seg_rows[q] && p < S.seg_rows[q + 1]) sg = q;
        if (enc != ~j) return 5;
        // ticket order: producer tile handed out no later than the layer of i
        const int tk_i = upper ? S.ntiles - 1 - tile_of[i] : tile_of[i];
        const int tk_j = upper ? S.ntiles - 1 - tile_of[j] : tile_of[j];
        if (!S.tile_layer.empty()) {  // wavefront order: explicit layers
          if (S.tile_layer[tile_of[j]] > S.tile_layer[tile_of[i]]) return 6;
        } else {
          const int layer = S.brick[0] ? (S.grid[0] + S.brick[0] - 1) / S.brick[0] *
                                             ((S.grid[1] + S.brick[1] - 1) / S.brick[1])
                                       : 1;
          if (tk_j / layer > tk_i / layer) return 6;
        }
        bool listed = false;
        for (int w = S.seg_wptr[sg]; w < S.seg_wptr[sg + 1]; ++w) listed = listed || S.seg_wt[w] == tile_of[j];
        if (!listed) return 7;
      }
    }
    if (d != S.p_nd[p]) return 8;
  }
  return 0;
}

}  // namespace igm
