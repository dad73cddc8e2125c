// pencil.hpp -- host-side record stream of the structured-grid "pencil"
// wavefront (csrc/tri_pencil.cuh).
//
// Applies to an ILU(0) triangular factor of a 7-point stencil in natural
// order on a gx x gy x gz grid: every off-diagonal entry of row (i,j,k) (in
// solve order: mirrored for the upper factor) is one of (i-1,j,k), (i,j-1,k),
// (i,j,k-1).  The substitution (ilu.cpp:122-155) is then a 3D wavefront whose
// level is i+j+k; the pencil kernel gives every thread one z-pencil (i,j,.)
// of a 16 x 16 brick and walks it one row per step, a lane's row at warp step
// s being k = s - (i mod 16) - (j mod 2): the x and y dependencies of a row
// are the values its neighbour lanes produced one step earlier (warp
// shuffles), the z dependency is the lane's own previous row.  The stream
// holds, per (brick, warp, step, lane), the row's three factor values and the
// exact reciprocal of its diagonal, so each warp step is two coalesced loads.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "fx_core.cuh"

namespace igm {

#ifndef PEN_WARPS
#define PEN_WARPS 4
#endif
constexpr int kPenWarps = PEN_WARPS;       // y-row pairs per brick
constexpr int kPenX = 16;                  // brick x extent (lanes per y-row)
constexpr int kPenY = 2 * kPenWarps;       // brick y extent
constexpr int kPenSkew = kPenX;            // max (i mod 16) + (j mod 2): steps beyond gz per warp

struct PencilStream {
  bool ok = false;
  int gx = 0, gy = 0, gz = 0, nbx = 0, nby = 0, nbricks = 0, S = 0;  // S = steps per warp
  int cy = 1;   // bricks per thread-block cluster along y (tri_pencil2.cuh)
  int pad = 0;  // idle blocks after each warp's S steps (the kernel's prefetch runs ahead)
  // [ticket][warp][step] blocks of 768 B: 32 lanes x {f_x, f_y, f_z, info}
  // (int32), then 32 lanes x the exact reciprocal of |diag| (u64)
  std::vector<std::uint64_t> blk;
  std::vector<int> brick_of_ticket;  // (by << 16) | bx, wavefront order (bx+by, then bx)
};

// info bits: sh1 | sh2 << 1 | den_neg << 8 | active << 9 | entry present toward -x, -y, -z << 10..12
inline std::int32_t pencil_info(const SDivMagic& g, bool active, int present = 0) {
  return (g.u.sh1 & 1) | ((g.u.sh2 & 127) << 1) | (g.den_neg << 8) | (active ? 1 << 9 : 0) | (present << 10);
}

// rp/ci/vals: the factor with its diagonal (dpos), natural row order; upper =
// backward substitution.  ok = false when the pattern is not the 7-point
// structure on the given grid, a factor value does not fit in int32, or a
// row has a duplicate column: the generic wavefront handles those.
inline PencilStream build_pencil_stream(int n, const int* rp, const int* ci, const std::int64_t* vals,
                                        const int* dpos, bool upper, int gx, int gy, int gz, int pad = 16,
                                        bool fp = false, int cy = 1) {
  PencilStream P;
  if (gx < 2 || gy < 2 || gz < 1 || static_cast<long long>(gx) * gy * gz != n || gx > 0xffff * kPenX ||
      gy > 0x7fff * kPenY)
    return P;
  const long long plane = static_cast<long long>(gx) * gy;
  // per solve-order row: factor values toward -x, -y, -z
  std::vector<std::int32_t> f(static_cast<size_t>(n) * 3, 0);
  std::vector<SDivMagic> dm(static_cast<size_t>(n));
  std::vector<double> dd(fp ? static_cast<size_t>(n) : 0);
  std::vector<unsigned char> pres(static_cast<size_t>(n), 0);
  for (int r = 0; r < n; ++r) {
    const long long rs = upper ? n - 1 - r : r;  // solve-order index of natural row r
    const long long i = rs % gx, j = (rs / gx) % gy, k = rs / plane;
    bool seen[3] = {false, false, false};
    for (int q = rp[r]; q < rp[r + 1]; ++q) {
      const int c = ci[q];
      if (q == dpos[r]) continue;
      if (c < 0 || c >= n) return P;
      if (upper ? c < r : c > r) continue;  // outside the triangle: never read (ilu.cpp:126-135)
      if (c == r) return P;                 // a second diagonal entry
      const long long d = rs - (upper ? n - 1 - c : c);
      int slot;
      if (d == 1 && i > 0) slot = 0;
      else if (d == gx && j > 0) slot = 1;
      else if (d == plane && k > 0) slot = 2;
      else return P;
      if (seen[slot]) return P;
      seen[slot] = true;
      pres[static_cast<size_t>(rs)] |= static_cast<unsigned char>(1 << slot);
      const std::int64_t v = vals[q];
      if (v < INT32_MIN || v > INT32_MAX) return P;
      f[static_cast<size_t>(rs) * 3 + slot] = static_cast<std::int32_t>(v);
    }
    if (dpos[r] < rp[r] || dpos[r] >= rp[r + 1] || ci[dpos[r]] != r || vals[dpos[r]] == 0) return P;
    dm[static_cast<size_t>(rs)] = make_sdiv(vals[dpos[r]]);
    if (fp) dd[static_cast<size_t>(rs)] = static_cast<double>(vals[dpos[r]]);
  }
  P.gx = gx;
  P.gy = gy;
  P.gz = gz;
  P.nbx = (gx + kPenX - 1) / kPenX;
  P.nby = (gy + kPenY - 1) / kPenY;
  // tickets: clusters of cy bricks stacked along y (cy = 1: single bricks) in
  // wavefront order (cbx + cby, then cbx), a cluster's bricks at consecutive
  // tickets by rank; the y extent is padded to whole clusters with idle bricks
  const int ncy = (P.nby + cy - 1) / cy;
  P.cy = cy;
  P.nbricks = P.nbx * ncy * cy;
  P.S = gz + kPenSkew;
  P.pad = pad;
  const int SB = P.S + pad;  // blocks per warp
  std::vector<int> clusters;
  for (int c = 0; c < P.nbx * ncy; ++c) clusters.push_back(((c / P.nbx) << 16) | (c % P.nbx));
  std::stable_sort(clusters.begin(), clusters.end(), [](int a, int b) {
    const int sa = (a & 0xffff) + (a >> 16), sb = (b & 0xffff) + (b >> 16);
    return sa != sb ? sa < sb : (a & 0xffff) < (b & 0xffff);
  });
  for (int c : clusters)
    for (int r = 0; r < cy; ++r) P.brick_of_ticket.push_back((((c >> 16) * cy + r) << 16) | (c & 0xffff));
  const size_t blocks = static_cast<size_t>(P.nbricks) * kPenWarps * SB;
  P.blk.assign(blocks * 96, 0);
  const SDivMagic one = make_sdiv(1);
  for (int t = 0; t < P.nbricks; ++t) {
    const int bx = P.brick_of_ticket[t] & 0xffff, by = P.brick_of_ticket[t] >> 16;
    for (int w = 0; w < kPenWarps; ++w)
      for (int s = 0; s < SB; ++s)
        for (int lane = 0; lane < 32; ++lane) {
          const int xl = lane & 15, jj = lane >> 4;
          const long long i = static_cast<long long>(bx) * kPenX + xl, j = static_cast<long long>(by) * kPenY + 2 * w + jj;
          const int k = s - xl - jj;
          const size_t b = (static_cast<size_t>(t) * kPenWarps + w) * SB + s;
          std::int32_t* rr = reinterpret_cast<std::int32_t*>(&P.blk[b * 96]) + lane * 4;
          std::uint64_t* mm = &P.blk[b * 96 + 64 + lane];
          if (i < gx && j < gy && k >= 0 && k < gz) {
            const size_t rs = static_cast<size_t>(k * plane + j * gx + i);
            rr[0] = f[rs * 3];
            rr[1] = f[rs * 3 + 1];
            rr[2] = f[rs * 3 + 2];
            rr[3] = pencil_info(dm[rs], true, pres[rs]);
            if (fp) std::memcpy(mm, &dd[rs], 8);
            else *mm = dm[rs].u.m;
          } else {  // idle lane-step: 0 / 1 = 0, nothing stored
            rr[3] = pencil_info(one, false);
            if (fp) {
              const double d1 = 1.0;
              std::memcpy(mm, &d1, 8);
            } else {
              *mm = one.u.m;
            }
          }
        }
  }
  P.ok = true;
  return P;
}

}  // namespace igm
