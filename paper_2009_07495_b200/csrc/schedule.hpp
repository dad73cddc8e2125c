// schedule.hpp -- host-side wavefront schedule of one ILU triangular factor.
//
// Built once at upload (igm_upload_ilu); pure host C++ so it is unit-testable
// on the CPU.  The factor's rows are partitioned into TILES; a CTA owns one
// tile, keeps the tile's solution values in shared memory, and walks the tile
// level by level (level = depth in the substitution DAG).  Cross-tile
// dependencies go through global memory with per-tile progress words.
//
// Tiling.  When the pattern is a structured-grid stencil in natural order
// (every dependency a +-1 neighbour of an inferred gx x gy x gz grid), tiles
// are cube-ish bricks: most of the 3*g DAG chain then stays inside shared
// memory, and a monotone path crosses only ~(gx/Bi + gy/Bj + gz/Bk) brick
// faces instead of one tile boundary per level.  Otherwise tiles are
// contiguous row blocks.  Either way the tile order handed out by the ticket
// counter is layer-major (z-layers of bricks, or row blocks), every
// dependency points to the same or an earlier layer, and no layer has more
// tiles than can be co-resident, which makes the spin-waits deadlock-free.
#pragma once

#include <cstdint>
#include <vector>

namespace igm {

struct TriSchedule {
  int n = 0, ntiles = 0, nlevels = 0, maxd = 0, stride = 0;  // stride = register deps per slot
  int grid[3] = {0, 0, 0};   // inferred grid (0 = unstructured)
  int brick[3] = {0, 0, 0};
  int tile_cap = 0;          // max rows per tile (shared memory slots)
  int max_tile_rows = 0;     // largest tile actually built
  std::vector<int> tile_layer;  // wavefront ticket order: layer of each tile (empty: z-layers)
  bool acyclic = false;         // every cross-tile dependency points to a strictly earlier ticket
  std::vector<int> tile_pbase;  // ntiles+1: first schedule slot of each tile
  std::vector<int> tile_seg;    // ntiles+1: first segment of each tile
  std::vector<int> seg_level;   // per segment (one DAG level of one tile)
  std::vector<int> seg_rows;    // nseg+1: first slot of each segment
  std::vector<int> seg_wptr;    // nseg+1 into seg_wt
  std::vector<int> seg_wt;      // producer tiles a segment waits on
  // per schedule slot p
  std::vector<int> p_row, p_nd;
  std::vector<int> p_dep;            // n*stride: >= 0 tile-local slot, < 0 ~global row
  std::vector<std::int64_t> p_val;   // n*stride
  std::vector<int> p_xrp;            // n+1: dependencies beyond `stride` (CSR)
  std::vector<int> p_xdep;
  std::vector<std::int64_t> p_xval;
  std::vector<std::uint64_t> p_mag;  // exact reciprocal of |diag|
  std::vector<int> p_info;  // sh1 | sh2<<1 | neg<<8 | (diag==-1)<<9 | exported<<10
  std::vector<std::int64_t> p_diag;
  // the same per-slot data as one packed record (what the kernel streams):
  //   int32 row, nd, info, xb | u64 mag | i64 diag | int32 dep[stride] | i64 val[stride]
  int rec_bytes = 0;                 // 32 + 12*stride (multiple of 16)
  // compact records (every factor value fits in int32, nd <= 255):
  //   int32 row | int32 info | (nd << 16) | u64 mag | int32 dep[stride] | int32 val[stride]
  // = 16 + 8*stride bytes; the rare extra-dependency index is read from p_xrp
  // and the FP path's diagonal from p_diag
  bool compact = false;
  std::vector<unsigned char> p_rec;  // n * rec_bytes
  // cross-tile dependencies of each segment: distinct producer rows; a
  // record's external dependency is encoded as ~(index into this list)
  std::vector<int> seg_xptr;  // nseg+1
  std::vector<int> seg_xrow;
  int max_seg_ext = 0;
  // the stripped factor in natural row order (checked-mode counting pass)
  std::vector<int> c_rp, c_ci;
  std::vector<std::int64_t> c_val, c_diag;
};

constexpr int kTriSegRows = 256;  // rows per segment (one per compute thread)

// rp/ci/vals: the factor (diagonal included); dpos: diagonal slot per row.
// upper = backward substitution.  Throws std::invalid_argument on bad input.
TriSchedule build_tri_schedule(int n, const int* rp, const int* ci, const std::int64_t* vals,
                               const int* dpos, bool upper, int num_sms, int tile_cap_override);

// shared-memory tile capacity (rows) for a dependency stride
inline int tri_tile_cap(int stride) { return stride <= 8 ? 16384 : 8192; }

// Structural check of a schedule (CPU tests): every row scheduled once,
// levels ascending inside a tile, tile-local dependencies resolved at a lower
// level of the same tile, cross-tile dependencies covered by the segment's
// wait list and pointing at the same or an earlier ticket layer.  Returns 0
// when valid, otherwise the number of the first failed property.
int validate_tri_schedule(const TriSchedule& S, const int* rp, const int* ci, bool upper);

}  // namespace igm
