// raster.cuh -- order in which the CTAs of a tiled contraction visit the tiles of c.
//
// The hardware dispatches CTAs in linear order (blockIdx.x fastest).  With a plain (x, y) -> (column
// tile, row tile) mapping the CTAs resident at one time form a thin strip: a few tile-rows of a against
// ALL of bt, so every strip streams the whole of bt from HBM again (measured at N = 4096 FP64 with 64 x 64
// tiles: 3.97 GB of DRAM traffic per launch against 0.54 GB algorithmic).  Grouped order sweeps `group`
// tile-rows column by column: the resident set is a near-square block, the group's rows of a stay in
// the 126 MB L2 for the whole sweep and bt is streamed once per group instead of once per strip.
#pragma once

namespace mmx {

// linear dispatch index `lin` over a gx x gy grid of tiles -> (bx, by)
__device__ __forceinline__ void raster_map(int group, int gx, int gy, int lin, int& bx, int& by) {
  if (group <= 1 || gy == 1) {
    bx = lin % gx;
    by = lin / gx;
    return;
  }
  const int per_group = group * gx;
  const int grp = lin / per_group;
  const int first = grp * group;
  const int h = min(group, gy - first);  // the last group may be shorter
  const int in = lin - grp * per_group;
  by = first + in % h;
  bx = in / h;
}

// (bx, by) = tile column / tile row served by this CTA; gridDim = (tile columns, tile rows)
__device__ __forceinline__ void raster_tile(int group, int& bx, int& by) {
  const int gx = static_cast<int>(gridDim.x), gy = static_cast<int>(gridDim.y);
  raster_map(group, gx, gy, static_cast<int>(blockIdx.y) * gx + static_cast<int>(blockIdx.x), bx, by);
}

// Tile-rows per group (16, measured; MMX_RASTER_GROUP overrides).
int raster_group(int tile_m, size_t row_bytes);

}  // namespace mmx
