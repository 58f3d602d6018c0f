// Edge-balanced (merge-path style) reduction over ALL rows of a CSR: the
// nonzero split of the reference's pull kernel (kernels.py:133-150) mapped
// onto warps.  The nnz range is cut into tiles of kRowTile consecutive
// entries; lane l of the warp owning a tile reads the 16 consecutive entries
// [e0 + 16 l, e0 + 16 l + 16) -- four 16-byte vector loads of column indices
// -- and folds them per row.  A row wholly inside one lane's chunk is stored
// directly; partial rows are combined with an atomic fold, so hub rows of
// power-law graphs spread over as many warps as their length needs.
//
// The tile's row starts (at most 33) are staged in shared memory, so finding
// the owner of an entry is a 5-step search and walking row boundaries is one
// LDS per boundary.  Tiles touching more than 32 rows fall back to one lane
// per row.  tile_first[t] = the row containing entry t*kRowTile
// (lbs_tile_first with S = offsets).  Blocks must be 256 threads.
//
// R must provide:
//   T identity();  T load(int64_t p, int32_t col);  T fold(T acc, T x);
//   void emit(int64_t row, T acc, bool whole_row);   // whole_row: plain store ok
#pragma once

#include "gb_common.cuh"

namespace gb {

constexpr int kRowItems = 16;
constexpr int kRowTile = 32 * kRowItems;  // 512 entries per warp tile

template <class T, class R>
__device__ __forceinline__ void row_tiles(int64_t nrows, const int64_t* __restrict__ off,
                                          const int32_t* __restrict__ idx,
                                          const int32_t* __restrict__ tile_first, R& red) {
  __shared__ int64_t s_st[8][33];
  const int lane = threadIdx.x & 31;
  int64_t* st = s_st[threadIdx.x >> 5];
  const int64_t E = off[nrows];
  const int64_t ntiles = (E + kRowTile - 1) / kRowTile;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = w0; t < ntiles; t += nw) {
    const int64_t e0 = t * kRowTile;
    const int64_t e1 = e0 + kRowTile < E ? e0 + kRowTile : E;
    const int64_t r0 = tile_first[t];
    const int64_t r1 = t + 1 < ntiles ? tile_first[t + 1] : nrows - 1;
    const int64_t nr = r1 - r0 + 1;
    if (nr <= 32) {
      st[lane] = lane <= nr ? off[r0 + lane] : INT64_MAX;
      if (lane == 0) st[32] = nr == 32 ? off[r0 + 32] : INT64_MAX;
      __syncwarp();
      const int64_t my0 = e0 + (int64_t)lane * kRowItems;
      const int64_t my1 = my0 + kRowItems < e1 ? my0 + kRowItems : e1;
      int32_t cols[kRowItems];
      if (my0 + kRowItems <= e1) {
        const int4* p4 = reinterpret_cast<const int4*>(idx + my0);  // e0 is 512-aligned
#pragma unroll
        for (int q = 0; q < kRowItems / 4; ++q) {
          int4 v;
          asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p4 + q));
          cols[4 * q] = v.x; cols[4 * q + 1] = v.y; cols[4 * q + 2] = v.z; cols[4 * q + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < kRowItems; ++q) cols[q] = my0 + q < e1 ? ld_stream(idx + my0 + q) : 0;
      }
      T vals[kRowItems];
#pragma unroll
      for (int q = 0; q < kRowItems; ++q)
        vals[q] = my0 + q < e1 ? red.load(my0 + q, cols[q]) : red.identity();
      if (my0 < e1) {
        // owner of my first entry: last row whose start <= my0 (empty rows
        // share their start with the next row; the last one is non-empty)
        int cur = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1)
          if (cur + step <= 32 && st[cur + step] <= my0) cur += step;
        int64_t row_start = st[cur];
        int64_t next = st[cur + 1];
        T acc = red.identity();
        bool any = false;
#pragma unroll
        for (int q = 0; q < kRowItems; ++q) {
          const int64_t e = my0 + q;
          if (e < my1) {
            while (e >= next) {
              if (any) red.emit(r0 + cur, acc, row_start >= my0 && next <= my1);
              acc = red.identity();
              any = false;
              ++cur;
              row_start = next;
              next = st[cur + 1];
            }
            acc = red.fold(acc, vals[q]);
            any = true;
          }
        }
        if (any) red.emit(r0 + cur, acc, row_start >= my0 && next <= my1);
      }
      __syncwarp();
    } else {
      // many short rows in this tile: one lane per row (partial first/last rows)
      for (int64_t i = lane; i < nr; i += 32) {
        const int64_t r = r0 + i;
        const int64_t a = off[r], b = off[r + 1];
        const int64_t lo = a > e0 ? a : e0;
        const int64_t hi = b < e1 ? b : e1;
        if (hi <= lo) continue;
        T acc = red.identity();
        for (int64_t p = lo; p < hi; ++p) acc = red.fold(acc, red.load(p, ld_stream(idx + p)));
        red.emit(r, acc, lo == a && hi == b);
      }
    }
  }
}

}  // namespace gb
