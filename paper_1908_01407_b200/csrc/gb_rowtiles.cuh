// Edge-balanced (merge-path style) reduction over the rows of a CSR: the
// nonzero split of the reference's pull kernel (kernels.py:133-150) mapped
// onto warps.
//
// The work list is the COMPRESSED row set (rows with >= 1 entry, built once
// per matrix orientation: nz_rows[i], nz_off[i]); empty rows -- 30-47% of an
// R-MAT graph -- never enter a tile.  The nnz range is cut into warp tiles of
// kRowTile = 512 consecutive entries, so a tile touches at most 512 compressed
// rows.  Their starts, relative to the tile, are staged in shared memory as
// uint16; lane l then reads its 16 consecutive entries with four 16-byte
// vector loads, finds the owner of its first entry with a 9-step search in
// shared memory, and folds its entries row by row.  A row wholly inside one
// lane's chunk is stored directly; rows that cross lanes are combined by a
// warp segmented scan and written once by the lane where they end; only rows
// that cross a tile boundary use an atomic fold, so hub rows spread over as
// many warps as their length needs at one atomic per 512 entries.
//
// tile_first[t] = compressed row containing entry t*kRowTile (lbs_tile_first
// with S = nz_off).  Blocks must be 256 threads.
//
// R must provide:
//   T identity();  T load(int64_t p, int32_t col);  T fold(T acc, T x);
//   void emit(int64_t row, T acc, bool whole_row);   // whole_row: plain store ok
#pragma once

#include "gb_common.cuh"

namespace gb {

#ifndef GB_ROW_SPLIT
#define GB_ROW_SPLIT 4  // gather waves per lane and tile (PR s22 x20: 1 wave 11.7 ms, 4 waves + 48 regs 10.6 ms)
#endif

constexpr int kRowItems = 16;
constexpr int kRowTile = 32 * kRowItems;  // 512 entries per warp tile

template <class T, class R>
__device__ __forceinline__ void row_tiles(int64_t R_rows, const int32_t* __restrict__ nz_rows,
                                          const int64_t* __restrict__ nz_off,
                                          const int32_t* __restrict__ idx,
                                          const int32_t* __restrict__ tile_first, R& red) {
  __shared__ uint16_t s_st[8][kRowTile + 8];
  const int lane = threadIdx.x & 31;
  uint16_t* st = s_st[threadIdx.x >> 5];
  const int64_t E = nz_off[R_rows];
  const int64_t ntiles = (E + kRowTile - 1) / kRowTile;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = w0; t < ntiles; t += nw) {
    const int64_t e0 = t * kRowTile;
    const int64_t e1 = e0 + kRowTile < E ? e0 + kRowTile : E;
    const int64_t my0 = e0 + (int64_t)lane * kRowItems;
    const int64_t my1 = my0 + kRowItems < e1 ? my0 + kRowItems : e1;
    // column loads first: they depend on nothing but the tile position
    int32_t cols[kRowItems];
    if (my0 + kRowItems <= e1) {
      // e0 is 512-aligned: two 256-bit loads per lane
#pragma unroll
      for (int q = 0; q < kRowItems / 8; ++q) {
        int32_t v[8];
        ld_stream8(idx + my0 + 8 * q, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) cols[8 * q + j] = v[j];
      }
    } else {
#pragma unroll
      for (int q = 0; q < kRowItems; ++q) cols[q] = my0 + q < e1 ? ld_stream(idx + my0 + q) : 0;
    }
    const int64_t r0 = tile_first[t];
    const int64_t r1 = t + 1 < ntiles ? tile_first[t + 1] : R_rows - 1;
    const int nr = (int)(r1 - r0 + 1);  // <= 512: every inner row owns >= 1 entry
    // relative row starts, clamped to [0, 512]; entry nr is the end of row r1
    for (int i = lane; i <= nr; i += 32) {
      const int64_t o = nz_off[r0 + i] - e0;
      st[i] = (uint16_t)(o < 0 ? 0 : (o > kRowTile ? kRowTile : o));
    }
    __syncwarp();
    // gathers in GB_ROW_SPLIT waves (fewer registers, more resident warps)
    constexpr int kGat = kRowItems / GB_ROW_SPLIT;
    T vals[kGat];
#pragma unroll
    for (int q = 0; q < kGat; ++q)
      vals[q] = my0 + q < e1 ? red.load(my0 + q, cols[q]) : red.identity();
    // Fold row segment by row segment (rows are non-empty: one step reaches
    // the next segment).  A segment closed inside the lane is a whole row
    // (emitted with a plain store) unless it continues a row from the
    // previous lane -- the lane's "head".  Open tail segments are combined
    // across lanes by a warp segmented scan; the lane where a row ends emits
    // it once, so only rows that cross a tile boundary use an atomic.
    const bool head_out = nz_off[r0] < e0;
    const bool tail_out = nz_off[r1 + 1] > e1;
    const int rel0 = lane * kRowItems, rel1 = (int)(my1 - e0);
    T acc = red.identity(), h_acc = red.identity();
    int h_row = -1;  // tile row of the head segment (-1 none, -2 a lane inside one row)
    int cur = -1;    // tile row of the open tail segment (-1 none)
    if (my0 < e1) {
      int lo = 0, hi = nr - 1;  // owner of my first entry: last row whose start <= rel0
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (st[mid] <= rel0) lo = mid; else hi = mid - 1;
      }
      cur = lo;
      int next = st[cur + 1];
      const bool cont = st[cur] < rel0 || (cur == 0 && head_out);
      bool first = true;
#pragma unroll
      for (int q = 0; q < kRowItems; ++q) {
        if (kGat < kRowItems && q > 0 && q % kGat == 0) {
#pragma unroll
          for (int j = 0; j < kGat; ++j)
            vals[j] = my0 + q + j < e1 ? red.load(my0 + q + j, cols[q + j]) : red.identity();
        }
        const int e = rel0 + q;
        if (e < rel1 && e >= next) {
          if (first && cont) {
            h_acc = acc;
            h_row = cur;
          } else {
            red.emit(nz_rows[r0 + cur], acc, true);
          }
          first = false;
          acc = red.identity();
          ++cur;
          next = st[cur + 1];
        }
        if (e < rel1) acc = red.fold(acc, vals[q % kGat]);
      }
      if (next <= rel1 && !(cur == nr - 1 && tail_out)) {
        // the last segment ends with my chunk
        if (first && cont) {
          h_acc = acc;
          h_row = cur;
        } else {
          red.emit(nz_rows[r0 + cur], acc, !(cur == 0 && head_out));
        }
        acc = red.identity();
        cur = -1;
      } else if (first && cont) {
        h_row = -2;
      }
    }
    // segmented inclusive scan of the open tails (equal keys are adjacent lanes)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int k2 = __shfl_up_sync(GB_FULL, cur, o);
      const T v2 = __shfl_up_sync(GB_FULL, acc, o);
      if (lane >= o && cur >= 0 && k2 == cur) acc = red.fold(acc, v2);
    }
    const int pk = __shfl_up_sync(GB_FULL, cur, 1);
    const T pv = __shfl_up_sync(GB_FULL, acc, 1);
    if (h_row >= 0) {
      const T v = lane > 0 && pk == h_row ? red.fold(h_acc, pv) : h_acc;
      red.emit(nz_rows[r0 + h_row], v, !(h_row == 0 && head_out));
    }
    const int nk = __shfl_down_sync(GB_FULL, cur, 1);
    const int nh = __shfl_down_sync(GB_FULL, h_row, 1);
    if (cur >= 0 && !(lane < 31 && (nk == cur || nh == cur)))
      red.emit(nz_rows[r0 + cur], acc, false);  // runs past the tile
    __syncwarp();
  }
}

// Compressed row set of a CSR (rows with at least one entry) + tile starts.
struct RowTilesPlan {
  int64_t R = 0;                 // number of non-empty rows
  int32_t* nz_rows = nullptr;    // [R] row ids
  int64_t* nz_off = nullptr;     // [R+1] their offsets (nz_off[R] = nnz)
  int32_t* tile_first = nullptr; // [nnz/kRowTile + 2]
};

gb_status row_tiles_plan(gb_ctx* ctx, Arena& ar, int64_t n, const int64_t* off, int64_t nnz,
                         RowTilesPlan* plan);

}  // namespace gb
