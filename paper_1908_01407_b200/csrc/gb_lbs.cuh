// Load-balanced expansion of a frontier's adjacency lists (edge-balanced
// partitioning, the GPU form of the reference's nonzero split,
// kernels.py:133-150, applied to the push gather kernels.py:254-262).
//
// Given K frontier entries ids[0..K) and the walked orientation `off`,
// the expansion space is the concatenation of their adjacency ranges:
// E = sum_k deg(ids[k]).  It is cut into tiles of exactly TE edges; every
// CTA processes whole tiles.  Owner lookup inside a tile is a shared-memory
// table filled cooperatively (one warp per frontier entry), so each edge
// costs one LDS for its owner plus a coalesced load of its column index.
#pragma once

#include <type_traits>

#include "gb_common.cuh"

namespace gb {

constexpr int kLbsThreads = 256;
constexpr int kLbsItems = 16;
constexpr int kLbsTile = kLbsThreads * kLbsItems;  // 4096 edges per tile
constexpr int kLbsCap = kLbsTile;                  // frontier entries per tile (fast path)

// rowstart[k] = off[ids[k]], deg[k] = off[ids[k]+1] - off[ids[k]]
__global__ void lbs_degrees(int64_t K, const int32_t* __restrict__ ids,
                            const int64_t* __restrict__ off, int64_t* __restrict__ rowstart,
                            int64_t* __restrict__ deg);

// S = exclusive scan of deg (K+1 entries, S[K] = E); tile_first[t] = the
// frontier entry whose range contains edge t*TE; tile_base[t] (optional) =
// rowstart - S of that entry, so a slot e of the tile sits at tile_base + e.
__global__ void lbs_tile_first(int64_t K, const int64_t* __restrict__ S,
                               const int64_t* __restrict__ rowstart, int64_t tile,
                               int32_t* __restrict__ tile_first, int64_t* __restrict__ tile_base);

// Expansion kernel.  f(k, p, e) is called once per edge e of the expansion,
// where k is the frontier position and p the position in the orientation's
// index/value arrays.
template <class F>
__global__ void __launch_bounds__(kLbsThreads)
lbs_expand(int64_t K, const int64_t* __restrict__ S, const int64_t* __restrict__ rowstart,
           const int32_t* __restrict__ tile_first, F f) {
  __shared__ int64_t s_delta[kLbsCap];
  __shared__ uint16_t s_own[kLbsTile];
  const int64_t E = S[K];
  const int64_t ntiles = (E + kLbsTile - 1) / kLbsTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = kLbsThreads / 32;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t e0 = t * kLbsTile;
    const int64_t e1 = e0 + kLbsTile < E ? e0 + kLbsTile : E;
    const int64_t k0 = tile_first[t];
    const int64_t k1 = t + 1 < ntiles ? tile_first[t + 1] : K - 1;
    const int64_t nk = k1 - k0 + 1;
    if (nk <= kLbsCap) {
      for (int64_t i = warp; i < nk; i += nwarps) {
        const int64_t k = k0 + i;
        const int64_t sk = S[k], sk1 = S[k + 1];
        const int64_t lo = sk > e0 ? sk : e0;
        const int64_t hi = sk1 < e1 ? sk1 : e1;
        if (lane == 0) s_delta[i] = rowstart[k] - sk;
        for (int64_t e = lo + lane; e < hi; e += 32) s_own[e - e0] = (uint16_t)i;
      }
      __syncthreads();
#pragma unroll 4
      for (int r = 0; r < kLbsItems; ++r) {
        const int64_t el = (int64_t)r * kLbsThreads + threadIdx.x;
        const int64_t e = e0 + el;
        if (e < e1) {
          const int i = s_own[el];
          f(k0 + i, s_delta[i] + e, e);
        }
      }
      __syncthreads();
    } else {
      // many empty frontier entries inside one tile: binary search per edge
      for (int64_t e = e0 + threadIdx.x; e < e1; e += kLbsThreads) {
        int64_t lo = k0, hi = k1;  // largest k with S[k] <= e
        while (lo < hi) {
          int64_t mid = (lo + hi + 1) >> 1;
          if (S[mid] <= e) lo = mid; else hi = mid - 1;
        }
        f(lo, rowstart[lo] + (e - S[lo]), e);
      }
    }
  }
}

// Host helper: degrees + scan + tile_first for K frontier entries.  Leaves
// S (K+1 entries, device) so the caller can read E = S[K] if it needs it.
struct LbsPlan {
  int64_t K = 0;
  int64_t* rowstart = nullptr;
  int64_t* S = nullptr;
  int32_t* tile_first = nullptr;
  int64_t* tile_base = nullptr;  // warp tiles only
  int grid = 0;
};

gb_status lbs_prepare(gb_ctx* ctx, Arena& ar, int64_t K, const int32_t* ids,
                      const int64_t* off, int64_t max_edges, LbsPlan* plan,
                      int64_t tile = kLbsTile);

// ---------------------------------------------------------------------------
// Warp tiles: each warp owns kWarpTile consecutive expansion slots and finds
// the owner of each slot by a 5-step binary search over the (at most 32)
// frontier entries of the tile, held one per lane and read with shuffles --
// no shared memory and no block barriers.  Tiles that touch more than 32
// frontier entries (many tiny adjacency lists) walk them one lane per entry.
// f.visit(p) is called for single edges; F must also provide
//   template <int B> void batch(const int64_t (&p)[B], const bool (&live)[B])
//   template <int B> void batch2(b0, b1, st1, rel_end, h)
// for the batched paths (batch2: slots h + r*32 + lane of a tile that lies in
// at most two lists, slot e at b0 + e before st1 and at b1 + e from st1 on).
// ---------------------------------------------------------------------------
constexpr int kWarpItems = 16;
constexpr int kWarpTile = 32 * kWarpItems;  // 512 slots

// Items per batch2 round trip in the one/two-list tiles: F::kTileBatch when
// the functor names one (the BFS push: 4), else half a lane's 16 items.
template <class F, class = void>
struct tile_batch {
  static constexpr int value = kWarpItems / 2;
};
template <class F>
struct tile_batch<F, std::void_t<decltype(F::kTileBatch)>> {
  static constexpr int value = F::kTileBatch;
};

// One warp tile [e0, e1) whose slots start in frontier entries k0..k1 (tb:
// the tile descriptor's base when has_tb).  Used by warp_tiles and by the
// TMA-prefetching BFS push for the tiles it does not stage.
template <class F>
__device__ __forceinline__ void warp_tile_one(const int64_t* S, const int64_t* rowstart, bool has_tb,
                                              int64_t e0, int64_t e1, int64_t k0, int64_t k1,
                                              int64_t tb, F& f) {
  const int lane = threadIdx.x & 31;
  const int64_t nk = k1 - k0 + 1;
  if (nk <= 2) {
    // Most tiles of a power-law push level lie inside one or two adjacency
    // lists (R-MAT s24 level 2: 69 % one, 22 % two): the owner is one
    // compare per item and the loads are warp-uniform broadcasts.
    const int64_t b0 = (has_tb ? tb : rowstart[k0] - S[k0]) + e0;
    int32_t st1 = INT32_MAX;
    int64_t b1 = b0;
    if (nk == 2) {
      const int64_t s1 = S[k0 + 1];
      st1 = (int32_t)(s1 - e0);
      b1 = rowstart[k0 + 1] - s1 + e0;
    }
    const int32_t rel_end = (int32_t)(e1 - e0);
    constexpr int B = tile_batch<F>::value;
#pragma unroll
    for (int h = 0; h < kWarpItems; h += B) f.template batch2<B>(b0, b1, st1, rel_end, h * 32);
  } else if (nk <= 32) {
    // Entry j of the tile (lane j) starts at st_rel (relative to e0; the
    // first entry's start is clamped to 0).  Slot e_rel = r*32 + lane
    // grows with r, so each lane finds its first owner by a 5-step
    // shuffle search and afterwards only advances when a row boundary
    // passes (warp-uniform loop, usually zero or one step per item):
    // ~2 ALU ops per edge instead of a 64-bit search per edge.
    int32_t st_rel = INT32_MAX;
    int64_t base_l = 0;
    if (lane < nk) {
      const int64_t sk = S[k0 + lane];
      st_rel = sk > e0 ? (int32_t)(sk - e0) : 0;
      base_l = rowstart[k0 + lane] - sk;
    }
    int own = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int32_t sv = __shfl_sync(GB_FULL, st_rel, (own + step) & 31);
      if (own + step < 32 && sv <= lane) own += step;
    }
    // empty entries share their start with the next one: the search and
    // the advance both land on the last entry whose start is <= e_rel
    int32_t nxt = __shfl_sync(GB_FULL, st_rel, (own + 1) & 31);
    if (own == 31) nxt = INT32_MAX;
    int64_t base = __shfl_sync(GB_FULL, base_l, own) + e0;
    const int32_t rel_end = (int32_t)(e1 - e0);
#pragma unroll
    for (int h = 0; h < kWarpItems; h += kWarpItems / 4) {
      constexpr int B = kWarpItems / 4;  // small batches keep the kernel's register count low
      int64_t p[B];
      bool live[B];
#pragma unroll
      for (int r = 0; r < B; ++r) {
        const int32_t er = (h + r) * 32 + lane;
        live[r] = er < rel_end;
        while (__any_sync(GB_FULL, er >= nxt)) {
          const bool adv = er >= nxt;
          own += adv;
          const int32_t n2 = __shfl_sync(GB_FULL, st_rel, (own + 1) & 31);
          const int64_t b2 = __shfl_sync(GB_FULL, base_l, own & 31);
          if (adv) {
            nxt = own == 31 ? INT32_MAX : n2;
            base = b2 + e0;
          }
        }
        p[r] = base + er;
      }
      f.template batch<B>(p, live);
    }
  } else {
    // many short lists: 4 entries per lane at a time, their bounds and first
    // edges batched (one round trip for 128 entries), the rest walked
    constexpr int B = 4;
    for (int64_t i0 = 0; i0 < nk; i0 += 32 * B) {
      int32_t len[B];  // edges of the entry inside this tile
      int64_t p[B];    // position of its first edge in the tile
#pragma unroll
      for (int r = 0; r < B; ++r) {
        const int64_t i = i0 + r * 32 + lane;
        len[r] = 0;
        p[r] = 0;
        if (i < nk) {
          const int64_t k = k0 + i;
          const int64_t sk = S[k], sk1 = S[k + 1];
          const int64_t lo = sk > e0 ? sk : e0;
          const int64_t hi = sk1 < e1 ? sk1 : e1;
          len[r] = hi > lo ? (int32_t)(hi - lo) : 0;
          p[r] = rowstart[k] - sk + lo;
        }
      }
      bool live[B];
#pragma unroll
      for (int r = 0; r < B; ++r) live[r] = len[r] > 0;
      f.template batch<B>(p, live);
#pragma unroll
      for (int r = 0; r < B; ++r)
        for (int32_t j = 1; j < len[r]; ++j) f.visit(p[r] + j);
    }
  }
}

template <class F>
__device__ __forceinline__ void warp_tiles(int64_t K, const int64_t* S, const int64_t* rowstart,
                                           const int32_t* tile_first, const int64_t* tile_base,
                                           F& f) {
  const int64_t E = S[K];
  const int64_t ntiles = (E + kWarpTile - 1) / kWarpTile;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // the next tile's descriptor is loaded one tile ahead (three independent
  // loads), so a tile inside one list starts without a dependent round trip
  int32_t k0n = 0, k1n = 0;
  int64_t bn = 0;
  // a single frontier entry owns every slot: no descriptors are read (the
  // BFS device loop does not stamp them for such levels)
  const bool single = K == 1;
  if (single) {
    // one list (a BFS's first level: the source's 406 K edges at R-MAT s24)
    // in 128-slot tiles, one batch per lane: 4x the warps of 512-slot tiles
    // on a level too small to fill the GPU with those
    constexpr int kT = 128;
    const int64_t b = rowstart[0] - S[0];
    for (int64_t t = w0; t * kT < E; t += nw) {
      const int64_t e0 = t * kT;
      const int32_t rel_end = (int32_t)(E - e0 < kT ? E - e0 : kT);
      f.template batch2<kT / 32>(b + e0, b + e0, INT32_MAX, rel_end, 0);
    }
    return;
  }
  if (w0 < ntiles) {
    k0n = tile_first[w0];
    k1n = w0 + 1 < ntiles ? tile_first[w0 + 1] : (int32_t)(K - 1);
    if (tile_base) bn = tile_base[w0];
  }
  for (int64_t t = w0; t < ntiles; t += nw) {
    const int64_t e0 = t * kWarpTile;
    const int64_t e1 = e0 + kWarpTile < E ? e0 + kWarpTile : E;
    const int64_t k0 = k0n, k1 = k1n, tb = bn;
    const int64_t tn = t + nw;
    if (tn < ntiles) {
      k0n = tile_first[tn];
      k1n = tn + 1 < ntiles ? tile_first[tn + 1] : (int32_t)(K - 1);
      if (tile_base) bn = tile_base[tn];
    }
    warp_tile_one(S, rowstart, tile_base != nullptr, e0, e1, k0, k1, tb, f);
  }
}

}  // namespace gb
