#include <cub/cub.cuh>

#include "gb_lbs.cuh"

namespace gb {

__global__ void lbs_degrees(int64_t K, const int32_t* __restrict__ ids,
                            const int64_t* __restrict__ off, int64_t* __restrict__ rowstart,
                            int64_t* __restrict__ deg) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = ids[k];
    const int64_t a = off[v], b = off[v + 1];
    rowstart[k] = a;
    deg[k] = b - a;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) deg[K] = 0;
}

__global__ void lbs_tile_first(int64_t K, const int64_t* __restrict__ S,
                               const int64_t* __restrict__ rowstart, int64_t tile,
                               int32_t* __restrict__ tile_first, int64_t* __restrict__ tile_base) {
  // one thread per TILE: binary search for the last entry whose start is <= the
  // tile's first slot (empty entries share a start with the next entry, so the
  // last one found is never empty).  Parallel over tiles, so a hub whose list
  // spans thousands of tiles costs no more than any other entry.
  const int64_t E = S[K];
  const int64_t ntiles = (E + tile - 1) / tile;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t * tile;
    int64_t lo = 0, hi = K - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (S[mid] <= e) lo = mid; else hi = mid - 1;
    }
    tile_first[t] = (int32_t)lo;
    if (tile_base) tile_base[t] = rowstart[lo] - S[lo];
  }
}

gb_status lbs_prepare(gb_ctx* ctx, Arena& ar, int64_t K, const int32_t* ids,
                      const int64_t* off, int64_t max_edges, LbsPlan* plan, int64_t tile) {
  cudaStream_t s = stream_of(ctx);
  plan->K = K;
  plan->rowstart = ar.alloc<int64_t>(K + 1);
  int64_t* deg = ar.alloc<int64_t>(K + 1);
  plan->S = ar.alloc<int64_t>(K + 1);
  plan->tile_first = ar.alloc<int32_t>(max_edges / tile + 2);
  plan->tile_base = tile == kWarpTile ? ar.alloc<int64_t>(max_edges / tile + 2) : nullptr;
  GB_ARENA_CHECK(ctx, ar);
  lbs_degrees<<<grid_for(ctx, K + 1, 256), 256, 0, s>>>(K, ids, off, plan->rowstart, deg);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, deg, plan->S, K + 1, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp, tb, deg, plan->S, K + 1, s));
  lbs_tile_first<<<grid_for(ctx, max_edges / tile + 1, 256), 256, 0, s>>>(
      K, plan->S, plan->rowstart, tile, plan->tile_first, plan->tile_base);
  GB_LAUNCH_CHECK(ctx);
  plan->grid = sm_count(ctx) * 4;
  return GB_OK;
}

}  // namespace gb
