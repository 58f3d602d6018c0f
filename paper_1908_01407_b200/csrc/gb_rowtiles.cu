// Compressed row set (rows with at least one entry) for the row-tile kernels.
#include <cub/cub.cuh>

#include "gb_lbs.cuh"
#include "gb_rowtiles.cuh"

namespace gb {

__global__ void nz_rows_flags(int64_t n, const int64_t* __restrict__ off, int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = i < n && off[i + 1] > off[i] ? 1 : 0;
}

__global__ void nz_rows_fill(int64_t n, const int64_t* __restrict__ off,
                             const int32_t* __restrict__ flag, const int64_t* __restrict__ pos,
                             int32_t* __restrict__ nz_rows, int64_t* __restrict__ nz_off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) {
      nz_rows[pos[i]] = (int32_t)i;
      nz_off[pos[i]] = off[i];
    }
  if (blockIdx.x == 0 && threadIdx.x == 0) nz_off[pos[n]] = off[n];
}

gb_status row_tiles_plan(gb_ctx* ctx, Arena& ar, int64_t n, const int64_t* off, int64_t nnz,
                         RowTilesPlan* plan) {
  cudaStream_t s = stream_of(ctx);
  int32_t* flag = ar.alloc<int32_t>(n + 1);
  int64_t* pos = ar.alloc<int64_t>(n + 1);
  // caller-provided output buffers are kept (gb_row_plan_build)
  if (!plan->nz_rows) plan->nz_rows = ar.alloc<int32_t>(n + 1);
  if (!plan->nz_off) plan->nz_off = ar.alloc<int64_t>(n + 1);
  if (!plan->tile_first) plan->tile_first = ar.alloc<int32_t>(nnz / kRowTile + 2);
  GB_ARENA_CHECK(ctx, ar);
  nz_rows_flags<<<grid_for(ctx, n + 1, 256), 256, 0, s>>>(n, off, flag);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, pos, n + 1, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp, tb, flag, pos, n + 1, s));
  nz_rows_fill<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, off, flag, pos, plan->nz_rows,
                                                     plan->nz_off);
  GB_TRY(read_i64(ctx, pos + n, &plan->R));
  if (plan->R > 0)
    lbs_tile_first<<<grid_for(ctx, nnz / kRowTile + 1, 256), 256, 0, s>>>(
        plan->R, plan->nz_off, nullptr, kRowTile, plan->tile_first, nullptr);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 5);
  return GB_OK;
}

}  // namespace gb

extern "C" gb_status gb_row_plan_build(gb_ctx* ctx, const gb_csr* a, int32_t* nz_rows,
                                       int64_t* nz_off, int32_t* tile_first,
                                       int64_t* nrows_nz_host) {
  gb::Arena ar(ctx);
  gb::RowTilesPlan plan;
  plan.nz_rows = nz_rows;
  plan.nz_off = nz_off;
  plan.tile_first = tile_first;
  GB_TRY(gb::row_tiles_plan(ctx, ar, a->nrows, a->offsets, a->nnz, &plan));
  *nrows_nz_host = plan.R;
  return GB_OK;
}
