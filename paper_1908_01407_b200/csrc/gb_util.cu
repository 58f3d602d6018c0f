// Element-wise utilities of the operator layer and the composed algorithms
// (what would otherwise be eager PyTorch ops on the device arrays):
//   gb_iota            arange                       (kernels.py:586-639 index vectors)
//   gb_cast            dtype conversion             (numpy astype; result_type promotions)
//   gb_select_flags    boolean compaction           (kernels.py:598-604 present entries)
//   gb_gather_i32      value gather by int32 index  (kernels.py:544-559)
//   gb_edges_clean     drop self loops + mirror     (io.py:220-249 weighted edges)
//   gb_scale_rows      alpha / outdeg per entry     (algorithms.py:122-129)
//   gb_lower_by_rank   degree-ranked lower triangle (algorithms.py:206-218)
// Dtype codes: GB_I64 = 0, GB_F64 = 1, GB_I32 = 2 (index vectors).
#include <cub/cub.cuh>

#include "gb_common.cuh"

namespace gb {

constexpr int kI32 = 2;

__global__ void iota_kernel(int64_t n, int code, void* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (code == kI32) static_cast<int32_t*>(out)[i] = (int32_t)i;
    else if (code == GB_I64) static_cast<int64_t*>(out)[i] = i;
    else static_cast<double*>(out)[i] = (double)i;
  }
}

__device__ __forceinline__ double load_as_f64(const void* p, int code, int64_t i) {
  if (code == kI32) return (double)static_cast<const int32_t*>(p)[i];
  if (code == GB_I64) return (double)static_cast<const int64_t*>(p)[i];
  return static_cast<const double*>(p)[i];
}
__device__ __forceinline__ int64_t load_as_i64(const void* p, int code, int64_t i) {
  if (code == kI32) return static_cast<const int32_t*>(p)[i];
  if (code == GB_I64) return static_cast<const int64_t*>(p)[i];
  // numpy float -> int astype: truncation toward zero (finite values)
  return (int64_t)static_cast<const double*>(p)[i];
}

__global__ void cast_kernel(int64_t n, int in_code, const void* in, int out_code, void* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (out_code == GB_F64) static_cast<double*>(out)[i] = load_as_f64(in, in_code, i);
    else if (out_code == GB_I64) static_cast<int64_t*>(out)[i] = load_as_i64(in, in_code, i);
    else static_cast<int32_t*>(out)[i] = (int32_t)load_as_i64(in, in_code, i);
  }
}

template <class T>
__global__ void select_kernel(int64_t k, const int32_t* __restrict__ flags,
                              const int64_t* __restrict__ pos, const int32_t* __restrict__ idx,
                              const T* __restrict__ vals, int32_t* __restrict__ out_idx,
                              T* __restrict__ out_vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flags[i]) {
      const int64_t p = pos[i];
      if (out_idx) out_idx[p] = idx ? idx[i] : (int32_t)i;
      if (out_vals) out_vals[p] = vals[i];
    }
}

template <class T>
__global__ void gather_i32_kernel(int64_t k, const int32_t* __restrict__ tgt,
                                  const T* __restrict__ src, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[tgt[i]];
}

// keep (src, dst, w) with src != dst; optionally append the mirror.  flags
// and the scan come from the caller; out arrays hold 2*kept when mirrored.
__global__ void edges_clean_kernel(int64_t m, const int32_t* __restrict__ src,
                                   const int32_t* __restrict__ dst, const double* __restrict__ w,
                                   const int64_t* __restrict__ pos, int64_t kept, int mirror,
                                   int64_t* __restrict__ os, int64_t* __restrict__ od,
                                   double* __restrict__ ow) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = src[i], b = dst[i];
    if (a == b) continue;
    const int64_t p = pos[i];
    os[p] = a;
    od[p] = b;
    if (ow) ow[p] = w[i];
    if (mirror) {
      os[kept + p] = b;
      od[kept + p] = a;
      if (ow) ow[kept + p] = w[i];
    }
  }
}

__global__ void not_loop_flags(int64_t m, const int32_t* __restrict__ src,
                               const int32_t* __restrict__ dst, int32_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = src[i] != dst[i];
}

// entry-wise alpha / outdeg(row): a warp per row
__global__ void scale_rows_kernel(int64_t n, const int64_t* __restrict__ off, double alpha,
                                  double* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n; r += nw) {
    const int64_t lo = off[r], hi = off[r + 1];
    if (hi == lo) continue;
    const double s = alpha / (double)(hi - lo);
    for (int64_t p = lo + lane; p < hi; p += 32) vals[p] = s;
  }
}

__global__ void degree_keys(int64_t n, const int64_t* __restrict__ off,
                            int64_t* __restrict__ deg, int32_t* __restrict__ id) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    deg[i] = off[i + 1] - off[i];
    id[i] = (int32_t)i;
  }
}

__global__ void rank_of_order(int64_t n, const int32_t* __restrict__ order,
                             int32_t* __restrict__ position) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    position[order[i]] = (int32_t)i;
}

// flags[p] = position[row(p)] > position[col(p)]; a warp per row
__global__ void lower_flags(int64_t n, const int64_t* __restrict__ off,
                            const int32_t* __restrict__ idx, const int32_t* __restrict__ position,
                            int32_t* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n; r += nw) {
    const int32_t pr = position[r];
    for (int64_t p = off[r] + lane; p < off[r + 1]; p += 32) flags[p] = pr > position[idx[p]];
  }
}

__global__ void lower_fill(int64_t n, const int64_t* __restrict__ off,
                           const int32_t* __restrict__ idx, const void* vals, int dtype,
                           int64_t iso_i, double iso_f, const int32_t* __restrict__ position,
                           const int32_t* __restrict__ flags, const int64_t* __restrict__ pos,
                           int64_t* __restrict__ orow, int64_t* __restrict__ ocol, void* ovals) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n; r += nw) {
    const int32_t pr = position[r];
    for (int64_t p = off[r] + lane; p < off[r + 1]; p += 32) {
      if (!flags[p]) continue;
      const int64_t q = pos[p];
      orow[q] = pr;
      ocol[q] = position[idx[p]];
      if (dtype == GB_I64)
        static_cast<int64_t*>(ovals)[q] = vals ? static_cast<const int64_t*>(vals)[p] : iso_i;
      else
        static_cast<double*>(ovals)[q] = vals ? static_cast<const double*>(vals)[p] : iso_f;
    }
  }
}

// exclusive scan of int32 flags into int64 positions; returns the total
static gb_status flag_scan(gb_ctx* ctx, Arena& ar, int64_t k, const int32_t* flags, int64_t** pos,
                           int64_t* total) {
  cudaStream_t s = stream_of(ctx);
  int64_t* p = ar.alloc<int64_t>(k + 1);
  GB_ARENA_CHECK(ctx, ar);
  // flags are 0/1: scan a widened copy (int64 positions)
  int64_t* wide = ar.alloc<int64_t>(k + 1);
  GB_ARENA_CHECK(ctx, ar);
  cast_kernel<<<grid_for(ctx, k, 256), 256, 0, s>>>(k, kI32, flags, GB_I64, wide);
  GB_CUDA(ctx, cudaMemsetAsync(wide + k, 0, sizeof(int64_t), s));
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, wide, p, k + 1, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp, tb, wide, p, k + 1, s));
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 3);
  GB_TRY(read_i64(ctx, p + k, total));
  *pos = p;
  return GB_OK;
}

}  // namespace gb

using namespace gb;

extern "C" {

gb_status gb_iota(gb_ctx* ctx, int32_t code, int64_t n, void* out) {
  if (n <= 0) return GB_OK;
  iota_kernel<<<grid_for(ctx, n, 256), 256, 0, stream_of(ctx)>>>(n, code, out);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

gb_status gb_cast(gb_ctx* ctx, int64_t n, int32_t in_code, const void* in, int32_t out_code,
                  void* out) {
  if (n <= 0) return GB_OK;
  cast_kernel<<<grid_for(ctx, n, 256), 256, 0, stream_of(ctx)>>>(n, in_code, in, out_code, out);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

gb_status gb_select_flags(gb_ctx* ctx, int64_t k, const int32_t* flags, const int32_t* idx,
                          const void* vals, int32_t dtype, int32_t* out_idx, void* out_vals,
                          int64_t* count_host) {
  *count_host = 0;
  if (k <= 0) return GB_OK;
  Arena ar(ctx);
  int64_t* pos;
  GB_TRY(flag_scan(ctx, ar, k, flags, &pos, count_host));
  cudaStream_t s = stream_of(ctx);
  if (dtype == GB_F64)
    select_kernel<double><<<grid_for(ctx, k, 256), 256, 0, s>>>(
        k, flags, pos, idx, (const double*)vals, out_idx, (double*)out_vals);
  else
    select_kernel<int64_t><<<grid_for(ctx, k, 256), 256, 0, s>>>(
        k, flags, pos, idx, (const int64_t*)vals, out_idx, (int64_t*)out_vals);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

gb_status gb_gather_i32(gb_ctx* ctx, int32_t dtype, int64_t k, const int32_t* tgt,
                        const void* src, void* out) {
  if (k <= 0) return GB_OK;
  cudaStream_t s = stream_of(ctx);
  if (dtype == GB_F64)
    gather_i32_kernel<double><<<grid_for(ctx, k, 256), 256, 0, s>>>(k, tgt, (const double*)src,
                                                                    (double*)out);
  else if (dtype == GB_I64)
    gather_i32_kernel<int64_t><<<grid_for(ctx, k, 256), 256, 0, s>>>(k, tgt, (const int64_t*)src,
                                                                     (int64_t*)out);
  else
    gather_i32_kernel<int32_t><<<grid_for(ctx, k, 256), 256, 0, s>>>(k, tgt, (const int32_t*)src,
                                                                     (int32_t*)out);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

gb_status gb_edges_clean(gb_ctx* ctx, int64_t m, const int32_t* src, const int32_t* dst,
                         const double* w, int32_t mirror, int64_t* out_src, int64_t* out_dst,
                         double* out_w, int64_t* count_host) {
  *count_host = 0;
  if (m <= 0) return GB_OK;
  Arena ar(ctx);
  int32_t* flags = ar.alloc<int32_t>(m);
  GB_ARENA_CHECK(ctx, ar);
  cudaStream_t s = stream_of(ctx);
  not_loop_flags<<<grid_for(ctx, m, 256), 256, 0, s>>>(m, src, dst, flags);
  int64_t* pos;
  int64_t kept = 0;
  GB_TRY(flag_scan(ctx, ar, m, flags, &pos, &kept));
  edges_clean_kernel<<<grid_for(ctx, m, 256), 256, 0, s>>>(m, src, dst, w, pos, kept, mirror,
                                                           out_src, out_dst, out_w);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 2);
  *count_host = mirror ? 2 * kept : kept;
  return GB_OK;
}

gb_status gb_scale_rows(gb_ctx* ctx, int64_t n, const int64_t* offsets, double alpha,
                        double* vals) {
  if (n <= 0) return GB_OK;
  scale_rows_kernel<<<grid_for(ctx, n * 32, 256, 8), 256, 0, stream_of(ctx)>>>(n, offsets, alpha,
                                                                              vals);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

gb_status gb_lower_by_rank(gb_ctx* ctx, const gb_csr* a, int64_t* out_rows, int64_t* out_cols,
                           void* out_vals, int64_t* count_host) {
  *count_host = 0;
  const int64_t n = a->nrows, m = a->nnz;
  if (n == 0 || m == 0) return GB_OK;
  cudaStream_t s = stream_of(ctx);
  Arena ar(ctx);
  int64_t* deg = ar.alloc<int64_t>(n);
  int64_t* deg2 = ar.alloc<int64_t>(n);
  int32_t* id = ar.alloc<int32_t>(n);
  int32_t* order = ar.alloc<int32_t>(n);
  int32_t* position = ar.alloc<int32_t>(n);
  int32_t* flags = ar.alloc<int32_t>(m);
  GB_ARENA_CHECK(ctx, ar);
  degree_keys<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, a->offsets, deg, id);
  // stable ascending sort by degree (radix sort is stable): numpy argsort(kind="stable")
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, deg, deg2, id, order, n, 0, 64, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceRadixSort::SortPairs(tmp, tb, deg, deg2, id, order, n, 0, 64, s));
  rank_of_order<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, order, position);
  lower_flags<<<grid_for(ctx, n * 32, 256, 8), 256, 0, s>>>(n, a->offsets, a->indices, position,
                                                            flags);
  int64_t* pos;
  GB_TRY(flag_scan(ctx, ar, m, flags, &pos, count_host));
  lower_fill<<<grid_for(ctx, n * 32, 256, 8), 256, 0, s>>>(
      n, a->offsets, a->indices, a->values, a->dtype, a->iso_i64, a->iso_f64, position, flags, pos,
      out_rows, out_cols, out_vals);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 5);
  return GB_OK;
}

}  // extern "C"
