// Vector storage conversions and masks.
//   gb_count_ne      Vector.nvals_for       containers.py:179-182
//   gb_compact       Vector.to_sparse       containers.py:242-252
//   gb_scatter_dense Vector.to_dense        containers.py:230-240
//   gb_mask_bitmap   _effective_mask        kernels.py:67-84
#include <string.h>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "gb_common.cuh"

namespace gb {

template <class T>
__global__ void count_ne_kernel(int64_t n, const T* __restrict__ v, T zero,
                                unsigned long long* __restrict__ out) {
  long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += v[i] != zero;
  c = warp_sum_ll(c);
  if (lane_id() == 0 && c) atomicAdd(out, (unsigned long long)c);
}

template <class T>
struct NotZeroAt {
  const T* v;
  T zero;
  __device__ bool operator()(int64_t i) const { return v[i] != zero; }
};

template <class T>
__global__ void gather_compacted(int64_t cnt, const int64_t* __restrict__ pos,
                                 const int32_t* __restrict__ idx, const T* __restrict__ vals,
                                 int32_t* __restrict__ out_idx, T* __restrict__ out_vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = pos[i];
    out_idx[i] = idx ? idx[p] : (int32_t)p;
    out_vals[i] = vals[p];
  }
}

template <class T>
__global__ void fill_kernel(int64_t n, T v, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v;
}

template <class T>
__global__ void scatter_kernel(int64_t k, const int32_t* __restrict__ idx,
                               const T* __restrict__ vals, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x)
    out[idx[i]] = vals[i];
}

template <class T>
__global__ void mask_dense_kernel(int64_t n, const T* __restrict__ v, int complement,
                                  uint32_t* __restrict__ out) {
  const int64_t W = (n + 31) / 32;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b) {
      int64_t i = w * 32 + b;
      if (i < n && v[i] != (T)0) bits |= 1u << b;
    }
    if (complement) bits = ~bits;
    int64_t rem = n - w * 32;
    if (rem < 32) bits &= (1u << rem) - 1u;
    out[w] = bits;
  }
}

template <class T>
__global__ void mask_sparse_kernel(int64_t k, const int32_t* __restrict__ idx,
                                   const T* __restrict__ v, uint32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x)
    if (v[i] != (T)0) atomicOr(&out[idx[i] >> 5], 1u << (idx[i] & 31));
}

__global__ void complement_kernel(int64_t n, uint32_t* __restrict__ bm) {
  const int64_t W = (n + 31) / 32;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bits = ~bm[w];
    int64_t rem = n - w * 32;
    if (rem < 32) bits &= (1u << rem) - 1u;
    bm[w] = bits;
  }
}

__global__ void nonempty_kernel(int64_t n, const int64_t* __restrict__ off,
                                uint32_t* __restrict__ out) {
  const int64_t W = (n + 31) / 32;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bits = 0;
    int64_t prev = off[w * 32];
    for (int b = 0; b < 32; ++b) {
      int64_t i = w * 32 + b;
      if (i >= n) break;
      int64_t nx = off[i + 1];
      if (nx > prev) bits |= 1u << b;
      prev = nx;
    }
    out[w] = bits;
  }
}

template <class T>
static gb_status compact_t(gb_ctx* ctx, int64_t n, int64_t k, const int32_t* idx,
                           const T* vals, T zero, int32_t* out_idx, T* out_vals,
                           int64_t* count) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const bool dense = k < 0;  // k < 0: dense input (n values); else k sparse entries
  if (dense) idx = nullptr;
  int64_t len = dense ? n : k;
  if (len == 0) { *count = 0; return GB_OK; }
  int64_t* pos = ar.alloc<int64_t>(len);
  int64_t* cnt = ar.alloc<int64_t>(1);
  GB_ARENA_CHECK(ctx, ar);
  thrust::counting_iterator<int64_t> it(0);
  NotZeroAt<T> pred{vals, zero};
  size_t tb = 0;
  cub::DeviceSelect::If(nullptr, tb, it, pos, cnt, len, pred, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceSelect::If(tmp, tb, it, pos, cnt, len, pred, s));
  int64_t c = 0;
  GB_TRY(read_i64(ctx, cnt, &c));
  if (c)
    gather_compacted<T><<<grid_for(ctx, c, 256), 256, 0, s>>>(c, pos, idx, vals, out_idx, out_vals);
  GB_LAUNCH_CHECK(ctx);
  *count = c;
  return GB_OK;
}

}  // namespace gb

using namespace gb;

extern "C" {

gb_status gb_count_ne(gb_ctx* ctx, int64_t n, const void* vals, int32_t dtype,
                      const void* zero_host, int64_t* count) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  int64_t* c = ar.alloc<int64_t>(1);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(c, 0, 8, s));
  if (n > 0) {
    if (dtype == GB_I64)
      count_ne_kernel<int64_t><<<grid_for(ctx, n, 256), 256, 0, s>>>(
          n, (const int64_t*)vals, *(const int64_t*)zero_host, (unsigned long long*)c);
    else
      count_ne_kernel<double><<<grid_for(ctx, n, 256), 256, 0, s>>>(
          n, (const double*)vals, *(const double*)zero_host, (unsigned long long*)c);
    GB_LAUNCH_CHECK(ctx);
  }
  return read_i64(ctx, c, count);
}

gb_status gb_compact(gb_ctx* ctx, int64_t n, int64_t k, const int32_t* idx, const void* vals,
                     int32_t dtype, const void* zero_host, int32_t* out_idx, void* out_vals,
                     int64_t* count) {
  if (dtype == GB_I64)
    return compact_t<int64_t>(ctx, n, k, idx, (const int64_t*)vals, *(const int64_t*)zero_host,
                              out_idx, (int64_t*)out_vals, count);
  return compact_t<double>(ctx, n, k, idx, (const double*)vals, *(const double*)zero_host,
                           out_idx, (double*)out_vals, count);
}

gb_status gb_scatter_dense(gb_ctx* ctx, int64_t n, int64_t k, const int32_t* idx,
                           const void* vals, int32_t dtype, const void* zero_host,
                           void* out_vals) {
  cudaStream_t s = stream_of(ctx);
  if (dtype == GB_I64) {
    if (n) fill_kernel<int64_t><<<grid_for(ctx, n, 256), 256, 0, s>>>(n, *(const int64_t*)zero_host, (int64_t*)out_vals);
    if (k) scatter_kernel<int64_t><<<grid_for(ctx, k, 256), 256, 0, s>>>(k, idx, (const int64_t*)vals, (int64_t*)out_vals);
  } else {
    if (n) fill_kernel<double><<<grid_for(ctx, n, 256), 256, 0, s>>>(n, *(const double*)zero_host, (double*)out_vals);
    if (k) scatter_kernel<double><<<grid_for(ctx, k, 256), 256, 0, s>>>(k, idx, (const double*)vals, (double*)out_vals);
  }
  GB_LAUNCH_CHECK(ctx);
  return GB_OK;
}

gb_status gb_mask_bitmap(gb_ctx* ctx, int64_t n, int64_t k, const int32_t* idx,
                         const void* vals, int32_t dtype, int32_t complement, uint32_t* out) {
  cudaStream_t s = stream_of(ctx);
  int64_t W = (n + 31) / 32;
  if (W == 0) return GB_OK;
  if (k < 0) {  // dense mask of n values
    if (dtype == GB_I64)
      mask_dense_kernel<int64_t><<<grid_for(ctx, W, 256), 256, 0, s>>>(n, (const int64_t*)vals, complement, out);
    else
      mask_dense_kernel<double><<<grid_for(ctx, W, 256), 256, 0, s>>>(n, (const double*)vals, complement, out);
  } else {
    GB_CUDA(ctx, cudaMemsetAsync(out, 0, sizeof(uint32_t) * W, s));
    if (k) {
      if (dtype == GB_I64)
        mask_sparse_kernel<int64_t><<<grid_for(ctx, k, 256), 256, 0, s>>>(k, idx, (const int64_t*)vals, out);
      else
        mask_sparse_kernel<double><<<grid_for(ctx, k, 256), 256, 0, s>>>(k, idx, (const double*)vals, out);
    }
    if (complement) complement_kernel<<<grid_for(ctx, W, 256), 256, 0, s>>>(n, out);
  }
  GB_LAUNCH_CHECK(ctx);
  return GB_OK;
}

gb_status gb_nonempty_rows(gb_ctx* ctx, int64_t n, const int64_t* offsets, uint32_t* out) {
  cudaStream_t s = stream_of(ctx);
  int64_t W = (n + 31) / 32;
  if (W) nonempty_kernel<<<grid_for(ctx, W, 256), 256, 0, s>>>(n, offsets, out);
  GB_LAUNCH_CHECK(ctx);
  return GB_OK;
}

}  // extern "C"

namespace gb {
__global__ void popc_kernel(int64_t W, const uint32_t* __restrict__ bm,
                            unsigned long long* __restrict__ out) {
  long long c = 0;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x)
    c += __popc(bm[w]);
  c = warp_sum_ll(c);
  if (lane_id() == 0 && c) atomicAdd(out, (unsigned long long)c);
}
}  // namespace gb

extern "C" gb_status gb_bitmap_count(gb_ctx* ctx, int64_t n, const uint32_t* bm, int64_t* count) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  int64_t* c = ar.alloc<int64_t>(1);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(c, 0, 8, s));
  const int64_t W = (n + 31) / 32;
  if (W) popc_kernel<<<grid_for(ctx, W, 256), 256, 0, s>>>(W, bm, (unsigned long long*)c);
  GB_LAUNCH_CHECK(ctx);
  return read_i64(ctx, c, count);
}
