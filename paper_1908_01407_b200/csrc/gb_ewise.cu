// Element-wise, assign, scatter/gather, apply and reduce kernels.
//
//   gb_ewise_dense      ewise_add / ewise_mult on dense operands   kernels.py:432-448, 468-478, 504-512
//   gb_union_sparse     ewise_add sparse+sparse (concat, stable sort, fold)  kernels.py:454-466
//   gb_intersect_sparse ewise_mult sparse*sparse                   kernels.py:489-494
//   gb_gather_pair      ewise_mult sparse*dense                    kernels.py:495-502
//   gb_filter_mask      _mask_sparse_result                        kernels.py:414-419
//   gb_assign_scalar    assign                                     kernels.py:519-535
//   gb_scatter_min      assign_scatter                             kernels.py:538-583
//   gb_gather / gb_gather_sparse   extract_gather                  kernels.py:586-619
//   gb_apply_affine     apply with an affine map                   kernels.py:622-639
//   gb_reduce           reduce / reduce_scalar_matrix              kernels.py:642-647, 663-665
//   gb_reduce_rows      reduce_rows                                kernels.py:650-660
#include <string.h>

#include <cub/cub.cuh>

#include "gb_common.cuh"

namespace gb {

template <class T>
__device__ __forceinline__ bool allowed(const uint32_t* m, int64_t i) {
  return !m || ((m[i >> 5] >> (i & 31)) & 1u);
}

template <class T>
__global__ void ewise_dense_kernel(int64_t n, int op, const T* __restrict__ a,
                                   const T* __restrict__ b, T bs, int swap,
                                   const uint32_t* __restrict__ mask, T zero, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T x = a[i];
    const T y = b ? b[i] : bs;
    T r = swap ? op_pair<T>(op, y, x) : op_pair<T>(op, x, y);
    out[i] = allowed<T>(mask, i) ? r : zero;
  }
}

// lower_bound of key in sorted idx[0..k)
__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* idx, int64_t k, int32_t key) {
  int64_t lo = 0, hi = k;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (idx[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// union of two sorted index sets: rank of each element in the merged output
// and a matched flag for elements of `a` present in `b`.
__global__ void union_rank_a(int64_t ka, const int32_t* __restrict__ ia, int64_t kb,
                             const int32_t* __restrict__ ib, int64_t* __restrict__ pos_in_b,
                             int32_t* __restrict__ matched) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ka;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = lower_bound_i32(ib, kb, ia[i]);
    pos_in_b[i] = p;
    matched[i] = (p < kb && ib[p] == ia[i]) ? 1 : 0;
  }
}

template <class T>
__global__ void union_write(int op, int64_t ka, const int32_t* __restrict__ ia,
                            const T* __restrict__ va, int64_t kb, const int32_t* __restrict__ ib,
                            const T* __restrict__ vb, const int64_t* __restrict__ pos_in_b,
                            const int32_t* __restrict__ matched,
                            const int64_t* __restrict__ matched_pre,  // exclusive scan, ka+1
                            int32_t* __restrict__ out_idx, T* __restrict__ out_vals) {
  const int64_t total = ka + kb;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t < ka) {
      const int64_t i = t;
      const int64_t r = i + pos_in_b[i] - matched_pre[i];
      out_idx[r] = ia[i];
      out_vals[r] = matched[i] ? op_fold<T>(op, va[i], vb[pos_in_b[i]]) : op_fold1<T>(op, va[i]);
    } else {
      const int64_t j = t - ka;
      const int64_t p = lower_bound_i32(ia, ka, ib[j]);
      if (p < ka && ia[p] == ib[j]) continue;  // written by the a-side
      const int64_t r = j + p - matched_pre[p];
      out_idx[r] = ib[j];
      out_vals[r] = op_fold1<T>(op, vb[j]);
    }
  }
}

template <class T>
__global__ void intersect_kernel(int op, int64_t ka, const int32_t* __restrict__ ia,
                                 const T* __restrict__ va, int64_t kb,
                                 const int32_t* __restrict__ ib, const T* __restrict__ vb,
                                 int32_t* __restrict__ flag, T* __restrict__ prod) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ka;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = lower_bound_i32(ib, kb, ia[i]);
    bool m = p < kb && ib[p] == ia[i];
    flag[i] = m ? 1 : 0;
    if (m) prod[i] = op_pair<T>(op, va[i], vb[p]);
  }
}

template <class T>
__global__ void gather_pair_kernel(int op, int64_t k, const int32_t* __restrict__ idx,
                                   const T* __restrict__ vals, const T* __restrict__ dense,
                                   int swap, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T d = dense[idx[i]];
    out[i] = swap ? op_pair<T>(op, d, vals[i]) : op_pair<T>(op, vals[i], d);
  }
}

template <class T>
__global__ void flag_by_mask(int64_t k, const int32_t* __restrict__ idx,
                             const uint32_t* __restrict__ mask, const int32_t* __restrict__ pre,
                             int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool ok = pre ? pre[i] != 0 : true;
    if (ok && mask) ok = (mask[idx[i] >> 5] >> (idx[i] & 31)) & 1u;
    flag[i] = ok ? 1 : 0;
  }
}

template <class T>
__global__ void select_flagged(int64_t k, const int32_t* __restrict__ flag,
                               const int64_t* __restrict__ pos, const int32_t* __restrict__ idx,
                               const T* __restrict__ vals, int32_t* __restrict__ out_idx,
                               T* __restrict__ out_vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) {
      out_idx[pos[i]] = idx ? idx[i] : (int32_t)i;
      out_vals[pos[i]] = vals[i];
    }
}

template <class T>
__global__ void assign_kernel(int64_t n, T* __restrict__ w, T value,
                              const uint32_t* __restrict__ mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (allowed<T>(mask, i)) w[i] = value;
}

__global__ void bounds_kernel(int64_t k, const int64_t* __restrict__ t, int64_t n,
                              int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x)
    if (t[i] < 0 || t[i] >= n) atomicOr(bad, 1);
}

template <class T>
__device__ __forceinline__ void atomic_min_any(T* addr, T v);
template <>
__device__ __forceinline__ void atomic_min_any<int64_t>(int64_t* addr, int64_t v) {
  atomicMin(reinterpret_cast<long long*>(addr), (long long)v);
}
template <>
__device__ __forceinline__ void atomic_min_any<double>(double* addr, double v) {
  // addr holds ordered bits (see ordered_bits)
  atomicMin(reinterpret_cast<unsigned long long*>(addr), ordered_bits(v));
}

template <class T>
__global__ void scatter_min_kernel(int64_t k, const int64_t* __restrict__ tgt,
                                   const T* __restrict__ val, const uint32_t* __restrict__ mask,
                                   T* __restrict__ tmp, uint32_t* __restrict__ touched) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = tgt[i];
    if (!allowed<T>(mask, t)) continue;
    atomic_min_any<T>(tmp + t, val[i]);
    atomicOr(touched + (t >> 5), 1u << (t & 31));
  }
}

template <class T>
__global__ void scatter_min_apply(int64_t n, const T* __restrict__ tmp,
                                  const uint32_t* __restrict__ touched, T* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if ((touched[i >> 5] >> (i & 31)) & 1u) {
      if (std::is_same<T, double>::value) {
        unsigned long long b;
        memcpy(&b, tmp + i, 8);
        w[i] = (T)from_ordered_bits(b);
      } else {
        w[i] = tmp[i];
      }
    }
}

template <class T>
__global__ void fill_bits_kernel(int64_t n, T* __restrict__ out, unsigned long long bits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    reinterpret_cast<unsigned long long*>(out)[i] = bits;
}

template <class T>
__global__ void gather_dense_kernel(int64_t k, const int64_t* __restrict__ tgt,
                                    const T* __restrict__ src, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[tgt[i]];
}

template <class T>
__global__ void gather_sparse_kernel(int64_t k, const int64_t* __restrict__ tgt, int64_t uk,
                                     const int32_t* __restrict__ uidx, const T* __restrict__ uval,
                                     int32_t* __restrict__ present, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = lower_bound_i32(uidx, uk, (int32_t)tgt[i]);
    const bool m = p < uk && uidx[p] == tgt[i];
    present[i] = m ? 1 : 0;
    if (m) out[i] = uval[p];
  }
}

template <class T>
__global__ void affine_kernel(int64_t n, const T* __restrict__ in, T scale, T shift,
                              T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = wrap_add(wrap_mul(in[i], scale), shift);
}

// block fold -> one partial per block; partial folds are combined on one block
template <class T>
__global__ void reduce_kernel(int64_t n, int op, const T* __restrict__ v, int use_zero, T zero,
                              T* __restrict__ partial, unsigned long long* __restrict__ count) {
  __shared__ T s[32];
  __shared__ long long sc[32];
  const T ident = op_identity<T>(op);
  T acc = ident;
  long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T x = v[i];
    if (use_zero && x == zero) continue;
    acc = op_fold<T>(op, acc, x);
    ++c;
  }
  acc = warp_fold<T>(op, acc);
  c = warp_sum_ll(c);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { s[wid] = acc; sc[wid] = c; }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    acc = lane < nw ? s[lane] : ident;
    c = lane < nw ? sc[lane] : 0;
    acc = warp_fold<T>(op, acc);
    c = warp_sum_ll(c);
    if (lane == 0) {
      partial[blockIdx.x] = acc;
      if (c) atomicAdd(count, (unsigned long long)c);
    }
  }
}

// sequential fold for order-dependent ops (one thread; host-decided)
template <class T>
__global__ void reduce_seq_kernel(int64_t n, int op, const T* __restrict__ v, int use_zero,
                                  T zero, T* __restrict__ out, unsigned long long* __restrict__ count) {
  if (blockIdx.x || threadIdx.x) return;
  T acc = op_identity<T>(op);
  long long c = 0;
  for (int64_t i = 0; i < n; ++i) {
    const T x = v[i];
    if (use_zero && x == zero) continue;
    acc = c == 0 ? x : op_fold<T>(op, acc, x);
    ++c;
  }
  *out = acc;
  *count = (unsigned long long)c;
}

template <class T>
__global__ void __launch_bounds__(256)
reduce_rows_kernel(int64_t nrows, const int64_t* __restrict__ off, const T* __restrict__ vals,
                   T iso, int op, T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T ident = op_identity<T>(op);
  for (int64_t i = w0; i < nrows; i += nw) {
    const int64_t lo = off[i], hi = off[i + 1];
    T acc = ident;
    for (int64_t p = lo + lane; p < hi; p += 32) acc = op_fold<T>(op, acc, vals ? vals[p] : iso);
    acc = warp_fold<T>(op, acc);
    if (lane == 0) out[i] = (hi - lo == 1) ? op_fold1<T>(op, vals ? vals[lo] : iso) : acc;
  }
}

template <class T>
static T host_val(const void* p) {
  T v;
  memcpy(&v, p, sizeof(T));
  return v;
}

template <class T>
static gb_status compact_flags(gb_ctx* ctx, Arena& ar, int64_t k, const int32_t* flag,
                               const int32_t* idx, const T* vals, int32_t* out_idx, T* out_vals,
                               int64_t* count) {
  cudaStream_t s = stream_of(ctx);
  int64_t* pos = ar.alloc<int64_t>(k + 1);
  int32_t* f1 = ar.alloc<int32_t>(k + 1);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemcpyAsync(f1, flag, sizeof(int32_t) * k, cudaMemcpyDeviceToDevice, s));
  GB_CUDA(ctx, cudaMemsetAsync(f1 + k, 0, sizeof(int32_t), s));
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, f1, pos, k + 1, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp, tb, f1, pos, k + 1, s));
  select_flagged<T><<<grid_for(ctx, k, 256), 256, 0, s>>>(k, f1, pos, idx, vals, out_idx, out_vals);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 5);
  return read_i64(ctx, pos + k, count);
}

}  // namespace gb

using namespace gb;

#define GB_DISPATCH(dtype, T, ...)        \
  if ((dtype) == GB_I64) {                \
    typedef int64_t T;                    \
    __VA_ARGS__                           \
  } else {                                \
    typedef double T;                     \
    __VA_ARGS__                           \
  }

extern "C" {

gb_status gb_ewise_dense(gb_ctx* ctx, int32_t op, int32_t dtype, int64_t n, const void* a,
                         const void* b, const void* b_scalar_host, int32_t swap,
                         const uint32_t* mask, const void* zero_host, void* out) {
  if (n == 0) return GB_OK;
  cudaStream_t s = stream_of(ctx);
  GB_DISPATCH(dtype, T, {
    const T bs = b ? (T)0 : host_val<T>(b_scalar_host);
    const T z = zero_host ? host_val<T>(zero_host) : (T)0;
    ewise_dense_kernel<T><<<grid_for(ctx, n, 256), 256, 0, s>>>(n, op, (const T*)a, (const T*)b, bs,
                                                               swap, mask, z, (T*)out);
  })
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx);
  return GB_OK;
}

gb_status gb_union_sparse(gb_ctx* ctx, int32_t op, int32_t dtype, int64_t ka, const int32_t* ia,
                          const void* va, int64_t kb, const int32_t* ib, const void* vb,
                          int32_t* out_idx, void* out_vals, int64_t* count) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  int64_t* pos_in_b = ar.alloc<int64_t>(ka + 1);
  int32_t* matched = ar.alloc<int32_t>(ka + 1);
  int64_t* pre = ar.alloc<int64_t>(ka + 1);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(matched, 0, sizeof(int32_t) * (ka + 1), s));
  if (ka) union_rank_a<<<grid_for(ctx, ka, 256), 256, 0, s>>>(ka, ia, kb, ib, pos_in_b, matched);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, matched, pre, ka + 1, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp, tb, matched, pre, ka + 1, s));
  if (ka + kb)
    GB_DISPATCH(dtype, T, {
      union_write<T><<<grid_for(ctx, ka + kb, 256), 256, 0, s>>>(
          op, ka, ia, (const T*)va, kb, ib, (const T*)vb, pos_in_b, matched, pre, out_idx,
          (T*)out_vals);
    })
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 4);
  int64_t m = 0;
  GB_TRY(read_i64(ctx, pre + ka, &m));
  *count = ka + kb - m;
  return GB_OK;
}

gb_status gb_intersect_sparse(gb_ctx* ctx, int32_t op, int32_t dtype, int64_t ka,
                              const int32_t* ia, const void* va, int64_t kb, const int32_t* ib,
                              const void* vb, const uint32_t* mask, int32_t* out_idx,
                              void* out_vals, int64_t* count) {
  *count = 0;
  if (ka == 0) return GB_OK;
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  int32_t* flag = ar.alloc<int32_t>(ka);
  int32_t* flag2 = ar.alloc<int32_t>(ka);
  GB_ARENA_CHECK(ctx, ar);
  GB_DISPATCH(dtype, T, {
    T* prod = ar.alloc<T>(ka);
    GB_ARENA_CHECK(ctx, ar);
    intersect_kernel<T><<<grid_for(ctx, ka, 256), 256, 0, s>>>(op, ka, ia, (const T*)va, kb, ib,
                                                               (const T*)vb, flag, prod);
    flag_by_mask<T><<<grid_for(ctx, ka, 256), 256, 0, s>>>(ka, ia, mask, flag, flag2);
    return compact_flags<T>(ctx, ar, ka, flag2, ia, prod, out_idx, (T*)out_vals, count);
  })
}

gb_status gb_gather_pair(gb_ctx* ctx, int32_t op, int32_t dtype, int64_t k, const int32_t* idx,
                         const void* vals, const void* dense, int32_t swap, void* out) {
  if (k == 0) return GB_OK;
  cudaStream_t s = stream_of(ctx);
  GB_DISPATCH(dtype, T, {
    gather_pair_kernel<T><<<grid_for(ctx, k, 256), 256, 0, s>>>(op, k, idx, (const T*)vals,
                                                                (const T*)dense, swap, (T*)out);
  })
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx);
  return GB_OK;
}

gb_status gb_filter_mask(gb_ctx* ctx, int32_t dtype, int64_t k, const int32_t* idx,
                         const void* vals, const uint32_t* mask, int32_t* out_idx, void* out_vals,
                         int64_t* count) {
  *count = 0;
  if (k == 0) return GB_OK;
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  int32_t* flag = ar.alloc<int32_t>(k);
  GB_ARENA_CHECK(ctx, ar);
  GB_DISPATCH(dtype, T, {
    flag_by_mask<T><<<grid_for(ctx, k, 256), 256, 0, s>>>(k, idx, mask, nullptr, flag);
    return compact_flags<T>(ctx, ar, k, flag, idx, (const T*)vals, out_idx, (T*)out_vals, count);
  })
}

gb_status gb_assign_scalar(gb_ctx* ctx, int32_t dtype, int64_t n, void* w,
                           const void* value_host, const uint32_t* mask) {
  if (n == 0) return GB_OK;
  cudaStream_t s = stream_of(ctx);
  GB_DISPATCH(dtype, T, {
    assign_kernel<T><<<grid_for(ctx, n, 256), 256, 0, s>>>(n, (T*)w, host_val<T>(value_host), mask);
  })
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx);
  return GB_OK;
}

gb_status gb_check_bounds(gb_ctx* ctx, int64_t k, const int64_t* t, int64_t n, int32_t* bad_host) {
  *bad_host = 0;
  if (k == 0) return GB_OK;
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  int* bad = ar.alloc<int>(2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(bad, 0, 8, s));
  bounds_kernel<<<grid_for(ctx, k, 256), 256, 0, s>>>(k, t, n, bad);
  int64_t h = 0;
  GB_TRY(read_i64(ctx, (const int64_t*)bad, &h));
  *bad_host = (int32_t)(h & 1);
  count_launch(ctx, 2);
  return GB_OK;
}

gb_status gb_scatter_min(gb_ctx* ctx, int32_t dtype, int64_t n, void* w, int64_t k,
                         const int64_t* tgt, const void* vals, const uint32_t* mask) {
  if (k == 0 || n == 0) return GB_OK;
  int32_t bad = 0;
  GB_TRY(gb_check_bounds(ctx, k, tgt, n, &bad));
  if (bad) return set_error(ctx, GB_ERR_INDEX, "scatter target index out of range");
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  uint32_t* touched = ar.alloc<uint32_t>(W);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(touched, 0, sizeof(uint32_t) * W, s));
  GB_DISPATCH(dtype, T, {
    T* tmp = ar.alloc<T>(n);
    GB_ARENA_CHECK(ctx, ar);
    const unsigned long long init = std::is_same<T, double>::value ? ~0ull
                                                                   : 0x7fffffffffffffffull;
    fill_bits_kernel<T><<<grid_for(ctx, n, 256), 256, 0, s>>>(n, tmp, init);
    scatter_min_kernel<T><<<grid_for(ctx, k, 256), 256, 0, s>>>(k, tgt, (const T*)vals, mask, tmp,
                                                               touched);
    scatter_min_apply<T><<<grid_for(ctx, n, 256), 256, 0, s>>>(n, tmp, touched, (T*)w);
  })
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 4);
  return GB_OK;
}

gb_status gb_gather(gb_ctx* ctx, int32_t dtype, int64_t k, const int64_t* tgt, int64_t usize,
                    const void* src, void* out) {
  if (k == 0) return GB_OK;
  int32_t bad = 0;
  GB_TRY(gb_check_bounds(ctx, k, tgt, usize, &bad));
  if (bad) return set_error(ctx, GB_ERR_INDEX, "gather index out of range");
  cudaStream_t s = stream_of(ctx);
  GB_DISPATCH(dtype, T, {
    gather_dense_kernel<T><<<grid_for(ctx, k, 256), 256, 0, s>>>(k, tgt, (const T*)src, (T*)out);
  })
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx);
  return GB_OK;
}

gb_status gb_gather_sparse(gb_ctx* ctx, int32_t dtype, int64_t k, const int64_t* tgt,
                           int64_t usize, int64_t uk, const int32_t* uidx, const void* uval,
                           int32_t* present, void* out) {
  if (k == 0) return GB_OK;
  int32_t bad = 0;
  GB_TRY(gb_check_bounds(ctx, k, tgt, usize, &bad));
  if (bad) return set_error(ctx, GB_ERR_INDEX, "gather index out of range");
  cudaStream_t s = stream_of(ctx);
  GB_DISPATCH(dtype, T, {
    gather_sparse_kernel<T><<<grid_for(ctx, k, 256), 256, 0, s>>>(k, tgt, uk, uidx, (const T*)uval,
                                                                 present, (T*)out);
  })
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx);
  return GB_OK;
}

gb_status gb_apply_affine(gb_ctx* ctx, int32_t dtype, int64_t n, const void* in,
                          const void* scale_host, const void* shift_host, void* out) {
  if (n == 0) return GB_OK;
  cudaStream_t s = stream_of(ctx);
  GB_DISPATCH(dtype, T, {
    affine_kernel<T><<<grid_for(ctx, n, 256), 256, 0, s>>>(n, (const T*)in, host_val<T>(scale_host),
                                                          host_val<T>(shift_host), (T*)out);
  })
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx);
  return GB_OK;
}

gb_status gb_reduce(gb_ctx* ctx, int32_t op, int32_t dtype, int64_t n, const void* vals,
                    const void* zero_host, void* out_host, int64_t* count_host) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  unsigned long long* cnt = ar.alloc<unsigned long long>(1);
  const int grid = n > 0 ? grid_for(ctx, n, 256, 4) : 1;
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(cnt, 0, 8, s));
  GB_DISPATCH(dtype, T, {
    T* part = ar.alloc<T>(grid + 1);
    GB_ARENA_CHECK(ctx, ar);
    const T z = zero_host ? host_val<T>(zero_host) : (T)0;
    T result;
    if (!fold_commutes(op)) {
      reduce_seq_kernel<T><<<1, 1, 0, s>>>(n, op, (const T*)vals, zero_host != nullptr, z, part, cnt);
      GB_LAUNCH_CHECK(ctx);
      GB_CUDA(ctx, cudaMemcpyAsync(pinned_slots(ctx), part, sizeof(T), cudaMemcpyDeviceToHost, s));
    } else {
      reduce_kernel<T><<<grid, 256, 0, s>>>(n, op, (const T*)vals, zero_host != nullptr, z, part, cnt);
      reduce_kernel<T><<<1, 256, 0, s>>>(grid, op, part, 0, z, part + grid, cnt + 0);
      GB_LAUNCH_CHECK(ctx);
      GB_CUDA(ctx, cudaMemcpyAsync(pinned_slots(ctx), part + grid, sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    GB_CUDA(ctx, cudaMemcpyAsync(pinned_slots(ctx) + 1, cnt, 8, cudaMemcpyDeviceToHost, s));
    GB_CUDA(ctx, cudaStreamSynchronize(s));
    memcpy(&result, pinned_slots(ctx), sizeof(T));
    memcpy(out_host, &result, sizeof(T));
  })
  // the second pass counted the partials; subtract them back out
  int64_t c = pinned_slots(ctx)[1];
  if (fold_commutes(op)) c -= grid;
  if (count_host) *count_host = c;
  count_launch(ctx, 3);
  return GB_OK;
}

gb_status gb_reduce_rows(gb_ctx* ctx, int32_t op, const gb_csr* a, void* out) {
  const int64_t n = a->nrows;
  if (n == 0) return GB_OK;
  cudaStream_t s = stream_of(ctx);
  GB_DISPATCH(a->dtype, T, {
    const T iso = std::is_same<T, double>::value ? (T)a->iso_f64 : (T)a->iso_i64;
    reduce_rows_kernel<T><<<grid_for(ctx, n * 32, 256, 16), 256, 0, s>>>(
        n, a->offsets, (const T*)a->values, iso, op, (T*)out);
  })
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx);
  return GB_OK;
}

}  // extern "C"
