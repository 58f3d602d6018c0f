// Output-masked SpGEMM and the fused triangle count.
//
//   gb_mxm_masked  mxm_masked (kernels.py:329-391): for every stored mask
//                  entry (i, j) with a non-zero value, intersect row i of A
//                  with column j of B (given as row j of the orientation
//                  `b`), multiply the matches and fold them.  Warp per mask
//                  row; each lane binary-searches elements of the shorter
//                  list in the longer one.  Output keeps mask order, so C is
//                  CSR-sorted without a sort.
//   gb_tc          triangle_count (algorithms.py:206-240) fused: degree
//                  ranking (stable by id), the upper (higher-rank) adjacency
//                  per vertex, and a warp-per-row intersection count with the
//                  row staged in shared memory.  The count is the same number
//                  the reference's L.L^T.*L reduction produces (each triangle
//                  once); only the orientation differs, which is free for an
//                  integer total (SURVEY §8(a) A-note 10).
#include <type_traits>

#include <cub/cub.cuh>

#include "gb_common.cuh"

namespace gb {

// first position with a[p] >= key (branchless halving: a select per step)
__device__ __forceinline__ int64_t lb32(const int32_t* a, int64_t n, int32_t key) {
  if (n <= 0) return 0;
  const int32_t* b = a;
  int64_t l = n;
  while (l > 1) {
    const int64_t h = l >> 1;
    b = b[h - 1] < key ? b + h : b;
    l -= h;
  }
  return (b - a) + (*b < key);
}

// One warp per mask row.  out_flag[e] = 1 when mask entry e produces an
// output entry (matches > 0, or the identity is non-zero), out_val[e] its value.
template <class T>
__global__ void __launch_bounds__(256)
mxm_masked_kernel(int64_t nrows, const int64_t* __restrict__ moff, const int32_t* __restrict__ midx,
                  const void* __restrict__ mval, int mdtype, int miso_live,
                  const int64_t* __restrict__ aoff,
                  const int32_t* __restrict__ aidx, const T* __restrict__ aval, T aiso,
                  const int64_t* __restrict__ boff, const int32_t* __restrict__ bidx,
                  const T* __restrict__ bval, T biso, int add_op, int mult_op,
                  int32_t* __restrict__ out_flag, T* __restrict__ out_val,
                  unsigned long long* __restrict__ counters) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T ident = op_identity<T>(add_op);
  for (int64_t i = w0; i < nrows; i += nw) {
    const int64_t alo = aoff[i], ahi = aoff[i + 1];
    const int64_t la = ahi - alo;
    long long mults = 0, adds = 0;
    for (int64_t e = moff[i]; e < moff[i + 1]; ++e) {
      const bool live = !mval ? miso_live != 0
                              : (mdtype == GB_I64 ? ((const int64_t*)mval)[e] != 0
                                                  : ((const double*)mval)[e] != 0.0);
      if (!live) {
        if (lane == 0) out_flag[e] = 0;
        continue;
      }
      const int32_t j = midx[e];
      const int64_t blo = boff[j], bhi = boff[j + 1];
      const int64_t lb = bhi - blo;
      // iterate the shorter list, search the longer
      const bool a_short = la <= lb;
      const int32_t* sidx = a_short ? aidx + alo : bidx + blo;
      const int32_t* lidx = a_short ? bidx + blo : aidx + alo;
      const int64_t ls = a_short ? la : lb, ll = a_short ? lb : la;
      T acc = ident;
      long long m = 0;
      for (int64_t q = lane; q < ls; q += 32) {
        const int32_t key = sidx[q];
        const int64_t p = lb32(lidx, ll, key);
        if (p < ll && lidx[p] == key) {
          const T x = a_short ? (aval ? aval[alo + q] : aiso) : (aval ? aval[alo + p] : aiso);
          const T y = a_short ? (bval ? bval[blo + p] : biso) : (bval ? bval[blo + q] : biso);
          acc = op_fold<T>(add_op, acc, op_pair<T>(mult_op, x, y));
          ++m;
        }
      }
      acc = warp_fold<T>(add_op, acc);
      m = warp_sum_ll(m);
      if (lane == 0) {
        if (m > 0) {
          out_flag[e] = 1;
          out_val[e] = acc;
          mults += m;
          adds += m - 1;
        } else {
          out_flag[e] = ident != (T)0 ? 1 : 0;
          out_val[e] = ident;
        }
      }
    }
    if (lane == 0 && counters && mults) {
      atomicAdd(counters + 1, (unsigned long long)mults);
      atomicAdd(counters + 2, (unsigned long long)adds);
    }
  }
}

__global__ void row_counts(int64_t nrows, const int64_t* __restrict__ off,
                           const int32_t* __restrict__ flag, int64_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < nrows; i += nw) {
    long long c = 0;
    for (int64_t p = off[i] + lane; p < off[i + 1]; p += 32) c += flag[p];
    c = warp_sum_ll(c);
    if (lane == 0) cnt[i] = c;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[nrows] = 0;
}

template <class T>
__global__ void compact_entries(int64_t nnz, const int32_t* __restrict__ flag,
                                const int64_t* __restrict__ pos, const int32_t* __restrict__ midx,
                                const T* __restrict__ val, int32_t* __restrict__ out_idx,
                                T* __restrict__ out_val) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    if (flag[e]) {
      out_idx[pos[e]] = midx[e];
      out_val[pos[e]] = val[e];
    }
}

// ---------------------------------------------------------------------------
// triangle count
// ---------------------------------------------------------------------------
__global__ void tc_degree_keys(int64_t n, const int64_t* __restrict__ off,
                               uint32_t* __restrict__ deg, int32_t* __restrict__ ids) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    deg[i] = (uint32_t)(off[i + 1] - off[i]);
    ids[i] = (int32_t)i;
  }
}

__global__ void tc_rank(int64_t n, const int32_t* __restrict__ order, int32_t* __restrict__ rank) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    rank[order[r]] = (int32_t)r;
}

// upper degree of vertex order[r] -> ucnt[r]
__global__ void tc_upper_count(int64_t n, const int64_t* __restrict__ off,
                               const int32_t* __restrict__ idx, const int32_t* __restrict__ order,
                               const int32_t* __restrict__ rank, int64_t* __restrict__ ucnt) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n; r += nw) {
    const int32_t v = order[r];
    long long c = 0;
    for (int64_t p = off[v] + lane; p < off[v + 1]; p += 32) c += rank[idx[p]] > r;
    c = warp_sum_ll(c);
    if (lane == 0) ucnt[r] = c;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ucnt[n] = 0;
}

__global__ void tc_upper_fill(int64_t n, const int64_t* __restrict__ off,
                              const int32_t* __restrict__ idx, const int32_t* __restrict__ order,
                              const int32_t* __restrict__ rank, const int64_t* __restrict__ uoff,
                              int32_t* __restrict__ uidx) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n; r += nw) {
    const int32_t v = order[r];
    int64_t out = uoff[r];
    for (int64_t base = off[v]; base < off[v + 1]; base += 32) {
      const int64_t p = base + lane;
      int32_t rj = -1;
      if (p < off[v + 1]) rj = rank[idx[p]];
      const bool keep = rj > r;
      const uint32_t bal = __ballot_sync(GB_FULL, keep);
      if (keep) uidx[out + __popc(bal & ((1u << lane) - 1u))] = rj;
      out += __popc(bal);
    }
  }
}

constexpr int kTcSmem = 1024;  // per-warp staged row capacity

// warp per upper row r: count |U(r) & U(j)| for every j in U(r)
__global__ void __launch_bounds__(256)
tc_count(int64_t n, const int64_t* __restrict__ uoff, const int32_t* __restrict__ uidx,
         unsigned long long* __restrict__ total) {
  __shared__ int32_t s_row[8][kTcSmem];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  long long c = 0;
  for (int64_t r = w0; r < n; r += nw) {
    const int64_t lo = uoff[r], hi = uoff[r + 1];
    const int64_t len = hi - lo;
    if (len < 2) continue;
    const bool staged = len <= kTcSmem;
    const int32_t* row = staged ? s_row[wid] : uidx + lo;
    if (staged) {
      for (int64_t q = lane; q < len; q += 32) s_row[wid][q] = uidx[lo + q];
      __syncwarp();
    }
    const int ilen = (int)len;
    const int32_t rmax = row[ilen - 1];
    int64_t mylo = 0, myhi = 0;  // bounds of U(row[a]) for a = (chunk of 32) + lane
    for (int a = 0; a < ilen; ++a) {
      if ((a & 31) == 0) {
        // the next 32 lists' bounds in one round of loads
        const int aa = a + lane;
        mylo = myhi = 0;
        if (aa < ilen) {
          const int32_t jj = row[aa];
          mylo = uoff[jj];
          myhi = uoff[jj + 1];
        }
      }
      const int64_t jlo = __shfl_sync(GB_FULL, mylo, a & 31);
      const int64_t jhi = __shfl_sync(GB_FULL, myhi, a & 31);
      // elements of U(j) are > j > r; search them in U(r) after position a
      // (branchless 32-bit lower bound: the kernel is issue-bound)
      const int32_t* base0 = row + a + 1;
      const int m = ilen - a - 1;
      if (m == 0) continue;
      for (int64_t q = jlo + lane; q < jhi; q += 32) {
        const int32_t key = uidx[q];
        if (key > rmax) break;  // sorted lists: no later key of U(j) is in U(r) either
        const int32_t* b = base0;
        int l = m;
        while (l > 1) {
          const int h = l >> 1;
          b = b[h - 1] < key ? b + h : b;
          l -= h;
        }
        c += *b == key;
      }
    }
    __syncwarp();
  }
  c = warp_sum_ll(c);
  if (lane == 0 && c) atomicAdd(total, (unsigned long long)c);
}

__global__ void diag_kernel(int64_t n, const int64_t* __restrict__ off,
                            const int32_t* __restrict__ idx, int* __restrict__ found) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = lb32(idx + off[i], off[i + 1] - off[i], (int32_t)i);
    if (p < off[i + 1] - off[i] && idx[off[i] + p] == i) *found = 1;
  }
}

template <class T>
static gb_status mxm_run(gb_ctx* ctx, Arena& ar, int add_op, int mult_op, const gb_csr* a,
                         const gb_csr* b, const gb_csr* m, int miso_live, int32_t* flag,
                         int64_t* rc, int64_t* pos, int32_t* flag1, int64_t* out_offsets,
                         int32_t* out_indices, void* out_vals, int64_t* counters) {
  cudaStream_t s = stream_of(ctx);
  const int64_t nr = m->nrows, nnz = m->nnz;
  const bool dbl = std::is_same<T, double>::value;
  T* val = ar.alloc<T>(nnz);
  GB_ARENA_CHECK(ctx, ar);
  mxm_masked_kernel<T><<<grid_for(ctx, nr * 32, 256, 16), 256, 0, s>>>(
      nr, m->offsets, m->indices, m->values, m->dtype, miso_live, a->offsets, a->indices,
      (const T*)a->values, dbl ? (T)a->iso_f64 : (T)a->iso_i64, b->offsets, b->indices,
      (const T*)b->values, dbl ? (T)b->iso_f64 : (T)b->iso_i64, add_op, mult_op, flag, val,
      (unsigned long long*)counters);
  row_counts<<<grid_for(ctx, nr * 32, 256, 16), 256, 0, s>>>(nr, m->offsets, flag, rc);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, rc, out_offsets, nr + 1, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp, tb, rc, out_offsets, nr + 1, s));
  GB_CUDA(ctx, cudaMemcpyAsync(flag1, flag, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, s));
  GB_CUDA(ctx, cudaMemsetAsync(flag1 + nnz, 0, 4, s));
  size_t tb2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, flag1, pos, nnz + 1, s);
  void* tmp2 = ar.raw(tb2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp2, tb2, flag1, pos, nnz + 1, s));
  compact_entries<T><<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, flag1, pos, m->indices, val,
                                                            out_indices, (T*)out_vals);
  return GB_OK;
}

}  // namespace gb

using namespace gb;

extern "C" {

gb_status gb_mxm_masked(gb_ctx* ctx, int32_t add_op, int32_t mult_op, const gb_csr* a,
                        const gb_csr* b, const gb_csr* m, int64_t* out_offsets,
                        int32_t* out_indices, void* out_vals, int64_t* nnz_host,
                        int64_t* counters) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int64_t nr = m->nrows, nnz = m->nnz;
  int32_t* flag = ar.alloc<int32_t>(nnz + 1);
  int64_t* rc = ar.alloc<int64_t>(nr + 1);
  int64_t* pos = ar.alloc<int64_t>(nnz + 1);
  int32_t* flag1 = ar.alloc<int32_t>(nnz + 1);
  GB_ARENA_CHECK(ctx, ar);
  if (a->dtype != b->dtype) return set_error(ctx, GB_ERR_ARG, "operand dtypes differ");
  if (nnz == 0) {
    GB_CUDA(ctx, cudaMemsetAsync(out_offsets, 0, sizeof(int64_t) * (nr + 1), s));
    *nnz_host = 0;
    return GB_OK;
  }
  const int miso_live = !m->values && (m->iso_i64 != 0 || m->iso_f64 != 0.0);
  if (a->dtype == GB_I64)
    GB_TRY(mxm_run<int64_t>(ctx, ar, add_op, mult_op, a, b, m, miso_live, flag, rc, pos, flag1,
                            out_offsets, out_indices, out_vals, counters));
  else
    GB_TRY(mxm_run<double>(ctx, ar, add_op, mult_op, a, b, m, miso_live, flag, rc, pos, flag1,
                           out_offsets, out_indices, out_vals, counters));
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 8);
  return read_i64(ctx, pos + nnz, nnz_host);
}

gb_status gb_has_diagonal(gb_ctx* ctx, const gb_csr* a, int32_t* found_host) {
  *found_host = 0;
  const int64_t n = a->nrows < a->ncols ? a->nrows : a->ncols;
  if (n == 0 || a->nnz == 0) return GB_OK;
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  int* f = ar.alloc<int>(2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(f, 0, 8, s));
  diag_kernel<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, a->offsets, a->indices, f);
  int64_t h = 0;
  GB_TRY(read_i64(ctx, (const int64_t*)f, &h));
  *found_host = (int32_t)(h & 1);
  count_launch(ctx, 2);
  return GB_OK;
}

gb_status gb_tc(gb_ctx* ctx, const gb_csr* a, int64_t* count_host) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int64_t n = a->nrows;
  *count_host = 0;
  if (n == 0 || a->nnz == 0) return GB_OK;
  uint32_t* deg = ar.alloc<uint32_t>(n);
  uint32_t* deg2 = ar.alloc<uint32_t>(n);
  int32_t* ids = ar.alloc<int32_t>(n);
  int32_t* order = ar.alloc<int32_t>(n);
  int32_t* rank = ar.alloc<int32_t>(n);
  int64_t* ucnt = ar.alloc<int64_t>(n + 1);
  int64_t* uoff = ar.alloc<int64_t>(n + 1);
  unsigned long long* total = ar.alloc<unsigned long long>(1);
  GB_ARENA_CHECK(ctx, ar);
  tc_degree_keys<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, a->offsets, deg, ids);
  // stable: ties keep ascending vertex id (algorithms.py:209-212)
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, deg, deg2, ids, order, n, 0, 32, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceRadixSort::SortPairs(tmp, tb, deg, deg2, ids, order, n, 0, 32, s));
  tc_rank<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, order, rank);
  tc_upper_count<<<grid_for(ctx, n * 32, 256, 16), 256, 0, s>>>(n, a->offsets, a->indices, order,
                                                                rank, ucnt);
  size_t tb2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, ucnt, uoff, n + 1, s);
  void* tmp2 = ar.raw(tb2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp2, tb2, ucnt, uoff, n + 1, s));
  int64_t m = 0;
  GB_TRY(read_i64(ctx, uoff + n, &m));
  int32_t* uidx = ar.alloc<int32_t>(m + 1);
  int32_t* uidx2 = ar.alloc<int32_t>(m + 1);
  GB_ARENA_CHECK(ctx, ar);
  tc_upper_fill<<<grid_for(ctx, n * 32, 256, 16), 256, 0, s>>>(n, a->offsets, a->indices, order,
                                                               rank, uoff, uidx);
  // sort each upper row ascending (rank order)
  size_t tb3 = 0;
  cub::DeviceSegmentedSort::SortKeys(nullptr, tb3, uidx, uidx2, m, n, uoff, uoff + 1, s);
  void* tmp3 = ar.raw(tb3);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceSegmentedSort::SortKeys(tmp3, tb3, uidx, uidx2, m, n, uoff, uoff + 1, s));
  GB_CUDA(ctx, cudaMemsetAsync(total, 0, 8, s));
  const int ps = prof_begin(ctx, PROF_TC, m);
  tc_count<<<resident_grid(ctx, tc_count, 256), 256, 0, s>>>(n, uoff, uidx2, total);
  prof_end(ctx, ps);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 12);
  return read_i64(ctx, (const int64_t*)total, count_host);
}

}  // extern "C"
