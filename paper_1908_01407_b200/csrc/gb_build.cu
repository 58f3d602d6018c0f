// Matrix construction and the R-MAT input pipeline.
//
//   gb_rmat_generate   io.py:275-295   counter-based SplitMix64, bit-exact
//   gb_edges_to_csr    io.py:220-249 + 298-315  loops, mirror, sort, dedup
//   gb_build_csr       containers.py:307-345    from_tuples with a dedup monoid
//   gb_transpose_csr   containers.py:357-364    CSC mirror (stable)
//   gb_assign_weights  io.py:252-272            first-appearance draw order
//
// These run once per graph (untimed setup).  Sorting uses CUB's radix sort
// (header-only, part of the CUDA toolkit); everything else is hand-written.
#include <cub/cub.cuh>

#include "gb_common.cuh"

namespace gb {

static const uint64_t kGamma = 0x9E3779B97F4A7C15ull;
static const uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;
static const uint64_t kMix2 = 0x94D049BB133111EBull;

__host__ __device__ __forceinline__ uint64_t splitmix_draw(uint64_t seed, uint64_t k) {
  // io.py:100-111: draw k (0-based) = mix(seed + (k+1)*gamma)
  uint64_t z = seed + (k + 1) * kGamma;
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  return z ^ (z >> 31);
}

__global__ void rmat_kernel(int scale, int64_t m, uint64_t seed, double a, double tab,
                            double tabc, int32_t* __restrict__ src, int32_t* __restrict__ dst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint32_t r = 0, c = 0;
    uint64_t k0 = (uint64_t)e * (uint64_t)scale;
    for (int l = 0; l < scale; ++l) {
      uint64_t z = splitmix_draw(seed, k0 + l);
      double x = (double)(z >> 11) * 0x1.0p-53;  // exact: 53-bit integer times 2^-53
      uint32_t rb = x >= tab;
      uint32_t cb = (x >= a && x < tab) || (x >= tabc);
      r = (r << 1) | rb;  // most significant bit first (io.py:292)
      c = (c << 1) | cb;
    }
    src[e] = (int32_t)r;
    dst[e] = (int32_t)c;
  }
}

static int bits_for(int64_t n) {
  int b = 1;
  while (((int64_t)1 << b) < n) ++b;
  return b;
}

__global__ void edge_keys_kernel(int64_t m, const int32_t* __restrict__ src,
                                 const int32_t* __restrict__ dst, int bits, int undirected,
                                 uint64_t sentinel, uint64_t* __restrict__ keys) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t s = (uint32_t)src[e], d = (uint32_t)dst[e];
    bool loop = s == d;
    if (undirected) {
      keys[2 * e] = loop ? sentinel : ((s << bits) | d);
      keys[2 * e + 1] = loop ? sentinel : ((d << bits) | s);
    } else {
      keys[e] = loop ? sentinel : ((s << bits) | d);
    }
  }
}

// offsets from sorted unique row keys: every row r gets the first position
// whose row >= r (rows with no entries repeat the next start).
template <class Row>
__global__ void offsets_from_sorted_rows(int64_t nnz, int64_t nrows, Row row_of,
                                         int64_t* __restrict__ offsets) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i < nnz ? (int64_t)row_of(i) : nrows;
    int64_t p = i == 0 ? -1 : (int64_t)row_of(i - 1);
    for (int64_t rr = p + 1; rr <= r; ++rr) offsets[rr] = i;
  }
}

struct KeyRow {
  const uint64_t* keys;
  int bits;
  __device__ int64_t operator()(int64_t i) const { return (int64_t)(keys[i] >> bits); }
};
struct IdxRow {
  const int32_t* idx;
  __device__ int64_t operator()(int64_t i) const { return idx[i]; }
};

__global__ void keys_to_cols(int64_t nnz, const uint64_t* __restrict__ keys, uint64_t mask,
                             int32_t* __restrict__ cols) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x)
    cols[i] = (int32_t)(keys[i] & mask);
}

// row id of every CSR entry: +1 at each row start, inclusive scan
__global__ void row_start_marks(int64_t nrows, int64_t nnz, const int64_t* __restrict__ off,
                                int32_t* __restrict__ marks) {
  for (int64_t r = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = off[r];
    if (p < nnz) atomicAdd(&marks[p], 1);
  }
}

template <class T>
__global__ void gather_kernel(int64_t n, const int64_t* __restrict__ perm,
                              const T* __restrict__ in, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[perm[i]];
}

__global__ void iota64(int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i;
}

__global__ void coo_keys(int64_t n, const int64_t* __restrict__ rows,
                         const int64_t* __restrict__ cols, int bits, uint64_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = ((uint64_t)rows[i] << bits) | (uint64_t)cols[i];
}

__global__ void coo_bounds(int64_t n, const int64_t* __restrict__ rows,
                           const int64_t* __restrict__ cols, int64_t nrows, int64_t ncols,
                           int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (rows[i] < 0 || rows[i] >= nrows) atomicOr(bad, 1);
    if (cols[i] < 0 || cols[i] >= ncols) atomicOr(bad, 2);
  }
}

__global__ void unique_flags(int64_t n, const uint64_t* __restrict__ keys,
                             int32_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// one thread per unique key: fold its duplicates in original order
template <class T>
__global__ void fold_segments(int64_t n, const uint64_t* __restrict__ keys,
                              const int32_t* __restrict__ flags, const int64_t* __restrict__ pos,
                              const int64_t* __restrict__ perm, const T* __restrict__ vals,
                              int op, int bits, uint64_t mask, int32_t* __restrict__ out_cols,
                              uint64_t* __restrict__ out_keys, T* __restrict__ out_vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!flags[i]) continue;
    int64_t o = pos[i];
    uint64_t k = keys[i];
    out_keys[o] = k;
    out_cols[o] = (int32_t)(k & mask);
    if (vals) {
      T acc = vals[perm[i]];
      int64_t j = i + 1;
      if (j < n && keys[j] == k) {
        for (; j < n && keys[j] == k; ++j) acc = op_fold<T>(op, acc, vals[perm[j]]);
      } else {
        acc = op_fold1<T>(op, acc);
      }
      out_vals[o] = acc;
    }
  }
}

template <class T>
__global__ void all_equal_kernel(int64_t n, const T* __restrict__ a, const T* __restrict__ b,
                                 int* __restrict__ diff) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (a[i] != b[i]) { *diff = 1; return; }
}

template <class T>
__global__ void iso_kernel(int64_t n, const T* __restrict__ v, int* __restrict__ diff) {
  T first = v[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (v[i] != first) { *diff = 1; return; }
}

template <class T>
__global__ void minmax_kernel(int64_t n, const T* __restrict__ v, double* __restrict__ out) {
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double x = (double)v[i];
    lo = fmin(lo, x);
    hi = fmax(hi, x);
  }
  for (int o = 16; o; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(GB_FULL, lo, o));
    hi = fmax(hi, __shfl_xor_sync(GB_FULL, hi, o));
  }
  if (lane_id() == 0) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(out);
    atomicMin(p, ordered_bits(lo));
    atomicMax(p + 1, ordered_bits(hi));
  }
}

__global__ void init_minmax(double* out) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(out);
  p[0] = ~0ull;
  p[1] = 0ull;
}

// ---- weights: draw index by first appearance of the unordered pair ----------
__global__ void pair_keys(int64_t nnz, const int32_t* __restrict__ src,
                          const int32_t* __restrict__ dst, int bits, uint64_t* __restrict__ keys,
                          int64_t* __restrict__ pos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t r = (uint32_t)src[i], c = (uint32_t)dst[i];
    uint64_t lo = r < c ? r : c, hi = r < c ? c : r;
    keys[i] = (lo << bits) | hi;
    pos[i] = i;
  }
}

// sorted (key, pos): segment starts hold the first appearance
__global__ void first_pos_kernel(int64_t n, const uint64_t* __restrict__ keys,
                                 const int64_t* __restrict__ pos, int64_t* __restrict__ first,
                                 int32_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool s = i == 0 || keys[i] != keys[i - 1];
    flags[i] = s ? 1 : 0;
    first[i] = s ? pos[i] : INT64_MAX;  // non-starts sort to the end
  }
}

// mark entries that are the first appearance of their pair
__global__ void mark_first(int64_t n, const int32_t* __restrict__ flags,
                           const int64_t* __restrict__ pos, int32_t* __restrict__ is_first) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flags[i]) is_first[pos[i]] = 1;
}

// entry i in list order: rank = #first appearances before i (exclusive scan)
// weight of a first appearance = draw[rank]; other entries copy their pair's.
__global__ void draw_firsts(int64_t n, const int32_t* __restrict__ is_first,
                            const int64_t* __restrict__ rank, uint64_t seed, int64_t low,
                            int64_t span, double* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (is_first[i]) w[i] = (double)(low + (int64_t)(splitmix_draw(seed, (uint64_t)rank[i]) % (uint64_t)span));
}

__global__ void copy_pair_weights(int64_t n, const uint64_t* __restrict__ keys,
                                  const int64_t* __restrict__ pos, const int32_t* __restrict__ flags,
                                  const int64_t* __restrict__ seg_first_pos, double* __restrict__ w) {
  // seg_first_pos[i] = position (in list order) of the first appearance of keys[i]'s pair
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!flags[i]) w[pos[i]] = w[seg_first_pos[i]];
}

__global__ void propagate_first(int64_t n, const int32_t* __restrict__ flags,
                                const int64_t* __restrict__ pos, const int64_t* __restrict__ segid,
                                const int64_t* __restrict__ seg_pos, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = seg_pos[segid[i] - 1];
}

__global__ void scatter_seg_pos(int64_t n, const int32_t* __restrict__ flags,
                                const int64_t* __restrict__ segid, const int64_t* __restrict__ pos,
                                int64_t* __restrict__ seg_pos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flags[i]) seg_pos[segid[i] - 1] = pos[i];
}


// ---------------------------------------------------------------------------
// Degree-ordered relabelling (the traversal layout of DESIGN.md §3).  Vertices
// are renumbered by descending degree (ties by id), so the vertices most
// traversals touch form a dense low-id prefix: at R-MAT s24 the first 1.5 M
// new ids (a 192 KB bitmap) receive 91 % of all edge endpoints.
// ---------------------------------------------------------------------------
__global__ void degree_keys(int64_t n, const int64_t* __restrict__ off, uint32_t* __restrict__ deg,
                            int32_t* __restrict__ ids) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    deg[i] = (uint32_t)(off[i + 1] - off[i]);
    ids[i] = (int32_t)i;
  }
}

__global__ void invert_order(int64_t n, const int32_t* __restrict__ order, int32_t* __restrict__ rank) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    rank[order[r]] = (int32_t)r;
}

__global__ void permuted_degrees(int64_t n, const int32_t* __restrict__ order,
                                 const int64_t* __restrict__ off, int64_t* __restrict__ deg) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    deg[r] = off[order[r] + 1] - off[order[r]];
}

// Warp per new row r = old row order[r]: its entries in their old order with
// columns renamed (key), the new row id and the source position.
__global__ void relabel_fill(int64_t n, const int32_t* __restrict__ order,
                             const int32_t* __restrict__ rank, const int64_t* __restrict__ off,
                             const int32_t* __restrict__ idx, const int64_t* __restrict__ uoff,
                             int32_t* __restrict__ ukey, int32_t* __restrict__ urow,
                             int64_t* __restrict__ usrc) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n; r += nw) {
    const int64_t o = order[r];
    const int64_t lo = off[o], hi = off[o + 1], base = uoff[r] - lo;
    for (int64_t p = lo + lane; p < hi; p += 32) {
      ukey[base + p] = rank[idx[p]];
      urow[base + p] = (int32_t)r;
      if (usrc) usrc[base + p] = p;
    }
  }
}

template <class T>
__global__ void gather_via(int64_t n, const int64_t* __restrict__ perm, const int64_t* __restrict__ via,
                           const T* __restrict__ in, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[via[perm[i]]];
}


static gb_status row_ids(gb_ctx* ctx, Arena& ar, int64_t nrows, int64_t nnz,
                         const int64_t* off, int32_t** out) {
  cudaStream_t s = stream_of(ctx);
  int32_t* marks = ar.alloc<int32_t>(nnz + 1);
  int32_t* rows = ar.alloc<int32_t>(nnz + 1);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(marks, 0, sizeof(int32_t) * (nnz + 1), s));
  row_start_marks<<<grid_for(ctx, nrows, 256), 256, 0, s>>>(nrows, nnz, off, marks);
  // entries before the first non-empty row belong to row 0 only when row 0 is
  // non-empty; the marks count every row start at or before the position.
  size_t tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, marks, rows, nnz, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::InclusiveSum(tmp, tb, marks, rows, nnz, s));
  *out = rows;
  return GB_OK;
}


}  // namespace gb

using namespace gb;

extern "C" {

gb_status gb_rmat_generate(gb_ctx* ctx, int32_t scale, int64_t nedges, uint64_t seed, double a,
                           double t_ab, double t_abc, int32_t* src, int32_t* dst) {
  if (scale < 0 || scale > 30) return set_error(ctx, GB_ERR_ARG, "scale out of range");
  cudaStream_t s = stream_of(ctx);
  rmat_kernel<<<grid_for(ctx, nedges, 256, 16), 256, 0, s>>>(scale, nedges, seed, a, t_ab,
                                                             t_abc, src, dst);
  GB_LAUNCH_CHECK(ctx);
  return GB_OK;
}

gb_status gb_edges_to_csr(gb_ctx* ctx, int64_t n, int64_t m, const int32_t* src,
                          const int32_t* dst, int32_t undirected, int64_t* out_offsets,
                          int32_t* out_indices, int64_t* nnz_out) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  int bits = bits_for(n);
  int64_t nk = undirected ? 2 * m : m;
  uint64_t sentinel = (uint64_t)1 << (2 * bits);
  uint64_t* k0 = ar.alloc<uint64_t>(nk);
  uint64_t* k1 = ar.alloc<uint64_t>(nk);
  int64_t* cnt = ar.alloc<int64_t>(1);
  GB_ARENA_CHECK(ctx, ar);
  if (nk > 0) {
    edge_keys_kernel<<<grid_for(ctx, m, 256), 256, 0, s>>>(m, src, dst, bits, undirected,
                                                           sentinel, k0);
    cub::DoubleBuffer<uint64_t> db(k0, k1);
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, db, nk, 0, 2 * bits + 1, s);
    void* tmp = ar.raw(tb);
    GB_ARENA_CHECK(ctx, ar);
    GB_CUDA(ctx, cub::DeviceRadixSort::SortKeys(tmp, tb, db, nk, 0, 2 * bits + 1, s));
    uint64_t* sorted = db.Current();
    uint64_t* uniq = db.Alternate();
    size_t tb2 = 0;
    cub::DeviceSelect::Unique(nullptr, tb2, sorted, uniq, cnt, nk, s);
    void* tmp2 = ar.raw(tb2);
    GB_ARENA_CHECK(ctx, ar);
    GB_CUDA(ctx, cub::DeviceSelect::Unique(tmp2, tb2, sorted, uniq, cnt, nk, s));
    int64_t nu = 0;
    GB_TRY(read_i64(ctx, cnt, &nu));
    // drop the sentinel (self loops) if present: it sorts last
    uint64_t last = 0;
    if (nu > 0) {
      GB_TRY(read_i64(ctx, (const int64_t*)(uniq + nu - 1), (int64_t*)&last));
      if (last == sentinel) --nu;
    }
    keys_to_cols<<<grid_for(ctx, nu, 256), 256, 0, s>>>(nu, uniq, ((uint64_t)1 << bits) - 1,
                                                        out_indices);
    offsets_from_sorted_rows<<<grid_for(ctx, nu + 1, 256), 256, 0, s>>>(
        nu, n, KeyRow{uniq, bits}, out_offsets);
    GB_LAUNCH_CHECK(ctx);
    *nnz_out = nu;
  } else {
    GB_CUDA(ctx, cudaMemsetAsync(out_offsets, 0, sizeof(int64_t) * (n + 1), s));
    *nnz_out = 0;
  }
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  return GB_OK;
}

gb_status gb_build_csr(gb_ctx* ctx, int64_t nrows, int64_t ncols, int64_t n,
                       const int64_t* rows, const int64_t* cols, const void* vals,
                       int32_t dtype, int32_t dedup_op, int64_t* out_offsets,
                       int32_t* out_indices, void* out_vals, int64_t* nnz_out) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  if (n == 0) {
    GB_CUDA(ctx, cudaMemsetAsync(out_offsets, 0, sizeof(int64_t) * (nrows + 1), s));
    GB_CUDA(ctx, cudaStreamSynchronize(s));
    *nnz_out = 0;
    return GB_OK;
  }
  int* bad = ar.alloc<int>(2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(bad, 0, sizeof(int), s));
  coo_bounds<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, rows, cols, nrows, ncols, bad);
  int hbad = 0;
  GB_CUDA(ctx, cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  if (hbad & 1) return set_error(ctx, GB_ERR_INDEX, "row index out of bounds for %lld rows", (long long)nrows);
  if (hbad & 2) return set_error(ctx, GB_ERR_INDEX, "column index out of bounds for %lld columns", (long long)ncols);

  int bits = bits_for(ncols > 1 ? ncols : 2);
  int rbits = bits_for(nrows > 1 ? nrows : 2);
  if (bits + rbits > 63) return set_error(ctx, GB_ERR_UNSUPPORTED, "matrix too large for 64-bit keys");
  uint64_t* ka = ar.alloc<uint64_t>(n);
  uint64_t* kb = ar.alloc<uint64_t>(n);
  int64_t* pa = ar.alloc<int64_t>(n);
  int64_t* pb = ar.alloc<int64_t>(n);
  int32_t* flags = ar.alloc<int32_t>(n + 1);
  int64_t* pos = ar.alloc<int64_t>(n + 1);
  uint64_t* ukeys = ar.alloc<uint64_t>(n);
  GB_ARENA_CHECK(ctx, ar);
  coo_keys<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, rows, cols, bits, ka);
  iota64<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, pa);
  cub::DoubleBuffer<uint64_t> dk(ka, kb);
  cub::DoubleBuffer<int64_t> dv(pa, pb);
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, n, 0, bits + rbits, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, n, 0, bits + rbits, s));
  const uint64_t* keys = dk.Current();
  const int64_t* perm = dv.Current();
  unique_flags<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, keys, flags);
  // exclusive positions of unique keys; flags[n] = 0 so pos[n] = unique count
  GB_CUDA(ctx, cudaMemsetAsync(flags + n, 0, sizeof(int32_t), s));
  size_t tb2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, flags, pos, n + 1, s);
  void* tmp2 = ar.raw(tb2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp2, tb2, flags, pos, n + 1, s));
  uint64_t cmask = ((uint64_t)1 << bits) - 1;
  if (dtype == GB_I64)
    fold_segments<int64_t><<<grid_for(ctx, n, 256), 256, 0, s>>>(
        n, keys, flags, pos, perm, (const int64_t*)vals, dedup_op, bits, cmask, out_indices,
        ukeys, (int64_t*)out_vals);
  else
    fold_segments<double><<<grid_for(ctx, n, 256), 256, 0, s>>>(
        n, keys, flags, pos, perm, (const double*)vals, dedup_op, bits, cmask, out_indices,
        ukeys, (double*)out_vals);
  int64_t nu = 0;
  GB_TRY(read_i64(ctx, pos + n, &nu));
  offsets_from_sorted_rows<<<grid_for(ctx, nu + 1, 256), 256, 0, s>>>(nu, nrows,
                                                                      KeyRow{ukeys, bits},
                                                                      out_offsets);
  GB_LAUNCH_CHECK(ctx);
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  *nnz_out = nu;
  return GB_OK;
}

gb_status gb_transpose_csr(gb_ctx* ctx, const gb_csr* a, int64_t* out_offsets,
                           int32_t* out_indices, void* out_vals) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  int64_t nnz = a->nnz;
  if (nnz == 0) {
    GB_CUDA(ctx, cudaMemsetAsync(out_offsets, 0, sizeof(int64_t) * (a->ncols + 1), s));
    return GB_OK;
  }
  int32_t* rows = nullptr;
  GB_TRY(row_ids(ctx, ar, a->nrows, nnz, a->offsets, &rows));
  int32_t* ka = ar.alloc<int32_t>(nnz);
  int32_t* kb = ar.alloc<int32_t>(nnz);
  int64_t* pa = ar.alloc<int64_t>(nnz);
  int64_t* pb = ar.alloc<int64_t>(nnz);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemcpyAsync(ka, a->indices, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, s));
  iota64<<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, pa);
  cub::DoubleBuffer<int32_t> dk(ka, kb);
  cub::DoubleBuffer<int64_t> dv(pa, pb);
  int cbits = bits_for(a->ncols > 1 ? a->ncols : 2);
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, nnz, 0, cbits, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, nnz, 0, cbits, s));
  const int32_t* scols = dk.Current();
  const int64_t* perm = dv.Current();
  gather_kernel<int32_t><<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, perm, rows, out_indices);
  if (a->values && out_vals)
    gather_kernel<int64_t><<<grid_for(ctx, nnz, 256), 256, 0, s>>>(
        nnz, perm, (const int64_t*)a->values, (int64_t*)out_vals);
  offsets_from_sorted_rows<<<grid_for(ctx, nnz + 1, 256), 256, 0, s>>>(
      nnz, a->ncols, IdxRow{scols}, out_offsets);
  GB_LAUNCH_CHECK(ctx);
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  return GB_OK;
}

gb_status gb_csr_row_ids(gb_ctx* ctx, int64_t nrows, int64_t nnz, const int64_t* offsets,
                         int32_t* out) {
  if (nnz == 0) return GB_OK;
  Arena ar(ctx);
  int32_t* rows = nullptr;
  GB_TRY(row_ids(ctx, ar, nrows, nnz, offsets, &rows));
  GB_CUDA(ctx, cudaMemcpyAsync(out, rows, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice,
                               stream_of(ctx)));
  return GB_OK;
}

gb_status gb_csr_equal(gb_ctx* ctx, const gb_csr* a, const gb_csr* b, int32_t* equal) {
  *equal = 0;
  if (a->nrows != b->nrows || a->ncols != b->ncols || a->nnz != b->nnz) return GB_OK;
  if ((a->values == nullptr) != (b->values == nullptr)) return GB_OK;
  if (!a->values && (a->iso_i64 != b->iso_i64 || a->iso_f64 != b->iso_f64)) return GB_OK;
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  int* diff = ar.alloc<int>(1);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(diff, 0, sizeof(int), s));
  all_equal_kernel<int64_t><<<grid_for(ctx, a->nrows + 1, 256), 256, 0, s>>>(
      a->nrows + 1, a->offsets, b->offsets, diff);
  if (a->nnz) {
    all_equal_kernel<int32_t><<<grid_for(ctx, a->nnz, 256), 256, 0, s>>>(a->nnz, a->indices,
                                                                         b->indices, diff);
    if (a->values)
      all_equal_kernel<int64_t><<<grid_for(ctx, a->nnz, 256), 256, 0, s>>>(
          a->nnz, (const int64_t*)a->values, (const int64_t*)b->values, diff);
  }
  int h = 0;
  GB_CUDA(ctx, cudaMemcpyAsync(&h, diff, sizeof(int), cudaMemcpyDeviceToHost, s));
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  *equal = h ? 0 : 1;
  return GB_OK;
}

gb_status gb_values_iso(gb_ctx* ctx, int64_t n, const void* vals, int32_t dtype, int32_t* iso) {
  *iso = 0;
  if (n == 0) { *iso = 1; return GB_OK; }
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  int* diff = ar.alloc<int>(1);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(diff, 0, sizeof(int), s));
  // bitwise comparison: -0.0 vs 0.0 and NaN payloads count as different
  iso_kernel<int64_t><<<grid_for(ctx, n, 256), 256, 0, s>>>(n, (const int64_t*)vals, diff);
  int h = 0;
  GB_CUDA(ctx, cudaMemcpyAsync(&h, diff, sizeof(int), cudaMemcpyDeviceToHost, s));
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  *iso = h ? 0 : 1;
  return GB_OK;
}

gb_status gb_values_minmax(gb_ctx* ctx, int64_t n, const void* vals, int32_t dtype,
                           double* mn, double* mx) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  double* out = ar.alloc<double>(2);
  GB_ARENA_CHECK(ctx, ar);
  init_minmax<<<1, 1, 0, s>>>(out);
  if (n > 0) {
    if (dtype == GB_I64)
      minmax_kernel<int64_t><<<grid_for(ctx, n, 256), 256, 0, s>>>(n, (const int64_t*)vals, out);
    else
      minmax_kernel<double><<<grid_for(ctx, n, 256), 256, 0, s>>>(n, (const double*)vals, out);
  }
  unsigned long long h[2];
  GB_CUDA(ctx, cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, s));
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  auto unmap = [](unsigned long long b) {
    b = (b & 0x8000000000000000ull) ? (b & 0x7fffffffffffffffull) : ~b;
    double d;
    memcpy(&d, &b, 8);
    return d;
  };
  *mn = n ? unmap(h[0]) : INFINITY;
  *mx = n ? unmap(h[1]) : -INFINITY;
  return GB_OK;
}

gb_status gb_assign_weights(gb_ctx* ctx, int64_t n, int64_t nnz, const int32_t* src,
                            const int32_t* dst, uint64_t seed, int64_t low, int64_t high,
                            double* w) {
  if (low > high) return set_error(ctx, GB_ERR_VALUE, "low %lld exceeds high %lld", (long long)low, (long long)high);
  if (nnz == 0) return GB_OK;
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  int bits = bits_for(n > 1 ? n : 2);
  uint64_t* ka = ar.alloc<uint64_t>(nnz);
  uint64_t* kb = ar.alloc<uint64_t>(nnz);
  int64_t* pa = ar.alloc<int64_t>(nnz);
  int64_t* pb = ar.alloc<int64_t>(nnz);
  int32_t* flags = ar.alloc<int32_t>(nnz);
  int32_t* is_first = ar.alloc<int32_t>(nnz);
  int64_t* rank = ar.alloc<int64_t>(nnz);
  int64_t* segid = ar.alloc<int64_t>(nnz);
  int64_t* seg_pos = ar.alloc<int64_t>(nnz);
  int64_t* firstpos = ar.alloc<int64_t>(nnz);
  GB_ARENA_CHECK(ctx, ar);
  pair_keys<<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, src, dst, bits, ka, pa);
  cub::DoubleBuffer<uint64_t> dk(ka, kb);
  cub::DoubleBuffer<int64_t> dv(pa, pb);
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, nnz, 0, 2 * bits, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, nnz, 0, 2 * bits, s));
  const uint64_t* keys = dk.Current();
  const int64_t* pos = dv.Current();  // stable: first entry of a key = first appearance
  unique_flags<<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, keys, flags);
  GB_CUDA(ctx, cudaMemsetAsync(is_first, 0, sizeof(int32_t) * nnz, s));
  mark_first<<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, flags, pos, is_first);
  size_t tb2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, is_first, rank, nnz, s);
  size_t tb3 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb3, flags, segid, nnz, s);
  void* tmp2 = ar.raw(tb2 > tb3 ? tb2 : tb3);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp2, tb2, is_first, rank, nnz, s));
  draw_firsts<<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, is_first, rank, seed, low,
                                                      high - low + 1, w);
  GB_CUDA(ctx, cub::DeviceScan::InclusiveSum(tmp2, tb3, flags, segid, nnz, s));
  scatter_seg_pos<<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, flags, segid, pos, seg_pos);
  propagate_first<<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, flags, pos, segid, seg_pos,
                                                          firstpos);
  copy_pair_weights<<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, keys, pos, flags, firstpos, w);
  GB_LAUNCH_CHECK(ctx);
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  return GB_OK;
}


gb_status gb_degree_order(gb_ctx* ctx, int64_t n, const int64_t* offsets, int32_t* order,
                          int32_t* rank) {
  if (n <= 0) return GB_OK;
  if (n > INT32_MAX) return set_error(ctx, GB_ERR_UNSUPPORTED, "degree order needs n < 2^31");
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  uint32_t* ka = ar.alloc<uint32_t>(n);
  uint32_t* kb = ar.alloc<uint32_t>(n);
  int32_t* va = ar.alloc<int32_t>(n);
  GB_ARENA_CHECK(ctx, ar);
  degree_keys<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, offsets, ka, va);
  // radix sort is stable: equal degrees keep ascending ids
  cub::DoubleBuffer<uint32_t> dk(ka, kb);
  cub::DoubleBuffer<int32_t> dv(va, order);
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, dk, dv, n, 0, 32, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceRadixSort::SortPairsDescending(tmp, tb, dk, dv, n, 0, 32, s));
  if (dv.Current() != order)
    GB_CUDA(ctx, cudaMemcpyAsync(order, dv.Current(), sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
  invert_order<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, order, rank);
  GB_LAUNCH_CHECK(ctx);
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  return GB_OK;
}

gb_status gb_csr_relabel_t(gb_ctx* ctx, const gb_csr* a, const int32_t* order, const int32_t* rank,
                           int64_t* out_offsets, int32_t* out_indices, void* out_vals) {
  const int64_t n = a->nrows, nnz = a->nnz;
  if (a->nrows != a->ncols) return set_error(ctx, GB_ERR_SHAPE, "relabelling needs a square matrix");
  cudaStream_t s = stream_of(ctx);
  if (nnz == 0) {
    GB_CUDA(ctx, cudaMemsetAsync(out_offsets, 0, sizeof(int64_t) * (n + 1), s));
    return GB_OK;
  }
  Arena ar(ctx);
  int64_t* deg = ar.alloc<int64_t>(n + 1);
  int64_t* uoff = ar.alloc<int64_t>(n + 1);
  int32_t* ka = ar.alloc<int32_t>(nnz);
  int32_t* kb = ar.alloc<int32_t>(nnz);
  int32_t* urow = ar.alloc<int32_t>(nnz);
  int64_t* pa = ar.alloc<int64_t>(nnz);
  int64_t* pb = ar.alloc<int64_t>(nnz);
  int64_t* usrc = a->values ? ar.alloc<int64_t>(nnz) : nullptr;
  GB_ARENA_CHECK(ctx, ar);
  // U = P A P^T with rows in new order, columns renamed but not yet sorted
  permuted_degrees<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, order, a->offsets, deg);
  GB_CUDA(ctx, cudaMemsetAsync(deg + n, 0, sizeof(int64_t), s));
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, deg, uoff, n + 1, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp, tb, deg, uoff, n + 1, s));
  relabel_fill<<<grid_for(ctx, n * 32, 256, 16), 256, 0, s>>>(n, order, rank, a->offsets, a->indices,
                                                              uoff, ka, urow, usrc);
  iota64<<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, pa);
  // stable sort by renamed column: the transpose of U, rows ascending in
  // every output row (P A^T P^T with sorted columns)
  cub::DoubleBuffer<int32_t> dk(ka, kb);
  cub::DoubleBuffer<int64_t> dv(pa, pb);
  size_t tb2 = 0;
  const int cbits = bits_for(n > 1 ? n : 2);
  cub::DeviceRadixSort::SortPairs(nullptr, tb2, dk, dv, nnz, 0, cbits, s);
  void* tmp2 = ar.raw(tb2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceRadixSort::SortPairs(tmp2, tb2, dk, dv, nnz, 0, cbits, s));
  const int32_t* skeys = dk.Current();
  const int64_t* perm = dv.Current();
  gather_kernel<int32_t><<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, perm, urow, out_indices);
  if (a->values && out_vals)
    gather_via<int64_t><<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, perm, usrc,
                                                                (const int64_t*)a->values,
                                                                (int64_t*)out_vals);
  offsets_from_sorted_rows<<<grid_for(ctx, nnz + 1, 256), 256, 0, s>>>(nnz, n, IdxRow{skeys},
                                                                       out_offsets);
  GB_LAUNCH_CHECK(ctx);
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  return GB_OK;
}


}  // extern "C"
