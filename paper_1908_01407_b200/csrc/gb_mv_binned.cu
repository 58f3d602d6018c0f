// Row-binned pull SpMV: the masked pull (kernels.py:153-229) and the
// reference's row split (Partition.ROW_SPLIT, kernels.py:142-143) as
// row-granular work.
//
// The edge-balanced row tiles (gb_rowtiles.cuh) walk every stored entry of
// the matrix: a masked-out row still costs its share of tile staging, owner
// search, fold slots and warp scan.  At R-MAT s24 with a 50 % mask that is
// half of 520 M slots for nothing, and with a 90 % mask the kernel spends
// 1.06 ms on 52 M entries.  Here the rows are binned ONCE per matrix by
// length and every bin tests the mask per row before touching an entry:
//
//   short  (1..16 entries, 6.4 M rows / 4.6 % of the entries at s24): one
//          lane per row, its entries loaded through L1 (a row is <= 2 sectors);
//   medium (17..512, 2.3 M rows / 31 %): a half-warp per row, two rows at a
//          time, 128 entries (8 loads + 8 gathers per lane) per pass; the 32
//          rows of a group are mask-tested with one ballot so only allowed
//          rows are walked;
//   long   (> 512, 190 K rows / 64 %): 512-entry tiles at absolute multiples of
//          512 (a full tile: lane l takes entries 32k + l, gathers in two
//          waves of 8), 32 tile descriptors loaded and mask-tested per warp batch,
//          warp fold, one atomic fold per tile (out is prefilled with the
//          identity).
//
// Each warp runs its stride of the long tiles, then of the medium groups,
// then of the short groups, so no bin waits for another.  Commutative folds
// only (the products of a row are combined in tree order).  Work counters
// are exact: reads = entries of allowed rows, multiplies = those with
// u(j) != identity, adds = multiplies - rows with >= 1 multiply (long rows
// through the `hasmul` bitmap, deduplicated by mv_pull_finish).
#include <type_traits>

#include <cub/cub.cuh>

#include "gb_common.cuh"

namespace gb {

constexpr int kBinShort = 16;
constexpr int kBinLong = 512;

#ifndef GB_MVB_MINB
#define GB_MVB_MINB 4
#endif


template <class T>
__device__ __forceinline__ T bin_aval(const T* vals, T iso, int64_t p) {
  return vals ? __ldg(vals + p) : iso;
}

// QM: medium rows a quarter-warp each, four per round trip (the column
// stripes of regular graphs: uniform s24 1.81 -> 1.70 ms), else a half-warp
// each, two per round trip (R-MAT s24: 1.22 vs 1.25 ms quartered)
template <class T, int ADD, int MUL, bool VALS, bool QM>
__global__ void __launch_bounds__(256, GB_MVB_MINB)
mv_pull_binned(int64_t nL, const int32_t* __restrict__ L_row, const int64_t* __restrict__ L_beg,
               const int64_t* __restrict__ L_end, int64_t nM, const int32_t* __restrict__ M_rows,
               int64_t nS, const int32_t* __restrict__ S_rows, const int64_t* __restrict__ off,
               const int32_t* __restrict__ idx, const T* __restrict__ vals, T iso,
               const T* __restrict__ u, const uint32_t* __restrict__ mask, int add_rt,
               int mult_rt, T* __restrict__ out, unsigned long long* __restrict__ counters,
               uint32_t* __restrict__ hasmul, int accumulate) {
  const int add_op = ADD >= 0 ? ADD : add_rt;
  const int mult_op = MUL >= 0 ? MUL : mult_rt;
  const T ident = op_identity<T>(add_op);
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long c_reads = 0, c_muls = 0, c_rows = 0;  // warp-wide work (lanes 0 / 16)
  unsigned long long s_reads = 0, s_muls = 0, s_rows = 0;  // per lane (short rows)
  // fold a gathered value (identity values are skipped, kernels.py:167)
  auto fold_one_v = [&](T& acc, int& cnt, T x, int64_t p) {
    if (x != ident) {
      acc = op_fold<T>(add_op, acc, op_pair<T>(mult_op, VALS ? bin_aval(vals, iso, p) : iso, x));
      ++cnt;
    }
  };

  // ---- long rows: 512-entry tiles, 32 tile descriptors per warp batch -----
  // Lane l loads descriptor g*32+l (coalesced) and tests its row's mask bit;
  // the warp then walks the allowed tiles of the batch.  Consecutive tiles
  // mostly belong to one hub row, so a batch is usually all-in or all-out.
  for (int64_t g = w0; g * 32 < nL; g += nw) {
    const int64_t ti = g * 32 + lane;
    int32_t row = -1;
    int64_t tb = 0, te = 0;
    if (ti < nL) {
      row = __ldg(L_row + ti);
      tb = __ldg(L_beg + ti);
      te = __ldg(L_end + ti);
    }
    uint32_t bal = __ballot_sync(GB_FULL, row >= 0 && (!mask || bit_test(mask, row)));
    while (bal) {
      const int j = __ffs(bal) - 1;
      bal &= bal - 1;
      const int32_t rr = __shfl_sync(GB_FULL, row, j);
      const int64_t beg = __shfl_sync(GB_FULL, tb, j), end = __shfl_sync(GB_FULL, te, j);
      T acc = ident;
      int cnt = 0;
      if (end - beg == kBinLong) {
        // a full 512-aligned tile, lane-consecutive: lane l takes entries
        // 32k + l (coalesced 128-byte index loads), so neighbouring sorted
        // columns that share a line of u coalesce into one L1 wavefront
        // (s24 50 % mask 1.27 -> 1.22 ms against two 256-bit loads per lane
        // of 16 consecutive entries); gathers in two waves of 8
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          int32_t cols[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) cols[k] = ld_stream(idx + beg + 256 * w + 32 * k + lane);
          T x[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) x[k] = ld_gather(u + cols[k]);
#pragma unroll
          for (int k = 0; k < 8; ++k) fold_one_v(acc, cnt, x[k], beg + 256 * w + 32 * k + lane);
        }
      } else {
        // a partial tile (the row's first or last): lane-strided, coalesced
        for (int64_t base = beg; base < end; base += 256) {
          int32_t cols[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int64_t p = base + 32 * k + lane;
            cols[k] = p < end ? ld_stream(idx + p) : 0;
          }
          T x[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) x[k] = base + 32 * k + lane < end ? ld_gather(u + cols[k]) : ident;
#pragma unroll
          for (int k = 0; k < 8; ++k) fold_one_v(acc, cnt, x[k], base + 32 * k + lane);
        }
      }
      acc = warp_fold<T>(add_op, acc);
      cnt = (int)__reduce_add_sync(GB_FULL, (unsigned)cnt);
      if (lane == 0) {
        c_reads += (unsigned long long)(end - beg);
        if (cnt > 0) {
          atomic_fold<T>(add_op, out + rr, acc);
          c_muls += cnt;
          if (hasmul) atomicOr(hasmul + (rr >> 5), 1u << (rr & 31));
        }
      }
    }
  }

  // ---- medium rows: a half-warp (QM: quarter-warp) per allowed row ---------
  for (int64_t g = w0; g * 32 < nM; g += nw) {
    const int64_t i = g * 32 + lane;
    const int32_t r = i < nM ? __ldg(M_rows + i) : -1;
    const bool ok = r >= 0 && (!mask || bit_test(mask, r));
    int64_t lo = 0, hi = 0;
    if (ok) {
      lo = __ldg(off + r);
      hi = __ldg(off + r + 1);
    }
    uint32_t bal = __ballot_sync(GB_FULL, ok);
    // QM: a quarter-warp per row, four rows at a time, 64 entries a pass
    if (QM) while (bal) {
      int js[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        js[k] = bal ? __ffs(bal) - 1 : -1;
        if (bal) bal &= bal - 1;
      }
      const int qq = lane >> 3, ql = lane & 7;
      const int mine = qq == 0 ? js[0] : qq == 1 ? js[1] : qq == 2 ? js[2] : js[3];
      const int src = mine >= 0 ? mine : js[0];
      const int32_t rr = __shfl_sync(GB_FULL, r, src);
      int64_t l = __shfl_sync(GB_FULL, lo, src), h = __shfl_sync(GB_FULL, hi, src);
      if (mine < 0) h = l;  // fewer than four rows left: this quarter idles
      T acc = ident;
      int cnt = 0;
      for (int64_t base = l; base < h; base += 64) {
        int32_t cols[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int64_t p = base + 8 * k + ql;
          cols[k] = p < h ? ld_stream(idx + p) : 0;
        }
        T x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = base + 8 * k + ql < h ? ld_gather(u + cols[k]) : ident;
#pragma unroll
        for (int k = 0; k < 8; ++k) fold_one_v(acc, cnt, x[k], base + 8 * k + ql);
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) acc = op_fold<T>(add_op, acc, __shfl_xor_sync(GB_FULL, acc, o));
      cnt = (int)__reduce_add_sync(0xffu << (8 * qq), (unsigned)cnt);
      if (ql == 0 && h > l) {
        c_reads += (unsigned long long)(h - l);
        if (cnt > 0) {
          c_muls += cnt;
          if (accumulate) {
            out[rr] = op_fold<T>(add_op, out[rr], acc);
            if (hasmul) atomicOr(hasmul + (rr >> 5), 1u << (rr & 31));
          } else {
            out[rr] = acc;
            ++c_rows;
          }
        }
      }
    }
    // else a half-warp per row, two rows at a time, 128 entries a pass
    const int half = lane >> 4, hl = lane & 15;
    if (!QM) while (bal) {
      const int j0 = __ffs(bal) - 1;
      bal &= bal - 1;
      const int j1 = bal ? __ffs(bal) - 1 : -1;
      if (bal) bal &= bal - 1;
      const int src = half ? (j1 >= 0 ? j1 : j0) : j0;
      const int32_t rr = __shfl_sync(GB_FULL, r, src);
      int64_t l = __shfl_sync(GB_FULL, lo, src), h = __shfl_sync(GB_FULL, hi, src);
      if (half && j1 < 0) h = l;  // no second row: the upper half idles
      T acc = ident;
      int cnt = 0;
      for (int64_t base = l; base < h; base += 128) {
        int32_t cols[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int64_t p = base + 16 * k + hl;
          cols[k] = p < h ? ld_stream(idx + p) : 0;
        }
        T x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = base + 16 * k + hl < h ? ld_gather(u + cols[k]) : ident;
#pragma unroll
        for (int k = 0; k < 8; ++k) fold_one_v(acc, cnt, x[k], base + 16 * k + hl);
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) acc = op_fold<T>(add_op, acc, __shfl_xor_sync(GB_FULL, acc, o));
      cnt = (int)__reduce_add_sync(0xffffu << (16 * half), (unsigned)cnt);
      if (hl == 0 && h > l) {
        c_reads += (unsigned long long)(h - l);
        if (cnt > 0) {
          c_muls += cnt;
          if (accumulate) {  // a column stripe: fold into the earlier stripes' value
            out[rr] = op_fold<T>(add_op, out[rr], acc);
            if (hasmul) atomicOr(hasmul + (rr >> 5), 1u << (rr & 31));
          } else {
            out[rr] = acc;
            ++c_rows;
          }
        }
      }
    }
  }

  // ---- short rows: a lane per row ------------------------------------------
  for (int64_t g = w0; g * 32 < nS; g += nw) {
    const int64_t i = g * 32 + lane;
    const int32_t r = i < nS ? __ldg(S_rows + i) : -1;
    if (r >= 0 && (!mask || bit_test(mask, r))) {
      const int64_t lo = __ldg(off + r);
      const int len = (int)(__ldg(off + r + 1) - lo);
      int32_t cols[kBinShort];
#pragma unroll
      for (int q = 0; q < kBinShort; ++q) cols[q] = q < len ? __ldg(idx + lo + q) : 0;
      T acc = ident;
      int cnt = 0;
      // gathers in two waves of 8, every load of a wave in flight together
#pragma unroll
      for (int w = 0; w < kBinShort / 8; ++w) {
        T x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = 8 * w + k < len ? ld_gather(u + cols[8 * w + k]) : ident;
#pragma unroll
        for (int k = 0; k < 8; ++k) fold_one_v(acc, cnt, x[k], lo + 8 * w + k);
      }
      s_reads += (unsigned long long)len;
      if (cnt > 0) {
        s_muls += cnt;
        if (accumulate) {
          out[r] = op_fold<T>(add_op, out[r], acc);
          if (hasmul) atomicOr(hasmul + (r >> 5), 1u << (r & 31));
        } else {
          out[r] = acc;
          ++s_rows;
        }
      }
    }
  }

  if (counters) {
    // warp-level totals straight to global: no block barrier, so a warp
    // that finishes its stride leaves at once
    const long long r_ = warp_sum_ll((long long)(s_reads + c_reads));
    const long long m_ = warp_sum_ll((long long)(s_muls + c_muls));
    const long long w_ = warp_sum_ll((long long)(s_rows + c_rows));
    if (lane == 0) {
      if (r_) atomicAdd(counters + 0, (unsigned long long)r_);
      if (m_) atomicAdd(counters + 1, (unsigned long long)m_);
      if (m_ - w_) atomicAdd(counters + 2, (unsigned long long)(m_ - w_));  // long rows: mv_pull_finish
    }
  }
}

// ---------------------------------------------------------------------------
// plan: per row, (short, medium) flags packed in one u64 (two 32-bit
// counters, n < 2^32) and the long tiles it spans in a second scan
// ---------------------------------------------------------------------------
__global__ void bin_count(int64_t n, const int64_t* __restrict__ off, uint64_t* __restrict__ sm,
                          int64_t* __restrict__ lt) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t a = 0;
    int64_t t = 0;
    if (r < n) {
      const int64_t lo = off[r], hi = off[r + 1], len = hi - lo;
      if (len >= 1 && len <= kBinShort) a = 1;
      else if (len > kBinShort && len <= kBinLong) a = 1ull << 32;
      else if (len > kBinLong) t = (hi - 1) / kBinLong - lo / kBinLong + 1;
    }
    sm[r] = a;
    lt[r] = t;
  }
}

__global__ void bin_fill(int64_t n, const int64_t* __restrict__ off, const uint64_t* __restrict__ sm,
                         const int64_t* __restrict__ lt, int32_t* __restrict__ S_rows,
                         int32_t* __restrict__ M_rows, int32_t* __restrict__ L_row,
                         int64_t* __restrict__ L_beg, int64_t* __restrict__ L_end) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = off[r], hi = off[r + 1], len = hi - lo;
    if (len >= 1 && len <= kBinShort) {
      S_rows[sm[r] & 0xffffffffull] = (int32_t)r;
    } else if (len > kBinShort && len <= kBinLong) {
      M_rows[sm[r] >> 32] = (int32_t)r;
    } else if (len > kBinLong) {
      int64_t p = lt[r];
      for (int64_t b = lo / kBinLong * kBinLong; b < hi; b += kBinLong, ++p) {
        L_row[p] = (int32_t)r;
        L_beg[p] = b > lo ? b : lo;
        L_end[p] = b + kBinLong < hi ? b + kBinLong : hi;
      }
    }
  }
}

// exclusive scans of the flags; returns the three totals on the host
static gb_status bin_scan(gb_ctx* ctx, Arena& ar, const gb_csr* a, uint64_t** sm_out,
                          int64_t** lt_out, int64_t* counts) {
  cudaStream_t s = stream_of(ctx);
  const int64_t n = a->nrows;
  uint64_t* sm = ar.alloc<uint64_t>(n + 1);
  uint64_t* smx = ar.alloc<uint64_t>(n + 1);
  int64_t* lt = ar.alloc<int64_t>(n + 1);
  int64_t* ltx = ar.alloc<int64_t>(n + 1);
  GB_ARENA_CHECK(ctx, ar);
  bin_count<<<grid_for(ctx, n + 1, 256), 256, 0, s>>>(n, a->offsets, sm, lt);
  size_t t1 = 0, t2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t1, sm, smx, n + 1, s);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, lt, ltx, n + 1, s);
  void* tmp = ar.raw(t1 > t2 ? t1 : t2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp, t1, sm, smx, n + 1, s));
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp, t2, lt, ltx, n + 1, s));
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 3);
  int64_t h[2];
  GB_CUDA(ctx, cudaMemcpyAsync(h, smx + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  GB_CUDA(ctx, cudaMemcpyAsync(h + 1, ltx + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  counts[0] = (int64_t)((uint64_t)h[0] & 0xffffffffull);  // short rows
  counts[1] = (int64_t)((uint64_t)h[0] >> 32);           // medium rows
  counts[2] = h[1];                                      // long tiles
  *sm_out = smx;
  *lt_out = ltx;
  return GB_OK;
}

template <class T, int ADD, int MUL, bool VALS>
static void launch_binned_k(gb_ctx* ctx, int add_op, int mult_op, const gb_bin_plan* p,
                            const gb_csr* a, T iso, const T* u, const uint32_t* mask, T* out,
                            unsigned long long* counters, uint32_t* hasmul, int accumulate) {
  // striped (regular) matrices: quarter-warp medium rows
  auto k = accumulate ? mv_pull_binned<T, ADD, MUL, VALS, true> : mv_pull_binned<T, ADD, MUL, VALS, false>;
  k<<<resident_grid(ctx, k, 256), 256, 0, stream_of(ctx)>>>(
      p->n_long_tiles, p->tile_row, p->tile_beg, p->tile_end, p->n_mid, p->mid_rows, p->n_short,
      p->short_rows, a->offsets, a->indices, (const T*)a->values, iso, u, mask, add_op, mult_op,
      out, counters, hasmul, accumulate);
}

template <class T, int ADD, int MUL>
static void launch_binned_v(gb_ctx* ctx, int add_op, int mult_op, const gb_bin_plan* p,
                            const gb_csr* a, T iso, const T* u, const uint32_t* mask, T* out,
                            unsigned long long* counters, uint32_t* hasmul, int accumulate) {
  if (a->values)
    launch_binned_k<T, ADD, MUL, true>(ctx, add_op, mult_op, p, a, iso, u, mask, out, counters,
                                       hasmul, accumulate);
  else
    launch_binned_k<T, ADD, MUL, false>(ctx, add_op, mult_op, p, a, iso, u, mask, out, counters,
                                        hasmul, accumulate);
}

// nstripes == 1: the whole matrix; > 1: column stripes of it (each a CSR
// over the same rows), folded into `out` one after the other so every
// stripe's slice of u stays L2-resident while it is gathered
template <class T>
static gb_status pull_binned_t(gb_ctx* ctx, int add_op, int mult_op, int nstripes,
                               const gb_csr* as, const gb_bin_plan* ps, const T* u,
                               const uint32_t* mask, T* out, int64_t* counters) {
  cudaStream_t s = stream_of(ctx);
  const int64_t n = as[0].nrows;
  const int64_t W = (n + 31) / 32;
  Arena ar(ctx);
  uint32_t* hasmul = counters ? ar.alloc<uint32_t>(W) : nullptr;
  GB_ARENA_CHECK(ctx, ar);
  if (hasmul) GB_CUDA(ctx, cudaMemsetAsync(hasmul, 0, sizeof(uint32_t) * W, s));
  fill_identity<T>(ctx, n, op_identity<T>(add_op), out);
  int64_t nnz = 0;
  for (int k = 0; k < nstripes; ++k) nnz += as[k].nnz;
  const int prof = prof_begin(ctx, PROF_MV, nnz);
  unsigned long long* c = (unsigned long long*)counters;
  const int accumulate = nstripes > 1;
  for (int k = 0; k < nstripes; ++k) {
    const gb_csr* a = as + k;
    const gb_bin_plan* p = ps + k;
    const T iso = std::is_same<T, double>::value ? (T)a->iso_f64 : (T)a->iso_i64;
#define GB_SR(A_, M_)                                                                  \
    if (add_op == A_ && mult_op == M_) {                                               \
      launch_binned_v<T, A_, M_>(ctx, add_op, mult_op, p, a, iso, u, mask, out, c, hasmul, \
                                 accumulate);                                          \
    } else
    GB_SR(GB_OP_PLUS, GB_OP_TIMES)
    GB_SR(GB_OP_LOR, GB_OP_LAND)
    GB_SR(GB_OP_MIN, GB_OP_PLUS)
    GB_SR(GB_OP_MAX, GB_OP_PLUS)
    GB_SR(GB_OP_MIN, GB_OP_TIMES)
    GB_SR(GB_OP_MIN, GB_OP_SECOND)
    GB_SR(GB_OP_PLUS, GB_OP_LESS)
    GB_SR(GB_OP_MIN, GB_OP_NE)
    launch_binned_v<T, -1, -1>(ctx, add_op, mult_op, p, a, iso, u, mask, out, c, hasmul,
                               accumulate);
#undef GB_SR
  }
  prof_end(ctx, prof);
  if (counters) mv_pull_finish_counts(ctx, W, hasmul, c);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1 + nstripes + (counters ? 1 : 0));
  return GB_OK;
}

}  // namespace gb

using namespace gb;

extern "C" {

gb_status gb_bin_plan_counts(gb_ctx* ctx, const gb_csr* a, int64_t* counts_host) {
  counts_host[0] = counts_host[1] = counts_host[2] = 0;
  if (a->nrows == 0) return GB_OK;
  Arena ar(ctx);
  uint64_t* sm;
  int64_t* lt;
  return bin_scan(ctx, ar, a, &sm, &lt, counts_host);
}

gb_status gb_bin_plan_fill(gb_ctx* ctx, const gb_csr* a, gb_bin_plan* plan) {
  if (a->nrows == 0) return GB_OK;
  Arena ar(ctx);
  uint64_t* sm;
  int64_t* lt;
  int64_t c[3];
  GB_TRY(bin_scan(ctx, ar, a, &sm, &lt, c));
  if (c[0] != plan->n_short || c[1] != plan->n_mid || c[2] != plan->n_long_tiles)
    return set_error(ctx, GB_ERR_VALUE, "gb_bin_plan_fill: plan sizes differ from the matrix");
  bin_fill<<<grid_for(ctx, a->nrows, 256), 256, 0, stream_of(ctx)>>>(
      a->nrows, a->offsets, sm, lt, const_cast<int32_t*>(plan->short_rows),
      const_cast<int32_t*>(plan->mid_rows), const_cast<int32_t*>(plan->tile_row),
      const_cast<int64_t*>(plan->tile_beg), const_cast<int64_t*>(plan->tile_end));
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  GB_CUDA(ctx, cudaStreamSynchronize(stream_of(ctx)));
  return GB_OK;
}

gb_status gb_mxv_pull_binned(gb_ctx* ctx, int32_t add_op, int32_t mult_op, const gb_csr* a,
                             const gb_bin_plan* plan, const void* u, const uint32_t* mask,
                             void* out, int64_t* counters) {
  if (a->nrows == 0) return GB_OK;
  if (!plan || !fold_commutes(add_op))
    return set_error(ctx, GB_ERR_VALUE, "gb_mxv_pull_binned: needs a plan and a commutative fold");
  if (a->dtype == GB_I64)
    return pull_binned_t<int64_t>(ctx, add_op, mult_op, 1, a, plan, (const int64_t*)u, mask,
                                  (int64_t*)out, counters);
  return pull_binned_t<double>(ctx, add_op, mult_op, 1, a, plan, (const double*)u, mask,
                               (double*)out, counters);
}

gb_status gb_mxv_pull_striped(gb_ctx* ctx, int32_t add_op, int32_t mult_op, int32_t nstripes,
                              const gb_csr* stripes, const gb_bin_plan* plans, const void* u,
                              const uint32_t* mask, void* out, int64_t* counters) {
  if (nstripes < 1 || !stripes || !plans)
    return set_error(ctx, GB_ERR_ARG, "gb_mxv_pull_striped: needs >= 1 stripe and its plan");
  if (stripes[0].nrows == 0) return GB_OK;
  if (!fold_commutes(add_op))
    return set_error(ctx, GB_ERR_VALUE, "gb_mxv_pull_striped: needs a commutative fold");
  for (int k = 1; k < nstripes; ++k)
    if (stripes[k].nrows != stripes[0].nrows || stripes[k].dtype != stripes[0].dtype)
      return set_error(ctx, GB_ERR_SHAPE, "gb_mxv_pull_striped: stripes differ in rows or dtype");
  if (stripes[0].dtype == GB_I64)
    return pull_binned_t<int64_t>(ctx, add_op, mult_op, nstripes, stripes, plans,
                                  (const int64_t*)u, mask, (int64_t*)out, counters);
  return pull_binned_t<double>(ctx, add_op, mult_op, nstripes, stripes, plans, (const double*)u,
                               mask, (double*)out, counters);
}

}  // extern "C"
