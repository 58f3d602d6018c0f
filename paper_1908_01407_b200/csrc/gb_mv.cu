// Generic masked matrix-vector multiply over any device-encodable semiring.
//
//   gb_mxv_pull   _spmv_pull / _pull_span   kernels.py:153-229
//   gb_mxv_push   _spmspv_push             kernels.py:242-280
//
// These are the unfused operator-layer kernels behind mxv / vxm / spmv_pull /
// spmspv_push.  They reproduce the reference exactly, including its work
// counters; the algorithms use their own fused drivers instead.
#include <stdlib.h>

#include <type_traits>

#include <cub/cub.cuh>

#include "gb_common.cuh"
#include "gb_lbs.cuh"
#include "gb_rowtiles.cuh"

namespace gb {

__host__ __device__ __forceinline__ bool fold_is_commutative(int op) { return fold_commutes(op); }

template <class T>
__device__ __forceinline__ T aval(const T* vals, T iso, int64_t p) {
  return vals ? vals[p] : iso;
}

// Warp per row.  counters: [entries read, multiplies, adds]
template <class T>
__global__ void __launch_bounds__(256)
mv_pull_rows(int64_t nrows, const int64_t* __restrict__ off, const int32_t* __restrict__ idx,
             const T* __restrict__ vals, T iso, const T* __restrict__ u,
             const uint32_t* __restrict__ mask, int add_op, int mult_op, int early,
             T* __restrict__ out, unsigned long long* __restrict__ counters) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T ident = op_identity<T>(add_op);
  const bool comm = fold_is_commutative(add_op);
  for (int64_t i = w0; i < nrows; i += nw) {
    if (mask && !((mask[i >> 5] >> (i & 31)) & 1u)) {
      if (lane == 0) out[i] = ident;
      continue;
    }
    const int64_t lo = off[i], hi = off[i + 1];
    T acc = ident;
    long long incl = 0;
    int64_t first_hit = hi;  // position of the first hit (early-exit read count)
    if (comm) {
      for (int64_t base = lo; base < hi; base += 32) {
        const int64_t p = base + lane;
        bool hit = false;
        if (p < hi) {
          const T uj = u[idx[p]];
          if (uj != ident) {
            const T prod = op_pair<T>(mult_op, aval(vals, iso, p), uj);
            acc = op_fold<T>(add_op, acc, prod);
            ++incl;
            hit = prod != ident;
          }
        }
        if (early) {
          const uint32_t hits = __ballot_sync(GB_FULL, hit);
          if (hits && first_hit == hi) first_hit = base + __ffs(hits) - 1;
          if (hits && !counters) break;  // results never depend on the rest
        }
      }
      acc = warp_fold<T>(add_op, acc);
    } else if (lane == 0) {
      // order-dependent fold (e.g. a user monoid on SelectSecond): sequential
      bool any = false;
      for (int64_t p = lo; p < hi; ++p) {
        const T uj = u[idx[p]];
        if (uj == ident) continue;
        const T prod = op_pair<T>(mult_op, aval(vals, iso, p), uj);
        acc = any ? op_fold<T>(add_op, acc, prod) : op_fold1<T>(add_op, prod);
        any = true;
        ++incl;
        if (early && prod != ident && first_hit == hi) first_hit = p;
      }
    }
    if (lane == 0) out[i] = acc;
    if (counters) {
      incl = warp_sum_ll(incl);
      if (lane == 0) {
        const long long reads = early ? (first_hit < hi ? first_hit - lo + 1 : hi - lo) : hi - lo;
        atomicAdd(counters + 0, (unsigned long long)reads);
        atomicAdd(counters + 1, (unsigned long long)incl);
        if (incl > 0) atomicAdd(counters + 2, (unsigned long long)(incl - 1));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Edge-balanced masked pull (commutative folds, no early exit): warp tiles of
// 512 consecutive entries over the non-empty rows (gb_rowtiles.cuh layout).
// Per tile the row starts and row-allowed flags are staged in shared memory;
// each lane owns 16 consecutive entries:
//   1. it walks its entries' rows and flags the allowed ones,
//   2. loads the column indices of the 4-entry groups that hold an allowed
//      entry (16-byte loads; masked-out rows cost no index traffic) and
//      issues all u gathers at once,
//   3. folds row segment by row segment.  A row wholly inside the lane is
//      stored directly; a row that crosses lanes is combined by a warp
//      segmented scan over the lanes' open segments and written once, by the
//      lane where it ends -- a plain store when the row lies inside the tile,
//      one atomic fold when it crosses a tile boundary.  Hub rows therefore
//      cost one atomic per 512 entries instead of one per lane.
// Rows with no contribution keep the identity `out` was filled with.
// Counters are exact: reads and multiplies are block-reduced; rows with >= 1
// multiply are counted where they are written (tile-crossing rows through
// the `hasmul` bitmap, deduplicated by mv_pull_finish): adds = multiplies -
// such rows (kernels.py:185-189).
// ADD / MUL >= 0 fix the semiring at compile time (the builtin semirings,
// algebra.py:161-179); -1 reads add_op / mult_op at run time.  VALS = false
// for iso (structure-only) matrices.
// ---------------------------------------------------------------------------
#ifndef GB_MV_MINB
#define GB_MV_MINB 4  // resident 256-thread CTAs per SM (4: 64 registers; measured best with 4 waves)
#endif
#ifndef GB_MV_SPLIT
#define GB_MV_SPLIT 4  // u gathers in waves of 16/SPLIT per lane (s24: 1 wave 1.80 ms, 2: 1.51, 4: 1.39, 8: 1.44)
#endif
// COMPACT: the rows are only the ALLOWED non-empty rows (mv_mask_plan):
// nz_off holds their offsets in the concatenation of just their entries and
// row_pos their first position in the matrix, so masked-out rows cost
// nothing.  Positions are contiguous only inside a row: a lane adds the
// tile row's (row_pos - nz_off) to its slot position.
// HOT (ordered layout, gb_mxv_pull_ordered): u is the degree-ordered copy of
// the input vector, whose first hot_n entries -- the highest-degree columns,
// ~31 % of all gathers at R-MAT s24 -- are staged once per CTA in dynamic
// shared memory; gathers of those columns never reach L2.  One 1024-thread
// CTA per SM (WPB = 32) shares the largest possible copy.
template <class T, int ADD, int MUL, bool VALS, bool COMPACT, int WPB, bool HOT>
__global__ void __launch_bounds__(WPB * 32, WPB == 8 ? GB_MV_MINB : 1)
mv_pull_tiles(DevI64 R_d, const int32_t* __restrict__ nz_rows, const int64_t* __restrict__ nz_off,
              const int64_t* __restrict__ row_pos,
              const int32_t* __restrict__ tile_first, const int32_t* __restrict__ idx,
              const T* __restrict__ vals, T iso, const T* __restrict__ u,
              const uint32_t* __restrict__ mask, int add_rt, int mult_rt, T* __restrict__ out,
              unsigned long long* __restrict__ counters, uint32_t* __restrict__ hasmul,
              int32_t hot_n) {
  const int add_op = ADD >= 0 ? ADD : add_rt;
  const int mult_op = MUL >= 0 ? MUL : mult_rt;
  __shared__ uint16_t s_st[WPB][kRowTile + 8];
  __shared__ uint32_t s_ok[WPB][COMPACT ? 1 : kRowTile / 32 + 1];  // mask bit of each tile row
  __shared__ int64_t s_sb[COMPACT ? WPB : 1][COMPACT ? kRowTile + 8 : 1];  // row_pos - nz_off
  __shared__ unsigned long long s_cnt[3];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  T* s_hot = reinterpret_cast<T*>(s_dyn);
  if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
  if (HOT) {
    // the hot prefix of u (L2-resident: written by the permutation just before)
    for (int i = 2 * threadIdx.x; i < hot_n; i += 2 * blockDim.x) {
      if (i + 1 < hot_n) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(u + i));
        *reinterpret_cast<double2*>(s_hot + i) = v;
      } else {
        s_hot[i] = __ldg(u + i);
      }
    }
  }
  __syncthreads();
  auto gather = [&](int32_t c) -> T {
    if (HOT) return c < hot_n ? s_hot[c] : ld_gather(u + c);
    return ld_gather(u + c);
  };
  const int lane = threadIdx.x & 31;
  uint16_t* st = s_st[threadIdx.x >> 5];
  uint32_t* okw = s_ok[threadIdx.x >> 5];
  int64_t* sb = s_sb[COMPACT ? threadIdx.x >> 5 : 0];
  const T ident = op_identity<T>(add_op);
  const int64_t R_rows = R_d.get();
  const int64_t E = nz_off[R_rows];
  const int64_t ntiles = (E + kRowTile - 1) / kRowTile;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long c_reads = 0, c_muls = 0, c_rows = 0;
  for (int64_t t = w0; t < ntiles; t += nw) {
    const int64_t e0 = t * kRowTile;
    const int32_t rel_end = (int32_t)((e0 + kRowTile < E ? e0 + kRowTile : E) - e0);
    const int64_t r0 = tile_first[t];
    const int64_t r1 = t + 1 < ntiles ? tile_first[t + 1] : R_rows - 1;
    const int nr = (int)(r1 - r0 + 1);
    // row starts relative to the tile, clamped to [0, kRowTile]; st[nr] ends the last row
    for (int i0 = 0; i0 <= nr; i0 += 32) {
      const int i = i0 + lane;
      bool ok = false;
      if (i <= nr) {
        const int64_t no = nz_off[r0 + i];
        const int64_t o = no - e0;
        st[i] = (uint16_t)(o < 0 ? 0 : (o > kRowTile ? kRowTile : o));
        if (i < nr) {
          if (COMPACT) {
            sb[i] = row_pos[r0 + i] - no;
          } else {
            const int32_t row = nz_rows[r0 + i];
            ok = !mask || ((__ldg(mask + (row >> 5)) >> (row & 31)) & 1u);
          }
        }
      }
      if (!COMPACT) {
        const uint32_t b = __ballot_sync(GB_FULL, ok);
        if (lane == 0) okw[i0 >> 5] = b;
      }
    }
    // does the tile's first row start before it / its last row end after it?
    const bool head_out = nz_off[r0] < e0;
    const bool tail_out = nz_off[r1 + 1] > e0 + rel_end;
    __syncwarp();
    const int rel0 = lane * kRowItems;
    const int rel1 = rel0 + kRowItems < rel_end ? rel0 + kRowItems : rel_end;
    int lo = 0;
    if (rel0 < rel1) {
      int hi = nr - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (st[mid] <= rel0) lo = mid; else hi = mid - 1;
      }
    }
    // pass 1 (per row segment, not per entry): which of my entries belong to
    // allowed rows
    uint32_t allowed = 0;
    if (COMPACT) {
      if (rel0 < rel1) allowed = rel1 - rel0 == 32 ? ~0u : (1u << (rel1 - rel0)) - 1u;
    } else if (rel0 < rel1) {
      int a = rel0, c = lo;
      do {
        const int b = st[c + 1] < rel1 ? st[c + 1] : rel1;
        if ((okw[c >> 5] >> (c & 31)) & 1u) allowed |= ((1u << (b - a)) - 1u) << (a - rel0);
        a = b;
        ++c;
      } while (a < rel1);
    }
    // pass 2: column indices of the 8-entry groups holding an allowed entry, then
    // every gather at once
    int32_t cols[kRowItems];
    const int64_t my0 = e0 + rel0;
    if (COMPACT) {
      // positions are contiguous inside a row only: add the row's shift
      int c = lo, next = rel0 < rel1 ? st[lo + 1] : 0;
      int64_t sh = rel0 < rel1 ? sb[lo] : 0;
#pragma unroll
      for (int q = 0; q < kRowItems; ++q) {
        const int e = rel0 + q;
        cols[q] = 0;
        if (e < rel1) {
          if (e >= next) {
            ++c;
            next = st[c + 1];
            sh = sb[c];
          }
          cols[q] = __ldg(idx + my0 + q + sh);  // L1-allocating: a lane's 16 loads share lines
        }
      }
    } else if (rel1 - rel0 == kRowItems) {
#pragma unroll
      for (int g = 0; g < kRowItems / 8; ++g) {
        int32_t v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if ((allowed >> (8 * g)) & 0xFFu) ld_stream8(idx + my0 + 8 * g, v);  // 256-bit loads
#pragma unroll
        for (int j = 0; j < 8; ++j) cols[8 * g + j] = v[j];
      }
    } else {
#pragma unroll
      for (int q = 0; q < kRowItems; ++q) cols[q] = (allowed >> q) & 1u ? ld_stream(idx + my0 + q) : 0;
    }
    // the u gathers: all 16 at once, or (GB_MV_SPLIT=2) 8 now and 8 halfway
    // through the fold -- fewer registers, more resident warps
    constexpr int kGat = kRowItems / GB_MV_SPLIT;
    T uv[kGat];
#pragma unroll
    for (int q = 0; q < kGat; ++q) uv[q] = (allowed >> q) & 1u ? gather(cols[q]) : ident;
    c_reads += __popc(allowed);
    // pass 3: fold segment by segment.  Rows are non-empty, so one step
    // always reaches the next segment.  A segment that ends inside the lane
    // is either the lane's head (it continues a row from the previous lane:
    // kept for the scan) or a whole row (stored: rows that end inside a lane
    // and start inside it lie inside the tile).
    T acc = ident;          // current segment
    int cnt = 0;            // its multiplies
    T h_acc = ident;        // head segment continuing a row from the previous lane
    int h_cnt = 0;
    int h_row = -1;         // its tile row index (-1: none, -2: a "through" lane)
    int cur = lo;
    if (rel0 < rel1) {
      int next = st[cur + 1];
      int64_t sh = COMPACT ? sb[cur] : 0;  // position shift of the current row (COMPACT)
      // the lane's first segment continues a row from an earlier lane / tile
      const bool cont = st[cur] < rel0 || (cur == 0 && head_out);
      bool first = true;
#pragma unroll
      for (int q = 0; q < kRowItems; ++q) {
        if (kGat < kRowItems && q > 0 && q % kGat == 0) {
#pragma unroll
          for (int j = 0; j < kGat; ++j)
            uv[j] = (allowed >> (q + j)) & 1u ? gather(cols[q + j]) : ident;
        }
        const int e = rel0 + q;
        if (e < rel1 && e >= next) {
          if (first && cont) {
            h_acc = acc;
            h_cnt = cnt;
            h_row = cur;
          } else if (cnt > 0) {
            out[nz_rows[r0 + cur]] = acc;
            c_muls += cnt;
            ++c_rows;
          }
          first = false;
          acc = ident;
          cnt = 0;
          ++cur;
          next = st[cur + 1];
          if (COMPACT && VALS) sh = sb[cur];
        }
        if (((allowed >> q) & 1u) && uv[q % kGat] != ident) {
          const T a = VALS ? __ldg(vals + my0 + q + sh) : iso;
          acc = op_fold<T>(add_op, acc, op_pair<T>(mult_op, a, uv[q % kGat]));
          ++cnt;
        }
      }
      // the last segment: closed when it ends at the lane end (and its row
      // does not run past the tile)
      if (next <= rel1 && !(cur == nr - 1 && tail_out)) {
        if (first && cont) {
          h_acc = acc;
          h_cnt = cnt;
          h_row = cur;
        } else if (cnt > 0) {
          const int32_t row = nz_rows[r0 + cur];
          if (cur == 0 && head_out) {
            atomic_fold<T>(add_op, out + row, acc);
            atomicOr(hasmul + (row >> 5), 1u << (row & 31));
          } else {
            out[row] = acc;
            ++c_rows;
          }
          c_muls += cnt;
        }
        acc = ident;
        cnt = 0;
        cur = -1;  // nothing open
      } else if (first && cont) {
        h_row = -2;  // one segment spanning the whole lane: it travels in the scan
      }
    } else {
      cur = -1;
    }
    // warp segmented scan of the open tail segments (key = tile row index)
    int key = cur;
    T cv = acc;
    int cc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int k2 = __shfl_up_sync(GB_FULL, key, o);
      const T v2 = __shfl_up_sync(GB_FULL, cv, o);
      const int c2 = __shfl_up_sync(GB_FULL, cc, o);
      if (lane >= o && key >= 0 && k2 == key) {
        cv = op_fold<T>(add_op, cv, v2);
        cc += c2;
      }
    }
    // the previous lane's scanned open segment completes my head segment
    const int pk = __shfl_up_sync(GB_FULL, key, 1);
    const T pv = __shfl_up_sync(GB_FULL, cv, 1);
    const int pc = __shfl_up_sync(GB_FULL, cc, 1);
    if (h_row >= 0) {
      T v = h_acc;
      int c = h_cnt;
      if (lane > 0 && pk == h_row) {
        v = op_fold<T>(add_op, v, pv);
        c += pc;
      }
      if (c > 0) {
        const int32_t row = nz_rows[r0 + h_row];
        const bool in_tile = !(h_row == 0 && head_out) && !(h_row == nr - 1 && tail_out);
        c_muls += c;
        if (in_tile) {
          out[row] = v;
          ++c_rows;
        } else {
          atomic_fold<T>(add_op, out + row, v);
          atomicOr(hasmul + (row >> 5), 1u << (row & 31));
        }
      }
    }
    // an open segment that no later lane closes (the row runs past the tile)
    const int nk = __shfl_down_sync(GB_FULL, key, 1);
    const int nh = __shfl_down_sync(GB_FULL, h_row, 1);
    if (key >= 0) {
      const bool continued = lane < 31 && (nk == key || nh == key);
      if (!continued && cc > 0) {
        const int32_t row = nz_rows[r0 + key];
        c_muls += cc;
        atomic_fold<T>(add_op, out + row, cv);
        atomicOr(hasmul + (row >> 5), 1u << (row & 31));
      }
    }
    __syncwarp();
  }
  if (counters) {
    c_reads = warp_sum_ll((long long)c_reads);
    c_muls = warp_sum_ll((long long)c_muls);
    c_rows = warp_sum_ll((long long)c_rows);
    if (lane == 0) {
      atomicAdd(&s_cnt[0], c_reads);
      atomicAdd(&s_cnt[1], c_muls);
      atomicAdd(&s_cnt[2], c_rows);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd(counters + 0, s_cnt[0]);
      atomicAdd(counters + 1, s_cnt[1]);
      // rows with a multiply so far (whole rows); tile-crossing rows are
      // added from `hasmul` by mv_pull_finish; adds = multiplies - rows
      atomicAdd(counters + 2, s_cnt[1] - s_cnt[2]);
    }
  }
}

template <class T>
__global__ void fill_value(int64_t n, T v, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v;
}

// counters[2] -= rows that were split across lanes and had a multiply
__global__ void mv_pull_finish(int64_t W, const uint32_t* __restrict__ hasmul,
                               unsigned long long* __restrict__ counters) {
  long long c = 0;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x)
    c += __popc(hasmul[w]);
  c = warp_sum_ll(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(counters + 2, (unsigned long long)(-c));
}

template <class T>
struct PushExpand {
  const int32_t* __restrict__ idx;
  const T* __restrict__ vals;
  T iso;
  const T* __restrict__ u_vals;
  int mult_op;
  int32_t* __restrict__ rows;
  T* __restrict__ prods;
  __device__ __forceinline__ void operator()(int64_t k, int64_t p, int64_t e) const {
    rows[e] = idx[p];
    prods[e] = op_pair<T>(mult_op, aval(vals, iso, p), u_vals[k]);
  }
};

__global__ void seg_flags(int64_t n, const int32_t* __restrict__ keys, int32_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// One thread per segment: fold in stable (expansion) order, keep non-identity,
// allowed results.  keep[s] = 1 when segment s survives.
template <class T>
__global__ void seg_fold(int64_t n, const int32_t* __restrict__ keys, const int32_t* __restrict__ flags,
                         const int64_t* __restrict__ segpos, const T* __restrict__ prods, int add_op,
                         const uint32_t* __restrict__ mask, int32_t* __restrict__ seg_row,
                         T* __restrict__ seg_val, int32_t* __restrict__ keep) {
  const T ident = op_identity<T>(add_op);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!flags[i]) continue;
    const int32_t r = keys[i];
    T acc = prods[i];
    int64_t j = i + 1;
    if (j < n && keys[j] == r) {
      for (; j < n && keys[j] == r; ++j) acc = op_fold<T>(add_op, acc, prods[j]);
    } else {
      acc = op_fold1<T>(add_op, acc);
    }
    const int64_t s = segpos[i];
    seg_row[s] = r;
    seg_val[s] = acc;
    bool ok = acc != ident;
    if (ok && mask) ok = (mask[r >> 5] >> (r & 31)) & 1u;
    keep[s] = ok ? 1 : 0;
  }
}

template <class T>
__global__ void select_kept(int64_t nseg, const int32_t* __restrict__ keep,
                            const int64_t* __restrict__ pos, const int32_t* __restrict__ seg_row,
                            const T* __restrict__ seg_val, int32_t* __restrict__ out_idx,
                            T* __restrict__ out_vals) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg;
       s += (int64_t)gridDim.x * blockDim.x)
    if (keep[s]) {
      out_idx[pos[s]] = seg_row[s];
      out_vals[pos[s]] = seg_val[s];
    }
}

// ---- push with an order-independent fold: a dense accumulator ------------
// When the add monoid gives the same result in any order (integer plus /
// times wrap, min, max, logical or / and -- fold_commutes on the stored
// type), the products fold straight into a dense accumulator with atomics;
// no expansion buffer, sort or segment scan.  The rows that received a
// product are marked in a bitmap (read before the atomicOr) for the adds
// counter; the output keeps, in index order, the rows whose fold is not the
// identity and that the mask allows -- exactly the sorted path's result.
__device__ __forceinline__ void acc_fold(int add_op, int64_t* a, int64_t x) {
  switch (add_op) {
    case GB_OP_PLUS:
    case GB_OP_PLUS_WRAP:
      atomicAdd(reinterpret_cast<unsigned long long*>(a), (unsigned long long)x);
      return;
    case GB_OP_MIN:
      if (x < *reinterpret_cast<volatile long long*>(a)) atomicMin(reinterpret_cast<long long*>(a), x);
      return;
    case GB_OP_MAX:
      if (x > *reinterpret_cast<volatile long long*>(a)) atomicMax(reinterpret_cast<long long*>(a), x);
      return;
    case GB_OP_LOR:
      if (x != 0 && *reinterpret_cast<volatile long long*>(a) == 0)
        atomicExch(reinterpret_cast<unsigned long long*>(a), 1ull);
      return;
    case GB_OP_LAND:
      if (x == 0 && *reinterpret_cast<volatile long long*>(a) != 0)
        atomicExch(reinterpret_cast<unsigned long long*>(a), 0ull);
      return;
    default: {  // TIMES (wrapping)
      unsigned long long* u = reinterpret_cast<unsigned long long*>(a);
      unsigned long long old = *u, assumed;
      do {
        assumed = old;
        old = atomicCAS(u, assumed, (unsigned long long)wrap_mul((int64_t)assumed, x));
      } while (old != assumed);
    }
  }
}

__device__ __forceinline__ void acc_fold(int add_op, double* a, double x) {
  unsigned long long* u = reinterpret_cast<unsigned long long*>(a);
  switch (add_op) {
    case GB_OP_LOR:
      if (x != 0.0) *reinterpret_cast<volatile double*>(a) = 1.0;  // idempotent store
      return;
    case GB_OP_LAND:
      if (x == 0.0) *reinterpret_cast<volatile double*>(a) = 0.0;
      return;
    default: {  // MIN / MAX: compare-and-swap on the value
      const bool mn = add_op == GB_OP_MIN;
      double cur = *reinterpret_cast<volatile double*>(a);
      while (mn ? x < cur : x > cur) {
        const unsigned long long old =
            atomicCAS(u, __double_as_longlong(cur), __double_as_longlong(x));
        if (old == (unsigned long long)__double_as_longlong(cur)) break;
        cur = __longlong_as_double(old);
      }
    }
  }
}

template <class T>
struct PushAccum {
  const int32_t* __restrict__ idx;
  const T* __restrict__ vals;
  T iso;
  const T* __restrict__ u_vals;
  int add_op, mult_op;
  T* acc;
  uint32_t* touched;
  __device__ __forceinline__ void operator()(int64_t k, int64_t p, int64_t) const {
    const int32_t r = __ldg(idx + p);
    acc_fold(add_op, acc + r, op_pair<T>(mult_op, aval(vals, iso, p), u_vals[k]));
    const uint32_t bit = 1u << (r & 31);
    if (!(ld_probe(touched + (r >> 5)) & bit)) atomicOr(touched + (r >> 5), bit);
  }
};

// kept bits per word (fold != identity, mask allows) and the word's count;
// the touched rows' count for the adds counter
template <class T>
__global__ void accum_keep(int64_t n, const T* __restrict__ acc, T ident,
                           const uint32_t* __restrict__ mask, const uint32_t* __restrict__ touched,
                           uint32_t* __restrict__ keep, int64_t* __restrict__ wcnt,
                           unsigned long long* __restrict__ ntouched) {
  const int64_t W = (n + 31) / 32;
  long long t = 0;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t tw = touched[w];
    uint32_t kb = 0;
    for (uint32_t b = tw; b; b &= b - 1) {
      const int j = __ffs(b) - 1;
      const int64_t r = w * 32 + j;
      if (acc[r] != ident && (!mask || ((mask[w] >> j) & 1u))) kb |= 1u << j;
    }
    keep[w] = kb;
    wcnt[w] = __popc(kb);
    t += __popc(tw);
  }
  t = warp_sum_ll(t);
  if ((threadIdx.x & 31) == 0 && t) atomicAdd(ntouched, (unsigned long long)t);
}

template <class T>
__global__ void accum_emit(int64_t n, const T* __restrict__ acc, const uint32_t* __restrict__ keep,
                           const int64_t* __restrict__ wpos, int32_t* __restrict__ out_idx,
                           T* __restrict__ out_vals) {
  const int64_t W = (n + 31) / 32;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x) {
    int64_t at = wpos[w];
    for (uint32_t b = keep[w]; b; b &= b - 1) {
      const int64_t r = w * 32 + (__ffs(b) - 1);
      out_idx[at] = (int32_t)r;
      out_vals[at] = acc[r];
      ++at;
    }
  }
}

template <class T>
static bool accum_fold_ok(int add_op) {
  if (std::is_same<T, int64_t>::value) return fold_commutes(add_op);
  return add_op == GB_OP_MIN || add_op == GB_OP_MAX || add_op == GB_OP_LOR || add_op == GB_OP_LAND;
}

template <class T>
static gb_status push_accum_t(gb_ctx* ctx, int add_op, int mult_op, const gb_csr* a,
                              int64_t out_size, int64_t k, const int32_t* u_idx, const T* u_vals,
                              const uint32_t* mask, int32_t* out_idx, T* out_vals, int64_t* count,
                              int64_t* counters, const LbsPlan& plan, Arena& ar, int64_t E) {
  cudaStream_t s = stream_of(ctx);
  const int64_t n = out_size, W = (n + 31) / 32;
  T* acc = ar.alloc<T>(n);
  uint32_t* touched = ar.alloc<uint32_t>(W);
  uint32_t* keep = ar.alloc<uint32_t>(W);
  int64_t* wcnt = ar.alloc<int64_t>(W + 1);
  int64_t* wpos = ar.alloc<int64_t>(W + 1);
  unsigned long long* nt = ar.alloc<unsigned long long>(1);
  GB_ARENA_CHECK(ctx, ar);
  const T ident = op_identity<T>(add_op);
  fill_value<T><<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(n, ident, acc);
  GB_CUDA(ctx, cudaMemsetAsync(touched, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(nt, 0, 8, s));
  GB_CUDA(ctx, cudaMemsetAsync(wcnt + W, 0, 8, s));
  const T iso = std::is_same<T, double>::value ? (T)a->iso_f64 : (T)a->iso_i64;
  PushAccum<T> f{a->indices, (const T*)a->values, iso, u_vals, add_op, mult_op, acc, touched};
  lbs_expand<PushAccum<T>><<<plan.grid, kLbsThreads, 0, s>>>(k, plan.S, plan.rowstart,
                                                             plan.tile_first, f);
  accum_keep<T><<<grid_for(ctx, W, 256, 8), 256, 0, s>>>(n, acc, ident, mask, touched, keep, wcnt,
                                                          nt);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, wcnt, wpos, W + 1, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp, tb, wcnt, wpos, W + 1, s));
  accum_emit<T><<<grid_for(ctx, W, 256, 8), 256, 0, s>>>(n, acc, keep, wpos, out_idx, out_vals);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 9);
  if (counters) {
    int64_t ntouched = 0;
    GB_TRY(read_i64(ctx, (const int64_t*)nt, &ntouched));
    int64_t c[3];
    GB_TRY(read_i64(ctx, counters, c, 3));
    c[2] += E - ntouched;
    GB_CUDA(ctx, cudaMemcpyAsync(counters, c, 24, cudaMemcpyHostToDevice, s));
  }
  return read_i64(ctx, wpos + W, count);
}

static int bits_for(int64_t n) {
  int b = 1;
  while (((int64_t)1 << b) < n) ++b;
  return b;
}

template <class T>
static gb_status push_t(gb_ctx* ctx, int add_op, int mult_op, const gb_csr* a, int64_t out_size,
                        int64_t k, const int32_t* u_idx, const T* u_vals, const uint32_t* mask,
                        int32_t* out_idx, T* out_vals, int64_t* count, int64_t* counters) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  *count = 0;
  if (k == 0) return GB_OK;
  LbsPlan plan;
  GB_TRY(lbs_prepare(ctx, ar, k, u_idx, a->offsets, a->nnz, &plan));
  int64_t E = 0;
  GB_TRY(read_i64(ctx, plan.S + k, &E));
  if (counters) {
    int64_t c[3];
    GB_TRY(read_i64(ctx, counters, c, 3));
    c[1] += E;
    GB_CUDA(ctx, cudaMemcpyAsync(counters, c, 24, cudaMemcpyHostToDevice, s));
  }
  if (E == 0) return GB_OK;
  if (accum_fold_ok<T>(add_op) && !getenv("GB_PUSH_SORTED"))
    return push_accum_t<T>(ctx, add_op, mult_op, a, out_size, k, u_idx, u_vals, mask, out_idx,
                           out_vals, count, counters, plan, ar, E);
  int32_t* ka = ar.alloc<int32_t>(E);
  int32_t* kb = ar.alloc<int32_t>(E);
  T* va = ar.alloc<T>(E);
  T* vb = ar.alloc<T>(E);
  int32_t* flags = ar.alloc<int32_t>(E + 1);
  int64_t* segpos = ar.alloc<int64_t>(E + 1);
  GB_ARENA_CHECK(ctx, ar);
  T iso = std::is_same<T, double>::value ? (T)a->iso_f64 : (T)a->iso_i64;
  PushExpand<T> f{a->indices, (const T*)a->values, iso, u_vals, mult_op, ka, va};
  lbs_expand<PushExpand<T>><<<plan.grid, kLbsThreads, 0, s>>>(k, plan.S, plan.rowstart,
                                                              plan.tile_first, f);
  cub::DoubleBuffer<int32_t> dk(ka, kb);
  cub::DoubleBuffer<T> dv(va, vb);
  size_t tb = 0;
  const int bits = bits_for(out_size > 1 ? out_size : 2);
  cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, E, 0, bits, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, E, 0, bits, s));
  const int32_t* keys = dk.Current();
  const T* prods = dv.Current();
  seg_flags<<<grid_for(ctx, E, 256), 256, 0, s>>>(E, keys, flags);
  GB_CUDA(ctx, cudaMemsetAsync(flags + E, 0, sizeof(int32_t), s));
  size_t tb2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, flags, segpos, E + 1, s);
  void* tmp2 = ar.raw(tb2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp2, tb2, flags, segpos, E + 1, s));
  int64_t nseg = 0;
  GB_TRY(read_i64(ctx, segpos + E, &nseg));
  // flags[E] = 0, so segpos[E] counts every segment
  if (counters) {
    int64_t c[3];
    GB_TRY(read_i64(ctx, counters, c, 3));
    c[2] += E - nseg;
    GB_CUDA(ctx, cudaMemcpyAsync(counters, c, 24, cudaMemcpyHostToDevice, s));
  }
  int32_t* seg_row = ar.alloc<int32_t>(nseg);
  T* seg_val = ar.alloc<T>(nseg);
  int32_t* keep = ar.alloc<int32_t>(nseg + 1);
  int64_t* kpos = ar.alloc<int64_t>(nseg + 1);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(keep + nseg, 0, sizeof(int32_t), s));
  seg_fold<T><<<grid_for(ctx, E, 256), 256, 0, s>>>(E, keys, flags, segpos, prods, add_op, mask,
                                                    seg_row, seg_val, keep);
  size_t tb3 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb3, keep, kpos, nseg + 1, s);
  void* tmp3 = ar.raw(tb3);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp3, tb3, keep, kpos, nseg + 1, s));
  select_kept<T><<<grid_for(ctx, nseg, 256), 256, 0, s>>>(nseg, keep, kpos, seg_row, seg_val,
                                                          out_idx, out_vals);
  GB_LAUNCH_CHECK(ctx);
  GB_TRY(read_i64(ctx, kpos + nseg, count));
  count_launch(ctx, 12);
  return GB_OK;
}

// Rows to reduce: the plan of all non-empty rows (mask tested per row), or,
// with `compact`, only the allowed ones (R read on the device).
struct MvRows {
  DevI64 R;
  const int32_t* rows;
  const int64_t* off;
  const int64_t* pos;  // compact: first matrix position of each row
  const int32_t* tile_first;
  bool compact;
};

// hot == 0: the original-layout kernel (4 x 256-thread CTAs per SM); hot > 0:
// the ordered-layout kernel with `hot` entries of u in shared memory
template <class T, int ADD, int MUL, bool VALS>
static gb_status launch_tiles_k(gb_ctx* ctx, int add_op, int mult_op, const MvRows& plan,
                                const gb_csr* a, T iso, const T* u, const uint32_t* mask, T* out,
                                unsigned long long* counters, uint32_t* hasmul, int32_t hot) {
  if (hot > 0) {
    auto k = mv_pull_tiles<T, ADD, MUL, VALS, false, 32, true>;
    const size_t smem = (size_t)hot * sizeof(T);
    GB_CUDA(ctx, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<resident_grid(ctx, k, 1024, smem), 1024, smem, stream_of(ctx)>>>(
        plan.R, plan.rows, plan.off, plan.pos, plan.tile_first, a->indices, (const T*)a->values,
        iso, u, mask, add_op, mult_op, out, counters, hasmul, hot);
    return GB_OK;
  }
  auto k = plan.compact ? mv_pull_tiles<T, ADD, MUL, VALS, true, 8, false>
                        : mv_pull_tiles<T, ADD, MUL, VALS, false, 8, false>;
  k<<<resident_grid(ctx, k, 256), 256, 0, stream_of(ctx)>>>(
      plan.R, plan.rows, plan.off, plan.pos, plan.tile_first, a->indices, (const T*)a->values, iso,
      u, mask, add_op, mult_op, out, counters, hasmul, 0);
  return GB_OK;
}

template <class T, int ADD, int MUL>
static gb_status launch_tiles_v(gb_ctx* ctx, int add_op, int mult_op, bool vals,
                                const MvRows& plan, const gb_csr* a, T iso, const T* u,
                                const uint32_t* mask, T* out, unsigned long long* counters,
                                uint32_t* hasmul, int32_t hot) {
  return vals ? launch_tiles_k<T, ADD, MUL, true>(ctx, add_op, mult_op, plan, a, iso, u, mask, out,
                                                  counters, hasmul, hot)
              : launch_tiles_k<T, ADD, MUL, false>(ctx, add_op, mult_op, plan, a, iso, u, mask, out,
                                                   counters, hasmul, hot);
}

// the builtin semirings get their own instantiation; anything else is generic
template <class T>
static gb_status launch_pull_tiles(gb_ctx* ctx, int add_op, int mult_op, bool vals,
                                   const MvRows& plan, const gb_csr* a, T iso, const T* u,
                                   const uint32_t* mask, T* out, unsigned long long* counters,
                                   uint32_t* hasmul, int32_t hot = 0) {
#define GB_SR(A_, M_)                                                                         \
  if (add_op == A_ && mult_op == M_)                                                          \
    return launch_tiles_v<T, A_, M_>(ctx, add_op, mult_op, vals, plan, a, iso, u, mask, out, \
                                     counters, hasmul, hot);
  GB_SR(GB_OP_PLUS, GB_OP_TIMES)    // PlusMultiplies
  GB_SR(GB_OP_LOR, GB_OP_LAND)      // LogicalOrAnd
  GB_SR(GB_OP_MIN, GB_OP_PLUS)      // MinPlus
  GB_SR(GB_OP_MAX, GB_OP_PLUS)      // MaxPlus
  GB_SR(GB_OP_MIN, GB_OP_TIMES)     // MinMultiplies
  GB_SR(GB_OP_MIN, GB_OP_SECOND)    // MinimumSelectSecond
  GB_SR(GB_OP_PLUS, GB_OP_LESS)     // PlusLess
  GB_SR(GB_OP_MIN, GB_OP_NE)        // MinimumNotEqualTo
#undef GB_SR
  return launch_tiles_v<T, -1, -1>(ctx, add_op, mult_op, vals, plan, a, iso, u, mask, out, counters,
                                   hasmul, hot);
}

// ---------------------------------------------------------------------------
// Compact plan of the allowed rows (per call: the mask changes).  One packed
// scan counts allowed rows (low 28 bits) and their entries (high 36 bits).
// ---------------------------------------------------------------------------
constexpr int kPackBits = 28;
constexpr uint64_t kPackMask = (1ull << kPackBits) - 1;

__global__ void mask_pack(int64_t R, const int32_t* __restrict__ nz_rows,
                          const int64_t* __restrict__ nz_off, const uint32_t* __restrict__ mask,
                          uint64_t* __restrict__ pk) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= R;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t v = 0;
    if (i < R) {
      const int32_t row = nz_rows[i];
      if ((__ldg(mask + (row >> 5)) >> (row & 31)) & 1u)
        v = ((uint64_t)(nz_off[i + 1] - nz_off[i]) << kPackBits) | 1u;
    }
    pk[i] = v;
  }
}

__global__ void mask_fill(int64_t R, const int32_t* __restrict__ nz_rows,
                          const int64_t* __restrict__ nz_off, const uint64_t* __restrict__ sc,
                          int32_t* __restrict__ a_rows, int64_t* __restrict__ a_off,
                          int64_t* __restrict__ a_pos, int64_t* __restrict__ A_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= R;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t c = sc[i];
    const int64_t p = (int64_t)(c & kPackMask);
    if (i == R) {
      *A_out = p;
      a_off[p] = (int64_t)(c >> kPackBits);
    } else if ((sc[i + 1] & kPackMask) != (uint64_t)p) {
      a_rows[p] = nz_rows[i];
      a_off[p] = (int64_t)(c >> kPackBits);
      a_pos[p] = nz_off[i];
    }
  }
}

// tile_first over the compact offsets, counts read on the device
__global__ void mask_tile_first(const int64_t* __restrict__ A_d, const int64_t* __restrict__ a_off,
                                int32_t* __restrict__ tf) {
  const int64_t A = *A_d;
  const int64_t E = a_off[A];
  const int64_t ntiles = (E + kRowTile - 1) / kRowTile;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t * kRowTile;
    int64_t lo = 0, hi = A - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (a_off[mid] <= e) lo = mid; else hi = mid - 1;
    }
    tf[t] = (int32_t)lo;
  }
}

static gb_status mv_mask_plan(gb_ctx* ctx, Arena& ar, const RowTilesPlan& plan, int64_t nnz,
                              const uint32_t* mask, MvRows* out) {
  cudaStream_t s = stream_of(ctx);
  const int64_t R = plan.R;
  uint64_t* pk = ar.alloc<uint64_t>(R + 1);
  uint64_t* sc = ar.alloc<uint64_t>(R + 1);
  int32_t* a_rows = ar.alloc<int32_t>(R > 0 ? R : 1);
  int64_t* a_off = ar.alloc<int64_t>(R + 1);
  int64_t* a_pos = ar.alloc<int64_t>(R > 0 ? R : 1);
  int32_t* tf = ar.alloc<int32_t>(nnz / kRowTile + 2);
  int64_t* A = ar.alloc<int64_t>(1);
  GB_ARENA_CHECK(ctx, ar);
  mask_pack<<<grid_for(ctx, R + 1, 256), 256, 0, s>>>(R, plan.nz_rows, plan.nz_off, mask, pk);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, pk, sc, R + 1, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp, tb, pk, sc, R + 1, s));
  mask_fill<<<grid_for(ctx, R + 1, 256), 256, 0, s>>>(R, plan.nz_rows, plan.nz_off, sc, a_rows, a_off,
                                                      a_pos, A);
  mask_tile_first<<<grid_for(ctx, nnz / kRowTile + 1, 256), 256, 0, s>>>(A, a_off, tf);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 5);
  *out = MvRows{dptr(A), a_rows, a_off, a_pos, tf, true};
  return GB_OK;
}

template <class T>
static gb_status pull_tiles_t(gb_ctx* ctx, int add_op, int mult_op, const gb_csr* a,
                              const gb_row_plan* given, const T* u, const uint32_t* mask, T* out,
                              int64_t* counters) {
  cudaStream_t s = stream_of(ctx);
  const int64_t n = a->nrows;
  const int64_t W = (n + 31) / 32;
  Arena ar(ctx);
  RowTilesPlan plan;
  if (given) {
    plan.R = given->nrows_nz;
    plan.nz_rows = const_cast<int32_t*>(given->nz_rows);
    plan.nz_off = const_cast<int64_t*>(given->nz_off);
    plan.tile_first = const_cast<int32_t*>(given->tile_first);
  } else {
    GB_TRY(row_tiles_plan(ctx, ar, n, a->offsets, a->nnz, &plan));
  }
  uint32_t* hasmul = counters ? ar.alloc<uint32_t>(W) : nullptr;
  GB_ARENA_CHECK(ctx, ar);
  const T ident = op_identity<T>(add_op);
  const T iso = std::is_same<T, double>::value ? (T)a->iso_f64 : (T)a->iso_i64;
  if (hasmul) GB_CUDA(ctx, cudaMemsetAsync(hasmul, 0, sizeof(uint32_t) * W, s));
  fill_value<T><<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(n, ident, out);
  const int ps = prof_begin(ctx, PROF_MV, a->nnz);
  if (plan.R > 0) {
    // a mask: reduce only the allowed rows (compact plan); otherwise every
    // non-empty row
    MvRows rows{dval(plan.R), plan.nz_rows, plan.nz_off, nullptr, plan.tile_first, false};
    // The compact plan skips masked-out rows entirely but loses the 16-byte
    // index loads; it measured slower at s24 with a 50 % mask (2.04 vs
    // 1.80 ms: the x gathers, not the masked rows, bound the kernel), so it
    // is opt-in (GB_MV_COMPACT=1) for sparse masks.
    static const bool compact = getenv("GB_MV_COMPACT") && atoi(getenv("GB_MV_COMPACT")) == 1;
    if (compact && mask && plan.R < (int64_t)kPackMask && (a->nnz >> (64 - kPackBits)) == 0)
      GB_TRY(mv_mask_plan(ctx, ar, plan, a->nnz, mask, &rows));
    GB_TRY(launch_pull_tiles<T>(ctx, add_op, mult_op, a->values != nullptr, rows, a, iso, u, mask,
                                out, (unsigned long long*)counters, hasmul));
  }
  prof_end(ctx, ps);
  if (counters)
    mv_pull_finish<<<grid_for(ctx, W, 256, 4), 256, 0, s>>>(W, hasmul,
                                                             (unsigned long long*)counters);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 2 + (counters ? 2 : 0));
  return GB_OK;
}

template <class T>
void fill_identity(gb_ctx* ctx, int64_t n, T v, T* out) {
  fill_value<T><<<grid_for(ctx, n, 256, 8), 256, 0, stream_of(ctx)>>>(n, v, out);
}
template void fill_identity<int64_t>(gb_ctx*, int64_t, int64_t, int64_t*);
template void fill_identity<double>(gb_ctx*, int64_t, double, double*);

void mv_pull_finish_counts(gb_ctx* ctx, int64_t W, const uint32_t* hasmul,
                           unsigned long long* counters) {
  mv_pull_finish<<<grid_for(ctx, W, 256, 4), 256, 0, stream_of(ctx)>>>(W, hasmul, counters);
}

// ---------------------------------------------------------------------------
// Masked pull on the degree-ordered layout (SparseMatrix.traversal()).  The
// matrix is P A P^T; the plan's rows are the ORIGINAL row ids of its
// non-empty rows, so the mask is probed and `out` written in the caller's
// labels, and only the column gathers use new ids -- on uo = u permuted into
// the new order (one pass over the `reach` columns that have entries).  In
// the new order the gathered part of u is a dense prefix (71 MB at R-MAT s24
// against 134 MB for u, so it stays in L2) and its highest-degree head sits
// in shared memory (HOT kernel above).
// ---------------------------------------------------------------------------
template <class T>
__global__ void perm_gather(int64_t m, const int32_t* __restrict__ order, const T* __restrict__ u,
                            T* __restrict__ uo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    uo[i] = __ldg(u + __ldg(order + i));
}

__global__ void remap_ids(int64_t m, const int32_t* __restrict__ ids, const int32_t* __restrict__ map,
                          int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = map[ids[i]];
}

__global__ void index_max(int64_t m, const int32_t* __restrict__ idx, int* __restrict__ out) {
  int v = -1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    v = max(v, ld_stream(idx + i));
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(GB_FULL, v, o));
  if ((threadIdx.x & 31) == 0 && v >= 0) atomicMax(out, v);
}

#ifndef GB_MV_HOT_MAX
#define GB_MV_HOT_MAX (1 << 30)  // cap on the shared-memory head (A/B knob)
#endif

template <class T>
static int32_t hot_entries(gb_ctx* ctx, int64_t reach) {
  static int cap = -1;
  if (cap < 0) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, mv_pull_tiles<T, GB_OP_PLUS, GB_OP_TIMES, false, false, 32, true>);
    cap = (int)((optin - (int)fa.sharedSizeBytes - 1024) / sizeof(T)) & ~1;
    if (cap < 0) cap = 0;
    const char* e = getenv("GB_MV_HOT");
    if (e) cap = cap < atoi(e) ? cap : atoi(e);
    if (cap > GB_MV_HOT_MAX) cap = GB_MV_HOT_MAX;
  }
  (void)ctx;
  return (int32_t)(reach < cap ? reach : cap);
}

template <class T>
static gb_status pull_ordered_t(gb_ctx* ctx, int add_op, int mult_op, const gb_csr* a,
                                const gb_row_plan* given, const int32_t* order, int64_t reach,
                                const T* u, const uint32_t* mask, T* out, int64_t* counters) {
  cudaStream_t s = stream_of(ctx);
  const int64_t n = a->nrows;
  const int64_t W = (n + 31) / 32;
  Arena ar(ctx);
  T* uo = ar.alloc<T>(reach > 0 ? reach : 1);
  uint32_t* hasmul = counters ? ar.alloc<uint32_t>(W) : nullptr;
  GB_ARENA_CHECK(ctx, ar);
  const T ident = op_identity<T>(add_op);
  const T iso = std::is_same<T, double>::value ? (T)a->iso_f64 : (T)a->iso_i64;
  if (hasmul) GB_CUDA(ctx, cudaMemsetAsync(hasmul, 0, sizeof(uint32_t) * W, s));
  fill_value<T><<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(n, ident, out);
  if (reach > 0)
    perm_gather<T><<<grid_for(ctx, reach, 256, 8), 256, 0, s>>>(reach, order, u, uo);
  const int ps = prof_begin(ctx, PROF_MV, a->nnz);
  if (given->nrows_nz > 0) {
    MvRows rows{dval(given->nrows_nz), given->nz_rows, given->nz_off, nullptr, given->tile_first,
                false};
    const int32_t hot = hot_entries<T>(ctx, reach);
    GB_TRY(launch_pull_tiles<T>(ctx, add_op, mult_op, a->values != nullptr, rows, a, iso, uo, mask,
                                out, (unsigned long long*)counters, hasmul, hot > 0 ? hot : 0));
  }
  prof_end(ctx, ps);
  if (counters)
    mv_pull_finish<<<grid_for(ctx, W, 256, 4), 256, 0, s>>>(W, hasmul,
                                                             (unsigned long long*)counters);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 3 + (counters ? 2 : 0));
  return GB_OK;
}

}  // namespace gb

using namespace gb;

extern "C" {

gb_status gb_mxv_pull(gb_ctx* ctx, int32_t add_op, int32_t mult_op, const gb_csr* a,
                      const gb_row_plan* plan, const void* u, const uint32_t* mask,
                      int32_t early_exit, int32_t partition, void* out, int64_t* counters) {
  (void)partition;  // both partition modes get the edge-balanced tiles (or warp per row)
  cudaStream_t s = stream_of(ctx);
  const int64_t n = a->nrows;
  if (n == 0) return GB_OK;
  const int early = early_exit && add_op == GB_OP_LOR;
  if (!early && fold_is_commutative(add_op)) {
    if (a->dtype == GB_I64)
      return pull_tiles_t<int64_t>(ctx, add_op, mult_op, a, plan, (const int64_t*)u, mask,
                                   (int64_t*)out, counters);
    return pull_tiles_t<double>(ctx, add_op, mult_op, a, plan, (const double*)u, mask,
                                (double*)out, counters);
  }
  const int grid = grid_for(ctx, n * 32, 256, 16);
  const int ps = prof_begin(ctx, PROF_MV, n);
  if (a->dtype == GB_I64)
    mv_pull_rows<int64_t><<<grid, 256, 0, s>>>(n, a->offsets, a->indices,
                                               (const int64_t*)a->values, a->iso_i64,
                                               (const int64_t*)u, mask, add_op, mult_op, early,
                                               (int64_t*)out, (unsigned long long*)counters);
  else
    mv_pull_rows<double><<<grid, 256, 0, s>>>(n, a->offsets, a->indices, (const double*)a->values,
                                              a->iso_f64, (const double*)u, mask, add_op, mult_op,
                                              early, (double*)out, (unsigned long long*)counters);
  prof_end(ctx, ps);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

gb_status gb_mxv_pull_ordered(gb_ctx* ctx, int32_t add_op, int32_t mult_op, const gb_csr* a,
                              const gb_row_plan* plan, const int32_t* order, int64_t reach,
                              const void* u, const uint32_t* mask, void* out, int64_t* counters) {
  if (a->nrows == 0) return GB_OK;
  if (!plan || !order || !fold_is_commutative(add_op))
    return set_error(ctx, GB_ERR_VALUE, "gb_mxv_pull_ordered: needs a plan, the order and a "
                     "commutative fold");
  if (a->dtype == GB_I64)
    return pull_ordered_t<int64_t>(ctx, add_op, mult_op, a, plan, order, reach, (const int64_t*)u,
                                   mask, (int64_t*)out, counters);
  return pull_ordered_t<double>(ctx, add_op, mult_op, a, plan, order, reach, (const double*)u,
                                mask, (double*)out, counters);
}

gb_status gb_row_plan_remap(gb_ctx* ctx, int64_t count, const int32_t* ids, const int32_t* map,
                            int32_t* out) {
  if (count > 0) {
    remap_ids<<<grid_for(ctx, count, 256, 8), 256, 0, stream_of(ctx)>>>(count, ids, map, out);
    GB_LAUNCH_CHECK(ctx);
    count_launch(ctx, 1);
  }
  return GB_OK;
}

gb_status gb_index_max(gb_ctx* ctx, int64_t count, const int32_t* idx, int64_t* max_host) {
  *max_host = -1;
  if (count == 0) return GB_OK;
  Arena ar(ctx);
  int* d = ar.alloc<int>(1);
  GB_ARENA_CHECK(ctx, ar);
  cudaStream_t s = stream_of(ctx);
  GB_CUDA(ctx, cudaMemsetAsync(d, 0xff, sizeof(int), s));
  index_max<<<grid_for(ctx, count, 256, 8), 256, 0, s>>>(count, idx, d);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  int h = -1;
  GB_CUDA(ctx, cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s));
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  *max_host = h;
  return GB_OK;
}

gb_status gb_mxv_push(gb_ctx* ctx, int32_t add_op, int32_t mult_op, const gb_csr* a,
                      int64_t out_size, int64_t k, const int32_t* u_idx, const void* u_vals,
                      const uint32_t* mask, int32_t* out_idx, void* out_vals, int64_t* count,
                      int64_t* counters) {
  if (a->dtype == GB_I64)
    return push_t<int64_t>(ctx, add_op, mult_op, a, out_size, k, u_idx, (const int64_t*)u_vals,
                           mask, out_idx, (int64_t*)out_vals, count, counters);
  return push_t<double>(ctx, add_op, mult_op, a, out_size, k, u_idx, (const double*)u_vals, mask,
                        out_idx, (double*)out_vals, count, counters);
}

}  // extern "C"
