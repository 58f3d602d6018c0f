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

// 32-bit form of lb32 for one row's list (the issue-bound inner search)
__device__ __forceinline__ int lb32i(const int32_t* a, int n, int32_t key) {
  if (n <= 0) return 0;
  const int32_t* b = a;
  int l = n;
  while (l > 1) {
    const int h = l >> 1;
    b = b[h - 1] < key ? b + h : b;
    l -= h;
  }
  return (int)(b - a) + (*b < key);
}

// Warp per task of kMxmTask consecutive mask entries (rows cut across
// tasks): a hub row's thousands of entries no longer serialise on one warp.
// out_flag[e] = 1 when mask entry e produces an output entry (matches > 0, or
// the identity is non-zero), out_val[e] its value.
constexpr int64_t kMxmTask = 32;
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
  const int64_t nnz_m = moff[nrows];
  const int64_t ntasks = (nnz_m + kMxmTask - 1) / kMxmTask;
  for (int64_t t = w0; t < ntasks; t += nw) {
    const int64_t e0 = t * kMxmTask, e1 = min(e0 + kMxmTask, nnz_m);
    // the row holding e0: last i with moff[i] <= e0
    int64_t i;
    {
      int64_t lo = 0, hi = nrows;
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (moff[mid] <= e0) lo = mid; else hi = mid;
      }
      i = lo;
    }
    long long mults = 0, adds = 0;
    int64_t rend = moff[i + 1];
    int64_t alo = aoff[i], la = aoff[i + 1] - alo;
    for (int64_t e = e0; e < e1; ++e) {
      while (e >= rend) {  // the task crossed into the next row(s)
        ++i;
        rend = moff[i + 1];
        alo = aoff[i];
        la = aoff[i + 1] - alo;
      }
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
      const int ll32 = (int)ll;  // a row's length fits 32 bits: the search stays 32-bit
      for (int64_t q = lane; q < ls; q += 32) {
        const int32_t key = sidx[q];
        const int p = lb32i(lidx, ll32, key);
        if (p < ll32 && lidx[p] == key) {
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

// Upper row of rank r (vertex v = order[r]): the ranks of v's higher-ranked
// neighbours, left in adjacency order -- tc_count tests membership, it does
// not merge.  Warp per row in rank order for rows up to kTcLong entries; the
// longer rows (the top of the degree order) are cut into kTcLong-entry tiles
// shared out over all warps, so a hub is not one warp's serial loop.
#ifndef GB_TC_LONG
#define GB_TC_LONG 2048
#endif
constexpr int kTcLong = GB_TC_LONG;

// Tile plan of the long rows: tstart[i] = first tile of rank first + i,
// meta = {first, tiles}; zeroes the long rows' lengths.
// One block; the degrees arrive sorted ascending.
__global__ void __launch_bounds__(1024)
tc_long_plan(int64_t n, const uint32_t* __restrict__ deg_sorted, int64_t* __restrict__ tstart,
             int64_t* __restrict__ meta, int64_t* __restrict__ ulen) {
  typedef cub::BlockScan<int64_t, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t s_first, s_carry;
  if (threadIdx.x == 0) {
    int64_t lo = 0, hi = n;  // first degree > kTcLong
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (deg_sorted[mid] > (uint32_t)kTcLong) hi = mid; else lo = mid + 1;
    }
    s_first = lo;
    s_carry = 0;
  }
  __syncthreads();
  const int64_t first = s_first, nlong = n - first;
  for (int64_t b = 0; b < nlong; b += 1024) {
    const int64_t i = b + threadIdx.x;
    const int64_t t = i < nlong ? (deg_sorted[first + i] + kTcLong - 1) / kTcLong : 0;
    int64_t x;
    Scan(tmp).ExclusiveSum(t, x);
    if (i < nlong) {
      tstart[i] = s_carry + x;
      ulen[first + i] = 0;  // the long rows' tiles reserve their slices on it
    }
    __syncthreads();
    if (threadIdx.x == 1023) s_carry += x + t;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tstart[nlong] = s_carry;
    meta[0] = first;
    meta[1] = s_carry;
  }
}

// long-row tile g -> (long row i, entries [p0, p1) of vertex order[first + i])
__device__ __forceinline__ int64_t tc_tile(int64_t g, const int64_t* __restrict__ tstart,
                                           int64_t nlong) {
  int64_t lo = 0, hi = nlong;  // last i with tstart[i] <= g
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (tstart[mid] <= g) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int64_t tc_fill_range(int64_t p0, int64_t p1, int32_t r,
                                                 const int32_t* __restrict__ idx,
                                                 const int32_t* __restrict__ rank,
                                                 int32_t* __restrict__ out_row, int lane) {
  int64_t out = 0;
  for (int64_t base = p0; base < p1; base += 32) {
    const int64_t p = base + lane;
    int32_t rj = -1;
    if (p < p1) rj = rank[idx[p]];
    const bool keep = rj > r;
    const uint32_t bal = __ballot_sync(GB_FULL, keep);
    if (keep) out_row[out + __popc(bal & ((1u << lane) - 1u))] = rj;
    out += __popc(bal);
  }
  return out;
}

// One pass: U(r) is written where vertex order[r]'s adjacency starts in the
// matrix (it holds at most deg entries), so no count pass, scan or read-back
// of the total is needed; ustart / ulen locate each row.
__global__ void tc_upper_build(int64_t n, const int64_t* __restrict__ off,
                               const int32_t* __restrict__ idx, const int32_t* __restrict__ order,
                               const int32_t* __restrict__ rank, const int64_t* __restrict__ tstart,
                               const int64_t* __restrict__ meta, int64_t* __restrict__ ustart,
                               int64_t* __restrict__ ulen, int32_t* __restrict__ uidx) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t first = meta[0], ntiles = meta[1], nlong = n - first;
  for (int64_t r = w0; r < first; r += nw) {
    const int32_t v = order[r];
    const int64_t p0 = off[v];
    const int64_t c = tc_fill_range(p0, off[v + 1], (int32_t)r, idx, rank, uidx + p0, lane);
    if (lane == 0) {
      ustart[r] = p0;
      ulen[r] = c;
    }
  }
  for (int64_t g = w0; g < ntiles; g += nw) {
    const int64_t i = tc_tile(g, tstart, nlong);
    const int64_t r = first + i;
    const int32_t v = order[r];
    const int64_t p0 = off[v] + (g - tstart[i]) * kTcLong;
    const int64_t p1 = min(p0 + kTcLong, off[v + 1]);
    long long c = 0;  // the tile's count reserves its slice of the row
    for (int64_t p = p0 + lane; p < p1; p += 32) c += rank[idx[p]] > r;
    c = warp_sum_ll(c);
    unsigned long long at = 0;
    if (lane == 0) {
      if (g == tstart[i]) ustart[r] = off[v];
      if (c) at = atomicAdd(reinterpret_cast<unsigned long long*>(ulen + r),
                            (unsigned long long)c);
    }
    at = __shfl_sync(GB_FULL, at, 0);
    if (c) tc_fill_range(p0, p1, (int32_t)r, idx, rank, uidx + off[v] + at, lane);
  }
}

// Top ranks held in a per-warp bitmap.  With the degree ordering the keys of
// the searched lists concentrate on the highest ranks (the hubs): on R-MAT s20
// 99.8 % of them fall in the top 32768, so membership in U(r) is one shared
// load and a bit test; the rest binary-search r's (sorted) adjacency for the
// key's vertex.  No list needs sorting and no search touches U(r) itself.
#ifndef GB_TC_TOP
#define GB_TC_TOP 32768
#endif
constexpr int kTcTopBits = GB_TC_TOP;
constexpr int kTcWords = kTcTopBits / 32;

// The top kTcDense ranks also get a dense adjacency bitmap (8 MB, L2-resident):
// row j holds U(j), whose keys all lie above j.  For a pair (r, j) with j in
// that range, |U(r) & U(j)| is the popcount of the AND of j's row with r's
// bitmap over the words above j -- fewer loads than walking U(j) whenever
// U(j) is denser than one key per 32 ranks (the hub-hub part of R-MAT: 3x
// fewer loads over the whole count at s20).
#ifndef GB_TC_DENSE
#define GB_TC_DENSE 8192
#endif
constexpr int kTcDense = GB_TC_DENSE;
#ifndef GB_TC_KEYS
#define GB_TC_KEYS 4
#endif
constexpr int kTcKeys = GB_TC_KEYS;

__global__ void tc_dense_rows(int64_t n, int32_t dbase, int32_t W, const int64_t* __restrict__ ustart,
                              const int64_t* __restrict__ ulen, const int32_t* __restrict__ uidx,
                              uint32_t* __restrict__ dense) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = dbase + w0; j < n; j += nw) {
    uint32_t* row = dense + (j - dbase) * W;
    for (int64_t q = ustart[j] + lane; q < ustart[j] + ulen[j]; q += 32) {
      const int32_t k = uidx[q] - dbase;
      atomicOr(&row[k >> 5], 1u << (k & 31));
    }
  }
}

// U(r)'s entries below the bitmap (low ranks) go to a per-warp open-address
// hash set when there are at most kTcLoSlots / 2 of them; the keys that miss
// the bitmap then probe it in shared memory instead of binary-searching r's
// adjacency in global memory (a divergent chain of dependent loads).
constexpr int kTcLoSlots = 128;
__device__ __forceinline__ uint32_t tc_hash(int32_t v) {
  return ((uint32_t)v * 2654435761u) >> 25;  // 7 bits: kTcLoSlots
}

// branchless 32-bit lower bound of vertex u in the sorted list nb[0, len)
__device__ __forceinline__ int tc_in_adjacency(const int32_t* __restrict__ nb, int len, int32_t u) {
  const int32_t* b = nb;
  while (len > 1) {
    const int h = len >> 1;
    b = b[h - 1] < u ? b + h : b;
    len -= h;
  }
  return *b == u;
}

// warp per upper row r: count |U(r) & U(j)| for every j in U(r)
__global__ void __launch_bounds__(256)
tc_count(int64_t n, const int64_t* __restrict__ ustart, const int64_t* __restrict__ ulen,
         const int32_t* __restrict__ uidx,
         const int64_t* __restrict__ off, const int32_t* __restrict__ idx,
         const int32_t* __restrict__ order, int32_t dbase, int32_t W,
         const uint32_t* __restrict__ dense, unsigned long long* __restrict__ total) {
  __shared__ uint32_t s_bm[8][kTcWords];
  __shared__ int32_t s_lo[8][kTcLoSlots];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int32_t base = n > kTcTopBits ? (int32_t)(n - kTcTopBits) : 0;
  const int boff = (dbase - base) >> 5;  // word of rank dbase in the row bitmap
  uint32_t* bm = s_bm[wid];
  int32_t* lo_set = s_lo[wid];
  for (int q = lane; q < kTcWords; q += 32) bm[q] = 0;
  for (int q = lane; q < kTcLoSlots; q += 32) lo_set[q] = -1;
  __syncwarp();
  long long c = 0;
  for (int64_t r = w0; r < n; r += nw) {
    const int64_t lo = ustart[r];
    const int64_t len = ulen[r];
    if (len < 2) continue;
    const int32_t* row = uidx + lo;
    int nlow = 0;  // entries of U(r) below the bitmap (warp-uniform count)
    for (int64_t q0 = 0; q0 < len; q0 += 32) {
      const int64_t q = q0 + lane;
      const int32_t v = q < len ? row[q] - base : 0;
      if (q < len && v >= 0) atomicOr(&bm[v >> 5], 1u << (v & 31));
      nlow += __popc(__ballot_sync(GB_FULL, q < len && v < 0));
    }
    // few of them: a shared hash set answers the keys below the bitmap
    const bool lo_hashed = nlow > 0 && nlow <= kTcLoSlots / 2;
    if (lo_hashed) {
      for (int64_t q = lane; q < len; q += 32) {
        const int32_t v = row[q];
        if (v >= base) continue;
        uint32_t h = tc_hash(v);
        while (atomicCAS(&lo_set[h], -1, v) != -1) h = (h + 1) & (kTcLoSlots - 1);
      }
    }
    __syncwarp();
    const int ilen = (int)len;
    const int32_t vr = order[r];  // for keys below the bitmap: search r's sorted adjacency
    const int32_t* nb = idx + off[vr];
    const int nlen = (int)(off[vr + 1] - off[vr]);
    // r's bitmap words of the 32-word window at the top of the dense range
    const int wt = (W > 32 ? W - 32 : 0) + lane;
    const uint32_t bmtop = wt < W ? bm[wt + boff] : 0u;
    uint32_t cr = 0;  // this lane's count for row r
    for (int c0 = 0; c0 < ilen; c0 += 32) {
      // lane = one pair (r, j) of the next 32; classify it
      const int a = c0 + lane;
      int32_t j = -1;
      int64_t jlo = 0, jhi = 0;
      if (a < ilen) {
        j = row[a];
        jlo = ustart[j];
        jhi = jlo + ulen[j];
      }
      int wj = W;  // first dense word holding ranks above j
      bool dn = false;
      if (j >= dbase) {
        wj = (j + 1 - dbase) >> 5;
        dn = W - wj < jhi - jlo;  // fewer words than keys: AND the dense row
      }
      uint32_t top = __ballot_sync(GB_FULL, dn && W - wj <= 32);
      const uint32_t wide = __ballot_sync(GB_FULL, dn && W - wj > 32);
      const uint32_t keyed = __ballot_sync(GB_FULL, !dn && jhi > jlo);
      // dense rows inside the top window: one coalesced word per lane, four
      // pairs' loads in flight
      while (top) {
        uint32_t word[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          word[u] = 0;
          if (top) {
            const int p = __ffs(top) - 1;
            top &= top - 1;
            const int32_t jp = __shfl_sync(GB_FULL, j, p);
            if (wt < W) word[u] = dense[(int64_t)(jp - dbase) * W + wt];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) cr += __popc(word[u] & bmtop);
      }
      for (uint32_t m = wide; m; m &= m - 1) {
        const int p = __ffs(m) - 1;
        const int32_t jp = __shfl_sync(GB_FULL, j, p);
        const int wp = __shfl_sync(GB_FULL, wj, p);
        const uint32_t* arow = dense + (int64_t)(jp - dbase) * W;
        for (int w = wp + lane; w < W; w += 32) cr += __popc(arow[w] & bm[w + boff]);
      }
      // every key k of U(j) has rank k > j > r, so k is in U(r) iff it is a
      // neighbour of r: |U(r) & U(j)| is the count of those memberships
      for (uint32_t m = keyed; m; m &= m - 1) {
        const int p = __ffs(m) - 1;
        const int64_t klo = __shfl_sync(GB_FULL, jlo, p);
        const int64_t khi = __shfl_sync(GB_FULL, jhi, p);
        // kTcKeys keys in flight per lane: the loop is bound by L2 latency
        for (int64_t q = klo + lane; q < khi; q += 32 * kTcKeys) {
          int32_t key[kTcKeys];
#pragma unroll
          for (int u = 0; u < kTcKeys; ++u) key[u] = q + 32 * u < khi ? uidx[q + 32 * u] : -1;
#pragma unroll
          for (int u = 0; u < kTcKeys; ++u) {
            if (key[u] < 0) continue;
            const int32_t v = key[u] - base;
            if (v >= 0) {
              cr += (bm[v >> 5] >> (v & 31)) & 1u;
            } else if (lo_hashed) {
              uint32_t h = tc_hash(key[u]);
              int32_t e;
              while ((e = lo_set[h]) != -1 && e != key[u]) h = (h + 1) & (kTcLoSlots - 1);
              cr += e == key[u];
            } else if (nlow > 0) {
              cr += tc_in_adjacency(nb, nlen, order[key[u]]);
            }
          }
        }
      }
    }
    c += cr;
    __syncwarp();
    for (int64_t q = lane; q < len; q += 32) {
      const int32_t v = row[q] - base;
      if (v >= 0) bm[v >> 5] = 0;
    }
    if (lo_hashed)
      for (int q = lane; q < kTcLoSlots; q += 32) lo_set[q] = -1;
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
  int64_t* ustart = ar.alloc<int64_t>(n);
  int64_t* ulen = ar.alloc<int64_t>(n);
  int32_t* uidx = ar.alloc<int32_t>(a->nnz);  // U(r) at its vertex's adjacency start
  unsigned long long* total = ar.alloc<unsigned long long>(1);
  const int64_t maxlong = a->nnz / kTcLong + 1;  // rows longer than kTcLong
  int64_t* tstart = ar.alloc<int64_t>(maxlong + 1);
  int64_t* meta = ar.alloc<int64_t>(2);
  GB_ARENA_CHECK(ctx, ar);
  tc_degree_keys<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, a->offsets, deg, ids);
  // stable: ties keep ascending vertex id (algorithms.py:209-212)
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, deg, deg2, ids, order, n, 0, 32, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceRadixSort::SortPairs(tmp, tb, deg, deg2, ids, order, n, 0, 32, s));
  tc_rank<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, order, rank);
  tc_long_plan<<<1, 1024, 0, s>>>(n, deg2, tstart, meta, ulen);
  tc_upper_build<<<grid_for(ctx, n * 32, 256, 16), 256, 0, s>>>(n, a->offsets, a->indices, order,
                                                                rank, tstart, meta, ustart, ulen,
                                                                uidx);
  // dense rows of the top ranks, word-aligned with tc_count's row bitmap
  const int64_t tbase = n > kTcTopBits ? n - kTcTopBits : 0;
  const int64_t lowest = n > kTcDense ? n - kTcDense : 0;
  const int32_t dbase = (int32_t)(tbase + ((lowest - tbase) >> 5 << 5));
  const int32_t W = (int32_t)((n - dbase + 31) / 32);
  uint32_t* dense = ar.alloc<uint32_t>((size_t)W * (n - dbase));
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(dense, 0, sizeof(uint32_t) * (size_t)W * (n - dbase), s));
  tc_dense_rows<<<grid_for(ctx, (n - dbase) * 32, 256, 16), 256, 0, s>>>(n, dbase, W, ustart,
                                                                         ulen, uidx, dense);
  GB_CUDA(ctx, cudaMemsetAsync(total, 0, 8, s));
  const int ps = prof_begin(ctx, PROF_TC, a->nnz / 2);
  tc_count<<<resident_grid(ctx, tc_count, 256), 256, 0, s>>>(n, ustart, ulen, uidx, a->offsets,
                                                               a->indices, order, dbase, W, dense,
                                                               total);
  prof_end(ctx, ps);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 9);
  return read_i64(ctx, (const int64_t*)total, count_host);
}

}  // extern "C"
