// Fused SSSP, PageRank and connected-components drivers.
//
//   gb_sssp      algorithms.py:80-119   min-plus relaxation, frontier = strictly
//                improved vertices.  Push: atomicMin on the distance bits
//                (non-negative doubles order like int64); the winning write
//                marks the vertex changed.  Pull: warp per row over in-edges.
//   gb_pagerank  algorithms.py:122-162  alpha/outdeg folded into a per-source
//                scale vector (products identical to the reference's
//                pre-scaled matrix), edge-balanced row tiles for the SpMV, the
//                teleport / delta / error / next-scale epilogue in one pass.
//   gb_cc        algorithms.py:165-203  FastSV: hooking SpMV (pull tiles or
//                push atomics), scatter-min folded into atomics on the parent
//                vector, grandparent + change count + sparsification in one
//                pass.
// Every driver logs the reference direction rule (gb_decide_direction) per
// multiply and synchronizes once per iteration for the loop-exit scalar.
#include <math.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

#include <type_traits>
#include <vector>

#include <cub/cub.cuh>

#include "gb_common.cuh"
#include "gb_lbs.cuh"
#include "gb_rowtiles.cuh"

#ifndef GB_ROW_MINB
#define GB_ROW_MINB 5  // resident 256-thread CTAs per SM of the row-tile pulls (48 registers)
#endif

extern "C" int32_t gb_decide_direction(int64_t nnz, int64_t nrows, int64_t nnz_u, double ratio,
                                       int32_t policy, int64_t* estimate_out);

namespace gb {

// ---------------------------------------------------------------------------
// SSSP
// ---------------------------------------------------------------------------
__device__ __forceinline__ double ld_weight(const void* vals, int dtype, double iso, int64_t p) {
  if (!vals) return iso;
  return dtype == GB_I64 ? (double)__ldg((const long long*)vals + p) : __ldg((const double*)vals + p);
}

__global__ void sssp_init(int64_t n, double* __restrict__ dist, double* __restrict__ fvd,
                          int64_t source, int32_t* __restrict__ F, double* __restrict__ Fv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    dist[i] = i == source ? 0.0 : INFINITY;
    fvd[i] = INFINITY;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    F[0] = (int32_t)source;
    Fv[0] = 0.0;
  }
}

// improve dist[v] to nd; returns true when this call lowered it.  Distances
// are >= 0 (positive weights are validated on the host), so the IEEE bit
// pattern orders like a signed integer.
__device__ __forceinline__ bool relax(double* dist, int32_t v, double nd,
                                      unsigned long long* reached) {
  long long* a = reinterpret_cast<long long*>(dist + v);
  const long long nb = __double_as_longlong(nd);
  if (nb >= *reinterpret_cast<volatile long long*>(a)) return false;
  const long long old = atomicMin(a, nb);
  if (nb < old) {
    if (old == 0x7ff0000000000000ll) atomicAdd(reached, 1ull);
    return true;
  }
  return false;
}

struct SsspPush {
  const int32_t* idx;
  const void* vals;
  int dtype;
  double iso;
  const double* Fv;
  double* dist;
  uint32_t* changed;
  unsigned long long* reached;
  __device__ __forceinline__ void operator()(int64_t k, int64_t p, int64_t e) const {
    const int32_t v = __ldg(idx + p);
    const double nd = ld_weight(vals, dtype, iso, p) + Fv[k];  // mult(A value, u value)
    if (relax(dist, v, nd, reached)) atomicOr(changed + (v >> 5), 1u << (v & 31));
  }
};

// Pull relaxation on edge-balanced row tiles: cand[row] = min over in-edges
// from frontier vertices of w + fvd[src] (non-negative doubles compare as
// int64 bits), then sssp_pull_apply folds cand into dist.
struct SsspMin {
  const void* vals;
  int dtype;
  double iso;
  const double* __restrict__ fvd;
  long long* __restrict__ cand;
  __device__ __forceinline__ double identity() const { return INFINITY; }
  __device__ __forceinline__ double load(int64_t p, int32_t col) const {
    const double u = ld_gather(fvd + col);
    return u == INFINITY ? INFINITY : ld_weight(vals, dtype, iso, p) + u;
  }
  __device__ __forceinline__ double fold(double a, double x) const { return fmin(a, x); }
  __device__ __forceinline__ void emit(int64_t row, double acc, bool whole) const {
    if (acc == INFINITY) return;
    const long long b = __double_as_longlong(acc);
    if (whole) cand[row] = b;
    else atomicMin(cand + row, b);
  }
};

__global__ void __launch_bounds__(256, GB_ROW_MINB)
sssp_pull_tiles(int64_t R, const int32_t* __restrict__ nz_rows, const int64_t* __restrict__ nz_off,
                const int32_t* __restrict__ idx, const int32_t* __restrict__ tile_first,
                const void* vals, int dtype, double iso, const double* __restrict__ fvd,
                long long* __restrict__ cand) {
  SsspMin red{vals, dtype, iso, fvd, cand};
  row_tiles<double>(R, nz_rows, nz_off, idx, tile_first, red);
}

constexpr long long kInfBits = 0x7ff0000000000000ll;

// Folds the pull's candidates into dist.  With `settled` (nullable): also
// totals the stored in-edges (pull offsets `off`) of the rows whose distance
// is now <= low -- the share of the matrix a bounded pull (sssp_pull_exit)
// with this bound would skip.  The next pull takes the bounded kernel when
// that share is large (the share only grows as distances settle).
__device__ __forceinline__ void sssp_apply_body(int64_t n, long long* __restrict__ cand,
                                                double* __restrict__ dist,
                                                uint32_t* __restrict__ changed,
                                                unsigned long long* __restrict__ reached,
                                                const int64_t* __restrict__ off, double low,
                                                unsigned long long* __restrict__ settled) {
  unsigned long long sd = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t ib = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); ib < n; ib += stride) {
    const int64_t i = ib + (threadIdx.x & 31);
    if (i >= n) continue;
    const long long c = cand[i];
    double d = dist[i];
    if (c != kInfBits) {
      cand[i] = kInfBits;
      const double nd = __longlong_as_double(c);
      if (nd < d) {
        if (d == INFINITY) atomicAdd(reached, 1ull);
        dist[i] = nd;
        d = nd;
        atomicOr(changed + (i >> 5), 1u << (i & 31));
      }
    }
    if (settled && d <= low) sd += (unsigned long long)(off[i + 1] - off[i]);
  }
  if (settled) {
    __shared__ unsigned long long s_sd[8];
    sd = (unsigned long long)warp_sum_ll((long long)sd);
    if ((threadIdx.x & 31) == 0) s_sd[threadIdx.x >> 5] = sd;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_sd[w];
      if (t) atomicAdd(settled, t);
    }
  }
}

__global__ void __launch_bounds__(256)
sssp_pull_apply(int64_t n, long long* __restrict__ cand, double* __restrict__ dist,
                uint32_t* __restrict__ changed, unsigned long long* __restrict__ reached,
                const int64_t* __restrict__ off, const long long* __restrict__ fmin,
                const double* __restrict__ wmin, unsigned long long* __restrict__ settled) {
  const double low = settled ? __longlong_as_double(*fmin) + *wmin : 0.0;
  sssp_apply_body(n, cand, dist, changed, reached, off, low, settled);
}

// warp per row over in-edges; contributions only from frontier vertices
__global__ void __launch_bounds__(256)
sssp_pull(int64_t n, const int64_t* __restrict__ off, const int32_t* __restrict__ idx,
          const void* vals, int dtype, double iso, const double* __restrict__ fvd,
          double* __restrict__ dist, uint32_t* __restrict__ changed,
          unsigned long long* __restrict__ reached) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < n; i += nw) {
    double best = INFINITY;
    for (int64_t p = off[i] + lane; p < off[i + 1]; p += 32) {
      const double u = fvd[__ldg(idx + p)];
      if (u != INFINITY) best = fmin(best, ld_weight(vals, dtype, iso, p) + u);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) best = fmin(best, __shfl_xor_sync(GB_FULL, best, o));
    if (lane == 0 && best < dist[i]) {
      if (dist[i] == INFINITY) atomicAdd(reached, 1ull);
      dist[i] = best;
      atomicOr(changed + (i >> 5), 1u << (i & 31));
    }
  }
}

// changed bitmap -> frontier list (+ values) and dense frontier values
__device__ __forceinline__ void sssp_finalize_body(int64_t n, uint32_t* __restrict__ changed,
                                                   const double* __restrict__ dist,
                                                   int32_t* __restrict__ F,
                                                   double* __restrict__ Fv,
                                                   double* __restrict__ fvd,
                                                   unsigned long long* __restrict__ count,
                                                   const int64_t* __restrict__ off,
                                                   unsigned long long* __restrict__ sumdeg,
                                                   long long* __restrict__ fmin);

__global__ void sssp_finalize(int64_t n, uint32_t* __restrict__ changed,
                              const double* __restrict__ dist, int32_t* __restrict__ F,
                              double* __restrict__ Fv, double* __restrict__ fvd,
                              unsigned long long* __restrict__ count,
                              const int64_t* __restrict__ off,
                              unsigned long long* __restrict__ sumdeg,
                              long long* __restrict__ fmin) {
  sssp_finalize_body(n, changed, dist, F, Fv, fvd, count, off, sumdeg, fmin);
}

__device__ __forceinline__ void sssp_finalize_body(int64_t n, uint32_t* __restrict__ changed,
                                                   const double* __restrict__ dist,
                                                   int32_t* __restrict__ F,
                                                   double* __restrict__ Fv,
                                                   double* __restrict__ fvd,
                                                   unsigned long long* __restrict__ count,
                                                   const int64_t* __restrict__ off,
                                                   unsigned long long* __restrict__ sumdeg,
                                                   long long* __restrict__ fmin) {
  // off / sumdeg: also total the new frontier's out-degrees (the edges a
  // push of it would relax).  fmin (nullable, reset to +inf bits before the
  // launch): the smallest listed distance, as bits (distances are >= 0)
  long long dmin = kInfBits;
  const int64_t W = (n + 31) / 32;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t wb = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); wb < W; wb += stride) {
    const int64_t w = wb + (threadIdx.x & 31);
    uint32_t bits = 0;
    if (w < W) {
      bits = changed[w];
      if (bits) changed[w] = 0;
    }
    const int c = __popc(bits);
    long long slot = warp_reserve(count, c);
    unsigned long long deg = 0;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int64_t v = w * 32 + b;
      const double dv = dist[v];
      F[slot] = (int32_t)v;
      Fv[slot] = dv;
      fvd[v] = dv;
      const long long db = __double_as_longlong(dv);
      dmin = db < dmin ? db : dmin;
      if (off) deg += (unsigned long long)(off[v + 1] - off[v]);
      ++slot;
    }
    if (sumdeg) {
      deg = warp_sum_ll((long long)deg);
      if ((threadIdx.x & 31) == 0 && deg) atomicAdd(sumdeg, deg);
    }
  }
  if (fmin) {
    // the wb loop is warp-uniform: every lane gets here
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const long long x = __shfl_xor_sync(GB_FULL, dmin, o);
      dmin = x < dmin ? x : dmin;
    }
    if ((threadIdx.x & 31) == 0 && dmin < *(volatile long long*)fmin) atomicMin(fmin, dmin);
  }
}

__global__ void reset_fvd(int64_t K, const int32_t* __restrict__ F, double* __restrict__ fvd,
                          long long* __restrict__ fmin_reset) {
  // the next finalize records the new frontier's smallest distance
  if (fmin_reset && blockIdx.x == 0 && threadIdx.x == 0) *fmin_reset = kInfBits;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K;
       i += (int64_t)gridDim.x * blockDim.x)
    fvd[F[i]] = INFINITY;
}

// ---------------------------------------------------------------------------
// PageRank
// ---------------------------------------------------------------------------
__global__ void pr_init(int64_t n, const int64_t* __restrict__ out_off, double alpha,
                        double* __restrict__ inv, double* __restrict__ rank,
                        double* __restrict__ y, double* __restrict__ spread) {
  const double r0 = 1.0 / (double)n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = out_off[i + 1] - out_off[i];
    const double s = d > 0 ? alpha / (double)d : 0.0;  // algorithms.py:124-127
    inv[i] = s;
    rank[i] = r0;
    y[i] = s * r0;
    spread[i] = 0.0;
  }
}

struct PrSum {
  const double* __restrict__ y;
  double* __restrict__ spread;
  __device__ __forceinline__ double identity() const { return 0.0; }
  __device__ __forceinline__ double load(int64_t, int32_t col) const { return ld_gather(y + col); }
  __device__ __forceinline__ double fold(double a, double x) const { return a + x; }
  __device__ __forceinline__ void emit(int64_t row, double acc, bool whole) const {
    if (whole) spread[row] = acc;
    else atomicAdd(spread + row, acc);
  }
};

__global__ void __launch_bounds__(256, GB_ROW_MINB)
pr_spmv(int64_t R, const int32_t* __restrict__ nz_rows, const int64_t* __restrict__ nz_off,
        const int32_t* __restrict__ idx, const int32_t* __restrict__ tile_first,
        const double* __restrict__ y, double* __restrict__ spread) {
  PrSum red{y, spread};
  row_tiles<double>(R, nz_rows, nz_off, idx, tile_first, red);
}

// ranks = spread + teleport; error^2 += (ranks - prev)^2; y = inv * ranks;
// spread reset for the next iteration; count of non-zero ranks (next decision)
__device__ __forceinline__ void pr_epilogue_body(int64_t n, double tele,
                                                 const double* __restrict__ inv,
                                                 double* __restrict__ spread,
                                                 const double* __restrict__ prev,
                                                 double* __restrict__ rank, double* __restrict__ y,
                                                 double* __restrict__ err2,
                                                 unsigned long long* __restrict__ nz);

__global__ void __launch_bounds__(256)
pr_epilogue(int64_t n, double tele, const double* __restrict__ inv, double* __restrict__ spread,
            const double* __restrict__ prev, double* __restrict__ rank, double* __restrict__ y,
            double* __restrict__ err2, unsigned long long* __restrict__ nz) {
  pr_epilogue_body(n, tele, inv, spread, prev, rank, y, err2, nz);
}

__device__ __forceinline__ void pr_epilogue_body(int64_t n, double tele,
                                                 const double* __restrict__ inv,
                                                 double* __restrict__ spread,
                                                 const double* __restrict__ prev,
                                                 double* __restrict__ rank, double* __restrict__ y,
                                                 double* __restrict__ err2,
                                                 unsigned long long* __restrict__ nz) {
  __shared__ double s_e[8];
  __shared__ long long s_c[8];
  double e = 0.0;
  long long c = 0;
  // 4 independent elements per thread per step: all loads issued first
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j0 < n; j0 += 4 * stride) {
    double sp[4], pv[4], iv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = j0 + u * stride;
      if (j < n) {
        sp[u] = __ldcs(spread + j);
        pv[u] = __ldcs(prev + j);
        iv[u] = __ldg(inv + j);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = j0 + u * stride;
      if (j < n) {
        const double r = sp[u] + tele;
        const double d = r - pv[u];
        e += d * d;
        c += r != 0.0;
        spread[j] = 0.0;
        rank[j] = r;
        y[j] = iv[u] * r;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    e += __shfl_xor_sync(GB_FULL, e, o);
    c += __shfl_xor_sync(GB_FULL, c, o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { s_e[wid] = e; s_c[wid] = c; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double te = 0.0;
    long long tc = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { te += s_e[i]; tc += s_c[i]; }
    atomicAdd(err2, te);
    atomicAdd(nz, (unsigned long long)tc);
  }
}

// ---------------------------------------------------------------------------
// Connected components (FastSV)
// ---------------------------------------------------------------------------
// Labels are vertex ids < n < 2^31: the driver keeps parent / grandparent /
// min-neighbour vectors as int32 (half the gather bytes, the 67 MB label
// vector of s24 stays L2-resident) and widens the result to int64 at the end.
// INT32_MAX plays the reference's INT64_MAX sparsification sentinel
// (algorithms.py:33, 201); it is never a valid label.
constexpr int kImax32 = 0x7fffffff;

struct CcMin {
  const int* __restrict__ gp;
  int* __restrict__ hook;
  __device__ __forceinline__ int identity() const { return kImax32; }
  __device__ __forceinline__ int load(int64_t, int32_t col) const { return ld_gather(gp + col); }
  __device__ __forceinline__ int fold(int a, int x) const { return x < a ? x : a; }
  __device__ __forceinline__ void emit(int64_t row, int acc, bool whole) const {
    if (acc == kImax32) return;  // hook was reset to the identity
    if (whole) hook[row] = acc;
    else atomicMin(hook + row, acc);
  }
};

__global__ void __launch_bounds__(256, GB_ROW_MINB)
cc_pull(int64_t R, const int32_t* __restrict__ nz_rows, const int64_t* __restrict__ nz_off,
        const int32_t* __restrict__ idx, const int32_t* __restrict__ tile_first,
        const int* __restrict__ gp, int* __restrict__ hook) {
  CcMin red{gp, hook};
  row_tiles<int>(R, nz_rows, nz_off, idx, tile_first, red);
}

// Pull when most grandparents are sparsified away (sentinel): a live bitmap
// (n/8 bytes, L1-friendly, written by the shortcut pass) is probed before the
// 4-byte gp gather, so the iterations with few live grandparents stop paying
// a random gather per entry (s24: 1.95 ms for every pull, at 100 %, 49 % and
// 12 % live, before).
struct CcMinLive {
  const int* __restrict__ gp;
  const uint32_t* __restrict__ live;
  int* __restrict__ hook;
  __device__ __forceinline__ int identity() const { return kImax32; }
  __device__ __forceinline__ int load(int64_t, int32_t col) const {
    return (ld_probe(live + (col >> 5)) >> (col & 31)) & 1u ? ld_gather(gp + col) : kImax32;
  }
  __device__ __forceinline__ int fold(int a, int x) const { return x < a ? x : a; }
  __device__ __forceinline__ void emit(int64_t row, int acc, bool whole) const {
    if (acc == kImax32) return;
    if (whole) hook[row] = acc;
    else atomicMin(hook + row, acc);
  }
};

__global__ void __launch_bounds__(256, GB_ROW_MINB)
cc_pull_live(int64_t R, const int32_t* __restrict__ nz_rows, const int64_t* __restrict__ nz_off,
             const int32_t* __restrict__ idx, const int32_t* __restrict__ tile_first,
             const int* __restrict__ gp, const uint32_t* __restrict__ live, int* __restrict__ hook) {
  CcMinLive red{gp, live, hook};
  row_tiles<int>(R, nz_rows, nz_off, idx, tile_first, red);
}

// The first iteration's pull: every grandparent is still its own id
// (cc_init), so min over neighbours of gp[j] is the smallest column id of the
// row -- the same hook values from the index stream alone, no gathers (s24:
// one full pull of 520 M random 4-byte gathers becomes a streaming read).
struct CcMinId {
  int* __restrict__ hook;
  __device__ __forceinline__ int identity() const { return kImax32; }
  __device__ __forceinline__ int load(int64_t, int32_t col) const { return col; }
  __device__ __forceinline__ int fold(int a, int x) const { return x < a ? x : a; }
  __device__ __forceinline__ void emit(int64_t row, int acc, bool whole) const {
    if (acc == kImax32) return;
    if (whole) hook[row] = acc;
    else atomicMin(hook + row, acc);
  }
};

__global__ void __launch_bounds__(256, GB_ROW_MINB)
cc_pull_first(int64_t R, const int32_t* __restrict__ nz_rows, const int64_t* __restrict__ nz_off,
              const int32_t* __restrict__ idx, const int32_t* __restrict__ tile_first,
              int* __restrict__ hook) {
  CcMinId red{hook};
  row_tiles<int>(R, nz_rows, nz_off, idx, tile_first, red);
}

// Bounded min pulls over the row bins (gb_mv_binned.cu's plan: short rows a
// lane each, medium rows a half-warp each, long rows in 512-entry tiles, 32
// tiles per warp batch).  A min pull whose consumer only uses a row's result
// when it is below some per-row value can skip rows and stop reading early
// given a lower bound `low` on every value the pull can gather:
//   * a row whose consumer value is <= low cannot change: skipped;
//   * a row whose running minimum reaches low has its minimum: it stops.
// Op supplies the value type T, identity(), skip(row), load(p, col),
// reached(acc) (acc <= low) and emit(row, acc, whole) (whole: the row is
// complete in this warp; else an atomic min of a partial tile).
template <class T>
__device__ __forceinline__ T group_min(unsigned mask, T v, int width) {
  if constexpr (std::is_same<T, int>::value) {
    return __reduce_min_sync(mask, v);
  } else {
    for (int o = width >> 1; o > 0; o >>= 1) {
      const T x = __shfl_xor_sync(mask, v, o);
      v = x < v ? x : v;
    }
    return v;
  }
}

template <class Op>
__device__ __forceinline__ void bins_min_pull(int64_t nL, const int32_t* __restrict__ L_row,
                                              const int64_t* __restrict__ L_beg,
                                              const int64_t* __restrict__ L_end, int64_t nM,
                                              const int32_t* __restrict__ M_rows, int64_t nS,
                                              const int32_t* __restrict__ S_rows,
                                              const int64_t* __restrict__ off,
                                              const int32_t* __restrict__ idx, const Op& op) {
  using T = typename Op::T;
  const T ident = op.identity();
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;

  // ---- long rows: 512-entry tiles in batches of Bt consecutive tiles per
  // warp (mostly one hub row); a row that reached the bound in an earlier
  // tile of the batch skips the rest of its tiles.  Bt = 32, halved until
  // the batches cover every warp (s20: 37 K tiles over 5.9 K warps -- 32-tile
  // batches had left 80 % of the warps idle and tripled a heavy SSSP pull)
  int Bt = 32;
  while (Bt > 1 && (nL + Bt - 1) / Bt < nw) Bt >>= 1;
  for (int64_t g = w0; g * Bt < nL; g += nw) {
    const int64_t ti = g * Bt + lane;
    int32_t row = -1;
    int64_t tb = 0, te = 0;
    if (lane < Bt && ti < nL) {
      row = __ldg(L_row + ti);
      tb = __ldg(L_beg + ti);
      te = __ldg(L_end + ti);
    }
    uint32_t bal = __ballot_sync(GB_FULL, row >= 0 && !op.skip(row));
    int32_t done = -1;
    while (bal) {
      const int j = __ffs(bal) - 1;
      bal &= bal - 1;
      const int32_t rr = __shfl_sync(GB_FULL, row, j);
      const int64_t beg = __shfl_sync(GB_FULL, tb, j), end = __shfl_sync(GB_FULL, te, j);
      if (rr == done) continue;
      T acc = ident;
      for (int64_t base = beg; base < end; base += 256) {
        int32_t c[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int64_t p = base + 32 * k + lane;
          c[k] = p < end ? ld_stream(idx + p) : -1;
        }
        T x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = c[k] >= 0 ? op.load(base + 32 * k + lane, c[k]) : ident;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = x[k] < acc ? x[k] : acc;
        acc = group_min<T>(GB_FULL, acc, 32);
        if (op.reached(acc)) break;
      }
      if (lane == 0) op.emit(rr, acc, false);
      if (op.reached(acc)) done = rr;
    }
  }

  // ---- medium rows (17..512 entries): each lane first probes its own row's
  // first 8 entries -- a row that meets the bound there costs one round trip
  // (a uniform graph's late pulls: most rows) -- and the rest continue a
  // half-warp per row, two rows at a time, 128 entries a pass
  const int half = lane >> 4, hl = lane & 15;
  const unsigned hmask = 0xffffu << (16 * half);
  for (int64_t g = w0; g * 32 < nM; g += nw) {
    const int64_t i = g * 32 + lane;
    const int32_t r = i < nM ? __ldg(M_rows + i) : -1;
    const bool ok = r >= 0 && !op.skip(r);
    int64_t lo = 0, hi = 0;
    T pacc = ident;  // the probe's minimum of my row
    if (ok) {
      lo = __ldg(off + r);
      hi = __ldg(off + r + 1);
      int32_t c[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) c[k] = __ldg(idx + lo + k);  // rows hold >= 17 entries
      T x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = op.load(lo + k, c[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) pacc = x[k] < pacc ? x[k] : pacc;
      lo += 8;
    }
    const bool more = ok && !op.reached(pacc);
    if (ok && !more) op.emit(r, pacc, true);
    uint32_t bal = __ballot_sync(GB_FULL, more);
    while (bal) {
      const int j0 = __ffs(bal) - 1;
      bal &= bal - 1;
      const int j1 = bal ? __ffs(bal) - 1 : -1;
      if (bal) bal &= bal - 1;
      const int src = half ? (j1 >= 0 ? j1 : j0) : j0;
      const int32_t rr = __shfl_sync(GB_FULL, r, src);
      const int64_t l = __shfl_sync(GB_FULL, lo, src);
      int64_t h = __shfl_sync(GB_FULL, hi, src);
      if (half && j1 < 0) h = l;  // no second row: the upper half idles
      T acc = __shfl_sync(GB_FULL, pacc, src);
      for (int64_t base = l; base < h; base += 128) {
        int32_t c[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int64_t p = base + 16 * k + hl;
          c[k] = p < h ? ld_stream(idx + p) : -1;
        }
        T x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = c[k] >= 0 ? op.load(base + 16 * k + hl, c[k]) : ident;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = x[k] < acc ? x[k] : acc;
        acc = group_min<T>(hmask, acc, 16);
        if (op.reached(acc)) break;
      }
      if (hl == 0 && h > l) op.emit(rr, acc, true);
    }
  }

  // ---- short rows: a lane per row
  for (int64_t g = w0; g * 32 < nS; g += nw) {
    const int64_t i = g * 32 + lane;
    const int32_t r = i < nS ? __ldg(S_rows + i) : -1;
    if (r >= 0 && !op.skip(r)) {
      const int64_t lo = __ldg(off + r);
      const int len = (int)(__ldg(off + r + 1) - lo);
      int32_t c[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) c[q] = q < len ? __ldg(idx + lo + q) : -1;
      T acc = ident;
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        T x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          x[k] = c[8 * w + k] >= 0 ? op.load(lo + 8 * w + k, c[8 * w + k]) : ident;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = x[k] < acc ? x[k] : acc;
      }
      op.emit(r, acc, true);
    }
  }
}

// CC: hook[u] only matters through min(mn[u], hook[u]) (cc_hook), and no
// gathered grandparent is below `low`, the smallest live grandparent (the
// previous shortcut pass records it; 0, the smallest label, is always a
// valid bound).  Rows with mn[u] <= low are skipped, a row stops once its
// minimum reaches low -- the proposals are exactly the full pull's.  In the
// first gathering pull of an R-MAT graph most grandparents are already the
// giant component's label 0: hub lists, which start at the hubs, stop within
// their first tile, and most rows after one pass.
struct CcBound {
  using T = int;
  const int* __restrict__ gp;
  const int* __restrict__ mn;
  int low;
  int* __restrict__ hook;
  __device__ __forceinline__ int identity() const { return kImax32; }
  __device__ __forceinline__ bool skip(int32_t r) const { return __ldg(mn + r) <= low; }
  __device__ __forceinline__ int load(int64_t, int32_t col) const { return ld_gather(gp + col); }
  __device__ __forceinline__ bool reached(int acc) const { return acc <= low; }
  __device__ __forceinline__ void emit(int32_t r, int acc, bool whole) const {
    if (acc == kImax32) return;
    if (whole) hook[r] = acc;
    else atomicMin(hook + r, acc);
  }
};

__global__ void __launch_bounds__(256, 4)
cc_pull_exit(int64_t nL, const int32_t* __restrict__ L_row, const int64_t* __restrict__ L_beg,
             const int64_t* __restrict__ L_end, int64_t nM, const int32_t* __restrict__ M_rows,
             int64_t nS, const int32_t* __restrict__ S_rows, const int64_t* __restrict__ off,
             const int32_t* __restrict__ idx, const int* __restrict__ gp,
             const int* __restrict__ mn, const int* __restrict__ lowp, int* __restrict__ hook) {
  const CcBound op{gp, mn, *lowp, hook};
  bins_min_pull(nL, L_row, L_beg, L_end, nM, M_rows, nS, S_rows, off, idx, op);
}

// SSSP: cand[u] = min over in-edges from the frontier of w + d(src) only
// matters where it is below dist[u] (sssp_pull_apply), and every candidate
// is at least low = (smallest frontier distance, recorded by the finalize
// that listed the frontier) + (smallest weight of the matrix).  Rows with
// dist[u] <= low are settled for this iteration and skipped; a row stops at
// low.  At R-MAT s20 the heavy pulls after the source skip 37 % / 81 % of the
// stored entries this way.
struct SsspBound {
  using T = double;
  const void* vals;
  int dtype;
  double iso;
  const double* __restrict__ fvd;
  const double* __restrict__ dist;
  double low;
  long long* __restrict__ cand;
  __device__ __forceinline__ double identity() const { return INFINITY; }
  __device__ __forceinline__ bool skip(int32_t r) const { return dist[r] <= low; }
  __device__ __forceinline__ double load(int64_t p, int32_t col) const {
    const double u = ld_gather(fvd + col);
    return u == INFINITY ? INFINITY : ld_weight(vals, dtype, iso, p) + u;
  }
  __device__ __forceinline__ bool reached(double acc) const { return acc <= low; }
  __device__ __forceinline__ void emit(int32_t r, double acc, bool whole) const {
    if (acc == INFINITY) return;
    const long long b = __double_as_longlong(acc);
    if (whole) cand[r] = b;
    else atomicMin(cand + r, b);
  }
};

__global__ void __launch_bounds__(256, 4)
sssp_pull_exit(int64_t nL, const int32_t* __restrict__ L_row, const int64_t* __restrict__ L_beg,
               const int64_t* __restrict__ L_end, int64_t nM, const int32_t* __restrict__ M_rows,
               int64_t nS, const int32_t* __restrict__ S_rows, const int64_t* __restrict__ off,
               const int32_t* __restrict__ idx, const void* vals, int dtype, double iso,
               const double* __restrict__ fvd, const double* dist, double* const* distp,
               const long long* __restrict__ fmin_bits, const double* __restrict__ wminp,
               long long* __restrict__ cand) {
  // dist: the distances, or null and *distp (the graph loop's state)
  const SsspBound op{vals, dtype, iso, fvd, dist ? dist : *distp,
                     __longlong_as_double(*fmin_bits) + *wminp, cand};
  bins_min_pull(nL, L_row, L_beg, L_end, nM, M_rows, nS, S_rows, off, idx, op);
}

// The row bins of a pull orientation (CC rows, SSSP in-edges) in one
// cudaMalloc block (*mem, the caller frees it); synchronises.  Leaves *mem
// null (every pull keeps the edge-balanced tiles) when the rows are empty or
// with GB_PULL_EXIT=0.  Whether a pull takes the bounded kernel is decided
// per iteration on the device from a predictor of how much it would skip
// (CC: live grandparents equal to the bound, cc_count_low; SSSP: edges of
// settled rows) -- with no early exits the bins' per-row round trips lose to
// the edge-balanced tiles (uniform s24 CC with bins on every full pull: 9.3
// vs 8.0 ms).  GB_PULL_EXIT=2 takes the bounded kernel for every CC full
// pull and every SSSP pull (tests).
static int pull_exit_mode() {
  static const int m = getenv("GB_PULL_EXIT") ? atoi(getenv("GB_PULL_EXIT")) : 1;
  return m;
}
// a full CC pull takes the bounded kernel when at least this share of the
// vertices have a live grandparent equal to the bound (GB_CC_EXIT_SHARE)
static double cc_exit_share() {
  static double v = -1.0;
  if (v < 0) {
    const char* e = getenv("GB_CC_EXIT_SHARE");
    v = pull_exit_mode() == 2 ? 0.0 : (e ? atof(e) : 0.2);
  }
  return v;
}
// ... or when at most this share of the vertices are non-empty rows above
// the bound (GB_CC_EXIT_ROWS)
static double cc_exit_rows() {
  static double v = -1.0;
  if (v < 0) {
    const char* e = getenv("GB_CC_EXIT_ROWS");
    v = e ? atof(e) : 0.1;
  }
  return v;
}
// ar: the storage comes from the caller's per-call arena (the host-driven
// loops; nothing to free, no device-wide synchronisation); null: one
// cudaMalloc block the caller frees (the cached loop graphs)
static gb_status pull_bins_build(gb_ctx* ctx, const gb_csr* rows, gb_bin_plan* b, void** mem,
                                 Arena* ar = nullptr) {
  *mem = nullptr;
  *b = gb_bin_plan{};
  if (pull_exit_mode() == 0 || rows->nrows == 0) return GB_OK;
  int64_t c[3];
  GB_TRY(gb_bin_plan_counts(ctx, rows, c));
  const size_t bytes = 4 * (size_t)(c[0] + c[1] + c[2]) + 16 * (size_t)c[2] + 64;
  if (ar) {
    *mem = ar->raw(bytes);
    if (ar->failed || !*mem) {
      *mem = nullptr;
      return set_error(ctx, GB_ERR_OOM, "pull bins: scratch allocation of %zu bytes", bytes);
    }
  } else if (cudaMalloc(mem, bytes) != cudaSuccess) {
    cudaGetLastError();
    *mem = nullptr;
    return set_error(ctx, GB_ERR_OOM, "pull bins: cudaMalloc of %zu bytes", bytes);
  }
  char* m = static_cast<char*>(*mem);
  b->n_short = c[0];
  b->n_mid = c[1];
  b->n_long_tiles = c[2];
  b->tile_beg = (const int64_t*)m;
  b->tile_end = (const int64_t*)(m + 8 * c[2]);
  int32_t* r = (int32_t*)(m + 16 * c[2]);
  b->tile_row = r;
  b->mid_rows = r + c[2];
  b->short_rows = r + c[2] + c[1];
  const gb_status st = gb_bin_plan_fill(ctx, rows, b);
  if (st != GB_OK) {
    if (!ar) cudaFree(*mem);
    *mem = nullptr;
  }
  return st;
}

static void cc_pull_exit_launch(gb_ctx* ctx, cudaStream_t s, const gb_bin_plan& b,
                                const gb_csr* rows, const int* gp, const int* mn, const int* low,
                                int* hook) {
  cc_pull_exit<<<resident_grid(ctx, cc_pull_exit, 256), 256, 0, s>>>(
      b.n_long_tiles, b.tile_row, b.tile_beg, b.tile_end, b.n_mid, b.mid_rows, b.n_short,
      b.short_rows, rows->offsets, rows->indices, gp, mn, low, hook);
}

// With rows that start at their minimum (any sorted CSR) the first pull is
// one load per row.
__global__ void cc_hook_first(int64_t n, const int64_t* __restrict__ off,
                              const int32_t* __restrict__ idx, int* __restrict__ hook) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = off[r];
    hook[r] = p < off[r + 1] ? idx[p] : kImax32;
  }
}

__global__ void cc_first_is_min(int64_t n, const int64_t* __restrict__ off,
                                const int32_t* __restrict__ idx, const int* __restrict__ rmin,
                                int* __restrict__ bad) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = off[r];
    if (p < off[r + 1] && idx[p] != rmin[r]) *bad = 1;
  }
}

// a pull iteration probes the live bitmap first when fewer than this share
// of the grandparents are live (GB_CC_LIVE_SHARE)
static double cc_live_share() {
  static double v = -1.0;
  if (v < 0) {
    const char* e = getenv("GB_CC_LIVE_SHARE");
    v = e ? atof(e) : 0.3;
  }
  return v;
}

// A pull iteration (the reference rule's decision, logged as such) whose
// live grandparents are fewer than this share of n runs as the transposed
// traversal: for each live j, min-fold gp[j] into hook[i] over column j of A.
// Column j lists exactly the rows i with A(i, j), so the hook values are the
// pull's, bit for bit, from sum(deg(live)) edges instead of a pass over all
// of A (GB_CC_PUSH_SHARE).
static double cc_push_share() {
  static double v = -1.0;
  if (v < 0) {
    const char* e = getenv("GB_CC_PUSH_SHARE");
    v = e ? atof(e) : 0.2;
  }
  return v;
}

struct CcPush {
  const int32_t* idx;
  const int32_t* F;
  const int* gp;
  int* hook;
  __device__ __forceinline__ void operator()(int64_t k, int64_t p, int64_t e) const {
    const int32_t i = __ldg(idx + p);
    const int g = gp[F[k]];
    if (g < hook[i]) atomicMin(hook + i, g);
  }
};

__global__ void iota_i32(int64_t n, int32_t* __restrict__ a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int32_t)i;
}

__global__ void fill_i64(int64_t n, long long v, long long* __restrict__ a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

__global__ void fill_i32(int64_t n, int v, int* __restrict__ a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

// Format check behind the gather-free first pull: does every row start at
// its smallest column (any sorted CSR; from_csr may wrap unsorted rows)?
// Computed once per matrix (the csr's content id `gen`) and shared by both
// loop engines.
struct CcFirstMin {
  uint64_t gen = 0;
  int64_t n = 0, nnz = 0;
  bool first_min = false;
};

static void cc_first_min_free(void* p) { delete static_cast<CcFirstMin*>(p); }

static gb_status cc_rows_start_at_min(gb_ctx* ctx, const gb_csr* rows, const RowTilesPlan& plan,
                                      bool* out) {
  void** slot = ctx_slot(ctx, SLOT_CC_FIRSTMIN, cc_first_min_free);
  auto* c = static_cast<CcFirstMin*>(*slot);
  if (c && rows->gen != 0 && c->gen == rows->gen && c->n == rows->nrows && c->nnz == rows->nnz) {
    *out = c->first_min;
    return GB_OK;
  }
  const int64_t n = rows->nrows;
  cudaStream_t s = stream_of(ctx);
  Arena ar(ctx);
  int* rmin = ar.alloc<int>(n);
  int* bad = ar.alloc<int>(2);
  GB_ARENA_CHECK(ctx, ar);
  fill_i32<<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(n, kImax32, rmin);
  GB_CUDA(ctx, cudaMemsetAsync(bad, 0, 8, s));
  if (plan.R)
    cc_pull_first<<<resident_grid(ctx, cc_pull_first, 256), 256, 0, s>>>(
        plan.R, plan.nz_rows, plan.nz_off, rows->indices, plan.tile_first, rmin);
  cc_first_is_min<<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(n, rows->offsets, rows->indices, rmin,
                                                             bad);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 4);
  int64_t h = 1;
  GB_TRY(read_i64(ctx, (const int64_t*)bad, &h));
  if (!c) *slot = c = new CcFirstMin();
  c->gen = rows->gen;
  c->n = n;
  c->nnz = rows->nnz;
  c->first_min = (h & 0xffffffff) == 0;
  *out = c->first_min;
  return GB_OK;
}


__global__ void cc_init(int64_t n, int* __restrict__ parent, int* __restrict__ mn,
                        int* __restrict__ gp, int* __restrict__ gpp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    parent[i] = mn[i] = gp[i] = gpp[i] = (int)i;
}

// mn = min(mn, hooked); parent = min(parent, mn); parent[pp[k]] = min(.., mn[k])
// (the scatter-min overwrite of kernels.py:538-583 followed by the two Min
// folds of algorithms.py:192-193 equals this atomic min)
__global__ void cc_hook(int64_t n, const int* __restrict__ hook, int* __restrict__ mn,
                        const int* __restrict__ pp, int* __restrict__ parent,
                        int* __restrict__ low_reset) {
  // the pull has read the bound; the shortcut pass after this recomputes it
  if (low_reset && blockIdx.x == 0 && threadIdx.x == 0) *low_reset = kImax32;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    int m = mn[k];
    const int h = hook[k];
    if (h < m) { m = h; mn[k] = m; }
    if (m == kImax32) continue;  // nothing to propose (sparsified / isolated)
    // read first: most targets already hold a smaller label (the giant
    // component's root is the target of millions of k), so the atomic --
    // which serialises on one L2 slice per address -- is rarely issued.  The
    // read goes through L1: parent only decreases inside the kernel, so a
    // stale cached value is never below the true one and at worst issues an
    // unneeded atomic (a volatile read sent every k to the root's L2 slice)
    if (m < __ldca(parent + k)) atomicMin(parent + k, m);
    const int t = pp[k];
    if (m < __ldca(parent + t)) atomicMin(parent + t, m);
  }
}

// gp = parent[parent]; changed = gp != gp_prev; gp_prev = gp; sparsify.
// Counts are reduced per block (one atomic per block, not per warp: the two
// counters are single addresses every block hits).
__device__ __forceinline__ void cc_shortcut_body(int64_t n, const int* __restrict__ parent,
                                                 int* __restrict__ gp, int* __restrict__ gpp,
                                                 int sparsify,
                                                 unsigned long long* __restrict__ changed,
                                                 unsigned long long* __restrict__ live,
                                                 uint32_t* __restrict__ livebm,
                                                 int* __restrict__ low);

__global__ void __launch_bounds__(256)
cc_shortcut(int64_t n, const int* __restrict__ parent, int* __restrict__ gp,
            int* __restrict__ gpp, int sparsify, unsigned long long* __restrict__ changed,
            unsigned long long* __restrict__ live, uint32_t* __restrict__ livebm,
            int* __restrict__ low) {
  cc_shortcut_body(n, parent, gp, gpp, sparsify, changed, live, livebm, low);
}

__device__ __forceinline__ void cc_shortcut_body(int64_t n, const int* __restrict__ parent,
                                                 int* __restrict__ gp, int* __restrict__ gpp,
                                                 int sparsify,
                                                 unsigned long long* __restrict__ changed,
                                                 unsigned long long* __restrict__ live,
                                                 uint32_t* __restrict__ livebm,
                                                 int* __restrict__ low) {
  // low (nullable): atomic min of the live grandparents (reset by cc_hook)
  __shared__ long long s_c[8], s_l[8];
  __shared__ int s_m[8];
  long long c = 0, l = 0;
  int lmin = kImax32;
  // four independent pointer jumps in flight per thread (latency-bound); the
  // loop bound is warp-uniform (the live-bitmap ballot needs every lane)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int lane_ = threadIdx.x & 31;
  for (int64_t kb = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); kb < n;
       kb += 4 * stride) {
    const int64_t k0 = kb + lane_;
    int p[4], g[4], q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t k = k0 + u * stride;
      p[u] = k < n ? parent[k] : 0;
      q[u] = k < n ? gpp[k] : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) g[u] = __ldg(parent + p[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t k = k0 + u * stride;
      bool is_live = false;
      if (k < n) {
        const bool ch = g[u] != q[u];
        gpp[k] = g[u];
        const int out = (sparsify && !ch) ? kImax32 : g[u];
        gp[k] = out;
        c += ch;
        is_live = out != kImax32;
        l += is_live;
        lmin = out < lmin ? out : lmin;
      }
      if (livebm) {
        // the 32 lanes hold 32 consecutive vertices (block and grid strides
        // are multiples of 32): one ballot is one bitmap word
        const uint32_t wbits = __ballot_sync(GB_FULL, is_live);
        const int64_t kw = k - (threadIdx.x & 31);
        if ((threadIdx.x & 31) == 0 && kw < n) livebm[kw >> 5] = wbits;
      }
    }
  }
  c = warp_sum_ll(c);
  l = warp_sum_ll(l);
  lmin = __reduce_min_sync(GB_FULL, lmin);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { s_c[wid] = c; s_l[wid] = l; s_m[wid] = lmin; }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tc = 0, tl = 0;
    int tm = kImax32;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      tc += s_c[i];
      tl += s_l[i];
      tm = s_m[i] < tm ? s_m[i] : tm;
    }
    if (tc) atomicAdd(changed, (unsigned long long)tc);
    if (tl) atomicAdd(live, (unsigned long long)tl);
    // read first: after the first blocks the bound is usually settled (0)
    if (low && tm < *(volatile int*)low) atomicMin(low, tm);
  }
}

// frontier list of live grandparents (gp != sentinel) for a push iteration.
// The order is free (the push folds with min), so a warp reserves once per
// 1024-vertex chunk: one counter atomic per warp and iteration measured
// 0.31-0.42 ms at s24, serialised on the single address.
__global__ void cc_list(int64_t n, const int* __restrict__ gp, int32_t* __restrict__ F,
                        unsigned long long* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = w0 * 1024; c < n; c += nw * 1024) {
    const int64_t end = c + 1024 < n ? c + 1024 : n;
    int cnt = 0;
    for (int64_t k = c + lane; k < end; k += 32) cnt += gp[k] != kImax32;
    cnt = __reduce_add_sync(GB_FULL, cnt);
    if (cnt == 0) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(count, (unsigned long long)cnt);
    base = __shfl_sync(GB_FULL, base, 0);
    for (int64_t k0 = c; k0 < end; k0 += 32) {
      const int64_t k = k0 + lane;
      const bool l = k < end && gp[k] != kImax32;
      const uint32_t bal = __ballot_sync(GB_FULL, l);
      if (l) F[base + __popc(bal & ((1u << lane) - 1u))] = (int32_t)k;
      base += __popc(bal);
    }
  }
}

// The predictors of the next bounded pull (cc_pull_exit), after the
// shortcut pass recorded the bound: out[0] = live grandparents equal to it
// (rows meet it early), out[1] = non-empty rows (the R ids of nz_rows) with
// mn at or below it (the rows the bounded pull skips) -- counted only when
// fewer than push_share of the grandparents are live (*livep, from the
// shortcut), the case where the bounded pull competes with the transposed
// push; otherwise out[1] stays 0
__global__ void __launch_bounds__(256)
cc_count_low(int64_t n, const int* __restrict__ gp, const int* __restrict__ mn, int64_t R,
             const int32_t* __restrict__ nz_rows, const int* __restrict__ lowp,
             const unsigned long long* __restrict__ livep, double push_share,
             unsigned long long* __restrict__ out) {
  __shared__ unsigned long long s_n[8], s_u[8];
  const int low = *lowp;
  const bool rows = (double)*livep < push_share * (double)n;
  unsigned long long c = 0, u = 0;
  // four independent elements per thread and pass (the mn lookups are
  // dependent gathers; one at a time the pass was latency-bound)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
    int g[4];
    int32_t r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t i = i0 + k * stride;
      g[k] = i < n ? gp[i] : kImax32;
      r[k] = rows && i < R ? nz_rows[i] : -1;
    }
    int m[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) m[k] = r[k] >= 0 ? __ldg(mn + r[k]) : kImax32;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      c += g[k] == low && low != kImax32;
      u += r[k] >= 0 && m[k] <= low;
    }
  }
  c = (unsigned long long)warp_sum_ll((long long)c);
  u = (unsigned long long)warp_sum_ll((long long)u);
  if ((threadIdx.x & 31) == 0) {
    s_n[threadIdx.x >> 5] = c;
    s_u[threadIdx.x >> 5] = u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0, tu = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      t += s_n[w];
      tu += s_u[w];
    }
    if (t) atomicAdd(out, t);
    if (tu) atomicAdd(out + 1, tu);
  }
}

__global__ void widen_i32(int64_t n, const int* __restrict__ a, long long* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i];
}

// ===========================================================================
// Device-resident iteration loops: PageRank, FastSV and
// SSSP as ONE CUDA-graph launch each -- a WHILE conditional node whose body
// runs an iteration and a single-thread step kernel that logs the reference
// direction rule (kernels.py:108-126, half-even rint), evaluates the loop
// exit (algorithms.py:160 / 196-197 / 114-118) and sets the loop handle;
// CC and SSSP pick their multiply in a two-way SWITCH node (pull | push).
// No host synchronisation inside the loop: the log and the iteration count
// are read once, after it.  The graphs are cached per context and matrix
// (gb_csr.gen) like the BFS graph; per-call parameters travel in a device
// state block written before each launch.  Push multiplies size themselves
// from a device count: a warp per frontier entry, entries longer than
// kLongPush edges cut into 512-edge tasks for a second pass.
// ===========================================================================
#ifndef GB_LONG_PUSH
#define GB_LONG_PUSH 1024  // A/B: 4096 / 1024 / 512 / 256 -> SSSP s20 1.63 / 1.56 / 1.57 / 1.60 ms, CC equal
#endif
constexpr int64_t kLongPush = GB_LONG_PUSH;
enum { kLoopGraph = 0, kLoopHost = 1 };
static int g_loop_engine = -1;
static int loop_engine() {
  if (g_loop_engine < 0) {
    const char* e = getenv("GB_LOOP_GRAPH");
    g_loop_engine = (e && atoi(e) == 0) ? kLoopHost : kLoopGraph;
  }
  return g_loop_engine;
}

__device__ __forceinline__ int32_t decide_dev(int64_t nnz, int64_t nrows, int64_t k, double ratio,
                                              int32_t policy, int64_t* est) {
  const double d = nrows ? (double)nnz / (double)nrows : 0.0;
  const int64_t e = (int64_t)rint(d * (double)k);  // Python round: half-even
  *est = e;
  int32_t dir = (double)e > (double)nnz * ratio ? GB_DIR_PULL : GB_DIR_PUSH;
  if (policy == GB_DIR_PUSH) dir = GB_DIR_PUSH;
  if (policy == GB_DIR_PULL) dir = GB_DIR_PULL;
  return dir;
}

__device__ __forceinline__ int32_t log_decision(int64_t* log, int64_t it, int64_t nnz,
                                                int64_t nrows, int64_t k, double ratio,
                                                int32_t policy) {
  int64_t est = 0;
  const int32_t dir = decide_dev(nnz, nrows, k, ratio, policy, &est);
  log[3 * it] = dir;
  log[3 * it + 1] = k;
  log[3 * it + 2] = est;
  return dir;
}

template <class Fn>
static cudaError_t loop_capture_into(cudaGraph_t g, cudaStream_t cs, Fn fn) {
  cudaError_t e = cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0,
                                                cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) return e;
  cudaError_t e2 = fn();
  cudaGraph_t out = g;
  e = cudaStreamEndCapture(cs, &out);
  return e2 != cudaSuccess ? e2 : e;
}

#define GB_LTRY(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) return e_; } while (0)

// add a conditional node (WHILE: size 1, SWITCH: size k) after the capture's
// current dependencies; returns its body graphs
static cudaError_t add_conditional(cudaStream_t s, cudaGraphConditionalHandle h,
                                   cudaGraphConditionalNodeType type, unsigned size,
                                   cudaGraph_t* bodies) {
  cudaStreamCaptureStatus status;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  GB_LTRY(cudaStreamGetCaptureInfo(s, &status, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = type;
  p.conditional.size = size;
  cudaGraphNode_t node;
  GB_LTRY(cudaGraphAddNode(&node, g, deps, nd, &p));
  for (unsigned i = 0; i < size; ++i) bodies[i] = p.conditional.phGraph_out[i];
  return cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
}

static cudaGraph_t capturing_graph(cudaStream_t s) {
  cudaStreamCaptureStatus status;
  cudaGraph_t g = nullptr;
  cudaStreamGetCaptureInfo(s, &status, nullptr, &g, nullptr, nullptr);
  return g;
}

static bool loop_same_csr(const gb_csr* a, const gb_csr* b) {
  if (!a || !b) return a == b;
  return a->gen != 0 && a->gen == b->gen && a->nrows == b->nrows && a->nnz == b->nnz &&
         a->offsets == b->offsets && a->indices == b->indices && a->values == b->values &&
         a->dtype == b->dtype && a->iso_i64 == b->iso_i64 && a->iso_f64 == b->iso_f64;
}

__global__ void copy_i32(int64_t n, const int* __restrict__ a, int* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// warp per frontier entry k < *count; a row longer than kLongPush edges is
// cut into kLongChunk-edge tasks (k, chunk) queued for push_long
constexpr int64_t kLongChunk = 512;
template <class Op>
__global__ void __launch_bounds__(256)
push_short(const unsigned long long* __restrict__ count, const int32_t* __restrict__ F,
           const int64_t* __restrict__ off, int32_t* __restrict__ longk,
           int32_t* __restrict__ longc, unsigned long long* __restrict__ nlong, Op op) {
  const int lane = threadIdx.x & 31;
  const int64_t K = (int64_t)*count;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = w0; k < K; k += nw) {
    const int32_t j = F[k];
    const int64_t lo = off[j], hi = off[j + 1];
    if (hi - lo > kLongPush) {
      const int64_t nc = (hi - lo + kLongChunk - 1) / kLongChunk;
      unsigned long long at = 0;
      if (lane == 0) at = atomicAdd(nlong, (unsigned long long)nc);
      at = __shfl_sync(GB_FULL, at, 0);
      for (int64_t c = lane; c < nc; c += 32) {
        longk[at + c] = (int32_t)k;
        longc[at + c] = (int32_t)c;
      }
      continue;
    }
    for (int64_t p = lo + lane; p < hi; p += 32) op(k, p);
  }
}

// warp per queued (entry, chunk) task of the long rows
template <class Op>
__global__ void __launch_bounds__(256)
push_long(const unsigned long long* __restrict__ nlong, const int32_t* __restrict__ longk,
          const int32_t* __restrict__ longc, const int32_t* __restrict__ F,
          const int64_t* __restrict__ off, Op op) {
  const int lane = threadIdx.x & 31;
  const int64_t L = (int64_t)*nlong;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = w0; t < L; t += nw) {
    const int64_t k = longk[t];
    const int32_t j = F[k];
    const int64_t lo = off[j] + (int64_t)longc[t] * kLongChunk;
    const int64_t hi = min(off[j + 1], lo + kLongChunk);
    for (int64_t p = lo + lane; p < hi; p += 32) op(k, p);
  }
}

// ---------------------------------------------------------------------------
// PageRank (algorithms.py:132-162)
// ---------------------------------------------------------------------------
struct PrState {
  // per call
  double alpha, tele, eps, ratio;
  int64_t max_iters;
  int64_t* log;   // [max_iters][3]
  double* errs;   // [max_iters]
  int32_t policy, pad_;
  // loop
  int64_t it, nz, iters;
  double e2;
  unsigned long long nzc;
};

__global__ void pr_init_g(int64_t n, const int64_t* __restrict__ out_off,
                          const PrState* __restrict__ st, double* __restrict__ inv,
                          double* __restrict__ rank, double* __restrict__ y,
                          double* __restrict__ spread) {
  const double alpha = st->alpha;
  const double r0 = 1.0 / (double)n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = out_off[i + 1] - out_off[i];
    const double sc = d > 0 ? alpha / (double)d : 0.0;  // algorithms.py:124-127
    inv[i] = sc;
    rank[i] = r0;
    y[i] = sc * r0;
    spread[i] = 0.0;
  }
}

__global__ void pr_start_g(PrState* st, int64_t n, int64_t nnz, cudaGraphConditionalHandle h) {
  st->it = 0;
  st->nz = n;
  st->iters = 0;
  st->e2 = 0.0;
  st->nzc = 0;
  if (st->max_iters > 0) log_decision(st->log, 0, nnz, n, n, st->ratio, st->policy);
  cudaGraphSetConditional(h, st->max_iters > 0 ? 1u : 0u);
}

__global__ void __launch_bounds__(256)
pr_epilogue_g(int64_t n, PrState* st, const double* __restrict__ inv, double* __restrict__ spread,
              double* __restrict__ rk0, double* __restrict__ rk1, double* __restrict__ y) {
  const bool odd = st->it & 1;
  pr_epilogue_body(n, st->tele, inv, spread, odd ? rk1 : rk0, odd ? rk0 : rk1, y, &st->e2,
                   &st->nzc);
}

__global__ void pr_step_g(PrState* st, int64_t n, int64_t nnz, cudaGraphConditionalHandle h) {
  const double err = sqrt(st->e2);
  const int64_t it = st->it;
  st->errs[it] = err;
  st->nz = (int64_t)st->nzc;
  st->it = it + 1;
  st->iters = it + 1;
  const bool cont = !(err <= st->eps) && it + 1 < st->max_iters;  // algorithms.py:160
  st->e2 = 0.0;
  st->nzc = 0;
  if (cont) log_decision(st->log, it + 1, nnz, n, st->nz, st->ratio, st->policy);
  cudaGraphSetConditional(h, cont ? 1u : 0u);
}

struct PrGraph {
  gb_csr pull{};
  const int64_t* out_off = nullptr;
  void* mem = nullptr;
  double *inv, *y, *spread, *rk[2];
  PrState* st;
  RowTilesPlan plan;
  cudaGraphExec_t exec = nullptr;
};

static void pr_graph_free(void* p) {
  auto* g = static_cast<PrGraph*>(p);
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->mem) cudaFree(g->mem);
  delete g;
}

static cudaError_t pr_graph_build(gb_ctx* ctx, PrGraph* G) {
  const int64_t n = G->pull.nrows, nnz = G->pull.nnz;
  cudaStream_t cs[2];
  for (auto& x : cs) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  cudaGraph_t top;
  cudaError_t err = cudaGraphCreate(&top, 0);
  if (err == cudaSuccess) err = loop_capture_into(top, cs[0], [&]() -> cudaError_t {
    cudaStream_t s = cs[0];
    pr_init_g<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, G->out_off, G->st, G->inv, G->rk[0], G->y,
                                                    G->spread);
    cudaGraphConditionalHandle h;
    GB_LTRY(cudaGraphConditionalHandleCreate(&h, capturing_graph(s), 0, cudaGraphCondAssignDefault));
    pr_start_g<<<1, 1, 0, s>>>(G->st, n, nnz, h);
    GB_LTRY(cudaGetLastError());
    cudaGraph_t body;
    GB_LTRY(add_conditional(s, h, cudaGraphCondTypeWhile, 1, &body));
    return loop_capture_into(body, cs[1], [&]() -> cudaError_t {
      if (G->plan.R)
        pr_spmv<<<resident_grid(ctx, pr_spmv, 256), 256, 0, cs[1]>>>(
            G->plan.R, G->plan.nz_rows, G->plan.nz_off, G->pull.indices, G->plan.tile_first, G->y,
            G->spread);
      pr_epilogue_g<<<grid_for(ctx, n, 256, 8), 256, 0, cs[1]>>>(n, G->st, G->inv, G->spread,
                                                                 G->rk[0], G->rk[1], G->y);
      pr_step_g<<<1, 1, 0, cs[1]>>>(G->st, n, nnz, h);
      return cudaGetLastError();
    });
  });
  if (err == cudaSuccess) err = cudaGraphInstantiate(&G->exec, top, 0);
  cudaGraphDestroy(top);
  for (auto& x : cs) cudaStreamDestroy(x);
  return err;
}

static gb_status pagerank_graph(gb_ctx* ctx, const gb_csr* pull, const int64_t* out_offsets,
                                double alpha, double eps, int64_t max_iters, double ratio,
                                int32_t policy, double* ranks_out, int32_t* log_dir,
                                int64_t* log_nvals, int64_t* log_est, double* err_out,
                                int64_t* iters_out) {
  const int64_t n = pull->nrows;
  void** slot = ctx_slot(ctx, SLOT_PR_GRAPH, pr_graph_free);
  PrGraph* G = static_cast<PrGraph*>(*slot);
  cudaStream_t s = stream_of(ctx);
  if (G && !(loop_same_csr(&G->pull, pull) && G->out_off == out_offsets)) {
    cudaStreamSynchronize(s);
    pr_graph_free(G);
    *slot = G = nullptr;
  }
  if (!G) {
    G = new PrGraph();
    G->pull = *pull;
    G->out_off = out_offsets;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += (b + 255) / 256 * 256; return o; };
    const size_t o_v = take(5 * 8 * (size_t)n), o_st = take(sizeof(PrState));
    const size_t o_r = take(4 * (size_t)n), o_o = take(8 * (size_t)(n + 1));
    const size_t o_t = take(4 * (size_t)(pull->nnz / kRowTile + 2));
    if (cudaMalloc(&G->mem, off) != cudaSuccess) {
      cudaGetLastError();
      delete G;
      return GB_ERR_UNSUPPORTED;
    }
    char* m = static_cast<char*>(G->mem);
    double* v = (double*)(m + o_v);
    G->inv = v;
    G->y = v + n;
    G->spread = v + 2 * n;
    G->rk[0] = v + 3 * n;
    G->rk[1] = v + 4 * n;
    G->st = (PrState*)(m + o_st);
    G->plan.nz_rows = (int32_t*)(m + o_r);
    G->plan.nz_off = (int64_t*)(m + o_o);
    G->plan.tile_first = (int32_t*)(m + o_t);
    Arena ar(ctx);
    gb_status st = row_tiles_plan(ctx, ar, n, pull->offsets, pull->nnz, &G->plan);
    cudaError_t e = st == GB_OK ? pr_graph_build(ctx, G) : cudaSuccess;
    if (st != GB_OK || e != cudaSuccess) {
      cudaGetLastError();
      pr_graph_free(G);
      return st != GB_OK ? st : set_error(ctx, GB_ERR_CUDA, "pagerank graph: %s", cudaGetErrorString(e));
    }
    *slot = G;
  }
  Arena ar(ctx);
  const int64_t cap = max_iters > 0 ? max_iters : 1;
  int64_t* dlog = ar.alloc<int64_t>(3 * cap + 1);
  double* derr = ar.alloc<double>(cap);
  GB_ARENA_CHECK(ctx, ar);
  PrState h{};
  h.alpha = alpha;
  h.tele = (1.0 - alpha) / (double)n;
  h.eps = eps;
  h.ratio = ratio;
  h.max_iters = max_iters;
  h.log = dlog;
  h.errs = derr;
  h.policy = policy;
  GB_CUDA(ctx, cudaMemcpyAsync(G->st, &h, offsetof(PrState, it), cudaMemcpyHostToDevice, s));
  GB_CUDA(ctx, cudaGraphLaunch(G->exec, s));
  count_launch(ctx, 3);  // init, start + the body kernels are booked below
  int64_t iters = 0;
  GB_CUDA(ctx, cudaMemcpyAsync(&iters, &G->st->iters, 8, cudaMemcpyDeviceToHost, s));
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  if (iters > 0) {
    std::vector<int64_t> lg(3 * iters);
    GB_CUDA(ctx, cudaMemcpyAsync(lg.data(), dlog, 8 * 3 * iters, cudaMemcpyDeviceToHost, s));
    if (err_out) GB_CUDA(ctx, cudaMemcpyAsync(err_out, derr, 8 * iters, cudaMemcpyDeviceToHost, s));
    GB_CUDA(ctx, cudaStreamSynchronize(s));
    for (int64_t i = 0; i < iters; ++i) {
      log_dir[i] = (int32_t)lg[3 * i];
      log_nvals[i] = lg[3 * i + 1];
      log_est[i] = lg[3 * i + 2];
    }
  }
  count_launch(ctx, (int)(3 * iters));
  // iteration i reads rk[i & 1] and writes the other: the result is rk[iters & 1]
  GB_CUDA(ctx, cudaMemcpyAsync(ranks_out, G->rk[iters & 1], 8 * (size_t)n, cudaMemcpyDeviceToDevice, s));
  *iters_out = iters;
  return GB_OK;
}

// ---------------------------------------------------------------------------
// Connected components, FastSV (algorithms.py:165-203)
// ---------------------------------------------------------------------------
struct CcState {
  double ratio;
  double live_share;  // pull with the live bitmap below this share of live grandparents
  double push_share;  // below this share a pull runs as the transposed push
  int32_t has_cols, pad_;
  int64_t max_iters;
  int64_t* log;
  int32_t policy, sparsify;
  double exit_share;  // a pull takes cc_pull_exit above this share of grandparents at the bound
  double exit_rows;   // ... or when at most this share of the rows is above it
  int64_t nz_rows;    // non-empty rows of the matrix
  int32_t has_bins, pad4_;
  // loop
  int64_t it, live, iters;
  unsigned long long cnt[3];  // changed, live, listed
  unsigned long long nlow[2];  // cc_count_low: grandparents at the bound, rows above it
  unsigned long long nlong;
  int64_t npush;  // iterations that ran the push branch (launch accounting)
  int32_t low;    // smallest live grandparent (cc_pull_exit's bound)
  int32_t pad2_;
};

struct CcPushOp {
  const int32_t* idx;
  const int32_t* F;
  const int* gp;
  int* hook;
  __device__ __forceinline__ void operator()(int64_t k, int64_t p) const {
    const int32_t i = __ldg(idx + p);
    const int g = gp[F[k]];
    if (g < hook[i]) atomicMin(hook + i, g);
  }
};

__global__ void cc_start_g(CcState* st, int64_t n, int64_t nnz, cudaGraphConditionalHandle h_loop,
                           cudaGraphConditionalHandle h_dir) {
  st->it = 0;
  st->live = n;
  st->iters = 0;
  st->nlow[0] = st->nlow[1] = 0;
  st->cnt[0] = st->cnt[1] = st->cnt[2] = 0;
  st->nlong = 0;
  st->npush = 0;
  st->low = 0;  // a valid bound until the first shortcut pass sets it
  const bool run = st->max_iters > 0;
  unsigned dir = 0;
  // branch 3: the first pull (grandparents are the identity)
  if (run) dir = log_decision(st->log, 0, nnz, n, n, st->ratio, st->policy) == GB_DIR_PULL ? 3 : 1;
  st->npush = dir == 1;
  cudaGraphSetConditional(h_loop, run ? 1u : 0u);
  cudaGraphSetConditional(h_dir, dir);
}

__global__ void cc_shortcut_g(int64_t n, const int* __restrict__ parent, int* __restrict__ gp,
                              int* __restrict__ gpp, CcState* st, uint32_t* __restrict__ livebm) {
  // sparsify read from the state: one graph serves both settings
  cc_shortcut_body(n, parent, gp, gpp, st->sparsify, &st->cnt[0], &st->cnt[1], livebm, &st->low);
}

__global__ void cc_step_g(CcState* st, int64_t n, int64_t nnz, cudaGraphConditionalHandle h_loop,
                          cudaGraphConditionalHandle h_dir) {
  const int64_t it = st->it;
  const unsigned long long changed = st->cnt[0];
  st->it = it + 1;
  st->iters = it + 1;
  bool cont = changed != 0 && it + 1 < st->max_iters;  // algorithms.py:196-197
  if (changed != 0) st->live = (int64_t)st->cnt[1];
  st->cnt[0] = st->cnt[1] = st->cnt[2] = 0;
  st->nlong = 0;
  const unsigned long long nlow = st->nlow[0];
  const int64_t nup = st->nz_rows - (int64_t)st->nlow[1];  // non-empty rows above the bound
  st->nlow[0] = st->nlow[1] = 0;
  unsigned dir = 5;  // no branch
  if (cont) {
    // branch 0: pull over row tiles, 1: push, 2: pull probing the live
    // bitmap first, 4: bounded pull over the row bins (enough grandparents
    // sit at the bound that most rows stop early)
    const int32_t d = log_decision(st->log, it + 1, nnz, n, st->live, st->ratio, st->policy);
    const double live = (double)st->live;
    dir = d != GB_DIR_PULL || (st->has_cols && live < st->push_share * (double)n)
              ? 1u
              : (live < st->live_share * (double)n ? 2u : 0u);
    // a pull the rule chose takes the bounded kernel (4) when most rows meet
    // the bound early or are skipped outright -- ahead of the live-count
    // variants: at R-MAT s24 iteration 3 (12 % live, so far the transposed
    // push) only the rows outside the giant component are left
    if (d == GB_DIR_PULL && st->has_bins &&
        ((double)nlow >= st->exit_share * (double)n || (double)nup <= st->exit_rows * (double)n))
      dir = 4u;
    st->npush += dir == 1;
  }
  cudaGraphSetConditional(h_loop, cont ? 1u : 0u);
  cudaGraphSetConditional(h_dir, dir);
}

struct CcGraph {
  gb_csr rows{}, cols{};
  bool has_cols = false;
  void* mem = nullptr;
  int *P, *mn, *gp, *gpp, *pp, *hook;
  bool first_min = false;  // every row's first stored column is its smallest (format check)
  int32_t *F, *longk, *longc;
  uint32_t* livebm;  // live grandparents (written by the shortcut pass)
  CcState* st;
  RowTilesPlan plan;
  gb_bin_plan bins{};      // row bins of `rows` for cc_pull_exit
  void* binmem = nullptr;  // their storage (null: full pulls run cc_pull)
  cudaGraphExec_t exec = nullptr;
};

static void cc_graph_free(void* p) {
  auto* g = static_cast<CcGraph*>(p);
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->mem) cudaFree(g->mem);
  if (g->binmem) cudaFree(g->binmem);
  delete g;
}

static cudaError_t cc_graph_build(gb_ctx* ctx, CcGraph* G) {
  const int64_t n = G->rows.nrows, nnz = G->rows.nnz;
  const int vec_grid = grid_for(ctx, n, 256, 8);
  cudaStream_t cs[3];
  for (auto& x : cs) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  cudaGraph_t top;
  cudaError_t err = cudaGraphCreate(&top, 0);
  if (err == cudaSuccess) err = loop_capture_into(top, cs[0], [&]() -> cudaError_t {
    cudaStream_t s = cs[0];
    cc_init<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, G->P, G->mn, G->gp, G->gpp);
    cudaGraphConditionalHandle h_loop, h_dir;
    cudaGraph_t g = capturing_graph(s);
    GB_LTRY(cudaGraphConditionalHandleCreate(&h_loop, g, 0, cudaGraphCondAssignDefault));
    GB_LTRY(cudaGraphConditionalHandleCreate(&h_dir, g, 0, cudaGraphCondAssignDefault));
    cc_start_g<<<1, 1, 0, s>>>(G->st, n, nnz, h_loop, h_dir);
    GB_LTRY(cudaGetLastError());
    cudaGraph_t body;
    GB_LTRY(add_conditional(s, h_loop, cudaGraphCondTypeWhile, 1, &body));
    return loop_capture_into(body, cs[1], [&]() -> cudaError_t {
      cudaStream_t b = cs[1];
      copy_i32<<<vec_grid, 256, 0, b>>>(n, G->P, G->pp);
      fill_i32<<<vec_grid, 256, 0, b>>>(n, kImax32, G->hook);
      cudaGraph_t br[5];
      GB_LTRY(add_conditional(b, h_dir, cudaGraphCondTypeSwitch, 5, br));
      GB_LTRY(loop_capture_into(br[3], cs[2], [&]() -> cudaError_t {
        // first pull (grandparents are the identity): each row's smallest
        // column id -- its first entry when the rows start at their minimum
        if (G->first_min)
          cc_hook_first<<<vec_grid, 256, 0, cs[2]>>>(n, G->rows.offsets, G->rows.indices, G->hook);
        else if (G->plan.R)
          cc_pull_first<<<resident_grid(ctx, cc_pull_first, 256), 256, 0, cs[2]>>>(
              G->plan.R, G->plan.nz_rows, G->plan.nz_off, G->rows.indices, G->plan.tile_first,
              G->hook);
        return cudaGetLastError();
      }));
      GB_LTRY(loop_capture_into(br[0], cs[2], [&]() -> cudaError_t {
        // pull: mxv walks rows of A (kernels.py:313-316)
        if (G->plan.R)
          cc_pull<<<resident_grid(ctx, cc_pull, 256), 256, 0, cs[2]>>>(
              G->plan.R, G->plan.nz_rows, G->plan.nz_off, G->rows.indices, G->plan.tile_first,
              G->gp, G->hook);
        return cudaGetLastError();
      }));
      GB_LTRY(loop_capture_into(br[4], cs[2], [&]() -> cudaError_t {
        if (G->binmem)
          cc_pull_exit_launch(ctx, cs[2], G->bins, &G->rows, G->gp, G->mn, &G->st->low, G->hook);
        return cudaGetLastError();
      }));
      GB_LTRY(loop_capture_into(br[2], cs[2], [&]() -> cudaError_t {
        if (G->plan.R)
          cc_pull_live<<<resident_grid(ctx, cc_pull_live, 256), 256, 0, cs[2]>>>(
              G->plan.R, G->plan.nz_rows, G->plan.nz_off, G->rows.indices, G->plan.tile_first,
              G->gp, G->livebm, G->hook);
        return cudaGetLastError();
      }));
      GB_LTRY(loop_capture_into(br[1], cs[2], [&]() -> cudaError_t {
        // push: columns of A from the live grandparents, listed on the device
        if (!G->has_cols) return cudaSuccess;
        cc_list<<<vec_grid, 256, 0, cs[2]>>>(n, G->gp, G->F, &G->st->cnt[2]);
        const CcPushOp op{G->cols.indices, G->F, G->gp, G->hook};
        push_short<CcPushOp><<<grid_for(ctx, n * 32, 256, 8), 256, 0, cs[2]>>>(
            &G->st->cnt[2], G->F, G->cols.offsets, G->longk, G->longc, &G->st->nlong, op);
        push_long<CcPushOp><<<grid_for(ctx, G->cols.nnz / 16 + 32, 256, 8), 256, 0, cs[2]>>>(
            &G->st->nlong, G->longk, G->longc, G->F, G->cols.offsets, op);
        return cudaGetLastError();
      }));
      cc_hook<<<vec_grid, 256, 0, b>>>(n, G->hook, G->mn, G->pp, G->P, &G->st->low);
      cc_shortcut_g<<<vec_grid, 256, 0, b>>>(n, G->P, G->gp, G->gpp, G->st, G->livebm);
      if (G->binmem)
        cc_count_low<<<vec_grid, 256, 0, b>>>(n, G->gp, G->mn, G->plan.R, G->plan.nz_rows,
                                              &G->st->low, &G->st->cnt[1], cc_push_share(),
                                              G->st->nlow);
      cc_step_g<<<1, 1, 0, b>>>(G->st, n, nnz, h_loop, h_dir);
      return cudaGetLastError();
    });
  });
  if (err == cudaSuccess) err = cudaGraphInstantiate(&G->exec, top, 0);
  cudaGraphDestroy(top);
  for (auto& x : cs) cudaStreamDestroy(x);
  return err;
}

static gb_status cc_graph(gb_ctx* ctx, const gb_csr* rows, const gb_csr* cols, int64_t max_iters,
                          double ratio, int32_t policy, int32_t sparsify, int64_t* parent,
                          int32_t* log_dir, int64_t* log_nvals, int64_t* log_est,
                          int64_t* iters_out) {
  const int64_t n = rows->nrows;
  void** slot = ctx_slot(ctx, SLOT_CC_GRAPH, cc_graph_free);
  CcGraph* G = static_cast<CcGraph*>(*slot);
  cudaStream_t s = stream_of(ctx);
  if (G && !(loop_same_csr(&G->rows, rows) && G->has_cols == (cols != nullptr) &&
             (!cols || loop_same_csr(&G->cols, cols)))) {
    cudaStreamSynchronize(s);
    cc_graph_free(G);
    *slot = G = nullptr;
  }
  if (!G) {
    G = new CcGraph();
    G->rows = *rows;
    G->has_cols = cols != nullptr;
    if (cols) G->cols = *cols;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += (b + 255) / 256 * 256; return o; };
    const size_t o_v = take(7 * 4 * (size_t)n), o_st = take(sizeof(CcState));
    const size_t o_lb = take(4 * (size_t)((n + 31) / 32 + 1));
    const size_t ntask = (size_t)n + (size_t)(rows->nnz / kLongChunk) + 1;
    const size_t o_lk = take(4 * ntask), o_lc = take(4 * ntask);
    const size_t o_r = take(4 * (size_t)n), o_o = take(8 * (size_t)(n + 1));
    const size_t o_t = take(4 * (size_t)(rows->nnz / kRowTile + 2));
    if (cudaMalloc(&G->mem, off) != cudaSuccess) {
      cudaGetLastError();
      delete G;
      return GB_ERR_UNSUPPORTED;
    }
    char* m = static_cast<char*>(G->mem);
    int* v = (int*)(m + o_v);
    G->P = v;
    G->mn = v + n;
    G->gp = v + 2 * n;
    G->gpp = v + 3 * n;
    G->pp = v + 4 * n;
    G->hook = v + 5 * n;
    G->F = v + 6 * n;
    G->longk = (int32_t*)(m + o_lk);
    G->longc = (int32_t*)(m + o_lc);
    G->livebm = (uint32_t*)(m + o_lb);
    G->st = (CcState*)(m + o_st);
    G->plan.nz_rows = (int32_t*)(m + o_r);
    G->plan.nz_off = (int64_t*)(m + o_o);
    G->plan.tile_first = (int32_t*)(m + o_t);
    Arena ar(ctx);
    gb_status st = row_tiles_plan(ctx, ar, n, rows->offsets, rows->nnz, &G->plan);
    if (st == GB_OK) st = cc_rows_start_at_min(ctx, rows, G->plan, &G->first_min);
    if (st == GB_OK) st = pull_bins_build(ctx, rows, &G->bins, &G->binmem);
    cudaError_t e = st == GB_OK ? cc_graph_build(ctx, G) : cudaSuccess;
    if (st != GB_OK || e != cudaSuccess) {
      cudaGetLastError();
      cc_graph_free(G);
      return st != GB_OK ? st : set_error(ctx, GB_ERR_CUDA, "cc graph: %s", cudaGetErrorString(e));
    }
    *slot = G;
  }
  Arena ar(ctx);
  const int64_t cap = max_iters > 0 ? max_iters : 1;
  int64_t* dlog = ar.alloc<int64_t>(3 * cap + 1);
  GB_ARENA_CHECK(ctx, ar);
  CcState h{};
  h.ratio = ratio;
  h.max_iters = max_iters;
  h.log = dlog;
  h.policy = policy;
  h.sparsify = sparsify;
  h.live_share = cc_live_share();
  h.push_share = cc_push_share();
  h.exit_share = cc_exit_share();
  h.exit_rows = cc_exit_rows();
  h.nz_rows = G->plan.R;
  h.has_bins = G->binmem != nullptr;
  h.has_cols = cols != nullptr;
  GB_CUDA(ctx, cudaMemcpyAsync(G->st, &h, offsetof(CcState, it), cudaMemcpyHostToDevice, s));
  GB_CUDA(ctx, cudaGraphLaunch(G->exec, s));
  widen_i32<<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(n, G->P, reinterpret_cast<long long*>(parent));
  GB_LAUNCH_CHECK(ctx);
  int64_t iters = 0, npush = 0;
  GB_CUDA(ctx, cudaMemcpyAsync(&iters, &G->st->iters, 8, cudaMemcpyDeviceToHost, s));
  GB_CUDA(ctx, cudaMemcpyAsync(&npush, &G->st->npush, 8, cudaMemcpyDeviceToHost, s));
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  if (iters > 0) {
    std::vector<int64_t> lg(3 * iters);
    GB_CUDA(ctx, cudaMemcpyAsync(lg.data(), dlog, 8 * 3 * iters, cudaMemcpyDeviceToHost, s));
    GB_CUDA(ctx, cudaStreamSynchronize(s));
    for (int64_t i = 0; i < iters; ++i) {
      log_dir[i] = (int32_t)lg[3 * i];
      log_nvals[i] = lg[3 * i + 1];
      log_est[i] = lg[3 * i + 2];
    }
  }
  // per iteration: copy, fill, the branch (1 kernel; push 3), hook, shortcut,
  // (the bound count,) step
  count_launch(ctx, (int)(3 + (G->binmem ? 7 : 6) * iters + 2 * npush));
  *iters_out = iters;
  return GB_OK;
}

// ---------------------------------------------------------------------------
// SSSP (algorithms.py:80-119)
// ---------------------------------------------------------------------------
struct SsspState {
  double ratio;
  int64_t max_iters, source;
  int64_t* log;
  double* dist;
  int32_t policy, has_pull;
  double pull_share;  // a push level relaxing more than this share of nnz runs as the pull
  double wmin;        // lower bound on the weights (sssp_pull_exit)
  double exit_share;  // a pull takes sssp_pull_exit above this settled share of nnz
  int32_t has_bins, pad3_;
  // loop
  int64_t it, K, reached, succ_last, iters;
  long long fmin;     // bits of the smallest frontier distance (finalize)
  unsigned long long settled;  // in-edges of settled rows at the last pull (apply)
  unsigned long long cnt[2];  // new frontier, newly reached
  unsigned long long nlong;
  unsigned long long sumdeg;  // out-degrees of the frontier (finalize)
  int64_t npull;              // levels run by the pull branch (launch accounting)
};

// A push level whose frontier's out-degrees exceed this share of the stored
// edges runs as the pull (GB_SSSP_PULL_SHARE; s20: the level after the
// source's pushes 64,602 vertices with 22 M out-edges, 70 % of nnz)
static double sssp_pull_share() {
  static double v = -1.0;
  if (v < 0) {
    const char* e = getenv("GB_SSSP_PULL_SHARE");
    v = e ? atof(e) : 0.3;
  }
  return v;
}

// A pull takes the bounded row-bin kernel when the previous pull left at
// least this share of the stored edges in settled rows (GB_SSSP_EXIT_SHARE).
static double sssp_exit_share() {
  static double v = -1.0;
  if (v < 0) {
    const char* e = getenv("GB_SSSP_EXIT_SHARE");
    v = pull_exit_mode() == 2 ? 0.0 : (e ? atof(e) : 0.3);
  }
  return v;
}

struct SsspPushOp {
  const int32_t* idx;
  const void* vals;
  int dtype;
  double iso;
  const double* Fv;
  double* const* dist;
  uint32_t* changed;
  unsigned long long* reached;
  __device__ __forceinline__ void operator()(int64_t k, int64_t p) const {
    const int32_t v = __ldg(idx + p);
    const double nd = ld_weight(vals, dtype, iso, p) + Fv[k];  // mult(A value, u value)
    if (relax(*dist, v, nd, reached)) atomicOr(changed + (v >> 5), 1u << (v & 31));
  }
};

__global__ void sssp_init_g(int64_t n, const SsspState* __restrict__ st, double* __restrict__ fvd,
                            int32_t* __restrict__ F, double* __restrict__ Fv,
                            long long* __restrict__ cand, uint32_t* __restrict__ changed) {
  double* dist = st->dist;
  const int64_t source = st->source;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    dist[i] = i == source ? 0.0 : INFINITY;
    fvd[i] = i == source ? 0.0 : INFINITY;  // the frontier's dense copy: the source
    cand[i] = kInfBits;
    if ((i & 31) == 0) changed[i >> 5] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    F[0] = (int32_t)source;
    Fv[0] = 0.0;
  }
}

// The logged decision is the reference rule's; a push whose frontier would
// relax more than pull_share of all stored edges runs as the pull -- the same
// min over the same candidates w + d(u), so the same distances.
__device__ __forceinline__ unsigned sssp_branch(SsspState* st, int64_t n, int64_t nnz) {
  const int32_t dir = log_decision(st->log, st->it, nnz, n, st->K, st->ratio, st->policy);
  st->cnt[0] = 0;
  st->nlong = 0;
  const bool heavy = st->has_pull && (double)st->sumdeg > st->pull_share * (double)nnz;
  st->sumdeg = 0;
  unsigned b = dir == GB_DIR_PULL || (st->K > 0 && heavy) ? 0u : (st->K > 0 ? 1u : 3u);
  // branch 2: the bounded pull, when the last pull left most stored edges in
  // settled rows
  if (b == 0 && st->has_bins && (double)st->settled >= st->exit_share * (double)nnz) b = 2u;
  if (b == 0 || b == 2) st->settled = 0;  // this pull's apply totals it afresh
  st->npull += b == 0 || b == 2;
  return b;
}

__global__ void sssp_start_g(SsspState* st, int64_t n, int64_t nnz,
                             cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_dir) {
  st->it = 0;
  st->K = 1;
  st->fmin = 0;  // the first frontier is the source at distance 0
  st->reached = 1;
  st->succ_last = -1;
  st->iters = 0;
  st->cnt[0] = st->cnt[1] = 0;
  st->sumdeg = 0;
  st->npull = 0;
  st->settled = 0;
  const bool run = st->max_iters > 0;
  const unsigned dir = run ? sssp_branch(st, n, nnz) : 3u;
  cudaGraphSetConditional(h_loop, run ? 1u : 0u);
  cudaGraphSetConditional(h_dir, dir);
}

__global__ void reset_fvd_g(SsspState* __restrict__ st, const int32_t* __restrict__ F,
                            double* __restrict__ fvd) {
  const int64_t K = st->K;
  if (blockIdx.x == 0 && threadIdx.x == 0) st->fmin = kInfBits;  // recorded by the finalize
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K;
       i += (int64_t)gridDim.x * blockDim.x)
    fvd[F[i]] = INFINITY;
}

__global__ void __launch_bounds__(256)
sssp_pull_apply_g(int64_t n, long long* __restrict__ cand, SsspState* st,
                  uint32_t* __restrict__ changed, const int64_t* __restrict__ off) {
  // the settled share is totalled only when a bounded pull is available
  // (sssp_branch zeroed it when it chose this pull)
  sssp_apply_body(n, cand, st->dist, changed, &st->cnt[1], off,
                  __longlong_as_double(st->fmin) + st->wmin, st->has_bins ? &st->settled : nullptr);
}

__global__ void sssp_finalize_g(int64_t n, uint32_t* __restrict__ changed, SsspState* st,
                                int32_t* __restrict__ F, double* __restrict__ Fv,
                                double* __restrict__ fvd, const int64_t* __restrict__ off) {
  sssp_finalize_body(n, changed, st->dist, F, Fv, fvd, &st->cnt[0], off, &st->sumdeg, &st->fmin);
}

__global__ void sssp_step_g(SsspState* st, int64_t n, int64_t nnz,
                            cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_dir) {
  const int64_t it = st->it;
  const int64_t K = (int64_t)st->cnt[0];
  const int64_t reached = st->reached + (int64_t)st->cnt[1];
  st->cnt[1] = 0;
  st->K = K;
  st->reached = reached;
  st->it = it + 1;
  st->iters = it + 1;
  // algorithms.py:114-118: count of finite distances stable and no frontier
  const bool done = reached == st->succ_last && K == 0;
  st->succ_last = reached;
  const bool cont = !done && it + 1 < st->max_iters;
  const unsigned dir = cont ? sssp_branch(st, n, nnz) : 3u;
  cudaGraphSetConditional(h_loop, cont ? 1u : 0u);
  cudaGraphSetConditional(h_dir, dir);
}

struct SsspGraph {
  gb_csr push{}, pull{};
  bool has_pull = false;
  void* mem = nullptr;
  uint32_t* changed;
  int32_t *F, *longk, *longc;
  double *Fv, *fvd;
  long long* cand;
  SsspState* st;
  RowTilesPlan plan;
  gb_bin_plan bins{};      // row bins of `pull` for sssp_pull_exit (skewed graphs)
  void* binmem = nullptr;
  cudaGraphExec_t exec = nullptr;
};

static void sssp_graph_free(void* p) {
  auto* g = static_cast<SsspGraph*>(p);
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->mem) cudaFree(g->mem);
  if (g->binmem) cudaFree(g->binmem);
  delete g;
}

static cudaError_t sssp_graph_build(gb_ctx* ctx, SsspGraph* G) {
  const int64_t n = G->push.nrows, nnz = G->push.nnz;
  const int64_t W = (n + 31) / 32;
  cudaStream_t cs[3];
  for (auto& x : cs) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  cudaGraph_t top;
  cudaError_t err = cudaGraphCreate(&top, 0);
  if (err == cudaSuccess) err = loop_capture_into(top, cs[0], [&]() -> cudaError_t {
    cudaStream_t s = cs[0];
    sssp_init_g<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, G->st, G->fvd, G->F, G->Fv, G->cand,
                                                      G->changed);
    cudaGraphConditionalHandle h_loop, h_dir;
    cudaGraph_t g = capturing_graph(s);
    GB_LTRY(cudaGraphConditionalHandleCreate(&h_loop, g, 0, cudaGraphCondAssignDefault));
    GB_LTRY(cudaGraphConditionalHandleCreate(&h_dir, g, 0, cudaGraphCondAssignDefault));
    sssp_start_g<<<1, 1, 0, s>>>(G->st, n, nnz, h_loop, h_dir);
    GB_LTRY(cudaGetLastError());
    cudaGraph_t body;
    GB_LTRY(add_conditional(s, h_loop, cudaGraphCondTypeWhile, 1, &body));
    return loop_capture_into(body, cs[1], [&]() -> cudaError_t {
      cudaStream_t b = cs[1];
      // branches: 0 pull over row tiles, 1 push, 2 bounded pull over the
      // row bins (skewed graphs, most edges in settled rows), 3 (none) skip
      cudaGraph_t br[3];
      GB_LTRY(add_conditional(b, h_dir, cudaGraphCondTypeSwitch, 3, br));
      GB_LTRY(loop_capture_into(br[0], cs[2], [&]() -> cudaError_t {
        if (!G->has_pull) return cudaSuccess;
        if (G->plan.R)
          sssp_pull_tiles<<<resident_grid(ctx, sssp_pull_tiles, 256), 256, 0, cs[2]>>>(
              G->plan.R, G->plan.nz_rows, G->plan.nz_off, G->pull.indices, G->plan.tile_first,
              G->pull.values, G->pull.dtype, G->pull.iso_f64, G->fvd, G->cand);
        sssp_pull_apply_g<<<grid_for(ctx, n, 256), 256, 0, cs[2]>>>(n, G->cand, G->st, G->changed,
                                                                    G->pull.offsets);
        return cudaGetLastError();
      }));
      GB_LTRY(loop_capture_into(br[2], cs[2], [&]() -> cudaError_t {
        if (!G->has_pull || !G->binmem) return cudaSuccess;
        sssp_pull_exit<<<resident_grid(ctx, sssp_pull_exit, 256), 256, 0, cs[2]>>>(
            G->bins.n_long_tiles, G->bins.tile_row, G->bins.tile_beg, G->bins.tile_end,
            G->bins.n_mid, G->bins.mid_rows, G->bins.n_short, G->bins.short_rows,
            G->pull.offsets, G->pull.indices, G->pull.values, G->pull.dtype, G->pull.iso_f64,
            G->fvd, nullptr, &G->st->dist, &G->st->fmin, &G->st->wmin, G->cand);
        sssp_pull_apply_g<<<grid_for(ctx, n, 256), 256, 0, cs[2]>>>(n, G->cand, G->st, G->changed,
                                                                    G->pull.offsets);
        return cudaGetLastError();
      }));
      GB_LTRY(loop_capture_into(br[1], cs[2], [&]() -> cudaError_t {
        const SsspPushOp op{G->push.indices, G->push.values, G->push.dtype, G->push.iso_f64,
                            G->Fv, &G->st->dist, G->changed, &G->st->cnt[1]};
        // the frontier size K: the previous finalize's count, kept in the state
        push_short<SsspPushOp><<<grid_for(ctx, n * 32, 256, 8), 256, 0, cs[2]>>>(
            reinterpret_cast<const unsigned long long*>(&G->st->K), G->F, G->push.offsets,
            G->longk, G->longc, &G->st->nlong, op);
        push_long<SsspPushOp><<<grid_for(ctx, G->push.nnz / 16 + 32, 256, 8), 256, 0, cs[2]>>>(
            &G->st->nlong, G->longk, G->longc, G->F, G->push.offsets, op);
        return cudaGetLastError();
      }));
      reset_fvd_g<<<grid_for(ctx, n, 256), 256, 0, b>>>(G->st, G->F, G->fvd);
      sssp_finalize_g<<<grid_for(ctx, W, 256), 256, 0, b>>>(n, G->changed, G->st, G->F, G->Fv,
                                                            G->fvd, G->push.offsets);
      sssp_step_g<<<1, 1, 0, b>>>(G->st, n, nnz, h_loop, h_dir);
      return cudaGetLastError();
    });
  });
  if (err == cudaSuccess) err = cudaGraphInstantiate(&G->exec, top, 0);
  cudaGraphDestroy(top);
  for (auto& x : cs) cudaStreamDestroy(x);
  return err;
}

static gb_status sssp_graph(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull, int64_t source,
                            int64_t max_iters, double ratio, int32_t policy, double wmin,
                            double* dist,
                            int32_t* log_dir, int64_t* log_nvals, int64_t* log_est,
                            int64_t* iters_out) {
  const int64_t n = push->nrows;
  void** slot = ctx_slot(ctx, SLOT_SSSP_GRAPH, sssp_graph_free);
  SsspGraph* G = static_cast<SsspGraph*>(*slot);
  cudaStream_t s = stream_of(ctx);
  if (G && !(loop_same_csr(&G->push, push) && G->has_pull == (pull != nullptr) &&
             (!pull || loop_same_csr(&G->pull, pull)))) {
    cudaStreamSynchronize(s);
    sssp_graph_free(G);
    *slot = G = nullptr;
  }
  if (!G) {
    G = new SsspGraph();
    G->push = *push;
    G->has_pull = pull != nullptr;
    if (pull) G->pull = *pull;
    const int64_t W = (n + 31) / 32;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += (b + 255) / 256 * 256; return o; };
    const size_t ntask = (size_t)n + (size_t)(push->nnz / kLongChunk) + 1;
    const size_t o_c = take(4 * (size_t)W), o_F = take(4 * (size_t)n), o_L = take(4 * ntask);
    const size_t o_LC = take(4 * ntask);
    const size_t o_Fv = take(8 * (size_t)n), o_fvd = take(8 * (size_t)n);
    const size_t o_cand = take(8 * (size_t)n), o_st = take(sizeof(SsspState));
    const size_t o_r = pull ? take(4 * (size_t)n) : 0, o_o = pull ? take(8 * (size_t)(n + 1)) : 0;
    const size_t o_t = pull ? take(4 * (size_t)(pull->nnz / kRowTile + 2)) : 0;
    if (cudaMalloc(&G->mem, off) != cudaSuccess) {
      cudaGetLastError();
      delete G;
      return GB_ERR_UNSUPPORTED;
    }
    char* m = static_cast<char*>(G->mem);
    G->changed = (uint32_t*)(m + o_c);
    G->F = (int32_t*)(m + o_F);
    G->longk = (int32_t*)(m + o_L);
    G->longc = (int32_t*)(m + o_LC);
    G->Fv = (double*)(m + o_Fv);
    G->fvd = (double*)(m + o_fvd);
    G->cand = (long long*)(m + o_cand);
    G->st = (SsspState*)(m + o_st);
    gb_status st = GB_OK;
    if (pull) {
      G->plan.nz_rows = (int32_t*)(m + o_r);
      G->plan.nz_off = (int64_t*)(m + o_o);
      G->plan.tile_first = (int32_t*)(m + o_t);
      Arena ar(ctx);
      st = row_tiles_plan(ctx, ar, n, pull->offsets, pull->nnz, &G->plan);
      if (st == GB_OK) st = pull_bins_build(ctx, pull, &G->bins, &G->binmem);
    }
    cudaError_t e = st == GB_OK ? sssp_graph_build(ctx, G) : cudaSuccess;
    if (st != GB_OK || e != cudaSuccess) {
      cudaGetLastError();
      sssp_graph_free(G);
      return st != GB_OK ? st : set_error(ctx, GB_ERR_CUDA, "sssp graph: %s", cudaGetErrorString(e));
    }
    *slot = G;
  }
  Arena ar(ctx);
  const int64_t cap = max_iters > 0 ? max_iters : 1;
  int64_t* dlog = ar.alloc<int64_t>(3 * cap + 1);
  GB_ARENA_CHECK(ctx, ar);
  SsspState h{};
  h.ratio = ratio;
  h.max_iters = max_iters;
  h.source = source;
  h.log = dlog;
  h.dist = dist;
  h.policy = policy;
  h.has_pull = pull != nullptr;
  h.pull_share = sssp_pull_share();
  h.wmin = wmin;
  h.exit_share = sssp_exit_share();
  h.has_bins = G->binmem != nullptr;
  GB_CUDA(ctx, cudaMemcpyAsync(G->st, &h, offsetof(SsspState, it), cudaMemcpyHostToDevice, s));
  GB_CUDA(ctx, cudaGraphLaunch(G->exec, s));
  int64_t iters = 0;
  GB_CUDA(ctx, cudaMemcpyAsync(&iters, &G->st->iters, 8, cudaMemcpyDeviceToHost, s));
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  std::vector<int64_t> lg(3 * (iters > 0 ? iters : 1));
  if (iters > 0) {
    GB_CUDA(ctx, cudaMemcpyAsync(lg.data(), dlog, 8 * 3 * iters, cudaMemcpyDeviceToHost, s));
    GB_CUDA(ctx, cudaStreamSynchronize(s));
  }
  for (int64_t i = 0; i < iters; ++i) {
    log_dir[i] = (int32_t)lg[3 * i];
    log_nvals[i] = lg[3 * i + 1];
    log_est[i] = lg[3 * i + 2];
  }
  // a pull iteration the graph met without the column orientation: report it
  // the way the host loop does
  for (int64_t i = 0; i < iters; ++i)
    if (log_dir[i] == GB_DIR_PULL && !pull)
      return set_error(ctx, GB_ERR_FORMAT, "column-oriented storage missing");
  count_launch(ctx, (int)(2 + 5 * iters));
  *iters_out = iters;
  return GB_OK;
}

}  // namespace gb

using namespace gb;

extern "C" {

typedef void (*gb_iter_cb)(int64_t iteration, void* user);

int32_t gb_loop_engine(int32_t engine) {
  const int32_t prev = loop_engine();
  if (engine == kLoopGraph || engine == kLoopHost) g_loop_engine = engine;
  return prev;
}

gb_status gb_sssp(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull, int64_t source,
                  int64_t max_iters, double ratio, int32_t policy, double min_weight, double* dist,
                  int32_t* log_dir, int64_t* log_nvals, int64_t* log_est, int64_t* iters_out,
                  gb_iter_cb cb, void* user) {
  const int64_t n = push->nrows;
  if (source < 0 || source >= n) return set_error(ctx, GB_ERR_INDEX, "source out of range");
  // a lower bound on the weights (positive by contract): anything else -> 0
  const double wmin = min_weight > 0.0 && min_weight < INFINITY ? min_weight : 0.0;
  // device-resident loop unless a per-iteration host callback is requested
  // or the kernels are being timed one by one
  if (!cb && loop_engine() == kLoopGraph && !prof_enabled(ctx)) {
    const gb_status st = sssp_graph(ctx, push, pull, source, max_iters, ratio, policy, wmin, dist,
                                    log_dir, log_nvals, log_est, iters_out);
    if (st != GB_ERR_UNSUPPORTED) return st;
  }
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  uint32_t* changed = ar.alloc<uint32_t>(W);
  int32_t* F = ar.alloc<int32_t>(n);
  double* Fv = ar.alloc<double>(n);
  double* fvd = ar.alloc<double>(n);
  // [frontier, reached, out-degrees, in-edges of settled rows]
  unsigned long long* cnt = ar.alloc<unsigned long long>(4);
  long long* fmin = ar.alloc<long long>(1);                   // smallest frontier distance (bits)
  double* wmin_d = ar.alloc<double>(1);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(fmin, 0, sizeof(long long), s));  // the source, at 0
  GB_CUDA(ctx, cudaMemcpyAsync(wmin_d, &wmin, sizeof(double), cudaMemcpyHostToDevice, s));
  GB_CUDA(ctx, cudaMemsetAsync(changed, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(cnt, 0, 32, s));
  sssp_init<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, dist, fvd, source, F, Fv);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 3);
  // the frontier's dense copy starts with the source
  const double zero = 0.0;
  GB_CUDA(ctx, cudaMemcpyAsync(fvd + source, &zero, 8, cudaMemcpyHostToDevice, s));
  RowTilesPlan pull_plan;    // built on the first pull iteration
  long long* cand = nullptr;  // pull candidates (+inf bits between iterations)
  gb_bin_plan bins{};         // row bins of `pull` (skewed graphs), with the plan
  void* binmem = nullptr;

  int64_t K = 1, reached = 1, succ_last = -1, iters = 0, sumdeg = 0, settled = 0;
  const double push_iso = push->iso_f64, pull_iso = pull ? pull->iso_f64 : 0.0;
  for (int64_t it = 0; it < max_iters; ++it) {
    int64_t est = 0;
    const int32_t dir = gb_decide_direction(push->nnz, push->nrows, K, ratio, policy, &est);
    log_dir[it] = dir;
    log_nvals[it] = K;
    log_est[it] = est;
    iters = it + 1;
    GB_CUDA(ctx, cudaMemsetAsync(cnt, 0, 8, s));
    // a heavy push runs as the pull (same candidates, same minima)
    const bool heavy = pull && K > 0 && (double)sumdeg > sssp_pull_share() * (double)push->nnz;
    if (dir == GB_DIR_PULL || heavy) {
      if (!pull) return set_error(ctx, GB_ERR_FORMAT, "column-oriented storage missing");
      const int ps = prof_begin(ctx, PROF_SSSP, K);
      if (!pull_plan.nz_rows) {
        GB_TRY(row_tiles_plan(ctx, ar, n, pull->offsets, pull->nnz, &pull_plan));
        cand = ar.alloc<long long>(n);
        GB_ARENA_CHECK(ctx, ar);
        fill_i64<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, kInfBits, cand);
        GB_TRY(pull_bins_build(ctx, pull, &bins, &binmem, &ar));
      }
      // the bounded pull when the last pull left most edges in settled rows
      const bool bounded = binmem && (double)settled >= sssp_exit_share() * (double)pull->nnz;
      if (bounded)
        sssp_pull_exit<<<resident_grid(ctx, sssp_pull_exit, 256), 256, 0, s>>>(
            bins.n_long_tiles, bins.tile_row, bins.tile_beg, bins.tile_end, bins.n_mid,
            bins.mid_rows, bins.n_short, bins.short_rows, pull->offsets, pull->indices,
            pull->values, pull->dtype, pull_iso, fvd, dist, nullptr, fmin, wmin_d, cand);
      else if (pull_plan.R)
        sssp_pull_tiles<<<resident_grid(ctx, sssp_pull_tiles, 256), 256, 0, s>>>(
            pull_plan.R, pull_plan.nz_rows, pull_plan.nz_off, pull->indices, pull_plan.tile_first,
            pull->values, pull->dtype, pull_iso, fvd, cand);
      GB_CUDA(ctx, cudaMemsetAsync(cnt + 3, 0, 8, s));
      sssp_pull_apply<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, cand, dist, changed, cnt + 1,
                                                            pull->offsets, fmin, wmin_d,
                                                            binmem ? cnt + 3 : nullptr);
      prof_end(ctx, ps);
      count_launch(ctx, 2);
    } else if (K > 0) {
      LbsPlan plan;
      GB_TRY(lbs_prepare(ctx, ar, K, F, push->offsets, push->nnz, &plan));
      SsspPush f{push->indices, push->values, push->dtype, push_iso, Fv, dist, changed, cnt + 1};
      const int ps = prof_begin(ctx, PROF_SSSP, K);
      lbs_expand<SsspPush><<<plan.grid, kLbsThreads, 0, s>>>(K, plan.S, plan.rowstart,
                                                             plan.tile_first, f);
      prof_end(ctx, ps);
      count_launch(ctx, 5);
    }
    reset_fvd<<<grid_for(ctx, K > 0 ? K : 1, 256), 256, 0, s>>>(K, F, fvd, fmin);
    sssp_finalize<<<grid_for(ctx, W, 256), 256, 0, s>>>(n, changed, dist, F, Fv, fvd, cnt,
                                                         push->offsets, cnt + 2, fmin);
    GB_LAUNCH_CHECK(ctx);
    count_launch(ctx, 2);
    int64_t h[4];
    GB_TRY(read_i64(ctx, (const int64_t*)cnt, h, 4));
    K = h[0];
    reached += h[1];
    sumdeg = h[2];
    if (dir == GB_DIR_PULL || heavy) settled = h[3];
    GB_CUDA(ctx, cudaMemsetAsync(cnt + 1, 0, 16, s));
    if (cb) cb(it, user);
    // algorithms.py:114-118: count of finite distances stable and no frontier
    if (reached == succ_last && K == 0) break;
    succ_last = reached;
  }
  *iters_out = iters;
  return GB_OK;
}

gb_status gb_pagerank(gb_ctx* ctx, const gb_csr* pull, const int64_t* out_offsets, double alpha,
                      double eps, int64_t max_iters, double ratio, int32_t policy,
                      double* ranks_out, int32_t* log_dir, int64_t* log_nvals, int64_t* log_est,
                      double* err_out, int64_t* iters_out) {
  const int64_t n = pull->nrows;
  if (loop_engine() == kLoopGraph && !prof_enabled(ctx) && n > 0) {
    const gb_status st = pagerank_graph(ctx, pull, out_offsets, alpha, eps, max_iters, ratio,
                                        policy, ranks_out, log_dir, log_nvals, log_est, err_out,
                                        iters_out);
    if (st != GB_ERR_UNSUPPORTED) return st;
  }
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  double* inv = ar.alloc<double>(n);
  double* y = ar.alloc<double>(n);
  double* spread = ar.alloc<double>(n);
  double* rk[2] = {ar.alloc<double>(n), ranks_out};
  double* scal = ar.alloc<double>(2);
  GB_ARENA_CHECK(ctx, ar);
  RowTilesPlan plan;
  GB_TRY(row_tiles_plan(ctx, ar, n, pull->offsets, pull->nnz, &plan));
  pr_init<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, out_offsets, alpha, inv, rk[0], y, spread);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  const double tele = (1.0 - alpha) / (double)n;
  const int spmv_grid = resident_grid(ctx, pr_spmv, 256);
  int64_t nz = n, iters = 0;
  int cur = 0;
  for (int64_t it = 0; it < max_iters; ++it) {
    int64_t est = 0;
    const int32_t dir = gb_decide_direction(pull->nnz, pull->nrows, nz, ratio, policy, &est);
    log_dir[it] = dir;
    log_nvals[it] = nz;
    log_est[it] = est;
    iters = it + 1;
    GB_CUDA(ctx, cudaMemsetAsync(scal, 0, 16, s));
    const int ps = prof_begin(ctx, PROF_PR, pull->nnz);
    if (plan.R) pr_spmv<<<spmv_grid, 256, 0, s>>>(plan.R, plan.nz_rows, plan.nz_off, pull->indices,
                                                  plan.tile_first, y, spread);
    prof_end(ctx, ps);
    // the last iteration must land in ranks_out: pick buffers so it does
    double* prev = rk[cur];
    double* next = rk[cur ^ 1];
    pr_epilogue<<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(n, tele, inv, spread, prev, next, y,
                                                         scal, (unsigned long long*)(scal + 1));
    GB_LAUNCH_CHECK(ctx);
    count_launch(ctx, 3);
    int64_t h[2];
    GB_TRY(read_i64(ctx, (const int64_t*)scal, h, 2));
    double e2;
    memcpy(&e2, &h[0], 8);
    nz = h[1];
    const double err = sqrt(e2);
    if (err_out) err_out[it] = err;
    cur ^= 1;
    if (err <= eps) break;
  }
  if (rk[cur] != ranks_out)
    GB_CUDA(ctx, cudaMemcpyAsync(ranks_out, rk[cur], sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  if (iters == 0)
    GB_CUDA(ctx, cudaMemcpyAsync(ranks_out, rk[0], sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  *iters_out = iters;
  return GB_OK;
}

gb_status gb_cc(gb_ctx* ctx, const gb_csr* rows, const gb_csr* cols, int64_t max_iters,
                double ratio, int32_t policy, int32_t sparsify, int64_t* parent,
                int32_t* log_dir, int64_t* log_nvals, int64_t* log_est, int64_t* iters_out) {
  const int64_t n = rows->nrows;
  if (n >= kImax32) return set_error(ctx, GB_ERR_UNSUPPORTED, "cc needs n < 2^31 - 1");
  if (loop_engine() == kLoopGraph && !prof_enabled(ctx) && n > 0) {
    const gb_status st = cc_graph(ctx, rows, cols, max_iters, ratio, policy, sparsify, parent,
                                  log_dir, log_nvals, log_est, iters_out);
    if (st != GB_ERR_UNSUPPORTED) return st;
  }
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  int* P = ar.alloc<int>(n);
  int* mn = ar.alloc<int>(n);
  int* gp = ar.alloc<int>(n);
  int* gpp = ar.alloc<int>(n);
  int* pp = ar.alloc<int>(n);
  int* hook = ar.alloc<int>(n);
  uint32_t* livebm = ar.alloc<uint32_t>((n + 31) / 32 + 1);
  int32_t* F = ar.alloc<int32_t>(n);
  // [changed, live, listed, grandparents at the bound, rows above it]
  unsigned long long* cnt = ar.alloc<unsigned long long>(5);
  GB_ARENA_CHECK(ctx, ar);
  int* low = ar.alloc<int>(1);
  GB_ARENA_CHECK(ctx, ar);
  RowTilesPlan plan;
  GB_TRY(row_tiles_plan(ctx, ar, n, rows->offsets, rows->nnz, &plan));
  bool first_min = false;
  GB_TRY(cc_rows_start_at_min(ctx, rows, plan, &first_min));
  gb_bin_plan bins;
  void* binmem = nullptr;
  GB_TRY(pull_bins_build(ctx, rows, &bins, &binmem, &ar));
  GB_CUDA(ctx, cudaMemsetAsync(low, 0, sizeof(int), s));
  cc_init<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, P, mn, gp, gpp);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  const int pull_grid = resident_grid(ctx, cc_pull, 256);
  const int vec_grid = grid_for(ctx, n, 256, 8);
  int64_t live = n, iters = 0, nlow = 0, nup = n;
  for (int64_t it = 0; it < max_iters; ++it) {
    int64_t est = 0;
    const int32_t dir = gb_decide_direction(rows->nnz, rows->nrows, live, ratio, policy, &est);
    log_dir[it] = dir;
    log_nvals[it] = live;
    log_est[it] = est;
    iters = it + 1;
    GB_CUDA(ctx, cudaMemcpyAsync(pp, P, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
    fill_i32<<<vec_grid, 256, 0, s>>>(n, kImax32, hook);
    const int ps = prof_begin(ctx, PROF_CC, live);
    // a pull whose rows mostly meet the bound early or are skipped takes the
    // bounded kernel; otherwise a pull over few live grandparents runs as
    // the transposed push (same hooks)
    const bool bounded = dir == GB_DIR_PULL && it > 0 && binmem &&
                         ((double)nlow >= cc_exit_share() * (double)n ||
                          (double)nup <= cc_exit_rows() * (double)n);
    const bool as_push = !bounded && (dir != GB_DIR_PULL ||
                                      (it > 0 && cols && (double)live < cc_push_share() * (double)n));
    if (bounded) {
      cc_pull_exit_launch(ctx, s, bins, rows, gp, mn, low, hook);
      count_launch(ctx, 1);
    } else if (!as_push) {
      // mxv pull walks rows of A (kernels.py:313-316, row_view(False))
      if (it == 0 && first_min)  // grandparents are the identity: each row's first column
        cc_hook_first<<<vec_grid, 256, 0, s>>>(n, rows->offsets, rows->indices, hook);
      else if (plan.R && it == 0)  // ... or its streaming minimum
        cc_pull_first<<<resident_grid(ctx, cc_pull_first, 256), 256, 0, s>>>(
            plan.R, plan.nz_rows, plan.nz_off, rows->indices, plan.tile_first, hook);
      else if (plan.R && (double)live < cc_live_share() * (double)n)
        cc_pull_live<<<resident_grid(ctx, cc_pull_live, 256), 256, 0, s>>>(
            plan.R, plan.nz_rows, plan.nz_off, rows->indices, plan.tile_first, gp, livebm, hook);
      else if (plan.R) cc_pull<<<pull_grid, 256, 0, s>>>(plan.R, plan.nz_rows, plan.nz_off, rows->indices,
                                                    plan.tile_first, gp, hook);
      count_launch(ctx, 1);
    } else if (live > 0) {
      // push walks columns of A (rows of the CSC orientation) from the live
      // grandparents, listed on demand
      if (!cols) return set_error(ctx, GB_ERR_FORMAT, "column-oriented storage missing");
      GB_CUDA(ctx, cudaMemsetAsync(cnt + 2, 0, 8, s));
      cc_list<<<vec_grid, 256, 0, s>>>(n, gp, F, cnt + 2);
      LbsPlan lp;
      GB_TRY(lbs_prepare(ctx, ar, live, F, cols->offsets, cols->nnz, &lp));
      CcPush f{cols->indices, F, gp, hook};
      lbs_expand<CcPush><<<lp.grid, kLbsThreads, 0, s>>>(live, lp.S, lp.rowstart, lp.tile_first, f);
      count_launch(ctx, 7);
    }
    prof_end(ctx, ps);
    cc_hook<<<vec_grid, 256, 0, s>>>(n, hook, mn, pp, P, low);
    GB_CUDA(ctx, cudaMemsetAsync(cnt, 0, 16, s));
    cc_shortcut<<<vec_grid, 256, 0, s>>>(n, P, gp, gpp, sparsify, cnt, cnt + 1, livebm, low);
    if (binmem) {
      GB_CUDA(ctx, cudaMemsetAsync(cnt + 3, 0, 16, s));
      cc_count_low<<<vec_grid, 256, 0, s>>>(n, gp, mn, plan.R, plan.nz_rows, low, cnt + 1,
                                            cc_push_share(), cnt + 3);
      count_launch(ctx, 2);
    }
    GB_LAUNCH_CHECK(ctx);
    count_launch(ctx, 5);
    int64_t h[5];
    GB_TRY(read_i64(ctx, (const int64_t*)cnt, h, 5));
    if (h[0] == 0) break;  // algorithms.py:196-197
    live = h[1];
    nlow = binmem ? h[3] : 0;
    nup = binmem ? plan.R - h[4] : n;
  }
  widen_i32<<<vec_grid, 256, 0, s>>>(n, P, reinterpret_cast<long long*>(parent));
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  *iters_out = iters;
  return GB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// 1D-partitioned connected components (one rank's steps; the loop and the
// all-reduce MIN of the parent proposals live in distributed.py).  Label
// vectors are int32, global-sized and replicated; hook/mn are meaningful on
// the rank's own vertices [lo, hi) only.
// ---------------------------------------------------------------------------
namespace gb {

struct CcMinBlock {
  const int* __restrict__ gp;
  int* __restrict__ hook;  // rebased: local row r writes hook[lo + r]
  __device__ __forceinline__ int identity() const { return kImax32; }
  __device__ __forceinline__ int load(int64_t, int32_t col) const { return ld_gather(gp + col); }
  __device__ __forceinline__ int fold(int a, int x) const { return x < a ? x : a; }
  __device__ __forceinline__ void emit(int64_t row, int acc, bool whole) const {
    if (acc == kImax32) return;
    if (whole) hook[row] = acc;
    else atomicMin(hook + row, acc);
  }
};

__global__ void __launch_bounds__(256, GB_ROW_MINB)
cc_pull_block(int64_t R, const int32_t* __restrict__ nz_rows, const int64_t* __restrict__ nz_off,
              const int32_t* __restrict__ idx, const int32_t* __restrict__ tile_first,
              const int* __restrict__ gp, int* __restrict__ hook_rebased) {
  CcMinBlock red{gp, hook_rebased};
  row_tiles<int>(R, nz_rows, nz_off, idx, tile_first, red);
}

// owned k: mn[k] = min(mn[k], hook[k]); prop[k] min= mn[k]; prop[pp[k]] min= mn[k]
__global__ void cc_propose(int64_t lo, int64_t hi, const int* __restrict__ hook,
                           int* __restrict__ mn, const int* __restrict__ pp,
                           int* __restrict__ prop) {
  for (int64_t k = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < hi;
       k += (int64_t)gridDim.x * blockDim.x) {
    int m = mn[k];
    const int h = hook[k];
    if (h < m) { m = h; mn[k] = m; }
    if (m < *reinterpret_cast<volatile int*>(prop + k)) atomicMin(prop + k, m);
    const int t = pp[k];
    if (m < *reinterpret_cast<volatile int*>(prop + t)) atomicMin(prop + t, m);
  }
}

// parent = min(pp, all-reduced proposals)
__global__ void cc_merge(int64_t n, const int* __restrict__ pp, const int* __restrict__ prop,
                         int* __restrict__ parent) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    parent[k] = min(pp[k], prop[k]);
}

}  // namespace gb

extern "C" {

gb_status gb_cc_dist_init(gb_ctx* ctx, int64_t n, int32_t* parent, int32_t* mn, int32_t* gp,
                          int32_t* gpp) {
  if (n >= kImax32) return set_error(ctx, GB_ERR_UNSUPPORTED, "cc needs n < 2^31 - 1");
  cc_init<<<grid_for(ctx, n, 256, 8), 256, 0, stream_of(ctx)>>>(n, parent, mn, gp, gpp);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

// hooked values of the owned vertices (pull over the row block, or push over
// the column block from the live grandparents).  hook is reset to the
// sentinel first; pp <- parent (the iteration's parent_prev snapshot).
gb_status gb_cc_dist_hook(gb_ctx* ctx, int32_t pull, const gb_csr* rowblock,
                          const gb_csr* colblock, int64_t lo, int64_t hi, int64_t n,
                          const int32_t* gp, const int32_t* parent, int32_t* pp, int32_t* hook) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int vg = grid_for(ctx, n, 256, 8);
  GB_CUDA(ctx, cudaMemcpyAsync(pp, parent, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
  fill_i32<<<vg, 256, 0, s>>>(n, kImax32, hook);
  count_launch(ctx, 2);
  if (pull) {
    if (rowblock->nnz == 0 || hi <= lo) return GB_OK;
    RowTilesPlan plan;
    GB_TRY(row_tiles_plan(ctx, ar, hi - lo, rowblock->offsets, rowblock->nnz, &plan));
    if (plan.R)
      cc_pull_block<<<resident_grid(ctx, cc_pull_block, 256), 256, 0, s>>>(
          plan.R, plan.nz_rows, plan.nz_off, rowblock->indices, plan.tile_first, gp, hook + lo);
    count_launch(ctx, 1);
  } else {
    if (colblock->nnz == 0) return GB_OK;
    int32_t* F = ar.alloc<int32_t>(n);
    unsigned long long* cnt = ar.alloc<unsigned long long>(1);
    GB_ARENA_CHECK(ctx, ar);
    GB_CUDA(ctx, cudaMemsetAsync(cnt, 0, 8, s));
    cc_list<<<vg, 256, 0, s>>>(n, gp, F, cnt);
    int64_t K = 0;
    GB_TRY(read_i64(ctx, (const int64_t*)cnt, &K));
    if (K > 0) {
      LbsPlan lp;
      GB_TRY(lbs_prepare(ctx, ar, K, F, colblock->offsets, colblock->nnz, &lp));
      CcPush f{colblock->indices, F, gp, hook};
      lbs_expand<CcPush><<<lp.grid, kLbsThreads, 0, s>>>(K, lp.S, lp.rowstart, lp.tile_first, f);
      count_launch(ctx, 6);
    }
  }
  GB_LAUNCH_CHECK(ctx);
  return GB_OK;
}

// proposals of the owned vertices for the all-reduce MIN (prop reset first)
gb_status gb_cc_dist_propose(gb_ctx* ctx, int64_t n, int64_t lo, int64_t hi, const int32_t* hook,
                             int32_t* mn, const int32_t* pp, int32_t* prop) {
  cudaStream_t s = stream_of(ctx);
  fill_i32<<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(n, kImax32, prop);
  if (hi > lo) cc_propose<<<grid_for(ctx, hi - lo, 256, 8), 256, 0, s>>>(lo, hi, hook, mn, pp, prop);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 2);
  return GB_OK;
}

// parent = min(pp, prop); gp = parent[parent]; changed / live counts (sync)
gb_status gb_cc_dist_shortcut(gb_ctx* ctx, int64_t n, const int32_t* pp, const int32_t* prop,
                              int32_t* parent, int32_t* gp, int32_t* gpp, int32_t sparsify,
                              int64_t* changed_host, int64_t* live_host) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  unsigned long long* cnt = ar.alloc<unsigned long long>(2);
  GB_ARENA_CHECK(ctx, ar);
  const int vg = grid_for(ctx, n, 256, 8);
  cc_merge<<<vg, 256, 0, s>>>(n, pp, prop, parent);
  GB_CUDA(ctx, cudaMemsetAsync(cnt, 0, 16, s));
  cc_shortcut<<<vg, 256, 0, s>>>(n, parent, gp, gpp, sparsify, cnt, cnt + 1, nullptr, nullptr);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 3);
  int64_t h[2];
  GB_TRY(read_i64(ctx, (const int64_t*)cnt, h, 2));
  *changed_host = h[0];
  *live_host = h[1];
  return GB_OK;
}

gb_status gb_widen_i32(gb_ctx* ctx, int64_t n, const int32_t* in, int64_t* out) {
  if (n) widen_i32<<<grid_for(ctx, n, 256, 8), 256, 0, stream_of(ctx)>>>(n, in, (long long*)out);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

}  // extern "C"
