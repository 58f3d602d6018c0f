// Fused direction-optimizing BFS: algorithms.py:48-77 with the dispatcher
// kernels.py:108-126 / 293-310 and both multiply kernels specialised to the
// LogicalOrAnd semiring with a complemented visited mask.
//
// Per level the reference does  assign(visited, depth, mask=f)  ->
// vxm(LogicalOrAnd, f, A, mask=~visited)  ->  reduce(Plus, f).  Here:
//   push level:  lbs_expand over the frontier list marks unvisited
//                neighbours in a byte array (plain stores, idempotent OR),
//                then bfs_finalize turns the marks into the next frontier
//                (bitmap + list + count), stamps levels and the visited
//                bitmap in one pass.
//   pull level:  bfs_pull walks in-edges of unvisited, non-isolated rows
//                (one lane per row, warp per 32 rows) and stops at the first
//                frontier hit (early exit, kernels.py:169-178); it writes the
//                next frontier directly -- no separate finalize.
// The direction of every level is decided on the host with the reference
// rule (gb_decide_direction) from the exact frontier count, so the direction
// trace equals the reference's.
#include <math.h>

#include "gb_common.cuh"
#include "gb_lbs.cuh"

#include <cub/cub.cuh>

namespace gb {

// A stored entry participates in LogicalAnd(a, u) iff a != 0.
struct EdgeOn {
  const void* vals;
  int dtype;
  __device__ __forceinline__ bool operator()(int64_t p) const {
    if (!vals) return true;
    return dtype == GB_I64 ? __ldg((const long long*)vals + p) != 0
                           : __ldg((const double*)vals + p) != 0.0;
  }
};

// ---------------------------------------------------------------------------
// push: load-balanced expansion of the frontier's out-edges
// ---------------------------------------------------------------------------
// Marking: the live visited bitmap `vbm` is probed through L1 (ld.ca: a stale
// clear bit only costs a redundant atomic) and a clear bit is set with one
// atomicOr, so a vertex reached by many frontier edges costs one read per edge
// but (almost) one write in total.  bfs_finalize recovers the new frontier as
// vbm & ~vprev.
__device__ __forceinline__ void mark(uint32_t* vbm, int32_t v, uint32_t word) {
  const uint32_t bit = 1u << (v & 31);
  if (!(word & bit)) atomicOr(vbm + (v >> 5), bit);
}

// Warp-tile push expansion (no shared memory, no barriers): a batch of
// column loads is issued before any visited probe.
template <bool VALS>
struct PushBits {
  const int32_t* __restrict__ idx;
  EdgeOn on;
  uint32_t* __restrict__ vbm;
  template <int B>
  __device__ __forceinline__ void batch(const int64_t (&p)[B], const bool (&live)[B]) {
    int32_t v[B];
#pragma unroll
    for (int r = 0; r < B; ++r) {
      v[r] = -1;
      if (live[r]) {
        const int32_t c = ld_stream(idx + p[r]);
        v[r] = (!VALS || on(p[r])) ? c : -1;
      }
    }
    uint32_t word[B];
#pragma unroll
    for (int r = 0; r < B; ++r) word[r] = v[r] >= 0 ? ld_probe(vbm + (v[r] >> 5)) : ~0u;
#pragma unroll
    for (int r = 0; r < B; ++r)
      if (v[r] >= 0) mark(vbm, v[r], word[r]);
  }
  __device__ __forceinline__ void visit(int64_t p) {
    const int32_t u = ld_stream(idx + p);
    if (!VALS || on(p)) mark(vbm, u, ld_probe(vbm + (u >> 5)));
  }
};

template <bool VALS>
__global__ void __launch_bounds__(256)
bfs_expand_warp(int64_t K, const int64_t* __restrict__ S, const int64_t* __restrict__ rowstart,
                const int32_t* __restrict__ tile_first, const int32_t* __restrict__ idx,
                EdgeOn on, uint32_t* __restrict__ vbm) {
  PushBits<VALS> f{idx, on, vbm};
  warp_tiles(K, S, rowstart, tile_first, f);
}

__global__ void bfs_init(int64_t source, int64_t* levels, uint32_t* vbm, uint32_t* vprev,
                         uint32_t* fbm, int32_t* F) {
  levels[source] = 1;
  vbm[source >> 5] |= 1u << (source & 31);
  vprev[source >> 5] |= 1u << (source & 31);
  fbm[source >> 5] |= 1u << (source & 31);
  F[0] = (int32_t)source;
}

// Warp per 32 words (1024 vertices): lane l diffs word w0+l of the live
// visited bitmap against the level-start snapshot, then the warp walks the
// non-empty words so level stamps and frontier-list writes are coalesced.
__global__ void __launch_bounds__(256)
bfs_finalize(int64_t n, int64_t depth, uint32_t* __restrict__ vbm,
             uint32_t* __restrict__ vprev, uint32_t* __restrict__ fbm_next,
             int64_t* __restrict__ levels, int32_t* __restrict__ F,
             unsigned long long* __restrict__ count,
             unsigned long long* __restrict__ count_clear, const uint32_t* __restrict__ xbm) {
  // xbm == NULL: new frontier = vbm & ~vprev (single GPU).  xbm != NULL: the
  // all-reduced new-frontier bitmap of a 1D-partitioned run is authoritative.
  if (blockIdx.x == 0 && threadIdx.x == 0) *count_clear = 0;
  const int lane = threadIdx.x & 31;
  const int64_t W = (n + 31) / 32;
  const int64_t G = (W + 31) / 32;
  const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g = g0; g < G; g += ng) {
    const int64_t w = g * 32 + lane;
    uint32_t bits = 0;
    if (w < W) {
      if (xbm) {
        bits = xbm[w];
        if (bits) {
          vbm[w] |= bits;
          vprev[w] |= bits;
        }
      } else {
        const uint32_t cur = vbm[w], old = vprev[w];
        bits = cur & ~old;
        if (bits) vprev[w] = cur;
      }
      fbm_next[w] = bits;
    }
    // frontier list slots for the whole group, in word order
    const int c = __popc(bits);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(GB_FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(GB_FULL, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && total) base = atomicAdd(count, (unsigned long long)total);
    base = __shfl_sync(GB_FULL, base, 31);
    uint32_t nonzero = __ballot_sync(GB_FULL, bits != 0);
    while (nonzero) {
      const int j = __ffs(nonzero) - 1;
      nonzero &= nonzero - 1;
      const uint32_t wb = __shfl_sync(GB_FULL, bits, j);
      const int start = __shfl_sync(GB_FULL, incl - c, j);
      if ((wb >> lane) & 1u) {
        const int64_t v = (g * 32 + j) * 32 + lane;
        levels[v] = depth;
        F[base + start + __popc(wb & ((1u << lane) - 1u))] = (int32_t)v;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// pull: warp per 32 words; candidate rows are compacted into a shared list
// and processed 8 per lane with their first loads batched
// ---------------------------------------------------------------------------
constexpr int kPullBatch = 8;                // rows per lane per pass
constexpr int kPullList = 32 * kPullBatch;   // rows per warp per pass
constexpr int kPullSerial = 8;               // entries a lane scans alone before the warp helps

__global__ void __launch_bounds__(256)
bfs_pull(int64_t n, int64_t depth, const int64_t* __restrict__ off,
         const int32_t* __restrict__ idx, EdgeOn on, const uint32_t* __restrict__ nonempty,
         uint32_t* __restrict__ vbm, uint32_t* __restrict__ vprev, const uint32_t* __restrict__ fbm,
         uint32_t* __restrict__ fbm_next, int64_t* __restrict__ levels,
         int32_t* __restrict__ F, unsigned long long* __restrict__ count,
         unsigned long long* __restrict__ count_clear, int64_t g_lo, int64_t g_hi) {
  // [g_lo, g_hi): groups of 32 words (1024 vertices) this launch owns; a
  // 1D-partitioned rank passes its vertex block with `off`/`nonempty`
  // pointers rebased so global vertex ids index them directly.
  __shared__ int32_t s_list[8][kPullList];
  __shared__ uint32_t s_new[8][32];
  if (blockIdx.x == 0 && threadIdx.x == 0) *count_clear = 0;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int64_t W = (n + 31) / 32;
  const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int32_t* list = s_list[wid];
  uint32_t* nw = s_new[wid];
  for (int64_t g = g_lo + g0; g < g_hi; g += ng) {
    const int64_t w = g * 32 + lane;
    uint32_t rem = w < W ? (~vbm[w] & __ldg(nonempty + w)) : 0u;
    nw[lane] = 0;
    __syncwarp();
    while (true) {
      const int c = __popc(rem);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(GB_FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const int total = __shfl_sync(GB_FULL, incl, 31);
      if (total == 0) break;
      int slot = incl - c;
      while (rem && slot < kPullList) {
        const int b = __ffs(rem) - 1;
        rem &= rem - 1;
        list[slot++] = (int32_t)(w * 32 + b);
      }
      __syncwarp();
      const int take = total < kPullList ? total : kPullList;
      int64_t lo[kPullBatch], hi[kPullBatch];
      int32_t v[kPullBatch];
#pragma unroll
      for (int r = 0; r < kPullBatch; ++r) {
        const int q = r * 32 + lane;
        v[r] = q < take ? list[q] : -1;
        lo[r] = hi[r] = 0;
        if (v[r] >= 0) {
          lo[r] = __ldg(off + v[r]);
          hi[r] = __ldg(off + v[r] + 1);
        }
      }
      int32_t j0[kPullBatch];
#pragma unroll
      for (int r = 0; r < kPullBatch; ++r) j0[r] = lo[r] < hi[r] ? __ldg(idx + lo[r]) : 0;
      uint32_t todo = 0;
#pragma unroll
      for (int r = 0; r < kPullBatch; ++r) {
        bool hit = false;
        if (lo[r] < hi[r]) {
          hit = ((__ldg(fbm + (j0[r] >> 5)) >> (j0[r] & 31)) & 1u) && on(lo[r]);
          int64_t p = lo[r] + 1;
          const int64_t stop = lo[r] + kPullSerial < hi[r] ? lo[r] + kPullSerial : hi[r];
          for (; !hit && p < stop; ++p) {
            const int32_t j = __ldg(idx + p);
            hit = ((__ldg(fbm + (j >> 5)) >> (j & 31)) & 1u) && on(p);
          }
          lo[r] = p;
          if (!hit && p < hi[r]) todo |= 1u << r;
        }
        if (hit) {
          atomicOr(&nw[(v[r] >> 5) - g * 32], 1u << (v[r] & 31));
          levels[v[r]] = depth;
        }
      }
      // long rows still unresolved: the warp scans them together
      for (int r = 0; r < kPullBatch; ++r) {
        uint32_t lanes = __ballot_sync(GB_FULL, (todo >> r) & 1u);
        while (lanes) {
          const int src = __ffs(lanes) - 1;
          lanes &= lanes - 1;
          const int64_t qlo = __shfl_sync(GB_FULL, lo[r], src);
          const int64_t qhi = __shfl_sync(GB_FULL, hi[r], src);
          const int32_t vv = __shfl_sync(GB_FULL, v[r], src);
          bool h = false;
          for (int64_t base = qlo; base < qhi && !h; base += 32) {
            const int64_t q = base + lane;
            bool mh = false;
            if (q < qhi) {
              const int32_t j = __ldg(idx + q);
              mh = ((__ldg(fbm + (j >> 5)) >> (j & 31)) & 1u) && on(q);
            }
            h = __ballot_sync(GB_FULL, mh) != 0;
          }
          if (h && lane == src) {
            atomicOr(&nw[(vv >> 5) - g * 32], 1u << (vv & 31));
            levels[vv] = depth;
          }
        }
      }
      __syncwarp();
    }
    __syncwarp();
    const uint32_t bits = nw[lane];
    if (w < W) {
      fbm_next[w] = bits;
      if (bits) {
        vbm[w] |= bits;
        vprev[w] |= bits;
      }
    }
    const int c = __popc(bits);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(GB_FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(GB_FULL, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && total) base = atomicAdd(count, (unsigned long long)total);
    base = __shfl_sync(GB_FULL, base, 31);
    int slot = incl - c;
    uint32_t b2 = bits;
    while (b2) {
      const int b = __ffs(b2) - 1;
      b2 &= b2 - 1;
      F[base + slot++] = (int32_t)(w * 32 + b);
    }
    __syncwarp();
  }
}

__global__ void bfs_unstamp(int64_t K, const int32_t* __restrict__ F, int64_t* __restrict__ levels) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K;
       i += (int64_t)gridDim.x * blockDim.x)
    levels[F[i]] = 0;
}

// (A shared-memory cache of the low-id visited words was tried here and lost:
// bank conflicts and halved occupancy cost more than the saved L1 sectors.)
template <bool VALS>
static gb_status launch_push_t(gb_ctx* ctx, int64_t K, const LbsPlan& plan, const gb_csr* a,
                               EdgeOn on, uint32_t* vbm) {
  bfs_expand_warp<VALS><<<resident_grid(ctx, bfs_expand_warp<VALS>, 256), 256, 0, stream_of(ctx)>>>(
      K, plan.S, plan.rowstart, plan.tile_first, a->indices, on, vbm);
  GB_LAUNCH_CHECK(ctx);
  return GB_OK;
}

static gb_status launch_push(gb_ctx* ctx, int64_t K, const LbsPlan& plan, const gb_csr* a,
                             EdgeOn on, uint32_t* vbm) {
  return a->values ? launch_push_t<true>(ctx, K, plan, a, on, vbm)
                   : launch_push_t<false>(ctx, K, plan, a, on, vbm);
}

}  // namespace gb

using namespace gb;

extern "C" {

int32_t gb_decide_direction(int64_t nnz, int64_t nrows, int64_t nnz_u, double ratio,
                            int32_t policy, int64_t* estimate_out) {
  // kernels.py:108-126.  d*nnz_u is rounded half-to-even like Python round():
  // nearbyint() under the default FE_TONEAREST mode.
  const double d = nrows ? (double)nnz / (double)nrows : 0.0;
  const int64_t est = (int64_t)nearbyint(d * (double)nnz_u);
  const double thr = (double)nnz * ratio;
  if (estimate_out) *estimate_out = est;
  if (policy == GB_DIR_PUSH) return GB_DIR_PUSH;
  if (policy == GB_DIR_PULL) return GB_DIR_PULL;
  return (double)est > thr ? GB_DIR_PULL : GB_DIR_PUSH;
}

gb_status gb_bfs(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull,
                 const uint32_t* pull_nonempty, int64_t source, int64_t max_iters,
                 double ratio, int32_t policy, int64_t* levels, int32_t* log_dir,
                 int64_t* log_nvals, int64_t* log_est, int64_t* iters_out) {
  const int64_t n = push->nrows;
  if (source < 0 || source >= n) return set_error(ctx, GB_ERR_INDEX, "source %lld out of range", (long long)source);
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  uint32_t* vbm = ar.alloc<uint32_t>(W);
  uint32_t* fbm[2] = {ar.alloc<uint32_t>(W), ar.alloc<uint32_t>(W)};
  int32_t* F = ar.alloc<int32_t>(n);
  uint32_t* vprev = ar.alloc<uint32_t>(W);
  unsigned long long* cnt = ar.alloc<unsigned long long>(2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(levels, 0, sizeof(int64_t) * n, s));
  GB_CUDA(ctx, cudaMemsetAsync(vbm, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(fbm[0], 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(vprev, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(cnt, 0, 16, s));
  bfs_init<<<1, 1, 0, s>>>(source, levels, vbm, vprev, fbm[0], F);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 6);  // 5 memsets + init

  const EdgeOn push_on{push->values, push->dtype};
  const EdgeOn pull_on{pull ? pull->values : nullptr, pull ? pull->dtype : 0};
  const bool push_dead = !push->values && push->iso_i64 == 0 && push->iso_f64 == 0.0;
  const bool pull_dead = pull && !pull->values && pull->iso_i64 == 0 && pull->iso_f64 == 0.0;
  int64_t K = 1, depth = 1, iters = 0;
  int cur = 0;
  for (int64_t it = 0; it < max_iters; ++it) {
    int64_t est = 0;
    const int32_t dir = gb_decide_direction(push->nnz, push->nrows, K, ratio, policy, &est);
    log_dir[it] = dir;
    log_nvals[it] = K;
    log_est[it] = est;
    iters = it + 1;
    unsigned long long* c = cnt + (it & 1);
    unsigned long long* c_next = cnt + ((it + 1) & 1);
    if (dir == GB_DIR_PULL) {
      if (!pull) return set_error(ctx, GB_ERR_FORMAT, "column-oriented storage missing");
      if (pull_dead) {
        GB_CUDA(ctx, cudaMemsetAsync(fbm[cur ^ 1], 0, sizeof(uint32_t) * W, s));
        GB_CUDA(ctx, cudaMemsetAsync(c, 0, 8, s));
        GB_CUDA(ctx, cudaMemsetAsync(c_next, 0, 8, s));
      } else {
        const int grid = grid_for(ctx, W, 256, 8);
        const int ps = prof_begin(ctx, PROF_BFS_PULL, K);
        bfs_pull<<<grid, 256, 0, s>>>(n, depth + 1, pull->offsets, pull->indices, pull_on,
                                      pull_nonempty, vbm, vprev, fbm[cur], fbm[cur ^ 1], levels, F,
                                      c, c_next, 0, (W + 31) / 32);
        prof_end(ctx, ps);
        count_launch(ctx, 1);
      }
    } else {
      if (!push_dead) {
        LbsPlan plan;
        GB_TRY(lbs_prepare(ctx, ar, K, F, push->offsets, push->nnz, &plan, kWarpTile));
        const int ps = prof_begin(ctx, PROF_BFS_PUSH, K);
        GB_TRY(launch_push(ctx, K, plan, push, push_on, vbm));
        prof_end(ctx, ps);
        count_launch(ctx, 5);  // degrees, scan (2), tile_first, expand
      }
      const int pf = prof_begin(ctx, PROF_BFS_FINALIZE, K);
      bfs_finalize<<<grid_for(ctx, W, 256, 8), 256, 0, s>>>(n, depth + 1, vbm, vprev, fbm[cur ^ 1],
                                                         levels, F, c, c_next, nullptr);
      prof_end(ctx, pf);
      count_launch(ctx, 1);
    }
    GB_LAUNCH_CHECK(ctx);
    GB_TRY(read_i64(ctx, (const int64_t*)c, &K));
    cur ^= 1;
    if (K == 0) break;
    ++depth;
    if (it + 1 == max_iters) {
      // loop cap reached: the reference never stamps the last frontier
      // (its assign happens at the start of the next iteration)
      bfs_unstamp<<<grid_for(ctx, K, 256), 256, 0, s>>>(K, F, levels);
      GB_LAUNCH_CHECK(ctx);
      count_launch(ctx, 1);
    }
  }
  *iters_out = iters;
  return GB_OK;
}

// ---------------------------------------------------------------------------
// 1D-partitioned BFS steps (one rank of P; the host loop and the NCCL
// exchange of the new-frontier bitmap live in distributed.py).  Rank p owns
// vertices [lo, hi) (lo, hi multiples of 1024 except hi = n) and stores
//   rowblock: rows lo..hi-1 of A^T (in-edges of owned vertices) for pull,
//   colblock: all n rows of A restricted to columns in [lo, hi) for push.
// Every bitmap / levels / frontier buffer is global-sized and replicated.
// ---------------------------------------------------------------------------

__global__ void bfs_collect(int64_t w_lo, int64_t w_hi, const uint32_t* __restrict__ vbm,
                            const uint32_t* __restrict__ vprev, uint32_t* __restrict__ xbm) {
  for (int64_t w = w_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < w_hi;
       w += (int64_t)gridDim.x * blockDim.x)
    xbm[w] = vbm[w] & ~vprev[w];
}

gb_status gb_bfs_dist_init(gb_ctx* ctx, int64_t n, int64_t source, int64_t* levels,
                           uint32_t* vbm, uint32_t* vprev, uint32_t* fbm, int32_t* F) {
  if (source < 0 || source >= n) return set_error(ctx, GB_ERR_INDEX, "source out of range");
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  GB_CUDA(ctx, cudaMemsetAsync(levels, 0, sizeof(int64_t) * n, s));
  GB_CUDA(ctx, cudaMemsetAsync(vbm, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(vprev, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(fbm, 0, sizeof(uint32_t) * W, s));
  bfs_init<<<1, 1, 0, s>>>(source, levels, vbm, vprev, fbm, F);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 5);
  return GB_OK;
}

gb_status gb_bfs_dist_push(gb_ctx* ctx, const gb_csr* colblock, int64_t K, const int32_t* F,
                           uint32_t* vbm) {
  if (K == 0 || colblock->nnz == 0) return GB_OK;
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  LbsPlan plan;
  GB_TRY(lbs_prepare(ctx, ar, K, F, colblock->offsets, colblock->nnz, &plan, kWarpTile));
  const EdgeOn on{colblock->values, colblock->dtype};
  const int ps = prof_begin(ctx, PROF_BFS_PUSH, K);
  GB_TRY(launch_push(ctx, K, plan, colblock, on, vbm));
  prof_end(ctx, ps);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 5);
  return GB_OK;
}

gb_status gb_bfs_dist_collect(gb_ctx* ctx, int64_t n, int64_t lo, int64_t hi,
                              const uint32_t* vbm, const uint32_t* vprev, uint32_t* xbm) {
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  const int64_t w_lo = lo / 32, w_hi = (hi + 31) / 32;
  GB_CUDA(ctx, cudaMemsetAsync(xbm, 0, sizeof(uint32_t) * W, s));
  if (w_hi > w_lo)
    bfs_collect<<<grid_for(ctx, w_hi - w_lo, 256), 256, 0, s>>>(w_lo, w_hi, vbm, vprev, xbm);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 2);
  return GB_OK;
}

gb_status gb_bfs_dist_pull(gb_ctx* ctx, const gb_csr* rowblock, int64_t lo, int64_t hi,
                           const uint32_t* nonempty_block, int64_t n, int64_t depth,
                           uint32_t* vbm, uint32_t* vprev, const uint32_t* fbm, uint32_t* xbm,
                           int64_t* levels) {
  if (lo % 1024) return set_error(ctx, GB_ERR_ARG, "partition start must be a multiple of 1024");
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  int32_t* F = ar.alloc<int32_t>(hi - lo + 1);
  unsigned long long* cnt = ar.alloc<unsigned long long>(2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(xbm, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(cnt, 0, 16, s));
  if (hi > lo && rowblock->nnz) {
    const EdgeOn on{rowblock->values, rowblock->dtype};
    // rebase so global vertex ids index the block's offsets / nonempty words
    const int64_t* off = rowblock->offsets - lo;
    const uint32_t* ne = nonempty_block - lo / 32;
    const int64_t g_lo = lo / 1024, g_hi = (hi + 1023) / 1024;
    const int ps = prof_begin(ctx, PROF_BFS_PULL, 0);
    bfs_pull<<<grid_for(ctx, (g_hi - g_lo) * 32, 256, 8), 256, 0, s>>>(
        hi, depth, off, rowblock->indices, on, ne, vbm, vprev, fbm, xbm, levels, F, cnt, cnt + 1,
        g_lo, g_hi);
    prof_end(ctx, ps);
  }
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 3);
  return GB_OK;
}

gb_status gb_bfs_dist_apply(gb_ctx* ctx, int64_t n, int64_t depth, const uint32_t* xbm,
                            uint32_t* vbm, uint32_t* vprev, uint32_t* fbm, int64_t* levels,
                            int32_t* F, int64_t* K_host) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  unsigned long long* cnt = ar.alloc<unsigned long long>(2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(cnt, 0, 16, s));
  bfs_finalize<<<grid_for(ctx, W, 256, 8), 256, 0, s>>>(n, depth, vbm, vprev, fbm, levels, F, cnt,
                                                        cnt + 1, xbm);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 2);
  return read_i64(ctx, (const int64_t*)cnt, K_host);
}

gb_status gb_bfs_dist_unstamp(gb_ctx* ctx, int64_t K, const int32_t* F, int64_t* levels) {
  if (K <= 0) return GB_OK;
  bfs_unstamp<<<grid_for(ctx, K, 256), 256, 0, stream_of(ctx)>>>(K, F, levels);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

// Column block of a CSR: every row keeps only its entries with column in
// [lo, hi) (columns stay global).  Two passes: counts, then copy.
__global__ void colblock_count(int64_t n, const int64_t* __restrict__ off,
                               const int32_t* __restrict__ idx, int32_t lo, int32_t hi,
                               int64_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n; r += nw) {
    long long c = 0;
    for (int64_t p = off[r] + lane; p < off[r + 1]; p += 32) c += idx[p] >= lo && idx[p] < hi;
    c = warp_sum_ll(c);
    if (lane == 0) cnt[r] = c;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[n] = 0;
}

__global__ void colblock_fill(int64_t n, const int64_t* __restrict__ off,
                              const int32_t* __restrict__ idx, int32_t lo, int32_t hi,
                              const int64_t* __restrict__ out_off, int32_t* __restrict__ out_idx) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n; r += nw) {
    int64_t o = out_off[r];
    for (int64_t base = off[r]; base < off[r + 1]; base += 32) {
      const int64_t p = base + lane;
      const bool keep = p < off[r + 1] && idx[p] >= lo && idx[p] < hi;
      const uint32_t bal = __ballot_sync(GB_FULL, keep);
      if (keep) out_idx[o + __popc(bal & ((1u << lane) - 1u))] = idx[p];
      o += __popc(bal);
    }
  }
}

gb_status gb_csr_column_block(gb_ctx* ctx, const gb_csr* a, int64_t lo, int64_t hi,
                              int64_t* out_offsets, int32_t* out_indices, int64_t* nnz_host) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int64_t n = a->nrows;
  int64_t* cnt = ar.alloc<int64_t>(n + 1);
  GB_ARENA_CHECK(ctx, ar);
  colblock_count<<<grid_for(ctx, n * 32, 256, 16), 256, 0, s>>>(n, a->offsets, a->indices,
                                                                (int32_t)lo, (int32_t)hi, cnt);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, out_offsets, n + 1, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, out_offsets, n + 1, s));
  GB_TRY(read_i64(ctx, out_offsets + n, nnz_host));
  if (out_indices)
    colblock_fill<<<grid_for(ctx, n * 32, 256, 16), 256, 0, s>>>(n, a->offsets, a->indices,
                                                                 (int32_t)lo, (int32_t)hi,
                                                                 out_offsets, out_indices);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 4);
  return GB_OK;
}

}  // extern "C"
