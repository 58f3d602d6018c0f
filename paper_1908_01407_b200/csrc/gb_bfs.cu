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

struct PushMark {
  const int32_t* __restrict__ idx;
  EdgeOn on;
  const uint32_t* __restrict__ vbm;
  uint8_t* __restrict__ nf;
  __device__ __forceinline__ void operator()(int64_t k, int64_t p, int64_t e) const {
    const int32_t v = __ldg(idx + p);
    if (!on(p)) return;
    if ((__ldg(vbm + (v >> 5)) >> (v & 31)) & 1u) return;
    nf[v] = 1;
  }
};

__global__ void bfs_init(int64_t source, int64_t* levels, uint32_t* vbm, uint32_t* fbm,
                         int32_t* F) {
  levels[source] = 1;
  vbm[source >> 5] |= 1u << (source & 31);
  fbm[source >> 5] |= 1u << (source & 31);
  F[0] = (int32_t)source;
}

// One thread per 32-vertex word: mark bytes -> next frontier.
__global__ void bfs_finalize(int64_t n, int64_t depth, uint8_t* __restrict__ nf,
                             uint32_t* __restrict__ vbm, uint32_t* __restrict__ fbm_next,
                             int64_t* __restrict__ levels, int32_t* __restrict__ F,
                             unsigned long long* __restrict__ count,
                             unsigned long long* __restrict__ count_clear) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *count_clear = 0;
  const int64_t W = (n + 31) / 32;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint4* p = reinterpret_cast<uint4*>(nf + w * 32);
    uint4 a = p[0], b = p[1];
    uint32_t bits = 0;
    if ((a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w) != 0) {
      uint32_t q[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if ((q[j] >> (8 * c)) & 0xffu) bits |= 1u << (4 * j + c);
      p[0] = make_uint4(0, 0, 0, 0);
      p[1] = make_uint4(0, 0, 0, 0);
      bits &= ~vbm[w];
      vbm[w] |= bits;
    }
    fbm_next[w] = bits;
    int c = __popc(bits);
    long long slot = warp_reserve(count, c);
    while (bits) {
      int b = __ffs(bits) - 1;
      bits &= bits - 1;
      int64_t v = w * 32 + b;
      levels[v] = depth;
      F[slot++] = (int32_t)v;
    }
  }
}

// Pull: warp per word of 32 candidate rows; lane = row.
constexpr int kPullSerial = 8;  // entries a lane scans alone before the warp helps

__global__ void __launch_bounds__(256)
bfs_pull(int64_t n, int64_t depth, const int64_t* __restrict__ off,
         const int32_t* __restrict__ idx, EdgeOn on, const uint32_t* __restrict__ nonempty,
         uint32_t* __restrict__ vbm, const uint32_t* __restrict__ fbm,
         uint32_t* __restrict__ fbm_next, int64_t* __restrict__ levels,
         int32_t* __restrict__ F, unsigned long long* __restrict__ count,
         unsigned long long* __restrict__ count_clear) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *count_clear = 0;
  const int lane = threadIdx.x & 31;
  const int64_t W = (n + 31) / 32;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp0; w < W; w += nwarps) {
    const uint32_t cand = ~vbm[w] & __ldg(nonempty + w);
    uint32_t found = 0;
    if (cand) {
      const int64_t v = w * 32 + lane;
      bool mine = (cand >> lane) & 1u;
      int64_t p = 0, hi = 0;
      bool hit = false;
      if (mine) {
        p = __ldg(off + v);
        hi = __ldg(off + v + 1);
        int64_t stop = p + kPullSerial < hi ? p + kPullSerial : hi;
        for (; p < stop; ++p) {
          const int32_t j = __ldg(idx + p);
          if (((__ldg(fbm + (j >> 5)) >> (j & 31)) & 1u) && on(p)) { hit = true; break; }
        }
      }
      // rows still unresolved after the serial phase: the warp scans them together
      uint32_t todo = __ballot_sync(GB_FULL, mine && !hit && p < hi);
      while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        int64_t q = __shfl_sync(GB_FULL, p, src);
        const int64_t qhi = __shfl_sync(GB_FULL, hi, src);
        bool h = false;
        for (q += lane; ; q += 32) {
          bool mh = false;
          if (q < qhi) {
            const int32_t j = __ldg(idx + q);
            mh = ((__ldg(fbm + (j >> 5)) >> (j & 31)) & 1u) && on(q);
          }
          const uint32_t any = __ballot_sync(GB_FULL, mh);
          if (any) { h = true; break; }
          if (__shfl_sync(GB_FULL, q, 0) + 32 >= qhi) break;
        }
        if (lane == src) hit = h;
      }
      found = __ballot_sync(GB_FULL, hit);
      if (hit) levels[v] = depth;
    }
    if (lane == 0) {
      fbm_next[w] = found;
      if (found) vbm[w] |= found;
    }
    const int c = lane == 0 ? __popc(found) : 0;
    long long base = 0;
    if (lane == 0 && c) base = (long long)atomicAdd(count, (unsigned long long)c);
    base = __shfl_sync(GB_FULL, base, 0);
    if ((found >> lane) & 1u) {
      const int rank = __popc(found & ((1u << lane) - 1u));
      F[base + rank] = (int32_t)(w * 32 + lane);
    }
  }
}

__global__ void bfs_unstamp(int64_t K, const int32_t* __restrict__ F, int64_t* __restrict__ levels) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K;
       i += (int64_t)gridDim.x * blockDim.x)
    levels[F[i]] = 0;
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
  uint8_t* nf = ar.alloc<uint8_t>(W * 32);
  unsigned long long* cnt = ar.alloc<unsigned long long>(2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(levels, 0, sizeof(int64_t) * n, s));
  GB_CUDA(ctx, cudaMemsetAsync(vbm, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(fbm[0], 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(nf, 0, (size_t)W * 32, s));
  GB_CUDA(ctx, cudaMemsetAsync(cnt, 0, 16, s));
  bfs_init<<<1, 1, 0, s>>>(source, levels, vbm, fbm[0], F);
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
        const int grid = grid_for(ctx, W * 32, 256, 16);
        const int ps = prof_begin(ctx, PROF_BFS_PULL, K);
        bfs_pull<<<grid, 256, 0, s>>>(n, depth + 1, pull->offsets, pull->indices, pull_on,
                                      pull_nonempty, vbm, fbm[cur], fbm[cur ^ 1], levels, F,
                                      c, c_next);
        prof_end(ctx, ps);
        count_launch(ctx, 1);
      }
    } else {
      if (!push_dead) {
        LbsPlan plan;
        GB_TRY(lbs_prepare(ctx, ar, K, F, push->offsets, push->nnz, &plan));
        PushMark f{push->indices, push_on, vbm, nf};
        const int ps = prof_begin(ctx, PROF_BFS_PUSH, K);
        lbs_expand<PushMark><<<plan.grid, kLbsThreads, 0, s>>>(K, plan.S, plan.rowstart,
                                                                plan.tile_first, f);
        prof_end(ctx, ps);
        count_launch(ctx, 5);  // degrees, scan (2), tile_first, expand
      }
      const int pf = prof_begin(ctx, PROF_BFS_FINALIZE, K);
      bfs_finalize<<<grid_for(ctx, W, 256), 256, 0, s>>>(n, depth + 1, nf, vbm, fbm[cur ^ 1],
                                                         levels, F, c, c_next);
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

}  // extern "C"
