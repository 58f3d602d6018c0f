// BFS parents and a Graph500-style validation of the BFS tree.
//
// The reference bfs returns levels only (algorithms.py:66-77; SURVEY A-note
// 6); BASELINE.json's north star asks for "BFS levels/parents-validity", so
// this is the extension beyond the oracle.  Parents are DERIVED from the
// levels so they are deterministic (and bit-comparable with the C oracle):
// parent[v] = the smallest id u adjacent to v with level[u] = level[v] - 1,
// parent[source] = source, -1 when v is unreached.  One warp per reached
// vertex walks v's sorted row until the first such u (early exit; hubs meet a
// frontier vertex within a few entries).  For a symmetric matrix the row of
// v lists its neighbours; in general the walked orientation is the IN-edge
// one (rows of A^T), so (parent[v], v) is an edge of A.
//
// Validation (Graph500 spec, section "validation"), all on the device, one
// pass over the vertices and one over the stored entries of A:
//   0: parent[source] == source and level[source] == 1
//   1: a reached vertex v != source has a reached parent with
//      level[v] == level[parent] + 1 and (parent, v) stored in A
//   2: an unreached vertex has parent -1 (and level 0)
//   3: every stored entry (u, v) (the search follows row u to column v,
//      vxm(f, A)) with u reached has v reached and level[v] <= level[u] + 1;
//      applied to both (u, v) and (v, u) of a symmetric matrix this is
//      Graph500's "both ends reached or neither, levels at most one apart"
#include <vector>

#include "gb_common.cuh"

namespace gb {

__global__ void bfs_parents_kernel(int64_t n, const int64_t* __restrict__ off,
                                   const int32_t* __restrict__ idx,
                                   const int64_t* __restrict__ levels, int64_t source,
                                   int64_t* __restrict__ parents) {
  const int lane = threadIdx.x & 31;
  const int grp = lane >> 3, gl = lane & 7;  // four 8-lane groups per warp
  const unsigned gmask = 0xffu << (8 * grp);
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // 32 vertices per warp step: lanes test their vertex, then each 8-lane
  // group walks one reached vertex's row 8 entries at a time (a parent is
  // usually among the first few in-neighbours: the lowest ids are the hubs)
  for (int64_t base = w0 * 32; base < n; base += nw * 32) {
    const int64_t v = base + lane;
    const int64_t lv = v < n ? levels[v] : 0;
    if (v < n && lv == 0) parents[v] = -1;
    if (v == source) parents[v] = source;
    uint32_t todo = __ballot_sync(GB_FULL, v < n && lv > 1 && v != source);
    while (todo) {
      // group g takes the g-th remaining vertex (if any)
      uint32_t t = todo;
      for (int g = 0; g < grp && t; ++g) t &= t - 1;
      const int j = t ? __ffs(t) - 1 : -1;
      for (int g = 0; g < 4 && todo; ++g) todo &= todo - 1;
      const int64_t want = __shfl_sync(GB_FULL, lv, j < 0 ? 0 : j) - 1;
      if (j >= 0) {
        const int64_t vv = base + j;
        const int64_t lo = off[vv], hi = off[vv + 1];
        int64_t found = -1;
        for (int64_t p0 = lo; p0 < hi; p0 += 8) {
          const int64_t p = p0 + gl;
          const int32_t u = p < hi ? idx[p] : -1;
          const bool hit = u >= 0 && levels[u] == want;
          const uint32_t b = __ballot_sync(gmask, hit) & gmask;
          if (b) {
            found = __shfl_sync(gmask, u, __ffs(b) - 1);  // rows ascend: the min id
            break;
          }
        }
        if (gl == 0) parents[vv] = found;  // -1 only for an inconsistent level vector
      }
    }
  }
}

__device__ __forceinline__ bool row_has(const int64_t* off, const int32_t* idx, int64_t r,
                                        int32_t c) {
  int64_t lo = off[r], hi = off[r + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int32_t x = idx[mid];
    if (x == c) return true;
    if (x < c) lo = mid + 1; else hi = mid;
  }
  return false;
}

// in_off / in_idx: rows of A^T (the in-edges of v, where (parent, v) must be)
__global__ void bfs_validate_vertices(int64_t n, const int64_t* __restrict__ in_off,
                                      const int32_t* __restrict__ in_idx,
                                      const int64_t* __restrict__ levels,
                                      const int64_t* __restrict__ parents, int64_t source,
                                      unsigned long long* __restrict__ err) {
  unsigned long long e0 = 0, e1 = 0, e2 = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lv = levels[v], pv = parents[v];
    if (v == source) {
      e0 += !(pv == source && lv == 1);
    } else if (lv > 0) {
      bool ok = pv >= 0 && pv < n;
      if (ok) {
        const int64_t lp = levels[pv];
        ok = lp > 0 && lv == lp + 1 && row_has(in_off, in_idx, v, (int32_t)pv);
      }
      e1 += !ok;
    } else {
      e2 += !(pv == -1 && lv == 0);
    }
  }
  if (e0) atomicAdd(err + 0, e0);
  if (e1) atomicAdd(err + 1, e1);
  if (e2) atomicAdd(err + 2, e2);
}

__global__ void bfs_validate_edges(int64_t n, const int64_t* __restrict__ off,
                                   const int32_t* __restrict__ idx,
                                   const int64_t* __restrict__ levels,
                                   unsigned long long* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long e3 = 0;
  for (int64_t u = w0; u < n; u += nw) {
    const int64_t lu = levels[u];
    for (int64_t p = off[u] + lane; p < off[u + 1]; p += 32) {
      const int64_t lv = levels[idx[p]];
      const bool bad = lu > 0 && (lv == 0 || lv > lu + 1);
      e3 += bad;
    }
  }
  e3 = (unsigned long long)warp_sum_ll((long long)e3);
  if (lane == 0 && e3) atomicAdd(err + 3, e3);
}

// ---------------------------------------------------------------------------
// Work counters of a fused BFS, exactly as the reference's kernels tally them
// (kernels.py:153-191 pull, :242-280 push), recomputed after the run from the
// final levels and the direction log: iteration t multiplies the frontier
// F_t = {level == t+1} under the mask "not visited" = {level == 0 or > t+1}.
//   push t: multiplies += sum of out-degrees of F_t; adds += multiplies -
//           |distinct out-neighbours of F_t| (one segment per output row)
//   pull t: for every allowed row x with in-edges: reads += position of its
//           first in-neighbour in F_t + 1 (early exit) or its length;
//           multiplies += its in-neighbours in F_t; adds += that - 1 if > 0.
// One warp per vertex walks its in-edge row once for every iteration: the
// push iterations as a 64-bit mask of the levels seen, up to kCntPull pull
// iterations with (count, first position).  acc[t] = {multiplies, reads,
// distinct outputs (push) / rows with a product (pull)}.
// ---------------------------------------------------------------------------
constexpr int kCntPull = 4;
constexpr int kCntLevels = 64;

__global__ void __launch_bounds__(256)
bfs_counters_kernel(int64_t n, const int64_t* __restrict__ in_off, const int32_t* __restrict__ in_idx,
                    const int64_t* __restrict__ out_off, const int64_t* __restrict__ levels,
                    int32_t T, unsigned long long push_mask, int32_t npl, int4 pl, int32_t early,
                    unsigned long long* __restrict__ acc) {
  __shared__ unsigned long long s_acc[kCntLevels * 3];
  for (int i = threadIdx.x; i < kCntLevels * 3; i += blockDim.x) s_acc[i] = 0;
  __syncthreads();
  const int pls[kCntPull] = {pl.x, pl.y, pl.z, pl.w};
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = w0; x < n; x += nw) {
    const int64_t lx = levels[x];
    if (lane == 0 && lx > 0 && lx <= T && ((push_mask >> (lx - 1)) & 1))
      atomicAdd(&s_acc[3 * (lx - 1)], (unsigned long long)(out_off[x + 1] - out_off[x]));
    const int64_t lo = in_off[x], hi = in_off[x + 1];
    unsigned long long seen = 0;
    unsigned cnt[kCntPull] = {0, 0, 0, 0};
    int64_t first[kCntPull] = {INT64_MAX, INT64_MAX, INT64_MAX, INT64_MAX};
    for (int64_t p = lo + lane; p < hi; p += 32) {
      const int64_t L = levels[in_idx[p]];
      if (L <= 0 || L > T) continue;
      const int t = (int)(L - 1);
      if ((push_mask >> t) & 1) {
        seen |= 1ull << t;
      } else {
#pragma unroll
        for (int j = 0; j < kCntPull; ++j)
          if (j < npl && pls[j] == t) {
            ++cnt[j];
            if (p - lo < first[j]) first[j] = p - lo;
          }
      }
    }
    const unsigned s_lo = __reduce_or_sync(GB_FULL, (unsigned)seen);
    const unsigned s_hi = __reduce_or_sync(GB_FULL, (unsigned)(seen >> 32));
#pragma unroll
    for (int j = 0; j < kCntPull; ++j) {
      cnt[j] = __reduce_add_sync(GB_FULL, cnt[j]);
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int64_t f = __shfl_xor_sync(GB_FULL, first[j], o);
        if (f < first[j]) first[j] = f;
      }
    }
    if (lane == 0) {
      unsigned long long m = ((unsigned long long)s_hi << 32) | s_lo;
      while (m) {
        const int t = __ffsll((long long)m) - 1;
        m &= m - 1;
        atomicAdd(&s_acc[3 * t + 2], 1ull);
      }
      const int64_t len = hi - lo;
      for (int j = 0; j < npl; ++j) {
        const int t = pls[j];
        const bool allowed = lx == 0 || lx > t + 1;
        if (!allowed || len == 0) continue;
        const int64_t reads = early && cnt[j] ? first[j] + 1 : len;
        atomicAdd(&s_acc[3 * t + 1], (unsigned long long)reads);
        atomicAdd(&s_acc[3 * t], (unsigned long long)cnt[j]);
        if (cnt[j]) atomicAdd(&s_acc[3 * t + 2], 1ull);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < T * 3; i += blockDim.x)
    if (s_acc[i]) atomicAdd(acc + i, s_acc[i]);
}

}  // namespace gb

using namespace gb;

extern "C" {

gb_status gb_bfs_parents(gb_ctx* ctx, const gb_csr* in_edges, const int64_t* levels,
                         int64_t source, int64_t* parents) {
  const int64_t n = in_edges->nrows;
  if (source < 0 || source >= n) return set_error(ctx, GB_ERR_INDEX, "source out of range");
  if (n == 0) return GB_OK;
  bfs_parents_kernel<<<grid_for(ctx, n, 256, 8), 256, 0, stream_of(ctx)>>>(
      n, in_edges->offsets, in_edges->indices, levels, source, parents);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

gb_status gb_bfs_counters(gb_ctx* ctx, const gb_csr* out_edges, const gb_csr* in_edges,
                          const int64_t* levels, int64_t iters, const int32_t* dirs_host,
                          int32_t early_exit, int64_t* totals_host) {
  totals_host[0] = totals_host[1] = totals_host[2] = 0;
  const int64_t n = in_edges->nrows;
  if (iters <= 0 || n == 0) return GB_OK;
  const bool iso_one = !in_edges->values && !out_edges->values && in_edges->iso_i64 != 0 &&
                       out_edges->iso_i64 != 0;
  if (iters > kCntLevels || !iso_one)
    return set_error(ctx, GB_ERR_UNSUPPORTED, "bfs counters: > %d iterations or a valued matrix",
                     kCntLevels);
  unsigned long long push_mask = 0;
  int pl[kCntPull] = {-1, -1, -1, -1};
  int npl = 0;
  for (int64_t t = 0; t < iters; ++t) {
    if (dirs_host[t] == GB_DIR_PULL) {
      if (npl == kCntPull)
        return set_error(ctx, GB_ERR_UNSUPPORTED, "bfs counters: > %d pull iterations", kCntPull);
      pl[npl++] = (int)t;
    } else {
      push_mask |= 1ull << t;
    }
  }
  cudaStream_t s = stream_of(ctx);
  Arena ar(ctx);
  unsigned long long* acc = ar.alloc<unsigned long long>(3 * kCntLevels);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(acc, 0, 8 * 3 * kCntLevels, s));
  bfs_counters_kernel<<<grid_for(ctx, n * 32, 256, 8), 256, 0, s>>>(
      n, in_edges->offsets, in_edges->indices, out_edges->offsets, levels, (int32_t)iters,
      push_mask, npl, make_int4(pl[0], pl[1], pl[2], pl[3]), early_exit, acc);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 2);
  std::vector<int64_t> h(3 * iters);
  GB_TRY(read_i64(ctx, (const int64_t*)acc, h.data(), (int)(3 * iters)));
  for (int64_t t = 0; t < iters; ++t) {
    const int64_t mult = h[3 * t], reads = h[3 * t + 1], segs = h[3 * t + 2];
    totals_host[0] += reads;  // push iterations read nothing (kernels.py:242-280)
    totals_host[1] += mult;
    totals_host[2] += mult - segs;
  }
  return GB_OK;
}

gb_status gb_bfs_validate(gb_ctx* ctx, const gb_csr* a, const gb_csr* in_edges, int64_t source,
                          const int64_t* levels, const int64_t* parents, int64_t* errors_host) {
  const int64_t n = a->nrows;
  for (int i = 0; i < 4; ++i) errors_host[i] = 0;
  if (n == 0) return GB_OK;
  if (source < 0 || source >= n) return set_error(ctx, GB_ERR_INDEX, "source out of range");
  cudaStream_t s = stream_of(ctx);
  Arena ar(ctx);
  unsigned long long* err = ar.alloc<unsigned long long>(4);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(err, 0, 32, s));
  bfs_validate_vertices<<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(
      n, in_edges->offsets, in_edges->indices, levels, parents, source, err);
  bfs_validate_edges<<<grid_for(ctx, n * 32, 256, 8), 256, 0, s>>>(n, a->offsets, a->indices,
                                                                   levels, err);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 3);
  return read_i64(ctx, (const int64_t*)err, errors_host, 4);
}

}  // extern "C"
