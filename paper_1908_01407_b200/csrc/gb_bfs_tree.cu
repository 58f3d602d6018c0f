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
#include "gb_common.cuh"

namespace gb {

__global__ void bfs_parents_kernel(int64_t n, const int64_t* __restrict__ off,
                                   const int32_t* __restrict__ idx,
                                   const int64_t* __restrict__ levels, int64_t source,
                                   int64_t* __restrict__ parents) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // 32 vertices per warp step: lanes test their vertex, then the warp walks
  // each reached one
  for (int64_t base = w0 * 32; base < n; base += nw * 32) {
    const int64_t v = base + lane;
    const int64_t lv = v < n ? levels[v] : 0;
    if (v < n && lv == 0) parents[v] = -1;
    if (v == source) parents[v] = source;
    uint32_t todo = __ballot_sync(GB_FULL, v < n && lv > 1 && v != source);
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const int64_t vv = base + j;
      const int64_t want = __shfl_sync(GB_FULL, lv, j) - 1;
      const int64_t lo = off[vv], hi = off[vv + 1];
      int64_t found = -1;
      for (int64_t p0 = lo; p0 < hi && found < 0; p0 += 32) {
        const int64_t p = p0 + lane;
        const int32_t u = p < hi ? idx[p] : -1;
        const bool hit = u >= 0 && levels[u] == want;
        const uint32_t b = __ballot_sync(GB_FULL, hit);
        if (b) found = __shfl_sync(GB_FULL, u, __ffs(b) - 1);  // rows ascend: min id
      }
      if (lane == 0) parents[vv] = found;  // -1 only for an inconsistent level vector
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
