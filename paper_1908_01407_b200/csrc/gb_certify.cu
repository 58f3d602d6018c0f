// Result certificates for the command-line harness's --verify (cli.py) --
// checks that prove a result correct from the graph alone, independent of the
// kernels that computed it (the reference verifies with separate pure-Python
// oracles, reference.py; this package has no CPU path).
//
//   gb_sssp_certify  distances are shortest paths iff dist[source] = 0, every
//                    stored edge (u, v, w) with dist[u] finite has
//                    dist[v] <= dist[u] + w, and every reached v != source
//                    has a tight in-edge (dist[v] == dist[u] + w); unreached
//                    vertices have no in-edge from a reached one.
//   gb_cc_certify    labels are the minimum-id component labels iff every
//                    stored edge joins equal labels, label[v] <= v,
//                    label[label[v]] == label[v] (the label is a member), and
//                    each class is connected -- the last is checked by the
//                    caller with BFS from chosen roots.
#include <math.h>

#include "gb_common.cuh"

namespace gb {

__device__ __forceinline__ double cert_weight(const void* vals, int dtype, double iso, int64_t p) {
  if (!vals) return iso;
  return dtype == GB_I64 ? (double)((const long long*)vals)[p] : ((const double*)vals)[p];
}

// rows of `in` are in-edges: row v lists u with (u, v) stored
__global__ void sssp_cert_kernel(int64_t n, const int64_t* __restrict__ off,
                                 const int32_t* __restrict__ idx, const void* vals, int dtype,
                                 double iso, const double* __restrict__ dist, int64_t source,
                                 unsigned long long* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long relaxable = 0, untight = 0;
  for (int64_t v = w0; v < n; v += nw) {
    const double dv = dist[v];
    bool tight = false;
    for (int64_t p = off[v] + lane; p < off[v + 1]; p += 32) {
      const double du = dist[idx[p]];
      if (!isinf(du)) {
        const double c = du + cert_weight(vals, dtype, iso, p);
        relaxable += c < dv;          // an edge that would still improve v
        tight |= c == dv;
      }
    }
    tight = __any_sync(GB_FULL, tight);
    if (lane == 0 && v != source && !isinf(dv) && !tight) ++untight;
  }
  relaxable = (unsigned long long)warp_sum_ll((long long)relaxable);
  if (lane == 0) {
    if (relaxable) atomicAdd(err + 1, relaxable);
    if (untight) atomicAdd(err + 2, untight);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && dist[source] != 0.0) atomicAdd(err + 0, 1ull);
}

__global__ void cc_cert_kernel(int64_t n, const int64_t* __restrict__ off,
                               const int32_t* __restrict__ idx, const int64_t* __restrict__ lab,
                               unsigned long long* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long cross = 0, bad = 0;
  for (int64_t v = w0; v < n; v += nw) {
    const int64_t l = lab[v];
    if (lane == 0) bad += !(l >= 0 && l <= v && lab[l] == l);
    for (int64_t p = off[v] + lane; p < off[v + 1]; p += 32) cross += lab[idx[p]] != l;
  }
  cross = (unsigned long long)warp_sum_ll((long long)cross);
  if (lane == 0) {
    if (bad) atomicAdd(err + 0, bad);
    if (cross) atomicAdd(err + 1, cross);
  }
}

}  // namespace gb

using namespace gb;

extern "C" {

gb_status gb_sssp_certify(gb_ctx* ctx, const gb_csr* in_edges, int64_t source, const double* dist,
                          int64_t* errors_host) {
  const int64_t n = in_edges->nrows;
  for (int i = 0; i < 3; ++i) errors_host[i] = 0;
  if (n == 0) return GB_OK;
  if (source < 0 || source >= n) return set_error(ctx, GB_ERR_INDEX, "source out of range");
  cudaStream_t s = stream_of(ctx);
  Arena ar(ctx);
  unsigned long long* err = ar.alloc<unsigned long long>(3);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(err, 0, 24, s));
  sssp_cert_kernel<<<grid_for(ctx, n * 32, 256, 8), 256, 0, s>>>(
      n, in_edges->offsets, in_edges->indices, in_edges->values, in_edges->dtype,
      in_edges->iso_f64, dist, source, err);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 2);
  return read_i64(ctx, (const int64_t*)err, errors_host, 3);
}

gb_status gb_cc_certify(gb_ctx* ctx, const gb_csr* a, const int64_t* labels,
                        int64_t* errors_host) {
  const int64_t n = a->nrows;
  errors_host[0] = errors_host[1] = 0;
  if (n == 0) return GB_OK;
  cudaStream_t s = stream_of(ctx);
  Arena ar(ctx);
  unsigned long long* err = ar.alloc<unsigned long long>(2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(err, 0, 16, s));
  cc_cert_kernel<<<grid_for(ctx, n * 32, 256, 8), 256, 0, s>>>(n, a->offsets, a->indices, labels,
                                                               err);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 2);
  return read_i64(ctx, (const int64_t*)err, errors_host, 2);
}

}  // extern "C"
