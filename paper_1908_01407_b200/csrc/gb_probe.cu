// Measurement support: the random-probe ceiling the BFS push runs against.
//
// The level-2 push of a BFS at R-MAT s24 performs one 4-byte probe of the
// visited bitmap per frontier edge (324 M probes into 2 MB).  Its speed is
// set by how many such scattered loads the L1/L2 path completes per second,
// not by HBM bandwidth.  gb_probe_rate measures that ceiling on the running
// GPU: every thread issues 8 independent uniformly random ld.global.ca probes
// of a `words`-word bitmap per step (the same load the push uses), grid = all
// SMs at full occupancy.  bench.py reports the push against it next to the
// HBM roofline.
#include <cstdlib>

#include "gb_common.cuh"

namespace gb {

__global__ void __launch_bounds__(256)
probe_kernel(const uint32_t* __restrict__ bm, uint32_t nbits, int iters, uint32_t* sink) {
  uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    uint32_t w[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = s * 1664525u + 1013904223u;
      const uint32_t v = __umulhi(s, nbits);
      w[u] = ld_probe(bm + (v >> 5));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= w[u];
  }
  if (acc == 0x9e3779b9u) sink[0] = acc;
}

// The gather ceiling of a pull SpMV on a given matrix: stream the column
// indices (256-bit loads, as the pull kernels do) and gather x[col] for every
// stored entry with nothing else -- no rows, mask, fold or output.  Its rate
// (gathers/s) is what a pull kernel over the same column sequence can at
// best reach when the random 8-byte gathers, not HBM bandwidth, bound it.
__global__ void __launch_bounds__(256)
gather_replay_kernel(int64_t nnz, const int32_t* __restrict__ idx, const double* __restrict__ x,
                     double* sink) {
  double acc = 0.0;
  const int64_t groups = nnz / 8;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    int32_t c[8];
    ld_stream8(idx + 8 * g, c);
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ld_gather(x + c[k]);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k];
  }
  if (acc == -1.2345) sink[0] = acc;
}

// The same replay with lane-consecutive entries (lane l of a warp gathers
// entries 32k + l of the warp's 256-entry chunk): sorted neighbours of one
// row that share a 128-byte line of x coalesce into one L1 wavefront.
__global__ void __launch_bounds__(256)
gather_replay_consec(int64_t nnz, const int32_t* __restrict__ idx, const double* __restrict__ x,
                     double* sink) {
  double acc = 0.0;
  const int lane = threadIdx.x & 31;
  const int64_t chunks = nnz / 256;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g = w0; g < chunks; g += nw) {
    int32_t c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = ld_stream(idx + 256 * g + 32 * k + lane);
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ld_gather(x + c[k]);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k];
  }
  if (acc == -1.2345) sink[0] = acc;
}

}  // namespace gb

using namespace gb;

extern "C" gb_status gb_gather_replay_rate(gb_ctx* ctx, const gb_csr* a, const double* x,
                                           double* gathers_per_s_host) {
  cudaStream_t s = stream_of(ctx);
  Arena ar(ctx);
  double* sink = ar.alloc<double>(1);
  GB_ARENA_CHECK(ctx, ar);
  // lane-consecutive by default (the higher of the two rates, and the
  // mapping of the row-bin pull's long tiles); GB_REPLAY_CONSEC=0: strided
  const char* cm = getenv("GB_REPLAY_CONSEC");
  auto k = (cm && cm[0] == '0') ? gather_replay_kernel : gather_replay_consec;
  const int grid = resident_grid(ctx, k, 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<grid, 256, 0, s>>>(a->nnz, a->indices, x, sink);  // warm-up
  cudaEventRecord(e0, s);
  k<<<grid, 256, 0, s>>>(a->nnz, a->indices, x, sink);
  cudaEventRecord(e1, s);
  GB_LAUNCH_CHECK(ctx);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  count_launch(ctx, 2);
  *gathers_per_s_host = (double)(a->nnz / 8 * 8) / (ms * 1e-3);
  return GB_OK;
}

extern "C" gb_status gb_probe_rate(gb_ctx* ctx, int64_t words, int64_t min_probes,
                                   double* probes_per_s_host) {
  if (words < 1 || words > (int64_t)1 << 26) return set_error(ctx, GB_ERR_VALUE, "probe bitmap size");
  cudaStream_t s = stream_of(ctx);
  Arena ar(ctx);
  uint32_t* bm = ar.alloc<uint32_t>(words + 1);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(bm, 0x5a, sizeof(uint32_t) * (words + 1), s));
  const int grid = resident_grid(ctx, probe_kernel, 256);
  const int64_t per_step = (int64_t)grid * 256 * 8;
  const int iters = (int)((min_probes + per_step - 1) / per_step);
  const uint32_t nbits = (uint32_t)(words * 32 > 0xffffffffLL ? 0xffffffffLL : words * 32);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  probe_kernel<<<grid, 256, 0, s>>>(bm, nbits, iters, bm + words);  // warm-up
  cudaEventRecord(a, s);
  probe_kernel<<<grid, 256, 0, s>>>(bm, nbits, iters, bm + words);
  cudaEventRecord(b, s);
  GB_LAUNCH_CHECK(ctx);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  count_launch(ctx, 3);
  *probes_per_s_host = (double)per_step * iters / (ms * 1e-3);
  return GB_OK;
}
