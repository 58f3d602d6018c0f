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

}  // namespace gb

using namespace gb;

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
