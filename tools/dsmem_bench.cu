// Microbenchmark: random 4-byte probes of a 2 MB bitmap held (a) in global
// memory (L1/L2 path, what bfs_expand_warp does today) and (b) spread over
// the distributed shared memory of a 16-CTA cluster (128 KB per CTA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bench dsmem_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

constexpr int kWords = (2 << 20) / 4;  // 2 MB bitmap = 512K words
constexpr int kCluster = 16;
constexpr int kPerCta = kWords / kCluster;  // 32K words = 128 KB

__device__ __forceinline__ uint32_t lcg(uint32_t& s) {
  s = s * 1664525u + 1013904223u;
  return s;
}

__global__ void probe_global(const uint32_t* __restrict__ bm, int iters, uint32_t* out) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    uint32_t w[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t v = lcg(s) >> 8;  // 24-bit vertex id (16.8M vertices)
      asm volatile("ld.global.ca.b32 %0, [%1];" : "=r"(w[u]) : "l"(bm + (v >> 5)));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= w[u];
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void __cluster_dims__(kCluster, 1, 1) probe_dsmem(const uint32_t* __restrict__ bm,
                                                             int iters, uint32_t* out) {
  extern __shared__ uint32_t s_bm[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank();
  for (int i = threadIdx.x; i < kPerCta; i += blockDim.x) s_bm[i] = bm[rank * kPerCta + i];
  cluster.sync();
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    uint32_t w[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t v = lcg(s) >> 8;
      const uint32_t word = v >> 5;
      const uint32_t* remote = cluster.map_shared_rank(s_bm, word / kPerCta);
      w[u] = remote[word % kPerCta];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= w[u];
  }
  cluster.sync();
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  uint32_t *bm, *out;
  cudaMalloc(&bm, kWords * 4);
  cudaMalloc(&out, 4);
  cudaMemset(bm, 0x5a, kWords * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 256;
  // global: 8 blocks of 256 per SM
  {
    const int grid = sms * 8, block = 256;
    probe_global<<<grid, block>>>(bm, iters, out);
    cudaEventRecord(a);
    probe_global<<<grid, block>>>(bm, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double probes = (double)grid * block * iters * 8;
    printf("global L1/L2 probes: %.1f Gprobe/s (%.3f ms)\n", probes / ms / 1e6, ms);
  }
  {
    cudaFuncSetAttribute(probe_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(probe_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, kPerCta * 4);
    const int block = 1024;
    int clusters = sms / kCluster;
    const int grid = clusters * kCluster;
    probe_dsmem<<<grid, block, kPerCta * 4>>>(bm, iters, out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("dsmem launch error: %s\n", cudaGetErrorString(e));
    cudaEventRecord(a);
    probe_dsmem<<<grid, block, kPerCta * 4>>>(bm, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    e = cudaGetLastError();
    if (e != cudaSuccess) printf("dsmem run error: %s\n", cudaGetErrorString(e));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double probes = (double)grid * block * iters * 8;
    printf("DSMEM cluster-16 probes: %.1f Gprobe/s (%.3f ms) on %d SMs\n", probes / ms / 1e6, ms,
           grid);
  }
  return 0;
}
