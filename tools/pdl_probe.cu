// Does programmatic dependent launch (PDL) work inside a CUDA-graph WHILE
// body, and what does it save per dependent kernel?  A WHILE node whose body
// is a chain of K small kernels (148 x 256 threads, one load/store each) and a
// one-thread step; the chain launched plainly or with the programmatic
// stream-serialization attribute (each kernel waits with griddepcontrol.wait
// before touching memory).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_step(int* x, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] += 1;
}

__global__ void k_loop(int* ctr, cudaGraphConditionalHandle h) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int c = --*ctr;
  cudaGraphSetConditional(h, c > 0 ? 1u : 0u);
}

static void launch(bool pdl, void (*k)(int*, int), dim3 g, dim3 b, cudaStream_t s, int* x, int n) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? at : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, x, n);
}

static float run(bool pdl, int K, int iters) {
  int n = 148 * 256;
  int *x, *ctr;
  cudaMalloc(&x, n * 4);
  cudaMalloc(&ctr, 4);
  cudaMemset(x, 0, n * 4);
  cudaStream_t s, s2;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaGraph_t top;
  cudaGraphCreate(&top, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, top, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  cudaError_t e = cudaGraphAddNode(&node, top, nullptr, 0, &p);
  if (e) { printf("add node: %s\n", cudaGetErrorString(e)); return -1; }
  cudaGraph_t body = p.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(s2, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  if (e) { printf("capture: %s\n", cudaGetErrorString(e)); return -1; }
  for (int i = 0; i < K; ++i) launch(pdl, k_step, dim3(148), dim3(256), s2, x, n);
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(1);
    cfg.stream = s2;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? at : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_loop, ctr, h);
  }
  cudaGraph_t out = body;
  e = cudaStreamEndCapture(s2, &out);
  if (e) { printf("end capture: %s\n", cudaGetErrorString(e)); return -1; }
  cudaGraphExec_t ex;
  e = cudaGraphInstantiate(&ex, top, 0);
  if (e) { printf("instantiate (pdl=%d): %s\n", pdl, cudaGetErrorString(e)); return -1; }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemcpyAsync(ctr, &iters, 4, cudaMemcpyHostToDevice, s);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ex, s);
    cudaEventRecord(b, s);
    cudaStreamSynchronize(s);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  int h0 = 0;
  cudaMemcpy(&h0, x, 4, cudaMemcpyDeviceToHost);
  e = cudaGetLastError();
  printf("pdl=%d K=%d iters=%d: %.3f ms, %.2f us per kernel (x[0]=%d, %s)\n", pdl, K, iters, best,
         best * 1e3 / (iters * (K + 1)), h0, cudaGetErrorString(e));
  return best;
}

int main() {
  for (int pdl = 0; pdl < 2; ++pdl) run(pdl, 8, 200);
  for (int pdl = 0; pdl < 2; ++pdl) run(pdl, 8, 200);
  return 0;
}
