#include <cstdio>
#include <cuda_runtime.h>
__global__ void setk(cudaGraphConditionalHandle h, int v) { cudaGraphSetConditional(h, v); }
__global__ void mark(int* p, int v) { *p = v; }
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s failed: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
int main() {
  int* d; CK(cudaMalloc(&d, 4)); CK(cudaMemset(d, 0, 4));
  cudaStream_t s; CK(cudaStreamCreate(&s));
  cudaGraph_t top; CK(cudaGraphCreate(&top, 0));
  // handle h2 created in TOP, used by an IF node inside the body of an IF node in TOP
  cudaGraphConditionalHandle h1, h2;
  CK(cudaGraphConditionalHandleCreate(&h1, top, 1, cudaGraphCondAssignDefault));
  CK(cudaGraphConditionalHandleCreate(&h2, top, 0, cudaGraphCondAssignDefault));
  // kernel in top sets h2 = 1
  CK(cudaStreamBeginCaptureToGraph(s, top, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  setk<<<1,1,0,s>>>(h2, 1);
  CK(cudaStreamEndCapture(s, &top));
  cudaGraphNode_t k0; size_t nn = 0; CK(cudaGraphGetNodes(top, nullptr, &nn));
  cudaGraphNode_t nodes[4]; nn = 4; CK(cudaGraphGetNodes(top, nodes, &nn)); k0 = nodes[0];
  cudaGraphNodeParams p = {}; p.type = cudaGraphNodeTypeConditional; p.conditional.handle = h1;
  p.conditional.type = cudaGraphCondTypeIf; p.conditional.size = 1;
  cudaGraphNode_t c1; CK(cudaGraphAddNode(&c1, top, &k0, 1, &p));
  cudaGraph_t b1 = p.conditional.phGraph_out[0];
  cudaGraphNodeParams p2 = {}; p2.type = cudaGraphNodeTypeConditional; p2.conditional.handle = h2;
  p2.conditional.type = cudaGraphCondTypeIf; p2.conditional.size = 1;
  cudaGraphNode_t c2; cudaError_t e = cudaGraphAddNode(&c2, b1, nullptr, 0, &p2);
  printf("add nested IF with parent handle: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 0;
  cudaGraph_t b2 = p2.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(s, b2, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  mark<<<1,1,0,s>>>(d, 7);
  cudaGraph_t o2 = b2; CK(cudaStreamEndCapture(s, &o2));
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, top, 0);
  printf("instantiate: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 0;
  CK(cudaGraphLaunch(ex, s)); CK(cudaStreamSynchronize(s));
  int h = 0; CK(cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost));
  printf("result %d (7 = nested IF ran on a handle set by a parent-graph kernel)\n", h);
  return 0;
}
