/* The drop-in boundary exercised from plain C, no Python and no PyTorch:
 * generate the reference's R-MAT graph on the GPU (gb_rmat_generate,
 * io.py:275-295), preprocess it into a CSR (gb_edges_to_csr, io.py:220-315),
 * run the fused BFS (gb_bfs, algorithms.py:48-77) and print one JSON line
 * (reached vertices, sum of levels, iterations, direction trace) that
 * tests/test_abi_c.py checks against the C oracle.
 *
 *   abi_bfs SCALE SOURCE */
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "graphblast.h"

#define CHECK(x)                                                              \
  do {                                                                        \
    gb_status s_ = (x);                                                       \
    if (s_ != GB_OK) {                                                        \
      fprintf(stderr, "%s failed (%d): %s\n", #x, s_, gb_last_error(ctx));   \
      return 1;                                                               \
    }                                                                         \
  } while (0)

int main(int argc, char** argv) {
  const int scale = argc > 1 ? atoi(argv[1]) : 14;
  const int64_t source = argc > 2 ? atoll(argv[2]) : 0;
  const int64_t n = (int64_t)1 << scale, m = (int64_t)16 << scale;
  gb_ctx* ctx = NULL;
  if (gb_ctx_create(0, &ctx) != GB_OK) {
    fprintf(stderr, "gb_ctx_create failed\n");
    return 1;
  }
  int32_t *src, *dst, *idx;
  int64_t *off, *levels;
  uint32_t* nonempty;
  if (cudaMalloc((void**)&src, 4 * m) || cudaMalloc((void**)&dst, 4 * m) ||
      cudaMalloc((void**)&idx, 8 * m) || cudaMalloc((void**)&off, 8 * (n + 1)) ||
      cudaMalloc((void**)&levels, 8 * n) || cudaMalloc((void**)&nonempty, 4 * ((n + 31) / 32))) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 1;
  }
  const double a = 0.57, b = 0.19, c = 0.19;
  CHECK(gb_rmat_generate(ctx, scale, m, 1, a, a + b, (a + b) + c, src, dst));
  int64_t nnz = 0;
  CHECK(gb_edges_to_csr(ctx, n, m, src, dst, 1, off, idx, &nnz));
  CHECK(gb_nonempty_rows(ctx, n, off, nonempty));
  gb_csr A = {0};
  A.nrows = A.ncols = n;
  A.nnz = nnz;
  A.offsets = off;
  A.indices = idx;
  A.values = NULL;
  A.dtype = GB_I64;
  A.iso_i64 = 1;
  A.iso_f64 = 1.0;
  A.gen = 1;
  enum { CAP = 64 };
  int32_t dirs[CAP];
  int64_t nv[CAP], est[CAP], iters = 0;
  /* symmetric: the push (rows = out-edges) and pull (rows = in-edges)
   * orientations are the same CSR */
  CHECK(gb_bfs(ctx, &A, &A, nonempty, source, CAP, 0.1, GB_DIR_AUTO, levels, dirs, nv, est,
               &iters));
  int64_t* h = (int64_t*)malloc(8 * n);
  cudaMemcpy(h, levels, 8 * n, cudaMemcpyDeviceToHost);
  long long reached = 0, sum = 0;
  for (int64_t i = 0; i < n; ++i) {
    reached += h[i] > 0;
    sum += h[i];
  }
  printf("{\"n\": %lld, \"nnz\": %lld, \"reached\": %lld, \"level_sum\": %lld, \"iters\": %lld, "
         "\"trace\": [", (long long)n, (long long)nnz, reached, sum, (long long)iters);
  for (int64_t i = 0; i < iters; ++i)
    printf("%s[\"%s\", %lld, %lld]", i ? ", " : "", dirs[i] == GB_DIR_PULL ? "pull" : "push",
           (long long)nv[i], (long long)est[i]);
  printf("]}\n");
  free(h);
  gb_ctx_destroy(ctx);
  return 0;
}
