// Small-graph BFS in ONE cooperative kernel (algorithms.py:48-77 with the
// reference direction rule, kernels.py:108-126).
//
// On a small graph a BFS is a few microseconds of work per level, and the
// device-graph loop's per-level cost -- a SWITCH node, the degree scan, the
// expansion, the bitmap finalize, the step kernel -- dominates (R-MAT s16:
// ~25 us per level).  Here a level is one grid-wide barrier inside one
// resident grid: the level's multiply (push: warps over the frontier
// entries' lists mark and append; pull: a thread per unvisited vertex scans
// its in-edges until a frontier vertex) while the buffers of the level after
// next are cleared.  Every thread computes the same decision from the same
// frontier size; thread 0 logs it.  The graph is the degree-ordered layout
// the default bfs() uses (`rank` maps original ids to new ones); levels are
// kept by new id and written by original id at the end, like bfs_unpermute.
#include <cooperative_groups.h>

#include "gb_common.cuh"

namespace cg = cooperative_groups;

namespace gb {

struct CoopBfs {
  int64_t n, nnz, source, cap;
  double ratio;
  int32_t policy, pad_;
  const int64_t *poff, *qoff;       // push rows (out-edges), pull rows (in-edges)
  const int32_t *pidx, *qidx;
  const void *pval, *qval;          // stored values (an edge with value 0 is absent), or NULL
  int32_t pdtype, qdtype;
  const uint32_t* nonempty;         // pull rows with >= 1 entry
  const int32_t* rank;              // original id -> new id
  uint32_t *vbm, *fbm[3];           // visited; frontier bitmaps, rotating by level
  int32_t *F[2], *lv;
  unsigned long long* cnt;          // [3]: list sizes, rotating by level
  int64_t* log;                     // [iters, (dir, K, est) x iters]
  int64_t* out;                     // levels by original id
};

__device__ __forceinline__ bool coop_on(const void* vals, int dtype, int64_t p) {
  if (!vals) return true;
  return dtype == GB_I64 ? ((const long long*)vals)[p] != 0 : ((const double*)vals)[p] != 0.0;
}

// append a warp's discoveries to the next frontier list (one atomic per warp)
__device__ __forceinline__ void coop_append(bool disc, int32_t v, unsigned long long* cn,
                                            int32_t* Fn) {
  const int lane = threadIdx.x & 31;
  const uint32_t bal = __ballot_sync(GB_FULL, disc);
  if (bal) {
    unsigned long long at = 0;
    if (lane == 0) at = atomicAdd(cn, (unsigned long long)__popc(bal));
    at = __shfl_sync(GB_FULL, at, 0);
    if (disc) Fn[at + __popc(bal & ((1u << lane) - 1u))] = v;
  }
}

// Level L reads frontier bitmap L%3 and list L%2, writes bitmap (L+1)%3 and
// list (L+1)%2, and clears bitmap / counter (L+2)%3 -- last read during level
// L-1 -- so ONE grid barrier separates two levels.
__global__ void __launch_bounds__(1024, 1) bfs_coop_kernel(CoopBfs a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int64_t gw = tid >> 5, nwarps = nth >> 5;
  const int64_t n = a.n, W = (n + 31) / 32;
  for (int64_t i = tid; i < W; i += nth) a.vbm[i] = a.fbm[0][i] = a.fbm[1][i] = a.fbm[2][i] = 0;
  for (int64_t i = tid; i < n; i += nth) a.lv[i] = 0;
  if (tid < 3) a.cnt[tid] = 0;
  grid.sync();
  const int32_t s = a.rank[a.source];
  if (tid == 0) {
    a.lv[s] = 1;
    a.vbm[s >> 5] |= 1u << (s & 31);
    a.fbm[0][s >> 5] |= 1u << (s & 31);
    a.F[0][0] = s;
  }
  grid.sync();
  const double d = n ? (double)a.nnz / (double)n : 0.0;
  int64_t K = 1, iters = 0;
  bool unstamp = false;
  for (int64_t it = 0; it < a.cap; ++it) {
    const int64_t est = (int64_t)rint(d * (double)K);  // Python round: half-even
    int32_t dir = (double)est > (double)a.nnz * a.ratio ? GB_DIR_PULL : GB_DIR_PUSH;
    if (a.policy == GB_DIR_PUSH) dir = GB_DIR_PUSH;
    if (a.policy == GB_DIR_PULL) dir = GB_DIR_PULL;
    if (tid == 0) {
      a.log[1 + 3 * it] = dir;
      a.log[2 + 3 * it] = K;
      a.log[3 + 3 * it] = est;
      a.cnt[(it + 2) % 3] = 0;
    }
    iters = it + 1;
    const int32_t* Fc = a.F[it & 1];
    int32_t* Fn = a.F[(it + 1) & 1];
    const uint32_t* fc = a.fbm[it % 3];
    uint32_t* fn = a.fbm[(it + 1) % 3];
    uint32_t* fz = a.fbm[(it + 2) % 3];
    unsigned long long* cn = a.cnt + (it + 1) % 3;
    const int32_t lvl = (int32_t)(it + 2);
    for (int64_t i = tid; i < W; i += nth) fz[i] = 0;
    if (dir == GB_DIR_PUSH) {
      // a warp per frontier entry; fewer entries than warps (the source's
      // level): several warps share an entry's list
      const int64_t wpe = K < nwarps ? nwarps / K : 1;
      for (int64_t t = gw; t < K * wpe; t += nwarps) {
        const int64_t k = t / wpe, part = t % wpe;
        const int32_t u = Fc[k];
        const int64_t hi = a.poff[u + 1];
        for (int64_t p0 = a.poff[u] + 32 * part; p0 < hi; p0 += 32 * wpe) {
          const int64_t p = p0 + lane;
          bool disc = false;
          int32_t v = 0;
          if (p < hi && coop_on(a.pval, a.pdtype, p)) {
            v = a.pidx[p];
            const uint32_t bit = 1u << (v & 31);
            if (!(ld_probe(a.vbm + (v >> 5)) & bit) && !(atomicOr(a.vbm + (v >> 5), bit) & bit)) {
              disc = true;
              a.lv[v] = lvl;
              atomicOr(fn + (v >> 5), bit);
            }
          }
          coop_append(disc, v, cn, Fn);
        }
      }
    } else {
      // a thread per unvisited vertex: its in-edges until a frontier vertex
      for (int64_t vb = tid - lane; vb < n; vb += nth) {
        const int64_t v = vb + lane;
        bool disc = false;
        if (v < n) {
          const uint32_t bit = 1u << (v & 31);
          if (!(a.vbm[v >> 5] & bit) && (a.nonempty[v >> 5] & bit)) {
            for (int64_t p = a.qoff[v]; p < a.qoff[v + 1]; ++p) {
              const int32_t j = a.qidx[p];
              if (((fc[j >> 5] >> (j & 31)) & 1u) && coop_on(a.qval, a.qdtype, p)) {
                disc = true;
                break;
              }
            }
          }
          if (disc) {
            atomicOr(a.vbm + (v >> 5), bit);
            atomicOr(fn + (v >> 5), bit);
            a.lv[v] = lvl;
          }
        }
        coop_append(disc, (int32_t)v, cn, Fn);
      }
    }
    grid.sync();
    const int64_t Kn = (int64_t)*cn;
    if (Kn == 0) break;
    K = Kn;
    if (it + 1 == a.cap) unstamp = true;  // the reference stamps a frontier one iteration later
  }
  if (unstamp)
    for (int64_t i = tid; i < K; i += nth) a.lv[a.F[iters & 1][i]] = 0;
  grid.sync();
  for (int64_t i = tid; i < n; i += nth) a.out[i] = a.lv[a.rank[i]];
  if (tid == 0) a.log[0] = iters;
}

struct CoopBuf {
  int64_t n = 0;
  void* mem = nullptr;
  uint32_t *vbm, *fbm[3];
  int32_t *F[2], *lv;
  unsigned long long* cnt;
};

static void coop_free(void* p) {
  auto* b = static_cast<CoopBuf*>(p);
  if (b->mem) cudaFree(b->mem);
  delete b;
}

// 0: off, else the largest n the cooperative kernel takes (GB_BFS_COOP_N,
// gb_bfs_coop_max_n)
static int64_t g_coop_max_n = -1;
int64_t bfs_coop_max_n() {
  if (g_coop_max_n < 0) {
    const char* e = getenv("GB_BFS_COOP_N");
    g_coop_max_n = e ? atoll(e) : ((int64_t)1 << 18);
  }
  return g_coop_max_n;
}

gb_status bfs_coop_run(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull,
                       const uint32_t* nonempty, const int32_t* rank, int64_t source,
                       int64_t cap, double ratio, int32_t policy, int64_t* levels,
                       int64_t* log_dev) {
  const int64_t n = push->nrows;
  void** slot = ctx_slot(ctx, SLOT_BFS_COOP, coop_free);
  CoopBuf* B = static_cast<CoopBuf*>(*slot);
  cudaStream_t s = stream_of(ctx);
  if (B && B->n < n) {
    cudaStreamSynchronize(s);
    coop_free(B);
    *slot = B = nullptr;
  }
  if (!B) {
    B = new CoopBuf();
    B->n = n;
    const int64_t W = (n + 31) / 32;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += (b + 255) / 256 * 256; return o; };
    const size_t o_v = take(4 * W), o_f0 = take(4 * W), o_f1 = take(4 * W), o_f2 = take(4 * W);
    const size_t o_F0 = take(4 * n), o_F1 = take(4 * n), o_lv = take(4 * n), o_c = take(24);
    if (cudaMalloc(&B->mem, off) != cudaSuccess) {
      cudaGetLastError();
      delete B;
      return GB_ERR_UNSUPPORTED;
    }
    char* m = static_cast<char*>(B->mem);
    B->vbm = (uint32_t*)(m + o_v);
    B->fbm[0] = (uint32_t*)(m + o_f0);
    B->fbm[1] = (uint32_t*)(m + o_f1);
    B->fbm[2] = (uint32_t*)(m + o_f2);
    B->F[0] = (int32_t*)(m + o_F0);
    B->F[1] = (int32_t*)(m + o_F1);
    B->lv = (int32_t*)(m + o_lv);
    B->cnt = (unsigned long long*)(m + o_c);
    *slot = B;
  }
  CoopBfs a;
  a.n = n;
  a.nnz = push->nnz;
  a.source = source;
  a.cap = cap;
  a.ratio = ratio;
  a.policy = policy;
  a.pad_ = 0;
  a.poff = push->offsets;
  a.pidx = push->indices;
  a.pval = push->values;
  a.pdtype = push->dtype;
  a.qoff = pull->offsets;
  a.qidx = pull->indices;
  a.qval = pull->values;
  a.qdtype = pull->dtype;
  a.nonempty = nonempty;
  a.rank = rank;
  a.vbm = B->vbm;
  a.fbm[0] = B->fbm[0];
  a.fbm[1] = B->fbm[1];
  a.fbm[2] = B->fbm[2];
  a.F[0] = B->F[0];
  a.F[1] = B->F[1];
  a.lv = B->lv;
  a.cnt = B->cnt;
  a.log = log_dev;
  a.out = levels;
  int per_sm = 0;
  GB_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_coop_kernel, 1024, 0));
  if (per_sm < 1) return GB_ERR_UNSUPPORTED;
  // one 1024-thread block per SM: the levels are small, a barrier costs per block
  const int grid = sm_count(ctx);
  void* args[] = {&a};
  GB_CUDA(ctx, cudaLaunchCooperativeKernel((void*)bfs_coop_kernel, grid, 1024, args, 0, s));
  count_launch(ctx, 1);
  return GB_OK;
}

}  // namespace gb

extern "C" int64_t gb_bfs_coop_max_n(int64_t n) {
  const int64_t prev = gb::bfs_coop_max_n();
  if (n >= 0) gb::g_coop_max_n = n;
  return prev;
}
