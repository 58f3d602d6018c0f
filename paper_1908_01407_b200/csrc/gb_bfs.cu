// Fused direction-optimizing BFS: algorithms.py:48-77 with the dispatcher
// kernels.py:108-126 / 293-310 and both multiply kernels specialised to the
// LogicalOrAnd semiring with a complemented visited mask.
//
// Per level the reference does  assign(visited, depth, mask=f)  ->
// vxm(LogicalOrAnd, f, A, mask=~visited)  ->  reduce(Plus, f).  Here:
//   push level:  warp-tile expansion of the frontier list sets unvisited
//                neighbours' bits in the visited bitmap (probe, then
//                atomicOr), then bfs_finalize turns vbm & ~vprev into the
//                next frontier (bitmap + list + count) and stamps levels.
//   pull level:  bfs_pull walks in-edges of unvisited, non-isolated rows
//                (candidate lists per warp of 32 words) and stops at the
//                first frontier hit (early exit, kernels.py:169-178); it
//                writes the next frontier directly -- no separate finalize.
// The direction of every level follows the reference rule on the exact
// frontier count, so the direction trace equals the reference's.  The level
// loop runs on the device inside one CUDA graph (bfs_graph_run); the
// host-driven loop below it remains for per-kernel profiling and the
// 1D-partitioned steps.
#include <math.h>
#include <stddef.h>
#include <stdlib.h>

#include <vector>

#include "gb_common.cuh"
#include "gb_lbs.cuh"

#include <cub/cub.cuh>

namespace gb {

// A stored entry participates in LogicalAnd(a, u) iff a != 0.
struct EdgeOn {
  const void* vals;
  int dtype;
  __device__ __forceinline__ bool operator()(int64_t p) const {
    if (!vals) return true;
    return dtype == GB_I64 ? __ldg((const long long*)vals + p) != 0
                           : __ldg((const double*)vals + p) != 0.0;
  }
};

// ---------------------------------------------------------------------------
// push: load-balanced expansion of the frontier's out-edges
// ---------------------------------------------------------------------------
// Marking: the live visited bitmap `vbm` is probed through L1 (ld.ca: a stale
// clear bit only costs a redundant atomic) and a clear bit is set with one
// atomicOr, so a vertex reached by many frontier edges costs one read per edge
// but (almost) one write in total.  bfs_finalize recovers the new frontier as
// vbm & ~vprev.
__device__ __forceinline__ void mark(uint32_t* vbm, int32_t v, uint32_t word) {
  const uint32_t bit = 1u << (v & 31);
  red_or_if(!(word & bit), vbm + (v >> 5), bit);
}

// Warp-tile push expansion (no shared memory, no barriers): a batch of
// column loads is issued before any visited probe.
template <bool VALS>
struct PushBits {
  // 4 items per round trip in one/two-list tiles: 0.4-1.6 % less per s24
  // BFS than 8 on two boxes (0.783 -> 0.780, 0.785 -> 0.772 ms), 2: 0.85 ms
  // (tools/ab_push_batch2.sh, same box, alternating)
#ifndef GB_PUSH_TILE_BATCH
#define GB_PUSH_TILE_BATCH 4
#endif
  static constexpr int kTileBatch = GB_PUSH_TILE_BATCH;
  const int32_t* __restrict__ idx;
  EdgeOn on;
  uint32_t* __restrict__ vbm;
  int32_t xs = 0;  // vertices below xs are known visited: no probe (dense visited prefix)
  template <int B>
  __device__ __forceinline__ void probe_mark(const int32_t (&v)[B]) {
    uint32_t word[B];
#pragma unroll
    for (int r = 0; r < B; ++r) word[r] = v[r] >= xs && v[r] >= 0 ? ld_probe(vbm + (v[r] >> 5)) : ~0u;
#pragma unroll
    for (int r = 0; r < B; ++r) mark(vbm, v[r] >= 0 ? v[r] : 0, word[r]);  // dead: word = ~0
  }
  template <int B>
  __device__ __forceinline__ void batch(const int64_t (&p)[B], const bool (&live)[B]) {
    int32_t v[B];
#pragma unroll
    for (int r = 0; r < B; ++r) {
      v[r] = -1;
      if (live[r]) {
        const int32_t c = ld_stream(idx + p[r]);
        v[r] = (!VALS || on(p[r])) ? c : -1;
      }
    }
    probe_mark<B>(v);
  }
  // slots h + r*32 + lane of a tile inside one or two lists (warp_tiles):
  // positions are formed on the fly, no per-item 64-bit array
  template <int B>
  __device__ __forceinline__ void batch2(int64_t b0, int64_t b1, int32_t st1, int32_t rel_end,
                                         int32_t h) {
    const int32_t lane = threadIdx.x & 31;
    int32_t v[B];
#pragma unroll
    for (int r = 0; r < B; ++r) {
      const int32_t er = h + r * 32 + lane;
      const int64_t pos = (er >= st1 ? b1 : b0) + er;
      v[r] = -1;
      if (er < rel_end) {
        const int32_t c = ld_stream(idx + pos);
        v[r] = (!VALS || on(pos)) ? c : -1;
      }
    }
    probe_mark<B>(v);
  }
  __device__ __forceinline__ void visit(int64_t p) {
    const int32_t u = ld_stream(idx + p);
    if (!VALS || on(p)) mark(vbm, u, ld_probe(vbm + (u >> 5)));
  }
};

template <bool VALS, int MINB>
__global__ void __launch_bounds__(256, MINB)
bfs_expand_warp(DevI64 Kd, const int64_t* __restrict__ S, const int64_t* __restrict__ rowstart,
                const int32_t* __restrict__ tile_first, const int64_t* __restrict__ tile_base,
                const int32_t* __restrict__ idx,
                EdgeOn on, uint32_t* __restrict__ vbm, DevI64 Xd) {
  const int64_t K = Kd.get();
  PushBits<VALS> f{idx, on, vbm, (int32_t)Xd.get()};
  if (K > 0 && S[K] < 4 * K) {
    // short lists (s24 level 4: 844 K entries, 1.04 M edges): one thread per
    // frontier entry beats 512-slot tiles that each hold hundreds of entries
    // four entries per thread per pass: their bounds, first edges and probes
    // are each one batched round trip
    constexpr int B = 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += B * stride) {
      int64_t p0[B], d[B];
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const int64_t kk = k + j * stride;
        p0[j] = 0;
        d[j] = 0;
        if (kk < K) {
          p0[j] = rowstart[kk];
          d[j] = S[kk + 1] - S[kk];
        }
      }
      int32_t v[B];
#pragma unroll
      for (int j = 0; j < B; ++j) {
        v[j] = -1;
        if (d[j] > 0) {
          const int32_t c = ld_stream(idx + p0[j]);
          v[j] = (!VALS || on(p0[j])) ? c : -1;
        }
      }
      f.template probe_mark<B>(v);
#pragma unroll
      for (int j = 0; j < B; ++j)
        for (int64_t e = 1; e < d[j]; ++e) f.visit(p0[j] + e);
    }
    return;
  }
  warp_tiles(K, S, rowstart, tile_first, tile_base, f);
}

// (A variant that staged each single-list tile's column range in shared
// memory with a 1D bulk copy (cp.async.bulk + mbarrier) one tile ahead was
// built and measured: 0.73-0.76 ms against 0.49 ms for the level-2 push --
// the staging buffers take L1 away from the hot visited prefix and each warp
// waits on its own barrier; the column stream is not the exposed latency.)

using ExpandKernel = void (*)(DevI64, const int64_t*, const int64_t*, const int32_t*,
                              const int64_t*, const int32_t*, EdgeOn, uint32_t*, DevI64);

// How an ordered BFS uses the dense visited prefix X (every vertex below X is
// visited): 1 = cut each sorted list at X in the degree scan (fewer index
// loads, one lower-bound search per frontier entry), 2 = expand the whole
// list but do not probe targets below X, 0 = ignore it.  GB_PREFIX_MODE.
static int prefix_mode() {
  static const int m = getenv("GB_PREFIX_MODE") ? atoi(getenv("GB_PREFIX_MODE")) : 1;
  return m;
}
// Degree window [lo, hi] of the lists that mode 1 cuts (GB_CUT_LO / GB_CUT_HI);
// lists outside it are expanded whole.  Lists under 32 entries are not cut by
// default: their search costs about what expanding the few prefix edges does
// (s24: 0.885 vs 0.909 ms per BFS).
// GB_CUT_SAMPLES=0: plain binary search for the cut (no column samples)
static bool use_samples() {
  static const bool v = !(getenv("GB_CUT_SAMPLES") && atoi(getenv("GB_CUT_SAMPLES")) == 0);
  return v;
}
static int64_t cut_lo() {
  static const int64_t v = getenv("GB_CUT_LO") ? atoll(getenv("GB_CUT_LO")) : 32;
  return v > 1 ? v : 1;
}
static int64_t cut_hi() {
  static const int64_t v = getenv("GB_CUT_HI") ? atoll(getenv("GB_CUT_HI")) : INT64_MAX;
  return v;
}

// Register budget of the push (GB_PUSH_MINB = minimum resident CTAs of 256
// threads per SM: 1 leaves the allocation to ptxas, 3 allows 80, 4 caps at 64,
// 5 (default, 40 warps per SM, measured best) at 48, 6 at 40).
template <bool VALS>
static ExpandKernel expand_kernel() {
  static const int minb = getenv("GB_PUSH_MINB") ? atoi(getenv("GB_PUSH_MINB")) : 5;
  switch (minb) {
    case 1: return bfs_expand_warp<VALS, 1>;
    case 4: return bfs_expand_warp<VALS, 4>;
    case 5: return bfs_expand_warp<VALS, 5>;
    case 6: return bfs_expand_warp<VALS, 6>;
    case 3: return bfs_expand_warp<VALS, 3>;
    default: return bfs_expand_warp<VALS, 5>;
  }
}

// Push over a degree-ordered graph: the visited bits of the
// low-id prefix -- the vertices that receive almost every probe -- live in
// shared memory for the whole launch.  One persistent CTA per SM copies the
// level-start prefix (vprev) in, probes and marks it with shared-memory
// loads / atomics, and at the end ORs what it discovered into the global
// visited bitmap with one atomic per changed word.  Probes past the prefix
// take the global path of PushBits.  A CTA may mark a vertex another CTA
// already found; the global OR makes that harmless (finalize diffs against
// vprev).  Small levels skip the prefix copy (E below the break-even).
constexpr int kSmemPushThreads = 768;
constexpr int64_t kPrefixWordsMax = 49152;  // 192 KB: 1.57 M vertices

template <bool VALS>
struct PushBitsSmem {
  const int32_t* __restrict__ idx;
  EdgeOn on;
  uint32_t* __restrict__ vbm;
  uint32_t* sbm;
  int32_t pbits;  // vertices [0, pbits) are tracked in shared memory
  template <int B>
  __device__ __forceinline__ void batch(const int64_t (&p)[B], const bool (&live)[B]) {
    int32_t v[B];
#pragma unroll
    for (int r = 0; r < B; ++r) {
      v[r] = -1;
      if (live[r]) v[r] = ld_stream(idx + p[r]);
      if (VALS && v[r] >= 0 && !on(p[r])) v[r] = -1;
    }
    probe_mark<B>(v);
  }
  template <int B>
  __device__ __forceinline__ void batch2(int64_t b0, int64_t b1, int32_t st1, int32_t rel_end,
                                         int32_t h) {
    const int32_t lane = threadIdx.x & 31;
    int32_t v[B];
#pragma unroll
    for (int r = 0; r < B; ++r) {
      const int32_t er = h + r * 32 + lane;
      const int64_t pos = (er >= st1 ? b1 : b0) + er;
      v[r] = -1;
      if (er < rel_end) v[r] = ld_stream(idx + pos);
      if (VALS && v[r] >= 0 && !on(pos)) v[r] = -1;
    }
    probe_mark<B>(v);
  }
  // Branch-free per item: every item reads a shared word (word 0 when its
  // vertex is outside the prefix), only suffix items issue a global probe,
  // and the marks are predicated atomics -- no divergent regions.
  template <int B>
  __device__ __forceinline__ void probe_mark(const int32_t (&v)[B]) {
    uint32_t word[B];
#pragma unroll
    for (int r = 0; r < B; ++r) {
      const bool pre = (uint32_t)v[r] < (uint32_t)pbits;  // v = -1 is never in the prefix
      word[r] = sbm[pre ? (v[r] >> 5) : 0];
      if (v[r] >= pbits) word[r] = ld_probe(vbm + (v[r] >> 5));
    }
#pragma unroll
    for (int r = 0; r < B; ++r) {
      const uint32_t bit = 1u << (v[r] & 31);
      const bool clear = !(word[r] & bit);
      const int32_t w = v[r] >= 0 ? v[r] >> 5 : 0;
      red_or_shared_if(clear && (uint32_t)v[r] < (uint32_t)pbits, sbm + (w < pbits / 32 ? w : 0), bit);
      red_or_if(clear && v[r] >= pbits, vbm + w, bit);
    }
  }
  __device__ __forceinline__ void visit(int64_t p) {
    const int32_t u = ld_stream(idx + p);
    if (VALS && !on(p)) return;
    const uint32_t bit = 1u << (u & 31);
    if (u < pbits) {
      if (!(sbm[u >> 5] & bit)) atomicOr(sbm + (u >> 5), bit);
    } else if (!(ld_probe(vbm + (u >> 5)) & bit)) {
      atomicOr(vbm + (u >> 5), bit);
    }
  }
};

template <bool VALS>
__global__ void __launch_bounds__(kSmemPushThreads, 1)
bfs_expand_smem(DevI64 Kd, const int64_t* __restrict__ S, const int64_t* __restrict__ rowstart,
                const int32_t* __restrict__ tile_first, const int64_t* __restrict__ tile_base,
                const int32_t* __restrict__ idx,
                EdgeOn on, uint32_t* __restrict__ vbm, const uint32_t* __restrict__ vprev,
                int64_t W) {
  extern __shared__ uint32_t sbm[];
  const int64_t K = Kd.get();
  if (K <= 0) return;
  const int64_t E = S[K];
  const int64_t P = W < kPrefixWordsMax ? W : kPrefixWordsMax;
  // the prefix copy-in / flush costs ~P/2 vector accesses per CTA
  const bool use = E >= P * (int64_t)gridDim.x / 4;
  if (use) {
    for (int64_t w = threadIdx.x; w < P; w += blockDim.x) sbm[w] = __ldg(vprev + w);
    __syncthreads();
  }
  PushBitsSmem<VALS> f{idx, on, vbm, sbm, use ? (int32_t)(P * 32) : 0};
  warp_tiles(K, S, rowstart, tile_first, tile_base, f);
  if (use) {
    __syncthreads();
    for (int64_t w = threadIdx.x; w < P; w += blockDim.x) {
      const uint32_t d = sbm[w] & ~__ldg(vprev + w);
      if (d) atomicOr(vbm + w, d);
    }
  }
}

template <bool VALS>
static int smem_push_setup(gb_ctx* ctx, int64_t W, size_t* smem) {
  const int64_t P = W < kPrefixWordsMax ? W : kPrefixWordsMax;
  *smem = (size_t)P * 4;
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(bfs_expand_smem<VALS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(kPrefixWordsMax * 4));
    done = true;
  }
  return sm_count(ctx);
}

// levels of the original vertex ids from a run over the relabelled graph:
// vertex i is new vertex rank[i]; the internal levels are cleared at the start
// of each run, so unvisited vertices read 0.  s24: ~50 us, the same with no
// gathers at all -- the 67 MB rank read + 134 MB int64 write stream at
// ~3.9 TB/s whatever the store flavour or grid (measured).
// Vertices without in-edges are never reached (only the source is): in the
// degree order they are the ids >= limit, read as 0 without a gather (47 %
// of R-MAT vertices are isolated).
template <class LT>
__global__ void bfs_unpermute(int64_t n, const int32_t* __restrict__ rank,
                              const LT* __restrict__ lv, int64_t limit, DevI64 srank_d,
                              DevP64 out_d) {
  int64_t* __restrict__ out = out_d.get();
  const int64_t srank = srank_d.get();
  // 8 vertices per thread, every load of the group in flight at once
  // (one vertex at a time leaves the loop latency-bound at ~3.4 TB/s)
  const bool aligned = ((reinterpret_cast<uintptr_t>(rank) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const int64_t n8 = aligned ? n / 8 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int4* r4 = reinterpret_cast<const int4*>(rank);
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int4 ra = make_int4(0, 0, 0, 0), rb = ra;
  if (g < n8) {
    ra = __ldcs(r4 + 2 * g);
    rb = __ldcs(r4 + 2 * g + 1);
  }
  for (; g < n8; g += stride) {
    // the next group's ranks are in flight while this group gathers
    int4 na = ra, nb = rb;
    if (g + stride < n8) {
      na = __ldcs(r4 + 2 * (g + stride));
      nb = __ldcs(r4 + 2 * (g + stride) + 1);
    }
    const int32_t r[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
    ra = na;
    rb = nb;
    int64_t l[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      l[j] = (r[j] < limit || r[j] == srank) ? (int64_t)lv[r[j]] : 0;
    longlong2* o = reinterpret_cast<longlong2*>(out + 8 * g);
#pragma unroll
    for (int j = 0; j < 4; ++j) __stcs(o + j, make_longlong2(l[2 * j], l[2 * j + 1]));
  }
  for (int64_t i = 8 * n8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rank[i];
    out[i] = (r < limit || r == srank) ? (int64_t)lv[r] : 0;
  }
}

// first vertex without in-edges of a degree-ordered graph (in-degrees are
// non-increasing in the new ids): lower bound of nnz in the pull offsets
__global__ void reach_limit(int64_t n, const int64_t* __restrict__ off, int64_t* out) {
  int64_t lo = 0, hi = n;  // off[hi] == nnz
  const int64_t nnz = off[n];
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (off[m] < nnz) lo = m + 1; else hi = m;
  }
  *out = lo;
}

// (Scattering instead -- new id r in order, out[order[r]] -- measured 3.7x
// slower at s24: 16.8 M scattered 8-byte writes cost more than gathers.)

template <class LT>
__global__ void bfs_init(int64_t source, LT* levels, uint32_t* vbm, uint32_t* vprev,
                         uint32_t* fbm, int32_t* F) {
  levels[source] = 1;
  vbm[source >> 5] |= 1u << (source & 31);
  vprev[source >> 5] |= 1u << (source & 31);
  fbm[source >> 5] |= 1u << (source & 31);
  F[0] = (int32_t)source;
}

// Warp per 32 words (1024 vertices): lane l diffs word w0+l of the live
// visited bitmap against the level-start snapshot, then the warp walks the
// non-empty words so level stamps and frontier-list writes are coalesced.
// Dense visited prefix: xmin (when given) receives, via one atomicMin per
// block, 32 x the index of the first visited-bitmap word that is not full
// after this level -- every vertex below it is visited.  wmin is the calling
// warp's candidate (groups are walked in increasing order per warp).
__device__ __forceinline__ void prefix_note(int64_t* wmin, int64_t g, uint32_t visited_after,
                                            bool valid) {
  const uint32_t nf = __ballot_sync(GB_FULL, valid && visited_after != ~0u);
  if (nf && *wmin == INT64_MAX) *wmin = (g * 32 + __ffs(nf) - 1) * 32;
}
__device__ __forceinline__ void prefix_flush(int64_t wmin, unsigned long long* xmin) {
  __shared__ unsigned long long s_min;
  if (threadIdx.x == 0) s_min = ~0ull;
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && wmin != INT64_MAX) atomicMin(&s_min, (unsigned long long)wmin);
  __syncthreads();
  if (threadIdx.x == 0 && s_min != ~0ull) atomicMin(xmin, s_min);
}

// The level stored for a vertex: 16-bit levels (relabelled runs) saturate at
// 65535; a run that deep is redone with int32 levels (bfs_run).
template <class LT>
__device__ __forceinline__ LT level_of(int64_t depth) {
  if constexpr (sizeof(LT) == 2) return (LT)(depth < 65535 ? depth : 65535);
  else return (LT)depth;
}
// a relabelled run of this many levels is redone with int32 internal levels;
// loop caps up to it cannot saturate (the asynchronous entry relies on that)
constexpr int64_t kNarrowLevelIters = 65000;

constexpr int kFinalizeWarps = 8;  // finalize blocks are 256 threads

// LT: int64 levels (the API vector) or 16-bit levels (a relabelled run; int32
// when it is deeper than kNarrowLevelIters levels)
template <class LT>
__device__ __forceinline__ void finalize_body(int64_t n, int64_t depth, uint32_t* vbm,
                                              uint32_t* vprev, uint32_t* fbm_next,
                                              LT* levels, int32_t* F,
                                              unsigned long long* count, const uint32_t* xbm,
                                              unsigned long long* xmin = nullptr) {
  // xbm == NULL: new frontier = vbm & ~vprev (single GPU).  xbm != NULL: the
  // all-reduced new-frontier bitmap of a 1D-partitioned run is authoritative.
  // The block walks 8 groups per step and reserves their frontier-list
  // slots with ONE atomic (one per warp-group put ~16 K same-address atomics
  // on the counter at s24 levels 1-2).
  __shared__ unsigned long long s_base;
  __shared__ int s_tot[kFinalizeWarps + 1];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  int64_t wmin = INT64_MAX;
  const int64_t W = (n + 31) / 32;
  const int64_t G = (W + 31) / 32;
  for (int64_t gb = (int64_t)blockIdx.x * kFinalizeWarps; gb < G;
       gb += (int64_t)gridDim.x * kFinalizeWarps) {
    const int64_t g = gb + wid;
    const int64_t w = g * 32 + lane;
    uint32_t bits = 0, visited = ~0u;
    if (w < W) {
      if (xbm) {
        bits = xbm[w];
        const uint32_t cur = vbm[w] | bits;
        if (bits) {
          vbm[w] = cur;
          vprev[w] |= bits;
        }
        visited = cur;
      } else {
        const uint32_t cur = vbm[w], old = vprev[w];
        bits = cur & ~old;
        if (bits) vprev[w] = cur;
        visited = cur;
      }
      fbm_next[w] = bits;
    }
    if (xmin) prefix_note(&wmin, g, visited, w < W);
    // frontier list slots for the whole group, in word order
    const int c = __popc(bits);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(GB_FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(GB_FULL, incl, 31);
    if (lane == 31) s_tot[wid] = total;
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int i = 0; i < kFinalizeWarps; ++i) {
        const int t = s_tot[i];
        s_tot[i] = run;
        run += t;
      }
      s_base = run ? atomicAdd(count, (unsigned long long)run) : 0ull;
    }
    __syncthreads();
    const unsigned long long base = s_base + (unsigned long long)s_tot[wid];
    uint32_t nonzero = __ballot_sync(GB_FULL, bits != 0);
    while (nonzero) {
      const int j = __ffs(nonzero) - 1;
      nonzero &= nonzero - 1;
      const uint32_t wb = __shfl_sync(GB_FULL, bits, j);
      const int start = __shfl_sync(GB_FULL, incl - c, j);
      if ((wb >> lane) & 1u) {
        const int64_t v = (g * 32 + j) * 32 + lane;
        levels[v] = level_of<LT>(depth);
        F[base + start + __popc(wb & ((1u << lane) - 1u))] = (int32_t)v;
      }
    }
  }
  if (xmin) prefix_flush(wmin, xmin);
}

template <class LT>
__global__ void __launch_bounds__(256)
bfs_finalize(int64_t n, DevI64 depth_d, uint32_t* __restrict__ vbm,
             uint32_t* __restrict__ vprev, uint32_t* __restrict__ fbm_next,
             DevP<LT> levels_d, int32_t* __restrict__ F,
             unsigned long long* __restrict__ count,
             unsigned long long* __restrict__ count_clear, const uint32_t* __restrict__ xbm,
             unsigned long long* __restrict__ xmin) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *count_clear = 0;
  finalize_body(n, depth_d.get(), vbm, vprev, fbm_next, levels_d.get(), F, count, xbm, xmin);
}

// ---------------------------------------------------------------------------
// pull: warp per 32 words; candidate rows are compacted into a shared list
// and processed 8 per lane with their first loads batched
// ---------------------------------------------------------------------------
constexpr int kPullBatch = 8;                // rows per lane per pass
constexpr int kPullList = 32 * kPullBatch;   // rows per warp per pass
constexpr int kPullSerial = 8;               // entries a lane scans alone before the warp helps

// The frontier bitmap is probed through L1 (ld.global.ca).
template <class LT>
__device__ __forceinline__ void pull_body(int64_t n, int64_t depth, const int64_t* __restrict__ off,
                                          const int32_t* __restrict__ idx, EdgeOn on,
                                          const uint32_t* __restrict__ nonempty, uint32_t* vbm,
                                          uint32_t* vprev, const uint32_t* fbm, uint32_t* fbm_next,
                                          LT* levels, int32_t* F, unsigned long long* count,
                                          int64_t g_lo, int64_t g_hi,
                                          unsigned long long* xmin = nullptr) {
  // [g_lo, g_hi): groups of 32 words (1024 vertices) this launch owns; a
  // 1D-partitioned rank passes its vertex block with `off`/`nonempty`
  // pointers rebased so global vertex ids index them directly.
  __shared__ int32_t s_list[8][kPullList];
  __shared__ uint32_t s_new[8][32];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int64_t W = (n + 31) / 32;
  const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int32_t* list = s_list[wid];
  uint32_t* nw = s_new[wid];
  int64_t wmin = INT64_MAX;
  for (int64_t g = g_lo + g0; g < g_hi; g += ng) {
    const int64_t w = g * 32 + lane;
    const uint32_t vb0 = w < W ? vbm[w] : ~0u;
    uint32_t rem = w < W ? (~vb0 & __ldg(nonempty + w)) : 0u;
    nw[lane] = 0;
    __syncwarp();
    while (true) {
      const int c = __popc(rem);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(GB_FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const int total = __shfl_sync(GB_FULL, incl, 31);
      if (total == 0) break;
      int slot = incl - c;
      while (rem && slot < kPullList) {
        const int b = __ffs(rem) - 1;
        rem &= rem - 1;
        list[slot++] = (int32_t)(w * 32 + b);
      }
      __syncwarp();
      const int take = total < kPullList ? total : kPullList;
      int64_t lo[kPullBatch], hi[kPullBatch];
      int32_t v[kPullBatch];
#pragma unroll
      for (int r = 0; r < kPullBatch; ++r) {
        const int q = r * 32 + lane;
        v[r] = q < take ? list[q] : -1;
        lo[r] = hi[r] = 0;
        if (v[r] >= 0) {
          lo[r] = __ldg(off + v[r]);
          hi[r] = __ldg(off + v[r] + 1);
        }
      }
      int32_t j0[kPullBatch];
#pragma unroll
      for (int r = 0; r < kPullBatch; ++r) j0[r] = lo[r] < hi[r] ? __ldg(idx + lo[r]) : 0;
      uint32_t todo = 0;
#pragma unroll
      for (int r = 0; r < kPullBatch; ++r) {
        bool hit = false;
        if (lo[r] < hi[r]) {
          hit = ((ld_probe(fbm + (j0[r] >> 5)) >> (j0[r] & 31)) & 1u) && on(lo[r]);
          int64_t p = lo[r] + 1;
          const int64_t stop = lo[r] + kPullSerial < hi[r] ? lo[r] + kPullSerial : hi[r];
          for (; !hit && p < stop; ++p) {
            const int32_t j = __ldg(idx + p);
            hit = ((ld_probe(fbm + (j >> 5)) >> (j & 31)) & 1u) && on(p);
          }
          lo[r] = p;
          if (!hit && p < hi[r]) todo |= 1u << r;
        }
        if (hit) {
          atomicOr(&nw[(v[r] >> 5) - g * 32], 1u << (v[r] & 31));
          levels[v[r]] = level_of<LT>(depth);
        }
      }
      // long rows still unresolved: the warp scans them together
      for (int r = 0; r < kPullBatch; ++r) {
        uint32_t lanes = __ballot_sync(GB_FULL, (todo >> r) & 1u);
        while (lanes) {
          const int src = __ffs(lanes) - 1;
          lanes &= lanes - 1;
          const int64_t qlo = __shfl_sync(GB_FULL, lo[r], src);
          const int64_t qhi = __shfl_sync(GB_FULL, hi[r], src);
          const int32_t vv = __shfl_sync(GB_FULL, v[r], src);
          bool h = false;
          for (int64_t base = qlo; base < qhi && !h; base += 32) {
            const int64_t q = base + lane;
            bool mh = false;
            if (q < qhi) {
              const int32_t j = __ldg(idx + q);
              mh = ((ld_probe(fbm + (j >> 5)) >> (j & 31)) & 1u) && on(q);
            }
            h = __ballot_sync(GB_FULL, mh) != 0;
          }
          if (h && lane == src) {
            atomicOr(&nw[(vv >> 5) - g * 32], 1u << (vv & 31));
            levels[vv] = level_of<LT>(depth);
          }
        }
      }
      __syncwarp();
    }
    __syncwarp();
    const uint32_t bits = nw[lane];
    if (w < W) {
      fbm_next[w] = bits;
      if (bits) {
        vbm[w] |= bits;
        vprev[w] |= bits;
      }
    }
    if (xmin) prefix_note(&wmin, g, vb0 | bits, w < W);
    const int c = __popc(bits);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(GB_FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(GB_FULL, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && total) base = atomicAdd(count, (unsigned long long)total);
    base = __shfl_sync(GB_FULL, base, 31);
    int slot = incl - c;
    uint32_t b2 = bits;
    while (b2) {
      const int b = __ffs(b2) - 1;
      b2 &= b2 - 1;
      F[base + slot++] = (int32_t)(w * 32 + b);
    }
    __syncwarp();
  }
  if (xmin) prefix_flush(wmin, xmin);
}

template <class LT>
__global__ void __launch_bounds__(256)
bfs_pull(int64_t n, DevI64 depth_d, const int64_t* __restrict__ off,
         const int32_t* __restrict__ idx, EdgeOn on, const uint32_t* __restrict__ nonempty,
         uint32_t* __restrict__ vbm, uint32_t* __restrict__ vprev, const uint32_t* __restrict__ fbm,
         uint32_t* __restrict__ fbm_next, DevP<LT> levels_d,
         int32_t* __restrict__ F, unsigned long long* __restrict__ count,
         unsigned long long* __restrict__ count_clear, int64_t g_lo, int64_t g_hi,
         unsigned long long* __restrict__ xmin) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *count_clear = 0;
  pull_body(n, depth_d.get(), off, idx, on, nonempty, vbm, vprev, fbm, fbm_next, levels_d.get(), F,
            count, g_lo, g_hi, xmin);
}

template <class LT>
__global__ void bfs_unstamp(DevI64 Kd, const int32_t* __restrict__ F, LT* __restrict__ levels) {
  const int64_t K = Kd.get();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K;
       i += (int64_t)gridDim.x * blockDim.x)
    levels[F[i]] = 0;
}

// (A shared-memory cache of the low-id visited words was tried here and lost:
// bank conflicts and halved occupancy cost more than the saved L1 sectors.)
template <bool VALS>
static gb_status launch_push_t(gb_ctx* ctx, int64_t K, const LbsPlan& plan, const gb_csr* a,
                               EdgeOn on, uint32_t* vbm, int64_t xskip) {
  const ExpandKernel k = expand_kernel<VALS>();
  k<<<resident_grid(ctx, k, 256), 256, 0, stream_of(ctx)>>>(
      dval(K), plan.S, plan.rowstart, plan.tile_first, plan.tile_base, a->indices, on, vbm,
      dval(xskip));
  GB_LAUNCH_CHECK(ctx);
  return GB_OK;
}

static gb_status launch_push(gb_ctx* ctx, int64_t K, const LbsPlan& plan, const gb_csr* a,
                             EdgeOn on, uint32_t* vbm, int64_t xskip = 0) {
  return a->values ? launch_push_t<true>(ctx, K, plan, a, on, vbm, xskip)
                   : launch_push_t<false>(ctx, K, plan, a, on, vbm, xskip);
}

template <bool VALS>
static gb_status launch_push_smem_t(gb_ctx* ctx, int64_t K, const LbsPlan& plan, const gb_csr* a,
                                    EdgeOn on, uint32_t* vbm, const uint32_t* vprev) {
  const int64_t W = (a->ncols + 31) / 32;
  size_t smem = 0;
  const int grid = smem_push_setup<VALS>(ctx, W, &smem);
  bfs_expand_smem<VALS><<<grid, kSmemPushThreads, smem, stream_of(ctx)>>>(
      dval(K), plan.S, plan.rowstart, plan.tile_first, plan.tile_base, a->indices, on, vbm, vprev, W);
  GB_LAUNCH_CHECK(ctx);
  return GB_OK;
}

// The ordered graph uses the global-probe push (its hot prefix stays in L1);
// GB_PUSH_SMEM=1 selects the shared-memory prefix kernel instead (A/B).
static bool push_smem_enabled() {
  static const bool on = getenv("GB_PUSH_SMEM") && atoi(getenv("GB_PUSH_SMEM")) == 1;
  return on;
}

static gb_status launch_push_smem(gb_ctx* ctx, int64_t K, const LbsPlan& plan, const gb_csr* a,
                                  EdgeOn on, uint32_t* vbm, const uint32_t* vprev) {
  if (!push_smem_enabled()) return launch_push(ctx, K, plan, a, on, vbm);
  return a->values ? launch_push_smem_t<true>(ctx, K, plan, a, on, vbm, vprev)
                   : launch_push_smem_t<false>(ctx, K, plan, a, on, vbm, vprev);
}

// ---------------------------------------------------------------------------
// Device-driven BFS.  The whole level loop is one CUDA
// graph: a WHILE conditional node whose body holds two unrolled iterations
// (even / odd, so the frontier-bitmap double buffer and the level counters
// are static pointers), each
//     decide  ->  IF push ELSE pull  ->  advance
// The reference direction rule (kernels.py:108-126, rint = half-even like
// Python round), the decision log, the loop cap min(max_niter, n+1) and the
// unstamp of the last frontier (algorithms.py:69-76) all run on the device,
// so a BFS is one graph launch plus one readback instead of a host round trip
// per level.  The push body's degree scan reads the frontier size from device
// memory (three small kernels instead of CUB, whose item count is a host
// value).  The instantiated graph and its scratch are cached per context and
// matrix; per-call inputs (source, cap, output and log pointers, rule
// parameters) live in a device state block written before each launch.
// ---------------------------------------------------------------------------
struct BfsState {
  int64_t* levels;      // per call
  int64_t* log;         // per call: [iters, (dir, K, est) x cap]
  int64_t source, cap;  // per call
  double ratio;         // per call
  int32_t policy, pad_;
  int64_t* out;         // per call, relabelled graphs: levels by original id
  uint16_t* lv16;       // relabelled graphs: internal (16-bit) levels by new id
  // single-entry push levels (K == 1) skip the degree scan: the decision
  // writes that entry's bounds itself (k1 == 0: disabled)
  const int64_t* off;
  const int32_t* F1;
  int64_t *rowstart1, *S1;
  int64_t k1;
  int64_t tiny;         // tiny push levels enabled (GB_BFS_TINY=0 disables)
  int32_t* Ft;          // tiny levels: the new frontier before it is committed to F
  int64_t it, K, depth, dnext, unstamp;  // loop state
  int64_t stopped;                        // the loop ended inside a body pass
  int64_t xcur;                 // dense visited prefix at the level start (ordered graphs)
  int64_t srank;                // relabelled graphs: the source's new id
  unsigned long long xnext;     // ... after the level (atomicMin target)
};

constexpr int kGScanBlocks = 2368;  // 16 per SM (the lower-bound searches want threads); each apply block folds its predecessors
constexpr int kGScanThreads = 256;
constexpr int kGScanItems = 4;
constexpr int64_t kSampleStride = 32;  // column samples: samp[j] = idx[32 j]
constexpr int kApplyRanges = 4;  // scan ranges per apply block
constexpr int kApplyBlocks = kGScanBlocks / kApplyRanges;
static_assert(kGScanBlocks % kApplyRanges == 0, "apply blocks cover the scan ranges");
constexpr int64_t kGraphMaxCap = 1 << 20;  // longer loop caps use the host-driven path


// column samples of a sorted-row (ordered) push matrix: samp[j] = idx[32 j]
__global__ void sample_columns(int64_t ns, const int32_t* __restrict__ idx,
                               int32_t* __restrict__ samp) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < ns;
       j += (int64_t)gridDim.x * blockDim.x)
    samp[j] = idx[j * kSampleStride];
}

// Per-matrix data of a relabelled BFS, built once and cached in the context
// (both engines use it): the push matrix's column samples and the reach limit.
struct OrderedAux {
  const int32_t* idx = nullptr;
  int64_t nnz = 0;
  const int64_t* pull_off = nullptr;
  int32_t* samp = nullptr;
  int64_t reach = 0;
  uint64_t gen = 0, pull_gen = 0;  // gb_csr.gen of the matrices (0: rebuilt every call)
};

static void ordered_aux_free(void* p) {
  auto* a = static_cast<OrderedAux*>(p);
  if (a->samp) cudaFree(a->samp);
  delete a;
}

static gb_status ordered_aux(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull,
                             const OrderedAux** out) {
  void** slot = ctx_slot(ctx, SLOT_BFS_AUX, ordered_aux_free);
  auto* a = static_cast<OrderedAux*>(*slot);
  const int64_t* poff = pull ? pull->offsets : nullptr;
  const uint64_t pgen = pull ? pull->gen : 0;
  if (a && push->gen != 0 && a->gen == push->gen && a->pull_gen == pgen && a->idx == push->indices &&
      a->nnz == push->nnz && a->pull_off == poff) {
    *out = a;
    return GB_OK;
  }
  cudaStream_t s = stream_of(ctx);
  if (a) {
    cudaStreamSynchronize(s);
    ordered_aux_free(a);
    *slot = nullptr;
  }
  a = new OrderedAux();
  a->idx = push->indices;
  a->nnz = push->nnz;
  a->gen = push->gen;
  a->pull_gen = pgen;
  a->pull_off = poff;
  a->reach = push->nrows;
  const int64_t ns = (push->nnz + kSampleStride - 1) / kSampleStride;
  if (ns > 0) {
    if (cudaMalloc(&a->samp, sizeof(int32_t) * ns) != cudaSuccess) {
      cudaGetLastError();
      delete a;
      return set_error(ctx, GB_ERR_OOM, "bfs column samples (%lld)", (long long)ns);
    }
    sample_columns<<<grid_for(ctx, ns, 256, 8), 256, 0, s>>>(ns, push->indices, a->samp);
  }
  if (poff) {
    Arena ar(ctx);
    int64_t* tmp = ar.alloc<int64_t>(1);
    GB_ARENA_CHECK(ctx, ar);
    reach_limit<<<1, 1, 0, s>>>(push->nrows, poff, tmp);
    const gb_status st = read_i64(ctx, tmp, &a->reach);
    if (st != GB_OK) {
      ordered_aux_free(a);
      return st;
    }
  }
  *slot = a;
  *out = a;
  return GB_OK;
}

// capacity of the stamp queue: a queued list spans > 4 tile starts, so it is
// longer than 4 * kWarpTile edges
static inline int64_t stamp_queue_cap(int64_t nnz) { return nnz / (4 * kWarpTile) + 2; }

// entries [lo, hi) of scan range b out of kGScanBlocks
__device__ __forceinline__ void g_range_of(int64_t K, int64_t b, int64_t* lo, int64_t* hi) {
  const int64_t per = (K + kGScanBlocks - 1) / kGScanBlocks;
  *lo = b * per < K ? b * per : K;
  *hi = *lo + per < K ? *lo + per : K;
}

// Per frontier entry k: the part of its (sorted) adjacency list the push must
// expand -- rowstart[k] and its length (kept in S[k] until the apply pass
// turns S into the exclusive scan) -- and the block's partial sum.  With
// X > 0 every vertex below X is already visited (the dense visited prefix of
// a degree-ordered graph: s24 level 2 has X = 13,043, and 24 % of the level's
// edges point below it), so the neighbours below X are skipped: they could
// only probe set bits.  A lower-bound search in the sorted row finds the cut.
__device__ __forceinline__ void scan_partials_body(int64_t K, const int32_t* F,
                                                   const int64_t* __restrict__ off,
                                                   const int32_t* __restrict__ idx, int64_t X,
                                                   int64_t clo, int64_t chi,
                                                   const int32_t* __restrict__ samp,
                                                   int64_t* rowstart, int64_t* deg, int64_t* part) {
  using BlockReduce = cub::BlockReduce<int64_t, kGScanThreads>;
  __shared__ typename BlockReduce::TempStorage tmp;
  int64_t lo, hi;
  g_range_of(K, blockIdx.x, &lo, &hi);
  int64_t sum = 0;
  for (int64_t k = lo + threadIdx.x; k < hi; k += kGScanThreads) {
    const int64_t v = F[k];
    int64_t a = __ldg(off + v);
    const int64_t b = __ldg(off + v + 1);
    if (X > 0 && b - a >= clo && b - a <= chi) {
      if (samp) {
        // lower bound of X in [a, b) narrowed through the column samples
        // (samp[j] = idx[32 j]): a search over the list's samples (one line
        // for a 512-entry list), then one 32-entry line of the list -- ~3
        // random lines per entry with the offsets, against ~6 for a plain
        // binary search (this search is DRAM-bound)
        int64_t l = a, h = b;
        const int64_t jl = (a + kSampleStride - 1) / kSampleStride, jh = (b - 1) / kSampleStride;
        if (jl <= jh) {
          int64_t ql = jl, qh = jh + 1;  // first sample >= X, or jh + 1
          while (ql < qh) {
            const int64_t m = (ql + qh) >> 1;
            if (__ldg(samp + m) < X) ql = m + 1; else qh = m;
          }
          if (ql <= jh) h = ql * kSampleStride;
          if (ql > jl) l = (ql - 1) * kSampleStride + 1;
        }
        while (l < h) {
          const int64_t m = (l + h) >> 1;
          if (__ldg(idx + m) < X) l = m + 1; else h = m;
        }
        a = l;
      } else if (__ldg(idx + a) < X) {
        if (__ldg(idx + b - 1) < X) {
          a = b;
        } else {  // first position in (a, b-1] holding a column >= X
          int64_t l = a + 1, h = b - 1;
          while (l < h) {
            const int64_t m = (l + h) >> 1;
            if (__ldg(idx + m) < X) l = m + 1; else h = m;
          }
          a = l;
        }
      }
    }
    rowstart[k] = a;
    deg[k] = b - a;
    sum += b - a;
  }
  const int64_t tot = BlockReduce(tmp).Sum(sum);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
  if (blockIdx.x == 0 && threadIdx.x == 0) part[kGScanBlocks] = 0;  // stamp queue length
}

__global__ void __launch_bounds__(kGScanThreads)
g_scan_partials(DevI64 Kd, const int32_t* __restrict__ F, const int64_t* __restrict__ off,
                const int32_t* __restrict__ idx, DevI64 Xd, int64_t clo, int64_t chi,
                const int32_t* __restrict__ samp, int64_t* __restrict__ rowstart,
                int64_t* __restrict__ deg, int64_t* __restrict__ part) {
  scan_partials_body(Kd.get(), F, off, idx, Xd.get(), clo, chi, samp, rowstart, deg, part);
}

// rowstart[k] = off[F[k]], S = exclusive scan of the degrees, S[K] = E, and
// tile_first[t] = the entry holding expansion slot t*kWarpTile.  Each block
// derives its own carry-in from the partials (no separate top-level scan),
// and every non-empty entry stamps the tiles that start inside its range, so
// one launch replaces scan-top / scan-apply / tile-first.
// rowstart[k] and the lengths (in S[k]) come from scan_partials_body.
__device__ __forceinline__ void scan_apply_body(int64_t K, const int64_t* part, const int64_t* rowstart,
                                                int64_t* S, int32_t* tile_first, int64_t* tile_base,
                                                int64_t* qcount, int64_t* queue) {
  using BlockScan = cub::BlockScan<int64_t, kGScanThreads>;
  using BlockReduce = cub::BlockReduce<int64_t, kGScanThreads>;
  __shared__ union {
    typename BlockScan::TempStorage scan;
    typename BlockReduce::TempStorage red;
  } tmp;
  __shared__ int64_t s_run;
  // block b applies scan ranges [b*kApplyRanges, (b+1)*kApplyRanges): one
  // wave of blocks instead of four
  const int r0 = blockIdx.x * kApplyRanges;
  int64_t lo, hi, dummy;
  g_range_of(K, r0, &lo, &dummy);
  g_range_of(K, r0 + kApplyRanges - 1, &dummy, &hi);
  // blocks past the end only matter for S[K] (the last block)
  if (lo >= hi && blockIdx.x != gridDim.x - 1) return;
  {
    int64_t c = 0;
    // all predecessor partials in flight at once
    constexpr int kCarry = (kGScanBlocks + kGScanThreads - 1) / kGScanThreads;
    int64_t pv[kCarry];
#pragma unroll
    for (int j = 0; j < kCarry; ++j) {
      const int i = threadIdx.x + j * kGScanThreads;
      pv[j] = i < r0 ? part[i] : 0;
    }
#pragma unroll
    for (int j = 0; j < kCarry; ++j) c += pv[j];
    const int64_t run0 = BlockReduce(tmp.red).Sum(c);
    if (threadIdx.x == 0) {
      s_run = run0;
      if (blockIdx.x == gridDim.x - 1) {
        int64_t t = run0;
        for (int i = r0; i < kGScanBlocks; ++i) t += part[i];
        S[K] = t;
      }
    }
    __syncthreads();
  }
  int64_t run = s_run;
  for (int64_t base = lo; base < hi; base += kGScanThreads * kGScanItems) {
    int64_t d[kGScanItems], r[kGScanItems];
    int64_t sum = 0;
#pragma unroll
    for (int i = 0; i < kGScanItems; ++i) {
      const int64_t k = base + threadIdx.x * kGScanItems + i;
      d[i] = k < hi ? S[k] : 0;
      r[i] = k < hi ? rowstart[k] : 0;
      sum += d[i];
    }
    int64_t pre, agg;
    BlockScan(tmp.scan).ExclusiveSum(sum, pre, agg);
    int64_t acc = run + pre;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < kGScanItems; ++i) {
      const int64_t k = base + threadIdx.x * kGScanItems + i;
      // tiles [t0, t1) start inside this entry's range; up to 4 are stamped
      // by the owning thread
      int64_t t0 = 0, t1 = 0, b = 0;
      if (k < hi) {
        S[k] = acc;
        if (d[i] > 0) {
          b = r[i] - acc;
          t0 = (acc + kWarpTile - 1) / kWarpTile;
          t1 = (acc + d[i] + kWarpTile - 1) / kWarpTile;
          if (t1 - t0 <= 4) {
            for (int64_t t = t0; t < t1; ++t) {
              tile_first[t] = (int32_t)k;
              tile_base[t] = b;
            }
          }
        }
      }
      // lists spanning more than 4 tiles go to the stamp queue (one warp
      // each in g_scan_stamp): stamped here they serialise on the warps that
      // hold the level's hubs
      const bool qb = t1 - t0 > 4;
      const uint32_t qm = __ballot_sync(GB_FULL, qb);
      if (qm) {
        const int leader = __ffs(qm) - 1;
        unsigned long long qbase = 0;
        if (lane == leader)
          qbase = atomicAdd(reinterpret_cast<unsigned long long*>(qcount), (unsigned long long)__popc(qm));
        qbase = __shfl_sync(GB_FULL, qbase, leader);
        if (qb) {
          int64_t* job = queue + 4 * (qbase + __popc(qm & ((1u << lane) - 1u)));
          job[0] = t0;
          job[1] = t1;
          job[2] = b;
          job[3] = k;
        }
      }
      acc += d[i];
    }
    run += agg;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kGScanThreads, 4)
g_scan_apply(DevI64 Kd, int64_t* __restrict__ part, const int64_t* __restrict__ rowstart,
             int64_t* __restrict__ S, int32_t* __restrict__ tile_first,
             int64_t* __restrict__ tile_base, int64_t* __restrict__ queue) {
  scan_apply_body(Kd.get(), part, rowstart, S, tile_first, tile_base, part + kGScanBlocks, queue);
}

// Stamp the queued long lists' tiles, one warp per list.  The queue length
// lives in part[kGScanBlocks] (reset by g_scan_partials).
__global__ void __launch_bounds__(256)
g_scan_stamp(const int64_t* __restrict__ part, const int64_t* __restrict__ queue,
             int32_t* __restrict__ tile_first, int64_t* __restrict__ tile_base) {
  const int64_t nq = part[kGScanBlocks];
  const int lane = threadIdx.x & 31;
  for (int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; e < nq;
       e += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t t0 = queue[4 * e], t1 = queue[4 * e + 1], b = queue[4 * e + 2];
    const int32_t k = (int32_t)queue[4 * e + 3];
    for (int64_t t = t0 + lane; t < t1; t += 32) {
      tile_first[t] = k;
      tile_base[t] = b;
    }
  }
}

__global__ void g_zero_levels(int64_t n, const BfsState* __restrict__ st) {
  int64_t* lv = st->levels;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    lv[i] = 0;
}

__device__ void decide_body(BfsState* st, int64_t nnz, int64_t nrows, unsigned long long* c,
                            cudaGraphConditionalHandle h_push);
// SWITCH values of a level node: its push body, its pull body, or nothing
constexpr unsigned kSwPush = 0, kSwPull = 1, kSwPush1 = 2, kSwTiny = 3, kSwSkip = 4;
// a push level with at most this many frontier entries takes the tiny path:
// one expansion kernel that appends each discovered vertex itself (no degree
// scan, no full-bitmap finalize) -- the s24 tail levels (3,034 and 9 entries)
constexpr int64_t kTinyK = 4096;

__global__ void g_start(BfsState* st, const int32_t* rank, uint32_t* vbm, uint32_t* vprev,
                        uint32_t* fbm0, int32_t* F, cudaGraphConditionalHandle h_loop,
                        int64_t nnz, int64_t nrows, unsigned long long* c0,
                        cudaGraphConditionalHandle h_push0) {
  const int64_t s = rank ? (int64_t)rank[st->source] : st->source;
  st->srank = s;
  if (rank) st->lv16[s] = 1;
  else st->levels[s] = 1;
  const uint32_t bit = 1u << (s & 31);
  vbm[s >> 5] |= bit;
  vprev[s >> 5] |= bit;
  fbm0[s >> 5] |= bit;
  F[0] = (int32_t)s;
  st->it = 0;
  st->K = 1;
  st->depth = 1;
  st->xcur = 0;
  st->unstamp = 0;
  st->stopped = 0;
  st->log[0] = 0;
  cudaGraphSetConditional(h_loop, st->cap > 0 ? 1u : 0u);
  if (st->cap > 0) decide_body(st, nnz, nrows, c0, h_push0);
}

// the reference rule (kernels.py:108-126) for iteration st->it; c: the
// counter that iteration's finalize / pull accumulates into
__device__ void decide_body(BfsState* st, int64_t nnz, int64_t nrows, unsigned long long* c,
                            cudaGraphConditionalHandle h_push) {
  const int64_t K = st->K, it = st->it;
  const double d = nrows ? (double)nnz / (double)nrows : 0.0;
  const int64_t est = (int64_t)rint(d * (double)K);
  const double thr = (double)nnz * st->ratio;
  int32_t dir = (double)est > thr ? GB_DIR_PULL : GB_DIR_PUSH;
  if (st->policy == GB_DIR_PUSH) dir = GB_DIR_PUSH;
  if (st->policy == GB_DIR_PULL) dir = GB_DIR_PULL;
  int64_t* e = st->log + 1 + 3 * it;
  e[0] = dir;
  e[1] = K;
  e[2] = est;
  st->dnext = st->depth + 1;
  st->xnext = ~0ull;
  *c = 0;
  unsigned sw = dir == GB_DIR_PUSH ? kSwPush : kSwPull;
  // (the single-entry level keeps push1 + finalize: finalize finds the dense
  // visited prefix the next push cuts at -- measured 0.79 vs 1.06 ms at s24)
  if (dir == GB_DIR_PUSH && K > 1 && K <= kTinyK && st->tiny) sw = kSwTiny;
  if (dir == GB_DIR_PUSH && K == 1 && st->k1) {
    // one frontier entry: its whole list (no prefix cut) as the expansion space
    const int64_t v = st->F1[0];
    const int64_t a = st->off[v], b = st->off[v + 1];
    st->rowstart1[0] = a;
    st->S1[0] = 0;
    st->S1[1] = b - a;
    sw = kSwPush1;
  }
  cudaGraphSetConditional(h_push, sw);
}

// after a level: new frontier size, loop continuation, cap handling; when the
// loop continues, the next iteration's decision (one node instead of two)
__global__ void g_step(BfsState* st, const unsigned long long* c, int64_t n,
                       cudaGraphConditionalHandle h_a, cudaGraphConditionalHandle h_b,
                       int64_t nnz, int64_t nrows, unsigned long long* c_next,
                       cudaGraphConditionalHandle h_push_next) {
  if (st->stopped) {  // the body's earlier level ended the loop
    cudaGraphSetConditional(h_a, 0);
    cudaGraphSetConditional(h_b, 0);
    cudaGraphSetConditional(h_push_next, kSwSkip);
    return;
  }
  const int64_t K = (int64_t)*c;
  st->xcur = st->xnext < (unsigned long long)n ? (int64_t)st->xnext : n;
  const int64_t it = st->it;
  st->log[0] = it + 1;
  st->K = K;
  unsigned cont = 0;
  if (K != 0) {
    st->depth += 1;
    if (it + 1 == st->cap) st->unstamp = 1;
    else cont = 1;
  }
  st->it = it + 1;
  cudaGraphSetConditional(h_a, cont);
  cudaGraphSetConditional(h_b, cont);
  if (cont) {
    decide_body(st, nnz, nrows, c_next, h_push_next);
  } else {
    st->stopped = 1;
    cudaGraphSetConditional(h_push_next, kSwSkip);
  }
}

__global__ void g_unstamp(const BfsState* __restrict__ st, const int32_t* __restrict__ F) {
  if (!st->unstamp) return;
  const int64_t K = st->K;
  int64_t* lv = st->levels;
  uint16_t* lv16 = st->lv16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (lv16) lv16[F[i]] = 0;
    else lv[F[i]] = 0;
  }
}

static bool tiny_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GB_BFS_TINY");
    v = !(e && atoi(e) == 0);
  }
  return v != 0;
}

// ---- tiny push levels (K <= kTinyK): a block per frontier entry expands its
// list; the thread that sets a vertex's visited bit owns the discovery and
// stamps its level, frontier bit and visited-at-level-start bit and appends
// it to Ft.  bfs_tiny_commit then moves Ft to F.  fbm_next was cleared
// before; the dense visited prefix is kept as it was (still valid).
template <class LT>
__global__ void __launch_bounds__(256)
bfs_tiny_expand(BfsState* st, const int32_t* __restrict__ F, const int64_t* __restrict__ off,
                const int32_t* __restrict__ idx, EdgeOn on, uint32_t* vbm, uint32_t* vprev,
                uint32_t* fbm_next, DevP<LT> levels_d, unsigned long long* count) {
  const int64_t K = st->K;
  const int64_t depth = st->dnext;
  LT* levels = levels_d.get();
  int32_t* Ft = st->Ft;
  // fewer entries than blocks (the source level: K = 1): several blocks share
  // an entry's list
  const int64_t bpe = K < gridDim.x ? gridDim.x / K : 1;
  for (int64_t b = blockIdx.x; b < K * bpe; b += gridDim.x) {
    const int64_t k = b / bpe, part = b % bpe;
    const int32_t u = F[k];
    const int64_t lo = off[u], hi = off[u + 1];
    for (int64_t p0 = lo + part * blockDim.x; p0 < hi; p0 += bpe * blockDim.x) {
      const int64_t p = p0 + threadIdx.x;
      bool disc = false;
      int32_t v = 0;
      if (p < hi && on(p)) {
        v = idx[p];
        const uint32_t bit = 1u << (v & 31);
        if (!(ld_probe(vbm + (v >> 5)) & bit) && !(atomicOr(vbm + (v >> 5), bit) & bit)) {
          disc = true;  // this thread set the bit: it owns the discovery
          atomicOr(vprev + (v >> 5), bit);
          atomicOr(fbm_next + (v >> 5), bit);
          levels[v] = level_of<LT>(depth);
        }
      }
      const uint32_t bal = __ballot_sync(__activemask(), disc);
      if (bal) {
        // one reservation per warp for its discoveries
        unsigned long long at = 0;
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(bal) - 1;
        if (lane == leader) at = atomicAdd(count, (unsigned long long)__popc(bal));
        at = __shfl_sync(__activemask(), at, leader);
        if (disc) Ft[at + __popc(bal & ((1u << lane) - 1u))] = v;
      }
    }
  }
}

__global__ void bfs_tiny_commit(BfsState* st, int32_t* __restrict__ F,
                                const unsigned long long* __restrict__ count,
                                unsigned long long* __restrict__ count_clear) {
  const int64_t c = (int64_t)*count;
  const int32_t* Ft = st->Ft;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c;
       i += (int64_t)gridDim.x * blockDim.x)
    F[i] = Ft[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *count_clear = 0;
    st->xnext = (unsigned long long)st->xcur;  // the prefix is unchanged (still a lower bound)
  }
}

struct BfsGraph {
  // key: the matrix orientations the graph was built for
  gb_csr push{}, pull{};
  const uint32_t* nonempty = nullptr;
  const int32_t* rank = nullptr;  // relabelled graph: original id -> new id
  // scratch (one allocation)
  void* mem = nullptr;
  uint32_t *vbm = nullptr, *vprev = nullptr, *fbm[2] = {nullptr, nullptr};
  int32_t* F = nullptr;
  int32_t* tile_first = nullptr;
  int64_t* tile_base = nullptr;
  unsigned long long* cnt = nullptr;
  int64_t *rowstart = nullptr, *S = nullptr, *part = nullptr;
  uint16_t* lv = nullptr;  // relabelled graph: 16-bit levels by new id
  const int32_t* samp = nullptr;  // relabelled graph: column samples (OrderedAux)
  int64_t* queue = nullptr;  // stamp queue of the long lists (4 x int64 per list)
  int32_t* Ft = nullptr;     // tiny levels' new frontier
  int64_t reach = 0;         // relabelled graph: vertices >= reach have no in-edges
  BfsState* st = nullptr;
  cudaGraphExec_t exec = nullptr;
  int launches_push = 0, launches_pull = 0, launches_fixed = 0;
  int unroll = 2;  // levels per WHILE pass (even)
  int launches_push1 = 0;  // a single-entry push level (expansion + finalize)
  int launches_tiny = 0;   // a tiny push level (memset, expansion, commit)
  int64_t k1 = 0;          // single-entry push levels skip the degree scan
};

static void bfs_graph_free(void* p) {
  auto* g = static_cast<BfsGraph*>(p);
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->mem) cudaFree(g->mem);
  delete g;
}

static bool same_csr(const gb_csr& a, const gb_csr& b) {
  return a.gen != 0 && a.gen == b.gen && a.nrows == b.nrows && a.ncols == b.ncols && a.nnz == b.nnz && a.offsets == b.offsets &&
         a.indices == b.indices && a.values == b.values && a.dtype == b.dtype &&
         a.iso_i64 == b.iso_i64 && a.iso_f64 == b.iso_f64;
}

template <class Fn>
static cudaError_t capture_into(cudaGraph_t g, cudaStream_t cs, Fn fn) {
  cudaError_t e = cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0,
                                                cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) return e;
  cudaError_t e2 = fn();
  cudaGraph_t out = g;
  e = cudaStreamEndCapture(cs, &out);
  return e2 != cudaSuccess ? e2 : e;
}

#define GB_GTRY(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) return e_; } while (0)

static cudaError_t bfs_graph_build(gb_ctx* ctx, BfsGraph* G, const cudaStream_t* cs) {
  const gb_csr& push = G->push;
  const gb_csr& pull = G->pull;
  const int64_t n = push.nrows;
  const int64_t W = (n + 31) / 32;
  const EdgeOn push_on{push.values, push.dtype};
  const EdgeOn pull_on{pull.values, pull.dtype};
  const bool push_dead = !push.values && push.iso_i64 == 0 && push.iso_f64 == 0.0;
  const bool pull_dead = !pull.values && pull.iso_i64 == 0 && pull.iso_f64 == 0.0;
  BfsState* st = G->st;
  const int grid_w = grid_for(ctx, W, 256, 8);
  const ExpandKernel expand = push.values ? expand_kernel<true>() : expand_kernel<false>();
  const int grid_expand = resident_grid(ctx, expand, 256);
  const bool ordered = G->rank != nullptr;
  const bool use_smem = ordered && push_smem_enabled();
  size_t smem = 0;
  const int grid_smem = push.values ? smem_push_setup<true>(ctx, W, &smem)
                                    : smem_push_setup<false>(ctx, W, &smem);
  G->launches_push = 4 + (push_dead ? 0 : 1);
  G->launches_push1 = 1 + (push_dead ? 0 : 1);
  G->launches_tiny = 2 + (push_dead ? 0 : 1);
  G->k1 = !use_smem && !(getenv("GB_BFS_K1") && atoi(getenv("GB_BFS_K1")) == 0);
  const int grid_stamp = grid_for(ctx, (int64_t)1 << 40, 256, 8);
  G->launches_pull = pull_dead ? 3 : 1;
  // 4 memsets, zero levels (or clear 16-bit levels + unpermute), start (with
  // the first decision), unstamp; each level adds its body and one g_step
  G->launches_fixed = ordered ? 8 : 7;
  {
    // 2 measured best (s24: 0.765 ms; 4: 0.797, 6: 0.774, 8: 0.805)
    const int u = getenv("GB_BFS_UNROLL") ? atoi(getenv("GB_BFS_UNROLL")) : 2;
    G->unroll = u >= 2 && u % 2 == 0 && u <= 16 ? u : 2;
  }

  auto push_body = [&](int h, cudaStream_t s, bool single) -> cudaError_t {
    // single: one frontier entry whose bounds g_step / g_start wrote (no scan)
    if (!single) {
    // ordered (sorted-row) graphs skip the dense visited prefix of each list
    g_scan_partials<<<kGScanBlocks, kGScanThreads, 0, s>>>(
        dptr(&st->K), G->F, push.offsets, push.indices,
        ordered && prefix_mode() == 1 ? dptr(&st->xcur) : dval(0), cut_lo(), cut_hi(),
        use_samples() ? G->samp : nullptr, G->rowstart, G->S, G->part);
    g_scan_apply<<<kApplyBlocks, kGScanThreads, 0, s>>>(dptr(&st->K), G->part, G->rowstart, G->S,
                                                        G->tile_first, G->tile_base, G->queue);
    g_scan_stamp<<<grid_stamp, 256, 0, s>>>(G->part, G->queue, G->tile_first, G->tile_base);
    }
    if (!push_dead && use_smem) {
      if (push.values)
        bfs_expand_smem<true><<<grid_smem, kSmemPushThreads, smem, s>>>(
            dptr(&st->K), G->S, G->rowstart, G->tile_first, G->tile_base, push.indices, push_on, G->vbm, G->vprev, W);
      else
        bfs_expand_smem<false><<<grid_smem, kSmemPushThreads, smem, s>>>(
            dptr(&st->K), G->S, G->rowstart, G->tile_first, G->tile_base, push.indices, push_on, G->vbm, G->vprev, W);
    } else if (!push_dead) {
      expand<<<grid_expand, 256, 0, s>>>(dptr(&st->K), G->S, G->rowstart, G->tile_first,
                                         G->tile_base, push.indices, push_on, G->vbm,
                                         ordered && prefix_mode() == 2 ? dptr(&st->xcur) : dval(0));
    }
    if (ordered)
      bfs_finalize<uint16_t><<<grid_w, 256, 0, s>>>(n, dptr(&st->dnext), G->vbm, G->vprev,
                                                   G->fbm[h ^ 1], pptr(&st->lv16), G->F, G->cnt + h,
                                                   G->cnt + (h ^ 1), nullptr, &st->xnext);
    else
      bfs_finalize<int64_t><<<grid_w, 256, 0, s>>>(n, dptr(&st->dnext), G->vbm, G->vprev,
                                                   G->fbm[h ^ 1], pptr(&st->levels), G->F, G->cnt + h,
                                                   G->cnt + (h ^ 1), nullptr, nullptr);
    return cudaGetLastError();
  };
  auto tiny_body = [&](int h, cudaStream_t s) -> cudaError_t {
    GB_GTRY(cudaMemsetAsync(G->fbm[h ^ 1], 0, sizeof(uint32_t) * W, s));
    if (!push_dead) {
      if (ordered)
        bfs_tiny_expand<uint16_t><<<grid_for(ctx, kTinyK, 1, 4), 256, 0, s>>>(
            st, G->F, push.offsets, push.indices, push_on, G->vbm, G->vprev, G->fbm[h ^ 1],
            pptr(&st->lv16), G->cnt + h);
      else
        bfs_tiny_expand<int64_t><<<grid_for(ctx, kTinyK, 1, 4), 256, 0, s>>>(
            st, G->F, push.offsets, push.indices, push_on, G->vbm, G->vprev, G->fbm[h ^ 1],
            pptr(&st->levels), G->cnt + h);
    }
    bfs_tiny_commit<<<4, 256, 0, s>>>(st, G->F, G->cnt + h, G->cnt + (h ^ 1));
    return cudaGetLastError();
  };
  auto pull_body = [&](int h, cudaStream_t s) -> cudaError_t {
    if (pull_dead) {
      GB_GTRY(cudaMemsetAsync(G->fbm[h ^ 1], 0, sizeof(uint32_t) * W, s));
      GB_GTRY(cudaMemsetAsync(G->cnt + h, 0, 8, s));
      GB_GTRY(cudaMemsetAsync(G->cnt + (h ^ 1), 0, 8, s));
    } else {
      if (ordered)
        bfs_pull<uint16_t><<<grid_w, 256, 0, s>>>(n, dptr(&st->dnext), pull.offsets, pull.indices,
                                                 pull_on, G->nonempty, G->vbm, G->vprev, G->fbm[h],
                                                 G->fbm[h ^ 1], pptr(&st->lv16), G->F, G->cnt + h,
                                                 G->cnt + (h ^ 1), 0, (W + 31) / 32, &st->xnext);
      else
        bfs_pull<int64_t><<<grid_w, 256, 0, s>>>(n, dptr(&st->dnext), pull.offsets, pull.indices,
                                                 pull_on, G->nonempty, G->vbm, G->vprev, G->fbm[h],
                                                 G->fbm[h ^ 1], pptr(&st->levels), G->F, G->cnt + h,
                                                 G->cnt + (h ^ 1), 0, (W + 31) / 32, nullptr);
    }
    return cudaGetLastError();
  };
  // one iteration on stream s (capturing into the graph that should hold it)
  auto iteration = [&](int h, cudaStream_t s, cudaStream_t s_inner,
                       cudaGraphConditionalHandle h_push, cudaGraphConditionalHandle h_a,
                       cudaGraphConditionalHandle h_b,
                       cudaGraphConditionalHandle h_push_next) -> cudaError_t {
    // h_push was set by the previous node that decided this iteration
    // (g_start or the previous g_step); the handles live in the top graph
    cudaGraph_t br[4];
    cudaStreamCaptureStatus status;
    cudaGraph_t g;
    {
      const cudaGraphNode_t* deps = nullptr;
      size_t nd = 0;
      GB_GTRY(cudaStreamGetCaptureInfo(s, &status, nullptr, &g, &deps, &nd));
      cudaGraphNodeParams p = {};
      p.type = cudaGraphNodeTypeConditional;
      p.conditional.handle = h_push;
      p.conditional.type = cudaGraphCondTypeSwitch;
      p.conditional.size = 4;  // kSwPush, kSwPull, kSwPush1, kSwTiny; kSwSkip runs none
      cudaGraphNode_t node;
      GB_GTRY(cudaGraphAddNode(&node, g, deps, nd, &p));
      for (int b = 0; b < 4; ++b) br[b] = p.conditional.phGraph_out[b];
      GB_GTRY(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    }
    GB_GTRY(capture_into(br[0], s_inner, [&] { return push_body(h, s_inner, false); }));
    GB_GTRY(capture_into(br[1], s_inner, [&] { return pull_body(h, s_inner); }));
    GB_GTRY(capture_into(br[2], s_inner, [&] { return push_body(h, s_inner, true); }));
    GB_GTRY(capture_into(br[3], s_inner, [&] { return tiny_body(h, s_inner); }));
    g_step<<<1, 1, 0, s>>>(st, G->cnt + h, n, h_a, h_b, push.nnz, push.nrows, G->cnt + (h ^ 1),
                           h_push_next);
    return cudaGetLastError();
  };

  cudaGraph_t top;
  GB_GTRY(cudaGraphCreate(&top, 0));
  cudaError_t err = capture_into(top, cs[0], [&]() -> cudaError_t {
    cudaStream_t s = cs[0];
    GB_GTRY(cudaMemsetAsync(G->vbm, 0, sizeof(uint32_t) * W, s));
    GB_GTRY(cudaMemsetAsync(G->vprev, 0, sizeof(uint32_t) * W, s));
    GB_GTRY(cudaMemsetAsync(G->fbm[0], 0, sizeof(uint32_t) * W, s));
    GB_GTRY(cudaMemsetAsync(G->cnt, 0, 16, s));
    // the API levels (int64) or the internal 16-bit levels of a relabelled run
    // start at 0: unvisited vertices read 0
    if (!ordered) g_zero_levels<<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(n, st);
    else GB_GTRY(cudaMemsetAsync(G->lv, 0, 2 * (size_t)n, s));  // unvisited read level 0
    cudaStreamCaptureStatus status;
    cudaGraph_t g;
    GB_GTRY(cudaStreamGetCaptureInfo(s, &status, nullptr, &g, nullptr, nullptr));
    // one SWITCH handle per level slot of a pass (a handle drives exactly one
    // conditional node); slot j's g_step decides slot j+1
    cudaGraphConditionalHandle h_loop, h_push[16];
    GB_GTRY(cudaGraphConditionalHandleCreate(&h_loop, g, 0, cudaGraphCondAssignDefault));
    for (int j = 0; j < G->unroll; ++j)
      GB_GTRY(cudaGraphConditionalHandleCreate(&h_push[j], g, 0, cudaGraphCondAssignDefault));
    g_start<<<1, 1, 0, s>>>(st, G->rank, G->vbm, G->vprev, G->fbm[0], G->F, h_loop, push.nnz,
                            push.nrows, G->cnt, h_push[0]);
    GB_GTRY(cudaGetLastError());
    cudaGraph_t body;
    {
      const cudaGraphNode_t* deps = nullptr;
      size_t nd = 0;
      GB_GTRY(cudaStreamGetCaptureInfo(s, &status, nullptr, &g, &deps, &nd));
      cudaGraphNodeParams p = {};
      p.type = cudaGraphNodeTypeConditional;
      p.conditional.handle = h_loop;
      p.conditional.type = cudaGraphCondTypeWhile;
      p.conditional.size = 1;
      cudaGraphNode_t node;
      GB_GTRY(cudaGraphAddNode(&node, g, deps, nd, &p));
      body = p.conditional.phGraph_out[0];
      GB_GTRY(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    }
    GB_GTRY(capture_into(body, cs[1], [&]() -> cudaError_t {
      // G->unroll (even) levels per pass; a level after the one that ended
      // the loop is a skipped SWITCH and a no-op g_step
      for (int j = 0; j < G->unroll; ++j)
        GB_GTRY(iteration(j & 1, cs[1], cs[2], h_push[j], h_loop, h_loop,
                          h_push[(j + 1) % G->unroll]));
      return cudaSuccess;
    }));
    g_unstamp<<<grid_for(ctx, n, 256, 4), 256, 0, s>>>(st, G->F);
    if (ordered)
      bfs_unpermute<<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(n, G->rank, G->lv, G->reach,
                                                             dptr(&st->srank), pptr(&st->out));
    return cudaGetLastError();
  });
  if (err == cudaSuccess) err = cudaGraphInstantiate(&G->exec, top, 0);
  cudaGraphDestroy(top);
  return err;
}

// Returns GB_OK after running the BFS, or GB_ERR_UNSUPPORTED when the graph
// path cannot be used (the caller then runs the host-driven loop).

// Asynchronous form (log_ext != NULL): the device writes the raw log
// [iters, (dir, K, est) x iters] to log_ext, its first kLogPrefix decisions
// are copied to the pinned log_pin behind the graph on the stream, and the
// call returns without synchronising; launch_info receives the launches of
// the fixed part and of one push / pull level.
constexpr int64_t kLogPrefix = 21;
static gb_status bfs_graph_run(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull,
                               const uint32_t* nonempty, const int32_t* rank, const OrderedAux* aux, int64_t source, int64_t cap,
                               double ratio, int32_t policy, int64_t* levels, int32_t* log_dir,
                               int64_t* log_nvals, int64_t* log_est, int64_t* iters_out,
                               int64_t* log_ext = nullptr, int64_t* log_pin = nullptr,
                               int64_t* launch_info = nullptr) {
  void** slot = ctx_slot(ctx, SLOT_BFS_GRAPH, bfs_graph_free);
  BfsGraph* G = static_cast<BfsGraph*>(*slot);
  if (G && !(same_csr(G->push, *push) && same_csr(G->pull, *pull) && G->nonempty == nonempty &&
             G->rank == rank)) {
    cudaStreamSynchronize(stream_of(ctx));
    bfs_graph_free(G);
    G = nullptr;
    *slot = nullptr;
  }
  if (!G) {
    G = new BfsGraph();
    G->push = *push;
    G->pull = *pull;
    G->nonempty = nonempty;
    G->rank = rank;
    const int64_t n = push->nrows;
    const int64_t W = (n + 31) / 32;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) / 256 * 256; return o; };
    const size_t o_vbm = take(4 * W), o_vprev = take(4 * W), o_f0 = take(4 * W), o_f1 = take(4 * W);
    const size_t o_F = take(4 * (size_t)n), o_tf = take(4 * (size_t)(push->nnz / kWarpTile + 2));
    const size_t o_tb = take(8 * (size_t)(push->nnz / kWarpTile + 2));
    const size_t o_cnt = take(32), o_rs = take(8 * (size_t)(n + 1)), o_S = take(8 * (size_t)(n + 1));
    const size_t o_part = take(8 * (kGScanBlocks + 1)), o_st = take(sizeof(BfsState));
    const size_t o_q = take(32 * (size_t)stamp_queue_cap(push->nnz));
    const size_t o_lv = rank ? take(2 * (size_t)n) : 0;
    const size_t o_Ft = take(4 * (size_t)n);
    if (cudaMalloc(&G->mem, off) != cudaSuccess) {
      cudaGetLastError();
      delete G;
      return GB_ERR_UNSUPPORTED;
    }
    char* m = static_cast<char*>(G->mem);
    G->vbm = (uint32_t*)(m + o_vbm);
    G->vprev = (uint32_t*)(m + o_vprev);
    G->fbm[0] = (uint32_t*)(m + o_f0);
    G->fbm[1] = (uint32_t*)(m + o_f1);
    G->F = (int32_t*)(m + o_F);
    G->tile_first = (int32_t*)(m + o_tf);
    G->tile_base = (int64_t*)(m + o_tb);
    G->cnt = (unsigned long long*)(m + o_cnt);
    G->rowstart = (int64_t*)(m + o_rs);
    G->S = (int64_t*)(m + o_S);
    G->part = (int64_t*)(m + o_part);
    G->queue = (int64_t*)(m + o_q);
    G->st = (BfsState*)(m + o_st);
    G->lv = rank ? (uint16_t*)(m + o_lv) : nullptr;
    G->Ft = (int32_t*)(m + o_Ft);
    G->samp = aux ? aux->samp : nullptr;
    G->reach = aux ? aux->reach : n;
    cudaStream_t cs[4];
    for (auto& x : cs) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    const cudaError_t e = bfs_graph_build(ctx, G, cs);
    for (auto& x : cs) cudaStreamDestroy(x);
    if (e != cudaSuccess) {
      cudaGetLastError();
      bfs_graph_free(G);
      return set_error(ctx, GB_ERR_CUDA, "bfs graph build: %s", cudaGetErrorString(e));
    }
    *slot = G;
  }
  if (!G->exec) {
    cudaStream_t cs[4];
    for (auto& x : cs) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    const cudaError_t e = bfs_graph_build(ctx, G, cs);
    for (auto& x : cs) cudaStreamDestroy(x);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return set_error(ctx, GB_ERR_CUDA, "bfs graph build: %s", cudaGetErrorString(e));
    }
  }
  cudaStream_t s = stream_of(ctx);
  Arena ar(ctx);
  int64_t* log = log_ext ? log_ext : ar.alloc<int64_t>(1 + 3 * cap);
  GB_ARENA_CHECK(ctx, ar);
  BfsState h{};
  h.levels = rank ? nullptr : levels;
  h.off = push->offsets;
  h.F1 = G->F;
  h.rowstart1 = G->rowstart;
  h.S1 = G->S;
  h.k1 = G->k1;
  h.tiny = tiny_enabled() ? 1 : 0;
  h.Ft = G->Ft;
  h.lv16 = rank ? G->lv : nullptr;
  h.out = levels;
  h.log = log;
  h.source = source;
  h.cap = cap;
  h.ratio = ratio;
  h.policy = policy;
  // the state block's per-call head (everything before the loop state)
  GB_CUDA(ctx, cudaMemcpyAsync(G->st, &h, offsetof(BfsState, it), cudaMemcpyHostToDevice, s));
  GB_CUDA(ctx, cudaGraphLaunch(G->exec, s));
  const int64_t first = cap < kLogPrefix ? cap : kLogPrefix;
  if (log_ext) {
    GB_CUDA(ctx, cudaMemcpyAsync(log_pin, log, sizeof(int64_t) * (1 + 3 * first),
                                 cudaMemcpyDeviceToHost, s));
    launch_info[0] = G->launches_fixed;
    launch_info[3] = G->unroll;
    launch_info[1] = 1 + G->launches_push;  // + g_step
    launch_info[2] = 1 + G->launches_pull;
    launch_info[4] = G->k1 ? 1 + G->launches_push1 : launch_info[1];
    launch_info[5] = h.tiny ? 1 + G->launches_tiny : launch_info[1];
    return GB_OK;
  }
  // one readback: iteration count and up to 21 decisions
  int64_t* pin = pinned_slots(ctx);
  GB_CUDA(ctx, cudaMemcpyAsync(pin, log, sizeof(int64_t) * (1 + 3 * first), cudaMemcpyDeviceToHost, s));
  GB_CUDA(ctx, cudaStreamSynchronize(s));
  const int64_t iters = pin[0];
  for (int64_t i = 0; i < iters && i < first; ++i) {
    log_dir[i] = (int32_t)pin[1 + 3 * i];
    log_nvals[i] = pin[2 + 3 * i];
    log_est[i] = pin[3 + 3 * i];
  }
  if (iters > first) {
    std::vector<int64_t> rest(3 * (iters - first));
    GB_CUDA(ctx, cudaMemcpyAsync(rest.data(), log + 1 + 3 * first, sizeof(int64_t) * rest.size(),
                                 cudaMemcpyDeviceToHost, s));
    GB_CUDA(ctx, cudaStreamSynchronize(s));
    for (int64_t i = first; i < iters; ++i) {
      log_dir[i] = (int32_t)rest[3 * (i - first)];
      log_nvals[i] = rest[3 * (i - first) + 1];
      log_est[i] = rest[3 * (i - first) + 2];
    }
  }
  *iters_out = iters;
  int64_t nl = G->launches_fixed;
  for (int64_t i = 0; i < iters; ++i)
    nl += 1 + (log_dir[i] != GB_DIR_PUSH ? G->launches_pull
               : (G->k1 && log_nvals[i] == 1) ? G->launches_push1
               : (h.tiny && log_nvals[i] <= kTinyK) ? G->launches_tiny : G->launches_push);
  nl += (G->unroll - iters % G->unroll) % G->unroll;  // no-op g_steps of the last pass
  count_launch(ctx, (int)nl);
  return GB_OK;
}

}  // namespace gb

using namespace gb;

extern "C" {

int32_t gb_decide_direction(int64_t nnz, int64_t nrows, int64_t nnz_u, double ratio,
                            int32_t policy, int64_t* estimate_out) {
  // kernels.py:108-126.  d*nnz_u is rounded half-to-even like Python round():
  // nearbyint() under the default FE_TONEAREST mode.
  const double d = nrows ? (double)nnz / (double)nrows : 0.0;
  const int64_t est = (int64_t)nearbyint(d * (double)nnz_u);
  const double thr = (double)nnz * ratio;
  if (estimate_out) *estimate_out = est;
  if (policy == GB_DIR_PUSH) return GB_DIR_PUSH;
  if (policy == GB_DIR_PULL) return GB_DIR_PULL;
  return (double)est > thr ? GB_DIR_PULL : GB_DIR_PUSH;
}

}  // extern "C"

namespace gb {

// A persistent cooperative kernel running every phase between grid barriers
// was built and measured here (s24: 1.38 ms against 1.09 ms for the graph):
// inside it the level-2 expansion took 0.84-0.90 ms instead of 0.55 ms -- the
// kernel's register cap is the maximum over all phases (pull, scans) and its
// static shared memory shrinks the L1 that holds the hot visited prefix.
enum { kEngineGraph = 0, kEngineHost = 1 };
static int g_bfs_engine = -1;  // -1: from the environment

static int bfs_engine_current() {
  if (g_bfs_engine < 0)
    g_bfs_engine = getenv("GB_BFS_GRAPH") && atoi(getenv("GB_BFS_GRAPH")) == 0 ? kEngineHost
                                                                               : kEngineGraph;
  return g_bfs_engine;
}

constexpr gb_status kTooDeep = -1000;  // internal: 16-bit levels would saturate

template <class LT>
static gb_status bfs_host_loop(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull,
                               const uint32_t* pull_nonempty, const int32_t* rank, const OrderedAux* aux, int64_t source,
                               int64_t max_iters, double ratio, int32_t policy, int64_t* levels_out,
                               int32_t* log_dir, int64_t* log_nvals, int64_t* log_est,
                               int64_t* iters_out) {
  const int64_t n = push->nrows;
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  // relabelled runs keep int32 levels by new id and unpermute at the end
  LT* levels = reinterpret_cast<LT*>(levels_out);
  if (rank) {
    // host-driven loop over the relabelled graph: internal levels by new id
    int32_t r = 0;
    GB_CUDA(ctx, cudaMemcpyAsync(&r, rank + source, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    GB_CUDA(ctx, cudaStreamSynchronize(s));
    source = r;
    levels = ar.alloc<LT>(n);
  }
  const int64_t reach = aux ? aux->reach : n;
  uint32_t* vbm = ar.alloc<uint32_t>(W);
  uint32_t* fbm[2] = {ar.alloc<uint32_t>(W), ar.alloc<uint32_t>(W)};
  int32_t* F = ar.alloc<int32_t>(n);
  uint32_t* vprev = ar.alloc<uint32_t>(W);
  // cnt[0..1]: frontier counters (alternating); cnt[2]: dense visited prefix
  unsigned long long* cnt = ar.alloc<unsigned long long>(3);
  // push scratch of the ordered path (same kernels as the graph engine)
  const bool ordered_push = rank && !push_smem_enabled();
  int64_t *rowstart = nullptr, *Sx = nullptr, *part = nullptr, *tbase = nullptr, *queue = nullptr;
  int32_t* tfirst = nullptr;
  const int32_t* samp = aux && use_samples() ? aux->samp : nullptr;
  if (ordered_push) {
    rowstart = ar.alloc<int64_t>(n + 1);
    Sx = ar.alloc<int64_t>(n + 1);
    part = ar.alloc<int64_t>(kGScanBlocks + 1);
    queue = ar.alloc<int64_t>(4 * stamp_queue_cap(push->nnz));
    tfirst = ar.alloc<int32_t>(push->nnz / kWarpTile + 2);
    tbase = ar.alloc<int64_t>(push->nnz / kWarpTile + 2);
  }
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(levels, 0, sizeof(LT) * n, s));
  GB_CUDA(ctx, cudaMemsetAsync(vbm, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(fbm[0], 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(vprev, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(cnt, 0, 24, s));
  bfs_init<<<1, 1, 0, s>>>(source, levels, vbm, vprev, fbm[0], F);
  int64_t X = 0;  // every vertex below X is visited (ordered graphs)
  unsigned long long* xmin = rank ? cnt + 2 : nullptr;
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 6);  // 5 memsets + init

  const EdgeOn push_on{push->values, push->dtype};
  const EdgeOn pull_on{pull ? pull->values : nullptr, pull ? pull->dtype : 0};
  const bool push_dead = !push->values && push->iso_i64 == 0 && push->iso_f64 == 0.0;
  const bool pull_dead = pull && !pull->values && pull->iso_i64 == 0 && pull->iso_f64 == 0.0;
  int64_t K = 1, depth = 1, iters = 0;
  int cur = 0;
  for (int64_t it = 0; it < max_iters; ++it) {
    if constexpr (sizeof(LT) == 2) {
      if (it >= kNarrowLevelIters) return kTooDeep;
    }
    int64_t est = 0;
    const int32_t dir = gb_decide_direction(push->nnz, push->nrows, K, ratio, policy, &est);
    log_dir[it] = dir;
    log_nvals[it] = K;
    log_est[it] = est;
    iters = it + 1;
    unsigned long long* c = cnt + (it & 1);
    unsigned long long* c_next = cnt + ((it + 1) & 1);
    if (dir == GB_DIR_PULL) {
      if (!pull) return set_error(ctx, GB_ERR_FORMAT, "column-oriented storage missing");
      if (pull_dead) {
        GB_CUDA(ctx, cudaMemsetAsync(fbm[cur ^ 1], 0, sizeof(uint32_t) * W, s));
        GB_CUDA(ctx, cudaMemsetAsync(c, 0, 8, s));
        GB_CUDA(ctx, cudaMemsetAsync(c_next, 0, 8, s));
      } else {
        if (xmin) GB_CUDA(ctx, cudaMemsetAsync(xmin, 0xff, 8, s));
        const int grid = grid_for(ctx, W, 256, 8);
        const int ps = prof_begin(ctx, PROF_BFS_PULL, K);
        bfs_pull<<<grid, 256, 0, s>>>(n, dval(depth + 1), pull->offsets, pull->indices, pull_on,
                                      pull_nonempty, vbm, vprev, fbm[cur], fbm[cur ^ 1], pval(levels), F,
                                      c, c_next, 0, (W + 31) / 32, xmin);
        prof_end(ctx, ps);
        count_launch(ctx, 1);
      }
    } else {
      if (!push_dead && ordered_push) {
        // the graph engine's kernels: sorted rows skip the dense visited prefix
        g_scan_partials<<<kGScanBlocks, kGScanThreads, 0, s>>>(dval(K), F, push->offsets,
                                                               push->indices,
                                                               dval(prefix_mode() == 1 ? X : 0),
                                                               cut_lo(), cut_hi(), samp,
                                                               rowstart, Sx,
                                                               part);
        g_scan_apply<<<kApplyBlocks, kGScanThreads, 0, s>>>(dval(K), part, rowstart, Sx, tfirst,
                                                            tbase, queue);
        g_scan_stamp<<<grid_for(ctx, (int64_t)1 << 40, 256, 8), 256, 0, s>>>(part, queue, tfirst,
                                                                              tbase);
        if (prof_enabled(ctx)) {
          int64_t E = 0;
          GB_TRY(read_i64(ctx, Sx + K, &E));
          prof_end(ctx, prof_begin(ctx, PROF_BFS_PUSH_EDGES, E));
        }
        const int ps = prof_begin(ctx, PROF_BFS_PUSH, K);
        LbsPlan plan;
        plan.K = K;
        plan.rowstart = rowstart;
        plan.S = Sx;
        plan.tile_first = tfirst;
        plan.tile_base = tbase;
        GB_TRY(launch_push(ctx, K, plan, push, push_on, vbm, prefix_mode() == 2 ? X : 0));
        prof_end(ctx, ps);
        count_launch(ctx, 4);  // scan (3), expand
      } else if (!push_dead) {
        LbsPlan plan;
        GB_TRY(lbs_prepare(ctx, ar, K, F, push->offsets, push->nnz, &plan, kWarpTile));
        const int ps = prof_begin(ctx, PROF_BFS_PUSH, K);
        if (rank) GB_TRY(launch_push_smem(ctx, K, plan, push, push_on, vbm, vprev));
        else GB_TRY(launch_push(ctx, K, plan, push, push_on, vbm));
        prof_end(ctx, ps);
        count_launch(ctx, 5);  // degrees, scan (2), tile_first, expand
      }
      if (xmin) GB_CUDA(ctx, cudaMemsetAsync(xmin, 0xff, 8, s));
      const int pf = prof_begin(ctx, PROF_BFS_FINALIZE, K);
      bfs_finalize<<<grid_for(ctx, W, 256, 8), 256, 0, s>>>(n, dval(depth + 1), vbm, vprev, fbm[cur ^ 1],
                                                         pval(levels), F, c, c_next, nullptr, xmin);
      prof_end(ctx, pf);
      count_launch(ctx, 1);
    }
    GB_LAUNCH_CHECK(ctx);
    GB_TRY(read_i64(ctx, (const int64_t*)c, &K));
    if (xmin) {
      int64_t x = 0;
      GB_TRY(read_i64(ctx, (const int64_t*)xmin, &x));
      X = (uint64_t)x < (uint64_t)n ? x : n;
    }
    cur ^= 1;
    if (K == 0) break;
    ++depth;
    if (it + 1 == max_iters) {
      // loop cap reached: the reference never stamps the last frontier
      // (its assign happens at the start of the next iteration)
      bfs_unstamp<<<grid_for(ctx, K, 256), 256, 0, s>>>(dval(K), F, levels);
      GB_LAUNCH_CHECK(ctx);
      count_launch(ctx, 1);
    }
  }
  *iters_out = iters;
  if constexpr (sizeof(LT) <= 4) {
    if (rank) {
      const int pu = prof_begin(ctx, PROF_BFS_UNPERMUTE, n);
      bfs_unpermute<<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(n, rank, levels, reach,
                                                             dval(source), pval(levels_out));
      prof_end(ctx, pu);
      GB_LAUNCH_CHECK(ctx);
      count_launch(ctx, 1);
    }
  }
  return GB_OK;
}

static gb_status bfs_run(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull,
                         const uint32_t* pull_nonempty, const int32_t* rank, int64_t source,
                         int64_t max_iters, double ratio, int32_t policy, int64_t* levels_out,
                         int32_t* log_dir, int64_t* log_nvals, int64_t* log_est, int64_t* iters_out) {
  const int64_t n = push->nrows;
  if (source < 0 || source >= n) return set_error(ctx, GB_ERR_INDEX, "source %lld out of range", (long long)source);
  if (rank && pull && bfs_engine_current() == kEngineGraph && !prof_enabled(ctx) && max_iters >= 1 &&
      n <= bfs_coop_max_n()) {
    // a small relabelled graph: the whole traversal in one cooperative kernel
    Arena ar(ctx);
    int64_t* log = ar.alloc<int64_t>(1 + 3 * max_iters);
    GB_ARENA_CHECK(ctx, ar);
    const gb_status st = bfs_coop_run(ctx, push, pull, pull_nonempty, rank, source, max_iters,
                                      ratio, policy, levels_out, log);
    if (st == GB_OK) {
      int64_t iters = 0;
      GB_TRY(read_i64(ctx, log, &iters));
      std::vector<int64_t> raw(3 * (iters > 0 ? iters : 1));
      if (iters > 0) {
        GB_CUDA(ctx, cudaMemcpyAsync(raw.data(), log + 1, sizeof(int64_t) * 3 * iters,
                                     cudaMemcpyDeviceToHost, stream_of(ctx)));
        GB_CUDA(ctx, cudaStreamSynchronize(stream_of(ctx)));
      }
      for (int64_t i = 0; i < iters; ++i) {
        log_dir[i] = (int32_t)raw[3 * i];
        log_nvals[i] = raw[3 * i + 1];
        log_est[i] = raw[3 * i + 2];
      }
      *iters_out = iters;
      return GB_OK;
    }
    if (st != GB_ERR_UNSUPPORTED) return st;
  }
  const OrderedAux* aux = nullptr;
  if (rank) GB_TRY(ordered_aux(ctx, push, pull, &aux));
  // Device-driven loop (one graph launch) unless profiling per kernel, the
  // pull orientation is missing (the host loop reports that error when pull
  // is chosen), or the engine is pinned (gb_bfs_engine; GB_BFS_GRAPH=0).
  if (pull && bfs_engine_current() == kEngineGraph && !prof_enabled(ctx) && max_iters >= 1 &&
      max_iters <= kGraphMaxCap) {
    const gb_status st = bfs_graph_run(ctx, push, pull, pull_nonempty, rank, aux, source, max_iters,
                                       ratio, policy, levels_out, log_dir, log_nvals, log_est,
                                       iters_out);
    // 16-bit levels saturate: a relabelled run this deep is redone with int32
    const bool deep = st == GB_OK && rank && *iters_out >= kNarrowLevelIters;
    if (deep)
      return bfs_host_loop<int32_t>(ctx, push, pull, pull_nonempty, rank, aux, source, max_iters,
                                    ratio, policy, levels_out, log_dir, log_nvals, log_est,
                                    iters_out);
    if (st != GB_ERR_UNSUPPORTED) return st;
  }
  if (rank) {
    const gb_status st = bfs_host_loop<uint16_t>(ctx, push, pull, pull_nonempty, rank, aux, source,
                                                max_iters, ratio, policy, levels_out, log_dir,
                                                log_nvals, log_est, iters_out);
    if (st != kTooDeep) return st;
    return bfs_host_loop<int32_t>(ctx, push, pull, pull_nonempty, rank, aux, source, max_iters, ratio,
                                  policy, levels_out, log_dir, log_nvals, log_est, iters_out);
  }
  return bfs_host_loop<int64_t>(ctx, push, pull, pull_nonempty, rank, aux, source, max_iters, ratio,
                                policy, levels_out, log_dir, log_nvals, log_est, iters_out);
}

}  // namespace gb

extern "C" {

int32_t gb_bfs_engine(int32_t engine) {
  const int32_t prev = bfs_engine_current();
  if (engine >= kEngineGraph && engine <= kEngineHost) g_bfs_engine = engine;
  return prev;
}

gb_status gb_bfs(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull,
                 const uint32_t* pull_nonempty, int64_t source, int64_t max_iters,
                 double ratio, int32_t policy, int64_t* levels, int32_t* log_dir,
                 int64_t* log_nvals, int64_t* log_est, int64_t* iters_out) {
  return bfs_run(ctx, push, pull, pull_nonempty, nullptr, source, max_iters, ratio, policy, levels,
                 log_dir, log_nvals, log_est, iters_out);
}

gb_status gb_bfs_ordered(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull,
                         const uint32_t* pull_nonempty, const int32_t* rank, int64_t source,
                         int64_t max_iters, double ratio, int32_t policy, int64_t* levels,
                         int32_t* log_dir, int64_t* log_nvals, int64_t* log_est,
                         int64_t* iters_out) {
  if (!rank) return set_error(ctx, GB_ERR_ARG, "gb_bfs_ordered needs the vertex rank array");
  return bfs_run(ctx, push, pull, pull_nonempty, rank, source, max_iters, ratio, policy, levels,
                 log_dir, log_nvals, log_est, iters_out);
}

gb_status gb_bfs_ordered_async(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull,
                               const uint32_t* pull_nonempty, const int32_t* rank, int64_t source,
                               int64_t max_iters, double ratio, int32_t policy, int64_t* levels,
                               int64_t* log_dev, int64_t* log_host, int64_t* launch_info) {
  if (!rank) return set_error(ctx, GB_ERR_ARG, "gb_bfs_ordered_async needs the vertex rank array");
  const int64_t n = push->nrows;
  if (source < 0 || source >= n)
    return set_error(ctx, GB_ERR_INDEX, "source %lld out of range", (long long)source);
  if (max_iters < 1) return set_error(ctx, GB_ERR_ARG, "max_iters must be >= 1");
  // a small graph: the whole traversal in one cooperative kernel
  if (pull && bfs_engine_current() == kEngineGraph && !prof_enabled(ctx) && n <= bfs_coop_max_n()) {
    const gb_status st = bfs_coop_run(ctx, push, pull, pull_nonempty, rank, source, max_iters,
                                      ratio, policy, levels, log_dev);
    if (st == GB_OK) {
      const int64_t first = max_iters < kLogPrefix ? max_iters : kLogPrefix;
      GB_CUDA(ctx, cudaMemcpyAsync(log_host, log_dev, sizeof(int64_t) * (1 + 3 * first),
                                   cudaMemcpyDeviceToHost, stream_of(ctx)));
      // its one launch is counted already: nothing to book when the log is read
      for (int i = 0; i < 6; ++i) launch_info[i] = 0;
      launch_info[3] = 1;
      return GB_OK;
    }
    if (st != GB_ERR_UNSUPPORTED) return st;
  }
  // the graph engine, with a loop cap its 16-bit levels cannot exceed
  if (pull && bfs_engine_current() == kEngineGraph && !prof_enabled(ctx) &&
      max_iters <= kGraphMaxCap && max_iters < kNarrowLevelIters) {
    const OrderedAux* aux = nullptr;
    GB_TRY(ordered_aux(ctx, push, pull, &aux));
    int64_t iters = 0;
    const gb_status st = bfs_graph_run(ctx, push, pull, pull_nonempty, rank, aux, source,
                                       max_iters, ratio, policy, levels, nullptr, nullptr,
                                       nullptr, &iters, log_dev, log_host, launch_info);
    if (st != GB_ERR_UNSUPPORTED) return st;
  }
  // otherwise synchronously: the raw log to log_dev, its prefix to log_host
  std::vector<int32_t> dir(max_iters);
  std::vector<int64_t> nv(max_iters), est(max_iters);
  int64_t iters = 0;
  GB_TRY(bfs_run(ctx, push, pull, pull_nonempty, rank, source, max_iters, ratio, policy, levels,
                 dir.data(), nv.data(), est.data(), &iters));
  std::vector<int64_t> raw(1 + 3 * iters);
  raw[0] = iters;
  for (int64_t i = 0; i < iters; ++i) {
    raw[1 + 3 * i] = dir[i];
    raw[2 + 3 * i] = nv[i];
    raw[3 + 3 * i] = est[i];
  }
  const int64_t first = iters < kLogPrefix ? iters : kLogPrefix;
  for (int64_t i = 0; i < 1 + 3 * first; ++i) log_host[i] = raw[i];
  GB_CUDA(ctx, cudaMemcpyAsync(log_dev, raw.data(), sizeof(int64_t) * raw.size(),
                               cudaMemcpyHostToDevice, stream_of(ctx)));
  GB_CUDA(ctx, cudaStreamSynchronize(stream_of(ctx)));
  // the synchronous path counted its own launches
  launch_info[0] = 0;
  launch_info[1] = 0;
  launch_info[2] = 0;
  launch_info[3] = 2;
  launch_info[4] = 0;
  launch_info[5] = 0;
  return GB_OK;
}

void gb_count_launches(gb_ctx* ctx, int64_t n) { count_launch(ctx, (int)n); }

// ---------------------------------------------------------------------------
// 1D-partitioned BFS steps (one rank of P; the host loop and the NCCL
// exchange of the new-frontier bitmap live in distributed.py).  Rank p owns
// vertices [lo, hi) (lo, hi multiples of 1024 except hi = n) and stores
//   rowblock: rows lo..hi-1 of A^T (in-edges of owned vertices) for pull,
//   colblock: all n rows of A restricted to columns in [lo, hi) for push.
// Every bitmap / levels / frontier buffer is global-sized and replicated.
// ---------------------------------------------------------------------------

__global__ void bfs_collect(int64_t w_lo, int64_t w_hi, const uint32_t* __restrict__ vbm,
                            const uint32_t* __restrict__ vprev, uint32_t* __restrict__ xbm) {
  for (int64_t w = w_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < w_hi;
       w += (int64_t)gridDim.x * blockDim.x)
    xbm[w] = vbm[w] & ~vprev[w];
}

gb_status gb_bfs_dist_init(gb_ctx* ctx, int64_t n, int64_t source, int64_t* levels,
                           uint32_t* vbm, uint32_t* vprev, uint32_t* fbm, int32_t* F) {
  if (source < 0 || source >= n) return set_error(ctx, GB_ERR_INDEX, "source out of range");
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  GB_CUDA(ctx, cudaMemsetAsync(levels, 0, sizeof(int64_t) * n, s));
  GB_CUDA(ctx, cudaMemsetAsync(vbm, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(vprev, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(fbm, 0, sizeof(uint32_t) * W, s));
  bfs_init<<<1, 1, 0, s>>>(source, levels, vbm, vprev, fbm, F);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 5);
  return GB_OK;
}

gb_status gb_bfs_dist_push(gb_ctx* ctx, const gb_csr* colblock, int64_t K, const int32_t* F,
                           uint32_t* vbm) {
  if (K == 0 || colblock->nnz == 0) return GB_OK;
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  LbsPlan plan;
  GB_TRY(lbs_prepare(ctx, ar, K, F, colblock->offsets, colblock->nnz, &plan, kWarpTile));
  const EdgeOn on{colblock->values, colblock->dtype};
  const int ps = prof_begin(ctx, PROF_BFS_PUSH, K);
  GB_TRY(launch_push(ctx, K, plan, colblock, on, vbm));
  prof_end(ctx, ps);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 5);
  return GB_OK;
}

gb_status gb_bfs_dist_collect(gb_ctx* ctx, int64_t n, int64_t lo, int64_t hi,
                              const uint32_t* vbm, const uint32_t* vprev, uint32_t* xbm) {
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  const int64_t w_lo = lo / 32, w_hi = (hi + 31) / 32;
  GB_CUDA(ctx, cudaMemsetAsync(xbm, 0, sizeof(uint32_t) * W, s));
  if (w_hi > w_lo)
    bfs_collect<<<grid_for(ctx, w_hi - w_lo, 256), 256, 0, s>>>(w_lo, w_hi, vbm, vprev, xbm);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 2);
  return GB_OK;
}

gb_status gb_bfs_dist_pull(gb_ctx* ctx, const gb_csr* rowblock, int64_t lo, int64_t hi,
                           const uint32_t* nonempty_block, int64_t n, int64_t depth,
                           uint32_t* vbm, uint32_t* vprev, const uint32_t* fbm, uint32_t* xbm,
                           int64_t* levels) {
  if (lo % 1024) return set_error(ctx, GB_ERR_ARG, "partition start must be a multiple of 1024");
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  int32_t* F = ar.alloc<int32_t>(hi - lo + 1);
  unsigned long long* cnt = ar.alloc<unsigned long long>(2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(xbm, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(cnt, 0, 16, s));
  if (hi > lo && rowblock->nnz) {
    const EdgeOn on{rowblock->values, rowblock->dtype};
    // rebase so global vertex ids index the block's offsets / nonempty words
    const int64_t* off = rowblock->offsets - lo;
    const uint32_t* ne = nonempty_block - lo / 32;
    const int64_t g_lo = lo / 1024, g_hi = (hi + 1023) / 1024;
    const int ps = prof_begin(ctx, PROF_BFS_PULL, 0);
    bfs_pull<<<grid_for(ctx, (g_hi - g_lo) * 32, 256, 8), 256, 0, s>>>(
        hi, dval(depth), off, rowblock->indices, on, ne, vbm, vprev, fbm, xbm, pval(levels), F, cnt, cnt + 1,
        g_lo, g_hi, nullptr);
    prof_end(ctx, ps);
  }
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 3);
  return GB_OK;
}

gb_status gb_bfs_dist_apply(gb_ctx* ctx, int64_t n, int64_t depth, const uint32_t* xbm,
                            uint32_t* vbm, uint32_t* vprev, uint32_t* fbm, int64_t* levels,
                            int32_t* F, int64_t* K_host) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  unsigned long long* cnt = ar.alloc<unsigned long long>(2);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cudaMemsetAsync(cnt, 0, 16, s));
  bfs_finalize<<<grid_for(ctx, W, 256, 8), 256, 0, s>>>(n, dval(depth), vbm, vprev, fbm, pval(levels), F,
                                                        cnt, cnt + 1, xbm, nullptr);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 2);
  if (!K_host) return GB_OK;  // the frontier size is known from the exchange: stay asynchronous
  return read_i64(ctx, (const int64_t*)cnt, K_host);
}

gb_status gb_bfs_dist_unstamp(gb_ctx* ctx, int64_t K, const int32_t* F, int64_t* levels) {
  if (K <= 0) return GB_OK;
  bfs_unstamp<<<grid_for(ctx, K, 256), 256, 0, stream_of(ctx)>>>(dval(K), F, levels);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

// ---- frontier exchange (distributed.FrontierExchange) ----------------------
// After a level each rank holds its OWNED new-frontier words xbm[w_lo, w_hi)
// (words outside are zero).  The exchange replicates the union: a dense
// allgather of the owned word slices when the frontier is large (|f|*32 > n,
// SURVEY §8(e)), else an allgather(v) of the owned vertex ids.

// count the owned new vertices and list them (unordered)
__global__ void dist_owned_ids(int64_t w_lo, int64_t w_hi, const uint32_t* __restrict__ xbm,
                               int32_t* __restrict__ ids, unsigned long long* __restrict__ count) {
  for (int64_t w = w_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < w_hi;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t b = xbm[w];
    if (!b) continue;
    unsigned long long at = atomicAdd(count, (unsigned long long)__popc(b));
    while (b) {
      const int k = __ffs(b) - 1;
      b &= b - 1;
      ids[at++] = (int32_t)(w * 32 + k);
    }
  }
}

__global__ void dist_pack_words(int64_t w_lo, int64_t w_hi, int64_t wmax,
                                const uint32_t* __restrict__ xbm, uint32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < wmax;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = w_lo + i < w_hi ? xbm[w_lo + i] : 0u;
}

// xbm[wb[p] + i] = gathered[p * wmax + i] for every rank p (slices tile [0, W))
__global__ void dist_unpack_words(int32_t P, int64_t wmax, const int64_t* __restrict__ wb,
                                  const uint32_t* __restrict__ gathered, uint32_t* __restrict__ xbm) {
  const int64_t total = (int64_t)P * wmax;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(j / wmax);
    const int64_t i = j - (int64_t)p * wmax;
    if (wb[p] + i < wb[p + 1]) xbm[wb[p] + i] = gathered[j];
  }
}

// set the bits of every gathered id (rank p's ids are gathered[p*kmax, +counts[p]))
__global__ void dist_set_ids(int32_t P, int64_t kmax, const int64_t* __restrict__ counts,
                             const int32_t* __restrict__ gathered, uint32_t* __restrict__ xbm) {
  const int64_t total = (int64_t)P * kmax;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(j / kmax);
    if (j - (int64_t)p * kmax < counts[p]) {
      const int32_t v = gathered[j];
      atomicOr(xbm + (v >> 5), 1u << (v & 31));
    }
  }
}

gb_status gb_bfs_dist_owned(gb_ctx* ctx, int64_t lo, int64_t hi, const uint32_t* xbm,
                            int32_t* ids, int64_t* count_dev) {
  cudaStream_t s = stream_of(ctx);
  GB_CUDA(ctx, cudaMemsetAsync(count_dev, 0, sizeof(int64_t), s));
  const int64_t w_lo = lo / 32, w_hi = (hi + 31) / 32;
  if (w_hi > w_lo)
    dist_owned_ids<<<grid_for(ctx, w_hi - w_lo, 256), 256, 0, s>>>(
        w_lo, w_hi, xbm, ids, (unsigned long long*)count_dev);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 2);
  return GB_OK;
}

gb_status gb_bfs_dist_pack_words(gb_ctx* ctx, int64_t lo, int64_t hi, int64_t wmax,
                                 const uint32_t* xbm, uint32_t* out) {
  if (wmax <= 0) return GB_OK;
  dist_pack_words<<<grid_for(ctx, wmax, 256), 256, 0, stream_of(ctx)>>>(lo / 32, (hi + 31) / 32,
                                                                         wmax, xbm, out);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

gb_status gb_bfs_dist_unpack_words(gb_ctx* ctx, int32_t P, int64_t wmax, const int64_t* wb,
                                   const uint32_t* gathered, uint32_t* xbm) {
  if (wmax <= 0 || P <= 0) return GB_OK;
  dist_unpack_words<<<grid_for(ctx, (int64_t)P * wmax, 256), 256, 0, stream_of(ctx)>>>(
      P, wmax, wb, gathered, xbm);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

gb_status gb_bfs_dist_set_ids(gb_ctx* ctx, int64_t n, int32_t P, int64_t kmax,
                              const int64_t* counts, const int32_t* gathered, uint32_t* xbm) {
  cudaStream_t s = stream_of(ctx);
  GB_CUDA(ctx, cudaMemsetAsync(xbm, 0, sizeof(uint32_t) * ((n + 31) / 32), s));
  if (kmax > 0 && P > 0)
    dist_set_ids<<<grid_for(ctx, (int64_t)P * kmax, 256), 256, 0, s>>>(P, kmax, counts, gathered,
                                                                       xbm);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 2);
  return GB_OK;
}

// ---- device-resident levels (distributed.bfs_partitioned_device) ---------
// The same level steps with every scalar the host used to hold -- the
// frontier size K, the depth, the iteration, the direction -- kept in a
// per-rank device state: the reference rule is evaluated on the device, the
// push / pull kernels run or return by the state's mode, and the exchange is
// the dense allgather of owned word slices (fixed size, so no count has to
// reach the host).  The host enqueues level after level and only watches a
// pinned copy of `done` a few levels behind.
struct DistBfsState {
  int64_t K;        // frontier size (replicated)
  int64_t Kpush;    // K when this level pushes, else 0
  int64_t mode;     // 0 none (finished), 1 push, 2 pull
  int64_t dnext;    // level stamped on this level's new vertices
  int64_t it, max_iters, done, Kun, iters;
  int64_t n, nnz, policy;
  double ratio;
  unsigned long long cnt[2];
  unsigned long long nlong;
  int64_t xcur;                // dense visited prefix: every vertex below it is visited
  unsigned long long xnext;    // ... after the level (finalize's atomicMin target)
};
static_assert(sizeof(DistBfsState) <= 24 * sizeof(int64_t), "state fits int64[24]");

__global__ void dist_state_init(DistBfsState* st, int64_t n, int64_t nnz, int64_t max_iters,
                                double ratio, int64_t policy, int64_t* log) {
  st->K = 1;
  st->Kpush = 0;
  st->mode = 0;
  st->dnext = 2;
  st->it = 0;
  st->max_iters = max_iters;
  st->done = max_iters <= 0;
  st->Kun = 0;
  st->iters = 0;
  st->n = n;
  st->nnz = nnz;
  st->policy = policy;
  st->ratio = ratio;
  st->cnt[0] = st->cnt[1] = 0;
  st->nlong = 0;
  st->xcur = 0;
  st->xnext = ~0ull;
  log[0] = 0;
}

// the reference rule (kernels.py:108-126) on the replicated K; raw log
// entries (dir, K, estimate) after the count, like gb_bfs_ordered_async's
__global__ void dist_decide(DistBfsState* st, int64_t* log) {
  st->nlong = 0;
  if (st->done) {
    st->mode = 0;
    st->Kpush = 0;
    return;
  }
  const double d = st->n ? (double)st->nnz / (double)st->n : 0.0;
  const int64_t est = (int64_t)rint(d * (double)st->K);  // Python round: half-even
  int32_t dir = (double)est > (double)st->nnz * st->ratio ? GB_DIR_PULL : GB_DIR_PUSH;
  if (st->policy == GB_DIR_PUSH) dir = GB_DIR_PUSH;
  if (st->policy == GB_DIR_PULL) dir = GB_DIR_PULL;
  const int64_t it = st->it;
  log[1 + 3 * it] = dir;
  log[2 + 3 * it] = st->K;
  log[3 + 3 * it] = est;
  log[0] = it + 1;
  st->mode = dir == GB_DIR_PULL ? 2 : 1;
  st->Kpush = dir == GB_DIR_PULL ? 0 : st->K;
}

// push over the column block: warp per frontier entry (K from the state),
// lists longer than kDistLong edges cut into kDistChunk-edge tasks
#ifndef GB_DIST_LONG
#define GB_DIST_LONG 4096
#endif
constexpr int64_t kDistLong = GB_DIST_LONG, kDistChunk = 512;
struct DistMark {
  const int32_t* idx;
  EdgeOn on;
  uint32_t* vbm;
  __device__ __forceinline__ void operator()(int64_t p) const {
    if (!on(p)) return;
    const int32_t v = __ldg(idx + p);
    const uint32_t bit = 1u << (v & 31);
    if (!(ld_probe(vbm + (v >> 5)) & bit)) atomicOr(vbm + (v >> 5), bit);
  }
};

// first position of idx[lo, hi) (sorted) holding a column >= key: 32-ary
// warp search, one coalesced round of probes per factor of 32
__device__ __forceinline__ int64_t warp_lower_bound(const int32_t* __restrict__ idx, int64_t lo,
                                                    int64_t hi, int32_t key, int lane) {
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = lo + lane * step;
    const uint32_t m = __ballot_sync(GB_FULL, p < hi && __ldg(idx + p) < key);
    if (!m) return lo;
    const int64_t last = lo + (int64_t)(__popc(m) - 1) * step;  // the last probe below key
    hi = min(hi, last + step);
    lo = last + 1;
  }
  const int64_t p = lo + lane;
  return lo + __popc(__ballot_sync(GB_FULL, p < hi && __ldg(idx + p) < key));
}

// cut: the rows are sorted -- skip each list's entries below the dense
// visited prefix (the single-GPU push's prefix cut, on the column block)
__global__ void __launch_bounds__(256)
dist_push_short(DistBfsState* st, const int32_t* __restrict__ F, const int64_t* __restrict__ off,
                int32_t* __restrict__ longk, int32_t* __restrict__ longc, DistMark op, int cut) {
  const int lane = threadIdx.x & 31;
  const int64_t K = st->Kpush;
  const int32_t xc = cut ? (int32_t)st->xcur : 0;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = w0; k < K; k += nw) {
    const int32_t j = F[k];
    int64_t lo = off[j];
    const int64_t hi = off[j + 1];
    if (xc > 0 && lo < hi && __ldg(op.idx + lo) < xc) lo = warp_lower_bound(op.idx, lo, hi, xc, lane);
    if (hi - lo > kDistLong) {
      const int64_t nc = (hi - lo + kDistChunk - 1) / kDistChunk;
      unsigned long long at = 0;
      if (lane == 0) at = atomicAdd(&st->nlong, (unsigned long long)nc);
      at = __shfl_sync(GB_FULL, at, 0);
      for (int64_t c = lane; c < nc; c += 32) {
        longk[at + c] = (int32_t)k;
        longc[at + c] = (int32_t)c;
      }
      continue;
    }
    for (int64_t p = lo + lane; p < hi; p += 32) op(p);
  }
}

__global__ void __launch_bounds__(256)
dist_push_long(const DistBfsState* st, const int32_t* __restrict__ longk,
               const int32_t* __restrict__ longc, const int32_t* __restrict__ F,
               const int64_t* __restrict__ off, DistMark op, int cut) {
  const int lane = threadIdx.x & 31;
  const int64_t L = (int64_t)st->nlong;
  const int32_t xc = cut ? (int32_t)st->xcur : 0;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = w0; t < L; t += nw) {
    const int32_t j = F[longk[t]];
    int64_t base = off[j];
    const int64_t end = off[j + 1];
    // the same cut push_short chunked from
    if (xc > 0 && base < end && __ldg(op.idx + base) < xc)
      base = warp_lower_bound(op.idx, base, end, xc, lane);
    const int64_t lo = base + (int64_t)longc[t] * kDistChunk;
    const int64_t hi = min(end, lo + kDistChunk);
    for (int64_t p = lo + lane; p < hi; p += 32) op(p);
  }
}

__global__ void dist_collect_if(const DistBfsState* st, int64_t w_lo, int64_t w_hi,
                                const uint32_t* __restrict__ vbm,
                                const uint32_t* __restrict__ vprev, uint32_t* __restrict__ xbm) {
  if (st->mode != 1) return;
  for (int64_t w = w_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < w_hi;
       w += (int64_t)gridDim.x * blockDim.x)
    xbm[w] = vbm[w] & ~vprev[w];
}

__global__ void __launch_bounds__(256)
dist_pull_if(const DistBfsState* st, int64_t n, const int64_t* __restrict__ off,
             const int32_t* __restrict__ idx, EdgeOn on, const uint32_t* __restrict__ nonempty,
             uint32_t* __restrict__ vbm, uint32_t* __restrict__ vprev,
             const uint32_t* __restrict__ fbm, uint32_t* __restrict__ xbm,
             int64_t* __restrict__ levels, int32_t* __restrict__ F,
             unsigned long long* __restrict__ count, int64_t g_lo, int64_t g_hi) {
  if (st->mode != 2) return;
  pull_body(n, st->dnext, off, idx, on, nonempty, vbm, vprev, fbm, xbm, levels, F, count, g_lo,
            g_hi, nullptr);
}

// after finalize: the new K; the loop cap (the reference stamps the last
// frontier at the next iteration, which never runs: unstamp it)
__global__ void dist_advance(DistBfsState* st) {
  st->Kun = 0;
  const int64_t K = (int64_t)st->cnt[0];
  st->cnt[0] = st->cnt[1] = 0;
  // the dense visited prefix after this level (replicated: finalize scanned
  // the whole replicated bitmap)
  if (st->xnext < (unsigned long long)st->n) st->xcur = (int64_t)st->xnext;
  st->xnext = ~0ull;
  if (st->done) return;
  st->K = K;
  st->it += 1;
  st->iters = st->it;
  if (K == 0) {
    st->done = 1;
    return;
  }
  st->dnext += 1;
  if (st->it == st->max_iters) {
    st->Kun = K;
    st->done = 1;
  }
}


// ---- device-resident levels: entry points ----------------------------------
gb_status gb_bfs_dist_dev_init(gb_ctx* ctx, int64_t* state, int64_t* log, int64_t n, int64_t nnz,
                               int64_t source, int64_t max_iters, double ratio, int32_t policy,
                               int64_t* levels, uint32_t* vbm, uint32_t* vprev, uint32_t* fbm,
                               int32_t* F) {
  GB_TRY(gb_bfs_dist_init(ctx, n, source, levels, vbm, vprev, fbm, F));
  dist_state_init<<<1, 1, 0, stream_of(ctx)>>>(reinterpret_cast<DistBfsState*>(state), n, nnz,
                                                max_iters, ratio, policy, log);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 1);
  return GB_OK;
}

gb_status gb_bfs_dist_dev_level(gb_ctx* ctx, int64_t* state, int64_t* log,
                                const gb_csr* rowblock, const gb_csr* colblock, int64_t lo,
                                int64_t hi, const uint32_t* nonempty_block, int64_t n,
                                uint32_t* vbm, uint32_t* vprev, const uint32_t* fbm,
                                uint32_t* xbm, int64_t* levels, const int32_t* F,
                                int32_t prefix_cut) {
  if (lo % 1024) return set_error(ctx, GB_ERR_ARG, "partition start must be a multiple of 1024");
  auto* st = reinterpret_cast<DistBfsState*>(state);
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  const int64_t ntask = n + colblock->nnz / kDistChunk + 1;
  int32_t* longk = ar.alloc<int32_t>(ntask);
  int32_t* longc = ar.alloc<int32_t>(ntask);
  int32_t* Fp = ar.alloc<int32_t>(hi - lo + 1);  // the pull's own list (unused)
  unsigned long long* pc = ar.alloc<unsigned long long>(1);
  GB_ARENA_CHECK(ctx, ar);
  dist_decide<<<1, 1, 0, s>>>(st, log);
  GB_CUDA(ctx, cudaMemsetAsync(xbm, 0, sizeof(uint32_t) * W, s));
  GB_CUDA(ctx, cudaMemsetAsync(pc, 0, sizeof(unsigned long long), s));
  if (colblock->nnz) {
    const DistMark op{colblock->indices, EdgeOn{colblock->values, colblock->dtype}, vbm};
    dist_push_short<<<grid_for(ctx, n * 32, 256, 8), 256, 0, s>>>(st, F, colblock->offsets,
                                                                 longk, longc, op, prefix_cut);
    dist_push_long<<<grid_for(ctx, colblock->nnz / 16 + 32, 256, 8), 256, 0, s>>>(
        st, longk, longc, F, colblock->offsets, op, prefix_cut);
  }
  const int64_t w_lo = lo / 32, w_hi = (hi + 31) / 32;
  if (w_hi > w_lo)
    dist_collect_if<<<grid_for(ctx, w_hi - w_lo, 256), 256, 0, s>>>(st, w_lo, w_hi, vbm, vprev,
                                                                    xbm);
  if (hi > lo && rowblock->nnz) {
    const EdgeOn on{rowblock->values, rowblock->dtype};
    const int64_t* off = rowblock->offsets - lo;
    const uint32_t* ne = nonempty_block - lo / 32;
    const int64_t g_lo = lo / 1024, g_hi = (hi + 1023) / 1024;
    dist_pull_if<<<grid_for(ctx, (g_hi - g_lo) * 32, 256, 8), 256, 0, s>>>(
        st, hi, off, rowblock->indices, on, ne, vbm, vprev, fbm, xbm, levels, Fp, pc, g_lo, g_hi);
  }
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 7);
  return GB_OK;
}

gb_status gb_bfs_dist_dev_apply(gb_ctx* ctx, int64_t* state, int64_t n, const uint32_t* xbm,
                                uint32_t* vbm, uint32_t* vprev, uint32_t* fbm, int64_t* levels,
                                int32_t* F) {
  auto* st = reinterpret_cast<DistBfsState*>(state);
  cudaStream_t s = stream_of(ctx);
  const int64_t W = (n + 31) / 32;
  bfs_finalize<<<grid_for(ctx, W, 256, 8), 256, 0, s>>>(n, dptr(&st->dnext), vbm, vprev, fbm,
                                                        pval(levels), F, &st->cnt[0], &st->cnt[1],
                                                        xbm, &st->xnext);
  dist_advance<<<1, 1, 0, s>>>(st);
  bfs_unstamp<<<grid_for(ctx, n, 256, 4), 256, 0, s>>>(dptr(&st->Kun), F, levels);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 3);
  return GB_OK;
}

// Column block of a CSR: every row keeps only its entries with column in
// [lo, hi) (columns stay global).  Two passes: counts, then copy.
__global__ void colblock_count(int64_t n, const int64_t* __restrict__ off,
                               const int32_t* __restrict__ idx, int32_t lo, int32_t hi,
                               int64_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n; r += nw) {
    long long c = 0;
    for (int64_t p = off[r] + lane; p < off[r + 1]; p += 32) c += idx[p] >= lo && idx[p] < hi;
    c = warp_sum_ll(c);
    if (lane == 0) cnt[r] = c;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[n] = 0;
}

__global__ void colblock_fill(int64_t n, const int64_t* __restrict__ off,
                              const int32_t* __restrict__ idx, int32_t lo, int32_t hi,
                              const int64_t* __restrict__ out_off, int32_t* __restrict__ out_idx) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n; r += nw) {
    int64_t o = out_off[r];
    for (int64_t base = off[r]; base < off[r + 1]; base += 32) {
      const int64_t p = base + lane;
      const bool keep = p < off[r + 1] && idx[p] >= lo && idx[p] < hi;
      const uint32_t bal = __ballot_sync(GB_FULL, keep);
      if (keep) out_idx[o + __popc(bal & ((1u << lane) - 1u))] = idx[p];
      o += __popc(bal);
    }
  }
}

gb_status gb_csr_column_block(gb_ctx* ctx, const gb_csr* a, int64_t lo, int64_t hi,
                              int64_t* out_offsets, int32_t* out_indices, int64_t* nnz_host) {
  Arena ar(ctx);
  cudaStream_t s = stream_of(ctx);
  const int64_t n = a->nrows;
  int64_t* cnt = ar.alloc<int64_t>(n + 1);
  GB_ARENA_CHECK(ctx, ar);
  colblock_count<<<grid_for(ctx, n * 32, 256, 16), 256, 0, s>>>(n, a->offsets, a->indices,
                                                                (int32_t)lo, (int32_t)hi, cnt);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, out_offsets, n + 1, s);
  void* tmp = ar.raw(tb);
  GB_ARENA_CHECK(ctx, ar);
  GB_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, out_offsets, n + 1, s));
  GB_TRY(read_i64(ctx, out_offsets + n, nnz_host));
  if (out_indices)
    colblock_fill<<<grid_for(ctx, n * 32, 256, 16), 256, 0, s>>>(n, a->offsets, a->indices,
                                                                 (int32_t)lo, (int32_t)hi,
                                                                 out_offsets, out_indices);
  GB_LAUNCH_CHECK(ctx);
  count_launch(ctx, 4);
  return GB_OK;
}

}  // extern "C"
