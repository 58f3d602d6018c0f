// Shared device/host helpers for libgraphblast_sm100a.
//
// Semiring arithmetic restates /root/reference/pkg/src/graphalg/algebra.py:
//   * pairwise ops (BinaryOp.pairwise, algebra.py:62-70): Plus saturates at the
//     int64 bounds (algebra.py:24-38), comparison / logical ops yield 0/1 in
//     the domain type;
//   * folds (Monoid.reduce / segment_reduce, algebra.py:98-126) use the plain
//     ufunc: int Plus wraps, logical folds yield 0/1 even for one element.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <limits.h>
#include <math.h>

#include <vector>

#include "../../include/graphblast.h"

#define GB_WARP 32
#define GB_FULL 0xffffffffu

namespace gb {

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
gb_status set_error(gb_ctx* ctx, gb_status st, const char* fmt, ...);

#define GB_CUDA(ctx, call)                                                          \
  do {                                                                              \
    cudaError_t _e = (call);                                                        \
    if (_e != cudaSuccess)                                                          \
      return ::gb::set_error((ctx), GB_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, \
                             #call, cudaGetErrorString(_e));                        \
  } while (0)

#define GB_LAUNCH_CHECK(ctx) GB_CUDA(ctx, cudaGetLastError())

#define GB_TRY(expr)               \
  do {                             \
    gb_status _s = (expr);         \
    if (_s != GB_OK) return _s;    \
  } while (0)

// ---------------------------------------------------------------------------
// operators
// ---------------------------------------------------------------------------
template <class T> struct Lim;
template <> struct Lim<int64_t> {
  __host__ __device__ static constexpr int64_t max() { return LLONG_MAX; }
  __host__ __device__ static constexpr int64_t min() { return LLONG_MIN; }
};
template <> struct Lim<double> {
  __host__ __device__ static double max() { return INFINITY; }
  __host__ __device__ static double min() { return -INFINITY; }
};

__host__ __device__ __forceinline__ int64_t sat_add(int64_t x, int64_t y) {
  // algebra.py:24-38: clamp instead of wrapping
  int64_t r;
  if (y > 0 && x > LLONG_MAX - y) return LLONG_MAX;
  if (y < 0 && x < LLONG_MIN - y) return LLONG_MIN;
  r = (int64_t)((uint64_t)x + (uint64_t)y);
  return r;
}
__host__ __device__ __forceinline__ double sat_add(double x, double y) { return x + y; }

__host__ __device__ __forceinline__ int64_t wrap_add(int64_t x, int64_t y) {
  return (int64_t)((uint64_t)x + (uint64_t)y);
}
__host__ __device__ __forceinline__ double wrap_add(double x, double y) { return x + y; }
__host__ __device__ __forceinline__ int64_t wrap_sub(int64_t x, int64_t y) {
  return (int64_t)((uint64_t)x - (uint64_t)y);
}
__host__ __device__ __forceinline__ double wrap_sub(double x, double y) { return x - y; }
__host__ __device__ __forceinline__ int64_t wrap_mul(int64_t x, int64_t y) {
  return (int64_t)((uint64_t)x * (uint64_t)y);
}
__host__ __device__ __forceinline__ double wrap_mul(double x, double y) { return x * y; }

// pairwise op (BinaryOp.pairwise semantics)
template <class T>
__host__ __device__ __forceinline__ T op_pair(int op, T a, T b) {
  switch (op) {
    case GB_OP_PLUS: return sat_add(a, b);
    case GB_OP_PLUS_WRAP: return wrap_add(a, b);
    case GB_OP_MINUS: return wrap_sub(a, b);
    case GB_OP_TIMES: return wrap_mul(a, b);
    case GB_OP_MIN: return a < b ? a : b;
    case GB_OP_MAX: return a > b ? a : b;
    case GB_OP_LOR: return (T)((a != (T)0) || (b != (T)0));
    case GB_OP_LAND: return (T)((a != (T)0) && (b != (T)0));
    case GB_OP_LESS: return (T)(a < b);
    case GB_OP_NE: return (T)(a != b);
    case GB_OP_SECOND: return b;
    case GB_OP_FIRST: return a;
    default: return a;
  }
}

// fold step (ufunc.reduce semantics): acc = op(acc, x); logical folds are 0/1
template <class T>
__host__ __device__ __forceinline__ T op_fold(int op, T acc, T x) {
  switch (op) {
    case GB_OP_PLUS:
    case GB_OP_PLUS_WRAP: return wrap_add(acc, x);
    case GB_OP_MINUS: return wrap_sub(acc, x);
    case GB_OP_TIMES: return wrap_mul(acc, x);
    case GB_OP_MIN: return acc < x ? acc : x;
    case GB_OP_MAX: return acc > x ? acc : x;
    case GB_OP_LOR: return (T)((acc != (T)0) || (x != (T)0));
    case GB_OP_LAND: return (T)((acc != (T)0) && (x != (T)0));
    case GB_OP_SECOND: return x;
    case GB_OP_FIRST: return acc;
    default: return acc;
  }
}

// folds whose result does not depend on the order of the operands
__host__ __device__ __forceinline__ bool fold_commutes(int op) {
  return op == GB_OP_PLUS || op == GB_OP_PLUS_WRAP || op == GB_OP_TIMES || op == GB_OP_MIN ||
         op == GB_OP_MAX || op == GB_OP_LOR || op == GB_OP_LAND;
}

// value of a one-element fold (reduceat on a length-1 segment)
template <class T>
__host__ __device__ __forceinline__ T op_fold1(int op, T x) {
  if (op == GB_OP_LOR || op == GB_OP_LAND) return (T)(x != (T)0);
  return x;
}

// monoid identity in domain T (algebra.py:88-96)
template <class T>
__host__ __device__ __forceinline__ T op_identity(int op);
template <>
__host__ __device__ __forceinline__ int64_t op_identity<int64_t>(int op) {
  switch (op) {
    case GB_OP_TIMES: case GB_OP_LAND: return 1;
    case GB_OP_MIN: return LLONG_MAX;
    case GB_OP_MAX: return LLONG_MIN;
    default: return 0;
  }
}
template <>
__host__ __device__ __forceinline__ double op_identity<double>(int op) {
  switch (op) {
    case GB_OP_TIMES: case GB_OP_LAND: return 1.0;
    case GB_OP_MIN: return INFINITY;
    case GB_OP_MAX: return -INFINITY;
    default: return 0.0;
  }
}

// Is the add monoid order-independent (exact under any reduction order)?
__host__ __device__ __forceinline__ bool op_idempotent(int op) {
  return op == GB_OP_MIN || op == GB_OP_MAX || op == GB_OP_LOR || op == GB_OP_LAND;
}

// ---------------------------------------------------------------------------
// atomics over the fold ops
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ordered_bits(double x) {
  // monotone map double -> uint64 (total order for non-NaN)
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_ordered_bits(unsigned long long b) {
  b = (b & 0x8000000000000000ull) ? (b & 0x7fffffffffffffffull) : ~b;
  return __longlong_as_double((long long)b);
}

template <class T>
__device__ __forceinline__ void atomic_fold(int op, T* addr, T x);

template <>
__device__ __forceinline__ void atomic_fold<int64_t>(int op, int64_t* addr, int64_t x) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
  switch (op) {
    case GB_OP_PLUS: case GB_OP_PLUS_WRAP: atomicAdd(a, (unsigned long long)x); return;
    case GB_OP_MIN: atomicMin(reinterpret_cast<long long*>(addr), (long long)x); return;
    case GB_OP_MAX: atomicMax(reinterpret_cast<long long*>(addr), (long long)x); return;
    case GB_OP_LOR: if (x != 0) *addr = 1; return;   // idempotent store
    case GB_OP_LAND: if (x == 0) *addr = 0; return;
    default: {
      unsigned long long old = *a, assumed;
      do {
        assumed = old;
        int64_t nv = op_fold<int64_t>(op, (int64_t)assumed, x);
        old = atomicCAS(a, assumed, (unsigned long long)nv);
      } while (old != assumed);
    }
  }
}

template <>
__device__ __forceinline__ void atomic_fold<double>(int op, double* addr, double x) {
  switch (op) {
    case GB_OP_PLUS: case GB_OP_PLUS_WRAP: atomicAdd(addr, x); return;
    case GB_OP_LOR: if (x != 0.0) *addr = 1.0; return;
    case GB_OP_LAND: if (x == 0.0) *addr = 0.0; return;
    default: {
      unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
      unsigned long long old = *a, assumed;
      do {
        assumed = old;
        double nv = op_fold<double>(op, __longlong_as_double((long long)assumed), x);
        if (__double_as_longlong(nv) == (long long)assumed) return;
        old = atomicCAS(a, assumed, (unsigned long long)__double_as_longlong(nv));
      } while (old != assumed);
    }
  }
}

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <class T>
__device__ __forceinline__ T warp_fold(int op, T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(GB_FULL, v, o);
    v = op_fold<T>(op, v, w);
  }
  return v;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(GB_FULL, v, o);
  return v;
}

// Warp-aggregated atomicAdd on a global counter: returns this lane's slot.
__device__ __forceinline__ long long warp_reserve(unsigned long long* counter, int want) {
  unsigned mask = __activemask();
  int lane = lane_id();
  // inclusive prefix of `want` among active lanes
  int pre = want;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(mask, pre, o);
    if (lane >= o && ((mask >> (lane - o)) & 1)) pre += v;
  }
  int leader = 31 - __clz(mask);
  int total = __shfl_sync(mask, pre, leader);
  unsigned long long base = 0;
  if (lane == leader && total) base = atomicAdd(counter, (unsigned long long)total);
  base = __shfl_sync(mask, base, leader);
  return (long long)base + pre - want;
}

// 32 consecutive bytes of a column-index stream in one 256-bit load (sm_100),
// L1-bypassing and marked evict-first in L2 (the matrix is read once per
// pass, the gathered vectors and bitmaps should stay resident).  p must be
// 32-byte aligned.  GB_STREAM_L2 selects the L2 policy (A/B builds).
#ifndef GB_STREAM_L2
#define GB_STREAM_L2 ".L2::evict_first"
#endif
__device__ __forceinline__ void ld_stream8(const int32_t* p, int32_t (&v)[8]) {
  asm("ld.global.nc.L1::no_allocate" GB_STREAM_L2 ".v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "l"(p));
}

// streaming read-only load that does not allocate in L1 (column-index
// streams).  Not volatile: the data is immutable during the kernel, so the
// compiler may predicate, batch and schedule these loads freely.
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
  int32_t v;
  asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
// L1-cached probe of a word other threads may be setting.  Staleness is
// benign (a stale clear bit only costs a redundant atomic), so the asm is not
// volatile either: it may be predicated and reordered.
__device__ __forceinline__ uint32_t ld_probe(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.ca.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Predicated fire-and-forget OR (one RED instruction, no branch region).
__device__ __forceinline__ void red_or_if(bool pred, uint32_t* addr, uint32_t bits) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p red.global.or.b32 [%0], %1; }"
               :: "l"(addr), "r"(bits), "r"((uint32_t)pred));
}
__device__ __forceinline__ void red_or_shared_if(bool pred, uint32_t* addr, uint32_t bits) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(addr);
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p red.shared.or.b32 [%0], %1; }"
               :: "r"(a), "r"(bits), "r"((uint32_t)pred));
}

// Random gather of a vector the pull kernels index by column.  GB_GATHER_NA=1
// bypasses L1 (the vectors are L2-sized; random 8-byte gathers rarely hit L1)
// -- an A/B knob, off by default.
#ifndef GB_GATHER_NA
#define GB_GATHER_NA 0
#endif
#ifndef GB_GATHER_EL
#define GB_GATHER_EL 0  // 1: gathers carry an L2 evict_last policy (A/B knob)
#endif
template <class T>
__device__ __forceinline__ T ld_gather(const T* p) {
#if GB_GATHER_EL
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  if (sizeof(T) == 8) {
    unsigned long long v;
    asm("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return *reinterpret_cast<T*>(&v);
  } else {
    unsigned v;
    asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return *reinterpret_cast<T*>(&v);
  }
#elif GB_GATHER_NA
  if (sizeof(T) == 8) {
    unsigned long long v;
    asm("ld.global.nc.L1::no_allocate.b64 %0, [%1];" : "=l"(v) : "l"(p));
    return *reinterpret_cast<T*>(&v);
  } else {
    unsigned v;
    asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return *reinterpret_cast<T*>(&v);
  }
#else
  return __ldg(p);
#endif
}

__device__ __forceinline__ bool bit_test(const uint32_t* bm, int64_t i) {
  return (__ldg(bm + (i >> 5)) >> (i & 31)) & 1u;
}

// ---------------------------------------------------------------------------
// host-side scratch arena (grow-only pool owned by the context)
// ---------------------------------------------------------------------------
struct Arena {
  gb_ctx* ctx;
  std::vector<size_t> used;
  bool failed;
  explicit Arena(gb_ctx* c);
  ~Arena();
  void* raw(size_t bytes);
  template <class T> T* alloc(size_t n) { return static_cast<T*>(raw(n * sizeof(T))); }
};

#define GB_ARENA_CHECK(ctx, arena) \
  do { if ((arena).failed) return ::gb::set_error((ctx), GB_ERR_OOM, "scratch allocation failed"); } while (0)

cudaStream_t stream_of(gb_ctx* ctx);
void count_launch(gb_ctx* ctx, int n = 1);
// event-timed region around a driver's main kernel (no-op unless profiling)
enum { PROF_BFS_PUSH = 1, PROF_BFS_PULL = 2, PROF_BFS_FINALIZE = 3, PROF_SSSP = 4, PROF_PR = 5,
       PROF_CC = 6, PROF_TC = 7, PROF_MV = 8,
       PROF_BFS_PUSH_EDGES = 9 /* zero-length marker: arg = edges the next push expands */,
       PROF_BFS_UNPERMUTE = 10 };
int prof_begin(gb_ctx* ctx, int kind, int64_t arg);
void prof_end(gb_ctx* ctx, int slot);
int sm_count(gb_ctx* ctx);
bool prof_enabled(gb_ctx* ctx);
// Per-context cached objects (e.g. instantiated CUDA graphs) that live until
// the context is destroyed: slot i holds a pointer and its destructor.
enum { SLOT_BFS_GRAPH = 0, SLOT_BFS_AUX = 1, SLOT_PR_GRAPH = 2, SLOT_CC_GRAPH = 3,
       SLOT_SSSP_GRAPH = 4, SLOT_BFS_COOP = 5, SLOT_CC_FIRSTMIN = 6, kCtxSlots = 8 };
void** ctx_slot(gb_ctx* ctx, int i, void (*destroy)(void*));
// pinned host scratch for small device->host reads (>= 64 int64 slots)
int64_t* pinned_slots(gb_ctx* ctx);
gb_status read_i64(gb_ctx* ctx, const int64_t* dptr, int64_t* out, int count = 1);

// grid that fills every SM exactly once at the kernel's achievable occupancy
template <class Kernel>
inline int resident_grid(gb_ctx* ctx, Kernel kernel, int block, size_t smem = 0) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  return per_sm * sm_count(ctx);
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// gb_bfs_coop.cu: small-graph BFS in one cooperative kernel (degree-ordered
// layout; levels by original id, raw log [iters, (dir, K, est) x iters])
int64_t bfs_coop_max_n();
gb_status bfs_coop_run(gb_ctx* ctx, const gb_csr* push, const gb_csr* pull,
                       const uint32_t* nonempty, const int32_t* rank, int64_t source,
                       int64_t cap, double ratio, int32_t policy, int64_t* levels,
                       int64_t* log_dev);

// gb_mv.cu: out[0..n) = v; counters[2] -= rows folded across tiles (hasmul bits)
template <class T>
void fill_identity(gb_ctx* ctx, int64_t n, T v, T* out);
void mv_pull_finish_counts(gb_ctx* ctx, int64_t W, const uint32_t* hasmul,
                           unsigned long long* counters);

// A scalar kernel argument that is either a value known at launch or a device
// location read when the kernel starts (graph-driven loops).
struct DevI64 {
  int64_t v;
  const int64_t* p;
  __device__ __forceinline__ int64_t get() const { return p ? *p : v; }
};
inline DevI64 dval(int64_t v) { return DevI64{v, nullptr}; }
inline DevI64 dptr(const int64_t* p) { return DevI64{0, p}; }
// Same for an output array pointer.
template <class T>
struct DevP {
  T* v;
  T* const* p;
  __device__ __forceinline__ T* get() const { return p ? *p : v; }
};
using DevP64 = DevP<int64_t>;
template <class T>
inline DevP<T> pval(T* v) { return DevP<T>{v, nullptr}; }
template <class T>
inline DevP<T> pptr(T* const* p) { return DevP<T>{nullptr, p}; }

// grid for a grid-stride kernel over n items
inline int grid_for(gb_ctx* ctx, int64_t n, int block, int per_sm = 8) {
  int64_t want = ceil_div(n > 0 ? n : 1, block);
  int64_t cap = (int64_t)sm_count(ctx) * per_sm;
  return (int)(want < cap ? want : cap);
}

}  // namespace gb
