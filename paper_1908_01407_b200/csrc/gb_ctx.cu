// Context: device binding, stream, grow-only scratch pool, pinned scalars,
// error text.  One context per device per host thread (not thread-safe),
// the equivalent of the paper's descriptor-attached memory pool
// without per-call cudaMalloc once warm.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <vector>

#include "gb_common.cuh"

struct gb_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t handoff = nullptr;  // orders a new stream after the previous one
  // scratch pool: blocks reused across calls; arena marks index into `blocks`
  struct Block {
    void* ptr;
    size_t size;
    size_t used;
  };
  std::vector<Block> blocks;
  int64_t* pinned = nullptr;   // 64 pinned int64 slots for scalar readback
  int* dev_err = nullptr;      // device-side error flag (index out of range)
  char msg[512] = {0};
  int64_t launches = 0;        // kernels launched by this context (all entry points)
  // optional per-kernel event timing of the fused drivers' main kernels
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> prof_kind;
  std::vector<int64_t> prof_arg;
  size_t prof_used = 0;
  void* slot[gb::kCtxSlots] = {nullptr};
  void (*slot_free[gb::kCtxSlots])(void*) = {nullptr};
};

namespace gb {

gb_status set_error(gb_ctx* ctx, gb_status st, const char* fmt, ...) {
  if (ctx) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(ctx->msg, sizeof(ctx->msg), fmt, ap);
    va_end(ap);
  }
  return st;
}

cudaStream_t stream_of(gb_ctx* ctx) { return ctx->stream; }

void count_launch(gb_ctx* ctx, int n) { ctx->launches += n; }

int prof_begin(gb_ctx* ctx, int kind, int64_t arg) {
  if (!ctx->prof) return -1;
  size_t need = 2 * (ctx->prof_used + 1);
  while (ctx->ev_pool.size() < need) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->ev_pool.push_back(e);
  }
  int slot = (int)ctx->prof_used++;
  ctx->prof_kind.resize(ctx->prof_used);
  ctx->prof_arg.resize(ctx->prof_used);
  ctx->prof_kind[slot] = kind;
  ctx->prof_arg[slot] = arg;
  cudaEventRecord(ctx->ev_pool[2 * slot], ctx->stream);
  return slot;
}

void prof_end(gb_ctx* ctx, int slot) {
  if (slot < 0) return;
  cudaEventRecord(ctx->ev_pool[2 * slot + 1], ctx->stream);
}
int sm_count(gb_ctx* ctx) { return ctx->sms; }
bool prof_enabled(gb_ctx* ctx) { return ctx->prof; }
void** ctx_slot(gb_ctx* ctx, int i, void (*destroy)(void*)) {
  if (destroy) ctx->slot_free[i] = destroy;
  return &ctx->slot[i];
}
int64_t* pinned_slots(gb_ctx* ctx) { return ctx->pinned; }

gb_status read_i64(gb_ctx* ctx, const int64_t* dptr, int64_t* out, int count) {
  GB_CUDA(ctx, cudaMemcpyAsync(ctx->pinned, dptr, sizeof(int64_t) * count,
                               cudaMemcpyDeviceToHost, ctx->stream));
  GB_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  memcpy(out, ctx->pinned, sizeof(int64_t) * count);
  return GB_OK;
}

// Arena: bump allocation across the context's blocks.  The constructor
// snapshots every block's usage and the destructor restores it, so scratch is
// reused by the next call.  All work is ordered on the context stream, which
// makes that reuse safe without synchronizing.
static const size_t kAlign = 256;

Arena::Arena(gb_ctx* c) : ctx(c), failed(false) {
  for (auto& b : ctx->blocks) used.push_back(b.used);
}

Arena::~Arena() {
  for (size_t i = 0; i < ctx->blocks.size(); ++i)
    ctx->blocks[i].used = i < used.size() ? used[i] : 0;
}

void* Arena::raw(size_t bytes) {
  bytes = (bytes + kAlign - 1) / kAlign * kAlign;
  if (bytes == 0) bytes = kAlign;
  for (auto& b : ctx->blocks) {
    if (b.size - b.used >= bytes) {
      void* p = (char*)b.ptr + b.used;
      b.used += bytes;
      return p;
    }
  }
  size_t want = bytes < ((size_t)64 << 20) ? ((size_t)64 << 20) : bytes;
  void* p = nullptr;
  if (cudaMalloc(&p, want) != cudaSuccess) {
    cudaGetLastError();
    failed = true;
    return nullptr;
  }
  ctx->blocks.push_back({p, want, bytes});
  return p;
}

}  // namespace gb

using namespace gb;

extern "C" {

int32_t gb_abi_version(void) { return 2; }

gb_status gb_ctx_create(int device, gb_ctx** out) {
  if (!out) return GB_ERR_ARG;
  gb_ctx* ctx = new gb_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete ctx;
    return GB_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMallocHost(&ctx->pinned, 64 * sizeof(int64_t)) != cudaSuccess ||
      cudaMalloc(&ctx->dev_err, sizeof(int)) != cudaSuccess) {
    delete ctx;
    return GB_ERR_CUDA;
  }
  cudaMemset(ctx->dev_err, 0, sizeof(int));
  cudaDeviceSynchronize();
  *out = ctx;
  return GB_OK;
}

gb_status gb_ctx_destroy(gb_ctx* ctx) {
  if (!ctx) return GB_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (int i = 0; i < gb::kCtxSlots; ++i)
    if (ctx->slot[i] && ctx->slot_free[i]) ctx->slot_free[i](ctx->slot[i]);
  for (auto& b : ctx->blocks) cudaFree(b.ptr);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->dev_err) cudaFree(ctx->dev_err);
  if (ctx->handoff) cudaEventDestroy(ctx->handoff);
  delete ctx;
  return GB_OK;
}

// Everything the context owns (scratch arena, cached BFS graph state, the
// pinned log slots) is ordered by its stream.  A switch to another stream
// therefore makes the new stream wait for all work already enqueued on the old
// one, so two calls issued under different torch streams never overlap on the
// shared state.
gb_status gb_ctx_set_stream(gb_ctx* ctx, void* s) {
  if (!ctx) return GB_ERR_ARG;
  cudaStream_t ns = (cudaStream_t)s;
  if (ns == ctx->stream) return GB_OK;
  if (!ctx->handoff) GB_CUDA(ctx, cudaEventCreateWithFlags(&ctx->handoff, cudaEventDisableTiming));
  GB_CUDA(ctx, cudaEventRecord(ctx->handoff, ctx->stream));
  GB_CUDA(ctx, cudaStreamWaitEvent(ns, ctx->handoff, 0));
  ctx->stream = ns;
  return GB_OK;
}

gb_status gb_ctx_sync(gb_ctx* ctx) {
  GB_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GB_OK;
}

const char* gb_last_error(gb_ctx* ctx) { return ctx ? ctx->msg : "no context"; }

int64_t gb_launch_count(gb_ctx* ctx) { return ctx ? ctx->launches : 0; }

gb_status gb_ctx_set_profiling(gb_ctx* ctx, int32_t on) {
  ctx->prof = on != 0;
  ctx->prof_used = 0;
  return GB_OK;
}

int32_t gb_prof_read(gb_ctx* ctx, int32_t max, int32_t* kind, int64_t* arg, float* ms) {
  cudaStreamSynchronize(ctx->stream);
  int32_t n = (int32_t)ctx->prof_used;
  if (n > max) n = max;
  for (int32_t i = 0; i < n; ++i) {
    kind[i] = ctx->prof_kind[i];
    arg[i] = ctx->prof_arg[i];
    float t = 0.f;
    cudaEventElapsedTime(&t, ctx->ev_pool[2 * i], ctx->ev_pool[2 * i + 1]);
    ms[i] = t;
  }
  ctx->prof_used = 0;
  return n;
}

gb_status gb_ctx_trim(gb_ctx* ctx) {
  cudaStreamSynchronize(ctx->stream);
  for (auto& b : ctx->blocks) cudaFree(b.ptr);
  ctx->blocks.clear();
  return GB_OK;
}

int64_t gb_scratch_bytes(gb_ctx* ctx) {
  int64_t s = 0;
  for (auto& b : ctx->blocks) s += (int64_t)b.size;
  return s;
}

}  // extern "C"

// Events recorded on a context's stream (the asynchronous bfs's completion
// marks): no per-record object on the Python side.
extern "C" gb_status gb_event_create(void** ev) {
  cudaEvent_t e;
  if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return GB_ERR_CUDA;
  *ev = (void*)e;
  return GB_OK;
}
extern "C" gb_status gb_event_record(gb_ctx* ctx, void* ev) {
  GB_CUDA(ctx, cudaEventRecord((cudaEvent_t)ev, ctx->stream));
  return GB_OK;
}
extern "C" gb_status gb_event_sync(void* ev) {
  return cudaEventSynchronize((cudaEvent_t)ev) == cudaSuccess ? GB_OK : GB_ERR_CUDA;
}
extern "C" gb_status gb_event_destroy(void* ev) {
  cudaEventDestroy((cudaEvent_t)ev);
  return GB_OK;
}
