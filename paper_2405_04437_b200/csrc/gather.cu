// Fused head all-gather over NVLink peer memory (north_star: "NCCL over NVLink is
// used only for the final head all-gather when the caller requests full outputs").
//
// Each rank (one process per GPU) owns one device buffer: two staging areas of its full decode
// output [max_batch, Hq_total, D] bf16, a rank-local front area, and a small signal area.  Ranks
// exchange CUDA IPC handles once (the host side does it over torch.distributed) and map every
// peer's buffer.  The decode kernel (kernels.cu, GatherSink) writes each output row of its head
// shard directly into every rank's staging area of the launch's parity as it is produced, and
// raises its flag in every peer's signal area when its grid is done; `vattn_gather_wait` then
// spins (bounded) until all ranks' flags reached this launch's epoch and copies the staging area
// into the caller's output (or the front area) on the caller's stream.
//
// Why two staging areas (write-after-read across ranks): rank A's launch e+1 may start as soon as
// A's wait for e saw every rank's rows of e.  A peer B may still be reading its launch-e output
// then (a slow consumer), so e+1 must not write where e's rows are: it writes the other parity.
// A's launch e+2, which does reuse e's area, starts only after A's wait for e+1 saw B's rows of
// e+1, and B issued its launch e+1 after its wait for e, which had finished copying e's area
// out (same stream).  The consumer never reads a staging area directly, so its own reads are
// ordered by its stream alone, exactly as with the NCCL all_gather this replaces.
//
// A "local" group places all `world` buffers on one device inside one process; it runs the
// identical kernels and protocol (peer pointers are simply local) and is how the single-GPU
// tests exercise the multi-rank path.

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "internal.h"
#include "vattn.h"

struct vattn_gather {
  int device = 0, rank = 0, world = 1;
  bool local_group = false;
  int64_t out_bytes = 0;       // bytes of one full output region [max_batch, Hq_total, D]
  int64_t stage_bytes = 0;     // staging area 1 offset (= area stride, 256-aligned)
  int64_t front_off = 0;       // rank-local front area (default destination of the wait copy)
  int64_t sig_off = 0;         // signal area offset inside every buffer
  void* base = nullptr;        // own buffer (owned)
  void* peer[vattn::kMaxGatherRanks] = {};
  bool opened[vattn::kMaxGatherRanks] = {};   // peer[r] came from cudaIpcOpenMemHandle
};

namespace vattn {
namespace {

constexpr int64_t kSigBytes = 512;   // flags[8] @0, counter @256, epoch @320, error @384
constexpr uint64_t kWaitTimeoutNs = 10ull * 1000 * 1000 * 1000;

uint32_t* flags_of(void* buf, int64_t sig_off) {
  return reinterpret_cast<uint32_t*>(static_cast<char*>(buf) + sig_off);
}
uint32_t* counter_of(void* buf, int64_t sig_off) {
  return reinterpret_cast<uint32_t*>(static_cast<char*>(buf) + sig_off + 256);
}
uint32_t* epoch_of(void* buf, int64_t sig_off) {
  return reinterpret_cast<uint32_t*>(static_cast<char*>(buf) + sig_off + 320);
}
uint32_t* error_of(void* buf, int64_t sig_off) {
  return reinterpret_cast<uint32_t*>(static_cast<char*>(buf) + sig_off + 384);
}

// Every CTA: one thread per source rank waits until rank r's flag in our signal area reached our
// own launch count (advanced by our last gathered launch, earlier on this stream); then the CTA
// copies its share of staging area (count & 1) to `out` with 16-byte loads and stores.  Bounded:
// after timeout_ns a waiter records a timeout instead of hanging the device (the copy then
// delivers whatever landed; vattn_gather_check reports the ranks).
__global__ void __launch_bounds__(256) gather_wait_kernel(const char* base, int64_t stage_bytes, const uint32_t* flags,
                                                          int world, const uint32_t* epoch_ptr, uint32_t* err,
                                                          uint64_t timeout_ns, uint4* out, int64_t chunks) {
  const int r = threadIdx.x;
  const uint32_t epoch = *epoch_ptr;
  if (r < world) {
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + r) : "memory");
      if ((int32_t)(v - epoch) >= 0) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicOr(err, 1u << r);
        break;
      }
      __nanosleep(200);
    }
  }
  __syncthreads();
  if (!out) return;
  const uint4* src = reinterpret_cast<const uint4*>(base + ((epoch & 1) ? stage_bytes : 0));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < chunks; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v;
    // peers wrote these bytes over NVLink; the acquire above orders them: bypass L1
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
    out[i] = v;
  }
}

void alloc_buffer(vattn_gather* g) {
  g->stage_bytes = (g->out_bytes + 255) / 256 * 256;
  g->front_off = 2 * g->stage_bytes;
  g->sig_off = 3 * g->stage_bytes;
  check_rt(cudaMalloc(&g->base, (size_t)(g->sig_off + kSigBytes)), "cudaMalloc(gather buffer)");
  check_rt(cudaMemset(g->base, 0, (size_t)(g->sig_off + kSigBytes)), "cudaMemset(gather buffer)");
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    check_rt(cudaGetDevice(&prev), "cudaGetDevice");
    if (prev != dev) check_rt(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

GatherSink gather_sink(vattn_gather* g, int hq_local, int batch, int head_dim) {
  if (!g) throw Fail(VATTN_BAD_STATE, "null gather handle");
  for (int r = 0; r < g->world; ++r)
    if (!g->peer[r]) throw Fail(VATTN_BAD_STATE, "gather: peer buffers not opened (call vattn_gather_open)");
  const int64_t need = (int64_t)batch * hq_local * g->world * head_dim * 2;
  if (need > g->out_bytes) throw Fail(VATTN_VALUE_ERROR, "gather: output buffer smaller than batch x Hq_total x D");
  GatherSink s{};
  for (int r = 0; r < g->world; ++r) {
    s.dst[r] = g->peer[r];
    s.flags[r] = flags_of(g->peer[r], g->sig_off);
  }
  s.counter = counter_of(g->base, g->sig_off);
  s.epoch = epoch_of(g->base, g->sig_off);
  s.stage_bytes = g->stage_bytes;
  s.n_ranks = g->world;
  s.rank = g->rank;
  s.hq_total = hq_local * g->world;
  s.head_off = g->rank * hq_local;
  return s;
}

}  // namespace vattn

using vattn::Fail;

template <typename F>
static vattn_status gguard(F&& f) {
  try {
    f();
    return VATTN_OK;
  } catch (const Fail& e) {
    vattn::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    vattn::set_last_error(e.what());
    return VATTN_BAD_STATE;
  }
}

extern "C" {

vattn_status vattn_gather_create(int32_t device, int32_t rank, int32_t world, int64_t out_bytes,
                                 vattn_gather_t** out, void* ipc_handle) {
  return gguard([&] {
    if (!out || !ipc_handle) throw Fail(VATTN_VALUE_ERROR, "null output pointer");
    if (world < 1 || world > vattn::kMaxGatherRanks || rank < 0 || rank >= world)
      throw Fail(VATTN_VALUE_ERROR, "gather: rank/world out of range (world <= 8)");
    if (out_bytes <= 0) throw Fail(VATTN_VALUE_ERROR, "gather: out_bytes must be positive");
    vattn::DeviceGuard dg(device);
    auto g = std::make_unique<vattn_gather>();
    g->device = device;
    g->rank = rank;
    g->world = world;
    g->out_bytes = out_bytes;
    vattn::alloc_buffer(g.get());
    g->peer[rank] = g->base;
    cudaIpcMemHandle_t h;
    vattn::check_rt(cudaIpcGetMemHandle(&h, g->base), "cudaIpcGetMemHandle");
    std::memcpy(ipc_handle, &h, sizeof(h));
    *out = g.release();
  });
}

vattn_status vattn_gather_open(vattn_gather_t* g, const void* handles) {
  return gguard([&] {
    if (!g || !handles) throw Fail(VATTN_VALUE_ERROR, "null argument");
    if (g->local_group) throw Fail(VATTN_BAD_STATE, "gather: a local group is already open");
    vattn::DeviceGuard dg(g->device);
    for (int r = 0; r < g->world; ++r) {
      if (r == g->rank || g->peer[r]) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const char*>(handles) + r * VATTN_IPC_HANDLE_BYTES, sizeof(h));
      void* p = nullptr;
      vattn::check_rt(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      g->peer[r] = p;
      g->opened[r] = true;
    }
  });
}

vattn_status vattn_gather_create_local(int32_t device, int32_t world, int64_t out_bytes,
                                       vattn_gather_t** out) {
  return gguard([&] {
    if (!out) throw Fail(VATTN_VALUE_ERROR, "null output pointer");
    if (world < 1 || world > vattn::kMaxGatherRanks) throw Fail(VATTN_VALUE_ERROR, "gather: world out of range");
    if (out_bytes <= 0) throw Fail(VATTN_VALUE_ERROR, "gather: out_bytes must be positive");
    vattn::DeviceGuard dg(device);
    std::vector<std::unique_ptr<vattn_gather>> gs;
    for (int r = 0; r < world; ++r) {
      auto g = std::make_unique<vattn_gather>();
      g->device = device;
      g->rank = r;
      g->world = world;
      g->out_bytes = out_bytes;
      g->local_group = true;
      vattn::alloc_buffer(g.get());
      gs.push_back(std::move(g));
    }
    for (int r = 0; r < world; ++r)
      for (int p = 0; p < world; ++p) gs[r]->peer[p] = gs[p]->base;
    for (int r = 0; r < world; ++r) out[r] = gs[r].release();
  });
}

vattn_status vattn_gather_output(vattn_gather_t* g, uint64_t* dptr) {
  return gguard([&] {
    if (!g || !dptr) throw Fail(VATTN_VALUE_ERROR, "null argument");
    *dptr = reinterpret_cast<uint64_t>(static_cast<char*>(g->base) + g->front_off);
  });
}

vattn_status vattn_gather_wait(vattn_gather_t* g, void* out, int64_t out_bytes, void* stream) {
  return gguard([&] {
    if (!g) throw Fail(VATTN_VALUE_ERROR, "null gather handle");
    if (out_bytes < 0 || out_bytes > g->out_bytes || out_bytes % 16)
      throw Fail(VATTN_VALUE_ERROR, "gather wait: out_bytes must be a multiple of 16 and at most the buffer size");
    if (out && reinterpret_cast<uintptr_t>(out) % 16) throw Fail(VATTN_VALUE_ERROR, "gather wait: out must be 16-byte aligned");
    if (!out) out = static_cast<char*>(g->base) + g->front_off;
    uint64_t timeout = vattn::kWaitTimeoutNs;
    if (const char* e = getenv("VATTN_GATHER_TIMEOUT_MS")) timeout = (uint64_t)std::max(1L, atol(e)) * 1000000ull;
    const int64_t chunks = out_bytes / 16;
    // ~8 chunks per thread, at most one wave of 148 x 256 threads (one CTA when nothing to copy)
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148, (chunks + 2047) / 2048));
    vattn::gather_wait_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        static_cast<const char*>(g->base), g->stage_bytes, vattn::flags_of(g->base, g->sig_off), g->world,
        vattn::epoch_of(g->base, g->sig_off), vattn::error_of(g->base, g->sig_off), timeout,
        chunks ? static_cast<uint4*>(out) : nullptr, chunks);
    vattn::check_rt(cudaGetLastError(), "gather wait launch");
  });
}

vattn_status vattn_gather_check(vattn_gather_t* g, uint32_t* timed_out_mask) {
  return gguard([&] {
    if (!g || !timed_out_mask) throw Fail(VATTN_VALUE_ERROR, "null argument");
    vattn::DeviceGuard dg(g->device);
    vattn::check_rt(cudaMemcpy(timed_out_mask, vattn::error_of(g->base, g->sig_off), 4, cudaMemcpyDeviceToHost),
                    "gather check");
  });
}

vattn_status vattn_gather_destroy(vattn_gather_t* g) {
  return gguard([&] {
    if (!g) return;
    std::unique_ptr<vattn_gather> own(g);
    vattn::DeviceGuard dg(g->device);
    for (int r = 0; r < g->world; ++r)
      if (g->opened[r]) cudaIpcCloseMemHandle(g->peer[r]);
    if (g->base) cudaFree(g->base);
  });
}

vattn_status vattn_decode_gather_raw(const vattn_cache_desc* c, const void* q, const void* k_new,
                                     const void* v_new, vattn_gather_t* g, int32_t batch, int32_t hq,
                                     const int32_t* cache_seqlens, const int32_t* batch_idx, float scale,
                                     int32_t num_splits, void* ws, int64_t ws_bytes, void* stream) {
  return gguard([&] {
    const vattn::CacheView v = vattn::view_from_desc(c);
    const vattn::GatherSink s = vattn::gather_sink(g, hq, batch, v.d);
    vattn::launch_decode(nullptr, -1, v, q, nullptr, batch, hq, cache_seqlens, batch_idx, scale, num_splits, ws,
                         ws_bytes, (cudaStream_t)stream, k_new, v_new, &s);
  });
}

}  // extern "C"
