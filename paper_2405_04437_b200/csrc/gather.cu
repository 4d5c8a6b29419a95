// Fused head all-gather over NVLink peer memory (north_star: "NCCL over NVLink is
// used only for the final head all-gather when the caller requests full outputs").
//
// Each rank (one process per GPU) owns one device buffer: its full decode output
// [max_batch, Hq_total, D] bf16 followed by a small signal area.  Ranks exchange CUDA IPC
// handles once (the host side does it over torch.distributed) and map every peer's buffer.
// The decode kernel (kernels.cu, GatherSink) then writes each output row of its head shard
// directly into every rank's buffer as it is produced and raises its flag in every peer's
// signal area when its grid is done; `vattn_gather_wait` launches one tiny kernel that spins
// (bounded) until all ranks' flags reached this launch's epoch.  There is no separate copy
// step: the transfer overlaps the attention of the CTAs still running.
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
  int64_t out_bytes = 0;       // bytes of the full output region
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

// One thread per source rank: wait until rank r's flag in our signal area reached our own
// launch count (advanced by our last gathered launch, earlier on this stream).  Bounded: after
// timeout_ns it records a timeout instead of hanging the device.
__global__ void gather_wait_kernel(const uint32_t* flags, int world, const uint32_t* epoch_ptr, uint32_t* err,
                                   uint64_t timeout_ns) {
  const int r = threadIdx.x;
  if (r >= world) return;
  const uint32_t epoch = *epoch_ptr;
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

void alloc_buffer(vattn_gather* g) {
  g->sig_off = (g->out_bytes + 255) / 256 * 256;
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
    *dptr = reinterpret_cast<uint64_t>(g->base);
  });
}

vattn_status vattn_gather_wait(vattn_gather_t* g, void* stream) {
  return gguard([&] {
    if (!g) throw Fail(VATTN_VALUE_ERROR, "null gather handle");
    uint64_t timeout = vattn::kWaitTimeoutNs;
    if (const char* e = getenv("VATTN_GATHER_TIMEOUT_MS")) timeout = (uint64_t)std::max(1L, atol(e)) * 1000000ull;
    vattn::gather_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(
        vattn::flags_of(g->base, g->sig_off), g->world, vattn::epoch_of(g->base, g->sig_off),
        vattn::error_of(g->base, g->sig_off), timeout);
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
