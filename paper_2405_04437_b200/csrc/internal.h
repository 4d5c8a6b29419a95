// Internal interfaces shared by the allocator core (core.cpp) and the kernels (kernels.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime_api.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "vattn.h"
#include <nvtx3/nvToolsExt.h>

namespace vattn {

// NVTX range for the allocator and launch paths (SURVEY §5 tracing): visible in Nsight Systems /
// ncu --nvtx; a no-op costing a few ns when no tool is attached.  Header-only NVTX v3.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

// Internal failure carrying a vattn_status; converted to a return code at the C ABI edge.
struct Fail : std::runtime_error {
  vattn_status code;
  Fail(vattn_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

// Driver API resolved at runtime through cudaGetDriverEntryPoint, so libvattn.so has no link
// dependency on libcuda (it loads on a CPU-only host for the shadow backend and ABI tests).
struct Driver {
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*MemAddressFree)(CUdeviceptr, size_t);
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                        unsigned long long);
  CUresult (*MemRelease)(CUmemGenericAllocationHandle);
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle,
                     unsigned long long);
  CUresult (*MemUnmap)(CUdeviceptr, size_t);
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*,
                                          CUmemAllocationGranularity_flags);
  CUresult (*CtxGetCurrent)(CUcontext*);
  CUresult (*CtxSetCurrent)(CUcontext);
  CUresult (*DevicePrimaryCtxRetain)(CUcontext*, CUdevice);
  CUresult (*DeviceGet)(CUdevice*, int);
  CUresult (*GetErrorString)(CUresult, const char**);
  CUresult (*TensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
};

// Loads the entry points on first use; throws Fail(VATTN_CUDA_ERROR) when no driver exists.
const Driver& driver();
void check_cu(CUresult r, const char* what);
void check_rt(cudaError_t e, const char* what);

// Geometry of one layer's K and V caches as the kernels see them: token-major rows of
// Hkv*D bf16 with an arbitrary token stride (per-layer or layer-sliced buffers) and a fixed
// per-slot stride (slot i starts at i * slot_stride; manager.py:137-138).
struct CacheView {
  uint64_t k_base = 0, v_base = 0;
  int64_t slot_stride = 0;
  int64_t token_stride = 0;
  int32_t slot_tokens = 0;
  int32_t n_slots = 0;
  int32_t hkv = 0;
  int32_t d = 0;
  // 1 = rows past a slot's length may sit in an unmapped page-group (a page-group is not a whole
  // number of 64-token decode tiles, e.g. the layer-sliced layout, manager.py:93-96): the decode
  // kernels then load a row's last, partial tile with bounded per-row loads instead of one TMA box
  int32_t tail_guard = 0;
  // read guard (manager caches): rows slot i may be read at, and the host-mapped words
  // [flag, slot, requested, readable] a kernel fills when asked for more (its reads are clamped)
  const int32_t* slot_rows = nullptr;
  uint32_t* err = nullptr;
};

CacheView view_from_desc(const vattn_cache_desc* c);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute
// belongs to the kernel in the current device's context, so a process driving several GPUs
// must set it on each.  Thread-safe (setting it twice is harmless).
template <auto Kern>
void ensure_smem_attr(int bytes) {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  check_rt(cudaGetDevice(&dev), "cudaGetDevice");
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  check_rt(cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "smem attribute");
  done.fetch_or(bit, std::memory_order_acq_rel);
}

// Kernel-side per-handle state (tensor-map cache, split-K workspace); defined in kernels.cu.
struct KernelState;
KernelState* kernel_state_new();
void kernel_state_free(KernelState*);

// Fused head all-gather (gather.cu): the decode epilogue stores every output row
// straight into each rank's [batch, Hq_total, D] staging area of this launch's parity over
// NVLink peer memory (16-byte P2P stores) at head offset rank*Hq_local, then the last CTA to
// finish raises this rank's flag in every peer's signal array.  n_ranks = 0 disables it (plain
// local output).
// Rotary embedding applied by the fused append+decode kernel to q and the new k at the token's
// position (flash_attn_with_kvcache rotary_cos / rotary_sin / rotary_interleaved semantics).
struct Rotary {
  const float* cos = nullptr;   // [positions, rotary_dim / 2] fp32; nullptr = no rotary
  const float* sin = nullptr;
  int32_t dim = 0;              // rotary_dim: even, multiple of 16, <= head_dim
  int32_t interleaved = 0;      // 0: GPT-NeoX halves (i, i + dim/2); 1: GPT-J pairs (2i, 2i + 1)
};

constexpr int kMaxGatherRanks = 8;
struct GatherSink {
  void* dst[kMaxGatherRanks];          // rank r's staging area 0 (peer-mapped; own included)
  uint32_t* flags[kMaxGatherRanks];    // rank r's signal words, indexed by the writing rank
  uint32_t* counter;                   // this rank's CTA-completion counter (reset by the last CTA)
  uint32_t* epoch;                     // this rank's launch count, advanced on the device by the
                                       // last CTA (graph-replay safe: no host-side epoch)
  int64_t stage_bytes;                 // staging area 1 = dst[r] + stage_bytes; launch e writes
                                       // area e & 1 (double buffer: see gather.cu)
  int32_t n_ranks, rank, hq_total, head_off;
};

// gather.cu: sink for a launch through `g` (every rank must issue the same sequence of
// gathered launches; the epoch lives on the device).
GatherSink gather_sink(vattn_gather_t* g, int hq_local, int batch, int head_dim);

// Decode row-order hint for the next launches on this thread (-1 none, 0 keep, 1 longest first).
void set_decode_order_hint(int h);
// PDL hint for the next decode launch on this thread: 1 = its K/V may be streamed before the
// previous kernel on the stream completes (the host knows that kernel wrote no row of the layer).
void set_decode_kv_early(int e);

// Entry points from kernels.cu used by the handle-based C ABI wrappers in core.cpp.
void launch_kv_append(KernelState* ks, int cache_key, const CacheView& v, const void* k_new,
                      const void* v_new, int batch, int n_new, const int32_t* seqlens,
                      const int32_t* batch_idx, cudaStream_t st, const Rotary* rot = nullptr);
void launch_decode(KernelState* ks, int cache_key, const CacheView& v, const void* q, void* out,
                   int batch, int hq, const int32_t* seqlens, const int32_t* batch_idx,
                   float scale, int num_splits, void* ws, int64_t ws_bytes, cudaStream_t st,
                   const void* k_new = nullptr, const void* v_new = nullptr,
                   const GatherSink* sink = nullptr, const Rotary* rot = nullptr);
void launch_prefill_varlen(const CacheView& v, const void* q, void* out, int hq, int n_req,
                           const int32_t* q_start, const int32_t* n_q, const int32_t* slots,
                           const int32_t* kv_len, float scale, bool causal, cudaStream_t st);
// merge split partials (fp32 O / l, log2-domain LSE; layout of decode_combine_kernel) into bf16
// rows of `out` [rows, D] (split-KV prefill)
void launch_split_combine(const float* part_o, const float* part_lse, void* out, int rows, int splits, int hq,
                          int d, cudaStream_t st);
void launch_prefill(KernelState* ks, int cache_key, const CacheView& v, const void* q, void* out,
                    int n_q, int hq, int slot, int kv_len, float scale, bool causal,
                    cudaStream_t st, const Rotary* rot = nullptr);

}  // namespace vattn
