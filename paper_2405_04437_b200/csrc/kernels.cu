// sm_100a kernels of the vAttention hot path: KV append, TMA-fed split-K GQA decode attention
// (contiguous virtual cache and paged comparison variant), split combine.  The tcgen05 prefill
// kernel lives in prefill.cu.
//
// Cache layout: per layer a K and a V region, token-major rows of Hkv*D bf16;
// slot i starts at i*slot_stride (manager.py:137-138 `slot_offset`), token p of a slot at
// p*token_stride.  No block table: the kernels address the virtual tensor directly.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <climits>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <tuple>

#include "internal.h"
#include "ptx.cuh"
#include "vattn.h"

namespace vattn {


// ------------------------------------------------------------------------------ KV append
// One 16-byte chunk per thread-iteration; rows are contiguous in both source and destination
// so warps issue fully coalesced 128-bit loads and stores.
struct AppendParams {
  const int32_t* slot_rows;   // read/write guard (CacheView): rows a slot backs; nullptr = slot_cap
  uint32_t* err;
  int32_t n_slots, slot_cap;
  const uint4* k_src;
  const uint4* v_src;
  char* k_dst;
  char* v_dst;
  const int32_t* seqlens;
  const int32_t* batch_idx;
  int64_t slot_stride, token_stride;
  int32_t n_new, chunks_per_row;
  int64_t total_chunks;  // batch * n_new * chunks_per_row
  Rotary rot;            // rotary of k at its position (cos == nullptr: plain copy)
  int32_t d;             // head dim (chunks per head = d / 8)
};

// One chunk of the append: chunk c of row (b, i) -> its slot row (skipped + reported if unbacked).
__device__ __forceinline__ void append_chunk(const AppendParams& p, int64_t c, uint4 kv, uint4 vv);

// U > 1: each thread loads U chunks of K and of V (grid-strided) before storing any, so a thread
// keeps 2U independent 16-byte loads in flight
template <int U>
__global__ void __launch_bounds__(256) kv_append_kernel_u(AppendParams p) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c0 < p.total_chunks; c0 += U * stride) {
    uint4 kv[U], vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t c = c0 + u * stride;
      if (c < p.total_chunks) {
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(kv[u].x), "=r"(kv[u].y), "=r"(kv[u].z), "=r"(kv[u].w)
                     : "l"(p.k_src + c));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(vv[u].x), "=r"(vv[u].y), "=r"(vv[u].z), "=r"(vv[u].w)
                     : "l"(p.v_src + c));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t c = c0 + u * stride;
      if (c < p.total_chunks) append_chunk(p, c, kv[u], vv[u]);
    }
  }
}

__device__ __forceinline__ void append_chunk(const AppendParams& p, int64_t c, uint4 kv, uint4 vv) {
  const int64_t row = c / p.chunks_per_row;
  const int32_t within = (int32_t)(c - row * p.chunks_per_row);
  const int32_t b = (int32_t)(row / p.n_new);
  const int32_t i = (int32_t)(row - (int64_t)b * p.n_new);
  const int32_t slot = p.batch_idx ? __ldg(p.batch_idx + b) : b;
  const int64_t pos = (int64_t)__ldg(p.seqlens + b) + i;
  const bool bad_slot = slot < 0 || slot >= p.n_slots;
  const int lim = bad_slot ? 0 : (p.slot_rows ? min(p.slot_cap, __ldg(p.slot_rows + slot)) : p.slot_cap);
  if (pos < 0 || pos >= lim) {
    if (p.err && within == 0) {
      p.err[1] = (uint32_t)slot;
      p.err[2] = (uint32_t)(pos + 1);
      p.err[3] = (uint32_t)lim;
      __threadfence_system();
      *reinterpret_cast<volatile uint32_t*>(p.err) = 1u;
    }
    return;
  }
  const int64_t dst = (int64_t)slot * p.slot_stride + pos * p.token_stride + (int64_t)within * 16;
  *reinterpret_cast<uint4*>(p.k_dst + dst) = kv;
  *reinterpret_cast<uint4*>(p.v_dst + dst) = vv;
}

__global__ void __launch_bounds__(256) kv_append_kernel(AppendParams p) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < p.total_chunks; c += stride) {
    const int64_t row = c / p.chunks_per_row;
    const int32_t within = (int32_t)(c - row * p.chunks_per_row);
    const int32_t b = (int32_t)(row / p.n_new);
    const int32_t i = (int32_t)(row - (int64_t)b * p.n_new);
    const int32_t slot = p.batch_idx ? __ldg(p.batch_idx + b) : b;
    const int64_t pos = (int64_t)__ldg(p.seqlens + b) + i;
    const bool bad_slot = slot < 0 || slot >= p.n_slots;
    const int lim = bad_slot ? 0 : (p.slot_rows ? min(p.slot_cap, __ldg(p.slot_rows + slot)) : p.slot_cap);
    if (pos < 0 || pos >= lim) {   // not backed: skip the row, report once per row
      if (p.err && within == 0) {
        p.err[1] = (uint32_t)slot;
        p.err[2] = (uint32_t)(pos + 1);
        p.err[3] = (uint32_t)lim;
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(p.err) = 1u;
      }
      continue;
    }
    const int64_t dst = (int64_t)slot * p.slot_stride + pos * p.token_stride + (int64_t)within * 16;
    uint4 kv, vv;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(kv.x), "=r"(kv.y), "=r"(kv.z), "=r"(kv.w)
                 : "l"(p.k_src + c));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(vv.x), "=r"(vv.y), "=r"(vv.z), "=r"(vv.w)
                 : "l"(p.v_src + c));
    if (p.rot.cos) {
      const int cc = within % (p.d / 8);          // chunk within this head
      if (cc * 8 < p.rot.dim) {
        const int half = p.rot.dim / 16;
        const int pc = p.rot.interleaved ? cc : (cc < half ? cc + half : cc - half);
        const uint4 w = __ldg(p.k_src + c - cc + pc);
        const int64_t t = pos * (p.rot.dim / 2);
        kv = ptx::rotary_chunk(kv, w, cc, p.rot.cos + t, p.rot.sin + t, p.rot.dim, p.rot.interleaved != 0);
      }
    }
    *reinterpret_cast<uint4*>(p.k_dst + dst) = kv;
    *reinterpret_cast<uint4*>(p.v_dst + dst) = vv;
  }
}

// PagedAttention-layout append (comparison path): row (b, i) goes to block
// table[b][pos / block_size], row pos % block_size, pools [num_blocks, block_size, Hkv, D].
struct PagedAppendParams {
  const uint4* k_src;
  const uint4* v_src;
  char* k_pool;
  char* v_pool;
  const int32_t* seqlens;
  const int32_t* block_table;
  int32_t max_blocks, block_size, n_new, chunks_per_row;
  int64_t total_chunks, row_bytes;
};

__global__ void __launch_bounds__(256) kv_append_paged_kernel(PagedAppendParams p) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < p.total_chunks; c += stride) {
    const int64_t row = c / p.chunks_per_row;
    const int32_t within = (int32_t)(c - row * p.chunks_per_row);
    const int32_t b = (int32_t)(row / p.n_new);
    const int32_t i = (int32_t)(row - (int64_t)b * p.n_new);
    const int32_t pos = __ldg(p.seqlens + b) + i;
    const int32_t blk = __ldg(p.block_table + (int64_t)b * p.max_blocks + pos / p.block_size);
    const int64_t dst = ((int64_t)blk * p.block_size + pos % p.block_size) * p.row_bytes + (int64_t)within * 16;
    const uint4 kv = __ldg(p.k_src + c), vv = __ldg(p.v_src + c);
    *reinterpret_cast<uint4*>(p.k_pool + dst) = kv;
    *reinterpret_cast<uint4*>(p.v_pool + dst) = vv;
  }
}

// ------------------------------------------------------------------------------ decode
constexpr int kTile = 64;        // tokens per pipeline stage
constexpr int kWarpsPerTile = 4;   // a group of 4 consumer warps owns a tile, 16 tokens each
// Consumer warps per CTA (template CW): 4 = one group, 2 CTAs per SM (the common case); 8 = two
// groups taking alternate tiles, for grids of at most one CTA per SM, where a single group per
// SM leaves each sub-partition one warp to hide the ldmatrix/mma/exp2 latencies with.
constexpr int decode_threads(int cw) { return (cw + 1) * 32; }   // + one TMA producer warp

struct DecodeParams {
  const __nv_bfloat16* q;     // [batch, hq, D]
  __nv_bfloat16* out;         // [batch, hq, D]
  float* part_o;              // [batch, hq, splits, D]  (split mode)
  float* part_lse;            // [batch, hq, splits]     log2 domain
  const int32_t* seqlens;
  const int32_t* batch_idx;   // contiguous: cache slot of row b (nullptr = b)
  const int32_t* block_table; // paged: [batch, max_blocks]
  int32_t max_blocks, block_size, box_tokens;
  int32_t hq, group, num_splits;
  float scale_log2;
  // fused append (flash-attn k=/v= semantics): seqlens are the lengths BEFORE the new token,
  // which is written to row seqlens[b] of the slot and attended to (nullptr = plain decode)
  const __nv_bfloat16* k_new;   // [batch, hkv, D]
  const __nv_bfloat16* v_new;
  __nv_bfloat16* k_cache;       // base of the layer's K region (row address computed below)
  __nv_bfloat16* v_cache;
  int64_t slot_stride, token_stride;
  GatherSink sink;              // fused head all-gather (n_ranks = 0: write `out` only)
  int32_t longest_first;        // schedule rows by descending length (B <= 256)
  int32_t tail_guard;           // contiguous: load a row's partial last tile per row (CacheView)
  int32_t kv_early;             // PDL: the producer may stream K/V before the previous kernel on
                                // the stream completed (it wrote no row of this layer's cache)
  // contiguous read guard (CacheView::slot_rows / err): rows are clamped to the slot's readable
  // rows (and to slot_cap); slots outside [0, n_slots) read nothing
  const int32_t* slot_rows;
  uint32_t* err;
  int32_t n_slots, slot_cap;
  Rotary rot;                   // rotary embedding of q and k_new (fused mode only)
  // split-K combine inside the cluster of a unit's splits (launched with cluster dims
  // (num_splits, 1, 1)): partials stay in shared memory and are merged over DSMEM, no
  // workspace round trip and no combine launch
  int32_t cluster_combine;
};

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(ptx::smem_u32(p)), "r"(rank));
  return a;
}


// ---- fused head all-gather epilogue (gather.cu owns the buffers and the wait) ----
// Output row (b, local head h) goes to row (b, head_off + h) of every rank's staging area of
// this launch's parity: one 16-byte P2P store per rank and 8 elements over NVLink, issued as the
// chunk is produced, so the exchange overlaps the other CTAs' attention instead of following it.
// The parity is (own launch count + 1) & 1; the count only moves when the last CTA of this launch
// signals, after every store of it (sink_signal), so all CTAs read the same value.
__device__ __forceinline__ int64_t sink_parity_off(const GatherSink& s) {
  return ((*reinterpret_cast<volatile uint32_t*>(s.epoch) + 1) & 1) ? s.stage_bytes : 0;
}
template <typename V>
__device__ __forceinline__ void sink_store(const GatherSink& s, int64_t par_off, int b, int head, int c, int D,
                                           V v) {
  const int64_t off = par_off + (((int64_t)b * s.hq_total + s.head_off + head) * D + c) * 2;
#pragma unroll 1
  for (int r = 0; r < s.n_ranks; ++r) *reinterpret_cast<V*>(static_cast<char*>(s.dst[r]) + off) = v;
}

// Called by all `nthreads` threads of a CTA (named barrier 1) after their last sink_store.
// Every writer fences at system scope; the CTA that completes the grid raises this rank's flag
// in every peer's signal array (release, system scope) and re-arms the counter for the next
// launch on the stream.
__device__ __forceinline__ void sink_signal(const GatherSink& s, uint32_t total_ctas, int nthreads) {
  __threadfence_system();
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(s.counter, 1u);
    if (prev == total_ctas - 1) {
      __threadfence_system();
      const uint32_t e = *s.epoch + 1;   // launches are stream-ordered: nobody else writes it now
      *s.epoch = e;
      for (int r = 0; r < s.n_ranks; ++r)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(s.flags[r] + s.rank), "r"(e) : "memory");
      atomicExch(s.counter, 0u);
    }
  }
}

template <int D, int STAGES, int CW = 4>
struct DecodeSmem {
  static constexpr int kHalfBytes = kTile * 128;             // 64 tokens x 64 dims x bf16
  static constexpr int kTileBytes = (D / 64) * kHalfBytes;   // one of K or V
  static constexpr int kStageBytes = 2 * kTileBytes;
  static constexpr int kQStride = D + 8;                     // bf16 elements, conflict-free ldmatrix
  static constexpr int kQBytes = 16 * kQStride * 2;
  static constexpr int kRedBytes = CW * 16 * 2 * 4;
  static_assert(CW * 16 * D * 4 <= STAGES * kStageBytes, "merge scratch reuses the pipeline smem");
  static constexpr int kBarOff = STAGES * kStageBytes + kQBytes + kRedBytes;
  static constexpr int kBytes = kBarOff + 2 * STAGES * 8 + 1024;  // + alignment slack
};

template <int D, int STAGES, bool PAGED, int CW = 4>
__global__ void __launch_bounds__(decode_threads(CW), CW == 4 ? 2 : 1) decode_kernel(const __grid_constant__ CUtensorMap kmap,
                                                          const __grid_constant__ CUtensorMap vmap,
                                                          DecodeParams p) {
  using L = DecodeSmem<D, STAGES, CW>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __nv_bfloat16* qs = reinterpret_cast<__nv_bfloat16*>(smem + STAGES * L::kStageBytes);
  float* red = reinterpret_cast<float*>(smem + STAGES * L::kStageBytes + L::kQBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* empty = full + STAGES;

  const int split = blockIdx.x, kvh = blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // Programmatic dependent launch: the next kernel on the stream (this layer's
  // split combine, or the next layer's decode) may launch once every CTA of this grid started, so
  // its K/V streaming fills the SMs this grid's tail leaves idle.  Everything a dependent reads
  // that this grid writes (out / partials / the appended row) is read after its
  // griddepcontrol.wait, which waits for this whole grid.
  asm volatile("griddepcontrol.launch_dependents;");
  // Longest rows first: CTA z takes the row with the z-th largest length (ties by index), so a
  // batch of mixed contexts does not finish on a tail of long rows started last (uniform(128,
  // 8192) contexts, B 64: 5.87 -> 6.5 TB/s, against 6.7 for equal lengths).
  int b = blockIdx.z;
  if (p.longest_first) {
    __shared__ int s_len[256];
    __shared__ int s_row;
    const int B = gridDim.z;
    for (int i = threadIdx.x; i < B; i += blockDim.x) s_len[i] = __ldg(p.seqlens + i);
    __syncthreads();
    for (int i = threadIdx.x; i < B; i += blockDim.x) {
      const int li = s_len[i];
      int rank = 0;
#pragma unroll 8
      for (int k = 0; k < B; ++k) rank += (s_len[k] > li) || (s_len[k] == li && k < i);
      if (rank == (int)blockIdx.z) s_row = i;
    }
    __syncthreads();
    b = s_row;
  }
  const int slot = (!PAGED && p.batch_idx) ? __ldg(p.batch_idx + b) : b;
  bool fused = p.k_new != nullptr;
  int pos_new = fused ? __ldg(p.seqlens + b) : -1;            // row receiving the new token
  int seqlen = fused ? pos_new + 1 : __ldg(p.seqlens + b);
  if constexpr (!PAGED) {
    // Read guard: never touch rows a slot does not back (a bad cache_seqlens / cache_batch_idx
    // would otherwise fault the context).  Clamp, and report through the host-mapped words.
    const bool bad_slot = slot < 0 || slot >= p.n_slots;
    const int lim = bad_slot ? 0 : (p.slot_rows ? min(p.slot_cap, __ldg(p.slot_rows + slot)) : p.slot_cap);
    if (bad_slot || seqlen > lim || seqlen < 0) {
      if (p.err && threadIdx.x == 0 && split == 0 && kvh == 0) {
        p.err[1] = (uint32_t)slot;
        p.err[2] = (uint32_t)seqlen;
        p.err[3] = (uint32_t)lim;
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(p.err) = 1u;
      }
      if (fused && (pos_new >= lim || pos_new < 0)) fused = false;   // no room for the new row
      seqlen = max(0, min(seqlen, lim));
      if (!fused) pos_new = -1;
    }
  }
  const int n_tiles_all = (seqlen + kTile - 1) / kTile;
  const int tps = (n_tiles_all + p.num_splits - 1) / p.num_splits;
  const int tile_begin = split * tps;
  const int n_tiles = max(0, min(n_tiles_all, tile_begin + tps) - tile_begin);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kWarpsPerTile);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp == CW) {
    // ===== TMA producer (lane 0; the whole warp for a guarded tail tile) =====
    if (n_tiles > 0) {
      if (lane == 0) {
        ptx::prefetch_tmap(&kmap);
        ptx::prefetch_tmap(&vmap);
      }
      // K/V rows may have been written by the previous kernel (a fused append of this same
      // layer): stream them early only when the host knows they were not (kv_early)
      if (!p.kv_early) asm volatile("griddepcontrol.wait;" ::: "memory");
      for (int it = 0; it < n_tiles; ++it) {
        const int st = it % STAGES;
        if (it >= STAGES) ptx::mbar_wait(&empty[st], ((it / STAGES) - 1) & 1);
        uint8_t* ks = smem + st * L::kStageBytes;
        uint8_t* vs = ks + L::kTileBytes;
        const int tok0 = (tile_begin + it) * kTile;
        if (!PAGED && p.tail_guard && tok0 + kTile > seqlen) {
          // The row's last tile where rows past its length may be unmapped (a page-group holds
          // a non-multiple of 64 tokens): 16-byte loads of rows [tok0, seqlen) only, stored in
          // the TMA box's 128B-swizzled layout; the consumers mask the rest.  Generic-proxy
          // writes; the arrive (release) after __syncwarp publishes them.
          const int rows = seqlen - tok0;
          const char* kb = reinterpret_cast<const char*>(p.k_cache) + (int64_t)slot * p.slot_stride +
                           (int64_t)kvh * D * 2;
          const char* vb = reinterpret_cast<const char*>(p.v_cache) + (int64_t)slot * p.slot_stride +
                           (int64_t)kvh * D * 2;
          const uint32_t ks_a = ptx::smem_u32(ks), vs_a = ptx::smem_u32(vs);
          for (int i = lane; i < rows * (D / 8); i += 32) {
            const int r = i / (D / 8), c = i % (D / 8);
            const int64_t off = (int64_t)(tok0 + r) * p.token_stride + c * 16;
            const uint4 kv = *reinterpret_cast<const uint4*>(kb + off);
            const uint4 vv = *reinterpret_cast<const uint4*>(vb + off);
            const uint32_t ka = ptx::swz128(ks_a + (c >> 3) * L::kHalfBytes, r, c & 7);
            const uint32_t va = ptx::swz128(vs_a + (c >> 3) * L::kHalfBytes, r, c & 7);
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(ka), "r"(kv.x), "r"(kv.y), "r"(kv.z), "r"(kv.w));
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(va), "r"(vv.x), "r"(vv.y), "r"(vv.z), "r"(vv.w));
          }
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&full[st]);
          continue;
        }
        if (lane != 0) continue;
        ptx::mbar_arrive_expect_tx(&full[st], L::kStageBytes);
        if constexpr (!PAGED) {
#pragma unroll
          for (int h = 0; h < D / 64; ++h) {
            ptx::tma_load_4d(ks + h * L::kHalfBytes, &kmap, &full[st], h * 64, kvh, tok0, slot);
            ptx::tma_load_4d(vs + h * L::kHalfBytes, &vmap, &full[st], h * 64, kvh, tok0, slot);
          }
        } else {
          const int last_blk = (seqlen - 1) / p.block_size;
          for (int sub = 0; sub < kTile / p.box_tokens; ++sub) {
            const int tok = tok0 + sub * p.box_tokens;
            const int bi = min(tok / p.block_size, last_blk);  // rows past seqlen are masked
            const int blk = __ldg(p.block_table + (int64_t)b * p.max_blocks + bi);
            const int within = tok % p.block_size;
#pragma unroll
            for (int h = 0; h < D / 64; ++h) {
              ptx::tma_load_4d(ks + h * L::kHalfBytes + sub * p.box_tokens * 128, &kmap, &full[st],
                               h * 64, kvh, within, blk);
              ptx::tma_load_4d(vs + h * L::kHalfBytes + sub * p.box_tokens * 128, &vmap, &full[st],
                               h * 64, kvh, within, blk);
            }
          }
        }
      }
    }
    if (p.cluster_combine) {   // the consumers' two cluster barriers (partials ready / read)
      cluster_sync_all();
      cluster_sync_all();
    }
    return;
  }

  // ===== consumers: 4 warps x 16 tokens of every tile =====
  // As a programmatic dependent of the previous kernel on the stream, q / k_new / v_new and the
  // output (or split partials / gather staging) belong to it until it completes: wait here.  The
  // producer warp above streams this layer's K/V meanwhile (a no-op for a normal launch).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // Q rows of this GQA group -> smem (rows >= group are zero padding of the m16 tile), rotated
  // at the new token's position when rotary tables are given
  const bool rotary = fused && p.rot.cos != nullptr;
  const int rhalf_chunks = p.rot.dim / 16;
  for (int i = threadIdx.x; i < 16 * (D / 8); i += CW * 32) {
    const int r = i / (D / 8), c = i % (D / 8);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < p.group) {
      const __nv_bfloat16* qrow = p.q + ((int64_t)b * p.hq + kvh * p.group + r) * D;
      v = *reinterpret_cast<const uint4*>(qrow + c * 8);
      if (rotary && c * 8 < p.rot.dim) {
        const int pc = p.rot.interleaved ? c : (c < rhalf_chunks ? c + rhalf_chunks : c - rhalf_chunks);
        const uint4 w = *reinterpret_cast<const uint4*>(qrow + pc * 8);
        const int64_t t = (int64_t)pos_new * (p.rot.dim / 2);
        v = ptx::rotary_chunk(v, w, c, p.rot.cos + t, p.rot.sin + t, p.rot.dim, p.rot.interleaved != 0);
      }
    }
    *reinterpret_cast<uint4*>(qs + r * L::kQStride + c * 8) = v;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(CW * 32));
  uint32_t qa[D / 16][4];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    const int r = ((lane >> 3) & 1) * 8 + (lane & 7);
    const int c = kk * 16 + (lane >> 4) * 8;
    ptx::ldsm_x4(ptx::smem_u32(qs + r * L::kQStride + c), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
  }

  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int g = lane >> 2, t4 = lane & 3;

  const int wr = warp % kWarpsPerTile;   // 16-token row block of the tile this warp owns
  for (int it = warp / kWarpsPerTile; it < n_tiles; it += CW / kWarpsPerTile) {
    const int st = it % STAGES;
    ptx::mbar_wait(&full[st], (it / STAGES) & 1);
    const uint32_t ks = ptx::smem_u32(smem + st * L::kStageBytes);
    const uint32_t vs = ks + L::kTileBytes;
    const int my_tok0 = (tile_begin + it) * kTile + wr * 16;
    const int valid = min(16, seqlen - my_tok0);
    if (fused && pos_new >= my_tok0 && pos_new < my_tok0 + 16) {
      // This warp owns the new token's row: patch it into the landed smem tile (the TMA copy
      // may predate the global write) and persist it to the cache.  Lanes 0-15 carry K,
      // 16-31 V; D/8 16-byte chunks per row.
      const int r = pos_new - (tile_begin + it) * kTile;
      const int64_t src = ((int64_t)b * (p.hq / p.group) + kvh) * D;
      const int64_t dst = (int64_t)slot * p.slot_stride + (int64_t)pos_new * p.token_stride +
                          (int64_t)kvh * D * 2;
      for (int c = lane % 16; c < D / 8; c += 16) {
        const bool is_v = lane >= 16;
        uint4 val = *reinterpret_cast<const uint4*>((is_v ? p.v_new : p.k_new) + src + c * 8);
        if (rotary && !is_v && c * 8 < p.rot.dim) {   // k is cached rotated (flash-attn semantics)
          const int pc = p.rot.interleaved ? c : (c < rhalf_chunks ? c + rhalf_chunks : c - rhalf_chunks);
          const uint4 w = *reinterpret_cast<const uint4*>(p.k_new + src + pc * 8);
          const int64_t t = (int64_t)pos_new * (p.rot.dim / 2);
          val = ptx::rotary_chunk(val, w, c, p.rot.cos + t, p.rot.sin + t, p.rot.dim, p.rot.interleaved != 0);
        }
        const uint32_t a = ptx::swz128((is_v ? vs : ks) + (c >> 3) * L::kHalfBytes, r, c & 7);
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(val.x), "r"(val.y), "r"(val.z),
                     "r"(val.w));
        *reinterpret_cast<uint4*>(reinterpret_cast<char*>(is_v ? p.v_cache : p.k_cache) + dst + c * 16) = val;
      }
      __syncwarp();
      ptx::fence_proxy_async();
    }
    if (valid > 0) {
      float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int row = wr * 16 + ((lane >> 4) << 3) + (lane & 7);
        const int chunk = ((kk & 3) << 1) + ((lane >> 3) & 1);
        uint32_t b0, b1, b2, b3;
        ptx::ldsm_x4(ptx::swz128(ks + (kk >> 2) * L::kHalfBytes, row, chunk), b0, b1, b2, b3);
        ptx::mma_bf16_16816(s[0], qa[kk], b0, b1);
        ptx::mma_bf16_16816(s[1], qa[kk], b2, b3);
      }
      // scale into the log2 domain and mask tokens past seqlen
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int col = j * 8 + 2 * t4 + (e & 1);
          s[j][e] = col < valid ? s[j][e] * p.scale_log2 : -INFINITY;
        }
      float mx0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
      float mx1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      const float c0 = ptx::fast_exp2(m0 - mn0), c1 = ptx::fast_exp2(m1 - mn1);  // m=-inf -> 0
      m0 = mn0;
      m1 = mn1;
      float p_[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        p_[j][0] = ptx::fast_exp2(s[j][0] - mn0);
        p_[j][1] = ptx::fast_exp2(s[j][1] - mn0);
        p_[j][2] = ptx::fast_exp2(s[j][2] - mn1);
        p_[j][3] = ptx::fast_exp2(s[j][3] - mn1);
      }
      l0 = l0 * c0 + (p_[0][0] + p_[0][1] + p_[1][0] + p_[1][1]);
      l1 = l1 * c1 + (p_[0][2] + p_[0][3] + p_[1][2] + p_[1][3]);
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        o[n][0] *= c0; o[n][1] *= c0;
        o[n][2] *= c1; o[n][3] *= c1;
      }
      if (valid < 16) {
        // rows past seqlen may hold stale bytes of a reused physical page: 0 * NaN must not
        // reach the accumulator, so zero them (they are the last rows this CTA reads).
        for (int i = lane; i < (16 - valid) * (D / 8); i += 32) {
          const int r = wr * 16 + valid + i / (D / 8);
          const int c = i % (D / 8);
          const uint32_t a = ptx::swz128(vs + (c >> 3) * L::kHalfBytes, r, c & 7);
          asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(a), "r"(0u));
        }
        __syncwarp();
      }
      uint32_t pa[4];
      pa[0] = ptx::pack_bf16(p_[0][0], p_[0][1]);
      pa[1] = ptx::pack_bf16(p_[0][2], p_[0][3]);
      pa[2] = ptx::pack_bf16(p_[1][0], p_[1][1]);
      pa[3] = ptx::pack_bf16(p_[1][2], p_[1][3]);
#pragma unroll
      for (int nd = 0; nd < D / 16; ++nd) {
        const int row = wr * 16 + (((lane >> 3) & 1) << 3) + (lane & 7);
        const int chunk = ((nd & 3) << 1) + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ptx::ldsm_x4_t(ptx::swz128(vs + (nd >> 2) * L::kHalfBytes, row, chunk), b0, b1, b2, b3);
        ptx::mma_bf16_16816(o[2 * nd], pa, b0, b1);
        ptx::mma_bf16_16816(o[2 * nd + 1], pa, b2, b3);
      }
      if (valid < 16) ptx::fence_proxy_async();
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[st]);
  }

  // ===== merge the 4 warps' (m, l, O) and write =====
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  float* red_m = red;
  float* red_l = red + CW * 16;
  if (t4 == 0) {
    red_m[warp * 16 + g] = m0;
    red_m[warp * 16 + g + 8] = m1;
    red_l[warp * 16 + g] = l0;
    red_l[warp * 16 + g + 8] = l1;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(CW * 32));
  float M0 = -INFINITY, M1 = -INFINITY;
#pragma unroll
  for (int w = 0; w < CW; ++w) {
    M0 = fmaxf(M0, red_m[w * 16 + g]);
    M1 = fmaxf(M1, red_m[w * 16 + g + 8]);
  }
  const float sc0 = (M0 == -INFINITY) ? 0.f : ptx::fast_exp2(m0 - M0);
  const float sc1 = (M1 == -INFINITY) ? 0.f : ptx::fast_exp2(m1 - M1);
  // every stage has been consumed: reuse the pipeline smem as [warp][16][D] fp32 scratch
  float* scratch = reinterpret_cast<float*>(smem);
#pragma unroll
  for (int n = 0; n < D / 8; ++n) {
    const int c = n * 8 + 2 * t4;
    float* r0 = scratch + (warp * 16 + g) * D + c;
    float* r1 = scratch + (warp * 16 + g + 8) * D + c;
    r0[0] = o[n][0] * sc0;
    r0[1] = o[n][1] * sc0;
    r1[0] = o[n][2] * sc1;
    r1[1] = o[n][3] * sc1;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(CW * 32));
  const int64_t par_off = (p.sink.n_ranks && p.num_splits == 1) ? sink_parity_off(p.sink) : 0;
  // cluster combine: this split's normalised partial [group][D] and lse [group] behind the scratch
  static_assert(CW * 16 * D * 4 + 16 * D * 4 + 16 * 4 <= STAGES * L::kStageBytes, "cluster staging fits");
  float* stg_o = scratch + CW * 16 * D;
  float* stg_lse = stg_o + 16 * D;
  // 8 consecutive output elements per thread-iteration: 16-byte stores (local or P2P)
  for (int i = threadIdx.x; i < p.group * (D / 8); i += CW * 32) {
    const int r = i / (D / 8), c = (i % (D / 8)) * 8;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < CW; ++w) M = fmaxf(M, red_m[w * 16 + r]);
    float lsum = 0.f, acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int w = 0; w < CW; ++w) {
      const float mw = red_m[w * 16 + r];
      const float f = (M == -INFINITY) ? 0.f : ptx::fast_exp2(mw - M);
      lsum += red_l[w * 16 + r] * f;
      const float4* src = reinterpret_cast<const float4*>(scratch + (w * 16 + r) * D + c);
      const float4 a = src[0], bb = src[1];
      acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
      acc[4] += bb.x; acc[5] += bb.y; acc[6] += bb.z; acc[7] += bb.w;
    }
    const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
    const int head = kvh * p.group + r;
    if (p.num_splits == 1) {
      uint4 pk;
      pk.x = ptx::pack_bf16(acc[0] * inv, acc[1] * inv);
      pk.y = ptx::pack_bf16(acc[2] * inv, acc[3] * inv);
      pk.z = ptx::pack_bf16(acc[4] * inv, acc[5] * inv);
      pk.w = ptx::pack_bf16(acc[6] * inv, acc[7] * inv);
      if (p.sink.n_ranks) sink_store(p.sink, par_off, b, head, c, D, pk);
      else *reinterpret_cast<uint4*>(p.out + ((int64_t)b * p.hq + head) * D + c) = pk;
    } else if (p.cluster_combine) {
      float4* dst = reinterpret_cast<float4*>(stg_o + r * D + c);
      dst[0] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
      dst[1] = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
      if (c == 0) stg_lse[r] = lsum > 0.f ? M + log2f(lsum) : -INFINITY;
    } else {
      const int64_t row = ((int64_t)b * p.hq + head) * p.num_splits + split;
      float4* dst = reinterpret_cast<float4*>(p.part_o + row * D + c);
      dst[0] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
      dst[1] = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
      if (c == 0) p.part_lse[row] = lsum > 0.f ? M + log2f(lsum) : -INFINITY;
    }
  }
  if (p.cluster_combine) {
    // Every split of this (row, KV head) is a CTA of this cluster; CTA `split` merges chunks
    // split, split + S, ... of the group's output over DSMEM, with the same arithmetic as
    // decode_combine_kernel (one batch of <= 16 splits against their max, in split order).
    cluster_sync_all();
    const int S = p.num_splits;
    for (int i = split * (CW * 32) + threadIdx.x; i < p.group * (D / 8); i += S * CW * 32) {
      const int r = i / (D / 8), c = (i % (D / 8)) * 8;
      float l[8];
      float M = -INFINITY;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        l[q] = -INFINITY;
        if (q < S) asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(l[q]) : "r"(dsmem_addr(stg_lse + r, q)));
        M = fmaxf(M, l[q]);
      }
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, wsum = 0.f;
      if (M != -INFINITY) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q >= S) break;
          const float w = exp2f(l[q] - M);
          if (w == 0.f) continue;   // an empty split holds no partial
          float4 a, bb;
          const uint32_t ra = dsmem_addr(stg_o + r * D + c, q);
          asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "r"(ra));
          asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(bb.x), "=f"(bb.y), "=f"(bb.z), "=f"(bb.w) : "r"(ra + 16));
          acc[0] += w * a.x; acc[1] += w * a.y; acc[2] += w * a.z; acc[3] += w * a.w;
          acc[4] += w * bb.x; acc[5] += w * bb.y; acc[6] += w * bb.z; acc[7] += w * bb.w;
          wsum += w;
        }
      }
      const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
      uint4 pk;
      pk.x = ptx::pack_bf16(acc[0] * inv, acc[1] * inv);
      pk.y = ptx::pack_bf16(acc[2] * inv, acc[3] * inv);
      pk.z = ptx::pack_bf16(acc[4] * inv, acc[5] * inv);
      pk.w = ptx::pack_bf16(acc[6] * inv, acc[7] * inv);
      *reinterpret_cast<uint4*>(p.out + ((int64_t)b * p.hq + kvh * p.group + r) * D + c) = pk;
    }
    cluster_sync_all();        // no CTA leaves while another still reads its partial
  }
  if (p.sink.n_ranks && p.num_splits == 1)
    sink_signal(p.sink, gridDim.x * gridDim.y * gridDim.z, CW * 32);
}

// merge split partials with log-sum-exp weights (log2 domain); with a gather sink the merged
// rows go straight to every rank's full output (rows = batch * hq_local)
template <int D>
__global__ void __launch_bounds__(128) decode_combine_kernel(const float* __restrict__ part_o,
                                                             const float* __restrict__ part_lse,
                                                             __nv_bfloat16* __restrict__ out,
                                                             int rows, int num_splits, int hq,
                                                             GatherSink sink) {
  const int row = blockIdx.x * (blockDim.x / (D / 4)) + threadIdx.x / (D / 4);
  const int c4 = threadIdx.x % (D / 4);
  // launched as a programmatic dependent of the decode grid: wait until its partials are visible
  // (a no-op for a normal launch); the next layer's decode may launch behind this grid
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (row < rows) {
    // One batch of up to 16 splits per round trip: every lse and partial of the batch is
    // loaded before any is used, so the L2/DRAM latencies overlap (a plain loop waits ~600
    // cycles per split).  Batches after the first rescale to a running max; with <= 16 splits
    // this is exactly the two-pass merge against the global max.
    constexpr int kB = 16;
    const float* lse = part_lse + (int64_t)row * num_splits;
    const float* po = part_o + (int64_t)row * num_splits * D + c4 * 4;
    float M = -INFINITY;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float wsum = 0.f;
    for (int s0 = 0; s0 < num_splits; s0 += kB) {
      float l[kB];
      float4 v[kB];
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        l[i] = -INFINITY;
        if (s0 + i < num_splits) {
          l[i] = lse[s0 + i];
          v[i] = *reinterpret_cast<const float4*>(po + (int64_t)(s0 + i) * D);
        }
      }
      float mb = M;
#pragma unroll
      for (int i = 0; i < kB; ++i) mb = fmaxf(mb, l[i]);
      if (mb == -INFINITY) continue;
      if (mb != M && M != -INFINITY) {
        const float f = exp2f(M - mb);
        acc.x *= f; acc.y *= f; acc.z *= f; acc.w *= f;
        wsum *= f;
      }
      M = mb;
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const float w = exp2f(l[i] - M);
        if (w != 0.f) {   // an empty split (lse -inf) may hold stale partials: never read into acc
          acc.x += w * v[i].x; acc.y += w * v[i].y; acc.z += w * v[i].z; acc.w += w * v[i].w;
          wsum += w;
        }
      }
    }
    const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
    __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    if (sink.n_ranks == 0) {
      *reinterpret_cast<uint2*>(out + (int64_t)row * D + c4 * 4) = pk;
    } else {
      sink_store(sink, sink_parity_off(sink), row / hq, row % hq, c4 * 4, D, pk);
    }
  }
  if (sink.n_ranks) sink_signal(sink, gridDim.x, blockDim.x);
}

// ------------------------------------------------------------------------------ compute proxy
// Stands in for the non-attention part of a model iteration (GEMMs) in the serving benchmark:
// holds the stream for `ns` nanoseconds of device time (globaltimer), calibrated by the caller
// to the reference's IterationModel (simulator.py:45-62).  One warp; does not touch memory.
__global__ void compute_proxy_kernel(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

// ------------------------------------------------------------------------------ host side
struct KernelState {
  std::mutex mu;
  std::map<std::tuple<uint64_t, int64_t, int64_t, int, int, int, int, int>, CUtensorMap> maps;
};
KernelState* kernel_state_new() { return new KernelState(); }
void kernel_state_free(KernelState* s) { delete s; }

thread_local int g_order_hint = -1;
void set_decode_order_hint(int h) { g_order_hint = h; }
thread_local int g_kv_early = 0;
void set_decode_kv_early(int e) { g_kv_early = e; }

static int g_num_sms = 0;
static int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      cudaGetLastError();
      return 148;       // no device (CPU host: only the labelling query gets here): B200's count
    }
    g_num_sms = n;
  }
  return g_num_sms;
}

// 4-D bf16 map over (D, Hkv, tokens, slots|blocks), 128B swizzle, box (64, 1, box_tokens, 1).
static CUtensorMap make_kv_map(uint64_t base, int d, int hkv, int64_t token_stride, int tokens,
                               int64_t outer_stride, int outer, int box_tokens) {
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)hkv, (cuuint64_t)tokens, (cuuint64_t)outer};
  cuuint64_t strides[3] = {(cuuint64_t)d * 2, (cuuint64_t)token_stride, (cuuint64_t)outer_stride};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)box_tokens, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  check_cu(driver().TensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                                         reinterpret_cast<void*>(base), dims, strides, box, estr,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
           "cuTensorMapEncodeTiled");
  return m;
}

static CUtensorMap cached_map(KernelState* ks, uint64_t base, int d, int hkv, int64_t token_stride,
                              int tokens, int64_t outer_stride, int outer, int box_tokens) {
  if (!ks) return make_kv_map(base, d, hkv, token_stride, tokens, outer_stride, outer, box_tokens);
  auto key = std::make_tuple(base, token_stride, outer_stride, tokens, outer, hkv, d, box_tokens);
  std::lock_guard<std::mutex> lk(ks->mu);
  auto it = ks->maps.find(key);
  if (it != ks->maps.end()) return it->second;
  CUtensorMap m = make_kv_map(base, d, hkv, token_stride, tokens, outer_stride, outer, box_tokens);
  ks->maps.emplace(key, m);
  return m;
}

static void check_view(const CacheView& v) {
  if (v.d != 64 && v.d != 128) throw Fail(VATTN_UNSUPPORTED, "head_dim must be 64 or 128");
  if (v.token_stride % 16 || v.slot_stride % 16 || (v.k_base | v.v_base) % 16)
    throw Fail(VATTN_UNSUPPORTED, "cache rows must be 16-byte aligned");
}

void launch_kv_append(KernelState*, int, const CacheView& v, const void* k_new, const void* v_new,
                      int batch, int n_new, const int32_t* seqlens, const int32_t* batch_idx,
                      cudaStream_t st, const Rotary* rot) {
  check_view(v);
  if (batch <= 0 || n_new <= 0) return;
  const int64_t row_bytes = (int64_t)v.hkv * v.d * 2;
  AppendParams p{};
  p.d = v.d;
  p.slot_rows = v.slot_rows;
  p.err = v.err;
  p.n_slots = v.n_slots;
  p.slot_cap = v.slot_tokens;
  if (rot && rot->cos) {
    if (!rot->sin || rot->dim <= 0 || rot->dim % 16 || rot->dim > v.d)
      throw Fail(VATTN_VALUE_ERROR, "rotary_dim must be a positive multiple of 16 and <= head_dim");
    p.rot = *rot;
  }
  p.k_src = reinterpret_cast<const uint4*>(k_new);
  p.v_src = reinterpret_cast<const uint4*>(v_new);
  p.k_dst = reinterpret_cast<char*>(v.k_base);
  p.v_dst = reinterpret_cast<char*>(v.v_base);
  p.seqlens = seqlens;
  p.batch_idx = batch_idx;
  p.slot_stride = v.slot_stride;
  p.token_stride = v.token_stride;
  p.n_new = n_new;
  p.chunks_per_row = (int32_t)(row_bytes / 16);
  p.total_chunks = (int64_t)batch * n_new * p.chunks_per_row;
  const int threads = 256;
  // Measured (tools/append_ab.py, 4 x 16K Yi-6B rows, 256 MiB moved, L2 flushed): two chunks of
  // K and of V in flight per thread and 16 blocks per SM: 41.0 us = 6.55 TB/s, against 47.1 us
  // for one chunk and 8 blocks per SM.  VATTN_APPEND_UNROLL (1/2/4) / VATTN_APPEND_BPS override.
  static const int unroll = [] {
    const char* e = getenv("VATTN_APPEND_UNROLL");
    return e ? atoi(e) : 2;
  }();
  static const int bps = [] {
    const char* e = getenv("VATTN_APPEND_BPS");
    return e ? std::max(1, atoi(e)) : 16;
  }();
  const int64_t want = (p.total_chunks + threads - 1) / threads;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms() * bps));
  if (!p.rot.cos && unroll == 2) kv_append_kernel_u<2><<<blocks, threads, 0, st>>>(p);
  else if (!p.rot.cos && unroll == 4) kv_append_kernel_u<4><<<blocks, threads, 0, st>>>(p);
  else kv_append_kernel<<<blocks, threads, 0, st>>>(p);
  check_rt(cudaGetLastError(), "kv_append launch");
}

constexpr int kMaxSplits = 64;

static int auto_splits(int units, int max_len) {
  // Measured on B200 (tools/decode_split_sweep.py): one CTA per (batch row, KV head) already
  // streams at full HBM bandwidth once ~128 of them run (deep 4-stage TMA ring per CTA), so
  // split only below that; keep >= 4 tiles (256 tokens) per split.
  const int tiles = std::max(1, (max_len + kTile - 1) / kTile);
  int s = (128 + units - 1) / units;
  // Rounding up past one CTA per SM drops the grid into the 2-CTA / 3-stage variant; when one
  // fewer split still keeps >= 100 CTAs the single-wave deep-ring variant is faster (B 5 x 32K:
  // 3 splits 98.6 vs 4 splits 101.3 us; B 7 x 16K: 2 vs 3, 71.2 vs 72.9; tools/split_fill_probe.py)
  const int sms = num_sms();
  if (s > 1 && units * s > sms && (sms / units) * units >= 100) s = sms / units;
  s = std::min(s, std::max(1, tiles / 4));
  return std::max(1, std::min(s, kMaxSplits));
}

template <int D, int STAGES, bool PAGED, int CW = 4>
static void run_decode(const CUtensorMap& km, const CUtensorMap& vm, DecodeParams p, int batch,
                       int hkv, cudaStream_t st) {
  using L = DecodeSmem<D, STAGES, CW>;
  auto kern = decode_kernel<D, STAGES, PAGED, CW>;
  ensure_smem_attr<decode_kernel<D, STAGES, PAGED, CW>>(L::kBytes);
  static const bool pdl = [] {
    const char* e = getenv("VATTN_DEC_PDL");
    return !e || atoi(e) != 0;
  }();
  // splits of a unit as one cluster, combined over DSMEM (VATTN_DEC_CLUSTER=0 disables)
  static const bool cl_env = [] {
    const char* e = getenv("VATTN_DEC_CLUSTER");
    return !e || atoi(e) != 0;
  }();
  // clusters of up to 8 splits (portable size).  16-CTA non-portable clusters were measured much
  // slower (B 1 x 32K, 16 splits: 49 vs 28 us with the combine kernel): the scheduler has to find
  // 16 free SMs of one GPC for each cluster.
  bool cl = cl_env && p.num_splits >= 2 && p.num_splits <= 8 && p.sink.n_ranks == 0;
  if (cl) {
    // Every unit's splits must be co-resident as one cluster: when the GPU cannot hold all the
    // units' clusters at once, the leftover clusters run as a second wave (B 2 x 64K with 8
    // splits: 125.6 vs 80.3 us; B 3 x 32K with 6 splits: 92.4 vs 62.6 us, tools/split_fill_probe.py).
    // Then the partials go through the combine kernel instead, whose CTAs need no co-scheduling.
    static std::map<int, int> max_clusters;   // per cluster size, for this kernel variant
    static std::mutex mc_mu;
    std::lock_guard<std::mutex> lk(mc_mu);
    auto it = max_clusters.find(p.num_splits);
    if (it == max_clusters.end()) {
      cudaLaunchConfig_t oc{};
      oc.gridDim = dim3(p.num_splits, 1, 1);
      oc.blockDim = dim3(decode_threads(CW));
      oc.dynamicSmemBytes = L::kBytes;
      cudaLaunchAttribute ca{};
      ca.id = cudaLaunchAttributeClusterDimension;
      ca.val.clusterDim.x = p.num_splits;
      ca.val.clusterDim.y = 1;
      ca.val.clusterDim.z = 1;
      oc.attrs = &ca;
      oc.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &oc) != cudaSuccess) {
        (void)cudaGetLastError();
        n = 0;
      }
      it = max_clusters.emplace(p.num_splits, n).first;
    }
    if ((int64_t)batch * hkv > it->second) cl = false;
  }
  p.cluster_combine = cl ? 1 : 0;
  {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.num_splits, hkv, batch);
    cfg.blockDim = dim3(decode_threads(CW));
    cfg.dynamicSmemBytes = L::kBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2]{};
    int na = 0;
    if (pdl) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    if (p.cluster_combine) {
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = p.num_splits;
      attr[na].val.clusterDim.y = 1;
      attr[na].val.clusterDim.z = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    check_rt(cudaLaunchKernelEx(&cfg, kern, km, vm, p), "decode launch");
  }
  check_rt(cudaGetLastError(), "decode launch");
  if (p.num_splits > 1 && !p.cluster_combine) {
    const int rows = batch * p.hq;
    const int per_block = 128 / (D / 4);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((rows + per_block - 1) / per_block);
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = pdl ? 1 : 0;
    check_rt(cudaLaunchKernelEx(&cfg, decode_combine_kernel<D>, (const float*)p.part_o, (const float*)p.part_lse,
                                p.out, rows, p.num_splits, p.hq, p.sink),
             "combine launch");
    check_rt(cudaGetLastError(), "combine launch");
  }
}

// Kernel variant for a D = 128 launch.  Measured (tools/decode_stage_sweep.py): with >= 2 CTAs per
// SM worth of work a 3-stage ring (97 KB smem, 2 CTAs/SM) beats the 4-stage one (L8 layer 6.9 vs
// 6.2 TB/s), so a grid of up to 2 x 148 runs in one wave (L8 at G = 2: 256 CTAs; 6.26 vs 6.12
// TB/s with 4 stages in two waves); with at most one CTA per SM the deeper pipeline wins
// (B 128 x 1 KV head: 6.6 vs 6.3 TB/s) and two consumer groups per CTA keep every sub-partition
// busy.  VATTN_DEC_STAGES / VATTN_DEC_CW=4 override.
struct DecodeChoice {
  int stages, cw;
};
static DecodeChoice choose_decode(int batch, int hkv, int num_splits) {
  static const int forced = [] {
    const char* e = getenv("VATTN_DEC_STAGES");
    return e ? atoi(e) : 0;
  }();
  static const int cw_env = [] {
    const char* e = getenv("VATTN_DEC_CW");
    return e ? atoi(e) : 0;
  }();
  const int64_t ctas = (int64_t)batch * hkv * num_splits;
  const int stages = forced ? forced : (ctas > num_sms() ? 3 : 4);
  const bool wide = stages == 4 && cw_env != 4 && ctas <= num_sms();
  return {stages, wide ? 8 : 4};
}

struct FusedAppend {
  const void* k_new;
  const void* v_new;
  const CacheView* view;
};

static void decode_common(const CUtensorMap& km, const CUtensorMap& vm, int d, int hkv, int hq,
                          const void* q, void* out, int batch, const int32_t* seqlens,
                          const int32_t* batch_idx, const int32_t* block_table, int max_blocks,
                          int block_size, int box_tokens, float scale, int num_splits,
                          int max_len, void* ws, int64_t ws_bytes, bool paged, cudaStream_t st,
                          const FusedAppend* fa = nullptr, const GatherSink* sink = nullptr,
                          const Rotary* rot = nullptr) {
  if (hq % hkv) throw Fail(VATTN_VALUE_ERROR, "n_q_heads must be a multiple of n_kv_heads");
  const int group = hq / hkv;
  if (group > 16) throw Fail(VATTN_UNSUPPORTED, "GQA group larger than 16");
  if (batch <= 0) return;
  if (num_splits <= 0) {
    static const int forced = [] {          // VATTN_DEC_SPLITS: fixed split count (experiments)
      const char* e = getenv("VATTN_DEC_SPLITS");
      return e ? atoi(e) : 0;
    }();
    num_splits = forced > 0 ? forced : auto_splits(batch * hkv, max_len);
  }
  num_splits = std::min(num_splits, kMaxSplits);
  DecodeParams p{};
  p.q = reinterpret_cast<const __nv_bfloat16*>(q);
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.seqlens = seqlens;
  p.batch_idx = batch_idx;
  p.block_table = block_table;
  p.max_blocks = max_blocks;
  p.block_size = block_size;
  p.box_tokens = box_tokens;
  p.hq = hq;
  p.group = group;
  p.num_splits = num_splits;
  // longest-first row order costs ~1 % on equal lengths (rank pass before the first TMA) and
  // gains ~11 % on mixed ones: on when the caller's hint says the lengths differ (the manager
  // knows its slots' contexts), forced by VATTN_DEC_LONGEST_FIRST=0/1
  static const int lf_env = [] {
    const char* e = getenv("VATTN_DEC_LONGEST_FIRST");
    return e ? atoi(e) : -1;
  }();
  const int hint = g_order_hint;
  g_order_hint = -1;                 // a hint applies to the one launch it was set for
  const int lf = lf_env >= 0 ? lf_env : (hint > 0 ? 1 : 0);
  p.longest_first = (lf && batch > 1 && batch <= 256) ? 1 : 0;
  p.kv_early = g_kv_early;
  g_kv_early = 0;                   // like the order hint: applies to the one launch
  if (scale <= 0.f) scale = 1.f / sqrtf((float)d);
  p.scale_log2 = scale * 1.4426950408889634f;
  if (fa) {   // contiguous cache: row addresses for the fused append and the guarded tail tile
    p.k_new = reinterpret_cast<const __nv_bfloat16*>(fa->k_new);   // nullptr: plain decode
    p.v_new = reinterpret_cast<const __nv_bfloat16*>(fa->v_new);
    p.k_cache = reinterpret_cast<__nv_bfloat16*>(fa->view->k_base);
    p.v_cache = reinterpret_cast<__nv_bfloat16*>(fa->view->v_base);
    p.slot_stride = fa->view->slot_stride;
    p.token_stride = fa->view->token_stride;
    p.tail_guard = fa->view->tail_guard;
    p.slot_rows = fa->view->slot_rows;
    p.err = fa->view->err;
    p.n_slots = fa->view->n_slots;
    p.slot_cap = fa->view->slot_tokens;
  }
  if (rot && rot->cos) {
    if (!fa || !fa->k_new) throw Fail(VATTN_VALUE_ERROR, "rotary embedding needs the fused append (k_new / v_new)");
    if (!rot->sin || rot->dim <= 0 || rot->dim % 16 || rot->dim > d)
      throw Fail(VATTN_VALUE_ERROR, "rotary_dim must be a positive multiple of 16 and <= head_dim");
    p.rot = *rot;
  }
  if (sink && sink->n_ranks) {
    if (sink->n_ranks > kMaxGatherRanks || sink->hq_total < hq * sink->n_ranks)
      throw Fail(VATTN_VALUE_ERROR, "gather: bad rank count or head total");
    p.sink = *sink;
  }
  if (num_splits > 1) {
    const int64_t need = vattn_decode_workspace_bytes(batch, hq, d, num_splits);
    if (!ws || ws_bytes < need) throw Fail(VATTN_VALUE_ERROR, "decode workspace too small");
    p.part_o = reinterpret_cast<float*>(ws);
    p.part_lse = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) +
                                          (int64_t)batch * hq * num_splits * d * 4);
  }
  if (d == 128) {
    const DecodeChoice ch = choose_decode(batch, hkv, p.num_splits);
    const int stages = ch.stages;
    const bool wide = ch.cw == 8;
    if (paged) {   // same rule, so the paged comparison differs from the contiguous path only in layout
      if (stages == 3) run_decode<128, 3, true>(km, vm, p, batch, hkv, st);
      else if (wide) run_decode<128, 4, true, 8>(km, vm, p, batch, hkv, st);
      else run_decode<128, 4, true>(km, vm, p, batch, hkv, st);
    } else if (stages == 3) {
      run_decode<128, 3, false>(km, vm, p, batch, hkv, st);
    } else if (wide) {
      run_decode<128, 4, false, 8>(km, vm, p, batch, hkv, st);
    } else {
      run_decode<128, 4, false>(km, vm, p, batch, hkv, st);
    }
  } else {
    if (paged) run_decode<64, 6, true>(km, vm, p, batch, hkv, st);
    else run_decode<64, 6, false>(km, vm, p, batch, hkv, st);
  }
}

void launch_split_combine(const float* part_o, const float* part_lse, void* out, int rows, int splits, int hq,
                          int d, cudaStream_t st) {
  if (rows <= 0) return;
  GatherSink none{};
  if (d == 128) {
    const int per_block = 128 / (128 / 4);
    decode_combine_kernel<128><<<(rows + per_block - 1) / per_block, 128, 0, st>>>(
        part_o, part_lse, reinterpret_cast<__nv_bfloat16*>(out), rows, splits, hq, none);
  } else if (d == 64) {
    const int per_block = 128 / (64 / 4);
    decode_combine_kernel<64><<<(rows + per_block - 1) / per_block, 128, 0, st>>>(
        part_o, part_lse, reinterpret_cast<__nv_bfloat16*>(out), rows, splits, hq, none);
  } else {
    throw Fail(VATTN_UNSUPPORTED, "split combine is built for head_dim 64 and 128");
  }
  check_rt(cudaGetLastError(), "split combine launch");
}

void launch_decode(KernelState* ks, int, const CacheView& v, const void* q, void* out, int batch,
                   int hq, const int32_t* seqlens, const int32_t* batch_idx, float scale,
                   int num_splits, void* ws, int64_t ws_bytes, cudaStream_t st, const void* k_new,
                   const void* v_new, const GatherSink* sink, const Rotary* rot) {
  check_view(v);
  // Token extent = every row inside the slot stride, so a 64-row tile that starts below seqlen
  // never takes TMA's out-of-bounds path (which faults on VMM-backed maps when the box
  // straddles the token bound); those rows sit in the slot's last mapped page and are masked.
  const int64_t rows = v.slot_stride / v.token_stride;
  const int tokens = (int)std::max<int64_t>(v.slot_tokens, std::min<int64_t>(rows, INT32_MAX));
  const CUtensorMap km = cached_map(ks, v.k_base, v.d, v.hkv, v.token_stride, tokens, v.slot_stride, v.n_slots, kTile);
  const CUtensorMap vm = cached_map(ks, v.v_base, v.d, v.hkv, v.token_stride, tokens, v.slot_stride, v.n_slots, kTile);
  FusedAppend fa{k_new, v_new, &v};
  decode_common(km, vm, v.d, v.hkv, hq, q, out, batch, seqlens, batch_idx, nullptr, 0, 0, kTile,
                scale, num_splits, v.slot_tokens, ws, ws_bytes, false, st, &fa, sink, rot);
}

}  // namespace vattn

// ================================================================================ C ABI
using vattn::Fail;

template <typename F>
static vattn_status kguard(F&& f) {
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

vattn_status vattn_compute_proxy(uint64_t ns, void* stream) {
  return kguard([&] {
    vattn::compute_proxy_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(ns);
    vattn::check_rt(cudaGetLastError(), "compute proxy launch");
  });
}

int32_t vattn_decode_num_splits(int32_t batch, int32_t hkv, int32_t max_seqlen) {
  try {
    return vattn::auto_splits(batch * hkv, max_seqlen);
  } catch (...) {
    return 1;
  }
}

int32_t vattn_decode_kernel_name(int32_t batch, int32_t hkv, int32_t max_seqlen, int32_t num_splits,
                                 int32_t head_dim, char* buf, int32_t cap) {
  try {
    if (num_splits <= 0) num_splits = vattn::auto_splits(batch * hkv, max_seqlen);
    num_splits = std::min(num_splits, vattn::kMaxSplits);
    char tmp[96];
    static const bool cl_env = [] {
      const char* e = getenv("VATTN_DEC_CLUSTER");
      return !e || atoi(e) != 0;
    }();
    // 2-8 splits merge inside their cluster (no combine kernel), more go through the combine kernel
    const char* tail = num_splits <= 1 ? ""
                       : (cl_env && num_splits <= 8) ? " (cluster combine)"
                       : (head_dim == 128 ? " + decode_combine_kernel<128>" : " + decode_combine_kernel<64>");
    if (head_dim == 128) {
      const vattn::DecodeChoice ch = vattn::choose_decode(batch, hkv, num_splits);
      snprintf(tmp, sizeof tmp, "decode_kernel<128,%d,false,%d>%s", ch.stages, ch.cw, tail);
    } else {
      snprintf(tmp, sizeof tmp, "decode_kernel<64,6,false,4>%s", tail);
    }
    if (buf && cap > 0) {
      strncpy(buf, tmp, (size_t)cap - 1);
      buf[cap - 1] = 0;
    }
    return num_splits;
  } catch (...) {
    return -1;
  }
}

int64_t vattn_decode_workspace_bytes(int32_t batch, int32_t hq, int32_t d, int32_t num_splits) {
  const int64_t s = num_splits > 0 ? num_splits : vattn::kMaxSplits;
  return (int64_t)batch * hq * s * (d + 1) * 4;
}

vattn_status vattn_kv_append_raw(const vattn_cache_desc* c, const void* k_new, const void* v_new,
                                 int32_t batch, int32_t n_new, const int32_t* seqlens,
                                 const int32_t* batch_idx, void* stream) {
  return kguard([&] {
    vattn::launch_kv_append(nullptr, -1, vattn::view_from_desc(c), k_new, v_new, batch, n_new,
                            seqlens, batch_idx, (cudaStream_t)stream);
  });
}

vattn_status vattn_decode_raw(const vattn_cache_desc* c, const void* q, void* out, int32_t batch,
                              int32_t hq, const int32_t* seqlens, const int32_t* batch_idx,
                              float scale, int32_t num_splits, void* ws, int64_t ws_bytes,
                              void* stream) {
  return kguard([&] {
    const vattn::CacheView v = vattn::view_from_desc(c);
    vattn::launch_decode(nullptr, -1, v, q, out, batch, hq, seqlens, batch_idx, scale, num_splits,
                         ws, ws_bytes, (cudaStream_t)stream, nullptr, nullptr);
  });
}

vattn_status vattn_decode_append_raw(const vattn_cache_desc* c, const void* q, const void* k_new,
                                     const void* v_new, void* out, int32_t batch, int32_t hq,
                                     const int32_t* cache_seqlens, const int32_t* batch_idx,
                                     float scale, int32_t num_splits, void* ws, int64_t ws_bytes,
                                     void* stream) {
  return kguard([&] {
    const vattn::CacheView v = vattn::view_from_desc(c);
    vattn::launch_decode(nullptr, -1, v, q, out, batch, hq, cache_seqlens, batch_idx, scale,
                         num_splits, ws, ws_bytes, (cudaStream_t)stream, k_new, v_new);
  });
}

vattn_status vattn_kv_append_rotary_raw(const vattn_cache_desc* c, const void* k_new, const void* v_new,
                                        int32_t batch, int32_t n_new, const int32_t* seqlens,
                                        const int32_t* batch_idx, const vattn_rotary* rotary, void* stream) {
  return kguard([&] {
    if (!rotary) throw Fail(VATTN_VALUE_ERROR, "null rotary descriptor");
    const vattn::Rotary rot{rotary->cos, rotary->sin, rotary->rotary_dim, rotary->interleaved};
    vattn::launch_kv_append(nullptr, -1, vattn::view_from_desc(c), k_new, v_new, batch, n_new, seqlens,
                            batch_idx, (cudaStream_t)stream, &rot);
  });
}

vattn_status vattn_decode_append_rotary_raw(const vattn_cache_desc* c, const void* q, const void* k_new,
                                            const void* v_new, void* out, int32_t batch, int32_t hq,
                                            const int32_t* cache_seqlens, const int32_t* batch_idx, float scale,
                                            int32_t num_splits, const vattn_rotary* rotary, void* ws,
                                            int64_t ws_bytes, void* stream) {
  return kguard([&] {
    if (!rotary) throw Fail(VATTN_VALUE_ERROR, "null rotary descriptor");
    const vattn::CacheView v = vattn::view_from_desc(c);
    const vattn::Rotary rot{rotary->cos, rotary->sin, rotary->rotary_dim, rotary->interleaved};
    vattn::launch_decode(nullptr, -1, v, q, out, batch, hq, cache_seqlens, batch_idx, scale, num_splits, ws,
                         ws_bytes, (cudaStream_t)stream, k_new, v_new, nullptr, &rot);
  });
}

vattn_status vattn_kv_append_paged(const void* k_new, const void* v_new, void* k_pool, void* v_pool,
                                   int32_t block_size, int32_t n_kv_heads, int32_t head_dim,
                                   const int32_t* block_table, int32_t max_blocks_per_seq, int32_t batch,
                                   int32_t n_new, const int32_t* cache_seqlens, void* stream) {
  return kguard([&] {
    if (batch <= 0 || n_new <= 0) return;
    vattn::PagedAppendParams p;
    p.k_src = reinterpret_cast<const uint4*>(k_new);
    p.v_src = reinterpret_cast<const uint4*>(v_new);
    p.k_pool = reinterpret_cast<char*>(k_pool);
    p.v_pool = reinterpret_cast<char*>(v_pool);
    p.seqlens = cache_seqlens;
    p.block_table = block_table;
    p.max_blocks = max_blocks_per_seq;
    p.block_size = block_size;
    p.n_new = n_new;
    p.row_bytes = (int64_t)n_kv_heads * head_dim * 2;
    p.chunks_per_row = (int32_t)(p.row_bytes / 16);
    p.total_chunks = (int64_t)batch * n_new * p.chunks_per_row;
    const int64_t want = (p.total_chunks + 255) / 256;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)vattn::num_sms() * 8));
    vattn::kv_append_paged_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(p);
    vattn::check_rt(cudaGetLastError(), "kv_append_paged launch");
  });
}

vattn_status vattn_decode_paged(const void* q, const void* k_pool, const void* v_pool,
                                int32_t num_blocks, int32_t block_size, int32_t hkv, int32_t d,
                                const int32_t* block_table, int32_t max_blocks, void* out,
                                int32_t batch, int32_t hq, const int32_t* seqlens, float scale,
                                int32_t num_splits, void* ws, int64_t ws_bytes, void* stream) {
  return kguard([&] {
    if (d != 64 && d != 128) throw Fail(VATTN_UNSUPPORTED, "head_dim must be 64 or 128");
    if (block_size <= 0 || (block_size < vattn::kTile && vattn::kTile % block_size) ||
        (block_size >= vattn::kTile && block_size % vattn::kTile))
      throw Fail(VATTN_UNSUPPORTED, "block_size must divide 64 or be a multiple of 64");
    const int box = std::min(block_size, vattn::kTile);
    const int64_t row = (int64_t)hkv * d * 2;
    const CUtensorMap km = vattn::make_kv_map((uint64_t)k_pool, d, hkv, row, block_size,
                                              row * block_size, num_blocks, box);
    const CUtensorMap vm = vattn::make_kv_map((uint64_t)v_pool, d, hkv, row, block_size,
                                              row * block_size, num_blocks, box);
    vattn::decode_common(km, vm, d, hkv, hq, q, out, batch, seqlens, nullptr, block_table,
                         max_blocks, block_size, box, scale, num_splits, max_blocks * block_size,
                         ws, ws_bytes, true, (cudaStream_t)stream);
  });
}

}  // extern "C"
