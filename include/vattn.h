/*
 * vattn.h — C ABI of the B200-native vAttention hot path (libvattn.so).
 *
 * Plain pointers and sizes only; no torch types.  Every entry point returns a vattn_status
 * (0 = OK).  On failure vattn_last_error() returns a message for the calling thread.
 *
 * Reference interface each group replaces (paths under /root/reference/pkg/src/kvsim/):
 *   vattn_create / vattn_destroy      KVCacheManager.__init__            manager.py:85-130
 *   vattn_alloc_reqid                 KVCacheManager.alloc_reqid         manager.py:163-178
 *   vattn_free_reqid                  KVCacheManager.free_reqid          manager.py:180-190
 *   vattn_step                        KVCacheManager.step                manager.py:255-296
 *   vattn_plan_overlap / _plan_fetch  KVCacheManager.plan_overlap        manager.py:298-311
 *   vattn_execute_plan                KVCacheManager.execute_plan        manager.py:313-333
 *   vattn_eager_prepare               KVCacheManager.eager_prepare       manager.py:335-361
 *   vattn_reclaim                     KVCacheManager.reclaim             manager.py:363-372
 *   vattn_reclaim_until               KVCacheManager._reclaim_until      manager.py:238-251
 *   vattn_bg_submit / vattn_bg_wait   _VattentionRuntime.background      simulator.py:199-203
 *                                     (execute_plan -> eager_prepare -> reclaim, on a real thread)
 *   vattn_slot_state / vattn_counters / vattn_api_stats / vattn_buffer_mappings / vattn_events
 *                                     introspection read by the reference tests: RequestSlot
 *                                     manager.py:66-75, PhysicalPool vmm.py:102-127,
 *                                     VmmDevice.calls/ledger_us vmm.py:172-173,
 *                                     VirtualKVBuffer.mappings vmm.py:141-147
 *   vattn_buffer_base                 Table 3 `init` "returns a list of KV cache tensors"
 *                                     (PAPER.md:434-437); the VA of buffer i never moves
 *   vattn_kv_append / vattn_decode / vattn_prefill
 *                                     no reference code; semantics of
 *                                     flash_attn_with_kvcache as used by PAPER.md:511
 *
 * Error codes map 1:1 onto the reference exceptions (manager.py:28-33, vmm.py:26-47).
 */
#ifndef VATTN_H_
#define VATTN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum vattn_status {
  VATTN_OK = 0,
  VATTN_BATCH_FULL = 1,        /* BatchFullError      manager.py:28 */
  VATTN_DOUBLE_FREE = 2,       /* DoubleFreeError     manager.py:32 */
  VATTN_VALUE_ERROR = 3,       /* ValueError          manager.py:86,100-109,265-272 */
  VATTN_POOL_EXHAUSTED = 4,    /* PoolExhaustedError  vmm.py:34 */
  VATTN_MAPPING_ERROR = 5,     /* MappingError        vmm.py:38 */
  VATTN_ALIGNMENT_ERROR = 6,   /* AlignmentError      vmm.py:30 */
  VATTN_INVALID_FREE = 7,      /* InvalidFreeError    vmm.py:42 */
  VATTN_LATENCY_CONFIG = 8,    /* LatencyConfigError  vmm.py:46 */
  VATTN_CUDA_ERROR = 9,        /* driver / runtime failure */
  VATTN_UNSUPPORTED = 10,      /* shape / layout the kernels do not cover */
  VATTN_BAD_STATE = 11         /* misuse (e.g. bg_wait without submit) */
} vattn_status;

typedef enum vattn_backend {
  VATTN_BACKEND_SHADOW = 0,    /* bookkeeping only (no device); used by CPU parity tests */
  VATTN_BACKEND_CUDA = 1       /* real cuMemAddressReserve/cuMemCreate/cuMemMap/cuMemSetAccess */
} vattn_backend;

typedef struct vattn_latency_entry {
  const char* api;             /* e.g. "cuMemMap" (vmm.py:55-68 names) */
  int64_t page_group_bytes;
  double us;
} vattn_latency_entry;

typedef struct vattn_config {
  /* ModelGeometry (geometry.py:64-117) */
  int32_t n_layers;
  int32_t kv_heads_total;
  int32_t head_dim;
  int32_t bytes_per_elem;
  int32_t tp_degree;
  int32_t n_q_heads_total;     /* build addition; 0 = kv_heads_total */
  int64_t max_context;
  int64_t max_batch;
  /* ManagerConfig (manager.py:42-63) */
  int64_t page_group_size;
  int64_t pool_bytes;
  double reclaim_threshold;
  double pre_create_fraction;
  int64_t eager_groups;
  int32_t sliced;
  /* build additions */
  int32_t backend;             /* vattn_backend */
  int32_t device;              /* CUDA ordinal for VATTN_BACKEND_CUDA */
  int32_t release_physical;    /* 1: cuMemRelease on unmap; 0: recycle the 2 MiB handle */
  int32_t log_events;          /* 1: keep the (op, buffer, offset) log for vattn_events */
  int32_t batch_set_access;    /* 1: coalesce cuMemSetAccess over contiguous page runs */
  const vattn_latency_entry* latency;  /* NULL = Table 2 defaults (vmm.py:55-68) */
  int32_t n_latency;
  /* B200 addition: physically pre-map pages each active slot needs within this many more tokens
   * (background jobs with VATTN_BG_PREFETCH); logical state stays the reference's. 0 = off. */
  int32_t prefetch_tokens;
  /* ...and physically pre-map the next `prefetch_slots` slots alloc_reqid would hand out, up to
   * `prefetch_slot_tokens` tokens of prompt (speculative eager; logical state untouched) */
  int32_t prefetch_slots;
  int32_t prefetch_slot_tokens;
  /* B200 addition: a trimmed or reclaimed page-group stays physically mapped as a speculative
   * page (logically released exactly as the reference does); the driver unmap happens only if
   * its handle is needed elsewhere, or never when the slot grows back over it.  Needs
   * release_physical = 0. */
  int32_t lazy_unmap;
  /* B200 addition: back `phys_chunk_groups` consecutive page-groups of a buffer with ONE physical
   * handle (cuMemCreate of phys_chunk_groups x page_group_size), mapped by one cuMemMap + one
   * cuMemSetAccess when the first of them is mapped (logically or speculatively) and unmapped when
   * the last one goes.  The page-group bookkeeping (shadow state, counters, events) is unchanged;
   * only the driver traffic and the physical footprint change.  0 or 1 = one handle per group. */
  int32_t phys_chunk_groups;
} vattn_config;

typedef struct vattn_t vattn_t;

typedef struct vattn_step_result {
  int32_t ok;                  /* StepResult.ok (manager.py:78-81) */
  double sync_us;              /* StepResult.sync_us: modelled Table-2 µs */
  double wall_us;              /* measured host wall time of this call (driver calls incl.) */
  double bg_wait_us;           /* time spent joining an outstanding background window */
} vattn_step_result;

typedef struct vattn_counters {
  int64_t created, mapped, precreated, total_mapped_bytes;
  int64_t capacity, page_group_size;
  int64_t buffer_count, groups_per_slot, slot_stride, buffer_size;
  int64_t per_buffer_token_bytes, max_batch, max_context;
  int64_t eager_slot;          /* -1 = None */
  int64_t next_handle_id;
  double init_us, charged_us;
  /* measured (real backend) */
  int64_t real_maps, real_unmaps, real_set_access_calls, real_creates, real_releases;
  double real_map_wall_us, real_unmap_wall_us, real_create_wall_us, real_set_access_wall_us;
  double init_wall_us;
  int64_t spec_maps, spec_hits, spec_steals, spec_pages;   /* physical prefetch */
  int64_t lazy_unmaps;         /* logical unmaps that kept the page mapped (lazy_unmap) */
  /* physical chunks (phys_chunk_groups > 1): groups per chunk, chunks mapped now, their bytes */
  int64_t phys_chunk_groups, phys_chunks_mapped, phys_mapped_bytes;
} vattn_counters;

typedef struct vattn_bg_result {
  double plan_us, eager_us, reclaim_us;   /* modelled µs per component */
  int64_t reclaimed_groups;
  double bg_wall_us;                      /* wall time the background thread worked */
  double waited_us;                       /* how long vattn_bg_wait blocked */
} vattn_bg_result;

/* background job flags, executed in this order (simulator.py:199-203) */
#define VATTN_BG_EXECUTE_PLAN 1u
#define VATTN_BG_EAGER 2u
#define VATTN_BG_RECLAIM 4u
/* execute_plan submitted ahead of the next admission: record per-slot credits so that
 * alloc_reqid ranks slots as if the plan ran after it (reference order, simulator.py:395-418) */
#define VATTN_BG_CREDIT 8u
/* vattn_iteration_step: defer eager/reclaim past step onto the background thread when the
 * result is provably identical */
#define VATTN_ITER_DEFER 16u
/* run the physical prefetch (see vattn_config.prefetch_tokens) at the end of the job */
#define VATTN_BG_PREFETCH 32u

typedef struct vattn_iteration_result {
  int32_t ok;                  /* step ok (preempt on 0) */
  int32_t deferred;            /* eager/reclaim were queued behind step */
  double sync_us;              /* modelled µs of step */
  double eager_us, reclaim_us; /* modelled µs of eager/reclaim when run synchronously */
  int64_t reclaimed_groups;
  double bg_wait_us;           /* joining the previous background window */
  double sync_bg_wall_us;      /* wall time of synchronous eager+reclaim */
  double wall_us;              /* wall time of the whole call = exposed allocation time */
} vattn_iteration_result;

/* ---- lifecycle --------------------------------------------------------------------- */
const char* vattn_last_error(void);
int32_t vattn_abi_version(void);
/* sizeof of the ABI structs, for binding checks: out[0..7] = vattn_config, vattn_counters,
 * vattn_step_result, vattn_bg_result, vattn_iteration_result, vattn_cache_desc, vattn_rotary,
 * vattn_latency_entry; returns how many were written (min(n, 8)) */
int32_t vattn_abi_sizes(int64_t* out, int32_t n);
vattn_status vattn_create(const vattn_config* cfg, vattn_t** out);
vattn_status vattn_destroy(vattn_t* h);

/* ---- Table 3 API + §6.1 optimisations ---------------------------------------------- */
vattn_status vattn_alloc_reqid(vattn_t* h, int32_t* req_id);
vattn_status vattn_free_reqid(vattn_t* h, int32_t req_id);
vattn_status vattn_step(vattn_t* h, const int64_t* seq_lens, int32_t n, vattn_step_result* out);
/* One serving iteration's allocation work in the reference order (simulator.py:414-426):
 * [join background] -> eager_prepare/reclaim per flags (sync, or deferred behind step when
 * VATTN_ITER_DEFER and provably equivalent) -> step. */
vattn_status vattn_iteration_step(vattn_t* h, const int64_t* seq_lens, int32_t n, uint32_t flags,
                                  int64_t eager_k, vattn_iteration_result* out);
vattn_status vattn_plan_overlap(vattn_t* h, const int64_t* next_seq_lens, int32_t n,
                                int64_t* n_entries);
vattn_status vattn_plan_fetch(vattn_t* h, int64_t* triples, int64_t cap_entries);
vattn_status vattn_execute_plan(vattn_t* h, const int64_t* triples, int64_t n_entries,
                                double* us);
vattn_status vattn_eager_prepare(vattn_t* h, int64_t k_groups /* <0: config */, double* us);
vattn_status vattn_reclaim(vattn_t* h, int64_t* freed, double* us);
vattn_status vattn_reclaim_until(vattn_t* h, int64_t target_available_bytes, int64_t* freed,
                                 double* us);
/* background thread: triples == NULL reuses the last vattn_plan_overlap result */
vattn_status vattn_bg_submit(vattn_t* h, const int64_t* triples, int64_t n_entries,
                             uint32_t flags, int64_t eager_k);
vattn_status vattn_bg_wait(vattn_t* h, vattn_bg_result* out);
/* unmap fence: record "the KV cache may be read by work queued on `stream` so far" (one event
 * per stream; unmaps wait for every stream's) */
vattn_status vattn_mark_use(vattn_t* h, void* stream);
/* Read guard: the decode / append kernels clamp every row to the rows its slot backs (and skip
 * slots outside [0, max_batch)) instead of faulting the context, and record the violation in
 * host-mapped words.  The next allocator call or kernel launch on the handle — or this call —
 * returns VATTN_VALUE_ERROR for it (after the kernel ran; synchronize first to be sure). */
vattn_status vattn_check_errors(vattn_t* h);

/* ---- introspection ------------------------------------------------------------------ */
vattn_status vattn_counters_get(vattn_t* h, vattn_counters* out);
/* same, without joining the background queue (monitoring; may race with a running job) */
vattn_status vattn_counters_peek(vattn_t* h, vattn_counters* out);
/* 5 int64 per slot: active, context_len, mapped_groups, phase(0 inactive,1 prefill,2 decode),
 * freed_seq */
vattn_status vattn_slot_state(vattn_t* h, int64_t* out, int64_t cap_slots);
int32_t vattn_api_count(void);
const char* vattn_api_name(int32_t i);
/* calls[i] and ledger_us[i] per API i (vattn_api_name order) + first-charge order */
vattn_status vattn_api_stats(vattn_t* h, int64_t* calls, double* ledger_us, int32_t* order,
                             int32_t* n_order);
vattn_status vattn_buffer_mappings(vattn_t* h, int32_t buffer_id, int64_t* offsets,
                                   int64_t* handle_ids, int64_t cap, int64_t* n);
/* drain the event log: triples (0=map|1=unmap, buffer_id, offset) */
vattn_status vattn_events(vattn_t* h, int64_t* triples, int64_t cap_entries, int64_t* n);
vattn_status vattn_buffer_base(vattn_t* h, int32_t buffer_id, uint64_t* dptr);

/* ---- admission-aware prefetch (B200 addition; logical state untouched) --------------------
 * The next `k` slots consecutive alloc_reqid calls would return now (eager slot first, then by
 * (mapped_groups, -req_id) with plan credits, manager.py:163-178); out[k], *n = how many. */
vattn_status vattn_predict_alloc(vattn_t* h, int32_t k, int32_t* out, int32_t* n);
/* Foreground launch window: while active != 0 the prefetch worker makes no new driver call
 * (cuMemSetAccess holds the kernel driver's lock for up to milliseconds on B200 and would stall
 * the caller's kernel launches).  Set around an iteration's launch burst. */
vattn_status vattn_set_foreground(vattn_t* h, int32_t active);
/* Ask the prefetch worker to back rows [0, tokens[i]) of slots[i] physically (queued prompts
 * about to be admitted there); replaces the previous hint set; used by the next background job
 * submitted with VATTN_BG_PREFETCH. */
vattn_status vattn_prefetch_hint(vattn_t* h, const int32_t* slots, const int64_t* tokens, int32_t n);
/* *ready = 1 when every page-group of rows [0, tokens) of `slot` is mapped in every buffer,
 * logically or speculatively (a step to that length then needs no driver call). */
vattn_status vattn_slot_ready(vattn_t* h, int32_t slot, int64_t tokens, int32_t* ready);

/* Table 2 analog measured on this device: mean µs per call at `page_bytes` (out[10]: reserve,
 * create, map, set_access, unmap, release, address_free, set_access-per-page batched by `run`,
 * map and set_access again on recycled (previously mapped) handles). */
vattn_status vattn_vmm_microbench(int32_t device, int64_t page_bytes, int32_t n_pages, int32_t run,
                                  double* out);

/* Probe: per-2MiB-slice map/set_access/unmap µs when slices come from one big physical handle
 * (big_handle=1) or one handle each, with `extra_handles` other live allocations. */
vattn_status vattn_vmm_slice_probe(int32_t device, int32_t n_pages, int32_t big_handle,
                                   int32_t extra_handles, double* out);

/* Probe: map + set_access of `n_pages` fresh 2 MiB pages from `n_threads` threads at once
 * (out[0] µs/page, out[1] total ms, out[2] unmap µs/page). */
vattn_status vattn_vmm_parallel_probe(int32_t device, int32_t n_pages, int32_t n_threads, double* out);

/* ---- kernels (bf16 K/V/Q/O; layouts in DESIGN.md §3) --------------------------------- */
/* Write k_new/v_new [batch, n_new, Hkv, D] at rows cache_seqlens[b] + i of slot
 * cache_batch_idx[b] (NULL = identity) of layer `layer`.  Device int32 arrays. */
vattn_status vattn_kv_append(vattn_t* h, int32_t layer, const void* k_new, const void* v_new,
                             int32_t batch, int32_t n_new, const int32_t* cache_seqlens,
                             const int32_t* cache_batch_idx, void* stream);
/* o[b, :, :] = softmax(q[b] K[slot, :seqlen]ᵀ · scale) V ; q/o [batch, Hq, D]. */
vattn_status vattn_decode(vattn_t* h, int32_t layer, const void* q, void* out, int32_t batch,
                          const int32_t* cache_seqlens, const int32_t* cache_batch_idx,
                          float scale, int32_t num_splits /* 0 = auto */, void* stream);
/* Fused KV-append + decode (flash_attn_with_kvcache k=/v= semantics):
 * k_new/v_new [batch, Hkv, D] go to row cache_seqlens[b] (length BEFORE the token) of slot
 * cache_batch_idx[b], and attention runs over cache_seqlens[b] + 1 rows.  One launch. */
vattn_status vattn_decode_append(vattn_t* h, int32_t layer, const void* q, const void* k_new,
                                 const void* v_new, void* out, int32_t batch,
                                 const int32_t* cache_seqlens, const int32_t* cache_batch_idx,
                                 float scale, int32_t num_splits, void* stream);
/* Rotary embedding for the fused append+decode (flash_attn_with_kvcache rotary_cos / rotary_sin /
 * rotary_interleaved, as the paper's kernels use it): q and k_new are rotated at
 * position cache_seqlens[b] before attention, and k is cached rotated.  Tables fp32
 * [positions, rotary_dim / 2]; rotary_dim a multiple of 16, <= head_dim. */
typedef struct vattn_rotary {
  const float* cos;
  const float* sin;
  int32_t rotary_dim;
  int32_t interleaved;         /* 0: GPT-NeoX halves, 1: GPT-J adjacent pairs */
} vattn_rotary;
vattn_status vattn_decode_append_rotary(vattn_t* h, int32_t layer, const void* q, const void* k_new,
                                        const void* v_new, void* out, int32_t batch,
                                        const int32_t* cache_seqlens, const int32_t* cache_batch_idx,
                                        float scale, int32_t num_splits, const vattn_rotary* rotary,
                                        void* stream);
/* Rotary at append / prefill (same tables and layouts): kv_append rotates each new k row at its
 * position cache_seqlens[b] + i before caching it; prefill rotates query row i at position
 * kv_len - n_q + i inside the tcgen05 kernel (in shared memory, before the first MMA). */
vattn_status vattn_kv_append_rotary(vattn_t* h, int32_t layer, const void* k_new, const void* v_new,
                                    int32_t batch, int32_t n_new, const int32_t* cache_seqlens,
                                    const int32_t* cache_batch_idx, const vattn_rotary* rotary,
                                    void* stream);
vattn_status vattn_prefill_rotary(vattn_t* h, int32_t layer, const void* q, void* out, int32_t n_q,
                                  int32_t req_slot, int32_t kv_len, float scale, int32_t causal,
                                  const vattn_rotary* rotary, void* stream);
/* Several requests' prefills in one launch (flash_attn_varlen_func-style packed queries): host
 * arrays of n_req entries; request i's query rows are q[q_start[i] .. + n_q[i]] (packed
 * [total, Hq, D]), attending causally over rows [0, kv_len[i]) of slot slots[i]; outputs at the
 * same packed rows.  The per-call schedule is uploaded on `stream` (not graph-capturable). */
vattn_status vattn_prefill_varlen(vattn_t* h, int32_t layer, const void* q, void* out, int32_t n_req,
                                  const int32_t* q_start, const int32_t* n_q, const int32_t* slots,
                                  const int32_t* kv_len, float scale, int32_t causal, void* stream);
/* causal (bottom-right) prefill of q [n_q, Hq, D] against slot rows [0, kv_len). */
vattn_status vattn_prefill(vattn_t* h, int32_t layer, const void* q, void* out, int32_t n_q,
                           int32_t req_slot, int32_t kv_len, float scale, int32_t causal,
                           void* stream);

/* ---- standalone kernels (no manager; caller-owned device memory) ------------------------ */
typedef struct vattn_cache_desc {
  const void* k_base;          /* token-major [slots, slot_tokens, Hkv, D] with slot stride */
  const void* v_base;
  int64_t slot_stride_bytes;
  int64_t token_stride_bytes;  /* 0 = Hkv*D*2 (per-layer buffers); N*Hkv*D*2 when layer-sliced */
  int32_t slot_tokens;         /* rows addressable per slot (>= every seqlen) */
  int32_t n_slots;
  int32_t n_kv_heads;
  int32_t head_dim;
} vattn_cache_desc;

vattn_status vattn_kv_append_raw(const vattn_cache_desc* c, const void* k_new, const void* v_new,
                                 int32_t batch, int32_t n_new, const int32_t* cache_seqlens,
                                 const int32_t* cache_batch_idx, void* stream);
vattn_status vattn_decode_raw(const vattn_cache_desc* c, const void* q, void* out,
                              int32_t batch, int32_t n_q_heads, const int32_t* cache_seqlens,
                              const int32_t* cache_batch_idx, float scale, int32_t num_splits,
                              void* workspace, int64_t workspace_bytes, void* stream);
vattn_status vattn_prefill_raw(const vattn_cache_desc* c, const void* q, void* out, int32_t n_q,
                               int32_t n_q_heads, int32_t req_slot, int32_t kv_len, float scale,
                               int32_t causal, void* stream);
vattn_status vattn_decode_append_raw(const vattn_cache_desc* c, const void* q, const void* k_new,
                                     const void* v_new, void* out, int32_t batch, int32_t n_q_heads,
                                     const int32_t* cache_seqlens, const int32_t* cache_batch_idx,
                                     float scale, int32_t num_splits, void* workspace,
                                     int64_t workspace_bytes, void* stream);
vattn_status vattn_decode_append_rotary_raw(const vattn_cache_desc* c, const void* q, const void* k_new,
                                            const void* v_new, void* out, int32_t batch, int32_t n_q_heads,
                                            const int32_t* cache_seqlens, const int32_t* cache_batch_idx,
                                            float scale, int32_t num_splits, const vattn_rotary* rotary,
                                            void* workspace, int64_t workspace_bytes, void* stream);
vattn_status vattn_kv_append_rotary_raw(const vattn_cache_desc* c, const void* k_new, const void* v_new,
                                        int32_t batch, int32_t n_new, const int32_t* cache_seqlens,
                                        const int32_t* cache_batch_idx, const vattn_rotary* rotary,
                                        void* stream);
vattn_status vattn_prefill_rotary_raw(const vattn_cache_desc* c, const void* q, void* out, int32_t n_q,
                                      int32_t n_q_heads, int32_t req_slot, int32_t kv_len, float scale,
                                      int32_t causal, const vattn_rotary* rotary, void* stream);
vattn_status vattn_prefill_varlen_raw(const vattn_cache_desc* c, const void* q, void* out,
                                      int32_t n_q_heads, int32_t n_req, const int32_t* q_start,
                                      const int32_t* n_q, const int32_t* slots, const int32_t* kv_len,
                                      float scale, int32_t causal, void* stream);
/* Paged-layout comparison kernel (PagedAttention block table; PAPER.md:602 block sizes):
 * pools [num_blocks, block_size, Hkv, D], block_table [batch, max_blocks] int32. */
vattn_status vattn_decode_paged(const void* q, const void* k_pool, const void* v_pool,
                                int32_t num_blocks, int32_t block_size, int32_t n_kv_heads,
                                int32_t head_dim, const int32_t* block_table,
                                int32_t max_blocks_per_seq, void* out, int32_t batch,
                                int32_t n_q_heads, const int32_t* seqlens, float scale,
                                int32_t num_splits, void* workspace, int64_t workspace_bytes,
                                void* stream);
/* serving benchmark only: occupy `stream` for `ns` ns of device time (dense-layer compute proxy) */
vattn_status vattn_compute_proxy(uint64_t ns, void* stream);
/* split count the auto heuristic picks for `batch` rows x Hkv heads at max_seqlen tokens */
int32_t vattn_decode_num_splits(int32_t batch, int32_t n_kv_heads, int32_t max_seqlen);
/* Paged-layout append (comparison path): row cache_seqlens[b] + i of sequence b goes to block
 * block_table[b][pos / block_size], row pos % block_size of pools [num_blocks, block_size, Hkv, D]. */
vattn_status vattn_kv_append_paged(const void* k_new, const void* v_new, void* k_pool, void* v_pool,
                                   int32_t block_size, int32_t n_kv_heads, int32_t head_dim,
                                   const int32_t* block_table, int32_t max_blocks_per_seq, int32_t batch,
                                   int32_t n_new, const int32_t* cache_seqlens, void* stream);
/* Paged-layout causal prefill (same tcgen05 kernel, K/V gathered per block): pools
 * [num_blocks, block_size, Hkv, D], block_table [max_blocks] int32 for the one request. */
vattn_status vattn_prefill_paged(const void* q, const void* k_pool, const void* v_pool,
                                 int32_t num_blocks, int32_t block_size, int32_t n_kv_heads,
                                 int32_t head_dim, const int32_t* block_table, int32_t kv_len,
                                 void* out, int32_t n_q, int32_t n_q_heads, float scale, int32_t causal,
                                 void* stream);
int64_t vattn_decode_workspace_bytes(int32_t batch, int32_t n_q_heads, int32_t head_dim,
                                     int32_t num_splits);
/* Name of the decode kernel variant (template arguments) a contiguous launch of this shape runs,
 * written to buf (NUL-terminated, at most cap bytes); returns the split count (num_splits 0 =
 * automatic) or -1.  For labelling measurements (bench.py roofline.kernel). */
int32_t vattn_decode_kernel_name(int32_t batch, int32_t hkv, int32_t max_seqlen, int32_t num_splits,
                                 int32_t head_dim, char* buf, int32_t cap);

/* ---- fused head all-gather over NVLink peer memory ----------------------------
 * Replaces the NCCL all-gather of the per-rank decode outputs [B, Hq/G, D] into [B, Hq, D]
 * (north_star: "NCCL over NVLink is used only for the final head all-gather when the caller
 * requests full outputs"; the reference has no multi-GPU code — every worker runs the same
 * allocator, geometry.py:96-98 kv_heads_per_worker).  The decode epilogue stores
 * each row into every rank's staging area (two, alternating per launch) over peer memory and
 * signals; vattn_gather_wait makes `stream` wait until all ranks' rows have landed and copies the
 * full output out.  Every rank issues the same sequence of gathered launches, each followed by a
 * vattn_gather_wait on the same stream before its next gathered launch; the output then has the
 * lifetime of any stream-ordered buffer (no peer writes into it). */
#define VATTN_IPC_HANDLE_BYTES 64
typedef struct vattn_gather vattn_gather_t;
/* one per rank (collective setup): allocates this rank's full-output buffer of out_bytes
 * (>= max_batch * Hq_total * D * 2) + signal words; writes its CUDA IPC handle
 * (VATTN_IPC_HANDLE_BYTES) to ipc_handle for the caller to all-gather across ranks. */
vattn_status vattn_gather_create(int32_t device, int32_t rank, int32_t world, int64_t out_bytes,
                                 vattn_gather_t** out, void* ipc_handle);
/* map every peer's buffer: handles = world x VATTN_IPC_HANDLE_BYTES in rank order */
vattn_status vattn_gather_open(vattn_gather_t* g, const void* handles);
/* `world` simulated ranks on one device in this process (out[world]); same kernels/protocol */
vattn_status vattn_gather_create_local(int32_t device, int32_t world, int64_t out_bytes,
                                       vattn_gather_t** out);
/* device address of this rank's front area [max_batch, Hq_total, D] bf16 (rank-local; the
 * destination of vattn_gather_wait when out is NULL) */
vattn_status vattn_gather_output(vattn_gather_t* g, uint64_t* dptr);
/* stream-ordered: wait (bounded: 10 s, env VATTN_GATHER_TIMEOUT_MS) until every rank's latest
 * gathered launch has landed, then copy the first out_bytes (batch * Hq_total * D * 2; multiple
 * of 16) of the full output to out (16-byte aligned; NULL = the front area).  out_bytes 0: wait
 * only. */
vattn_status vattn_gather_wait(vattn_gather_t* g, void* out, int64_t out_bytes, void* stream);
/* bit r set = the wait for rank r timed out (a rank skipped a launch) */
vattn_status vattn_gather_check(vattn_gather_t* g, uint32_t* timed_out_mask);
vattn_status vattn_gather_destroy(vattn_gather_t* g);
/* decode (k_new/v_new non-NULL: fused append, as vattn_decode_append) of this rank's Hq_local
 * heads, rows stored into every rank's full output at head offset rank * Hq_local */
vattn_status vattn_decode_gather(vattn_t* h, int32_t layer, const void* q, const void* k_new,
                                 const void* v_new, vattn_gather_t* g, int32_t batch,
                                 const int32_t* cache_seqlens, const int32_t* cache_batch_idx,
                                 float scale, int32_t num_splits, void* stream);
vattn_status vattn_decode_gather_raw(const vattn_cache_desc* c, const void* q, const void* k_new,
                                     const void* v_new, vattn_gather_t* g, int32_t batch,
                                     int32_t n_q_heads, const int32_t* cache_seqlens,
                                     const int32_t* cache_batch_idx, float scale, int32_t num_splits,
                                     void* workspace, int64_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VATTN_H_ */
