// vAttention allocator core: policy state machine, driver bookkeeping shadow, real CUDA VMM
// backend and the background mapping thread, exported through the C ABI in include/vattn.h.
//
// The policy is the reference KVCacheManager (/root/reference/pkg/src/kvsim/manager.py) and
// its mock driver VmmDevice (vmm.py); each method below cites the lines it reproduces.  The
// shadow (counters, handle ids, per-API call counts, modelled Table-2 µs) is always kept, so
// the reference's state is reproducible bit for bit; with VATTN_BACKEND_CUDA every shadow
// map/unmap/create/release is also issued to the real driver at 2 MiB granularity.

#include <cuda.h>
#include <cuda_runtime_api.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "internal.h"
#include "vattn.h"

namespace vattn {

static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

// ------------------------------------------------------------------------------ driver
static Driver g_drv;
static bool g_drv_loaded = false;
static std::mutex g_drv_mu;

template <typename F>
static void load_sym(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaError_t e = cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q);
  if (e != cudaSuccess || p == nullptr || q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    throw Fail(VATTN_CUDA_ERROR, std::string("driver entry point unavailable: ") + name);
  }
  *fn = reinterpret_cast<F>(p);
}

const Driver& driver() {
  std::lock_guard<std::mutex> lk(g_drv_mu);
  if (!g_drv_loaded) {
    load_sym("cuMemAddressReserve", &g_drv.MemAddressReserve);
    load_sym("cuMemAddressFree", &g_drv.MemAddressFree);
    load_sym("cuMemCreate", &g_drv.MemCreate);
    load_sym("cuMemRelease", &g_drv.MemRelease);
    load_sym("cuMemMap", &g_drv.MemMap);
    load_sym("cuMemUnmap", &g_drv.MemUnmap);
    load_sym("cuMemSetAccess", &g_drv.MemSetAccess);
    load_sym("cuMemGetAllocationGranularity", &g_drv.MemGetAllocationGranularity);
    load_sym("cuCtxGetCurrent", &g_drv.CtxGetCurrent);
    load_sym("cuCtxSetCurrent", &g_drv.CtxSetCurrent);
    load_sym("cuDevicePrimaryCtxRetain", &g_drv.DevicePrimaryCtxRetain);
    load_sym("cuDeviceGet", &g_drv.DeviceGet);
    load_sym("cuGetErrorString", &g_drv.GetErrorString);
    load_sym("cuTensorMapEncodeTiled", &g_drv.TensorMapEncodeTiled);
    g_drv_loaded = true;
  }
  return g_drv;
}

void check_cu(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* s = "?";
  if (g_drv_loaded && g_drv.GetErrorString) g_drv.GetErrorString(r, &s);
  throw Fail(VATTN_CUDA_ERROR, std::string(what) + ": CUresult " + std::to_string(int(r)) + " " + s);
}

void check_rt(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  throw Fail(VATTN_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

static double now_us() {
  using namespace std::chrono;
  return duration<double, std::micro>(steady_clock::now().time_since_epoch()).count();
}

// CPython >= 3.12 `sum()` of floats (Neumaier compensated summation).  The reference totals
// its ledger with sum() (vmm.py:191-195, :301-302), so the modelled µs are reproduced bit for
// bit only with the same algorithm.
struct PySum {
  double s = 0.0, c = 0.0;
  void add(double x) {
    const double t = s + x;
    if (std::fabs(s) >= std::fabs(x)) c += (s - t) + x;
    else c += (x - t) + s;
    s = t;
  }
  double value() const { return (c != 0.0 && std::isfinite(c)) ? s + c : s; }
};

// ------------------------------------------------------------------------------ latency model
// Table 2 of the paper as encoded in vmm.py:55-68.
enum Api {
  A_vMemReserve, A_cuMemAddressReserve, A_vMemCreate, A_cuMemCreate, A_vMemMap, A_cuMemMap,
  A_cuMemSetAccess, A_cuMemUnmap, A_vMemRelease, A_cuMemRelease, A_vMemFree, A_cuMemAddressFree,
  A_COUNT
};
static const char* kApiNames[A_COUNT] = {
    "vMemReserve", "cuMemAddressReserve", "vMemCreate", "cuMemCreate", "vMemMap", "cuMemMap",
    "cuMemSetAccess", "cuMemUnmap", "vMemRelease", "cuMemRelease", "vMemFree",
    "cuMemAddressFree"};

struct LatencyTable {
  std::vector<std::pair<int64_t, double>> rows[A_COUNT];
  void set(int api, int64_t size, double us) {
    for (auto& r : rows[api])
      if (r.first == size) { r.second = us; return; }
    rows[api].push_back({size, us});
  }
  double get(int api, int64_t size) const {
    for (auto& r : rows[api])
      if (r.first == size) return r.second;
    throw Fail(VATTN_LATENCY_CONFIG, std::string("no latency configured for (") + kApiNames[api] +
                                         ", " + std::to_string(size) + ")");
  }
  static LatencyTable table2() {
    LatencyTable t;
    const int64_t K64 = 65536, K128 = 131072, K256 = 262144, M2 = 2097152;
    t.set(A_vMemReserve, K64, 18); t.set(A_vMemReserve, K128, 17); t.set(A_vMemReserve, K256, 16);
    t.set(A_cuMemAddressReserve, M2, 2);
    t.set(A_vMemCreate, K64, 1.7); t.set(A_vMemCreate, K128, 2); t.set(A_vMemCreate, K256, 2.1);
    t.set(A_cuMemCreate, M2, 29);
    t.set(A_vMemMap, K64, 8); t.set(A_vMemMap, K128, 8.5); t.set(A_vMemMap, K256, 9);
    t.set(A_cuMemMap, M2, 2);
    t.set(A_cuMemSetAccess, M2, 38);
    t.set(A_cuMemUnmap, M2, 34);
    t.set(A_vMemRelease, K64, 2); t.set(A_vMemRelease, K128, 3); t.set(A_vMemRelease, K256, 4);
    t.set(A_cuMemRelease, M2, 23);
    t.set(A_vMemFree, K64, 35); t.set(A_vMemFree, K128, 35); t.set(A_vMemFree, K256, 35);
    t.set(A_cuMemAddressFree, M2, 1);
    return t;
  }
};

static int api_index(const char* name) {
  for (int i = 0; i < A_COUNT; ++i)
    if (std::strcmp(name, kApiNames[i]) == 0) return i;
  return -1;
}

// ------------------------------------------------------------------------------ manager
enum Phase : int64_t { INACTIVE = 0, PREFILL = 1, DECODE = 2 };

struct Slot {  // manager.py:66-75
  bool active = false;
  int64_t context_len = 0;
  int64_t mapped_groups = 0;
  Phase phase = INACTIVE;
  int64_t freed_seq = 0;
};

// alloc_reqid's ranking key (see Manager::alloc_reqid): mapped groups minus plan credits
static inline int64_t ranked(const Slot& s, int64_t credit) { return s.mapped_groups - credit; }

struct Handle {  // vmm.py:130-138 plus the real driver handle
  bool mapped = false;
  int32_t buf = -1;
  int64_t off = -1;
  CUmemGenericAllocationHandle real = 0;
};

struct BgJob {
  std::vector<int64_t> plan;
  uint32_t flags = 0;
  int64_t eager_k = -1;
  uint64_t seq = 0;
};

class Manager {
 public:
  explicit Manager(const vattn_config& c);
  ~Manager();

  // Table 3 + §6.1 API (all called from the control thread; they join the bg window first)
  int32_t alloc_reqid();
  void free_reqid(int32_t rid);
  bool step(const int64_t* seq, int32_t n, double* sync_us);
  int64_t plan_overlap(const int64_t* next, int32_t n);
  double execute_plan(const int64_t* trip, int64_t n);
  double eager_prepare(int64_t k);
  std::pair<int64_t, double> reclaim();
  std::pair<int64_t, double> reclaim_until(int64_t target);

  // background thread
  void bg_submit(const int64_t* trip, int64_t n, uint32_t flags, int64_t eager_k);
  void bg_wait(vattn_bg_result* out);
  double join_bg();                 // wait until every submitted job retired
  double join_noncommuting();       // wait for queued eager/reclaim jobs only
  bool deferral_safe(const int64_t* seq, int32_t n, int64_t eager_k) const;
  void reset_credits() { std::fill(plan_credit_.begin(), plan_credit_.end(), 0); }

  void mark_use(cudaStream_t st, bool explicit_mark = true);
  // Device-side read guard: rows each slot may be read at (backed page-groups), published to the
  // device for the decode / append kernels, which clamp to it and record a violation in a
  // host-mapped word instead of faulting the context; check_device_errors() raises it.
  void publish_rows();                          // grow to the slots' backed rows
  void shrink_rows(int64_t off);                // before unmapping the page at buffer offset off
  void check_device_errors();
  int32_t rows_of(int64_t groups) const {
    return (int32_t)std::min<int64_t>(max_context_, groups * t_ / per_buffer_token_bytes_);
  }
  int64_t mapped_rows(int32_t slot) const { return rows_of(slots_.at(slot).mapped_groups); }
  // prefill takes kv_len on the host: check it against the slot's backed rows before launching
  void check_prefill_rows(int32_t slot, int64_t kv_len) const {
    if (slot < 0 || slot >= (int32_t)slots_.size())
      throw Fail(VATTN_VALUE_ERROR, "slot " + std::to_string(slot) + " out of range");
    if (real() && kv_len > mapped_rows(slot))
      throw Fail(VATTN_VALUE_ERROR, "prefill over " + std::to_string(kv_len) + " rows of slot " +
                                        std::to_string(slot) + ", which backs " + std::to_string(mapped_rows(slot)) +
                                        " (call step() with the prompt length first)");
  }
  void begin_call() { fenced_ = false; }
  void end_call() { flush_access(); }

  // introspection
  void counters(vattn_counters* o) const;
  void slot_state(int64_t* out) const;
  void api_stats(int64_t* calls, double* ledger, int32_t* order, int32_t* n_order) const;
  int64_t buffer_mappings(int32_t b, int64_t* offs, int64_t* hids, int64_t cap) const;
  int64_t drain_events(int64_t* out, int64_t cap);
  uint64_t buffer_base(int32_t b) const;
  const std::vector<int64_t>& last_plan() const { return last_plan_; }
  CacheView layer_view(int32_t layer) const;
  void check_decode_tiling() const;
  // active slots' contexts differ by more than a quarter of the longest (decode row ordering)
  bool mixed_lengths() const {
    int64_t lo = INT64_MAX, hi = 0;
    for (const Slot& s : slots_)
      if (s.active) {
        lo = std::min(lo, s.context_len);
        hi = std::max(hi, s.context_len);
      }
    return hi > 0 && (hi - lo) * 4 > hi;
  }
  bool real() const { return backend_ == VATTN_BACKEND_CUDA; }
  int64_t max_batch() const { return (int64_t)slots_.size(); }
  int32_t hq_local() const { return hq_local_; }

  KernelState* ks = nullptr;

 private:
  // ---- shadow driver (vmm.py:150-302) ----
  double bill(const std::vector<int>& apis, int64_t count = 1);
  double unit_cost(const std::vector<int>& apis) const;
  int64_t available() const { return capacity_ - mapped_ * t_; }   // vmm.py:124-127
  int64_t free_bytes() const { return capacity_ - created_ * t_; }   // vmm.py:118-121
  int64_t new_handle_id();
  int64_t dev_create();                      // vmm.py:213-225
  double dev_precreate(int64_t count);       // vmm.py:227-239
  int64_t dev_take_precreated();             // vmm.py:245-253
  double dev_map(int32_t b, int64_t off, int64_t hid);   // vmm.py:255-283
  double dev_unmap_release(int32_t b, int64_t off);       // vmm.py:285-297
  double charged_total() const;

  // ---- real driver ----
  CUmemGenericAllocationHandle real_create();
  CUmemGenericAllocationHandle take_unattached();
  CUmemGenericAllocationHandle steal_spec();
  void real_release(CUmemGenericAllocationHandle hnd);
 public:
  void prefetch();
  std::vector<int32_t> predict_alloc(int32_t k) const;
  void prefetch_hint(const int32_t* slots, const int64_t* tokens, int32_t n);
  bool slot_ready(int32_t slot, int64_t tokens) const;
 private:
  CUmemGenericAllocationHandle steal_spec_locked(std::unique_lock<std::mutex>& lk);
  void real_map(int32_t b, int64_t off, CUmemGenericAllocationHandle hnd);
  void real_unmap(int32_t b, int64_t off);
  void flush_access();
  void fence_unmap();

  // ---- policy (manager.py) ----
  int64_t groups_required(int64_t seq) const;
  int64_t slot_offset(int64_t rid, int64_t g) const { return rid * slot_stride_ + g * t_; }
  int64_t reclaim_floor() const { return (int64_t)(reclaim_threshold_ * (double)pool_bytes_); }
  int32_t best_inactive() const;
  std::pair<int64_t, double> acquire_handle();
  double map_group(int64_t rid, int64_t g);
  double release_top_group(int64_t rid);
  std::vector<int32_t> reclaim_victims() const;
  void bg_loop();

  // config / geometry
  int32_t backend_;
  int64_t t_, pool_bytes_, capacity_;
  double reclaim_threshold_;
  int64_t eager_groups_;
  bool sliced_;
  int64_t max_context_;
  int32_t n_layers_, hkv_local_, hq_local_, head_dim_, elem_bytes_;
  int64_t buffer_count_, per_buffer_token_bytes_, groups_per_slot_, slot_stride_, buffer_size_;
  bool release_physical_, log_events_, batch_access_;
  LatencyTable lat_;
  std::vector<int> api_reserve_, api_create_, api_map_, api_release_;

  // shadow state
  int64_t created_ = 0, mapped_ = 0, precreated_ = 0, total_mapped_bytes_ = 0, next_hid_ = 0;
  std::vector<std::unordered_map<int64_t, int64_t>> buf_maps_;
  std::unordered_map<int64_t, Handle> handles_;
  int64_t calls_[A_COUNT] = {};
  double ledger_[A_COUNT] = {};
  bool ledger_seen_[A_COUNT] = {};
  std::vector<int32_t> ledger_order_;
  std::vector<int64_t> events_;
  std::vector<Slot> slots_;
  int64_t eager_slot_ = -1;
  int64_t freed_counter_ = 0;
  std::deque<int64_t> handle_cache_;  // manager.py:130 rollback leftovers
  std::vector<int64_t> last_plan_;

  double init_us_ = 0.0, init_wall_us_ = 0.0;

  // real backend state
  CUdevice cu_dev_ = 0;
  CUcontext ctx_ = nullptr;
  std::vector<CUdeviceptr> va_;
  // Physical 2 MiB handles not attached to a shadow handle (pre-created reserve + recycled),
  // and speculative mappings: pages mapped ahead of the reference's schedule by prefetch().
  // Invariant: phys_free_.size() + spec_.size() == handles the shadow considers unattached.
  std::vector<CUmemGenericAllocationHandle> phys_free_;
  std::unordered_map<int64_t, CUmemGenericAllocationHandle> spec_;   // key b*buffer_size+off
  std::deque<int64_t> spec_order_;
  int64_t prefetch_tokens_ = 0;
  int64_t prefetch_slots_ = 0, prefetch_slot_tokens_ = 0;   // speculative eager for likely-next slots
  bool lazy_unmap_ = false;
  // Physical chunks (phys_chunk_groups): chunk_ consecutive page-groups of a buffer share one
  // physical handle, mapped (cuMemMap + cuMemSetAccess over chunk_ * t_ bytes) when its first group
  // is referenced and unmapped when its last reference goes.  The per-group handles the logical
  // layer passes around (phys_free_, spec_, Handle::real) are then plain tokens.
  int64_t chunk_ = 1;
  struct Chunk {
    int32_t refs = 0;
    bool busy = false;                 // a driver call on it is in flight (ch_mu_ released)
    CUmemGenericAllocationHandle h = 0;
  };
  std::unordered_map<int64_t, Chunk> chunks_;                                        // ch_mu_
  std::unordered_map<int64_t, std::vector<CUmemGenericAllocationHandle>> ch_free_;  // by bytes
  mutable std::mutex ch_mu_;
  std::condition_variable ch_cv_;
  std::atomic<uint64_t> next_token_{0};
  int64_t ch_mapped_ = 0, ch_mapped_bytes_ = 0;
  bool chunked() const { return chunk_ > 1; }
  CUmemGenericAllocationHandle make_token() { return (1ull << 62) | ++next_token_; }
  int64_t chunk_bytes(int64_t c) const { return std::min(chunk_ * t_, buffer_size_ - c * chunk_ * t_); }
  void chunk_ref(int32_t b, int64_t off);
  void chunk_unref(int32_t b, int64_t off);
  void prop_size_create(CUmemGenericAllocationHandle* h, int64_t bytes);
  int64_t lazy_unmaps_ = 0;
  std::vector<std::pair<int32_t, int64_t>> pf_hints_;       // (slot, tokens) of queued prompts (pf_mu_)
  std::atomic<bool> prefetch_cancel_{false};   // legacy; the detached worker never blocks a join
  int64_t spec_maps_ = 0, spec_hits_ = 0, spec_steals_ = 0;
  // Detached prefetch worker: maps the speculative pages the bg thread chose, holding no state
  // but its own (pf_mu_ guards phys_free_, spec_, spec_order_ and everything pf_*), so a slow
  // or stalled driver call never blocks step / alloc / free; a control-thread map waits only
  // when it needs exactly the page in flight.
  std::thread pf_thread_;
  mutable std::mutex pf_mu_;
  std::condition_variable pf_cv_;
  std::vector<int64_t> pf_targets_;
  size_t pf_next_ = 0;
  std::unordered_set<int64_t> pf_pending_;
  int64_t pf_inflight_ = -1;
  size_t pf_reserve_ = 0;
  bool pf_stop_ = false;
  bool pf_hold_ = false;          // foreground launch window: the worker makes no driver call
 public:
  void set_foreground(bool on) {
    {
      std::lock_guard<std::mutex> lk(pf_mu_);
      pf_hold_ = on;
    }
    pf_cv_.notify_all();
  }
 private:
  int64_t pf_maps_ = 0, pf_access_ = 0, pf_errors_ = 0;
  double pf_map_us_ = 0, pf_access_us_ = 0;
  void pf_loop();
  void pf_stop();
  CUmemAllocationProp prop_{};
  CUmemAccessDesc access_{};
  std::vector<int64_t> run_begin_, run_end_;  // pending cuMemSetAccess page runs per buffer
  // Unmap fence: one "last use" event per stream that launched kernels on this cache (a reclaim
  // or trim must wait for decode on stream A and prefill on stream B alike).
  std::mutex use_mu_;
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> use_events_;
  std::vector<char> use_dirty_;                     // launches on stream i since its last record
  std::unordered_set<unsigned long long> open_captures_;   // captures with launches, no mark yet
  std::atomic<bool> use_recorded_{false};
  cudaEvent_t use_event_locked(cudaStream_t st, size_t* idx);
  bool fenced_ = false;
  // read guard (publish_rows): device copy of every slot's readable rows, its pinned staging
  // buffer and host shadow, a private stream for the copy, and the host-mapped violation words
  // [flag, slot, requested rows, readable rows]
  std::mutex pub_mu_;
  std::mutex slot_mu_;   // free_reqid's writes vs the prefetch job's slot snapshot
  int32_t* d_rows_ = nullptr;
  int32_t* h_rows_ = nullptr;
  std::vector<int32_t> pub_rows_;
  cudaStream_t pub_stream_ = nullptr;
  uint32_t* h_err_ = nullptr;
  uint32_t* d_err_ = nullptr;
  // measured real-driver statistics
  int64_t real_maps_ = 0, real_unmaps_ = 0, real_access_ = 0, real_creates_ = 0,
          real_releases_ = 0;
  double real_map_us_ = 0, real_unmap_us_ = 0, real_create_us_ = 0, real_access_us_ = 0;

  // background thread
  std::thread bg_thread_;
  std::mutex bg_mu_;
  std::condition_variable bg_cv_;
  std::deque<BgJob> bg_queue_;
  uint64_t bg_submitted_ = 0, bg_completed_ = 0, bg_last_noncommuting_ = 0;
  bool bg_stop_ = false;
  vattn_bg_result bg_res_{};        // accumulated since the last bg_wait
  vattn_status bg_status_ = VATTN_OK;
  std::string bg_error_;
  // groups mapped per slot by a plan executed ahead of the reference's position (credit mode)
  std::vector<int64_t> plan_credit_;
  bool credit_mode_ = false;
};

// ---- construction (manager.py:85-130) --------------------------------------------------
Manager::Manager(const vattn_config& c) {
  if (c.reclaim_threshold < 0.0 || c.reclaim_threshold > 1.0)
    throw Fail(VATTN_VALUE_ERROR, "reclaim_threshold must be in [0, 1]");
  if (c.pre_create_fraction < 0.0 || c.pre_create_fraction > 1.0)
    throw Fail(VATTN_VALUE_ERROR, "pre_create_fraction must be in [0, 1]");
  if (c.eager_groups < 0) throw Fail(VATTN_VALUE_ERROR, "eager_groups must be >= 0");
  if (c.n_layers < 1 || c.kv_heads_total < 1 || c.head_dim < 1 || c.bytes_per_elem < 1 ||
      c.tp_degree < 1)
    throw Fail(VATTN_VALUE_ERROR, "geometry fields must be >= 1");
  if (c.kv_heads_total % c.tp_degree != 0)
    throw Fail(VATTN_VALUE_ERROR, "kv_heads_total must be divisible by tp_degree");
  if (c.max_context < 0) throw Fail(VATTN_VALUE_ERROR, "max_context must be >= 0");
  if (c.max_batch < 1) throw Fail(VATTN_VALUE_ERROR, "geometry.max_batch must be >= 1 to serve requests");
  if (c.page_group_size < 1) throw Fail(VATTN_VALUE_ERROR, "page_group_size must be >= 1");
  if (c.pool_bytes < 0) throw Fail(VATTN_VALUE_ERROR, "capacity must be >= 0");

  backend_ = c.backend;
  t_ = c.page_group_size;
  pool_bytes_ = capacity_ = c.pool_bytes;
  reclaim_threshold_ = c.reclaim_threshold;
  eager_groups_ = c.eager_groups;
  sliced_ = c.sliced != 0;
  max_context_ = c.max_context;
  n_layers_ = c.n_layers;
  hkv_local_ = c.kv_heads_total / c.tp_degree;
  int32_t hq_total = c.n_q_heads_total > 0 ? c.n_q_heads_total : c.kv_heads_total;
  if (hq_total % c.tp_degree != 0 || hq_total % c.kv_heads_total != 0)
    throw Fail(VATTN_VALUE_ERROR, "n_q_heads_total must be a multiple of kv_heads_total and tp");
  hq_local_ = hq_total / c.tp_degree;
  head_dim_ = c.head_dim;
  elem_bytes_ = c.bytes_per_elem;
  release_physical_ = c.release_physical != 0;
  log_events_ = c.log_events != 0;
  batch_access_ = c.batch_set_access != 0;
  prefetch_tokens_ = std::max<int64_t>(0, c.prefetch_tokens);
  prefetch_slots_ = std::max<int64_t>(0, c.prefetch_slots);
  prefetch_slot_tokens_ = std::max<int64_t>(0, c.prefetch_slot_tokens);
  lazy_unmap_ = c.lazy_unmap != 0 && c.release_physical == 0;
  chunk_ = std::max<int64_t>(1, c.phys_chunk_groups);

  lat_ = LatencyTable::table2();
  if (c.latency && c.n_latency > 0) {
    lat_ = LatencyTable{};
    for (int i = 0; i < c.n_latency; ++i) {
      int a = api_index(c.latency[i].api);
      if (a < 0) continue;  // unknown names are kept out of the model, as LatencyModel does
      if (c.latency[i].us < 0) throw Fail(VATTN_VALUE_ERROR, "negative latency");
      lat_.set(a, c.latency[i].page_group_bytes, c.latency[i].us);
    }
  }
  const bool large = t_ == 2097152;  // vmm.py:178-182
  api_reserve_ = {large ? A_cuMemAddressReserve : A_vMemReserve};
  api_create_ = {large ? A_cuMemCreate : A_vMemCreate};
  if (large) api_map_ = {A_cuMemMap, A_cuMemSetAccess}; else api_map_ = {A_vMemMap};
  if (large) api_release_ = {A_cuMemUnmap, A_cuMemRelease}; else api_release_ = {A_vMemRelease};

  const int64_t token_layer_bytes = (int64_t)hkv_local_ * head_dim_ * elem_bytes_;
  if (sliced_) {  // manager.py:93-99
    buffer_count_ = 2;
    per_buffer_token_bytes_ = (int64_t)n_layers_ * token_layer_bytes;
  } else {
    buffer_count_ = 2 * (int64_t)n_layers_;
    per_buffer_token_bytes_ = token_layer_bytes;
  }
  if (t_ < per_buffer_token_bytes_)
    throw Fail(VATTN_VALUE_ERROR, "page-group size smaller than one token's cache in this layout");
  if (pool_bytes_ < buffer_count_ * t_)
    throw Fail(VATTN_VALUE_ERROR, "pool cannot back one page-group in each buffer");
  groups_per_slot_ = (max_context_ * per_buffer_token_bytes_ + t_ - 1) / t_;  // :111-115
  slot_stride_ = groups_per_slot_ * t_;
  buffer_size_ = c.max_batch * slot_stride_;

  const double t0 = now_us();
  if (real()) {
    if (t_ != 2097152)
      throw Fail(VATTN_UNSUPPORTED, "the stock-driver backend maps 2 MiB page-groups only");
    const Driver& d = driver();
    check_rt(cudaSetDevice(c.device), "cudaSetDevice");
    check_rt(cudaFree(nullptr), "cudaFree(0) context init");
    check_cu(d.DeviceGet(&cu_dev_, c.device), "cuDeviceGet");
    check_cu(d.CtxGetCurrent(&ctx_), "cuCtxGetCurrent");
    if (!ctx_) {
      check_cu(d.DevicePrimaryCtxRetain(&ctx_, cu_dev_), "cuDevicePrimaryCtxRetain");
      check_cu(d.CtxSetCurrent(ctx_), "cuCtxSetCurrent");
    }
    prop_.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop_.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop_.location.id = c.device;
    size_t gran = 0;
    check_cu(d.MemGetAllocationGranularity(&gran, &prop_, CU_MEM_ALLOC_GRANULARITY_MINIMUM),
             "cuMemGetAllocationGranularity");
    if ((int64_t)gran > t_ || t_ % (int64_t)gran != 0)
      throw Fail(VATTN_UNSUPPORTED, "page-group size is not a multiple of the driver granularity");
    access_.location = prop_.location;
    access_.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }

  buf_maps_.resize(buffer_count_);
  run_begin_.assign(buffer_count_, -1);
  run_end_.assign(buffer_count_, -1);
  for (int64_t i = 0; i < buffer_count_; ++i) {  // :119-122 — reserve(max_batch * slot_stride)
    if (buffer_size_ % t_ != 0) throw Fail(VATTN_ALIGNMENT_ERROR, "buffer size misaligned");
    if (real()) {
      CUdeviceptr p = 0;
      check_cu(driver().MemAddressReserve(&p, (size_t)buffer_size_, (size_t)t_, 0, 0),
               "cuMemAddressReserve");
      va_.push_back(p);
    }
    bill(api_reserve_);
  }
  init_us_ = 0.0;
  init_us_ += charged_total();
  const int64_t pre = (int64_t)(c.pre_create_fraction * (double)c.pool_bytes) / t_;  // :124-125
  init_us_ += dev_precreate(pre);
  slots_.resize(c.max_batch);
  plan_credit_.assign(c.max_batch, 0);
  // counters_peek walks ledger_order_ while a background job may append to it: never reallocate
  ledger_order_.reserve(A_COUNT);
  if (real()) {
    const size_t n = (size_t)c.max_batch;
    check_rt(cudaMalloc(reinterpret_cast<void**>(&d_rows_), n * 4), "cudaMalloc(read guard)");
    check_rt(cudaMemset(d_rows_, 0, n * 4), "cudaMemset(read guard)");
    check_rt(cudaHostAlloc(reinterpret_cast<void**>(&h_rows_), n * 4, cudaHostAllocDefault), "cudaHostAlloc(read guard)");
    check_rt(cudaStreamCreateWithFlags(&pub_stream_, cudaStreamNonBlocking), "cudaStreamCreate(read guard)");
    check_rt(cudaHostAlloc(reinterpret_cast<void**>(&h_err_), 64, cudaHostAllocMapped), "cudaHostAlloc(error words)");
    std::memset(h_err_, 0, 64);
    check_rt(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_err_), h_err_, 0), "cudaHostGetDevicePointer");
    pub_rows_.assign(n, 0);
  }
  init_wall_us_ = now_us() - t0;

  bg_thread_ = std::thread([this] { bg_loop(); });
  if (real()) pf_thread_ = std::thread([this] { pf_loop(); });
}

void Manager::pf_stop() {
  {
    std::lock_guard<std::mutex> lk(pf_mu_);
    pf_stop_ = true;
  }
  pf_cv_.notify_all();
  if (pf_thread_.joinable()) pf_thread_.join();
}

void Manager::pf_loop() {
  const Driver& d = driver();
  if (d.CtxSetCurrent(ctx_) != CUDA_SUCCESS) return;
  std::unique_lock<std::mutex> lk(pf_mu_);
  for (;;) {
    // cuMemMap/cuMemSetAccess take the kernel driver's lock for up to milliseconds; while the
    // caller is launching an iteration's kernels the worker holds back so launches never queue
    // behind it
    pf_cv_.wait(lk, [&] { return pf_stop_ || (!pf_hold_ && pf_next_ < pf_targets_.size()); });
    if (pf_stop_) return;
    const int64_t key = pf_targets_[pf_next_++];
    if (!pf_pending_.erase(key) || spec_.count(key)) continue;   // claimed by a logical map meanwhile
    if (phys_free_.size() <= pf_reserve_) {                       // keep handles for the reference path
      pf_next_ = pf_targets_.size();
      pf_pending_.clear();
      continue;
    }
    const auto h = phys_free_.back();
    phys_free_.pop_back();
    pf_inflight_ = key;
    lk.unlock();
    const int64_t b = key / buffer_size_, off = key % buffer_size_;
    const double t0 = now_us();
    bool ok;
    double t1, t2;
    if (chunked()) {           // one reference on the page's chunk: a driver call only if unmapped
      try {
        chunk_ref((int32_t)b, off);
        ok = true;
      } catch (...) {
        ok = false;
      }
      t1 = t2 = now_us();
    } else {
      ok = d.MemMap(va_[b] + off, (size_t)t_, 0, h, 0) == CUDA_SUCCESS;
      t1 = now_us();
      if (ok && d.MemSetAccess(va_[b] + off, (size_t)t_, &access_, 1) != CUDA_SUCCESS) {
        d.MemUnmap(va_[b] + off, (size_t)t_);
        ok = false;
      }
      t2 = now_us();
    }
    lk.lock();
    pf_inflight_ = -1;
    pf_map_us_ += t1 - t0;
    pf_access_us_ += t2 - t1;
    if (ok) {
      pf_maps_ += 1;
      pf_access_ += 1;
      spec_[key] = h;
      spec_order_.push_back(key);
      spec_maps_ += 1;
    } else {
      pf_errors_ += 1;
      phys_free_.push_back(h);
    }
    pf_cv_.notify_all();
  }
}

Manager::~Manager() {
  {
    std::unique_lock<std::mutex> lk(bg_mu_);
    bg_cv_.wait(lk, [&] { return bg_completed_ == bg_submitted_; });
    bg_stop_ = true;
  }
  bg_cv_.notify_all();
  if (bg_thread_.joinable()) bg_thread_.join();
  pf_stop();
  if (!real()) return;
  const Driver& d = driver();
  d.CtxSetCurrent(ctx_);
  cudaDeviceSynchronize();
  if (chunked()) {
    const int64_t per_buf = buffer_size_ / t_ + 1;
    for (auto& kv : chunks_)
      if (kv.second.h) {
        const int64_t b = kv.first / per_buf, c = kv.first % per_buf;
        d.MemUnmap(va_[b] + (CUdeviceptr)(c * chunk_ * t_), (size_t)chunk_bytes(c));
        d.MemRelease(kv.second.h);
      }
    for (auto& fl : ch_free_)
      for (auto h : fl.second) d.MemRelease(h);
    for (size_t b = 0; b < va_.size(); ++b) d.MemAddressFree(va_[b], (size_t)buffer_size_);
    for (auto& se : use_events_) cudaEventDestroy(se.second);
    if (d_rows_) cudaFree(d_rows_);
    if (h_rows_) cudaFreeHost(h_rows_);
    if (h_err_) cudaFreeHost(h_err_);
    if (pub_stream_) cudaStreamDestroy(pub_stream_);
    return;
  }
  for (int32_t b = 0; b < (int32_t)buf_maps_.size(); ++b)
    for (auto& kv : buf_maps_[b]) d.MemUnmap(va_[b] + kv.first, (size_t)t_);
  for (auto& kv : handles_)
    if (kv.second.real) d.MemRelease(kv.second.real);
  for (auto& kv : spec_) {
    const int64_t b = kv.first / buffer_size_, off = kv.first % buffer_size_;
    d.MemUnmap(va_[b] + off, (size_t)t_);
    d.MemRelease(kv.second);
  }
  for (auto h : phys_free_) d.MemRelease(h);
  for (size_t b = 0; b < va_.size(); ++b) d.MemAddressFree(va_[b], (size_t)buffer_size_);
  for (auto& se : use_events_) cudaEventDestroy(se.second);
  if (d_rows_) cudaFree(d_rows_);
  if (h_rows_) cudaFreeHost(h_rows_);
  if (h_err_) cudaFreeHost(h_err_);
  if (pub_stream_) cudaStreamDestroy(pub_stream_);
}

// ---- shadow driver ------------------------------------------------------------------------
// vmm.py:186-195: each API charged count times; a composite charge sums from integer 0.
double Manager::bill(const std::vector<int>& apis, int64_t count) {
  PySum total;
  for (int a : apis) {
    const double us = lat_.get(a, t_) * (double)count;
    if (!ledger_seen_[a]) { ledger_seen_[a] = true; ledger_order_.push_back(a); }
    ledger_[a] = ledger_[a] + us;
    calls_[a] += count;
    total.add(us);
  }
  return total.value();
}

double Manager::unit_cost(const std::vector<int>& apis) const {  // manager.py:201-203
  PySum total;
  for (int a : apis) total.add(lat_.get(a, t_));
  return total.value();
}

double Manager::charged_total() const {  // vmm.py:301-302 sum(ledger_us.values())
  PySum s;
  for (int32_t a : ledger_order_) s.add(ledger_[a]);
  return s.value();
}

int64_t Manager::new_handle_id() {
  const int64_t id = next_hid_++;
  handles_.emplace(id, Handle{});
  return id;
}

int64_t Manager::dev_create() {
  if (free_bytes() < t_) throw Fail(VATTN_POOL_EXHAUSTED, "pool exhausted");
  CUmemGenericAllocationHandle r = real() ? real_create() : 0;
  const int64_t id = new_handle_id();
  handles_[id].real = r;
  created_ += 1;
  bill(api_create_);
  return id;
}

double Manager::dev_precreate(int64_t count) {
  if (count < 0) throw Fail(VATTN_VALUE_ERROR, "count must be >= 0");
  if (free_bytes() < count * t_) throw Fail(VATTN_POOL_EXHAUSTED, "cannot pre-create page-groups");
  if (real() && chunked()) {
    // tokens for the logical layer; full-size chunk handles for the physical one
    std::lock_guard<std::mutex> lk(pf_mu_);
    for (int64_t i = 0; i < count; ++i) phys_free_.push_back(make_token());
    const int64_t n = (count + chunk_ - 1) / chunk_;
    std::lock_guard<std::mutex> lc(ch_mu_);
    for (int64_t i = 0; i < n; ++i) {
      CUmemGenericAllocationHandle h = 0;
      const double t0 = now_us();
      prop_size_create(&h, chunk_ * t_);
      real_create_us_ += now_us() - t0;
      real_creates_ += 1;
      ch_free_[chunk_ * t_].push_back(h);
    }
  } else if (real()) {
    phys_free_.reserve(phys_free_.size() + (size_t)count);
    for (int64_t i = 0; i < count; ++i) {
      CUmemGenericAllocationHandle h = 0;
      const double t0 = now_us();
      check_cu(driver().MemCreate(&h, (size_t)t_, &prop_, 0), "cuMemCreate");
      real_create_us_ += now_us() - t0;
      real_creates_ += 1;
      std::lock_guard<std::mutex> lk(pf_mu_);
      phys_free_.push_back(h);
    }
  }
  created_ += count;
  precreated_ += count;
  return count ? bill(api_create_, count) : 0.0;
}

int64_t Manager::dev_take_precreated() {
  if (precreated_ < 1) throw Fail(VATTN_POOL_EXHAUSTED, "no pre-created handles available");
  precreated_ -= 1;
  const int64_t id = new_handle_id();
  if (real()) handles_[id].real = take_unattached();
  return id;
}

double Manager::dev_map(int32_t b, int64_t off, int64_t hid) {
  auto it = handles_.find(hid);
  if (it == handles_.end()) throw Fail(VATTN_MAPPING_ERROR, "handle released");
  Handle& h = it->second;
  if (h.mapped) throw Fail(VATTN_MAPPING_ERROR, "handle already mapped");
  if (off % t_ != 0) throw Fail(VATTN_ALIGNMENT_ERROR, "offset not aligned");
  if (off < 0 || off + t_ > buffer_size_) throw Fail(VATTN_MAPPING_ERROR, "offset out of range");
  if (buf_maps_[b].count(off)) throw Fail(VATTN_MAPPING_ERROR, "offset already backed");
  if (real()) {
    const int64_t key = (int64_t)b * buffer_size_ + off;
    std::unique_lock<std::mutex> lk(pf_mu_);
    pf_pending_.erase(key);                                     // the worker must not map it now
    pf_cv_.wait(lk, [&] { return pf_inflight_ != key; });       // unless it already is
    auto sp = spec_.find(key);
    if (sp != spec_.end()) {            // prefetched: already mapped and accessible, adopt it
      if (h.real) phys_free_.push_back(h.real);
      h.real = sp->second;
      spec_.erase(sp);
      spec_hits_ += 1;
    } else {
      if (!h.real) h.real = steal_spec_locked(lk);
      lk.unlock();
      real_map(b, off, h.real);
    }
  }
  h.mapped = true;
  h.buf = b;
  h.off = off;
  buf_maps_[b][off] = hid;
  mapped_ += 1;
  total_mapped_bytes_ += t_;
  if (log_events_) { events_.push_back(0); events_.push_back(b); events_.push_back(off); }
  return bill(api_map_);
}

double Manager::dev_unmap_release(int32_t b, int64_t off) {
  auto it = buf_maps_[b].find(off);
  if (it == buf_maps_[b].end()) throw Fail(VATTN_INVALID_FREE, "no mapping at offset");
  const int64_t hid = it->second;
  Handle h = handles_[hid];
  if (real()) {
    if (lazy_unmap_) {     // keep it mapped as a speculative page: no driver call now
      std::lock_guard<std::mutex> lk(pf_mu_);
      const int64_t key = (int64_t)b * buffer_size_ + off;
      spec_[key] = h.real;
      spec_order_.push_back(key);
      lazy_unmaps_ += 1;
    } else {
      real_unmap(b, off);
      real_release(h.real);
    }
  }
  buf_maps_[b].erase(it);
  handles_.erase(hid);
  mapped_ -= 1;
  created_ -= 1;  // capacity returns to the pool, not the pre-created reserve (vmm.py:295-296)
  if (log_events_) { events_.push_back(1); events_.push_back(b); events_.push_back(off); }
  return bill(api_release_);
}

// ---- real driver ----------------------------------------------------------------------------
// An unattached physical handle for a shadow handle; 0 = "all of them are holding speculative
// pages": resolved in dev_map (adopt the page if it is the one being mapped, else steal one).
CUmemGenericAllocationHandle Manager::take_unattached() {
  std::lock_guard<std::mutex> lk(pf_mu_);
  if (!phys_free_.empty()) {
    auto h = phys_free_.back();
    phys_free_.pop_back();
    return h;
  }
  if (spec_.empty() && pf_inflight_ < 0) throw Fail(VATTN_BAD_STATE, "physical pool accounting error");
  return 0;
}

CUmemGenericAllocationHandle Manager::steal_spec() {
  std::unique_lock<std::mutex> lk(pf_mu_);
  return steal_spec_locked(lk);
}

// Take a speculative page's handle back for the reference path (unmapping it); waits for the
// worker's page in flight when it holds the last one.  Called and returns with `lk` held.
CUmemGenericAllocationHandle Manager::steal_spec_locked(std::unique_lock<std::mutex>& lk) {
  for (;;) {
    if (!phys_free_.empty()) {        // a failed prefetch may have returned one meanwhile
      auto h = phys_free_.back();
      phys_free_.pop_back();
      return h;
    }
    while (!spec_order_.empty()) {
      const int64_t key = spec_order_.front();
      spec_order_.pop_front();
      auto it = spec_.find(key);
      if (it == spec_.end()) continue;   // already adopted
      const auto h = it->second;
      spec_.erase(it);
      spec_steals_ += 1;
      lk.unlock();
      real_unmap((int32_t)(key / buffer_size_), key % buffer_size_);
      lk.lock();
      return h;
    }
    if (pf_inflight_ < 0) throw Fail(VATTN_BAD_STATE, "no speculative page to steal");
    pf_cv_.wait(lk, [&] { return pf_inflight_ < 0; });
  }
}

// Physical prefetch (B200 addition, not in the reference): map the pages each active slot will
// need within `prefetch_tokens_` more tokens ahead of the reference's schedule, from handles the
// shadow considers unattached.  Logical state (slots, counters, events) is untouched; when the
// reference logic maps such a page later it adopts the mapping with no driver call.  Keeps one
// group's worth of handles free so the reference path rarely has to steal.
std::vector<int32_t> Manager::predict_alloc(int32_t k) const {
  std::vector<int32_t> out;
  std::vector<char> taken(slots_.size(), 0);
  if (k > 0 && eager_slot_ >= 0 && !slots_[eager_slot_].active) {
    out.push_back((int32_t)eager_slot_);
    taken[eager_slot_] = 1;
  }
  while ((int32_t)out.size() < k) {
    int32_t rid = -1;
    for (int32_t r = 0; r < (int32_t)slots_.size(); ++r) {
      if (slots_[r].active || taken[r]) continue;
      if (rid < 0 || ranked(slots_[r], plan_credit_[r]) > ranked(slots_[rid], plan_credit_[rid])) rid = r;
    }
    if (rid < 0) break;
    out.push_back(rid);
    taken[rid] = 1;
  }
  return out;
}

void Manager::prefetch_hint(const int32_t* slots, const int64_t* tokens, int32_t n) {
  std::lock_guard<std::mutex> lk(pf_mu_);
  pf_hints_.clear();
  for (int32_t i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= (int32_t)slots_.size()) throw Fail(VATTN_VALUE_ERROR, "hint slot out of range");
    if (tokens[i] < 0 || tokens[i] > max_context_) throw Fail(VATTN_VALUE_ERROR, "hint tokens out of range");
    pf_hints_.emplace_back(slots[i], tokens[i]);
  }
}

bool Manager::slot_ready(int32_t slot, int64_t tokens) const {
  if (slot < 0 || slot >= (int32_t)slots_.size()) throw Fail(VATTN_VALUE_ERROR, "slot out of range");
  const int64_t need = std::min(groups_required(tokens), groups_per_slot_);
  std::lock_guard<std::mutex> lk(pf_mu_);
  for (int64_t g = 0; g < need; ++g) {
    const int64_t off = slot_offset(slot, g);
    for (int64_t b = 0; b < buffer_count_; ++b)
      if (!buf_maps_[b].count(off) && !(real() && spec_.count(b * buffer_size_ + off))) return false;
  }
  return true;
}

void Manager::prefetch() {
  Nvtx nv("vattn.prefetch");
  if (!real()) return;
  // free_reqid may run concurrently (it does not join prefetch jobs): work on a snapshot of the
  // slot table taken under slot_mu_ (ADVICE r1 core.cpp:1554)
  std::vector<Slot> slots;
  int32_t eager_slot;
  {
    std::lock_guard<std::mutex> lk(slot_mu_);
    slots = slots_;
    eager_slot = eager_slot_;
  }
  // Runs inside a bg window (state owned): choose the pages, hand them to the worker, return.
  // (urgency, key): pages are mapped soonest-needed first — decode growth by the tokens left
  // before the row reaches the page, then the speculative-eager slots in alloc_reqid order
  std::vector<std::pair<int64_t, int64_t>> targets;
  const int64_t tokens_per_group = t_ / per_buffer_token_bytes_;
  auto spec_range = [&](int32_t r, int64_t g0, int64_t g1, int64_t urgency0, int64_t ctx) {
    for (int64_t g = g0; g < g1; ++g) {
      const int64_t off = slot_offset(r, g);
      const int64_t urgency = urgency0 + (ctx >= 0 ? g * tokens_per_group - ctx : g);
      for (int64_t b = 0; b < buffer_count_; ++b)
        if (!buf_maps_[b].count(off)) targets.emplace_back(urgency, b * buffer_size_ + off);
    }
  };
  // 1. decode growth of active slots within prefetch_tokens_ more tokens
  if (prefetch_tokens_ > 0)
    for (int32_t r = 0; r < (int32_t)slots.size(); ++r) {
      const Slot& s = slots[r];
      if (!s.active) continue;
      spec_range(r, s.mapped_groups, std::min(groups_required(s.context_len + prefetch_tokens_), groups_per_slot_),
                 0, s.context_len);
    }
  // 2. speculative eager: the slots alloc_reqid would hand out next (eager slot first, then by
  //    (mapped_groups, -req_id), manager.py:166-174) up to prefetch_slot_tokens_ of prompt
  if (prefetch_slots_ > 0 && prefetch_slot_tokens_ > 0) {
    std::vector<int32_t> cand;
    for (int32_t r = 0; r < (int32_t)slots.size(); ++r)
      if (!slots[r].active) cand.push_back(r);
    std::stable_sort(cand.begin(), cand.end(), [&](int32_t a, int32_t b) {
      const bool ea = a == eager_slot, eb = b == eager_slot;
      if (ea != eb) return ea;
      return slots[a].mapped_groups > slots[b].mapped_groups;
    });
    const int64_t target = std::min(groups_required(prefetch_slot_tokens_), groups_per_slot_);
    for (size_t i = 0; i < cand.size() && (int64_t)i < prefetch_slots_; ++i)
      spec_range(cand[i], slots[cand[i]].mapped_groups, target, (int64_t)(1 + i) << 40, -1);
  }
  // 3. prompts queued for admission, at the slots they are predicted to get (after growth)
  std::vector<std::pair<int32_t, int64_t>> hints;
  {
    std::lock_guard<std::mutex> lk(pf_mu_);
    hints = pf_hints_;
  }
  for (size_t i = 0; i < hints.size(); ++i) {
    const auto& hs = hints[i];
    if (slots[hs.first].active) continue;
    spec_range(hs.first, 0, std::min(groups_required(hs.second), groups_per_slot_), ((int64_t)1 << 38) + ((int64_t)i << 20), -1);
  }
  std::stable_sort(targets.begin(), targets.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  {
    std::lock_guard<std::mutex> lk(pf_mu_);
    pf_reserve_ = (size_t)(2 * buffer_count_);   // one group's worth of handles stays free
    pf_targets_.clear();
    pf_pending_.clear();
    for (const auto& t : targets)
      if (!spec_.count(t.second) && t.second != pf_inflight_ && pf_pending_.insert(t.second).second)
        pf_targets_.push_back(t.second);
    pf_next_ = 0;
  }
  pf_cv_.notify_all();
}

CUmemGenericAllocationHandle Manager::real_create() {
  bool none_unattached;
  {
    std::lock_guard<std::mutex> lk(pf_mu_);
    none_unattached = phys_free_.empty() && spec_.empty() && pf_inflight_ < 0;
  }
  if (!none_unattached) return take_unattached();
  if (chunked()) return make_token();
  CUmemGenericAllocationHandle h = 0;
  const double t0 = now_us();
  check_cu(driver().MemCreate(&h, (size_t)t_, &prop_, 0), "cuMemCreate");
  real_create_us_ += now_us() - t0;
  real_creates_ += 1;
  return h;
}

void Manager::real_release(CUmemGenericAllocationHandle h) {
  if (chunked()) {                 // a token: the physical chunk is released in chunk_unref
    if (!release_physical_) {
      std::lock_guard<std::mutex> lk(pf_mu_);
      phys_free_.push_back(h);
    }
    return;
  }
  if (!release_physical_) {
    std::lock_guard<std::mutex> lk(pf_mu_);
    phys_free_.push_back(h);
    return;
  }
  check_cu(driver().MemRelease(h), "cuMemRelease");
  real_releases_ += 1;
}

void Manager::real_map(int32_t b, int64_t off, CUmemGenericAllocationHandle h) {
  if (chunked()) {
    chunk_ref(b, off);
    return;
  }
  const Driver& d = driver();
  const double t0 = now_us();
  check_cu(d.MemMap(va_[b] + off, (size_t)t_, 0, h, 0), "cuMemMap");
  real_map_us_ += now_us() - t0;
  real_maps_ += 1;
  if (!batch_access_) {
    const double t1 = now_us();
    check_cu(d.MemSetAccess(va_[b] + off, (size_t)t_, &access_, 1), "cuMemSetAccess");
    real_access_us_ += now_us() - t1;
    real_access_ += 1;
    return;
  }
  // coalesce contiguous pages of the same buffer into one cuMemSetAccess call
  if (run_begin_[b] >= 0 && run_end_[b] == off) { run_end_[b] = off + t_; return; }
  if (run_begin_[b] >= 0) {
    const double t1 = now_us();
    check_cu(d.MemSetAccess(va_[b] + run_begin_[b], (size_t)(run_end_[b] - run_begin_[b]), &access_, 1),
             "cuMemSetAccess");
    real_access_us_ += now_us() - t1;
    real_access_ += 1;
  }
  run_begin_[b] = off;
  run_end_[b] = off + t_;
}

void Manager::flush_access() {
  if (!real() || !batch_access_) return;
  const Driver& d = driver();
  for (size_t b = 0; b < run_begin_.size(); ++b) {
    if (run_begin_[b] < 0) continue;
    const double t1 = now_us();
    check_cu(d.MemSetAccess(va_[b] + run_begin_[b], (size_t)(run_end_[b] - run_begin_[b]), &access_, 1),
             "cuMemSetAccess");
    real_access_us_ += now_us() - t1;
    real_access_ += 1;
    run_begin_[b] = run_end_[b] = -1;
  }
}

void Manager::fence_unmap() {
  Nvtx nv("vattn.unmap_fence");
  // Never unmap a page that queued kernels may still read (SURVEY §7 hard part 3).
  if (fenced_) return;
  flush_access();
  if (use_recorded_) {
    // Launches only flag their stream (a per-launch event record would sit between consecutive
    // kernels and cancel their programmatic dependent launch); the record happens here, so it
    // covers every kernel queued on the stream so far.  A graph captured without a closing
    // mark_use may be replayed on any stream: then only a device-wide sync is safe.
    std::vector<cudaEvent_t> evs;
    bool device_sync = false;
    {
      std::lock_guard<std::mutex> lk(use_mu_);
      device_sync = !open_captures_.empty();
      for (size_t i = 0; i < use_events_.size(); ++i) {
        if (use_dirty_[i]) {
          cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
          if (cudaStreamIsCapturing(use_events_[i].first, &cs) != cudaSuccess) {
            // the stream was destroyed after its launches (its work may still run): sync all
            cudaGetLastError();
            device_sync = true;
            use_dirty_[i] = 0;
            continue;
          }
          if (cs == cudaStreamCaptureStatusNone) {
            check_rt(cudaEventRecord(use_events_[i].second, use_events_[i].first), "cudaEventRecord(fence)");
            use_dirty_[i] = 0;
          } else {
            device_sync = true;      // its earlier eager work cannot be marked now
          }
        }
        evs.push_back(use_events_[i].second);
      }
    }
    if (device_sync) check_rt(cudaDeviceSynchronize(), "cudaDeviceSynchronize(unmap fence)");
    for (cudaEvent_t e : evs) check_rt(cudaEventSynchronize(e), "cudaEventSynchronize(unmap fence)");
  }
  fenced_ = true;
}

void Manager::real_unmap(int32_t b, int64_t off) {
  if (chunked()) {
    // the read guard shrinks now, so kernels still queued on the old row count must finish
    // first even if the chunk stays mapped (found by test_gpu_unmap_fence [eager-4])
    fence_unmap();
    shrink_rows(off);
    chunk_unref(b, off);        // unmaps only when the chunk's last group goes
    return;
  }
  fence_unmap();
  shrink_rows(off);
  const double t0 = now_us();
  check_cu(driver().MemUnmap(va_[b] + off, (size_t)t_), "cuMemUnmap");
  real_unmap_us_ += now_us() - t0;
  real_unmaps_ += 1;
}

void Manager::prop_size_create(CUmemGenericAllocationHandle* h, int64_t bytes) {
  check_cu(driver().MemCreate(h, (size_t)bytes, &prop_, 0), "cuMemCreate(chunk)");
}

// Reference one page-group of chunk (b, off / (chunk_ * t_)); the first reference maps the chunk.
// Driver calls run with ch_mu_ released (the chunk is marked busy), so a concurrent reference to
// another chunk never waits behind them.
void Manager::chunk_ref(int32_t b, int64_t off) {
  const int64_t c = off / (chunk_ * t_);
  const int64_t key = (int64_t)b * (buffer_size_ / t_ + 1) + c;
  std::unique_lock<std::mutex> lk(ch_mu_);
  Chunk& ch = chunks_[key];                  // node-based map: the reference stays valid
  ch_cv_.wait(lk, [&] { return !ch.busy; });
  ch.refs += 1;
  if (ch.refs > 1) return;
  const int64_t bytes = chunk_bytes(c);
  CUmemGenericAllocationHandle h = 0;
  auto& fl = ch_free_[bytes];
  if (!fl.empty()) {
    h = fl.back();
    fl.pop_back();
  }
  ch.busy = true;
  lk.unlock();
  const Driver& d = driver();
  CUresult e = CUDA_SUCCESS;
  double t_create = 0, t_map = 0, t_acc = 0;
  const bool fresh = h == 0;              // no recycled handle of this size: create one
  const double t0 = now_us();
  if (fresh) e = d.MemCreate(&h, (size_t)bytes, &prop_, 0);
  const double t1 = now_us();
  const CUdeviceptr va = va_[b] + (CUdeviceptr)(c * chunk_ * t_);
  bool mapped = false;
  if (e == CUDA_SUCCESS) {
    e = d.MemMap(va, (size_t)bytes, 0, h, 0);
    mapped = e == CUDA_SUCCESS;
  }
  const double t2 = now_us();
  if (e == CUDA_SUCCESS) e = d.MemSetAccess(va, (size_t)bytes, &access_, 1);
  const double t3 = now_us();
  if (e != CUDA_SUCCESS && mapped) d.MemUnmap(va, (size_t)bytes);
  t_create = t1 - t0;
  t_map = t2 - t1;
  t_acc = t3 - t2;
  lk.lock();
  ch.busy = false;
  if (e != CUDA_SUCCESS) {
    ch.refs -= 1;
    if (h) ch_free_[bytes].push_back(h);
    ch_cv_.notify_all();
    lk.unlock();
    check_cu(e, "cuMemCreate/cuMemMap/cuMemSetAccess(chunk)");
  }
  ch.h = h;
  if (fresh) {
    real_create_us_ += t_create;
    real_creates_ += 1;
  }
  real_map_us_ += t_map;
  real_maps_ += 1;
  real_access_us_ += t_acc;
  real_access_ += 1;
  ch_mapped_ += 1;
  ch_mapped_bytes_ += bytes;
  ch_cv_.notify_all();
}

void Manager::chunk_unref(int32_t b, int64_t off) {
  const int64_t c = off / (chunk_ * t_);
  const int64_t key = (int64_t)b * (buffer_size_ / t_ + 1) + c;
  std::unique_lock<std::mutex> lk(ch_mu_);
  auto it = chunks_.find(key);
  if (it == chunks_.end() || it->second.refs < 1) throw Fail(VATTN_BAD_STATE, "chunk reference count underflow");
  Chunk& ch = it->second;
  ch_cv_.wait(lk, [&] { return !ch.busy; });
  ch.refs -= 1;
  if (ch.refs > 0) return;
  ch.busy = true;
  const CUmemGenericAllocationHandle h = ch.h;
  const int64_t bytes = chunk_bytes(c);
  lk.unlock();
  CUresult e = CUDA_SUCCESS;
  double t_unmap = 0;
  try {
    fence_unmap();            // queued kernels may still read the chunk
    const double t0 = now_us();
    e = driver().MemUnmap(va_[b] + (CUdeviceptr)(c * chunk_ * t_), (size_t)bytes);
    t_unmap = now_us() - t0;
  } catch (...) {
    lk.lock();
    ch.refs += 1;
    ch.busy = false;
    ch_cv_.notify_all();
    throw;
  }
  lk.lock();
  ch.busy = false;
  if (e != CUDA_SUCCESS) {
    ch.refs += 1;             // still mapped: keep the reference so state stays consistent
    ch_cv_.notify_all();
    lk.unlock();
    check_cu(e, "cuMemUnmap(chunk)");
  }
  ch.h = 0;
  CUresult er = CUDA_SUCCESS;
  if (!release_physical_) {
    ch_free_[bytes].push_back(h);
  } else {
    er = driver().MemRelease(h);   // unmapped either way; a failed release only leaks the handle
    if (er == CUDA_SUCCESS) real_releases_ += 1;
  }
  real_unmap_us_ += t_unmap;
  real_unmaps_ += 1;
  ch_mapped_ -= 1;
  ch_mapped_bytes_ -= bytes;
  ch_cv_.notify_all();
  if (er != CUDA_SUCCESS) {
    lk.unlock();
    check_cu(er, "cuMemRelease(chunk)");
  }
}

cudaEvent_t Manager::use_event_locked(cudaStream_t st, size_t* idx) {
  for (size_t i = 0; i < use_events_.size(); ++i)
    if (use_events_[i].first == st) {
      *idx = i;
      return use_events_[i].second;
    }
  cudaEvent_t ev = nullptr;
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;   // first use may be inside a capture
  check_rt(cudaThreadExchangeStreamCaptureMode(&mode), "cudaThreadExchangeStreamCaptureMode");
  const cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaThreadExchangeStreamCaptureMode(&mode);
  check_rt(e, "cudaEventCreate(use)");
  use_events_.emplace_back(st, ev);
  use_dirty_.push_back(0);
  *idx = use_events_.size() - 1;
  return ev;
}

// Unmap fence bookkeeping.  A kernel launch through the manager (explicit_mark = false) only flags
// its stream, or, inside a graph capture, the capture; fence_unmap records the stream's event
// when it needs it.  An explicit mark (vattn_mark_use) records now: inside a capture that is an
// external event node (every replay re-arms the fence) and it covers the capture's launches so
// far, so a captured region should end with one.
void Manager::mark_use(cudaStream_t st, bool explicit_mark) {
  if (!real()) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  unsigned long long cap_id = 0;
  check_rt(cudaStreamGetCaptureInfo(st, &cs, &cap_id), "cudaStreamGetCaptureInfo");
  const bool capturing = cs == cudaStreamCaptureStatusActive;
  std::lock_guard<std::mutex> lk(use_mu_);
  size_t i = 0;
  cudaEvent_t ev = use_event_locked(st, &i);
  if (!explicit_mark) {
    if (capturing) open_captures_.insert(cap_id);
    else use_dirty_[i] = 1;
    use_recorded_ = true;
    return;
  }
  if (capturing) {
    check_rt(cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal), "cudaEventRecord(use, graph)");
    open_captures_.erase(cap_id);
  } else {
    check_rt(cudaEventRecord(ev, st), "cudaEventRecord(use)");
    use_dirty_[i] = 0;
  }
  use_recorded_ = true;
}

// ---- policy ------------------------------------------------------------------------------------
int64_t Manager::groups_required(int64_t seq) const {  // manager.py:134-135, geometry.py:177-183
  return (seq * per_buffer_token_bytes_ + t_ - 1) / t_;
}

int32_t Manager::best_inactive() const {  // max over inactive of (mapped_groups, -req_id)
  int32_t best = -1;
  for (int32_t r = 0; r < (int32_t)slots_.size(); ++r) {
    if (slots_[r].active) continue;
    if (best < 0 || slots_[r].mapped_groups > slots_[best].mapped_groups) best = r;
  }
  return best;
}

// alloc_reqid's choice as the reference makes it: admission precedes execute_plan
// (simulator.py:395-418), so a plan executed early (during the previous iteration's compute)
// must not influence which inactive slot is reused.  Credits undo its effect on the ranking.

int32_t Manager::alloc_reqid() {  // manager.py:163-178
  int32_t rid;
  if (eager_slot_ >= 0 && !slots_[eager_slot_].active) {
    rid = (int32_t)eager_slot_;
    eager_slot_ = -1;
  } else {
    rid = -1;
    for (int32_t r = 0; r < (int32_t)slots_.size(); ++r) {
      if (slots_[r].active) continue;
      if (rid < 0 || ranked(slots_[r], plan_credit_[r]) > ranked(slots_[rid], plan_credit_[rid])) rid = r;
    }
    if (rid < 0)
      throw Fail(VATTN_BATCH_FULL, "all " + std::to_string(slots_.size()) + " request slots active");
  }
  Slot& s = slots_[rid];
  s.active = true;
  s.context_len = 0;
  s.phase = PREFILL;
  return rid;
}

void Manager::free_reqid(int32_t rid) {  // manager.py:180-190 — no driver calls
  if (rid < 0 || rid >= (int32_t)slots_.size()) throw Fail(VATTN_VALUE_ERROR, "req_id out of range");
  Slot& s = slots_[rid];
  if (!s.active) throw Fail(VATTN_DOUBLE_FREE, "slot " + std::to_string(rid) + " is not active");
  std::lock_guard<std::mutex> lk(slot_mu_);   // a prefetch job may be snapshotting the table
  s.active = false;
  s.context_len = 0;
  s.phase = INACTIVE;
  freed_counter_ += 1;
  s.freed_seq = freed_counter_;
}

std::pair<int64_t, double> Manager::acquire_handle() {  // manager.py:194-204
  if (!handle_cache_.empty()) {
    const int64_t h = handle_cache_.front();
    handle_cache_.pop_front();
    return {h, 0.0};
  }
  if (precreated_ > 0) return {dev_take_precreated(), 0.0};
  const int64_t h = dev_create();
  return {h, unit_cost(api_create_)};
}

double Manager::map_group(int64_t rid, int64_t g) {  // manager.py:206-220, all-or-nothing
  std::vector<int64_t> got;
  got.reserve((size_t)buffer_count_);
  double us = 0.0;
  try {
    for (int64_t i = 0; i < buffer_count_; ++i) {
      auto hc = acquire_handle();
      got.push_back(hc.first);
      us += hc.second;
    }
  } catch (const Fail& f) {
    if (f.code != VATTN_POOL_EXHAUSTED) throw;
    for (int64_t h : got) handle_cache_.push_back(h);
    throw;
  }
  const int64_t off = slot_offset(rid, g);
  for (int64_t b = 0; b < buffer_count_; ++b) us += dev_map((int32_t)b, off, got[b]);
  return us;
}

double Manager::release_top_group(int64_t rid) {  // manager.py:222-230
  Slot& s = slots_[rid];
  const int64_t g = s.mapped_groups - 1;
  const int64_t off = slot_offset(rid, g);
  double us = 0.0;
  for (int64_t b = 0; b < buffer_count_; ++b) us += dev_unmap_release((int32_t)b, off);
  s.mapped_groups = g;
  return us;
}

std::vector<int32_t> Manager::reclaim_victims() const {  // manager.py:232-236
  std::vector<int32_t> v;
  for (int32_t r = 0; r < (int32_t)slots_.size(); ++r)
    if (!slots_[r].active && slots_[r].mapped_groups > 0) v.push_back(r);
  std::stable_sort(v.begin(), v.end(), [&](int32_t a, int32_t b) {
    const bool ea = a == eager_slot_, eb = b == eager_slot_;
    if (ea != eb) return !ea;  // eager slot harvested last
    if (slots_[a].freed_seq != slots_[b].freed_seq) return slots_[a].freed_seq < slots_[b].freed_seq;
    return a < b;
  });
  return v;
}

std::pair<int64_t, double> Manager::reclaim_until(int64_t target) {  // manager.py:238-251
  int64_t freed = 0;
  double us = 0.0;
  for (int32_t r : reclaim_victims()) {
    Slot& s = slots_[r];
    while (s.mapped_groups > 0 && available() < target) {
      us += release_top_group(r);
      freed += 1;
    }
    if (s.mapped_groups == 0 && eager_slot_ == r) eager_slot_ = -1;
    if (available() >= target) break;
  }
  return {freed, us};
}

bool Manager::step(const int64_t* seq, int32_t n, double* sync_out) {  // manager.py:255-296
  Nvtx nv("vattn.step");
  if (n != (int32_t)slots_.size())
    throw Fail(VATTN_VALUE_ERROR, "expected " + std::to_string(slots_.size()) + " sequence lengths, got " +
                                      std::to_string(n));
  for (int32_t r = 0; r < n; ++r) {
    if (!slots_[r].active && seq[r] != 0)
      throw Fail(VATTN_VALUE_ERROR, "inactive slot " + std::to_string(r) + " has nonzero length");
    if (seq[r] < 0 || seq[r] > max_context_)
      throw Fail(VATTN_VALUE_ERROR, "slot " + std::to_string(r) + " length outside [0, max_context]");
  }
  double sync_us = 0.0;
  for (int32_t r = 0; r < n; ++r) {
    Slot& s = slots_[r];
    if (!s.active) continue;
    const int64_t required = groups_required(seq[r]);
    if (s.phase == PREFILL)
      while (s.mapped_groups > required) sync_us += release_top_group(r);
    while (s.mapped_groups < required) {
      try {
        sync_us += map_group(r, s.mapped_groups);
      } catch (const Fail& f) {
        if (f.code != VATTN_POOL_EXHAUSTED) throw;
        auto fr = reclaim_until(buffer_count_ * t_);
        sync_us += fr.second;
        if (fr.first == 0) {
          *sync_out = sync_us;
          publish_rows();   // earlier slots of this step did grow
          return false;
        }
        continue;
      }
      s.mapped_groups += 1;
    }
    s.context_len = seq[r];
    s.phase = DECODE;
  }
  *sync_out = sync_us;
  publish_rows();
  return true;
}

// The published rows track what is PHYSICALLY readable without a fault: they grow with the
// logical state (end of step / of a background job) and shrink only in real_unmap, after the
// unmap fence, for the page about to go.  A lazily kept page (lazy_unmap) stays readable until
// it is really unmapped.  Copies go through a private non-blocking stream, so a publish never
// waits for the caller's in-flight kernels.
static void push_rows(int32_t* d, int32_t* h, const std::vector<int32_t>& v, cudaStream_t st) {
  std::memcpy(h, v.data(), v.size() * 4);
  check_rt(cudaMemcpyAsync(d, h, v.size() * 4, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync(read guard)");
  check_rt(cudaStreamSynchronize(st), "cudaStreamSynchronize(read guard)");
}

void Manager::publish_rows() {
  if (!real()) return;
  std::lock_guard<std::mutex> lk(pub_mu_);
  bool changed = false;
  for (int32_t r = 0; r < (int32_t)slots_.size(); ++r) {
    const int32_t v = rows_of(slots_[r].mapped_groups);
    if (v > pub_rows_[r]) {
      pub_rows_[r] = v;
      changed = true;
    }
  }
  if (changed) push_rows(d_rows_, h_rows_, pub_rows_, pub_stream_);
}

void Manager::shrink_rows(int64_t off) {
  if (!d_rows_) return;
  const int64_t r = off / slot_stride_, g = (off % slot_stride_) / t_;
  if (r < 0 || r >= (int64_t)pub_rows_.size()) return;
  std::lock_guard<std::mutex> lk(pub_mu_);
  const int32_t v = rows_of(g);
  if (v >= pub_rows_[r]) return;
  pub_rows_[r] = v;
  push_rows(d_rows_, h_rows_, pub_rows_, pub_stream_);
}

void Manager::check_device_errors() {
  if (!h_err_) return;
  volatile uint32_t* e = h_err_;
  if (e[0] == 0) return;
  const uint32_t slot = e[1], want = e[2], have = e[3];
  e[0] = 0;
  throw Fail(VATTN_VALUE_ERROR, "a kernel was asked to read " + std::to_string(want) + " rows of slot " +
                                    std::to_string(slot) + ", which has " + std::to_string(have) +
                                    " backed rows (or the slot index is out of range); its reads were clamped"
                                    " (call step() with the grown lengths first)");
}

int64_t Manager::plan_overlap(const int64_t* next, int32_t n) {  // manager.py:298-311
  if (n != (int32_t)slots_.size()) throw Fail(VATTN_VALUE_ERROR, "plan length mismatch");
  last_plan_.clear();
  for (int32_t r = 0; r < n; ++r) {
    const Slot& s = slots_[r];
    if (!s.active) continue;
    if (next[r] < 0) throw Fail(VATTN_VALUE_ERROR, "negative length");
    const int64_t req = std::min(groups_required(next[r]), groups_per_slot_);
    for (int64_t g = s.mapped_groups; g < req; ++g)
      for (int64_t b = 0; b < buffer_count_; ++b) {
        last_plan_.push_back(r);
        last_plan_.push_back(b);
        last_plan_.push_back(slot_offset(r, g));
      }
  }
  return (int64_t)last_plan_.size() / 3;
}

double Manager::execute_plan(const int64_t* trip, int64_t n) {  // manager.py:313-333
  Nvtx nv("vattn.execute_plan");
  double us = 0.0;
  std::unordered_set<int64_t> done;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t rid = trip[3 * i], off = trip[3 * i + 2];
    if (rid < 0 || rid >= (int64_t)slots_.size()) throw Fail(VATTN_VALUE_ERROR, "plan req_id out of range");
    Slot& s = slots_[rid];
    const int64_t rel = off - rid * slot_stride_;
    // Python floor division
    const int64_t g = rel >= 0 ? rel / t_ : -((-rel + t_ - 1) / t_);
    const int64_t key = rid * (groups_per_slot_ + 1) + g;
    if ((g >= 0 && done.count(key)) || g < s.mapped_groups) continue;
    if (g >= groups_per_slot_) continue;
    while (s.mapped_groups <= g) {  // grow strictly in order; the mapped prefix stays contiguous
      try {
        us += map_group(rid, s.mapped_groups);
      } catch (const Fail& f) {
        if (f.code != VATTN_POOL_EXHAUSTED) throw;
        return us;
      }
      s.mapped_groups += 1;
      if (credit_mode_) plan_credit_[rid] += 1;
    }
    done.insert(key);
  }
  return us;
}

double Manager::eager_prepare(int64_t k) {  // manager.py:335-361
  Nvtx nv("vattn.eager_prepare");
  if (k < 0) k = eager_groups_;
  if (k <= 0) return 0.0;
  k = std::min(k, groups_per_slot_);
  if (eager_slot_ >= 0 && slots_[eager_slot_].mapped_groups >= k) return 0.0;
  const int32_t rid = best_inactive();
  if (rid < 0) return 0.0;
  eager_slot_ = rid;
  Slot& s = slots_[rid];
  double us = 0.0;
  const int64_t group_bytes = buffer_count_ * t_;
  while (s.mapped_groups < k) {
    if (available() - group_bytes < reclaim_floor()) break;
    try {
      us += map_group(rid, s.mapped_groups);
    } catch (const Fail& f) {
      if (f.code != VATTN_POOL_EXHAUSTED) throw;
      break;
    }
    s.mapped_groups += 1;
  }
  return us;
}

std::pair<int64_t, double> Manager::reclaim() {  // manager.py:363-372
  const int64_t floor = reclaim_floor();
  if (available() >= floor) return {0, 0.0};
  return reclaim_until(floor);
}

// ---- background thread (simulator.py:199-203 on a real thread) ----------------------------
// A FIFO of jobs; each runs execute_plan -> eager_prepare -> reclaim per its flags.  API calls
// join the queue before touching state, except free_reqid, which only waits for queued
// eager/reclaim jobs (execute_plan never reads the fields free_reqid writes, and vice versa).
void Manager::bg_loop() {
  bool ctx_set = false;
  for (;;) {
    BgJob job;
    {
      std::unique_lock<std::mutex> lk(bg_mu_);
      bg_cv_.wait(lk, [&] { return !bg_queue_.empty() || bg_stop_; });
      if (bg_queue_.empty()) return;
      job = std::move(bg_queue_.front());
      bg_queue_.pop_front();
    }
    Nvtx nv("vattn.bg_job");
    vattn_bg_result res{};
    vattn_status st = VATTN_OK;
    std::string err;
    const double t0 = now_us();
    try {
      if (real() && !ctx_set) {
        check_cu(driver().CtxSetCurrent(ctx_), "cuCtxSetCurrent(bg)");
        ctx_set = true;
      }
      fenced_ = false;
      if (job.flags & VATTN_BG_EXECUTE_PLAN) {
        credit_mode_ = (job.flags & VATTN_BG_CREDIT) != 0;
        res.plan_us = execute_plan(job.plan.data(), (int64_t)job.plan.size() / 3);
        credit_mode_ = false;
      }
      if (job.flags & VATTN_BG_EAGER) res.eager_us = eager_prepare(job.eager_k);
      if (job.flags & VATTN_BG_RECLAIM) {
        auto r = reclaim();
        res.reclaimed_groups = r.first;
        res.reclaim_us = r.second;
      }
      flush_access();
      publish_rows();
      if (job.flags & VATTN_BG_PREFETCH) prefetch();
    } catch (const Fail& f) {
      st = f.code;
      err = f.what();
    } catch (const std::exception& e) {
      st = VATTN_BAD_STATE;
      err = e.what();
    }
    res.bg_wall_us = now_us() - t0;
    {
      std::lock_guard<std::mutex> lk(bg_mu_);
      bg_res_.plan_us += res.plan_us;
      bg_res_.eager_us += res.eager_us;
      bg_res_.reclaim_us += res.reclaim_us;
      bg_res_.reclaimed_groups += res.reclaimed_groups;
      bg_res_.bg_wall_us += res.bg_wall_us;
      if (st != VATTN_OK && bg_status_ == VATTN_OK) {
        bg_status_ = st;
        bg_error_ = err;
      }
      bg_completed_ = job.seq;
    }
    bg_cv_.notify_all();
  }
}

double Manager::join_bg() {
  std::unique_lock<std::mutex> lk(bg_mu_);
  if (bg_completed_ == bg_submitted_) return 0.0;
  Nvtx nv("vattn.bg_join_wait");
  prefetch_cancel_.store(true, std::memory_order_relaxed);
  const double t0 = now_us();
  bg_cv_.wait(lk, [&] { return bg_completed_ == bg_submitted_; });
  return now_us() - t0;
}

double Manager::join_noncommuting() {
  std::unique_lock<std::mutex> lk(bg_mu_);
  if (bg_completed_ >= bg_last_noncommuting_) return 0.0;
  prefetch_cancel_.store(true, std::memory_order_relaxed);
  const double t0 = now_us();
  bg_cv_.wait(lk, [&] { return bg_completed_ >= bg_last_noncommuting_; });
  return now_us() - t0;
}

void Manager::bg_submit(const int64_t* trip, int64_t n, uint32_t flags, int64_t eager_k) {
  std::lock_guard<std::mutex> lk(bg_mu_);
  BgJob job;
  if (trip) job.plan.assign(trip, trip + 3 * n);
  else if (flags & VATTN_BG_EXECUTE_PLAN) job.plan = last_plan_;
  job.flags = flags;
  job.eager_k = eager_k;
  job.seq = ++bg_submitted_;
  if (flags & (VATTN_BG_EAGER | VATTN_BG_RECLAIM)) bg_last_noncommuting_ = job.seq;
  prefetch_cancel_.store(false, std::memory_order_relaxed);
  bg_queue_.push_back(std::move(job));
  bg_cv_.notify_all();
}

void Manager::bg_wait(vattn_bg_result* out) {
  std::unique_lock<std::mutex> lk(bg_mu_);
  const double t0 = now_us();
  if (bg_completed_ != bg_submitted_) prefetch_cancel_.store(true, std::memory_order_relaxed);
  bg_cv_.wait(lk, [&] { return bg_completed_ == bg_submitted_; });
  const double waited = now_us() - t0;
  vattn_bg_result r = bg_res_;
  r.waited_us = waited;
  bg_res_ = vattn_bg_result{};
  const vattn_status st = bg_status_;
  const std::string err = bg_error_;
  bg_status_ = VATTN_OK;
  bg_error_.clear();
  if (out) *out = r;
  if (st != VATTN_OK) throw Fail(st, "background job failed: " + err);
}

// Deferring eager_prepare/reclaim past step (so they run during compute) yields the same state
// as the reference order (eager -> reclaim -> step, simulator.py:414-426) when nothing can hit
// the pool floor or run dry: with A = available bytes, E eager groups and S step groups still
// to map, A - (E + S)·G >= floor keeps every eager floor check passing and reclaim a no-op in
// both orders, and enough cached/pre-created handles keep the modelled create charges in place.
bool Manager::deferral_safe(const int64_t* seq, int32_t n, int64_t eager_k) const {
  if (n != (int32_t)slots_.size()) return false;
  int64_t k = eager_k < 0 ? eager_groups_ : eager_k;
  int64_t E = 0;
  if (k > 0) {
    k = std::min(k, groups_per_slot_);
    const bool done = eager_slot_ >= 0 && slots_[eager_slot_].mapped_groups >= k;
    if (!done) {
      const int32_t x = best_inactive();
      if (x >= 0) E = std::max<int64_t>(0, k - slots_[x].mapped_groups);
    }
  }
  int64_t S = 0;
  for (int32_t r = 0; r < n; ++r) {
    if (!slots_[r].active) continue;
    if (seq[r] < 0 || seq[r] > max_context_) return false;
    S += std::max<int64_t>(0, groups_required(seq[r]) - slots_[r].mapped_groups);
  }
  const int64_t G = buffer_count_ * t_;
  if (available() - (E + S) * G < reclaim_floor()) return false;
  const int64_t free_handles = (int64_t)handle_cache_.size() + precreated_;
  return free_handles >= (E + S) * buffer_count_;
}

// ---- introspection ------------------------------------------------------------------------------
void Manager::counters(vattn_counters* o) const {
  std::memset(o, 0, sizeof(*o));
  o->created = created_;
  o->mapped = mapped_;
  o->precreated = precreated_;
  o->total_mapped_bytes = total_mapped_bytes_;
  o->capacity = capacity_;
  o->page_group_size = t_;
  o->buffer_count = buffer_count_;
  o->groups_per_slot = groups_per_slot_;
  o->slot_stride = slot_stride_;
  o->buffer_size = buffer_size_;
  o->per_buffer_token_bytes = per_buffer_token_bytes_;
  o->max_batch = (int64_t)slots_.size();
  o->max_context = max_context_;
  o->eager_slot = eager_slot_;
  o->next_handle_id = next_hid_;
  o->init_us = init_us_;
  o->charged_us = charged_total();
  std::lock_guard<std::mutex> lk(pf_mu_);
  // chunk mode: every driver call (control thread and prefetch worker) goes through chunk_ref /
  // chunk_unref, which count them in real_*; pf_* then count the worker's logical pages only
  const bool ck = chunked();
  o->real_maps = real_maps_ + (ck ? 0 : pf_maps_);
  o->real_unmaps = real_unmaps_;
  o->real_set_access_calls = real_access_ + (ck ? 0 : pf_access_);
  o->real_creates = real_creates_;
  o->real_releases = real_releases_;
  o->real_map_wall_us = real_map_us_ + (ck ? 0 : pf_map_us_);
  o->real_unmap_wall_us = real_unmap_us_;
  o->real_create_wall_us = real_create_us_;
  o->real_set_access_wall_us = real_access_us_ + (ck ? 0 : pf_access_us_);
  o->init_wall_us = init_wall_us_;
  o->spec_maps = spec_maps_;
  o->spec_hits = spec_hits_;
  o->spec_steals = spec_steals_;
  o->spec_pages = (int64_t)spec_.size();
  o->lazy_unmaps = lazy_unmaps_;
  o->phys_chunk_groups = chunk_;
  if (chunked()) {
    std::lock_guard<std::mutex> lc(ch_mu_);   // lock order pf_mu_ -> ch_mu_, as in dev_precreate
    o->phys_chunks_mapped = ch_mapped_;
    o->phys_mapped_bytes = ch_mapped_bytes_;
  } else {
    o->phys_chunks_mapped = 0;
    o->phys_mapped_bytes = real() ? (mapped_ + (int64_t)spec_.size()) * t_ : 0;
  }
}

void Manager::slot_state(int64_t* out) const {
  for (size_t r = 0; r < slots_.size(); ++r) {
    out[5 * r + 0] = slots_[r].active ? 1 : 0;
    out[5 * r + 1] = slots_[r].context_len;
    out[5 * r + 2] = slots_[r].mapped_groups;
    out[5 * r + 3] = (int64_t)slots_[r].phase;
    out[5 * r + 4] = slots_[r].freed_seq;
  }
}

void Manager::api_stats(int64_t* calls, double* ledger, int32_t* order, int32_t* n_order) const {
  for (int a = 0; a < A_COUNT; ++a) {
    if (calls) calls[a] = calls_[a];
    if (ledger) ledger[a] = ledger_[a];
  }
  if (order)
    for (size_t i = 0; i < ledger_order_.size(); ++i) order[i] = ledger_order_[i];
  if (n_order) *n_order = (int32_t)ledger_order_.size();
}

int64_t Manager::buffer_mappings(int32_t b, int64_t* offs, int64_t* hids, int64_t cap) const {
  if (b < 0 || b >= (int32_t)buf_maps_.size()) throw Fail(VATTN_VALUE_ERROR, "buffer id out of range");
  std::vector<std::pair<int64_t, int64_t>> v(buf_maps_[b].begin(), buf_maps_[b].end());
  std::sort(v.begin(), v.end());
  for (int64_t i = 0; i < (int64_t)v.size() && i < cap; ++i) {
    if (offs) offs[i] = v[i].first;
    if (hids) hids[i] = v[i].second;
  }
  return (int64_t)v.size();
}

int64_t Manager::drain_events(int64_t* out, int64_t cap) {
  const int64_t n = (int64_t)events_.size() / 3;
  if (out == nullptr) return n;
  const int64_t k = std::min(n, cap);
  std::copy(events_.begin(), events_.begin() + 3 * k, out);
  events_.erase(events_.begin(), events_.begin() + 3 * k);
  return k;
}

uint64_t Manager::buffer_base(int32_t b) const {
  if (b < 0 || b >= (int32_t)buffer_count_) throw Fail(VATTN_VALUE_ERROR, "buffer id out of range");
  if (!real()) throw Fail(VATTN_BAD_STATE, "shadow backend has no device buffers");
  return (uint64_t)va_[b];
}

// The decode kernels stream 64-token TMA boxes (kernels.cu kTile); a box that starts below a
// row's length ends inside its mapped page-groups for every length only when a page-group spans
// a whole number of 64-token tiles.  Otherwise (layer-sliced layout: 32 tokens per 2 MiB group at
// Llama-3-8B, 17.07 at Yi-34B) layer_view sets tail_guard and the kernels load each row's last,
// partial tile with per-row loads bounded by the row's length.
void Manager::check_decode_tiling() const {}

CacheView Manager::layer_view(int32_t layer) const {
  if (!real()) throw Fail(VATTN_BAD_STATE, "kernels need the CUDA backend");
  if (layer < 0 || layer >= n_layers_) throw Fail(VATTN_VALUE_ERROR, "layer out of range");
  if (elem_bytes_ != 2) throw Fail(VATTN_UNSUPPORTED, "kernels compute on bf16 caches");
  CacheView v;
  const int64_t row = (int64_t)hkv_local_ * head_dim_ * elem_bytes_;
  if (sliced_) {  // [B, L, N, H, D]: layer l sits at l*row inside each token's N*row bytes
    v.k_base = va_[0] + (uint64_t)layer * row;
    v.v_base = va_[1] + (uint64_t)layer * row;
    v.token_stride = (int64_t)n_layers_ * row;
  } else {  // buffer id 2*layer + {0: K, 1: V}
    v.k_base = va_[2 * layer];
    v.v_base = va_[2 * layer + 1];
    v.token_stride = row;
  }
  v.slot_stride = slot_stride_;
  v.tail_guard = (t_ % (64 * per_buffer_token_bytes_) != 0) ? 1 : 0;
  v.slot_rows = d_rows_;
  v.err = d_err_;
  v.slot_tokens = (int32_t)max_context_;
  v.n_slots = (int32_t)slots_.size();
  v.hkv = hkv_local_;
  v.d = head_dim_;
  return v;
}

CacheView view_from_desc(const vattn_cache_desc* c) {
  if (!c) throw Fail(VATTN_VALUE_ERROR, "null cache descriptor");
  CacheView v;
  v.k_base = (uint64_t)c->k_base;
  v.v_base = (uint64_t)c->v_base;
  v.slot_stride = c->slot_stride_bytes;
  v.token_stride = c->token_stride_bytes ? c->token_stride_bytes : (int64_t)c->n_kv_heads * c->head_dim * 2;
  v.slot_tokens = c->slot_tokens;
  v.n_slots = c->n_slots;
  v.hkv = c->n_kv_heads;
  v.d = c->head_dim;
  return v;
}

}  // namespace vattn

// ================================================================================ C ABI
using vattn::Fail;
using vattn::Manager;

struct vattn_t {
  Manager* m = nullptr;
  // per launching stream, the layer the last decode through this handle appended a row to (-1
  // none): the next decode of a DIFFERENT layer may stream its K/V under PDL before that kernel
  // completes (kernels.cu DecodeParams::kv_early)
  std::mutex early_mu;
  std::unordered_map<cudaStream_t, int32_t> last_append_layer;
  // Split-K decode workspaces, one per launching stream (concurrent decodes on two streams must
  // not share part_o/part_lse).  Never freed before vattn_destroy: a CUDA graph captured with a
  // workspace keeps its address, so a grown one only retires the old (ADVICE r1 core.cpp:1783).
  std::mutex ws_mu;
  std::unordered_map<cudaStream_t, std::pair<void*, int64_t>> ws;
  std::vector<void*> ws_all;
};

// Decide kv_early for a decode of `layer` on `st` and record whether it appends (fused).
static void decode_pdl_hint(vattn_t* h, cudaStream_t st, int32_t layer, bool appends) {
  static const bool on = [] {
    const char* e = getenv("VATTN_DEC_PDL");
    return !e || atoi(e) != 0;
  }();
  std::lock_guard<std::mutex> lk(h->early_mu);
  auto it = h->last_append_layer.find(st);
  const int32_t prev = it == h->last_append_layer.end() ? -2 : it->second;
  vattn::set_decode_kv_early(on && prev != -2 && prev != layer ? 1 : 0);
  h->last_append_layer[st] = appends ? layer : -1;
}

// Workspace for a decode of `need` bytes on stream st.  The first one of a stream is sized for the
// manager's max_batch, so it normally never grows; cudaMalloc runs with the thread's capture mode
// relaxed, so a first decode inside a graph capture is legal too.
static void* decode_workspace(vattn_t* h, cudaStream_t st, int64_t need, int64_t max_need, int64_t* bytes) {
  std::lock_guard<std::mutex> lk(h->ws_mu);
  auto it = h->ws.find(st);
  if (it != h->ws.end() && it->second.second >= need) {
    *bytes = it->second.second;
    return it->second.first;
  }
  const int64_t size = std::max(need, max_need);
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  vattn::check_rt(cudaThreadExchangeStreamCaptureMode(&mode), "cudaThreadExchangeStreamCaptureMode");
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, (size_t)size);
  cudaThreadExchangeStreamCaptureMode(&mode);
  vattn::check_rt(e, "cudaMalloc(decode workspace)");
  h->ws_all.push_back(p);
  h->ws[st] = {p, size};
  *bytes = size;
  return p;
}

template <typename F>
static vattn_status guard(F&& f) {
  try {
    f();
    return VATTN_OK;
  } catch (const Fail& e) {
    vattn::set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    vattn::set_last_error("out of host memory");
    return VATTN_BAD_STATE;
  } catch (const std::exception& e) {
    vattn::set_last_error(e.what());
    return VATTN_BAD_STATE;
  }
}

template <typename F>
static vattn_status api_call(vattn_t* h, F&& f) {
  if (!h || !h->m) {
    vattn::set_last_error("null handle");
    return VATTN_BAD_STATE;
  }
  return guard([&] {
    h->m->join_bg();
    h->m->check_device_errors();
    h->m->begin_call();
    try {
      f(*h->m);
    } catch (...) {
      try { h->m->end_call(); } catch (...) {}
      throw;
    }
    h->m->end_call();
  });
}

extern "C" {

const char* vattn_last_error(void) { return vattn::g_last_error.c_str(); }
int32_t vattn_abi_version(void) { return 1; }

int32_t vattn_abi_sizes(int64_t* out, int32_t n) {
  const int64_t sz[8] = {(int64_t)sizeof(vattn_config),       (int64_t)sizeof(vattn_counters),
                         (int64_t)sizeof(vattn_step_result),  (int64_t)sizeof(vattn_bg_result),
                         (int64_t)sizeof(vattn_iteration_result), (int64_t)sizeof(vattn_cache_desc),
                         (int64_t)sizeof(vattn_rotary),       (int64_t)sizeof(vattn_latency_entry)};
  const int32_t k = n < 8 ? n : 8;
  for (int32_t i = 0; i < k && out; ++i) out[i] = sz[i];
  return k;
}

vattn_status vattn_create(const vattn_config* cfg, vattn_t** out) {
  return guard([&] {
    if (!cfg || !out) throw Fail(VATTN_VALUE_ERROR, "null argument");
    auto h = std::make_unique<vattn_t>();
    h->m = new Manager(*cfg);
    h->m->ks = vattn::kernel_state_new();
    *out = h.release();
  });
}

vattn_status vattn_destroy(vattn_t* h) {
  if (!h) return VATTN_OK;
  return guard([&] {
    if (h->m) {
      if (h->m->ks) vattn::kernel_state_free(h->m->ks);
      delete h->m;
    }
    for (void* p : h->ws_all) cudaFree(p);
    delete h;
  });
}

vattn_status vattn_alloc_reqid(vattn_t* h, int32_t* rid) {
  return api_call(h, [&](Manager& m) { *rid = m.alloc_reqid(); });
}

vattn_status vattn_free_reqid(vattn_t* h, int32_t rid) {
  // free_reqid commutes with a queued execute_plan (disjoint fields), so it waits only for
  // queued eager/reclaim jobs, which read `active` (manager.py:232-236, :347-349).
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] {
    h->m->join_noncommuting();
    h->m->free_reqid(rid);
  });
}

vattn_status vattn_step(vattn_t* h, const int64_t* seq, int32_t n, vattn_step_result* out) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] {
    const double t0 = vattn::now_us();
    const double waited = h->m->join_bg();
    h->m->check_device_errors();
    h->m->begin_call();
    double us = 0.0;
    bool ok;
    try {
      h->m->reset_credits();
      ok = h->m->step(seq, n, &us);
    } catch (...) {
      try { h->m->end_call(); } catch (...) {}
      throw;
    }
    h->m->end_call();
    if (out) {
      out->ok = ok ? 1 : 0;
      out->sync_us = us;
      out->bg_wait_us = waited;
      out->wall_us = vattn::now_us() - t0;
    }
  });
}

vattn_status vattn_iteration_step(vattn_t* h, const int64_t* seq, int32_t n, uint32_t flags,
                                  int64_t eager_k, vattn_iteration_result* out) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] {
    Manager& m = *h->m;
    const double t0 = vattn::now_us();
    vattn_iteration_result r{};
    r.bg_wait_us = m.join_bg();
    m.check_device_errors();
    m.begin_call();
    try {
      const bool want = (flags & (VATTN_BG_EAGER | VATTN_BG_RECLAIM)) != 0;
      const bool defer = want && (flags & VATTN_ITER_DEFER) && m.deferral_safe(seq, n, eager_k);
      if (want && !defer) {
        const double t1 = vattn::now_us();
        if (flags & VATTN_BG_EAGER) r.eager_us = m.eager_prepare(eager_k);
        if (flags & VATTN_BG_RECLAIM) {
          auto rc = m.reclaim();
          r.reclaimed_groups = rc.first;
          r.reclaim_us = rc.second;
        }
        r.sync_bg_wall_us = vattn::now_us() - t1;
      }
      m.reset_credits();
      double us = 0.0;
      r.ok = m.step(seq, n, &us) ? 1 : 0;
      r.sync_us = us;
      m.end_call();
      if (defer) {
        m.bg_submit(nullptr, 0, flags & (VATTN_BG_EAGER | VATTN_BG_RECLAIM), eager_k);
        r.deferred = 1;
      }
    } catch (...) {
      try { m.end_call(); } catch (...) {}
      throw;
    }
    r.wall_us = vattn::now_us() - t0;
    if (out) *out = r;
  });
}

vattn_status vattn_plan_overlap(vattn_t* h, const int64_t* next, int32_t n, int64_t* n_entries) {
  return api_call(h, [&](Manager& m) {
    const int64_t k = m.plan_overlap(next, n);
    if (n_entries) *n_entries = k;
  });
}

vattn_status vattn_plan_fetch(vattn_t* h, int64_t* trip, int64_t cap) {
  return api_call(h, [&](Manager& m) {
    const auto& p = m.last_plan();
    const int64_t k = std::min<int64_t>(cap, (int64_t)p.size() / 3);
    std::copy(p.begin(), p.begin() + 3 * k, trip);
  });
}

vattn_status vattn_execute_plan(vattn_t* h, const int64_t* trip, int64_t n, double* us) {
  return api_call(h, [&](Manager& m) {
    const double u = m.execute_plan(trip, n);
    if (us) *us = u;
  });
}

vattn_status vattn_eager_prepare(vattn_t* h, int64_t k, double* us) {
  return api_call(h, [&](Manager& m) {
    const double u = m.eager_prepare(k);
    if (us) *us = u;
  });
}

vattn_status vattn_reclaim(vattn_t* h, int64_t* freed, double* us) {
  return api_call(h, [&](Manager& m) {
    auto r = m.reclaim();
    if (freed) *freed = r.first;
    if (us) *us = r.second;
  });
}

vattn_status vattn_reclaim_until(vattn_t* h, int64_t target, int64_t* freed, double* us) {
  return api_call(h, [&](Manager& m) {
    auto r = m.reclaim_until(target);
    if (freed) *freed = r.first;
    if (us) *us = r.second;
  });
}

vattn_status vattn_bg_submit(vattn_t* h, const int64_t* trip, int64_t n, uint32_t flags,
                             int64_t eager_k) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] { h->m->bg_submit(trip, n, flags, eager_k); });
}

vattn_status vattn_bg_wait(vattn_t* h, vattn_bg_result* out) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] { h->m->bg_wait(out); });
}

vattn_status vattn_check_errors(vattn_t* h) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] { h->m->check_device_errors(); });
}

vattn_status vattn_mark_use(vattn_t* h, void* stream) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] { h->m->mark_use((cudaStream_t)stream, true); });
}

vattn_status vattn_counters_get(vattn_t* h, vattn_counters* out) {
  return api_call(h, [&](Manager& m) { m.counters(out); });
}

vattn_status vattn_counters_peek(vattn_t* h, vattn_counters* out) {
  // No join: a snapshot that may race with a running background job (monitoring only).
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] { h->m->counters(out); });
}

vattn_status vattn_slot_state(vattn_t* h, int64_t* out, int64_t cap) {
  return api_call(h, [&](Manager& m) {
    if (cap < m.max_batch()) throw Fail(VATTN_VALUE_ERROR, "slot buffer too small");
    m.slot_state(out);
  });
}

int32_t vattn_api_count(void) { return vattn::A_COUNT; }
const char* vattn_api_name(int32_t i) {
  return (i >= 0 && i < vattn::A_COUNT) ? vattn::kApiNames[i] : "";
}

vattn_status vattn_api_stats(vattn_t* h, int64_t* calls, double* ledger, int32_t* order,
                             int32_t* n_order) {
  return api_call(h, [&](Manager& m) { m.api_stats(calls, ledger, order, n_order); });
}

vattn_status vattn_buffer_mappings(vattn_t* h, int32_t b, int64_t* offs, int64_t* hids,
                                   int64_t cap, int64_t* n) {
  return api_call(h, [&](Manager& m) {
    const int64_t k = m.buffer_mappings(b, offs, hids, cap);
    if (n) *n = k;
  });
}

vattn_status vattn_events(vattn_t* h, int64_t* trip, int64_t cap, int64_t* n) {
  return api_call(h, [&](Manager& m) {
    const int64_t k = m.drain_events(trip, cap);
    if (n) *n = k;
  });
}

vattn_status vattn_set_foreground(vattn_t* h, int32_t active) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] { h->m->set_foreground(active != 0); });
}

vattn_status vattn_predict_alloc(vattn_t* h, int32_t k, int32_t* out, int32_t* n) {
  return api_call(h, [&](Manager& m) {
    if (!out || !n) throw Fail(VATTN_VALUE_ERROR, "null argument");
    const auto v = m.predict_alloc(k);
    std::copy(v.begin(), v.end(), out);
    *n = (int32_t)v.size();
  });
}

vattn_status vattn_prefetch_hint(vattn_t* h, const int32_t* slots, const int64_t* tokens, int32_t n) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] {
    if (n > 0 && (!slots || !tokens)) throw Fail(VATTN_VALUE_ERROR, "null argument");
    h->m->prefetch_hint(slots, tokens, n);
  });
}

vattn_status vattn_slot_ready(vattn_t* h, int32_t slot, int64_t tokens, int32_t* ready) {
  return api_call(h, [&](Manager& m) {
    if (!ready) throw Fail(VATTN_VALUE_ERROR, "null argument");
    *ready = m.slot_ready(slot, tokens) ? 1 : 0;
  });
}

vattn_status vattn_buffer_base(vattn_t* h, int32_t b, uint64_t* dptr) {
  return api_call(h, [&](Manager& m) { *dptr = m.buffer_base(b); });
}

// ---- handle-based kernel entry points ------------------------------------------------------
vattn_status vattn_kv_append(vattn_t* h, int32_t layer, const void* k_new, const void* v_new,
                             int32_t batch, int32_t n_new, const int32_t* seqlens,
                             const int32_t* batch_idx, void* stream) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] {
    vattn::Nvtx nv("vattn.kv_append");
    h->m->check_device_errors();
    const vattn::CacheView v = h->m->layer_view(layer);
    vattn::launch_kv_append(h->m->ks, layer, v, k_new, v_new, batch, n_new, seqlens, batch_idx,
                            (cudaStream_t)stream);
    h->m->mark_use((cudaStream_t)stream, false);
  });
}

vattn_status vattn_decode(vattn_t* h, int32_t layer, const void* q, void* out, int32_t batch,
                          const int32_t* seqlens, const int32_t* batch_idx, float scale,
                          int32_t num_splits, void* stream) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] {
    h->m->check_decode_tiling();
    vattn::set_decode_order_hint(h->m->mixed_lengths() ? 1 : 0);
    vattn::Nvtx nv("vattn.decode");
    h->m->check_device_errors();
    const vattn::CacheView v = h->m->layer_view(layer);
    const int hq = h->m->hq_local();
    int64_t ws_bytes = 0;
    void* ws = decode_workspace(h, (cudaStream_t)stream, vattn_decode_workspace_bytes(batch, hq, v.d, 0),
                                vattn_decode_workspace_bytes(h->m->max_batch(), hq, v.d, 0), &ws_bytes);
    decode_pdl_hint(h, (cudaStream_t)stream, layer, false);
    vattn::launch_decode(h->m->ks, layer, v, q, out, batch, hq, seqlens, batch_idx, scale,
                         num_splits, ws, ws_bytes, (cudaStream_t)stream);
    h->m->mark_use((cudaStream_t)stream, false);
  });
}

vattn_status vattn_decode_append(vattn_t* h, int32_t layer, const void* q, const void* k_new,
                                 const void* v_new, void* out, int32_t batch,
                                 const int32_t* cache_seqlens, const int32_t* batch_idx, float scale,
                                 int32_t num_splits, void* stream) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] {
    h->m->check_decode_tiling();
    vattn::set_decode_order_hint(h->m->mixed_lengths() ? 1 : 0);
    vattn::Nvtx nv("vattn.decode_append");
    h->m->check_device_errors();
    const vattn::CacheView v = h->m->layer_view(layer);
    const int hq = h->m->hq_local();
    int64_t ws_bytes = 0;
    void* ws = decode_workspace(h, (cudaStream_t)stream, vattn_decode_workspace_bytes(batch, hq, v.d, 0),
                                vattn_decode_workspace_bytes(h->m->max_batch(), hq, v.d, 0), &ws_bytes);
    decode_pdl_hint(h, (cudaStream_t)stream, layer, k_new != nullptr);
    vattn::launch_decode(h->m->ks, layer, v, q, out, batch, hq, cache_seqlens, batch_idx, scale,
                         num_splits, ws, ws_bytes, (cudaStream_t)stream, k_new, v_new);
    h->m->mark_use((cudaStream_t)stream, false);
  });
}

vattn_status vattn_kv_append_rotary(vattn_t* h, int32_t layer, const void* k_new, const void* v_new,
                                    int32_t batch, int32_t n_new, const int32_t* seqlens,
                                    const int32_t* batch_idx, const vattn_rotary* rotary, void* stream) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] {
    if (!rotary) throw Fail(VATTN_VALUE_ERROR, "null rotary descriptor");
    vattn::Nvtx nv("vattn.kv_append");
    h->m->check_device_errors();
    const vattn::CacheView v = h->m->layer_view(layer);
    const vattn::Rotary rot{rotary->cos, rotary->sin, rotary->rotary_dim, rotary->interleaved};
    vattn::launch_kv_append(h->m->ks, layer, v, k_new, v_new, batch, n_new, seqlens, batch_idx,
                            (cudaStream_t)stream, &rot);
    h->m->mark_use((cudaStream_t)stream, false);
  });
}

vattn_status vattn_prefill_varlen(vattn_t* h, int32_t layer, const void* q, void* out, int32_t n_req,
                                  const int32_t* q_start, const int32_t* n_q, const int32_t* slots,
                                  const int32_t* kv_len, float scale, int32_t causal, void* stream) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] {
    if (n_req > 0 && (!q_start || !n_q || !slots || !kv_len)) throw Fail(VATTN_VALUE_ERROR, "null argument");
    vattn::Nvtx nv("vattn.prefill_varlen");
    h->m->check_device_errors();
    const vattn::CacheView v = h->m->layer_view(layer);
    for (int32_t i = 0; i < n_req; ++i) h->m->check_prefill_rows(slots[i], kv_len[i]);
    vattn::launch_prefill_varlen(v, q, out, h->m->hq_local(), n_req, q_start, n_q, slots, kv_len, scale,
                                 causal != 0, (cudaStream_t)stream);
    h->m->mark_use((cudaStream_t)stream, false);
  });
}

vattn_status vattn_prefill_rotary(vattn_t* h, int32_t layer, const void* q, void* out, int32_t n_q,
                                  int32_t slot, int32_t kv_len, float scale, int32_t causal,
                                  const vattn_rotary* rotary, void* stream) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] {
    if (!rotary) throw Fail(VATTN_VALUE_ERROR, "null rotary descriptor");
    vattn::Nvtx nv("vattn.prefill");
    h->m->check_device_errors();
    const vattn::CacheView v = h->m->layer_view(layer);
    const vattn::Rotary rot{rotary->cos, rotary->sin, rotary->rotary_dim, rotary->interleaved};
    h->m->check_prefill_rows(slot, kv_len);
    vattn::launch_prefill(h->m->ks, layer, v, q, out, n_q, h->m->hq_local(), slot, kv_len, scale,
                          causal != 0, (cudaStream_t)stream, &rot);
    h->m->mark_use((cudaStream_t)stream, false);
  });
}

vattn_status vattn_decode_append_rotary(vattn_t* h, int32_t layer, const void* q, const void* k_new,
                                        const void* v_new, void* out, int32_t batch,
                                        const int32_t* cache_seqlens, const int32_t* batch_idx, float scale,
                                        int32_t num_splits, const vattn_rotary* rotary, void* stream) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] {
    if (!rotary) throw Fail(VATTN_VALUE_ERROR, "null rotary descriptor");
    h->m->check_decode_tiling();
    vattn::set_decode_order_hint(h->m->mixed_lengths() ? 1 : 0);
    vattn::Nvtx nv("vattn.decode_append");
    h->m->check_device_errors();
    const vattn::CacheView v = h->m->layer_view(layer);
    const int hq = h->m->hq_local();
    int64_t ws_bytes = 0;
    void* ws = decode_workspace(h, (cudaStream_t)stream, vattn_decode_workspace_bytes(batch, hq, v.d, 0),
                                vattn_decode_workspace_bytes(h->m->max_batch(), hq, v.d, 0), &ws_bytes);
    const vattn::Rotary rot{rotary->cos, rotary->sin, rotary->rotary_dim, rotary->interleaved};
    decode_pdl_hint(h, (cudaStream_t)stream, layer, k_new != nullptr);
    vattn::launch_decode(h->m->ks, layer, v, q, out, batch, hq, cache_seqlens, batch_idx, scale, num_splits,
                         ws, ws_bytes, (cudaStream_t)stream, k_new, v_new, nullptr, &rot);
    h->m->mark_use((cudaStream_t)stream, false);
  });
}

vattn_status vattn_decode_gather(vattn_t* h, int32_t layer, const void* q, const void* k_new,
                                 const void* v_new, vattn_gather_t* g, int32_t batch,
                                 const int32_t* cache_seqlens, const int32_t* batch_idx, float scale,
                                 int32_t num_splits, void* stream) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] {
    h->m->check_decode_tiling();
    vattn::set_decode_order_hint(h->m->mixed_lengths() ? 1 : 0);
    vattn::Nvtx nv("vattn.decode_gather");
    h->m->check_device_errors();
    const vattn::CacheView v = h->m->layer_view(layer);
    const int hq = h->m->hq_local();
    int64_t ws_bytes = 0;
    void* ws = decode_workspace(h, (cudaStream_t)stream, vattn_decode_workspace_bytes(batch, hq, v.d, 0),
                                vattn_decode_workspace_bytes(h->m->max_batch(), hq, v.d, 0), &ws_bytes);
    const vattn::GatherSink s = vattn::gather_sink(g, hq, batch, v.d);
    decode_pdl_hint(h, (cudaStream_t)stream, layer, k_new != nullptr);
    vattn::launch_decode(h->m->ks, layer, v, q, nullptr, batch, hq, cache_seqlens, batch_idx, scale,
                         num_splits, ws, ws_bytes, (cudaStream_t)stream, k_new, v_new, &s);
    h->m->mark_use((cudaStream_t)stream, false);
  });
}

vattn_status vattn_prefill(vattn_t* h, int32_t layer, const void* q, void* out, int32_t n_q,
                           int32_t slot, int32_t kv_len, float scale, int32_t causal,
                           void* stream) {
  if (!h || !h->m) { vattn::set_last_error("null handle"); return VATTN_BAD_STATE; }
  return guard([&] {
    vattn::Nvtx nv("vattn.prefill");
    h->m->check_device_errors();
    const vattn::CacheView v = h->m->layer_view(layer);
    h->m->check_prefill_rows(slot, kv_len);
    vattn::launch_prefill(h->m->ks, layer, v, q, out, n_q, h->m->hq_local(), slot, kv_len, scale,
                          causal != 0, (cudaStream_t)stream);
    h->m->mark_use((cudaStream_t)stream, false);
  });
}


// Table 2 analog on the real driver: mean µs per call of every cuMem* API at `page_bytes`,
// plus cuMemSetAccess over runs of `run` contiguous pages (one call per run).
// out[0..7] = reserve, create, map, set_access(1 page), unmap, release, address_free,
//             set_access per page when batched over `run` pages.
vattn_status vattn_vmm_microbench(int32_t device, int64_t page_bytes, int32_t n_pages, int32_t run,
                                  double* out) {
  return guard([&] {
    using vattn::check_cu;
    const vattn::Driver& d = vattn::driver();
    vattn::check_rt(cudaSetDevice(device), "cudaSetDevice");
    vattn::check_rt(cudaFree(nullptr), "context init");
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    CUmemAccessDesc acc{};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (n_pages < 1 || run < 1 || n_pages % run) throw Fail(VATTN_VALUE_ERROR, "n_pages must be a multiple of run");
    const size_t pg = (size_t)page_bytes, total = pg * (size_t)n_pages;
    std::vector<CUmemGenericAllocationHandle> h((size_t)n_pages);
    double t0 = vattn::now_us();
    CUdeviceptr va = 0;
    check_cu(d.MemAddressReserve(&va, total, pg, 0, 0), "cuMemAddressReserve");
    out[0] = vattn::now_us() - t0;
    t0 = vattn::now_us();
    for (auto& x : h) check_cu(d.MemCreate(&x, pg, &prop, 0), "cuMemCreate");
    out[1] = (vattn::now_us() - t0) / n_pages;
    t0 = vattn::now_us();
    for (int i = 0; i < n_pages; ++i) check_cu(d.MemMap(va + i * pg, pg, 0, h[i], 0), "cuMemMap");
    out[2] = (vattn::now_us() - t0) / n_pages;
    t0 = vattn::now_us();
    for (int i = 0; i < n_pages; ++i) check_cu(d.MemSetAccess(va + i * pg, pg, &acc, 1), "cuMemSetAccess");
    out[3] = (vattn::now_us() - t0) / n_pages;
    t0 = vattn::now_us();
    for (int i = 0; i < n_pages; ++i) check_cu(d.MemUnmap(va + i * pg, pg), "cuMemUnmap");
    out[4] = (vattn::now_us() - t0) / n_pages;
    // batched access: map again, one cuMemSetAccess per run of `run` pages
    for (int i = 0; i < n_pages; ++i) check_cu(d.MemMap(va + i * pg, pg, 0, h[i], 0), "cuMemMap");
    t0 = vattn::now_us();
    for (int i = 0; i < n_pages; i += run) check_cu(d.MemSetAccess(va + i * pg, pg * run, &acc, 1), "cuMemSetAccess(run)");
    out[7] = (vattn::now_us() - t0) / n_pages;
    for (int i = 0; i < n_pages; ++i) check_cu(d.MemUnmap(va + i * pg, pg), "cuMemUnmap");
    // recycled handles: map the same physical pages again at shifted slots
    t0 = vattn::now_us();
    for (int i = 0; i < n_pages; ++i) check_cu(d.MemMap(va + ((i + 1) % n_pages) * pg, pg, 0, h[i], 0), "cuMemMap(re)");
    out[8] = (vattn::now_us() - t0) / n_pages;
    t0 = vattn::now_us();
    for (int i = 0; i < n_pages; ++i) check_cu(d.MemSetAccess(va + i * pg, pg, &acc, 1), "cuMemSetAccess(re)");
    out[9] = (vattn::now_us() - t0) / n_pages;
    for (int i = 0; i < n_pages; ++i) check_cu(d.MemUnmap(va + i * pg, pg), "cuMemUnmap");
    t0 = vattn::now_us();
    for (auto& x : h) check_cu(d.MemRelease(x), "cuMemRelease");
    out[5] = (vattn::now_us() - t0) / n_pages;
    t0 = vattn::now_us();
    check_cu(d.MemAddressFree(va, total), "cuMemAddressFree");
    out[6] = vattn::now_us() - t0;
  });
}


// Probe: map+SetAccess+unmap cost of `n_pages` 2 MiB slices when the physical memory comes
// from one big handle (cuMemMap offset) vs one handle per slice, with `extra_handles` other
// live allocations in the context.  out[0..2] = per-slice map, set_access, unmap µs.
vattn_status vattn_vmm_slice_probe(int32_t device, int32_t n_pages, int32_t big_handle,
                                   int32_t extra_handles, double* out) {
  return guard([&] {
    using vattn::check_cu;
    const vattn::Driver& d = vattn::driver();
    vattn::check_rt(cudaSetDevice(device), "cudaSetDevice");
    vattn::check_rt(cudaFree(nullptr), "context init");
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    CUmemAccessDesc acc{};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    const size_t pg = 2u << 20;
    // `extra_handles` other live 2 MiB allocations, mapped and accessible (a populated cache)
    std::vector<CUmemGenericAllocationHandle> extra((size_t)extra_handles);
    CUdeviceptr xva = 0;
    if (extra_handles > 0) check_cu(d.MemAddressReserve(&xva, pg * extra_handles, pg, 0, 0), "reserve(extra)");
    for (int i = 0; i < extra_handles; ++i) {
      check_cu(d.MemCreate(&extra[i], pg, &prop, 0), "cuMemCreate(extra)");
      check_cu(d.MemMap(xva + (size_t)i * pg, pg, 0, extra[i], 0), "cuMemMap(extra)");
    }
    if (extra_handles > 0) check_cu(d.MemSetAccess(xva, pg * extra_handles, &acc, 1), "cuMemSetAccess(extra)");
    std::vector<CUmemGenericAllocationHandle> h;
    if (big_handle) {
      h.resize(1);
      check_cu(d.MemCreate(&h[0], pg * n_pages, &prop, 0), "cuMemCreate(big)");
    } else {
      h.resize((size_t)n_pages);
      for (auto& x : h) check_cu(d.MemCreate(&x, pg, &prop, 0), "cuMemCreate");
    }
    CUdeviceptr va = 0;
    check_cu(d.MemAddressReserve(&va, pg * n_pages * 2, pg, 0, 0), "reserve");
    double tm = 0, ta = 0, tu = 0;
    for (int rep = 0; rep < 2; ++rep) {
      double t0 = vattn::now_us();
      for (int i = 0; i < n_pages; ++i) {
        const CUdeviceptr p = va + (size_t)(2 * i + rep) * pg;   // non-contiguous slots
        if (big_handle) check_cu(d.MemMap(p, pg, pg * i, h[0], 0), "cuMemMap(slice)");
        else check_cu(d.MemMap(p, pg, 0, h[i], 0), "cuMemMap");
      }
      tm += vattn::now_us() - t0;
      t0 = vattn::now_us();
      for (int i = 0; i < n_pages; ++i)
        check_cu(d.MemSetAccess(va + (size_t)(2 * i + rep) * pg, pg, &acc, 1), "cuMemSetAccess");
      ta += vattn::now_us() - t0;
      t0 = vattn::now_us();
      for (int i = 0; i < n_pages; ++i) check_cu(d.MemUnmap(va + (size_t)(2 * i + rep) * pg, pg), "cuMemUnmap");
      tu += vattn::now_us() - t0;
    }
    out[0] = tm / (2.0 * n_pages);
    out[1] = ta / (2.0 * n_pages);
    out[2] = tu / (2.0 * n_pages);
    d.MemAddressFree(va, pg * n_pages * 2);
    for (auto x : h) d.MemRelease(x);
    for (int i = 0; i < extra_handles; ++i) d.MemUnmap(xva + (size_t)i * pg, pg);
    for (auto x : extra) d.MemRelease(x);
    if (extra_handles > 0) d.MemAddressFree(xva, pg * extra_handles);
  });
}


// Probe: wall time to map + set access `n_pages` 2 MiB pages (fresh handles) using `n_threads`
// threads concurrently (out[0] = µs per page, out[1] = total ms), then unmap (out[2] µs/page).
vattn_status vattn_vmm_parallel_probe(int32_t device, int32_t n_pages, int32_t n_threads, double* out) {
  return guard([&] {
    using vattn::check_cu;
    const vattn::Driver& d = vattn::driver();
    vattn::check_rt(cudaSetDevice(device), "cudaSetDevice");
    vattn::check_rt(cudaFree(nullptr), "context init");
    CUcontext ctx = nullptr;
    check_cu(d.CtxGetCurrent(&ctx), "ctx");
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    CUmemAccessDesc acc{};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    const size_t pg = 2u << 20;
    std::vector<CUmemGenericAllocationHandle> h((size_t)n_pages);
    for (auto& x : h) check_cu(d.MemCreate(&x, pg, &prop, 0), "cuMemCreate");
    CUdeviceptr va = 0;
    check_cu(d.MemAddressReserve(&va, pg * n_pages * 2, pg, 0, 0), "reserve");
    auto work = [&](int t) {
      d.CtxSetCurrent(ctx);
      for (int i = t; i < n_pages; i += n_threads) {
        const CUdeviceptr p = va + (size_t)(2 * i) * pg;
        if (d.MemMap(p, pg, 0, h[i], 0) != CUDA_SUCCESS) return;
        d.MemSetAccess(p, pg, &acc, 1);
      }
    };
    double t0 = vattn::now_us();
    std::vector<std::thread> th;
    for (int t = 0; t < n_threads; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
    out[1] = (vattn::now_us() - t0) / 1e3;
    out[0] = out[1] * 1e3 / n_pages;
    t0 = vattn::now_us();
    for (int i = 0; i < n_pages; ++i) d.MemUnmap(va + (size_t)(2 * i) * pg, pg);
    out[2] = (vattn::now_us() - t0) / n_pages;
    d.MemAddressFree(va, pg * n_pages * 2);
    for (auto x : h) d.MemRelease(x);
  });
}

}  // extern "C"
