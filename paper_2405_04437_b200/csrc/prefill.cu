// tcgen05/TMEM causal prefill attention (placeholder until the tcgen05 kernel lands).
#include "internal.h"

namespace vattn {
void launch_prefill(KernelState*, int, const CacheView&, const void*, void*, int, int, int, int,
                    float, bool, cudaStream_t) {
  throw Fail(VATTN_UNSUPPORTED, "prefill kernel not built yet");
}
}  // namespace vattn

extern "C" vattn_status vattn_prefill_raw(const vattn_cache_desc*, const void*, void*, int32_t,
                                          int32_t, int32_t, int32_t, float, int32_t, void*) {
  vattn::set_last_error("prefill kernel not built yet");
  return VATTN_UNSUPPORTED;
}
