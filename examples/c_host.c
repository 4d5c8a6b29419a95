/* A C host driving the vAttention allocator through the C ABI (include/vattn.h) — what a
 * non-Python integration of the reference's KVCacheManager API (kvsim/manager.py:84-372) binds.
 * Shadow backend (bookkeeping only, no GPU), so it runs anywhere:
 *   gcc -std=c11 -I include examples/c_host.c -L paper_2405_04437_b200/_lib -lvattn \
 *       -Wl,-rpath,$PWD/paper_2405_04437_b200/_lib -o c_host && ./c_host
 * Prints one line per call; tests/test_c_abi_host.py replays the same calls through the Python
 * facade and compares. */
#include <stdio.h>
#include <string.h>

#include "vattn.h"

#define CHECK(x)                                                           \
  do {                                                                     \
    vattn_status s_ = (x);                                                 \
    if (s_ != VATTN_OK) {                                                  \
      printf("error %d %s: %s\n", (int)s_, #x, vattn_last_error());        \
      return 1;                                                            \
    }                                                                      \
  } while (0)

int main(void) {
  vattn_config c;
  memset(&c, 0, sizeof c);
  c.n_layers = 2; c.kv_heads_total = 2; c.head_dim = 64; c.bytes_per_elem = 2; c.tp_degree = 1;
  c.max_context = 8192; c.max_batch = 4;
  c.page_group_size = 64 * 1024; c.pool_bytes = 64ll << 20;
  c.reclaim_threshold = 0.1; c.pre_create_fraction = 1.0; c.eager_groups = 2;
  c.backend = VATTN_BACKEND_SHADOW; c.log_events = 1; c.batch_set_access = 1;
  vattn_t* h = NULL;
  CHECK(vattn_create(&c, &h));
  int32_t r0, r1, r2, r3;
  CHECK(vattn_alloc_reqid(h, &r0));
  CHECK(vattn_alloc_reqid(h, &r1));
  CHECK(vattn_alloc_reqid(h, &r2));
  printf("alloc %d %d %d\n", r0, r1, r2);
  int64_t seq[4] = {0, 0, 0, 0};
  seq[r0] = 1000; seq[r1] = 3000; seq[r2] = 10;
  vattn_step_result sr;
  CHECK(vattn_step(h, seq, 4, &sr));
  printf("step %d %.3f\n", sr.ok, sr.sync_us);
  CHECK(vattn_free_reqid(h, r1));
  seq[r1] = 0;
  double us = 0;
  CHECK(vattn_eager_prepare(h, -1, &us));
  printf("eager %.3f\n", us);
  CHECK(vattn_alloc_reqid(h, &r3));
  printf("realloc %d\n", r3);
  seq[r3] = 500; seq[r0] = 1001; seq[r2] = 11;
  CHECK(vattn_step(h, seq, 4, &sr));
  printf("step %d %.3f\n", sr.ok, sr.sync_us);
  int64_t freed = 0;
  CHECK(vattn_reclaim(h, &freed, &us));
  printf("reclaim %lld %.3f\n", (long long)freed, us);
  vattn_counters k;
  CHECK(vattn_counters_get(h, &k));
  printf("counters %lld %lld %lld %lld\n", (long long)k.created, (long long)k.mapped,
         (long long)k.total_mapped_bytes, (long long)k.eager_slot);
  CHECK(vattn_free_reqid(h, r3));
  int32_t st = vattn_free_reqid(h, r3);   /* already free: DoubleFreeError */
  printf("double_free %d\n", (int)st);
  CHECK(vattn_destroy(h));
  return 0;
}
