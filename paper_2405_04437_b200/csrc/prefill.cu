// Causal prefill attention on 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// One CTA = one query head x 256 query rows, split into two 128-row tiles A and B that
// ping-pong (FA4-style): while the softmax warpgroup of tile A turns S_A = Q_A·Kᵀ into P_A, the
// tensor core works on tile B, and vice versa.  Everything that is a contraction runs on
// tcgen05.mma with fp32 accumulators in TMEM:
//   S_X(j)  = Q_X · K_jᵀ      A = Q (smem, K-major), B = K_j (smem, K-major), D = TMEM
//   O_X    += P_X(j) · V_j    A = P (TMEM, bf16, aliased on S_X), B = V_j (smem, MN-major)
// K/V tiles of 128 tokens are read straight out of the request's slot of the virtual KV cache
// by TMA (4-D map over [D, Hkv, tokens, slots]; no block table).  The online softmax keeps one
// query row per thread (TMEM lane), so row max / row sum need no shuffles; the O rescale is
// lazy (only when the running max grows by more than 2^8).
//
// Warp roles (320 threads): warps 0-3 softmax A, 4-7 softmax B, 8 TMA producer, 9 MMA issuer
// (+ TMEM allocator).  TMEM: S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512) columns.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <vector>
#include <cmath>
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"
#include "vattn.h"

namespace vattn {
namespace pf {

constexpr int kBM = 128;           // query rows per tile
constexpr int kBN = 128;           // keys per KV tile
constexpr int kD = 128;            // head dim (Yi-6B / Llama / Yi-34B)
constexpr int kStages = 2;         // V ring depth
constexpr int kKStages = 3;        // K ring depth: K runs one tile ahead of V, each stage released
                                   // after its own last MMA (K: both S; V: both PV).  Measured +1.5 %
                                   // (16K) over a shared 2-deep K/V ring (tools/pf_var_ab.py)
constexpr int kThreads = 320;
constexpr int kHalf = kBN * 128;               // one 64-column half of a 128-row tile (16 KB)
constexpr float kRescaleThreshold = 8.0f;      // log2 domain: rescale O when max grows > 2^8

// Shared-memory layout for head dim D (64 or 128): every 128-row tile is D/64 swizzled 64-column
// halves of 16 KB.
template <int D, int KS = kKStages>
struct PfL {
  static constexpr int kTile = (D / 64) * kHalf;
  static constexpr int kKS = KS;                                // K ring depth
  static constexpr int kQOff = 0;                               // Q_A, Q_B
  static constexpr int kKOff = 2 * kTile;                       // K stages
  static constexpr int kVOff = kKOff + KS * kTile;
  static constexpr int kBarOff = kVOff + kStages * kTile;
  static constexpr int kSmem = kBarOff + 256 + 1024;
};

struct Params {
  __nv_bfloat16* out;      // [n_q, hq, D]
  int n_q, hq, group, kv_len, slot, n_pairs;
  int q_off;               // kv_len - n_q  (bottom-right causal alignment)
  int causal;
  float scale_log2;
  // paged comparison variant: K/V tiles gathered block by block through a block table
  const int32_t* block_table;
  int block_size, box_tokens;
  // rotary of the query rows at their absolute positions q_off + i (k is rotated at append)
  const float* rot_cos;
  const float* rot_sin;
  int rot_dim, rot_inter;
  // varlen (several requests per launch): blockIdx.x indexes work = (request, pair), requests
  // hold (first packed query row, n_q, kv_len), maps hold each request's K and V tensor maps
  const int4* work;
  const int4* reqs;
  const CUtensorMap* maps;
  // grid order: 1 = heads vary fastest (blockIdx.x = head, blockIdx.y = work item), so the
  // hardware's linear CTA order is heaviest-first across ALL heads and the CTAs of one GQA group
  // read the same K/V tiles at the same time; 0 = work items fastest (per-head heaviest-first)
  int head_fast;
  // head pairs (single-request kernel): tile A / B = the same 128 query rows of two query heads
  // of one GQA group (2h, 2h+1) instead of two consecutive row tiles of one head.  Both tiles
  // then need the same K/V tiles (equal step counts: no lone last step on the causal diagonal)
  // and a prompt of <= 128 rows fills both tiles.  n_pairs counts 128-row tiles in this mode.
  int head_pair;
  // early PV (prefill_kernel): the softmax releases keys 0..63 of P once stored, and the issuer
  // starts their PV MMAs while keys 64..127 are exponentiated.  1 always, 0 never, -1 in CTAs
  // that run a single tile (tools/pf_earlypv_ab.py)
  int early_pv;
  // split-KV (single-request kernel, small grids): blockIdx.z = split; each CTA runs its tiles'
  // KV range [j0, j0 + T) and writes fp32 O / l and lse = m + log2(l) (log2 domain) per row and
  // split into part_o [n_q * hq][splits][D] / part_lse [n_q * hq][splits]; the decode combine
  // kernel merges them (kv_splits <= 1: plain bf16 output)
  int kv_splits;
  float* part_o;
  float* part_lse;
};

static int head_fast_order() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("VATTN_PF_HEAD_FAST");
    v = e ? (atoi(e) != 0) : 1;
  }
  return v;
}
static dim3 pf_grid(Params& p, unsigned n_work, unsigned hq) {
  p.head_fast = head_fast_order();
  return p.head_fast ? dim3(hq, n_work) : dim3(n_work, hq);
}

// ---- tcgen05 wrappers -------------------------------------------------------------------
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // SM100 UMMA shared-memory descriptor, SWIZZLE_128B, version 1 (cute UMMA::SmemDescriptor)
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor, kind::f16: bf16 x bf16 -> f32, M=128, N=128
__host__ __device__ constexpr uint32_t idesc(bool b_mn_major, int n = 128) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) |
         ((kBM >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   ptx::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

#define TMEM_LD32(taddr, r)                                                                            \
  asm volatile(                                                                                        \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                       \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),           \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),       \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),    \
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),    \
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                            \
      : "r"(taddr))

#define TMEM_ST32(taddr, r)                                                                             \
  asm volatile(                                                                                         \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"   \
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),         \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),          \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),    \
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),  \
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) \
      : "memory")

#define TMEM_ST16(taddr, r)                                                                             \
  asm volatile(                                                                                         \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"   \
      "%15,%16};" ::"r"(taddr),                                                                         \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),          \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])     \
      : "memory")

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 2^x on the FMA pipe (FA4-style MUFU offload): round-to-nearest via the 1.5·2^23 magic add,
// degree-3 polynomial on [-0.5, 0.5] (max rel. err 2.2e-4, far below bf16's 3.9e-3), exponent
// via integer add.  Inputs below -127 flush to ~0 (masked entries are zeroed explicitly).
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 n = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-n.x, -n.y));
  float2 q = __ffma2_rn(f, make_float2(0.05286731580314504f, 0.05286731580314504f),
                        make_float2(0.2421521458456525f, 0.2421521458456525f));
  q = __ffma2_rn(q, f, make_float2(0.6935868335103712f, 0.6935868335103712f));
  q = __ffma2_rn(q, f, make_float2(0.9999627473381362f, 0.9999627473381362f));
  const int ex = (__float_as_int(t.x) - 0x4B400000) << 23;
  const int ey = (__float_as_int(t.y) - 0x4B400000) << 23;
  return make_float2(__int_as_float(__float_as_int(q.x) + ex), __int_as_float(__float_as_int(q.y) + ey));
}

__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// Pass 2 of the online softmax for one 128-column S row: P = exp2(S*scale - m) packed to bf16
// and stored over the S columns already consumed; returns the (pairwise) row sum.  MASK=false
// (all but the diagonal/tail tiles) carries no per-element compare/select.
template <bool MASK, int POLY>
__device__ __forceinline__ float2 softmax_p_pass(uint32_t tS, float2 sc2, float2 nm2, int lim) {
  float2 acc2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int c0 = 0; c0 < kBN; c0 += 32) {
    uint32_t r[32], pk[16];
    TMEM_LD32(tS + c0, r);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < 32; c += 2) {
      const float2 x = __ffma2_rn(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), sc2, nm2);
      float p0, p1;
      if (((c / 2) & 3) < POLY) {       // this share of the exps runs on the FMA pipe
        const float2 e = exp2_poly2(x);
        p0 = e.x;
        p1 = e.y;
      } else {
        p0 = ptx::fast_exp2(x.x);
        p1 = ptx::fast_exp2(x.y);
      }
      if (MASK) {
        p0 = (c0 + c < lim) ? p0 : 0.f;
        p1 = (c0 + c + 1 < lim) ? p1 : 0.f;
      }
      acc2 = __fadd2_rn(acc2, make_float2(p0, p1));
      pk[c / 2] = ptx::pack_bf16(p0, p1);
    }
    TMEM_ST16(tS + c0 / 2, pk);
  }
  return acc2;
}

#ifdef VATTN_PF_TRACE
// debug timeline of CTA (0, 0): [role][j][event] clock64 stamps (build with -DVATTN_PF_TRACE)
__device__ unsigned long long g_pf_trace[4][160][8];
// per-CTA record of the last traced launch: [globaltimer start, end, smid, kv tiles]
// [0] start (work item known), [1] end of work, [2] smid, [3] kv tiles, [4] kernel entry,
// [5] prologue done (barriers, TMEM), [6] TMEM released (exit)
__device__ unsigned long long g_pf_cta[8192][12];
__device__ __forceinline__ unsigned long long pf_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long pf_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
#define PF_TRACE(role, j, ev) \
  if (blockIdx.x == 0 && blockIdx.y == 0 && (j) < 160) g_pf_trace[role][j][ev] = pf_clock()
#else
#define PF_TRACE(role, j, ev)
#endif

// Half a row (64 keys at TMEM columns [tS, tS+64)): P = exp2(S*scale - m) packed into pk[32],
// row max of the raw scores into m3, pairwise sum into acc.
template <int POLY>
__device__ __forceinline__ void softmax_half(uint32_t tS, float2 sc2, float2 nm2, uint32_t* pk, float& m3,
                                             float2& acc) {
#pragma unroll
  for (int c0 = 0; c0 < 64; c0 += 32) {
    uint32_t r[32];
    TMEM_LD32(tS + c0, r);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < 32; c += 2) {
      m3 = max3(m3, __uint_as_float(r[c]), __uint_as_float(r[c + 1]));
      const float2 xx = __ffma2_rn(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), sc2, nm2);
      float p0, p1;
      if (((c / 2) & 3) < POLY) {
        const float2 e = exp2_poly2(xx);
        p0 = e.x;
        p1 = e.y;
      } else {
        p0 = ptx::fast_exp2(xx.x);
        p1 = ptx::fast_exp2(xx.y);
      }
      acc = __fadd2_rn(acc, make_float2(p0, p1));
      pk[(c0 + c) / 2] = ptx::pack_bf16(p0, p1);
    }
  }
}

// number of KV tiles a query tile starting at row q0 needs
__device__ __forceinline__ int kv_tiles_for(const Params& p, int q0) {
  if (q0 >= p.n_q) return 0;
  int last_key = p.kv_len - 1;
  if (p.causal) {
    const int q_last = min(q0 + kBM, p.n_q) - 1;
    last_key = min(last_key, q_last + p.q_off);
  }
  if (last_key < 0) return 0;
  return last_key / kBN + 1;
}

// Arrive on a barrier of the CTA pair's leader (rank 0) when PAIR, else on the local one.
template <bool PAIR>
__device__ __forceinline__ void arrive_lead(uint64_t* bar) {
  if constexpr (PAIR) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(a) : "r"(ptx::smem_u32(bar)));
    // default (.release.cta) semantics, as CUTLASS's umma_arrive_2x1SM_sm0: the P columns are
    // ordered by tcgen05.wait::st + fence::before_thread_sync, and the leader's MMA reads them
    // through the tensor core; a .cluster-scope release costs ~1000 cycles per arrival here
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
  } else {
    ptx::mbar_arrive(bar);
  }
}

// ===================== softmax warpgroups (A: warps 0-3, B: warps 4-7) =====================
// One query row per thread (TMEM lane); used by the single-CTA kernel and by both CTAs of the
// pair kernel (PAIR: P-ready / Q-ready arrivals go to the leader's barriers).
// Persistent kernel (o_free != nullptr): s_full / o_final phases continue across work items
// (s_base = tiles this Q tile ran before this item, o_par = items with tiles before it), O goes
// out with direct stores (the Q buffer may already hold the next item's Q), and o_free is
// arrived once O has been read out of TMEM so the next item's first PV may overwrite it.
template <int POLY, int D, bool VARLEN, bool PAIR, class L>
__device__ __forceinline__ void softmax_role(const Params& p, uint8_t* smem, uint64_t* s_full, uint64_t* p_full,
                                             uint64_t* o_final, uint64_t* q_full, uint64_t* q_ready, uint32_t tmem,
                                             int warp, int lane, int head, int q_row0, int q0A, int q0B, int nA,
                                             int nB, int n_kv, const CUtensorMap& omap, uint32_t s_base = 0,
                                             uint32_t o_par = 0, uint64_t* o_free = nullptr, int headB = -1,
                                             uint64_t* p_lo = nullptr, uint64_t* pv_lo = nullptr, int j0 = 0) {
  const int x = warp / 4;
  const int row = (warp % 4) * 32 + lane;          // TMEM lane == row of the query tile
  const int q0 = x == 0 ? q0A : q0B;
  const int n = x == 0 ? nA : nB;
  const int qpos = q0 + row;
  const uint32_t lane_base = tmem + (((warp % 4) * 32) << 16);
  const uint32_t tS = lane_base + x * 128;
  const uint32_t tO = lane_base + 256 + x * D;
  float m_run = -INFINITY, l_run = 0.f;
  if (p.rot_cos && n_kv > 0) {
    // rotary: each thread rotates its own query row of tile x in the swizzled smem tile, then
    // hands the tiles to the async proxy (tcgen05.mma reads Q from smem) and signals the issuer
    ptx::mbar_wait(q_full, 0);
    if (qpos < p.n_q) {
      const uint32_t qt = ptx::smem_u32(smem + L::kQOff + x * L::kTile);
      const int64_t t = (int64_t)(qpos + p.q_off) * (p.rot_dim / 2);
      const int nch = p.rot_dim / 8, half = p.rot_dim / 16;
      for (int cc = 0; cc < nch; ++cc) {
        if (!p.rot_inter && cc >= half) break;     // NeoX: the first-half chunk rotates both
        const int pc = p.rot_inter ? cc : cc + half;
        const uint32_t a0 = ptx::swz128(qt + (cc >> 3) * kHalf, row, cc & 7);
        const uint32_t a1 = ptx::swz128(qt + (pc >> 3) * kHalf, row, pc & 7);
        uint4 v0, v1;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v0.x), "=r"(v0.y), "=r"(v0.z), "=r"(v0.w) : "r"(a0));
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v1.x), "=r"(v1.y), "=r"(v1.z), "=r"(v1.w) : "r"(a1));
        const uint4 r0 = ptx::rotary_chunk(v0, v1, cc, p.rot_cos + t, p.rot_sin + t, p.rot_dim, p.rot_inter != 0);
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a0), "r"(r0.x), "r"(r0.y), "r"(r0.z), "r"(r0.w));
        if (!p.rot_inter) {
          const uint4 r1 = ptx::rotary_chunk(v1, v0, pc, p.rot_cos + t, p.rot_sin + t, p.rot_dim, false);
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a1), "r"(r1.x), "r"(r1.y), "r"(r1.z), "r"(r1.w));
        }
      }
    }
    ptx::fence_proxy_async();
    arrive_lead<PAIR>(q_ready);
  }
  for (int j = 0; j < n; ++j) {
    if (lane == 0 && (warp % 4) == 0) PF_TRACE(x, j, 0);
    ptx::mbar_wait(&s_full[x], (s_base + j) & 1);
    if (lane == 0 && (warp % 4) == 0) PF_TRACE(x, j, 1);
    fence_after();
    // pass 1: row max (chunks of 32 columns keep register pressure low; TMEM reads are cheap).
    // Only diagonal / tail tiles need the per-element mask; the others take the plain path.
    const int k0 = (j0 + j) * kBN;
    const bool need_mask = (k0 + kBN > p.kv_len) || (p.causal && k0 + kBN - 1 > qpos + p.q_off);
    const int lim = need_mask ? min(p.kv_len, p.causal ? qpos + p.q_off + 1 : p.kv_len) - k0 : kBN;
    const bool warp_mask = __any_sync(0xffffffffu, need_mask);
    if (!warp_mask && m_run != -INFINITY) {
      // Single pass (common case): exponentiate against the running max while tracking the
      // row max, half a row (64 keys) at a time; each half's P is stored only once its keys
      // are known not to raise the max by more than 2^8 (then the stale max is kept, as the
      // lazy rescale would).  S columns a half still needs are never overwritten early.
      const float2 sc2f = make_float2(p.scale_log2, p.scale_log2);
      const float2 nm2f = make_float2(-m_run, -m_run);
      float m_lo = -INFINITY;
      float2 acc_lo = make_float2(0.f, 0.f);
      uint32_t pk[32];
      softmax_half<POLY>(tS + 0, sc2f, nm2f, pk, m_lo, acc_lo);
      if (!__any_sync(0xffffffffu, m_lo * p.scale_log2 > m_run + kRescaleThreshold)) {
        TMEM_ST16(tS + 0, pk);
        TMEM_ST16(tS + 16, (pk + 16));
        if (p_lo) {   // early PV: keys 0..63 of P go to the tensor core while keys 64..127 run
          tmem_wait_st();
          fence_before();
          arrive_lead<PAIR>(&p_lo[x]);
        }
        float m_hi = -INFINITY;
        float2 acc_hi = make_float2(0.f, 0.f);
        softmax_half<POLY>(tS + 64, sc2f, nm2f, pk, m_hi, acc_hi);
        const float mx_hi = m_hi * p.scale_log2;
        if (!__any_sync(0xffffffffu, mx_hi > m_run + kRescaleThreshold)) {
          TMEM_ST16(tS + 32, pk);
          TMEM_ST16(tS + 48, (pk + 16));
          l_run += (acc_lo.x + acc_lo.y) + (acc_hi.x + acc_hi.y);
        } else {
          // rare: keys 64..127 raised the max.  Rescale O and l, rescale the stored P of keys
          // 0..63 in place, recompute keys 64..127 from S (intact) against the new max.
          const float m_new = fmaxf(m_run, fmaxf(mx_hi, m_lo * p.scale_log2));
          const float f = ptx::fast_exp2(m_run - m_new);
          if (p_lo) {
            // P_lo was released at the old max and may already be in O: let that PV retire,
            // then O (which holds it) is rescaled below like every earlier contribution
            ptx::mbar_wait(&pv_lo[x], (s_base + j) & 1);
            fence_after();
          }
          if (j > 0 || p_lo) {
#pragma unroll 1
            for (int c0 = 0; c0 < D; c0 += 32) {
              uint32_t o[32];
              TMEM_LD32(tO + c0, o);
              tmem_wait_ld();
#pragma unroll
              for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
              TMEM_ST32(tO + c0, o);
            }
          }
          if (!p_lo) {
            uint32_t pl[32];
            TMEM_LD32(tS + 0, pl);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&pl[c]);
              const float2 fv = __bfloat1622float2(v);
              pl[c] = ptx::pack_bf16(fv.x * f, fv.y * f);
            }
            TMEM_ST32(tS + 0, pl);
          }
          float m_dummy = -INFINITY;
          float2 acc_new = make_float2(0.f, 0.f);
          softmax_half<POLY>(tS + 64, sc2f, make_float2(-m_new, -m_new), pk, m_dummy, acc_new);
          TMEM_ST16(tS + 32, pk);
          TMEM_ST16(tS + 48, (pk + 16));
          l_run = l_run * f + (acc_lo.x + acc_lo.y) * f + (acc_new.x + acc_new.y);
          m_run = m_new;
        }
        tmem_wait_st();
        fence_before();
        arrive_lead<PAIR>(&p_full[x]);
        if (lane == 0 && (warp % 4) == 0) PF_TRACE(x, j, 2);
        continue;
      }
      // rare: the first half already raised the max: two-pass path below (nothing stored yet)
    }
    float mx = -INFINITY;
    if (!warp_mask) {
      float m3 = -INFINITY;
#pragma unroll
      for (int c0 = 0; c0 < kBN; c0 += 32) {
        uint32_t r[32];
        TMEM_LD32(tS + c0, r);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; c += 2) m3 = max3(m3, __uint_as_float(r[c]), __uint_as_float(r[c + 1]));
      }
      mx = m3 * p.scale_log2;     // scale > 0: max commutes with the scaling
    } else {
#pragma unroll
      for (int c0 = 0; c0 < kBN; c0 += 32) {
        uint32_t r[32];
        TMEM_LD32(tS + c0, r);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float v = (c0 + c < lim) ? __uint_as_float(r[c]) * p.scale_log2 : -INFINITY;
          mx = fmaxf(mx, v);
        }
      }
    }
    // lazy rescale: keep the stale max unless it grows by more than 2^8 (warp-uniform decision)
    const bool grow = (m_run == -INFINITY) ? (mx > -INFINITY) : (mx > m_run + kRescaleThreshold);
    if (__any_sync(0xffffffffu, grow)) {
      const float m_new = fmaxf(m_run, mx);
      const float f = (m_run == -INFINITY) ? 0.f : ptx::fast_exp2(m_run - m_new);
      l_run *= f;
      if (j > 0 && __any_sync(0xffffffffu, f != 1.f)) {
        // O_x(j-1) is complete: S_x(j) was issued after PV_x(j-1) and has retired
#pragma unroll 1
        for (int c0 = 0; c0 < D; c0 += 32) {
          uint32_t o[32];
          TMEM_LD32(tO + c0, o);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
          TMEM_ST32(tO + c0, o);
        }
        tmem_wait_st();
      }
      m_run = m_new;
    }
    // pass 2: P = exp2(S*scale - m) -> bf16 into TMEM over the S columns already consumed.
    // Packed f32x2 FMA/ADD (FFMA2/FADD2) halve the FMA-pipe instructions; MUFU does the exp2.
    const float neg_m = m_run == -INFINITY ? 0.f : -m_run;
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    const float2 nm2 = make_float2(neg_m, neg_m);
    const float2 acc2 = warp_mask ? softmax_p_pass<true, POLY>(tS, sc2, nm2, lim)
                                  : softmax_p_pass<false, POLY>(tS, sc2, nm2, lim);
    const float lsum = acc2.x + acc2.y;
    l_run += lsum;
    tmem_wait_st();
    fence_before();
    if (p_lo) arrive_lead<PAIR>(&p_lo[x]);   // both halves at once on this path
    arrive_lead<PAIR>(&p_full[x]);
    if (lane == 0 && (warp % 4) == 0) PF_TRACE(x, j, 2);
  }
  // ---- epilogue: O / l -> bf16 -> global ----
  if (n > 0) {
    ptx::mbar_wait(&o_final[x], o_par & 1);
    fence_after();
  }
  const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
  if (!VARLEN && o_free == nullptr && p.kv_splits > 1) {
    // split-KV partial of this row: O / l in fp32 and its log2-domain LSE (-inf: no keys here)
    // (tcgen05.ld is warp-collective: every lane loads, only rows < n_q store)
    const int hd = (x == 1 && headB >= 0) ? headB : head;
    const bool live_row = qpos < p.n_q;
    const int64_t prow = ((int64_t)(live_row ? qpos : 0) * p.hq + hd) * p.kv_splits + blockIdx.z;
    float* po = p.part_o + prow * D;
#pragma unroll 1
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t o[32];
      if (n > 0) {
        TMEM_LD32(tO + c0, o);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) o[c] = 0u;
      }
      if (live_row) {
#pragma unroll
        for (int c = 0; c < 32; c += 4)
          *reinterpret_cast<float4*>(po + c0 + c) =
              make_float4(__uint_as_float(o[c]) * inv, __uint_as_float(o[c + 1]) * inv,
                          __uint_as_float(o[c + 2]) * inv, __uint_as_float(o[c + 3]) * inv);
      }
    }
    if (live_row) p.part_lse[prow] = l_run > 0.f ? m_run + __log2f(l_run) : -INFINITY;
    return;
  }
  // Full tiles (and any tile of a single-request launch: the map clips rows >= n_q) go out
  // through shared memory and one TMA store: the tile's Q buffer is free once o_final landed
  // (every MMA reading it has retired), and whole 128-byte rows reach L2 instead of the
  // half-sector 16-byte stores of one row per thread.  Varlen tail tiles store directly so
  // they cannot spill into the next request's rows.  A tile that sees no keys (n == 0) also
  // stores its zeros directly: it never waited for its Q load, which may still be landing in
  // that buffer (found under compute-sanitizer's slowed timing).
  const bool via_tma = o_free == nullptr && n > 0 && (!VARLEN || q0 + kBM <= p.n_q);
  const uint32_t qt = ptx::smem_u32(smem + L::kQOff + x * L::kTile);
  const int hd = (x == 1 && headB >= 0) ? headB : head;   // head pairs: tile B is the odd head
  __nv_bfloat16* dst = p.out + ((int64_t)qpos * p.hq + hd) * D;
  const bool live = qpos < p.n_q;
#pragma unroll
  for (int c0 = 0; c0 < D; c0 += 32) {
    uint32_t o[32];
    if (n > 0) {
      TMEM_LD32(tO + c0, o);
      tmem_wait_ld();
      if (o_free != nullptr && c0 + 32 == D) {   // all of O read: the next item may overwrite it
        fence_before();
        ptx::mbar_arrive(&o_free[x]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < 32; ++c) o[c] = 0u;
    }
#pragma unroll
    for (int c = 0; c < 32; c += 8) {
      uint4 v;
      v.x = ptx::pack_bf16(__uint_as_float(o[c + 0]) * inv, __uint_as_float(o[c + 1]) * inv);
      v.y = ptx::pack_bf16(__uint_as_float(o[c + 2]) * inv, __uint_as_float(o[c + 3]) * inv);
      v.z = ptx::pack_bf16(__uint_as_float(o[c + 4]) * inv, __uint_as_float(o[c + 5]) * inv);
      v.w = ptx::pack_bf16(__uint_as_float(o[c + 6]) * inv, __uint_as_float(o[c + 7]) * inv);
      if (via_tma) {
        const int cc = (c0 + c) / 8;
        const uint32_t a = ptx::swz128(qt + (cc >> 3) * kHalf, row, cc & 7);
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
      } else if (live) {
        *reinterpret_cast<uint4*>(dst + c0 + c) = v;
      }
    }
  }
  if (via_tma) {
    ptx::fence_proxy_async();
    asm volatile("bar.sync %0, 128;" ::"r"(1 + x) : "memory");   // the 4 warps of tile x
    if (warp % 4 == 0 && lane == 0) {
#pragma unroll
      for (int h = 0; h < D / 64; ++h)
        ptx::tma_store_3d(&omap, smem + L::kQOff + x * L::kTile + h * kHalf, h * 64, hd, q_row0 + q0);
      ptx::tma_store_commit();
      ptx::tma_store_wait_read();
    }
  }
}

template <int POLY, bool PAGED = false, int D = 128, bool VARLEN = false>
__global__ void __launch_bounds__(kThreads, 1)
prefill_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
               const __grid_constant__ CUtensorMap vmap, const __grid_constant__ CUtensorMap omap, Params p) {
  // the paged comparison variant keeps one shared 2-deep K/V ring (K_j and V_j loaded together)
  constexpr int KS = PAGED ? kStages : kKStages;     // K ring depth
  constexpr bool SPLIT = !PAGED;                     // K / V stages released separately
  using L = PfL<D, KS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;            // [KS]
  uint64_t* v_full = bars + 5;            // [kStages]
  uint64_t* k_empty = bars + 7;           // [KS]; releases K and V together unless SPLIT
  uint64_t* v_empty = bars + 11;          // [kStages] (SPLIT only)
  uint64_t* s_full = bars + 13;           // [2] tiles A, B
  uint64_t* p_full = bars + 15;           // [2]
  uint64_t* o_final = bars + 17;          // [2]
  uint64_t* q_ready = bars + 19;          // rotary: both Q tiles rotated in shared memory
  uint64_t* p_lo = bars + 20;             // [2] early PV: keys 0..63 of P stored
  uint64_t* pv_lo = bars + 22;            // [2] early PV: the PV MMAs of keys 0..63 retired
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
#ifdef VATTN_PF_TRACE
  if (threadIdx.x == 0 && blockIdx.y * gridDim.x + blockIdx.x < 8192)
    g_pf_cta[blockIdx.y * gridDim.x + blockIdx.x][4] = pf_gtime();
#endif
  const int witem = p.head_fast ? blockIdx.y : blockIdx.x;
  int pair = p.n_pairs - 1 - witem;        // heaviest (latest) query rows first
  int q_row0 = 0;                          // packed row of this request's query row 0
  const CUtensorMap* kmp = &kmap;
  const CUtensorMap* vmp = &vmap;
  if constexpr (VARLEN) {                  // work list is sorted heaviest first on the host
    const int4 w = p.work[witem];
    const int4 r = p.reqs[w.x];
    pair = w.y;
    q_row0 = r.x;
    p.n_q = r.y;
    p.kv_len = r.z;
    p.q_off = r.z - r.y;
    p.out += (int64_t)r.x * p.hq * D;
    kmp = p.maps + 2 * w.x;
    vmp = kmp + 1;
  }
  const int hsel = p.head_fast ? blockIdx.x : blockIdx.y;
  const bool hp = p.head_pair != 0;
  const int head = hp ? 2 * hsel : hsel;   // tile A's head
  const int headB = hp ? head + 1 : head;  // tile B's head (same GQA group: group is even)
  const int kvh = head / p.group;
  const int q0A = hp ? pair * kBM : pair * 2 * kBM, q0B = hp ? q0A : q0A + kBM;
  int nA = kv_tiles_for(p, q0A), nB = kv_tiles_for(p, q0B);
  int j0 = 0;                              // split-KV: first KV tile of this CTA's range
  if (!VARLEN && !PAGED && p.kv_splits > 1) {
    const int per = (max(nA, nB) + p.kv_splits - 1) / p.kv_splits;
    j0 = blockIdx.z * per;
    nA = max(0, min(nA - j0, per));
    nB = max(0, min(nB - j0, per));
  }
  const int n_kv = max(nA, nB);
  // early PV pays only where a CTA runs one tile (no ping-pong partner to fill the tensor core
  // during the softmax): 128-row chunks over a 16K prefix 1.067x; with two tiles 0.98-1.00x
  const bool early = !PAGED && (p.early_pv > 0 || (p.early_pv < 0 && min(nA, nB) == 0));

#ifdef VATTN_PF_TRACE
  const int cta_lin = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0 && cta_lin < 8192) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_pf_cta[cta_lin][0] = pf_gtime();
    g_pf_cta[cta_lin][2] = smid;
    g_pf_cta[cta_lin][3] = (unsigned long long)n_kv;
  }
#endif
  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < KS; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
    }
    for (int x = 0; x < 2; ++x) {
      ptx::mbar_init(&s_full[x], 1);
      ptx::mbar_init(&p_full[x], kBM);
      ptx::mbar_init(&o_final[x], 1);
    }
    ptx::mbar_init(q_ready, 2 * kBM);
    for (int x = 0; x < 2; ++x) {
      ptx::mbar_init(&p_lo[x], kBM);
      ptx::mbar_init(&pv_lo[x], 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     ptx::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
#ifdef VATTN_PF_TRACE
  if (threadIdx.x == 0 && cta_lin < 8192) g_pf_cta[cta_lin][5] = pf_gtime();
#endif

  if (warp == 8) {
    // ===================== TMA producer =====================
    if (lane == 0 && n_kv > 0) {
      ptx::prefetch_tmap(&qmap);
      ptx::prefetch_tmap(kmp);
      ptx::prefetch_tmap(vmp);
      ptx::mbar_arrive_expect_tx(q_full, 2 * L::kTile);
#pragma unroll
      for (int h = 0; h < D / 64; ++h) {
        ptx::tma_load_3d(smem + L::kQOff + h * kHalf, &qmap, q_full, h * 64, head, q_row0 + q0A);
        ptx::tma_load_3d(smem + L::kQOff + L::kTile + h * kHalf, &qmap, q_full, h * 64, headB, q_row0 + q0B);
      }
      if constexpr (!PAGED) {
        // K runs KS - kStages tiles ahead of V (K_j then V_{j-ahead}); each stage waits for its
        // own release (K and V share one release when !SPLIT)
        constexpr int ahead = KS - kStages;
        for (int j = 0; j < n_kv + ahead; ++j) {
          if (j < n_kv) {
            const int s = j % KS;
            if (j >= KS) ptx::mbar_wait(&k_empty[s], ((j / KS) - 1) & 1);
            ptx::mbar_arrive_expect_tx(&k_full[s], L::kTile);
#pragma unroll
            for (int h = 0; h < D / 64; ++h)
              ptx::tma_load_3d(smem + L::kKOff + s * L::kTile + h * kHalf, kmp, &k_full[s], h * 64, kvh, (j0 + j) * kBN);
          }
          const int jv = j - ahead;
          if (jv >= 0) {
            const int s = jv % kStages;
            if (SPLIT && jv >= kStages) ptx::mbar_wait(&v_empty[s], ((jv / kStages) - 1) & 1);
            ptx::mbar_arrive_expect_tx(&v_full[s], L::kTile);
#pragma unroll
            for (int h = 0; h < D / 64; ++h)
              ptx::tma_load_3d(smem + L::kVOff + s * L::kTile + h * kHalf, vmp, &v_full[s], h * 64, kvh, (j0 + jv) * kBN);
          }
        }
      }
      for (int j = 0; PAGED && j < n_kv; ++j) {
        const int s = j % kStages;
        if (j >= kStages) ptx::mbar_wait(&k_empty[s], ((j / kStages) - 1) & 1);
        ptx::mbar_arrive_expect_tx(&k_full[s], L::kTile);
        {
          // PagedAttention layout: one TMA box per KV block (4-D map over [D, Hkv, block, n_blocks])
          const int last_blk = (p.kv_len - 1) / p.block_size;
          for (int sub = 0; sub < kBN / p.box_tokens; ++sub) {
            const int tok = j * kBN + sub * p.box_tokens;
            const int blk = __ldg(p.block_table + min(tok / p.block_size, last_blk));
            const int within = tok % p.block_size;
#pragma unroll
            for (int h = 0; h < D / 64; ++h)
              ptx::tma_load_4d(smem + L::kKOff + s * L::kTile + h * kHalf + sub * p.box_tokens * 128, &kmap,
                               &k_full[s], h * 64, kvh, within, blk);
          }
          ptx::mbar_arrive_expect_tx(&v_full[s], L::kTile);
          for (int sub = 0; sub < kBN / p.box_tokens; ++sub) {
            const int tok = j * kBN + sub * p.box_tokens;
            const int blk = __ldg(p.block_table + min(tok / p.block_size, last_blk));
            const int within = tok % p.block_size;
#pragma unroll
            for (int h = 0; h < D / 64; ++h)
              ptx::tma_load_4d(smem + L::kVOff + s * L::kTile + h * kHalf + sub * p.box_tokens * 128, &vmap,
                               &v_full[s], h * 64, kvh, within, blk);
          }
        }
      }
    }
  } else if (warp == 9) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0 && n_kv > 0) {
      const uint32_t id_qk = idesc(false), id_pv = idesc(true, D);
      const uint32_t sbase = ptx::smem_u32(smem);
      const uint32_t tS[2] = {tmem + 0, tmem + 128};
      const uint32_t tO[2] = {tmem + 256, tmem + 256 + D};
      const int nX[2] = {nA, nB};
      auto issue_s = [&](int x, int j) {   // S_x(j) = Q_x K_j^T
        const int s = j % KS;
        const uint32_t qa = sbase + L::kQOff + x * L::kTile;
        const uint32_t kb = sbase + L::kKOff + s * L::kTile;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
          mma_ss(tS[x], sdesc(qa + off, 16, 1024), sdesc(kb + off, 16, 1024), id_qk, kk > 0);
        }
        mma_commit(&s_full[x]);
      };
      auto issue_pv = [&](int x, int j, int k_lo, int k_hi) {  // O_x += P_x(j) V_j, keys [16 k_lo, 16 k_hi)
        const int s = j % kStages;
        const uint32_t vb = sbase + L::kVOff + s * L::kTile;
#pragma unroll
        for (int kk = k_lo; kk < k_hi; ++kk)
          mma_ts(tO[x], tS[x] + kk * 8, sdesc(vb + kk * 2048, kHalf, 1024), id_pv, (j > 0 || kk > 0) ? 1u : 0u);
      };
      ptx::mbar_wait(q_full, 0);
      if (p.rot_cos) ptx::mbar_wait(q_ready, 0);
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % kStages;
        if (j == 0) {
          ptx::mbar_wait(&k_full[0], 0);
          fence_after();
          for (int x = 0; x < 2; ++x)
            if (nX[x] > 0) issue_s(x, 0);
          if (SPLIT) mma_commit(&k_empty[0]);
        }
        ptx::mbar_wait(&v_full[s], (j / kStages) & 1);
        fence_after();
        for (int x = 0; x < 2; ++x) {
          if (j >= nX[x]) continue;
          PF_TRACE(2 + x, j, 0);
          if (early) {
            // keys 0..63 of P as soon as the softmax stored them, the rest when it is done
            ptx::mbar_wait_poll(&p_lo[x], j & 1);
            fence_after();
            issue_pv(x, j, 0, kBN / 32);
            mma_commit(&pv_lo[x]);
            ptx::mbar_wait_poll(&p_full[x], j & 1);
            PF_TRACE(2 + x, j, 1);
            fence_after();
            issue_pv(x, j, kBN / 32, kBN / 16);
          } else {
            // polled without a suspend hint: the issuer wakes sooner (measured 1229 vs 1220 TF)
            ptx::mbar_wait_poll(&p_full[x], j & 1);
            PF_TRACE(2 + x, j, 1);
            fence_after();
            issue_pv(x, j, 0, kBN / 16);
          }
          PF_TRACE(2 + x, j, 2);
          if (j + 1 == nX[x]) {
            mma_commit(&o_final[x]);
          } else {
            // S_x(j+1) needs K_{j+1}
            const int s1 = (j + 1) % KS;
            ptx::mbar_wait(&k_full[s1], ((j + 1) / KS) & 1);
            fence_after();
            issue_s(x, j + 1);
            PF_TRACE(2 + x, j, 3);
          }
        }
        if (SPLIT) {
          mma_commit(&v_empty[s]);                               // V_j: its last PV was issued
          if (j + 1 < n_kv) mma_commit(&k_empty[(j + 1) % KS]);  // K_{j+1}: both its S issued
        } else {
          mma_commit(&k_empty[s]);   // K_j / V_j fully consumed once these MMAs retire
        }
      }
    }
  } else {
    softmax_role<POLY, D, VARLEN, false, L>(p, smem, s_full, p_full, o_final, q_full, q_ready, tmem, warp, lane,
                                            head, q_row0, q0A, q0B, nA, nB, n_kv, omap, 0, 0, nullptr,
                                            hp ? headB : -1, early ? p_lo : nullptr, early ? pv_lo : nullptr, j0);
  }
#ifdef VATTN_PF_TRACE
  __syncthreads();
  if (threadIdx.x == 0 && cta_lin < 8192) g_pf_cta[cta_lin][1] = pf_gtime();
#endif
  fence_before();
#ifdef VATTN_PF_TRACE
  if (threadIdx.x == 0 && cta_lin < 8192) g_pf_cta[cta_lin][8] = pf_gtime();
  if (threadIdx.x == 32 * 9 && cta_lin < 8192) g_pf_cta[cta_lin][10] = pf_gtime();
#endif
  __syncthreads();
#ifdef VATTN_PF_TRACE
  if (threadIdx.x == 0 && cta_lin < 8192) g_pf_cta[cta_lin][9] = pf_gtime();
#endif
  if (warp == 9) {
#ifdef VATTN_PF_TRACE
    if (lane == 0 && cta_lin < 8192) g_pf_cta[cta_lin][7] = pf_gtime();
#endif
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
#ifdef VATTN_PF_TRACE
    if (lane == 0 && cta_lin < 8192) g_pf_cta[cta_lin][6] = pf_gtime();
#endif
  }
}



// ===================== persistent varlen kernel: one CTA per SM walks the work list =============
// Short prompts give CTAs of 1-4 KV tiles, where a CTA's fixed costs (launch, barrier / TMEM
// setup, two dependent loads for its work item, the Q and first K/V latencies, the epilogue)
// rival its work (tools/prefill_cta_timeline_varlen.py).  Here a CTA keeps TMEM,
// barriers and the K / V rings across items (head, request, 256-row pair): item i+1's Q load,
// first K / V tiles and first S MMAs run under item i's softmax tail and epilogue.  Items are
// the normal grid's (head-fastest, heaviest-first) order dealt to the CTAs in snake order.  Ring
// indices and barrier phases run on across items; Q is released (q_empty) once an item's last S
// MMA retired and O (o_free) once the epilogue read it out of TMEM.  D = 128, no rotary.
__device__ __forceinline__ int persist_item(int r, int c, int G) { return r * G + ((r & 1) ? G - 1 - c : c); }

struct VarItem {
  int head, headB, q_row0, q0A, q0B, nA, nB;
  const CUtensorMap* kmp;
  Params p;      // the launch's Params with this item's request fields (n_q, kv_len, q_off, out)
};

__device__ __forceinline__ VarItem varlen_item(const Params& p, int w) {
  VarItem it;
  const int hper = p.head_pair ? p.hq / 2 : p.hq;   // items per work entry
  const int4 wk = p.work[w / hper];
  const int4 rq = p.reqs[wk.x];
  it.head = p.head_pair ? 2 * (w % hper) : w % hper;
  it.headB = p.head_pair ? it.head + 1 : it.head;
  it.q_row0 = rq.x;
  it.p = p;
  it.p.n_q = rq.y;
  it.p.kv_len = rq.z;
  it.p.q_off = rq.z - rq.y;
  it.p.out = p.out + (int64_t)rq.x * p.hq * 128;
  it.q0A = p.head_pair ? wk.y * kBM : wk.y * 2 * kBM;
  it.q0B = p.head_pair ? it.q0A : it.q0A + kBM;
  it.nA = kv_tiles_for(it.p, it.q0A);
  it.nB = kv_tiles_for(it.p, it.q0B);
  it.kmp = p.maps + 2 * wk.x;
  return it;
}

__global__ void __launch_bounds__(kThreads, 1)
prefill_persist_varlen_kernel(const __grid_constant__ CUtensorMap qmap, Params p, int n_items) {
  constexpr int D = 128;
  constexpr int KS = kKStages;
  using L = PfL<D, KS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;            // [KS]
  uint64_t* v_full = bars + 5;            // [kStages]
  uint64_t* k_empty = bars + 7;           // [KS]
  uint64_t* v_empty = bars + 11;          // [kStages]
  uint64_t* s_full = bars + 13;           // [2]
  uint64_t* p_full = bars + 15;           // [2]
  uint64_t* o_final = bars + 17;          // [2]
  uint64_t* q_empty = bars + 19;
  uint64_t* o_free = bars + 20;           // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int c = blockIdx.x, G = gridDim.x;

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int st = 0; st < KS; ++st) {
      ptx::mbar_init(&k_full[st], 1);
      ptx::mbar_init(&k_empty[st], 1);
    }
    for (int st = 0; st < kStages; ++st) {
      ptx::mbar_init(&v_full[st], 1);
      ptx::mbar_init(&v_empty[st], 1);
    }
    for (int x = 0; x < 2; ++x) {
      ptx::mbar_init(&s_full[x], 1);
      ptx::mbar_init(&p_full[x], kBM);
      ptx::mbar_init(&o_final[x], 1);
      ptx::mbar_init(&o_free[x], kBM);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     ptx::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ===================== TMA producer =====================
    // Per item: the first K / V stages first (their previous occupants belong to earlier items, so
    // they are released without this item's MMAs), then Q once the previous item's last S MMA
    // retired, then the rest of the K / V stream.  The next item's descriptor (two dependent
    // loads) is fetched while the current one streams.
    if (lane == 0) {
      ptx::prefetch_tmap(&qmap);
      int kt = 0, qi = 0;                  // K/V tiles and Q loads issued so far
      constexpr int ahead = KS - kStages;
      int w = persist_item(0, c, G);
      VarItem it{};
      if (w < n_items) it = varlen_item(p, w);
      for (int r = 0; w < n_items; ++r) {
        const int w_next = persist_item(r + 1, c, G);
        VarItem nxt{};
        if (w_next < n_items) nxt = varlen_item(p, w_next);
        const int n_kv = max(it.nA, it.nB);
        if (n_kv > 0) {
          const int kvh = it.head / p.group;
          const CUtensorMap* kmp = it.kmp;
          const CUtensorMap* vmp = it.kmp + 1;
          ptx::prefetch_tmap(kmp);
          ptx::prefetch_tmap(vmp);
          auto load_k = [&](int j) {
            const int t = kt + j, st = t % KS;
            if (t >= KS) ptx::mbar_wait(&k_empty[st], ((t / KS) - 1) & 1);
            ptx::mbar_arrive_expect_tx(&k_full[st], L::kTile);
#pragma unroll
            for (int h = 0; h < D / 64; ++h)
              ptx::tma_load_3d(smem + L::kKOff + st * L::kTile + h * kHalf, kmp, &k_full[st], h * 64, kvh, j * kBN);
          };
          auto load_v = [&](int jv) {
            const int t = kt + jv, st = t % kStages;
            if (t >= kStages) ptx::mbar_wait(&v_empty[st], ((t / kStages) - 1) & 1);
            ptx::mbar_arrive_expect_tx(&v_full[st], L::kTile);
#pragma unroll
            for (int h = 0; h < D / 64; ++h)
              ptx::tma_load_3d(smem + L::kVOff + st * L::kTile + h * kHalf, vmp, &v_full[st], h * 64, kvh, jv * kBN);
          };
          const int k_early = min(n_kv, KS), v_early = min(n_kv, kStages);
          for (int j = 0; j < k_early; ++j) load_k(j);
          for (int jv = 0; jv < v_early; ++jv) load_v(jv);
          if (qi > 0) ptx::mbar_wait(q_empty, (qi - 1) & 1);
          ptx::mbar_arrive_expect_tx(q_full, 2 * L::kTile);
#pragma unroll
          for (int h = 0; h < D / 64; ++h) {
            ptx::tma_load_3d(smem + L::kQOff + h * kHalf, &qmap, q_full, h * 64, it.head, it.q_row0 + it.q0A);
            ptx::tma_load_3d(smem + L::kQOff + L::kTile + h * kHalf, &qmap, q_full, h * 64, it.headB,
                             it.q_row0 + it.q0B);
          }
          ++qi;
          for (int j = k_early; j < n_kv + ahead; ++j) {
            if (j < n_kv) load_k(j);
            const int jv = j - ahead;
            if (jv >= v_early && jv < n_kv) load_v(jv);
          }
          kt += n_kv;
        }
        w = w_next;
        it = nxt;
      }
    }
  } else if (warp == 9) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      const uint32_t id_qk = idesc(false), id_pv = idesc(true, D);
      const uint32_t sbase = ptx::smem_u32(smem);
      const uint32_t tS[2] = {tmem + 0, tmem + 128};
      const uint32_t tO[2] = {tmem + 256, tmem + 256 + D};
      int kt = 0, qi = 0;
      uint32_t cntS[2] = {0, 0}, cntO[2] = {0, 0};   // tiles / items with tiles, per Q tile
      int w = persist_item(0, c, G);
      VarItem it{};
      if (w < n_items) it = varlen_item(p, w);
      for (int r = 0; w < n_items; ++r, w = persist_item(r, c, G)) {
        const int w_next = persist_item(r + 1, c, G);
        VarItem nxt{};
        if (w_next < n_items) nxt = varlen_item(p, w_next);   // next item's descriptor, fetched early
        const VarItem cur = it;
        it = nxt;
        const int n_kv = max(cur.nA, cur.nB);
        if (n_kv == 0) continue;
        const int nX[2] = {cur.nA, cur.nB};
        auto issue_s = [&](int x, int j) {
          const int st = (kt + j) % KS;
          const uint32_t qa = sbase + L::kQOff + x * L::kTile;
          const uint32_t kb = sbase + L::kKOff + st * L::kTile;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
            mma_ss(tS[x], sdesc(qa + off, 16, 1024), sdesc(kb + off, 16, 1024), id_qk, kk > 0);
          }
          mma_commit(&s_full[x]);
        };
        ptx::mbar_wait(q_full, qi & 1);
        for (int j = 0; j < n_kv; ++j) {
          const int t = kt + j, sv = t % kStages;
          if (j == 0) {
            ptx::mbar_wait(&k_full[t % KS], (t / KS) & 1);
            fence_after();
            for (int x = 0; x < 2; ++x)
              if (nX[x] > 0) issue_s(x, 0);
            mma_commit(&k_empty[t % KS]);
          }
          ptx::mbar_wait(&v_full[sv], (t / kStages) & 1);
          fence_after();
          for (int x = 0; x < 2; ++x) {
            if (j >= nX[x]) continue;
            ptx::mbar_wait_poll(&p_full[x], (cntS[x] + j) & 1);
            if (j == 0 && cntO[x] > 0) ptx::mbar_wait(&o_free[x], (cntO[x] - 1) & 1);   // previous O read out
            fence_after();
            const uint32_t vb = sbase + L::kVOff + sv * L::kTile;
#pragma unroll
            for (int kk = 0; kk < kBN / 16; ++kk)
              mma_ts(tO[x], tS[x] + kk * 8, sdesc(vb + kk * 2048, kHalf, 1024), id_pv, (j > 0 || kk > 0) ? 1u : 0u);
            if (j + 1 == nX[x]) {
              mma_commit(&o_final[x]);
            } else {
              const int t1 = t + 1;
              ptx::mbar_wait(&k_full[t1 % KS], (t1 / KS) & 1);
              fence_after();
              issue_s(x, j + 1);
            }
          }
          mma_commit(&v_empty[sv]);
          if (j + 1 < n_kv) mma_commit(&k_empty[(t + 1) % KS]);
        }
        mma_commit(q_empty);                 // Q no longer read once these MMAs retire
        for (int x = 0; x < 2; ++x) {
          cntS[x] += nX[x];
          cntO[x] += nX[x] > 0 ? 1u : 0u;
        }
        kt += n_kv;
        ++qi;
      }
    }
  } else {
    const int x = warp / 4;
    uint32_t cntS = 0, cntO = 0;
    for (int r = 0;; ++r) {
      const int w = persist_item(r, c, G);
      if (w >= n_items) break;
      const VarItem it = varlen_item(p, w);
      const int n_kv = max(it.nA, it.nB);
      softmax_role<0, D, true, false, L>(it.p, smem, s_full, p_full, o_final, q_full, nullptr, tmem, warp, lane,
                                         it.head, it.q_row0, it.q0A, it.q0B, it.nA, it.nB, n_kv, qmap, cntS,
                                         cntO, o_free, p.head_pair ? it.headB : -1);
      const int n = x == 0 ? it.nA : it.nB;
      cntS += n;
      cntO += n > 0 ? 1u : 0u;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 9) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}



// ===================== CTA-pair kernel (tcgen05 cta_group::2) =====================
// Two CTAs of a cluster = two query heads of one GQA group over the same 256 query rows.  The
// leader (rank 0) issues every MMA for both with M = 256 (rows 0-127 = leader's head, 128-255 =
// peer's): each SM supplies its own Q tile as its half of A and HALF of the B operand (K: 64 of
// the 128 keys of a tile; V: 64 of the 128 head-dim columns), and the hardware multicasts the B
// halves between the pair.  Per SM and 128-key step that halves the B-operand reads and the TMA
// writes of the single-CTA kernel, whose S MMAs are shared-memory bound.  S, P and O
// of a head live in its own CTA's TMEM, so the softmax warps are the single-CTA ones.
template <int D>
struct PairL {
  static_assert(D == 128, "the pair kernel is built for head_dim 128");
  static constexpr int kKS = 4, kVS = 3;               // ring depths (stages of half tiles)
  static constexpr int kTile = 2 * kHalf;              // one Q tile: 128 rows x 128 d (32 KB)
  static constexpr int kKHalf = 64 * 128;              // K half-tile, one 64-d half: 64 keys x 128 B
  static constexpr int kKStage = 2 * kKHalf;           // 16 KB
  static constexpr int kVStage = kHalf;                // V half-tile: 128 keys x 64 d (16 KB)
  static constexpr int kQOff = 0;
  static constexpr int kKOff = 2 * kTile;
  static constexpr int kVOff = kKOff + kKS * kKStage;
  static constexpr int kBarOff = kVOff + kVS * kVStage;
  static constexpr int kSmem = kBarOff + 256 + 1024;
};

__host__ __device__ constexpr uint32_t idesc2(bool b_mn_major) {   // M = 256 (pair), N = 128
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(128 >> 3) << 17) |
         ((uint32_t)(256 >> 4) << 24);
}
__device__ __forceinline__ void mma2_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma2_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
// completion of the leader's MMAs so far -> the barrier at this offset in BOTH CTAs of the pair
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
          ptx::smem_u32(bar))
      : "memory");
}
// TMA load into this CTA's shared memory whose bytes complete on the LEADER's barrier
__device__ __forceinline__ void tma2_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(ptx::smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = ptx::smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAITC:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@p bra.uni DONEC;\n"
      "bra.uni LAB_WAITC;\n"
      "DONEC:\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

template <bool VARLEN = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
prefill_pair_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                    const __grid_constant__ CUtensorMap vmap, const __grid_constant__ CUtensorMap omap, Params p) {
  constexpr int D = 128;
  using L = PairL<D>;
  constexpr int KS = L::kKS, VS = L::kVS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  // *_full / p_full / q_ready are used in the leader only; *_empty, s_full, o_final in both
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;            // [KS]
  uint64_t* v_full = bars + 5;            // [VS]
  uint64_t* k_empty = bars + 8;           // [KS]
  uint64_t* v_empty = bars + 12;          // [VS]
  uint64_t* s_full = bars + 15;           // [2]
  uint64_t* p_full = bars + 17;           // [2]
  uint64_t* o_final = bars + 19;          // [2]
  uint64_t* q_ready = bars + 21;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const bool leader = rank == 0;
  const int witem = blockIdx.y;            // pair kernel: heads along x (cluster), work along y
  int pair = p.n_pairs - 1 - witem;
  int q_row0 = 0;
  const CUtensorMap* kmp = &kmap;
  const CUtensorMap* vmp = &vmap;
  if constexpr (VARLEN) {
    const int4 w = p.work[witem];
    const int4 r = p.reqs[w.x];
    pair = w.y;
    q_row0 = r.x;
    p.n_q = r.y;
    p.kv_len = r.z;
    p.q_off = r.z - r.y;
    p.out += (int64_t)r.x * p.hq * D;
    kmp = p.maps + 2 * w.x;
    vmp = kmp + 1;
  }
  const int head = blockIdx.x;
  const int kvh = head / p.group;          // both heads of the pair share it (group even)
  const int q0A = pair * 2 * kBM, q0B = q0A + kBM;
  const int nA = kv_tiles_for(p, q0A), nB = kv_tiles_for(p, q0B);
  const int n_kv = max(nA, nB);

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < KS; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < VS; ++s) {
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
    }
    for (int x = 0; x < 2; ++x) {
      ptx::mbar_init(&s_full[x], 1);
      ptx::mbar_init(&p_full[x], 2 * kBM);         // both CTAs' softmax threads of tile x
      ptx::mbar_init(&o_final[x], 1);
    }
    ptx::mbar_init(q_ready, 2 * 2 * kBM);
    ptx::fence_mbar_init();
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     ptx::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  cluster_sync();                          // barriers of both CTAs initialised, TMEM allocated
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ===================== TMA producer (both CTAs: own Q, own halves of K and V) ============
    if (lane == 0 && n_kv > 0) {
      ptx::prefetch_tmap(&qmap);
      ptx::prefetch_tmap(kmp);
      ptx::prefetch_tmap(vmp);
      if (leader) ptx::mbar_arrive_expect_tx(q_full, 2 * 2 * L::kTile);
#pragma unroll
      for (int h = 0; h < D / 64; ++h) {
        tma2_load_3d(smem + L::kQOff + h * kHalf, &qmap, q_full, h * 64, head, q_row0 + q0A);
        tma2_load_3d(smem + L::kQOff + L::kTile + h * kHalf, &qmap, q_full, h * 64, head, q_row0 + q0B);
      }
      constexpr int ahead = KS - VS;       // K runs ahead of V
      for (int j = 0; j < n_kv + ahead; ++j) {
        if (j < n_kv) {
          const int s = j % KS;
          if (j >= KS) ptx::mbar_wait(&k_empty[s], ((j / KS) - 1) & 1);
          if (leader) ptx::mbar_arrive_expect_tx(&k_full[s], 2 * L::kKStage);
#pragma unroll
          for (int h = 0; h < D / 64; ++h)   // keys [64 rank, 64 rank + 64) of tile j, d-half h
            tma2_load_3d(smem + L::kKOff + s * L::kKStage + h * L::kKHalf, kmp, &k_full[s], h * 64, kvh,
                         j * kBN + 64 * (int)rank);
        }
        const int jv = j - ahead;
        if (jv >= 0) {
          const int s = jv % VS;
          if (jv >= VS) ptx::mbar_wait(&v_empty[s], ((jv / VS) - 1) & 1);
          if (leader) ptx::mbar_arrive_expect_tx(&v_full[s], 2 * L::kVStage);
          // all 128 keys of tile jv, head-dim columns [64 rank, 64 rank + 64)
          tma2_load_3d(smem + L::kVOff + s * L::kVStage, vmp, &v_full[s], 64 * (int)rank, kvh, jv * kBN);
        }
      }
    }
  } else if (warp == 9) {
    // ===================== MMA issuer (leader, one thread, for both CTAs) =====================
    if (leader && lane == 0 && n_kv > 0) {
      const uint32_t id_qk = idesc2(false), id_pv = idesc2(true);
      const uint32_t sbase = ptx::smem_u32(smem);
      const uint32_t tS[2] = {tmem + 0, tmem + 128};
      const uint32_t tO[2] = {tmem + 256, tmem + 256 + D};
      const int nX[2] = {nA, nB};
      auto issue_s = [&](int x, int j) {   // S_x(j) = Q_x K_j^T (M = 256: this tile of both heads)
        const int s = j % KS;
        const uint32_t qa = sbase + L::kQOff + x * L::kTile;
        const uint32_t kb = sbase + L::kKOff + s * L::kKStage;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma2_ss(tS[x], sdesc(qa + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024),
                  sdesc(kb + (kk >> 2) * L::kKHalf + (kk & 3) * 32, 16, 1024), id_qk, kk > 0);
        commit2(&s_full[x]);
      };
      auto issue_pv = [&](int x, int j) {  // O_x += P_x(j) V_j
        const int s = j % VS;
        const uint32_t vb = sbase + L::kVOff + s * L::kVStage;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)
          mma2_ts(tO[x], tS[x] + kk * 8, sdesc(vb + kk * 2048, kHalf, 1024), id_pv, (j > 0 || kk > 0) ? 1u : 0u);
      };
      mbar_wait_cluster(q_full, 0);
      if (p.rot_cos) mbar_wait_cluster(q_ready, 0);
      for (int j = 0; j < n_kv; ++j) {
        const int sv = j % VS;
        if (j == 0) {
          mbar_wait_cluster(&k_full[0], 0);
          fence_after();
          for (int x = 0; x < 2; ++x)
            if (nX[x] > 0) issue_s(x, 0);
          commit2(&k_empty[0]);
        }
        mbar_wait_cluster(&v_full[sv], (j / VS) & 1);
        fence_after();
        for (int x = 0; x < 2; ++x) {
          if (j >= nX[x]) continue;
          PF_TRACE(2 + x, j, 0);
          {   // P_x(j) from both CTAs' softmax warps
            const uint32_t a = ptx::smem_u32(&p_full[x]);
            asm volatile(
                "{\n.reg .pred p;\nLAB_WAITPP:\n"
                "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
                "@p bra.uni DONEPP;\nbra.uni LAB_WAITPP;\nDONEPP:\n}\n" ::"r"(a), "r"((uint32_t)(j & 1))
                : "memory");
          }
          PF_TRACE(2 + x, j, 1);
          fence_after();
          issue_pv(x, j);
          PF_TRACE(2 + x, j, 2);
          if (j + 1 == nX[x]) {
            commit2(&o_final[x]);
          } else {
            const int s1 = (j + 1) % KS;
            mbar_wait_cluster(&k_full[s1], ((j + 1) / KS) & 1);
            fence_after();
            issue_s(x, j + 1);
            PF_TRACE(2 + x, j, 3);
          }
        }
        commit2(&v_empty[sv]);
        if (j + 1 < n_kv) commit2(&k_empty[(j + 1) % KS]);
      }
    }
  } else {
    softmax_role<0, D, VARLEN, true, L>(p, smem, s_full, p_full, o_final, q_full, q_ready, tmem, warp, lane, head,
                                        q_row0, q0A, q0B, nA, nB, n_kv, omap);
  }
  fence_before();
  __syncthreads();
  cluster_sync();                          // the peer's shared memory / TMEM stay live until both are done
  if (warp == 9) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}


}  // namespace pf

static CUtensorMap make_map(void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                            const cuuint32_t* box) {
  CUtensorMap m;
  const char* promo_env = getenv("VATTN_PF_L2PROMO");
  const CUtensorMapL2promotion promo = (promo_env && promo_env[0] == '0') ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                                                          : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  check_cu(driver().TensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, base, dims, strides,
                                         box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                         CU_TENSOR_MAP_SWIZZLE_128B, promo,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
           "cuTensorMapEncodeTiled(prefill)");
  return m;
}

// Head pairs (Params::head_pair) for the single-request kernel: VATTN_PF_HEADPAIR=0/1 forces
// the tiling.  By default pairs are used when the GQA group is even and the prompt spans more
// than one 128-row tile (tools/pf_headpair_ab.py, B200: Yi-6B 4K causal 1.056x, Llama-3-8B 4K
// 1.096x, 16K 1.006x, bit-identical).  At <= 128 rows the row tiling launches twice as many
// CTAs (one per head, tile B empty) on a grid far below the SM count, which is faster there
// (0.86-0.94x with pairs).
static int early_pv_mode() {
  static int v = -1;   // 2 = automatic
  if (v < 0) {
    const char* e = getenv("VATTN_PF_EARLYPV");
    v = e ? (atoi(e) != 0 ? 1 : 0) : 2;
  }
  return v == 2 ? -1 : v;
}

static int head_pair_env() {   // -1 automatic, 0 / 1 forced (VATTN_PF_HEADPAIR)
  static int mode = -2;
  if (mode == -2) {
    const char* e = getenv("VATTN_PF_HEADPAIR");
    mode = e ? atoi(e) : -1;
  }
  return mode;
}

static int split_kv_mode() {   // VATTN_PF_SPLITKV: 0 off, 1 automatic (default), N > 1 forced
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("VATTN_PF_SPLITKV");
    mode = e ? std::max(0, atoi(e)) : 1;
  }
  return mode;
}

static int num_sms_cached();
// rows_items / pair_items: CTAs (work items) of the launch under each tiling.  Pairs never have
// more; they are taken when they keep the count or still fill every SM.
static bool use_head_pairs(int64_t rows_items, int64_t pair_items, int hq, int group) {
  const int mode = head_pair_env();
  if (group % 2 || hq % 2 || mode == 0) return false;
  if (mode > 0) return true;
  return pair_items >= rows_items || pair_items >= num_sms_cached();
}

void launch_prefill(KernelState*, int, const CacheView& v, const void* q, void* out, int n_q, int hq,
                    int slot, int kv_len, float scale, bool causal, cudaStream_t st, const Rotary* rot) {
  if (v.d != 128 && v.d != 64) throw Fail(VATTN_UNSUPPORTED, "prefill kernel is built for head_dim 64 and 128");
  const int D = v.d;
  if (hq % v.hkv) throw Fail(VATTN_VALUE_ERROR, "n_q_heads must be a multiple of n_kv_heads");
  if (slot < 0 || slot >= v.n_slots) throw Fail(VATTN_VALUE_ERROR, "slot out of range");
  if (kv_len < 0 || kv_len > v.slot_tokens) throw Fail(VATTN_VALUE_ERROR, "kv_len out of range");
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(out)) % 16)
    throw Fail(VATTN_UNSUPPORTED, "q/out must be 16-byte aligned");
  if (n_q <= 0) return;
  // Per-call maps: the K/V token extent is exactly kv_len, so rows past it are zero-filled by
  // TMA instead of being read from (possibly stale or unmapped) pages.
  const int kvl = std::max(kv_len, 1);
  cuuint64_t qd[3] = {(cuuint64_t)D, (cuuint64_t)hq, (cuuint64_t)n_q};
  cuuint64_t qs[2] = {(cuuint64_t)D * 2, (cuuint64_t)hq * D * 2};
  cuuint32_t qb[3] = {64, 1, (cuuint32_t)pf::kBM};
  const CUtensorMap qmap = make_map(const_cast<void*>(q), 3, qd, qs, qb);
  const CUtensorMap omap = make_map(out, 3, qd, qs, qb);
  // 3-D map rooted at the request's slot: [D, Hkv, kv_len] (the slot index is folded into the base)
  cuuint64_t kd[3] = {(cuuint64_t)D, (cuuint64_t)v.hkv, (cuuint64_t)kvl};
  cuuint64_t ks[2] = {(cuuint64_t)D * 2, (cuuint64_t)v.token_stride};
  cuuint32_t kb[3] = {64, 1, (cuuint32_t)pf::kBN};
  const uint64_t slot_off = (uint64_t)slot * (uint64_t)v.slot_stride;
  const CUtensorMap kmap = make_map(reinterpret_cast<void*>(v.k_base + slot_off), 3, kd, ks, kb);
  const CUtensorMap vmap = make_map(reinterpret_cast<void*>(v.v_base + slot_off), 3, kd, ks, kb);
  pf::Params p{};
  if (rot && rot->cos) {
    if (!rot->sin || rot->dim <= 0 || rot->dim % 16 || rot->dim > D)
      throw Fail(VATTN_VALUE_ERROR, "rotary_dim must be a positive multiple of 16 and <= head_dim");
    p.rot_cos = rot->cos;
    p.rot_sin = rot->sin;
    p.rot_dim = rot->dim;
    p.rot_inter = rot->interleaved;
  }
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.n_q = n_q;
  p.hq = hq;
  p.group = hq / v.hkv;
  p.kv_len = kv_len;
  p.slot = slot;
  p.q_off = kv_len - n_q;
  p.causal = causal ? 1 : 0;
  if (scale <= 0.f) scale = 1.f / sqrtf((float)D);
  p.scale_log2 = scale * 1.4426950408889634f;
  p.head_pair = use_head_pairs((int64_t)hq * ((n_q + 2 * pf::kBM - 1) / (2 * pf::kBM)),
                               (int64_t)(hq / 2) * ((n_q + pf::kBM - 1) / pf::kBM), hq, p.group) ? 1 : 0;
  static int pair_mode = -1;
  if (pair_mode < 0) {
    const char* e = getenv("VATTN_PF_PAIR");   // 1: CTA-pair kernel (cta_group::2) where it applies
    pair_mode = e ? (atoi(e) != 0) : 0;
  }
  const bool use_pair_kernel = D == 128 && pair_mode && !(rot && rot->cos) && p.group % 2 == 0 && hq % 2 == 0;
  // Split-KV for grids far below the SM count with long KV ranges (e.g. a 128-row chunk over a
  // long prefix: 32 CTAs of one tile each): head pairs first (two tiles per CTA), then the KV
  // range of every CTA is split so the grid fills the SMs; partials merge in the combine kernel.
  auto n_ctas = [&](bool hp_) {
    return (int64_t)(hp_ ? hq / 2 : hq) * (hp_ ? (n_q + pf::kBM - 1) / pf::kBM : (n_q + 2 * pf::kBM - 1) / (2 * pf::kBM));
  };
  const int nkv_max = (std::max(kv_len, 1) + pf::kBN - 1) / pf::kBN;
  const int split_env = split_kv_mode();
  int splits = 1;
  if (!use_pair_kernel && split_env != 0) {
    if (split_env > 1) {
      splits = split_env;
    } else if (n_ctas(p.head_pair != 0) * 2 <= num_sms_cached() && nkv_max >= 16) {
      if (p.group % 2 == 0 && hq % 2 == 0 && head_pair_env() != 0) p.head_pair = 1;
      splits = (int)std::min<int64_t>(std::min<int64_t>(16, num_sms_cached() / n_ctas(p.head_pair != 0)), nkv_max / 8);
    }
    splits = std::max(1, std::min(splits, nkv_max));
  }
  p.n_pairs = p.head_pair ? (n_q + pf::kBM - 1) / pf::kBM : (n_q + 2 * pf::kBM - 1) / (2 * pf::kBM);
  dim3 grid = pf::pf_grid(p, p.n_pairs, p.head_pair ? hq / 2 : hq);
  p.early_pv = early_pv_mode();
  void* ws = nullptr;
  if (splits > 1) {
    const int64_t rows = (int64_t)n_q * hq;
    check_rt(cudaMallocAsync(&ws, (size_t)rows * splits * (D + 1) * sizeof(float), st), "cudaMallocAsync(split prefill)");
    p.kv_splits = splits;
    p.part_o = static_cast<float*>(ws);
    p.part_lse = p.part_o + rows * splits * D;
    grid.z = splits;
  }
  auto finish = [&]() {
    if (splits > 1) {
      launch_split_combine(p.part_o, p.part_lse, out, n_q * hq, splits, hq, D, st);
      check_rt(cudaFreeAsync(ws, st), "cudaFreeAsync(split prefill)");
    }
  };
  if (D == 64) {
    ensure_smem_attr<pf::prefill_kernel<0, false, 64>>(pf::PfL<64>::kSmem);
    pf::prefill_kernel<0, false, 64><<<grid, pf::kThreads, pf::PfL<64>::kSmem, st>>>(qmap, kmap, vmap, omap, p);
    check_rt(cudaGetLastError(), "prefill launch");
    finish();
    return;
  }
  if (use_pair_kernel) {
    p.head_pair = 0;   // the CTA-pair kernel tiles rows (two consecutive 128-row tiles)
    p.n_pairs = (n_q + 2 * pf::kBM - 1) / (2 * pf::kBM);
    // the pair kernel's K half-tiles: boxes of 64 keys
    cuuint32_t kb2[3] = {64, 1, 64};
    const CUtensorMap kmap2 = make_map(reinterpret_cast<void*>(v.k_base + slot_off), 3, kd, ks, kb2);
    constexpr int kS2 = pf::PairL<128>::kSmem;
    ensure_smem_attr<pf::prefill_pair_kernel<false>>(kS2);
    pf::prefill_pair_kernel<false><<<dim3(hq, p.n_pairs), pf::kThreads, kS2, st>>>(qmap, kmap2, vmap, omap, p);
    check_rt(cudaGetLastError(), "prefill (pair) launch");
    return;
  }
  static int poly = -1;
  if (poly < 0) {
    const char* e = getenv("VATTN_PF_POLY");   // share of exp2 on the FMA pipe, in quarters
    poly = e ? std::max(0, std::min(3, atoi(e))) : 0;
  }
  constexpr int kS = pf::PfL<128>::kSmem;
  if (poly == 0) {
    ensure_smem_attr<pf::prefill_kernel<0>>(kS);
    pf::prefill_kernel<0><<<grid, pf::kThreads, kS, st>>>(qmap, kmap, vmap, omap, p);
  } else if (poly == 1) {
    ensure_smem_attr<pf::prefill_kernel<1>>(kS);
    pf::prefill_kernel<1><<<grid, pf::kThreads, kS, st>>>(qmap, kmap, vmap, omap, p);
  } else if (poly == 2) {
    ensure_smem_attr<pf::prefill_kernel<2>>(kS);
    pf::prefill_kernel<2><<<grid, pf::kThreads, kS, st>>>(qmap, kmap, vmap, omap, p);
  } else {
    ensure_smem_attr<pf::prefill_kernel<3>>(kS);
    pf::prefill_kernel<3><<<grid, pf::kThreads, kS, st>>>(qmap, kmap, vmap, omap, p);
  }
  check_rt(cudaGetLastError(), "prefill launch");
  finish();
}

static int num_sms_cached() {
  static const int sms = [] {
    int d = 0, n = 148;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    return n;
  }();
  return sms;
}

// Several requests' prefills in one launch (flash_attn_varlen_func-style packing of the query
// rows): q [total, Hq, D] packed, request i's rows at q_start[i] .. + n_q[i], attending over rows
// [0, kv_len[i]) of slot slots[i].  The host builds each request's K/V tensor maps (rooted at its
// slot, extent exactly kv_len) and a work list of (request, 256-row pair) sorted by descending
// KV tiles, copied to a device buffer on the stream before the launch.
void launch_prefill_varlen(const CacheView& v, const void* q, void* out, int hq, int n_req, const int32_t* q_start,
                           const int32_t* n_q, const int32_t* slots, const int32_t* kv_len, float scale,
                           bool causal, cudaStream_t st) {
  if (v.d != 128 && v.d != 64) throw Fail(VATTN_UNSUPPORTED, "prefill kernel is built for head_dim 64 and 128");
  if (hq % v.hkv) throw Fail(VATTN_VALUE_ERROR, "n_q_heads must be a multiple of n_kv_heads");
  if (n_req <= 0) return;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(out)) % 16)
    throw Fail(VATTN_UNSUPPORTED, "q/out must be 16-byte aligned");
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  check_rt(cudaStreamIsCapturing(st, &cs), "cudaStreamIsCapturing");
  if (cs != cudaStreamCaptureStatusNone)
    throw Fail(VATTN_UNSUPPORTED, "varlen prefill uploads a per-call schedule and cannot be graph-captured");
  const int D = v.d;
  int total = 0;
  std::vector<CUtensorMap> maps(2 * (size_t)n_req);
  std::vector<int4> reqs(n_req);
  std::vector<std::pair<int, int4>> work;   // (kv tiles, item)
  int64_t rows_items = 0, pair_items = 0;
  for (int i = 0; i < n_req; ++i) {
    if (slots[i] < 0 || slots[i] >= v.n_slots) throw Fail(VATTN_VALUE_ERROR, "slot out of range");
    if (kv_len[i] < 0 || kv_len[i] > v.slot_tokens) throw Fail(VATTN_VALUE_ERROR, "kv_len out of range");
    if (n_q[i] < 0 || q_start[i] < 0) throw Fail(VATTN_VALUE_ERROR, "bad query rows");
    total = std::max(total, q_start[i] + n_q[i]);
    const int kvl = std::max(kv_len[i], 1);
    cuuint64_t kd[3] = {(cuuint64_t)D, (cuuint64_t)v.hkv, (cuuint64_t)kvl};
    cuuint64_t ks[2] = {(cuuint64_t)D * 2, (cuuint64_t)v.token_stride};
    cuuint32_t kb[3] = {64, 1, (cuuint32_t)pf::kBN};
    const uint64_t off = (uint64_t)slots[i] * (uint64_t)v.slot_stride;
    maps[2 * i] = make_map(reinterpret_cast<void*>(v.k_base + off), 3, kd, ks, kb);
    maps[2 * i + 1] = make_map(reinterpret_cast<void*>(v.v_base + off), 3, kd, ks, kb);
    reqs[i] = make_int4(q_start[i], n_q[i], kv_len[i], 0);
    rows_items += (int64_t)hq * ((n_q[i] + 2 * pf::kBM - 1) / (2 * pf::kBM));
    pair_items += (int64_t)(hq / 2) * ((n_q[i] + pf::kBM - 1) / pf::kBM);
  }
  const bool hp = use_head_pairs(rows_items, pair_items, hq, hq / v.hkv);
  const int rows_per_item = hp ? pf::kBM : 2 * pf::kBM;
  for (int i = 0; i < n_req; ++i) {
    const int pairs = (n_q[i] + rows_per_item - 1) / rows_per_item;
    for (int pr = 0; pr < pairs; ++pr) {
      const int q_last = std::min((pr + 1) * rows_per_item, n_q[i]) - 1;
      const int last_key = causal ? std::min(kv_len[i] - 1, q_last + kv_len[i] - n_q[i]) : kv_len[i] - 1;
      work.push_back({last_key < 0 ? 0 : last_key / pf::kBN + 1, make_int4(i, pr, 0, 0)});
    }
  }
  if (work.empty() || total == 0) return;
  std::stable_sort(work.begin(), work.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
  // device copy: [maps (64-B aligned)][reqs][work]
  const size_t maps_b = maps.size() * sizeof(CUtensorMap), reqs_b = reqs.size() * sizeof(int4),
               work_b = work.size() * sizeof(int4);
  std::vector<uint8_t> blob(maps_b + reqs_b + work_b);
  std::memcpy(blob.data(), maps.data(), maps_b);
  std::memcpy(blob.data() + maps_b, reqs.data(), reqs_b);
  for (size_t k = 0; k < work.size(); ++k) std::memcpy(blob.data() + maps_b + reqs_b + k * sizeof(int4), &work[k].second, sizeof(int4));
  // Schedule buffers per (thread, device): a ring of pinned host staging slots, each with a
  // device copy and an event, so a call never waits on the previous launch and the H2D copy is
  // a true async DMA (a pageable source may make the driver stage or serialise it).
  constexpr int kSlots = 4;
  struct Ring {
    void* host[kSlots] = {};
    void* dev[kSlots] = {};
    cudaEvent_t done[kSlots] = {};
    size_t cap[kSlots] = {};
    int next = 0;
  };
  static thread_local std::map<int, Ring> rings;
  int dev = 0;
  check_rt(cudaGetDevice(&dev), "cudaGetDevice");
  Ring& ring = rings[dev];
  const int k = ring.next;
  ring.next = (k + 1) % kSlots;
  if (ring.done[k]) check_rt(cudaEventSynchronize(ring.done[k]), "varlen slot reuse");   // 4 launches back
  else check_rt(cudaEventCreateWithFlags(&ring.done[k], cudaEventDisableTiming), "cudaEventCreate(varlen)");
  if (blob.size() > ring.cap[k]) {
    if (ring.host[k]) check_rt(cudaFreeHost(ring.host[k]), "cudaFreeHost(varlen)");
    if (ring.dev[k]) check_rt(cudaFree(ring.dev[k]), "cudaFree(varlen)");
    ring.cap[k] = std::max(blob.size(), (size_t)1 << 16);
    check_rt(cudaMallocHost(&ring.host[k], ring.cap[k]), "cudaMallocHost(varlen)");
    check_rt(cudaMalloc(&ring.dev[k], ring.cap[k]), "cudaMalloc(varlen)");
  }
  std::memcpy(ring.host[k], blob.data(), blob.size());
  void* dbuf = ring.dev[k];
  check_rt(cudaMemcpyAsync(dbuf, ring.host[k], blob.size(), cudaMemcpyHostToDevice, st), "varlen params H2D");
  cuuint64_t qd[3] = {(cuuint64_t)D, (cuuint64_t)hq, (cuuint64_t)total};
  cuuint64_t qs[2] = {(cuuint64_t)D * 2, (cuuint64_t)hq * D * 2};
  cuuint32_t qb[3] = {64, 1, (cuuint32_t)pf::kBM};
  const CUtensorMap qmap = make_map(const_cast<void*>(q), 3, qd, qs, qb);
  const CUtensorMap omap = make_map(out, 3, qd, qs, qb);
  pf::Params p{};
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.hq = hq;
  p.group = hq / v.hkv;
  p.head_pair = hp ? 1 : 0;
  const int heads_per_item = hp ? hq / 2 : hq;   // CTAs (items) per work entry
  p.causal = causal ? 1 : 0;
  if (scale <= 0.f) scale = 1.f / sqrtf((float)D);
  p.scale_log2 = scale * 1.4426950408889634f;
  p.maps = reinterpret_cast<const CUtensorMap*>(dbuf);
  p.reqs = reinterpret_cast<const int4*>(static_cast<uint8_t*>(dbuf) + maps_b);
  p.work = reinterpret_cast<const int4*>(static_cast<uint8_t*>(dbuf) + maps_b + reqs_b);
  // Persistent CTAs when the items are many and short (measured, tools/pf_persist_varlen_check.py:
  // 64 x 128 1.28x, 32 x 256 1.18x, 16 x 512 1.13x, 8 x 2048 1.08x, 4 x 3072 1.05x, bit-equal;
  // 2 x 8192 and 1 x 16384 (33 / 65 KV tiles per item) on par).  VATTN_PF_PERSIST=0 / 1 forces.
  static const int persist_env = [] {
    const char* e = getenv("VATTN_PF_PERSIST");
    return e ? atoi(e) : -1;
  }();
  int64_t tiles = 0;
  for (const auto& w_ : work) tiles += w_.first;
  const bool persist = persist_env >= 0 ? persist_env != 0
                                        : (int64_t)work.size() * heads_per_item > num_sms_cached() &&
                                              tiles <= 24 * (int64_t)work.size();
  if (D == 128 && persist) {
    const int n_items = (int)work.size() * heads_per_item;
    const int G = std::min(n_items, num_sms_cached());
    ensure_smem_attr<pf::prefill_persist_varlen_kernel>(pf::PfL<128>::kSmem);
    pf::prefill_persist_varlen_kernel<<<G, pf::kThreads, pf::PfL<128>::kSmem, st>>>(qmap, p, n_items);
    check_rt(cudaGetLastError(), "prefill (varlen, persistent) launch");
    check_rt(cudaEventRecord(ring.done[k], st), "varlen slot event");
    return;
  }
  const dim3 grid = pf::pf_grid(p, (unsigned)work.size(), heads_per_item);
  p.early_pv = early_pv_mode();
  if (D == 128) {
    ensure_smem_attr<pf::prefill_kernel<0, false, 128, true>>(pf::PfL<128>::kSmem);
    pf::prefill_kernel<0, false, 128, true><<<grid, pf::kThreads, pf::PfL<128>::kSmem, st>>>(qmap, qmap, qmap, omap, p);
  } else {
    ensure_smem_attr<pf::prefill_kernel<0, false, 64, true>>(pf::PfL<64>::kSmem);
    pf::prefill_kernel<0, false, 64, true><<<grid, pf::kThreads, pf::PfL<64>::kSmem, st>>>(qmap, qmap, qmap, omap, p);
  }
  check_rt(cudaGetLastError(), "prefill (varlen) launch");
  check_rt(cudaEventRecord(ring.done[k], st), "varlen slot event");
}

void launch_prefill_paged(const void* q, const void* k_pool, const void* v_pool, int num_blocks,
                          int block_size, int hkv, const int32_t* block_table, int kv_len, void* out,
                          int n_q, int hq, float scale, bool causal, cudaStream_t st) {
  if (hq % hkv) throw Fail(VATTN_VALUE_ERROR, "n_q_heads must be a multiple of n_kv_heads");
  if (block_size <= 0 || (block_size < pf::kBN && pf::kBN % block_size) ||
      (block_size >= pf::kBN && block_size % pf::kBN))
    throw Fail(VATTN_UNSUPPORTED, "block_size must divide 128 or be a multiple of 128");
  if (n_q <= 0 || kv_len <= 0) return;
  const int box = std::min(block_size, pf::kBN);
  cuuint64_t qd[3] = {(cuuint64_t)pf::kD, (cuuint64_t)hq, (cuuint64_t)n_q};
  cuuint64_t qs[2] = {(cuuint64_t)pf::kD * 2, (cuuint64_t)hq * pf::kD * 2};
  cuuint32_t qb[3] = {64, 1, (cuuint32_t)pf::kBM};
  const CUtensorMap qmap = make_map(const_cast<void*>(q), 3, qd, qs, qb);
  const CUtensorMap omap = make_map(out, 3, qd, qs, qb);
  const uint64_t row = (uint64_t)hkv * pf::kD * 2;
  cuuint64_t kd[4] = {(cuuint64_t)pf::kD, (cuuint64_t)hkv, (cuuint64_t)block_size, (cuuint64_t)num_blocks};
  cuuint64_t ks[3] = {(cuuint64_t)pf::kD * 2, row, row * block_size};
  cuuint32_t kb[4] = {64, 1, (cuuint32_t)box, 1};
  const CUtensorMap kmap = make_map(const_cast<void*>(k_pool), 4, kd, ks, kb);
  const CUtensorMap vmap = make_map(const_cast<void*>(v_pool), 4, kd, ks, kb);
  pf::Params p{};
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.n_q = n_q;
  p.hq = hq;
  p.group = hq / hkv;
  p.kv_len = kv_len;
  p.n_pairs = (n_q + 2 * pf::kBM - 1) / (2 * pf::kBM);
  p.q_off = kv_len - n_q;
  p.causal = causal ? 1 : 0;
  if (scale <= 0.f) scale = 1.f / sqrtf((float)pf::kD);
  p.scale_log2 = scale * 1.4426950408889634f;
  p.block_table = block_table;
  p.block_size = block_size;
  p.box_tokens = box;
  ensure_smem_attr<pf::prefill_kernel<0, true>>(pf::PfL<128, pf::kStages>::kSmem);
  const dim3 grid = pf::pf_grid(p, p.n_pairs, hq);
  pf::prefill_kernel<0, true><<<grid, pf::kThreads, pf::PfL<128, pf::kStages>::kSmem, st>>>(qmap, kmap, vmap, omap, p);
  check_rt(cudaGetLastError(), "prefill (paged) launch");
}

}  // namespace vattn

extern "C" vattn_status vattn_prefill_paged(const void* q, const void* k_pool, const void* v_pool,
                                            int32_t num_blocks, int32_t block_size, int32_t n_kv_heads,
                                            int32_t head_dim, const int32_t* block_table, int32_t kv_len,
                                            void* out, int32_t n_q, int32_t n_q_heads, float scale,
                                            int32_t causal, void* stream) {
  try {
    if (head_dim != vattn::pf::kD) throw vattn::Fail(VATTN_UNSUPPORTED, "prefill kernel is built for head_dim 128");
    vattn::launch_prefill_paged(q, k_pool, v_pool, num_blocks, block_size, n_kv_heads, block_table, kv_len, out,
                                n_q, n_q_heads, scale, causal != 0, (cudaStream_t)stream);
    return VATTN_OK;
  } catch (const vattn::Fail& e) {
    vattn::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    vattn::set_last_error(e.what());
    return VATTN_BAD_STATE;
  }
}

#ifdef VATTN_PF_TRACE
extern "C" int vattn_debug_prefill_cta(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, vattn::pf::g_pf_cta, sizeof(vattn::pf::g_pf_cta));
}
extern "C" int vattn_debug_prefill_trace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, vattn::pf::g_pf_trace, sizeof(vattn::pf::g_pf_trace));
}
#endif

extern "C" vattn_status vattn_prefill_varlen_raw(const vattn_cache_desc* c, const void* q, void* out,
                                                 int32_t n_q_heads, int32_t n_req, const int32_t* q_start,
                                                 const int32_t* n_q, const int32_t* slots, const int32_t* kv_len,
                                                 float scale, int32_t causal, void* stream) {
  try {
    vattn::launch_prefill_varlen(vattn::view_from_desc(c), q, out, n_q_heads, n_req, q_start, n_q, slots, kv_len,
                                 scale, causal != 0, (cudaStream_t)stream);
    return VATTN_OK;
  } catch (const vattn::Fail& e) {
    vattn::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    vattn::set_last_error(e.what());
    return VATTN_BAD_STATE;
  }
}

extern "C" vattn_status vattn_prefill_rotary_raw(const vattn_cache_desc* c, const void* q, void* out, int32_t n_q,
                                                 int32_t hq, int32_t slot, int32_t kv_len, float scale,
                                                 int32_t causal, const vattn_rotary* rotary, void* stream) {
  try {
    if (!rotary) throw vattn::Fail(VATTN_VALUE_ERROR, "null rotary descriptor");
    const vattn::Rotary rot{rotary->cos, rotary->sin, rotary->rotary_dim, rotary->interleaved};
    vattn::launch_prefill(nullptr, -1, vattn::view_from_desc(c), q, out, n_q, hq, slot, kv_len, scale,
                          causal != 0, (cudaStream_t)stream, &rot);
    return VATTN_OK;
  } catch (const vattn::Fail& e) {
    vattn::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    vattn::set_last_error(e.what());
    return VATTN_BAD_STATE;
  }
}

extern "C" vattn_status vattn_prefill_raw(const vattn_cache_desc* c, const void* q, void* out, int32_t n_q,
                                          int32_t hq, int32_t slot, int32_t kv_len, float scale,
                                          int32_t causal, void* stream) {
  try {
    vattn::launch_prefill(nullptr, -1, vattn::view_from_desc(c), q, out, n_q, hq, slot, kv_len, scale,
                          causal != 0, (cudaStream_t)stream);
    return VATTN_OK;
  } catch (const vattn::Fail& e) {
    vattn::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    vattn::set_last_error(e.what());
    return VATTN_BAD_STATE;
  }
}
