// tcgen05 issue-pattern probe: cycles per 128x128x128 bf16 unit for the MMA sequences the
// prefill pipelines issue, with and without a TMEM write-after-read hazard between a TS-MMA that
// reads P from TMEM and the next SS-MMA that overwrites those columns.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2405_04437_b200/csrc \
//        tools/mma_probe.cu -o /tmp/mma_probe -lcuda && /tmp/mma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#include "ptx.cuh"

using namespace vattn;

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(bool b_mn_major, int n = 128) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) |
         ((128 >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
               ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   ptx::smem_u32(bar)) : "memory");
}

constexpr int kReps = 64;
constexpr int kHalf = 16384, kTile = 32768;

__global__ void __launch_bounds__(288, 1) probe(int mode, int bg, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 3 * kTile);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  volatile int* stop = reinterpret_cast<volatile int*>(bar + 3);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { ptx::mbar_init(bar, 1); ptx::fence_mbar_init(); *stop = 0; }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(ptx::smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *slot;
  if (warp < 8 && bg != 0) {
    // background "softmax" warps on TMEM lanes (warp%4)*32, columns of tile warp/4 (S region)
    const uint32_t base = tmem + (((warp % 4) * 32) << 16) + (warp / 4) * 128;
    float acc = 0.f;
    uint32_t r[32];
    while (*stop == 0) {
      for (int c0 = 0; c0 < 128; c0 += 32) {
        if (bg == 1 || bg == 3) {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                       "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                       : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                         "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                         "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
                         "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
                         "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                       : "r"(base + c0));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        } else {
          for (int c = 0; c < 32; ++c) r[c] = __float_as_uint(acc + c);
        }
        for (int c = 0; c < 32; ++c) acc += ptx::fast_exp2(__uint_as_float(r[c]) * 1e-3f);
        if (bg == 3) {
          asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                       ::"r"(base + c0 / 2), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
                         "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),
                         "r"(r[14]), "r"(r[15]) : "memory");
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
      }
    }
    if (acc == 12345.f) out[15] = 1;
  }
  if (threadIdx.x == 256) {
    const uint32_t sb = ptx::smem_u32(sm);
    const uint32_t qa = sb, kb = sb + kTile, vb = sb + 2 * kTile;
    const uint32_t iq = idesc(false), iq64 = idesc(false, 64), iv = idesc(true);
    auto S = [&](uint32_t dcol, int keys0, int n) {     // S[:, dcol:dcol+n] = Q K[keys0:keys0+n]^T
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
        mma_ss(tmem + dcol, sdesc(qa + off, 16, 1024), sdesc(kb + keys0 * 128 + off, 16, 1024),
               n == 64 ? iq64 : iq, kk > 0);
      }
    };
    auto PV = [&](uint32_t pcol, int k0, int k1) {    // O(256) += P[pcol..] V[k-steps k0..k1)
      for (int kk = k0; kk < k1; ++kk)
        mma_ts(tmem + 256, tmem + pcol + (kk - k0) * 8, sdesc(vb + kk * 2048, kHalf, 1024), iv, 1);
    };
    const long long t0 = clock64();
    for (int r = 0; r < kReps; ++r) {
      switch (mode) {
        case 0: S(0, 0, 128); break;                                        // 1 unit
        case 1: S(0, 0, 64); S(64, 64, 64); break;                          // 1 unit, N=64 halves
        case 2: PV(0, 0, 8); S(0, 0, 128); break;                           // 2 units, WAR on cols 0-63
        case 3: PV(0, 0, 8); S(128, 0, 128); break;                         // 2 units, no hazard
        case 4: PV(0, 0, 8); break;                                         // 1 unit
        case 5: PV(0, 0, 4); S(0, 0, 64); PV(64, 4, 8); S(64, 64, 64); break;       // split, hazards
        case 6: PV(0, 0, 4); S(128, 0, 64); PV(64, 4, 8); S(192, 64, 64); break;    // split, none
        case 7: PV(0, 0, 8); S(0, 0, 128); PV(128, 0, 8); S(128, 0, 128); break;    // A/B ping-pong (old)
      }
    }
    commit(bar);
    ptx::mbar_wait(bar, 0);
    const long long t1 = clock64();
    out[mode] = (unsigned long long)(t1 - t0);
    *stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16 * sizeof(unsigned long long));
  const int smem = 3 * kTile + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"S N=128", "S 2x N=64", "PV+S WAR", "PV+S no-hazard", "PV only",
                         "split PV/S halves WAR", "split PV/S halves no-hazard", "ping-pong A/B (old)"};
  const double units[] = {1, 1, 2, 2, 1, 2, 2, 4};
  const char* bgn[] = {"idle", "tmem.ld", "mufu only", "tmem.ld+st"};
  for (int bg = 0; bg < 4; ++bg)
    for (int m = 0; m < 8; ++m) {
      if (bg && !(m == 5 || m == 7 || m == 0)) continue;
      for (int it = 0; it < 3; ++it) probe<<<1, 288, smem>>>(m, bg, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long c[16];
      cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
      printf("[bg %-10s] %-30s %8.1f cycles per 128^3 unit (ideal 512)\n", bgn[bg], names[m], c[m] / (kReps * units[m]));
    }
  // same, all SMs busy (148 CTAs) -- clocks under load
  return 0;
}
