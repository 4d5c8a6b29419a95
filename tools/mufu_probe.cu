// MUFU exp2 throughput on B200: f32 vs packed bf16x2 / f16x2 (results per SM per cycle).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_probe.cu -o tools/mufu_probe.bin
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

constexpr int kIters = 4096;

// the prefill kernel's FMA-pipe exp2 (prefill.cu exp2_poly2), on a pair
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 n = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-n.x, -n.y));
  float2 q = __ffma2_rn(f, make_float2(0.05286731580314504f, 0.05286731580314504f),
                        make_float2(0.2421521458456525f, 0.2421521458456525f));
  q = __ffma2_rn(q, f, make_float2(0.6935868335103712f, 0.6935868335103712f));
  q = __ffma2_rn(q, f, make_float2(0.9999627473381362f, 0.9999627473381362f));
  const int ex = __float_as_int(t.x) << 23, ey = __float_as_int(t.y) << 23;
  return make_float2(__int_as_float(__float_as_int(q.x) + ex), __int_as_float(__float_as_int(q.y) + ey));
}

template <int MODE>
__global__ void probe(float* out, long long* cyc) {
  uint32_t v[8];
  for (int i = 0; i < 8; ++i) v[i] = __float_as_uint(-0.001f * (threadIdx.x + i));
  if (MODE != 0)
    for (int i = 0; i < 8; ++i) v[i] = 0x3c003c00u ^ (threadIdx.x + i);   // small packed halves
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(v[i]));
      if (MODE == 1) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[i]));
      if (MODE == 2) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
      if (MODE == 3) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f38000000;" : "+r"(v[i]));
      if (MODE == 4 && (i & 1) == 0) {   // 4 independent packed chains (pairs 0-1, 2-3, ...)
        float2 a = make_float2(__uint_as_float(v[i]), __uint_as_float(v[i + 1]));
        a = __ffma2_rn(a, make_float2(0.99999f, 0.99999f), make_float2(1e-5f, 1e-5f));
        v[i] = __float_as_uint(a.x); v[i + 1] = __float_as_uint(a.y);
      }
      if (MODE == 6 && (i & 1) == 0) {   // F2FP pack (cvt.rn.bf16x2.f32) on 4 independent pairs
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(__uint_as_float(v[i])), "f"(__uint_as_float(v[i + 1])));
        v[i] ^= r;
      }
      if (MODE == 7 && (i & 1) == 0) {   // 2 x MUFU ex2 + 1 F2FP per pair
        float e0, e1;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(__uint_as_float(v[i])));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(__uint_as_float(v[i + 1])));
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(e1), "f"(e0));
        v[i] ^= r;
        v[i + 1] = __float_as_uint(e1) & 0xBFFFFFFFu;
      }
      if (MODE == 8 && (i & 1) == 0) {   // the prefill softmax mix per pair: FMNMX3, FFMA2, 2 MUFU, FADD2, F2FP
        const float a = __uint_as_float(v[i]), b = __uint_as_float(v[i + 1]);
        float m;
        asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(m) : "f"(__uint_as_float(v[(i + 2) & 7])), "f"(a), "f"(b));
        const float2 x = __ffma2_rn(make_float2(a, b), make_float2(0.125f, 0.125f), make_float2(-m, -m));
        float e0, e1;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(x.x));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(x.y));
        const float2 acc = __fadd2_rn(make_float2(e0, e1), make_float2(a, b));
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(e1), "f"(e0));
        v[i] = (__float_as_uint(acc.x) ^ r) & 0xBFFFFFFFu;
        v[i + 1] = __float_as_uint(acc.y) & 0xBFFFFFFFu;
      }
      if (MODE == 5 && (i & 1) == 0) {   // polynomial exp2 on 4 independent pairs; input kept in [-1, 0]
        float2 a = make_float2(__uint_as_float(v[i]), __uint_as_float(v[i + 1]));
        a = exp2_poly2(a);
        v[i] = __float_as_uint(-a.x); v[i + 1] = __float_as_uint(-a.y);
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  uint32_t acc = 0;
  for (int i = 0; i < 8; ++i) acc ^= v[i];
  if (acc == 0x12345) out[0] = 1.f;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* o;
  long long* c;
  cudaMalloc(&o, 4);
  cudaMalloc(&c, 1024 * 8);
  const char* names[] = {"ex2.approx.ftz.f32", "ex2.approx.ftz.bf16x2", "ex2.approx.f16x2", "fma.rn.f32",
                         "ffma2 (f32x2)", "exp2_poly2 (per pair)", "cvt.rn.bf16x2.f32", "2 ex2 + 1 cvt (pair)",
                         "softmax mix (pair)"};
  for (int threads : {512, 128}) {
    printf("--- %d threads per SM (%d warps per sub-partition)\n", threads, threads / 128);
    for (int m = 0; m < 9; ++m) {
      for (int rep = 0; rep < 2; ++rep) {
        if (m == 0) probe<0><<<148, threads>>>(o, c);
        if (m == 1) probe<1><<<148, threads>>>(o, c);
        if (m == 2) probe<2><<<148, threads>>>(o, c);
        if (m == 3) probe<3><<<148, threads>>>(o, c);
        if (m == 4) probe<4><<<148, threads>>>(o, c);
        if (m == 5) probe<5><<<148, threads>>>(o, c);
        if (m == 6) probe<6><<<148, threads>>>(o, c);
        if (m == 7) probe<7><<<148, threads>>>(o, c);
        if (m == 8) probe<8><<<148, threads>>>(o, c);
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s: %s\n", names[m], cudaGetErrorString(e)); continue; }
      long long h[148];
      cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < 148; ++i) cyc += h[i];
      cyc /= 148;
      // thread-level operations per SM (one CTA per SM); modes >= 4 do 4 packed ops per 8 registers
      const double instr = (double)threads * kIters * ((m >= 4) ? 4 : 8);
      const double results = instr * ((m == 0 || m == 3 || m == 6) ? 1 : 2);
      printf("%-24s %6.2f instr/clk/SM  %6.2f results/clk/SM\n", names[m], instr / cyc, results / cyc);
    }
  }
  return 0;
}
