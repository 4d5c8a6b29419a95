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
                         "ffma2 (f32x2)", "exp2_poly2 (per pair)"};
  for (int m = 0; m < 6; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) probe<0><<<148, 512>>>(o, c);
      if (m == 1) probe<1><<<148, 512>>>(o, c);
      if (m == 2) probe<2><<<148, 512>>>(o, c);
      if (m == 3) probe<3><<<148, 512>>>(o, c);
      if (m == 4) probe<4><<<148, 512>>>(o, c);
      if (m == 5) probe<5><<<148, 512>>>(o, c);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", names[m], cudaGetErrorString(e)); continue; }
    long long h[148];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < 148; ++i) cyc += h[i];
    cyc /= 148;
    // thread-level operations per SM (one CTA per SM); modes 4/5 do 4 packed ops per 8 registers
    const double instr = 512.0 * kIters * ((m >= 4) ? 4 : 8);
    const double results = instr * ((m == 0 || m == 3) ? 1 : 2);
    printf("%-24s %6.2f instr/clk/SM  %6.2f results/clk/SM\n", names[m], instr / cyc, results / cyc);
  }
  return 0;
}
