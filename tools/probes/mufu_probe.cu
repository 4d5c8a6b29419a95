// MUFU.EX2 issue/throughput probe: cycles per warp-level ex2 with W warps per SM sub-partition,
// alone and interleaved with the FFMA2/FMNMX3/FADD2/F2FP mix the prefill softmax issues per pair.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int MODE>
__global__ void probe(float* out, long long* cyc, int iters) {
  float v[16];
  for (int i = 0; i < 16; ++i) v[i] = -0.001f * (threadIdx.x + i);
  float m = -1e30f;
  float2 acc = make_float2(0.f, 0.f);
  unsigned pk = 0;
  float pp[16];
  for (int i = 0; i < 16; ++i) pp[i] = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) {
        v[i] = ex2(v[i]);
        v[i + 1] = ex2(v[i + 1]);
      } else if (MODE == 8) {   // full mix, consumers one iteration behind the ex2s
        float mm;
        asm("max.f32 %0, %1, %2, %3;" : "=f"(mm) : "f"(m), "f"(v[i]), "f"(v[i + 1]));
        m = mm;
        acc = __fadd2_rn(acc, make_float2(pp[i], pp[i + 1]));
        __nv_bfloat162 b = __floats2bfloat162_rn(pp[i], pp[i + 1]);
        pk ^= *reinterpret_cast<unsigned*>(&b);
        float2 xx = __ffma2_rn(make_float2(v[i], v[i + 1]), make_float2(0.5f, 0.5f), make_float2(-0.25f, -0.25f));
        pp[i] = ex2(xx.x);
        pp[i + 1] = ex2(xx.y);
        v[i] = __uint_as_float(__float_as_uint(v[i]) ^ 1u);
        v[i + 1] = __uint_as_float(__float_as_uint(v[i + 1]) ^ 1u);
      } else if (MODE == 4) {   // ex2 + FFMA2 only
        float2 xx = __ffma2_rn(make_float2(v[i], v[i + 1]), make_float2(0.5f, 0.5f), make_float2(-0.25f, -0.25f));
        v[i] = ex2(xx.x);
        v[i + 1] = ex2(xx.y);
      } else if (MODE == 5) {   // ex2 + FMNMX3 only
        float mm;
        asm("max.f32 %0, %1, %2, %3;" : "=f"(mm) : "f"(m), "f"(v[i]), "f"(v[i + 1]));
        m = mm;
        v[i] = ex2(v[i]);
        v[i + 1] = ex2(v[i + 1]);
      } else if (MODE == 6) {   // ex2 + FADD2 only
        float p0 = ex2(v[i]), p1 = ex2(v[i + 1]);
        acc = __fadd2_rn(acc, make_float2(p0, p1));
        v[i] = p0;
        v[i + 1] = p1;
      } else if (MODE == 7) {   // ex2 + F2FP only
        float p0 = ex2(v[i]), p1 = ex2(v[i + 1]);
        __nv_bfloat162 b = __floats2bfloat162_rn(p0, p1);
        pk ^= *reinterpret_cast<unsigned*>(&b);
        v[i] = p0;
        v[i + 1] = p1;
      } else {
        float mm;
        asm("max.f32 %0, %1, %2, %3;" : "=f"(mm) : "f"(m), "f"(v[i]), "f"(v[i + 1]));
        m = mm;
        float2 xx = __ffma2_rn(make_float2(v[i], v[i + 1]), make_float2(0.5f, 0.5f), make_float2(-0.25f, -0.25f));
        float p0 = ex2(xx.x), p1 = ex2(xx.y);
        acc = __fadd2_rn(acc, make_float2(p0, p1));
        if (MODE == 1) {          // F2FP.BF16.F32.PACK_AB
          __nv_bfloat162 b = __floats2bfloat162_rn(p0, p1);
          pk ^= *reinterpret_cast<unsigned*>(&b);
        } else if (MODE == 2) {   // truncating pack on the integer pipe (PRMT)
          unsigned r;
          asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(__float_as_uint(p0)), "r"(__float_as_uint(p1)));
          pk ^= r;
        } else if (MODE == 3) {   // round-to-nearest-even on the integer pipe, then PRMT
          unsigned u0 = __float_as_uint(p0), u1 = __float_as_uint(p1);
          u0 = u0 + 0x7FFFu + ((u0 >> 16) & 1u);
          u1 = u1 + 0x7FFFu + ((u1 >> 16) & 1u);
          unsigned r;
          asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(u0), "r"(u1));
          pk ^= r;
        }
        v[i] = p0 - 0.5f;
        v[i + 1] = p1 - 0.5f;
      }
    }
  }
  long long t1 = clock64();
  float s = m + acc.x + acc.y + __uint_as_float(pk);
  for (int i = 0; i < 16; ++i) s += pp[i];
  for (int i = 0; i < 16; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x % 32 == 0) cyc[blockIdx.x * 64 + threadIdx.x / 32] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 64 * 8);
  const int iters = 4096;
  for (int mode : {0, 1, 2, 3, 4, 5, 6, 7, 8}) {
    for (int warps : {4, 8}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) probe<0><<<148, warps * 32>>>(out, cyc, iters);
        else if (mode == 1) probe<1><<<148, warps * 32>>>(out, cyc, iters);
        else if (mode == 2) probe<2><<<148, warps * 32>>>(out, cyc, iters);
        else if (mode == 3) probe<3><<<148, warps * 32>>>(out, cyc, iters);
        else if (mode == 4) probe<4><<<148, warps * 32>>>(out, cyc, iters);
        else if (mode == 5) probe<5><<<148, warps * 32>>>(out, cyc, iters);
        else if (mode == 6) probe<6><<<148, warps * 32>>>(out, cyc, iters);
        else if (mode == 7) probe<7><<<148, warps * 32>>>(out, cyc, iters);
        else probe<8><<<148, warps * 32>>>(out, cyc, iters);
      }
      cudaDeviceSynchronize();
      long long h[64];
      cudaMemcpy(h, cyc, 64 * 8, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
      const double ex2_per_warp = 16.0 * iters;
      printf("mode %s warps/SM %2d (per SMSP %d): %.2f cycles per warp-ex2 per warp; SMSP ex2 rate %.2f lanes/clk\n",
             mode == 0 ? "ex2-only" : mode == 1 ? "mix F2FP" : mode == 2 ? "mix PRMT-trunc" : mode == 3 ? "mix int-RN" : mode == 4 ? "ex2+FFMA2" : mode == 5 ? "ex2+FMNMX3" : mode == 6 ? "ex2+FADD2" : mode == 7 ? "ex2+F2FP" : "mix pipelined", warps, warps / 4, mx / ex2_per_warp,
             (warps / 4) * ex2_per_warp * 32 / mx);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
