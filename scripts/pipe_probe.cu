// Issue-throughput probe for the fp8 decode instructions (not part of the library):
// each thread runs 8 independent chains of the op under test; reports ops/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

template <int OP>
__global__ void probe(uint32_t* out, int iters) {
  uint32_t x[8];
  float f[8];
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 2654435761u + i; f[i] = float(i); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) {  // F2FP e4m3x2 -> f16x2
        uint32_t h;
        asm volatile("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h) : "h"(static_cast<unsigned short>(x[i])));
        x[i] = h;
      } else if (OP == 1) {  // f16 -> f32 (HADD2.F32)
        __half hh = __ushort_as_half(static_cast<unsigned short>(x[i]));
        float v = __half2float(hh);
        x[i] = __float_as_uint(v) >> 16;
      } else if (OP == 2) {  // FFMA2
        unsigned long long a, c;
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(f[i]), "f"(f[(i + 1) & 7]));
        asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(c) : "l"(a));
        float lo, hi;
        asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(c));
        f[i] = lo + hi;
      } else if (OP == 3) {  // PRMT
        uint32_t p;
        asm volatile("prmt.b32 %0, %1, 0, 0x9180;" : "=r"(p) : "r"(x[i]));
        x[i] = p;
      } else if (OP == 4) {  // FFMA
        f[i] = fmaf(f[i], 1.0001f, 0.5f);
      }
    }
  }
  uint32_t acc = 0;
  for (int i = 0; i < 8; ++i) acc ^= x[i] ^ __float_as_uint(f[i]);
  if (acc == 0x12345678u) out[0] = acc;
}

template <int OP>
void run(const char* name, int warps) {
  uint32_t* out;
  cudaMalloc(&out, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096;
  probe<OP><<<sms, warps * 32>>>(out, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<OP><<<sms, warps * 32>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = double(sms) * warps * 32 * iters * 8;
  const double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
  printf("%-6s warps %2d: %.1f ops/clk/SM (%.3f ms)\n", name, warps, per_clk_sm, ms);
  cudaFree(out);
}

int main() {
  for (int w : {8, 16, 32}) {
    run<0>("F2FP", w);
    run<1>("H2F32", w);
    run<2>("FFMA2", w);
    run<3>("PRMT", w);
    run<4>("FFMA", w);
  }
  return 0;
}
