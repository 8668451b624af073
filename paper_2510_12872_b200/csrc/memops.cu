// Insert-path and concatenation kernels:
//   * measure_kernel — offset measurement of Algorithm 1's fallback branch:
//       ΔK = R_{-(s_real - s_base)} K_real - K_base,  ΔV = V_real - V_base   (step a0)
//     written straight into the pool slab, fp32 math, one RNE rounding to bf16.
//   * copy_rows_kernel — strided [Ls][Hs][rows][d] row-block copy (p_(m,0) into the
//     consumer's prompt cache for the concatenation, P:304 / Alg. 1; GIVEN
//     offsets and embeddings into the pool slab).
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include "kvcomm_internal.h"
#include "ptx.cuh"

namespace kvc {

// One thread per 16-byte vector; rows are d elements = d/8 vectors.
__global__ void copy_rows_kernel(const bf16* __restrict__ src, int64_t src_ld, bf16* __restrict__ dst,
                                 int64_t dst_ld, int Hs, int rows, int vpr, int64_t total) {
  for (int64_t x = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < total;
       x += int64_t(gridDim.x) * blockDim.x) {
    const int v = int(x % vpr);
    int64_t r = x / vpr;
    const int i = int(r % rows);
    const int64_t lh = r / rows;
    const uint4 val = ldg128_nc(src + (lh * src_ld + i) * (vpr * 8) + v * 8);
    *reinterpret_cast<uint4*>(dst + (lh * dst_ld + i) * (vpr * 8) + v * 8) = val;
  }
}

__global__ void copy_flat_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t nvec) {
  for (int64_t x = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < nvec;
       x += int64_t(gridDim.x) * blockDim.x)
    dst[x] = ldg128_nc(src + x);
}

static int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  const int64_t cap = 148 * 16;
  if (g > cap) g = cap;
  return g < 1 ? 1 : int(g);
}

cudaError_t launch_copy_rows(const bf16* src, int64_t src_ld, bf16* dst, int64_t dst_ld, int Ls, int Hs,
                             int rows, int d, cudaStream_t s) {
  const int vpr = d / 8;
  const int64_t total = int64_t(Ls) * Hs * rows * vpr;
  if (total == 0) return cudaSuccess;
  copy_rows_kernel<<<grid_for(total, 256), 256, 0, s>>>(src, src_ld, dst, dst_ld, Hs, rows, vpr, total);
  return cudaGetLastError();
}

cudaError_t launch_copy_flat(const bf16* src, bf16* dst, int64_t n, cudaStream_t s) {
  const int64_t nvec = n / 8;
  if (nvec == 0) return cudaSuccess;
  copy_flat_kernel<<<grid_for(nvec, 256), 256, 0, s>>>(reinterpret_cast<const uint4*>(src),
                                                       reinterpret_cast<uint4*>(dst), nvec);
  return cudaGetLastError();
}

// Items = (row, vector-pair v): 8 elements of the first half and the matching 8 of
// the second half of a d-element row, so the rotate_half pair (f, f+d/2) stays in
// one thread.  cos/sin of δ·inv_freq[f] (fp64 angle) are tabled in shared memory.
__global__ void measure_kernel(const bf16* __restrict__ kr, const bf16* __restrict__ vr, int64_t real_ld,
                               const bf16* __restrict__ kb, const bf16* __restrict__ vb, int64_t base_ld,
                               int rows, int Hs, int d, int delta, const double* __restrict__ inv_freq,
                               bf16* __restrict__ dk, bf16* __restrict__ dv, int64_t dst_ld, int64_t total) {
  __shared__ float2 cs[128];
  const int half = d / 2;
  for (int f = threadIdx.x; f < half; f += blockDim.x) {
    double sn, cn;
    sincos(double(delta) * inv_freq[f], &sn, &cn);
    cs[f] = make_float2(float(cn), float(sn));
  }
  __syncthreads();
  const int vph = d / 16;  // vector pairs per row
  for (int64_t x = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < total;
       x += int64_t(gridDim.x) * blockDim.x) {
    const int v = int(x % vph);
    const int64_t r = x / vph;
    const int i = int(r % rows);
    const int64_t lh = r / rows;
    const int64_t ro = (lh * real_ld + i) * d + v * 8;
    const int64_t bo = (lh * base_ld + i) * d + v * 8;
    const int64_t oo = (lh * dst_ld + i) * d + v * 8;
    const uint4 ka = ldg128_nc(kr + ro), kb2 = ldg128_nc(kr + ro + half);
    const uint4 ba = ldg128_nc(kb + bo), bb = ldg128_nc(kb + bo + half);
    const uint4 va = ldg128_nc(vr + ro), vb2 = ldg128_nc(vr + ro + half);
    const uint4 wa = ldg128_nc(vb + bo), wb = ldg128_nc(vb + bo + half);
    const uint32_t k0[4] = {ka.x, ka.y, ka.z, ka.w}, k1[4] = {kb2.x, kb2.y, kb2.z, kb2.w};
    const uint32_t b0[4] = {ba.x, ba.y, ba.z, ba.w}, b1[4] = {bb.x, bb.y, bb.z, bb.w};
    const uint32_t v0[4] = {va.x, va.y, va.z, va.w}, v1[4] = {vb2.x, vb2.y, vb2.z, vb2.w};
    const uint32_t w0[4] = {wa.x, wa.y, wa.z, wa.w}, w1[4] = {wb.x, wb.y, wb.z, wb.w};
    uint32_t ok0[4], ok1[4], ov0[4], ov1[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float y0[2], y1[2];
      const float x0[2] = {bf_lo(k0[e]), bf_hi(k0[e])};
      const float x1[2] = {bf_lo(k1[e]), bf_hi(k1[e])};
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const float2 c = cs[v * 8 + 2 * e + t];
        y0[t] = x0[t] * c.x - x1[t] * c.y;
        y1[t] = x1[t] * c.x + x0[t] * c.y;
      }
      ok0[e] = pack_bf16_rn(y0[0] - bf_lo(b0[e]), y0[1] - bf_hi(b0[e]));
      ok1[e] = pack_bf16_rn(y1[0] - bf_lo(b1[e]), y1[1] - bf_hi(b1[e]));
      ov0[e] = pack_bf16_rn(bf_lo(v0[e]) - bf_lo(w0[e]), bf_hi(v0[e]) - bf_hi(w0[e]));
      ov1[e] = pack_bf16_rn(bf_lo(v1[e]) - bf_lo(w1[e]), bf_hi(v1[e]) - bf_hi(w1[e]));
    }
    *reinterpret_cast<uint4*>(dk + oo) = make_uint4(ok0[0], ok0[1], ok0[2], ok0[3]);
    *reinterpret_cast<uint4*>(dk + oo + half) = make_uint4(ok1[0], ok1[1], ok1[2], ok1[3]);
    *reinterpret_cast<uint4*>(dv + oo) = make_uint4(ov0[0], ov0[1], ov0[2], ov0[3]);
    *reinterpret_cast<uint4*>(dv + oo + half) = make_uint4(ov1[0], ov1[1], ov1[2], ov1[3]);
  }
}

cudaError_t launch_measure(const bf16* k_real, const bf16* v_real, int64_t real_ld, const bf16* k_base,
                           const bf16* v_base, int64_t base_ld, int rows, int Ls, int Hs, int d, int delta,
                           const double* inv_freq, bf16* dk, bf16* dv, int64_t dst_ld, cudaStream_t s) {
  const int64_t total = int64_t(Ls) * Hs * rows * (d / 16);
  if (total == 0) return cudaSuccess;
  measure_kernel<<<grid_for(total, 256), 256, 0, s>>>(k_real, v_real, real_ld, k_base, v_base, base_ld, rows,
                                                       Hs, d, delta, inv_freq, dk, dv, dst_ld, total);
  return cudaGetLastError();
}

}  // namespace kvc
