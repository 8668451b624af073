// HBM bandwidth probe for the realign roofline (not part of the product library).
// Measures, on one B200, the achievable DRAM bandwidth of access patterns the
// realign kernel could use:
//   tma_read   : persistent CTAs stream CHUNK-byte cp.async.bulk tiles through an
//                NSTAGE ring (data discarded) — read-only roofline of the TMA path
//   ldg_read   : LDG.128 x UNROLL per thread, grid-stride, xor-reduced
//   tma_mix    : TMA read of 22 chunks per 1 chunk written (realign's 21:1 ratio)
//   copy       : LDG/STG copy (what MEASURED_PEAKS.json's hbm_gbs measures)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o bw_probe bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(
                   smem_u32(b)),
               "r"(ph)
               : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(n), "r"(smem_u32(b)), "l"(pol)
      : "memory");
}

// Each CTA: 1 producer lane + 1 consumer warp.  Streams chunks ids blockIdx.x, +grid...
__global__ void tma_read(const uint8_t* src, int64_t nchunks, int chunk, int nstage, uint8_t* wdst, int wevery) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(nstage) * chunk);
  uint64_t* empty = full + nstage;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nstage; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (threadIdx.x >= 32) {
    if (threadIdx.x == 32) {
      int st = 0; uint32_t ph = 0;
      for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        mbar_wait(&empty[st], ph ^ 1);
        mbar_expect(&full[st], chunk);
        bulk(sm + size_t(st) * chunk, src + c * chunk, chunk, &full[st], pol);
        if (++st == nstage) { st = 0; ph ^= 1; }
      }
    }
    return;
  }
  int st = 0; uint32_t ph = 0;
  int64_t k = 0;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
    mbar_wait(&full[st], ph);
    if (wevery > 0 && (k % wevery) == 0) {
      // write one chunk from smem (realign's output share)
      const uint4* s = reinterpret_cast<const uint4*>(sm + size_t(st) * chunk);
      // k-th write of this CTA -> a distinct chunk (no L2 merging of writes)
      const int64_t wi = (k / wevery) * gridDim.x + blockIdx.x;
      uint4* d = reinterpret_cast<uint4*>(wdst + wi * chunk);
      for (int i = threadIdx.x; i < chunk / 16; i += 32) d[i] = s[i];
    }
    __syncwarp();
    if (threadIdx.x == 0) mbar_arrive(&empty[st]);
    if (++st == nstage) { st = 0; ph ^= 1; }
  }
}

// Read stream of 16 KiB TMA tiles; every `wevery`-th tile is written back to a
// distinct destination with a TMA bulk store (mode 0: no hint, 1: evict_first,
// 2: evict_last, 3: per-thread st.global.cs, 4: per-thread st.global.wb).
__global__ void tma_mix_store(const uint8_t* src, int64_t nchunks, int chunk, int nstage, uint8_t* wdst, int wevery,
                              int mode) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(nstage) * chunk);
  uint64_t* empty = full + nstage;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nstage; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t pol, pst;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (mode == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pst));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pst));
  if (threadIdx.x >= 32) {
    if (threadIdx.x == 32) {
      int st = 0; uint32_t ph = 0;
      for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        mbar_wait(&empty[st], ph ^ 1);
        mbar_expect(&full[st], chunk);
        bulk(sm + size_t(st) * chunk, src + c * chunk, chunk, &full[st], pol);
        if (++st == nstage) { st = 0; ph ^= 1; }
      }
    }
    return;
  }
  int st = 0; uint32_t ph = 0;
  int64_t k = 0;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
    mbar_wait(&full[st], ph);
    bool wrote = false;
    if ((k % wevery) == 0) {
      const int64_t wi = (k / wevery) * gridDim.x + blockIdx.x;
      uint8_t* d = wdst + wi * chunk;
      const uint8_t* sp = sm + size_t(st) * chunk;
      if (mode <= 2) {
        if (threadIdx.x == 0) {
          if (mode == 0)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(smem_u32(sp)),
                         "r"(chunk) : "memory");
          else
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(d),
                         "r"(smem_u32(sp)), "r"(chunk), "l"(pst) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        wrote = true;
      } else {
        const uint4* s4 = reinterpret_cast<const uint4*>(sp);
        uint4* d4 = reinterpret_cast<uint4*>(d);
        for (int i = threadIdx.x; i < chunk / 16; i += 32) {
          uint4 v = s4[i];
          if (mode == 3)
            asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(d4 + i), "r"(v.x), "r"(v.y), "r"(v.z),
                         "r"(v.w) : "memory");
          else
            d4[i] = v;
        }
      }
    }
    __syncwarp();
    if (threadIdx.x == 0) mbar_arrive(&empty[st]);
    (void)wrote;
    if (++st == nstage) { st = 0; ph ^= 1; }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA read of `chunk`-byte tiles where every tile also pulls `nsmall` 256-byte side
// slices (one from an L2-resident table, the rest from DRAM), as the fp8 realign does.
// Realign's anchor-major access: CTA b takes units u = b, b + grid, ...; per unit it
// streams the unit's chunk of each of K anchors, anchor j at j * stride + u * chunk
// (the pool slab layout [slot][...]), or at (u * K + j) * chunk when stride == 0
// (anchors of one unit contiguous).
__global__ void tma_gather(const uint8_t* src, int64_t units, int K, int64_t stride, int chunk, int nstage) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(nstage) * chunk);
  uint64_t* empty = full + nstage;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nstage; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (threadIdx.x >= 32) {
    if (threadIdx.x == 32) {
      int st = 0; uint32_t ph = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x)
        for (int j = 0; j < K; ++j) {
          const int64_t off = stride ? j * stride + u * chunk : (u * K + j) * chunk;
          mbar_wait(&empty[st], ph ^ 1);
          mbar_expect(&full[st], chunk);
          bulk(sm + size_t(st) * chunk, src + off, chunk, &full[st], pol);
          if (++st == nstage) { st = 0; ph ^= 1; }
        }
    }
    return;
  }
  int st = 0; uint32_t ph = 0;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x)
    for (int j = 0; j < K; ++j) {
      mbar_wait(&full[st], ph);
      __syncwarp();
      if (threadIdx.x == 0) mbar_arrive(&empty[st]);
      if (++st == nstage) { st = 0; ph ^= 1; }
    }
}
__global__ void tma_read_side(const uint8_t* src, int64_t nchunks, int chunk, int nstage, const uint8_t* side,
                              int64_t side_bytes, int nsmall) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int sstride = chunk + 1024;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(nstage) * sstride);
  uint64_t* empty = full + nstage;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nstage; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (threadIdx.x >= 32) {
    if (threadIdx.x == 32) {
      int st = 0; uint32_t ph = 0;
      for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        mbar_wait(&empty[st], ph ^ 1);
        mbar_expect(&full[st], chunk + 256 * nsmall);
        uint8_t* d = sm + size_t(st) * sstride;
        bulk(d, src + c * chunk, chunk, &full[st], pol);
        for (int k = 0; k < nsmall; ++k) {
          const int64_t off = (k == 0) ? (c % 64) * 256 : ((c * 7919 + k * 104729) % (side_bytes / 256)) * 256;
          bulk(d + chunk + 256 * k, side + off, 256, &full[st], pol);
        }
        if (++st == nstage) { st = 0; ph ^= 1; }
      }
    }
    return;
  }
  int st = 0; uint32_t ph = 0;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    mbar_wait(&full[st], ph);
    __syncwarp();
    if (threadIdx.x == 0) mbar_arrive(&empty[st]);
    if (++st == nstage) { st = 0; ph ^= 1; }
  }
}

template <int U>
__global__ void ldg_read(const uint4* src, int64_t n, uint32_t* out) {
  uint32_t acc = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x * U;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x * U + threadIdx.x; i < n; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + int64_t(u) * blockDim.x;
      if (j < n) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                              : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + j));
      else v[u] = make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void copy_k(const uint4* src, uint4* dst, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

int main() {
  const int64_t bytes = int64_t(8) << 30;  // 8 GiB read region
  uint8_t *src, *dst;
  uint32_t* out;
  cudaMalloc(&src, bytes);
  cudaMalloc(&dst, bytes / 2);
  cudaMalloc(&out, 64);
  cudaMemset(src, 1, bytes);
  cudaMemset(dst, 0, bytes / 2);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto fn, double moved, const char* name) {
    fn();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      fn();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("%-40s %8.1f GB/s  (%.3f ms)%s\n", name, moved / (best * 1e-3) / 1e9, best,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  {  // anchor-major gather (realign's pattern) vs anchors of a unit contiguous
    const int chunk = 16384, nst = 9;
    size_t smem = size_t(nst) * chunk + 2 * nst * 8;
    cudaFuncSetAttribute(tma_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (int K : {20, 64, 256}) {
      const int64_t per = (bytes / K) / chunk * chunk;   // slot size, a multiple of the chunk
      const int64_t units = per / chunk - 2;
      for (int mode = 0; mode < 4; ++mode) {
        // 0: slot stride = per (as allocated), 1: per + 16 KiB pad, 2: per rounded down to a
        // power of two, 3: contiguous anchors per unit
        int64_t stride = per;
        if (mode == 1) stride = per - 2 * chunk + chunk;   // per minus one chunk: shifted alignment
        if (mode == 2) { stride = 1; while (stride * 2 <= per) stride *= 2; }
        if (mode == 3) stride = 0;
        const int64_t u = mode == 2 ? stride / chunk - 2 : units;
        char name[128];
        snprintf(name, sizeof(name), "tma_gather K=%d %s", K,
                 mode == 0 ? "slot-major" : mode == 1 ? "slot-major (shifted)" : mode == 2 ? "slot-major pow2" : "unit-major");
        timeit([&] { tma_gather<<<sms, 64, smem>>>(src, u, K, stride, chunk, nst); }, double(u) * K * chunk, name);
      }
    }
  }
  const int chunks[] = {4096, 8192, 16384, 32768};
  for (int chunk : chunks) {
    for (int nst : {4, 8, 12}) {
      size_t smem = size_t(nst) * chunk + 2 * nst * 8;
      if (smem > 220 * 1024) continue;
      cudaFuncSetAttribute(tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      for (int cps : {1, 2}) {
        if (smem * cps > 225 * 1024) continue;
        int64_t n = bytes / chunk;
        char name[128];
        snprintf(name, sizeof(name), "tma_read chunk=%d stages=%d ctas/sm=%d", chunk, nst, cps);
        timeit([&] { tma_read<<<sms * cps, 64, smem>>>(src, n, chunk, nst, dst, 0); }, double(bytes), name);
      }
    }
  }
  {
    int chunk = 16384, nst = 11;
    size_t smem = size_t(nst) * chunk + 2 * nst * 8;
    cudaFuncSetAttribute(tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int64_t n = bytes / chunk;
    for (int we : {22, 11, 4}) {
      char name[96];
      snprintf(name, sizeof(name), "tma_mix %d:1 chunk=16K stages=11", we);
      timeit([&] { tma_read<<<sms, 64, smem>>>(src, n, chunk, nst, dst, we); }, double(bytes) * (1.0 + 1.0 / we),
             name);
    }
  }
  {
    int chunk = 16384, nst = 11;
    size_t smem = size_t(nst) * chunk + 2 * nst * 8;
    cudaFuncSetAttribute(tma_mix_store, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int64_t n = bytes / chunk;
    const char* names[] = {"bulk store", "bulk store evict_first", "bulk store evict_last", "st.global.cs",
                           "st.global (wb)"};
    for (int we : {22, 17}) {
      for (int mode = 0; mode < 5; ++mode) {
        char name[96];
        snprintf(name, sizeof(name), "mix %d:1 %s", we, names[mode]);
        timeit([&] { tma_mix_store<<<sms, 64, smem>>>(src, n, chunk, nst, dst, we, mode); },
               double(bytes) * (1.0 + 1.0 / we), name);
      }
    }
  }
  {
    for (int chunk : {8192, 16384}) {
      for (int nsmall : {0, 1, 2, 4}) {
        const int nst = 11;
        size_t smem = size_t(nst) * (chunk + 1024) + 2 * nst * 8;
        cudaFuncSetAttribute(tma_read_side, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        int64_t n = bytes / chunk;
        char name[96];
        snprintf(name, sizeof(name), "tma_read chunk=%d + %d x 256B side", chunk, nsmall);
        timeit([&] { tma_read_side<<<sms, 64, smem>>>(src, n, chunk, nst, dst, bytes / 2, nsmall); },
               double(bytes) * (1.0 + 256.0 * nsmall / chunk), name);
      }
    }
  }
  int64_t nv = bytes / 16;
  timeit([&] { ldg_read<8><<<sms * 8, 256>>>((const uint4*)src, nv, out); }, double(bytes), "ldg_read U=8 8x256/sm");
  timeit([&] { ldg_read<16><<<sms * 4, 256>>>((const uint4*)src, nv, out); }, double(bytes), "ldg_read U=16 4x256/sm");
  timeit([&] { ldg_read<4><<<sms * 8, 256>>>((const uint4*)src, nv, out); }, double(bytes), "ldg_read U=4 8x256/sm");
  timeit([&] { copy_k<<<sms * 8, 256>>>((const uint4*)src, (uint4*)dst, nv / 2); }, double(bytes), "copy (read+write)");
  return 0;
}
