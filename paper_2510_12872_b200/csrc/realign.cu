// Fused anchor-offset blend + RoPE-δ + add (SURVEY §8(a) a4+a5), plus the verbatim
// copies of the concatenation step (a6):
//
//   K̂[l,h,i,:] = R_δ( K_base[l,h,i,:] + Σ_j w[i,j] ΔK_j[l,h,i,:] )     (Eq. 6 P:289 / Eq. 7 P:297,
//   V̂[l,h,i,:] =      V_base[l,h,i,:] + Σ_j w[i,j] ΔV_j[l,h,i,:]        alignment P:141)
//
// The path is pure HBM streaming: per output row it reads k offset rows + 1 base
// row and writes 1 row, ≈ k FMAs per 2(k+2) bytes.  Design:
//   * one persistent CTA per SM walks a static round-robin list of work units
//     (segment, layer, head, K|V plane, 16 KiB tile of token rows);
//   * warp 8 (one elected lane) is the TMA producer: for every unit it streams the
//     k anchor tiles (each with the matching weight slice) and finally the base
//     tile into an 11-deep shared-memory ring with cp.async.bulk (UBLKCP) +
//     mbarrier complete_tx, L2 evict-first;
//   * warps 0-7 consume: each thread owns two 32-byte "items" (8 elements of the
//     first half of a row and the matching 8 of the second half, so the
//     rotate_half pair (f, f+d/2) sits in one thread), accumulates Σ w Δ in fp32
//     registers; on the base tile it adds, rotates (K only), rounds to bf16 (RNE)
//     in place in shared memory, and one thread writes the whole tile back with a
//     single TMA bulk store (cp.async.bulk.global.shared), which measured 2-3 %
//     faster than per-thread STG (profiles/).
//   * COPY segments (n_cand = 0, δ = 0) move rows verbatim through the same ring
//     (bit-exact: no arithmetic is applied), so p_(m,0) rides in the same launch.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdlib>
#include "kvcomm_internal.h"
#include "ptx.cuh"

namespace kvc {

constexpr int kNStage = 11;
constexpr int kItems = kStageBytes / 32;                         // 512 items of 32 B per stage
constexpr int kConsumerBar = 1;                                  // named barrier id (consumers only)

constexpr size_t realign_smem_bytes() {
  return size_t(kNStage) * (kStageBytes + kStageWBytes) + 2 * kNStage * sizeof(uint64_t);
}

__device__ __forceinline__ int find_segment(const SegDev* segs, int n_seg, int64_t u) {
  int lo = 0, hi = n_seg - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (segs[mid].unit_begin <= u) lo = mid; else hi = mid - 1;
  }
  return lo;
}

struct Unit {
  int s, l, h, p, t;
};

// unit -> (segment, layer, head, plane, tile), tile fastest so that neighbouring CTAs
// stream neighbouring 16 KiB tiles of the same anchor at the same time.  Segments that
// share one base cache (one sample realigned for several consumers) form a group whose
// members are interleaved just outside the tile index: all members' units of one
// (layer, head, plane) fall in the same round of CTAs, so the shared base tile is
// fetched from HBM once and hit in L2 by the other members.
__device__ __forceinline__ Unit decode_unit(const SegDev* segs, int n_seg, int Hs, int64_t u) {
  Unit r;
  const int last = find_segment(segs, n_seg, u);   // last member of the unit's group
  int64_t rem = u - segs[last].unit_begin;
  const int G = segs[last].group_size;
  const int tiles = segs[last].tiles;              // equal for every member
  r.t = int(rem % tiles);
  rem /= tiles;
  const int member = int(rem % G);
  rem /= G;
  r.s = last - (G - 1) + member;
  r.p = int(rem & 1);
  rem >>= 1;
  r.h = int(rem % Hs);
  r.l = int(rem / Hs);
  return r;
}

// Device-side branch of Algorithm 1: a segment of an agent is realigned only
// if every placeholder pool the agent depends on was matched Shareable.
__device__ __forceinline__ bool seg_open(const TableHdr& hdr, const int32_t* ints, const SegDev& g) {
  for (int i = 0; i < g.n_gate; ++i)
    if (hdr.gate_results[ints[g.gate_off + i]].verdict != 0) return false;
  return true;
}

// Per-segment preparation: cos/sin of δ·inv_freq (fp64 angle, reading A13) and,
// for PREFIX segments, the scalar weights w̄[cand[j]] expanded into rows of the
// same shape as a placeholder W slice so the main kernel treats both kinds alike.
__global__ void realign_prep_kernel(uint8_t* tab) {
  const TableHdr* hdr = reinterpret_cast<const TableHdr*>(tab);
  SegDev* segs = reinterpret_cast<SegDev*>(tab + hdr->seg_off);
  const int32_t* cand = reinterpret_cast<const int32_t*>(tab + hdr->cand_off);
  float2* cs = reinterpret_cast<float2*>(tab + hdr->cs_off);
  float* wexp = reinterpret_cast<float*>(tab + hdr->wexp_off);
  const int s = blockIdx.x;
  const SegDev& g = segs[s];
  const int half = hdr->d / 2;
  if (g.delta != 0) {
    for (int f = threadIdx.x; f < half; f += blockDim.x) {
      double sn, cn;
      sincos(double(g.delta) * g.inv_freq[f], &sn, &cn);
      cs[g.cs_off + f] = make_float2(float(cn), float(sn));
    }
  }
  if (!g.w_by_slot && g.n_cand > 0) {
    const int ld = int(g.ld_w);
    for (int x = threadIdx.x; x < g.n_cand * ld; x += blockDim.x) {
      const int j = x / ld;
      wexp[g.wexp_off + x] = g.wbar[cand[g.cand_off + j]];
    }
  }
}

// variant (probe knob, KVCOMM_REALIGN_VARIANT): bit0 = per-thread STG.cs stores instead
// of the TMA bulk store; bit1 = skip output stores (bandwidth probe only, wrong results).
// kConsumerWarps consumer warps (8: two items per thread; 16: one item per thread, twice the
// issue slots for the e4m3 decode of fp8 pools) + one producer warp.
template <int kConsumerWarps>
__global__ void __launch_bounds__((kConsumerWarps + 1) * 32, 1)
    realign_kernel(const uint8_t* __restrict__ tab, int variant) {
  constexpr int kItemsPerThread = kItems / (kConsumerWarps * 32);
  static_assert(kItemsPerThread * kConsumerWarps * 32 == kItems, "item split");
  const TableHdr hdr = *reinterpret_cast<const TableHdr*>(tab);
  const SegDev* segs = reinterpret_cast<const SegDev*>(tab + hdr.seg_off);
  const int32_t* cand = reinterpret_cast<const int32_t*>(tab + hdr.cand_off);
  const float2* cs = reinterpret_cast<const float2*>(tab + hdr.cs_off);

  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sdata = smem;
  float* sw = reinterpret_cast<float*>(smem + size_t(kNStage) * kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(kNStage) * (kStageBytes + kStageWBytes));
  uint64_t* empty = full + kNStage;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kNStage; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int d = hdr.d;
  const int Hs = hdr.Hs;
  const int rpt = hdr.rows_per_tile;
  const int64_t total = hdr.total_units;
  const int row_bytes = 2 * d;
  const bool tma_store = !(variant & 3);

  if (warp == kConsumerWarps) {
    // ---------------- TMA producer (one lane) ----------------
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();  // offsets: read once per request
      const uint64_t pol_shared = (variant & 4) ? policy_evict_first()
                                  : (variant & 8) ? policy_evict_normal() : policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = blockIdx.x; u < total; u += gridDim.x) {
        const Unit un = decode_unit(segs, hdr.n_seg, Hs, u);
        const SegDev& g = segs[un.s];
        if (!seg_open(hdr, cand, g)) continue;
        const int i0 = un.t * rpt;
        const int nrows = min(rpt, g.L_seg - i0);
        const uint32_t bytes = uint32_t(nrows) * row_bytes;
        const uint32_t wbytes = (uint32_t(nrows) * 4u + 15u) & ~15u;
        const int64_t lh = int64_t(un.l) * Hs + un.h;
        if (g.fp8) {
          // e4m3 anchor tiles are half a stage: two anchors per stage, each with its
          // weight slice and its per-row scale slice in the stage's side area
          const uint32_t cbytes = uint32_t(nrows) * d;
          // per-unit parts of the addresses (rows of the tile; codes are 1 byte per element)
          const int64_t unit_rows = int64_t(un.p) * g.sc_plane_stride + lh * g.off_ld + i0;
          const uint8_t* code0 = reinterpret_cast<const uint8_t*>(g.off) + unit_rows * d;
          const float* scale0 = g.scales + unit_rows;
          const float* w0 = g.w + i0;
          for (int c = 0; c < g.n_cand; c += 2) {
            mbar_wait(&empty[stage], phase ^ 1u);
            const int na = min(2, g.n_cand - c);
            uint8_t* dst = sdata + size_t(stage) * kStageBytes;
            float* swst = sw + size_t(stage) * (kStageWBytes / 4);
            mbar_arrive_expect_tx(&full[stage], uint32_t(na) * (cbytes + 2 * wbytes));
            for (int a = 0; a < na; ++a) {
              const int slot = cand[g.cand_off + c + a];
              bulk_g2s(dst + a * (kStageBytes / 2), code0 + int64_t(slot) * g.slot_stride, cbytes, &full[stage],
                       pol_stream);
              bulk_g2s(swst + a * rpt, w0 + int64_t(g.w_by_slot ? slot : c + a) * g.ld_w, wbytes, &full[stage],
                       pol_stream);
              bulk_g2s(swst + (2 + a) * rpt, scale0 + int64_t(slot) * g.sc_slot_stride, wbytes, &full[stage],
                       pol_stream);
            }
            if (++stage == kNStage) { stage = 0; phase ^= 1u; }
          }
          mbar_wait(&empty[stage], phase ^ 1u);
          const bf16* src = g.base[un.p] + (lh * g.base_ld + i0) * d;
          mbar_arrive_expect_tx(&full[stage], bytes);
          bulk_g2s(sdata + size_t(stage) * kStageBytes, src, bytes, &full[stage],
                   g.group_size > 1 ? pol_shared : pol_stream);
          if (++stage == kNStage) { stage = 0; phase ^= 1u; }
          continue;
        }
        for (int c = 0; c <= g.n_cand; ++c) {
          mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t* dst = sdata + size_t(stage) * kStageBytes;
          if (c < g.n_cand) {
            const int slot = cand[g.cand_off + c];
            const bf16* src = g.off + int64_t(slot) * g.slot_stride + int64_t(un.p) * g.plane_stride +
                              (lh * g.off_ld + i0) * d;
            const float* wsrc = g.w + int64_t(g.w_by_slot ? slot : c) * g.ld_w + i0;
            mbar_arrive_expect_tx(&full[stage], bytes + wbytes);
            bulk_g2s(dst, src, bytes, &full[stage], pol_stream);
            bulk_g2s(sw + size_t(stage) * (kStageWBytes / 4), wsrc, wbytes, &full[stage], pol_stream);
          } else {
            const bf16* src = g.base[un.p] + (lh * g.base_ld + i0) * d;
            mbar_arrive_expect_tx(&full[stage], bytes);
            bulk_g2s(dst, src, bytes, &full[stage], g.group_size > 1 ? pol_shared : pol_stream);
          }
          if (++stage == kNStage) { stage = 0; phase ^= 1u; }
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int vpr = d >> 4;  // items per row
  const int ct = threadIdx.x;
  int irow[kItemsPerThread], ivec[kItemsPerThread];
#pragma unroll
  for (int q = 0; q < kItemsPerThread; ++q) {
    const int it = ct + q * kConsumerWarps * 32;
    irow[q] = it / vpr;
    ivec[q] = it - irow[q] * vpr;
  }
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t u = blockIdx.x; u < total; u += gridDim.x) {
    const Unit un = decode_unit(segs, hdr.n_seg, Hs, u);
    const SegDev& g = segs[un.s];
    if (!seg_open(hdr, cand, g)) continue;
    const int i0 = un.t * rpt;
    const int nrows = min(rpt, g.L_seg - i0);
    float acc[kItemsPerThread][16];
#pragma unroll
    for (int q = 0; q < kItemsPerThread; ++q)
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[q][e] = 0.f;

    const int n_cand = g.n_cand;
    if (g.fp8) {
      for (int c = 0; c < n_cand; c += 2) {
        mbar_wait(&full[stage], phase);
        const uint8_t* buf = sdata + size_t(stage) * kStageBytes;
        const float* swst = sw + size_t(stage) * (kStageWBytes / 4);
        const int na = min(2, n_cand - c);
        for (int a = 0; a < na; ++a) {
          const uint8_t* ab = buf + a * (kStageBytes / 2);
#pragma unroll
          for (int q = 0; q < kItemsPerThread; ++q) {
            const float w = swst[a * rpt + irow[q]] * swst[(2 + a) * rpt + irow[q]];  // weight x row scale
            const uint2 lo = lds64(ab + irow[q] * d + ivec[q] * 8);
            const uint2 hi = lds64(ab + irow[q] * d + d / 2 + ivec[q] * 8);
            const uint32_t lw[2] = {lo.x, lo.y}, hw[2] = {hi.x, hi.y};
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              float f[4];
              e4m3x4_to_float(lw[t], f);
#pragma unroll
              for (int e = 0; e < 4; ++e) acc[q][4 * t + e] = fmaf(w, f[e], acc[q][4 * t + e]);
              e4m3x4_to_float(hw[t], f);
#pragma unroll
              for (int e = 0; e < 4; ++e) acc[q][8 + 4 * t + e] = fmaf(w, f[e], acc[q][8 + 4 * t + e]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == kNStage) { stage = 0; phase ^= 1u; }
      }
    }
    for (int c = 0; c < (g.fp8 ? 0 : n_cand); ++c) {
      mbar_wait(&full[stage], phase);
      const uint8_t* buf = sdata + size_t(stage) * kStageBytes;
      const float* wv = sw + size_t(stage) * (kStageWBytes / 4);
#pragma unroll
      for (int q = 0; q < kItemsPerThread; ++q) {
        const float w = wv[irow[q]];
        const uint4 a = lds128(buf + irow[q] * row_bytes + ivec[q] * 16);
        const uint4 b = lds128(buf + irow[q] * row_bytes + d + ivec[q] * 16);
        const uint32_t av[4] = {a.x, a.y, a.z, a.w};
        const uint32_t bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          acc[q][2 * e] = fmaf(w, bf_lo(av[e]), acc[q][2 * e]);
          acc[q][2 * e + 1] = fmaf(w, bf_hi(av[e]), acc[q][2 * e + 1]);
          acc[q][8 + 2 * e] = fmaf(w, bf_lo(bv[e]), acc[q][8 + 2 * e]);
          acc[q][8 + 2 * e + 1] = fmaf(w, bf_hi(bv[e]), acc[q][8 + 2 * e + 1]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kNStage) { stage = 0; phase ^= 1u; }
    }

    // base tile: add, rotate (K), round, store
    mbar_wait(&full[stage], phase);
    uint8_t* buf = sdata + size_t(stage) * kStageBytes;
    const int64_t lh = int64_t(un.l) * Hs + un.h;
    const bool rotate = un.p == 0 && g.delta != 0;
    if (n_cand > 0 || rotate) {  // COPY segments leave the staged rows untouched (bit-exact)
#pragma unroll
      for (int q = 0; q < kItemsPerThread; ++q) {
        if (irow[q] >= nrows) continue;
        uint8_t* pa = buf + irow[q] * row_bytes + ivec[q] * 16;
        uint8_t* pb = pa + d;
        const uint4 a = lds128(pa);
        const uint4 b = lds128(pb);
        const uint32_t av[4] = {a.x, a.y, a.z, a.w};
        const uint32_t bv[4] = {b.x, b.y, b.z, b.w};
        float y0[8], y1[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          y0[2 * e] = bf_lo(av[e]) + acc[q][2 * e];
          y0[2 * e + 1] = bf_hi(av[e]) + acc[q][2 * e + 1];
          y1[2 * e] = bf_lo(bv[e]) + acc[q][8 + 2 * e];
          y1[2 * e + 1] = bf_hi(bv[e]) + acc[q][8 + 2 * e + 1];
        }
        if (rotate) {
          const float2* csr = cs + g.cs_off + ivec[q] * 8;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float2 r = csr[e];
            const float x0 = y0[e], x1 = y1[e];
            y0[e] = x0 * r.x - x1 * r.y;
            y1[e] = x1 * r.x + x0 * r.y;
          }
        }
        const uint4 r0 = make_uint4(pack_bf16_rn(y0[0], y0[1]), pack_bf16_rn(y0[2], y0[3]),
                                    pack_bf16_rn(y0[4], y0[5]), pack_bf16_rn(y0[6], y0[7]));
        const uint4 r1 = make_uint4(pack_bf16_rn(y1[0], y1[1]), pack_bf16_rn(y1[2], y1[3]),
                                    pack_bf16_rn(y1[4], y1[5]), pack_bf16_rn(y1[6], y1[7]));
        if (tma_store) {
          sts128(pa, r0);  // in place; the whole tile leaves with one bulk store below
          sts128(pb, r1);
        } else if (!(variant & 2)) {
          bf16* o = g.dst[un.p] + (lh * g.dst_ld + g.target_start + i0 + irow[q]) * d + ivec[q] * 8;
          stg128_cs(o, r0);
          stg128_cs(o + d / 2, r1);
        }
        if (g.dbg[un.p] != nullptr) {
          float* od = g.dbg[un.p] + (lh * g.L_seg + i0 + irow[q]) * d + ivec[q] * 8;
          float4* o0 = reinterpret_cast<float4*>(od);
          float4* o1 = reinterpret_cast<float4*>(od + d / 2);
          o0[0] = make_float4(acc[q][0], acc[q][1], acc[q][2], acc[q][3]);
          o0[1] = make_float4(acc[q][4], acc[q][5], acc[q][6], acc[q][7]);
          o1[0] = make_float4(acc[q][8], acc[q][9], acc[q][10], acc[q][11]);
          o1[1] = make_float4(acc[q][12], acc[q][13], acc[q][14], acc[q][15]);
        }
      }
    } else if (!tma_store && !(variant & 2)) {
#pragma unroll
      for (int q = 0; q < kItemsPerThread; ++q) {
        if (irow[q] >= nrows) continue;
        const uint8_t* pa = buf + irow[q] * row_bytes + ivec[q] * 16;
        bf16* o = g.dst[un.p] + (lh * g.dst_ld + g.target_start + i0 + irow[q]) * d + ivec[q] * 8;
        stg128_cs(o, lds128(pa));
        stg128_cs(o + d / 2, lds128(pa + d));
      }
    }
    if (tma_store) {
      // all consumer writes of the tile -> visible to the async proxy, then one bulk store;
      // the stage is released only once the store has finished reading shared memory
      fence_proxy_async_smem();
      named_bar_sync(kConsumerBar, kConsumerWarps * 32);
      if (threadIdx.x == 0) {
        bf16* o = g.dst[un.p] + (lh * g.dst_ld + g.target_start + i0) * d;
        bulk_s2g(o, buf, uint32_t(nrows) * row_bytes);
        bulk_wait_read_all();
        mbar_arrive_cnt(&empty[stage], kConsumerWarps);
      }
    } else {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
    }
    if (++stage == kNStage) { stage = 0; phase ^= 1u; }
  }
  if (tma_store && threadIdx.x == 0) bulk_wait_all();  // global writes complete before exit
}

int realign_grid_size(int device) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return sms > 0 ? sms : 148;
}

cudaError_t launch_realign(const void* table_dev, const TableHdr& hdr, int grid, cudaStream_t s) {
  static bool attr_set[64] = {false};
  static int variant = -1, cw = 16;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(realign_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(realign_smem_bytes()));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(realign_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(realign_smem_bytes()));
    if (e != cudaSuccess) return e;
    attr_set[dev & 63] = true;
  }
  if (variant < 0) {
    const char* v = getenv("KVCOMM_REALIGN_VARIANT");
    variant = v ? atoi(v) : 0;
    const char* c = getenv("KVCOMM_REALIGN_CONSUMER_WARPS");
    if (c && atoi(c) == 8) cw = 8;
  }
  realign_prep_kernel<<<hdr.n_seg, 128, 0, s>>>(reinterpret_cast<uint8_t*>(const_cast<void*>(table_dev)));
  if (hdr.total_units <= 0) return cudaGetLastError();
  const int64_t g = hdr.total_units < grid ? hdr.total_units : grid;
  const uint8_t* t = reinterpret_cast<const uint8_t*>(table_dev);
  if (cw == 8)
    realign_kernel<8><<<int(g), 9 * 32, realign_smem_bytes(), s>>>(t, variant);
  else
    realign_kernel<16><<<int(g), 17 * 32, realign_smem_bytes(), s>>>(t, variant);
  return cudaGetLastError();
}

}  // namespace kvc
