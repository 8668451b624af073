// Fused anchor-offset blend + RoPE-δ + add (SURVEY §8(a) a4+a5), plus the verbatim
// copies of the concatenation step (a6):
//
//   K̂[l,h,i,:] = R_δ( K_base[l,h,i,:] + Σ_j w[i,j] ΔK_j[l,h,i,:] )     (Eq. 6 P:289 / Eq. 7 P:297,
//   V̂[l,h,i,:] =      V_base[l,h,i,:] + Σ_j w[i,j] ΔV_j[l,h,i,:]        alignment P:141)
//
// The path is pure HBM streaming: per output row it reads k offset rows + 1 base
// row and writes 1 row, ≈ k FMAs per 2(k+2) bytes.  Design:
//   * one persistent CTA per SM walks a static round-robin list of work units
//     (segment, layer, head, K|V plane, tile of token rows: 16 KiB of bf16 rows, or
//     two such tiles for fp8 pools so that each anchor tile is again ~16 KiB);
//   * the last warp (one elected lane) is the TMA producer: it streams the unit's
//     weights [n_cand][rows] in chunks of up to 16 KiB (one copy each, double
//     buffered), then the anchor tiles (one contiguous copy per anchor: bf16 rows, or
//     an fp8 block of e4m3 codes followed by their row scales) and finally the base
//     tile(s) into a shared-memory ring of 7 (bf16) / 9 (fp8) stages (ring_stages: fewer
//     bytes in flight, less DRAM contention) with cp.async.bulk (UBLKCP) + mbarrier
//     complete_tx, L2 evict-first for anchor tiles, evict-last for the weight blocks
//     (re-read by every (layer, head, plane) unit of a tile) and for shared bases; the
//     pool's slab pads 64 rows between slots so that consecutive anchors' tiles do not
//     sit a power-of-two multiple apart (config 4: +3.5 %);
//   * 8 consumer warps (16 for tables that read fp8 pools): each thread owns two
//     32-byte "items" per 64-row tile (8 elements of the first half of a row and the
//     matching 8 of the second half, so the rotate_half pair (f, f+d/2) sits in one
//     thread).  Per anchor tile it loads its operands into registers, arrives on the
//     stage's empty barrier (the stage is held only for the shared-memory loads),
//     then accumulates Σ w Δ in fp32 registers with packed FFMA2 (fp8 codes decoded
//     exactly by F2FP + HADD2.F32).  On a base tile it adds, rotates (K only), rounds
//     to bf16 (RNE) in place in shared memory, and one thread writes the whole tile
//     back with a single TMA bulk store (cp.async.bulk.global.shared, 2-3 % faster than
//     per-thread STG); rows bound for a peer GPU (the fused gather) use per-thread
//     stores over NVLink instead.
//   * COPY segments (n_cand = 0, δ = 0) move rows verbatim through the same ring
//     (bit-exact: no arithmetic is applied), so p_(m,0) rides in the same launch.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include "kvcomm_internal.h"
#include "ptx.cuh"

namespace kvc {

// Ring depth per instantiation (stages of kStageStride): fewer bytes in flight means less
// DRAM contention, as long as the ring still covers the latency.  Measured at config 2
// (profiles/r02g_ring_depth.jsonl, r02h_fp8_warps.txt): the bf16 stream is fastest with 7
// stages (9: 2 % slower, 11: 5 %), the fp8 decode (slower consumers) with 10 (7: 1.5 %, 8:
// 0.8 % slower; 11 would leave no room for a match CTA beside it when pipelined).
#ifndef KVC_NSTAGE_BF16
#define KVC_NSTAGE_BF16 7
#endif
#ifndef KVC_NSTAGE_FP8
#define KVC_NSTAGE_FP8 10
#endif
template <bool kFp8>
constexpr int ring_stages() { return kFp8 ? KVC_NSTAGE_FP8 : KVC_NSTAGE_BF16; }
constexpr int kItems = kStageBytes / 32;  // 512 items of 32 B per 16 KiB bf16 tile
constexpr int kConsumerBar = 1;           // named barrier id (consumers only)

constexpr size_t realign_smem_bytes(int stages) {
  return size_t(stages) * kStageStride + 2 * size_t(kUnitWBytes) + (2 * size_t(stages) + 4) * sizeof(uint64_t);
}
static_assert(realign_smem_bytes(ring_stages<false>()) <= 227 * 1024, "realign shared memory");
static_assert(realign_smem_bytes(ring_stages<true>()) <= 227 * 1024, "realign shared memory");

struct Unit {
  int s, l, h, p, t;
};

// Device-side branch of Algorithm 1: a segment of an agent is realigned only
// if every placeholder pool the agent depends on was matched Shareable.
__device__ __forceinline__ bool seg_open(const TableHdr& hdr, const int32_t* ints, const SegDev& g) {
  for (int i = 0; i < g.n_gate; ++i)
    if (hdr.gate_results[ints[g.gate_off + i]].verdict != 0) return false;
  return true;
}

// The prep kernel's unit list (UnitDev at unit_off): tile fastest so that neighbouring
// CTAs stream neighbouring tiles of the same anchor at the same time.  Segments that
// share one base cache (one sample realigned for several consumers) form a group whose
// members are interleaved just outside the tile index: all members' units of one
// (layer, head, plane) fall in the same round of CTAs, so the shared base tile is
// fetched from HBM once and hit in L2 by the other members.
//   u = unit_begin + (((l * Hs + h) * 2 + p) * group_size + member) * tiles + t
__device__ __forceinline__ Unit load_unit(const UnitDev* units, int64_t u) {
  const int4 v = __ldg(reinterpret_cast<const int4*>(units + u));
  Unit r;
  r.s = v.x;
  r.l = v.y;
  r.h = v.z;
  r.p = v.w & 1;
  r.t = v.w >> 1;
  return r;
}

// Per-segment preparation (grid n_seg x kPrepY): the segment's entries of the unit list,
// cos/sin of δ·inv_freq (fp64 angle, reading A13) and the weight blocks wt[tile][j][row] = weight of candidate j at the
// tile's token row (0 past L_seg), from W[slot] (PLACEHOLDER) or w̄[slot] (PREFIX),
// so the main kernel fetches a unit's weights as contiguous chunks.
#ifndef KVC_PREP_Y
#define KVC_PREP_Y 8
#endif
constexpr int kPrepY = KVC_PREP_Y;  // block rows per segment
__global__ void realign_prep_kernel(uint8_t* tab) {
  const TableHdr* hdr = reinterpret_cast<const TableHdr*>(tab);
  SegDev* segs = reinterpret_cast<SegDev*>(tab + hdr->seg_off);
  const int32_t* cand = reinterpret_cast<const int32_t*>(tab + hdr->cand_off);
  float2* cs = reinterpret_cast<float2*>(tab + hdr->cs_off);
  float* wt = reinterpret_cast<float*>(tab + hdr->wt_off);
  const SegDev& g = segs[blockIdx.x];
  const int half = hdr->d / 2;
  if (g.delta != 0 && blockIdx.y == 0) {
    for (int f = threadIdx.x; f < half; f += blockDim.x) {
      double sn, cn;
      sincos(double(g.delta) * g.inv_freq[f], &sn, &cn);
      cs[g.cs_off + f] = make_float2(float(cn), float(sn));
    }
  }
  {  // this segment's entries of the unit list (s = -1: gate closed, every unit skipped)
    UnitDev* units = reinterpret_cast<UnitDev*>(tab + hdr->unit_off);
    const int32_t* ints = cand;
    const bool open = seg_open(*hdr, ints, g);
    const uint32_t tiles = uint32_t(g.tiles), G = uint32_t(g.group_size);
    const uint32_t nu = uint32_t(hdr->Ls) * uint32_t(hdr->Hs) * 2u * tiles;  // < 2^31: host-validated sizes
    for (uint32_t x = blockIdx.y * blockDim.x + threadIdx.x; x < nu; x += gridDim.y * blockDim.x) {
      const uint32_t lhp = x / tiles;
      const uint32_t t = x - lhp * tiles;
      const uint32_t lh = lhp >> 1;
      const uint32_t l = lh / uint32_t(hdr->Hs);
      UnitDev v;
      v.s = open ? int32_t(blockIdx.x) : -1;
      v.l = int32_t(l);
      v.h = int32_t(lh - l * uint32_t(hdr->Hs));
      v.tp = int32_t((t << 1) | (lhp & 1u));
      units[g.unit_begin + (int64_t(lhp) * G + uint32_t(g.group_member)) * tiles + t] = v;
    }
  }
  if (g.n_cand == 0) return;
  const int rpu = unit_rows(hdr->d, g.fp8);
  const int rw = weight_row_stride(rpu);
  // 32-bit index math: with rpu >= 4 rows per unit (rpu <= 2 * rows_per_tile), tiles * rw <=
  // (L_seg / rpu + 1) * (rpu + 3) < 2 * (L_seg + 2 * rows_per_tile), and validate_segment
  // (kvcomm_api.cu) rejects any segment with (L_seg + 2 * rows_per_tile) * n_cand * 2 >= 2^31
  // before a launch, so tiles * n_cand * rw < 2^31
  const uint32_t n = uint32_t(g.tiles) * uint32_t(g.n_cand) * uint32_t(rw);
  const uint32_t urw = uint32_t(rw), unc = uint32_t(g.n_cand);
  for (uint32_t x = blockIdx.y * blockDim.x + threadIdx.x; x < n; x += gridDim.y * blockDim.x) {
    const uint32_t tj = x / urw;
    const int r = int(x - tj * urw);
    const uint32_t t = tj / unc;
    const int j = int(tj - t * unc);
    const int row = int(t) * rpu + r;
    const int slot = cand[g.cand_off + j];
    float w = 0.f;
    if (r < rpu && row < g.L_seg) w = g.w_by_slot ? g.w[int64_t(slot) * g.ld_w + row] : g.wbar[slot];
    wt[g.wt_off + x] = w;
  }
}

// One anchor tile of an fp8 pool: two 64-row tiles of a block (codes, then row scales);
// every thread's item is one 16-byte chunk of a row (8 codes of the first half of the
// row and the matching 8 of the second half, stored interleaved), so a warp's loads are
// contiguous and conflict-free.  fp8_load pulls a thread's codes and weight x row scale
// into registers (the stage can be released right after), fp8_accum decodes with F2FP
// (e4m3x2 -> f16x2, exact) + HADD2.F32 (f16 -> f32, exact) and accumulates with packed
// FFMA2.  (An all-integer decode with 2^120 folded into the weight measured 15 % slower:
// it loads the ALU pipe.)
template <int NI>
__device__ __forceinline__ void fp8_load(float (&w)[2][NI], uint4 (&code)[2][NI], const uint8_t* blk,
                                         const uint8_t* wv, const uint8_t* scl, const int (&coff)[2][NI],
                                         const int (&roff)[2][NI]) {
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int q = 0; q < NI; ++q) {
      // weight x row scale
      w[s][q] = *reinterpret_cast<const float*>(wv + roff[s][q]) * *reinterpret_cast<const float*>(scl + roff[s][q]);
      code[s][q] = lds128(blk + coff[s][q]);
    }
}

template <int NI>
__device__ __forceinline__ void fp8_accum(float (&acc)[2][NI][16], const float (&w)[2][NI],
                                          const uint4 (&code)[2][NI]) {
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int q = 0; q < NI; ++q) {
      const uint32_t cw[4] = {code[s][q].x, code[s][q].y, code[s][q].z, code[s][q].w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {  // word t: elements 4t..4t+3 of the item's 16
        float f[4];
        e4m3x4_to_float(cw[t], f);
        ffma2(acc[s][q][4 * t], acc[s][q][4 * t + 1], w[s][q], w[s][q], f[0], f[1]);
        ffma2(acc[s][q][4 * t + 2], acc[s][q][4 * t + 3], w[s][q], w[s][q], f[2], f[3]);
      }
    }
}

// variant (measurement knob, KVCOMM_REALIGN_VARIANT): bit0 = per-thread STG.cs stores
// instead of the TMA bulk store; bits 2/3 = L2 policy of shared bases; bit8 = generic-d
// kernel — all of them give the same results.  Bandwidth probes that give WRONG results
// (bit1 = skip the output stores, bit5 = skip the anchor math) exist only in probe builds
// (make EXTRA=-DKVC_PROBE_VARIANTS=1 OUT=<dir>/libkvcomm.so OBJDIR=<dir>/obj); the product
// library compiles them out, so no environment variable can make it write wrong caches.
// Stage release: every consumer thread arrives on the empty barrier itself after its own
// shared-memory reads (same speed as a warp-elected arrive after __syncwarp, and the
// ordering is then visible to compute-sanitizer racecheck, which does not model the
// __syncwarp hand-off).
// kConsumerWarps consumer warps (8: two items per thread; 16: one item per thread) + one
// producer warp.
// kD: head_dim fixed at compile time (128: the Llama shapes; all tile geometry and
// thread offsets fold into immediates), 0: read from the table (any supported d).
// KVC_WARP_ARRIVE=1: one elected arrive per consumer warp after __syncwarp instead of one
// per thread — measured no faster (bf16 config 2 and 4) and 1.5 % slower with fp8 pools
// (r01g), and the per-thread form keeps the ordering visible to racecheck.
#ifndef KVC_WARP_ARRIVE
#define KVC_WARP_ARRIVE 0
#endif
constexpr int kArrivals = KVC_WARP_ARRIVE ? 1 : 32;  // empty-barrier arrivals per consumer warp
#ifndef KVC_PROBE_VARIANTS
#define KVC_PROBE_VARIANTS 0
#endif
constexpr bool kProbeVariants = KVC_PROBE_VARIANTS != 0;
#ifndef KVC_FP8_UNROLL
#define KVC_FP8_UNROLL 2
#endif
constexpr int kFp8Unroll = KVC_FP8_UNROLL;  // fp8 anchor tiles per iteration (4 measured no faster than 2, and spills)
#ifndef KVC_WAIT_HINT
#define KVC_WAIT_HINT 0
#endif
// consumers' waits on full stages: suspend-time hint in ns (0 = plain try_wait polling)
__device__ __forceinline__ void consumer_wait(uint64_t* b, uint32_t parity) {
  mbar_wait_hint<KVC_WAIT_HINT>(b, parity);
}
__device__ __forceinline__ void stage_release(uint64_t* b) {
#if KVC_WARP_ARRIVE
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(b);
#else
  mbar_arrive(b);
#endif
}

template <int kConsumerWarps, int kD, bool kFp8>
__device__ __forceinline__ void realign_body(const uint8_t* __restrict__ tab, int variant) {
  constexpr int kItemsPerThread = kItems / (kConsumerWarps * 32);
  // tables that read an fp8 pool always launch the 16-warp instantiation (launch_realign), so
  // the 8-warp one carries no e4m3 decode (keeps its registers for the bf16 stream)
  constexpr bool kFp8Path = kFp8;
  constexpr int kNStage = ring_stages<kFp8>();
  static_assert(kItemsPerThread * kConsumerWarps * 32 == kItems, "item split");
  const TableHdr hdr = *reinterpret_cast<const TableHdr*>(tab);
  const SegDev* segs = reinterpret_cast<const SegDev*>(tab + hdr.seg_off);
  const int32_t* cand = reinterpret_cast<const int32_t*>(tab + hdr.cand_off);
  const float2* cs = reinterpret_cast<const float2*>(tab + hdr.cs_off);
  const UnitDev* units = reinterpret_cast<const UnitDev*>(tab + hdr.unit_off);

  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sdata = smem;                                                       // [kNStage][kStageStride]
  float* suw = reinterpret_cast<float*>(smem + size_t(kNStage) * kStageStride);  // [2][kUnitWBytes/4]
  uint64_t* full = reinterpret_cast<uint64_t*>(suw + 2 * (kUnitWBytes / 4));
  uint64_t* empty = full + kNStage;
  uint64_t* uw_full = empty + kNStage;
  uint64_t* uw_empty = uw_full + 2;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kNStage; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kConsumerWarps * kArrivals);  // every consumer thread (or warp) arrives
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&uw_full[i], 1);
      mbar_init(&uw_empty[i], kConsumerWarps * kArrivals);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int d = kD ? kD : hdr.d;
  const int Hs = hdr.Hs;
  const int rpt = kD ? rows_per_tile(kD) : hdr.rows_per_tile;
  const int fblk = fp8_block_bytes(d);
  const int64_t total = hdr.total_units;
  const int row_bytes = 2 * d;
  const bool skip_store = kProbeVariants && (variant & 2);  // probe builds only
  const bool skip_math = kProbeVariants && (variant & 32);   // probe builds only
  const bool tma_store = !(variant & 1) && !skip_store;

  if (warp == kConsumerWarps) {
    // ---------------- TMA producer (one lane) ----------------
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();  // offsets: read once per request
      // weight blocks: re-read by every (layer, head, plane) unit of the same tile, so they
      // stay in L2 (evict_first measured 0.4 % slower at config 2, 0.9 % at config 4)
      const uint64_t pol_weights = policy_evict_last();
      const uint64_t pol_shared = (variant & 4) ? policy_evict_first()
                                  : (variant & 8) ? policy_evict_normal() : policy_evict_last();
      int stage = 0, ub = 0;
      uint32_t phase = 0, uphase = 0;
      for (int64_t u = blockIdx.x; u < total; u += gridDim.x) {
        const Unit un = load_unit(units, u);
        if (un.s < 0) continue;  // gate closed
        const SegDev& g = segs[un.s];
        // segment fields -> registers (the barrier asm's memory clobbers would reload them)
        const bool fp8 = g.fp8;
        const int n_cand = g.n_cand;
        const int* cands = cand + g.cand_off;
        const int rpu = unit_rows(d, fp8);
        const int i0 = un.t * rpu;
        const int nrows = min(rpu, g.L_seg - i0);
        const int64_t lh = int64_t(un.l) * Hs + un.h;
        const int rw = weight_row_stride(rpu);
        const int chunk = kUnitWBytes / (rw * 4);  // anchors per weight chunk
        const float* wt = g.wt + int64_t(un.t) * n_cand * rw;
        // anchor tile of slot s at anchor0 + s * slot_bytes
        const uint8_t* anchor0 = fp8 ? reinterpret_cast<const uint8_t*>(g.off) + int64_t(un.p) * g.plane_stride +
                                           lh * g.off_ld + int64_t(un.t) * fblk
                                     : reinterpret_cast<const uint8_t*>(g.off + int64_t(un.p) * g.plane_stride +
                                                                        (lh * g.off_ld + i0) * d);
        const int64_t slot_bytes = fp8 ? g.slot_stride : g.slot_stride * int64_t(sizeof(bf16));
        const uint32_t full_bytes = fp8 ? uint32_t(fblk) : uint32_t(nrows) * row_bytes;
        const bool split = fp8 && nrows < rpu;  // fp8 tail tile: only its rows' codes and scales
        const uint32_t cb = (uint32_t(nrows * d) + 15u) & ~15u, sb = (uint32_t(nrows) * 4u + 15u) & ~15u;
        const bf16* base = g.base[un.p] + (lh * g.base_ld + i0) * d;
        const uint64_t pol_base = g.group_size > 1 ? pol_shared : pol_stream;
        int slot = n_cand > 0 ? cands[0] : 0;
        for (int c0 = 0; c0 < n_cand; c0 += chunk) {
          const int c1 = min(n_cand, c0 + chunk);
          mbar_wait(&uw_empty[ub], uphase ^ 1u);
          const uint32_t wbytes = uint32_t((c1 - c0) * rw) * 4u;
          mbar_arrive_expect_tx(&uw_full[ub], wbytes);
          bulk_g2s(suw + ub * (kUnitWBytes / 4), wt + int64_t(c0) * rw, wbytes, &uw_full[ub], pol_weights);
          if (++ub == 2) { ub = 0; uphase ^= 1u; }
          for (int c = c0; c < c1; ++c) {
            const int next = c + 1 < n_cand ? cands[c + 1] : 0;  // in flight during the wait
            mbar_wait(&empty[stage], phase ^ 1u);
            uint8_t* dst = sdata + size_t(stage) * kStageStride;
            const uint8_t* src = anchor0 + int64_t(slot) * slot_bytes;
            if (!split) {
              mbar_arrive_expect_tx(&full[stage], full_bytes);
              bulk_g2s(dst, src, full_bytes, &full[stage], pol_stream);
            } else {
              mbar_arrive_expect_tx(&full[stage], cb + sb);
              bulk_g2s(dst, src, cb, &full[stage], pol_stream);
              bulk_g2s(dst + rpu * d, src + rpu * d, sb, &full[stage], pol_stream);
            }
            slot = next;
            if (++stage == kNStage) { stage = 0; phase ^= 1u; }
          }
        }
        for (int r0 = 0; r0 < nrows; r0 += rpt) {  // base tile(s)
          mbar_wait(&empty[stage], phase ^ 1u);
          const uint32_t bytes = uint32_t(min(rpt, nrows - r0)) * row_bytes;
          mbar_arrive_expect_tx(&full[stage], bytes);
          bulk_g2s(sdata + size_t(stage) * kStageStride, base + int64_t(r0) * d, bytes, &full[stage], pol_base);
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
  // fp8 blocks: byte offsets of the thread's code chunks and of its rows' weights / scales
  int coff[2][kItemsPerThread], roff[2][kItemsPerThread];
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int q = 0; q < kItemsPerThread; ++q) {
      coff[s][q] = (s * rpt + irow[q]) * d + ivec[q] * 16;
      roff[s][q] = (s * rpt + irow[q]) * 4;
    }
  const int scale_off = 2 * rpt * d;
  int stage = 0, ub = 0;
  uint32_t phase = 0, uphase = 0;
  for (int64_t u = blockIdx.x; u < total; u += gridDim.x) {
    const Unit un = load_unit(units, u);
    if (un.s < 0) continue;  // gate closed
    const SegDev& g = segs[un.s];
    // segment fields -> registers (the barrier asm's memory clobbers would reload them)
    const bool fp8 = g.fp8;
    const int n_cand = g.n_cand;
    const int rpu = unit_rows(d, fp8);
    const int i0 = un.t * rpu;
    const int nrows = min(rpu, g.L_seg - i0);
    const int rw = weight_row_stride(rpu);
    const int chunk = kUnitWBytes / (rw * 4);
    const int64_t lh = int64_t(un.l) * Hs + un.h;
    const bool rotate = un.p == 0 && g.delta != 0;
    const bool rope_il = g.rope_il;
    const float2* csg = cs + g.cs_off;
    bf16* const dst = g.dst[un.p] + ((int64_t(un.l) * g.dst_heads + un.h) * g.dst_ld + g.target_start + i0) * d;
    const bool tstore = tma_store && g.dst_stg != 1;  // dst_stg 1: peer rows with per-thread stores
    float* const dbg = g.dbg[un.p] != nullptr ? g.dbg[un.p] + (lh * g.L_seg + i0) * d : nullptr;
    float acc[2][kItemsPerThread][16];  // [64-row tile of the unit][item][element]
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int q = 0; q < kItemsPerThread; ++q)
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[s][q][e] = 0.f;

    for (int c0 = 0; c0 < n_cand; c0 += chunk) {
      const int c1 = min(n_cand, c0 + chunk);
      consumer_wait(&uw_full[ub], uphase);
      const float* wv = suw + ub * (kUnitWBytes / 4);
      int c = c0;
      if (kFp8Path && fp8) {
        // kFp8Unroll anchor tiles per iteration, all loaded and released before the decode
        // (amortises the per-tile barrier / stage bookkeeping over more elements)
        for (; c + kFp8Unroll - 1 < c1; c += kFp8Unroll, wv += kFp8Unroll * rw) {
          float wq[kFp8Unroll][2][kItemsPerThread];
          uint4 cq[kFp8Unroll][2][kItemsPerThread];
#pragma unroll
          for (int a = 0; a < kFp8Unroll; ++a) {
            consumer_wait(&full[stage], phase);
            const uint8_t* ba = sdata + size_t(stage) * kStageStride;
            fp8_load<kItemsPerThread>(wq[a], cq[a], ba, reinterpret_cast<const uint8_t*>(wv + a * rw), ba + scale_off,
                                      coff, roff);
            stage_release(&empty[stage]);
            if (++stage == kNStage) { stage = 0; phase ^= 1u; }
          }
          if (!skip_math) {
#pragma unroll
            for (int a = 0; a < kFp8Unroll; ++a) fp8_accum<kItemsPerThread>(acc, wq[a], cq[a]);
          }
        }
      }
      for (; c < c1; ++c, wv += rw) {
        consumer_wait(&full[stage], phase);
        const uint8_t* buf = sdata + size_t(stage) * kStageStride;
        // operands -> registers, release the stage to the producer, then the math: the
        // stage is held only for the shared-memory loads (more bytes in flight)
        if (kFp8Path && fp8) {
          float w[2][kItemsPerThread];
          uint4 code[2][kItemsPerThread];
          fp8_load<kItemsPerThread>(w, code, buf, reinterpret_cast<const uint8_t*>(wv), buf + scale_off, coff, roff);
          stage_release(&empty[stage]);  // this thread's reads of the stage are done
          if (!skip_math) fp8_accum<kItemsPerThread>(acc, w, code);
        } else {
          float w[kItemsPerThread];
          uint4 va[kItemsPerThread], vb[kItemsPerThread];
#pragma unroll
          for (int q = 0; q < kItemsPerThread; ++q) {
            w[q] = wv[irow[q]];
            va[q] = lds128(buf + irow[q] * row_bytes + ivec[q] * 16);
            vb[q] = lds128(buf + irow[q] * row_bytes + d + ivec[q] * 16);
          }
          stage_release(&empty[stage]);  // this thread's reads of the stage are done
          if (!skip_math) {
#pragma unroll
            for (int q = 0; q < kItemsPerThread; ++q) {
              const uint32_t av[4] = {va[q].x, va[q].y, va[q].z, va[q].w};
              const uint32_t bv[4] = {vb[q].x, vb[q].y, vb[q].z, vb[q].w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                ffma2(acc[0][q][2 * e], acc[0][q][2 * e + 1], w[q], w[q], bf_lo(av[e]), bf_hi(av[e]));
                ffma2(acc[0][q][8 + 2 * e], acc[0][q][8 + 2 * e + 1], w[q], w[q], bf_lo(bv[e]), bf_hi(bv[e]));
              }
            }
          }
        }
        if (++stage == kNStage) { stage = 0; phase ^= 1u; }
      }
      stage_release(&uw_empty[ub]);  // weight chunk consumed
      if (++ub == 2) { ub = 0; uphase ^= 1u; }
    }

    // base tile(s): add, rotate (K), round, store
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int r0 = s * rpt;
      if (r0 >= nrows) break;
      const int srows = min(rpt, nrows - r0);
      consumer_wait(&full[stage], phase);
      uint8_t* buf = sdata + size_t(stage) * kStageStride;
      if (n_cand > 0 || rotate) {  // COPY segments leave the staged rows untouched (bit-exact)
#pragma unroll
        for (int q = 0; q < kItemsPerThread; ++q) {
          if (irow[q] >= srows) continue;
          uint8_t* pa = buf + irow[q] * row_bytes + ivec[q] * 16;
          uint8_t* pb = pa + d;
          const uint4 a = lds128(pa);
          const uint4 b = lds128(pb);
          const uint32_t av[4] = {a.x, a.y, a.z, a.w};
          const uint32_t bv[4] = {b.x, b.y, b.z, b.w};
          float y0[8], y1[8];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            y0[2 * e] = bf_lo(av[e]) + acc[s][q][2 * e];
            y0[2 * e + 1] = bf_hi(av[e]) + acc[s][q][2 * e + 1];
            y1[2 * e] = bf_lo(bv[e]) + acc[s][q][8 + 2 * e];
            y1[2 * e + 1] = bf_hi(bv[e]) + acc[s][q][8 + 2 * e + 1];
          }
          if (rotate && !rope_il) {  // rotate_half: pair (f, f + d/2), f = 8·ivec + e
            const float2* csr = csg + ivec[q] * 8;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float2 r = csr[e];
              const float x0 = y0[e], x1 = y1[e];
              y0[e] = x0 * r.x - x1 * r.y;
              y1[e] = x1 * r.x + x0 * r.y;
            }
          } else if (rotate) {       // interleaved: pairs (2f, 2f + 1) inside each half
            const float2* ca = csg + ivec[q] * 4;           // f = 4·ivec + e/2
            const float2* cb = csg + (d >> 2) + ivec[q] * 4;  // f = d/4 + 4·ivec + e/2
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const float2 ra = ca[e >> 1], rb = cb[e >> 1];
              const float a0 = y0[e], a1 = y0[e + 1], b0 = y1[e], b1 = y1[e + 1];
              y0[e] = a0 * ra.x - a1 * ra.y;
              y0[e + 1] = a1 * ra.x + a0 * ra.y;
              y1[e] = b0 * rb.x - b1 * rb.y;
              y1[e + 1] = b1 * rb.x + b0 * rb.y;
            }
          }
          const uint4 o0 = make_uint4(pack_bf16_rn(y0[0], y0[1]), pack_bf16_rn(y0[2], y0[3]),
                                      pack_bf16_rn(y0[4], y0[5]), pack_bf16_rn(y0[6], y0[7]));
          const uint4 o1 = make_uint4(pack_bf16_rn(y1[0], y1[1]), pack_bf16_rn(y1[2], y1[3]),
                                      pack_bf16_rn(y1[4], y1[5]), pack_bf16_rn(y1[6], y1[7]));
          const int row = r0 + irow[q];  // within the unit
          if (tstore) {
            sts128(pa, o0);  // in place; the whole tile leaves with one bulk store below
            sts128(pb, o1);
          } else if (!skip_store) {
            bf16* o = dst + int64_t(row) * d + ivec[q] * 8;
            stg128_cs(o, o0);
            stg128_cs(o + d / 2, o1);
          }
          if (dbg != nullptr) {
            float* od = dbg + int64_t(row) * d + ivec[q] * 8;
            float4* p0 = reinterpret_cast<float4*>(od);
            float4* p1 = reinterpret_cast<float4*>(od + d / 2);
            p0[0] = make_float4(acc[s][q][0], acc[s][q][1], acc[s][q][2], acc[s][q][3]);
            p0[1] = make_float4(acc[s][q][4], acc[s][q][5], acc[s][q][6], acc[s][q][7]);
            p1[0] = make_float4(acc[s][q][8], acc[s][q][9], acc[s][q][10], acc[s][q][11]);
            p1[1] = make_float4(acc[s][q][12], acc[s][q][13], acc[s][q][14], acc[s][q][15]);
          }
        }
      } else if (!tstore && !skip_store) {
#pragma unroll
        for (int q = 0; q < kItemsPerThread; ++q) {
          if (irow[q] >= srows) continue;
          const uint8_t* pa = buf + irow[q] * row_bytes + ivec[q] * 16;
          bf16* o = dst + int64_t(r0 + irow[q]) * d + ivec[q] * 8;
          stg128_cs(o, lds128(pa));
          stg128_cs(o + d / 2, lds128(pa + d));
        }
      }
      if (tstore) {
        // all consumer writes of the tile -> visible to the async proxy, then one bulk store;
        // the stage is released only once the store has finished reading shared memory
        fence_proxy_async_smem();
        named_bar_sync(kConsumerBar, kConsumerWarps * 32);
        if (threadIdx.x == 0) {
          bulk_s2g(dst + int64_t(r0) * d, buf, uint32_t(srows) * row_bytes);
          bulk_wait_read_all();
          mbar_arrive_cnt(&empty[stage], kConsumerWarps * kArrivals);  // for all consumers (named barrier above)
        }
      } else {
        stage_release(&empty[stage]);
      }
      if (++stage == kNStage) { stage = 0; phase ^= 1u; }
    }
  }
  if (tma_store && threadIdx.x == 0) bulk_wait_all();  // global writes complete before exit
  if (hdr.any_stg) __threadfence_system();  // peer-GPU rows: visible system-wide before the kernel ends
}

// The instantiations (one CTA per SM): 8 + 1 warps for bf16 tables; 16 + 1 for tables that
// read an fp8 pool at a generic head_dim (17 warps leave 96 registers per thread, as ptxas
// allocates for 20 warps); realign_kernel_fp8w8 below for fp8 at head_dim 128.
template <int kConsumerWarps, int kD>
__global__ void __launch_bounds__((kConsumerWarps + 1) * 32, 1)
    realign_kernel(const uint8_t* __restrict__ tab, int variant) {
  realign_body<kConsumerWarps, kD, kConsumerWarps == 16>(tab, variant);
}

// fp8 tables (head_dim 128, the default): 8 consumer warps with two items per thread under
// a 144-register cap.  ptxas rounds a CTA to 12 warps, so 12 x 32 x 144 = 55,296 registers
// leave 10,240 for one CTA of the next request's match kernel beside the realign when
// requests are pipelined.  Measured at config 2 (profiles/r02h_fp8_warps.txt): step 2.90 ->
// 2.82 ms against the 16-warp kernel; at 152 registers (no cap needed, 149 used) the
// realign alone is 1 % faster but the match no longer fits beside it, at 128 it spills.
// KVCOMM_REALIGN_FP8_WARPS=16 selects the 16-warp kernel.
#ifndef KVC_FP8W8_REGS
#define KVC_FP8W8_REGS 144
#endif
__global__ void __maxnreg__(KVC_FP8W8_REGS) realign_kernel_fp8w8(const uint8_t* __restrict__ tab, int variant) {
  realign_body<8, 128, true>(tab, variant);
}

int realign_grid_size(int device) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (sms <= 0) sms = 148;
  const char* e = getenv("KVCOMM_REALIGN_GRID");  // measurement knob: persistent CTAs (<= SMs)
  const int g = e ? atoi(e) : 0;
  return g > 0 && g < sms ? g : sms;
}

cudaError_t launch_realign(const void* table_dev, const TableHdr& hdr, int grid, cudaStream_t s) {
  cudaError_t e = launch_realign_prep(table_dev, hdr, s);
  return e != cudaSuccess ? e : launch_realign_main(table_dev, hdr, grid, s);
}

cudaError_t launch_realign_prep(const void* table_dev, const TableHdr& hdr, cudaStream_t s) {
  if (hdr.n_seg <= 0) return cudaSuccess;
  realign_prep_kernel<<<dim3(hdr.n_seg, kPrepY), 256, 0, s>>>(reinterpret_cast<uint8_t*>(const_cast<void*>(table_dev)));
  return cudaGetLastError();
}

cudaError_t launch_realign_main(const void* table_dev, const TableHdr& hdr, int grid, cudaStream_t s) {
  static bool attr_set[64] = {false};
  static int variant = -1, cw_env = 0, fp8w_env = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    const int smem8 = int(realign_smem_bytes(ring_stages<false>())), smem16 = int(realign_smem_bytes(ring_stages<true>()));
    cudaError_t e = cudaFuncSetAttribute(realign_kernel<8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem8);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(realign_kernel<16, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem16);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(realign_kernel<8, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem8);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(realign_kernel<16, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem16);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(realign_kernel_fp8w8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem16);
    // all of the SM's 228 KiB as shared memory: the realign CTA takes ~153 KiB (bf16 ring), and
    // the rest must stay free for the CTAs of the next request's match / prep kernels that run
    // beside it when requests are pipelined (kvcomm_plan_set_realign_stream); at the default
    // carveout the SM is configured just large enough for the realign CTA alone
    for (const void* k : {(const void*)realign_kernel<8, 0>, (const void*)realign_kernel<16, 0>,
                          (const void*)realign_kernel<8, 128>, (const void*)realign_kernel<16, 128>,
                          (const void*)realign_kernel_fp8w8})
      if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    attr_set[dev & 63] = true;
  }
  if (variant < 0) {
    const char* v = getenv("KVCOMM_REALIGN_VARIANT");
    variant = v ? atoi(v) : 0;
    if (!kProbeVariants && (variant & (2 | 32)))
      fprintf(stderr, "libkvcomm: KVCOMM_REALIGN_VARIANT bits 1/5 (skip stores / math) exist only in probe "
                      "builds; ignored\n");
    const char* c = getenv("KVCOMM_REALIGN_CONSUMER_WARPS");
    if (c) cw_env = atoi(c);
    const char* f = getenv("KVCOMM_REALIGN_FP8_WARPS");
    if (f) fp8w_env = atoi(f);
  }
  // 8 consumer warps stream bf16 pools at the HBM roofline; fp8 pools at head_dim 128 take
  // realign_kernel_fp8w8 (8 warps, two items per thread), other head_dims the 16-warp kernel
  const int cw = hdr.any_fp8 ? 16 : (cw_env == 16 ? 16 : 8);
  if (hdr.n_seg <= 0 || hdr.total_units <= 0) return cudaSuccess;
  const int64_t g = hdr.total_units < grid ? hdr.total_units : grid;
  const uint8_t* t = reinterpret_cast<const uint8_t*>(table_dev);
  const size_t smem = realign_smem_bytes(hdr.any_fp8 ? ring_stages<true>() : ring_stages<false>());
  const bool d128 = hdr.d == 128 && !(variant & 256);  // bit8: generic-d kernel (probe)
  if (hdr.any_fp8 && d128 && fp8w_env != 16)
    realign_kernel_fp8w8<<<int(g), 9 * 32, smem, s>>>(t, variant);
  else if (cw == 8 && d128)
    realign_kernel<8, 128><<<int(g), 9 * 32, smem, s>>>(t, variant);
  else if (cw == 8)
    realign_kernel<8, 0><<<int(g), 9 * 32, smem, s>>>(t, variant);
  else if (d128)
    realign_kernel<16, 128><<<int(g), 17 * 32, smem, s>>>(t, variant);
  else
    realign_kernel<16, 0><<<int(g), 17 * 32, smem, s>>>(t, variant);
  return cudaGetLastError();
}

}  // namespace kvc
