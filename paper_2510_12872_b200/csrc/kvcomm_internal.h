// Internal structures shared between the C-ABI layer (kvcomm_api.cu) and the kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace kvc {

using bf16 = __nv_bfloat16;

// Bytes of data one realign pipeline stage carries (a tile of rows_per_tile token
// rows of one (layer, head, K|V) plane): 16 KiB = 64 rows of d=128 bf16.
constexpr int kStageBytes = 16384;
constexpr int kStageStride = kStageBytes + 1024;  // an fp8 block (codes + row scales) fits too
#ifndef KVC_UNITW
#define KVC_UNITW 16384
#endif
constexpr int kUnitWBytes = KVC_UNITW;  // weight chunk buffer: [anchors][weight_row_stride] floats
constexpr int kMaxCapDev = 1024;    // == KVCOMM_MAX_CAPACITY
constexpr int kMaxTopK = 32;        // == KVCOMM_MAX_TOPK
constexpr int kMatchChunks = 32;    // position-block chunks of the two-pass d̄ reduction
constexpr int kMatchStageBytes = 16384;  // TMA distance kernel: bytes per ring stage
constexpr int kMatchTmaMaxCand = 256;    // TMA distance kernel: candidates per job
constexpr int kMatchTmaMaxDe = 8192;     // TMA distance kernel: embedding width
constexpr int kMatchRingWarps = 8;       // row-ring distance kernel: consumer warps (ring depth: a multiple)

// rows per realign tile (16 KiB of bf16 rows) for head_dim d
__host__ __device__ constexpr int rows_per_tile(int d) { return kStageBytes / (2 * d); }
// fp8 storage block: two tiles' rows of d e4m3 codes, then their fp32 row scales, padded
// to 16 bytes (TMA bulk granularity) — about 16 KiB, one contiguous copy per anchor tile
__host__ __device__ constexpr int fp8_rows_per_block(int d) { return 2 * rows_per_tile(d); }
__host__ __device__ constexpr int fp8_block_bytes(int d) { return (fp8_rows_per_block(d) * (d + 4) + 15) & ~15; }
// token rows of one realign work unit: one bf16 tile, or one fp8 block
__host__ __device__ constexpr int unit_rows(int d, int fp8) { return fp8 ? fp8_rows_per_block(d) : rows_per_tile(d); }
// row stride of the weight blocks (16-byte multiple)
__host__ __device__ constexpr int weight_row_stride(int rows) { return (rows + 3) & ~3; }

// One segment of a realign batch, as the kernels see it (device resident).
struct SegDev {
  const bf16* base[2];  // K, V base rows, [Ls][Hs][base_ld][d]
  bf16* dst[2];         // destination rows: (l, h, row) at ((l*dst_heads + h)*dst_ld + row)*d
  float* dbg[2];        // optional fp32 blended offsets [Ls][Hs][L_seg][d]
  const float* w;       // PLACEHOLDER: W rows by slot, row r at w + r*ld_w (w_by_slot = 1)
  const float* wt;      // weight blocks [tiles][n_cand][weight_row_stride(unit rows)] (prep kernel)
  const bf16* off;      // offsets of (consumer, kind).  bf16: element (slot, plane, l, h, row, e) at
                        //   slot*slot_stride + plane*plane_stride + (lh*off_ld + row)*d + e;
                        //   fp8: a byte pointer, block (slot, plane, lh, tile) at
                        //   slot*slot_stride + plane*plane_stride + lh*off_ld + tile*fp8_block_bytes
  const double* inv_freq;  // [d/2] of the owning pool
  const float* wbar;    // PREFIX: scalar weights [capacity] (expanded by the prep kernel)
  int64_t base_ld, dst_ld, ld_w;
  int64_t slot_stride, plane_stride, off_ld;  // bf16: elements / rows; fp8: bytes
  int64_t unit_begin;   // first work unit of this segment's group (same for every member)
  int32_t L_seg, target_start, delta, n_cand;
  int32_t cand_off;     // index of this segment's first candidate in Table::cand
  int32_t cs_off;       // index (in float2) of its cos/sin table in Table::cs
  int32_t w_by_slot;    // 1: weights from W[slot] (PLACEHOLDER); 0: from w̄[slot] (PREFIX)
  int32_t tiles;        // ceil(L_seg / unit_rows)
  int32_t n_gate;       // segment runs iff every listed match verdict is SHAREABLE (device-side
  int32_t gate_off;     //   branch of Alg. 1); indices into Table::cand area, n_gate = 0: always
  int32_t group_size;   // segments sharing this base tile (consecutive in the table; units interleave
                        //   members so the shared base tile is read from HBM once and hit in L2 after)
  int32_t fp8;          // offsets stored as blocked e4m3 codes + row scales
  int64_t wt_off;       // float offset of this segment's weight blocks in Table::wt
  int32_t dst_stg;      // 0: local rows, TMA bulk store; 2: peer rows, TMA bulk store to the peer address;
                        // 1: write rows with per-thread stores (destination on a peer GPU, mapped by
                        //   CUDA IPC: the fused gather of SURVEY §8(e)), 0: TMA bulk store
  int32_t rope_il;      // K's RoPE pairs: 0 (f, f + d/2) rotate_half, 1 (2f, 2f + 1) interleaved
  int32_t dst_heads;    // heads per layer of the destination layout (>= Hs): a head shard writes its
                        //   [Ls][Hs] block into a consumer's full [L][H][N][d] cache (70B grid, §9)
  int32_t group_member;  // index of this segment within its group (0 .. group_size-1)
};

// One realign work unit as the prep kernel lays it out (UnitDev[total_units] at
// TableHdr::unit_off): the persistent kernel reads one 16-byte descriptor per unit
// instead of decoding the unit index (binary search over segments + 64-bit divisions,
// once per warp per unit).  s = -1: the segment's gate is closed (Alg. 1 branch).
struct UnitDev {
  int32_t s, l, h, tp;  // segment, layer, head, (tile << 1) | plane
};

struct MatchResultDev {
  double entropy, threshold;
  int32_t verdict, tie_flag, tie_count;
  int32_t shard_mismatch;  // sharded matching: another rank matched a different job layout
};

// Device-side work table for one realign launch (lives in one contiguous buffer).
struct TableHdr {
  int32_t n_seg, d, Ls, Hs;
  int32_t rows_per_tile, any_fp8;  // any_fp8: some segment reads an fp8 pool
  int32_t any_stg, _pad1;          // any_stg: some segment writes peer rows (system-scope fence at the end)
  int64_t total_units;
  // byte offsets from the table base
  int64_t seg_off, cand_off, cs_off, wt_off, unit_off;
  const MatchResultDev* gate_results;  // verdicts the segments' gates index (device), or null
};

// Launchers (stream-ordered).  Return cudaGetLastError().
cudaError_t launch_realign(const void* table_dev, const TableHdr& hdr, int grid, cudaStream_t s);
// the two halves of launch_realign: the prep kernel (unit list, cos/sin, weight blocks), then
// the persistent realign kernel (callers may put them on different streams, ordered by an event)
cudaError_t launch_realign_prep(const void* table_dev, const TableHdr& hdr, cudaStream_t s);
cudaError_t launch_realign_main(const void* table_dev, const TableHdr& hdr, int grid, cudaStream_t s);
int realign_grid_size(int device);

constexpr int kMaxMatchPeers = 7;   // one box: 8 GPUs

// One matching job (one query sample against one pool), as the kernels see it.
struct MatchJob {
  const bf16* query;        // [L_phi][De]
  const bf16* emb;          // pool slab [cap][maxlen][De]
  int64_t slot_stride;      // elements between slots of emb
  float* W;                 // [cap][ld_w]
  int64_t ld_w;
  int32_t* idx;             // [L_phi][top_k] or null
  double* dist_user;        // optional [cap][ld_w]
  double* partial;          // pool scratch [n_blocks][stride]: stride n_cand (l2) or 2 n_cand + 1 (cosine)
  double* chunks;           // pool scratch [kMatchChunks][stride]: fixed-order sums of chunks of blocks
  float* wbar;              // [cap]
  double gamma;
  int32_t n_cand, cap, L_phi, De;
  int32_t top_k;            // effective k (0 = dense, paper default)
  int32_t scalar_mode;      // 0 Frobenius: partial = Σ d², 1 mean-ℓ2: partial = Σ d
  int32_t cosine;           // 1: d = 1 - cos; partials Σ q·a, Σ a·a (per candidate) and Σ q·q
  int32_t cand_off;         // into MatchHdr ints: candidate slot ids [n_cand]
  int32_t s2c_off;          // into MatchHdr ints: slot -> candidate index or -1 [cap]
  int32_t block_begin, n_blocks;  // block_begin: first work item of this job; n_blocks: ALL position blocks
  // Sharded matching: this launch computes position blocks
  // own_lo + k * own_step (k < n_own) only and stores their W columns and partial rows into
  // this GPU's buffers AND every peer's copy (IPC-mapped) — the chunk/finalize passes
  // then run on the complete arrays on every rank.  Unsharded: own_lo 0, own_step 1,
  // n_own = n_blocks, n_peer 0.
  int32_t own_lo, n_own;    // position blocks own_lo, own_lo + own_step, ... (n_own of them)
  int32_t own_step;
  int32_t emb_world;        // > 1: the pool stores only its blocks' rows, compacted (emb_shard)
  int32_t n_peer, _pad_peer;
  // Sharded: a block's W columns travel to the peers position-major, X[i][cap] (row i =
  // the cap weights of position i, one coalesced run per warp store) instead of as
  // scattered 4-byte stores into the slot-major W; each rank's chunk kernel then copies
  // the positions it does not own from its own X into W.
  float* X;                            // this rank's exchange rows [n_blocks * P][cap] (peers write them)
  float* X_peer[kMaxMatchPeers];       // the same rows in every peer's plan buffer
  double* partial_peer[kMaxMatchPeers];
};

// Device-side table of one batched match launch.
struct MatchHdr {
  int32_t n_jobs, total_blocks, P, any_peer;   // total_blocks: work items of this launch (owned blocks)
  int64_t job_off, int_off, res_off, tie_off;   // byte offsets from the table base
  // Sharded matching: every rank stores a fingerprint of its job layout (candidates,
  // lengths, modes) into slot `shard_rank` of every rank's fingerprint array; finalize
  // compares all `shard_world` slots with its own and, on any difference, reports the
  // job NewAnchor with shard_mismatch set (the realign gate then skips its segments).
  uint64_t fingerprint;
  int32_t shard_rank, shard_world;
  // TMA-streamed distance kernel (l2 jobs with n_cand <= kMatchTmaMaxCand, D_e <= 8192): ring
  // stages of kMatchStageBytes, query double buffer of tma_qbytes each, partial table for
  // tma_cmax candidates; tma = 0 selects the register-streaming kernel
  int32_t tma, tma_stages, tma_qbytes, tma_cmax;
  int32_t max_de;                         // largest D_e of the launch's jobs (selects the kernel)
  int32_t ring_row_bytes;                 // tma = 2 (row-ring kernel): bytes per ring stage (max D_e x 2)
  int32_t beside_realign;                 // pipelined plan run: the match shares the SMs with a realign
  int32_t _pad_br;
  uint64_t* fp_dst[kMaxMatchPeers + 1];   // [r]: this rank's slot in rank r's array
  const uint64_t* fp_mine;                // this rank's array [shard_world]
};

// distance + per-position weights over all jobs' blocks, then one finalize block per job
cudaError_t launch_match_batch(const void* table_dev, const MatchHdr& hdr, size_t smem_bytes, cudaStream_t s);
// the two halves of launch_match_batch (sharded plans put the cross-rank sync between them)
cudaError_t launch_match_dist(const void* table_dev, const MatchHdr& hdr, size_t smem_bytes, cudaStream_t s);
cudaError_t launch_match_reduce(const void* table_dev, const MatchHdr& hdr, cudaStream_t s);
// dynamic shared memory of the TMA distance kernel (ring stages, query buffers, partials)
size_t match_tma_smem(int stages, int qbytes, int cmax);
// dynamic shared memory of the row-ring distance kernel (stages of one anchor row each)
size_t match_ring_smem(int stages, int row_bytes, int qbytes, int cmax, int P);

// Strided row-block copy: for l<Ls, h<Hs, i<rows: dst[(l*Hs+h)*dst_ld + i] = src[(l*Hs+h)*src_ld + i]
cudaError_t launch_copy_rows(const bf16* src, int64_t src_ld, bf16* dst, int64_t dst_ld, int Ls, int Hs,
                             int rows, int d, cudaStream_t s);
// Batched insert-path jobs (one launch per insert instead of one per (consumer, kind,
// plane)); passed by value as kernel parameters.
struct CopyJob {
  const bf16* src;
  void* dst;                // bf16 rows, or (fp8 pools) the blocked e4m3 region
  int64_t src_ld, dst_ld;   // rows; fp8: dst_ld = bytes per (layer, head) region
  int32_t rows, _pad;
};
constexpr int kMaxCopyJobs = 64;
struct CopyJobs {
  CopyJob j[kMaxCopyJobs];
};
struct MeasureJob {
  const bf16 *kr, *vr, *kb, *vb;
  void *dk, *dv;            // bf16 rows, or (fp8 pools) blocked e4m3 regions
  int64_t real_ld, base_ld, dst_ld;  // fp8: dst_ld = bytes per (layer, head) region
  int32_t rows, delta;
};
constexpr int kMaxMeasureJobs = 32;
struct MeasureJobs {
  MeasureJob j[kMaxMeasureJobs];
};
cudaError_t launch_copy_rows_batch(const CopyJobs& jobs, int n, int Ls, int Hs, int d, cudaStream_t s);
cudaError_t launch_measure_batch(const MeasureJobs& jobs, int n, int Ls, int Hs, int d, int interleaved,
                                 const double* inv_freq, cudaStream_t s);
cudaError_t launch_quantize_rows_batch(const CopyJobs& jobs, int n, int Ls, int Hs, int d, cudaStream_t s);
cudaError_t launch_measure_fp8_batch(const MeasureJobs& jobs, int n, int Ls, int Hs, int d, int interleaved,
                                     const double* inv_freq, cudaStream_t s);
// Contiguous copy of n bf16 elements (multiple of 8).
cudaError_t launch_copy_flat(const bf16* src, bf16* dst, int64_t n, cudaStream_t s);
// fp8 (e4m3 + per-row fp32 scale) offset storage in blocks of fp8_rows_per_block(d) rows
// (codes, then the block's row scales); lh_bytes = bytes per (layer, head) region.
// Blocked e4m3 rows -> dense codes [lh][rows][d] + scales [lh][rows] (inspection / tests).
cudaError_t launch_read_fp8(const uint8_t* src, int64_t lh_bytes, uint8_t* codes, float* scales, int Ls, int Hs,
                            int rows, int d, cudaStream_t s);
}  // namespace kvc
