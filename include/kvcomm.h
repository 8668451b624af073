/*
 * kvcomm.h — C ABI of the B200-native KVComm anchor-realignment hot path.
 *
 * KVComm (arXiv 2510.12872) reuses the KV-cache of a text segment that an agent
 * shares with other agents: the segment's *base* cache (computed standalone) is
 * moved under a new prefix by adding an *offset* interpolated from anchors.
 * "P:n" below is a line of the paper text, with the
 * equation or section it falls in.  The library implements:
 *
 *   a0  anchor-pool store + insert (Alg. 1 fallback branch P:786-796; §3.3)
 *   a1  candidate filter / length clause of Eq. 5
 *   a2  embedding distances ‖h_φ - h_ψ‖₂                   (Eq. 5/6)
 *   a3  softmax weights, entropy, NewAnchor verdict         (Eq. 5, Eq. 6)
 *   a4  offset blend                                        (Eq. 6, Eq. 7)
 *   a5  RoPE position delta + add into the base cache
 *   a6  concatenation of the updated segments + ledger      (Alg. 1)
 *
 * Conventions for every call
 *   - Pointers named "device" must be CUDA device pointers on the pool's device,
 *     16-byte aligned.  "host" pointers are ordinary host memory, only read during
 *     the call.  The caller owns every buffer it passes; the pool owns its slabs.
 *   - Tensors of one model shard use the layout [Ls][Hs][ld][d] bf16 (token rows
 *     of d elements, d fastest; `ld` = row stride between consecutive (layer,
 *     head) blocks, >= the number of rows used).  Ls/Hs are the pool's shard sizes.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call is
 *     stream-ordered and asynchronous except kvcomm_match_anchors, which
 *     synchronises `stream` to fill its host `info` (Algorithm 1's reuse/fallback
 *     branch is a host decision).
 *   - Errors never throw across the ABI: each call returns a kvcomm_status and sets
 *     a thread-local message (kvcomm_last_error_message).  Contract violations are
 *     errors, never silent fallbacks.
 *   - Thread safety: a pool admits many concurrent readers (match, realign) or one
 *     writer (insert, set_offsets, evict, record_access, destroy).
 */
#ifndef KVCOMM_H
#define KVCOMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVCOMM_API __attribute__((visibility("default")))

#define KVCOMM_VERSION 1
#define KVCOMM_MAX_CAPACITY 1024  /* anchors per pool (𝒱) */
#define KVCOMM_MAX_CONSUMERS 64   /* (agent, slot) consumers per pool */
#define KVCOMM_MAX_TOPK 32
#define KVCOMM_ALL_CONSUMERS (-1)

typedef enum {
  KVCOMM_OK = 0,
  KVCOMM_ERR_INVALID_ARGUMENT = 1, /* null pointer, odd d, gamma outside [0,1], misaligned */
  KVCOMM_ERR_SHAPE_MISMATCH = 2,   /* length / layer / head mismatch          */
  KVCOMM_ERR_NO_CANDIDATES = 3,    /* realign with an empty candidate set                    */
  KVCOMM_ERR_MISSING_OFFSET = 4,   /* reuse needs an offset the anchor lacks          */
  KVCOMM_ERR_POSITION_GAP = 5,     /* concat ledger: segments leave a hole                   */
  KVCOMM_ERR_POSITION_OVERLAP = 6, /* concat ledger: segments overlap                        */
  KVCOMM_ERR_NOT_FOUND = 7,        /* empty slot / unknown consumer                                  */
  KVCOMM_ERR_OUT_OF_MEMORY = 8,
  KVCOMM_ERR_CUDA = 9,
  KVCOMM_ERR_NCCL = 10,
  KVCOMM_ERR_IO = 11               /* checkpoint file missing, unreadable, truncated or corrupt       */
} kvcomm_status;

typedef enum { KVCOMM_SHAREABLE = 0, KVCOMM_NEW_ANCHOR = 1 } kvcomm_verdict;

typedef enum {
  KVCOMM_REASON_OK = 0,
  KVCOMM_REASON_EMPTY_POOL = 1,     /* pool holds no anchor                                   */
  KVCOMM_REASON_TOO_LONG = 2,       /* L_φ > max_{ψ∈𝒜} L_ψ  (Eq. 5 first clause)             */
  KVCOMM_REASON_NO_CANDIDATES = 3,  /* no anchor with L_ψ >= L_φ and the consumer's offsets  */
  KVCOMM_REASON_HIGH_ENTROPY = 4,   /* H_{φ|𝒜} > γ log|𝒜_φ|  (Eq. 5 second clause)           */
  KVCOMM_REASON_SHARD_MISMATCH = 5  /* sharded matching: the ranks' job layouts differ (pools
                                       out of step across ranks); treated as NewAnchor        */
} kvcomm_reason;

typedef enum { KVCOMM_SCALAR_FROBENIUS = 0, KVCOMM_SCALAR_MEAN_L2 = 1 } kvcomm_scalar_distance;
typedef enum { KVCOMM_SIM_L2 = 0, KVCOMM_SIM_COSINE = 1 } kvcomm_similarity;
typedef enum { KVCOMM_OFFSET_BF16 = 0, KVCOMM_OFFSET_FP8_E4M3 = 1 } kvcomm_offset_format;
typedef enum { KVCOMM_PLACE_DEVICE = 0, KVCOMM_PLACE_HOST = 1 } kvcomm_placement;
typedef enum { KVCOMM_ROPE_HALF = 0, KVCOMM_ROPE_INTERLEAVED = 1 } kvcomm_rope_layout;
/* COPY: rows copied verbatim (no offsets, no rotation; bit-exact), e.g. p_(m,0) of the
 * concatenation (reading A20) riding in the same launch as the realignment. */
typedef enum { KVCOMM_PLACEHOLDER = 0, KVCOMM_PREFIX = 1, KVCOMM_COPY = 2 } kvcomm_segment_kind;
typedef enum { KVCOMM_OFFSET_GIVEN = 0, KVCOMM_OFFSET_MEASURE = 1 } kvcomm_offset_mode;

typedef struct kvcomm_pool_s* kvcomm_pool_t;

/* Pool geometry.  One pool per placeholder name ("Each placeholder initializes
 * an individual anchor pool"); consumer c = one (agent m, slot i) that reads the pool.
 * The pool holds layers [layer_begin, layer_end) and KV heads [head_begin, head_end)
 * of the model (Ls = layer_end-layer_begin, Hs = head_end-head_begin). */
typedef struct {
  int32_t device;          /* CUDA device ordinal                                        */
  int32_t num_layers;      /* L of the model                                             */
  int32_t layer_begin, layer_end;
  int32_t num_kv_heads;    /* H of the model                                             */
  int32_t head_begin, head_end;
  int32_t head_dim;        /* d: multiple of 16, <= 256                                   */
  int32_t emb_dim;         /* D_e of the token embeddings h (reading A1): multiple of 8  */
  int32_t capacity;        /* 𝒱, 1..KVCOMM_MAX_CAPACITY (paper default 20)        */
  int32_t max_anchor_len;  /* longest anchor sample L_ψ the pool will store             */
  int32_t num_consumers;   /* 1..KVCOMM_MAX_CONSUMERS                                     */
  int32_t scalar_distance; /* sample-level distance d̄ of Eq. 5/7 (reading A4):
                              KVCOMM_SCALAR_FROBENIUS (0, default) d̄_j = sqrt(Σ_i d[i,j]²),
                              KVCOMM_SCALAR_MEAN_L2  (1)           d̄_j = mean_i d[i,j]     */
  int32_t similarity;      /* matching score (Table A.4):
                              KVCOMM_SIM_L2 (0, paper default): d = ‖h_φ[i] - h_ψ[i]‖₂, w = softmax(-d);
                              KVCOMM_SIM_COSINE (1): d = 1 - cos(h_φ[i], h_ψ[i]), w = softmax(cos);
                              sample level: 1 - <h_φ,h_ψ>_F / (‖h_φ‖_F ‖h_ψ‖_F)            */
  int32_t offset_format;   /* KVCOMM_OFFSET_BF16 (0, default, exact storage) |
                              KVCOMM_OFFSET_FP8_E4M3 (1): each stored offset row of d values is
                              e4m3 codes + one fp32 scale = max|x|/448, code = RNE_sat(x/scale)
                              (the compression P:1518 names as future work; lossy, ~1.9x fewer
                              offset bytes; requires head_dim >= 64)                      */
  int32_t placement;       /* KVCOMM_PLACE_DEVICE (0, default) | KVCOMM_PLACE_HOST (1): the offset
                              slabs live in pinned, mapped host memory and the same kernels
                              stream them over the host link (the CPU-offloaded anchors of
                              A.4.4: pools larger than HBM)                  */
  int32_t rope_layout;     /* RoPE pairing of K's head dimension (reading A12):
                              KVCOMM_ROPE_HALF (0, default): HF rotate_half, pairs (f, f + d/2);
                              KVCOMM_ROPE_INTERLEAVED (1): GPT-J style, pairs (2f, 2f + 1).
                              Both rotate pair f by δ·inv_freq[f].                        */
  int16_t emb_shard_rank;  /* embedding rows held by this pool ("sharded
                              embeddings").  emb_shard_world <= 1 (default 0): every row.  G =
                              emb_shard_world in [2, 8]: only rows i with (i / 2) mod G ==
                              emb_shard_rank — the position blocks this rank matches under
                              sharded matching (kvcomm_plan_match_shard with the same rank and
                              world; any other match of the pool is INVALID_ARGUMENT) — so each
                              of G GPUs stores 1/G of the embeddings instead of all of them.   */
  int16_t emb_shard_world;
  const int32_t* prefix_len; /* host [num_consumers]: |p_(m,i)| following this placeholder */
  const double* inv_freq;  /* host [head_dim/2]: RoPE inverse frequencies (copied)        */
} kvcomm_pool_config;

/* A strided view of K and V rows of one shard: element (l, h, i, e) lives at
 * ptr + ((l*Hs + h)*ld + i)*d + e.  `start` = absolute position of row 0. */
typedef struct {
  const void* k;   /* device bf16 */
  const void* v;   /* device bf16 */
  int64_t ld;      /* rows between (l,h) blocks; 0 means "= the segment length"   */
  int32_t start;   /* absolute token position of row 0 (MEASURE mode only)         */
  int32_t _pad;
} kvcomm_kv_view;

/* Offsets of one anchor for one consumer (Table A.1: agent_id_ph / agent_id_pf).
 * GIVEN:   ph_delta / pf_delta hold ΔK,ΔV already in the base frame (reading A10).
 * MEASURE: the device measures them (Alg. 1; step a0):
 *          ΔK = R_{-(s_real - s_base)} K_real - K_base,  ΔV = V_real - V_base,
 *          fp32 arithmetic, one RNE rounding to bf16.
 * Either part may be omitted by passing k == NULL (it stays absent/unchanged). */
typedef struct {
  int32_t consumer;
  int32_t mode;            /* kvcomm_offset_mode */
  kvcomm_kv_view ph_delta; /* [Ls,Hs,L_ψ,d]  (GIVEN)      */
  kvcomm_kv_view pf_delta; /* [Ls,Hs,P_c,d]  (GIVEN)      */
  kvcomm_kv_view ph_real, ph_base; /* [Ls,Hs,L_ψ,d] (MEASURE) */
  kvcomm_kv_view pf_real, pf_base; /* [Ls,Hs,P_c,d] (MEASURE) */
} kvcomm_offset_desc;

typedef struct {
  int32_t occupied;
  int32_t length;          /* L_ψ */
  int64_t access_count;
  int64_t insertion_index;
  uint64_t ph_present_mask; /* bit c: placeholder offsets of consumer c present */
  uint64_t pf_present_mask; /* bit c: prefix offsets of consumer c present      */
} kvcomm_slot_info;

typedef struct {
  int32_t verdict;         /* kvcomm_verdict                                             */
  int32_t reason;          /* kvcomm_reason                                              */
  int32_t n_candidates;    /* |𝒜_φ|                                                       */
  int32_t top_k;           /* effective k (n_candidates when top_k = 0)                  */
  int32_t candidates[KVCOMM_MAX_CAPACITY]; /* slot ids of 𝒜_φ, ascending               */
  double entropy;          /* H = -Σ w̄ log w̄ (reading A5)                                */
  double threshold;        /* γ log|𝒜_φ|                                                  */
  int32_t verdict_in_tie_band; /* |H - threshold| <= 1e-6 * threshold                   */
  int32_t tie_band_count;  /* positions whose top-k boundary/order has a relative
                              distance gap <= 1e-6 (0 when top_k = 0)                   */
} kvcomm_match_info;

/* One segment to realign (step a4+a5).  PLACEHOLDER (Eq. 6): token i of the
 * segment uses weights W[slot][i].  PREFIX (Eq. 7, reading A3): every token uses
 * the scalar w̄[slot].  Output rows target_start .. target_start+L_seg-1 of dst:
 *   K̂ = R_δ(K_base + Σ_j w_j ΔK_j),  V̂ = V_base + Σ_j w_j ΔV_j,  δ = target_start - base_start,
 * accumulated in fp32, rounded once (RNE) to bf16.
 * COPY: base rows are copied to dst unchanged; consumer/weights/candidates/base_start
 * are ignored (pool only supplies the geometry and device). */
typedef struct {
  kvcomm_pool_t pool;
  int32_t consumer;        /* 0..num_consumers-1                                          */
  int32_t kind;            /* kvcomm_segment_kind                                         */
  const float* weights;    /* device. PLACEHOLDER: W [capacity][ld_w] (slot-major, as
                              written by kvcomm_match_anchors).  PREFIX: w̄ [capacity]  */
  int64_t ld_w;            /* PLACEHOLDER: row stride of W, multiple of 4, >= L_seg        */
  const int32_t* candidates; /* host [n_candidates]: slot ids to blend (info.candidates) */
  int32_t n_candidates;
  int32_t L_seg;           /* tokens; PREFIX requires L_seg == prefix_len[consumer]; 0 = no-op */
  kvcomm_kv_view base;     /* device [Ls,Hs,ld,d] base K/V rows 0..L_seg-1               */
  int32_t base_start;      /* placeholder base: 0; prefix base: |p_(m,0)| (reading A11)   */
  int32_t target_start;    /* first destination row (absolute position in the prompt)     */
  void* dst_k;             /* device bf16 [Ls,Hs,dst_ld,d]                                 */
  void* dst_v;
  int64_t dst_ld;          /* prompt length N of the consumer                             */
  float* debug_delta_k;    /* optional device fp32 [Ls,Hs,L_seg,d]: Σ_j w_j ΔK_j (parity) */
  float* debug_delta_v;
  int32_t dst_heads;       /* heads per layer of the destination layout; 0 = the pool's Hs.
                              Element (l, h, row) of this shard lands at
                              dst + ((l*dst_heads + h)*dst_ld + row)*d, so a KV-head shard
                              (pool head_range [h0,h1)) writes straight into a consumer's full
                              [L][H][N][d] cache: dst = cache + ((l0*H + h0)*N)*d, dst_heads = H
                              (SURVEY §8(e) 70B layer x KV-head grid).  SHAPE_MISMATCH if < Hs. */
  int32_t _pad;
} kvcomm_realign_desc;

/* A segment of the consumer's prompt for the concatenation ledger (step a6).
 * src.k != NULL: rows are copied verbatim from src (e.g. p_(m,0), reading A20);
 * src.k == NULL: rows were already written in place (by realign). */
typedef struct {
  int32_t start;
  int32_t length;
  kvcomm_kv_view src;
} kvcomm_segment_ref;

/* ---- status / diagnostics ------------------------------------------------- */
KVCOMM_API const char* kvcomm_status_string(kvcomm_status s);
KVCOMM_API const char* kvcomm_last_error_message(void);      /* thread-local */
KVCOMM_API int32_t kvcomm_version(void);
/* Number of CUDA kernels this library has launched in this process. */
KVCOMM_API int64_t kvcomm_kernel_launch_count(void);

/* ---- a0: anchor-pool store ------------------------------------------------- */
/* Allocates the pool's device slabs (embeddings [𝒱][max_len][D_e], placeholder
 * offsets [C][𝒱][2][Ls][Hs][max_len][d] with 64 rows of padding between slots, prefix
 * offsets [C][𝒱][2][Ls][Hs][P_c][d], bf16; fp8 pools: blocked e4m3 codes + row scales) on
 * config->device (offset slabs in pinned host memory with placement HOST).  With
 * emb_shard_world G > 1 the embedding slab holds ceil(max_len / 2G) * 2 rows per slot.
 * OUT_OF_MEMORY if they do not fit. */
KVCOMM_API kvcomm_status kvcomm_anchor_pool_create(const kvcomm_pool_config* config,
                                                   kvcomm_pool_t* out);
KVCOMM_API kvcomm_status kvcomm_anchor_pool_destroy(kvcomm_pool_t pool);
/* Bytes of device memory the pool owns. */
KVCOMM_API kvcomm_status kvcomm_anchor_pool_bytes(kvcomm_pool_t pool, int64_t* bytes);

/* Insert a new anchor ψ ("the newly-generated cache becomes a new anchor"):
 * copies its embeddings emb (device bf16 [L_psi][D_e]) and the given/measured offsets
 * into a free slot.  If the pool is full, first evicts the anchor with the smallest
 * access count, ties to the earliest inserted (reading A17); the incoming
 * anchor is never its own victim.  *slot_out = slot used; *evicted_out = evicted
 * slot or -1.  L_psi in [1, max_anchor_len]. */
KVCOMM_API kvcomm_status kvcomm_anchor_pool_insert(kvcomm_pool_t pool, int32_t L_psi,
                                                   const void* emb,
                                                   const kvcomm_offset_desc* offs, int32_t n_offs,
                                                   void* stream, int32_t* slot_out,
                                                   int32_t* evicted_out);
/* Fill in (or replace) offsets of an existing anchor ("dependent agents fill in
 * deviations under their respective contexts"). */
KVCOMM_API kvcomm_status kvcomm_anchor_pool_set_offsets(kvcomm_pool_t pool, int32_t slot,
                                                        const kvcomm_offset_desc* offs,
                                                        int32_t n_offs, void* stream);
/* Drop an anchor (LFU pruning, happens inside insert when the pool is full;
 * this is the explicit form).  NOT_FOUND if the slot is empty. */
KVCOMM_API kvcomm_status kvcomm_anchor_pool_evict(kvcomm_pool_t pool, int32_t slot);
/* +1 access for each listed slot (reading A18: once per Shareable turn). */
KVCOMM_API kvcomm_status kvcomm_anchor_pool_record_access(kvcomm_pool_t pool,
                                                          const int32_t* slots, int32_t n);
/* Host metadata of one slot (occupancy, length, access count, insertion index,
 * per-consumer offset-presence masks). */
KVCOMM_API kvcomm_status kvcomm_anchor_pool_slot_info(kvcomm_pool_t pool, int32_t slot,
                                                      kvcomm_slot_info* info);
/* Device view of a stored offset (which: 0 placeholder, 1 prefix) of a bf16 pool:
 * *k, *v point at [Ls][Hs][*ld][d] bf16 rows of the slot (INVALID_ARGUMENT for fp8). */
KVCOMM_API kvcomm_status kvcomm_anchor_pool_offset_view(kvcomm_pool_t pool, int32_t slot,
                                                        int32_t consumer, int32_t which,
                                                        const void** k, const void** v,
                                                        int64_t* ld);

/* Copy a stored offset of (slot, consumer) out for inspection (which: 0 placeholder,
 * 1 prefix), first `rows` rows, stream-ordered: bf16 pools write bf16 [Ls][Hs][rows][d]
 * to k_out/v_out; fp8 pools write the e4m3 codes (uint8 [Ls][Hs][rows][d]) and the row
 * scales (fp32 [Ls][Hs][rows]) to sk_out/sv_out. */
KVCOMM_API kvcomm_status kvcomm_anchor_pool_read_offsets(kvcomm_pool_t pool, int32_t slot, int32_t consumer,
                                                         int32_t which, int32_t rows, void* k_out,
                                                         void* v_out, float* sk_out, float* sv_out,
                                                         void* stream);

/* ---- pool checkpoint (SURVEY §5 "optional pool dump/load"; SPEC S:293 dumps pools
 * for its CPU program) ---------------------------------------------------------------
 * save: synchronises `stream` (so inserts issued on it are included), then writes the
 * pool's configuration, LFU metadata (lengths, access counts, insertion indices and
 * counter, offset-presence masks) and every occupied slot's embeddings and present
 * offsets, exactly as stored (bf16 rows, or fp8 codes + row scales), to `path`.  The
 * caller orders any other stream's writes to the pool before the call.  Holds the
 * pool's reader lock.  IO: the file cannot be created or written. */
KVCOMM_API kvcomm_status kvcomm_anchor_pool_save(kvcomm_pool_t pool, const char* path, void* stream);
/* load: creates a pool on `device` with the saved configuration (layer/head shard,
 * capacity, formats, placement) and restores every slot bit for bit at its saved slot
 * index with its metadata, so later matches, realignments and LFU evictions behave
 * exactly as in the saved pool.  IO: missing, truncated, corrupt or wrong-version file;
 * OUT_OF_MEMORY / CUDA as for create.  Synchronous. */
KVCOMM_API kvcomm_status kvcomm_anchor_pool_load(const char* path, int32_t device, kvcomm_pool_t* out);
/* The pool's configuration; prefix_len (host int32 [num_consumers]) and inv_freq (host
 * double [head_dim/2]) are filled when non-NULL (config->prefix_len / inv_freq are set
 * to NULL). */
KVCOMM_API kvcomm_status kvcomm_anchor_pool_get_config(kvcomm_pool_t pool, kvcomm_pool_config* config,
                                                       int32_t* prefix_len, double* inv_freq);

/* ---- a1-a3: anchor matching (Eq. 5, Eq. 6 weights) -------------------------- */
/* query_emb: device bf16 [L_phi][D_e] (the sample's token embeddings h_φ).
 * consumer: candidates must hold that consumer's placeholder+prefix offsets;
 *   KVCOMM_ALL_CONSUMERS requires every consumer's (weights are then shared by all
 *   consumers of the sample, reading A21).
 * Computes, on the device, d[i,j] = ‖h_φ[i] - h_ψj[i]‖₂ (fp32 differences, fp64
 * accumulation), W[j][i] = softmax_j(-d[i,j]) (fp64, stored fp32), optional top-k
 * (distance asc, slot asc; KVCOMM_MAX_TOPK), d̄_j per config.scalar_distance, w̄ = softmax(-d̄),
 * H = -Σ w̄ log w̄ and the verdict.
 * Outputs (device): W [capacity][ld_w] fp32 (rows of non-candidate slots = 0),
 * idx [L_phi][top_k] int32 slot ids (may be NULL; ignored if top_k = 0),
 * wbar [capacity] fp32 (0 for non-candidates), dist (optional fp64 [capacity][ld_w]).
 * When the verdict is decided by the length clause / empty pool, no kernel runs and
 * the device outputs are left untouched. */
KVCOMM_API kvcomm_status kvcomm_match_anchors(kvcomm_pool_t pool, const void* query_emb,
                                              int32_t L_phi, int32_t consumer, float gamma,
                                              int32_t top_k, float* W, int64_t ld_w,
                                              int32_t* idx, float* wbar, double* dist,
                                              kvcomm_match_info* info, void* stream);

/* Several matches with ONE device synchronisation (e.g. every placeholder pool of a
 * request, Alg. 1 P:765 evaluates Eq. 5 for all placeholders before branching).
 * Each request has the arguments of kvcomm_match_anchors; every pool may appear at
 * most once per batch (its scratch is reused).  On error no info is valid. */
typedef struct {
  kvcomm_pool_t pool;
  const void* query_emb;
  int32_t L_phi;
  int32_t consumer;
  float gamma;
  int32_t top_k;
  float* W;
  int64_t ld_w;
  int32_t* idx;
  float* wbar;
  double* dist;
  kvcomm_match_info* info;   /* host, filled on return */
} kvcomm_match_request;

/* kvcomm_match_anchors for n requests in one batched launch (distances + weights,
 * chunk sums, finalize), then one host synchronisation to fill every info.  Each pool
 * may appear once per batch (its match scratch is per pool); all pools on one device. */
KVCOMM_API kvcomm_status kvcomm_match_anchors_batch(const kvcomm_match_request* reqs, int32_t n,
                                                    void* stream);

/* ---- a4-a5: fused blend + RoPE-δ + add ------------------------------------ */
/* One segment (Eq. 6 placeholder, Eq. 7 prefix, or a verbatim COPY) into its
 * destination rows, stream-ordered, no host synchronisation.  Validation errors
 * (SHAPE_MISMATCH, NO_CANDIDATES, MISSING_OFFSET, ...) return before any launch. */
KVCOMM_API kvcomm_status kvcomm_realign_segment(const kvcomm_realign_desc* seg, void* stream);
/* All segments of one request in ONE persistent kernel launch.  Segments may come
 * from different pools but must share (Ls, Hs, d) and device. */
KVCOMM_API kvcomm_status kvcomm_realign_segments(const kvcomm_realign_desc* segs, int32_t n,
                                                 void* stream);

/* ---- a6: concatenation + ledger ------------------------------------------- */
/* Checks that segs tile [0, N_total) in order (POSITION_GAP / POSITION_OVERLAP
 * otherwise, nothing launched) and copies the rows of segments with src.k != NULL
 * into dst [Ls][Hs][dst_ld][d] (dst_ld >= N_total) with the realign kernel's TMA ring
 * (one launch).  `device` = the CUDA device that runs the copy, normally dst's.
 * Across GPUs (Alg. 1 P:777's concatenation on the GPU that prefills the consumer, with
 * the request sharded by layer): dst may be the consumer's cache mapped into this
 * process with kvcomm_ipc_open, offset to this rank's layer block; `device` stays the
 * local device, the rows then leave with stores over NVLink and the launch ends with a
 * system-scope fence — the caller orders the consumer's reads after it (e.g. a
 * stream-ordered NCCL all-reduce of one word), as shard.PeerCaches does. */
KVCOMM_API kvcomm_status kvcomm_concat_prefill_cache(const kvcomm_segment_ref* segs, int32_t n,
                                                     int32_t N_total, int32_t Ls, int32_t Hs,
                                                     int32_t d, void* dst_k, void* dst_v,
                                                     int64_t dst_ld, int32_t device, void* stream);

/* ---- request plan: Algorithm 1's reuse branch as one native executor -------- */
/* A plan fixes, for a multi-agent prompt layout, which placeholder pools are matched
 * per request and which segments every agent realigns (Eq. 1: p_(m,0), φ_(m,1),
 * p_(m,1), ...).  kvcomm_plan_run then issues, stream-ordered and without host
 * synchronisation: the candidate filter (host), ONE batched match launch, and ONE
 * realign launch covering every agent's placeholder, prefix and COPY (p_(m,0))
 * segments.  The reuse/fallback branch of Alg. 1 is taken ON THE DEVICE:
 * an agent's segments run only if every pool it depends on was matched Shareable
 * (agents decided NewAnchor by the host-side length clause are skipped outright).
 * Their prompt caches are left untouched and reported as fallback (dense prefill,
 * P:784, is outside this library).  Every agent's segments must tile [0, N)
 * exactly (checked at create).  The plan owns its W / w̄ buffers and two work
 * tables, so one run may be in flight while the next is prepared. */
typedef struct kvcomm_plan_s* kvcomm_plan_t;

typedef struct {
  kvcomm_pool_t pool;      /* each pool at most once per plan                           */
  int32_t L_phi;           /* length of the sample matched against this pool per request */
  int32_t consumer;        /* KVCOMM_ALL_CONSUMERS (weights shared by all consumers)    */
  float gamma;             /* Eq. 5 threshold (paper default 0.3)                 */
  int32_t top_k;           /* 0 = all candidates (paper)                                 */
} kvcomm_plan_match;

typedef struct {
  int32_t agent;           /* index into the agents array                                */
  int32_t match;           /* pool (index into matches) the segment belongs to; ignored
                              for COPY                                                   */
  int32_t kind;            /* PLACEHOLDER (L_seg == L_phi) | PREFIX | COPY               */
  int32_t consumer;        /* consumer index of this (agent, slot) in the pool          */
  kvcomm_kv_view base;     /* device [Ls,Hs,ld,d]: base cache (COPY: rows to copy)       */
  int32_t L_seg;
  int32_t base_start;
  int32_t target_start;
  int32_t _pad;
} kvcomm_plan_segment;

typedef struct {
  int32_t N;               /* prompt length                                              */
  int32_t dst_heads;       /* heads per layer of the destination layout, 0 = the pools' Hs
                              (kvcomm_realign_desc.dst_heads: head shards of a full cache) */
  void* dst_k;             /* device bf16 [Ls,dst_heads,dst_ld,d] (this shard's block)   */
  void* dst_v;
  int64_t dst_ld;
} kvcomm_plan_agent;

/* Compile a request layout into a native executor: validates every segment and
 * checks each agent's ledger (segments tile [0, N) exactly) once; allocates the
 * plan's weight buffers and match scratch (owned by the plan, so plans over shared
 * pools may run concurrently on different streams).  Destinations may be peer-GPU
 * memory mapped with kvcomm_ipc_open (the fused gather). */
KVCOMM_API kvcomm_status kvcomm_plan_create(const kvcomm_plan_match* matches, int32_t n_matches,
                                            const kvcomm_plan_segment* segs, int32_t n_segs,
                                            const kvcomm_plan_agent* agents, int32_t n_agents,
                                            kvcomm_plan_t* out);
/* Waits for in-flight runs, frees the plan's buffers. */
KVCOMM_API kvcomm_status kvcomm_plan_destroy(kvcomm_plan_t plan);
/* query_embs: host array of n_matches device pointers (bf16 [L_phi][D_e]).  sync != 0
 * waits for the run to finish.  Pool metadata is read at call time. */
KVCOMM_API kvcomm_status kvcomm_plan_run(kvcomm_plan_t plan, const void* const* query_embs, int32_t sync,
                                         void* stream);
/* Waits for the last run and reports it: infos [n_matches], agent_reused [n_agents]
 * (1 = realigned, 0 = fallback).  Either may be NULL. */
KVCOMM_API kvcomm_status kvcomm_plan_results(kvcomm_plan_t plan, kvcomm_match_info* infos,
                                             int32_t* agent_reused);
/* Optional CUDA events (cudaEvent_t, created by the caller) recorded immediately before
 * and after the realign kernel (a4-a6; the prep kernel excluded) of every later run, on
 * the stream that runs it (the run's own, or the realign stream below); NULL disables.
 * Lets a caller time the realign kernel alone inside a pipelined run. */
KVCOMM_API kvcomm_status kvcomm_plan_set_events(kvcomm_plan_t plan, void* before_realign, void* after_realign);
/* Same for the distance kernel of Eq. 5/6 (a2, match_dist_kernel): events recorded right
 * before and after it in every later run (NULL disables), so a caller can time the
 * matching kernel alone (bench.py's roofline.match). */
KVCOMM_API kvcomm_status kvcomm_plan_set_match_events(kvcomm_plan_t plan, void* before_match, void* after_match);
/* Request pipelining (Algorithm 1's reuse branch, for consecutive requests;
 * "pipelining ... orthogonal"): with enable != 0, every later run launches its realign kernel on
 * `stream` (a cudaStream_t; NULL = the legacy default stream) instead of the run's own
 * stream.  The run's own stream keeps the table upload, matching, reduction, results copy
 * and the prep kernel, then records an event the realign stream waits on; the run's
 * completion (kvcomm_plan_results, the next-but-one run's buffer reuse) is ordered after
 * the realign.  A caller that issues run t+1 on the run stream while run t's realign
 * occupies the realign stream overlaps t+1's matching with t's realign — every kernel of
 * a run still sees exactly the same inputs (runs alternate between two table and weight
 * buffer sets; the run after next waits on the host for this run's completion).  enable = 0
 * restores single-stream runs.  INVALID_ARGUMENT between run_begin and run_end. */
KVCOMM_API kvcomm_status kvcomm_plan_set_realign_stream(kvcomm_plan_t plan, void* stream, int32_t enable);
/* Device pointers of the LAST run's weights for match `match` (W [capacity][ld_w], w̄;
 * runs alternate between two buffer sets). */
KVCOMM_API kvcomm_status kvcomm_plan_weights(kvcomm_plan_t plan, int32_t match, const float** W,
                                             int64_t* ld_w, const float** wbar);

/* ---- sharded matching across the ranks of a layer-sharded request -------
 * The weights of Eq. 5/6 depend only on the sample, so a plan replicated on
 * G ranks (same pools' slots and lengths, same matches, each rank its own layer block)
 * would compute the same distances G times.  After kvcomm_plan_match_shard, each rank
 * computes only the position blocks b = rank (mod G) of every job (2 positions per block;
 * a pool created with emb_shard_rank/world = rank/G needs only those embedding rows) and stores those
 * W columns into its own W and d̄ partial rows into its own buffers, AND both into every
 * peer's (NVLink stores into the peers' match buffers, mapped by CUDA IPC; W columns travel
 * position-major — one contiguous run of `capacity` weights per position, coalesced — into
 * an exchange area that run_end's first kernel copies into W); the fixed-order d̄ reduction, w̄, H and
 * the verdict then run on the complete arrays on every rank, so every rank's weights and
 * verdicts are bit-identical to an unsharded run.  A sharded run is split in two:
 *   kvcomm_plan_run_begin  (candidate filter, table upload, distance+weight kernel)
 *   -- caller: a stream-ordered cross-rank barrier, e.g. an NCCL all-reduce of one word --
 *   kvcomm_plan_run_end    (d̄ reduction + verdict, gated realign)
 * and kvcomm_plan_run refuses a sharded plan.  Every rank must call begin/end once per
 * request in lockstep (buffer parities alternate; kvcomm_plan_match_shard resets them).
 * The per-job tie_band_count then counts this rank's positions only.  Every rank also
 * publishes a fingerprint of its job layout (candidate slots, lengths, k, γ, modes) into
 * every rank's buffers; a job whose fingerprints differ across ranks is reported
 * NewAnchor with reason SHARD_MISMATCH (its agents are not realigned) and
 * kvcomm_plan_results returns SHAPE_MISMATCH — never silently blended weights. */
/* Export the plan's match buffers (W, w̄ and scratch of both parities, one allocation):
 * `bytes` (may be NULL) lets ranks check that their plans have the same layout. */
struct kvcomm_ipc_handle;  /* defined with the fused gather below */
KVCOMM_API kvcomm_status kvcomm_plan_match_handle(kvcomm_plan_t plan, struct kvcomm_ipc_handle* handle,
                                                  int64_t* bytes);
/* handles[world]: every rank's kvcomm_plan_match_handle (this rank's entry ignored).
 * Opens the peers' buffers (closing any earlier mapping, after in-flight runs finish).
 * world = 1 returns the plan to unsharded matching (handles may be NULL).
 * INVALID_ARGUMENT: world outside [1, 8], rank outside [0, world), a run begun; CUDA:
 * a handle cannot be opened (nothing stays mapped). */
KVCOMM_API kvcomm_status kvcomm_plan_match_shard(kvcomm_plan_t plan, int32_t rank, int32_t world,
                                                 const struct kvcomm_ipc_handle* handles);
/* The two halves of kvcomm_plan_run (same arguments); also usable unsharded.
 * INVALID_ARGUMENT: begin twice, or end without begin. */
KVCOMM_API kvcomm_status kvcomm_plan_run_begin(kvcomm_plan_t plan, const void* const* query_embs, void* stream);
KVCOMM_API kvcomm_status kvcomm_plan_run_end(kvcomm_plan_t plan, int32_t sync, void* stream);

/* ---- the fused gather (SURVEY §8(e) "fuse the gather into the realign epilogue with
 * NVLink P2P stores"; north star: realigned caches land on the GPU that prefills the
 * consuming agent) ------------------------------------------------------------------
 * With the path layer-sharded over G GPUs (one process each), the rank hosting agent m
 * allocates m's full-depth caches with kvcomm_ipc_alloc and shares the 64-byte handles
 * over any host channel; every other rank maps them with kvcomm_ipc_open and passes
 * (mapped pointer + its layer block's offset) as the destination of its segments.  The
 * library detects destinations that live on another GPU (cudaPointerGetAttributes) and
 * the realign kernel writes those rows with per-thread stores straight into the peer's
 * HBM over NVLink, then fences system-wide before it exits: there is no separate gather
 * pass.  The caller orders the consumer's reads after every writer's launch (e.g. a
 * stream-ordered all-reduce of one word).  Setting KVCOMM_STORE_STG=1 in the
 * environment forces the per-thread store path for every destination (tests). */
typedef struct kvcomm_ipc_handle {
  char bytes[64]; /* cudaIpcMemHandle_t */
} kvcomm_ipc_handle;

/* cudaMalloc `bytes` on `device` (owned by the caller until kvcomm_ipc_free) and export it. */
KVCOMM_API kvcomm_status kvcomm_ipc_alloc(int32_t device, int64_t bytes, void** ptr, kvcomm_ipc_handle* handle);
KVCOMM_API kvcomm_status kvcomm_ipc_free(void* ptr);
/* Map another process's allocation into this process (peer access enabled lazily);
 * *ptr is valid on `device` until kvcomm_ipc_close. */
KVCOMM_API kvcomm_status kvcomm_ipc_open(int32_t device, const kvcomm_ipc_handle* handle, void** ptr);
KVCOMM_API kvcomm_status kvcomm_ipc_close(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* KVCOMM_H */
