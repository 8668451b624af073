// C ABI of libkvcomm (include/kvcomm.h): anchor-pool store (host metadata + device
// slabs), argument validation, work-table construction and kernel launches.
// No exception crosses the ABI; every entry point returns a kvcomm_status.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <shared_mutex>
#include <string>
#include <vector>

#include "../../include/kvcomm.h"
#include "kvcomm_internal.h"

using namespace kvc;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
namespace {
thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

kvcomm_status fail(kvcomm_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

kvcomm_status ok() {
  g_err.clear();
  return KVCOMM_OK;
}

#define KV_CUDA(expr)                                                                          \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess) return fail(KVCOMM_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

#define KV_TRY(expr)                  \
  do {                                \
    kvcomm_status _s = (expr);        \
    if (_s != KVCOMM_OK) return _s;   \
  } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Makes `dev` current for the scope of a call and restores the caller's device.
// NVTX range per public call (header-only nvtx3: a no-op unless a profiler attaches)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

// ---------------------------------------------------------------------------
// pool
// ---------------------------------------------------------------------------
struct SlotMeta {
  bool occupied = false;
  int32_t length = 0;
  int64_t access = 0;
  int64_t inserted = 0;
  uint64_t ph_mask = 0, pf_mask = 0;
};

struct kvcomm_pool_s {
  kvcomm_pool_config cfg{};
  int Ls = 0, Hs = 0, d = 0, De = 0, cap = 0, maxlen = 0, C = 0;
  int ph_ld = 0;            // rows per (layer, head) block of a stored placeholder offset (>= maxlen)
  int64_t slot_pad = 0;     // extra elements between slots (breaks power-of-two strides)
  std::vector<int32_t> prefix_len;
  std::vector<double> inv_freq;
  // embedding sharding (config emb_shard_*): rows of position blocks b with b % emb_world ==
  // emb_rank only, block b stored at b / emb_world; emb_rows = stored rows per slot
  int emb_rank = 0, emb_world = 1;
  int64_t emb_rows = 0;
  int64_t emb_pad_rows = 0;  // rows of padding between embedding slots (KVCOMM_EMB_SLOT_PAD_ROWS)
  int64_t emb_slot() const { return (emb_rows + emb_pad_rows) * De; }  // elements between slots
  // device slabs
  bf16* emb = nullptr;                 // [cap][emb_rows][De]
  bool fp8 = false;                    // offset_format == KVCOMM_OFFSET_FP8_E4M3
  bf16* ph = nullptr;                  // [C][cap][2][Ls][Hs][ph_ld][d]  (bf16 pools)
  std::vector<bf16*> pf;               // per consumer: [cap][2][Ls][Hs][P_c][d]
  uint8_t* ph8 = nullptr;              // fp8 pools: blocked e4m3 codes + row scales
  std::vector<uint8_t*> pf8;           //   [C][cap][2][Ls][Hs][blocks][rpt*d codes | rpt fp32 scales]
  std::vector<void*> host_allocs;      // offset slabs placed in pinned host memory (f4)
  double* inv_freq_dev = nullptr;
  // match scratch
  double* d_partial = nullptr;         // [n_blocks_max][cap]
  int64_t bytes = 0;
  std::vector<SlotMeta> slots;
  int64_t next_index = 0;
  mutable std::shared_mutex mu;        // metadata: many readers / one writer
  std::mutex match_mu;                 // match scratch buffers

  int64_t ph_slot_stride() const { return int64_t(2) * Ls * Hs * ph_ld * d + slot_pad; }
  int64_t ph_plane_stride() const { return int64_t(Ls) * Hs * ph_ld * d; }
  bf16* ph_base(int c) const { return ph + int64_t(c) * cap * ph_slot_stride(); }
  int64_t pf_ld(int c) const { return prefix_len[c]; }
  // fp8 blocked geometry (bytes): a (layer, head) region holds ceil(ld / rpt) blocks
  int64_t f8_lh(int64_t ld) const {
    return (ld + fp8_rows_per_block(d) - 1) / fp8_rows_per_block(d) * fp8_block_bytes(d);
  }
  int64_t f8_ph_plane() const { return int64_t(Ls) * Hs * f8_lh(ph_ld); }
  int64_t f8_slot_pad = 0;  // fp8 pools: extra bytes between slots
  int64_t f8_ph_slot() const { return 2 * f8_ph_plane() + f8_slot_pad; }
  int64_t f8_pf_plane(int c) const { return int64_t(Ls) * Hs * f8_lh(prefix_len[c]); }
  int64_t f8_pf_slot(int c) const { return 2 * f8_pf_plane(c); }
  int64_t pf_slot_stride(int c) const { return int64_t(2) * Ls * Hs * pf_ld(c) * d; }
  // rows stored for an anchor of length L (all of them unless the embeddings are sharded)
  int64_t emb_row_count(int64_t L) const;
  int64_t pf_plane_stride(int c) const { return int64_t(Ls) * Hs * pf_ld(c) * d; }
};

#ifndef KVC_MATCH_P
#define KVC_MATCH_P 2
#endif
static constexpr int kMatchP = KVC_MATCH_P;  // positions per match work item

int64_t kvcomm_pool_s::emb_row_count(int64_t L) const {
  if (emb_world <= 1) return L;
  const int64_t cyc = int64_t(kMatchP) * emb_world, rem = L % cyc;
  return L / cyc * kMatchP + std::max<int64_t>(0, std::min<int64_t>(kMatchP, rem - int64_t(emb_rank) * kMatchP));
}

static void pool_free(kvcomm_pool_s* p) {
  if (!p) return;
  DeviceGuard g(p->cfg.device);
  auto release = [p](void* x) {
    if (!x) return;
    if (std::find(p->host_allocs.begin(), p->host_allocs.end(), x) != p->host_allocs.end()) cudaFreeHost(x);
    else cudaFree(x);
  };
  cudaFree(p->emb);
  release(p->ph);
  for (auto* x : p->pf) release(x);
  release(p->ph8);
  for (auto* x : p->pf8) release(x);
  cudaFree(p->inv_freq_dev);
  cudaFree(p->d_partial);
  delete p;
}

template <typename T>
static kvcomm_status dev_alloc(kvcomm_pool_s* p, T** out, int64_t count, const char* what, bool host = false) {
  const size_t bytes = size_t(std::max<int64_t>(count, 1)) * sizeof(T);
  // host placement (f4): pinned, mapped host memory; with UVA the pointer is valid on the device
  cudaError_t e = host ? cudaHostAlloc(reinterpret_cast<void**>(out), bytes, cudaHostAllocMapped)
                       : cudaMalloc(reinterpret_cast<void**>(out), bytes);
  if (e == cudaSuccess && host) p->host_allocs.push_back(*out);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    return fail(e == cudaErrorMemoryAllocation ? KVCOMM_ERR_OUT_OF_MEMORY : KVCOMM_ERR_CUDA,
                "allocating %s (%zu bytes): %s", what, bytes, cudaGetErrorString(e));
  }
  p->bytes += int64_t(bytes);
  return KVCOMM_OK;
}

extern "C" {

KVCOMM_API const char* kvcomm_status_string(kvcomm_status s) {
  switch (s) {
    case KVCOMM_OK: return "OK";
    case KVCOMM_ERR_INVALID_ARGUMENT: return "INVALID_ARGUMENT";
    case KVCOMM_ERR_SHAPE_MISMATCH: return "SHAPE_MISMATCH";
    case KVCOMM_ERR_NO_CANDIDATES: return "NO_CANDIDATES";
    case KVCOMM_ERR_MISSING_OFFSET: return "MISSING_OFFSET";
    case KVCOMM_ERR_POSITION_GAP: return "POSITION_GAP";
    case KVCOMM_ERR_POSITION_OVERLAP: return "POSITION_OVERLAP";
    case KVCOMM_ERR_NOT_FOUND: return "NOT_FOUND";
    case KVCOMM_ERR_OUT_OF_MEMORY: return "OUT_OF_MEMORY";
    case KVCOMM_ERR_CUDA: return "CUDA";
    case KVCOMM_ERR_NCCL: return "NCCL";
    case KVCOMM_ERR_IO: return "IO";
  }
  return "UNKNOWN";
}

KVCOMM_API const char* kvcomm_last_error_message(void) { return g_err.c_str(); }
KVCOMM_API int32_t kvcomm_version(void) { return KVCOMM_VERSION; }
KVCOMM_API int64_t kvcomm_kernel_launch_count(void) { return g_launches.load(); }

KVCOMM_API kvcomm_status kvcomm_anchor_pool_create(const kvcomm_pool_config* c, kvcomm_pool_t* out) {
  if (!c || !out) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null config/out");
  *out = nullptr;
  const int Ls = c->layer_end - c->layer_begin, Hs = c->head_end - c->head_begin;
  if (c->num_layers <= 0 || c->layer_begin < 0 || c->layer_end > c->num_layers || Ls <= 0)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "bad layer shard [%d,%d) of %d", c->layer_begin, c->layer_end,
                c->num_layers);
  if (c->num_kv_heads <= 0 || c->head_begin < 0 || c->head_end > c->num_kv_heads || Hs <= 0)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "bad head shard [%d,%d) of %d", c->head_begin, c->head_end,
                c->num_kv_heads);
  if (c->head_dim <= 0 || c->head_dim % 16 != 0 || c->head_dim > 256)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "head_dim %d must be a multiple of 16 in [16,256]", c->head_dim);
  if (c->emb_dim <= 0 || c->emb_dim % 8 != 0)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "emb_dim %d must be a positive multiple of 8", c->emb_dim);
  if (c->capacity < 1 || c->capacity > KVCOMM_MAX_CAPACITY)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "capacity %d outside [1,%d]", c->capacity, KVCOMM_MAX_CAPACITY);
  if (c->max_anchor_len < 1) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "max_anchor_len %d", c->max_anchor_len);
  if (c->num_consumers < 1 || c->num_consumers > KVCOMM_MAX_CONSUMERS)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "num_consumers %d outside [1,%d]", c->num_consumers,
                KVCOMM_MAX_CONSUMERS);
  if (!c->prefix_len || !c->inv_freq) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null prefix_len/inv_freq");
  if (c->scalar_distance != KVCOMM_SCALAR_FROBENIUS && c->scalar_distance != KVCOMM_SCALAR_MEAN_L2)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "scalar_distance %d", c->scalar_distance);
  if (c->similarity != KVCOMM_SIM_L2 && c->similarity != KVCOMM_SIM_COSINE)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "similarity %d", c->similarity);
  if (c->offset_format != KVCOMM_OFFSET_BF16 && c->offset_format != KVCOMM_OFFSET_FP8_E4M3)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "offset_format %d", c->offset_format);
  if (c->placement != KVCOMM_PLACE_DEVICE && c->placement != KVCOMM_PLACE_HOST)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "placement %d", c->placement);
  if (c->rope_layout != KVCOMM_ROPE_HALF && c->rope_layout != KVCOMM_ROPE_INTERLEAVED)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "rope_layout %d", c->rope_layout);
  if (c->offset_format == KVCOMM_OFFSET_FP8_E4M3 && c->head_dim < 64)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "fp8 offsets need head_dim >= 64 (got %d)", c->head_dim);
  for (int i = 0; i < c->num_consumers; ++i)
    if (c->prefix_len[i] < 0) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "prefix_len[%d] < 0", i);
  if (c->emb_shard_world > 1 &&
      (c->emb_shard_world > kMaxMatchPeers + 1 || c->emb_shard_rank < 0 || c->emb_shard_rank >= c->emb_shard_world))
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "emb_shard rank %d / world %d (world <= %d)", c->emb_shard_rank,
                c->emb_shard_world, kMaxMatchPeers + 1);
  if (c->emb_shard_world <= 1 && c->emb_shard_rank != 0)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "emb_shard_rank %d without emb_shard_world", c->emb_shard_rank);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || c->device < 0 || c->device >= ndev) {
    cudaGetLastError();
    return fail(KVCOMM_ERR_CUDA, "device %d not available (%d devices)", c->device, ndev);
  }
  DeviceGuard guard(c->device);
  if (!guard.ok) return fail(KVCOMM_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);

  auto* p = new kvcomm_pool_s();
  p->cfg = *c;
  p->Ls = Ls; p->Hs = Hs; p->d = c->head_dim; p->De = c->emb_dim; p->cap = c->capacity;
  p->maxlen = c->max_anchor_len; p->C = c->num_consumers;
  p->fp8 = c->offset_format == KVCOMM_OFFSET_FP8_E4M3;
  {
    // Tuning knobs: KVCOMM_PH_PAD_ROWS pads each (layer, head) block of a
    // stored offset, KVCOMM_SLOT_PAD_ROWS adds rows between anchor slots.
    const char* e1 = getenv("KVCOMM_PH_PAD_ROWS");
    const char* e2 = getenv("KVCOMM_SLOT_PAD_ROWS");
    p->ph_ld = p->maxlen + (e1 ? atoi(e1) : 0);
    // Default: 64 rows between consecutive slots of the placeholder slab (one fp8 block
    // for fp8 pools).  Without it, the tiles the ring keeps in flight (the same
    // (layer, head, tile) of consecutive anchors) sit a large power-of-two multiple
    // apart; measured (profiles/r01g_slot_pad.jsonl): config-4 realign 5.26 -> 5.08 ms,
    // config 2 4.68 -> 4.65 ms.
    const int pad_rows = e2 ? atoi(e2) : 64;
    p->slot_pad = int64_t(pad_rows) * p->d;
    const char* e3 = getenv("KVCOMM_F8_SLOT_PAD_BLOCKS");
    p->f8_slot_pad = int64_t(e3 ? atoi(e3) : 1) * fp8_block_bytes(p->d);

  }
  p->prefix_len.assign(c->prefix_len, c->prefix_len + c->num_consumers);
  p->inv_freq.assign(c->inv_freq, c->inv_freq + c->head_dim / 2);
  p->cfg.prefix_len = nullptr;
  p->cfg.inv_freq = nullptr;
  p->slots.resize(p->cap);
  kvcomm_status st;
#define ALLOC(ptr, n, what)                          \
  if ((st = dev_alloc(p, &(ptr), (n), what)) != KVCOMM_OK) { pool_free(p); return st; }
  const bool host = c->placement == KVCOMM_PLACE_HOST;
#define ALLOC_OFF(ptr, n, what)                      \
  if ((st = dev_alloc(p, &(ptr), (n), what, host)) != KVCOMM_OK) { pool_free(p); return st; }
  if (c->emb_shard_world > 1) {
    p->emb_rank = c->emb_shard_rank;
    p->emb_world = c->emb_shard_world;
  }
  {
    const int64_t cyc = int64_t(kMatchP) * p->emb_world;
    p->emb_rows = p->emb_world > 1 ? (p->maxlen + cyc - 1) / cyc * kMatchP : p->maxlen;
    const char* e = getenv("KVCOMM_EMB_SLOT_PAD_ROWS");
    p->emb_pad_rows = e ? atoi(e) : 0;
  }
  ALLOC(p->emb, int64_t(p->cap) * p->emb_slot(), "embedding slab");
  if (!p->fp8) {
    ALLOC_OFF(p->ph, int64_t(p->C) * p->cap * p->ph_slot_stride(), "placeholder offset slab");
    p->pf.assign(p->C, nullptr);
    for (int i = 0; i < p->C; ++i) ALLOC_OFF(p->pf[i], int64_t(p->cap) * p->pf_slot_stride(i), "prefix offset slab");
  } else {
    ALLOC_OFF(p->ph8, int64_t(p->C) * p->cap * p->f8_ph_slot(), "placeholder offset slab (e4m3)");
    p->pf8.assign(p->C, nullptr);
    for (int i = 0; i < p->C; ++i)
      ALLOC_OFF(p->pf8[i], int64_t(p->cap) * p->f8_pf_slot(i), "prefix offset slab (e4m3)");
    // blocks are read whole (tail rows past a segment's length included): keep them finite
    auto zero = [&](uint8_t* x, int64_t n) {
      if (host) std::memset(x, 0, size_t(n));
      else cudaMemset(x, 0, size_t(n));
    };
    zero(p->ph8, int64_t(p->C) * p->cap * p->f8_ph_slot());
    for (int i = 0; i < p->C; ++i) zero(p->pf8[i], int64_t(p->cap) * p->f8_pf_slot(i));
  }
  ALLOC(p->inv_freq_dev, p->d / 2, "inv_freq");
  // [position blocks][2cap+1] partial sums, then [kMatchChunks][2cap+1] chunk sums
  ALLOC(p->d_partial, (int64_t((p->maxlen + kMatchP - 1) / kMatchP) + kMatchChunks) * (2 * p->cap + 1),
        "partial sums");
#undef ALLOC
#undef ALLOC_OFF
  cudaError_t e = cudaMemcpy(p->inv_freq_dev, p->inv_freq.data(), sizeof(double) * (p->d / 2),
                             cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    pool_free(p);
    return fail(KVCOMM_ERR_CUDA, "inv_freq upload: %s", cudaGetErrorString(e));
  }
  *out = p;
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_anchor_pool_destroy(kvcomm_pool_t p) {
  if (!p) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null pool");
  {
    DeviceGuard g(p->cfg.device);
    cudaDeviceSynchronize();
  }
  pool_free(p);
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_anchor_pool_bytes(kvcomm_pool_t p, int64_t* bytes) {
  if (!p || !bytes) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null argument");
  *bytes = p->bytes;
  return ok();
}

// ---- offsets -----------------------------------------------------------------
static kvcomm_status check_view(const kvcomm_kv_view& v, int rows, const char* what) {
  if (!v.k || !v.v) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "%s: null k/v", what);
  if (!aligned16(v.k) || !aligned16(v.v)) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "%s: not 16-byte aligned", what);
  if (v.ld != 0 && v.ld < rows)
    return fail(KVCOMM_ERR_SHAPE_MISMATCH, "%s: ld %lld < rows %d", what, (long long)v.ld, rows);
  return KVCOMM_OK;
}

static int64_t ld_of(const kvcomm_kv_view& v, int rows) { return v.ld ? v.ld : rows; }

// Writes the offsets of one consumer into slot `slot` (caller holds the writer lock).
// Where the offsets of (slot, consumer) live: bf16 rows, or blocked e4m3 codes + row scales.
struct OffDst {
  bf16 *k = nullptr, *v = nullptr;       // bf16: [Ls][Hs][ld][d]
  uint8_t *k8 = nullptr, *v8 = nullptr;  // fp8: (layer, head) regions of lh_bytes
  int64_t ld = 0, lh_bytes = 0;
};

static OffDst offsets_of(const kvcomm_pool_s* p, int c, int slot, bool prefix) {
  OffDst o;
  o.ld = prefix ? p->pf_ld(c) : p->ph_ld;
  if (!p->fp8) {
    const int64_t e0 = prefix ? int64_t(slot) * p->pf_slot_stride(c)
                              : int64_t(c) * p->cap * p->ph_slot_stride() + int64_t(slot) * p->ph_slot_stride();
    const int64_t plane = prefix ? p->pf_plane_stride(c) : p->ph_plane_stride();
    bf16* b = prefix ? p->pf[c] : p->ph;
    o.k = b + e0;
    o.v = o.k + plane;
  } else {
    const int64_t b0 = prefix ? int64_t(slot) * p->f8_pf_slot(c)
                              : (int64_t(c) * p->cap + slot) * p->f8_ph_slot();
    const int64_t plane = prefix ? p->f8_pf_plane(c) : p->f8_ph_plane();
    uint8_t* b = prefix ? p->pf8[c] : p->ph8;
    o.k8 = b + b0;
    o.v8 = o.k8 + plane;
    o.lh_bytes = p->f8_lh(o.ld);
  }
  return o;
}

// Every copy (or quantisation) and measurement of one insert is collected and issued
// as one batched launch of each kind (flush_insert) instead of one launch per
// (consumer, kind, plane).
struct InsertJobs {
  std::vector<CopyJob> copies;
  std::vector<MeasureJob> measures;
};

static kvcomm_status flush_insert(kvcomm_pool_s* p, InsertJobs& jobs, cudaStream_t s) {
  for (size_t i = 0; i < jobs.copies.size(); i += kMaxCopyJobs) {
    CopyJobs b{};
    const int n = int(std::min<size_t>(kMaxCopyJobs, jobs.copies.size() - i));
    for (int k = 0; k < n; ++k) b.j[k] = jobs.copies[i + k];
    if (!p->fp8) KV_CUDA(launch_copy_rows_batch(b, n, p->Ls, p->Hs, p->d, s));
    else KV_CUDA(launch_quantize_rows_batch(b, n, p->Ls, p->Hs, p->d, s));
    g_launches += 1;
  }
  const int il = p->cfg.rope_layout == KVCOMM_ROPE_INTERLEAVED;
  for (size_t i = 0; i < jobs.measures.size(); i += kMaxMeasureJobs) {
    MeasureJobs b{};
    const int n = int(std::min<size_t>(kMaxMeasureJobs, jobs.measures.size() - i));
    for (int k = 0; k < n; ++k) b.j[k] = jobs.measures[i + k];
    if (!p->fp8) KV_CUDA(launch_measure_batch(b, n, p->Ls, p->Hs, p->d, il, p->inv_freq_dev, s));
    else KV_CUDA(launch_measure_fp8_batch(b, n, p->Ls, p->Hs, p->d, il, p->inv_freq_dev, s));
    g_launches += 1;
  }
  jobs.copies.clear();
  jobs.measures.clear();
  return KVCOMM_OK;
}

// Queue the copies (bf16) or quantisations (fp8) of GIVEN offsets.
static void queue_given(kvcomm_pool_s* p, const kvcomm_kv_view& src, int rows, const OffDst& d, InsertJobs& jobs) {
  const int64_t ld = ld_of(src, rows);
  const bf16* k = static_cast<const bf16*>(src.k);
  const bf16* v = static_cast<const bf16*>(src.v);
  if (!p->fp8) {
    jobs.copies.push_back({k, d.k, ld, d.ld, rows, 0});
    jobs.copies.push_back({v, d.v, ld, d.ld, rows, 0});
  } else {
    jobs.copies.push_back({k, d.k8, ld, d.lh_bytes, rows, 0});
    jobs.copies.push_back({v, d.v8, ld, d.lh_bytes, rows, 0});
  }
}

// Queue a device measurement ΔK = R_{-(s_real - s_base)} K_real - K_base, ΔV = V_real - V_base.
static void queue_measured(kvcomm_pool_s* p, const kvcomm_kv_view& real, const kvcomm_kv_view& base, int rows,
                           const OffDst& d, InsertJobs& jobs) {
  const int delta = -(real.start - base.start);
  const auto* kr = static_cast<const bf16*>(real.k);
  const auto* vr = static_cast<const bf16*>(real.v);
  const auto* kb = static_cast<const bf16*>(base.k);
  const auto* vb = static_cast<const bf16*>(base.v);
  if (!p->fp8)
    jobs.measures.push_back({kr, vr, kb, vb, d.k, d.v, ld_of(real, rows), ld_of(base, rows), d.ld, rows, delta});
  else
    jobs.measures.push_back({kr, vr, kb, vb, d.k8, d.v8, ld_of(real, rows), ld_of(base, rows), d.lh_bytes, rows,
                             delta});
}

static kvcomm_status write_offsets(kvcomm_pool_s* p, int slot, int L_psi, const kvcomm_offset_desc& o,
                                   uint64_t* ph_set, uint64_t* pf_set, InsertJobs& jobs) {
  const int c = o.consumer;
  if (c < 0 || c >= p->C) return fail(KVCOMM_ERR_NOT_FOUND, "consumer %d outside [0,%d)", c, p->C);
  const int P = p->prefix_len[c];
  const OffDst ph = offsets_of(p, c, slot, false), pf = offsets_of(p, c, slot, true);
  if (P == 0) *pf_set |= 1ull << c;  // an empty prefix segment needs no offsets
  if (o.mode == KVCOMM_OFFSET_GIVEN) {
    if (o.ph_delta.k) {
      KV_TRY(check_view(o.ph_delta, L_psi, "ph_delta"));
      queue_given(p, o.ph_delta, L_psi, ph, jobs);
      *ph_set |= 1ull << c;
    }
    if (o.pf_delta.k) {
      KV_TRY(check_view(o.pf_delta, P, "pf_delta"));
      queue_given(p, o.pf_delta, P, pf, jobs);
      *pf_set |= 1ull << c;
    }
  } else if (o.mode == KVCOMM_OFFSET_MEASURE) {
    if (o.ph_real.k) {
      KV_TRY(check_view(o.ph_real, L_psi, "ph_real"));
      KV_TRY(check_view(o.ph_base, L_psi, "ph_base"));
      queue_measured(p, o.ph_real, o.ph_base, L_psi, ph, jobs);
      *ph_set |= 1ull << c;
    }
    if (o.pf_real.k) {
      KV_TRY(check_view(o.pf_real, P, "pf_real"));
      KV_TRY(check_view(o.pf_base, P, "pf_base"));
      queue_measured(p, o.pf_real, o.pf_base, P, pf, jobs);
      *pf_set |= 1ull << c;
    }
  } else {
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "offset mode %d", o.mode);
  }
  return KVCOMM_OK;
}

static int lfu_victim(const kvcomm_pool_s* p) {
  int best = -1;
  for (int s = 0; s < p->cap; ++s) {
    const SlotMeta& m = p->slots[s];
    if (!m.occupied) continue;
    if (best < 0 || m.access < p->slots[best].access ||
        (m.access == p->slots[best].access && m.inserted < p->slots[best].inserted))
      best = s;
  }
  return best;
}

KVCOMM_API kvcomm_status kvcomm_anchor_pool_insert(kvcomm_pool_t p, int32_t L_psi, const void* emb,
                                                   const kvcomm_offset_desc* offs, int32_t n_offs, void* stream,
                                                   int32_t* slot_out, int32_t* evicted_out) {
  NvtxRange nvtx_("kvcomm_anchor_pool_insert");
  if (!p || !emb || (n_offs > 0 && !offs)) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null argument");
  if (L_psi < 1 || L_psi > p->maxlen)
    return fail(KVCOMM_ERR_SHAPE_MISMATCH, "L_psi %d outside [1,%d]", L_psi, p->maxlen);
  if (!aligned16(emb)) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "emb not 16-byte aligned");
  DeviceGuard guard(p->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::unique_lock<std::shared_mutex> lk(p->mu);
  int evicted = -1;
  int slot = -1;
  for (int i = 0; i < p->cap; ++i)
    if (!p->slots[i].occupied) { slot = i; break; }
  if (slot < 0) {
    evicted = lfu_victim(p);
    p->slots[evicted] = SlotMeta();
    slot = evicted;
  }
  bf16* edst = p->emb + int64_t(slot) * p->emb_slot();
  if (p->emb_world <= 1) {
    KV_CUDA(launch_copy_flat(static_cast<const bf16*>(emb), edst, int64_t(L_psi) * p->De, s));
    g_launches += 1;
  } else {  // this rank's position blocks only: block b = rank + k * world -> stored block k
    const int64_t P = kMatchP, G = p->emb_world, row = int64_t(p->De) * sizeof(bf16);
    const int64_t stored = p->emb_row_count(L_psi), full = stored / P, tail = stored - full * P;
    const uint8_t* src = static_cast<const uint8_t*>(emb) + int64_t(p->emb_rank) * P * row;
    if (full > 0)
      KV_CUDA(cudaMemcpy2DAsync(edst, size_t(P * row), src, size_t(G * P * row), size_t(P * row), size_t(full),
                                cudaMemcpyDeviceToDevice, s));
    if (tail > 0)
      KV_CUDA(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(edst) + full * P * row, src + full * G * P * row,
                              size_t(tail * row), cudaMemcpyDeviceToDevice, s));
  }
  uint64_t phm = 0, pfm = 0;
  InsertJobs jobs;
  for (int i = 0; i < n_offs; ++i) {
    kvcomm_status st = write_offsets(p, slot, L_psi, offs[i], &phm, &pfm, jobs);
    if (st != KVCOMM_OK) {
      if (evicted < 0) p->slots[slot] = SlotMeta();  // leave the pool as it was (minus the victim)
      return st;
    }
  }
  KV_TRY(flush_insert(p, jobs, s));
  SlotMeta& m = p->slots[slot];
  m.occupied = true;
  m.length = L_psi;
  m.access = 0;
  m.inserted = p->next_index++;
  m.ph_mask = phm;
  m.pf_mask = pfm;
  if (slot_out) *slot_out = slot;
  if (evicted_out) *evicted_out = evicted;
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_anchor_pool_set_offsets(kvcomm_pool_t p, int32_t slot,
                                                        const kvcomm_offset_desc* offs, int32_t n_offs,
                                                        void* stream) {
  if (!p || (n_offs > 0 && !offs)) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null argument");
  std::unique_lock<std::shared_mutex> lk(p->mu);
  if (slot < 0 || slot >= p->cap || !p->slots[slot].occupied)
    return fail(KVCOMM_ERR_NOT_FOUND, "slot %d is empty", slot);
  DeviceGuard guard(p->cfg.device);
  SlotMeta& m = p->slots[slot];
  InsertJobs jobs;
  uint64_t phm = m.ph_mask, pfm = m.pf_mask;  // published only once every job is issued
  for (int i = 0; i < n_offs; ++i)
    KV_TRY(write_offsets(p, slot, m.length, offs[i], &phm, &pfm, jobs));
  KV_TRY(flush_insert(p, jobs, static_cast<cudaStream_t>(stream)));
  m.ph_mask = phm;
  m.pf_mask = pfm;
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_anchor_pool_evict(kvcomm_pool_t p, int32_t slot) {
  if (!p) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null pool");
  std::unique_lock<std::shared_mutex> lk(p->mu);
  if (slot < 0 || slot >= p->cap || !p->slots[slot].occupied)
    return fail(KVCOMM_ERR_NOT_FOUND, "slot %d is empty", slot);
  p->slots[slot] = SlotMeta();
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_anchor_pool_record_access(kvcomm_pool_t p, const int32_t* slots, int32_t n) {
  if (!p || (n > 0 && !slots)) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null argument");
  std::unique_lock<std::shared_mutex> lk(p->mu);
  for (int i = 0; i < n; ++i)
    if (slots[i] < 0 || slots[i] >= p->cap || !p->slots[slots[i]].occupied)
      return fail(KVCOMM_ERR_NOT_FOUND, "slot %d is empty", slots[i]);
  for (int i = 0; i < n; ++i) p->slots[slots[i]].access += 1;
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_anchor_pool_slot_info(kvcomm_pool_t p, int32_t slot, kvcomm_slot_info* info) {
  if (!p || !info) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null argument");
  if (slot < 0 || slot >= p->cap) return fail(KVCOMM_ERR_NOT_FOUND, "slot %d outside [0,%d)", slot, p->cap);
  std::shared_lock<std::shared_mutex> lk(p->mu);
  const SlotMeta& m = p->slots[slot];
  info->occupied = m.occupied;
  info->length = m.length;
  info->access_count = m.access;
  info->insertion_index = m.inserted;
  info->ph_present_mask = m.ph_mask;
  info->pf_present_mask = m.pf_mask;
  return ok();
}

// ---- pool checkpoint (SURVEY §5 "pool dump/load"): host file IO ------------------
// File layout (native endianness): "KVCPOOL1", u32 version, the config's integer fields,
// prefix_len[C], inv_freq[d/2], next insertion index, per-slot metadata, then for every
// occupied slot: its L_ψ embedding rows (bf16 [L_ψ][D_e]) and, per consumer whose bit
// is set, the placeholder region (bf16: rows [0, L_ψ) of every (plane, layer, head)
// block; fp8: the blocks holding those rows, codes + scales as stored) and the prefix
// region (whole).  Rows are written in a dense canonical layout, so a checkpoint loads
// into a pool whose row padding (KVCOMM_PH_PAD_ROWS / KVCOMM_SLOT_PAD_ROWS) differs.
namespace {
constexpr char kCkptMagic[8] = {'K', 'V', 'C', 'P', 'O', 'O', 'L', '1'};
constexpr uint32_t kCkptVersion = 2;  // 2: + embedding shard (rank, world)

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

kvcomm_status fwrite_all(FILE* f, const void* p, size_t n, const char* what) {
  if (n && fwrite(p, 1, n, f) != n) return fail(KVCOMM_ERR_IO, "writing %s", what);
  return KVCOMM_OK;
}
kvcomm_status fread_all(FILE* f, void* p, size_t n, const char* what) {
  if (n && fread(p, 1, n, f) != n) return fail(KVCOMM_ERR_IO, "reading %s: truncated or not a pool checkpoint", what);
  return KVCOMM_OK;
}

// One region of a slot as `rows` strided blocks of `width` bytes (dense in the file).
struct Region {
  void* base;
  size_t width, pitch, rows;
};

// Regions of (slot, consumer, prefix?) holding rows [0, len).
Region offset_region(const kvcomm_pool_s* p, int c, int slot, bool prefix, int len) {
  const OffDst o = offsets_of(p, c, slot, prefix);
  const size_t blocks = size_t(2) * p->Ls * p->Hs;  // K plane then V plane: uniformly spaced
  if (!p->fp8) {
    return {o.k, size_t(len) * p->d * sizeof(bf16), size_t(o.ld) * p->d * sizeof(bf16), blocks};
  }
  const int rpb = fp8_rows_per_block(p->d);
  return {o.k8, size_t((len + rpb - 1) / rpb) * fp8_block_bytes(p->d), size_t(o.lh_bytes), blocks};
}

kvcomm_status region_io(const Region& r, std::vector<uint8_t>& buf, bool save, FILE* f) {
  const size_t n = r.width * r.rows;
  if (n == 0) return KVCOMM_OK;
  buf.resize(n);
  if (save) {
    KV_CUDA(cudaMemcpy2D(buf.data(), r.width, r.base, r.pitch, r.width, r.rows, cudaMemcpyDefault));
    return fwrite_all(f, buf.data(), n, "offset region");
  }
  KV_TRY(fread_all(f, buf.data(), n, "offset region"));
  KV_CUDA(cudaMemcpy2D(r.base, r.pitch, buf.data(), r.width, r.width, r.rows, cudaMemcpyDefault));
  return KVCOMM_OK;
}

int32_t* cfg_ints(kvcomm_pool_config& c, int i) {
  int32_t* f[] = {&c.num_layers, &c.layer_begin, &c.layer_end, &c.num_kv_heads, &c.head_begin, &c.head_end,
                  &c.head_dim, &c.emb_dim, &c.capacity, &c.max_anchor_len, &c.num_consumers, &c.scalar_distance,
                  &c.similarity, &c.offset_format, &c.placement, &c.rope_layout};
  return i < int(sizeof(f) / sizeof(f[0])) ? f[i] : nullptr;
}
constexpr int kCfgInts = 16;

// the slot data of one pool, saved or loaded in file order
kvcomm_status slots_io(kvcomm_pool_s* p, bool save, FILE* f) {
  std::vector<uint8_t> buf;
  for (int s = 0; s < p->cap; ++s) {
    const SlotMeta& m = p->slots[s];
    if (!m.occupied) continue;
    const size_t ew = size_t(p->emb_row_count(m.length)) * p->De * sizeof(bf16);  // rows as stored
    const Region er{p->emb + int64_t(s) * p->emb_slot(), ew, ew, 1};
    KV_TRY(region_io(er, buf, save, f));
    for (int c = 0; c < p->C; ++c) {
      if (m.ph_mask >> c & 1) KV_TRY(region_io(offset_region(p, c, s, false, m.length), buf, save, f));
      if (m.pf_mask >> c & 1) KV_TRY(region_io(offset_region(p, c, s, true, p->prefix_len[c]), buf, save, f));
    }
  }
  return KVCOMM_OK;
}
}  // namespace

KVCOMM_API kvcomm_status kvcomm_anchor_pool_save(kvcomm_pool_t p, const char* path, void* stream) {
  NvtxRange nvtx_("kvcomm_anchor_pool_save");
  if (!p || !path) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null pool/path");
  std::shared_lock<std::shared_mutex> lk(p->mu);
  DeviceGuard guard(p->cfg.device);
  KV_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));  // prior inserts on `stream` land first
  // ... and those issued on any other stream of the pool's device (a checkpoint must never
  // capture half-written embedding or offset rows)
  KV_CUDA(cudaDeviceSynchronize());
  File F;
  F.f = fopen(path, "wb");
  if (!F.f) return fail(KVCOMM_ERR_IO, "cannot create %s", path);
  kvcomm_pool_config c = p->cfg;
  KV_TRY(fwrite_all(F.f, kCkptMagic, sizeof(kCkptMagic), "magic"));
  KV_TRY(fwrite_all(F.f, &kCkptVersion, sizeof(kCkptVersion), "version"));
  for (int i = 0; i < kCfgInts; ++i) KV_TRY(fwrite_all(F.f, cfg_ints(c, i), sizeof(int32_t), "config"));
  const int32_t es[2] = {c.emb_shard_rank, c.emb_shard_world};
  KV_TRY(fwrite_all(F.f, es, sizeof(es), "config"));
  KV_TRY(fwrite_all(F.f, p->prefix_len.data(), sizeof(int32_t) * p->C, "prefix_len"));
  KV_TRY(fwrite_all(F.f, p->inv_freq.data(), sizeof(double) * (p->d / 2), "inv_freq"));
  KV_TRY(fwrite_all(F.f, &p->next_index, sizeof(int64_t), "insertion counter"));
  for (const SlotMeta& m : p->slots) {
    const int32_t occ = m.occupied ? 1 : 0;
    KV_TRY(fwrite_all(F.f, &occ, sizeof(occ), "slot"));
    KV_TRY(fwrite_all(F.f, &m.length, sizeof(m.length), "slot"));
    KV_TRY(fwrite_all(F.f, &m.access, sizeof(m.access), "slot"));
    KV_TRY(fwrite_all(F.f, &m.inserted, sizeof(m.inserted), "slot"));
    KV_TRY(fwrite_all(F.f, &m.ph_mask, sizeof(m.ph_mask), "slot"));
    KV_TRY(fwrite_all(F.f, &m.pf_mask, sizeof(m.pf_mask), "slot"));
  }
  KV_TRY(slots_io(p, true, F.f));
  if (fflush(F.f) != 0) return fail(KVCOMM_ERR_IO, "flushing %s", path);
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_anchor_pool_load(const char* path, int32_t device, kvcomm_pool_t* out) {
  NvtxRange nvtx_("kvcomm_anchor_pool_load");
  if (!path || !out) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null path/out");
  *out = nullptr;
  File F;
  F.f = fopen(path, "rb");
  if (!F.f) return fail(KVCOMM_ERR_IO, "cannot open %s", path);
  char magic[8];
  uint32_t ver = 0;
  KV_TRY(fread_all(F.f, magic, sizeof(magic), "magic"));
  if (std::memcmp(magic, kCkptMagic, sizeof(magic)) != 0) return fail(KVCOMM_ERR_IO, "%s: not a pool checkpoint", path);
  KV_TRY(fread_all(F.f, &ver, sizeof(ver), "version"));
  if (ver != kCkptVersion) return fail(KVCOMM_ERR_IO, "%s: checkpoint version %u (expected %u)", path, ver, kCkptVersion);
  kvcomm_pool_config c{};
  for (int i = 0; i < kCfgInts; ++i) KV_TRY(fread_all(F.f, cfg_ints(c, i), sizeof(int32_t), "config"));
  int32_t es[2];
  KV_TRY(fread_all(F.f, es, sizeof(es), "config"));
  c.emb_shard_rank = int16_t(es[0]);
  c.emb_shard_world = int16_t(es[1]);
  if (c.num_consumers < 1 || c.num_consumers > KVCOMM_MAX_CONSUMERS || c.head_dim < 2 || c.head_dim > 256 ||
      c.capacity < 1 || c.capacity > KVCOMM_MAX_CAPACITY)
    return fail(KVCOMM_ERR_IO, "%s: corrupt configuration", path);
  std::vector<int32_t> plen(c.num_consumers);
  std::vector<double> inv(c.head_dim / 2);
  KV_TRY(fread_all(F.f, plen.data(), sizeof(int32_t) * plen.size(), "prefix_len"));
  KV_TRY(fread_all(F.f, inv.data(), sizeof(double) * inv.size(), "inv_freq"));
  c.device = device;
  c.prefix_len = plen.data();
  c.inv_freq = inv.data();
  kvcomm_pool_t p = nullptr;
  KV_TRY(kvcomm_anchor_pool_create(&c, &p));
  auto bail = [&](kvcomm_status st) {
    const std::string msg = g_err;
    pool_free(p);
    g_err = msg;
    return st;
  };
  kvcomm_status st;
  if ((st = fread_all(F.f, &p->next_index, sizeof(int64_t), "insertion counter")) != KVCOMM_OK) return bail(st);
  for (SlotMeta& m : p->slots) {
    int32_t occ = 0;
    if ((st = fread_all(F.f, &occ, sizeof(occ), "slot")) != KVCOMM_OK ||
        (st = fread_all(F.f, &m.length, sizeof(m.length), "slot")) != KVCOMM_OK ||
        (st = fread_all(F.f, &m.access, sizeof(m.access), "slot")) != KVCOMM_OK ||
        (st = fread_all(F.f, &m.inserted, sizeof(m.inserted), "slot")) != KVCOMM_OK ||
        (st = fread_all(F.f, &m.ph_mask, sizeof(m.ph_mask), "slot")) != KVCOMM_OK ||
        (st = fread_all(F.f, &m.pf_mask, sizeof(m.pf_mask), "slot")) != KVCOMM_OK)
      return bail(st);
    m.occupied = occ != 0;
    if (m.occupied && (m.length < 1 || m.length > p->maxlen)) return bail(fail(KVCOMM_ERR_IO, "%s: corrupt slot", path));
  }
  {  // the LFU metadata must describe a pool this library could have produced (reading A17's
     // tie-break runs on insertion indices): unique indices below the counter, masks < 2^C
    const uint64_t cmask = p->C >= 64 ? ~0ull : (1ull << p->C) - 1;
    std::vector<int64_t> seen;
    for (const SlotMeta& m : p->slots) {
      if (!m.occupied) continue;
      if (m.inserted < 0 || m.inserted >= p->next_index || m.access < 0 || (m.ph_mask & ~cmask) ||
          (m.pf_mask & ~cmask))
        return bail(fail(KVCOMM_ERR_IO, "%s: corrupt slot metadata", path));
      seen.push_back(m.inserted);
    }
    std::sort(seen.begin(), seen.end());
    if (std::adjacent_find(seen.begin(), seen.end()) != seen.end())
      return bail(fail(KVCOMM_ERR_IO, "%s: two slots share an insertion index", path));
  }
  {
    DeviceGuard guard(device);
    if ((st = slots_io(p, false, F.f)) != KVCOMM_OK) return bail(st);
  }
  char extra;
  if (fread(&extra, 1, 1, F.f) != 0) return bail(fail(KVCOMM_ERR_IO, "%s: trailing bytes", path));
  *out = p;
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_anchor_pool_get_config(kvcomm_pool_t p, kvcomm_pool_config* config,
                                                       int32_t* prefix_len, double* inv_freq) {
  if (!p || !config) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null pool/config");
  *config = p->cfg;
  config->prefix_len = nullptr;
  config->inv_freq = nullptr;
  if (prefix_len) std::memcpy(prefix_len, p->prefix_len.data(), sizeof(int32_t) * p->C);
  if (inv_freq) std::memcpy(inv_freq, p->inv_freq.data(), sizeof(double) * (p->d / 2));
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_anchor_pool_offset_view(kvcomm_pool_t p, int32_t slot, int32_t consumer,
                                                        int32_t which, const void** k, const void** v,
                                                        int64_t* ld) {
  if (!p || !k || !v || !ld) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null argument");
  if (p->fp8) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "fp8 pools store blocked codes: use read_offsets");
  if (slot < 0 || slot >= p->cap) return fail(KVCOMM_ERR_NOT_FOUND, "slot %d", slot);
  if (consumer < 0 || consumer >= p->C) return fail(KVCOMM_ERR_NOT_FOUND, "consumer %d", consumer);
  const OffDst o = offsets_of(p, consumer, slot, which != 0);
  *k = o.k;
  *v = o.v;
  *ld = o.ld;
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_anchor_pool_read_offsets(kvcomm_pool_t p, int32_t slot, int32_t consumer,
                                                         int32_t which, int32_t rows, void* k_out, void* v_out,
                                                         float* sk_out, float* sv_out, void* stream) {
  if (!p || !k_out || !v_out) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null argument");
  if (p->fp8 && (!sk_out || !sv_out)) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "fp8 pools need scale outputs");
  if (slot < 0 || slot >= p->cap) return fail(KVCOMM_ERR_NOT_FOUND, "slot %d", slot);
  if (consumer < 0 || consumer >= p->C) return fail(KVCOMM_ERR_NOT_FOUND, "consumer %d", consumer);
  const OffDst o = offsets_of(p, consumer, slot, which != 0);
  if (rows < 0 || rows > o.ld) return fail(KVCOMM_ERR_SHAPE_MISMATCH, "rows %d outside [0,%lld]", rows,
                                           (long long)o.ld);
  DeviceGuard guard(p->cfg.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::shared_lock<std::shared_mutex> lk(p->mu);
  if (!p->fp8) {
    KV_CUDA(launch_copy_rows(o.k, o.ld, static_cast<bf16*>(k_out), rows, p->Ls, p->Hs, rows, p->d, s));
    KV_CUDA(launch_copy_rows(o.v, o.ld, static_cast<bf16*>(v_out), rows, p->Ls, p->Hs, rows, p->d, s));
  } else {
    KV_CUDA(launch_read_fp8(o.k8, o.lh_bytes, static_cast<uint8_t*>(k_out), sk_out, p->Ls, p->Hs, rows, p->d, s));
    KV_CUDA(launch_read_fp8(o.v8, o.lh_bytes, static_cast<uint8_t*>(v_out), sv_out, p->Ls, p->Hs, rows, p->d, s));
  }
  g_launches += 2;
  return ok();
}

// ---- work tables (match and realign) -------------------------------------------
namespace {

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// A pair of (pinned host, device) buffers holding one launch's work table; reusing
// it waits on the event recorded after the kernels that consumed it.
struct RingEntry {
  void* host = nullptr;
  void* dev = nullptr;
  size_t cap = 0;
  cudaEvent_t done = nullptr;
  bool used = false;
};

kvcomm_status entry_reserve(RingEntry& E, size_t bytes) {
  if (E.used) KV_CUDA(cudaEventSynchronize(E.done));
  E.used = false;
  if (!E.done) KV_CUDA(cudaEventCreateWithFlags(&E.done, cudaEventDisableTiming));
  if (E.cap < bytes) {
    if (E.host) cudaFreeHost(E.host);
    if (E.dev) cudaFree(E.dev);
    E.host = E.dev = nullptr;
    E.cap = 0;
    const size_t cap = std::max<size_t>(align_up(bytes, 1 << 16), 1 << 16);
    if (cudaMallocHost(&E.host, cap) != cudaSuccess || cudaMalloc(&E.dev, cap) != cudaSuccess) {
      cudaGetLastError();
      return fail(KVCOMM_ERR_OUT_OF_MEMORY, "work table (%zu bytes)", cap);
    }
    E.cap = cap;
  }
  return KVCOMM_OK;
}

void entry_free(RingEntry& E) {
  if (E.used && E.done) cudaEventSynchronize(E.done);
  if (E.host) cudaFreeHost(E.host);
  if (E.dev) cudaFree(E.dev);
  if (E.done) cudaEventDestroy(E.done);
  E = RingEntry();
}

struct TableRing {
  static constexpr int kN = 8;
  RingEntry e[kN];
  int next = 0;
  std::mutex mu;
};
TableRing g_rings[64];

std::vector<kvcomm_pool_s*> distinct(std::vector<kvcomm_pool_s*> pools) {
  std::sort(pools.begin(), pools.end());
  pools.erase(std::unique(pools.begin(), pools.end()), pools.end());
  return pools;
}

void lock_readers(const std::vector<kvcomm_pool_s*>& pools, std::vector<std::shared_lock<std::shared_mutex>>& l) {
  for (kvcomm_pool_s* p : distinct(pools)) l.emplace_back(p->mu);
}

void lock_match_scratch(const std::vector<kvcomm_pool_s*>& pools, std::vector<std::unique_lock<std::mutex>>& l) {
  for (kvcomm_pool_s* p : distinct(pools)) l.emplace_back(p->match_mu);
}

// ---- a1: candidate filter + length clause (host, integer metadata) ----------
// Fills info->{candidates, n_candidates, verdict, reason}; returns true when the
// verdict still needs the device (entropy clause).
bool candidate_filter(const kvcomm_pool_s* p, int L_phi, int consumer, kvcomm_match_info* info) {
  std::memset(info, 0, sizeof(*info));
  int32_t maxL = 0, n_occ = 0, n_cand = 0;
  const uint64_t need = consumer == KVCOMM_ALL_CONSUMERS ? (p->C >= 64 ? ~0ull : ((1ull << p->C) - 1))
                                                         : (1ull << consumer);
  for (int s = 0; s < p->cap; ++s) {
    const SlotMeta& m = p->slots[s];
    if (!m.occupied) continue;
    ++n_occ;
    maxL = std::max(maxL, m.length);
    if (m.length >= L_phi && (m.ph_mask & need) == need && (m.pf_mask & need) == need)
      info->candidates[n_cand++] = s;
  }
  info->n_candidates = n_cand;
  info->verdict = KVCOMM_NEW_ANCHOR;
  if (n_occ == 0) { info->reason = KVCOMM_REASON_EMPTY_POOL; return false; }
  if (L_phi > maxL) { info->reason = KVCOMM_REASON_TOO_LONG; return false; }
  if (n_cand == 0) { info->reason = KVCOMM_REASON_NO_CANDIDATES; return false; }
  info->reason = KVCOMM_REASON_OK;
  return true;
}

void fill_info_from_result(kvcomm_match_info* info, const MatchResultDev& r) {
  info->entropy = r.entropy;
  info->threshold = r.threshold;
  info->verdict = r.verdict ? KVCOMM_NEW_ANCHOR : KVCOMM_SHAREABLE;
  info->reason = r.shard_mismatch ? KVCOMM_REASON_SHARD_MISMATCH
                 : r.verdict      ? KVCOMM_REASON_HIGH_ENTROPY
                                  : KVCOMM_REASON_OK;
  info->verdict_in_tie_band = r.tie_flag;
  info->tie_band_count = r.tie_count;
}

// ---- match work table ---------------------------------------------------------
struct MatchItem {
  kvcomm_pool_s* p;
  const void* query;
  int L_phi;
  float gamma;
  int top_k;  // effective k, 0 = dense
  float* W;
  int64_t ld_w;
  int32_t* idx;
  float* wbar;
  double* dist;
  const kvcomm_match_info* info;  // candidates
  double* scratch = nullptr;      // partial + chunk sums owned by the caller (plans), else the pool's
  // sharded matching (plans only): own position blocks [own_lo, own_lo + n_own), n_own < 0 = all;
  // W columns and partial rows also stored into the peers' copies
  int own_lo = 0, n_own = -1, own_step = 1, n_peer = 0;
  float* X = nullptr;                   // exchange rows (position-major), sharded only
  float* X_peer[kMaxMatchPeers] = {};
  double* partial_peer[kMaxMatchPeers] = {};
};

static int match_blocks(int L_phi) { return (L_phi + kMatchP - 1) / kMatchP; }

struct MatchLayout {
  MatchHdr hdr{};
  size_t bytes = 0;
  size_t smem = 0;
};

MatchLayout layout_match(const std::vector<MatchItem>& items) {
  MatchLayout L;
  const int nj = int(items.size());
  L.hdr.n_jobs = nj;
  L.hdr.P = kMatchP;
  size_t n_ints = 0;
  int blocks = 0;
  for (const MatchItem& it : items) {
    n_ints += it.info->n_candidates + it.p->cap;
    blocks += it.n_own >= 0 ? it.n_own : match_blocks(it.L_phi);
    if (it.n_peer > 0) L.hdr.any_peer = 1;
    L.hdr.max_de = std::max(L.hdr.max_de, int32_t(it.p->De));
    L.smem = std::max(L.smem, align_up(size_t(kMatchP) * it.p->De * 2, 16) +
                                  size_t(kMatchP) * (3 * it.info->n_candidates + 1) * sizeof(double));
  }
  L.hdr.total_blocks = blocks;
  {  // the TMA-streamed distance kernel takes l2 jobs up to 256 candidates and D_e 8192
    static const int tma_env = [] {
      // measurement knob, off by default: 1 = the TMA tile-ring distance kernel, 2 = the TMA
      // row-ring kernel; both measured SLOWER than the register-streaming kernel (1: config 4
      // 3.13 vs 1.99 ms, one config-2 pool 86 vs 60 us, profiles/r02_match_tma.json; 2: config 2
      // 121 vs 103 us, config 4 2.30 vs 2.00 ms, profiles/r02h_match_ring.txt) — DESIGN §7
      const char* e = getenv("KVCOMM_MATCH_TMA");
      return e ? atoi(e) : 0;
    }();
    bool ok = tma_env != 0 && kMatchP == 2 && nj > 0;
    int de = 0, cm = 1;
    for (const MatchItem& it : items) {
      ok = ok && it.p->cfg.similarity == KVCOMM_SIM_L2 && it.info->n_candidates <= kMatchTmaMaxCand &&
           it.p->De <= kMatchTmaMaxDe;
      de = std::max(de, it.p->De);
      cm = std::max(cm, it.info->n_candidates);
    }
    if (ok && tma_env == 2) {  // row-ring kernel: one ring stage per anchor row
      const int rb = int(align_up(size_t(de) * 2, 128));
      const int qb = int(align_up(size_t(kMatchP) * de * 2, 128));
      const size_t fixed = match_ring_smem(0, rb, qb, cm, kMatchP);
      int stages = fixed < 227 * 1024 ? int(std::min<size_t>(16, (227 * 1024 - fixed) / (size_t(rb) + 16))) : 0;
      stages -= stages % kMatchRingWarps;  // parity safety: a stage's consecutive uses belong to one warp
      if (stages >= kMatchRingWarps) {
        L.hdr.tma = 2;
        L.hdr.tma_stages = stages;
        L.hdr.tma_qbytes = qb;
        L.hdr.tma_cmax = cm;
        L.hdr.ring_row_bytes = rb;
      }
    } else if (ok) {
      const int qb = int(align_up(size_t(kMatchP) * de * 2, 16));
      const size_t fixed = match_tma_smem(0, qb, cm);
      const int stages = int(std::min<size_t>(8, (227 * 1024 - fixed) / (kMatchStageBytes + 16)));
      if (stages >= 3) {
        L.hdr.tma = 1;
        L.hdr.tma_stages = stages;
        L.hdr.tma_qbytes = qb;
        L.hdr.tma_cmax = cm;
      }
    }
  }
  size_t off = align_up(sizeof(MatchHdr), 64);
  L.hdr.job_off = int64_t(off);
  off = align_up(off + sizeof(MatchJob) * nj, 64);
  L.hdr.int_off = int64_t(off);
  off = align_up(off + sizeof(int32_t) * n_ints, 64);
  L.hdr.res_off = int64_t(off);
  off = align_up(off + sizeof(MatchResultDev) * nj, 64);
  L.hdr.tie_off = int64_t(off);
  off = align_up(off + sizeof(int32_t) * (nj + 1), 64);  // per-job tie counters + the item counter
  L.bytes = off;
  return L;
}

void write_match(uint8_t* h, const MatchLayout& L, const std::vector<MatchItem>& items) {
  std::memset(h, 0, L.bytes);
  std::memcpy(h, &L.hdr, sizeof(L.hdr));
  MatchJob* jobs = reinterpret_cast<MatchJob*>(h + L.hdr.job_off);
  int32_t* ints = reinterpret_cast<int32_t*>(h + L.hdr.int_off);
  int ipos = 0, blocks = 0;
  for (size_t t = 0; t < items.size(); ++t) {
    const MatchItem& it = items[t];
    kvcomm_pool_s* p = it.p;
    MatchJob& a = jobs[t];
    a.query = static_cast<const bf16*>(it.query);
    a.emb = p->emb;
    a.slot_stride = p->emb_slot();
    a.emb_world = p->emb_world;
    a.W = it.W;
    a.ld_w = it.ld_w;
    a.top_k = it.top_k;
    a.idx = it.top_k > 0 ? it.idx : nullptr;
    a.dist_user = it.dist;
    if (it.scratch) {  // plan-owned: concurrent plans sharing a pool never share scratch
      a.partial = it.scratch;
      a.chunks = it.scratch + int64_t((it.L_phi + kMatchP - 1) / kMatchP) * (2 * p->cap + 1);
    } else {           // the pool's (guarded by its match-scratch lock until the results are read)
      a.partial = p->d_partial;
      a.chunks = p->d_partial + int64_t((p->maxlen + kMatchP - 1) / kMatchP) * (2 * p->cap + 1);
    }
    a.wbar = it.wbar;
    a.gamma = double(it.gamma);
    a.n_cand = it.info->n_candidates;
    a.cap = p->cap;
    a.L_phi = it.L_phi;
    a.De = p->De;
    a.scalar_mode = p->cfg.scalar_distance;
    a.cosine = p->cfg.similarity == KVCOMM_SIM_COSINE;
    a.cand_off = ipos;
    std::memcpy(ints + ipos, it.info->candidates, sizeof(int32_t) * a.n_cand);
    ipos += a.n_cand;
    a.s2c_off = ipos;
    for (int sl = 0; sl < p->cap; ++sl) ints[ipos + sl] = -1;
    for (int j = 0; j < a.n_cand; ++j) ints[ipos + it.info->candidates[j]] = j;
    ipos += p->cap;
    a.n_blocks = match_blocks(it.L_phi);
    a.block_begin = blocks;
    a.own_lo = it.n_own >= 0 ? it.own_lo : 0;
    a.own_step = it.n_own >= 0 ? it.own_step : 1;
    a.n_own = it.n_own >= 0 ? it.n_own : a.n_blocks;
    blocks += a.n_own;
    a.n_peer = it.n_peer;
    a.X = it.X;
    for (int r = 0; r < it.n_peer; ++r) {
      a.X_peer[r] = it.X_peer[r];
      a.partial_peer[r] = it.partial_peer[r];
    }
  }
}

// ---- realign work table -------------------------------------------------------
struct HostSeg {
  SegDev x;
  const int32_t* cand = nullptr;
  bool prefix = false;
  std::vector<int32_t> gates;  // indices into the gate results (match jobs)
};

struct RealignLayout {
  TableHdr hdr{};
  size_t bytes = 0;
};

RealignLayout layout_realign(int d, int Ls, int Hs, const std::vector<HostSeg>& hs) {
  RealignLayout L;
  const int n_seg = int(hs.size());
  const int rpt = rows_per_tile(d);
  size_t n_ints = 0, n_wt = 0, n_units = 0;
  for (const HostSeg& g : hs) {
    n_ints += g.x.n_cand + g.gates.size();
    if (g.x.fp8) L.hdr.any_fp8 = 1;
    if (g.x.dst_stg) L.hdr.any_stg = 1;
    const int rpu = unit_rows(d, g.x.fp8);
    n_wt += size_t((g.x.L_seg + rpu - 1) / rpu) * g.x.n_cand * weight_row_stride(rpu);
    n_units += size_t(Ls) * Hs * 2 * size_t((g.x.L_seg + rpu - 1) / rpu);
  }
  TableHdr& hdr = L.hdr;
  hdr.n_seg = n_seg;
  hdr.d = d;
  hdr.Ls = Ls;
  hdr.Hs = Hs;
  hdr.rows_per_tile = rpt;
  size_t off = align_up(sizeof(TableHdr), 64);
  hdr.seg_off = int64_t(off);
  off = align_up(off + sizeof(SegDev) * n_seg, 64);
  hdr.cand_off = int64_t(off);
  off = align_up(off + sizeof(int32_t) * std::max<size_t>(n_ints, 1), 64);
  hdr.cs_off = int64_t(off);
  off = align_up(off + sizeof(float2) * (d / 2) * n_seg, 64);
  hdr.wt_off = int64_t(off);
  off = align_up(off + sizeof(float) * n_wt, 64);
  hdr.unit_off = int64_t(off);
  off = align_up(off + sizeof(UnitDev) * std::max<size_t>(n_units, 1), 64);
  L.bytes = off;
  return L;
}

// h/dev: host image and device address of the realign part of a table.
void write_realign(uint8_t* h, uint8_t* dev, RealignLayout& L, const std::vector<HostSeg>& hs_in,
                   const MatchResultDev* gate_results) {
  TableHdr& hdr = L.hdr;
  const int d = hdr.d;
  // group segments that share a base cache (and hence its tiles): consecutive in the table
  std::vector<int> order(hs_in.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = int(i);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    const SegDev &x = hs_in[a].x, &y = hs_in[b].x;
    if (x.base[0] != y.base[0]) return x.base[0] < y.base[0];
    if (x.fp8 != y.fp8) return x.fp8 < y.fp8;
    return x.L_seg < y.L_seg;
  });
  SegDev* segs = reinterpret_cast<SegDev*>(h + hdr.seg_off);
  int32_t* ints = reinterpret_cast<int32_t*>(h + hdr.cand_off);
  const float* dwt = reinterpret_cast<const float*>(dev + hdr.wt_off);
  int64_t units = 0, tpos = 0;
  int ipos = 0;
  const int n = int(order.size());
  for (int t0 = 0; t0 < n;) {
    int t1 = t0 + 1;
    const SegDev& lead = hs_in[order[t0]].x;
    while (t1 < n && hs_in[order[t1]].x.base[0] == lead.base[0] && hs_in[order[t1]].x.base[1] == lead.base[1] &&
           hs_in[order[t1]].x.base_ld == lead.base_ld && hs_in[order[t1]].x.L_seg == lead.L_seg &&
           hs_in[order[t1]].x.fp8 == lead.fp8)
      ++t1;
    const int G = t1 - t0;
    const int rpu = unit_rows(d, lead.fp8);  // equal tiles for every member
    const int tiles = (lead.L_seg + rpu - 1) / rpu;
    for (int t = t0; t < t1; ++t) {
      const HostSeg& src = hs_in[order[t]];
      SegDev x = src.x;
      x.cand_off = ipos;
      if (x.n_cand) std::memcpy(ints + ipos, src.cand, sizeof(int32_t) * x.n_cand);
      ipos += x.n_cand;
      x.n_gate = int32_t(src.gates.size());
      x.gate_off = ipos;
      for (int32_t gi : src.gates) ints[ipos++] = gi;
      x.cs_off = t * (d / 2);
      x.tiles = tiles;
      x.unit_begin = units;
      x.group_size = G;
      x.group_member = t - t0;
      x.wt = dwt + tpos;
      x.wt_off = tpos;
      tpos += int64_t(tiles) * x.n_cand * weight_row_stride(rpu);
      segs[t] = x;
    }
    units += int64_t(hdr.Ls) * hdr.Hs * 2 * tiles * G;
    t0 = t1;
  }
  hdr.total_units = units;
  hdr.gate_results = gate_results;
  std::memcpy(h, &hdr, sizeof(hdr));
}

int grid_for_device(int dev) {
  static int grid_cache[64] = {0};
  if (!grid_cache[dev & 63]) grid_cache[dev & 63] = realign_grid_size(dev);
  return grid_cache[dev & 63];
}

}  // namespace

// ---- match -------------------------------------------------------------------
static kvcomm_status check_match_request(const kvcomm_match_request& q, int r) {
  kvcomm_pool_s* p = q.pool;
  if (!p || !q.info) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "request %d: null pool/info", r);
  if (p->emb_world > 1)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT,
                "request %d: the pool holds 1/%d of the embedding rows; match it through a plan sharded the same way "
                "(kvcomm_plan_match_shard)", r, p->emb_world);
  if (!(q.gamma >= 0.f && q.gamma <= 1.f))
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "request %d: gamma %g outside [0,1]", r, q.gamma);
  if (q.L_phi < 1) return fail(KVCOMM_ERR_SHAPE_MISMATCH, "request %d: L_phi %d < 1", r, q.L_phi);
  if (q.top_k < 0 || q.top_k > KVCOMM_MAX_TOPK)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "request %d: top_k %d outside [0,%d]", r, q.top_k, KVCOMM_MAX_TOPK);
  if (q.consumer != KVCOMM_ALL_CONSUMERS && (q.consumer < 0 || q.consumer >= p->C))
    return fail(KVCOMM_ERR_NOT_FOUND, "request %d: consumer %d", r, q.consumer);
  if (q.L_phi > p->maxlen && q.query_emb == nullptr) return KVCOMM_OK;
  return KVCOMM_OK;
}

static kvcomm_status check_match_buffers(const kvcomm_match_request& q, int r) {
  if (!q.query_emb || !q.W || !q.wbar) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "request %d: null query/W/wbar", r);
  if (!aligned16(q.query_emb))
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "request %d: query_emb not 16-byte aligned", r);
  if (q.ld_w < q.L_phi)
    return fail(KVCOMM_ERR_SHAPE_MISMATCH, "request %d: ld_w %lld < L_phi %d", r, (long long)q.ld_w, q.L_phi);
  return KVCOMM_OK;
}

KVCOMM_API kvcomm_status kvcomm_match_anchors_batch(const kvcomm_match_request* reqs, int32_t n, void* stream) {
  NvtxRange nvtx_("kvcomm_match_anchors_batch");
  if (n < 0 || (n > 0 && !reqs)) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "bad request list");
  std::vector<kvcomm_pool_s*> pools;
  for (int r = 0; r < n; ++r) {
    KV_TRY(check_match_request(reqs[r], r));
    kvcomm_pool_s* p = reqs[r].pool;
    if (std::find(pools.begin(), pools.end(), p) != pools.end())
      return fail(KVCOMM_ERR_INVALID_ARGUMENT, "request %d: pool appears twice in one batch", r);
    if (!pools.empty() && p->cfg.device != pools[0]->cfg.device)
      return fail(KVCOMM_ERR_INVALID_ARGUMENT, "request %d: pools on different devices", r);
    pools.push_back(p);
  }
  if (n == 0) return ok();
  std::vector<std::shared_lock<std::shared_mutex>> rlocks;
  lock_readers(pools, rlocks);
  std::vector<MatchItem> items;
  std::vector<int> active;
  for (int r = 0; r < n; ++r) {
    const kvcomm_match_request& q = reqs[r];
    if (!candidate_filter(q.pool, q.L_phi, q.consumer, q.info)) continue;
    KV_TRY(check_match_buffers(q, r));
    const int k_eff = q.top_k > 0 ? std::min(q.top_k, q.info->n_candidates) : 0;
    q.info->top_k = k_eff > 0 ? k_eff : q.info->n_candidates;
    items.push_back({q.pool, q.query_emb, q.L_phi, q.gamma, k_eff, q.W, q.ld_w, q.idx, q.wbar, q.dist, q.info});
    active.push_back(r);
  }
  if (items.empty()) return ok();
  const MatchLayout L = layout_match(items);
  const int dev = pools[0]->cfg.device;
  DeviceGuard guard(dev);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<std::unique_lock<std::mutex>> mlocks;
  lock_match_scratch(pools, mlocks);
  TableRing& ring = g_rings[dev & 63];
  std::lock_guard<std::mutex> rlk(ring.mu);
  RingEntry& E = ring.e[ring.next];
  ring.next = (ring.next + 1) % TableRing::kN;
  KV_TRY(entry_reserve(E, L.bytes));
  uint8_t* h = static_cast<uint8_t*>(E.host);
  write_match(h, L, items);
  KV_CUDA(cudaMemcpyAsync(E.dev, E.host, L.bytes, cudaMemcpyHostToDevice, s));
  KV_CUDA(launch_match_batch(E.dev, L.hdr, L.smem, s));
  g_launches += 3;  // distances + weights, chunk sums, finalize
  KV_CUDA(cudaMemcpyAsync(h + L.hdr.res_off, static_cast<uint8_t*>(E.dev) + L.hdr.res_off,
                          L.bytes - size_t(L.hdr.res_off), cudaMemcpyDeviceToHost, s));
  KV_CUDA(cudaEventRecord(E.done, s));
  E.used = true;
  KV_CUDA(cudaStreamSynchronize(s));
  const MatchResultDev* res = reinterpret_cast<const MatchResultDev*>(h + L.hdr.res_off);
  for (size_t t = 0; t < active.size(); ++t) fill_info_from_result(reqs[active[t]].info, res[t]);
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_match_anchors(kvcomm_pool_t p, const void* query_emb, int32_t L_phi,
                                              int32_t consumer, float gamma, int32_t top_k, float* W,
                                              int64_t ld_w, int32_t* idx, float* wbar, double* dist,
                                              kvcomm_match_info* info, void* stream) {
  kvcomm_match_request q{p, query_emb, L_phi, consumer, gamma, top_k, W, ld_w, idx, wbar, dist, info};
  return kvcomm_match_anchors_batch(&q, 1, stream);
}

// ---- realign -----------------------------------------------------------------
static kvcomm_status validate_segment(const kvcomm_realign_desc& g, int idx) {
  kvcomm_pool_s* p = g.pool;
  if (!p) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "segment %d: null pool", idx);
  if (g.kind != KVCOMM_PLACEHOLDER && g.kind != KVCOMM_PREFIX && g.kind != KVCOMM_COPY)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "segment %d: kind %d", idx, g.kind);
  if (g.L_seg < 0) return fail(KVCOMM_ERR_SHAPE_MISMATCH, "segment %d: L_seg %d", idx, g.L_seg);
  if (g.L_seg == 0) return KVCOMM_OK;
  KV_TRY(check_view(g.base, g.L_seg, "base"));
  if (!g.dst_k || !g.dst_v || !aligned16(g.dst_k) || !aligned16(g.dst_v))
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "segment %d: dst null or misaligned", idx);
  if (g.target_start < 0 || int64_t(g.target_start) + g.L_seg > g.dst_ld)
    return fail(KVCOMM_ERR_SHAPE_MISMATCH, "segment %d: rows [%d,%d) outside dst_ld %lld", idx, g.target_start,
                g.target_start + g.L_seg, (long long)g.dst_ld);
  if (g.dst_heads != 0 && (g.dst_heads < p->Hs || g.dst_heads > 1 << 20))
    return fail(KVCOMM_ERR_SHAPE_MISMATCH, "segment %d: dst_heads %d < the pool's %d heads", idx, g.dst_heads, p->Hs);
  if (g.kind == KVCOMM_COPY) return KVCOMM_OK;
  if (g.consumer < 0 || g.consumer >= p->C)
    return fail(KVCOMM_ERR_NOT_FOUND, "segment %d: consumer %d outside [0,%d)", idx, g.consumer, p->C);
  if (g.n_candidates < 1 || !g.candidates)
    return fail(KVCOMM_ERR_NO_CANDIDATES, "segment %d: empty candidate set", idx);
  if (g.n_candidates > p->cap) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "segment %d: n_candidates", idx);
  if (!g.weights) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "segment %d: null weights", idx);
  // the per-tile weight blocks are indexed in 32 bits (realign_prep_kernel)
  if ((int64_t(g.L_seg) + 2 * rows_per_tile(p->d)) * g.n_candidates * 2 >= (int64_t(1) << 31))
    return fail(KVCOMM_ERR_SHAPE_MISMATCH, "segment %d: %d rows x %d anchors exceeds the weight table", idx,
                g.L_seg, g.n_candidates);
  if (g.kind == KVCOMM_PREFIX) {
    if (g.L_seg != p->prefix_len[g.consumer])
      return fail(KVCOMM_ERR_SHAPE_MISMATCH, "segment %d: prefix L_seg %d != prefix_len %d", idx, g.L_seg,
                  p->prefix_len[g.consumer]);
  } else {
    if (g.L_seg > p->maxlen)
      return fail(KVCOMM_ERR_SHAPE_MISMATCH, "segment %d: L_seg %d > max_anchor_len %d", idx, g.L_seg, p->maxlen);
    if (g.ld_w % 4 != 0 || g.ld_w < ((g.L_seg + 3) & ~3))
      return fail(KVCOMM_ERR_SHAPE_MISMATCH, "segment %d: ld_w %lld must be a multiple of 4 >= L_seg", idx,
                  (long long)g.ld_w);
    if (!aligned16(g.weights)) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "segment %d: W not 16-byte aligned", idx);
  }
  if ((g.debug_delta_k && !aligned16(g.debug_delta_k)) || (g.debug_delta_v && !aligned16(g.debug_delta_v)))
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "segment %d: debug buffers misaligned", idx);
  const uint64_t bit = 1ull << g.consumer;
  for (int j = 0; j < g.n_candidates; ++j) {
    const int s = g.candidates[j];
    if (s < 0 || s >= p->cap || !p->slots[s].occupied)
      return fail(KVCOMM_ERR_NOT_FOUND, "segment %d: candidate slot %d is empty", idx, s);
    const SlotMeta& m = p->slots[s];
    if (g.kind == KVCOMM_PLACEHOLDER) {
      if (m.length < g.L_seg)
        return fail(KVCOMM_ERR_SHAPE_MISMATCH, "segment %d: anchor slot %d has L=%d < L_seg %d", idx, s, m.length,
                    g.L_seg);
      if (!(m.ph_mask & bit))
        return fail(KVCOMM_ERR_MISSING_OFFSET, "segment %d: slot %d lacks placeholder offsets of consumer %d", idx,
                    s, g.consumer);
    } else if (!(m.pf_mask & bit)) {
      return fail(KVCOMM_ERR_MISSING_OFFSET, "segment %d: slot %d lacks prefix offsets of consumer %d", idx, s,
                  g.consumer);
    }
  }
  return KVCOMM_OK;
}

// Destinations on another GPU (a consumer's cache mapped by CUDA IPC: the fused gather,
// SURVEY §8(e)) are written with per-thread stores (mode 1) by default, or — measurement
// knob KVCOMM_PEER_STORE=bulk, for the first multi-GPU run — with the same TMA bulk store
// as local rows, issued to the peer address (mode 2; one 16 KiB transfer per tile instead
// of 1,024 16-byte stores).  Either way the kernel ends with a system-scope fence.
// KVCOMM_STORE_STG=1 forces per-thread stores everywhere (tests compare that path with
// the TMA bulk-store path bit for bit).
static int32_t dst_store_mode(const void* dst, int device) {
  const char* e = getenv("KVCOMM_STORE_STG");
  if (e && atoi(e) == 1) return 1;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, dst) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (!(at.type == cudaMemoryTypeDevice && at.device != device)) return 0;
  static const bool bulk = [] {
    const char* v = getenv("KVCOMM_PEER_STORE");
    return v && std::strcmp(v, "bulk") == 0;
  }();
  return bulk ? 2 : 1;
}

static HostSeg host_segment(const kvcomm_realign_desc& g, int32_t dst_stg = -1) {
  kvcomm_pool_s* p = g.pool;
  HostSeg h{};
  SegDev& x = h.x;
  x.base[0] = static_cast<const bf16*>(g.base.k);
  x.base[1] = static_cast<const bf16*>(g.base.v);
  x.base_ld = ld_of(g.base, g.L_seg);
  x.dst[0] = static_cast<bf16*>(g.dst_k);
  x.dst[1] = static_cast<bf16*>(g.dst_v);
  x.dst_ld = g.dst_ld;
  x.dst_heads = g.dst_heads > 0 ? g.dst_heads : p->Hs;
  x.dst_stg = dst_stg >= 0 ? dst_stg : dst_store_mode(g.dst_k, p->cfg.device);
  x.rope_il = p->cfg.rope_layout == KVCOMM_ROPE_INTERLEAVED;
  x.inv_freq = p->inv_freq_dev;
  x.L_seg = g.L_seg;
  x.target_start = g.target_start;
  x.w_by_slot = 1;
  if (g.kind == KVCOMM_COPY) return h;  // delta 0, no candidates: verbatim rows
  x.dbg[0] = g.debug_delta_k;
  x.dbg[1] = g.debug_delta_v;
  x.delta = g.target_start - g.base_start;
  x.n_cand = g.n_candidates;
  h.cand = g.candidates;
  x.fp8 = p->fp8 ? 1 : 0;
  if (g.kind == KVCOMM_PLACEHOLDER) {
    x.w = g.weights;
    x.ld_w = g.ld_w;
    if (!p->fp8) {
      x.off = p->ph_base(g.consumer);
      x.slot_stride = p->ph_slot_stride();
      x.plane_stride = p->ph_plane_stride();
      x.off_ld = p->ph_ld;
    } else {
      x.off = reinterpret_cast<const bf16*>(p->ph8 + int64_t(g.consumer) * p->cap * p->f8_ph_slot());
      x.slot_stride = p->f8_ph_slot();
      x.plane_stride = p->f8_ph_plane();
      x.off_ld = p->f8_lh(p->ph_ld);
    }
  } else {
    h.prefix = true;
    x.w_by_slot = 0;
    x.wbar = g.weights;
    if (!p->fp8) {
      x.off = p->pf[g.consumer];
      x.slot_stride = p->pf_slot_stride(g.consumer);
      x.plane_stride = p->pf_plane_stride(g.consumer);
      x.off_ld = p->pf_ld(g.consumer);
    } else {
      x.off = reinterpret_cast<const bf16*>(p->pf8[g.consumer]);
      x.slot_stride = p->f8_pf_slot(g.consumer);
      x.plane_stride = p->f8_pf_plane(g.consumer);
      x.off_ld = p->f8_lh(p->prefix_len[g.consumer]);
    }
  }
  return h;
}

// Builds the work table of `hs` in a ring entry and launches prep + realign kernels.
static kvcomm_status launch_segments(int dev, int d, int Ls, int Hs, const std::vector<HostSeg>& hs,
                                     cudaStream_t s) {
  if (hs.empty()) return KVCOMM_OK;
  RealignLayout L = layout_realign(d, Ls, Hs, hs);
  TableRing& ring = g_rings[dev & 63];
  std::lock_guard<std::mutex> rlk(ring.mu);
  RingEntry& E = ring.e[ring.next];
  ring.next = (ring.next + 1) % TableRing::kN;
  KV_TRY(entry_reserve(E, L.bytes));
  write_realign(static_cast<uint8_t*>(E.host), static_cast<uint8_t*>(E.dev), L, hs, nullptr);
  KV_CUDA(cudaMemcpyAsync(E.dev, E.host, size_t(L.hdr.cs_off), cudaMemcpyHostToDevice, s));
  KV_CUDA(launch_realign(E.dev, L.hdr, grid_for_device(dev), s));
  g_launches += L.hdr.total_units > 0 ? 2 : 1;
  KV_CUDA(cudaEventRecord(E.done, s));
  E.used = true;
  return KVCOMM_OK;
}

KVCOMM_API kvcomm_status kvcomm_realign_segments(const kvcomm_realign_desc* segs, int32_t n, void* stream) {
  NvtxRange nvtx_("kvcomm_realign_segments");
  if (n < 0 || (n > 0 && !segs)) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "bad segment list");
  kvcomm_pool_s* p0 = nullptr;
  std::vector<kvcomm_pool_s*> pools;
  for (int i = 0; i < n; ++i) {
    kvcomm_pool_s* p = segs[i].pool;
    if (!p) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "segment %d: null pool", i);
    if (!p0) p0 = p;
    if (p->Ls != p0->Ls || p->Hs != p0->Hs || p->d != p0->d || p->cfg.device != p0->cfg.device)
      return fail(KVCOMM_ERR_SHAPE_MISMATCH, "segment %d: pool geometry differs from segment 0", i);
    pools.push_back(p);
  }
  if (!p0) return ok();
  std::vector<std::shared_lock<std::shared_mutex>> locks;
  lock_readers(pools, locks);
  std::vector<HostSeg> hs;
  hs.reserve(n);
  for (int i = 0; i < n; ++i) {
    KV_TRY(validate_segment(segs[i], i));
    if (segs[i].L_seg > 0) hs.push_back(host_segment(segs[i]));
  }
  DeviceGuard guard(p0->cfg.device);
  KV_TRY(launch_segments(p0->cfg.device, p0->d, p0->Ls, p0->Hs, hs, static_cast<cudaStream_t>(stream)));
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_realign_segment(const kvcomm_realign_desc* seg, void* stream) {
  if (!seg) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null segment");
  return kvcomm_realign_segments(seg, 1, stream);
}

// ---- concat ------------------------------------------------------------------
static kvcomm_status check_ledger(const int32_t* starts, const int32_t* lengths, int n, int32_t N_total) {
  int64_t pos = 0;  // segments tile [0, N_total) in order
  for (int i = 0; i < n; ++i) {
    if (lengths[i] < 0) return fail(KVCOMM_ERR_SHAPE_MISMATCH, "segment %d: negative length", i);
    if (starts[i] > pos) return fail(KVCOMM_ERR_POSITION_GAP, "gap at position %lld (segment %d)", (long long)pos, i);
    if (starts[i] < pos) return fail(KVCOMM_ERR_POSITION_OVERLAP, "overlap at position %d (segment %d)", starts[i], i);
    pos = int64_t(starts[i]) + lengths[i];
  }
  if (pos < N_total) return fail(KVCOMM_ERR_POSITION_GAP, "gap at position %lld (end)", (long long)pos);
  if (pos > N_total) return fail(KVCOMM_ERR_POSITION_OVERLAP, "segments run past N_total %d", N_total);
  return KVCOMM_OK;
}

KVCOMM_API kvcomm_status kvcomm_concat_prefill_cache(const kvcomm_segment_ref* segs, int32_t n, int32_t N_total,
                                                     int32_t Ls, int32_t Hs, int32_t d, void* dst_k, void* dst_v,
                                                     int64_t dst_ld, int32_t device, void* stream) {
  NvtxRange nvtx_("kvcomm_concat_prefill_cache");
  if (n < 0 || (n > 0 && !segs)) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "bad segment list");
  if (Ls < 1 || Hs < 1 || d < 16 || d % 16 != 0 || d > 256) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "bad geometry");
  if (N_total < 0 || dst_ld < N_total)
    return fail(KVCOMM_ERR_SHAPE_MISMATCH, "dst_ld %lld < N_total %d", (long long)dst_ld, N_total);
  std::vector<int32_t> st(n), ln(n);
  for (int i = 0; i < n; ++i) {
    st[i] = segs[i].start;
    ln[i] = segs[i].length;
  }
  KV_TRY(check_ledger(st.data(), ln.data(), n, N_total));
  if (!dst_k || !dst_v || !aligned16(dst_k) || !aligned16(dst_v))
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "dst null or misaligned");
  std::vector<HostSeg> hs;
  const int32_t stg = dst_store_mode(dst_k, device);
  for (int i = 0; i < n; ++i) {
    if (!segs[i].src.k || segs[i].length == 0) continue;
    KV_TRY(check_view(segs[i].src, segs[i].length, "concat src"));
    HostSeg h{};
    SegDev& x = h.x;
    x.base[0] = static_cast<const bf16*>(segs[i].src.k);
    x.base[1] = static_cast<const bf16*>(segs[i].src.v);
    x.base_ld = ld_of(segs[i].src, segs[i].length);
    x.dst[0] = static_cast<bf16*>(dst_k);
    x.dst[1] = static_cast<bf16*>(dst_v);
    x.dst_ld = dst_ld;
    x.dst_heads = Hs;
    x.dst_stg = stg;
    x.L_seg = segs[i].length;
    x.target_start = segs[i].start;
    x.w_by_slot = 1;
    hs.push_back(h);
  }
  if (hs.empty()) return ok();
  DeviceGuard guard(device);
  KV_TRY(launch_segments(device, d, Ls, Hs, hs, static_cast<cudaStream_t>(stream)));
  return ok();
}

// ---- request plan (native executor of Algorithm 1's reuse branch) --------------
struct kvcomm_plan_s {
  int dev = 0, d = 0, Ls = 0, Hs = 0;
  std::vector<kvcomm_plan_match> matches;
  std::vector<kvcomm_plan_segment> segs;
  std::vector<kvcomm_plan_agent> agents;
  std::vector<std::vector<int>> agent_matches;  // distinct matches each agent depends on
  // Match buffers, one set per table parity (run t uses set t % 2), all in ONE allocation
  // (`xbuf`, exportable by CUDA IPC for sharded matching): per parity and match
  // W [cap][ld_w] f32, w̄ [cap] f32, scratch [ceil(L_phi/P) + kMatchChunks][2 cap + 1] f64.
  void* xbuf = nullptr;
  int64_t xbytes = 0;
  std::vector<int64_t> W_off[2], wbar_off[2], sc_off[2], X_off[2];  // byte offsets into xbuf
  int64_t fp_off[2] = {0, 0};     // per parity: uint64 fingerprints [kMaxMatchPeers + 1] (sharded runs)
  std::vector<int64_t> ld_w;
  // sharded matching: this rank's position blocks, and the peers' xbuf mappings
  int rank = 0, world = 1;
  std::vector<char*> peer_x;   // world - 1 mapped peer buffers (this process's addresses)
  RingEntry tab[2];
  int next = 0;
  // a run between kvcomm_plan_run_begin and kvcomm_plan_run_end
  bool pending = false;
  MatchLayout pML;
  RealignLayout pRL;
  size_t proff = 0;
  size_t n_items = 0, n_hs = 0;
  // last run
  int last = -1;
  std::vector<kvcomm_match_info> infos;
  std::vector<int> job_of;        // match -> job index in the last run (-1: decided on host)
  std::vector<int32_t> agent_state;  // 0 reuse pending/ok, 1 fallback (host-decided)
  std::vector<int32_t> agent_stg;    // destination store mode per agent (dst_store_mode at create)
  int64_t res_off = 0;
  cudaEvent_t ev_before = nullptr, ev_after = nullptr;
  cudaEvent_t ev_mbefore = nullptr, ev_mafter = nullptr;  // around the distance kernel
  // kvcomm_plan_set_realign_stream: the realign kernel of every run goes to rstream (after
  // the run's prep, by ev_prep[parity]) so that the next run's matching can overlap it
  cudaStream_t rstream = nullptr;
  bool rstream_set = false;
  cudaEvent_t ev_prep[2] = {nullptr, nullptr};
  std::mutex mu;

  char* xb() const { return static_cast<char*>(xbuf); }
  float* W(int par, int i) const { return reinterpret_cast<float*>(xb() + W_off[par][i]); }
  float* wbar(int par, int i) const { return reinterpret_cast<float*>(xb() + wbar_off[par][i]); }
  double* scratch(int par, int i) const { return reinterpret_cast<double*>(xb() + sc_off[par][i]); }
};

static void plan_close_peers(kvcomm_plan_s* pl) {
  for (char* x : pl->peer_x) cudaIpcCloseMemHandle(x);
  pl->peer_x.clear();
  pl->rank = 0;
  pl->world = 1;
}

static void plan_free(kvcomm_plan_s* pl) {
  if (!pl) return;
  DeviceGuard g(pl->dev);
  for (auto& e : pl->tab) entry_free(e);
  for (cudaEvent_t& e : pl->ev_prep)
    if (e) cudaEventDestroy(e);
  plan_close_peers(pl);
  cudaFree(pl->xbuf);
  delete pl;
}

KVCOMM_API kvcomm_status kvcomm_plan_create(const kvcomm_plan_match* matches, int32_t n_matches,
                                            const kvcomm_plan_segment* segs, int32_t n_segs,
                                            const kvcomm_plan_agent* agents, int32_t n_agents, kvcomm_plan_t* out) {
  if (!out || n_matches < 1 || !matches || n_segs < 0 || (n_segs > 0 && !segs) || n_agents < 1 || !agents)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "bad plan arguments");
  *out = nullptr;
  kvcomm_pool_s* p0 = matches[0].pool;
  for (int i = 0; i < n_matches; ++i) {
    const kvcomm_plan_match& m = matches[i];
    kvcomm_pool_s* p = m.pool;
    if (!p) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "match %d: null pool", i);
    if (p->Ls != p0->Ls || p->Hs != p0->Hs || p->d != p0->d || p->cfg.device != p0->cfg.device)
      return fail(KVCOMM_ERR_SHAPE_MISMATCH, "match %d: pool geometry differs from match 0", i);
    for (int j = 0; j < i; ++j)
      if (matches[j].pool == p) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "match %d: pool used twice", i);
    if (!(m.gamma >= 0.f && m.gamma <= 1.f)) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "match %d: gamma", i);
    if (m.L_phi < 1 || m.L_phi > p->maxlen) return fail(KVCOMM_ERR_SHAPE_MISMATCH, "match %d: L_phi %d", i, m.L_phi);
    if (m.top_k < 0 || m.top_k > KVCOMM_MAX_TOPK) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "match %d: top_k", i);
    if (m.consumer != KVCOMM_ALL_CONSUMERS && (m.consumer < 0 || m.consumer >= p->C))
      return fail(KVCOMM_ERR_NOT_FOUND, "match %d: consumer %d", i, m.consumer);
  }
  std::vector<std::vector<int>> am(n_agents);
  std::vector<std::vector<std::pair<int32_t, int32_t>>> ledger(n_agents);
  for (int i = 0; i < n_segs; ++i) {
    const kvcomm_plan_segment& s = segs[i];
    if (s.agent < 0 || s.agent >= n_agents) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "segment %d: agent", i);
    const kvcomm_plan_agent& a = agents[s.agent];
    if (s.kind != KVCOMM_COPY) {
      if (s.match < 0 || s.match >= n_matches) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "segment %d: match", i);
      kvcomm_pool_s* p = matches[s.match].pool;
      if (s.kind == KVCOMM_PLACEHOLDER && s.L_seg != matches[s.match].L_phi)
        return fail(KVCOMM_ERR_SHAPE_MISMATCH, "segment %d: placeholder length %d != L_phi %d", i, s.L_seg,
                    matches[s.match].L_phi);
      if (s.consumer < 0 || s.consumer >= p->C) return fail(KVCOMM_ERR_NOT_FOUND, "segment %d: consumer", i);
      if (s.kind == KVCOMM_PREFIX && s.L_seg != p->prefix_len[s.consumer])
        return fail(KVCOMM_ERR_SHAPE_MISMATCH, "segment %d: prefix length %d != %d", i, s.L_seg,
                    p->prefix_len[s.consumer]);
      if (std::find(am[s.agent].begin(), am[s.agent].end(), s.match) == am[s.agent].end())
        am[s.agent].push_back(s.match);
    } else if (s.kind != KVCOMM_COPY) {
      return fail(KVCOMM_ERR_INVALID_ARGUMENT, "segment %d: kind", i);
    }
    if (s.L_seg > 0) KV_TRY(check_view(s.base, s.L_seg, "plan segment base"));
    if (!a.dst_k || !a.dst_v || !aligned16(a.dst_k) || !aligned16(a.dst_v) || a.dst_ld < a.N)
      return fail(KVCOMM_ERR_INVALID_ARGUMENT, "agent %d: bad destination", s.agent);
    if (a.dst_heads != 0 && (a.dst_heads < p0->Hs || a.dst_heads > 1 << 20))
      return fail(KVCOMM_ERR_SHAPE_MISMATCH, "agent %d: dst_heads %d < the pools' %d heads", s.agent, a.dst_heads,
                  p0->Hs);
    ledger[s.agent].push_back({s.target_start, s.L_seg});
  }
  for (int a = 0; a < n_agents; ++a) {  // every prompt must be tiled exactly (reading A20 + P:304)
    auto& l = ledger[a];
    std::sort(l.begin(), l.end());
    std::vector<int32_t> st, ln;
    for (auto& x : l) {
      st.push_back(x.first);
      ln.push_back(x.second);
    }
    kvcomm_status s = check_ledger(st.data(), ln.data(), int(st.size()), agents[a].N);
    if (s != KVCOMM_OK) {
      g_err = "agent " + std::to_string(a) + ": " + g_err;
      return s;
    }
  }
  DeviceGuard guard(p0->cfg.device);
  auto* pl = new kvcomm_plan_s();
  pl->dev = p0->cfg.device;
  pl->d = p0->d;
  pl->Ls = p0->Ls;
  pl->Hs = p0->Hs;
  pl->matches.assign(matches, matches + n_matches);
  pl->segs.assign(segs, segs + n_segs);
  pl->agents.assign(agents, agents + n_agents);
  for (int a = 0; a < n_agents; ++a) pl->agent_stg.push_back(dst_store_mode(agents[a].dst_k, p0->cfg.device));
  pl->agent_matches = am;
  pl->infos.resize(n_matches);
  pl->job_of.assign(n_matches, -1);
  pl->agent_state.assign(n_agents, 1);
  int64_t off = 0;
  for (int i = 0; i < n_matches; ++i) pl->ld_w.push_back((matches[i].L_phi + 3) & ~3);
  for (int par = 0; par < 2; ++par)
    for (int i = 0; i < n_matches; ++i) {
      const int cap = matches[i].pool->cap;
      pl->W_off[par].push_back(off);
      off = int64_t(align_up(size_t(off + int64_t(sizeof(float)) * pl->ld_w[i] * cap), 256));
      pl->wbar_off[par].push_back(off);
      off = int64_t(align_up(size_t(off + int64_t(sizeof(float)) * cap), 256));
      pl->sc_off[par].push_back(off);
      off = int64_t(align_up(size_t(off + int64_t(sizeof(double)) * (match_blocks(matches[i].L_phi) + kMatchChunks) *
                                              (2 * cap + 1)),
                             256));
      pl->X_off[par].push_back(off);  // sharded matching's exchange rows [blocks * P][cap]
      off = int64_t(align_up(size_t(off + int64_t(sizeof(float)) * match_blocks(matches[i].L_phi) * kMatchP * cap), 256));
    }
  for (int par = 0; par < 2; ++par) {
    pl->fp_off[par] = off;
    off += int64_t(align_up(sizeof(uint64_t) * (kMaxMatchPeers + 1), 256));
  }
  pl->xbytes = off;
  if (cudaMalloc(&pl->xbuf, size_t(off)) != cudaSuccess ||
      cudaMemset(static_cast<char*>(pl->xbuf) + pl->fp_off[0], 0, size_t(off - pl->fp_off[0])) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(pl->xbuf);
    pl->xbuf = nullptr;
    plan_free(pl);
    return fail(KVCOMM_ERR_OUT_OF_MEMORY, "plan weight buffers (%lld bytes)", (long long)off);
  }
  *out = pl;
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_plan_destroy(kvcomm_plan_t pl) {
  if (!pl) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null plan");
  plan_free(pl);
  return ok();
}

// First half of a run: the candidate filter (a1, host), the work table upload and the
// distance + weight kernel over this rank's position blocks.
static kvcomm_status plan_begin(kvcomm_plan_s* pl, const void* const* query_embs, cudaStream_t s) {
  if (pl->pending) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "plan run already begun (call kvcomm_plan_run_end)");
  const int nm = int(pl->matches.size());
  for (int i = 0; i < nm; ++i)
    if (!query_embs[i] || !aligned16(query_embs[i]))
      return fail(KVCOMM_ERR_INVALID_ARGUMENT, "query %d null or misaligned", i);
  std::vector<kvcomm_pool_s*> pools;
  for (auto& m : pl->matches) pools.push_back(m.pool);
  std::vector<std::shared_lock<std::shared_mutex>> rlocks;
  lock_readers(pools, rlocks);
  DeviceGuard guard(pl->dev);
  const int par = pl->next;
  RingEntry& E = pl->tab[par];
  KV_TRY(entry_reserve(E, 0));  // waits for the run that used this table two runs ago
  // job_of / infos are rebuilt below; until this run completes there is no result to report
  // (a failure part-way must not leave plan_results reading the old table through new jobs)
  pl->last = -1;
  // a1 on the host; jobs for the entropy clause
  std::vector<MatchItem> items;
  std::vector<bool> host_new(nm, false);
  for (int i = 0; i < nm; ++i) {
    const kvcomm_plan_match& m = pl->matches[i];
    kvcomm_match_info* info = &pl->infos[i];
    pl->job_of[i] = -1;
    if (!candidate_filter(m.pool, m.L_phi, m.consumer, info)) {
      host_new[i] = true;
      continue;
    }
    const int k_eff = m.top_k > 0 ? std::min(m.top_k, info->n_candidates) : 0;
    info->top_k = k_eff > 0 ? k_eff : info->n_candidates;
    pl->job_of[i] = int(items.size());
    MatchItem it{m.pool, query_embs[i], m.L_phi, m.gamma, k_eff, pl->W(par, i), pl->ld_w[i], nullptr,
                 pl->wbar(par, i), nullptr, info, pl->scratch(par, i)};
    if (m.pool->emb_world > 1 && (m.pool->emb_world != pl->world || m.pool->emb_rank != pl->rank))
      return fail(KVCOMM_ERR_INVALID_ARGUMENT,
                  "match %d: the pool holds the embeddings of rank %d of %d; the plan matches as rank %d of %d", i,
                  m.pool->emb_rank, m.pool->emb_world, pl->rank, pl->world);
    if (pl->world > 1) {  // position blocks b = rank (mod world); the rest comes from the peers
      const int nb = match_blocks(m.L_phi);
      it.own_lo = pl->rank;
      it.own_step = pl->world;
      it.n_own = pl->rank < nb ? (nb - pl->rank + pl->world - 1) / pl->world : 0;
      it.n_peer = int(pl->peer_x.size());
      it.X = reinterpret_cast<float*>(pl->xb() + pl->X_off[par][i]);
      for (int r = 0; r < it.n_peer; ++r) {
        it.X_peer[r] = reinterpret_cast<float*>(pl->peer_x[r] + pl->X_off[par][i]);
        it.partial_peer[r] = reinterpret_cast<double*>(pl->peer_x[r] + pl->sc_off[par][i]);
      }
    }
    items.push_back(it);
  }
  // segments of agents not already decided by the length clause, gated on device
  std::vector<HostSeg> hs;
  for (size_t a = 0; a < pl->agents.size(); ++a) {
    bool closed = false;
    for (int mi : pl->agent_matches[a]) closed |= host_new[mi];
    pl->agent_state[a] = closed ? 1 : 0;
  }
  for (const kvcomm_plan_segment& g : pl->segs) {
    if (g.L_seg == 0 || pl->agent_state[g.agent]) continue;
    const kvcomm_plan_agent& a = pl->agents[g.agent];
    kvcomm_realign_desc d{};
    d.pool = g.kind == KVCOMM_COPY ? pl->matches[0].pool : pl->matches[g.match].pool;
    d.consumer = g.consumer;
    d.kind = g.kind;
    d.L_seg = g.L_seg;
    d.base = g.base;
    d.base_start = g.base_start;
    d.target_start = g.target_start;
    d.dst_k = a.dst_k;
    d.dst_v = a.dst_v;
    d.dst_ld = a.dst_ld;
    d.dst_heads = a.dst_heads;
    if (g.kind != KVCOMM_COPY) {
      const kvcomm_match_info* info = &pl->infos[g.match];
      d.weights = g.kind == KVCOMM_PLACEHOLDER ? pl->W(par, g.match) : pl->wbar(par, g.match);
      d.ld_w = pl->ld_w[g.match];
      d.candidates = info->candidates;
      d.n_candidates = info->n_candidates;
      KV_TRY(validate_segment(d, int(&g - pl->segs.data())));
    }
    HostSeg h = host_segment(d, pl->agent_stg[g.agent]);
    for (int mi : pl->agent_matches[g.agent]) h.gates.push_back(pl->job_of[mi]);
    hs.push_back(std::move(h));
  }
  // one table: [match part][realign part]
  // Sharded plans always launch the distance kernel, even with no job (every match decided
  // on the host): its fingerprint tells the peers this rank's layout differs from theirs.
  const bool match_table = !items.empty() || pl->world > 1;
  MatchLayout ML = match_table ? layout_match(items) : MatchLayout();
  if (pl->world > 1) {  // layout fingerprint, compared across ranks by finalize
    uint64_t h = 1469598103934665603ull;
    auto mix = [&h](uint64_t v) {
      for (int b = 0; b < 8; ++b) {
        h ^= (v >> (8 * b)) & 0xffu;
        h *= 1099511628211ull;
      }
    };
    mix(items.size());
    for (const MatchItem& it : items) {
      uint32_t gb;
      std::memcpy(&gb, &it.gamma, sizeof(gb));
      mix(uint64_t(it.p->cap) << 32 | uint32_t(it.L_phi));
      mix(uint64_t(it.top_k) << 32 | gb);
      mix(uint64_t(it.p->cfg.scalar_distance) << 32 | uint32_t(it.p->cfg.similarity));
      mix(uint64_t(it.info->n_candidates) << 32 | uint32_t(it.p->emb_world));
      // which anchor occupies each candidate slot: once a pool is full every insert reuses an
      // evicted slot id, so the ids alone would not tell two ranks' different anchors apart
      // (a missed or reordered insert, or LFU counts that diverged and evicted other victims)
      for (int j = 0; j < it.info->n_candidates; ++j) {
        const SlotMeta& sm = it.p->slots[it.info->candidates[j]];
        mix(uint64_t(uint32_t(it.info->candidates[j])) << 32 | uint32_t(sm.length));
        mix(uint64_t(sm.inserted));
      }
    }
    ML.hdr.fingerprint = h;
    ML.hdr.shard_rank = pl->rank;
    ML.hdr.shard_world = pl->world;
    for (int r = 0, q = 0; r < pl->world; ++r) {
      char* base = r == pl->rank ? pl->xb() : pl->peer_x[q++];
      ML.hdr.fp_dst[r] = reinterpret_cast<uint64_t*>(base + pl->fp_off[par]) + pl->rank;
    }
    ML.hdr.fp_mine = reinterpret_cast<const uint64_t*>(pl->xb() + pl->fp_off[par]);
    ML.hdr.any_peer = 1;  // system-scope fence after the (peer) fingerprint stores
  }
  // Pipelined runs: the next run's match runs beside the realign only in the 40-register
  // build, at one or two CTAs per SM — worth it while the match is small next to the
  // realign (config 2: 0.53 vs 30.5 GB; a sharded 70B match: 1.6 vs 33 GB); a large one
  // (config 4's replicated 12.9 GB) would outlast the realign there, so it keeps the
  // faster build and follows the realign (measured: profiles/r02h_config4.json)
  if (pl->rstream_set && match_table) {
    double mb = 0.0, rb = 0.0;
    for (const MatchItem& it : items)
      mb += double(it.n_own >= 0 ? int64_t(it.n_own) * kMatchP : it.L_phi) * (it.info->n_candidates + 1) *
            it.p->De * 2.0;
    for (const HostSeg& g : hs) rb += double(g.x.L_seg) * (g.x.n_cand + 2) * 2.0 * pl->Ls * pl->Hs * pl->d * 2.0;
    ML.hdr.beside_realign = mb * 8.0 <= rb ? 1 : 0;
  }
  RealignLayout RL = layout_realign(pl->d, pl->Ls, pl->Hs, hs);
  const size_t roff = align_up(ML.bytes, 256);
  KV_TRY(entry_reserve(E, roff + RL.bytes));
  uint8_t* h = static_cast<uint8_t*>(E.host);
  uint8_t* dv = static_cast<uint8_t*>(E.dev);
  if (match_table) write_match(h, ML, items);
  const MatchResultDev* gres = items.empty() ? nullptr
                                             : reinterpret_cast<const MatchResultDev*>(dv + ML.hdr.res_off);
  if (!hs.empty()) write_realign(h + roff, dv + roff, RL, hs, gres);
  KV_CUDA(cudaMemcpyAsync(dv, h, hs.empty() ? ML.bytes : roff + size_t(RL.hdr.cs_off), cudaMemcpyHostToDevice, s));
  if (match_table) {
    if (pl->ev_mbefore) KV_CUDA(cudaEventRecord(pl->ev_mbefore, s));
    KV_CUDA(launch_match_dist(dv, ML.hdr, ML.smem, s));
    if (pl->ev_mafter) KV_CUDA(cudaEventRecord(pl->ev_mafter, s));
    g_launches += 1;
  }
  pl->pML = ML;
  pl->pRL = RL;
  pl->proff = roff;
  pl->n_items = items.size();
  pl->n_hs = hs.size();
  pl->pending = true;
  return ok();
}

// Second half: d̄ / w̄ / H / verdict (chunk + finalize), then the gated realign.
static kvcomm_status plan_end(kvcomm_plan_s* pl, int32_t sync, cudaStream_t s) {
  if (!pl->pending) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "plan run not begun (call kvcomm_plan_run_begin)");
  pl->pending = false;
  DeviceGuard guard(pl->dev);
  RingEntry& E = pl->tab[pl->next];
  uint8_t* h = static_cast<uint8_t*>(E.host);
  uint8_t* dv = static_cast<uint8_t*>(E.dev);
  const MatchLayout& ML = pl->pML;
  const RealignLayout& RL = pl->pRL;
  const size_t roff = pl->proff;
  // the realign kernel's stream: the run's own, or the plan's realign stream (pipelined
  // runs: this run's matching, reduction and prep on s overlap the previous run's realign
  // on rs; the realign waits for this run's prep through ev_prep)
  const bool split = pl->rstream_set;
  cudaStream_t rs = split ? pl->rstream : s;
  const int par = pl->next;
  if (pl->n_items) {
    KV_CUDA(launch_match_reduce(dv, ML.hdr, s));
    g_launches += 2;
    KV_CUDA(cudaMemcpyAsync(h + ML.hdr.res_off, dv + ML.hdr.res_off, ML.bytes - size_t(ML.hdr.res_off),
                            cudaMemcpyDeviceToHost, s));
  }
  const bool realign = pl->n_hs && RL.hdr.n_seg > 0;
  if (realign) {
    KV_CUDA(launch_realign_prep(dv + roff, RL.hdr, s));
    g_launches += 1;
  }
  if (split) {
    if (!pl->ev_prep[par]) KV_CUDA(cudaEventCreateWithFlags(&pl->ev_prep[par], cudaEventDisableTiming));
    KV_CUDA(cudaEventRecord(pl->ev_prep[par], s));
    KV_CUDA(cudaStreamWaitEvent(rs, pl->ev_prep[par], 0));
  }
  if (pl->ev_before) KV_CUDA(cudaEventRecord(pl->ev_before, rs));  // brackets the realign kernel alone
  if (realign && RL.hdr.total_units > 0) {
    KV_CUDA(launch_realign_main(dv + roff, RL.hdr, grid_for_device(pl->dev), rs));
    g_launches += 1;
  }
  if (pl->ev_after) KV_CUDA(cudaEventRecord(pl->ev_after, rs));
  KV_CUDA(cudaEventRecord(E.done, rs));
  E.used = true;
  pl->res_off = pl->n_items ? ML.hdr.res_off : -1;
  pl->last = pl->next;
  pl->next ^= 1;
  if (sync) KV_CUDA(cudaEventSynchronize(E.done));
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_plan_run(kvcomm_plan_t pl, const void* const* query_embs, int32_t sync,
                                         void* stream) {
  NvtxRange nvtx_("kvcomm_plan_run");
  if (!pl || !query_embs) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null plan/queries");
  std::lock_guard<std::mutex> plk(pl->mu);
  if (pl->world > 1)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "sharded plan: use kvcomm_plan_run_begin / sync / kvcomm_plan_run_end");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  KV_TRY(plan_begin(pl, query_embs, s));
  return plan_end(pl, sync, s);
}

KVCOMM_API kvcomm_status kvcomm_plan_run_begin(kvcomm_plan_t pl, const void* const* query_embs, void* stream) {
  NvtxRange nvtx_("kvcomm_plan_run_begin");
  if (!pl || !query_embs) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null plan/queries");
  std::lock_guard<std::mutex> plk(pl->mu);
  return plan_begin(pl, query_embs, static_cast<cudaStream_t>(stream));
}

KVCOMM_API kvcomm_status kvcomm_plan_run_end(kvcomm_plan_t pl, int32_t sync, void* stream) {
  NvtxRange nvtx_("kvcomm_plan_run_end");
  if (!pl) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null plan");
  std::lock_guard<std::mutex> plk(pl->mu);
  return plan_end(pl, sync, static_cast<cudaStream_t>(stream));
}

KVCOMM_API kvcomm_status kvcomm_plan_results(kvcomm_plan_t pl, kvcomm_match_info* infos, int32_t* agent_reused) {
  if (!pl) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null plan");
  std::lock_guard<std::mutex> plk(pl->mu);
  if (pl->last < 0) return fail(KVCOMM_ERR_NOT_FOUND, "plan has not run");
  RingEntry& E = pl->tab[pl->last];
  KV_CUDA(cudaEventSynchronize(E.done));
  const int nm = int(pl->matches.size());
  bool mismatch = false;
  if (pl->res_off >= 0) {
    const MatchResultDev* res = reinterpret_cast<const MatchResultDev*>(static_cast<uint8_t*>(E.host) + pl->res_off);
    for (int i = 0; i < nm; ++i)
      if (pl->job_of[i] >= 0) {
        fill_info_from_result(&pl->infos[i], res[pl->job_of[i]]);
        mismatch |= res[pl->job_of[i]].shard_mismatch != 0;
      }
  }
  if (infos)
    for (int i = 0; i < nm; ++i) infos[i] = pl->infos[i];
  if (agent_reused)
    for (size_t a = 0; a < pl->agents.size(); ++a) {
      bool okk = pl->agent_state[a] == 0;
      for (int mi : pl->agent_matches[a]) okk &= pl->infos[mi].verdict == KVCOMM_SHAREABLE;
      agent_reused[a] = okk ? 1 : 0;
    }
  if (mismatch)
    return fail(KVCOMM_ERR_SHAPE_MISMATCH,
                "sharded matching: the ranks matched different candidate sets or lengths (pools out of step); "
                "those agents were not realigned");
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_plan_set_events(kvcomm_plan_t pl, void* before_realign, void* after_realign) {
  if (!pl) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null plan");
  std::lock_guard<std::mutex> plk(pl->mu);
  pl->ev_before = static_cast<cudaEvent_t>(before_realign);
  pl->ev_after = static_cast<cudaEvent_t>(after_realign);
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_plan_set_realign_stream(kvcomm_plan_t pl, void* stream, int32_t enable) {
  if (!pl) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null plan");
  std::lock_guard<std::mutex> plk(pl->mu);
  if (pl->pending) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "a run is in progress (between run_begin and run_end)");
  pl->rstream = static_cast<cudaStream_t>(stream);
  pl->rstream_set = enable != 0;
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_plan_set_match_events(kvcomm_plan_t pl, void* before_match, void* after_match) {
  if (!pl) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null plan");
  std::lock_guard<std::mutex> plk(pl->mu);
  pl->ev_mbefore = static_cast<cudaEvent_t>(before_match);
  pl->ev_mafter = static_cast<cudaEvent_t>(after_match);
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_plan_weights(kvcomm_plan_t pl, int32_t match, const float** W, int64_t* ld_w,
                                             const float** wbar) {
  if (!pl || match < 0 || match >= int32_t(pl->matches.size())) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "bad match");
  std::lock_guard<std::mutex> plk(pl->mu);
  const int par = pl->last >= 0 ? pl->last : 0;  // the last run's buffers
  if (W) *W = pl->W(par, match);
  if (ld_w) *ld_w = pl->ld_w[match];
  if (wbar) *wbar = pl->wbar(par, match);
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_plan_match_handle(kvcomm_plan_t pl, kvcomm_ipc_handle* handle, int64_t* bytes) {
  if (!pl || !handle) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null plan/handle");
  std::lock_guard<std::mutex> plk(pl->mu);
  DeviceGuard guard(pl->dev);
  cudaIpcMemHandle_t h;
  KV_CUDA(cudaIpcGetMemHandle(&h, pl->xbuf));
  std::memcpy(handle->bytes, &h, sizeof(h));
  if (bytes) *bytes = pl->xbytes;
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_plan_match_shard(kvcomm_plan_t pl, int32_t rank, int32_t world,
                                                 const kvcomm_ipc_handle* handles) {
  if (!pl) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null plan");
  if (world < 1 || world > kMaxMatchPeers + 1 || rank < 0 || rank >= world)
    return fail(KVCOMM_ERR_INVALID_ARGUMENT, "rank %d / world %d (world <= %d)", rank, world, kMaxMatchPeers + 1);
  if (world > 1 && !handles) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "null handles");
  std::lock_guard<std::mutex> plk(pl->mu);
  if (pl->pending) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "plan run in progress");
  DeviceGuard guard(pl->dev);
  for (auto& e : pl->tab)  // no run may still read the old mappings
    if (e.used) KV_CUDA(cudaEventSynchronize(e.done));
  plan_close_peers(pl);
  pl->next = 0;  // every rank's runs use buffer parity 0, 1, 0, ... in lockstep from here
  if (world == 1) return ok();
  for (int r = 0; r < world; ++r) {
    if (r == rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles[r].bytes, sizeof(h));
    void* x = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&x, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      plan_close_peers(pl);
      return fail(KVCOMM_ERR_CUDA, "rank %d: opening peer %d's match buffers: %s", rank, r, cudaGetErrorString(e));
    }
    pl->peer_x.push_back(static_cast<char*>(x));
  }
  pl->rank = rank;
  pl->world = world;
  return ok();
}

// ---- fused gather: IPC-shared destinations ------------------------------------
static_assert(sizeof(kvcomm_ipc_handle) == sizeof(cudaIpcMemHandle_t), "ipc handle size");

KVCOMM_API kvcomm_status kvcomm_ipc_alloc(int32_t device, int64_t bytes, void** ptr, kvcomm_ipc_handle* handle) {
  if (!ptr || !handle || bytes <= 0) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "bad ipc_alloc arguments");
  DeviceGuard guard(device);
  *ptr = nullptr;
  cudaError_t e = cudaMalloc(ptr, size_t(bytes));
  if (e != cudaSuccess) {
    cudaGetLastError();
    *ptr = nullptr;
    return fail(e == cudaErrorMemoryAllocation ? KVCOMM_ERR_OUT_OF_MEMORY : KVCOMM_ERR_CUDA, "ipc_alloc %lld bytes: %s",
                (long long)bytes, cudaGetErrorString(e));
  }
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, *ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    cudaFree(*ptr);
    *ptr = nullptr;
    return fail(KVCOMM_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  }
  std::memcpy(handle->bytes, &h, sizeof(h));
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_ipc_free(void* ptr) {
  if (!ptr) return ok();
  KV_CUDA(cudaFree(ptr));
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_ipc_open(int32_t device, const kvcomm_ipc_handle* handle, void** ptr) {
  if (!ptr || !handle) return fail(KVCOMM_ERR_INVALID_ARGUMENT, "bad ipc_open arguments");
  DeviceGuard guard(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle->bytes, sizeof(h));
  *ptr = nullptr;
  KV_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return ok();
}

KVCOMM_API kvcomm_status kvcomm_ipc_close(void* ptr) {
  if (!ptr) return ok();
  KV_CUDA(cudaIpcCloseMemHandle(ptr));
  return ok();
}

}  // extern "C"
