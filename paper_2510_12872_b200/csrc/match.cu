// Anchor matching (SURVEY §8(a) a2+a3; Eq. 5, Eq. 6):
//
//   d[i,j]  = ‖h_φ[i] - h_ψj[i]‖₂          i < L_φ, ψ_j ∈ 𝒜_φ (first L_φ rows, reading A8)
//   W[j][i] = softmax_j(-d[i,j])            per position (reading A2); optional top-k (A16)
//   d̄_j     = sqrt(Σ_i d[i,j]²)            Frobenius (reading A4; or mean_i d[i,j])
//   (cosine variant, Table A.4: d = 1 - cos per position, d̄ = 1 - <h_φ,h_ψ>_F/(‖h_φ‖_F‖h_ψ‖_F))
//   w̄ = softmax(-d̄),  H = -Σ w̄ log w̄,  NewAnchor ⇔ H > γ log|𝒜_φ|
//
// One launch covers every (sample, pool) job of a request: blocks of P positions of
// every job, then one finalize block per job.
//
// Numerics: each lane forms 8 differences of bf16 values in fp32 (exact unless the
// exponents are >16 binades apart), squares/accumulates those 8 with fp32 FMA
// (relative error <= 8·2^-24 on a sum of positive terms), and adds the partials in
// fp64.  The resulting distance has a relative error below 3e-7, inside the 1e-6
// tie band of the parity contract.  Softmax, sums and entropy run in fp64 with
// fixed-order reductions, so the verdict is deterministic run to run.
//
// Why not tensor cores: the distance compares row i of φ only with row i of each
// anchor (a batched GEMV, ~0.5 FLOP/byte) — it is HBM-bound, not a dense GEMM, and
// the ‖a‖²+‖b‖²-2a·b expansion would cancel catastrophically near ties.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdlib>
#include <cfloat>
#include <algorithm>
#include "kvcomm_internal.h"
#include "ptx.cuh"

namespace kvc {

constexpr int kMatchThreads = 256;
constexpr int kMatchWarps = kMatchThreads / 32;
constexpr double kTieRel = 1e-6;
#ifndef KVC_MATCH_UNROLL
#define KVC_MATCH_UNROLL 8
#endif
constexpr int kMatchUnroll = KVC_MATCH_UNROLL;
// Two instantiations of the distance kernel by D_e (measured, profiles/r02g_match_ctas.txt):
// rows of D_e <= kMatchWideDe (8 KiB at 4096) run 6 CTAs per SM at 40 registers (config 2:
// 120 -> 104 us); longer rows keep the unbounded 110-register build at 2 CTAs per SM,
// whose warps hold more loads in flight (config 4: 2.02 ms vs 2.23-3.45 ms at 2-6 CTAs of
// the 40-register build).
constexpr int kMatchWideDe = 4096;
#ifndef KVC_MATCH_L2PF
#define KVC_MATCH_L2PF 0  // TMA L2 prefetch of each warp's next anchor row (measurement knob)
#endif
#ifndef KVC_MATCH_PROBE_NOTAIL
#define KVC_MATCH_PROBE_NOTAIL 0
#endif
#ifndef KVC_MATCH_MINB
#define KVC_MATCH_MINB 6
#endif  // 16-byte anchor loads in flight per lane (8 vs 4: match 2-5 % faster)

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// (d, slot) lexicographic "less than"
__device__ __forceinline__ bool key_less(double da, int sa, double db, int sb) {
  return da < db || (da == db && sa < sb);
}

// Σ over 8 bf16 pairs of (q - a)²: exact fp32 differences (almost always: unless the
// exponents are > 16 binades apart) and squares accumulated with packed FADD2 / FFMA2 in
// two fp32 lanes (even / odd elements, 4 terms each), summed once at the end — 8 terms in
// fp32 as before, half the math instructions of scalar FADD + FFMA (measured: match 1 %
// faster; the kernel is bound by its loads, not its math).  KVC_MATCH_PACKED=0: scalar.
#ifndef KVC_MATCH_PACKED
#define KVC_MATCH_PACKED 1
#endif
__device__ __forceinline__ float sq_diff8(const uint4& qv, const uint4& av) {
  const uint32_t aw[4] = {av.x, av.y, av.z, av.w};
  const uint32_t qw[4] = {qv.x, qv.y, qv.z, qv.w};
  if (!KVC_MATCH_PACKED) {
    float part = 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float d0 = bf_lo(qw[t]) - bf_lo(aw[t]);
      const float d1 = bf_hi(qw[t]) - bf_hi(aw[t]);
      part = fmaf(d0, d0, part);
      part = fmaf(d1, d1, part);
    }
    return part;
  }
  float p0 = 0.f, p1 = 0.f;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    float d0, d1;
    fsub2(d0, d1, bf_lo(qw[t]), bf_hi(qw[t]), bf_lo(aw[t]), bf_hi(aw[t]));
    ffma2(p0, p1, d0, d1, d0, d1);
  }
  return p0 + p1;
}

// q·a, a·a, q·q over 8 bf16 pairs.  A product of two bf16 values is exact in fp32
// (8 + 8 significant bits); the products are summed in fp64, so 1 - cos keeps ~1e-12
// absolute accuracy and the 1e-6 relative tie band holds down to tiny distances (an
// fp32 running sum lost ~1e-7 absolute, > 1e-6 relative once 1 - cos < 0.1).
__device__ __forceinline__ void dots8(const uint4& qv, const uint4& av, double& qa, double& aa, double& qq) {
  const uint32_t aw[4] = {av.x, av.y, av.z, av.w};
  const uint32_t qw[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const float a0 = bf_lo(aw[t]), a1 = bf_hi(aw[t]), q0 = bf_lo(qw[t]), q1 = bf_hi(qw[t]);
    qa += double(q0 * a0) + double(q1 * a1);
    aa += double(a0 * a0) + double(a1 * a1);
    qq += double(q0 * q0) + double(q1 * q1);
  }
}

__device__ __forceinline__ int find_job(const MatchJob* jobs, int n, int b) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].block_begin <= b) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void match_tail(const MatchJob& a, int jb, int lb, int i0, int np, const double* sd,
                                           const double* s_qa, const double* s_aa, const double* s_qq,
                                           const int32_t* cand, const int32_t* slot2cand, int32_t* ties, int warp,
                                           int lane, int tid);

// One work item = P consecutive positions of one job.
__device__ __forceinline__ void match_item(const uint8_t* __restrict__ tab, const int item) {
  const MatchHdr* hdr = reinterpret_cast<const MatchHdr*>(tab);
  const MatchJob* jobs = reinterpret_cast<const MatchJob*>(tab + hdr->job_off);
  const int32_t* ints = reinterpret_cast<const int32_t*>(tab + hdr->int_off);
  int32_t* ties = reinterpret_cast<int32_t*>(const_cast<uint8_t*>(tab) + hdr->tie_off);
  const int jb = find_job(jobs, hdr->n_jobs, item);
  const MatchJob& a = jobs[jb];
  const int P = hdr->P;
  const int lb = a.own_lo + (item - a.block_begin) * a.own_step;  // position block (sharded: this rank's)
  const int32_t* cand = ints + a.cand_off;
  const int32_t* slot2cand = ints + a.s2c_off;

  extern __shared__ __align__(16) uint8_t smem[];
  const int De = a.De;
  const int n_cand = a.n_cand;
  bf16* q = reinterpret_cast<bf16*>(smem);
  double* sd = reinterpret_cast<double*>(smem + ((size_t(P) * De * 2 + 15) & ~size_t(15)));
  double* s_qa = sd + P * n_cand;      // cosine only: Σ q·a, Σ a·a per (position, candidate), Σ q·q
  double* s_aa = s_qa + P * n_cand;
  double* s_qq = s_aa + P * n_cand;
  const int i0 = lb * P;
  const int np = min(P, a.L_phi - i0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // stage the query rows of this block's positions
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.query + size_t(i0) * De);
    uint4* dst = reinterpret_cast<uint4*>(q);
    const int nvec = np * De / 8;
    for (int x = threadIdx.x; x < nvec; x += kMatchThreads) dst[x] = src[x];
  }
  __syncthreads();

  // distances: one warp per (position, candidate) task
  const int ntask = np * n_cand;
  // anchor row of task t: row i0 + p of candidate j; a pool holding only this rank's blocks
  // stores block lb at lb / G
  auto task_row = [&](int t) {
    const int p = t / n_cand;
    const int j = t - p * n_cand;
    const int64_t erow = a.emb_world > 1 ? int64_t(lb / a.emb_world) * P + p : int64_t(i0 + p);
    return a.emb + int64_t(cand[j]) * a.slot_stride + erow * De;
  };
  if (KVC_MATCH_L2PF && lane == 0 && warp < ntask) bulk_prefetch_l2(task_row(warp), uint32_t(De) * 2u);
  for (int task = warp; task < ntask; task += kMatchWarps) {
    const int p = task / n_cand;
    const int j = task - p * n_cand;
    const bf16* arow = task_row(task);
    // this warp's next row streams into L2 by TMA while the warp reduces this one
    if (KVC_MATCH_L2PF && lane == 0 && task + kMatchWarps < ntask)
      bulk_prefetch_l2(task_row(task + kMatchWarps), uint32_t(De) * 2u);
    const bf16* qrow = q + size_t(p) * De;
    if (!a.cosine) {
      double s = 0.0;
      int e = lane * 8;
      for (; e + (kMatchUnroll - 1) * 256 < De; e += kMatchUnroll * 256) {  // independent 16-byte loads in flight
        uint4 av[kMatchUnroll];
#pragma unroll
        for (int r = 0; r < kMatchUnroll; ++r) av[r] = ldg128_nc(arow + e + r * 256);
#pragma unroll
        for (int r = 0; r < kMatchUnroll; ++r) s += double(sq_diff8(lds128(qrow + e + r * 256), av[r]));
      }
      for (; e < De; e += 256) s += double(sq_diff8(lds128(qrow + e), ldg128_nc(arow + e)));
      s = warp_sum_d(s);
      if (lane == 0) sd[p * n_cand + j] = sqrt(s);
    } else {
      double qa = 0.0, aa = 0.0, qq = 0.0;
      for (int e = lane * 8; e < De; e += 256) {
        dots8(lds128(qrow + e), ldg128_nc(arow + e), qa, aa, qq);
      }
      qa = warp_sum_d(qa);
      aa = warp_sum_d(aa);
      qq = warp_sum_d(qq);
      if (lane == 0) {
        const double den = sqrt(qq * aa);
        sd[p * n_cand + j] = 1.0 - (den > 0.0 ? qa / den : 0.0);
        s_qa[p * n_cand + j] = qa;
        s_aa[p * n_cand + j] = aa;
        if (j == 0) s_qq[p] = qq;
      }
    }
  }
  __syncthreads();
#if KVC_MATCH_PROBE_NOTAIL  // bandwidth probe only (wrong results): the loads and distances without the tail
  if (np < 0)
#endif
  match_tail(a, jb, lb, i0, np, sd, s_qa, s_aa, s_qq, cand, slot2cand, ties, warp, lane, threadIdx.x);
}

// Per-position weights (Eq. 6 / top-k) and the block's deterministic partial sums of
// d̄, from this block's distances sd[p * n_cand + j] (both distance kernels end here).
// 8 warps (threads 0..255) take part; no block-level barrier inside.
__device__ __forceinline__ void match_tail(const MatchJob& a, int jb, int lb, int i0, int np, const double* sd,
                                           const double* s_qa, const double* s_aa, const double* s_qq,
                                           const int32_t* cand, const int32_t* slot2cand, int32_t* ties, int warp,
                                           int lane, int tid) {
  const int n_cand = a.n_cand;
  // per-position weights (one warp per position)
  for (int p = warp; p < np; p += kMatchWarps) {
    const int i = i0 + p;
    const double* dr = sd + p * n_cand;
    if (a.dist_user)
      for (int j = lane; j < n_cand; j += 32) a.dist_user[int64_t(cand[j]) * a.ld_w + i] = dr[j];
    if (a.top_k <= 0) {
      double mn = DBL_MAX;
      for (int j = lane; j < n_cand; j += 32) mn = fmin(mn, dr[j]);
      mn = warp_min_d(mn);
      double sum = 0.0;
      for (int j = lane; j < n_cand; j += 32) sum += exp(-(dr[j] - mn));
      sum = warp_sum_d(sum);
      for (int sl = lane; sl < a.cap; sl += 32) {
        const int j = slot2cand[sl];
        const float w = j >= 0 ? float(exp(-(dr[j] - mn)) / sum) : 0.f;
        a.W[int64_t(sl) * a.ld_w + i] = w;
        const int64_t x = int64_t(i) * a.cap + sl;  // position-major exchange row: lanes contiguous
        for (int r = 0; r < a.n_peer; ++r) a.X_peer[r][x] = w;
      }
    } else {
      // top-k: k rounds of lexicographic (distance, slot) argmin over the unselected
      const int k = a.top_k;
      double sel_d = 0.0;  // lane r < k keeps the r-th selected distance / slot
      int sel_s = -1;
      double prev_d = -1.0;
      int prev_s = -1;
      bool tie = false;
      double last_d = 0.0;
      for (int r = 0; r <= k && r < n_cand; ++r) {
        double bd = DBL_MAX;
        int bs = INT32_MAX;
        for (int j = lane; j < n_cand; j += 32) {
          const double dj = dr[j];
          const int sj = cand[j];
          // unselected == strictly after (prev_d, prev_s) in the lexicographic order
          const bool after = (prev_s < 0) || key_less(prev_d, prev_s, dj, sj);
          if (after && key_less(dj, sj, bd, bs)) { bd = dj; bs = sj; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double od = __shfl_xor_sync(0xffffffffu, bd, o);
          const int os = __shfl_xor_sync(0xffffffffu, bs, o);
          if (key_less(od, os, bd, bs)) { bd = od; bs = os; }
        }
        if (r > 0 && (bd - last_d) <= kTieRel * fmax(bd, 1e-300)) tie = true;
        last_d = bd;
        if (r == k) break;  // the (k+1)-th only serves the boundary tie test
        if (lane == r) { sel_d = bd; sel_s = bs; }
        prev_d = bd;
        prev_s = bs;
      }
      const double mn = __shfl_sync(0xffffffffu, sel_d, 0);
      const double ev = (lane < k) ? exp(-(sel_d - mn)) : 0.0;
      const double sum = warp_sum_d(ev);
      for (int sl = lane; sl < a.cap; sl += 32) a.W[int64_t(sl) * a.ld_w + i] = 0.f;
      __syncwarp();
      if (lane < k) {
        a.W[int64_t(sel_s) * a.ld_w + i] = float(ev / sum);
        if (a.idx) a.idx[int64_t(i) * k + lane] = sel_s;
      }
      if (a.n_peer > 0) {  // peers receive the finished column: one store per address
        __syncwarp();
        for (int sl = lane; sl < a.cap; sl += 32) {
          const float w = a.W[int64_t(sl) * a.ld_w + i];
          for (int r = 0; r < a.n_peer; ++r) a.X_peer[r][int64_t(i) * a.cap + sl] = w;
        }
      }
      if (lane == 0 && tie) atomicAdd(&ties[jb], 1);  // sharded: this rank's positions only
    }
  }

  // deterministic per-block partial sums (Σ d² for Frobenius, Σ d for mean-ℓ2;
  // cosine: Σ q·a and Σ a·a per candidate, Σ q·q once)
  if (!a.cosine) {
    for (int j = tid; j < n_cand; j += kMatchThreads) {
      double s = 0.0;
      for (int p = 0; p < np; ++p) {
        const double dv = sd[p * n_cand + j];
        s += a.scalar_mode == 0 ? dv * dv : dv;
      }
      a.partial[int64_t(lb) * n_cand + j] = s;
      for (int r = 0; r < a.n_peer; ++r) a.partial_peer[r][int64_t(lb) * n_cand + j] = s;
    }
  } else {
    const int64_t stride = 2 * n_cand + 1;
    for (int j = tid; j < n_cand; j += kMatchThreads) {
      double sqa = 0.0, saa = 0.0;
      for (int p = 0; p < np; ++p) {
        sqa += s_qa[p * n_cand + j];
        saa += s_aa[p * n_cand + j];
      }
      a.partial[int64_t(lb) * stride + j] = sqa;
      a.partial[int64_t(lb) * stride + n_cand + j] = saa;
      for (int r = 0; r < a.n_peer; ++r) {
        a.partial_peer[r][int64_t(lb) * stride + j] = sqa;
        a.partial_peer[r][int64_t(lb) * stride + n_cand + j] = saa;
      }
    }
    if (tid == 0) {
      double sqq = 0.0;
      for (int p = 0; p < np; ++p) sqq += s_qq[p];
      a.partial[int64_t(lb) * stride + 2 * n_cand] = sqq;
      for (int r = 0; r < a.n_peer; ++r) a.partial_peer[r][int64_t(lb) * stride + 2 * n_cand] = sqq;
    }
  }
}

// Persistent blocks pull items from an atomic counter (the table's word after the
// per-job tie counters, zeroed by the host upload), so the last wave has no tail of
// idle SMs.  Sharded matching: the items are this rank's position blocks only.  The processing order does not affect any result: every item writes its
// own W columns and partial sums.
template <int kMinBlocks>
__global__ void __launch_bounds__(kMatchThreads, kMinBlocks) match_dist_kernel(const uint8_t* __restrict__ tab) {
  const MatchHdr* hdr = reinterpret_cast<const MatchHdr*>(tab);
  int32_t* counter = reinterpret_cast<int32_t*>(const_cast<uint8_t*>(tab) + hdr->tie_off) + hdr->n_jobs;
  __shared__ int s_item;
  if (hdr->shard_world > 1 && blockIdx.x == 0 && threadIdx.x == 0)
    for (int r = 0; r < hdr->shard_world; ++r) *hdr->fp_dst[r] = hdr->fingerprint;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= hdr->total_blocks) break;
    match_item(tab, item);
    __syncthreads();  // shared memory is reused by the next item
  }
  if (hdr->any_peer) __threadfence_system();  // peer stores visible before the caller's cross-rank sync
}

// ---- TMA-streamed distance kernel (l2 jobs) --------------------------------------
// Persistent CTAs of 8 consumer warps + 1 producer warp walk the work items (P = 2
// positions of one job) round-robin.  The producer's elected lane copies each item's
// query rows (one bulk copy into a double buffer) and, per candidate anchor, the
// anchor's P contiguous embedding rows (the same positions, reading A8) as 16 KiB
// chunks into a ring of stages (cp.async.bulk + mbarrier complete_tx, L2 evict-first),
// running ahead across items so the stream has no per-item bubble.  Consumer thread t
// keeps its query vectors of the item in registers (vectors g = c * 1024 + t + 256 k of
// the flattened [P][De] tile) and, per anchor, accumulates Σ (q - a)² per position with
// the same numerics as the register kernel (groups of 8 in fp32 FMA, fp64 beyond), warp-
// reduces, and stores one fp64 partial per (anchor, warp, position); the item's
// distances are the fixed-order sums of the 8 warp partials, so results are
// deterministic and independent of the grid (sharded ranks agree bit for bit).
constexpr int kMatchTmaVec = 8;  // query vectors per thread: P * De * 2 / (16 * 256) <= 8 at De 8192

__device__ __forceinline__ void match_tma_geom(const MatchHdr* hdr, const MatchJob* jobs, int item, int& jb,
                                               int& lb, int& i0, int& np) {
  jb = find_job(jobs, hdr->n_jobs, item);
  const MatchJob& a = jobs[jb];
  lb = a.own_lo + (item - a.block_begin) * a.own_step;
  i0 = lb * hdr->P;
  np = min(hdr->P, a.L_phi - i0);
}

__global__ void __launch_bounds__(kMatchThreads + 32, 1) match_dist_tma_kernel(const uint8_t* __restrict__ tab) {
  const MatchHdr* hdr = reinterpret_cast<const MatchHdr*>(tab);
  const MatchJob* jobs = reinterpret_cast<const MatchJob*>(tab + hdr->job_off);
  const int32_t* ints = reinterpret_cast<const int32_t*>(tab + hdr->int_off);
  int32_t* ties = reinterpret_cast<int32_t*>(const_cast<uint8_t*>(tab) + hdr->tie_off);
  const int NS = hdr->tma_stages, QB = hdr->tma_qbytes, CM = hdr->tma_cmax;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;                                                  // [NS][kMatchStageBytes]
  uint8_t* qbuf = ring + size_t(NS) * kMatchStageBytes;                  // [2][QB]
  double* part = reinterpret_cast<double*>(qbuf + 2 * size_t(QB));       // [CM][kMatchWarps][2]
  double* sd = part + size_t(CM) * kMatchWarps * 2;                      // [2][CM]
  uint64_t* full = reinterpret_cast<uint64_t*>(sd + 2 * size_t(CM));
  uint64_t* empty = full + NS;
  uint64_t* qfull = empty + NS;
  uint64_t* qempty = qfull + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kMatchThreads);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], 1);
    }
    fence_mbar_init();
  }
  if (hdr->shard_world > 1 && blockIdx.x == 0 && threadIdx.x == 0)
    for (int r = 0; r < hdr->shard_world; ++r) *hdr->fp_dst[r] = hdr->fingerprint;
  __syncthreads();
  const int total = hdr->total_blocks;

  if (warp == kMatchWarps) {
    // ---------------- TMA producer (one lane) ----------------
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();
      int stage = 0, qb = 0;
      uint32_t phase = 0, qphase = 0;
      for (int item = blockIdx.x; item < total; item += gridDim.x) {
        int jb, lb, i0, np;
        match_tma_geom(hdr, jobs, item, jb, lb, i0, np);
        const MatchJob& a = jobs[jb];
        const uint32_t tile = uint32_t(np) * uint32_t(a.De) * 2u;
        mbar_wait(&qempty[qb], qphase ^ 1u);
        mbar_arrive_expect_tx(&qfull[qb], tile);
        bulk_g2s(qbuf + size_t(qb) * QB, a.query + int64_t(i0) * a.De, tile, &qfull[qb], pol_stream);
        if (++qb == 2) { qb = 0; qphase ^= 1u; }
        const int32_t* cand = ints + a.cand_off;
        const int64_t erow = a.emb_world > 1 ? int64_t(lb / a.emb_world) * hdr->P : int64_t(i0);
        for (int j = 0; j < a.n_cand; ++j) {
          const uint8_t* src = reinterpret_cast<const uint8_t*>(a.emb + int64_t(cand[j]) * a.slot_stride + erow * a.De);
          for (uint32_t off = 0; off < tile; off += kMatchStageBytes) {
            const uint32_t bytes = min(uint32_t(kMatchStageBytes), tile - off);
            mbar_wait(&empty[stage], phase ^ 1u);
            mbar_arrive_expect_tx(&full[stage], bytes);
            bulk_g2s(ring + size_t(stage) * kMatchStageBytes, src + off, bytes, &full[stage], pol_stream);
            if (++stage == NS) { stage = 0; phase ^= 1u; }
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers (threads 0..255) ----------------
  const int tid = threadIdx.x;
  int stage = 0, qb = 0;
  uint32_t phase = 0, qphase = 0;
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    int jb, lb, i0, np;
    match_tma_geom(hdr, jobs, item, jb, lb, i0, np);
    const MatchJob& a = jobs[jb];
    const int De = a.De;
    const int n_cand = a.n_cand;
    const int tile_vec = np * De / 8;                    // 16-byte vectors of the [np][De] tile
    const int chunks = (tile_vec + 1023) / 1024;         // 16 KiB chunks per anchor
    mbar_wait(&qfull[qb], qphase);
    const uint8_t* qsm = qbuf + size_t(qb) * QB;
    uint4 qv[kMatchTmaVec];
    int qpos = 0;                                        // bit v: vector v lies in position 1
#pragma unroll
    for (int v = 0; v < kMatchTmaVec; ++v) {
      const int g = (v >> 2) * 1024 + tid + 256 * (v & 3);
      qv[v] = g < tile_vec ? lds128(qsm + size_t(g) * 16) : make_uint4(0, 0, 0, 0);
      qpos |= (g * 8 >= De ? 1 : 0) << v;
    }
    named_bar_sync(1, kMatchThreads);                   // every consumer holds its query vectors
    if (tid == 0) mbar_arrive(&qempty[qb]);              // the producer may refill this buffer
    if (++qb == 2) { qb = 0; qphase ^= 1u; }
    for (int j = 0; j < n_cand; ++j) {
      double acc0 = 0.0, acc1 = 0.0;
      for (int c = 0; c < chunks; ++c) {
        mbar_wait(&full[stage], phase);
        const uint8_t* buf = ring + size_t(stage) * kMatchStageBytes;
        float part8[4];
        bool has[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int g = c * 1024 + tid + 256 * k;
          has[k] = g < tile_vec;
          part8[k] = 0.f;
        }
        uint4 av[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          av[k] = has[k] ? lds128(buf + size_t(tid + 256 * k) * 16) : make_uint4(0, 0, 0, 0);
        mbar_arrive(&empty[stage]);                      // this thread's reads of the stage are done
        if (++stage == NS) { stage = 0; phase ^= 1u; }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
          for (int cc = 0; cc < kMatchTmaVec / 4; ++cc) {  // select the query vector of chunk c (unrolled)
            if (cc == c && has[k]) {
              part8[k] = sq_diff8(qv[cc * 4 + k], av[k]);
              if ((qpos >> (cc * 4 + k)) & 1) acc1 += double(part8[k]); else acc0 += double(part8[k]);
            }
          }
        }
      }
      acc0 = warp_sum_d(acc0);
      acc1 = warp_sum_d(acc1);
      if (lane == 0) {
        part[(size_t(j) * kMatchWarps + warp) * 2] = acc0;
        part[(size_t(j) * kMatchWarps + warp) * 2 + 1] = acc1;
      }
    }
    named_bar_sync(1, kMatchThreads);                   // all warp partials of the item are in place
    for (int t = tid; t < np * n_cand; t += kMatchThreads) {
      const int p = t / n_cand, j = t - p * n_cand;
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kMatchWarps; ++w) s += part[(size_t(j) * kMatchWarps + w) * 2 + p];
      sd[p * n_cand + j] = sqrt(s);
    }
    named_bar_sync(1, kMatchThreads);
    match_tail(a, jb, lb, i0, np, sd, nullptr, nullptr, nullptr, ints + a.cand_off, ints + a.s2c_off, ties, warp,
               lane, tid);
    named_bar_sync(1, kMatchThreads);                   // sd / part are reused by the next item
  }
  if (hdr->any_peer) __threadfence_system();
}

// ---- row-ring distance kernel (l2 jobs; round 2) ----------------------------------
// The register kernel's task model (one warp reduces one whole anchor row of one position)
// fed by TMA instead of per-lane loads, so the bytes in flight are bounded by a shared-memory
// ring, not by registers or the LSU's outstanding misses.  One persistent CTA per SM of 8
// consumer warps + 1 producer warp walks the work items (P positions of one job)
// round-robin.  The producer's elected lane copies the item's query rows into a double
// buffer and then, for every task (candidate j, position p) of the item in order, the
// anchor's row into the next ring stage (one cp.async.bulk of D_e x 2 bytes, L2
// evict-first).  Tasks are numbered across items; consumer warp w takes the tasks
// g = w (mod 8), so its ring stage advances by 8 per task.  Per task the warp computes the
// distance exactly as the register kernel does (lane-strided 16-byte vectors, groups of 8
// in fp32 with packed FADD2 / FFMA2, fp64 accumulation in the same order, the same
// butterfly), so both kernels give bit-identical distances; lane 0 releases the stage.
// The item's distances go to one of two sd buffers; after a consumer-only barrier the 8
// warps run the same tail (per-position weights, partial sums) as the register kernel
// while the producer streams the next item.
// Consumer warps of the row-ring kernel.  The ring depth must be a multiple of it (host,
// layout_match): task g + NS reuses task g's stage, and the parity wait is only safe if the
// same warp, in order, consumes both (another warp could otherwise see task g's completed
// phase as its own).  16 warps measured 117 us at config 2 (8: 121 us; register kernel 103).
constexpr int kRingWarps = kMatchRingWarps;
__global__ void __launch_bounds__(kRingWarps * 32 + 32, 1) match_dist_ring_kernel(const uint8_t* __restrict__ tab) {
  const MatchHdr* hdr = reinterpret_cast<const MatchHdr*>(tab);
  const MatchJob* jobs = reinterpret_cast<const MatchJob*>(tab + hdr->job_off);
  const int32_t* ints = reinterpret_cast<const int32_t*>(tab + hdr->int_off);
  int32_t* ties = reinterpret_cast<int32_t*>(const_cast<uint8_t*>(tab) + hdr->tie_off);
  const int NS = hdr->tma_stages, QB = hdr->tma_qbytes, CM = hdr->tma_cmax, RB = hdr->ring_row_bytes;
  const int P = hdr->P;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;                                                  // [NS][RB]
  uint8_t* qbuf = ring + size_t(NS) * RB;                                // [2][QB]
  double* sdb = reinterpret_cast<double*>(qbuf + 2 * size_t(QB));        // [2][P * CM]
  uint64_t* full = reinterpret_cast<uint64_t*>(sdb + 2 * size_t(P) * CM);
  uint64_t* empty = full + NS;
  uint64_t* qfull = empty + NS;
  uint64_t* qempty = qfull + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);           // lane 0 of the consuming warp, after __syncwarp
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], 1);
    }
    fence_mbar_init();
  }
  if (hdr->shard_world > 1 && blockIdx.x == 0 && threadIdx.x == 0)
    for (int r = 0; r < hdr->shard_world; ++r) *hdr->fp_dst[r] = hdr->fingerprint;
  __syncthreads();
  const int total = hdr->total_blocks;

  if (warp == kRingWarps) {
    // ---------------- TMA producer (one lane) ----------------
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();
      int stage = 0, qb = 0;
      uint32_t phase = 0, qphase = 0;
      for (int item = blockIdx.x; item < total; item += gridDim.x) {
        int jb, lb, i0, np;
        match_tma_geom(hdr, jobs, item, jb, lb, i0, np);
        const MatchJob& a = jobs[jb];
        const uint32_t row = uint32_t(a.De) * 2u;
        mbar_wait(&qempty[qb], qphase ^ 1u);
        mbar_arrive_expect_tx(&qfull[qb], uint32_t(np) * row);
        bulk_g2s(qbuf + size_t(qb) * QB, a.query + int64_t(i0) * a.De, uint32_t(np) * row, &qfull[qb], pol_stream);
        if (++qb == 2) { qb = 0; qphase ^= 1u; }
        const int32_t* cand = ints + a.cand_off;
        const int64_t erow = a.emb_world > 1 ? int64_t(lb / a.emb_world) * P : int64_t(i0);
        for (int j = 0; j < a.n_cand; ++j) {
          const bf16* src = a.emb + int64_t(cand[j]) * a.slot_stride + erow * a.De;
          for (int p = 0; p < np; ++p) {
            mbar_wait(&empty[stage], phase ^ 1u);
            mbar_arrive_expect_tx(&full[stage], row);
            bulk_g2s(ring + size_t(stage) * RB, src + int64_t(p) * a.De, row, &full[stage], pol_stream);
            if (++stage == NS) { stage = 0; phase ^= 1u; }
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers (threads 0 .. kRingWarps * 32 - 1) ----------------
  const int tid = threadIdx.x;
  int64_t gbase = 0;               // tasks of all earlier items of this CTA
  int stage = warp % NS;           // stage and phase of this warp's next task g = warp + kRingWarps k
  uint32_t phase = uint32_t((warp / NS) & 1);
  int64_t gnext = warp;
  int qb = 0, sb = 0;
  uint32_t qphase = 0;
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    int jb, lb, i0, np;
    match_tma_geom(hdr, jobs, item, jb, lb, i0, np);
    const MatchJob& a = jobs[jb];
    const int De = a.De;
    const int n_cand = a.n_cand;
    const int ntask = n_cand * np;
    double* sd = sdb + size_t(sb) * P * CM;
    mbar_wait(&qfull[qb], qphase);
    const bf16* qsm = reinterpret_cast<const bf16*>(qbuf + size_t(qb) * QB);
    for (; gnext < gbase + ntask; gnext += kRingWarps) {
      const int t = int(gnext - gbase);
      const int j = t / np, p = t - j * np;
      mbar_wait(&full[stage], phase);
      const bf16* arow = reinterpret_cast<const bf16*>(ring + size_t(stage) * RB);
      const bf16* qrow = qsm + size_t(p) * De;
      double sacc = 0.0;
      for (int e = lane * 8; e < De; e += 256) sacc += double(sq_diff8(lds128(qrow + e), lds128(arow + e)));
      sacc = warp_sum_d(sacc);
      __syncwarp();
      if (lane == 0) {
        sd[p * n_cand + j] = sqrt(sacc);
        mbar_arrive(&empty[stage]);    // the whole warp's reads of the stage are done (__syncwarp)
      }
      stage += kRingWarps;
      while (stage >= NS) { stage -= NS; phase ^= 1u; }
    }
    gbase += ntask;
    named_bar_sync(1, kRingWarps * 32);                 // the item's distances are in sd
    if (tid == 0) mbar_arrive(&qempty[qb]);              // the producer may refill this query buffer
    if (++qb == 2) { qb = 0; qphase ^= 1u; }
    if (warp < kMatchWarps)                              // the tail is written for 8 warps
      match_tail(a, jb, lb, i0, np, sd, nullptr, nullptr, nullptr, ints + a.cand_off, ints + a.s2c_off, ties, warp,
                 lane, tid);
    sb ^= 1;  // the next item writes the other sd buffer; the barrier of the item after it
              // orders every warp's tail of this item before this buffer is written again
  }
  if (hdr->any_peer) __threadfence_system();
}

size_t match_ring_smem(int stages, int row_bytes, int qbytes, int cmax, int P) {
  return size_t(stages) * row_bytes + 2 * size_t(qbytes) + 2 * size_t(P) * cmax * sizeof(double) +
         (2 * size_t(stages) + 4) * sizeof(uint64_t);
}

size_t match_tma_smem(int stages, int qbytes, int cmax) {
  return size_t(stages) * kMatchStageBytes + 2 * size_t(qbytes) + size_t(cmax) * kMatchWarps * 2 * sizeof(double) +
         2 * size_t(cmax) * sizeof(double) + (2 * size_t(stages) + 4) * sizeof(uint64_t);
}

// First pass of d̄ (and the cosine sums): block (job, c) sums position blocks
// [c*per, (c+1)*per) of every partial column in order (4 interleaved accumulators,
// combined in order) into chunk row c.  Columns are coalesced across threads.  Sharded
// runs also copy the peers' W columns of those blocks from the exchange rows X into W.
__global__ void __launch_bounds__(256) match_chunk_kernel(const uint8_t* __restrict__ tab) {
  const MatchHdr* hdr = reinterpret_cast<const MatchHdr*>(tab);
  const MatchJob& a = reinterpret_cast<const MatchJob*>(tab + hdr->job_off)[blockIdx.x];
  const int c = blockIdx.y;
  const int per = (a.n_blocks + kMatchChunks - 1) / kMatchChunks;
  const int b0 = c * per, b1 = min(a.n_blocks, b0 + per);
  const int stride = a.cosine ? 2 * a.n_cand + 1 : a.n_cand;
  if (a.n_peer > 0) {
    // sharded: W columns of the positions this rank does not own arrived position-major in X
    // (peers' distance kernels, ordered before this launch by the caller's cross-rank barrier)
    const int P = hdr->P;
    for (int b = b0 + int(threadIdx.x >> 5); b < b1; b += blockDim.x >> 5) {
      if (b >= a.own_lo && (b - a.own_lo) % a.own_step == 0) continue;  // own block: W written locally
      const int i1 = min(a.L_phi, (b + 1) * P);
      for (int i = b * P; i < i1; ++i)
        for (int sl = int(threadIdx.x & 31); sl < a.cap; sl += 32)
          a.W[int64_t(sl) * a.ld_w + i] = a.X[int64_t(i) * a.cap + sl];
    }
  }
  for (int col = threadIdx.x; col < stride; col += blockDim.x) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    int b = b0;
    for (; b + 4 <= b1; b += 4) {
#pragma unroll
      for (int k = 0; k < 4; ++k) s[k] += a.partial[int64_t(b + k) * stride + col];
    }
    if (b < b1) s[0] += a.partial[int64_t(b) * stride + col];
    if (b + 1 < b1) s[1] += a.partial[int64_t(b + 1) * stride + col];
    if (b + 2 < b1) s[2] += a.partial[int64_t(b + 2) * stride + col];
    a.chunks[int64_t(c) * stride + col] = (s[0] + s[1]) + (s[2] + s[3]);
  }
}

// Fixed-order tree reduction over 1024 entries in shared memory.
template <bool kMin>
__device__ double block_reduce_1024(double* buf, double v) {
  const int t = threadIdx.x;
  buf[t] = v;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (t < o) buf[t] = kMin ? fmin(buf[t], buf[t + o]) : buf[t] + buf[t + o];
    __syncthreads();
  }
  const double r = buf[0];
  __syncthreads();
  return r;
}

// One block (1024 threads) per job: d̄, w̄, H and the verdict.
__global__ void __launch_bounds__(1024) match_finalize_kernel(uint8_t* tab) {
  const MatchHdr* hdr = reinterpret_cast<const MatchHdr*>(tab);
  const MatchJob& a = reinterpret_cast<const MatchJob*>(tab + hdr->job_off)[blockIdx.x];
  const int32_t* ints = reinterpret_cast<const int32_t*>(tab + hdr->int_off);
  MatchResultDev* res = reinterpret_cast<MatchResultDev*>(tab + hdr->res_off) + blockIdx.x;
  const int32_t* ties = reinterpret_cast<const int32_t*>(tab + hdr->tie_off);
  __shared__ double buf[1024];
  __shared__ double dsh[kMaxCapDev];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // per candidate: lanes stride over the position blocks in a fixed order, then a
  // butterfly (identical in every lane, deterministic)
  if (!a.cosine) {
    static_assert(kMatchChunks == 32, "one chunk per lane");
    for (int j = warp; j < a.n_cand; j += 32) {
      double s = a.chunks[int64_t(lane) * a.n_cand + j];
      s = warp_sum_d(s);
      if (lane == 0) dsh[j] = a.scalar_mode == 0 ? sqrt(s) : s / double(a.L_phi);
    }
  } else {
    const int64_t stride = 2 * a.n_cand + 1;
    double sqq = a.chunks[int64_t(lane) * stride + 2 * a.n_cand];  // every warp: same order, same value
    sqq = warp_sum_d(sqq);
    for (int j = warp; j < a.n_cand; j += 32) {
      double sqa = a.chunks[int64_t(lane) * stride + j];
      double saa = a.chunks[int64_t(lane) * stride + a.n_cand + j];
      sqa = warp_sum_d(sqa);
      saa = warp_sum_d(saa);
      const double den = sqrt(sqq * saa);
      if (lane == 0) dsh[j] = 1.0 - (den > 0.0 ? sqa / den : 0.0);
    }
  }
  __syncthreads();
  const int j = threadIdx.x;
  const bool valid = j < a.n_cand;
  const double dbar = valid ? dsh[j] : 0.0;
  const double mn = block_reduce_1024<true>(buf, valid ? dbar : DBL_MAX);
  const double e = valid ? exp(-(dbar - mn)) : 0.0;
  const double S = block_reduce_1024<false>(buf, e);
  const double w = e / S;
  const double t = (valid && w > 0.0) ? -w * log(w) : 0.0;
  const double H = block_reduce_1024<false>(buf, t);
  if (valid) dsh[j] = w;
  __syncthreads();
  const int32_t* slot2cand = ints + a.s2c_off;
  for (int sl = threadIdx.x; sl < a.cap; sl += blockDim.x) {
    const int jj = slot2cand[sl];
    a.wbar[sl] = jj >= 0 ? float(dsh[jj]) : 0.f;
  }
  if (threadIdx.x == 0) {
    const double thr = a.gamma * log(double(a.n_cand));
    int mismatch = 0;
    for (int r = 0; r < hdr->shard_world && hdr->shard_world > 1; ++r) mismatch |= hdr->fp_mine[r] != hdr->fingerprint;
    res->entropy = H;
    res->threshold = thr;
    // γ = 0 is "the original no-cache-sharing method" (Table 6; reading A19): NewAnchor
    // even when |𝒜_φ| = 1 makes H = 0 = threshold
    res->verdict = (H > thr || a.gamma == 0.0 || mismatch) ? 1 : 0;
    res->shard_mismatch = mismatch;
    res->tie_flag = (a.n_cand > 1 && fabs(H - thr) <= kTieRel * thr) ? 1 : 0;  // |𝒜|=1: H = 0 = thr exactly
    res->tie_count = ties[blockIdx.x];
  }
}

cudaError_t launch_match_dist(const void* table_dev, const MatchHdr& hdr, size_t smem, cudaStream_t s) {
  // (a rank that owns no position block still launches one block: it publishes its fingerprint)
  if (hdr.tma == 2) {
    const size_t sm = match_ring_smem(hdr.tma_stages, hdr.ring_row_bytes, hdr.tma_qbytes, hdr.tma_cmax, hdr.P);
    static bool attr2[64] = {false};
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    if (!attr2[dev & 63]) {
      cudaError_t e = cudaFuncSetAttribute(match_dist_ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(227 * 1024));
      if (e != cudaSuccess) return e;
      attr2[dev & 63] = true;
    }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::max(1, std::min(hdr.total_blocks, sms));
    match_dist_ring_kernel<<<grid, kRingWarps * 32 + 32, sm, s>>>(reinterpret_cast<const uint8_t*>(table_dev));
    return cudaGetLastError();
  }
  if (hdr.tma) {
    const size_t sm = match_tma_smem(hdr.tma_stages, hdr.tma_qbytes, hdr.tma_cmax);
    static bool attr[64] = {false};
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    if (!attr[dev & 63]) {
      cudaError_t e = cudaFuncSetAttribute(match_dist_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(227 * 1024));
      if (e != cudaSuccess) return e;
      attr[dev & 63] = true;
    }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::max(1, std::min(hdr.total_blocks, sms));
    match_dist_tma_kernel<<<grid, kMatchThreads + 32, sm, s>>>(reinterpret_cast<const uint8_t*>(table_dev));
    return cudaGetLastError();
  }
  // beside a realign (pipelined plan runs) only the 40-register build fits next to the
  // realign CTA on an SM, whatever the row length: slower alone at D_e 8192, but hidden
  const auto kern = (hdr.max_de <= kMatchWideDe || hdr.beside_realign) ? match_dist_kernel<KVC_MATCH_MINB>
                                                                         : match_dist_kernel<1>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
  }
  uint8_t* t = reinterpret_cast<uint8_t*>(const_cast<void*>(table_dev));
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMatchThreads, smem);
  static const int ctas_env = [] {  // measurement knob: CTAs per SM (<= occupancy)
    const char* e = getenv("KVCOMM_MATCH_CTAS");
    return e ? atoi(e) : 0;
  }();
  if (ctas_env > 0) per_sm = std::min(per_sm, ctas_env);
  const int grid = std::max(1, std::min(hdr.total_blocks, sms * std::max(per_sm, 1)));  // >= 1
  kern<<<grid, kMatchThreads, smem, s>>>(t);
  return cudaGetLastError();
}

cudaError_t launch_match_reduce(const void* table_dev, const MatchHdr& hdr, cudaStream_t s) {
  uint8_t* t = reinterpret_cast<uint8_t*>(const_cast<void*>(table_dev));
  match_chunk_kernel<<<dim3(hdr.n_jobs, kMatchChunks), 256, 0, s>>>(t);
  match_finalize_kernel<<<hdr.n_jobs, 1024, 0, s>>>(t);
  return cudaGetLastError();
}

cudaError_t launch_match_batch(const void* table_dev, const MatchHdr& hdr, size_t smem, cudaStream_t s) {
  cudaError_t e = launch_match_dist(table_dev, hdr, smem, s);
  return e != cudaSuccess ? e : launch_match_reduce(table_dev, hdr, s);
}

}  // namespace kvc
