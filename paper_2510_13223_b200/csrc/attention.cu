// H4 (+ H6 for co-located shards): paged GQA split decode attention over KV shards
// (split attention of PAPER.md:216-231, eqs. 6-9, with readings R-A1..R-A11: token-range
// split, explicit scale, max-shifted exponentials, shard-local block tables, masked pad
// slots).
//
// Outputs per (request b, q-head h): the partial triple (o~ normalised by the local
// denominator, m, l) in fp32, natural-log units -- what bs_merge_partials (eq. 10)
// consumes -- or, for shards that live on this GPU (bs_split_decode_attention_local),
// the LSE-merged bf16 O and lse directly.
//
// Design:
//  * grid = (CTA ranges over all shards of the launch, kv heads, requests); a CTA owns one
//    (request, kv-head, block range) and serves all G query heads of the group, so every
//    K/V page is read from HBM exactly once.
//  * 4 warps per CTA, each an independent pipeline over every 4th block of the range:
//    the block's K and V pages stream into a STAGES-deep shared-memory ring by TMA,
//    completing on an mbarrier; block ids come from a shared-memory copy of the table.
//  * split_decode_attn_mma (default): the per-block contractions S^T = K q^T and
//    O^T += V^T P^T on the tensor cores (mma.sync m16n8k16 bf16 -> fp32, heads in N),
//    pages by 2-D tensor TMA with 128-byte swizzle so ldmatrix is conflict-free.
//  * split_decode_attn (CUDA cores, BS_ATTN_MMA=0): lane-owned head dims, a select-free
//    16-shuffle reduce-scatter, online softmax in log2 units, packed FFMA2.
//  * the 4 warp states merge in shared memory; with several CTA ranges per
//    (request, kv-head) -- intra-GPU split-K and/or several local shards -- each CTA
//    writes a partial to the workspace and the last-arriving CTA merges them in fixed
//    order (deterministic), re-arms the arrival counter and writes the output; one-wave
//    launches with 2..8 ranges instead run each (request, kv-head)'s ranges as one
//    thread-block cluster and merge through distributed shared memory (same arithmetic).
//  * launches flagged BS_ATTN_PDL are programmatic dependents of the previous layer's
//    launch (prologue and first K/V stages overlap its tail); grids of <= 1 CTA per SM then
//    run a 6-stage ring that prefetches most of their range before griddepcontrol.wait.
//  * ragged plans may pack short requests four to a CTA, one warp each (no combine).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "internal.h"
#include "ptx.cuh"

namespace bs {
namespace {

constexpr float kLn2 = 0.6931471805599453f;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kWarps = 4;
constexpr int kBtMax = 512;     // blocks per CTA range (bt cached in smem)
constexpr int kMaxSplit = 64;   // intra-GPU split-K limit
constexpr int kPackMaxBlocks = 8;  // ragged plan: requests of <= 8 blocks are packed, one per warp

constexpr int kMaxLocal = 8;  // shards (tasks) / problems of one launch

#ifdef BS_TIMELINE
// Diagnostics build only: per-CTA %globaltimer stamps (ns) of the tensor-core kernel --
// [0] entry, [1] first K/V stage landed (warp 0), [2] all warps' loops done, [3] arrival
// counter resolved (cluster merge: leader's partials all landed / producer released),
// [4] exit, [5] smid | last-arriver << 16 | blocks << 20, [6] griddepcontrol.wait returned
// (PDL launches).  Rows from AttnParams::tl_base: consecutive launches alternate between the
// two halves (bs_timeline_reset restarts at the first), so a PDL pair can be read back.
// Read by bs_timeline_read.
constexpr int kTlCtas = 16384;
constexpr int kTlCols = 8;
__device__ unsigned long long g_timeline[kTlCtas][kTlCols];
std::atomic<int> g_tl_launches{0};  // host: launches since bs_timeline_reset
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define BS_TL(k)                                                                              \
  do {                                                                                        \
    const unsigned _lin = tl_base_ + blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); \
    if (threadIdx.x == 0 && _lin < kTlCtas) g_timeline[_lin][k] = tl_now();                  \
  } while (0)
#else
#define BS_TL(k) \
  do {           \
  } while (0)
#endif

// One attention problem: a set of requests whose KV is split into shards, some of which
// may be processed by other launches (on other GPUs).  All ranges of a (request, kv-head)
// arrive on one counter; the last arriver merges.  Every pointer may be a peer mapping.
struct ProbDesc {
  const __nv_bfloat16* q;
  const int32_t* kv_split;
  int32_t n_shards;
  int32_t nsplit;  // CTA ranges of the problem over all its shards (all launches / GPUs)
  int32_t merged;  // 1: write bf16 O + lse; 0: (o~, m, l)
  int32_t sys;     // shards on several GPUs: system-scope arrival / done counters
  float* o;
  float* m;
  float* l;
  __nv_bfloat16* out;
  float* lse;
  float* ws_o;
  float* ws_ml;
  int32_t* ws_cnt;
  int32_t* done;   // +1 per merged (request, kv-head), monotonic; or NULL
};

// One KV shard of the launch: where its pages live and how its blocks are cut into CTAs.
struct ShardDesc {
  const uint8_t* kv;  // pool base + layer * layer_bytes
  int64_t chunk_bytes;
  int64_t v_off;      // Hkv * page bytes: K page -> V page of the same head
  const int32_t* bt;
  int32_t max_blocks;
  int32_t shard_id;    // column of kv_split
  int32_t bps;         // blocks per CTA range
  int32_t split_off;   // first grid.x index of this shard
  int32_t layer_row0;  // tensor-map row of (layer, block 0, K, head 0, slot 0)
  int32_t pool_hkv;    // kv heads of the pool (tensor-map addressing)
  int32_t pool_head_lo;  // first kv head of this launch inside the pool
  int32_t prob;        // problem of this shard (index into AttnParams::pb)
  int32_t range_base;  // problem range index of this shard's first CTA range
  const int32_t* order;  // uniform grid: request of grid row z (longest first), or NULL
};

struct AttnParams {
  ShardDesc sh[kMaxLocal];
  ProbDesc pb[kMaxLocal];
  int32_t n_local;
  float scale_log2;
  int32_t hq, hkv;          // hq: q heads of the MODEL (row stride); hkv: kv heads in this launch
  int32_t model_head_lo;    // first kv head of the launch in the model (q / output rows)
  int32_t grid_x;           // CTA ranges of this launch over its shards
  int32_t pdl;              // launched as a programmatic dependent: prefetch, then wait
  int32_t cl;               // cluster merge: grid.x = ranges = cluster size (cluster_combine_merge)
  int32_t tl_base;          // timeline build only: first g_timeline row of this launch
  int32_t trig_late;        // tensor-core kernel: let the next (PDL) launch start once every
                            // CTA has started (0), finished its main loop (1), or exited (2)
  int32_t deep;             // at most one CTA per SM: the 6-stage ring variant (d = 128)
  const int4* work;         // ragged plan (bs_attention_ragged_plan) or NULL: one item per
                            // item = (request, shard << 16 | slot, first block,
                            // blocks << 8 | ranges of the request); grid.x = items * hkv
};

struct TMaps {
  CUtensorMap m[kMaxLocal];
};

// grid.x index -> (shard of the launch, CTA range inside it)
__device__ __forceinline__ int shard_of(const AttnParams& p, int spg) {
  int j = 0;
#pragma unroll
  for (int i = 1; i < kMaxLocal; ++i)
    if (i < p.n_local && spg >= p.sh[i].split_off) j = i;
  return j;
}

// What one CTA computes: request b, shard js of the launch, blocks [blo, blo + nb) of the
// shard, partial slot, and the request's range count (-1: the problem's uniform nsplit).
struct CtaWork {
  int b, g, js, blo, nb, slot, nparts;
  int packed;  // ragged plan, short requests: each warp serves its own request b (-1: none)
};

__device__ __forceinline__ CtaWork cta_work(const AttnParams& p) {
  CtaWork w;
  w.packed = 0;
  if (p.work) {  // ragged plan: grid.x = item * Hkv + kv head (heads of an item adjacent:
                 // they read neighbouring pages of the same blocks)
    const int item = blockIdx.x / p.hkv;
    w.g = blockIdx.x - item * p.hkv;
    const int4 it = __ldg(p.work + item);
    if ((it.w & 0xff) == 0) {  // packed item (parts field 0): up to kWarps short requests of
      w.packed = 1;            // shard 0, one per warp -- (b0, b1, b2, b3 << 8), -1 = none
      const int wp = threadIdx.x >> 5;
      w.b = wp == 0 ? it.x : wp == 1 ? it.y : wp == 2 ? it.z : (it.w >> 8);
      w.js = 0;
      w.slot = 0;
      w.blo = 0;
      w.nb = 0;
      w.nparts = 1;
      return w;
    }
    w.b = it.x;
    w.js = it.y >> 16;
    w.slot = it.y & 0xffff;
    w.blo = it.z;
    w.nb = it.w >> 8;
    w.nparts = it.w & 0xff;
  } else {       // uniform plan: grid = (ranges over the launch's shards, kv heads, requests)
    const int spg = blockIdx.x;
    w.g = blockIdx.y;
    w.js = shard_of(p, spg);
    // rows are dispatched in z order: a task's request order puts its longest requests in
    // the first CTAs (longest-processing-time first), the merge order stays the slot order
    w.b = p.sh[w.js].order ? __ldg(p.sh[w.js].order + blockIdx.z) : (int)blockIdx.z;
    const int sp = spg - p.sh[w.js].split_off;
    w.blo = sp * p.sh[w.js].bps;
    w.nb = p.sh[w.js].bps;
    w.slot = p.sh[w.js].range_base + sp;
    w.nparts = -1;
  }
  return w;
}

template <int D, int G, int STAGES>
struct Smem {
  static constexpr int kPage = 16 * D * 2;
  static constexpr int kStage = 2 * kPage;
  static constexpr int kRing = kWarps * STAGES * kStage;
  static constexpr int kBtOff = kRing;
  static constexpr int kPOff = kBtOff + kBtMax * 4;
  static constexpr int kBarOff = kPOff + kWarps * G * 16 * 4;
  static constexpr int kMlOff = kBarOff + kWarps * STAGES * 8;
  static constexpr int kWOff = kMlOff + kWarps * G * 2 * 4;
  static constexpr int kFlagOff = kWOff + G * kMaxSplit * 4;
  static constexpr int kTotal = kFlagOff + 16;
  static_assert(kWarps * G * D * 4 <= kRing, "combine buffer must fit in the ring");
};

__device__ __forceinline__ float2 bf2_to_f2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  return __ffma2_rn(a, b, c);
}

// Sum 16 per-lane partials over the 32 lanes.  Slot i of lane L holds token i ^ (L >> 1)
// (the K rows are loaded in that lane-permuted order), so every butterfly step keeps the
// low half of its slots and sends the high half -- no per-lane selects -- and lane pair
// (2t, 2t+1) ends with token t's total.  Adds are packed (FADD2) on slot pairs.
__device__ __forceinline__ float reduce_scatter16(float (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    const float2 r = make_float2(__shfl_xor_sync(0xffffffffu, v[i + 8], 16),
                                 __shfl_xor_sync(0xffffffffu, v[i + 9], 16));
    const float2 x = __fadd2_rn(make_float2(v[i], v[i + 1]), r);
    v[i] = x.x;
    v[i + 1] = x.y;
  }
#pragma unroll
  for (int i = 0; i < 4; i += 2) {
    const float2 r = make_float2(__shfl_xor_sync(0xffffffffu, v[i + 4], 8),
                                 __shfl_xor_sync(0xffffffffu, v[i + 5], 8));
    const float2 x = __fadd2_rn(make_float2(v[i], v[i + 1]), r);
    v[i] = x.x;
    v[i + 1] = x.y;
  }
  {
    const float2 r = make_float2(__shfl_xor_sync(0xffffffffu, v[2], 4),
                                 __shfl_xor_sync(0xffffffffu, v[3], 4));
    const float2 x = __fadd2_rn(make_float2(v[0], v[1]), r);
    v[0] = x.x;
    v[1] = x.y;
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[1], 2);
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// Merge the kWarps per-warp states of one CTA (s_acc [kWarps][G][D] unnormalised, s_ml
// [kWarps][G] (m log2, l)) and write the shard output -- or, with intra-GPU split-K, the
// CTA's partial; the last-arriving CTA of the (request, kv-head) then merges all partials
// in fixed order, re-arms the arrival counter and writes the output.  Called by every
// thread of the CTA after a __syncthreads.
__device__ __forceinline__ void count_done(const ProbDesc& P) {  // P: a local copy
  // the caller's barrier orders every thread's output stores before this; the release is
  // cumulative, so a waiter that acquires the counter sees the outputs
  if (P.sys)
    asm volatile("red.release.sys.global.add.s32 [%0], 1;" ::"l"(P.done) : "memory");
  else
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(P.done) : "memory");
}

// The eq. 10 merge of a (request, kv-head)'s nparts partials (o~ normalised by its own l,
// m in log2 units, l) in fixed order 0..nparts-1, and the output store (bf16 O + lse, or the
// (o~, m, l) triple).  `src` says where the partials are: the workspace (last-arriver
// merge, WsParts) or this CTA's shared memory (cluster merge, SmemParts) -- the arithmetic
// is the same, so both paths give bitwise the same result.  s_red: KiB-sized scratch.
struct WsParts {  // P.ws_o [row][nsplit][D], P.ws_ml [row][nsplit][2], read through L2
  const float* ws_o;
  const float* ws_ml;
  int nsplit;
  __device__ __forceinline__ float m(int64_t row, int, int j) const { return __ldcg(ws_ml + (row * nsplit + j) * 2); }
  __device__ __forceinline__ float l(int64_t row, int, int j) const { return __ldcg(ws_ml + (row * nsplit + j) * 2 + 1); }
  template <int D>
  __device__ __forceinline__ float4 o4(int64_t row, int, int x, int j) const {
    return __ldcg(reinterpret_cast<const float4*>(ws_o + (row * nsplit + j) * D + x));
  }
};

template <int D, int G>
struct SmemParts {  // part j at base + j * kPF floats: o~ [G][D], then (m, l) per head
  static constexpr int kPF = (G * D + 2 * G + 3) & ~3;
  const float* base;
  __device__ __forceinline__ float m(int64_t, int h, int j) const { return base[j * kPF + G * D + 2 * h]; }
  __device__ __forceinline__ float l(int64_t, int h, int j) const { return base[j * kPF + G * D + 2 * h + 1]; }
  template <int DD>
  __device__ __forceinline__ float4 o4(int64_t, int h, int x, int j) const {
    return *reinterpret_cast<const float4*>(base + j * kPF + h * D + x);
  }
};

template <int D, int G, class Src>
__device__ __forceinline__ void merge_parts_store(const ProbDesc& P, int hq, int b, int gm, int nparts,
                                                  const Src& src, float* s_w, float4* s_red) {
  // per-head weights w_j = l_j 2^(m_j - M) / L: one warp per head, lanes over the ranges
  // (<= kMaxSplit = 64 -> 2 per lane); butterfly reductions keep the result deterministic
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int h = warp; h < G; h += kWarps) {
      const int64_t row = (int64_t)b * hq + gm * G + h;
      float mj[2], lj[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int j = lane + 32 * t;
        mj[t] = j < nparts ? src.m(row, h, j) : -INFINITY;
        lj[t] = j < nparts ? src.l(row, h, j) : 0.f;
      }
      float M = fmaxf(mj[0], mj[1]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      float w[2], L = 0.f;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        w[t] = mj[t] == -INFINITY ? 0.f : lj[t] * exp2f(mj[t] - M);
        L += w[t];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int j = lane + 32 * t;
        if (j < nparts) s_w[h * kMaxSplit + j] = L > 0.f ? w[t] / L : 0.f;
      }
      if (lane == 0) {
        if (P.merged) {
          if (P.lse) P.lse[row] = L > 0.f ? M * kLn2 + logf(L) : -INFINITY;
        } else {
          P.m[row] = L > 0.f ? M * kLn2 : -INFINITY;
          P.l[row] = L;
        }
      }
    }
  }
  __syncthreads();
  // O = sum_j w_j o~_j over float4 columns: every load of the loop is independent (16 in
  // flight per thread), so the merge costs ~nparts/16 L2 round trips instead of one per
  // 8 ranges per column.  NV float4 columns per (request, kv-head); with NV < 128 the
  // threads also split the ranges (JS interleaved groups) and sum the groups in fixed order.
  {
    constexpr int NV = G * D / 4;
    constexpr int E = NV < kWarps * 32 ? NV : kWarps * 32;
    constexpr int JS = kWarps * 32 / E;
    const int e0 = threadIdx.x % E, jo = threadIdx.x / E;
#pragma unroll
    for (int e = e0; e < NV; e += E) {
      const int h = (e * 4) / D, x = e * 4 - h * D;
      const int64_t row = (int64_t)b * hq + gm * G + h;
      const float* w = s_w + h * kMaxSplit;
      float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 16
      for (int j = jo; j < nparts; j += JS) {
        const float4 v = src.template o4<D>(row, h, x, j);
        const float wj = w[j];
        O.x += wj * v.x;
        O.y += wj * v.y;
        O.z += wj * v.z;
        O.w += wj * v.w;
      }
      if constexpr (JS > 1) {
        s_red[jo * E + e0] = O;
        __syncthreads();
        if (jo == 0) {
#pragma unroll
          for (int k = 1; k < JS; ++k) {
            const float4 r = s_red[k * E + e0];
            O.x += r.x;
            O.y += r.y;
            O.z += r.z;
            O.w += r.w;
          }
        }
      }
      if (jo == 0) {
        if (P.merged) {
          const __nv_bfloat162 lo = __floats2bfloat162_rn(O.x, O.y), hi = __floats2bfloat162_rn(O.z, O.w);
          uint2 pk;
          pk.x = *reinterpret_cast<const uint32_t*>(&lo);
          pk.y = *reinterpret_cast<const uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(P.out + row * D + x) = pk;
        } else {
          *reinterpret_cast<float4*>(P.o + row * D + x) = O;
        }
      }
    }
  }
  if (P.done) {
    __syncthreads();
    if (threadIdx.x == 0) count_done(P);
  }
}


template <int D, int G>
// sp: this CTA's partial slot; nparts: ranges of the request to merge (P.nsplit, or the
// request's own count under a ragged plan); P.nsplit is the workspace slot stride.
__device__ __forceinline__ void cta_combine_and_store(const ProbDesc P, int hq, int hkv, int b, int g,
                                                      int gm, int sp, int nparts, const float* s_acc,
                                                      const float* s_ml, float* s_w, int* s_flag,
                                                      int tl_base_ = 0) {
  (void)tl_base_;
  for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
    const int h = idx / D, x = idx - h * D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, s_ml[(w * G + h) * 2]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float mw = s_ml[(w * G + h) * 2];
      if (mw != -INFINITY) {
        const float f = exp2f(mw - M);
        L += s_ml[(w * G + h) * 2 + 1] * f;
        O += s_acc[(w * G + h) * D + x] * f;
      }
    }
    const int64_t row = (int64_t)b * hq + gm * G + h;
    const bool any = L > 0.f;
    if (nparts == 1) {
      if (P.merged) {
        P.out[row * D + x] = __float2bfloat16_rn(any ? O / L : 0.f);
        if (x == 0 && P.lse) P.lse[row] = any ? M * kLn2 + logf(L) : -INFINITY;
      } else {
        P.o[row * D + x] = any ? O / L : 0.f;
        if (x == 0) {
          P.m[row] = any ? M * kLn2 : -INFINITY;
          P.l[row] = L;
        }
      }
    } else {
      const int64_t part = row * P.nsplit + sp;
      P.ws_o[part * D + x] = any ? O / L : 0.f;
      if (x == 0) {
        P.ws_ml[part * 2] = any ? M : -INFINITY;  // log2 units
        P.ws_ml[part * 2 + 1] = L;
      }
    }
  }
  if (nparts == 1) {
    if (P.done) {
      __syncthreads();
      if (threadIdx.x == 0) count_done(P);
    }
    return;
  }

  // ---- split-K / several shards: the last CTA of this (request, kv-head) merges --------
  // The barrier orders every thread's partial stores before thread 0's acq_rel atomic
  // (release is cumulative), and the winner's acquire + barrier order the other CTAs'
  // partials before this CTA's loads -- one atomic per CTA instead of a full fence
  // (CCTL.IVALL) in every thread.  System scope when the problem's shards run on several
  // GPUs: the other ranges' partials then arrive over NVLink from the peers' CTAs.
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t* cnt = P.ws_cnt + (int64_t)b * hkv + g;
    int prev;
    if (P.sys)
      asm volatile("atom.acq_rel.sys.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(cnt) : "memory");
    else
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(cnt) : "memory");
    const int last = prev == nparts - 1;
    if (last) *cnt = 0;  // every CTA has arrived: re-arm for the next call
    s_flag[0] = last;
  }
  __syncthreads();
  BS_TL(3);
  if (!s_flag[0]) return;
  merge_parts_store<D, G>(P, hq, b, gm, nparts, WsParts{P.ws_o, P.ws_ml, P.nsplit}, s_w,
                          reinterpret_cast<float4*>(const_cast<float*>(s_acc)));  // rings idle
}
// Cluster merge (AttnParams::cl, single-GPU problems with 2..16 CTA ranges per (request,
// kv-head)): the ranges of one (request, kv-head) form one thread-block cluster (grid.x =
// ranges = cluster size, rank = range slot).  Instead of publishing every partial to the
// workspace and electing the last arriver (the partial stores, an acq_rel atomic and the
// merge's loads: three dependent L2 round trips after the slowest range), each CTA combines
// its warps as usual and the non-leaders store their partial straight into the leader's
// (rank 0) shared memory with st.async, counted on the leader's mbarrier; the leader merges
// from shared memory (merge_parts_store, the same arithmetic as the workspace path).  The
// receive area is the leader's idle K/V ring, so the leader releases each producer (a
// remote arrive on the producer's "go" mbarrier) once its own loop is done.  No CTA's
// shared memory is touched after it exits: producers write only into the leader, which
// waits for all their bytes; the leader arrives only on producers that wait for it.
// cbar: [0] go (producers), [1] receive (leader), initialised before the cluster barrier's
// arrive in the prologue.
template <int D, int G>
__device__ __forceinline__ void cluster_combine_merge(const ProbDesc& P, int hq, int b, int gm,
                                                      int nparts, const float* s_acc,
                                                      const float* s_ml, float* s_w,
                                                      float* s_recv, uint64_t* cbar,
                                                      int tl_base_ = 0) {
  (void)tl_base_;
  using SP = SmemParts<D, G>;
  constexpr int NV = G * D / 4;
  constexpr int PER = (NV + kWarps * 32 - 1) / (kWarps * 32);
  float4 val[PER];
  float2 mlv[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {  // the CTA's partial, as cta_combine_and_store computes it
    const int e = threadIdx.x + k * kWarps * 32;
    if (e < NV) {
      const int h = (e * 4) / D, x = e * 4 - h * D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) M = fmaxf(M, s_ml[(w * G + h) * 2]);
      float L = 0.f, O[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const float mw = s_ml[(w * G + h) * 2];
        if (mw != -INFINITY) {
          const float f = exp2f(mw - M);
          L += s_ml[(w * G + h) * 2 + 1] * f;
#pragma unroll
          for (int c = 0; c < 4; ++c) O[c] += s_acc[(w * G + h) * D + x + c] * f;
        }
      }
      const bool any = L > 0.f;
      val[k] = any ? make_float4(O[0] / L, O[1] / L, O[2] / L, O[3] / L) : make_float4(0.f, 0.f, 0.f, 0.f);
      mlv[k] = make_float2(any ? M : -INFINITY, L);  // log2 units
    }
  }
  const uint32_t rank = ptx::cluster_ctarank();
  ptx::cluster_wait_acquire();  // every CTA of the cluster has initialised its barriers
  uint64_t* go = cbar;
  uint64_t* rv = cbar + 1;
  if (rank == 0) {
    if (threadIdx.x == 0) ptx::mbar_expect_tx(rv, (uint32_t)(nparts - 1) * (G * D * 4 + G * 8));
    if (threadIdx.x >= 1 && threadIdx.x < nparts) ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(go), threadIdx.x));
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int e = threadIdx.x + k * kWarps * 32;
      if (e < NV) {
        const int h = (e * 4) / D, x = e * 4 - h * D;
        *reinterpret_cast<float4*>(s_recv + h * D + x) = val[k];
        if (x == 0) *reinterpret_cast<float2*>(s_recv + G * D + 2 * h) = mlv[k];
      }
    }
    ptx::mbar_wait_cluster(rv, 0);
    __syncthreads();  // the leader's own partial (other threads' stores) too
    BS_TL(3);
    merge_parts_store<D, G>(P, hq, b, gm, nparts, SP{s_recv}, s_w,
                            reinterpret_cast<float4*>(s_recv + nparts * SP::kPF));
  } else {
    ptx::mbar_wait_cluster(go, 0);
    BS_TL(3);
    const uint32_t rbar = ptx::mapa(ptx::smem_u32(rv), 0);
    const uint32_t rbase = ptx::mapa(ptx::smem_u32(s_recv + rank * SP::kPF), 0);
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int e = threadIdx.x + k * kWarps * 32;
      if (e < NV) {
        const int h = (e * 4) / D, x = e * 4 - h * D;
        ptx::st_async_v4(rbase + (uint32_t)(h * D + x) * 4, val[k], rbar);
        if (x == 0) ptx::st_async_v2(rbase + (uint32_t)(G * D + 2 * h) * 4, mlv[k].x, mlv[k].y, rbar);
      }
    }
  }
}

template <int D, int G, int STAGES, int MINB>
__global__ void __launch_bounds__(kWarps * 32, MINB) split_decode_attn(const AttnParams p) {
  using S = Smem<D, G, STAGES>;
  constexpr int DPL = D / 32;  // head dims per lane (4 or 2)
  constexpr int DP2 = DPL / 2;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const CtaWork cw = cta_work(p);
  if (cw.packed) asm volatile("trap;");  // packed ragged items are for the tensor-core kernel
  const int g = cw.g, b = cw.b, js = cw.js;
  const ShardDesc& sd = p.sh[js];
  const ProbDesc& P = p.pb[sd.prob];

  // One memory round trip before the first TMA: the CTA's block-table row (independent
  // of the length), each warp's first STAGES block ids and the shard length are loaded
  // together; lane 0 of every warp then issues its first copies before the CTA barrier.
  const int32_t blo = cw.blo;
  const int64_t row0 = (int64_t)b * sd.max_blocks + blo;
  const int nb_tab = max(min(cw.nb, sd.max_blocks - blo), 0);
  constexpr int kIdPerThread = kBtMax / (kWarps * 32);
  int32_t idv[kIdPerThread];
#pragma unroll
  for (int r = 0; r < kIdPerThread; ++r) {
    const int i = threadIdx.x + r * kWarps * 32;
    idv[r] = i < nb_tab ? __ldg(sd.bt + row0 + i) : 0;
  }
  int32_t first[STAGES];
#pragma unroll
  for (int k = 0; k < STAGES; ++k)
    first[k] = (lane == 0 && warp + k * kWarps < nb_tab) ? __ldg(sd.bt + row0 + warp + k * kWarps) : 0;
  const int32_t* ks = P.kv_split + (int64_t)b * (P.n_shards + 1) + sd.shard_id;
  const int32_t len = max(__ldg(ks + 1) - __ldg(ks), 0);
  const int32_t nblk = (len + 15) >> 4;
  const int32_t nb_cta = max(min(nblk, blo + cw.nb) - blo, 0);
  const int nparts = cw.nparts < 0 ? P.nsplit : cw.nparts;

  int32_t* s_bt = reinterpret_cast<int32_t*>(smem + S::kBtOff);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kBarOff) + warp * STAGES;
  float* s_p = reinterpret_cast<float*>(smem + S::kPOff) + warp * G * 16;
  uint8_t* ring = smem + warp * STAGES * S::kStage;

  const int nmine = nb_cta > warp ? (nb_cta - warp + kWarps - 1) / kWarps : 0;
  const uint8_t* kv_head = sd.kv + (int64_t)(sd.pool_head_lo + g) * S::kPage;
  const int gm = p.model_head_lo + g;  // kv head index in the model
  uint64_t policy = 0;
  auto issue = [&](int k, int64_t phys) {  // lane 0 only
    const int s = k % STAGES;
    const uint8_t* kp = kv_head + phys * sd.chunk_bytes;
    uint8_t* dst = ring + s * S::kStage;
    ptx::mbar_expect_tx(&bars[s], 2 * S::kPage);
    ptx::bulk_g2s_evict_first(dst, kp, S::kPage, &bars[s], policy);
    ptx::bulk_g2s_evict_first(dst + S::kPage, kp + sd.v_off, S::kPage, &bars[s], policy);
  };
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) ptx::mbar_init(&bars[s], 1);
    ptx::fence_mbar_init();
    policy = ptx::policy_evict_first();
#pragma unroll
    for (int k = 0; k < STAGES; ++k)
      if (k < nmine) issue(k, first[k]);
  }
#pragma unroll
  for (int r = 0; r < kIdPerThread; ++r) {
    const int i = threadIdx.x + r * kWarps * 32;
    if (i < nb_cta) s_bt[i] = idv[r];
  }
  __syncthreads();  // block table + barrier inits visible to the CTA
  // Programmatic dependent launch (BS_ATTN_PDL): this grid may start while the previous
  // kernel on the stream drains.  Everything above -- block table, kv_split, the first
  // K/V stages in flight -- reads only step inputs (the caller's contract); q, the outputs
  // and the workspace (which the previous launch may still be merging from) come after the
  // wait, which returns once that kernel has completed and its writes are visible.
  if (p.pdl) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }

  // q for the G heads of this group, this lane's dims, pre-scaled into log2 units and
  // duplicated into both halves of a packed pair ({q_e, q_e}) for token-pair FFMA2
  float2 qq[G][DPL];
  {
    const __nv_bfloat16* qp = P.q + ((int64_t)b * p.hq + gm * G) * D + lane * DPL;
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float qf[DPL];
      if constexpr (DPL == 4) {
        const uint2 w = *reinterpret_cast<const uint2*>(qp + h * D);
        const float2 a = bf2_to_f2(w.x), c = bf2_to_f2(w.y);
        qf[0] = a.x; qf[1] = a.y; qf[2] = c.x; qf[3] = c.y;
      } else {
        const float2 a = bf2_to_f2(*reinterpret_cast<const uint32_t*>(qp + h * D));
        qf[0] = a.x; qf[1] = a.y;
      }
#pragma unroll
      for (int e = 0; e < DPL; ++e) qq[h][e] = make_float2(qf[e] * p.scale_log2, qf[e] * p.scale_log2);
    }
  }

  // running state; acc[h][e] = {sum over even tokens, sum over odd tokens} for dim e
  float m_run[G], l_run[G];
  float2 acc[G][DPL];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    m_run[h] = -INFINITY;
    l_run[h] = 0.f;
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[h][e] = make_float2(0.f, 0.f);
  }

  // two rows (tokens) of a page, this lane's DPL dims -> DPL packed {row0, row1} pairs
  auto load_pair = [&](const uint8_t* r0, const uint8_t* r1, float2 (&out)[DPL]) {
    if constexpr (DPL == 4) {
      const uint2 w0 = *reinterpret_cast<const uint2*>(r0 + lane * 8);
      const uint2 w1 = *reinterpret_cast<const uint2*>(r1 + lane * 8);
      out[0] = make_float2(__uint_as_float(w0.x << 16), __uint_as_float(w1.x << 16));
      out[1] = make_float2(__uint_as_float(w0.x & 0xffff0000u), __uint_as_float(w1.x & 0xffff0000u));
      out[2] = make_float2(__uint_as_float(w0.y << 16), __uint_as_float(w1.y << 16));
      out[3] = make_float2(__uint_as_float(w0.y & 0xffff0000u), __uint_as_float(w1.y & 0xffff0000u));
    } else {
      const uint32_t w0 = *reinterpret_cast<const uint32_t*>(r0 + lane * 4);
      const uint32_t w1 = *reinterpret_cast<const uint32_t*>(r1 + lane * 4);
      out[0] = make_float2(__uint_as_float(w0 << 16), __uint_as_float(w1 << 16));
      out[1] = make_float2(__uint_as_float(w0 & 0xffff0000u), __uint_as_float(w1 & 0xffff0000u));
    }
  };

  for (int k = 0; k < nmine; ++k) {
    const int s = k % STAGES;
    ptx::mbar_wait(&bars[s], (uint32_t)((k / STAGES) & 1));
    __syncwarp();
    const uint8_t* sk = ring + s * S::kStage;
    const uint8_t* sv = sk + S::kPage;
    const int blk = blo + warp + k * kWarps;  // block index within the shard
    const int nvalid = min(16, len - blk * 16);

    // ---- scores: s_t = <q_h, k_t> (log2 units) -------------------------------------
    // slot i holds token i ^ (lane >> 1) (see reduce_scatter16); slots paired (2j, 2j+1)
    float2 kp[8][DPL];
    const uint32_t kswz = (uint32_t)((lane >> 1) & 15) * (D * 2);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      load_pair(sk + ((uint32_t)(2 * j * D * 2) ^ kswz), sk + ((uint32_t)((2 * j + 1) * D * 2) ^ kswz),
                kp[j]);
    const bool valid = (lane >> 1) < nvalid;
    float alpha[G];
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float v[16];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float2 a = __fmul2_rn(qq[h][0], kp[j][0]);
#pragma unroll
        for (int e = 1; e < DPL; ++e) a = ffma2(qq[h][e], kp[j][e], a);
        v[2 * j] = a.x;
        v[2 * j + 1] = a.y;
      }
      float sc = reduce_scatter16(v);
      sc = valid ? sc : -INFINITY;
      float mb = sc;
      mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 2));
      mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 4));
      mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 8));
      mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 16));
      const float mn = fmaxf(m_run[h], mb);  // finite: slot 0 of every block is valid
      alpha[h] = exp2f(m_run[h] - mn);
      const float pr = exp2f(sc - mn);
      l_run[h] = l_run[h] * alpha[h] + ((lane & 1) ? 0.f : pr);
      m_run[h] = mn;
      if (!(lane & 1)) s_p[h * 16 + (lane >> 1)] = pr;
    }
    __syncwarp();

    // ---- o = alpha * o + sum_t p_t v_t  (token pairs: {p_2j, p_2j+1} x {v_2j, v_2j+1})
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const float2 a2 = make_float2(alpha[h], alpha[h]);
#pragma unroll
      for (int e = 0; e < DPL; ++e) acc[h][e] = __fmul2_rn(acc[h][e], a2);
    }
    auto pv = [&](auto full) {
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {  // 4 tokens per float4 of p
        float4 pp[G];
#pragma unroll
        for (int h = 0; h < G; ++h) pp[h] = *reinterpret_cast<const float4*>(s_p + h * 16 + 4 * j4);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int t0 = 4 * j4 + 2 * half;
          if (!decltype(full)::value && t0 >= nvalid) continue;
          float2 vp[DPL];
          load_pair(sv + t0 * D * 2, sv + (t0 + 1) * D * 2, vp);
          if (!decltype(full)::value && t0 + 1 >= nvalid) {  // odd token is a pad slot
#pragma unroll
            for (int e = 0; e < DPL; ++e) vp[e].y = 0.f;
          }
#pragma unroll
          for (int h = 0; h < G; ++h) {
            const float2 p2 = half == 0 ? make_float2(pp[h].x, pp[h].y) : make_float2(pp[h].z, pp[h].w);
#pragma unroll
            for (int e = 0; e < DPL; ++e) acc[h][e] = ffma2(p2, vp[e], acc[h][e]);
          }
        }
      }
    };
    // pad slots hold garbage (NaN-poisoned in tests): the partial last block masks V too
    if (nvalid == 16) pv(std::true_type{});
    else pv(std::false_type{});
    __syncwarp();
    if (lane == 0 && k + STAGES < nmine) {
      ptx::fence_proxy_async_smem();
      issue(k + STAGES, s_bt[warp + (k + STAGES) * kWarps]);
    }
    __syncwarp();
  }

  // ---- merge the 4 warp states in shared memory ------------------------------------
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float x = l_run[h];
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 4);
    x += __shfl_xor_sync(0xffffffffu, x, 8);
    x += __shfl_xor_sync(0xffffffffu, x, 16);
    l_run[h] = x;
  }
  __syncthreads();  // every warp finished with its ring; reuse it for the combine
  float* s_acc = reinterpret_cast<float*>(smem);  // [kWarps][G][D]
  float* s_ml = reinterpret_cast<float*>(smem + S::kMlOff);
  float* s_w = reinterpret_cast<float*>(smem + S::kWOff);
  int* s_flag = reinterpret_cast<int*>(smem + S::kFlagOff);
#pragma unroll
  for (int h = 0; h < G; ++h) {
#pragma unroll
    for (int e = 0; e < DP2; ++e)
      *reinterpret_cast<float2*>(s_acc + (warp * G + h) * D + lane * DPL + 2 * e) =
          make_float2(acc[h][2 * e].x + acc[h][2 * e].y, acc[h][2 * e + 1].x + acc[h][2 * e + 1].y);
    if (lane == 0) {
      s_ml[(warp * G + h) * 2] = m_run[h];
      s_ml[(warp * G + h) * 2 + 1] = l_run[h];
    }
  }
  __syncthreads();
  cta_combine_and_store<D, G>(P, p.hq, p.hkv, b, g, gm, cw.slot, nparts, s_acc, s_ml, s_w,
                              s_flag);
}

// ---------------------------------------------------------------------------------------
// Tensor-core variant for GQA groups G in {4, 8} (at G >= 4 the CUDA-core
// kernel is issue-bound -- ncu: 724 instructions per 8 KiB block at G=4 -- so the two
// per-block contractions go to mma.sync.m16n8k16 (bf16 in, fp32 accumulate)):
//   S^T[16 tok x 8 heads] = K[16 x d] . Q^T[d x 8]   (A = K rows via ldmatrix, B = q in regs)
//   O^T[d x 8 heads]     += V^T[d x 16] . P^T[16 x 8] (A = V via ldmatrix.trans, B = P bf16)
// The G heads of the group fill N = 8 (G = 4: half the columns are padding).  Scores are
// scaled in fp32 after the MMA (q stays exact bf16); P is rounded to bf16 for the PV MMA
// (the denominator l sums the fp32 p).  K/V pages land in shared memory as 16 rows of
// d*2 bytes padded to d*2+16 (one 256/128-byte TMA bulk copy per row, issued by 32 lanes
// in parallel), which makes every ldmatrix row phase conflict-free.  Pipeline, split-K
// and epilogue are those of split_decode_attn.
// ---------------------------------------------------------------------------------------

template <int D, int G, int STAGES>
struct MmaSmem {
  static constexpr int kBoxes = D / 64;       // 128-byte-wide TMA boxes per page
  static constexpr int kBox = 16 * 128;       // one box: 16 rows x 128 B, 128B-swizzled
  static constexpr int kStage = 2 * kBoxes * kBox;  // K boxes then V boxes
  static constexpr int kRing = kWarps * STAGES * kStage;
  static constexpr int kBtOff = kRing;
  static constexpr int kPOff = kBtOff + kBtMax * 4;  // P^T bf16 [8][16] per warp
  static constexpr int kBarOff = kPOff + kWarps * 8 * 16 * 2;
  static constexpr int kMlOff = kBarOff + kWarps * STAGES * 8;
  static constexpr int kWOff = kMlOff + kWarps * G * 2 * 4;
  static constexpr int kFlagOff = kWOff + G * kMaxSplit * 4;
  static constexpr int kClBarOff = kFlagOff + 16;     // cluster merge: go / receive mbarriers
  static constexpr int kRecvOff = kWarps * G * D * 4;  // cluster merge: partials, in the idle ring
  static constexpr int kTotal = kClBarOff + 16 + 1024;  // + alignment slack (swizzle atoms)
  static_assert(kWarps * G * D * 4 <= kRing, "combine buffer must fit in the ring");
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// 2D tensor TMA (pool viewed as [rows][D] bf16, box [16 rows][64 elems], 128B swizzle)
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(ptx::smem_u32(bar)), "l"(policy)
      : "memory");
}

// byte offset of (row, 16-byte chunk) inside a 128B-swizzled box
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
}

template <int D, int G, int STAGES, int MINB>
__global__ void __launch_bounds__(kWarps * 32, MINB)
    split_decode_attn_mma(const AttnParams p, const __grid_constant__ TMaps tm) {
  using S = MmaSmem<D, G, STAGES>;
  constexpr int KS = D / 16;  // k-steps of the QK MMA == m-tiles of the PV MMA
  constexpr int NB = S::kBoxes;
  static_assert(G <= 8, "one n8 tile of heads");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tl_base_ = p.tl_base;
  (void)tl_base_;
  BS_TL(0);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;  // mma groupID / thread-in-group
  const CtaWork cw = cta_work(p);
  const int g = cw.g, js = cw.js;
  const ShardDesc& sd = p.sh[js];
  const ProbDesc& P = p.pb[sd.prob];
  // packed item (ragged plan, short requests): this warp serves its own request alone --
  // all its blocks (boff 0, stride 1) from its own slice of the block-id table -- and
  // writes its output itself; otherwise the warps interleave over the CTA's range
  const int b = cw.b;  // (packed items: this warp's own request)
  const int bstride = cw.packed ? 1 : kWarps, boff = cw.packed ? 0 : warp;

  // One memory round trip before the first TMA: the CTA's block-table row (independent
  // of the length), each warp's first STAGES block ids and the shard length are loaded
  // together; lane 0 of every warp then issues its first copies before the CTA barrier.
  const int32_t blo = cw.blo;
  const int64_t row0 = (int64_t)max(b, 0) * sd.max_blocks + blo;
  const int nb_tab = cw.packed ? (b < 0 ? 0 : min(kPackMaxBlocks, sd.max_blocks))
                               : max(min(cw.nb, sd.max_blocks - blo), 0);
  constexpr int kIdPerThread = kBtMax / (kWarps * 32);
  int32_t idv[kIdPerThread];
#pragma unroll
  for (int r = 0; r < kIdPerThread; ++r) {
    const int i = cw.packed ? lane + 32 * r : threadIdx.x + r * kWarps * 32;
    idv[r] = i < nb_tab ? __ldg(sd.bt + row0 + i) : 0;
  }
  int32_t first[STAGES];
#pragma unroll
  for (int k = 0; k < STAGES; ++k)
    first[k] = (lane == 0 && boff + k * bstride < nb_tab) ? __ldg(sd.bt + row0 + boff + k * bstride) : 0;
  const int32_t* ks = P.kv_split + (int64_t)max(b, 0) * (P.n_shards + 1) + sd.shard_id;
  const int32_t len = b < 0 ? 0 : max(__ldg(ks + 1) - __ldg(ks), 0);
  const int32_t nblk = (len + 15) >> 4;
  const int32_t nb_cta = cw.packed ? min(nblk, nb_tab) : max(min(nblk, blo + cw.nb) - blo, 0);
  const int nparts = cw.nparts < 0 ? P.nsplit : cw.nparts;

  int32_t* s_bt = reinterpret_cast<int32_t*>(smem + S::kBtOff) + (cw.packed ? warp * (kBtMax / kWarps) : 0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kBarOff) + warp * STAGES;
  uint8_t* s_pt = smem + S::kPOff + warp * 8 * 16 * 2;
  uint8_t* ring = smem + warp * STAGES * S::kStage;

  const int nmine = cw.packed ? nb_cta : (nb_cta > warp ? (nb_cta - warp + kWarps - 1) / kWarps : 0);
  const int gm = p.model_head_lo + g;
  const int head = sd.pool_head_lo + g;
  const CUtensorMap* tmap = &tm.m[js];
  uint64_t policy = 0;
  const uint32_t ring_u32 = ptx::smem_u32(ring);
  auto issue = [&](int k, int32_t phys) {  // lane 0 only
    const int s = k % STAGES;
    const int32_t row_k = sd.layer_row0 + ((phys * 2 + 0) * sd.pool_hkv + head) * 16;
    const int32_t row_v = row_k + sd.pool_hkv * 16;
    const uint32_t st = ring_u32 + s * S::kStage;
    ptx::mbar_expect_tx(&bars[s], 2 * 16 * D * 2);
#pragma unroll
    for (int bx = 0; bx < NB; ++bx) {
      tma_load_2d(st + bx * S::kBox, tmap, 64 * bx, row_k, &bars[s], policy);
      tma_load_2d(st + (NB + bx) * S::kBox, tmap, 64 * bx, row_v, &bars[s], policy);
    }
  };
  uint64_t* cbar = reinterpret_cast<uint64_t*>(smem + S::kClBarOff);
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) ptx::mbar_init(&bars[s], 1);
    if (p.cl && warp == 0) {
      ptx::mbar_init(&cbar[0], 1);
      ptx::mbar_init(&cbar[1], 1);
    }
    ptx::fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
    policy = ptx::policy_evict_first();
#pragma unroll
    for (int k = 0; k < STAGES; ++k)
      if (k < nmine) issue(k, first[k]);
  }
#pragma unroll
  for (int r = 0; r < kIdPerThread; ++r) {
    const int i = cw.packed ? lane + 32 * r : threadIdx.x + r * kWarps * 32;
    if (i < nb_cta) s_bt[i] = idv[r];
  }
  __syncthreads();  // block table + barrier inits visible to the CTA
  if (p.cl) ptx::cluster_arrive_release();  // ... and the cluster barriers to the cluster
  // Programmatic dependent launch (BS_ATTN_PDL): this grid may start while the previous
  // kernel on the stream drains.  Everything above -- block table, kv_split, the first
  // K/V stages in flight -- reads only step inputs (the caller's contract); q, the outputs
  // and the workspace (which the previous launch may still be merging from) come after the
  // wait, which returns once that kernel has completed and its writes are visible.
  // The next launch on the stream, if it is a programmatic dependent, may start once every
  // CTA of this grid has triggered: right away for multi-wave grids (it fills the slots of
  // the last wave's tail), after the main loop for single-wave grids (its prologue and first
  // K/V stages then overlap this grid's epilogue instead of competing with its streaming).
  if (p.trig_late == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (p.pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    BS_TL(6);
  }

  // q^T B-fragments (bf16 pairs) for head n = gq (zero padding for n >= G)
  uint32_t bq[KS][2];
  {
    const uint32_t* qrow = reinterpret_cast<const uint32_t*>(P.q + ((int64_t)max(b, 0) * p.hq + gm * G + gq) * D);
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      bq[kk][0] = gq < G && b >= 0 ? __ldg(qrow + 8 * kk + tq) : 0u;
      bq[kk][1] = gq < G && b >= 0 ? __ldg(qrow + 8 * kk + 4 + tq) : 0u;
    }
  }

  float oacc[KS][4];  // O^T: rows dims 16*mt + gq (+8), cols heads 2*tq, 2*tq+1
#pragma unroll
  for (int mt = 0; mt < KS; ++mt) oacc[mt][0] = oacc[mt][1] = oacc[mt][2] = oacc[mt][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};

  const uint32_t pt_u32 = ptx::smem_u32(s_pt);
  const int lr = (lane & 7) + 8 * ((lane >> 3) & 1);  // K rows (ldmatrix matrix = lane / 8)
  const int kh = lane >> 4;                          // K: which 8-dim half of the k-step
  const int vtok = (lane & 7) + 8 * (lane >> 4);     // V rows (tokens)
  const int vh = (lane >> 3) & 1;                    // V: which 8-dim half of the m-tile

  for (int k = 0; k < nmine; ++k) {
    const int s = k % STAGES;
    ptx::mbar_wait(&bars[s], (uint32_t)((k / STAGES) & 1));
    __syncwarp();
    if (k == 0 && warp == 0) BS_TL(1);
    const int blk = blo + boff + k * bstride;
    const int nvalid = min(16, len - blk * 16);
    const uint32_t st = ring_u32 + s * S::kStage;

    // ---- S^T = K q^T ----------------------------------------------------------------
    float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      uint32_t a[4];
      ldsm_x4(st + (kk / 4) * S::kBox + swz(lr, 2 * (kk % 4) + kh), a);
      mma_bf16_16816(sc, a, bq[kk][0], bq[kk][1]);
    }
    // sc[0] = (tok gq, head 2tq), sc[1] = (gq, 2tq+1), sc[2] = (gq+8, 2tq), sc[3] = (gq+8, 2tq+1)
    const bool v0 = gq < nvalid, v1 = gq + 8 < nvalid;
    sc[0] = v0 ? sc[0] * p.scale_log2 : -INFINITY;
    sc[1] = v0 ? sc[1] * p.scale_log2 : -INFINITY;
    sc[2] = v1 ? sc[2] * p.scale_log2 : -INFINITY;
    sc[3] = v1 ? sc[3] * p.scale_log2 : -INFINITY;
    float mx0 = fmaxf(sc[0], sc[2]), mx1 = fmaxf(sc[1], sc[3]);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    }
    const float mn0 = fmaxf(m_run[0], mx0), mn1 = fmaxf(m_run[1], mx1);  // finite
    const float al0 = exp2f(m_run[0] - mn0), al1 = exp2f(m_run[1] - mn1);
    m_run[0] = mn0;
    m_run[1] = mn1;
    const float p0 = exp2f(sc[0] - mn0), p1 = exp2f(sc[1] - mn1);
    const float p2 = exp2f(sc[2] - mn0), p3 = exp2f(sc[3] - mn1);
    l_run[0] = l_run[0] * al0 + (p0 + p2);
    l_run[1] = l_run[1] * al1 + (p1 + p3);
    // P^T (bf16) -> smem [head][16 tokens]
    {
      const uint32_t a = pt_u32 + ((2 * tq) * 16 + gq) * 2;
      const __nv_bfloat16 b0 = __float2bfloat16_rn(p0), b1 = __float2bfloat16_rn(p1);
      const __nv_bfloat16 b2 = __float2bfloat16_rn(p2), b3 = __float2bfloat16_rn(p3);
      asm volatile("st.shared.b16 [%0], %1;" ::"r"(a), "h"(*reinterpret_cast<const uint16_t*>(&b0)));
      asm volatile("st.shared.b16 [%0], %1;" ::"r"(a + 32), "h"(*reinterpret_cast<const uint16_t*>(&b1)));
      asm volatile("st.shared.b16 [%0], %1;" ::"r"(a + 16), "h"(*reinterpret_cast<const uint16_t*>(&b2)));
      asm volatile("st.shared.b16 [%0], %1;" ::"r"(a + 48), "h"(*reinterpret_cast<const uint16_t*>(&b3)));
    }
    if (nvalid < 16) {  // pad rows of the V page may hold anything (NaN): zero them
      for (int i = lane; i < (16 - nvalid) * NB * 8; i += 32) {
        const int r = nvalid + i / (NB * 8), rem = i % (NB * 8);
        *reinterpret_cast<uint4*>(ring + s * S::kStage + (NB + rem / 8) * S::kBox + r * 128 +
                                  (rem % 8) * 16) = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    __syncwarp();
    uint32_t bp0, bp1;  // P^T B-fragment: head n = gq, tokens 2tq(+1), 2tq+8(+9)
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(bp0) : "r"(pt_u32 + gq * 32 + 4 * tq));
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(bp1) : "r"(pt_u32 + gq * 32 + 16 + 4 * tq));

    // ---- O^T = alpha O^T + V^T P^T ------------------------------------------------------
    const uint32_t vb = st + NB * S::kBox;
#pragma unroll
    for (int mt = 0; mt < KS; ++mt) {
      oacc[mt][0] *= al0;
      oacc[mt][1] *= al1;
      oacc[mt][2] *= al0;
      oacc[mt][3] *= al1;
      uint32_t a[4];
      ldsm_x4_t(vb + (mt / 4) * S::kBox + swz(vtok, 2 * (mt % 4) + vh), a);
      mma_bf16_16816(oacc[mt], a, bp0, bp1);
    }
    __syncwarp();
    if (lane == 0 && k + STAGES < nmine) {
      ptx::fence_proxy_async_smem();
      issue(k + STAGES, s_bt[boff + (k + STAGES) * bstride]);
    }
    __syncwarp();
  }
  if (p.trig_late == 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ---- per-warp state -> shared memory, then the common CTA epilogue --------------------
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    float x = l_run[j];
    x += __shfl_xor_sync(0xffffffffu, x, 4);
    x += __shfl_xor_sync(0xffffffffu, x, 8);
    x += __shfl_xor_sync(0xffffffffu, x, 16);
    l_run[j] = x;
  }
  if (cw.packed) {  // this warp's request is complete: O = O~ / l, lse = m + ln l (merged out)
    if (b >= 0) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int h = 2 * tq + j;
        if (h < G) {
          const int64_t row = (int64_t)b * p.hq + gm * G + h;
          const float L = l_run[j];
          const bool any = L > 0.f;
#pragma unroll
          for (int mt = 0; mt < KS; ++mt) {
            P.out[row * D + 16 * mt + gq] = __float2bfloat16_rn(any ? oacc[mt][j] / L : 0.f);
            P.out[row * D + 16 * mt + gq + 8] = __float2bfloat16_rn(any ? oacc[mt][2 + j] / L : 0.f);
          }
          if (gq == 0 && P.lse) P.lse[row] = any ? m_run[j] * kLn2 + logf(L) : -INFINITY;
        }
      }
    }
    return;
  }
  __syncthreads();  // rings idle: reuse them for the combine
  BS_TL(2);
  float* s_acc = reinterpret_cast<float*>(smem);  // [kWarps][G][D]
  float* s_ml = reinterpret_cast<float*>(smem + S::kMlOff);
  float* s_w = reinterpret_cast<float*>(smem + S::kWOff);
  int* s_flag = reinterpret_cast<int*>(smem + S::kFlagOff);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int h = 2 * tq + j;
    if (h < G) {
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        s_acc[(warp * G + h) * D + 16 * mt + gq] = oacc[mt][j];
        s_acc[(warp * G + h) * D + 16 * mt + gq + 8] = oacc[mt][2 + j];
      }
      if (gq == 0) {
        s_ml[(warp * G + h) * 2] = m_run[j];
        s_ml[(warp * G + h) * 2 + 1] = l_run[j];
      }
    }
  }
  __syncthreads();
  if (p.cl)
    cluster_combine_merge<D, G>(P, p.hq, b, gm, nparts, s_acc, s_ml, s_w,
                                reinterpret_cast<float*>(smem + S::kRecvOff), cbar, tl_base_);
  else
    cta_combine_and_store<D, G>(P, p.hq, p.hkv, b, g, gm, cw.slot, nparts, s_acc, s_ml, s_w,
                                s_flag, tl_base_);
#ifdef BS_TIMELINE
  BS_TL(4);
  {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const unsigned lin = tl_base_ + blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (threadIdx.x == 0 && lin < kTlCtas)
      g_timeline[lin][5] = smid | ((unsigned long long)(nparts == 1 || (p.cl ? ptx::cluster_ctarank() == 0 : s_flag[0])) << 16) |
                           ((unsigned long long)nb_cta << 20);
  }
#endif
}

// Pipeline depth / residency per (head_dim, group): STAGES blocks (K+V pages) per warp in
// flight, MINB CTAs per SM.  G <= 4 fits 3 CTAs/SM (registers <= 168) with a 2-deep ring
// (d=128); G = 8 needs more registers and keeps 2 CTAs/SM with a 3-deep ring.  Both give
// ~192 KiB of KV in flight per SM.  BS_ATTN_VARIANT=1 forces the 2-CTA/3-deep variant.
struct Variant {
  int stages, minb;
  bool mma;
};

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

int alt_variant() {
  static int v = env_int("BS_ATTN_VARIANT", 0);
  return v;
}

bool use_mma(int G) {
  // 2 (default): tensor cores for every G; 1: only for G >= 4; 0: CUDA cores for every G
  static int v = env_int("BS_ATTN_MMA", 2);
  return (v == 1 && G >= 4) || v == 2;
}

// The default (tensor-core) variant, independent of the environment: the range plan of a
// problem shared by several GPUs uses it (rank-invariant inputs only).
Variant default_variant(int d) { return d == 128 ? Variant{2, 3, true} : Variant{4, 3, true}; }

Variant variant_for(int d, int G) {
  if (use_mma(G)) return default_variant(d);
  if (alt_variant() == 1) return d == 128 ? Variant{3, 2, false} : Variant{6, 2, false};
  if (d == 128) return G <= 4 ? Variant{2, 3, false} : Variant{3, 2, false};
  return G <= 4 ? Variant{4, 3, false} : Variant{6, 2, false};
}

constexpr int kMaxProbShards = 16;  // shards of one problem (over all GPUs)

struct Plan {
  int bps;                        // blocks per CTA range (common to the problem's shards)
  int nsplit;                     // total CTA ranges per (request, kv-head)
  int split_off[kMaxProbShards];  // first range of each shard
  int nsplit_s[kMaxProbShards];   // ranges of each shard
  size_t ws_bytes, off_ml, off_cnt;
};

// Split-K planning over the launch's shards (one for bs_split_decode_attention, all the
// local shards for bs_split_decode_attention_local): pick the CTA range length that
// minimises waves x blocks-per-CTA (+ a fixed per-CTA cost), i.e. fills the SM slots.
// hkv: kv heads handled by the launch (grid.y); hq: q heads of the model (partial rows).
// Problems whose shards live on several GPUs (bs_split_decode_attention_tasks) are planned
// by every GPU that runs one of their shards, and the last-arriver merge needs the same
// range cut everywhere: their plan uses only rank-invariant inputs -- the problem's shape,
// a fixed slot count (a B200's 148 SMs x 3 resident CTAs) and no environment switches.
constexpr int kInvariantSlots = 148 * 3;

bs_status make_plan(int batch, int G, int hq, int hkv, int d, int n_local, const int* max_blocks,
                    bool merged, Plan* out, bool rank_invariant = false) {
  if (n_local < 1 || n_local > kMaxProbShards)
    return set_error(BS_ERR_INVALID_ARG, "attention plan: %d shards (1..%d)", n_local, kMaxProbShards);
  const int64_t slots = rank_invariant ? (int64_t)kInvariantSlots
                                       : (int64_t)sm_count(current_device()) * variant_for(d, G).minb;
  const int64_t base = (int64_t)batch * hkv;
  int mb_max = 1;
  for (int j = 0; j < n_local; ++j) mb_max = std::max(mb_max, max_blocks[j]);
  const int min_bps = kWarps;
  // cap the blocks per CTA range: with mixed lengths the longest request's CTA is the
  // critical path; shorter ranges let the hardware scheduler balance them (BS_ATTN_MAX_BPS)
  static const int max_bps = [] {
    const char* e = getenv("BS_ATTN_MAX_BPS");
    const int x = e ? atoi(e) : 0;
    return x > 0 ? x : kBtMax;
  }();
  // experiment switch: force the number of ranges per shard width
  static const int forced_ns = [] {
    const char* e = getenv("BS_ATTN_NSPLIT");
    return e ? atoi(e) : 0;
  }();
  static const int plan_model = env_int("BS_ATTN_PLAN", 1);  // 0: round-1 planner everywhere
  int best_bps = -1;
  double best = 1e300;
  if (forced_ns > 0 && !rank_invariant)
    best_bps = std::min(kBtMax, std::max(min_bps, (mb_max + forced_ns - 1) / forced_ns));
  // Few (request, kv-head) pairs -- fewer than the CTA slots, so the blocks of each pair
  // are cut into ranges to fill the GPU (C3: 8 or 64 pairs).  Among the cuts that run as
  // ONE wave, a bandwidth / latency model picks (r02 planner sweep).
  // Streaming takes the longer of
  //   * all KV bytes at min(HBM read ceiling, bytes in flight / latency), the bytes in flight
  //     being every CTA's ring (kWarps x STAGES blocks), and
  //   * the busiest SM's bytes (CTAs spread evenly over the SMs) at one SM's rate;
  // ranges are a multiple of kWarps blocks (the slowest of the four warp pipelines sets a
  // CTA's time), and the last arriver's merge costs a round trip plus every partial at one
  // SM's L2 rate.  Constants measured on a B200: 7.0 TB/s, 1.5 us, 45 GB/s per SM, merge
  // 1.5 us + 25 GB/s.
  if (best_bps < 0 && plan_model && base < slots) {
    const Variant v = rank_invariant ? default_variant(d) : variant_for(d, G);
    const int sms = rank_invariant ? kInvariantSlots / 3 : sm_count(current_device());
    const double blk = 2.0 * 16 * d * 2;                      // K + V page of one block
    const double inflight_cta = (double)kWarps * v.stages * blk;
    const double bw = 7.0e12, lat = 1.5e-6, r_sm = 45e9;
    double all_blocks = 0;
    for (int j = 0; j < n_local; ++j) all_blocks += max_blocks[j];
    const double total_bytes = (double)base * all_blocks * blk;
    for (int bps = min_bps; bps <= kBtMax; bps += kWarps) {
      int total = 0;
      for (int j = 0; j < n_local; ++j) total += (max_blocks[j] + bps - 1) / bps;
      const int64_t ctas = base * total;
      if (total > kMaxSplit || ctas > slots) continue;   // one wave only
      const double bw_eff = std::min(bw, (double)ctas * inflight_cta / lat);
      const int64_t per_sm = (ctas + sms - 1) / sms;     // CTAs on the busiest SM
      double t = std::max(total_bytes / bw_eff, (double)per_sm * bps * blk / r_sm);
      if (total > 1) t += 1.5e-6 + (double)total * G * d * 4 / 25e9;
      if (t < best * (1 - 1e-9)) {
        best = t;
        best_bps = bps;
      }
      if (bps >= mb_max) break;  // one range per shard: longer ranges change nothing
    }
  }
  for (int pass = 0; pass < 2 && best_bps < 0; ++pass) {  // pass 1: without the cap
    const int cap =
        pass == 0 && !rank_invariant ? std::min(kBtMax, std::max(max_bps, min_bps)) : kBtMax;
    int last_bps = -1;
    for (int ns = 1; ns <= kMaxSplit; ++ns) {
      const int bps = std::max(min_bps, (mb_max + ns - 1) / ns);
      if (bps > cap || bps == last_bps) continue;
      last_bps = bps;
      int total = 0;
      for (int j = 0; j < n_local; ++j) total += (max_blocks[j] + bps - 1) / bps;
      if (total > kMaxSplit) continue;
      const int64_t ctas = base * total;
      const int64_t waves = (ctas + slots - 1) / slots;
      const bool partial = total > 1;
      const double cost = (double)waves * ((double)bps / kWarps + 2.0 + (partial ? 1.0 : 0.0));
      if (cost < best - 1e-9) {
        best = cost;
        best_bps = bps;
      }
      if (bps == min_bps) break;
    }
  }
  if (best_bps < 0)
    return set_error(BS_ERR_UNSUPPORTED, "max_blocks %d exceeds %d", mb_max, kBtMax * kMaxSplit);
  Plan pl{};
  pl.bps = best_bps;
  int off = 0;
  for (int j = 0; j < n_local; ++j) {
    pl.split_off[j] = off;
    pl.nsplit_s[j] = (max_blocks[j] + best_bps - 1) / best_bps;
    off += pl.nsplit_s[j];
  }
  pl.nsplit = off;
  (void)merged;
  if (pl.nsplit > 1) {
    const size_t parts = (size_t)batch * hq * pl.nsplit;
    pl.off_ml = parts * d * 4;
    pl.off_cnt = pl.off_ml + parts * 2 * 4;
    pl.ws_bytes = pl.off_cnt + (size_t)batch * hkv * 4;
  }
  *out = pl;
  return BS_OK;
}

// Launch with cudaLaunchKernelEx: programmatic stream serialisation (PDL: the grid may
// begin as soon as every CTA of the previous kernel on the stream has started and
// triggered; the kernel's griddepcontrol.wait orders what depends on that kernel) and / or
// a cluster of `cluster_x` CTAs along grid.x (cluster merge).
template <typename... KArgs, typename... Args>
bs_status launch_ex(void (*kern)(KArgs...), dim3 grid, int smem, cudaStream_t stream, bool pdl,
                    int cluster_x, const char* what, const Args&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kWarps * 32, 1, 1);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = (unsigned)cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = (unsigned)n;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
  if (e != cudaSuccess) return set_error(BS_ERR_CUDA, "%s (launch_ex): %s", what, cudaGetErrorString(e));
  return BS_OK;
}

template <typename... KArgs, typename... Args>
bs_status launch_pdl(void (*kern)(KArgs...), dim3 grid, int smem, cudaStream_t stream,
                     const char* what, const Args&... args) {
  return launch_ex(kern, grid, smem, stream, true, 1, what, args...);
}

// What the calling thread's last attention launch ran (bs_attention_last_launch).
struct LaunchInfo {
  int32_t ranges, merge, pdl, tensor_cores, stages;  // merge: 0 none, 1 last arriver, 2 cluster
};
int32_t merge_kind(const AttnParams& p) {
  if (p.pb[0].nsplit < 2) return 0;  // one range (or one per request, ragged): no merge
  return p.cl ? 2 : 1;
}
thread_local LaunchInfo g_last_launch{0, 0, 0, 0, 0};

int cluster_env() {  // A/B switch BS_ATTN_CLUSTER: 0 never, 1 single-wave launches, 2 always
  static int v = env_int("BS_ATTN_CLUSTER", 1);
  return v;
}

// Largest cluster the merge uses (BS_ATTN_CLUSTER_MAX, <= 16).  Clusters must sit in one
// GPC: 16-CTA clusters of a C3 B=1 launch (8 x 16 CTAs) were placed two CTAs to an SM on 28
// SMs (114 SMs used instead of 128) and lost more in the loop than the merge saved.
int cluster_max() {
  static int v = std::min(16, std::max(2, env_int("BS_ATTN_CLUSTER_MAX", 8)));
  return v;
}

int trig_exit_mode() {  // A/B switch BS_ATTN_TRIG_EXIT: 1 (default) trigger at exit for
  static int v = env_int("BS_ATTN_TRIG_EXIT", 1);  // one-wave grids too large to start beside
  return v ? 2 : 1;                                  // their predecessor; 0: after the loop
}

int deep_env() {  // A/B switch BS_ATTN_DEEP: 0 never use the 6-stage one-CTA-per-SM variant
  static int v = env_int("BS_ATTN_DEEP", 1);
  return v;
}

int pdl_env() {  // A/B switch BS_ATTN_PDL: 0 never, 1 every attention launch, unset: flags
  static int v = env_int("BS_ATTN_PDL", -1);
  return v;
}

template <int D, int G, int STAGES, int MINB>
bs_status launch_attn_v(const AttnParams& p, int batch, cudaStream_t stream) {
  using S = Smem<D, G, STAGES>;
  static std::atomic<uint64_t> configured{0};  // per-device function attribute
  const uint64_t bit = 1ull << (current_device() & 63);
  if (!(configured.load() & bit)) {
    cudaFuncSetAttribute(split_decode_attn<D, G, STAGES, MINB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, S::kTotal);
    configured.fetch_or(bit);
  }
  const dim3 grid = p.work ? dim3(p.grid_x * p.hkv, 1, 1) : dim3(p.grid_x, p.hkv, batch);
  g_last_launch = LaunchInfo{p.grid_x, merge_kind(p), p.pdl, 0, STAGES};
  if (p.pdl) return launch_pdl(split_decode_attn<D, G, STAGES, MINB>, grid, S::kTotal, stream,
                               "split_decode_attn", p);
  split_decode_attn<D, G, STAGES, MINB><<<grid, kWarps * 32, S::kTotal, stream>>>(p);
  return check_launch("split_decode_attn");
}

// Can clusters of `n` CTAs of this kernel be resident (GPC size, shared memory)?  Asked
// once per (device, n) with cudaOccupancyMaxActiveClusters.
template <int D, int G, int STAGES, int MINB>
bool cluster_fits(int n, int smem) {
  static std::mutex mu;
  static int known[64][17];  // 0 unknown, 1 yes, 2 no
  const int dev = current_device() & 63;
  std::lock_guard<std::mutex> g(mu);
  if (!known[dev][n]) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n, 1, 1);
    cfg.blockDim = dim3(kWarps * 32, 1, 1);
    cfg.dynamicSmemBytes = (size_t)smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)n;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    const cudaError_t e =
        cudaOccupancyMaxActiveClusters(&clusters, split_decode_attn_mma<D, G, STAGES, MINB>, &cfg);
    cudaGetLastError();
    known[dev][n] = (e == cudaSuccess && clusters > 0) ? 1 : 2;
  }
  return known[dev][n] == 1;
}

template <int D, int G, int STAGES, int MINB>
bs_status launch_attn_mma(const AttnParams& p_in, const TMaps& tm, int batch, cudaStream_t stream) {
  using S = MmaSmem<D, G, STAGES>;
  static std::atomic<uint64_t> configured{0};  // per-device function attributes
  const uint64_t bit = 1ull << (current_device() & 63);
  if (!(configured.load() & bit)) {
    cudaFuncSetAttribute(split_decode_attn_mma<D, G, STAGES, MINB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, S::kTotal);
    cudaFuncSetAttribute(split_decode_attn_mma<D, G, STAGES, MINB>,
                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    configured.fetch_or(bit);
  }
  AttnParams p = p_in;
  // cluster merge: the partials of a (request, kv-head) must fit in the leader's idle ring
  // (plus the merge's 2 KiB scratch), and clusters of grid.x CTAs must be schedulable
  if (p.cl) {
    const int need = S::kRecvOff + p.grid_x * SmemParts<D, G>::kPF * 4 + 2048;
    if (p.work || p.grid_x < 2 || p.grid_x > 16 || need > S::kRing ||
        !cluster_fits<D, G, STAGES, MINB>(p.grid_x, S::kTotal))
      p.cl = 0;
  }
  const dim3 grid = p.work ? dim3(p.grid_x * p.hkv, 1, 1) : dim3(p.grid_x, p.hkv, batch);
  g_last_launch = LaunchInfo{p.grid_x, merge_kind(p), p.pdl, 1, STAGES};
  if (p.pdl || p.cl)
    return launch_ex(split_decode_attn_mma<D, G, STAGES, MINB>, grid, S::kTotal, stream, p.pdl != 0,
                     p.cl ? p.grid_x : 1, "split_decode_attn_mma", p, tm);
  split_decode_attn_mma<D, G, STAGES, MINB><<<grid, kWarps * 32, S::kTotal, stream>>>(p, tm);
  return check_launch("split_decode_attn_mma");
}

template <int D, int G>
bs_status launch_attn_t(const AttnParams& p, const TMaps* tm, int batch, cudaStream_t stream) {
  const Variant v = variant_for(D, G);
  if (v.mma && tm) {
    // one CTA per SM: 6 K/V stages per warp (192 KiB of ring) -- a programmatic dependent
    // then prefetches most of its range while the previous launch finishes
    if constexpr (D == 128)
      if (p.deep) return launch_attn_mma<D, G, 6, 1>(p, *tm, batch, stream);
    if constexpr (D == 128) return launch_attn_mma<D, G, 2, 3>(p, *tm, batch, stream);
    else return launch_attn_mma<D, G, 4, 3>(p, *tm, batch, stream);
  }
  if constexpr (D == 128) {
    if (v.stages == 2) return launch_attn_v<D, G, 2, 3>(p, batch, stream);
    return launch_attn_v<D, G, 3, 2>(p, batch, stream);
  } else {
    if (v.stages == 4) return launch_attn_v<D, G, 4, 3>(p, batch, stream);
    return launch_attn_v<D, G, 6, 2>(p, batch, stream);
  }
}

template <int D>
bs_status launch_attn_d(const AttnParams& p, const TMaps* tm, int G, int batch, cudaStream_t stream) {
  switch (G) {
    case 1: return launch_attn_t<D, 1>(p, tm, batch, stream);
    case 2: return launch_attn_t<D, 2>(p, tm, batch, stream);
    case 4: return launch_attn_t<D, 4>(p, tm, batch, stream);
    case 8: return launch_attn_t<D, 8>(p, tm, batch, stream);
  }
  return set_error(BS_ERR_UNSUPPORTED, "query group G=%d not in {1,2,4,8}", G);
}

}  // namespace
}  // namespace bs

// Encode (once) a 2D tensor map over the whole pool -- rows = (layer, block, K|V, head,
// slot), inner dim = head_dim -- with 16 x 64 boxes and the 128-byte swizzle the
// tensor-core kernel's ldmatrix addressing expects.
static const CUtensorMap* pool_tensor_map(const bs_kv_pool* cpool) {
  bs_kv_pool* pool = const_cast<bs_kv_pool*>(cpool);
  std::lock_guard<std::mutex> g(pool->mu);
  if (pool->tmap_state == 0) {
    using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);
    static Enc enc = nullptr;
    if (!enc) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess)
        enc = reinterpret_cast<Enc>(fn);
    }
    const bs_kv_pool_desc& d = pool->desc;
    const uint64_t rows = (uint64_t)d.num_layers * d.num_blocks * 2 * d.num_kv_heads * 16;
    pool->tmap_state = -1;
    if (enc && !pool->host && rows < (1ull << 31)) {
      const cuuint64_t dims[2] = {(cuuint64_t)d.head_dim, rows};
      const cuuint64_t strides[1] = {(cuuint64_t)d.head_dim * 2};
      const cuuint32_t box[2] = {64, 16};
      const cuuint32_t estr[2] = {1, 1};
      if (enc(&pool->tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pool->base, dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
        pool->tmap_state = 1;
    }
    cudaGetLastError();
    if (pool->tmap_state != 1 && !pool->host && !getenv("BS_QUIET"))
      // not silent: the CUDA-core kernel (correct, slower at G >= 4) serves this pool; the
      // launch is also visible as tensor_cores = 0 in bs_attention_last_launch
      fprintf(stderr,
              "banaserve: no TMA tensor map for a pool (%llu rows%s); its attention launches use "
              "the CUDA-core kernel\n",
              (unsigned long long)rows, enc ? "" : ", cuTensorMapEncodeTiled unavailable");
  }
  return pool->tmap_state == 1 ? &pool->tmap : nullptr;
}

namespace {

struct LaunchArgs {
  int n_local;
  const bs_kv_pool* pools[bs::kMaxLocal];
  const int32_t* bts[bs::kMaxLocal];
  int32_t max_blocks[bs::kMaxLocal];
  int32_t shard_ids[bs::kMaxLocal];
  int32_t pool_head_lo, model_head_lo, n_kv_heads, num_kv_heads_total;
  int32_t layer, batch, num_q_heads, n_shards;
  const void* q;
  const int32_t* kv_split;
  float scale;
  bool merged;
  float *o, *m, *l;
  void* out;
  float* lse;
  void* workspace;
  size_t workspace_bytes;
  void* stream;
  const int32_t* work;  // ragged plan (device int4 items) or NULL
  int32_t n_work, max_parts;
  uint32_t flags;       // BS_ATTN_PDL | BS_ATTN_NO_CLUSTER
};

bs_status validate_common(const LaunchArgs& a, int* G_out) {
  BS_REQUIRE(a.n_local >= 1 && a.n_local <= bs::kMaxLocal, "attention: %d local shards (1..%d)",
             a.n_local, bs::kMaxLocal);
  const bs_kv_pool* p0 = a.pools[0];
  for (int j = 0; j < a.n_local; ++j) {
    const bs_kv_pool* pj = a.pools[j];
    BS_REQUIRE(pj, "attention: NULL pool");
    BS_REQUIRE(!pj->host, "attention: host-tier pools are fetched first, not read");
    BS_REQUIRE(pj->desc.head_dim == p0->desc.head_dim && pj->desc.num_layers == p0->desc.num_layers,
               "attention: local shards must share head_dim / num_layers");
    BS_REQUIRE(a.pool_head_lo >= 0 && a.pool_head_lo + a.n_kv_heads <= pj->desc.num_kv_heads,
               "attention: head range [%d,+%d) outside pool (%d)", a.pool_head_lo, a.n_kv_heads,
               pj->desc.num_kv_heads);
    BS_REQUIRE(a.max_blocks[j] >= 1, "attention: max_blocks < 1");
    BS_REQUIRE(a.shard_ids[j] >= 0 && a.shard_ids[j] < a.n_shards, "attention: shard %d of %d",
               a.shard_ids[j], a.n_shards);
  }
  BS_REQUIRE(a.layer >= 0 && a.layer < p0->desc.num_layers, "attention: layer %d out of range", a.layer);
  BS_REQUIRE(a.batch >= 0, "attention: batch < 0");
  BS_REQUIRE(a.num_kv_heads_total >= 1 && a.num_q_heads >= a.num_kv_heads_total &&
                 a.num_q_heads % a.num_kv_heads_total == 0,
             "attention: num_q_heads %d not a multiple of Hkv %d", a.num_q_heads, a.num_kv_heads_total);
  BS_REQUIRE(a.n_kv_heads >= 1 && a.model_head_lo >= 0 &&
                 a.model_head_lo + a.n_kv_heads <= a.num_kv_heads_total,
             "attention: model head range [%d,+%d) outside %d", a.model_head_lo, a.n_kv_heads,
             a.num_kv_heads_total);
  BS_REQUIRE(a.n_shards >= 1, "attention: n_shards < 1");
  BS_REQUIRE(a.scale > 0.f && a.scale == a.scale, "attention: bad scale");
  const int G = a.num_q_heads / a.num_kv_heads_total;
  if (G != 1 && G != 2 && G != 4 && G != 8)
    return bs::set_error(BS_ERR_UNSUPPORTED, "query group G=%d not in {1,2,4,8}", G);
  *G_out = G;
  return BS_OK;
}

bs_status run_attention(const LaunchArgs& a) {
  int G = 0;
  bs_status st = validate_common(a, &G);
  if (st != BS_OK) return st;
  if (a.batch == 0) return BS_OK;
  BS_REQUIRE(a.q && a.kv_split, "attention: NULL q / kv_split");
  for (int j = 0; j < a.n_local; ++j) BS_REQUIRE(a.bts[j], "attention: NULL block table");
  if (a.merged) BS_REQUIRE(a.out, "attention: NULL out");
  else BS_REQUIRE(a.o && a.m && a.l, "attention: NULL o / m / l");
  BS_REQUIRE(((uintptr_t)a.q & 15) == 0 && ((uintptr_t)(a.merged ? a.out : (void*)a.o) & 15) == 0,
             "attention: q / output must be 16-B aligned");
  const int d = a.pools[0]->desc.head_dim;
  bs::Plan pl;
  if (a.work) {  // ragged plan: ranges come from the work list, slots up to max_parts
    BS_REQUIRE(a.n_work >= 1 && a.max_parts >= 1 && a.max_parts <= bs::kMaxSplit,
               "attention: ragged plan with %d items / %d parts", a.n_work, a.max_parts);
    BS_REQUIRE(((uintptr_t)a.work & 15) == 0, "attention: work list must be 16-B aligned");
    pl = bs::Plan{};
    pl.bps = bs::kBtMax;
    pl.nsplit = a.max_parts;
    for (int j = 0; j < a.n_local; ++j) pl.split_off[j] = 0;
    if (a.max_parts > 1) {
      const size_t parts = (size_t)a.batch * a.num_q_heads * a.max_parts;
      pl.off_ml = parts * d * 4;
      pl.off_cnt = pl.off_ml + parts * 2 * 4;
      pl.ws_bytes = pl.off_cnt + (size_t)a.batch * a.n_kv_heads * 4;
    }
  } else {
    st = bs::make_plan(a.batch, G, a.num_q_heads, a.n_kv_heads, d, a.n_local, a.max_blocks, a.merged, &pl);
    if (st != BS_OK) return st;
  }
  BS_REQUIRE(pl.ws_bytes == 0 || (a.workspace && a.workspace_bytes >= pl.ws_bytes &&
                                  ((uintptr_t)a.workspace & 15) == 0),
             "attention: workspace needs %zu bytes (got %zu)", pl.ws_bytes, a.workspace_bytes);
  bs::AttnParams p{};
  p.n_local = a.n_local;
  bs::TMaps tm;
  bool have_maps = bs::variant_for(d, G).mma;
  for (int j = 0; j < a.n_local; ++j) {
    const bs_kv_pool* pool = a.pools[j];
    bs::ShardDesc& sd = p.sh[j];
    sd.kv = pool->base + (size_t)a.layer * pool->layer_bytes;
    sd.chunk_bytes = (int64_t)pool->chunk_bytes;
    sd.v_off = (int64_t)pool->desc.num_kv_heads * pool->page_bytes;
    sd.bt = a.bts[j];
    sd.max_blocks = a.max_blocks[j];
    sd.shard_id = a.shard_ids[j];
    sd.bps = pl.bps;
    sd.split_off = pl.split_off[j];
    sd.prob = 0;
    sd.range_base = pl.split_off[j];
    sd.pool_hkv = pool->desc.num_kv_heads;
    sd.pool_head_lo = a.pool_head_lo;
    sd.layer_row0 =
        (int32_t)((int64_t)a.layer * pool->desc.num_blocks * 2 * pool->desc.num_kv_heads * 16);
    if (have_maps) {
      const CUtensorMap* m = pool_tensor_map(pool);
      if (m) tm.m[j] = *m;
      else have_maps = false;
    }
  }
  p.scale_log2 = a.scale * bs::kLog2e;
  p.hq = a.num_q_heads;
  p.hkv = a.n_kv_heads;
  p.model_head_lo = a.model_head_lo;
  p.grid_x = a.work ? a.n_work : pl.nsplit;
  p.work = reinterpret_cast<const int4*>(a.work);
  {  // programmatic dependent launch of flagged launches (BS_ATTN_PDL=0/1 overrides)
    const int64_t ctas = (int64_t)p.grid_x * a.n_kv_heads * (a.work ? 1 : a.batch);
    const int64_t slots = (int64_t)bs::sm_count(bs::current_device()) * bs::variant_for(d, G).minb;
    const int env = bs::pdl_env();
    const int64_t sms = bs::sm_count(bs::current_device());
    // Where THIS grid lets its dependent (the next layer's launch) start -- trig_late:
    //  0 multi-wave: once every CTA has started (the next grid fills the last wave's tail);
    //  1 one wave within half the slots: after the main loops, so the next grid's prologue
    //    and first K/V stages overlap this grid's epilogue, not its streaming (C3 B=1: 11.9
    //    -> 10.8 us; triggering at entry gained nothing);
    //  2 larger one-wave grids: at exit -- a next grid started earlier would be placed in
    //    whatever slots are free, unevenly, and lose its tail (C3 B=8: 42.9 -> 44.9 us).
    // The flag never changes the range cut: flagged and plain launches are bitwise identical.
    p.pdl = env >= 0 ? env : ((a.flags & BS_ATTN_PDL) ? 1 : 0);
    p.trig_late = ctas > slots ? 0 : (2 * ctas <= slots ? 1 : bs::trig_exit_mode());
    // ... and, for such a PDL launch of at most one CTA per SM, 6 K/V stages per warp: it
    // prefetches 24 of a 32-block range before the wait (C3 B=1 10.8 -> 9.9 us; without PDL
    // the deeper ring is slower, 11.8 -> 12.5 us)
    p.deep = (p.pdl && !a.work && d == 128 && ctas <= sms && bs::deep_env()) ? 1 : 0;
    // cluster merge: single-wave launches with 2..16 ranges per (request,
    // kv-head) -- the epilogue is their critical path; BS_ATTN_CLUSTER=0 off, 2 any wave count
    const int cl_env = bs::cluster_env();
    p.cl = (!a.work && !(a.flags & BS_ATTN_NO_CLUSTER) && pl.nsplit >= 2 &&
            pl.nsplit <= bs::cluster_max() && cl_env != 0 &&
            (cl_env == 2 || ctas <= slots)) ? 1 : 0;
  }
#ifdef BS_TIMELINE
  p.tl_base = (bs::g_tl_launches.fetch_add(1) & 1) * (bs::kTlCtas / 2);
#endif
  bs::ProbDesc& P = p.pb[0];
  P.q = static_cast<const __nv_bfloat16*>(a.q);
  P.kv_split = a.kv_split;
  P.n_shards = a.n_shards;
  P.nsplit = pl.nsplit;
  P.merged = a.merged ? 1 : 0;
  P.o = a.o;
  P.m = a.m;
  P.l = a.l;
  P.out = static_cast<__nv_bfloat16*>(a.out);
  P.lse = a.lse;
  if (pl.ws_bytes) {
    uint8_t* ws = static_cast<uint8_t*>(a.workspace);
    P.ws_o = reinterpret_cast<float*>(ws);
    P.ws_ml = reinterpret_cast<float*>(ws + pl.off_ml);
    P.ws_cnt = reinterpret_cast<int32_t*>(ws + pl.off_cnt);
  }
  cudaStream_t s = static_cast<cudaStream_t>(a.stream);
  for (int j = 0; j < a.n_local; ++j)
    BS_DEBUG_CHECK(bs::debug_check_table(a.kv_split, a.n_shards, a.shard_ids[j], a.batch, a.bts[j],
                                         a.max_blocks[j], a.pools[j]->desc.num_blocks, s,
                                         "attention block table / kv_split"));
  const bs::TMaps* tmp = have_maps ? &tm : nullptr;
  if (d == 128) return bs::launch_attn_d<128>(p, tmp, G, a.batch, s);
  return bs::launch_attn_d<64>(p, tmp, G, a.batch, s);
}

bs_status workspace_impl(int n_local, const bs_kv_pool* const* pools, const int32_t* max_blocks,
                         int32_t batch, int32_t n_kv_heads, int32_t num_kv_heads_total,
                         int32_t num_q_heads, bool merged, size_t* bytes) {
  BS_REQUIRE(pools && bytes && max_blocks, "attention workspace size: NULL argument");
  BS_REQUIRE(n_local >= 1 && n_local <= bs::kMaxLocal, "attention workspace size: %d shards", n_local);
  for (int j = 0; j < n_local; ++j)
    BS_REQUIRE(pools[j] && max_blocks[j] >= 1, "attention workspace size: bad pool / max_blocks");
  BS_REQUIRE(batch >= 0 && n_kv_heads >= 1 && num_kv_heads_total >= 1 &&
                 num_q_heads >= num_kv_heads_total && num_q_heads % num_kv_heads_total == 0,
             "attention workspace size: bad batch / heads");
  bs::Plan pl;
  bs_status st = bs::make_plan(batch, num_q_heads / num_kv_heads_total, num_q_heads, n_kv_heads,
                               pools[0]->desc.head_dim, n_local, max_blocks, merged, &pl);
  if (st != BS_OK) return st;
  *bytes = pl.ws_bytes;
  return BS_OK;
}

}  // namespace

extern "C" {

#ifdef BS_TIMELINE
// Diagnostics build only (not declared in include/banaserve.h): copy / clear the stamps.
bs_status bs_timeline_read(void* host, size_t bytes) {
  const size_t n = std::min(bytes, sizeof(bs::g_timeline));
  const cudaError_t e = cudaMemcpyFromSymbol(host, bs::g_timeline, n);
  return e == cudaSuccess ? BS_OK : bs::set_error(BS_ERR_CUDA, "timeline: %s", cudaGetErrorString(e));
}
bs_status bs_timeline_reset(void) {
  bs::g_tl_launches = 0;
  static unsigned long long zeros[bs::kTlCtas][bs::kTlCols];
  const cudaError_t e = cudaMemcpyToSymbol(bs::g_timeline, zeros, sizeof(zeros));
  return e == cudaSuccess ? BS_OK : bs::set_error(BS_ERR_CUDA, "timeline: %s", cudaGetErrorString(e));
}
#endif

bs_status bs_attention_last_launch(int32_t* ranges, int32_t* merge, int32_t* pdl,
                                   int32_t* tensor_cores, int32_t* stages) {
  BS_REQUIRE(ranges && merge && pdl && tensor_cores && stages,
             "bs_attention_last_launch: NULL argument");
  const bs::LaunchInfo& i = bs::g_last_launch;
  *ranges = i.ranges;
  *merge = i.merge;
  *pdl = i.pdl;
  *tensor_cores = i.tensor_cores;
  *stages = i.stages;
  return BS_OK;
}

bs_status bs_split_decode_attention_workspace_size(const bs_kv_pool* pool, int32_t batch,
                                                   int32_t num_q_heads, int32_t max_blocks,
                                                   size_t* bytes) {
  BS_REQUIRE(pool, "bs_split_decode_attention_workspace_size: NULL pool");
  return workspace_impl(1, &pool, &max_blocks, batch, pool->desc.num_kv_heads,
                        pool->desc.num_kv_heads, num_q_heads, false, bytes);
}

bs_status bs_split_decode_attention(const bs_kv_pool* pool, int32_t layer, const void* q,
                                    int32_t batch, int32_t num_q_heads,
                                    const int32_t* block_tables, int32_t max_blocks,
                                    const int32_t* kv_split, int32_t n_shards, int32_t shard_id,
                                    float scale, float* o_part, float* m, float* l,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  BS_REQUIRE(pool, "bs_split_decode_attention: NULL pool");
  LaunchArgs a{};
  a.n_local = 1;
  a.pools[0] = pool;
  a.bts[0] = block_tables;
  a.max_blocks[0] = max_blocks;
  a.shard_ids[0] = shard_id;
  a.pool_head_lo = 0;
  a.model_head_lo = 0;
  a.n_kv_heads = pool->desc.num_kv_heads;
  a.num_kv_heads_total = pool->desc.num_kv_heads;
  a.layer = layer;
  a.batch = batch;
  a.num_q_heads = num_q_heads;
  a.n_shards = n_shards;
  a.q = q;
  a.kv_split = kv_split;
  a.scale = scale;
  a.merged = false;
  a.o = o_part;
  a.m = m;
  a.l = l;
  a.workspace = workspace;
  a.workspace_bytes = workspace_bytes;
  a.stream = stream;
  return run_attention(a);
}

bs_status bs_split_decode_attention_heads_workspace_size(const bs_kv_pool* pool, int32_t batch,
                                                         int32_t n_kv_heads,
                                                         int32_t num_kv_heads_total,
                                                         int32_t num_q_heads, int32_t max_blocks,
                                                         size_t* bytes) {
  return workspace_impl(1, &pool, &max_blocks, batch, n_kv_heads, num_kv_heads_total, num_q_heads,
                        false, bytes);
}

bs_status bs_split_decode_attention_heads(const bs_kv_pool* pool, int32_t layer,
                                          int32_t pool_head_lo, int32_t model_head_lo,
                                          int32_t n_kv_heads, int32_t num_kv_heads_total,
                                          const void* q, int32_t batch, int32_t num_q_heads,
                                          const int32_t* block_tables, int32_t max_blocks,
                                          const int32_t* kv_split, int32_t n_shards,
                                          int32_t shard_id, float scale, float* o_part, float* m,
                                          float* l, void* workspace, size_t workspace_bytes,
                                          void* stream) {
  LaunchArgs a{};
  a.n_local = 1;
  a.pools[0] = pool;
  a.bts[0] = block_tables;
  a.max_blocks[0] = max_blocks;
  a.shard_ids[0] = shard_id;
  a.pool_head_lo = pool_head_lo;
  a.model_head_lo = model_head_lo;
  a.n_kv_heads = n_kv_heads;
  a.num_kv_heads_total = num_kv_heads_total;
  a.layer = layer;
  a.batch = batch;
  a.num_q_heads = num_q_heads;
  a.n_shards = n_shards;
  a.q = q;
  a.kv_split = kv_split;
  a.scale = scale;
  a.merged = false;
  a.o = o_part;
  a.m = m;
  a.l = l;
  a.workspace = workspace;
  a.workspace_bytes = workspace_bytes;
  a.stream = stream;
  return run_attention(a);
}

bs_status bs_split_decode_attention_local_workspace_size(int32_t n_local,
                                                         const bs_kv_pool* const* pools,
                                                         const int32_t* max_blocks, int32_t batch,
                                                         int32_t num_q_heads, size_t* bytes) {
  BS_REQUIRE(pools && pools[0], "bs_split_decode_attention_local_workspace_size: NULL pool");
  const int hkv = pools[0]->desc.num_kv_heads;
  return workspace_impl(n_local, pools, max_blocks, batch, hkv, hkv, num_q_heads, true, bytes);
}

bs_status bs_split_decode_attention_local(int32_t n_local, const bs_kv_pool* const* pools,
                                          int32_t layer, const void* q, int32_t batch,
                                          int32_t num_q_heads, const int32_t* const* block_tables,
                                          const int32_t* max_blocks, const int32_t* shard_ids,
                                          const int32_t* kv_split, int32_t n_shards, float scale,
                                          void* out, float* lse, void* workspace,
                                          size_t workspace_bytes, void* stream) {
  return bs_split_decode_attention_local_ex(n_local, pools, layer, q, batch, num_q_heads,
                                            block_tables, max_blocks, shard_ids, kv_split,
                                            n_shards, scale, out, lse, workspace, workspace_bytes,
                                            0u, stream);
}

bs_status bs_split_decode_attention_local_ex(int32_t n_local, const bs_kv_pool* const* pools,
                                             int32_t layer, const void* q, int32_t batch,
                                             int32_t num_q_heads,
                                             const int32_t* const* block_tables,
                                             const int32_t* max_blocks, const int32_t* shard_ids,
                                             const int32_t* kv_split, int32_t n_shards, float scale,
                                             void* out, float* lse, void* workspace,
                                             size_t workspace_bytes, uint32_t flags, void* stream) {
  BS_REQUIRE((flags & ~(BS_ATTN_PDL | BS_ATTN_NO_CLUSTER)) == 0,
             "bs_split_decode_attention_local: unknown flags 0x%x", flags);
  BS_REQUIRE(pools && block_tables && max_blocks && shard_ids,
             "bs_split_decode_attention_local: NULL array");
  BS_REQUIRE(n_local >= 1 && n_local <= bs::kMaxLocal, "bs_split_decode_attention_local: %d shards",
             n_local);
  BS_REQUIRE(pools[0], "bs_split_decode_attention_local: NULL pool");
  LaunchArgs a{};
  a.n_local = n_local;
  for (int j = 0; j < n_local; ++j) {
    a.pools[j] = pools[j];
    a.bts[j] = block_tables[j];
    a.max_blocks[j] = max_blocks[j];
    a.shard_ids[j] = shard_ids[j];
    BS_REQUIRE(pools[j] && pools[j]->desc.num_kv_heads == pools[0]->desc.num_kv_heads,
               "bs_split_decode_attention_local: shards must share num_kv_heads");
  }
  a.pool_head_lo = 0;
  a.model_head_lo = 0;
  a.n_kv_heads = pools[0]->desc.num_kv_heads;
  a.num_kv_heads_total = a.n_kv_heads;
  a.layer = layer;
  a.batch = batch;
  a.num_q_heads = num_q_heads;
  a.n_shards = n_shards;
  a.q = q;
  a.kv_split = kv_split;
  a.scale = scale;
  a.merged = true;
  a.out = out;
  a.lse = lse;
  a.workspace = workspace;
  a.workspace_bytes = workspace_bytes;
  a.stream = stream;
  a.flags = flags;
  return run_attention(a);
}

bs_status bs_attention_problem_workspace_size(int32_t batch, int32_t num_q_heads,
                                              int32_t num_kv_heads, int32_t head_dim,
                                              int32_t n_shards, const int32_t* max_blocks,
                                              size_t* bytes) {
  BS_REQUIRE(bytes && max_blocks, "bs_attention_problem_workspace_size: NULL argument");
  BS_REQUIRE(batch >= 0 && num_kv_heads >= 1 && num_q_heads >= num_kv_heads &&
                 num_q_heads % num_kv_heads == 0,
             "bs_attention_problem_workspace_size: bad batch / heads");
  BS_REQUIRE(n_shards >= 1 && n_shards <= bs::kMaxProbShards,
             "bs_attention_problem_workspace_size: %d shards (1..%d)", n_shards, bs::kMaxProbShards);
  for (int j = 0; j < n_shards; ++j)
    BS_REQUIRE(max_blocks[j] >= 1, "bs_attention_problem_workspace_size: max_blocks < 1");
  const int G = num_q_heads / num_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8)
    return bs::set_error(BS_ERR_UNSUPPORTED, "query group G=%d not in {1,2,4,8}", G);
  if (head_dim != 64 && head_dim != 128)
    return bs::set_error(BS_ERR_UNSUPPORTED, "head_dim %d not in {64,128}", head_dim);
  bs::Plan pl;
  bs_status st = bs::make_plan(batch, G, num_q_heads, num_kv_heads, head_dim, n_shards, max_blocks,
                               true, &pl, /*rank_invariant=*/true);
  if (st != BS_OK) return st;
  *bytes = pl.ws_bytes;
  return BS_OK;
}

bs_status bs_split_decode_attention_tasks(int32_t n_problems, const bs_attn_problem* problems,
                                          int32_t n_tasks, const bs_attn_task* tasks,
                                          int32_t layer, int32_t batch, int32_t num_q_heads,
                                          float scale, void* stream) {
  BS_REQUIRE(problems && tasks, "bs_split_decode_attention_tasks: NULL array");
  BS_REQUIRE(n_problems >= 1 && n_problems <= bs::kMaxLocal && n_tasks >= 1 && n_tasks <= bs::kMaxLocal,
             "bs_split_decode_attention_tasks: %d problems / %d tasks (1..%d each)", n_problems,
             n_tasks, bs::kMaxLocal);
  BS_REQUIRE(tasks[0].pool, "bs_split_decode_attention_tasks: NULL pool");
  const bs_kv_pool_desc& d0 = tasks[0].pool->desc;
  const int hkv = d0.num_kv_heads, d = d0.head_dim;
  for (int t = 0; t < n_tasks; ++t) {
    const bs_attn_task& k = tasks[t];
    BS_REQUIRE(k.pool && k.block_tables, "bs_split_decode_attention_tasks: task %d: NULL pool / table", t);
    BS_REQUIRE(!k.pool->host, "bs_split_decode_attention_tasks: host-tier pools are fetched first");
    BS_REQUIRE(k.pool->desc.num_kv_heads == hkv && k.pool->desc.head_dim == d &&
                   k.pool->desc.num_layers == d0.num_layers,
               "bs_split_decode_attention_tasks: pools must share geometry");
    BS_REQUIRE(k.problem >= 0 && k.problem < n_problems, "bs_split_decode_attention_tasks: task %d: problem %d",
               t, k.problem);
    BS_REQUIRE(k.shard_id >= 0 && k.shard_id < problems[k.problem].n_shards,
               "bs_split_decode_attention_tasks: task %d: shard %d", t, k.shard_id);
  }
  BS_REQUIRE(layer >= 0 && layer < d0.num_layers, "bs_split_decode_attention_tasks: layer %d", layer);
  BS_REQUIRE(batch >= 0, "bs_split_decode_attention_tasks: batch < 0");
  BS_REQUIRE(num_q_heads >= hkv && num_q_heads % hkv == 0,
             "bs_split_decode_attention_tasks: num_q_heads %d not a multiple of Hkv %d", num_q_heads, hkv);
  BS_REQUIRE(scale > 0.f && scale == scale, "bs_split_decode_attention_tasks: bad scale");
  const int G = num_q_heads / hkv;
  if (G != 1 && G != 2 && G != 4 && G != 8)
    return bs::set_error(BS_ERR_UNSUPPORTED, "query group G=%d not in {1,2,4,8}", G);
  bs::Plan plans[bs::kMaxLocal];
  bs::AttnParams p{};
  for (int i = 0; i < n_problems; ++i) {
    const bs_attn_problem& pr = problems[i];
    BS_REQUIRE(pr.q && pr.kv_split && pr.max_blocks && pr.out,
               "bs_split_decode_attention_tasks: problem %d: NULL q / kv_split / max_blocks / out", i);
    BS_REQUIRE(((uintptr_t)pr.q & 15) == 0 && ((uintptr_t)pr.out & 15) == 0,
               "bs_split_decode_attention_tasks: q / out must be 16-B aligned");
    BS_REQUIRE(pr.n_shards >= 1 && pr.n_shards <= bs::kMaxProbShards,
               "bs_split_decode_attention_tasks: problem %d: %d shards", i, pr.n_shards);
    for (int j = 0; j < pr.n_shards; ++j)
      BS_REQUIRE(pr.max_blocks[j] >= 1, "bs_split_decode_attention_tasks: max_blocks < 1");
    bs_status st = bs::make_plan(batch, G, num_q_heads, hkv, d, pr.n_shards, pr.max_blocks, true, &plans[i],
                                 /*rank_invariant=*/true);
    if (st != BS_OK) return st;
    BS_REQUIRE(plans[i].ws_bytes == 0 || (pr.workspace && pr.workspace_bytes >= plans[i].ws_bytes &&
                                          ((uintptr_t)pr.workspace & 15) == 0),
               "bs_split_decode_attention_tasks: problem %d: workspace needs %zu bytes (got %zu)", i,
               plans[i].ws_bytes, pr.workspace_bytes);
    bs::ProbDesc& P = p.pb[i];
    P.q = static_cast<const __nv_bfloat16*>(pr.q);
    P.kv_split = pr.kv_split;
    P.n_shards = pr.n_shards;
    P.nsplit = plans[i].nsplit;
    P.merged = 1;
    P.sys = pr.cross_device ? 1 : 0;
    P.out = static_cast<__nv_bfloat16*>(pr.out);
    P.lse = pr.lse;
    P.done = pr.done;
    if (plans[i].ws_bytes) {
      uint8_t* ws = static_cast<uint8_t*>(pr.workspace);
      P.ws_o = reinterpret_cast<float*>(ws);
      P.ws_ml = reinterpret_cast<float*>(ws + plans[i].off_ml);
      P.ws_cnt = reinterpret_cast<int32_t*>(ws + plans[i].off_cnt);
    }
  }
  if (batch == 0) return BS_OK;
  bs::TMaps tm;
  bool have_maps = bs::variant_for(d, G).mma;
  int off = 0;
  for (int t = 0; t < n_tasks; ++t) {
    const bs_attn_task& k = tasks[t];
    const bs_kv_pool* pool = k.pool;
    const bs::Plan& pl = plans[k.problem];
    bs::ShardDesc& sd = p.sh[t];
    sd.kv = pool->base + (size_t)layer * pool->layer_bytes;
    sd.chunk_bytes = (int64_t)pool->chunk_bytes;
    sd.v_off = (int64_t)pool->desc.num_kv_heads * pool->page_bytes;
    sd.bt = k.block_tables;
    sd.max_blocks = problems[k.problem].max_blocks[k.shard_id];
    sd.shard_id = k.shard_id;
    sd.bps = pl.bps;
    sd.split_off = off;
    off += pl.nsplit_s[k.shard_id];
    sd.pool_hkv = hkv;
    sd.pool_head_lo = 0;
    sd.layer_row0 = (int32_t)((int64_t)layer * pool->desc.num_blocks * 2 * hkv * 16);
    sd.prob = k.problem;
    sd.range_base = pl.split_off[k.shard_id];
    sd.order = k.order;
    if (have_maps) {
      const CUtensorMap* m = pool_tensor_map(pool);
      if (m) tm.m[t] = *m;
      else have_maps = false;
    }
  }
  p.n_local = n_tasks;
  p.scale_log2 = scale * bs::kLog2e;
  p.hq = num_q_heads;
  p.hkv = hkv;
  p.model_head_lo = 0;
  p.grid_x = off;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int t = 0; t < n_tasks; ++t) {
    const bs_attn_problem& pr = problems[tasks[t].problem];
    BS_DEBUG_CHECK(bs::debug_check_table(pr.kv_split, pr.n_shards, tasks[t].shard_id, batch,
                                         tasks[t].block_tables, pr.max_blocks[tasks[t].shard_id],
                                         tasks[t].pool->desc.num_blocks, s,
                                         "attention task block table / kv_split"));
  }
  const bs::TMaps* tmp = have_maps ? &tm : nullptr;
  if (d == 128) return bs::launch_attn_d<128>(p, tmp, G, batch, s);
  return bs::launch_attn_d<64>(p, tmp, G, batch, s);
}

bs_status bs_attention_ragged_plan(int32_t batch, int32_t n_shards, const int32_t* kv_split_host,
                                   int32_t n_local, const int32_t* shard_ids, int32_t num_q_heads,
                                   int32_t num_kv_heads, int32_t head_dim,
                                   int32_t max_blocks_per_range, int32_t* work, int32_t capacity,
                                   int32_t* n_work, int32_t* max_parts, size_t* workspace_bytes) {
  return bs_attention_ragged_plan_ex(batch, n_shards, kv_split_host, n_local, shard_ids, num_q_heads,
                                     num_kv_heads, head_dim, max_blocks_per_range, 0u, work, capacity,
                                     n_work, max_parts, workspace_bytes);
}

bs_status bs_attention_ragged_plan_ex(int32_t batch, int32_t n_shards, const int32_t* kv_split_host,
                                      int32_t n_local, const int32_t* shard_ids, int32_t num_q_heads,
                                      int32_t num_kv_heads, int32_t head_dim,
                                      int32_t max_blocks_per_range, uint32_t flags, int32_t* work,
                                      int32_t capacity, int32_t* n_work, int32_t* max_parts,
                                      size_t* workspace_bytes) {
  BS_REQUIRE((flags & ~BS_PLAN_PACK_SHORT) == 0, "bs_attention_ragged_plan: unknown flags 0x%x", flags);
  BS_REQUIRE(kv_split_host && shard_ids && n_work && max_parts && workspace_bytes,
             "bs_attention_ragged_plan: NULL argument");
  BS_REQUIRE(batch >= 1 && n_shards >= 1 && n_local >= 1 && n_local <= bs::kMaxLocal,
             "bs_attention_ragged_plan: batch %d / %d shards / %d local", batch, n_shards, n_local);
  BS_REQUIRE(num_kv_heads >= 1 && num_q_heads >= num_kv_heads && num_q_heads % num_kv_heads == 0,
             "bs_attention_ragged_plan: bad heads");
  BS_REQUIRE(head_dim == 64 || head_dim == 128, "bs_attention_ragged_plan: head_dim %d", head_dim);
  BS_REQUIRE(max_blocks_per_range >= 0 && max_blocks_per_range <= bs::kBtMax,
             "bs_attention_ragged_plan: max_blocks_per_range %d (0..%d)", max_blocks_per_range,
             bs::kBtMax);
  for (int t = 0; t < n_local; ++t)
    BS_REQUIRE(shard_ids[t] >= 0 && shard_ids[t] < n_shards, "bs_attention_ragged_plan: shard %d",
               shard_ids[t]);
  const int G = num_q_heads / num_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8)
    return bs::set_error(BS_ERR_UNSUPPORTED, "query group G=%d not in {1,2,4,8}", G);
  std::vector<int32_t> nblk((size_t)batch * n_local);
  for (int b = 0; b < batch; ++b)
    for (int t = 0; t < n_local; ++t) {
      const int32_t* ks = kv_split_host + (int64_t)b * (n_shards + 1) + shard_ids[t];
      const int32_t len = std::max(ks[1] - ks[0], 0);
      nblk[(size_t)b * n_local + t] = (len + 15) / 16;
    }
  // range length (automatic): the uniform planner's choice for the same shard widths
  // (its wave model), so balanced batches get the uniform grid's cut; the ragged list then
  // drops the empty (request, shard) CTAs and gives short requests a single range
  int bps = max_blocks_per_range;
  if (bps == 0) {
    int mb[bs::kMaxProbShards];
    for (int t = 0; t < n_local; ++t) {
      mb[t] = 1;
      for (int b = 0; b < batch; ++b) mb[t] = std::max(mb[t], nblk[(size_t)b * n_local + t]);
    }
    bs::Plan pl;
    bs_status st = bs::make_plan(batch, G, num_q_heads, num_kv_heads, head_dim, n_local, mb, true, &pl);
    if (st != BS_OK) return st;
    bps = std::min(bs::kBtMax, std::max(16, pl.bps));
  }
  int32_t most = 1;
  std::vector<int4> items;
  std::vector<int32_t> keys;  // dispatch-order key: the CTA's longest per-warp block run x 4
  auto emit = [&](int b, int t, int slot, int blo, int nb, int parts) {
    items.push_back(make_int4(b, (t << 16) | slot, blo, (nb << 8) | parts));
    keys.push_back(nb);
  };
  // BS_PLAN_PACK_SHORT: requests whose (only) shard has <= kPackMaxBlocks blocks go into
  // packed items -- up to 4 requests per CTA, one warp each, no cross-warp combine (the
  // tensor-core kernel; a one-CTA-per-(request, kv-head) item with 1-8 blocks is prologue-
  // and epilogue-bound)
  const bool pack = (flags & BS_PLAN_PACK_SHORT) && n_local == 1 && bs::variant_for(head_dim, G).mma;
  std::vector<int32_t> short_reqs;
  for (int b = 0; b < batch; ++b) {
    if (pack && nblk[(size_t)b] <= bs::kPackMaxBlocks) {
      short_reqs.push_back(b);
      continue;
    }
    int pb = bps, parts = 0;
    for (;;) {  // a request's ranges must fit kMaxSplit slots: widen its ranges if not
      parts = 0;
      for (int t = 0; t < n_local; ++t) parts += (nblk[(size_t)b * n_local + t] + pb - 1) / pb;
      if (parts <= bs::kMaxSplit) break;
      pb = std::min(bs::kBtMax, pb * 2);
      if (pb == bs::kBtMax) {
        parts = 0;
        for (int t = 0; t < n_local; ++t) parts += (nblk[(size_t)b * n_local + t] + pb - 1) / pb;
        if (parts > bs::kMaxSplit)
          return bs::set_error(BS_ERR_UNSUPPORTED, "request %d: %d ranges > %d", b, parts, bs::kMaxSplit);
        break;
      }
    }
    if (parts == 0) {  // empty everywhere: one item writes the empty result
      emit(b, 0, 0, 0, 0, 1);
      continue;
    }
    most = std::max(most, parts);
    int slot = 0;
    for (int t = 0; t < n_local; ++t) {  // shard-major, then range: the fixed merge order
      const int nb = nblk[(size_t)b * n_local + t];
      if (nb == 0) continue;
      const int nr = (nb + pb - 1) / pb, base = nb / nr, rem = nb % nr;
      int blo = 0;
      for (int r = 0; r < nr; ++r) {
        const int len = base + (r < rem ? 1 : 0);
        emit(b, t, slot++, blo, len, parts);
        blo += len;
      }
    }
  }
  // Launch order = CTA dispatch order.  Longest ranges first (LPT): the hardware hands out
  // CTAs in grid order, so the long ranges of mixed-length batches start in the first wave
  // and the short ones fill the tail.  The merge order is the slot order, not the arrival
  // order, so the results do not depend on it.  BS_RAGGED_ORDER=0 keeps request order.
  for (size_t i = 0; i < short_reqs.size(); i += bs::kWarps) {
    int32_t r[bs::kWarps];
    int32_t longest = 0;
    for (int k = 0; k < bs::kWarps; ++k) {
      r[k] = i + k < short_reqs.size() ? short_reqs[i + k] : -1;
      if (r[k] >= 0) longest = std::max(longest, nblk[(size_t)r[k]]);
    }
    items.push_back(make_int4(r[0], r[1], r[2], (int32_t)((uint32_t)r[3] << 8)));  // parts 0
    keys.push_back(longest * bs::kWarps);  // one warp streams all of its request's blocks
  }
  const char* oe = getenv("BS_RAGGED_ORDER");
  if (!(oe && atoi(oe) == 0)) {
    std::vector<size_t> idx(items.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](size_t x, size_t y) { return keys[x] > keys[y]; });
    std::vector<int4> sorted(items.size());
    for (size_t i = 0; i < idx.size(); ++i) sorted[i] = items[idx[i]];
    items.swap(sorted);
  }
  const int32_t count = (int32_t)items.size();
  if (work)
    for (int32_t i = 0; i < std::min(count, capacity); ++i) {
      int32_t* w = work + 4 * (size_t)i;
      w[0] = items[i].x;
      w[1] = items[i].y;
      w[2] = items[i].z;
      w[3] = items[i].w;
    }
  *n_work = count;
  *max_parts = most;
  *workspace_bytes = most > 1 ? (size_t)batch * num_q_heads * most * (head_dim + 2) * 4 +
                                    (size_t)batch * num_kv_heads * 4
                              : 0;
  if (work && count > capacity)
    return bs::set_error(BS_ERR_INVALID_ARG, "bs_attention_ragged_plan: %d items > capacity %d", count,
                         capacity);
  return BS_OK;
}

bs_status bs_split_decode_attention_local_ragged(
    int32_t n_local, const bs_kv_pool* const* pools, int32_t layer, const void* q, int32_t batch,
    int32_t num_q_heads, const int32_t* const* block_tables, const int32_t* max_blocks,
    const int32_t* shard_ids, const int32_t* kv_split, int32_t n_shards, float scale,
    const int32_t* work, int32_t n_work, int32_t max_parts, void* out, float* lse, void* workspace,
    size_t workspace_bytes, void* stream) {
  return bs_split_decode_attention_local_ragged_ex(n_local, pools, layer, q, batch, num_q_heads,
                                                   block_tables, max_blocks, shard_ids, kv_split,
                                                   n_shards, scale, work, n_work, max_parts, out,
                                                   lse, workspace, workspace_bytes, 0u, stream);
}

bs_status bs_split_decode_attention_local_ragged_ex(
    int32_t n_local, const bs_kv_pool* const* pools, int32_t layer, const void* q, int32_t batch,
    int32_t num_q_heads, const int32_t* const* block_tables, const int32_t* max_blocks,
    const int32_t* shard_ids, const int32_t* kv_split, int32_t n_shards, float scale,
    const int32_t* work, int32_t n_work, int32_t max_parts, void* out, float* lse, void* workspace,
    size_t workspace_bytes, uint32_t flags, void* stream) {
  BS_REQUIRE((flags & ~(BS_ATTN_PDL | BS_ATTN_NO_CLUSTER)) == 0,
             "bs_split_decode_attention_local_ragged: unknown flags 0x%x", flags);
  BS_REQUIRE(pools && block_tables && max_blocks && shard_ids && work,
             "bs_split_decode_attention_local_ragged: NULL array");
  BS_REQUIRE(n_local >= 1 && n_local <= bs::kMaxLocal, "bs_split_decode_attention_local_ragged: %d shards",
             n_local);
  BS_REQUIRE(pools[0], "bs_split_decode_attention_local_ragged: NULL pool");
  LaunchArgs a{};
  a.n_local = n_local;
  for (int j = 0; j < n_local; ++j) {
    a.pools[j] = pools[j];
    a.bts[j] = block_tables[j];
    a.max_blocks[j] = max_blocks[j];
    a.shard_ids[j] = shard_ids[j];
    BS_REQUIRE(pools[j] && pools[j]->desc.num_kv_heads == pools[0]->desc.num_kv_heads,
               "bs_split_decode_attention_local_ragged: shards must share num_kv_heads");
  }
  a.n_kv_heads = a.num_kv_heads_total = pools[0]->desc.num_kv_heads;
  a.layer = layer;
  a.batch = batch;
  a.num_q_heads = num_q_heads;
  a.n_shards = n_shards;
  a.q = q;
  a.kv_split = kv_split;
  a.scale = scale;
  a.merged = true;
  a.out = out;
  a.lse = lse;
  a.workspace = workspace;
  a.workspace_bytes = workspace_bytes;
  a.stream = stream;
  a.work = work;
  a.n_work = n_work;
  a.max_parts = max_parts;
  a.flags = flags;
  return run_attention(a);
}

}  // extern "C"
