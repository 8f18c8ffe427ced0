// H2: per-layer KV block migration -- gather -> send -> scatter fused into one copy
// kernel (attention-level migration, eq. 11; the copy is
// "without semantic change", eq. 5).
//
// The unit of work is one page (one (layer, block, K|V, kv_head) = 16*d*2 bytes, 4 KiB
// at d=128): pages are contiguous in the pool layout, so every copy is a straight
// 16-byte-aligned memcpy.  Two kernels:
//   * copy_pages_vec16: warp per page, 16-byte LDG (L1::no_allocate) / STG, all loads of
//     a page issued before its stores (8 x 16 B in flight per lane at d=128).  When the
//     destination (or source) base is a peer-mapped pointer the stores (loads) travel over
//     NVLink -- the P2P "push" (or "pull") transport with no staging.
//   * copy_pages_bulk: one elected thread per CTA streams pages through a shared-memory
//     ring with TMA bulk copies (cp.async.bulk global->shared with an mbarrier, then
//     cp.async.bulk shared->global in bulk groups); no registers touch the payload.
#include <cuda_runtime.h>

#include <atomic>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "append.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace bs {
namespace {

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Cache-policy experiment (BS_COPY_HINT): 0 default stores; 1 streaming
// stores (st.global.cs: evict-first); 2 loads and stores with an L2 evict_first policy.
// The hand-off's 100 MB of writes per layer otherwise sit dirty in L2 and are written back
// while the next layer's attention streams its reads (read/write interference, §7).
__device__ __forceinline__ int4 ld_stream_hint(const int4* p, int hint, uint64_t pol) {
  if (hint == 2) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
  }
  return ld_stream(p);
}

__device__ __forceinline__ void st_stream_hint(int4* p, const int4& v, int hint, uint64_t pol) {
  if (hint == 1) {
    asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
  } else if (hint == 2) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.s32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
  } else {
    st_stream(p, v);
  }
}

// The page loop of the vec16 copy for CTA `cta` of `nctas` (shared by the plain copy and
// the fused copy + append launch).
template <int PAGE_BYTES, int U>
__device__ __forceinline__ void copy_pages_body(const uint8_t* __restrict__ src_base,
                                                const int32_t* __restrict__ src_ids,
                                                uint8_t* __restrict__ dst_base,
                                                const int32_t* __restrict__ dst_ids, int32_t n,
                                                int32_t pages_per_chunk, int64_t chunk_bytes,
                                                int32_t n_layers, int64_t src_layer_stride,
                                                int64_t dst_layer_stride, int cta, int nctas,
                                                int hint = 0) {
  constexpr int V = PAGE_BYTES / (16 * 32);  // int4 per lane per page
  uint64_t pol = 0;
  if (hint == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int lane = threadIdx.x & 31;
  const int wpc = blockDim.x >> 5;
  const int64_t per_layer = (int64_t)n * pages_per_chunk;
  const int64_t total = per_layer * n_layers;
  // a warp moves U pages per iteration: U * V 16-byte loads in flight per lane
  for (int64_t p0 = ((int64_t)cta * wpc + (threadIdx.x >> 5)) * U; p0 < total;
       p0 += (int64_t)nctas * wpc * U) {
    int4 r[U][V];
    int4* dst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = p0 + u;
      dst[u] = nullptr;
      if (p < total) {
        const int32_t ly = (int32_t)(p / per_layer);
        const int64_t q = p - (int64_t)ly * per_layer;
        const int32_t i = (int32_t)(q / pages_per_chunk);
        const int32_t j = (int32_t)(q - (int64_t)i * pages_per_chunk);
        const int64_t si = src_ids ? __ldg(src_ids + i) : i;
        const int64_t di = dst_ids ? __ldg(dst_ids + i) : i;
        const int4* s = reinterpret_cast<const int4*>(src_base + ly * src_layer_stride +
                                                      si * chunk_bytes + (int64_t)j * PAGE_BYTES) + lane;
        dst[u] = reinterpret_cast<int4*>(dst_base + ly * dst_layer_stride + di * chunk_bytes +
                                         (int64_t)j * PAGE_BYTES) + lane;
#pragma unroll
        for (int v = 0; v < V; ++v) r[u][v] = ld_stream_hint(s + v * 32, hint, pol);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (dst[u])
#pragma unroll
        for (int v = 0; v < V; ++v) st_stream_hint(dst[u] + v * 32, r[u][v], hint, pol);
  }
}

template <int PAGE_BYTES, int U>
__global__ void __launch_bounds__(256) copy_pages_vec16(const uint8_t* __restrict__ src_base,
                                                        const int32_t* __restrict__ src_ids,
                                                        uint8_t* __restrict__ dst_base,
                                                        const int32_t* __restrict__ dst_ids,
                                                        int32_t n, int32_t pages_per_chunk,
                                                        int64_t chunk_bytes, int32_t n_layers,
                                                        int64_t src_layer_stride,
                                                        int64_t dst_layer_stride) {
  copy_pages_body<PAGE_BYTES, U>(src_base, src_ids, dst_base, dst_ids, n, pages_per_chunk,
                                 chunk_bytes, n_layers, src_layer_stride, dst_layer_stride,
                                 blockIdx.x, gridDim.x);
}

// H2 + H7 in one launch (bs_kv_migrate_append_layer): CTAs [0, batch) write request b's
// decoded-token K/V rows into the append pool, the others run the hand-off page copy.
struct AppendArgs {
  uint8_t* layer_base;
  int64_t chunk_bytes;
  int32_t hkv, d;
  const uint4* k_new;
  const uint4* v_new;
  const int32_t* bt;
  int32_t max_blocks;
  const int32_t* pos;
  int32_t batch;
};

template <int PAGE_BYTES, int U>
__global__ void __launch_bounds__(256) migrate_append_vec16(const uint8_t* __restrict__ src_base,
                                                            const int32_t* __restrict__ src_ids,
                                                            uint8_t* __restrict__ dst_base,
                                                            const int32_t* __restrict__ dst_ids,
                                                            int32_t n, int32_t pages_per_chunk,
                                                            int64_t chunk_bytes, const AppendArgs a,
                                                            int hint) {
  if ((int)blockIdx.x < a.batch) {
    append_token_rows(a.layer_base, a.chunk_bytes, a.hkv, a.d, a.k_new, a.v_new, a.bt, a.max_blocks,
                      a.pos, blockIdx.x, threadIdx.x, blockDim.x);
    return;
  }
  copy_pages_body<PAGE_BYTES, U>(src_base, src_ids, dst_base, dst_ids, n, pages_per_chunk,
                                 chunk_bytes, 1, 0, 0, blockIdx.x - a.batch, gridDim.x - a.batch,
                                 hint);
}

// NEXT F2: head-granular pages (K and V of n_heads kv-heads of each pair), between pools
// whose kv-head counts may differ (a cold pool can keep only the migrated heads).
template <int PAGE_BYTES>
__global__ void __launch_bounds__(256) copy_head_pages_vec16(
    const uint8_t* __restrict__ src_base, const int32_t* __restrict__ src_ids, int64_t src_chunk,
    int32_t src_hkv, int32_t src_head_lo, uint8_t* __restrict__ dst_base,
    const int32_t* __restrict__ dst_ids, int64_t dst_chunk, int32_t dst_hkv, int32_t dst_head_lo,
    int32_t n, int32_t n_heads) {
  constexpr int V = PAGE_BYTES / (16 * 32);
  const int lane = threadIdx.x & 31;
  const int wpc = blockDim.x >> 5;
  const int32_t ppp = 2 * n_heads;  // pages per pair
  const int64_t total = (int64_t)n * ppp;
  for (int64_t p = (int64_t)blockIdx.x * wpc + (threadIdx.x >> 5); p < total;
       p += (int64_t)gridDim.x * wpc) {
    const int32_t i = (int32_t)(p / ppp);
    const int32_t r = (int32_t)(p - (int64_t)i * ppp);
    const int32_t kv = r / n_heads, h = r - kv * n_heads;
    const int4* s = reinterpret_cast<const int4*>(
        src_base + (int64_t)__ldg(src_ids + i) * src_chunk +
        (int64_t)(kv * src_hkv + src_head_lo + h) * PAGE_BYTES) + lane;
    int4* d = reinterpret_cast<int4*>(dst_base + (int64_t)__ldg(dst_ids + i) * dst_chunk +
                                      (int64_t)(kv * dst_hkv + dst_head_lo + h) * PAGE_BYTES) + lane;
    int4 rg[V];
#pragma unroll
    for (int v = 0; v < V; ++v) rg[v] = ld_stream(s + v * 32);
#pragma unroll
    for (int v = 0; v < V; ++v) st_stream(d + v * 32, rg[v]);
  }
}

// ---- TMA bulk ring -------------------------------------------------------------------

using ptx::bulk_g2s;
using ptx::mbar_expect_tx;
using ptx::mbar_init;
using ptx::mbar_wait;
using ptx::smem_u32;

__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

constexpr int kBulkStages = 24;  // ring slots (pages)
constexpr int kBulkAhead = 16;   // loads in flight ahead of the store front

template <int PAGE_BYTES>
__global__ void __launch_bounds__(32) copy_pages_bulk(const uint8_t* __restrict__ src_base,
                                                      const int32_t* __restrict__ src_ids,
                                                      uint8_t* __restrict__ dst_base,
                                                      const int32_t* __restrict__ dst_ids,
                                                      int32_t n, int32_t pages_per_chunk,
                                                      int64_t chunk_bytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kBulkStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kBulkStages; ++s) mbar_init(&bars[s], 1);
  ptx::fence_mbar_init();

  const int64_t total = (int64_t)n * pages_per_chunk;
  // this CTA's pages: p = blockIdx.x + k * gridDim.x, k = 0..mine-1
  const int64_t mine = total > blockIdx.x ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto src_of = [&](int64_t k) {
    const int64_t p = blockIdx.x + k * gridDim.x;
    const int32_t i = (int32_t)(p / pages_per_chunk);
    const int32_t j = (int32_t)(p - (int64_t)i * pages_per_chunk);
    const int64_t si = src_ids ? __ldg(src_ids + i) : i;
    return src_base + si * chunk_bytes + (int64_t)j * PAGE_BYTES;
  };
  auto dst_of = [&](int64_t k) {
    const int64_t p = blockIdx.x + k * gridDim.x;
    const int32_t i = (int32_t)(p / pages_per_chunk);
    const int32_t j = (int32_t)(p - (int64_t)i * pages_per_chunk);
    const int64_t di = dst_ids ? __ldg(dst_ids + i) : i;
    return dst_base + di * chunk_bytes + (int64_t)j * PAGE_BYTES;
  };
  auto issue_load = [&](int64_t k) {
    const int s = (int)(k % kBulkStages);
    mbar_expect_tx(&bars[s], PAGE_BYTES);
    bulk_g2s(smem + (size_t)s * PAGE_BYTES, src_of(k), PAGE_BYTES, &bars[s]);
  };
  for (int64_t k = 0; k < mine && k < kBulkAhead; ++k) issue_load(k);
  for (int64_t k = 0; k < mine; ++k) {
    const int s = (int)(k % kBulkStages);
    mbar_wait(&bars[s], (uint32_t)((k / kBulkStages) & 1));
    bulk_s2g(dst_of(k), smem + (size_t)s * PAGE_BYTES, PAGE_BYTES);
    bulk_commit();
    const int64_t nk = k + kBulkAhead;
    if (nk < mine) {
      // slot of nk was last read by the store of page nk - kBulkStages; at most
      // kBulkStages - kBulkAhead - 1 younger stores may still be reading smem.
      bulk_wait_read<kBulkStages - kBulkAhead - 1>();
      issue_load(nk);
    }
  }
  bulk_wait_all();
}

template <int PAGE_BYTES>
bs_status launch_copy_t(const uint8_t* src_base, const int32_t* src_ids, uint8_t* dst_base,
                        const int32_t* dst_ids, int32_t n, int32_t ppc, int64_t chunk, int method,
                        cudaStream_t stream, int max_ctas, int32_t n_layers, int64_t src_ls,
                        int64_t dst_ls) {
  const int64_t total = (int64_t)n * ppc * n_layers;
  if (method == BS_MIGRATE_BULK && n_layers != 1) method = BS_MIGRATE_VEC16;
  const int sms = sm_count(current_device());
  if (method == BS_MIGRATE_BULK) {
    const int smem = kBulkStages * PAGE_BYTES;
    // the shared-memory opt-in is a per-device function attribute: track it per device
    static std::atomic<uint64_t> configured{0};
    const int dev = current_device();
    const uint64_t bit = 1ull << (dev & 63);
    if (!(configured.load() & bit)) {
      cudaFuncSetAttribute(copy_pages_bulk<PAGE_BYTES>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      configured.fetch_or(bit);
    }
    int64_t grid = std::min<int64_t>(total, (int64_t)sms * 2);
    if (max_ctas > 0) grid = std::min<int64_t>(grid, max_ctas);
    copy_pages_bulk<PAGE_BYTES><<<(unsigned)grid, 32, smem, stream>>>(
        src_base, src_ids, dst_base, dst_ids, n, ppc, chunk);
    return check_launch("copy_pages_bulk");
  }
  const int wpc = 8;
  static const int unroll = [] {
    const char* e = getenv("BS_COPY_UNROLL");
    return e && atoi(e) == 1 ? 1 : 2;
  }();
  int64_t grid = std::min<int64_t>((total + wpc * unroll - 1) / (wpc * unroll), (int64_t)sms * 8);
  if (max_ctas > 0) grid = std::min<int64_t>(grid, max_ctas);
  if (unroll == 2)
    copy_pages_vec16<PAGE_BYTES, 2><<<(unsigned)grid, wpc * 32, 0, stream>>>(
        src_base, src_ids, dst_base, dst_ids, n, ppc, chunk, n_layers, src_ls, dst_ls);
  else
    copy_pages_vec16<PAGE_BYTES, 1><<<(unsigned)grid, wpc * 32, 0, stream>>>(
        src_base, src_ids, dst_base, dst_ids, n, ppc, chunk, n_layers, src_ls, dst_ls);
  return check_launch("copy_pages_vec16");
}

}  // namespace

bs_status launch_copy_chunks(const uint8_t* src_base, const int32_t* src_ids, uint8_t* dst_base,
                             const int32_t* dst_ids, int32_t n, size_t chunk_bytes,
                             size_t page_bytes, int method, cudaStream_t stream, int max_ctas,
                             int32_t n_layers, int64_t src_layer_stride, int64_t dst_layer_stride) {
  if (n == 0 || n_layers == 0) return BS_OK;
  const int32_t ppc = (int32_t)(chunk_bytes / page_bytes);
  if (method == BS_MIGRATE_AUTO) {
    static const int dflt = [] {  // BS_MIGRATE_AUTO_METHOD: 1 vec16 (default), 2 bulk
      const char* e = getenv("BS_MIGRATE_AUTO_METHOD");
      return e && atoi(e) == BS_MIGRATE_BULK ? BS_MIGRATE_BULK : BS_MIGRATE_VEC16;
    }();
    method = dflt;
  }
  if (page_bytes == 4096)
    return launch_copy_t<4096>(src_base, src_ids, dst_base, dst_ids, n, ppc, (int64_t)chunk_bytes,
                               method, stream, max_ctas, n_layers, src_layer_stride, dst_layer_stride);
  if (page_bytes == 2048)
    return launch_copy_t<2048>(src_base, src_ids, dst_base, dst_ids, n, ppc, (int64_t)chunk_bytes,
                               method, stream, max_ctas, n_layers, src_layer_stride, dst_layer_stride);
  return set_error(BS_ERR_UNSUPPORTED, "page size %zu", page_bytes);
}

}  // namespace bs

// CTAs for a copy that touches a host-tier pool: ~8 x 8 warps x 4 KiB in flight covers
// PCIe latency x bandwidth (~2 us x 55 GB/s); the other SMs keep the layer's compute.
static int host_copy_ctas() {
  static int v = [] {
    const char* e = getenv("BS_HOST_COPY_CTAS");
    int x = e ? atoi(e) : 8;
    return x > 0 ? x : 8;
  }();
  return v;
}
#define kHostCopyCtas host_copy_ctas()

// Optional cap on the CTAs of a device-side migration (BS_MIGRATE_MAX_CTAS, 0 = none): a
// hand-off that runs beside attention only needs ~96 MiB per layer, so a few dozen CTAs
// keep it on time while leaving the SM slots to the attention launch.
static int dev_copy_ctas() {
  static int v = [] {
    const char* e = getenv("BS_MIGRATE_MAX_CTAS");
    int x = e ? atoi(e) : 0;
    return x > 0 ? x : 0;
  }();
  return v;
}

// A push into a pool owned by another GPU (a peer-mapped view, desc.device = the owner's
// ordinal) is NVLink-bound, not HBM-bound: one 8-warp CTA per SM keeps >= 9 MB of loads
// and stores in flight -- far more than 900 GB/s x the link's round trip needs -- while a
// full grid (8 CTAs x 256 threads per SM) would hold every SM's thread slots for the
// whole, slower, transfer and starve the attention launch beside it
// (BS_REMOTE_COPY_CTAS overrides; 0 = no cap).
static int remote_copy_ctas() {
  const char* e = getenv("BS_REMOTE_COPY_CTAS");
  return e ? std::max(0, atoi(e)) : bs::sm_count(bs::current_device());
}

static bool is_remote(const bs_kv_pool* p) {
  return !p->host && p->desc.device >= 0 && p->desc.device != bs::current_device();
}

static bool same_geometry(const bs_kv_pool* a, const bs_kv_pool* b) {
  return a->desc.num_layers == b->desc.num_layers && a->desc.num_kv_heads == b->desc.num_kv_heads &&
         a->desc.head_dim == b->desc.head_dim && a->desc.block_size == b->desc.block_size &&
         a->desc.dtype == b->desc.dtype;
}

extern "C" {

bs_status bs_kv_migrate_layer_ex(const bs_kv_pool* src, bs_kv_pool* dst, int32_t layer,
                                 const int32_t* src_ids, const int32_t* dst_ids, int32_t n,
                                 int32_t method, void* stream) {
  BS_REQUIRE(src && dst, "bs_kv_migrate_layer: NULL pool");
  BS_REQUIRE(same_geometry(src, dst), "bs_kv_migrate_layer: src/dst geometry differs");
  BS_REQUIRE(layer >= 0 && layer < src->desc.num_layers, "bs_kv_migrate_layer: layer %d out of [0,%d)",
             layer, src->desc.num_layers);
  BS_REQUIRE(n >= 0, "bs_kv_migrate_layer: n < 0");
  BS_REQUIRE(n == 0 || (src_ids && dst_ids), "bs_kv_migrate_layer: NULL ids");
  BS_REQUIRE(method >= BS_MIGRATE_AUTO && method <= BS_MIGRATE_BULK,
             "bs_kv_migrate_layer: bad method %d", method);
  // a host-tier pool is behind PCIe / C2C: a few CTAs keep it saturated, the rest of the
  // SMs stay with the layer's compute (three-stage pipeline, Fig. 6)
  int max_ctas = (src->host || dst->host) ? kHostCopyCtas : dev_copy_ctas();
  if (max_ctas == 0 && (is_remote(src) || is_remote(dst))) max_ctas = remote_copy_ctas();
  BS_DEBUG_CHECK(bs::debug_check_ids(src_ids, n, src->desc.num_blocks, static_cast<cudaStream_t>(stream),
                                     "bs_kv_migrate_layer src_ids"));
  BS_DEBUG_CHECK(bs::debug_check_ids(dst_ids, n, dst->desc.num_blocks, static_cast<cudaStream_t>(stream),
                                     "bs_kv_migrate_layer dst_ids"));
  return bs::launch_copy_chunks(src->base + (size_t)layer * src->layer_bytes, src_ids,
                                dst->base + (size_t)layer * dst->layer_bytes, dst_ids, n,
                                src->chunk_bytes, src->page_bytes, method,
                                static_cast<cudaStream_t>(stream), max_ctas);
}

bs_status bs_kv_migrate_append_layer(const bs_kv_pool* src, bs_kv_pool* dst, int32_t layer,
                                     const int32_t* src_ids, const int32_t* dst_ids, int32_t n,
                                     bs_kv_pool* app_pool, const void* k_new, const void* v_new,
                                     int32_t batch, const int32_t* block_tables,
                                     int32_t max_blocks, const int32_t* pos, void* stream) {
  BS_REQUIRE(src && dst && app_pool, "bs_kv_migrate_append_layer: NULL pool");
  BS_REQUIRE(batch >= 0 && n >= 0, "bs_kv_migrate_append_layer: negative count");
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  // host-tier / remote pools, an empty side or an unusual page size: the two launches
  const bool fuse = batch > 0 && n > 0 && !src->host && !dst->host && !app_pool->host &&
                    !is_remote(src) && !is_remote(dst) && !is_remote(app_pool) &&
                    same_geometry(src, dst) && (src->page_bytes == 4096 || src->page_bytes == 2048);
  if (!fuse) {
    bs_status st = bs_kv_migrate_layer(src, dst, layer, src_ids, dst_ids, n, stream);
    if (st != BS_OK) return st;
    return bs_kv_append_token(app_pool, layer, k_new, v_new, batch, block_tables, max_blocks, pos,
                              stream);
  }
  BS_REQUIRE(layer >= 0 && layer < src->desc.num_layers && layer < app_pool->desc.num_layers,
             "bs_kv_migrate_append_layer: layer %d out of range", layer);
  BS_REQUIRE(src_ids && dst_ids && k_new && v_new && block_tables && pos,
             "bs_kv_migrate_append_layer: NULL argument");
  BS_REQUIRE(max_blocks >= 1, "bs_kv_migrate_append_layer: max_blocks < 1");
  BS_REQUIRE(((uintptr_t)k_new & 15) == 0 && ((uintptr_t)v_new & 15) == 0,
             "bs_kv_migrate_append_layer: k_new / v_new must be 16-B aligned");
  BS_DEBUG_CHECK(bs::debug_check_ids(src_ids, n, src->desc.num_blocks, s, "bs_kv_migrate_append_layer src_ids"));
  BS_DEBUG_CHECK(bs::debug_check_ids(dst_ids, n, dst->desc.num_blocks, s, "bs_kv_migrate_append_layer dst_ids"));
  BS_DEBUG_CHECK(bs::debug_check_append(pos, batch, block_tables, max_blocks, app_pool->desc.num_blocks, s,
                                        "bs_kv_migrate_append_layer positions / block table"));
  bs::AppendArgs a;
  a.layer_base = app_pool->base + (size_t)layer * app_pool->layer_bytes;
  a.chunk_bytes = (int64_t)app_pool->chunk_bytes;
  a.hkv = app_pool->desc.num_kv_heads;
  a.d = app_pool->desc.head_dim;
  a.k_new = static_cast<const uint4*>(k_new);
  a.v_new = static_cast<const uint4*>(v_new);
  a.bt = block_tables;
  a.max_blocks = max_blocks;
  a.pos = pos;
  a.batch = batch;
  const int32_t ppc = (int32_t)(src->chunk_bytes / src->page_bytes);
  const int64_t total = (int64_t)n * ppc;
  const int sms = bs::sm_count(bs::current_device());
  int64_t grid = std::min<int64_t>((total + 8 * 2 - 1) / (8 * 2), (int64_t)sms * 8);
  const int cap = dev_copy_ctas();
  if (cap > 0) grid = std::min<int64_t>(grid, cap);
  const uint8_t* sb = src->base + (size_t)layer * src->layer_bytes;
  uint8_t* db = dst->base + (size_t)layer * dst->layer_bytes;
  static const int hint = [] {
    const char* e = getenv("BS_COPY_HINT");
    return e ? atoi(e) : 0;
  }();
  if (src->page_bytes == 4096)
    bs::migrate_append_vec16<4096, 2><<<(unsigned)(grid + batch), 256, 0, s>>>(
        sb, src_ids, db, dst_ids, n, ppc, (int64_t)src->chunk_bytes, a, hint);
  else
    bs::migrate_append_vec16<2048, 2><<<(unsigned)(grid + batch), 256, 0, s>>>(
        sb, src_ids, db, dst_ids, n, ppc, (int64_t)src->chunk_bytes, a, hint);
  return bs::check_launch("migrate_append_vec16");
}

bs_status bs_kv_migrate_layers(const bs_kv_pool* src, bs_kv_pool* dst, int32_t layer_lo,
                               int32_t n_layers, const int32_t* src_ids, const int32_t* dst_ids,
                               int32_t n, void* stream) {
  BS_REQUIRE(src && dst, "bs_kv_migrate_layers: NULL pool");
  BS_REQUIRE(same_geometry(src, dst), "bs_kv_migrate_layers: src/dst geometry differs");
  BS_REQUIRE(n_layers >= 0 && layer_lo >= 0 && layer_lo + n_layers <= src->desc.num_layers,
             "bs_kv_migrate_layers: layers [%d,+%d) out of range", layer_lo, n_layers);
  BS_REQUIRE(n >= 0, "bs_kv_migrate_layers: n < 0");
  BS_REQUIRE(n == 0 || (src_ids && dst_ids), "bs_kv_migrate_layers: NULL ids");
  const int max_ctas = (src->host || dst->host) ? kHostCopyCtas : 0;
  BS_DEBUG_CHECK(bs::debug_check_ids(src_ids, n, src->desc.num_blocks, static_cast<cudaStream_t>(stream),
                                     "bs_kv_migrate_layers src_ids"));
  BS_DEBUG_CHECK(bs::debug_check_ids(dst_ids, n, dst->desc.num_blocks, static_cast<cudaStream_t>(stream),
                                     "bs_kv_migrate_layers dst_ids"));
  return bs::launch_copy_chunks(src->base + (size_t)layer_lo * src->layer_bytes, src_ids,
                                dst->base + (size_t)layer_lo * dst->layer_bytes, dst_ids, n,
                                src->chunk_bytes, src->page_bytes, BS_MIGRATE_VEC16,
                                static_cast<cudaStream_t>(stream), max_ctas, n_layers,
                                (int64_t)src->layer_bytes, (int64_t)dst->layer_bytes);
}

bs_status bs_copy_bytes(void* dst, const void* src, size_t bytes, void* stream) {
  BS_REQUIRE(bytes == 0 || (dst && src), "bs_copy_bytes: NULL pointer");
  if (bytes == 0) return BS_OK;
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return bs::set_error(BS_ERR_CUDA, "bs_copy_bytes: %s", cudaGetErrorString(e));
  return BS_OK;
}

bs_status bs_kv_migrate_layer(const bs_kv_pool* src, bs_kv_pool* dst, int32_t layer,
                              const int32_t* src_ids, const int32_t* dst_ids, int32_t n,
                              void* stream) {
  return bs_kv_migrate_layer_ex(src, dst, layer, src_ids, dst_ids, n, BS_MIGRATE_AUTO, stream);
}

bs_status bs_kv_migrate_layer_ce(const bs_kv_pool* src, bs_kv_pool* dst, int32_t layer,
                                 const int32_t* src_ids, const int32_t* dst_ids, int32_t n,
                                 void* stream) {
  BS_REQUIRE(src && dst, "bs_kv_migrate_layer_ce: NULL pool");
  BS_REQUIRE(same_geometry(src, dst), "bs_kv_migrate_layer_ce: src/dst geometry differs");
  BS_REQUIRE(layer >= 0 && layer < src->desc.num_layers, "bs_kv_migrate_layer_ce: layer out of range");
  BS_REQUIRE(n >= 0, "bs_kv_migrate_layer_ce: n < 0");
  if (n == 0) return BS_OK;
  BS_REQUIRE(src_ids && dst_ids, "bs_kv_migrate_layer_ce: NULL ids");
  const size_t chunk = src->chunk_bytes;
  std::vector<void*> dsts, srcs;
  std::vector<size_t> sizes;
  dsts.reserve(n);
  srcs.reserve(n);
  sizes.reserve(n);
  for (int32_t i = 0; i < n;) {
    const int32_t s0 = src_ids[i], d0 = dst_ids[i];
    BS_REQUIRE(s0 >= 0 && s0 < src->desc.num_blocks && d0 >= 0 && d0 < dst->desc.num_blocks,
               "bs_kv_migrate_layer_ce: pair %d (%d -> %d) out of range", i, s0, d0);
    int32_t run = 1;  // coalesce runs of consecutive ids on both sides into one copy
    while (i + run < n && src_ids[i + run] == s0 + run && dst_ids[i + run] == d0 + run &&
           s0 + run < src->desc.num_blocks && d0 + run < dst->desc.num_blocks)
      ++run;
    srcs.push_back(src->base + (size_t)layer * src->layer_bytes + (size_t)s0 * chunk);
    dsts.push_back(dst->base + (size_t)layer * dst->layer_bytes + (size_t)d0 * chunk);
    sizes.push_back((size_t)run * chunk);
    i += run;
  }
  // one cudaMemcpyAsync per coalesced run (the batched-descriptor API is not used: it
  // faulted GPUs of this pool, F1)
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  for (size_t k = 0; k < sizes.size(); ++k) {
    e = cudaMemcpyAsync(dsts[k], srcs[k], sizes[k], cudaMemcpyDefault, s);
    if (e != cudaSuccess) break;
  }
  if (e != cudaSuccess) return bs::set_error(BS_ERR_CUDA, "bs_kv_migrate_layer_ce: %s", cudaGetErrorString(e));
  return BS_OK;
}

bs_status bs_kv_migrate_heads_layer(const bs_kv_pool* src, bs_kv_pool* dst, int32_t layer,
                                    const int32_t* src_ids, const int32_t* dst_ids, int32_t n,
                                    int32_t src_head_lo, int32_t dst_head_lo, int32_t n_heads,
                                    void* stream) {
  BS_REQUIRE(src && dst, "bs_kv_migrate_heads_layer: NULL pool");
  BS_REQUIRE(src->desc.num_layers == dst->desc.num_layers && src->desc.head_dim == dst->desc.head_dim,
             "bs_kv_migrate_heads_layer: layers / head_dim differ");
  BS_REQUIRE(layer >= 0 && layer < src->desc.num_layers, "bs_kv_migrate_heads_layer: layer out of range");
  BS_REQUIRE(n_heads >= 1 && src_head_lo >= 0 && src_head_lo + n_heads <= src->desc.num_kv_heads &&
                 dst_head_lo >= 0 && dst_head_lo + n_heads <= dst->desc.num_kv_heads,
             "bs_kv_migrate_heads_layer: head range outside a pool");
  BS_REQUIRE(n >= 0, "bs_kv_migrate_heads_layer: n < 0");
  if (n == 0) return BS_OK;
  BS_REQUIRE(src_ids && dst_ids, "bs_kv_migrate_heads_layer: NULL ids");
  BS_DEBUG_CHECK(bs::debug_check_ids(src_ids, n, src->desc.num_blocks, static_cast<cudaStream_t>(stream),
                                     "bs_kv_migrate_heads_layer src_ids"));
  BS_DEBUG_CHECK(bs::debug_check_ids(dst_ids, n, dst->desc.num_blocks, static_cast<cudaStream_t>(stream),
                                     "bs_kv_migrate_heads_layer dst_ids"));
  const int sms = bs::sm_count(bs::current_device());
  const int64_t total = (int64_t)n * 2 * n_heads;
  const int wpc = 8;
  int64_t grid = std::min<int64_t>((total + wpc - 1) / wpc, (int64_t)sms * 8);
  if (src->host || dst->host) grid = std::min<int64_t>(grid, kHostCopyCtas);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint8_t* sb = src->base + (size_t)layer * src->layer_bytes;
  uint8_t* db = dst->base + (size_t)layer * dst->layer_bytes;
  if (src->page_bytes == 4096)
    bs::copy_head_pages_vec16<4096><<<(unsigned)grid, wpc * 32, 0, s>>>(
        sb, src_ids, (int64_t)src->chunk_bytes, src->desc.num_kv_heads, src_head_lo, db, dst_ids,
        (int64_t)dst->chunk_bytes, dst->desc.num_kv_heads, dst_head_lo, n, n_heads);
  else
    bs::copy_head_pages_vec16<2048><<<(unsigned)grid, wpc * 32, 0, s>>>(
        sb, src_ids, (int64_t)src->chunk_bytes, src->desc.num_kv_heads, src_head_lo, db, dst_ids,
        (int64_t)dst->chunk_bytes, dst->desc.num_kv_heads, dst_head_lo, n, n_heads);
  return bs::check_launch("copy_head_pages_vec16");
}

bs_status bs_kv_gather_layer(const bs_kv_pool* src, int32_t layer, const int32_t* ids, int32_t n,
                             void* staging, void* stream) {
  BS_REQUIRE(src, "bs_kv_gather_layer: NULL pool");
  BS_REQUIRE(layer >= 0 && layer < src->desc.num_layers, "bs_kv_gather_layer: layer out of range");
  BS_REQUIRE(n >= 0, "bs_kv_gather_layer: n < 0");
  BS_REQUIRE(n == 0 || (ids && staging), "bs_kv_gather_layer: NULL ids/staging");
  BS_REQUIRE(((uintptr_t)staging & 15) == 0, "bs_kv_gather_layer: staging not 16-B aligned");
  BS_DEBUG_CHECK(bs::debug_check_ids(ids, n, src->desc.num_blocks, static_cast<cudaStream_t>(stream),
                                     "bs_kv_gather_layer ids"));
  return bs::launch_copy_chunks(src->base + (size_t)layer * src->layer_bytes, ids,
                                static_cast<uint8_t*>(staging), nullptr, n, src->chunk_bytes,
                                src->page_bytes, BS_MIGRATE_AUTO, static_cast<cudaStream_t>(stream),
                                src->host ? kHostCopyCtas : 0);
}

bs_status bs_kv_scatter_layer(bs_kv_pool* dst, int32_t layer, const int32_t* ids, int32_t n,
                              const void* staging, void* stream) {
  BS_REQUIRE(dst, "bs_kv_scatter_layer: NULL pool");
  BS_REQUIRE(layer >= 0 && layer < dst->desc.num_layers, "bs_kv_scatter_layer: layer out of range");
  BS_REQUIRE(n >= 0, "bs_kv_scatter_layer: n < 0");
  BS_REQUIRE(n == 0 || (ids && staging), "bs_kv_scatter_layer: NULL ids/staging");
  BS_REQUIRE(((uintptr_t)staging & 15) == 0, "bs_kv_scatter_layer: staging not 16-B aligned");
  BS_DEBUG_CHECK(bs::debug_check_ids(ids, n, dst->desc.num_blocks, static_cast<cudaStream_t>(stream),
                                     "bs_kv_scatter_layer ids"));
  return bs::launch_copy_chunks(static_cast<const uint8_t*>(staging), nullptr,
                                dst->base + (size_t)layer * dst->layer_bytes, ids, n,
                                dst->chunk_bytes, dst->page_bytes, BS_MIGRATE_AUTO,
                                static_cast<cudaStream_t>(stream), dst->host ? kHostCopyCtas : 0);
}

}  // extern "C"
