// H0: pool descriptor + host block allocator, and the library's error plumbing.
// Paged KV blocks as in vLLM's PagedAttention; the per-migration
// "time to reallocate buffers" T_mem_realloc of eq. 28 is this
// allocator's cost.  Policy (reading R-A12): lowest free id first, all-or-nothing.
#include <algorithm>
#include <vector>

#include "internal.h"

namespace bs {

static thread_local std::string g_last_error;

bs_status set_error(bs_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

bs_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(BS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return BS_OK;
}

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

int sm_count(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (cache[device] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0)
      n = 148;
    cache[device] = n;
  }
  return cache[device];
}

}  // namespace bs

static bool desc_ok(const bs_kv_pool_desc* d) {
  return d && d->num_layers >= 1 && d->num_blocks >= 1 && d->block_size == 16 &&
         d->num_kv_heads >= 1 && (d->head_dim == 64 || d->head_dim == 128) &&
         d->dtype == BS_DTYPE_BF16 && (d->device >= 0 || d->device == BS_DEVICE_HOST);
}

extern "C" {

const char* bs_last_error(void) { return bs::g_last_error.c_str(); }

int32_t bs_abi_version(void) { return BS_ABI_VERSION; }

size_t bs_kv_chunk_bytes(const bs_kv_pool_desc* d) {
  if (!desc_ok(d)) return 0;
  return (size_t)2 * d->num_kv_heads * d->block_size * d->head_dim * 2;
}

size_t bs_kv_pool_bytes(const bs_kv_pool_desc* d) {
  if (!desc_ok(d)) return 0;
  return (size_t)d->num_layers * d->num_blocks * bs_kv_chunk_bytes(d);
}

bs_status bs_kv_pool_create(const bs_kv_pool_desc* desc, void* base, bs_kv_pool** out) {
  BS_REQUIRE(out != nullptr, "bs_kv_pool_create: out is NULL");
  *out = nullptr;
  BS_REQUIRE(desc != nullptr, "bs_kv_pool_create: desc is NULL");
  if (desc->block_size != 16 || (desc->head_dim != 64 && desc->head_dim != 128) ||
      desc->dtype != BS_DTYPE_BF16)
    return bs::set_error(BS_ERR_UNSUPPORTED,
                         "bs_kv_pool_create: need block_size 16, head_dim 64|128, bf16 "
                         "(got bs=%d d=%d dtype=%d)",
                         desc->block_size, desc->head_dim, desc->dtype);
  BS_REQUIRE(desc_ok(desc), "bs_kv_pool_create: bad geometry (L=%d blocks=%d Hkv=%d dev=%d)",
             desc->num_layers, desc->num_blocks, desc->num_kv_heads, desc->device);
  BS_REQUIRE(base != nullptr, "bs_kv_pool_create: base is NULL");
  BS_REQUIRE(((uintptr_t)base & 255) == 0, "bs_kv_pool_create: base must be 256-byte aligned");
  uint8_t* dbase = static_cast<uint8_t*>(base);
  if (desc->device == BS_DEVICE_HOST) {
    // Global KV Cache Store tier: page-locked host memory, reached by the copy kernels
    // through its UVA device mapping (zero-copy over PCIe / C2C)
    cudaPointerAttributes attr{};
    cudaError_t e = cudaPointerGetAttributes(&attr, base);
    if (e != cudaSuccess || attr.type != cudaMemoryTypeHost || !attr.devicePointer) {
      cudaGetLastError();
      return bs::set_error(BS_ERR_INVALID_ARG,
                           "bs_kv_pool_create: host pool base must be page-locked, mapped memory");
    }
    dbase = static_cast<uint8_t*>(attr.devicePointer);
  }
  bs_kv_pool* p = new (std::nothrow) bs_kv_pool();
  if (!p) return bs::set_error(BS_ERR_INVALID_ARG, "bs_kv_pool_create: host OOM");
  p->desc = *desc;
  p->base = dbase;
  p->host = desc->device == BS_DEVICE_HOST;
  p->chunk_bytes = bs_kv_chunk_bytes(desc);
  p->page_bytes = (size_t)desc->block_size * desc->head_dim * 2;
  p->layer_bytes = (size_t)desc->num_blocks * p->chunk_bytes;
  for (int32_t i = 0; i < desc->num_blocks; ++i) p->free_ids.insert(p->free_ids.end(), i);
  *out = p;
  return BS_OK;
}

bs_status bs_kv_pool_destroy(bs_kv_pool* pool) {
  delete pool;
  return BS_OK;
}

bs_status bs_kv_pool_alloc(bs_kv_pool* pool, int32_t n, int32_t* out_ids) {
  BS_REQUIRE(pool != nullptr, "bs_kv_pool_alloc: pool is NULL");
  BS_REQUIRE(n >= 0, "bs_kv_pool_alloc: n < 0");
  BS_REQUIRE(n == 0 || out_ids != nullptr, "bs_kv_pool_alloc: out_ids is NULL");
  std::lock_guard<std::mutex> g(pool->mu);
  if ((size_t)n > pool->free_ids.size())
    return bs::set_error(BS_ERR_OUT_OF_BLOCKS, "bs_kv_pool_alloc: want %d blocks, %zu free", n,
                         pool->free_ids.size());
  auto it = pool->free_ids.begin();
  for (int32_t i = 0; i < n; ++i) out_ids[i] = *it++;
  pool->free_ids.erase(pool->free_ids.begin(), it);
  return BS_OK;
}

bs_status bs_kv_pool_free(bs_kv_pool* pool, int32_t n, const int32_t* ids) {
  BS_REQUIRE(pool != nullptr, "bs_kv_pool_free: pool is NULL");
  BS_REQUIRE(n >= 0, "bs_kv_pool_free: n < 0");
  BS_REQUIRE(n == 0 || ids != nullptr, "bs_kv_pool_free: ids is NULL");
  std::lock_guard<std::mutex> g(pool->mu);
  std::vector<int32_t> v(ids, ids + n);
  std::sort(v.begin(), v.end());
  for (int32_t i = 0; i < n; ++i) {
    BS_REQUIRE(v[i] >= 0 && v[i] < pool->desc.num_blocks, "bs_kv_pool_free: id %d out of range",
               v[i]);
    BS_REQUIRE(i == 0 || v[i] != v[i - 1], "bs_kv_pool_free: id %d repeated", v[i]);
    BS_REQUIRE(pool->free_ids.count(v[i]) == 0, "bs_kv_pool_free: id %d is not allocated", v[i]);
  }
  for (int32_t x : v) pool->free_ids.insert(x);
  return BS_OK;
}

int32_t bs_kv_pool_num_free(const bs_kv_pool* pool) {
  if (!pool) return -1;
  std::lock_guard<std::mutex> g(const_cast<bs_kv_pool*>(pool)->mu);
  return (int32_t)pool->free_ids.size();
}

}  // extern "C"
