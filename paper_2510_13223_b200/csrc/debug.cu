// Debug build only (BS_DEBUG=1, libbanaserve_debug.so; SURVEY.md §8(b) "a debug build adds
// device-side bounds checks that set an error flag the harness reads"): before a kernel
// consumes DEVICE index arrays (block ids, block tables, kv_split, append positions), a small validation
// kernel checks them on the device; the call then synchronises its stream, and on a
// violation records the code (bs_debug_error_code) and returns BS_ERR_INVALID_ARG without
// launching the real kernel.  Release builds compile none of this (bs_debug_build() == 0).
#include <atomic>

#include "internal.h"

namespace {
std::atomic<int32_t> g_code{0};
}

#ifdef BS_DEBUG
namespace bs {
namespace {

__global__ void check_ids_kernel(const int32_t* ids, int32_t n, int32_t limit, int32_t* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t x = ids[i];
    if (x < 0 || x >= limit) atomicOr(bad, 4);
  }
}

// one CTA per request: the shard's length must be >= 0 and fit the table width; every
// block id the shard uses must lie in [0, num_blocks)
__global__ void check_table_kernel(const int32_t* kv_split, int32_t n_shards, int32_t shard,
                                   const int32_t* bt, int32_t max_blocks, int32_t num_blocks,
                                   int32_t* bad) {
  const int b = blockIdx.x;
  const int32_t* ks = kv_split + (int64_t)b * (n_shards + 1) + shard;
  const int32_t len = ks[1] - ks[0];
  if (len < 0) {
    if (threadIdx.x == 0) atomicOr(bad, 2);
    return;
  }
  const int32_t nblk = (len + 15) / 16;
  if (nblk > max_blocks && threadIdx.x == 0) atomicOr(bad, 2);
  for (int i = threadIdx.x; i < min(nblk, max_blocks); i += blockDim.x) {
    const int32_t x = bt[(int64_t)b * max_blocks + i];
    if (x < 0 || x >= num_blocks) atomicOr(bad, 1);
  }
}

// H7 append: pos[b] < 0 (skip) or pos[b] / 16 < max_blocks, and its block id in range
__global__ void check_append_kernel(const int32_t* pos, int32_t batch, const int32_t* bt,
                                    int32_t max_blocks, int32_t num_blocks, int32_t* bad) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < batch; b += gridDim.x * blockDim.x) {
    const int32_t p = pos[b];
    if (p < 0) continue;
    if (p / 16 >= max_blocks) {
      atomicOr(bad, 8);
      continue;
    }
    const int32_t x = bt[(int64_t)b * max_blocks + p / 16];
    if (x < 0 || x >= num_blocks) atomicOr(bad, 1);
  }
}

// The checks synchronise the stream, which a stream capture forbids: launches enqueued while
// capturing a CUDA graph are not checked (the same launches run checked when issued eagerly).
bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return st != cudaStreamCaptureStatusNone;
}

int32_t* flag_buffer() {
  static int32_t* buf[64] = {nullptr};
  const int d = current_device();
  if (!buf[d]) cudaMalloc(&buf[d], sizeof(int32_t));
  return buf[d];
}

bs_status finish(int32_t* flag, cudaStream_t s, const char* what) {
  int32_t host = 0;
  cudaMemcpyAsync(&host, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_error(BS_ERR_CUDA, "%s (debug check): %s", what, cudaGetErrorString(e));
  if (host) {
    g_code.fetch_or(host);
    return set_error(BS_ERR_INVALID_ARG, "%s: device index arrays invalid (debug code %d)", what, host);
  }
  return BS_OK;
}

}  // namespace

bs_status debug_check_ids(const int32_t* ids, int32_t n, int32_t limit, cudaStream_t s,
                          const char* what) {
  if (capturing(s)) return BS_OK;
  if (n <= 0) return BS_OK;
  int32_t* flag = flag_buffer();
  cudaMemsetAsync(flag, 0, sizeof(int32_t), s);
  check_ids_kernel<<<std::min<int64_t>((n + 255) / 256, 1024), 256, 0, s>>>(ids, n, limit, flag);
  return finish(flag, s, what);
}

bs_status debug_check_table(const int32_t* kv_split, int32_t n_shards, int32_t shard, int32_t batch,
                            const int32_t* bt, int32_t max_blocks, int32_t num_blocks, cudaStream_t s,
                            const char* what) {
  if (capturing(s)) return BS_OK;
  if (batch <= 0) return BS_OK;
  int32_t* flag = flag_buffer();
  cudaMemsetAsync(flag, 0, sizeof(int32_t), s);
  check_table_kernel<<<batch, 128, 0, s>>>(kv_split, n_shards, shard, bt, max_blocks, num_blocks, flag);
  return finish(flag, s, what);
}

bs_status debug_check_append(const int32_t* pos, int32_t batch, const int32_t* bt, int32_t max_blocks,
                             int32_t num_blocks, cudaStream_t s, const char* what) {
  if (capturing(s)) return BS_OK;
  if (batch <= 0) return BS_OK;
  int32_t* flag = flag_buffer();
  cudaMemsetAsync(flag, 0, sizeof(int32_t), s);
  check_append_kernel<<<(batch + 255) / 256, 256, 0, s>>>(pos, batch, bt, max_blocks, num_blocks, flag);
  return finish(flag, s, what);
}

}  // namespace bs
#endif  // BS_DEBUG

extern "C" {

int32_t bs_debug_build(void) {
#ifdef BS_DEBUG
  return 1;
#else
  return 0;
#endif
}

int32_t bs_debug_error_code(int32_t reset) {
  return reset ? g_code.exchange(0) : g_code.load();
}

}  // extern "C"
