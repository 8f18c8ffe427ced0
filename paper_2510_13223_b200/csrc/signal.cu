// Cross-instance signalling for the P2P transport: a producer pushes data
// straight into a peer-mapped buffer (remote-view pool, q or partial buffer) and then
// raises a flag in the consumer's memory; the consumer's stream waits on its local flag.
// Flags carry a monotonically increasing epoch (the decode step), so they never need
// resetting.  A waiter gives up after `timeout_ns` and records the failure in `err`
// instead of hanging the GPU.
#include <cuda_runtime.h>

#include "internal.h"

namespace bs {
namespace {

__global__ void signal_kernel(int32_t* flag, int32_t value) {
  // every write enqueued before this kernel on the stream is complete (kernel boundary);
  // make it visible system-wide, then publish the flag with release semantics
  __threadfence_system();
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

__global__ void wait_kernel(const int32_t* flag, int32_t value, uint64_t timeout_ns, int32_t* err) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned ns = 32;
  while (true) {
    int32_t v;
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= value) break;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (timeout_ns && t - t0 > timeout_ns) {
      if (err) atomicExch(err, 1);
      break;
    }
    __nanosleep(ns);
    if (ns < 4096) ns <<= 1;
  }
}

constexpr int kMaxWaits = 16;

struct Flags {
  int32_t* flag[kMaxWaits];
  int32_t n;
};

__global__ void signal_many_kernel(const Flags f, int32_t value) {
  if ((int)threadIdx.x >= f.n) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(f.flag[threadIdx.x]), "r"(value) : "memory");
}

struct Waits {
  const int32_t* flag[kMaxWaits];
  int32_t value[kMaxWaits];
  int32_t n;
};

__global__ void wait_many_kernel(const Waits w, uint64_t timeout_ns, int32_t* err) {
  if ((int)threadIdx.x >= w.n) return;
  const int32_t* flag = w.flag[threadIdx.x];
  const int32_t value = w.value[threadIdx.x];
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned ns = 32;
  while (true) {
    int32_t v;
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= value) break;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (timeout_ns && t - t0 > timeout_ns) {
      if (err) atomicExch(err, 1);
      break;
    }
    __nanosleep(ns);
    if (ns < 4096) ns <<= 1;
  }
}

}  // namespace
}  // namespace bs

extern "C" {

bs_status bs_signal(int32_t* flag, int32_t value, void* stream) {
  BS_REQUIRE(flag, "bs_signal: NULL flag");
  bs::signal_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(flag, value);
  return bs::check_launch("signal_kernel");
}

bs_status bs_wait_signal(const int32_t* flag, int32_t value, uint64_t timeout_ns, int32_t* err,
                         void* stream) {
  BS_REQUIRE(flag, "bs_wait_signal: NULL flag");
  bs::wait_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(flag, value, timeout_ns, err);
  return bs::check_launch("wait_kernel");
}

bs_status bs_signals(int32_t n, int32_t* const* flags, int32_t value, void* stream) {
  BS_REQUIRE(n >= 1 && n <= bs::kMaxWaits, "bs_signals: n=%d (1..%d)", n, bs::kMaxWaits);
  BS_REQUIRE(flags, "bs_signals: NULL array");
  bs::Flags f{};
  for (int i = 0; i < n; ++i) {
    BS_REQUIRE(flags[i], "bs_signals: NULL flag %d", i);
    f.flag[i] = flags[i];
  }
  f.n = n;
  bs::signal_many_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(f, value);
  return bs::check_launch("signal_many_kernel");
}

bs_status bs_wait_signals(int32_t n, const int32_t* const* flags, const int32_t* values,
                          uint64_t timeout_ns, int32_t* err, void* stream) {
  BS_REQUIRE(n >= 1 && n <= bs::kMaxWaits, "bs_wait_signals: n=%d (1..%d)", n, bs::kMaxWaits);
  BS_REQUIRE(flags && values, "bs_wait_signals: NULL array");
  bs::Waits w{};
  for (int i = 0; i < n; ++i) {
    BS_REQUIRE(flags[i], "bs_wait_signals: NULL flag %d", i);
    w.flag[i] = flags[i];
    w.value[i] = values[i];
  }
  w.n = n;
  bs::wait_many_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(w, timeout_ns, err);
  return bs::check_launch("wait_many_kernel");
}

}  // extern "C"
