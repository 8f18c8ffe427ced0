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

// Flags and counters are int32 and grow without bound (epochs, merge counts): they wrap
// after 2^31.  "reached" is therefore a wrap-safe comparison -- the signed distance from
// the target -- valid while the two values are within 2^31 of each other (always: a
// waiter is at most a few steps behind its producer).
__device__ __forceinline__ bool reached(int32_t v, int32_t target) {
  return (int32_t)((uint32_t)v - (uint32_t)target) >= 0;
}

// A timed-out waiter records the failure with a plain system-scope store (err may live in
// device memory or in page-locked host memory the host polls without synchronising).
__device__ __forceinline__ void raise_err(int32_t* err) {
  if (err) asm volatile("st.relaxed.sys.global.s32 [%0], %1;" ::"l"(err), "r"(1) : "memory");
}

__device__ void spin_until(const int32_t* flag, int32_t value, uint64_t timeout_ns, int32_t* err) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned ns = 32;
  while (true) {
    int32_t v;
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (reached(v, value)) break;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (timeout_ns && t - t0 > timeout_ns) {
      raise_err(err);
      break;
    }
    __nanosleep(ns);
    if (ns < 4096) ns <<= 1;
  }
}

__global__ void wait_kernel(const int32_t* flag, int32_t value, uint64_t timeout_ns, int32_t* err) {
  spin_until(flag, value, timeout_ns, err);
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
  spin_until(w.flag[threadIdx.x], w.value[threadIdx.x], timeout_ns, err);
}

// Device-epoch variants (CUDA-graph capturable steps): the value is computed on the device
// from the step counter, value = (*epoch) * mul + add (int32, wrapping), so a captured
// graph replays with the current step's values.
struct EpochFlags {
  int32_t* flag[kMaxWaits];
  int32_t mul[kMaxWaits], add[kMaxWaits];
  int32_t n;
};

__global__ void signal_epoch_kernel(const EpochFlags f, const int32_t* epoch) {
  if ((int)threadIdx.x >= f.n) return;
  const uint32_t e = (uint32_t)*epoch;
  const int32_t v = (int32_t)(e * (uint32_t)f.mul[threadIdx.x] + (uint32_t)f.add[threadIdx.x]);
  __threadfence_system();
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(f.flag[threadIdx.x]), "r"(v) : "memory");
}

__global__ void wait_epoch_kernel(const EpochFlags f, const int32_t* epoch, uint64_t timeout_ns,
                                  int32_t* err) {
  if ((int)threadIdx.x >= f.n) return;
  const uint32_t e = (uint32_t)*epoch;
  const int32_t v = (int32_t)(e * (uint32_t)f.mul[threadIdx.x] + (uint32_t)f.add[threadIdx.x]);
  spin_until(f.flag[threadIdx.x], v, timeout_ns, err);
}

__global__ void epoch_advance_kernel(int32_t* epoch) {
  *epoch = (int32_t)((uint32_t)*epoch + 1u);
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

static bs_status fill_epoch_flags(const char* who, int32_t n, const void* const* flags,
                                  const int32_t* mul, const int32_t* add, bs::EpochFlags* f) {
  BS_REQUIRE(n >= 1 && n <= bs::kMaxWaits, "%s: n=%d (1..%d)", who, n, bs::kMaxWaits);
  BS_REQUIRE(flags && mul && add, "%s: NULL array", who);
  for (int i = 0; i < n; ++i) {
    BS_REQUIRE(flags[i], "%s: NULL flag %d", who, i);
    f->flag[i] = const_cast<int32_t*>(static_cast<const int32_t*>(flags[i]));
    f->mul[i] = mul[i];
    f->add[i] = add[i];
  }
  f->n = n;
  return BS_OK;
}

bs_status bs_signals_epoch(int32_t n, int32_t* const* flags, const int32_t* mul, const int32_t* add,
                           const int32_t* epoch, void* stream) {
  BS_REQUIRE(epoch, "bs_signals_epoch: NULL epoch");
  bs::EpochFlags f{};
  bs_status st = fill_epoch_flags("bs_signals_epoch", n, reinterpret_cast<const void* const*>(flags),
                                  mul, add, &f);
  if (st != BS_OK) return st;
  bs::signal_epoch_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(f, epoch);
  return bs::check_launch("signal_epoch_kernel");
}

bs_status bs_wait_signals_epoch(int32_t n, const int32_t* const* flags, const int32_t* mul,
                                const int32_t* add, const int32_t* epoch, uint64_t timeout_ns,
                                int32_t* err, void* stream) {
  BS_REQUIRE(epoch, "bs_wait_signals_epoch: NULL epoch");
  bs::EpochFlags f{};
  bs_status st = fill_epoch_flags("bs_wait_signals_epoch", n,
                                  reinterpret_cast<const void* const*>(flags), mul, add, &f);
  if (st != BS_OK) return st;
  bs::wait_epoch_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(f, epoch, timeout_ns, err);
  return bs::check_launch("wait_epoch_kernel");
}

bs_status bs_epoch_advance(int32_t* epoch, void* stream) {
  BS_REQUIRE(epoch, "bs_epoch_advance: NULL epoch");
  bs::epoch_advance_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(epoch);
  return bs::check_launch("epoch_advance_kernel");
}

}  // extern "C"
