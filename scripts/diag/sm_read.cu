// Diagnostics only (not part of the library): how fast can ONE SM pull data from HBM?
// Each CTA (one per SM: 200 KB of dynamic shared memory) streams its own contiguous
// `per_cta` bytes, either with 16-byte LDGs (512 threads, U loads in flight per thread) or
// with 1-D TMA bulk copies (one thread, a ring of `stages` 8-KiB slots completing on
// mbarriers).  With few CTAs the HBM is far from saturated, so the per-CTA rate is the SM's
// own ceiling for that load path -- the question behind the small C3 launches.
#include <cuda_runtime.h>
#include <cstdint>

template <int U>
__global__ void __launch_bounds__(512, 1) ldg_kernel(const int4* __restrict__ p, int64_t per_cta16, int* sink) {
  const int4* base = p + (int64_t)blockIdx.x * per_cta16;
  int acc = 0;
  for (int64_t i = threadIdx.x; i < per_cta16; i += (int64_t)blockDim.x * U) {
    int4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + (int64_t)u * blockDim.x;
      if (j < per_cta16)
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[u].x), "=r"(r[u].y), "=r"(r[u].z), "=r"(r[u].w)
                     : "l"(base + j));
      else
        r[u] = make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
  }
  if (acc == 0x7fffffff) sink[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32, 1) tma_kernel(const uint8_t* __restrict__ p, int64_t per_cta, int stages,
                                                    int* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int kChunk = 8192;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + stages * kChunk);
  const uint8_t* base = p + (int64_t)blockIdx.x * per_cta;
  const int64_t n = per_cta / kChunk;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto issue = [&](int64_t k) {
    const int s = (int)(k % stages);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[s])), "r"(kChunk)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(smem + s * kChunk)),
                 "l"(base + k * kChunk), "r"(kChunk), "r"(su32(&bars[s]))
                 : "memory");
  };
  for (int64_t k = 0; k < stages && k < n; ++k) issue(k);
  int acc = 0;
  for (int64_t k = 0; k < n; ++k) {
    const int s = (int)(k % stages);
    const uint32_t par = (uint32_t)((k / stages) & 1);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n}"
                   : "=r"(ok) : "r"(su32(&bars[s])), "r"(par) : "memory");
    acc ^= smem[s * kChunk];
    if (k + stages < n) issue(k + stages);
  }
  if (acc == 0x7fffffff) sink[0] = acc;
}

extern "C" int sm_read(const void* p, int64_t per_cta, int nctas, int mode, int param, int* sink, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int smem_pad = 200 * 1024;  // one CTA per SM
  if (mode == 0) {  // LDG, param = loads in flight per thread
    static bool cfg = false;
    if (!cfg) {
      cudaFuncSetAttribute(ldg_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_pad);
      cudaFuncSetAttribute(ldg_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_pad);
      cudaFuncSetAttribute(ldg_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_pad);
      cfg = true;
    }
    const int64_t n16 = per_cta / 16;
    if (param == 8) ldg_kernel<8><<<nctas, 512, smem_pad, s>>>(static_cast<const int4*>(p), n16, sink);
    else if (param == 16) ldg_kernel<16><<<nctas, 512, smem_pad, s>>>(static_cast<const int4*>(p), n16, sink);
    else ldg_kernel<32><<<nctas, 512, smem_pad, s>>>(static_cast<const int4*>(p), n16, sink);
  } else {          // TMA bulk, param = ring stages of 8 KiB
    static bool cfg = false;
    if (!cfg) {
      cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      cfg = true;
    }
    const int smem = param * 8192 + param * 8;
    tma_kernel<<<nctas, 32, smem < smem_pad ? smem_pad : smem, s>>>(static_cast<const uint8_t*>(p), per_cta,
                                                                    param, sink);
  }
  return (int)cudaGetLastError();
}
