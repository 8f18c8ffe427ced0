// Diagnostics only (not part of the library): pure-read HBM bandwidth on this GPU, the
// ceiling for the read-dominated attention kernel (MEASURED_PEAKS.json's hbm_gbs is a
// read+write copy).  16-byte non-allocating loads, U in flight per thread, grid-stride.
#include <cuda_runtime.h>
#include <cstdint>

template <int U>
__global__ void __launch_bounds__(512) read_kernel(const int4* __restrict__ p, int64_t n, int* sink) {
  int acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x) * U + threadIdx.x; i < n; i += stride) {
    int4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + (int64_t)u * blockDim.x;
      if (j < n)
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[u].x), "=r"(r[u].y), "=r"(r[u].z), "=r"(r[u].w)
                     : "l"(p + j));
      else
        r[u] = make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
  }
  if (acc == 0x7fffffff) sink[0] = acc;
}

extern "C" int hbm_read(const void* p, int64_t bytes, int ctas_per_sm, int unroll, int* sink, void* stream) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t n = bytes / 16;
  const dim3 grid(sms * ctas_per_sm);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (unroll == 4) read_kernel<4><<<grid, 512, 0, s>>>(static_cast<const int4*>(p), n, sink);
  else if (unroll == 8) read_kernel<8><<<grid, 512, 0, s>>>(static_cast<const int4*>(p), n, sink);
  else read_kernel<16><<<grid, 512, 0, s>>>(static_cast<const int4*>(p), n, sink);
  return (int)cudaGetLastError();
}
