// Read-only HBM stream: the denominator the HBM-bound kernels' roofline is
// reported against besides the driver's copy figure (MEASURED_PEAKS.json
// hbm_gbs, read + write) and the 8 TB/s datasheet number. K1 and K4 only
// read, so their ceiling is this stream, not the copy.
//
// Persistent grid (4 CTAs x 512 threads per SM), eight independent 16-byte
// non-coherent loads in flight per thread (256 KB per SM), L1 not allocated.
#include <cstdlib>

#include "common.cuh"
#include "../../include/duchess_b200.h"

namespace duchess {

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

__global__ void __launch_bounds__(512) read_stream_kernel(const uint4* __restrict__ p,
                                                          int64_t n16, uint32_t* out) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ld_stream(p + i + k * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  for (; i < n16; i += stride) {
    const uint4 v = ld_stream(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9E3779B9u) out[0] = acc;   // keeps the loads; practically never stores
}

// Write-only HBM stream (measurement): the ceiling of write-dominated kernels
// (K3's fork copies write ~4x what they read). Persistent grid, 16-byte
// streaming stores, eight per thread per iteration.
template <bool STCS>
__device__ __forceinline__ void st16(uint4* p, uint4 v) {
  if constexpr (STCS) __stcs(p, v);
  else *p = v;
}
template <bool STCS>
__global__ void __launch_bounds__(512) write_stream_kernel(uint4* __restrict__ p, int64_t n16,
                                                           uint32_t seed) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint4 v = make_uint4(seed, seed ^ 0x9E3779B9u, seed + 1u, ~seed);
  for (; i + 7 * stride < n16; i += 8 * stride) {
#pragma unroll
    for (int k = 0; k < 8; ++k) st16<STCS>(p + i + k * stride, v);
  }
  for (; i < n16; i += stride) st16<STCS>(p + i, v);
}

// Launch gate (measurement): one thread waits until the host sets *flag
// (pinned host memory, read through its device mapping) or `timeout_ns`
// passes, so a benchmark can enqueue its whole timed region before the GPU
// starts it (device time then excludes host launch latency, as a blocking
// kernel does in nvbench). Writes 1 to *timed_out on timeout.
__global__ void gate_kernel(const volatile int32_t* flag, int64_t timeout_ns, int32_t* timed_out) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*flag == 0) {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (int64_t(t - t0) > timeout_ns) {
      *timed_out = 1;
      return;
    }
  }
}

}  // namespace duchess

using namespace duchess;

extern "C" int duchess_write_stream(void* buf, int64_t bytes, uint32_t seed, void* stream) {
  if (!buf || bytes < 16 || (reinterpret_cast<uintptr_t>(buf) & 15)) return DUCHESS_EINVAL;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // store flavour (env DUCHESS_WS_STCS=1: streaming .cs stores; default write-back)
  static const bool stcs = [] { const char* e = getenv("DUCHESS_WS_STCS"); return e && atoi(e) != 0; }();
  auto k = stcs ? write_stream_kernel<true> : write_stream_kernel<false>;
  k<<<unsigned(4 * sms), 512, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint4*>(buf), bytes / 16, seed);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_gate(const int32_t* host_flag, int64_t timeout_ns, int32_t* timed_out,
                            void* stream) {
  if (!host_flag || !timed_out || timeout_ns <= 0) return DUCHESS_EINVAL;
  gate_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(host_flag, timeout_ns, timed_out);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}

extern "C" int duchess_read_stream(const void* buf, int64_t bytes, uint32_t* sink, void* stream) {
  if (!buf || !sink || bytes < 16 || (reinterpret_cast<uintptr_t>(buf) & 15)) return DUCHESS_EINVAL;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  read_stream_kernel<<<unsigned(4 * sms), 512, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(buf), bytes / 16, sink);
  return cudaGetLastError() == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}
