// Measurement helper (not part of the method): the achievable HBM *read*
// bandwidth of this device, the denominator SURVEY.md 8(d) asks for beside
// the copy peak of MEASURED_PEAKS.json (the attention kernel reads pages and
// writes comparatively little, so a read-only stream is its roofline).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "tts_internal.cuh"

namespace tts {
namespace {

// Grid-stride 16-byte loads, 4 in flight per thread, folded into one word per
// thread that is stored (4 B per thread: ~1 MB against GBs read) so that the
// loads stay live.  Three load flavours (the measured peak is the best):
// 0 = ld.global.nc with an L2 256-B prefetch hint, 1 = __ldg, 2 = __ldcs.
template <int kMode>
__device__ __forceinline__ uint4 ld16(const uint4* p) {
  if constexpr (kMode == 0) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
  } else if constexpr (kMode == 1) {
    return __ldg(p);
  } else {
    return __ldcs(p);
  }
}

template <int kMode>
__global__ void __launch_bounds__(512) k_read_stream(const uint4* __restrict__ p, int64_t n, uint32_t* sink) {
  uint32_t acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = ld16<kMode>(p + i), b = ld16<kMode>(p + i + stride), c = ld16<kMode>(p + i + 2 * stride),
          d = ld16<kMode>(p + i + 3 * stride);
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
  }
  for (; i < n; i += stride) {
    uint4 a = ld16<kMode>(p + i);
    acc ^= a.x ^ a.y ^ a.z ^ a.w;
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// One-shot variant: every thread reads 4 consecutive 16-B vectors (64 B) once.
__global__ void __launch_bounds__(256) k_read_once(const uint4* __restrict__ p, int64_t n, uint32_t* sink) {
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4;
  uint32_t acc = 0;
  if (i + 3 < n) {
    const uint4 a = __ldg(p + i), b = __ldg(p + i + 1), c = __ldg(p + i + 2), d = __ldg(p + i + 3);
    acc = a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
  }
  if (acc == 0x9E3779B9u) sink[threadIdx.x] = acc;
}

}  // namespace
}  // namespace tts

extern "C" tts_status_t tts_stream_read_gbs(const void* buf, size_t bytes, int32_t iters, double* gbs_h,
                                            void* stream) {
  if (!buf || bytes < 16 || iters <= 0 || !gbs_h) return TTS_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  TTS_CUDA(cudaGetDevice(&dev));
  TTS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t n = (int64_t)(bytes / 16);
  uint32_t* sink = nullptr;
  const int max_grid = 8 * sms;
  TTS_CUDA(cudaMalloc(&sink, (size_t)max_grid * 512 * 4));
  cudaEvent_t e0, e1;
  TTS_CUDA(cudaEventCreate(&e0));
  TTS_CUDA(cudaEventCreate(&e1));
  double best = 0.0;
  for (int mode = 0; mode < 3; ++mode)
    for (int per_sm : {2, 4, 8}) {
      const int grid = per_sm * sms;
      auto launch = [&]() {
        if (mode == 0) tts::k_read_stream<0><<<grid, 512, 0, st>>>((const uint4*)buf, n, sink);
        else if (mode == 1) tts::k_read_stream<1><<<grid, 512, 0, st>>>((const uint4*)buf, n, sink);
        else tts::k_read_stream<2><<<grid, 512, 0, st>>>((const uint4*)buf, n, sink);
      };
      launch();  // warm-up
      TTS_CUDA(cudaEventRecord(e0, st));
      for (int k = 0; k < iters; ++k) launch();
      TTS_CUDA(cudaEventRecord(e1, st));
      TTS_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      TTS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      best = std::max(best, (double)n * 16 * iters / (ms * 1e-3) / 1e9);
    }
  {
    const int64_t threads = n / 4;
    const int64_t blocks = (threads + 255) / 256;
    tts::k_read_once<<<(unsigned)blocks, 256, 0, st>>>((const uint4*)buf, n, sink);
    TTS_CUDA(cudaEventRecord(e0, st));
    for (int k = 0; k < iters; ++k) tts::k_read_once<<<(unsigned)blocks, 256, 0, st>>>((const uint4*)buf, n, sink);
    TTS_CUDA(cudaEventRecord(e1, st));
    TTS_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    TTS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    const double gbs = (double)(threads * 4) * 16 * iters / (ms * 1e-3) / 1e9;
    if (getenv("TTS_PROBE_VERBOSE")) fprintf(stderr, "read probe one-shot: %.0f GB/s (loop best %.0f)\n", gbs, best);
    best = std::max(best, gbs);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  *gbs_h = best;
  return TTS_OK;
}
