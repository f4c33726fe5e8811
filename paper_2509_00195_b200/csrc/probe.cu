// Measurement helper (not part of the method): the achievable HBM *read*
// bandwidth of this device, the denominator SURVEY.md 8(d) asks for beside
// the copy peak of MEASURED_PEAKS.json (the attention kernel reads pages and
// writes comparatively little, so a read-only stream is its roofline).
#include "tts_internal.cuh"

namespace tts {
namespace {

// Grid-stride 16-byte loads, 4 in flight per thread, folded into one word per
// thread that is stored (4 B per thread: ~1 MB against GBs read) so that the
// loads stay live.
__global__ void __launch_bounds__(512) k_read_stream(const uint4* __restrict__ p, int64_t n, uint32_t* sink) {
  uint32_t acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride),
          d = __ldcs(p + i + 3 * stride);
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
  }
  for (; i < n; i += stride) {
    uint4 a = __ldcs(p + i);
    acc ^= a.x ^ a.y ^ a.z ^ a.w;
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
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
  const int grid = 4 * sms;  // 4 x 512 threads per SM
  uint32_t* sink = nullptr;
  TTS_CUDA(cudaMalloc(&sink, (size_t)grid * 512 * 4));
  cudaEvent_t e0, e1;
  TTS_CUDA(cudaEventCreate(&e0));
  TTS_CUDA(cudaEventCreate(&e1));
  tts::k_read_stream<<<grid, 512, 0, st>>>((const uint4*)buf, n, sink);  // warm-up
  TTS_CUDA(cudaEventRecord(e0, st));
  for (int k = 0; k < iters; ++k) tts::k_read_stream<<<grid, 512, 0, st>>>((const uint4*)buf, n, sink);
  TTS_CUDA(cudaEventRecord(e1, st));
  TTS_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  TTS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  *gbs_h = (double)n * 16 * iters / (ms * 1e-3) / 1e9;
  return TTS_OK;
}
