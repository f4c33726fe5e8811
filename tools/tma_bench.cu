// TMA request-rate microbenchmark for the attention kernel's load pattern
// (one CTA per SM, a producer warp whose lanes 0-7 each issue one page's
// requests, a consumer warp that releases each slot as soon as it lands).
// Per unit: 64 KiB (8 pages x K + V) from random page ids of a large pool.
//   mode 0: 16 x 2D K half-boxes (2 KiB) + 8 x 3D V boxes (4 KiB)  (24 requests, the kernel's)
//   mode 1: 16 x 3D boxes of 4 KiB (one per page for K and V)       (16 requests)
//   mode 2: 4 x 2D boxes of 16 KiB (8 contiguous pages per box)      (4 requests)
//   mode 3: 16 x cp.async.bulk of 4 KiB (no tensor map)              (16 requests)
// usage: tma_bench [units_per_cta] ; prints GB/s per mode
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#include "../paper_2509_00195_b200/csrc/sm100.cuh"
using namespace tts::sm100;

constexpr int kSlots = 3;
constexpr int kSlot = 64 * 1024;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

template <int kMode>
__global__ void __launch_bounds__(64, 1)
    k_bench(const __grid_constant__ CUtensorMap t2, const __grid_constant__ CUtensorMap t3,
            const __grid_constant__ CUtensorMap t16, const uint8_t* pool, int npages, int units, int* sink) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (su32(smem_raw) + 1023u) & ~1023u;
  __shared__ uint64_t bars[2 * kSlots];
  const uint32_t b_full = su32(bars), b_empty = b_full + 8 * kSlots;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) {
      bar_init(b_full + 8 * i, 1);
      bar_init(b_empty + 8 * i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    int slot = 0;
    uint32_t ph = 0;
    for (int u = 0; u < units; ++u) {
      bar_wait(b_empty + 8 * slot, ph ^ 1u);
      const uint32_t fb = b_full + 8 * slot;
      if (lane == 0) bar_expect(fb, kSlot);
      __syncwarp();
      const uint32_t sb = base + slot * kSlot;
      const uint32_t h = hash32((uint32_t)(blockIdx.x * 1000003u + u * 8u + lane));
      if (kMode == 2) {
        if (lane < 4) {
          const int run = (int)(h % (uint32_t)(npages / 8 - 1));
          tma2d(sb + lane * 16384, &t16, 0, run * 8 * 32, fb);  // 128 rows of 128 B (half 0 view)
        }
      } else if (lane < 8) {
        const int page = (int)(h % (uint32_t)npages);
        const int y = page * 32;  // a page = 32 rows of 128 B (K 16 tokens x 256 B as two halves)
        if (kMode == 0) {
          tma2d(sb + lane * 2048, &t2, 0, y / 2, fb);
          tma2d(sb + 16384 + lane * 2048, &t2, 64, y / 2, fb);
          const int page2 = (int)(hash32(h) % (uint32_t)npages);
          tma3d(sb + 32768 + lane * 4096, &t3, 0, page2 * 16, 0, fb);
        } else if (kMode == 1) {
          tma3d(sb + lane * 4096, &t3, 0, page * 16, 0, fb);
          const int page2 = (int)(hash32(h) % (uint32_t)npages);
          tma3d(sb + 32768 + lane * 4096, &t3, 0, page2 * 16, 0, fb);
        } else {
          bulk_g2s(sb + lane * 4096, pool + (size_t)page * 4096, 4096, fb);
          const int page2 = (int)(hash32(h) % (uint32_t)npages);
          bulk_g2s(sb + 32768 + lane * 4096, pool + (size_t)page2 * 4096, 4096, fb);
        }
      }
      __syncwarp();
      if (++slot == kSlots) {
        slot = 0;
        ph ^= 1u;
      }
    }
  } else {
    int slot = 0;
    uint32_t ph = 0;
    int acc = 0;
    for (int u = 0; u < units; ++u) {
      bar_wait(b_full + 8 * slot, ph);
      acc += smem_raw[(base - su32(smem_raw)) + slot * kSlot + lane * 4];
      __syncwarp();
      if (lane == 0) bar_arrive(b_empty + 8 * slot);
      if (++slot == kSlots) {
        slot = 0;
        ph ^= 1u;
      }
    }
    if (acc == 123456789) sink[0] = acc;
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int units = argc > 1 ? atoi(argv[1]) : 400;
  const size_t pool_bytes = (size_t)8 << 30;  // 8 GiB >> L2
  const int npages = (int)(pool_bytes / 4096);
  uint8_t* pool;
  cudaMalloc(&pool, pool_bytes);
  cudaMemset(pool, 1, pool_bytes);
  int* sink;
  cudaMalloc(&sink, 4);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
  const cuuint64_t rows = pool_bytes / 256;  // rows of 128 bf16
  CUtensorMap t2, t3, t16;
  {
    cuuint64_t dims[2] = {128, rows};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, 16};
    cuuint32_t es[2] = {1, 1};
    enc(&t2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pool, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t dims[3] = {64, rows, 2};
    cuuint64_t strides[2] = {256, 128};
    cuuint32_t box[3] = {64, 16, 2};
    cuuint32_t es[3] = {1, 1, 1};
    enc(&t3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, pool, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t dims[2] = {64, rows * 2};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    enc(&t16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pool, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = kSlots * kSlot + 1024;
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int grid : {sms, 2 * sms}) {
      if (grid == 2 * sms) continue;
      kern<<<grid, 64, smem>>>(t2, t3, t16, pool, npages, units, sink);
      cudaDeviceSynchronize();
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      for (int it = 0; it < 5; ++it) kern<<<grid, 64, smem>>>(t2, t3, t16, pool, npages, units, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = 5.0 * grid * units * (double)kSlot;
      printf("%-44s grid %d: %.1f GB/s  (%.2f us per unit per CTA)  err=%s\n", name, grid, bytes / ms / 1e6,
             ms * 1e3 / 5 / units, cudaGetErrorString(cudaGetLastError()));
    }
  };
  run(k_bench<0>, "mode0 16x2KiB K halves + 8x4KiB V (24 req)");
  run(k_bench<1>, "mode1 16x4KiB 3D boxes (16 req)");
  run(k_bench<2>, "mode2 4x16KiB boxes (4 req)");
  run(k_bench<3>, "mode3 16x4KiB cp.async.bulk (16 req)");
  return 0;
}
