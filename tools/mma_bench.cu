// Microbenchmark: cycles per tcgen05.mma (kind::f16, cta_group::1, M=128, K=16)
// as a function of N, with A from TMEM (TS) or shared memory (SS), issued back
// to back by one thread and drained with tcgen05.commit -> mbarrier.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../include -o mma_bench mma_bench.cu
#include <cstdio>
#include <cstdint>

#include "../paper_2509_00195_b200/csrc/sm100.cuh"

using namespace tts::sm100;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k_bench(int n_mma, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t base = (su32(sm) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    bar_init(su32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  long long t0 = 0, t1 = 0;
  if (warp == 0) {
    constexpr uint32_t id = idesc_bf16(128, N, false);
    const uint64_t da = sdesc(base, 16, 1024, 2);
    const uint64_t db = sdesc(base + 32768, 16, 1024, 2);
    uint32_t ph = 0;
    for (int r = 0; r < reps; ++r) {
      __syncwarp();
      if (r == 1) t0 = clock64();
      if (elect_one()) {
        for (int i = 0; i < n_mma; ++i) {
          if (TS)
            mma_ts(tmem, tmem + 128, db, id, i > 0);
          else
            mma_ss(tmem, da, db, id, i > 0);
        }
        tc_commit(su32(&bar));
      }
      __syncwarp();
      bar_wait(su32(&bar), ph);
      ph ^= 1u;
    }
    t1 = clock64();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0);
}

template <int N, bool TS>
void run(int ctas, int n_mma) {
  long long* d;
  cudaMalloc(&d, ctas * sizeof(long long));
  const int smem = 70 * 1024;
  cudaFuncSetAttribute(k_bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 21;
  k_bench<N, TS><<<ctas, 128, smem>>>(n_mma, reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[512];
  cudaMemcpy(h, d, ctas * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < ctas; ++i) avg += h[i];
  avg /= ctas;
  printf("%s N=%3d ctas=%3d n_mma=%3d: %.1f cycles per mma (per CTA)  err=%d\n", TS ? "TS" : "SS", N, ctas, n_mma,
         avg / (reps - 1) / n_mma, (int)e);
  cudaFree(d);
}

int main() {
  for (int ctas : {1, 148, 296}) {
    for (int n_mma : {2, 16, 64}) {
      run<16, true>(ctas, n_mma);
      run<32, true>(ctas, n_mma);
      run<64, true>(ctas, n_mma);
      run<128, true>(ctas, n_mma);
      run<16, false>(ctas, n_mma);
      run<128, false>(ctas, n_mma);
    }
  }
  return 0;
}
