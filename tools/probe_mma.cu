// tcgen05.mma issue-to-completion throughput per SM for the FMHA shapes:
// cycles per 128 x N x 16 bf16 MMA, A from shared memory (SS) or TMEM (TS),
// B K-major or MN-major SW128 in shared memory.  One CTA per SM, 1024 MMAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_18750_b200/csrc -o tools/bin/probe_mma tools/probe_mma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100_ptx.cuh"

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int N, int TS, int BMN>
__global__ void __launch_bounds__(128, 1) probe(long long* out, int n_mma) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { sm100::mbar_init(&bar, 1); sm100::fence_barrier_init(); }
  if (warp == 0) sm100::tmem_alloc<512>(&tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0 && lane == 0) {
    constexpr uint32_t idesc = sm100::idesc_bf16(128, N, 0, BMN);
    const uint32_t a_s = sm100::smem_u32(smem), b_s = sm100::smem_u32(smem + 65536);
    long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int k = i & 7;
      const uint64_t bd = BMN ? sm100::umma_desc_sw128(b_s + k * 2048, 16384, 1024)
                              : sm100::umma_desc_sw128(b_s + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
      const uint32_t d = tmem + 256 + ((i >> 3) & 1) * 128;   // D in columns 256..511
      if (TS) mma_ts(d, tmem + k * 8, bd, idesc, k != 0);
      else sm100::mma_bf16(d, sm100::umma_desc_sw128(a_s + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), bd, idesc, k != 0);
    }
    sm100::mma_commit(&bar);
    sm100::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) { sm100::tc_fence_after(); sm100::tmem_dealloc<512>(tmem); }
}

template <int N, int TS, int BMN>
void run(const char* name, long long* d, int grid) {
  auto k = probe<N, TS, BMN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const int n = 4096;
  for (int rep = 0; rep < 3; ++rep) k<<<grid, 128, 140 * 1024>>>(d, n);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  long long mx = 0, mn = 1LL << 60;
  for (int i = 0; i < grid; ++i) { mx = h[i] > mx ? h[i] : mx; mn = h[i] < mn ? h[i] : mn; }
  printf("%-34s grid %3d: %6.1f cycles/MMA (min CTA %6.1f)  -> %5.0f FLOP/clk/SM  err=%s\n", name, grid,
         (double)mx / n, (double)mn / n, 2.0 * 128 * N * 16 * n / mx, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  for (int grid : {1, 148}) {
    run<128, 0, 0>("SS 128x128x16, B K-major", d, grid);
    run<128, 0, 1>("SS 128x128x16, B MN-major", d, grid);
    run<128, 1, 1>("TS 128x128x16, B MN-major", d, grid);
    run<128, 1, 0>("TS 128x128x16, B K-major", d, grid);
    run<256, 0, 0>("SS 128x256x16, B K-major", d, grid);
    run<64, 0, 0>("SS 128x64x16, B K-major", d, grid);
  }
  return 0;
}
