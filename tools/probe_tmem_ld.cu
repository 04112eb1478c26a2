// Does a tcgen05.ld wait behind tcgen05.mma already queued by the CTA (to other
// TMEM columns)?  Warp 0 issues N MMAs (128x128x16, D in columns 256..383);
// warp 4 then times tcgen05.ld + wait::ld of 32 columns in 0..127.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_18750_b200/csrc -o tools/bin/probe_tmem_ld tools/probe_tmem_ld.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100_ptx.cuh"

__global__ void __launch_bounds__(256, 1) probe(long long* out, int n_mma) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int go;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { sm100::mbar_init(&bar, 1); sm100::fence_barrier_init(); go = 0; }
  if (warp == 0) sm100::tmem_alloc<512>(&tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0 && lane == 0) {
    constexpr uint32_t idesc = sm100::idesc_bf16(128, 128, 0, 0);
    const uint32_t a_s = sm100::smem_u32(smem), b_s = sm100::smem_u32(smem + 65536);
    for (int i = 0; i < n_mma; ++i) {
      const int k = i & 7;
      sm100::mma_bf16(tmem + 256, sm100::umma_desc_sw128(a_s + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024),
                      sm100::umma_desc_sw128(b_s + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), idesc, k != 0);
    }
    go = 1;
    sm100::mma_commit(&bar);
    long long t0 = clock64();
    sm100::mbar_wait(&bar, 0);
    out[blockIdx.x * 4 + 1] = clock64() - t0;   // time until the queued MMAs completed
  }
  if (warp == 4) {
    while (!go) {}
    long long t0 = clock64();
    uint32_t r[32];
    sm100::tmem_ld32(tmem, r);
    sm100::tmem_ld_wait();
    long long t1 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < 32; ++i) acc ^= r[i];
    if (lane == 0) { out[blockIdx.x * 4] = t1 - t0; out[blockIdx.x * 4 + 2] = acc; }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) { sm100::tc_fence_after(); sm100::tmem_dealloc<512>(tmem); }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 4 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  for (int n : {0, 8, 16, 32, 64}) {
    probe<<<1, 256, 140 * 1024>>>(d, n);
    probe<<<1, 256, 140 * 1024>>>(d, n);
    cudaDeviceSynchronize();
    long long h[4];
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("MMAs queued %3d: tcgen05.ld+wait %6lld cycles; MMA queue drained after %6lld cycles (%s)\n", n, h[0], h[1],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
