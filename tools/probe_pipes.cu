// Per-SM issue throughput of the softmax's instruction kinds on this part:
// MUFU.EX2, F2FP.BF16 pack, FFMA2, FADD2, FMNMX, IMAD (results / clock / SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_pipes tools/probe_pipes.cu && /tmp/probe_pipes
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

constexpr int ITERS = 4096;

template <int KIND>
__global__ void probe(float* out, long long* cyc, float seed) {
  float a[8];
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + i) * 1e-3f; u[i] = __float_as_uint(a[i]); }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (KIND == 1) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        u[i] ^= r;
      }
      if (KIND == 2) {
        uint64_t x = (uint64_t)u[i] | ((uint64_t)u[(i + 1) & 7] << 32), y;
        asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(y) : "l"(x));
        u[i] = (uint32_t)y ^ (uint32_t)(y >> 32);
      }
      if (KIND == 3) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      if (KIND == 4) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i + 3) & 7]));
      if (KIND == 5) asm volatile("mad.lo.u32 %0, %0, 8388608, %0;" : "+r"(u[i]));
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"MUFU.EX2", "F2FP.BF16 (cvt.rn.bf16x2.f32)", "FFMA2 (fma.rn.f32x2)", "FFMA", "FMNMX", "IMAD"};
  for (int warps : {4, 8, 16}) {
    for (int k = 0; k < 6; ++k) {
      void (*f)(float*, long long*, float) = k == 0 ? probe<0> : k == 1 ? probe<1> : k == 2 ? probe<2> : k == 3 ? probe<3> : k == 4 ? probe<4> : probe<5>;
      f<<<148, warps * 32>>>(out, cyc, 1.0f);
      f<<<148, warps * 32>>>(out, cyc, 1.0f);
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double ops = (double)ITERS * 8 * warps * 32;
      printf("warps/SM %2d  %-32s %7.1f results/clk/SM  (%lld cycles)\n", warps, names[k], ops / c, c);
    }
  }
  return 0;
}
