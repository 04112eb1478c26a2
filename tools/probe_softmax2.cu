// Which part of the softmax step costs what (cycles per 128-column row step, one
// warp per SM sub-partition): variants of the same arithmetic.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/probe_softmax2 tools/probe_softmax2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ uint64_t u2pack(uint32_t lo, uint32_t hi) { return (uint64_t)lo | ((uint64_t)hi << 32); }
__device__ __forceinline__ float f2lo(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2hi(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int V>
__global__ void __launch_bounds__(512, 1) probe(const float* in, uint32_t* out, long long* cyc, int steps, float sl2) {
  uint32_t r0[128];
  for (int i = 0; i < 128; ++i) r0[i] = __float_as_uint(in[(threadIdx.x * 7 + i) & 4095]);
  __shared__ uint32_t sink[512 * 17];
  float l = 0.f;
  const float m = 1.5f;
  const uint64_t sl2_2 = f2pack(sl2, sl2), negm2 = f2pack(-m, -m);
  __syncthreads();
  long long t0 = clock64();
  for (int st = 0; st < steps; ++st) {
    uint32_t r[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) r[i] = r0[i] ^ (st & 1);
    uint32_t acc = 0;
    if (V == 0) {        // interleaved per pair: FFMA2, 2 MUFU, FADD2, F2FP
      uint64_t l2[4] = {0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < 128; i += 2) {
        const uint64_t x2 = ffma2(u2pack(r[i], r[i + 1]), sl2_2, negm2);
        const uint64_t p2 = f2pack(ex2(f2lo(x2)), ex2(f2hi(x2)));
        l2[(i >> 1) & 3] = fadd2(l2[(i >> 1) & 3], p2);
        acc ^= pack_bf16(f2lo(p2), f2hi(p2));
      }
      const uint64_t ls = fadd2(fadd2(l2[0], l2[1]), fadd2(l2[2], l2[3]));
      l += f2lo(ls) + f2hi(ls);
    } else if (V == 1) { // scalar FFMA / FADD
      float la[4] = {0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < 128; i += 2) {
        const float p0 = ex2(fmaf(__uint_as_float(r[i]), sl2, -m));
        const float p1 = ex2(fmaf(__uint_as_float(r[i + 1]), sl2, -m));
        la[(i >> 1) & 3] += p0 + p1;
        acc ^= pack_bf16(p0, p1);
      }
      l += (la[0] + la[1]) + (la[2] + la[3]);
    } else if (V == 2) { // MUFU only
#pragma unroll
      for (int i = 0; i < 128; ++i) acc ^= __float_as_uint(ex2(__uint_as_float(r[i])));
    } else if (V == 3) { // everything but MUFU
      uint64_t l2[4] = {0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < 128; i += 2) {
        const uint64_t p2 = ffma2(u2pack(r[i], r[i + 1]), sl2_2, negm2);
        l2[(i >> 1) & 3] = fadd2(l2[(i >> 1) & 3], p2);
        acc ^= pack_bf16(f2lo(p2), f2hi(p2));
      }
      const uint64_t ls = fadd2(fadd2(l2[0], l2[1]), fadd2(l2[2], l2[3]));
      l += f2lo(ls) + f2hi(ls);
    } else if (V == 4) { // V0 but packs stored (16 x st.shared.v4) instead of xor
      uint64_t l2[4] = {0, 0, 0, 0};
      uint32_t pk[64];
#pragma unroll
      for (int i = 0; i < 128; i += 2) {
        const uint64_t x2 = ffma2(u2pack(r[i], r[i + 1]), sl2_2, negm2);
        const uint64_t p2 = f2pack(ex2(f2lo(x2)), ex2(f2hi(x2)));
        l2[(i >> 1) & 3] = fadd2(l2[(i >> 1) & 3], p2);
        pk[i >> 1] = pack_bf16(f2lo(p2), f2hi(p2));
      }
#pragma unroll
      for (int c = 0; c < 16; ++c)
        *reinterpret_cast<uint4*>(&sink[(threadIdx.x * 17 + c) & ~3]) = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      const uint64_t ls = fadd2(fadd2(l2[0], l2[1]), fadd2(l2[2], l2[3]));
      l += f2lo(ls) + f2hi(ls);
    }
    sink[threadIdx.x] ^= acc;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(l) ^ sink[threadIdx.x];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name, int threads, float* in, uint32_t* out, long long* cyc) {
  const int steps = 200;
  probe<V><<<148, threads>>>(in, out, cyc, steps, 0.127f);
  probe<V><<<148, threads>>>(in, out, cyc, steps, 0.127f);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-40s warps/SMSP %d: %6.0f cycles per step (%s)\n", name, threads / 128, (double)c / steps,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* in; uint32_t* out; long long* cyc;
  cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 8);
  float h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = (float)((i * 2654435761u) % 1000) / 100.f - 5.f;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int t : {128, 256}) {
    run<0>("interleaved FFMA2/MUFU/FADD2/F2FP", t, in, out, cyc);
    run<1>("scalar FFMA/MUFU/FADD/F2FP", t, in, out, cyc);
    run<2>("MUFU only (128)", t, in, out, cyc);
    run<3>("no MUFU (FFMA2/FADD2/F2FP)", t, in, out, cyc);
    run<4>("interleaved + st.shared.v4 of P", t, in, out, cyc);
  }
  return 0;
}
