// Cycles per softmax step of the attention forward (one 128-wide S row per
// thread, one warp per SM sub-partition), isolated from TMEM and the MMAs:
// max, x = s*c - m (FFMA2), 2^x (MUFU / FMA-pipe polynomial), row sum (FADD2),
// bf16 pack.  Variants: POLY = bit mask over pair index mod 8 of the pairs
// emulated on the FMA pipe; WARPS = warps per SM sharing the work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/probe_softmax tools/probe_softmax.cu
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
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t x2) {
  const float a = fmaxf(f2lo(x2), -127.f), b = fmaxf(f2hi(x2), -127.f);
  const uint64_t x = f2pack(a, b);
  const uint64_t t = fadd2(x, f2pack(12582912.f, 12582912.f));
  const uint64_t jn = fadd2(t, f2pack(-12582912.f, -12582912.f));
  const uint64_t f = ffma2(jn, f2pack(-1.f, -1.f), x);
  uint64_t p = ffma2(f2pack(0.05500882f, 0.05500882f), f, f2pack(0.24221077f, 0.24221077f));
  p = ffma2(p, f, f2pack(0.69328291f, 0.69328291f));
  p = ffma2(p, f, f2pack(1.f, 1.f));
  const uint32_t lo = (uint32_t)t * 8388608u + (uint32_t)p;
  const uint32_t hi = (uint32_t)(t >> 32) * 8388608u + (uint32_t)(p >> 32);
  return u2pack(lo, hi);
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <uint32_t POLY, int COLS>
__global__ void __launch_bounds__(512, 1) probe(const float* in, uint32_t* out, long long* cyc, int steps, float sl2) {
  uint32_t r0[COLS];
  for (int i = 0; i < COLS; ++i) r0[i] = __float_as_uint(in[(threadIdx.x * 7 + i) & 4095]);
  __shared__ uint32_t sink[512 * 4];
  float l = 0.f, m_used = -1e30f;
  const uint64_t sl2_2 = f2pack(sl2, sl2);
  __syncthreads();
  long long t0 = clock64();
  for (int st = 0; st < steps; ++st) {
    uint32_t r[COLS];
#pragma unroll
    for (int i = 0; i < COLS; ++i) r[i] = r0[i] ^ (st & 1);   // fresh "S" each step
    float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int i = 0; i < COLS; i += 2)
      mx4[(i >> 1) & 3] = fmaxf(mx4[(i >> 1) & 3], fmaxf(__uint_as_float(r[i]), __uint_as_float(r[i + 1])));
    const float m_new = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * sl2;
    if (m_new > m_used + 8.f) m_used = m_new;
    const uint64_t negm2 = f2pack(-m_used, -m_used);
#pragma unroll
    for (int i = 0; i < COLS; i += 2) {
      const uint64_t x2 = ffma2(u2pack(r[i], r[i + 1]), sl2_2, negm2);
      r[i] = (uint32_t)x2; r[i + 1] = (uint32_t)(x2 >> 32);
    }
#pragma unroll
    for (int i = 0; i < COLS; i += 2) {
      if ((POLY >> ((i >> 1) & 7)) & 1) {
        const uint64_t p2 = ex2_poly2(u2pack(r[i], r[i + 1]));
        r[i] = (uint32_t)p2; r[i + 1] = (uint32_t)(p2 >> 32);
      } else {
        r[i] = __float_as_uint(ex2(__uint_as_float(r[i])));
        r[i + 1] = __float_as_uint(ex2(__uint_as_float(r[i + 1])));
      }
    }
    uint64_t l2[4] = {0, 0, 0, 0};
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < COLS; i += 2) {
      const uint64_t p2 = u2pack(r[i], r[i + 1]);
      l2[(i >> 1) & 3] = fadd2(l2[(i >> 1) & 3], p2);
      acc ^= pack_bf16(f2lo(p2), f2hi(p2));
    }
    const uint64_t ls = fadd2(fadd2(l2[0], l2[1]), fadd2(l2[2], l2[3]));
    l += f2lo(ls) + f2hi(ls);
    sink[threadIdx.x] = acc;   // stands in for the tcgen05.st of P
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(l) ^ sink[threadIdx.x];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <uint32_t POLY, int COLS>
void run(const char* name, int threads, float* in, uint32_t* out, long long* cyc) {
  const int steps = 200;
  probe<POLY, COLS><<<148, threads>>>(in, out, cyc, steps, 0.127f);
  probe<POLY, COLS><<<148, threads>>>(in, out, cyc, steps, 0.127f);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  // rows per SM-step: threads; elements = threads * COLS; report cycles per 128x128 tile
  const double tiles = (double)threads * COLS / (128.0 * 128.0);
  printf("%-28s threads %3d cols %3d: %7.0f cycles/step  = %6.0f cycles per 128x128 tile   %s\n", name, threads,
         COLS, (double)c / steps, (double)c / steps / tiles, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* in; uint32_t* out; long long* cyc;
  cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 8);
  float h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = (float)((i * 2654435761u) % 1000) / 100.f - 5.f;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  run<0x00, 128>("no poly", 128, in, out, cyc);
  run<0x80, 128>("poly 1/8", 128, in, out, cyc);
  run<0x88, 128>("poly 2/8", 128, in, out, cyc);
  run<0xA4, 128>("poly 3/8", 128, in, out, cyc);
  run<0xAA, 128>("poly 4/8", 128, in, out, cyc);
  run<0x00, 128>("no poly", 256, in, out, cyc);
  run<0x88, 128>("poly 2/8", 256, in, out, cyc);
  run<0xA4, 128>("poly 3/8", 256, in, out, cyc);
  run<0x00, 64>("no poly", 256, in, out, cyc);
  run<0x88, 64>("poly 2/8", 256, in, out, cyc);
  run<0xA4, 64>("poly 3/8", 256, in, out, cyc);
  run<0xA4, 64>("poly 3/8", 512, in, out, cyc);
  return 0;
}
