// microbenchmark: cross-entropy forward variants on [2048 x 50304] bf16 logits (dev tool)
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* f) {
  uint4 q = __ldcs(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) { float2 t = __bfloat1622float2(h[i]); f[2 * i] = t.x; f[2 * i + 1] = t.y; }
}
__device__ __forceinline__ void merge(float& m, float& s, float om, float os) {
  const float nm = fmaxf(m, om);
  s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
  m = nm;
}
template <int NT, int U>
__global__ void __launch_bounds__(NT) xent(const __nv_bfloat16* __restrict__ logits, long long ld, int V,
                                            float* __restrict__ lse_out) {
  __shared__ float shm[32], shs[32];
  const __nv_bfloat16* row = logits + (size_t)blockIdx.x * ld;
  float m = -INFINITY, s = 0.f;
  const int stride = NT * 8;
  for (int c0 = threadIdx.x * 8; c0 < V; c0 += U * stride) {
    float f[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + u * stride < V) load8(row + c0 + u * stride, f[u]);
      else for (int j = 0; j < 8; ++j) f[u][j] = -INFINITY;
    float cm = m;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) cm = fmaxf(cm, f[u][j]);
    s *= __expf(m - cm);   // (m = -inf first: 0 * 0)
    if (cm == -INFINITY) s = 0.f;
    m = cm;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) s += __expf(f[u][j] - m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) merge(m, s, __shfl_xor_sync(~0u, m, o), __shfl_xor_sync(~0u, s, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { shm[w] = m; shs[w] = s; }
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < NT / 32 ? shm[threadIdx.x] : -INFINITY;
    s = threadIdx.x < NT / 32 ? shs[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) merge(m, s, __shfl_xor_sync(~0u, m, o), __shfl_xor_sync(~0u, s, o));
    if (threadIdx.x == 0) lse_out[blockIdx.x] = m + __logf(s);
  }
}
template <typename K>
float timeit(K k, int nt, const __nv_bfloat16* x, float* o, int S, int V) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<<<S, nt>>>(x, V, V, o);
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) k<<<S, nt>>>(x, V, V, o);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 20 * 1e3f;
}
int main() {
  const int S = 2048, V = 50304;
  __nv_bfloat16* x; float* o;
  cudaMalloc(&x, (size_t)S * V * 2); cudaMalloc(&o, S * 4);
  cudaMemset(x, 0x3c, (size_t)S * V * 2);
  const double gb = (double)S * V * 2 / 1e3;
  float t;
  t = timeit(xent<512, 1>, 512, x, o, S, V); printf("512 thr, 1 load  : %6.1f us %6.0f GB/s\n", t, gb / t);
  t = timeit(xent<512, 4>, 512, x, o, S, V); printf("512 thr, 4 loads : %6.1f us %6.0f GB/s\n", t, gb / t);
  t = timeit(xent<256, 4>, 256, x, o, S, V); printf("256 thr, 4 loads : %6.1f us %6.0f GB/s\n", t, gb / t);
  t = timeit(xent<1024, 2>, 1024, x, o, S, V); printf("1024 thr, 2 loads: %6.1f us %6.0f GB/s\n", t, gb / t);
  t = timeit(xent<256, 8>, 256, x, o, S, V); printf("256 thr, 8 loads : %6.1f us %6.0f GB/s\n", t, gb / t);
  return 0;
}
