// ops.cu -- HBM-bound stage-compute kernels of the synthetic GPT block
// (SURVEY.md K7 LayerNorm fwd/bwd, K10 softmax cross-entropy, embedding,
// bias-gradient reduction).  bf16 I/O, fp32 statistics and accumulation.
// Each kernel is a single pass over its tensors: one warp per row, 16-byte
// vector loads, per-block partial reductions for parameter gradients.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/rrfp_b200.h"
#include "rrfp_common.h"
#include "sm100_ptx.cuh"

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* f) {
  uint4 q = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float* f) {
  uint4 q;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = q;
}

// ------------------------------------------------------------- LayerNorm
// One CTA per row, D/8 threads (one 16-byte chunk of x / dy / g each): every
// load is issued up front, 8+ CTAs per SM keep enough bytes in flight to run at
// HBM/L2 speed (the previous warp-per-row kernels held a whole row per thread
// group in ~150 registers: one CTA per SM, latency-bound).

// sum of a and b over the CTA (warp shuffles, then one smem exchange)
__device__ __forceinline__ void block_sum2(float& a, float& b, float* sh) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (l == 0) { sh[w] = a; sh[32 + w] = b; }
  __syncthreads();
  float ta = 0.f, tb = 0.f;
  for (int i = 0; i < nw; ++i) { ta += sh[i]; tb += sh[32 + i]; }
  a = ta;
  b = tb;
  __syncthreads();   // sh may be reused by the caller
}

// Forward: one WARP per row (the row in registers, no CTA barrier): measured
// faster than the row-per-CTA form, whose two CTA reductions cost more than
// they save on a 16 MB pass.
// y = (x - mean) * rstd * g + b; one warp per row; D = 256 * NV.
template <int NV>
__global__ void __launch_bounds__(256) ln_fwd_warp_kernel(const __nv_bfloat16* __restrict__ x,
                                                     const __nv_bfloat16* __restrict__ g,
                                                     const __nv_bfloat16* __restrict__ b,
                                                     __nv_bfloat16* __restrict__ y,
                                                     float* __restrict__ mean_out,
                                                     float* __restrict__ rstd_out, int rows,
                                                     float eps) {
  sm100::griddep_launch();
  sm100::griddep_wait();
  constexpr int D = 256 * NV;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const __nv_bfloat16* xr = x + (size_t)warp * D;
  float v[NV][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    load8(xr + (i * 32 + lane) * 8, v[i]);
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[i][j];
  }
  const float mean = warp_sum(s) * (1.f / D);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) { float d = v[i][j] - mean; q += d * d; }
  const float rstd = rsqrtf(warp_sum(q) * (1.f / D) + eps);
  __nv_bfloat16* yr = y + (size_t)warp * D;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * 8;
    float gg[8], bb[8], o[8];
    load8(g + c, gg);
    load8(b + c, bb);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (v[i][j] - mean) * rstd * gg[j] + bb[j];
    store8(yr + c, o);
  }
  if (lane == 0) { mean_out[warp] = mean; rstd_out[warp] = rstd; }
}


// dx = rstd * (dxh - xhat * mean(dxh * xhat) - mean(dxh)) + dres, dxh = dy * g
__global__ void __launch_bounds__(1024) ln_bwd_dx_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
    const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
    const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ dres,
    __nv_bfloat16* __restrict__ dx, int D) {
  __shared__ float sh[64];
  sm100::griddep_launch();
  sm100::griddep_wait();
  const int row = blockIdx.x, c = threadIdx.x * 8;
  const size_t off = (size_t)row * D + c;
  float xv[8], dv[8], gv[8], rv[8];
  load8(x + off, xv);
  load8(dy + off, dv);
  load8(g + c, gv);
  if (dres) load8(dres + off, rv);
  const float mean = mean_in[row], rstd = rstd_in[row];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    xv[j] = (xv[j] - mean) * rstd;   // xhat
    dv[j] *= gv[j];                  // dxh
    s1 += dv[j] * xv[j];
    s2 += dv[j];
  }
  block_sum2(s1, s2, sh);
  s1 *= 1.f / D;
  s2 *= 1.f / D;
  float o[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j] = rstd * (dv[j] - xv[j] * s1 - s2) + (dres ? rv[j] : 0.f);
  store8(dx + off, o);
}

// dg[c] += sum_r dy[r,c] * (x[r,c]-mean[r])*rstd[r];  db[c] += sum_r dy[r,c]
// Block = 8 warps over a slab of rows; each thread owns 8 consecutive columns
// (16-byte loads, a warp covers 256 columns per row); warps reduce via smem,
// then one atomicAdd per column per block.
__global__ void __launch_bounds__(256) ln_param_grad_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
    const float* __restrict__ mean_in, const float* __restrict__ rstd_in, float* __restrict__ dg,
    float* __restrict__ db, int rows, int D, int rows_per_block) {
  sm100::griddep_launch();
  sm100::griddep_wait();
  __shared__ float sg[8][256], sb[8][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * 256 + lane * 8;
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  float ag[8], ab[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { ag[j] = 0.f; ab[j] = 0.f; }
  if (c0 < D) {
#pragma unroll 4
    for (int r = r0 + warp; r < r1; r += 8) {
      float xv[8], dv[8];
      load8(x + (size_t)r * D + c0, xv);
      load8(dy + (size_t)r * D + c0, dv);
      const float m = mean_in[r], rs = rstd_in[r];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        ag[j] += dv[j] * (xv[j] - m) * rs;
        ab[j] += dv[j];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) { sg[warp][lane * 8 + j] = ag[j]; sb[warp][lane * 8 + j] = ab[j]; }
  __syncthreads();
  const int t = threadIdx.x;   // one column of this block's 256
  float tg = 0.f, tb = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) { tg += sg[w][t]; tb += sb[w][t]; }
  const int c = blockIdx.x * 256 + t;
  if (c < D) {
    if (dg) atomicAdd(&dg[c], tg);
    if (db) atomicAdd(&db[c], tb);
  }
}

// Fused LayerNorm backward over a slab of rows per CTA (D/8 threads, 8
// consecutive columns each, G rows in flight per step):
//   dx[r]   = rstd (dxh - xhat mean(dxh xhat) - mean(dxh)) + dres[r],  dxh = dy g
//   dg     += sum_r dy xhat,   db += sum_r dy          (LN parameter gradients)
//   cs_res += sum_r dres[r],   cs_dx += sum_r dx[r]    (bias gradients of the
//             linear layers the residual gradients feed: b_2 from LN2's dres,
//             b_o from LN1's dres)
// One pass over dy / x / dres instead of three kernels (dx, parameter
// gradients, bias-gradient column sums) each re-reading them; the column
// partials stay in registers for the whole slab and leave with one vector
// reduction (red.global.add.v4.f32) per 4 columns per CTA.  dx == NULL: the
// reductions only (dres then only feeds cs_res).
__device__ __forceinline__ void red_add8(float* p, const float* v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
               "f"(v[3]) : "memory");
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p + 4), "f"(v[4]), "f"(v[5]), "f"(v[6]),
               "f"(v[7]) : "memory");
}

__device__ __forceinline__ void unpack8(const uint4& q, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// raw 16-byte loads of one row group (G rows of dy / x / dres + the row statistics):
// kept packed in registers so the NEXT group's loads are in flight while the
// current group is reduced (the block barrier of the row sums would otherwise
// expose the full memory latency once per group)
template <int G>
struct LnGroup {
  uint4 d[G], x[G], r[G];
  float mu[G], rs[G];
};

template <int G>
__device__ __forceinline__ void ln_group_load(LnGroup<G>& q, int rb, int r1, int D, int c,
                                              const __nv_bfloat16* __restrict__ dy,
                                              const __nv_bfloat16* __restrict__ x,
                                              const __nv_bfloat16* __restrict__ dres,
                                              const float* __restrict__ mean_in,
                                              const float* __restrict__ rstd_in, bool want_x) {
#pragma unroll
  for (int i = 0; i < G; ++i) {
    const int r = rb + i;
    const size_t off = (size_t)r * D + c;
    q.d[i] = q.x[i] = q.r[i] = make_uint4(0, 0, 0, 0);   // (bf16 zeros)
    q.mu[i] = 0.f;
    q.rs[i] = 0.f;
    if (r < r1) {
      q.d[i] = *reinterpret_cast<const uint4*>(dy + off);
      if (want_x) {
        q.x[i] = *reinterpret_cast<const uint4*>(x + off);
        q.mu[i] = mean_in[r];
        q.rs[i] = rstd_in[r];
      }
      if (dres) q.r[i] = *reinterpret_cast<const uint4*>(dres + off);
    }
  }
}

template <int G>
__global__ void __launch_bounds__(512, 1) ln_bwd_fused_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
    const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
    const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ dres,
    __nv_bfloat16* __restrict__ dx, float* __restrict__ dg, float* __restrict__ db,
    float* __restrict__ cs_res, float* __restrict__ cs_dx, int rows, int D, int rows_per_cta) {
  __shared__ float sh[2][16][2 * G];   // per-warp row partials, double-buffered by step parity
  sm100::griddep_launch();
  sm100::griddep_wait();
  const int c = threadIdx.x * 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool want_x = dx || dg;
  float gv[8];
  if (dx) load8(g + c, gv);
  float adg[8], adb[8], ares[8], adx[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { adg[j] = 0.f; adb[j] = 0.f; ares[j] = 0.f; adx[j] = 0.f; }
  const int r0 = blockIdx.x * rows_per_cta;
  const int r1 = min(rows, r0 + rows_per_cta);
  if (r0 >= r1) return;
  LnGroup<G> nxt;
  ln_group_load<G>(nxt, r0, r1, D, c, dy, x, dres, mean_in, rstd_in, want_x);
  int parity = 0;
  for (int rb = r0; rb < r1; rb += G, parity ^= 1) {
    const LnGroup<G> cur = nxt;
    if (rb + G < r1) ln_group_load<G>(nxt, rb + G, r1, D, c, dy, x, dres, mean_in, rstd_in, want_x);
    float xv[G][8], dv[G][8], rv[G][8];
    float s[2 * G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      unpack8(cur.d[i], dv[i]);
      unpack8(cur.x[i], xv[i]);
      unpack8(cur.r[i], rv[i]);
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float xh = (xv[i][j] - cur.mu[i]) * cur.rs[i];
        xv[i][j] = xh;
        adg[j] += dv[i][j] * xh;
        adb[j] += dv[i][j];
        ares[j] += rv[i][j];
        if (dx) {
          const float d = dv[i][j] * gv[j];
          dv[i][j] = d;
          s1 += d * xh;
          s2 += d;
        }
      }
      s[2 * i] = s1;
      s[2 * i + 1] = s2;
    }
    if (dx) {
#pragma unroll
      for (int k = 0; k < 2 * G; ++k) s[k] = warp_sum(s[k]);
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 2 * G; ++k) sh[parity][warp][k] = s[k];
      }
      __syncthreads();   // (the other parity buffer is rewritten only after the next barrier)
#pragma unroll
      for (int k = 0; k < 2 * G; ++k) {
        float t = 0.f;
        for (int w = 0; w < nw; ++w) t += sh[parity][w][k];
        s[k] = t * (1.f / D);
      }
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const int r = rb + i;
        if (r >= r1) break;
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          o[j] = cur.rs[i] * (dv[i][j] - xv[i][j] * s[2 * i] - s[2 * i + 1]) + rv[i][j];
          adx[j] += o[j];
        }
        store8(dx + (size_t)r * D + c, o);
      }
    }
  }
  if (dg) red_add8(dg + c, adg);
  if (db) red_add8(db + c, adb);
  if (cs_res) red_add8(cs_res + c, ares);
  if (cs_dx) red_add8(cs_dx + c, adx);
}

// ------------------------------------------------------------- embedding
__global__ void embed_fwd_kernel(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ E,
                                 const __nv_bfloat16* __restrict__ P, __nv_bfloat16* __restrict__ x,
                                 int rows, int D) {
  sm100::griddep_launch();
  sm100::griddep_wait();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= rows) return;
  const __nv_bfloat16* e = E + (size_t)tok[row] * D;
  const __nv_bfloat16* p = P + (size_t)row * D;
  for (int c = lane * 8; c < D; c += 256) {
    float a[8], b[8];
    load8(e + c, a);
    load8(p + c, b);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] += b[j];
    store8(x + (size_t)row * D + c, a);
  }
}

__global__ void embed_bwd_kernel(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ dx,
                                 float* __restrict__ dE, float* __restrict__ dP, int rows, int D) {
  sm100::griddep_launch();
  sm100::griddep_wait();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= rows) return;
  float* e = dE + (size_t)tok[row] * D;
  float* p = dP + (size_t)row * D;
  for (int c = lane * 8; c < D; c += 256) {
    float a[8];
    load8(dx + (size_t)row * D + c, a);
    // token rows collide across positions: vector reductions (2 x 16 B per 8 columns);
    // position rows are this thread's alone: plain 16-byte read-modify-write
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(e + c + 4 * h), "f"(a[4 * h]),
                   "f"(a[4 * h + 1]), "f"(a[4 * h + 2]), "f"(a[4 * h + 3])
                   : "memory");
      float4* q = reinterpret_cast<float4*>(p + c + 4 * h);
      float4 v = *q;
      v.x += a[4 * h]; v.y += a[4 * h + 1]; v.z += a[4 * h + 2]; v.w += a[4 * h + 3];
      *q = v;
    }
  }
}

// ------------------------------------------------------- bias gradients
// db[n] += sum_r dy[r, n]; each thread owns 8 consecutive columns (16-byte
// loads), 8 warps split a slab of rows, smem reduction, 1 atomic / column / block.
__global__ void __launch_bounds__(256) colsum_kernel(const __nv_bfloat16* __restrict__ dy, long long ld,
                                                     float* __restrict__ db, int rows, int cols,
                                                     int rows_per_block) {
  sm100::griddep_launch();
  sm100::griddep_wait();
  __shared__ float sb[8][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * 256 + lane * 8;
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = 0.f;
  if (c0 < cols) {
#pragma unroll 4
    for (int r = r0 + warp; r < r1; r += 8) {
      float v[8];
      load8(dy + (size_t)r * ld + c0, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] += v[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) sb[warp][lane * 8 + j] = a[j];
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) t += sb[w][threadIdx.x];
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c < cols) atomicAdd(&db[c], t);
}

// ------------------------------------------------------- cross entropy
// one 512-thread block per row; loss[r] = lse - logit[target]
__device__ __forceinline__ float block_reduce(float v, bool is_max, float* sh) {
  v = is_max ? warp_max(v) : warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  float t = threadIdx.x < nw ? sh[threadIdx.x] : (is_max ? -INFINITY : 0.f);
  if (w == 0) t = is_max ? warp_max(t) : warp_sum(t);
  if (threadIdx.x == 0) sh[0] = t;
  __syncthreads();
  float r = sh[0];
  __syncthreads();
  return r;
}

// single pass over the row: each thread keeps an online (max, sum-exp) pair,
// rescaled once per group of four 16-byte chunks (all four loads in flight,
// streaming / evict-first: the logits are read once here and once in the
// backward); pairs are merged by warp shuffles, then across the warps.
// 256 threads per row: 49 us for [2048 x 50304] (4.2 TB/s) vs 81 us for the
// per-chunk-rescale 512-thread form (tools/xent_variants.cu).
__device__ __forceinline__ void load8_stream(const __nv_bfloat16* p, float* f) {
  uint4 q = __ldcs(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ void lse_merge(float& m, float& s, float om, float os) {
  const float nm = fmaxf(m, om);
  s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
  m = nm;
}
constexpr int XENT_FWD_THREADS = 256;
__global__ void __launch_bounds__(XENT_FWD_THREADS) xent_fwd_kernel(
    const __nv_bfloat16* __restrict__ logits, long long ld, const int32_t* __restrict__ target, int V,
    float* __restrict__ loss, float* __restrict__ lse_out) {
  sm100::griddep_launch();
  sm100::griddep_wait();
  constexpr int U = 4, NW = XENT_FWD_THREADS / 32;
  __shared__ float shm[NW], shs[NW];
  const __nv_bfloat16* row = logits + (size_t)blockIdx.x * ld;
  float m = -INFINITY, s = 0.f;
  const int stride = XENT_FWD_THREADS * 8;
  for (int c0 = threadIdx.x * 8; c0 < V; c0 += U * stride) {
    float f[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (c0 + u * stride < V) {
        load8_stream(row + c0 + u * stride, f[u]);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[u][j] = -INFINITY;
      }
    }
    float cm = m;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) cm = fmaxf(cm, f[u][j]);
    s = cm == -INFINITY ? 0.f : s * __expf(m - cm);
    m = cm;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) s += __expf(f[u][j] - m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    lse_merge(m, s, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, s, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { shm[w] = m; shs[w] = s; }
  __syncthreads();
  if (w == 0) {
    m = l < NW ? shm[l] : -INFINITY;
    s = l < NW ? shs[l] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      lse_merge(m, s, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, s, o));
    if (l == 0) {
      const float lse = m + __logf(s);
      lse_out[blockIdx.x] = lse;
      loss[blockIdx.x] = lse - __bfloat162float(row[target[blockIdx.x]]);
    }
  }
}

// Cross-entropy forward from the LM-head GEMM's per-slot softmax statistics
// (gemm EPI_BF16_LSE: float2 (max, sum exp) per row and 128-column slot): one
// warp per row merges the slots -> lse, loss = lse - logit[target].  Reads
// 8 B per slot instead of the 206 MB logits pass of xent_fwd_kernel.
__global__ void __launch_bounds__(256) xent_combine_kernel(const float2* __restrict__ part, long long ldp,
                                                           int slots, const __nv_bfloat16* __restrict__ logits,
                                                           long long ld, const int32_t* __restrict__ target,
                                                           int rows, float* __restrict__ loss,
                                                           float* __restrict__ lse_out) {
  sm100::griddep_launch();
  sm100::griddep_wait();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float2* p = part + (size_t)row * ldp;
  float m = -INFINITY, s = 0.f;
  for (int i = lane; i < slots; i += 32) {
    const float2 q = __ldcs(p + i);
    lse_merge(m, s, q.x, q.y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    lse_merge(m, s, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, s, o));
  if (lane == 0) {
    const float l = m + __logf(s);
    lse_out[row] = l;
    loss[row] = l - __bfloat162float(logits[(size_t)row * ld + target[row]]);
  }
}

// dlogits = (softmax - onehot) * scale, written in place
__global__ void __launch_bounds__(512) xent_bwd_kernel(__nv_bfloat16* __restrict__ logits, long long ld,
                                                       const int32_t* __restrict__ target, int V,
                                                       const float* __restrict__ lse_in, float scale) {
  sm100::griddep_launch();
  sm100::griddep_wait();
  __nv_bfloat16* row = logits + (size_t)blockIdx.x * ld;
  const float lse = lse_in[blockIdx.x];
  const int t = target[blockIdx.x];
  for (int c = threadIdx.x * 8; c < V; c += blockDim.x * 8) {
    float f[8];
    load8(row + c, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = (__expf(f[j] - lse) - (c + j == t ? 1.f : 0.f)) * scale;
    store8(row + c, f);
  }
}

// strided 2-D copy, 16-byte vectors: dst[r, :w] = src[r, :w]   (w in bytes)
__global__ void copy_rows_kernel(char* __restrict__ dst, long long ldd, const char* __restrict__ src,
                                 long long lds, int rows, int w16) {
  sm100::griddep_launch();
  sm100::griddep_wait();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n = (long long)rows * w16;
  for (long long k = i; k < n; k += (long long)gridDim.x * blockDim.x) {
    const long long r = k / w16, c = k % w16;
    *reinterpret_cast<uint4*>(dst + r * ldd + c * 16) =
        __ldg(reinterpret_cast<const uint4*>(src + r * lds + c * 16));
  }
}

}  // namespace

// LayerNorm widths: multiples of 256 up to 8192 (D/8 threads per row-CTA)
static int ln_width_ok(int D) {
  if (D < 256 || D > 8192 || D % 256)
    return rrfp_fail(RRFP_E_INVALID, "LayerNorm width %d unsupported (multiple of 256, <= 8192)", D);
  return RRFP_OK;
}

extern "C" int rrfp_layernorm_fwd(const void* x, const void* g, const void* b, void* y, float* mean,
                                  float* rstd, int rows, int D, float eps, void* stream) {
  if (int rc = ln_width_ok(D)) return rc;
  if (rows <= 0) return RRFP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 grid((rows + 7) / 8), block(256);
  const __nv_bfloat16 *xx = (const __nv_bfloat16*)x, *gg = (const __nv_bfloat16*)g, *bb = (const __nv_bfloat16*)b;
  __nv_bfloat16* yy = (__nv_bfloat16*)y;
  switch (D / 256) {
    case 1: RRFP_CUDA_TRY(rrfp_launch(ln_fwd_warp_kernel<1>, grid, block, 0, st, xx, gg, bb, yy, mean, rstd, rows, eps)); break;
    case 2: RRFP_CUDA_TRY(rrfp_launch(ln_fwd_warp_kernel<2>, grid, block, 0, st, xx, gg, bb, yy, mean, rstd, rows, eps)); break;
    case 3: RRFP_CUDA_TRY(rrfp_launch(ln_fwd_warp_kernel<3>, grid, block, 0, st, xx, gg, bb, yy, mean, rstd, rows, eps)); break;
    case 4: RRFP_CUDA_TRY(rrfp_launch(ln_fwd_warp_kernel<4>, grid, block, 0, st, xx, gg, bb, yy, mean, rstd, rows, eps)); break;
    case 5: RRFP_CUDA_TRY(rrfp_launch(ln_fwd_warp_kernel<5>, grid, block, 0, st, xx, gg, bb, yy, mean, rstd, rows, eps)); break;
    case 6: RRFP_CUDA_TRY(rrfp_launch(ln_fwd_warp_kernel<6>, grid, block, 0, st, xx, gg, bb, yy, mean, rstd, rows, eps)); break;
    case 8: RRFP_CUDA_TRY(rrfp_launch(ln_fwd_warp_kernel<8>, grid, block, 0, st, xx, gg, bb, yy, mean, rstd, rows, eps)); break;
    case 16: RRFP_CUDA_TRY(rrfp_launch(ln_fwd_warp_kernel<16>, grid, block, 0, st, xx, gg, bb, yy, mean, rstd, rows, eps)); break;
    default: return rrfp_fail(RRFP_E_INVALID, "LayerNorm width %d unsupported", D);
  }
  RRFP_CUDA_TRY(cudaGetLastError());
  return RRFP_OK;
}

extern "C" int rrfp_layernorm_bwd(const void* dy, const void* x, const float* mean, const float* rstd,
                                  const void* g, const void* dres, void* dx, float* dg, float* db,
                                  int rows, int D, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (int rc = ln_width_ok(D)) return rc;
  if (rows <= 0) return RRFP_OK;
  if (dx) {   // dx == NULL: parameter gradients only (e.g. on a side stream)
    RRFP_CUDA_TRY(rrfp_launch(ln_bwd_dx_kernel, dim3(rows), dim3(D / 8), 0, st, (const __nv_bfloat16*)dy,
                              (const __nv_bfloat16*)x, mean, rstd, (const __nv_bfloat16*)g,
                              (const __nv_bfloat16*)dres, (__nv_bfloat16*)dx, D));
    RRFP_CUDA_TRY(cudaGetLastError());
  }
  if (dg || db) {
    const int rpb = 32;   // 2 rows per warp (unrolled): enough CTAs in flight per SM (64 / 128: slower)
    dim3 g2((D + 255) / 256, (rows + rpb - 1) / rpb);
    RRFP_CUDA_TRY(rrfp_launch(ln_param_grad_kernel, g2, dim3(256), 0, st, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, mean,
                                             rstd, dg, db, rows, D, rpb));
    RRFP_CUDA_TRY(cudaGetLastError());
  }
  return RRFP_OK;
}

// Fused LayerNorm backward (ln_bwd_fused_kernel): any of dx / dg / db / cs_res /
// cs_dx may be NULL; the fp32 outputs are accumulated (+=).  Slabs of rows sized
// so two CTAs per SM cover the rows in one wave.
extern "C" int rrfp_layernorm_bwd_fused(const void* dy, const void* x, const float* mean, const float* rstd,
                                        const void* g, const void* dres, void* dx, float* dg, float* db,
                                        float* cs_res, float* cs_dx, int rows, int D, void* stream) {
  if (int rc = ln_width_ok(D)) return rc;
  if (D > 4096) return rrfp_fail(RRFP_E_INVALID, "layernorm_bwd_fused: width %d > 4096", D);
  if (rows <= 0) return RRFP_OK;
  if (dx && !g) return rrfp_fail(RRFP_E_INVALID, "layernorm_bwd_fused: dx needs gamma");
  if ((dx || dg) && (!x || !mean || !rstd)) return rrfp_fail(RRFP_E_INVALID, "layernorm_bwd_fused: needs x/mean/rstd");
  if (cs_res && !dres) return rrfp_fail(RRFP_E_INVALID, "layernorm_bwd_fused: cs_res needs dres");
  if (!dx && cs_dx) return rrfp_fail(RRFP_E_INVALID, "layernorm_bwd_fused: cs_dx needs dx");
  constexpr int G = 2;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int per_sm = D <= 2048 ? 2 : 1;
  int rpc = (rows + per_sm * sms - 1) / (per_sm * sms);
  // reductions only (no dx, no per-row barrier): taller slabs, fewer column partials
  // to reduce-add (env RRFP_LN_RPC_MUL, default 2)
  static int mul = -1;
  if (mul < 0) {
    const char* e = getenv("RRFP_LN_RPC_MUL");
    mul = e ? atoi(e) : 2;
    if (mul < 1) mul = 1;
  }
  if (!dx) rpc *= mul;
  rpc = (rpc + G - 1) / G * G;
  const int grid = (rows + rpc - 1) / rpc;
  RRFP_CUDA_TRY(rrfp_launch(ln_bwd_fused_kernel<G>, dim3(grid), dim3(D / 8), 0, (cudaStream_t)stream,
                            (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, mean, rstd,
                            (const __nv_bfloat16*)g, (const __nv_bfloat16*)dres, (__nv_bfloat16*)dx, dg, db,
                            cs_res, cs_dx, rows, D, rpc));
  RRFP_CUDA_TRY(cudaGetLastError());
  return RRFP_OK;
}

extern "C" int rrfp_embedding_fwd(const int32_t* tok, const void* E, const void* P, void* x, int rows,
                                  int D, void* stream) {
  if (D % 8) return rrfp_fail(RRFP_E_INVALID, "embedding width must be a multiple of 8");
  RRFP_CUDA_TRY(rrfp_launch(embed_fwd_kernel, dim3((rows + 7) / 8), dim3(256), 0, (cudaStream_t)stream, tok, (const __nv_bfloat16*)E, (const __nv_bfloat16*)P, (__nv_bfloat16*)x, rows, D));
  RRFP_CUDA_TRY(cudaGetLastError());
  return RRFP_OK;
}

extern "C" int rrfp_embedding_bwd(const int32_t* tok, const void* dx, float* dE, float* dP, int rows,
                                  int D, void* stream) {
  if (D % 8) return rrfp_fail(RRFP_E_INVALID, "embedding width must be a multiple of 8");
  RRFP_CUDA_TRY(rrfp_launch(embed_bwd_kernel, dim3((rows + 7) / 8), dim3(256), 0, (cudaStream_t)stream, tok, (const __nv_bfloat16*)dx, dE, dP, rows, D));
  RRFP_CUDA_TRY(cudaGetLastError());
  return RRFP_OK;
}

extern "C" int rrfp_bias_grad(const void* dy, long long ld, float* db, int rows, int cols, void* stream) {
  if (cols % 8 || ld % 8) return rrfp_fail(RRFP_E_INVALID, "bias grad needs cols, ld multiples of 8");
  const int rpb = 64;
  dim3 grid((cols + 255) / 256, (rows + rpb - 1) / rpb);
  RRFP_CUDA_TRY(rrfp_launch(colsum_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream, (const __nv_bfloat16*)dy, ld, db, rows, cols, rpb));
  RRFP_CUDA_TRY(cudaGetLastError());
  return RRFP_OK;
}

extern "C" int rrfp_xent_combine(const void* part, long long ldp, int slots, const void* logits, long long ld,
                                 const int32_t* target, int rows, float* loss, float* lse, void* stream) {
  if (slots <= 0 || ldp < slots) return rrfp_fail(RRFP_E_INVALID, "xent_combine: bad slot count");
  if (rows <= 0) return RRFP_OK;
  RRFP_CUDA_TRY(rrfp_launch(xent_combine_kernel, dim3((rows + 7) / 8), dim3(256), 0, (cudaStream_t)stream,
                            (const float2*)part, ldp, slots, (const __nv_bfloat16*)logits, ld, target, rows, loss,
                            lse));
  RRFP_CUDA_TRY(cudaGetLastError());
  return RRFP_OK;
}

extern "C" int rrfp_xent_fwd(const void* logits, long long ld, const int32_t* target, int rows, int V,
                             float* loss, float* lse, void* stream) {
  if (V % 8 || ld % 8) return rrfp_fail(RRFP_E_INVALID, "vocab / ld must be multiples of 8");
  RRFP_CUDA_TRY(rrfp_launch(xent_fwd_kernel, dim3(rows), dim3(XENT_FWD_THREADS), 0, (cudaStream_t)stream, (const __nv_bfloat16*)logits, ld, target, V,
                                                          loss, lse));
  RRFP_CUDA_TRY(cudaGetLastError());
  return RRFP_OK;
}

extern "C" int rrfp_xent_bwd(void* logits, long long ld, const int32_t* target, int rows, int V,
                             const float* lse, float scale, void* stream) {
  if (V % 8 || ld % 8) return rrfp_fail(RRFP_E_INVALID, "vocab / ld must be multiples of 8");
  RRFP_CUDA_TRY(rrfp_launch(xent_bwd_kernel, dim3(rows), dim3(512), 0, (cudaStream_t)stream, (__nv_bfloat16*)logits, ld, target, V, lse,
                                                          scale));
  RRFP_CUDA_TRY(cudaGetLastError());
  return RRFP_OK;
}

extern "C" int rrfp_copy_rows(void* dst, long long ldd_bytes, const void* src, long long lds_bytes,
                              int rows, long long width_bytes, void* stream) {
  if (width_bytes % 16 || ldd_bytes % 16 || lds_bytes % 16 || (uintptr_t)dst % 16 || (uintptr_t)src % 16)
    return rrfp_fail(RRFP_E_INVALID, "copy_rows needs 16-byte aligned rows");
  const int w16 = (int)(width_bytes / 16);
  long long n = (long long)rows * w16;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  RRFP_CUDA_TRY(rrfp_launch(copy_rows_kernel, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, (char*)dst, ldd_bytes, (const char*)src,
                                                              lds_bytes, rows, w16));
  RRFP_CUDA_TRY(cudaGetLastError());
  return RRFP_OK;
}
