// gemm_sm100.cu -- hand-written tcgen05 + TMA bf16 GEMM for the synthetic
// GPT stage compute, with fused epilogues (K8 bias+GELU,
// residual add, GELU backward, fp32 weight-grad accumulation).
//
//   C[M,N] = sum_k A[m,k] * B[n,k]      (bf16 in, fp32 accumulate in TMEM)
//
// Operand majors are template parameters so the three GEMM families of a
// transformer block map onto the tensor cores without transposes:
//   forward  Y  = X  . W^T   A K-major  (X [T,K]),  B K-major  (W [N,K])
//   dgrad    dX = dY . W     A K-major  (dY [T,N]), B MN-major (W [N,K] read as [K x N])
//   wgrad    dW = dY^T . X   A MN-major (dY [T,N]), B MN-major (X [T,K])
//
// Warp-specialised persistent CTA (256 threads, 1 CTA/SM):
//   warp 0  TMA producer  (4-stage smem ring, mbarrier full/empty)
//   warp 1  MMA issuer    (one thread, tcgen05.mma 128x256x16, accumulators in TMEM)
//   warp 2  TMEM allocator (512 columns = 2 accumulator buffers)
//   warps 4-7 epilogue    (tcgen05.ld -> fused epilogue -> global)
// The epilogue of tile i overlaps the MMAs of tile i+1 (double-buffered TMEM).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <mutex>
#include <utility>

#include "../../include/rrfp_b200.h"
#include "rrfp_common.h"
#include "sm100_ptx.cuh"

namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_STAGE_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_STAGE_BYTES = BN * BK * 2;   // 32 KB
constexpr int SMEM_BYTES = STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + 1024 + 256;
constexpr int TMEM_COLS = 2 * BN;            // two fp32 accumulators of 128 x 256

enum Epi : int {
  EPI_BF16 = 0,        // C = acc (+ bias)                         -> bf16
  EPI_BIAS_GELU = 1,   // C = acc + bias (pre-act), C2 = gelu(C)   -> bf16, bf16
  EPI_RESID = 2,       // C = acc (+ bias) + R                     -> bf16
  EPI_ACC_F32 = 3,     // C (f32) (+)= acc                         -> f32
  EPI_GELU_BWD = 4,    // C = acc * gelu'(R)                       -> bf16;  C2 (optional, f32 [N])
                       //   += column sums of C as stored (the FC1 bias gradient)
  EPI_F32 = 5,         // C = acc                                  -> f32
  EPI_BF16_LSE = 6,    // C = acc (+ bias) -> bf16, and per row and 128-column slot the
                       // online softmax statistics (max, sum exp) of the bf16 values:
                       // float2 C2[row * ldc2 + col / 128] (LM head + cross-entropy)
};

struct GemmArgs {
  int M, N, K;
  int tiles_m, tiles_n;
  void* C;
  long long ldc;
  void* C2;
  long long ldc2;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* R;
  long long ldr;
  int accumulate;
  int vec;   // 1 when C/C2/R rows are 16-byte aligned (vector epilogue path allowed)
  int vec_bias;
  int tma_st;  // pair-kernel epilogue: 0 per-thread stores, 1 smem box + TMA store / reduce-add,
               // 2 smem box + coalesced st.global (bf16 output on a peer GPU: NVLink writes)
  // stream-K tail (pair kernel): tiles [0, sk_full) run data-parallel, one per
  // cluster per round; the sk_W = (tiles - sk_full) * kblocks k-block iterations
  // of the last, partial round are split evenly over all clusters.  A tile split
  // between clusters is finished by its "owner" (the cluster holding its last
  // k-block), which adds the other contributors' fp32 partials from `ws`
  // (one 256 KB slot per cluster) after they signal `cnt`.  sk_W = 0: plain
  // data-parallel persistent schedule.
  int sk_full;
  int sk_W;
  float4* ws;
  int* cnt;
  // half-width tail (pair kernel, data-parallel schedule): after half_rounds full
  // rounds of 256x256 tiles the last half_tail tiles (2*half_tail <= clusters) run
  // as 256x128 halves, one round: the last wave takes half a tile time instead of
  // a full one (256 tiles on 74 pairs: 3.5 tile times instead of 4).  -1: off.
  int half_rounds;
  int half_tail;
  int rpref;   // 1: epilogue loads R one 32-column chunk ahead (env RRFP_GEMM_RPREF, default 1)
};

enum Role : int { ROLE_FULL = 0, ROLE_OWNER = 1, ROLE_PARTIAL = 2 };

struct Unit {
  int tile, k0, k1, role;
  int n0, bn;      // first output column of the unit and its width (256, or 128 for a half tile)
  int tail;        // tail-tile index (counter slot), owner / partial only
  int first;       // owner: first contributing cluster (partials in slots first .. cluster-1)
};

__device__ __forceinline__ long long sk_start(const GemmArgs& g, int c, int C) {
  return (long long)c * g.sk_W / C;
}

// The i-th work unit of cluster `cid` (of C).  Producer, MMA issuer and
// epilogue all walk the same sequence.  Tail order: a cluster's range covers
// at most two tiles (range < one tile); the partial segment of the second tile
// is done FIRST, the owner segment of the first tile LAST, so a partial writer
// never waits on anything and an owner waits only for segments other clusters
// run first.
template <int MC>
__device__ __forceinline__ bool get_unit(const GemmArgs& g, int num_tiles, int kblocks, int cid, int C,
                                         int i, bool direct, Unit& u, int pairi) {
  if (MC == 2) {   // double tiles: (mb, 2*nb2 + pair); odd tiles_n: the last pair's
                   // tile lies past N (zero-filled loads, no stores)
    const int t2 = cid + i * C;
    if (t2 >= g.tiles_m * ((g.tiles_n + 1) >> 1)) return false;
    const int mb = t2 % g.tiles_m, nb = 2 * (t2 / g.tiles_m) + pairi;
    u.tile = mb + nb * g.tiles_m; u.k0 = 0; u.k1 = kblocks; u.role = ROLE_FULL; u.tail = 0; u.first = 0;
    u.n0 = nb * 256; u.bn = 256;
    return true;
  }
  if (!g.sk_W) {
    if (g.half_rounds >= 0 && i >= g.half_rounds) {
      const int h = cid + (i - g.half_rounds) * C;
      if (h >= 2 * g.half_tail) return false;   // (several rounds when every tile runs as halves)
      const int t = g.half_rounds * C + (h >> 1);
      u.tile = t; u.k0 = 0; u.k1 = kblocks; u.role = ROLE_FULL; u.tail = 0; u.first = 0;
      u.n0 = (t / g.tiles_m) * 256 + (h & 1) * 128; u.bn = 128;
      return true;
    }
    const int t = cid + i * C;
    if (t >= num_tiles) return false;
    u.tile = t; u.k0 = 0; u.k1 = kblocks; u.role = ROLE_FULL; u.tail = 0; u.first = 0;
    u.n0 = (t / g.tiles_m) * 256; u.bn = 256;
    return true;
  }
  const int n_dp = g.sk_full / C;
  if (i < n_dp) {
    u.tile = cid + i * C; u.k0 = 0; u.k1 = kblocks; u.role = ROLE_FULL; u.tail = 0; u.first = 0;
    u.n0 = (u.tile / g.tiles_m) * 256; u.bn = 256;
    return true;
  }
  const int j = i - n_dp;
  const long long s = sk_start(g, cid, C), e = sk_start(g, cid + 1, C);
  if (s >= e) return false;
  const int tA = (int)(s / kblocks);
  const bool hasB = e > (long long)(tA + 1) * kblocks;
  int t, k0, k1;
  if (hasB && j == 0) {
    t = tA + 1; k0 = 0; k1 = (int)(e - (long long)(tA + 1) * kblocks);
  } else if (j == (hasB ? 1 : 0)) {
    t = tA; k0 = (int)(s - (long long)tA * kblocks);
    k1 = (int)min((long long)kblocks, e - (long long)tA * kblocks);
  } else {
    return false;
  }
  u.tile = g.sk_full + t; u.k0 = k0; u.k1 = k1; u.tail = t; u.first = cid;
  u.n0 = (u.tile / g.tiles_m) * 256; u.bn = 256;
  if (direct || (k0 == 0 && k1 == kblocks)) {
    u.role = ROLE_FULL;
  } else if (k1 == kblocks) {
    u.role = ROLE_OWNER;
    const long long x = (long long)t * kblocks;   // the tile's first iteration
    int c = (int)(x * C / g.sk_W);
    while (c + 1 < C && sk_start(g, c + 1, C) <= x) ++c;
    while (c > 0 && sk_start(g, c, C) > x) --c;
    u.first = c;
  } else {
    u.role = ROLE_PARTIAL;
  }
  return true;
}

// fp32 partial accumulators: slot (cluster, cta rank) = 128 rows x 256 cols
// laid out so that thread (warp ew, lane) of the writer and of the owner touch
// the same float4s and every warp access is 512 contiguous bytes.
__device__ __forceinline__ float4* ws_chunk(const GemmArgs& g, int slot, int rank, int c32, int ew, int lane) {
  return g.ws + (size_t)(slot * 2 + rank) * 8192 + (size_t)((c32 * 4 + ew) * 8) * 32 + lane;
}
__device__ __forceinline__ void ws_add(const GemmArgs& g, const Unit& u, int cid, int rank, int c32, int ew,
                                       int lane, float (&v)[32]) {
  for (int p = u.first; p < cid; ++p) {
    const float4* q = ws_chunk(g, p, rank, c32, ew, lane);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 a = __ldcg(q + j * 32);
      v[4 * j] += a.x; v[4 * j + 1] += a.y; v[4 * j + 2] += a.z; v[4 * j + 3] += a.w;
    }
  }
}

// MUFU.TANH (rel. error ~2^-11, far below the bf16 output rounding)
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float u = k0 * (x + k1 * x * x * x);
  return 0.5f * x * (1.f + tanh_fast(u));
}
__device__ __forceinline__ float gelu_tanh_grad(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float x2 = x * x;
  float u = k0 * (x + k1 * x2 * x);
  float t = tanh_fast(u);
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x2);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Pull this thread's residual / pre-activation row segment of the next tile
// into L2 before the accumulator is ready (hides the epilogue's load latency).
template <int EPI>
__device__ __forceinline__ void epilogue_prefetch(const GemmArgs& g, int row, int col0, int ncols) {
  if (EPI != EPI_RESID && EPI != EPI_GELU_BWD) return;
  if (row >= g.M) return;
  const char* p = reinterpret_cast<const char*>(g.R + (size_t)row * g.ldr + col0);
  const int bytes = min(ncols, g.N - col0) * 2;
  for (int b = 0; b < bytes; b += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + b));
}

// Fused epilogue math on one 32-column chunk of a row, in registers: bias,
// residual add or GELU' (the f32 epilogues and GELU itself are applied by the
// caller).  Loops have compile-time trip counts with predicated tails.
template <int EPI>
__device__ __forceinline__ void epi_apply(const GemmArgs& g, int row, int col0, float (&v)[32]) {
  if (EPI == EPI_ACC_F32 || EPI == EPI_F32) return;
  if (row >= g.M || col0 >= g.N) return;
  const bool full = g.vec && col0 + 32 <= g.N;
  const int nvalid = g.N - col0;
  if (g.bias && EPI != EPI_GELU_BWD) {
    if (full && g.vec_bias) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 q = __ldg(reinterpret_cast<const uint4*>(g.bias + col0 + j));
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          float2 f = __bfloat1622float2(h[t]);
          v[j + 2 * t] += f.x;
          v[j + 2 * t + 1] += f.y;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) v[j] += __bfloat162float(g.bias[col0 + j]);
    }
  }
  if (EPI == EPI_RESID || EPI == EPI_GELU_BWD) {
    const __nv_bfloat16* rp = g.R + (size_t)row * g.ldr + col0;
    if (full) {
      uint4 q[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) q[j] = *reinterpret_cast<const uint4*>(rp + 8 * j);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q[j]);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 x = __bfloat1622float2(h[t]);
          if (EPI == EPI_RESID) {
            v[8 * j + 2 * t] += x.x;
            v[8 * j + 2 * t + 1] += x.y;
          } else {
            v[8 * j + 2 * t] *= gelu_tanh_grad(x.x);
            v[8 * j + 2 * t + 1] *= gelu_tanh_grad(x.y);
          }
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < nvalid) {
          const float x = __bfloat162float(rp[j]);
          if (EPI == EPI_RESID) v[j] += x;
          else v[j] *= gelu_tanh_grad(x);
        }
      }
    }
  }
}

// Residual / pre-activation operand of one 32-column chunk, loaded ahead of use
// (the epilogue issues chunk c+1's loads before it works on chunk c, so the L2
// latency of R is hidden behind the TMEM read-out and the stores instead of
// being paid once per chunk: on a GEMM with one tile per CTA the whole
// epilogue is exposed).  Rows / columns outside C load zeros.
template <int EPI>
__device__ __forceinline__ void epi_load_r(const GemmArgs& g, int row, int col0, uint4 (&q)[4]) {
  if (EPI != EPI_RESID && EPI != EPI_GELU_BWD) return;
  if (row < g.M && g.vec && col0 + 32 <= g.N) {
    const __nv_bfloat16* rp = g.R + (size_t)row * g.ldr + col0;
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = __ldcg(reinterpret_cast<const uint4*>(rp + 8 * j));
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = make_uint4(0, 0, 0, 0);
  }
}

// epi_apply with the R chunk already in registers (full vector chunks only;
// ragged chunks take epi_apply's scalar path)
template <int EPI>
__device__ __forceinline__ void epi_apply_q(const GemmArgs& g, int row, int col0, float (&v)[32],
                                            const uint4 (&q)[4]) {
  if (EPI != EPI_RESID && EPI != EPI_GELU_BWD) { epi_apply<EPI>(g, row, col0, v); return; }
  if (row >= g.M || col0 >= g.N) return;
  if (!(g.vec && col0 + 32 <= g.N)) { epi_apply<EPI>(g, row, col0, v); return; }
  if (g.bias && EPI != EPI_GELU_BWD) {
    if (g.vec_bias) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 b = __ldg(reinterpret_cast<const uint4*>(g.bias + col0 + j));
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          float2 f = __bfloat1622float2(h[t]);
          v[j + 2 * t] += f.x;
          v[j + 2 * t + 1] += f.y;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += __bfloat162float(g.bias[col0 + j]);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q[j]);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float2 x = __bfloat1622float2(h[t]);
      if (EPI == EPI_RESID) {
        v[8 * j + 2 * t] += x.x;
        v[8 * j + 2 * t + 1] += x.y;
      } else {
        v[8 * j + 2 * t] *= gelu_tanh_grad(x.x);
        v[8 * j + 2 * t + 1] *= gelu_tanh_grad(x.y);
      }
    }
  }
}

// Column sums of a warp's 32 rows x 32 columns (one row per lane, v[c] = column
// c): 31 shuffles (halving exchange); lane l returns the sum of column l.
__device__ __forceinline__ float warp_colsum32(float (&v)[32], int lane) {
#pragma unroll
  for (int k = 16; k >= 1; k >>= 1) {
    const bool upper = lane & k;
#pragma unroll
    for (int i = 0; i < k; ++i) {
      const float send = upper ? v[i] : v[i + k];
      const float keep = upper ? v[i + k] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
    }
  }
  return v[0];
}

// Write one 128-byte row segment (8 x 16 B) of a SWIZZLE_128B staging box:
// chunk j of row `lane` lands at chunk position j ^ (lane % 8), so the 32
// lanes of a warp (32 rows) hit all 32 banks every 8 rows (4 wavefronts / store).
__device__ __forceinline__ void stage_row_sw128(uint8_t* box, int lane, const uint32_t (&w)[32]) {
  uint8_t* rowp = box + lane * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t a = sm100::smem_u32(rowp + ((j ^ (lane & 7)) << 4));
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w[4 * j]), "r"(w[4 * j + 1]),
                 "r"(w[4 * j + 2]), "r"(w[4 * j + 3])
                 : "memory");
  }
}

// Copy a warp's staged SWIZZLE_128B box (32 rows x 128 B) to global memory with
// coalesced 16-byte stores: 8 lanes cover one 128-byte row segment, so each warp
// instruction writes 4 whole row segments (what NVLink peer writes want; the
// per-thread path writes 32 rows x 16 B per instruction).
__device__ __forceinline__ void box_store_coalesced(const uint8_t* box, int lane, char* gbase, long long ld_bytes,
                                                    int rows_valid, int bytes_valid) {
  const int c16 = lane & 7;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = (lane >> 3) + 4 * i;
    if (r < rows_valid && c16 * 16 < bytes_valid) {
      uint4 v;
      const uint32_t a = sm100::smem_u32(box + r * 128 + ((c16 ^ (r & 7)) << 4));
      asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
      *reinterpret_cast<uint4*>(gbase + (long long)r * ld_bytes + c16 * 16) = v;
    }
  }
}

// All loops below have compile-time trip counts (tails are predicated), so the
// 32-wide value arrays stay in registers (no local-memory spill).
template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmArgs& g, int row, int col0,
                                               uint32_t (&r)[32]) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  if (row >= g.M) return;
  const bool full = g.vec && col0 + 32 <= g.N;
  const int nvalid = g.N - col0;   // >= 1
  if (EPI == EPI_ACC_F32 || EPI == EPI_F32) {
    float* c = reinterpret_cast<float*>(g.C) + (size_t)row * g.ldc + col0;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        if (EPI == EPI_ACC_F32 && g.accumulate) {
          // fire-and-forget vector reduction in L2: no load latency in the epilogue
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(c + j), "f"(v[j]),
                       "f"(v[j + 1]), "f"(v[j + 2]), "f"(v[j + 3])
                       : "memory");
        } else {
          *reinterpret_cast<float4*>(c + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) c[j] = (EPI == EPI_ACC_F32 && g.accumulate) ? c[j] + v[j] : v[j];
    }
    return;
  }
  if (g.bias && EPI != EPI_GELU_BWD) {
    if (full && g.vec_bias) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 q = __ldg(reinterpret_cast<const uint4*>(g.bias + col0 + j));
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          float2 f = __bfloat1622float2(h[t]);
          v[j + 2 * t] += f.x;
          v[j + 2 * t + 1] += f.y;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) v[j] += __bfloat162float(g.bias[col0 + j]);
    }
  }
  if (EPI == EPI_RESID || EPI == EPI_GELU_BWD) {
    const __nv_bfloat16* rp = g.R + (size_t)row * g.ldr + col0;
    if (full) {
      uint4 q[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) q[j] = *reinterpret_cast<const uint4*>(rp + 8 * j);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q[j]);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 x = __bfloat1622float2(h[t]);
          if (EPI == EPI_RESID) {
            v[8 * j + 2 * t] += x.x;
            v[8 * j + 2 * t + 1] += x.y;
          } else {
            v[8 * j + 2 * t] *= gelu_tanh_grad(x.x);
            v[8 * j + 2 * t + 1] *= gelu_tanh_grad(x.y);
          }
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < nvalid) {
          const float x = __bfloat162float(rp[j]);
          if (EPI == EPI_RESID) v[j] += x;
          else v[j] *= gelu_tanh_grad(x);
        }
      }
    }
  }
  __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(g.C) + (size_t)row * g.ldc + col0;
  __nv_bfloat16* c2 = EPI == EPI_BIAS_GELU
                          ? reinterpret_cast<__nv_bfloat16*>(g.C2) + (size_t)row * g.ldc2 + col0
                          : nullptr;
  if (full) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint4 o;
      o.x = pack_bf16(v[j], v[j + 1]); o.y = pack_bf16(v[j + 2], v[j + 3]);
      o.z = pack_bf16(v[j + 4], v[j + 5]); o.w = pack_bf16(v[j + 6], v[j + 7]);
      *reinterpret_cast<uint4*>(c + j) = o;
      if (EPI == EPI_BIAS_GELU) {
        uint4 q;
        q.x = pack_bf16(gelu_tanh(v[j]), gelu_tanh(v[j + 1]));
        q.y = pack_bf16(gelu_tanh(v[j + 2]), gelu_tanh(v[j + 3]));
        q.z = pack_bf16(gelu_tanh(v[j + 4]), gelu_tanh(v[j + 5]));
        q.w = pack_bf16(gelu_tanh(v[j + 6]), gelu_tanh(v[j + 7]));
        *reinterpret_cast<uint4*>(c2 + j) = q;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j < nvalid) {
        c[j] = __float2bfloat16(v[j]);
        if (EPI == EPI_BIAS_GELU) c2[j] = __float2bfloat16(gelu_tanh(v[j]));
      }
    }
  }
}

template <int EPI, int A_MN, int B_MN>
__global__ void __launch_bounds__(256, 1)
    gemm_bf16_sm100(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    GemmArgs g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE_BYTES);
  uint64_t* full = bars;                  // [STAGES]
  uint64_t* empty = bars + STAGES;        // [STAGES]
  uint64_t* tfull = bars + 2 * STAGES;    // [2]
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tmA);
    sm100::tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { sm100::mbar_init(&tfull[a], 1); sm100::mbar_init(&tempty[a], 128); }
    sm100::fence_barrier_init();
  }
  if (warp == 2) sm100::tmem_alloc<TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  sm100::griddep_launch();
  sm100::griddep_wait();

  const int num_tiles = g.tiles_m * g.tiles_n;
  const int kblocks = (g.K + BK - 1) / BK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int mb = tile % g.tiles_m, nb = tile / g.tiles_m;
        for (int kb = 0; kb < kblocks; ++kb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          sm100::mbar_arrive_expect_tx(&full[stage], A_STAGE_BYTES + B_STAGE_BYTES);
          uint8_t* a_dst = sA + stage * A_STAGE_BYTES;
          uint8_t* b_dst = sB + stage * B_STAGE_BYTES;
          if (!A_MN) {
            sm100::tma_load_2d(a_dst, &tmA, &full[stage], kb * BK, mb * BM);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              sm100::tma_load_2d(a_dst + j * 64 * BK * 2, &tmA, &full[stage], mb * BM + j * 64, kb * BK);
          }
          if (!B_MN) {
            sm100::tma_load_2d(b_dst, &tmB, &full[stage], kb * BK, nb * BN);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              sm100::tma_load_2d(b_dst + j * 64 * BK * 2, &tmB, &full[stage], nb * BN + j * 64, kb * BK);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = sm100::idesc_bf16(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t a_base = sm100::smem_u32(sA + stage * A_STAGE_BYTES);
          const uint32_t b_base = sm100::smem_u32(sB + stage * B_STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t ad = A_MN ? sm100::umma_desc_sw128(a_base + k * 16 * 128, 64 * BK * 2, 1024)
                               : sm100::umma_desc_sw128(a_base + k * 32, 16, 1024);
            uint64_t bd = B_MN ? sm100::umma_desc_sw128(b_base + k * 16 * 128, 64 * BK * 2, 1024)
                               : sm100::umma_desc_sw128(b_base + k * 32, 16, 1024);
            sm100::mma_bf16(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          sm100::mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        sm100::mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int mb = tile % g.tiles_m, nb = tile / g.tiles_m;
      const int row = mb * BM + ew * 32 + lane;
      epilogue_prefetch<EPI>(g, row, nb * BN, BN);
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        sm100::tmem_ld32(t_row + c, r);
        sm100::tmem_ld_wait();
        if (nb * BN + c < g.N) epilogue_chunk<EPI>(g, row, nb * BN + c, r);
      }
      sm100::tc_fence_before();
      sm100::mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}


// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs computes a 256 x 256
// tile with tcgen05.mma.cta_group::2 (UMMA M = 256).  Each CTA loads its own
// 128 rows of A and 128 rows (half of N) of B, so a CTA moves 32 KB per
// 64-deep k-block instead of 48 KB: 1.5x the arithmetic intensity of the
// 1-CTA 128x256 tile against the L2 (the 1-CTA kernel is L2-bandwidth bound).
// The leader CTA issues the MMAs; TMA completions of both CTAs land on the
// leader's full barrier; MMA commits multicast to both CTAs' empty / tmem-full
// barriers; both epilogues release the leader's tmem-empty barrier.
// k-block depth PBK (64 or 128; same 192 KB of operand ring: 6 or 3 stages).
// A K-major operand stage holds PBK/64 SW128 panels of [128 rows x 64 k]; an
// MN-major one two 64-wide MN panels of [PBK k-rows x 64].
constexpr int P_BM = 256, P_BN = 256;
constexpr int P_RING_BYTES = 6 * 2 * 128 * 64 * 2;   // 192 KB
template <int PBK> struct PairCfg {
  static constexpr int STAGES = 6 * 64 / PBK;
  static constexpr int A_BYTES = 128 * PBK * 2;      // this CTA's 128 rows of A
  static constexpr int B_BYTES = 128 * PBK * 2;      // this CTA's 128 rows (N/2) of B
};
constexpr int P_STAGES = 6;                          // (barrier array size: max stages)
constexpr int P_EPI_BYTES = 4 * 2 * 4096;     // per epilogue warp: two 32-row x 128-byte staging boxes
constexpr int P_SMEM_BYTES = P_RING_BYTES + P_EPI_BYTES + 1024 + 256;
constexpr int P_TMEM_COLS = 2 * P_BN;

// MC = 2: a cluster of two CTA pairs on adjacent N tiles of the same M rows;
// each A k-block is loaded once per cluster (each pair loads one 64-row half and
// multicasts it to the same-rank CTA of the other pair), halving A's L2->SM
// traffic.  Both pairs walk the same unit list (double tiles) in lock step; a
// stage is free once BOTH pairs' MMAs consumed it (empty barriers count 2).
template <int EPI, int A_MN, int B_MN, int PBK, int MC>
__global__ void __cluster_dims__(2 * MC, 1, 1) __launch_bounds__(256, 1)
    gemm_bf16_sm100_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2,
                         const __grid_constant__ CUtensorMap tmBh,   // K-major B, 64-row box (half tiles)
                         const __grid_constant__ CUtensorMap tmAh,   // K-major A, 64-row box (MC = 2)
                         GemmArgs g) {
  constexpr int NST = PairCfg<PBK>::STAGES;
  constexpr int P_A_BYTES = PairCfg<PBK>::A_BYTES, P_B_BYTES = PairCfg<PBK>::B_BYTES;
  constexpr int PANEL = 128 * 64 * 2;   // one SW128 K-major panel of 128 rows
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + NST * P_A_BYTES;
  uint8_t* sEpi = smem + P_RING_BYTES;   // 1024-aligned
  uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + P_EPI_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + P_STAGES;
  uint64_t* tfull = bars + 2 * P_STAGES;
  uint64_t* tempty = bars + 2 * P_STAGES + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * P_STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = sm100::cluster_ctarank();
  const uint32_t rank = crank & 1;              // rank inside the CTA pair
  const uint32_t pairi = crank >> 1;            // which pair of the cluster (MC = 2)
  const uint32_t lead = crank & ~1u;            // this pair's leader CTA
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tmA);
    sm100::tma_prefetch(&tmB);
    for (int s = 0; s < NST; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], MC); }
    for (int a = 0; a < 2; ++a) { sm100::mbar_init(&tfull[a], 1); sm100::mbar_init(&tempty[a], 8); }
    sm100::fence_barrier_init();
  }
  if (warp == 2) sm100::tmem_alloc_pair<P_TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  sm100::griddep_launch();
  sm100::griddep_wait();

  const int num_tiles = g.tiles_m * g.tiles_n;
  const int kblocks = (g.K + PBK - 1) / PBK;
  const int cluster_id = blockIdx.x / (2 * MC), num_clusters = gridDim.x / (2 * MC);
  // f32 accumulate: every split segment reduce-adds into C by itself (no fix-up)
  const bool direct = EPI == EPI_ACC_F32 && g.accumulate && (g.tma_st || g.vec);

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t lead_full0 = sm100::mapa_shared(sm100::smem_u32(&full[0]), lead);
      const uint16_t mask_a = (uint16_t)((1u << rank) | (1u << (rank + 2)));   // same-rank CTAs (MC = 2)
      int stage = 0;
      uint32_t phase = 0;
      Unit u;
      for (int ui = 0; get_unit<MC>(g, num_tiles, kblocks, cluster_id, num_clusters, ui, direct, u, pairi); ++ui) {
        const int mb = u.tile % g.tiles_m;
        // (a half tile still loads 128-row B boxes; the MMA reads the first 64 rows of each)
        const int m0 = mb * P_BM + rank * 128, n0 = u.n0 + rank * (u.bn >> 1);
        const bool half = u.bn != P_BN;   // 64 rows of B per CTA (one 64-wide MN panel)
        for (int kb = u.k0; kb < u.k1; ++kb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          if (leader) sm100::mbar_arrive_expect_tx(&full[stage], 2 * (P_A_BYTES + (half ? P_B_BYTES / 2 : P_B_BYTES)));
          const uint32_t bar = lead_full0 + stage * 8;
          uint8_t* a_dst = sA + stage * P_A_BYTES;
          uint8_t* b_dst = sB + stage * P_B_BYTES;
          if (MC == 2) {   // this CTA's 64-row (K-major) / 64-col (MN-major) half of A, to both pairs
            if (!A_MN) {
#pragma unroll
              for (int h = 0; h < PBK / 64; ++h)
                sm100::tma_load_2d_pair_mc(a_dst + h * PANEL + pairi * 64 * 128, &tmAh, bar, kb * PBK + h * 64,
                                           m0 + pairi * 64, mask_a);
            } else {
              sm100::tma_load_2d_pair_mc(a_dst + pairi * 64 * PBK * 2, &tmA, bar, m0 + pairi * 64, kb * PBK,
                                         mask_a);
            }
          } else if (!A_MN) {
#pragma unroll
            for (int h = 0; h < PBK / 64; ++h)
              sm100::tma_load_2d_pair(a_dst + h * PANEL, &tmA, bar, kb * PBK + h * 64, m0);
          } else {
            sm100::tma_load_2d_pair(a_dst, &tmA, bar, m0, kb * PBK);
            sm100::tma_load_2d_pair(a_dst + 64 * PBK * 2, &tmA, bar, m0 + 64, kb * PBK);
          }
          if (!B_MN) {
#pragma unroll
            for (int h = 0; h < PBK / 64; ++h)   // (a 64-row panel keeps the 128-row panel stride)
              sm100::tma_load_2d_pair(b_dst + h * PANEL, half ? &tmBh : &tmB, bar, kb * PBK + h * 64, n0);
          } else {
            sm100::tma_load_2d_pair(b_dst, &tmB, bar, n0, kb * PBK);
            if (!half) sm100::tma_load_2d_pair(b_dst + 64 * PBK * 2, &tmB, bar, n0 + 64, kb * PBK);
          }
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc_full = sm100::idesc_bf16(P_BM, P_BN, A_MN, B_MN);
      constexpr uint32_t idesc_half = sm100::idesc_bf16(P_BM, P_BN / 2, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      Unit u;
      for (int ui = 0; get_unit<MC>(g, num_tiles, kblocks, cluster_id, num_clusters, ui, direct, u, pairi); ++ui) {
        sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * P_BN;
        const uint32_t idesc = u.bn == P_BN ? idesc_full : idesc_half;
        for (int kb = u.k0; kb < u.k1; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t a_base = sm100::smem_u32(sA + stage * P_A_BYTES);
          const uint32_t b_base = sm100::smem_u32(sB + stage * P_B_BYTES);
#pragma unroll
          for (int k = 0; k < PBK / 16; ++k) {
            const uint32_t kp = (k >> 2) * PANEL + (k & 3) * 32;   // K-major: panel, then 32 B per k16
            uint64_t ad = A_MN ? sm100::umma_desc_sw128(a_base + k * 16 * 128, 64 * PBK * 2, 1024)
                               : sm100::umma_desc_sw128(a_base + kp, 16, 1024);
            uint64_t bd = B_MN ? sm100::umma_desc_sw128(b_base + k * 16 * 128, 64 * PBK * 2, 1024)
                               : sm100::umma_desc_sw128(b_base + kp, 16, 1024);
            sm100::mma_bf16_pair(d_tmem, ad, bd, idesc, (kb != u.k0) || (k != 0));
          }
          sm100::mma_commit_pair(&empty[stage], MC == 2 ? 0xF : 0x3);   // (MC = 2: both pairs' producers)
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
        sm100::mma_commit_pair(&tfull[acc], (uint16_t)(0x3u << lead));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const uint32_t lead_tempty0 = sm100::mapa_shared(sm100::smem_u32(&tempty[0]), lead);
    uint8_t* wbuf = sEpi + ew * 8192;     // this warp's two staging boxes
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t unit = 0;                    // staging-box round robin
    Unit u;
    for (int ui = 0; get_unit<MC>(g, num_tiles, kblocks, cluster_id, num_clusters, ui, direct, u, pairi); ++ui) {
      const int tile = u.tile;
      const int mb = tile % g.tiles_m;
      const int row0 = mb * P_BM + rank * 128 + ew * 32;
      const int row = row0 + lane;
      int* cnt = g.cnt ? g.cnt + u.tail * 8 + rank * 4 + ew : nullptr;
      if (u.role != ROLE_PARTIAL) epilogue_prefetch<EPI>(g, row, u.n0, u.bn);
      uint4 qn[2][4];   // R of the next two 32-column chunks (EPI_RESID / EPI_GELU_BWD, TMA-store path)
      if (g.rpref && g.tma_st && u.role != ROLE_PARTIAL) {
        epi_load_r<EPI>(g, row, u.n0, qn[0]);
        epi_load_r<EPI>(g, row, u.n0 + 32, qn[1]);
      }
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * P_BN;
      if (u.role == ROLE_OWNER) {
        // wait until every other contributor's warp (same rank, same rows) published its partial
        if (lane == 0) {
          const int need = cluster_id - u.first;
          int got;
          do {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(got) : "l"(cnt) : "memory");
          } while (got < need);
        }
        __syncwarp();
      }
      if (u.role == ROLE_PARTIAL) {
        // raw fp32 partial -> this cluster's workspace slot (coalesced), then signal
#pragma unroll 1
        for (int c = 0; c < u.bn; c += 32) {
          uint32_t r[32];
          sm100::tmem_ld32(t_row + c, r);
          sm100::tmem_ld_wait();
          float4* q = ws_chunk(g, cluster_id, rank, c >> 5, ew, lane);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            __stcg(q + j * 32, make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                           __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(cnt) : "memory");
      } else if (!g.tma_st) {
#pragma unroll 1
        for (int c = 0; c < u.bn; c += 32) {
          uint32_t r[32];
          sm100::tmem_ld32(t_row + c, r);
          sm100::tmem_ld_wait();
          if (u.role == ROLE_OWNER) {
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            ws_add(g, u, cluster_id, rank, c >> 5, ew, lane, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(v[j]);
          }
          if (u.n0 + c < g.N) epilogue_chunk<EPI>(g, row, u.n0 + c, r);
        }
      } else if (EPI == EPI_ACC_F32 || EPI == EPI_F32) {
        // 32 f32 columns per box: TMA reduce-add (weight-gradient accumulate) or store
#pragma unroll 1
        for (int c = 0; c < u.bn; c += 32) {
          const int col = u.n0 + c;
          if (col >= g.N) break;
          uint32_t r[32];
          sm100::tmem_ld32(t_row + c, r);
          uint8_t* box = wbuf + (unit & 1) * 4096;
          if (lane == 0) sm100::bulk_wait_read<1>();
          __syncwarp();
          sm100::tmem_ld_wait();
          if (u.role == ROLE_OWNER) {
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            ws_add(g, u, cluster_id, rank, c >> 5, ew, lane, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(v[j]);
          }
          stage_row_sw128(box, lane, r);
          sm100::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (EPI == EPI_ACC_F32 && g.accumulate) sm100::tma_reduce_add_2d(&tmC, box, col, row0);
            else sm100::tma_store_2d(&tmC, box, col, row0);
            sm100::bulk_commit();
          }
          ++unit;
        }
      } else {
        // 64 bf16 columns per box (two TMEM chunks); GELU also stages gelu(C) for C2.
        // R (residual / pre-activation) runs one 32-column chunk ahead in qn[h]
        // (its first chunk was requested before the accumulator wait, below).
        float lse_m = -INFINITY, lse_s = 0.f;   // EPI_BF16_LSE: this row's (max, sum exp) over the unit
#pragma unroll 1
        for (int c = 0; c < u.bn; c += 64) {
          const int col = u.n0 + c;
          if (col >= g.N) break;
          uint32_t w[32];
          uint32_t w2[32];   // gelu(C) (EPI_BIAS_GELU only; dead otherwise)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t r[32];
            sm100::tmem_ld32(t_row + c + 32 * h, r);
            sm100::tmem_ld_wait();
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            if (u.role == ROLE_OWNER) ws_add(g, u, cluster_id, rank, (c >> 5) + h, ew, lane, v);
            if (g.rpref) {
              epi_apply_q<EPI>(g, row, col + 32 * h, v, qn[h]);
              if (c + 64 < u.bn) epi_load_r<EPI>(g, row, col + 64 + 32 * h, qn[h]);
            } else {
              epi_apply<EPI>(g, row, col + 32 * h, v);
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              w[16 * h + j] = pack_bf16(v[2 * j], v[2 * j + 1]);
              if (EPI == EPI_BIAS_GELU) w2[16 * h + j] = pack_bf16(gelu_tanh(v[2 * j]), gelu_tanh(v[2 * j + 1]));
            }
            if (EPI == EPI_GELU_BWD && g.C2) {
              // FC1 bias gradient: column sums of d_pre as stored (bf16), rows past M excluded
              float cv[32];
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[16 * h + j]));
                cv[2 * j] = row < g.M ? f.x : 0.f;
                cv[2 * j + 1] = row < g.M ? f.y : 0.f;
              }
              const float cs = warp_colsum32(cv, lane);
              const int cc = col + 32 * h + lane;
              if (cc < g.N) atomicAdd(reinterpret_cast<float*>(g.C2) + cc, cs);
            }
            if (EPI == EPI_BF16_LSE) {
              // statistics of the values as stored (bf16), columns past N excluded
              const int nv = g.N - (col + 32 * h);
              float xr[32];
              float cm = lse_m;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[16 * h + j]));
                xr[2 * j] = 2 * j < nv ? f.x : -INFINITY;
                xr[2 * j + 1] = 2 * j + 1 < nv ? f.y : -INFINITY;
                cm = fmaxf(cm, fmaxf(xr[2 * j], xr[2 * j + 1]));
              }
              if (cm != -INFINITY) {
                float acc = lse_s * __expf(lse_m - cm);
#pragma unroll
                for (int j = 0; j < 32; ++j) acc += __expf(xr[j] - cm);
                lse_s = acc;
                lse_m = cm;
              }
            }
          }
          uint8_t* box = wbuf + (EPI == EPI_BIAS_GELU ? 0 : (unit & 1) * 4096);
          if (lane == 0) {
            if (EPI == EPI_BIAS_GELU) sm100::bulk_wait_read<0>();
            else sm100::bulk_wait_read<1>();
          }
          __syncwarp();
          stage_row_sw128(box, lane, w);
          if (EPI == EPI_BIAS_GELU) stage_row_sw128(wbuf + 4096, lane, w2);
          sm100::fence_proxy_async_smem();
          __syncwarp();
          if (g.tma_st == 1) {
            if (lane == 0) {
              sm100::tma_store_2d(&tmC, box, col, row0);
              if (EPI == EPI_BIAS_GELU) sm100::tma_store_2d(&tmC2, wbuf + 4096, col, row0);
              sm100::bulk_commit();
            }
          } else {   // peer-GPU destination: coalesced generic stores from the box
            const int rv = min(32, g.M - row0), bv = min(128, (g.N - col) * 2);
            box_store_coalesced(box, lane, reinterpret_cast<char*>(g.C) + ((long long)row0 * g.ldc + col) * 2,
                                g.ldc * 2, rv, bv);
            if (EPI == EPI_BIAS_GELU)
              box_store_coalesced(wbuf + 4096, lane,
                                  reinterpret_cast<char*>(g.C2) + ((long long)row0 * g.ldc2 + col) * 2,
                                  g.ldc2 * 2, rv, bv);
            __syncwarp();
          }
          ++unit;
        }
        if (EPI == EPI_BF16_LSE && row < g.M && u.n0 < g.N) {
          float2* part = reinterpret_cast<float2*>(g.C2) + (size_t)row * g.ldc2 + (u.n0 >> 7);
          part[0] = make_float2(lse_m, lse_s);
          if (u.bn == P_BN) part[1] = make_float2(-INFINITY, 0.f);
        }
      }
      if (u.role == ROLE_OWNER && lane == 0) *cnt = 0;   // ready for the next launch on this stream
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive_remote(lead_tempty0 + acc * 8);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) sm100::bulk_wait<0>();
  }
  sm100::tc_fence_before();
  sm100::cluster_sync();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc_pair<P_TMEM_COLS>(tmem_base);
  }
}

// ------------------------------------------------------------------- host
typedef CUresult (*encode_fn_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

encode_fn_t get_encode() {
  static encode_fn_t fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (encode_fn_t)p;
  }
  return fn;
}

// 2-D bf16 tensor map over a row-major [rows, cols] matrix with leading dim ld
// (elements); box = {box_cols, box_rows}, 128-byte swizzle.
int make_map(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld,
             int box_cols, int box_rows, bool f32 = false) {
  encode_fn_t enc = get_encode();
  if (!enc) return rrfp_fail(RRFP_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return rrfp_fail(RRFP_E_INVALID, "tensor map encode failed (%d): rows=%lld cols=%lld ld=%lld", (int)r,
                     rows, cols, ld);
  return RRFP_OK;
}

int g_num_sms = 0;
int g_reserve_sms = 0;
int g_pair = -1;   // 1: use the CTA-pair kernel (env RRFP_GEMM_PAIR, default on)

int g_tma_store = -1;   // 1: TMA-store epilogue (env RRFP_GEMM_TMA_STORE, default on)

bool use_tma_store() {
  if (g_tma_store < 0) {
    const char* e = getenv("RRFP_GEMM_TMA_STORE");
    g_tma_store = e ? atoi(e) : 1;
  }
  return g_tma_store != 0;
}

int g_pair_bk = -1;   // pair-kernel k-block depth: 64 (6 stages) or 128 (3 stages); env RRFP_GEMM_BK

int pair_bk() {
  if (g_pair_bk < 0) {
    const char* e = getenv("RRFP_GEMM_BK");
    g_pair_bk = (e && atoi(e) == 128) ? 128 : 64;
  }
  return g_pair_bk;
}

bool use_pair() {
  if (g_pair < 0) {
    const char* e = getenv("RRFP_GEMM_PAIR");
    g_pair = e ? atoi(e) : 1;
  }
  return g_pair != 0;
}

// Stream-K workspace, one per (device, stream): kernels on one stream never
// overlap (PDL dependents wait in griddepcontrol.wait before touching it), and
// concurrent branches of a graph were captured from different streams.
struct SkWorkspace {
  float4* ws = nullptr;
  int* cnt = nullptr;
};
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, SkWorkspace> g_ws;
// env RRFP_GEMM_STREAMK (default 0).  Measured on B200 (profiles/r01_gemm_ab.txt):
// the 256x256 pair kernel is bound by L2->SM (TMA) throughput (~11 TB/s of operand
// traffic at 1.8 GHz), not by wave quantization, so idle SMs in the last round cost
// little and the fix-up traffic of the split costs more (-10% on one layer).
int g_tail_split = 1;   // half-width last wave (rrfp_gemm_set_tail_split)
// Shapes whose tiles fill less than one wave of CTA pairs (2048^3: 64 tiles on
// 74 pairs; rrfp_gemm_set_small, env RRFP_GEMM_SMALL, bit mask, default 0 --
// both measured SLOWER than the two-pair multicast clusters on one B200,
// profiles/r02_gemm_small_ab.txt: halves 17.8 -> 25.9 us on the 2048^3 dgrad
// (a 256x128 half reads all of A for half the MMAs: L2 -> SM bound), stream-K
// 18.5 -> 20.8 us on the 2048^3 wgrad (partial-tile reduce-add traffic)):
//   1: f32-accumulate outputs (weight gradients) run stream-K over every pair;
//      each k-segment TMA-reduce-adds its partial tile itself, no fix-up
//   2: other outputs run as 256x128 halves (twice the units: the epilogue of
//      a CTA's first half overlaps the MMAs of its second)
int g_small = -1;
int g_rpref = -1;   // R operand loaded one chunk ahead in the bf16 epilogues (rrfp_gemm_set_rpref)
int small_mode() {
  if (g_small < 0) {
    const char* e = getenv("RRFP_GEMM_SMALL");
    g_small = e ? atoi(e) : 0;
  }
  return g_small;
}
int g_mc = 1;           // 2-pair clusters with A multicast (rrfp_gemm_set_multicast)
int g_streamk = -1;

bool use_streamk() {
  if (g_streamk < 0) {
    const char* e = getenv("RRFP_GEMM_STREAMK");
    g_streamk = e ? atoi(e) : 0;
  }
  return g_streamk != 0;
}

// workspace for `st`, allocated on first (eager) use; never allocates while
// the stream is being captured (returns null -> no stream-K fix-up then)
SkWorkspace* sk_workspace(cudaStream_t st, int clusters) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_ws_mu);
  auto key = std::make_pair(dev, st);
  auto it = g_ws.find(key);
  if (it != g_ws.end()) return &it->second;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
  SkWorkspace w;
  const size_t ws_bytes = (size_t)148 * 128 * 256 * 4;   // one 128x256 f32 slot per CTA (>= clusters * 2)
  const size_t cnt_bytes = (size_t)148 * 8 * sizeof(int);
  (void)clusters;
  if (cudaMalloc(&w.ws, ws_bytes) != cudaSuccess) return nullptr;
  if (cudaMalloc(&w.cnt, cnt_bytes) != cudaSuccess) { cudaFree(w.ws); return nullptr; }
  if (cudaMemset(w.cnt, 0, cnt_bytes) != cudaSuccess) return nullptr;
  cudaDeviceSynchronize();
  return &(g_ws[key] = w);
}

// co-resident clusters of `kern` (cluster of `csize` CTAs, 1 CTA per SM): a
// persistent grid larger than this would run its surplus clusters as a second
// wave.  Clusters are packed per GPC, so this can be below num_SMs / csize.
template <typename K>
int max_clusters(K kern, int csize) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize * 1024);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = P_SMEM_BYTES;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (void*)kern, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

template <int EPI, int A_MN, int B_MN, int PBK>
int launch_pair_mc(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const CUtensorMap& tc2,
                   const CUtensorMap& tbh, const CUtensorMap& tah, GemmArgs g, cudaStream_t st) {
  auto kern = gemm_bf16_sm100_pair<EPI, A_MN, B_MN, PBK, 2>;
  static bool attr = false;
  if (!attr) {
    RRFP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM_BYTES));
    attr = true;
  }
  const int dtiles = g.tiles_m * ((g.tiles_n + 1) / 2);
  static int resident = max_clusters(kern, 4);
  int clusters = (g_num_sms - g_reserve_sms) / 4;
  if (resident > 0 && clusters > resident) clusters = resident;
  if (clusters < 1) clusters = 1;
  g.sk_full = 0; g.sk_W = 0; g.ws = nullptr; g.cnt = nullptr;
  g.half_rounds = -1; g.half_tail = 0;
  const int grid = 4 * (dtiles < clusters ? dtiles : clusters);
  RRFP_CUDA_TRY(rrfp_launch(kern, dim3(grid), dim3(256), P_SMEM_BYTES, st, ta, tb, tc, tc2, tbh, tah, g));
  return RRFP_OK;
}

template <int EPI, int A_MN, int B_MN, int PBK>
int launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const CUtensorMap& tc2,
                const CUtensorMap& tbh, const CUtensorMap& tah,
                GemmArgs g, cudaStream_t st) {
  g.tiles_m = (g.M + P_BM - 1) / P_BM;
  g.tiles_n = (g.N + P_BN - 1) / P_BN;
  // (not under an SM cap: a capped grid shares the GPU, possibly inside a green-context
  // partition, where 4-CTA clusters may not be placeable)
  const bool direct_acc = EPI == EPI_ACC_F32 && g.accumulate && (g.tma_st || g.vec);
  int all_pairs = (g_num_sms - g_reserve_sms) / 2;
  const int tiles0 = g.tiles_m * g.tiles_n;
  const bool small = g_reserve_sms == 0 && tiles0 < all_pairs &&
                     (direct_acc ? (small_mode() & 1) : ((small_mode() & 2) && g_tail_split));
  if (!small && PBK == 64 && g_mc && g_reserve_sms == 0 && g.tiles_n > 1)
    return launch_pair_mc<EPI, A_MN, B_MN, PBK>(ta, tb, tc, tc2, tbh, tah, g, st);
  auto kern = gemm_bf16_sm100_pair<EPI, A_MN, B_MN, PBK, 1>;
  static bool attr = false;
  if (!attr) {
    RRFP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM_BYTES));
    attr = true;
  }
  g.tiles_n = (g.N + P_BN - 1) / P_BN;
  int tiles = g.tiles_m * g.tiles_n;
  static int resident = max_clusters(kern, 2);
  int pairs = (g_num_sms - g_reserve_sms) / 2;
  if (resident > 0 && pairs > resident) pairs = resident;
  if (pairs < 1) pairs = 1;
  const int kblocks = (g.K + PBK - 1) / PBK;
  g.sk_full = 0; g.sk_W = 0; g.ws = nullptr; g.cnt = nullptr;
  g.half_rounds = -1; g.half_tail = 0;
  int grid = 2 * (tiles < pairs ? tiles : pairs);
  const int tail = tiles % pairs;
  if (small && direct_acc) {
    // every k-block of every tile split evenly over all pairs (reduce-add epilogue)
    g.sk_full = 0;
    g.sk_W = tiles * kblocks;
    grid = 2 * pairs;
    RRFP_CUDA_TRY(rrfp_launch(kern, dim3(grid), dim3(256), P_SMEM_BYTES, st, ta, tb, tc, tc2, tbh, tah, g));
    return RRFP_OK;
  }
  if (small) {
    // every tile as two 256x128 halves, rounds of `pairs` halves
    g.half_rounds = 0;
    g.half_tail = tiles;
    grid = 2 * (2 * tiles < pairs ? 2 * tiles : pairs);
    RRFP_CUDA_TRY(rrfp_launch(kern, dim3(grid), dim3(256), P_SMEM_BYTES, st, ta, tb, tc, tc2, tbh, tah, g));
    return RRFP_OK;
  }
  if (g_tail_split && tail != 0 && 2 * tail <= pairs) {
    // last partial wave as 256x128 halves: ceil(tiles / pairs) - 0.5 tile times
    g.half_rounds = tiles / pairs;
    g.half_tail = tail;
    grid = 2 * (g.half_rounds > 0 ? pairs : 2 * tail);
  }
  if (g.half_rounds < 0 && use_streamk() && tail != 0 && (long long)tail * kblocks >= 2LL * pairs) {
    const bool direct = EPI == EPI_ACC_F32 && g.accumulate && (g.tma_st || g.vec);
    SkWorkspace* w = direct ? nullptr : sk_workspace(st, pairs);
    if (direct || w) {
      g.sk_full = tiles - tail;
      g.sk_W = tail * kblocks;
      if (w) { g.ws = w->ws; g.cnt = w->cnt; }
      grid = 2 * pairs;
    }
  }
  RRFP_CUDA_TRY(rrfp_launch(kern, dim3(grid), dim3(256), P_SMEM_BYTES, st, ta, tb, tc, tc2, tbh, tah, g));
  return RRFP_OK;
}

template <int EPI, int A_MN, int B_MN>
int launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, cudaStream_t st) {
  auto kern = gemm_bf16_sm100<EPI, A_MN, B_MN>;
  static bool attr = false;
  if (!attr) {
    RRFP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    attr = true;
  }
  int tiles = g.tiles_m * g.tiles_n;
  int sms = g_num_sms - g_reserve_sms;
  if (sms < 1) sms = 1;
  int grid = tiles < sms ? tiles : sms;
  RRFP_CUDA_TRY(rrfp_launch(kern, dim3(grid), dim3(256), SMEM_BYTES, st, ta, tb, g));
  return RRFP_OK;
}

template <int EPI>
int dispatch_majors(int a_mn, int b_mn, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tbh,
                    const CUtensorMap& tah, const CUtensorMap& tc,
                    const CUtensorMap& tc2, const GemmArgs& g, cudaStream_t st) {
  if (!g_num_sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (use_pair()) {
    if (pair_bk() == 128) {
      if (!a_mn && !b_mn) return launch_pair<EPI, 0, 0, 128>(ta, tb, tc, tc2, tbh, tah, g, st);
      if (!a_mn && b_mn) return launch_pair<EPI, 0, 1, 128>(ta, tb, tc, tc2, tbh, tah, g, st);
      if (a_mn && b_mn) return launch_pair<EPI, 1, 1, 128>(ta, tb, tc, tc2, tbh, tah, g, st);
      return launch_pair<EPI, 1, 0, 128>(ta, tb, tc, tc2, tbh, tah, g, st);
    }
    if (!a_mn && !b_mn) return launch_pair<EPI, 0, 0, 64>(ta, tb, tc, tc2, tbh, tah, g, st);
    if (!a_mn && b_mn) return launch_pair<EPI, 0, 1, 64>(ta, tb, tc, tc2, tbh, tah, g, st);
    if (a_mn && b_mn) return launch_pair<EPI, 1, 1, 64>(ta, tb, tc, tc2, tbh, tah, g, st);
    return launch_pair<EPI, 1, 0, 64>(ta, tb, tc, tc2, tbh, tah, g, st);
  }
  if (!a_mn && !b_mn) return launch<EPI, 0, 0>(ta, tb, g, st);
  if (!a_mn && b_mn) return launch<EPI, 0, 1>(ta, tb, g, st);
  if (a_mn && b_mn) return launch<EPI, 1, 1>(ta, tb, g, st);
  return launch<EPI, 1, 0>(ta, tb, g, st);
}

}  // namespace

// C[M,N] = sum_k A(m,k) B(n,k) with
//   A(m,k) = a_mn ? A[k*lda + m] : A[m*lda + k]
//   B(n,k) = b_mn ? B[k*ldb + n] : B[n*ldb + k]
extern "C" int rrfp_gemm_bf16(int epi, int a_mn, int b_mn, int M, int N, int K, const void* A,
                              long long lda, const void* B, long long ldb, void* C, long long ldc,
                              void* C2, long long ldc2, const void* bias, const void* R,
                              long long ldr, int accumulate, void* stream) {
  if (M <= 0 || N <= 0 || K <= 0 || !A || !B || !C) return rrfp_fail(RRFP_E_INVALID, "bad gemm args");
  if ((lda * 2) % 16 || (ldb * 2) % 16) return rrfp_fail(RRFP_E_INVALID, "leading dims must be 16-byte multiples");
  if (epi == EPI_BIAS_GELU && !C2) return rrfp_fail(RRFP_E_INVALID, "gelu epilogue needs C2");
  if ((epi == EPI_RESID || epi == EPI_GELU_BWD) && !R) return rrfp_fail(RRFP_E_INVALID, "epilogue needs R");
  CUtensorMap ta, tb;
  const int brows = use_pair() ? 128 : BN;   // rows of B per CTA (the pair splits N)
  const int mn_krows = use_pair() ? pair_bk() : BK;   // k-rows per MN-major box
  int rc = a_mn ? make_map(&ta, A, K, M, lda, 64, mn_krows) : make_map(&ta, A, M, K, lda, BK, BM);
  if (rc) return rc;
  rc = b_mn ? make_map(&tb, B, K, N, ldb, 64, mn_krows) : make_map(&tb, B, N, K, ldb, BK, brows);
  if (rc) return rc;
  CUtensorMap tbh = tb;   // K-major B with a 64-row box: each CTA's half of a 256x128 tile
  if (use_pair() && !b_mn && (rc = make_map(&tbh, B, N, K, ldb, BK, 64))) return rc;
  CUtensorMap tah = ta;   // K-major A with a 64-row box: one pair's half of a multicast A slice
  if (use_pair() && g_mc && !a_mn && (rc = make_map(&tah, A, M, K, lda, BK, 64))) return rc;
  GemmArgs g;
  g.M = M; g.N = N; g.K = K;
  g.tiles_m = (M + BM - 1) / BM;
  g.tiles_n = (N + BN - 1) / BN;
  g.C = C; g.ldc = ldc; g.C2 = C2; g.ldc2 = ldc2;
  g.bias = (const __nv_bfloat16*)bias;
  g.R = (const __nv_bfloat16*)R; g.ldr = ldr;
  g.accumulate = accumulate;
  if (g_rpref < 0) {
    const char* e = getenv("RRFP_GEMM_RPREF");
    g_rpref = e ? atoi(e) : 1;
  }
  g.rpref = g_rpref;
  const int esz = (epi == EPI_ACC_F32 || epi == EPI_F32) ? 4 : 2;
  g.vec = ((uintptr_t)C % 16 == 0) && ((ldc * esz) % 16 == 0) &&
          (!C2 || epi == EPI_BF16_LSE || epi == EPI_GELU_BWD ||
           (((uintptr_t)C2 % 16 == 0) && (ldc2 * 2) % 16 == 0)) &&
          (!R || (((uintptr_t)R % 16 == 0) && (ldr * 2) % 16 == 0));
  g.vec_bias = ((uintptr_t)bias % 16) == 0;
  // TMA-store epilogue (pair kernel): C (and C2) must be valid TMA globals
  CUtensorMap tc, tc2;
  memset(&tc, 0, sizeof(tc));
  memset(&tc2, 0, sizeof(tc2));
  g.tma_st = 0;
  // The TMA-store epilogue is used for memory of this device only; a C (or C2)
  // that lives on a peer GPU (a neighbour stage's mailbox over NVLink) takes the
  // per-thread st.global epilogue, the path P2P stores are defined for.
  auto local = [](const void* p) {
    int dev = -1;
    cudaGetDevice(&dev);
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice && a.device == dev;
  };
  const bool f32 = (epi == EPI_ACC_F32 || epi == EPI_F32);
  if (use_pair() && use_tma_store() && g.vec) {
    if (g_tma_store != 2 && local(C) && (!C2 || local(C2))) {
      bool ok = make_map(&tc, C, M, N, ldc, f32 ? 32 : 64, 32, f32) == RRFP_OK;
      if (ok && epi == EPI_BIAS_GELU) ok = make_map(&tc2, C2, M, N, ldc2, 64, 32) == RRFP_OK;
      g.tma_st = ok ? 1 : 0;
    } else if (!f32) {
      g.tma_st = 2;
    }
  }
  if (epi == EPI_GELU_BWD && C2 && !g.tma_st)
    return rrfp_fail(RRFP_E_INVALID, "EPI_GELU_BWD column sums (C2) need the staged (TMA-store) epilogue");
  cudaStream_t st = (cudaStream_t)stream;
  switch (epi) {
    case EPI_BF16: return dispatch_majors<EPI_BF16>(a_mn, b_mn, ta, tb, tbh, tah, tc, tc2, g, st);
    case EPI_BIAS_GELU: return dispatch_majors<EPI_BIAS_GELU>(a_mn, b_mn, ta, tb, tbh, tah, tc, tc2, g, st);
    case EPI_RESID: return dispatch_majors<EPI_RESID>(a_mn, b_mn, ta, tb, tbh, tah, tc, tc2, g, st);
    case EPI_ACC_F32: return dispatch_majors<EPI_ACC_F32>(a_mn, b_mn, ta, tb, tbh, tah, tc, tc2, g, st);
    case EPI_GELU_BWD: return dispatch_majors<EPI_GELU_BWD>(a_mn, b_mn, ta, tb, tbh, tah, tc, tc2, g, st);
    case EPI_F32: return dispatch_majors<EPI_F32>(a_mn, b_mn, ta, tb, tbh, tah, tc, tc2, g, st);
    case EPI_BF16_LSE:
      // pair kernel, TMA-store epilogue, K-major operands only (the LM head forward)
      if (!use_pair() || g.tma_st != 1 || a_mn || b_mn || !C2 || ldc2 < 2 * ((N + 255) / 256))
        return rrfp_fail(RRFP_E_INVALID, "EPI_BF16_LSE needs the pair kernel, a TMA-store C, K-major "
                         "operands and C2 with >= 2 * ceil(N / 256) float2 slots per row");
      if (!g_num_sms) {
        int dev;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
      }
      if (pair_bk() == 128) return launch_pair<EPI_BF16_LSE, 0, 0, 128>(ta, tb, tc, tc2, tbh, tah, g, st);
      return launch_pair<EPI_BF16_LSE, 0, 0, 64>(ta, tb, tc, tc2, tbh, tah, g, st);
  }
  return rrfp_fail(RRFP_E_INVALID, "unknown epilogue %d", epi);
}

// 1 = run the last partial wave of 256x256 tiles as 256x128 halves when they fit
// in one round (default), 0 = plain data-parallel waves
extern "C" int rrfp_gemm_set_tail_split(int on) {
  g_tail_split = on ? 1 : 0;
  return RRFP_OK;
}

// 1 (default) = clusters of two CTA pairs on adjacent N tiles sharing A through
// TMA multicast (N tile count even, no SM cap), 0 = one pair per cluster.
// Measured (profiles/r01_gemm_multicast_ab.txt): one layer's ten GEMMs 518 us vs
// 534 us with pairs (half-width tail) under sustained clocks; only 33 two-pair
// clusters are co-resident (GPC packing), the grid is capped to that.
extern "C" int rrfp_gemm_set_multicast(int on) {
  g_mc = on ? 1 : 0;
  return RRFP_OK;
}

// co-resident clusters of the pair kernel: mc = 1 (CTA pairs) or 2 (two pairs)
extern "C" int rrfp_gemm_max_clusters(int mc) {
  auto k1 = gemm_bf16_sm100_pair<EPI_BF16, 0, 0, 64, 1>;
  auto k2 = gemm_bf16_sm100_pair<EPI_BF16, 0, 0, 64, 2>;
  for (auto k : {(const void*)k1, (const void*)k2})
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM_BYTES) != cudaSuccess)
      return rrfp_fail(RRFP_E_CUDA, "cudaFuncSetAttribute failed");
  return mc == 2 ? max_clusters(k2, 4) : max_clusters(k1, 2);
}

// sub-wave shapes (see g_small): bit 1 stream-K for f32 accumulate, bit 2 half tiles
extern "C" int rrfp_gemm_set_small(int mode) {
  g_small = mode < 0 ? 0 : mode;
  return RRFP_OK;
}

// 1 (default) = residual / pre-activation loads run one 32-column chunk ahead
// in the bf16 epilogues (first chunk before the accumulator wait), 0 = loaded
// where used
extern "C" int rrfp_gemm_set_rpref(int on) {
  g_rpref = on ? 1 : 0;
  return RRFP_OK;
}

// 1 = CTA-pair (cta_group::2) kernel, 0 = single-CTA kernel
extern "C" int rrfp_gemm_set_variant(int pair) {
  g_pair = pair ? 1 : 0;
  return RRFP_OK;
}

// 1 = stream-K split of the last partial round of tiles, 0 = data-parallel only (default)
extern "C" int rrfp_gemm_set_streamk(int on) {
  g_streamk = on ? 1 : 0;
  return RRFP_OK;
}

// 1 = smem-staged TMA store / reduce-add epilogue, 0 = per-thread global stores
extern "C" int rrfp_gemm_set_epilogue(int tma_store) {
  g_tma_store = tma_store < 0 ? 0 : tma_store;
  return RRFP_OK;
}

// pair-kernel k-block depth: 64 (default) or 128
extern "C" int rrfp_gemm_set_bk(int bk) {
  g_pair_bk = bk == 128 ? 128 : 64;
  return RRFP_OK;
}

extern "C" int rrfp_gemm_reserve_sms(int n) {
  g_reserve_sms = n < 0 ? 0 : n;
  return RRFP_OK;
}
