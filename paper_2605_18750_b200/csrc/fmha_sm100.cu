// fmha_sm100.cu -- the attention core of the GPT stage bodies,
// hand-written for sm_100a: tcgen05.mma with TMEM accumulators, TMA-fed
// shared-memory operands, d_head = 128, causal or bidirectional, reading Q/K/V
// straight out of the packed QKV GEMM output [T, 3*D] and writing O [T, D] and
// the packed dQKV [T, 3*D] (no layout copies).  It fills the compute slot the
// reference times as a no-op (engine.py:272-273) / a spin (live.py:388-390).
//
// Forward (one CTA per (head, pair of 128-row query tiles)):
//   warp 0      TMA producer: both Q tiles once, then K_j / V_j tiles through a
//               4-stage ring of 32 KB tiles (two SW128 panels of 128 x 64)
//   warp 1      MMA issuer (one thread):  S = Q K^T  (SS, 128x128x128) into a
//               TMEM S buffer;  O += P V  (TS: P read from TMEM, V from smem)
//   warp 2      TMEM allocator (512 columns: S buffers 0/1, O0, O1)
//   warps 4-7   softmax of query tile 0, warps 8-11 softmax of query tile 1
//               (one thread per query row; P written back over its S columns
//               as packed bf16 with tcgen05.st, the A operand of the PV MMA)
// The two tiles ping-pong on the tensor core: issue order QK0_j, PV1_{j-1},
// QK1_j, PV0_j, so each softmax has a full QK+PV of the other tile to hide
// behind.  Causal pairs are (u, n_qt-1-u): every CTA has n_qt+1 tile steps.
// Once the short tile is done, the long one alternates between both S buffers
// (QK_{j+1} is issued before PV_j) so its softmax still overlaps the MMAs.
// Row max uses a lazy rescale: O and l are rescaled only when the running max
// grows by more than 8 (log2 units), so P <= 256 and the O correction (a TMEM
// read-modify-write) happens on the first tiles only.
// Statistics: lse[h][t] = logsumexp of the scaled scores of row t (natural log,
// the softmax-stats layout cuDNN's SDPA backward also reads).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/rrfp_b200.h"
#include "rrfp_common.h"
#include "sm100_ptx.cuh"

namespace {

constexpr int FT = 128;                      // query / key tile rows
constexpr int DH = 128;                      // head dimension
constexpr int PANEL = FT * 128;              // 16 KB: 128 rows x 64 bf16 (one SW128 panel)
constexpr int TILE = 2 * PANEL;              // 32 KB: 128 rows x 128 bf16
constexpr int F_RING = 4;
constexpr int F_SMEM = (2 + F_RING) * TILE + 1024 + 256;
constexpr int F_THREADS = 384;

struct FwdArgs {
  int T, H, D, n_qt, causal;
  float sl2;                   // softmax scale * log2(e)
  __nv_bfloat16* o;
  long long ldo;
  float* lse;
  long long lse_ld;
  int experiment;    // test hook: 1 = P from a copy instead of exp (pipeline-bound time)
  long long* dbg;    // optional event log of one CTA: [4][512] (code<<56 | j<<40 | clock)
  int dbg_cta;
};

// mbarrier wait that traps after ~4 s instead of hanging the device.  Plain
// try_wait (no suspend-time hint): a hinted wait parks the thread in
// NANOSLEEP.SYNCS and the hand-offs between the roles pick up its wake-up latency.
__device__ __forceinline__ uint32_t try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
  return ok;
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = sm100::smem_u32(bar);
  if (try_wait(addr, parity)) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    if (try_wait(addr, parity)) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 4000000000ull) __trap();
  }
}

// whole-warp callers: one elected lane issues the op
__device__ __forceinline__ void mma_ss_e(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_ts_e(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// N = 4 or 8 SS MMAs of one product (K = 16 N) in ONE asm block: one elect, the
// descriptor bases moved to uniform registers once, per-k offsets as immediates
// ((k / 4) * P + (k % 4) * S, in 16-byte units).  mma_ss_e per instruction costs
// ~11 SASS (R2UR / ELECT / VOTEU per MMA): ~50 issue cycles each in the backward.
template <int SA, int PA, int SB, int PB>
__device__ __forceinline__ void mma_ss_x8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, q, e;\n"
      ".reg .b64 ra, rb;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "setp.eq.u32 q, 0, 0;\n"
      "add.s64 ra, %1, %5;  add.s64 rb, %2, %13;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, p;\n"
      "add.s64 ra, %1, %6;  add.s64 rb, %2, %14;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, q;\n"
      "add.s64 ra, %1, %7;  add.s64 rb, %2, %15;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, q;\n"
      "add.s64 ra, %1, %8;  add.s64 rb, %2, %16;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, q;\n"
      "add.s64 ra, %1, %9;  add.s64 rb, %2, %17;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, q;\n"
      "add.s64 ra, %1, %10; add.s64 rb, %2, %18;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, q;\n"
      "add.s64 ra, %1, %11; add.s64 rb, %2, %19;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, q;\n"
      "add.s64 ra, %1, %12; add.s64 rb, %2, %20;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, q;\n"
      "}\n" ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate),
      "n"(0), "n"(SA), "n"(2 * SA), "n"(3 * SA), "n"(PA), "n"(PA + SA), "n"(PA + 2 * SA), "n"(PA + 3 * SA),
      "n"(0), "n"(SB), "n"(2 * SB), "n"(3 * SB), "n"(PB), "n"(PB + SB), "n"(PB + 2 * SB), "n"(PB + 3 * SB));
}
template <int SA, int SB>
__device__ __forceinline__ void mma_ss_x4(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, q, e;\n"
      ".reg .b64 ra, rb;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "setp.eq.u32 q, 0, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "add.s64 ra, %1, %5;  add.s64 rb, %2, %8;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, q;\n"
      "add.s64 ra, %1, %6;  add.s64 rb, %2, %9;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, q;\n"
      "add.s64 ra, %1, %7;  add.s64 rb, %2, %10;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, q;\n"
      "}\n" ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate),
      "n"(SA), "n"(2 * SA), "n"(3 * SA), "n"(SB), "n"(2 * SB), "n"(3 * SB));
}

__device__ __forceinline__ void commit_e(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(sm100::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA pipe for 3 of every 8 exponential pairs of the softmax (the
// MUFU unit, 16 results / clock / SM, bounds it otherwise): x = j + f,
// j = rint(x), 2^f by a degree-3 minimax polynomial on [-0.5, 0.5] (max rel.
// error 1.0e-4, far below the bf16 rounding of P), 2^j added into the exponent.
// packed fp32x2 arithmetic (FFMA2 / FADD2 on sm_100): half the issue slots
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ uint64_t u2pack(uint32_t lo, uint32_t hi) { return (uint64_t)lo | ((uint64_t)hi << 32); }
__device__ __forceinline__ float f2lo(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2hi(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// two exponentials per MUFU op: 2^x on packed halves (ex2.approx.f16x2).  The
// fp16 input keeps 11 significant bits of x <= 8 (|error in 2^x| <= 0.27 %, the
// size of the bf16 rounding P gets anyway), the result 11 bits; P in [0, 256].
__device__ __forceinline__ uint64_t ex2_h2(uint64_t x2) {
  uint32_t h, e;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(f2hi(x2)), "f"(f2lo(x2)));
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(e) : "r"(h));
  float lo, hi;
  asm("{\n.reg .f16 a, b;\nmov.b32 {a, b}, %2;\ncvt.f32.f16 %0, a;\ncvt.f32.f16 %1, b;\n}" : "=f"(lo), "=f"(hi) : "r"(e));
  return f2pack(lo, hi);
}
// pairs of exponentials emulated on the FMA pipe (bit mask over pair index mod 8): 3/8
constexpr uint32_t POLY_PAIRS = 0xA4;
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

// causal mask of the diagonal tile: key column i > query row -> -inf
__device__ __forceinline__ void mask_diag(uint32_t (&r)[128], int row) {
#pragma unroll
  for (int i = 0; i < 128; ++i)
    if (i > row) r[i] = __float_as_uint(-INFINITY);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// The query tiles of a CTA: slot 0 (short) and slot 1 (long); len = kv tiles.
struct FwdPlan {
  int h, q0, q1, len0, len1;
};
__device__ __forceinline__ FwdPlan fwd_plan(const FwdArgs& g) {
  FwdPlan p;
  const int n_pairs = (g.n_qt + 1) >> 1;
  p.h = blockIdx.x % g.H;
  const int u = blockIdx.x / g.H;
  if (g.causal) {
    p.q0 = u; p.q1 = g.n_qt - 1 - u;
  } else {
    p.q0 = 2 * u; p.q1 = 2 * u + 1;
    if (p.q1 >= g.n_qt) { p.q1 = p.q0; }
  }
  if (p.q0 == p.q1) {   // a single tile: it runs as the long one
    p.len0 = 0;
  } else {
    p.len0 = g.causal ? p.q0 + 1 : g.n_qt;
  }
  p.len1 = g.causal ? p.q1 + 1 : g.n_qt;
  (void)n_pairs;
  return p;
}
// S/P buffer of slot 1 at kv step j (slot 0 always uses buffer 0)
__device__ __forceinline__ int buf1(const FwdPlan& p, int j) { return j < p.len0 ? 1 : ((j - p.len0) & 1); }

__global__ void __launch_bounds__(F_THREADS, 1)
    fmha_fwd_sm100(const __grid_constant__ CUtensorMap tmQKV, FwdArgs g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = smem;                         // [2][TILE]
  uint8_t* ring = smem + 2 * TILE;            // [F_RING][TILE]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + F_RING * TILE);
  uint64_t* full = bars;                      // [F_RING]
  uint64_t* empty = bars + F_RING;            // [F_RING]
  uint64_t* q_full = bars + 2 * F_RING;       // [2]
  uint64_t* s_full = q_full + 2;              // [2] per S buffer
  uint64_t* p_full = s_full + 2;              // [2] per S buffer
  uint64_t* o_done = p_full + 2;              // [2] per slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const FwdPlan pl = fwd_plan(g);
  int dbg_n = 0;
  const bool dbg_on = g.dbg && (int)blockIdx.x == g.dbg_cta && (lane == 0) &&
                      (warp == 1 || warp == 0 || warp == 4 || warp == 8);
#define DBG(stream, code, j)                                                                        \
  do {                                                                                              \
    if (dbg_on && dbg_n < 512)                                                                      \
      g.dbg[(stream) * 512 + dbg_n++] = ((long long)(code) << 56) | ((long long)(j) << 40) |        \
                                        (long long)(clock64() & 0xffffffffffLL);                     \
  } while (0)
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tmQKV);
    for (int s = 0; s < F_RING; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], 1); }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&q_full[i], 1);
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&p_full[i], 128);
      sm100::mbar_init(&o_done[i], 1);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 2) sm100::tmem_alloc<512>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  sm100::griddep_launch();
  sm100::griddep_wait();

  const int n_iter = pl.len1;
  const int kcol = g.D + pl.h * DH, vcol = 2 * g.D + pl.h * DH;

  // registers: producer / MMA / allocator warpgroup down, the two softmax warpgroups up
  if (warp == 0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (lane == 0) {
      if (pl.len0) {
        sm100::mbar_arrive_expect_tx(&q_full[0], TILE);
        for (int p = 0; p < 2; ++p)
          sm100::tma_load_2d(sQ + p * PANEL, &tmQKV, &q_full[0], pl.h * DH + 64 * p, pl.q0 * FT);
      }
      sm100::mbar_arrive_expect_tx(&q_full[1], TILE);
      for (int p = 0; p < 2; ++p)
        sm100::tma_load_2d(sQ + TILE + p * PANEL, &tmQKV, &q_full[1], pl.h * DH + 64 * p, pl.q1 * FT);
      for (int n = 0; n < 2 * n_iter; ++n) {
        const int st = n % F_RING, j = n >> 1;
        DBG(0, 20, n);
        wait(&empty[st], ((n / F_RING) & 1) ^ 1);
        DBG(0, 21, n);
        sm100::mbar_arrive_expect_tx(&full[st], TILE);
        const int col = (n & 1) ? vcol : kcol;
        for (int p = 0; p < 2; ++p)
          sm100::tma_load_2d(ring + st * TILE + p * PANEL, &tmQKV, &full[st], col + 64 * p, j * FT);
      }
    }
  } else if (warp == 1) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    // the whole warp walks the schedule (warp-uniform values stay in uniform
    // registers); one elected lane issues each tcgen05 op
    constexpr uint32_t idS = sm100::idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t idO = sm100::idesc_bf16(128, 128, 0, 1);
    const uint64_t dQ0 = sm100::umma_desc_sw128(sm100::smem_u32(sQ), 16, 1024);
    const uint64_t dQ1 = sm100::umma_desc_sw128(sm100::smem_u32(sQ + TILE), 16, 1024);
    const uint64_t dK0 = sm100::umma_desc_sw128(sm100::smem_u32(ring), 16, 1024);
    const uint64_t dV0 = sm100::umma_desc_sw128(sm100::smem_u32(ring), PANEL, 1024);
    int pc0 = 0, pc1 = 0;     // p_full consumptions per S buffer
    auto ring_wait = [&](int n) {
      DBG(1, 10, n);
      wait(&full[n % F_RING], (n / F_RING) & 1);
      sm100::tc_fence_after();
      DBG(1, 11, n);
    };
    auto qk = [&](uint64_t dq, int n, int b) {
      const uint64_t dk = dK0 + (uint64_t)(((n % F_RING) * TILE) >> 4);
      const uint32_t d = tmem + b * 128;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = ((k >> 2) * PANEL + (k & 3) * 32) >> 4;
        mma_ss_e(d, dq + off, dk + off, idS, k != 0);
      }
      commit_e(&s_full[b]);
    };
    auto pv = [&](int slot, int n, int b, int j) {
      DBG(1, 12, j);
      const int c = b ? pc1 : pc0;
      wait(&p_full[b], c & 1);
      if (b) ++pc1; else ++pc0;
      sm100::tc_fence_after();
      DBG(1, 13, j);
      const uint64_t dv = dV0 + (uint64_t)(((n % F_RING) * TILE) >> 4);
      const uint32_t d = tmem + 256 + slot * 128, a = tmem + b * 128;
#pragma unroll
      for (int k = 0; k < 8; ++k) mma_ts_e(d, a + k * 8, dv + ((k * 16 * 128) >> 4), idO, (j | k) != 0);
      commit_e(&o_done[slot]);
    };
    for (int j = 0; j < n_iter; ++j) {
      ring_wait(2 * j);
      if (j < pl.len0) {
        if (j == 0) { wait(&q_full[0], 0); sm100::tc_fence_after(); }
        qk(dQ0, 2 * j, 0);
        if (j >= 1) {
          pv(1, 2 * (j - 1) + 1, buf1(pl, j - 1), j - 1);
          commit_e(&empty[(2 * (j - 1) + 1) % F_RING]);
        }
        if (j == 0) { wait(&q_full[1], 0); sm100::tc_fence_after(); }
        qk(dQ1, 2 * j, 1);
        commit_e(&empty[(2 * j) % F_RING]);
        ring_wait(2 * j + 1);
        pv(0, 2 * j + 1, 0, j);
      } else {
        if (j == 0) { wait(&q_full[1], 0); sm100::tc_fence_after(); }
        qk(dQ1, 2 * j, buf1(pl, j));
        commit_e(&empty[(2 * j) % F_RING]);
        if (j >= 1) {
          if (j - 1 >= pl.len0) ring_wait(2 * (j - 1) + 1);
          pv(1, 2 * (j - 1) + 1, buf1(pl, j - 1), j - 1);
          commit_e(&empty[(2 * (j - 1) + 1) % F_RING]);
        }
      }
    }
    const int j = n_iter - 1;
    if (j >= pl.len0) ring_wait(2 * j + 1);
    pv(1, 2 * j + 1, buf1(pl, j), j);
    commit_e(&empty[(2 * j + 1) % F_RING]);
  } else if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  } else {
    // (the pool is what warpgroup 0 released: 128 x (168 - 56) = 256 x (224 - 168))
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    // softmax: warpgroup 1 = query tile of slot 0, warpgroup 2 = slot 1; one
    // thread per query row (TMEM lane)
    const int slot = (warp - 4) >> 2, q = warp & 3;
    const int row = q * 32 + lane;
    const int qi = slot ? pl.q1 : pl.q0;
    const int len = slot ? pl.len1 : pl.len0;
    int cnt[2] = {slot ? pl.len0 : 0, 0};   // s_full completions seen per buffer (slot 0 used buffer 0 len0 times)
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t o_t = tmem + lane_off + 256 + slot * 128;
    float m_used = -INFINITY, l = 0.f;
    const uint64_t sl2_2 = f2pack(g.sl2, g.sl2);
    for (int j = 0; j < len; ++j) {
      const int b = slot ? buf1(pl, j) : 0;
      DBG(2 + slot, 0, j);
      wait(&s_full[b], cnt[b] & 1);
      ++cnt[b];
      sm100::tc_fence_after();
      const uint32_t s_t = tmem + lane_off + b * 128;
      const bool diag = g.causal && j == qi;
      DBG(2 + slot, 1, j);
      // the whole S row in registers: four loads in flight, one wait
      uint32_t r[128];
      sm100::tmem_ld32(s_t, *reinterpret_cast<uint32_t(*)[32]>(r));
      sm100::tmem_ld32(s_t + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
      sm100::tmem_ld32(s_t + 64, *reinterpret_cast<uint32_t(*)[32]>(r + 64));
      sm100::tmem_ld32(s_t + 96, *reinterpret_cast<uint32_t(*)[32]>(r + 96));
      sm100::tmem_ld_wait();
      DBG(2 + slot, 2, j);
      if (diag) mask_diag(r, row);
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < 128; i += 2)
        mx4[(i >> 1) & 3] = fmaxf(mx4[(i >> 1) & 3], fmaxf(__uint_as_float(r[i]), __uint_as_float(r[i + 1])));
      const float m_new = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * g.sl2;
      const bool need = m_new > m_used + 8.f;
      if (__any_sync(0xffffffffu, need)) {
        const float alpha = need ? ex2(m_used - m_new) : 1.f;
        if (need) { m_used = m_new; l *= alpha; }
        if (j > 0) {   // O holds P V of earlier tiles: wait for the last PV, then scale
          wait(&o_done[slot], (j - 1) & 1);
          sm100::tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            sm100::tmem_ld32(o_t + 32 * c, o);
            sm100::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(o_t + 32 * c, o);
          }
          tmem_st_wait();
        }
      }
      // exponentials on pairs (FFMA2 / FADD2): x = s*scale*log2e - m; 3 of every 8
      // pairs on the FMA pipe (ex2_poly2), the rest on MUFU.  P (bf16 pairs) goes
      // over the first 64 columns of the S buffer: the A operand of the PV MMA
      // phase 1: x = s*scale*log2e - m in place (FFMA2); phase 2: 2^x in place, 3 of
      // every 8 pairs on the FMA pipe (ex2_poly2), the rest on MUFU; phase 3: row
      // sum (FADD2), bf16 pairs of P over the first 64 columns of the S buffer (the
      // A operand of the PV MMA).  Phases keep producer and consumer far apart: one
      // warp per SM sub-partition has nothing else to hide latencies with.
      const uint64_t negm2 = f2pack(-m_used, -m_used);
#pragma unroll
      for (int i = 0; i < 128; i += 2) {
        const uint64_t x2 = ffma2(u2pack(r[i], r[i + 1]), sl2_2, negm2);
        r[i] = (uint32_t)x2;
        r[i + 1] = (uint32_t)(x2 >> 32);
      }
#pragma unroll
      for (int i = 0; i < 128; i += 2) {
        if ((POLY_PAIRS >> ((i >> 1) & 7)) & 1) {
          const uint64_t p2 = ex2_poly2(u2pack(r[i], r[i + 1]));
          r[i] = (uint32_t)p2;
          r[i + 1] = (uint32_t)(p2 >> 32);
        } else {
          r[i] = __float_as_uint(ex2(__uint_as_float(r[i])));
          r[i + 1] = __float_as_uint(ex2(__uint_as_float(r[i + 1])));
        }
      }
      uint64_t l2[4] = {0, 0, 0, 0};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const uint64_t p2 = u2pack(r[32 * c + i], r[32 * c + i + 1]);
          l2[(i >> 1) & 3] = fadd2(l2[(i >> 1) & 3], p2);
          pk[i >> 1] = pack_bf16(f2lo(p2), f2hi(p2));
        }
        tmem_st16(s_t + 16 * c, pk);
      }
      {
        const uint64_t ls = fadd2(fadd2(l2[0], l2[1]), fadd2(l2[2], l2[3]));
        l += f2lo(ls) + f2hi(ls);
      }
      DBG(2 + slot, 3, j);
      tmem_st_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&p_full[b]);
      DBG(2 + slot, 4, j);
    }
    if (len > 0) {
      wait(&o_done[slot], (len - 1) & 1);
      sm100::tc_fence_after();
      const float inv = 1.f / l;
      const int t = qi * FT + row;
      __nv_bfloat16* orow = g.o + (size_t)t * g.ldo + pl.h * DH;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        sm100::tmem_ld32(o_t + 32 * c, r);
        sm100::tmem_ld_wait();
        uint4* dst = reinterpret_cast<uint4*>(orow + 32 * c);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(r[8 * v + 0]) * inv, __uint_as_float(r[8 * v + 1]) * inv);
          w.y = pack_bf16(__uint_as_float(r[8 * v + 2]) * inv, __uint_as_float(r[8 * v + 3]) * inv);
          w.z = pack_bf16(__uint_as_float(r[8 * v + 4]) * inv, __uint_as_float(r[8 * v + 5]) * inv);
          w.w = pack_bf16(__uint_as_float(r[8 * v + 6]) * inv, __uint_as_float(r[8 * v + 7]) * inv);
          dst[v] = w;
        }
      }
      g.lse[(size_t)pl.h * g.lse_ld + t] = (m_used + __log2f(l)) * 0.6931471805599453f;
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem);
  }
}

typedef CUresult (*encode_fn_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

encode_fn_t encode() {
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

// bf16 [rows, cols] row-major (leading dim ld), box {64 cols, box_rows}, SW128
int map_bf16(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, int box_rows) {
  encode_fn_t enc = encode();
  if (!enc) return rrfp_fail(RRFP_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return rrfp_fail(RRFP_E_INVALID, "fmha tensor map encode failed (%d)", (int)r);
  return RRFP_OK;
}


// ---------------------------------------------------------------------------
// Backward (FA2-style key/value-stationary): one CTA per (head, pair of 128-row
// key tiles (u, n-1-u)), processed one after the other (every CTA does the same
// number of steps under the causal mask).  For a key tile j the CTA walks the
// 64-row query sub-tiles i it sees:
//   S^T  = K Q_i^T,  dP^T = V dO_i^T          (SS, 128 x 64 x 128, TMEM)
//   P^T  = exp2(S^T * scale*log2e - lse2_i),   dS^T = scale * P^T (dP^T - D_i)
//          (elementwise warpgroups 1-2, one thread per key row, 32 query columns
//           each; bf16 P^T / dS^T to shared memory, SW128 K-major)
//   dV  += P^T dO_i,  dK += dS^T Q_i            (SS, 128 x 128 x 64, TMEM accumulators)
//   dQ_i^T = K^T dS^T                          (SS, 128 x 64 x 128, double-buffered TMEM)
//          -> warpgroup 3 reduces it into the fp32 dQ accumulator (TMA reduce-add)
// TMEM: dV [0,128) dK [128,256) S^T [256,320) dP^T [320,384) dQ^T x2 [384,512).
// MMA issue order per step: S^T_i, dP^T_i, dV_{i-1}, dK_{i-1}, dQ^T_{i-1}, so the
// elementwise pass of step i overlaps the gradient MMAs of step i-1.
// D_i = rowsum(dO * O) and lse2 = lse * log2(e) come from attn_bwd_prep_kernel;
// attn_bwd_dq_kernel converts the fp32 dQ into the packed dQKV afterwards.
constexpr int B_QT = 64;                        // query sub-tile rows
constexpr int B_QTILE = B_QT * DH * 2;          // 16 KB
constexpr int B_STAGES = 3;
constexpr int B_STAGE = 2 * B_QTILE;            // Q_i, dO_i (1024-aligned SW128 tiles)
constexpr int B_VEC = 512;                      // lse2_i[64], D_i[64] per stage
constexpr int B_SMEM = 2 * TILE + B_STAGES * (B_STAGE + B_VEC) + 2 * (FT * B_QT * 2) + B_QT * DH * 4 + 1024 + 256;
constexpr int B_EWG = 2;                        // elementwise warpgroups (query columns split B_EWG ways)
constexpr int B_EWC = B_QT / B_EWG;             // query columns per elementwise thread
constexpr int B_RD0 = 4 + 4 * B_EWG;            // first dQ read-out warp
constexpr int B_THREADS = 32 * (B_RD0 + 4);

struct BwdArgs {
  int T, H, D, n_kt, causal;
  float sl2, scale;
  const float* lse2;    // [H][T]
  const float* dsum;    // [H][T]  D = rowsum(dO * O)
  __nv_bfloat16* dqkv;
  long long lddqkv;
  long long* dbg;    // optional event log of CTA dbg_cta: [4][512]
  int dbg_cta;
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sm100::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(sm100::smem_u32(bar))
               : "memory");
}

// key tiles of a CTA and their query sub-tile ranges
struct BwdPlan {
  int h, n_units, kt[2];
};
__device__ __forceinline__ BwdPlan bwd_plan(const BwdArgs& g) {
  BwdPlan p;
  p.h = blockIdx.x % g.H;
  const int u = blockIdx.x / g.H;
  if (g.causal) { p.kt[0] = u; p.kt[1] = g.n_kt - 1 - u; }
  else { p.kt[0] = 2 * u; p.kt[1] = 2 * u + 1; }
  p.n_units = (p.kt[1] == p.kt[0] || p.kt[1] >= g.n_kt) ? 1 : 2;
  return p;
}
// first query sub-tile of key tile kt, and the count
__device__ __forceinline__ int bwd_i0(const BwdArgs& g, int kt) { return g.causal ? 2 * kt : 0; }
__device__ __forceinline__ int bwd_ni(const BwdArgs& g, int kt) { return 2 * g.n_kt - bwd_i0(g, kt); }

__global__ void __launch_bounds__(B_THREADS, 1)
    fmha_bwd_sm100(const __grid_constant__ CUtensorMap tmKV,    // qkv, box {64, 128}
                   const __grid_constant__ CUtensorMap tmQ,     // qkv, box {64, 64}
                   const __grid_constant__ CUtensorMap tmDO,    // dO,  box {64, 64}
                   const __grid_constant__ CUtensorMap tmDQ,    // fp32 dQ accumulator, box {128, 64}
                   BwdArgs g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sK = smem;
  uint8_t* sV = smem + TILE;
  uint8_t* stg = smem + 2 * TILE;                       // [B_STAGES][Q | dO]
  uint8_t* sP = stg + B_STAGES * B_STAGE;               // P^T  [128 keys x 64 q] bf16 SW128
  uint8_t* sDS = sP + FT * B_QT * 2;                    // dS^T
  float* sDQ = reinterpret_cast<float*>(sDS + FT * B_QT * 2);   // dQ staging [64 q][128 d]
  uint8_t* svec = reinterpret_cast<uint8_t*>(sDQ) + B_QT * DH * 4;   // [B_STAGES][lse2 | D]
  uint64_t* bars = reinterpret_cast<uint64_t*>(svec + B_STAGES * B_VEC);
  uint64_t* kv_full = bars;                 // K, V of the unit loaded
  uint64_t* kv_free = bars + 1;             // the unit's MMAs are done with K, V
  uint64_t* full = bars + 2;                // [B_STAGES]
  uint64_t* empty = full + B_STAGES;        // [B_STAGES]
  uint64_t* s_full = empty + B_STAGES;      // S^T, dP^T of the step in TMEM
  uint64_t* sd_free = s_full + 1;           // ... loaded into registers (256 arrivals)
  uint64_t* ds_full = sd_free + 1;          // P^T, dS^T in smem (256 arrivals)
  uint64_t* pds_free = ds_full + 1;         // the MMAs reading P^T, dS^T are done
  uint64_t* dq_full = pds_free + 1;         // [2] dQ^T in TMEM
  uint64_t* dq_free = dq_full + 2;          // [2] ... read out (128 arrivals)
  uint64_t* acc_full = dq_free + 2;         // dV, dK of the unit complete
  uint64_t* acc_free = acc_full + 1;        // ... written out (256 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const BwdPlan pl = bwd_plan(g);
  int dbg_n = 0;
  const bool dbg_on = g.dbg && (int)blockIdx.x == g.dbg_cta && (lane == 0) &&
                      (warp == 1 || warp == 0 || warp == 4 || warp == B_RD0);
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tmKV); sm100::tma_prefetch(&tmQ); sm100::tma_prefetch(&tmDO); sm100::tma_prefetch(&tmDQ);
    sm100::mbar_init(kv_full, 1); sm100::mbar_init(kv_free, 1);
    for (int s = 0; s < B_STAGES; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], 1); }
    sm100::mbar_init(s_full, 1); sm100::mbar_init(sd_free, 128 * B_EWG); sm100::mbar_init(ds_full, 128 * B_EWG);
    sm100::mbar_init(pds_free, 1);
    for (int b = 0; b < 2; ++b) { sm100::mbar_init(&dq_full[b], 1); sm100::mbar_init(&dq_free[b], 128); }
    sm100::mbar_init(acc_full, 1); sm100::mbar_init(acc_free, 128 * B_EWG);
    sm100::fence_barrier_init();
  }
  if (warp == 2) sm100::tmem_alloc<512>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  sm100::griddep_launch();
  sm100::griddep_wait();
  const int kcol = g.D + pl.h * DH, vcol = 2 * g.D + pl.h * DH, qcol = pl.h * DH;

  if (warp == 0) {
    if (lane == 0) {
      int n = 0;
      for (int un = 0; un < pl.n_units; ++un) {
        const int kt = pl.kt[un];
        if (un) wait(kv_free, (un - 1) & 1);
        sm100::mbar_arrive_expect_tx(kv_full, 2 * TILE);
        for (int p = 0; p < 2; ++p) {
          sm100::tma_load_2d(sK + p * PANEL, &tmKV, kv_full, kcol + 64 * p, kt * FT);
          sm100::tma_load_2d(sV + p * PANEL, &tmKV, kv_full, vcol + 64 * p, kt * FT);
        }
        const int i0 = bwd_i0(g, kt), ni = bwd_ni(g, kt);
        for (int ii = 0; ii < ni; ++ii, ++n) {
          const int i = i0 + ii, st = n % B_STAGES;
          wait(&empty[st], ((n / B_STAGES) & 1) ^ 1);
          uint8_t* d = stg + st * B_STAGE;
          sm100::mbar_arrive_expect_tx(&full[st], 2 * B_QTILE + B_VEC);
          for (int p = 0; p < 2; ++p) {
            sm100::tma_load_2d(d + p * (B_QTILE / 2), &tmQ, &full[st], qcol + 64 * p, i * B_QT);
            sm100::tma_load_2d(d + B_QTILE + p * (B_QTILE / 2), &tmDO, &full[st], qcol + 64 * p, i * B_QT);
          }
          bulk_g2s(svec + st * B_VEC, g.lse2 + (size_t)pl.h * g.T + i * B_QT, 256, &full[st]);
          bulk_g2s(svec + st * B_VEC + 256, g.dsum + (size_t)pl.h * g.T + i * B_QT, 256, &full[st]);
        }
      }
    }
  } else if (warp == 1 || warp == 3) {
    // Two MMA issuers: warp 1 issues S^T / dP^T of each step, warp 3 the gradient
    // MMAs (dV, dK, dQ^T) of the step the elementwise pass finished.  One issuer
    // spent ~1,800 of ~3,000 cycles per step issuing these 32 small MMAs
    // (tools/attn_timeline.py --bwd); split, the two streams of issues overlap.
    // Each warp commits only its own MMAs (tcgen05.commit tracks the issuing
    // thread's operations); the barriers order what the two share: S^T / dP^T
    // TMEM (s_full -> sd_free), P^T / dS^T smem (ds_full -> pds_free), the Q / dO
    // stage (released by the gradient MMAs, which follow the stage's S^T / dP^T
    // through ds_full), K / V (kv_free after the unit's last gradient MMAs).
    // S^T / dP^T: M=128 keys, N=64 queries, K=128 (A K-major keys/values, B K-major Q/dO)
    constexpr uint32_t idSD = sm100::idesc_bf16(128, 64, 0, 0);
    // dV / dK: M=128 keys, N=128 (d), K=64 queries (A = P^T / dS^T K-major, B = dO / Q MN-major)
    constexpr uint32_t idVK = sm100::idesc_bf16(128, 128, 0, 1);
    // dQ^T: M=128 (d), N=64 queries, K=128 keys (A = K MN-major, B = dS^T MN-major)
    constexpr uint32_t idQ = sm100::idesc_bf16(128, 64, 1, 1);
    const uint32_t tS = tmem + 256, tP = tmem + 320;
    const uint64_t dK_k = sm100::umma_desc_sw128(sm100::smem_u32(sK), 16, 1024);
    const uint64_t dV_k = sm100::umma_desc_sw128(sm100::smem_u32(sV), 16, 1024);
    const uint64_t dK_mn = sm100::umma_desc_sw128(sm100::smem_u32(sK), PANEL, 1024);
    const uint64_t dP_a = sm100::umma_desc_sw128(sm100::smem_u32(sP), 16, 1024);
    const uint64_t dDS_a = sm100::umma_desc_sw128(sm100::smem_u32(sDS), 16, 1024);
    const uint64_t dDS_b = sm100::umma_desc_sw128(sm100::smem_u32(sDS), PANEL, 1024);
    const uint64_t dStg_k = sm100::umma_desc_sw128(sm100::smem_u32(stg), 16, 1024);
    const uint64_t dStg_mn = sm100::umma_desc_sw128(sm100::smem_u32(stg), B_QTILE / 2, 1024);
    int n = 0, step = 0;   // ring index, global step (sd/ds/pds/dq parities)
    if (warp == 1) {
      for (int un = 0; un < pl.n_units; ++un) {
        const int ni = bwd_ni(g, pl.kt[un]);
        wait(kv_full, un & 1);
        sm100::tc_fence_after();
        for (int ii = 0; ii < ni; ++ii, ++n, ++step) {
          const int st = n % B_STAGES;
          DBG(1, 10, step);
          wait(&full[st], (n / B_STAGES) & 1);
          DBG(1, 11, step);
          if (step) wait(sd_free, (step - 1) & 1);   // the elementwise pass has S^T / dP^T of the last step
          DBG(1, 12, step);
          sm100::tc_fence_after();
          const uint64_t so = (uint64_t)((st * B_STAGE) >> 4);
          // (k-block offsets: K-major panels of 128 rows (A) / 64 rows (B), 32 B per k16)
          mma_ss_x8<2, (PANEL >> 4), 2, ((B_QTILE / 2) >> 4)>(tS, dK_k, dStg_k + so, idSD, 0);
          mma_ss_x8<2, (PANEL >> 4), 2, ((B_QTILE / 2) >> 4)>(tP, dV_k, dStg_k + so + (B_QTILE >> 4), idSD, 0);
          commit_e(s_full);
          DBG(1, 13, step);
        }
      }
    } else {
      for (int un = 0; un < pl.n_units; ++un) {
        const int ni = bwd_ni(g, pl.kt[un]);
        wait(kv_full, un & 1);
        if (un) wait(acc_free, (un - 1) & 1);   // the previous unit's dV / dK are written out
        sm100::tc_fence_after();
        for (int ii = 0; ii < ni; ++ii, ++n, ++step) {
          const int st = n % B_STAGES;
          const bool first = ii == 0;
          wait(ds_full, step & 1);
          sm100::tc_fence_after();
          const uint64_t so = (uint64_t)((st * B_STAGE) >> 4);
          // dV += P^T dO, dK += dS^T Q  (A K-major: 32 B per k16; B MN-major: 16 rows x 128 B per k16)
          mma_ss_x4<2, 128>(tmem, dP_a, dStg_mn + so + (B_QTILE >> 4), idVK, !first);
          mma_ss_x4<2, 128>(tmem + 128, dDS_a, dStg_mn + so, idVK, !first);
          const int b = step & 1;
          if (step >= 2) wait(&dq_free[b], ((step - 2) >> 1) & 1);
          sm100::tc_fence_after();
          // dQ^T = K^T dS^T (both MN-major: 16 rows x 128 B per k16)
          mma_ss_x8<128, 512, 128, 512>(tmem + 384 + 64 * b, dK_mn, dDS_b, idQ, 0);
          commit_e(pds_free);
          commit_e(&dq_full[b]);
          commit_e(&empty[st]);
        }
        commit_e(acc_full);
        commit_e(kv_free);
      }
    }
  } else if (warp >= 4 && warp < B_RD0) {
    // elementwise: thread = key row, B_EWC query columns of the sub-tile
    const int wg = (warp - 4) >> 2, q4 = warp & 3, row = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint64_t sl2_2 = f2pack(g.sl2, g.sl2);
    int n = 0, step = 0;
    for (int un = 0; un < pl.n_units; ++un) {
      const int kt = pl.kt[un], i0 = bwd_i0(g, kt), ni = bwd_ni(g, kt);
      const int key = kt * FT + row;
      for (int ii = 0; ii < ni; ++ii, ++n, ++step) {
        const int st = n % B_STAGES, i = i0 + ii;
        const float* vec = reinterpret_cast<const float*>(svec + st * B_VEC);
        DBG(2, 0, step);
        wait(&full[st], (n / B_STAGES) & 1);   // (the stage's lse2 / D vectors)
        wait(s_full, step & 1);
        DBG(2, 1, step);
        sm100::tc_fence_after();
        uint32_t s[B_EWC], dp[B_EWC];
        if (B_EWC == 32) {
          sm100::tmem_ld32(tmem + lane_off + 256 + wg * B_EWC, *reinterpret_cast<uint32_t(*)[32]>(s));
          sm100::tmem_ld32(tmem + lane_off + 320 + wg * B_EWC, *reinterpret_cast<uint32_t(*)[32]>(dp));
        } else {
          tmem_ld16(tmem + lane_off + 256 + wg * B_EWC, *reinterpret_cast<uint32_t(*)[16]>(s));
          tmem_ld16(tmem + lane_off + 320 + wg * B_EWC, *reinterpret_cast<uint32_t(*)[16]>(dp));
        }
        sm100::tmem_ld_wait();
        sm100::tc_fence_before();
        sm100::mbar_arrive(sd_free);
        DBG(2, 5, step);
        const int qb = i * B_QT + wg * B_EWC;
        const bool mask = g.causal && qb < key;   // some query of this warp's columns precedes the key
        uint32_t pw[B_EWC / 2], dw[B_EWC / 2];
#pragma unroll
        for (int c = 0; c < B_EWC; c += 2) {
          const uint64_t l2 = *reinterpret_cast<const uint64_t*>(vec + wg * B_EWC + c);
          const uint64_t d2 = *reinterpret_cast<const uint64_t*>(vec + 64 + wg * B_EWC + c);
          const uint64_t x2 = ffma2(u2pack(s[c], s[c + 1]), sl2_2, l2 ^ 0x8000000080000000ull);
          float p0 = ex2(f2lo(x2)), p1 = ex2(f2hi(x2));
          if (mask) {
            if (qb + c < key) p0 = 0.f;
            if (qb + c + 1 < key) p1 = 0.f;
          }
          const uint64_t p2 = f2pack(p0, p1);
          const uint64_t t2 = fadd2(u2pack(dp[c], dp[c + 1]), d2 ^ 0x8000000080000000ull);   // dP - D
          const uint64_t ds2 = ffma2(ffma2(p2, t2, 0), f2pack(g.scale, g.scale), 0);   // scale * P (dP - D)
          pw[c >> 1] = pack_bf16(p0, p1);
          dw[c >> 1] = pack_bf16(f2lo(ds2), f2hi(ds2));
        }
        DBG(2, 2, step);
        if (step) wait(pds_free, (step - 1) & 1);   // the last step's MMAs have read P^T / dS^T
        DBG(2, 3, step);
        // row `row` of the SW128 K-major tiles: 128 B = 8 chunks of 16 B, chunk c at c ^ (row & 7)
        uint8_t* prow = sP + row * 128;
        uint8_t* drow = sDS + row * 128;
#pragma unroll
        for (int c = 0; c < B_EWC / 8; ++c) {
          const int ch = ((wg * (B_EWC / 8) + c) ^ (row & 7)) * 16;
          *reinterpret_cast<uint4*>(prow + ch) = make_uint4(pw[4 * c], pw[4 * c + 1], pw[4 * c + 2], pw[4 * c + 3]);
          *reinterpret_cast<uint4*>(drow + ch) = make_uint4(dw[4 * c], dw[4 * c + 1], dw[4 * c + 2], dw[4 * c + 3]);
        }
        sm100::fence_proxy_async_smem();
        sm100::mbar_arrive(ds_full);
        DBG(2, 4, step);
      }
      // unit epilogue: the elementwise warpgroups write dV (TMEM columns [0,128)) and dK
      // ([128,256)), 256 / B_EWG columns each, bf16 into the packed dQKV
      wait(acc_full, un & 1);
      sm100::tc_fence_after();
      constexpr int EC = 256 / B_EWG;
      const int c0 = wg * EC;
      __nv_bfloat16* dst = g.dqkv + (size_t)key * g.lddqkv + (c0 < 128 ? vcol + c0 : kcol + c0 - 128);
#pragma unroll 1
      for (int c = 0; c < EC / 32; ++c) {
        uint32_t r[32];
        sm100::tmem_ld32(tmem + lane_off + c0 + 32 * c, r);
        sm100::tmem_ld_wait();
        uint4* o4 = reinterpret_cast<uint4*>(dst + 32 * c);
#pragma unroll
        for (int v = 0; v < 4; ++v)
          o4[v] = make_uint4(pack_bf16(__uint_as_float(r[8 * v]), __uint_as_float(r[8 * v + 1])),
                             pack_bf16(__uint_as_float(r[8 * v + 2]), __uint_as_float(r[8 * v + 3])),
                             pack_bf16(__uint_as_float(r[8 * v + 4]), __uint_as_float(r[8 * v + 5])),
                             pack_bf16(__uint_as_float(r[8 * v + 6]), __uint_as_float(r[8 * v + 7])));
      }
      sm100::tc_fence_before();
      sm100::mbar_arrive(acc_free);
    }
  } else if (warp >= B_RD0) {
    // dQ^T read-out: thread = head-dim lane d, 64 query columns -> staging [q][d] ->
    // TMA reduce-add into the fp32 dQ accumulator
    const int q4 = warp & 3, d = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const bool issuer = warp == B_RD0 && lane == 0;
    int step = 0;
    for (int un = 0; un < pl.n_units; ++un) {
      const int kt = pl.kt[un], i0 = bwd_i0(g, kt), ni = bwd_ni(g, kt);
      for (int ii = 0; ii < ni; ++ii, ++step) {
        const int b = step & 1;
        DBG(3, 30, step);
        wait(&dq_full[b], (step >> 1) & 1);
        DBG(3, 31, step);
        sm100::tc_fence_after();
        uint32_t r[64];
        sm100::tmem_ld32(tmem + lane_off + 384 + 64 * b, *reinterpret_cast<uint32_t(*)[32]>(r));
        sm100::tmem_ld32(tmem + lane_off + 384 + 64 * b + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        sm100::tmem_ld_wait();
        sm100::tc_fence_before();
        sm100::mbar_arrive(&dq_free[b]);
        if (issuer) sm100::bulk_wait_read<0>();   // the last reduce has read the staging tile
        named_bar(1, 128);
#pragma unroll
        for (int c = 0; c < 64; ++c) sDQ[c * DH + d] = __uint_as_float(r[c]);
        sm100::fence_proxy_async_smem();
        named_bar(1, 128);
        if (issuer) {
          sm100::tma_reduce_add_2d(&tmDQ, sDQ, pl.h * DH, (i0 + ii) * B_QT);
          sm100::bulk_commit();
        }
        DBG(3, 32, step);
      }
    }
    if (issuer) sm100::bulk_wait<0>();
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem);
  }
}

// D[h][t] = sum_d dO[t, h*128 + d] * O[t, h*128 + d];  lse2 = lse * log2(e).  One warp per (t, h).
__global__ void attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ o, long long ldo,
                                     const __nv_bfloat16* __restrict__ dout, long long lddo,
                                     const float* __restrict__ lse, long long lse_ld, float* __restrict__ lse2,
                                     float* __restrict__ dsum, int T, int H) {
  sm100::griddep_wait();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= T * H) return;
  const int t = w / H, h = w % H;
  const uint2 a = *reinterpret_cast<const uint2*>(o + (size_t)t * ldo + h * DH + lane * 4);
  const uint2 b = *reinterpret_cast<const uint2*>(dout + (size_t)t * lddo + h * DH + lane * 4);
  const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float2 x = __bfloat1622float2(a2[k]), y = __bfloat1622float2(b2[k]);
    acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) {
    dsum[(size_t)h * T + t] = acc;
    lse2[(size_t)h * T + t] = lse[(size_t)h * lse_ld + t] * 1.4426950408889634f;
  }
}

// dQ (fp32 [T, D]) -> bf16 columns [0, D) of the packed dQKV
__global__ void attn_bwd_dq_kernel(const float4* __restrict__ dq, __nv_bfloat16* __restrict__ dqkv, long long ld,
                                   int T, int D) {
  sm100::griddep_wait();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;   // 8 elements per thread
  const long long n8 = (long long)T * D / 8;
  if (i >= n8) return;
  const long long e = i * 8;
  const int t = (int)(e / D), c = (int)(e % D);
  const float4 a = dq[2 * i], b = dq[2 * i + 1];
  *reinterpret_cast<uint4*>(dqkv + (size_t)t * ld + c) =
      make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y), pack_bf16(b.z, b.w));
}

int map_f32(CUtensorMap* m, const void* ptr, long long rows, long long cols, int box_cols, int box_rows) {
  encode_fn_t enc = encode();
  if (!enc) return rrfp_fail(RRFP_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return rrfp_fail(RRFP_E_INVALID, "fmha dq tensor map encode failed (%d)", (int)r);
  return RRFP_OK;
}

long long* g_attn_dbg = nullptr;
long long* g_attn_dbg_bwd = nullptr;
int g_attn_dbg_cta = 0;

}  // namespace

/* test hook: log the event timeline of CTA `cta` into buf ([4][512] int64), NULL: off */
extern "C" int rrfp_attn_debug(long long* buf, int cta) {
  const char* e = getenv("RRFP_ATTN_DEBUG_BWD");
  if (e && atoi(e)) { g_attn_dbg_bwd = buf; g_attn_dbg_cta = cta; return RRFP_OK; }
  g_attn_dbg = buf;
  g_attn_dbg_cta = cta;
  return RRFP_OK;
}

extern "C" int rrfp_attn_fwd(const void* qkv, long long ldqkv, void* o, long long ldo, float* lse,
                             long long lse_ld, int T, int H, int d_head, int causal, float scale, void* stream) {
  if (d_head != DH) return rrfp_fail(RRFP_E_INVALID, "attn_fwd: d_head %d unsupported (128 only)", d_head);
  if (T <= 0 || T % FT) return rrfp_fail(RRFP_E_INVALID, "attn_fwd: T=%d must be a positive multiple of 128", T);
  if (!qkv || !o || !lse || ldqkv < 3LL * H * DH || ldo < (long long)H * DH || (ldqkv % 8) || (ldo % 8))
    return rrfp_fail(RRFP_E_INVALID, "attn_fwd: bad pointers / leading dims");
  static bool attr = false;
  if (!attr) {
    RRFP_CUDA_TRY(cudaFuncSetAttribute(fmha_fwd_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM));
    attr = true;
  }
  CUtensorMap m;
  int rc = map_bf16(&m, qkv, T, 3LL * H * DH, ldqkv, FT);
  if (rc) return rc;
  FwdArgs g;
  g.T = T; g.H = H; g.D = H * DH; g.n_qt = T / FT; g.causal = causal ? 1 : 0;
  g.sl2 = scale * 1.4426950408889634f;
  g.o = reinterpret_cast<__nv_bfloat16*>(o); g.ldo = ldo;
  g.lse = lse; g.lse_ld = lse_ld;
  g.dbg = g_attn_dbg; g.dbg_cta = g_attn_dbg_cta;
  g.experiment = 0;
  const int grid = H * ((g.n_qt + 1) / 2);
  RRFP_CUDA_TRY(rrfp_launch(fmha_fwd_sm100, dim3(grid), dim3(F_THREADS), F_SMEM, (cudaStream_t)stream, m, g));
  return RRFP_OK;
}

/* workspace of rrfp_attn_bwd: fp32 dQ accumulator [T, H*128] + lse2 [H, T] + D [H, T] */
extern "C" size_t rrfp_attn_bwd_workspace_bytes(int T, int H) {
  return (size_t)T * H * DH * 4 + 2 * (size_t)H * T * 4;
}

extern "C" int rrfp_attn_bwd(const void* qkv, long long ldqkv, const void* o, long long ldo, const void* dout,
                             long long lddo, const float* lse, long long lse_ld, void* dqkv, long long lddqkv,
                             void* workspace, int T, int H, int d_head, int causal, float scale, void* stream) {
  if (d_head != DH) return rrfp_fail(RRFP_E_INVALID, "attn_bwd: d_head %d unsupported (128 only)", d_head);
  if (T <= 0 || T % FT) return rrfp_fail(RRFP_E_INVALID, "attn_bwd: T=%d must be a positive multiple of 128", T);
  const long long D = (long long)H * DH;
  if (!qkv || !o || !dout || !lse || !dqkv || !workspace || ldqkv < 3 * D || lddqkv < 3 * D || ldo < D ||
      lddo < D || (ldqkv % 8) || (lddqkv % 8) || (ldo % 8) || (lddo % 8))
    return rrfp_fail(RRFP_E_INVALID, "attn_bwd: bad pointers / leading dims");
  static bool attr = false;
  if (!attr) {
    RRFP_CUDA_TRY(cudaFuncSetAttribute(fmha_bwd_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, B_SMEM));
    attr = true;
  }
  cudaStream_t st = (cudaStream_t)stream;
  float* dq = reinterpret_cast<float*>(workspace);
  float* lse2 = dq + (size_t)T * D;
  float* dsum = lse2 + (size_t)H * T;
  CUtensorMap mKV, mQ, mDO, mDQ;
  int rc = map_bf16(&mKV, qkv, T, 3 * D, ldqkv, FT);
  if (!rc) rc = map_bf16(&mQ, qkv, T, 3 * D, ldqkv, B_QT);
  if (!rc) rc = map_bf16(&mDO, dout, T, D, lddo, B_QT);
  if (!rc) rc = map_f32(&mDQ, dq, T, D, DH, B_QT);
  if (rc) return rc;
  RRFP_CUDA_TRY(cudaMemsetAsync(dq, 0, (size_t)T * D * 4, st));
  const int warps = T * H;
  RRFP_CUDA_TRY(rrfp_launch(attn_bwd_prep_kernel, dim3((warps + 7) / 8), dim3(256), 0, st,
                            reinterpret_cast<const __nv_bfloat16*>(o), ldo,
                            reinterpret_cast<const __nv_bfloat16*>(dout), lddo, lse, lse_ld, lse2, dsum, T, H));
  BwdArgs g;
  g.T = T; g.H = H; g.D = (int)D; g.n_kt = T / FT; g.causal = causal ? 1 : 0;
  g.sl2 = scale * 1.4426950408889634f; g.scale = scale;
  g.lse2 = lse2; g.dsum = dsum;
  g.dqkv = reinterpret_cast<__nv_bfloat16*>(dqkv); g.lddqkv = lddqkv;
  g.dbg = g_attn_dbg_bwd; g.dbg_cta = g_attn_dbg_cta;
  const int grid = H * ((g.n_kt + 1) / 2);
  RRFP_CUDA_TRY(rrfp_launch(fmha_bwd_sm100, dim3(grid), dim3(B_THREADS), B_SMEM, st, mKV, mQ, mDO, mDQ, g));
  const long long n8 = (long long)T * D / 8;
  RRFP_CUDA_TRY(rrfp_launch(attn_bwd_dq_kernel, dim3((unsigned)((n8 + 255) / 256)), dim3(256), 0, st,
                            reinterpret_cast<const float4*>(dq), reinterpret_cast<__nv_bfloat16*>(dqkv), lddqkv,
                            T, (int)D));
  return RRFP_OK;
}
