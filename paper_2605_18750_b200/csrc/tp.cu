// tp.cu -- tensor-parallel all-reduce inside one pipeline stage's TP group
// (BASELINE config 3, SURVEY.md 8e "K5"), over peer memory: no NCCL, no host.
//
// Each TP rank's row-parallel GEMM writes its fp32-accumulated bf16 partial
// [rows, cols] into its own `part` buffer.  The all-reduce kernel then
//   1. publishes READY(seq) into every peer's board (st.release.sys) and waits
//      for every peer's READY(seq) (ld.acquire.sys) -- one thread per CTA;
//   2. sums the R partials IN RANK ORDER (0..R-1, fp32), so every rank computes
//      bit-identical outputs, and fuses the row-parallel bias and the residual:
//      out = sum_q part_q + bias + resid, written to up to four destinations
//      (the local activation and the next stage's mailbox slots of every TP
//      rank: peer memory over NVLink when the ranks live on other GPUs);
//   3. the last CTA (atomic ticket) publishes DONE(seq) and waits for every
//      peer's DONE(seq): when the kernel retires, no peer still reads `part`,
//      so the next GEMM on the stream may overwrite it.
// `seq` is a per-rank device counter advanced by the kernel itself, so the
// kernel is replayable inside captured CUDA graphs.  Both ranks issue the same
// all-reduce sequence because the device dispatchers agree on every F/B task
// (tp_coordinate, arbitration.py:323-334) before running it.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "../../include/rrfp_b200.h"
#include "rrfp_common.h"
#include "sm100_ptx.cuh"

namespace {

constexpr int TP_MAX = 8;
constexpr int READY = 0, DONE = TP_MAX;   // board layout: ready[8], done[8] (u64)
constexpr unsigned long long SPIN_LIMIT_NS = 20ull * 1000 * 1000 * 1000;   // never hang the GPU

struct TpArgs {
  const __nv_bfloat16* part[TP_MAX];
  unsigned long long* board[TP_MAX];   // every rank's board (own included)
  unsigned long long* seq;             // own counter
  unsigned int* ticket;                // own CTA ticket
  int* err;                            // own error word (spin timeout)
  int R, rank;
};

struct TpOuts {
  __nv_bfloat16* out[4];
  int n;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// wait until every peer's board[slot + q] >= seq; false on timeout
__device__ bool wait_peers(const TpArgs& a, int slot, unsigned long long seq) {
  const unsigned long long t0 = now_ns();
  for (int q = 0; q < a.R; ++q) {
    if (q == a.rank) continue;
    while (ld_acquire_sys64(&a.board[a.rank][slot + q]) < seq) {
      if (now_ns() - t0 > SPIN_LIMIT_NS) { atomicExch(a.err, 1); return false; }
      __nanosleep(64);
    }
  }
  return true;
}

__device__ __forceinline__ void add8(const __nv_bfloat16* p, float* f) {
  uint4 q = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] += t.x;
    f[2 * i + 1] += t.y;
  }
}

__global__ void __launch_bounds__(512) tp_allreduce_kernel(TpArgs a, TpOuts o, const __nv_bfloat16* bias,
                                                           const __nv_bfloat16* resid, long long ld_resid,
                                                           int rows, int cols) {
  sm100::griddep_wait();   // the partial GEMM (previous kernel on this stream) has completed
  const unsigned long long seq = *reinterpret_cast<volatile unsigned long long*>(a.seq) + 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < a.R; ++q)
      if (q != a.rank) st_release_sys64(&a.board[q][READY + a.rank], seq);
  }
  if (threadIdx.x == 0) wait_peers(a, READY, seq);
  __syncthreads();

  const int c8n = cols >> 3;
  const long long total = (long long)rows * c8n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(i / c8n), c = (int)(i % c8n) * 8;
    const size_t off = (size_t)row * cols + c;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = 0.f;
    for (int q = 0; q < a.R; ++q) add8(a.part[q] + off, v);   // fixed rank order
    if (bias) add8(bias + c, v);
    if (resid) add8(resid + (size_t)row * ld_resid + c, v);
    uint4 w;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
    for (int k = 0; k < o.n; ++k) *reinterpret_cast<uint4*>(o.out[k] + off) = w;
  }

  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned int t = atomicAdd(a.ticket, 1u);
    if (t == gridDim.x - 1) {   // every CTA finished reading the peers' partials
      for (int q = 0; q < a.R; ++q)
        if (q != a.rank) st_release_sys64(&a.board[q][DONE + a.rank], seq);
      wait_peers(a, DONE, seq);
      *a.ticket = 0u;
      *a.seq = seq;
    }
  }
}

}  // namespace

struct rrfp_tp {
  int R, rank, dev;
  size_t part_bytes;
  void* part;                    // own partial (cudaMalloc: IPC exportable)
  unsigned long long* board;     // own board [2 * TP_MAX] (peers write it)
  unsigned long long* seq;       // own counter, ticket, error word
  const void* peer_part[TP_MAX];
  unsigned long long* peer_board[TP_MAX];
  bool connected;
};

extern "C" int rrfp_tp_create(int rank, int R, size_t part_bytes, rrfp_tp** out) {
  if (!out || R < 1 || R > TP_MAX || rank < 0 || rank >= R || part_bytes == 0)
    return rrfp_fail(RRFP_E_INVALID, "rrfp_tp_create: bad arguments (rank %d, R %d)", rank, R);
  rrfp_tp* t = new rrfp_tp();
  memset(t, 0, sizeof(*t));
  t->R = R; t->rank = rank; t->part_bytes = part_bytes;
  cudaGetDevice(&t->dev);
  RRFP_CUDA_TRY(cudaMalloc(&t->part, part_bytes));
  RRFP_CUDA_TRY(cudaMalloc(&t->board, 2 * TP_MAX * sizeof(unsigned long long)));
  RRFP_CUDA_TRY(cudaMemset(t->board, 0, 2 * TP_MAX * sizeof(unsigned long long)));
  RRFP_CUDA_TRY(cudaMalloc(&t->seq, 4 * sizeof(unsigned long long)));
  RRFP_CUDA_TRY(cudaMemset(t->seq, 0, 4 * sizeof(unsigned long long)));
  // load the kernel now (lazy module loading must never happen while a peer spins)
  cudaFuncAttributes fa;
  RRFP_CUDA_TRY(cudaFuncGetAttributes(&fa, tp_allreduce_kernel));
  RRFP_CUDA_TRY(cudaDeviceSynchronize());
  *out = t;
  return RRFP_OK;
}

extern "C" int rrfp_tp_buffers(rrfp_tp* t, void** part, void** board) {
  if (!t) return rrfp_fail(RRFP_E_INVALID, "null tp handle");
  if (part) *part = t->part;
  if (board) *board = t->board;
  return RRFP_OK;
}

extern "C" int rrfp_tp_connect(rrfp_tp* t, void* const* parts, void* const* boards) {
  if (!t || !parts || !boards) return rrfp_fail(RRFP_E_INVALID, "rrfp_tp_connect: null argument");
  for (int q = 0; q < t->R; ++q) {
    if (!parts[q] || !boards[q]) return rrfp_fail(RRFP_E_INVALID, "rrfp_tp_connect: rank %d missing", q);
    t->peer_part[q] = parts[q];
    t->peer_board[q] = (unsigned long long*)boards[q];
  }
  t->connected = true;
  return RRFP_OK;
}

// local_only != 0: no rendezvous -- out = own partial + bias + resid.  Used to
// warm up a rank's bodies eagerly (module loading of every kernel happens here,
// never while a peer spins); the sequence counter advances exactly as in the
// collective so the ranks stay in step.
extern "C" int rrfp_tp_allreduce(rrfp_tp* t, int rows, int cols, const void* bias, const void* resid,
                                 long long ld_resid, void* const* outs, int n_out, int local_only,
                                 void* stream) {
  if (!t || (!t->connected && !local_only)) return rrfp_fail(RRFP_E_INVALID, "tp group not connected");
  if (rows <= 0 || cols <= 0 || cols % 8 || (size_t)rows * cols * 2 > t->part_bytes)
    return rrfp_fail(RRFP_E_INVALID, "tp all-reduce: bad shape %dx%d", rows, cols);
  if (n_out < 1 || n_out > 4 || !outs) return rrfp_fail(RRFP_E_INVALID, "tp all-reduce: 1..4 outputs");
  if (resid && ld_resid % 8) return rrfp_fail(RRFP_E_INVALID, "tp all-reduce: residual ld %% 8");
  TpArgs a;
  memset(&a, 0, sizeof(a));
  for (int q = 0; q < t->R; ++q) {
    a.part[q] = (const __nv_bfloat16*)t->peer_part[q];
    a.board[q] = t->peer_board[q];
  }
  a.seq = t->seq;
  a.ticket = reinterpret_cast<unsigned int*>(t->seq + 1);
  a.err = reinterpret_cast<int*>(t->seq + 2);
  a.R = t->R; a.rank = t->rank;
  if (local_only) {
    memset(a.part, 0, sizeof(a.part));
    memset(a.board, 0, sizeof(a.board));
    a.part[0] = (const __nv_bfloat16*)t->part;
    a.board[0] = t->board;
    a.R = 1; a.rank = 0;
  }
  TpOuts o;
  memset(&o, 0, sizeof(o));
  for (int k = 0; k < n_out; ++k) o.out[k] = (__nv_bfloat16*)outs[k];
  o.n = n_out;
  // enough CTAs to keep ~1-2 MB of peer reads in flight, few enough that the
  // spinning CTAs never crowd out a co-resident peer's GEMM (same-GPU TP groups)
  const int grid = 64;
  RRFP_CUDA_TRY(rrfp_launch(tp_allreduce_kernel, dim3(grid), dim3(512), 0, (cudaStream_t)stream, a, o,
                            (const __nv_bfloat16*)bias, (const __nv_bfloat16*)resid, ld_resid, rows, cols));
  RRFP_CUDA_TRY(cudaGetLastError());
  return RRFP_OK;
}

// 0 ok, 1 a spin wait timed out (a peer never arrived) since creation
extern "C" int rrfp_tp_error(rrfp_tp* t, int* err) {
  if (!t || !err) return rrfp_fail(RRFP_E_INVALID, "null argument");
  int v = 0;
  RRFP_CUDA_TRY(cudaMemcpy(&v, reinterpret_cast<int*>(t->seq + 2), sizeof(int), cudaMemcpyDeviceToHost));
  *err = v;
  return RRFP_OK;
}

extern "C" void rrfp_tp_destroy(rrfp_tp* t) {
  if (!t) return;
  cudaFree(t->part);
  cudaFree(t->board);
  cudaFree(t->seq);
  delete t;
}

// ------------------------------------------------------------------------
// Cross-GPU %globaltimer calibration (wall traces from
// several GPUs on one clock, so validate_trace precedence (validate.py:117-131)
// and the breakdown can run on them).  NTP-style ping-pong between two
// single-thread kernels over peer memory: the initiator stamps t0, the
// responder answers with its own timer t_r, the initiator stamps t1;
// offset = t_r - (t0 + t1) / 2 of the round with the smallest t1 - t0.
// slot layout (u64): [0] round, [1] responder stamp.
namespace {
__global__ void clock_pingpong_kernel(unsigned long long* mine, unsigned long long* peer, int role, int rounds,
                                      unsigned long long base, long long* out) {
  if (threadIdx.x != 0) return;
  long long best_rtt = -1, best_off = 0;
  for (int i = 1; i <= rounds; ++i) {
    const unsigned long long want = base + i;
    const unsigned long long t_start = now_ns();
    if (role == 0) {
      const unsigned long long t0 = now_ns();
      st_release_sys64(&peer[0], want);
      while (ld_acquire_sys64(&mine[0]) < want) {
        if (now_ns() - t_start > 5000000000ull) { out[2] = -1; return; }
      }
      const unsigned long long t1 = now_ns();
      const long long tr = (long long)ld_acquire_sys64(&mine[1]);
      const long long rtt = (long long)(t1 - t0);
      if (best_rtt < 0 || rtt < best_rtt) { best_rtt = rtt; best_off = tr - (long long)((t0 + t1) / 2); }
    } else {
      while (ld_acquire_sys64(&mine[0]) < want) {
        if (now_ns() - t_start > 5000000000ull) { out[2] = -1; return; }
      }
      peer[1] = now_ns();
      __threadfence_system();
      st_release_sys64(&peer[0], want);
    }
  }
  out[0] = best_off;
  out[1] = best_rtt;
  out[2] = 0;
}
}  // namespace

// role 0: initiator (reference clock) -> *offset_ns = peer clock - my clock,
// *rtt_ns = best round trip; role 1: responder.  `mine` / `peer` are 16-byte
// slots (own memory / the other GPU's slot through IPC); round ids are
// base+1 .. base+rounds and must grow from call to call on a slot (both sides
// pass the same base).  Blocks until done.
extern "C" int rrfp_clock_pingpong(void* mine, void* peer, int role, int rounds, long long base,
                                   long long* offset_ns, long long* rtt_ns) {
  if (!mine || !peer || rounds < 1) return rrfp_fail(RRFP_E_INVALID, "clock ping-pong: bad arguments");
  long long* out = nullptr;
  RRFP_CUDA_TRY(cudaMalloc(&out, 3 * sizeof(long long)));
  clock_pingpong_kernel<<<1, 32>>>((unsigned long long*)mine, (unsigned long long*)peer, role, rounds,
                                   (unsigned long long)base, out);
  RRFP_CUDA_TRY(cudaGetLastError());
  long long h[3];
  RRFP_CUDA_TRY(cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost));
  cudaFree(out);
  if (h[2] != 0) return rrfp_fail(RRFP_E_CUDA, "clock ping-pong timed out (peer not running?)");
  if (offset_ns) *offset_ns = role == 0 ? h[0] : 0;
  if (rtt_ns) *rtt_ns = role == 0 ? h[1] : 0;
  return RRFP_OK;
}

// Single-process multi-GPU pipelines (GpuPipeline(devices=[...])): neighbour
// stages store into each other's mailboxes / inboxes with plain pointers, which
// needs peer access enabled in both directions (the multi-process path gets it
// from cudaIpcMemLazyEnablePeerAccess).  Idempotent.
extern "C" int rrfp_enable_peer_access(int dev, int peer) {
  if (dev == peer) return RRFP_OK;
  int can = 0;
  RRFP_CUDA_TRY(cudaDeviceCanAccessPeer(&can, dev, peer));
  if (!can) return rrfp_fail(RRFP_E_CUDA, "GPU %d cannot access GPU %d (no P2P / NVLink)", dev, peer);
  int cur = 0;
  cudaGetDevice(&cur);
  RRFP_CUDA_TRY(cudaSetDevice(dev));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) { cudaGetLastError(); e = cudaSuccess; }
  cudaSetDevice(cur);
  RRFP_CUDA_TRY(e);
  return RRFP_OK;
}
