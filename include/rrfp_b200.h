/*
 * rrfp_b200.h -- C ABI of the B200-native RRFP pipeline runtime
 * (arXiv 2605.18750).  Plain pointers and sizes only; no torch types.
 *
 * Every entry point replaces a function of the reference's Python
 * scheduling path (/root/reference/pkg/src/rrfp); the citation is given
 * per function.  All functions return 0 on success and a negative
 * RRFP_E_* code on failure; rrfp_last_error() returns a thread-local
 * message.  No C++ exception crosses this boundary.
 *
 * Task encoding (rrfp_task_t, uint32):
 *   bits 0-1  direction (0 = B, 1 = F, 2 = W; the reference's
 *             DISPATCH_RANK order, workload.py:37-40)
 *   bits 2-5  model chunk   (C <= 16)
 *   bits 6-15 microbatch    (M <= 1024)
 *   bits 16-21 stage        (N <= 32)
 * Keys index per-stage bitmasks: key = chunk * (32*MW) + mb, MW = ceil(M/32).
 */
#ifndef RRFP_B200_H
#define RRFP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RRFP_OK 0
#define RRFP_E_INVALID -1      /* bad argument / config (ValueError in the reference) */
#define RRFP_E_DEADLOCK -2     /* EngineDeadlockError, engine.py:62-67            */
#define RRFP_E_WATCHDOG -3     /* LiveWatchdogError, live.py:58-63                 */
#define RRFP_E_CUDA -4         /* CUDA runtime failure                             */
#define RRFP_E_CAPACITY -5     /* a device ring/heap would overflow                */
#define RRFP_E_NOGPU -6        /* no CUDA device / kernel image                    */

#define RRFP_DIR_B 0
#define RRFP_DIR_F 1
#define RRFP_DIR_W 2
#define RRFP_WAIT 3

#define RRFP_MAX_STAGES 32
#define RRFP_MAX_RANKS 8
#define RRFP_MAX_CHUNKS 16
#define RRFP_MAX_MB 1024
#define RRFP_MAX_WORDS 128     /* bitmask words per ready set: C*MW <= 128 */
#define RRFP_MAX_RANKED 8

/* hint kinds, arbitration.py:37 HINT_KINDS */
#define RRFP_HINT_BF 0
#define RRFP_HINT_FB 1
#define RRFP_HINT_BPRIO 2
#define RRFP_HINT_FPRIO 3
#define RRFP_HINT_BFW 4
#define RRFP_HINT_EXTERNAL 5

/* backpressure modes, arbitration.py:32-34 */
#define RRFP_BP_NORMAL 0
#define RRFP_BP_DRAIN 1
#define RRFP_BP_FOCUS 2

typedef uint32_t rrfp_task_t;

/* HintOrder, arbitration.py:40-66. ranked_dir uses RRFP_DIR_*, ranked_desc 1 = "desc". */
typedef struct {
  int32_t kind;
  int32_t n_ranked;
  int32_t ranked_dir[RRFP_MAX_RANKED];
  int32_t ranked_desc[RRFP_MAX_RANKED];
} rrfp_hint;

/* One (stage, rank) arbitration snapshot: StageBuffers + BackpressureState +
 * ArbiterState + StageProgress (arbitration.py:93-229) as bitmasks. */
typedef struct {
  int32_t M, C, MW, decompose;     /* shape; MW = ceil(M/32), C*MW <= RRFP_MAX_WORDS */
  int32_t admission;               /* next chunk-0 mb at stage 0, or -1 */
  int32_t mode, focus;             /* RRFP_BP_*, focus microbatch (-1) */
  int32_t phase;                   /* next direction to probe: RRFP_DIR_F/B, or -1 = round start */
  uint32_t fready[RRFP_MAX_WORDS];
  uint32_t bready[RRFP_MAX_WORDS];
  uint32_t wpend[RRFP_MAX_WORDS];
  uint32_t doneF[RRFP_MAX_WORDS];
  uint32_t doneB[RRFP_MAX_WORDS];
} rrfp_stage_state;

typedef struct {
  int32_t kind;                    /* RRFP_DIR_B/F/W or RRFP_WAIT */
  int32_t mb, chunk;
} rrfp_decision;

/* ---- arbitration twin -------------------------------------------------- */

/* arbitrate + _weight_fallback, arbitration.py:232-303.  Pure.  The same
 * __host__ __device__ code runs inside the device dispatcher. */
int rrfp_arbitrate(const rrfp_stage_state* st, const rrfp_hint* hint, rrfp_decision* out);

/* next_by_priority, arbitration.py:119-129: the first key of a chunk-major
 * set (C*MW words) in forward order min(chunk, mb) (forward = 1) or backward
 * order min(-chunk, mb) (forward = 0); kind RRFP_WAIT if the set is empty. */
int rrfp_next_by_priority(const uint32_t* words, int32_t C, int32_t MW, int32_t forward, rrfp_decision* out);

/* update_backpressure, arbitration.py:188-215.  In/out on mode/focus. */
int rrfp_update_backpressure(rrfp_stage_state* st, int32_t limit, int32_t n_f, int32_t n_b);

/* ---- replay engine (virtual clock) --------------------------------------- */

/* Static description of one iteration plus the host-built tables
 * (Workload.latency + build_injection_table, CommDelay.sample, TP skew).
 * All int64 tables are microseconds.  Index helpers:
 *   dur  [((s*3 + dir) * KEYS) + key]          latency + injected delay
 *   comm [((s*2 + dir) * KEYS) + key]          delay of the message SENT by task (s,dir,key), dir in {B,F}
 *   skew [(((s*2 + dir) * KEYS) + key) * R + r] arrival skew of message TO task (s,dir,key) at rank r
 *   fixed[s * per_stage + i]                   FIXED-mode order (rrfp_task_t)
 * KEYS = C * MW * 32.
 */
typedef struct {
  int32_t N, M, C, R, MW, decompose;
  int32_t buffer_limit;
  int32_t fixed_mode;              /* 0 = RRFP arbitration, 1 = fixed per-stage order */
  int32_t per_stage;               /* tasks per stage = M*C*(2 or 3) */
  int32_t pad0;
  int64_t coord_cost;              /* TpGroup.coordination_round_cost */
  rrfp_hint hint;
} rrfp_iter_desc;

/* One trace record.  kind: 0 exec, 1 send, 2 recv, 3 coord(agreed), 4 coord(deferred). */
typedef struct {
  int64_t t0, t1;
  int32_t kind, stage, rank;
  rrfp_task_t task;
} rrfp_event;

typedef struct {
  int64_t makespan;
  int64_t agreed, deferred;
  int32_t status;                  /* RRFP_OK / RRFP_E_DEADLOCK / RRFP_E_CAPACITY */
  int32_t n_events;
  int64_t compute[RRFP_MAX_STAGES];
  int64_t coord[RRFP_MAX_STAGES];
  int32_t n_f[RRFP_MAX_STAGES], n_b[RRFP_MAX_STAGES], n_w[RRFP_MAX_STAGES];
  int32_t remaining[RRFP_MAX_STAGES];
} rrfp_replay_result;

/* Device workspace bytes for one replay of this shape. */
size_t rrfp_replay_workspace_bytes(const rrfp_iter_desc* d);
/* Max trace records a replay of this shape can emit. */
int32_t rrfp_replay_event_capacity(const rrfp_iter_desc* d);

/* engine.run_rrfp / baselines.run_fixed semantics (engine.py:344-367,
 * baselines.py:94-172) on the CPU, using the same __host__ __device__
 * state machine as the device kernel.  Host pointers. */
int rrfp_replay_host(const rrfp_iter_desc* d, const int64_t* dur, const int64_t* comm,
                     const int64_t* skew, const rrfp_task_t* fixed,
                     rrfp_event* events, int32_t event_cap, rrfp_replay_result* res);

/* The same replay as ONE device kernel (one CTA, one thread per stage,
 * lockstep ticks).  All table/event/workspace pointers are DEVICE
 * pointers; res is a device pointer.  Enqueued on `stream` (cudaStream_t). */
int rrfp_replay_device(const rrfp_iter_desc* d, const int64_t* dur, const int64_t* comm,
                       const int64_t* skew, const rrfp_task_t* fixed, void* workspace,
                       rrfp_event* events, int32_t event_cap, rrfp_replay_result* res,
                       void* stream);

/* ---- free-running device runtime (live.run_live replacement) ------------ */

typedef struct rrfp_runtime rrfp_runtime;

/* Per-stage executor description (one per (stage, rank) lane).  */
typedef struct {
  int32_t N, M, C, R, MW, decompose;
  int32_t buffer_limit;
  int32_t fixed_mode;              /* 0 = arbitrate (FREE), 1 = follow order list (FIXED / replay) */
  int32_t per_stage;
  int32_t stage, rank;
  int32_t device;                  /* CUDA ordinal */
  int32_t compute_kind;            /* 0 = spin tasks (latency table), 1 = caller body graphs */
  int32_t trace_cap;
  double time_scale;               /* live.run_live time_scale */
  int64_t coord_cost_ns;
  rrfp_hint hint;
  /* virtual_clock = 1: replay mode.  The lane makes EVERY decision itself
   * (rrfp_arbitrate_core + the K4 TP round) at the reference engine's
   * virtual times (engine.py:298-367): messages carry their virtual arrival
   * time (end + comm delay + rank skew, engine.py:211-221), each lane
   * publishes a lower bound on the virtual time of its future sends, and a
   * lane processes tick T only when every in-neighbour's bound exceeds T
   * (conservative parallel discrete-event simulation).  Tables are then in
   * integer microseconds (virtual), trace records carry virtual times.
   * v_dmin = the stage's smallest task duration, v_la = the smallest
   * comm delay + skew of the lane's sends (v_dmin + v_la >= 1 for progress),
   * v_horizon = an upper bound of the makespan (beyond it: deadlock). */
  int32_t virtual_clock;
  int32_t declog_cap;              /* > 0: log every arbitration (inputs + decision), records */
  int64_t v_dmin, v_la, v_horizon;
} rrfp_lane_desc;

int rrfp_runtime_create(const rrfp_lane_desc* desc, rrfp_runtime** out);
void rrfp_runtime_destroy(rrfp_runtime* rt);
/* Device address of this lane's inbox block (flags + visible-at stamps), to be
 * exported to peers (same process: plain pointer; other process: CUDA IPC). */
int rrfp_runtime_inbox(rrfp_runtime* rt, void** dev_ptr, size_t* bytes);
/* CUDA IPC handle (64 bytes) of the inbox allocation. */
int rrfp_runtime_inbox_ipc(rrfp_runtime* rt, void* handle64);
/* Open a peer's IPC handle; returns a device pointer usable in this process. */
int rrfp_ipc_open(const void* handle64, void** dev_ptr);
/* Unmap a pointer returned by rrfp_ipc_open (every opener closes before its peer's
 * next allocation can be opened again). */
int rrfp_ipc_close(void* dev_ptr);
/* cudaMalloc'd (IPC-exportable) buffer for mailbox slots; handle of such a buffer. */
int rrfp_ipc_alloc(size_t bytes, void** dev_ptr);
int rrfp_ipc_handle(void* dev_ptr, void* handle64);
void rrfp_ipc_free(void* dev_ptr);

/* ---- tensor-parallel group of one pipeline stage (csrc/tp.cu; BASELINE config 3) ----
 * Replaces the reference's TP collective step that follows tp_coordinate
 * (arbitration.py:323-334; live.py:246-277 resolves the group, the collective
 * itself is the Megatron all-reduce the paper times).
 * Each rank owns a partial buffer (row-parallel GEMM output) and a flag board;
 * rrfp_tp_allreduce sums the R partials in rank order over peer memory, fuses
 * bias + residual, and writes up to 4 destinations; replayable in CUDA graphs. */
typedef struct rrfp_tp rrfp_tp;
int rrfp_tp_create(int rank, int R, size_t part_bytes, rrfp_tp** out);
/* own partial buffer and flag board (cudaMalloc'd: export with rrfp_ipc_handle) */
int rrfp_tp_buffers(rrfp_tp* t, void** part, void** board);
/* every rank's partial and board, indexed by TP rank (own included; peer pointers ok) */
int rrfp_tp_connect(rrfp_tp* t, void* const* parts, void* const* boards);
/* local_only: no rendezvous (out = own partial + bias + resid) -- eager warm-up */
int rrfp_tp_allreduce(rrfp_tp* t, int rows, int cols, const void* bias, const void* resid,
                      long long ld_resid, void* const* outs, int n_out, int local_only, void* stream);
/* *err = 1 if a peer wait timed out (20 s) since creation */
int rrfp_tp_error(rrfp_tp* t, int* err);
void rrfp_tp_destroy(rrfp_tp* t);

/* Cross-GPU %globaltimer calibration for wall traces (replaces the single
 * process clock the reference's validate_trace assumes, validate.py:117-131):
 * NTP-style ping-pong over peer memory between two ranks' 16-byte slots
 * (cudaMalloc'd, IPC-exchanged).  role 0 (initiator) returns offset = peer
 * clock - own clock and the best round trip; role 1 responds.  Round ids are
 * base+1..base+rounds, growing across calls on a slot.  Blocking. */
int rrfp_clock_pingpong(void* mine, void* peer, int role, int rounds, long long base, long long* offset_ns,
                        long long* rtt_ns);
/* One process driving several GPUs (GpuPipeline(devices=[...])): enable dev -> peer
 * access for the neighbours' plain-pointer mailbox / inbox stores.  Idempotent. */
int rrfp_enable_peer_access(int dev, int peer);
/* Single-GPU pipeline emulation: n disjoint SM partitions (green contexts) of
 * >= min_sms SMs; two streams per partition in streams[2i], streams[2i+1]. */
int rrfp_green_streams(int device, int n, int min_sms, void** streams, int* sms);
/* Destroy the 2n streams and n green contexts rrfp_green_streams returned
 * (streams as returned, after the caller synchronised them). */
int rrfp_green_destroy(void* const* streams, int n);
/* Wire neighbours: inbox of the lanes that receive this lane's F output
 * (next stage, all R ranks) and B output (previous stage, all R ranks), and
 * the TP group's agreement board slots.  Pointers may be peer pointers. */
int rrfp_runtime_connect(rrfp_runtime* rt, void* const* fwd_dst_inboxes, void* const* bwd_dst_inboxes,
                         void* const* tp_peer_inboxes);
/* Load host tables (per-lane): dur_ns[3*KEYS] (spin length incl. injected
 * delay; with caller bodies: the additive jitter pad), comm_ns[2*KEYS] (flag
 * visibility delay of sent messages), skew_ns[2*KEYS*R] (arrival skew per
 * destination rank), fixed order, min_ns[3*KEYS] (optional task floor:
 * end >= start + min_ns, the lognormal compute jitter).  May be reloaded
 * between iterations. */
int rrfp_runtime_load_tables(rrfp_runtime* rt, const int64_t* dur_ns, const int64_t* comm_ns,
                             const int64_t* skew_ns, const rrfp_task_t* fixed, const int64_t* min_ns);
/* Register caller-captured compute bodies: graphs[kind * M*C + chunk * M + mb]
 * is the cudaGraph_t run for task (kind, mb, chunk) (kind: 0 = B, 1 = F, 2 = W;
 * NULL = no work), n = 3 * M * C.  The dispatcher selects the branch with
 * cudaGraphSetConditional.  Must be called before the first launch. */
int rrfp_runtime_set_bodies(rrfp_runtime* rt, void* const* graphs, int32_t n);
int rrfp_runtime_task_ptr(rrfp_runtime* rt, void** dev_ptr);
/* Build, instantiate and upload the lane graph (call for every lane of the job
 * before the first launch of any lane). */
int rrfp_runtime_prepare(rrfp_runtime* rt, void* stream);
/* Build (first call) and launch one iteration's executor graph on the lane's
 * stream; epoch must increase by one per iteration. Asynchronous. */
int rrfp_runtime_launch(rrfp_runtime* rt, int64_t epoch, void* stream);
/* Wait for the lane to finish (host poll with watchdog); copies the trace. */
int rrfp_runtime_wait(rrfp_runtime* rt, double watchdog_secs, rrfp_event* events, int32_t cap,
                      int32_t* n_events, int64_t* t0_ns);
int rrfp_runtime_status(rrfp_runtime* rt, char* dump, size_t cap);
/* Decision log of the last iteration (desc.declog_cap > 0): one record per
 * arbitration the lane evaluated, uint32 words, stride = 16 + 5*nwords:
 *   [0] stage [1] rank [2] n_f [3] n_b [4] bp mode before update_backpressure
 *   [5] focus before [6] mode after [7] focus after [8] phase (-1/B/F)
 *   [9] admission (-1) [10] decision kind [11] mb [12] chunk [13] nwords
 *   [14..15] time (virtual us, or %globaltimer ns in free mode)
 *   then fready, bready, wpend, doneF, doneB (nwords each, chunk-major keys).
 * The inputs are exactly what rrfp_arbitrate_core saw, so the host can
 * re-evaluate each decision with the reference's arbitrate (tests/). */
int rrfp_runtime_declog(rrfp_runtime* rt, uint32_t* out, int32_t cap_words, int32_t* n_records,
                        int32_t* stride_words);

/* Dispatcher profile (free mode): cap > 0 records, for the next iterations,
 * one record per lane_step_kernel run: uint64 {entry, completion done, decision
 * made (%globaltimer ns), kind << 32 | view polls}; cap = 0 disables.  (ncu does
 * not profile kernel nodes of graphs with conditional nodes.) */
int rrfp_runtime_profile(rrfp_runtime* rt, int32_t cap);
int rrfp_runtime_profile_read(rrfp_runtime* rt, uint64_t* out, int32_t cap, int32_t* n_records);

/* ---- stage-compute kernel entry points (unit-test surface) ------------- */

/* Stage GEMM (tcgen05/TMA, csrc/gemm_sm100.cu): C[M,N] = sum_k A(m,k) B(n,k),
 * A(m,k) = a_mn ? A[k*lda+m] : A[m*lda+k], B(n,k) = b_mn ? B[k*ldb+n] : B[n*ldb+k];
 * epi: 0 bf16 (+bias), 1 bias+GELU (C=pre, C2=gelu), 2 +bias+R, 3 f32 (+)=,
 * 4 *gelu'(R), 5 f32.  Replaces the timed no-op compute (engine.py:272-273). */
int rrfp_gemm_bf16(int epi, int a_mn, int b_mn, int M, int N, int K, const void* A, long long lda,
                   const void* B, long long ldb, void* C, long long ldc, void* C2, long long ldc2,
                   const void* bias, const void* R, long long ldr, int accumulate, void* stream);
int rrfp_gemm_set_variant(int pair);
/* Programmatic dependent launch for the stage kernels (default on; env RRFP_PDL=0 disables). */
int rrfp_set_pdl(int on);
int rrfp_gemm_reserve_sms(int n);
/* 1 = smem-staged TMA store / reduce-add epilogue (default; outputs on a peer GPU
 * use staged coalesced st.global), 0 = per-thread global stores, 2 = force the
 * staged coalesced st.global path for every bf16 output (test hook). */
int rrfp_gemm_set_epilogue(int tma_store);
/* 1 = stream-K split of the last partial round of 256x256 tiles over all CTA pairs (default 0). */
int rrfp_gemm_set_streamk(int on);
/* 1 (default): the last partial wave of 256x256 output tiles runs as 256x128
   halves when they fit in one round of CTA pairs; 0: plain waves. */
int rrfp_gemm_set_tail_split(int on);
/* 1 (default): clusters of two CTA pairs on adjacent N tiles, A multicast
   between them (N tile count even, no SM cap); 0: one CTA pair per cluster. */
int rrfp_gemm_set_multicast(int on);
/* Co-resident clusters of the pair GEMM kernel (mc = 1: CTA pairs, 2: two
   pairs); the persistent grid is capped to it.  < 0: error. */
int rrfp_gemm_max_clusters(int mc);
/* pair-kernel k-block depth: 64 (6-stage ring, default) or 128 (3 stages). */
int rrfp_gemm_set_bk(int bk);
/* GEMMs whose 256x256 tiles fill less than one wave of CTA pairs (bit mask,
   default 0 -- both modes measured slower; env RRFP_GEMM_SMALL): 1 = f32-accumulate outputs stream-K over
   every pair (each k-segment reduce-adds its partial tile), 2 = other outputs
   as 256x128 halves. */
int rrfp_gemm_set_small(int mode);
/* 1 (default): the bf16 epilogues load R (residual / GELU pre-activation) one
   32-column chunk ahead; 0: where used. */
int rrfp_gemm_set_rpref(int on);
/* LayerNorm / embedding / bias-grad / softmax cross-entropy (csrc/ops.cu). */
int rrfp_layernorm_fwd(const void* x, const void* g, const void* b, void* y, float* mean, float* rstd,
                       int rows, int D, float eps, void* stream);
/* layernorm_bwd: dx = NULL computes only the parameter gradients (dg, db += ...). */
int rrfp_layernorm_bwd(const void* dy, const void* x, const float* mean, const float* rstd,
                       const void* g, const void* dres, void* dx, float* dg, float* db, int rows,
                       int D, void* stream);
/* layernorm_bwd_fused: one pass over a slab of rows per CTA computing any of
   dx (+ dres), the parameter gradients dg/db (+=) and the column sums
   cs_res += sum_r dres, cs_dx += sum_r dx (the bias gradients of the linear
   layers on either side of the residual); NULL skips an output.  D <= 4096. */
int rrfp_layernorm_bwd_fused(const void* dy, const void* x, const float* mean, const float* rstd,
                             const void* g, const void* dres, void* dx, float* dg, float* db,
                             float* cs_res, float* cs_dx, int rows, int D, void* stream);
int rrfp_embedding_fwd(const int32_t* tok, const void* E, const void* P, void* x, int rows, int D,
                       void* stream);
int rrfp_embedding_bwd(const int32_t* tok, const void* dx, float* dE, float* dP, int rows, int D,
                       void* stream);
int rrfp_bias_grad(const void* dy, long long ld, float* db, int rows, int cols, void* stream);
int rrfp_copy_rows(void* dst, long long ldd_bytes, const void* src, long long lds_bytes, int rows,
                   long long width_bytes, void* stream);
/* Cross-entropy forward from the LM-head GEMM's softmax statistics (rrfp_gemm_bf16
   epilogue 6, EPI_BF16_LSE: float2 (max, sum exp) per row and 128-column slot,
   ldp float2 per row): lse[r], loss[r] = lse - logits[r, target[r]].  Replaces
   rrfp_xent_fwd's pass over the logits. */
int rrfp_xent_combine(const void* part, long long ldp, int slots, const void* logits, long long ld,
                      const int32_t* target, int rows, float* loss, float* lse, void* stream);
int rrfp_xent_fwd(const void* logits, long long ld, const int32_t* target, int rows, int V,
                  float* loss, float* lse, void* stream);
int rrfp_xent_bwd(void* logits, long long ld, const int32_t* target, int rows, int V,
                  const float* lse, float scale, void* stream);

/* Attention core of the stage bodies (csrc/fmha_sm100.cu; fills the
 * compute slot of engine.py:272-273 / live.py:388-390).  tcgen05 flash attention,
 * d_head = 128, T a multiple of 128.  qkv: packed [T, ldqkv] bf16 with Q, K, V of
 * head h at columns h*128, D + h*128, 2D + h*128 (D = H*128); o: [T, ldo] bf16
 * (head h at columns h*128); lse: fp32 [H, lse_ld], the natural-log logsumexp of
 * each row of scaled scores. */
int rrfp_attn_fwd(const void* qkv, long long ldqkv, void* o, long long ldo, float* lse,
                  long long lse_ld, int T, int H, int d_head, int causal, float scale, void* stream);
/* Attention backward (csrc/fmha_sm100.cu): dQ, dK, dV of the forward above written
 * into the packed dqkv [T, lddqkv] (same column layout as qkv); o / dout [T, ld*] bf16,
 * lse the forward's statistics; workspace of rrfp_attn_bwd_workspace_bytes(T, H)
 * device bytes (fp32 dQ accumulator + per-row vectors), owned by the caller. */
size_t rrfp_attn_bwd_workspace_bytes(int T, int H);
int rrfp_attn_bwd(const void* qkv, long long ldqkv, const void* o, long long ldo, const void* dout,
                  long long lddo, const float* lse, long long lse_ld, void* dqkv, long long lddqkv,
                  void* workspace, int T, int H, int d_head, int causal, float scale, void* stream);
/* test hook: log the forward's event timeline of CTA `cta` ([4][512] int64), NULL: off */
int rrfp_attn_debug(long long* buf, int cta);

/* Synthetic spin task: busy-wait `ns` on the device (%globaltimer). */
int rrfp_spin(int64_t ns, void* stream);

const char* rrfp_last_error(void);
int rrfp_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif
