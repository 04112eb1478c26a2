// rrfp_replay.cu -- C-ABI entry points for the arbitration twin and the
// virtual-clock replay engine (host twin + single-CTA device kernel).
//
// rrfp_replay_device runs engine.run_rrfp's tick loop (engine.py:344-362) on
// the B200: one thread per pipeline stage inside ONE CTA; each tick is two
// lock-step phases separated by __syncthreads():
//   A) completions -> sends (arrivals appended to the destination's inbox)
//   B) inbox drain, arrivals/releases/coord-ends at T, then dispatch
// which reproduces "apply every event of the tick, then dispatch touched
// stages in ascending order" because a dispatch only schedules the stage's
// own completion (engine.py:270-296) and so cannot affect another stage in
// the same tick.  The next tick is the block-wide min of the per-stage next
// event times.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <string>

#include "rrfp_core.cuh"
#include "rrfp_common.h"

// ----------------------------------------------------------- error plumbing
static thread_local std::string g_last_error;
extern "C" const char* rrfp_last_error(void) { return g_last_error.c_str(); }
int rrfp_fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}
extern "C" int rrfp_abi_version(void) { return 1; }

static int g_pdl = -1;
bool rrfp_pdl() {
  if (g_pdl < 0) {
    const char* e = getenv("RRFP_PDL");
    g_pdl = e ? atoi(e) : 1;
  }
  return g_pdl != 0;
}
extern "C" int rrfp_set_pdl(int on) {
  g_pdl = on ? 1 : 0;
  return RRFP_OK;
}

static int check_desc(const rrfp_iter_desc* d) {
  if (!d) return rrfp_fail(RRFP_E_INVALID, "null iter desc");
  if (d->N < 1 || d->N > RRFP_MAX_STAGES) return rrfp_fail(RRFP_E_INVALID, "N out of range: %d", d->N);
  if (d->R < 1 || d->R > RRFP_MAX_RANKS) return rrfp_fail(RRFP_E_INVALID, "R out of range: %d", d->R);
  if (d->C < 1 || d->C > RRFP_MAX_CHUNKS) return rrfp_fail(RRFP_E_INVALID, "C out of range: %d", d->C);
  if (d->M < 1 || d->M > RRFP_MAX_MB) return rrfp_fail(RRFP_E_INVALID, "M out of range: %d", d->M);
  if (d->MW != (d->M + 31) / 32) return rrfp_fail(RRFP_E_INVALID, "MW must be ceil(M/32)");
  if (d->C * d->MW > RRFP_MAX_WORDS) return rrfp_fail(RRFP_E_INVALID, "C*MW exceeds %d", RRFP_MAX_WORDS);
  if (d->buffer_limit < 1) return rrfp_fail(RRFP_E_INVALID, "buffer_limit must be >= 1");
  if (d->fixed_mode && d->R != 1) return rrfp_fail(RRFP_E_INVALID, "fixed mode needs R == 1");
  if (d->hint.n_ranked < 0 || d->hint.n_ranked > RRFP_MAX_RANKED)
    return rrfp_fail(RRFP_E_INVALID, "bad ranked hint length");
  return RRFP_OK;
}

// ------------------------------------------------------------ arbitration
extern "C" int rrfp_arbitrate(const rrfp_stage_state* st, const rrfp_hint* hint, rrfp_decision* out) {
  if (!st || !hint || !out) return rrfp_fail(RRFP_E_INVALID, "null argument");
  if (st->C * st->MW > RRFP_MAX_WORDS || st->MW != (st->M + 31) / 32)
    return rrfp_fail(RRFP_E_INVALID, "bad snapshot shape");
  rrfp_view_ref v;
  v.fready = st->fready; v.bready = st->bready; v.wpend = st->wpend;
  v.doneF = st->doneF; v.doneB = st->doneB; v.admission = st->admission;
  *out = rrfp_arbitrate_core(v, *hint, st->mode, st->focus, st->phase, st->M, st->C, st->MW,
                             st->decompose);
  return RRFP_OK;
}

extern "C" int rrfp_next_by_priority(const uint32_t* words, int32_t C, int32_t MW, int32_t forward,
                                     rrfp_decision* out) {
  if (!words || !out) return rrfp_fail(RRFP_E_INVALID, "null argument");
  if (C < 1 || MW < 1 || C * MW > RRFP_MAX_WORDS) return rrfp_fail(RRFP_E_INVALID, "bad set shape");
  int k = forward ? first_asc(words, C, MW) : first_desc(words, C, MW);
  *out = mk_dec(k < 0 ? RRFP_WAIT : (forward ? RRFP_DIR_F : RRFP_DIR_B), k, MW);
  return RRFP_OK;
}

extern "C" int rrfp_update_backpressure(rrfp_stage_state* st, int32_t limit, int32_t n_f, int32_t n_b) {
  if (!st) return rrfp_fail(RRFP_E_INVALID, "null argument");
  rrfp_bp_update(&st->mode, &st->focus, limit, n_f, n_b, st->doneF, st->doneB, st->M, st->C, st->MW);
  return RRFP_OK;
}

// -------------------------------------------------------------- workspace
struct ws_layout {
  size_t st, heap, mbox, nev, ctr, total;
};
static ws_layout layout_for(const rrfp_iter_desc& d) {
  ws_layout L;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = (off + bytes + 255) & ~(size_t)255; return o; };
  L.st = take(sizeof(des_stage) * d.N);
  L.heap = take(sizeof(des_hent) * (size_t)des_heap_cap(d) * d.N);
  L.mbox = take(sizeof(des_mbox) * (size_t)des_mbox_cap(d) * d.N);
  L.nev = take(sizeof(int32_t) * 4);
  L.ctr = take(sizeof(int64_t) * 4);
  L.total = off;
  return L;
}

extern "C" size_t rrfp_replay_workspace_bytes(const rrfp_iter_desc* d) {
  if (check_desc(d)) return 0;
  return layout_for(*d).total;
}
extern "C" int32_t rrfp_replay_event_capacity(const rrfp_iter_desc* d) {
  if (check_desc(d)) return 0;
  return des_event_cap(*d);
}

static des_ctx make_ctx(const rrfp_iter_desc& d, const int64_t* dur, const int64_t* comm,
                        const int64_t* skew, const rrfp_task_t* fixed, char* ws,
                        rrfp_event* events, int32_t cap) {
  ws_layout L = layout_for(d);
  des_ctx x;
  x.d = d;
  x.KEYS = d.C * d.MW * 32;
  x.heap_cap = des_heap_cap(d);
  x.mbox_cap = des_mbox_cap(d);
  x.event_cap = cap;
  x.dur = dur; x.comm = comm; x.skew = skew; x.fixed = fixed;
  x.st = (des_stage*)(ws + L.st);
  x.heap = (des_hent*)(ws + L.heap);
  x.mbox = (des_mbox*)(ws + L.mbox);
  x.events = events;
  x.n_events = (int32_t*)(ws + L.nev);
  x.counters = (int64_t*)(ws + L.ctr);
  return x;
}

RHD void fill_result(const des_ctx& x, int64_t makespan, bool deadlock, rrfp_replay_result* r) {
  bool overflow = false;
  r->makespan = makespan;
  r->agreed = x.counters[0];
  r->deferred = x.counters[1];
  for (int s = 0; s < RRFP_MAX_STAGES; ++s) {
    if (s < x.d.N) {
      const des_stage& S = x.st[s];
      r->compute[s] = S.compute; r->coord[s] = S.coord_time;
      r->n_f[s] = S.n_f; r->n_b[s] = S.n_b; r->n_w[s] = S.n_w; r->remaining[s] = S.remaining;
      overflow = overflow || S.overflow;
    } else {
      r->compute[s] = r->coord[s] = 0;
      r->n_f[s] = r->n_b[s] = r->n_w[s] = r->remaining[s] = 0;
    }
  }
  int ne = *x.n_events;
  if (ne > x.event_cap) overflow = true;
  r->n_events = ne > x.event_cap ? x.event_cap : ne;
  r->status = overflow ? RRFP_E_CAPACITY : (deadlock ? RRFP_E_DEADLOCK : RRFP_OK);
}

// ----------------------------------------------------------------- host twin
extern "C" int rrfp_replay_host(const rrfp_iter_desc* d, const int64_t* dur, const int64_t* comm,
                                const int64_t* skew, const rrfp_task_t* fixed,
                                rrfp_event* events, int32_t event_cap, rrfp_replay_result* res) {
  int rc = check_desc(d);
  if (rc) return rc;
  if (!dur || !comm || !skew || !events || !res || (d->fixed_mode && !fixed))
    return rrfp_fail(RRFP_E_INVALID, "null table pointer");
  ws_layout L = layout_for(*d);
  std::string ws(L.total, '\0');
  des_ctx x = make_ctx(*d, dur, comm, skew, fixed, &ws[0], events, event_cap);
  for (int s = 0; s < d->N; ++s) des_init_stage(x, s);
  *x.n_events = 0;
  x.counters[0] = x.counters[1] = 0;
  for (int s = 0; s < d->N; ++s) des_dispatch(x, s, 0);
  int64_t last = 0;
  while (true) {
    int64_t T = RRFP_T_INF;
    for (int s = 0; s < d->N; ++s) {
      int64_t t = des_next_time(x, s);
      if (t < T) T = t;
    }
    if (T == RRFP_T_INF) break;
    for (int s = 0; s < d->N; ++s) des_phase_a(x, s, T);
    for (int s = 0; s < d->N; ++s) des_phase_b(x, s, T);
    last = T;
  }
  bool dead = false;
  for (int s = 0; s < d->N; ++s) dead = dead || x.st[s].remaining != 0;
  fill_result(x, last, dead, res);
  if (res->status == RRFP_E_CAPACITY) return rrfp_fail(RRFP_E_CAPACITY, "replay capacity exceeded");
  if (dead) return rrfp_fail(RRFP_E_DEADLOCK, "quiescent with unfinished tasks");
  return RRFP_OK;
}

// ------------------------------------------------------------- device run
__global__ void __launch_bounds__(32, 1) rrfp_replay_kernel(des_ctx x, rrfp_replay_result* res) {
  const int s = threadIdx.x;
  const int N = x.d.N;
  if (s < N) des_init_stage(x, s);
  if (s == 0) { *x.n_events = 0; x.counters[0] = x.counters[1] = 0; }
  __syncthreads();
  if (s < N) des_dispatch(x, s, 0);
  __syncthreads();
  int64_t last = 0;
  while (true) {
    int64_t t = s < N ? des_next_time(x, s) : RRFP_T_INF;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      long long other = __shfl_xor_sync(0xffffffffu, (long long)t, o);
      t = other < t ? other : t;
    }
    if (t == RRFP_T_INF) break;
    if (s < N) des_phase_a(x, s, t);
    __syncthreads();
    if (s < N) des_phase_b(x, s, t);
    __syncthreads();
    last = t;
  }
  if (s == 0) {
    bool dead = false;
    for (int i = 0; i < N; ++i) dead = dead || x.st[i].remaining != 0;
    fill_result(x, last, dead, res);
  }
}

extern "C" int rrfp_replay_device(const rrfp_iter_desc* d, const int64_t* dur, const int64_t* comm,
                                  const int64_t* skew, const rrfp_task_t* fixed, void* workspace,
                                  rrfp_event* events, int32_t event_cap, rrfp_replay_result* res,
                                  void* stream) {
  int rc = check_desc(d);
  if (rc) return rc;
  if (!workspace || !dur || !comm || !skew || !events || !res || (d->fixed_mode && !fixed))
    return rrfp_fail(RRFP_E_INVALID, "null device pointer");
  des_ctx x = make_ctx(*d, dur, comm, skew, fixed, (char*)workspace, events, event_cap);
  rrfp_replay_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(x, res);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return rrfp_fail(RRFP_E_CUDA, "replay launch: %s", cudaGetErrorString(e));
  return RRFP_OK;
}
