// rrfp_core.cuh -- the RRFP decision layer and virtual-clock replay engine as
// __host__ __device__ code.  The same source is compiled into the host twin
// (rrfp_arbitrate / rrfp_replay_host) and into the device kernels
// (replay kernel, free-running dispatcher), so CPU parity of the host twin
// against the reference carries over to the device by construction and is
// re-checked on the B200 by tests/test_gpu_*.py.
//
// Reference semantics (/root/reference/pkg/src/rrfp):
//   next_by_priority   arbitration.py:119-129   -> first_*() over ordered bitmasks
//   update_backpressure arbitration.py:188-215  -> rrfp_bp_update()
//   arbitrate/_weight_fallback arbitration.py:232-303 -> rrfp_arbitrate_core()
//   advance_round_phase arbitration.py:306-320  -> rrfp_advance_phase()
//   engine._Run (send/arrival/complete/commit/dispatch/run) engine.py:150-367
//                                              -> des_* below
//   baselines.run_fixed  baselines.py:94-172   -> fixed_mode dispatch
#pragma once
#include <stdint.h>
#include "../../include/rrfp_b200.h"

#ifdef __CUDACC__
#define RHD __host__ __device__ __forceinline__
#else
#define RHD inline
#endif

// ------------------------------------------------------------------ tasks --
RHD rrfp_task_t rrfp_make_task(int dir, int stage, int mb, int chunk) {
  return (rrfp_task_t)((dir & 3) | ((chunk & 15) << 2) | ((mb & 1023) << 6) | ((stage & 63) << 16));
}
RHD int rrfp_task_dir(rrfp_task_t t) { return (int)(t & 3u); }
RHD int rrfp_task_chunk(rrfp_task_t t) { return (int)((t >> 2) & 15u); }
RHD int rrfp_task_mb(rrfp_task_t t) { return (int)((t >> 6) & 1023u); }
RHD int rrfp_task_stage(rrfp_task_t t) { return (int)((t >> 16) & 63u); }
#define RRFP_NO_TASK 0xFFFFFFFFu

RHD int rrfp_key(int mb, int chunk, int MW) { return chunk * MW * 32 + mb; }
RHD int rrfp_key_mb(int key, int MW) { return key % (MW * 32); }
RHD int rrfp_key_chunk(int key, int MW) { return key / (MW * 32); }

RHD bool bit_get(const uint32_t* w, int k) { return (w[k >> 5] >> (k & 31)) & 1u; }
RHD void bit_set(uint32_t* w, int k) { w[k >> 5] |= (1u << (k & 31)); }
RHD void bit_clr(uint32_t* w, int k) { w[k >> 5] &= ~(1u << (k & 31)); }

RHD int rrfp_ffs(uint32_t x) {
#ifdef __CUDA_ARCH__
  return __ffs(x) - 1;
#else
  return __builtin_ffs((int)x) - 1;
#endif
}

// first set key in words [lo, hi) (key order == chunk-major, then mb)
RHD int first_set(const uint32_t* w, int lo, int hi) {
  for (int i = lo; i < hi; ++i)
    if (w[i]) return i * 32 + rrfp_ffs(w[i]);
  return -1;
}

// min (chunk, mb) over a set (forward order, or backward "asc" rule)
RHD int first_asc(const uint32_t* w, int C, int MW) { return first_set(w, 0, C * MW); }
// min (-chunk, mb) over a set (backward order, weight order, forward "desc")
RHD int first_desc(const uint32_t* w, int C, int MW) {
  for (int c = C - 1; c >= 0; --c) {
    int k = first_set(w, c * MW, (c + 1) * MW);
    if (k >= 0) return k;
  }
  return -1;
}
RHD bool any_set(const uint32_t* w, int nwords) {
  for (int i = 0; i < nwords; ++i)
    if (w[i]) return true;
  return false;
}

// forward candidates = fready U {admission (mb, chunk 0)}; arbitration.py:109-113
RHD int fcand_first(const uint32_t* fready, int admission, int C, int MW, bool desc) {
  int k = desc ? first_desc(fready, C, MW) : first_asc(fready, C, MW);
  if (admission < 0) return k;
  int ka = rrfp_key(admission, 0, MW);
  if (k < 0) return ka;
  int kc = rrfp_key_chunk(k, MW), km = rrfp_key_mb(k, MW);
  if (!desc) {  // (chunk, mb): admission has chunk 0
    if (kc > 0 || admission < km) return ka;
    return k;
  }
  // (-chunk, mb): admission only wins against chunk-0 entries
  if (kc == 0 && admission < km) return ka;
  return k;
}

// ----------------------------------------------------------- arbitration --
RHD bool mb_finished(const uint32_t* doneF, const uint32_t* doneB, int mb, int C, int MW) {
  for (int c = 0; c < C; ++c) {
    int k = rrfp_key(mb, c, MW);
    if (!bit_get(doneF, k) || !bit_get(doneB, k)) return false;
  }
  return true;
}

// next_in_completion_order: F_0..F_{C-1}, B_{C-1}..B_0 (arbitration.py:174-185)
RHD void next_step(const uint32_t* doneF, const uint32_t* doneB, int mb, int C, int MW, int* dir,
                   int* chunk) {
  for (int c = 0; c < C; ++c)
    if (!bit_get(doneF, rrfp_key(mb, c, MW))) { *dir = RRFP_DIR_F; *chunk = c; return; }
  for (int c = C - 1; c >= 0; --c)
    if (!bit_get(doneB, rrfp_key(mb, c, MW))) { *dir = RRFP_DIR_B; *chunk = c; return; }
  *dir = RRFP_WAIT;
  *chunk = -1;
}

// update_backpressure (arbitration.py:188-215).  lead = n_f - n_b.
RHD void rrfp_bp_update(int32_t* mode, int32_t* focus, int limit, int n_f, int n_b,
                        const uint32_t* doneF, const uint32_t* doneB, int M, int C, int MW) {
  if (n_f - n_b < limit) { *mode = RRFP_BP_NORMAL; *focus = -1; return; }
  if (C == 1) { *mode = RRFP_BP_DRAIN; *focus = -1; return; }
  int f = *focus;
  if (*mode != RRFP_BP_FOCUS || f < 0 || mb_finished(doneF, doneB, f, C, MW)) {
    f = -1;
    for (int j = 0; j < M; ++j)
      if (!mb_finished(doneF, doneB, j, C, MW)) { f = j; break; }
    if (f < 0) { *mode = RRFP_BP_NORMAL; *focus = -1; return; }
  }
  *mode = RRFP_BP_FOCUS;
  *focus = f;
}

struct rrfp_view_ref {       // pointers into one rank's view + stage-shared sets
  const uint32_t* fready;
  const uint32_t* bready;
  const uint32_t* wpend;
  const uint32_t* doneF;
  const uint32_t* doneB;
  int admission;
};

RHD rrfp_decision mk_dec(int kind, int key, int MW) {
  rrfp_decision d;
  d.kind = kind;
  d.mb = key < 0 ? -1 : rrfp_key_mb(key, MW);
  d.chunk = key < 0 ? -1 : rrfp_key_chunk(key, MW);
  return d;
}

RHD rrfp_decision weight_fallback(const rrfp_view_ref& v, int C, int MW, int dec) {
  if (dec) {
    int k = first_desc(v.wpend, C, MW);
    if (k >= 0) return mk_dec(RRFP_DIR_W, k, MW);
  }
  return mk_dec(RRFP_WAIT, -1, MW);
}

// arbitrate (arbitration.py:232-294) over one rank's view; pure.
RHD rrfp_decision rrfp_arbitrate_core(const rrfp_view_ref& v, const rrfp_hint& h, int mode,
                                      int focus, int phase, int M, int C, int MW, int dec) {
  (void)M;
  if (mode == RRFP_BP_DRAIN) {
    int k = first_desc(v.bready, C, MW);
    return mk_dec(k >= 0 ? RRFP_DIR_B : RRFP_WAIT, k, MW);
  }
  if (mode == RRFP_BP_FOCUS) {
    int dir, c;
    next_step(v.doneF, v.doneB, focus, C, MW, &dir, &c);
    if (dir == RRFP_WAIT) return mk_dec(RRFP_WAIT, -1, MW);
    int k = rrfp_key(focus, c, MW);
    if (dir == RRFP_DIR_F) {
      bool present = bit_get(v.fready, k) || (c == 0 && v.admission == focus);
      return mk_dec(present ? RRFP_DIR_F : RRFP_WAIT, present ? k : -1, MW);
    }
    bool present = bit_get(v.bready, k);
    return mk_dec(present ? RRFP_DIR_B : RRFP_WAIT, present ? k : -1, MW);
  }
  if (h.kind == RRFP_HINT_EXTERNAL) {
    for (int i = 0; i < h.n_ranked; ++i) {
      int d = h.ranked_dir[i];
      bool desc = h.ranked_desc[i] != 0;
      int k;
      if (d == RRFP_DIR_F) k = fcand_first(v.fready, v.admission, C, MW, desc);
      else if (d == RRFP_DIR_B) k = desc ? first_desc(v.bready, C, MW) : first_asc(v.bready, C, MW);
      else k = dec ? first_desc(v.wpend, C, MW) : -1;
      if (k >= 0) return mk_dec(d, k, MW);
    }
    return weight_fallback(v, C, MW, dec);
  }
  int first, second;
  if (h.kind == RRFP_HINT_BPRIO) { first = RRFP_DIR_B; second = RRFP_DIR_F; }
  else if (h.kind == RRFP_HINT_FPRIO) { first = RRFP_DIR_F; second = RRFP_DIR_B; }
  else {
    first = phase >= 0 ? phase : (h.kind == RRFP_HINT_FB ? RRFP_DIR_F : RRFP_DIR_B);
    second = first == RRFP_DIR_F ? RRFP_DIR_B : RRFP_DIR_F;
  }
  int order[2] = {first, second};
  for (int i = 0; i < 2; ++i) {
    int k = order[i] == RRFP_DIR_B ? first_desc(v.bready, C, MW)
                                   : fcand_first(v.fready, v.admission, C, MW, false);
    if (k >= 0) return mk_dec(order[i], k, MW);
  }
  return weight_fallback(v, C, MW, dec);
}

// advance_round_phase (arbitration.py:306-320); phase -1 == "" (round start)
RHD void rrfp_advance_phase(int32_t* phase, const rrfp_hint& h, int kind) {
  if (h.kind != RRFP_HINT_BF && h.kind != RRFP_HINT_FB && h.kind != RRFP_HINT_BFW) return;
  if (kind == RRFP_DIR_B) *phase = RRFP_DIR_F;
  else if (kind == RRFP_DIR_F) *phase = RRFP_DIR_B;
  else *phase = -1;
}

// ------------------------------------------------------- replay engine ---
// Event heap entry (arrivals and send-release touches); COMPLETE and
// COORD_END are at most one per stage and kept as scalars.
struct des_hent {
  int64_t time;
  int32_t kind;          // 0 arrival, 1 release
  int32_t rank;
  rrfp_task_t task;
  int32_t pad;
};
struct des_mbox {
  int64_t time;
  int32_t rank;
  rrfp_task_t task;
};

struct des_stage {
  int64_t busy_until, coord_until, compute, coord_time;
  int64_t complete_time;            // -1: nothing running
  int64_t coord_end_time;           // -1: none pending
  rrfp_task_t complete_task;
  int32_t awaiting, remaining, n_w, n_f, n_b, next_adm, fixed_head, touched;
  int32_t mode, focus, phase;
  int32_t heap_n, mbox_n, mbox_drained, overflow, pad;
  uint32_t doneF[RRFP_MAX_WORDS], doneB[RRFP_MAX_WORDS], wpend[RRFP_MAX_WORDS];
  uint32_t fready[RRFP_MAX_RANKS][RRFP_MAX_WORDS];
  uint32_t bready[RRFP_MAX_RANKS][RRFP_MAX_WORDS];
  uint32_t pend[RRFP_MAX_RANKS][RRFP_MAX_WORDS];
};

struct des_ctx {
  rrfp_iter_desc d;
  int KEYS, heap_cap, mbox_cap, event_cap;
  const int64_t* dur;
  const int64_t* comm;
  const int64_t* skew;
  const rrfp_task_t* fixed;
  des_stage* st;          // [N]
  des_hent* heap;         // [N][heap_cap]
  des_mbox* mbox;         // [N][mbox_cap]
  rrfp_event* events;
  int32_t* n_events;
  int64_t* counters;      // [0] agreed, [1] deferred
};

RHD int des_heap_cap(const rrfp_iter_desc& d) {
  int keys = d.C * d.M;
  return (2 * d.R + 2) * keys + 8;
}
RHD int des_mbox_cap(const rrfp_iter_desc& d) { return 2 * d.R * d.C * d.M + 8; }
RHD int des_event_cap(const rrfp_iter_desc& d) {
  int keys = d.C * d.M;
  // exec R*3K + send 2K + recv 2RK + coord (<= one per arrival + per task)
  return d.N * (3 * d.R + 2 + 2 * d.R + 2 * d.R + 4) * keys + 64;
}

RHD int32_t atomic_inc(int32_t* p) {
#ifdef __CUDA_ARCH__
  return atomicAdd(p, 1);
#else
  return (*p)++;
#endif
}

RHD void atomic_add64(int64_t* p, int64_t v) {
#ifdef __CUDA_ARCH__
  atomicAdd((unsigned long long*)p, (unsigned long long)v);
#else
  *p += v;
#endif
}

RHD void des_emit(des_ctx& x, int kind, int64_t t0, int64_t t1, int stage, int rank,
                  rrfp_task_t task) {
  int i = atomic_inc(x.n_events);
  if (i < x.event_cap) {
    rrfp_event& e = x.events[i];
    e.t0 = t0; e.t1 = t1; e.kind = kind; e.stage = stage; e.rank = rank; e.task = task;
  }
}

RHD void heap_push(des_ctx& x, int s, const des_hent& e) {
  des_stage& S = x.st[s];
  des_hent* h = x.heap + (size_t)s * x.heap_cap;
  if (S.heap_n >= x.heap_cap) { S.overflow = 1; return; }
  int i = S.heap_n++;
  while (i > 0) {
    int p = (i - 1) >> 1;
    if (h[p].time <= e.time) break;
    h[i] = h[p];
    i = p;
  }
  h[i] = e;
}
RHD des_hent heap_pop(des_ctx& x, int s) {
  des_stage& S = x.st[s];
  des_hent* h = x.heap + (size_t)s * x.heap_cap;
  des_hent top = h[0];
  des_hent last = h[--S.heap_n];
  int i = 0, n = S.heap_n;
  while (true) {
    int l = 2 * i + 1;
    if (l >= n) break;
    int c = (l + 1 < n && h[l + 1].time < h[l].time) ? l + 1 : l;
    if (h[c].time >= last.time) break;
    h[i] = h[c];
    i = c;
  }
  if (n > 0) h[i] = last;
  return top;
}

RHD int64_t tbl_dur(const des_ctx& x, int s, int dir, int key) {
  return x.dur[((size_t)s * 3 + dir) * x.KEYS + key];
}

RHD void des_init_stage(des_ctx& x, int s) {
  const rrfp_iter_desc& d = x.d;
  des_stage& S = x.st[s];
  S.busy_until = S.coord_until = S.compute = S.coord_time = 0;
  S.complete_time = -1; S.coord_end_time = -1; S.complete_task = RRFP_NO_TASK;
  S.awaiting = 0; S.remaining = d.per_stage; S.n_w = S.n_f = S.n_b = 0;
  S.next_adm = s == 0 ? 0 : -1; S.fixed_head = 0; S.touched = 0;
  S.mode = RRFP_BP_NORMAL; S.focus = -1; S.phase = -1;
  S.heap_n = 0; S.mbox_n = 0; S.mbox_drained = 0; S.overflow = 0;
  for (int i = 0; i < RRFP_MAX_WORDS; ++i) {
    S.doneF[i] = S.doneB[i] = S.wpend[i] = 0;
    for (int r = 0; r < RRFP_MAX_RANKS; ++r) S.fready[r][i] = S.bready[r][i] = S.pend[r][i] = 0;
  }
}

// engine._send (engine.py:181-221)
RHD void des_send(des_ctx& x, int s, int dir, int mb, int c, int64_t end) {
  const rrfp_iter_desc& d = x.d;
  int MW = d.MW;
  int dst_s, dst_c, dst_dir = dir;
  if (dir == RRFP_DIR_F) {
    if (s < d.N - 1) { dst_s = s + 1; dst_c = c; }
    else if (c < d.C - 1) { dst_s = 0; dst_c = c + 1; }
    else {  // pipeline turn-around: local grad input at `end`
      int k = rrfp_key(mb, c, MW);
      for (int r = 0; r < d.R; ++r) bit_set(x.st[s].bready[r], k);
      return;
    }
  } else {
    if (s > 0) { dst_s = s - 1; dst_c = c; }
    else if (c > 0) { dst_s = d.N - 1; dst_c = c - 1; }
    else return;  // gradient leaves the pipeline
  }
  int key = rrfp_key(mb, c, MW);
  int dkey = rrfp_key(mb, dst_c, MW);
  int64_t deliver = end + x.comm[((size_t)s * 2 + dir) * x.KEYS + key];
  rrfp_task_t src = rrfp_make_task(dir, s, mb, c);
  rrfp_task_t dst = rrfp_make_task(dst_dir, dst_s, mb, dst_c);
  des_emit(x, 1, end, deliver, s, -1, src);
  des_hent rel; rel.time = deliver; rel.kind = 1; rel.rank = 0; rel.task = src; rel.pad = 0;
  heap_push(x, s, rel);
  des_stage& D = x.st[dst_s];
  for (int r = 0; r < d.R; ++r) {
    int64_t sk = x.skew[(((size_t)dst_s * 2 + dst_dir) * x.KEYS + dkey) * d.R + r];
    int i = atomic_inc(&D.mbox_n);
    if (i >= x.mbox_cap) { D.overflow = 1; continue; }
    des_mbox& m = x.mbox[(size_t)dst_s * x.mbox_cap + i];
    m.time = deliver + sk; m.rank = r; m.task = dst;
  }
}

// engine._apply_complete (engine.py:240-266)
RHD void des_complete(des_ctx& x, int s, int64_t t, rrfp_task_t task) {
  const rrfp_iter_desc& d = x.d;
  des_stage& S = x.st[s];
  int dir = rrfp_task_dir(task), mb = rrfp_task_mb(task), c = rrfp_task_chunk(task);
  int k = rrfp_key(mb, c, d.MW);
  S.remaining -= 1;
  if (dir == RRFP_DIR_F) {
    bit_set(S.doneF, k);
    S.n_f += 1;
    for (int r = 0; r < d.R; ++r)
      if (bit_get(S.pend[r], k)) { bit_clr(S.pend[r], k); bit_set(S.bready[r], k); }
    des_send(x, s, dir, mb, c, t);
  } else if (dir == RRFP_DIR_B) {
    bit_set(S.doneB, k);
    S.n_b += 1;
    if (d.decompose) bit_set(S.wpend, k);
    des_send(x, s, dir, mb, c, t);
  } else {
    S.n_w += 1;
  }
}

// engine._apply_arrival (engine.py:225-238)
RHD void des_arrival(des_ctx& x, int s, int64_t t, int r, rrfp_task_t task) {
  des_stage& S = x.st[s];
  S.awaiting = 0;
  int k = rrfp_key(rrfp_task_mb(task), rrfp_task_chunk(task), x.d.MW);
  if (rrfp_task_dir(task) == RRFP_DIR_F) bit_set(S.fready[r], k);
  else if (bit_get(S.doneF, k)) bit_set(S.bready[r], k);
  else bit_set(S.pend[r], k);
  des_emit(x, 2, t, t, s, r, task);
}

// engine._commit (engine.py:270-296)
RHD void des_commit(des_ctx& x, int s, int kind, int mb, int c, int64_t start) {
  const rrfp_iter_desc& d = x.d;
  des_stage& S = x.st[s];
  int k = rrfp_key(mb, c, d.MW);
  int64_t dur = tbl_dur(x, s, kind, k);
  if (kind == RRFP_DIR_F) {
    if (s == 0 && c == 0) {
      // stage-0 chunk-0 forwards come only from the admission cursor
      S.next_adm += 1;
      if (S.next_adm >= d.M) S.next_adm = -1;
    } else {
      for (int r = 0; r < d.R; ++r) bit_clr(S.fready[r], k);
    }
  } else if (kind == RRFP_DIR_B) {
    for (int r = 0; r < d.R; ++r) bit_clr(S.bready[r], k);
  } else {
    bit_clr(S.wpend, k);
  }
  rrfp_advance_phase(&S.phase, d.hint, kind);
  S.busy_until = start + dur;
  S.compute += dur;
  rrfp_task_t task = rrfp_make_task(kind, s, mb, c);
  for (int r = 0; r < d.R; ++r) des_emit(x, 0, start, start + dur, s, d.R > 1 ? r : -1, task);
  S.complete_time = start + dur;
  S.complete_task = task;
}

RHD rrfp_view_ref des_view(const des_ctx& x, int s, int r) {
  const des_stage& S = x.st[s];
  rrfp_view_ref v;
  v.fready = S.fready[r]; v.bready = S.bready[r]; v.wpend = S.wpend;
  v.doneF = S.doneF; v.doneB = S.doneB;
  v.admission = (s == 0) ? S.next_adm : -1;
  return v;
}

RHD bool same_dec(const rrfp_decision& a, const rrfp_decision& b) {
  return a.kind == b.kind && a.mb == b.mb && a.chunk == b.chunk;
}

// engine._dispatch (engine.py:298-340) and the FIXED head rule (baselines.py:121-143)
RHD void des_dispatch(des_ctx& x, int s, int64_t now) {
  const rrfp_iter_desc& d = x.d;
  des_stage& S = x.st[s];
  if (S.busy_until > now || S.coord_until > now || S.remaining == 0) return;
  int MW = d.MW;
  if (d.fixed_mode) {
    if (S.fixed_head >= d.per_stage) return;
    rrfp_task_t t = x.fixed[(size_t)s * d.per_stage + S.fixed_head];
    int dir = rrfp_task_dir(t), mb = rrfp_task_mb(t), c = rrfp_task_chunk(t);
    int k = rrfp_key(mb, c, MW);
    bool ready;
    if (dir == RRFP_DIR_F) ready = (s == 0 && c == 0) ? true : bit_get(S.fready[0], k);
    else if (dir == RRFP_DIR_B) ready = bit_get(S.bready[0], k);
    else ready = bit_get(S.wpend, k);
    if (!ready) return;
    S.fixed_head += 1;
    des_commit(x, s, dir, mb, c, now);
    return;
  }
  rrfp_bp_update(&S.mode, &S.focus, d.buffer_limit, S.n_f, S.n_b, S.doneF, S.doneB, d.M, d.C, MW);
  if (d.R == 1) {
    rrfp_decision dec = rrfp_arbitrate_core(des_view(x, s, 0), d.hint, S.mode, S.focus, S.phase,
                                            d.M, d.C, MW, d.decompose);
    if (dec.kind == RRFP_WAIT) { S.phase = -1; return; }
    des_commit(x, s, dec.kind, dec.mb, dec.chunk, now);
    return;
  }
  rrfp_decision ds[RRFP_MAX_RANKS];
  bool all_wait = true, all_w = true;
  for (int r = 0; r < d.R; ++r) {
    ds[r] = rrfp_arbitrate_core(des_view(x, s, r), d.hint, S.mode, S.focus, S.phase, d.M, d.C,
                                MW, d.decompose);
    all_wait = all_wait && ds[r].kind == RRFP_WAIT;
    all_w = all_w && ds[r].kind == RRFP_DIR_W;
  }
  if (all_wait) { S.phase = -1; return; }
  if (all_w) { des_commit(x, s, RRFP_DIR_W, ds[0].mb, ds[0].chunk, now); return; }
  if (S.awaiting) return;
  // tp_coordinate (arbitration.py:323-334): agreed iff all present and equal
  bool agreed = ds[0].kind == RRFP_DIR_F || ds[0].kind == RRFP_DIR_B;
  for (int r = 1; r < d.R && agreed; ++r) agreed = same_dec(ds[r], ds[0]);
  int64_t cost = d.coord_cost;
  S.coord_time += cost;
  if (agreed) {
    atomic_add64(&x.counters[0], 1);
    des_emit(x, 3, now, now + cost, s, -1, rrfp_make_task(ds[0].kind, s, ds[0].mb, ds[0].chunk));
    des_commit(x, s, ds[0].kind, ds[0].mb, ds[0].chunk, now + cost);
  } else {
    atomic_add64(&x.counters[1], 1);
    des_emit(x, 4, now, now + cost, s, -1, RRFP_NO_TASK);
    S.coord_until = now + cost;
    S.awaiting = 1;
    S.phase = -1;
    S.coord_end_time = now + cost;
  }
}

// Phase A of a tick: completions (which create sends/arrivals for others).
RHD void des_phase_a(des_ctx& x, int s, int64_t T) {
  des_stage& S = x.st[s];
  S.touched = 0;
  if (S.complete_time == T) {
    rrfp_task_t t = S.complete_task;
    S.complete_time = -1;
    S.complete_task = RRFP_NO_TASK;
    des_complete(x, s, T, t);
    S.touched = 1;
  }
}

// Phase B: drain inbox, apply arrivals/releases/coord-ends at T, dispatch.
RHD void des_phase_b(des_ctx& x, int s, int64_t T) {
  des_stage& S = x.st[s];
  int n = S.mbox_n < x.mbox_cap ? S.mbox_n : x.mbox_cap;
  for (int i = S.mbox_drained; i < n; ++i) {
    const des_mbox& m = x.mbox[(size_t)s * x.mbox_cap + i];
    des_hent e; e.time = m.time; e.kind = 0; e.rank = m.rank; e.task = m.task; e.pad = 0;
    heap_push(x, s, e);
  }
  S.mbox_drained = n;
  while (S.heap_n > 0 && x.heap[(size_t)s * x.heap_cap].time == T) {
    des_hent e = heap_pop(x, s);
    if (e.kind == 0) des_arrival(x, s, T, e.rank, e.task);
    S.touched = 1;
  }
  if (S.coord_end_time == T) { S.coord_end_time = -1; S.touched = 1; }
  if (S.touched) des_dispatch(x, s, T);
}

#define RRFP_T_INF ((int64_t)0x7fffffffffffffffLL)

RHD int64_t des_next_time(const des_ctx& x, int s) {
  const des_stage& S = x.st[s];
  int64_t t = RRFP_T_INF;
  if (S.complete_time >= 0 && S.complete_time < t) t = S.complete_time;
  if (S.coord_end_time >= 0 && S.coord_end_time < t) t = S.coord_end_time;
  if (S.heap_n > 0 && x.heap[(size_t)s * x.heap_cap].time < t) t = x.heap[(size_t)s * x.heap_cap].time;
  return t;
}
