// rrfp_exec.cu -- the free-running device runtime that replaces live.run_live
// (/root/reference/pkg/src/rrfp/live.py:111-523).
//
// One *lane* = one (stage, TP rank) executor on one GPU.  Per iteration the
// lane runs ONE CUDA graph, launched once by the host:
//
//   init ─► WHILE(h_while) { dispatch ─► SWITCH(h_switch){B-body, F-body, W-body} ─► complete } ─► final
//
// * dispatch  (K2+K3, and K4 for TP): one warp polls the lane's inbox flags
//   (ld.acquire.sys), ballots them into ready bitmasks, runs the shared
//   __host__ __device__ arbiter (rrfp_core.cuh) and selects the body with
//   cudaGraphSetConditional -- no host round trip per task.
//   live.py:_worker/_resolve_round/_commit_locked (331-421, 246-297).
// * bodies    caller compute graphs (GPT stage F/B/W) or synthetic spins of
//   the latency table (live.py:388-390 semantics, time_scale applied).
// * complete  (K1 + K11 + K12): optional jitter pad, completion bookkeeping
//   (live._complete_locked 299-329), then the send: the payload was already
//   written into the receiver's mailbox by the body; here the lane
//   publishes visible-at stamp + epoch flag with st.release.sys into every
//   destination rank's inbox (live._sender/_receiver 203-244).  A comm-delay
//   is a visible-at time in the future, never a blocking sleep.
//
// Inbox flags carry the iteration epoch, so nothing is ever reset; an
// iteration barrier in `init` keeps epochs of a lane group in step.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "rrfp_common.h"
#include "rrfp_core.cuh"

#define RRFP_MAX_KEYS (RRFP_MAX_WORDS * 32)
#define RRFP_MAX_LANES 64
#define LANE_NONE 3

struct lane_inbox {
  uint32_t fflag[RRFP_MAX_KEYS];
  uint32_t bflag[RRFP_MAX_KEYS];
  unsigned long long fvis[RRFP_MAX_KEYS];
  unsigned long long bvis[RRFP_MAX_KEYS];
  // proposals double-buffered by round parity: a rank can run at most ONE round
  // ahead of a peer still gathering (it needs the peer's proposal of the
  // current round to finish it), so slot (round & 1) is never overwritten
  // before every peer has read it.
  unsigned long long tp_prop[2][RRFP_MAX_RANKS];  // (round << 32) | decision code
  uint32_t tp_cnt[2][RRFP_MAX_RANKS];             // proposer's view count at proposal
  uint32_t view_count;                          // monotone count of visible arrivals
  uint32_t done_epoch;                          // iteration barrier
  uint32_t pad[2];
  // replay (virtual-clock) mode: (epoch << 44) | lower bound of the virtual
  // time of any message this lane has not sent yet (conservative PDES)
  unsigned long long vsafe;
};

#define V_TBITS 44
#define V_INF ((1LL << V_TBITS) - 1)

struct lane_state {
  rrfp_lane_desc d;
  int KEYS, nwords;
  uint32_t epoch;
  int32_t n_f, n_b, n_w, mode, focus, phase, next_adm, remaining, fixed_head, status;
  int32_t cur_kind;
  rrfp_task_t cur_task;
  unsigned long long t_start, t_iter0, t_iter1;
  unsigned long long tp_round;
  uint32_t tp_snap;
  int32_t n_lanes;
  lane_inbox* inbox;                        // own inbox (local)
  lane_inbox* fwd_dst[RRFP_MAX_RANKS];      // receivers of F output
  lane_inbox* bwd_dst[RRFP_MAX_RANKS];      // receivers of B output
  lane_inbox* tp_peer[RRFP_MAX_RANKS];      // TP group boards (incl. self)
  lane_inbox* all[RRFP_MAX_LANES];          // every lane (iteration barrier)
  const long long* dur_ns;                  // [3][KEYS] spin / jitter pad
  const long long* comm_ns;                 // [2][KEYS]
  const long long* dskew_ns;                // [2][KEYS][R] arrival skew of a sent msg at each dest rank
  const long long* min_ns;                  // [3][KEYS] task floor: end >= start + min_ns (lognormal jitter)
  const rrfp_task_t* fixed;                 // [per_stage]
  rrfp_event* ring;
  int32_t ring_n, ring_cap;
  volatile int32_t* abort_flag;             // host-mapped
  volatile int32_t* mon;                    // host-mapped monitor: [0] where, [1] task, [2] remaining, [3] epoch
  cudaGraphConditionalHandle h_while, h_switch;
  uint32_t doneF[RRFP_MAX_WORDS], doneB[RRFP_MAX_WORDS], wpend[RRFP_MAX_WORDS];
  uint32_t fdisp[RRFP_MAX_WORDS], bdisp[RRFP_MAX_WORDS];
  uint32_t recvF[RRFP_MAX_WORDS], recvB[RRFP_MAX_WORDS];
  // ---- replay (virtual-clock) mode: engine._Stage of this lane (engine.py:70-90)
  long long v_now, v_busy_until, v_coord_until, v_coord_end, v_touch, v_start, v_end, v_H;
  int32_t v_await, v_nin;
  lane_inbox* v_in[2 * RRFP_MAX_RANKS];          // in-neighbour lanes (their vsafe words)
  uint32_t vF[RRFP_MAX_WORDS], vB[RRFP_MAX_WORDS], vP[RRFP_MAX_WORDS];   // own view + pending grads
  uint32_t procF[RRFP_MAX_RANKS][RRFP_MAX_WORDS], procB[RRFP_MAX_RANKS][RRFP_MAX_WORDS];
  // ---- decision log (desc.declog_cap records)
  uint32_t* declog;
  int32_t declog_n;
  uint32_t declog_sig;     // free mode: inputs of the last logged WAIT (re-polls are not logged)
  // ---- dispatcher profile (rrfp_runtime_profile): per step kernel 4 x u64
  //      {entry, completion done, decision made, kind << 32 | view polls}
  unsigned long long* prof;
  int32_t prof_n, prof_cap, polls;
};

// ------------------------------------------------------------ primitives
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_volatile64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ void ring_emit(lane_state* L, int kind, unsigned long long t0, unsigned long long t1,
                          int rank, rrfp_task_t task) {
  int i = atomicAdd(&L->ring_n, 1);
  if (i < L->ring_cap) {
    rrfp_event& e = L->ring[i];
    e.t0 = (long long)t0; e.t1 = (long long)t1; e.kind = kind; e.stage = L->d.stage;
    e.rank = rank; e.task = task;
  }
}

__device__ __forceinline__ void spin_until(unsigned long long deadline) {
  while (gtimer() < deadline) __nanosleep(64);
}

// ------------------------------------------------------------------ init
__global__ void lane_init_kernel(lane_state* L) {
  const int lane = threadIdx.x;
  // iteration barrier: every lane of the job finished the previous epoch
  if (lane == 0) {
    L->epoch += 1;
    uint32_t prev = L->epoch - 1;
    unsigned long long t_guard = gtimer();
    for (int i = 0; i < L->n_lanes; ++i) {
      while (ld_acquire_sys(&L->all[i]->done_epoch) < prev) {
        if (*L->abort_flag) break;
        __nanosleep(128);
      }
    }
    (void)t_guard;
    L->n_f = L->n_b = L->n_w = 0;
    L->mode = RRFP_BP_NORMAL; L->focus = -1; L->phase = -1;
    L->next_adm = L->d.stage == 0 ? 0 : -1;
    L->remaining = L->d.per_stage;
    L->fixed_head = 0; L->status = 0; L->cur_kind = LANE_NONE;
    L->ring_n = 0;
    L->prof_n = 0;
    L->declog_n = 0;
    L->declog_sig = 0xFFFFFFFFu;
    L->v_now = 0; L->v_busy_until = 0; L->v_coord_until = 0; L->v_coord_end = -1;
    L->v_touch = 0;       // engine.run dispatches every stage at t = 0 (engine.py:345-346)
    L->v_start = L->v_end = 0; L->v_H = 0; L->v_await = 0;
    L->t_iter0 = gtimer();
    L->mon[0] = 1; L->mon[2] = L->remaining; L->mon[3] = (int32_t)L->epoch;
  }
  for (int i = lane; i < RRFP_MAX_WORDS; i += 32) {
    L->doneF[i] = L->doneB[i] = L->wpend[i] = 0;
    L->fdisp[i] = L->bdisp[i] = 0;
    L->recvF[i] = L->recvB[i] = 0;
    L->vF[i] = L->vB[i] = L->vP[i] = 0;
    for (int r = 0; r < RRFP_MAX_RANKS; ++r) L->procF[r][i] = L->procB[r][i] = 0;
  }
}

__global__ void lane_final_kernel(lane_state* L) {
  if (threadIdx.x == 0) {
    L->mon[0] = 4;
    L->t_iter1 = gtimer();
    __threadfence_system();
    st_release_sys(&L->inbox->done_epoch, L->epoch);
  }
}

// ---------------------------------------------------------------- dispatch
// Builds this lane's ready bitmasks from the inbox (warp-parallel), logs new
// arrivals, returns the number of visible arrivals.
__device__ void build_view(lane_state* L, uint32_t* sF, uint32_t* sB, unsigned long long now) {
  const int lane = threadIdx.x;
  const rrfp_lane_desc& d = L->d;
  const int MW = d.MW;
  const uint32_t ep = L->epoch;
  const lane_inbox* in = L->inbox;
  uint32_t count = 0;
  for (int w = 0; w < L->nwords; ++w) {
    int key = w * 32 + lane;
    int mb = rrfp_key_mb(key, MW), c = rrfp_key_chunk(key, MW);
    bool valid = mb < d.M;
    bool af = valid && ld_acquire_sys(&in->fflag[key]) == ep && in->fvis[key] <= now;
    bool ab = valid && ld_acquire_sys(&in->bflag[key]) == ep && in->bvis[key] <= now;
    bool turn = valid && d.stage == d.N - 1 && c == d.C - 1;
    uint32_t mF = __ballot_sync(0xffffffffu, af);
    uint32_t mB = __ballot_sync(0xffffffffu, ab);
    uint32_t mT = __ballot_sync(0xffffffffu, turn);
    uint32_t newF = mF & ~L->recvF[w];
    uint32_t newB = mB & ~L->recvB[w];
    if ((newF >> lane) & 1u)
      ring_emit(L, 2, in->fvis[key], in->fvis[key], d.rank, rrfp_make_task(RRFP_DIR_F, d.stage, mb, c));
    if ((newB >> lane) & 1u)
      ring_emit(L, 2, in->bvis[key], in->bvis[key], d.rank, rrfp_make_task(RRFP_DIR_B, d.stage, mb, c));
    __syncwarp();
    if (lane == 0) {
      L->recvF[w] |= newF;
      L->recvB[w] |= newB;
      sF[w] = mF & ~L->fdisp[w];
      sB[w] = (mB | mT) & L->doneF[w] & ~L->bdisp[w];
    }
    count += __popc(mF) + __popc(mB);
  }
  __syncwarp();
  if (lane == 0 && count != L->inbox->view_count) {
    st_release_sys(&L->inbox->view_count, count);
  }
  __syncwarp();
}

// One record per evaluated arbitration: the exact inputs of rrfp_bp_update +
// rrfp_arbitrate_core and the result (layout: include/rrfp_b200.h,
// rrfp_runtime_declog).  Thread 0 only.
__device__ __noinline__ void declog_put(lane_state* L, long long t, int mode_in, int focus_in, const uint32_t* fr,
                           const uint32_t* br, const rrfp_decision& dec) {
  if (!L->declog) return;
  const int nw = L->nwords;
  if (L->declog_n < L->d.declog_cap) {
    uint32_t* r = L->declog + (size_t)L->declog_n * (16 + 5 * nw);
    r[0] = L->d.stage; r[1] = L->d.rank; r[2] = L->n_f; r[3] = L->n_b;
    r[4] = mode_in; r[5] = (uint32_t)focus_in; r[6] = L->mode; r[7] = (uint32_t)L->focus;
    r[8] = (uint32_t)L->phase; r[9] = (uint32_t)L->next_adm;
    r[10] = dec.kind; r[11] = (uint32_t)dec.mb; r[12] = (uint32_t)dec.chunk; r[13] = nw;
    r[14] = (uint32_t)(unsigned long long)t; r[15] = (uint32_t)((unsigned long long)t >> 32);
    for (int w = 0; w < nw; ++w) {
      r[16 + w] = fr[w]; r[16 + nw + w] = br[w]; r[16 + 2 * nw + w] = L->wpend[w];
      r[16 + 3 * nw + w] = L->doneF[w]; r[16 + 4 * nw + w] = L->doneB[w];
    }
  }
  L->declog_n += 1;   // counts past the capacity: the host reports an overflow
}

__device__ rrfp_decision lane_arbitrate(lane_state* L, const uint32_t* sF, const uint32_t* sB,
                                        long long t) {
  const rrfp_lane_desc& d = L->d;
  const int mode_in = L->mode, focus_in = L->focus;
  rrfp_bp_update(&L->mode, &L->focus, d.buffer_limit, L->n_f, L->n_b, L->doneF, L->doneB, d.M,
                 d.C, d.MW);
  rrfp_view_ref v;
  v.fready = sF; v.bready = sB; v.wpend = L->wpend; v.doneF = L->doneF; v.doneB = L->doneB;
  v.admission = L->next_adm;
  rrfp_decision dec =
      rrfp_arbitrate_core(v, d.hint, L->mode, L->focus, L->phase, d.M, d.C, d.MW, d.decompose);
  if (L->declog) {
    // a WAIT is re-evaluated on every poll: log it once per distinct input
    // (inputs only grow between dispatches, so the ready-bit count + the
    // remaining-task count identify them)
    uint32_t sig = (uint32_t)L->remaining << 20;
    for (int w = 0; w < L->nwords; ++w) sig += __popc(sF[w]) + __popc(sB[w]) + __popc(L->wpend[w]);
    if (dec.kind != RRFP_WAIT || sig != L->declog_sig) declog_put(L, t, mode_in, focus_in, sF, sB, dec);
    L->declog_sig = dec.kind == RRFP_WAIT ? sig : 0xFFFFFFFFu;
  }
  return dec;
}

__device__ rrfp_decision lane_fixed_head(lane_state* L, const uint32_t* sF, const uint32_t* sB) {
  rrfp_decision dec; dec.kind = RRFP_WAIT; dec.mb = dec.chunk = -1;
  if (L->fixed_head >= L->d.per_stage) return dec;
  rrfp_task_t t = L->fixed[L->fixed_head];
  int dir = rrfp_task_dir(t), mb = rrfp_task_mb(t), c = rrfp_task_chunk(t);
  int k = rrfp_key(mb, c, L->d.MW);
  bool ready;
  if (dir == RRFP_DIR_F) ready = (L->d.stage == 0 && c == 0) || bit_get(sF, k);
  else if (dir == RRFP_DIR_B) ready = bit_get(sB, k);
  else ready = bit_get(L->wpend, k);
  if (ready) { dec.kind = dir; dec.mb = mb; dec.chunk = c; }
  return dec;
}

__device__ void lane_commit(lane_state* L, const rrfp_decision& dec) {
  const rrfp_lane_desc& d = L->d;
  int k = rrfp_key(dec.mb, dec.chunk, d.MW);
  if (dec.kind == RRFP_DIR_F) {
    if (d.stage == 0 && dec.chunk == 0) {
      L->next_adm = (L->next_adm + 1 < d.M) ? L->next_adm + 1 : -1;
      // FIXED mode may admit out of order: keep the cursor monotone past it
    }
    bit_set(L->fdisp, k);
  } else if (dec.kind == RRFP_DIR_B) {
    bit_set(L->bdisp, k);
  } else {
    bit_clr(L->wpend, k);
  }
  if (d.fixed_mode) L->fixed_head += 1;
  else rrfp_advance_phase(&L->phase, d.hint, dec.kind);
  L->cur_kind = dec.kind;
  L->cur_task = rrfp_make_task(dec.kind, d.stage, dec.mb, dec.chunk);
}

__device__ __forceinline__ uint32_t dec_code(const rrfp_decision& d) {
  return (uint32_t)d.kind | ((uint32_t)(d.mb & 1023) << 2) | ((uint32_t)(d.chunk & 15) << 12);
}

// K4: one TP agreement round over the group's boards (arbitration.py:323-334,
// live._resolve_round 246-277): publish this rank's proposal into every
// peer's board, gather all R (the same vector on every rank).  Returns the
// sum of the proposers' arrival counts (free mode's retry snapshot).
__device__ __noinline__ uint32_t tp_exchange(lane_state* L, const rrfp_decision& dec, rrfp_decision* ds) {
  const rrfp_lane_desc& d = L->d;
  const int R = d.R;
  unsigned long long round = ++L->tp_round;
  unsigned long long word = (round << 32) | dec_code(dec);
  uint32_t mycnt = L->inbox->view_count;
  const int par = (int)(round & 1);
  for (int r = 0; r < R; ++r) {
    L->tp_peer[r]->tp_cnt[par][d.rank] = mycnt;
    __threadfence_system();
    st_release_sys64(&L->tp_peer[r]->tp_prop[par][d.rank], word);
  }
  uint32_t snap = 0;
  for (int r = 0; r < R; ++r) {
    unsigned long long w;
    while (((w = ld_acquire_sys64(&L->inbox->tp_prop[par][r])) >> 32) != round) {
      if (*L->abort_flag) break;
      __nanosleep(32);
    }
    uint32_t code = (uint32_t)w;
    ds[r].kind = code & 3; ds[r].mb = (code >> 2) & 1023; ds[r].chunk = (code >> 12) & 15;
    snap += L->inbox->tp_cnt[par][r];
  }
  return snap;
}

__device__ void lane_dispatch(lane_state* L) {
  __shared__ uint32_t sF[RRFP_MAX_WORDS], sB[RRFP_MAX_WORDS];
  __shared__ int s_kind, s_exit;
  const int lane = threadIdx.x;
  const rrfp_lane_desc& d = L->d;
  const int R = d.R;
  if (lane == 0) L->polls = 0;
  while (true) {
    if (lane == 0) {
      L->polls += 1;
      s_exit = 0;
      if (*L->abort_flag) { L->status = RRFP_E_WATCHDOG; s_exit = 1; }
      else if (L->remaining == 0) s_exit = 1;
    }
    __syncwarp();
    if (s_exit) {
      if (lane == 0) {
        L->cur_kind = LANE_NONE;
        cudaGraphSetConditional(L->h_switch, 0xFFFFFFFFu);
        cudaGraphSetConditional(L->h_while, 0);
      }
      return;
    }
    unsigned long long now = gtimer();
    build_view(L, sF, sB, now);
    if (lane == 0) {
      rrfp_decision dec =
          d.fixed_mode ? lane_fixed_head(L, sF, sB) : lane_arbitrate(L, sF, sB, (long long)now);
      s_kind = RRFP_WAIT;
      if (R == 1) {
        if (dec.kind == RRFP_WAIT) {
          if (!d.fixed_mode) L->phase = -1;
        } else {
          lane_commit(L, dec);
          s_kind = dec.kind;
        }
      } else {
        // K4: TP agreement round over the group's boards (arbitration.py:323-334,
        // live._resolve_round 246-277): publish, gather all R, same verdict everywhere.
        rrfp_decision ds[RRFP_MAX_RANKS];
        uint32_t snap = tp_exchange(L, dec, ds);
        bool all_wait = true, all_w = true;
        for (int r = 0; r < R; ++r) {
          all_wait = all_wait && ds[r].kind == RRFP_WAIT;
          all_w = all_w && ds[r].kind == RRFP_DIR_W;
        }
        if (all_wait) {
          L->phase = -1;
        } else if (all_w) {
          lane_commit(L, ds[0]);
          s_kind = RRFP_DIR_W;
        } else {
          bool agreed = ds[0].kind == RRFP_DIR_F || ds[0].kind == RRFP_DIR_B;
          for (int r = 1; r < R && agreed; ++r)
            agreed = ds[r].kind == ds[0].kind && ds[r].mb == ds[0].mb && ds[r].chunk == ds[0].chunk;
          unsigned long long t0 = gtimer();
          spin_until(t0 + (unsigned long long)d.coord_cost_ns);
          if (d.rank == 0)
            ring_emit(L, agreed ? 3 : 4, t0, gtimer(), -1,
                      agreed ? rrfp_make_task(ds[0].kind, d.stage, ds[0].mb, ds[0].chunk)
                             : RRFP_NO_TASK);
          if (agreed) {
            lane_commit(L, ds[0]);
            s_kind = ds[0].kind;
          } else {
            L->phase = -1;
          }
        }
        L->tp_snap = snap;
        // wait / deferral: retry only after a new arrival at ANY rank of the
        // group (live.py:398-407); -1 tells the warp to enter that wait.
        if (s_kind == RRFP_WAIT) s_kind = -1;
      }
      if (s_kind >= 0 && s_kind != RRFP_WAIT) {
        L->mon[0] = 2;
        L->mon[1] = (int32_t)L->cur_task;
        L->t_start = gtimer();
        unsigned branch = (unsigned)s_kind;
        if (d.compute_kind == 1)   // body (kind, chunk, mb): kind * M*C + chunk * M + mb
          branch = (unsigned)(s_kind * d.M * d.C + rrfp_task_chunk(L->cur_task) * d.M + rrfp_task_mb(L->cur_task));
        cudaGraphSetConditional(L->h_switch, branch);
      }
    }
    __syncwarp();
    int k = s_kind;
    if (k >= 0 && k != RRFP_WAIT) return;
    if (R > 1 && k < 0) {
      // TP wait: rebuild the view until any rank's arrival count changes
      while (true) {
        __syncwarp();
        build_view(L, sF, sB, gtimer());
        int go = 0;
        if (lane == 0) {
          uint32_t cur = 0;
          for (int r = 0; r < R; ++r) cur += ld_acquire_sys(&L->tp_peer[r]->view_count);
          go = (cur != L->tp_snap) || *L->abort_flag;
        }
        go = __shfl_sync(0xffffffffu, go, 0);
        if (go) break;
        __nanosleep(256);
      }
    } else {
      __nanosleep(128);
    }
  }
}

// ======================================================== replay (virtual clock)
// The lane runs the reference engine's per-stage semantics itself
// (engine.py:181-340) at virtual times, and makes every decision with the
// same rrfp_arbitrate_core + K4 round as free mode.  Cross-lane knowledge is
// only what physically arrived: a message carries its virtual arrival time
// (vt = end + comm delay + rank skew, engine.py:211-221) in the inbox's
// visible-at stamp; each lane publishes vsafe = a lower bound of the vt of
// anything it has not sent yet; a lane processes tick T only when every
// in-neighbour's vsafe exceeds T, so every arrival with vt <= T has landed
// (Chandy-Misra-Bryant conservative PDES, lookahead = min task duration +
// min comm delay).  Within a tick the engine applies all events, then
// dispatches (engine.py:347-362); a stage's arrivals and its own completion
// commute (no dispatch happens while it is busy), so a lane applies its
// completion as soon as the body has run and its arrivals tick by tick.

__device__ __noinline__ void lane_send(lane_state* L, int dir, int mb, int c, unsigned long long end);

__device__ __forceinline__ long long v_min(long long a, long long b) { return a < b ? a : b; }
__device__ __forceinline__ long long v_max(long long a, long long b) { return a > b ? a : b; }

__device__ void v_publish(lane_state* L, long long h) {   // thread 0; monotone
  if (h > V_INF) h = V_INF;
  if (h <= L->v_H) return;
  L->v_H = h;
  unsigned long long w = ((unsigned long long)(L->epoch & 0xFFFFFu) << V_TBITS) | (unsigned long long)h;
  __threadfence_system();            // every message sent so far is visible before the bound
  st_release_sys64(&L->inbox->vsafe, w);
}

// min over the in-neighbours' bounds (V_INF without in-neighbours)
__device__ long long v_safe(lane_state* L) {
  long long S = V_INF;
  for (int i = 0; i < L->v_nin; ++i) {
    unsigned long long w = ld_acquire_sys64(&L->v_in[i]->vsafe);
    long long h = ((w >> V_TBITS) == (L->epoch & 0xFFFFFu)) ? (long long)(w & (unsigned long long)V_INF) : 0;
    S = v_min(S, h);
  }
  return S;
}

__device__ __forceinline__ long long warp_min64(long long v) {
  for (int o = 16; o; o >>= 1) v = v_min(v, (long long)__shfl_xor_sync(0xffffffffu, (unsigned long long)v, o));
  return v;
}

// Earliest vt of a landed, unprocessed arrival at ANY rank of this stage (the
// stage is touched by every rank's arrivals, engine.py:225-238).  Warp.
__device__ long long v_scan(lane_state* L) {
  const int lane = threadIdx.x;
  const rrfp_lane_desc& d = L->d;
  const uint32_t ep = L->epoch;
  long long best = V_INF;
  for (int q = 0; q < d.R; ++q) {
    const lane_inbox* in = L->tp_peer[q];
    for (int w = 0; w < L->nwords; ++w) {
      int key = w * 32 + lane;
      if (rrfp_key_mb(key, d.MW) >= d.M) continue;
      if (!((L->procF[q][w] >> lane) & 1u) && ld_acquire_sys(&in->fflag[key]) == ep)
        best = v_min(best, (long long)ld_volatile64(&in->fvis[key]));
      if (!((L->procB[q][w] >> lane) & 1u) && ld_acquire_sys(&in->bflag[key]) == ep)
        best = v_min(best, (long long)ld_volatile64(&in->bvis[key]));
    }
  }
  return warp_min64(best);
}

// Apply every landed arrival with vt == T (engine._apply_arrival): own rank's
// into the view (B gated on the local F, else pending), all ranks' marked
// processed.  Returns whether any rank had one (stage touched).  Warp.
__device__ bool v_arrivals(lane_state* L, long long T) {
  const int lane = threadIdx.x;
  const rrfp_lane_desc& d = L->d;
  const uint32_t ep = L->epoch;
  bool any = false;
  for (int q = 0; q < d.R; ++q) {
    const lane_inbox* in = L->tp_peer[q];
    for (int w = 0; w < L->nwords; ++w) {
      int key = w * 32 + lane;
      int mb = rrfp_key_mb(key, d.MW), c = rrfp_key_chunk(key, d.MW);
      bool valid = mb < d.M;
      bool af = valid && !((L->procF[q][w] >> lane) & 1u) && ld_acquire_sys(&in->fflag[key]) == ep &&
                (long long)ld_volatile64(&in->fvis[key]) == T;
      bool ab = valid && !((L->procB[q][w] >> lane) & 1u) && ld_acquire_sys(&in->bflag[key]) == ep &&
                (long long)ld_volatile64(&in->bvis[key]) == T;
      uint32_t mF = __ballot_sync(0xffffffffu, af);
      uint32_t mB = __ballot_sync(0xffffffffu, ab);
      if (q == d.rank) {
        if (af) ring_emit(L, 2, T, T, d.rank, rrfp_make_task(RRFP_DIR_F, d.stage, mb, c));
        if (ab) ring_emit(L, 2, T, T, d.rank, rrfp_make_task(RRFP_DIR_B, d.stage, mb, c));
      }
      __syncwarp();
      if (lane == 0) {
        L->procF[q][w] |= mF;
        L->procB[q][w] |= mB;
        if (q == d.rank) {
          L->vF[w] |= mF;
          L->vB[w] |= mB & L->doneF[w];
          L->vP[w] |= mB & ~L->doneF[w];
        }
      }
      any = any || mF || mB;
      __syncwarp();
    }
  }
  return any;
}

// engine._apply_complete (engine.py:240-266) for the task whose body just ran.
__device__ void v_complete(lane_state* L) {
  const rrfp_lane_desc& d = L->d;
  const int kind = L->cur_kind;
  rrfp_task_t t = L->cur_task;
  int mb = rrfp_task_mb(t), c = rrfp_task_chunk(t);
  int k = rrfp_key(mb, c, d.MW);
  const long long end = L->v_end;
  L->remaining -= 1;
  L->mon[0] = 3;
  L->mon[2] = L->remaining;
  if (kind == RRFP_DIR_F) {
    bit_set(L->doneF, k);
    L->n_f += 1;
    if (bit_get(L->vP, k)) { bit_clr(L->vP, k); bit_set(L->vB, k); }
    if (d.stage == d.N - 1 && c == d.C - 1) bit_set(L->vB, k);   // turn-around (engine.py:193-199)
    else lane_send(L, kind, mb, c, (unsigned long long)end);
  } else if (kind == RRFP_DIR_B) {
    bit_set(L->doneB, k);
    L->n_b += 1;
    if (d.decompose) bit_set(L->wpend, k);
    lane_send(L, kind, mb, c, (unsigned long long)end);
  } else {
    L->n_w += 1;
  }
  L->cur_kind = LANE_NONE;
  L->v_touch = end;                  // the completion touches the stage at `end`
  // next send: after a task that starts >= end
  v_publish(L, end + d.v_dmin + d.v_la);
}

// engine._commit (engine.py:270-296): virtual start/end, exec record per rank.
__device__ void v_commit(lane_state* L, const rrfp_decision& dec, long long start) {
  const rrfp_lane_desc& d = L->d;
  int k = rrfp_key(dec.mb, dec.chunk, d.MW);
  long long dur = L->dur_ns[(size_t)dec.kind * L->KEYS + k];     // integer us in replay mode
  if (dec.kind == RRFP_DIR_F) {
    if (d.stage == 0 && dec.chunk == 0) L->next_adm = (L->next_adm + 1 < d.M) ? L->next_adm + 1 : -1;
    else bit_clr(L->vF, k);
  } else if (dec.kind == RRFP_DIR_B) {
    bit_clr(L->vB, k);
  } else {
    bit_clr(L->wpend, k);
  }
  if (d.fixed_mode) L->fixed_head += 1;
  else rrfp_advance_phase(&L->phase, d.hint, dec.kind);
  rrfp_task_t task = rrfp_make_task(dec.kind, d.stage, dec.mb, dec.chunk);
  L->v_start = start;
  L->v_end = start + dur;
  L->v_busy_until = start + dur;
  ring_emit(L, 0, (unsigned long long)start, (unsigned long long)(start + dur), d.R > 1 ? d.rank : -1, task);
  L->cur_kind = dec.kind;
  L->cur_task = task;
  v_publish(L, start + dur + d.v_la);
}

// engine._dispatch (engine.py:298-340) / the FIXED head rule (baselines.py:121-143)
// at virtual time T; returns the committed kind or RRFP_WAIT.  Thread 0.
__device__ int v_dispatch(lane_state* L, long long T) {
  const rrfp_lane_desc& d = L->d;
  rrfp_decision dec;
  if (d.fixed_mode) {
    if (L->fixed_head >= d.per_stage) return RRFP_WAIT;
    rrfp_task_t t = L->fixed[L->fixed_head];
    int dir = rrfp_task_dir(t), mb = rrfp_task_mb(t), c = rrfp_task_chunk(t);
    int k = rrfp_key(mb, c, d.MW);
    bool ready = dir == RRFP_DIR_F ? ((d.stage == 0 && c == 0) || bit_get(L->vF, k))
               : dir == RRFP_DIR_B ? bit_get(L->vB, k) : bit_get(L->wpend, k);
    if (!ready) return RRFP_WAIT;
    dec.kind = dir; dec.mb = mb; dec.chunk = c;
    v_commit(L, dec, T);
    return dir;
  }
  const int mode_in = L->mode, focus_in = L->focus;
  rrfp_bp_update(&L->mode, &L->focus, d.buffer_limit, L->n_f, L->n_b, L->doneF, L->doneB, d.M, d.C, d.MW);
  rrfp_view_ref v;
  v.fready = L->vF; v.bready = L->vB; v.wpend = L->wpend; v.doneF = L->doneF; v.doneB = L->doneB;
  v.admission = L->next_adm;
  dec = rrfp_arbitrate_core(v, d.hint, L->mode, L->focus, L->phase, d.M, d.C, d.MW, d.decompose);
  declog_put(L, T, mode_in, focus_in, L->vF, L->vB, dec);
  if (d.R == 1) {
    if (dec.kind == RRFP_WAIT) { L->phase = -1; return RRFP_WAIT; }
    v_commit(L, dec, T);
    return dec.kind;
  }
  // a blocking round: nothing this lane sends can precede T + dmin (+ la)
  v_publish(L, T + d.v_dmin + d.v_la);
  rrfp_decision ds[RRFP_MAX_RANKS];
  tp_exchange(L, dec, ds);
  bool all_wait = true, all_w = true;
  for (int r = 0; r < d.R; ++r) {
    all_wait = all_wait && ds[r].kind == RRFP_WAIT;
    all_w = all_w && ds[r].kind == RRFP_DIR_W;
  }
  if (all_wait) { L->phase = -1; return RRFP_WAIT; }
  if (all_w) { v_commit(L, ds[0], T); return RRFP_DIR_W; }
  if (L->v_await) return RRFP_WAIT;             // a deferred round retries after an arrival
  bool agreed = ds[0].kind == RRFP_DIR_F || ds[0].kind == RRFP_DIR_B;
  for (int r = 1; r < d.R && agreed; ++r)
    agreed = ds[r].kind == ds[0].kind && ds[r].mb == ds[0].mb && ds[r].chunk == ds[0].chunk;
  const long long cost = d.coord_cost_ns;        // integer us in replay mode
  if (d.rank == 0)
    ring_emit(L, agreed ? 3 : 4, (unsigned long long)T, (unsigned long long)(T + cost), -1,
              agreed ? rrfp_make_task(ds[0].kind, d.stage, ds[0].mb, ds[0].chunk) : RRFP_NO_TASK);
  if (agreed) { v_commit(L, ds[0], T + cost); return ds[0].kind; }
  L->v_coord_until = T + cost;
  L->v_coord_end = T + cost;
  L->v_await = 1;
  L->phase = -1;
  return RRFP_WAIT;
}

// The replay-mode step: complete the body that just ran, then advance the
// virtual clock tick by tick until this lane commits its next task (SWITCH
// branch set) or finishes (WHILE ends).
__device__ __noinline__ void lane_virtual(lane_state* L) {
  __shared__ long long s_T;
  __shared__ int s_state;           // 0 wait, 1 process s_T, 2 exit
  __shared__ int s_kind;
  const int lane = threadIdx.x;
  const rrfp_lane_desc& d = L->d;
  if (lane == 0 && L->cur_kind != LANE_NONE) v_complete(L);
  __syncwarp();
  __shared__ long long s_S;
  while (true) {
    // the bound first, then the inbox: every message with vt < S was written
    // before its sender published S (release / acquire, then __syncwarp)
    if (lane == 0) s_S = v_safe(L);
    __syncwarp();
    long long amin = v_scan(L);
    if (lane == 0) {
      s_state = 0;
      if (*L->abort_flag) {
        L->status = RRFP_E_WATCHDOG; s_state = 2;
      } else if (L->remaining == 0) {
        s_state = 2;
      } else {
        const long long S = s_S;
        long long T = amin;
        if (L->v_touch >= 0) T = v_min(T, L->v_touch);
        if (L->v_coord_end >= 0) T = v_min(T, L->v_coord_end);
        if (T < S && T < V_INF) {
          s_T = T; s_state = 1;
        } else {
          long long base = v_max(L->v_now, v_min(T, S));
          if (base > d.v_horizon) {            // quiescent with unfinished tasks (engine.py:363-367)
            L->status = RRFP_E_DEADLOCK; s_state = 2;
          } else {
            v_publish(L, base + d.v_dmin + d.v_la);
          }
        }
      }
    }
    __syncwarp();
    const int st = s_state;
    if (st == 2) {
      if (lane == 0) {
        v_publish(L, V_INF);
        L->cur_kind = LANE_NONE;
        cudaGraphSetConditional(L->h_switch, 0xFFFFFFFFu);
        cudaGraphSetConditional(L->h_while, 0);
      }
      return;
    }
    if (st == 0) { __nanosleep(64); continue; }
    const long long T = s_T;
    bool any = v_arrivals(L, T);
    if (lane == 0) {
      bool touched = any;
      if (any) L->v_await = 0;
      if (L->v_coord_end == T) { L->v_coord_end = -1; touched = true; }
      if (L->v_touch == T) { L->v_touch = -1; touched = true; }
      L->v_now = T;
      s_kind = RRFP_WAIT;
      if (touched && T >= L->v_busy_until && T >= L->v_coord_until && L->remaining > 0) {
        L->mon[0] = 1;
        s_kind = v_dispatch(L, T);
      }
      if (s_kind != RRFP_WAIT) {
        L->mon[0] = 2;
        L->mon[1] = (int32_t)L->cur_task;
        L->t_start = gtimer();
        unsigned branch = (unsigned)s_kind;
        if (d.compute_kind == 1)
          branch = (unsigned)(s_kind * d.M * d.C + rrfp_task_chunk(L->cur_task) * d.M + rrfp_task_mb(L->cur_task));
        cudaGraphSetConditional(L->h_switch, branch);
      }
    }
    __syncwarp();
    if (s_kind != RRFP_WAIT) return;
  }
}

// ---------------------------------------------------------------- bodies
// Synthetic compute: spin the task's table duration (latency+jitter, scaled).
__global__ void lane_spin_body_kernel(lane_state* L) {
  if (threadIdx.x == 0) {
    rrfp_task_t t = L->cur_task;
    int k = rrfp_key(rrfp_task_mb(t), rrfp_task_chunk(t), L->d.MW);
    long long ns = L->dur_ns[(size_t)rrfp_task_dir(t) * L->KEYS + k];
    if (L->d.virtual_clock) ns = (long long)((double)ns * 1000.0 * L->d.time_scale);
    spin_until(L->t_start + (unsigned long long)ns);
  }
}

// ---------------------------------------------------------------- complete
__device__ __noinline__ void lane_send(lane_state* L, int dir, int mb, int c, unsigned long long end) {
  const rrfp_lane_desc& d = L->d;
  int dst_c, dst_s;
  lane_inbox* const* dsts;
  if (dir == RRFP_DIR_F) {
    if (d.stage < d.N - 1) { dst_s = d.stage + 1; dst_c = c; }
    else if (c < d.C - 1) { dst_s = 0; dst_c = c + 1; }
    else return;  // turn-around: B readiness derives from doneF locally
    dsts = L->fwd_dst;
  } else {
    if (d.stage > 0) { dst_s = d.stage - 1; dst_c = c; }
    else if (c > 0) { dst_s = d.N - 1; dst_c = c - 1; }
    else return;
    dsts = L->bwd_dst;
  }
  (void)dst_s;
  int key = rrfp_key(mb, c, d.MW);
  int dkey = rrfp_key(mb, dst_c, d.MW);
  long long delay = L->comm_ns[(size_t)dir * L->KEYS + key];
  // TP: rank r flags only rank r of the neighbour stage (the reference's
  // per-rank delivery, arrival = this rank's end + delay + skew[r]); the bytes
  // were written to every receiver rank's mailbox by every sender rank
  for (int r = d.rank; r == d.rank; ++r) {
    lane_inbox* in = dsts[r];
    long long sk = L->dskew_ns[((size_t)dir * L->KEYS + dkey) * d.R + r];
    unsigned long long vis = end + (unsigned long long)(delay + sk);
    if (dir == RRFP_DIR_F) {
      in->fvis[dkey] = vis;
      __threadfence_system();
      st_release_sys(&in->fflag[dkey], L->epoch);
    } else {
      in->bvis[dkey] = vis;
      __threadfence_system();
      st_release_sys(&in->bflag[dkey], L->epoch);
    }
  }
  if (d.rank == 0)
    ring_emit(L, 1, end, end + (unsigned long long)delay, -1, rrfp_make_task(dir, d.stage, mb, c));
}

// (thread 0) record + publish the task the SWITCH body just ran
__device__ void lane_complete(lane_state* L) {
  int kind = L->cur_kind;
  if (kind == LANE_NONE) return;
  const rrfp_lane_desc& d = L->d;
  rrfp_task_t t = L->cur_task;
  int mb = rrfp_task_mb(t), c = rrfp_task_chunk(t);
  int k = rrfp_key(mb, c, d.MW);
  if (d.compute_kind == 1) {
    // K11: injected jitter pads real compute: an additive delay (the J-level
    // injection table) and a floor start + nominal * X (lognormal compute jitter)
    long long pad = L->dur_ns[(size_t)kind * L->KEYS + k];
    long long floor_ns = L->min_ns[(size_t)kind * L->KEYS + k];
    unsigned long long until = gtimer() + (unsigned long long)(pad > 0 ? pad : 0);
    if (floor_ns > 0 && L->t_start + (unsigned long long)floor_ns > until)
      until = L->t_start + (unsigned long long)floor_ns;
    spin_until(until);
  }
  unsigned long long end = gtimer();
  ring_emit(L, 0, L->t_start, end, d.R > 1 ? d.rank : -1, t);
  L->remaining -= 1;
  L->mon[0] = 3;
  L->mon[2] = L->remaining;
  if (kind == RRFP_DIR_F) {
    bit_set(L->doneF, k);
    L->n_f += 1;
    lane_send(L, kind, mb, c, end);
  } else if (kind == RRFP_DIR_B) {
    bit_set(L->doneB, k);
    L->n_b += 1;
    if (d.decompose) bit_set(L->wpend, k);
    lane_send(L, kind, mb, c, end);
  } else {
    L->n_w += 1;
  }
  L->cur_kind = LANE_NONE;
}

// One dispatcher step per loop iteration: complete the task the previous
// iteration's SWITCH ran (end stamp, jitter pad, sends), then arbitrate the
// next one and set the SWITCH branch (or end the WHILE).  One kernel node per
// task instead of a dispatch and a completion kernel: ~1 device-side launch
// less per decision (tools/dispatch_bench.py).
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  bytes &= ~15u;
  if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(32, 1) lane_step_kernel(lane_state* L) {
  // Between two decisions the task body streams its working set through L2, so
  // the lane state and the inbox are usually cold: pull them into L2 in bulk
  // before the dependent chain of state reads starts (one HBM latency instead
  // of one per access).
  if (threadIdx.x == 0) {
    l2_prefetch(L, (uint32_t)sizeof(lane_state));
    lane_inbox* in = L->inbox;
    const uint32_t keys = (uint32_t)L->KEYS;
    l2_prefetch(in->fflag, keys * 4 + 12);
    l2_prefetch(in->bflag, keys * 4 + 12);
    l2_prefetch(in->fvis, keys * 8);
    l2_prefetch(in->bvis, keys * 8);
    l2_prefetch(in->tp_prop, (uint32_t)(sizeof(lane_inbox) - offsetof(lane_inbox, tp_prop)));
  }
  if (L->d.virtual_clock) {
    lane_virtual(L);
    return;
  }
  const unsigned long long t_in = gtimer();
  if (threadIdx.x == 0) lane_complete(L);
  const unsigned long long t_c = gtimer();
  __syncwarp();
  lane_dispatch(L);
  if (L->prof && threadIdx.x == 0) {
    const int i = L->prof_n++;
    if (i < L->prof_cap) {
      unsigned long long* p = L->prof + 4 * (size_t)i;
      p[0] = t_in; p[1] = t_c; p[2] = gtimer();
      p[3] = ((unsigned long long)(uint32_t)L->cur_kind << 32) | (uint32_t)L->polls;
    }
  }
}

// ================================================================ host side
struct rrfp_runtime {
  rrfp_lane_desc d;
  int dev;
  lane_state* L;            // device
  lane_inbox* inbox;        // device (separate allocation: IPC-exportable)
  long long* tables;        // device
  rrfp_task_t* fixed;       // device
  rrfp_event* ring;         // device
  int32_t* abort_host;      // mapped host memory
  int32_t* abort_dev;
  int32_t* mon_host;        // mapped monitor block (readable while the GPU is busy)
  int32_t* mon_dev;
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  uint32_t* declog;         // device, desc.declog_cap records
  std::vector<cudaGraph_t> bodies;   // [3 * M] per-(kind, mb) compute graphs
  bool built;
  cudaEvent_t done_ev;
  int KEYS;
  std::vector<void*> opened;
};

static int lane_check_desc(const rrfp_lane_desc* d) {
  if (!d) return rrfp_fail(RRFP_E_INVALID, "null lane desc");
  if (d->N < 1 || d->N > RRFP_MAX_STAGES || d->R < 1 || d->R > RRFP_MAX_RANKS || d->C < 1 ||
      d->C > RRFP_MAX_CHUNKS || d->M < 1 || d->M > RRFP_MAX_MB || d->MW != (d->M + 31) / 32 ||
      d->C * d->MW > RRFP_MAX_WORDS)
    return rrfp_fail(RRFP_E_INVALID, "lane shape out of range");
  if (d->N * d->R > RRFP_MAX_LANES) return rrfp_fail(RRFP_E_INVALID, "too many lanes");
  if (d->stage < 0 || d->stage >= d->N || d->rank < 0 || d->rank >= d->R)
    return rrfp_fail(RRFP_E_INVALID, "stage/rank out of range");
  if (d->buffer_limit < 1) return rrfp_fail(RRFP_E_INVALID, "buffer_limit must be >= 1");
  if (d->trace_cap < 16) return rrfp_fail(RRFP_E_INVALID, "trace_cap too small");
  if (d->declog_cap < 0) return rrfp_fail(RRFP_E_INVALID, "declog_cap must be >= 0");
  if (d->virtual_clock) {
    if (d->fixed_mode && d->R > 1)
      return rrfp_fail(RRFP_E_INVALID, "replay of a fixed schedule is rank-agnostic (R must be 1)");
    if (d->v_dmin + d->v_la < 1)
      return rrfp_fail(RRFP_E_INVALID, "replay mode needs a positive lookahead (min task + comm delay >= 1 us)");
    if (d->v_horizon < 1 || d->v_horizon >= V_INF) return rrfp_fail(RRFP_E_INVALID, "bad replay horizon");
  }
  return RRFP_OK;
}

extern "C" int rrfp_runtime_create(const rrfp_lane_desc* desc, rrfp_runtime** out) {
  int rc = lane_check_desc(desc);
  if (rc) return rc;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return rrfp_fail(RRFP_E_NOGPU, "no CUDA device");
  RRFP_CUDA_TRY(cudaSetDevice(desc->device));
  rrfp_runtime* rt = new rrfp_runtime();
  rt->d = *desc;
  rt->dev = desc->device;
  rt->KEYS = desc->C * desc->MW * 32;
  rt->built = false;
  RRFP_CUDA_TRY(cudaMalloc(&rt->L, sizeof(lane_state)));
  RRFP_CUDA_TRY(cudaMalloc(&rt->inbox, sizeof(lane_inbox)));
  RRFP_CUDA_TRY(cudaMemset(rt->inbox, 0, sizeof(lane_inbox)));
  size_t tbytes = sizeof(long long) * (size_t)rt->KEYS * (3 + 2 + 2 * desc->R + 3);
  RRFP_CUDA_TRY(cudaMalloc(&rt->tables, tbytes));
  RRFP_CUDA_TRY(cudaMemset(rt->tables, 0, tbytes));
  RRFP_CUDA_TRY(cudaMalloc(&rt->fixed, sizeof(rrfp_task_t) * (size_t)(desc->per_stage + 1)));
  RRFP_CUDA_TRY(cudaMalloc(&rt->ring, sizeof(rrfp_event) * (size_t)desc->trace_cap));
  rt->declog = nullptr;
  if (desc->declog_cap > 0)
    RRFP_CUDA_TRY(cudaMalloc(&rt->declog, sizeof(uint32_t) * (size_t)desc->declog_cap *
                                              (16 + 5 * desc->C * desc->MW)));
  RRFP_CUDA_TRY(cudaHostAlloc(&rt->abort_host, sizeof(int32_t), cudaHostAllocMapped));
  *rt->abort_host = 0;
  RRFP_CUDA_TRY(cudaHostGetDevicePointer(&rt->abort_dev, rt->abort_host, 0));
  RRFP_CUDA_TRY(cudaHostAlloc(&rt->mon_host, 16 * sizeof(int32_t), cudaHostAllocMapped));
  memset(rt->mon_host, 0, 16 * sizeof(int32_t));
  RRFP_CUDA_TRY(cudaHostGetDevicePointer(&rt->mon_dev, rt->mon_host, 0));
  RRFP_CUDA_TRY(cudaEventCreateWithFlags(&rt->done_ev, cudaEventDisableTiming));
  // host image of the lane state
  lane_state h;
  memset(&h, 0, sizeof(h));
  h.d = *desc;
  h.KEYS = rt->KEYS;
  h.nwords = desc->C * desc->MW;
  h.epoch = 0;
  h.inbox = rt->inbox;
  h.dur_ns = rt->tables;
  h.comm_ns = rt->tables + 3 * rt->KEYS;
  h.dskew_ns = rt->tables + 5 * (size_t)rt->KEYS;
  h.min_ns = rt->tables + (5 + 2 * desc->R) * (size_t)rt->KEYS;
  h.fixed = rt->fixed;
  h.ring = rt->ring;
  h.ring_cap = desc->trace_cap;
  h.abort_flag = rt->abort_dev;
  h.mon = rt->mon_dev;
  h.declog = rt->declog;
  h.v_nin = 0;
  h.n_lanes = 1;
  h.all[0] = rt->inbox;
  for (int r = 0; r < RRFP_MAX_RANKS; ++r) h.fwd_dst[r] = h.bwd_dst[r] = h.tp_peer[r] = rt->inbox;
  RRFP_CUDA_TRY(cudaMemcpy(rt->L, &h, sizeof(h), cudaMemcpyHostToDevice));
  *out = rt;
  return RRFP_OK;
}

extern "C" void rrfp_runtime_destroy(rrfp_runtime* rt) {
  if (!rt) return;
  cudaSetDevice(rt->dev);
  if (rt->exec) cudaGraphExecDestroy(rt->exec);
  if (rt->graph) cudaGraphDestroy(rt->graph);
  for (void* p : rt->opened) cudaIpcCloseMemHandle(p);
  unsigned long long* prof = nullptr;
  if (cudaMemcpy(&prof, (char*)rt->L + offsetof(lane_state, prof), sizeof(prof), cudaMemcpyDeviceToHost) ==
          cudaSuccess && prof)
    cudaFree(prof);
  cudaFree(rt->L); cudaFree(rt->inbox); cudaFree(rt->tables); cudaFree(rt->fixed);
  cudaFree(rt->ring); cudaFreeHost(rt->abort_host); cudaFreeHost(rt->mon_host);
  if (rt->declog) cudaFree(rt->declog);
  cudaEventDestroy(rt->done_ev);
  delete rt;
}

extern "C" int rrfp_runtime_inbox(rrfp_runtime* rt, void** dev_ptr, size_t* bytes) {
  if (!rt || !dev_ptr) return rrfp_fail(RRFP_E_INVALID, "null argument");
  *dev_ptr = rt->inbox;
  if (bytes) *bytes = sizeof(lane_inbox);
  return RRFP_OK;
}

extern "C" int rrfp_runtime_inbox_ipc(rrfp_runtime* rt, void* handle64) {
  if (!rt || !handle64) return rrfp_fail(RRFP_E_INVALID, "null argument");
  RRFP_CUDA_TRY(cudaSetDevice(rt->dev));
  cudaIpcMemHandle_t h;
  RRFP_CUDA_TRY(cudaIpcGetMemHandle(&h, rt->inbox));
  memcpy(handle64, &h, sizeof(h));
  return RRFP_OK;
}

extern "C" int rrfp_ipc_open(const void* handle64, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return rrfp_fail(RRFP_E_INVALID, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  RRFP_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return RRFP_OK;
}

// Unmap a peer buffer opened with rrfp_ipc_open (a later pipeline that opens the
// peer's next buffer -- possibly at the same address -- would otherwise fail with
// "resource already mapped").
extern "C" int rrfp_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return RRFP_OK;
  RRFP_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
  return RRFP_OK;
}

extern "C" int rrfp_ipc_alloc(size_t bytes, void** dev_ptr) {
  if (!dev_ptr || !bytes) return rrfp_fail(RRFP_E_INVALID, "bad ipc alloc");
  RRFP_CUDA_TRY(cudaMalloc(dev_ptr, bytes));
  RRFP_CUDA_TRY(cudaMemset(*dev_ptr, 0, bytes));
  return RRFP_OK;
}

extern "C" int rrfp_ipc_handle(void* dev_ptr, void* handle64) {
  if (!dev_ptr || !handle64) return rrfp_fail(RRFP_E_INVALID, "null argument");
  cudaIpcMemHandle_t h;
  RRFP_CUDA_TRY(cudaIpcGetMemHandle(&h, dev_ptr));
  memcpy(handle64, &h, sizeof(h));
  return RRFP_OK;
}

extern "C" void rrfp_ipc_free(void* dev_ptr) {
  if (dev_ptr) cudaFree(dev_ptr);
}

// all_lanes: N*R inbox pointers (lane index = stage*R + rank), used for the
// iteration barrier; fwd/bwd: R receivers each (NULL where no send exists).
extern "C" int rrfp_runtime_connect(rrfp_runtime* rt, void* const* fwd_dst, void* const* bwd_dst,
                                    void* const* tp_peer) {
  if (!rt) return rrfp_fail(RRFP_E_INVALID, "null runtime");
  RRFP_CUDA_TRY(cudaSetDevice(rt->dev));
  lane_state h;
  RRFP_CUDA_TRY(cudaMemcpy(&h, rt->L, sizeof(h), cudaMemcpyDeviceToHost));
  int R = rt->d.R, NL = rt->d.N * R;
  for (int r = 0; r < R; ++r) {
    h.fwd_dst[r] = fwd_dst && fwd_dst[r] ? (lane_inbox*)fwd_dst[r] : rt->inbox;
    h.bwd_dst[r] = bwd_dst && bwd_dst[r] ? (lane_inbox*)bwd_dst[r] : rt->inbox;
    h.tp_peer[r] = tp_peer && tp_peer[r] ? (lane_inbox*)tp_peer[r] : rt->inbox;
  }
  // the iteration-barrier list follows the R tp peers in tp_peer[R..R+NL)
  h.n_lanes = 1;
  h.all[0] = rt->inbox;
  if (tp_peer) {
    h.n_lanes = NL;
    for (int i = 0; i < NL; ++i) h.all[i] = tp_peer[R + i] ? (lane_inbox*)tp_peer[R + i] : rt->inbox;
  }
  // replay mode: the lanes whose messages reach this stage (any rank) --
  // F from the previous stage (from N-1 at stage 0 when C > 1: the chunk
  // wrap), B from the next (from 0 at N-1 when C > 1); never itself.
  {
    const int s = rt->d.stage, N = rt->d.N, C = rt->d.C;
    h.v_nin = 0;
    if (s > 0 || C > 1)
      for (int r = 0; r < R; ++r)
        if (h.bwd_dst[r] != rt->inbox) h.v_in[h.v_nin++] = h.bwd_dst[r];
    if (s < N - 1 || C > 1)
      for (int r = 0; r < R; ++r)
        if (h.fwd_dst[r] != rt->inbox) h.v_in[h.v_nin++] = h.fwd_dst[r];
  }
  RRFP_CUDA_TRY(cudaMemcpy(rt->L, &h, sizeof(h), cudaMemcpyHostToDevice));
  return RRFP_OK;
}

// dur_ns[3*KEYS]; comm_ns[2*KEYS] (indexed by the sending task);
// skew_ns[2*KEYS*R]: arrival skew at each destination rank, indexed by
// [send direction][destination key][rank].
extern "C" int rrfp_runtime_load_tables(rrfp_runtime* rt, const int64_t* dur_ns, const int64_t* comm_ns,
                                        const int64_t* skew_ns, const rrfp_task_t* fixed,
                                        const int64_t* min_ns) {
  if (!rt || !dur_ns || !comm_ns || !skew_ns) return rrfp_fail(RRFP_E_INVALID, "null table");
  RRFP_CUDA_TRY(cudaSetDevice(rt->dev));
  size_t K = rt->KEYS, R = rt->d.R;
  RRFP_CUDA_TRY(cudaMemcpy(rt->tables, dur_ns, sizeof(long long) * 3 * K, cudaMemcpyHostToDevice));
  RRFP_CUDA_TRY(cudaMemcpy(rt->tables + 3 * K, comm_ns, sizeof(long long) * 2 * K, cudaMemcpyHostToDevice));
  RRFP_CUDA_TRY(cudaMemcpy(rt->tables + 5 * K, skew_ns, sizeof(long long) * 2 * K * R,
                           cudaMemcpyHostToDevice));
  if (min_ns)
    RRFP_CUDA_TRY(cudaMemcpy(rt->tables + (5 + 2 * R) * K, min_ns, sizeof(long long) * 3 * K,
                             cudaMemcpyHostToDevice));
  else
    RRFP_CUDA_TRY(cudaMemset(rt->tables + (5 + 2 * R) * K, 0, sizeof(long long) * 3 * K));
  if (fixed && rt->d.per_stage > 0)
    RRFP_CUDA_TRY(cudaMemcpy(rt->fixed, fixed, sizeof(rrfp_task_t) * rt->d.per_stage,
                             cudaMemcpyHostToDevice));
  return RRFP_OK;
}

extern "C" int rrfp_runtime_set_bodies(rrfp_runtime* rt, void* const* graphs, int32_t n) {
  if (!rt || !graphs) return rrfp_fail(RRFP_E_INVALID, "null argument");
  if (rt->built) return rrfp_fail(RRFP_E_INVALID, "bodies must be set before the first launch");
  if (n != 3 * rt->d.M * rt->d.C)
    return rrfp_fail(RRFP_E_INVALID, "need 3*M*C body graphs, got %d", n);
  rt->bodies.assign(n, nullptr);
  for (int i = 0; i < n; ++i) rt->bodies[i] = (cudaGraph_t)graphs[i];
  return RRFP_OK;
}

extern "C" int rrfp_runtime_task_ptr(rrfp_runtime* rt, void** dev_ptr) {
  if (!rt || !dev_ptr) return rrfp_fail(RRFP_E_INVALID, "null argument");
  *dev_ptr = (char*)rt->L + offsetof(lane_state, cur_task);
  return RRFP_OK;
}

static int add_kernel(cudaGraphNode_t* node, cudaGraph_t g, const cudaGraphNode_t* dep, int ndep,
                      void* fn, lane_state* L) {
  cudaKernelNodeParams kp;
  memset(&kp, 0, sizeof(kp));
  void* args[1] = {&L};
  kp.func = fn;
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(32);
  kp.kernelParams = args;
  RRFP_CUDA_TRY(cudaGraphAddKernelNode(node, g, dep, ndep, &kp));
  return RRFP_OK;
}

static int build_graph(rrfp_runtime* rt) {
  cudaGraph_t g;
  RRFP_CUDA_TRY(cudaGraphCreate(&g, 0));
  cudaGraphNode_t n_init, n_while, n_final, n_dec, n_sw;
  int rc = add_kernel(&n_init, g, nullptr, 0, (void*)lane_init_kernel, rt->L);
  if (rc) return rc;
  cudaGraphConditionalHandle hw, hs;
  RRFP_CUDA_TRY(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hw;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  RRFP_CUDA_TRY(cudaGraphAddNode(&n_while, g, &n_init, 1, &cp));
  cudaGraph_t loop = cp.conditional.phGraph_out[0];
  if ((rc = add_kernel(&n_dec, loop, nullptr, 0, (void*)lane_step_kernel, rt->L))) return rc;
  RRFP_CUDA_TRY(cudaGraphConditionalHandleCreate(&hs, loop, 0xFFFFFFFFu, cudaGraphCondAssignDefault));
  cudaGraphNodeParams sp = {};
  sp.type = cudaGraphNodeTypeConditional;
  sp.conditional.handle = hs;
  sp.conditional.type = cudaGraphCondTypeSwitch;
  const bool per_mb = rt->d.compute_kind == 1;
  const int nb = per_mb ? 3 * rt->d.M * rt->d.C : 3;
  sp.conditional.size = nb;
  RRFP_CUDA_TRY(cudaGraphAddNode(&n_sw, loop, &n_dec, 1, &sp));
  for (int k = 0; k < nb; ++k) {
    cudaGraph_t b = sp.conditional.phGraph_out[k];
    cudaGraphNode_t n;
    if (per_mb) {
      cudaGraph_t body = k < (int)rt->bodies.size() ? rt->bodies[k] : nullptr;
      if (body) RRFP_CUDA_TRY(cudaGraphAddChildGraphNode(&n, b, nullptr, 0, body));
      else RRFP_CUDA_TRY(cudaGraphAddEmptyNode(&n, b, nullptr, 0));
    } else {
      if ((rc = add_kernel(&n, b, nullptr, 0, (void*)lane_spin_body_kernel, rt->L))) return rc;
    }
  }
  if ((rc = add_kernel(&n_final, g, &n_while, 1, (void*)lane_final_kernel, rt->L))) return rc;
  // store the handles in the device lane state
  RRFP_CUDA_TRY(cudaMemcpy((char*)rt->L + offsetof(lane_state, h_while), &hw, sizeof(hw),
                           cudaMemcpyHostToDevice));
  RRFP_CUDA_TRY(cudaMemcpy((char*)rt->L + offsetof(lane_state, h_switch), &hs, sizeof(hs),
                           cudaMemcpyHostToDevice));
  RRFP_CUDA_TRY(cudaGraphInstantiate(&rt->exec, g, 0));
  rt->graph = g;
  rt->built = true;
  return RRFP_OK;
}

// Build + instantiate + upload the lane graph while the device is idle (every
// lane of a job must be prepared before any lane is launched: a running lane
// spins on its peers, and graph instantiation/upload must not queue behind it).
// A lane whose stream belongs to a green context (single-GPU pipeline emulation,
// green.cu) builds its graph with that context current, so the dispatcher's
// kernel nodes share the context of the captured bodies (a conditional body
// mixing contexts does not instantiate).
static int build_graph_on_stream_ctx(rrfp_runtime* rt, cudaStream_t st) {
  using get_g_t = CUresult (*)(CUstream, CUgreenCtx*);
  using from_g_t = CUresult (*)(CUcontext*, CUgreenCtx);
  using push_t = CUresult (*)(CUcontext);
  using pop_t = CUresult (*)(CUcontext*);
  static get_g_t get_g = nullptr;
  static from_g_t from_g = nullptr;
  static push_t push = nullptr;
  static pop_t pop = nullptr;
  static bool looked = false;
  if (!looked) {
    looked = true;
    cudaDriverEntryPointQueryResult q;
    void* p;
    if (cudaGetDriverEntryPoint("cuStreamGetGreenCtx", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) get_g = (get_g_t)p;
    if (cudaGetDriverEntryPoint("cuCtxFromGreenCtx", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) from_g = (from_g_t)p;
    if (cudaGetDriverEntryPoint("cuCtxPushCurrent", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) push = (push_t)p;
    if (cudaGetDriverEntryPoint("cuCtxPopCurrent", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) pop = (pop_t)p;
  }
  CUgreenCtx g = nullptr;
  CUcontext c = nullptr;
  if (get_g && from_g && push && pop && st && get_g((CUstream)st, &g) == CUDA_SUCCESS && g &&
      from_g(&c, g) == CUDA_SUCCESS && c) {
    if (push(c) != CUDA_SUCCESS) return rrfp_fail(RRFP_E_CUDA, "cuCtxPushCurrent(green) failed");
    int rc = build_graph(rt);
    CUcontext dummy;
    pop(&dummy);
    return rc;
  }
  return build_graph(rt);
}

extern "C" int rrfp_runtime_prepare(rrfp_runtime* rt, void* stream) {
  if (!rt) return rrfp_fail(RRFP_E_INVALID, "null runtime");
  RRFP_CUDA_TRY(cudaSetDevice(rt->dev));
  if (!rt->built) {
    int rc = build_graph_on_stream_ctx(rt, (cudaStream_t)stream);
    if (rc) return rc;
  }
  RRFP_CUDA_TRY(cudaGraphUpload(rt->exec, (cudaStream_t)stream));
  RRFP_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return RRFP_OK;
}

extern "C" int rrfp_runtime_launch(rrfp_runtime* rt, int64_t epoch, void* stream) {
  if (!rt) return rrfp_fail(RRFP_E_INVALID, "null runtime");
  RRFP_CUDA_TRY(cudaSetDevice(rt->dev));
  (void)epoch;
  if (!rt->built) {
    int rc = build_graph_on_stream_ctx(rt, (cudaStream_t)stream);
    if (rc) return rc;
  }
  *rt->abort_host = 0;
  RRFP_CUDA_TRY(cudaGraphLaunch(rt->exec, (cudaStream_t)stream));
  RRFP_CUDA_TRY(cudaEventRecord(rt->done_ev, (cudaStream_t)stream));
  return RRFP_OK;
}

extern "C" int rrfp_runtime_wait(rrfp_runtime* rt, double watchdog_secs, rrfp_event* events,
                                 int32_t cap, int32_t* n_events, int64_t* t0_ns) {
  if (!rt) return rrfp_fail(RRFP_E_INVALID, "null runtime");
  RRFP_CUDA_TRY(cudaSetDevice(rt->dev));
  struct timespec a, b;
  clock_gettime(CLOCK_MONOTONIC, &a);
  bool fired = false;
  while (true) {
    cudaError_t q = cudaEventQuery(rt->done_ev);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) return rrfp_fail(RRFP_E_CUDA, "lane: %s", cudaGetErrorString(q));
    clock_gettime(CLOCK_MONOTONIC, &b);
    double el = (b.tv_sec - a.tv_sec) + 1e-9 * (b.tv_nsec - a.tv_nsec);
    if (!fired && watchdog_secs > 0 && el > watchdog_secs) {
      *(volatile int32_t*)rt->abort_host = 1;  // dispatcher exits its loop
      fired = true;
    }
    if (fired && el > watchdog_secs + 10.0) {
      volatile int32_t* m = rt->mon_host;
      const char* where[] = {"?", "dispatch", "body", "complete", "final"};
      int w = m[0] >= 0 && m[0] <= 4 ? m[0] : 0;
      rrfp_task_t t = (rrfp_task_t)m[1];
      return rrfp_fail(RRFP_E_WATCHDOG,
                       "lane stage %d rank %d stuck in %s (task %c mb %d chunk %d), remaining %d, epoch %d",
                       rt->d.stage, rt->d.rank, where[w], "BFW?"[rrfp_task_dir(t)], rrfp_task_mb(t),
                       rrfp_task_chunk(t), m[2], m[3]);
    }
    struct timespec ts = {0, 20000};
    nanosleep(&ts, nullptr);
  }
  lane_state h;
  RRFP_CUDA_TRY(cudaMemcpy(&h, rt->L, sizeof(h), cudaMemcpyDeviceToHost));
  int n = h.ring_n < h.ring_cap ? h.ring_n : h.ring_cap;
  if (n > cap) n = cap;
  if (events && n > 0)
    RRFP_CUDA_TRY(cudaMemcpy(events, rt->ring, sizeof(rrfp_event) * n, cudaMemcpyDeviceToHost));
  if (n_events) *n_events = n;
  if (t0_ns) *t0_ns = (int64_t)h.t_iter0;
  if (h.status == RRFP_E_DEADLOCK && !fired)
    return rrfp_fail(RRFP_E_DEADLOCK, "replay: stage %d rank %d quiescent with %d unfinished tasks",
                     rt->d.stage, rt->d.rank, h.remaining);
  if (fired || h.status == RRFP_E_WATCHDOG)
    return rrfp_fail(RRFP_E_WATCHDOG, "watchdog: stage %d rank %d remaining=%d n_f=%d n_b=%d",
                     rt->d.stage, rt->d.rank, h.remaining, h.n_f, h.n_b);
  if (h.ring_n > h.ring_cap) return rrfp_fail(RRFP_E_CAPACITY, "trace ring overflow");
  return RRFP_OK;
}

// Dispatcher profile: cap records of {step-kernel entry, completion done, decision
// made, kind << 32 | view polls} (%globaltimer ns) per lane_step_kernel run of the
// next iterations (cap = 0 disables).  Device-side stamps: ncu does not profile
// the kernel nodes of a graph with conditional nodes.
extern "C" int rrfp_runtime_profile(rrfp_runtime* rt, int32_t cap) {
  if (!rt || cap < 0) return rrfp_fail(RRFP_E_INVALID, "bad argument");
  RRFP_CUDA_TRY(cudaSetDevice(rt->dev));
  unsigned long long* buf = nullptr;
  unsigned long long* old = nullptr;
  RRFP_CUDA_TRY(cudaMemcpy(&old, (char*)rt->L + offsetof(lane_state, prof), sizeof(old), cudaMemcpyDeviceToHost));
  if (old) RRFP_CUDA_TRY(cudaFree(old));
  if (cap > 0) RRFP_CUDA_TRY(cudaMalloc(&buf, sizeof(unsigned long long) * 4 * (size_t)cap));
  RRFP_CUDA_TRY(cudaMemcpy((char*)rt->L + offsetof(lane_state, prof), &buf, sizeof(buf), cudaMemcpyHostToDevice));
  RRFP_CUDA_TRY(cudaMemcpy((char*)rt->L + offsetof(lane_state, prof_cap), &cap, sizeof(cap), cudaMemcpyHostToDevice));
  return RRFP_OK;
}

extern "C" int rrfp_runtime_profile_read(rrfp_runtime* rt, uint64_t* out, int32_t cap, int32_t* n_records) {
  if (!rt || !n_records) return rrfp_fail(RRFP_E_INVALID, "null argument");
  RRFP_CUDA_TRY(cudaSetDevice(rt->dev));
  lane_state h;
  RRFP_CUDA_TRY(cudaMemcpy(&h, rt->L, sizeof(h), cudaMemcpyDeviceToHost));
  int n = h.prof ? (h.prof_n < h.prof_cap ? h.prof_n : h.prof_cap) : 0;
  if (n > cap) n = cap;
  if (n > 0 && out)
    RRFP_CUDA_TRY(cudaMemcpy(out, h.prof, sizeof(uint64_t) * 4 * (size_t)n, cudaMemcpyDeviceToHost));
  *n_records = n;
  return RRFP_OK;
}

extern "C" int rrfp_runtime_declog(rrfp_runtime* rt, uint32_t* out, int32_t cap_words, int32_t* n_records,
                                   int32_t* stride_words) {
  if (!rt || !n_records) return rrfp_fail(RRFP_E_INVALID, "null argument");
  RRFP_CUDA_TRY(cudaSetDevice(rt->dev));
  const int stride = 16 + 5 * rt->d.C * rt->d.MW;
  if (stride_words) *stride_words = stride;
  *n_records = 0;
  if (!rt->declog) return RRFP_OK;
  int32_t n = 0;
  RRFP_CUDA_TRY(cudaMemcpy(&n, (char*)rt->L + offsetof(lane_state, declog_n), sizeof(n), cudaMemcpyDeviceToHost));
  if (n > rt->d.declog_cap) return rrfp_fail(RRFP_E_CAPACITY, "decision log overflow (%d > %d)", n, rt->d.declog_cap);
  if (out && (long long)n * stride > cap_words) return rrfp_fail(RRFP_E_CAPACITY, "output buffer too small");
  if (n > 0 && out)
    RRFP_CUDA_TRY(cudaMemcpy(out, rt->declog, sizeof(uint32_t) * (size_t)n * stride, cudaMemcpyDeviceToHost));
  *n_records = n;
  return RRFP_OK;
}

// Reads only the host-mapped monitor block: safe while the GPU is busy or hung.
extern "C" int rrfp_runtime_status(rrfp_runtime* rt, char* dump, size_t cap) {
  if (!rt) return rrfp_fail(RRFP_E_INVALID, "null runtime");
  volatile int32_t* m = rt->mon_host;
  const char* where[] = {"idle", "dispatch", "body", "complete", "final"};
  int w = m[0] >= 0 && m[0] <= 4 ? m[0] : 0;
  rrfp_task_t t = (rrfp_task_t)m[1];
  if (dump && cap)
    snprintf(dump, cap, "stage %d rank %d: epoch=%d where=%s last_task=%c%d.%d remaining=%d",
             rt->d.stage, rt->d.rank, m[3], where[w], "BFW?"[rrfp_task_dir(t)], rrfp_task_mb(t),
             rrfp_task_chunk(t), m[2]);
  return RRFP_OK;
}

__global__ void spin_kernel(long long ns) {
  unsigned long long t0 = gtimer();
  spin_until(t0 + (unsigned long long)ns);
}

extern "C" int rrfp_spin(int64_t ns, void* stream) {
  spin_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(ns);
  RRFP_CUDA_TRY(cudaGetLastError());
  return RRFP_OK;
}
