"""ctypes binding of the C-ABI library `_rrfp_b200.so` (include/rrfp_b200.h).

The library is built in-tree by `paper_2605_18750_b200.build`.  There is no
fallback: if the library is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_rrfp_b200.so")

MAX_STAGES = 32
MAX_RANKS = 8
MAX_WORDS = 128
MAX_RANKED = 8
E_CODES = {0: "ok", -1: "invalid", -2: "deadlock", -3: "watchdog", -4: "cuda",
           -5: "capacity", -6: "nogpu"}

DIR_B, DIR_F, DIR_W, WAIT = 0, 1, 2, 3
DIR_CODE = {"B": DIR_B, "F": DIR_F, "W": DIR_W}
CODE_DIR = {DIR_B: "B", DIR_F: "F", DIR_W: "W", WAIT: "wait"}
HINT_CODE = {"bf": 0, "fb": 1, "bprio": 2, "fprio": 3, "bfw": 4, "external": 5}


class Hint(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_ranked", C.c_int32),
                ("ranked_dir", C.c_int32 * MAX_RANKED), ("ranked_desc", C.c_int32 * MAX_RANKED)]


class StageState(C.Structure):
    _fields_ = [("M", C.c_int32), ("C", C.c_int32), ("MW", C.c_int32), ("decompose", C.c_int32),
                ("admission", C.c_int32), ("mode", C.c_int32), ("focus", C.c_int32),
                ("phase", C.c_int32),
                ("fready", C.c_uint32 * MAX_WORDS), ("bready", C.c_uint32 * MAX_WORDS),
                ("wpend", C.c_uint32 * MAX_WORDS), ("doneF", C.c_uint32 * MAX_WORDS),
                ("doneB", C.c_uint32 * MAX_WORDS)]


class Decision_(C.Structure):
    _fields_ = [("kind", C.c_int32), ("mb", C.c_int32), ("chunk", C.c_int32)]


class IterDesc(C.Structure):
    _fields_ = [("N", C.c_int32), ("M", C.c_int32), ("C", C.c_int32), ("R", C.c_int32),
                ("MW", C.c_int32), ("decompose", C.c_int32), ("buffer_limit", C.c_int32),
                ("fixed_mode", C.c_int32), ("per_stage", C.c_int32), ("pad0", C.c_int32),
                ("coord_cost", C.c_int64), ("hint", Hint)]


class Event(C.Structure):
    _fields_ = [("t0", C.c_int64), ("t1", C.c_int64), ("kind", C.c_int32), ("stage", C.c_int32),
                ("rank", C.c_int32), ("task", C.c_uint32)]


class ReplayResult(C.Structure):
    _fields_ = [("makespan", C.c_int64), ("agreed", C.c_int64), ("deferred", C.c_int64),
                ("status", C.c_int32), ("n_events", C.c_int32),
                ("compute", C.c_int64 * MAX_STAGES), ("coord", C.c_int64 * MAX_STAGES),
                ("n_f", C.c_int32 * MAX_STAGES), ("n_b", C.c_int32 * MAX_STAGES),
                ("n_w", C.c_int32 * MAX_STAGES), ("remaining", C.c_int32 * MAX_STAGES)]


class LaneDesc(C.Structure):
    _fields_ = [("N", C.c_int32), ("M", C.c_int32), ("C", C.c_int32), ("R", C.c_int32),
                ("MW", C.c_int32), ("decompose", C.c_int32), ("buffer_limit", C.c_int32),
                ("fixed_mode", C.c_int32), ("per_stage", C.c_int32), ("stage", C.c_int32),
                ("rank", C.c_int32), ("device", C.c_int32), ("compute_kind", C.c_int32),
                ("trace_cap", C.c_int32), ("time_scale", C.c_double),
                ("coord_cost_ns", C.c_int64), ("hint", Hint),
                ("virtual_clock", C.c_int32), ("declog_cap", C.c_int32),
                ("v_dmin", C.c_int64), ("v_la", C.c_int64), ("v_horizon", C.c_int64)]


EVENT_KINDS = {0: "exec", 1: "send", 2: "recv", 3: "coord", 4: "coord"}

# exported symbols declared in include/rrfp_b200.h (checked by the CPU test-suite)
EXPORTS = [
    "rrfp_arbitrate", "rrfp_next_by_priority", "rrfp_update_backpressure", "rrfp_replay_workspace_bytes",
    "rrfp_replay_event_capacity", "rrfp_replay_host", "rrfp_replay_device",
    "rrfp_runtime_create", "rrfp_runtime_destroy", "rrfp_runtime_inbox", "rrfp_runtime_inbox_ipc",
    "rrfp_ipc_open", "rrfp_ipc_close", "rrfp_ipc_alloc", "rrfp_ipc_handle", "rrfp_ipc_free", "rrfp_runtime_connect", "rrfp_runtime_load_tables", "rrfp_runtime_set_bodies",
    "rrfp_runtime_task_ptr", "rrfp_runtime_prepare", "rrfp_runtime_launch", "rrfp_runtime_wait", "rrfp_runtime_status", "rrfp_runtime_declog", "rrfp_runtime_profile", "rrfp_runtime_profile_read",
    "rrfp_spin", "rrfp_last_error", "rrfp_abi_version", "rrfp_gemm_bf16", "rrfp_gemm_set_variant", "rrfp_set_pdl",
    "rrfp_gemm_reserve_sms", "rrfp_gemm_set_epilogue", "rrfp_gemm_set_streamk", "rrfp_gemm_set_tail_split", "rrfp_gemm_set_multicast", "rrfp_gemm_max_clusters", "rrfp_gemm_set_bk", "rrfp_gemm_set_small", "rrfp_gemm_set_rpref", "rrfp_layernorm_fwd", "rrfp_layernorm_bwd", "rrfp_layernorm_bwd_fused", "rrfp_xent_combine", "rrfp_embedding_fwd",
    "rrfp_embedding_bwd", "rrfp_bias_grad", "rrfp_copy_rows", "rrfp_xent_fwd", "rrfp_xent_bwd", "rrfp_attn_fwd", "rrfp_attn_debug", "rrfp_attn_bwd", "rrfp_attn_bwd_workspace_bytes",
    "rrfp_tp_create", "rrfp_tp_buffers", "rrfp_tp_connect", "rrfp_tp_allreduce", "rrfp_tp_error",
    "rrfp_tp_destroy", "rrfp_clock_pingpong", "rrfp_enable_peer_access", "rrfp_green_streams", "rrfp_green_destroy",
]

_lib = None


class RrfpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"rrfp error {code} ({E_CODES.get(code, '?')}): {msg}")
        self.code = code


def lib():
    """Load the library (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2605_18750_b200.build`")
        L = C.CDLL(LIB_PATH)
        L.rrfp_last_error.restype = C.c_char_p
        L.rrfp_replay_workspace_bytes.restype = C.c_size_t
        L.rrfp_replay_event_capacity.restype = C.c_int32
        L.rrfp_attn_bwd_workspace_bytes.restype = C.c_size_t
        L.rrfp_runtime_destroy.restype = None
        L.rrfp_ipc_free.restype = None
        L.rrfp_tp_destroy.restype = None
        _lib = L
    return _lib


def check(rc):
    if rc != 0:
        raise RrfpError(rc, lib().rrfp_last_error().decode())
    return rc


def make_hint(hint) -> Hint:
    h = Hint()
    h.kind = HINT_CODE[hint.kind]
    h.n_ranked = len(hint.ranked)
    if h.n_ranked > MAX_RANKED:
        raise ValueError("at most 8 ranked hint entries")
    for i, (d, rule) in enumerate(hint.ranked):
        h.ranked_dir[i] = DIR_CODE[d]
        h.ranked_desc[i] = 1 if rule == "desc" else 0
    return h


def task_code(d: str, stage: int, mb: int, chunk: int) -> int:
    return (DIR_CODE[d] & 3) | ((chunk & 15) << 2) | ((mb & 1023) << 6) | ((stage & 63) << 16)


def task_fields(code: int):
    return CODE_DIR[code & 3], (code >> 16) & 63, (code >> 6) & 1023, (code >> 2) & 15
