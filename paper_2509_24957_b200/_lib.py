"""ctypes binding of the C-ABI in include/duchess_b200.h.

The library is built in-tree (``make`` or ``__graft_entry__.build()``) as
``paper_2509_24957_b200/libduchess_b200.so``. There is no CPU fallback: if the
library is missing, or no CUDA device is present when a kernel is launched,
the call raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libduchess_b200.so"

DUCHESS_OK = 0
F32, BF16, F64 = 0, 1, 2
ACTIVE, EARLY_TERMINATED, NATURAL_END, CAPPED, CANCELLED = range(5)
REASON_NONE, REASON_CONSENSUS, REASON_COVERAGE, REASON_EXHAUSTED = range(4)
ACT_CONTINUE, ACT_TERMINATE, ACT_BRANCH_OUT = 1, 2, 3
PRED_DEVICE, PRED_TRACE, PRED_HOST = 0, 1, 2
FLAG_EXACT_CDF = 1
SCORE_NO_INPUT_WAIT = 1
POLICY_DUCHESS, POLICY_DEFAULT_SC, POLICY_SHORT_MK, POLICY_DYNASOR = 0, 1, 2, 3
MT_WORDS = 625
MAX_SLOTS = 64
REC_WORDS = 12
(REC_ROUND, REC_DECODING, REC_MAX_CHUNK, REC_DECODE, REC_PROBES, REC_NACTIONS, REC_DONE,
 REC_NFORKS, REC_NSURV, REC_REQ, REC_REASON, REC_FINAL) = range(12)
CNT_AMBIGUOUS, CNT_ERRORS, CNT_FINISHED, CNT_BRANCH_STEPS, CNT_FORKS, CNT_NEAR_TAU = range(6)
N_COUNTERS = 8

_i32p = C.POINTER(C.c_int32)
_u32p = C.POINTER(C.c_uint32)
_f64p = C.POINTER(C.c_double)


class Policy(C.Structure):
    _fields_ = [
        ("max_branches", C.c_int32), ("interval_tokens", C.c_int32),
        ("early_term_rounds", C.c_int32), ("token_cap", C.c_int32),
        ("probe_cost_tokens", C.c_int32), ("need_consensus", C.c_int32),
        ("need_coverage", C.c_int32), ("pred_source", C.c_int32),
        ("n_layers", C.c_int32), ("combine", C.c_int32),
        ("flags", C.c_int32), ("policy_kind", C.c_int32), ("short_m", C.c_int32),
        ("dynasor_window", C.c_int32), ("_pad2", C.c_int32 * 2),
        ("early_term_threshold", C.c_double), ("inv_temperature", C.c_double),
        ("rho", C.c_double),
    ]


class Workload(C.Structure):
    _fields_ = [
        ("n_requests", C.c_int32), ("queue_len", C.c_int32), ("cycle", C.c_int32),
        ("_pad", C.c_int32),
        ("tmpl_off", C.c_void_p), ("ground_truth", C.c_void_p), ("mt_init", C.c_void_p),
        ("nat_len", C.c_void_p), ("final_ans", C.c_void_p), ("conv", C.c_void_p),
        ("probe_off", C.c_void_p), ("probe_at", C.c_void_p), ("probe_ans", C.c_void_p),
        ("pred_off", C.c_void_p), ("pred_at", C.c_void_p), ("pred_p", C.c_void_p),
        ("queue", C.c_void_p), ("queue_rec", C.c_void_p),
    ]


STATE_PTR_FIELDS = [
    "slot_req", "needs_refill", "n_branches", "next_template", "tokens_decode",
    "tokens_probe", "rounds", "done", "tally", "mt",
    "br_offset", "br_decoded", "br_streak", "br_status", "br_final", "br_npred", "br_slot",
    "br_last_pred", "br_probe_last", "br_probe_run", "slot_aux",
    "slot_branch", "row_mask", "row_pos", "row_tmpl", "row_req",
    "p1_rec", "round_rec", "actions", "forks", "step_pred", "queue_head", "active_rows", "active_count",
    "out_final", "out_reason", "out_tokens_decode", "out_tokens_probe", "out_rounds",
    "out_error", "out_tally", "counters", "trace",
]


class State(C.Structure):
    _fields_ = [("n_slots", C.c_int32), ("branch_cap", C.c_int32),
                ("answer_cap", C.c_int32), ("_pad", C.c_int32)] + [
        (name, C.c_void_p) for name in STATE_PTR_FIELDS]


KV_CNT_ALLOC, KV_CNT_FREE, KV_CNT_TAIL_BYTES, KV_CNT_OVERFLOW = range(4)
KV_N_COUNTERS = 4
KV_OVERLAP = 1
KV_LEAD = 2
TRACE_WORDS = 24    # DUCHESS_TRACE_WORDS
KV_PTR_FIELDS = ["table", "kv_tokens", "refcount", "free_stack", "arena", "jobs", "job_count",
                 "kv_pool", "counters"]


class KV(C.Structure):
    _fields_ = [("block_tokens", C.c_int32), ("blocks_per_slot", C.c_int32),
                ("max_blocks", C.c_int32), ("flags", C.c_int32),
                ("kv_bytes_per_token", C.c_int64)] + [(n, C.c_void_p) for n in KV_PTR_FIELDS]


SYMBOLS = {
    # name: (restype, argtypes)
    "duchess_score_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int32]),
    "duchess_score": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_size_t, C.c_int32, C.c_int32, C.c_void_p]),
    "duchess_score_list": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                     C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p]),
    "duchess_score_active": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                       C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p]),
    "duchess_score_active_ex": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                       C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_int32, C.c_void_p]),
    "duchess_gather_active": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                        C.c_void_p, C.c_int64, C.c_void_p]),
    "duchess_upload_rows": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                      C.c_int32, C.c_int64, C.c_void_p]),
    "duchess_fill_activations": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int32,
                                           C.c_int32, C.c_int32, C.c_int64, C.c_int64,
                                           C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p]),
    "duchess_advance": (C.c_int, [C.POINTER(Policy), C.POINTER(Workload), C.POINTER(State),
                                  C.c_void_p]),
    "duchess_decide": (C.c_int, [C.POINTER(Policy), C.POINTER(Workload), C.POINTER(State),
                                 C.c_void_p, C.c_void_p]),
    "duchess_round": (C.c_int, [C.POINTER(Policy), C.POINTER(Workload), C.POINTER(State),
                                C.c_void_p, C.c_void_p]),
    "duchess_read_stream": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "duchess_gate": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "duchess_write_stream": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint32, C.c_void_p]),
    "duchess_baseline_round": (C.c_int, [C.POINTER(Policy), C.POINTER(Workload),
                                         C.POINTER(State), C.c_void_p]),
    "duchess_branch_out_sample": (C.c_int, [C.c_void_p, C.c_int32, C.c_double, C.c_void_p,
                                            C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p]),
    "duchess_vote": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                               C.c_void_p, C.c_void_p, C.c_void_p]),
    "duchess_template_lookup": (C.c_int, [C.POINTER(Workload), C.c_void_p, C.c_void_p,
                                          C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "duchess_sort_keys_workspace_bytes": (C.c_size_t, [C.c_int64]),
    "duchess_sort_keys": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_size_t,
                                    C.c_void_p]),
    "duchess_sort_difficulty": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                          C.c_void_p]),
    "duchess_fork_workspace_bytes": (C.c_size_t, [C.c_int32, C.c_int32]),
    "duchess_fork_cow": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                                   C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                   C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "duchess_kv_round": (C.c_int, [C.POINTER(Policy), C.POINTER(State), C.POINTER(KV),
                                   C.c_void_p]),
    "duchess_lr_grad_workspace_bytes": (C.c_size_t, [C.c_int32]),
    "duchess_lr_grad": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64,
                                  C.c_int32, C.c_float, C.c_void_p, C.c_void_p, C.c_size_t,
                                  C.c_void_p]),
    "duchess_sgd_update": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_float,
                                     C.c_void_p]),
    "duchess_synthetic_predict": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_double,
                                            C.c_void_p, C.c_void_p]),
    "duchess_confused_level": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p]),
    "duchess_mt_seed": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "duchess_confused_levels": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]),
    "duchess_timeline": (C.c_int, [C.c_void_p, C.c_int32, C.c_double, C.c_double, C.c_int64,
                                   C.c_void_p, C.c_void_p, C.c_void_p]),
    "duchess_early_termination": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_double,
                                            C.c_int32, C.c_void_p, C.c_void_p]),
    "duchess_mlp_forward": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_int32,
                                      C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.c_void_p,
                                      C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "duchess_mlp_probe_tc_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int32]),
    "duchess_mlp_probe_tc": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int32,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_float,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                       C.c_void_p]),
    "duchess_mlp_probe_tc_grouped_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int32,
                                                                    C.c_int32]),
    "duchess_mlp_probe_tc_grouped": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                               C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                               C.c_void_p]),
    "duchess_tc_linear_grouped_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int32, C.c_int32]),
    "duchess_tc_linear_grouped": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                            C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t,
                                            C.c_void_p]),
    "duchess_tc_linear_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int32]),
    "duchess_tc_linear": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int32,
                                    C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "duchess_row_normalize": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int32,
                                        C.c_void_p, C.c_void_p]),
    "duchess_head_logits": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_int32, C.c_void_p, C.c_void_p]),
    "duchess_version": (C.c_char_p, []),
    "duchess_device_arch": (C.c_int, []),
}

_LIB: C.CDLL | None = None


class DuchessError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


def load() -> C.CDLL:
    """Load the in-tree sm_100a library; raises if it was not built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = Path(os.environ.get("DUCHESS_B200_LIB", LIB_PATH))
    if not path.exists():
        raise ImportError(
            f"duchess_b200 CUDA library not found at {path}; build it with `make` "
            f"(or __graft_entry__.build()). There is no CPU fallback.")
    lib = C.CDLL(str(path))
    for name, (restype, argtypes) in SYMBOLS.items():
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    _LIB = lib
    return lib


def check(status: int, what: str) -> None:
    if status != DUCHESS_OK:
        raise DuchessError(f"{what} failed with status {status}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda(tensor=None) -> None:
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("duchess_b200 needs a CUDA device (sm_100a); no CPU fallback")
    if tensor is not None and not tensor.is_cuda:
        raise ValueError("expected a CUDA tensor")
