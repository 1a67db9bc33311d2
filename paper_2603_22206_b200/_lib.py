"""ctypes binding of libchimera_sm100a.so (declared in include/chimera_b200.h).

The structs below mirror the C structs field for field. Pointers are passed
as integers taken from torch tensors (`tensor.data_ptr()`); streams as the raw
`cudaStream_t` handle (`torch.cuda.current_stream().cuda_stream`).

There is no fallback: if the shared library is missing, importing the GPU
path raises immediately.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int32, c_int64, c_uint32, c_void_p

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libchimera_sm100a.so")

MAX_MODELS = 8
MAX_STAGES = 32

# chm_status codes (include/chimera_b200.h)
CHM_OK = 0
CHM_ERR_INVALID_ARG = 1
CHM_ERR_VALIDATION = 2
CHM_ERR_NEGATIVE_PREDICTION = 3
CHM_ERR_DUPLICATE_REQUEST = 4
CHM_ERR_TIME_BACKWARDS = 5
CHM_ERR_NAN_PREDICTION = 6
CHM_ERR_INVALID_STATE = 7
CHM_ERR_CAPACITY = 8
CHM_ERR_UNSUPPORTED = 9
CHM_ERR_CUDA = 10
CHM_ERR_UNKNOWN_REQUEST = 11
CHM_ERR_UNKNOWN_STAGE = 12
CHM_ERR_NCCL = 13
COMM_ID_BYTES = 128


class Pool(ctypes.Structure):
    _fields_ = [
        ("n_models", c_int32),
        ("max_batch_size", c_int32 * MAX_MODELS),
        ("decode_ms_per_token", c_double * MAX_MODELS),
    ]


class BalancerCfg(ctypes.Structure):
    _fields_ = [("latency_slack", c_double), ("confidence_margin", c_double),
                ("tie_tolerance", c_double)]


class AgingCfg(ctypes.Structure):
    _fields_ = [
        ("enabled", c_int32),
        ("starvation_threshold", c_int32),
        ("running_quantum", c_int32),
        ("demote_while_queued", c_int32),
    ]


class MonitorState(ctypes.Structure):
    _fields_ = [
        ("n_programs", c_int32),
        ("inflight_sum", c_void_p),
        ("inflight_comp", c_void_p),
        ("inflight_count", c_void_p),
        ("assignment", c_void_p),
        ("stage_bits", c_void_p),
        ("batch_stamp", c_void_p),
        ("engine_clock", c_void_p),
        ("engine_seq", c_void_p),
        ("engine_running", c_void_p),
        ("engine_queued", c_void_p),
        ("engine_iterations", c_void_p),
        ("inflight_capacity", c_int32),
        ("inflight_key", c_void_p),
        ("inflight_yhat", c_void_p),
        ("inflight_progress", c_void_p),
        ("inflight_stamp", c_void_p),
        ("stamp_base", c_void_p),
    ]


class Rows(ctypes.Structure):
    _fields_ = [
        ("n_rows", c_int32),
        ("program", c_void_p),
        ("stage", c_void_p),
        ("arrival", c_void_p),
        ("out_tokens", c_void_p),
        ("handle", c_void_p),
        ("input_tokens", c_void_p),
    ]


class RowScratch(ctypes.Structure):
    _fields_ = [
        ("first_row", c_void_p),
        ("pre_model", c_void_p),
        ("route_rows", c_void_p),
        ("n_route", c_void_p),
        ("qual", c_void_p),
        ("rank", c_void_p),
        ("flags", c_void_p),
        ("lnew", c_void_p),
    ]


class Decisions(ctypes.Structure):
    _fields_ = [
        ("model", c_void_p),
        ("priority", c_void_p),
        ("flags", c_void_p),
        ("seq", c_void_p),
        ("loads", c_void_p),
        ("n_committed", c_void_p),
        ("error", c_void_p),
        ("tie_counts", c_void_p),
    ]


class QueueState(ctypes.Structure):
    _fields_ = [
        ("capacity", c_int32),
        ("priority", c_void_p),
        ("arrival", c_void_p),
        ("seq", c_void_p),
        ("handle", c_void_p),
        ("out_tokens", c_void_p),
        ("level", c_void_p),
        ("count", c_void_p),
        ("quantum", c_void_p),
        ("order", c_void_p),
        ("admitted", c_void_p),
        ("n_admitted", c_void_p),
        ("n_promoted", c_void_p),
        ("arrival_unsorted", c_void_p),
        ("scratch", c_void_p),
        ("run", c_void_p),
    ]


class EngineRun(ctypes.Structure):
    _fields_ = [
        ("capacity", c_int32),
        ("done_capacity", c_int32),
        ("prefill_ms_per_token", c_double * MAX_MODELS),
        ("queue_input_tokens", c_void_p),
        ("handle", c_void_p),
        ("seq", c_void_p),
        ("stint_end", c_void_p),
        ("decode_start", c_void_p),
        ("stint_tokens", c_void_p),
        ("n", c_void_p),
        ("tokens_emitted", c_void_p),
        ("served", c_void_p),
        ("done_handle", c_void_p),
        ("done_time", c_void_p),
        ("n_done", c_void_p),
    ]



class Trace(ctypes.Structure):
    _fields_ = [
        ("n_programs", c_int32),
        ("max_stages", c_int32),
        ("n_models", c_int32),
        ("n_stages", c_void_p),
        ("workflow", c_void_p),
        ("user_arrival", c_void_p),
        ("base_input", c_void_p),
        ("out_tokens", c_void_p),
        ("carried", c_void_p),
        ("remaining", c_void_p),
        ("carried_prefix", c_void_p),
    ]


class EncoderCfg(ctypes.Structure):
    _fields_ = [
        ("n_layers", c_int32),
        ("hidden", c_int32),
        ("n_heads", c_int32),
        ("ffn", c_int32),
        ("vocab", c_int32),
        ("max_pos", c_int32),
        ("n_models", c_int32),
        ("ln_eps", c_float),
        ("flags", c_int32),
    ]


ENC_UNFUSED_ATTENTION = 1
ENC_CLUSTER_LN = 2
ENC_DEFERRED_LN = 4


class EncoderWeights(ctypes.Structure):
    _fields_ = [
        ("word_emb", c_void_p),
        ("pos_emb", c_void_p),
        ("type_emb", c_void_p),
        ("emb_ln_g", c_void_p),
        ("emb_ln_b", c_void_p),
        ("w_qkv", c_void_p),
        ("b_qkv", c_void_p),
        ("w_o", c_void_p),
        ("b_o", c_void_p),
        ("ln1_g", c_void_p),
        ("ln1_b", c_void_p),
        ("w_1", c_void_p),
        ("b_1", c_void_p),
        ("w_2", c_void_p),
        ("b_2", c_void_p),
        ("ln2_g", c_void_p),
        ("ln2_b", c_void_p),
        ("head_w", c_void_p),
        ("head_b", c_void_p),
    ]


class EncoderWorkspace(ctypes.Structure):
    _fields_ = [
        ("max_tokens", c_int64),
        ("x", c_void_p),
        ("qkv", c_void_p),
        ("ctx", c_void_p),
        ("tmp", c_void_p),
        ("ffn", c_void_p),
        ("stats", c_void_p),
        ("folded", c_void_p),
    ]


# (name, restype, argtypes) of every exported symbol declared in the header.
_SIGNATURES = [
    ("chm_version", c_char_p, []),
    ("chm_status_string", c_char_p, [c_int32]),
    ("chm_device_info", c_int32, [c_int32, POINTER(c_int32), POINTER(c_int32), POINTER(c_int32)]),
    ("chm_prepare_rows", c_int32,
     [POINTER(MonitorState), POINTER(Rows), POINTER(RowScratch), c_void_p, c_void_p]),
    ("chm_predict_quantile", c_int32,
     [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_int32, c_void_p, c_void_p]),
    ("chm_predict_oracle", c_int32,
     [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
    ("chm_predict_input_length", c_int32, [c_void_p, c_int32, c_int32, c_void_p, c_void_p]),
    ("chm_schedule_rows", c_int32,
     [POINTER(Pool), POINTER(BalancerCfg), POINTER(MonitorState), POINTER(Rows),
      POINTER(RowScratch), c_void_p, c_void_p, POINTER(Decisions), c_void_p]),
    ("chm_queue_complete", c_int32,
     [POINTER(Pool), POINTER(AgingCfg), POINTER(MonitorState), POINTER(QueueState),
      c_void_p, c_void_p, c_void_p]),
    ("chm_queue_tick", c_int32,
     [POINTER(Pool), POINTER(AgingCfg), POINTER(MonitorState), POINTER(QueueState),
      POINTER(Rows), POINTER(Decisions), c_int32, c_void_p, c_void_p]),
    ("chm_queue_candidates", c_int32,
     [POINTER(Pool), POINTER(MonitorState), POINTER(QueueState), c_int32, c_void_p, c_void_p]),
    ("chm_queue_admit_merged", c_int32,
     [POINTER(Pool), POINTER(AgingCfg), POINTER(MonitorState), POINTER(QueueState), c_void_p,
      c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
    ("chm_engine_advance", c_int32,
     [POINTER(Pool), POINTER(AgingCfg), POINTER(MonitorState), POINTER(QueueState), c_void_p,
      c_void_p, c_void_p]),
    ("chm_encoder_forward", c_int32,
     [POINTER(EncoderCfg), POINTER(EncoderWeights), POINTER(EncoderWorkspace), c_void_p,
      c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p]),
    ("chm_gemm_bf16", c_int32,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_int32, c_int32,
      c_void_p]),
    ("chm_gemm_bf16_ln", c_int32,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_float, c_int32,
      c_int32, c_int32, c_void_p]),
    ("chm_gemm_bf16_deferred_ln", c_int32,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
      c_int32, c_void_p, c_void_p, c_float, c_int32, c_int32, c_int32, c_void_p]),
    ("chm_encoder_folded_bytes", ctypes.c_uint64, [POINTER(EncoderCfg)]),
    ("chm_encoder_stats_bytes", ctypes.c_uint64, [POINTER(EncoderCfg), ctypes.c_int64]),
    ("chm_encoder_fold_weights", c_int32,
     [POINTER(EncoderCfg), POINTER(EncoderWeights), POINTER(EncoderWorkspace), c_void_p]),
    ("chm_queue_scratch_bytes", ctypes.c_uint64, [c_int32]),
    ("chm_queue_fast_calls", ctypes.c_uint64, []),
    ("chm_trace_derive", c_int32, [POINTER(Trace), c_void_p, c_void_p]),
    ("chm_kendall_tau_scratch_bytes", ctypes.c_uint64, [ctypes.c_int64]),
    ("chm_quantile_train_scratch_bytes", ctypes.c_uint64,
     [ctypes.c_int64, c_int32, c_int32, c_int32]),
    ("chm_quantile_train", c_int32,
     [POINTER(Trace), c_void_p, c_int32, c_int32, ctypes.c_double, ctypes.c_int64, c_void_p,
      ctypes.c_uint64, c_void_p, c_void_p]),
    ("chm_kendall_tau_distance", c_int32,
     [c_void_p, c_void_p, ctypes.c_int64, c_void_p, ctypes.c_uint64, c_void_p, c_void_p,
      c_void_p]),
    ("chm_monitor_note_progress", c_int32,
     [POINTER(Pool), POINTER(MonitorState), c_void_p, c_void_p, c_void_p, c_int32, c_void_p,
      c_void_p]),
    ("chm_trace_gather_rows", c_int32,
     [POINTER(Trace), c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
      c_void_p, c_void_p]),
    ("chm_trace_next_stage", c_int32,
     [POINTER(Trace), c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_void_p,
      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("chm_trace_first_stage", c_int32,
     [POINTER(Trace), c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
      c_void_p]),
    ("chm_monitor_complete", c_int32,
     [POINTER(Pool), POINTER(MonitorState), c_void_p, c_void_p, c_int32, c_void_p, c_void_p,
      c_void_p]),
    ("chm_attention_bf16", c_int32,
     [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p]),
    ("chm_qkv_attention_bf16", c_int32,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_void_p]),
    ("chm_ffn_fused_bf16", c_int32,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, ctypes.c_float,
      c_int32, c_int32, c_int32, c_void_p]),
    ("chm_comm_available", c_int32, []),
    ("chm_comm_unique_id", c_int32, [c_void_p]),
    ("chm_comm_init", c_int32, [c_void_p, c_int32, c_int32, c_int32, c_void_p]),
    ("chm_comm_destroy", c_int32, [c_void_p]),
    ("chm_comm_allgather", c_int32, [c_void_p, c_void_p, c_void_p, ctypes.c_uint64, c_void_p]),
    ("chm_comm_allreduce_i64", c_int32, [c_void_p, c_void_p, c_int32, c_void_p]),
    ("chm_inflight_record_bytes", ctypes.c_uint64, [c_int32, c_int32]),
    ("chm_inflight_pack", c_int32,
     [POINTER(Pool), POINTER(Decisions), c_int32, c_void_p, c_void_p]),
    ("chm_inflight_fold", c_int32,
     [POINTER(Pool), POINTER(MonitorState), c_void_p, c_void_p, c_void_p, c_int32, c_int32,
      c_void_p, c_void_p]),
    ("chm_allreduce_inflight", c_int32,
     [c_void_p, POINTER(Pool), POINTER(MonitorState), c_void_p, c_void_p, POINTER(Decisions),
      c_int32, c_void_p, c_void_p, c_void_p]),
    ("chm_inflight_relay_recv", c_int32, [c_void_p, c_void_p, c_int32, c_void_p]),
    ("chm_inflight_relay_send", c_int32, [c_void_p, c_void_p, c_int32, c_void_p]),
    ("chm_inflight_local_sum", c_int32,
     [POINTER(Pool), POINTER(MonitorState), c_void_p, c_void_p]),
    ("chm_inflight_set_sum", c_int32,
     [POINTER(Pool), POINTER(MonitorState), c_void_p, c_void_p, c_void_p]),
    ("chm_inflight_pack_live", c_int32,
     [POINTER(Pool), POINTER(MonitorState), c_int32, c_void_p, c_void_p]),
    ("chm_inflight_merge_sum", c_int32,
     [POINTER(Pool), POINTER(MonitorState), c_void_p, c_void_p, c_int32, c_int32, c_void_p]),
    ("chm_profile_enable", c_int32, [c_int32]),
    ("chm_profile_read", c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
]

PROFILE_KINDS = ["gemm", "attention", "rowwise", "predict", "prepare", "select", "queue",
                 "qkv_attention", "trace", "eval"]


def profile_enable(on: bool) -> None:
    check(load().chm_profile_enable(1 if on else 0), "chm_profile_enable")


def profile_read() -> dict:
    """{kind: {"timed", "ms", "work", "launches"}} since the last read."""
    n = len(PROFILE_KINDS)
    timed = (ctypes.c_int32 * n)()
    ms = (ctypes.c_double * n)()
    work = (ctypes.c_double * n)()
    launches = (ctypes.c_int64 * n)()
    check(load().chm_profile_read(ctypes.addressof(timed), ctypes.addressof(ms),
                                  ctypes.addressof(work), ctypes.addressof(launches)),
          "chm_profile_read")
    return {k: {"timed": timed[i], "ms": ms[i], "work": work[i], "launches": launches[i]}
            for i, k in enumerate(PROFILE_KINDS)}

EXPORTED_SYMBOLS = [name for name, _, _ in _SIGNATURES]

_lib: ctypes.CDLL | None = None


def load(path: str | None = None) -> ctypes.CDLL:
    """Load the shared library (once) and attach the prototypes.

    Raises RuntimeError when the library has not been built: the product path
    has no CPU fallback.
    """
    global _lib
    if _lib is not None:
        return _lib
    # CHM_LIB: an alternative build of the same library (A/B measurement)
    path = path or os.environ.get("CHM_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_2603_22206_b200.build` "
            "(the GPU path has no CPU fallback)"
        )
    lib = ctypes.CDLL(path)
    for name, restype, argtypes in _SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    """Map a host-side chm_status to an exception."""
    if status == CHM_OK:
        return
    msg = load().chm_status_string(status).decode()
    if status == CHM_ERR_CUDA:
        raise RuntimeError(f"{what}: CUDA launch failed ({msg})")
    if status == CHM_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    if status == CHM_ERR_NCCL:
        raise RuntimeError(f"{what}: {msg}")
    raise errors.ValidationError(f"{what}: {msg} (status {status})")


def raise_device_error(err: list[int], context: str = "") -> None:
    """Raise the hetsched exception matching a device error word {code,row,model,aux}."""
    code, row, model, aux = (int(x) for x in err)
    if code == CHM_OK:
        return
    where = f"row {row}" + (f" model {model}" if model >= 0 else "")
    if context:
        where = f"{context}: {where}"
    if code == CHM_ERR_VALIDATION:
        what = "score outside [0,1]" if aux == 1 else "out_tokens must be >= 0"
        raise errors.ValidationError(f"{where}: {what}")
    if code == CHM_ERR_NEGATIVE_PREDICTION:
        raise ValueError(f"{where}: predicted_tokens must be >= 0")
    if code == CHM_ERR_NAN_PREDICTION:
        raise ValueError(f"{where}: predicted_tokens is NaN")
    if code == CHM_ERR_DUPLICATE_REQUEST:
        raise errors.DuplicateRequest(f"{where}: request already in flight")
    if code == CHM_ERR_TIME_BACKWARDS:
        raise ValueError(f"{where}: time going backwards")
    if code == CHM_ERR_UNKNOWN_STAGE:
        raise errors.UnknownStage(f"{where}: stage {aux} outside the program")
    if code == CHM_ERR_UNKNOWN_REQUEST:
        raise errors.UnknownRequest(f"{where}: request not in flight")
    if code == CHM_ERR_CAPACITY:
        raise errors.ValidationError(f"{where}: queue capacity exceeded ({aux} entries)")
    if code == CHM_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{where}: unsupported on device (aux {aux})")
    if code == CHM_ERR_INVALID_STATE:
        raise errors.ValidationError(f"{where}: invalid device state (aux {aux})")
    if code == CHM_ERR_INVALID_ARG:
        raise errors.ValidationError(f"{where}: invalid argument")
    raise RuntimeError(f"{where}: device error code {code}")
