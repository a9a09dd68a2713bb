"""ctypes mirror of include/orloj.h and the loader for liborloj.so.

Argument marshalling only: every step of the path runs in the CUDA library.
There is no CPU fallback — if liborloj.so is missing or fails to load, every
call raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.environ.get("ORLOJ_LIB") or os.path.join(PKG, "liborloj.so")
HEADER = os.path.join(ROOT, "include", "orloj.h")

NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-shared", "-Xcompiler", "-fPIC"]

ABI_VERSION = 5  # include/orloj.h ORLOJ_ABI_VERSION: the struct layouts below

STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "COLD_START", 3: "UNSORTED", 4: "CAPACITY", 5: "CUDA", 6: "OOM"}


class OrlojError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"orloj {STATUS.get(status, status)}: {msg}")
        self.status = status


def build(nvcc: str = "nvcc", verbose: bool = False, out: str | None = None, defines=(), only=None) -> str:
    """Compile every csrc/*.cu translation unit for sm_100a in parallel and link
    liborloj.so (each TU's kernels are launched only from that TU: no
    relocatable device code).  out / defines: a variant library built with
    extra -D flags (loaded through ORLOJ_LIB) for experiments; only: rebuild
    just these TUs (the other objects are reused)."""
    from concurrent.futures import ThreadPoolExecutor
    csrc = os.path.join(PKG, "csrc")
    out = out or LIB_PATH
    objdir = os.path.join(PKG, "build", os.path.basename(out).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    srcs = sorted(f for f in os.listdir(csrc) if f.endswith(".cu"))
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"] + [f"-D{d}" for d in defines]

    def one(f):
        obj = os.path.join(objdir, f[:-3] + ".o")
        if only is not None and f not in only and os.path.exists(obj):
            return obj
        cmd = [nvcc, *compile_flags, "-c", "-o", obj, os.path.join(csrc, f)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        return obj

    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        objs = list(ex.map(one, srcs))
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    tmp = out + ".tmp"
    subprocess.check_call([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs])
    os.replace(tmp, out)
    return out


class Store(ctypes.Structure):
    _fields_ = [("num_dists", ctypes.c_int32), ("num_bins", ctypes.c_int32), ("bin_ticks", ctypes.c_int64),
                ("log2_cdf", ctypes.c_void_p)]


class LatencyProfile(ctypes.Structure):
    _fields_ = [("kmax", ctypes.c_int32), ("offset_ticks", ctypes.c_void_p), ("ticks_per_bin", ctypes.c_void_p)]


class QueuesC(ctypes.Structure):
    _fields_ = [("num_queues", ctypes.c_int64), ("queue_offsets", ctypes.c_void_p),
                ("arrival_ticks", ctypes.c_void_p), ("deadline_ticks", ctypes.c_void_p),
                ("dist_id", ctypes.c_void_p), ("now_ticks", ctypes.c_void_p)]


class TraceC(ctypes.Structure):
    _fields_ = [("num_scenarios", ctypes.c_int64), ("arrival_offsets", ctypes.c_void_p),
                ("arrival_ticks", ctypes.c_void_p), ("dist_id", ctypes.c_void_p), ("true_bin", ctypes.c_void_p),
                ("slo_ticks", ctypes.c_void_p), ("bucket", ctypes.c_void_p), ("num_buckets", ctypes.c_int32)]


class ReplayPolicyC(ctypes.Structure):
    _fields_ = [("objective", ctypes.c_int32), ("drop_threshold_ticks", ctypes.c_void_p),
                ("size_threshold_ticks", ctypes.c_void_p), ("priority_table", ctypes.c_void_p),
                ("priority_log_expected", ctypes.c_void_p), ("priority_b_per_tick", ctypes.c_double)]


class CostSteps(ctypes.Structure):
    _fields_ = [("num_steps", ctypes.c_int32), ("offset_ticks", ctypes.c_void_p), ("cost", ctypes.c_void_p)]


SCORE_MODEL_PLAN_BYTES = 512  # ORLOJ_SCORE_MODEL_PLAN_BYTES


class ScoreModelC(ctypes.Structure):
    _fields_ = [("kmax", ctypes.c_int32), ("duration_ticks", ctypes.c_void_p), ("interpolate", ctypes.c_int32),
                ("num_steps", ctypes.c_int32), ("step_offset_ticks", ctypes.c_void_p), ("step_cost", ctypes.c_void_p),
                ("plan", ctypes.c_void_p)]


class ReplayEpochC(ctypes.Structure):
    _fields_ = [("epoch", ctypes.c_int32), ("num_epochs", ctypes.c_int32), ("worker_free_ticks", ctypes.c_void_p),
                ("outcome", ctypes.c_void_p)]


class FeedbackC(ctypes.Structure):
    _fields_ = [("num_epochs", ctypes.c_int32), ("window_epochs", ctypes.c_int32), ("min_samples", ctypes.c_uint32),
                ("sample_mask", ctypes.c_void_p)]


class Counters(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("total", "finished", "dropped", "late", "batches", "busy_ticks", "span_ticks")]


# symbol -> (restype, argtypes)
_P = ctypes.c_void_p
SIGNATURES = {
    "orloj_last_error": (ctypes.c_char_p, []),
    "orloj_abi_version": (ctypes.c_int32, []),
    "orloj_store_build": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, _P, _P]),
    "orloj_score_batches": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(LatencyProfile),
                                           ctypes.POINTER(QueuesC), _P, _P, _P, _P]),
    "orloj_pick_batch": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(LatencyProfile),
                                        ctypes.POINTER(QueuesC), _P, _P, _P]),
    "orloj_pick_batch_host_workspace": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int64]),
    "orloj_pick_batch_host": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(LatencyProfile), ctypes.c_int64,
                                             _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "orloj_replay_trace": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(LatencyProfile),
                                          ctypes.POINTER(TraceC), _P, _P, _P]),
    "orloj_replay_trace_ex": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(LatencyProfile),
                                             ctypes.POINTER(TraceC), ctypes.POINTER(ReplayPolicyC), _P, _P, _P]),
    "orloj_replay_seg_workspace": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                                     ctypes.c_int32]),
    "orloj_replay_trace_seg": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(LatencyProfile),
                                              ctypes.POINTER(TraceC), ctypes.POINTER(ReplayPolicyC), ctypes.c_int32,
                                              ctypes.c_int64, _P, ctypes.c_size_t, _P, _P, _P]),
    "orloj_score_model_batches": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(QueuesC),
                                                 ctypes.POINTER(ScoreModelC), _P, _P, _P, _P]),
    "orloj_score_model_prepare": (ctypes.c_int, [ctypes.POINTER(ScoreModelC), ctypes.c_int32, _P, _P]),
    "orloj_priority_table": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(LatencyProfile), ctypes.c_int32,
                                            _P, ctypes.c_double, _P, _P, _P]),
    "orloj_priority_scores": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(LatencyProfile), ctypes.c_int32,
                                             ctypes.c_double, _P, _P, ctypes.POINTER(QueuesC), _P, _P]),
    "orloj_priority_scores_steps": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(LatencyProfile),
                                                   ctypes.c_int32, ctypes.c_double, _P, _P, ctypes.POINTER(QueuesC),
                                                   ctypes.POINTER(CostSteps), _P, _P]),
    "orloj_pop_batch": (ctypes.c_int, [ctypes.POINTER(QueuesC), _P, ctypes.c_int32, _P, _P, _P]),
    "orloj_histogram_accumulate": (ctypes.c_int, [_P, _P, ctypes.c_int64, ctypes.c_int64, _P, ctypes.c_int32,
                                                  ctypes.c_int32, _P]),
    "orloj_replay_trace_epoch": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(LatencyProfile),
                                                ctypes.POINTER(TraceC), ctypes.POINTER(ReplayPolicyC),
                                                ctypes.POINTER(ReplayEpochC), _P, _P, _P]),
    "orloj_profile_outcomes": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_int64, _P, ctypes.c_int32, ctypes.c_int32,
                                              _P]),
    "orloj_store_refresh": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, _P, _P]),
    "orloj_replay_feedback_workspace": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                                          ctypes.c_int32]),
    "orloj_replay_feedback": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(LatencyProfile),
                                             ctypes.POINTER(TraceC), ctypes.POINTER(ReplayPolicyC),
                                             ctypes.POINTER(FeedbackC), _P, ctypes.c_size_t, _P, _P, _P, _P]),
    "orloj_expected_latency_thresholds": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32,
                                                         ctypes.POINTER(LatencyProfile), _P]),
    "orloj_alg1_size_thresholds": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, _P,
                                                  ctypes.POINTER(LatencyProfile), _P]),
    "orloj_validate_store": (ctypes.c_int, [ctypes.POINTER(Store), _P]),
    "orloj_validate_queues": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(QueuesC), _P]),
    "orloj_validate_trace": (ctypes.c_int, [ctypes.POINTER(Store), ctypes.POINTER(TraceC), _P]),
}

_lib = None


def lib():
    """Load liborloj.so (fails loudly: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OrlojError(5, f"{LIB_PATH} not built: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.orloj_abi_version() != ABI_VERSION:
            raise OrlojError(1, f"{LIB_PATH} has ABI {L.orloj_abi_version()}, the binding expects {ABI_VERSION}: "
                                "rebuild with __graft_entry__.build()")
        _lib = L
    return _lib


def check(status: int):
    if status != 0:
        raise OrlojError(status, lib().orloj_last_error().decode())
