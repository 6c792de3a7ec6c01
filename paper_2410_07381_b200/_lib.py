"""ctypes binding of libtally_b200.so (include/tally_b200.h).

The library is the product: there is no Python or CPU fallback for anything
it implements.  If the shared object is missing this module raises at import
with the build command; if it is present but no sm_100 GPU is visible, every
device call fails loudly with the library's own error.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TALLY_LIB_PATH: an alternative build of the same library (tools/gemm_variants.py experiments)
LIB_PATH = os.environ.get("TALLY_LIB_PATH") or os.path.join(HERE, "_lib", "libtally_b200.so")

OK = 0
EINVAL = -22
ETRANSFORM = -95
ENODEV = -19
ECUDA = -5
ENOMEM = -12
EBUSY = -16

HIGH_CLASS = 0
BEST_EFFORT_CLASS = 1

SHAPE_ORIGINAL, SHAPE_SLICED, SHAPE_PTB = 0, 1, 2
EV_LAUNCH_ISSUED, EV_BLOCK_STARTED, EV_BLOCK_FINISHED = 0, 1, 2
EV_KERNEL_FINISHED, EV_PREEMPT_SIGNALED, EV_WORKER_PARKED = 3, 4, 5
POLICY_CODES = {"Tally": 0, "Eager": 1, "KernelPriority": 2, "TimeSliced": 3}


class TallyError(RuntimeError):
    """A CUDA / driver / device failure reported by libtally_b200."""


class TransformError(ValueError):
    """A transformation was refused (ref transforms.py:27-28)."""


class c_gpu_info(C.Structure):
    _fields_ = [("device", C.c_int), ("num_sms", C.c_int), ("max_threads_per_sm", C.c_int),
                ("max_blocks_per_sm", C.c_int), ("cc_major", C.c_int), ("cc_minor", C.c_int),
                ("smem_per_sm", C.c_longlong), ("hbm_bytes", C.c_longlong),
                ("stream_mem_ops", C.c_int), ("stream_mem_ops_probe", C.c_int),
                ("name", C.c_char * 96)]


class c_kernel_args(C.Structure):
    _fields_ = [("ptr", C.c_void_p * 8), ("i", C.c_longlong * 8), ("f", C.c_double * 4)]


class c_gemm_layout(C.Structure):
    _fields_ = [("a_rows", C.c_longlong), ("a_cols", C.c_longlong), ("a_ld", C.c_longlong),
                ("b_rows", C.c_longlong), ("b_cols", C.c_longlong), ("b_ld", C.c_longlong),
                ("ldc", C.c_longlong), ("batches", C.c_int), ("hdiv", C.c_int),
                ("a_row_off", C.c_longlong * 2), ("a_col_off", C.c_longlong * 2),
                ("b_row_off", C.c_longlong * 2), ("b_col_off", C.c_longlong * 2),
                ("c_row_off", C.c_longlong * 2), ("c_col_off", C.c_longlong * 2)]


class c_conv_geometry(C.Structure):
    _fields_ = [("n", C.c_int), ("h", C.c_int), ("w", C.c_int), ("c", C.c_int),
                ("k", C.c_int), ("stride", C.c_int), ("pad", C.c_int)]


class c_bn_stats(C.Structure):
    _fields_ = [("part", C.c_void_p), ("gamma", C.c_void_p), ("beta", C.c_void_p), ("mean", C.c_void_p),
                ("invstd", C.c_void_p), ("scale_shift", C.c_void_p), ("eps", C.c_double), ("rb", C.c_longlong)]


class c_kernel_info(C.Structure):
    _fields_ = [("grid_x", C.c_uint), ("grid_y", C.c_uint), ("grid_z", C.c_uint),
                ("total_blocks", C.c_longlong), ("threads_per_block", C.c_int),
                ("smem_bytes", C.c_longlong), ("occupancy_ptb", C.c_int),
                ("occupancy_original", C.c_int), ("alg_bytes", C.c_double),
                ("alg_flops", C.c_double), ("preempt_units", C.c_int), ("cluster", C.c_int)]


class c_launch_desc(C.Structure):
    _fields_ = [("shape", C.c_int), ("linear", C.c_int), ("linear_offset", C.c_longlong),
                ("count", C.c_longlong), ("off_x", C.c_uint), ("off_y", C.c_uint),
                ("off_z", C.c_uint), ("sub_x", C.c_uint), ("sub_y", C.c_uint),
                ("sub_z", C.c_uint), ("workers", C.c_int), ("start_count", C.c_longlong),
                ("preempt_at", C.c_longlong), ("exec_count", C.c_void_p),
                ("pausable", C.c_int), ("worker_log", C.c_void_p), ("timed", C.c_int),
                ("chain", C.c_int), ("block_log", C.c_void_p)]


class c_launch_state(C.Structure):
    _fields_ = [("done", C.c_int), ("parked", C.c_int), ("preempted", C.c_int),
                ("task_counter", C.c_longlong), ("claims", C.c_longlong),
                ("gt_first_start", C.c_longlong), ("gt_first_stop", C.c_longlong),
                ("gt_last_exit", C.c_longlong), ("host_submit_ns", C.c_longlong),
                ("host_preempt_ns", C.c_longlong), ("gt_last_busy_exit", C.c_longlong)]


class c_cost(C.Structure):
    _fields_ = [("block_duration_ns", C.c_longlong), ("launch_overhead_ns", C.c_longlong),
                ("ptb_iteration_overhead_ns", C.c_longlong), ("threads_per_block", C.c_int),
                ("total_blocks", C.c_longlong)]


class c_candidate(C.Structure):
    _fields_ = [("variant", C.c_int), ("frac_num", C.c_longlong), ("frac_den", C.c_longlong),
                ("worker_count", C.c_int)]


class c_work(C.Structure):
    _fields_ = [("kernel_id", C.c_char_p), ("cost", c_cost), ("exempt", C.c_int),
                ("device_kernel", C.c_int), ("has_config", C.c_int), ("config", c_candidate),
                ("est_ns", C.c_longlong)]


class c_submit_desc(C.Structure):
    _fields_ = [("task", C.c_int), ("task_id", C.c_char_p), ("kernel_id", C.c_char_p),
                ("priority", C.c_int), ("shape", C.c_int), ("worker_count", C.c_int),
                ("start_count", C.c_longlong), ("cost", c_cost), ("block_offset", C.c_longlong),
                ("is_slice", C.c_int), ("device_kernel", C.c_int)]


class c_handle_state(C.Structure):
    _fields_ = [("done", C.c_int), ("parked", C.c_int), ("preempted", C.c_int),
                ("is_ptb", C.c_int), ("task_counter", C.c_longlong), ("finish_time", C.c_longlong)]


NOW_FN = C.CFUNCTYPE(C.c_longlong, C.c_void_p)
SUBMIT_FN = C.CFUNCTYPE(C.c_longlong, C.c_void_p, C.POINTER(c_submit_desc))
PREEMPT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_longlong)
QUERY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_longlong, C.POINTER(c_handle_state))
CALL_AT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_longlong, C.c_longlong)
FILTER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int)
KICK_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)
RUN_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)


class c_device_vtbl(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("now", NOW_FN), ("submit", SUBMIT_FN),
                ("signal_preempt", PREEMPT_FN), ("query", QUERY_FN), ("call_at", CALL_AT_FN),
                ("set_dispatch_filter", FILTER_FN), ("kick", KICK_FN),
                ("run_to_completion", RUN_FN)]


class c_event(C.Structure):
    _fields_ = [("time_ns", C.c_longlong), ("kind", C.c_int), ("task", C.c_int),
                ("kernel_index", C.c_int), ("block", C.c_longlong)]


class c_launch_record(C.Structure):
    _fields_ = [("task", C.c_int), ("kernel_index", C.c_int), ("priority", C.c_int),
                ("shape", C.c_int), ("workers", C.c_int), ("count", C.c_longlong),
                ("start_count", C.c_longlong), ("task_counter", C.c_longlong),
                ("submit_ns", C.c_longlong), ("issue_ns", C.c_longlong),
                ("complete_ns", C.c_longlong), ("preempt_ns", C.c_longlong),
                ("gt_first_start", C.c_longlong), ("gt_first_stop", C.c_longlong),
                ("gt_last_exit", C.c_longlong), ("parked", C.c_int),
                ("gpu_start_ns", C.c_longlong), ("gpu_end_ns", C.c_longlong),
                ("handle", C.c_longlong), ("gt_last_busy_exit", C.c_longlong)]


_SIGNATURES = {
    "tally_abi_version": (C.c_int, []),
    "tally_stream_handle": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "tally_last_error": (C.c_char_p, []),
    "tally_now_ns": (C.c_longlong, []),
    "tally_init": (C.c_int, [C.c_int, C.POINTER(c_gpu_info)]),
    "tally_shutdown": (C.c_int, []),
    "tally_clock_offset": (C.c_int, [C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    "tally_set_flag_mode": (C.c_int, [C.c_int]),
    "tally_l2_persist": (C.c_int, [C.c_void_p, C.c_void_p, C.c_longlong, C.c_float, C.POINTER(C.c_longlong)]),
    "tally_graph_l2_persist": (C.c_int, [C.c_void_p, C.c_void_p, C.c_longlong, C.c_float, C.POINTER(C.c_int)]),
    "tally_l2_prefetch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_longlong]),
    "tally_probe_flag_latency": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_longlong),
                                           C.POINTER(C.c_longlong)]),
    "tally_kernel_kind_count": (C.c_int, []),
    "tally_kernel_kind_name": (C.c_char_p, [C.c_int]),
    "tally_kernel_create": (C.c_int, [C.c_char_p, C.POINTER(c_kernel_args), C.POINTER(C.c_int)]),
    "tally_kernel_info_get": (C.c_int, [C.c_int, C.POINTER(c_kernel_info)]),
    "tally_kernel_destroy": (C.c_int, [C.c_int]),
    "tally_jit_register": (C.c_int, [C.c_char_p, C.c_void_p, C.c_char_p, C.c_char_p, C.c_char_p,
                                     C.c_uint, C.c_uint, C.c_uint, C.c_int, C.c_longlong,
                                     C.POINTER(C.c_int)]),
    "tally_stream_create": (C.c_int, [C.c_int, C.POINTER(C.c_int)]),
    "tally_stream_sync": (C.c_int, [C.c_int]),
    "tally_stream_destroy": (C.c_int, [C.c_int]),
    "tally_launch": (C.c_int, [C.c_int, C.c_int, C.POINTER(c_launch_desc), C.POINTER(C.c_int)]),
    "tally_launch_query": (C.c_int, [C.c_int, C.POINTER(c_launch_state)]),
    "tally_launch_wait": (C.c_int, [C.c_int, C.POINTER(c_launch_state)]),
    "tally_launch_elapsed_ns": (C.c_int, [C.c_int, C.POINTER(C.c_longlong)]),
    "tally_preempt": (C.c_int, [C.c_int]),
    "tally_set_pause": (C.c_int, [C.c_int]),
    "tally_launch_release": (C.c_int, [C.c_int]),
    "tally_runner_create": (C.c_int, [C.c_int, C.c_longlong, C.c_longlong, C.c_longlong,
                                      C.POINTER(C.c_int)]),
    "tally_runner_add_task": (C.c_int, [C.c_int, C.c_char_p, C.c_int, C.POINTER(c_work), C.c_int,
                                        C.POINTER(C.c_longlong), C.c_int]),
    "tally_runner_run": (C.c_int, [C.c_int, C.POINTER(c_device_vtbl)]),
    "tally_runner_fire": (C.c_int, [C.c_int, C.c_longlong]),
    "tally_runner_on_event": (C.c_int, [C.c_int, C.c_int, C.c_longlong]),
    "tally_runner_filter": (C.c_int, [C.c_int, C.c_longlong]),
    "tally_runner_request_count": (C.c_int, [C.c_int, C.c_int]),
    "tally_runner_requests": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_longlong), C.c_int]),
    "tally_runner_iteration_count": (C.c_int, [C.c_int, C.c_int]),
    "tally_runner_iterations": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_longlong), C.c_int]),
    "tally_runner_destroy": (C.c_int, [C.c_int]),
    "tally_runner_set_option": (C.c_int, [C.c_int, C.c_char_p, C.c_longlong]),
    "tally_device_run_origin_ns": (C.c_longlong, [C.c_int]),
    "tally_device_event_count": (C.c_int, [C.c_int]),
    "tally_device_events": (C.c_int, [C.c_int, C.POINTER(c_event), C.c_int]),
    "tally_device_launch_count": (C.c_int, [C.c_int]),
    "tally_device_launches": (C.c_int, [C.c_int, C.POINTER(c_launch_record), C.c_int]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2410_07381_b200.build` "
            "(there is deliberately no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.tally_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> int:
    """Map a library return code to the reference's exception types."""
    if rc >= 0:
        return rc
    msg = last_error() or what
    if rc == ETRANSFORM:
        raise TransformError(msg)
    if rc == EINVAL:
        raise ValueError(msg)
    raise TallyError(f"{what}: {msg} (code {rc})" if what else f"{msg} (code {rc})")


def exported_symbols():
    return list(_SIGNATURES)
