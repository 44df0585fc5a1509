"""ctypes binding of libes_b200.so (include/es_b200.h).

There is no CPU fallback: if the library is missing or cannot be loaded, every
engine call raises.  ctypes releases the GIL for the duration of each call, so
the engine can race SAT/BDD threads exactly like the reference's ES thread
(sched.py:232-257).
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libes_b200.so")

ES_OK = 0
ES_E_TOO_MANY_INPUTS = -1
ES_E_CUDA = -2
ES_E_BAD_PROGRAM = -3
ES_E_BAD_ARG = -4
ES_E_NO_DEVICE = -5
ES_E_WITNESS = -6
ES_E_AIGER, ES_E_AIGER_HEADER, ES_E_AIGER_LATCHES, ES_E_AIGER_DANGLING = -7, -8, -9, -10

ENGINE_AUTO, ENGINE_JIT, ENGINE_INTERP = 0, 1, 2
# es_run_opts.cofactor_pis (include/es_b200.h)
COFACTOR_AUTO, COFACTOR_NONE, COFACTOR_THROUGHPUT = 0, -1, -2
COFACTOR_MODES = {"auto": COFACTOR_AUTO, "none": COFACTOR_NONE, "throughput": COFACTOR_THROUGHPUT}
ENGINES = {"auto": ENGINE_AUTO, "jit": ENGINE_JIT, "interp": ENGINE_INTERP}

# every symbol include/es_b200.h declares
EXPORTS = ("es_compile", "es_run", "es_run_batch", "es_session_open", "es_session_geometry",
           "es_session_launch", "es_session_close", "es_map_stats", "es_map_pipes", "es_map_eval", "es_k2_stats", "es_k2_eval",
           "es_emit_ptx", "es_jit_check", "es_alu_peak", "es_fma_peak", "es_smem_peak", "es_batch_extract", "es_batch_size",
           "es_batch_info", "es_batch_table", "es_batch_k2_stats", "es_batch_k2_traffic", "es_xag_eval", "es_batch_xag", "es_batch_select", "es_batch_run", "es_batch_merge", "es_batch_free",
           "es_ipc_alloc", "es_ipc_open", "es_ipc_close", "es_word_write", "es_word_read",
           "es_map_stats_k", "es_map_pipes_k", "es_map_eval_k", "es_map_stats_kc", "es_map_eval_kc", "es_emit_ptx_k", "es_emit_body_k", "es_sass_cubin", "es_k4_cubin", "es_jit_check_k", "es_jit_check_split",
           "es_k2_eval_k", "es_k2_cofactor_pis", "es_batch_prepare",
           "es_sim", "es_sim_ones", "es_sim_device", "es_sim_prog_free", "es_sim_classes", "es_sim_levels",
           "es_aiger_parse", "es_detect_xors", "es_xag_size", "es_xag_read", "es_xag_free",
           "es_aiger_write",
           "es_peer_arm", "es_peer_arrive_wait", "es_device_count", "es_last_error", "es_version", "es_shutdown")

_P = ctypes.c_void_p


class EsProg(ctypes.Structure):
    _fields_ = [("num_instrs", ctypes.c_int32), ("num_registers", ctypes.c_int32),
                ("num_pis", ctypes.c_int32), ("op", _P), ("dst", _P), ("src0", _P),
                ("neg0", _P), ("src1", _P), ("neg1", _P), ("pi", _P)]


class EsRunOpts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("engine", ctypes.c_int32),
                ("budget_s", ctypes.c_double), ("cancel_flag", _P),
                ("slice_ms", ctypes.c_double), ("block_threads", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("cofactor_pis", ctypes.c_int32),
                ("n_devices", ctypes.c_int32), ("devices", _P), ("jit_parts", ctypes.c_int32)]


class EsResult(ctypes.Structure):
    _fields_ = [("verdict", ctypes.c_int32), ("reason", ctypes.c_int32),
                ("engine", ctypes.c_int32), ("num_luts", ctypes.c_int32),
                ("witness_index", ctypes.c_uint64), ("patterns_evaluated", ctypes.c_uint64),
                ("patterns_swept", ctypes.c_uint64), ("compile_ms", ctypes.c_double),
                ("jit_ms", ctypes.c_double), ("device_ms", ctypes.c_double),
                ("wall_ms", ctypes.c_double), ("launches", ctypes.c_int32),
                ("regs_per_thread", ctypes.c_int32), ("cofactor_pis", ctypes.c_int32),
                ("jit_opt", ctypes.c_int32), ("witness_minimal", ctypes.c_int32),
                ("n_devices", ctypes.c_int32), ("phases", ctypes.c_int32),
                ("phase2_cofactor_pis", ctypes.c_int32), ("phase2_copies", ctypes.c_int32),
                ("jit_parts", ctypes.c_int32)]


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"es_b200 error {code}: {msg}")
        self.code = code


_lib = None
_lock = threading.Lock()


def lib():
    """Load the native engine (fails loudly; never falls back)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeError(ES_E_CUDA, f"{LIB_PATH} is missing: run "
                              "`python -m paper_2512_06627_b200.build` (or __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        L.es_compile.argtypes = [ctypes.c_int32, ctypes.c_int32, _P, _P, _P, ctypes.c_uint32,
                                 _P, _P, _P, _P, _P, _P, _P, _P]
        L.es_compile.restype = ctypes.c_int32
        L.es_run.argtypes = [ctypes.POINTER(EsProg), ctypes.POINTER(EsRunOpts),
                             ctypes.POINTER(EsResult)]
        L.es_run.restype = ctypes.c_int32
        L.es_run_batch.argtypes = [ctypes.c_int32, ctypes.POINTER(EsProg),
                                   ctypes.POINTER(EsRunOpts), ctypes.POINTER(EsResult)]
        L.es_run_batch.restype = ctypes.c_int32
        L.es_peer_arm.argtypes = [_P, _P]
        L.es_peer_arm.restype = ctypes.c_int32
        L.es_peer_arrive_wait.argtypes = [_P, _P, ctypes.c_int32, _P]
        L.es_peer_arrive_wait.restype = ctypes.c_int32
        L.es_map_stats_kc.argtypes = [ctypes.POINTER(EsProg), ctypes.c_int32, ctypes.c_int32, _P, _P]
        L.es_map_stats_kc.restype = ctypes.c_int32
        L.es_map_eval_kc.argtypes = [ctypes.POINTER(EsProg), ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_uint64, ctypes.c_uint64, _P]
        L.es_map_eval_kc.restype = ctypes.c_int32
        L.es_batch_k2_traffic.argtypes = [_P, _P, _P]
        L.es_batch_k2_traffic.restype = ctypes.c_int32
        L.es_device_count.argtypes = [ctypes.POINTER(ctypes.c_int32)]
        L.es_device_count.restype = ctypes.c_int32
        L.es_session_open.argtypes = [ctypes.POINTER(EsProg), ctypes.POINTER(EsRunOpts),
                                      ctypes.POINTER(_P)]
        L.es_session_open.restype = ctypes.c_int32
        L.es_session_geometry.argtypes = [_P, ctypes.POINTER(ctypes.c_uint64),
                                          ctypes.POINTER(ctypes.c_uint64),
                                          ctypes.POINTER(ctypes.c_int32),
                                          ctypes.POINTER(ctypes.c_int32)]
        L.es_session_geometry.restype = ctypes.c_int32
        L.es_session_launch.argtypes = [_P, _P, _P, ctypes.c_uint64, ctypes.c_uint64,
                                        ctypes.c_int32, ctypes.c_int32]
        L.es_session_launch.restype = ctypes.c_int32
        L.es_session_close.argtypes = [_P]
        L.es_session_close.restype = None
        L.es_map_stats.argtypes = [ctypes.POINTER(EsProg), ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
        L.es_map_stats.restype = ctypes.c_int32
        L.es_map_pipes.argtypes = [ctypes.POINTER(EsProg), ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(ctypes.c_int32)]
        L.es_map_pipes.restype = ctypes.c_int32
        L.es_map_eval.argtypes = [ctypes.POINTER(EsProg), ctypes.c_uint64, ctypes.c_uint64, _P]
        L.es_map_eval.restype = ctypes.c_int32
        L.es_k2_stats.argtypes = [ctypes.POINTER(EsProg), _P, _P, _P, _P]
        L.es_k2_stats.restype = ctypes.c_int32
        L.es_k2_eval.argtypes = [ctypes.POINTER(EsProg), ctypes.c_uint64, ctypes.c_uint64, _P]
        L.es_k2_eval.restype = ctypes.c_int32
        L.es_emit_ptx.argtypes = [ctypes.POINTER(EsProg), ctypes.c_int32, ctypes.c_char_p,
                                  ctypes.c_int64]
        L.es_emit_ptx.restype = ctypes.c_int64
        L.es_jit_check.argtypes = [ctypes.POINTER(EsProg), ctypes.c_int32,
                                   ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                   ctypes.c_char_p, ctypes.c_int64]
        L.es_jit_check.restype = ctypes.c_int64
        _I = ctypes.c_int32
        L.es_map_stats_k.argtypes = [ctypes.POINTER(EsProg), _I, _P, _P, _P, _P]
        L.es_map_stats_k.restype = _I
        L.es_map_pipes_k.argtypes = [ctypes.POINTER(EsProg), _I, _P, _P]
        L.es_map_pipes_k.restype = _I
        L.es_map_eval_k.argtypes = [ctypes.POINTER(EsProg), _I, ctypes.c_uint64, ctypes.c_uint64, _P]
        L.es_map_eval_k.restype = _I
        L.es_emit_ptx_k.argtypes = [ctypes.POINTER(EsProg), _I, _I, ctypes.c_char_p, ctypes.c_int64]
        L.es_emit_ptx_k.restype = ctypes.c_int64
        L.es_sass_cubin.argtypes = [ctypes.POINTER(EsProg), _I, _I, _P, ctypes.c_char_p, ctypes.c_int64]
        L.es_sass_cubin.restype = ctypes.c_int64
        L.es_k4_cubin.argtypes = [ctypes.POINTER(EsProg), _I, _P, _I, _P, ctypes.c_char_p, ctypes.c_int64]
        L.es_k4_cubin.restype = ctypes.c_int64
        L.es_emit_body_k.argtypes = [ctypes.POINTER(EsProg), _I, _I, _I, _P, ctypes.c_char_p, ctypes.c_int64]
        L.es_emit_body_k.restype = ctypes.c_int64
        L.es_jit_check_k.argtypes = [ctypes.POINTER(EsProg), _I, _I, _P, _P, ctypes.c_char_p,
                                     ctypes.c_int64]
        L.es_jit_check_k.restype = ctypes.c_int64
        L.es_jit_check_split.argtypes = [ctypes.POINTER(EsProg), _I, _I, _I, _P, _P, _P, _P, _P]
        L.es_jit_check_split.restype = ctypes.c_int64
        L.es_k2_eval_k.argtypes = [ctypes.POINTER(EsProg), _I, ctypes.c_uint64, ctypes.c_uint64, _P]
        L.es_k2_eval_k.restype = _I
        L.es_k2_cofactor_pis.argtypes = [ctypes.POINTER(EsProg)]
        L.es_k2_cofactor_pis.restype = _I
        L.es_smem_peak.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_double)]
        L.es_smem_peak.restype = ctypes.c_int32
        L.es_fma_peak.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_double)]
        L.es_fma_peak.restype = ctypes.c_int32
        L.es_alu_peak.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_double)]
        L.es_alu_peak.restype = ctypes.c_int32
        L.es_batch_extract.argtypes = [ctypes.c_int32, ctypes.c_int32, _P, _P, _P, ctypes.c_int32,
                                       _P, _P, ctypes.c_int32, _P, _P, _P, ctypes.c_int32,
                                       ctypes.POINTER(_P)]
        L.es_batch_extract.restype = ctypes.c_int32
        L.es_sim.argtypes = [_I, _I, _P, _P, _P, _P, ctypes.c_int64, _I, _P, _P]
        L.es_sim.restype = _I
        L.es_sim_ones.argtypes = [_I, _I, _P, _P, _P, _P, ctypes.c_int64, _I, _P, _P]
        L.es_sim_ones.restype = _I
        L.es_sim_device.argtypes = [_I, _I, _P, _P, _P, _P, ctypes.c_int64, _P, _P, _P]
        L.es_sim_device.restype = _I
        L.es_sim_prog_free.argtypes = [_P]
        L.es_sim_prog_free.restype = None
        L.es_sim_classes.argtypes = [_I, _I, _P, _P, _P, _P, ctypes.c_int64, _I, _P, _P, _P, _P]
        L.es_sim_classes.restype = _I
        L.es_sim_levels.argtypes = [_I, _I, _P, _P, _P]
        L.es_sim_levels.restype = _I
        L.es_aiger_parse.argtypes = [_P, ctypes.c_int64, _I, ctypes.POINTER(_P)]
        L.es_aiger_parse.restype = _I
        L.es_detect_xors.argtypes = [_I, _I, _P, _P, _P, _I, _P, ctypes.POINTER(_P)]
        L.es_detect_xors.restype = _I
        L.es_xag_size.argtypes = [_P, _P, _P, _P]
        L.es_xag_size.restype = _I
        L.es_xag_read.argtypes = [_P, _P, _P, _P, _P]
        L.es_xag_read.restype = _I
        L.es_xag_free.argtypes = [_P]
        L.es_xag_free.restype = None
        L.es_aiger_write.argtypes = [_I, _I, _P, _P, _P, _I, _P, ctypes.c_char_p, ctypes.c_int64]
        L.es_aiger_write.restype = ctypes.c_int64
        L.es_batch_prepare.argtypes = [_P, ctypes.c_int32]
        L.es_batch_prepare.restype = ctypes.c_int32
        L.es_batch_size.argtypes = [_P]
        L.es_batch_size.restype = ctypes.c_int32
        L.es_batch_info.argtypes = [_P, ctypes.c_int32, _P, _P, _P, _P, _P, _P]
        L.es_batch_info.restype = ctypes.c_int32
        L.es_xag_eval.argtypes = [_I, _I, _P, _P, _P, ctypes.c_uint32, ctypes.c_uint64]
        L.es_xag_eval.restype = _I
        L.es_batch_k2_stats.argtypes = [_P, _P, _P, _P]
        L.es_batch_k2_stats.restype = ctypes.c_int32
        L.es_batch_table.argtypes = [_P, _P, _P, _P, _P]
        L.es_batch_table.restype = ctypes.c_int32
        L.es_batch_xag.argtypes = [_P, ctypes.c_int32, _P, _P, _P, _P, _P]
        L.es_batch_xag.restype = ctypes.c_int32
        L.es_batch_select.argtypes = [_P, ctypes.c_int32, _P]
        L.es_batch_select.restype = ctypes.c_int32
        L.es_batch_run.argtypes = [_P, ctypes.POINTER(EsRunOpts), ctypes.POINTER(EsResult)]
        L.es_batch_run.restype = ctypes.c_int32
        L.es_batch_merge.argtypes = [_P, _P]
        L.es_batch_merge.restype = ctypes.c_int32
        L.es_batch_free.argtypes = [_P]
        L.es_batch_free.restype = None
        L.es_ipc_alloc.argtypes = [ctypes.c_int32, ctypes.POINTER(_P), _P]
        L.es_ipc_alloc.restype = ctypes.c_int32
        L.es_ipc_open.argtypes = [ctypes.c_int32, _P, ctypes.POINTER(_P)]
        L.es_ipc_open.restype = ctypes.c_int32
        L.es_ipc_close.argtypes = [ctypes.c_int32, _P, ctypes.c_int32]
        L.es_ipc_close.restype = ctypes.c_int32
        L.es_word_write.argtypes = [ctypes.c_int32, _P, ctypes.c_uint64]
        L.es_word_write.restype = ctypes.c_int32
        L.es_word_read.argtypes = [ctypes.c_int32, _P, ctypes.POINTER(ctypes.c_uint64)]
        L.es_word_read.restype = ctypes.c_int32
        L.es_last_error.argtypes = []
        L.es_last_error.restype = ctypes.c_char_p
        L.es_version.argtypes = []
        L.es_version.restype = ctypes.c_char_p
        L.es_shutdown.argtypes = []
        L.es_shutdown.restype = None
        _lib = L
        return L


def last_error() -> str:
    return lib().es_last_error().decode(errors="replace")


def check(rc: int) -> int:
    if rc < 0:
        raise NativeError(rc, last_error())
    return rc
