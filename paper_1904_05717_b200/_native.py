"""Loader for the native library (lib/libtilemul_b200.so) and its C ABI.

There is no Python fallback: if the library is missing the import fails
loudly. The signatures mirror include/tilemul_b200.h one to one.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# TILEMUL_B200_LIB: load another build of the library (A/B kernel experiments)
DEFAULT_LIB = os.path.join(PKG, "lib", "libtilemul_b200.so")
LIB_PATH = os.environ.get("TILEMUL_B200_LIB") or DEFAULT_LIB


class tm_level(C.Structure):
    _fields_ = [("capacity_elements", C.c_int64), ("granularity", C.c_int64), ("inclusive", C.c_int32),
                ("write_allocate", C.c_int32), ("write_back", C.c_int32)]


class tm_blocksize(C.Structure):
    _fields_ = [("level", C.c_int32), ("dim", C.c_char), ("value", C.c_int64)]


class tm_loop(C.Structure):
    _fields_ = [("level", C.c_int32), ("dim", C.c_char), ("blocksize", C.c_int64), ("cap", C.c_int32)]


class tm_tier(C.Structure):
    _fields_ = [("level", C.c_int32), ("resident", C.c_char), ("outer_dim", C.c_char), ("inner_dim", C.c_char)]


class tm_derive_opts(C.Structure):
    _fields_ = [("slack", C.c_double), ("m_r", C.c_int64), ("n_r", C.c_int64), ("beta_a", C.c_double),
                ("beta_b", C.c_double), ("beta_c", C.c_double)]


class tm_exec_opts(C.Structure):
    _fields_ = [("numerics", C.c_int32), ("schedule", C.c_int32), ("split_k", C.c_int32), ("ctas", C.c_int32),
                ("tile", C.c_int32), ("tile_n", C.c_int32), ("parallel_loop", C.c_int32),
                ("staging", C.c_int32)]


class tm_sim_level(C.Structure):
    _fields_ = [("level", C.c_int32), ("capacity_lines", C.c_int64), ("granularity", C.c_int64),
                ("hits", C.c_int64), ("read_misses", C.c_int64), ("write_misses", C.c_int64),
                ("fetched_lines", C.c_int64), ("passthrough_writes", C.c_int64), ("writebacks", C.c_int64),
                ("per_operand_misses", C.c_int64 * 3), ("per_operand_writebacks", C.c_int64 * 3)]


# (name, restype, argtypes) for every symbol declared in include/tilemul_b200.h
P = C.c_void_p
i32, i64, dbl, cstr = C.c_int32, C.c_int64, C.c_double, C.c_char_p
SIGNATURES = [
    ("tm_last_error", cstr, []),
    ("tm_last_rules", cstr, []),
    ("tm_version", cstr, []),
    ("tm_build_id", cstr, []),
    ("tm_kernel_id", cstr, []),
    ("tm_parse_name", C.c_int, [cstr, C.c_int, C.POINTER(tm_tier), C.c_int, C.POINTER(C.c_int)]),
    ("tm_compose", C.c_int, [C.POINTER(i32), cstr, C.c_int, C.c_int, C.c_char_p, C.c_int, C.POINTER(tm_tier), C.c_int,
                             C.POINTER(C.c_int)]),
    ("tm_validate_structure", C.c_int, [C.POINTER(tm_tier), C.c_int, C.c_int]),
    ("tm_skip_level", C.c_int, [cstr, C.c_int, C.c_char_p, C.c_int]),
    ("tm_select_outer", C.c_int, [i64, i64, i64, i64, C.c_char_p]),
    ("tm_derive", C.c_int, [cstr, C.POINTER(tm_level), C.c_int, i64, i64, i64, C.POINTER(tm_derive_opts),
                            C.POINTER(tm_blocksize), C.c_int, C.POINTER(tm_blocksize), C.c_int, C.POINTER(C.c_int)]),
    ("tm_validate", C.c_int, [cstr, C.POINTER(tm_level), C.c_int, i64, i64, i64, C.POINTER(tm_blocksize), C.c_int]),
    ("tm_gpu_hierarchy", C.c_int, [C.c_int, C.POINTER(tm_level), C.c_int, C.POINTER(C.c_int)]),
    ("tm_plan_create", C.c_int, [cstr, C.POINTER(tm_level), C.c_int, i64, i64, i64, C.POINTER(tm_blocksize), C.c_int,
                                 C.POINTER(P)]),
    ("tm_plan_create_loops", C.c_int, [cstr, C.POINTER(tm_loop), C.c_int, i64, i64, i64, i64, i64, C.POINTER(P)]),
    ("tm_plan_destroy", None, [P]),
    ("tm_plan_gpu_model", C.c_int, [P, C.POINTER(tm_exec_opts), C.c_int, i64, C.POINTER(dbl), C.POINTER(i64), C.c_int]),
    ("tm_plan_gpu_model_tc", C.c_int, [P, C.c_int, C.POINTER(tm_exec_opts), C.c_int, i64, C.POINTER(i64), C.c_int]),
    ("tm_plan_tasks", C.c_int, [P, C.POINTER(tm_exec_opts), C.c_int, C.POINTER(i32), i64, C.POINTER(i64),
                                C.POINTER(i32), C.POINTER(i32), C.c_int]),
    ("tm_ipc_export", C.c_int, [P, P, C.POINTER(i64)]),
    ("tm_ipc_open", C.c_int, [P, i64, C.POINTER(P)]),
    ("tm_ipc_close", C.c_int, [P, i64]),
    ("tm_copy_async", C.c_int, [P, P, i64, P]),
    ("tm_plan_loops", C.c_int, [P, C.POINTER(tm_loop), C.c_int, C.POINTER(C.c_int)]),
    ("tm_plan_cells", i64, [P]),
    ("tm_plan_model", C.c_int, [P, C.POINTER(i64), C.c_int]),
    ("tm_model", C.c_int, [cstr, C.c_int, C.POINTER(tm_level), C.c_int, i64, i64, i64, C.POINTER(tm_blocksize),
                           C.c_int, C.POINTER(i64), C.c_int]),
    ("tm_plan_levels", C.c_int, [P]),
    ("tm_io_lower_bound", C.c_int, [i64, i64, i64, i64, C.POINTER(i64), C.POINTER(i64)]),
    ("tm_resident_cost", C.c_int, [C.c_char, i64, i64, i64, i64, i64, C.POINTER(i64)]),
    ("tm_streaming_efficiency", dbl, [C.c_char, i64, i64]),
    ("tm_goto_efficiency", dbl, [i64, i64]),
    ("tm_roofline_bound", dbl, [dbl, dbl, dbl]),
    ("tm_execute", C.c_int, [P, P, i64, P, i64, P, i64, C.POINTER(tm_exec_opts), P]),
    ("tm_execute_host", C.c_int, [P, P, P, P, C.POINTER(tm_exec_opts)]),
    ("tm_host_pipe_steps", C.c_int, [P, C.POINTER(i64), i64, C.POINTER(i64)]),
    ("tm_execute_tc", C.c_int, [P, C.c_int, P, i64, P, i64, P, i64, C.POINTER(tm_exec_opts), P]),
    ("tm_round_inputs", C.c_int, [C.c_int, P, P, i64, P]),
    ("tm_layout_address", C.c_int, [i64, i64, C.POINTER(i32), C.POINTER(i64), C.c_int, i64, i64, C.POINTER(i64)]),
    ("tm_plan_layout", C.c_int, [P, C.c_char, C.POINTER(i32), C.POINTER(i64), C.c_int, C.POINTER(C.c_int)]),
    ("tm_pack", C.c_int, [P, C.c_char, P, P, P]),
    ("tm_unpack", C.c_int, [P, C.c_char, P, P, P]),
    ("tm_execute_packed", C.c_int, [P, P, P, P, C.POINTER(tm_exec_opts), P]),
    ("tm_plan_last_launch", C.c_int, [P, C.POINTER(i64), C.POINTER(i32), C.POINTER(i32)]),
    ("tm_plan_last_staging", C.c_int, [P, C.POINTER(i32)]),
    ("tm_fill_seeded", C.c_int, [C.c_uint64, P, i64, P, i64, P, i64]),
    ("tm_measure_fp64_peak", C.c_int, [C.c_int, C.POINTER(dbl)]),
    ("tm_measure_tc_peak", C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(dbl)]),
    ("tm_fill_uniform_device", C.c_int, [P, i64, C.c_uint64, C.c_uint64, P]),
    ("tm_fill_uniform_block", C.c_int, [P, i64, i64, i64, C.c_uint64, i64, i64, i64, P]),
    ("tm_trace_event_count", i64, [P]),
    ("tm_trace", C.c_int, [P, C.c_int, i64, P, P, P, C.POINTER(i64)]),
    ("tm_sim_create", C.c_int, [C.POINTER(tm_level), C.c_int, i64, i64, i64, C.c_int, C.c_int, C.POINTER(P)]),
    ("tm_sim_destroy", None, [P]),
    ("tm_sim_access", C.c_int, [P, P, P, P, i64]),
    ("tm_sim_replay", C.c_int, [P, P, C.c_int]),
    ("tm_sim_finish", C.c_int, [P, C.POINTER(tm_sim_level), C.c_int, C.POINTER(C.c_int), C.POINTER(i64)]),
    ("tm_sim_resident_lines", C.c_int, [P, C.c_int, C.POINTER(i64), C.c_int, C.POINTER(C.c_int)]),
]

_lib = None


def lib():
    """The loaded library. Raises ImportError when it was never built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1904_05717_b200.build` "
                              "(or __graft_entry__.build()); there is no fallback implementation")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if LIB_PATH == DEFAULT_LIB:
            from . import build as _b

            want, have = _b.source_hash(), L.tm_build_id().decode()
            if want != have:
                raise ImportError(f"{LIB_PATH} was built from other sources (build id {have}, sources {want}): "
                                  "rebuild with `python -m paper_1904_05717_b200.build`")
        _lib = L
    return _lib


def build_id() -> str:
    """The loaded library's build id (sha256[:16] of its sources)."""
    return lib().tm_build_id().decode()


def kernel_id() -> str:
    """The loaded library's kernel id (sha256[:16] of the device-work sources)."""
    return lib().tm_kernel_id().decode()


def declared_symbols():
    return [s[0] for s in SIGNATURES]
