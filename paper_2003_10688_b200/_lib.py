"""ctypes binding of the C ABI in include/solb200.h (libsolb200.so, built in-tree).

The product path fails loudly when the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsolb200.so")

SOL_OK = 0
SOL_E_USE_AFTER_FREE = 1
SOL_E_UNKNOWN_REF = 2
SOL_E_OUT_OF_BOUNDS = 3
SOL_E_INVALID_ARGUMENT = 10
SOL_E_SHAPE_MISMATCH = 11
SOL_E_UNSUPPORTED = 12
SOL_E_OVERFLOW = 13
SOL_E_OUT_OF_REFS = 14
SOL_E_NCCL = 50
SOL_E_CUDA = 100

MODOPT_UPDATE_BN_RUNNING_STATS = 1
MODOPT_TILE_N = 2

DT_F32 = 0
DT_BF16 = 1
MAX_OP_IN = 40

# Exported symbols (must match include/solb200.h; checked by tests/test_abi.py).
SYMBOLS = [
    "sol_b200_last_error", "sol_b200_device_count", "sol_b200_set_device",
    "sol_b200_module_create", "sol_b200_module_destroy", "sol_b200_module_info", "sol_b200_module_run",
    "sol_b200_queue_create", "sol_b200_queue_destroy", "sol_b200_malloc_async", "sol_b200_free_async",
    "sol_b200_vptr_add", "sol_b200_memcpy_h2d", "sol_b200_memcpy_d2h", "sol_b200_launch",
    "sol_b200_barrier", "sol_b200_synchronize", "sol_b200_stats", "sol_b200_queue_stream",
    "sol_b200_plan_create", "sol_b200_plan_destroy", "sol_b200_plan_add_buffer", "sol_b200_plan_add_step",
    "sol_b200_plan_add_allreduce", "sol_b200_plan_finalize", "sol_b200_plan_buffer_ptr",
    "sol_b200_plan_set_frozen", "sol_b200_plan_run", "sol_b200_plan_stream", "sol_b200_plan_sync",
    "sol_b200_plan_profile", "sol_b200_plan_num_steps", "sol_b200_plan_step_info",
    "sol_b200_plan_arena_bytes", "sol_b200_nccl_unique_id", "sol_b200_plan_set_comm",
    "sol_b200_conv_packed_elems", "sol_b200_conv_pack_weight", "sol_b200_conv_fprop", "sol_b200_conv_dgrad",
    "sol_b200_conv_wgrad_workspace", "sol_b200_conv_wgrad",
    "sol_b200_plan_h2d", "sol_b200_plan_d2h", "sol_b200_plan_event_record", "sol_b200_plan_event_elapsed",
    "sol_b200_host_alloc", "sol_b200_host_free", "sol_b200_set_conv_debug", "sol_b200_plan_stage_h2d",
    "sol_b200_module_set_sibling_outputs", "sol_b200_plan_comm_info",
    "sol_b200_plan_copy_fence", "sol_b200_plan_copy_wait", "sol_b200_module_set_option",
    "sol_b200_plan_set_lr", "sol_b200_plan_time_step", "sol_b200_plan_step_set_option",
    "sol_b200_plan_link_bn_stats",
]


class Attrs(C.Structure):
    _fields_ = [("out_channels", C.c_int64), ("out_features", C.c_int64),
                ("kh", C.c_int64), ("kw", C.c_int64), ("sh", C.c_int64), ("sw", C.c_int64),
                ("ph", C.c_int64), ("pw", C.c_int64), ("groups", C.c_int64),
                ("has_bias", C.c_int32), ("min_init", C.c_float), ("count_padding", C.c_int32),
                ("eps", C.c_float), ("momentum", C.c_float), ("training", C.c_int32),
                ("lr", C.c_float), ("offset", C.c_int64)]


class UnitOp(C.Structure):
    _fields_ = [("op", C.c_int32), ("n_inputs", C.c_int32), ("inputs", C.c_int32 * MAX_OP_IN),
                ("n_params", C.c_int32), ("params", C.c_int32 * 4), ("attrs", Attrs),
                ("saved_dims", C.c_int64 * 4), ("saved_rank", C.c_int32),
                ("out_dims", C.c_int64 * 4), ("out_rank", C.c_int32)]


class Binding(C.Structure):
    _fields_ = [("is_param", C.c_int32), ("dtype", C.c_int32), ("rank", C.c_int32),
                ("dims", C.c_int64 * 4), ("ld", C.c_int64)]


class UnitDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_ops", C.c_int32), ("ops", C.POINTER(UnitOp)),
                ("n_bindings", C.c_int32), ("bindings", C.POINTER(Binding)), ("output", Binding),
                ("dtype", C.c_int32)]


class ModuleInfo(C.Structure):
    _fields_ = [("family", C.c_char * 32), ("n_args", C.c_int32), ("scratch_bytes", C.c_uint64),
                ("launches", C.c_int64), ("algo_bytes", C.c_double), ("algo_flops", C.c_double),
                ("launches_frozen", C.c_int64)]


class TransferStats(C.Structure):
    _fields_ = [("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("h2d_ops", C.c_uint64),
                ("d2h_ops", C.c_uint64), ("packed_transfers", C.c_uint64), ("launches", C.c_uint64),
                ("device_time_us", C.c_double), ("pinned_slabs", C.c_uint64), ("device_slabs", C.c_uint64)]


class ConvDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("N", "Cin", "H", "W", "Cout", "OH", "OW", "kh", "kw", "sh", "sw",
                                         "ph", "pw", "cin_ld", "dtype", "cout_ld")]


class SolError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"solb200 error {code}: {msg}")
        self.code = code


class UnsupportedError(SolError):
    pass


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 backend has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.sol_b200_last_error.restype = C.c_char_p
        vp, i32, u64, i64 = C.c_void_p, C.c_int32, C.c_uint64, C.c_int64
        sig = {
            "sol_b200_device_count": [C.POINTER(C.c_int)],
            "sol_b200_set_device": [C.c_int],
            "sol_b200_module_create": [C.POINTER(UnitDesc), C.POINTER(vp)],
            "sol_b200_module_destroy": [vp],
            "sol_b200_module_info": [vp, C.POINTER(ModuleInfo)],
            "sol_b200_module_run": [vp, C.POINTER(vp), i32, vp, vp, i32],
            "sol_b200_queue_create": [C.c_int, u64, i32, C.POINTER(vp)],
            "sol_b200_queue_destroy": [vp],
            "sol_b200_malloc_async": [vp, u64, C.POINTER(u64)],
            "sol_b200_free_async": [vp, u64],
            "sol_b200_vptr_add": [u64, u64, C.POINTER(u64)],
            "sol_b200_memcpy_h2d": [vp, u64, vp, u64],
            "sol_b200_memcpy_d2h": [vp, vp, u64, u64],
            "sol_b200_launch": [vp, vp, C.POINTER(u64), i32],
            "sol_b200_barrier": [vp],
            "sol_b200_synchronize": [vp, C.c_char_p, C.c_size_t],
            "sol_b200_stats": [vp, C.POINTER(TransferStats)],
            "sol_b200_queue_stream": [vp, C.POINTER(vp)],
            "sol_b200_plan_create": [C.c_int, C.POINTER(vp)],
            "sol_b200_plan_destroy": [vp],
            "sol_b200_plan_add_buffer": [vp, u64, i32, C.POINTER(i32)],
            "sol_b200_plan_add_step": [vp, vp, C.POINTER(i32), i32],
            "sol_b200_plan_add_allreduce": [vp, i32, u64, i32, C.c_float],
            "sol_b200_plan_finalize": [vp],
            "sol_b200_plan_buffer_ptr": [vp, i32, C.POINTER(vp)],
            "sol_b200_plan_set_frozen": [vp, i32],
            "sol_b200_plan_run": [vp, i32],
            "sol_b200_plan_stream": [vp, C.POINTER(vp)],
            "sol_b200_plan_sync": [vp],
            "sol_b200_plan_profile": [vp, C.POINTER(C.c_double), i32],
            "sol_b200_plan_num_steps": [vp, C.POINTER(i32)],
            "sol_b200_plan_step_info": [vp, i32, C.POINTER(ModuleInfo)],
            "sol_b200_plan_arena_bytes": [vp, C.POINTER(u64)],
            "sol_b200_nccl_unique_id": [C.POINTER(C.c_uint8)],
            "sol_b200_plan_set_comm": [vp, C.POINTER(C.c_uint8), i32, i32],
            "sol_b200_plan_comm_info": [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)],
            "sol_b200_conv_packed_elems": [C.POINTER(ConvDesc), i32, C.POINTER(i64)],
            "sol_b200_conv_pack_weight": [C.POINTER(ConvDesc), vp, vp, i32, vp],
            "sol_b200_conv_fprop": [C.POINTER(ConvDesc), vp, vp, vp, vp, i32, vp],
            "sol_b200_conv_dgrad": [C.POINTER(ConvDesc), vp, vp, vp, vp],
            "sol_b200_conv_wgrad_workspace": [C.POINTER(ConvDesc), C.POINTER(u64)],
            "sol_b200_conv_wgrad": [C.POINTER(ConvDesc), vp, vp, vp, vp, vp],
            "sol_b200_plan_h2d": [vp, i32, vp, u64],
            "sol_b200_plan_stage_h2d": [vp, i32, vp, u64],
            "sol_b200_plan_copy_fence": [vp, C.POINTER(C.c_uint64)],
            "sol_b200_plan_copy_wait": [vp, u64],
            "sol_b200_module_set_sibling_outputs": [vp, i32],
            "sol_b200_module_set_option": [vp, i32, i32],
            "sol_b200_plan_link_bn_stats": [vp, i32, i32, i32],
            "sol_b200_plan_set_lr": [vp, C.c_float, C.POINTER(i32)],
            "sol_b200_plan_time_step": [vp, i32, i32, C.POINTER(C.c_double)],
            "sol_b200_plan_step_set_option": [vp, i32, i32, i32],
            "sol_b200_plan_d2h": [vp, vp, i32, u64],
            "sol_b200_plan_event_record": [vp, i32],
            "sol_b200_plan_event_elapsed": [vp, i32, i32, C.POINTER(C.c_float)],
            "sol_b200_host_alloc": [u64, C.POINTER(vp)],
            "sol_b200_host_free": [vp],
            "sol_b200_set_conv_debug": [i32],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        _lib = L
    return _lib


def check(rc: int):
    if rc != SOL_OK:
        msg = lib().sol_b200_last_error().decode(errors="replace")
        if rc == SOL_E_UNSUPPORTED:
            raise UnsupportedError(rc, msg)
        raise SolError(rc, msg)
    return rc
