"""ctypes binding of the C ABI in include/fgt1d_b200.h (libfgt1d_b200.so).

This is the "reference-side binding a maintainer would add" for a Python host
(see INTEGRATION.md).  The library is built in-tree by __graft_entry__.build()
(paper_1909_09825_b200/csrc/Makefile -> paper_1909_09825_b200/lib/).  There is
no fallback: if the library is missing the import fails loudly.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FGT1D_LIB") or os.path.join(_HERE, "lib", "libfgt1d_b200.so")

FGT_OK = 0
FGT_ERR_DOMAIN = 1
FGT_ERR_INVALID = 2
FGT_ERR_NUMERICAL = 3
FGT_ERR_CUDA = 4
FGT_ERR_NOMEM = 5

FGT_DEVICE_PTRS = 1
FGT_ASSUME_SORTED = 2
FGT_BORROW = 4
FGT_DEVICE_AGGS = 8

FGT_SOE_FULL = 0
FGT_SOE_FOLDED = 1

# name -> (restype, argtypes); mirrors include/fgt1d_b200.h exactly.
_D = ctypes.c_double
_PD = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PU8 = ctypes.POINTER(ctypes.c_uint8)
_PI32 = ctypes.POINTER(ctypes.c_int32)
_I = ctypes.c_int
_PI = ctypes.POINTER(ctypes.c_int)
_U32 = ctypes.c_uint32
_U64 = ctypes.c_uint64
_VP = ctypes.c_void_p
_PVP = ctypes.POINTER(ctypes.c_void_p)

SIGNATURES = {
    "fgt_last_error": (ctypes.c_char_p, []),
    "fgt_device_count": (_I, []),
    "fgt_cf_soe": (_I, [_I, _I, _PD, _PD, _PD, _PD, _PU8]),
    "fgt_preset_mode_count": (_I, [_I]),
    "fgt_mode_count_for_tolerance": (_I, [_D]),
    "fgt_plan_create": (_I, [_PD, _I64, _PD, _I64, _D, _PD, _PD, _PD, _PD, _PU8, _I, _I, _U32,
                             _I, _VP, _PVP]),
    "fgt_plan_create_chunk": (_I, [_PD, _I64, _PD, _I64, _D, _I, _D, _PD, _PD, _PD, _PD, _PU8,
                                   _I, _I, _U32, _I, _VP, _PVP]),
    "fgt_plan_destroy": (None, [_VP]),
    "fgt_plan_info": (_I, [_VP, _PI64, _PI64, _PI, _PI, _PI, _PI, _PI64]),
    "fgt_plan_copy_sorted": (_I, [_VP, _PD, _PI64, _PD, _PI64]),
    "fgt_plan_copy_soe": (_I, [_VP, _PD, _PD, _PD, _PD, _PU8]),
    "fgt_apply_general": (_I, [_VP, _PD, _I64, _PD, _I, _U32, _VP]),
    "fgt_apply_same": (_I, [_VP, _PD, _I64, _PD, _I, _U32, _VP]),
    "fgt_plan_gap_table": (_I, [_VP, _PD]),
    "fgt_mode_sums": (_I, [_VP, _PD, _PD, _PD]),
    "fgt_apply_chunk_aggregate": (_I, [_VP, _PD, _PD, _U32, _VP]),
    "fgt_apply_chunk_finish": (_I, [_VP, _PD, _PD, _PD, _U32, _VP]),
    "fgt_chunk_carries": (_I, [_PD, _I, _I, _PD]),
    "fgt_gauss_transform": (_I, [_PD, _I64, _PD, _I64, _PD, _D, _PD, _PD, _PD, _PD, _PU8, _I, _I,
                                 _I, _I, _PD]),
    "fgt_chunk_carries_device": (_I, [_VP, _I, _I, _I, _VP, _VP]),
    "fgt_transform_host": (_I, [_PD, _I64, _PD, _I64, _PD, _D, _PD, _PD, _PD, _PD, _PU8, _I, _I,
                                _PD, _I, _VP]),
    "fgt_direct": (_I, [_PD, _I64, _PD, _I64, _PD, _D, _PI64, _I64, _PD]),
    "fgt_uniform_points_device": (_I, [_VP, _I64, _U64, _U64, _U64, _VP]),
    "fgt_sort_device": (_I, [_VP, _I64, _VP, _VP, _VP]),
    "fgt_gather_device": (_I, [_VP, _VP, _I64, _VP, _VP]),
    "fgt_scatter_device": (_I, [_VP, _VP, _I64, _VP, _VP]),
    "fgt_merge_runs_device": (_I, [_VP, _PI64, _I, _VP, _VP, _VP]),
    "fgt_batch_create": (_I, [_I, _PD, _PI64, _PD, _PI64, _PD, _PD, _PD, _PD, _PD, _PU8, _I, _I,
                              _U32, _I, _VP, _PVP]),
    "fgt_launch_counter": (ctypes.c_longlong, []),
    "fgt_profile_enable": (None, [_I]),
    "fgt_profile_read": (_I, [_PD, ctypes.POINTER(ctypes.c_longlong), _I]),
    "fgt_fp64_peak": (_I, [_PD, _PD]),
}


def load(path=LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = load()
    return _lib


class NumericalError(ArithmeticError):
    """fgt::numerical_error (proj/include/fgt1d/errors.hpp:12-15); the reference
    binding registers it as an ArithmeticError (pymodule.cpp:81-82)."""


class DeviceError(RuntimeError):
    """No usable CUDA device or a CUDA failure (no CPU fallback)."""


def check(rc):
    if rc == FGT_OK:
        return
    msg = lib().fgt_last_error()
    msg = msg.decode() if msg else ""
    if rc in (FGT_ERR_DOMAIN, FGT_ERR_INVALID):
        # pybind11 maps std::domain_error and std::invalid_argument to ValueError
        raise ValueError(msg)
    if rc == FGT_ERR_NUMERICAL:
        raise NumericalError(msg)
    if rc == FGT_ERR_NOMEM:
        raise MemoryError(msg)
    raise DeviceError(msg)
