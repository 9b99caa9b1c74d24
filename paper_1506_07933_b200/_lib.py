"""ctypes binding of libdfftb.so (the C ABI in include/dfftb/dfftb.h).

The library is built in-tree (``python __graft_entry__.py`` / ``make -C
paper_1506_07933_b200/csrc``).  There is no fallback: if the CUDA extension is
missing, importing the API raises.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DFFTB_LIB_OVERRIDE") or os.path.join(HERE, "libdfftb.so")

_c = ctypes
i64p = _c.POINTER(_c.c_int64)
ip = _c.POINTER(_c.c_int)
vp = _c.c_void_p


class PlanOptionsC(_c.Structure):
    _fields_ = [("exchange", _c.c_int), ("normalize", _c.c_int),
                ("chunks_per_peer", _c.c_int), ("staging_buffers", _c.c_int),
                ("validate_finite", _c.c_int)]


class TimingC(_c.Structure):
    _fields_ = [("local_fft", _c.c_double), ("pack", _c.c_double), ("unpack", _c.c_double),
                ("staging_copy", _c.c_double), ("wire_comm", _c.c_double),
                ("total", _c.c_double)]


_SIGS = {
    "dfftb_plan_options_default": (None, [_c.POINTER(PlanOptionsC)]),
    "dfftb_plan_create": (_c.c_int, [_c.c_int, i64p, _c.c_int, _c.c_int, ip, _c.c_int, _c.c_int,
                                     _c.c_int, _c.POINTER(PlanOptionsC), _c.POINTER(vp)]),
    "dfftb_plan_destroy": (None, [vp]),
    "dfftb_plan_signature": (_c.c_int, [vp, _c.c_char_p, _c.c_size_t]),
    "dfftb_plan_fft_stage_count": (_c.c_int, [vp]),
    "dfftb_plan_transpose_stage_count": (_c.c_int, [vp]),
    "dfftb_plan_nranks": (_c.c_int, [vp]),
    "dfftb_plan_precision": (_c.c_int, [vp]),
    "dfftb_plan_kind": (_c.c_int, [vp]),
    "dfftb_plan_direction": (_c.c_int, [vp]),
    "dfftb_plan_warning_count": (_c.c_int, [vp]),
    "dfftb_plan_warning": (_c.c_char_p, [vp, _c.c_int]),
    "dfftb_block_map": (_c.c_int, [_c.c_int64, _c.c_int, i64p, i64p]),
    "dfftb_plan_layout": (_c.c_int, [vp, _c.c_int, i64p, ip, ip, ip]),
    "dfftb_plan_local_extents": (_c.c_int, [vp, _c.c_int, _c.c_int, i64p, i64p]),
    "dfftb_plan_local_count": (_c.c_int64, [vp, _c.c_int, _c.c_int]),
    "dfftb_local_index": (_c.c_int, [vp, _c.c_int, i64p, ip, i64p]),
    "dfftb_plan_exchange_counts": (_c.c_int, [vp, _c.c_int, _c.c_int, i64p, i64p, ip]),
    "dfftb_ctx_create": (_c.c_int, [vp, _c.c_int, _c.c_int, _c.POINTER(vp)]),
    "dfftb_ctx_handle_size": (_c.c_size_t, []),
    "dfftb_ctx_export_handle": (_c.c_int, [vp, vp]),
    "dfftb_ctx_connect": (_c.c_int, [vp, vp]),
    "dfftb_ctx_destroy": (None, [vp]),
    "dfftb_execute": (_c.c_int, [vp, vp, vp, vp, vp, _c.c_int, _c.POINTER(TimingC)]),
    "dfftb_ctx_check": (_c.c_int, [vp, vp]),
    "dfftb_world_create": (_c.c_int, [vp, _c.c_int, _c.POINTER(vp)]),
    "dfftb_world_create_devices": (_c.c_int, [vp, _c.c_int, ip, _c.POINTER(vp)]),
    "dfftb_ctx_last_ops": (_c.c_int, [vp, ip, ip, ip, _c.POINTER(_c.c_double), _c.POINTER(_c.c_double),
                                      _c.POINTER(_c.c_double), _c.c_int]),
    "dfftb_execute_world": (_c.c_int, [vp, _c.POINTER(vp), _c.POINTER(vp), _c.POINTER(vp), vp,
                                       _c.c_int]),
    "dfftb_fill_seeded": (_c.c_int, [vp, _c.c_int, _c.c_int, _c.c_uint64, _c.c_int, vp, vp]),
    "dfftb_error_name": (_c.c_char_p, [_c.c_int]),
    "dfftb_last_error_message": (_c.c_char_p, []),
    "dfftb_kernel_launch_count": (_c.c_uint64, []),
    "dfftb_spectral_apply": (_c.c_int, [vp, _c.c_int, _c.c_int, _c.c_int,
                                        _c.POINTER(_c.c_double), vp, vp, _c.c_int, vp]),
    "dfftb_workspace_bytes": (_c.c_int, [vp, _c.c_int, _c.POINTER(_c.c_uint64)]),
    "dfftb_execute_spectral": (_c.c_int, [vp, vp, vp, vp, _c.c_int, _c.c_int, _c.POINTER(_c.c_double),
                                          _c.c_int, vp, _c.c_int]),
    "dfftb_execute_world_spectral": (_c.c_int, [vp, _c.POINTER(vp), _c.POINTER(vp), _c.POINTER(vp), _c.c_int,
                                                _c.c_int, _c.POINTER(_c.c_double), _c.c_int, vp, _c.c_int]),
    "dfftb_wavenumbers": (_c.c_int, [vp, _c.c_int, _c.c_int, _c.c_int,
                                     _c.POINTER(_c.c_double), _c.POINTER(_c.c_double)]),
}

_LIB = None


def lib():
    """Load libdfftb.so (fails loudly when the CUDA extension is not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"dfftb CUDA extension not found at {LIB_PATH}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` or "
                "`make -C paper_1506_07933_b200/csrc`")
        L = _c.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("DFFTB_LIB_OVERRIDE") and not hasattr(L, name):
                continue  # A/B builds of older revisions may lack newer entry points
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def exported_symbols():
    return list(_SIGS)
