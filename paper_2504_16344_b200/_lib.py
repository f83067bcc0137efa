"""Loader for libltb.so (the sm_100a hot path behind include/ltb.h).

There is no CPU fallback: if the library is missing or no CUDA device is
usable, every compute call raises.  ``build()`` compiles the library in-tree
with nvcc (``paper_2504_16344_b200/Makefile``).
"""
import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libltb.so")

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p

# every symbol declared in include/ltb.h, with its ctypes signature
SIGNATURES = {
    "ltb_last_error": ([], C.c_char_p),
    "ltb_version": ([], C.c_char_p),
    "ltb_kernel_launches": ([], C.c_uint64),
    "ltb_plan_create": ([_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _vp, C.POINTER(_vp)], C.c_int),
    "ltb_plan_create_generated": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                   C.c_longlong, C.c_longlong, _vp, C.POINTER(_vp)], C.c_int),
    "ltb_plan_create_premultiplied": ([_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                       C.c_double, C.c_double, _vp, C.POINTER(_vp)], C.c_int),
    "ltb_plan_create_generated_premultiplied": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                                 C.c_uint64, C.c_double, C.c_double, C.c_double,
                                                 _vp, C.POINTER(_vp)], C.c_int),
    "ltb_plan_load_btpz": ([C.c_char_p, _dp, _vp, C.POINTER(_vp)], C.c_int),
    "ltb_plan_destroy": ([_vp], C.c_int),
    "ltb_plan_dims": ([_vp] + [C.POINTER(C.c_int)] * 6, C.c_int),
    "ltb_plan_bytes": ([_vp, C.POINTER(C.c_size_t)], C.c_int),
    "ltb_kernel_hat_sqnorm": ([_vp, _dp], C.c_int),
    "ltb_plan_copy_kernel_hat": ([_vp, C.c_int, C.c_int, _dp], C.c_int),
    "ltb_scratch_create": ([_vp, _vp, C.POINTER(_vp)], C.c_int),
    "ltb_scratch_destroy": ([_vp], C.c_int),
    "ltb_scratch_sync": ([_vp], C.c_int),
    "ltb_scratch_stream": ([_vp], _vp),
    "ltb_scratch_timing": ([_vp, C.c_int], C.c_int),
    "ltb_scratch_stage_ms": ([_vp, _dp, C.POINTER(C.c_int)], C.c_int),
    "ltb_apply": ([_vp, _vp, _vp, _vp, C.c_int], C.c_int),
    "ltb_apply_adjoint": ([_vp, _vp, _vp, _vp, C.c_int], C.c_int),
    "ltb_apply_series": ([_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, _vp, C.c_int], C.c_int),
    "ltb_apply_adjoint_series": ([_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, _vp, C.c_int], C.c_int),
    "ltb_dense_apply": ([_vp, C.c_int, C.c_int, C.c_int, _vp, C.c_int, C.c_ulonglong, _vp,
                         C.c_int], C.c_int),
    "ltb_engine_create": ([_vp, _vp, _vp, C.POINTER(_vp)], C.c_int),
    "ltb_engine_destroy": ([_vp], C.c_int),
    "ltb_engine_set_factor": ([_vp, _vp, C.c_int, C.c_size_t, C.c_int], C.c_int),
    "ltb_engine_set_world": ([_vp, C.c_int, C.c_int], C.c_int),
    "ltb_engine_ipc_handle": ([_vp, _vp], C.c_int),
    "ltb_engine_connect": ([_vp, _vp], C.c_int),
    "ltb_engine_set_factor_generated": ([_vp, C.c_int, C.c_uint64], C.c_int),
    "ltb_engine_solve_k": ([_vp, _vp, _vp, C.c_int], C.c_int),
    "ltb_engine_form_k": ([_vp, _vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int], C.c_int),
    "ltb_engine_form_k_generated": ([_vp, C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                     C.c_double], C.c_int),
    "ltb_engine_factorize": ([_vp], C.c_int),
    "ltb_engine_offline_ms": ([_vp, _dp, _dp, _dp], C.c_int),
    "ltb_engine_form_q": ([_vp, _vp, _vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int], C.c_int),
    "ltb_engine_form_q_generated": ([_vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_double,
                                     C.c_double, C.c_double], C.c_int),
    "ltb_engine_export_phase3": ([_vp, _vp, C.c_size_t, _vp, _vp, C.c_size_t, C.c_int], C.c_int),
    "ltb_engine_set_residual_model": ([_vp, _vp, C.c_double, C.c_double, C.c_double, C.c_double], C.c_int),
    "ltb_engine_map_residual": ([_vp, _vp, _vp, _vp, _dp, C.c_int], C.c_int),
    "ltb_integrate_displacement": ([_vp, C.c_int, C.c_int, C.c_double, _vp, C.c_int], C.c_int),
    "ltb_write_btpz": ([C.c_char_p, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int], C.c_int),
    "ltb_write_dnsm": ([C.c_char_p, _vp, C.c_int, C.c_int, C.c_size_t, C.c_int, C.c_int], C.c_int),
    "ltb_engine_export_lower": ([_vp, _vp, C.c_size_t, C.c_int], C.c_int),
    "ltb_engine_infer_map": ([_vp, _vp, _vp, _vp, _dp, C.c_int], C.c_int),
    "ltb_engine_forecast": ([_vp, _vp, _vp, _vp, C.c_int], C.c_int),
    "ltb_engine_trsv_trace": ([_vp, C.c_int, C.POINTER(C.c_ulonglong), C.c_int], C.c_int),
    "ltb_debug_dtrsv_emulated": ([C.c_int, C.c_int, C.c_uint64, _dp, _dp, _dp, _dp], C.c_int),
    "ltb_engine_set_phase3": ([_vp, _vp, C.c_size_t, _vp, C.c_int], C.c_int),
    "ltb_engine_predict_qoi": ([_vp, _vp, _vp, C.c_double, _vp, _vp, _vp, _dp, C.c_int], C.c_int),
    "ltb_normal_quantile": ([C.c_double, _dp], C.c_int),
    "ltb_fnv1a64_file": ([C.c_char_p, C.POINTER(C.c_uint64)], C.c_int),
    "ltb_engine_load_factor_dnsm": ([_vp, C.c_char_p], C.c_int),
    "ltb_engine_load_phase3_dnsm": ([_vp, C.c_char_p, C.c_char_p], C.c_int),
    "ltb_engine_infer_and_forecast": ([_vp, _vp, _vp, _vp, _vp, _dp, C.c_int], C.c_int),
    "ltb_plan_create_sharded": ([_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), _vp,
                                 C.POINTER(_vp)], C.c_int),
    "ltb_plan_create_generated_sharded": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                           C.POINTER(C.c_int), _vp, C.POINTER(_vp)], C.c_int),
    "ltb_splan_destroy": ([_vp], C.c_int),
    "ltb_splan_dims": ([_vp] + [C.POINTER(C.c_int)] * 4, C.c_int),
    "ltb_splan_shard": ([_vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                         C.POINTER(C.c_int)], C.c_int),
    "ltb_splan_kernel_hat_sqnorm": ([_vp, _dp], C.c_int),
    "ltb_sscratch_create": ([_vp, _vp, C.POINTER(_vp)], C.c_int),
    "ltb_sscratch_destroy": ([_vp], C.c_int),
    "ltb_sscratch_sync": ([_vp], C.c_int),
    "ltb_sscratch_stream": ([_vp], _vp),
    "ltb_apply_sharded": ([_vp, _vp, _vp, _vp, C.c_int], C.c_int),
    "ltb_apply_adjoint_sharded": ([_vp, _vp, _vp, _vp, C.c_int], C.c_int),
    "ltb_reindex": ([_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, C.c_int, _vp], C.c_int),
    "ltb_nccl_unique_id": ([_vp], C.c_int),
    "ltb_plan_create_generated_premultiplied_shard": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                                       C.c_longlong, C.c_longlong, C.c_double, C.c_double,
                                                       C.c_double, _vp, C.POINTER(_vp)], C.c_int),
    "ltb_engine_set_comm": ([_vp, _vp], C.c_int),
    "ltb_engine_form_k_generated_dist": ([_vp, C.c_longlong, C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                          C.c_double, C.c_double], C.c_int),
    "ltb_engine_factorize_dist": ([_vp], C.c_int),
}

_lib = None


class LtbOpts(C.Structure):
    _fields_ = [("device", C.c_int), ("unit_cols", C.c_int)]


def build(force=False):
    """Compile libltb.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", HERE])
    else:
        subprocess.check_call(["make", "-s", "-C", HERE], stdout=subprocess.DEVNULL)


def load():
    """Load libltb.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                "libltb.so not built (%s); run __graft_entry__.build() or make -C %s" % (LIB_PATH, HERE))
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def last_error():
    return load().ltb_last_error().decode(errors="replace")


def kernel_launches():
    return int(load().ltb_kernel_launches())
