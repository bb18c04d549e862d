"""ctypes binding of lib/libpencil_b200.so (C ABI: include/pencil_b200.h).

The product path is the CUDA library; there is no CPU fallback.  If the shared object is
missing, loading fails loudly with instructions to build it.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PENCIL_B200_LIB: load another build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("PENCIL_B200_LIB") or os.path.join(_HERE, "lib", "libpencil_b200.so")
SYNTH_PATH = os.path.join(_HERE, "lib", "libpencil_synth.so")

c_int, c_ll, c_float, c_double, c_void_p, c_char_p = (
    ctypes.c_int, ctypes.c_longlong, ctypes.c_float, ctypes.c_double, ctypes.c_void_p, ctypes.c_char_p)
P = c_void_p  # every array crosses the ABI as a plain pointer

# name -> (restype, argtypes); the drop-in section mirrors the emitted-C signatures exactly
SIGNATURES = {
    # §1 drop-in
    "gemv": (None, [c_int, c_int, c_float, c_float, P, P, P]),
    "gemv_t": (None, [c_int, c_int, c_int, c_int, c_int, c_float, c_float, P, P, P]),
    "dot": (c_float, [c_int, P, P]),
    "axpy": (None, [c_int, c_float, P, P]),
    "spmv_vec": (None, [c_int, c_int, c_int, P, P, P, P, P]),
    "spmv_inline": (None, [c_int, c_int, c_int, P, P, P, P, P]),
    "spmv": (None, [c_int, c_int, c_int, P, P, P, P, P]),
    "spmv_row": (None, [c_int, c_int, c_int, c_int, P, P, P, P, P]),
    "conv5x5_u8": (None, [c_int, c_int, c_int, P, P, P]),
    "conv5x5_f32": (None, [c_int, c_int, P, P, P]),
    "gemm": (None, [c_int, c_int, c_int, c_float, c_float, P, P, P]),
    # §2 status
    "pencil_cuda_last_status": (c_int, []),
    "pencil_cuda_last_error": (c_char_p, []),
    "pencil_cuda_clear_status": (None, []),
    "pencil_status_code": (c_char_p, [c_int]),
    # §3 device API
    "pencil_gemv_dev": (c_int, [P, c_int, c_int, c_float, c_float, P, P, P]),
    "pencil_gemv_t_dev": (c_int, [P, c_int, c_int, c_int, c_int, c_int, c_float, c_float, P, P, P]),
    "pencil_dot_dev": (c_int, [P, c_ll, P, P, P]),
    "pencil_axpy_dev": (c_int, [P, c_ll, c_float, P, P]),
    "pencil_axpy_dev_ptr": (c_int, [P, c_ll, P, P, P]),
    "pencil_conv5x5_u8_dev": (c_int, [P, c_int, c_int, c_int, P, P, P]),
    "pencil_conv5x5_u8_bytes_dev": (c_int, [P, c_int, c_int, c_int, P, P, P]),
    "pencil_conv5x5_u8_bytes": (c_int, [c_int, c_int, c_int, P, P, P]),
    "pencil_conv5x5_f32_dev": (c_int, [P, c_int, c_int, P, P, P]),
    "pencil_conv5x5_u8_band_dev": (c_int, [P, c_int, c_int, c_int, P, P, P, P, P]),
    "pencil_conv5x5_f32_band_dev": (c_int, [P, c_int, c_int, c_int, c_int, P, P, P, P, P]),
    "pencil_gemm_dev": (c_int, [P, c_int, c_int, c_int, c_float, c_float, P, P, P]),
    "pencil_gemm_strided_dev": (c_int, [P, c_int, c_int, c_int, c_float, c_float, P, c_ll, P, c_ll, P, c_ll]),
    "pencil_csr_plan_create": (c_int, [P, c_int, c_int, c_int, P, c_int, ctypes.POINTER(c_void_p)]),
    "pencil_csr_plan_destroy": (c_int, [P]),
    "pencil_csr_plan_info": (c_int, [P, ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
    "pencil_spmv_dev": (c_int, [P, P, P, P, P, P, P]),
    "pencil_spmv_dev_dist": (c_int, [P, P, P, P, P, P, P, ctypes.POINTER(c_void_p), c_int, P]),
    "pencil_sync_status": (c_int, [P]),
    # §4 name dispatch
    "pencil_runtime_create": (c_void_p, [c_int]),
    "pencil_runtime_destroy": (None, [P]),
    "pencil_runtime_set_array": (c_int, [P, c_char_p, c_int, P, c_ll]),
    "pencil_runtime_bind_array": (c_int, [P, c_char_p, c_int, P, c_ll]),
    "pencil_runtime_get_array": (c_int, [P, c_char_p, P, c_ll]),
    "pencil_runtime_array_info": (c_int, [P, c_char_p, ctypes.POINTER(c_int), ctypes.POINTER(c_ll),
                                          ctypes.POINTER(c_void_p)]),
    "pencil_runtime_call": (c_int, [P, c_char_p, c_int, P, P]),
    "pencil_runtime_fp_reordered": (c_int, [P]),
    "pencil_runtime_last_kernel": (c_char_p, [P]),
    "pencil_runtime_array_desc": (c_void_p, [P, c_char_p]),
    # §10 descriptors
    "pencil_affine_accesses": (c_int, [c_char_p, c_char_p, c_int, P, P, P, c_int]),
    "pencil_fixture_source": (c_char_p, [c_char_p]),
    "pencil_dist_plan": (c_ll, [c_char_p, c_char_p, c_char_p, c_ll]),
    "pencil_view_slice": (c_int, [P, c_int, c_ll, c_ll, P]),
    "pencil_gemv_t_view_dev": (c_int, [P, c_float, c_float, P, P, P]),
    "pencil_gemv_t_views": (c_int, [c_int, c_int, c_int, c_int, c_int, P]),
    "pencil_array_create": (c_void_p, [c_int, c_ll, c_int, P]),
    "pencil_array_destroy": (None, [P]),
    "pencil_array_attach": (c_int, [P, c_int, c_int, P]),
    "pencil_array_set_mirror": (c_int, [P, P]),
    "pencil_array_info": (c_int, [P, P, P, P, P]),
    "pencil_array_shard": (c_int, [P, c_int, P, P, P, P]),
    "pencil_array_owner": (c_int, [P, c_ll]),
    "pencil_array_sync": (c_int, [P, c_int, c_int, P]),
    "pencil_array_view": (c_int, [P, c_int, P]),
    # §5 mapper
    "pencil_map_nest": (c_int, [c_char_p, P, c_int, P]),
    "pencil_fixture_verdicts": (c_int, [c_char_p, P, c_int]),
    # §6 partitioners
    "pencil_shard_rows_by_nnz": (c_int, [P, c_int, c_int, P]),
    "pencil_shard_bands": (c_int, [c_int, c_int, P]),
    "pencil_shard_gemm_grid": (c_int, [c_int, c_int, c_int, ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
    # §7
    "pencil_version": (c_char_p, []),
    "pencil_last_transfer_bytes": (c_int, [ctypes.POINTER(c_ll), ctypes.POINTER(c_ll)]),
    "pencil_l2_flush": (c_int, [P]),
    "pencil_micro_gather": (c_int, [P, c_int, c_ll, P, P, P]),
    "pencil_micro_copy": (c_int, [P, c_ll, P, P]),
    "pencil_micro_gather_val": (c_int, [P, c_ll, P, P, P, P]),
    # §8 OP2 mesh loops
    "pencil_op2_load": (c_void_p, [c_char_p]),
    "pencil_op2_free": (None, [P]),
    "pencil_op2_num_loops": (c_int, [P]),
    "pencil_op2_loop_info": (c_int, [P, c_int, ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
    "pencil_op2_prepare": (c_int, [P]),
    "pencil_op2_run": (c_int, [P]),
    "pencil_op2_run_loop_async": (c_int, [P, c_int]),
    "pencil_op2_sync": (c_int, [P]),
    "pencil_op2_dat_size": (c_ll, [P, c_char_p]),
    "pencil_op2_get_dat": (c_int, [P, c_char_p, P, c_ll]),
    "pencil_op2_set_dat": (c_int, [P, c_char_p, P, c_ll]),
    "pencil_op2_cuda_source": (c_char_p, [P]),
    "pencil_op2_lowered": (c_char_p, [P]),
    "pencil_op2_stream": (c_void_p, [P]),
    # §9 PENCIL units (general mapper)
    "pencil_jit_load": (c_void_p, [c_char_p]),
    "pencil_jit_free": (None, [P]),
    "pencil_jit_set_array": (c_int, [P, c_char_p, c_int, P, c_ll]),
    "pencil_jit_array_size": (c_ll, [P, c_char_p]),
    "pencil_jit_get_array": (c_int, [P, c_char_p, P, P, P, c_ll]),
    "pencil_jit_call": (c_int, [P, c_char_p, c_int, P, P]),
    "pencil_jit_schedule": (c_int, [P, c_char_p, c_char_p, c_int]),
    "pencil_jit_cuda_source": (c_char_p, [P]),
    "pencil_optiml_lower": (c_ll, [c_char_p, c_char_p, c_ll]),
    "pencil_jit_access": (c_int, [P, c_char_p, c_char_p, c_int]),
    "pencil_jit_call_host": (c_int, [P, c_char_p, c_int, P, P, P, P, P]),
    "pencil_jit_last_traffic": (c_int, [P, ctypes.POINTER(c_ll), ctypes.POINTER(c_ll)]),
    "pencil_jit_set_rand_sequence": (c_int, [P, P, c_ll]),
    "pencil_jit_set_array_values": (c_int, [P, c_char_p, P, P, P, c_ll]),
    "pencil_jit_enable_trace": (c_int, [P, c_int]),
    "pencil_jit_trace_size": (c_ll, [P]),
    "pencil_jit_trace_get": (c_int, [P, c_ll, c_ll, P, P, P]),
    "pencil_jit_trace_clear": (c_int, [P]),
    # introspection used by the boundary tests (not in the public header)
    "pencil_fixture_signature": (c_int, [c_char_p, c_char_p, c_int]),
    "pencil_fixture_count": (c_int, []),
    "pencil_fixture_name": (c_char_p, [c_int]),
}


class pencil_arg(ctypes.Structure):
    _fields_ = [("kind", c_int), ("i", c_ll), ("f", c_double), ("array", c_char_p)]


class pencil_value(ctypes.Structure):
    _fields_ = [("kind", c_int), ("i", c_ll), ("f", c_double)]


class pencil_loop_verdict(ctypes.Structure):
    _fields_ = [("loop_id", c_int), ("depth", c_int), ("verdict", c_int), ("reduction_op", ctypes.c_char)]


class pencil_view(ctypes.Structure):
    _fields_ = [("base", c_void_p), ("offset", c_ll), ("rank", c_int), ("dtype", c_int),
                ("extent", c_ll * 2), ("stride", c_ll * 2)]


class pencil_access_form(ctypes.Structure):
    _fields_ = [("array", ctypes.c_char * 32), ("is_write", c_int), ("affine", c_int), ("nloops", c_int),
                ("loop", (ctypes.c_char * 16) * 8), ("lo", c_ll * 8), ("hi", c_ll * 8), ("stride", c_ll * 8),
                ("offset", c_ll), ("form", ctypes.c_char * 128)]


class pencil_schedule(ctypes.Structure):
    _fields_ = [("nloops", c_int), ("role", c_int * 8), ("grid_dims", c_int), ("reassociates", c_int),
                ("kernel", ctypes.c_char * 48)]


_lib = None
_synth = None


def load():
    """Load the CUDA backend library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make -C {_HERE}` (or __graft_entry__.build()); "
                "there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def load_synth():
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_PATH):
            raise RuntimeError(f"{SYNTH_PATH} is missing: run `make -C {_HERE}`")
        s = ctypes.CDLL(SYNTH_PATH)
        s.pencil_synth_f32.argtypes = [P, c_ll, ctypes.c_ulonglong, c_ll]
        s.pencil_synth_u8_i32.argtypes = [P, c_ll, ctypes.c_ulonglong, c_ll]
        s.pencil_synth_u8.argtypes = [P, c_ll, ctypes.c_ulonglong, c_ll]
        s.pencil_synth_csr_rowptr.argtypes = [c_int, c_double, c_double, c_int, ctypes.c_ulonglong, P,
                                              ctypes.POINTER(c_double)]
        s.pencil_synth_csr_rowptr.restype = c_ll
        s.pencil_synth_csr_fill.argtypes = [c_int, c_int, ctypes.c_ulonglong, P, P, P]
        _synth = s
    return _synth
