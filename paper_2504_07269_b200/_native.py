"""ctypes binding of the C-ABI library `_lib/libstfem_b200.so` (include/stfem_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, every compute entry point raises `NativeUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libstfem_b200.so")

OK, ERR_ARG, ERR_DIM, ERR_SINGULAR, ERR_CUDA, ERR_NOMEM, ERR_INTERNAL, ERR_NCCL = range(8)


class NativeUnavailable(RuntimeError):
    """The CUDA extension is not built or no GPU is present (no fallback)."""


class StfemError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[stfem error {code}] {msg}")
        self.code = code


class DimensionMismatch(StfemError, ValueError):
    """SPEC.md:336, :390, :396 dimension mismatch."""


class SingularPivot(StfemError, ArithmeticError):
    """numerically singular shifted system; names the shift."""


class bv_layout(C.Structure):
    _fields_ = [("rhs_stride", C.c_int64), ("shift_stride", C.c_int64),
                ("chunk_cols", C.c_int64), ("chunk_stride", C.c_int64)]


class plan_stats(C.Structure):
    _fields_ = [("n", C.c_int32), ("num_fronts", C.c_int32), ("depth", C.c_int32),
                ("max_front", C.c_int32), ("max_pivots", C.c_int32),
                ("nnz_factor", C.c_int64), ("factor_elems", C.c_int64),
                ("update_elems", C.c_int64), ("flops_factor", C.c_double),
                ("nnz_pattern", C.c_int64)]


class plan_options(C.Structure):
    """stfem_plan_options (include/stfem_b200.h): tuning knobs of one plan."""
    _fields_ = [("small_front_n", C.c_int32), ("fused_min_p", C.c_int32), ("panel_group", C.c_int32),
                ("asm_whole_n", C.c_int32), ("level_timing", C.c_int32), ("tiles_per_cta", C.c_int32),
                ("ws_stages", C.c_int32), ("front_syrk_max_p", C.c_int32), ("bwd_dmma_min_p", C.c_int32),
                ("workspace_fraction", C.c_double), ("pivot_tol", C.c_double)]


class fd_factors(C.Structure):
    """stfem_fd_factors (include/stfem_b200.h): device pointers of the temporal factors."""
    _fields_ = [("nt", C.c_int32), ("lam", C.c_void_p), ("X", C.c_void_p), ("Y", C.c_void_p),
                ("A_fwd", C.c_void_p), ("mrows_fwd", C.c_int32), ("rows_fwd", C.c_void_p),
                ("scale_fwd", C.c_void_p), ("nsrc", C.c_int32), ("A_back", C.c_void_p),
                ("mix_rows", C.c_void_p), ("mix_coef", C.c_void_p), ("nmix", C.c_int32)]


_lib = None


def _declare(lib):
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "stfem_last_error": (C.c_char_p, []),
        "stfem_version": (C.c_int, []),
        "stfem_cuda_device_count": (C.c_int, []),
        "stfem_time_transform": (C.c_int, [P, C.c_int, P, I64, P, I64, I64, C.c_int, I64, I64, P]),
        "stfem_transform_pair_fwd": (C.c_int, [P, C.c_int, C.c_int, P, P, C.c_int, P, I64, P, I64, I64, C.c_int,
                                               I64, I64, P]),
        "stfem_transform_pair_fwd_map": (C.c_int, [P, C.c_int, C.c_int, P, P, C.c_int, P, I64, P, I64, I64, C.c_int,
                                                  I64, I64, P, P]),
        "stfem_pair_mix": (C.c_int, [P, P, C.c_int, P, I64, I64, C.c_int, I64, P]),
        "stfem_transform_pair_back_map": (C.c_int, [P, C.c_int, P, P, C.c_int, P, I64, P, I64, I64, C.c_int, I64, I64,
                                                   P, P]),
        "stfem_plan_set_io_permuted": (C.c_int, [P, I32]),
        "stfem_plan_device_iperm": (C.c_int, [P, C.POINTER(P)]),
        "stfem_transform_pair_back": (C.c_int, [P, C.c_int, P, P, C.c_int, P, I64, P, I64, I64, C.c_int, I64, I64,
                                                P]),
        "stfem_copy_cols": (C.c_int, [P, I64, P, I64, I64, I64, I32, P]),
        "stfem_plan_create": (C.c_int, [I32, P, P, P, I32, I32, C.POINTER(P)]),
        "stfem_plan_destroy": (C.c_int, [P]),
        "stfem_plan_stats_get": (C.c_int, [P, C.POINTER(plan_stats)]),
        "stfem_plan_perm": (C.c_int, [P, P]),
        "stfem_plan_fronts": (C.c_int, [P, P]),
        "stfem_plan_front_rows": (C.c_int, [P, P, P]),
        "stfem_probe_launch": (C.c_int, [C.c_int, C.c_int, C.c_int, P, C.POINTER(D), P]),
        "stfem_plan_set_batch": (C.c_int, [P, I32, C.POINTER(I64)]),
        "stfem_plan_last_launches": (C.c_int, [P, C.POINTER(I64)]),
        "stfem_plan_last_batches": (C.c_int, [P, C.POINTER(I32)]),
        "stfem_plan_max_rhs": (C.c_int, [P, C.POINTER(I32)]),
        "stfem_plan_record_levels": (C.c_int, [P, I32]),
        "stfem_plan_level_report": (C.c_int, [P, P, P, P]),
        "stfem_plan_kernel_report": (C.c_int, [P, I32, P, P, P]),
        "stfem_plan_set_spectral": (C.c_int, [P, I32, P, P, P, P, I64, P, I64, P, I64, P, I64]),
        "stfem_plan_spectral_stats": (C.c_int, [P, C.POINTER(I32), C.POINTER(D), C.POINTER(D),
                                                C.POINTER(I64)]),
        "stfem_factor_solve": (C.c_int, [P, P, P, P, I32, I32, P, P, bv_layout, P]),
        "stfem_plan_check": (C.c_int, [P, P]),
        "stfem_comm_unique_id": (C.c_int, [P]),
        "stfem_comm_init": (C.c_int, [P, I32, I32, C.POINTER(P)]),
        "stfem_comm_destroy": (C.c_int, [P]),
        "stfem_comm_info": (C.c_int, [P, C.POINTER(I32), C.POINTER(I32), C.POINTER(I32)]),
        "stfem_comm_all_to_all": (C.c_int, [P, P, P, I64, P]),
        "stfem_fdm_solve": (C.c_int, [P, P, P, P, C.POINTER(fd_factors), P, P, P, I32, P]),
        "stfem_plan_set_shift_base": (C.c_int, [P, I32]),
        "stfem_plan_reserve": (C.c_int, [P, I32, I32]),
        "stfem_plan_get_options": (C.c_int, [P, C.POINTER(plan_options)]),
        "stfem_plan_set_options": (C.c_int, [P, C.POINTER(plan_options)]),
        "stfem_asm_create": (C.c_int, [I32, I32, P, I32, P, P, C.POINTER(P)]),
        "stfem_asm_destroy": (C.c_int, [P]),
        "stfem_mesh_refine2d": (C.c_int, [I32, P, I32, P, P, P, P, P, P, C.POINTER(I32), C.POINTER(I32), P]),
        "stfem_asm_pattern": (C.c_int, [P, C.POINTER(I32), C.POINTER(I64), P, P]),
        "stfem_asm_spatial": (C.c_int, [P, P, P, P]),
        "stfem_asm_rhs": (C.c_int, [P, I32, P, I32, P, I64, P]),
        "stfem_csr_spmv_c": (C.c_int, [P, P, P, I64, P, I64, I32, D, D, D, P]),
        "stfem_apply_global": (C.c_int, [P, P, P, P, P, I32, P, P, P, P]),
        "stfem_bs_update": (C.c_int, [P, P, P, I64, I32, P, I32, P, I64, I64, P]),
        "stfem_spacetime_errors": (C.c_int, [P, I32, P, I32, P, I64, P, P, P]),
    }
    for name, (res, args) in sig.items():
        if not hasattr(lib, name):
            continue
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args


def lib():
    """The loaded library (loads on first use; raises NativeUnavailable)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is not built: run `python -m paper_2504_07269_b200.build` "
                "(there is no CPU fallback)")
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def exported_symbols():
    """Dynamic symbols of the .so that start with stfem_ (via nm -D)."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True).stdout
    return sorted({ln.split()[-1] for ln in out.splitlines() if ln.split() and ln.split()[-1].startswith("stfem_")})


def require_cuda(t: torch.Tensor | None = None):
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the stfem_b200 path runs only on the GPU")
    if t is not None and not t.is_cuda:
        raise NativeUnavailable("tensor is not on a CUDA device (no CPU fallback)")


def check(rc: int):
    if rc == OK:
        return
    msg = lib().stfem_last_error().decode(errors="replace")
    if rc == ERR_DIM:
        raise DimensionMismatch(rc, msg)
    if rc == ERR_SINGULAR:
        raise SingularPivot(rc, msg)
    raise StfemError(rc, msg)


def ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)
