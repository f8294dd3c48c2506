"""ctypes binding of the C ABI in include/sgtk_cuda.h (libsgtk_b200.so).

The product path: every call lands in hand-written sm_100a kernels.  There is
no CPU fallback — if the shared library is missing or no CUDA device is
visible, calls raise instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SGTK_LIB", os.path.join(HERE, "libsgtk_b200.so"))

# sgtk_status -> exception (mirrors the reference pybind mapping,
# /root/reference/proj/src/python/bindings.cpp:88-100).


class SgtkError(RuntimeError):
    """sgtk::Error (errors.hpp:10-13)."""

    code = 1


class GraphIoError(SgtkError, OSError):
    code = 2


class GraphParseError(SgtkError, ValueError):
    code = 3


class NodeIdOverflowError(SgtkError, OverflowError):
    code = 4


class DegreeError(SgtkError, ValueError):
    code = 5


class GeometryError(SgtkError, ValueError):
    code = 6


class TileIndexError(SgtkError, IndexError):
    code = 7


class RangeError(SgtkError, ValueError):
    code = 8


class ShapeError(SgtkError, ValueError):
    code = 9


class NonFiniteError(SgtkError, FloatingPointError):
    code = 10


class CudaError(SgtkError):
    code = 11


_BY_CODE = {c.code: c for c in (SgtkError, GraphIoError, GraphParseError, NodeIdOverflowError,
                                DegreeError, GeometryError, TileIndexError, RangeError,
                                ShapeError, NonFiniteError, CudaError)}

FP32, TF32 = 0, 1  # Precision (tile_exec.hpp:12-15)
PRECISIONS = {"fp32": FP32, "tf32": TF32}

_lib = None

u64 = C.c_uint64
u32 = C.c_uint32
vp = C.c_void_p

_SIGS = {
    "sgtk_graph_create": [vp, vp, vp, u64, u64, u32, u32, C.c_int, vp, C.POINTER(vp)],
    "sgtk_graph_create_rows": [vp, vp, vp, u64, u64, u64, u64, u32, u32, C.c_int, vp,
                               C.POINTER(vp)],
    "sgtk_graph_import": [vp, vp, vp, u64, u64, u32, u32, vp, vp, vp, vp, C.POINTER(vp)],
    "sgtk_graph_info": [vp, vp],
    "sgtk_graph_save_panels": [vp, C.c_char_p, vp],
    "sgtk_graph_import_panels": [vp, vp, vp, u64, u64, u32, u32, vp, vp, vp, C.c_char_p, vp,
                                 C.POINTER(vp)],
    "sgtk_graph_panels_loaded": [vp, C.POINTER(C.c_int)],
    "sgtk_graph_build_times": [vp, vp],
    "sgtk_graph_device_ptrs": [vp, vp],
    "sgtk_panel_info": [vp, vp],
    "sgtk_panel_info_for": [vp, u64, vp],
    "sgtk_debug_set": [C.c_int],
    "sgtk_panel_download": [vp, vp, vp, vp, vp, vp, vp],
    "sgtk_graph_download": [vp, vp, vp, vp, vp, vp],
    "sgtk_graph_reblock": [vp, u32, vp, C.POINTER(vp)],
    "sgtk_block_stats": [vp, vp, C.POINTER(C.c_double)],
    "sgtk_split_plan": [vp, C.c_double, vp],
    "sgtk_gather_tile": [vp, u64, u64, vp, vp],
    "sgtk_spmm": [vp, vp, u64, u64, vp, vp, C.c_int, vp, u64, vp, vp],
    "sgtk_sddmm": [vp, vp, u64, vp, u64, u64, vp, vp, C.c_int, C.c_float, vp, vp],
    "sgtk_edge_softmax": [vp, vp, vp, vp],
    "sgtk_l2_normalize_rows": [vp, u64, u64, u64, vp, u64, vp, vp, vp],
    "sgtk_gemm": [vp, u64, vp, u64, u64, u64, C.c_int, C.c_int, vp, u64, vp],
    "sgtk_gcn_forward": [vp, vp, u64, u32, vp, vp, vp, vp, C.c_int, C.c_int, vp, u64, vp, u64, vp],
    "sgtk_gcn_forward_async": [vp, vp, u64, u32, vp, vp, vp, vp, C.c_int, C.c_int, vp, u64, vp,
                               u64, vp, vp],
    "sgtk_agnn_forward": [vp, vp, u64, u64, u32, vp, vp, C.c_int, C.c_int, vp, u64, vp, u64, vp,
                          vp],
    "sgtk_gcn_normalize_values": [vp, vp, u64, vp, vp],
    "sgtk_tf32_round": [vp, vp, u64, vp],
    "sgtk_relu_inplace": [vp, u64, u64, u64, vp],
    "sgtk_csr_softmax": [vp, u64, vp, vp, vp],
    "sgtk_normalize_graph": [vp, vp, vp, u64, u64, C.c_int, C.c_int, C.c_int, C.c_int, vp,
                             C.POINTER(vp)],
    "sgtk_csr_info": [vp, vp],
    "sgtk_csr_download": [vp, vp, vp, vp],
    "sgtk_csr_device_ptrs": [vp, vp],
    "sgtk_gcn_forward_host": [vp, vp, u32, vp, vp, vp, C.c_double, C.c_int, vp, vp],
    "sgtk_agnn_forward_host": [vp, vp, u64, u32, vp, C.c_double, C.c_int, C.c_int, vp, vp, vp],
    "sgtk_spmm_host": [vp, vp, u64, C.c_double, C.c_int, vp, vp, vp],
    "sgtk_partition_windows": [vp, u64, u32, u32, vp],
    "sgtk_synth_create": [u64, C.c_double, C.c_double, C.c_double, C.c_double, u64, C.POINTER(vp)],
    "sgtk_synth_info": [vp, C.POINTER(u64), C.POINTER(u64)],
    "sgtk_synth_copy": [vp, vp, vp],
}


def lib() -> C.CDLL:
    """Load libsgtk_b200.so (fails loudly; there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C paper_2412_12218_b200/csrc -j` "
                "(or __graft_entry__.build()); the CUDA path has no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.sgtk_last_error.restype = C.c_char_p
        L.sgtk_version.restype = C.c_char_p
        L.sgtk_graph_destroy.argtypes = [vp]
        L.sgtk_graph_destroy.restype = None
        L.sgtk_synth_destroy.argtypes = [vp]
        L.sgtk_synth_destroy.restype = None
        L.sgtk_csr_destroy.argtypes = [vp]
        L.sgtk_csr_destroy.restype = None
        L.sgtk_gcn_workspace.argtypes = [vp, u32, vp]
        L.sgtk_gcn_workspace.restype = u64
        L.sgtk_agnn_workspace.argtypes = [vp, u64]
        L.sgtk_agnn_workspace.restype = u64
        L.sgtk_dense_random.argtypes = [u64, u64, u64, C.c_float, C.c_float, vp]
        L.sgtk_dense_random.restype = None
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc:
        msg = lib().sgtk_last_error().decode(errors="replace")
        raise _BY_CODE.get(rc, SgtkError)(msg)


def exported_symbols() -> list[str]:
    """Names declared in include/sgtk_cuda.h (for the CPU load/export test)."""
    return sorted(set(_SIGS) | {"sgtk_last_error", "sgtk_version", "sgtk_graph_destroy",
                                "sgtk_csr_destroy",
                                "sgtk_gcn_workspace", "sgtk_agnn_workspace", "sgtk_synth_destroy",
                                "sgtk_dense_random"})
