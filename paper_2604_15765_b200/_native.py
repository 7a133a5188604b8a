"""ctypes binding of the in-tree native libraries.

``lib/libhermsim_b200.so``  -- CUDA engine (C-ABI ``include/hs_cuda.h``) + C++ host API and its C
                              facade (``include/hermsim_b200_c.h``).
``lib/libhs_harness.so``    -- host-only seeded input generators (``csrc/harness.c``).

There is no fallback: if the CUDA library is missing or no device is visible, every call that
needs the engine raises.  Build with ``__graft_entry__.build()`` (or ``make -C
paper_2604_15765_b200/csrc``).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "lib")
# HS_ENGINE_LIB: another build of the engine (diagnostics: A/B of kernel variants on one box)
ENGINE_PATH = os.environ.get("HS_ENGINE_LIB") or os.path.join(LIB_DIR, "libhermsim_b200.so")
HARNESS_PATH = os.path.join(LIB_DIR, "libhs_harness.so")

c_double_p = ctypes.POINTER(ctypes.c_double)
c_u32_p = ctypes.POINTER(ctypes.c_uint32)
c_u64_p = ctypes.POINTER(ctypes.c_uint64)
c_i32_p = ctypes.POINTER(ctypes.c_int32)
c_int_p = ctypes.POINTER(ctypes.c_int)


class HsPlan(ctypes.Structure):
    """hs_plan (include/hs_cuda.h): ApplyPlan plus launch facts."""

    _fields_ = [
        ("path", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("targets", ctypes.c_uint32 * 3),
        ("subcases", ctypes.c_uint64 * 3),
        ("grid_bits", ctypes.c_int32),
        ("launches", ctypes.c_int32),
        ("touched_bytes", ctypes.c_uint64),
    ]


class IoError(RuntimeError):
    """hermsim::IoError (storage_io.hpp:11-20): `kind` is the IoErrorKind name."""

    def __init__(self, text: str):
        super().__init__(text)
        tail = text.split(": ", 1)[-1] if ": " in text else text
        self.kind = next((k for k in ("bad_magic", "bad_version", "bad_header", "truncated", "length_mismatch",
                                      "io_failure") if k in tail), "io_failure")


class NativeError(RuntimeError):
    pass


_engine = None
_harness = None


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args


def engine() -> ctypes.CDLL:
    """Load libhermsim_b200.so (raises if it has not been built)."""
    global _engine
    if _engine is not None:
        return _engine
    if not os.path.exists(ENGINE_PATH):
        raise ImportError(f"CUDA engine not built: {ENGINE_PATH} missing (run __graft_entry__.build())")
    L = ctypes.CDLL(ENGINE_PATH)
    vp, i, u32, u64, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double
    pp = ctypes.POINTER(ctypes.c_void_p)
    plan = ctypes.POINTER(HsPlan)
    _sig(L, "hs_last_error", ctypes.c_char_p, [])
    _sig(L, "hs_version", ctypes.c_char_p, [])
    _sig(L, "hs_device_count", i, [c_int_p])
    _sig(L, "hs_launch_count", u64, [])
    _sig(L, "hs_set_plan_subcases", i, [i])
    _sig(L, "hs_state_create", i, [i, i, i, pp])
    _sig(L, "hs_state_free", i, [vp])
    _sig(L, "hs_state_info", i, [vp, c_int_p, c_int_p, c_u64_p, c_u64_p])
    for nm in ("hs_state_upload", "hs_state_download", "hs_state_upload_async", "hs_state_download_async"):
        _sig(L, nm, i, [vp, c_double_p, u64])
    for nm in ("hs_state_upload_range", "hs_state_download_range"):
        _sig(L, nm, i, [vp, c_double_p, u64, u64])
    _sig(L, "hs_state_copy", i, [vp, vp])
    _sig(L, "hs_state_zero", i, [vp])
    _sig(L, "hs_state_synchronize", i, [vp])
    _sig(L, "hs_state_set_stream", i, [vp, vp])
    _sig(L, "hs_state_stream", vp, [vp])
    _sig(L, "hs_state_device_ptr", vp, [vp])
    _sig(L, "hs_host_alloc", i, [u64, pp])
    _sig(L, "hs_host_free", i, [vp])
    _sig(L, "hs_apply_transfer", i, [vp, i, c_double_p, c_u32_p, plan])
    _sig(L, "hs_apply_unitary", i, [vp, i, c_double_p, c_u32_p, plan])
    _sig(L, "hs_apply_kraus", i, [vp, i, i, c_double_p, c_u32_p, plan])
    _sig(L, "hs_apply_hadamard", i, [vp, u32, plan])
    _sig(L, "hs_apply_diagonal_phase", i, [vp, u32, c_double_p, plan])
    _sig(L, "hs_apply_pauli", i, [vp, u32, i, plan])
    _sig(L, "hs_apply_permutation", i, [vp, i, c_u32_p, c_u32_p, plan])
    _sig(L, "hs_apply_monomial", i, [vp, i, c_u32_p, c_double_p, c_u32_p, plan])
    _sig(L, "hs_expectation", i, [vp, vp, c_double_p])
    _sig(L, "hs_trace", i, [vp, c_double_p])
    _sig(L, "hs_frobenius", i, [vp, c_double_p])
    _sig(L, "hs_state_fill_mixture", i, [vp, i, c_double_p])
    _sig(L, "hs_state_fill_pauli_sum", i, [vp, i, c_u64_p, c_u64_p, c_i32_p, c_double_p])
    _sig(L, "hs_state_distance_mixture", i, [vp, i, c_double_p, c_double_p])
    _sig(L, "hs_state_create_sharded", i, [i, i, i, i, i, pp])
    _sig(L, "hs_state_shard_info", i, [vp, c_int_p, c_int_p, c_u64_p])
    _sig(L, "hs_op_partner", i, [vp, i, c_u32_p, c_int_p])
    _sig(L, "hs_state_recv_alloc", i, [vp])
    _sig(L, "hs_state_exchange_from", i, [vp, vp])
    _sig(L, "hs_nccl_unique_id", i, [vp])
    _sig(L, "hs_state_comm_init", i, [vp, vp, i, i])
    _sig(L, "hs_state_exchange", i, [vp, i])
    _sig(L, "hs_op_group", i, [vp, i, c_u32_p, c_u32_p])
    _sig(L, "hs_apply_program", i, [vp, i, c_i32_p, c_u32_p, c_double_p, plan])
    _sig(L, "hs_apply_grid_program", i, [vp, i, c_i32_p, c_u32_p, c_double_p, plan])
    _sig(L, "hs_apply_cx_layer", i, [vp, i, c_u32_p, c_u32_p, plan])
    _sig(L, "hs_state_peer_enable", i, [vp])
    _sig(L, "hs_state_peer_buffers", i, [vp, pp, pp])
    _sig(L, "hs_state_set_peer", i, [vp, i, vp, vp])
    _sig(L, "hs_state_peer_flip", i, [vp, c_int_p])
    _sig(L, "hs_ipc_handles", i, [vp, vp])
    _sig(L, "hs_ipc_open", i, [vp, i, pp])
    _sig(L, "hs_ipc_close", i, [vp, i])
    _sig(L, "hs_peer_access", i, [i, i])
    _sig(L, "hs_state_fill_random_hermitian", i, [vp, ctypes.c_uint64])
    _sig(L, "hs_state_fill_basis_projector", i, [vp, ctypes.c_uint64])
    _sig(L, "hs_graph_begin", i, [vp])
    _sig(L, "hs_graph_end", i, [vp, pp])
    _sig(L, "hs_graph_launch", i, [vp, vp])
    _sig(L, "hs_graph_nodes", i, [vp, c_u64_p])
    _sig(L, "hs_graph_free", i, [vp])
    _sig(L, "hs_state_save", i, [vp, ctypes.c_char_p])
    for fn in ("hs_state_to_dense", "hs_state_to_packed", "hs_state_from_dense", "hs_state_from_packed"):
        _sig(L, fn, i, [vp, vp, i])
    _sig(L, "hs_state_convert", i, [vp, vp])
    _sig(L, "hs_device_alloc", i, [i, u64, pp])
    _sig(L, "hs_device_free", i, [i, vp])
    _sig(L, "hs_copy_d2h", i, [i, vp, vp, u64])
    _sig(L, "hs_state_load", i, [ctypes.c_char_p, i, pp])
    _sig(L, "hs_state_recv_reserve", i, [vp, i])
    _sig(L, "hs_state_exchange_group_from", i, [vp, vp, ctypes.c_uint32])
    _sig(L, "hs_state_exchange_group", i, [vp, ctypes.c_uint32])
    _sig(L, "hs_reduce_partial", i, [vp, vp, i, c_double_p])
    _sig(L, "hs_event_create", i, [pp])
    _sig(L, "hs_event_destroy", i, [vp])
    _sig(L, "hs_event_record", i, [vp, vp])
    _sig(L, "hs_event_elapsed_ms", i, [vp, vp, ctypes.POINTER(ctypes.c_float)])
    # C facade of the C++ host API
    _sig(L, "hb_last_error", ctypes.c_char_p, [])
    _sig(L, "hb_channel_native", i, [ctypes.c_char_p, d, pp])
    _sig(L, "hb_channel_depolarising", i, [d, pp])
    _sig(L, "hb_channel_generic", i, [ctypes.c_char_p, i, i, c_double_p, i, d, pp])
    _sig(L, "hb_channel_dual", i, [vp, pp])
    _sig(L, "hb_channel_free", i, [vp])
    _sig(L, "hb_channel_info", i, [vp, c_int_p, c_int_p, c_int_p])
    _sig(L, "hb_channel_kraus", i, [vp, c_double_p])
    _sig(L, "hb_channel_transfer", i, [vp, c_double_p])
    _sig(L, "hb_channel_phases", i, [vp, c_double_p])
    _sig(L, "hb_channel_perm", i, [vp, c_u32_p])
    _sig(L, "hb_bind", i, [vp, c_u32_p, i, c_u32_p, c_double_p, c_u32_p])
    _sig(L, "hb_validate_cptni", i, [vp, d, c_int_p, c_double_p, c_double_p])
    _sig(L, "hb_apply", i, [vp, vp, c_u32_p, i, i, i, plan])
    _engine = L
    return L


def harness() -> ctypes.CDLL:
    global _harness
    if _harness is not None:
        return _harness
    if not os.path.exists(HARNESS_PATH):
        raise ImportError(f"harness library not built: {HARNESS_PATH} missing")
    L = ctypes.CDLL(HARNESS_PATH)
    u64, i = ctypes.c_uint64, ctypes.c_int
    _sig(L, "hsg_gaussian_entry", None, [u64, u64, c_double_p])
    _sig(L, "hsg_uniform", ctypes.c_double, [u64, u64])
    _sig(L, "hsg_rank_psi", None, [i, u64, i, c_double_p])
    _sig(L, "hsg_payload_count", u64, [i, i])
    _sig(L, "hsg_rho_payload", None, [i, i, i, c_double_p, c_double_p])
    _sig(L, "hsg_rho_payload_range", None, [i, i, i, c_double_p, c_double_p, u64, u64])
    _sig(L, "hsg_haar", None, [i, u64, c_double_p])
    _sig(L, "hsg_isometry", i, [i, i, u64, c_double_p])
    _sig(L, "hsg_permutation", None, [i, u64, c_u32_p])
    _sig(L, "hsg_pauli_strings", None, [i, i, u64, c_u64_p, c_u64_p, c_i32_p, c_double_p])
    _sig(L, "hsg_pauli_payload", None, [i, i, i, c_u64_p, c_u64_p, c_i32_p, c_double_p, c_double_p])
    _harness = L
    return L


def check(rc: int, where: str = "", facade: bool = False) -> None:
    """Raise the reference's exception type for a non-zero status (hs_* or, with facade, hb_*)."""
    if rc == 0:
        return
    L = engine()
    msg = ((L.hb_last_error() if facade else L.hs_last_error()) or b"").decode()
    text = f"{where}: {msg}" if where else msg
    if rc == -1:
        raise ValueError(text)  # std::invalid_argument
    if rc == -2:
        raise IndexError(text)  # std::out_of_range
    if rc == -4:
        raise MemoryError(text)
    if rc == -5:
        raise NotImplementedError(text)
    if rc == -6:
        raise IoError(text)
    raise NativeError(text)
