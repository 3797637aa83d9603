"""ctypes binding of libdlb_b200.so (include/dlb.h).

The shared library is built in-tree by ``paper_2506_09242_b200.build`` (or
``__graft_entry__.build()``). There is no fallback: if the library is missing
or a CUDA call fails, the error is raised.
"""
from __future__ import annotations

import ctypes as C
import os

from .build import LIB

DLB_OK = 0
STATUS_NAMES = {
    1: "INVALID_ARGUMENT", 2: "CONFIG", 3: "IO", 4: "DISPATCH", 5: "EXCHANGE", 6: "INTERNAL",
}
LAYOUT_TWO_POP, LAYOUT_AA = 0, 1
ARITH_EXACT, ARITH_FAST = 0, 1


class DlbError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[{STATUS_NAMES.get(status, status)}] {message}")
        self.status = status
        self.message = message


class DispatchError(DlbError):
    """A present dynamics tag is not in the dispatch set (accelerated_lattice.hpp:16-26)."""

    @property
    def chain_name(self) -> str:
        m = self.message
        return m.split('"')[1] if '"' in m else m


class ExchangeError(DlbError):
    """Halo exchange failure (multiblock.hpp:17-20)."""


class ConfigError(DlbError):
    pass


class LatticeDesc(C.Structure):
    _fields_ = [
        ("dims", C.c_int64 * 3), ("periodic", C.c_int32 * 3), ("q", C.c_int32),
        ("precision_bits", C.c_int32), ("layout", C.c_int32), ("arith", C.c_int32),
        ("device", C.c_int32), ("z_origin", C.c_int64), ("global_nz", C.c_int64),
        ("flags", C.c_int32), ("reserved", C.c_int32),
    ]


FLAG_SKIP_NODYNAMICS = 1
FLAG_TMA = 2
FLAG_SPARSE_LISTS = 4


class BlockView(C.Structure):
    _fields_ = [
        ("precision_bits", C.c_int32), ("q", C.c_int32), ("interior", C.c_int64 * 3),
        ("f_in", C.c_void_p), ("f_out", C.c_void_p), ("tag", C.c_void_p),
        ("param_index", C.c_void_p),
    ]


class ReduceArgs(C.Structure):
    _fields_ = [
        ("quantity", C.c_int32), ("periodic", C.c_int32 * 3), ("x_begin", C.c_int64),
        ("x_end", C.c_int64), ("halo_below", C.c_void_p), ("halo_above", C.c_void_p),
    ]


class TreePart(C.Structure):
    _fields_ = [("lo", C.c_int64), ("len", C.c_int64), ("value", C.c_double)]


Q_KINETIC, Q_ENSTROPHY, Q_DU_NUM, Q_DU_DEN = 0, 1, 2, 3
Q_PRESSURE_FLUID, Q_UX_FLUID, Q_UX_ALL, Q_RHO_FLUID = 4, 5, 6, 7

_lib = None

_SIGS = {
    "dlb_version": ([], C.c_char_p),
    "dlb_last_error": ([], C.c_char_p),
    "dlb_chain_canonical": ([C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "dlb_registry_new": ([C.POINTER(C.c_void_p)], C.c_int),
    "dlb_registry_free": ([C.c_void_p], None),
    "dlb_registry_register": ([C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_int32)], C.c_int),
    "dlb_registry_tag_for": ([C.c_void_p, C.c_char_p, C.POINTER(C.c_int32)], C.c_int),
    "dlb_registry_chain_for": ([C.c_void_p, C.c_int32, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "dlb_registry_tag_of_slot": ([C.c_void_p, C.c_int32, C.POINTER(C.c_int32)], C.c_int),
    "dlb_registry_counts": ([C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)], C.c_int),
    "dlb_registry_slot_params": ([C.c_void_p, C.c_int32, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "dlb_lattice_create": ([C.POINTER(LatticeDesc), C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
    "dlb_lattice_free": ([C.c_void_p], None),
    "dlb_lattice_set_slots": ([C.c_void_p, C.c_void_p], C.c_int),
    "dlb_lattice_set_uniform_slot": ([C.c_void_p, C.c_int32], C.c_int),
    "dlb_lattice_set_dispatch": ([C.c_void_p, C.c_void_p, C.c_size_t], C.c_int),
    "dlb_lattice_fill_equilibrium": ([C.c_void_p] + [C.c_void_p] * 4, C.c_int),
    "dlb_lattice_fill_tgv": ([C.c_void_p, C.c_int64, C.c_double], C.c_int),
    "dlb_lattice_upload_populations": ([C.c_void_p, C.c_void_p], C.c_int),
    "dlb_lattice_download_populations": ([C.c_void_p, C.c_void_p], C.c_int),
    "dlb_lattice_download_raw": ([C.c_void_p, C.c_void_p], C.c_int),
    "dlb_lattice_step": ([C.c_void_p, C.c_int64], C.c_int),
    "dlb_lattice_synchronize": ([C.c_void_p], C.c_int),
    "dlb_lattice_stream": ([C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
    "dlb_lattice_steps_done": ([C.c_void_p, C.POINTER(C.c_int64)], C.c_int),
    "dlb_lattice_traffic": ([C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int32)], C.c_int),
    "dlb_lattice_gather_macroscopic": ([C.c_void_p] * 5, C.c_int),
    "dlb_lattice_checksum": ([C.c_void_p, C.c_void_p], C.c_int),
    "dlb_lattice_checksum_active": ([C.c_void_p, C.c_void_p], C.c_int),
    "dlb_lattice_set_halo_timeout": ([C.c_void_p, C.c_double], C.c_int),
    "dlb_lattices_exchange": ([C.c_void_p, C.c_size_t], C.c_int),
    "dlb_block_cache_release": ([], None),
    "dlb_block_cache_info": ([C.c_void_p, C.c_void_p], C.c_int),
    "dlb_lattice_links": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "dlb_lattice_halo_trace": ([C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p], C.c_int),
    "dlb_lattice_reduce_count": ([C.c_void_p, C.POINTER(ReduceArgs), C.POINTER(C.c_int64)], C.c_int),
    "dlb_lattice_reduce_parts": ([C.c_void_p, C.POINTER(ReduceArgs), C.c_int64, C.c_int64, C.c_void_p,
                                  C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "dlb_lattice_reduce": ([C.c_void_p, C.POINTER(ReduceArgs), C.POINTER(C.c_double), C.POINTER(C.c_int64)], C.c_int),
    "dlb_tree_combine": ([C.c_int64, C.c_void_p, C.c_size_t, C.POINTER(C.c_double)], C.c_int),
    "dlb_tree_plan": ([C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "dlb_tree_sum": ([C.c_void_p, C.c_int64, C.POINTER(C.c_double)], C.c_int),
    "dlb_lattice_snapshot_velocity": ([C.c_void_p], C.c_int),
    "dlb_lattice_request_kinetic": ([C.c_void_p, C.POINTER(C.c_int32)], C.c_int),
    "dlb_lattice_velocity_planes": ([C.c_void_p, C.c_int32, C.c_int32, C.c_void_p], C.c_int),
    "dlb_lattice_step_bytes": ([C.c_void_p, C.POINTER(C.c_int64)], C.c_int),
    "dlb_lattice_time_steps": ([C.c_void_p, C.c_int64, C.POINTER(C.c_double)], C.c_int),
    "dlb_lattice_kernel_name": ([C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "dlb_lattice_link_local": ([C.c_void_p, C.c_void_p], C.c_int),
    "dlb_lattice_exchange": ([C.c_void_p], C.c_int),
    "dlb_lattice_export_ipc": ([C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "dlb_lattice_link_ipc": ([C.c_void_p, C.c_int32, C.c_void_p, C.c_size_t], C.c_int),
    "dlb_lattices_step": ([C.c_void_p, C.c_size_t, C.c_int64], C.c_int),
    "dlb_collide_and_stream": ([C.c_void_p, C.POINTER(BlockView), C.c_void_p, C.c_size_t, C.c_int32], C.c_int),
    "dlb_refresh_envelope_periodic": ([C.POINTER(BlockView), C.c_void_p], C.c_int),
    "dlb_host_alloc": ([C.c_size_t, C.POINTER(C.c_void_p)], C.c_int),
    "dlb_host_free": ([C.c_void_p], None),
    "dlb_case_sphere_pack": ([C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_uint64,
                              C.c_void_p, C.POINTER(C.c_double)], C.c_int),
}

EXPORTED = sorted(_SIGS)


def lib():
    """Load libdlb_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(status: int):
    if status == DLB_OK:
        return
    msg = lib().dlb_last_error().decode(errors="replace")
    cls = {4: DispatchError, 5: ExchangeError, 2: ConfigError}.get(status, DlbError)
    raise cls(status, msg)


def get_string(fn, *args) -> str:
    n = C.c_size_t()
    check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    check(fn(*args, buf, n.value, C.byref(n)))
    return buf.value.decode()
