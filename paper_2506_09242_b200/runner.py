"""ctypes binding of the reference-compatible benchmark interface (include/dolb.h).

``Dolb(path)`` wraps any library exporting dolb.h -- by default this package's
``_lib/libdolb.so`` (the device runner, csrc/runner.cpp). The methods mirror the
C calls one to one and raise ``DolbError`` with the status code and
``dolb_last_error()`` text, so tests written against the reference's
tests/test_capi.cpp read the same. ``run(config)`` is the one-call form:
dict of "section.key" -> value in, (steps, MLUPS) out, artefacts in run.out.
"""
from __future__ import annotations

import ctypes as C
import os

from .build import LIBDIR

DOLB_LIB = os.path.join(LIBDIR, "libdolb.so")

DOLB_OK, INVALID_ARGUMENT, CONFIG, IO, DISPATCH, EXCHANGE, INTERNAL = range(7)


class DolbError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"dolb status {status}: {message}")
        self.status = status
        self.message = message


class Dolb:
    def __init__(self, path: str = DOLB_LIB):
        if not os.path.exists(path):
            raise OSError(f"{path} is missing: run paper_2506_09242_b200.build.build() first")
        lib = C.CDLL(path)
        lib.dolb_version.restype = C.c_char_p
        lib.dolb_last_error.restype = C.c_char_p
        lib.dolb_config_new.restype = C.c_void_p
        lib.dolb_config_free.argtypes = [C.c_void_p]
        lib.dolb_config_load.argtypes = [C.c_void_p, C.c_char_p]
        lib.dolb_config_set.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p]
        lib.dolb_config_get.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_size_t]
        lib.dolb_run.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        lib.dolb_show_models.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        lib.dolb_bytes_per_cell.argtypes = [C.c_int, C.POINTER(C.c_int64)]
        lib.dolb_peak_glups.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_double)]
        lib.dolb_memory_fraction.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int64, C.POINTER(C.c_double)]
        self.lib = lib

    # -- raw calls (status codes) ------------------------------------------------
    def last_error(self) -> str:
        return self.lib.dolb_last_error().decode()

    def version(self) -> str:
        return self.lib.dolb_version().decode()

    def check(self, status: int):
        if status != DOLB_OK:
            raise DolbError(status, self.last_error())

    # -- configuration handle ------------------------------------------------------
    def config(self, values: dict | None = None) -> "DolbConfig":
        return DolbConfig(self, values)

    def run(self, values: dict):
        with self.config(values) as cfg:
            return cfg.run()

    def show_models(self, values: dict) -> list:
        with self.config(values) as cfg:
            return cfg.show_models()

    def bytes_per_cell(self, bits: int) -> int:
        out = C.c_int64()
        self.check(self.lib.dolb_bytes_per_cell(bits, C.byref(out)))
        return out.value

    def peak_glups(self, device: str, bits: int, catalog: str | None = None) -> float:
        out = C.c_double()
        self.check(self.lib.dolb_peak_glups(device.encode(), catalog.encode() if catalog else None, bits,
                                            C.byref(out)))
        return out.value

    def memory_fraction(self, device: str, bits: int, L: int, catalog: str | None = None) -> float:
        out = C.c_double()
        self.check(self.lib.dolb_memory_fraction(device.encode(), catalog.encode() if catalog else None, bits, L,
                                                 C.byref(out)))
        return out.value


class DolbConfig:
    def __init__(self, api: Dolb, values: dict | None = None):
        self.api = api
        self.handle = C.c_void_p(api.lib.dolb_config_new())
        for k, v in (values or {}).items():
            self.set(k, v)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.free()

    def free(self):
        if self.handle:
            self.api.lib.dolb_config_free(self.handle)
            self.handle = C.c_void_p()

    def set(self, key: str, value):
        self.api.check(self.api.lib.dolb_config_set(self.handle, key.encode(), str(value).encode()))

    def load(self, path: str):
        self.api.check(self.api.lib.dolb_config_load(self.handle, path.encode()))

    def get(self, key: str, capacity: int = 4096) -> str:
        buf = C.create_string_buffer(capacity)
        self.api.check(self.api.lib.dolb_config_get(self.handle, key.encode(), buf, capacity))
        return buf.value.decode()

    def run(self):
        steps, mlups = C.c_int64(), C.c_double()
        self.api.check(self.api.lib.dolb_run(self.handle, C.byref(steps), C.byref(mlups)))
        return steps.value, mlups.value

    def show_models(self) -> list:
        n = C.c_size_t()
        self.api.check(self.api.lib.dolb_show_models(self.handle, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        self.api.check(self.api.lib.dolb_show_models(self.handle, buf, n.value, None))
        return [s for s in buf.value.decode().split("\n") if s]


def run(values: dict):
    """dolb_run on this package's device runner: (steps, MLUPS)."""
    return Dolb().run(values)


def show_models(values: dict) -> list:
    return Dolb().show_models(values)
