"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the CPU oracle.

Two checkers live here:

* ``Oracle``  -> ``oracle/build/liblbm_oracle.so``: the plain-C restatement of
  the reference algorithm (oracle/lbm_oracle.c).
* ``Reference`` -> ``oracle/_ref/libdolb_refshim.so``: the UNMODIFIED reference
  sources (/root/reference/proj) compiled by oracle/Makefile, driven through
  their public C++ API by oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg import this module. The product (paper_2506_09242_b200) never does.

Case helpers restate the reference input generators so both checkers and the
product see identical inputs:
  convective scaling ..... proj/src/cases.cpp:16-50
  cavity chains .......... proj/src/cases.cpp:160-189
  porous chains .......... proj/src/cases.cpp:191-260
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liblbm_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdolb_refshim.so")

KCS = 0.57735026918962576451  # cases.cpp:12

# recipe kinds / bases, chain.hpp:88 and chain.hpp:14-24
NODYN, BB, MBB, COLLIDE = 0, 1, 2, 3
BGK, TRT, RR = 0, 1, 2
BASE_NAMES = {BGK: "BGK", TRT: "TRT", RR: "RR"}


class OrcRecipe(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("base", C.c_int32), ("has_regularized", C.c_int32),
        ("reg_is_pressure", C.c_int32), ("reg_axis", C.c_int32), ("reg_orient", C.c_int32),
        ("has_les", C.c_int32), ("pad", C.c_int32),
        ("omega", C.c_double), ("lambda_", C.c_double), ("smagorinsky_c", C.c_double),
        ("omega_bulk_ho", C.c_double), ("wall_velocity", C.c_double * 3),
        ("target_rho", C.c_double),
    ]


@dataclass
class Recipe:
    """Python image of ChainRecipe (chain.hpp:86-102) plus its chain string and
    serialized parameter record (chain.cpp:87-98, 153-186)."""
    kind: int = COLLIDE
    base: int = BGK
    has_regularized: bool = False
    reg_is_pressure: bool = False
    reg_axis: int = 0
    reg_orient: int = 1
    has_les: bool = False
    omega: float = 1.0
    lambda_: float = 3.0 / 16.0
    smagorinsky_c: float = 0.0
    omega_bulk_ho: float = 1.0
    wall_velocity: tuple = (0.0, 0.0, 0.0)
    target_rho: float = 1.0

    def chain_string(self) -> str:
        if self.kind == NODYN:
            return "NoDynamics"
        if self.kind == BB:
            return "BounceBack"
        if self.kind == MBB:
            return "MovingBounceBack"
        links = []
        if self.has_regularized:
            kind = "Pressure" if self.reg_is_pressure else "Velocity"
            o = "1" if self.reg_orient > 0 else "M1"
            reg = f"Boundary_Regularized{kind}_{self.reg_axis}_{o}"
            if not self.has_les:
                return reg + "__" + BASE_NAMES[self.base]
            links.append(reg)
        if self.has_les:
            links.append("LES_Smagorinsky")
        links.append("COLL_" + BASE_NAMES[self.base])
        return "|".join(links)

    def params(self) -> list:
        """serialize_params (chain.cpp:153-186): each link appends its values."""
        out = []
        if self.kind == MBB:
            return list(self.wall_velocity)
        if self.kind != COLLIDE:
            return out
        if self.has_regularized:
            out += [self.target_rho] if self.reg_is_pressure else list(self.wall_velocity)
        if self.has_les:
            out.append(self.smagorinsky_c)
        out.append(self.omega)
        if self.base == TRT:
            out.append(self.lambda_)
        elif self.base == RR:
            out.append(self.omega_bulk_ho)
        return out

    def c_struct(self) -> OrcRecipe:
        r = OrcRecipe()
        r.kind, r.base = self.kind, self.base
        r.has_regularized, r.reg_is_pressure = int(self.has_regularized), int(self.reg_is_pressure)
        r.reg_axis, r.reg_orient, r.has_les = self.reg_axis, self.reg_orient, int(self.has_les)
        r.omega, r.lambda_, r.smagorinsky_c = self.omega, self.lambda_, self.smagorinsky_c
        r.omega_bulk_ho, r.target_rho = self.omega_bulk_ho, self.target_rho
        for a in range(3):
            r.wall_velocity[a] = self.wall_velocity[a]
        return r


def omega_from_viscosity(nu: float) -> float:  # collision.hpp:34-36
    return 1.0 / (3.0 * nu + 0.5)


@dataclass
class Case:
    """Flat mirror of dolb::CaseConfig (cases.hpp:22-54)."""
    kind: str = "tgv"            # tgv | cavity | porous
    L: int = 64
    Re: float = 1600.0
    Ma: float = 0.2
    collision: int = BGK
    smagorinsky_c: float | None = None
    lambda_: float = 3.0 / 16.0
    omega_bulk_ho: float = 1.0
    drive: str = "velocity"
    tau: float = 1.0
    delta_rho: float = 2e-3
    upstream: int = 40
    downstream: int = 40
    plate_layers: int = 11
    geometry: str = "plates"     # "plates" or raw voxel path
    voxel_dims: tuple = (0, 0, 0)
    q: int = 19
    mask: np.ndarray | None = field(default=None, repr=False)  # solid mask (z,y,x) for porous

    # cases.cpp:16-50
    def lattice_velocity(self) -> float:
        return KCS * self.Ma

    def char_length(self) -> float:
        if self.kind == "tgv":
            return float(self.L) / (2.0 * math.pi)
        return float(self.L)

    def viscosity(self) -> float:
        if self.kind == "porous":
            return (self.tau - 0.5) / 3.0
        return self.lattice_velocity() * self.char_length() / self.Re

    def omega(self) -> float:
        if self.kind == "porous":
            return 1.0 / self.tau
        return omega_from_viscosity(self.viscosity())

    def bulk_recipe(self) -> Recipe:
        r = Recipe(kind=COLLIDE, base=self.collision, omega=self.omega())
        if self.collision == TRT:
            r.lambda_ = self.lambda_
        if self.collision == RR:
            r.omega_bulk_ho = self.omega_bulk_ho
        if self.smagorinsky_c is not None and self.kind != "porous":
            r.has_les, r.smagorinsky_c = True, self.smagorinsky_c
        return r

    def solid_mask(self) -> np.ndarray:
        """Solid occupancy of the porous box (z, y, x), cases.cpp:229-236."""
        if self.mask is not None:
            return self.mask
        if self.geometry == "plates":
            gd = (self.L, self.L, self.plate_layers + 2)
        else:
            gd = tuple(self.voxel_dims)
        nx = gd[0] + self.upstream + self.downstream
        m = np.zeros((gd[2], gd[1], nx), dtype=bool)
        if self.geometry == "plates":
            m[0, :, :] = True
            m[gd[2] - 1, :, :] = True
        else:
            raw = np.fromfile(self.geometry, dtype=np.uint8).reshape(gd[2], gd[1], gd[0])
            m[:, :, self.upstream:self.upstream + gd[0]] = raw.astype(np.float64) > 0.5 * 255.0
        return m

    def setup(self):
        """(dims, periodic, recipes, slot[z,y,x]) — slot indexes recipes."""
        if self.kind == "tgv":
            L = self.L
            return (L, L, L), (1, 1, 1), [self.bulk_recipe()], np.zeros((L, L, L), np.int32)
        if self.kind == "cavity":
            L = self.L
            bulk = self.bulk_recipe()
            wall = Recipe(kind=BB)
            lid = Recipe(kind=MBB, wall_velocity=(self.lattice_velocity(), 0.0, 0.0))
            slot = np.zeros((L, L, L), np.int32)
            z, y, x = np.meshgrid(np.arange(L), np.arange(L), np.arange(L), indexing="ij")
            walls = (x == 0) | (x == L - 1) | (y == 0) | (y == L - 1) | (z == 0)
            slot[walls] = 1
            slot[z == L - 1] = 2
            return (L, L, L), (0, 0, 0), [bulk, wall, lid], slot
        # porous, cases.cpp:191-260
        solid = self.solid_mask()
        nz, ny, nx = solid.shape
        bulk = self.bulk_recipe()
        u_in = self.lattice_velocity()
        mk = dict(kind=COLLIDE, base=self.collision, omega=bulk.omega, lambda_=bulk.lambda_,
                  omega_bulk_ho=bulk.omega_bulk_ho, has_regularized=True, reg_axis=0)
        if self.drive == "velocity":
            inlet = Recipe(reg_orient=1, wall_velocity=(u_in, 0.0, 0.0), **mk)
            outlet = Recipe(reg_orient=-1, wall_velocity=(u_in, 0.0, 0.0), **mk)
        else:
            inlet = Recipe(reg_orient=1, reg_is_pressure=True, target_rho=1.0 + self.delta_rho, **mk)
            outlet = Recipe(reg_orient=-1, reg_is_pressure=True, target_rho=1.0 - self.delta_rho, **mk)
        recipes = [bulk, Recipe(kind=BB), Recipe(kind=NODYN), inlet, outlet]
        c = descriptor(19)[0]
        fluid_nb = np.zeros_like(solid)
        for i in range(1, 19):
            cx, cy, cz = c[i]
            sh = np.roll(solid, shift=(-cz, -cy), axis=(0, 1))  # y/z periodic wrap
            nbr = np.ones_like(solid)  # outside in x: ignored (continue)
            if cx == 0:
                nbr = sh
            elif cx == 1:
                nbr[:, :, :-1] = sh[:, :, 1:]
            else:
                nbr[:, :, 1:] = sh[:, :, :-1]
            fluid_nb |= ~nbr
        slot = np.zeros(solid.shape, np.int32)
        slot[:, :, 0] = 3
        slot[:, :, nx - 1] = 4
        slot[solid & fluid_nb] = 1
        slot[solid & ~fluid_nb] = 2
        return (nx, ny, nz), (0, 1, 1), recipes, slot

    def ref_struct(self):
        rc = RefCase()
        rc.kind = {"tgv": 0, "cavity": 1, "porous": 2}[self.kind]
        rc.collision = self.collision
        rc.L, rc.Re, rc.Ma = self.L, self.Re, self.Ma
        rc.lambda_, rc.omega_bulk_ho = self.lambda_, self.omega_bulk_ho
        rc.smagorinsky_c = float("nan") if self.smagorinsky_c is None else self.smagorinsky_c
        rc.drive = 0 if self.drive == "velocity" else 1
        rc.tau, rc.delta_rho = self.tau, self.delta_rho
        rc.upstream, rc.downstream, rc.plate_layers = self.upstream, self.downstream, self.plate_layers
        for a in range(3):
            rc.voxel_dims[a] = self.voxel_dims[a]
        rc._geom = self.geometry.encode()
        rc.geometry = rc._geom
        return rc


class RefCase(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("collision", C.c_int32), ("L", C.c_int64),
        ("Re", C.c_double), ("Ma", C.c_double), ("lambda_", C.c_double),
        ("omega_bulk_ho", C.c_double), ("smagorinsky_c", C.c_double),
        ("drive", C.c_int32), ("pad0", C.c_int32), ("tau", C.c_double), ("delta_rho", C.c_double),
        ("upstream", C.c_int64), ("downstream", C.c_int64), ("plate_layers", C.c_int64),
        ("voxel_dims", C.c_int64 * 3), ("geometry", C.c_char_p),
    ]


_DESC = {}


def descriptor(q: int):
    if q not in _DESC:
        o = Oracle()
        c = np.zeros(q * 3, np.int32)
        w = np.zeros(q, np.float64)
        opp = np.zeros(q, np.int32)
        o.lib.orc_descriptor(q, c.ctypes.data, w.ctypes.data, opp.ctypes.data)
        _DESC[q] = (c.reshape(q, 3), w, opp)
    return _DESC[q]


def _ptr(a):
    return C.c_void_p(a.ctypes.data)


class Oracle:
    _lib = None

    def __init__(self):
        if Oracle._lib is None:
            if not os.path.exists(ORACLE_SO):
                raise RuntimeError(f"oracle not built: {ORACLE_SO} (run make -C oracle)")
            lib = C.CDLL(ORACLE_SO)
            # every pointer argument declared: an undeclared one is passed as a
            # 32-bit C int (the descriptor call segfaulted whenever numpy placed
            # its arrays above 4 GiB)
            lib.orc_descriptor.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
            lib.orc_derive_omega_minus.restype = C.c_double
            lib.orc_derive_omega_minus.argtypes = [C.c_double, C.c_double]
            for fn in ("orc_equilibrium_d",):
                getattr(lib, fn).argtypes = [C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_void_p]
            lib.orc_equilibrium_f.argtypes = [C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_void_p]
            for fn in ("orc_apply_d", "orc_apply_f"):
                getattr(lib, fn).argtypes = [C.c_int, C.POINTER(OrcRecipe), C.c_void_p, C.c_int64]
            for fn in ("orc_fill_equilibrium_d", "orc_fill_equilibrium_f"):
                getattr(lib, fn).argtypes = [C.c_int, C.c_int64] + [C.c_void_p] * 5
            for fn in ("orc_step_d", "orc_step_f"):
                getattr(lib, fn).argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.POINTER(OrcRecipe),
                                             C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_int64, C.c_int]
            lib.orc_tgv_state.argtypes = [C.c_int64, C.c_double, C.c_int64, C.c_int64] + [C.c_void_p] * 4
            Oracle._lib = lib
        self.lib = Oracle._lib

    def derive_omega_minus(self, omega, lam):
        return self.lib.orc_derive_omega_minus(omega, lam)

    def equilibrium(self, q, order, rho, u, dtype=np.float64):
        out = np.zeros(q, dtype)
        uu = np.asarray(u, dtype)
        if dtype == np.float64:
            self.lib.orc_equilibrium_d(q, order, rho, _ptr(uu), _ptr(out))
        else:
            self.lib.orc_equilibrium_f(q, order, rho, _ptr(uu), _ptr(out))
        return out

    def apply(self, q, recipe: Recipe, f: np.ndarray) -> np.ndarray:
        """f: (n, q) cell-major; returns a new array."""
        g = np.ascontiguousarray(f).copy()
        r = recipe.c_struct()
        fn = self.lib.orc_apply_d if g.dtype == np.float64 else self.lib.orc_apply_f
        fn(q, C.byref(r), _ptr(g), g.shape[0])
        return g

    def tgv_state(self, L, u_inf, z0=0, nz=None):
        nz = L if nz is None else nz
        n = L * L * nz
        arrs = [np.zeros(n) for _ in range(4)]
        self.lib.orc_tgv_state(L, u_inf, z0, nz, *[_ptr(a) for a in arrs])
        return arrs

    def fill_equilibrium(self, q, rho, ux, uy, uz, dtype):
        n = rho.size
        f = np.zeros(q * n, dtype)
        fn = self.lib.orc_fill_equilibrium_d if dtype == np.float64 else self.lib.orc_fill_equilibrium_f
        fn(q, n, *[_ptr(np.ascontiguousarray(a, np.float64)) for a in (rho, ux, uy, uz)], _ptr(f))
        return f

    def initial_state(self, case: Case, dtype):
        dims, _, _, _ = case.setup()
        n = dims[0] * dims[1] * dims[2]
        if case.kind == "tgv":
            rho, ux, uy, uz = self.tgv_state(case.L, case.lattice_velocity())
        else:
            rho, ux, uy, uz = np.ones(n), np.zeros(n), np.zeros(n), np.zeros(n)
        return self.fill_equilibrium(case.q, rho, ux, uy, uz, dtype)

    def step(self, q, dims, periodic, recipes, slot, f, nsteps, nthreads=None):
        """In place on f (canonical, direction-major, x fastest)."""
        nthreads = nthreads or min(8, os.cpu_count() or 1)
        dims_a = np.asarray(dims, np.int64)
        per = np.asarray(periodic, np.int32)
        arr = (OrcRecipe * len(recipes))(*[r.c_struct() for r in recipes])
        sl = np.ascontiguousarray(slot, np.int32)
        scratch = np.empty_like(f)
        fn = self.lib.orc_step_d if f.dtype == np.float64 else self.lib.orc_step_f
        rc = fn(q, _ptr(dims_a), _ptr(per), arr, len(recipes), _ptr(sl), _ptr(f), _ptr(scratch),
                nsteps, nthreads)
        if rc != 0:
            raise RuntimeError(f"orc_step failed ({rc})")
        return f

    def run_case(self, case: Case, dtype, nsteps, nthreads=None):
        dims, periodic, recipes, slot = case.setup()
        f = self.initial_state(case, dtype)
        return self.step(case.q, dims, periodic, recipes, slot, f, nsteps, nthreads)


class Reference:
    """The unmodified reference solver (oracle/_ref, built from /root/reference)."""
    _lib = None

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        if Reference._lib is None:
            if not os.path.exists(REF_SO):
                raise RuntimeError(f"reference shim not built: {REF_SO}")
            lib = C.CDLL(REF_SO)
            lib.ref_last_error.restype = C.c_char_p
            lib.ref_case_dims.argtypes = [C.POINTER(RefCase), C.c_void_p]
            lib.ref_case_tags.argtypes = [C.POINTER(RefCase), C.c_void_p, C.c_char_p, C.c_size_t]
            lib.ref_case_run.argtypes = [C.POINTER(RefCase), C.c_int, C.c_void_p, C.c_int,
                                         C.c_int64, C.c_void_p]
            lib.ref_case_bench.argtypes = [C.POINTER(RefCase), C.c_int, C.c_int, C.c_int64,
                                           C.c_int64, C.c_int, C.c_void_p, C.POINTER(C.c_double)]
            lib.ref_apply_chain.argtypes = [C.c_char_p, C.c_void_p, C.c_size_t, C.c_int,
                                            C.c_void_p, C.c_int64]
            lib.ref_equilibrium.argtypes = [C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_void_p]
            lib.ref_derive_omega_minus.restype = C.c_double
            lib.ref_derive_omega_minus.argtypes = [C.c_double, C.c_double]
            lib.ref_chain_roundtrip.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
            lib.ref_case_macro.argtypes = [C.POINTER(RefCase), C.c_int, C.c_int64] + [C.c_void_p] * 4
            lib.ref_case_dump.argtypes = [C.POINTER(RefCase), C.c_int, C.c_int64, C.c_char_p]
            lib.ref_case_checksum.argtypes = [C.POINTER(RefCase), C.c_int, C.c_void_p, C.c_int,
                                              C.c_int64, C.c_void_p]
            lib.ref_case_checksum_masked.argtypes = [C.POINTER(RefCase), C.c_int, C.c_void_p, C.c_int,
                                                     C.c_int64, C.c_void_p, C.c_void_p]
            lib.ref_case_sample.argtypes = [C.POINTER(RefCase), C.c_int, C.c_int64, C.c_int64, C.c_void_p]
            lib.ref_tree_sum.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_double)]
            Reference._lib = lib
        self.lib = Reference._lib

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def dims(self, case: Case):
        d = np.zeros(3, np.int64)
        rc = case.ref_struct()
        self._check(self.lib.ref_case_dims(C.byref(rc), _ptr(d)))
        return tuple(int(v) for v in d)

    def tags(self, case: Case):
        d = self.dims(case)
        tags = np.zeros(d[0] * d[1] * d[2], np.int32)
        buf = C.create_string_buffer(1 << 16)
        rc = case.ref_struct()
        self._check(self.lib.ref_case_tags(C.byref(rc), _ptr(tags), buf, len(buf)))
        models = [m for m in buf.value.decode().split("\n") if m]
        return tags.reshape(d[2], d[1], d[0]), models

    def run_case(self, case: Case, precision_bits: int, nsteps: int, grid=(1, 1, 1), workers=1):
        d = self.dims(case)
        out = np.zeros(19 * d[0] * d[1] * d[2], np.float64)
        g = np.asarray(grid, np.int32)
        rc = case.ref_struct()
        self._check(self.lib.ref_case_run(C.byref(rc), precision_bits, _ptr(g), workers, nsteps, _ptr(out)))
        return out

    def macroscopic(self, case: Case, precision_bits: int, nsteps: int):
        d = self.dims(case)
        n = d[0] * d[1] * d[2]
        arrs = [np.zeros(n) for _ in range(4)]
        rc = case.ref_struct()
        self._check(self.lib.ref_case_macro(C.byref(rc), precision_bits, nsteps, *[_ptr(a) for a in arrs]))
        return tuple(arrs)

    def sample(self, case: Case, precision_bits: int, steps_a: int, steps_b: int) -> dict:
        """The runner's sampling step on the reference's own fields
        (runner.cpp:346-448): kinetic energy and enstrophy after steps_a + steps_b,
        the cavity convergence sums between the two samples, porous extras."""
        out = np.zeros(9)
        rc = case.ref_struct()
        self._check(self.lib.ref_case_sample(C.byref(rc), precision_bits, steps_a, steps_b, _ptr(out)))
        keys = ["k", "eps", "nn", "dd", "k_perm", "ubar", "dp", "ux_in", "ux_out"]
        return dict(zip(keys, (float(v) for v in out)))

    def tree_sum(self, values: np.ndarray) -> float:
        v = np.ascontiguousarray(values, np.float64)
        out = C.c_double()
        self._check(self.lib.ref_tree_sum(_ptr(v), v.size, C.byref(out)))
        return out.value

    def dump(self, case: Case, precision_bits: int, nsteps: int, path: str):
        rc = case.ref_struct()
        self._check(self.lib.ref_case_dump(C.byref(rc), precision_bits, nsteps, path.encode()))

    def checksum(self, case: Case, precision_bits: int, nsteps: int, grid=(1, 1, 1), workers=1):
        out = np.zeros(19, np.uint64)
        g = np.asarray(grid, np.int32)
        rc = case.ref_struct()
        self._check(self.lib.ref_case_checksum(C.byref(rc), precision_bits, _ptr(g), workers, nsteps,
                                               _ptr(out)))
        return [int(v) for v in out]

    def checksum_masked(self, case: Case, precision_bits: int, nsteps: int, grid=(1, 1, 1), workers=1):
        """(checksum of every cell, checksum of the cells whose chain is not
        NoDynamics), streamed over the reference's blocks (no gather copy)."""
        out = np.zeros(19, np.uint64)
        act = np.zeros(19, np.uint64)
        g = np.asarray(grid, np.int32)
        rc = case.ref_struct()
        self._check(self.lib.ref_case_checksum_masked(C.byref(rc), precision_bits, _ptr(g), workers, nsteps,
                                                      _ptr(out), _ptr(act)))
        return [int(v) for v in out], [int(v) for v in act]

    def bench(self, case: Case, precision_bits: int, workers: int, warmup: int, steps: int, reps: int = 3):
        reps_out = np.zeros(reps)
        mean = C.c_double()
        rc = case.ref_struct()
        self._check(self.lib.ref_case_bench(C.byref(rc), precision_bits, workers, warmup, steps, reps,
                                            _ptr(reps_out), C.byref(mean)))
        return mean.value, list(reps_out)

    def apply_chain(self, chain: str, params, precision_bits: int, f: np.ndarray):
        g = np.ascontiguousarray(f, np.float64).copy()
        p = np.asarray(params, np.float64)
        self._check(self.lib.ref_apply_chain(chain.encode(), _ptr(p), p.size, precision_bits,
                                             _ptr(g), g.shape[0]))
        return g

    def equilibrium(self, order, precision_bits, rho, u):
        out = np.zeros(19)
        uu = np.asarray(u, np.float64)
        self._check(self.lib.ref_equilibrium(order, precision_bits, rho, _ptr(uu), _ptr(out)))
        return out

    def derive_omega_minus(self, omega, lam):
        return self.lib.ref_derive_omega_minus(omega, lam)

    def chain_roundtrip(self, s: str) -> str:
        buf = C.create_string_buffer(4096)
        self._check(self.lib.ref_chain_roundtrip(s.encode(), buf, len(buf)))
        return buf.value.decode()


def canonical_hash(pops: np.ndarray) -> str:
    """sha256 of the canonical population array as float64 with -0.0 folded to
    +0.0 (values, not zero signs, define parity)."""
    import hashlib
    a = np.ascontiguousarray(pops, dtype=np.float64) + 0.0
    return hashlib.sha256(a.tobytes()).hexdigest()


def canonical_checksum(pops: np.ndarray, q: int = 19) -> list:
    """Per-direction sum of bits(f + 0.0) * (cell index + 1) mod 2^64 — the
    dlb_lattice_checksum definition, from a canonical population array."""
    a = (np.ascontiguousarray(pops, dtype=np.float64) + 0.0).reshape(q, -1)
    n = a.shape[1]
    w = np.arange(1, n + 1, dtype=np.uint64)
    bits = a.view(np.uint64)
    with np.errstate(over="ignore"):
        return [int(np.sum(bits[i] * w, dtype=np.uint64)) for i in range(q)]
