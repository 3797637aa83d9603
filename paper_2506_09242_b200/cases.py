"""Benchmark case input generators (the reference's cases layer).

  CaseConfig + convective scaling ...... proj/include/dolb/cases.hpp:22-54, src/cases.cpp:16-50
  init_tgv ............................. src/cases.cpp:127-158
  init_cavity .......................... src/cases.cpp:160-189
  init_porous .......................... src/cases.cpp:191-260
  load_voxels / make_plate_geometry .... src/cases.cpp:86-125
  build_run ............................ src/cases.cpp:279-297 (DeviceRun instead of MultiBlockRun)
  sphere_pack (new: SURVEY.md §8d c4) .. seeded Boolean sphere model in the raw voxel format

Chain assignment is computed with numpy over the whole grid; the TGV state is
evaluated on the device from glibc sin/cos tables (bit-identical to the
reference's host evaluation), other cases start at rest.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from .dolb import (D3Q19, CollisionParams, DeviceRun, DispatchSet, DynamicsRegistry, LinkType,
                   make_bounce_back, make_collision_chain, make_moving_bounce_back,
                   make_no_dynamics, make_regularized_pressure, make_regularized_velocity)

KCS = 0.57735026918962576451  # 1/sqrt(3), cases.cpp:12


def omega_from_viscosity(nu: float) -> float:
    return 1.0 / (3.0 * nu + 0.5)


@dataclass
class CaseConfig:
    kind: str = "tgv"  # tgv | cavity | porous
    L: int = 64
    Re: float = 1600.0
    Ma: float = 0.2
    collision: LinkType = LinkType.BGK
    smagorinsky_c: float | None = None
    lambda_: float = 3.0 / 16.0
    omega_bulk_ho: float = 1.0
    q: int = 19
    # porous
    drive: str = "velocity"
    geometry: str = "plates"
    plate_layers: int = 11
    tau: float = 1.0
    delta_rho: float = 2e-3
    upstream: int = 40
    downstream: int = 40
    voxel_dims: tuple = (0, 0, 0)
    voxel_threshold: float = 0.5
    mask: np.ndarray | None = field(default=None, repr=False)  # raw voxels (z, y, x) u8

    def lattice_velocity(self) -> float:
        return KCS * self.Ma

    def char_length(self) -> float:
        return float(self.L) / (2.0 * math.pi) if self.kind == "tgv" else float(self.L)

    def viscosity(self) -> float:
        if self.kind == "porous":
            return (self.tau - 0.5) / 3.0
        return self.lattice_velocity() * self.char_length() / self.Re

    def omega(self) -> float:
        return 1.0 / self.tau if self.kind == "porous" else omega_from_viscosity(self.viscosity())

    def t_c(self) -> float:
        return self.char_length() / self.lattice_velocity()

    def validate(self):
        if self.kind == "tgv" and self.L < 8:
            raise ValueError("tgv requires L >= 8")
        if self.kind == "cavity" and self.L < 16:
            raise ValueError("cavity requires L >= 16")
        if not (0.0 < self.Ma < 0.5):
            raise ValueError("Mach number must lie in (0, 0.5)")
        om = self.omega()
        if not (0.0 < om < 2.0):
            raise ValueError(f"relaxation rate {om} outside the stable range (0, 2)")

    def collision_params(self) -> CollisionParams:
        p = CollisionParams().set_trt(self.omega(), self.lambda_)
        p.omega_bulk_ho = self.omega_bulk_ho
        return p


@dataclass
class CaseSetup:
    dims: tuple
    periodic: tuple
    chains: list            # DynamicsChain per local chain index
    chain_index: np.ndarray | int  # (nz, ny, nx) index into chains, or a scalar
    state: tuple            # ('tgv', L, u) | ('rest',)
    t_c: float = 1.0
    q: int = 19
    sample_begin: int = 0
    sample_end: int = 0


def init_tgv(cfg: CaseConfig) -> CaseSetup:
    cfg.validate()
    L = cfg.L
    bulk = make_collision_chain(cfg.collision, cfg.collision_params(), cfg.smagorinsky_c)
    return CaseSetup((L, L, L), (1, 1, 1), [bulk], 0, ("tgv", L, cfg.lattice_velocity()),
                     cfg.t_c(), cfg.q)


def init_cavity(cfg: CaseConfig) -> CaseSetup:
    cfg.validate()
    L = cfg.L
    bulk = make_collision_chain(cfg.collision, cfg.collision_params(), cfg.smagorinsky_c)
    wall = make_bounce_back()
    lid = make_moving_bounce_back((cfg.lattice_velocity(), 0.0, 0.0))
    idx = np.zeros((L, L, L), np.int32)
    r = np.arange(L)
    edge = (r == 0) | (r == L - 1)
    walls = edge[None, None, :] | edge[None, :, None] | (r == 0)[:, None, None]
    idx[walls] = 1
    idx[L - 1] = 2
    return CaseSetup((L, L, L), (0, 0, 0), [bulk, wall, lid], idx, ("rest",), cfg.t_c(), cfg.q)


def make_plate_mask(length: int, width: int, layers: int) -> np.ndarray:
    """Parallel plates: solid rows at z = 0 and z = H + 1 (cases.cpp:113-125); (z, y, x) bool."""
    m = np.zeros((layers + 2, width, length), bool)
    m[0] = True
    m[layers + 1] = True
    return m


def load_voxels(path: str, dims, threshold: float = 0.5) -> np.ndarray:
    """Raw 8-bit occupancy, x fastest; value > threshold*255 is solid (cases.cpp:86-111)."""
    raw = np.fromfile(path, dtype=np.uint8)
    n = int(dims[0]) * int(dims[1]) * int(dims[2])
    if raw.size != n:
        raise OSError(f'voxel file "{path}" has {raw.size} bytes, expected {n}')
    solid = raw.astype(np.float64).reshape(dims[2], dims[1], dims[0]) > threshold * 255.0
    phi = 1.0 - solid.mean()
    if phi <= 0.0 or phi >= 1.0:
        raise OSError(f"degenerate medium: porosity {phi}")
    return solid


def sphere_pack(dims, radius: float = 8.0, porosity: float = 0.20, seed: int = 20250611):
    """Seeded Boolean sphere pack in the raw voxel format (u8, 255 = solid,
    x fastest). Returns (voxels (nz, ny, nx) u8, achieved porosity)."""
    nx, ny, nz = (int(v) for v in dims)
    out = np.zeros(nx * ny * nz, np.uint8)
    phi = C.c_double()
    _capi.check(_capi.lib().dlb_case_sphere_pack(nx, ny, nz, radius, porosity, seed,
                                                 out.ctypes.data, C.byref(phi)))
    return out.reshape(nz, ny, nx), phi.value


def init_porous(cfg: CaseConfig, solid: np.ndarray | None = None) -> CaseSetup:
    """Porous sample between `upstream` / `downstream` fluid buffers along x,
    lateral periodic, regularized inlet / outlet (cases.cpp:191-260).
    `solid` is the (z, y, x) bool mask of the sample (plates if None)."""
    cfg.validate()
    plates = solid is None and cfg.geometry == "plates"
    if solid is None:
        if plates:
            solid = make_plate_mask(cfg.L, cfg.L, cfg.plate_layers)
        else:
            solid = load_voxels(cfg.geometry, cfg.voxel_dims, cfg.voxel_threshold)
    gz, gy, gx = solid.shape
    nx = gx + cfg.upstream + cfg.downstream
    full = np.zeros((gz, gy, nx), bool)
    if plates:
        full[0] = True
        full[gz - 1] = True
    else:
        full[:, :, cfg.upstream:cfg.upstream + gx] = solid
    params = cfg.collision_params()
    bulk = make_collision_chain(cfg.collision, params)
    u_in = cfg.lattice_velocity()
    if cfg.drive == "velocity":
        inlet = make_regularized_velocity(0, 1, (u_in, 0.0, 0.0), cfg.collision, params)
        outlet = make_regularized_velocity(0, -1, (u_in, 0.0, 0.0), cfg.collision, params)
    else:
        inlet = make_regularized_pressure(0, 1, 1.0 + cfg.delta_rho, cfg.collision, params)
        outlet = make_regularized_pressure(0, -1, 1.0 - cfg.delta_rho, cfg.collision, params)
    chains = [bulk, make_bounce_back(), make_no_dynamics(), inlet, outlet]
    # a solid cell with any fluid neighbour (y/z periodic, x bounded) bounces back
    c = D3Q19[0]
    fluid_nb = np.zeros_like(full)
    for i in range(1, 19):
        cx, cy, cz = (int(v) for v in c[i])
        sh = np.roll(full, shift=(-cz, -cy), axis=(0, 1))
        nbr = np.ones_like(full)
        if cx == 0:
            nbr = sh
        elif cx == 1:
            nbr[:, :, :-1] = sh[:, :, 1:]
        else:
            nbr[:, :, 1:] = sh[:, :, :-1]
        fluid_nb |= ~nbr
    idx = np.zeros(full.shape, np.int32)
    idx[:, :, 0] = 3
    idx[:, :, nx - 1] = 4
    idx[full & fluid_nb] = 1
    idx[full & ~fluid_nb] = 2
    return CaseSetup((nx, gy, gz), (0, 1, 1), chains, idx, ("rest",), cfg.t_c(), cfg.q,
                     cfg.upstream, cfg.upstream + gx)


def build_run(setup: CaseSetup, registry: DynamicsRegistry | None = None, precision: int = 64,
              slabs: int = 1, dispatch: DispatchSet | None = None, arith: str = "exact",
              dist=None, devices=None, layout: str = "twopop",
              skip_nodynamics: bool = False, tma: bool = False, sparse_lists: bool = False) -> DeviceRun:
    """Register the setup's chains, build the device run, fill tags and state
    (cases.cpp:279-297 + multiblock.cpp:252-287)."""
    registry = registry or DynamicsRegistry()
    slot_of = [registry.register_chain(ch) for ch in setup.chains]
    run = DeviceRun(setup.dims, setup.periodic, registry, dispatch, q=setup.q, precision=precision,
                    slabs=slabs, arith=arith, dist=dist, devices=devices, layout=layout,
                    skip_nodynamics=skip_nodynamics, tma=tma, sparse_lists=sparse_lists)
    if np.isscalar(setup.chain_index):
        slots = slot_of[int(setup.chain_index)]
    else:
        slots = np.asarray(slot_of, np.int32)[setup.chain_index]
    run.fill(slots, setup.state)
    return run


def setup_models(setup: CaseSetup) -> list:
    """Distinct chain strings the setup assigns, sorted (cases.cpp:299-311)."""
    used = {0} if np.isscalar(setup.chain_index) else set(np.unique(setup.chain_index).tolist())
    return sorted({setup.chains[i].chain_string() for i in used})
