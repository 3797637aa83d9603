"""Reference-facing interface of the B200 collide-and-stream path.

Mirrors the names, argument meaning and error behaviour of the reference's
dynamics / data-processor API so that code written against it ports directly:

  LinkType, ChainLink, CollisionParams, ChainParams, DynamicsChain
        proj/include/dolb/chain.hpp:14-53, collision.hpp:12-31
  make_collision_chain / make_bounce_back / make_no_dynamics /
  make_moving_bounce_back / make_regularized_velocity / make_regularized_pressure
        proj/src/chain.cpp:249-297
  chain_string / parse_chain_string / serialize_params
        proj/src/chain.cpp:87-186
  DynamicsRegistry, DispatchSet, DispatchError
        proj/include/dolb/accelerated_lattice.hpp:16-79
  DeviceRun (the device twin of MultiBlockRun<T>: fill, advance,
  gather_populations, gather_macroscopic)   proj/include/dolb/multiblock.hpp:119-176
  partition (balanced split)                proj/src/multiblock.cpp:10-49
  collide_and_stream on a host block        proj/include/dolb/accelerated_lattice.hpp:124-127

Everything below the Python surface runs in libdlb_b200.so (C++ host runtime +
sm_100a kernels); this module only marshals arguments.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import (ARITH_EXACT, ARITH_FAST, LAYOUT_TWO_POP, ConfigError, DispatchError, DlbError,
                    ExchangeError, check)

__all__ = [
    "LinkType", "ChainLink", "CollisionParams", "ChainParams", "DynamicsChain",
    "make_collision_chain", "make_bounce_back", "make_no_dynamics", "make_moving_bounce_back",
    "make_regularized_velocity", "make_regularized_pressure", "chain_string", "serialize_params",
    "DynamicsRegistry", "DispatchSet", "DispatchError", "ExchangeError", "ConfigError", "DlbError",
    "DeviceRun", "partition", "collide_and_stream", "block_cache_release", "block_cache_info", "refresh_envelope_periodic", "read_field_dump", "D3Q19", "D3Q27",
]


class LinkType(enum.Enum):
    NoDynamics = "NoDynamics"
    BounceBack = "BounceBack"
    MovingBounceBack = "MovingBounceBack"
    BGK = "COLL_BGK"
    TRT = "COLL_TRT"
    RR = "COLL_RR"
    Smagorinsky = "LES_Smagorinsky"
    RegularizedVelocity = "Boundary_RegularizedVelocity"
    RegularizedPressure = "Boundary_RegularizedPressure"


BASES = (LinkType.BGK, LinkType.TRT, LinkType.RR)


@dataclass(frozen=True)
class ChainLink:
    type: LinkType
    axis: int = 0
    orient: int = 1

    def link_id(self) -> str:
        if self.type in (LinkType.RegularizedVelocity, LinkType.RegularizedPressure):
            return f"{self.type.value}_{self.axis}_{'1' if self.orient > 0 else 'M1'}"
        return self.type.value


def derive_omega_minus(omega: float, lam: float) -> float:
    """collision.hpp:19-22"""
    half_minus = lam / (1.0 / omega - 0.5)
    return 1.0 / (half_minus + 0.5)


@dataclass
class CollisionParams:
    omega: float = 1.0
    omega_minus: float = 1.0
    lambda_: float = 3.0 / 16.0
    smagorinsky_c: float = 0.0
    omega_bulk_ho: float = 1.0

    def set_trt(self, omega: float, lam: float):
        self.omega, self.lambda_ = omega, lam
        self.omega_minus = derive_omega_minus(omega, lam)
        return self


@dataclass
class ChainParams:
    collision: CollisionParams = field(default_factory=CollisionParams)
    wall_velocity: tuple = (0.0, 0.0, 0.0)
    target_rho: float = 1.0


@dataclass
class DynamicsChain:
    links: list
    params: ChainParams = field(default_factory=ChainParams)

    def chain_string(self) -> str:
        return chain_string(self)


def chain_string(chain: DynamicsChain) -> str:
    """Canonical chain string (chain.cpp:87-98), rendered by the C++ runtime."""
    raw = "|".join(l.link_id() for l in chain.links)
    return _capi.get_string(_capi.lib().dlb_chain_canonical, raw.encode())


def serialize_params(chain: DynamicsChain) -> list:
    """Parameter record, each link appending the values it consumes (chain.cpp:153-186)."""
    p = chain.params
    out = []
    for l in chain.links:
        t = l.type
        if t == LinkType.BGK:
            out.append(p.collision.omega)
        elif t == LinkType.TRT:
            out += [p.collision.omega, p.collision.lambda_]
        elif t == LinkType.RR:
            out += [p.collision.omega, p.collision.omega_bulk_ho]
        elif t == LinkType.Smagorinsky:
            out.append(p.collision.smagorinsky_c)
        elif t in (LinkType.MovingBounceBack, LinkType.RegularizedVelocity):
            out += [float(v) for v in p.wall_velocity]
        elif t == LinkType.RegularizedPressure:
            out.append(p.target_rho)
    return out


def _canonical_collision(base: LinkType, params: CollisionParams) -> CollisionParams:
    """chain.cpp:236-245: keep only what the base consumes."""
    c = CollisionParams(omega=params.omega)
    if base == LinkType.TRT:
        c.set_trt(params.omega, params.lambda_)
    elif base == LinkType.RR:
        c.omega_bulk_ho = params.omega_bulk_ho
    return c


def make_collision_chain(base: LinkType, params: CollisionParams, smagorinsky_c=None) -> DynamicsChain:
    coll = _canonical_collision(base, params)
    links = []
    if smagorinsky_c is not None:
        coll.smagorinsky_c = smagorinsky_c
        links.append(ChainLink(LinkType.Smagorinsky))
    links.append(ChainLink(base))
    return DynamicsChain(links, ChainParams(collision=coll))


def make_bounce_back() -> DynamicsChain:
    return DynamicsChain([ChainLink(LinkType.BounceBack)])


def make_no_dynamics() -> DynamicsChain:
    return DynamicsChain([ChainLink(LinkType.NoDynamics)])


def make_moving_bounce_back(u_wall) -> DynamicsChain:
    return DynamicsChain([ChainLink(LinkType.MovingBounceBack)],
                         ChainParams(wall_velocity=tuple(float(v) for v in u_wall)))


def make_regularized_velocity(axis, orient, u, base, params) -> DynamicsChain:
    return DynamicsChain([ChainLink(LinkType.RegularizedVelocity, axis, orient), ChainLink(base)],
                         ChainParams(collision=_canonical_collision(base, params),
                                     wall_velocity=tuple(float(v) for v in u)))


def make_regularized_pressure(axis, orient, rho, base, params) -> DynamicsChain:
    return DynamicsChain([ChainLink(LinkType.RegularizedPressure, axis, orient), ChainLink(base)],
                         ChainParams(collision=_canonical_collision(base, params), target_rho=rho))


class DynamicsRegistry:
    """Chain strings <-> tags plus the parameter table (accelerated_lattice.hpp:32-60).
    Tags are indices into the sorted chain-string set; slots are (chain, params) instances."""

    def __init__(self):
        h = C.c_void_p()
        check(_capi.lib().dlb_registry_new(C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _capi._lib is not None:
            _capi._lib.dlb_registry_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def register_chain(self, chain: DynamicsChain) -> int:
        raw = "|".join(l.link_id() for l in chain.links)
        rec = np.asarray(serialize_params(chain), np.float64)
        slot = C.c_int32()
        check(_capi.lib().dlb_registry_register(self._h, raw.encode(),
                                                rec.ctypes.data if rec.size else None,
                                                rec.size, C.byref(slot)))
        return slot.value

    def tag_for(self, chain_str: str) -> int:
        t = C.c_int32()
        check(_capi.lib().dlb_registry_tag_for(self._h, chain_str.encode(), C.byref(t)))
        return t.value

    def chain_for(self, tag: int) -> str:
        return _capi.get_string(_capi.lib().dlb_registry_chain_for, self._h, tag)

    def tag_of_slot(self, slot: int) -> int:
        t = C.c_int32()
        check(_capi.lib().dlb_registry_tag_of_slot(self._h, slot, C.byref(t)))
        return t.value

    def _counts(self):
        a, b = C.c_int32(), C.c_int32()
        check(_capi.lib().dlb_registry_counts(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def num_tags(self) -> int:
        return self._counts()[0]

    def num_instances(self) -> int:
        return self._counts()[1]

    def chain_strings(self) -> list:
        return [self.chain_for(t) for t in range(self.num_tags())]

    def slot_params(self, slot: int) -> list:
        n = C.c_size_t()
        check(_capi.lib().dlb_registry_slot_params(self._h, slot, None, 0, C.byref(n)))
        buf = np.zeros(max(n.value, 1))
        check(_capi.lib().dlb_registry_slot_params(self._h, slot, buf.ctypes.data, buf.size, C.byref(n)))
        return list(buf[:n.value])


class DispatchSet:
    """Explicit subset of registry tags admitted by the step kernel."""

    def __init__(self, tags=()):
        self.tags = set(int(t) for t in tags)

    @staticmethod
    def all_of(registry: DynamicsRegistry) -> "DispatchSet":
        return DispatchSet(range(registry.num_tags()))

    @staticmethod
    def from_strings(registry: DynamicsRegistry, names) -> "DispatchSet":
        return DispatchSet(registry.tag_for(n) for n in names)

    def contains(self, tag: int) -> bool:
        return tag in self.tags


def partition(n: int, k: int):
    """Balanced split: the first n % k parts are one cell longer (multiblock.cpp:24-31).
    Returns [(origin, extent), ...]."""
    if k < 1 or k > n:
        raise ValueError("partition: block grid must be between 1 and the extent")
    out, at = [], 0
    for b in range(k):
        ln = n // k + (1 if b < n % k else 0)
        out.append((at, ln))
        at += ln
    return out


def halo_neighbours(rank: int, world: int, periodic_z: bool):
    """(lower, upper) neighbour ranks of a z-slab (None at a non-periodic end).
    The plan of the reference's z sweep (multiblock.cpp:51-101) restricted to
    one block per rank along z."""
    lower = rank - 1 if rank > 0 else (world - 1 if periodic_z and world > 1 else None)
    upper = rank + 1 if rank < world - 1 else (0 if periodic_z and world > 1 else None)
    return lower, upper


def exchange_blobs(blob: bytes):
    """All-gather one opaque byte blob per rank over torch.distributed (the
    transport for CUDA IPC handles; the data path itself is peer memory)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, blob)
    return out


class _Lattice:
    """One z-slab handle."""

    def __init__(self, desc: _capi.LatticeDesc, registry: DynamicsRegistry):
        h = C.c_void_p()
        check(_capi.lib().dlb_lattice_create(C.byref(desc), registry.handle, C.byref(h)))
        self._h = h
        self.desc = desc
        self.registry = registry  # keep alive

    def __del__(self):
        if getattr(self, "_h", None) and _capi._lib is not None:
            _capi._lib.dlb_lattice_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def ncells(self):
        d = self.desc.dims
        return int(d[0] * d[1] * d[2])


class DeviceRun:
    """Device twin of MultiBlockRun<T> for a z-slab decomposition.

    ``slabs`` z-slabs are created in this process (on ``devices``, default all
    on device 0) and linked through peer memory; ``dist=(rank, world)`` instead
    creates only this rank's slab and links it to its neighbours' slabs in
    other processes via CUDA IPC handles exchanged over torch.distributed.
    """

    def __init__(self, dims, periodic, registry: DynamicsRegistry, dispatch: DispatchSet | None = None,
                 q: int = 19, precision: int = 64, slabs: int = 1, devices=None, arith: str = "exact",
                 dist=None, layout: str = "twopop", skip_nodynamics: bool = False, tma: bool = False,
                 sparse_lists: bool = False):
        self.dims = tuple(int(v) for v in dims)
        self.periodic = tuple(int(bool(p)) for p in periodic)
        self.registry = registry
        self.q, self.precision = q, precision
        self.dist = dist
        world = dist[1] if dist else slabs
        parts = partition(self.dims[2], world)
        self.parts = parts
        mine = [dist[0]] if dist else list(range(world))
        if devices is None:
            devices = [0] * len(mine)
        self.slabs = []
        for k, r in enumerate(mine):
            d = _capi.LatticeDesc()
            d.dims[0], d.dims[1], d.dims[2] = self.dims[0], self.dims[1], parts[r][1]
            for a in range(3):
                d.periodic[a] = self.periodic[a]
            d.q, d.precision_bits = q, precision
            d.layout = _capi.LAYOUT_AA if layout == "aa" else LAYOUT_TWO_POP
            d.arith = ARITH_FAST if arith == "fast" else ARITH_EXACT
            d.device = devices[k]
            d.z_origin, d.global_nz = parts[r][0], self.dims[2]
            d.flags = ((_capi.FLAG_SKIP_NODYNAMICS if skip_nodynamics else 0) | (_capi.FLAG_TMA if tma else 0)
                       | (_capi.FLAG_SPARSE_LISTS if sparse_lists else 0))
            self.slabs.append(_Lattice(d, registry))
        self.ranks = mine
        if dist is None and world > 1:
            for r in range(world - 1):
                check(_capi.lib().dlb_lattice_link_local(self.slabs[r].handle, self.slabs[r + 1].handle))
            if self.periodic[2]:
                check(_capi.lib().dlb_lattice_link_local(self.slabs[world - 1].handle, self.slabs[0].handle))
        elif dist is not None and world > 1:
            self._link_distributed()
        self.set_dispatch(dispatch if dispatch is not None else DispatchSet.all_of(registry))

    # -- distributed linking over torch.distributed (plumbing only) --------------
    def _link_distributed(self):
        rank, world = self.dist
        lat = self.slabs[0]
        n = C.c_size_t()
        check(_capi.lib().dlb_lattice_export_ipc(lat.handle, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        check(_capi.lib().dlb_lattice_export_ipc(lat.handle, buf, n.value, C.byref(n)))
        blobs = exchange_blobs(bytes(buf))
        for side, nb in enumerate(halo_neighbours(rank, world, bool(self.periodic[2]))):
            if nb is None:
                continue
            b = blobs[nb]
            cb = (C.c_uint8 * len(b)).from_buffer_copy(b)
            check(_capi.lib().dlb_lattice_link_ipc(lat.handle, side, cb, len(b)))
        import torch.distributed as dist
        dist.barrier()

    # -- setup ------------------------------------------------------------------
    def set_dispatch(self, dispatch: DispatchSet):
        self.dispatch = dispatch
        tags = np.asarray(sorted(dispatch.tags), np.int32)
        for s in self.slabs:
            check(_capi.lib().dlb_lattice_set_dispatch(s.handle, tags.ctypes.data if tags.size else None, tags.size))

    def _slab_range(self, k):
        r = self.ranks[k]
        return self.parts[r]

    def fill_slots(self, slots: np.ndarray | int):
        """slots: (nz, ny, nx) registry slots over the GLOBAL domain, or one slot for all."""
        for k, s in enumerate(self.slabs):
            if np.isscalar(slots):
                check(_capi.lib().dlb_lattice_set_uniform_slot(s.handle, int(slots)))
                continue
            z0, nz = self._slab_range(k)
            part = np.ascontiguousarray(np.asarray(slots, np.int32)[z0:z0 + nz])
            check(_capi.lib().dlb_lattice_set_slots(s.handle, part.ctypes.data))

    def fill_state(self, rho=None, ux=None, uy=None, uz=None):
        """Equilibrium from per-cell (rho, u) over the global domain; default rest."""
        for k, s in enumerate(self.slabs):
            z0, nz = self._slab_range(k)
            n = self.dims[0] * self.dims[1] * nz
            sl = slice(z0 * self.dims[0] * self.dims[1], (z0 + nz) * self.dims[0] * self.dims[1])

            def part(a, default):
                if a is None:
                    return np.full(n, default, np.float64)
                return np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1)[sl])
            arrs = [part(rho, 1.0), part(ux, 0.0), part(uy, 0.0), part(uz, 0.0)]
            check(_capi.lib().dlb_lattice_fill_equilibrium(s.handle, *[a.ctypes.data for a in arrs]))

    def fill_tgv(self, L: int, u_inf: float):
        for s in self.slabs:
            check(_capi.lib().dlb_lattice_fill_tgv(s.handle, L, u_inf))

    def fill(self, slot_of, state):
        """MultiBlockRun::fill analogue: slot_of array/scalar, state = ('tgv', L, u) | ('rest',) |
        (rho, ux, uy, uz) arrays."""
        self.fill_slots(slot_of)
        tag = state[0] if isinstance(state, tuple) and state and isinstance(state[0], str) else None
        if tag == "tgv":
            self.fill_tgv(state[1], state[2])
        elif tag == "rest":
            self.fill_state()
        else:
            self.fill_state(*state)
        self.exchange()

    def exchange(self):
        """Envelope (halo) exchange only, valid before the first step
        (MultiBlockRun::exchange, multiblock.hpp:142-143). Called after every
        state fill / upload of a decomposed run."""
        if len(self.slabs) == 1 and self.dist is None:
            return
        if len(self.slabs) > 1:
            arr = (C.c_void_p * len(self.slabs))(*[s.handle.value for s in self.slabs])
            check(_capi.lib().dlb_lattices_exchange(arr, len(self.slabs)))
        else:
            check(_capi.lib().dlb_lattice_exchange(self.slabs[0].handle))
        if self.dist is not None and self.dist[1] > 1:
            import torch.distributed as dist
            dist.barrier()

    def upload_populations(self, canon: np.ndarray):
        canon = np.asarray(canon, np.float64).reshape(self.q, -1)
        nxy = self.dims[0] * self.dims[1]
        for k, s in enumerate(self.slabs):
            z0, nz = self._slab_range(k)
            part = np.ascontiguousarray(canon[:, z0 * nxy:(z0 + nz) * nxy])
            check(_capi.lib().dlb_lattice_upload_populations(s.handle, part.ctypes.data))
        self.exchange()

    # -- stepping ---------------------------------------------------------------
    def advance(self, nsteps: int):
        if len(self.slabs) == 1:
            check(_capi.lib().dlb_lattice_step(self.slabs[0].handle, nsteps))
        else:
            arr = (C.c_void_p * len(self.slabs))(*[s.handle.value for s in self.slabs])
            check(_capi.lib().dlb_lattices_step(arr, len(self.slabs), nsteps))

    def set_halo_timeout(self, seconds: float, k: int | None = None):
        """Halo wait limit of slab k (all slabs if None); a neighbour that stays
        silent longer fails the step with ExchangeError (state kept at the last
        completed step)."""
        for j, s in enumerate(self.slabs):
            if k is None or j == k:
                check(_capi.lib().dlb_lattice_set_halo_timeout(s.handle, float(seconds)))

    def links(self, k: int = 0) -> dict:
        """Link state of slab k: lower / upper = 'none' | 'same_gpu' | 'peer_gpu',
        and the halo bytes it pushes per step."""
        lo, up, hb = C.c_int32(), C.c_int32(), C.c_int64()
        check(_capi.lib().dlb_lattice_links(self.slabs[k].handle, C.byref(lo), C.byref(up), C.byref(hb)))
        name = {0: "none", 1: "same_gpu", 2: "peer_gpu"}
        return {"lower": name[lo.value], "upper": name[up.value], "halo_bytes_per_step": hb.value}

    def step_slab(self, k: int, nsteps: int):
        """Advance slab k alone (its neighbours must keep up; fault tests)."""
        check(_capi.lib().dlb_lattice_step(self.slabs[k].handle, nsteps))

    def synchronize(self):
        for s in self.slabs:
            check(_capi.lib().dlb_lattice_synchronize(s.handle))

    def time_steps(self, nsteps: int) -> float:
        """CUDA-event milliseconds for nsteps on the (single) slab's stream."""
        ms = C.c_double()
        check(_capi.lib().dlb_lattice_time_steps(self.slabs[0].handle, nsteps, C.byref(ms)))
        return ms.value

    def stream_handle(self, k: int = 0) -> int:
        p = C.c_void_p()
        check(_capi.lib().dlb_lattice_stream(self.slabs[k].handle, C.byref(p)))
        return p.value or 0

    def kernel_name(self, k: int = 0) -> str:
        return _capi.get_string(_capi.lib().dlb_lattice_kernel_name, self.slabs[k].handle)

    def traffic(self, k: int = 0):
        b, d, l = C.c_int64(), C.c_int64(), C.c_int32()
        check(_capi.lib().dlb_lattice_traffic(self.slabs[k].handle, C.byref(b), C.byref(d), C.byref(l)))
        return b.value, d.value, l.value

    def checksum(self, active_only: bool = False) -> list:
        """Per-direction exact checksums of this process's cells (sum of slab
        checksums mod 2^64; equal to the reference's for identical states).
        active_only: only the cells whose chain is not NoDynamics."""
        tot = np.zeros(self.q, np.uint64)
        fn = _capi.lib().dlb_lattice_checksum_active if active_only else _capi.lib().dlb_lattice_checksum
        for s in self.slabs:
            buf = np.zeros(self.q, np.uint64)
            check(fn(s.handle, buf.ctypes.data))
            tot = tot + buf  # uint64 wraps
        return [int(v) for v in tot]

    def step_bytes(self) -> int:
        """Algorithmic HBM bytes per step summed over this process's slabs."""
        tot = 0
        for s in self.slabs:
            b = C.c_int64()
            check(_capi.lib().dlb_lattice_step_bytes(s.handle, C.byref(b)))
            tot += b.value
        return tot

    def num_cells(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    # -- gathers ----------------------------------------------------------------
    def gather_populations(self) -> np.ndarray:
        """Canonical order (direction-major, x fastest) over the cells this process owns."""
        nxy = self.dims[0] * self.dims[1]
        z_lo = self._slab_range(0)[0]
        z_hi = sum(self._slab_range(len(self.slabs) - 1))
        out = np.zeros((self.q, (z_hi - z_lo) * nxy), np.float64)
        for k, s in enumerate(self.slabs):
            z0, nz = self._slab_range(k)
            buf = np.zeros(self.q * nz * nxy, np.float64)
            check(_capi.lib().dlb_lattice_download_populations(s.handle, buf.ctypes.data))
            out[:, (z0 - z_lo) * nxy:(z0 - z_lo + nz) * nxy] = buf.reshape(self.q, -1)
        return out.reshape(-1)

    def gather_macroscopic(self):
        """rho, ux, uy, uz over this process's cells (multiblock.cpp:443-484)."""
        nxy = self.dims[0] * self.dims[1]
        outs = []
        for k, s in enumerate(self.slabs):
            _, nz = self._slab_range(k)
            arrs = [np.zeros(nz * nxy) for _ in range(4)]
            check(_capi.lib().dlb_lattice_gather_macroscopic(s.handle, *[a.ctypes.data for a in arrs]))
            outs.append(arrs)
        return tuple(np.concatenate([o[j] for o in outs]) for j in range(4))

    def write_field_dump(self, path: str):
        """DOLB1 field dump of the whole (single-process) domain in the storage
        precision: magic, u8 precision, u32 q, 3 x u64 dims, then the q SoA
        arrays x fastest (accelerated_lattice.cpp:313-341)."""
        import struct
        raw = self.gather_raw()
        with open(path, "wb") as fh:
            fh.write(b"DOLB1")
            fh.write(struct.pack("<BI3Q", self.precision // 8, self.q, *self.dims))
            fh.write(raw.tobytes())

    # -- GPU-resident diagnostics (runner.cpp:346-448, diagnostics.cpp:10-131) --
    def _all_gather(self, obj):
        if self.dist is None or self.dist[1] == 1:
            return [obj]
        import torch.distributed as dist
        out = [None] * self.dist[1]
        dist.all_gather_object(out, obj)
        return out

    def _args(self, quantity, x_range=None, halos=(None, None)):
        a = _capi.ReduceArgs()
        a.quantity = quantity
        for ax in range(3):
            a.periodic[ax] = self.periodic[ax]
        a.x_begin, a.x_end = x_range if x_range is not None else (0, self.dims[0])
        a.halo_below = halos[0].ctypes.data if halos[0] is not None else None
        a.halo_above = halos[1].ctypes.data if halos[1] is not None else None
        return a

    def velocity_planes(self, z0: int, nz: int, k: int = 0) -> np.ndarray:
        """(nz, 3, ny, nx) velocity of local planes [z0, z0 + nz) of slab k."""
        out = np.zeros((nz, 3, self.dims[1], self.dims[0]))
        check(_capi.lib().dlb_lattice_velocity_planes(self.slabs[k].handle, z0, nz, out.ctypes.data))
        return out

    def _enstrophy_halos(self):
        """Per local slab: the 4 global velocity planes below and above it
        (the FD8 stencil's reach), gathered from the slabs that own them."""
        nz_g = self.dims[2]
        if len(self.parts) == 1:
            return [(None, None)]
        # every slab publishes its (up to) 4 bottom and 4 top planes
        mine = {}
        for k in range(len(self.slabs)):
            z0, nz = self._slab_range(k)
            want = sorted(set(list(range(min(4, nz))) + list(range(max(0, nz - 4), nz))))
            planes = self.velocity_planes(want[0], want[-1] - want[0] + 1, k) if want else None
            for j in want:
                mine[z0 + j] = planes[j - want[0]]
        have = {}
        for d in self._all_gather(mine):
            have.update(d)
        zero = np.zeros((3, self.dims[1], self.dims[0]))
        out = []
        for k in range(len(self.slabs)):
            z0, nz = self._slab_range(k)

            def block(zs):
                rows = []
                for zg in zs:
                    if not self.periodic[2] and not 0 <= zg < nz_g:
                        rows.append(zero)
                        continue
                    rows.append(have[zg % nz_g])
                return np.ascontiguousarray(np.stack(rows))
            out.append((block(range(z0 - 4, z0)), block(range(z0 + nz, z0 + nz + 4))))
        return out

    def tree_reduce(self, quantity: int, x_range=None):
        """(tree_sum, count) of a quantity's value sequence over the whole
        (possibly decomposed) domain, bit-identical to diag::tree_sum over the
        vector the reference's runner builds."""
        halos = self._enstrophy_halos() if quantity == _capi.Q_ENSTROPHY else [(None, None)] * len(self.slabs)
        args = [self._args(quantity, x_range, halos[k]) for k in range(len(self.slabs))]
        counts = []
        for k, s in enumerate(self.slabs):
            c = C.c_int64()
            check(_capi.lib().dlb_lattice_reduce_count(s.handle, C.byref(args[k]), C.byref(c)))
            counts.append((self.ranks[k], c.value))
        allc = sorted(c for part in self._all_gather(counts) for c in part)
        n_total = sum(c for _, c in allc)
        begin = {}
        acc = 0
        for r, c in allc:
            begin[r] = acc
            acc += c
        parts = []
        for k, s in enumerate(self.slabs):
            n = C.c_size_t()
            check(_capi.lib().dlb_lattice_reduce_parts(s.handle, C.byref(args[k]), n_total, begin[self.ranks[k]],
                                                       None, 0, C.byref(n)))
            buf = (_capi.TreePart * max(n.value, 1))()
            check(_capi.lib().dlb_lattice_reduce_parts(s.handle, C.byref(args[k]), n_total, begin[self.ranks[k]],
                                                       buf, n.value, C.byref(n)))
            parts.extend((p.lo, p.len, p.value) for p in buf[:n.value])
        allp = [p for part in self._all_gather(parts) for p in part]
        arr = (_capi.TreePart * max(len(allp), 1))(*[_capi.TreePart(*p) for p in allp])
        out = C.c_double()
        check(_capi.lib().dlb_tree_combine(n_total, arr, len(allp), C.byref(out)))
        return out.value, n_total

    def _tree_mean(self, quantity, x_range=None, empty=None):
        s, n = self.tree_reduce(quantity, x_range)
        if n == 0:
            if empty is None:
                raise ValueError("mean of an empty set")  # diagnostics.cpp:21
            return empty
        return s / float(n)

    def kinetic_energy(self) -> float:
        """diag::kinetic_energy of the gathered velocity (diagnostics.cpp:25-31)."""
        return self._tree_mean(_capi.Q_KINETIC)

    def enstrophy(self) -> float:
        """diag::enstrophy(diag::vorticity_fd8(u, periodic)) (diagnostics.cpp:65-120)."""
        return self._tree_mean(_capi.Q_ENSTROPHY)

    def request_kinetic(self) -> bool:
        """Fuse the next kinetic-energy reduction into the last step of the next
        advance() (dlb_lattice_request_kinetic); False when unfused."""
        fused = True
        for s in self.slabs:
            f = C.c_int32()
            check(_capi.lib().dlb_lattice_request_kinetic(s.handle, C.byref(f)))
            fused = fused and bool(f.value)
        return fused

    def snapshot_velocity(self):
        """Keep the current velocity on the device (the runner's prev_u, runner.cpp:445-448)."""
        for s in self.slabs:
            check(_capi.lib().dlb_lattice_snapshot_velocity(s.handle))

    def convergence_sums(self):
        """(tree_sum |u - u_prev|^2, tree_sum |u|^2) against the last snapshot (runner.cpp:433-444)."""
        return self.tree_reduce(_capi.Q_DU_NUM)[0], self.tree_reduce(_capi.Q_DU_DEN)[0]

    def porous_extras(self, sample_begin: int, sample_end: int, nu: float, aperture_mean: bool = False):
        """Driver::porous_extras (runner.cpp:346-399): [k_perm, ubar, dp, ux_in, ux_out]."""
        x0, x1 = sample_begin, sample_end - 1

        def plane_mean_p(x):
            return self._tree_mean(_capi.Q_PRESSURE_FLUID, (x, x + 1), empty=0.0)

        def plane_mean_ux(x):
            return self._tree_mean(_capi.Q_UX_FLUID, (x, x + 1), empty=0.0)
        win = (sample_begin, sample_end)
        ubar = self._tree_mean(_capi.Q_UX_FLUID if aperture_mean else _capi.Q_UX_ALL, win)
        rho_bar = self._tree_mean(_capi.Q_RHO_FLUID, win, empty=1.0)
        dp = (plane_mean_p(x0) - plane_mean_p(x1)) / rho_bar
        lx = float(x1 - x0)
        if abs(dp) < 1e-300:
            k_perm = 0.0
        else:
            k_perm = ubar * nu * lx / dp  # diag::permeability (diagnostics.cpp:122-127)
        return [k_perm, ubar, dp, plane_mean_ux(1), plane_mean_ux(self.dims[0] - 2)]

    def gather_raw(self) -> np.ndarray:
        """Like gather_populations but in the storage precision."""
        dt = np.float64 if self.precision == 64 else np.float32
        nxy = self.dims[0] * self.dims[1]
        parts = []
        for k, s in enumerate(self.slabs):
            _, nz = self._slab_range(k)
            buf = np.zeros(self.q * nz * nxy, dt)
            check(_capi.lib().dlb_lattice_download_raw(s.handle, buf.ctypes.data))
            parts.append(buf.reshape(self.q, -1))
        return np.concatenate(parts, axis=1).reshape(-1)


def collide_and_stream(registry: DynamicsRegistry, f_in: np.ndarray, tag: np.ndarray,
                       param_index: np.ndarray, dispatch: DispatchSet, f_out: np.ndarray | None = None,
                       q: int = 19):
    """Drop-in for collide_and_stream<T>(AcceleratedBlock<T>&, ...) on host arrays
    (accelerated_lattice.hpp:124-127). f_in: (q, ez, ey, ex) envelope-inclusive,
    tag / param_index: (ez, ey, ex). Without f_out the new state overwrites
    f_in's interior and f_in is returned. With f_out the new state is written
    into f_out (f_in keeps the previous state) and (f_out, f_in) is returned:
    the reference's swap -- the first is the block's new f_in."""
    assert f_in.flags.c_contiguous and f_in.ndim == 4
    ez, ey, ex = f_in.shape[1:]
    v = _capi.BlockView()
    v.precision_bits = 64 if f_in.dtype == np.float64 else 32
    v.q = q
    v.interior[0], v.interior[1], v.interior[2] = ex - 2, ey - 2, ez - 2
    v.f_in = f_in.ctypes.data
    v.f_out = f_out.ctypes.data if f_out is not None else None
    tag = np.ascontiguousarray(tag, np.int32)
    pidx = np.ascontiguousarray(param_index, np.int32)
    v.tag, v.param_index = tag.ctypes.data, pidx.ctypes.data
    tags = np.asarray(sorted(dispatch.tags), np.int32)
    check(_capi.lib().dlb_collide_and_stream(registry.handle, C.byref(v),
                                             tags.ctypes.data if tags.size else None, tags.size, 1))
    if f_out is None:
        return f_in
    assert v.f_in == f_out.ctypes.data  # the view came back swapped
    return f_out, f_in


def block_cache_release():
    """Free the device contexts dlb_collide_and_stream keeps per block shape."""
    _capi.lib().dlb_block_cache_release()


def block_cache_info():
    """(entries, device bytes) held by the host-block device cache."""
    n, b = C.c_size_t(), C.c_int64()
    check(_capi.lib().dlb_block_cache_info(C.byref(n), C.byref(b)))
    return n.value, b.value


def read_field_dump(path: str):
    """read_field_dump (accelerated_lattice.cpp:343-374): (dims, precision_bytes,
    q x N doubles)."""
    import struct
    with open(path, "rb") as fh:
        if fh.read(5) != b"DOLB1":
            raise OSError(f'"{path}" is not a DOLB1 field dump')
        prec, q, nx, ny, nz = struct.unpack("<BI3Q", fh.read(29))
        if prec not in (4, 8):
            raise OSError(f'unsupported field dump header in "{path}"')
        dt = np.float64 if prec == 8 else np.float32
        n = q * nx * ny * nz
        data = np.frombuffer(fh.read(n * prec), dtype=dt)
        if data.size != n:
            raise OSError(f'truncated field dump "{path}"')
    return (nx, ny, nz), prec, data.astype(np.float64)


def refresh_envelope_periodic(f_in: np.ndarray, periodic=(1, 1, 1), q: int = 19):
    """refresh_envelope_periodic<T> (accelerated_lattice.cpp:202-238) on a host
    block (q, ez, ey, ex), done by the C++ runtime with one thread per direction."""
    assert f_in.flags.c_contiguous and f_in.ndim == 4
    ez, ey, ex = f_in.shape[1:]
    v = _capi.BlockView()
    v.precision_bits = 64 if f_in.dtype == np.float64 else 32
    v.q = q
    v.interior[0], v.interior[1], v.interior[2] = ex - 2, ey - 2, ez - 2
    v.f_in = f_in.ctypes.data
    per = np.asarray(periodic, np.int32)
    check(_capi.lib().dlb_refresh_envelope_periodic(C.byref(v), per.ctypes.data))


def _descriptor(q):
    if q == 19:
        c = [(0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1),
             (-1, -1, 0), (1, 1, 0), (-1, 1, 0), (1, -1, 0), (-1, 0, -1), (1, 0, 1), (-1, 0, 1),
             (1, 0, -1), (0, -1, -1), (0, 1, 1), (0, -1, 1), (0, 1, -1)]
        w = [1 / 3] + [1 / 18] * 6 + [1 / 36] * 12
    else:
        c = _descriptor(19)[0].tolist() + [(-1, -1, -1), (1, 1, 1), (-1, -1, 1), (1, 1, -1),
                                           (-1, 1, -1), (1, -1, 1), (1, -1, -1), (-1, 1, 1)]
        w = [8 / 27] + [2 / 27] * 6 + [1 / 54] * 12 + [1 / 216] * 8
    return np.asarray(c, np.int64), np.asarray(w)


D3Q19 = _descriptor(19)
D3Q27 = _descriptor(27)
