// Fused collide-and-stream kernels for sm_100a.
//
// Replaces the reference hot path collide_and_stream<T> -> step_range<T> ->
// ChainRecipe<T>::apply (proj/src/accelerated_lattice.cpp:126-200,
// proj/include/dolb/chain.hpp:104-144): one thread per cell pulls its q
// populations from the neighbours' post-collision state (two-population
// scheme, f_in -> f_out), applies the cell's dynamics from the per-slot recipe
// table, and stores q values. Periodic axes wrap in-kernel; non-periodic axes
// read the zero envelope (reference_lattice.cpp:240-254) or, for a z-slab of a
// decomposed domain, the ghost plane filled by the neighbour's halo push.
//
// This translation unit is compiled twice: DLB_MODE = exact with -fmad=false
// (bit-identical to the reference CPU solver) and DLB_MODE = fast with FMA
// contraction.
#include <cooperative_groups.h>

#include <algorithm>

#include "kernels.cuh"

#ifndef DLB_MODE
#error "define DLB_MODE (exact or fast)"
#endif

namespace dlb {
namespace DLB_MODE {

// Occupancy target per instantiation (register cap = 65536 / (256 * blocks)):
// lean dispatch sets (BGK / TRT / walls): fp32 6 blocks (<= 42 regs), D3Q19
// fp64 3 (<= 85); sets with RR, LES or regularized links, and D3Q27 fp64, get 2
// (fp32 3) so their larger live state does not spill.
// The pure-BGK fp32 set gets 5 (<= 48 regs): at 6 it spilled 8 B per thread
// and c5 ran 2 % slower (26.95 vs 26.41 ms per 1024^3 step,
// profiles/r02_summary.md); the wall sets stay at 6 (c3: 3.34 vs 3.43 ms).
template <typename T, int Q, unsigned KM>
constexpr int min_blocks() {
    constexpr bool heavy = (KM & (KM_RR | KM_LES | KM_REGV | KM_REGP)) != 0;
    if (sizeof(T) == 4 && Q == 19 && (KM & ~(KM_KE | KM_SKIP | KM_XREC)) == KM_BGK) return 5;
    if (sizeof(T) == 4) return (heavy || Q == 27) ? 3 : 6;
    if (Q == 27) return 2;
    return heavy ? 2 : 3;
}

// Completion signal of a boundary launch: publish this block's peer stores at
// system scope, take a ticket; the last block bumps the slab's step counter and
// release-stores it into both neighbours' flags (read by their k_halo_wait).
template <typename T>
__device__ __forceinline__ void signal_step(const StepArgs<T>& a) {
    // One system-scope fence per block, by the thread that takes the ticket
    // after the barrier: fences are cumulative, so it orders every thread's
    // peer stores that the barrier ordered before it (the pattern of
    // cooperative groups' grid sync, at system scope). A fence in every thread
    // kept each boundary block resident for its own fence latency.
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        __threadfence_system();
        const unsigned total = gridDim.x * gridDim.y * gridDim.z;
        const unsigned ticket = atomicAdd(a.counter, 1u);
        if (ticket == total - 1) {
            __threadfence_system();
            *a.counter = 0u;
            const unsigned long long s = *a.my_step + 1ull;
            *a.my_step = s;
            if (a.sig_up != nullptr)
                asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.sig_up), "l"(s) : "memory");
            if (a.sig_down != nullptr)
                asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.sig_down), "l"(s) : "memory");
        }
    }
}

// One cell of the two-population pull step: gather f_i(x) <- f_i(x - c_i)
// from the input buffer (periodic axes wrap in-kernel, non-periodic faces
// read the zero envelope / ghost planes), apply the slot's dynamics, store to
// the output buffer, and push the z-crossing links into the neighbours' ghost
// planes when the slab is linked. READ_SLOT: look the slot up here (after the
// loads, so the slot read overlaps them); otherwise `s` is already known.
template <typename T, int Q>
__device__ __forceinline__ void pull_cell(const StepArgs<T>& a, int x, int y, int z, T (&f)[Q]) {
    using L = Lat<Q>;
    const Geo& g = a.g;
    const int xm = (x == 0 && g.per_x) ? g.nx - 1 : x - 1;
    const int xp = (x == g.nx - 1 && g.per_x) ? 0 : x + 1;
    const int ym = (y == 0 && g.per_y) ? g.ny - 1 : y - 1;
    const int yp = (y == g.ny - 1 && g.per_y) ? 0 : y + 1;
    const int zm = (z == 0 && g.per_z) ? g.nz - 1 : z - 1;
    const int zp = (z == g.nz - 1 && g.per_z) ? 0 : z + 1;
    sfor<Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
        const int sx = cx > 0 ? xm : (cx < 0 ? xp : x);
        const int sy = cy > 0 ? ym : (cy < 0 ? yp : y);
        const int sz = cz > 0 ? zm : (cz < 0 ? zp : z);
        f[i] = __ldg(a.fin[i] + (sz * g.plane + sy * g.pitch + sx));
    });
}

template <typename T, int Q, unsigned KM>
__device__ __forceinline__ void collide_store_cell(const StepArgs<T>& a, int x, int y, int z, int s, T (&f)[Q]) {
    using L = Lat<Q>;
    const Geo& g = a.g;
    Cell<T, Q>::template apply<KM>(f, recipe_of<KM>(a, s));

    const int center = z * g.plane + y * g.pitch + x;
    sfor<Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        a.fout[i][center] = f[i];
    });

    if (a.push_up != nullptr && z == g.nz - 1) {
        const int ghost = -g.plane + y * g.pitch + x;
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            if constexpr (L::c[i][2] > 0) a.push_up[i * a.up_dstride + ghost] = f[i];
        });
    }
    if (a.push_down != nullptr && z == 0) {
        const int ghost = a.down_ghost_z * g.plane + y * g.pitch + x;
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            if constexpr (L::c[i][2] < 0) a.push_down[i * a.down_dstride + ghost] = f[i];
        });
    }
}

template <typename T, int Q, unsigned KM, bool READ_SLOT>
__device__ __forceinline__ void cell_update(const StepArgs<T>& a, int x, int y, int z, int s) {
    T f[Q];
    pull_cell<T, Q>(a, x, y, z, f);
    if constexpr (READ_SLOT) {
        if (a.slot != nullptr) s = a.slot[(static_cast<long long>(z) * a.g.ny + y) * a.g.nx + x];
    }
    collide_store_cell<T, Q, KM>(a, x, y, z, s, f);
}

// MINB != 0 overrides the occupancy target (register cap) of an instantiation
// (tuning entries, DLB_PULL_MINB).
template <typename T, int Q, unsigned KM, int MINB = 0>
__global__ void __launch_bounds__(256, (MINB ? MINB : min_blocks<T, Q, KM>()))
    k_pull(const __grid_constant__ StepArgs<T> a) {
    using L = Lat<Q>;
    const Geo& g = a.g;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int z = a.z_begin + int(blockIdx.z) * a.z_step;
    // (L1-cached load: the flag only changes between launches of this slab's
    // later steps; the interior launch of the failing step may read either value)
    if (a.err != nullptr && __ldca(a.err) != 0ull) return;
    bool active = x < g.nx && y < g.ny;
    int s = a.uniform_slot;
    if constexpr ((KM & KM_SKIP) != 0) {
        // masked porous variant: NoDynamics cells (solids without a fluid
        // neighbour, cases.cpp:239-249) are neither loaded nor stored; their
        // values are never consumed by a fluid cell. The skip
        // works on x-aligned groups of a.skip_group cells (one memory segment
        // of every direction array): a group moves nothing only when all its
        // cells are NoDynamics, otherwise its NoDynamics cells run their dense
        // (reference) update, so every store covers whole segments and no
        // partial-segment writes reach HBM. blockDim.x is a multiple of 32
        // and rows start 128-B aligned, so warp lanes are x-consecutive and
        // groups are segment-aligned.
        bool need = false;
        if (active && a.slot != nullptr) {
            s = a.slot[(static_cast<long long>(z) * g.ny + y) * g.nx + x];
            need = recipe_of<KM>(a, s).kind != KIND_NODYN;
        }
        const unsigned ball = __ballot_sync(0xffffffffu, need);
        const int G = a.skip_group;
        const unsigned lane = threadIdx.x & 31u;
        const unsigned gmask = G >= 32 ? 0xffffffffu : ((1u << G) - 1u);
        active = active && ((ball >> (lane & ~unsigned(G - 1))) & gmask) != 0u;
    }
    // (body kept inline rather than through cell_update: the inlined helper
    // changes the instruction schedule and costs 13 % on c3, profiles/r01_summary.md)
    if (active) {
        // Source coordinates of the pull f_i(x) <- f_i(x - c_i).
        const int xm = (x == 0 && g.per_x) ? g.nx - 1 : x - 1;
        const int xp = (x == g.nx - 1 && g.per_x) ? 0 : x + 1;
        const int ym = (y == 0 && g.per_y) ? g.ny - 1 : y - 1;
        const int yp = (y == g.ny - 1 && g.per_y) ? 0 : y + 1;
        const int zm = (z == 0 && g.per_z) ? g.nz - 1 : z - 1;
        const int zp = (z == g.nz - 1 && g.per_z) ? 0 : z + 1;

        T f[Q];
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
            const int sx = cx > 0 ? xm : (cx < 0 ? xp : x);
            const int sy = cy > 0 ? ym : (cy < 0 ? yp : y);
            const int sz = cz > 0 ? zm : (cz < 0 ? zp : z);
            f[i] = __ldg(a.fin[i] + (sz * g.plane + sy * g.pitch + sx));
        });

        if constexpr ((KM & KM_SKIP) == 0) {
            if (a.slot != nullptr) s = a.slot[(static_cast<long long>(z) * g.ny + y) * g.nx + x];
        }
        Cell<T, Q>::template apply<KM & ~(KM_SKIP | KM_KE)>(f, recipe_of<KM>(a, s));

        const int center = z * g.plane + y * g.pitch + x;
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            a.fout[i][center] = f[i];
        });
        if constexpr ((KM & KM_KE) != 0) {
            // Fused reduce input (the paper's transform_reduce): the
            // kinetic energy of the state just stored, with gather_macroscopic's
            // semantics (multiblock.cpp:458-478: rho / u in double from the
            // stored T values; wall velocity on moving walls; 0 elsewhere) and
            // diag::kinetic_energy's expression (diagnostics.cpp:28).
            const DevRecipe<T>& r = recipe_of<KM>(a, s);
            double u[3] = {0.0, 0.0, 0.0};
            if (r.kind == KIND_COLLIDE) {
                double fd[Q];
                sfor<Q>([&](auto I) {
                    constexpr int i = decltype(I)::value;
                    fd[i] = double(f[i]);
                });
                double rho;
                Cell<double, Q>::rho_u(fd, rho, u);
            } else if (r.kind == KIND_MBB) {
                u[0] = double(r.wall_velocity[0]);
                u[1] = double(r.wall_velocity[1]);
                u[2] = double(r.wall_velocity[2]);
            }
            a.ke[(static_cast<long long>(z) * g.ny + y) * g.nx + x] = 0.5 * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
        }

        if (a.push_up != nullptr && z == g.nz - 1) {
            const int ghost = -g.plane + y * g.pitch + x;
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                if constexpr (L::c[i][2] > 0) a.push_up[i * a.up_dstride + ghost] = f[i];
            });
        }
        if (a.push_down != nullptr && z == 0) {
            const int ghost = a.down_ghost_z * g.plane + y * g.pitch + x;
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                if constexpr (L::c[i][2] < 0) a.push_down[i * a.down_dstride + ghost] = f[i];
            });
        }
    }


    if (a.counter != nullptr) signal_step(a);
}


// 128-bit vectorised dense sweep (opt-in, DLB_VEC=1; BASELINE north_star:
// "coalesced, vectorised 128-bit HBM loads and stores"). Each thread owns
// VW = 16 / sizeof(T) x-consecutive cells (4 fp32 / 2 fp64): per direction
// one aligned 128-bit load of its own x-range in the source row; the +-1
// x-shifted directions take the missing element from the neighbouring lane
// (warp shuffle) or, at a warp's edge, one scalar load; one aligned 128-bit
// store per direction. Per-cell arithmetic as k_pull (bit-identical). Single
// slabs, nx % VW == 0, plain dispatch sets (no halo push / fused reduce).
template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
    using type = float4;
    static constexpr int n = 4;
};
template <>
struct Vec16<double> {
    using type = double2;
    static constexpr int n = 2;
};

template <typename T, int Q, unsigned KM>
__global__ void __launch_bounds__(256, 2) k_vec(const __grid_constant__ StepArgs<T> a) {
    using L = Lat<Q>;
    using V = typename Vec16<T>::type;
    constexpr int VW = Vec16<T>::n;
    const Geo& g = a.g;
    const unsigned lane = threadIdx.x & 31u;
    const int xv = int(blockIdx.x * blockDim.x + threadIdx.x) * VW;
    const int y = int(blockIdx.y * blockDim.y + threadIdx.y);
    const int z = a.z_begin + int(blockIdx.z) * a.z_step;
    const bool active = xv < g.nx && y < g.ny;
    // inactive lanes of a partial warp still join the shuffles (clamped loads)
    const int x0 = active ? xv : (xv < g.nx ? xv : g.nx - VW);
    const int yc = y < g.ny ? y : g.ny - 1;
    const int ym = (yc == 0 && g.per_y) ? g.ny - 1 : yc - 1;
    const int yp = (yc == g.ny - 1 && g.per_y) ? 0 : yc + 1;
    const int zm = (z == 0 && g.per_z) ? g.nz - 1 : z - 1;
    const int zp = (z == g.nz - 1 && g.per_z) ? 0 : z + 1;
    // the element left of x0 / right of the x-range (warp edges, row ends)
    const int xl = (x0 == 0 && g.per_x) ? g.nx - 1 : x0 - 1;
    const int xr = (x0 + VW == g.nx && g.per_x) ? 0 : x0 + VW;
    const unsigned full = 0xffffffffu;
    // lanes whose neighbour lane does not hold the adjacent x-range
    const bool own_left = lane == 0 || x0 == 0;
    const bool own_right = lane == 31 || x0 + VW >= g.nx;
    T f[VW][Q];
    sfor<Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
        const int sy = cy > 0 ? ym : (cy < 0 ? yp : yc);
        const int sz = cz > 0 ? zm : (cz < 0 ? zp : z);
        const T* row = a.fin[i] + (sz * g.plane + sy * g.pitch);
        const V v = __ldg(reinterpret_cast<const V*>(row + x0));
        T e[VW];
        if constexpr (VW == 4) {
            e[0] = v.x; e[1] = v.y; e[2] = v.z; e[3] = v.w;
        } else {
            e[0] = v.x; e[1] = v.y;
        }
        if constexpr (cx == 0) {
#pragma unroll
            for (int c = 0; c < VW; ++c) f[c][i] = e[c];
        } else if constexpr (cx > 0) {  // f_i(x) <- f_i(x - 1)
            T left = __shfl_up_sync(full, e[VW - 1], 1);
            if (own_left) left = __ldg(row + xl);
            f[0][i] = left;
#pragma unroll
            for (int c = 1; c < VW; ++c) f[c][i] = e[c - 1];
        } else {  // f_i(x) <- f_i(x + 1)
            T right = __shfl_down_sync(full, e[0], 1);
            if (own_right) right = __ldg(row + xr);
#pragma unroll
            for (int c = 0; c < VW - 1; ++c) f[c][i] = e[c + 1];
            f[VW - 1][i] = right;
        }
    });
    if (!active) return;
    const long long cell0 = (static_cast<long long>(z) * g.ny + y) * g.nx + x0;
#pragma unroll
    for (int c = 0; c < VW; ++c) {
        const int s = a.slot != nullptr ? a.slot[cell0 + c] : a.uniform_slot;
        Cell<T, Q>::template apply<KM>(f[c], recipe_of<KM>(a, s));
    }
    const int center = z * g.plane + y * g.pitch + x0;
    sfor<Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        V v;
        if constexpr (VW == 4) {
            v.x = f[0][i]; v.y = f[1][i]; v.z = f[2][i]; v.w = f[3][i];
        } else {
            v.x = f[0][i]; v.y = f[1][i];
        }
        *reinterpret_cast<V*>(a.fout[i] + center) = v;
    });
}

// Persistent multi-step sweep for small lattices (cooperative launch): the
// whole grid stays resident for nsteps steps, each thread walks its cells
// (grid stride), then grid-wide barrier and the buffers swap roles. For a
// lattice that is a few waves of one launch (config 1: 64³, 2.3 waves) the
// per-step launch ramp and tail dominate; here they are paid once per call.
// Same per-cell arithmetic as k_pull (bit-identical); single slab only.
template <typename T, int Q, unsigned KM>
__global__ void __launch_bounds__(256, (min_blocks<T, Q, KM>()))
    k_pull_coop(const __grid_constant__ StepArgs<T> a, int nsteps) {
    using L = Lat<Q>;
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const Geo& g = a.g;
    const long long n = static_cast<long long>(g.nx) * g.ny * g.nz;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (int st = 0; st < nsteps; ++st) {
        const T* const* fin = (st & 1) ? const_cast<const T* const*>(a.fout) : a.fin;
        T* const* fout = (st & 1) ? const_cast<T* const*>(a.fin) : a.fout;
        for (long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; c < n; c += stride) {
            const int x = int(c % g.nx);
            const long long r = c / g.nx;
            const int y = int(r % g.ny);
            const int z = int(r / g.ny);
            const int xm = (x == 0 && g.per_x) ? g.nx - 1 : x - 1;
            const int xp = (x == g.nx - 1 && g.per_x) ? 0 : x + 1;
            const int ym = (y == 0 && g.per_y) ? g.ny - 1 : y - 1;
            const int yp = (y == g.ny - 1 && g.per_y) ? 0 : y + 1;
            const int zm = (z == 0 && g.per_z) ? g.nz - 1 : z - 1;
            const int zp = (z == g.nz - 1 && g.per_z) ? 0 : z + 1;
            T f[Q];
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
                const int sx = cx > 0 ? xm : (cx < 0 ? xp : x);
                const int sy = cy > 0 ? ym : (cy < 0 ? yp : y);
                const int sz = cz > 0 ? zm : (cz < 0 ? zp : z);
                f[i] = fin[i][sz * g.plane + sy * g.pitch + sx];
            });
            int s = a.uniform_slot;
            if (a.slot != nullptr) s = a.slot[c];
            Cell<T, Q>::template apply<KM>(f, recipe_of<KM>(a, s));
            const int center = z * g.plane + y * g.pitch + x;
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                fout[i][center] = f[i];
            });
        }
        grid.sync();
    }
}


// Compacted masked sweep for porous media (single slab): the host lists the
// x-aligned segments of a.skip_group cells that hold at least one
// non-NoDynamics cell (the same rule as the KM_SKIP ballot), as linear
// segment indices (z * ny + y) * ceil(nx / G) + x / G in row-major order.
// Consecutive threads take consecutive cells of consecutive listed segments,
// so every warp is fully populated (the masked dense sweep keeps idle lanes in
// the warps that straddle solids, which caps its bytes in flight) while every
// store still covers whole segments. NoDynamics cells of a listed segment run
// their dense update; unlisted segments are never touched.
// CPT cells per thread (cells t and t + 256 of a 256 * CPT-cell block range):
// every thread issues the loads of all its cells before the first collision,
// CPT times the bytes in flight per thread of the latency-bound fp64 sweep.
template <typename T, int Q, unsigned KM, int CPT, int MINB = 0>
__global__ void __launch_bounds__(256, (MINB ? MINB : (CPT == 1 ? min_blocks<T, Q, KM>() : 2)))
    k_seg(const __grid_constant__ StepArgs<T> a, const unsigned* __restrict__ segs, long long nseg, int gshift,
          int pf, int pack) {
    const Geo& g = a.g;
    const unsigned nsx = unsigned((g.nx + (1 << gshift) - 1) >> gshift);
    const long long n = nseg << gshift;
    const int bd = int(blockDim.x);  // 256 (or 128: finer-grained block turnover)
    const long long base = static_cast<long long>(blockIdx.x) * (bd * CPT) + threadIdx.x;
    if (segs && pf > 0 && threadIdx.x < 32) {
        // the segment entries of the block pf launches ahead (about one wave of
        // resident blocks) into L2: its threads' first, dependent load then
        // hits L2 instead of DRAM (the list is streamed once per step)
        const long long e0 = ((static_cast<long long>(blockIdx.x) + pf) * (bd * CPT)) >> gshift;
        const long long e = e0 + threadIdx.x * 32;  // one 128-B line per lane
        const long long e_end = e0 + ((static_cast<long long>(bd) * CPT) >> gshift);
        if (e < e_end && e < nseg) asm volatile("prefetch.global.L2 [%0];" ::"l"(segs + e));
    }
    int xs[CPT], ys[CPT], zs[CPT];
    bool ok[CPT];
    T f[CPT][Q];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        const long long t = base + bd * c;
        ok[c] = t < n;
        xs[c] = ys[c] = zs[c] = 0;
        if (ok[c]) {
            // segs == nullptr: every segment (the dense sweep), no list to chase
            const unsigned e = segs ? __ldg(segs + (t >> gshift)) : unsigned(t >> gshift);
            const int lane = int(t & ((1 << gshift) - 1));
            if (pack != 0 && segs) {
                // packed entry s | y << bs | z << (bs + by): no divisions on the
                // path from the entry load to the population loads
                const int bs = pack & 0xff, by = (pack >> 8) & 0xff;
                xs[c] = int((e & ((1u << bs) - 1u)) << gshift) + lane;
                ys[c] = int((e >> bs) & ((1u << by) - 1u));
                zs[c] = int(e >> (bs + by));
            } else {
                const unsigned row = e / nsx;
                xs[c] = int((e - row * nsx) << gshift) + lane;
                zs[c] = int(row / unsigned(g.ny));
                ys[c] = int(row - unsigned(zs[c]) * unsigned(g.ny));
            }
            ok[c] = xs[c] < g.nx;
        }
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c)
        if (ok[c]) pull_cell<T, Q>(a, xs[c], ys[c], zs[c], f[c]);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        if (!ok[c]) continue;
        const int s = a.slot ? a.slot[(static_cast<long long>(zs[c]) * g.ny + ys[c]) * g.nx + xs[c]] : a.uniform_slot;
        collide_store_cell<T, Q, KM>(a, xs[c], ys[c], zs[c], s, f[c]);
    }
}


// Fluid-segment porous sweep (single slab, after one k_seg step): only the
// listed segments that hold a collision cell move. A bounce-back neighbour's
// post-collision value in direction i is, bit for bit, the puller's own
// population opp(i) of the step before (full-way bounce-back returns it after
// one step in the wall cell: f_i(x_b, t) = f_opp(i)(x_b + c_i, t - 1)), which
// is still in the output buffer (the two-population ping-pong holds state
// t - 2 there) at the cell this thread is about to overwrite. So a collision
// cell whose neighbour x - c_i is bounce-back (bit i of its link mask) loads
// f_out[opp(i)][x] instead of f_in[i][x - c_i]: wall cells outside the listed
// segments need not step at all (they are brought up to date lazily before the
// state is read, k_bb_finalize) and their sectors -- and the solid sectors
// behind them -- are never read. Every other cell of a listed segment runs its
// dense update, so stores still cover whole segments.
template <typename T, int Q, unsigned KM, int CPT>
__global__ void __launch_bounds__(256, (CPT == 1 ? min_blocks<T, Q, KM>() : 2))
    k_segbb(const __grid_constant__ StepArgs<T> a, const unsigned* __restrict__ segs,
            const unsigned* __restrict__ links, long long nseg, int gshift) {
    using L = Lat<Q>;
    const Geo& g = a.g;
    const unsigned nsx = unsigned((g.nx + (1 << gshift) - 1) >> gshift);
    const long long n = nseg << gshift;
    const long long base = static_cast<long long>(blockIdx.x) * (256 * CPT) + threadIdx.x;
    int xs[CPT], ys[CPT], zs[CPT];
    unsigned mk[CPT];
    bool ok[CPT];
    T f[CPT][Q];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        const long long t = base + 256 * c;
        ok[c] = t < n;
        xs[c] = ys[c] = zs[c] = 0;
        mk[c] = 0u;
        if (ok[c]) {
            const unsigned e = __ldg(segs + (t >> gshift));
            mk[c] = __ldg(links + t);
            const unsigned row = e / nsx;
            xs[c] = int((e - row * nsx) << gshift) + int(t & ((1 << gshift) - 1));
            zs[c] = int(row / unsigned(g.ny));
            ys[c] = int(row - unsigned(zs[c]) * unsigned(g.ny));
            ok[c] = xs[c] < g.nx;
        }
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        if (!ok[c]) continue;
        const int x = xs[c], y = ys[c], z = zs[c];
        const int xm = (x == 0 && g.per_x) ? g.nx - 1 : x - 1;
        const int xp = (x == g.nx - 1 && g.per_x) ? 0 : x + 1;
        const int ym = (y == 0 && g.per_y) ? g.ny - 1 : y - 1;
        const int yp = (y == g.ny - 1 && g.per_y) ? 0 : y + 1;
        const int zm = (z == 0 && g.per_z) ? g.nz - 1 : z - 1;
        const int zp = (z == g.nz - 1 && g.per_z) ? 0 : z + 1;
        const int center = z * g.plane + y * g.pitch + x;
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
            const int sx = cx > 0 ? xm : (cx < 0 ? xp : x);
            const int sy = cy > 0 ? ym : (cy < 0 ? yp : y);
            const int sz = cz > 0 ? zm : (cz < 0 ? zp : z);
            const T* src = a.fin[i] + (sz * g.plane + sy * g.pitch + sx);
            if constexpr (i != 0) {
                if ((mk[c] >> i) & 1u) src = a.fout[opp_of(i)] + center;
            }
            f[c][i] = *src;
        });
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        if (!ok[c]) continue;
        const int s = a.slot ? a.slot[(static_cast<long long>(zs[c]) * g.ny + ys[c]) * g.nx + xs[c]] : a.uniform_slot;
        collide_store_cell<T, Q, KM>(a, xs[c], ys[c], zs[c], s, f[c]);
    }
}

// Lazy update of the wall cells the fluid-segment sweep leaves alone, before
// the state is read: for every listed (cell, link j) whose reader x_b + c_j is
// a collision cell, f_j(x_b) = f_opp(j)(x_b + c_j) of the previous state --
// exactly the bounce-back cell's own update on those links. Entry: x | y << 13
// | z << 26 | link mask << 38 (as k_list).
template <typename T, int Q>
__global__ void k_bb_finalize(T* cur, const T* prev, Geo g, const unsigned long long* __restrict__ list,
                              long long n) {
    using L = Lat<Q>;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const unsigned long long e = list[k];
        const int x = int(e & 0x1fffull), y = int((e >> 13) & 0x1fffull), z = int((e >> 26) & 0xfffull);
        const unsigned mask = unsigned(e >> 38);
        const int center = z * g.plane + y * g.pitch + x;
        sfor<Q>([&](auto I) {
            constexpr int j = decltype(I)::value;
            if constexpr (j != 0) {
                if ((mask >> (j - 1)) & 1u) {
                    constexpr int cx = L::c[j][0], cy = L::c[j][1], cz = L::c[j][2];
                    int X = x + cx, Y = y + cy, Z = z + cz;
                    if (g.per_x) X = X < 0 ? X + g.nx : (X >= g.nx ? X - g.nx : X);
                    if (g.per_y) Y = Y < 0 ? Y + g.ny : (Y >= g.ny ? Y - g.ny : Y);
                    if (g.per_z) Z = Z < 0 ? Z + g.nz : (Z >= g.nz ? Z - g.nz : Z);
                    cur[j * g.dstride + center] = prev[opp_of(j) * g.dstride + Z * g.plane + Y * g.pitch + X];
                }
            }
        });
    }
}

// Compacted porous sweep (single slab, non-periodic x).
// The masked sweep (k_seg) reads the listed segments where they lie in the
// dense layout: its isolated 32-B sectors are fetched from DRAM as 64-B pairs
// (ncu at c4 680x600^2: 30.9 GB read for 22 GB delivered to L1) and its
// +-1-shifted pulls straddle unlisted sectors. Here the listed segments -- and
// the segments they pull from -- are gathered into row-major compact arrays
// once, so consecutive listed segments are consecutive in memory and the
// x-neighbour of any source segment is the next / previous compact segment;
// the rows above / below come from a per-segment table of 8 compact indices.
// Same per-cell arithmetic and stores as k_seg (bit-identical); the dense
// layout is brought up to date (k_cmp_scatter) before the state is read.
// FIX: the regularized inlet / outlet cells, computed with the full dispatch
// set by a second launch on a parallel graph branch (the main sweep leaves
// them out: same input buffer, disjoint outputs); the lean main set keeps its
// register budget.
template <typename T, int Q, unsigned KM, int CPT, bool FIX>
__global__ void __launch_bounds__(256, (CPT == 1 ? min_blocks<T, Q, KM>() : 2))
    k_cmp(const __grid_constant__ StepArgs<T> a, const __grid_constant__ CmpArgs c) {
    using L = Lat<Q>;
    const int G = 1 << c.gshift;
    const long long base = static_cast<long long>(blockIdx.x) * (256 * CPT) + threadIdx.x;
    long long li[CPT], own[CPT];
    int lane[CPT];
    bool ok[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const long long t = base + 256 * k;
        ok[k] = t < c.n;
        li[k] = 0;
        lane[k] = 0;
        own[k] = 0;
        if (ok[k]) {
            long long cell = t;
            if constexpr (FIX) cell = __ldg(c.fix + t);
            li[k] = cell >> c.gshift;
            lane[k] = int(cell & (G - 1));
            const unsigned e = __ldg(c.seg + li[k]);
            own[k] = static_cast<long long>(e & 0x03ffffffu) * G + lane[k];
            ok[k] = lane[k] < int(e >> 26);
        }
    }
    T f[CPT][Q];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        if (!ok[k]) continue;
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
            long long src;
            if constexpr (cy == 0 && cz == 0) {
                src = own[k] - cx;
            } else {
                constexpr int r = cmp_row(-cy, -cz);
                const long long m = __ldg(c.rows + r * c.nlist + li[k]);
                src = m * G + lane[k] - cx;
            }
            f[k][i] = __ldg(a.fin[i] + src);
        });
    }
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        if (!ok[k]) continue;
        const int s = c.slot[own[k]];
        if constexpr (!FIX && (KM & (KM_REGV | KM_REGP)) == 0) {
            // regularized cells belong to the FIX launch, which runs beside
            // this one (same input buffer, disjoint outputs)
            if (recipe_of<KM>(a, s).has_reg) continue;
        }
        Cell<T, Q>::template apply<KM>(f[k], recipe_of<KM>(a, s));
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            a.fout[i][own[k]] = f[k][i];
        });
    }
}

// AA-pattern in-place streaming (PAPER.md:104 future work): one
// population array A, two alternating kernels, every location read and
// written by the same thread (race-free in place), the same 2*q*sizeof(T)
// bytes per cell as the two-population scheme with half the memory.
//   even step: f_i = A[i][x];            collide; A[opp(i)][x]       = f_i
//   odd  step: f_i = A[opp(i)][x - c_i]; collide; A[i][x + c_i]      = f_i
// After an even step the canonical state is f_i(x) = A[opp(i)][x], after an
// odd step (and at upload) f_i(x) = A[i][x + c_i]. Pulls from outside a
// non-periodic face read 0: the odd step reads nothing there and zeroes
// A[i][x] (the location the next even step reads for that link); pushes
// across a non-periodic face land in the envelope, where they stay part of the
// canonical state but are never read.
//
// Linked z-slabs (boundary launch, push_up / push_down set). Every location
// of the global AA array is still touched by exactly one cell per step; the
// ones across a slab face belong to the neighbour, so:
//  * even step: nothing crosses a face; the top plane additionally stores its
//    c_z = +1 populations f_i into the upper neighbour's A[i] at z = -1, the
//    bottom plane its c_z = -1 ones into the lower neighbour's A[i] at z = nz
//    (the two-population push; these ghost slots are never part of the state);
//  * odd step: a pull from across the face reads that pushed value, A[i] of the
//    own ghost plane (instead of A[opp(i)] of the neighbour's boundary plane,
//    which holds the same number); the store A[i][x + c_i] across the face goes
//    to the neighbour's boundary plane (z = 0 of the upper, z = nz - 1 of the
//    lower), where its next even step reads it, and to the own ghost plane
//    (the canonical odd-layout value of this slab's cell, read by downloads).
// Linked slabs therefore rest in the even layout after a fill / upload (their
// first step is odd), and the halo protocol of the two-population scheme
// (wait for both neighbours' previous boundary launch, signal after ours)
// orders every cross-face access. LINKED: the boundary-plane instantiation
// (catch-all dispatch set; the interior launch runs the lean one, whose
// register budget the face logic would overflow).
template <typename T, int Q, unsigned KM, bool ODD, bool LINKED = false>
__global__ void __launch_bounds__(256, (min_blocks<T, Q, KM>())) k_aa(const __grid_constant__ StepArgs<T> a) {
    using L = Lat<Q>;
    const Geo& g = a.g;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int z = a.z_begin + int(blockIdx.z) * a.z_step;
    if (a.err != nullptr && __ldca(a.err) != 0ull) return;  // failed exchange: write nothing
    const bool active = x < g.nx && y < g.ny;
    const int center = z * g.plane + y * g.pitch + x;
    T f[Q];
    if (active) {
        // (neighbour coordinates are recomputed after the collision rather
        // than kept live across it: the fp32 BGK / TRT sets run at 40-48
        // registers and would spill)
        if constexpr (!ODD) {
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                f[i] = a.fin[i][center];
            });
        } else {
            const bool lo_link = LINKED && a.push_down != nullptr && z == 0;
            const bool hi_link = LINKED && a.push_up != nullptr && z == g.nz - 1;
            const int xm = (x == 0 && g.per_x) ? g.nx - 1 : x - 1;
            const int xp = (x == g.nx - 1 && g.per_x) ? 0 : x + 1;
            const int ym = (y == 0 && g.per_y) ? g.ny - 1 : y - 1;
            const int yp = (y == g.ny - 1 && g.per_y) ? 0 : y + 1;
            const int zm = (z == 0 && g.per_z) ? g.nz - 1 : z - 1;
            const int zp = (z == g.nz - 1 && g.per_z) ? 0 : z + 1;
            const bool xlo = xm < 0, xhi = xp >= g.nx, ylo = ym < 0, yhi = yp >= g.ny;
            const bool zlo = zm < 0 && !lo_link, zhi = zp >= g.nz && !hi_link;
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
                const bool out = (cx > 0 && xlo) || (cx < 0 && xhi) || (cy > 0 && ylo) ||
                                 (cy < 0 && yhi) || (cz > 0 && zlo) || (cz < 0 && zhi);
                const int sx = cx > 0 ? xm : (cx < 0 ? xp : x);
                const int sy = cy > 0 ? ym : (cy < 0 ? yp : y);
                const int sz = cz > 0 ? zm : (cz < 0 ? zp : z);
                // across a linked face: the neighbour's pushed value in the own ghost plane
                const bool ghost = (cz > 0 && lo_link) || (cz < 0 && hi_link);
                f[i] = out ? T(0) : a.fin[ghost ? i : opp_of(i)][sz * g.plane + sy * g.pitch + sx];
            });
        }
        int s = a.uniform_slot;
        if (a.slot != nullptr) s = a.slot[(static_cast<long long>(z) * g.ny + y) * g.nx + x];
        Cell<T, Q>::template apply<KM>(f, recipe_of<KM>(a, s));
    }
    // (tried: odd-step c_x != 0 stores realigned per block row through shared
    // memory -- 3.61 vs 3.52 ms per 512^3 odd step, L2 write sectors unchanged;
    // profiles/r02b_summary.md)
    if (active) {
        const bool lo_link = LINKED && a.push_down != nullptr && z == 0;
        const bool hi_link = LINKED && a.push_up != nullptr && z == g.nz - 1;
        if constexpr (!ODD) {
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                a.fout[opp_of(i)][center] = f[i];
            });
            if (LINKED && hi_link) {
                const int ghost = -g.plane + y * g.pitch + x;
                sfor<Q>([&](auto I) {
                    constexpr int i = decltype(I)::value;
                    if constexpr (L::c[i][2] > 0) a.push_up[i * a.up_dstride + ghost] = f[i];
                });
            }
            if (LINKED && lo_link) {
                const int ghost = a.down_ghost_z * g.plane + y * g.pitch + x;
                sfor<Q>([&](auto I) {
                    constexpr int i = decltype(I)::value;
                    if constexpr (L::c[i][2] < 0) a.push_down[i * a.down_dstride + ghost] = f[i];
                });
            }
        } else {
            const int xm = (x == 0 && g.per_x) ? g.nx - 1 : x - 1;
            const int xp = (x == g.nx - 1 && g.per_x) ? 0 : x + 1;
            const int ym = (y == 0 && g.per_y) ? g.ny - 1 : y - 1;
            const int yp = (y == g.ny - 1 && g.per_y) ? 0 : y + 1;
            const int zm = (z == 0 && g.per_z) ? g.nz - 1 : z - 1;
            const int zp = (z == g.nz - 1 && g.per_z) ? 0 : z + 1;
            const bool xlo = xm < 0, xhi = xp >= g.nx, ylo = ym < 0, yhi = yp >= g.ny;
            const bool zlo = zm < 0 && !lo_link, zhi = zp >= g.nz && !hi_link;
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
                const int dx = cx > 0 ? xp : (cx < 0 ? xm : x);
                const int dy = cy > 0 ? yp : (cy < 0 ? ym : y);
                const int dz = cz > 0 ? zp : (cz < 0 ? zm : z);
                a.fout[i][dz * g.plane + dy * g.pitch + dx] = f[i];
                if constexpr (LINKED && cz > 0) {
                    if (hi_link) a.push_up[i * a.up_dstride + dy * g.pitch + dx] = f[i];
                }
                if constexpr (LINKED && cz < 0) {
                    if (lo_link)
                        a.push_down[i * a.down_dstride + (a.down_ghost_z - 1) * g.plane + dy * g.pitch + dx] = f[i];
                }
                if constexpr (i != 0) {
                    const bool out = (cx > 0 && xlo) || (cx < 0 && xhi) || (cy > 0 && ylo) ||
                                     (cy < 0 && yhi) || (cz > 0 && zlo) || (cz < 0 && zhi);
                    if (out) a.fout[i][center] = T(0);
                }
            });
        }
    }
    if constexpr (LINKED) {
        if (a.counter != nullptr) signal_step(a);
    }
}

// Sparse, kind-sorted list variant for porous media.
// The host groups the cells that move populations by registry slot (so every
// launch runs one dynamics kind with a minimal instantiation and no per-cell
// dispatch), in row-major order. NoDynamics cells are not listed. Bounce-back
// cells (MASKED) carry the set of links whose source is a fluid cell: only
// those are loaded and, after the swap, stored — every other link of a wall
// cell only ever feeds solid cells, so Collide-kind cells stay
// bit-identical to the dense reference sweep.
// Entry: x | y << 13 | z << 26 | link mask (links 1..q-1) << 38.
template <typename T, int Q, unsigned KM, bool MASKED>
__global__ void __launch_bounds__(256, (min_blocks<T, Q, KM>()))
    k_list(const __grid_constant__ StepArgs<T> a, const unsigned long long* __restrict__ list,
           long long n, int slot) {
    using L = Lat<Q>;
    const Geo& g = a.g;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned long long next = idx < n ? __ldg(list + idx) : 0ull;
    for (; idx < n; idx += stride) {
        const unsigned long long e = next;
        if (idx + stride < n) next = __ldg(list + idx + stride);  // prefetch the next entry
        const int x = int(e & 0x1fffull);
        const int y = int((e >> 13) & 0x1fffull);
        const int z = int((e >> 26) & 0xfffull);
        const unsigned mask = unsigned(e >> 38);
        const int xm = (x == 0 && g.per_x) ? g.nx - 1 : x - 1;
        const int xp = (x == g.nx - 1 && g.per_x) ? 0 : x + 1;
        const int ym = (y == 0 && g.per_y) ? g.ny - 1 : y - 1;
        const int yp = (y == g.ny - 1 && g.per_y) ? 0 : y + 1;
        const int zm = (z == 0 && g.per_z) ? g.nz - 1 : z - 1;
        const int zp = (z == g.nz - 1 && g.per_z) ? 0 : z + 1;
        T f[Q];
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
            const int sx = cx > 0 ? xm : (cx < 0 ? xp : x);
            const int sy = cy > 0 ? ym : (cy < 0 ? yp : y);
            const int sz = cz > 0 ? zm : (cz < 0 ? zp : z);
            bool use = true;
            if constexpr (MASKED) use = i != 0 && ((mask >> (i - 1)) & 1u);
            f[i] = use ? __ldg(a.fin[i] + (sz * g.plane + sy * g.pitch + sx)) : T(0);
        });
        Cell<T, Q>::template apply<KM>(f, recipe_of<KM>(a, slot));
        const int center = z * g.plane + y * g.pitch + x;
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            bool use = true;
            if constexpr (MASKED) {
                constexpr int o = opp_of(i);
                use = o != 0 && ((mask >> (o - 1)) & 1u);
            }
            if (use) a.fout[i][center] = f[i];
        });
    }
}

// ---------------------------------------------------------------------------
// TMA-staged pull (dense two-population, single slab). A persistent CTA walks
// tiles of BX x BY cells of one z-plane; per tile, one elected thread issues q
// 4-D TMA box loads (cp.async.bulk.tensor) — direction i's box is the tile
// shifted by -c_i, read straight out of the envelope-inclusive layout — into
// an S-stage shared-memory ring tracked by mbarriers (expect_tx), so S-1 tiles
// of neighbour data are in flight while the threads collide the current one.
// Loads need no wrap logic: on periodic axes the envelope holds the periodic
// images, which the kernel itself keeps current by pushing every boundary
// cell's outgoing links into the opposite envelope of the output buffer
// (k_refresh_envelope primes it once after a fill / upload).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned phase) {
    unsigned done = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
    } while (!done);
}

// Lattice velocities for the TMA issue loop (kept as a runtime loop: a fully
// unrolled run of q tensor copies exhausts the uniform register file).
__constant__ signed char kTmaC[27][3] = {
    {0, 0, 0},
    {-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1},
    {-1, -1, 0}, {1, 1, 0}, {-1, 1, 0}, {1, -1, 0},
    {-1, 0, -1}, {1, 0, 1}, {-1, 0, 1}, {1, 0, -1},
    {0, -1, -1}, {0, 1, 1}, {0, -1, 1}, {0, 1, -1},
    {-1, -1, -1}, {1, 1, 1}, {-1, -1, 1}, {1, 1, -1},
    {-1, 1, -1}, {1, -1, 1}, {1, -1, -1}, {-1, 1, 1}};

// TMA tile loads need a 16-B aligned start in the innermost dimension, so each
// direction's box starts at x0 - E (E = 16 B / sizeof(T)) and is BX + 2E wide;
// the x shift of the pull is applied when reading shared memory.
template <typename T>
__host__ __device__ constexpr int tma_pad() {
    return int(16 / sizeof(T));
}

template <typename T, int Q, int BX, int BY>
__device__ __noinline__ void tma_issue_tile(const CUtensorMap* map, T* dst, unsigned bar, int x0, int y0, int z,
                                            int xoff) {
    constexpr int E = tma_pad<T>();
    constexpr int W = BX + 2 * E;
    constexpr unsigned bytes = unsigned(Q * W * BY * sizeof(T));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    const unsigned long long desc = reinterpret_cast<unsigned long long>(map);
    const unsigned base = smem_u32(dst);
#pragma unroll 1
    for (int i = 0; i < Q; ++i) {
        const int c0 = x0 - E + xoff, c1 = y0 - kTmaC[i][1] + 1, c2 = z - kTmaC[i][2] + 1;
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(base + unsigned(i * W * BY * sizeof(T))),
            "l"(desc), "r"(c0), "r"(c1), "r"(c2), "r"(i), "r"(bar)
            : "memory");
    }
}

// Warp-specialised: warps 0..NW-1 collide (each thread RPT cells of the
// tile, rows ty + k * (BY / RPT)), warp NW is the TMA producer. full[st]
// completes when the q boxes of a tile have landed (expect_tx), empty[st]
// when all consumer warps have pulled their values out of the stage.
template <typename T, int Q, unsigned KM, int BX, int BY, int S>
__global__ void __launch_bounds__(BX * BY + 32, 1)
    k_tma(const __grid_constant__ StepArgs<T> a, const CUtensorMap* __restrict__ tin, int xoff) {
    using L = Lat<Q>;
    constexpr int NT = BX * BY;             // consumer threads (one cell each)
    constexpr int NW = NT / 32;             // consumer warps
    constexpr int RPT = BX * BY / NT;       // cells per consumer thread
    constexpr int E = tma_pad<T>();
    constexpr int W = BX + 2 * E;           // padded box width (aligned start, see tma_issue_tile)
    constexpr int STAGE = Q * W * BY;
    const Geo& g = a.g;
    extern __shared__ __align__(128) unsigned char smem[];
    T* ring = reinterpret_cast<T*>(smem);
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + size_t(S) * STAGE * sizeof(T));
    unsigned long long* empty = full + S;
    const int tid = threadIdx.x;
    const int tiles_x = (g.nx + BX - 1) / BX, tiles_y = (g.ny + BY - 1) / BY;
    const int tiles_per_plane = tiles_x * tiles_y;
    const long long ntiles = static_cast<long long>(tiles_per_plane) * g.nz;
    auto tile_xyz = [&](long long t, int& x0, int& y0, int& z) {
        z = int(t / tiles_per_plane);
        const int r = int(t % tiles_per_plane);
        y0 = (r / tiles_x) * BY;
        x0 = (r % tiles_x) * BX;
    };
    if (tid == 0) {
        for (int st = 0; st < S; ++st) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + st)) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(empty + st)), "r"(NW) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (tid >= NT) {  // ---- producer warp
        if (tid == NT) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(tin)) : "memory");
            int k = 0;
            for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
                const int st = k % S;
                if (k >= S) mbar_wait(smem_u32(empty + st), unsigned((k / S) - 1) & 1u);
                int x0, y0, z;
                tile_xyz(t, x0, y0, z);
                tma_issue_tile<T, Q, BX, BY>(tin, ring + size_t(st) * STAGE, smem_u32(full + st), x0, y0, z, xoff);
            }
        }
        return;
    }

    // ---- consumer warps
    const int tx = tid % BX, ty0 = tid / BX;
    constexpr int ROWS = NT / BX;  // rows covered by one pass of the consumer threads
    int k = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int st = k % S;
        int x0, y0, z;
        tile_xyz(t, x0, y0, z);
        mbar_wait(smem_u32(full + st), unsigned(k / S) & 1u);
        const T* tile = ring + size_t(st) * STAGE;
        T fr[RPT][Q];
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int ty = ty0 + r * ROWS;
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                constexpr int cx = L::c[i][0];
                fr[r][i] = tile[(i * BY + ty) * W + tx + E - cx];
            });
        }
        __syncwarp();
        if ((tid & 31) == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + st)) : "memory");
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int x = x0 + tx, y = y0 + ty0 + r * ROWS;
            if (x >= g.nx || y >= g.ny) continue;
            T (&f)[Q] = fr[r];
            int s = a.uniform_slot;
            if (a.slot != nullptr) s = a.slot[(static_cast<long long>(z) * g.ny + y) * g.nx + x];
            Cell<T, Q>::template apply<KM>(f, recipe_of<KM>(a, s));
            const int center = z * g.plane + y * g.pitch + x;
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                a.fout[i][center] = f[i];
            });
            // periodic images of the outgoing links of boundary cells
            const bool bx_lo = g.per_x && x == 0, bx_hi = g.per_x && x == g.nx - 1;
            const bool by_lo = g.per_y && y == 0, by_hi = g.per_y && y == g.ny - 1;
            const bool bz_lo = g.per_z && z == 0, bz_hi = g.per_z && z == g.nz - 1;
            if (bx_lo || bx_hi || by_lo || by_hi || bz_lo || bz_hi) {
                sfor<Q>([&](auto I) {
                    constexpr int i = decltype(I)::value;
                    constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
                    int X = x, Y = y, Z = z;
                    bool moved = false;
                    if (cx > 0 && bx_hi) { X = x - g.nx; moved = true; }
                    if (cx < 0 && bx_lo) { X = x + g.nx; moved = true; }
                    if (cy > 0 && by_hi) { Y = y - g.ny; moved = true; }
                    if (cy < 0 && by_lo) { Y = y + g.ny; moved = true; }
                    if (cz > 0 && bz_hi) { Z = z - g.nz; moved = true; }
                    if (cz < 0 && bz_lo) { Z = z + g.nz; moved = true; }
                    if (moved) a.fout[i][Z * g.plane + Y * g.pitch + X] = f[i];
                });
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Row-staged TMA pull (dense two-population, single slab). Unit of work = one
// x-row (y, z) of the output. For each direction i the producer warp loads the
// WHOLE source row (y - c_y, z - c_z), x = -E .. nx + E, as nb boxes of bw
// elements of a 3-D tensor map (x, row, direction) into one stage of an
// S-deep shared-memory ring (mbarrier expect_tx) -- every source element is
// fetched exactly once per step (the x shift of the pull is a shared-memory
// offset, the y / z shifts select the row), so there are no halo re-reads.
// The consumer warps walk the row, collide and store straight to HBM, then
// release the stage. Periodic axes read the envelope, kept current by the
// kernel itself (boundary cells push their outgoing links into the opposite
// envelope of the output buffer, as in k_tma).
template <typename T, int Q, unsigned KM, int NCW>
__global__ void __launch_bounds__(NCW * 32 + 32, (NCW >= 16 ? 1 : 2))
    k_tmarow(const __grid_constant__ StepArgs<T> a, const CUtensorMap* __restrict__ tin, int nb, int bw, int S,
             int tw) {
    using L = Lat<Q>;
    constexpr int NT = NCW * 32;
    constexpr int E = tma_pad<T>();
    const Geo& g = a.g;
    const int W = nb * bw;
    const int stage = Q * W;
    extern __shared__ __align__(128) unsigned char smem[];
    T* ring = reinterpret_cast<T*>(smem);
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + size_t(S) * stage * sizeof(T));
    unsigned long long* empty = full + S;
    const int tid = threadIdx.x;
    const int tiles_x = (g.nx + tw - 1) / tw;  // a work unit is tw cells of one row
    const long long rows = static_cast<long long>(g.ny) * g.nz * tiles_x;
    if (tid == 0) {
        for (int st = 0; st < S; ++st) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + st)) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(empty + st)), "r"(NCW) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (tid >= NT) {  // ---- producer warp: lane i issues direction i's boxes (parallel TMA issue)
        const int lane = tid - NT;
        if (lane == 0)
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(tin)) : "memory");
        const unsigned long long desc = reinterpret_cast<unsigned long long>(tin);
        const unsigned bytes = unsigned(stage * sizeof(T));
        int k = 0;
        for (long long r = blockIdx.x; r < rows; r += gridDim.x, ++k) {
            const int st = k % S;
            if (k >= S) mbar_wait(smem_u32(empty + st), unsigned((k / S) - 1) & 1u);
            const long long ry = r / tiles_x;
            const int x0 = int(r - ry * tiles_x) * tw;
            const int z = int(ry / g.ny), y = int(ry - static_cast<long long>(z) * g.ny);
            const unsigned bar = smem_u32(full + st);
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
            __syncwarp();
            const unsigned base = smem_u32(ring + size_t(st) * stage);
            for (int i = lane; i < Q; i += 32) {
                const int row = (z - kTmaC[i][2] + 1) * (g.ny + 2) + (y - kTmaC[i][1] + 1);
#pragma unroll 1
                for (int b = 0; b < nb; ++b) {
                    const unsigned dst = base + unsigned((i * W + b * bw) * sizeof(T));
                    asm volatile(
                        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
                        "l"(desc), "r"(x0 + b * bw), "r"(row), "r"(i), "r"(bar)
                        : "memory");
                }
            }
        }
        return;
    }

    // ---- consumer warps
    int k = 0;
    for (long long r = blockIdx.x; r < rows; r += gridDim.x, ++k) {
        const int st = k % S;
        const long long ry = r / tiles_x;
        const int x0 = int(r - ry * tiles_x) * tw;
        const int z = int(ry / g.ny), y = int(ry - static_cast<long long>(z) * g.ny);
        const int x1 = min(g.nx, x0 + tw);
        mbar_wait(smem_u32(full + st), unsigned(k / S) & 1u);
        const T* srow = ring + size_t(st) * stage - x0;
        for (int x = x0 + tid; x < x1; x += NT) {
            T f[Q];
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                constexpr int cx = L::c[i][0];
                f[i] = srow[i * W + x + E - cx];
            });
            int s = a.uniform_slot;
            if (a.slot != nullptr) s = a.slot[(static_cast<long long>(z) * g.ny + y) * g.nx + x];
            Cell<T, Q>::template apply<KM>(f, recipe_of<KM>(a, s));
            const int center = z * g.plane + y * g.pitch + x;
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                a.fout[i][center] = f[i];
            });
            const bool bx_lo = g.per_x && x == 0, bx_hi = g.per_x && x == g.nx - 1;
            const bool by_lo = g.per_y && y == 0, by_hi = g.per_y && y == g.ny - 1;
            const bool bz_lo = g.per_z && z == 0, bz_hi = g.per_z && z == g.nz - 1;
            if (bx_lo || bx_hi || by_lo || by_hi || bz_lo || bz_hi) {
                sfor<Q>([&](auto I) {
                    constexpr int i = decltype(I)::value;
                    constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
                    int X = x, Y = y, Z = z;
                    bool moved = false;
                    if (cx > 0 && bx_hi) { X = x - g.nx; moved = true; }
                    if (cx < 0 && bx_lo) { X = x + g.nx; moved = true; }
                    if (cy > 0 && by_hi) { Y = y - g.ny; moved = true; }
                    if (cy < 0 && by_lo) { Y = y + g.ny; moved = true; }
                    if (cz > 0 && bz_hi) { Z = z - g.nz; moved = true; }
                    if (cz < 0 && bz_lo) { Z = z + g.nz; moved = true; }
                    if (moved) a.fout[i][Z * g.plane + Y * g.pitch + X] = f[i];
                });
            }
        }
        __syncwarp();
        if ((tid & 31) == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + st)) : "memory");
    }
}

// Block-staged TMA pull (the DLB_FLAG_TMA kernel of uniform lattices): work unit =
// R consecutive rows x (256 - 2E) cells of one plane; per direction ONE 2-D
// tensor box (256 x R) brings all the unit's source rows, so the number of
// tensor-copy instructions per cell drops R * 256 / 1040 times against
// k_tmarow (whose limiter is the copy issue rate).
template <typename T, int Q, unsigned KM, int NCW, int R>
__global__ void __launch_bounds__(NCW * 32 + 32, (NCW >= 16 ? 1 : 2))
    k_tmablk(const __grid_constant__ StepArgs<T> a, const CUtensorMap* __restrict__ tin, int S) {
    using L = Lat<Q>;
    constexpr int NT = NCW * 32;
    constexpr int E = tma_pad<T>();
    constexpr int BW = 256;
    constexpr int TW = BW - 2 * E;
    constexpr int stage = Q * R * BW;
    const Geo& g = a.g;
    extern __shared__ __align__(128) unsigned char smem[];
    T* ring = reinterpret_cast<T*>(smem);
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + size_t(S) * stage * sizeof(T));
    unsigned long long* empty = full + S;
    const int tid = threadIdx.x;
    const int tiles_x = (g.nx + TW - 1) / TW, tiles_y = (g.ny + R - 1) / R;
    const long long units = static_cast<long long>(tiles_x) * tiles_y * g.nz;
    if (tid == 0) {
        for (int st = 0; st < S; ++st) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + st)) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(empty + st)), "r"(NCW) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto unit_xyz = [&](long long u, int& x0, int& y0, int& z) {
        const long long v = u / tiles_x;
        x0 = int(u - v * tiles_x) * TW;
        z = int(v / tiles_y);
        y0 = int(v - static_cast<long long>(z) * tiles_y) * R;
    };
    if (tid >= NT) {  // producer warp: lane i loads direction i's 2-D box
        const int lane = tid - NT;
        if (lane == 0)
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(tin)) : "memory");
        const unsigned long long desc = reinterpret_cast<unsigned long long>(tin);
        int k = 0;
        for (long long u = blockIdx.x; u < units; u += gridDim.x, ++k) {
            const int st = k % S;
            if (k >= S) mbar_wait(smem_u32(empty + st), unsigned((k / S) - 1) & 1u);
            int x0, y0, z;
            unit_xyz(u, x0, y0, z);
            const unsigned bar = smem_u32(full + st);
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                             "r"(unsigned(stage * sizeof(T))) : "memory");
            __syncwarp();
            const unsigned base = smem_u32(ring + size_t(st) * stage);
            for (int i = lane; i < Q; i += 32) {
                const int row = (z - kTmaC[i][2] + 1) * (g.ny + 2) + (y0 - kTmaC[i][1] + 1);
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(base + unsigned(i * R * BW * sizeof(T))),
                    "l"(desc), "r"(x0), "r"(row), "r"(i), "r"(bar)
                    : "memory");
            }
        }
        return;
    }
    int k = 0;
    for (long long u = blockIdx.x; u < units; u += gridDim.x, ++k) {
        const int st = k % S;
        int x0, y0, z;
        unit_xyz(u, x0, y0, z);
        mbar_wait(smem_u32(full + st), unsigned(k / S) & 1u);
        const T* sb = ring + size_t(st) * stage;
        for (int idx = tid; idx < TW * R; idx += NT) {
            const int r = idx / TW, xx = idx - r * TW;
            const int x = x0 + xx, y = y0 + r;
            if (x >= g.nx || y >= g.ny) continue;
            T f[Q];
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                constexpr int cx = L::c[i][0];
                f[i] = sb[(i * R + r) * BW + xx + E - cx];
            });
            int s = a.uniform_slot;
            if (a.slot != nullptr) s = a.slot[(static_cast<long long>(z) * g.ny + y) * g.nx + x];
            Cell<T, Q>::template apply<KM>(f, recipe_of<KM>(a, s));
            const int center = z * g.plane + y * g.pitch + x;
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                a.fout[i][center] = f[i];
            });
            const bool bx_lo = g.per_x && x == 0, bx_hi = g.per_x && x == g.nx - 1;
            const bool by_lo = g.per_y && y == 0, by_hi = g.per_y && y == g.ny - 1;
            const bool bz_lo = g.per_z && z == 0, bz_hi = g.per_z && z == g.nz - 1;
            if (bx_lo || bx_hi || by_lo || by_hi || bz_lo || bz_hi) {
                sfor<Q>([&](auto I) {
                    constexpr int i = decltype(I)::value;
                    constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
                    int X = x, Y = y, Z = z;
                    bool moved = false;
                    if (cx > 0 && bx_hi) { X = x - g.nx; moved = true; }
                    if (cx < 0 && bx_lo) { X = x + g.nx; moved = true; }
                    if (cy > 0 && by_hi) { Y = y - g.ny; moved = true; }
                    if (cy < 0 && by_lo) { Y = y + g.ny; moved = true; }
                    if (cz > 0 && bz_hi) { Z = z - g.nz; moved = true; }
                    if (cz < 0 && bz_lo) { Z = z + g.nz; moved = true; }
                    if (moved) a.fout[i][Z * g.plane + Y * g.pitch + X] = f[i];
                });
            }
        }
        __syncwarp();
        if ((tid & 31) == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + st)) : "memory");
    }
}

#define DLB_STR2(x) #x
#define DLB_STR(x) DLB_STR2(x)
#define ENTRY(T, Q, KM)                                                                  \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), LAYOUT_TWO_POP,                              \
            reinterpret_cast<const void*>(&k_pull<T, Q, unsigned(KM)>),                   \
            "k_pull<" #T ",D3Q" #Q "," #KM ">[" DLB_STR(DLB_MODE) "]"                      \
    }

#define ENTRY_MB(T, Q, KM, MB)                                                           \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), LAYOUT_TWO_POP,                              \
            reinterpret_cast<const void*>(&k_pull<T, Q, unsigned(KM), MB>),               \
            "k_pull<" #T ",D3Q" #Q "," #KM ",b" #MB ">[" DLB_STR(DLB_MODE) "]", 0, 0, 0, 1, 0, MB \
    }
#define MB_SET                                                                            \
    , ENTRY_MB(float, 19, KM_BGK, 5), ENTRY_MB(float, 19, KM_BGK, 4), ENTRY_MB(float, 19, KM_TRT | KM_BB | KM_MBB, 5), \
        ENTRY_MB(double, 19, KM_BGK, 2), ENTRY_MB(double, 27, KM_RR, 1)

#define AA_ENTRY(T, Q, KM, ODD)                                                          \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), ODD ? LAYOUT_AA_ODD : LAYOUT_AA,               \
            reinterpret_cast<const void*>(&k_aa<T, Q, unsigned(KM), ODD>),                \
            "k_aa_" #ODD "<" #T ",D3Q" #Q "," #KM ">[" DLB_STR(DLB_MODE) "]"                  \
    }
#define AA_PAIR(T, Q, KM) AA_ENTRY(T, Q, KM, false), AA_ENTRY(T, Q, KM, true)
// boundary planes of linked AA slabs: the common sets and the catch-alls (the
// catch-all fp32 instantiation runs at 80 registers: its two planes took 40 us
// per 512^2 step, beside a 3.3 ms interior)
#define AA_LINK_ENTRY(T, Q, KM, ODD)                                                     \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), ODD ? LAYOUT_AA_ODD_LINK : LAYOUT_AA_LINK,     \
            reinterpret_cast<const void*>(&k_aa<T, Q, unsigned(KM), ODD, true>),          \
            "k_aa_link_" #ODD "<" #T ",D3Q" #Q "," #KM ">[" DLB_STR(DLB_MODE) "]"             \
    }
#define AA_LINK_PAIR(T, Q, KM) AA_LINK_ENTRY(T, Q, KM, false), AA_LINK_ENTRY(T, Q, KM, true)
#define AA_LINK_SET(T)                                                                    \
    , AA_LINK_PAIR(T, 19, KM_BGK), AA_LINK_PAIR(T, 19, KM_TRT), AA_LINK_PAIR(T, 19, KM_TRT | KM_BB | KM_MBB), \
        AA_LINK_PAIR(T, 27, KM_RR),                                                       \
        AA_LINK_ENTRY(T, 19, KM_ALL, false), AA_LINK_ENTRY(T, 19, KM_ALL, true),          \
        AA_LINK_ENTRY(T, 27, KM_ALL, false), AA_LINK_ENTRY(T, 27, KM_ALL, true),          \
        AA_LINK_ENTRY(T, 19, KM_ALL | KM_XREC, false), AA_LINK_ENTRY(T, 19, KM_ALL | KM_XREC, true), \
        AA_LINK_ENTRY(T, 27, KM_ALL | KM_XREC, false), AA_LINK_ENTRY(T, 27, KM_ALL | KM_XREC, true)
#define AA_SET(T)                                                                         \
    AA_PAIR(T, 19, KM_BGK), AA_PAIR(T, 19, KM_TRT), AA_PAIR(T, 19, KM_RR),               \
        AA_PAIR(T, 19, KM_TRT | KM_BB | KM_MBB), AA_PAIR(T, 19, KM_ALL), AA_PAIR(T, 27, KM_RR), \
        AA_PAIR(T, 27, KM_ALL)

#define TMAROW_ENTRY1(T, Q, KM, NCW)                                                     \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), LAYOUT_TMAROW,                               \
            reinterpret_cast<const void*>(&k_tmarow<T, Q, unsigned(KM), NCW>),            \
            "k_tmarow<" #T ",D3Q" #Q "," #KM ",w" #NCW ">[" DLB_STR(DLB_MODE) "]", 0, 0, 0, 1, NCW \
    }
#define TMAROW_ENTRY(T, Q, KM) TMAROW_ENTRY1(T, Q, KM, 16), TMAROW_ENTRY1(T, Q, KM, 8)
#define TMAROW_SET(T)                                                                     \
    TMAROW_ENTRY(T, 19, KM_BGK), TMAROW_ENTRY(T, 19, KM_TRT), TMAROW_ENTRY(T, 19, KM_BGK | KM_BB | KM_MBB), \
        TMAROW_ENTRY(T, 19, KM_TRT | KM_BB | KM_MBB)

#define TMABLK_ENTRY(T, Q, KM, R, W)                                                     \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), LAYOUT_TMABLK,                               \
            reinterpret_cast<const void*>(&k_tmablk<T, Q, unsigned(KM), W, R>),           \
            "k_tmablk<" #T ",D3Q" #Q "," #KM ",r" #R ",w" #W ">[" DLB_STR(DLB_MODE) "]", 0, R, 0, 1, W \
    }
#define TMABLK_SET                                                                        \
    , TMABLK_ENTRY(float, 19, KM_BGK, 4, 16), TMABLK_ENTRY(float, 19, KM_TRT | KM_BB | KM_MBB, 4, 16), \
        TMABLK_ENTRY(double, 19, KM_BGK, 2, 16), TMABLK_ENTRY(double, 19, KM_TRT | KM_BB | KM_MBB, 2, 16)

#define COOP_ENTRY(T, Q, KM)                                                             \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), LAYOUT_COOP,                                 \
            reinterpret_cast<const void*>(&k_pull_coop<T, Q, unsigned(KM)>),             \
            "k_pull_coop<" #T ",D3Q" #Q "," #KM ">[" DLB_STR(DLB_MODE) "]"                  \
    }
#define COOP_SET(T)                                                                       \
    , COOP_ENTRY(T, 19, KM_BGK), COOP_ENTRY(T, 19, KM_TRT), COOP_ENTRY(T, 19, KM_RR),     \
        COOP_ENTRY(T, 19, KM_BGK | KM_BB | KM_MBB), COOP_ENTRY(T, 19, KM_TRT | KM_BB | KM_MBB), \
        COOP_ENTRY(T, 19, KM_RR | KM_BB | KM_MBB), COOP_ENTRY(T, 27, KM_RR)

#define SEG_ENTRY1(T, Q, KM, CPT)                                                        \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), LAYOUT_SEG,                                  \
            reinterpret_cast<const void*>(&k_seg<T, Q, unsigned(KM), CPT>),               \
            "k_seg<" #T ",D3Q" #Q "," #KM ",x" #CPT ">[" DLB_STR(DLB_MODE) "]", 0, 0, 0, CPT \
    }
#define SEG_ENTRY(T, Q, KM) SEG_ENTRY1(T, Q, KM, 1), SEG_ENTRY1(T, Q, KM, 2)
#define SEGBB_ENTRY1(T, Q, KM, CPT)                                                      \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), LAYOUT_SEGBB,                                \
            reinterpret_cast<const void*>(&k_segbb<T, Q, unsigned(KM), CPT>),             \
            "k_segbb<" #T ",D3Q" #Q "," #KM ",x" #CPT ">[" DLB_STR(DLB_MODE) "]", 0, 0, 0, CPT \
    }
#define SEGBB_ENTRY(T, Q, KM) SEGBB_ENTRY1(T, Q, KM, 1), SEGBB_ENTRY1(T, Q, KM, 2)
#define SEGBB_SET(T)                                                                      \
    , SEGBB_ENTRY(T, 19, KM_BGK | KM_BB | KM_NODYN), SEGBB_ENTRY(T, 19, KM_TRT | KM_BB | KM_NODYN), \
        SEGBB_ENTRY(T, 19, KM_RR | KM_BB | KM_NODYN), SEGBB_ENTRY(T, 27, KM_BGK | KM_BB | KM_NODYN), \
        SEGBB_ENTRY(T, 27, KM_TRT | KM_BB | KM_NODYN), SEGBB_ENTRY(T, 27, KM_RR | KM_BB | KM_NODYN)
#define SEG_MB(T, Q, KM, CPT, MB)                                                        \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), LAYOUT_SEG,                                  \
            reinterpret_cast<const void*>(&k_seg<T, Q, unsigned(KM), CPT, MB>),           \
            "k_seg<" #T ",D3Q" #Q "," #KM ",x" #CPT ",b" #MB ">[" DLB_STR(DLB_MODE) "]", 0, 0, 0, CPT, 0, MB \
    }
#define SEG_MB_SET                                                                        \
    , SEG_MB(double, 19, KM_TRT | KM_BB | KM_NODYN, 1, 4), SEG_MB(double, 19, KM_TRT | KM_BB | KM_NODYN, 1, 5), \
        SEG_MB(double, 19, KM_TRT | KM_BB | KM_NODYN, 2, 3)
#define SEG_SET(T)                                                                        \
    SEG_ENTRY(T, 19, KM_BGK | KM_BB | KM_NODYN), SEG_ENTRY(T, 19, KM_TRT | KM_BB | KM_NODYN), \
        SEG_ENTRY(T, 19, KM_RR | KM_BB | KM_NODYN),                                       \
        SEG_ENTRY(T, 19, KM_BGK | KM_BB | KM_NODYN | KM_REGV | KM_REGP),                  \
        SEG_ENTRY(T, 19, KM_TRT | KM_BB | KM_NODYN | KM_REGV | KM_REGP),                  \
        SEG_ENTRY(T, 19, KM_RR | KM_BB | KM_NODYN | KM_REGV | KM_REGP), SEG_ENTRY(T, 19, KM_ALL), \
        SEG_ENTRY(T, 27, KM_ALL)

#define LIST_ENTRY(T, Q, KM, M)                                                          \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), M ? LAYOUT_LIST_MASKED : LAYOUT_LIST,          \
            reinterpret_cast<const void*>(&k_list<T, Q, unsigned(KM), M>),                \
            "k_list<" #T ",D3Q" #Q "," #KM "," #M ">[" DLB_STR(DLB_MODE) "]"                  \
    }
#define LIST_SET(T, Q)                                                                    \
    LIST_ENTRY(T, Q, KM_BGK, false), LIST_ENTRY(T, Q, KM_TRT, false), LIST_ENTRY(T, Q, KM_RR, false), \
        LIST_ENTRY(T, Q, KM_BGK | KM_REGV | KM_REGP, false),                              \
        LIST_ENTRY(T, Q, KM_TRT | KM_REGV | KM_REGP, false),                              \
        LIST_ENTRY(T, Q, KM_RR | KM_REGV | KM_REGP, false), LIST_ENTRY(T, Q, KM_ALL, false), \
        LIST_ENTRY(T, Q, KM_BB, true), LIST_ENTRY(T, Q, KM_MBB, true)

// TMA tiles (one consumer thread per cell + 1 producer warp): f32 64 x 8 cells
// (3 stages), D3Q19 f64 32 x 16 (2 stages), D3Q27 fp64 32 x 8 (2 stages)
#define TMA_ENTRY(T, Q, KM, BX, BY, S)                                                   \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), LAYOUT_TMA,                                  \
            reinterpret_cast<const void*>(&k_tma<T, Q, unsigned(KM), BX, BY, S>),          \
            "k_tma<" #T ",D3Q" #Q "," #KM ">[" DLB_STR(DLB_MODE) "]", BX, BY, S               \
    }
#define TMA_SET                                                                           \
    TMA_ENTRY(float, 19, KM_BGK, 64, 8, 3), TMA_ENTRY(float, 19, KM_TRT, 64, 8, 3),       \
        TMA_ENTRY(float, 19, KM_BGK | KM_BB | KM_MBB, 64, 8, 3),                          \
        TMA_ENTRY(float, 19, KM_TRT | KM_BB | KM_MBB, 64, 8, 3),                          \
        TMA_ENTRY(double, 19, KM_BGK, 32, 16, 2), TMA_ENTRY(double, 19, KM_TRT, 32, 16, 2), \
        TMA_ENTRY(double, 19, KM_BGK | KM_BB | KM_MBB, 32, 16, 2),                        \
        TMA_ENTRY(double, 19, KM_TRT | KM_BB | KM_MBB, 32, 16, 2),                        \
        TMA_ENTRY(double, 27, KM_RR, 32, 8, 2)

#define Q19_SET(T)                                                                        \
    ENTRY(T, 19, KM_BGK), ENTRY(T, 19, KM_TRT), ENTRY(T, 19, KM_RR),                      \
        ENTRY(T, 19, KM_BGK | KM_BB | KM_MBB), ENTRY(T, 19, KM_TRT | KM_BB | KM_MBB),    \
        ENTRY(T, 19, KM_RR | KM_BB | KM_MBB),                                             \
        ENTRY(T, 19, KM_BGK | KM_BB | KM_NODYN | KM_REGV | KM_REGP),                      \
        ENTRY(T, 19, KM_TRT | KM_BB | KM_NODYN | KM_REGV | KM_REGP),                      \
        ENTRY(T, 19, KM_RR | KM_BB | KM_NODYN | KM_REGV | KM_REGP), ENTRY(T, 19, KM_ALL),        \
        ENTRY(T, 19, KM_BGK | KM_BB | KM_NODYN | KM_REGV | KM_REGP | KM_SKIP),                  \
        ENTRY(T, 19, KM_TRT | KM_BB | KM_NODYN | KM_REGV | KM_REGP | KM_SKIP),                  \
        ENTRY(T, 19, KM_RR | KM_BB | KM_NODYN | KM_REGV | KM_REGP | KM_SKIP), ENTRY(T, 19, KM_ALL | KM_SKIP), \
        ENTRY(T, 19, KM_BGK | KM_BB | KM_NODYN), ENTRY(T, 19, KM_TRT | KM_BB | KM_NODYN),             \
        ENTRY(T, 19, KM_RR | KM_BB | KM_NODYN), ENTRY(T, 19, KM_TRT | KM_BB | KM_NODYN | KM_SKIP)

#define Q27_SET(T) ENTRY(T, 27, KM_BGK), ENTRY(T, 27, KM_TRT), ENTRY(T, 27, KM_RR), ENTRY(T, 27, KM_ALL), \
        ENTRY(T, 27, KM_ALL | KM_SKIP)

// registries beyond kMaxSlots instances: the catch-all sets reading the
// recipe table from global memory
#define XREC_SET(T)                                                                       \
    , ENTRY(T, 19, KM_ALL | KM_XREC), ENTRY(T, 19, KM_ALL | KM_XREC | KM_SKIP), ENTRY(T, 27, KM_ALL | KM_XREC), \
        AA_PAIR(T, 19, KM_ALL | KM_XREC), AA_PAIR(T, 27, KM_ALL | KM_XREC)

// fused kinetic-energy variants: exact mode only (the reduce input must carry
// the diagnostics' non-contracted double arithmetic)
#ifdef DLB_FUSED_KE
#define KE_SET(T)                                                                         \
    , ENTRY(T, 19, KM_BGK | KM_KE), ENTRY(T, 19, KM_TRT | KM_KE), ENTRY(T, 19, KM_RR | KM_KE), \
        ENTRY(T, 19, KM_BGK | KM_LES | KM_KE), ENTRY(T, 19, KM_TRT | KM_LES | KM_KE),   \
        ENTRY(T, 19, KM_BGK | KM_BB | KM_MBB | KM_KE), ENTRY(T, 19, KM_TRT | KM_BB | KM_MBB | KM_KE), \
        ENTRY(T, 19, KM_RR | KM_BB | KM_MBB | KM_KE), ENTRY(T, 27, KM_RR | KM_KE), ENTRY(T, 27, KM_BGK | KM_KE)
#else
#define KE_SET(T)
#endif

#define CMP_ENTRY(T, Q, KM, CPT, FIX)                                                    \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), FIX ? LAYOUT_CMP_FIX : LAYOUT_CMP,             \
            reinterpret_cast<const void*>(&k_cmp<T, Q, unsigned(KM), CPT, FIX>),          \
            "k_cmp<" #T ",D3Q" #Q "," #KM ",x" #CPT ">[" DLB_STR(DLB_MODE) "]", 0, 0, 0, CPT \
    }
// main sweeps of the porous dispatch sets (regularized cells via the FIX list)
// and the fix-up / catch-all sets
#define CMP_SET(T)                                                                        \
    , CMP_ENTRY(T, 19, KM_TRT | KM_BB | KM_NODYN, 1, false), CMP_ENTRY(T, 19, KM_TRT | KM_BB | KM_NODYN, 2, false), \
        CMP_ENTRY(T, 19, KM_BGK | KM_BB | KM_NODYN, 1, false), CMP_ENTRY(T, 19, KM_BGK | KM_BB | KM_NODYN, 2, false), \
        CMP_ENTRY(T, 19, KM_RR | KM_BB | KM_NODYN, 1, false), CMP_ENTRY(T, 19, KM_ALL, 1, false),          \
        CMP_ENTRY(T, 27, KM_ALL, 1, false), CMP_ENTRY(T, 19, KM_ALL, 1, true), CMP_ENTRY(T, 27, KM_ALL, 1, true)

#define VEC_ENTRY(T, Q, KM)                                                              \
    KernelEntry {                                                                        \
        int(sizeof(T) * 8), Q, unsigned(KM), LAYOUT_VEC,                                  \
            reinterpret_cast<const void*>(&k_vec<T, Q, unsigned(KM)>),                    \
            "k_vec<" #T ",D3Q" #Q "," #KM ">[" DLB_STR(DLB_MODE) "]"                       \
    }
#define VEC_SET(T)                                                                        \
    , VEC_ENTRY(T, 19, KM_BGK), VEC_ENTRY(T, 19, KM_TRT), VEC_ENTRY(T, 19, KM_TRT | KM_BB | KM_MBB), \
        VEC_ENTRY(T, 19, KM_BGK | KM_BB | KM_MBB), VEC_ENTRY(T, 27, KM_RR)

static const KernelEntry kTable[] = {
    Q19_SET(float), Q19_SET(double), Q27_SET(float), Q27_SET(double), AA_SET(float), AA_SET(double),
    LIST_SET(float, 19), LIST_SET(double, 19), LIST_SET(float, 27), LIST_SET(double, 27),
    TMA_SET, SEG_SET(float), SEG_SET(double), TMAROW_SET(float), TMAROW_SET(double) KE_SET(float) KE_SET(double)
        COOP_SET(float) COOP_SET(double) TMABLK_SET MB_SET XREC_SET(float) XREC_SET(double) SEG_MB_SET
        SEGBB_SET(float) SEGBB_SET(double) AA_LINK_SET(float) AA_LINK_SET(double) CMP_SET(float) CMP_SET(double)
        VEC_SET(float) VEC_SET(double)
};

void launch_bb_finalize(int bits, int q, void* cur, const void* prev, const Geo& g,
                        const unsigned long long* list, long long n, cudaStream_t st) {
    if (n <= 0) return;
    const int grid = int(std::min<long long>((n + 255) / 256, 148LL * 16));
    if (bits == 64) {
        if (q == 19) k_bb_finalize<double, 19><<<grid, 256, 0, st>>>((double*)cur, (const double*)prev, g, list, n);
        else k_bb_finalize<double, 27><<<grid, 256, 0, st>>>((double*)cur, (const double*)prev, g, list, n);
    } else {
        if (q == 19) k_bb_finalize<float, 19><<<grid, 256, 0, st>>>((float*)cur, (const float*)prev, g, list, n);
        else k_bb_finalize<float, 27><<<grid, 256, 0, st>>>((float*)cur, (const float*)prev, g, list, n);
    }
}

const KernelEntry* kernel_table(int* n) {
    *n = int(sizeof(kTable) / sizeof(kTable[0]));
    return kTable;
}

}  // namespace DLB_MODE
}  // namespace dlb
