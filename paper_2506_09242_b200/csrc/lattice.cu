// Device lattice runtime (see lattice.hpp). Compiled with -fmad=false: the
// initialisation kernels evaluate equilibrium2<T> and the TGV state with the
// reference's operation order (multiblock.cpp:278-281, cases.cpp:145-156).
#include "lattice.hpp"

#include <atomic>
#include <mutex>
#include "canon.cuh"

#include <cstddef>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <cstdlib>
#include <random>
#include <thread>

namespace dlb {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {

constexpr std::size_t kStagingBytes = std::size_t(256) << 20;
// graph versions: unique across lattices (the multi-slab graph cache key)
std::atomic<uint64_t> g_graph_version{1};
constexpr int kCz19[19] = {0, 0, 0, 0, 0, -1, 1, 0, 0, 0, 0, -1, 1, 1, -1, -1, 1, 1, -1};
constexpr int kCz27[27] = {0, 0, 0, 0, 0, -1, 1, 0, 0, 0, 0, -1, 1, 1, -1, -1, 1, 1, -1,
                           -1, 1, 1, -1, -1, 1, -1, 1};
constexpr int kCx19[19] = {0, -1, 1, 0, 0, 0, 0, -1, 1, -1, 1, -1, 1, -1, 1, 0, 0, 0, 0};
constexpr int kCy19[19] = {0, 0, 0, -1, 1, 0, 0, -1, 1, 1, -1, 0, 0, 0, 0, -1, 1, -1, 1};
constexpr int kCx27[27] = {0, -1, 1, 0, 0, 0, 0, -1, 1, -1, 1, -1, 1, -1, 1, 0, 0, 0, 0,
                           -1, 1, -1, 1, -1, 1, 1, -1};
constexpr int kCy27[27] = {0, 0, 0, -1, 1, 0, 0, -1, 1, 1, -1, 0, 0, 0, 0, -1, 1, -1, 1,
                           -1, 1, -1, 1, 1, -1, -1, 1};

// ---------------------------------------------------------------------------
// auxiliary kernels

template <typename T>
__device__ __forceinline__ long long lin(const Geo& g, int x, int y, int z) {
    return static_cast<long long>(z) * g.plane + static_cast<long long>(y) * g.pitch + x;
}

// Where a fill stores canonical f_i(x, y, z) (aa_mode as canon_load: 0
// two-population, 1 AA even layout A[opp(i)][x], 2 AA odd layout A[i][x + c_i]).
template <int Q, int i>
__device__ __forceinline__ long long fill_pos(const Geo& g, int x, int y, int z, int aa_mode) {
    using L = Lat<Q>;
    constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
    const long long dir = aa_mode == 1 ? opp_of(i) : i;
    if (aa_mode == 2) return i * g.dstride + shifted(g, x, y, z, cx, cy, cz);
    return dir * g.dstride + static_cast<long long>(z) * g.plane + static_cast<long long>(y) * g.pitch + x;
}

// Stored state := equilibrium2<T>(T(rho), T(u)) for planes [z0, z0 + nzc).
template <typename T, int Q>
__global__ void k_fill_eq(T* origin, Geo g, const double* rho, const double* ux,
                          const double* uy, const double* uz, int z0, int nzc, int aa) {
    const long long n = static_cast<long long>(g.nx) * g.ny * nzc;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int x = int(c % g.nx);
        const int y = int((c / g.nx) % g.ny);
        const int z = z0 + int(c / (static_cast<long long>(g.nx) * g.ny));
        const T r = T(rho[c]);
        const T u[3] = {T(ux[c]), T(uy[c]), T(uz[c])};
        const T usqr = Cell<T, Q>::usqr_of(u);
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            origin[fill_pos<Q, i>(g, x, y, z, aa)] = Cell<T, Q>::template eq2<i>(r, u, usqr);
        });
    }
}

// Taylor-Green vortex state (cases.cpp:145-156) from host-evaluated per-index
// sin / cos / cos(2x) tables (glibc, as the reference), then equilibrium2<T>.
template <typename T, int Q>
__global__ void k_fill_tgv(T* origin, Geo g, const double* s1, const double* c1,
                           const double* c2, long long z_origin, double u_inf, int aa) {
    const long long n = static_cast<long long>(g.nx) * g.ny * g.nz;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int x = int(c % g.nx);
        const int y = int((c / g.nx) % g.ny);
        const int z = int(c / (static_cast<long long>(g.nx) * g.ny));
        const long long k = z_origin + z;
        const double dp = u_inf * u_inf / 16.0 * (c2[k] + 2.0) * (c2[x] + c2[y]);
        const double rho = 1.0 + dp / (1.0 / 3.0);
        const double ux = u_inf * s1[x] * c1[y] * c1[k];
        const double uy = -u_inf * c1[x] * s1[y] * c1[k];
        const T r = T(rho);
        const T u[3] = {T(ux), T(uy), T(0.0)};
        const T usqr = Cell<T, Q>::usqr_of(u);
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            origin[fill_pos<Q, i>(g, x, y, z, aa)] = Cell<T, Q>::template eq2<i>(r, u, usqr);
        });
    }
}

// Box copy between the padded layout of one direction and a dense buffer
// (x fastest). The box origin (bx0, by0, bz0) may be -1 (envelope).
// (sx, sy, sz) shifts the layout position (AA odd layout), wrapped on periodic axes.
template <typename TD, typename TS, bool TO_LAYOUT>
__global__ void k_box_copy(TD* dst, const TS* src, Geo g, int bx0, int by0, int bz0, int ex,
                           int ey, int ez, int sx = 0, int sy = 0, int sz = 0) {
    const long long n = static_cast<long long>(ex) * ey * ez;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int x = bx0 + int(c % ex);
        const int y = by0 + int((c / ex) % ey);
        const int z = bz0 + int(c / (static_cast<long long>(ex) * ey));
        const long long at = (sx | sy | sz) ? shifted(g, x, y, z, sx, sy, sz) : lin<TD>(g, x, y, z);
        if constexpr (TO_LAYOUT) dst[at] = TD(src[c]);
        else dst[c] = TD(src[at]);
    }
}

// Halo wait: block the stream until both neighbours finished the boundary
// planes of the step this slab completed last (flags[0] from the lower,
// flags[1] from the upper neighbour; flags[2] = own completed steps). Gives up
// after `timeout_ns` and raises flags[3] (reported as an exchange error).
__global__ void k_halo_wait(unsigned long long* flags, int have_lower, int have_upper,
                            unsigned long long timeout_ns) {
    if (*reinterpret_cast<volatile unsigned long long*>(flags + 3) != 0ull) return;  // already failed
    const unsigned long long target = flags[2];
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned long long lo = target, up = target;
        if (have_lower) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(lo) : "l"(flags));
        if (have_upper)
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(up) : "l"(flags + 1));
        if (lo >= target && up >= target) return;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) {
            flags[3] = target + 1;
            return;
        }
        __nanosleep(200);
    }
}

// Order-independent exact checksum of the canonical state: per direction
// S_i = sum over cells of bits(double(f_i) + 0.0) * (global cell index + 1)
// (mod 2^64). Integer sums commute, so the result does not depend on the
// reduction order, the slab decomposition or the layout (two-population / AA
// even / AA odd), and sums of slab checksums equal the monolithic one.
// skip (optional): per-slot flags; cells whose slot is flagged (NoDynamics)
// are left out (the masked porous sweep never writes them).
template <typename T, int Q>
__global__ void k_checksum(const T* origin0, Geo g, int aa_mode, long long z_origin, long long gnx,
                           long long gny, unsigned long long* out, const uint8_t* slot, int uniform_slot,
                           const uint8_t* skip) {
    using L = Lat<Q>;
    unsigned long long acc[Q];
    for (int i = 0; i < Q; ++i) acc[i] = 0ull;
    const long long n = static_cast<long long>(g.nx) * g.ny * g.nz;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        if (skip != nullptr && skip[slot ? slot[c] : uniform_slot]) continue;
        const int x = int(c % g.nx);
        const int y = int((c / g.nx) % g.ny);
        const int z = int(c / (static_cast<long long>(g.nx) * g.ny));
        const unsigned long long w = static_cast<unsigned long long>(((z_origin + z) * gny + y) * gnx + x) + 1ull;
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
            long long at;
            int dir = i;
            if (aa_mode == 2) at = shifted(g, x, y, z, cx, cy, cz);          // AA odd layout
            else {
                at = static_cast<long long>(z) * g.plane + static_cast<long long>(y) * g.pitch + x;
                if (aa_mode == 1) dir = opp_of(i);                              // AA even layout
            }
            const double v = double(origin0[dir * g.dstride + at]) + 0.0;
            acc[i] += static_cast<unsigned long long>(__double_as_longlong(v)) * w;
        });
    }
    for (int i = 0; i < Q; ++i) {
        unsigned long long v = acc[i];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) atomicAdd(out + i, v);
    }
}

// MultiBlockRun::gather_macroscopic (multiblock.cpp:443-484): populations
// converted to double; Collide cells report compute_rho_u, moving walls their
// (T-cast) wall velocity with rho = 1, other cells rho = 1, u = 0.
template <typename T, int Q>
__global__ void k_macro(const T* origin0, Geo g, int aa_mode, const uint8_t* slot, int uniform_slot,
                        const MacroSlot* ms, int z0, int nzc, double* rho, double* ux, double* uy,
                        double* uz) {
    const long long n = static_cast<long long>(g.nx) * g.ny * nzc;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int x = int(c % g.nx);
        const int y = int((c / g.nx) % g.ny);
        const int z = z0 + int(c / (static_cast<long long>(g.nx) * g.ny));
        const int s = slot ? slot[(static_cast<long long>(z) * g.ny + y) * g.nx + x] : uniform_slot;
        double r = 1.0, u[3] = {0.0, 0.0, 0.0};
        if (ms[s].kind == KIND_COLLIDE) {
            double f[Q];
            sfor<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                f[i] = double(canon_load<T, Q, i>(origin0, g, x, y, z, aa_mode));
            });
            Cell<double, Q>::rho_u(f, r, u);
        } else if (ms[s].kind == KIND_MBB) {
            u[0] = ms[s].uw[0];
            u[1] = ms[s].uw[1];
            u[2] = ms[s].uw[2];
        }
        rho[c] = r;
        ux[c] = u[0];
        uy[c] = u[1];
        uz[c] = u[2];
    }
}

// Device refresh_envelope_periodic (accelerated_lattice.cpp:202-238): every
// envelope cell whose out-of-range coordinates all lie on periodic axes gets
// the value of its periodic image (edges and corners included).
template <typename T>
__global__ void k_refresh_envelope(T* origin0, Geo g, int q) {
    const long long ex = g.nx + 2, ey = g.ny + 2, ez = g.nz + 2;
    const long long n = ex * ey * ez;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        int x = int(c % ex) - 1, y = int((c / ex) % ey) - 1, z = int(c / (ex * ey)) - 1;
        const bool env = x < 0 || x >= g.nx || y < 0 || y >= g.ny || z < 0 || z >= g.nz;
        if (!env) continue;
        int X = x, Y = y, Z = z;
        if (X < 0 || X >= g.nx) { if (!g.per_x) continue; X = X < 0 ? X + g.nx : X - g.nx; }
        if (Y < 0 || Y >= g.ny) { if (!g.per_y) continue; Y = Y < 0 ? Y + g.ny : Y - g.ny; }
        if (Z < 0 || Z >= g.nz) { if (!g.per_z) continue; Z = Z < 0 ? Z + g.nz : Z - g.nz; }
        const long long dst = static_cast<long long>(z) * g.plane + static_cast<long long>(y) * g.pitch + x;
        const long long src = static_cast<long long>(Z) * g.plane + static_cast<long long>(Y) * g.pitch + X;
        for (int i = 0; i < q; ++i) origin0[i * g.dstride + dst] = origin0[i * g.dstride + src];
    }
}

// Host-block pipeline: the x / y envelope cells of host planes [p0, p1) of the
// input mirror into the output mirror (blockIdx.y = direction * planes + plane),
// so the whole-plane copy-back hands the caller's envelope back unchanged
// instead of stale mirror memory (the kernels write interior cells only).
template <typename T>
__global__ void k_carry_envelope_xy(const T* __restrict__ din, T* __restrict__ dout, long long vol, int pitch,
                                    int plane, int nx, int ny, int p0, int np) {
    const int i = int(blockIdx.y) / np, p = p0 + int(blockIdx.y) % np;
    const int per = 2 * pitch + 2 * ny;  // rows y = 0 and y = ny + 1, then x = 0 / nx + 1 of rows 1..ny
    for (int k = int(blockIdx.x * blockDim.x + threadIdx.x); k < per; k += int(gridDim.x * blockDim.x)) {
        int x, y;
        if (k < 2 * pitch) {
            y = k < pitch ? 0 : ny + 1;
            x = k < pitch ? k : k - pitch;
        } else {
            const int r = k - 2 * pitch;
            y = 1 + (r >> 1);
            x = (r & 1) ? nx + 1 : 0;
        }
        const long long at = i * vol + static_cast<long long>(p) * plane + static_cast<long long>(y) * pitch + x;
        dout[at] = din[at];
    }
}

int grid_for(long long n) {
    long long b = (n + 255) / 256;
    return int(std::min<long long>(std::max<long long>(b, 1), 148LL * 32));
}

const KernelEntry* find_kernel(int arith, int bits, int q, unsigned km, int layout) {
    int n = 0;
    const KernelEntry* t = arith == DLB_ARITH_FAST ? fast::kernel_table(&n) : exact::kernel_table(&n);
    const KernelEntry* best = nullptr;
    for (int k = 0; k < n; ++k) {
        const KernelEntry& e = t[k];
        if (e.precision_bits != bits || e.q != q || e.layout != layout || e.minb != 0) continue;
        constexpr unsigned variant = KM_SKIP | KM_KE | KM_XREC;
        if ((e.km & km) != km || (e.km & variant) != (km & variant)) continue;
        if (!best || __builtin_popcount(e.km) < __builtin_popcount(best->km)) best = &e;
    }
    return best;
}

template <typename T>
DevRecipe<T> compile_recipe(const DynamicsChain& ch) {
    // compile_chain<T> (chain.hpp:147-187): parameters cast to T; the TRT odd
    // rate derived in double from the T-cast values (chain.hpp:132-135).
    DevRecipe<T> r{};
    const ChainParams& p = ch.params;
    r.omega = T(p.omega);
    r.lambda = T(p.lambda);
    r.smagorinsky_c = T(p.smagorinsky_c);
    r.omega_bulk_ho = T(p.omega_bulk_ho);
    r.target_rho = T(p.target_rho);
    for (int a = 0; a < 3; ++a) r.wall_velocity[a] = T(p.wall_velocity[a]);
    r.omega_minus = T(derive_omega_minus(double(r.omega), double(r.lambda)));
    r.kind = KIND_NODYN;
    for (const ChainLink& l : ch.links) {
        switch (l.type) {
            case LinkType::NoDynamics: r.kind = KIND_NODYN; break;
            case LinkType::BounceBack: r.kind = KIND_BB; break;
            case LinkType::MovingBounceBack: r.kind = KIND_MBB; break;
            case LinkType::BGK: r.kind = KIND_COLLIDE; r.base = BASE_BGK; break;
            case LinkType::TRT: r.kind = KIND_COLLIDE; r.base = BASE_TRT; break;
            case LinkType::RR: r.kind = KIND_COLLIDE; r.base = BASE_RR; break;
            case LinkType::Smagorinsky: r.has_les = 1; break;
            case LinkType::RegularizedVelocity:
            case LinkType::RegularizedPressure:
                r.has_reg = 1;
                r.reg_is_pressure = l.type == LinkType::RegularizedPressure;
                r.reg_axis = l.axis;
                r.reg_orient = l.orient;
                break;
        }
    }
    return r;
}

unsigned kind_bits(const DynamicsChain& ch) {
    unsigned km = 0;
    for (const ChainLink& l : ch.links) {
        switch (l.type) {
            case LinkType::NoDynamics: km |= KM_NODYN; break;
            case LinkType::BounceBack: km |= KM_BB; break;
            case LinkType::MovingBounceBack: km |= KM_MBB; break;
            case LinkType::BGK: km |= KM_BGK; break;
            case LinkType::TRT: km |= KM_TRT; break;
            case LinkType::RR: km |= KM_RR; break;
            case LinkType::Smagorinsky: km |= KM_LES; break;
            case LinkType::RegularizedVelocity: km |= KM_REGV; break;
            case LinkType::RegularizedPressure: km |= KM_REGP; break;
        }
    }
    return km;
}

}  // namespace

// ---------------------------------------------------------------------------

Lattice::Lattice(const dlb_lattice_desc& desc, const DynamicsRegistry& reg) : d_(desc) {
    if (d_.q != 19 && d_.q != 27) throw std::invalid_argument("q must be 19 or 27");
    if (d_.precision_bits != 32 && d_.precision_bits != 64)
        throw std::invalid_argument("precision must be 32 or 64");
    if (d_.layout != DLB_LAYOUT_TWO_POP && d_.layout != DLB_LAYOUT_AA)
        throw std::invalid_argument("layout must be DLB_LAYOUT_TWO_POP or DLB_LAYOUT_AA");
    if (d_.arith != DLB_ARITH_EXACT && d_.arith != DLB_ARITH_FAST)
        throw std::invalid_argument("arith must be DLB_ARITH_EXACT or DLB_ARITH_FAST");
    for (int a = 0; a < 3; ++a)
        if (d_.dims[a] < 1) throw std::invalid_argument("block extents must be >= 1");
    if (d_.global_nz < d_.dims[2] || d_.z_origin < 0 || d_.z_origin + d_.dims[2] > d_.global_nz)
        throw std::invalid_argument("slab z range outside the global domain");
    if (reg.num_instances() > kMaxInstances)
        throw std::invalid_argument("registry holds " + std::to_string(reg.num_instances()) +
                                    " instances; the per-cell u8 slot array addresses at most " +
                                    std::to_string(kMaxInstances));
    xrec_ = reg.num_instances() > kMaxSlots;
    for (int s = 0; s < reg.num_instances(); ++s) {
        chains_.push_back(reg.chain_at_slot(s));
        tag_of_slot_.push_back(reg.tag_of_slot(s));
    }
    for (int t = 0; t < reg.num_tags(); ++t) tag_names_.push_back(reg.chain_for(t));

    device_ = d_.device;
    graph_version_ = g_graph_version.fetch_add(1);
    DeviceGuard dg(device_);
    cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    {
        // z-slab halo work (wait + boundary planes + peer push) runs on a
        // high-priority stream beside the interior launch
        int lo = 0, hi = 0;
        cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
        cuda_check(cudaStreamCreateWithPriority(&halo_stream_, cudaStreamNonBlocking, hi), "cudaStreamCreate");
        cuda_check(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&ev_wait_, cudaEventDisableTiming), "cudaEventCreate");
        trace_halo_ = std::getenv("DLB_TRACE_HALO") != nullptr;
        const char* oe = std::getenv("DLB_HALO_OVERLAP");
        overlap_ = !(oe && oe[0] == '0');
        const char* te = std::getenv("DLB_HALO_TIMEOUT_MS");
        if (te && std::atof(te) > 0) halo_timeout_ns_ = static_cast<unsigned long long>(std::atof(te) * 1e6);
    }
    cuda_check(cudaEventCreate(&ev0_), "cudaEventCreate");
    cuda_check(cudaEventCreate(&ev1_), "cudaEventCreate");
    if (const char* fg = std::getenv("DLB_L2_FETCH")) {
        // L2 fetch granularity hint (bytes; tuning experiment for the sector-
        // scattered porous sweep)
        cuda_check(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, std::size_t(std::atoi(fg))), "L2 fetch limit");
    }

    const int s = d_.precision_bits / 8;
    align_ = 128 / s;
    {
        // masked porous sweep: skip granularity in bytes of one direction
        // array (default one 32-B sector; DLB_SKIP_GROUP_BYTES overrides, 4..128)
        const char* e = std::getenv("DLB_SKIP_GROUP_BYTES");
        int gb = e ? std::atoi(e) : 32;
        gb = std::min(128, std::max(int(s), gb));
        int g = 1;
        while (g * 2 <= std::min(32, gb / int(s))) g *= 2;
        skip_group_ = g;
    }
    const long long nx = d_.dims[0], ny = d_.dims[1], nz = d_.dims[2];
    const long long pitch = (nx + 2 + align_ - 1) / align_ * align_;
    const long long plane = pitch * (ny + 2);
    const long long dstride = plane * (nz + 2) + align_;  // + align: room for x = -1 of row 0
    if (plane * (nz + 2) + 2 * align_ > (1LL << 31) - 1)
        throw std::invalid_argument("slab too large for 32-bit in-array offsets");
    geo_.nx = int(nx);
    geo_.ny = int(ny);
    geo_.nz = int(nz);
    geo_.pitch = int(pitch);
    geo_.plane = int(plane);
    geo_.dstride = dstride;
    geo_.per_x = d_.periodic[0] != 0;
    geo_.per_y = d_.periodic[1] != 0;
    geo_.per_z = d_.periodic[2] != 0 && !split();
    base_off_ = align_ + plane + pitch;  // interior (0,0,0)

    const std::size_t bytes = std::size_t(d_.q) * std::size_t(dstride) * std::size_t(s);
    const int nbuf = d_.layout == DLB_LAYOUT_AA ? 1 : 2;
    for (int b = 0; b < nbuf; ++b) {
        cuda_check(cudaMalloc(&buf_[b], bytes), "cudaMalloc populations");
        cuda_check(cudaMemsetAsync(buf_[b], 0, bytes, stream_), "cudaMemset populations");
    }
    if (nbuf == 1) buf_[1] = buf_[0];
    device_bytes_ = int64_t(nbuf * bytes);
    cuda_check(cudaMalloc(&d_flags_, 4 * sizeof(unsigned long long)), "cudaMalloc flags");
    cuda_check(cudaMemsetAsync(d_flags_, 0, 4 * sizeof(unsigned long long), stream_), "memset");
    cuda_check(cudaMalloc(&d_counter_, sizeof(unsigned int)), "cudaMalloc counter");
    cuda_check(cudaMemsetAsync(d_counter_, 0, sizeof(unsigned int), stream_), "memset");
    staging_bytes_ = kStagingBytes;
    cuda_check(cudaMalloc(&staging_, staging_bytes_), "cudaMalloc staging");
    if (xrec_) {
        // the whole recipe table in global memory for the KM_XREC kernels
        const std::size_t rb = d_.precision_bits == 64 ? sizeof(DevRecipe<double>) : sizeof(DevRecipe<float>);
        std::vector<uint8_t> host(rb * chains_.size());
        for (std::size_t k = 0; k < chains_.size(); ++k) {
            if (d_.precision_bits == 64) {
                const DevRecipe<double> r = compile_recipe<double>(chains_[k]);
                std::memcpy(host.data() + k * rb, &r, rb);
            } else {
                const DevRecipe<float> r = compile_recipe<float>(chains_[k]);
                std::memcpy(host.data() + k * rb, &r, rb);
            }
        }
        cuda_check(cudaMalloc(&d_xrec_, host.size()), "cudaMalloc recipes");
        cuda_check(cudaMemcpy(d_xrec_, host.data(), host.size(), cudaMemcpyHostToDevice), "upload recipes");
    }
    setup_tma();
    cuda_check(cudaStreamSynchronize(stream_), "init");
}

Lattice::~Lattice() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    if (halo_stream_) cudaStreamSynchronize(halo_stream_);
    if (stream_) cudaStreamSynchronize(stream_);
    invalidate_graph();
    for (Peer* p : {&lower_, &upper_})
        for (void* v : p->ipc_opened) cudaIpcCloseMemHandle(v);
    cudaFree(buf_[0]);
    if (buf_[1] != buf_[0]) cudaFree(buf_[1]);
    cudaFree(d_slot_);
    cudaFree(d_list_);
    cudaFree(d_seg_);
    cudaFree(d_fseg_);
    cudaFree(d_flink_);
    cudaFree(d_bbfin_);
    cudaFree(d_ke_);
    cudaFree(d_fix_);
    cudaFree(d_tmap_);
    cudaFree(d_xrec_);
    free_compact();
    cudaFree(d_flags_);
    cudaFree(d_counter_);
    cudaFree(staging_);
    cudaFree(blk_out_);
    cudaFree(d_uprev_);
    cudaFree(diag_buf_);
    for (cudaEvent_t e : blk_ev_) cudaEventDestroy(e);
    if (copy_stream_) cudaStreamDestroy(copy_stream_);
    if (h2d_stream_) cudaStreamDestroy(h2d_stream_);
    if (ev0_) cudaEventDestroy(ev0_);
    if (ev1_) cudaEventDestroy(ev1_);
    for (cudaEvent_t e : trace_ev_) cudaEventDestroy(e);
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (ev_wait_) cudaEventDestroy(ev_wait_);
    if (halo_stream_) cudaStreamDestroy(halo_stream_);
    if (stream_) cudaStreamDestroy(stream_);
    if (prev >= 0) cudaSetDevice(prev);
}

void* Lattice::origin(int which) const {
    return static_cast<char*>(buf_[which]) + base_off_ * (d_.precision_bits / 8);
}

int64_t Lattice::bytes_per_cell() const {
    // populations read once + written once; the u8 slot read when not uniform
    return int64_t(2) * d_.q * (d_.precision_bits / 8) + (d_slot_ ? 1 : 0);
}

int64_t Lattice::step_bytes() const {
    if (sparse_) return step_bytes_;
    if (dense_seg_ && !(lower_.linked || upper_.linked)) return bytes_per_cell() * cells();  // no list read
    if (kernel_segbb_ && !(lower_.linked || upper_.linked))  // listed cells: populations, slot, link mask; 4 B / segment
        return (int64_t(2) * d_.q * (d_.precision_bits / 8) + 1 + 4) * fseg_cells_ + 4 * nfseg_;
    if (kernel_seg_ && !(lower_.linked || upper_.linked))  // listed cells + their slot bytes + 4 B per segment
        return (int64_t(2) * d_.q * (d_.precision_bits / 8) + 1) * masked_cells_ + 4 * nseg_;
    if ((km_needed_ & KM_SKIP) && masked_cells_ >= 0)
        return int64_t(2) * d_.q * (d_.precision_bits / 8) * masked_cells_ + (d_slot_ ? cells() : 0);
    return bytes_per_cell() * cells();
}

int Lattice::launches_per_step() const {
    if (sparse_) return int(lists_.size());
    const bool linked = lower_.linked || upper_.linked;
    if (kernel_cmp_ && !linked) return 1 + (kernel_cmp_fix_ ? 1 : 0);
    if (kernel_seg_ && seg_fused_reg_ && !linked) return 1;
    if (!linked) return 1 + ((kernel_main_ && !fixups_.empty()) ? int(fixups_.size()) : 0);
    return 1 + 1 + (geo_.nz > 2 ? 1 : 0);  // wait + boundary + interior
}

void Lattice::set_periodic_override(bool x, bool y, bool z) {
    invalidate_graph();
    envelope_valid_ = false;
    geo_.per_x = x;
    geo_.per_y = y;
    geo_.per_z = z;
}

void Lattice::set_slots(const int32_t* slots) {
    DeviceGuard dg(device_);
    invalidate_graph();
    const long long n = cells();
    std::vector<uint8_t> u8(std::size_t(n), 0);
    std::vector<char> seen(chains_.size(), 0);
    untagged_ = false;
    int first = -2;
    bool uniform = true;
    for (long long c = 0; c < n; ++c) {
        const int32_t s = slots[c];
        if (s < 0) {
            untagged_ = true;
            uniform = false;
            continue;
        }
        if (s >= int32_t(chains_.size()))
            throw std::invalid_argument("slot " + std::to_string(s) + " is not registered");
        seen[std::size_t(s)] = 1;
        u8[std::size_t(c)] = uint8_t(s);
        if (first == -2) first = s;
        else if (s != first) uniform = false;
    }
    present_slots_.clear();
    for (std::size_t s = 0; s < seen.size(); ++s)
        if (seen[s]) present_slots_.push_back(int32_t(s));
    cudaFree(d_slot_);
    d_slot_ = nullptr;
    masked_cells_ = -1;
    free_compact();
    if ((d_.flags & (DLB_FLAG_SKIP_NODYNAMICS | DLB_FLAG_SPARSE_LISTS)) && !aa()) {
        // cells the masked sweep moves: x-aligned groups of skip_group_ cells
        // that hold at least one non-NoDynamics cell (k_pull KM_SKIP rule)
        std::vector<uint8_t> nodyn(chains_.size(), 0);
        for (std::size_t k = 0; k < chains_.size(); ++k) nodyn[k] = kind_bits(chains_[k]) == KM_NODYN;
        if (!untagged_) check_skip_precondition(u8, nodyn);
        const int G = skip_group_;
        const long long nsx = (geo_.nx + G - 1) / G;
        // compacted segment list for the single-slab masked sweep (k_seg)
        const char* ce = std::getenv("DLB_MASKED_COMPACT");
        const bool compact = !(ce && ce[0] == '0');
        const bool want_segs = compact && !split() && !(d_.flags & DLB_FLAG_SPARSE_LISTS) &&
                               (n / G) < (1LL << 32) - 1;
        std::vector<uint32_t> segs;
        long long moved = 0;
        // packed entries (segment | y << bs | z << (bs + by)) when they fit 32 bits
        auto bits = [](long long v) { int b = 0; while ((1LL << b) < v) ++b; return b; };
        const int bs = bits(nsx), by = bits(geo_.ny), bz = bits(geo_.nz);
        const char* pe = std::getenv("DLB_SEG_PACK");  // 0: linear entries decoded by division (tuning)
        seg_pack_ = (bs + by + bz <= 32 && bs < 32 && by < 32 && !(pe && pe[0] == '0')) ? (bs | (by << 8)) : 0;
        for (long long r = 0; r < n / geo_.nx; ++r) {
            const uint8_t* row = u8.data() + r * geo_.nx;
            const long long ry = r % geo_.ny, rz = r / geo_.ny;
            for (int x0 = 0; x0 < geo_.nx; x0 += G) {
                const int x1 = std::min(geo_.nx, x0 + G);
                bool any = untagged_;
                for (int x = x0; x < x1 && !any; ++x) any = !nodyn[row[x]];
                if (!any) continue;
                moved += x1 - x0;
                if (want_segs)
                    segs.push_back(seg_pack_ ? uint32_t(x0 / G) | uint32_t(ry << bs) | uint32_t(rz << (bs + by))
                                             : uint32_t(r * nsx + x0 / G));
            }
        }
        masked_cells_ = moved;
        cudaFree(d_seg_);
        d_seg_ = nullptr;
        nseg_ = 0;
        if (want_segs && !segs.empty() && !untagged_) {
            cuda_check(cudaMalloc(&d_seg_, segs.size() * sizeof(uint32_t)), "cudaMalloc segments");
            cuda_check(cudaMemcpy(d_seg_, segs.data(), segs.size() * sizeof(uint32_t), cudaMemcpyHostToDevice),
                       "upload segments");
            nseg_ = (long long)segs.size();
            build_fluid_segments(u8);
            build_compact(u8, nodyn);
        } else {
            build_fluid_segments({});
        }
    }
    sparse_ = (d_.flags & DLB_FLAG_SPARSE_LISTS) && !split() && !aa() && !(uniform && first >= 0) && !xrec_ &&
              !untagged_ && geo_.nx <= 8192 && geo_.ny <= 8192 && geo_.nz <= 4096;
    if (sparse_) {
        uniform_slot_ = 0;
        slots_set_ = true;
        build_lists(u8);
        // the list kernels carry their slot; the per-cell array serves the diagnostics
        cuda_check(cudaMalloc(&d_slot_, std::size_t(n)), "cudaMalloc slots");
        cuda_check(cudaMemcpy(d_slot_, u8.data(), std::size_t(n), cudaMemcpyHostToDevice), "upload slots");
        return;
    }
    build_fixups(u8);
    // Dense porous sweep (every cell, the reference's behaviour) with
    // regularized planes in fp64: the segment sweep over ALL segments runs it
    // at two cells per thread with the regularized cells inside (126 registers
    // either way), instead of the one-cell k_pull plus two fix-up list launches
    // that re-read every source line of those isolated cells.
    dense_seg_ = false;
    if (!(d_.flags & (DLB_FLAG_SKIP_NODYNAMICS | DLB_FLAG_SPARSE_LISTS)) && !split() && !aa() && !xrec_ &&
        !untagged_ && d_.precision_bits == 64 && !fixups_.empty()) {
        const char* de = std::getenv("DLB_DENSE_SEG");
        const long long nsx = (geo_.nx + skip_group_ - 1) / skip_group_;
        const long long nseg = (n / geo_.nx) * nsx;
        if (!(de && de[0] == '0') && nseg < (1LL << 32) - 1) {
            // no segment list: k_seg maps thread -> segment arithmetically
            cudaFree(d_seg_);
            d_seg_ = nullptr;
            nseg_ = nseg;
            masked_cells_ = n;
            dense_seg_ = true;
        }
    }
    if (uniform && first >= 0) {
        uniform_slot_ = first;
    } else {
        uniform_slot_ = 0;
        cuda_check(cudaMalloc(&d_slot_, std::size_t(n)), "cudaMalloc slots");
        cuda_check(cudaMemcpy(d_slot_, u8.data(), std::size_t(n), cudaMemcpyHostToDevice),
                   "upload slots");
    }
    slots_set_ = true;
    select_kernel();
}

// The masked / sparse porous sweeps never update NoDynamics cells, which is
// exact only when no collision (Collide-kind) cell pulls from one: the
// reference's porous setup guarantees it (a solid cell with a fluid neighbour
// is BounceBack, cases.cpp:239-249), and bounce-back cells only ever return a
// cell's own populations to it. Reject layouts that break it (within this
// slab; z neighbours in other slabs are not visible here).
void Lattice::check_skip_precondition(const std::vector<uint8_t>& u8, const std::vector<uint8_t>& nodyn) const {
    std::vector<uint8_t> collide(chains_.size(), 0);
    for (std::size_t k = 0; k < chains_.size(); ++k)
        collide[k] = (kind_bits(chains_[k]) & (KM_BGK | KM_TRT | KM_RR)) != 0;
    const int nx = geo_.nx, ny = geo_.ny, nz = geo_.nz, q = d_.q;
    const int* cx = q == 19 ? kCx19 : kCx27;
    const int* cy = q == 19 ? kCy19 : kCy27;
    const int* cz = q == 19 ? kCz19 : kCz27;
    const bool px = geo_.per_x, py = geo_.per_y, pz = d_.periodic[2] && !split();
    const int nw = std::max(1, std::min<int>(nz, int(std::thread::hardware_concurrency())));
    std::vector<long long> bad(std::size_t(nw), -1);
    std::vector<std::thread> th;
    for (int w = 0; w < nw; ++w)
        th.emplace_back([&, w] {
            for (int z = nz * w / nw; z < nz * (w + 1) / nw && bad[std::size_t(w)] < 0; ++z)
                for (int y = 0; y < ny; ++y)
                    for (int x = 0; x < nx; ++x) {
                        const long long c = (long long)(z * ny + y) * nx + x;
                        if (!collide[u8[std::size_t(c)]]) continue;
                        for (int i = 1; i < q; ++i) {
                            int X = x - cx[i], Y = y - cy[i], Z = z - cz[i];
                            if (X < 0 || X >= nx) { if (!px) continue; X = (X + nx) % nx; }
                            if (Y < 0 || Y >= ny) { if (!py) continue; Y = (Y + ny) % ny; }
                            if (Z < 0 || Z >= nz) { if (!pz) continue; Z = (Z + nz) % nz; }
                            if (nodyn[u8[std::size_t((long long)(Z * ny + Y) * nx + X)]]) {
                                bad[std::size_t(w)] = c;
                                return;
                            }
                        }
                    }
        });
    for (auto& t : th) t.join();
    for (long long c : bad)
        if (c >= 0)
            throw std::invalid_argument(
                "skipping NoDynamics cells needs every collision cell's neighbours to be non-NoDynamics "
                "(a solid cell next to fluid must bounce back, cases.cpp:239-249); cell " + std::to_string(c) +
                " of this slab pulls from a NoDynamics cell");
}

// Fluid-segment sweep (k_segbb, single slab, DLB_FLUID_SEGMENTS=1): the
// x-aligned segments holding a collision cell, a per-listed-cell mask of the
// links whose source is a bounce-back cell (read from the puller's own previous
// state instead), and the wall cells outside those segments that face a
// collision cell (brought up to date by k_bb_finalize before the state is
// read). Needs: no moving wall, no regularized cell next to a wall (its list
// fix-up pulls directly), registry within the parameter-space table.
void Lattice::build_fluid_segments(const std::vector<uint8_t>& u8) {
    cudaFree(d_fseg_);
    cudaFree(d_flink_);
    cudaFree(d_bbfin_);
    d_fseg_ = nullptr;
    d_flink_ = nullptr;
    d_bbfin_ = nullptr;
    nfseg_ = nbbfin_ = fseg_cells_ = 0;
    bb_prologue_ = true;
    cmp_valid_ = false;
    bb_dirty_ = false;
    // opt-in (DLB_FLUID_SEGMENTS=1): on c4 it writes 23 % fewer bytes but reads
    // 15 % more (the puller's own previous sector for every wall link), for the
    // same time as k_seg (profiles/r02_summary.md)
    const char* fe = std::getenv("DLB_FLUID_SEGMENTS");
    if (u8.empty() || !(fe && fe[0] == '1') || xrec_ || aa() || split()) return;
    const int nsl = int(chains_.size());
    std::vector<uint8_t> collide(std::size_t(nsl), 0), bb(std::size_t(nsl), 0), reg(std::size_t(nsl), 0);
    for (int k = 0; k < nsl; ++k) {
        const unsigned kb = kind_bits(chains_[std::size_t(k)]);
        if (kb & KM_MBB) return;
        collide[std::size_t(k)] = (kb & (KM_BGK | KM_TRT | KM_RR)) != 0;
        bb[std::size_t(k)] = kb == KM_BB;
        reg[std::size_t(k)] = (kb & (KM_REGV | KM_REGP)) != 0;
    }
    const int nx = geo_.nx, ny = geo_.ny, nz = geo_.nz, q = d_.q, G = skip_group_;
    if (nx > 8192 || ny > 8192 || nz > 4096) return;
    const int* cx = q == 19 ? kCx19 : kCx27;
    const int* cy = q == 19 ? kCy19 : kCy27;
    const int* cz = q == 19 ? kCz19 : kCz27;
    const bool px = geo_.per_x, py = geo_.per_y, pz = geo_.per_z;
    auto at = [&](int x, int y, int z, int* out) {  // neighbour (x, y, z) inside the lattice, wrapped
        if (x < 0 || x >= nx) { if (!px) return false; x = (x + nx) % nx; }
        if (y < 0 || y >= ny) { if (!py) return false; y = (y + ny) % ny; }
        if (z < 0 || z >= nz) { if (!pz) return false; z = (z + nz) % nz; }
        *out = u8[std::size_t((long long)(z * ny + y) * nx + x)];
        return true;
    };
    const long long nsx = (nx + G - 1) / G;
    const int nw = std::max(1, std::min<int>(nz, int(std::thread::hardware_concurrency())));
    struct Part {
        std::vector<uint32_t> segs, links;
        std::vector<unsigned long long> fin;
        long long cells = 0;
        bool bad = false;
    };
    std::vector<Part> part(static_cast<std::size_t>(nw));
    std::vector<std::thread> th;
    for (int w = 0; w < nw; ++w)
        th.emplace_back([&, w] {
            Part& P = part[std::size_t(w)];
            for (int z = nz * w / nw; z < nz * (w + 1) / nw && !P.bad; ++z)
                for (int y = 0; y < ny; ++y) {
                    const uint8_t* row = u8.data() + (long long)(z * ny + y) * nx;
                    for (int x0 = 0; x0 < nx; x0 += G) {
                        const int x1 = std::min(nx, x0 + G);
                        bool listed = false;
                        for (int x = x0; x < x1 && !listed; ++x) listed = collide[row[x]];
                        if (listed) {
                            P.segs.push_back(uint32_t((long long)(z * ny + y) * nsx + x0 / G));
                            P.cells += x1 - x0;
                        }
                        for (int x = x0; x < x0 + G; ++x) {
                            const int sl = x < nx ? row[x] : -1;
                            if (listed) {
                                unsigned mask = 0;
                                if (sl >= 0 && collide[std::size_t(sl)])
                                    for (int i = 1; i < q; ++i) {
                                        int nb;
                                        if (at(x - cx[i], y - cy[i], z - cz[i], &nb) && bb[std::size_t(nb)]) {
                                            if (reg[std::size_t(sl)]) P.bad = true;  // its list fix-up pulls directly
                                            mask |= 1u << i;
                                        }
                                    }
                                P.links.push_back(mask);
                            } else if (sl >= 0 && bb[std::size_t(sl)]) {
                                unsigned long long mask = 0;
                                for (int j = 1; j < q; ++j) {
                                    int nb;
                                    if (at(x + cx[j], y + cy[j], z + cz[j], &nb) && collide[std::size_t(nb)])
                                        mask |= 1ull << (j - 1);
                                }
                                if (mask)
                                    P.fin.push_back((unsigned long long)x | ((unsigned long long)y << 13) |
                                                    ((unsigned long long)z << 26) | (mask << 38));
                            }
                        }
                    }
                }
        });
    for (auto& t : th) t.join();
    std::vector<uint32_t> segs, links;
    std::vector<unsigned long long> fin;
    for (auto& P : part) {
        if (P.bad) return;
        segs.insert(segs.end(), P.segs.begin(), P.segs.end());
        links.insert(links.end(), P.links.begin(), P.links.end());
        fin.insert(fin.end(), P.fin.begin(), P.fin.end());
        fseg_cells_ += P.cells;
    }
    if (segs.empty() || segs.size() >= (1ull << 32) / std::size_t(G)) return;
    cuda_check(cudaMalloc(&d_fseg_, segs.size() * 4), "cudaMalloc fluid segments");
    cuda_check(cudaMemcpy(d_fseg_, segs.data(), segs.size() * 4, cudaMemcpyHostToDevice), "upload");
    cuda_check(cudaMalloc(&d_flink_, links.size() * 4), "cudaMalloc link masks");
    cuda_check(cudaMemcpy(d_flink_, links.data(), links.size() * 4, cudaMemcpyHostToDevice), "upload");
    if (!fin.empty()) {
        cuda_check(cudaMalloc(&d_bbfin_, fin.size() * 8), "cudaMalloc wall list");
        cuda_check(cudaMemcpy(d_bbfin_, fin.data(), fin.size() * 8, cudaMemcpyHostToDevice), "upload");
    }
    nfseg_ = (long long)segs.size();
    nbbfin_ = (long long)fin.size();
}

// Bring the wall cells the fluid-segment sweep skipped up to date (their
// collision-facing links) before anything reads the state.
void Lattice::finalize_walls() {
    scatter_compact();
    if (!bb_dirty_) return;
    DeviceGuard dg(device_);
    exact::launch_bb_finalize(d_.precision_bits, d_.q, origin(cur_), origin(1 - cur_), geo_, d_bbfin_, nbbfin_,
                              stream_);
    cuda_check(cudaGetLastError(), "k_bb_finalize");
    bb_dirty_ = false;
}

// Sparse porous lists (see k_list): cells grouped by slot in row-major order,
// NoDynamics dropped, wall cells tagged with their fluid-source links.
void Lattice::build_lists(const std::vector<uint8_t>& u8) {
    const int nx = geo_.nx, ny = geo_.ny, nz = geo_.nz, q = d_.q;
    const int nslots = int(chains_.size());
    std::vector<int> kind(static_cast<std::size_t>(nslots), 0);
    for (int s = 0; s < nslots; ++s) {
        const LinkType t = chains_[size_t(s)].links.back().type;
        kind[size_t(s)] = t == LinkType::NoDynamics ? KIND_NODYN
                        : t == LinkType::BounceBack ? KIND_BB
                        : t == LinkType::MovingBounceBack ? KIND_MBB : KIND_COLLIDE;
    }
    const int* cx = q == 19 ? kCx19 : kCx27;
    const int* cy = q == 19 ? kCy19 : kCy27;
    const int* cz = q == 19 ? kCz19 : kCz27;
    auto fluid = [&](int x, int y, int z) {
        if (x < 0 || x >= nx) { if (!geo_.per_x) return false; x = (x + nx) % nx; }
        if (y < 0 || y >= ny) { if (!geo_.per_y) return false; y = (y + ny) % ny; }
        if (z < 0 || z >= nz) { if (!geo_.per_z) return false; z = (z + nz) % nz; }
        return kind[u8[size_t((long long)(z * ny + y) * nx + x)]] == KIND_COLLIDE;
    };
    const int nw = std::max(1, std::min<int>(nz, int(std::thread::hardware_concurrency())));
    std::vector<std::vector<std::vector<unsigned long long>>> part(static_cast<std::size_t>(nw));
    for (auto& p : part) p.resize(static_cast<std::size_t>(nslots));
    std::vector<std::vector<int64_t>> bytes(static_cast<std::size_t>(nw), std::vector<int64_t>(1, 0));
    const int s = d_.precision_bits / 8;
    std::vector<std::thread> th;
    for (int w = 0; w < nw; ++w) {
        th.emplace_back([&, w] {
            for (int z = nz * w / nw; z < nz * (w + 1) / nw; ++z)
                for (int y = 0; y < ny; ++y)
                    for (int x = 0; x < nx; ++x) {
                        const int sl = u8[size_t((long long)(z * ny + y) * nx + x)];
                        const int k = kind[size_t(sl)];
                        if (k == KIND_NODYN) continue;
                        unsigned long long mask = 0;
                        if (k == KIND_BB || k == KIND_MBB) {
                            for (int i = 1; i < q; ++i)
                                if (fluid(x - cx[i], y - cy[i], z - cz[i])) mask |= 1ull << (i - 1);
                            if (!mask) continue;  // feeds no fluid cell
                            bytes[size_t(w)][0] += 2LL * __builtin_popcountll(mask) * s + 8;
                        } else {
                            bytes[size_t(w)][0] += 2LL * q * s + 8;
                        }
                        part[size_t(w)][size_t(sl)].push_back(
                            (unsigned long long)x | ((unsigned long long)y << 13) |
                            ((unsigned long long)z << 26) | (mask << 38));
                    }
        });
    }
    for (auto& t : th) t.join();
    std::vector<unsigned long long> all;
    lists_.clear();
    step_bytes_ = 0;
    for (int w = 0; w < nw; ++w) step_bytes_ += bytes[size_t(w)][0];
    present_slots_.clear();
    for (int sl = 0; sl < nslots; ++sl) {
        const long long off = (long long)all.size();
        for (int w = 0; w < nw; ++w)
            all.insert(all.end(), part[size_t(w)][size_t(sl)].begin(), part[size_t(w)][size_t(sl)].end());
        const long long cnt = (long long)all.size() - off;
        bool present = cnt > 0;
        if (!present) {  // still present for the dispatch check when any cell has it
            for (std::size_t c = 0; c < u8.size() && !present; ++c) present = u8[c] == sl;
        }
        if (present) present_slots_.push_back(sl);
        if (cnt == 0) continue;
        const int k = kind[size_t(sl)];
        const unsigned km = kind_bits(chains_[size_t(sl)]);
        const int layout = (k == KIND_BB || k == KIND_MBB) ? LAYOUT_LIST_MASKED : LAYOUT_LIST;
        const KernelEntry* e = find_kernel(d_.arith, d_.precision_bits, q, km, layout);
        if (!e) throw std::invalid_argument("no list kernel instantiation covers slot " + std::to_string(sl));
        lists_.push_back({sl, off, cnt, e});
    }
    std::sort(lists_.begin(), lists_.end(),
              [](const ListLaunch& a, const ListLaunch& b) { return a.count > b.count; });
    cudaFree(d_list_);
    d_list_ = nullptr;
    cuda_check(cudaMalloc(&d_list_, std::max<std::size_t>(1, all.size()) * 8), "cudaMalloc lists");
    cuda_check(cudaMemcpy(d_list_, all.data(), all.size() * 8, cudaMemcpyHostToDevice), "upload lists");
    kernel_ = lists_.empty() ? nullptr : lists_.front().kernel;
    if (!kernel_) kernel_ = find_kernel(d_.arith, d_.precision_bits, q, KM_BB, LAYOUT_LIST_MASKED);
}

void Lattice::build_fixups(const std::vector<uint8_t>& u8) {
    fixups_.clear();
    cudaFree(d_fix_);
    d_fix_ = nullptr;
    if (aa() || xrec_) return;
    if (const char* rs = std::getenv("DLB_RARE_SPLIT"))  // 0: regularized cells in the main sweep (tuning)
        if (rs[0] == '0') return;
    std::vector<char> reg(chains_.size(), 0);
    bool any = false;
    for (std::size_t s = 0; s < chains_.size(); ++s)
        for (const ChainLink& l : chains_[s].links)
            if (l.type == LinkType::RegularizedVelocity || l.type == LinkType::RegularizedPressure)
                reg[s] = 1, any = true;
    if (!any) return;
    std::vector<std::vector<unsigned long long>> per(chains_.size());
    for (int z = 0; z < geo_.nz; ++z)
        for (int y = 0; y < geo_.ny; ++y)
            for (int x = 0; x < geo_.nx; ++x) {
                const int sl = u8[std::size_t((long long)(z * geo_.ny + y) * geo_.nx + x)];
                if (reg[std::size_t(sl)])
                    per[std::size_t(sl)].push_back((unsigned long long)x | ((unsigned long long)y << 13) |
                                                   ((unsigned long long)z << 26));
            }
    std::vector<unsigned long long> all;
    for (std::size_t sl = 0; sl < per.size(); ++sl) {
        if (per[sl].empty()) continue;
        const KernelEntry* e =
            find_kernel(d_.arith, d_.precision_bits, d_.q, kind_bits(chains_[sl]), LAYOUT_LIST);
        if (!e) return;  // no list instantiation: keep the full dense kernel
        fixups_.push_back({int(sl), (long long)all.size(), (long long)per[sl].size(), e});
        all.insert(all.end(), per[sl].begin(), per[sl].end());
    }
    if (all.empty() || geo_.nx > 8192 || geo_.ny > 8192 || geo_.nz > 4096) {
        fixups_.clear();
        return;
    }
    cuda_check(cudaMalloc(&d_fix_, all.size() * 8), "cudaMalloc fixups");
    cuda_check(cudaMemcpy(d_fix_, all.data(), all.size() * 8, cudaMemcpyHostToDevice), "upload fixups");
}

// Tensor map of one population buffer as a 4-D tensor (x, y, z, direction).
// The base sits 16 B before interior x = 0 so that x = -1 .. nx are in range
// (needs pitch >= nx + 2 + 16 B / s).
void Lattice::setup_tma() {
    tma_ok_ = false;
    if (aa() || !(d_.flags & DLB_FLAG_TMA)) return;
    const int s = d_.precision_bits / 8;
    const int e = 16 / s;
    if (geo_.pitch < geo_.nx + 2 + e) return;
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
        cudaGetLastError();
        return;
    }
    const int bx = (s == 4 ? 64 : 32) + 2 * e, by = (s == 4 || d_.q == 27) ? 8 : 16;  // padded box (kernel: W x BY)
    for (int b = 0; b < 2; ++b) {
        char* base = static_cast<char*>(buf_[b]) + std::size_t(align_ - e) * s;
        const cuuint64_t dims[4] = {cuuint64_t(geo_.pitch), cuuint64_t(geo_.ny + 2), cuuint64_t(geo_.nz + 2),
                                    cuuint64_t(d_.q)};
        const cuuint64_t strides[3] = {cuuint64_t(geo_.pitch) * s, cuuint64_t(geo_.plane) * s,
                                       cuuint64_t(geo_.dstride) * s};
        const cuuint32_t box[4] = {cuuint32_t(bx), cuuint32_t(by), 1u, 1u};
        const cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
        const CUresult r = reinterpret_cast<EncodeFn>(fn)(
            &tmap_[b], s == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims,
            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return;
    }
    // Row-staged variant (k_tmarow, DLB_TMA_ROW != 0): the buffer as a 3-D
    // tensor (x, row = (z + 1)(ny + 2) + y + 1, direction), boxes of row_bw_ x 1 x 1
    // covering x = -e .. nx + e of one row in row_nb_ pieces.
    const char* re = std::getenv("DLB_TMA_ROW");
    row_ok_ = false;
    if (!(re && re[0] == '0') && geo_.pitch >= geo_.nx + e + 1) {
        // work unit = row_tw_ cells of one row, as many x-splits as it takes
        // for two ring stages to fit the per-CTA budget (DLB_TMAROW_SMEM_KB)
        const char* be = std::getenv("DLB_TMAROW_SMEM_KB");
        const std::size_t budget = std::size_t(be ? std::atoi(be) : 200) << 10;
        int splits = 1;
        auto tile_w = [&](int sp) { return ((geo_.nx + sp - 1) / sp + 31) / 32 * 32; };
        while (splits < 16 &&
               std::size_t(2) * d_.q * std::size_t(tile_w(splits) + 2 * (128 / s)) * s > budget)
            ++splits;
        row_tw_ = splits == 1 ? geo_.nx : tile_w(splits);
        const int span = row_tw_ + e + 1;
        // TMA shared-memory destinations must be 128-B aligned: box widths are
        // multiples of 128 B (elements past the row's pitch are zero-filled
        // out-of-bounds reads, no HBM traffic)
        const int al = 128 / s;
        row_nb_ = (span + 255) / 256;
        row_bw_ = ((span + row_nb_ - 1) / row_nb_ + al - 1) / al * al;
        if (row_bw_ > 256) row_bw_ = 256, row_nb_ = (span + 255) / 256;
        bool ok = true;
        for (int b = 0; b < 2 && ok; ++b) {
            char* base = static_cast<char*>(buf_[b]) + std::size_t(align_ - e) * s;
            const cuuint64_t dims[3] = {cuuint64_t(geo_.pitch), cuuint64_t(geo_.ny + 2) * cuuint64_t(geo_.nz + 2),
                                        cuuint64_t(d_.q)};
            const cuuint64_t strides[2] = {cuuint64_t(geo_.pitch) * s, cuuint64_t(geo_.dstride) * s};
            const cuuint32_t box[3] = {cuuint32_t(row_bw_), 1u, 1u};
            const cuuint32_t estr[3] = {1u, 1u, 1u};
            ok = reinterpret_cast<EncodeFn>(fn)(
                     &tmap_[2 + b], s == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                     base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
        row_ok_ = ok;
    }
    // Block-staged variant (k_tmablk; DLB_TMA_BLOCKS=0 disables): the same 3-D
    // tensor with 2-D boxes of 256 x R rows (R = 4 fp32, 2 fp64).
    blk_ok_ = false;
    const char* bke = std::getenv("DLB_TMA_BLOCKS");
    if (!(bke && bke[0] == '0') && geo_.pitch >= geo_.nx + e + 1) {
        const int R = s == 4 ? 4 : 2;  // rows per work unit (k_tmablk's R)
        bool ok = true;
        for (int b = 0; b < 2 && ok; ++b) {
            char* base = static_cast<char*>(buf_[b]) + std::size_t(align_ - e) * s;
            const cuuint64_t dims[3] = {cuuint64_t(geo_.pitch), cuuint64_t(geo_.ny + 2) * cuuint64_t(geo_.nz + 2),
                                        cuuint64_t(d_.q)};
            const cuuint64_t strides[2] = {cuuint64_t(geo_.pitch) * s, cuuint64_t(geo_.dstride) * s};
            const cuuint32_t box[3] = {256u, cuuint32_t(R), 1u};
            const cuuint32_t estr[3] = {1u, 1u, 1u};
            ok = reinterpret_cast<EncodeFn>(fn)(
                     &tmap_[4 + b], s == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                     base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
        blk_ok_ = ok;
    }
    cuda_check(cudaMalloc(&d_tmap_, 6 * sizeof(CUtensorMap)), "cudaMalloc tensor maps");
    cuda_check(cudaMemcpy(d_tmap_, tmap_, 6 * sizeof(CUtensorMap), cudaMemcpyHostToDevice), "tensor maps");
    tma_xoff_ = e;
    tma_ok_ = true;
}

void Lattice::refresh_envelope(int which) {
    const long long n = (long long)(geo_.nx + 2) * (geo_.ny + 2) * (geo_.nz + 2);
    const int grid = grid_for(n);
    if (d_.precision_bits == 64)
        k_refresh_envelope<double><<<grid, 256, 0, stream_>>>(static_cast<double*>(origin(which)), geo_, d_.q);
    else
        k_refresh_envelope<float><<<grid, 256, 0, stream_>>>(static_cast<float*>(origin(which)), geo_, d_.q);
    cuda_check(cudaGetLastError(), "k_refresh_envelope");
}

template <typename T>
void Lattice::launch_tma(StepArgs<T>& a, int parity) {
    const KernelEntry* k = kernel_tma_;
    const int e = int(16 / sizeof(T));
    if (k->layout == LAYOUT_TMABLK) {
        const int S = 2;
        const std::size_t stage = std::size_t(d_.q) * k->tile_y * 256 * sizeof(T);
        const std::size_t smem = std::size_t(S) * stage + std::size_t(2 * S) * 8 + 128;
        if (tma_grid_ == 0) {
            cuda_check(cudaFuncSetAttribute(k->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
                       "smem attr");
            int sms = 0, per_sm = 0;
            cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_), "sm count");
            cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k->fn, k->warps * 32 + 32, smem),
                       "occupancy");
            tma_grid_ = std::max(1, per_sm) * sms;
        }
        if (!envelope_valid_) refresh_envelope(parity);
        const CUtensorMap* map = d_tmap_ + 4 + parity;
        int ns = S;
        void* args[] = {&a, &map, &ns};
        cuda_check(cudaLaunchKernel(k->fn, dim3(unsigned(tma_grid_)), dim3(unsigned(k->warps * 32 + 32)), args, smem,
                                    stream_), "launch tma blocks");
        envelope_valid_ = true;
        return;
    }
    if (k->layout == LAYOUT_TMAROW) {
        const std::size_t stage = std::size_t(d_.q) * row_nb_ * row_bw_ * sizeof(T);
        // two ring stages per CTA by default (DLB_TMAROW_STAGES); one CTA of a
        // producer warp + 16 consumer warps (96 registers) per SM
        static const int stages_env = [] {
            const char* e = std::getenv("DLB_TMAROW_STAGES");
            return e ? std::max(2, std::atoi(e)) : 2;
        }();
        const int S = stages_env;
        const std::size_t smem = std::size_t(S) * stage + std::size_t(2 * S) * 8 + 128;
        if (tma_grid_ == 0) {
            cuda_check(cudaFuncSetAttribute(k->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
                       "smem attr");
            int sms = 0, per_sm = 0;
            cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_), "sm count");
            cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k->fn, k->warps * 32 + 32, smem),
                       "occupancy");
            tma_grid_ = std::max(1, per_sm) * sms;
        }
        if (!envelope_valid_) refresh_envelope(parity);
        const CUtensorMap* map = d_tmap_ + 2 + parity;
        int nb = row_nb_, bw = row_bw_, ns = S, tw = row_tw_;
        void* args[] = {&a, &map, &nb, &bw, &ns, &tw};
        cuda_check(cudaLaunchKernel(k->fn, dim3(unsigned(tma_grid_)), dim3(unsigned(k->warps * 32 + 32)), args, smem,
                                    stream_), "launch tma rows");
        envelope_valid_ = true;
        return;
    }
    const std::size_t smem = std::size_t(k->stages) * d_.q * (k->tile_x + 2 * e) * k->tile_y * sizeof(T) + 128;
    if (tma_grid_ == 0) {
        cuda_check(cudaFuncSetAttribute(k->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "smem attr");
        int per_sm = 0;
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k->fn, k->tile_x * k->tile_y + 32, smem),
                   "occupancy");
        int sms = 0;
        cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_), "sm count");
        tma_grid_ = std::max(1, per_sm) * sms;
    }
    if (!envelope_valid_) refresh_envelope(parity);
    const CUtensorMap* map = d_tmap_ + parity;
    int xoff = tma_xoff_;
    void* args[] = {&a, &map, &xoff};
    cuda_check(cudaLaunchKernel(k->fn, dim3(unsigned(tma_grid_)), dim3(unsigned(k->tile_x * k->tile_y + 32)), args,
                                smem, stream_), "launch tma");
    envelope_valid_ = true;  // the kernel pushed the periodic images into the output buffer
}

void Lattice::set_uniform_slot(int32_t slot) {
    DeviceGuard dg(device_);
    if (slot < 0 || slot >= int32_t(chains_.size()))
        throw std::invalid_argument("slot " + std::to_string(slot) + " is not registered");
    cudaFree(d_slot_);
    d_slot_ = nullptr;
    cudaFree(d_seg_);
    d_seg_ = nullptr;
    nseg_ = 0;
    build_fluid_segments({});
    // every per-cell structure of an earlier set_slots goes with it
    free_compact();
    dense_seg_ = false;
    fixups_.clear();
    cudaFree(d_fix_);
    d_fix_ = nullptr;
    sparse_ = false;
    lists_.clear();
    cudaFree(d_list_);
    d_list_ = nullptr;
    masked_cells_ = -1;
    uniform_slot_ = slot;
    untagged_ = false;
    present_slots_ = {slot};
    slots_set_ = true;
    select_kernel();
}

void Lattice::select_kernel() {
    invalidate_graph();
    // launch-shape knobs, read whenever the kernels are chosen (per lattice)
    {
        // segment sweep: entry prefetch distance in blocks (37-148 best on c4:
        // 27.6 vs 26.8 GLUPS without; DLB_SEG_PREFETCH, 0 = off)
        const char* pe = std::getenv("DLB_SEG_PREFETCH");
        seg_prefetch_ = pe ? std::max(0, std::atoi(pe)) : 74;
        // segment sweep threads per block: 64 for the every-segment dense sweep
        // (c4 dense 20.0 / 19.5 / 18.8 GLUPS at 64 / 128 / 256; 32 as 64), 256
        // for the masked one (27.6 vs 27.5 at 128, 27.2 at 64); DLB_SEG_BLOCK
        const char* be = std::getenv("DLB_SEG_BLOCK");
        const int b = be ? std::atoi(be) : 0;
        seg_block_ = (b == 32 || b == 64 || b == 128 || b == 256) ? b : (dense_seg_ ? 64 : 256);
    }
    kernel_ke_ = nullptr;
    ke_requested_ = false;
    if (sparse_) return;
    km_needed_ = xrec_ ? KM_XREC : 0u;
    for (int32_t s : present_slots_) km_needed_ |= kind_bits(chains_[std::size_t(s)]);
    if ((d_.flags & (DLB_FLAG_SKIP_NODYNAMICS | DLB_FLAG_SPARSE_LISTS)) && (km_needed_ & KM_NODYN) && !aa())
        km_needed_ |= KM_SKIP;
    {
        // dense / AA sweeps: 128-thread blocks for the low-occupancy sets -- the
        // same threads per SM as 256 (launch bounds are per 256 threads), but a
        // retiring block frees its SM slot at half the granularity: c2 14.4 ->
        // 14.9 GLUPS, c1 +1.8 %, c3 +0.6 %, AA c5 38.6 -> 40.8; the pure-BGK fp32
        // set (c5, 10 blocks of 128 per SM) keeps 256: +0.55 % under power
        // capping (40.82 vs 40.59 GLUPS), equal otherwise. DLB_PULL_THREADS
        const char* e = std::getenv("DLB_PULL_THREADS");
        const int v = e ? std::atoi(e) : 0;
        const bool light = d_.precision_bits == 32 && d_.q == 19 && !aa() &&
                           (km_needed_ & ~(KM_SKIP | KM_KE | KM_XREC)) == KM_BGK;
        pull_threads_ = (v == 64 || v == 128 || v == 256) ? v : (light ? 256 : 128);
    }
    if (aa()) {
        kernel_ = find_kernel(d_.arith, d_.precision_bits, d_.q, km_needed_, LAYOUT_AA);
        kernel_odd_ = find_kernel(d_.arith, d_.precision_bits, d_.q, km_needed_, LAYOUT_AA_ODD);
        if (kernel_ && kernel_odd_ && kernel_->km != kernel_odd_->km) kernel_odd_ = nullptr;
        if (!kernel_ || !kernel_odd_)
            throw std::invalid_argument("no AA kernel instantiation covers this dynamics set");
        // boundary planes of linked slabs: the face-crossing instantiations
        kernel_link_ = find_kernel(d_.arith, d_.precision_bits, d_.q, km_needed_, LAYOUT_AA_LINK);
        kernel_odd_link_ = find_kernel(d_.arith, d_.precision_bits, d_.q, km_needed_, LAYOUT_AA_ODD_LINK);
        if (!kernel_link_ || !kernel_odd_link_)
            throw std::invalid_argument("no linked AA kernel instantiation covers this dynamics set");
        return;
    }
    kernel_ = find_kernel(d_.arith, d_.precision_bits, d_.q, km_needed_, LAYOUT_TWO_POP);
    if (!kernel_) throw std::invalid_argument("no kernel instantiation covers this dynamics set");
    if (const char* mb = std::getenv("DLB_PULL_MINB")) {
        // occupancy-target variant of the same instantiation (tuning knob)
        int nt = 0;
        const KernelEntry* t = d_.arith == DLB_ARITH_FAST ? fast::kernel_table(&nt) : exact::kernel_table(&nt);
        for (int k = 0; k < nt; ++k)
            if (t[k].layout == LAYOUT_TWO_POP && t[k].km == kernel_->km && t[k].minb == std::atoi(mb) &&
                t[k].precision_bits == kernel_->precision_bits && t[k].q == kernel_->q)
                kernel_ = &t[k];
    }
    kernel_main_ = nullptr;
    if (!fixups_.empty())
        kernel_main_ = find_kernel(d_.arith, d_.precision_bits, d_.q, km_needed_ & ~(KM_REGV | KM_REGP),
                                   LAYOUT_TWO_POP);
    kernel_seg_ = nullptr;
    seg_fused_reg_ = false;
    if ((d_seg_ && (km_needed_ & KM_SKIP)) || dense_seg_) {
        unsigned km = km_needed_ & ~KM_SKIP;
        // the regularized cells stay in the segment sweep when it runs two
        // cells per thread (fp64): that instantiation has the same 126
        // registers with or without them, and the separate fix-up launches
        // re-read every source line of those isolated cells
        const char* fr = std::getenv("DLB_SEG_FUSE_REG");
        const char* ce0 = std::getenv("DLB_SEG_CPT");
        const int cpt0 = ce0 ? std::atoi(ce0) : (d_.precision_bits == 64 ? 2 : 1);
        const char* fs = std::getenv("DLB_FLUID_SEGMENTS");  // k_segbb has no regularized sets
        seg_fused_reg_ = kernel_main_ && cpt0 == 2 && !(fr && fr[0] == '0') && !(fs && fs[0] == '1');
        if (kernel_main_ && !seg_fused_reg_) km &= ~(KM_REGV | KM_REGP);
        kernel_seg_ = find_kernel(d_.arith, d_.precision_bits, d_.q, km, LAYOUT_SEG);
        // cells per thread of the segment sweep (DLB_SEG_CPT): 2 for fp64
        // (c4: 24.96 vs 23.76 GLUPS, profiles/r01_summary.md), 1 for fp32
        const char* ce = std::getenv("DLB_SEG_CPT");
        const int cpt = ce ? std::atoi(ce) : (d_.precision_bits == 64 ? 2 : 1);
        const char* me = std::getenv("DLB_SEG_MINB");  // occupancy-target variant (tuning)
        const int minb = me ? std::atoi(me) : 0;
        if (kernel_seg_ && (kernel_seg_->cpt != cpt || minb)) {
            int nt = 0;
            const KernelEntry* t = d_.arith == DLB_ARITH_FAST ? fast::kernel_table(&nt) : exact::kernel_table(&nt);
            for (int k = 0; k < nt; ++k)
                if (t[k].layout == LAYOUT_SEG && t[k].km == kernel_seg_->km && t[k].cpt == cpt &&
                    t[k].minb == minb && t[k].precision_bits == kernel_seg_->precision_bits &&
                    t[k].q == kernel_seg_->q)
                    kernel_seg_ = &t[k];
        }
    }
    kernel_cmp_ = kernel_cmp_fix_ = nullptr;
    if (kernel_seg_ && d_cseg_) {
        // compacted sweep: the main set without the regularized kinds (they run
        // as the FIX list with the full set), cells per thread as k_seg
        unsigned km = km_needed_ & ~KM_SKIP;
        const bool reg = (km & (KM_REGV | KM_REGP)) != 0;
        if (reg) km &= ~(KM_REGV | KM_REGP);
        const int cpt = kernel_seg_->cpt;
        int nt = 0;
        const KernelEntry* t = d_.arith == DLB_ARITH_FAST ? fast::kernel_table(&nt) : exact::kernel_table(&nt);
        const KernelEntry* best = nullptr;
        for (int k = 0; k < nt; ++k) {
            const KernelEntry& e = t[k];
            if (e.layout != LAYOUT_CMP || e.precision_bits != d_.precision_bits || e.q != d_.q) continue;
            if ((e.km & km) != km || (e.km & KM_XREC)) continue;
            const bool better = !best || __builtin_popcount(e.km) < __builtin_popcount(best->km) ||
                                (__builtin_popcount(e.km) == __builtin_popcount(best->km) && e.cpt == cpt);
            if (better) best = &e;
        }
        const KernelEntry* fix = reg ? find_kernel(d_.arith, d_.precision_bits, d_.q, km_needed_ & ~KM_SKIP,
                                                   LAYOUT_CMP_FIX) : nullptr;
        if (best && (!reg || (fix && ncfix_ > 0))) {
            kernel_cmp_ = best;
            kernel_cmp_fix_ = reg ? fix : nullptr;
        }
    }
    kernel_segbb_ = nullptr;
    if (kernel_seg_ && d_fseg_) {
        int nt = 0;
        const KernelEntry* t = d_.arith == DLB_ARITH_FAST ? fast::kernel_table(&nt) : exact::kernel_table(&nt);
        for (int k = 0; k < nt; ++k)
            if (t[k].layout == LAYOUT_SEGBB && t[k].km == kernel_seg_->km && t[k].cpt == kernel_seg_->cpt &&
                t[k].precision_bits == kernel_seg_->precision_bits && t[k].q == kernel_seg_->q)
                kernel_segbb_ = &t[k];
    }
    // fused kinetic-energy variant of the dense sweep (exact mode, single
    // two-population slab, no regularized fix-ups): used for the steps a
    // kinetic-energy reduction is requested for (request_kinetic)
    kernel_ke_ = nullptr;
    if (!aa() && !split() && fixups_.empty() && !(km_needed_ & KM_SKIP) && d_.arith == DLB_ARITH_EXACT)
        kernel_ke_ = find_kernel(d_.arith, d_.precision_bits, d_.q, km_needed_ | KM_KE, LAYOUT_TWO_POP);
    // persistent cooperative sweep for small single-slab lattices (whole call
    // in one launch). Opt-in (DLB_COOP_MAX_CELLS = largest lattice, default 0):
    // config 1 runs 11.6 vs 12.5 us per step over 1000 steps but 14.7 vs 12.7
    // over 100 (cooperative launch cost), profiles/r01_summary.md
    kernel_coop_ = nullptr;
    coop_grid_ = 0;
    {
        const char* ce = std::getenv("DLB_COOP_MAX_CELLS");
        const long long maxc = ce ? std::atoll(ce) : 0;
        if (cells() <= maxc && !aa() && !split() && fixups_.empty() && !(km_needed_ & KM_SKIP))
            kernel_coop_ = find_kernel(d_.arith, d_.precision_bits, d_.q, km_needed_, LAYOUT_COOP);
    }
    // 128-bit vectorised dense sweep (opt-in): unlinked single slabs whose rows
    // hold whole 16-B vectors, plain dispatch sets
    kernel_vec_ = nullptr;
    if (const char* ve = std::getenv("DLB_VEC")) {
        const int vw = 16 / (d_.precision_bits / 8);
        if (ve[0] == '1' && !aa() && !split() && fixups_.empty() && !(km_needed_ & (KM_SKIP | KM_XREC)) &&
            geo_.nx % vw == 0)
            kernel_vec_ = find_kernel(d_.arith, d_.precision_bits, d_.q, km_needed_, LAYOUT_VEC);
    }
    kernel_tma_ = nullptr;
    tma_grid_ = 0;
    if (tma_ok_ && fixups_.empty() && !(km_needed_ & KM_SKIP)) {
        const std::size_t stage = std::size_t(d_.q) * row_nb_ * row_bw_ * std::size_t(d_.precision_bits / 8);
        // uniform lattices: 2-D block boxes (c5 0.84-0.85 vs 0.79-0.82 for rows); with a
        // slot array the row kernel wins (its slot reads hide behind 2 CTAs per SM)
        if (blk_ok_ && !d_slot_) {
            kernel_tma_ = find_kernel(d_.arith, d_.precision_bits, d_.q, km_needed_, LAYOUT_TMABLK);
        }
        if (!kernel_tma_ && row_ok_ && 2 * stage <= (std::size_t(200) << 10)) {
            kernel_tma_ = find_kernel(d_.arith, d_.precision_bits, d_.q, km_needed_, LAYOUT_TMAROW);
            // rows short enough for two 2-stage CTAs per SM: 8 consumer warps each
            // (c3 512-wide rows: 0.75 vs 0.55 of copy bandwidth with one 16-warp CTA)
            const char* se = std::getenv("DLB_TMAROW_STAGES");
            const std::size_t ring = std::size_t(se ? std::max(2, std::atoi(se)) : 2) * stage + 1024;
            const int want = 2 * ring <= (std::size_t(220) << 10) ? 8 : 16;
            if (kernel_tma_ && kernel_tma_->warps != want) {
                int nt = 0;
                const KernelEntry* t = d_.arith == DLB_ARITH_FAST ? fast::kernel_table(&nt) : exact::kernel_table(&nt);
                for (int k = 0; k < nt; ++k)
                    if (t[k].layout == LAYOUT_TMAROW && t[k].km == kernel_tma_->km && t[k].warps == want &&
                        t[k].precision_bits == kernel_tma_->precision_bits && t[k].q == kernel_tma_->q)
                        kernel_tma_ = &t[k];
            }
        }
        if (!kernel_tma_) kernel_tma_ = find_kernel(d_.arith, d_.precision_bits, d_.q, km_needed_, LAYOUT_TMA);
    }
}

void Lattice::set_dispatch(const int32_t* tags, std::size_t n) {
    dispatch_.clear();
    for (std::size_t k = 0; k < n; ++k) dispatch_.insert(tags[k]);
    dispatch_set_ = true;
}

// accelerated_lattice.cpp:161-181: fail before any write, naming the chain.
void Lattice::check_dispatch() const {
    if (!slots_set_) throw std::invalid_argument("cell dynamics not assigned (set slots first)");
    if (untagged_) throw DispatchError("<untagged cell>");
    std::set<int> present;
    for (int32_t s : present_slots_) present.insert(tag_of_slot_[std::size_t(s)]);
    for (int t : present) {
        const bool ok = dispatch_set_ ? dispatch_.count(t) != 0 : true;
        if (!ok) throw DispatchError(tag_names_[std::size_t(t)]);
    }
    if (split() && d_.periodic[2] && !(lower_.linked && upper_.linked))
        throw ExchangeError("periodic z-slab is not linked to both neighbours");
    if (exchange_failed_)
        throw ExchangeError("a halo exchange failed; bring the slabs to one step count and call exchange first");
}

void Lattice::reset_aa() {
    envelope_valid_ = false;
    if (!aa()) return;
    DeviceGuard dg(device_);
    const std::size_t bytes = std::size_t(d_.q) * std::size_t(geo_.dstride) * (d_.precision_bits / 8);
    cuda_check(cudaMemsetAsync(buf_[0], 0, bytes, stream_), "memset");
    // unlinked: the odd layout (the first step is even); linked z-slabs rest
    // in the even layout, which needs no neighbour data (k_aa)
    aa_odd_layout_ = !(lower_.linked || upper_.linked);
}

void Lattice::fill_equilibrium(const double* rho, const double* ux, const double* uy,
                               const double* uz) {
    bb_prologue_ = true;
    cmp_valid_ = false;
    bb_dirty_ = false;
    envelope_valid_ = false;
    DeviceGuard dg(device_);
    reset_aa();
    const long long plane_cells = (long long)geo_.nx * geo_.ny;
    const int zc = int(std::max<long long>(1, (long long)(staging_bytes_ / 32) / plane_cells));
    double* st = static_cast<double*>(staging_);
    for (int z0 = 0; z0 < geo_.nz; z0 += zc) {
        const int nzc = std::min(zc, geo_.nz - z0);
        const long long n = plane_cells * nzc;
        if (n * 32 > (long long)staging_bytes_) throw std::invalid_argument("plane too large");
        const long long off = plane_cells * z0;
        cuda_check(cudaMemcpyAsync(st, rho + off, n * 8, cudaMemcpyHostToDevice, stream_), "h2d");
        cuda_check(cudaMemcpyAsync(st + n, ux + off, n * 8, cudaMemcpyHostToDevice, stream_), "h2d");
        cuda_check(cudaMemcpyAsync(st + 2 * n, uy + off, n * 8, cudaMemcpyHostToDevice, stream_), "h2d");
        cuda_check(cudaMemcpyAsync(st + 3 * n, uz + off, n * 8, cudaMemcpyHostToDevice, stream_), "h2d");
        const int grid = grid_for(n);
        void* o = origin(cur_);
        if (d_.precision_bits == 64) {
            if (d_.q == 19) k_fill_eq<double, 19><<<grid, 256, 0, stream_>>>((double*)o, geo_, st, st + n, st + 2 * n, st + 3 * n, z0, nzc, aa_fill_mode());
            else k_fill_eq<double, 27><<<grid, 256, 0, stream_>>>((double*)o, geo_, st, st + n, st + 2 * n, st + 3 * n, z0, nzc, aa_fill_mode());
        } else {
            if (d_.q == 19) k_fill_eq<float, 19><<<grid, 256, 0, stream_>>>((float*)o, geo_, st, st + n, st + 2 * n, st + 3 * n, z0, nzc, aa_fill_mode());
            else k_fill_eq<float, 27><<<grid, 256, 0, stream_>>>((float*)o, geo_, st, st + n, st + 2 * n, st + 3 * n, z0, nzc, aa_fill_mode());
        }
        cuda_check(cudaGetLastError(), "k_fill_eq");
        cuda_check(cudaStreamSynchronize(stream_), "fill_equilibrium");
    }
}

// Uniform equilibrium state (rho, u) in every cell: the chunked equilibrium
// fill with constant staging arrays (same k_fill_eq arithmetic).
void Lattice::fill_uniform(double rho, double ux, double uy, double uz) {
    bb_prologue_ = true;
    cmp_valid_ = false;
    bb_dirty_ = false;
    const long long plane_cells = (long long)geo_.nx * geo_.ny;
    const int zc = int(std::max<long long>(1, std::min<long long>(geo_.nz, (long long)(staging_bytes_ / 32) / plane_cells)));
    const long long n = plane_cells * zc;
    if (n * 32 > (long long)staging_bytes_) throw std::invalid_argument("plane too large");
    std::vector<double> h(std::size_t(4 * n));
    std::fill(h.begin(), h.begin() + n, rho);
    std::fill(h.begin() + n, h.begin() + 2 * n, ux);
    std::fill(h.begin() + 2 * n, h.begin() + 3 * n, uy);
    std::fill(h.begin() + 3 * n, h.end(), uz);
    // k_fill_eq indexes the staging arrays chunk-locally: one upload serves every chunk
    DeviceGuard dg(device_);
    envelope_valid_ = false;
    reset_aa();
    double* st = static_cast<double*>(staging_);
    cuda_check(cudaMemcpyAsync(st, h.data(), h.size() * 8, cudaMemcpyHostToDevice, stream_), "h2d");
    for (int z0 = 0; z0 < geo_.nz; z0 += zc) {
        const int nzc = std::min(zc, geo_.nz - z0);
        const long long m = plane_cells * nzc;
        const int grid = grid_for(m);
        void* o = origin(cur_);
        if (d_.precision_bits == 64) {
            if (d_.q == 19) k_fill_eq<double, 19><<<grid, 256, 0, stream_>>>((double*)o, geo_, st, st + n, st + 2 * n, st + 3 * n, z0, nzc, aa_fill_mode());
            else k_fill_eq<double, 27><<<grid, 256, 0, stream_>>>((double*)o, geo_, st, st + n, st + 2 * n, st + 3 * n, z0, nzc, aa_fill_mode());
        } else {
            if (d_.q == 19) k_fill_eq<float, 19><<<grid, 256, 0, stream_>>>((float*)o, geo_, st, st + n, st + 2 * n, st + 3 * n, z0, nzc, aa_fill_mode());
            else k_fill_eq<float, 27><<<grid, 256, 0, stream_>>>((float*)o, geo_, st, st + n, st + 2 * n, st + 3 * n, z0, nzc, aa_fill_mode());
        }
        cuda_check(cudaGetLastError(), "k_fill_eq");
    }
    cuda_check(cudaStreamSynchronize(stream_), "fill_uniform");
}

void Lattice::fill_tgv(int64_t L, double u_inf) {
    bb_prologue_ = true;
    cmp_valid_ = false;
    bb_dirty_ = false;
    if (d_.dims[0] != L || d_.dims[1] != L || d_.global_nz != L)
        throw std::invalid_argument("TGV fill needs an L^3 domain");
    DeviceGuard dg(device_);
    reset_aa();
    envelope_valid_ = false;
    // cases.cpp:145-156: x = 2 pi / L * (i + 0.5); glibc sin / cos on the host.
    const double scale = 2.0 * 3.14159265358979323846 / double(L);
    std::vector<double> tab(std::size_t(3 * L));
    for (int64_t i = 0; i < L; ++i) {
        const double x = scale * (double(i) + 0.5);
        tab[std::size_t(i)] = std::sin(x);
        tab[std::size_t(L + i)] = std::cos(x);
        tab[std::size_t(2 * L + i)] = std::cos(2.0 * x);
    }
    double* st = static_cast<double*>(staging_);
    cuda_check(cudaMemcpyAsync(st, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, stream_), "h2d");
    const int grid = grid_for(cells());
    void* o = origin(cur_);
    if (d_.precision_bits == 64) {
        if (d_.q == 19) k_fill_tgv<double, 19><<<grid, 256, 0, stream_>>>((double*)o, geo_, st, st + L, st + 2 * L, d_.z_origin, u_inf, aa_fill_mode());
        else k_fill_tgv<double, 27><<<grid, 256, 0, stream_>>>((double*)o, geo_, st, st + L, st + 2 * L, d_.z_origin, u_inf, aa_fill_mode());
    } else {
        if (d_.q == 19) k_fill_tgv<float, 19><<<grid, 256, 0, stream_>>>((float*)o, geo_, st, st + L, st + 2 * L, d_.z_origin, u_inf, aa_fill_mode());
        else k_fill_tgv<float, 27><<<grid, 256, 0, stream_>>>((float*)o, geo_, st, st + L, st + 2 * L, d_.z_origin, u_inf, aa_fill_mode());
    }
    cuda_check(cudaGetLastError(), "k_fill_tgv");
    cuda_check(cudaStreamSynchronize(stream_), "fill_tgv");
}

// Canonical (direction-major, x fastest, interior only) <-> device layout,
// chunked over z planes through the staging buffer.
void Lattice::copy_canonical(void* host, bool to_device, bool as_double, int elem_bytes) {
    DeviceGuard dg(device_);
    if (to_device) {
        reset_aa();
        envelope_valid_ = false;
        bb_prologue_ = true;
        cmp_valid_ = false;
        bb_dirty_ = false;
    } else {
        finalize_walls();
    }
    const long long plane_cells = (long long)geo_.nx * geo_.ny;
    const long long n = cells();
    const int zc = int(std::max<long long>(1, (long long)staging_bytes_ / (8 * plane_cells)));
    const int* cz_tab = d_.q == 19 ? kCz19 : kCz27;
    for (int i = 0; i < d_.q; ++i) {
        // canonical direction i lives in layout direction li, shifted by sh (AA)
        int li = i, sx = 0, sy = 0, sz = 0;
        if (aa() && !aa_odd_layout_) li = i == 0 ? 0 : ((i & 1) ? i + 1 : i - 1);
        if (aa() && aa_odd_layout_) {
            sx = (d_.q == 19 ? kCx19 : kCx27)[i];
            sy = (d_.q == 19 ? kCy19 : kCy27)[i];
            sz = cz_tab[i];
        }
        for (int z0 = 0; z0 < geo_.nz; z0 += zc) {
            const int nzc = std::min(zc, geo_.nz - z0);
            const long long cnt = plane_cells * nzc;
            char* h = static_cast<char*>(host) + (std::size_t(i) * n + plane_cells * z0) * elem_bytes;
            const int grid = grid_for(cnt);
            char* o = static_cast<char*>(origin(cur_)) + std::size_t(li) * geo_.dstride * (d_.precision_bits / 8);
            if (to_device) {
                cuda_check(cudaMemcpyAsync(staging_, h, cnt * elem_bytes, cudaMemcpyHostToDevice, stream_), "h2d");
                if (d_.precision_bits == 64)
                    k_box_copy<double, double, true><<<grid, 256, 0, stream_>>>((double*)o, (const double*)staging_, geo_, 0, 0, z0, geo_.nx, geo_.ny, nzc, sx, sy, sz);
                else if (as_double)
                    k_box_copy<float, double, true><<<grid, 256, 0, stream_>>>((float*)o, (const double*)staging_, geo_, 0, 0, z0, geo_.nx, geo_.ny, nzc, sx, sy, sz);
                else
                    k_box_copy<float, float, true><<<grid, 256, 0, stream_>>>((float*)o, (const float*)staging_, geo_, 0, 0, z0, geo_.nx, geo_.ny, nzc, sx, sy, sz);
                cuda_check(cudaGetLastError(), "k_box_copy");
            } else {
                if (d_.precision_bits == 64)
                    k_box_copy<double, double, false><<<grid, 256, 0, stream_>>>((double*)staging_, (const double*)o, geo_, 0, 0, z0, geo_.nx, geo_.ny, nzc, sx, sy, sz);
                else if (as_double)
                    k_box_copy<double, float, false><<<grid, 256, 0, stream_>>>((double*)staging_, (const float*)o, geo_, 0, 0, z0, geo_.nx, geo_.ny, nzc, sx, sy, sz);
                else
                    k_box_copy<float, float, false><<<grid, 256, 0, stream_>>>((float*)staging_, (const float*)o, geo_, 0, 0, z0, geo_.nx, geo_.ny, nzc, sx, sy, sz);
                cuda_check(cudaGetLastError(), "k_box_copy");
                cuda_check(cudaMemcpyAsync(h, staging_, cnt * elem_bytes, cudaMemcpyDeviceToHost, stream_), "d2h");
            }
            cuda_check(cudaStreamSynchronize(stream_), "copy_canonical");
        }
    }
}

void Lattice::upload(const double* canon) { copy_canonical(const_cast<double*>(canon), true, true, 8); }
void Lattice::download(double* canon) { copy_canonical(canon, false, true, 8); }
void Lattice::download_raw(void* canon) {
    copy_canonical(canon, false, d_.precision_bits == 64, d_.precision_bits / 8);
}

// Envelope-inclusive AcceleratedBlock arrays: the whole (nx+2)(ny+2)(nz+2)
// box of every direction, including the envelope the caller refreshed.
void Lattice::upload_block(const void* f, const int64_t ext[3]) {
    bb_prologue_ = true;
    cmp_valid_ = false;
    bb_dirty_ = false;
    envelope_valid_ = false;
    DeviceGuard dg(device_);
    const int s = d_.precision_bits / 8;
    const long long vol = ext[0] * ext[1] * ext[2];
    const long long plane_cells = ext[0] * ext[1];
    const int zc = int(std::max<long long>(1, (long long)staging_bytes_ / (s * plane_cells)));
    for (int i = 0; i < d_.q; ++i) {
        for (int z0 = 0; z0 < ext[2]; z0 += zc) {
            const int nzc = int(std::min<long long>(zc, ext[2] - z0));
            const long long cnt = plane_cells * nzc;
            const char* h = static_cast<const char*>(f) + (std::size_t(i) * vol + plane_cells * z0) * s;
            char* o = static_cast<char*>(origin(cur_)) + std::size_t(i) * geo_.dstride * s;
            cuda_check(cudaMemcpyAsync(staging_, h, cnt * s, cudaMemcpyHostToDevice, stream_), "h2d");
            const int grid = grid_for(cnt);
            if (s == 8)
                k_box_copy<double, double, true><<<grid, 256, 0, stream_>>>((double*)o, (const double*)staging_, geo_, -1, -1, z0 - 1, int(ext[0]), int(ext[1]), nzc);
            else
                k_box_copy<float, float, true><<<grid, 256, 0, stream_>>>((float*)o, (const float*)staging_, geo_, -1, -1, z0 - 1, int(ext[0]), int(ext[1]), nzc);
            cuda_check(cudaGetLastError(), "k_box_copy");
            cuda_check(cudaStreamSynchronize(stream_), "upload_block");
        }
    }
}

// Interior of buffer `which` (0 = current state) back into an envelope-
// inclusive host block; the host envelope is left untouched.
void Lattice::download_block_interior(void* f, const int64_t ext[3], int which) {
    DeviceGuard dg(device_);
    const int s = d_.precision_bits / 8;
    const long long vol = ext[0] * ext[1] * ext[2];
    const long long plane_cells = ext[0] * ext[1];
    const int buf = which == 0 ? cur_ : 1 - cur_;
    const int zc = int(std::max<long long>(1, (long long)staging_bytes_ / (s * plane_cells)));
    for (int i = 0; i < d_.q; ++i) {
        for (int z0 = 1; z0 < ext[2] - 1; z0 += zc) {
            const int nzc = int(std::min<long long>(zc, ext[2] - 1 - z0));
            const long long cnt = plane_cells * nzc;
            const char* o = static_cast<const char*>(origin(buf)) + std::size_t(i) * geo_.dstride * s;
            const int grid = grid_for(cnt);
            // gather full rows (envelope columns included) of planes z0..z0+nzc-1
            if (s == 8)
                k_box_copy<double, double, false><<<grid, 256, 0, stream_>>>((double*)staging_, (const double*)o, geo_, -1, -1, z0 - 1, int(ext[0]), int(ext[1]), nzc);
            else
                k_box_copy<float, float, false><<<grid, 256, 0, stream_>>>((float*)staging_, (const float*)o, geo_, -1, -1, z0 - 1, int(ext[0]), int(ext[1]), nzc);
            cuda_check(cudaGetLastError(), "k_box_copy");
            // copy back the interior of those planes (the caller's envelope is kept)
            cudaMemcpy3DParms p{};
            p.srcPtr = make_cudaPitchedPtr(staging_, ext[0] * s, ext[0], ext[1]);
            p.srcPos = make_cudaPos(s, 1, 0);
            p.dstPtr = make_cudaPitchedPtr(static_cast<char*>(f) + std::size_t(i) * vol * s, ext[0] * s,
                                           ext[0], ext[1]);
            p.dstPos = make_cudaPos(s, 1, z0);
            p.extent = make_cudaExtent((ext[0] - 2) * s, ext[1] - 2, nzc);
            p.kind = cudaMemcpyDeviceToHost;
            cuda_check(cudaMemcpy3DAsync(&p, stream_), "d2h");
            cuda_check(cudaStreamSynchronize(stream_), "download_block");
        }
    }
}

template <typename T>
void Lattice::fill_recipes(StepArgs<T>& a) const {
    a.slot = d_slot_;
    a.uniform_slot = uniform_slot_;
    a.skip_group = skip_group_;
    for (std::size_t s = 0; s < chains_.size() && s < std::size_t(kMaxSlots); ++s)
        a.rec[s] = compile_recipe<T>(chains_[s]);
    a.xrec = static_cast<const DevRecipe<T>*>(d_xrec_);
}

// Three-stage pipeline over z-chunks of a pinned host block (host layout kept
// on the device, so every transfer is one contiguous range per direction):
//   copy engine 1: host planes needed by chunk k -> device input mirror
//   SMs:           collide-and-stream of chunk k (input mirror -> output mirror)
//   copy engine 2: finished planes of chunk k -> the caller's f_out (or back
//                  into f_in: those planes are no longer read by later chunks)
// The two PCIe directions run concurrently with the compute. The H2D copies
// run at most `ahead` chunks in front of the copy-back (each waits for the
// D2H of chunk k - ahead): left alone the H2D direction wins the link
// arbitration and the copy-back finishes alone at the end.
template <typename T>
void Lattice::launch_host_block(void* f_in, const int64_t ext[3], void* f_out) {
    const long long vol = ext[0] * ext[1] * ext[2];
    Geo hg{};
    hg.nx = geo_.nx;
    hg.ny = geo_.ny;
    hg.nz = geo_.nz;
    hg.pitch = int(ext[0]);
    hg.plane = int(ext[0] * ext[1]);
    hg.dstride = vol;
    hg.per_x = hg.per_y = hg.per_z = 0;  // the caller's envelope is authoritative
    const std::size_t bytes = std::size_t(d_.q) * vol * sizeof(T);
    T* din;
    T* dout;
    if (!aa() && std::size_t(d_.q) * std::size_t(geo_.dstride) * sizeof(T) >= bytes) {
        // the lattice's own two population buffers hold the host-layout
        // mirrors (each call uploads the whole input state, so nothing else
        // lives there between calls): no second pair of state-sized buffers
        din = static_cast<T*>(buf_[0]);
        dout = static_cast<T*>(buf_[1]);
        envelope_valid_ = false;
    } else {
        if (blk_out_bytes_ < 2 * bytes) {
            cudaFree(blk_out_);
            blk_out_ = nullptr;
            cuda_check(cudaMalloc(&blk_out_, 2 * bytes), "cudaMalloc block mirrors");
            blk_out_bytes_ = 2 * bytes;
        }
        din = static_cast<T*>(blk_out_);
        dout = din + std::size_t(d_.q) * vol;
    }
    if (!copy_stream_) cuda_check(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking), "stream");
    if (!h2d_stream_) cuda_check(cudaStreamCreateWithFlags(&h2d_stream_, cudaStreamNonBlocking), "stream");
    StepArgs<T> a{};
    fill_recipes(a);
    a.g = hg;
    const long long org = hg.plane + hg.pitch + 1;
    for (int i = 0; i < d_.q; ++i) {
        a.fin[i] = din + i * vol + org;
        a.fout[i] = dout + i * vol + org;
    }
    a.z_step = 1;
    blk_args_.resize(sizeof(a));
    std::memcpy(blk_args_.data(), &a, sizeof(a));
    blk_.bx = hg.nx >= 128 ? 128 : (hg.nx > 32 ? 64 : 32);
    blk_.by = 256 / blk_.bx;
    blk_.gx = unsigned((hg.nx + blk_.bx - 1) / blk_.bx);
    blk_.gy = unsigned((hg.ny + blk_.by - 1) / blk_.by);
    // 32 z-chunks (2-D copies keep the per-chunk cost low; shorter fill / drain), >= 1 plane each
    static const int kChunks = [] {
        const char* e = std::getenv("DLB_BLOCK_CHUNKS");
        return e ? std::max(1, std::atoi(e)) : 32;
    }();
    static const int kAhead = [] {
        const char* e = std::getenv("DLB_BLOCK_AHEAD");
        return e ? std::max(0, std::atoi(e)) : 2;
    }();
    const int zc = std::max(1, (hg.nz + kChunks - 1) / kChunks);
    const int nchunks = (hg.nz + zc - 1) / zc;
    while (int(blk_ev_.size()) < 3 * nchunks) {
        cudaEvent_t e;
        cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        blk_ev_.push_back(e);
    }
    blk_.f_in = f_in;
    blk_.f_out = f_out ? f_out : f_in;
    blk_.din = din;
    blk_.dout = dout;
    blk_.vol = vol;
    blk_.plane = hg.plane;
    blk_.pitch = hg.pitch;
    blk_.nx = hg.nx;
    blk_.ny = hg.ny;
    blk_.nz = hg.nz;
    blk_.zc = zc;
    blk_.nchunks = nchunks;
    blk_.elem = int(sizeof(T));
    blk_.ahead = kAhead == 0 ? nchunks : kAhead;
    blk_.issued = 0;
    blk_.loaded = 0;
    blk_.pending = true;
    static const bool trace = std::getenv("DLB_TRACE_BLOCK") != nullptr;
    if (trace) {  // timeline events (DLB_TRACE_BLOCK): begin, end of H2D, end of compute
        for (auto& e : blk_tr_)
            if (!e) cuda_check(cudaEventCreate(&e), "event");
        cuda_check(cudaEventRecord(blk_tr_[0], h2d_stream_), "event");
    }
    // speculative part (device-side writes only, runs while the caller's tag
    // scan decides): the first max(ahead, DLB_BLOCK_SPEC = 4) chunks
    static const int kSpec = [] {
        const char* e = std::getenv("DLB_BLOCK_SPEC");
        return e ? std::max(1, std::atoi(e)) : 4;
    }();
    blk_.copied = 0;
    while (blk_.issued < std::min(std::max(blk_.ahead, kSpec), nchunks)) issue_block_chunk(blk_.issued++);
}

// H2D of the host planes chunk c reads (after the D2H of chunk c - ahead) and
// its compute. Events per chunk: [3c] H2D done, [3c+1] compute done, [3c+2] D2H done.
void Lattice::issue_block_chunk(int c) {
    const int z0 = c * blk_.zc, z1 = std::min(blk_.nz, z0 + blk_.zc);
    if (c >= blk_.ahead && c - blk_.ahead < blk_.copied)
        cuda_check(cudaStreamWaitEvent(h2d_stream_, blk_ev_[3 * (c - blk_.ahead) + 2], 0), "wait");
    // chunk [z0, z1) reads host planes [z0, z1 + 2)
    block_copy(h2d_stream_, blk_.f_in, blk_.din, true, blk_.loaded, z1 + 2);
    blk_.loaded = z1 + 2;
    cuda_check(cudaEventRecord(blk_ev_[3 * c], h2d_stream_), "event");
    if (c == blk_.nchunks - 1 && blk_tr_[1]) cuda_check(cudaEventRecord(blk_tr_[1], h2d_stream_), "event");
    cuda_check(cudaStreamWaitEvent(stream_, blk_ev_[3 * c], 0), "wait");
    // the kernel reads z_begin from its argument block (StepArgs<T> is a POD image)
    std::vector<uint8_t> args(blk_args_);
    const std::size_t zoff = d_.precision_bits == 64 ? offsetof(StepArgs<double>, z_begin)
                                                     : offsetof(StepArgs<float>, z_begin);
    std::memcpy(args.data() + zoff, &z0, sizeof(int));
    void* kargs[] = {args.data()};
    cuda_check(cudaLaunchKernel(kernel_->fn, dim3(blk_.gx, blk_.gy, unsigned(z1 - z0)), dim3(blk_.bx, blk_.by, 1),
                                kargs, 0, stream_), "launch");
    {   // host planes [z0 + 1, z1 + 1): their x / y envelope rides along to the copy-back
        const int np = z1 - z0, per = 2 * blk_.pitch + 2 * blk_.ny;
        const dim3 grid(unsigned(std::min(8, (per + 255) / 256)), unsigned(d_.q * np));
        if (blk_.elem == 8)
            k_carry_envelope_xy<double><<<grid, 256, 0, stream_>>>(static_cast<const double*>(blk_.din),
                static_cast<double*>(blk_.dout), blk_.vol, blk_.pitch, blk_.plane, blk_.nx, blk_.ny, z0 + 1, np);
        else
            k_carry_envelope_xy<float><<<grid, 256, 0, stream_>>>(static_cast<const float*>(blk_.din),
                static_cast<float*>(blk_.dout), blk_.vol, blk_.pitch, blk_.plane, blk_.nx, blk_.ny, z0 + 1, np);
        cuda_check(cudaGetLastError(), "k_carry_envelope_xy");
    }
    cuda_check(cudaEventRecord(blk_ev_[3 * c + 1], stream_), "event");
    if (c == blk_.nchunks - 1 && blk_tr_[2]) cuda_check(cudaEventRecord(blk_tr_[2], stream_), "event");
}

// One direction-strided copy of host planes [p0, p1) between a caller block
// and a device mirror (the same envelope-inclusive layout).
void Lattice::block_copy(cudaStream_t st, void* host, void* dev, bool up, int p0, int p1) {
    if (p1 <= p0) return;
    const std::size_t plane_bytes = std::size_t(blk_.plane) * blk_.elem;
    static const bool one_d = [] {
        const char* e = std::getenv("DLB_BLOCK_1D");  // tuning: per-direction 1-D copies
        return e && e[0] == '1';
    }();
    if (!one_d) {
        // all q direction arrays in one 2-D copy (rows = directions, pitch = one array)
        const std::size_t off = std::size_t(p0) * blk_.plane * blk_.elem;
        const std::size_t pitch = std::size_t(blk_.vol) * blk_.elem;
        char* h = static_cast<char*>(host) + off;
        char* d = static_cast<char*>(dev) + off;
        const cudaError_t e = cudaMemcpy2DAsync(up ? d : h, pitch, up ? h : d, pitch, std::size_t(p1 - p0) * plane_bytes,
                                                d_.q, up ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) return;
        cudaGetLastError();  // pitch beyond the 2-D copy limit: one copy per direction
    }
    for (int i = 0; i < d_.q; ++i) {
        const std::size_t off = (std::size_t(i) * blk_.vol + std::size_t(p0) * blk_.plane) * blk_.elem;
        char* h = static_cast<char*>(host) + off;
        char* d = static_cast<char*>(dev) + off;
        cuda_check(cudaMemcpyAsync(up ? d : h, up ? h : d, std::size_t(p1 - p0) * plane_bytes,
                                   up ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, st),
                   up ? "h2d" : "d2h");
    }
}

// Copy-back of host planes [p0, p1). Default: whole planes (one 2-D copy for
// all directions), whose x / y envelope cells carry f_in's envelope
// (k_carry_envelope_xy): in place that is the caller's envelope unchanged;
// into f_out it is f_in's envelope where the reference's step_range (interior
// cells only, accelerated_lattice.cpp:126-153) leaves f_out's -- equal
// whenever the two buffers hold the same envelope (a bounded block's, or one
// refreshed before each step). DLB_BLOCK_D2H_ROWS=1: interior rows only (one
// 3-D copy per direction), f_out's envelope never written; measured 20-30 %
// slower end to end (row-sized DMA pieces; profiles/r02c_summary.md).
void Lattice::block_copy_back_interior(cudaStream_t st, int p0, int p1) {
    if (p1 <= p0) return;
    static const bool by_rows = [] {
        const char* v = std::getenv("DLB_BLOCK_D2H_ROWS");
        return v && v[0] == '1';
    }();
    if (!by_rows) return block_copy(st, blk_.f_out, blk_.dout, false, p0, p1);
    const std::size_t e = std::size_t(blk_.elem);
    const std::size_t pitch = std::size_t(blk_.pitch) * e;
    const std::size_t rows = std::size_t(blk_.plane / blk_.pitch);
    for (int i = 0; i < d_.q; ++i) {
        const std::size_t off = std::size_t(i) * std::size_t(blk_.vol) * e;
        cudaMemcpy3DParms m{};
        m.srcPtr = make_cudaPitchedPtr(static_cast<char*>(blk_.dout) + off, pitch, pitch, rows);
        m.dstPtr = make_cudaPitchedPtr(static_cast<char*>(blk_.f_out) + off, pitch, pitch, rows);
        m.srcPos = m.dstPos = make_cudaPos(e, 1, std::size_t(p0));
        m.extent = make_cudaExtent(std::size_t(blk_.nx) * e, std::size_t(blk_.ny), std::size_t(p1 - p0));
        m.kind = cudaMemcpyDeviceToHost;
        cuda_check(cudaMemcpy3DAsync(&m, st), "d2h interior");
    }
}

void Lattice::begin_host_block(void* f_in, const int64_t ext[3], void* f_out) {
    DeviceGuard dg(device_);
    if (aa()) throw std::invalid_argument("host-block stepping uses the two-population layout");
    if (blk_.pending) abort_host_block();
    if (d_.precision_bits == 64) launch_host_block<double>(f_in, ext, f_out);
    else launch_host_block<float>(f_in, ext, f_out);
}

// Copy-back: finished planes go back as soon as their chunk is computed, on a
// second copy engine, interleaved with the remaining H2D chunks.
void Lattice::finish_host_block(const std::function<int(int)>& gate, const std::function<void()>& reslot) {
    DeviceGuard dg(device_);
    if (!blk_.pending) throw std::logic_error("finish_host_block without begin_host_block");
    int written = 1;  // host planes [1, written) copied back (plane 0 is envelope)
    bool gated = static_cast<bool>(gate);
    for (int c = 0; c < blk_.nchunks; ++c) {
        const int z1 = std::min(blk_.nz, (c + 1) * blk_.zc);
        if (gated && gate(z1) >= 0) {
            // the slots of a plane of chunk c (or later) changed: the chunks
            // before c were stepped with their confirmed slots and stay; drain,
            // install the new slots, recompute from chunk c on
            cuda_check(cudaStreamSynchronize(h2d_stream_), "block reslot");
            cuda_check(cudaStreamSynchronize(stream_), "block reslot");
            cuda_check(cudaStreamSynchronize(copy_stream_), "block reslot");
            reslot();
            if (d_.precision_bits == 64) refill_block_recipes<double>();
            else refill_block_recipes<float>();
            blk_.issued = c;
            while (blk_.issued < blk_.nchunks && blk_.issued <= c + blk_.ahead) issue_block_chunk(blk_.issued++);
            gated = false;
        }
        cuda_check(cudaStreamWaitEvent(copy_stream_, blk_ev_[3 * c + 1], 0), "wait");
        if (c == 0 && blk_tr_[3]) cuda_check(cudaEventRecord(blk_tr_[3], copy_stream_), "event");
        block_copy_back_interior(copy_stream_, written, z1 + 1);
        written = z1 + 1;
        cuda_check(cudaEventRecord(blk_ev_[3 * c + 2], copy_stream_), "event");
        blk_.copied = c + 1;
        while (blk_.issued < blk_.nchunks && blk_.issued <= c + blk_.ahead) issue_block_chunk(blk_.issued++);
    }
    if (blk_tr_[4]) cuda_check(cudaEventRecord(blk_tr_[4], copy_stream_), "event");
    blk_.pending = false;
    cuda_check(cudaStreamSynchronize(copy_stream_), "block copy-back");
    cuda_check(cudaStreamSynchronize(stream_), "block step");
    if (blk_tr_[4]) {
        float t[5] = {0, 0, 0, 0, 0};
        for (int k = 1; k < 5; ++k) cudaEventElapsedTime(&t[k], blk_tr_[0], blk_tr_[k]);
        std::fprintf(stderr, "[dlb block] H2D done %.1f ms, compute done %.1f ms, D2H start %.1f ms, D2H done %.1f ms\n",
                     t[1], t[2], t[3], t[4]);
    }
    ++steps_;
}

// The pending block step's kernel arguments after new slots: the recipe /
// slot fields again, geometry and mirror pointers kept.
template <typename T>
void Lattice::refill_block_recipes() {
    StepArgs<T> a;
    std::memcpy(&a, blk_args_.data(), sizeof(a));
    fill_recipes(a);
    std::memcpy(blk_args_.data(), &a, sizeof(a));
}

// Drop a begun step: nothing was written to the caller's block.
void Lattice::abort_host_block() {
    DeviceGuard dg(device_);
    blk_.pending = false;
    cuda_check(cudaStreamSynchronize(h2d_stream_), "block abort");
    cuda_check(cudaStreamSynchronize(stream_), "block abort");
}

void Lattice::step_host_block(void* f_in, const int64_t ext[3], void* f_out) {
    begin_host_block(f_in, ext, f_out);
    finish_host_block();
}

template <typename T>
void Lattice::launch_coop(int64_t nsteps) {
    StepArgs<T> a{};
    for (int i = 0; i < d_.q; ++i) {
        a.fin[i] = static_cast<const T*>(origin(cur_)) + i * geo_.dstride;
        a.fout[i] = static_cast<T*>(origin(1 - cur_)) + i * geo_.dstride;
    }
    a.slot = d_slot_;
    a.uniform_slot = uniform_slot_;
    a.skip_group = skip_group_;
    a.g = geo_;
    for (std::size_t s = 0; s < chains_.size() && s < std::size_t(kMaxSlots); ++s)
        a.rec[s] = compile_recipe<T>(chains_[s]);
    a.xrec = static_cast<const DevRecipe<T>*>(d_xrec_);
    if (coop_grid_ == 0) {
        int per_sm = 0, sms = 0;
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel_coop_->fn, 256, 0), "occupancy");
        cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_), "sm count");
        coop_grid_ = int(std::min<long long>(std::max(1, per_sm) * (long long)sms, (cells() + 255) / 256));
    }
    // chunks of at most 2^30 steps (int argument); parity follows the step count
    int64_t done = 0;
    while (done < nsteps) {
        int n = int(std::min<int64_t>(nsteps - done, 1 << 30));
        void* args[] = {&a, &n};
        cuda_check(cudaLaunchCooperativeKernel(kernel_coop_->fn, dim3(unsigned(coop_grid_)), dim3(256), args, 0,
                                               stream_), "launch cooperative");
        if (n & 1)  // an odd chunk leaves the state in the other buffer
            for (int i = 0; i < d_.q; ++i) {
                T* t = a.fout[i];
                a.fout[i] = const_cast<T*>(a.fin[i]);
                a.fin[i] = t;
            }
        done += n;
    }
    if (nsteps & 1) cur_ = 1 - cur_;
    steps_ += nsteps;
    envelope_valid_ = false;
}

template <typename T>
void Lattice::launch_step(int parity) {
    StepArgs<T> a{};
    for (int i = 0; i < d_.q; ++i) {
        a.fin[i] = static_cast<const T*>(origin(parity)) + i * geo_.dstride;
        a.fout[i] = static_cast<T*>(origin(1 - parity)) + i * geo_.dstride;
    }
    a.slot = d_slot_;
    a.uniform_slot = uniform_slot_;
    a.skip_group = skip_group_;
    a.g = geo_;
    for (std::size_t s = 0; s < chains_.size() && s < std::size_t(kMaxSlots); ++s)
        a.rec[s] = compile_recipe<T>(chains_[s]);
    a.xrec = static_cast<const DevRecipe<T>*>(d_xrec_);

    const int bx0 = geo_.nx >= 128 ? 128 : (geo_.nx > 32 ? 64 : 32);
    const int bx = std::min(bx0, pull_threads_);
    const int by = std::max(1, pull_threads_ / bx);
    const dim3 block(bx, by, 1);
    const unsigned gx = unsigned((geo_.nx + bx - 1) / bx);
    const unsigned gy = unsigned((geo_.ny + by - 1) / by);
    const bool linked = lower_.linked || upper_.linked;
    // AA: the state's layout picks the kernel (odd layout -> even kernel)
    const void* fn = !aa() ? kernel_->fn : (aa_odd_layout_ ? kernel_->fn : kernel_odd_->fn);
    if (sparse_) {
        for (const ListLaunch& l : lists_) {
            const unsigned long long* lp = d_list_ + l.offset;
            long long n = l.count;
            int slot = l.slot;
            void* args[] = {&a, &lp, &n, &slot};
            const long long blocks = std::min<long long>((n + 255) / 256, 148LL * 8);
            cuda_check(cudaLaunchKernel(l.kernel->fn, dim3(unsigned(blocks)), dim3(256), args, 0, stream_),
                       "launch list");
        }
        return;
    }
    if (aa() && !linked) {
        a.z_begin = 0;
        a.z_step = 1;
        void* args[] = {&a};
        cuda_check(cudaLaunchKernel(fn, dim3(gx, gy, geo_.nz), block, args, 0, stream_), "launch");
        aa_odd_layout_ = !aa_odd_layout_;
        return;
    }
    if (!linked && kernel_tma_ && !(ke_requested_ && kernel_ke_)) {
        launch_tma<T>(a, parity);
        return;
    }
    envelope_valid_ = false;  // the other kernels wrap in-kernel and leave the envelope stale
    if (!linked) {
        a.z_begin = 0;
        a.z_step = 1;
        void* args[] = {&a};
        bool split_rare = kernel_main_ != nullptr && !fixups_.empty();
        if (kernel_cmp_) {
            // compacted porous sweep (+ the regularized cells with the full set)
            prepare_compact();
            StepArgs<T> c = a;
            for (int i = 0; i < d_.q; ++i) {
                c.fin[i] = static_cast<const T*>(cbuf_[parity]) + i * cstride_;
                c.fout[i] = static_cast<T*>(cbuf_[1 - parity]) + i * cstride_;
            }
            c.slot = nullptr;
            CmpArgs ca{d_cseg_, d_crows_, d_cslot_, d_cfix_, ncl_ << cgshift_, ncl_, cgshift_};
            void* cargs[] = {&c, &ca};
            const long long per_block = 256LL * kernel_cmp_->cpt;
            cuda_check(cudaLaunchKernel(kernel_cmp_->fn, dim3(unsigned((ca.n + per_block - 1) / per_block)),
                                        dim3(256), cargs, 0, stream_), "launch compact");
            if (kernel_cmp_fix_) {
                // (as a parallel high-priority branch it slowed the main sweep:
                // 10.06 vs 9.65 ms per c4 step, profiles/r02b_summary.md)
                ca.n = ncfix_;
                cuda_check(cudaLaunchKernel(kernel_cmp_fix_->fn, dim3(unsigned((ca.n + 255) / 256)), dim3(256),
                                            cargs, 0, stream_), "launch compact fix-up");
            }
            cmp_dirty_ = true;
            return;
        }
        if (kernel_segbb_ && !bb_prologue_) {
            // fluid-segment sweep: wall cells outside the listed segments skip
            const unsigned* sp = d_fseg_;
            const unsigned* lp = d_flink_;
            long long ns = nfseg_;
            int gshift = 0;
            while ((1 << gshift) < skip_group_) ++gshift;
            void* sargs[] = {&a, &sp, &lp, &ns, &gshift};
            const long long threads = ns << gshift;
            const long long per_block = 256LL * kernel_segbb_->cpt;
            cuda_check(cudaLaunchKernel(kernel_segbb_->fn, dim3(unsigned((threads + per_block - 1) / per_block)),
                                        dim3(256), sargs, 0, stream_), "launch fluid segments");
            bb_dirty_ = true;
        } else if (kernel_seg_) {
            // (regularized cells fused: no fix-up launches after it)
            if (seg_fused_reg_) split_rare = false;
            // compacted masked sweep: one thread per cell of the listed segments
            // (also the first step of the fluid-segment sweep: it leaves every
            // listed cell current in both buffers)
            const unsigned* sp = d_seg_;
            long long ns = nseg_;
            int gshift = 0;
            while ((1 << gshift) < skip_group_) ++gshift;
            // segment-entry prefetch distance in blocks (DLB_SEG_PREFETCH; 0 = off)
            int pf = seg_prefetch_;
            int pack = seg_pack_;
            void* sargs[] = {&a, &sp, &ns, &gshift, &pf, &pack};
            const int sb = seg_block_;
            const long long threads = ns << gshift;
            const long long per_block = (long long)sb * kernel_seg_->cpt;
            cuda_check(cudaLaunchKernel(kernel_seg_->fn, dim3(unsigned((threads + per_block - 1) / per_block)),
                                        dim3(unsigned(sb)), sargs, 0, stream_), "launch segments");
            bb_prologue_ = false;
            bb_dirty_ = false;
        } else if (ke_requested_ && kernel_ke_) {
            if (!d_ke_) {
                cuda_check(cudaMalloc(&d_ke_, std::size_t(cells()) * sizeof(double)), "cudaMalloc kinetic energy");
                device_bytes_ += cells() * int64_t(sizeof(double));
            }
            a.ke = d_ke_;
            cuda_check(cudaLaunchKernel(kernel_ke_->fn, dim3(gx, gy, geo_.nz), block, args, 0, stream_),
                       "launch fused kinetic energy");
            ke_requested_ = false;
            ke_step_ = steps_ + 1;  // valid for the state after this step
        } else if (kernel_vec_ && !split_rare) {
            const int vw = 16 / int(sizeof(T));
            const unsigned vx = unsigned((geo_.nx / vw + 63) / 64), vy = unsigned((geo_.ny + 3) / 4);
            cuda_check(cudaLaunchKernel(kernel_vec_->fn, dim3(vx, vy, geo_.nz), dim3(64, 4, 1), args, 0, stream_),
                       "launch vectorised");
        } else {
            cuda_check(cudaLaunchKernel(split_rare ? kernel_main_->fn : fn, dim3(gx, gy, geo_.nz), block, args, 0,
                                        stream_), "launch");
        }
        if (split_rare) {
            // the main sweep treated the regularized cells as plain bulk cells;
            // recompute them (same f_in, later in stream order) with the full chain
            for (const ListLaunch& l : fixups_) {
                const unsigned long long* lp = d_fix_ + l.offset;
                long long n = l.count;
                int slot = l.slot;
                void* largs[] = {&a, &lp, &n, &slot};
                const long long blocks = std::min<long long>((n + 255) / 256, 148LL * 8);
                cuda_check(cudaLaunchKernel(l.kernel->fn, dim3(unsigned(blocks)), dim3(256), largs, 0, stream_),
                           "launch fixup");
            }
        }
        return;
    }
    // Linked z-slab (halo exchange over peer memory), per step:
    //   halo_stream_ (high priority): k_halo_wait (both neighbours finished the
    //     boundary planes of the previous step, i.e. our ghost planes are
    //     current) -> boundary launch (planes 0 and nz-1, peer push of the
    //     z-crossing links into the neighbours' ghost planes, completion signal)
    //   stream_: interior launch (planes 1..nz-2; reads no ghost plane)
    // forked after the previous step and joined before the next one: the
    // interior of step s needs both launches of step s-1 (its input planes, and
    // the boundary launch's reads of the buffer it overwrites), so the wait,
    // the boundary sweep and the NVLink transfer all overlap the interior.
    a.err = d_flags_ + 3;
    ++halo_steps_;
    // DLB_TRACE_HALO: timing events around the two branches (graphs disabled)
    cudaEvent_t* tr = nullptr;
    if (trace_halo_ && trace_ev_.size() + 5 <= 5 * 256) {
        for (int k = 0; k < 5; ++k) {
            cudaEvent_t e;
            cuda_check(cudaEventCreate(&e), "event");
            trace_ev_.push_back(e);
        }
        tr = trace_ev_.data() + trace_ev_.size() - 5;
    }
    // DLB_HALO_OVERLAP=0: the serialised variant (wait, boundary, interior on
    // one stream), kept for comparison
    const cudaStream_t hs = overlap_ ? halo_stream_ : stream_;
    if (overlap_) {
        cuda_check(cudaEventRecord(ev_fork_, stream_), "fork");
        cuda_check(cudaStreamWaitEvent(halo_stream_, ev_fork_, 0), "fork");
    }
    if (tr) cuda_check(cudaEventRecord(tr[0], hs), "trace");
    k_halo_wait<<<1, 1, 0, hs>>>(d_flags_, lower_.linked, upper_.linked, halo_timeout_ns_);
    cuda_check(cudaGetLastError(), "k_halo_wait");
    if (tr) cuda_check(cudaEventRecord(tr[1], hs), "trace");
    // AA updates in place: the interior launch of a step whose halo wait fails
    // would overwrite the kept state, so it starts after the wait (the wait
    // returns within microseconds when the neighbours keep pace); the
    // two-population interior writes the other buffer and need not wait
    if (aa() && overlap_) {
        cuda_check(cudaEventRecord(ev_wait_, hs), "wait event");
        cuda_check(cudaStreamWaitEvent(stream_, ev_wait_, 0), "wait event");
    }
    StepArgs<T> b = a;
    b.z_begin = 0;
    b.z_step = geo_.nz > 1 ? geo_.nz - 1 : 1;
    if (upper_.linked) {
        b.push_up = static_cast<T*>(upper_.buf[1 - parity]);
        b.up_dstride = upper_.dstride;
        b.sig_up = upper_.flag;
    }
    if (lower_.linked) {
        b.push_down = static_cast<T*>(lower_.buf[1 - parity]);
        b.down_dstride = lower_.dstride;
        b.down_ghost_z = lower_.nz;
        b.sig_down = lower_.flag;
    }
    b.counter = d_counter_;
    b.my_step = d_flags_ + 2;
    {
        void* args[] = {&b};
        const void* bfn = !aa() ? fn : (aa_odd_layout_ ? kernel_link_->fn : kernel_odd_link_->fn);
        cuda_check(cudaLaunchKernel(bfn, dim3(gx, gy, geo_.nz > 1 ? 2 : 1), block, args, 0, hs),
                   "launch boundary");
    }
    if (tr) cuda_check(cudaEventRecord(tr[2], hs), "trace");
    if (overlap_) cuda_check(cudaEventRecord(ev_join_, halo_stream_), "join");
    if (tr) cuda_check(cudaEventRecord(tr[3], stream_), "trace");
    if (geo_.nz > 2) {
        a.z_begin = 1;
        a.z_step = 1;
        void* args[] = {&a};
        cuda_check(cudaLaunchKernel(fn, dim3(gx, gy, geo_.nz - 2), block, args, 0, stream_),
                   "launch interior");
    }
    if (tr) cuda_check(cudaEventRecord(tr[4], stream_), "trace");
    if (overlap_) cuda_check(cudaStreamWaitEvent(stream_, ev_join_, 0), "join");
    if (aa()) aa_odd_layout_ = !aa_odd_layout_;
}

void Lattice::enqueue_step() {
    DeviceGuard dg(device_);
    if (d_.precision_bits == 64) launch_step<double>(cur_);
    else launch_step<float>(cur_);
    if (!aa()) cur_ = 1 - cur_;
    ++steps_;
}

void Lattice::invalidate_graph() {
    if (graph_) cudaGraphExecDestroy(graph_);
    graph_ = nullptr;
    graph_version_ = g_graph_version.fetch_add(1);
}

namespace {
// The one cached multi-slab graph (dlb_lattices_step / DeviceRun::advance), kGroupSteps steps:
// keyed by the slabs, their graph versions and buffer parities at capture.
struct GroupGraph {
    std::vector<const void*> lats;
    std::vector<uint64_t> versions;
    std::vector<int> parity;
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t fork = nullptr;
    std::vector<cudaEvent_t> join;
    int device = -1;
};
GroupGraph g_group;
std::mutex g_group_mu;
}  // namespace

void Lattice::step_group(const std::vector<Lattice*>& lats, int64_t nsteps) {
    if (lats.empty() || nsteps <= 0) return;
    if (lats.size() == 1) {
        lats[0]->step(nsteps);
        return;
    }
    // steps per replay: the slabs meet at the graph's end (the first slab's
    // stream waits for all), so a longer graph keeps them pipelined longer
    constexpr int kGroupSteps = 8;
    const int dev = lats[0]->device_;
    bool graphable = nsteps >= kGroupSteps;
    for (Lattice* l : lats)
        graphable = graphable && l->device_ == dev && !l->trace_halo_ && !l->ke_requested_ && !l->kernel_segbb_ &&
                    !l->kernel_tma_;  // (the TMA kernels' one-off envelope refresh stays out of graphs)
    // Only where the host is the bottleneck: enqueueing a slab's step costs
    // ~9 us of host time; slabs moving more than ~64 MB per step (~10 us of
    // HBM time) keep the device busy without a graph, and there the graph's
    // barrier every kGroupSteps steps costs more than it saves (8 slabs of a
    // 256^3 fp32 lattice: 444 vs 429 us per step; 8 slabs of config 1's 64^3
    // fp64 cavity: 37 vs 74 us per step, profiles/r02b_summary.md)
    int64_t max_bytes = 0;
    for (Lattice* l : lats) max_bytes = std::max(max_bytes, l->step_bytes());
    const char* ge = std::getenv("DLB_GROUP_GRAPH");
    if (ge) graphable = graphable && ge[0] == '1';
    else graphable = graphable && max_bytes <= (int64_t(64) << 20);
    int64_t k = 0;
    auto eager = [&] {
        for (Lattice* l : lats) l->enqueue_step();
        ++k;
    };
    if (!graphable) {
        for (; k < nsteps;) eager();
        return;
    }
    for (Lattice* l : lats) {
        DeviceGuard dg(l->device_);
        l->prepare_compact();  // gathers stay out of the graph
    }
    auto parity_of = [](const Lattice* l) { return l->aa() ? int(l->aa_odd_layout_) : l->cur_; };
    std::lock_guard<std::mutex> lock(g_group_mu);
    GroupGraph& G = g_group;
    auto matches = [&] {
        if (!G.exec || G.lats.size() != lats.size() || G.device != dev) return false;
        for (std::size_t i = 0; i < lats.size(); ++i)
            if (G.lats[i] != lats[i] || G.versions[i] != lats[i]->graph_version_ ||
                G.parity[i] != parity_of(lats[i]))
                return false;
        return true;
    };
    DeviceGuard dg(dev);
    if (!matches()) {
        // a graph of the other parity: one eager step aligns every slab with it
        if (G.exec && G.lats.size() == lats.size()) {
            bool same = G.device == dev;
            for (std::size_t i = 0; same && i < lats.size(); ++i)
                same = G.lats[i] == lats[i] && G.versions[i] == lats[i]->graph_version_;
            if (same) eager();
        }
    }
    if (!matches()) {
        if (G.exec) cudaGraphExecDestroy(G.exec);
        G.exec = nullptr;
        if (!G.fork) cuda_check(cudaEventCreateWithFlags(&G.fork, cudaEventDisableTiming), "event");
        while (G.join.size() < lats.size()) {
            cudaEvent_t e;
            cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            G.join.push_back(e);
        }
        struct Saved {
            int cur;
            bool odd, bb_dirty, bb_prologue, cmp_dirty;
            int64_t steps, halo_steps;
        };
        std::vector<Saved> saved;
        for (Lattice* l : lats)
            saved.push_back({l->cur_, l->aa_odd_layout_, l->bb_dirty_, l->bb_prologue_, l->cmp_dirty_, l->steps_,
                             l->halo_steps_});
        cudaStream_t origin = lats[0]->stream_;
        cudaGraph_t g = nullptr;
        auto restore = [&] {
            for (std::size_t i = 0; i < lats.size(); ++i) {
                Lattice* l = lats[i];
                const Saved& v = saved[i];
                l->cur_ = v.cur;
                l->aa_odd_layout_ = v.odd;
                l->bb_dirty_ = v.bb_dirty;
                l->bb_prologue_ = v.bb_prologue;
                l->cmp_dirty_ = v.cmp_dirty;
                l->steps_ = v.steps;
                l->halo_steps_ = v.halo_steps;
            }
        };
        cuda_check(cudaStreamBeginCapture(origin, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
            cuda_check(cudaEventRecord(G.fork, origin), "fork");
            for (std::size_t i = 1; i < lats.size(); ++i)
                cuda_check(cudaStreamWaitEvent(lats[i]->stream_, G.fork, 0), "fork");
            for (int s = 0; s < kGroupSteps; ++s)
                for (Lattice* l : lats) {
                    if (l->d_.precision_bits == 64) l->launch_step<double>(l->cur_);
                    else l->launch_step<float>(l->cur_);
                    if (!l->aa()) l->cur_ = 1 - l->cur_;
                }
            for (std::size_t i = 1; i < lats.size(); ++i) {
                cuda_check(cudaEventRecord(G.join[i], lats[i]->stream_), "join");
                cuda_check(cudaStreamWaitEvent(origin, G.join[i], 0), "join");
            }
        } catch (...) {
            // close the capture so the streams stay usable, then report
            cudaGraph_t bad = nullptr;
            cudaStreamEndCapture(origin, &bad);
            if (bad) cudaGraphDestroy(bad);
            cudaGetLastError();
            restore();
            throw;
        }
        cuda_check(cudaStreamEndCapture(origin, &g), "end capture");
        restore();
        cuda_check(cudaGraphInstantiateWithFlags(&G.exec, g, cudaGraphInstantiateFlagUseNodePriority),
                   "graph instantiate");
        cudaGraphDestroy(g);
        G.lats.assign(lats.begin(), lats.end());
        G.versions.clear();
        G.parity.clear();
        for (Lattice* l : lats) {
            G.versions.push_back(l->graph_version_);
            G.parity.push_back(parity_of(l));
        }
        G.device = dev;
    }
    if (nsteps - k >= kGroupSteps) {
        cudaStream_t origin = lats[0]->stream_;
        // the graph runs on the first slab's stream: order it after every
        // slab's earlier work, and every slab's later work after it
        for (std::size_t i = 1; i < lats.size(); ++i) {
            cuda_check(cudaEventRecord(G.join[i], lats[i]->stream_), "order");
            cuda_check(cudaStreamWaitEvent(origin, G.join[i], 0), "order");
        }
        for (; k + kGroupSteps <= nsteps; k += kGroupSteps) {
            cuda_check(cudaGraphLaunch(G.exec, origin), "graph launch");
            for (Lattice* l : lats) {
                l->steps_ += kGroupSteps;
                if (l->lower_.linked || l->upper_.linked) l->halo_steps_ += kGroupSteps;
                if (l->kernel_cmp_) l->cmp_dirty_ = true;
            }
        }
        cuda_check(cudaEventRecord(G.fork, origin), "order");
        for (std::size_t i = 1; i < lats.size(); ++i) cuda_check(cudaStreamWaitEvent(lats[i]->stream_, G.fork, 0), "order");
    }
    for (; k < nsteps;) eager();
}

void Lattice::ensure_graph() {
    if (graph_) return;
    prepare_compact();  // the gather stays out of the replayed graph
    if (kernel_tma_ && !envelope_valid_ && !(lower_.linked || upper_.linked)) {
        refresh_envelope(cur_);  // keep the one-off refresh out of the replayed graph
        envelope_valid_ = true;
    }
    const int cur = cur_;
    const bool odd = aa_odd_layout_;
    const int64_t steps = steps_, halo_steps = halo_steps_;
    const bool bb_dirty = bb_dirty_, bb_prologue = bb_prologue_, cmp_dirty = cmp_dirty_;
    cudaGraph_t g = nullptr;
    cuda_check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
        enqueue_step();
        enqueue_step();
    } catch (...) {
        // close the capture so the stream stays usable, restore, report
        cudaGraph_t bad = nullptr;
        cudaStreamEndCapture(stream_, &bad);
        if (bad) cudaGraphDestroy(bad);
        cudaGetLastError();
        cur_ = cur;
        aa_odd_layout_ = odd;
        steps_ = steps;
        halo_steps_ = halo_steps;
        bb_dirty_ = bb_dirty;
        bb_prologue_ = bb_prologue;
        cmp_dirty_ = cmp_dirty;
        throw;
    }
    cuda_check(cudaStreamEndCapture(stream_, &g), "end capture");
    cur_ = cur;
    aa_odd_layout_ = odd;
    steps_ = steps;
    halo_steps_ = halo_steps;
    bb_dirty_ = bb_dirty;
    bb_prologue_ = bb_prologue;
    cmp_dirty_ = cmp_dirty;
    // keep the halo branch's stream priority inside the replayed graph
    cuda_check(cudaGraphInstantiateWithFlags(&graph_, g, cudaGraphInstantiateFlagUseNodePriority),
               "graph instantiate");
    cudaGraphDestroy(g);
}

// Steps are replayed as a CUDA graph of two consecutive steps (launch latency
// and host overhead amortised; the halo wait / push / signal nodes are
// device-side, so linked slabs replay safely too).
bool Lattice::request_kinetic() {
    if (!kernel_ke_ || lower_.linked || upper_.linked) return false;
    ke_requested_ = true;
    return true;
}

void Lattice::step(int64_t nsteps) {
    if (nsteps <= 0) return;
    check_dispatch();
    DeviceGuard dg(device_);
    // a requested fused kinetic energy belongs to the LAST step of this call;
    // the others (and any captured graph) run the plain kernel
    const bool ke_last = ke_requested_;
    ke_requested_ = false;
    if (ke_last) --nsteps;
    int64_t k = 0;
    if (kernel_coop_ && nsteps >= 2 && !(lower_.linked || upper_.linked) && !kernel_tma_) {
        // small lattice: all nsteps in one persistent cooperative launch
        if (d_.precision_bits == 64) launch_coop<double>(nsteps);
        else launch_coop<float>(nsteps);
        k = nsteps;
    }
    if (kernel_segbb_ && bb_prologue_ && k < nsteps && !(lower_.linked || upper_.linked)) {
        enqueue_step();  // the fluid-segment sweep's first step (k_seg) stays out of the graph
        ++k;
    }
    if (nsteps - k >= 4 && !trace_halo_) {
        const bool aligned = aa() ? aa_odd_layout_ : cur_ == 0;
        if (!aligned) {
            enqueue_step();
            ++k;
        }
        ensure_graph();
        for (; k + 2 <= nsteps; k += 2) {
            cuda_check(cudaGraphLaunch(graph_, stream_), "graph launch");
            steps_ += 2;
            if (lower_.linked || upper_.linked) halo_steps_ += 2;
            if (kernel_segbb_) bb_dirty_ = true;
            if (kernel_cmp_) cmp_dirty_ = true;
        }
    }
    for (; k < nsteps; ++k) enqueue_step();
    if (ke_last) {
        ke_requested_ = true;
        enqueue_step();
        ke_requested_ = false;
    }
}

// MultiBlockRun::exchange (multiblock.hpp:142-143) for a z-slab: copy this
// slab's top / bottom interior planes into the neighbours' ghost planes of the
// CURRENT state buffer (whole planes; only the c_z-crossing directions are
// read from there). Needed once before the first step after (re)filling the
// state; afterwards every step's boundary launch pushes the halo itself.
// Neighbours must be quiescent (lockstep, as in the reference).
void Lattice::quiesce() {
    DeviceGuard dg(device_);
    cuda_check(cudaStreamSynchronize(halo_stream_), "sync");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
}

void Lattice::exchange() {
    DeviceGuard dg(device_);
    quiesce();
    // (re)priming the ghosts clears a previous exchange error: the caller has
    // brought the slabs back to one step count (MultiBlockRun::exchange)
    cuda_check(cudaMemsetAsync(d_flags_ + 3, 0, sizeof(unsigned long long), stream_), "clear error");
    exchange_failed_ = false;
    const int s = d_.precision_bits / 8;
    const std::size_t plane_bytes = std::size_t(geo_.plane) * s;
    auto plane_ptr = [&](void* origin_dir0, long long dstride, int i, int z) {
        return static_cast<char*>(origin_dir0) +
               (std::size_t(i) * dstride + std::size_t(z) * geo_.plane - geo_.pitch - 1) * s;
    };
    for (int i = 0; i < d_.q; ++i) {
        const int cz = i == 0 ? 0 : (d_.q == 19 ? kCz19[i] : kCz27[i]);
        // AA (linked slabs rest in the even layout, f_i(x) = A[opp(i)][x]): the
        // neighbour's odd step reads our boundary cell's f_i from its ghost slot
        // A[i] (k_aa); in the odd layout the next step is even and reads no ghost
        const int src = aa() ? (i == 0 ? 0 : ((i & 1) ? i + 1 : i - 1)) : i;
        if (aa() && aa_odd_layout_) break;
        if (cz > 0 && upper_.linked)
            cuda_check(cudaMemcpyAsync(plane_ptr(upper_.buf[cur_], upper_.dstride, i, -1),
                                       plane_ptr(origin(cur_), geo_.dstride, src, geo_.nz - 1),
                                       plane_bytes, cudaMemcpyDefault, stream_), "halo exchange");
        if (cz < 0 && lower_.linked)
            cuda_check(cudaMemcpyAsync(plane_ptr(lower_.buf[cur_], lower_.dstride, i, lower_.nz),
                                       plane_ptr(origin(cur_), geo_.dstride, src, 0),
                                       plane_bytes, cudaMemcpyDefault, stream_), "halo exchange");
    }
    cuda_check(cudaStreamSynchronize(stream_), "halo exchange");
}

void Lattice::checksum(unsigned long long* per_dir, bool active_only) {
    DeviceGuard dg(device_);
    finalize_walls();
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    unsigned long long* d = static_cast<unsigned long long*>(staging_);
    cuda_check(cudaMemsetAsync(d, 0, 27 * 8, stream_), "memset");
    const uint8_t* skip = nullptr;
    if (active_only) {
        std::vector<uint8_t> nd(256, 0);
        for (std::size_t k = 0; k < chains_.size(); ++k) nd[k] = kind_bits(chains_[k]) == KM_NODYN;
        uint8_t* dsk = static_cast<uint8_t*>(staging_) + 4096;
        cuda_check(cudaMemcpyAsync(dsk, nd.data(), nd.size(), cudaMemcpyHostToDevice, stream_), "h2d");
        skip = dsk;
    }
    const int mode = !aa() ? 0 : (aa_odd_layout_ ? 2 : 1);
    const int grid = grid_for(cells());
    const void* o = origin(cur_);
    const long long gnx = geo_.nx, gny = geo_.ny;
    if (d_.precision_bits == 64) {
        if (d_.q == 19) k_checksum<double, 19><<<grid, 256, 0, stream_>>>((const double*)o, geo_, mode, d_.z_origin, gnx, gny, d, d_slot_, uniform_slot_, skip);
        else k_checksum<double, 27><<<grid, 256, 0, stream_>>>((const double*)o, geo_, mode, d_.z_origin, gnx, gny, d, d_slot_, uniform_slot_, skip);
    } else {
        if (d_.q == 19) k_checksum<float, 19><<<grid, 256, 0, stream_>>>((const float*)o, geo_, mode, d_.z_origin, gnx, gny, d, d_slot_, uniform_slot_, skip);
        else k_checksum<float, 27><<<grid, 256, 0, stream_>>>((const float*)o, geo_, mode, d_.z_origin, gnx, gny, d, d_slot_, uniform_slot_, skip);
    }
    cuda_check(cudaGetLastError(), "k_checksum");
    cuda_check(cudaMemcpyAsync(per_dir, d, size_t(d_.q) * 8, cudaMemcpyDeviceToHost, stream_), "d2h");
    cuda_check(cudaStreamSynchronize(stream_), "checksum");
}

void Lattice::gather_macroscopic(double* rho, double* ux, double* uy, double* uz) {
    DeviceGuard dg(device_);
    finalize_walls();
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    std::vector<MacroSlot> ms(std::max<std::size_t>(chains_.size(), 1));
    for (std::size_t s = 0; s < chains_.size(); ++s) {
        const LinkType t = chains_[s].links.back().type;
        ms[s].kind = t == LinkType::MovingBounceBack ? KIND_MBB
                   : (t == LinkType::BGK || t == LinkType::TRT || t == LinkType::RR) ? KIND_COLLIDE
                                                                                      : KIND_BB;
        for (int a = 0; a < 3; ++a) {
            const double w = chains_[s].params.wall_velocity[a];
            ms[s].uw[a] = d_.precision_bits == 64 ? w : double(float(w));  // T-cast, as the recipe holds it
        }
    }
    const std::size_t ms_bytes = ms.size() * sizeof(MacroSlot);
    char* st = static_cast<char*>(staging_);
    cuda_check(cudaMemcpyAsync(st, ms.data(), ms_bytes, cudaMemcpyHostToDevice, stream_), "h2d");
    const long long plane_cells = (long long)geo_.nx * geo_.ny;
    const std::size_t room = staging_bytes_ - 4096;
    const int zc = int(std::max<long long>(1, (long long)(room / 32) / plane_cells));
    double* out = reinterpret_cast<double*>(st + 4096);
    const int mode = !aa() ? 0 : (aa_odd_layout_ ? 2 : 1);
    for (int z0 = 0; z0 < geo_.nz; z0 += zc) {
        const int nzc = std::min(zc, geo_.nz - z0);
        const long long n = plane_cells * nzc;
        const int grid = grid_for(n);
        const void* o = origin(cur_);
        const MacroSlot* dms = reinterpret_cast<const MacroSlot*>(st);
        if (d_.precision_bits == 64) {
            if (d_.q == 19) k_macro<double, 19><<<grid, 256, 0, stream_>>>((const double*)o, geo_, mode, d_slot_, uniform_slot_, dms, z0, nzc, out, out + n, out + 2 * n, out + 3 * n);
            else k_macro<double, 27><<<grid, 256, 0, stream_>>>((const double*)o, geo_, mode, d_slot_, uniform_slot_, dms, z0, nzc, out, out + n, out + 2 * n, out + 3 * n);
        } else {
            if (d_.q == 19) k_macro<float, 19><<<grid, 256, 0, stream_>>>((const float*)o, geo_, mode, d_slot_, uniform_slot_, dms, z0, nzc, out, out + n, out + 2 * n, out + 3 * n);
            else k_macro<float, 27><<<grid, 256, 0, stream_>>>((const float*)o, geo_, mode, d_slot_, uniform_slot_, dms, z0, nzc, out, out + n, out + 2 * n, out + 3 * n);
        }
        cuda_check(cudaGetLastError(), "k_macro");
        const long long off = plane_cells * z0;
        double* dst[4] = {rho, ux, uy, uz};
        for (int k = 0; k < 4; ++k)
            cuda_check(cudaMemcpyAsync(dst[k] + off, out + k * n, n * 8, cudaMemcpyDeviceToHost, stream_), "d2h");
        cuda_check(cudaStreamSynchronize(stream_), "gather_macroscopic");
    }
}

void Lattice::check_error_flag() {
    DeviceGuard dg(device_);
    if (!(lower_.linked || upper_.linked)) return;
    if (exchange_failed_) return;  // reported once; the kept state stays readable
    unsigned long long fl[4] = {0, 0, 0, 0};
    cuda_check(cudaMemcpy(fl, d_flags_, sizeof(fl), cudaMemcpyDeviceToHost), "read flags");
    if (!fl[3]) return;
    exchange_failed_ = true;
    // flags[3] = 1-based index of the step whose halo wait timed out; that step
    // and every later one wrote nothing, so the state after the last completed
    // step (flags[2] of them) is intact in the buffer of its parity.
    const int64_t done = int64_t(fl[3]) - 1;
    const int64_t failed = halo_steps_ - done;  // enqueued linked steps that wrote nothing
    if (failed > 0) {
        if (failed & 1) {
            if (aa()) aa_odd_layout_ = !aa_odd_layout_;
            else cur_ = 1 - cur_;
        }
        steps_ -= failed;
        halo_steps_ = done;
        invalidate_graph();
    }
    throw ExchangeError("halo exchange timed out waiting for a neighbour at step " + std::to_string(fl[3]) +
                        " (state kept after step " + std::to_string(done) + ")");
}

std::vector<double> Lattice::halo_trace(bool consume) {
    DeviceGuard dg(device_);
    quiesce();
    std::vector<double> out;
    if (trace_ev_.empty()) return out;
    if (!consume) {
        out.resize(trace_ev_.size());
        return out;
    }
    for (std::size_t k = 0; k < trace_ev_.size(); ++k) {
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, trace_ev_[0], trace_ev_[k]), "elapsed");
        out.push_back(double(ms));
    }
    for (cudaEvent_t e : trace_ev_) cudaEventDestroy(e);
    trace_ev_.clear();
    return out;
}

void Lattice::links(int* lower, int* upper, int64_t* halo_bytes) const {
    auto code = [](const Peer& p) { return p.linked ? (p.other_gpu ? 2 : 1) : 0; };
    *lower = code(lower_);
    *upper = code(upper_);
    const int cross = d_.q == 19 ? 5 : 9;  // links with c_z = +1 (or -1)
    *halo_bytes = int64_t(int(lower_.linked) + int(upper_.linked)) * geo_.nx * geo_.ny * cross *
                  (d_.precision_bits / 8);
}

void Lattice::set_halo_timeout(double seconds) {
    if (!(seconds > 0)) throw std::invalid_argument("halo timeout must be positive");
    halo_timeout_ns_ = static_cast<unsigned long long>(seconds * 1e9);
    invalidate_graph();
}

void Lattice::synchronize() {
    DeviceGuard dg(device_);
    cuda_check(cudaStreamSynchronize(stream_), "step");
    check_error_flag();
}

double Lattice::time_steps(int64_t nsteps) {
    check_dispatch();
    DeviceGuard dg(device_);
    if (nsteps >= 4) {  // build the graph outside the timed region
        const bool aligned = aa() ? aa_odd_layout_ : cur_ == 0;
        if (!aligned) step(1);
        ensure_graph();
    }
    cuda_check(cudaEventRecord(ev0_, stream_), "event");
    step(nsteps);
    cuda_check(cudaEventRecord(ev1_, stream_), "event");
    cuda_check(cudaEventSynchronize(ev1_), "event sync");
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, ev0_, ev1_), "elapsed");
    check_error_flag();
    return double(ms);
}

void Lattice::link_lower(Lattice& lower) {
    invalidate_graph();
    lower.invalidate_graph();
    if (aa() != lower.aa()) throw std::invalid_argument("linked slabs must share the storage layout");
    // `lower` sits directly below this slab: lower's top plane feeds our ghost
    // z = -1, our bottom plane feeds lower's ghost z = lower.nz.
    if (lower.geo_.nx != geo_.nx || lower.geo_.ny != geo_.ny || lower.d_.q != d_.q ||
        lower.d_.precision_bits != d_.precision_bits)
        throw std::invalid_argument("linked slabs must share nx, ny, q and precision");
    if (lower.device_ != device_) {
        int ok = 0;
        cuda_check(cudaDeviceCanAccessPeer(&ok, device_, lower.device_), "peer query");
        if (!ok) throw ExchangeError("devices have no peer access");
        cudaSetDevice(device_);
        cudaDeviceEnablePeerAccess(lower.device_, 0);
        cudaSetDevice(lower.device_);
        cudaDeviceEnablePeerAccess(device_, 0);
        cudaGetLastError();
    }
    lower_.linked = true;
    lower_.other_gpu = lower.upper_.other_gpu = lower.device_ != device_;
    // the z neighbours now provide the wrap (a single slab may be linked to
    // itself: the one-slab-per-GPU step on one GPU)
    geo_.per_z = lower.geo_.per_z = 0;
    lower_.buf[0] = lower.origin(0);
    lower_.buf[1] = lower.origin(1);
    lower_.dstride = lower.geo_.dstride;
    lower_.nz = lower.geo_.nz;
    lower_.flag = lower.d_flags_ + 1;  // we are lower's upper neighbour
    lower.upper_.linked = true;
    lower.upper_.buf[0] = origin(0);
    lower.upper_.buf[1] = origin(1);
    lower.upper_.dstride = geo_.dstride;
    lower.upper_.nz = geo_.nz;
    lower.upper_.flag = d_flags_ + 0;  // lower is our lower neighbour
    // an AA slab's state crosses the faces in the odd layout: linking clears
    // the state (fill / upload after linking, as MultiBlockRun does)
    reset_aa();
    lower.reset_aa();
}

namespace {
struct IpcBlob {
    uint32_t magic;
    int32_t q, bits, nx, ny, nz;
    int32_t device;
    int32_t aa;        // storage layout (AA slabs link only to AA slabs)
    char pci_bus[32];  // the exporting slab's GPU (reported by links(): peer on another GPU or not)
    long long dstride, base_off_bytes;
    cudaIpcMemHandle_t buf[2];
    cudaIpcMemHandle_t flags;
};
constexpr uint32_t kIpcMagic = 0x444c4231;  // "DLB1"
}  // namespace

std::vector<uint8_t> Lattice::export_ipc() const {
    IpcBlob b{};
    b.magic = kIpcMagic;
    b.q = d_.q;
    b.bits = d_.precision_bits;
    b.nx = geo_.nx;
    b.ny = geo_.ny;
    b.nz = geo_.nz;
    b.aa = int(aa());
    b.dstride = geo_.dstride;
    b.base_off_bytes = base_off_ * (d_.precision_bits / 8);
    DeviceGuard dg(device_);
    b.device = device_;
    cuda_check(cudaDeviceGetPCIBusId(b.pci_bus, int(sizeof(b.pci_bus)), device_), "pci bus id");
    for (int k = 0; k < 2; ++k) cuda_check(cudaIpcGetMemHandle(&b.buf[k], buf_[k]), "ipc handle");
    cuda_check(cudaIpcGetMemHandle(&b.flags, d_flags_), "ipc handle");
    std::vector<uint8_t> out(sizeof(b));
    std::memcpy(out.data(), &b, sizeof(b));
    return out;
}

void Lattice::link_ipc(int side, const void* blob, std::size_t len) {
    invalidate_graph();
    if (len != sizeof(IpcBlob)) throw std::invalid_argument("bad IPC blob size");
    IpcBlob b;
    std::memcpy(&b, blob, sizeof(b));
    if (b.magic != kIpcMagic) throw std::invalid_argument("bad IPC blob");
    if (b.nx != geo_.nx || b.ny != geo_.ny || b.q != d_.q || b.bits != d_.precision_bits)
        throw std::invalid_argument("linked slabs must share nx, ny, q and precision");
    if (b.aa != int(aa())) throw std::invalid_argument("linked slabs must share the storage layout");
    DeviceGuard dg(device_);
    Peer& p = side == 0 ? lower_ : upper_;
    void* bases[3];
    // an AA slab has one population array (both handles name it): open it once
    cuda_check(cudaIpcOpenMemHandle(&bases[0], b.buf[0], cudaIpcMemLazyEnablePeerAccess), "ipc open");
    if (b.aa) bases[1] = bases[0];
    else cuda_check(cudaIpcOpenMemHandle(&bases[1], b.buf[1], cudaIpcMemLazyEnablePeerAccess), "ipc open");
    cuda_check(cudaIpcOpenMemHandle(&bases[2], b.flags, cudaIpcMemLazyEnablePeerAccess), "ipc open");
    p.ipc_opened = b.aa ? std::vector<void*>{bases[0], bases[2]} : std::vector<void*>{bases[0], bases[1], bases[2]};
    p.linked = true;
    p.buf[0] = static_cast<char*>(bases[0]) + b.base_off_bytes;
    p.buf[1] = static_cast<char*>(bases[1]) + b.base_off_bytes;
    p.dstride = b.dstride;
    p.nz = b.nz;
    char mine[32] = {0};
    cuda_check(cudaDeviceGetPCIBusId(mine, int(sizeof(mine)), device_), "pci bus id");
    p.other_gpu = std::strncmp(mine, b.pci_bus, sizeof(mine)) != 0;
    // we are the peer's upper neighbour if it is our lower one, and vice versa
    p.flag = static_cast<unsigned long long*>(bases[2]) + (side == 0 ? 1 : 0);
    reset_aa();  // see link_lower
}

// ---------------------------------------------------------------------------
// Random Boolean sphere pack: spheres of radius r with
// uniform centres (mt19937_64, periodic placement) are added until the pore
// fraction drops to target or below; written as raw u8, 255 = solid, x fastest.
double sphere_pack(int64_t nx, int64_t ny, int64_t nz, double radius, double target_porosity,
                   uint64_t seed, uint8_t* out) {
    if (nx < 1 || ny < 1 || nz < 1 || radius <= 0 || target_porosity <= 0 || target_porosity >= 1)
        throw std::invalid_argument("invalid sphere-pack parameters");
    const int64_t n = nx * ny * nz;
    std::memset(out, 0, std::size_t(n));
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> ux(0.0, double(nx)), uy(0.0, double(ny)), uz(0.0, double(nz));
    int64_t solid = 0;
    const int r = int(std::ceil(radius));
    const double r2 = radius * radius;
    while (double(n - solid) / double(n) > target_porosity) {
        const double cx = ux(rng), cy = uy(rng), cz = uz(rng);
        for (int dz = -r - 1; dz <= r + 1; ++dz) {
            const int64_t z = int64_t(std::floor(cz)) + dz;
            const double ddz = (double(z) + 0.5) - cz;
            if (ddz * ddz > r2) continue;
            const int64_t zz = ((z % nz) + nz) % nz;
            for (int dy = -r - 1; dy <= r + 1; ++dy) {
                const int64_t y = int64_t(std::floor(cy)) + dy;
                const double ddy = (double(y) + 0.5) - cy;
                if (ddz * ddz + ddy * ddy > r2) continue;
                const int64_t yy = ((y % ny) + ny) % ny;
                for (int dx = -r - 1; dx <= r + 1; ++dx) {
                    const int64_t x = int64_t(std::floor(cx)) + dx;
                    const double ddx = (double(x) + 0.5) - cx;
                    if (ddz * ddz + ddy * ddy + ddx * ddx > r2) continue;
                    const int64_t xx = ((x % nx) + nx) % nx;
                    uint8_t& v = out[std::size_t((zz * ny + yy) * nx + xx)];
                    if (!v) {
                        v = 255;
                        ++solid;
                    }
                }
            }
        }
    }
    return double(n - solid) / double(n);
}

}  // namespace dlb
