// GPU-resident diagnostics: the sampling step after the update.
//
// The reference gathers rho / u of the whole domain to the host
// (MultiBlockRun::gather_macroscopic, proj/src/multiblock.cpp:443-484) and then
// reduces them there (Driver::sample / porous_extras, proj/src/runner.cpp:
// 346-423; diag::kinetic_energy / vorticity_fd8 / enstrophy,
// proj/src/diagnostics.cpp:25-120). Here the per-cell values are produced from
// the resident populations chunk by chunk (z planes) into a device scratch
// buffer and reduced on the device with the reference's tree order
// (diagnostics.cpp:10-18): the host plans which tree nodes each chunk owns
// (tree.hpp), the device sums them, the host combines the nodes above.
//
// Compiled with -fmad=false: every value is the reference's double
// expression with the same association (no contraction).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "canon.cuh"
#include "lattice.hpp"
#include "tree.hpp"

namespace dlb {
namespace {

struct DiagSlot {
    int kind;   // KIND_* of the chain's recipe
    int fluid;  // runner.cpp:668-676: last link not BounceBack / NoDynamics / MovingBounceBack
    double uw[3];
};

// gather_macroscopic semantics for one cell (multiblock.cpp:458-478).
template <typename T, int Q>
__device__ __forceinline__ void cell_macro(const T* origin0, const Geo& g, int aa_mode, const DiagSlot& s,
                                           int x, int y, int z, double& r, double (&u)[3]) {
    r = 1.0;
    u[0] = u[1] = u[2] = 0.0;
    if (s.kind == KIND_COLLIDE) {
        double f[Q];
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            f[i] = double(canon_load<T, Q, i>(origin0, g, x, y, z, aa_mode));
        });
        Cell<double, Q>::rho_u(f, r, u);
    } else if (s.kind == KIND_MBB) {
        u[0] = s.uw[0];
        u[1] = s.uw[1];
        u[2] = s.uw[2];
    }
}

// Per-cell values of the cell quantities over x in [xb, xe), all y, local
// planes [z0, z0 + nzc), x fastest; flag = 1 where the cell is in the sequence.
template <typename T, int Q>
__global__ void k_cell_values(const T* origin0, Geo g, int aa_mode, const uint8_t* slot, int uniform_slot,
                              const DiagSlot* ds, int quantity, int z0, int nzc, int xb, int xe,
                              const double* uprev, long long ncell, double* val, uint8_t* flag) {
    const int w = xe - xb;
    const long long n = static_cast<long long>(w) * g.ny * nzc;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int x = xb + int(c % w);
        const int y = int((c / w) % g.ny);
        const int z = z0 + int(c / (static_cast<long long>(w) * g.ny));
        const long long cell = (static_cast<long long>(z) * g.ny + y) * g.nx + x;
        const DiagSlot& s = ds[slot ? slot[cell] : uniform_slot];
        double r, u[3];
        cell_macro<T, Q>(origin0, g, aa_mode, s, x, y, z, r, u);
        double v;
        switch (quantity) {
            case DLB_Q_KINETIC:  // diagnostics.cpp:28
                v = 0.5 * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
                break;
            case DLB_Q_DU_NUM: {  // runner.cpp:436-439
                const double dx = u[0] - uprev[cell];
                const double dy = u[1] - uprev[ncell + cell];
                const double dz = u[2] - uprev[2 * ncell + cell];
                v = dx * dx + dy * dy + dz * dz;
                break;
            }
            case DLB_Q_DU_DEN:  // runner.cpp:440
                v = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
                break;
            case DLB_Q_PRESSURE_FLUID:  // runner.cpp:358 (D3Q19::cs2 = 1.0 / 3.0)
                v = (1.0 / 3.0) * r;
                break;
            case DLB_Q_RHO_FLUID:
                v = r;
                break;
            default:  // UX_FLUID, UX_ALL
                v = u[0];
        }
        val[c] = v;
        if (flag) flag[c] = uint8_t(s.fluid);
    }
}

// Velocity of local planes [z0, z0 + np) as [plane][ux|uy|uz][y][x].
template <typename T, int Q>
__global__ void k_u_planes(const T* origin0, Geo g, int aa_mode, const uint8_t* slot, int uniform_slot,
                           const DiagSlot* ds, int z0, int np, double* out) {
    const long long pc = static_cast<long long>(g.nx) * g.ny;
    const long long n = pc * np;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int x = int(c % g.nx);
        const int y = int((c / g.nx) % g.ny);
        const int p = int(c / pc);
        const int z = z0 + p;
        const long long cell = (static_cast<long long>(z) * g.ny + y) * g.nx + x;
        double r, u[3];
        cell_macro<T, Q>(origin0, g, aa_mode, ds[slot ? slot[cell] : uniform_slot], x, y, z, r, u);
        double* o = out + p * 3 * pc + static_cast<long long>(y) * g.nx + x;
        o[0] = u[0];
        o[pc] = u[1];
        o[2 * pc] = u[2];
    }
}

// diag::vorticity_fd8 + enstrophy values (diagnostics.cpp:33-120) of the valid
// box [vx0, vx1) x [vy0, vy1) x window planes [4, 4 + nzc), from the velocity
// window U ([plane][comp][y][x], 4 extra planes on each side).
__device__ __forceinline__ double fd8_along(const double* comp, int nx, int ny, long long pc, int x, int y,
                                            int p, int axis) {
    const double coeff[4] = {4.0 / 5.0, -1.0 / 5.0, 4.0 / 105.0, -1.0 / 280.0};
    double d = 0.0;
#pragma unroll
    for (int k = 1; k <= 4; ++k) {
        long long ip, im;
        if (axis == 0) {
            ip = static_cast<long long>(y) * nx + (x + k) % nx;
            im = static_cast<long long>(y) * nx + (x - k + 4 * nx) % nx;
            ip += p * 3 * pc;
            im += p * 3 * pc;
        } else if (axis == 1) {
            ip = static_cast<long long>((y + k) % ny) * nx + x + p * 3 * pc;
            im = static_cast<long long>((y - k + 4 * ny) % ny) * nx + x + p * 3 * pc;
        } else {
            ip = static_cast<long long>(y) * nx + x + (p + k) * 3 * pc;
            im = static_cast<long long>(y) * nx + x + (p - k) * 3 * pc;
        }
        d += coeff[k - 1] * (comp[ip] - comp[im]);
    }
    return d;
}

__global__ void k_enstrophy_values(const double* U, int nx, int ny, int vx0, int vx1, int vy0, int vy1,
                                   int nzc, double* val) {
    const long long pc = static_cast<long long>(nx) * ny;
    const int bx = vx1 - vx0, by = vy1 - vy0;
    const long long n = static_cast<long long>(bx) * by * nzc;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int x = vx0 + int(c % bx);
        const int y = vy0 + int((c / bx) % by);
        const int p = 4 + int(c / (static_cast<long long>(bx) * by));
        const double* ux = U;
        const double* uy = U + pc;
        const double* uz = U + 2 * pc;
        const double duz_dy = fd8_along(uz, nx, ny, pc, x, y, p, 1);
        const double duy_dz = fd8_along(uy, nx, ny, pc, x, y, p, 2);
        const double dux_dz = fd8_along(ux, nx, ny, pc, x, y, p, 2);
        const double duz_dx = fd8_along(uz, nx, ny, pc, x, y, p, 0);
        const double duy_dx = fd8_along(uy, nx, ny, pc, x, y, p, 0);
        const double dux_dy = fd8_along(ux, nx, ny, pc, x, y, p, 1);
        const double wx = duz_dy - duy_dz;
        const double wy = dux_dz - duz_dx;
        const double wz = duy_dx - dux_dy;
        val[c] = 0.5 * (wx * wx + wy * wy + wz * wz);
    }
}

// ---- device tree sums (diagnostics.cpp:10-18) --------------------------------

__device__ double tree_rec(const double* v, long long n) {
    if (n <= 8) {
        double s = 0.0;
        for (long long j = 0; j < n; ++j) s += v[j];
        return s;
    }
    const long long h = n / 2;
    const double a = tree_rec(v, h);
    return a + tree_rec(v + h, n - h);
}

// Small parts (len <= kSmall, or raw values with len 0), one thread each.
__global__ void k_tree_small(const double* v, const long long* lo_len, int n, double* out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const long long lo = lo_len[2 * t], len = lo_len[2 * t + 1];
    out[t] = len == 0 ? v[lo] : tree_rec(v + lo, len);
}

// The 2^D depth-D nodes of a large part, one thread each: descend by the bits
// of t (most significant first: left = 0), then sum the node sequentially-tree.
__global__ void k_tree_leaves(const double* v, long long len, int D, double* out) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (1ll << D)) return;
    long long l = 0, m = len;
    for (int d = D - 1; d >= 0; --d) {
        const long long h = m / 2;
        if ((t >> d) & 1) {
            l += h;
            m -= h;
        } else {
            m = h;
        }
    }
    out[t] = tree_rec(v + l, m);
}

__global__ void k_tree_pairs(const double* in, double* out, long long m) {
    const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (j < m) out[j] = in[2 * j] + in[2 * j + 1];
}

int grid_of(long long n) {
    long long b = (n + 255) / 256;
    return int(std::min<long long>(std::max<long long>(b, 1), 148LL * 32));
}

constexpr int64_t kSmall = 2048;

// Reduce the parts (global indices) of the chunk whose values start at global
// index `base` in `v` (device). Results land in parts[k].value.
void reduce_chunk(const double* v, int64_t base, dlb_tree_part* parts, std::size_t n, char* scratch,
                  std::size_t scratch_bytes, cudaStream_t st) {
    if (n == 0) return;
    std::vector<long long> small;
    std::vector<std::size_t> small_idx, large_idx;
    for (std::size_t k = 0; k < n; ++k) {
        if (parts[k].len <= kSmall) {
            small.push_back(parts[k].lo - base);
            small.push_back(parts[k].len);
            small_idx.push_back(k);
        } else {
            large_idx.push_back(k);
        }
    }
    // scratch: [results n doubles][small lo/len][level ping-pong]
    double* d_res = reinterpret_cast<double*>(scratch);
    long long* d_ll = reinterpret_cast<long long*>(scratch + n * 8);
    char* rest = scratch + n * 8 + small.size() * 8;
    rest = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(rest) + 255) & ~uintptr_t(255));
    const std::size_t rest_bytes = scratch_bytes - std::size_t(rest - scratch);
    if (!small.empty()) {
        cuda_check(cudaMemcpyAsync(d_ll, small.data(), small.size() * 8, cudaMemcpyHostToDevice, st), "h2d");
        const int m = int(small_idx.size());
        // results of the small parts first, in small order
        k_tree_small<<<(m + 127) / 128, 128, 0, st>>>(v, d_ll, m, d_res);
        cuda_check(cudaGetLastError(), "k_tree_small");
    }
    for (std::size_t j = 0; j < large_idx.size(); ++j) {
        const dlb_tree_part& p = parts[large_idx[j]];
        int D = 0;
        while (((p.len + (1ll << D) - 1) >> D) > 512) ++D;  // depth-D nodes hold <= 512 values
        const long long m = 1ll << D;
        if (std::size_t(m) * 16 > rest_bytes) throw DeviceError("diagnostics scratch too small");
        double* a = reinterpret_cast<double*>(rest);
        double* b = a + m;
        k_tree_leaves<<<int((m + 127) / 128), 128, 0, st>>>(v + (p.lo - base), p.len, D, a);
        cuda_check(cudaGetLastError(), "k_tree_leaves");
        for (long long w = m / 2; w >= 1; w /= 2) {
            double* dst = w == 1 ? d_res + small_idx.size() + j : b;
            k_tree_pairs<<<int((w + 255) / 256), 256, 0, st>>>(a, dst, w);
            cuda_check(cudaGetLastError(), "k_tree_pairs");
            std::swap(a, b);
        }
        if (m == 1) cuda_check(cudaMemcpyAsync(d_res + small_idx.size() + j, a, 8, cudaMemcpyDeviceToDevice, st), "d2d");
    }
    std::vector<double> res(n);
    cuda_check(cudaMemcpyAsync(res.data(), d_res, n * 8, cudaMemcpyDeviceToHost, st), "d2h");
    cuda_check(cudaStreamSynchronize(st), "tree reduce");
    for (std::size_t j = 0; j < small_idx.size(); ++j) parts[small_idx[j]].value = res[j];
    for (std::size_t j = 0; j < large_idx.size(); ++j) parts[large_idx[j]].value = res[small_idx.size() + j];
}

bool masked(int q) {
    return q == DLB_Q_PRESSURE_FLUID || q == DLB_Q_UX_FLUID || q == DLB_Q_RHO_FLUID;
}
bool windowed(int q) { return masked(q) || q == DLB_Q_UX_ALL; }

}  // namespace

void* Lattice::diag_scratch(std::size_t min_bytes) {
    if (diag_bytes_ >= min_bytes) return diag_buf_;
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    cudaFree(diag_buf_);
    diag_buf_ = nullptr;
    diag_bytes_ = 0;
    std::size_t free_b = 0, total_b = 0;
    cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    std::size_t want = std::max<std::size_t>(min_bytes, std::size_t(1) << 30);  // 1 GiB when it fits
    if (const char* e = std::getenv("DLB_DIAG_SCRATCH_BYTES"))  // tests: force many chunks
        want = std::max<std::size_t>(min_bytes, std::strtoull(e, nullptr, 10));
    const std::size_t reserve = std::size_t(256) << 20;
    if (free_b > reserve && want > free_b - reserve) want = std::max(min_bytes, free_b - reserve);
    cuda_check(cudaMalloc(&diag_buf_, want), "cudaMalloc(diagnostics scratch)");
    diag_bytes_ = want;
    return diag_buf_;
}

void* Lattice::diag_slots() {
    std::vector<DiagSlot> ds(std::max<std::size_t>(chains_.size(), 1));
    for (std::size_t s = 0; s < chains_.size(); ++s) {
        const LinkType t = chains_[s].links.back().type;
        ds[s].kind = t == LinkType::MovingBounceBack ? KIND_MBB
                   : (t == LinkType::BGK || t == LinkType::TRT || t == LinkType::RR) ? KIND_COLLIDE
                                                                                      : KIND_BB;
        ds[s].fluid = !(t == LinkType::BounceBack || t == LinkType::NoDynamics || t == LinkType::MovingBounceBack);
        for (int a = 0; a < 3; ++a) {
            const double w = chains_[s].params.wall_velocity[a];
            ds[s].uw[a] = d_.precision_bits == 64 ? w : double(float(w));  // T-cast, as the recipe holds it
        }
    }
    // the slot table lives at the head of the staging buffer
    cuda_check(cudaMemcpyAsync(staging_, ds.data(), ds.size() * sizeof(DiagSlot), cudaMemcpyHostToDevice, stream_),
               "h2d");
    return staging_;
}

namespace {
struct Box {
    int x0, x1, y0, y1;
    long long z0, z1;  // global
};
Box valid_box(const dlb_lattice_desc& d, const dlb_reduce_args& a) {
    const long long dims[3] = {d.dims[0], d.dims[1], d.global_nz};
    for (int ax = 0; ax < 3; ++ax)
        if (!a.periodic[ax] && dims[ax] < 9)
            throw std::invalid_argument("vorticity_fd8: non-periodic extent below the 9-point stencil width");
    Box b;
    b.x0 = a.periodic[0] ? 0 : 4;
    b.x1 = a.periodic[0] ? d.dims[0] : d.dims[0] - 4;
    b.y0 = a.periodic[1] ? 0 : 4;
    b.y1 = a.periodic[1] ? d.dims[1] : d.dims[1] - 4;
    b.z0 = a.periodic[2] ? 0 : 4;
    b.z1 = a.periodic[2] ? d.global_nz : d.global_nz - 4;
    return b;
}
void check_args(const dlb_lattice_desc& d, const dlb_reduce_args& a) {
    if (a.quantity < DLB_Q_KINETIC || a.quantity > DLB_Q_RHO_FLUID)
        throw std::invalid_argument("reduce: unknown quantity " + std::to_string(a.quantity));
    if (windowed(a.quantity) && (a.x_begin < 0 || a.x_end > d.dims[0] || a.x_begin > a.x_end))
        throw std::invalid_argument("reduce: x window outside the lattice");
}
}  // namespace

int64_t Lattice::reduce_count(const dlb_reduce_args& a) const {
    check_args(d_, a);
    const int64_t nx = d_.dims[0], ny = d_.dims[1], nz = d_.dims[2];
    if (a.quantity == DLB_Q_ENSTROPHY) {
        const Box b = valid_box(d_, a);
        const long long z0 = std::max<long long>(b.z0, d_.z_origin), z1 = std::min<long long>(b.z1, d_.z_origin + nz);
        return z1 > z0 ? int64_t(b.x1 - b.x0) * (b.y1 - b.y0) * (z1 - z0) : 0;
    }
    if (a.quantity == DLB_Q_UX_ALL) return (a.x_end - a.x_begin) * ny * nz;
    if (!masked(a.quantity)) return nx * ny * nz;
    // fluid cells in the window: from the slot array (host snapshot of the registry)
    std::vector<uint8_t> fluid(std::max<std::size_t>(chains_.size(), 1), 0);
    for (std::size_t s = 0; s < chains_.size(); ++s) {
        const LinkType t = chains_[s].links.back().type;
        fluid[s] = !(t == LinkType::BounceBack || t == LinkType::NoDynamics || t == LinkType::MovingBounceBack);
    }
    if (!d_slot_) return uniform_slot_ >= 0 && fluid[std::size_t(uniform_slot_)] ? (a.x_end - a.x_begin) * ny * nz : 0;
    std::vector<uint8_t> sl(std::size_t(nx * ny * nz));
    cuda_check(cudaMemcpy(sl.data(), d_slot_, sl.size(), cudaMemcpyDeviceToHost), "d2h slots");
    int64_t cnt = 0;
    for (int64_t r = 0; r < ny * nz; ++r)
        for (int64_t x = a.x_begin; x < a.x_end; ++x) cnt += fluid[sl[std::size_t(r * nx + x)]];
    return cnt;
}

void Lattice::reduce_parts(const dlb_reduce_args& a, int64_t n_total, int64_t seg_begin,
                           std::vector<dlb_tree_part>& out) {
    finalize_walls();
    DeviceGuard dg(device_);
    check_args(d_, a);
    if (!slots_set_) throw std::invalid_argument("diagnostics: dynamics slots not set");
    if (a.quantity == DLB_Q_DU_NUM && !d_uprev_)
        throw std::invalid_argument("diagnostics: DU_NUM needs a velocity snapshot (dlb_lattice_snapshot_velocity)");
    if (n_total < 0 || seg_begin < 0) throw std::invalid_argument("reduce: negative sizes");
    if (d_.precision_bits == 64) diag_impl<double>(a, n_total, seg_begin, out);
    else diag_impl<float>(a, n_total, seg_begin, out);
}

template <typename T>
void Lattice::diag_impl(const dlb_reduce_args& a, int64_t n_total, int64_t seg_begin,
                        std::vector<dlb_tree_part>& out) {
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    const int nx = d_.dims[0], ny = d_.dims[1], nz = d_.dims[2];
    const long long pc = static_cast<long long>(nx) * ny;
    const int mode = !aa() ? 0 : (aa_odd_layout_ ? 2 : 1);
    const T* o = static_cast<const T*>(origin(cur_));
    const DiagSlot* ds = static_cast<const DiagSlot*>(diag_slots());
    const int q = a.quantity;
    const bool ens = q == DLB_Q_ENSTROPHY;
    const int xb = windowed(q) ? int(a.x_begin) : 0, xe = windowed(q) ? int(a.x_end) : nx;
    const long long row = static_cast<long long>(xe - xb) * ny;  // values per plane (before compaction)

    // per-plane scratch: values (8) [+ flags (1) + compacted (8)] or U (24) + values (8)
    const std::size_t per_plane = ens ? std::size_t(pc) * 32 : std::size_t(row) * (masked(q) ? 17 : 8);
    const std::size_t fixed = (ens ? std::size_t(pc) * 24 * 8 : 0) + (std::size_t(64) << 20);
    char* buf = static_cast<char*>(diag_scratch(fixed + per_plane * 2));
    const int zc = int(std::max<long long>(1, std::min<long long>(nz, (diag_bytes_ - fixed) / per_plane)));

    long long vz0 = 0, vz1 = nz;  // local planes whose values enter the sequence
    Box box{};
    if (ens) {
        box = valid_box(d_, a);
        vz0 = std::max<long long>(box.z0 - d_.z_origin, 0);
        vz1 = std::min<long long>(box.z1 - d_.z_origin, nz);
    }
    int64_t cursor = seg_begin;
    auto align = [](char* p) { return reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255)); };
    for (long long za = vz0; za < vz1; za += zc) {
        const int nzc = int(std::min<long long>(zc, vz1 - za));
        char* p = buf;
        double* val = nullptr;
        long long cnt = 0;
        if (ens) {
            // velocity window: local planes [za - 4, za + nzc + 4)
            double* U = reinterpret_cast<double*>(p);
            const int W = nzc + 8;
            p = align(p + std::size_t(W) * pc * 24);
            val = reinterpret_cast<double*>(p);
            p = align(p + std::size_t(box.x1 - box.x0) * (box.y1 - box.y0) * nzc * 8);
            int w = 0;
            while (w < W) {
                const long long lz = za - 4 + w;
                if (lz >= 0 && lz < nz) {  // run of resident planes
                    const int run = int(std::min<long long>(W - w, nz - lz));
                    velocity_planes_impl<T>(int(lz), run, U + std::size_t(w) * pc * 3);
                    w += run;
                    continue;
                }
                if (!split()) {  // whole z extent here: periodic image
                    const long long sz = ((lz % nz) + nz) % nz;
                    velocity_planes_impl<T>(int(sz), 1, U + std::size_t(w) * pc * 3);
                } else {
                    const double* h = lz < 0 ? a.halo_below : a.halo_above;
                    const long long hp = lz < 0 ? lz + 4 : lz - nz;
                    const long long gz = d_.z_origin + lz;
                    const bool needed = a.periodic[2] || (gz >= 0 && gz < d_.global_nz);
                    if (h) {
                        cuda_check(cudaMemcpyAsync(U + std::size_t(w) * pc * 3, h + std::size_t(hp) * pc * 3, pc * 24,
                                                   cudaMemcpyHostToDevice, stream_), "h2d halo");
                    } else if (needed) {
                        throw std::invalid_argument("enstrophy: velocity halo planes required on a split slab");
                    } else {
                        cuda_check(cudaMemsetAsync(U + std::size_t(w) * pc * 3, 0, pc * 24, stream_), "memset");
                    }
                }
                ++w;
            }
            cnt = static_cast<long long>(box.x1 - box.x0) * (box.y1 - box.y0) * nzc;
            k_enstrophy_values<<<grid_of(cnt), 256, 0, stream_>>>(U, nx, ny, box.x0, box.x1, box.y0, box.y1, nzc, val);
            cuda_check(cudaGetLastError(), "k_enstrophy_values");
        } else if (q == DLB_Q_KINETIC && kinetic_fused_current()) {
            // the collide-stream kernel already wrote these values (KM_KE variant)
            val = d_ke_ + za * pc;
            cnt = row * nzc;
        } else {
            const long long n = row * nzc;
            val = reinterpret_cast<double*>(p);
            p = align(p + n * 8);
            uint8_t* flag = nullptr;
            double* comp = nullptr;
            if (masked(q)) {
                flag = reinterpret_cast<uint8_t*>(p);
                p = align(p + n);
                comp = reinterpret_cast<double*>(p);
                p = align(p + n * 8);
            }
            if (d_.q == 19)
                k_cell_values<T, 19><<<grid_of(n), 256, 0, stream_>>>(o, geo_, mode, d_slot_, uniform_slot_, ds, q,
                                                                      int(za), nzc, xb, xe, d_uprev_, pc * nz, val, flag);
            else
                k_cell_values<T, 27><<<grid_of(n), 256, 0, stream_>>>(o, geo_, mode, d_slot_, uniform_slot_, ds, q,
                                                                      int(za), nzc, xb, xe, d_uprev_, pc * nz, val, flag);
            cuda_check(cudaGetLastError(), "k_cell_values");
            cnt = n;
            if (masked(q)) {  // order-preserving compaction of the fluid cells
                long long* d_num = reinterpret_cast<long long*>(p);
                p = align(p + 8);
                std::size_t tb = 0;
                cuda_check(cub::DeviceSelect::Flagged(nullptr, tb, val, flag, comp, d_num, n, stream_), "cub size");
                if (std::size_t(p - buf) + tb + (std::size_t(32) << 20) > diag_bytes_)
                    throw DeviceError("diagnostics scratch too small for the compaction");
                cuda_check(cub::DeviceSelect::Flagged(p, tb, val, flag, comp, d_num, n, stream_), "cub select");
                cuda_check(cudaMemcpyAsync(&cnt, d_num, 8, cudaMemcpyDeviceToHost, stream_), "d2h");
                cuda_check(cudaStreamSynchronize(stream_), "select");
                p = align(p + tb);
                val = comp;
            }
        }
        std::vector<dlb_tree_part> parts;
        tree_plan(0, n_total, cursor, cursor + cnt, parts);
        if (!parts.empty()) {
            reduce_chunk(val, cursor, parts.data(), parts.size(), p, diag_bytes_ - std::size_t(p - buf), stream_);
            out.insert(out.end(), parts.begin(), parts.end());
        }
        cursor += cnt;
    }
    if (cursor > n_total) throw std::invalid_argument("reduce: segment exceeds the global sequence");
}

template <typename T>
void Lattice::velocity_planes_impl(int z0, int np, double* dev_out) {
    const int mode = !aa() ? 0 : (aa_odd_layout_ ? 2 : 1);
    const T* o = static_cast<const T*>(origin(cur_));
    const DiagSlot* ds = static_cast<const DiagSlot*>(staging_);  // diag_slots() uploaded it
    const long long n = static_cast<long long>(d_.dims[0]) * d_.dims[1] * np;
    if (d_.q == 19) k_u_planes<T, 19><<<grid_of(n), 256, 0, stream_>>>(o, geo_, mode, d_slot_, uniform_slot_, ds, z0, np, dev_out);
    else k_u_planes<T, 27><<<grid_of(n), 256, 0, stream_>>>(o, geo_, mode, d_slot_, uniform_slot_, ds, z0, np, dev_out);
    cuda_check(cudaGetLastError(), "k_u_planes");
}

void Lattice::velocity_planes(int z0, int np, double* out) {
    finalize_walls();
    DeviceGuard dg(device_);
    if (!slots_set_) throw std::invalid_argument("diagnostics: dynamics slots not set");
    if (z0 < 0 || np < 0 || z0 + np > d_.dims[2]) throw std::invalid_argument("velocity_planes: planes outside the slab");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    diag_slots();
    const std::size_t pb = std::size_t(d_.dims[0]) * d_.dims[1] * 24;
    char* buf = static_cast<char*>(diag_scratch(pb + (std::size_t(64) << 20)));
    const int chunk = int(std::max<std::size_t>(1, diag_bytes_ / pb));
    for (int z = z0; z < z0 + np; z += chunk) {
        const int m = std::min(chunk, z0 + np - z);
        if (d_.precision_bits == 64) velocity_planes_impl<double>(z, m, reinterpret_cast<double*>(buf));
        else velocity_planes_impl<float>(z, m, reinterpret_cast<double*>(buf));
        cuda_check(cudaMemcpyAsync(out + std::size_t(z - z0) * pb / 8, buf, pb * m, cudaMemcpyDeviceToHost, stream_), "d2h");
        cuda_check(cudaStreamSynchronize(stream_), "velocity_planes");
    }
}

void Lattice::snapshot_velocity() {
    finalize_walls();
    DeviceGuard dg(device_);
    if (!slots_set_) throw std::invalid_argument("diagnostics: dynamics slots not set");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    const long long pc = static_cast<long long>(d_.dims[0]) * d_.dims[1];
    const long long n = pc * d_.dims[2];
    if (!d_uprev_) {
        cuda_check(cudaMalloc(&d_uprev_, std::size_t(n) * 24), "cudaMalloc(velocity snapshot)");
        device_bytes_ += n * 24;
    }
    diag_slots();
    // planes one by one into [ux | uy | uz] x cells via the plane layout
    const std::size_t pb = std::size_t(pc) * 24;
    char* buf = static_cast<char*>(diag_scratch(pb + (std::size_t(64) << 20)));
    const int chunk = int(std::max<std::size_t>(1, diag_bytes_ / pb));
    for (int z = 0; z < d_.dims[2]; z += chunk) {
        const int m = std::min(chunk, int(d_.dims[2]) - z);
        if (d_.precision_bits == 64) velocity_planes_impl<double>(z, m, reinterpret_cast<double*>(buf));
        else velocity_planes_impl<float>(z, m, reinterpret_cast<double*>(buf));
        for (int c = 0; c < 3; ++c)
            cuda_check(cudaMemcpy2DAsync(d_uprev_ + c * n + z * pc, pc * 8, buf + c * pc * 8, pb, pc * 8, m,
                                         cudaMemcpyDeviceToDevice, stream_), "snapshot copy");
    }
    cuda_check(cudaStreamSynchronize(stream_), "snapshot");
}

}  // namespace dlb
