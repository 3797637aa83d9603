// Compacted storage for the porous masked sweep (k_cmp, collide_stream.cu).
//
// The reference steps every cell of the porous block (step_range over the
// whole AcceleratedBlock, proj/src/accelerated_lattice.cpp:126-153), NoDynamics
// solids included; the masked sweep skips the x-aligned segments of G cells
// (one 32-B sector of every direction array) that hold only NoDynamics cells
// (cases.cpp:239-249 makes every solid next to a fluid cell BounceBack, so no
// collision cell ever pulls from a skipped cell; check_skip_precondition).
// In the dense layout the listed segments are scattered sectors; here they are
// gathered, together with every segment they pull from ("frozen" sources:
// skipped segments and envelope segments, whose values never change), into
// compact arrays in row-major segment order over the envelope-inclusive
// segment grid. Row-major order keeps x-neighbours adjacent, so a pull shifted
// by +-1 cell reads the previous / next compact segment; the rows above and
// below come from an 8-entry table per listed segment.
//
// Life cycle: built with the slots (set_slots); gathered from the dense
// current buffer before the first compact step after any state write
// (prepare_compact, outside graph capture); the dense layout is brought up to
// date by scattering the listed segments (finalize_walls) before every read of
// the state. Single slabs with a non-periodic x axis (the porous case's inlet /
// outlet axis); opt-in with DLB_POROUS_COMPACT=1.
//
// Measured (profiles/r02b_summary.md): DRAM reads of these sparse sweeps follow
// whole 128-B lines -- at c4 (680 x 600^2, 31.8 M listed segments) a
// line-granular model of the pulls predicts 30.5 GB per step for the dense
// layout (k_seg; ncu 30.9 GB) and 28.8 + 1.3 GB (tables) for the compact one
// (ncu 30.2 GB), against 21.5 GB at sector granularity: the sphere pack's runs
// of listed segments (4.7 segments on average) are too short for any row
// ordering to fill the lines. k_cmp runs 9.65 vs 9.80 ms per step.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "lattice.hpp"

namespace dlb {
namespace {

// dense (current buffer) -> both compact buffers, every compact segment; lanes
// outside the dense row's x range [-1, nx] hold 0 (never read)
template <typename T>
__global__ void k_cmp_gather(T* c0, T* c1, long long cstride, const T* d0, long long dstride, const long long* off,
                             const int* x0, long long ncomp, int gshift, int q, int nx) {
    const long long n = ncomp << gshift;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const long long k = t >> gshift;
        const int lane = int(t & ((1 << gshift) - 1));
        const int x = x0[k] + lane;
        const bool in = x >= -1 && x <= nx;
        const long long at = off[k] + lane;
        for (int i = 0; i < q; ++i) {
            const T v = in ? d0[i * dstride + at] : T(0);
            c0[i * cstride + t] = v;
            c1[i * cstride + t] = v;
        }
    }
}

// current compact buffer -> current dense buffer, the listed segments' interior cells
template <typename T>
__global__ void k_cmp_scatter(T* d0, long long dstride, const T* c0, long long cstride, const unsigned* seg,
                              const long long* off, const int* x0, long long nlist, int gshift, int q, int nx) {
    const long long n = nlist << gshift;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const long long li = t >> gshift;
        const int lane = int(t & ((1 << gshift) - 1));
        const unsigned e = seg[li];
        const long long k = e & 0x03ffffffu;
        if (lane >= int(e >> 26)) continue;
        const int x = x0[k] + lane;
        if (x < 0 || x >= nx) continue;
        const long long src = (k << gshift) + lane;
        const long long at = off[k] + lane;
        for (int i = 0; i < q; ++i) d0[i * dstride + at] = c0[i * cstride + src];
    }
}

int grid_of(long long n) { return int(std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 16))); }

}  // namespace

void Lattice::free_compact() {
    for (void*& b : cbuf_) {
        cudaFree(b);
        b = nullptr;
    }
    cudaFree(d_cseg_);
    cudaFree(d_crows_);
    cudaFree(d_coff_);
    cudaFree(d_cx0_);
    cudaFree(d_cslot_);
    cudaFree(d_cfix_);
    d_cseg_ = d_crows_ = d_cfix_ = nullptr;
    d_coff_ = nullptr;
    d_cx0_ = nullptr;
    d_cslot_ = nullptr;
    device_bytes_ -= cmp_bytes_;
    cmp_bytes_ = 0;
    ncomp_ = ncl_ = ncfix_ = 0;
    cstride_ = 0;
    cmp_valid_ = cmp_dirty_ = false;
}

void Lattice::build_compact(const std::vector<uint8_t>& u8, const std::vector<uint8_t>& nodyn) {
    free_compact();
    const char* env = std::getenv("DLB_POROUS_COMPACT");  // opt-in (measured: +1.6 % on c4 for 60 GB)
    if (!(env && env[0] == '1')) return;
    const char* fs = std::getenv("DLB_FLUID_SEGMENTS");  // the opt-in fluid-segment sweep keeps the dense layout
    if (fs && fs[0] == '1') return;
    if (geo_.per_x || split() || aa() || untagged_ || xrec_ || u8.empty()) return;
    const int G = skip_group_;
    int gshift = 0;
    while ((1 << gshift) < G) ++gshift;
    const int nx = geo_.nx, ny = geo_.ny, nz = geo_.nz, q = d_.q;
    const long long nsx = (nx + G - 1) / G;
    const long long EX = nsx + 2, EY = ny + 2, EZ = nz + 2;
    const long long ne = EX * EY * EZ;
    if (ne >= (1LL << 26)) return;  // compact indices carry 26 bits
    const bool py = geo_.per_y, pz = geo_.per_z;
    auto eid = [&](long long z, long long y, long long s) { return ((z + 1) * EY + (y + 1)) * EX + (s + 1); };
    auto wrap = [](int v, int n, bool per) { return per ? (v < 0 ? v + n : (v >= n ? v - n : v)) : v; };

    // listed interior segments
    std::vector<uint8_t> listed(std::size_t(ne), 0), inset(std::size_t(ne), 0);
    const int nw = std::max(1, std::min<int>(nz + 2, int(std::thread::hardware_concurrency())));
    auto par = [&](int lo, int hi, auto&& fn) {
        std::vector<std::thread> th;
        for (int w = 0; w < nw; ++w)
            th.emplace_back([&, w] {
                for (int z = lo + (hi - lo) * w / nw; z < lo + (hi - lo) * (w + 1) / nw; ++z) fn(z);
            });
        for (auto& t : th) t.join();
    };
    par(0, nz, [&](int z) {
        for (int y = 0; y < ny; ++y) {
            const uint8_t* row = u8.data() + (long long)(z * ny + y) * nx;
            for (long long s = 0; s < nsx; ++s) {
                bool any = false;
                for (long long x = s * G; x < std::min<long long>(nx, (s + 1) * G) && !any; ++x) any = !nodyn[row[x]];
                listed[std::size_t(eid(z, y, s))] = any;
            }
        }
    });
    // source rows: dest row (y, z) pulls direction i from row (y - cy, z - cz);
    // need[r] = some direction uses row offset r, with an x-shift of +1 (the
    // segment to the left, nm) or -1 (to the right, np)
    bool need[3][3] = {}, nm[3][3] = {}, np[3][3] = {};
    for (int i = 0; i < q; ++i) {
        const int* c = q == 19 ? Lat<19>::c[i] : Lat<27>::c[i];
        const int dy = -c[1] + 1, dz = -c[2] + 1;
        need[dy][dz] = true;
        if (c[0] > 0) nm[dy][dz] = true;
        if (c[0] < 0) np[dy][dz] = true;
    }
    // the set: listed segments and every segment a listed one pulls from
    // (formulated per target row, so threads never write the same row)
    par(-1, nz + 1, [&](int Z) {
        if ((Z < 0 || Z >= nz) && pz) return;  // periodic: envelope planes are never sources
        for (int Y = -1; Y <= ny; ++Y) {
            if ((Y < 0 || Y >= ny) && py) continue;
            for (int dz = -1; dz <= 1; ++dz)
                for (int dy = -1; dy <= 1; ++dy) {
                    if (!need[dy + 1][dz + 1]) continue;
                    // dest rows whose row offset (dy, dz) lands on (Y, Z)
                    const int z = wrap(Z - dz, nz, pz), y = wrap(Y - dy, ny, py);
                    if (z < 0 || z >= nz || y < 0 || y >= ny) continue;
                    const uint8_t* L = listed.data() + eid(z, y, -1);  // L[s + 1]
                    uint8_t* S = inset.data() + eid(Z, Y, -1);
                    for (long long s = -1; s <= nsx; ++s) {
                        bool v = s >= 0 && s < nsx && L[s + 1];
                        if (!v && nm[dy + 1][dz + 1] && s + 1 < nsx) v = L[s + 2];  // dest s+1 reads its left neighbour s
                        if (!v && np[dy + 1][dz + 1] && s - 1 >= 0) v = L[s];      // dest s-1 reads its right neighbour s
                        if (v) S[s + 1] = 1;
                    }
                }
        }
    });
    for (long long e = 0; e < ne; ++e) inset[std::size_t(e)] |= listed[std::size_t(e)];
    // compact index of every set member, row-major
    std::vector<uint32_t> cidx(std::size_t(ne), 0);
    long long ncomp = 0;
    for (long long e = 0; e < ne; ++e)
        if (inset[std::size_t(e)]) cidx[std::size_t(e)] = uint32_t(ncomp++);
    std::vector<long long> off(static_cast<std::size_t>(ncomp));
    std::vector<int> x0(static_cast<std::size_t>(ncomp));
    std::vector<uint8_t> slotc(std::size_t(ncomp) << gshift, 0);
    for (long long Z = -1; Z <= nz; ++Z)
        for (long long Y = -1; Y <= ny; ++Y)
            for (long long s = -1; s <= nsx; ++s) {
                const long long e = eid(Z, Y, s);
                if (!inset[std::size_t(e)]) continue;
                const uint32_t k = cidx[std::size_t(e)];
                off[k] = Z * geo_.plane + Y * geo_.pitch + s * G;
                x0[k] = int(s * G);
                if (Z >= 0 && Z < nz && Y >= 0 && Y < ny && s >= 0 && s < nsx)
                    for (int l = 0; l < G && s * G + l < nx; ++l)
                        slotc[(std::size_t(k) << gshift) + l] = u8[std::size_t((Z * ny + Y) * nx + s * G + l)];
            }
    // listed segments in row-major order: compact index, valid lanes, row table
    std::vector<uint32_t> seg, rows;
    std::vector<uint32_t> fix;
    std::vector<char> reg(chains_.size(), 0);
    for (std::size_t sl = 0; sl < chains_.size(); ++sl)
        for (const ChainLink& l : chains_[sl].links)
            if (l.type == LinkType::RegularizedVelocity || l.type == LinkType::RegularizedPressure) reg[sl] = 1;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (long long s = 0; s < nsx; ++s) {
                const long long e = eid(z, y, s);
                if (!listed[std::size_t(e)]) continue;
                const int valid = int(std::min<long long>(G, nx - s * G));
                const uint32_t li = uint32_t(seg.size());
                seg.push_back(cidx[std::size_t(e)] | (uint32_t(valid) << 26));
                for (int l = 0; l < valid; ++l)
                    if (reg[u8[std::size_t((long long)(z * ny + y) * nx + s * G + l)]])
                        fix.push_back((li << gshift) | uint32_t(l));
            }
    const long long nl = (long long)seg.size();
    if (nl == 0 || (nl << gshift) >= (1LL << 32)) return;
    rows.assign(std::size_t(8 * nl), 0);
    {
        long long li = 0;
        for (int z = 0; z < nz; ++z)
            for (int y = 0; y < ny; ++y)
                for (long long s = 0; s < nsx; ++s) {
                    if (!listed[std::size_t(eid(z, y, s))]) continue;
                    for (int dz = -1; dz <= 1; ++dz)
                        for (int dy = -1; dy <= 1; ++dy) {
                            if (dy == 0 && dz == 0) continue;
                            uint32_t v = 0;
                            if (need[dy + 1][dz + 1]) {
                                const long long e = eid(wrap(z + dz, nz, pz), wrap(y + dy, ny, py), s);
                                if (!inset[std::size_t(e)]) throw std::logic_error("compact porous set incomplete");
                                v = cidx[std::size_t(e)];
                            }
                            rows[std::size_t(cmp_row(dy, dz) * nl + li)] = v;
                        }
                    ++li;
                }
    }
    // device copies
    const int es = d_.precision_bits / 8;
    cstride_ = ((ncomp << gshift) + 31) / 32 * 32 + 32;  // + one segment of slack past the last x-neighbour
    const std::size_t pop_bytes = std::size_t(q) * std::size_t(cstride_) * std::size_t(es);
    auto up = [&](void** dst, const void* src, std::size_t bytes, const char* what) {
        cuda_check(cudaMalloc(dst, std::max<std::size_t>(bytes, 4)), what);
        if (bytes) cuda_check(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice), what);
        cmp_bytes_ += int64_t(bytes);
    };
    for (void*& b : cbuf_) {
        // the compact arrays sit beside the dense layout: without room for
        // them the masked sweep stays on the dense layout (k_seg)
        if (cudaMalloc(&b, pop_bytes) != cudaSuccess) {
            cudaGetLastError();
            free_compact();
            return;
        }
        cmp_bytes_ += int64_t(pop_bytes);
    }
    up(reinterpret_cast<void**>(&d_cseg_), seg.data(), seg.size() * 4, "compact segments");
    up(reinterpret_cast<void**>(&d_crows_), rows.data(), rows.size() * 4, "compact rows");
    up(reinterpret_cast<void**>(&d_coff_), off.data(), off.size() * 8, "compact offsets");
    up(reinterpret_cast<void**>(&d_cx0_), x0.data(), x0.size() * 4, "compact x");
    up(reinterpret_cast<void**>(&d_cslot_), slotc.data(), slotc.size(), "compact slots");
    up(reinterpret_cast<void**>(&d_cfix_), fix.data(), fix.size() * 4, "compact fix-ups");
    device_bytes_ += cmp_bytes_;
    ncomp_ = ncomp;
    ncl_ = nl;
    ncfix_ = (long long)fix.size();
    cgshift_ = gshift;
    cmp_valid_ = cmp_dirty_ = false;
}

void Lattice::prepare_compact() {
    if (!kernel_cmp_ || cmp_valid_) return;
    DeviceGuard dg(device_);
    const int es = d_.precision_bits / 8;
    const long long n = ncomp_ << cgshift_;
    const int c = cur_;
    if (es == 8)
        k_cmp_gather<double><<<grid_of(n), 256, 0, stream_>>>(
            static_cast<double*>(cbuf_[c]), static_cast<double*>(cbuf_[1 - c]), cstride_,
            static_cast<const double*>(origin(c)), geo_.dstride, d_coff_, d_cx0_, ncomp_, cgshift_, d_.q, geo_.nx);
    else
        k_cmp_gather<float><<<grid_of(n), 256, 0, stream_>>>(
            static_cast<float*>(cbuf_[c]), static_cast<float*>(cbuf_[1 - c]), cstride_,
            static_cast<const float*>(origin(c)), geo_.dstride, d_coff_, d_cx0_, ncomp_, cgshift_, d_.q, geo_.nx);
    cuda_check(cudaGetLastError(), "k_cmp_gather");
    cmp_valid_ = true;
    cmp_dirty_ = false;
}

void Lattice::scatter_compact() {
    if (!cmp_dirty_) return;
    DeviceGuard dg(device_);
    const long long n = ncl_ << cgshift_;
    const int c = cur_;
    if (d_.precision_bits == 64)
        k_cmp_scatter<double><<<grid_of(n), 256, 0, stream_>>>(
            static_cast<double*>(origin(c)), geo_.dstride, static_cast<const double*>(cbuf_[c]), cstride_, d_cseg_,
            d_coff_, d_cx0_, ncl_, cgshift_, d_.q, geo_.nx);
    else
        k_cmp_scatter<float><<<grid_of(n), 256, 0, stream_>>>(
            static_cast<float*>(origin(c)), geo_.dstride, static_cast<const float*>(cbuf_[c]), cstride_, d_cseg_,
            d_coff_, d_cx0_, ncl_, cgshift_, d_.q, geo_.nx);
    cuda_check(cudaGetLastError(), "k_cmp_scatter");
    cmp_dirty_ = false;
}

}  // namespace dlb
