// Canonical-state access shared by the runtime (lattice.cu) and the
// diagnostics (diag.cu): where f_i(x, y, z) of the reference's canonical
// post-collision state lives in each storage layout.
#pragma once

#include "kernels.cuh"
#include "lbm_cell.cuh"

namespace dlb {
namespace {

// Position of canonical f_i(x, y, z) in the AA array after an odd step /
// at upload: A[i][x + c_i] (wrapped on periodic axes, envelope otherwise).
__device__ __forceinline__ long long shifted(const Geo& g, int x, int y, int z, int cx, int cy,
                                             int cz) {
    int X = x + cx, Y = y + cy, Z = z + cz;
    if (g.per_x) X = X < 0 ? X + g.nx : (X >= g.nx ? X - g.nx : X);
    if (g.per_y) Y = Y < 0 ? Y + g.ny : (Y >= g.ny ? Y - g.ny : Y);
    if (g.per_z) Z = Z < 0 ? Z + g.nz : (Z >= g.nz ? Z - g.nz : Z);
    return static_cast<long long>(Z) * g.plane + static_cast<long long>(Y) * g.pitch + X;
}

// Canonical f_i(x, y, z) of the current state for any layout
// (aa_mode: 0 two-population, 1 AA even layout, 2 AA odd layout).
template <typename T, int Q, int i>
__device__ __forceinline__ T canon_load(const T* origin0, const Geo& g, int x, int y, int z, int aa_mode) {
    using L = Lat<Q>;
    constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
    if (aa_mode == 2) return origin0[i * g.dstride + shifted(g, x, y, z, cx, cy, cz)];
    const long long at = static_cast<long long>(z) * g.plane + static_cast<long long>(y) * g.pitch + x;
    return origin0[(aa_mode == 1 ? opp_of(i) : i) * g.dstride + at];
}

struct MacroSlot {
    int kind;
    double uw[3];
};

}  // namespace
}  // namespace dlb
