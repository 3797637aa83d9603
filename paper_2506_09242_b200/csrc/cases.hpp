// Benchmark cases on the host side of the device runtime (C++ twin of the
// Python `cases` module). Same inputs, chain assignment and initial state as
// the reference's cases layer:
//   CaseConfig + convective scaling ... proj/include/dolb/cases.hpp:22-54, src/cases.cpp:16-68
//   load_voxels / make_plate_geometry . src/cases.cpp:86-125
//   init_tgv / init_cavity / init_porous src/cases.cpp:127-260
//   chain factories ................... src/chain.cpp:236-281
//   setup_models ...................... src/cases.cpp:299-311
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "chain.hpp"

namespace dlb {

enum class CaseKind { Tgv, Cavity, Porous };
enum class DriveKind { Velocity, Pressure };

struct CaseConfig {
    CaseKind kind = CaseKind::Tgv;
    int64_t L = 64;
    double Re = 1600.0;
    double Ma = 0.2;
    LinkType collision = LinkType::BGK;
    std::optional<double> smagorinsky_c;
    double lambda = 3.0 / 16.0;
    double omega_bulk_ho = 1.0;
    int precision_bits = 64;
    int q = 19;  // device-runtime extension (case.lattice = d3q27): the reference is D3Q19 only
    std::array<int, 3> block_grid = {1, 1, 1};
    int workers = 1;
    // porous
    DriveKind drive = DriveKind::Velocity;
    std::string geometry;
    int64_t plate_layers = 11;
    double tau = 1.0;
    double delta_rho = 2e-3;
    int64_t upstream = 40;
    int64_t downstream = 40;
    std::array<int64_t, 3> voxel_dims = {0, 0, 0};
    double voxel_dx = 0.0;
    double voxel_threshold = 0.5;

    double lattice_velocity() const;
    double char_length() const;
    double viscosity() const;
    double omega() const;
    double t_c() const;
    void validate() const;
};

// 1 = solid, x fastest (cases.hpp:57-66)
struct VoxelGeometry {
    std::array<int64_t, 3> dims = {0, 0, 0};
    std::vector<uint8_t> solid;
    double dx_meters = 0.0;
    double porosity() const;
};

VoxelGeometry load_voxels(const std::string& path, std::array<int64_t, 3> dims, double threshold,
                          double dx_meters);
VoxelGeometry make_plate_geometry(int64_t length, int64_t width, int64_t layers);

struct CollisionParams {
    double omega = 1.0;
    double lambda = 3.0 / 16.0;
    double omega_bulk_ho = 1.0;
};

DynamicsChain make_collision_chain(LinkType base, const CollisionParams& p,
                                   std::optional<double> smagorinsky_c = std::nullopt);
DynamicsChain make_bounce_back();
DynamicsChain make_no_dynamics();
DynamicsChain make_moving_bounce_back(std::array<double, 3> u_wall);
DynamicsChain make_regularized_velocity(int axis, int orient, std::array<double, 3> u, LinkType base,
                                        const CollisionParams& p);
DynamicsChain make_regularized_pressure(int axis, int orient, double rho, LinkType base,
                                        const CollisionParams& p);

// Initial state of a case: the TGV field (evaluated on the device from glibc
// sin/cos tables, bit-identical to cases.cpp:145-156) or rest (rho 1, u 0).
enum class InitState { Tgv, Rest };

struct CaseSetup {
    std::array<int64_t, 3> dims = {0, 0, 0};
    std::array<bool, 3> periodic = {false, false, false};
    std::vector<DynamicsChain> chains;
    std::vector<uint8_t> chain_index;  // per cell, x fastest; empty = chain 0 everywhere
    InitState state = InitState::Rest;
    double u_inf = 0.0;                // TGV amplitude
    double t_c = 1.0;
    int64_t sample_begin = 0, sample_end = 0;

    int chain_at(int64_t g) const { return chain_index.empty() ? 0 : chain_index[std::size_t(g)]; }
    int64_t cells() const { return dims[0] * dims[1] * dims[2]; }
};

CaseSetup init_tgv(const CaseConfig& cfg);
CaseSetup init_cavity(const CaseConfig& cfg);
CaseSetup init_porous(const CaseConfig& cfg, const VoxelGeometry& geometry);
// The runner's geometry choice (runner.cpp:276-287): "plates" or a voxel file.
CaseSetup make_setup(const CaseConfig& cfg);
// Chain strings the setup assigns to at least one cell, sorted.
std::vector<std::string> setup_models(const CaseSetup& setup);

}  // namespace dlb
