// Benchmark cases (see cases.hpp for the reference line map).
#include "cases.hpp"

#include <cmath>
#include <fstream>
#include <set>
#include <stdexcept>

namespace dlb {

namespace {
constexpr double kCs = 0.57735026918962576451;  // 1/sqrt(3), cases.cpp:12
constexpr double kPi = 3.14159265358979323846;

// D3Q19 velocities (descriptor.hpp:13-33) for the solid-neighbour test.
constexpr int kC19[19][3] = {{0, 0, 0},   {-1, 0, 0}, {1, 0, 0},  {0, -1, 0}, {0, 1, 0},
                             {0, 0, -1},  {0, 0, 1},  {-1, -1, 0}, {1, 1, 0}, {-1, 1, 0},
                             {1, -1, 0},  {-1, 0, -1}, {1, 0, 1},  {-1, 0, 1}, {1, 0, -1},
                             {0, -1, -1}, {0, 1, 1},  {0, -1, 1}, {0, 1, -1}};

// chain.cpp:236-245: a chain keeps only the collision parameters its base consumes.
ChainParams collision_params_for(LinkType base, const CollisionParams& p) {
    ChainParams c;
    c.omega = p.omega;
    if (base == LinkType::TRT) {
        c.lambda = p.lambda;
        c.omega_minus = derive_omega_minus(p.omega, p.lambda);
    } else if (base == LinkType::RR) {
        c.omega_bulk_ho = p.omega_bulk_ho;
    }
    return c;
}

CollisionParams case_params(const CaseConfig& cfg) {
    CollisionParams p;
    p.omega = cfg.omega();
    p.lambda = cfg.lambda;
    p.omega_bulk_ho = cfg.omega_bulk_ho;
    return p;
}
}  // namespace

double CaseConfig::lattice_velocity() const { return kCs * Ma; }

double CaseConfig::char_length() const {
    // TGV: cell centres map to [0, 2 pi), the length is the inverse wavenumber
    return kind == CaseKind::Tgv ? double(L) / (2.0 * kPi) : double(L);
}

double CaseConfig::viscosity() const {
    if (kind == CaseKind::Porous) return (tau - 0.5) / 3.0;
    return lattice_velocity() * char_length() / Re;
}

double CaseConfig::omega() const {
    if (kind == CaseKind::Porous) return 1.0 / tau;
    return 1.0 / (3.0 * viscosity() + 0.5);  // omega_from_viscosity
}

double CaseConfig::t_c() const { return char_length() / lattice_velocity(); }

void CaseConfig::validate() const {
    if (kind == CaseKind::Tgv && L < 8) throw std::invalid_argument("tgv requires L >= 8");
    if (kind == CaseKind::Cavity && L < 16) throw std::invalid_argument("cavity requires L >= 16");
    if (Ma <= 0.0 || Ma >= 0.5) throw std::invalid_argument("Mach number must lie in (0, 0.5)");
    const double om = omega();
    if (!(om > 0.0 && om < 2.0))
        throw std::invalid_argument("relaxation rate " + std::to_string(om) + " outside the stable range (0, 2)");
    if (kind == CaseKind::Porous && geometry.empty())
        throw std::invalid_argument("porous case requires a geometry");
}

double VoxelGeometry::porosity() const {
    int64_t fluid = 0;
    for (uint8_t s : solid) fluid += s == 0;
    return double(fluid) / double(solid.size());
}

VoxelGeometry load_voxels(const std::string& path, std::array<int64_t, 3> dims, double threshold,
                          double dx_meters) {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw std::runtime_error("cannot open voxel file \"" + path + "\"");
    const int64_t expected = dims[0] * dims[1] * dims[2];
    const int64_t size = int64_t(in.tellg());
    if (size != expected)
        throw std::runtime_error("voxel file \"" + path + "\" has " + std::to_string(size) + " bytes, expected " +
                                 std::to_string(expected));
    in.seekg(0);
    std::vector<uint8_t> raw(static_cast<std::size_t>(expected));
    in.read(reinterpret_cast<char*>(raw.data()), expected);
    VoxelGeometry g;
    g.dims = dims;
    g.dx_meters = dx_meters;
    g.solid.resize(raw.size());
    for (std::size_t k = 0; k < raw.size(); ++k) g.solid[k] = double(raw[k]) > threshold * 255.0 ? 1 : 0;
    const double phi = g.porosity();
    if (phi <= 0.0 || phi >= 1.0) throw std::runtime_error("degenerate medium: porosity " + std::to_string(phi));
    return g;
}

VoxelGeometry make_plate_geometry(int64_t length, int64_t width, int64_t layers) {
    VoxelGeometry g;
    g.dims = {length, width, layers + 2};
    g.solid.assign(std::size_t(length * width * (layers + 2)), 0);
    const int64_t plane = length * width;
    for (int64_t k = 0; k < plane; ++k) {
        g.solid[std::size_t(k)] = 1;                         // z = 0
        g.solid[std::size_t((layers + 1) * plane + k)] = 1;  // z = H + 1
    }
    return g;
}

DynamicsChain make_collision_chain(LinkType base, const CollisionParams& p, std::optional<double> smagorinsky_c) {
    DynamicsChain ch;
    ch.params = collision_params_for(base, p);
    if (smagorinsky_c) {
        ch.params.smagorinsky_c = *smagorinsky_c;
        ch.links.push_back({LinkType::Smagorinsky});
    }
    ch.links.push_back({base});
    validate_chain(ch.links);
    return ch;
}

DynamicsChain make_bounce_back() { return DynamicsChain{{{LinkType::BounceBack}}, {}}; }

DynamicsChain make_no_dynamics() { return DynamicsChain{{{LinkType::NoDynamics}}, {}}; }

DynamicsChain make_moving_bounce_back(std::array<double, 3> u_wall) {
    DynamicsChain ch{{{LinkType::MovingBounceBack}}, {}};
    ch.params.wall_velocity = u_wall;
    return ch;
}

DynamicsChain make_regularized_velocity(int axis, int orient, std::array<double, 3> u, LinkType base,
                                        const CollisionParams& p) {
    DynamicsChain ch;
    ch.links = {{LinkType::RegularizedVelocity, axis, orient}, {base}};
    ch.params = collision_params_for(base, p);
    ch.params.wall_velocity = u;
    validate_chain(ch.links);
    return ch;
}

DynamicsChain make_regularized_pressure(int axis, int orient, double rho, LinkType base,
                                        const CollisionParams& p) {
    DynamicsChain ch;
    ch.links = {{LinkType::RegularizedPressure, axis, orient}, {base}};
    ch.params = collision_params_for(base, p);
    ch.params.target_rho = rho;
    validate_chain(ch.links);
    return ch;
}

CaseSetup init_tgv(const CaseConfig& cfg) {
    cfg.validate();
    CaseSetup s;
    s.dims = {cfg.L, cfg.L, cfg.L};
    s.periodic = {true, true, true};
    s.t_c = cfg.t_c();
    s.chains.push_back(make_collision_chain(cfg.collision, case_params(cfg), cfg.smagorinsky_c));
    s.state = InitState::Tgv;
    s.u_inf = cfg.lattice_velocity();
    return s;
}

CaseSetup init_cavity(const CaseConfig& cfg) {
    cfg.validate();
    CaseSetup s;
    const int64_t L = cfg.L;
    s.dims = {L, L, L};
    s.t_c = cfg.t_c();
    s.chains = {make_collision_chain(cfg.collision, case_params(cfg), cfg.smagorinsky_c), make_bounce_back(),
                make_moving_bounce_back({cfg.lattice_velocity(), 0.0, 0.0})};
    s.chain_index.assign(std::size_t(L * L * L), 0);
    for (int64_t z = 0; z < L; ++z)
        for (int64_t y = 0; y < L; ++y)
            for (int64_t x = 0; x < L; ++x) {
                uint8_t c = 0;
                if (z == L - 1) c = 2;  // lid
                else if (x == 0 || x == L - 1 || y == 0 || y == L - 1 || z == 0) c = 1;
                s.chain_index[std::size_t((z * L + y) * L + x)] = c;
            }
    return s;
}

CaseSetup init_porous(const CaseConfig& cfg, const VoxelGeometry& geo) {
    cfg.validate();
    const auto gd = geo.dims;
    CaseSetup s;
    const int64_t nx = gd[0] + cfg.upstream + cfg.downstream, ny = gd[1], nz = gd[2];
    s.dims = {nx, ny, nz};
    s.periodic = {false, true, true};
    s.t_c = cfg.t_c();
    s.sample_begin = cfg.upstream;
    s.sample_end = cfg.upstream + gd[0];
    const CollisionParams p = case_params(cfg);
    const double u_in = cfg.lattice_velocity();
    DynamicsChain inlet, outlet;
    if (cfg.drive == DriveKind::Velocity) {
        inlet = make_regularized_velocity(0, 1, {u_in, 0.0, 0.0}, cfg.collision, p);
        outlet = make_regularized_velocity(0, -1, {u_in, 0.0, 0.0}, cfg.collision, p);
    } else {
        inlet = make_regularized_pressure(0, 1, 1.0 + cfg.delta_rho, cfg.collision, p);
        outlet = make_regularized_pressure(0, -1, 1.0 - cfg.delta_rho, cfg.collision, p);
    }
    // the porous bulk never carries the LES link (cases.cpp:215)
    s.chains = {make_collision_chain(cfg.collision, p), make_bounce_back(), make_no_dynamics(), inlet, outlet};
    const bool plates = cfg.geometry == "plates";
    const int64_t up = cfg.upstream;
    std::vector<uint8_t> solid(std::size_t(nx * ny * nz), 0);
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) {
                bool sol;
                if (plates) sol = z == 0 || z == nz - 1;  // plates span the buffers too
                else sol = x >= up && x < up + gd[0] && geo.solid[std::size_t((z * ny + y) * gd[0] + (x - up))];
                solid[std::size_t((z * ny + y) * nx + x)] = sol;
            }
    s.chain_index.assign(solid.size(), 0);
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) {
                const int64_t g = (z * ny + y) * nx + x;
                uint8_t c;
                if (solid[std::size_t(g)]) {
                    // solids with no fluid neighbour need no collision work (cases.cpp:239-249)
                    c = 2;
                    for (int i = 1; i < 19; ++i) {
                        const int64_t sx = x + kC19[i][0];
                        const int64_t sy = (y + kC19[i][1] + ny) % ny;
                        const int64_t sz = (z + kC19[i][2] + nz) % nz;
                        if (sx < 0 || sx >= nx) continue;
                        if (!solid[std::size_t((sz * ny + sy) * nx + sx)]) {
                            c = 1;
                            break;
                        }
                    }
                } else if (x == 0) {
                    c = 3;
                } else if (x == nx - 1) {
                    c = 4;
                } else {
                    c = 0;
                }
                s.chain_index[std::size_t(g)] = c;
            }
    return s;
}

CaseSetup make_setup(const CaseConfig& cfg) {
    switch (cfg.kind) {
        case CaseKind::Tgv: return init_tgv(cfg);
        case CaseKind::Cavity: return init_cavity(cfg);
        case CaseKind::Porous: {
            if (cfg.geometry == "plates")
                return init_porous(cfg, make_plate_geometry(cfg.L, std::max<int64_t>(4, cfg.L / 5), cfg.plate_layers));
            if (cfg.voxel_dims[0] < 1) throw std::invalid_argument("voxel geometry needs case.voxel_dims");
            return init_porous(cfg, load_voxels(cfg.geometry, cfg.voxel_dims, cfg.voxel_threshold, cfg.voxel_dx));
        }
    }
    throw std::logic_error("unreachable");
}

std::vector<std::string> setup_models(const CaseSetup& setup) {
    std::vector<uint8_t> used(setup.chains.size(), 0);
    if (setup.chain_index.empty()) used[0] = 1;
    for (uint8_t c : setup.chain_index) used[c] = 1;
    std::set<std::string> names;
    for (std::size_t k = 0; k < used.size(); ++k)
        if (used[k]) names.insert(chain_string(setup.chains[k].links));
    return {names.begin(), names.end()};
}

}  // namespace dlb
