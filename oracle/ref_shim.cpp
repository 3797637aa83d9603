// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference solver ("dolb",
// /root/reference/proj), compiled from the reference sources where they lie
// by oracle/Makefile into oracle/_ref/libdolb_refshim.so. It uses only the
// reference's public C++ API:
//   - case generators   init_tgv / init_cavity / init_porous  (proj/src/cases.cpp:127-260)
//   - build_run<T>      (proj/src/cases.cpp:279-297) + MultiBlockRun<T>::advance
//                       (proj/src/multiblock.cpp:376-419) + gather_populations (:421-441)
//   - compile_chain<T> / ChainRecipe<T>::apply (proj/include/dolb/chain.hpp:104-187)
//   - equilibrium2/4 (proj/include/dolb/descriptor.hpp:79-121)
//   - perf::measure_mlups (proj/src/perfmodel.cpp:94-121)
// Python tests and bench.py (--impl reference / cpu_baseline) call it via ctypes.
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "dolb/accelerated_lattice.hpp"
#include "dolb/cases.hpp"
#include "dolb/chain.hpp"
#include "dolb/descriptor.hpp"
#include "dolb/diagnostics.hpp"
#include "dolb/multiblock.hpp"
#include "dolb/perfmodel.hpp"

namespace {

thread_local std::string g_err;

// Flat case description (mirrors dolb::CaseConfig, proj/include/dolb/cases.hpp:22-54).
struct RefCase {
    int32_t kind;        // 0 tgv, 1 cavity, 2 porous
    int32_t collision;   // 0 BGK, 1 TRT, 2 RR
    int64_t L;
    double Re, Ma, lambda, omega_bulk_ho;
    double smagorinsky_c;  // NaN => no LES link
    int32_t drive;         // 0 velocity, 1 pressure
    int32_t pad0;
    double tau, delta_rho;
    int64_t upstream, downstream, plate_layers;
    int64_t voxel_dims[3];
    const char* geometry;  // "plates" or a raw voxel path
};

dolb::LinkType base_of(int c) {
    switch (c) {
        case 0: return dolb::LinkType::BGK;
        case 1: return dolb::LinkType::TRT;
        case 2: return dolb::LinkType::RR;
    }
    throw std::invalid_argument("collision must be 0 (BGK), 1 (TRT) or 2 (RR)");
}

dolb::CaseConfig make_config(const RefCase& rc) {
    dolb::CaseConfig cfg;
    cfg.kind = rc.kind == 0 ? dolb::CaseKind::Tgv
             : rc.kind == 1 ? dolb::CaseKind::Cavity
                            : dolb::CaseKind::Porous;
    cfg.L = rc.L;
    cfg.Re = rc.Re;
    cfg.Ma = rc.Ma;
    cfg.collision = base_of(rc.collision);
    if (!std::isnan(rc.smagorinsky_c)) cfg.smagorinsky_c = rc.smagorinsky_c;
    cfg.lambda = rc.lambda;
    cfg.omega_bulk_ho = rc.omega_bulk_ho;
    cfg.drive = rc.drive == 0 ? dolb::DriveKind::Velocity : dolb::DriveKind::Pressure;
    cfg.tau = rc.tau;
    cfg.delta_rho = rc.delta_rho;
    cfg.upstream = rc.upstream;
    cfg.downstream = rc.downstream;
    cfg.plate_layers = rc.plate_layers;
    cfg.geometry = rc.geometry ? rc.geometry : "";
    return cfg;
}

dolb::CaseSetup make_setup(const RefCase& rc) {
    dolb::CaseConfig cfg = make_config(rc);
    if (rc.kind == 0) return dolb::init_tgv(cfg);
    if (rc.kind == 1) return dolb::init_cavity(cfg);
    std::shared_ptr<const dolb::VoxelGeometry> geom;
    if (cfg.geometry == "plates") {
        geom = std::make_shared<dolb::VoxelGeometry>(
            dolb::make_plate_geometry(rc.L, rc.L, rc.plate_layers));
    } else {
        geom = std::make_shared<dolb::VoxelGeometry>(dolb::load_voxels(
            cfg.geometry, {rc.voxel_dims[0], rc.voxel_dims[1], rc.voxel_dims[2]}, 0.5, 1e-6));
    }
    return dolb::init_porous(cfg, geom);
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    } catch (...) {
        g_err = "unknown error";
        return 1;
    }
}

template <typename T>
void run_case(const RefCase& rc, const int grid[3], int workers, int64_t steps, double* out) {
    const dolb::CaseSetup setup = make_setup(rc);
    auto registry = std::make_shared<dolb::DynamicsRegistry>();
    auto run = dolb::build_run<T>(setup, {grid[0], grid[1], grid[2]}, workers, registry);
    run.advance(steps);
    const std::vector<double> pops = run.gather_populations();
    std::memcpy(out, pops.data(), pops.size() * sizeof(double));
}

// Streamed over the run's blocks (public MultiBlockRun::blocks() + the
// blocks' cell_index): no gather_populations copy, so full-size configs fit in
// host RAM. out_all: every interior cell; out_active (optional): cells whose
// chain is not NoDynamics (the masked porous sweep leaves those stale).
template <typename T>
void checksum_case(const RefCase& rc, const int grid[3], int workers, int64_t steps, uint64_t* out_all,
                   uint64_t* out_active) {
    const dolb::CaseSetup setup = make_setup(rc);
    auto registry = std::make_shared<dolb::DynamicsRegistry>();
    auto run = dolb::build_run<T>(setup, {grid[0], grid[1], grid[2]}, workers, registry);
    run.advance(steps);
    const auto& blocks = run.blocks();
    const int ntags = registry->num_tags();
    std::vector<char> nodyn(std::size_t(std::max(ntags, 1)), 0);
    for (int t = 0; t < ntags; ++t) nodyn[std::size_t(t)] = registry->chain_for(t) == "NoDynamics";
    std::vector<std::array<uint64_t, 38>> part(blocks.size());
    std::vector<std::thread> th;
    for (std::size_t b = 0; b < blocks.size(); ++b) {
        th.emplace_back([&, b] {
            const auto& blk = blocks[b];
            std::array<uint64_t, 38> acc{};
            const std::size_t vol = std::size_t(blk.vol());
            for (int64_t z = 1; z <= blk.interior[2]; ++z)
                for (int64_t y = 1; y <= blk.interior[1]; ++y)
                    for (int64_t x = 1; x <= blk.interior[0]; ++x) {
                        const int64_t at = blk.idx(x, y, z);
                        const uint64_t w = uint64_t(blk.cell_index[std::size_t(at)]) + 1u;
                        const int32_t tg = blk.tag[std::size_t(at)];
                        const bool active = !(tg >= 0 && tg < ntags && nodyn[std::size_t(tg)]);
                        for (int i = 0; i < 19; ++i) {
                            const double v = double(blk.f_in[std::size_t(i) * vol + std::size_t(at)]) + 0.0;
                            uint64_t bits;
                            std::memcpy(&bits, &v, 8);
                            acc[std::size_t(i)] += bits * w;
                            if (active) acc[std::size_t(19 + i)] += bits * w;
                        }
                    }
            part[b] = acc;
        });
    }
    for (auto& t : th) t.join();
    for (int i = 0; i < 19; ++i) {
        uint64_t a = 0, m = 0;
        for (const auto& p : part) {
            a += p[std::size_t(i)];
            m += p[std::size_t(19 + i)];
        }
        out_all[i] = a;
        if (out_active) out_active[i] = m;
    }
}

template <typename T>
void macro_case(const RefCase& rc, int64_t steps, double* rho, double* ux, double* uy, double* uz) {
    const dolb::CaseSetup setup = make_setup(rc);
    auto registry = std::make_shared<dolb::DynamicsRegistry>();
    auto run = dolb::build_run<T>(setup, {1, 1, 2}, 2, registry);
    run.advance(steps);
    std::vector<double> r, x, y, z;
    run.gather_macroscopic(r, x, y, z);
    std::memcpy(rho, r.data(), r.size() * 8);
    std::memcpy(ux, x.data(), x.size() * 8);
    std::memcpy(uy, y.data(), y.size() * 8);
    std::memcpy(uz, z.data(), z.size() * 8);
}

template <typename T>
void dump_case(const RefCase& rc, int64_t steps, const char* path) {
    const dolb::CaseSetup setup = make_setup(rc);
    auto registry = std::make_shared<dolb::DynamicsRegistry>();
    auto run = dolb::build_run<T>(setup, {1, 1, 2}, 2, registry);
    run.advance(steps);
    dolb::write_field_dump(path, run.gather_block());
}


// The runner's sampling step (Driver::sample / porous_extras,
// proj/src/runner.cpp:346-448) on the reference's own gathered fields after
// steps_a and steps_a + steps_b steps: out = {k, eps, nn, dd, k_perm, ubar, dp,
// ux_in, ux_out} (nn / dd between the two samples; porous extras zero for
// other cases).
template <typename T>
void sample_case(const RefCase& rc, int64_t steps_a, int64_t steps_b, double* out) {
    const dolb::CaseConfig cfg = make_config(rc);
    const dolb::CaseSetup setup = make_setup(rc);
    auto registry = std::make_shared<dolb::DynamicsRegistry>();
    auto run = dolb::build_run<T>(setup, {1, 1, 2}, 2, registry);
    run.advance(steps_a);
    std::vector<double> r0, x0, y0, z0;
    run.gather_macroscopic(r0, x0, y0, z0);
    run.advance(steps_b);
    std::vector<double> rho, ux, uy, uz;
    run.gather_macroscopic(rho, ux, uy, uz);
    dolb::diag::VectorField u;
    u.dims = setup.dims;
    u.x = ux;
    u.y = uy;
    u.z = uz;
    out[0] = dolb::diag::kinetic_energy(u);
    out[1] = dolb::diag::enstrophy(dolb::diag::vorticity_fd8(u, setup.periodic));
    std::vector<double> num(ux.size()), den(ux.size());
    for (std::size_t i = 0; i < ux.size(); ++i) {
        const double dx = ux[i] - x0[i];
        const double dy = uy[i] - y0[i];
        const double dz = uz[i] - z0[i];
        num[i] = dx * dx + dy * dy + dz * dz;
        den[i] = ux[i] * ux[i] + uy[i] * uy[i] + uz[i] * uz[i];
    }
    out[2] = dolb::diag::tree_sum(num);
    out[3] = dolb::diag::tree_sum(den);
    for (int k = 4; k < 9; ++k) out[k] = 0.0;
    if (rc.kind != 2) return;
    const auto& dims = setup.dims;
    std::vector<uint8_t> fluid(std::size_t(dims[0] * dims[1] * dims[2]));
    for (int64_t z = 0; z < dims[2]; ++z)
        for (int64_t y = 0; y < dims[1]; ++y)
            for (int64_t x = 0; x < dims[0]; ++x) {
                const dolb::LinkType t = setup.chain_of(x, y, z)->links.back().type;
                const bool solid = t == dolb::LinkType::BounceBack || t == dolb::LinkType::NoDynamics ||
                                   t == dolb::LinkType::MovingBounceBack;
                fluid[std::size_t((z * dims[1] + y) * dims[0] + x)] = solid ? 0 : 1;
            }
    const bool aperture = cfg.geometry == "plates";
    auto plane_mean = [&](int64_t x, const std::vector<double>& f, double scale) {
        std::vector<double> vals;
        for (int64_t z = 0; z < dims[2]; ++z)
            for (int64_t y = 0; y < dims[1]; ++y) {
                const int64_t g = (z * dims[1] + y) * dims[0] + x;
                if (fluid[std::size_t(g)]) vals.push_back(scale == 0.0 ? f[std::size_t(g)] : scale * f[std::size_t(g)]);
            }
        return vals.empty() ? 0.0 : dolb::diag::tree_mean(vals);
    };
    std::vector<double> vals, density;
    for (int64_t z = 0; z < dims[2]; ++z)
        for (int64_t y = 0; y < dims[1]; ++y)
            for (int64_t x = setup.sample_begin; x < setup.sample_end; ++x) {
                const int64_t g = (z * dims[1] + y) * dims[0] + x;
                if (fluid[std::size_t(g)]) density.push_back(rho[std::size_t(g)]);
                if (aperture && !fluid[std::size_t(g)]) continue;
                vals.push_back(ux[std::size_t(g)]);
            }
    const int64_t x0p = setup.sample_begin, x1p = setup.sample_end - 1;
    const double ubar = dolb::diag::tree_mean(vals);
    const double rho_bar = density.empty() ? 1.0 : dolb::diag::tree_mean(density);
    const double dp = (plane_mean(x0p, rho, dolb::D3Q19::cs2) - plane_mean(x1p, rho, dolb::D3Q19::cs2)) / rho_bar;
    const double lx = double(x1p - x0p);
    const double nu = cfg.viscosity();
    out[4] = std::abs(dp) < 1e-300 ? 0.0 : dolb::diag::permeability(ubar, nu, lx, dp);
    out[5] = ubar;
    out[6] = dp;
    out[7] = plane_mean(1, ux, 0.0);
    out[8] = plane_mean(dims[0] - 2, ux, 0.0);
}

template <typename T>
void bench_case(const RefCase& rc, int workers, int64_t warmup, int64_t steps, int reps,
                double* rep_mlups, double* mean) {
    const dolb::CaseSetup setup = make_setup(rc);
    auto registry = std::make_shared<dolb::DynamicsRegistry>();
    // N workers and N z-blocks: the only way the reference uses N cores
    // (MultiBlockRun never passes nthreads > 1, proj/src/multiblock.cpp:367,397).
    auto run = dolb::build_run<T>(setup, {1, 1, workers}, workers, registry);
    const auto report = dolb::perf::measure_mlups(
        [&run](std::int64_t n) { run.advance(n); }, run.num_cells(), warmup, steps, reps);
    for (int r = 0; r < reps; ++r) rep_mlups[r] = report.repetition_mlups[std::size_t(r)];
    *mean = report.mlups;
}

template <typename T>
void apply_chain(const char* chain_str, const double* params, size_t nparams, double* f,
                 int64_t n) {
    dolb::DynamicsChain chain;
    chain.links = dolb::parse_chain_string(chain_str);
    chain.params = dolb::deserialize_params(chain.links, params, nparams);
    const dolb::ChainRecipe<T> recipe = dolb::compile_chain<T>(chain);
    for (int64_t c = 0; c < n; ++c) {
        dolb::Populations<T> p;
        for (int i = 0; i < 19; ++i) p[i] = T(f[c * 19 + i]);
        recipe.apply(p);
        for (int i = 0; i < 19; ++i) f[c * 19 + i] = double(p[i]);
    }
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* ref_last_error(void) { return g_err.c_str(); }

__attribute__((visibility("default"))) int ref_case_dims(const RefCase* rc, int64_t* dims) {
    return guarded([&] {
        const auto s = make_setup(*rc);
        for (int a = 0; a < 3; ++a) dims[a] = s.dims[a];
    });
}

// Per-cell registry tags (x fastest) plus the newline-joined sorted model list.
__attribute__((visibility("default"))) int ref_case_tags(const RefCase* rc, int32_t* tags,
                                                         char* models, size_t cap) {
    return guarded([&] {
        const auto s = make_setup(*rc);
        dolb::DynamicsRegistry reg;
        for (const auto& ch : s.chains) reg.register_chain(*ch);
        int64_t k = 0;
        for (int64_t z = 0; z < s.dims[2]; ++z)
            for (int64_t y = 0; y < s.dims[1]; ++y)
                for (int64_t x = 0; x < s.dims[0]; ++x, ++k)
                    tags[k] = reg.tag_for(dolb::chain_string(*s.chain_of(x, y, z)));
        std::string joined;
        for (const auto& m : reg.chain_strings()) joined += m + "\n";
        if (joined.size() + 1 > cap) throw std::invalid_argument("model buffer too small");
        std::memcpy(models, joined.c_str(), joined.size() + 1);
    });
}

// Runs `steps` steps of the reference accelerated path (MultiBlockRun<T>) and
// writes gather_populations() (19*N doubles, direction-major, x fastest).
__attribute__((visibility("default"))) int ref_case_run(const RefCase* rc, int precision_bits,
                                                        const int* grid, int workers,
                                                        int64_t steps, double* out) {
    return guarded([&] {
        if (precision_bits == 64) run_case<double>(*rc, grid, workers, steps, out);
        else if (precision_bits == 32) run_case<float>(*rc, grid, workers, steps, out);
        else throw std::invalid_argument("precision must be 32 or 64");
    });
}

// dlb_lattice_checksum of the reference's state after `steps` steps.
__attribute__((visibility("default"))) int ref_case_checksum(const RefCase* rc, int precision_bits,
                                                             const int* grid, int workers,
                                                             int64_t steps, uint64_t* out) {
    return guarded([&] {
        if (precision_bits == 64) checksum_case<double>(*rc, grid, workers, steps, out, nullptr);
        else checksum_case<float>(*rc, grid, workers, steps, out, nullptr);
    });
}

// The same, plus the checksum restricted to cells whose chain is not
// NoDynamics (compare with the masked porous sweep).
__attribute__((visibility("default"))) int ref_case_checksum_masked(const RefCase* rc, int precision_bits,
                                                                    const int* grid, int workers,
                                                                    int64_t steps, uint64_t* out_all,
                                                                    uint64_t* out_active) {
    return guarded([&] {
        if (precision_bits == 64) checksum_case<double>(*rc, grid, workers, steps, out_all, out_active);
        else checksum_case<float>(*rc, grid, workers, steps, out_all, out_active);
    });
}

__attribute__((visibility("default"))) int ref_case_macro(const RefCase* rc, int precision_bits,
                                                          int64_t steps, double* rho, double* ux,
                                                          double* uy, double* uz) {
    return guarded([&] {
        if (precision_bits == 64) macro_case<double>(*rc, steps, rho, ux, uy, uz);
        else macro_case<float>(*rc, steps, rho, ux, uy, uz);
    });
}

__attribute__((visibility("default"))) int ref_case_dump(const RefCase* rc, int precision_bits,
                                                         int64_t steps, const char* path) {
    return guarded([&] {
        if (precision_bits == 64) dump_case<double>(*rc, steps, path);
        else dump_case<float>(*rc, steps, path);
    });
}

__attribute__((visibility("default"))) int ref_case_sample(const RefCase* rc, int precision_bits,
                                                           int64_t steps_a, int64_t steps_b,
                                                           double* out) {
    return guarded([&] {
        if (precision_bits == 64) sample_case<double>(*rc, steps_a, steps_b, out);
        else sample_case<float>(*rc, steps_a, steps_b, out);
    });
}

__attribute__((visibility("default"))) int ref_tree_sum(const double* v, int64_t n, double* out) {
    return guarded([&] { *out = dolb::diag::tree_sum(std::span<const double>(v, std::size_t(n))); });
}

__attribute__((visibility("default"))) int ref_case_bench(const RefCase* rc, int precision_bits,
                                                          int workers, int64_t warmup,
                                                          int64_t steps, int reps,
                                                          double* rep_mlups, double* mean) {
    return guarded([&] {
        if (precision_bits == 64) bench_case<double>(*rc, workers, warmup, steps, reps, rep_mlups, mean);
        else bench_case<float>(*rc, workers, warmup, steps, reps, rep_mlups, mean);
    });
}

// ChainRecipe<T>::apply on n population sets (input/output as doubles, cast to T).
__attribute__((visibility("default"))) int ref_apply_chain(const char* chain_str,
                                                           const double* params, size_t nparams,
                                                           int precision_bits, double* f,
                                                           int64_t n) {
    return guarded([&] {
        if (precision_bits == 64) apply_chain<double>(chain_str, params, nparams, f, n);
        else apply_chain<float>(chain_str, params, nparams, f, n);
    });
}

__attribute__((visibility("default"))) int ref_equilibrium(int order, int precision_bits,
                                                           double rho, const double* u,
                                                           double* out) {
    return guarded([&] {
        auto go = [&](auto tag) {
            using T = decltype(tag);
            const std::array<T, 3> uu = {T(u[0]), T(u[1]), T(u[2])};
            const auto feq = order == 4 ? dolb::equilibrium4<T>(T(rho), uu)
                                        : dolb::equilibrium2<T>(T(rho), uu);
            for (int i = 0; i < 19; ++i) out[i] = double(feq[i]);
        };
        if (precision_bits == 64) go(double{});
        else go(float{});
    });
}

__attribute__((visibility("default"))) double ref_derive_omega_minus(double omega, double lambda) {
    return dolb::CollisionParams::derive_omega_minus(omega, lambda);
}

// Registry-level behaviour, for pinning the product's host-side mirror:
// chain string of a (chain string, params) after a parse/serialize round trip.
__attribute__((visibility("default"))) int ref_chain_roundtrip(const char* chain_str,
                                                               char* out, size_t cap) {
    return guarded([&] {
        dolb::DynamicsChain chain;
        chain.links = dolb::parse_chain_string(chain_str);
        dolb::validate_chain(chain);
        const std::string s = dolb::chain_string(chain);
        if (s.size() + 1 > cap) throw std::invalid_argument("buffer too small");
        std::memcpy(out, s.c_str(), s.size() + 1);
    });
}

}  // extern "C"
