// Reference-side C++ call sites swapped onto the B200 path (include/dlb_dolb.hpp).
//
// Compiled against the UNMODIFIED reference headers and objects
// (/root/reference/proj, built by oracle/Makefile into oracle/_ref/obj) plus
// libdlb_b200.so; run by tests/test_cpp_dropin.py on the GPU. Each case is a
// port of a reference test with only the solver call replaced:
//   1. test_accelerated.cpp:131-168  golden TGV16 trajectory through a DOLB1 dump (<= 1e-12)
//   2. test_accelerated.cpp:171-186  hybrid: 50 reference steps + 50 accelerated == 100 reference
//   3. test_accelerated.cpp:223-244  a tag outside the dispatch set throws DispatchError before any write
//   4. acceptance.cpp:70-105         criterion 1: oracle equivalence, TGV32 Re 1600, 100 steps
//   5. acceptance.cpp:108-131        criterion 2: decomposition invariance, bit-identical every step
//   6. the device run against the reference's own MultiBlockRun on a bounded domain (cavity, walls + lid)
#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <string>

#include "dlb_dolb.hpp"
#include "dolb/cases.hpp"
#include "dolb/reference_lattice.hpp"

using namespace dolb;

namespace {

int g_failures = 0;

#define CHECK(cond)                                                                  \
    do {                                                                             \
        if (!(cond)) {                                                               \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
            ++g_failures;                                                            \
        }                                                                            \
    } while (0)

CaseSetup small_tgv(std::int64_t L) {
    CaseConfig config;
    config.kind = CaseKind::Tgv;
    config.L = L;
    config.Re = 8.0;
    config.Ma = 0.1;
    return init_tgv(config);
}

CaseConfig tgv_config(std::int64_t L, double Re, double Ma, LinkType coll) {
    CaseConfig c;
    c.kind = CaseKind::Tgv;
    c.L = L;
    c.Re = Re;
    c.Ma = Ma;
    c.collision = coll;
    return c;
}

double max_abs_diff(const ReferenceLattice& ref, const AcceleratedBlock<double>& block) {
    double worst = 0.0;
    const std::int64_t vol = block.vol();
    for (std::int64_t z = 0; z < block.interior[2]; ++z)
        for (std::int64_t y = 0; y < block.interior[1]; ++y)
            for (std::int64_t x = 0; x < block.interior[0]; ++x) {
                const auto& cell = ref.cell(x, y, z);
                const std::int64_t at = block.idx(x + 1, y + 1, z + 1);
                for (int i = 0; i < 19; ++i)
                    worst = std::max(worst, std::abs(cell.f[i] - block.f_in[std::size_t(i) * std::size_t(vol) +
                                                                             std::size_t(at)]));
            }
    return worst;
}

double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// 1. test_accelerated.cpp:131-168
void golden_dump() {
    const CaseSetup setup = small_tgv(16);
    ReferenceLattice ref = build_reference(setup);
    for (int t = 0; t < 10; ++t) ref.collide_and_stream();
    DynamicsRegistry golden_registry;
    const auto golden_block = mirror_to_accelerated<double>(ref, golden_registry);
    const std::string golden = (std::filesystem::temp_directory_path() / "dlb_dropin_golden_tgv16.dolb").string();
    write_field_dump(golden, golden_block);

    auto registry = std::make_shared<DynamicsRegistry>();
    auto run = dlb_dolb::build_device_run<double>(setup, {1, 1, 1}, 1, registry);  // was build_run<double>
    run.advance(10);
    const auto mono = run.gather_block();

    const FieldDump dump = read_field_dump(golden);
    CHECK((dump.dims == std::array<std::int64_t, 3>{16, 16, 16}));
    CHECK(dump.precision_bytes == 8);
    const std::int64_t vol = mono.vol();
    double worst = 0.0;
    std::int64_t cell = 0;
    for (std::int64_t z = 0; z < 16; ++z)
        for (std::int64_t y = 0; y < 16; ++y)
            for (std::int64_t x = 0; x < 16; ++x, ++cell) {
                const std::int64_t at = mono.idx(x + 1, y + 1, z + 1);
                for (int i = 0; i < 19; ++i)
                    worst = std::max(worst, std::abs(dump.value(i, cell) -
                                                     mono.f_in[std::size_t(i) * std::size_t(vol) + std::size_t(at)]));
            }
    CHECK(worst <= 1e-12);
    std::filesystem::remove(golden);
    std::printf("golden_dump: max |diff| = %.3g\n", worst);
}

// 2. test_accelerated.cpp:171-186
void hybrid() {
    const CaseSetup setup = small_tgv(12);
    ReferenceLattice pure = build_reference(setup);
    for (int t = 0; t < 100; ++t) pure.collide_and_stream();

    ReferenceLattice half = build_reference(setup);
    for (int t = 0; t < 50; ++t) half.collide_and_stream();
    DynamicsRegistry registry;
    auto block = mirror_to_accelerated<double>(half, registry);
    const auto recipes = compile_recipes<double>(registry);
    const DispatchSet all = DispatchSet::all_of(registry);
    for (int t = 0; t < 50; ++t) {
        refresh_envelope_periodic(block);                                    // the reference's own
        dlb_dolb::collide_and_stream(block, registry, recipes, all);         // was collide_and_stream
    }
    const double d = max_abs_diff(pure, block);
    CHECK(d <= 1e-12);
    std::printf("hybrid: max |diff| = %.3g\n", d);
}

// 3. test_accelerated.cpp:223-244
void dispatch_error_before_any_write() {
    ReferenceLattice ref({4, 4, 4}, {true, true, true});
    CollisionParams p;
    p.omega = 1.0;
    ref.set_chain({{0, 0, 0}, {4, 4, 4}}, make_collision_chain(LinkType::BGK, p));
    ref.set_chain({{1, 1, 1}, {2, 2, 2}}, make_bounce_back());
    DynamicsRegistry registry;
    auto block = mirror_to_accelerated<double>(ref, registry);
    const auto recipes = compile_recipes<double>(registry);
    const DispatchSet only_bgk = DispatchSet::from_strings(registry, {"COLL_BGK"});
    refresh_envelope_periodic(block);
    const auto before = block.f_in;
    bool thrown = false;
    try {
        dlb_dolb::collide_and_stream(block, registry, recipes, only_bgk);  // was collide_and_stream
    } catch (const DispatchError& e) {
        thrown = true;
        CHECK(e.chain_name() == "BounceBack");
        CHECK(std::string(e.what()).find("BounceBack") != std::string::npos);
    }
    CHECK(thrown);
    CHECK(block.f_in == before);  // eager scan fails before any write
    std::printf("dispatch_error: %s\n", thrown ? "DispatchError(BounceBack), block untouched" : "MISSING");
}

// 4. acceptance.cpp:70-105
void oracle_equivalence() {
    const double t0 = now();
    const CaseSetup setup = init_tgv(tgv_config(32, 1600.0, 0.2, LinkType::BGK));
    ReferenceLattice reference = build_reference(setup);
    auto registry = std::make_shared<DynamicsRegistry>();
    auto run = dlb_dolb::build_device_run<double>(setup, {1, 1, 1}, 1, registry);
    for (int step = 0; step < 100; ++step) reference.collide_and_stream();
    run.advance(100);
    const std::vector<double> acc = run.gather_populations();
    const std::int64_t n = run.num_cells();
    double worst = 0.0;
    for (std::int64_t z = 0; z < 32; ++z)
        for (std::int64_t y = 0; y < 32; ++y)
            for (std::int64_t x = 0; x < 32; ++x) {
                const auto& cell = reference.cell(x, y, z);
                const std::int64_t g = (z * 32 + y) * 32 + x;
                for (int i = 0; i < 19; ++i)
                    worst = std::max(worst, std::abs(cell.f[i] - acc[std::size_t(i) * std::size_t(n) + std::size_t(g)]));
            }
    const double elapsed = now() - t0;
    CHECK(worst <= 1e-12);
    CHECK(elapsed < 30.0);
    std::printf("criterion 1 (oracle equivalence): max-abs %.3g, %.2f s\n", worst, elapsed);
}

// 5. acceptance.cpp:108-131 (the device run decomposes along z: 4 z-slabs
// here; the reference's {2, 2, 1} grid is run beside it as a third witness)
void decomposition_invariance() {
    const double t0 = now();
    const CaseSetup setup = init_tgv(tgv_config(32, 1600.0, 0.2, LinkType::BGK));
    auto reg_mono = std::make_shared<DynamicsRegistry>();
    auto reg_part = std::make_shared<DynamicsRegistry>();
    auto reg_ref = std::make_shared<DynamicsRegistry>();
    auto mono = dlb_dolb::build_device_run<double>(setup, {1, 1, 1}, 1, reg_mono);
    auto part = dlb_dolb::build_device_run<double>(setup, {1, 1, 4}, 4, reg_part);
    auto ref = build_run<double>(setup, {2, 2, 1}, 4, reg_ref);
    bool identical = true;
    int step = 0;
    for (; step < 100 && identical; ++step) {
        mono.advance(1);
        part.advance(1);
        ref.advance(1);
        const auto a = mono.gather_populations();
        identical = a == part.gather_populations() && a == ref.gather_populations();
    }
    const double elapsed = now() - t0;
    CHECK(identical);
    CHECK(elapsed < 60.0);
    std::printf("criterion 2 (decomposition invariance): %s after %d steps, %.2f s\n",
                identical ? "bit-identical" : "MISMATCH", step, elapsed);
}

// 6. bounded domain: walls, moving lid (cases.cpp:160-189), fp32 and fp64
template <typename T>
void cavity_vs_multiblock() {
    CaseConfig c;
    c.kind = CaseKind::Cavity;
    c.L = 24;
    c.Re = 400.0;
    c.Ma = 0.1;
    c.collision = LinkType::TRT;
    const CaseSetup setup = init_cavity(c);
    auto reg_a = std::make_shared<DynamicsRegistry>();
    auto reg_b = std::make_shared<DynamicsRegistry>();
    auto dev = dlb_dolb::build_device_run<T>(setup, {1, 1, 3}, 3, reg_a);
    auto ref = build_run<T>(setup, {1, 1, 3}, 3, reg_b);
    dev.advance(60);
    ref.advance(60);
    const bool same = dev.gather_populations() == ref.gather_populations();
    std::vector<double> r1, u1, v1, w1, r2, u2, v2, w2;
    dev.gather_macroscopic(r1, u1, v1, w1);
    ref.gather_macroscopic(r2, u2, v2, w2);
    CHECK(same);
    CHECK(r1 == r2 && u1 == u2 && v1 == v2 && w1 == w2);
    std::printf("cavity24 TRT fp%d, 3 z-slabs vs MultiBlockRun: %s\n", int(8 * sizeof(T)),
                same ? "bit-identical" : "MISMATCH");
}

}  // namespace

int main() {
    golden_dump();
    hybrid();
    dispatch_error_before_any_write();
    oracle_equivalence();
    decomposition_invariance();
    cavity_vs_multiblock<double>();
    cavity_vs_multiblock<float>();
    if (g_failures) {
        std::fprintf(stderr, "%d check(s) failed\n", g_failures);
        return 1;
    }
    std::printf("all drop-in checks passed\n");
    return 0;
}
