// Benchmark runner on the device runtime (runner.hpp; reference semantics from
// proj/src/runner.cpp, proj/src/diagnostics.cpp:164-193, proj/src/perfmodel.cpp).
#include "runner.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <set>
#include <sstream>
#include <stdexcept>

#include "device_run.hpp"
#include "tree.hpp"

namespace dlb::run {

namespace {

std::string trim(const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r\n");
    if (b == std::string::npos) return "";
    const auto e = s.find_last_not_of(" \t\r\n");
    return s.substr(b, e - b + 1);
}

std::string g17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

std::vector<std::string> split(const std::string& s, char sep) {
    std::vector<std::string> out;
    std::istringstream in(s);
    std::string tok;
    while (std::getline(in, tok, sep)) {
        tok = trim(tok);
        if (!tok.empty()) out.push_back(tok);
    }
    return out;
}

double parse_double(const Config& c, const std::string& key, double fallback) {
    const auto v = c.get(key);
    if (!v) return fallback;
    try {
        std::size_t used = 0;
        const double d = std::stod(*v, &used);
        if (used != v->size()) throw std::invalid_argument("");
        return d;
    } catch (...) {
        throw std::invalid_argument("config key " + key + ": \"" + *v + "\" is not a number");
    }
}

int64_t parse_int(const Config& c, const std::string& key, int64_t fallback) {
    const auto v = c.get(key);
    if (!v) return fallback;
    try {
        std::size_t used = 0;
        const long long n = std::stoll(*v, &used);
        if (used != v->size()) throw std::invalid_argument("");
        return n;
    } catch (...) {
        throw std::invalid_argument("config key " + key + ": \"" + *v + "\" is not an integer");
    }
}

bool parse_bool(const Config& c, const std::string& key, bool fallback) {
    const auto v = c.get(key);
    if (!v) return fallback;
    if (*v == "true" || *v == "1" || *v == "yes") return true;
    if (*v == "false" || *v == "0" || *v == "no") return false;
    throw std::invalid_argument("config key " + key + ": \"" + *v + "\" is not a boolean");
}

CaseKind parse_case_kind(const std::string& n) {
    if (n == "tgv") return CaseKind::Tgv;
    if (n == "cavity") return CaseKind::Cavity;
    if (n == "porous") return CaseKind::Porous;
    throw std::invalid_argument("unknown case \"" + n + "\"; valid cases: tgv, cavity, porous");
}

LinkType parse_collision(const std::string& n) {
    if (n == "bgk") return LinkType::BGK;
    if (n == "trt") return LinkType::TRT;
    if (n == "rr") return LinkType::RR;
    throw std::invalid_argument("unknown collision model \"" + n + "\"; valid models: bgk, trt, rr");
}

int parse_precision(const std::string& n) {
    if (n == "f32") return 32;
    if (n == "f64") return 64;
    throw std::invalid_argument("unknown precision \"" + n + "\"; valid precisions: f32, f64");
}

// steps, "<N>tc" (convective units) or "steady" (runner.cpp:168-193)
void parse_tmax(const std::string& text, double t_c, RunPlan& plan) {
    if (text == "steady") {
        plan.until_steady = true;
        plan.tmax_steps = 0;
        return;
    }
    std::string num = text;
    bool in_tc = false;
    if (num.size() > 2) {
        std::string suf = num.substr(num.size() - 2);
        for (char& ch : suf) ch = char(std::tolower(static_cast<unsigned char>(ch)));
        if (suf == "tc") {
            in_tc = true;
            num = num.substr(0, num.size() - 2);
        }
    }
    try {
        std::size_t used = 0;
        const double v = std::stod(num, &used);
        if (used != num.size() || v < 0) throw std::invalid_argument("");
        plan.tmax_steps = in_tc ? std::llround(v * t_c) : std::llround(v);
    } catch (...) {
        throw std::invalid_argument("cannot parse time specification \"" + text +
                                    "\": use steps, \"<N>tc\" or \"steady\"");
    }
}

const char* kind_name(CaseKind k) {
    return k == CaseKind::Tgv ? "tgv" : (k == CaseKind::Cavity ? "cavity" : "porous");
}

const char* collision_name(LinkType t) {
    return t == LinkType::BGK ? "bgk" : (t == LinkType::TRT ? "trt" : "rr");
}

// diagnostics rows (diagnostics.cpp:164-193)
struct Row {
    int64_t step = 0;
    double t_c = 0, k = 0, eps = 0;
    std::vector<double> extras;
};

}  // namespace

// ---------------------------------------------------------------------------- Config
Config Config::from_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open config file \"" + path + "\"");
    std::stringstream b;
    b << in.rdbuf();
    return from_string(b.str());
}

Config Config::from_string(const std::string& text) {
    Config c;
    std::istringstream in(text);
    std::string line, section;
    while (std::getline(in, line)) {
        const auto hash = line.find('#');
        if (hash != std::string::npos) line.resize(hash);
        line = trim(line);
        if (line.empty()) continue;
        if (line.front() == '[' && line.back() == ']') {
            section = trim(line.substr(1, line.size() - 2));
            continue;
        }
        const auto eq = line.find('=');
        if (eq == std::string::npos) throw std::runtime_error("config line without '=': \"" + line + "\"");
        const std::string key = trim(line.substr(0, eq)), value = trim(line.substr(eq + 1));
        c.set(section.empty() ? key : section + "." + key, value);
    }
    return c;
}

std::optional<std::string> Config::get(const std::string& key) const {
    const auto it = values_.find(key);
    if (it == values_.end()) return std::nullopt;
    return it->second;
}

std::string Config::get_or(const std::string& key, const std::string& fallback) const {
    const auto v = get(key);
    return v ? *v : fallback;
}

std::string Config::render() const {
    std::map<std::string, std::vector<std::pair<std::string, std::string>>> sections;
    for (const auto& [key, value] : values_) {
        const auto dot = key.find('.');
        sections[dot == std::string::npos ? "" : key.substr(0, dot)].push_back(
            {dot == std::string::npos ? key : key.substr(dot + 1), value});
    }
    std::string out;
    for (const auto& [section, entries] : sections) {
        if (!section.empty()) out += "[" + section + "]\n";
        for (const auto& [name, value] : entries) out += name + " = " + value + "\n";
        out += "\n";
    }
    return out;
}

// ---------------------------------------------------------------------------- resolve
RunPlan resolve(const Config& config) {
    RunPlan plan;
    CaseConfig& cc = plan.case_config;
    cc.kind = parse_case_kind(config.get_or("case.kind", "tgv"));
    cc.L = parse_int(config, "case.L", 64);
    cc.Ma = parse_double(config, "case.Ma", cc.kind == CaseKind::Porous ? 0.01 : 0.2);
    cc.Re = parse_double(config, "case.Re", cc.kind == CaseKind::Cavity ? 1000.0 : 1600.0);
    cc.collision = parse_collision(config.get_or("case.collision", cc.kind == CaseKind::Porous ? "trt" : "bgk"));
    if (config.has("case.smagorinsky")) cc.smagorinsky_c = parse_double(config, "case.smagorinsky", 0.0);
    cc.lambda = parse_double(config, "case.lambda", 3.0 / 16.0);
    cc.omega_bulk_ho = parse_double(config, "case.omega_bulk_ho", 1.0);
    cc.precision_bits = parse_precision(config.get_or("case.precision", "f64"));
    {
        const std::string d = config.get_or("case.drive", "velocity");
        if (d == "velocity") cc.drive = DriveKind::Velocity;
        else if (d == "pressure") cc.drive = DriveKind::Pressure;
        else throw std::invalid_argument("unknown drive \"" + d + "\"; valid drives: velocity, pressure");
    }
    cc.geometry = config.get_or("case.geometry", "");
    cc.plate_layers = parse_int(config, "case.H", 11);
    {
        const std::string lat = config.get_or("case.lattice", "d3q19");
        if (lat == "d3q19") cc.q = 19;
        else if (lat == "d3q27") cc.q = 27;
        else throw std::invalid_argument("unknown lattice \"" + lat + "\"; valid lattices: d3q19, d3q27");
        if (cc.q == 27 && cc.kind == CaseKind::Porous)
            throw std::invalid_argument("case.lattice d3q27: porous media use the D3Q19 wall classification");
    }
    cc.tau = parse_double(config, "case.tau", 1.0);
    cc.delta_rho = parse_double(config, "case.delta_rho", 2e-3);
    cc.upstream = parse_int(config, "case.upstream", 40);
    cc.downstream = parse_int(config, "case.downstream", 40);
    if (config.has("case.voxel_dims")) {
        const auto p = split(*config.get("case.voxel_dims"), ',');
        if (p.size() != 3) throw std::invalid_argument("case.voxel_dims needs three comma-separated extents");
        for (int a = 0; a < 3; ++a) cc.voxel_dims[std::size_t(a)] = std::stoll(p[std::size_t(a)]);
    }
    cc.voxel_dx = parse_double(config, "case.voxel_dx", 0.0);
    cc.voxel_threshold = parse_double(config, "case.voxel_threshold", 0.5);
    if (config.has("run.blocks")) {
        const auto p = split(*config.get("run.blocks"), ',');
        if (p.size() != 3) throw std::invalid_argument("run.blocks needs three comma-separated counts");
        for (int a = 0; a < 3; ++a) cc.block_grid[std::size_t(a)] = int(std::stoll(p[std::size_t(a)]));
    }
    cc.workers = int(parse_int(config, "run.workers", 1));
    cc.validate();

    const std::string default_tmax =
        cc.kind == CaseKind::Porous ? "steady" : (cc.kind == CaseKind::Tgv ? "12tc" : "20tc");
    parse_tmax(config.get_or("run.tmax", default_tmax), cc.t_c(), plan);
    plan.steady_tol = parse_double(config, "run.steady_tol", 1e-8);
    plan.max_steps = parse_int(config, "run.max_steps", 200000);
    const int64_t default_every =
        cc.kind == CaseKind::Porous
            ? 200
            : std::max<int64_t>(1, std::llround(cc.t_c() / (cc.kind == CaseKind::Tgv ? 8.0 : 1.0)));
    plan.output_every = parse_int(config, "run.output_every", default_every);
    if (plan.output_every < 1) throw std::invalid_argument("run.output_every must be >= 1");
    plan.dump_every = parse_int(config, "run.dump_every", 0);
    plan.avg_from_tc = parse_double(config, "run.avg_from", 50.0);
    plan.out_dir = config.get_or("run.out", "out");
    if (config.has("run.perf_device")) plan.perf_device = *config.get("run.perf_device");
    if (config.has("run.device_catalog")) plan.device_catalog = *config.get("run.device_catalog");
    plan.reference_check = parse_bool(config, "run.reference_check", false);
    if (plan.reference_check)
        throw std::invalid_argument(
            "run.reference_check: the in-run CPU reference lattice is not part of the device runtime "
            "(parity is checked by the test suite against the reference solver)");
    if (config.has("dispatch.models")) plan.dispatch_models = split(*config.get("dispatch.models"), ',');
    // device-runtime keys
    if (config.has("run.devices")) {
        for (const std::string& d : split(*config.get("run.devices"), ',')) {
            try {
                plan.devices.push_back(int(std::stoi(d)));
            } catch (...) {
                throw std::invalid_argument("config key run.devices: \"" + d + "\" is not a device ordinal");
            }
        }
    }
    plan.layout_name = config.get_or("run.layout", "twopop");
    if (plan.layout_name == "twopop") plan.layout = DLB_LAYOUT_TWO_POP;
    else if (plan.layout_name == "aa") plan.layout = DLB_LAYOUT_AA;
    else throw std::invalid_argument("unknown layout \"" + plan.layout_name + "\"; valid layouts: twopop, aa");
    plan.porous_name = config.get_or("run.porous", "dense");
    if (plan.porous_name == "dense") plan.flags = 0;
    else if (plan.porous_name == "masked") plan.flags = DLB_FLAG_SKIP_NODYNAMICS;
    else if (plan.porous_name == "lists") plan.flags = DLB_FLAG_SPARSE_LISTS;
    else throw std::invalid_argument("unknown porous sweep \"" + plan.porous_name + "\"; valid sweeps: dense, masked, lists");
    {
        const std::string a = config.get_or("run.arith", "exact");
        if (a == "exact") plan.arith = DLB_ARITH_EXACT;
        else if (a == "fast") plan.arith = DLB_ARITH_FAST;
        else throw std::invalid_argument("unknown arithmetic mode \"" + a + "\"; valid modes: exact, fast");
    }
    return plan;
}

// ---------------------------------------------------------------------------- perf model
int64_t model_bytes_per_cell(int bits) {
    if (bits != 32 && bits != 64) throw std::invalid_argument("precision must be 32 or 64 bits");
    return 2 * 19 * (bits / 8) + 8 + 4;  // populations + cell_index + tag (perfmodel.cpp:47-56)
}

DeviceSpec lookup_device(const std::string& name, const char* catalog_path) {
    std::vector<DeviceSpec> catalog = {{"A100-SXM4-40GB", 1555e9, 40e9}};
    if (catalog_path) {
        std::ifstream in(catalog_path);
        if (!in) throw std::runtime_error("cannot open device catalog \"" + std::string(catalog_path) + "\"");
        std::string line;
        while (std::getline(in, line)) {
            const auto hash = line.find('#');
            if (hash != std::string::npos) line.resize(hash);
            std::istringstream f(line);
            DeviceSpec d;
            double bw = 0, cap = 0;
            if (f >> d.name >> bw >> cap) {
                d.bandwidth_bytes = bw * 1e9;
                d.capacity_bytes = cap * 1e9;
                if (d.bandwidth_bytes <= 0.0 || d.capacity_bytes <= 0.0)
                    throw std::runtime_error("device \"" + d.name + "\" needs positive bandwidth and capacity");
                catalog.push_back(d);
            }
        }
    }
    for (const DeviceSpec& d : catalog)
        if (d.name == name) return d;
    throw std::invalid_argument("unknown device \"" + name + "\"");
}

double peak_glups(const DeviceSpec& d, int bits) { return d.bandwidth_bytes / double(model_bytes_per_cell(bits)) / 1e9; }

double memory_fraction(const DeviceSpec& d, int bits, int64_t L) {
    return double(model_bytes_per_cell(bits)) * double(L) * double(L) * double(L) / d.capacity_bytes;
}

// ---------------------------------------------------------------------------- driver
namespace {

class Driver {
  public:
    Driver(const RunPlan& plan, const CaseSetup& setup, DynamicsRegistry& reg, DeviceRun& run,
           const std::set<int>& dispatch)
        : plan_(plan), setup_(setup), reg_(reg), run_(run), dispatch_(dispatch) {}

    RunArtifacts execute();

  private:
    void sample(int64_t step);
    std::string path(const std::string& n) const { return (std::filesystem::path(plan_.out_dir) / n).string(); }
    void write_series() const;
    void write_profiles() const;
    void write_perf(double seconds, int64_t steps) const;
    void write_manifest() const;
    void center_lines(std::vector<double>& line_ux, std::vector<double>& line_uz);

    const RunPlan& plan_;
    const CaseSetup& setup_;
    DynamicsRegistry& reg_;
    DeviceRun& run_;
    std::set<int> dispatch_;
    std::vector<std::string> extra_names_;
    std::vector<Row> rows_;
    double k0_ = 0, eps0_ = 0;
    bool have_prev_ = false;
    std::vector<std::vector<double>> prof_ux_, prof_uz_;
    std::vector<double> prof_t_;
    double last_perm_ = 0;
    int steady_hits_ = 0;
    std::vector<std::string> files_;
};

// Centre lines of the cavity (runner.cpp:449-462): ux(L/2, L/2, z) over z and
// uz(x, L/2, L/2) over x, read plane by plane from the device.
void Driver::center_lines(std::vector<double>& line_ux, std::vector<double>& line_uz) {
    const int64_t L = setup_.dims[0], nx = setup_.dims[0], ny = setup_.dims[1];
    line_ux.assign(std::size_t(L), 0.0);
    line_uz.assign(std::size_t(L), 0.0);
    const std::size_t pl = std::size_t(3 * nx * ny);
    int64_t z0 = 0;
    for (int k = 0; k < run_.slabs(); ++k) {
        Lattice& s = run_.slab(k);
        const int nz = s.slab_planes();
        const int chunk = 16;
        std::vector<double> buf(std::size_t(chunk) * pl);
        for (int z = 0; z < nz; z += chunk) {
            const int m = std::min(chunk, nz - z);
            s.velocity_planes(z, m, buf.data());
            for (int j = 0; j < m; ++j) {
                const int64_t zg = z0 + z + j;
                const double* p = buf.data() + std::size_t(j) * pl;  // [ux|uy|uz][y][x]
                line_ux[std::size_t(zg)] = p[(L / 2) * nx + L / 2];
                if (zg == L / 2)
                    for (int64_t x = 0; x < L; ++x) line_uz[std::size_t(x)] = p[2 * nx * ny + (L / 2) * nx + x];
            }
        }
        z0 += nz;
    }
}

void Driver::sample(int64_t step) {
    Row row;
    row.step = step;
    row.t_c = double(step) / setup_.t_c;
    row.k = run_.kinetic_energy();
    row.eps = run_.enstrophy();
    if (step == 0) {
        k0_ = row.k;
        eps0_ = row.eps;
    }
    const CaseKind kind = plan_.case_config.kind;
    if (kind == CaseKind::Tgv) {
        row.extras.push_back(k0_ == 0.0 ? 0.0 : row.k / k0_);
        row.extras.push_back(eps0_ == 0.0 ? 0.0 : row.eps / eps0_);
    } else if (kind == CaseKind::Cavity) {
        double du = 0.0;
        if (have_prev_) {
            double nn = 0, dd = 0;
            run_.convergence_sums(&nn, &dd);
            if (dd > 0.0) du = std::sqrt(nn / dd) * setup_.t_c / double(plan_.output_every);
        }
        row.extras.push_back(du);
        run_.snapshot_velocity();
        have_prev_ = true;
        std::vector<double> lx, lz;
        center_lines(lx, lz);
        prof_ux_.push_back(std::move(lx));
        prof_uz_.push_back(std::move(lz));
        prof_t_.push_back(row.t_c);
    } else {
        row.extras = run_.porous_extras(setup_.sample_begin, setup_.sample_end, plan_.case_config.viscosity(),
                                        plan_.case_config.geometry == "plates");
        const double k_perm = row.extras[0];
        if (step > 0) {
            const double prev = last_perm_;
            if (k_perm != 0.0 && prev != 0.0 && std::abs(k_perm - prev) <= plan_.steady_tol * std::abs(k_perm))
                ++steady_hits_;
            else
                steady_hits_ = 0;
        }
        last_perm_ = k_perm;
    }
    // DiagnosticsSeries::append (diagnostics.cpp:164-179)
    if (!rows_.empty() && row.step <= rows_.back().step)
        throw std::invalid_argument("diagnostics steps must be strictly increasing");
    if (!std::isfinite(row.k) || !std::isfinite(row.eps))
        throw std::invalid_argument("diagnostics values must be finite");
    for (double v : row.extras)
        if (!std::isfinite(v)) throw std::invalid_argument("diagnostics values must be finite");
    if (row.extras.size() != extra_names_.size()) throw std::invalid_argument("diagnostics row arity mismatch");
    rows_.push_back(std::move(row));
}

void Driver::write_series() const {
    std::string out = "step,t_c,k,eps";
    for (const std::string& n : extra_names_) out += "," + n;
    out += "\n";
    for (const Row& r : rows_) {
        out += std::to_string(r.step);
        out += "," + g17(r.t_c);
        out += "," + g17(r.k);
        out += "," + g17(r.eps);
        for (double v : r.extras) out += "," + g17(v);
        out += "\n";
    }
    std::ofstream f(path("series.csv"), std::ios::binary);
    f << out;
}

void Driver::write_profiles() const {
    const int64_t L = setup_.dims[0];
    std::vector<std::size_t> pick;
    for (std::size_t s = 0; s < prof_t_.size(); ++s)
        if (prof_t_[s] >= plan_.avg_from_tc) pick.push_back(s);
    if (pick.empty() && !prof_ux_.empty()) pick.push_back(prof_ux_.size() - 1);
    if (pick.empty()) return;
    // diag::averaged_profile: tree_mean over the snapshots, point by point
    auto mean_at = [&](const std::vector<std::vector<double>>& snaps, int64_t p) {
        std::vector<double> col;
        for (std::size_t s : pick) col.push_back(snaps[s][std::size_t(p)]);
        return tree_sum_host(col.data(), int64_t(col.size())) / double(col.size());
    };
    const double u0 = plan_.case_config.lattice_velocity();
    std::string out = "z_c,ux_over_u0,x_c,uz_over_u0\n";
    for (int64_t i = 0; i < L; ++i) {
        const double coord = 2.0 * (double(i) + 0.5) / double(L) - 1.0;  // normalized_coordinate
        out += g17(coord) + "," + g17(mean_at(prof_ux_, i) / u0) + "," + g17(coord) + "," +
               g17(mean_at(prof_uz_, i) / u0) + "\n";
    }
    std::ofstream f(path("profiles.csv"), std::ios::binary);
    f << out;
}

void Driver::write_perf(double seconds, int64_t steps) const {
    const int64_t cells = run_.num_cells();
    const double mlups = seconds > 0.0 ? double(cells) * double(steps) / seconds / 1e6 : 0.0;
    const int bits = plan_.case_config.precision_bits;
    std::ostringstream out;
    out << "cells,steps,seconds,mlups,device,bytes_per_cell,peak_glups,fraction_of_peak,memory_fraction\n";
    out << cells << "," << steps << "," << g17(seconds) << "," << g17(mlups);
    if (plan_.perf_device) {
        DeviceSpec d;
        try {
            d = lookup_device(*plan_.perf_device, plan_.device_catalog ? plan_.device_catalog->c_str() : nullptr);
        } catch (const std::invalid_argument&) {
            throw std::invalid_argument("unknown device \"" + *plan_.perf_device +
                                        "\"; list entries in the catalog file or use A100-SXM4-40GB");
        }
        const double peak = peak_glups(d, bits);
        out << "," << d.name << "," << model_bytes_per_cell(bits) << "," << g17(peak) << ","
            << g17(mlups / (peak * 1e3)) << "," << g17(memory_fraction(d, bits, plan_.case_config.L));
    } else {
        out << ",," << model_bytes_per_cell(bits) << ",,,";
    }
    out << "\n";
    std::ofstream f(path("perf.csv"), std::ios::binary);
    f << out.str();
}

// Replayable manifest (runner.cpp:578-647): the resolved configuration, the
// registry's tags and the artefact list.
void Driver::write_manifest() const {
    Config m;
    const CaseConfig& cc = plan_.case_config;
    m.set("case.kind", kind_name(cc.kind));
    m.set("case.L", std::to_string(cc.L));
    m.set("case.Re", g17(cc.Re));
    m.set("case.Ma", g17(cc.Ma));
    m.set("case.collision", collision_name(cc.collision));
    if (cc.smagorinsky_c) m.set("case.smagorinsky", g17(*cc.smagorinsky_c));
    m.set("case.lambda", g17(cc.lambda));
    m.set("case.omega_bulk_ho", g17(cc.omega_bulk_ho));
    m.set("case.precision", cc.precision_bits == 32 ? "f32" : "f64");
    if (cc.q == 27) m.set("case.lattice", "d3q27");
    if (cc.kind == CaseKind::Porous) {
        m.set("case.drive", cc.drive == DriveKind::Velocity ? "velocity" : "pressure");
        m.set("case.geometry", cc.geometry);
        m.set("case.H", std::to_string(cc.plate_layers));
        m.set("case.tau", g17(cc.tau));
        m.set("case.delta_rho", g17(cc.delta_rho));
        m.set("case.upstream", std::to_string(cc.upstream));
        m.set("case.downstream", std::to_string(cc.downstream));
        if (cc.voxel_dims[0] > 0) {
            m.set("case.voxel_dims", std::to_string(cc.voxel_dims[0]) + "," + std::to_string(cc.voxel_dims[1]) + "," +
                                         std::to_string(cc.voxel_dims[2]));
            m.set("case.voxel_dx", g17(cc.voxel_dx));
            m.set("case.voxel_threshold", g17(cc.voxel_threshold));
        }
    }
    m.set("run.blocks", std::to_string(cc.block_grid[0]) + "," + std::to_string(cc.block_grid[1]) + "," +
                            std::to_string(cc.block_grid[2]));
    m.set("run.workers", std::to_string(cc.workers));
    m.set("run.tmax", plan_.until_steady ? "steady" : std::to_string(plan_.tmax_steps));
    m.set("run.steady_tol", g17(plan_.steady_tol));
    m.set("run.max_steps", std::to_string(plan_.max_steps));
    m.set("run.output_every", std::to_string(plan_.output_every));
    m.set("run.dump_every", std::to_string(plan_.dump_every));
    m.set("run.avg_from", g17(plan_.avg_from_tc));
    m.set("run.out", plan_.out_dir);
    if (plan_.perf_device) m.set("run.perf_device", *plan_.perf_device);
    if (plan_.device_catalog) m.set("run.device_catalog", *plan_.device_catalog);
    m.set("run.reference_check", plan_.reference_check ? "true" : "false");
    // device-runtime keys only when configured (a default manifest matches the reference's)
    if (!plan_.devices.empty()) {
        std::string d;
        for (int v : plan_.devices) d += (d.empty() ? "" : ",") + std::to_string(v);
        m.set("run.devices", d);
    }
    if (plan_.arith == DLB_ARITH_FAST) m.set("run.arith", "fast");
    if (plan_.layout == DLB_LAYOUT_AA) m.set("run.layout", "aa");
    if (plan_.flags) m.set("run.porous", plan_.porous_name);
    std::string models;
    for (int t = 0; t < reg_.num_tags(); ++t) {
        if (!dispatch_.count(t)) continue;
        if (!models.empty()) models += ",";
        models += reg_.chain_for(t);
    }
    m.set("dispatch.models", models);
    std::string out = m.render();
    out += "[registry]\n";
    for (int t = 0; t < reg_.num_tags(); ++t) out += "tag_" + std::to_string(t) + " = " + reg_.chain_for(t) + "\n";
    out += "\n[files]\n";
    int idx = 0;
    for (const std::string& f : files_) out += "file_" + std::to_string(idx++) + " = " + f + "\n";
    std::ofstream f(path("manifest"), std::ios::binary);
    f << out;
}

RunArtifacts Driver::execute() {
    std::filesystem::create_directories(plan_.out_dir);
    switch (plan_.case_config.kind) {
        case CaseKind::Tgv: extra_names_ = {"k_over_k0", "eps_over_eps0"}; break;
        case CaseKind::Cavity: extra_names_ = {"du_per_tc"}; break;
        case CaseKind::Porous: extra_names_ = {"k_perm", "ubar", "dp", "ux_in", "ux_out"}; break;
    }
    sample(0);
    double seconds = 0.0;
    int64_t step = 0;
    const int64_t limit = plan_.until_steady ? plan_.max_steps : plan_.tmax_steps;
    while (step < limit) {
        const int64_t chunk = std::min(plan_.output_every, limit - step);
        const auto t0 = std::chrono::steady_clock::now();
        run_.advance(chunk, true);  // the sample's kinetic energy fused into the chunk's last step
        run_.synchronize();         // the chunk's device work is inside the timed region
        seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        step += chunk;
        sample(step);
        if (plan_.dump_every > 0 && step % plan_.dump_every == 0) {
            char name[32];
            std::snprintf(name, sizeof name, "dump_%08lld.dolb", static_cast<long long>(step));
            run_.write_field_dump(path(name));
            files_.push_back(name);
        }
        if (plan_.until_steady && steady_hits_ >= 3) break;
    }
    write_series();
    files_.insert(files_.begin(), "series.csv");
    if (plan_.case_config.kind == CaseKind::Cavity) {
        write_profiles();
        files_.push_back("profiles.csv");
    }
    write_perf(seconds, step);
    files_.push_back("perf.csv");
    write_manifest();
    files_.push_back("manifest");
    RunArtifacts a;
    a.out_dir = plan_.out_dir;
    a.files = files_;
    a.steps = step;
    a.mlups = seconds > 0.0 ? double(run_.num_cells()) * double(step) / seconds / 1e6 : 0.0;
    return a;
}

}  // namespace

RunArtifacts execute(const Config& config) {
    const RunPlan plan = resolve(config);
    const CaseSetup setup = make_setup(plan.case_config);
    DynamicsRegistry reg;
    std::vector<int32_t> slot_of(setup.chains.size());
    for (std::size_t k = 0; k < setup.chains.size(); ++k) slot_of[k] = reg.register_chain(setup.chains[k]);
    // the configured dispatch set (unknown names fail here; missing-but-used
    // chains fail at the first step with the chain string)
    std::set<int> dispatch;
    if (plan.dispatch_models.empty()) {
        for (int t = 0; t < reg.num_tags(); ++t) dispatch.insert(t);
    } else {
        for (const std::string& n : plan.dispatch_models) dispatch.insert(reg.tag_for(n));
    }
    // z-slab decomposition: as many slabs as the reference's block grid has
    // blocks (the update is decomposition-invariant), over the listed devices
    const CaseConfig& cc = plan.case_config;
    const int64_t blocks = int64_t(cc.block_grid[0]) * cc.block_grid[1] * cc.block_grid[2];
    if (blocks < 1) throw std::invalid_argument("run.blocks counts must be >= 1");
    const int slabs = int(std::min<int64_t>(blocks, setup.dims[2]));
    std::vector<int> devices = plan.devices;
    if (devices.empty()) {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
            cudaGetLastError();
            throw DeviceError("no CUDA device available for the run");
        }
        for (int d = 0; d < n; ++d) devices.push_back(d);
    }
    DeviceRun run(setup.dims, setup.periodic, reg, cc.q, cc.precision_bits, slabs, devices, plan.arith, plan.flags,
                  plan.layout);
    std::vector<int32_t> slots;
    if (!setup.chain_index.empty()) {
        slots.resize(setup.chain_index.size());
        for (std::size_t g = 0; g < slots.size(); ++g) slots[g] = slot_of[setup.chain_index[g]];
    }
    run.fill(slots, slot_of[0], setup);
    run.set_dispatch(dispatch);
    Driver driver(plan, setup, reg, run, dispatch);
    return driver.execute();
}

std::vector<std::string> show_models(const Config& config) {
    const RunPlan plan = resolve(config);
    return setup_models(make_setup(plan.case_config));
}

}  // namespace dlb::run
