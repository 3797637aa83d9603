// DeviceRun (device_run.hpp): single-process multi-slab run over dlb::Lattice.
#include "device_run.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <stdexcept>

#include "tree.hpp"

namespace dlb {

std::vector<std::pair<int64_t, int64_t>> balanced_partition(int64_t n, int k) {
    if (k < 1) throw std::invalid_argument("partition: at least one block");
    if (n < k) throw std::invalid_argument("partition: more blocks than cells along z");
    std::vector<std::pair<int64_t, int64_t>> out;
    int64_t z = 0;
    for (int b = 0; b < k; ++b) {
        const int64_t len = n / k + (b < n % k ? 1 : 0);
        out.push_back({z, len});
        z += len;
    }
    return out;
}

DeviceRun::DeviceRun(std::array<int64_t, 3> dims, std::array<bool, 3> periodic, const DynamicsRegistry& reg, int q,
                     int precision_bits, int slabs, const std::vector<int>& devices, int arith, int flags,
                     int layout)
    : dims_(dims), periodic_(periodic), q_(q), bits_(precision_bits) {
    parts_ = balanced_partition(dims[2], slabs);
    for (int k = 0; k < slabs; ++k) {
        dlb_lattice_desc d{};
        d.dims[0] = dims[0];
        d.dims[1] = dims[1];
        d.dims[2] = parts_[std::size_t(k)].second;
        for (int a = 0; a < 3; ++a) d.periodic[a] = periodic[std::size_t(a)];
        d.q = q;
        d.precision_bits = precision_bits;
        d.layout = layout;
        d.arith = arith;
        d.device = devices.empty() ? 0 : devices[std::size_t(k) % devices.size()];
        d.z_origin = parts_[std::size_t(k)].first;
        d.global_nz = dims[2];
        d.flags = flags;
        slabs_.push_back(std::make_unique<Lattice>(d, reg));
    }
    for (int k = 0; k + 1 < slabs; ++k) slabs_[std::size_t(k + 1)]->link_lower(*slabs_[std::size_t(k)]);
    if (slabs > 1 && periodic[2]) slabs_.front()->link_lower(*slabs_.back());
}

void DeviceRun::fill(const std::vector<int32_t>& slot_of_cell, int32_t uniform_slot, const CaseSetup& setup) {
    const int64_t nxy = dims_[0] * dims_[1];
    for (std::size_t k = 0; k < slabs_.size(); ++k) {
        Lattice& s = *slabs_[k];
        if (slot_of_cell.empty()) s.set_uniform_slot(uniform_slot);
        else s.set_slots(slot_of_cell.data() + parts_[k].first * nxy);
        if (setup.state == InitState::Tgv) s.fill_tgv(dims_[0], setup.u_inf);
        else s.fill_uniform(1.0, 0.0, 0.0, 0.0);
    }
    exchange();
}

void DeviceRun::set_dispatch(const std::set<int>& tags) {
    const std::vector<int32_t> t(tags.begin(), tags.end());
    for (auto& s : slabs_) s->set_dispatch(t.data(), t.size());
}

void DeviceRun::exchange() {
    if (slabs_.size() == 1) return;
    for (auto& s : slabs_) s->quiesce();
    for (auto& s : slabs_) s->exchange();
}

void DeviceRun::advance(int64_t nsteps, bool kinetic_last) {
    if (nsteps <= 0) return;
    if (slabs_.size() == 1) {
        if (kinetic_last) slabs_.front()->request_kinetic();
        slabs_.front()->step(nsteps);
    } else {
        // eager dispatch check on every slab before any of them writes
        std::vector<Lattice*> group;
        for (auto& s : slabs_) {
            s->check_dispatch();
            group.push_back(s.get());
        }
        Lattice::step_group(group, nsteps);
    }
    steps_ += nsteps;
}

void DeviceRun::synchronize() {
    for (auto& s : slabs_) s->synchronize();
}

int64_t DeviceRun::step_bytes() const {
    int64_t b = 0;
    for (const auto& s : slabs_) b += s->step_bytes();
    return b;
}

std::vector<double> DeviceRun::gather_populations() {
    const int64_t nxy = dims_[0] * dims_[1], n = num_cells();
    std::vector<double> out(std::size_t(q_ * n));
    for (std::size_t k = 0; k < slabs_.size(); ++k) {
        const int64_t z0 = parts_[k].first, nz = parts_[k].second, m = nz * nxy;
        std::vector<double> buf(std::size_t(q_ * m));
        slabs_[k]->download(buf.data());
        for (int i = 0; i < q_; ++i)
            std::memcpy(out.data() + i * n + z0 * nxy, buf.data() + i * m, std::size_t(m) * 8);
    }
    return out;
}

std::vector<uint8_t> DeviceRun::gather_raw() {
    const int64_t nxy = dims_[0] * dims_[1], n = num_cells();
    const int s = bits_ / 8;
    std::vector<uint8_t> out(std::size_t(q_ * n * s));
    for (std::size_t k = 0; k < slabs_.size(); ++k) {
        const int64_t z0 = parts_[k].first, nz = parts_[k].second, m = nz * nxy;
        std::vector<uint8_t> buf(std::size_t(q_ * m * s));
        slabs_[k]->download_raw(buf.data());
        for (int i = 0; i < q_; ++i)
            std::memcpy(out.data() + (i * n + z0 * nxy) * s, buf.data() + i * m * s, std::size_t(m * s));
    }
    return out;
}

// DOLB1 field dump (accelerated_lattice.cpp:313-341): magic "DOLB1", u8 bytes
// per value, u32 q, 3 x u64 dims, then the q arrays x fastest in the storage type.
void DeviceRun::write_field_dump(const std::string& path) {
    const std::vector<uint8_t> raw = gather_raw();
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write field dump \"" + path + "\"");
    const uint8_t prec = uint8_t(bits_ / 8);
    const uint32_t q = uint32_t(q_);
    const uint64_t d[3] = {uint64_t(dims_[0]), uint64_t(dims_[1]), uint64_t(dims_[2])};
    out.write("DOLB1", 5);
    out.write(reinterpret_cast<const char*>(&prec), 1);
    out.write(reinterpret_cast<const char*>(&q), 4);
    out.write(reinterpret_cast<const char*>(d), 24);
    out.write(reinterpret_cast<const char*>(raw.data()), std::streamsize(raw.size()));
    if (!out) throw std::runtime_error("short write to field dump \"" + path + "\"");
}

void DeviceRun::gather_macroscopic(std::vector<double>& rho, std::vector<double>& ux, std::vector<double>& uy,
                                   std::vector<double>& uz) {
    const int64_t nxy = dims_[0] * dims_[1], n = num_cells();
    for (auto* v : {&rho, &ux, &uy, &uz}) v->assign(std::size_t(n), 0.0);
    for (std::size_t k = 0; k < slabs_.size(); ++k) {
        const std::size_t off = std::size_t(parts_[k].first * nxy);
        slabs_[k]->gather_macroscopic(rho.data() + off, ux.data() + off, uy.data() + off, uz.data() + off);
    }
}

// The runner's diagnostics reduce one value sequence over the whole domain with
// diag::tree_sum; every slab reduces the tree nodes inside its own segment of
// that sequence and the host combines them (tree.hpp), so the result has the
// bits of the single-array sum for any decomposition.
double DeviceRun::tree_reduce(int quantity, int64_t x_begin, int64_t x_end, int64_t* count_out) {
    const bool ens = quantity == DLB_Q_ENSTROPHY;
    const int64_t nx = dims_[0], ny = dims_[1], nz_g = dims_[2];
    // FD8 enstrophy on a decomposed domain: the 4 global velocity planes below
    // and above each slab, gathered from the slabs that own them
    std::vector<std::vector<double>> below(slabs_.size()), above(slabs_.size());
    if (ens && slabs_.size() > 1) {
        const std::size_t pl = std::size_t(3 * nx * ny);
        std::map<int64_t, std::vector<double>> have;
        for (std::size_t k = 0; k < slabs_.size(); ++k) {
            const int64_t z0 = parts_[k].first, nz = parts_[k].second;
            const int lo = int(std::min<int64_t>(4, nz)), hi0 = int(std::max<int64_t>(0, nz - 4));
            std::set<int> want;
            for (int j = 0; j < lo; ++j) want.insert(j);
            for (int j = hi0; j < nz; ++j) want.insert(j);
            const int a = *want.begin(), b = *want.rbegin();
            std::vector<double> planes(std::size_t(b - a + 1) * pl);
            slabs_[k]->velocity_planes(a, b - a + 1, planes.data());
            for (int j : want)
                have[z0 + j].assign(planes.begin() + std::ptrdiff_t(std::size_t(j - a) * pl),
                                    planes.begin() + std::ptrdiff_t(std::size_t(j - a + 1) * pl));
        }
        auto block = [&](int64_t zf, std::vector<double>& dst) {
            dst.assign(4 * pl, 0.0);
            for (int r = 0; r < 4; ++r) {
                const int64_t zg = zf + r;
                if (!periodic_[2] && (zg < 0 || zg >= nz_g)) continue;
                const auto& src = have.at(((zg % nz_g) + nz_g) % nz_g);
                std::copy(src.begin(), src.end(), dst.begin() + std::ptrdiff_t(r * pl));
            }
        };
        for (std::size_t k = 0; k < slabs_.size(); ++k) {
            block(parts_[k].first - 4, below[k]);
            block(parts_[k].first + parts_[k].second, above[k]);
        }
    }
    std::vector<dlb_reduce_args> args(slabs_.size());
    for (std::size_t k = 0; k < slabs_.size(); ++k) {
        dlb_reduce_args& a = args[k];
        a = dlb_reduce_args{};
        a.quantity = quantity;
        for (int ax = 0; ax < 3; ++ax) a.periodic[ax] = periodic_[std::size_t(ax)];
        a.x_begin = x_begin;
        a.x_end = x_end;
        a.halo_below = below[k].empty() ? nullptr : below[k].data();
        a.halo_above = above[k].empty() ? nullptr : above[k].data();
    }
    std::vector<int64_t> counts(slabs_.size());
    int64_t n_total = 0;
    for (std::size_t k = 0; k < slabs_.size(); ++k) {
        counts[k] = slabs_[k]->reduce_count(args[k]);
        n_total += counts[k];
    }
    std::vector<dlb_tree_part> parts;
    int64_t begin = 0;
    for (std::size_t k = 0; k < slabs_.size(); ++k) {
        std::vector<dlb_tree_part> p;
        slabs_[k]->reduce_parts(args[k], n_total, begin, p);
        parts.insert(parts.end(), p.begin(), p.end());
        begin += counts[k];
    }
    if (count_out) *count_out = n_total;
    return tree_combine(n_total, parts.data(), parts.size());
}

double DeviceRun::tree_mean(int quantity, int64_t x_begin, int64_t x_end, const double* empty) {
    int64_t n = 0;
    const double s = tree_reduce(quantity, x_begin, x_end, &n);
    if (n == 0) {
        if (!empty) throw std::invalid_argument("mean of an empty set");  // diagnostics.cpp:21
        return *empty;
    }
    return s / double(n);
}

double DeviceRun::kinetic_energy() { return tree_mean(DLB_Q_KINETIC, 0, dims_[0], nullptr); }

double DeviceRun::enstrophy() { return tree_mean(DLB_Q_ENSTROPHY, 0, dims_[0], nullptr); }

void DeviceRun::snapshot_velocity() {
    for (auto& s : slabs_) s->snapshot_velocity();
}

void DeviceRun::convergence_sums(double* num, double* den) {
    *num = tree_reduce(DLB_Q_DU_NUM, 0, dims_[0], nullptr);
    *den = tree_reduce(DLB_Q_DU_DEN, 0, dims_[0], nullptr);
}

// Driver::porous_extras (runner.cpp:346-399): [k_perm, ubar, dp, ux_in, ux_out].
std::vector<double> DeviceRun::porous_extras(int64_t sample_begin, int64_t sample_end, double nu,
                                             bool aperture_mean) {
    const double zero = 0.0, one = 1.0;
    const int64_t x0 = sample_begin, x1 = sample_end - 1;
    auto plane_mean_p = [&](int64_t x) { return tree_mean(DLB_Q_PRESSURE_FLUID, x, x + 1, &zero); };
    auto plane_mean_ux = [&](int64_t x) { return tree_mean(DLB_Q_UX_FLUID, x, x + 1, &zero); };
    const double ubar = tree_mean(aperture_mean ? DLB_Q_UX_FLUID : DLB_Q_UX_ALL, sample_begin, sample_end, nullptr);
    const double rho_bar = tree_mean(DLB_Q_RHO_FLUID, sample_begin, sample_end, &one);
    const double dp = (plane_mean_p(x0) - plane_mean_p(x1)) / rho_bar;
    const double lx = double(x1 - x0);
    const double k_perm = std::abs(dp) < 1e-300 ? 0.0 : ubar * nu * lx / dp;  // diag::permeability
    return {k_perm, ubar, dp, plane_mean_ux(1), plane_mean_ux(dims_[0] - 2)};
}

}  // namespace dlb
