// dlb_dolb.hpp — header-only C++ drop-in of the B200 path for code written
// against the reference's own C++ API ("dolb", proj/include/dolb/*.hpp).
//
// Include it next to the reference's headers and link libdlb_b200.so:
//
//   g++ -std=gnu++20 app.cpp -I<dolb>/include -I<repo>/include <dolb objects>
//       -L<repo>/paper_2506_09242_b200/_lib -ldlb_b200 -Wl,-rpath,<...>/_lib -pthread
//
// What it replaces (file:line under /root/reference/proj):
//   dlb_dolb::collide_and_stream<T>   collide_and_stream<T>(AcceleratedBlock<T>&, const
//                                     DynamicsRegistry&, const std::vector<ChainRecipe<T>>&,
//                                     const DispatchSet&, int)   include/dolb/accelerated_lattice.hpp:124-127
//   dlb_dolb::DeviceRun<T>            MultiBlockRun<T>             include/dolb/multiblock.hpp:119-176
//   dlb_dolb::build_device_run<T>     build_run<T>                 include/dolb/cases.hpp:103-108, src/cases.cpp:279-297
//
// Everything below is marshalling over the C ABI (include/dlb.h): the state
// lives in HBM (DeviceRun) or is streamed through it (collide_and_stream on a
// host block); the arithmetic is the device kernels', bit-identical to the
// reference in the exact mode used here. Errors come back as the reference's
// exception types: dolb::DispatchError (chain name), dolb::ExchangeError,
// std::invalid_argument (configuration), std::runtime_error (device / other).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dlb.h"
#include "dolb/accelerated_lattice.hpp"
#include "dolb/cases.hpp"
#include "dolb/chain.hpp"
#include "dolb/multiblock.hpp"

namespace dlb_dolb {

// dlb_status -> the reference's exception types (proj/src/capi.cpp:20-39 in reverse).
inline void check(dlb_status s) {
    if (s == DLB_OK) return;
    const std::string msg = dlb_last_error();
    switch (s) {
        case DLB_ERROR_DISPATCH: {
            // "collision model \"<chain>\" is not part of the dispatch set"
            const auto a = msg.find('"'), b = msg.rfind('"');
            throw dolb::DispatchError(a != std::string::npos && b > a ? msg.substr(a + 1, b - a - 1) : msg);
        }
        case DLB_ERROR_EXCHANGE: throw dolb::ExchangeError(msg);
        case DLB_ERROR_CONFIG:
        case DLB_ERROR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        default: throw std::runtime_error(msg);
    }
}

// The reference registry mirrored into a dlb_registry: same instances in the
// same slot order (chain string + serialize_params record, i.e. the
// registry's own parameter table), hence the same tags (sorted chain strings).
class Registry {
  public:
    explicit Registry(const dolb::DynamicsRegistry& ref) {
        check(dlb_registry_new(&h_));
        sync(ref);
    }
    ~Registry() { dlb_registry_free(h_); }
    Registry(const Registry&) = delete;
    Registry& operator=(const Registry&) = delete;

    // Registers the instances the reference registry gained since the last call.
    void sync(const dolb::DynamicsRegistry& ref) {
        for (int slot = mirrored_; slot < ref.num_instances(); ++slot) {
            const auto& in = ref.instance(slot);
            const double* p = ref.params_table().data() + in.param_offset;
            int32_t got = -1;
            check(dlb_registry_register(h_, in.chain_str.c_str(), in.param_len ? p : nullptr,
                                        size_t(in.param_len), &got));
            if (got != slot) throw std::logic_error("registry mirror out of slot order");
        }
        mirrored_ = ref.num_instances();
    }
    // Same content as `ref` (slots, chain strings, parameters)?
    bool mirrors(const dolb::DynamicsRegistry& ref) const {
        return mirrored_ == ref.num_instances() && chains_ == snapshot(ref).first && params_ == snapshot(ref).second;
    }
    void remember(const dolb::DynamicsRegistry& ref) { std::tie(chains_, params_) = snapshot(ref); }
    dlb_registry* get() const { return h_; }

  private:
    static std::pair<std::vector<std::string>, std::vector<double>> snapshot(const dolb::DynamicsRegistry& ref) {
        std::vector<std::string> c;
        for (int s = 0; s < ref.num_instances(); ++s) c.push_back(ref.instance(s).chain_str);
        return {c, ref.params_table()};
    }
    dlb_registry* h_ = nullptr;
    int mirrored_ = 0;
    std::vector<std::string> chains_;
    std::vector<double> params_;
};

namespace detail {
// One mirror per reference registry (re-validated against its content on
// every call, so a registry freed and reallocated at the same address is
// never mistaken for the old one).
inline const Registry& mirror_of(const dolb::DynamicsRegistry& ref) {
    thread_local std::map<const dolb::DynamicsRegistry*, std::unique_ptr<Registry>> cache;
    auto& m = cache[&ref];
    if (!m || !m->mirrors(ref)) {
        m = std::make_unique<Registry>(ref);
        m->remember(ref);
    }
    return *m;
}
}  // namespace detail

// Drop-in for dolb::collide_and_stream<T> on an AcceleratedBlock<T>: same
// pre-condition (envelope of f_in current), same post-condition (f_in holds
// the new state, f_out the previous one: the arrays are swapped as in
// accelerated_lattice.cpp:199), same eager DispatchError before any write.
// `recipes` are not read: the device compiles the same recipes from the
// registry (compile_chain<T> semantics, chain.hpp:147-187). `nthreads` has no
// meaning on the GPU (results never depend on it, accelerated_lattice.cpp:183-198).
template <typename T>
void collide_and_stream(dolb::AcceleratedBlock<T>& block, const dolb::DynamicsRegistry& registry,
                        const std::vector<dolb::ChainRecipe<T>>& recipes, const dolb::DispatchSet& dispatch,
                        int nthreads = 1) {
    (void)recipes;
    const Registry& reg = detail::mirror_of(registry);
    std::vector<int32_t> tags(dispatch.tags().begin(), dispatch.tags().end());
    dlb_block_view v{};
    v.precision_bits = int32_t(8 * sizeof(T));
    v.q = 19;
    for (int a = 0; a < 3; ++a) v.interior[a] = block.interior[std::size_t(a)];
    v.f_in = block.f_in.data();
    v.f_out = block.f_out.data();
    v.tag = block.tag.data();
    v.param_index = block.param_index.data();
    check(dlb_collide_and_stream(reg.get(), &v, tags.empty() ? nullptr : tags.data(), tags.size(), nthreads));
    if (v.f_in == static_cast<void*>(block.f_out.data())) std::swap(block.f_in, block.f_out);
}

// Device twin of dolb::MultiBlockRun<T>: the global domain as z-slabs (the
// reference's balanced split along z, multiblock.cpp:24-31), each resident in
// HBM on one GPU, linked through peer memory (the halo is pushed by the
// boundary-plane kernel every step). Public surface follows MultiBlockRun.
template <typename T>
class DeviceRun {
  public:
    DeviceRun(std::array<std::int64_t, 3> dims, std::array<bool, 3> periodic,
              std::shared_ptr<const dolb::DynamicsRegistry> registry, dolb::DispatchSet dispatch, int slabs = 1,
              std::vector<int> devices = {0})
        : dims_(dims), periodic_(periodic), registry_(std::move(registry)), dispatch_(std::move(dispatch)),
          mirror_(std::make_unique<Registry>(*registry_)) {
        if (slabs < 1 || slabs > dims[2]) throw std::invalid_argument("partition: bad slab count");
        if (devices.empty()) devices = {0};
        std::int64_t z = 0;
        for (int k = 0; k < slabs; ++k) {
            const std::int64_t nz = dims[2] / slabs + (k < dims[2] % slabs ? 1 : 0);
            dlb_lattice_desc d{};
            d.dims[0] = dims[0];
            d.dims[1] = dims[1];
            d.dims[2] = nz;
            for (int a = 0; a < 3; ++a) d.periodic[a] = periodic[std::size_t(a)] ? 1 : 0;
            d.q = 19;
            d.precision_bits = int32_t(8 * sizeof(T));
            d.layout = DLB_LAYOUT_TWO_POP;
            d.arith = DLB_ARITH_EXACT;
            d.device = devices[std::size_t(k) % devices.size()];
            d.z_origin = z;
            d.global_nz = dims[2];
            dlb_lattice* h = nullptr;
            check(dlb_lattice_create(&d, mirror_->get(), &h));
            slabs_.push_back(h);
            parts_.push_back({z, nz});
            z += nz;
        }
        for (int k = 0; k + 1 < slabs; ++k) check(dlb_lattice_link_local(slabs_[std::size_t(k)], slabs_[std::size_t(k + 1)]));
        if (slabs > 1 && periodic[2]) check(dlb_lattice_link_local(slabs_.back(), slabs_.front()));
        set_dispatch(dispatch_);
    }
    ~DeviceRun() {
        for (dlb_lattice* h : slabs_) dlb_lattice_free(h);
    }
    DeviceRun(DeviceRun&& o) noexcept { *this = std::move(o); }
    DeviceRun& operator=(DeviceRun&& o) noexcept {
        std::swap(dims_, o.dims_);
        std::swap(periodic_, o.periodic_);
        std::swap(registry_, o.registry_);
        std::swap(dispatch_, o.dispatch_);
        std::swap(mirror_, o.mirror_);
        std::swap(slabs_, o.slabs_);
        std::swap(parts_, o.parts_);
        std::swap(slot_, o.slot_);
        return *this;
    }
    DeviceRun(const DeviceRun&) = delete;
    DeviceRun& operator=(const DeviceRun&) = delete;

    const dolb::DynamicsRegistry& registry() const { return *registry_; }
    const dolb::DispatchSet& dispatch() const { return dispatch_; }
    void set_dispatch(dolb::DispatchSet d) {
        dispatch_ = std::move(d);
        std::vector<int32_t> t(dispatch_.tags().begin(), dispatch_.tags().end());
        for (dlb_lattice* h : slabs_) check(dlb_lattice_set_dispatch(h, t.empty() ? nullptr : t.data(), t.size()));
    }
    std::int64_t num_cells() const { return dims_[0] * dims_[1] * dims_[2]; }
    int slabs() const { return int(slabs_.size()); }

    // MultiBlockRun::fill (multiblock.cpp:252-287): slot and equilibrium2<T>(T(rho), T(u)) per cell.
    void fill(const std::function<int(std::int64_t, std::int64_t, std::int64_t)>& slot_of,
              const std::function<void(std::int64_t, std::int64_t, std::int64_t, double&, std::array<double, 3>&)>&
                  state_of) {
        const std::int64_t nxy = dims_[0] * dims_[1];
        slot_.assign(std::size_t(num_cells()), 0);
        for (std::size_t k = 0; k < slabs_.size(); ++k) {
            const auto [z0, nz] = parts_[k];
            const std::size_t n = std::size_t(nz * nxy);
            std::vector<double> rho(n), ux(n), uy(n), uz(n);
            for (std::int64_t z = 0; z < nz; ++z)
                for (std::int64_t y = 0; y < dims_[1]; ++y)
                    for (std::int64_t x = 0; x < dims_[0]; ++x) {
                        const std::size_t c = std::size_t((z * dims_[1] + y) * dims_[0] + x);
                        slot_[std::size_t(z0 * nxy) + c] = slot_of(x, y, z0 + z);
                        double r = 1.0;
                        std::array<double, 3> u = {0, 0, 0};
                        state_of(x, y, z0 + z, r, u);
                        rho[c] = r;
                        ux[c] = u[0];
                        uy[c] = u[1];
                        uz[c] = u[2];
                    }
            check(dlb_lattice_set_slots(slabs_[k], slot_.data() + z0 * nxy));
            check(dlb_lattice_fill_equilibrium(slabs_[k], rho.data(), ux.data(), uy.data(), uz.data()));
        }
        exchange();
    }

    // Envelope (halo) exchange only; valid before the first step.
    void exchange() { check(dlb_lattices_exchange(slabs_.data(), slabs_.size())); }

    // MultiBlockRun::advance (multiblock.cpp:376-419): sample(step) after every
    // sample_every-th step, with the state quiescent.
    void advance(std::int64_t nsteps, std::int64_t sample_every = 0,
                 const std::function<void(std::int64_t)>& sample = nullptr) {
        if (nsteps <= 0) return;
        std::int64_t done = 0;
        while (done < nsteps) {
            std::int64_t chunk = nsteps - done;
            if (sample_every > 0) chunk = std::min(chunk, sample_every - (steps_ % sample_every));
            if (slabs_.size() == 1) check(dlb_lattice_step(slabs_[0], chunk));
            else check(dlb_lattices_step(slabs_.data(), slabs_.size(), chunk));
            done += chunk;
            steps_ += chunk;
            if (sample_every > 0 && steps_ % sample_every == 0 && sample) {
                synchronize();
                sample(done);
            }
        }
        synchronize();
    }
    void synchronize() {
        for (dlb_lattice* h : slabs_) check(dlb_lattice_synchronize(h));
    }

    // Canonical order: direction-major, x fastest (multiblock.cpp:421-441).
    std::vector<double> gather_populations() const {
        const std::int64_t nxy = dims_[0] * dims_[1], n = num_cells();
        std::vector<double> out(std::size_t(19 * n));
        for (std::size_t k = 0; k < slabs_.size(); ++k) {
            const auto [z0, nz] = parts_[k];
            const std::int64_t m = nz * nxy;
            std::vector<double> buf(std::size_t(19 * m));
            check(dlb_lattice_download_populations(slabs_[k], buf.data()));
            for (int i = 0; i < 19; ++i)
                std::copy(buf.begin() + i * m, buf.begin() + (i + 1) * m, out.begin() + i * n + z0 * nxy);
        }
        return out;
    }
    void gather_macroscopic(std::vector<double>& rho, std::vector<double>& ux, std::vector<double>& uy,
                            std::vector<double>& uz) const {
        const std::int64_t nxy = dims_[0] * dims_[1];
        for (auto* v : {&rho, &ux, &uy, &uz}) v->assign(std::size_t(num_cells()), 0.0);
        for (std::size_t k = 0; k < slabs_.size(); ++k) {
            const std::int64_t off = parts_[k].first * nxy;
            check(dlb_lattice_gather_macroscopic(slabs_[k], rho.data() + off, ux.data() + off, uy.data() + off,
                                                 uz.data() + off));
        }
    }
    // MultiBlockRun::gather_block (multiblock.cpp:487-511): one monolithic
    // block with the interior state, tags and parameter slots.
    dolb::AcceleratedBlock<T> gather_block() const {
        dolb::AcceleratedBlock<T> mono(dims_, {0, 0, 0}, dims_, periodic_);
        const std::int64_t nxy = dims_[0] * dims_[1], mvol = mono.vol();
        for (std::size_t k = 0; k < slabs_.size(); ++k) {
            const auto [z0, nz] = parts_[k];
            const std::int64_t m = nz * nxy;
            std::vector<T> buf(std::size_t(19 * m));
            check(dlb_lattice_download_raw(slabs_[k], buf.data()));
            for (std::int64_t z = 0; z < nz; ++z)
                for (std::int64_t y = 0; y < dims_[1]; ++y)
                    for (std::int64_t x = 0; x < dims_[0]; ++x) {
                        const std::int64_t c = (z * dims_[1] + y) * dims_[0] + x;
                        const std::int64_t at = mono.idx(x + 1, y + 1, z0 + z + 1);
                        const int s = slot_.empty() ? 0 : slot_[std::size_t(z0 * nxy + c)];
                        mono.param_index[std::size_t(at)] = s;
                        mono.tag[std::size_t(at)] = registry_->tag_of_slot(s);
                        for (int i = 0; i < 19; ++i)
                            mono.f_in[std::size_t(i) * std::size_t(mvol) + std::size_t(at)] =
                                buf[std::size_t(i * m + c)];
                    }
        }
        return mono;
    }

  private:
    std::array<std::int64_t, 3> dims_{};
    std::array<bool, 3> periodic_{};
    std::shared_ptr<const dolb::DynamicsRegistry> registry_;
    dolb::DispatchSet dispatch_;
    std::unique_ptr<Registry> mirror_;
    std::vector<dlb_lattice*> slabs_;
    std::vector<std::pair<std::int64_t, std::int64_t>> parts_;
    std::vector<int32_t> slot_;
    std::int64_t steps_ = 0;
};

// Drop-in for dolb::build_run<T> (src/cases.cpp:279-297): registers the
// setup's chains, builds the device run, fills tags and state. The device run
// decomposes along z only: block_grid[2] z-slabs (the x / y splits of the
// grid do not change any value, test_multiblock.cpp:234-256), spread over
// `devices` (round robin).
template <typename T>
DeviceRun<T> build_device_run(const dolb::CaseSetup& setup, std::array<int, 3> block_grid, int workers,
                              std::shared_ptr<dolb::DynamicsRegistry> registry,
                              std::optional<dolb::DispatchSet> dispatch = std::nullopt,
                              std::vector<int> devices = {0}) {
    (void)workers;
    std::map<const dolb::DynamicsChain*, int> slot_of;
    for (const auto& chain : setup.chains) slot_of[chain.get()] = registry->register_chain(*chain);
    dolb::DispatchSet ds = dispatch ? *dispatch : dolb::DispatchSet::all_of(*registry);
    DeviceRun<T> run(setup.dims, setup.periodic, registry, std::move(ds), std::max(1, block_grid[2]),
                     std::move(devices));
    run.fill([&](std::int64_t x, std::int64_t y, std::int64_t z) { return slot_of.at(setup.chain_of(x, y, z)); },
             setup.state_of);
    return run;
}

}  // namespace dlb_dolb
