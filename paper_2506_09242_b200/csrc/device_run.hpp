// DeviceRun: the device twin of MultiBlockRun<T> (proj/include/dolb/multiblock.hpp:119-176)
// for one process — the global domain split into z-slabs (the reference's
// balanced rule, multiblock.cpp:24-31), one dlb::Lattice per slab, slabs on
// the listed CUDA devices (round robin) and linked through peer memory so
// every step's halo moves inside the boundary launch. Public methods follow
// MultiBlockRun: fill, exchange, advance, gather_populations,
// gather_macroscopic, set_dispatch, plus the GPU-resident diagnostics the
// runner samples (runner.cpp:401-510) as split deterministic tree reductions.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "cases.hpp"
#include "chain.hpp"
#include "lattice.hpp"

namespace dlb {

// Balanced split of n into k parts: the first n % k get one extra (multiblock.cpp:24-31).
std::vector<std::pair<int64_t, int64_t>> balanced_partition(int64_t n, int k);

class DeviceRun {
  public:
    DeviceRun(std::array<int64_t, 3> dims, std::array<bool, 3> periodic, const DynamicsRegistry& reg, int q,
              int precision_bits, int slabs, const std::vector<int>& devices, int arith = DLB_ARITH_EXACT,
              int flags = 0, int layout = DLB_LAYOUT_TWO_POP);
    DeviceRun(const DeviceRun&) = delete;
    DeviceRun& operator=(const DeviceRun&) = delete;

    // Registry slot of every cell (global, x fastest) or one slot for all; then
    // the state (multiblock.cpp:252-287) and the halo exchange.
    void fill(const std::vector<int32_t>& slot_of_cell, int32_t uniform_slot, const CaseSetup& setup);
    void set_dispatch(const std::set<int>& tags);
    void exchange();
    // kinetic_last: fuse the kinetic-energy values into the last step (single
    // slab; multi-slab runs reduce unfused)
    void advance(int64_t nsteps, bool kinetic_last = false);
    void synchronize();

    std::vector<double> gather_populations();
    void gather_macroscopic(std::vector<double>& rho, std::vector<double>& ux, std::vector<double>& uy,
                            std::vector<double>& uz);
    // raw storage-precision populations, canonical order (the DOLB1 payload)
    std::vector<uint8_t> gather_raw();
    void write_field_dump(const std::string& path);

    // diagnostics (diagnostics.cpp / runner.cpp semantics, bit-identical tree sums)
    double tree_reduce(int quantity, int64_t x_begin, int64_t x_end, int64_t* count_out);
    double kinetic_energy();
    double enstrophy();
    void snapshot_velocity();
    void convergence_sums(double* num, double* den);
    std::vector<double> porous_extras(int64_t sample_begin, int64_t sample_end, double nu, bool aperture_mean);

    int64_t num_cells() const { return dims_[0] * dims_[1] * dims_[2]; }
    int64_t steps_done() const { return steps_; }
    const std::array<int64_t, 3>& dims() const { return dims_; }
    int slabs() const { return int(slabs_.size()); }
    Lattice& slab(int k) { return *slabs_[std::size_t(k)]; }
    std::string kernel_name() const { return slabs_.front()->kernel_name(); }
    int64_t step_bytes() const;

  private:
    double tree_mean(int quantity, int64_t x_begin, int64_t x_end, const double* empty);
    std::array<int64_t, 3> dims_;
    std::array<bool, 3> periodic_;
    int q_, bits_;
    std::vector<std::pair<int64_t, int64_t>> parts_;  // (z0, nz) per slab
    std::vector<std::unique_ptr<Lattice>> slabs_;
    int64_t steps_ = 0;
};

}  // namespace dlb
