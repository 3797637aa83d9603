// Host-side dynamics-chain model and registry.
//
// Same semantics (ids, composite names, validation, parameter records, tag
// order, error texts) as the reference's chain / registry layer:
//   LinkType / ChainLink / ChainParams .. proj/include/dolb/chain.hpp:14-53
//   link_id / parse / chain_string ..... proj/src/chain.cpp:38-119
//   validate_chain ..................... proj/src/chain.cpp:121-151
//   serialize / deserialize_params ..... proj/src/chain.cpp:153-230
//   DynamicsRegistry ................... proj/include/dolb/accelerated_lattice.hpp:32-60,
//                                        proj/src/accelerated_lattice.cpp:10-71
//   DispatchError ...................... accelerated_lattice.hpp:16-26
#pragma once

#include <array>
#include <cstdint>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

namespace dlb {

enum class LinkType {
    NoDynamics,
    BounceBack,
    MovingBounceBack,
    BGK,
    TRT,
    RR,
    Smagorinsky,
    RegularizedVelocity,
    RegularizedPressure,
};

struct ChainLink {
    LinkType type = LinkType::BGK;
    int axis = 0;
    int orient = 1;
    bool operator==(const ChainLink& o) const {
        return type == o.type && axis == o.axis && orient == o.orient;
    }
};

struct ChainParams {
    double omega = 1.0;
    double omega_minus = 1.0;
    double lambda = 3.0 / 16.0;
    double smagorinsky_c = 0.0;
    double omega_bulk_ho = 1.0;
    std::array<double, 3> wall_velocity = {0, 0, 0};
    double target_rho = 1.0;
};

struct DynamicsChain {
    std::vector<ChainLink> links;
    ChainParams params;
};

class DispatchError : public std::runtime_error {
  public:
    explicit DispatchError(const std::string& chain_name)
        : std::runtime_error("collision model \"" + chain_name +
                             "\" is not part of the dispatch set"),
          chain_name_(chain_name) {}
    const std::string& chain_name() const { return chain_name_; }

  private:
    std::string chain_name_;
};

class ExchangeError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

// CUDA / device-side failure (maps to DLB_ERROR_INTERNAL).
class DeviceError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

double derive_omega_minus(double omega, double lambda);

std::string link_id(const ChainLink& link);
ChainLink parse_link_id(const std::string& id);
std::string chain_string(const std::vector<ChainLink>& links);
std::vector<ChainLink> parse_chain_string(const std::string& s);
void validate_chain(const std::vector<ChainLink>& links);
std::vector<double> serialize_params(const DynamicsChain& chain);
ChainParams deserialize_params(const std::vector<ChainLink>& links, const double* data,
                               std::size_t len);

class DynamicsRegistry {
  public:
    struct Instance {
        std::string chain_str;
        std::vector<ChainLink> links;
        std::int64_t param_offset = 0;
        std::int64_t param_len = 0;
    };

    int register_chain(const DynamicsChain& chain);
    int tag_for(const std::string& chain_str) const;
    const std::string& chain_for(int tag) const;
    int tag_of_slot(int slot) const { return tag_for(instances_.at(std::size_t(slot)).chain_str); }
    DynamicsChain chain_at_slot(int slot) const;
    int num_instances() const { return int(instances_.size()); }
    int num_tags() const { return int(strings_.size()); }
    const std::vector<double>& params_table() const { return params_table_; }
    const Instance& instance(int slot) const { return instances_.at(std::size_t(slot)); }

  private:
    std::set<std::string> strings_;
    std::vector<Instance> instances_;
    std::vector<double> params_table_;
};

}  // namespace dlb
