// Host-side chain model + registry; behaviour pinned to the reference by
// tests/test_host_api.py (ids, composite names, tags, parameter records and
// error categories). See chain.hpp for the reference map.
#include "chain.hpp"

#include <algorithm>
#include <iterator>

namespace dlb {

namespace {

bool terminal(LinkType t) {
    switch (t) {
        case LinkType::NoDynamics:
        case LinkType::BounceBack:
        case LinkType::MovingBounceBack:
        case LinkType::BGK:
        case LinkType::TRT:
        case LinkType::RR:
            return true;
        default:
            return false;
    }
}

bool base_collision(LinkType t) {
    return t == LinkType::BGK || t == LinkType::TRT || t == LinkType::RR;
}

bool regularized(LinkType t) {
    return t == LinkType::RegularizedVelocity || t == LinkType::RegularizedPressure;
}

const char* short_base(LinkType t) {
    if (t == LinkType::BGK) return "BGK";
    if (t == LinkType::TRT) return "TRT";
    if (t == LinkType::RR) return "RR";
    throw std::invalid_argument("not a base collision link");
}

struct NamedLink {
    const char* id;
    LinkType type;
};

constexpr NamedLink kPlainLinks[] = {
    {"NoDynamics", LinkType::NoDynamics},     {"BounceBack", LinkType::BounceBack},
    {"MovingBounceBack", LinkType::MovingBounceBack}, {"COLL_BGK", LinkType::BGK},
    {"COLL_TRT", LinkType::TRT},              {"COLL_RR", LinkType::RR},
    {"LES_Smagorinsky", LinkType::Smagorinsky},
};

constexpr const char* kVelPrefix = "Boundary_RegularizedVelocity_";
constexpr const char* kPresPrefix = "Boundary_RegularizedPressure_";

}  // namespace

double derive_omega_minus(double omega, double lambda) {
    // Lambda = (1/omega - 1/2)(1/omega_minus - 1/2)   (collision.hpp:19-22)
    const double half_minus = lambda / (1.0 / omega - 0.5);
    return 1.0 / (half_minus + 0.5);
}

std::string link_id(const ChainLink& link) {
    for (const NamedLink& n : kPlainLinks)
        if (n.type == link.type) return n.id;
    if (regularized(link.type)) {
        const std::string prefix =
            link.type == LinkType::RegularizedVelocity ? kVelPrefix : kPresPrefix;
        return prefix + std::to_string(link.axis) + (link.orient > 0 ? "_1" : "_M1");
    }
    throw std::invalid_argument("unknown link type");
}

ChainLink parse_link_id(const std::string& id) {
    for (const NamedLink& n : kPlainLinks)
        if (id == n.id) return ChainLink{n.type, 0, 1};
    for (const char* prefix : {kVelPrefix, kPresPrefix}) {
        const std::string p(prefix);
        if (id.compare(0, p.size(), p) != 0) continue;
        // "<axis>_<1|M1>"
        const std::string tail = id.substr(p.size());
        if (tail.size() < 3 || tail[1] != '_' || tail[0] < '0' || tail[0] > '2') break;
        const std::string o = tail.substr(2);
        if (o != "1" && o != "M1") break;
        const LinkType t =
            prefix == kVelPrefix ? LinkType::RegularizedVelocity : LinkType::RegularizedPressure;
        return ChainLink{t, tail[0] - '0', o == "1" ? 1 : -1};
    }
    throw std::invalid_argument("unknown model identifier: \"" + id + "\"");
}

std::string chain_string(const std::vector<ChainLink>& links) {
    if (links.size() == 2 && regularized(links[0].type) && base_collision(links[1].type))
        return link_id(links[0]) + "__" + short_base(links[1].type);
    std::string out;
    for (std::size_t k = 0; k < links.size(); ++k) {
        if (k) out.push_back('|');
        out += link_id(links[k]);
    }
    return out;
}

std::vector<ChainLink> parse_chain_string(const std::string& s) {
    std::vector<ChainLink> links;
    const std::size_t cut = s.rfind("__");
    if (cut != std::string::npos && s.compare(0, 20, "Boundary_Regularized") == 0) {
        links.push_back(parse_link_id(s.substr(0, cut)));
        links.push_back(parse_link_id("COLL_" + s.substr(cut + 2)));
        return links;
    }
    std::size_t at = 0;
    for (;;) {
        const std::size_t bar = s.find('|', at);
        links.push_back(parse_link_id(s.substr(at, bar == std::string::npos ? std::string::npos
                                                                            : bar - at)));
        if (bar == std::string::npos) break;
        at = bar + 1;
    }
    return links;
}

void validate_chain(const std::vector<ChainLink>& links) {
    if (links.empty()) throw std::invalid_argument("dynamics chain must contain at least one link");
    int terminals = 0;
    for (std::size_t k = 0; k < links.size(); ++k) {
        if (terminal(links[k].type)) {
            ++terminals;
            if (k + 1 != links.size())
                throw std::invalid_argument("terminal link \"" + link_id(links[k]) +
                                            "\" must be the last link of the chain");
        }
        if (regularized(links[k].type) && links[k].orient != 1 && links[k].orient != -1)
            throw std::invalid_argument("regularized boundary orientation must be +1 or -1");
    }
    if (terminals != 1)
        throw std::invalid_argument("dynamics chain \"" + chain_string(links) +
                                    "\" needs exactly one terminal link");
    const bool collides = base_collision(links.back().type);
    for (std::size_t k = 0; k + 1 < links.size(); ++k) {
        const LinkType t = links[k].type;
        if ((regularized(t) || t == LinkType::Smagorinsky) && !collides)
            throw std::invalid_argument("link \"" + link_id(links[k]) +
                                        "\" requires a base collision terminal");
    }
}

// Record layout: each link appends the values it consumes, in chain order.
std::vector<double> serialize_params(const DynamicsChain& chain) {
    std::vector<double> rec;
    const ChainParams& p = chain.params;
    for (const ChainLink& l : chain.links) {
        switch (l.type) {
            case LinkType::BGK: rec.push_back(p.omega); break;
            case LinkType::TRT: rec.insert(rec.end(), {p.omega, p.lambda}); break;
            case LinkType::RR: rec.insert(rec.end(), {p.omega, p.omega_bulk_ho}); break;
            case LinkType::Smagorinsky: rec.push_back(p.smagorinsky_c); break;
            case LinkType::MovingBounceBack:
            case LinkType::RegularizedVelocity:
                rec.insert(rec.end(), p.wall_velocity.begin(), p.wall_velocity.end());
                break;
            case LinkType::RegularizedPressure: rec.push_back(p.target_rho); break;
            case LinkType::NoDynamics:
            case LinkType::BounceBack: break;
        }
    }
    return rec;
}

ChainParams deserialize_params(const std::vector<ChainLink>& links, const double* data,
                               std::size_t len) {
    ChainParams p;
    std::size_t k = 0;
    auto take = [&]() -> double {
        if (k >= len) throw std::invalid_argument("parameter record too short for chain");
        return data[k++];
    };
    for (const ChainLink& l : links) {
        switch (l.type) {
            case LinkType::BGK: p.omega = take(); break;
            case LinkType::TRT:
                p.omega = take();
                p.lambda = take();
                p.omega_minus = derive_omega_minus(p.omega, p.lambda);
                break;
            case LinkType::RR:
                p.omega = take();
                p.omega_bulk_ho = take();
                break;
            case LinkType::Smagorinsky: p.smagorinsky_c = take(); break;
            case LinkType::MovingBounceBack:
            case LinkType::RegularizedVelocity:
                for (double& v : p.wall_velocity) v = take();
                break;
            case LinkType::RegularizedPressure: p.target_rho = take(); break;
            case LinkType::NoDynamics:
            case LinkType::BounceBack: break;
        }
    }
    if (k != len) throw std::invalid_argument("parameter record too long for chain");
    return p;
}

int DynamicsRegistry::register_chain(const DynamicsChain& chain) {
    validate_chain(chain.links);
    const bool has_base = std::any_of(chain.links.begin(), chain.links.end(),
                                      [](const ChainLink& l) { return base_collision(l.type); });
    if (has_base) {
        const double om = chain.params.omega;
        if (!(om > 0.0 && om < 2.0))
            throw std::invalid_argument("relaxation rate " + std::to_string(om) +
                                        " outside the stable range (0, 2)");
    }
    const std::string name = chain_string(chain.links);
    const std::vector<double> rec = serialize_params(chain);
    for (std::size_t slot = 0; slot < instances_.size(); ++slot) {
        const Instance& in = instances_[slot];
        if (in.chain_str == name && in.param_len == std::int64_t(rec.size()) &&
            std::equal(rec.begin(), rec.end(), params_table_.begin() + in.param_offset))
            return int(slot);
    }
    strings_.insert(name);
    Instance in;
    in.chain_str = name;
    in.links = chain.links;
    in.param_offset = rec.empty() ? 0 : std::int64_t(params_table_.size());
    in.param_len = std::int64_t(rec.size());
    params_table_.insert(params_table_.end(), rec.begin(), rec.end());
    instances_.push_back(std::move(in));
    return int(instances_.size()) - 1;
}

int DynamicsRegistry::tag_for(const std::string& chain_str) const {
    const auto it = strings_.find(chain_str);
    if (it == strings_.end())
        throw std::invalid_argument("chain \"" + chain_str + "\" is not registered");
    return int(std::distance(strings_.begin(), it));
}

const std::string& DynamicsRegistry::chain_for(int tag) const {
    if (tag < 0 || tag >= int(strings_.size()))
        throw std::out_of_range("tag " + std::to_string(tag) + " is not registered");
    return *std::next(strings_.begin(), tag);
}

DynamicsChain DynamicsRegistry::chain_at_slot(int slot) const {
    const Instance& in = instances_.at(std::size_t(slot));
    DynamicsChain c;
    c.links = in.links;
    c.params = deserialize_params(in.links, params_table_.data() + in.param_offset,
                                  std::size_t(in.param_len));
    return c;
}

}  // namespace dlb
