// Host side of the split tree reductions (see tree.hpp). Compiled without FMA
// contraction: every addition is the reference's double addition.
#include "tree.hpp"

#include <stdexcept>
#include <string>
#include <unordered_map>

namespace dlb {

void tree_plan(int64_t lo, int64_t n, int64_t a, int64_t b, std::vector<dlb_tree_part>& out) {
    if (n <= 0 || lo >= b || lo + n <= a) return;
    if (a <= lo && lo + n <= b) {
        out.push_back({lo, n, 0.0});
        return;
    }
    if (n <= 8) {  // a leaf cut by the segment: its values go out raw
        const int64_t j0 = lo > a ? lo : a, j1 = lo + n < b ? lo + n : b;
        for (int64_t j = j0; j < j1; ++j) out.push_back({j, 0, 0.0});
        return;
    }
    const int64_t h = n / 2;
    tree_plan(lo, h, a, b, out);
    tree_plan(lo + h, n - h, a, b, out);
}

namespace {

struct Combiner {
    std::unordered_map<int64_t, std::vector<std::pair<int64_t, double>>> nodes;  // lo -> (len, sum)
    std::unordered_map<int64_t, double> raw;

    bool node(int64_t lo, int64_t n, double& v) const {
        auto it = nodes.find(lo);
        if (it == nodes.end()) return false;
        for (const auto& [len, s] : it->second) {
            if (len == n) {
                v = s;
                return true;
            }
        }
        return false;
    }

    double eval(int64_t lo, int64_t n) const {
        double v;
        if (node(lo, n, v)) return v;
        if (n <= 8) {
            double s = 0.0;
            for (int64_t j = lo; j < lo + n; ++j) {
                auto it = raw.find(j);
                if (it == raw.end())
                    throw std::invalid_argument("tree_combine: no part covers value " + std::to_string(j));
                s += it->second;
            }
            return s;
        }
        const int64_t h = n / 2;
        return eval(lo, h) + eval(lo + h, n - h);
    }
};

}  // namespace

double tree_combine(int64_t n_total, const dlb_tree_part* parts, std::size_t n) {
    if (n_total < 0) throw std::invalid_argument("tree_combine: negative length");
    Combiner c;
    for (std::size_t k = 0; k < n; ++k) {
        if (parts[k].len > 0) c.nodes[parts[k].lo].push_back({parts[k].len, parts[k].value});
        else c.raw[parts[k].lo] = parts[k].value;
    }
    return c.eval(0, n_total);
}

double tree_sum_host(const double* v, int64_t n) {
    if (n <= 8) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) s += v[j];
        return s;
    }
    const int64_t h = n / 2;
    return tree_sum_host(v, h) + tree_sum_host(v + h, n - h);
}

}  // namespace dlb
