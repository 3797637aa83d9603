// Deterministic tree reductions split across segments (host side).
//
// diag::tree_sum (proj/src/diagnostics.cpp:10-18) sums <= 8 values
// sequentially from 0.0 and otherwise returns tree(first n/2) + tree(rest).
// A segment [a, b) of the global sequence (one slab, one device chunk) owns
// the maximal tree nodes that lie inside it; a leaf cut by a segment boundary
// cannot be split, so its values inside the segment are shipped raw (len 0).
// tree_combine re-evaluates the nodes above the parts, giving the same bits
// as tree_sum over the whole sequence.
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/dlb.h"

namespace dlb {

// Parts of segment [a, b) of the tree over [lo, lo + n) (values left 0).
void tree_plan(int64_t lo, int64_t n, int64_t a, int64_t b, std::vector<dlb_tree_part>& out);
// tree_sum of the n_total-value sequence from the parts of all segments.
double tree_combine(int64_t n_total, const dlb_tree_part* parts, std::size_t n);
// diag::tree_sum of a host array.
double tree_sum_host(const double* v, int64_t n);

}  // namespace dlb
