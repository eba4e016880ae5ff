// Host-side log-singular product-integration weights (reference
// logquad.cpp:16-112); see logquad.cpp.
#pragma once

#include <vector>

#include "geometry.hpp"

namespace sbx {

// lambda_j(u), j < q, for a target at panel-local parameter u (cached by value).
const std::vector<double>& log_weights(int q, double u);
// q x q row-major table: row i = weights for the target at Gauss node i.
const std::vector<double>& log_self_table(int q);

// Single-layer tables of g for the components flagged in sl_comp (cached on g).
const SlTables& single_layer_tables(const Geom& g, const std::vector<char>& sl_comp, cudaStream_t s);

}  // namespace sbx
