// mrlbm_internal.h — declarations shared by the host and device translation units.
#pragma once
#include "../../include/mrlbm_gpu.h"
#include <vector>

namespace mrlbm_b200 {

struct TableEntry {
    int off[2];
    double w;
};

// exactness sets of a table: bounding box of the level-l dependency cells (must
// be inside the domain) and parents of the level-(l+1) funnel (must not be internal)
struct TableSets {
    int dep_lo[2], dep_hi[2];
    std::vector<std::pair<int, int>> par;
};

// exact dyadic flattened table (push formulation), see host_configs.cpp
int build_stream_table(int d, int g, const int32_t* eta, int side, std::vector<TableEntry>& out,
                       TableSets* sets = nullptr);
// Gauss-Jordan with partial pivoting in the reference's elimination order
bool gauss_jordan_inverse(int n, const double* a, double* out);

} // namespace mrlbm_b200
