// mrlbm_internal.h — declarations shared by the host and device translation units.
#pragma once
#include "../../include/mrlbm_gpu.h"
#include <vector>

namespace mrlbm_b200 {

struct TableEntry {
    int off[2];
    double w;
};

// exact dyadic flattened table (push formulation), see host_configs.cpp
int build_stream_table(int d, int g, const int32_t* eta, int side, std::vector<TableEntry>& out);
// Gauss-Jordan with partial pivoting in the reference's elimination order
bool gauss_jordan_inverse(int n, const double* a, double* out);

} // namespace mrlbm_b200
