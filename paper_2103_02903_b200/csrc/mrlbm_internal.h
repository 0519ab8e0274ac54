// mrlbm_internal.h — declarations shared by the host and device translation units.
#pragma once
#include "../../include/mrlbm_gpu.h"
#include <array>
#include <string>
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

// ---- 3D (D3Q6 path): flattened table of one (gap, velocity, side) ----
struct TableEntry3 {
    int off[3];
    double w;
};
struct TableSets3 {
    int dep_lo[3], dep_hi[3];            // bounding box of the level-l dependency cells
    std::vector<std::array<int, 3>> par; // parents (level l) of the touched level-(l+1) cells
};
int build_stream_table3(int g, const int32_t* eta, int side, std::vector<TableEntry3>& out, TableSets3* sets);

// 3D engine (mrlbm_step3d.cu), reached through the mrlbm_* entry points when scheme.d == 3
struct Engine3D;
int e3_create(const mrlbm_scheme_spec* sc, const mrlbm_run_config* rc, Engine3D** out, std::string& err);
int e3_load_leaves(Engine3D* e, int level, int64_t n, const int32_t* idx, const double* f);
int e3_commit(Engine3D* e);
int e3_step(Engine3D* e, int nsteps, mrlbm_step_stats* stats);
int e3_level_count(Engine3D* e, int level, int64_t* n);
int e3_read_leaves(Engine3D* e, int level, int32_t* idx, double* f);
int e3_tie_log(Engine3D* e, mrlbm_tie_record* out, int cap, int64_t* n, int reset);
int e3_finest_count(const Engine3D* e, int64_t* n);
void* e3_stream(Engine3D* e);
int e3_synchronize(Engine3D* e);
const char* e3_last_error(const Engine3D* e);
void e3_destroy(Engine3D* e);

} // namespace mrlbm_b200
