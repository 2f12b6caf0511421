// host_model.h — host-side model helpers shared by the ABI translation units.
#pragma once

#include <cstdint>
#include <vector>

#include "wavegrid_b200.h"

namespace wg {

struct RunGeometry {
    uint32_t m = 1;         // components
    uint64_t splits[2] = {1, 1};
    uint64_t n[2] = {0, 0};  // logical points per patch side
    uint64_t npatch = 0;
    uint64_t tcount = 0;     // true cells per component (n+2)^2
    uint64_t tiles = 1;      // periodic copies along dim 0 (wg_run_config::tile_rows)
};

bool valid_signal_length(uint64_t n);
int signal_level(uint64_t n);
void plan_validate(const uint64_t* dims, uint32_t rank, int levels);
double band_threshold(const int* scales, uint32_t rank, int mode, double c, double alpha);
void threshold_table_2d(int levels, int mode, double c, double alpha, double* out);
uint32_t scheme_components(int scheme);
void sim_validate(const wg_run_config& c);
double sim_dx(const wg_run_config& c);
RunGeometry run_geometry(const wg_run_config& c);
std::vector<double> transport_dts(const wg_run_config& c);
double exact_transport_at(const wg_run_config& c, double t, uint64_t i, uint64_t j);
void initial_state(const wg_run_config& c, uint64_t row_begin, uint64_t row_end, double* buf);

}  // namespace wg
