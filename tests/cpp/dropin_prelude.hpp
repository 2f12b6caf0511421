// dropin_prelude.hpp — force-included (g++ -include) in front of each of the
// reference's own test files (proj/tests/*.cpp), so that the unchanged test
// sources call the DROP-IN for every function it replaces
// (include/wavegrid_b200_reference.hpp) instead of the reference's CPU code.
// TEST INFRASTRUCTURE (tests/cpp/Makefile).
//
// How: while the reference headers are parsed, each replaced name is a
// function-like macro, so the reference's own definition and its internal
// callers become wavegrid::ref_cpu_<name> (a function-like macro never
// touches a member or a string of the same name, e.g. MetricsRow::
// global_mass).  The macros are then removed and the drop-in's
// wavegrid::b200::<name> is declared as wavegrid::<name>: the tests' `using
// namespace wavegrid;` and unqualified calls (dwt_nd(f, plan), run(cfg), ...)
// resolve to the drop-in, i.e. to the C ABI of the linked implementation —
// the sm_100a product on the GPU box, the C oracle on CPU.
//
// Routed: dwt_nd, idwt_nd, band_threshold, apply_threshold, csr_encode,
// csr_decode, lz_encode, lz_decode, sync_ghosts, global_mass, run, sweep
// (its runs through the drop-in's run).  Not routed: the per-patch fv_step template (the drop-in's fv_step is per grid) and the reference's
// non-path helpers (decompose, fill, assemble, lz_*, file formats).
#pragma once

// every standard header the reference headers include, before the macros
#include <algorithm>
#include <array>
#include <atomic>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <filesystem>
#include <fstream>
#include <functional>
#include <limits>
#include <memory>
#include <numbers>
#include <numeric>
#include <ostream>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#define dwt_nd(...) ref_cpu_dwt_nd(__VA_ARGS__)
#define idwt_nd(...) ref_cpu_idwt_nd(__VA_ARGS__)
#define band_threshold(...) ref_cpu_band_threshold(__VA_ARGS__)
#define apply_threshold(...) ref_cpu_apply_threshold(__VA_ARGS__)
#define csr_encode(...) ref_cpu_csr_encode(__VA_ARGS__)
#define csr_decode(...) ref_cpu_csr_decode(__VA_ARGS__)
#define sync_ghosts(...) ref_cpu_sync_ghosts(__VA_ARGS__)
#define global_mass(...) ref_cpu_global_mass(__VA_ARGS__)
#define run(...) ref_cpu_run(__VA_ARGS__)
#define sweep(...) ref_cpu_sweep(__VA_ARGS__)
#define lz_encode(...) ref_cpu_lz_encode(__VA_ARGS__)
#define lz_decode(...) ref_cpu_lz_decode(__VA_ARGS__)

#include "wavegrid/codec.hpp"
#include "wavegrid/field.hpp"
#include "wavegrid/patchgrid.hpp"
#include "wavegrid/pipeline.hpp"
#include "wavegrid/solver.hpp"
#include "wavegrid/threshold.hpp"
#include "wavegrid/wavelet.hpp"

#undef dwt_nd
#undef idwt_nd
#undef band_threshold
#undef apply_threshold
#undef csr_encode
#undef csr_decode
#undef sync_ghosts
#undef global_mass
#undef run
#undef sweep
#undef lz_encode
#undef lz_decode

#include "wavegrid_b200_reference.hpp"

namespace wavegrid {
using b200::apply_threshold;
using b200::band_threshold;
using b200::csr_decode;
using b200::csr_encode;
using b200::dwt_nd;
using b200::global_mass;
using b200::idwt_nd;
using b200::lz_decode;
using b200::lz_encode;
using b200::run;
using b200::sweep;
using b200::sync_ghosts;
}  // namespace wavegrid
