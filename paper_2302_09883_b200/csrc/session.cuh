// session.cuh — device data layout of the compressed patch store.
//
// HBM layout (per shard):
//   store[2]   byte pools, double-buffered (read step k-1, write step k).
//              One block per (patch, component): CSR exactly as the
//              reference's CsrBlock (codec.hpp:24-34) — v[nnz] f64,
//              col[nnz] u32, row[n+1] u32, 16-byte aligned — or, for a raw
//              patch (skip rule, pipeline.hpp:243-249; initial state),
//              the n*n dense logical block.
//   dir[2]     DirEntry per (patch, component): byte offset, nnz, flags.
//   edges[2]   reconstructed boundary lines of every patch (logical rows 1
//              and n-2, columns 1 and n-2): the ghost-ring source of the
//              next step (sync_ghosts, patchgrid.hpp:131-201).  Row lines
//              have R+2 patch-row slots: slot 0 and R+1 are the halo rows
//              received from the neighbouring shards (multi-GPU).
//   partials   per-CTA metric sums of a step, reduced by the last CTA into
//              the step's metrics row.
#pragma once

#include <cstdint>

namespace wg {

constexpr uint32_t DIR_RAW = 1u;
constexpr uint32_t DIR_DEAD = 2u;   // block lost to a store overflow: decodes as zeros, error raised
constexpr uint32_t DIR_CONST = 4u;  // a raw block whose n*n values are bitwise equal: off holds the
                                    // value's bits, nothing in the pool (SWE's flat regions)

struct DirEntry {
    uint64_t off;    // byte offset in the pool
    uint32_t nnz;    // CSR entries (0 for raw)
    uint32_t flags;  // DIR_RAW / DIR_DEAD / DIR_CONST (with DIR_RAW)
};

struct EdgeSet {
    double* rowlo;  // [(R+2) slots][P1][m][n]: logical row 1
    double* rowhi;  // [(R+2) slots][P1][m][n]: logical row n-2
    double* collo;  // [R][P1][m][n]: logical column 1
    double* colhi;  // [R][P1][m][n]: logical column n-2
    // peer halo mode (multi-GPU, opt-in): the ring neighbours' halo slots of
    // the same buffer parity, mapped into this process (NVLink P2P / IPC).
    // The line of owned slot 1 (rowlo) is also stored into peer_lo = the
    // above neighbour's rowlo slot R_above + 1; the line of owned slot R
    // (rowhi) into peer_hi = the below neighbour's rowhi slot 0.  Null: the
    // halo blocks are exchanged by the host (NCCL) instead.
    double* peer_lo;
    double* peer_hi;
};

struct ShardGeom {
    uint32_t R;       // owned patch rows
    uint32_t P1;      // patches per row
    uint32_t m;       // components
    int world;        // 1: periodic wrap is local
    uint32_t npatch;  // R * P1
    uint32_t me;      // components stored per edge line (D2Q9: the 3 crossing that side)
    uint32_t row0;    // global index of the first owned patch row
};

// D2Q9 edge lines carry only the populations a neighbour pulls across that
// side (pull streaming f_q(x) <- f_q(x - c_q) reads ghost row 0 only for
// c_x = +1, row N+1 for c_x = -1, column 0 for c_y = +1, column N+1 for
// c_y = -1).  Slot of population q in each line, -1 if not stored.
//   rowlo (logical row 1, read as the upper neighbour's ghost row N+1): q in {2,6,8}
//   rowhi (logical row n-2, the lower neighbour's ghost row 0):         q in {1,5,7}
//   collo (logical column 1, the left neighbour's ghost column N+1):    q in {4,6,7}
//   colhi (logical column n-2, the right neighbour's ghost column 0):   q in {3,5,8}
__host__ __device__ constexpr int lbm_slot_rowlo(int q) { return q == 2 ? 0 : q == 6 ? 1 : q == 8 ? 2 : -1; }
__host__ __device__ constexpr int lbm_slot_rowhi(int q) { return q == 1 ? 0 : q == 5 ? 1 : q == 7 ? 2 : -1; }
__host__ __device__ constexpr int lbm_slot_collo(int q) { return q == 4 ? 0 : q == 6 ? 1 : q == 7 ? 2 : -1; }
__host__ __device__ constexpr int lbm_slot_colhi(int q) { return q == 3 ? 0 : q == 5 ? 1 : q == 8 ? 2 : -1; }

__host__ __device__ inline uint64_t round16(uint64_t b) { return (b + 15) & ~uint64_t(15); }

// Row slot of local patch row a' in [-1, R] (halo rows for world > 1; the
// periodic wrap for world == 1, patchgrid.hpp:143-161).
__device__ __forceinline__ uint32_t row_slot(int a, const ShardGeom& g) {
    if (g.world == 1) {
        const int R = (int)g.R;
        a = (a + R) % R;
    }
    return (uint32_t)(a + 1);
}

}  // namespace wg
