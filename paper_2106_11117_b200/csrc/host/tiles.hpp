// Spatial tiling of R for the temporally blocked LF-LTS step (config 3 and
// any box level whose R does not fit one SM).
//
// One global step of the reference's lts_step (src/integrators.cpp:117-157)
// on the rows of R needs, for an owned set O of R rows, d_p on O only; d_p
// depends on d_{p-1} on the P-neighbours of O, ..., d_1 = -c0 A z_n on the
// rows within p - 1 hops, and z_n one hop further.  A tile therefore owns a
// rectangle of the refined-square lattice (plus the R rows outside the box
// closest to it) and computes all p substeps on the rectangle grown by a
// halo, keeping every intermediate on chip; values near the halo's outer
// edge are wrong (their neighbours are missing) but the error travels one
// hop per substep and never reaches O.  The planner checks exactly that on
// the level's graph: every "source" of a wrong value (a lattice position
// whose stencil leaves the rectangle, a generic row with a P-column outside
// the tile) must be at least p hops from every owned row.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "level.hpp"

namespace wmc {

struct TilePlan {
    bool ok = false;
    std::string reason;
    // region geometry (fixed per plan): Wz x Hz box positions, thread = 2
    // columns x K rows; local slot of region column c, row r:
    //   colpos(c) * kTileHs + r + 1, colpos(c) = c even ? c/2 + 1 : Wz/2 + 2 + c/2
    // (even and odd columns apart, guard columns 0, Wz/2 + 1, Wz + 2; guard
    // rows 0 and Hz + 1), generic rows outside the box at kTileBoxSlots + k
    // shapes: 0 wide (wz columns x hz rows), 1 tall (hz columns x wz rows),
    // 2 square (sqrt(wz hz) each way: the box corners of the thin-frame layout)
    int wz = 0, hz = 0, k = 0;
    int hs = 0;          // column stride of the wide shape (odd); the tall one uses (wz + 2) | 1
    int jres = 0;        // region row origins are = jres (mod k)
    std::string notes;   // why the layouts tried before this one failed
    std::string layout;  // "grid" or "frame"
    int box_slots = 0;   // slots of the region rectangle incl. guards
    int max_gen = 0;     // generic rows per tile (<= threads)
    int max_app = 0;     // appended (outside-rectangle) slots per tile
    int max_ent = 0;     // generic SELL entries per tile
    int n_tiles = 0;
    // per tile
    std::vector<int> tiles_shape;       // 0 wide, 1 tall, 2 square
    std::vector<int> i0, j0;            // region origin (box coordinates, may be < 0)
    std::vector<int> oi0, oi1, oj0, oj1;  // owned rectangle [oi0, oi1) x [oj0, oj1) (box coordinates)
    std::vector<int> gen_off;           // generic rows of tile t: [gen_off[t], gen_off[t+1])
    // per tile and thread (threads = wide / 2 * narrow / k): the thread's
    // first column ia, first row jr0, lattice mask | owned mask << 16 (bit
    // r: column ia row jr0 + r, bit k + r: column ia + 1), see the kernel
    std::vector<int> thr_geo;           // [tile][thread][4]
    // per generic row
    std::vector<int> g_slot, g_dof, g_owned, g_ent_off, g_rem_off;  // ent / rem offsets: [off[r], off[r+1])
    std::vector<double> g_rs;
    // per generic SELL entry (P columns): local slot of the column, and the
    // weight recipe w = sum_t c[cell_t] a0_t (a0 already times sqrt(M_col))
    std::vector<int> e_slot, e_rc_off;
    std::vector<int> rc_cell;
    std::vector<double> rc_a0;
    // per remainder entry (columns outside P: z_n read from HBM): dof and
    // recipe A_ij = sum_t c[cell_t] a0_t
    std::vector<int> r_dof, r_rc_off;
    std::vector<int> rr_cell;
    std::vector<double> rr_a0;
    // line rows: box rows j in [1, m-1] starting a new coefficient row; a
    // strip starting on one takes separate first-row conductances
    std::vector<std::uint8_t> line_row;  // per box row
    double work_factor = 0.0;           // region positions per owned lattice node (diagnostics)
    // streamed interior (stream_step_kernel): slabs of at most `slab_rows`
    // box rows swept along the columns; region (I0, NX, J0, NY) and owned
    // region columns [x0, x1), rows [y0, y1); tiles own the rest of the box
    int slab_rows = 0, n_slabs = 0, max_nx = 0;
    int slab_threads = 0;       // rows of the tallest slab region rounded up to a warp (the kernel's CTA size)
    std::vector<int> slab;      // [slab][4]
    std::vector<int> slab_own;  // [slab][4]
};

// Plans the tiling for a box level (t.box) with the fixed kernel shape
// (region wz x hz, K rows per strip).  ok = false (with reason) when the
// level does not qualify or a tile fails the halo check.
// slab_rows > 0 (the stream kernel's rows per slab, p <= stream_max_p):
// frame layouts hand the interior to streamed slabs.
TilePlan plan_tiles(const LevelTables& t, int wide, int narrow, int k, int slab_rows = 0, int stream_max_p = 0);

}  // namespace wmc
