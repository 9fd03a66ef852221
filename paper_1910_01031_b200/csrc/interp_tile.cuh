// interp_tile.cuh -- Catmull-Rom interpolation of a coarse field onto one 32x16 fine tile
// (+1-cell halo) in shared memory, shared by q_half_apply (model error / posterior) and
// pull_apply (IEWPF pull). Included only by --fmad=false translation units.
//
// interpolate_bicubic (stochastic.hpp:93-118) computes, per fine cell, four x-direction
// Catmull-Rom evaluations col[m] (one per coarse row bs[m]) and one y-direction
// evaluation. col[m] depends only on (fine column, coarse row), so pass 1 evaluates it
// once per (coarse row, fine column) of the tile into X, and pass 2 combines four rows of
// X per fine cell -- the same operands in the same order, hence bit-identical results.
// All per-column / per-row index bookkeeping (floor, wrap, slots) is done once per
// thread-owned column/row, not per element.
#pragma once

#include "dc_internal.h"
#include "detmath.cuh"

namespace dcg {
namespace tile {

constexpr int TX = 32, TY = 16;
constexpr int NBMAX = TY + 2 + 3;  // coarse rows a tile can touch (c_omega = 1 worst case)
constexpr int XW = TX + 2;         // tile width incl. halo

// Thread layout: 256 threads = 32 (x) x 8 (y). Thread tx owns halo columns jl = tx and,
// for tx < 2, jl = tx + 32; thread ty owns rows ty, ty+8, ty+16 (< TY+2).
struct Col {
    int a[4];   // wrapped coarse column indices a0-1 .. a0+2
    double t;   // x fraction
};

__device__ __forceinline__ void col_setup(const ErrParams& ep, int nx, int j0, int oj, int jl,
                                          Col& c) {
    const int jw = det::wrap1(j0 - 1 + jl, nx);
    const double xc = static_cast<double>(jw - oj) * ep.inv_c;  // stochastic.hpp:104-106
    const int a0 = static_cast<int>(floor(xc));
    c.t = xc - a0;
#pragma unroll
    for (int q = 0; q < 4; ++q) c.a[q] = det::wrapf(a0 - 1 + q, ep.nxc);
}

// coarse-row window of a tile: X row s holds coarse row b(s)
struct Rows {
    bool whole;
    int bstart, nb;
};

__device__ __forceinline__ void row_b0(const ErrParams& ep, int kk, int ok, int* b0, double* ty) {
    const double yc = static_cast<double>(kk - ok) * ep.inv_c;  // stochastic.hpp:98-100
    *b0 = static_cast<int>(floor(yc));
    *ty = yc - *b0;
}

__device__ __forceinline__ Rows rows_setup(const ErrParams& ep, int ny, int k0, int ok) {
    int bfirst, blast;
    double td;
    row_b0(ep, det::wrap1(k0 - 1, ny), ok, &bfirst, &td);
    row_b0(ep, det::wrap1(k0 + TY, ny), ok, &blast, &td);
    Rows R;
    R.whole = ep.nyc <= NBMAX;
    R.bstart = R.whole ? 0 : det::wrapf(bfirst - 1, ep.nyc);
    R.nb = R.whole ? ep.nyc : det::wrapf(blast - bfirst, ep.nyc) + 4;
    return R;
}

__device__ __forceinline__ int row_of_slot(const ErrParams& ep, const Rows& R, int s) {
    return R.whole ? s : det::wrap1(R.bstart + s, ep.nyc);
}

// Interpolate into D[TY+2][XW]. COARSE(a, b) returns the coarse value at wrapped (a, b).
// ROWVAL(b) precomputes a per-coarse-row handle consumed by COLVAL(handle, a).
// COLMAP maps a wrapped coarse column index to the index VALF expects (once per column).
template <class RowH, class ROWF, class VALF, class COLMAP>
__device__ __forceinline__ void interpolate(const ErrParams& ep, int nx, int ny, int j0, int k0,
                                            int oj, int ok, ROWF rowf, VALF valf, COLMAP colmap,
                                            double (*X)[XW], double (*D)[XW]) {
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    Col c0;
    col_setup(ep, nx, j0, oj, tx, c0);
    Col c1 = c0;
    const bool has1 = tx < XW - 32;
    if (has1) col_setup(ep, nx, j0, oj, tx + 32, c1);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        c0.a[q] = colmap(c0.a[q]);
        c1.a[q] = colmap(c1.a[q]);
    }
    const Rows R = rows_setup(ep, ny, k0, ok);
    // pass 1: X[s][jl] = catmull over the coarse row b(s) at column jl
    for (int s = ty; s < R.nb; s += 8) {
        const RowH h = rowf(row_of_slot(ep, R, s));
        X[s][tx] = det::catmull(valf(h, c0.a[0]), valf(h, c0.a[1]), valf(h, c0.a[2]),
                                valf(h, c0.a[3]), c0.t);
        if (has1)
            X[s][tx + 32] = det::catmull(valf(h, c1.a[0]), valf(h, c1.a[1]), valf(h, c1.a[2]),
                                         valf(h, c1.a[3]), c1.t);
    }
    __syncthreads();
    // pass 2: D[r][jl] = catmull over four X rows (stochastic.hpp:114)
    for (int r = ty; r < TY + 2; r += 8) {
        const int kk = det::wrap1(k0 - 1 + r, ny);
        int b0;
        double t;
        row_b0(ep, kk, ok, &b0, &t);
        int sl[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int b = det::wrapf(b0 - 1 + q, ep.nyc);
            sl[q] = R.whole ? b : det::wrapf(b - R.bstart, ep.nyc);
        }
        D[r][tx] = det::catmull(X[sl[0]][tx], X[sl[1]][tx], X[sl[2]][tx], X[sl[3]][tx], t);
        if (has1)
            D[r][tx + 32] = det::catmull(X[sl[0]][tx + 32], X[sl[1]][tx + 32], X[sl[2]][tx + 32],
                                         X[sl[3]][tx + 32], t);
    }
    __syncthreads();
}

} // namespace tile
} // namespace dcg
