// interp_tile.cuh -- Catmull-Rom interpolation of a coarse field onto one 32x30 fine tile
// (+1-cell halo) in shared memory, shared by q_half_apply (model error / posterior) and
// pull_apply (IEWPF pull). Included only by --fmad=false translation units.
//
// interpolate_bicubic (stochastic.hpp:93-118) computes, per fine cell, four x-direction
// Catmull-Rom evaluations col[m] (one per coarse row bs[m]) and one y-direction
// evaluation. col[m] depends only on (fine column, coarse row), so pass 1 evaluates it
// once per (coarse row, fine column) of the tile into X, and pass 2 combines four rows of
// X per fine cell -- the same operands in the same order, hence bit-identical results.
// The per-column / per-row index bookkeeping (floor, wrap, row slots) is done once per
// column / row into shared tables; the element loops are flat and evenly split.
#pragma once

#include "dc_internal.h"
#include "detmath.cuh"

namespace dcg {
namespace tile {

constexpr int TX = 32, TY = 30;    // output tile (TY+2 = 32 halo rows: 4 per thread row)
constexpr int NBMAX = TY + 2 + 3;  // coarse rows a tile can touch (c_omega = 1 worst case)
constexpr int XW = TX + 2;         // tile width incl. halo
constexpr int YH = TY + 2;         // tile height incl. halo
constexpr int NT = 256;            // threads

struct ColInfo {
    int a[4];  // coarse column indices a0-1 .. a0+2 (wrapped, then mapped)
    double t;  // x fraction
};
struct RowInfo {
    int sl[4];  // X slots of coarse rows b0-1 .. b0+2
    double t;   // y fraction
};

struct Smem {
    double X[NBMAX][XW];
    double D[YH][XW];
    ColInfo col[XW];
    RowInfo row[YH];
    int brow[NBMAX];  // coarse row of each X slot (mapped)
    int nb;
};

__device__ __forceinline__ void row_b0(const ErrParams& ep, int kk, int ok, int* b0, double* ty) {
    const double yc = static_cast<double>(kk - ok) * ep.inv_c;  // stochastic.hpp:98-100
    *b0 = static_cast<int>(floor(yc));
    *ty = yc - *b0;
}

// Tables for one (tile, coarse offset): COLMAP / ROWMAP turn wrapped coarse indices into
// whatever the value accessor expects. Ends with a barrier.
template <class COLMAP, class ROWMAP>
__device__ __forceinline__ void setup(Smem& S, const ErrParams& ep, int nx, int ny, int j0,
                                      int k0, int oj, int ok, COLMAP colmap, ROWMAP rowmap) {
    const int tid = threadIdx.x;
    int bfirst, blast;
    double td;
    row_b0(ep, det::wrap1(k0 - 1, ny), ok, &bfirst, &td);
    row_b0(ep, det::wrap1(k0 + TY, ny), ok, &blast, &td);
    const bool whole = ep.nyc <= NBMAX;
    const int bstart = whole ? 0 : det::wrapf(bfirst - 1, ep.nyc);
    const int nb = whole ? ep.nyc : det::wrapf(blast - bfirst, ep.nyc) + 4;
    if (tid < XW) {  // column tables (stochastic.hpp:104-108)
        const int jw = det::wrap1(j0 - 1 + tid, nx);
        const double xc = static_cast<double>(jw - oj) * ep.inv_c;
        const int a0 = static_cast<int>(floor(xc));
        ColInfo c;
        c.t = xc - a0;
#pragma unroll
        for (int q = 0; q < 4; ++q) c.a[q] = colmap(det::wrapf(a0 - 1 + q, ep.nxc));
        S.col[tid] = c;
    } else if (tid >= 64 && tid < 64 + YH) {  // row tables (stochastic.hpp:98-102)
        const int r = tid - 64;
        int b0;
        RowInfo ri;
        row_b0(ep, det::wrap1(k0 - 1 + r, ny), ok, &b0, &ri.t);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int b = det::wrapf(b0 - 1 + q, ep.nyc);
            ri.sl[q] = whole ? b : det::wrapf(b - bstart, ep.nyc);
        }
        S.row[r] = ri;
    } else if (tid >= 128 && tid < 128 + nb) {
        const int s = tid - 128;
        S.brow[s] = rowmap(whole ? s : det::wrap1(bstart + s, ep.nyc));
    }
    if (tid == 0) S.nb = nb;
    __syncthreads();
}

// Passes 1 and 2 into S.D. VALF(mapped row, mapped col) returns the coarse value.
// Ends with a barrier.
template <class VALF>
__device__ __forceinline__ void interpolate(Smem& S, VALF valf) {
    const int tid = threadIdx.x;
    const int n1 = S.nb * XW;
    for (int i = tid; i < n1; i += NT) {
        const int s = i / XW, jl = i - s * XW;
        const ColInfo& c = S.col[jl];
        const int b = S.brow[s];
        S.X[s][jl] = det::catmull(valf(b, c.a[0]), valf(b, c.a[1]), valf(b, c.a[2]),
                                  valf(b, c.a[3]), c.t);
    }
    __syncthreads();
    for (int i = tid; i < YH * XW; i += NT) {
        const int r = i / XW, jl = i - r * XW;
        const RowInfo& ri = S.row[r];
        S.D[r][jl] = det::catmull(S.X[ri.sl[0]][jl], S.X[ri.sl[1]][jl], S.X[ri.sl[2]][jl],
                                  S.X[ri.sl[3]][jl], ri.t);
    }
    __syncthreads();
}

} // namespace tile
} // namespace dcg
