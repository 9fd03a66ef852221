// interp_tile.cuh -- the pieces of the Catmull-Rom interpolation of a coarse field onto a
// 32x30 fine tile (+1-cell halo) shared by q_half_apply (stochastic.cu: column strips) and
// the IEWPF pull (iewpf.cu: pull_tables / pull_apply): the tile geometry, the column /
// row group tables and the Catmull-Rom coefficients. Included only by --fmad=false
// translation units.
//
// interpolate_bicubic (stochastic.hpp:93-118) computes, per fine cell, four x-direction
// Catmull-Rom evaluations col[m] (one per coarse row bs[m]) and one y-direction
// evaluation. col[m] depends only on (fine column, coarse row), so pass 1 evaluates it
// once per (coarse row, fine column) of the tile into X, and pass 2 combines four rows of
// X per fine cell.
//
// catmull (stochastic.hpp:81-87) is 0.5*(a + t*(b + t*(c + t*d))) with a..d functions of
// the four points only. Consecutive fine columns (rows) with the same coarse cell a0 (b0)
// -- c_omega of them -- share the four points, so each pass evaluates a..d once per run
// ("group") and only the t-polynomial per fine column (row). Same operands, same order:
// bit-identical to the reference's per-cell evaluation.
#pragma once

#include "dc_internal.h"
#include "detmath.cuh"

namespace dcg {
namespace tile {

constexpr int TX = 32, TY = 30;    // output tile (TY+2 = 32 halo rows)
constexpr int NBMAX = TY + 2 + 3;  // coarse rows a tile can touch (c_omega = 1 worst case)
constexpr int XW = TX + 2;         // tile width incl. halo
constexpr int YH = TY + 2;         // tile height incl. halo (= 32: one lane per row)
#ifndef DC_TILE_NT
#define DC_TILE_NT 256
#endif
constexpr int NT = DC_TILE_NT;     // threads (a multiple of 32, >= 96)
constexpr int kWarps = NT / 32;    // warps; an add gives warp w rows w, w + kWarps, ..
constexpr int kRowsPerThread = (TY + kWarps - 1) / kWarps;

// the interpolation tables of one (tile, coarse alignment) as setup_cols / setup_rows
// build them (pull_tables_kernel compacts them into the pull's per-entry PullTab)
struct Tab {
    double ct[XW];           // x fraction per halo column
    double rt[YH];           // y fraction per halo row
    int cg_a[XW][4];         // per column group: coarse columns a0-1 .. a0+2 (mapped)
    int rg_sl[YH][4];        // per row group: X slots of coarse rows b0-1 .. b0+2
    int cg_first[XW + 1];    // first halo column of each column group (+ end sentinel)
    int rg_first[YH + 1];    // first halo row of each row group (+ end sentinel)
    int brow[NBMAX];         // coarse row of each X slot (mapped)
    int nb, ncg, nrg;
};
struct Cm {
    double a, b, c, d;
};

// the t-independent part of catmull (stochastic.hpp:82-85)
__device__ __forceinline__ Cm coef(double fm1, double f0, double f1, double f2) {
    Cm m;
    m.a = 2.0 * f0;
    m.b = f1 - fm1;
    m.c = 2.0 * fm1 - 5.0 * f0 + 4.0 * f1 - f2;
    m.d = -fm1 + 3.0 * f0 - 3.0 * f1 + f2;
    return m;
}
// stochastic.hpp:86
__device__ __forceinline__ double eval(const Cm& m, double t) {
    return 0.5 * (m.a + t * (m.b + t * (m.c + t * m.d)));
}

__device__ __forceinline__ void row_b0(const ErrParams& ep, int kk, int ok, int* b0, double* ty) {
    const double yc = static_cast<double>(kk - ok) * ep.inv_c;  // stochastic.hpp:98-100
    *b0 = static_cast<int>(floor(yc));
    *ty = yc - *b0;
}

__device__ __forceinline__ unsigned lanemask_le() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}

// Column tables of one tile (warp 0): depend only on the tile's columns and the coarse
// column offset, so a CTA that streams down a column strip builds them once. No barrier.
template <class TabT, class COLMAP>
__device__ __forceinline__ void setup_cols(TabT& S, const ErrParams& ep, int nx, int j0, int oj,
                                           COLMAP colmap) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {  // columns l and 32+l (l < 2) (stochastic.hpp:104-108)
        int a1, a2 = 0;
        double t1, t2 = 0.0;
        {
            const double xc = static_cast<double>(det::wrap1(j0 - 1 + lane, nx) - oj) * ep.inv_c;
            a1 = static_cast<int>(floor(xc));
            t1 = xc - a1;
        }
        if (lane < XW - 32) {
            const double xc =
                static_cast<double>(det::wrap1(j0 + 31 + lane, nx) - oj) * ep.inv_c;
            a2 = static_cast<int>(floor(xc));
            t2 = xc - a2;
        }
        const int up1 = __shfl_up_sync(0xffffffffu, a1, 1);
        const int last1 = __shfl_sync(0xffffffffu, a1, 31);
        const int first2 = __shfl_sync(0xffffffffu, a2, 0);
        const bool s1 = lane == 0 || a1 != up1;
        const bool s2 = lane < XW - 32 && a2 != (lane == 0 ? last1 : first2);
        const unsigned b1 = __ballot_sync(0xffffffffu, s1), b2 = __ballot_sync(0xffffffffu, s2);
        const unsigned le = lanemask_le();
        S.ct[lane] = t1;
        if (s1) {
            const int g = __popc(b1 & le) - 1;
            S.cg_first[g] = lane;
#pragma unroll
            for (int q = 0; q < 4; ++q) S.cg_a[g][q] = colmap(det::wrapf(a1 - 1 + q, ep.nxc));
        }
        if (lane < XW - 32) S.ct[32 + lane] = t2;
        if (s2) {
            const int g = __popc(b1) + __popc(b2 & le) - 1;
            S.cg_first[g] = 32 + lane;
#pragma unroll
            for (int q = 0; q < 4; ++q) S.cg_a[g][q] = colmap(det::wrapf(a2 - 1 + q, ep.nxc));
        }
        if (lane == 0) {
            const int n = __popc(b1) + __popc(b2);
            S.ncg = n;
            S.cg_first[n] = XW;
        }
    }
}

// Row tables of one tile (warps 1, 2). No barrier.
template <class ROWMAP>
__device__ __forceinline__ void setup_rows(Tab& S, const ErrParams& ep, int ny, int k0, int ok,
                                           ROWMAP rowmap) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool whole = ep.nyc <= NBMAX;
    if (warp == 1 || warp == 2) {
        int bfirst, blast;
        double td;
        row_b0(ep, det::wrap1(k0 - 1, ny), ok, &bfirst, &td);
        row_b0(ep, det::wrap1(k0 + TY, ny), ok, &blast, &td);
        const int bstart = whole ? 0 : det::wrapf(bfirst - 1, ep.nyc);
        const int nb = whole ? ep.nyc : det::wrapf(blast - bfirst, ep.nyc) + 4;
        if (warp == 1) {  // halo row = lane (stochastic.hpp:98-102)
            int b0;
            double t;
            row_b0(ep, det::wrap1(k0 - 1 + lane, ny), ok, &b0, &t);
            const int up = __shfl_up_sync(0xffffffffu, b0, 1);
            const bool s = lane == 0 || b0 != up;
            const unsigned bl = __ballot_sync(0xffffffffu, s);
            S.rt[lane] = t;
            if (s) {
                const int g = __popc(bl & lanemask_le()) - 1;
                S.rg_first[g] = lane;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int b = det::wrapf(b0 - 1 + q, ep.nyc);
                    S.rg_sl[g][q] = whole ? b : det::wrapf(b - bstart, ep.nyc);
                }
            }
            if (lane == 0) {
                const int n = __popc(bl);
                S.nrg = n;
                S.rg_first[n] = YH;
            }
        } else {
            for (int s = lane; s < nb; s += 32)
                S.brow[s] = rowmap(whole ? s : det::wrap1(bstart + s, ep.nyc));
            if (lane == 0) S.nb = nb;
        }
    }
}

} // namespace tile
} // namespace dcg
