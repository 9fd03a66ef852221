// iewpf.cu -- observation operators, drifter advection and the two-stage IEWPF analysis
// on sm_100a (compiled --fmad=false: fp64 expressions follow the restated order exactly).
//
// Stage map, all particles at once:
//   obs_locate      locate_cell of every observation (grid.hpp:55-69), bit-exact fp64
//   innovations     d = y(H+eta)/H - (hu,hv), S d, phi = sum_o d^T S d in id order, c = phi + log N_e
//   pull_windows    per (particle, obs): SOAR(SOAR(GB^T dipole(S d))) on the obs-aligned
//                   coarse grid, kept as an 11x11 window (stochastic.hpp:178-202, 49-69)
//   tile_lists      per 32x16 fine tile: the observations whose pull footprint covers it
//   pull_apply      per (particle, tile): for each covering obs in ascending id, Catmull-Rom
//                   interpolation + geostrophic balance + float-rounded add -- a GATHER
//                   that reproduces the sequential per-observation add_q_half exactly
//                   (each cell sees the same ordered sequence of roundings), atomic-free
//   perp_pair       xi, nu~ (Philox, filter stream), three fixed-order dot products,
//                   in-place nu transform, gamma, zeta
//   barrier_alpha   w_target = mean c, beta = min((w-c)/zeta + 1) in particle-id order,
//                   c*, alpha by Lambert-W Halley iteration
//   local_blocks    z = beta^1/2 nu + alpha^1/2 xi; 7x7 coarse blocks <- U Sigma^1/2 block,
//                   ascending obs id
// then coarse_soar + q_half_apply (stochastic.cu) add P^{1/2} z to the pulled state.
#include <cuda_runtime.h>
#include <cstdint>

#include "dc_internal.h"
#include "detmath.cuh"
#include "iewpf_kernels.h"
#include "interp_tile.cuh"
#include "tma.cuh"

namespace dcg {

namespace {

using det::wrap1;
using det::wrapf;
using det::wrapi;

using tile::TX;
using tile::TY;
constexpr int WIN = 11;   // pull window: coarse offsets -5..5
constexpr int WH = 5;

// locate_cell (grid.hpp:55-69)
__device__ __forceinline__ bool locate(const SweParams& sp, double x, double y, int* j, int* k) {
    if (!isfinite(x) || !isfinite(y)) return false;
    const double lx = sp.nx * sp.dx, ly = sp.ny * sp.dy;
    double xm = fmod(x, lx);
    if (xm < 0.0) xm += lx;
    double ym = fmod(y, ly);
    if (ym < 0.0) ym += ly;
    int jj = static_cast<int>(floor(xm / sp.dx));
    int kk = static_cast<int>(floor(ym / sp.dy));
    if (jj >= sp.nx) jj = 0;
    if (kk >= sp.ny) kk = 0;
    *j = jj;
    *k = kk;
    return true;
}

__global__ void obs_locate_kernel(SweParams sp, const double* __restrict__ obs, int n_obs,
                                  int* cells, int* bad) {
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < n_obs; o += gridDim.x * blockDim.x) {
        int j = 0, k = 0;
        if (!locate(sp, obs[4 * o], obs[4 * o + 1], &j, &k)) atomicExch(bad, 1);
        cells[2 * o] = j;
        cells[2 * o + 1] = k;
    }
}

// stage 1 + phi/c: one CTA per particle
__global__ void innovations_kernel(SweParams sp, const float* __restrict__ eta,
                                   const float* __restrict__ hu, const float* __restrict__ hv,
                                   const double* __restrict__ obs, const int* __restrict__ cells,
                                   int n_obs, const double* __restrict__ S, double log_ne,
                                   double* d, double* sd, double* scal, const int* err) {
    const int m = blockIdx.x;
    if (err[m]) return;
    const size_t mbase = static_cast<size_t>(m) * sp.mstride;
    const double S0 = S[0], S1 = S[1], S2 = S[2], S3 = S[3];
    for (int o = threadIdx.x; o < n_obs; o += blockDim.x) {
        const int j = cells[2 * o], k = cells[2 * o + 1];
        const size_t c = mbase + static_cast<size_t>(k) * sp.pitch + j;
        const double h = sp.h_eq + static_cast<double>(eta[c]);
        const double d0 = obs[4 * o + 2] * h / sp.h_eq - static_cast<double>(hu[c]);
        const double d1 = obs[4 * o + 3] * h / sp.h_eq - static_cast<double>(hv[c]);
        const size_t q = (static_cast<size_t>(m) * n_obs + o) * 2;
        d[q] = d0;
        d[q + 1] = d1;
        sd[q] = S0 * d0 + S1 * d1;
        sd[q + 1] = S2 * d0 + S3 * d1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double phi = 0.0;
        for (int o = 0; o < n_obs; ++o) {
            const size_t q = (static_cast<size_t>(m) * n_obs + o) * 2;
            phi += d[q] * sd[q] + d[q + 1] * sd[q + 1];
        }
        scal[8 * m + 1] = phi;
        scal[8 * m + 0] = phi + log_ne;
    }
}

// SOAR(SOAR(GB^T dipole)) of one (particle, obs) on its aligned coarse grid, as an
// 11x11 window centred on the obs coarse point (requires nxc, nyc >= 11 so nothing
// aliases). Sums keep apply_soar's order (db outer, da inner, from 0.0); the exact
// zeros of the reference's full-grid sums do not change any rounding.
__global__ void pull_windows_kernel(ErrParams ep, const double* __restrict__ sd, int n_obs,
                                    double* win, const int* err) {
    const int m = blockIdx.y, o = blockIdx.x;
    if (err[m]) return;
    __shared__ double s1[WIN * WIN];
    const size_t q = (static_cast<size_t>(m) * n_obs + o) * 2;
    const double yhu = sd[q], yhv = sd[q + 1];
    // adjoint_geo_balance values (stochastic.hpp:181-186), accumulated onto 0.0
    const double vN = 0.0 + (-ep.cyc * yhu);  // (a, b+1)
    const double vS = 0.0 + (ep.cyc * yhu);   // (a, b-1)
    const double vE = 0.0 + (ep.cxc * yhv);   // (a+1, b)
    const double vW = 0.0 + (-ep.cxc * yhv);  // (a-1, b)
    // the first SOAR sees four non-zero inputs: its 25-term sum (db outer, da inner, from
    // 0.0) is the sum of the (at most four) dipole terms in that order -- S (db = -1-pb),
    // W and E (db = -pb), N (db = 1-pb) -- because the other terms add w * (+0) = +-0 to a
    // partial sum that is never -0 (the dipole values are 0.0 + x, never -0; a sum that
    // cancels is +0 under round-to-nearest), which leaves it unchanged
    auto term = [&](int da, int db, double v, double s) {
        return (da >= -2 && da <= 2 && db >= -2 && db <= 2) ? s + ep.w[(db + 2) * 5 + (da + 2)] * v
                                                            : s;
    };
    for (int i = threadIdx.x; i < WIN * WIN; i += blockDim.x) {
        const int pa = i % WIN - WH, pb = i / WIN - WH;  // offset from the obs point
        double s = 0.0;
        s = term(-pa, -1 - pb, vS, s);
        s = term(-1 - pa, -pb, vW, s);
        s = term(1 - pa, -pb, vE, s);
        s = term(-pa, 1 - pb, vN, s);
        s1[i] = s;
    }
    __syncthreads();
    double* out = win + (static_cast<size_t>(m) * n_obs + o) * (WIN * WIN);
    for (int i = threadIdx.x; i < WIN * WIN; i += blockDim.x) {
        const int pa = i % WIN - WH, pb = i / WIN - WH;
        double s = 0.0;
        for (int db = -2; db <= 2; ++db)
            for (int da = -2; da <= 2; ++da) {
                const int ra = pa + da + WH, rb = pb + db + WH;
                const double v = (ra >= 0 && ra < WIN && rb >= 0 && rb < WIN) ? s1[rb * WIN + ra] : 0.0;
                s += ep.w[(db + 2) * 5 + (da + 2)] * v;
            }
        out[i] = s;
    }
}

// periodic interval [lo, hi] (unwrapped, hi - lo < n) intersects [t0, t1] (t1 < n)?
__device__ __forceinline__ bool overlaps(int lo, int hi, int t0, int t1, int n) {
    if (hi - lo + 1 >= n) return true;
    const int a = wrapi(lo, n);
    const int b = a + (hi - lo);  // may exceed n-1
    if (b < n) return !(b < t0 || a > t1);
    return !(t1 < a && t0 > b - n);  // [a, n-1] U [0, b-n]
}

// per fine tile: ascending ids of the observations whose pull footprint may touch it, with
// each observation's coarse alignment (align_coarse_offset / coarse_point_of,
// grid.hpp:106-117) so the pull does no integer division
__global__ void tile_lists_kernel(SweParams sp, ErrParams ep, const int* __restrict__ cells,
                                  int n_obs, int tiles_x, int n_tiles, int4* lists, int* counts) {
    // one warp per tile; lanes test 32 observations at a time and a ballot prefix keeps
    // the list in ascending id
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (t >= n_tiles) return;
    const int tx = t % tiles_x, ty = t / tiles_x;
    const int j0 = tx * TX, j1 = min(j0 + TX, sp.nx) - 1;
    const int k0 = ty * TY, k1 = min(k0 + TY, sp.ny) - 1;
    const int r = 7 * ep.c + 1;  // footprint radius
    int n = 0;
    for (int base = 0; base < n_obs; base += 32) {
        const int o = base + lane;
        bool hit = false;
        int jo = 0, ko = 0;
        if (o < n_obs) {
            jo = cells[2 * o];
            ko = cells[2 * o + 1];
            hit = overlaps(jo - r, jo + r, j0, j1, sp.nx) && overlaps(ko - r, ko + r, k0, k1, sp.ny);
        }
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        if (hit) {
            const int oj = jo % ep.c, ok = ko % ep.c;
            lists[static_cast<size_t>(t) * n_obs + n + __popc(b & ((1u << lane) - 1u))] =
                make_int4(o, oj | (ok << 16), wrapi((jo - oj) / ep.c, ep.nxc),
                          wrapi((ko - ok) / ep.c, ep.nyc));
        }
        n += __popc(b);
    }
    if (lane == 0) counts[t] = n;
}

// Sequential-equivalent gather of every covering observation's pull into one tile of one
// particle (optimal_proposal_pull, SPEC.md:455-463 + add_q_half, stochastic.hpp:144-160).
constexpr int WP = 16;  // padded window pitch: indices 11..15 read exact zeros
using tile::kRowsPerThread;
using tile::kWarps;

#ifndef DC_PULL_MIN_BLOCKS
#define DC_PULL_MIN_BLOCKS 5
#endif

__device__ __forceinline__ void cp_async8d(double* dst, const double* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}

// The interpolation tables of one (tile, covering observation) in the compact form the
// pull reads (~1 KB), plus everything derived from the window's reach, precomputed so
// pull_apply's loop carries no searches or divisions: the column groups pass 1 evaluates,
// the coarse rows ("slots") pass 2 reads -- numbered compactly -- the row groups and
// columns pass 2 evaluates, and the box the add covers.
struct alignas(16) PullTab {
    double ct[tile::XW];             // x fraction per halo column
    double rt[tile::YH];             // y fraction per halo row
    uint8_t cg_a[tile::XW][4];       // per column group: window columns of its 4 coarse points
    uint8_t cg_first[tile::XW + 1];  // first halo column of each column group (+ end)
    uint8_t rg_si[tile::YH][4];      // per row group: compact slots of its 4 coarse rows
    uint8_t rg_first[tile::YH + 1];  // first halo row of each row group (+ end)
    uint8_t wrow[tile::NBMAX + 1];   // window row of each compact slot
    int ns, npg, g0;                 // pass 1: slots 0..ns-1 x column groups g0..g0+npg-1
    int nh, h0, ca, w;               // pass 2: row groups h0..h0+nh-1 x halo columns ca..ca+w-1
    int ar0, ar1, ac0, ac1;          // the add: halo rows ar0..ar1 x halo columns ac0..ac1
    float inv_npg, inv_w;            // 1/npg, 1/w: exact flat-index splits (index < 2^11)
};
constexpr int kPullTabChunks = (sizeof(PullTab) + 15) / 16;
// compact slots a tile can need: (row groups over 32 halo rows) + 3
__host__ __device__ constexpr int pull_slots(int c) {
    return 32 / c + 5 < tile::NBMAX + 1 ? 32 / c + 5 : tile::NBMAX + 1;
}

// Interpolation tables of every (tile, covering observation): they depend on the tile and
// the observation's coarse alignment only, not on the particle, so they are built once per
// analysis here instead of in every (particle, tile) CTA. One 96-thread CTA per entry
// (warp 0 columns, warps 1-2 rows, as tile::setup_cols / setup_rows) into shared memory,
// then the compact table.
__global__ void __launch_bounds__(96)
pull_tables_kernel(SweParams sp, ErrParams ep, const int4* __restrict__ lists,
                   const int* __restrict__ counts, int n_obs, int tiles_x, PullTab* tabs) {
    const int tl = blockIdx.x, li = blockIdx.y;
    if (li >= counts[tl]) return;
    __shared__ tile::Tab F;
    __shared__ int map[tile::NBMAX];
    const int4 ent = lists[static_cast<size_t>(tl) * n_obs + li];
    const int oj = ent.y & 0xffff, ok = ent.y >> 16, ao = ent.z, bo = ent.w;
    const int j0 = (tl % tiles_x) * TX, k0 = (tl / tiles_x) * TY;
    const int nxc = ep.nxc, nyc = ep.nyc;
    PullTab& T = tabs[static_cast<size_t>(tl) * n_obs + li];
    // coarse indices -> the padded window (indices 11..15 read exact zeros)
    tile::setup_cols(F, ep, sp.nx, j0, oj, [&](int a) {
        const int da = wrapf(a - ao + WH, nxc);
        return da < WIN ? da : WP - 1;
    });
    tile::setup_rows(F, ep, sp.ny, k0, ok, [&](int b) {
        const int db = wrapf(b - bo + WH, nyc);
        return db < WIN ? db : WP - 1;
    });
    __syncthreads();
    const int tid = threadIdx.x;
    // the window's reach inside the tile: column groups / row groups with at least one of
    // their four coarse points inside the 11x11 window (the others interpolate to exactly 0)
    if (tid < 32) {
        const int l = tid;
        bool ca_ = false, ra_ = false;
        if (l < F.ncg)
            for (int q = 0; q < 4; ++q) ca_ |= F.cg_a[l][q] != WP - 1;
        if (l < F.nrg)
            for (int q = 0; q < 4; ++q) ra_ |= F.brow[F.rg_sl[l][q]] != WP - 1;
        const unsigned bc = __ballot_sync(0xffffffffu, ca_), br = __ballot_sync(0xffffffffu, ra_);
        if (l == 0) {
            if (bc && br) {
                const int c0 = F.cg_first[__ffs(bc) - 1], c1 = F.cg_first[32 - __clz(bc)] - 1;
                const int r0 = F.rg_first[__ffs(br) - 1], r1 = F.rg_first[32 - __clz(br)] - 1;
                // D is needed on the reach + 2 (the geostrophic differences of the cells
                // next to it read one more D); the add covers the reach + 1
                const int ra = max(r0 - 2, 0), rb = min(r1 + 2, tile::YH - 1);
                const int ca = max(c0 - 2, 0), cb = min(c1 + 2, tile::XW - 1);
                int g0 = 0, g1 = F.ncg - 1;
                while (g0 < g1 && F.cg_first[g0 + 1] <= ca) ++g0;
                while (g1 > g0 && F.cg_first[g1] > cb) --g1;
                int h0 = 0, h1 = F.nrg - 1;
                while (h0 < h1 && F.rg_first[h0 + 1] <= ra) ++h0;
                while (h1 > h0 && F.rg_first[h1] > rb) --h1;
                unsigned long long need = 0;
                for (int g = h0; g <= h1; ++g)
                    for (int q = 0; q < 4; ++q) need |= 1ull << F.rg_sl[g][q];
                int ns = 0;
                for (int sl = 0; sl < F.nb; ++sl) {
                    map[sl] = ns;
                    if (need >> sl & 1ull) T.wrow[ns++] = static_cast<uint8_t>(F.brow[sl]);
                }
                if (ns > pull_slots(ep.c)) __trap();  // the slot bound of the launcher
                T.ns = ns;
                T.g0 = g0;
                T.npg = g1 - g0 + 1;
                T.h0 = h0;
                T.nh = h1 - h0 + 1;
                T.ca = ca;
                T.w = cb - ca + 1;
                T.ar0 = max(r0 - 1, 1);
                T.ar1 = min(r1 + 1, TY);
                T.ac0 = max(c0 - 1, 1);
                T.ac1 = min(c1 + 1, TX);
                T.inv_npg = 1.0f / static_cast<float>(T.npg);
                T.inv_w = 1.0f / static_cast<float>(T.w);
            } else {
                T.ns = T.npg = T.nh = T.w = 0;
                T.ar0 = 1;
                T.ar1 = 0;
                T.ac0 = 1;
                T.ac1 = 0;
            }
        }
    }
    __syncthreads();
    // the compact arrays (entries past the used groups are never read)
    for (int i = tid; i < tile::XW; i += 96) {
        T.ct[i] = F.ct[i];
        for (int q = 0; q < 4; ++q) T.cg_a[i][q] = static_cast<uint8_t>(F.cg_a[i][q]);
    }
    for (int i = tid; i <= tile::XW; i += 96) T.cg_first[i] = static_cast<uint8_t>(F.cg_first[min(i, F.ncg)]);
    for (int i = tid; i < tile::YH; i += 96) {
        T.rt[i] = F.rt[i];
        if (i < F.nrg)
            for (int q = 0; q < 4; ++q) T.rg_si[i][q] = static_cast<uint8_t>(map[F.rg_sl[i][q]]);
    }
    for (int i = tid; i <= tile::YH; i += 96) T.rg_first[i] = static_cast<uint8_t>(F.rg_first[min(i, F.nrg)]);
}

constexpr int kStw = TX + 4;  // TMA box width: cells j0-2 .. j0+TX+1 (16-byte aligned start)

// i / n for i < 2^11 by a float reciprocal: (i + 0.5) * RN(1/n) stays inside
// [q + 0.5/n, q + 1 - 0.5/n] up to a relative error of 2^-23, so truncation is exact
__device__ __forceinline__ int div_small(int i, float inv_n) {
    return __float2int_rz(__fmul_rn(static_cast<float>(i) + 0.5f, inv_n));
}

// pass 1 of one entry (the observation's window W through its tables T): X for the
// entry's slots x the column groups of the reach (interp_tile.cuh: one Catmull-Rom
// coefficient set per (slot, group), the t-polynomial per fine column)
__device__ __forceinline__ void pull_pass1(const PullTab& T, const double* __restrict__ W,
                                           double (*X)[tile::XW]) {
    const int n = T.ns * T.npg;
    // from the last thread down: the segment's add gives the last two warps one row fewer
    // (30 rows over 8 warps), so pass 1 (~2.5 rows' worth per item) goes there first
    for (int i = tile::NT - 1 - threadIdx.x; i < n; i += tile::NT) {
        const int si = div_small(i, T.inv_npg);
        const int g = T.g0 + (i - si * T.npg);
        const double* wr = W + T.wrow[si] * WP;
        const tile::Cm m = tile::coef(wr[T.cg_a[g][0]], wr[T.cg_a[g][1]], wr[T.cg_a[g][2]],
                                      wr[T.cg_a[g][3]]);
        const int j1 = T.cg_first[g + 1];
        for (int jl = T.cg_first[g]; jl < j1; ++jl) X[si][jl] = tile::eval(m, T.ct[jl]);
    }
}

// pass 2 of one entry: D on the row groups x columns of the reach + 2
__device__ __forceinline__ void pull_pass2(const PullTab& T, const double (*X)[tile::XW],
                                           double (*D)[tile::XW]) {
    const int n = T.nh * T.w;
    for (int i = threadIdx.x; i < n; i += tile::NT) {
        const int gi = div_small(i, T.inv_w);
        const int g = T.h0 + gi, jl = T.ca + (i - gi * T.w);
        const tile::Cm m = tile::coef(X[T.rg_si[g][0]][jl], X[T.rg_si[g][1]][jl],
                                      X[T.rg_si[g][2]][jl], X[T.rg_si[g][3]][jl]);
        const int r1 = T.rg_first[g + 1];
        for (int r = T.rg_first[g]; r < r1; ++r) D[r][jl] = tile::eval(m, T.rt[r]);
    }
}

// Sequential-equivalent gather of every covering observation's pull into one tile of one
// particle (optimal_proposal_pull, SPEC.md:455-463 + add_q_half, stochastic.hpp:144-160):
// each thread keeps its cells' state in registers across all of the tile's observations
// and adds them in ascending id, rounding to float after every add as the reference's
// per-observation add_q_half does. The observations run as a three-stage software
// pipeline with one barrier per observation: in the segment of entry i, entry i+2's
// pass 1 fills one X, entry i+1's pass 2 reads the other X into one D, entry i is added
// from the other D, and entry i+3's window and tables stream into the fourth buffer.
struct PullSmem {
    union alignas(128) {  // the TMA box of the tile's state (128-byte aligned), then (once
        float ST[3][TY][kStw];  // in registers) the second D
        double D1[tile::YH][tile::XW];
    } u;
    double D0[tile::YH][tile::XW];
    double W[4][WP * WP];
    PullTab T[4];
    unsigned long long bar;
    // then X[2][slots][XW] doubles (dynamic, pull_slots(c) rows each)
};
size_t pull_smem_bytes(int c) {
    return (sizeof(PullSmem) + 7) / 8 * 8 + 2ull * pull_slots(c) * tile::XW * sizeof(double);
}

__global__ void __launch_bounds__(tile::NT, DC_PULL_MIN_BLOCKS)
pull_apply_kernel(const __grid_constant__ CUtensorMap smap, SweParams sp, ErrParams ep,
                  const double* __restrict__ win, int n_obs,
                  const int4* __restrict__ lists, const int* __restrict__ counts, int tiles_x,
                  const PullTab* __restrict__ tabs, float* eta, float* hu, float* hv,
                  int* err, int* err_pos) {
    extern __shared__ __align__(128) unsigned char pull_raw[];
    PullSmem& P = *reinterpret_cast<PullSmem*>(pull_raw);
    const int xr = pull_slots(ep.c);
    double(*X0)[tile::XW] =
        reinterpret_cast<double(*)[tile::XW]>(pull_raw + (sizeof(PullSmem) + 7) / 8 * 8);
    double(*X1)[tile::XW] = X0 + xr;
    const int m = blockIdx.y;
    // another tile of the member may raise E_DRY_ADD meanwhile: decide once per CTA
    if (__syncthreads_or(err[m] != 0)) return;
    const int tl = blockIdx.x;
    const int cnt = counts[tl];
    if (cnt == 0) return;
    const int j0 = (tl % tiles_x) * TX, k0 = (tl / tiles_x) * TY;
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    const int j = j0 + tx;
    const uint32_t b = smem_u32(&P.bar);
    if (tid == 0) {
        mbar_init(b, 1);
        mbar_fence_init();
        mbar_expect_tx(b, sizeof(P.u.ST));
        tma_row(smem_u32(&P.u.ST[0][0][0]), &smap, j0, m * (sp.ny + 4) + 2 + k0, b);
    }
    // the windows' pad (da or db >= WIN) stays zero; the copies touch only da, db < WIN
    for (int i = tid; i < 4 * WP * WP; i += tile::NT) {
        const int e = i & (WP * WP - 1);
        if ((e & (WP - 1)) >= WIN || (e >> 4) >= WIN) P.W[i >> 8][e] = 0.0;
    }
    const int4* tlist = lists + static_cast<size_t>(tl) * n_obs;
    const PullTab* ttab = tabs + static_cast<size_t>(tl) * n_obs;
    const double* wbase = win + static_cast<size_t>(m) * n_obs * (WIN * WIN);
    auto load = [&](int li) {  // entry li's 11x11 window and tables into buffer li & 3
        const int q = li & 3;
        if (li < cnt) {
            if (tid < WIN * WIN)
                cp_async8d(&P.W[q][(tid / WIN) * WP + tid % WIN],
                           wbase + static_cast<size_t>(tlist[li].x) * (WIN * WIN) + tid);
            for (int c = tid; c < kPullTabChunks; c += tile::NT)
                cp_async16(reinterpret_cast<char*>(&P.T[q]) + 16 * c,
                           reinterpret_cast<const char*>(ttab + li) + 16 * c);
        }
        asm volatile("cp.async.commit_group;\n" ::);  // (empty past the list: uniform counts)
    };
    load(0);
    load(1);
    load(2);
    // the thread's cells: halo row ty + 1 + kWarps q, halo column tx + 1
    float se[kRowsPerThread], su[kRowsPerThread], sv[kRowsPerThread];
    __syncthreads();  // the mbarrier is initialised
    mbar_wait(b, 0);
#pragma unroll
    for (int q = 0; q < kRowsPerThread; ++q) {
        const int r = min(ty + kWarps * q, TY - 1);
        se[q] = P.u.ST[0][r][tx + 2];
        su[q] = P.u.ST[1][r][tx + 2];
        sv[q] = P.u.ST[2][r][tx + 2];
    }
    asm volatile("cp.async.wait_group 2;\n" ::);
    __syncthreads();  // entry 0 landed; the state box is in registers (D1 may be written)
    pull_pass1(P.T[0], P.W[0], X0);
    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncthreads();  // X of entry 0 complete; entry 1 landed
    if (cnt > 1) pull_pass1(P.T[1], P.W[1], X1);
    pull_pass2(P.T[0], X0, P.D0);
    bool dryq[kRowsPerThread], rowok[kRowsPerThread];
#pragma unroll
    for (int q = 0; q < kRowsPerThread; ++q) {
        const int r = ty + kWarps * q;
        dryq[q] = false;
        rowok[q] = r < TY && k0 + r < sp.ny;
    }
    const double cy = ep.cy, cx = ep.cx, heq = ep.h_eq;
    const bool colok = j < sp.nx;
    for (int li = 0; li < cnt; ++li) {
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();  // D of entry li, X of entry li+1 complete; entry li+2 landed
        if (li + 2 < cnt) pull_pass1(P.T[(li + 2) & 3], P.W[(li + 2) & 3], (li & 1) ? X1 : X0);
        if (li + 1 < cnt)
            pull_pass2(P.T[(li + 1) & 3], (li & 1) ? X0 : X1, (li & 1) ? P.D0 : P.u.D1);
        // entry li's add on its box (outside it the pull is an exact zero, whose add leaves
        // the float state unchanged)
        {
            const PullTab& T = P.T[li & 3];
            // this thread's D entries: one base, rows kWarps apart (immediate offsets)
            const double* Dc = ((li & 1) ? &P.u.D1[0][0] : &P.D0[0][0]) + (ty + 1) * tile::XW + tx + 1;
            const int ar0 = T.ar0, ar1 = T.ar1;
            const bool colin = colok && tx + 1 >= T.ac0 && tx + 1 <= T.ac1;
#pragma unroll
            for (int q = 0; q < kRowsPerThread; ++q) {
                const int rr = ty + 1 + kWarps * q;
                if (!rowok[q] || rr < ar0 || rr > ar1) continue;  // warp-uniform
                if (!colin) continue;
                const double* d = Dc + q * kWarps * tile::XW;
                const double de = d[0];
                const double dhu = -cy * (d[tile::XW] - d[-tile::XW]);
                const double dhv = cx * (d[1] - d[-1]);
                const double ee = static_cast<double>(se[q]) + 1.0 * de;
                dryq[q] |= !(heq + ee > 0.0);
                se[q] = static_cast<float>(ee);
                su[q] = static_cast<float>(static_cast<double>(su[q]) + 1.0 * dhu);
                sv[q] = static_cast<float>(static_cast<double>(sv[q]) + 1.0 * dhv);
            }
        }
        load(li + 3);  // into the buffer entry li-1 used (its add ended before the barrier)
    }
    const size_t mbase = static_cast<size_t>(m) * sp.mstride;
#pragma unroll
    for (int q = 0; q < kRowsPerThread; ++q) {
        const int r = ty + kWarps * q, k = k0 + r;
        if (r >= TY || k >= sp.ny || !colok) continue;
        const size_t o = mbase + static_cast<size_t>(k) * sp.pitch + j;
        eta[o] = se[q];
        hu[o] = su[q];
        hv[o] = sv[q];
    }
    bool dry = false;
    int dry_at = 0x7fffffff;
#pragma unroll
    for (int q = kRowsPerThread - 1; q >= 0; --q)
        if (dryq[q]) {
            dry = true;
            dry_at = (k0 + ty + kWarps * q) * sp.nx + j;  // the thread's first dry cell
        }
    if (dry) {
        atomicCAS(err + m, 0, E_DRY_ADD);
        atomicMin(err_pos + m, dry_at);
    }
}

// Stage 3: perpendicular pair + fixed-order dot products (256 strided partials, then a
// halving tree -- the order the CPU checker restates). One CTA of 256 per particle.
__global__ void __launch_bounds__(256)
perp_pair_kernel(ErrParams ep, uint64_t seed, long long member_base, uint64_t cycle,
                 double ratio, double* xi, double* nu, int* foffs, double* scal,
                 const int* /*err*/) {
    // state independent: computed for every member (it runs concurrently with the pull
    // chain, whose error flags it must not depend on)
    const int m = blockIdx.x;
    const int nr = ep.nxc * ep.nyc;
    const uint64_t key = det::stream_key(seed, 2 /*filter*/, static_cast<uint64_t>(member_base + m));
    double* X = xi + static_cast<size_t>(m) * nr;
    double* N = nu + static_cast<size_t>(m) * nr;
    const int npairs = (nr + 1) / 2;
    for (int p = threadIdx.x; p < npairs; p += 256) {
        double a, b;
        det::normal_pair(key, 0, cycle, static_cast<uint32_t>(p), &a, &b);
        X[2 * p] = a;
        if (2 * p + 1 < nr) X[2 * p + 1] = b;
        det::normal_pair(key, 1, cycle, static_cast<uint32_t>(p), &a, &b);
        N[2 * p] = a;
        if (2 * p + 1 < nr) N[2 * p + 1] = b;
    }
    if (threadIdx.x == 0) {
        int oj, ok;
        det::draw_offsets(key, 0, cycle, ep.c, &oj, &ok);
        foffs[2 * m] = oj;
        foffs[2 * m + 1] = ok;
    }
    __syncthreads();
    __shared__ double pxx[256], pnn[256], pnx[256];
    const int l = threadIdx.x;
    double sxx = 0.0, snn = 0.0, snx = 0.0;
    for (int i = l; i < nr; i += 256) {
        const double x = X[i], n = N[i];
        sxx += x * x;
        snn += n * n;
        snx += n * x;
    }
    pxx[l] = sxx;
    pnn[l] = snn;
    pnx[l] = snx;
    __syncthreads();
    for (int s = 128; s >= 1; s >>= 1) {
        if (l < s) {
            pxx[l] = pxx[l] + pxx[l + s];
            pnn[l] = pnn[l] + pnn[l + s];
            pnx[l] = pnx[l] + pnx[l + s];
        }
        __syncthreads();
    }
    const double xx = pxx[0], nn = pnn[0], nxv = pnx[0];
    const double a = nxv / xx;
    const double sc = sqrt(nn / (nn - a * nxv));
    for (int i = l; i < nr; i += 256) N[i] = sc * (N[i] - a * X[i]);
    if (l == 0) {
        scal[8 * m + 2] = xx * ratio;  // gamma
        scal[8 * m + 3] = nn * ratio;  // zeta
    }
}

__global__ void gather_cz_kernel(int M, const double* __restrict__ scal, double* cz) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M) return;
    cz[2 * m] = scal[8 * m + 0];
    cz[2 * m + 1] = scal[8 * m + 3];
}

// Lambert W0 by Halley iteration, fp64, tol 1e-12, clamp within 1e-9 of -1/e
__device__ bool lambert_w0(double x, double* w_out) {
    const double em1 = 0.36787944117144233;
    if (x < -em1) {
        if (x >= -em1 - 1e-9) x = -em1;
        else return false;
    }
    if (x == -em1) {
        *w_out = -1.0;
        return true;
    }
    double w;
    if (x < -0.32) {
        const double p = sqrt(2.0 * (2.71828182845904509080 * x + 1.0));
        w = -1.0 + p * (1.0 + p * (-1.0 / 3.0 + p * (11.0 / 72.0)));
    } else {
        w = x - x * x;
    }
    for (int it = 0; it < 100; ++it) {
        const double ew = det::exp_det(w);
        const double f = w * ew - x;
        const double wp1 = w + 1.0;
        if (wp1 == 0.0) break;
        const double den = ew * wp1 - (w + 2.0) * f / (2.0 * wp1);
        const double dw = f / den;
        w = w - dw;
        if (fabs(dw) <= 1e-12 * (1.0 + fabs(w))) {
            *w_out = w;
            return true;
        }
    }
    return false;
}

// Stage 4 (the barrier) + stage 5. Single CTA: the sum for w_target and the beta min
// run in particle-id order over all N_e particles; every rank computes them identically.
constexpr int kBarrierStage = 2048;  // particles staged in shared memory (32 KB)

// Stage 4 + 5. Two-stage (default): w_target = mean c, beta = min((w - c)/zeta + 1),
// c* = (w - c) - (beta - 1) zeta. One-stage IEWPF:
// w_target = max c, c* = w - c, no nu term (beta reported as 0).
__global__ void barrier_alpha_kernel(const double* __restrict__ cz_all, int n_total, int M,
                                     double n_psi, double* scal, double* wb, int* aerr,
                                     int one_stage) {
    __shared__ double s_w, s_b;
    __shared__ int s_bad;
    // the (c, zeta) pairs are staged in shared memory by all threads, so the fixed-order
    // sequential reductions below do not wait on a global load per particle
    __shared__ double cz_s[2 * kBarrierStage];
    const bool staged = n_total <= kBarrierStage;
    if (staged)
        for (int i = threadIdx.x; i < 2 * n_total; i += blockDim.x) cz_s[i] = cz_all[i];
    __syncthreads();
    const double* cz = staged ? cz_s : cz_all;
    if (threadIdx.x == 0) {
        double w, beta;
        int bad = 0;
        if (one_stage) {
            w = -__longlong_as_double(0x7ff0000000000000ll);
            for (int i = 0; i < n_total; ++i) w = (cz[2 * i] > w) ? cz[2 * i] : w;
            beta = 0.0;
        } else {
            double sum = 0.0;
            for (int i = 0; i < n_total; ++i) sum += cz[2 * i];
            w = sum / n_total;
            beta = __longlong_as_double(0x7ff0000000000000ll);
            for (int i = 0; i < n_total; ++i) {
                const double z = cz[2 * i + 1];
                if (!(z > 0.0)) bad = 1;
                const double b = (w - cz[2 * i]) / z + 1.0;
                beta = (b < beta) ? b : beta;
            }
            if (!(beta >= 0.0)) bad = 1;
        }
        s_w = w;
        s_b = beta;
        s_bad = bad;
        wb[0] = w;
        wb[1] = beta;
    }
    __syncthreads();
    // errors go to aerr (merged into err after the pull chain joined, merge_err_kernel)
    for (int m = threadIdx.x; m < M; m += blockDim.x) {
        if (s_bad) {
            aerr[m] = E_BETA;
            continue;
        }
        const double c = scal[8 * m + 0], gamma = scal[8 * m + 2], zeta = scal[8 * m + 3];
        const double cstar = one_stage ? s_w - c : (s_w - c) - (s_b - 1.0) * zeta;
        const double t = gamma / n_psi;
        const double x = -((t * det::exp_det(-t)) * det::exp_det(-cstar / n_psi));
        double w;
        if (!lambert_w0(x, &w)) {
            aerr[m] = E_ALPHA;
            continue;
        }
        scal[8 * m + 4] = -(n_psi / gamma) * w;
    }
}

// nearest coarse point of fine index j on an offset-o grid
__device__ __forceinline__ int nearest_coarse(int j, int o, int c, int n) {
    const int v = j - o + (c - 1) / 2;
    const int q = (v >= 0) ? v / c : -((-v + c - 1) / c);
    return wrapi(q, n);
}

// Stage 6a: z = beta^1/2 nu + alpha^1/2 xi, then the local U Sigma^1/2 blocks in ascending
// obs id. One CTA per member holds z in shared memory; the blocks run
// level by level (iewpf_api.inc: build_block_schedule) with kLbGroups observations of a
// level at a time, one 64-thread group each -- the blocks of a level are disjoint, so this
// equals the sequential ascending-id application bit for bit.
constexpr int kObsTab = 1024;
constexpr int kLbGroups = 8;

__global__ void __launch_bounds__(64 * kLbGroups)
local_blocks_kernel(ErrParams ep, const double* __restrict__ xi, const double* __restrict__ nu,
                    const double* __restrict__ scal, const double* __restrict__ wb,
                    const int* __restrict__ cells, int n_obs, const int* __restrict__ order,
                    const int* __restrict__ level_start, int n_levels,
                    const int* __restrict__ foffs, const double* __restrict__ usig, double* z,
                    const int* aerr, int z_in_smem, int one_stage) {
    const int m = blockIdx.x;
    if (aerr[m]) return;  // no alpha for this member
    extern __shared__ double dyn[];  // [49*49] U, then [nr] z when it fits
    double* U = dyn;
    __shared__ double bin[kLbGroups][49];
    __shared__ int idx[kLbGroups][49];
    __shared__ int ab[kObsTab][2];
    __shared__ int ord[kObsTab];
    __shared__ int lst[kObsTab + 1];
    const int nr = ep.nxc * ep.nyc;
    for (int i = threadIdx.x; i < 49 * 49; i += blockDim.x) U[i] = usig[i];
    const double sqb = sqrt(wb[1]);
    const double sqa = sqrt(scal[8 * m + 4]);
    const double* X = xi + static_cast<size_t>(m) * nr;
    const double* N = nu + static_cast<size_t>(m) * nr;
    double* Zg = z + static_cast<size_t>(m) * nr;
    double* Z = z_in_smem ? dyn + 49 * 49 : Zg;
    for (int i = threadIdx.x; i < nr; i += blockDim.x)
        Z[i] = one_stage ? sqa * X[i] : sqb * N[i] + sqa * X[i];
    const int oj = foffs[2 * m], ok = foffs[2 * m + 1];
    for (int o = threadIdx.x; o < n_obs; o += blockDim.x) {  // block centres (member offsets)
        ab[o][0] = nearest_coarse(cells[2 * o], oj, ep.c, ep.nxc);
        ab[o][1] = nearest_coarse(cells[2 * o + 1], ok, ep.c, ep.nyc);
        ord[o] = order[o];
    }
    for (int l = threadIdx.x; l <= n_levels; l += blockDim.x) lst[l] = level_start[l];
    __syncthreads();
    const int g = threadIdx.x >> 6, r = threadIdx.x & 63;
    for (int l = 0; l < n_levels; ++l) {
        const int le = lst[l + 1];
        for (int q0 = lst[l]; q0 < le; q0 += kLbGroups) {
            const bool act = (q0 + g < le) && r < 49;
            if (act) {
                const int o = ord[q0 + g];
                const int id = wrapf(ab[o][1] + r / 7 - 3, ep.nyc) * ep.nxc +
                               wrapf(ab[o][0] + r % 7 - 3, ep.nxc);
                idx[g][r] = id;
                bin[g][r] = Z[id];
            }
            __syncthreads();
            if (act) {
                double s = 0.0;
#pragma unroll 7
                for (int c = 0; c < 49; ++c) s += U[r * 49 + c] * bin[g][c];
                Z[idx[g][r]] = s;
            }
            __syncthreads();
        }
    }
    if (z_in_smem)
        for (int i = threadIdx.x; i < nr; i += blockDim.x) Zg[i] = Z[i];
}

// advect_drifters: forward Euler at the containing cell, fp64
__global__ void drifters_kernel(SweParams sp, const float* __restrict__ eta,
                                const float* __restrict__ hu, const float* __restrict__ hv,
                                int M, int n_d, double dt, double* pos, int* wind, int* err,
                                int* err_pos) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M * n_d) return;
    const int m = i / n_d;
    if (err[m]) return;
    double* p = pos + 2 * static_cast<size_t>(i);
    int j, k;
    if (!locate(sp, p[0], p[1], &j, &k)) {
        atomicCAS(err + m, 0, E_DRY_DRIFTER);
        return;
    }
    const size_t c = static_cast<size_t>(m) * sp.mstride + static_cast<size_t>(k) * sp.pitch + j;
    const double h = sp.h_eq + static_cast<double>(eta[c]);
    if (!(h > 0.0)) {
        atomicCAS(err + m, 0, E_DRY_DRIFTER);
        atomicMin(err_pos + m, k * sp.nx + j);
        return;
    }
    const double u = static_cast<double>(hu[c]) / h;
    const double v = static_cast<double>(hv[c]) / h;
    const double lx = sp.nx * sp.dx, ly = sp.ny * sp.dy;
    const double xs[2] = {p[0] + dt * u, p[1] + dt * v};
    const double ls[2] = {lx, ly};
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        const double xn = xs[a], len = ls[a];
        double xm = fmod(xn, len);
        if (xm < 0.0) xm += len;
        if (xm >= len) xm = 0.0;
        wind[2 * static_cast<size_t>(i) + a] += (xn >= len) ? 1 : ((xn < 0.0) ? -1 : 0);
        p[a] = xm;
    }
}

// observe_mooring without noise, one member
__global__ void observe_mooring_kernel(SweParams sp, const float* __restrict__ eta,
                                       const float* __restrict__ hu, const float* __restrict__ hv,
                                       int m, const double* __restrict__ xy, int n, double* y,
                                       int* bad) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n) return;
    int j, k;
    if (!locate(sp, xy[2 * o], xy[2 * o + 1], &j, &k)) {
        atomicExch(bad, 1);
        return;
    }
    const size_t c = static_cast<size_t>(m) * sp.mstride + static_cast<size_t>(k) * sp.pitch + j;
    const double h = sp.h_eq + static_cast<double>(eta[c]);
    y[2 * o] = static_cast<double>(hu[c]) * sp.h_eq / h;
    y[2 * o + 1] = static_cast<double>(hv[c]) * sp.h_eq / h;
}

} // namespace

void launch_obs_locate(cudaStream_t s, const SweParams& sp, const double* obs, int n_obs,
                       int* cells, int* bad) {
    KScope ks(s, "obs_locate", 40.0 * n_obs);
    obs_locate_kernel<<<(n_obs + 127) / 128, 128, 0, s>>>(sp, obs, n_obs, cells, bad);
}

void launch_innovations(cudaStream_t s, const SweParams& sp, const float* eta, const float* hu,
                        const float* hv, const double* obs, const int* cells, int n_obs,
                        const double* S, double log_ne, double* d, double* sd, double* scal,
                        const int* err, int M) {
    // per (member, obs): a 12 B state gather, d and S d written (32 B)
    KScope ks(s, "innovations", 44.0 * n_obs * M + 40.0 * n_obs);
    innovations_kernel<<<M, 256, 0, s>>>(sp, eta, hu, hv, obs, cells, n_obs, S, log_ne, d, sd,
                                          scal, err);
}

void launch_pull_windows(cudaStream_t s, const ErrParams& ep, const double* sd, int n_obs,
                         double* win, const int* err, int M) {
    KScope ks(s, "pull_windows", (16.0 + 8.0 * WIN * WIN) * n_obs * M);
    pull_windows_kernel<<<dim3(n_obs, M), 128, 0, s>>>(ep, sd, n_obs, win, err);
}

void launch_tile_lists(cudaStream_t s, const SweParams& sp, const ErrParams& ep, const int* cells,
                       int n_obs, int* lists, int* counts, int* n_tiles_out, int* tiles_x_out) {
    const int tiles_x = (sp.nx + TX - 1) / TX, tiles_y = (sp.ny + TY - 1) / TY;
    const int n_tiles = tiles_x * tiles_y;
    KScope ks(s, "tile_lists", 16.0 * n_tiles * n_obs + 8.0 * n_obs);
    tile_lists_kernel<<<(n_tiles * 32 + 127) / 128, 128, 0, s>>>(
        sp, ep, cells, n_obs, tiles_x, n_tiles, reinterpret_cast<int4*>(lists), counts);
    *n_tiles_out = n_tiles;
    *tiles_x_out = tiles_x;
}

size_t pull_table_bytes() { return sizeof(PullTab); }

void launch_pull_apply(cudaStream_t s, const CUtensorMap* smap, const SweParams& sp,
                       const ErrParams& ep, const double* win,
                       const int* cells, int n_obs, const int* lists, const int* counts,
                       int n_tiles, int tiles_x, void* tabs, float* eta, float* hu, float* hv,
                       int* err, int* err_pos, int M, double entries, double touched_cells) {
    PullTab* T = static_cast<PullTab*>(tabs);
    {
        KScope ks(s, "pull_tables", entries * (sizeof(PullTab) + 16.0));
        pull_tables_kernel<<<dim3(n_tiles, n_obs), 96, 0, s>>>(
            sp, ep, reinterpret_cast<const int4*>(lists), counts, n_obs, tiles_x, T);
    }
    // the touched tiles' state read and written once (24 B/cell), every (member, obs)
    // window once, the tables once
    KScope ks(s, "pull_apply", (24.0 * touched_cells + 8.0 * WIN * WIN * n_obs) * M +
                                   entries * sizeof(PullTab));
    const size_t smem = pull_smem_bytes(ep.c);
    smem_opt_in(pull_apply_kernel, pull_smem_bytes(1));  // the largest (c_omega = 1)
    pull_apply_kernel<<<dim3(n_tiles, M), tile::NT, smem, s>>>(*smap, sp, ep, win, n_obs,
                                                       reinterpret_cast<const int4*>(lists), counts,
                                                       tiles_x, T, eta, hu, hv, err, err_pos);
}

void launch_perp_pair(cudaStream_t s, const ErrParams& ep, uint64_t seed, int64_t member_base,
                      uint64_t cycle, double ratio, double* xi, double* nu, int* foffs,
                      double* scal, const int* err, int M) {
    // xi, nu~ written, read back for the dot products, nu written again
    KScope ks(s, "perp_pair", 40.0 * ep.nxc * ep.nyc * M);
    perp_pair_kernel<<<M, 256, 0, s>>>(ep, seed, member_base, cycle, ratio, xi, nu, foffs, scal,
                                       err);
}

void launch_gather_cz(cudaStream_t s, int M, const double* scal, double* cz) {
    KScope ks(s, "gather_cz", 32.0 * M);
    gather_cz_kernel<<<(M + 127) / 128, 128, 0, s>>>(M, scal, cz);
}

void launch_barrier_alpha(cudaStream_t s, const double* cz_all, int n_total, int M, double n_psi,
                          int one_stage, double* scal, double* wb, int* aerr) {
    KScope ks(s, "barrier_alpha", 16.0 * n_total + 40.0 * M);
    barrier_alpha_kernel<<<1, 256, 0, s>>>(cz_all, n_total, M, n_psi, scal, wb, aerr, one_stage);
}

namespace {
__global__ void merge_err_kernel(int M, const int* __restrict__ aerr, int* err) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m < M && aerr[m] && !err[m]) err[m] = aerr[m];
}
}  // namespace

void launch_merge_err(cudaStream_t s, int M, const int* aerr, int* err) {
    KScope ks(s, "merge_err", 12.0 * M);
    merge_err_kernel<<<(M + 127) / 128, 128, 0, s>>>(M, aerr, err);
}

void launch_local_blocks(cudaStream_t s, const ErrParams& ep, const double* xi, const double* nu,
                         const double* scal, const double* wb, const int* cells, int n_obs,
                         const int* order, const int* level_start, int n_levels,
                         const int* foffs, const double* usig, double* z, const int* err,
                         const int* aerr, int M, int one_stage) {
    const size_t nr = static_cast<size_t>(ep.nxc) * ep.nyc;
    const size_t full = (49 * 49 + nr) * sizeof(double);
    const int in_smem = full <= 160 * 1024;
    smem_opt_in(local_blocks_kernel, 160 * 1024);
    KScope ks(s, "local_blocks", 24.0 * nr * M);  // xi, nu read, z written
    local_blocks_kernel<<<M, 64 * kLbGroups, in_smem ? full : 49 * 49 * sizeof(double), s>>>(
        ep, xi, nu, scal, wb, cells, n_obs, order, level_start, n_levels, foffs, usig, z, aerr,
        in_smem, one_stage);
    (void)err;
}

void launch_drifters(cudaStream_t s, const SweParams& sp, const float* eta, const float* hu,
                     const float* hv, int M, int n_d, double dt, double* pos, int* wind, int* err,
                     int* err_pos) {
    const int n = M * n_d;
    // per drifter: 12 B state gather, position and winding counts read and written
    KScope ks(s, "drifters", 60.0 * n);
    drifters_kernel<<<(n + 127) / 128, 128, 0, s>>>(sp, eta, hu, hv, M, n_d, dt, pos, wind, err,
                                                    err_pos);
}

void launch_observe_mooring(cudaStream_t s, const SweParams& sp, const float* eta, const float* hu,
                            const float* hv, int m, const double* xy, int n, double* y, int* bad) {
    KScope ks(s, "observe_mooring", 44.0 * n);
    observe_mooring_kernel<<<(n + 127) / 128, 128, 0, s>>>(sp, eta, hu, hv, m, xy, n, y, bad);
}

} // namespace dcg
