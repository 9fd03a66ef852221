// stochastic.cu -- model-error covariance Q^{1/2} on sm_100a (compiled --fmad=false).
//
// Three kernels per draw, all members at once:
//   philox_noise : xi ~ N(0,I) on the coarse grid + per-draw offsets, counter-based
//                  (Philox4x32-10 keyed by stream_seed(seed, tag, member)); replaces the
//                  sequential NoiseStream consumption of perturb_state
//                  (stochastic.hpp:168-171, rng.hpp:57-84).
//   coarse_soar  : the 5x5 SOAR stencil (stochastic.hpp:49-69), one thread per point.
//   q_half_apply : Catmull-Rom interpolation to the fine grid, geostrophic balance and
//                  the in-place add (stochastic.hpp:93-160) fused in one HBM pass:
//                  read 12 B + write 12 B per cell. The interpolation is separable --
//                  the x-pass over the coarse rows a tile needs is staged in shared
//                  memory and reused by every fine row (identical operands and order as
//                  the reference's per-cell col[m], so bit-identical results).
// All arithmetic is fp64 as in the reference; --fmad=false keeps the reference's
// evaluation order without contraction, so results match bit-for-bit.
#include <cuda_runtime.h>
#include <cstdint>

#include "dc_internal.h"
#include "detmath.cuh"
#include "fp32_rn.cuh"
#include "interp_tile.cuh"
#include "tma.cuh"

namespace dcg {

namespace {

using det::wrap1;
using det::wrapi;

__global__ void philox_noise_kernel(ErrParams ep, int M, uint64_t seed, uint64_t tag,
                                    long long member_base, uint32_t substream, uint64_t draw,
                                    double* __restrict__ xi, int* __restrict__ offsets,
                                    const int* __restrict__ err) {
    const int m = blockIdx.y;
    if (err && err[m]) return;
    const uint64_t key = det::stream_key(seed, tag, static_cast<uint64_t>(member_base + m));
    const int nr = ep.nxc * ep.nyc;
    const int npairs = (nr + 1) / 2;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npairs; p += gridDim.x * blockDim.x) {
        double z0, z1;
        det::normal_pair(key, substream, draw, static_cast<uint32_t>(p), &z0, &z1);
        double* o = xi + static_cast<size_t>(m) * nr;
        o[2 * p] = z0;
        if (2 * p + 1 < nr) o[2 * p + 1] = z1;
    }
    if (offsets && blockIdx.x == 0 && threadIdx.x == 0) {
        int oj, ok;
        det::draw_offsets(key, substream, draw, ep.c, &oj, &ok);
        offsets[2 * m] = oj;
        offsets[2 * m + 1] = ok;
    }
}

// apply_soar (stochastic.hpp:49-69): s = 0; db outer, da inner.
__global__ void coarse_soar_kernel(ErrParams ep, int M, const double* __restrict__ in,
                                   double* __restrict__ out, const int* __restrict__ err) {
    const int m = blockIdx.y;
    if (err && err[m]) return;
    const int nr = ep.nxc * ep.nyc;
    const double* src = in + static_cast<size_t>(m) * nr;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += gridDim.x * blockDim.x) {
        const int a = i % ep.nxc, b = i / ep.nxc;
        double s = 0.0;
#pragma unroll
        for (int db = -2; db <= 2; ++db) {
            const int bb = det::wrapf(b + db, ep.nyc);
#pragma unroll
            for (int da = -2; da <= 2; ++da)
                s += ep.w[(db + 2) * 5 + (da + 2)] * __ldg(src + bb * ep.nxc + det::wrapf(a + da, ep.nxc));
        }
        out[static_cast<size_t>(m) * nr + i] = s;
    }
}

// Philox noise + SOAR fused for the model-error draw (perturb_state, stochastic.hpp:164-173):
// one CTA per (band of kBand coarse rows, member). The band's xi rows and a 2-row periodic
// halo are generated straight into shared memory (pair p gives elements 2p, 2p+1 as
// philox_noise does; a pair straddling a row boundary is generated for both rows), then
// the 5x5 SOAR stencil (db outer, da inner, from 0.0 -- coarse_soar_kernel's order) writes
// the band of the correlated field. xi never goes to HBM.
constexpr int kBand = 16;

__global__ void __launch_bounds__(256)
philox_soar_kernel(ErrParams ep, int M, uint64_t seed, uint64_t tag, long long member_base,
                   uint32_t substream, uint64_t draw, double* __restrict__ corr,
                   int* __restrict__ offsets, const int* __restrict__ err) {
    extern __shared__ double X[];  // [kBand + 4][nxc]
    const int m = blockIdx.y;
    if (err && err[m]) return;
    const uint64_t key = det::stream_key(seed, tag, static_cast<uint64_t>(member_base + m));
    const int nxc = ep.nxc, nyc = ep.nyc;
    const int b0 = blockIdx.x * kBand;
    const int nb = min(kBand, nyc - b0);
    const int rows = nb + 4;
    const int ppr = nxc / 2 + 2;  // pair slots per row (covers a row of either parity)
    for (int it = threadIdx.x; it < rows * ppr; it += blockDim.x) {
        const int sr = it / ppr, q = it - sr * ppr;
        const int gb = det::wrapf(b0 - 2 + sr, nyc);
        const int lo = gb * nxc;                   // first element of the row
        const int p = (lo >> 1) + q;               // pair index
        if (2 * p >= lo + nxc) continue;           // past the row
        double z0, z1;
        det::normal_pair(key, substream, draw, static_cast<uint32_t>(p), &z0, &z1);
        const int e0 = 2 * p - lo, e1 = e0 + 1;    // row-local element indices
        if (e0 >= 0 && e0 < nxc) X[sr * nxc + e0] = z0;
        if (e1 >= 0 && e1 < nxc) X[sr * nxc + e1] = z1;
    }
    if (offsets && blockIdx.x == 0 && threadIdx.x == 0) {
        int oj, ok;
        det::draw_offsets(key, substream, draw, ep.c, &oj, &ok);
        offsets[2 * m] = oj;
        offsets[2 * m + 1] = ok;
    }
    __syncthreads();
    double* out = corr + static_cast<size_t>(m) * nxc * nyc + static_cast<size_t>(b0) * nxc;
    for (int i = threadIdx.x; i < nb * nxc; i += blockDim.x) {
        const int bl = i / nxc, a = i - bl * nxc;
        double sum = 0.0;
#pragma unroll
        for (int db = -2; db <= 2; ++db) {
            const double* row = X + (bl + 2 + db) * nxc;
#pragma unroll
            for (int da = -2; da <= 2; ++da)
                sum += ep.w[(db + 2) * 5 + (da + 2)] * row[det::wrapf(a + da, nxc)];
        }
        out[i] = sum;
    }
}

using tile::TX;
using tile::TY;

__device__ __forceinline__ unsigned ordered_bits(float f) {
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Q^{1/2} tail + add (stochastic.hpp:144-160) for one (member, 32x30 tile). When mx is
// given, also reduces the CFL statistics of the NEW state (Stepper::load,
// swe.hpp:306-317) so the next model step needs no separate scan.
using tile::kRowsPerThread;
using tile::kWarps;
#ifndef DC_QHALF_WAVES
#define DC_QHALF_WAVES 8.0
#endif
#ifndef DC_QHALF_MIN_BLOCKS
#define DC_QHALF_MIN_BLOCKS 5
#endif

// The tile's state arrives by TMA: one box {TX+4 columns from cell j0-2, TY rows, 3 fields}
// of the state set's map (storage column j0 is 16-byte aligned; the box's first two and
// last two columns are not used).
constexpr int kStw = TX + 4;
static_assert(kStw * sizeof(float) % 16 == 0, "TMA box rows must be 16-byte multiples");

// Strip form: one CTA streams down a column strip of S tiles of one member (32 columns x
// S*30 rows). The column tables are built once per strip; the x pass (X, one row per
// coarse row) lives in a ring keyed by the coarse row's unwrapped index, so a coarse row
// shared by consecutive tiles is evaluated once; the tiles run as a two-barrier software
// pipeline -- the add of tile i beside the x pass of tile i+1's new coarse rows, then the
// y pass of tile i+1 into the other D while tile i+1's state arrives by TMA.
struct QhCols {  // column tables of the strip (interp_tile.cuh setup_cols, identity map)
    double ct[tile::XW];
    int cg_a[tile::XW][4];
    int cg_first[tile::XW + 1];
    int ncg;
};
struct QhRows {  // row tables of one tile: one lane of warp 1 per halo row
    double rt[tile::YH];
    int rg_first[tile::YH + 1];
    int rg_u[tile::YH];  // unwrapped coarse row b0 of each row group
    int rg_slot[tile::YH][4];  // ring slots of its four coarse rows b0-1 .. b0+2
    int nrg, u_last;     // u_last: the last coarse row the tile reads (b0 of row 31, + 2)
};
struct QhSmem {
    float ST[3][TY][kStw];       // the tile's state box (TMA), 128-byte aligned at offset 0
    double D[2][tile::YH][tile::XW];
    QhCols C;
    QhRows R[3];  // tile i in R[i % 3]
    float red[3][kWarps];
    unsigned long long bar;
    // then X[ring][XW] doubles (dynamic)
};
__host__ __device__ constexpr int qh_ring(int c) { return 31 / c + 6; }

__device__ __forceinline__ int qh_slot(int u, int ring) { return (u + 4 * ring) % ring; }

// halo rows of the tile starting at fine row k0 (warp 1, lane = halo row): b0 and t as
// interpolate_bicubic computes them (stochastic.hpp:98-102) from the wrapped row, and the
// unwrapped coarse index u = b0 -/+ nyc for halo rows above / below the domain
__device__ __forceinline__ void qh_rows(QhRows& R, const ErrParams& ep, int ny, int k0, int ok,
                                        int ring) {
    const int lane = threadIdx.x & 31;
    const int k = k0 - 1 + lane;
    int b0;
    double t;
    tile::row_b0(ep, wrap1(k, ny), ok, &b0, &t);
    const int u = b0 + (k < 0 ? -ep.nyc : (k >= ny ? ep.nyc : 0));
    const int up = __shfl_up_sync(0xffffffffu, u, 1);
    const bool st = lane == 0 || u != up;
    const unsigned bl = __ballot_sync(0xffffffffu, st);
    R.rt[lane] = t;
    if (st) {
        const int g = __popc(bl & tile::lanemask_le()) - 1;
        R.rg_first[g] = lane;
        R.rg_u[g] = u;
#pragma unroll
        for (int q = 0; q < 4; ++q) R.rg_slot[g][q] = qh_slot(u - 1 + q, ring);
    }
    if (lane == 31) {
        const int n = __popc(bl);
        R.nrg = n;
        R.rg_first[n] = tile::YH;
        R.u_last = u + 2;
    }
}

// x pass of coarse rows u0 .. u1 (unwrapped) into their ring slots
__device__ __forceinline__ void qh_xpass(const QhCols& C, const ErrParams& ep,
                                         const double* __restrict__ cf, double (*X)[tile::XW],
                                         int ring, int u0, int u1) {
    const int ncg = C.ncg, n = (u1 - u0 + 1) * ncg;
    const float inv_ncg = 1.0f / static_cast<float>(ncg);
    // from the last thread down: the add gives the last two warps one row fewer
    for (int i = tile::NT - 1 - threadIdx.x; i < n; i += tile::NT) {
        const int ui = __float2int_rz(__fmul_rn(static_cast<float>(i) + 0.5f, inv_ncg));
        const int g = i - ui * ncg;
        const int u = u0 + ui;
        const double* row = cf + det::wrapf(u, ep.nyc) * ep.nxc;
        const tile::Cm m = tile::coef(__ldg(row + C.cg_a[g][0]), __ldg(row + C.cg_a[g][1]),
                                      __ldg(row + C.cg_a[g][2]), __ldg(row + C.cg_a[g][3]));
        double* x = X[qh_slot(u, ring)];
        const int j1 = C.cg_first[g + 1];
        for (int jl = C.cg_first[g]; jl < j1; ++jl) x[jl] = tile::eval(m, C.ct[jl]);
    }
}

// y pass of one tile: D on all 32 halo rows x 34 halo columns
__device__ __forceinline__ void qh_ypass(const QhRows& R, const double (*X)[tile::XW],
                                         double (*D)[tile::XW]) {
    const int n = R.nrg * tile::XW;
    for (int i = threadIdx.x; i < n; i += tile::NT) {
        const int g = i / tile::XW, jl = i - g * tile::XW;
        const tile::Cm m = tile::coef(X[R.rg_slot[g][0]][jl], X[R.rg_slot[g][1]][jl],
                                      X[R.rg_slot[g][2]][jl], X[R.rg_slot[g][3]][jl]);
        const int r1 = R.rg_first[g + 1];
        for (int r = R.rg_first[g]; r < r1; ++r) D[r][jl] = tile::eval(m, R.rt[r]);
    }
}

// UNIT: scale == 1.0 (model error, posterior): scale * x == x exactly, so the three
// products are dropped (bitwise the same)
template <bool UNIT>
__global__ void __launch_bounds__(tile::NT, DC_QHALF_MIN_BLOCKS)
q_half_apply_kernel(const __grid_constant__ CUtensorMap smap, SweParams sp, ErrParams ep,
                    const double* __restrict__ corr, const int* __restrict__ offsets,
                    double scale, float* eta, float* hu, float* hv, int* err, int* err_pos,
                    unsigned* mx, int strip_tiles) {
    extern __shared__ __align__(128) unsigned char qh_raw[];
    QhSmem& S = *reinterpret_cast<QhSmem*>(qh_raw);
    double(*X)[tile::XW] = reinterpret_cast<double(*)[tile::XW]>(qh_raw + sizeof(QhSmem));
    const int m = blockIdx.z;
    // another tile of the member may raise E_DRY_ADD meanwhile: decide once per CTA
    if (__syncthreads_or(err[m] != 0)) return;
    const int n_tiles_y = (sp.ny + TY - 1) / TY;
    const int t0 = blockIdx.y * strip_tiles, nt = min(strip_tiles, n_tiles_y - t0);
    const int j0 = blockIdx.x * TX;
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5, warp = ty;
    const int j = j0 + tx;
    const int ring = qh_ring(ep.c);
    const size_t pitch = sp.pitch;
    const int oj = offsets[2 * m], ok = offsets[2 * m + 1];
    const double* cf = corr + static_cast<size_t>(m) * ep.nxc * ep.nyc;
    // the member's fields (a member's storage is < 2^31 cells: 32-bit offsets below)
    float* const Em = eta + static_cast<size_t>(m) * sp.mstride;
    float* const Um = hu + static_cast<size_t>(m) * sp.mstride;
    float* const Vm = hv + static_cast<size_t>(m) * sp.mstride;
    const uint32_t b = smem_u32(&S.bar);
    if (tid == 0) {
        mbar_init(b, 1);
        mbar_fence_init();
        mbar_expect_tx(b, sizeof(S.ST));
        // storage row of cell row k0 of member m (the map starts at row -2 of member 0)
        tma_row(smem_u32(&S.ST[0][0][0]), &smap, j0, m * (sp.ny + 4) + 2 + t0 * TY, b);
    }
    tile::setup_cols(S.C, ep, sp.nx, j0, oj, [](int a) { return a; });
    if (warp == kWarps - 1) qh_rows(S.R[0], ep, sp.ny, t0 * TY, ok, ring);
    __syncthreads();
    qh_xpass(S.C, ep, cf, X, ring, S.R[0].rg_u[0] - 1, S.R[0].u_last);
    if (warp == 0 && nt > 1) qh_rows(S.R[1], ep, sp.ny, (t0 + 1) * TY, ok, ring);
    __syncthreads();
    qh_ypass(S.R[0], X, S.D[0]);
    bool dry = false;
    int dry_at = 0x7fffffff;
    float mx_u = 0.0f, mx_v = 0.0f, mn_h = 3.402823466e+38f;
    const double cy = ep.cy, cx = ep.cx, heq = ep.h_eq;
    for (int i = 0; i < nt; ++i) {
        __syncthreads();  // D of tile i complete; tile i+1's row tables published
        const int k0 = (t0 + i) * TY;
        if (i + 1 < nt) qh_xpass(S.C, ep, cf, X, ring, S.R[i % 3].u_last + 1, S.R[(i + 1) % 3].u_last);
        // tile i+2's row tables (into the buffer tile i-1 used) on a warp with one row fewer
        if (warp == kWarps - 1 && i + 2 < nt) qh_rows(S.R[(i + 2) % 3], ep, sp.ny, k0 + 2 * TY, ok, ring);
        // geostrophic balance (stochastic.hpp:122-139) + add in fp64, cast to float
        mbar_wait(b, i & 1);
        const double(*D)[tile::XW] = S.D[i & 1];
        // cells within 2 of a domain edge also go to their ghost copies, so
        // the next model step needs no fix_ghosts pass; interior tiles skip that (uniform)
        const bool edge = j0 < 2 || j0 + TX > sp.nx - 2 || k0 < 2 || k0 + TY > sp.ny - 2;
        const int cell0 = (k0 + ty) * static_cast<int>(pitch) + j;  // offset in the member
#pragma unroll
        for (int q = 0; q < kRowsPerThread; ++q) {
            const int r = ty + kWarps * q;
            if (!((r < TY) && (k0 + r < sp.ny) && (j < sp.nx))) continue;
            const int rr = r + 1, jl = tx + 1;
            const double de = D[rr][jl];
            const double dhu = -cy * (D[rr + 1][jl] - D[rr - 1][jl]);
            const double dhv = cx * (D[rr][jl + 1] - D[rr][jl - 1]);
            const float s0 = S.ST[0][r][tx + 2], s1 = S.ST[1][r][tx + 2], s2 = S.ST[2][r][tx + 2];
            const double e = static_cast<double>(s0) + (UNIT ? de : scale * de);
            if (!(heq + e > 0.0)) {
                dry = true;
                dry_at = min(dry_at, (k0 + r) * sp.nx + j);
            }
            const float fe = static_cast<float>(e);
            const float fu = static_cast<float>(static_cast<double>(s1) + (UNIT ? dhu : scale * dhu));
            const float fv = static_cast<float>(static_cast<double>(s2) + (UNIT ? dhv : scale * dhv));
            const int o = cell0 + q * kWarps * static_cast<int>(pitch);
            Em[o] = fe;
            Um[o] = fu;
            Vm[o] = fv;
            if (edge) {
                const int kk = k0 + r;
                const int gc = j < 2 ? sp.nx : (j >= sp.nx - 2 ? -sp.nx : 0);
                const int gr = kk < 2 ? sp.ny : (kk >= sp.ny - 2 ? -sp.ny : 0);
                if (gc) {
                    Em[o + gc] = fe;
                    Um[o + gc] = fu;
                    Vm[o + gc] = fv;
                }
                if (gr) {
                    const int g = gr * static_cast<int>(pitch);
                    Em[o + g] = fe;
                    Um[o + g] = fu;
                    Vm[o + g] = fv;
                    if (gc) {
                        Em[o + g + gc] = fe;
                        Um[o + g + gc] = fu;
                        Vm[o + g + gc] = fv;
                    }
                }
            }
            if (mx) {  // load() statistics of the new state, IEEE float (swe.hpp:307-316)
                const float h = __fadd_rn(sp.H, fe);
                mn_h = fminf(mn_h, h);
                const float inv = rcp_rn(h);
                const float c = sqrt_rn(__fmul_rn(sp.g, fmaxf(h, 0.0f)));
                mx_u = fmaxf(mx_u, __fadd_rn(fabsf(__fmul_rn(fu, inv)), c));
                mx_v = fmaxf(mx_v, __fadd_rn(fabsf(__fmul_rn(fv, inv)), c));
            }
        }
        __syncthreads();  // the state box is consumed; tile i+1's new X rows are complete
        if (i + 1 < nt) {
            if (tid == 0) {
                mbar_expect_tx(b, sizeof(S.ST));
                tma_row(smem_u32(&S.ST[0][0][0]), &smap, j0, m * (sp.ny + 4) + 2 + k0 + TY, b);
            }
            qh_ypass(S.R[(i + 1) % 3], X, S.D[(i + 1) & 1]);
        }
    }
    if (dry) {
        atomicCAS(err + m, 0, E_DRY_ADD);
        atomicMin(err_pos + m, dry_at);
    }
    if (mx) {
        // warp maxima / minimum in one CREDUX each (order-free: max / min are exact)
        float a_, b_, c_;
        asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(a_) : "f"(mx_u));
        asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(b_) : "f"(mx_v));
        asm("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(c_) : "f"(mn_h));
        if (tx == 0) {
            S.red[0][ty] = a_;
            S.red[1][ty] = b_;
            S.red[2][ty] = c_;
        }
        __syncthreads();
        if (tid == 0) {
            float a = S.red[0][0], bb = S.red[1][0], c = S.red[2][0];
            for (int w = 1; w < kWarps; ++w) {
                a = fmaxf(a, S.red[0][w]);
                bb = fmaxf(bb, S.red[1][w]);
                c = fminf(c, S.red[2][w]);
            }
            atomicMax(mx + 4 * m + 0, __float_as_uint(a));
            atomicMax(mx + 4 * m + 1, __float_as_uint(bb));
            atomicMin(mx + 4 * m + 2, ordered_bits(c));
        }
    }
}

} // namespace

void launch_philox_noise(cudaStream_t s, const ErrParams& ep, int M, uint64_t seed, uint64_t tag,
                         int64_t member_base, uint32_t substream, uint64_t draw, double* xi,
                         int* offsets, const int* err) {
    const int npairs = (ep.nxc * ep.nyc + 1) / 2;
    int bx = (npairs + 255) / 256;
    KScope ks(s, "philox_noise", 8.0 * ep.nxc * ep.nyc * M);
    philox_noise_kernel<<<dim3(bx, M), 256, 0, s>>>(ep, M, seed, tag, member_base, substream,
                                                    draw, xi, offsets, err);
}

void launch_philox_soar(cudaStream_t s, const ErrParams& ep, int M, uint64_t seed, uint64_t tag,
                        int64_t member_base, uint32_t substream, uint64_t draw, double* corr,
                        int* offsets, const int* err) {
    const size_t bytes = static_cast<size_t>(kBand + 4) * ep.nxc * sizeof(double);
    smem_opt_in(philox_soar_kernel, 200 * 1024);
    KScope ks(s, "philox_soar", 8.0 * ep.nxc * ep.nyc * M);  // xi stays on chip
    philox_soar_kernel<<<dim3((ep.nyc + kBand - 1) / kBand, M), 256, bytes, s>>>(
        ep, M, seed, tag, member_base, substream, draw, corr, offsets, err);
}

void launch_coarse_soar(cudaStream_t s, const ErrParams& ep, int M, const double* in,
                        double* out, const int* err) {
    const int nr = ep.nxc * ep.nyc;
    KScope ks(s, "coarse_soar", 16.0 * nr * M);
    coarse_soar_kernel<<<dim3((nr + 255) / 256, M), 256, 0, s>>>(ep, M, in, out, err);
}

void launch_q_half_apply(cudaStream_t s, const CUtensorMap* smap, const SweParams& sp,
                         const ErrParams& ep, const double* corr, const int* offsets,
                         double scale, float* eta, float* hu, float* hv, int* err,
                         int* err_pos, int M, unsigned* mx, const char* prof_name) {
    // strips of S tiles: long enough to amortise the strip prologue, short enough to keep
    // >= ~8 waves of resident CTAs
    const int tiles_x = (sp.nx + TX - 1) / TX, tiles_y = (sp.ny + TY - 1) / TY;
    const double slots = 148.0 * DC_QHALF_MIN_BLOCKS;
    int S = static_cast<int>(static_cast<double>(tiles_x) * tiles_y * M / (DC_QHALF_WAVES * slots));
    S = S < 1 ? 1 : (S > tiles_y ? tiles_y : S);
    const int strips = (tiles_y + S - 1) / S;
    S = (tiles_y + strips - 1) / strips;  // balance the strips
    dim3 grid(tiles_x, strips, M);
    // < 48 KB for every c_omega (ring <= 37 rows): no opt-in
    const size_t smem = sizeof(QhSmem) + static_cast<size_t>(qh_ring(ep.c)) * tile::XW * sizeof(double);
    // the state read and written once (24 B/cell) + the coarse field
    KScope ks(s, prof_name,
              (24.0 * sp.nx * sp.ny + 8.0 * ep.nxc * ep.nyc) * M);
    if (scale == 1.0) {
        q_half_apply_kernel<true><<<grid, tile::NT, smem, s>>>(*smap, sp, ep, corr, offsets, scale,
                                                            eta, hu, hv, err, err_pos, mx, S);
    } else {
        q_half_apply_kernel<false><<<grid, tile::NT, smem, s>>>(*smap, sp, ep, corr, offsets, scale,
                                                             eta, hu, hv, err, err_pos, mx, S);
    }
}

} // namespace dcg
