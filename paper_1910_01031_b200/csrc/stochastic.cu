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
#ifndef DC_QHALF_MIN_BLOCKS
#define DC_QHALF_MIN_BLOCKS 6
#endif

// The tile's state arrives by TMA: one box {TX+4 columns from cell j0-2, TY rows, 3 fields}
// of the state set's map (storage column j0 is 16-byte aligned; the box's first two and
// last two columns are not used).
constexpr int kStw = TX + 4;
static_assert(kStw * sizeof(float) % 16 == 0, "TMA box rows must be 16-byte multiples");

// UNIT: scale == 1.0 (model error, posterior): scale * x == x exactly, so the three
// products are dropped (bitwise the same)
template <bool UNIT>
__global__ void __launch_bounds__(tile::NT, DC_QHALF_MIN_BLOCKS)
q_half_apply_kernel(const __grid_constant__ CUtensorMap smap, SweParams sp, ErrParams ep,
                    const double* __restrict__ corr, const int* __restrict__ offsets,
                    double scale, float* eta, float* hu, float* hv, int* err, int* err_pos,
                    unsigned* mx) {
    __shared__ tile::Smem S;
    __shared__ alignas(128) float ST[3][TY][kStw];
    __shared__ float red[3][kWarps];
    __shared__ alignas(8) unsigned long long bar;
    const int m = blockIdx.z;
    // another tile of the member may raise E_DRY_ADD meanwhile: decide once per CTA
    if (__syncthreads_or(err[m] != 0)) return;
    const int j0 = blockIdx.x * TX, k0 = blockIdx.y * TY;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int j = j0 + tx;
    const size_t pitch = sp.pitch;
    // this thread's cells: column j, rows k0 + ty + 8q
    const size_t cell0 = static_cast<size_t>(m) * sp.mstride + static_cast<size_t>(k0 + ty) * pitch + j;
    const size_t step = static_cast<size_t>(kWarps) * pitch;
    const uint32_t b = smem_u32(&bar);
    if (threadIdx.x == 0) {
        mbar_init(b, 1);
        mbar_fence_init();
        mbar_expect_tx(b, sizeof(ST));
        // storage row of cell row k0 of member m (the map starts at row -2 of member 0)
        tma_row(smem_u32(&ST[0][0][0]), &smap, j0, m * (sp.ny + 4) + 2 + k0, b);
    }
    const int oj = offsets[2 * m], ok = offsets[2 * m + 1];
    const double* cf = corr + static_cast<size_t>(m) * ep.nxc * ep.nyc;
    const int nxc = ep.nxc;
    tile::setup(S, ep, sp.nx, sp.ny, j0, k0, oj, ok, [](int a) { return a; },
                [&](int bb) { return bb * nxc; });  // (its barrier publishes the mbarrier)
    tile::interpolate(S, [&](int brow, int a) { return __ldg(cf + brow + a); });
    // geostrophic balance (stochastic.hpp:122-139) + add in fp64, cast to float
    bool dry = false;
    int dry_at = 0x7fffffff;
    float mx_u = 0.0f, mx_v = 0.0f, mn_h = 3.402823466e+38f;
    const double cy = ep.cy, cx = ep.cx, heq = ep.h_eq;
    mbar_wait(b, 0);
    // cells within 2 of a domain edge also go to their ghost copies, so the
    // next model step needs no fix_ghosts pass; interior tiles skip that (uniform branch)
    const bool edge = j0 < 2 || j0 + TX > sp.nx - 2 || k0 < 2 || k0 + TY > sp.ny - 2;
#pragma unroll
    for (int q = 0; q < kRowsPerThread; ++q) {
        const int r = ty + kWarps * q;
        if (!((r < TY) && (k0 + r < sp.ny) && (j < sp.nx))) continue;
        const int rr = r + 1, jl = tx + 1;
        const double de = S.D[rr][jl];
        const double dhu = -cy * (S.D[rr + 1][jl] - S.D[rr - 1][jl]);
        const double dhv = cx * (S.D[rr][jl + 1] - S.D[rr][jl - 1]);
        const double e = static_cast<double>(ST[0][r][tx + 2]) + (UNIT ? de : scale * de);
        if (!(heq + e > 0.0)) {
            dry = true;
            dry_at = min(dry_at, (k0 + r) * sp.nx + j);
        }
        const float fe = static_cast<float>(e);
        const float fu = static_cast<float>(static_cast<double>(ST[1][r][tx + 2]) +
                                            (UNIT ? dhu : scale * dhu));
        const float fv = static_cast<float>(static_cast<double>(ST[2][r][tx + 2]) +
                                            (UNIT ? dhv : scale * dhv));
        const size_t o = cell0 + q * step;
        eta[o] = fe;
        hu[o] = fu;
        hv[o] = fv;
        if (edge) {
            const int kk = k0 + r;
            const ptrdiff_t gc = j < 2 ? sp.nx : (j >= sp.nx - 2 ? -sp.nx : 0);
            const ptrdiff_t gr = kk < 2 ? sp.ny : (kk >= sp.ny - 2 ? -sp.ny : 0);
            if (gc) {
                eta[o + gc] = fe;
                hu[o + gc] = fu;
                hv[o + gc] = fv;
            }
            if (gr) {
                const ptrdiff_t g = gr * static_cast<ptrdiff_t>(pitch);
                eta[o + g] = fe;
                hu[o + g] = fu;
                hv[o + g] = fv;
                if (gc) {
                    eta[o + g + gc] = fe;
                    hu[o + g + gc] = fu;
                    hv[o + g + gc] = fv;
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
            red[0][ty] = a_;
            red[1][ty] = b_;
            red[2][ty] = c_;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            float a = red[0][0], bb = red[1][0], c = red[2][0];
            for (int i = 1; i < kWarps; ++i) {
                a = fmaxf(a, red[0][i]);
                bb = fmaxf(bb, red[1][i]);
                c = fminf(c, red[2][i]);
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
    dim3 grid((sp.nx + TX - 1) / TX, (sp.ny + TY - 1) / TY, M);
    // the state read and written once (24 B/cell) + the coarse field
    KScope ks(s, prof_name,
              (24.0 * sp.nx * sp.ny + 8.0 * ep.nxc * ep.nyc) * M);
    if (scale == 1.0)
        q_half_apply_kernel<true><<<grid, tile::NT, 0, s>>>(*smap, sp, ep, corr, offsets, scale,
                                                            eta, hu, hv, err, err_pos, mx);
    else
        q_half_apply_kernel<false><<<grid, tile::NT, 0, s>>>(*smap, sp, ep, corr, offsets, scale, eta, hu,
                                                  hv, err, err_pos, mx);
}

} // namespace dcg
