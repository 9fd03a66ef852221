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

constexpr int TX = 32, TY = 16;
constexpr int NBMAX = TY + 2 + 3;  // coarse rows a tile can touch (c_omega = 1 worst case)

// Fine-row -> coarse-row bookkeeping of interpolate_bicubic (stochastic.hpp:97-102),
// computed from the WRAPPED fine index exactly as the reference does.
__device__ __forceinline__ void row_coords(const ErrParams& ep, int kk, int ok, int* b0, double* ty) {
    const double yc = static_cast<double>(kk - ok) * ep.inv_c;
    *b0 = static_cast<int>(floor(yc));
    *ty = yc - *b0;
}

// Q^{1/2} tail + add (stochastic.hpp:144-160) for one (member, 32x16 tile).
__global__ void __launch_bounds__(256)
q_half_apply_kernel(SweParams sp, ErrParams ep, const double* __restrict__ corr,
                    const int* __restrict__ offsets, double scale, float* eta, float* hu,
                    float* hv, int* err, int* err_pos) {
    __shared__ double X[NBMAX][TX + 2];
    __shared__ double D[TY + 2][TX + 2];
    const int m = blockIdx.z;
    if (err[m]) return;
    const int j0 = blockIdx.x * TX, k0 = blockIdx.y * TY;
    const int oj = offsets[2 * m], ok = offsets[2 * m + 1];
    const double* cf = corr + static_cast<size_t>(m) * ep.nxc * ep.nyc;
    const int tid = threadIdx.x;

    // coarse-row window of this tile
    int bfirst, blast;
    double tdummy;
    row_coords(ep, wrapi(k0 - 1, sp.ny), ok, &bfirst, &tdummy);
    row_coords(ep, wrapi(k0 + TY, sp.ny), ok, &blast, &tdummy);
    const bool whole = ep.nyc <= NBMAX;
    const int bstart = whole ? 0 : wrapi(bfirst - 1, ep.nyc);
    const int nb = whole ? ep.nyc : wrapi(blast - bfirst, ep.nyc) + 4;

    // pass 1: x-interpolation of the needed coarse rows at the tile's fine columns
    for (int i = tid; i < nb * (TX + 2); i += blockDim.x) {
        const int s = i / (TX + 2), jl = i % (TX + 2);
        const int b = whole ? s : wrap1(bstart + s, ep.nyc);
        const int jw = wrap1(j0 - 1 + jl, sp.nx);
        const double xc = static_cast<double>(jw - oj) * ep.inv_c;
        const int a0 = static_cast<int>(floor(xc));
        const double tx = xc - a0;
        const double* row = cf + b * ep.nxc;
        X[s][jl] = det::catmull(__ldg(row + det::wrapf(a0 - 1, ep.nxc)), __ldg(row + det::wrapf(a0, ep.nxc)),
                                __ldg(row + det::wrapf(a0 + 1, ep.nxc)), __ldg(row + det::wrapf(a0 + 2, ep.nxc)),
                                tx);
    }
    __syncthreads();
    // pass 2: y-interpolation -> delta eta on the tile + 1-cell halo
    for (int i = tid; i < (TY + 2) * (TX + 2); i += blockDim.x) {
        const int r = i / (TX + 2), jl = i % (TX + 2);
        const int kk = wrap1(k0 - 1 + r, sp.ny);
        int b0;
        double ty;
        row_coords(ep, kk, ok, &b0, &ty);
        int sl[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int b = det::wrapf(b0 - 1 + q, ep.nyc);
            sl[q] = whole ? b : det::wrapf(b - bstart, ep.nyc);
        }
        D[r][jl] = det::catmull(X[sl[0]][jl], X[sl[1]][jl], X[sl[2]][jl], X[sl[3]][jl], ty);
    }
    __syncthreads();
    // pass 3: geostrophic balance (stochastic.hpp:122-139) + add in fp64, cast to float
    bool dry = false;
    int dry_at = 0x7fffffff;
    const size_t mbase = static_cast<size_t>(m) * sp.ny * sp.pitch;
    for (int i = tid; i < TY * TX; i += blockDim.x) {
        const int r = i / TX + 1, jl = i % TX + 1;
        const int k = k0 + r - 1, j = j0 + jl - 1;
        if (k >= sp.ny || j >= sp.nx) continue;
        const double de = D[r][jl];
        const double dhu = -ep.cy * (D[r + 1][jl] - D[r - 1][jl]);
        const double dhv = ep.cx * (D[r][jl + 1] - D[r][jl - 1]);
        const size_t o = mbase + static_cast<size_t>(k) * sp.pitch + j;
        const double e = static_cast<double>(eta[o]) + scale * de;
        if (!(ep.h_eq + e > 0.0)) {
            dry = true;
            dry_at = min(dry_at, k * sp.nx + j);
        }
        eta[o] = static_cast<float>(e);
        hu[o] = static_cast<float>(static_cast<double>(hu[o]) + scale * dhu);
        hv[o] = static_cast<float>(static_cast<double>(hv[o]) + scale * dhv);
    }
    if (dry) {
        atomicCAS(err + m, 0, E_DRY_ADD);
        atomicMin(err_pos + m, dry_at);
    }
}

} // namespace

void launch_philox_noise(cudaStream_t s, const ErrParams& ep, int M, uint64_t seed, uint64_t tag,
                         int64_t member_base, uint32_t substream, uint64_t draw, double* xi,
                         int* offsets, const int* err) {
    const int npairs = (ep.nxc * ep.nyc + 1) / 2;
    int bx = (npairs + 255) / 256;
    philox_noise_kernel<<<dim3(bx, M), 256, 0, s>>>(ep, M, seed, tag, member_base, substream,
                                                    draw, xi, offsets, err);
}

void launch_coarse_soar(cudaStream_t s, const ErrParams& ep, int M, const double* in,
                        double* out, const int* err) {
    const int nr = ep.nxc * ep.nyc;
    coarse_soar_kernel<<<dim3((nr + 255) / 256, M), 256, 0, s>>>(ep, M, in, out, err);
}

void launch_q_half_apply(cudaStream_t s, const SweParams& sp, const ErrParams& ep,
                         const double* corr, const int* offsets, double scale, float* eta,
                         float* hu, float* hv, int* err, int* err_pos, int M) {
    dim3 grid((sp.nx + TX - 1) / TX, (sp.ny + TY - 1) / TY, M);
    q_half_apply_kernel<<<grid, 256, 0, s>>>(sp, ep, corr, offsets, scale, eta, hu, hv, err,
                                             err_pos);
}

} // namespace dcg
