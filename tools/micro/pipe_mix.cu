// Issue rate of an FFMA2 + FMNMX3 + FMNMX mix on sm_100a at several warps per SM
// (development aid): what a dependency-light stream of the stencil's instruction mix
// (packed FP32 on the fma-heavy pipe, 3-input / 2-input min-max on the alu pipe) can
// reach, to compare with the stage kernels' 61 % issue / 62 % fma-pipe utilisation.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 6, kIters = 2048;

template <int MIX>
__global__ void k(float2* out, float2 p, float2 nz) {
    float2 d[kChains];
    float m[kChains];
    float2 x = make_float2(threadIdx.x * 1e-7f + 1.0f, 1.0f - threadIdx.x * 1e-7f);
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        d[c] = make_float2(c * 0.1f, c * 0.2f);
        m[c] = c;
    }
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            d[c] = __ffma2_rn(d[c], x, nz);                   // fma-heavy, 2 cycles
            if (MIX >= 1) {                                   // + alu: 3-input min/max
                float r;
                asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(m[c]), "f"(d[c].x), "f"(p.x));
                m[c] = r;
            }
            if (MIX >= 2) d[c] = __fadd2_rn(d[c], p);         // second packed op
            if (MIX >= 3) m[c] = fminf(m[c], d[c].y);         // 2-input min
        }
    }
    float2 s = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < kChains; ++c) s = make_float2(s.x + d[c].x + m[c], s.y + d[c].y);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MIX>
void run(float2* out, int ctas_per_sm, int threads) {
    const int blocks = 148 * ctas_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float2 p = make_float2(0.999f, 0.998f), nz = make_float2(-0.0f, -0.0f);
    k<MIX><<<blocks, threads>>>(out, p, nz);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<MIX><<<blocks, threads>>>(out, p, nz);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const int per_iter = 1 + (MIX >= 1) + (MIX >= 2) + (MIX >= 3);
    const int fma_per_iter = 1 + (MIX >= 2);
    const double warps = 5.0 * blocks * threads / 32.0;
    const double inst = warps * kIters * kChains * per_iter;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double smsp_cycles = ms * 1e-3 * clk * 1e3 * 148 * 4;
    const double fma_cycles = warps * kIters * kChains * fma_per_iter * 2;
    std::printf("mix %d  warps/SM %3d : issue %.2f inst/cycle/SMSP, fma pipe %.2f\n", MIX,
                ctas_per_sm * threads / 32, inst / smsp_cycles, fma_cycles / smsp_cycles);
}

int main() {
    float2* out;
    cudaMalloc(&out, 148 * 32 * 1024 * sizeof(float2));
    for (int w : {4, 8, 12, 16, 24}) {
        run<0>(out, w / 4, 128);
        run<1>(out, w / 4, 128);
        run<2>(out, w / 4, 128);
        run<3>(out, w / 4, 128);
    }
    return 0;
}
