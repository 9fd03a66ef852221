// Throughput of packed FP32 instruction forms on sm_100a (development aid): FFMA2 with
// three vector registers, with a kernel-parameter addend, FMUL2, FADD2, scalar FFMA.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8, kIters = 4096;

template <int FORM>
__global__ void __launch_bounds__(256) k(float2* out, float2 p, float2 q, float2 nz) {
    float2 d[kChains];
    float2 x = make_float2(threadIdx.x * 1e-7f + 1.0f, 1.0f - threadIdx.x * 1e-7f);
    float2 y = make_float2(p.x + threadIdx.x * 1e-9f, p.y - threadIdx.x * 1e-9f);
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c] = make_float2(c * 0.1f, c * 0.2f);
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (FORM == 0) d[c] = __ffma2_rn(d[c], x, y);        // R, R, R
            if (FORM == 1) d[c] = __ffma2_rn(d[c], x, nz);       // R, R, param
            if (FORM == 2) d[c] = __fmul2_rn(d[c], x);           // FMUL2
            if (FORM == 3) d[c] = __fadd2_rn(d[c], y);           // FADD2
            if (FORM == 4) d[c] = __ffma2_rn(d[c], q, y);        // R, param, R
            if (FORM == 5) {                                      // scalar FFMA x2
                d[c].x = __fmaf_rn(d[c].x, x.x, y.x);
                d[c].y = __fmaf_rn(d[c].y, x.y, y.y);
            }
        }
    }
    float2 s = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < kChains; ++c) s = make_float2(s.x + d[c].x, s.y + d[c].y);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int FORM>
void run(const char* name, float2* out) {
    const int blocks = 148 * 8;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float2 p = make_float2(0.999f, 0.998f), q = make_float2(1.0001f, 0.9999f), nz = make_float2(-0.0f, -0.0f);
    k<FORM><<<blocks, 256>>>(out, p, q, nz);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<FORM><<<blocks, 256>>>(out, p, q, nz);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double inst = 5.0 * blocks * 8.0 /*warps*/ * kIters * kChains * (FORM == 5 ? 2 : 1);
    const double lane_ops = 5.0 * blocks * 256.0 * kIters * kChains * 2;
    printf("%-28s %8.3f ms  %7.2f T warp-inst/s  %7.2f T lane-ops/s\n", name, ms / 5,
           inst / (ms / 1e3) / 5 / 1e12 * 5, lane_ops / (ms / 1e3) / 1e12);
}

int main() {
    float2* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(float2));
    run<0>("FFMA2 R,R,R", out);
    run<1>("FFMA2 R,R,param(-0)", out);
    run<4>("FFMA2 R,param,R", out);
    run<2>("FMUL2 R,R", out);
    run<3>("FADD2 R,R", out);
    run<5>("2x FFMA R,R,R", out);
    return 0;
}
