// Back-to-back dependent launch cost on one stream (development aid): N launches of a
// kernel of G CTAs x 128 threads that does almost nothing, timed with CUDA events, plus
// the same inside a CUDA graph. Usage: launch_gap [G]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void tiny(int* p) {
    if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}

int main(int argc, char** argv) {
    const int G = argc > 1 ? std::atoi(argv[1]) : 2400;
    const int N = 200;
    int* p;
    cudaMalloc(&p, 4);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 10; ++i) tiny<<<G, 128, 0, s>>>(p);
    cudaEventRecord(a, s);
    for (int i = 0; i < N; ++i) tiny<<<G, 128, 0, s>>>(p);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::printf("stream: %d CTAs: %.2f us per launch\n", G, 1e3 * ms / N);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) tiny<<<G, 128, 0, s>>>(p);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    std::printf("graph : %d CTAs: %.2f us per launch\n", G, 1e3 * ms / N);
    return 0;
}
