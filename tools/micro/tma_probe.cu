// TMA probe (development aid): 3-D box loads with the stage kernel's PTX helpers.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

struct Maps { CUtensorMap a, w; };

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ unsigned g_wbytes;
template <int MODE>
__global__ void probe(const __grid_constant__ Maps mp, const CUtensorMap* gmap, float* out, int c0, int r) {
    extern __shared__ __align__(128) unsigned char sm[];
    float* buf = reinterpret_cast<float*>(sm + 128);
    uint32_t bar = smem_u32(sm);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(1) : "memory");
        if (MODE & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((MODE & 8) ? 3072u + g_wbytes : (MODE & 16) ? g_wbytes : 3072u) : "memory");
        if (MODE & 24) {
            const uint64_t wmap = (MODE & 4) ? reinterpret_cast<uint64_t>(gmap + 1) : reinterpret_cast<uint64_t>(&mp.w);
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(smem_u32(buf) + 3072), "l"(wmap), "r"(c0 + 10), "r"(r), "r"(0), "r"(bar) : "memory");
        }
        const uint64_t map = (MODE & 4) ? reinterpret_cast<uint64_t>(gmap) : reinterpret_cast<uint64_t>(&mp.a);
        if (MODE & 16) {}
        else if (MODE & 32)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(smem_u32(buf)), "l"(reinterpret_cast<uint64_t>(&mp.w)), "r"(c0), "r"(r), "r"(0), "r"(bar) : "memory");
        else if (MODE & 2)
            asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(smem_u32(buf)), "l"(map), "r"(c0), "r"(r), "r"(0), "r"(bar) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(smem_u32(buf)), "l"(map), "r"(c0), "r"(r), "r"(0), "r"(bar) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(bar), "r"(0) : "memory");
    for (int i = threadIdx.x; i < 768; i += blockDim.x) out[i] = (MODE & 16) ? 0.f : buf[i];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

#include <cstdlib>
int main(int argc, char** argv) {
    const int nx = 500, rows = 600, pitch = 512;
    const size_t fs = (size_t)rows * pitch;
    std::vector<float> h(3 * fs);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float* d; cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    float* o; cudaMalloc(&o, 768 * 4);
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    Enc enc = (Enc)p;
    Maps mp;
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)rows, 3};
    cuuint64_t str[2] = {(cuuint64_t)pitch * 4, (cuuint64_t)fs * 4};
    cuuint32_t box[3] = {256, 1, 3}, es[3] = {1, 1, 1};
    CUresult rc = enc(&mp.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)rc);
    const int ww = argc > 3 ? atoi(argv[3]) : 4;
    cuuint32_t boxw[3] = {(cuuint32_t)ww, 1, 3};
    rc = enc(&mp.w, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, boxw, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode w rc=%d\n", (int)rc);
    CUtensorMap* gm; cudaMalloc(&gm, 2 * sizeof(CUtensorMap)); cudaMemcpy(gm, &mp.a, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    cudaMemcpy(gm + 1, &mp.w, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    const int mode = atoi(argv[1]);
    { unsigned wb = ww * 12; cudaMemcpyToSymbol(g_wbytes, &wb, 4); }
    const int c0 = atoi(argv[2]);
    {
        void (*ks[32])(Maps, const CUtensorMap*, float*, int, int) = {probe<0>, probe<1>, probe<2>, probe<3>, probe<4>, probe<5>, probe<6>, probe<7>,
        probe<8>, probe<9>, probe<10>, probe<11>, probe<12>, probe<13>, probe<14>, probe<15>, probe<16>, probe<17>, probe<18>, probe<19>, probe<20>, probe<21>, probe<22>, probe<23>,
        probe<24>, probe<25>, probe<26>, probe<27>, probe<28>, probe<29>, probe<30>, probe<31>};
    void (*k2)(Maps, const CUtensorMap*, float*, int, int) = mode == 20 ? probe<20> : mode == 32 ? probe<32> : mode == 36 ? probe<36> : nullptr;
        void (*k)(Maps, const CUtensorMap*, float*, int, int) = k2 ? k2 : ks[mode];
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096);
        k<<<1, 128, 4096>>>(mp, gm, o, c0, 7);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> r(768);
        cudaMemcpy(r.data(), o, 768 * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int f = 0; f < 3; ++f) for (int c = 0; c < 256; ++c) {
            int col = c + c0; float want = (col < 0 || col >= nx) ? 0.f : h[f * fs + 7 * pitch + col];
            if (r[f * 256 + c] != want) ++bad;
        }
        printf("mode %d: %s, mismatches %d\n", mode, cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
