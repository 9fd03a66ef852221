// guard.cu -- guard-banded device allocations (DC_GUARD=1): the memory checker of this
// repo. compute-sanitizer is not available on the GPU pool, so every device buffer of the
// library can be allocated with 64 KB guard bands on both sides, filled with a byte
// pattern, and the user region poisoned with 0xFF bytes (NaN floats / doubles, -1 ints),
// so that
//   * an out-of-bounds WRITE by any kernel changes a guard band -> dc_check_guards()
//     names the buffer (allocation site) and the first corrupted offset;
//   * an out-of-bounds or uninitialised READ feeds NaN / garbage into the arithmetic ->
//     the bitwise comparisons against the CPU oracle fail.
// Without DC_GUARD the allocator is plain cudaMalloc / cudaFree.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "dc_internal.h"

namespace dcg {

namespace {
constexpr size_t kGuard = 64 * 1024;
constexpr unsigned char kPattern = 0xA5;

struct Alloc {
    size_t bytes;
    const char* file;
    int line;
};

std::mutex g_mu;
std::map<char*, Alloc>& registry() {  // user pointer -> allocation
    static std::map<char*, Alloc> r;
    return r;
}

bool guard_mode() {
    static const bool on = [] {
        const char* e = std::getenv("DC_GUARD");
        return e && e[0] == '1';
    }();
    return on;
}
}  // namespace

cudaError_t dmalloc_impl(void** p, size_t bytes, const char* file, int line) {
    if (!guard_mode()) return cudaMalloc(p, bytes);
    char* base = nullptr;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&base), bytes + 2 * kGuard);
    if (e != cudaSuccess) return e;
    // the fills run on the legacy stream, which the library's non-blocking streams do not
    // wait for: finish them before any stream can touch the buffer -- by synchronising that
    // stream only (a device-wide synchronisation would also wait for other contexts' work,
    // which in a multi-rank process may be waiting for this rank's collective)
    if ((e = cudaMemsetAsync(base, kPattern, kGuard, cudaStreamLegacy)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(base + kGuard, 0xFF, bytes, cudaStreamLegacy)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(base + kGuard + bytes, kPattern, kGuard, cudaStreamLegacy)) != cudaSuccess)
        return e;
    if ((e = cudaStreamSynchronize(cudaStreamLegacy)) != cudaSuccess) return e;
    char* user = base + kGuard;
    std::lock_guard<std::mutex> lk(g_mu);
    registry()[user] = Alloc{bytes, file, line};
    *p = user;
    return cudaSuccess;
}

cudaError_t dfree(void* p) {
    if (!p) return cudaSuccess;
    if (guard_mode()) {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = registry().find(static_cast<char*>(p));
        if (it != registry().end()) {
            registry().erase(it);
            return cudaFree(static_cast<char*>(p) - kGuard);
        }
    }
    return cudaFree(p);
}

// Checks every live guard band (synchronises the device). Returns the number of corrupted
// allocations and describes the first ones in msg.
int check_guards(std::string* msg) {
    if (!guard_mode()) return 0;
    cudaDeviceSynchronize();
    std::lock_guard<std::mutex> lk(g_mu);
    std::vector<unsigned char> h(kGuard);
    int bad = 0;
    for (auto& [user, a] : registry()) {
        int dev = -1;
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, user) == cudaSuccess) dev = at.device;
        int prev = -1;
        cudaGetDevice(&prev);
        if (dev >= 0 && dev != prev) cudaSetDevice(dev);
        for (int side = 0; side < 2; ++side) {
            const char* g = side == 0 ? user - kGuard : user + a.bytes;
            if (cudaMemcpy(h.data(), g, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) continue;
            for (size_t i = 0; i < kGuard; ++i)
                if (h[i] != kPattern) {
                    if (bad < 8) {
                        char b[256];
                        std::snprintf(b, sizeof(b), "%s:%d (%zu B): %s guard band written at %s%zu B; ",
                                      a.file, a.line, a.bytes, side ? "upper" : "lower",
                                      side ? "+" : "-", side ? i : kGuard - i);
                        *msg += b;
                    }
                    ++bad;
                    break;
                }
        }
        if (dev >= 0 && dev != prev) cudaSetDevice(prev);
    }
    return bad;
}

}  // namespace dcg
