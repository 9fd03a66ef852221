// kprof.cu -- per-kernel timing for the roofline table (dc_profile_begin / dc_profile_end).
//
// While a profile window is open on the calling host thread, every launcher's KScope
// brackets its kernel with two CUDA events on the launch stream and records the kernel's
// algorithmic HBM bytes (the launcher knows its sizes). Launches inside a stream capture
// are not bracketed (dc_step uses its host-driven substep loop while profiling, so the
// stage kernels are launched, and timed, one by one). Each interval is the kernel's own
// device time: the events sit directly before and after it on the same stream.
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "dc_internal.h"

namespace dcg {

struct KProf {
    struct Rec {
        const char* name;
        double bytes;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;  // events created for this window
    size_t used = 0;
    cudaEvent_t take() {
        if (used == pool.size()) {
            cudaEvent_t e = nullptr;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        return pool[used++];
    }
};

thread_local KProf* g_kprof = nullptr;

namespace {
bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone;
}
} // namespace

bool kprof_active() { return g_kprof != nullptr; }

KScope::KScope(cudaStream_t s_, const char* name_, double bytes_) : s(s_), rec(-1) {
    if (!g_kprof || capturing(s)) return;
    KProf::Rec r{name_, bytes_, g_kprof->take(), g_kprof->take()};
    cudaEventRecord(r.a, s);
    rec = static_cast<int>(g_kprof->recs.size());
    g_kprof->recs.push_back(r);
}

KScope::~KScope() {
    if (rec >= 0 && g_kprof) cudaEventRecord(g_kprof->recs[rec].b, s);
}

void kprof_begin() {
    delete g_kprof;
    g_kprof = new KProf();
}

// Ends the window: synchronises the recorded events and folds them per kernel name
// (first-seen order).
int kprof_end(dc_kernel_time* out, int cap) {
    KProf* p = g_kprof;
    g_kprof = nullptr;
    if (!p) return 0;
    std::vector<std::string> order;
    std::map<std::string, dc_kernel_time> acc;
    for (const KProf::Rec& r : p->recs) {
        cudaEventSynchronize(r.b);
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        const std::string n(r.name);
        auto it = acc.find(n);
        if (it == acc.end()) {
            dc_kernel_time k{};
            std::strncpy(k.name, r.name, sizeof(k.name) - 1);
            it = acc.emplace(n, k).first;
            order.push_back(n);
        }
        it->second.launches += 1;
        it->second.ms += ms;
        it->second.bytes += r.bytes;
    }
    for (cudaEvent_t e : p->pool) cudaEventDestroy(e);
    delete p;
    int n = 0;
    for (const std::string& k : order) {
        if (n < cap && out) out[n] = acc[k];
        ++n;
    }
    return n;
}

} // namespace dcg
