// fake_nccl.cpp -- test infrastructure only: an in-process stand-in for the subset of NCCL
// the library uses (csrc/comm_api.inc), so that SEVERAL RANKS ON ONE GPU -- one thread and
// one dc_ctx per rank -- run the library's real multi-GPU code path (dc_comm_attach, the
// (c, zeta) exchange at the IEWPF barrier, the drifter gather to rank 0). Real NCCL refuses
// two ranks on one device, and the test box has one GPU.
//
// Semantics kept from NCCL: communicators over a shared unique id (CommInitRank blocks until
// every rank joined); AllGather; grouped Send / Recv matched per (source, destination) pair
// in posting order; completion ordered on the caller's stream. Transfers are device-to-
// device copies on the receiver's stream after the sender's data is ready (events); a
// sender's stream then waits until its buffers were read. Unlike NCCL, the host calls
// rendezvous (every rank reaches the same collective), which is what a correct driver does.
// Built by tests (g++ ... -shared -o libfake_nccl.so) and loaded through DC_NCCL_LIB.
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <vector>

extern "C" {
typedef struct { char internal[128]; } ncclUniqueId;
typedef enum { ncclSuccess = 0, ncclInvalidArgument = 4, ncclInvalidUsage = 5 } ncclResult_t;
typedef enum { ncclInt8 = 0, ncclUint8 = 1, ncclInt32 = 2, ncclUint32 = 3, ncclInt64 = 4,
               ncclUint64 = 5, ncclFloat16 = 6, ncclFloat32 = 7, ncclFloat64 = 8 } ncclDataType_t;
struct FakeComm;
typedef FakeComm* ncclComm_t;
}

namespace {

size_t type_size(ncclDataType_t t) {
    switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
    }
}

struct Msg {  // one posted send
    const void* buf;
    size_t bytes;
    cudaEvent_t ready;   // the sender's data is complete
    cudaEvent_t done;    // the receiver's copy is complete (set by the receiver)
    bool consumed = false;
};

struct World {
    int nranks = 0, joined = 0;
    std::mutex mu;
    std::condition_variable cv;
    std::map<std::pair<int, int>, std::deque<Msg*>> box;  // (src, dst) -> posted sends
};

std::mutex g_mu;
std::map<std::string, World*> g_worlds;
uint64_t g_next_id = 1;

}  // namespace

struct FakeComm {
    World* w;
    int rank;
};

namespace {
struct Op {
    bool send;
    void* buf;
    size_t bytes;
    int peer;
    ncclComm_t comm;
    cudaStream_t s;
};
thread_local int t_group = 0;
thread_local std::vector<Op> t_ops;

ncclResult_t run_ops(std::vector<Op>& ops) {
    // post every send, then serve every receive, then wait until the sends were read
    std::vector<Msg*> mine;
    for (Op& o : ops) {
        if (!o.send) continue;
        Msg* m = new Msg{o.buf, o.bytes, nullptr, nullptr};
        cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&m->done, cudaEventDisableTiming);
        cudaEventRecord(m->ready, o.s);
        World* w = o.comm->w;
        std::lock_guard<std::mutex> lk(w->mu);
        w->box[{o.comm->rank, o.peer}].push_back(m);
        w->cv.notify_all();
        mine.push_back(m);
    }
    for (Op& o : ops) {
        if (o.send) continue;
        World* w = o.comm->w;
        std::unique_lock<std::mutex> lk(w->mu);
        auto& q = w->box[{o.peer, o.comm->rank}];
        w->cv.wait(lk, [&] { return !q.empty(); });
        Msg* m = q.front();
        q.pop_front();
        lk.unlock();
        if (m->bytes != o.bytes) return ncclInvalidUsage;
        cudaStreamWaitEvent(o.s, m->ready, 0);
        cudaMemcpyAsync(o.buf, m->buf, o.bytes, cudaMemcpyDeviceToDevice, o.s);
        cudaEventRecord(m->done, o.s);
        lk.lock();
        m->consumed = true;
        w->cv.notify_all();
    }
    for (size_t i = 0, k = 0; i < ops.size(); ++i) {
        Op& o = ops[i];
        if (!o.send) continue;
        Msg* m = mine[k++];
        World* w = o.comm->w;
        std::unique_lock<std::mutex> lk(w->mu);
        w->cv.wait(lk, [&] { return m->consumed; });
        lk.unlock();
        cudaStreamWaitEvent(o.s, m->done, 0);
        // the events may still be pending on the streams; release them lazily (tiny leak in
        // a test process is acceptable, destroying pending events is legal anyway)
        cudaEventDestroy(m->ready);
        cudaEventDestroy(m->done);
        delete m;
    }
    return ncclSuccess;
}
}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    std::memset(id->internal, 0, sizeof(id->internal));
    std::lock_guard<std::mutex> lk(g_mu);
    const uint64_t v = g_next_id++;
    std::memcpy(id->internal, "fakenccl", 8);
    std::memcpy(id->internal + 8, &v, sizeof(v));
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    World* w;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        const std::string key(id.internal, sizeof(id.internal));
        auto it = g_worlds.find(key);
        if (it == g_worlds.end()) {
            w = new World();
            w->nranks = nranks;
            g_worlds[key] = w;
        } else {
            w = it->second;
        }
    }
    std::unique_lock<std::mutex> lk(w->mu);
    if (w->nranks != nranks) return ncclInvalidUsage;
    w->joined += 1;
    w->cv.notify_all();
    w->cv.wait(lk, [&] { return w->joined >= w->nranks; });
    *comm = new FakeComm{w, rank};
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
    delete comm;  // the world stays (ids are never reused)
    return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) {
    return r == ncclSuccess ? "success (fake NCCL)" : "error (fake NCCL)";
}

ncclResult_t ncclGroupStart() {
    ++t_group;
    return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
    if (t_group <= 0) return ncclInvalidUsage;
    if (--t_group > 0) return ncclSuccess;
    std::vector<Op> ops;
    ops.swap(t_ops);
    return run_ops(ops);
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t type, int peer,
                      ncclComm_t comm, cudaStream_t s) {
    Op o{true, const_cast<void*>(buf), count * type_size(type), peer, comm, s};
    if (t_group > 0) {
        t_ops.push_back(o);
        return ncclSuccess;
    }
    std::vector<Op> v{o};
    return run_ops(v);
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t type, int peer, ncclComm_t comm,
                      cudaStream_t s) {
    Op o{false, buf, count * type_size(type), peer, comm, s};
    if (t_group > 0) {
        t_ops.push_back(o);
        return ncclSuccess;
    }
    std::vector<Op> v{o};
    return run_ops(v);
}

ncclResult_t ncclAllGather(const void* send, void* recv, size_t count, ncclDataType_t type,
                           ncclComm_t comm, cudaStream_t s) {
    // every rank sends its block to every other rank; its own block is a local copy
    World* w = comm->w;
    const size_t bytes = count * type_size(type);
    std::vector<Op> ops;
    for (int r = 0; r < w->nranks; ++r) {
        if (r == comm->rank) continue;
        ops.push_back(Op{true, const_cast<void*>(send), bytes, r, comm, s});
        ops.push_back(Op{false, static_cast<char*>(recv) + r * bytes, bytes, r, comm, s});
    }
    cudaMemcpyAsync(static_cast<char*>(recv) + comm->rank * bytes, send, bytes,
                    cudaMemcpyDeviceToDevice, s);
    return run_ops(ops);
}

}  // extern "C"
