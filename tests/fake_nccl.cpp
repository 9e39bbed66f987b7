// Test double for libnccl.so.2 (test infrastructure, never shipped or loaded by
// the product unless TMG_NCCL_LIB points at it).
//
// The slab code's rank-per-process branch (csrc/slabs.inc: State::run with
// ncclSend / ncclRecv groups, the norm gather in SlabGroup::cycle) needs one
// GPU per rank under real NCCL.  This library implements the eight NCCL entry
// points that branch binds so that the ranks can be THREADS of one process on
// one GPU: a send posts (buffer, byte count, "ready" event recorded on the
// sender's stream) into the mailbox of its (src, dst) pair; the matching
// receive -- matched in posting order per pair, as NCCL matches point-to-point
// operations -- makes the receiver's stream wait for that event, enqueues a
// device-to-device copy and hands back a "done" event the sender's stream
// waits on before it may overwrite the buffer.  No kernel waits on another
// rank; only stream-event dependencies.  A receive whose byte count differs
// from its send fails both sides with ncclInvalidArgument.
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

namespace {

struct Msg {
    const void* buf = nullptr;
    size_t bytes = 0;
    cudaEvent_t ready = nullptr, done = nullptr;
    bool consumed = false, bad = false;
};

struct World {
    int n = 0, joined = 0;
    std::mutex mu;
    std::condition_variable cv;
    std::map<std::pair<int, int>, std::deque<std::shared_ptr<Msg>>> box;
};

std::mutex gMu;
std::map<std::string, std::shared_ptr<World>> gWorlds;
std::atomic<unsigned long long> gSends{0}, gBytes{0}, gGroups{0}, gIds{0};

struct Op {
    bool send;
    const void* sbuf;
    void* rbuf;
    size_t bytes;
    int peer;
    cudaStream_t stream;
    ncclComm_t comm;
};

thread_local int tDepth = 0;
thread_local std::vector<Op> tPending;

constexpr auto kTimeout = std::chrono::seconds(120);

size_t type_size(ncclDataType_t t) {
    switch (t) {
        case ncclInt8:
        case ncclUint8: return 1;
        case ncclFloat16: return 2;
        case ncclInt32:
        case ncclUint32:
        case ncclFloat32: return 4;
        case ncclInt64:
        case ncclUint64:
        case ncclFloat64: return 8;
        default: return 0;
    }
}

}  // namespace

struct ncclComm {
    std::shared_ptr<World> w;
    int rank = 0;
};

namespace {

ncclResult_t flush() {
    std::vector<Op> ops;
    ops.swap(tPending);
    if (ops.empty()) return ncclSuccess;
    ++gGroups;
    ncclResult_t result = ncclSuccess;
    struct Sent {
        std::shared_ptr<Msg> msg;
        cudaStream_t stream;
        World* w;
    };
    std::vector<Sent> mine;
    for (const Op& op : ops) {  // 1. post every send
        if (!op.send) continue;
        World& w = *op.comm->w;
        auto m = std::make_shared<Msg>();
        m->buf = op.sbuf;
        m->bytes = op.bytes;
        if (cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventRecord(m->ready, op.stream) != cudaSuccess)
            return ncclUnhandledCudaError;
        {
            std::lock_guard<std::mutex> lk(w.mu);
            w.box[{op.comm->rank, op.peer}].push_back(m);
        }
        w.cv.notify_all();
        mine.push_back(Sent{m, op.stream, &w});
        ++gSends;
        gBytes += op.bytes;
    }
    for (const Op& op : ops) {  // 2. match every receive with the peer's next send to this rank
        if (op.send) continue;
        World& w = *op.comm->w;
        std::shared_ptr<Msg> m;
        {
            std::unique_lock<std::mutex> lk(w.mu);
            auto& q = w.box[{op.peer, op.comm->rank}];
            if (!w.cv.wait_for(lk, kTimeout, [&] { return !q.empty(); })) return ncclInternalError;
            m = q.front();
            q.pop_front();
        }
        const bool ok = m->bytes == op.bytes;
        cudaEvent_t done = nullptr;
        cudaError_t e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
        if (ok && e == cudaSuccess) e = cudaStreamWaitEvent(op.stream, m->ready, 0);
        if (ok && e == cudaSuccess) e = cudaMemcpyAsync(op.rbuf, m->buf, op.bytes, cudaMemcpyDeviceToDevice, op.stream);
        if (e == cudaSuccess) e = cudaEventRecord(done, op.stream);
        {
            std::lock_guard<std::mutex> lk(w.mu);
            m->done = done;
            m->consumed = true;
            m->bad = !ok || e != cudaSuccess;
        }
        w.cv.notify_all();
        if (!ok) result = ncclInvalidArgument;
        else if (e != cudaSuccess) result = ncclUnhandledCudaError;
    }
    for (Sent& sn : mine) {  // 3. the send buffers may be rewritten once the copies are done
        Msg& m = *sn.msg;
        {
            std::unique_lock<std::mutex> lk(sn.w->mu);
            if (!sn.w->cv.wait_for(lk, kTimeout, [&] { return m.consumed; })) return ncclInternalError;
        }
        if (m.done) {
            if (cudaStreamWaitEvent(sn.stream, m.done, 0) != cudaSuccess) result = ncclUnhandledCudaError;
            cudaEventDestroy(m.done);
        }
        cudaEventDestroy(m.ready);
        if (m.bad && result == ncclSuccess) result = ncclInvalidArgument;
    }
    return result;
}

ncclResult_t enqueue(bool send, const void* sbuf, void* rbuf, size_t count, ncclDataType_t type, int peer,
                     ncclComm_t comm, cudaStream_t stream) {
    const size_t ts = type_size(type);
    if (!comm || ts == 0 || peer < 0 || peer >= comm->w->n || peer == comm->rank) return ncclInvalidArgument;
    tPending.push_back(Op{send, sbuf, rbuf, count * ts, peer, stream, comm});
    return tDepth > 0 ? ncclSuccess : flush();
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    std::memset(id, 0, sizeof(*id));
    const unsigned long long k = ++gIds;
    std::snprintf(id->internal, sizeof(id->internal), "fake-nccl-%llu-%p", k, static_cast<void*>(&gIds));
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
    if (!comm || nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    const std::string key(id.internal, sizeof(id.internal));
    std::shared_ptr<World> w;
    {
        std::lock_guard<std::mutex> lk(gMu);
        auto& slot = gWorlds[key];
        if (!slot) {
            slot = std::make_shared<World>();
            slot->n = nranks;
        }
        w = slot;
    }
    if (w->n != nranks) return ncclInvalidArgument;
    {
        std::unique_lock<std::mutex> lk(w->mu);
        ++w->joined;
        w->cv.notify_all();
        if (!w->cv.wait_for(lk, kTimeout, [&] { return w->joined >= w->n; })) return ncclInternalError;
    }
    *comm = new ncclComm{w, rank};
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
    delete comm;
    return ncclSuccess;
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t type, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
    return enqueue(true, buf, nullptr, count, type, peer, comm, stream);
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t type, int peer, ncclComm_t comm, cudaStream_t stream) {
    return enqueue(false, nullptr, buf, count, type, peer, comm, stream);
}

ncclResult_t ncclGroupStart() {
    ++tDepth;
    return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
    if (tDepth <= 0) return ncclInvalidUsage;
    return --tDepth == 0 ? flush() : ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) {
    switch (r) {
        case ncclSuccess: return "no error";
        case ncclUnhandledCudaError: return "fake nccl: CUDA error";
        case ncclInternalError: return "fake nccl: timed out waiting for the peer";
        case ncclInvalidArgument: return "fake nccl: invalid argument (peer, type, or send / recv size mismatch)";
        case ncclInvalidUsage: return "fake nccl: invalid usage";
        default: return "fake nccl: error";
    }
}

// counters for the test: point-to-point sends, their bytes, non-empty groups
void fake_nccl_stats(unsigned long long* out3) {
    out3[0] = gSends.load();
    out3[1] = gBytes.load();
    out3[2] = gGroups.load();
}

}  // extern "C"
