// comm.cu — NCCL and in-process shard exchange (comm.h).
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <climits>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "device.cuh"

namespace lpsg {

namespace {

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw CommError(std::string(what) + ": " + cudaGetErrorString(e));
    }
}

// ---------------------------------------------------------------- NCCL ---
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
    bool ok = false;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
            return a;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
        a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
        a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.AllReduce &&
               a.Broadcast && a.GetErrorString;
        if (!a.ok) a.error = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    return api;
}

void nccl_ok(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw CommError(std::string(what) + ": " + nccl().GetErrorString(r));
}

class NcclComm final : public Comm {
public:
    NcclComm(const unsigned char id[128], int r, int n, int device) {
        const NcclApi& a = nccl();
        if (!a.ok) throw CommError(a.error);
        cuda_ok(cudaSetDevice(device), "cudaSetDevice");
        ncclUniqueId uid;
        std::memcpy(uid.internal, id, sizeof(uid.internal));
        nccl_ok(a.CommInitRank(&comm_, n, uid, r), "ncclCommInitRank");
        rank = r;
        size = n;
    }
    ~NcclComm() override {
        if (comm_) nccl().CommDestroy(comm_);
    }
    void allgather(const void* send, void* recv, size_t b, cudaStream_t st) override {
        nccl_ok(nccl().AllGather(send, recv, b, ncclUint8, comm_, st), "ncclAllGather");
        ++calls;
        bytes += (double)b;
    }
    void sum_i64(long long* buf, size_t n, cudaStream_t st) override {
        nccl_ok(nccl().AllReduce(buf, buf, n, ncclInt64, ncclSum, comm_, st), "ncclAllReduce");
        ++calls;
        bytes += 8.0 * n;
    }
    void min_i32(int* buf, size_t n, cudaStream_t st) override {
        nccl_ok(nccl().AllReduce(buf, buf, n, ncclInt32, ncclMin, comm_, st), "ncclAllReduce");
        ++calls;
        bytes += 4.0 * n;
    }
    void bcast(void* buf, size_t b, int root, cudaStream_t st) override {
        nccl_ok(nccl().Broadcast(buf, buf, b, ncclUint8, root, comm_, st), "ncclBroadcast");
        ++calls;
        bytes += (double)b;
    }

private:
    ncclComm_t comm_ = nullptr;
};

// ------------------------------------------------------------ in-process ---
// Three-step exchange per collective (every rank, in order):
//   1. record ready[rank] on the stream, publish the source pointer, barrier;
//   2. wait for the sources' ready events, copy, record done[rank], barrier;
//   3. wait for every rank's done event before touching the source again.
// A rank can re-record its events only after passing the next collective's
// first barrier, i.e. after every other rank has issued its waits.
class LocalComm final : public Comm {
public:
    LocalComm(LocalHub* hub, int r) : hub_(hub) {
        rank = r;
        size = hub->n;
        cuda_ok(cudaEventCreateWithFlags(&hub_->ready[r], cudaEventDisableTiming), "cudaEventCreate");
        cuda_ok(cudaEventCreateWithFlags(&hub_->done[r], cudaEventDisableTiming), "cudaEventCreate");
    }
    ~LocalComm() override {
        if (scratch_) cudaFree(scratch_);
    }
    void allgather(const void* send, void* recv, size_t b, cudaStream_t st) override {
        exchange(send, st, [&](int g, const void* src) {
            cuda_ok(cudaMemcpyAsync(static_cast<char*>(recv) + (size_t)g * b, src, b, cudaMemcpyDefault, st),
                    "cudaMemcpyAsync");
        });
        ++calls;
        bytes += (double)b;
    }
    void sum_i64(long long* buf, size_t n, cudaStream_t st) override {
        long long* tmp = static_cast<long long*>(scratch(8 * n * size));
        allgather(buf, tmp, 8 * n, st);
        launch_sum_i64(tmp, size, n, buf, st);
        cuda_ok(cudaGetLastError(), "k_sum_i64");
    }
    void min_i32(int* buf, size_t n, cudaStream_t st) override {
        int* tmp = static_cast<int*>(scratch(4 * n * size));
        allgather(buf, tmp, 4 * n, st);
        launch_min_i32(tmp, size, n, buf, st);
        cuda_ok(cudaGetLastError(), "k_min_i32");
    }
    void bcast(void* buf, size_t b, int root, cudaStream_t st) override {
        exchange(buf, st, [&](int g, const void* src) {
            if (g == root && rank != root)
                cuda_ok(cudaMemcpyAsync(buf, src, b, cudaMemcpyDefault, st), "cudaMemcpyAsync");
        });
        ++calls;
        bytes += (double)b;
    }

private:
    template <class F>
    void exchange(const void* mine, cudaStream_t st, F&& copy) {
        const int n = size;
        cuda_ok(cudaEventRecord(hub_->ready[rank], st), "cudaEventRecord");
        hub_->ptr[rank] = mine;
        hub_->barrier();
        for (int g = 0; g < n; ++g) {
            cuda_ok(cudaStreamWaitEvent(st, hub_->ready[g], 0), "cudaStreamWaitEvent");
            copy(g, hub_->ptr[g]);
        }
        cuda_ok(cudaEventRecord(hub_->done[rank], st), "cudaEventRecord");
        hub_->barrier();
        for (int g = 0; g < n; ++g)
            if (g != rank) cuda_ok(cudaStreamWaitEvent(st, hub_->done[g], 0), "cudaStreamWaitEvent");
        if (debug_sync_) cuda_ok(cudaStreamSynchronize(st), "debug sync");
    }
    bool debug_sync_ = getenv("LPSG_LOCAL_SYNC") != nullptr;
    void* scratch(size_t b) {
        if (b > scratch_bytes_) {
            if (scratch_) cudaFree(scratch_);
            scratch_ = nullptr;
            cuda_ok(cudaMalloc(&scratch_, b), "cudaMalloc");
            scratch_bytes_ = b;
        }
        return scratch_;
    }
    LocalHub* hub_;
    void* scratch_ = nullptr;
    size_t scratch_bytes_ = 0;
};

}  // namespace

LocalHub::LocalHub(int count) : n(count), ptr(count, nullptr), ready(count, nullptr), done(count, nullptr) {}

LocalHub::~LocalHub() {
    for (auto e : ready)
        if (e) cudaEventDestroy(e);
    for (auto e : done)
        if (e) cudaEventDestroy(e);
}

void LocalHub::barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == n) {
        arrived = 0;
        ++gen;
        cv.notify_all();
    } else {
        cv.wait(lk, [&] { return gen != g; });
    }
}

bool nccl_unique_id(unsigned char out[128], std::string* err) {
    const NcclApi& a = nccl();
    if (!a.ok) {
        if (err) *err = a.error;
        return false;
    }
    ncclUniqueId id;
    const ncclResult_t r = a.GetUniqueId(&id);
    if (r != ncclSuccess) {
        if (err) *err = a.GetErrorString(r);
        return false;
    }
    std::memcpy(out, id.internal, sizeof(id.internal));
    return true;
}

std::unique_ptr<Comm> make_nccl_comm(const unsigned char id[128], int rank, int size, int device) {
    return std::unique_ptr<Comm>(new NcclComm(id, rank, size, device));
}

std::unique_ptr<Comm> make_local_comm(LocalHub* hub, int rank) {
    return std::unique_ptr<Comm>(new LocalComm(hub, rank));
}

}  // namespace lpsg
