// comm.cu — NCCL and in-process shard exchange (comm.h).
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "device.cuh"
#include "peer.cuh"

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
    const char* transport() const override { return "nccl"; }
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
    const char* transport() const override { return "local-events"; }
    void host_barrier() override { hub_->barrier(); }
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
    bool debug_sync_ = xp_env("LPSG_LOCAL_SYNC") != nullptr;
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

// ------------------------------------------------------------------ P2P ---
// Heap layout (identical on every rank):
//   [0, 4 KB)                 flags: u64 per source rank (last sequence it raised here)
//   [4 KB, 4 KB + 2 MB_)      two mailboxes (by sequence parity)
//   [4 KB + 2 MB_, bytes)     symmetric allocations (owner_bcast targets)
constexpr int kSmallThreads = 512;

enum PeerOp : int { OP_GATHER = 0, OP_SUM_I64 = 1, OP_MIN_I32 = 2, OP_BCAST = 3, OP_OWNER = 4 };

// copy `bytes` from src to dst with the threads [t0, t0 + nt) (16-byte lanes when aligned)
__device__ __forceinline__ void peer_copy(char* dst, const char* src, size_t bytes, size_t t0, size_t nt) {
    if ((((uintptr_t)dst | (uintptr_t)src | bytes) & 15) == 0) {
        const size_t n = bytes / 16;
        for (size_t k = t0; k < n; k += nt)
            reinterpret_cast<int4*>(dst)[k] = __ldcg(reinterpret_cast<const int4*>(src) + k);
    } else {
        for (size_t k = t0; k < bytes; k += nt) dst[k] = src[k];
    }
}

// Phase 1 (put): this rank's contribution into every peer's mailbox slot (or,
// for OP_OWNER, straight into the peers' copy of the symmetric buffer).
__device__ void peer_put(const PeerArgs& a, int op, const char* send, size_t bytes, int root, const int* is_owner,
                         size_t sym_off, size_t t0, size_t nt) {
    for (int g = 0; g < a.size; ++g) {
        char* peer = a.peers[g];
        switch (op) {
            case OP_GATHER:
            case OP_SUM_I64:
            case OP_MIN_I32: peer_copy(peer + a.mbox + (size_t)a.rank * bytes, send, bytes, t0, nt); break;
            case OP_BCAST:
                if (a.rank == root && g != a.rank) peer_copy(peer + a.mbox, send, bytes, t0, nt);
                break;
            case OP_OWNER:
                if (*is_owner && g != a.rank) peer_copy(peer + sym_off, send, bytes, t0, nt);
                break;
        }
    }
}

// Phase 3 (post): mailbox -> caller's buffer.
__device__ void peer_post(const PeerArgs& a, int op, char* out, size_t bytes, int root, size_t t0, size_t nt) {
    const char* mb = a.peers[a.rank] + a.mbox;
    switch (op) {
        case OP_GATHER: peer_copy(out, mb, bytes * a.size, t0, nt); break;
        case OP_SUM_I64: {
            const size_t n = bytes / 8;
            for (size_t k = t0; k < n; k += nt) {
                long long v = 0;
                for (int g = 0; g < a.size; ++g) v += __ldcg(reinterpret_cast<const long long*>(mb + (size_t)g * bytes) + k);
                reinterpret_cast<long long*>(out)[k] = v;
            }
            break;
        }
        case OP_MIN_I32: {
            const size_t n = bytes / 4;
            for (size_t k = t0; k < n; k += nt) {
                int v = INT_MAX;
                for (int g = 0; g < a.size; ++g) v = min(v, __ldcg(reinterpret_cast<const int*>(mb + (size_t)g * bytes) + k));
                reinterpret_cast<int*>(out)[k] = v;
            }
            break;
        }
        case OP_BCAST:
            if (a.rank != root) peer_copy(out, mb, bytes, t0, nt);
            break;
        default: break;
    }
}

// Small messages: the whole collective in one CTA (one launch).
__global__ void __launch_bounds__(kSmallThreads) k_peer_small(PeerArgs a, int op, const char* send, char* out,
                                                              size_t bytes, int root, const int* is_owner,
                                                              size_t sym_off) {
    peer_put(a, op, send, bytes, root, is_owner, sym_off, threadIdx.x, blockDim.x);
    __syncthreads();
    peer_signal(a);
    peer_wait(a);
    peer_post(a, op, out, bytes, root, threadIdx.x, blockDim.x);
}

// Large messages: multi-CTA put, the last CTA raises the flags ...
__global__ void __launch_bounds__(256) k_peer_put(PeerArgs a, int op, const char* send, size_t bytes, int root,
                                                  const int* is_owner, size_t sym_off, unsigned int* ticket) {
    peer_put(a, op, send, bytes, root, is_owner, sym_off, (size_t)blockIdx.x * blockDim.x + threadIdx.x,
             (size_t)gridDim.x * blockDim.x);
    __threadfence_system();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    if (threadIdx.x == 0) *ticket = 0;
    peer_signal(a);
}

// ... one CTA waits (so a waiting rank holds at most one SM) ...
__global__ void k_peer_wait(PeerArgs a) { peer_wait(a); }

// ... and a grid drains the mailbox.
__global__ void __launch_bounds__(256) k_peer_post(PeerArgs a, int op, char* out, size_t bytes, int root) {
    peer_post(a, op, out, bytes, root, (size_t)blockIdx.x * blockDim.x + threadIdx.x, (size_t)gridDim.x * blockDim.x);
}

class PeerComm final : public Comm {
public:
    explicit PeerComm(PeerHeap* h) : h_(h) {
        rank = h->rank;
        size = h->size;
        // same carveout as the solver kernels (kernels.cu configure_kernels)
        const void* ks[] = {(const void*)k_peer_small, (const void*)k_peer_put, (const void*)k_peer_wait,
                            (const void*)k_peer_post};
        for (const void* f : ks) cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cuda_ok(cudaMalloc(&peers_dev_, sizeof(char*) * size), "cudaMalloc");
        cuda_ok(cudaMemcpy(peers_dev_, h->peers.data(), sizeof(char*) * size, cudaMemcpyHostToDevice), "cudaMemcpy");
        cuda_ok(cudaMalloc(&ticket_, sizeof(unsigned int)), "cudaMalloc");
        cuda_ok(cudaMemset(ticket_, 0, sizeof(unsigned int)), "cudaMemset");
        // flags were zeroed by peer_heap_create, before any peer could map the heap
        sym_next_ = kFlagBytes + 2 * kMailbox;
        if (h->bytes < sym_next_ + ((size_t)1 << 20)) throw CommError("peer heap too small");
    }
    ~PeerComm() override {
        if (peers_dev_) cudaFree(peers_dev_);
        if (ticket_) cudaFree(ticket_);
    }
    const char* transport() const override { return "p2p"; }
    void host_barrier() override {
        if (h_->hub) h_->hub->barrier();
    }
    // Shards sharing one GPU in one process keep to one batch in flight: their
    // spin-waiting exchange kernels compete for the same SMs.
    bool allows_pipelining() const override { return h_->hub == nullptr; }
    void wait_slot(const PeerArgs& a, cudaStream_t st) override {
        k_peer_wait<<<1, 32, 0, st>>>(a);
        cuda_ok(cudaGetLastError(), "k_peer_wait");
    }
    size_t sym_offset(const void* p) const override { return (size_t)(static_cast<const char*>(p) - h_->base); }
    bool fused_slot(PeerArgs* out) override {
        const unsigned long long seq = ++h_->seq;
        *out = PeerArgs{peers_dev_, rank, size, seq, kFlagBytes + (seq & 1) * kMailbox, trace_ ? 1 : 0, timeout_ns_};
        ++calls;
        return true;
    }
    void check(cudaStream_t st) override {
        unsigned long long e = 0;
        cuda_ok(cudaMemcpyAsync(&e, reinterpret_cast<unsigned long long*>(h_->base) + kErrorWord, 8,
                                cudaMemcpyDeviceToHost, st),
                "cudaMemcpyAsync");
        cuda_ok(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        if (e) throw CommError("p2p exchange timed out waiting for a peer (LPSG_P2P_TIMEOUT_S)");
    }

    void* sym_alloc(size_t b) override {
        const size_t off = (sym_next_ + 255) & ~(size_t)255;
        if (off + b > h_->bytes) throw CommError("peer heap exhausted (raise the heap size)");
        sym_next_ = off + b;
        return h_->base + off;
    }
    void sym_free(void*) override {}

    void allgather(const void* send, void* recv, size_t b, cudaStream_t st) override {
        run(OP_GATHER, send, recv, b, 0, nullptr, st);
    }
    void sum_i64(long long* buf, size_t n, cudaStream_t st) override { run(OP_SUM_I64, buf, buf, 8 * n, 0, nullptr, st); }
    void min_i32(int* buf, size_t n, cudaStream_t st) override { run(OP_MIN_I32, buf, buf, 4 * n, 0, nullptr, st); }
    void bcast(void* buf, size_t b, int root, cudaStream_t st) override { run(OP_BCAST, buf, buf, b, root, nullptr, st); }
    void owner_bcast(void* buf, size_t b, const int* is_owner, cudaStream_t st) override {
        const char* p = static_cast<const char*>(buf);
        if (p < h_->base || p + b > h_->base + h_->bytes) throw CommError("owner_bcast: buffer is not in the peer heap");
        one(OP_OWNER, buf, buf, b, 0, is_owner, (size_t)(p - h_->base), st);
    }

private:
    // split so each rank's piece times `size` fits one mailbox
    void run(int op, const void* send, void* out, size_t b, int root, const int* owner, cudaStream_t st) {
        const size_t per = op == OP_BCAST ? kMailbox : (kMailbox / size) & ~(size_t)15;
        if (b <= per) {
            one(op, send, out, b, root, owner, 0, st);
            return;
        }
        if (op == OP_GATHER) {
            // chunk k of every rank lands in recv[g*b + k*per ...]: gather into a
            // temporary of size*chunk per round and scatter (rare: large gathers)
            char* tmp = nullptr;
            cuda_ok(cudaMallocAsync(reinterpret_cast<void**>(&tmp), per * size, st), "cudaMallocAsync");
            for (size_t o = 0; o < b; o += per) {
                const size_t c = std::min(per, b - o);
                one(op, static_cast<const char*>(send) + o, tmp, c, root, owner, 0, st);
                for (int g = 0; g < size; ++g)
                    cuda_ok(cudaMemcpyAsync(static_cast<char*>(out) + (size_t)g * b + o, tmp + (size_t)g * c, c,
                                            cudaMemcpyDeviceToDevice, st),
                            "cudaMemcpyAsync");
            }
            cuda_ok(cudaFreeAsync(tmp, st), "cudaFreeAsync");
            return;
        }
        const size_t unit = op == OP_MIN_I32 ? 4 : 8;
        const size_t step = std::max(unit, per / unit * unit);
        for (size_t o = 0; o < b; o += step) {
            const size_t c = std::min(step, b - o);
            one(op, static_cast<const char*>(send) + o, static_cast<char*>(out) + o, c, root, owner, 0, st);
        }
    }

    void one(int op, const void* send, void* out, size_t b, int root, const int* owner, size_t sym_off,
             cudaStream_t st) {
        const unsigned long long seq = ++h_->seq;
        PeerArgs a{peers_dev_, rank, size, seq, kFlagBytes + (seq & 1) * kMailbox, trace_ ? 1 : 0, timeout_ns_};
        if (trace_)
            fprintf(stderr, "[p2p r%d] seq %llu op %d bytes %zu peers %p %p\n", rank, seq, op, b,
                    (void*)h_->peers[0], (void*)h_->peers[size > 1 ? 1 : 0]);
        const size_t moved = op == OP_GATHER || op == OP_SUM_I64 || op == OP_MIN_I32 ? b * size : b * (size - 1);
        ++calls;
        bytes += (double)b;
        if (moved <= ((size_t)64 << 10)) {
            k_peer_small<<<1, kSmallThreads, 0, st>>>(a, op, static_cast<const char*>(send), static_cast<char*>(out),
                                                       b, root, owner, sym_off);
        } else {
            const unsigned grid = (unsigned)std::min<size_t>(128, (moved / 16 + 255) / 256 + 1);
            k_peer_put<<<grid, 256, 0, st>>>(a, op, static_cast<const char*>(send), b, root, owner, sym_off, ticket_);
            k_peer_wait<<<1, 32, 0, st>>>(a);
            if (op != OP_OWNER) {
                const size_t post = op == OP_GATHER ? b * size : b;
                const unsigned g2 = (unsigned)std::min<size_t>(256, (post / 16 + 255) / 256 + 1);
                k_peer_post<<<g2, 256, 0, st>>>(a, op, static_cast<char*>(out), b, root);
            }
        }
        cuda_ok(cudaGetLastError(), "peer collective launch");
    }

    PeerHeap* h_;
    bool trace_ = getenv("LPSG_TRACE_COMM") != nullptr;
    unsigned long long timeout_ns_ = (unsigned long long)(1e9 * (getenv("LPSG_P2P_TIMEOUT_S")
                                                                      ? atof(getenv("LPSG_P2P_TIMEOUT_S"))
                                                                      : 30.0));
    char** peers_dev_ = nullptr;
    unsigned int* ticket_ = nullptr;
    size_t sym_next_ = 0;
};

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

void* Comm::sym_alloc(size_t b) {
    void* p = nullptr;
    cuda_ok(cudaMalloc(&p, std::max<size_t>(b, 16)), "cudaMalloc");
    return p;
}

void Comm::sym_free(void* p) {
    if (p) cudaFree(p);
}

PeerHeap::~PeerHeap() {
    for (size_t g = 0; g < peers.size(); ++g)
        if (opened[g] && peers[g]) cudaIpcCloseMemHandle(peers[g]);
    if (base) cudaFree(base);
}

std::unique_ptr<PeerHeap> peer_heap_create(int rank, int size, int device, size_t bytes, unsigned char handle[64]) {
    std::unique_ptr<PeerHeap> h(new PeerHeap);
    h->rank = rank;
    h->size = size;
    h->device = device;
    h->bytes = bytes ? bytes : kPeerHeapDefault;
    cuda_ok(cudaSetDevice(device), "cudaSetDevice");
    cuda_ok(cudaMalloc(reinterpret_cast<void**>(&h->base), h->bytes), "cudaMalloc(peer heap)");
    cuda_ok(cudaMemset(h->base, 0, kFlagBytes), "cudaMemset");
    cuda_ok(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    h->peers.assign(size, nullptr);
    h->opened.assign(size, false);
    h->peers[rank] = h->base;
    if (handle) {
        cudaIpcMemHandle_t ih;
        cuda_ok(cudaIpcGetMemHandle(&ih, h->base), "cudaIpcGetMemHandle");
        static_assert(sizeof(ih) == 64, "cudaIpcMemHandle_t is 64 bytes");
        std::memcpy(handle, &ih, 64);
    }
    return h;
}

void peer_heap_connect(PeerHeap* h, const unsigned char* handles) {
    cuda_ok(cudaSetDevice(h->device), "cudaSetDevice");
    for (int g = 0; g < h->size; ++g) {
        if (g == h->rank) continue;
        cudaIpcMemHandle_t ih;
        std::memcpy(&ih, handles + 64 * (size_t)g, 64);
        void* p = nullptr;
        cuda_ok(cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        h->peers[g] = static_cast<char*>(p);
        h->opened[g] = true;
    }
}

void peer_heap_connect_local(PeerHeap* h, const std::vector<char*>& bases) {
    for (int g = 0; g < h->size; ++g) h->peers[g] = bases[g];
    for (int g = 0; g < h->size; ++g) {
        if (g == h->rank) continue;
        int dev_g = -1;
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, bases[g]) == cudaSuccess) dev_g = at.device;
        if (dev_g >= 0 && dev_g != h->device) {
            const cudaError_t e = cudaDeviceEnablePeerAccess(dev_g, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                throw CommError(std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
            cudaGetLastError();
        }
    }
}

std::unique_ptr<Comm> make_peer_comm(PeerHeap* heap) { return std::unique_ptr<Comm>(new PeerComm(heap)); }

std::unique_ptr<Comm> make_local_comm(LocalHub* hub, int rank) {
    return std::unique_ptr<Comm>(new LocalComm(hub, rank));
}

}  // namespace lpsg
