// comm.h — shard exchange for the sharded solver.
//
// Every collective is stream-ordered on the caller's stream and must be
// issued by every rank in the same order (the solver's decisions are
// replicated, so all ranks walk the same host code path). Two transports:
//
//   NcclComm   one process (or thread) per GPU, NCCL over NVLink / NVSwitch.
//              libnccl.so.2 is dlopen'ed: the library has no link-time NCCL
//              dependency and single-GPU use never loads it.
//   LocalComm  G shards inside one process, one host thread each, on one or
//              several devices; exchanges are device-to-device copies ordered
//              by CUDA events and host barriers. This is how the sharded path
//              is parity-tested on a single B200.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "peer.cuh"

namespace lpsg {

struct CommError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

class Comm {
public:
    int rank = 0, size = 1;
    long long calls = 0;
    double bytes = 0.0;  // payload bytes this rank contributed
    virtual ~Comm() = default;
    // recv[g*bytes .. (g+1)*bytes) = send of rank g
    virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
    // in place, element-wise over ranks; used with a single non-zero
    // contributor to deliver doubles bit for bit (int64 patterns)
    virtual void sum_i64(long long* buf, size_t n, cudaStream_t st) = 0;
    virtual void min_i32(int* buf, size_t n, cudaStream_t st) = 0;
    virtual void bcast(void* buf, size_t bytes, int root, cudaStream_t st) = 0;
    // Broadcast from the rank whose *is_owner (device int) is non-zero; the
    // owner is known on the device only. Default: the int64 bit-pattern sum
    // (non-owners must have zero-filled buf).
    virtual void owner_bcast(void* buf, size_t bytes, const int* is_owner, cudaStream_t st) {
        (void)is_owner;
        sum_i64(static_cast<long long*>(buf), bytes / 8, st);
    }
    // Device memory that collectives may write remotely (owner_bcast targets).
    // Every rank must make the same sequence of calls (symmetric heaps).
    virtual void* sym_alloc(size_t bytes);
    virtual void sym_free(void* p);
    virtual const char* transport() const = 0;
    // Host-side barrier of shards that share a process (no-op across processes).
    virtual void host_barrier() {}
    // Throws CommError when the transport recorded a failure (called after syncs;
    // stream-ordered: a legacy-stream copy here can stall behind another shard's
    // spin-waiting kernel on a shared GPU).
    virtual void check(cudaStream_t st) { (void)st; }
    // Device-initiated transports: reserve the next exchange for a kernel that
    // stores its payload straight into the peers' mailboxes (returns false if
    // the transport cannot). Every rank must reserve in the same order.
    virtual bool fused_slot(PeerArgs* out) {
        (void)out;
        return false;
    }
    // Completes a reserved exchange whose payload and flags the kernels stored:
    // waits (stream-ordered, one CTA) until every rank raised the flag.
    virtual void wait_slot(const PeerArgs& a, cudaStream_t st) {
        (void)a;
        (void)st;
    }
    // Offset of a sym_alloc'ed pointer in the symmetric heap (P2P), else 0.
    virtual size_t sym_offset(const void* p) const {
        (void)p;
        return 0;
    }
    // Whether the solver may keep a second pivot batch in flight while it
    // drains the first (pipelined host loop).
    virtual bool allows_pipelining() const { return true; }
};

struct LocalHub;

// ---- device-initiated peer transport (NVLink / NVSwitch P2P stores + flags) ----
// Every rank owns a symmetric heap (same size, same allocation sequence); each
// collective is one or a few kernels that store straight into the peers'
// heaps and raise a per-source sequence flag there, then spin on the local
// flags. No host synchronisation, no NCCL kernel. Peers are mapped with CUDA
// IPC (multi-process) or shared directly (shards of one process).
struct PeerHeap {
    int rank = 0, size = 1, device = 0;
    size_t bytes = 0;
    char* base = nullptr;                // this rank's heap
    std::vector<char*> peers;            // every rank's heap as seen from this device
    std::vector<bool> opened;            // peers[g] came from cudaIpcOpenMemHandle
    LocalHub* hub = nullptr;             // in-process shards: their host barrier
    unsigned long long seq = 0;          // last exchange sequence (persists across solvers on this heap)
    ~PeerHeap();
};
constexpr size_t kPeerHeapDefault = (size_t)96 << 20;
// allocate this rank's heap; `handle` (64 bytes) is its cudaIpcMemHandle
std::unique_ptr<PeerHeap> peer_heap_create(int rank, int size, int device, size_t bytes,
                                           unsigned char handle[64]);
// map the other ranks' heaps from their handles (size x 64 bytes, rank order)
void peer_heap_connect(PeerHeap* h, const unsigned char* handles);
// in-process shards: adopt each other's heap pointers directly
void peer_heap_connect_local(PeerHeap* h, const std::vector<char*>& bases);
std::unique_ptr<Comm> make_peer_comm(PeerHeap* heap);

// NCCL unique id (128 bytes) for rank 0 to hand to the others.
bool nccl_unique_id(unsigned char out[128], std::string* err);
std::unique_ptr<Comm> make_nccl_comm(const unsigned char id[128], int rank, int size, int device);

struct LocalHub {
    explicit LocalHub(int n);
    ~LocalHub();
    void barrier();
    int n;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long long gen = 0;
    std::vector<const void*> ptr;
    std::vector<cudaEvent_t> ready, done;
};
std::unique_ptr<Comm> make_local_comm(LocalHub* hub, int rank);

}  // namespace lpsg
