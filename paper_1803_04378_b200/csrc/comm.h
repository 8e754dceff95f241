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
};

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
