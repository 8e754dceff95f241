// peer.cuh — device-side primitives of the P2P transport (comm.cu), shared with
// the solver kernels that fuse their exchange into the producing kernel
// (kernels.cu: k_price / k_update put their messages straight into the peers'
// mailboxes; k_price_final / k_ratio_final wait for the flags).
//
// Heap layout (identical on every rank):
//   [0, 4 KB)                 flags: u64 per source rank (last sequence it raised here);
//                             u64 kErrorWord: set when a wait timed out
//   [4 KB, 4 KB + 2 MB_)      two mailboxes (by sequence parity)
//   [4 KB + 2 MB_, bytes)     symmetric allocations (owner_bcast targets)
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdio>

namespace lpsg {

constexpr size_t kFlagBytes = 4096;
constexpr int kErrorWord = 480;
constexpr size_t kMailbox = (size_t)8 << 20;

struct PeerArgs {
    char* const* peers;  // device array: every rank's heap base
    int rank, size;
    unsigned long long seq;
    size_t mbox;         // mailbox offset for this sequence's parity
    int watchdog;        // debug: report timeouts
    unsigned long long timeout_ns;
};

__device__ __forceinline__ void st_flag(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_flag(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Raise this rank's flag for a.seq at every peer (after a system-scope fence
// that orders the payload stores before it). Threads [0, size) do the stores.
__device__ __forceinline__ void peer_signal(const PeerArgs& a) {
    __threadfence_system();
    if (threadIdx.x < (unsigned)a.size)
        st_flag(reinterpret_cast<unsigned long long*>(a.peers[threadIdx.x]) + a.rank, a.seq);
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Spin until every source raised this sequence. A peer that never arrives
// (crashed rank, mismatched call sequence) ends the wait after timeout_ns with
// the error word set, so the host fails the solve instead of hanging the GPU.
__device__ __forceinline__ void peer_wait(const PeerArgs& a) {
    if (threadIdx.x < (unsigned)a.size) {
        unsigned long long* heap = reinterpret_cast<unsigned long long*>(a.peers[a.rank]);
        const unsigned long long* f = heap + threadIdx.x;
        const unsigned long long t0 = globaltimer_ns();
        unsigned long long v;
        unsigned spins = 0;
        while ((v = ld_flag(f)) < a.seq) {
            if ((++spins & 1023u) == 0 && globaltimer_ns() - t0 > a.timeout_ns) {
                if (a.watchdog)
                    printf("[p2p] rank %d timed out at seq %llu: flag[%d] = %llu\n", a.rank, a.seq,
                           (int)threadIdx.x, v);
                atomicExch(heap + kErrorWord, 1ull);
                break;
            }
        }
    }
    __syncthreads();
    __threadfence_system();
}


}  // namespace lpsg
