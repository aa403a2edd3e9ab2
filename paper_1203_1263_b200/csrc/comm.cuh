// comm.cuh -- slab-mode synchronisation and small exchanges over peer memory
// (SURVEY §8(e), §8(a) row a9).
//
// The halo data itself moves inside the stage kernels: every stage kernel stores the
// outputs of its first / last w owned planes also into the neighbours' ghost planes
// (store_out, common.cuh).  What remains is ordering: after each stage a rank must
// not start the next stage before both neighbours have finished the current one
// (their remote stores are then complete: a kernel boundary flushes them, and the
// release below orders this rank's flag after them), and the neighbour must not
// overwrite a ghost plane this rank is still reading (the stage outputs alternate
// between buffers, so the same one-stage barrier also covers this write-after-read).
//
// Every rank owns a small "comm block" in its device memory: flags[NLSE_MAX_RANKS]
// (monotone epochs; flags[j] is written by rank j) and xbuf[NLSE_MAX_RANKS][2]
// (diagnostic partial sums; xbuf[j] is written by rank j).  Peers map it through
// CUDA IPC (one process per GPU) or use it directly (virtual ranks in one process).
#pragma once
#include <cstdint>
#include "common.cuh"

namespace nlse {

constexpr int MAX_RANKS = 16;

struct CommBlock {
    unsigned long long flags[MAX_RANKS];
    double xbuf[MAX_RANKS][2];
    unsigned long long my_epoch;   // this rank's barrier count (written by its own launches only)
    unsigned int abort;            // nonzero: a rank gave up (nlse_dist_abort); waiters stop waiting
    unsigned int status;           // barrier outcome of this rank: 0 ok, 1 timed out, 2 aborted
};

// Barrier arguments: signal the next epoch into sig[i]->flags[me] for every listed peer,
// then wait until own->flags[w] >= epoch for every listed waiter rank w.  The epoch
// counter lives in the rank's own comm block (advanced by the signalling launch), so
// the launch parameters are the same every step and a captured CUDA graph can replay.
struct BarrierArgs {
    CommBlock *own;
    CommBlock *sig[MAX_RANKS];
    int wait_rank[MAX_RANKS];
    int nsig, nwait, me;
    unsigned long long timeout_ns;   // give up waiting after this long (NLSE_BARRIER_TIMEOUT_S)
};

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int ld_relaxed_sys(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;\n" : "=l"(t));
    return t;
}

// mode bit 1: signal, bit 2: wait.  Slab mode on separate GPUs launches both in one
// kernel; virtual ranks sharing one stream launch every rank's signal before any wait
// (a spinning kernel must never sit in front of the work that releases it).
static __global__ void __launch_bounds__(32) peer_barrier(BarrierArgs b, int mode) {
    const int t = threadIdx.x;
    const unsigned long long epoch = b.own->my_epoch + ((mode & 1) ? 1ull : 0ull);
    __syncwarp();
    if ((mode & 1) && t == 0) b.own->my_epoch = epoch;
    if ((mode & 1) && t < b.nsig) {
        __threadfence_system();
        st_release_sys(&b.sig[t]->flags[b.me], epoch);
    }
    // bounded wait: exponential __nanosleep backoff (64 ns .. 4 us); a set abort flag or the
    // timeout ends it and records why in own->status (the host turns that into NLSE_ERR_COMM
    // instead of hanging every rank on one failed or late peer)
    if ((mode & 2) && t < b.nwait) {
        const unsigned long long *f = &b.own->flags[b.wait_rank[t]];
        const unsigned long long t0 = globaltimer_ns();
        unsigned ns = 64;
        while (ld_acquire_sys(f) < epoch) {
            if (ld_relaxed_sys(&b.own->abort)) { atomicMax(&b.own->status, 2u); break; }
            if (ld_relaxed_sys(&b.own->status)) break;   // an earlier barrier already gave up
            if (globaltimer_ns() - t0 > b.timeout_ns) { atomicMax(&b.own->status, 1u); break; }
            __nanosleep(ns);
            if (ns < 4096) ns <<= 1;
        }
    }
    __syncwarp();
}

// Advance the device step counter after a launch sequence of n steps.
static __global__ void add_steps(int *counter, int n) {
    if (threadIdx.x == 0) *counter += n;
}

// Push this rank's (mass, energy) partial pair into every rank's xbuf[me].
struct PushArgs {
    CommBlock *dst[MAX_RANKS];
    int n, me;
};
static __global__ void __launch_bounds__(32) diag_push(const double *__restrict__ local, PushArgs a) {
    const int t = threadIdx.x;
    if (t < a.n) {
        a.dst[t]->xbuf[a.me][0] = local[0];
        a.dst[t]->xbuf[a.me][1] = local[1];
    }
}

// Sum the nranks partial pairs in rank order (identical on every rank) and scale by h^d.
static __global__ void __launch_bounds__(32) diag_sum(const CommBlock *__restrict__ own, int n, double hd,
                                               double *__restrict__ result) {
    if (threadIdx.x == 0) {
        double m = 0.0, e = 0.0;
        for (int j = 0; j < n; j++) { m += own->xbuf[j][0]; e += own->xbuf[j][1]; }
        result[0] = hd * m;
        result[1] = hd * e;
    }
}

}  // namespace nlse
