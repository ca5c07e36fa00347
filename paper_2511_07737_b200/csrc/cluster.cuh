// cluster.cuh - exchanges between the CTAs of a thread-block cluster over
// distributed shared memory: k_update MODE 3 splits every variable row's N
// candidates over the CL CTAs of a cluster (DESIGN.md §7 "cluster-split rows"),
// so each CTA keeps the g table of its N / CL candidates in shared memory and
// the row's J_v and Q_{t+1,v} partials (exact int64) are summed over DSMEM.
//
// Each warp group owns, in its shared scratch, one slot per (kind, rank):
// [2 kinds: J, Q][CL ranks][2 words].  The group pair with the same index in
// the other CTAs processes the same rows in the same order (static row
// schedule), so message `seq` (= row iteration + 1) of a kind is written by
// rank r into slot [kind][r] of every other CTA.  An int64 travels as two
// self-validating u64 words (seq << 32 | 32-bit half): an aligned 8-byte
// shared store is single-copy atomic, so a reader that sees `seq` in both
// words has the value.  One slot per kind suffices: a rank writes kind k of
// row i + 1 only after it received every rank's other kind of row i (Q after
// J, J of the next row after Q), which each rank sends after reading row i's
// kind k.  Slots are zeroed at kernel start before a cluster barrier (seq >=
// 1 never matches), and a cluster barrier precedes exit (no DSMEM write can
// target an exited CTA).  A wait longer than kClusterTimeoutNs sets
// DevScalars::xerr (the step returns an error) instead of hanging the GPU.
#pragma once

#include <cstdint>

#include "tsat_internal.h"

namespace tsat {

#ifndef TSAT_CL_SLEEP
#define TSAT_CL_SLEEP 0            // ns between polls (0: spin)
#endif
constexpr unsigned long long kClusterTimeoutNs = 5ull * 1000 * 1000 * 1000;
constexpr int kMaxCluster = 16;

__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_id_x() {
    unsigned r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_count_x() {
    unsigned r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
// Every thread of every CTA of the cluster (convergent: kernel start / end).
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned long long cl_globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void dsmem_st_u64(const void* local_slot, unsigned rank, unsigned long long v) {
    const unsigned l = (unsigned)__cvta_generic_to_shared(local_slot);
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(l), "r"(rank));
    asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(r), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long smem_ld_relaxed_u64(const void* p) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    unsigned long long v;
    asm volatile("ld.relaxed.cluster.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}

// Send this rank's int64 partial x (message seq) into slot [me] of every
// other CTA's copy of `slots` ([CL][2] words of one kind).
__device__ __forceinline__ void cl_send(unsigned long long* slots, unsigned CL, unsigned me, unsigned seq, long long x) {
    const unsigned long long ux = (unsigned long long)x;
    const unsigned long long w0 = ((unsigned long long)seq << 32) | (ux & 0xffffffffull);
    const unsigned long long w1 = ((unsigned long long)seq << 32) | (ux >> 32);
    for (unsigned r = 0; r < CL; ++r) {
        if (r == me) continue;
        dsmem_st_u64(slots + 2 * me, r, w0);
        dsmem_st_u64(slots + 2 * me + 1, r, w1);
    }
}

// One thread polls (optionally with a sleep between polls).
__device__ __forceinline__ unsigned long long cl_wait_word(const unsigned long long* p, unsigned seq, DevScalars* ds) {
    unsigned long long w = smem_ld_relaxed_u64(p);
    if ((unsigned)(w >> 32) == seq) return w;
    const unsigned long long t0 = cl_globaltimer();
    for (unsigned i = 1;; ++i) {
#if TSAT_CL_SLEEP
        __nanosleep(TSAT_CL_SLEEP);
#endif
        w = smem_ld_relaxed_u64(p);
        if ((unsigned)(w >> 32) == seq) return w;
        if ((i & 1023u) == 0) {
            if (*(volatile unsigned*)&ds->xerr) return w;          // already failed: do not wait again
            if (cl_globaltimer() - t0 > kClusterTimeoutNs) {
                atomicExch(&ds->xerr, 1u);
                return w;
            }
        }
    }
}

// own + the CL - 1 partials of message seq in `slots` (exact int64: the sum
// does not depend on the order, every rank gets the same value).  Called by
// one thread (the caller broadcasts).
__device__ __forceinline__ long long cl_recv_sum(const unsigned long long* slots, unsigned CL, unsigned me, unsigned seq,
                                                 long long own, DevScalars* ds) {
    long long s = own;
    for (unsigned r = 0; r < CL; ++r) {
        if (r == me) continue;
        const unsigned long long w0 = cl_wait_word(slots + 2 * r, seq, ds);
        const unsigned long long w1 = cl_wait_word(slots + 2 * r + 1, seq, ds);
        s += (long long)((w0 & 0xffffffffull) | (w1 << 32));
    }
    return s;
}

}  // namespace tsat
