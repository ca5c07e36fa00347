// peer.cuh - exchanges over NVLink peer memory inside the step kernels
// (SURVEY §8(e)).
//
// Each rank owns one exchange buffer (PeerLayout); every rank writes its own
// slot of every rank's buffer with system-scope stores and publishes it with
// a release store of the exchange generation into the slot's flag.  A reader
// acquires the W flags of its local buffer and sums the W slots in rank
// order.  Reduced values are int64 (fixed point) or maxima, so every rank
// computes identical results, bit for bit equal to W = 1.
//
// Row values (J, Q) need no fence: each int64 travels as two u64 words
// (generation << 32 | 32-bit half), and a naturally aligned 8-byte store is
// single-copy atomic, so a reader that sees the expected generation in both
// words has the value (relaxed.sys stores and loads, L1 bypassed).  The
// per-step scalars use a release-stored flag instead (4 words, once a step).
// Row slots are reused every iteration: a rank writes the rows
// of generation g+1 only after receiving every rank's g+1 scalars, which each
// rank sends after its k_update(g) has completed, so no row slot is
// overwritten before it is read.  The scalar slots themselves are
// double-buffered by generation parity (a rank can be at most one generation
// ahead of a CTA that has not yet read them).
//
// A wait that exceeds kPeerTimeoutNs sets DevScalars::xerr and returns (the
// host reports TSAT_E_NCCL): a broken peer can never hang the GPU.
#pragma once

#include <cstdint>

#include "tsat_internal.h"

namespace tsat {

constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys(long long* p, long long v) {
    asm volatile("st.relaxed.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ long long ld_relaxed_sys(const long long* p) {
    long long v;
    asm volatile("ld.relaxed.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Wait until flag >= gen (wrap-safe); false on timeout or a previous error.
__device__ __forceinline__ bool peer_wait(const unsigned* flag, unsigned gen, DevScalars* ds) {
    if ((int)(ld_acquire_sys(flag) - gen) >= 0) return true;
    const unsigned long long t0 = globaltimer_ns();
    unsigned ns = 64;
    while ((int)(ld_acquire_sys(flag) - gen) < 0) {
        if (*(volatile unsigned*)&ds->xerr) return false;
        __nanosleep(ns);
        if (ns < 2048) ns <<= 1;
        if (globaltimer_ns() - t0 > kPeerTimeoutNs) {
            atomicExch(&ds->xerr, 1u);
            return false;
        }
    }
    return true;
}

// Row all-reduce (sum of one int64 per rank), which = 0 (J) or 1 (Q); one
// thread sends, later one thread receives (they may be apart in time).  A
// rank's own partial never goes through memory: the receiver adds it locally
// (int64 sums are exact in any order), so only the W - 1 remote slots are
// written and awaited.
__device__ __forceinline__ void peer_row_send(const PeerArgs& px, int which, int v, long long val, unsigned gen) {
    const size_t slot = 2 * ((size_t)px.rank * px.V + v);
    const unsigned long long g = (unsigned long long)gen << 32;
    const unsigned long long w0 = g | (unsigned long long)(unsigned)val;
    const unsigned long long w1 = g | (unsigned long long)(unsigned)((unsigned long long)val >> 32);
    for (int p = 0; p < px.W; ++p) {
        if (p == px.rank) continue;
        unsigned long long* d = reinterpret_cast<unsigned long long*>(px.xb[p] + (which ? px.L.qx : px.L.jx)) + slot;
        st_relaxed_sys_u64(d, w0);
        st_relaxed_sys_u64(d + 1, w1);
    }
}

__device__ __forceinline__ long long peer_row_recv(const PeerArgs& px, int which, int v, unsigned gen,
                                                   DevScalars* ds, long long own) {
    const unsigned long long* xs =
        reinterpret_cast<const unsigned long long*>(px.xb[px.rank] + (which ? px.L.qx : px.L.jx));
    long long s = own;
    for (int r = 0; r < px.W; ++r) {
        if (r == px.rank) continue;
        const unsigned long long* q = xs + 2 * ((size_t)r * px.V + v);
        unsigned long long w0 = ld_relaxed_sys_u64(q), w1 = ld_relaxed_sys_u64(q + 1);
        if ((unsigned)(w0 >> 32) != gen || (unsigned)(w1 >> 32) != gen) {
            const unsigned long long t0 = globaltimer_ns();
            unsigned ns = 32;
            while ((unsigned)(w0 >> 32) != gen || (unsigned)(w1 >> 32) != gen) {
                if (*(volatile unsigned*)&ds->xerr) return 0;
                __nanosleep(ns);
                if (ns < 1024) ns <<= 1;
                if (globaltimer_ns() - t0 > kPeerTimeoutNs) {
                    atomicExch(&ds->xerr, 1u);
                    return 0;
                }
                w0 = ld_relaxed_sys_u64(q);
                w1 = ld_relaxed_sys_u64(q + 1);
            }
        }
        s += (long long)(((w1 & 0xffffffffull) << 32) | (w0 & 0xffffffffull));
    }
    return s;
}

// Per-iteration scalars: x = {~best key, gmax bits, thmax bits, loss fixed point};
// the own rank's values are combined locally by the receiver.
__device__ __forceinline__ void peer_send_scalars(const PeerArgs& px, const unsigned long long (&x)[4], unsigned gen) {
    const int par = (int)(gen & 1u);
    for (int p = 0; p < px.W; ++p) {
        if (p == px.rank) continue;
        long long* d = reinterpret_cast<long long*>(px.xb[p] + px.L.sx) + 4 * ((size_t)par * px.W + px.rank);
#pragma unroll
        for (int k = 0; k < 4; ++k) st_relaxed_sys(d + k, (long long)x[k]);
        st_release_sys(reinterpret_cast<unsigned*>(px.xb[p] + px.L.sf) + (size_t)par * px.W + px.rank, gen);
    }
}

// Combine: max of ~key, gmax, thmax (non-negative bit patterns order like
// their values); sum of the loss.  Returns false on timeout.
__device__ __forceinline__ bool peer_recv_scalars(const PeerArgs& px, unsigned gen, DevScalars* ds,
                                                  const unsigned long long (&own)[4], unsigned long long (&out)[4]) {
    const int par = (int)(gen & 1u);
    const long long* xs = reinterpret_cast<const long long*>(px.xb[px.rank] + px.L.sx) + (size_t)4 * par * px.W;
    const unsigned* fs = reinterpret_cast<const unsigned*>(px.xb[px.rank] + px.L.sf) + (size_t)par * px.W;
#pragma unroll
    for (int k = 0; k < 4; ++k) out[k] = own[k];
    for (int r = 0; r < px.W; ++r) {
        if (r == px.rank) continue;
        if (!peer_wait(fs + r, gen, ds)) return false;
        unsigned long long x[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = (unsigned long long)ld_relaxed_sys(xs + 4 * r + k);
        out[0] = x[0] > out[0] ? x[0] : out[0];
        out[1] = x[1] > out[1] ? x[1] : out[1];
        out[2] = x[2] > out[2] ? x[2] : out[2];
        out[3] += x[3];
    }
    return true;
}

}  // namespace tsat
