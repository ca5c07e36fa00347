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
// Ordering: slot store (relaxed.sys) -> flag store (release.sys) on the
// writer; flag load (acquire.sys) -> slot load (relaxed.sys, bypasses L1) on
// the reader.  Row slots are reused every iteration: a rank writes the rows
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

// All-reduce (sum) of one int64 row value: which = 0 (J) or 1 (Q).
// Called by one thread.
__device__ __forceinline__ long long peer_row_sum(const PeerArgs& px, int which, int v, long long val, unsigned gen,
                                                  DevScalars* ds) {
    const size_t ox = which ? px.L.qx : px.L.jx, of = which ? px.L.qf : px.L.jf;
    const size_t slot = (size_t)px.rank * px.V + v;
    for (int p = 0; p < px.W; ++p) {
        st_relaxed_sys(reinterpret_cast<long long*>(px.xb[p] + ox) + slot, val);
        st_release_sys(reinterpret_cast<unsigned*>(px.xb[p] + of) + slot, gen);
    }
    const long long* xs = reinterpret_cast<const long long*>(px.xb[px.rank] + ox);
    const unsigned* fs = reinterpret_cast<const unsigned*>(px.xb[px.rank] + of);
    long long s = 0;
    for (int r = 0; r < px.W; ++r) {
        const size_t i = (size_t)r * px.V + v;
        if (!peer_wait(fs + i, gen, ds)) return val;
        s += ld_relaxed_sys(xs + i);
    }
    return s;
}

// Per-iteration scalars: x = {~best key, gmax bits, thmax bits, loss fixed point}.
__device__ __forceinline__ void peer_send_scalars(const PeerArgs& px, const unsigned long long (&x)[4], unsigned gen) {
    const int par = (int)(gen & 1u);
    for (int p = 0; p < px.W; ++p) {
        long long* d = reinterpret_cast<long long*>(px.xb[p] + px.L.sx) + 4 * ((size_t)par * px.W + px.rank);
#pragma unroll
        for (int k = 0; k < 4; ++k) st_relaxed_sys(d + k, (long long)x[k]);
        st_release_sys(reinterpret_cast<unsigned*>(px.xb[p] + px.L.sf) + (size_t)par * px.W + px.rank, gen);
    }
}

// Combine: max of ~key, gmax, thmax (non-negative bit patterns order like
// their values); sum of the loss.  Returns false on timeout.
__device__ __forceinline__ bool peer_recv_scalars(const PeerArgs& px, unsigned gen, DevScalars* ds,
                                                  unsigned long long (&out)[4]) {
    const int par = (int)(gen & 1u);
    const long long* xs = reinterpret_cast<const long long*>(px.xb[px.rank] + px.L.sx) + (size_t)4 * par * px.W;
    const unsigned* fs = reinterpret_cast<const unsigned*>(px.xb[px.rank] + px.L.sf) + (size_t)par * px.W;
    out[0] = out[1] = out[2] = out[3] = 0ull;
    for (int r = 0; r < px.W; ++r) {
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
