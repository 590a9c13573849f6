// The one exchange step of the multi-GPU path (MMH is linear over a
// partition of the blocks, "split and separately handle").
//
// Each rank holds the transform-domain accumulator of its blocks, acc = sum_{i in shard}
// NTT(x_i) (.) NTT(a_i) mod q_j for every NTT prime q_j (the row MAC's output, in up to
// nslot partial slots, each value < 4 q_j).  Because the transform is linear, the sum of
// the ranks' accumulators mod q_j is the whole key's accumulator: one reduction replaces
// the per-rank inverse transform, CRT and carries (only the root runs them).
//
//   acc_export<T>: slots -> one canonical word per element (< q_j), as uint32 (reduced
//                  with a 32-bit NCCL sum while world * q_j < 2^32, i.e. world <= 4) or
//                  uint64 (any world);
//   acc_import_u64: the 64-bit sums -> canonical uint32 residues for the inverse pass.
#pragma once
#include <cstdint>
#include "modarith.cuh"

namespace pa {

// out[e] = (sum_s acc[s * slot_stride + e]) mod q_{e >> log2L}, e < P << log2L
template <class T>
__global__ void __launch_bounds__(256) acc_export(const uint32_t *__restrict__ acc, uint32_t nslot, uint64_t slot_stride,
                                                  uint32_t log2L, uint64_t total, const PrimeSet ks, T *__restrict__ out) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t pi = (uint32_t)(e >> log2L);
        const uint32_t q = ks.k[pi].p, q2 = ks.k[pi].p2;
        uint32_t v = 0;
        for (uint32_t s = 0; s < nslot; s++) {
            const uint32_t a = red1p(red2p(PA_AT(acc + s * slot_stride + e), q2), q);   // < 4q -> < q
            v = red1p(v + a, q);
        }
        PA_AT(out + e) = (T)v;
    }
}

// in[e] < 2^64 (a sum of canonical residues over the ranks) -> in[e] mod q_{e >> log2L};
// ZERO: the input is cleared as it is read (the P2P receive buffer, ready for its next use)
template <bool ZERO = false>
__global__ void __launch_bounds__(256) acc_import_u64(uint64_t *__restrict__ in, uint32_t log2L, uint64_t total,
                                                      const PrimeSet ks, uint32_t *__restrict__ out) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = ks.k[e >> log2L].p;
        PA_AT(out + e) = (uint32_t)(PA_AT(in + e) % q);
        if (ZERO) PA_AT(in + e) = 0ull;
    }
}

// ---- P2P exchange (pa_params.p2p): the ranks' row MACs add their partial accumulators
// straight into the root's 64-bit receive buffer over NVLink (row_mac mode 3, so the transfer
// overlaps the multiply-accumulate), and 32-bit counters in each GPU's own memory order the
// uses of a buffer.  A counter is incremented by a remote (or local) release atomic and
// waited on locally; every counter has a local "expected" companion that the wait advances,
// so every kernel argument stays the same from one use to the next (graph replay).
constexpr int kMaxWorld = 64;
constexpr uint32_t kFlagWords = 32;          // one counter per 128-byte line
struct PeerFlags {
    uint32_t *p[kMaxWorld];
};

// for i < n: wait until flags[i] >= expected[i] + 1 (wrap-safe), then expected[i] += 1.
// A peer that never signals (a rank that stopped calling) must not hang the GPU: after
// kP2PTimeoutNs the wait gives up and traps, which fails the stream with an error.
constexpr uint64_t kP2PTimeoutNs = 20ull * 1000 * 1000 * 1000;
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__global__ void __launch_bounds__(64) p2p_wait(const uint32_t *flags, uint32_t *expected, uint32_t n) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t want = PA_AT(expected + (size_t)i * kFlagWords) + 1u;
        const uint32_t *f = flags + (size_t)i * kFlagWords;
        PA_CK(f, 4);
        const uint64_t t0 = globaltimer_ns();
        for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
            if ((int32_t)(v - want) >= 0) break;
            if (globaltimer_ns() - t0 > kP2PTimeoutNs) {
                printf("pa p2p_wait: counter %u stuck at %u, expected %u (a rank stopped?)\n", i, v, want);
                __trap();
            }
            __nanosleep(256);
        }
        PA_AT(expected + (size_t)i * kFlagWords) = want;
    }
}

// for i < n: counter P.p[i] += 1, a system-scope release after everything this stream did
// before (the preceding kernels' peer writes ended with a system fence)
__global__ void __launch_bounds__(64) p2p_signal(PeerFlags P, uint32_t n) {
    const uint32_t i = threadIdx.x;
    if (i < n) {
        __threadfence_system();
        uint32_t old;
        asm volatile("atom.add.release.sys.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(P.p[i]) : "memory");
        (void)old;
    }
}

}  // namespace pa
