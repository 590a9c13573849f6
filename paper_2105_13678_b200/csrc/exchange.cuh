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

// in[e] < 2^64 (a sum of canonical residues over the ranks) -> in[e] mod q_{e >> log2L}
__global__ void __launch_bounds__(256) acc_import_u64(const uint64_t *__restrict__ in, uint32_t log2L, uint64_t total,
                                                      const PrimeSet ks, uint32_t *__restrict__ out) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = ks.k[e >> log2L].p;
        PA_AT(out + e) = (uint32_t)(PA_AT(in + e) % q);
    }
}

}  // namespace pa
