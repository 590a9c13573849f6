// Fresh hash keys per job on the GPU: the hash-key expansion of
// reading A7 -- Philox4x64-10 with numpy's counter convention, stream (seed, s), ceil(w/64)
// little-endian words per draw, masked to w bits; a_i redrawn while equal to 2^gamma - 1
// (PAPER.md:142); b with bit 0 set; c as drawn -- computed
// by device kernels so a context can be re-keyed without a host round trip.
#pragma once
#include <cstdint>
#include "debug.cuh"

namespace pa {

__device__ __forceinline__ void philox4x64_10_dev(uint64_t ctr0, uint64_t k0, uint64_t k1, uint64_t out[4]) {
    uint64_t c0 = ctr0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
    for (int round = 0; round < 10; round++) {
        if (round) { k0 += 0x9E3779B97F4A7C15ull; k1 += 0xBB67AE8584CAA73Bull; }
        const uint64_t m0 = 0xD2E7470EE14C6C93ull, m1 = 0xCA5A826395121157ull;
        const uint64_t hi0 = __umul64hi(m0, c0), lo0 = m0 * c0;
        const uint64_t hi1 = __umul64hi(m1, c2), lo1 = m1 * c2;
        const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// First draw of every vector, all vectors at once: out[v][0..nw32) = draw 0 of stream
// (seed, s0 + v); ok[v] = 1 if it is not all ones (ok zeroed by the caller).  Grid-stride
// over (vector, philox block): one philox call yields 8 output words.  The 64-bit word e of
// philox block blk is out words 8 blk + 2e, +1 (little-endian), so a warp whose 32 blocks lie
// inside one vector (8-byte aligned, top word excluded) transposes its 4 x 32 words through
// shared memory and stores 128 consecutive 64-bit words; other warps store word by word.
constexpr int kExpT = 256;
__global__ void __launch_bounds__(kExpT) expand_keys_first(uint64_t seed, uint64_t s0, uint64_t bits, uint32_t nw32,
                                                         uint32_t nvec, int force_odd, uint32_t *__restrict__ out,
                                                         uint32_t *ok) {
    __shared__ uint64_t sbuf[kExpT / 32][4 * 33];
    const uint64_t nw64 = (bits + 63) >> 6;
    const uint64_t nblk = (nw64 + 3) >> 2;                     // philox blocks per draw 0
    const uint32_t topmask = (bits % 32) ? (uint32_t)((1ull << (bits % 32)) - 1) : 0xFFFFFFFFu;
    const uint64_t total = nblk * nvec;
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    uint64_t *sw = sbuf[wq];
    const uint64_t stride = (uint64_t)gridDim.x * kExpT;
    for (uint64_t tb = blockIdx.x * (uint64_t)kExpT + (threadIdx.x & ~31u); tb < total; tb += stride) {
        const uint64_t t = tb + lane;
        const bool live = t < total;
        const uint32_t v = !live ? 0u : (t >> 32) ? (uint32_t)(t / nblk) : (uint32_t)t / (uint32_t)nblk;
        const uint64_t blk = t - (uint64_t)v * nblk;
        uint64_t r[4];
        philox4x64_10_dev(blk + 1, seed, s0 + v, r);
        uint32_t differs = 0;
#pragma unroll
        for (int e = 0; e < 4; e++) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint64_t i32 = 8 * blk + 2 * e + h;
                uint32_t x = (uint32_t)(r[e] >> (32 * h));
                if (i32 == nw32 - 1) x &= topmask;
                if (i32 == 0 && force_odd) x |= 1u;
                if (i32 < nw32) differs |= (x != (i32 == nw32 - 1 ? topmask : 0xFFFFFFFFu));
                r[e] = h ? ((r[e] & 0xFFFFFFFFull) | ((uint64_t)x << 32)) : ((r[e] & ~0xFFFFFFFFull) | x);
            }
        }
        if (live && differs && !ok[v]) ok[v] = 1u;           // benign race: all writers store 1
        const uint32_t v0 = __shfl_sync(0xFFFFFFFFu, v, 0);
        const uint64_t blk0 = __shfl_sync(0xFFFFFFFFu, blk, 0);
        const bool fast = __all_sync(0xFFFFFFFFu, live && v == v0 && 8 * (blk + 1) < nw32) &&
                          (((uint64_t)v0 * nw32) & 1) == 0;
        if (fast) {
#pragma unroll
            for (int e = 0; e < 4; e++) sw[e * 33 + lane] = r[e];
            __syncwarp();
            uint64_t *o64 = reinterpret_cast<uint64_t *>(out + (size_t)v0 * nw32) + 4 * blk0;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int q = 32 * k + lane;                    // word q of the warp's 128
                PA_AT(o64 + q) = sw[(q & 3) * 33 + (q >> 2)];
            }
            __syncwarp();
        } else if (live) {
            uint32_t *o = out + (size_t)v * nw32;
#pragma unroll
            for (int e = 0; e < 4; e++)
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const uint64_t i32 = 8 * blk + 2 * e + h;
                    if (i32 < nw32) PA_AT(o + i32) = (uint32_t)(r[e] >> (32 * h));
                }
        }
    }
}

// Redraws of the rejected vectors (ok[v] == 0: draw 0 was all ones, probability 2^-bits):
// out[v] = the first later draw of stream (seed, s0 + v) that is not all ones (PAPER.md:142,
// reading A7).  One CTA per vector; accepted vectors return at once.
__global__ void __launch_bounds__(256) expand_keys_dev(uint64_t seed, uint64_t s0, uint64_t bits, uint32_t nw32,
                                                       int reject, int force_odd, uint32_t *__restrict__ out,
                                                       const uint32_t *ok = nullptr) {
    if (ok && ok[blockIdx.x]) return;
    const uint64_t s = s0 + blockIdx.x;
    uint32_t *o = out + (size_t)blockIdx.x * nw32;
    const uint64_t nw64 = (bits + 63) >> 6;
    const uint32_t topmask = (bits % 32) ? (uint32_t)((1ull << (bits % 32)) - 1) : 0xFFFFFFFFu;
    for (uint64_t draw = ok ? 1 : 0;; draw++) {
        // stream words [draw nw64, (draw + 1) nw64); philox block b holds words 4b .. 4b+3
        const uint64_t w0 = draw * nw64;
        int allones = 1;
        for (uint64_t q = threadIdx.x; q < (nw64 + 3) / 4 + 1; q += blockDim.x) {
            const uint64_t blk = (w0 >> 2) + q;                 // philox block (counter blk + 1)
            uint64_t r[4];
            philox4x64_10_dev(blk + 1, seed, s, r);
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const uint64_t gw = 4 * blk + e;                  // stream word index
                if (gw < w0 || gw >= w0 + nw64) continue;
                const uint64_t lw = gw - w0;                      // word within the draw
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const uint64_t i32 = 2 * lw + h;
                    if (i32 >= nw32) continue;
                    uint32_t v = (uint32_t)(r[e] >> (32 * h));
                    if (i32 == nw32 - 1) v &= topmask;
                    if (i32 == 0 && force_odd) v |= 1u;
                    PA_AT(o + i32) = v;
                    allones &= (v == (i32 == nw32 - 1 ? topmask : 0xFFFFFFFFu));
                }
            }
        }
        if (!reject) return;
        if (!__syncthreads_and(allones)) return;            // accepted (uniform)
    }
}

}  // namespace pa
