// Toeplitz-hashing PA, the comparator of Table 1 / Fig. 3 (SURVEY.md
// §8(f) NEXT-4): output_j = XOR_i d[m-1-j+i] x_i over GF(2) (reading A14).
//
// Exact integer convolution, no floating point: every key bit and every
// diagonal bit is one coefficient, so each needed convolution coefficient is a count <= n
// below the single NTT prime, and its parity is the output bit.  The m x n matrix is cut
// into r x r Toeplitz blocks (the Table 1 split): block (o, b) only depends on
// delta = b - o, so with e'_delta the reversed diagonal window of that block,
//   y_o = sum_b e'_(b-o) (*) x_b,   output bit o r + j' = coefficient r - 1 + j' of y_o,
// and a cyclic length L = 2r keeps the needed coefficients free of wrap-around.  The sum
// over b is taken in the transform domain (toeplitz_mac), one inverse per output block.
#pragma once
#include <cstdint>
#include "modarith.cuh"

namespace pa {

// x_b[j] = key bit b r + j (MSB-first within bytes, reading A4), 0 beyond n; out [nb][r]
// (the natural order the forward column pass reads, r = rows * N1).  A thread expands one
// nibble (4 coefficients) into one 16-byte store, so a warp writes 512 contiguous bytes.
__global__ void __launch_bounds__(256) toeplitz_pack_bits(const uint8_t *__restrict__ key, uint64_t n,
                                                          uint64_t total, uint32_t *__restrict__ out) {
    const uint64_t nchunks = total >> 2;                     // total is a multiple of r >= 512
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nchunks;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t0 = i << 2;                          // first bit of the nibble
        uint32_t nib = 0;
        if (t0 < n) {
            const uint32_t byte = PA_LDG(key + (t0 >> 3));
            nib = (i & 1) ? (byte & 0xFu) : (byte >> 4);      // MSB-first: even chunk = high nibble
            if (t0 + 4 > n) nib &= (0xF0u >> (n - t0)) & 0xFu;   // bits >= n are 0
        }
        PA_AT(reinterpret_cast<uint4 *>(out) + i) = make_uint4((nib >> 3) & 1u, (nib >> 2) & 1u, (nib >> 1) & 1u, nib & 1u);
    }
}

// Reversed diagonal windows: out[dp][s] = d[m + (dp - (O-1)) r + r - 2 - s] for s <= 2r - 2,
// 0 for s = 2r - 1 and for indices outside [0, n + m - 1).  d is LSB-first in 32-bit words
// (reading A15).  out [ne][L], L = 2r.
__global__ void __launch_bounds__(256) toeplitz_pack_diag(const uint32_t *__restrict__ dw, uint64_t nd, uint64_t m,
                                                          uint32_t log2r, uint32_t O, uint32_t ne,
                                                          uint32_t *__restrict__ out) {
    const uint64_t r = 1ull << log2r, L = 2 * r;
    const uint64_t total = (uint64_t)ne * L;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t dp = t >> (log2r + 1), s = t & (L - 1);
        uint32_t v = 0;
        if (s + 1 < L) {
            const int64_t idx = (int64_t)m + ((int64_t)dp - (int64_t)(O - 1)) * (int64_t)r + (int64_t)r - 2 - (int64_t)s;
            if (idx >= 0 && (uint64_t)idx < nd) v = (PA_LDG(dw + (idx >> 5)) >> (idx & 31)) & 1u;
        }
        PA_AT(out + t) = v;
    }
}

// acc[o'][e] = sum_{b in [b0, b1)} Xh[b][e] * Eh[b - o + no - 1][e] mod p for the output blocks
// o = o0 + o' (o' < O) of a group, i.e. the transform-domain sum over the input blocks of a
// group (canonical).  Eh holds T(e') L^-1 R (Montgomery), Xh plain transforms, so mul_mont
// leaves T(x) T(e') / L.  ebase = b0 - o0 + no - O: for a fixed e the E index window
// ebase + (b - b0) .. + O - 1 slides by one per input block: O registers, one new load.
// The products are summed as plain 64-bit integers (one wide multiply-add each): x, w < p <
// 2^30, so seven products stay below 3 p 2^32 and one REDC per seven blocks turns the group
// into sum x w R^-1 mod p -- the same value as seven Montgomery products, at a fraction of
// the instructions.
constexpr int kTzMaxOut = 16;                 // output blocks per MAC launch (O registers)
constexpr int kTzGroup = 7;
template <int O>
__global__ void __launch_bounds__(256) toeplitz_mac(const uint32_t *__restrict__ Xh, const uint32_t *__restrict__ Eh,
                                                    uint32_t b0, uint32_t b1, uint32_t ebase, uint32_t L, uint32_t p,
                                                    uint32_t pinv, uint32_t *__restrict__ acc) {
    const uint32_t p2 = 2 * p;
    const uint32_t nb = b1 - b0;
    Xh += (size_t)b0 * L;
    Eh += (size_t)ebase * L;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < L; e += gridDim.x * blockDim.x) {
        uint32_t a[O], w[O];
        uint64_t t[O];
#pragma unroll
        for (int o = 0; o < O; o++) {
            a[o] = 0;
            t[o] = 0;
            w[o] = PA_LDG(Eh + (size_t)(O - 1 - o) * L + e);        // w[o] = E[ebase + b + O - 1 - o] at b = b0
        }
        uint32_t g = 0;
#pragma unroll 7
        for (uint32_t b = 0; b < nb; b++) {
            const uint32_t x = PA_LDG(Xh + (size_t)b * L + e);
#pragma unroll
            for (int o = 0; o < O; o++) t[o] = mad_wide(x, w[o], t[o]);
            if (++g == kTzGroup) {
                g = 0;
#pragma unroll
                for (int o = 0; o < O; o++) {
                    a[o] = red2p(a[o] + red2p(redc64(t[o], p, pinv), p2), p2);
                    t[o] = 0;
                }
            }
            if (b + 1 < nb) {
#pragma unroll
                for (int o = O - 1; o > 0; o--) w[o] = w[o - 1];
                w[0] = PA_LDG(Eh + (size_t)(b + O) * L + e);
            }
        }
#pragma unroll
        for (int o = 0; o < O; o++) {
            a[o] = red2p(a[o] + red2p(redc64(t[o], p, pinv), p2), p2);
            PA_AT(acc + (size_t)o * L + e) = red1p(a[o], p);
        }
    }
}

// Output bit j < m = parity of coefficient r - 1 + (j mod r) of block j / r (canonical
// residues = exact counts < p).  One warp per 32 output bits: ballot, emitted MSB-first.
// With several input-block groups (their counts each below p, the sum possibly not) every
// group's parities are XORed into the output (xor_in): the parity of a sum is the XOR of the
// parities.
__global__ void __launch_bounds__(256) toeplitz_extract(const uint32_t *__restrict__ acc, uint32_t log2r, uint32_t L,
                                                        uint64_t m, uint8_t *__restrict__ out, uint64_t nbytes,
                                                        uint32_t xor_in) {
    const uint64_t r = 1ull << log2r;
    const int lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t wq = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; wq * 32 < m; wq += nwarps) {
        const uint64_t j = wq * 32 + lane;
        uint32_t bit = 0;
        if (j < m) bit = PA_LDG(acc + (j >> log2r) * L + (r - 1) + (j & (r - 1))) & 1u;
        const uint32_t mask = __brev(__ballot_sync(0xFFFFFFFFu, bit));   // bit 31 = output bit 32 wq
        if (lane < 4) {
            const uint64_t q = wq * 4 + lane;
            if (q < nbytes) {
                const uint8_t v = (uint8_t)(mask >> (24 - 8 * lane));
                PA_AT(out + q) = xor_in ? (uint8_t)(PA_AT(out + q) ^ v) : v;
            }
        }
    }
}

}  // namespace pa
