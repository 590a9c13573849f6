// Modular arithmetic for 30-bit NTT primes p < 2^30 on 32-bit integer pipes.
//
// Why 30-bit primes: the MMH/MH products ("its main part is large
// number multiplications") are exact integer convolutions.  On sm_100a the integer
// datapath is 32 bits wide; a butterfly mod a 30-bit prime is ~7 IMAD/ALU
// instructions (Shoup multiply + lazy Harvey reduction), against ~35 for a 64-bit
// Goldilocks butterfly.  Several primes are recombined by CRT (crt_carry.cuh).
//
// Value ranges ("lazy" representation): residues live in [0, 2p) between
// operations; 4p < 2^32 so a sum of two never overflows.
#pragma once
#include <cstdint>
#include "debug.cuh"

namespace pa {

constexpr int kMaxPrimes = 16;   // NTT primes per product (CRT modulus <= 16 words)

struct alignas(16) PrimeK {  // per-prime constants passed to kernels
    uint32_t p;            // prime, < 2^30
    uint32_t p2;           // 2p
    uint32_t pinv;         // p^{-1} mod 2^32   (Montgomery, R = 2^32)
    uint32_t r2;           // R^2 mod p         (to Montgomery form)
    uint32_t pw[8];        // 2^(32 i) mod p, i < 8 (multiword limb reduction)
    uint32_t pw24[10];     // 2^(24 j) mod p, j < 10 (the same, over 24-bit chunks)
    uint32_t pw28[10];     // 2^(28 j) mod p, j < 10 (over 28-bit chunks)
    uint32_t pad_[4];
};

// All primes of a stage by value: passed as a kernel parameter, so the per-prime constants
// are constant-bank operands of the multiply instructions (no shared/global loads)
struct PrimeSet {
    PrimeK k[kMaxPrimes];
};

// a * b + c with a 32x32 -> 64-bit multiply (one IMAD.WIDE.U32)
__device__ __forceinline__ uint64_t mad_wide(uint32_t a, uint32_t b, uint64_t c) {
    uint64_t r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
    return r;
}

// REDC of t < 3 p 2^32: t 2^-32 mod p in [0, 4p)
__device__ __forceinline__ uint32_t redc64(uint64_t t, uint32_t p, uint32_t pinv) {
    const uint32_t lo = (uint32_t)t, hi = (uint32_t)(t >> 32);
    return hi - __umulhi(lo * pinv, p) + p;
}

// s in [0, 4p) -> [0, 2p)
__device__ __forceinline__ uint32_t red2p(uint32_t s, uint32_t p2) { return min(s, s - p2); }
// s in [0, 2p) -> [0, p)
__device__ __forceinline__ uint32_t red1p(uint32_t s, uint32_t p) { return min(s, s - p); }

// Shoup multiplication by a constant w < p with wp = floor(w 2^32 / p):
// returns x*w mod p in [0, 2p) for any 32-bit x.
__device__ __forceinline__ uint32_t mul_shoup(uint32_t x, uint32_t w, uint32_t wp, uint32_t p) {
    uint32_t q = __umulhi(x, wp);
    return x * w - q * p;
}

// Montgomery product x*y*2^-32 mod p in (0, 2p), valid for any 32-bit x and y < p.
__device__ __forceinline__ uint32_t mul_mont(uint32_t x, uint32_t y, uint32_t p, uint32_t pinv) {
    uint64_t t = (uint64_t)x * y;
    uint32_t lo = (uint32_t)t, hi = (uint32_t)(t >> 32);
    uint32_t q = lo * pinv;
    return hi - __umulhi(q, p) + p;
}

// Gentleman-Sande (DIF) butterfly: (a, b) -> (a + b, (a - b) w), inputs/outputs in [0, 2p).
__device__ __forceinline__ void bfly_dif(uint32_t &a, uint32_t &b, uint32_t w, uint32_t wp,
                                         uint32_t p, uint32_t p2) {
    uint32_t s = red2p(a + b, p2);
    uint32_t d = a - b + p2;
    b = mul_shoup(d, w, wp, p);
    a = s;
}
__device__ __forceinline__ void bfly_dif1(uint32_t &a, uint32_t &b, uint32_t p2) {
    uint32_t s = red2p(a + b, p2);
    uint32_t d = red2p(a - b + p2, p2);
    a = s;
    b = d;
}

}  // namespace pa
