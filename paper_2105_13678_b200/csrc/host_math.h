// Host-side number theory and the Philox4x64-10 generator (no CUDA).
#pragma once
#include <cstdint>
#include <vector>

namespace pa {

// ---------------------------------------------------------------- Philox4x64-10
// Reading A7: numpy.random.Philox convention.  Block b of stream
// (key0, key1) encrypts counter (b + 1, 0, 0, 0); words are the 4 outputs in order.
struct Philox4x64 {
    static void block(uint64_t ctr0, uint64_t key0, uint64_t key1, uint64_t out[4]) {
        uint64_t c[4] = {ctr0, 0, 0, 0};
        uint64_t k0 = key0, k1 = key1;
        for (int round = 0; round < 10; round++) {
            if (round) { k0 += 0x9E3779B97F4A7C15ull; k1 += 0xBB67AE8584CAA73Bull; }
            const __uint128_t p0 = (__uint128_t)0xD2E7470EE14C6C93ull * c[0];
            const __uint128_t p1 = (__uint128_t)0xCA5A826395121157ull * c[2];
            const uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
            const uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
            c[0] = hi1 ^ c[1] ^ k0;
            c[1] = lo1;
            c[2] = hi0 ^ c[3] ^ k1;
            c[3] = lo0;
        }
        for (int i = 0; i < 4; i++) out[i] = c[i];
    }
    // words [w0, w0 + n) of the stream
    static void words(uint64_t key0, uint64_t key1, uint64_t w0, uint64_t n, uint64_t *out) {
        uint64_t blk[4];
        uint64_t cur = ~0ull;
        for (uint64_t w = w0; w < w0 + n; w++) {
            const uint64_t b = w >> 2;
            if (b != cur) { block(b + 1, key0, key1, blk); cur = b; }
            out[w - w0] = blk[w & 3];
        }
    }
};

// ---------------------------------------------------------------- modular helpers
inline uint64_t mulmod64(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((__uint128_t)a * b % m); }
inline uint64_t powmod64(uint64_t a, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    a %= m;
    while (e) { if (e & 1) r = mulmod64(r, a, m); a = mulmod64(a, a, m); e >>= 1; }
    return r;
}
inline uint32_t inv_mod(uint32_t a, uint32_t p) { return (uint32_t)powmod64(a, p - 2, p); }
inline uint32_t to_mont(uint32_t a, uint32_t p) { return (uint32_t)(((uint64_t)a << 32) % p); }
inline uint32_t shoup_of(uint32_t w, uint32_t p) { return (uint32_t)(((uint64_t)w << 32) / p); }

inline uint32_t primitive_root(uint32_t p) {
    std::vector<uint32_t> f;
    uint32_t n = p - 1;
    for (uint32_t d = 2; (uint64_t)d * d <= n; d++)
        if (n % d == 0) { f.push_back(d); while (n % d == 0) n /= d; }
    if (n > 1) f.push_back(n);
    for (uint32_t g = 2;; g++) {
        bool ok = true;
        for (uint32_t q : f) if (powmod64(g, (p - 1) / q, p) == 1) { ok = false; break; }
        if (ok) return g;
    }
}

inline int two_adic(uint32_t p) { int v = 0; uint32_t q = p - 1; while (!(q & 1)) { q >>= 1; v++; } return v; }

// NTT primes p < 2^30 (so 4p < 2^32 for lazy butterflies), p = c 2^v + 1 with
// v >= 20, in decreasing order (the planner takes the largest usable ones first).  Any subset whose 2-adic valuations cover log2 L
// can serve a transform of length L.
static const uint32_t kPrimes[] = {
    1053818881u, 1051721729u, 1045430273u, 1012924417u, 1007681537u, 1004535809u,
    998244353u, 985661441u, 976224257u, 975175681u, 972029953u, 962592769u,
    957349889u, 950009857u, 943718401u, 940572673u, 938475521u, 935329793u,
    925892609u, 924844033u, 919601153u, 918552577u, 913309697u, 907018241u,
    899678209u, 897581057u, 883949569u, 880803841u,
    // smaller primes with 2-adicity >= 22, for transforms of length 2^22 / 2^23
    // (the MH-only comparator over a whole 2.6e8-bit key)
    754974721u, 683671553u, 666894337u, 645922817u, 595591169u, 469762049u, 415236097u,
    377487361u,
};

// Mersenne exponents.
static const uint64_t kMersenne[] = {
    3, 5, 7, 13, 17, 19, 31, 61, 89, 107, 127, 521, 607, 1279, 2203, 2281, 3217,
    4253, 4423, 9689, 9941, 11213, 19937, 21701, 23209, 44497, 86243, 110503,
    132049, 216091, 756839, 859433, 1257787, 1398269, 2976221, 3021377, 6972593,
    13466917, 20996011, 24036583, 25964951, 30402457, 32582657, 37156667,
    42643801, 43112609, 57885161, 74207281,
};

}  // namespace pa
