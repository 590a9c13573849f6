// Column and row pass kernels of the four-step NTT (see ntt.cuh), with the hot-path
// fusions:  S1 pack (key bits -> B-bit limbs -> residues) inside the forward column
// pass, S3 multiply-accumulate against the precomputed transforms of the a_i inside
// the forward row pass (Eq. 2's sum done in the transform domain), and
// the inverse four-step twiddle inside the inverse row pass.
#pragma once
#include <cstdint>
#include "modarith.cuh"
#include "ntt.cuh"
#include "bulk.cuh"

namespace pa {

// ---------------------------------------------------------------- limb sources
// S1 ("split the input bit sequence and map it to a prime field"):
// block i of the key = bytes [i R, (i+1) R) of the slice, a big-endian integer
// (MSB-first bits, reading A4); limb j = bits [B j, B j + B) of that integer.
struct KeySrc {
    const uint8_t *key;     // slice base
    uint64_t nbytes;        // valid bytes in the slice (bytes beyond read as 0)
    uint32_t last_mask;     // mask of the byte nbytes-1 (bits >= n ignored)
    uint32_t blk_bytes;     // R = r / 8
    uint32_t limb_bytes;    // B / 8
    uint32_t wx;            // limbs per block = ceil(r / B)
    uint32_t aligned;       // key pointer 4-byte aligned
};

__device__ __forceinline__ uint32_t key_word(const KeySrc &s, int64_t widx) {
    const int64_t base = widx * 4;
    if (base < 0) return 0;
    if (s.aligned && base + 4 < (int64_t)s.nbytes)
        return PA_LDG(reinterpret_cast<const uint32_t *>(s.key) + widx);
    uint32_t w = 0;
#pragma unroll
    for (int b = 0; b < 4; b++) {
        const int64_t pos = base + b;
        if (pos < (int64_t)s.nbytes) {
            uint32_t v = PA_AT(s.key + pos);
            if (pos == (int64_t)s.nbytes - 1) v &= s.last_mask;
            w |= v << (8 * b);
        }
    }
    return w;
}

__device__ __forceinline__ uint64_t key_limb(const KeySrc &s, uint32_t blk, uint32_t j) {
    if (j >= s.wx) return 0;
    const int64_t start = (int64_t)blk * s.blk_bytes;
    const int64_t end = start + s.blk_bytes;
    int64_t lo = end - (int64_t)(j + 1) * s.limb_bytes;
    const int64_t hi = end - (int64_t)j * s.limb_bytes;
    if (lo < start) lo = start;
    const int nb = (int)(hi - lo);                          // 1..8 bytes
    const int64_t w0 = lo >> 2;
    const int sh = (int)(lo & 3) * 8;
    const uint32_t a0 = key_word(s, w0), a1 = key_word(s, w0 + 1), a2 = key_word(s, w0 + 2);
    const uint32_t lo32 = __funnelshift_r(a0, a1, sh);      // bytes lo..lo+3 (memory order)
    const uint32_t hi32 = __funnelshift_r(a1, a2, sh);      // bytes lo+4..lo+7
    // big-endian value of the first nb bytes
    const uint64_t be = ((uint64_t)__byte_perm(lo32, 0, 0x0123) << 32) | __byte_perm(hi32, 0, 0x0123);
    return be >> (64 - 8 * nb);
}

// Multiword limb (B > 56 bits): w[i] = bits [32 i, 32 i + 32) of limb j, i < NW.
// Word i is the big-endian value of the 4 key bytes ending 4 i bytes before the limb's
// last byte; bytes before the limb (or the block) read as 0.
template <int NW>
__device__ __forceinline__ void key_limb_words(const KeySrc &s, uint32_t blk, uint32_t j, uint32_t (&w)[NW]) {
    if (j >= s.wx) {
#pragma unroll
        for (int i = 0; i < NW; i++) w[i] = 0;
        return;
    }
    const int64_t start = (int64_t)blk * s.blk_bytes;
    const int64_t end = start + s.blk_bytes;
    const int64_t hi = end - (int64_t)j * s.limb_bytes;
    int64_t lo = hi - (int64_t)s.limb_bytes;
    if (lo < start) lo = start;
#pragma unroll
    for (int i = 0; i < NW; i++) {
        const int64_t pos = hi - 4 * (i + 1);               // first (most significant) byte
        const int64_t wi = pos >> 2;                          // floor for negative too
        const int sh = (int)(pos & 3) * 8;
        const uint32_t a0 = key_word(s, wi), a1 = key_word(s, wi + 1);
        uint32_t v = __byte_perm(__funnelshift_r(a0, a1, sh), 0, 0x0123);
        const int64_t below = lo - pos;                       // leading bytes outside the limb
        if (below >= 4) v = 0;
        else if (below > 0) v &= 0xFFFFFFFFu >> (8 * below);
        w[i] = v;
    }
}

// Little-endian 32-bit word vectors (a_i, b, y): limb j = bits [B j, B j + B).
struct WordSrc {
    const uint32_t *w;
    uint32_t words;         // words per vector (stride); words beyond are read as 0
    uint32_t limb_bits;     // B
    uint32_t nlimbs;        // limbs per vector
};

__device__ __forceinline__ uint64_t word_limb(const WordSrc &s, uint32_t vec, uint32_t j) {
    if (j >= s.nlimbs) return 0;
    const uint64_t bit = (uint64_t)j * s.limb_bits;
    const uint32_t wi = (uint32_t)(bit >> 5);
    const int sh = (int)(bit & 31);
    const uint32_t *base = s.w + (size_t)vec * s.words;
    const uint32_t a0 = wi < s.words ? PA_LDG(base + wi) : 0u;
    const uint32_t a1 = wi + 1 < s.words ? PA_LDG(base + wi + 1) : 0u;
    const uint32_t a2 = wi + 2 < s.words ? PA_LDG(base + wi + 2) : 0u;
    const uint64_t v = ((uint64_t)__funnelshift_r(a1, a2, sh) << 32) | __funnelshift_r(a0, a1, sh);
    return s.limb_bits >= 64 ? v : (v & ((1ull << s.limb_bits) - 1));
}

template <int NW>
__device__ __forceinline__ void word_limb_words(const WordSrc &s, uint32_t vec, uint32_t j, uint32_t (&w)[NW]) {
    if (j >= s.nlimbs) {
#pragma unroll
        for (int i = 0; i < NW; i++) w[i] = 0;
        return;
    }
    const uint64_t bit = (uint64_t)j * s.limb_bits;
    const uint32_t wi = (uint32_t)(bit >> 5);
    const int sh = (int)(bit & 31);
    const uint32_t *base = s.w + (size_t)vec * s.words;
    uint32_t prev = wi < s.words ? PA_LDG(base + wi) : 0u;
#pragma unroll
    for (int i = 0; i < NW; i++) {
        const uint32_t nx = wi + i + 1 < s.words ? PA_LDG(base + wi + i + 1) : 0u;
        uint32_t v = __funnelshift_r(prev, nx, sh);
        const int left = (int)s.limb_bits - 32 * i;          // limb bits from this word up
        if (left <= 0) v = 0;
        else if (left < 32) v &= (1u << left) - 1u;
        w[i] = v;
        prev = nx;
    }
}

// Montgomery reduction of a limb value v < 2^56 (hi < 2^24 < p): v 2^-32 mod p in (0, 2p).
// The factor 2^-32 is common to every element of a packed vector and is compensated in
// the scale of the precomputed operand (pa_api.cu, setup_stage).
__device__ __forceinline__ uint32_t limb_redc(uint64_t v, uint32_t p, uint32_t pinv) {
    const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
    return hi - __umulhi(lo * pinv, p) + p;
}

// Multiword limb v = sum_i w_i 2^(32 i) -> v 2^-32 mod p in [0, 2p) (the same factor as
// limb_redc): groups of <= 3 products w_i (2^(32 i) mod p) summed in 64 bits (< 3 p 2^32),
// each group REDC-reduced and the groups added lazily.
template <int NW>
__device__ __forceinline__ uint32_t limb_words_redc(const uint32_t (&w)[NW], const PrimeK &k) {
    uint32_t s = 0;
#pragma unroll
    for (int g = 0; g < NW; g += 3) {
        uint64_t t = 0;
#pragma unroll
        for (int i = g; i < g + 3 && i < NW; i++) t = mad_wide(w[i], k.pw[i], t);
        s = red2p(s + red2p(redc64(t, k.p, k.pinv), k.p2), k.p2);
    }
    return s;
}

// The same from the limb's 24-bit chunks c_j (NC <= 10): sum_j c_j (2^(24 j) mod p) < 10 2^54
// fits one 64-bit accumulator far below p 2^32, so a single REDC gives v 2^-32 mod p in
// (0, 2p) -- one multiply-add per chunk and one reduction per (limb, prime), against a
// reduction per three 32-bit words.
template <int NW>
__host__ __device__ constexpr int chunks24() { return (32 * NW + 23) / 24; }
template <int NW>
__device__ __forceinline__ void limb_chunks24(const uint32_t (&w)[NW], uint32_t (&c)[chunks24<NW>()]) {
#pragma unroll
    for (int j = 0; j < chunks24<NW>(); j++) {
        const int i = (24 * j) >> 5, sh = (24 * j) & 31;
        const uint32_t lo = w[i], hi = (i + 1 < NW) ? w[i + 1] : 0u;
        c[j] = __funnelshift_r(lo, hi, sh) & 0xFFFFFFu;
    }
}
template <int NC>
__device__ __forceinline__ uint32_t limb_chunks_redc(const uint32_t (&c)[NC], const PrimeK &k) {
    static_assert(NC <= 10, "pw24 holds 10 chunk weights");
    uint64_t t = 0;
#pragma unroll
    for (int j = 0; j < NC; j++) t = mad_wide(c[j], k.pw24[j], t);
    return redc64(t, k.p, k.pinv);
}

// The same over NC 28-bit chunks (key limbs; B <= 28 NC): sum_j c_j (2^(28 j) mod p) <=
// 10 (2^28 - 1)(p - 1) < p 2^32, so one REDC still gives v 2^-32 mod p in (0, 2p); a 168-bit
// limb takes 6 multiply-adds per prime instead of the 8 of its 24-bit chunks.
template <int NW, int NC>
__device__ __forceinline__ void limb_chunks28(const uint32_t (&w)[NW], uint32_t (&c)[NC]) {
#pragma unroll
    for (int j = 0; j < NC; j++) {
        const int i = (28 * j) >> 5, sh = (28 * j) & 31;
        const uint32_t lo = i < NW ? w[i] : 0u, hi = (i + 1 < NW) ? w[i + 1] : 0u;
        c[j] = __funnelshift_r(lo, hi, sh) & 0xFFFFFFFu;
    }
}
template <int NC>
__device__ __forceinline__ uint32_t limb_chunks28_redc(const uint32_t (&c)[NC], const PrimeK &k) {
    static_assert(NC <= 10, "pw28 holds 10 chunk weights");
    uint64_t t = 0;
#pragma unroll
    for (int j = 0; j < NC; j++) t = mad_wide(c[j], k.pw28[j], t);
    return redc64(t, k.p, k.pinv);
}

// The residues of one multiword limb modulo all P primes, stored P x wxp apart from o.
template <int NW>
__device__ __forceinline__ void store_residues(uint32_t *o, uint32_t wxp, uint32_t P, uint32_t any,
                                               const uint32_t (&w)[NW], const PrimeSet &ks) {
    if (any) {
#pragma unroll
        for (uint32_t pi = 0; pi < kMaxPrimes; pi++) {
            if (pi >= P) break;
            PA_AT(o) = limb_words_redc<NW>(w, ks.k[pi]);
            o += wxp;
        }
    } else {
        for (uint32_t pi = 0; pi < P; pi++, o += wxp) PA_AT(o) = 0u;
    }
}

// S1 ("split the input bit sequence and map it to a prime field"): every
// limb of every vector is extracted once and reduced modulo all P primes.
// res layout: [vec][prime][wxp] with wxp = rows * N1 (zero beyond the vector's limbs).
// NW = 0: limbs of <= 56 bits (one 64-bit value, limb_redc); else NW 32-bit words.
template <class Src, int NW>
__global__ void __launch_bounds__(256) pack_residues(const Src src, const PrimeSet ks,
                                                     uint32_t P, uint32_t nvec, uint32_t wxp,
                                                     uint32_t *__restrict__ res) {
    PA_TMARK(0x7000 | NW, 0);
    const uint64_t total = (uint64_t)nvec * wxp;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        // 32-bit quotient whenever the index fits (a 64-bit division is a software call)
        const uint32_t iv = (t >> 32) ? (uint32_t)(t / wxp) : (uint32_t)t / wxp;
        const uint32_t j = (uint32_t)(t - (uint64_t)iv * wxp);
        uint32_t *o = res + (size_t)iv * P * wxp + j;
        if constexpr (NW == 0) {
            const uint64_t v = src(iv, j);
#pragma unroll
            for (uint32_t pi = 0; pi < kMaxPrimes; pi++)
                if (pi < P) PA_AT(o + (size_t)pi * wxp) = v ? limb_redc(v, ks.k[pi].p, ks.k[pi].pinv) : 0u;
        } else {
            uint32_t w[NW];
            src.template words<NW>(iv, j, w);
            uint32_t any = 0;
#pragma unroll
            for (int i = 0; i < NW; i++) any |= w[i];
            store_residues<NW>(o, wxp, P, any, w, ks);
        }
    }
}

// S1 for key blocks with multiword limbs (B > 56): CTA (tile of 256 limbs, block iv).
// The tile's key bytes are staged in shared memory with coalesced 32-bit loads; each
// thread assembles its limb's NW words (big-endian bytes, readings A3/A4) from there and
// reduces them modulo every prime.  res layout as pack_residues.
constexpr int kPackT = 256;
#ifndef PA_PACKL
#define PA_PACKL 2
#endif
constexpr int kPackL = PA_PACKL;                               // limbs per thread in pack_key_residues
#ifndef PA_PACK_V4
#define PA_PACK_V4 1                           // 128-bit key loads in pack_key_residues
#endif
#ifndef PA_PACK_CHUNK24
#define PA_PACK_CHUNK24 1                      // reduce limbs over 24-bit chunks (one REDC per prime)
#endif
// Residues of kPackL limbs (j0 + q kPackT) modulo all P primes, stored P x wxp apart.
// A zero limb among non-zero ones reduces to p (== 0 mod p, inside the [0, 2p) range the
// column pass takes); an all-zero set stores zeros.
// NC28 > 0: the limbs hold at most 28 NC28 bits; reduce them over 28-bit chunks.
template <int NW, int NC28 = 0>
__device__ __forceinline__ void store_residues_multi(uint32_t *o, uint32_t j0, uint32_t wxp, uint32_t P, uint32_t any,
                                                     const uint32_t (&w)[kPackL][NW], const PrimeSet &ks) {
    if (!any) {
        for (uint32_t pi = 0; pi < P; pi++, o += wxp)
#pragma unroll
            for (int q = 0; q < kPackL; q++)
                if (j0 + q * kPackT < wxp) PA_AT(o + q * kPackT) = 0u;
        return;
    }
    if constexpr (NC28 > 0) {
        uint32_t c[kPackL][NC28];
#pragma unroll
        for (int q = 0; q < kPackL; q++) limb_chunks28<NW, NC28>(w[q], c[q]);
#pragma unroll
        for (uint32_t pi = 0; pi < kMaxPrimes; pi++) {
            if (pi >= P) break;
#pragma unroll
            for (int q = 0; q < kPackL; q++) {
                const uint32_t r = limb_chunks28_redc<NC28>(c[q], ks.k[pi]);
                if (j0 + q * kPackT < wxp) PA_AT(o + q * kPackT) = r;
            }
            o += wxp;
        }
        return;
    }
#if PA_PACK_CHUNK24
    if constexpr (NW <= 7) {
        constexpr int NC = chunks24<NW>();
        uint32_t c[kPackL][NC];
#pragma unroll
        for (int q = 0; q < kPackL; q++) limb_chunks24<NW>(w[q], c[q]);
#pragma unroll
        for (uint32_t pi = 0; pi < kMaxPrimes; pi++) {
            if (pi >= P) break;
#pragma unroll
            for (int q = 0; q < kPackL; q++) {
                const uint32_t r = limb_chunks_redc<NC>(c[q], ks.k[pi]);
                if (j0 + q * kPackT < wxp) PA_AT(o + q * kPackT) = r;
            }
            o += wxp;
        }
    } else
#endif
    {
#pragma unroll
        for (uint32_t pi = 0; pi < kMaxPrimes; pi++) {
            if (pi >= P) break;
#pragma unroll
            for (int q = 0; q < kPackL; q++) {
                const uint32_t r = limb_words_redc<NW>(w[q], ks.k[pi]);
                if (j0 + q * kPackT < wxp) PA_AT(o + q * kPackT) = r;
            }
            o += wxp;
        }
    }
}

#ifndef PA_PACK_MINB
#define PA_PACK_MINB 8        // resident CTAs per SM the key pack's register budget is sized for (limbs of <= 6
#endif                        // words fit 32 registers without spills; wider limbs keep the default budget)
template <int NW, int NC28 = 0>
__global__ void __launch_bounds__(kPackT, ((NW <= 5 || (NW == 6 && NC28 > 0)) ? PA_PACK_MINB : 1)) pack_key_residues(const KeySrc s, const PrimeSet ks, uint32_t P,
                                                          uint32_t wxp, uint32_t *__restrict__ res) {
    PA_TMARK(0x6000 | NW, 0);
    // a tile is kPackL kPackT limbs, kPackL per thread (limbs t + q kPackT): the per-prime
    // constants, loop and addressing are shared by the limbs' reductions
    constexpr int TL = kPackL * kPackT;
    // staged words (LB <= 4 NW bytes per limb), plus up to 3 words back to a 16-byte boundary
    // and the round-up of the 16-byte loads
    constexpr int MAXW = ((TL * NW + 4 + 6 + 3) / 4) * 4;
    __shared__ __align__(16) uint32_t sw[MAXW];
    const uint32_t iv = blockIdx.y;
    const uint32_t jt0 = blockIdx.x * TL;
    const int64_t start = (int64_t)iv * s.blk_bytes;
    const int64_t end = start + s.blk_bytes;
    const int LB = (int)s.limb_bytes;
    const uint32_t jt1 = min(jt0 + TL, s.wx);               // limbs with data in this tile
    int64_t tlo = end - (int64_t)LB * jt1 - 4;               // lowest byte any word may touch
    if (tlo < start - 4) tlo = start - 4;
    int64_t gw0 = tlo >> 2;                                  // floor
    const int64_t thi = end - (int64_t)LB * jt0;
    int nw = (jt0 < jt1) ? (int)(((thi + 3) >> 2) - gw0 + 1) : 0;
    // interior tiles: plain aligned loads; tiles touching the key's ends: key_word
    const bool interior = s.aligned && gw0 >= 0 && (gw0 + nw + 1) * 4 < (int64_t)s.nbytes;
#if PA_PACK_V4
    // 128-bit loads (north_star (1)): the staged window starts at the 16-byte boundary at or
    // below its first word, so every load and every shared store is one aligned uint4
    const int dl = (int)((((uintptr_t)s.key + (uintptr_t)(gw0 * 4)) & 15) >> 2);
    const bool vec = interior && nw > 0 && gw0 - dl >= 0 &&
                     (gw0 - dl + 4 * (int64_t)((nw + dl + 3) >> 2) + 1) * 4 < (int64_t)s.nbytes;
    if (vec) {
        gw0 -= dl;
        nw += dl;
        const int nv = (nw + 3) >> 2;
        const uint4 *kv = reinterpret_cast<const uint4 *>(reinterpret_cast<const uint32_t *>(s.key) + gw0);
        constexpr int KV = (MAXW / 4 + kPackT - 1) / kPackT;
        uint4 q[KV];
#pragma unroll
        for (int u = 0; u < KV; u++) {
            const int k = threadIdx.x + u * kPackT;
            if (k < nv) q[u] = PA_LDG(kv + k);
        }
#pragma unroll
        for (int u = 0; u < KV; u++) {
            const int k = threadIdx.x + u * kPackT;
            if (k < nv) { PA_IDX_CK(4 * k + 3, MAXW); reinterpret_cast<uint4 *>(sw)[k] = q[u]; }
        }
    } else
#endif
    {
        const uint32_t *kw = reinterpret_cast<const uint32_t *>(s.key) + (interior ? gw0 : 0);
        // all of a thread's loads are issued before its stores (no load->store serialisation)
        constexpr int KU = (MAXW + kPackT - 1) / kPackT;
        uint32_t v[KU];
        if (interior) {
#pragma unroll
            for (int u = 0; u < KU; u++) {
                const int k = threadIdx.x + u * kPackT;
                v[u] = (k < nw) ? PA_LDG(kw + k) : 0u;
            }
        } else {
            for (int u = 0; u < KU; u++) {
                const int k = threadIdx.x + u * kPackT;
                v[u] = (k < nw) ? key_word(s, gw0 + k) : 0u;
            }
        }
#pragma unroll
        for (int u = 0; u < KU; u++) {
            const int k = threadIdx.x + u * kPackT;
            if (k < nw) { PA_IDX_CK(k, MAXW); sw[k] = v[u]; }
        }
    }
    __syncthreads();
    // limb j's NW words (big-endian bytes, readings A3/A4).  Byte offsets relative to the
    // staged base 4 gw0 (all < 4 MAXW).  Word i of the limb is the big-endian value of the
    // 4 bytes ending 4 i bytes before the limb's end, so all words share the byte shift
    // (hi & 3) and walk down the staged words by one.
    auto extract = [&](uint32_t j, uint32_t (&w)[NW]) -> uint32_t {
        uint32_t any = 0;
        if (j >= s.wx) {
#pragma unroll
            for (int i = 0; i < NW; i++) w[i] = 0u;
            return 0u;
        }
        const int base = (int)(4 * gw0 - start);
        const int hi = (int)(s.blk_bytes - (uint32_t)LB * j) - base;
        const int sh = (hi & 3) * 8;
        const int wtop = (hi >> 2) - 1;                       // staged word holding byte hi - 4
        PA_IDX_CK(wtop + 1, MAXW);
        uint32_t nxt = sw[wtop + 1];
#pragma unroll
        for (int i = 0; i < NW; i++) {
            PA_IDX_CK(max(wtop - i, 0), MAXW);
            const uint32_t cur = sw[max(wtop - i, 0)];
            w[i] = __byte_perm(__funnelshift_r(cur, nxt, sh), 0, 0x0123);
            nxt = cur;
        }
        // the block's top limb is shorter than B: clear the bytes before the block start
        int lo = hi - LB;
        if (lo < -base) {
            lo = -base;
#pragma unroll
            for (int i = 0; i < NW; i++) {
                const int below = lo - (hi - 4 * (i + 1));
                if (below >= 4) w[i] = 0;
                else if (below > 0) w[i] &= 0xFFFFFFFFu >> (8 * below);
            }
        }
        // a limb narrower than its NW words (B % 32): mask the top word
        if (LB < 4 * NW) {
            const int topbytes = LB - 4 * (NW - 1);
            w[NW - 1] &= 0xFFFFFFFFu >> (8 * (4 - topbytes));
        }
#pragma unroll
        for (int i = 0; i < NW; i++) any |= w[i];
        return any;
    };
    const uint32_t j0 = jt0 + threadIdx.x;
    if (j0 >= wxp) return;
    uint32_t w[kPackL][NW];
    uint32_t any = 0;
#pragma unroll
    for (int q = 0; q < kPackL; q++) any |= extract(j0 + q * kPackT, w[q]);
    store_residues_multi<NW, NC28>(res + (size_t)iv * P * wxp + j0, j0, wxp, P, any, w, ks);
}

// S1 for many word-sourced vectors (pa_ctx_rekey's a_i): CTA (tile of kPackL kPackT limbs,
// vector blockIdx.y), kPackL limbs per thread sharing the per-prime loop (pack_key_residues'
// scheme without the byte staging).  res layout as pack_residues.
template <class Src, int NW>
__global__ void __launch_bounds__(kPackT) pack_residues_tiled(const Src src, const PrimeSet ks, uint32_t P,
                                                              uint32_t wxp, uint32_t *__restrict__ res) {
    const uint32_t iv = blockIdx.y;
    const uint32_t j0 = blockIdx.x * (kPackL * kPackT) + threadIdx.x;
    if (j0 >= wxp) return;
    uint32_t w[kPackL][NW];
    uint32_t any = 0;
#pragma unroll
    for (int q = 0; q < kPackL; q++) {
        const uint32_t j = j0 + q * kPackT;
        if (j < wxp) {
            src.template words<NW>(iv, j, w[q]);
        } else {
#pragma unroll
            for (int i = 0; i < NW; i++) w[q][i] = 0u;
        }
#pragma unroll
        for (int i = 0; i < NW; i++) any |= w[q][i];
    }
    store_residues_multi<NW>(res + (size_t)iv * P * wxp + j0, j0, wxp, P, any, w, ks);
}

// ---------------------------------------------------------------- paper mode (NEXT-1)
// Algorithm 1 as written: gamma-bit windows t = key bits
// [t gamma, (t+1) gamma) (MSB-first); a window equal to 2^gamma - 1 is cast
// away and the next one consumed (reading A10).  Windows stay at
// multiples of gamma, so the reload rule is: block i = the i-th window with a zero bit.

// flags[t] = 1 if window t contains a zero bit.  CTA t scans window t in chunks of
// blockDim words and stops at the first chunk holding a zero bit: for keys of i.i.d.
// bits that is the first chunk, so the check reads ~1 KB per window; an all-ones window
// (the reload case) is scanned completely (correct, proportionally slower).
// The last CTA to finish (done counter, zeroed by the caller) then resolves the offsets:
// offs[i] = bit offset of block i (the i-th window with a zero bit); status 1 if fewer than k
// windows qualify (SPEC.md:74 InsufficientInput), else 0.
__global__ void __launch_bounds__(256) window_flags(const KeySrc s, uint32_t gamma, uint32_t T, uint32_t *flags,
                                                    uint32_t *done, uint32_t k, uint64_t *offs, uint32_t *status) {
    __shared__ uint32_t s_last;
    const uint32_t t = blockIdx.x;
    const uint64_t lo = (uint64_t)t * gamma, hi = lo + gamma;  // window bits [lo, hi)
    const uint64_t w0 = lo >> 5, w1 = (hi + 31) >> 5;
    uint32_t found = 0;
    for (uint64_t base = w0; base < w1 && !found; base += blockDim.x) {
        const uint64_t wi = base + threadIdx.x;
        uint32_t z = 0;
        if (wi < w1) {
            z = ~__byte_perm(key_word(s, (int64_t)wi), 0, 0x0123);     // bit 31 = position 32 wi
            const uint64_t p0 = 32 * wi;
            if (p0 < lo) z &= 0xFFFFFFFFu >> (lo - p0);                 // positions before the window
            if (p0 + 32 > hi) z &= 0xFFFFFFFFu << (p0 + 32 - hi);       // positions after it
        }
        found = __syncthreads_or(z != 0) ? 1u : 0u;
    }
    if (threadIdx.x == 0) {
        PA_AT(flags + t) = found;
        __threadfence();
        s_last = (atomicAdd(done, 1u) == T - 1);
    }
    __syncthreads();
    if (!s_last || threadIdx.x) return;
    __threadfence();
    uint32_t i = 0;
    for (uint32_t u = 0; u < T && i < k; u++)
        if (((volatile uint32_t *)flags)[u]) { PA_CK(offs + i, 8); offs[i++] = (uint64_t)u * gamma; }
    *status = (i < k) ? 1u : 0u;
    for (; i < k; i++) PA_AT(offs + i) = 0;                            // output undefined; reads stay in bounds
}

// S1 in paper mode: block iv = the gamma-bit window at key bit offs[iv]; limb j, word w =
// integer bits [B j + 32 w, + 32) = the 32 key bits starting at
// q = offs[iv] + gamma - (B j + 32 w) - 32 (MSB-first), bits before the window read 0.
template <int NW>
__global__ void __launch_bounds__(kPackT) pack_bits_residues(const KeySrc s, const uint64_t *__restrict__ offs,
                                                           uint32_t gamma, uint32_t B, uint32_t wx,
                                                           const PrimeSet ks, uint32_t P, uint32_t wxp,
                                                           uint32_t *__restrict__ res) {
    constexpr int TL = kPackL * kPackT;                       // limbs per tile, kPackL per thread
    constexpr int MAXW = TL * NW + 8;
    __shared__ uint32_t sw[MAXW];
    const uint32_t iv = blockIdx.y;
    const uint32_t jt0 = blockIdx.x * TL;
    const int64_t off = (int64_t)offs[iv];
    const uint32_t jt1 = min(jt0 + TL, wx);
    // key bits of the tile: [off + gamma - B jt1, off + gamma - B jt0), clipped at off
    int64_t blo = off + (int64_t)gamma - (int64_t)B * jt1 - 32;
    if (blo < off - 32) blo = off - 32;
    const int64_t bhi = off + (int64_t)gamma - (int64_t)B * jt0;
    const int64_t gw0 = (blo >> 3) >> 2;                      // first staged word (floor)
    const int nw = (jt0 < jt1) ? (int)((((bhi + 7) >> 3) + 3) / 4 - gw0 + 2) : 0;
    constexpr int KU = (MAXW + kPackT - 1) / kPackT;
    {
        uint32_t v[KU];
#pragma unroll
        for (int u = 0; u < KU; u++) {
            const int k = threadIdx.x + u * kPackT;
            v[u] = (k < nw && k < MAXW) ? key_word(s, gw0 + k) : 0u;
        }
#pragma unroll
        for (int u = 0; u < KU; u++) {
            const int k = threadIdx.x + u * kPackT;
            if (k < nw && k < MAXW) { PA_IDX_CK(k, MAXW); sw[k] = v[u]; }
        }
    }
    __syncthreads();
    // word i of limb j = window bits [B j + 32 i, +32) = the 32 key bits whose MSB is key bit
    // q_i = off + gamma - B j - 32 (i + 1): every word shares q_0's byte and bit shift and
    // sits one staged word lower than the previous one
    auto extract = [&](uint32_t j, uint32_t (&w)[NW]) -> uint32_t {
        uint32_t any = 0;
        if (j >= wx) {
#pragma unroll
            for (int i = 0; i < NW; i++) w[i] = 0u;
            return 0u;
        }
        const int64_t q0 = off + (int64_t)gamma - (int64_t)B * j - 32;
        const int64_t rb0 = (q0 >> 3) - 4 * gw0;               // staged byte of word 0
        const int sh = (int)(q0 & 7), bb = (int)(rb0 & 3);
        const int wi0 = (int)(rb0 >> 2);
        const int rem = (int)((int64_t)gamma - (int64_t)B * j); // window bits from the limb up
        uint32_t a1 = sw[wi0 + 1], a2 = sw[wi0 + 2];
#pragma unroll
        for (int i = 0; i < NW; i++) {
            const int wi = wi0 - i;
            const uint32_t a0 = (wi >= 0) ? sw[wi] : 0u;
            const uint32_t lo = __funnelshift_r(a0, a1, 8 * bb), hi = __funnelshift_r(a1, a2, 8 * bb);
            const uint64_t be = ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32) | __byte_perm(hi, 0, 0x0123);
            uint32_t v = (uint32_t)(be >> (32 - sh));
            const int valid = min(rem - 32 * i, (int)B - 32 * i);   // bits inside window and limb
            if (valid <= 0) v = 0u;
            else if (valid < 32) v &= (1u << valid) - 1u;
            w[i] = v;
            any |= v;
            a2 = a1;
            a1 = a0;
        }
        return any;
    };
    const uint32_t j0 = jt0 + threadIdx.x;
    if (j0 >= wxp) return;
    uint32_t w[kPackL][NW];
    uint32_t any = 0;
#pragma unroll
    for (int q = 0; q < kPackL; q++) any |= extract(j0 + q * kPackT, w[q]);
    store_residues_multi<NW>(res + (size_t)iv * P * wxp + j0, j0, wxp, P, any, w, ks);
}

// MH-only comparator: out[u] = bits [32 u, 32 u + 32) of x, the integer of key bits
// [0, n) read MSB-first, i.e. key bits [n - 32 u - 32, n - 32 u).
__global__ void key_to_words(const KeySrc s, uint64_t n, uint32_t W, uint32_t *__restrict__ out) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= W) return;
    const int64_t q = (int64_t)n - 32 * ((int64_t)u + 1);      // key bit of the word's MSB
    const int64_t bq = q >> 3;                                  // floor (q may be negative)
    const int sh = (int)(q & 7);
    const int64_t wi = bq >> 2;
    const int bb = (int)(bq & 3);
    const uint32_t a0 = key_word(s, wi), a1 = key_word(s, wi + 1), a2 = key_word(s, wi + 2);
    const uint32_t lo = __funnelshift_r(a0, a1, 8 * bb), hi = __funnelshift_r(a1, a2, 8 * bb);
    const uint64_t be = ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32) | __byte_perm(hi, 0, 0x0123);
    uint32_t v = (uint32_t)(be >> (32 - sh));
    if (q < 0) v &= 0xFFFFFFFFu >> (-q);                        // positions before bit 0 of the key
    PA_AT(out + u) = v;
}

struct KeyLimbs {
    KeySrc s;
    __device__ __forceinline__ uint64_t operator()(uint32_t iv, uint32_t j) const { return key_limb(s, iv, j); }
    template <int NW>
    __device__ __forceinline__ void words(uint32_t iv, uint32_t j, uint32_t (&w)[NW]) const { key_limb_words<NW>(s, iv, j, w); }
};
struct WordLimbs {
    WordSrc s;
    __device__ __forceinline__ uint64_t operator()(uint32_t iv, uint32_t j) const { return word_limb(s, iv, j); }
    template <int NW>
    __device__ __forceinline__ void words(uint32_t iv, uint32_t j, uint32_t (&w)[NW]) const { word_limb_words<NW>(s, iv, j, w); }
};

// ---------------------------------------------------------------- column pass
enum ColMode { COL_FWD = 0, COL_INV = 2 };

struct ColArgs {
    NttArgs nt;
    const uint32_t *src;     // FWD: residues [nvec][P][rows*N1];  INV: [P][L]
    uint32_t rows;           // FWD: rows holding non-zero limbs (<= N2)
    const uint2 *tw4;        // FWD: omega_L^(j1 k2) table [P][L], Shoup pairs (w, floor(w 2^32/p))
    uint32_t *dst;           // FWD: [nvec][P][L];  INV: [P][L]
    uint32_t nvec;           // vectors (blocks) per prime
    uint32_t units;          // (N1/32) * P * nvec
    uint32_t lanes;          // co-resident CTAs per SM slot (launcher: grid = lanes * slots), else 1
};

// One CTA = 32 adjacent columns (one lane each) x S/E threads per column.  The row
// length N1 = 2^N1_LOG is a template parameter so every element address is a per-unit
// base plus a compile-time offset (no per-element 64-bit index arithmetic).
// ZH (template, chosen by the launcher): the forward input's rows all lie in the first half
// of each column (see below); each instantiation carries only its own load and first stage
template <int S_LOG, int E_LOG, int N1_LOG, int MODE, bool ZH = false>
#ifndef PA_COL8_MINB
#define PA_COL8_MINB 4
#endif
#ifndef PA_COL8E4_MINB
#define PA_COL8E4_MINB 2
#endif
__global__ void __launch_bounds__(32 * (1 << (S_LOG - E_LOG)),
                                  S_LOG == 8 ? (E_LOG == 5 ? PA_COL8_MINB : PA_COL8E4_MINB) : (S_LOG < 8 ? 3 : 1))
col_pass(const ColArgs A) {
    PA_TMARK(0x1000 | (S_LOG << 8) | (E_LOG << 4) | MODE, 0);
    using SP = SubPlan<S_LOG, E_LOG>;
    constexpr int E = SP::E;
    constexpr uint32_t N1 = 1u << N1_LOG;
    constexpr uint32_t L = (1u << S_LOG) * N1;
    extern __shared__ uint32_t sm[];
    const int c = threadIdx.x & 31;
    const int v = threadIdx.x >> 5;
    const NttArgs &a = A.nt;
    const uint32_t P = a.nprimes;
    const uint32_t nvec = A.nvec;
    const uint32_t rows = A.rows;
    const uint32_t units = A.units;
    // CTAs b, b + slots, b + 2 slots, ... of a full-occupancy grid are resident on one SM (the
    // first wave fills SM (b mod slots) with them): they share one contiguous unit range and
    // take its units round robin, so the co-resident CTAs work on the same (column group,
    // prime) for successive vectors and read the same four-step twiddles (one L1-resident
    // tile instead of one per CTA).  Any placement gives the same results.
    const uint32_t lanes = A.lanes;
    const uint32_t slots = gridDim.x / lanes;
    const uint32_t slot = blockIdx.x % slots, lane = blockIdx.x / slots;
    const uint32_t u0 = (uint32_t)(((uint64_t)slot * units) / slots) + lane;
    const uint32_t u1 = (uint32_t)(((uint64_t)(slot + 1) * units) / slots);
    auto sidx = [c](int pos) { return pos * 32 + c; };

    uint32_t tw[E / 2], twp[E / 2];
    int cur_pi = -1;
    Ctx32 cx{};
    const uint32_t *rtw_p = nullptr;

    // unit u = ((cg P + pi) nvec + iv): stepped incrementally, no division in the loop
    uint32_t iv = 0, pi = 0, cg = 0;
    if (u0 < u1) {
        const uint32_t pair0 = u0 / nvec;
        iv = u0 - pair0 * nvec;
        pi = pair0 % P;
        cg = pair0 / P;
    }
    for (uint32_t u = u0; u < u1; u += lanes) {
        if (u != u0) {
            iv += lanes;
            while (iv >= nvec) {
                iv -= nvec;
                if (++pi == P) { pi = 0; cg++; }
            }
        }
        const uint32_t j1 = cg * 32 + c;
        if ((int)pi != cur_pi) {
            cur_pi = (int)pi;
            const PrimeK pk = a.pk[pi];
            cx.p = pk.p; cx.p2 = pk.p2; cx.pinv = pk.pinv;
            load_regtw<E>(a, pi, tw, twp);
            rtw_p = a.rtw + (size_t)pi * a.rtw_stride;
        }
        uint32_t x[E];
        // round 0's first stage pairs rows q and q + S/2: with all non-zero rows in the
        // first half (the zero-padded upper half of every packed vector) it is (a, a w), and the
        // upper half (m >= R/2 in every group) is neither loaded nor read.  Its loads are left
        // out of this branch altogether: a predicated-off load still holds its destination
        // register on the scoreboard, and a later reuse of that register waited on it.
        constexpr bool zh = ZH;
        {
            constexpr int R = 1 << SP::rlog(0);
#if defined(PA_COL_DBG) && (PA_COL_DBG & 4)
            const uint32_t *src = ((MODE == COL_INV) ? A.src + (size_t)pi * L
                                                     : A.src + ((size_t)0 * P + pi) * ((size_t)rows * N1)) +
#else
            const uint32_t *src = ((MODE == COL_INV) ? A.src + (size_t)pi * L
                                                     : A.src + ((size_t)iv * P + pi) * ((size_t)rows * N1)) +
#endif
                                  ((size_t)v << N1_LOG) + j1;
            if constexpr (zh) {
#pragma unroll
                for (int h = 0; h < E / R; h++) {
#pragma unroll
                    for (int m = 0; m < R; m++) {
                        const int rel = SP::TPV * h + (SP::S / R) * m;      // in_pos - v, < S/2 iff m < R/2
                        uint32_t val = 0;
                        if (m < R / 2 && (uint32_t)(v + rel) < rows) val = PA_AT(src + ((size_t)rel << N1_LOG));
                        x[h * R + m] = val;
                    }
                }
            } else {
#pragma unroll
                for (int h = 0; h < E / R; h++) {
#pragma unroll
                    for (int m = 0; m < R; m++) {
                        const int rel = SP::TPV * h + (SP::S / R) * m;      // in_pos - v
                        uint32_t val = 0;
                        if (MODE == COL_INV || (uint32_t)(v + rel) < rows) val = PA_AT(src + ((size_t)rel << N1_LOG));
                        x[h * R + m] = val;
                    }
                }
            }
        }
        __syncthreads();    // previous unit's last-round smem reads are done
        if constexpr (zh)
            round0_finish<S_LOG, E_LOG, true>(x, sm, sidx, v, tw, twp, rtw_p, a, cx);
        else
            round0_finish<S_LOG, E_LOG>(x, sm, sidx, v, tw, twp, rtw_p, a, cx);
        // forward: the outputs meet a Montgomery multiply by the four-step twiddle next, so
        // the last stage skips its reductions
        rounds_rest<S_LOG, E_LOG, 1, MODE == COL_FWD>(x, sm, sidx, v, tw, twp, rtw_p, a, cx);
        {
            constexpr int R = 1 << SP::rlog(SP::Q - 1);
            constexpr int G = 1 << SP::glog(SP::Q - 1);
            const size_t vb = ((size_t)v << N1_LOG) + j1;
            uint32_t *dst = ((MODE == COL_INV) ? A.dst + (size_t)pi * L : A.dst + ((size_t)iv * P + pi) * L) + vb;
            const uint2 *tw4 = A.tw4 + (size_t)pi * L + vb;
#pragma unroll
            for (int h = 0; h < E / R; h++) {
#pragma unroll
                for (int mm = 0; mm < R; mm++) {
                    const int rel = SP::TPV * h + G * bitrev<R>(mm);        // out_pos - v
                    const size_t o = (size_t)rel << N1_LOG;
                    uint32_t val = x[h * R + mm];
                    if constexpr (MODE != COL_INV) {
#if defined(PA_COL_DBG) && (PA_COL_DBG & 1)
                        const uint2 w = make_uint2(j1 + 3u, (j1 + 3u) * 5u);   // timing-only ablation
#else
                        const uint2 w = PA_LDG(tw4 + o);
#endif
                        val = mul_shoup(val, w.x, w.y, cx.p);
                    }
                    else val = red1p(val, cx.p);
                    PA_AT(dst + o) = val;
                }
            }
        }
    }
}

// ---------------------------------------------------------------- row pass
enum RowMode { ROW_MAC = 0, ROW_STORE = 1, ROW_INV = 2 };

struct RowArgs {
    NttArgs nt;
    const uint32_t *src;      // MAC/STORE: [nvec][P][L];  INV: [P][L]
    uint32_t *dst;            // MAC: [P][L] accumulators;  STORE: [nvec][P][L];  INV: [P][L]
    const uint32_t *ahat;     // MAC: [nvec][P][L] (Montgomery form, times 1/L)
    const uint32_t *scale;    // STORE: [P] Montgomery constant multiplied into outputs
    const uint32_t *tw4;      // INV: omega_L^(-j1 k2) table [P][L] (Montgomery, canonical)
    uint32_t nsrc;            // INV: the input is the sum of nsrc slots src + s * src_stride (each < 4p)
    uint32_t src_stride;
    uint32_t nvec;
    uint32_t units;           // (N2 / V) * P
};

template <int S_LOG, int E_LOG, int V, int MODE>
__global__ void __launch_bounds__(V * (1 << (S_LOG - E_LOG)))
row_pass(const RowArgs A) {
    PA_TMARK(0x2000 | (S_LOG << 8) | (E_LOG << 4) | MODE, 0);
    using SP = SubPlan<S_LOG, E_LOG>;
    constexpr int S = SP::S, E = SP::E;
    constexpr int RS = S + S / 32;                       // padded row stride in smem
    extern __shared__ uint32_t sm[];
    const int w = threadIdx.x / SP::TPV;
    const int v = threadIdx.x % SP::TPV;
    const NttArgs &a = A.nt;
    const uint32_t L = 1u << a.log2L;
    const uint32_t P = a.nprimes;
    auto sidx = [w](int pos) { return w * RS + pos + (pos >> 5); };

    // ROW_STORE: the vectors are independent, so (unit, vector) pairs are spread over the
    // grid (iv = uu / units); MAC accumulates over all vectors inside a unit
    const uint32_t nflat = (MODE == ROW_STORE) ? A.units * A.nvec : A.units;
    for (uint32_t uu = blockIdx.x; uu < nflat; uu += gridDim.x) {
        const uint32_t u = (MODE == ROW_STORE) ? uu % A.units : uu;
        const uint32_t pi = u % P;
        const uint32_t rg = u / P;
        const uint32_t k2 = rg * V + w;                  // row index
        const PrimeK pk = a.pk[pi];
        const Ctx32 cx{pk.p, pk.p2, pk.pinv};
        uint32_t tw[E / 2], twp[E / 2];
        load_regtw<E>(a, pi, tw, twp);
        const uint32_t *rtw_p = a.rtw + (size_t)pi * a.rtw_stride;
        uint32_t acc[E];
#pragma unroll
        for (int e = 0; e < E; e++) acc[e] = 0;
        const uint32_t iv0 = (MODE == ROW_STORE) ? uu / A.units : 0u;
        const uint32_t nv = (MODE == ROW_INV) ? 1u : ((MODE == ROW_STORE) ? iv0 + 1 : A.nvec);
        for (uint32_t iv = iv0; iv < nv; iv++) {
            const size_t vbase = (MODE == ROW_INV) ? (size_t)pi * L : ((size_t)iv * P + pi) * L;
            const uint32_t *src = A.src + vbase + (size_t)k2 * S;
            uint32_t x[E];
            {
                constexpr int R = 1 << SP::rlog(0);
#pragma unroll
                for (int h = 0; h < E / R; h++)
#pragma unroll
                    for (int m = 0; m < R; m++) {
                        const uint32_t t = PA_AT(src + in_pos<S_LOG, E_LOG>(v, h, m));
                        // ROW_INV input: accumulators merged with red.add, in [0, 4p)
                        x[h * R + m] = (MODE == ROW_INV) ? red2p(t, cx.p2) : t;
                    }
            }
            if constexpr (MODE == ROW_INV) {
                // the row MAC's further accumulator slots (each < 4p), one batch of loads each
                for (uint32_t q = 1; q < A.nsrc; q++) {
                    constexpr int R = 1 << SP::rlog(0);
                    const uint32_t *sq = src + (size_t)q * A.src_stride;
#pragma unroll
                    for (int h = 0; h < E / R; h++)
#pragma unroll
                        for (int m = 0; m < R; m++)
                            x[h * R + m] = red2p(x[h * R + m] + red2p(PA_AT(sq + in_pos<S_LOG, E_LOG>(v, h, m)), cx.p2), cx.p2);
                }
            }
            __syncthreads();
            round0_finish<S_LOG, E_LOG>(x, sm, sidx, v, tw, twp, rtw_p, a, cx);
            rounds_rest<S_LOG, E_LOG, 1, true>(x, sm, sidx, v, tw, twp, rtw_p, a, cx);   // mul_mont next
            constexpr int R = 1 << SP::rlog(SP::Q - 1);
            if constexpr (MODE == ROW_MAC) {
                const uint32_t *ah = A.ahat + vbase + (size_t)k2 * S;
#pragma unroll
                for (int h = 0; h < E / R; h++)
#pragma unroll
                    for (int mm = 0; mm < R; mm++) {
                        const int k1 = out_pos<S_LOG, E_LOG>(v, h, mm);
                        acc[h * R + mm] = red2p(acc[h * R + mm] + mul_mont(x[h * R + mm], PA_LDG(ah + k1), cx.p, cx.pinv), cx.p2);
                    }
            } else if constexpr (MODE == ROW_STORE) {
                const uint32_t sc = A.scale[pi];
                uint32_t *dst = A.dst + vbase + (size_t)k2 * S;
#pragma unroll
                for (int h = 0; h < E / R; h++)
#pragma unroll
                    for (int mm = 0; mm < R; mm++) {
                        const int k1 = out_pos<S_LOG, E_LOG>(v, h, mm);
                        PA_AT(dst + k1) = red1p(mul_mont(x[h * R + mm], sc, cx.p, cx.pinv), cx.p);
                    }
            } else {
                uint32_t *dst = A.dst + vbase + (size_t)k2 * S;
#pragma unroll
                for (int h = 0; h < E / R; h++)
#pragma unroll
                    for (int mm = 0; mm < R; mm++) {
                        const uint32_t j1 = (uint32_t)out_pos<S_LOG, E_LOG>(v, h, mm);
                        const uint32_t w = PA_LDG(A.tw4 + (size_t)pi * L + (size_t)k2 * S + j1);
                        PA_AT(dst + j1) = mul_mont(x[h * R + mm], w, cx.p, cx.pinv);
                    }
            }
        }
        if constexpr (MODE == ROW_MAC) {
            constexpr int R = 1 << SP::rlog(SP::Q - 1);
            uint32_t *dst = A.dst + (size_t)pi * L + (size_t)k2 * S;
#pragma unroll
            for (int h = 0; h < E / R; h++)
#pragma unroll
                for (int mm = 0; mm < R; mm++) PA_AT(dst + out_pos<S_LOG, E_LOG>(v, h, mm)) = acc[h * R + mm];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- single-vector row MAC + inverse row
// S7 (Eq. 4), the MH product b y: the single vector's forward row DFT,
// the transform-domain product with B^ (b's precomputed transform), the inverse row DFT
// and the inverse four-step twiddle, in one pass over each row.  With one vector there is
// nothing to accumulate across CTAs, so the row stays on chip between the two DFTs (one
// shared-memory reorder from the forward DFT's output positions to the inverse DFT's input
// positions) instead of a store, a kernel boundary and a reload.  Output as ROW_INV.
struct MacInvArgs {
    NttArgs fw;               // forward row tables
    NttArgs iv;               // inverse row tables
    const uint32_t *src;      // [P][L] forward column-pass output
    const uint32_t *bhat;     // [P][L] precomputed transform (Montgomery, x 1/L)
    const uint32_t *tw4;      // omega_L^(-j1 k2) [P][L] (Montgomery, canonical)
    uint32_t *dst;            // [P][L]
    uint32_t units;           // (N2 / V) * P
};

template <int S_LOG, int E_LOG, int V>
__global__ void __launch_bounds__(V * (1 << (S_LOG - E_LOG)))
row_macinv(const MacInvArgs A) {
    PA_TMARK(0x2800 | (S_LOG << 4) | E_LOG, 0);
    using SP = SubPlan<S_LOG, E_LOG>;
    constexpr int S = SP::S, E = SP::E;
    constexpr int RS = S + S / 32;                       // padded row stride in smem
    extern __shared__ uint32_t sm[];
    const int w = threadIdx.x / SP::TPV;
    const int v = threadIdx.x % SP::TPV;
    const uint32_t L = 1u << A.fw.log2L;
    const uint32_t P = A.fw.nprimes;
    auto sidx = [w](int pos) { return w * RS + pos + (pos >> 5); };
    constexpr int R0 = 1 << SP::rlog(0);
    constexpr int RL = 1 << SP::rlog(SP::Q - 1);
    for (uint32_t u = blockIdx.x; u < A.units; u += gridDim.x) {
        const uint32_t pi = u % P;
        const uint32_t k2 = (u / P) * V + w;             // row index
        const PrimeK pk = A.fw.pk[pi];
        const Ctx32 cx{pk.p, pk.p2, pk.pinv};
        const size_t rb = (size_t)pi * L + (size_t)k2 * S;
        uint32_t tw[E / 2], twp[E / 2];
        uint32_t x[E];
#pragma unroll
        for (int h = 0; h < E / R0; h++)
#pragma unroll
            for (int m = 0; m < R0; m++) x[h * R0 + m] = PA_AT(A.src + rb + in_pos<S_LOG, E_LOG>(v, h, m));
        load_regtw<E>(A.fw, pi, tw, twp);
        __syncthreads();                                 // the previous row's shared reads are done
        round0_finish<S_LOG, E_LOG>(x, sm, sidx, v, tw, twp, A.fw.rtw + (size_t)pi * A.fw.rtw_stride, A.fw, cx);
        rounds_rest<S_LOG, E_LOG, 1, true>(x, sm, sidx, v, tw, twp, A.fw.rtw + (size_t)pi * A.fw.rtw_stride, A.fw, cx);
        __syncthreads();                                 // last-round shared reads before the reorder
#pragma unroll
        for (int h = 0; h < E / RL; h++)
#pragma unroll
            for (int mm = 0; mm < RL; mm++) {
                const int k1 = out_pos<S_LOG, E_LOG>(v, h, mm);
                PA_SMEM_PTR_CK(sm + sidx(k1), 4);
                sm[sidx(k1)] = mul_mont(x[h * RL + mm], PA_LDG(A.bhat + rb + k1), cx.p, cx.pinv);   // (0, 2p)
            }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < E / R0; h++)
#pragma unroll
            for (int m = 0; m < R0; m++) {
                PA_SMEM_PTR_CK(sm + sidx(in_pos<S_LOG, E_LOG>(v, h, m)), 4);
                x[h * R0 + m] = sm[sidx(in_pos<S_LOG, E_LOG>(v, h, m))];
            }
        load_regtw<E>(A.iv, pi, tw, twp);
        __syncthreads();                                 // reorder reads before round 0's writes
        round0_finish<S_LOG, E_LOG>(x, sm, sidx, v, tw, twp, A.iv.rtw + (size_t)pi * A.iv.rtw_stride, A.iv, cx);
        rounds_rest<S_LOG, E_LOG, 1, true>(x, sm, sidx, v, tw, twp, A.iv.rtw + (size_t)pi * A.iv.rtw_stride, A.iv, cx);
#pragma unroll
        for (int h = 0; h < E / RL; h++)
#pragma unroll
            for (int mm = 0; mm < RL; mm++) {
                const uint32_t j1 = (uint32_t)out_pos<S_LOG, E_LOG>(v, h, mm);
                PA_AT(A.dst + rb + j1) = mul_mont(x[h * RL + mm], PA_LDG(A.tw4 + rb + j1), cx.p, cx.pinv);
            }
    }
}

// ---------------------------------------------------------------- row pass + MAC
// S2+S3 (Eq. 2): second NTT pass of every block and the transform-
// domain multiply-accumulate acc += X_i (.) A^_i, for all blocks i.
// Iteration space (unit = V rows of one prime, block iv) flattened with iv fastest and
// split evenly over persistent CTAs.  A CTA streams its iterations' X rows (2-stage
// ring) and A^ rows (single buffer, loaded while the X rows are transformed) into
// shared memory with bulk asynchronous copies (cp.async.bulk, mbarrier completion),
// so HBM reads overlap the butterflies.  The radix-round exchange happens in place in
// the X stage, XOR-swizzled (bank-conflict free for every round pattern, checked by
// scripts/dev/swizzle_sim.py), so a CTA needs only 3 V*S words of shared memory.
// A unit's accumulators are added into dst with red.add (dst zeroed by the caller);
// a unit split between CTAs is thereby merged.  Partials are canonical (< p) and the
// launcher keeps gridDim.x <= 3 nunits (no unit spans more than four CTAs): values < 4p.
struct MacArgs {
    NttArgs nt;
    const uint32_t *src;      // [nvec][P][L] forward column-pass output
    const uint32_t *ahat;     // [nvec][P][L] precomputed transforms (Montgomery, x 1/L)
    uint32_t *dst;            // [P][L] accumulators (zeroed), results in [0, 4p)
    uint32_t nvec;
    uint32_t nunits;          // (N2 / V) * P
    uint32_t mode;            // 0: iterations split evenly, red.add into zeroed dst (< 4p)
                              // 1: whole units per CTA, dst = sum (canonical)
                              // 2: whole units per CTA, dst = (dst + sum) mod p (dst canonical)
                              // 3: iterations split evenly, 64-bit red.add of the canonical
                              //    partials into dst64 (a peer GPU's receive buffer, the
                              //    multi-GPU P2P exchange), then a system-scope fence
    unsigned long long *dst64;
    uint32_t nslot;           // mode 0: CTA b adds into slot b mod nslot (dst + slot * slot_stride),
    uint32_t slot_stride;     // so that no slot receives more than four partials of a unit
};

// rows per CTA: V*S = kMacWords words per operand and stage, and V <= S/2 <= N2 (planner)
#ifndef PA_MAC_WORDS
#define PA_MAC_WORDS 2048
#endif
constexpr int kMacWords = PA_MAC_WORDS;
__host__ __device__ constexpr int mac_v(int slog) {
    return ((1 << slog) >= kMacWords ? 1 : (kMacWords >> slog)) < (1 << (slog - 1))
               ? ((1 << slog) >= kMacWords ? 1 : (kMacWords >> slog))
               : (1 << (slog - 1));
}
// exchange layout: a separate padded buffer (fewer instructions than the in-place XOR
// swizzle, measured 118 vs 135 us for C4) whenever it fits; in place for 2^14-point rows
__host__ __device__ constexpr int mac_pad(int slog) { return slog <= 13 ? 1 : 0; }
#ifndef PA_MAC_NSX
#define PA_MAC_NSX 2
#endif
template <int S_LOG, int PAD = mac_pad(S_LOG), int NSX = PA_MAC_NSX, int AIN = 0>
constexpr size_t mac_smem_bytes() {
    return (size_t)(NSX + (AIN ? 0 : 1)) * mac_v(S_LOG) * (1 << S_LOG) * 4 + 4 * 8 +
           (PAD ? (size_t)mac_v(S_LOG) * ((1 << S_LOG) + (1 << S_LOG) / 32) * 4 : 0);
}
__device__ __forceinline__ int swz32(int P) { return P ^ ((P >> 5) & 31); }

__host__ __device__ constexpr int mac_threads(int slog, int elog) { return mac_v(slog) * (1 << (slog - elog)); }
// CTAs per SM as shared memory admits them (227 KB usable, 1 KB reserved per CTA); the
// register budget per thread follows from it (65536 / (minb * threads), e.g. 6 CTAs of 64
// threads -> 167 registers: measured 124 -> 118 us for the C4 row_mac against a 128 cap)
__host__ __device__ constexpr int mac_minb(size_t smem_bytes) {
    return (int)(232448 / (smem_bytes + 1024)) < 1 ? 1 : ((int)(232448 / (smem_bytes + 1024)) > 8 ? 8 : (int)(232448 / (smem_bytes + 1024)));
}
// MODE: A.mode as a template parameter, so each instantiation carries only its own flush and
// iteration split (the P2P mode's branch in the shared kernel cost the default C4 row MAC 6
// registers and 4.5 us)
#ifndef PA_MAC_AIN
#define PA_MAC_AIN 0          // A^ rows land in the X stage (needs the padded exchange buffer): two stages, not three
#endif
#ifndef PA_MAC_MINB_CAP
#define PA_MAC_MINB_CAP 8     // most CTAs per SM the register budget is sized for
#endif
__host__ __device__ constexpr int mac_ain(int slog) { return PA_MAC_AIN && mac_pad(slog); }
__host__ __device__ constexpr int mac_minb_cap(int b) { return b > PA_MAC_MINB_CAP ? PA_MAC_MINB_CAP : b; }
template <int S_LOG, int E_LOG, int DBG = 0, int PAD = mac_pad(S_LOG), int NSX = PA_MAC_NSX, int AIN = mac_ain(S_LOG), int MODE = 0>
__global__ void __launch_bounds__(mac_threads(S_LOG, E_LOG), mac_minb_cap(mac_minb(mac_smem_bytes<S_LOG, PAD, NSX, AIN>())))
row_mac(const MacArgs A) {
    PA_TMARK(0x3000 | (S_LOG << 8) | (E_LOG << 4), 0);
    using SP = SubPlan<S_LOG, E_LOG>;
    constexpr int S = SP::S, E = SP::E;
    constexpr int V = mac_v(S_LOG);
    constexpr uint32_t SW = V * S;                       // words per operand per stage
    extern __shared__ __align__(128) uint32_t smem[];
    uint32_t *xs = smem;                                 // [2][SW] X ring (exchange in place)
    // AIN: A^ rows are copied into the X stage once its natural-order reads are done
    // (the exchange is in the separate padded buffer), saving a third stage of smem
    static_assert(!AIN || PAD, "AIN needs the separate exchange buffer");
    constexpr int NST = NSX + (AIN ? 0 : 1);
    uint32_t *as = smem + NSX * SW;                      // [SW]   A^ (unless AIN)
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + NST * SW);   // fullX[NSX], fullA
    uint32_t *exb = smem + NST * SW + 8;                 // PAD: [V][S + S/32] exchange
    const int w = threadIdx.x / SP::TPV;
    const int v = threadIdx.x % SP::TPV;
    const NttArgs &a = A.nt;
    const uint32_t L = 1u << a.log2L;
    const uint32_t P = a.nprimes;
    const uint32_t nvec = A.nvec;
    const uint64_t total = (uint64_t)A.nunits * nvec;
    constexpr bool whole = MODE == 1 || MODE == 2;
    const uint64_t it0 = whole ? (uint64_t)(blockIdx.x * (uint64_t)A.nunits / gridDim.x) * nvec
                               : blockIdx.x * total / gridDim.x;
    const uint64_t it1 = whole ? (uint64_t)((blockIdx.x + 1) * (uint64_t)A.nunits / gridDim.x) * nvec
                               : (blockIdx.x + 1) * total / gridDim.x;
    auto sidx = [w](int pos) {
        if constexpr (PAD) return w * (S + S / 32) + pos + (pos >> 5);
        else return swz32(w * S + pos);
    };
    // iteration it = (unit, iv), unit = (rg, pi): cursors stepped incrementally (the loop
    // does no integer division; one set of divisions per cursor at the start)
    struct Cur {
        uint32_t iv, pi, rg;
    };
    auto cur_at = [&](uint64_t it) -> Cur {
        const uint32_t unit = (uint32_t)(it / nvec);
        return Cur{(uint32_t)(it - (uint64_t)unit * nvec), unit % P, unit / P};
    };
    auto step = [&](Cur &c) {
        if (++c.iv == nvec) {
            c.iv = 0;
            if (++c.pi == P) { c.pi = 0; c.rg++; }
        }
    };
    auto offset_of = [&](const Cur &c) -> size_t { return ((size_t)c.iv * P + c.pi) * L + (size_t)c.rg * SW; };
    auto issue_x = [&](const Cur &c, int s) {
        mbar_arrive_expect_tx(&bars[s], SW * 4);
        bulk_g2s(xs + s * SW, A.src + offset_of(c), SW * 4, &bars[s]);
    };
    auto issue_a = [&](const Cur &c, uint32_t *dst) {
        mbar_arrive_expect_tx(&bars[NSX], SW * 4);
        bulk_g2s(dst, A.ahat + offset_of(c), SW * 4, &bars[NSX]);
    };
    Cur cc = cur_at(it0);                                // iteration it
    Cur cn = cc;                                         // next X to issue (it + NSX)
    Cur ca = cc;                                         // next A^ to issue (it + 1)
    if (threadIdx.x == 0) {
        for (int s = 0; s <= NSX; s++) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    for (int s = 0; s < NSX; s++) {
        if (threadIdx.x == 0 && it0 + s < it1) issue_x(cn, s);
        step(cn);
    }
    if (threadIdx.x == 0 && !AIN && it0 < it1) issue_a(ca, as);
    step(ca);

    uint32_t tw[E / 2], twp[E / 2];
    uint32_t acc[E];
    Ctx32 cx{};
    uint32_t *const dslot = A.dst + (size_t)(blockIdx.x % A.nslot) * A.slot_stride;   // mode 0 slot
    auto flush_one = [&](uint32_t *d, uint32_t v) {
        v = red1p(v, cx.p);
        PA_CK(d, 4);
        if constexpr (MODE == 3) {
            const size_t e = (size_t)(d - dslot);                  // element of the [P][L] accumulator
            PA_CK(A.dst64 + e, 8);
            atomicAdd(A.dst64 + e, (unsigned long long)v);
        } else if constexpr (MODE == 0) atomicAdd(d, v);
        else if constexpr (MODE == 1) *d = v;
        else *d = red1p(*d + v, cx.p);
    };
    const uint32_t *rtw_p = nullptr;
    bool have_unit = false;
    uint32_t fpi = 0, frg = 0;                           // unit being accumulated
    uint32_t cur_pi = 0;
    for (uint64_t it = it0; it < it1; it++, step(cc)) {
        if (!have_unit || cc.iv == 0) {
            if (have_unit) {
                constexpr int R = 1 << SP::rlog(SP::Q - 1);
                uint32_t *dst = dslot + (size_t)fpi * L + (size_t)(frg * V + w) * S;
#pragma unroll
                for (int h = 0; h < E / R; h++)
#pragma unroll
                    for (int mm = 0; mm < R; mm++) flush_one(dst + out_pos<S_LOG, E_LOG>(v, h, mm), acc[h * R + mm]);
            }
            fpi = cc.pi;
            frg = cc.rg;
            const uint32_t pi = cc.pi;
            if (rtw_p == nullptr || pi != cur_pi) {
                cur_pi = pi;
                const PrimeK pk = a.pk[pi];
                cx = Ctx32{pk.p, pk.p2, pk.pinv};
                load_regtw<E>(a, pi, tw, twp);
                rtw_p = a.rtw + (size_t)pi * a.rtw_stride;
            }
            have_unit = true;
#pragma unroll
            for (int e = 0; e < E; e++) acc[e] = 0;
        }
        const uint32_t k = (DBG == 2 || DBG == 3) ? 0u : (uint32_t)(it - it0);
        const int s = (int)(k % NSX);
        mbar_wait(&bars[s], (k / NSX) & 1);
        uint32_t *xst = xs + s * SW;
        uint32_t x[E];
        {
            constexpr int R = 1 << SP::rlog(0);
#pragma unroll
            for (int h = 0; h < E / R; h++)
#pragma unroll
                for (int m = 0; m < R; m++) { PA_SMEM_PTR_CK((xst + w * S + in_pos<S_LOG, E_LOG>(v, h, m)), 4); x[h * R + m] = xst[w * S + in_pos<S_LOG, E_LOG>(v, h, m)]; }
        }
        if constexpr (AIN) {
            __syncthreads();                             // X stage s read: A^(it) may land there
            if (threadIdx.x == 0) issue_a(cc, xst);
        }
        if constexpr (DBG != 1) {
            uint32_t *exch = PAD ? exb : xst;
            if constexpr (SP::Q > 1 && !PAD) __syncthreads();   // natural-order reads before in-place writes
            round0_finish<S_LOG, E_LOG>(x, exch, sidx, v, tw, twp, rtw_p, a, cx);
            rounds_rest<S_LOG, E_LOG, 1, true>(x, exch, sidx, v, tw, twp, rtw_p, a, cx);   // mul_mont next
        }
        mbar_wait(&bars[NSX], k & 1);
        {
            constexpr int R = 1 << SP::rlog(SP::Q - 1);
            const uint32_t *arow = (AIN ? xst : as) + w * S;
#pragma unroll
            for (int h = 0; h < E / R; h++)
#pragma unroll
                for (int mm = 0; mm < R; mm++) {
                    const int k1 = out_pos<S_LOG, E_LOG>(v, h, mm);
                    if constexpr (DBG == 3) acc[h * R + mm] += x[h * R + mm];
                    else acc[h * R + mm] = red2p(acc[h * R + mm] + mul_mont(x[h * R + mm], (PA_SMEM_PTR_CK(arow + k1, 4), arow[k1]), cx.p, cx.pinv), cx.p2);
                }
        }
        __syncthreads();                                 // X stage s and A^ are free
        if (threadIdx.x == 0 && DBG != 2 && DBG != 3) {
            if (it + NSX < it1) issue_x(cn, s);
            if (!AIN && it + 1 < it1) issue_a(ca, as);
        }
        step(cn);
        step(ca);
    }
    if (have_unit) {
        constexpr int R = 1 << SP::rlog(SP::Q - 1);
        uint32_t *dst = dslot + (size_t)fpi * L + (size_t)(frg * V + w) * S;
#pragma unroll
        for (int h = 0; h < E / R; h++)
#pragma unroll
            for (int mm = 0; mm < R; mm++) flush_one(dst + out_pos<S_LOG, E_LOG>(v, h, mm), acc[h * R + mm]);
    }
    // mode 3: the peer atomics are performed (system scope) before this CTA exits, so the
    // p2p_signal kernel that follows in stream order publishes complete sums
    if constexpr (MODE == 3) __threadfence_system();
}

}  // namespace pa
