// Exact reconstruction of the product integers and the Mersenne / power-of-two
// reductions of the MMH-MH pipeline.
//
//  * CRT (Garner) turns the P residues of every convolution coefficient into the
//    exact coefficient c_j < prod p_i (the plan guarantees the bound).
//  * Column sums: word u of  sum_j c_j 2^(B j)  (+ an optional addend, MH's c) is
//    gathered as a 64-bit sum of 32-bit windows of the coefficients.
//  * Carry resolution: the 64-bit column sums become 32-bit words with a
//    generate/propagate carry-lookahead scan (warp ballots, block, grid).
//  * Fold: y = Y mod (2^gamma - 1) = sum of gamma-bit chunks of Y, folded again
//    (PAPER.md:130-132), canonical zero (reading A6).
//  * MH extract: bits [alpha - m, alpha) of (b y + c) mod 2^alpha, MSB-first bytes
//    (Eq. 4; readings A5, A8).
#pragma once
#include <cstdint>
#include "modarith.cuh"

namespace pa {

constexpr int kMaxPrimes = 8;

struct CrtK {
    uint32_t P;
    uint32_t p[kMaxPrimes];
    uint32_t pinv[kMaxPrimes];
    // inv[i][l] = (p_0 ... p_{l-1})^{-1} mod p_i   for l <= i, Montgomery form
    // pm[i][l]  = (p_0 ... p_{l-1}) mod p_i        Montgomery form (l < i)
    uint32_t inv[kMaxPrimes];         // (p_0 ... p_{i-1})^{-1} mod p_i  (Montgomery form)
    uint32_t pmod[kMaxPrimes][kMaxPrimes];  // pmod[i][l] = p_l mod p_i (Montgomery form)
    // prod[l] = p_0 ... p_{l-1} as little-endian 32-bit words (l <= P), P words each
    uint32_t prod[kMaxPrimes + 1][kMaxPrimes];
};

// Garner: exact c (P 32-bit words, little-endian) from canonical residues r[i].
// u_0 = r_0; u_i = (r_i - (u_0 + p_0 (u_1 + p_1 (...)))) * (p_0...p_{i-1})^{-1} mod p_i;
// c = u_0 + p_0 u_1 + p_0 p_1 u_2 + ...
__device__ __forceinline__ void garner(const CrtK &K, const uint32_t *r, uint32_t *c) {
    uint32_t u[kMaxPrimes];
    for (uint32_t i = 0; i < K.P; i++) {
        const uint32_t p = K.p[i], pinv = K.pinv[i];
        // partial = u_0 + p_0 (u_1 + p_1 (... u_{i-1})) mod p_i, Horner from the inside
        uint32_t acc = 0;
        for (int l = (int)i - 1; l >= 0; l--) {
            // acc = u_l + p_l * acc
            acc = red1p(mul_mont(acc, K.pmod[i][l], p, pinv), p);
            acc = red1p(acc + (u[l] >= p ? u[l] - p : u[l]) % p, p);  // u_l < p_l may exceed p_i
        }
        uint32_t d = r[i] + p - acc;            // in (0, 2p)
        d = red1p(d, p);
        u[i] = (i == 0) ? r[0] : red1p(mul_mont(d, K.inv[i], p, pinv), p);
    }
    for (uint32_t w = 0; w < K.P; w++) c[w] = 0;
    for (uint32_t i = 0; i < K.P; i++) {       // c += u_i * prod[i]
        uint64_t carry = 0;
        for (uint32_t w = 0; w < K.P; w++) {
            const uint64_t t = (uint64_t)c[w] + (uint64_t)u[i] * K.prod[i][w] + carry;
            c[w] = (uint32_t)t;
            carry = t >> 32;
        }
    }
}

// 32-bit window of a multiword value x (nw words) starting at bit offset `off`
// (may be negative: the value starts inside the window).
__device__ __forceinline__ uint32_t window32(const uint32_t *x, int nw, int off) {
    if (off <= -32) return 0;
    if (off < 0) return x[0] << (-off);
    const int wi = off >> 5, sh = off & 31;
    if (wi >= nw) return 0;
    const uint32_t lo = x[wi];
    const uint32_t hi = (wi + 1 < nw) ? x[wi + 1] : 0u;
    return __funnelshift_r(lo, hi, sh);
}

// Column sums of Y = sum_{j < ncoef} c_j 2^(B j) (+ addend) for words [0, W).
// res: [P][L] canonical residues (natural coefficient order).
__global__ void crt_colsum(const uint32_t *__restrict__ res, uint32_t L, uint32_t ncoef,
                           uint32_t B, const CrtK K, const uint32_t *__restrict__ addend,
                           uint32_t n_addend, uint64_t *__restrict__ S, uint32_t W) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= W) return;
    const int64_t cbits = 32 * (int64_t)K.P;
    const int64_t lo_bit = 32 * (int64_t)u, hi_bit = lo_bit + 32;
    int64_t jlo = (lo_bit - cbits + 1 + B - 1);
    jlo = jlo <= 0 ? 0 : jlo / B;
    int64_t jhi = (hi_bit - 1) / B;
    if (jhi >= (int64_t)ncoef) jhi = (int64_t)ncoef - 1;
    uint64_t s = (addend && u < n_addend) ? addend[u] : 0ull;
    for (int64_t j = jlo; j <= jhi; j++) {
        uint32_t r[kMaxPrimes], c[kMaxPrimes];
        for (uint32_t i = 0; i < K.P; i++) r[i] = res[(size_t)i * L + j];
        garner(K, r, c);
        s += window32(c, (int)K.P, (int)(lo_bit - (int64_t)B * j));
    }
    S[u] = s;
}

// ---------------------------------------------------------------- carry resolution
// Words t_u = lo(S_u) + hi(S_{u-1}) < 2^32 + 2^31: generate g_u = t_u >> 32,
// propagate p_u = (uint32)t_u == 0xFFFFFFFF.  Final word = (uint32)t_u + carry_in_u.
constexpr int kTile = 1024;

__device__ __forceinline__ void word_gp(const uint64_t *S, uint32_t W, uint32_t u, uint32_t &w, int &g, int &pp) {
    uint64_t t = 0;
    if (u < W) {
        t = (S[u] & 0xFFFFFFFFull) + (u > 0 ? (S[u - 1] >> 32) : 0ull);
    }
    w = (uint32_t)t;
    g = (int)(t >> 32);
    pp = (u < W) && (w == 0xFFFFFFFFu);
}

// (g, p) of a whole warp / block given bit masks: carry-in to each lane and carry out.
__device__ __forceinline__ uint32_t lane_carries(uint32_t Gm, uint32_t Pm, uint32_t cin, uint32_t &cout) {
    const uint64_t A = (uint64_t)(Gm | Pm), Bm = Gm;
    const uint64_t sum = A + Bm + cin;
    cout = (uint32_t)(sum >> 32);
    return (uint32_t)sum ^ (uint32_t)A ^ (uint32_t)Bm;
}

// Block-level carry resolution of one tile of kTile words with block carry-in `cin`
// (uniform).  Returns this thread's word carry-in; block carry-out in *bcout.
__device__ __forceinline__ uint32_t block_carries(int g, int pp, uint32_t cin, uint32_t *bcout) {
    __shared__ uint32_t wg[32], wp[32], wc[32];
    __shared__ uint32_t s_cout;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t Gm = __ballot_sync(0xFFFFFFFFu, g), Pm = __ballot_sync(0xFFFFFFFFu, pp);
    uint32_t co0;
    (void)lane_carries(Gm, Pm, 0, co0);            // warp generate (cin = 0)
    if (lane == 0) { wg[wid] = co0; wp[wid] = (Pm == 0xFFFFFFFFu); }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        const uint32_t G2 = __ballot_sync(0xFFFFFFFFu, lane < nw ? wg[lane] : 0);
        const uint32_t P2 = __ballot_sync(0xFFFFFFFFu, lane < nw ? wp[lane] : 0);
        uint32_t co;
        const uint32_t C2 = lane_carries(G2, P2, cin, co);
        wc[lane] = (C2 >> lane) & 1;
        if (lane == 0) {
            // carry out of the last active warp
            uint32_t c = cin;
            for (int i = 0; i < nw; i++) c = ((G2 >> i) & 1) | (((P2 >> i) & 1) & c);
            s_cout = c;
        }
    }
    __syncthreads();
    uint32_t co;
    const uint32_t C = lane_carries(Gm, Pm, wc[wid], co);
    if (bcout) *bcout = s_cout;
    return (C >> lane) & 1;
}

// Phase A: (g, p) summary per tile.
__global__ void carry_tiles(const uint64_t *__restrict__ S, uint32_t W, uint8_t *__restrict__ tg,
                            uint8_t *__restrict__ tp) {
    const uint32_t u = blockIdx.x * kTile + threadIdx.x;
    uint32_t w; int g, pp;
    word_gp(S, W, u, w, g, pp);
    // tile propagate = all words propagate (out-of-range words count as propagate so
    // the last partial tile passes carries through; they are never written)
    const int pfull = (u < W) ? pp : 1;
    const int allp = __syncthreads_and(pfull);
    uint32_t cout;
    (void)block_carries(g, pp, 0, &cout);
    if (threadIdx.x == 0) { tg[blockIdx.x] = (uint8_t)cout; tp[blockIdx.x] = (uint8_t)allp; }
}

// Phase B: carry-in of every tile (single block, sequential chunks + block scan).
__global__ void carry_scan(const uint8_t *__restrict__ tg, const uint8_t *__restrict__ tp, uint32_t ntiles,
                           const uint32_t *__restrict__ cin0, uint8_t *__restrict__ tcin,
                           uint32_t *__restrict__ carry_out) {
    const uint32_t T = blockDim.x;
    const uint32_t per = (ntiles + T - 1) / T;
    const uint32_t b0 = threadIdx.x * per;
    const uint32_t b1 = min(ntiles, b0 + per);
    int G = 0, Pp = 1;
    for (uint32_t t = b0; t < b1; t++) { G = tg[t] | (tp[t] & G); Pp &= tp[t]; }
    const uint32_t cin = cin0 ? (*cin0 & 1u) : 0u;
    uint32_t bcout;
    uint32_t c = block_carries(G, (b0 < b1) ? Pp : 1, cin, &bcout);
    for (uint32_t t = b0; t < b1; t++) { tcin[t] = (uint8_t)c; c = tg[t] | (tp[t] & c); }
    if (threadIdx.x == 0 && carry_out) *carry_out = bcout;
}

// Phase C: final words.
__global__ void carry_apply(const uint64_t *__restrict__ S, uint32_t W, const uint8_t *__restrict__ tcin,
                            uint32_t *__restrict__ out) {
    const uint32_t u = blockIdx.x * kTile + threadIdx.x;
    uint32_t w; int g, pp;
    word_gp(S, W, u, w, g, pp);
    const uint32_t c = block_carries(g, pp, tcin[blockIdx.x], nullptr);
    if (u < W) out[u] = w + c;
}

// ---------------------------------------------------------------- fold mod 2^gamma - 1
// bits [start, start + 32) of X (nw words), zero beyond nw words.
__device__ __forceinline__ uint32_t bits32(const uint32_t *X, uint64_t nw, uint64_t start) {
    const uint64_t wi = start >> 5;
    const int sh = (int)(start & 31);
    const uint32_t lo = wi < nw ? X[wi] : 0u;
    const uint32_t hi = wi + 1 < nw ? X[wi + 1] : 0u;
    return __funnelshift_r(lo, hi, sh);
}

// S_u = sum over gamma-bit chunks t of word u of chunk_t(X), u < Wg = ceil(gamma/32),
// plus S_{Wg} = 0 (room for the overflow).
__global__ void fold_colsum(const uint32_t *__restrict__ X, uint64_t nwx, uint64_t gamma,
                            uint64_t *__restrict__ S, uint32_t Wout) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= Wout) return;
    const uint64_t Wg = (gamma + 31) >> 5;
    uint64_t s = 0;
    if (u < Wg) {
        const uint64_t nbits = 32 * nwx;
        const uint64_t nch = (nbits + gamma - 1) / gamma;
        const uint64_t off = 32 * (uint64_t)u;
        uint32_t mask = 0xFFFFFFFFu;
        if (off + 32 > gamma) mask = (uint32_t)((1ull << (gamma - off)) - 1);
        for (uint64_t t = 0; t < nch; t++) s += bits32(X, nwx, t * gamma + off) & mask;
    }
    S[u] = s;
}

// y (Wout words) -> S_u = (y mod 2^gamma)_u + [u == 0] * (y >> gamma).
__global__ void fold_final_colsum(const uint32_t *__restrict__ y, uint64_t gamma,
                                  uint64_t *__restrict__ S, uint32_t Wout) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= Wout) return;
    const uint64_t off = 32 * (uint64_t)u;
    uint64_t s = 0;
    if (off < gamma) {
        uint32_t mask = 0xFFFFFFFFu;
        if (off + 32 > gamma) mask = (uint32_t)((1ull << (gamma - off)) - 1);
        s = y[u] & mask;
    }
    if (u == 0) {
        // y >> gamma: at most 64 bits are ever non-zero here
        s += bits32(y, Wout, gamma) + ((uint64_t)bits32(y, Wout, gamma + 32) << 32);
    }
    S[u] = s;
}

// flag = (y == 2^gamma - 1) over the low gamma bits (y < 2^gamma guaranteed).
__global__ void allones_check(const uint32_t *__restrict__ y, uint64_t gamma, uint32_t *flag) {
    const uint64_t Wg = (gamma + 31) >> 5;
    int bad = 0;
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < Wg; u += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t want = 0xFFFFFFFFu;
        if (32 * u + 32 > gamma) want = (uint32_t)((1ull << (gamma - 32 * u)) - 1);
        if (y[u] != want) bad = 1;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

// canonical zero (reading A6): if y == p, y := 0.  flag = 0 means "not all ones".
__global__ void zero_if_allones(uint32_t *__restrict__ y, uint32_t W, const uint32_t *flag) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < W && *flag == 0) y[u] = 0;
}

// ---------------------------------------------------------------- MH output
// out byte q = bits of z = Z mod 2^alpha >> (alpha - m), MSB-first (reading A5).
// Each thread writes one byte (bytes are few: ceil(m/8)).
__global__ void mh_extract(const uint32_t *__restrict__ Z, uint64_t nwz, uint64_t alpha, uint64_t m,
                           uint8_t *__restrict__ out, uint64_t nbytes) {
    const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (q >= nbytes) return;
    // output bits 8q .. 8q+7 are z bits m-1-8q ... m-8-8q = Z bits alpha-1-8q ... alpha-8-8q
    const int64_t top = (int64_t)alpha - 1 - 8 * (int64_t)q;          // Z bit of the byte's MSB
    const int64_t lowb = top - 7;
    uint32_t v;
    if (lowb >= 0) {
        v = (bits32(Z, nwz, (uint64_t)lowb) & 0xFFu);
    } else {
        v = (bits32(Z, nwz, 0) << (-lowb)) & 0xFFu;
    }
    // pad bits (output bit index >= m) are zero
    const int64_t valid = (int64_t)m - 8 * (int64_t)q;                  // bits of this byte that exist
    if (valid < 8) v &= (0xFFu << (8 - valid)) & 0xFFu;
    out[q] = (uint8_t)v;
}

}  // namespace pa
