// Exact reconstruction of the product integers and the Mersenne / power-of-two
// reductions of the MMH-MH pipeline.
//
//  * CRT (approximate-quotient form, no Garner chain) turns the P residues of every
//    convolution coefficient into the exact coefficient c_j < prod p_i (the plan
//    guarantees the bound), one thread per coefficient; a second kernel forms the
//    64-bit column sums of the 32-bit output words from those coefficients.
//  * MMH (S4+S5): the column sums are taken on the gamma-bit ring directly: coefficient j
//    sits at bit (B j) mod gamma, and a piece that crosses bit gamma wraps to bit 0 --
//    this is the fold x mod M_gamma = floor(x / 2^gamma) + x mod 2^gamma
//    applied to each coefficient before the carries.
//  * MH (S7): plain column sums of b*y plus the addend c, words below alpha
//    (Eq. 4).
//  * Carry resolution: 64-bit column sums -> 32-bit words with a generate/propagate
//    carry-lookahead: 8 words per thread, warp ballots inside a tile, single-pass
//    decoupled look-back between tiles (a tile that does not propagate ends the look-back).
//  * Mersenne finish: the residual fold (x >> gamma) + (x mod 2^gamma) and canonical zero
//    (reading A6) in one CTA; MH bit extraction (readings A5, A8).
#pragma once
#include <cstdint>
#include "modarith.cuh"

namespace pa {

struct CrtK {
    uint32_t P;
    uint32_t p[kMaxPrimes];
    uint32_t pinv[kMaxPrimes];
    uint32_t qinv[kMaxPrimes];                // (M / p_i)^{-1} mod p_i, Montgomery form
    uint64_t G[kMaxPrimes];                   // floor(2^64 / p_i)
    uint32_t MI[kMaxPrimes][kMaxPrimes];      // M / p_i, little-endian words
    uint32_t M[kMaxPrimes];                   // M = p_0 ... p_{P-1}, little-endian words
};

// Exact coefficient c < M' (M' = 2^-0.5 M at most, the planner's margin) from its
// residues r_i (canonical), CRT with an approximate quotient:
//   y_i = r_i (M/p_i)^{-1} mod p_i,   c = sum_i y_i (M/p_i) - k M,
//   k = floor(sum_i y_i / p_i) evaluated in 64-bit fixed point (q_i = y_i floor(2^64/p_i),
//   error < P 2^-34 per unit) with a bias of 2^-24: exact because c/M <= 2^-0.5 keeps the
//   fractional part away from 1.  All coefficients are independent (no Garner chain).
// One thread per coefficient; word-major layout coef[w][j] (coalesced), P words each.
template <int P>
#ifndef PA_CRT_MINB
#define PA_CRT_MINB 1
#endif
__global__ void __launch_bounds__(128, PA_CRT_MINB) crt_coeffs(const uint32_t *__restrict__ res, uint32_t L, uint32_t ncoef,
                                                  const CrtK K, uint32_t *__restrict__ coef) {
    PA_TMARK(0x4000 | P, 0);
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ncoef) return;
    uint32_t y[P];
    uint64_t slo = 1ull << 40, shi = 0;                // bias 2^-24
#pragma unroll
    for (int i = 0; i < P; i++) {
        const uint32_t r = PA_AT(res + (size_t)i * L + j);
        y[i] = red1p(mul_mont(r, K.qinv[i], K.p[i], K.pinv[i]), K.p[i]);
        const uint64_t q = (uint64_t)y[i] * K.G[i];
        slo += q;
        shi += (slo < q);
    }
    const uint32_t k = (uint32_t)shi;
    // sum_i y_i (M/p_i): products < 2^62, so four of them are summed in one 64-bit
    // accumulator per word (one mad.wide each) before being split into 32-bit columns
    uint64_t acc[P + 1];
#pragma unroll
    for (int w = 0; w <= P; w++) acc[w] = 0;
#pragma unroll
    for (int g = 0; g < P; g += 4) {
        uint64_t t[P];
#pragma unroll
        for (int w = 0; w < P; w++) t[w] = 0;
#pragma unroll
        for (int i = g; i < g + 4 && i < P; i++)
#pragma unroll
            for (int w = 0; w < P; w++) t[w] = mad_wide(y[i], K.MI[i][w], t[w]);
#pragma unroll
        for (int w = 0; w < P; w++) {
            acc[w] += (uint32_t)t[w];
            acc[w + 1] += t[w] >> 32;
        }
    }
    // words of sum_i y_i M_i (P + 1 words) minus k M
    uint64_t carry = 0;
    int64_t borrow = 0;
    uint32_t *out = coef + j;
#pragma unroll
    for (int w = 0; w < P; w++) {
        const uint64_t v = acc[w] + carry;
        carry = v >> 32;
        const uint64_t km = (uint64_t)k * K.M[w];
        // subtract low word of k M (its high part carries into the next word via `borrow`)
        const int64_t d = (int64_t)(uint32_t)v - (int64_t)(uint32_t)km + borrow;
        PA_AT(out + (size_t)w * ncoef) = (uint32_t)d;
        borrow = (d >> 32) - (int64_t)(km >> 32);       // arithmetic shift: -1 on underflow
    }
}

// ---------------------------------------------------------------- carry resolution
// (g, p) over 32 lanes given ballot masks: per-lane carry-in (bit i) and carry out.
__device__ __forceinline__ uint32_t lane_carries(uint32_t Gm, uint32_t Pm, uint32_t cin, uint32_t &cout) {
    const uint64_t A = (uint64_t)(Gm | Pm), Bm = Gm;
    const uint64_t sum = A + Bm + cin;
    cout = (uint32_t)(sum >> 32);
    return (uint32_t)sum ^ (uint32_t)A ^ (uint32_t)Bm;
}

// Carry-in of this thread's word within a block of kTile words with block carry-in
// `cin`; block aggregate (generate with cin = 0) in *bg.
__device__ __forceinline__ uint32_t block_carries(int g, int pp, uint32_t cin, uint32_t *bg) {
    __shared__ uint32_t wg[32], wp[32], wc[32];
    __shared__ uint32_t s_bg;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t Gm = __ballot_sync(0xFFFFFFFFu, g), Pm = __ballot_sync(0xFFFFFFFFu, pp);
    uint32_t co0;
    (void)lane_carries(Gm, Pm, 0, co0);
    __syncthreads();
    if (lane == 0) { wg[wid] = co0; wp[wid] = (Pm == 0xFFFFFFFFu); }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        const uint32_t G2 = __ballot_sync(0xFFFFFFFFu, lane < nw ? wg[lane] : 0);
        const uint32_t P2 = __ballot_sync(0xFFFFFFFFu, lane < nw ? wp[lane] : 1);
        uint32_t co;
        const uint32_t C2 = lane_carries(G2, P2, cin, co);
        wc[lane] = (C2 >> lane) & 1;
        uint32_t co_g;
        (void)lane_carries(G2, P2, 0, co_g);
        if (lane == 0) s_bg = co_g;
    }
    __syncthreads();
    uint32_t co;
    const uint32_t C = lane_carries(Gm, Pm, wc[wid], co);
    if (bg) *bg = s_bg;
    return (C >> lane) & 1;
}

// block_carries for both block carry-ins at once: *c0 / *c1 = this thread's carry-in with
// block carry-in 0 / 1, *bg = block generate.  One scan, so a caller that learns its carry-in
// later (decoupled look-back) only selects.
__device__ __forceinline__ void block_carries2(int g, int pp, uint32_t *c0, uint32_t *c1, uint32_t *bg) {
    __shared__ uint32_t wc0[32], wc1[32];
    __shared__ uint32_t wg2[32], wp2[32];
    __shared__ uint32_t s_bg2;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t Gm = __ballot_sync(0xFFFFFFFFu, g), Pm = __ballot_sync(0xFFFFFFFFu, pp);
    uint32_t co0;
    (void)lane_carries(Gm, Pm, 0, co0);
    if (lane == 0) { wg2[wid] = co0; wp2[wid] = (Pm == 0xFFFFFFFFu); }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        const uint32_t G2 = __ballot_sync(0xFFFFFFFFu, lane < nw ? wg2[lane] : 0);
        const uint32_t P2 = __ballot_sync(0xFFFFFFFFu, lane < nw ? wp2[lane] : 1);
        uint32_t co;
        wc0[lane] = (lane_carries(G2, P2, 0, co) >> lane) & 1;
        s_bg2 = co;                                           // same for every lane
        wc1[lane] = (lane_carries(G2, P2, 1, co) >> lane) & 1;
    }
    __syncthreads();
    uint32_t co;
    *c0 = (lane_carries(Gm, Pm, wc0[wid], co) >> lane) & 1;
    *c1 = (lane_carries(Gm, Pm, wc1[wid], co) >> lane) & 1;
    *bg = s_bg2;
}

// Sources of 64-bit column sums for the carry kernel.
struct SrcArr {
    const uint64_t *S;
    uint32_t n;            // words present; S_u = 0 for u >= n
    __device__ __forceinline__ uint64_t operator()(uint32_t u) const { return u < n ? PA_AT(S + u) : 0ull; }
};
// Sum of G residues (S6): S_u = sum_g parts[g][u].
struct SrcParts {
    const uint32_t *parts;
    uint32_t G, Wg;
    __device__ __forceinline__ uint64_t operator()(uint32_t u) const {
        uint64_t s = 0;
        if (u < Wg)
            for (uint32_t g = 0; g < G; g++) s += PA_AT(parts + (size_t)g * Wg + u);
        return s;
    }
};

// ---------------------------------------------------------------- multiword carry scan
// out[u] = word u of sum_u S_u 2^(32u) for u < W (the caller sizes W so nothing is
// lost above).  One thread owns kCarryV consecutive words; a tile is 256 threads.
// Word u: t_u = lo32(S_u) + hi32(S_{u-1}) < 2^33 -> digit w_u = lo32(t_u) with a
// generate bit g_u = t_u >> 32 and a propagate bit p_u = (w_u == 2^32 - 1).  Thread
// aggregates are scanned with warp ballots; tiles chain through decoupled look-back.
constexpr int kCarryV = 8;
constexpr int kCarryT = 256;
constexpr int kCarryTile = kCarryV * kCarryT;

template <class Src>
__global__ void __launch_bounds__(kCarryT) carry_mw(const Src src, uint32_t W, uint32_t *__restrict__ out,
                                                  uint32_t *state, uint32_t *ticket) {
    __shared__ uint32_t s_tile, s_cin;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t u0 = tile * kCarryTile + threadIdx.x * kCarryV;
    uint32_t w[kCarryV];
    uint32_t gm = 0, pm = 0;                       // per-word generate / propagate bits
    uint64_t prev = (u0 > 0 && u0 - 1 < W) ? src(u0 - 1) : 0ull;
#pragma unroll
    for (int j = 0; j < kCarryV; j++) {
        const uint32_t u = u0 + j;
        const uint64_t s = (u < W) ? src(u) : 0ull;
        const uint64_t t = (s & 0xFFFFFFFFull) + (prev >> 32);
        prev = s;
        w[j] = (uint32_t)t;
        gm |= (uint32_t)(t >> 32) << j;
        pm |= (uint32_t)((u >= W) || (w[j] == 0xFFFFFFFFu)) << j;
    }
    // thread aggregate (carry out with carry-in 0; all-propagate)
    uint32_t G = 0;
#pragma unroll
    for (int j = 0; j < kCarryV; j++) G = ((gm >> j) & 1u) | (((pm >> j) & 1u) & G);
    const int Pall = (pm == (1u << kCarryV) - 1u);
    const int allp = __syncthreads_and(Pall);
    uint32_t bg;
    (void)block_carries((int)G, Pall, 0, &bg);
    if (threadIdx.x == 0) {
        volatile uint32_t *vs = state;
        const uint32_t ntiles = (W + kCarryTile - 1) / kCarryTile;
        uint32_t cin = 0;
        if (tile > 0) {
            PA_CK(vs + tile, 4);
            vs[tile] = 1u | (bg << 1) | ((uint32_t)allp << 2);
            __threadfence();
            uint32_t accG = 0, accP = 1;
            int64_t j = (int64_t)tile - 1;
            for (;;) {
                if (j < 0) { cin = accG; break; }
                PA_CK(vs + j, 4);
                const uint32_t st = vs[j];
                if (st == 0) continue;
                if (st & 8u) { cin = accG | (accP & ((st >> 4) & 1u)); break; }
                accG |= accP & ((st >> 1) & 1u);
                accP &= (st >> 2) & 1u;
                if (!accP) { cin = accG; break; }
                j--;
            }
        }
        const uint32_t incl = bg | ((uint32_t)allp & cin);
        __threadfence();
        vs[tile] = 1u | (bg << 1) | ((uint32_t)allp << 2) | 8u | (incl << 4);
        s_cin = cin;
        (void)ntiles;
    }
    __syncthreads();
    uint32_t c = block_carries((int)G, Pall, s_cin, nullptr);
#pragma unroll
    for (int j = 0; j < kCarryV; j++) {
        const uint32_t u = u0 + j;
        if (u < W) PA_AT(out + u) = w[j] + c;
        c = ((gm >> j) & 1u) | (((pm >> j) & 1u) & c);
    }
}

// ---------------------------------------------------------------- Mersenne finish
// y (Wtot words, y < 2^(32 Wtot)) -> y mod (2^gamma - 1), canonical in [0, p-1]
// (reading A6), in place, by the fold x mod M_gamma = (x >> gamma) + (x mod 2^gamma)
// repeated until nothing is left above bit gamma.  Run by one CTA (any
// block size): the fold adds a short number (Wtot - floor(gamma/32) <= 64 words) at bit
// 0, whose carry ripples only through a run of all-ones words -- one chunk of blockDim
// words almost always, more chunks only for such runs (correct either way).
constexpr int kFinT = 1024;

__device__ __forceinline__ void fin_ripple(uint32_t *y, uint32_t Wtot, uint32_t from) {
    // add 1 at word `from`, rippling through all-ones words
    __shared__ uint32_t s_first;
    for (uint32_t base = from; base < Wtot; base += blockDim.x) {
        if (threadIdx.x == 0) s_first = 0xFFFFFFFFu;
        __syncthreads();
        const uint32_t u = base + threadIdx.x;
        const uint32_t v = (u < Wtot) ? PA_AT(y + u) : 0u;
        if (u < Wtot && v != 0xFFFFFFFFu) atomicMin(&s_first, u);
        __syncthreads();
        const uint32_t f = s_first;
        if (u < Wtot && u < f) PA_AT(y + u) = 0u;
        if (u == f) PA_AT(y + u) = v + 1u;
        __syncthreads();
        if (f != 0xFFFFFFFFu) return;     // carry absorbed (uniform)
    }
}

__device__ void mersenne_finish_dev(uint32_t *y, uint32_t Wtot, uint64_t gamma) {
    __shared__ uint32_t T[64];
    __shared__ uint32_t s_nz, s_carry, s_bad;
    const uint32_t gw = (uint32_t)(gamma >> 5);
    const int gs = (int)(gamma & 31);
    const uint32_t nT = Wtot - gw;                       // words of y >> gamma (<= 64)
    for (;;) {
        if (threadIdx.x == 0) s_nz = 0;
        __syncthreads();
        for (uint32_t t = threadIdx.x; t < nT; t += blockDim.x) {
            const uint32_t i = gw + t;
            const uint32_t lo = PA_AT(y + i), hi = (i + 1 < Wtot) ? PA_AT(y + i + 1) : 0u;
            const uint32_t v = gs ? __funnelshift_r(lo, hi, gs) : lo;
            T[t] = v;
            if (v) atomicOr(&s_nz, 1u);
        }
        __syncthreads();
        if (!s_nz) break;
        for (uint32_t t = threadIdx.x; t < nT; t += blockDim.x) {     // clear bits >= gamma
            const uint32_t i = gw + t;
            if (t == 0 && gs) PA_AT(y + i) &= (1u << gs) - 1u;
            else PA_AT(y + i) = 0u;
        }
        __syncthreads();
        // y += T (short add, nT <= 64 words) by the first two warps: one word per lane, the
        // carries by generate/propagate ballots, warp 0's carry-out into warp 1; the carry out
        // of word lim-1 (= the carry into lane lim) continues in fin_ripple
        {
            __shared__ uint32_t s_Cw[2], s_co[2];
            const uint32_t t = threadIdx.x;
            const uint32_t lim = min(nT, Wtot);
            uint64_t sum = 0;
            uint32_t Gm = 0, Pm = 0;
            if (t < 64) {
                const uint32_t yv = (t < lim) ? PA_AT(y + t) : 0u;
                sum = (uint64_t)yv + ((t < lim) ? T[t] : 0u);
                Gm = __ballot_sync(0xFFFFFFFFu, (uint32_t)(sum >> 32));
                Pm = __ballot_sync(0xFFFFFFFFu, (uint32_t)sum == 0xFFFFFFFFu);
                if (t == 0) {
                    uint32_t co;
                    s_Cw[0] = lane_carries(Gm, Pm, 0, co);
                    s_co[0] = co;
                }
            }
            __syncthreads();
            if (t == 32) {
                uint32_t co;
                s_Cw[1] = lane_carries(Gm, Pm, s_co[0], co);
                s_co[1] = co;
            }
            __syncthreads();
            if (t < 64 && t < lim) PA_AT(y + t) = (uint32_t)sum + ((s_Cw[t >> 5] >> (t & 31)) & 1u);
            if (t == 0) s_carry = (lim < 64) ? ((s_Cw[lim >> 5] >> (lim & 31)) & 1u) : s_co[1];
        }
        __syncthreads();
        if (s_carry && nT < Wtot) fin_ripple(y, Wtot, nT);
        __syncthreads();
    }
    // canonical zero: y == 2^gamma - 1 -> 0
    const uint32_t Wg = (uint32_t)((gamma + 31) >> 5);
    for (uint32_t base = 0; base < Wg; base += blockDim.x) {
        if (threadIdx.x == 0) s_bad = 0;
        __syncthreads();
        const uint32_t u = base + threadIdx.x;
        if (u < Wg) {
            const uint32_t want = (u == Wg - 1 && gs) ? ((1u << gs) - 1u) : 0xFFFFFFFFu;
            if (PA_AT(y + u) != want) atomicOr(&s_bad, 1u);
        }
        __syncthreads();
        if (s_bad) return;
    }
    for (uint32_t u = threadIdx.x; u < Wg; u += blockDim.x) PA_AT(y + u) = 0u;
}

__global__ void __launch_bounds__(kFinT) mersenne_finish_k(uint32_t *__restrict__ y, uint32_t Wtot, uint64_t gamma) {
    mersenne_finish_dev(y, Wtot, gamma);
}

// ---------------------------------------------------------------- fused CRT + carries
// S4/S5 (MMH) and S7 (MH) tail after crt_coeffs.  A CTA (ticket order) owns kCarryTile
// output words [u0, u1).  For each chunk of the ring it stages the exact coefficients
// (from crt_coeffs) whose pieces meet its words in shared memory, forms the 64-bit column
// sums S_u of its words (RING: pieces cut at bit gamma, high parts land at bit 0 -- the
// Mersenne fold of PAPER.md:130-132 per coefficient; LINEAR: plus the addend c), then
// resolves the carries: digit d_u = lo32(S_u) + hi32(S_{u-1}) inside the tile, binary
// generate/propagate scan over words u0+1.., and a small multi-bit carry between tiles:
//   C_out = hi32(S_{u1-1}) + carry_out(c1),  c1 = [w_{u0} + C_in >= 2^32].
// A tile whose carry-out does not depend on C_in (it generates, or some word does not
// propagate) publishes C_out before waiting for its predecessor, so the chain is
// almost never serial.  RING: the last CTA to finish runs the Mersenne finish.
// state: [0] ticket, [kFlagStride] done counter, [kFlagStride (2 + t)] tile t: bit 31 ready,
// bits 0..30 C_out -- one 128-byte line per word, so the publishers' stores and the
// successors' polls of different tiles (and the two counters) do not contend for a line.
constexpr uint32_t kFlagStride = 32;
__device__ __forceinline__ void st_relaxed_gpu(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// bits [off, off + 32) of a coefficient held in shared memory (P words at stride 1)
template <int P>
__device__ __forceinline__ uint32_t coef_window_s(const uint32_t *c, int off, int len) {
    if (off <= -32 || off >= len) return 0;
    uint32_t v;
    if (off < 0) {
        v = c[0] << (-off);
    } else {
        const int wi = off >> 5, sh = off & 31;
        const uint32_t lo = c[wi];
        const uint32_t hi = (wi + 1 < P) ? c[wi + 1] : 0u;
        v = __funnelshift_r(lo, hi, sh);
    }
    const int top = len - off;
    if (top < 32) v &= (top <= 0) ? 0u : ((1u << top) - 1u);
    return v;
}

template <int P>
__host__ __device__ constexpr int crt_cstride() { return P | 1; }
#ifndef PA_CCV
#define PA_CCV 4
#endif
constexpr int kCCV = PA_CCV;                   // words per thread in crt_carry
constexpr int kCCT = 256;                      // threads per tile
constexpr int kCCTile = kCCV * kCCT;                 // odd stride: fewer bank conflicts

template <int P, bool RING, int DBG = 0>
__global__ void __launch_bounds__(kCCT) crt_carry(const uint32_t *__restrict__ coefT, uint32_t L, uint32_t ncoef,
                                                     uint32_t B, uint32_t gamma,
                                                     const uint32_t *__restrict__ addend, uint32_t n_addend,
                                                     uint32_t *__restrict__ out, uint32_t W, uint32_t cap,
                                                     uint32_t *state, uint32_t Wfin, uint32_t *__restrict__ obe) {
    (void)cap;
    // column sums of the tile's words, scatter form: a thread owns whole coefficients
    // (P words loaded from coefT, coalesced) and adds their P + 1 bit-shifted words into
    // the tile's 64-bit sums in shared memory (shared-memory atomics: <= ceil(32(P+1)/B)+1
    // contributions per word)
    // 64-bit column sums as two 32-bit words: a native 32-bit shared atomicAdd on the low
    // word (its old value reveals the carry) instead of a 64-bit add, which sm_100a only has
    // as a compare-and-swap loop
    __shared__ uint32_t s_clo[kCCTile], s_chi[kCCTile];
    constexpr uint32_t cbits = 32 * P;
    __shared__ uint32_t s_tile, s_cin, s_c1, s_last;
    __shared__ uint32_t s_hi[kCCT];
    constexpr uint32_t kKid = 0x5000 | P | (RING ? 0x80 : 0);
    PA_TMARK(kKid, 0);
    if (threadIdx.x == 0) { PA_CK(state, 4); s_tile = atomicAdd(&state[0], 1u); }
    for (uint32_t i = threadIdx.x; i < kCCTile; i += blockDim.x) s_clo[i] = s_chi[i] = 0u;
    __syncthreads();
    const uint32_t tile = s_tile;
    PA_TMARK_B(kKid, 7, 0x100000 | tile);               // ticket known (scripts/tprof.py phase base)
    const uint32_t u0 = tile * kCCTile;
    const uint32_t ub = u0 + threadIdx.x * kCCV;            // this thread's first word
    const uint32_t nchunks = (DBG & 8) ? 0u : RING ? (uint32_t)(((uint64_t)B * ncoef + gamma - 1) / gamma) : 1u;
    const uint32_t tb0 = 32 * u0, tb1 = 32 * min(u0 + kCCTile, W);   // tile bits
    // adds bits [0, len) of coefficient c, placed at tile-relative bit d, into the sums
    auto scatter = [&](const uint32_t (&c)[P], int64_t d, int64_t len) {
        uint32_t m[P];
#pragma unroll
        for (int w = 0; w < P; w++) {
            const int64_t top = len - 32 * w;                  // bits of word w inside [0, len)
            m[w] = top >= 32 ? c[w] : (top <= 0 ? 0u : (c[w] & ((1u << top) - 1u)));
        }
        const int64_t wq = d >> 5;                            // floor
        const int s = (int)(d & 31);
#pragma unroll
        for (int i = 0; i <= P; i++) {
            const int64_t wi = wq + i;
            if (wi < 0 || wi >= (int64_t)kCCTile) continue;
            PA_IDX_CK(wi, kCCTile);
            const uint32_t lo = (i > 0) ? m[i - 1] : 0u, hi = (i < P) ? m[i] : 0u;
            const uint32_t val = s ? __funnelshift_l(lo, hi, s) : hi;
            if (val) {
                const uint32_t old = atomicAdd(&s_clo[wi], val);
                if (old + val < old) atomicAdd(&s_chi[wi], 1u);
            }
        }
    };
    for (uint32_t t = 0; t < nchunks; t++) {
        const uint32_t base = RING ? t * gamma : 0u;
        const uint32_t jc0 = (base + B - 1) / B;
        uint32_t jc1 = ncoef - 1;
        if (RING) jc1 = min(jc1, (uint32_t)(((uint64_t)(t + 1) * gamma + B - 1) / B) - 1);
        uint32_t ja = (tb0 + base > cbits) ? (tb0 + base - cbits) / B : 0u;
        uint32_t jb = (tb1 - 1 + base) / B;
        if (ja < jc0) ja = jc0;
        if (jb > jc1) jb = jc1;
        if (jb < ja || jb == 0xFFFFFFFFu) continue;           // uniform
        for (uint32_t j = ja + threadIdx.x; j <= jb; j += blockDim.x) {
            uint32_t c[P];
#pragma unroll
            for (int w = 0; w < P; w++) c[w] = (DBG & 1) ? 0u : PA_LDG(coefT + (size_t)w * ncoef + j);
            const int64_t pos = (int64_t)B * j - base;        // ring / linear bit of the piece
            int64_t len = cbits;
            if (RING && pos + len > (int64_t)gamma) len = (int64_t)gamma - pos;
            scatter(c, pos - (int64_t)tb0, len);
        }
    }
    if (RING && tb0 < cbits + 32 && !(DBG & 8)) {
        // wrapped pieces: the bits of a coefficient above the ring top land at ring bit 0
        for (uint32_t t = 0; t < nchunks; t++) {
            const int64_t base = (int64_t)t * gamma;
            const int64_t top = base + (int64_t)gamma;
            int64_t jx = (top - (int64_t)cbits) / (int64_t)B;
            const int64_t jc0 = (base + B - 1) / B;
            if (jx < jc0) jx = jc0;
            int64_t jy = (top - 1) / (int64_t)B;
            if (jy > (int64_t)ncoef - 1) jy = (int64_t)ncoef - 1;
            for (int64_t j = jx + threadIdx.x; j <= jy; j += blockDim.x) {
                const int64_t pos = (int64_t)B * j - base;
                if (pos + (int64_t)cbits <= (int64_t)gamma) continue;
                const int cut = (int)((int64_t)gamma - pos);
                uint32_t c[P], h[P];
#pragma unroll
                for (int w = 0; w < P; w++) c[w] = PA_AT(coefT + (size_t)w * ncoef + j);
                // h = c >> cut (the part above the ring top), placed at ring bit 0
                const int cw = cut >> 5, cs = cut & 31;
#pragma unroll
                for (int w = 0; w < P; w++) {
                    uint32_t lo = 0, hi = 0;
#pragma unroll
                    for (int q = 0; q < P; q++) { if (q == w + cw) lo = c[q]; if (q == w + cw + 1) hi = c[q]; }
                    h[w] = cs ? __funnelshift_r(lo, hi, cs) : lo;
                }
                scatter(h, -(int64_t)tb0, cbits);
            }
        }
    }
    __syncthreads();
    PA_TMARK_B(kKid, 2, 0x100000 | tile);
    uint64_t S[kCCV];
#pragma unroll
    for (int v = 0; v < kCCV; v++) {
        const uint32_t u = ub + v;
        const uint32_t iw = threadIdx.x * kCCV + v;
        S[v] = (((uint64_t)s_chi[iw] << 32) | s_clo[iw]) + ((!RING && addend && u < n_addend) ? PA_AT(addend + u) : 0ull);
    }
    // ---- carries inside the tile (cin of word u0 handled separately, see above)
    uint32_t w[kCCV];
    uint32_t gm = 0, pm = 0;
    s_hi[threadIdx.x] = (uint32_t)(S[kCCV - 1] >> 32);
    __syncthreads();
    uint32_t hprev = threadIdx.x ? s_hi[threadIdx.x - 1] : 0u;
#pragma unroll
    for (int v = 0; v < kCCV; v++) {
        const uint32_t u = ub + v;
        const uint64_t t = (S[v] & 0xFFFFFFFFull) + hprev;
        hprev = (uint32_t)(S[v] >> 32);
        w[v] = (uint32_t)t;
        const bool first = (threadIdx.x == 0 && v == 0);       // word u0: transparent in the scan
        gm |= (uint32_t)(first ? 0u : (uint32_t)(t >> 32)) << v;
        pm |= (uint32_t)(first || u >= W || w[v] == 0xFFFFFFFFu) << v;
    }
    uint32_t G = 0;
#pragma unroll
    for (int v = 0; v < kCCV; v++) G = ((gm >> v) & 1u) | (((pm >> v) & 1u) & G);
    const int Pall = (pm == (1u << kCCV) - 1u);
    const int allp = __syncthreads_and(Pall);
    uint32_t bg, cc0, cc1;
    block_carries2((int)G, Pall, &cc0, &cc1, &bg);          // both carry-ins before the look-back
    PA_TMARK_B(kKid, 3, 0x100000 | tile);
    const uint32_t hi_last = s_hi[kCCT - 1];               // hi32 of the tile's last sum
    // the look-back flags carry their whole payload (ready bit + C_out), so relaxed gpu-scope
    // accesses suffice: no fence orders other data behind them
    uint32_t *vs = state + 2 * kFlagStride;
    if (threadIdx.x == 0) {
        const bool indep = bg || !allp;
        const uint32_t cout_indep = hi_last + bg;
        PA_TMARK_B(kKid, 10 + (indep ? 1 : 0) + (allp ? 2 : 0) + (bg ? 4 : 0), 0x100000 | tile);
        if (indep) st_relaxed_gpu(vs + kFlagStride * tile, 0x80000000u | cout_indep);
        uint32_t cin = 0;
        if (tile > 0 && !(DBG & 2)) {
            uint32_t st;
            PA_CK(vs + kFlagStride * (tile - 1), 4);
            while (!((st = ld_relaxed_gpu(vs + kFlagStride * (tile - 1))) & 0x80000000u)) __nanosleep(32);
            cin = st & 0x7FFFFFFFu;
        }
        const uint32_t c1 = (uint32_t)(((uint64_t)w[0] + cin) >> 32);     // thread 0 owns word u0
        s_cin = cin;
        s_c1 = c1;
        PA_TMARK_B(kKid, 4, 0x100000 | tile);
        if (!indep) st_relaxed_gpu(vs + kFlagStride * tile, 0x80000000u | (hi_last + (bg | ((uint32_t)allp & c1))));
    }
    __syncthreads();
    const uint32_t cin = s_cin;
    uint32_t c = s_c1 ? cc1 : cc0;
    // LINEAR with obe: the caller wants the W words as the MSB-first bit string of the whole
    // W-word integer (m = alpha = 32 W, readings A5/A8): word u lands byte-swapped at W-1-u
    auto store = [&](uint32_t u, uint32_t val) {
        if (!RING && obe) PA_AT(obe + (W - 1 - u)) = __byte_perm(val, 0, 0x0123);
        else PA_AT(out + u) = val;
    };
#pragma unroll
    for (int v = 0; v < kCCV; v++) {
        const uint32_t u = ub + v;
        const bool first = (threadIdx.x == 0 && v == 0);
        if (first) {
            if (u < W) store(u, w[v] + cin);
            continue;
        }
        if (u < W) store(u, w[v] + c);
        c = ((gm >> v) & 1u) | (((pm >> v) & 1u) & c);
    }
    if (RING && !(DBG & 4)) {
        // the CTA barrier orders every thread's output stores before thread 0's fence, which
        // (cumulatively) publishes them before the done-counter increment
        // acq_rel atomic (cumulative release of what bar.sync made thread 0 observe; acquire
        // for the last CTA) instead of a full sequentially-consistent fence per CTA
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t ntiles = (W + kCCTile - 1) / kCCTile;
            uint32_t old;
            PA_CK(state + kFlagStride, 4);
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(state + kFlagStride) : "memory");
            s_last = (old == ntiles - 1);
        }
        __syncthreads();
        if (s_last) {
            __threadfence();                                  // one CTA: acquire for every thread
            mersenne_finish_dev(out, Wfin, gamma);
            PA_TMARK_B(kKid, 6, 0x100000 | tile);
        }
    }
    PA_TMARK_B(kKid, 5, 0x100000 | tile);
}

// ---------------------------------------------------------------- MH output
// out word q (4 bytes, big-endian) = bits [alpha - 32(q+1), alpha - 32q) of Z, i.e. the
// next 32 output bits MSB-first (reading A5); bits beyond m are zero.
__global__ void mh_extract(const uint32_t *__restrict__ Z, uint64_t nwz, uint64_t alpha, uint64_t m,
                           uint8_t *__restrict__ out, uint64_t nbytes) {
    const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (4 * q >= nbytes) return;
    const int64_t lowb = (int64_t)alpha - 32 * (int64_t)(q + 1);   // Z bit of the word's LSB
    uint32_t v;
    auto zw = [&](int64_t wi) -> uint32_t { return (wi >= 0 && (uint64_t)wi < nwz) ? PA_AT(Z + wi) : 0u; };
    if (lowb >= 0) {
        const int64_t wi = lowb >> 5;
        v = __funnelshift_r(zw(wi), zw(wi + 1), (int)(lowb & 31));
    } else {
        v = zw(0) << (-lowb);
    }
    const int64_t valid = (int64_t)m - 32 * (int64_t)q;              // output bits present here
    if (valid < 32) v &= valid <= 0 ? 0u : ~((1u << (32 - valid)) - 1u);
    const uint32_t be = __byte_perm(v, 0, 0x0123);
    if (4 * q + 4 <= nbytes && !(reinterpret_cast<uintptr_t>(out) & 3)) {
        PA_AT(reinterpret_cast<uint32_t *>(out) + q) = be;                 // coalesced word store
        return;
    }
#pragma unroll
    for (int b = 0; b < 4; b++)
        if (4 * q + b < nbytes) PA_AT(out + 4 * q + b) = (uint8_t)(be >> (8 * b));
}

}  // namespace pa
