// Number-theoretic transforms of length L = N1 * N2 modulo 30-bit primes (sm_100a).
//
// Role in the method: the MMH products a_i * x_i (Eq. 2) and the MH
// product b * y (Eq. 4) are exact big-integer multiplications: "its main
// part is large number multiplications, which means it can be accelerated by
// algorithms such as the Schonhage and Strassen algorithm".  Each
// product is a cyclic convolution of B-bit limb vectors computed with NTTs; the MMH
// sum over blocks is accumulated in the transform domain so that one inverse
// transform serves all blocks.
//
// Four-step structure (no explicit transposes, no bit reversal):
//   column pass: for each column j1 < N1, an N2-point DFT over j2 of x[j1 + N1 j2],
//                times omega_L^(j1 k2), stored at j1 + N1 k2;
//   row pass:    for each row k2, an N1-point DFT of the contiguous row; the result
//                X[k2 + N2 k1] is stored at k2 N1 + k1.
// The inverse runs row pass (omega^-1, then times omega_L^(-j1 k2)) and column pass
// (omega^-1) and lands in natural order; 1/L is folded into the precomputed operand.
// Each pass is a sub-DFT of S = 2^S_LOG points: a thread holds E = 2^E_LOG elements
// in registers and runs radix-2^r DIF networks (Shoup butterflies), with one shared
// memory exchange and one twiddle multiply per additional round.  The sub-DFT maps
// natural order to natural order (positions g + G l).
#pragma once
#include <cstdint>
#include "modarith.cuh"

namespace pa {

constexpr int kMaxRounds = 4;

struct NttArgs {
    const PrimeK *pk;          // [P]
    const uint32_t *regtw;     // [P][E/2] omega_E^j of this direction
    const uint32_t *regtwp;    // [P][E/2] Shoup companions
    uint32_t regtw_stride;     // E/2 entries per prime in the table (allocated for E=32)
    // the same omega_32^j Shoup pairs by value: kernel parameters live in the constant bank,
    // so a warp-uniform prime index reads them as uniform constant loads (no per-thread
    // registers or global loads for the in-register DFT twiddles)
    uint32_t ctw[kMaxPrimes][16];
    uint32_t ctwp[kMaxPrimes][16];
    const uint32_t *rtw;       // round twiddles, Shoup pairs (w, floor(w 2^32/p)): [P][rtw_stride]
    uint32_t rtw_stride;
    uint32_t rtw_off[kMaxRounds];
    uint32_t rtw_off4[kMaxRounds];   // the same pass's offsets for 16-element threads (E_LOG = 4)
    const uint32_t *ltw_lo;    // omega_L^(+-e_lo), e_lo < 2^h   (Montgomery form)
    const uint32_t *ltw_hi;    // omega_L^(+-e_hi 2^h)
    uint32_t ltw_lo_stride, ltw_hi_stride, ltw_h;
    uint32_t log2L;
    uint32_t n1;               // row length (number of columns)
    uint32_t n2;               // column length (number of rows)
    uint32_t nprimes;
};

template <int S_LOG, int E_LOG>
struct SubPlan {
    static constexpr int S = 1 << S_LOG;
    static constexpr int E = 1 << E_LOG;
    static constexpr int Q = (S_LOG + E_LOG - 1) / E_LOG;     // radix rounds
    static constexpr int TPV = S / E;                          // threads per vector
    __host__ __device__ static constexpr int rlog(int rho) { return (rho < Q - 1) ? E_LOG : (S_LOG - E_LOG * (Q - 1)); }
    __host__ __device__ static constexpr int glog(int rho) { return rho == 0 ? 0 : glog(rho - 1) + rlog(rho - 1); }
};

template <int R>
__host__ __device__ constexpr int bitrev(int q) {
    int r = 0;
    for (int b = 1; b < R; b <<= 1) { r = (r << 1) | (q & 1); q >>= 1; }
    return r;
}

// In-register DIF DFT of radix R = 2^RLOG on x[0..R): natural order in, X[bitrev(q)]
// in x[q] out.  tw[j] = omega_E^j, twp[j] its Shoup companion (j < E/2).
// ZH: the upper half x[R/2..R) is known to be zero (a column whose non-zero rows all lie in
// the first half): the first stage is then (a, a w), no sums or differences.
// LAZY: the last stage's outputs are left in [0, 4p) (no final reductions) -- for callers
// whose next step is a Montgomery multiply, which takes any 32-bit operand.  LAZY0: the
// same except output 0, the one inter-round output that is not twiddled (k = bitrev(0) = 0).
template <int RLOG, int E, bool ZH = false, bool LAZY = false, bool LAZY0 = false>
__device__ __forceinline__ void dft_reg(uint32_t *x, const uint32_t *tw, const uint32_t *twp,
                                        uint32_t p, uint32_t p2) {
    constexpr int R = 1 << RLOG;
#pragma unroll
    for (int h = R / 2; h >= 1; h >>= 1) {
#pragma unroll
        for (int s = 0; s < R; s += 2 * h) {
#pragma unroll
            for (int i = 0; i < h; i++) {
                if (ZH && h == R / 2) {
                    const int j = i * (E / (2 * h));
                    x[s + i + h] = (i == 0) ? x[s + i] : mul_shoup(x[s + i], tw[j], twp[j], p);
                } else if (i == 0) {
                    if ((LAZY || LAZY0) && h == 1) {
                        const uint32_t u = x[s], w = x[s + 1];
                        x[s] = (LAZY0 && !LAZY && s == 0) ? red2p(u + w, p2) : u + w;   // < 4p
                        x[s + 1] = u - w + p2;                                          // < 4p
                    } else {
                        bfly_dif1(x[s], x[s + h], p2);
                    }
                } else {
                    const int j = i * (E / (2 * h));
                    bfly_dif(x[s + i], x[s + i + h], tw[j], twp[j], p, p2);
                }
            }
        }
    }
}

// omega_L^e (direction of the tables) in Montgomery form, canonical (< p).
__device__ __forceinline__ uint32_t ltw_mont(const NttArgs &a, int pi, uint32_t e, uint32_t p,
                                             uint32_t pinv) {
    const uint32_t lo = PA_LDG(a.ltw_lo + (size_t)pi * a.ltw_lo_stride + (e & ((1u << a.ltw_h) - 1)));
    const uint32_t hi = PA_LDG(a.ltw_hi + (size_t)pi * a.ltw_hi_stride + (e >> a.ltw_h));
    return red1p(mul_mont(lo, hi, p, pinv), p);
}

struct Ctx32 {  // per-prime constants held in registers by a thread
    uint32_t p, p2, pinv;
};

#ifndef PA_CTW
#define PA_CTW 1
#endif
// omega_E^j (j < E/2) of prime pi for an in-register radix-E DFT (E <= 32)
template <int E>
__device__ __forceinline__ void load_regtw(const NttArgs &a, uint32_t pi, uint32_t *tw, uint32_t *twp) {
#pragma unroll
    for (int j = 0; j < E / 2; j++) {
#if PA_CTW
        tw[j] = a.ctw[pi][j * (32 / E)];
        twp[j] = a.ctwp[pi][j * (32 / E)];
#else
        tw[j] = PA_LDG(a.regtw + pi * a.regtw_stride + j * (32 / E));
        twp[j] = PA_LDG(a.regtwp + pi * a.regtw_stride + j * (32 / E));
#endif
    }
}

// Round rho >= 1 of a sub-DFT (recursive over rho).  Round rho-1 left its outputs in
// shared memory; the last round leaves its outputs in x[] (group h, register mm <->
// position v + TPV h + G_last * bitrev(mm)), in [0, 2p), or [0, 4p) with LAZY.
template <int S_LOG, int E_LOG, int RHO, bool LAZY = false, class SIdx>
__device__ __forceinline__ void rounds_rest(uint32_t *x, uint32_t *sm, const SIdx &sidx, int v,
                                            const uint32_t *tw, const uint32_t *twp,
                                            const uint32_t *rtw_p, const NttArgs &a,
                                            const Ctx32 &c) {
    using SP = SubPlan<S_LOG, E_LOG>;
    if constexpr (RHO < SP::Q) {
        constexpr int S = SP::S, E = SP::E;
        constexpr int RL = SP::rlog(RHO);
        constexpr int R = 1 << RL;
        constexpr int G = 1 << SP::glog(RHO);
        constexpr int T = S / (G * R);
        constexpr int NG = E / R;
        __syncthreads();
#pragma unroll
        for (int h = 0; h < NG; h++) {
            const int q = v + SP::TPV * h;
#pragma unroll
            for (int m = 0; m < R; m++) { PA_SMEM_PTR_CK(sm + sidx(q + (S / R) * m), 4); x[h * R + m] = sm[sidx(q + (S / R) * m)]; }
        }
#pragma unroll
        for (int h = 0; h < NG; h++)
            dft_reg<RL, E, false, LAZY && RHO == SP::Q - 1, (RHO < SP::Q - 1) && (T > 1)>(x + h * R, tw, twp, c.p, c.p2);
        if constexpr (RHO < SP::Q - 1) {
            __syncthreads();
#pragma unroll
            for (int h = 0; h < NG; h++) {
                const int q = v + SP::TPV * h;
                const int g = q % G, t = q / G;
#pragma unroll
                for (int mm = 0; mm < R; mm++) {
                    const int k = bitrev<R>(mm);
                    uint32_t val = x[h * R + mm];
                    if (T > 1 && k != 0) {
                        const uint2 w = PA_LDG(reinterpret_cast<const uint2 *>(rtw_p + a.rtw_off[RHO]) + k * T + t);
                        val = mul_shoup(val, w.x, w.y, c.p);
                    }
                    PA_SMEM_PTR_CK(sm + sidx(g + G * k + G * R * t), 4);
                    sm[sidx(g + G * k + G * R * t)] = val;
                }
            }
        }
        rounds_rest<S_LOG, E_LOG, RHO + 1, LAZY>(x, sm, sidx, v, tw, twp, rtw_p, a, c);
    }
}

// Round 0 post-processing: DFT of the loaded groups, twiddle, store to shared memory.
template <int S_LOG, int E_LOG, bool ZH = false, class SIdx>
__device__ __forceinline__ void round0_finish(uint32_t *x, uint32_t *sm, const SIdx &sidx, int v,
                                              const uint32_t *tw, const uint32_t *twp,
                                              const uint32_t *rtw_p, const NttArgs &a,
                                              const Ctx32 &c) {
    using SP = SubPlan<S_LOG, E_LOG>;
    constexpr int S = SP::S, E = SP::E;
    constexpr int RL = SP::rlog(0);
    constexpr int R = 1 << RL;
    constexpr int T = S / R;
    constexpr int NG = E / R;
    // with a further round, every output but k = 0 is twiddled next (Montgomery): LAZY0
#pragma unroll
    for (int h = 0; h < NG; h++) dft_reg<RL, E, ZH, false, (SP::Q > 1) && (T > 1)>(x + h * R, tw, twp, c.p, c.p2);
    if constexpr (SP::Q > 1) {
#pragma unroll
        for (int h = 0; h < NG; h++) {
            const int t = v + SP::TPV * h;
#pragma unroll
            for (int mm = 0; mm < R; mm++) {
                const int k = bitrev<R>(mm);
                uint32_t val = x[h * R + mm];
                if (T > 1 && k != 0) {
#if defined(PA_COL_DBG) && (PA_COL_DBG & 2)
                    const uint2 w = make_uint2(k * 7u + t, k * 11u + t);   // timing-only ablation
#else
                    const uint2 w = PA_LDG(reinterpret_cast<const uint2 *>(rtw_p + a.rtw_off[0]) + k * T + t);
#endif
                    val = mul_shoup(val, w.x, w.y, c.p);
                }
                PA_SMEM_PTR_CK(sm + sidx(k + R * t), 4);
                sm[sidx(k + R * t)] = val;
            }
        }
    }
}

// Position of register (h, mm) after the last round.
template <int S_LOG, int E_LOG>
__device__ __forceinline__ int out_pos(int v, int h, int mm) {
    using SP = SubPlan<S_LOG, E_LOG>;
    constexpr int RL = SP::rlog(SP::Q - 1);
    constexpr int R = 1 << RL;
    constexpr int G = 1 << SP::glog(SP::Q - 1);
    return (v + SP::TPV * h) + G * bitrev<R>(mm);
}

// Position of register (h, m) in round 0 (input order).
template <int S_LOG, int E_LOG>
__device__ __forceinline__ int in_pos(int v, int h, int m) {
    using SP = SubPlan<S_LOG, E_LOG>;
    constexpr int R = 1 << SP::rlog(0);
    return (v + SP::TPV * h) + (SP::S / R) * m;
}

}  // namespace pa
