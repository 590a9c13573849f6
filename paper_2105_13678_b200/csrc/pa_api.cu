// C ABI of the MMH-MH privacy-amplification library (include/pa.h): parameter
// validation, transform planning, hash-key expansion, context lifecycle and the
// stream-ordered orchestration of the sm_100a kernels of one hash.
//
// Hot path of one pa_hash (Algorithm 1), all on the ctx stream:
//   S1     pack_key_residues  key blocks -> B-bit limbs -> residues mod P primes
//   S2     col_pass<FWD>   first (column) NTT pass, four-step twiddle
//   S2+S3  row_mac         second NTT pass, multiply by the precomputed transforms of
//                          the a_i and accumulate over blocks (bulk-copy pipeline)
//   S4     row_pass<INV>, col_pass<INV>   one inverse transform for all blocks
//          crt_coeffs (exact coefficients) + crt_carry (column sums on the gamma-bit
//          ring, carries with look-back)                  exact Y = sum_i a_i x_i
//   S5     inside crt_carry: ring fold per coefficient, last CTA: residual fold and
//          canonical zero                                 -> y = Y mod p
//   S7     pack(y), col_pass, row_mac(B^), inverse, crt_coeffs + crt_carry (+c, linear),
//          mh_extract -> out_bits = top m bits of (b y + c) mod 2^alpha
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/pa.h"
#include "carry.cuh"
#include "host_math.h"
#include "modarith.cuh"
#include "ntt.cuh"
#include "passes.cuh"
#include "rekey.cuh"
#include "toeplitz.cuh"
#include "exchange.cuh"
#include "nccl_dl.h"

using namespace pa;

// ====================================================================== errors
static thread_local int g_err = 0;
static thread_local char g_msg[512];

static int set_err(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
static int set_err(int code, const char *fmt, ...) {
    g_err = code;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_msg, sizeof g_msg, fmt, ap);
    va_end(ap);
    return code;
}

#define CUDA_TRY(expr)                                                                      \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            return set_err(PA_E_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                           __FILE__, __LINE__);                                             \
    } while (0)

#define NCCL_TRY(expr)                                                                      \
    do {                                                                                    \
        const ncclResult_t r_ = (expr);                                                     \
        if (r_ != ncclSuccess)                                                              \
            return set_err(PA_E_NCCL, "%s: %s", #expr, pa::nccl_api().GetErrorString(r_));  \
    } while (0)

#define TRY(expr)                      \
    do {                               \
        int _rc = (expr);              \
        if (_rc != PA_OK) return _rc;  \
    } while (0)

extern "C" int pa_last_error(char *buf, size_t len) {
    if (buf && len) {
        strncpy(buf, g_msg, len - 1);
        buf[len - 1] = 0;
    }
    return g_err;
}

// ====================================================================== debug build
// PA_DEBUG (debug.cuh): the device-side table of valid global ranges -- every allocation of
// every context on the device, plus the caller's buffers of the current call.  Uploaded
// (after a device synchronize) whenever it changes; graphs are off in this build.
#ifdef PA_DEBUG
#include <mutex>
namespace {
struct DbgDev {
    std::vector<pa::DbgRange> perm, user;
};
std::mutex g_dbg_mu;
std::map<int, DbgDev> g_dbg_dev;
void dbg_upload_locked(int dev) {
    DbgDev &d = g_dbg_dev[dev];
    std::vector<pa::DbgRange> all = d.perm;
    for (const auto &r : d.user) if (all.size() < (size_t)pa::kDbgMaxRanges) all.push_back(r);
    if (all.size() > (size_t)pa::kDbgMaxRanges) all.resize(pa::kDbgMaxRanges);
    const uint32_t n = (uint32_t)all.size();
    cudaDeviceSynchronize();
    if (n) cudaMemcpyToSymbol(pa::g_dbg_ranges, all.data(), n * sizeof(pa::DbgRange));
    cudaMemcpyToSymbol(pa::g_dbg_n, &n, sizeof n);
}
}  // namespace
static void dbg_add(const void *p, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_dbg_mu);
    g_dbg_dev[dev].perm.push_back({(uint64_t)p, (uint64_t)p + bytes});
    dbg_upload_locked(dev);
}
static void dbg_remove(const void *p) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_dbg_mu);
    auto &v = g_dbg_dev[dev].perm;
    for (size_t i = 0; i < v.size(); i++)
        if (v[i].lo == (uint64_t)p) { v.erase(v.begin() + i); break; }
    dbg_upload_locked(dev);
}
// the caller's buffers of this call (replaces those of the previous call)
static void dbg_user(std::initializer_list<std::pair<const void *, uint64_t>> bufs) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_dbg_mu);
    auto &u = g_dbg_dev[dev].user;
    u.clear();
    for (const auto &b : bufs)
        if (b.first && b.second) u.push_back({(uint64_t)b.first, (uint64_t)b.first + b.second});
    dbg_upload_locked(dev);
}
static void dbg_user_add(const void *p, uint64_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_dbg_mu);
    if (p && bytes) g_dbg_dev[dev].user.push_back({(uint64_t)p, (uint64_t)p + bytes});
    dbg_upload_locked(dev);
}
#else
static inline void dbg_add(const void *, size_t) {}
static inline void dbg_remove(const void *) {}
static inline void dbg_user(std::initializer_list<std::pair<const void *, uint64_t>>) {}
static inline void dbg_user_add(const void *, uint64_t) {}
#endif

// ====================================================================== planning
static constexpr int kMinLog2L = 10;
static constexpr int kMaxLog2L = 23;
static constexpr int kColMaxLog = 8;      // column pass length cap (2^9 only when the row would exceed 2^14)
static uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
static constexpr int kMaxRowLog = 14;
static constexpr int kMaxLimbBits = 256;

static double log2_bound(uint64_t nterms, uint64_t overlap, uint32_t B) {
    // log2(nterms * overlap * (2^B - 1)^2)  (upper bound of a convolution coefficient)
    return std::log2((double)nterms) + std::log2((double)overlap) + 2.0 * std::log2(std::ldexp(1.0, (int)B) - 1.0);
}

// Choose (B, P, L) for the product of an `abits`-bit and a `bbits`-bit operand, summed
// over `nterms` products; only coefficients below `need_coef` limbs... (all are needed:
// the cyclic length must cover the full product so nothing wraps).
// nvec: vectors transformed per hash (blocks for MMH, 1 for MH).  A single vector gets a
// short column (many column groups, many row units) so the passes fill the GPU.
static int plan_product(uint64_t abits, uint64_t bbits, uint64_t nterms, int force_B, uint64_t nvec,
                        pa_stage_plan *out) {
    // B <= 56: one 64-bit limb (limb_redc); larger B: multiword limbs (<= 8 words)
    double best = 1e300;
    pa_stage_plan bp{};
    for (uint32_t B = 16; B <= (uint32_t)kMaxLimbBits; B += 8) {
        if (force_B && (int)B != force_B) continue;
        const uint64_t wa = (abits + B - 1) / B, wb = (bbits + B - 1) / B;
        const uint64_t len = wa + wb - 1;
        int lg = kMinLog2L;
        while ((1ull << lg) < len) lg++;
        if (lg > kMaxLog2L) continue;
        const double bound = log2_bound(nterms, std::min(wa, wb), B);
        // primes usable at this length, largest first
        std::vector<uint32_t> ps;
        for (uint32_t p : kPrimes) if (two_adic(p) >= lg) ps.push_back(p);
        double mod = 0;
        uint32_t P = 0;
        while (P < ps.size() && P < (uint32_t)kMaxPrimes && mod <= bound + 0.5) { mod += std::log2((double)ps[P]); P++; }
        if (mod <= bound + 0.5) continue;                   // not enough primes
        const double cost = (double)P * std::ldexp(1.0, lg) * (lg + 2);
        if (cost < best) {
            best = cost;
            bp = pa_stage_plan{};
            bp.limb_bits = B;
            bp.nprimes = P;
            bp.log2_len = (uint32_t)lg;
            // 2^8-point columns at most unless the row would exceed 2^14: the 512-thread
            // 2^9 column pass runs one CTA per SM (C5c 2.34 -> 2.18 ms, P1 412 -> 399 us at 2^8);
            // single-vector stages (MH) likewise (C4 MH 2^8 x 2^10 353.7 us, 2^7 x 2^11 359.5 us)
            const int cl = std::max(std::min(kColMaxLog, lg / 2), lg - kMaxRowLog);
            bp.n_col = 1u << cl;
            bp.n_row = 1u << (lg - cl);
            for (uint32_t i = 0; i < P; i++) bp.primes[i] = ps[i];
            bp.bound_log2 = bound;
            bp.modulus_log2 = mod;
        }
    }
    if (best == 1e300) return PA_E_BOUND;
    *out = bp;
    return PA_OK;
}

struct Plan {
    uint64_t n, r, m, gamma, alpha, k, b0, b1, seed;
    uint64_t paper_k;        // paper mode (gamma-bit blocks, reload rule) when nonzero
    uint64_t mh_only;        // comparator: MH-only PA over the whole n-bit key
    uint64_t toeplitz;       // comparator: Toeplitz-hashing PA (tz_nb input, tz_no output blocks of r bits)
    uint64_t tz_nb, tz_no;
    uint32_t tz_group = 0;   // input blocks per accumulation (counts below the prime)
    int strict, force_B;
    int world, rank;         // multi-GPU context (world >= 1): NCCL rank of a world-rank job
    pa_stage_plan mmh, mh;
};

static bool is_mersenne(uint64_t g) {
    for (uint64_t e : kMersenne) if (e == g) return true;
    return false;
}

static int make_plan(const pa_params *prm, Plan *P) {
    if (!prm) return set_err(PA_E_PARAM, "params is NULL");
    Plan p{};
    p.n = prm->n; p.r = prm->r; p.m = prm->m; p.seed = prm->seed;
    p.strict = prm->strict; p.force_B = prm->limb_bits;
    p.paper_k = prm->paper_k;
    p.mh_only = prm->mh_only;
    p.toeplitz = prm->toeplitz;
    p.world = prm->world;
    p.rank = prm->rank;
    if (p.n < 1) return set_err(PA_E_PARAM, "n must be >= 1");
    if (p.world < 0 || (p.world > 0 && (p.rank < 0 || p.rank >= p.world)) || (p.world == 0 && p.rank != 0))
        return set_err(PA_E_PARAM, "multi-GPU: need 0 <= rank < world (got rank %d, world %d)", p.rank, p.world);
    if (p.world > 0 && (p.paper_k || p.mh_only || p.toeplitz))
        return set_err(PA_E_PARAM, "multi-GPU contexts hash in r-bit mode (no paper_k, mh_only or toeplitz)");
    if (prm->p2p && (p.world < 1 || p.world > kMaxWorld))
        return set_err(PA_E_PARAM, "p2p needs a multi-GPU context with 1 <= world <= %d", kMaxWorld);
    if (p.m < 1) return set_err(PA_E_PARAM, "m must be >= 1");
    if (p.toeplitz) {
        // comparator: Toeplitz-hashing PA, r x r blocks, one prime
        if (prm->gamma || prm->r || p.paper_k || p.mh_only || prm->block_begin || prm->block_end)
            return set_err(PA_E_PARAM, "Toeplitz PA takes no gamma, r, paper_k, mh_only or shard");
        if (p.m >= (1ull << 31)) return set_err(PA_E_PARAM, "Toeplitz PA: m < 2^31");
        const uint64_t big = std::max(p.n, p.m);
        int lr = 9;
        while (lr < 22 && (1ull << lr) < big) lr++;
        if (prm->limb_bits) {               // forced block size r = 2^limb_bits (tests, tuning)
            if (prm->limb_bits < 9 || prm->limb_bits > 22) return set_err(PA_E_PARAM, "Toeplitz: limb_bits = log2 r in [9, 22]");
            lr = prm->limb_bits;
        }
        const int lg = lr + 1;
        p.r = 1ull << lr;
        p.tz_nb = cdiv(p.n, p.r);
        p.tz_no = cdiv(p.m, p.r);
        p.k = p.tz_nb;
        p.alpha = p.tz_no;
        p.gamma = 0;
        p.b0 = 0; p.b1 = p.k;
        uint32_t prime = 0;
        // a prime above n keeps every count exact in one accumulation; else the largest prime
        // of the transform length, and the input blocks are summed in groups of
        // floor((prime - 1) / r) blocks whose counts stay below it (parities XORed)
        for (uint32_t q : kPrimes) if (two_adic(q) >= lg && q > p.n) { prime = q; break; }
        if (!prime)
            for (uint32_t q : kPrimes) if (two_adic(q) >= lg && q > p.r && q > prime) prime = q;
        if (!prime) return set_err(PA_E_BOUND, "no NTT prime for Toeplitz length 2^%d", lg);
        p.tz_group = (uint32_t)std::min<uint64_t>((prime - 1) / p.r, p.tz_nb);
        if (prm->tz_group_blocks) p.tz_group = (uint32_t)std::min<uint64_t>(prm->tz_group_blocks, p.tz_group);
        pa_stage_plan &sp = p.mmh;
        sp = pa_stage_plan{};
        sp.limb_bits = 1;
        sp.nprimes = 1;
        sp.log2_len = (uint32_t)lg;
        const int cl = std::max(std::min(kColMaxLog, lg / 2), lg - kMaxRowLog);
        sp.n_col = 1u << cl;
        sp.n_row = 1u << (lg - cl);
        sp.primes[0] = prime;
        sp.bound_log2 = std::log2((double)p.n);
        sp.modulus_log2 = std::log2((double)prime);
        *P = p;
        return PA_OK;
    }
    if (p.force_B && (p.force_B < 16 || p.force_B > kMaxLimbBits || p.force_B % 8))
        return set_err(PA_E_PARAM, "limb_bits must be a multiple of 8 in [16, %d]", kMaxLimbBits);
    uint64_t g = prm->gamma;
    if (p.mh_only) {
        // comparator: z = top m bits of (b x + c) mod 2^n
        if (prm->gamma || prm->r || p.paper_k || prm->block_begin || prm->block_end)
            return set_err(PA_E_PARAM, "MH-only PA takes no gamma, r, paper_k or shard");
        if (p.m > p.n) return set_err(PA_E_PARAM, "MH-only PA: m must be <= n (SPEC.md:309)");
        if (p.n > (1ull << 31)) return set_err(PA_E_PARAM, "MH-only PA: n <= 2^31");
        p.gamma = p.n;                  // width of the MH operand y (= x)
        p.alpha = p.n;
        p.r = p.n;
        p.k = 0;
        p.b0 = p.b1 = 0;
        if (plan_product(p.n, p.n, 1, p.force_B, 1, &p.mh) != PA_OK)
            return set_err(PA_E_BOUND, "no transform plan covers the MH-only product");
        *P = p;
        return PA_OK;
    }
    if (p.paper_k) {
        // paper mode: Algorithm 1 as written, gamma-bit blocks
        if (!g) return set_err(PA_E_PARAM, "paper mode needs an explicit gamma (p = 2^gamma - 1)");
        if (!is_mersenne(g)) return set_err(PA_E_PARAM, "gamma=%llu is not a known Mersenne exponent (SPEC.md:33)", (unsigned long long)g);
        if (p.m >= g) return set_err(PA_E_PARAM, "paper mode: m must be < gamma (PAPER.md:143)");
        if (p.paper_k > p.n / g) return set_err(PA_E_PARAM, "paper mode: n must be >= paper_k * gamma (n = gamma k, PAPER.md:282)");
        if (prm->block_begin || prm->block_end) return set_err(PA_E_PARAM, "paper mode is not available for shard contexts");
        p.gamma = g;
        p.r = g;
        p.alpha = g;
        p.k = p.paper_k;
        p.b0 = 0; p.b1 = p.k;
        if (plan_product(g, g, p.k, p.force_B, p.k, &p.mmh) != PA_OK)
            return set_err(PA_E_BOUND, "no transform plan covers the MMH coefficient bound");
        if (plan_product(g, g, 1, p.force_B, 1, &p.mh) != PA_OK)
            return set_err(PA_E_BOUND, "no transform plan covers the MH product");
        *P = p;
        return PA_OK;
    }
    if (p.r < 16 || p.r % 16) return set_err(PA_E_PARAM, "r must be >= 16 and a multiple of 16 (got %llu)", (unsigned long long)p.r);
    if (g == 0) {
        for (uint64_t e : kMersenne) if (e > p.r) { g = e; break; }
        if (g == 0) return set_err(PA_E_PARAM, "no known Mersenne exponent > r");
    }
    if (!is_mersenne(g)) return set_err(PA_E_PARAM, "gamma=%llu is not a known Mersenne exponent (SPEC.md:33)", (unsigned long long)g);
    if (g <= p.r) return set_err(PA_E_PARAM, "gamma must exceed r so every r-bit block lies in Z_p (reading A2)");
    if (p.strict && p.m >= g) return set_err(PA_E_PARAM, "strict: m must be < gamma (PAPER.md:143)");
    p.gamma = g;
    p.alpha = std::max<uint64_t>(g, p.m);
    p.k = (p.n + p.r - 1) / p.r;
    p.b0 = prm->block_begin; p.b1 = prm->block_end;
    if (p.world > 0) {
        // rank g owns blocks [floor(k g / G), floor(k (g+1) / G))
        if ((uint64_t)p.world > p.k) return set_err(PA_E_PARAM, "multi-GPU: world %d > k = %llu blocks", p.world, (unsigned long long)p.k);
        const uint64_t s0 = p.k * (uint64_t)p.rank / (uint64_t)p.world, s1 = p.k * (uint64_t)(p.rank + 1) / (uint64_t)p.world;
        if ((p.b0 || p.b1) && (p.b0 != s0 || p.b1 != s1))
            return set_err(PA_E_PARAM, "multi-GPU: block range must be 0 or [%llu, %llu) for rank %d of %d",
                           (unsigned long long)s0, (unsigned long long)s1, p.rank, p.world);
        p.b0 = s0; p.b1 = s1;
    }
    if (p.b0 == 0 && p.b1 == 0) p.b1 = p.k;
    if (p.b0 >= p.b1 || p.b1 > p.k) return set_err(PA_E_PARAM, "bad shard [%llu, %llu) of %llu blocks",
                                                  (unsigned long long)p.b0, (unsigned long long)p.b1, (unsigned long long)p.k);
    // every shard plans the transform of the whole key (all k blocks in the coefficient bound,
    // the whole key's split): the transform-domain accumulators of the shards are then
    // compatible and their sum is the whole key's (pa_mmh_acc, multi-GPU reduce)
    if (plan_product(p.r, p.gamma, p.k, p.force_B, p.k, &p.mmh) != PA_OK)
        return set_err(PA_E_BOUND, "no transform plan covers the MMH coefficient bound");
    if (plan_product(p.gamma, p.alpha, 1, p.force_B, 1, &p.mh) != PA_OK)
        return set_err(PA_E_BOUND, "no transform plan covers the MH product");
    *P = p;
    return PA_OK;
}

// ====================================================================== stage tables
struct StageDev {
    pa_stage_plan pl{};
    uint32_t L = 0, lg = 0;
    PrimeK *pk = nullptr;
    PrimeSet pks{};                     // host copy, passed by value to the pack kernels
    uint32_t *scale = nullptr;
    uint32_t *regtw[2] = {}, *regtwp[2] = {};
    uint32_t ctw[2][kMaxPrimes][16] = {}, ctwp[2][kMaxPrimes][16] = {};   // host copies (NttArgs by value)
    uint32_t *rtw = nullptr;            // [P][stride]: col fwd, col inv, row fwd, row inv
    uint32_t rtw_stride = 0;
    uint32_t rtw_off[2][4][kMaxRounds] = {};   // [E_LOG - 4][col fwd, col inv, row fwd, row inv]
    uint32_t *ltw_lo[2] = {}, *ltw_hi[2] = {};
    uint32_t ltw_h = 0, ltw_lo_n = 0, ltw_hi_n = 0;
    uint2 *tw4f = nullptr;              // omega_L^(j1 k2) at k2 N1 + j1, [P][L] Shoup pairs (forward)
    uint32_t *tw4i = nullptr;           // omega_L^(-j1 k2), [P][L] Montgomery form (inverse)
    CrtK crt{};
};

// Device memory of a context: the caller's allocator (pa_params.dev_alloc / dev_free, e.g.
// PyTorch's caching allocator) or the stream-ordered cudaMallocAsync / cudaFreeAsync on the
// context stream (the device's default memory pool).
struct DevAlloc {
    struct Blk {
        void *p;
        size_t bytes;
    };
    std::vector<Blk> blks;
    uint64_t bytes = 0;
    cudaStream_t stream = nullptr;
    void *(*fn_alloc)(size_t, void *, void *) = nullptr;
    void (*fn_free)(void *, size_t, void *, void *) = nullptr;
    void *user = nullptr;
    template <class T>
    int alloc(T **p, size_t count) {
        void *q = nullptr;
        const size_t b = (std::max<size_t>(count * sizeof(T), 16) + 255) & ~(size_t)255;
        if (fn_alloc) {
            q = fn_alloc(b, (void *)stream, user);
            if (!q) return set_err(PA_E_NOMEM, "dev_alloc(%zu) returned NULL", b);
            if ((uintptr_t)q & 15) {
                if (fn_free) fn_free(q, b, (void *)stream, user);
                return set_err(PA_E_PARAM, "dev_alloc returned a pointer that is not 16-byte aligned");
            }
        } else {
            cudaError_t e = cudaMallocAsync(&q, b, stream);
            if (e != cudaSuccess) return set_err(PA_E_NOMEM, "cudaMallocAsync(%zu) failed: %s", b, cudaGetErrorString(e));
        }
        blks.push_back({q, b});
        bytes += b;
        dbg_add(q, b);
        *p = (T *)q;
        return PA_OK;
    }
    void free_all() {
        for (const Blk &k : blks) {
            dbg_remove(k.p);
            if (fn_alloc) {
                if (fn_free) fn_free(k.p, k.bytes, (void *)stream, user);
            } else {
                cudaFreeAsync(k.p, stream);
            }
        }
        if (!fn_alloc && !blks.empty()) cudaStreamSynchronize(stream);
        blks.clear();
        bytes = 0;
    }
};

// Round twiddles of a sub-DFT of 2^S_LOG points with radix 2^5 rounds: for round rho,
// table[k][t] = omega_{S_rho}^(t k), S_rho = S / G_rho.
static void round_tables(uint32_t p, uint32_t wL, int lg, int slog, int E_LOG, std::vector<uint32_t> &tab,
                         uint32_t off[kMaxRounds]) {
    const int Q = (slog + E_LOG - 1) / E_LOG;
    int glog = 0;
    for (int rho = 0; rho < kMaxRounds; rho++) off[rho] = 0;
    for (int rho = 0; rho < Q; rho++) {
        const int rl = (rho < Q - 1) ? E_LOG : slog - E_LOG * (Q - 1);
        const int srho_log = slog - glog;
        const uint32_t R = 1u << rl, T = 1u << (srho_log - rl);
        const uint32_t w = (uint32_t)powmod64(wL, 1ull << (lg - srho_log), p);   // omega_{S_rho}
        off[rho] = (uint32_t)tab.size();
        for (uint32_t k = 0; k < R; k++) {
            uint64_t wk = powmod64(w, k, p), cur = 1;
            // Shoup pairs (w, floor(w 2^32 / p)), interleaved: one 8-byte load per twiddle
            for (uint32_t t = 0; t < T; t++) {
                tab.push_back((uint32_t)cur);
                tab.push_back(shoup_of((uint32_t)cur, p));
                cur = mulmod64(cur, wk, p);
            }
        }
        glog += rl;
    }
}

// tw4[pi][k2 N1 + j1] = omega_L^(j1 k2) from the two-level Montgomery tables: as a Shoup
// pair (w canonical, floor(w 2^32 / p)) for the forward column pass (one fewer instruction per
// multiply, measured 96 -> 95 us), in Montgomery form for the inverse row pass (its 8-byte
// loads measured 2 us slower there).
template <class T>
__global__ void gen_tw4(const uint32_t *__restrict__ lo, const uint32_t *__restrict__ hi, uint32_t lo_n,
                        uint32_t hi_n, uint32_t h, const PrimeK *__restrict__ pk, uint32_t P, uint32_t lg,
                        uint32_t n1, T *__restrict__ out) {
    const uint64_t L = 1ull << lg;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < P * L; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t pi = (uint32_t)(t >> lg);
        const uint32_t pos = (uint32_t)(t & (L - 1));
        const uint32_t k2 = pos / n1, j1 = pos % n1;
        const uint32_t e = (uint32_t)(((uint64_t)j1 * k2) & (L - 1));
        const uint32_t p = pk[pi].p, pinv = pk[pi].pinv;
        const uint32_t a = lo[(size_t)pi * lo_n + (e & ((1u << h) - 1))];
        const uint32_t b = hi[(size_t)pi * hi_n + (e >> h)];
        const uint32_t wm = red1p(mul_mont(a, b, p, pinv), p);      // omega R mod p
        if constexpr (sizeof(T) == 8) {
            const uint32_t w = red1p(mul_mont(wm, 1u, p, pinv), p);  // omega
            out[t] = T{w, (uint32_t)(((uint64_t)w << 32) / p)};
        } else {
            out[t] = wm;
        }
    }
}

static int setup_stage(DevAlloc &da, const pa_stage_plan &pl, StageDev &sd, cudaStream_t st) {
    sd.pl = pl;
    sd.lg = pl.log2_len;
    sd.L = 1u << sd.lg;
    const uint32_t P = pl.nprimes;
    const int lg = (int)sd.lg;
    const int clog = __builtin_ctz(pl.n_col), rlog = __builtin_ctz(pl.n_row);
    std::vector<PrimeK> pk(P);
    std::vector<uint32_t> scale(P);
    std::vector<uint32_t> regtw[2], regtwp[2];
    std::vector<std::vector<uint32_t>> rt(P);
    sd.ltw_h = (uint32_t)((lg + 1) / 2);
    sd.ltw_lo_n = 1u << sd.ltw_h;
    sd.ltw_hi_n = 1u << (lg - sd.ltw_h);
    std::vector<uint32_t> lo[2], hi[2];
    for (uint32_t i = 0; i < P; i++) {
        const uint32_t p = pl.primes[i];
        pk[i].p = p;
        pk[i].p2 = 2 * p;
        uint32_t inv = 1;                             // p^{-1} mod 2^32 by Newton
        for (int it = 0; it < 5; it++) inv *= 2 - p * inv;
        pk[i].pinv = inv;
        pk[i].r2 = (uint32_t)powmod64(2, 64, p);
        for (int w = 0; w < 8; w++) pk[i].pw[w] = (uint32_t)powmod64(2, 32ull * w, p);
        for (int w = 0; w < 10; w++) pk[i].pw24[w] = (uint32_t)powmod64(2, 24ull * w, p);
        for (int w = 0; w < 10; w++) pk[i].pw28[w] = (uint32_t)powmod64(2, 28ull * w, p);
        const uint32_t g = primitive_root(p);
        const uint32_t wf = (uint32_t)powmod64(g, (p - 1) >> lg, p);     // omega_L
        const uint32_t wi = inv_mod(wf, p);
        const uint32_t Linv = inv_mod(sd.L, p);
        // packed operands carry 2^-32 (limb_redc); stored hat = T(a) L^-1 R^2 needs
        // mont(T(a) R^-1, L^-1 R^4)
        scale[i] = (uint32_t)mulmod64(Linv, powmod64(2, 128, p), p);
        for (int dir = 0; dir < 2; dir++) {
            const uint32_t wL = dir ? wi : wf;
            const uint32_t w32 = (uint32_t)powmod64(wL, sd.L / 32, p);
            for (int j = 0; j < 16; j++) {
                const uint32_t t = (uint32_t)powmod64(w32, j, p);
                regtw[dir].push_back(t);
                regtwp[dir].push_back(shoup_of(t, p));
                sd.ctw[dir][i][j] = t;
                sd.ctwp[dir][i][j] = shoup_of(t, p);
            }
            uint64_t cur = 1;
            for (uint32_t e = 0; e < sd.ltw_lo_n; e++) { lo[dir].push_back(to_mont((uint32_t)cur, p)); cur = mulmod64(cur, wL, p); }
            const uint64_t step = powmod64(wL, 1ull << sd.ltw_h, p);
            cur = 1;
            for (uint32_t e = 0; e < sd.ltw_hi_n; e++) { hi[dir].push_back(to_mont((uint32_t)cur, p)); cur = mulmod64(cur, step, p); }
        }
        for (int el = 4; el <= 5; el++) {
            round_tables(p, wf, lg, clog, el, rt[i], sd.rtw_off[el - 4][0]);
            round_tables(p, wi, lg, clog, el, rt[i], sd.rtw_off[el - 4][1]);
            round_tables(p, wf, lg, rlog, el, rt[i], sd.rtw_off[el - 4][2]);
            round_tables(p, wi, lg, rlog, el, rt[i], sd.rtw_off[el - 4][3]);
        }
    }
    sd.rtw_stride = (uint32_t)rt[0].size();
    std::vector<uint32_t> rtall;
    for (uint32_t i = 0; i < P; i++) rtall.insert(rtall.end(), rt[i].begin(), rt[i].end());

    TRY(da.alloc(&sd.pk, P));
    TRY(da.alloc(&sd.scale, P));
    TRY(da.alloc(&sd.rtw, rtall.size()));
    CUDA_TRY(cudaMemcpy(sd.pk, pk.data(), P * sizeof(PrimeK), cudaMemcpyHostToDevice));
    for (uint32_t i = 0; i < P; i++) sd.pks.k[i] = pk[i];
    CUDA_TRY(cudaMemcpy(sd.scale, scale.data(), P * 4, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(sd.rtw, rtall.data(), rtall.size() * 4, cudaMemcpyHostToDevice));
    for (int dir = 0; dir < 2; dir++) {
        TRY(da.alloc(&sd.regtw[dir], regtw[dir].size()));
        TRY(da.alloc(&sd.regtwp[dir], regtwp[dir].size()));
        TRY(da.alloc(&sd.ltw_lo[dir], lo[dir].size()));
        TRY(da.alloc(&sd.ltw_hi[dir], hi[dir].size()));
        CUDA_TRY(cudaMemcpy(sd.regtw[dir], regtw[dir].data(), regtw[dir].size() * 4, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(sd.regtwp[dir], regtwp[dir].data(), regtwp[dir].size() * 4, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(sd.ltw_lo[dir], lo[dir].data(), lo[dir].size() * 4, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(sd.ltw_hi[dir], hi[dir].data(), hi[dir].size() * 4, cudaMemcpyHostToDevice));
        if (dir == 0) {
            TRY(da.alloc(&sd.tw4f, (size_t)P * sd.L));
            gen_tw4<uint2><<<1024, 256, 0, st>>>(sd.ltw_lo[dir], sd.ltw_hi[dir], sd.ltw_lo_n, sd.ltw_hi_n, sd.ltw_h,
                                                 sd.pk, P, sd.lg, pl.n_row, sd.tw4f);
        } else {
            TRY(da.alloc(&sd.tw4i, (size_t)P * sd.L));
            gen_tw4<uint32_t><<<1024, 256, 0, st>>>(sd.ltw_lo[dir], sd.ltw_hi[dir], sd.ltw_lo_n, sd.ltw_hi_n, sd.ltw_h,
                                                    sd.pk, P, sd.lg, pl.n_row, sd.tw4i);
        }
        CUDA_TRY(cudaGetLastError());
    }
    // CRT constants (approximate-quotient CRT, carry.cuh crt_coeffs)
    CrtK &K = sd.crt;
    memset(&K, 0, sizeof K);
    K.P = P;
    auto mul_words = [](std::vector<uint32_t> &x, uint32_t m) {   // x *= m (little-endian)
        uint64_t carry = 0;
        for (auto &w : x) { const uint64_t t = (uint64_t)w * m + carry; w = (uint32_t)t; carry = t >> 32; }
        if (carry) x.push_back((uint32_t)carry);
    };
    std::vector<uint32_t> M{1};
    for (uint32_t i = 0; i < P; i++) mul_words(M, pl.primes[i]);
    if (M.size() > (size_t)kMaxPrimes) return set_err(PA_E_BOUND, "CRT modulus exceeds %d words", kMaxPrimes);
    for (size_t w = 0; w < M.size(); w++) K.M[w] = M[w];
    for (uint32_t i = 0; i < P; i++) {
        const uint32_t p = pl.primes[i];
        K.p[i] = p;
        K.pinv[i] = pk[i].pinv;
        std::vector<uint32_t> Mi{1};
        uint64_t mimod = 1;
        for (uint32_t l = 0; l < P; l++)
            if (l != i) { mul_words(Mi, pl.primes[l]); mimod = mulmod64(mimod, pl.primes[l] % p, p); }
        for (size_t w = 0; w < Mi.size() && w < (size_t)kMaxPrimes; w++) K.MI[i][w] = Mi[w];
        K.qinv[i] = to_mont(inv_mod((uint32_t)mimod, p), p);
        K.G[i] = (uint64_t)(((unsigned __int128)1 << 64) / p);
    }
    return PA_OK;
}

static NttArgs ntt_args(const StageDev &sd, int dir, int pass /*0 col, 1 row*/, int elog = 5) {
    NttArgs a{};
    a.pk = sd.pk;
    a.regtw = sd.regtw[dir];
    a.regtwp = sd.regtwp[dir];
    a.regtw_stride = 16;
    memcpy(a.ctw, sd.ctw[dir], sizeof a.ctw);
    memcpy(a.ctwp, sd.ctwp[dir], sizeof a.ctwp);
    a.rtw = sd.rtw;
    a.rtw_stride = sd.rtw_stride;
    for (int r = 0; r < kMaxRounds; r++) a.rtw_off[r] = sd.rtw_off[elog - 4][pass * 2 + dir][r];
    for (int r = 0; r < kMaxRounds; r++) a.rtw_off4[r] = sd.rtw_off[0][pass * 2 + dir][r];
    a.ltw_lo = sd.ltw_lo[dir];
    a.ltw_hi = sd.ltw_hi[dir];
    a.ltw_lo_stride = sd.ltw_lo_n;
    a.ltw_hi_stride = sd.ltw_hi_n;
    a.ltw_h = sd.ltw_h;
    a.log2L = sd.lg;
    a.n1 = sd.pl.n_row;
    a.n2 = sd.pl.n_col;
    a.nprimes = sd.pl.nprimes;
    return a;
}

// ====================================================================== launchers
// SM count of the device the current pa_* call runs on: set per call by DevGuard from the
// context (a process may drive several GPUs), read by the launchers for grid sizing
static thread_local int g_num_sms = 0;

struct KInfo {
    int threads = 0;
    size_t smem = 0;
    int occ = 0;
};

// Launch attributes and occupancy are per device: callers keep one KInfo per device
// (kMaxDevices) and pass the current device's entry.
static constexpr int kMaxDevices = 16;
static KInfo &kinfo_slot(KInfo (&tab)[kMaxDevices]) {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
    return tab[d];
}

template <class F>
static int kinfo(F *fn, int threads, size_t smem, KInfo &ki) {
    if (ki.occ) return PA_OK;
    if (smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem));
    if (occ < 1) return set_err(PA_E_CUDA, "kernel cannot be resident (threads=%d smem=%zu)", threads, smem);
    ki.threads = threads;
    ki.smem = smem;
    ki.occ = occ;
    return PA_OK;
}

#ifndef PA_COL_LANES
#define PA_COL_LANES 1
#endif
template <int S_LOG, int E_LOG, int N1_LOG, int MODE, bool ZH>
static int launch_col_z(const ColArgs &A0, cudaStream_t st) {
    static KInfo kis[kMaxDevices];
    KInfo &ki = kinfo_slot(kis);
    auto fn = col_pass<S_LOG, E_LOG, N1_LOG, MODE, ZH>;
    TRY(kinfo(fn, 32 * (1 << (S_LOG - E_LOG)), (size_t)(1 << S_LOG) * 32 * 4, ki));
    ColArgs A = A0;
    if (E_LOG == 4)
        for (int r = 0; r < kMaxRounds; r++) A.nt.rtw_off[r] = A.nt.rtw_off4[r];
    const int grid = (int)std::min<uint64_t>(A.units, (uint64_t)ki.occ * g_num_sms);
    // co-resident CTAs share their SM slot's units round robin (col_pass) when the grid is
    // the full occupancy and every CTA of a slot gets work
    A.lanes = (PA_COL_LANES && grid == ki.occ * g_num_sms && A.units >= (uint64_t)grid * 2) ? (uint32_t)ki.occ : 1u;
    fn<<<grid, ki.threads, ki.smem, st>>>(A);
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

// A pass with few units (the single-vector MH forward and both inverses: one unit per CTA)
// is as long as one unit takes; 16-element threads (twice the threads per column) halve
// that.  Many-unit passes keep 32 elements per thread (fewer instructions per point).
// Measured on C4: the MMH inverse (192 units) 20.8 -> 18.9 us with E = 16, but the MH
// passes (352 units) slower (forward 14.8 -> 18.9 us), so only passes below 1.5 units per SM.
#ifndef PA_COL_E4_UNITS
#define PA_COL_E4_UNITS 3                          // E = 16 while 2 units <= this x SMs
#endif
template <int S_LOG, int E_LOG, int N1_LOG, int MODE>
static int launch_col_e(const ColArgs &A, cudaStream_t st) {
    // the zero-half forward instantiation when every packed row lies in the first half
    if constexpr (MODE == COL_FWD)
        if (2ull * A.rows <= (1ull << S_LOG)) return launch_col_z<S_LOG, E_LOG, N1_LOG, MODE, true>(A, st);
    return launch_col_z<S_LOG, E_LOG, N1_LOG, MODE, false>(A, st);
}

template <int S_LOG, int N1_LOG, int MODE>
static int launch_col_t(const ColArgs &A, cudaStream_t st) {
    if constexpr (S_LOG == 8) {
        if (2ull * A.units <= (uint64_t)PA_COL_E4_UNITS * g_num_sms) return launch_col_e<S_LOG, 4, N1_LOG, MODE>(A, st);
    }
    return launch_col_e<S_LOG, 5, N1_LOG, MODE>(A, st);
}

// (column log, row log) pairs the planner produces (plan_product: MMH and single-vector rules)
template <int MODE>
static int launch_col(int slog, int n1log, const ColArgs &A, cudaStream_t st) {
#define PA_COL(S, N) \
    if (slog == S && n1log == N) return launch_col_t<S, N, MODE>(A, st);
    PA_COL(5, 5) PA_COL(5, 6) PA_COL(6, 6) PA_COL(6, 7) PA_COL(7, 7) PA_COL(7, 8) PA_COL(8, 8) PA_COL(8, 9)
    PA_COL(8, 10) PA_COL(8, 11) PA_COL(8, 12) PA_COL(8, 13) PA_COL(8, 14) PA_COL(9, 14)
#undef PA_COL
    return set_err(PA_E_PARAM, "unsupported column/row split 2^%d x 2^%d", slog, n1log);
}

constexpr int inv_v(int slog) {
    return slog >= 10 ? 1 : ((1024 >> slog) < (1 << (slog - 1)) ? (1024 >> slog) : (1 << (slog - 1)));
}
constexpr int row_v(int slog) {
    return (256 >> (slog - 5)) < 1 ? 1 : ((256 >> (slog - 5)) > 32 ? 32 : (256 >> (slog - 5)));
}

template <int S_LOG, int MODE>
static int launch_row_t(const RowArgs &A0, cudaStream_t st) {
    constexpr int E_LOG = 5;
    // the inverse transforms a single vector: small CTAs (V S = 1024 words; 2048 measured
    // 21.0 vs 19.0 us for the C4 MMH inverse) give enough units
    // ROW_STORE (precomputed transforms, comparators): half the rows of the MAC-era default
    // (C4 re-key: 108 -> 102 us for the 372 vectors of 2^9-point rows)
    constexpr int V = MODE == ROW_INV ? inv_v(S_LOG) : MODE == ROW_STORE ? (row_v(S_LOG) > 1 ? row_v(S_LOG) / 2 : 1) : row_v(S_LOG);
    static KInfo kis[kMaxDevices];
    KInfo &ki = kinfo_slot(kis);
    auto fn = row_pass<S_LOG, E_LOG, V, MODE>;
    constexpr int S = 1 << S_LOG;
    TRY(kinfo(fn, V * (S >> E_LOG), (size_t)V * (S + S / 32) * 4, ki));
    RowArgs A = A0;
    A.units = (A.nt.n2 / V) * A.nt.nprimes;
    const uint64_t work = MODE == ROW_STORE ? (uint64_t)A.units * A.nvec : A.units;
    const int grid = (int)std::min<uint64_t>(work, (uint64_t)ki.occ * g_num_sms);
    fn<<<grid, ki.threads, ki.smem, st>>>(A);
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

template <int MODE>
static int launch_row(int slog, const RowArgs &A, cudaStream_t st) {
    switch (slog) {
        case 5: return launch_row_t<5, MODE>(A, st);
        case 6: return launch_row_t<6, MODE>(A, st);
        case 7: return launch_row_t<7, MODE>(A, st);
        case 8: return launch_row_t<8, MODE>(A, st);
        case 9: return launch_row_t<9, MODE>(A, st);
        case 10: return launch_row_t<10, MODE>(A, st);
        case 11: return launch_row_t<11, MODE>(A, st);
        case 12: return launch_row_t<12, MODE>(A, st);
        case 13: return launch_row_t<13, MODE>(A, st);
        case 14: return launch_row_t<14, MODE>(A, st);
    }
    return set_err(PA_E_PARAM, "unsupported row length 2^%d", slog);
}

template <int S_LOG>
static int launch_macinv_t(const MacInvArgs &A0, cudaStream_t st) {
    constexpr int E_LOG = 5;
    constexpr int V = inv_v(S_LOG);                     // as the inverse row pass
    static KInfo kis[kMaxDevices];
    KInfo &ki = kinfo_slot(kis);
    auto fn = row_macinv<S_LOG, E_LOG, V>;
    constexpr int S = 1 << S_LOG;
    TRY(kinfo(fn, V * (S >> E_LOG), (size_t)V * (S + S / 32) * 4, ki));
    MacInvArgs A = A0;
    A.units = (A.fw.n2 / V) * A.fw.nprimes;
    const int grid = (int)std::min<uint64_t>(A.units, (uint64_t)ki.occ * g_num_sms);
    fn<<<grid, ki.threads, ki.smem, st>>>(A);
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

static int launch_macinv(int slog, const MacInvArgs &A, cudaStream_t st) {
    switch (slog) {
#define PA_LMI(S) case S: return launch_macinv_t<S>(A, st);
        PA_LMI(5) PA_LMI(6) PA_LMI(7) PA_LMI(8) PA_LMI(9) PA_LMI(10) PA_LMI(11) PA_LMI(12) PA_LMI(13) PA_LMI(14)
#undef PA_LMI
    }
    return set_err(PA_E_PARAM, "unsupported row length 2^%d", slog);
}

// Grid of the row MAC.  Mode 0 splits the (unit, vector) iterations evenly: a unit then
// spans at most ceil(grid / nunits) + 1 consecutive CTAs, and CTA b adds its canonical
// partials (< p) into slot b mod nslot, so a slot sees at most four partials of a unit
// (< 4p < 2^32).  nslot = 1 while grid <= 3 nunits; few units and many vectors (C5a: 88
// units of 2048 vectors) take up to kMacSlots slots to keep every SM busy.  Modes 1/2
// (whole units per CTA): grid <= nunits, one slot.
#ifndef PA_MAC_DBG
#define PA_MAC_DBG 0     // timing-only ablations of the row MAC (1: no DFT, 2: no loads, 3: no loads, no MAC); results are wrong when set
#endif
static constexpr uint32_t kMacSlots = 4;
template <int S_LOG>
static int mac_grid_t(uint32_t nunits, uint32_t nvec, uint32_t mode, int *grid, uint32_t *nslot) {
    constexpr int E_LOG = 5;
    static KInfo kis[kMaxDevices];
    KInfo &ki = kinfo_slot(kis);
    auto fn = row_mac<S_LOG, E_LOG>;
    TRY(kinfo(fn, mac_v(S_LOG) * (1 << (S_LOG - E_LOG)), mac_smem_bytes<S_LOG, mac_pad(S_LOG), PA_MAC_NSX, mac_ain(S_LOG)>(), ki));
    const uint64_t full = (uint64_t)ki.occ * g_num_sms;
    *nslot = 1;
    if (mode == 3) {                                     // 64-bit sums: no partial-count bound
        *grid = (int)std::min<uint64_t>(full, (uint64_t)nunits * nvec);
        return PA_OK;
    }
    if (mode) {
        *grid = (int)std::min<uint64_t>(nunits, full);
        return PA_OK;
    }
    // one slot: grid <= 3 nunits, every CTA runs >= nvec/3 iterations, a unit touches <= 4 CTAs
    uint64_t g = std::min<uint64_t>(full, 3ull * nunits);
    const uint64_t T = (uint64_t)nunits * nvec;
    if (g < full && nvec >= 8) {
        uint64_t gs = std::min<uint64_t>(full, T);
        for (;;) {
            const uint64_t q = T / gs;                       // fewest iterations a CTA runs
            const uint64_t span = cdiv(nvec, q) + 1;         // most CTAs a unit touches
            const uint64_t ns = cdiv(span, 4);
            if (ns <= kMacSlots) {
                if (ns > 1) { g = gs; *nslot = (uint32_t)ns; }
                break;
            }
            gs = gs * 3 / 4;
        }
    }
    *grid = (int)g;
    return PA_OK;
}

template <int S_LOG, int MODE>
static int launch_mac_m(const MacArgs &A, int grid, cudaStream_t st) {
    constexpr int E_LOG = 5;
    static KInfo kis[kMaxDevices];
    KInfo &ki = kinfo_slot(kis);
    auto fn = row_mac<S_LOG, E_LOG, PA_MAC_DBG, mac_pad(S_LOG), PA_MAC_NSX, mac_ain(S_LOG), MODE>;
    TRY(kinfo(fn, mac_v(S_LOG) * (1 << (S_LOG - E_LOG)), mac_smem_bytes<S_LOG, mac_pad(S_LOG), PA_MAC_NSX, mac_ain(S_LOG)>(), ki));
    fn<<<grid, ki.threads, ki.smem, st>>>(A);
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}
template <int S_LOG>
static int launch_mac_t(const MacArgs &A, int grid, cudaStream_t st) {
    switch (A.mode) {
        case 0: return launch_mac_m<S_LOG, 0>(A, grid, st);
        case 1: return launch_mac_m<S_LOG, 1>(A, grid, st);
        case 2: return launch_mac_m<S_LOG, 2>(A, grid, st);
        case 3: return launch_mac_m<S_LOG, 3>(A, grid, st);
    }
    return set_err(PA_E_PARAM, "row MAC mode %u", A.mode);
}
static int mac_grid(int slog, uint32_t nunits, uint32_t nvec, uint32_t mode, int *grid, uint32_t *nslot) {
    switch (slog) {
#define PA_MG(S) case S: return mac_grid_t<S>(nunits, nvec, mode, grid, nslot);
        PA_MG(5) PA_MG(6) PA_MG(7) PA_MG(8) PA_MG(9) PA_MG(10) PA_MG(11) PA_MG(12) PA_MG(13) PA_MG(14)
#undef PA_MG
    }
    return set_err(PA_E_PARAM, "unsupported row length 2^%d", slog);
}

static int launch_mac(int slog, const MacArgs &A, int grid, cudaStream_t st) {
    switch (slog) {
#define PA_LM(S) case S: return launch_mac_t<S>(A, grid, st);
        PA_LM(5) PA_LM(6) PA_LM(7) PA_LM(8) PA_LM(9) PA_LM(10) PA_LM(11) PA_LM(12) PA_LM(13) PA_LM(14)
#undef PA_LM
    }
    return set_err(PA_E_PARAM, "unsupported row length 2^%d", slog);
}

template <int P, bool RING>
static int launch_crt_carry_t(const uint32_t *res, const StageDev &sd, uint32_t ncoef, uint64_t gamma,
                              const uint32_t *addend, uint32_t n_addend, uint32_t *coef, uint32_t *out, uint32_t W,
                              uint32_t *state, uint32_t Wfin, cudaStream_t st, uint32_t *obe) {
    const uint32_t B = sd.pl.limb_bits;
    const uint32_t cap = (32u * kCCTile + 32u * P) / B + 3;
    crt_coeffs<P><<<(ncoef + 127) / 128, 128, 0, st>>>(res, sd.L, ncoef, sd.crt, coef);
    CUDA_TRY(cudaGetLastError());
#ifndef PA_CC_DBG
#define PA_CC_DBG 0
#endif
    auto fn = crt_carry<P, RING, PA_CC_DBG>;            // PA_CC_DBG: timing-only ablations (carry.cuh)
    const uint32_t ntiles = (W + kCCTile - 1) / kCCTile;
    fn<<<ntiles, kCCT, 0, st>>>(coef, sd.L, ncoef, B, (uint32_t)gamma, addend, n_addend, out, W, cap,
                                      state, Wfin, obe);
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

template <bool RING>
static int launch_crt_carry(const uint32_t *res, const StageDev &sd, uint32_t ncoef, uint64_t gamma,
                            const uint32_t *addend, uint32_t n_addend, uint32_t *coef, uint32_t *out, uint32_t W,
                            uint32_t *state, uint32_t Wfin, cudaStream_t st, uint32_t *obe = nullptr) {
#define PA_CC_CASE(P) \
    case P: return launch_crt_carry_t<P, RING>(res, sd, ncoef, gamma, addend, n_addend, coef, out, W, state, Wfin, st, obe);
    switch (sd.pl.nprimes) {
        PA_CC_CASE(2) PA_CC_CASE(3) PA_CC_CASE(4) PA_CC_CASE(5) PA_CC_CASE(6) PA_CC_CASE(7) PA_CC_CASE(8)
        PA_CC_CASE(9) PA_CC_CASE(10) PA_CC_CASE(11) PA_CC_CASE(12) PA_CC_CASE(13) PA_CC_CASE(14)
        PA_CC_CASE(15) PA_CC_CASE(16)
    }
#undef PA_CC_CASE
    return set_err(PA_E_PARAM, "unsupported prime count %u", sd.pl.nprimes);
}


// ====================================================================== context
struct ProfRec {
    const char *name;
    cudaEvent_t a, b;
};

// Per-hash working buffers (everything a hash writes).  A context has one active set;
// pa_hash_batch adds a second set + stream and alternates keys between them.
struct HashBufs {
    uint32_t *res = nullptr, *scratch = nullptr, *acc = nullptr, *scratch_mh = nullptr, *acc_mh = nullptr;
    uint64_t *S = nullptr;
    uint32_t *coef = nullptr, *y1 = nullptr, *Z = nullptr, *cstate = nullptr;
    cudaStream_t stream = nullptr;
};

// A captured CUDA graph of one call shape.  The graph is keyed on the pointers the call
// bakes into kernel arguments; a call with new pointers re-captures (host work only) and
// updates the executable graph in place (cudaGraphExecUpdate: same topology, new kernel
// parameters) instead of re-instantiating it.  Counters: pa_info.graph_*.
struct GraphSlot {
    cudaGraphExec_t exec = nullptr;
    std::vector<const void *> key;
    uint32_t launches = 0;
    void reset() {
        if (exec) cudaGraphExecDestroy(exec);
        exec = nullptr;
        key.clear();
    }
};

struct pa_ctx {
    Plan pl{};
    int device = 0;
    int num_sms = 0;                          // SMs of `device` (grid sizing)
    cudaStream_t stream = nullptr;
    DevAlloc da;
    StageDev smmh, smh;
    uint32_t nblk = 0;
    uint32_t rows_mmh = 0, rows_mh = 0;       // column-pass rows holding limbs
    uint32_t *res = nullptr;                  // packed residues [nvec][P][rows N1]
    uint32_t *ahat = nullptr, *scratch = nullptr, *acc = nullptr;
    uint32_t *bhat = nullptr, *scratch_mh = nullptr, *acc_mh = nullptr;
    uint32_t *c_words = nullptr;
    uint64_t *S = nullptr;
    uint32_t *coef = nullptr;                 // exact convolution coefficients [ncoef][P]
    uint32_t *y1 = nullptr, *Z = nullptr;
    uint32_t *cstate = nullptr;               // carry look-back: [kCarrySlots][1 + ntiles]
    uint32_t cstate_stride = 0;
    int cslot = 0;
    uint32_t *a_words_dev = nullptr, *b_words_dev = nullptr;   // pa_ctx_rekey expansions
    uint32_t *rekey_ok = nullptr;             // per vector: first draw accepted
    uint64_t *offs = nullptr;                 // paper mode: bit offset of each block's window
    uint32_t *wflags = nullptr;               // paper mode: window has a zero bit, [T]
    uint32_t *status = nullptr;               // device status of the last hash (paper mode)
    uint32_t T = 0;                           // paper mode: windows in the key
    uint32_t *tz_scale = nullptr;             // Toeplitz: [R, L^-1 R^2] (ROW_STORE scales of x and e')
    uint8_t *key_dev = nullptr;               // staging for pa_hash_host
    cudaStream_t copy_stream = nullptr;       // pa_hash_host H2D copies
    GraphSlot g_hash, g_host, g_batch;        // captured pa_hash / pa_hash_host / pa_hash_batch
    GraphSlot g_mg_pre[2], g_mg_post[2];      // multi-GPU, per buffer set: S1-S3 + export; S4-S7 (root)
    GraphSlot g_mg_host;                      // multi-GPU pa_hash_host: grouped H2D + S1-S3 + export
    // multi-GPU (pa_params.world >= 1): the NCCL communicator and, per buffer set, the
    // exported accumulator (send) and the reduced sum (recv; significant on the root)
    ncclComm_t comm = nullptr;
    bool x_u64 = false;                       // reduce 64-bit words (world * max prime >= 2^32)
    void *xsend[2] = {}, *xrecv[2] = {};
    // P2P exchange (pa_params.p2p, exchange.cuh): this GPU's receive region (cudaMalloc, shared
    // by CUDA IPC): two 64-bit receive buffers [P][L] and the counters (p2p_flag_word); every
    // rank's region as mapped in this process (own: p2p_region)
    bool p2p = false;
    uint8_t *p2p_region = nullptr;
    size_t p2p_recv_bytes = 0;
    uint8_t *p2p_peer[kMaxWorld] = {};
    uint32_t *p2p_tmp[2] = {};                // root: the imported accumulator [P][L], per hashing buffer set
    uint32_t p2p_uses[kMaxWorld] = {};        // keys rooted at rank q so far (the same on all ranks)
    GraphSlot g_p2p_pre[kMaxWorld][2][2];     // [root][receive buffer][hashing buffer set]
    GraphSlot g_p2p_post[2][2];               // [receive buffer][hashing buffer set]
    cudaEvent_t copy_ev[9] = {};
    uint8_t *out_dev = nullptr;
    uint8_t *key_dev2 = nullptr, *out_dev2 = nullptr;   // pa_hash_host_batch second staging set
    cudaEvent_t hb_copy[2] = {}, hb_done[2] = {};
    uint64_t Wg = 0, W_ring = 0, W_fold = 0, W_Z = 0, ncoef_mmh = 0;
    uint32_t mac_slots = 1;           // accumulator slots of the last MMH row MAC (mac_grid)
    uint32_t launches = 0;            // launches of the current / last hash call
    uint32_t launches_total = 0;      // since creation
    uint32_t graph_captures = 0, graph_updates = 0, graph_instantiations = 0;
    bool prof = false;
    std::vector<ProfRec> recs;
    std::vector<cudaEvent_t> evpool;
    std::map<std::string, std::pair<double, uint32_t>> acc_ms;
    // pa_hash_batch: second buffer set (own stream), fork/join events, captured batch graph
    bool alt_ready = false;
    HashBufs alt;
    size_t res_words = 0;
    cudaEvent_t bev[2] = {};
};
static constexpr int kCarrySlots = 8;

// Every pa_* call on a context runs on the context's device: the guard makes it current
// (restoring the caller's device on return) and selects its SM count for the launchers.
struct DevGuard {
    int prev = -1;
    bool switched = false;
    explicit DevGuard(const pa_ctx *c) {
        if (!c) return;
        g_num_sms = c->num_sms;
        if (cudaGetDevice(&prev) == cudaSuccess && prev != c->device && cudaSetDevice(c->device) == cudaSuccess)
            switched = true;
    }
    ~DevGuard() {
        if (switched) cudaSetDevice(prev);
    }
    DevGuard(const DevGuard &) = delete;
    DevGuard &operator=(const DevGuard &) = delete;
};

// exchange the active per-hash buffers (and stream) with the alternate set
static void swap_bufs(pa_ctx *c) {
    std::swap(c->res, c->alt.res);
    std::swap(c->scratch, c->alt.scratch);
    std::swap(c->acc, c->alt.acc);
    std::swap(c->scratch_mh, c->alt.scratch_mh);
    std::swap(c->acc_mh, c->alt.acc_mh);
    std::swap(c->S, c->alt.S);
    std::swap(c->coef, c->alt.coef);
    std::swap(c->y1, c->alt.y1);
    std::swap(c->Z, c->alt.Z);
    std::swap(c->cstate, c->alt.cstate);
    std::swap(c->stream, c->alt.stream);
}

static cudaEvent_t ev_get(pa_ctx *c) {
    if (!c->evpool.empty()) { cudaEvent_t e = c->evpool.back(); c->evpool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

struct ProfScope {
    pa_ctx *c;
    const char *name;
    cudaEvent_t a = nullptr;
    ProfScope(pa_ctx *c_, const char *n) : c(c_), name(n) {
        if (c->prof) { a = ev_get(c); cudaEventRecord(a, c->stream); }
    }
    ~ProfScope() {
        if (c->prof) {
            cudaEvent_t b = ev_get(c);
            cudaEventRecord(b, c->stream);
            c->recs.push_back({name, a, b});
        }
    }
};


// zero all look-back state slots used by one hash (one memset)
static int carry_reset(pa_ctx *c) {
    CUDA_TRY(cudaMemsetAsync(c->cstate, 0, (size_t)c->cstate_stride * kCarrySlots * 4, c->stream));
    c->cslot = 0;
    return PA_OK;
}

template <class Src>
static int run_carry(pa_ctx *c, const Src &src, uint32_t W, uint32_t *out) {
    if (c->cslot >= kCarrySlots) return set_err(PA_E_STATE, "carry slots exhausted");
    uint32_t *base = c->cstate + (size_t)c->cslot * c->cstate_stride;
    c->cslot++;
    const uint32_t nt = (uint32_t)cdiv(W, kCarryTile);
    carry_mw<Src><<<nt, kCarryT, 0, c->stream>>>(src, W, out, base + 1, base);
    c->launches++;
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

// a zeroed look-back state slot ([ticket, done, tiles...]) for one fused launch
static uint32_t *next_state(pa_ctx *c) {
    if (c->cslot >= kCarrySlots) return nullptr;
    return c->cstate + (size_t)(c->cslot++) * c->cstate_stride;
}

// y (W_fold words, resolved) -> y mod p, canonical (reading A6), in place
static int mersenne_finish(pa_ctx *c, uint32_t *y) {
    mersenne_finish_k<<<1, kFinT, 0, c->stream>>>(y, (uint32_t)c->W_fold, c->pl.gamma);
    c->launches++;
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

static uint32_t mac_v_rt(int slog) {
    switch (slog) {
        case 5: return mac_v(5); case 6: return mac_v(6); case 7: return mac_v(7); case 8: return mac_v(8);
        case 9: return mac_v(9); case 10: return mac_v(10); default: return 1;
    }
}

#ifndef PA_PACK_CW28
#define PA_PACK_CW28 1                 // key limbs reduced over 28-bit chunks where that saves one
#endif
template <int NW>
static void launch_pack_key(const KeySrc &s, uint32_t nvec, const PrimeSet &pk, uint32_t P, uint32_t wxp, uint32_t *res,
                            cudaStream_t st) {
    const dim3 grid((wxp + kPackL * kPackT - 1) / (kPackL * kPackT), nvec);   // kPackL limbs per thread
    // a limb of B <= 28 (NW - 1) + 28 bits... : ceil(B / 28) 28-bit chunks when that is fewer
    // than the ceil(32 NW / 24) 24-bit ones (B = 168: 6 against 8)
    constexpr int NCLO = (32 * (NW - 1) + 8 + 27) / 28;       // chunks of the narrowest B with NW words
    const uint32_t B = 8 * s.limb_bytes;
    if (PA_PACK_CW28 && NCLO <= 10 && B <= 28u * NCLO)
        pack_key_residues<NW, (NCLO <= 10 ? NCLO : 10)><<<grid, kPackT, 0, st>>>(s, pk, P, wxp, res);
    else if (PA_PACK_CW28 && (32 * NW + 27) / 28 <= 10)
        pack_key_residues<NW, ((32 * NW + 27) / 28 <= 10 ? (32 * NW + 27) / 28 : 10)><<<grid, kPackT, 0, st>>>(s, pk, P, wxp, res);
    else
        pack_key_residues<NW><<<grid, kPackT, 0, st>>>(s, pk, P, wxp, res);
}

static int launch_pack(const KeyLimbs &src, uint32_t B, uint32_t grid, const PrimeSet &pk, uint32_t P, uint32_t nvec,
                       uint32_t wxp, uint32_t *res, cudaStream_t st) {
    const int nw = B <= 56 ? 0 : (int)((B + 31) / 32);
    switch (nw) {
        case 0: pack_residues<KeyLimbs, 0><<<grid, 256, 0, st>>>(src, pk, P, nvec, wxp, res); break;
        case 2: launch_pack_key<2>(src.s, nvec, pk, P, wxp, res, st); break;
        case 3: launch_pack_key<3>(src.s, nvec, pk, P, wxp, res, st); break;
        case 4: launch_pack_key<4>(src.s, nvec, pk, P, wxp, res, st); break;
        case 5: launch_pack_key<5>(src.s, nvec, pk, P, wxp, res, st); break;
        case 6: launch_pack_key<6>(src.s, nvec, pk, P, wxp, res, st); break;
        case 7: launch_pack_key<7>(src.s, nvec, pk, P, wxp, res, st); break;
        case 8: launch_pack_key<8>(src.s, nvec, pk, P, wxp, res, st); break;
        default: return set_err(PA_E_PARAM, "unsupported limb width %u", B);
    }
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

template <class Src>
static int launch_pack(const Src &src, uint32_t B, uint32_t grid, const PrimeSet &pk, uint32_t P, uint32_t nvec,
                       uint32_t wxp, uint32_t *res, cudaStream_t st) {
    const int nw = B <= 56 ? 0 : (int)((B + 31) / 32);
    const uint32_t tiles = (uint32_t)cdiv(wxp, (uint64_t)kPackL * kPackT);
    if (nw >= 2 && nvec <= 65535 && (uint64_t)tiles * nvec >= 2ull * g_num_sms) {
        // many vectors (re-key): kPackL limbs per thread; the single-vector MH pack keeps
        // one limb per thread (more CTAs for its ~170 tiles)
        const dim3 tg(tiles, nvec);
        switch (nw) {
            case 2: pack_residues_tiled<Src, 2><<<tg, kPackT, 0, st>>>(src, pk, P, wxp, res); break;
            case 3: pack_residues_tiled<Src, 3><<<tg, kPackT, 0, st>>>(src, pk, P, wxp, res); break;
            case 4: pack_residues_tiled<Src, 4><<<tg, kPackT, 0, st>>>(src, pk, P, wxp, res); break;
            case 5: pack_residues_tiled<Src, 5><<<tg, kPackT, 0, st>>>(src, pk, P, wxp, res); break;
            case 6: pack_residues_tiled<Src, 6><<<tg, kPackT, 0, st>>>(src, pk, P, wxp, res); break;
            case 7: pack_residues_tiled<Src, 7><<<tg, kPackT, 0, st>>>(src, pk, P, wxp, res); break;
            case 8: pack_residues_tiled<Src, 8><<<tg, kPackT, 0, st>>>(src, pk, P, wxp, res); break;
            default: return set_err(PA_E_PARAM, "unsupported limb width %u", B);
        }
        CUDA_TRY(cudaGetLastError());
        return PA_OK;
    }
    switch (nw) {
        case 0: pack_residues<Src, 0><<<grid, 256, 0, st>>>(src, pk, P, nvec, wxp, res); break;
        case 2: pack_residues<Src, 2><<<grid, 256, 0, st>>>(src, pk, P, nvec, wxp, res); break;
        case 3: pack_residues<Src, 3><<<grid, 256, 0, st>>>(src, pk, P, nvec, wxp, res); break;
        case 4: pack_residues<Src, 4><<<grid, 256, 0, st>>>(src, pk, P, nvec, wxp, res); break;
        case 5: pack_residues<Src, 5><<<grid, 256, 0, st>>>(src, pk, P, nvec, wxp, res); break;
        case 6: pack_residues<Src, 6><<<grid, 256, 0, st>>>(src, pk, P, nvec, wxp, res); break;
        case 7: pack_residues<Src, 7><<<grid, 256, 0, st>>>(src, pk, P, nvec, wxp, res); break;
        case 8: pack_residues<Src, 8><<<grid, 256, 0, st>>>(src, pk, P, nvec, wxp, res); break;
        default: return set_err(PA_E_PARAM, "unsupported limb width %u", B);
    }
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

// ---- pack -> forward column pass -> row pass with MAC -> inverse; residues in acc
// ---- S1+S2 (first pass) of vectors [0, nvec) of src: pack -> residues -> forward
// column pass into scratch.  `res` / `scratch` point at the first vector's slots.
template <class Src>
static int stage_pack_col(pa_ctx *c, StageDev &sd, const Src &src, uint32_t nvec, uint32_t rows, uint32_t *res,
                          uint32_t *scratch, const char *tag_pack, const char *tag_fwd1) {
    const int clog = __builtin_ctz(sd.pl.n_col);
    const uint32_t P = sd.pl.nprimes;
    const uint32_t wxp = rows * sd.pl.n_row;
    {
        ProfScope ps(c, tag_pack);
        const uint64_t total = (uint64_t)nvec * wxp;
        const uint32_t grid = (uint32_t)std::min<uint64_t>(cdiv(total, 256), (uint64_t)g_num_sms * 8);
        TRY(launch_pack(src, sd.pl.limb_bits, grid, sd.pks, P, nvec, wxp, res, c->stream));
        c->launches++;
    }
    {
        ProfScope ps(c, tag_fwd1);
        ColArgs A{};
        A.nt = ntt_args(sd, 0, 0);
        A.src = res;
        A.rows = rows;
        A.tw4 = sd.tw4f;
        A.dst = scratch;
        A.nvec = nvec;
        A.units = (sd.pl.n_row / 32) * P * nvec;
        TRY(launch_col<COL_FWD>(clog, __builtin_ctz(sd.pl.n_row), A, c->stream));
        c->launches++;
    }
    return PA_OK;
}

// ---- S2 (second pass) + S3 for vectors [0, nvec) (pointers at the first vector):
// acc (+)= sum_i X_i (.) hat_i.  only: the single accumulation (balanced split, red.add
// into zeroed acc); else first / later call of a multi-call accumulation (whole units per
// CTA, store / modular read-modify-write, no atomics).
static int stage_mac(pa_ctx *c, StageDev &sd, uint32_t nvec, const uint32_t *scratch, const uint32_t *hat,
                     uint32_t *acc, bool first, const char *tag, bool only = true, bool zero = true,
                     unsigned long long *dst64 = nullptr) {
    const int rlog = __builtin_ctz(sd.pl.n_row);
    const uint32_t P = sd.pl.nprimes;
    ProfScope ps(c, tag);
    MacArgs M{};
    M.mode = dst64 ? 3u : only ? 0u : (first ? 1u : 2u);
    M.dst64 = dst64;
    M.nt = ntt_args(sd, 0, 1);
    M.src = scratch;
    M.ahat = hat;
    M.dst = acc;
    M.nvec = nvec;
    M.nunits = (sd.pl.n_col / mac_v_rt(rlog)) * P;
    int grid = 0;
    TRY(mac_grid(rlog, M.nunits, nvec, M.mode, &grid, &M.nslot));
    M.slot_stride = P * sd.L;
    if (only && zero && !dst64) CUDA_TRY(cudaMemsetAsync(acc, 0, (size_t)M.nslot * P * sd.L * 4, c->stream));
    if (&sd == &c->smmh && !dst64) c->mac_slots = M.nslot;
    TRY(launch_mac(rlog, M, grid, c->stream));
    c->launches++;
    return PA_OK;
}

// ---- S4: one inverse transform of acc (in place, natural order, canonical residues)
// src (default acc): nslot slots src_stride words apart (default P L), each < 4p, summed
static int stage_inverse(pa_ctx *c, StageDev &sd, uint32_t *acc, const char *tag, uint32_t nslot = 1,
                         const uint32_t *src = nullptr, uint64_t src_stride = 0) {
    const int clog = __builtin_ctz(sd.pl.n_col), rlog = __builtin_ctz(sd.pl.n_row);
    const uint32_t P = sd.pl.nprimes;
    ProfScope ps(c, tag);
    RowArgs R{};
    R.nt = ntt_args(sd, 1, 1);
    R.src = src ? src : acc;
    R.nsrc = nslot;
    R.src_stride = src_stride ? (uint32_t)src_stride : P * sd.L;
    R.dst = acc;
    R.tw4 = sd.tw4i;
    R.nvec = 1;
    TRY(launch_row<ROW_INV>(rlog, R, c->stream));
    ColArgs A{};
    A.nt = ntt_args(sd, 1, 0);
    A.src = acc;
    A.dst = acc;
    A.nvec = 1;
    A.units = (sd.pl.n_row / 32) * P;
    TRY(launch_col<COL_INV>(clog, rlog, A, c->stream));
    c->launches += 2;
    return PA_OK;
}

// ---- S3+S4 of a single vector (the MH product): forward row DFT x hat, inverse row DFT
// (one kernel, row_macinv), then the inverse column pass -> canonical residues in dst,
// natural order
static int stage_macinv(pa_ctx *c, StageDev &sd, const uint32_t *scratch, const uint32_t *hat, uint32_t *dst,
                        const char *tag_row, const char *tag_col) {
    const int clog = __builtin_ctz(sd.pl.n_col), rlog = __builtin_ctz(sd.pl.n_row);
    const uint32_t P = sd.pl.nprimes;
    {
        ProfScope ps(c, tag_row);
        MacInvArgs M{};
        M.fw = ntt_args(sd, 0, 1);
        M.iv = ntt_args(sd, 1, 1);
        M.src = scratch;
        M.bhat = hat;
        M.tw4 = sd.tw4i;
        M.dst = dst;
        TRY(launch_macinv(rlog, M, c->stream));
        c->launches++;
    }
    {
        ProfScope ps(c, tag_col);
        ColArgs A{};
        A.nt = ntt_args(sd, 1, 0);
        A.src = dst;
        A.dst = dst;
        A.nvec = 1;
        A.units = (sd.pl.n_row / 32) * P;
        TRY(launch_col<COL_INV>(clog, rlog, A, c->stream));
        c->launches++;
    }
    return PA_OK;
}

// ---- precompute transforms of word vectors (a_i or b) into hat (Montgomery, x 1/L)
static int precompute_hat(pa_ctx *c, StageDev &sd, const WordSrc &ws, uint32_t nvec, uint32_t rows,
                          uint32_t *scratch, uint32_t *hat) {
    TRY(stage_pack_col(c, sd, WordLimbs{ws}, nvec, rows, c->res, scratch, "pre_pack", "pre_col"));
    RowArgs R{};
    R.nt = ntt_args(sd, 0, 1);
    R.src = scratch;
    R.dst = hat;
    R.scale = sd.scale;
    R.nvec = nvec;
    TRY(launch_row<ROW_STORE>(__builtin_ctz(sd.pl.n_row), R, c->stream));
    return PA_OK;
}

static int expand_words(uint64_t key0, uint64_t key1, uint64_t bits, std::vector<uint32_t> &w, bool reject_allones) {
    const uint64_t nw64 = cdiv(bits, 64), nw32 = cdiv(bits, 32);
    std::vector<uint64_t> raw(nw64);
    uint64_t off = 0;
    for (;;) {
        Philox4x64::words(key0, key1, off, nw64, raw.data());
        off += nw64;
        w.assign(nw32, 0);
        for (uint64_t i = 0; i < nw32; i++) w[i] = (uint32_t)(raw[i / 2] >> (32 * (i & 1)));
        if (bits % 32) w[nw32 - 1] &= (uint32_t)((1ull << (bits % 32)) - 1);
        if (!reject_allones) return PA_OK;
        bool all = true;
        for (uint64_t i = 0; i < nw32 && all; i++) {
            const uint32_t want = (i == nw32 - 1 && bits % 32) ? (uint32_t)((1ull << (bits % 32)) - 1) : 0xFFFFFFFFu;
            all = (w[i] == want);
        }
        if (!all) return PA_OK;
    }
}

static const uint64_t kStreamB = 1ull << 63, kStreamC = (1ull << 63) + 1;
static const uint64_t kStreamT = (1ull << 63) + 2;       // Toeplitz diagonal (reading A15)

// ====================================================================== Toeplitz comparator
// (NEXT-4; toeplitz.cuh).  Forward transform of nvec bit vectors (one prime): column pass
// from the packed coefficients, then the row pass in place with the output scale.
static int tz_forward(pa_ctx *c, const uint32_t *res, uint32_t nvec, uint32_t rows, uint32_t *dst,
                      const uint32_t *scale, const char *tag_col, const char *tag_row) {
    StageDev &sd = c->smmh;
    const int clog = __builtin_ctz(sd.pl.n_col), rlog = __builtin_ctz(sd.pl.n_row);
    {
        ProfScope ps(c, tag_col);
        ColArgs A{};
        A.nt = ntt_args(sd, 0, 0);
        A.src = res;
        A.rows = rows;
        A.tw4 = sd.tw4f;
        A.dst = dst;
        A.nvec = nvec;
        A.units = (sd.pl.n_row / 32) * nvec;
        TRY(launch_col<COL_FWD>(clog, rlog, A, c->stream));
        c->launches++;
    }
    {
        ProfScope ps(c, tag_row);
        RowArgs R{};
        R.nt = ntt_args(sd, 0, 1);
        R.src = dst;
        R.dst = dst;
        R.scale = scale;
        R.nvec = nvec;
        TRY(launch_row<ROW_STORE>(rlog, R, c->stream));
        c->launches++;
    }
    return PA_OK;
}

static int toeplitz_alloc_and_precompute(pa_ctx *c) {
    const Plan &p = c->pl;
    TRY(setup_stage(c->da, p.mmh, c->smmh, c->stream));
    const StageDev &sd = c->smmh;
    const uint32_t L = sd.L, lr = sd.lg - 1, nb = (uint32_t)p.tz_nb, no = (uint32_t)p.tz_no;
    const uint32_t ne = nb + no - 1;
    c->nblk = nb;
    TRY(c->da.alloc(&c->res, std::max<size_t>((size_t)nb << lr, (size_t)ne * L)));
    TRY(c->da.alloc(&c->scratch, (size_t)nb * L));             // X^ (in place after the column pass)
    TRY(c->da.alloc(&c->ahat, (size_t)ne * L));                // E'^ = T(e') L^-1 R
    TRY(c->da.alloc(&c->acc, (size_t)no * L));
    TRY(c->da.alloc(&c->tz_scale, 2));
    TRY(c->da.alloc(&c->status, 4));
    const uint32_t q = p.mmh.primes[0];
    const uint32_t sc[2] = {(uint32_t)powmod64(2, 32, q),
                            (uint32_t)mulmod64(inv_mod(L % q, q), powmod64(2, 64, q), q)};
    CUDA_TRY(cudaMemcpyAsync(c->tz_scale, sc, sizeof sc, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemsetAsync(c->status, 0, 4, c->stream));
    // diagonal d: n + m - 1 bits of stream (seed, 2^63 + 2), LSB-first words (reading A15)
    const uint64_t nd = p.n + p.m - 1;
    std::vector<uint32_t> dw;
    TRY(expand_words(p.seed, kStreamT, nd, dw, false));
    uint32_t *dw_dev = nullptr;
    CUDA_TRY(cudaMallocAsync(&dw_dev, dw.size() * 4, c->stream));
    dbg_add(dw_dev, dw.size() * 4);
    CUDA_TRY(cudaMemcpyAsync(dw_dev, dw.data(), dw.size() * 4, cudaMemcpyHostToDevice, c->stream));
    const uint64_t tot = (uint64_t)ne * L;
    toeplitz_pack_diag<<<(uint32_t)std::min<uint64_t>(cdiv(tot, 256), (uint64_t)g_num_sms * 16), 256, 0,
                         c->stream>>>(dw_dev, nd, p.m, lr, no, ne, c->res);
    int rc = cudaGetLastError() == cudaSuccess ? PA_OK : set_err(PA_E_CUDA, "toeplitz_pack_diag launch failed");
    if (rc == PA_OK) rc = tz_forward(c, c->res, ne, sd.pl.n_col, c->ahat, c->tz_scale + 1, "pre_col", "pre_row");
    const cudaError_t e = cudaStreamSynchronize(c->stream);
    dbg_remove(dw_dev);
    cudaFreeAsync(dw_dev, c->stream);
    if (rc != PA_OK) return rc;
    if (e != cudaSuccess) return set_err(PA_E_CUDA, "Toeplitz precompute failed: %s", cudaGetErrorString(e));
    return PA_OK;
}

template <int O>
static void launch_tz_mac(const pa_ctx *c, uint32_t grid, uint32_t b0, uint32_t b1, uint32_t o0) {
    const StageDev &sd = c->smmh;
    const uint32_t ebase = b0 - o0 + (uint32_t)c->pl.tz_no - O;        // >= 0: o0 + O <= no
    toeplitz_mac<O><<<grid, 256, 0, c->stream>>>(c->scratch, c->ahat, b0, b1, ebase, sd.L, sd.pl.primes[0],
                                                 sd.pks.k[0].pinv, c->acc + (size_t)o0 * sd.L);
}

static int run_toeplitz(pa_ctx *c, const uint8_t *key, uint8_t *out_bits) {
    const Plan &p = c->pl;
    StageDev &sd = c->smmh;
    const uint32_t L = sd.L, lr = sd.lg - 1, nb = (uint32_t)p.tz_nb, no = (uint32_t)p.tz_no;
    {
        ProfScope ps(c, "tz_pack");
        const uint64_t tot = (uint64_t)nb << lr;
        toeplitz_pack_bits<<<(uint32_t)std::min<uint64_t>(cdiv(tot / 4, 256), (uint64_t)g_num_sms * 16), 256, 0,
                             c->stream>>>(key, p.n, tot, c->res);
        c->launches++;
        CUDA_TRY(cudaGetLastError());
    }
    TRY(tz_forward(c, c->res, nb, sd.pl.n_col / 2, c->scratch, c->tz_scale, "tz_fwd_col", "tz_fwd_row"));
    // input blocks in groups whose counts stay below the prime (one group unless n >= prime),
    // output blocks in groups of at most kTzMaxOut per MAC launch
    const uint32_t gb = std::max<uint32_t>(1, p.tz_group);
    for (uint32_t b0 = 0; b0 < nb; b0 += gb) {
        const uint32_t b1 = std::min(nb, b0 + gb);
        {
            ProfScope ps(c, "tz_mac");
            const uint32_t grid = (uint32_t)cdiv(L, 256);      // one element per thread
            for (uint32_t o0 = 0; o0 < no; o0 += kTzMaxOut) {
                const uint32_t O = std::min<uint32_t>(kTzMaxOut, no - o0);
                switch (O) {
#define PA_TZ(Q) case Q: launch_tz_mac<Q>(c, grid, b0, b1, o0); break;
                    PA_TZ(1) PA_TZ(2) PA_TZ(3) PA_TZ(4) PA_TZ(5) PA_TZ(6) PA_TZ(7) PA_TZ(8)
                    PA_TZ(9) PA_TZ(10) PA_TZ(11) PA_TZ(12) PA_TZ(13) PA_TZ(14) PA_TZ(15) PA_TZ(16)
#undef PA_TZ
                }
                c->launches++;
                CUDA_TRY(cudaGetLastError());
            }
        }
        for (uint32_t o = 0; o < no; o++) TRY(stage_inverse(c, sd, c->acc + (size_t)o * L, "tz_inverse"));
        {
            ProfScope ps(c, "tz_extract");
            const uint64_t nbytes = cdiv(p.m, 8), nwarp = cdiv(p.m, 32);
            toeplitz_extract<<<(uint32_t)std::min<uint64_t>(cdiv(nwarp, 8), (uint64_t)g_num_sms * 16), 256, 0,
                               c->stream>>>(c->acc, lr, L, p.m, out_bits, nbytes, b0 > 0 ? 1u : 0u);
            c->launches++;
            CUDA_TRY(cudaGetLastError());
        }
    }
    return PA_OK;
}

static uint32_t rows_for(uint64_t limbs, uint32_t n1, uint32_t n2) {
    return (uint32_t)std::min<uint64_t>(n2, cdiv(limbs, n1));
}

static int toeplitz_alloc_and_precompute(pa_ctx *c);

static int ctx_alloc_and_precompute(pa_ctx *c, const pa_params *prm) {
    Plan &p = c->pl;
    if (p.toeplitz) return toeplitz_alloc_and_precompute(c);
    if (!p.mh_only) TRY(setup_stage(c->da, p.mmh, c->smmh, c->stream));   // MH-only: no MMH stage
    TRY(setup_stage(c->da, p.mh, c->smh, c->stream));
    c->nblk = (uint32_t)(p.b1 - p.b0);
    const uint32_t Lm = c->smmh.L, Pm = p.mmh.nprimes;
    const uint32_t Lh = c->smh.L, Ph = p.mh.nprimes;
    const uint32_t Bm = p.mmh.limb_bits, Bh = p.mh.limb_bits;
    const uint64_t wx = Bm ? cdiv(p.r, Bm) : 0, wa = Bm ? cdiv(p.gamma, Bm) : 0;
    c->ncoef_mmh = Bm ? wx + wa - 1 : 0;
    c->Wg = cdiv(p.gamma, 32);
    c->W_ring = c->Wg + Pm + 2;              // wrapped pieces of tiny rings may pass the top
    c->W_fold = c->W_ring + 2;               // 64-bit column sums carry into 2 more words
    c->W_Z = cdiv(p.alpha, 32);
    const uint64_t Wa32 = cdiv(p.gamma, 32), Wal32 = cdiv(p.alpha, 32);
    const uint32_t rows_x = Bm ? rows_for(wx, p.mmh.n_row, p.mmh.n_col) : 0;
    const uint32_t rows_a = Bm ? rows_for(wa, p.mmh.n_row, p.mmh.n_col) : 0;
    c->rows_mmh = rows_x;
    const uint32_t rows_y = rows_for(cdiv(p.gamma, Bh), p.mh.n_row, p.mh.n_col);
    const uint32_t rows_b = rows_for(cdiv(p.alpha, Bh), p.mh.n_row, p.mh.n_col);
    c->rows_mh = rows_y;
    const uint64_t res_words = std::max<uint64_t>(
        (uint64_t)c->nblk * Pm * std::max(rows_x, rows_a) * p.mmh.n_row,
        (uint64_t)Ph * std::max(rows_y, rows_b) * p.mh.n_row);
    c->res_words = res_words;
    TRY(c->da.alloc(&c->res, res_words));
    TRY(c->da.alloc(&c->ahat, (size_t)c->nblk * Pm * Lm));
    TRY(c->da.alloc(&c->scratch, (size_t)c->nblk * Pm * Lm));
    TRY(c->da.alloc(&c->acc, (size_t)kMacSlots * Pm * Lm));     // row MAC slots (mac_grid)
    TRY(c->da.alloc(&c->bhat, (size_t)Ph * Lh));
    TRY(c->da.alloc(&c->scratch_mh, (size_t)Ph * Lh));
    TRY(c->da.alloc(&c->acc_mh, (size_t)Ph * Lh));
    TRY(c->da.alloc(&c->c_words, Wal32));
    const uint64_t Smax = std::max<uint64_t>(c->W_fold, c->W_Z);
    TRY(c->da.alloc(&c->S, Smax));
    TRY(c->da.alloc(&c->coef, std::max<size_t>((size_t)Pm * Lm, (size_t)Ph * Lh)));
    TRY(c->da.alloc(&c->y1, std::max<uint64_t>(c->W_fold, c->Wg)));
    TRY(c->da.alloc(&c->Z, c->W_Z));
    // crt_carry: ticket, done counter and one flag per tile, each on its own 128-byte line
    c->cstate_stride = (uint32_t)((cdiv(Smax, std::min(kCarryTile, kCCTile)) + 2) * kFlagStride);
    TRY(c->da.alloc(&c->cstate, (size_t)c->cstate_stride * kCarrySlots));
    TRY(c->da.alloc(&c->status, 4));
    CUDA_TRY(cudaMemsetAsync(c->status, 0, 4, c->stream));
    if (p.paper_k) {
        c->T = (uint32_t)(p.n / p.gamma);
        TRY(c->da.alloc(&c->offs, p.k));
        TRY(c->da.alloc(&c->wflags, c->T));
    }

    // ---- hash keys (reading A7): a_i for the shard's blocks, b, c
    std::vector<uint32_t> aw((size_t)c->nblk * Wa32), bw, cw, tmp;
    for (uint32_t i = 0; i < c->nblk; i++) {
        if (prm->a_words) {
            memcpy(&aw[(size_t)i * Wa32], prm->a_words + (size_t)i * Wa32, Wa32 * 4);
        } else {
            TRY(expand_words(p.seed, p.b0 + i, p.gamma, tmp, true));
            memcpy(&aw[(size_t)i * Wa32], tmp.data(), Wa32 * 4);
        }
    }
    if (prm->b_words) bw.assign(prm->b_words, prm->b_words + Wal32);
    else { TRY(expand_words(p.seed, kStreamB, p.alpha, bw, false)); bw[0] |= 1u; }
    if (prm->c_words) cw.assign(prm->c_words, prm->c_words + Wal32);
    else TRY(expand_words(p.seed, kStreamC, p.alpha, cw, false));
    if (!(bw[0] & 1u)) return set_err(PA_E_PARAM, "b must be odd (PAPER.md:97)");
    if (p.alpha % 32) {
        const uint32_t mask = (uint32_t)((1ull << (p.alpha % 32)) - 1);
        if ((bw[Wal32 - 1] & ~mask) || (cw[Wal32 - 1] & ~mask)) return set_err(PA_E_PARAM, "b, c must be < 2^alpha");
    }
    if (prm->a_words) {
        for (uint32_t i = 0; i < c->nblk; i++) {
            bool all = true;
            for (uint64_t w = 0; w < Wa32 && all; w++) {
                const uint32_t want = (w == Wa32 - 1 && p.gamma % 32) ? (uint32_t)((1ull << (p.gamma % 32)) - 1) : 0xFFFFFFFFu;
                const uint32_t got = aw[(size_t)i * Wa32 + w];
                if (w == Wa32 - 1 && p.gamma % 32 && (got & ~want)) return set_err(PA_E_PARAM, "a_i must be < p");
                all = (got == want);
            }
            if (all) return set_err(PA_E_PARAM, "a_i must be < p (got p)");
        }
    }
    uint32_t *a_dev = nullptr, *b_dev = nullptr;
    CUDA_TRY(cudaMallocAsync(&a_dev, std::max<size_t>(aw.size() * 4, 16), c->stream));
    CUDA_TRY(cudaMallocAsync(&b_dev, Wal32 * 4, c->stream));
    dbg_add(a_dev, std::max<size_t>(aw.size() * 4, 16));
    dbg_add(b_dev, Wal32 * 4);
    CUDA_TRY(cudaMemcpyAsync(a_dev, aw.data(), aw.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(b_dev, bw.data(), Wal32 * 4, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->c_words, cw.data(), Wal32 * 4, cudaMemcpyHostToDevice, c->stream));
    WordSrc wsa{a_dev, (uint32_t)Wa32, Bm, (uint32_t)wa};
    int rc = p.mh_only ? PA_OK : precompute_hat(c, c->smmh, wsa, c->nblk, rows_a, c->scratch, c->ahat);
    WordSrc wsb{b_dev, (uint32_t)Wal32, Bh, (uint32_t)cdiv(p.alpha, Bh)};
    if (rc == PA_OK) rc = precompute_hat(c, c->smh, wsb, 1, rows_b, c->scratch_mh, c->bhat);
    cudaError_t e = cudaStreamSynchronize(c->stream);
    dbg_remove(a_dev);
    dbg_remove(b_dev);
    cudaFreeAsync(a_dev, c->stream);
    cudaFreeAsync(b_dev, c->stream);
    if (rc != PA_OK) return rc;
    if (e != cudaSuccess) return set_err(PA_E_CUDA, "precompute failed: %s", cudaGetErrorString(e));
    return PA_OK;
}

extern "C" int pa_plan(const pa_params *prm, pa_info *info) {
    Plan p;
    TRY(make_plan(prm, &p));
    if (info) {
        memset(info, 0, sizeof *info);
        info->n = p.n; info->r = p.r; info->m = p.m; info->gamma = p.gamma; info->alpha = p.alpha;
        info->k = p.k; info->block_begin = p.b0; info->block_end = p.b1;
        info->mmh = p.mmh; info->mh = p.mh;
        info->insecure_length = (!p.mh_only && !p.toeplitz && p.m >= p.gamma) ? 1u : 0u;
        info->world = p.world; info->rank = p.rank;
        info->acc_words = (uint64_t)p.mmh.nprimes << p.mmh.log2_len;
        info->tz_group_blocks = p.toeplitz ? p.tz_group : 0u;
        const uint64_t nb = p.b1 - p.b0;
        info->device_bytes = 4ull * (3 * nb + 3) * p.mmh.nprimes * (1ull << p.mmh.log2_len) +
                             4ull * 5 * p.mh.nprimes * (1ull << p.mh.log2_len);
    }
    return PA_OK;
}

static int mg_init(pa_ctx *c, const pa_params *prm);

extern "C" int pa_ctx_create_ex(const pa_params *prm, pa_ctx **out) {
    if (!out) return set_err(PA_E_PARAM, "out is NULL");
    *out = nullptr;
    Plan p;
    TRY(make_plan(prm, &p));
    pa_ctx *c = new (std::nothrow) pa_ctx();
    if (!c) return set_err(PA_E_NOMEM, "host allocation failed");
    c->pl = p;
    c->stream = (cudaStream_t)prm->stream;
    int rc = PA_OK;
    if (cudaGetDevice(&c->device) != cudaSuccess) rc = set_err(PA_E_CUDA, "no CUDA device");
    if (rc == PA_OK) {
        int nsm = 0;
        if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess || nsm <= 0)
            rc = set_err(PA_E_CUDA, "cudaDeviceGetAttribute(multiProcessorCount) failed");
        c->num_sms = g_num_sms = nsm;
    }
    c->da.stream = c->stream;
    c->da.fn_alloc = prm->dev_alloc;
    c->da.fn_free = prm->dev_free;
    c->da.user = prm->alloc_user;
    if (rc == PA_OK && (!prm->dev_alloc) != (!prm->dev_free)) rc = set_err(PA_E_PARAM, "dev_alloc and dev_free go together");
    if (rc == PA_OK) rc = ctx_alloc_and_precompute(c, prm);
    if (rc == PA_OK && p.world > 0) rc = mg_init(c, prm);
    if (rc != PA_OK) {
        cudaStreamSynchronize(c->stream);
        c->da.free_all();
        delete c;
        return rc;
    }
    *out = c;
    return PA_OK;
}

extern "C" pa_ctx *pa_ctx_create(uint64_t n, uint64_t r, uint64_t m, uint64_t p, uint64_t seed) {
    pa_params prm{};
    prm.n = n; prm.r = r; prm.m = m; prm.gamma = p; prm.seed = seed;
    pa_ctx *c = nullptr;
    if (pa_ctx_create_ex(&prm, &c) != PA_OK) return nullptr;
    return c;
}

extern "C" void pa_ctx_destroy(pa_ctx *c) {
    if (!c) return;
    DevGuard dg_(c);
    cudaStreamSynchronize(c->stream);
    if (c->p2p_region) {
        for (int q = 0; q < kMaxWorld; q++)
            if (c->p2p_peer[q] && c->p2p_peer[q] != c->p2p_region) cudaIpcCloseMemHandle(c->p2p_peer[q]);
        cudaFree(c->p2p_region);
    }
    for (auto &row : c->g_p2p_pre)
        for (auto &pair : row)
            for (GraphSlot &g : pair) g.reset();
    for (auto &pair : c->g_p2p_post)
        for (GraphSlot &g : pair) g.reset();
    if (c->comm) nccl_api().CommDestroy(c->comm);
    for (auto &r : c->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : c->evpool) cudaEventDestroy(e);
    for (GraphSlot *g : {&c->g_hash, &c->g_host, &c->g_batch, &c->g_mg_pre[0], &c->g_mg_pre[1], &c->g_mg_post[0],
                         &c->g_mg_post[1], &c->g_mg_host})
        g->reset();
    if (c->alt_ready) {
        cudaStreamSynchronize(c->alt.stream);
        cudaStreamDestroy(c->alt.stream);
        for (auto e : c->bev) cudaEventDestroy(e);
    }
    if (c->copy_stream) {
        cudaStreamSynchronize(c->copy_stream);
        for (auto e : c->copy_ev) if (e) cudaEventDestroy(e);
        cudaStreamDestroy(c->copy_stream);
    }
    for (auto e : c->hb_copy) if (e) cudaEventDestroy(e);
    for (auto e : c->hb_done) if (e) cudaEventDestroy(e);
    c->da.free_all();
    delete c;
}

// ---- fresh hash keys per job (NEXT-2): expand a_i, b, c from `seed` on the GPU (reading
// A7, bit-identical to pa_expand_a / pa_expand_bc) and recompute the transforms of the a_i
// and of b.  Asynchronous on the context stream; later hashes use the new function.
#ifndef PA_EXP_CTAS
#define PA_EXP_CTAS 8                              // expand_keys_first CTAs per SM (full occupancy)
#endif
extern "C" int pa_ctx_rekey(pa_ctx *c, uint64_t seed) {
    if (!c) return set_err(PA_E_PARAM, "NULL ctx");
    DevGuard dg_(c);
    if (c->pl.toeplitz) return set_err(PA_E_STATE, "rekey: not for the Toeplitz comparator");
    const Plan &p = c->pl;
    const uint32_t Wa32 = (uint32_t)cdiv(p.gamma, 32), Wal32 = (uint32_t)cdiv(p.alpha, 32);
    if (!c->a_words_dev) {
        TRY(c->da.alloc(&c->a_words_dev, std::max<size_t>((size_t)c->nblk * Wa32, 1)));
        TRY(c->da.alloc(&c->b_words_dev, Wal32));
        TRY(c->da.alloc(&c->rekey_ok, (size_t)c->nblk + 2));
    }
    c->g_hash.reset();
    const uint32_t launches0 = c->launches;
    c->launches = 0;
    {
        ProfScope ps(c, "rekey_expand");
        const uint32_t grid = (uint32_t)g_num_sms * PA_EXP_CTAS;
        if (c->nblk) {
            CUDA_TRY(cudaMemsetAsync(c->rekey_ok, 0, (size_t)c->nblk * 4, c->stream));
            expand_keys_first<<<grid, 256, 0, c->stream>>>(seed, p.b0, p.gamma, Wa32, c->nblk, 0, c->a_words_dev,
                                                           c->rekey_ok);
            expand_keys_dev<<<c->nblk, 256, 0, c->stream>>>(seed, p.b0, p.gamma, Wa32, 1, 0, c->a_words_dev, c->rekey_ok);
        }
        CUDA_TRY(cudaMemsetAsync(c->rekey_ok + c->nblk, 0, 8, c->stream));
        expand_keys_first<<<grid, 256, 0, c->stream>>>(seed, kStreamB, p.alpha, Wal32, 1, 1, c->b_words_dev,
                                                       c->rekey_ok + c->nblk);
        expand_keys_first<<<grid, 256, 0, c->stream>>>(seed, kStreamC, p.alpha, Wal32, 1, 0, c->c_words,
                                                       c->rekey_ok + c->nblk + 1);
        c->launches += c->nblk ? 4 : 2;
        CUDA_TRY(cudaGetLastError());
    }
    c->pl.seed = seed;
    int rc = PA_OK;
    {
        ProfScope ps(c, "rekey_transforms");
        if (c->nblk) {
            const uint32_t Bm = p.mmh.limb_bits;
            WordSrc wsa{c->a_words_dev, Wa32, Bm, (uint32_t)cdiv(p.gamma, Bm)};
            rc = precompute_hat(c, c->smmh, wsa, c->nblk, rows_for(cdiv(p.gamma, Bm), p.mmh.n_row, p.mmh.n_col),
                                c->scratch, c->ahat);
        }
        const uint32_t Bh = p.mh.limb_bits;
        WordSrc wsb{c->b_words_dev, Wal32, Bh, (uint32_t)cdiv(p.alpha, Bh)};
        if (rc == PA_OK)
            rc = precompute_hat(c, c->smh, wsb, 1, rows_for(cdiv(p.alpha, Bh), p.mh.n_row, p.mh.n_col), c->scratch_mh,
                                c->bhat);
        c->launches += 5 + (c->nblk ? 3 : 0);
    }
    c->launches_total += c->launches;
    c->launches = launches0;
    return rc;
}

extern "C" int pa_ctx_status(pa_ctx *c) {
    if (!c) return set_err(PA_E_PARAM, "NULL ctx");
    DevGuard dg_(c);
    uint32_t st = 0;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    CUDA_TRY(cudaMemcpy(&st, c->status, 4, cudaMemcpyDeviceToHost));
    if (st) return set_err(PA_E_INSUFFICIENT_INPUT, "paper mode: fewer than %llu windows of the key differ from 2^gamma - 1 (SPEC.md:74)",
                           (unsigned long long)c->pl.k);
    return PA_OK;
}

extern "C" int pa_ctx_paper_stats(pa_ctx *c, uint64_t *consumed_bits, uint64_t *rejected_windows) {
    if (!c) return set_err(PA_E_PARAM, "NULL ctx");
    DevGuard dg_(c);
    if (!c->pl.paper_k) return set_err(PA_E_STATE, "paper stats: not a paper-mode context");
    TRY(pa_ctx_status(c));                                   // synchronizes; insufficient input
    uint64_t last = 0;
    CUDA_TRY(cudaMemcpy(&last, c->offs + (c->pl.k - 1), 8, cudaMemcpyDeviceToHost));
    const uint64_t consumed = last + c->pl.gamma;
    if (consumed_bits) *consumed_bits = consumed;
    if (rejected_windows) *rejected_windows = consumed / c->pl.gamma - c->pl.k;
    return PA_OK;
}

extern "C" int pa_ctx_query(const pa_ctx *c, pa_info *info) {
    if (!c || !info) return set_err(PA_E_PARAM, "NULL argument");
    memset(info, 0, sizeof *info);
    const Plan &p = c->pl;
    info->n = p.n; info->r = p.r; info->m = p.m; info->gamma = p.gamma; info->alpha = p.alpha;
    info->k = p.k; info->block_begin = p.b0; info->block_end = p.b1;
    info->mmh = p.mmh; info->mh = p.mh;
    info->insecure_length = (!p.mh_only && !p.toeplitz && p.m >= p.gamma) ? 1u : 0u;
    info->world = p.world; info->rank = p.rank;
    info->acc_words = (p.mh_only || p.toeplitz) ? 0 : (uint64_t)p.mmh.nprimes << p.mmh.log2_len;
    info->device_bytes = c->da.bytes;
    info->graph_captures = c->graph_captures;
    info->graph_updates = c->graph_updates;
    info->graph_instantiations = c->graph_instantiations;
    info->p2p = c->p2p ? 1u : 0u;
    info->tz_group_blocks = p.toeplitz ? p.tz_group : 0u;
    info->kernels_per_hash = c->launches;
    info->launches_total = c->launches_total;
    return PA_OK;
}

extern "C" int pa_ctx_set_stream(pa_ctx *c, void *stream) {
    if (!c) return set_err(PA_E_PARAM, "NULL ctx");
    DevGuard dg_(c);
    for (GraphSlot *g : {&c->g_hash, &c->g_host, &c->g_batch, &c->g_mg_pre[0], &c->g_mg_pre[1], &c->g_mg_post[0],
                         &c->g_mg_post[1], &c->g_mg_host})
        g->reset();
    c->stream = (cudaStream_t)stream;
    c->da.stream = c->stream;
    return PA_OK;
}

// ---- S1-S5 on this ctx's blocks -> canonical y in the returned buffer (Wg words)
// key source of this ctx's blocks [v0, v1) (shard-relative), key_slice = the shard's bytes
static KeySrc key_src(const pa_ctx *c, const uint8_t *key_slice, uint32_t v0, uint32_t v1) {
    const Plan &p = c->pl;
    const uint64_t total_bytes = cdiv(p.n, 8);
    const uint64_t R = p.r / 8;
    const uint64_t off = (p.b0 + v0) * R;                       // global byte offset of block v0
    const uint64_t nbytes = std::min<uint64_t>(total_bytes - std::min(off, total_bytes), (uint64_t)(v1 - v0) * R);
    KeySrc ks{};
    ks.key = key_slice + (uint64_t)v0 * R;
    ks.nbytes = nbytes;
    const bool has_last = (off + nbytes == total_bytes);      // bits >= n ignored
    ks.last_mask = (has_last && (p.n % 8)) ? ((0xFFu << (8 - p.n % 8)) & 0xFFu) : 0xFFu;
    ks.blk_bytes = (uint32_t)R;
    ks.limb_bytes = p.mmh.limb_bits / 8;
    ks.wx = (uint32_t)cdiv(p.r, p.mmh.limb_bits);
    ks.aligned = (((uintptr_t)ks.key) & 3) == 0;
    return ks;
}

template <int NW>
static void launch_pack_bits(const KeySrc &s, const uint64_t *offs, uint32_t gamma, uint32_t B, uint32_t wx,
                             uint32_t nvec, const PrimeSet &pk, uint32_t P, uint32_t wxp, uint32_t *res, cudaStream_t st) {
    const dim3 grid((wxp + kPackL * kPackT - 1) / (kPackL * kPackT), nvec);
    pack_bits_residues<NW><<<grid, kPackT, 0, st>>>(s, offs, gamma, B, wx, pk, P, wxp, res);
}

// ---- paper mode S1: windows with a zero bit -> block offsets (reload rule), pack
static int paper_pack(pa_ctx *c, const uint8_t *key) {
    const Plan &p = c->pl;
    KeySrc ks{};
    ks.key = key;
    ks.nbytes = cdiv(p.n, 8);
    ks.last_mask = (p.n % 8) ? ((0xFFu << (8 - p.n % 8)) & 0xFFu) : 0xFFu;
    ks.aligned = (((uintptr_t)key) & 3) == 0;
    {
        ProfScope ps(c, "mmh_reload_windows");
        uint32_t *done = next_state(c);                     // zeroed by carry_reset
        if (!done) return set_err(PA_E_STATE, "carry slots exhausted");
        window_flags<<<c->T, 256, 0, c->stream>>>(ks, (uint32_t)p.gamma, c->T, c->wflags, done, (uint32_t)p.k, c->offs,
                                                  c->status);
        c->launches += 1;
        CUDA_TRY(cudaGetLastError());
    }
    ProfScope ps(c, "mmh_pack");
    const uint32_t B = p.mmh.limb_bits, P = p.mmh.nprimes;
    const uint32_t wx = (uint32_t)cdiv(p.gamma, B);
    const uint32_t wxp = c->rows_mmh * p.mmh.n_row;
    const int nw = (int)cdiv(B, 32);
    switch (nw) {
#define PA_PB(N) case N: launch_pack_bits<N>(ks, c->offs, (uint32_t)p.gamma, B, wx, c->nblk, c->smmh.pks, P, wxp, c->res, c->stream); break;
        PA_PB(1) PA_PB(2) PA_PB(3) PA_PB(4) PA_PB(5) PA_PB(6) PA_PB(7) PA_PB(8)
#undef PA_PB
        default: return set_err(PA_E_PARAM, "unsupported limb width %u", B);
    }
    c->launches++;
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

// ---- S1+S2 first pass for blocks [v0, v1) of the shard
static int mmh_forward(pa_ctx *c, const uint8_t *key_slice, uint32_t v0, uint32_t v1) {
    const uint32_t P = c->pl.mmh.nprimes;
    const size_t wxp = (size_t)c->rows_mmh * c->pl.mmh.n_row;
    if (c->pl.paper_k) {
        if (v0 != 0 || v1 != c->nblk) return set_err(PA_E_STATE, "paper mode hashes all blocks at once");
        TRY(paper_pack(c, key_slice));
        ProfScope ps(c, "mmh_fwd_col");
        ColArgs A{};
        A.nt = ntt_args(c->smmh, 0, 0);
        A.src = c->res;
        A.rows = c->rows_mmh;
        A.tw4 = c->smmh.tw4f;
        A.dst = c->scratch;
        A.nvec = c->nblk;
        A.units = (c->pl.mmh.n_row / 32) * P * c->nblk;
        TRY(launch_col<COL_FWD>(__builtin_ctz(c->pl.mmh.n_col), __builtin_ctz(c->pl.mmh.n_row), A, c->stream));
        c->launches++;
        return PA_OK;
    }
    return stage_pack_col(c, c->smmh, KeyLimbs{key_src(c, key_slice, v0, v1)}, v1 - v0, c->rows_mmh,
                          c->res + (size_t)v0 * P * wxp, c->scratch + (size_t)v0 * P * c->smmh.L, "mmh_pack",
                          "mmh_fwd_col");
}

static int mmh_mac(pa_ctx *c, uint32_t v0, uint32_t v1, bool first, bool only, bool zero = true) {
    const size_t off = (size_t)v0 * c->pl.mmh.nprimes * c->smmh.L;
    return stage_mac(c, c->smmh, v1 - v0, c->scratch + off, c->ahat + off, c->acc, first, "mmh_fwd_row_mac", only,
                     zero);
}

// ---- S4+S5 after all blocks are accumulated -> canonical y.  The accumulator is c->acc
// (c->mac_slots slots) unless src is given: nsrc slots src_stride words apart, each < 4p
// (the merged accumulators of several shards)
static int mmh_tail(pa_ctx *c, uint32_t **y_out, const uint32_t *src = nullptr, uint32_t nsrc = 0,
                    uint64_t src_stride = 0) {
    const Plan &p = c->pl;
    TRY(stage_inverse(c, c->smmh, c->acc, "mmh_inverse", src ? nsrc : c->mac_slots, src, src_stride));
    {
        ProfScope ps(c, "mmh_crt_carry_fold");
        TRY(launch_crt_carry<true>(c->acc, c->smmh, (uint32_t)c->ncoef_mmh, p.gamma, nullptr, 0, c->coef, c->y1,
                                   (uint32_t)c->W_fold, next_state(c), (uint32_t)c->W_fold, c->stream));
        c->launches += 2;
    }
    *y_out = c->y1;
    return PA_OK;
}

// ---- S1-S3 on this ctx's blocks -> transform-domain accumulator c->acc (c->mac_slots slots)
static int run_mmh_acc(pa_ctx *c, const uint8_t *key_slice) {
    // accumulators zeroed first: the chain pack -> col -> row_mac is back-to-back kernels
    {
        const uint32_t P = c->pl.mmh.nprimes;
        const int rlog = __builtin_ctz(c->pl.mmh.n_row);
        int grid = 0;
        uint32_t nslot = 1;
        TRY(mac_grid(rlog, (c->pl.mmh.n_col / mac_v_rt(rlog)) * P, c->nblk, 0, &grid, &nslot));
        CUDA_TRY(cudaMemsetAsync(c->acc, 0, (size_t)nslot * P * c->smmh.L * 4, c->stream));
    }
    TRY(mmh_forward(c, key_slice, 0, c->nblk));
    return mmh_mac(c, 0, c->nblk, true, true, false);
}

// ---- S1-S5 on this ctx's blocks -> canonical y in the returned buffer (Wg words)
static int run_mmh(pa_ctx *c, const uint8_t *key_slice, uint32_t **y_out) {
    TRY(run_mmh_acc(c, key_slice));
    return mmh_tail(c, y_out);
}

// ---- S7 on canonical y -> out_bits
#ifndef PA_MH_MACINV
#define PA_MH_MACINV 1            // fused single-vector row MAC + inverse row pass (row_macinv)
#endif
static int run_mh(pa_ctx *c, const uint32_t *y, uint8_t *out_bits) {
    const Plan &p = c->pl;
    const uint32_t Bh = p.mh.limb_bits;
    WordSrc ws{y, (uint32_t)c->Wg, Bh, (uint32_t)cdiv(p.gamma, Bh)};
    TRY(stage_pack_col(c, c->smh, WordLimbs{ws}, 1, c->rows_mh, c->res, c->scratch_mh, "mh_pack", "mh_fwd_col"));
#if PA_MH_MACINV
    TRY(stage_macinv(c, c->smh, c->scratch_mh, c->bhat, c->acc_mh, "mh_row_mac_inv", "mh_inverse_col"));
#else
    TRY(stage_mac(c, c->smh, 1, c->scratch_mh, c->bhat, c->acc_mh, true, "mh_fwd_row_mac", false));
    TRY(stage_inverse(c, c->smh, c->acc_mh, "mh_inverse"));
#endif
    const uint32_t W = (uint32_t)c->W_Z;
    {
        ProfScope ps(c, "mh_crt_carry_extract");
        // only (b y + c) mod 2^alpha is needed: coefficients j with j B >= alpha cannot reach it
        const uint64_t ncoef = std::min<uint64_t>(std::min<uint64_t>(c->smh.L, cdiv(p.alpha, Bh) + cdiv(p.gamma, Bh) - 1),
                                                  cdiv(p.alpha, Bh));
        // m = alpha, a whole number of words, aligned output: the carry kernel writes the
        // output bits itself (byte-swapped words in reverse order), no extract pass
        const bool direct = p.m == p.alpha && p.alpha % 32 == 0 && !((uintptr_t)out_bits & 3);
        TRY(launch_crt_carry<false>(c->acc_mh, c->smh, (uint32_t)ncoef, 0, c->c_words, W, c->coef, c->Z, W,
                                    next_state(c), 0, c->stream, direct ? reinterpret_cast<uint32_t *>(out_bits) : nullptr));
        c->launches += 2;
        if (!direct) {
            const uint64_t nb = cdiv(p.m, 8), nw = cdiv(nb, 4);
            mh_extract<<<(uint32_t)cdiv(nw, 256), 256, 0, c->stream>>>(c->Z, c->W_Z, p.alpha, p.m, out_bits, nb);
            c->launches++;
            CUDA_TRY(cudaGetLastError());
        }
    }
    return PA_OK;
}

static int hash_enqueue(pa_ctx *c, const uint8_t *key_bits, uint8_t *out_bits) {
    c->launches = 0;
    if (c->pl.toeplitz) return run_toeplitz(c, key_bits, out_bits);
    TRY(carry_reset(c));
    if (c->pl.mh_only) {
        // comparator: y := x, the n-bit key integer, then the MH stage with alpha = n
        KeySrc ks{};
        ks.key = key_bits;
        ks.nbytes = cdiv(c->pl.n, 8);
        ks.last_mask = (c->pl.n % 8) ? ((0xFFu << (8 - c->pl.n % 8)) & 0xFFu) : 0xFFu;
        ks.aligned = (((uintptr_t)key_bits) & 3) == 0;
        {
            ProfScope ps(c, "mh_only_key_words");
            key_to_words<<<(uint32_t)cdiv(c->Wg, 256), 256, 0, c->stream>>>(ks, c->pl.n, (uint32_t)c->Wg, c->y1);
            c->launches++;
            CUDA_TRY(cudaGetLastError());
        }
        return run_mh(c, c->y1, out_bits);
    }
    uint32_t *y = nullptr;
    TRY(run_mmh(c, key_bits, &y));
    return run_mh(c, y, out_bits);
}

// On a non-default stream (and without stage profiling) the ~20 launches of one hash are
// captured once into a CUDA graph per (key, out) pointer pair and replayed: no host
// launch overhead, no inter-kernel launch gaps.  PA_NO_GRAPH=1 disables it.
static bool graphs_enabled(const pa_ctx *c) {
#ifdef PA_DEBUG
    (void)c;
    return false;                         // the range table is uploaded per call
#endif
    static const bool off = getenv("PA_NO_GRAPH") && atoi(getenv("PA_NO_GRAPH"));
    return !off && c->stream != nullptr && !c->prof;
}

// End-to-end hash from host buffers.  The key is copied in kCopyGroups block groups on a
// copy stream; the pack, both forward passes and the multiply-accumulate of group g start
// as soon as group g has landed (stream-ordered by events), so the PCIe transfer overlaps
// the MMH transforms.
#ifndef PA_COPY_GROUPS
#define PA_COPY_GROUPS 8
#endif
static constexpr int kCopyGroups = PA_COPY_GROUPS;

// First block of copy group g of G: group sizes fall linearly (weights G, G-1, ..., 1), so the
// last group -- whose transforms are all that is left to do once the last byte has arrived --
// is the smallest (C4: 7, 6, 5, 4, 4, 2, 2, 1 blocks).  The H2D copy outruns nothing: the
// GPU finishes each group's transforms before the next group's bytes land.
#ifndef PA_COPY_GEOM
#define PA_COPY_GEOM 0        // 1: group sizes halve (weights 2^(G-1), ..., 2, 1) instead of falling linearly
#endif
static uint32_t group_begin(uint32_t nblk, int G, int g) {
#if PA_COPY_GEOM
    const uint64_t W = (1ull << G) - 1;
    uint64_t cum = 0;
    for (int i = 0; i < g; i++) cum += 1ull << (G - 1 - i);
    return (uint32_t)((nblk * cum + W / 2) / W);
#else
    const uint64_t W = (uint64_t)G * (G + 1) / 2;
    uint64_t cum = 0;
    for (int i = 0; i < g; i++) cum += (uint64_t)(G - i);
    return (uint32_t)((nblk * cum + W / 2) / W);
#endif
}

static int mg_hash(pa_ctx *c, const uint8_t *key, uint8_t *out, int root, int set, const uint8_t *key_host = nullptr);
static int mg_hash_p2p(pa_ctx *c, const uint8_t *key, uint8_t *out, int root, int set);
static int mg_hash_batch(pa_ctx *c, const uint8_t *const *keys, uint8_t *const *outs, uint32_t count);

// Enqueue `enqueue()` on the context stream through the graph slot `gs` (captured once per
// pointer key, updated in place for new pointers) or directly when graphs are off.
template <class F>
static int graph_run(pa_ctx *c, GraphSlot &gs, const std::vector<const void *> &key, F &&enqueue) {
    if (!graphs_enabled(c)) return enqueue();
    if (!gs.exec || key != gs.key) {
        cudaGraph_t g = nullptr;
        CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        const int rc = enqueue();
        const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
        if (rc != PA_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (e != cudaSuccess) return set_err(PA_E_CUDA, "graph capture failed: %s", cudaGetErrorString(e));
        c->graph_captures++;
        bool updated = false;
        if (gs.exec) {
            cudaGraphExecUpdateResultInfo info{};
            if (cudaGraphExecUpdate(gs.exec, g, &info) == cudaSuccess) {
                updated = true;
                c->graph_updates++;
            } else {
                cudaGetLastError();
                gs.reset();
            }
        }
        if (!updated) {
            const cudaError_t e2 = cudaGraphInstantiate(&gs.exec, g, 0);
            if (e2 != cudaSuccess) {
                gs.exec = nullptr;
                cudaGraphDestroy(g);
                return set_err(PA_E_CUDA, "graph instantiate failed: %s", cudaGetErrorString(e2));
            }
            c->graph_instantiations++;
        }
        cudaGraphDestroy(g);
        gs.key = key;
        gs.launches = c->launches;
    }
    CUDA_TRY(cudaGraphLaunch(gs.exec, c->stream));
    c->launches = gs.launches;
    return PA_OK;
}

// bytes of the key (slice) a call on this context reads
static uint64_t key_slice_len(const pa_ctx *c) {
    const Plan &p = c->pl;
    const uint64_t nb = cdiv(p.n, 8);
    if (p.paper_k || p.mh_only || p.toeplitz) return nb;
    const uint64_t R = p.r / 8;
    return std::min(p.b1 * R, nb) - std::min(p.b0 * R, nb);
}

extern "C" int pa_hash(pa_ctx *c, const uint8_t *key_bits, uint8_t *out_bits) {
    if (!c || !key_bits) return set_err(PA_E_PARAM, "NULL argument");
    DevGuard dg_(c);
    dbg_user({{key_bits, key_slice_len(c)}, {out_bits, cdiv(c->pl.m, 8)}});
    if (c->comm) return c->p2p ? mg_hash_p2p(c, key_bits, out_bits, 0, 0) : mg_hash(c, key_bits, out_bits, 0, 0);
    if (!out_bits) return set_err(PA_E_PARAM, "NULL argument");
    if (c->pl.b0 != 0 || c->pl.b1 != c->pl.k)
        return set_err(PA_E_STATE, "shard context: use pa_mmh_partial + pa_mh_merge or pa_mmh_acc + pa_tail_merge");
    const int rc = graph_run(c, c->g_hash, {key_bits, out_bits}, [&] { return hash_enqueue(c, key_bits, out_bits); });
    c->launches_total += c->launches;
    return rc;
}

extern "C" int pa_mmh_partial(pa_ctx *c, const uint8_t *key_slice, uint32_t *y_out) {
    if (!c || !key_slice || !y_out) return set_err(PA_E_PARAM, "NULL argument");
    DevGuard dg_(c);
    dbg_user({{key_slice, key_slice_len(c)}, {y_out, c->Wg * 4}});
    if (c->pl.mh_only || c->pl.toeplitz) return set_err(PA_E_STATE, "comparator context: use pa_hash");
    c->launches = 0;
    TRY(carry_reset(c));
    uint32_t *y = nullptr;
    const int rc = run_mmh(c, key_slice, &y);
    c->launches_total += c->launches;
    TRY(rc);
    CUDA_TRY(cudaMemcpyAsync(y_out, y, c->Wg * 4, cudaMemcpyDeviceToDevice, c->stream));
    return PA_OK;
}

extern "C" int pa_mh_merge(pa_ctx *c, const uint32_t *y_parts, uint32_t G, uint8_t *out_bits) {
    if (!c || !y_parts || !out_bits || G == 0) return set_err(PA_E_PARAM, "bad argument");
    DevGuard dg_(c);
    dbg_user({{y_parts, (uint64_t)G * c->Wg * 4}, {out_bits, cdiv(c->pl.m, 8)}});
    if (G > (1u << 24)) return set_err(PA_E_PARAM, "too many parts");
    if (c->pl.mh_only || c->pl.toeplitz) return set_err(PA_E_STATE, "comparator context: use pa_hash");
    c->launches = 0;
    TRY(carry_reset(c));
    int rc;
    {
        ProfScope ps(c, "merge_sum_fold");
        rc = run_carry(c, SrcParts{y_parts, G, (uint32_t)c->Wg}, (uint32_t)c->W_fold, c->y1);
        if (rc == PA_OK) rc = mersenne_finish(c, c->y1);
    }
    if (rc == PA_OK) rc = run_mh(c, c->y1, out_bits);
    c->launches_total += c->launches;
    return rc;
}

// ---- stream mode: `count` independent keys, hashed with the same
// function, alternately on two buffer sets / streams so that one key's latency-bound
// MH and tail kernels overlap the next key's MMH transforms.
static int alloc_alt(pa_ctx *c) {
    if (c->alt_ready) return PA_OK;
    const Plan &p = c->pl;
    const size_t Pm = p.mmh.nprimes, Lm = c->smmh.L, Ph = p.mh.nprimes, Lh = c->smh.L;
    HashBufs &b = c->alt;
    TRY(c->da.alloc(&b.res, c->res_words));
    TRY(c->da.alloc(&b.scratch, (size_t)c->nblk * Pm * Lm));
    TRY(c->da.alloc(&b.acc, (size_t)kMacSlots * Pm * Lm));
    TRY(c->da.alloc(&b.scratch_mh, Ph * Lh));
    TRY(c->da.alloc(&b.acc_mh, Ph * Lh));
    TRY(c->da.alloc(&b.S, std::max<uint64_t>(c->W_fold, c->W_Z)));
    TRY(c->da.alloc(&b.coef, std::max(Pm * Lm, Ph * Lh)));
    TRY(c->da.alloc(&b.y1, c->W_fold));
    TRY(c->da.alloc(&b.Z, c->W_Z));
    TRY(c->da.alloc(&b.cstate, (size_t)c->cstate_stride * kCarrySlots));
    CUDA_TRY(cudaStreamCreateWithFlags(&b.stream, cudaStreamNonBlocking));
    for (auto &e : c->bev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->alt_ready = true;
    return PA_OK;
}

static int batch_enqueue(pa_ctx *c, const uint8_t *const *keys, uint8_t *const *outs, uint32_t count) {
    // fork: the alternate stream starts after the work already on the ctx stream
    CUDA_TRY(cudaEventRecord(c->bev[0], c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->alt.stream, c->bev[0], 0));
    uint32_t total = 0;
    for (uint32_t j = 0; j < count; j++) {
        if (j & 1) swap_bufs(c);
        const int rc = hash_enqueue(c, keys[j], outs[j]);
        total += c->launches;
        if (j & 1) swap_bufs(c);
        TRY(rc);
    }
    // join
    CUDA_TRY(cudaEventRecord(c->bev[1], c->alt.stream));
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->bev[1], 0));
    c->launches = total;
    return PA_OK;
}

extern "C" int pa_hash_batch(pa_ctx *c, const uint8_t *const *keys, uint8_t *const *outs, uint32_t count) {
    if (!c || (count && (!keys || !outs))) return set_err(PA_E_PARAM, "NULL argument");
    DevGuard dg_(c);
    dbg_user({});
    for (uint32_t j = 0; j < count; j++) {
        dbg_user_add(keys[j], key_slice_len(c));
        dbg_user_add(outs[j], cdiv(c->pl.m, 8));
    }
    if (c->pl.mh_only || c->pl.toeplitz) return set_err(PA_E_STATE, "comparator context: use pa_hash");
    if (c->comm) return mg_hash_batch(c, keys, outs, count);
    if (c->pl.b0 != 0 || c->pl.b1 != c->pl.k) return set_err(PA_E_STATE, "shard context: use pa_mmh_partial + pa_mh_merge");
    for (uint32_t j = 0; j < count; j++)
        if (!keys[j] || !outs[j]) return set_err(PA_E_PARAM, "NULL key or output in batch");
    if (count == 0) return PA_OK;
    if (count == 1) return pa_hash(c, keys[0], outs[0]);
    TRY(alloc_alt(c));
    std::vector<const void *> ptrs;
    for (uint32_t j = 0; j < count; j++) { ptrs.push_back(keys[j]); ptrs.push_back(outs[j]); }
    const int rc = graph_run(c, c->g_batch, ptrs, [&] { return batch_enqueue(c, keys, outs, count); });
    c->launches_total += c->launches;
    return rc;
}

// ====================================================================== multi-GPU
// rank g hashes its blocks' S1-S3 into the transform-domain accumulator,
// the ranks' accumulators are summed by one ncclReduce to the key's root (MMH is linear over
// a partition of the blocks), and the root alone runs S4-S7.

// canonical export of the accumulator (c->mac_slots slots) into `dst` (u32 or u64 words)
static int launch_export(pa_ctx *c, void *dst, bool u64) {
    const uint64_t total = (uint64_t)c->pl.mmh.nprimes * c->smmh.L;
    const uint32_t grid = (uint32_t)std::min<uint64_t>(cdiv(total, 256), (uint64_t)g_num_sms * 8);
    const uint32_t lg = c->pl.mmh.log2_len;
    ProfScope ps(c, "mmh_acc_export");
    if (u64)
        acc_export<uint64_t><<<grid, 256, 0, c->stream>>>(c->acc, c->mac_slots, total, lg, total, c->smmh.pks,
                                                          static_cast<uint64_t *>(dst));
    else
        acc_export<uint32_t><<<grid, 256, 0, c->stream>>>(c->acc, c->mac_slots, total, lg, total, c->smmh.pks,
                                                          static_cast<uint32_t *>(dst));
    c->launches++;
    CUDA_TRY(cudaGetLastError());
    return PA_OK;
}

// S4-S7 from the reduced accumulator `recv` (u32 sums < 4p, or u64 sums converted into tmp32)
static int mg_post_enqueue(pa_ctx *c, const void *recv, uint32_t *tmp32, uint8_t *out) {
    c->launches = 0;
    TRY(carry_reset(c));
    const uint32_t *src = static_cast<const uint32_t *>(recv);
    if (c->x_u64) {
        const uint64_t total = (uint64_t)c->pl.mmh.nprimes * c->smmh.L;
        const uint32_t grid = (uint32_t)std::min<uint64_t>(cdiv(total, 256), (uint64_t)g_num_sms * 8);
        ProfScope ps(c, "mmh_acc_import");
        acc_import_u64<<<grid, 256, 0, c->stream>>>(static_cast<uint64_t *>(const_cast<void *>(recv)), c->pl.mmh.log2_len,
                                                     total, c->smmh.pks, tmp32);
        c->launches++;
        CUDA_TRY(cudaGetLastError());
        src = tmp32;
    }
    uint32_t *y = nullptr;
    TRY(mmh_tail(c, &y, src, 1, 0));
    return run_mh(c, y, out);
}

// one key on a multi-GPU context, reduced to and finished on `root`, with buffer set `set`
// (the caller has swapped the set in: c->acc, c->stream, ... are the set's)
// key_host (pa_hash_host, pinned memory): the slice is first copied into `key` in block groups on
// the copy stream, each group's transforms waiting only for its own bytes
static int mg_hash(pa_ctx *c, const uint8_t *key, uint8_t *out, int root, int set, const uint8_t *key_host) {
    const int rank = c->pl.rank;
    if (rank == root && !out) return set_err(PA_E_PARAM, "NULL output on the root rank");
    const uint64_t total = (uint64_t)c->pl.mmh.nprimes * c->smmh.L;
    uint32_t launched = 0;
    if (key_host) {
        TRY(graph_run(c, c->g_mg_host, {key_host, key}, [&] {
            c->launches = 0;
            const uint64_t sb = key_slice_len(c), R = c->pl.r / 8;
            const uint32_t nblk = c->nblk;
            const int G = (int)std::min<uint32_t>(kCopyGroups, nblk);
            uint8_t *kd = const_cast<uint8_t *>(key);
            CUDA_TRY(cudaEventRecord(c->copy_ev[kCopyGroups], c->stream));
            CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->copy_ev[kCopyGroups], 0));
            for (int g = 0; g < G; g++) {
                const uint64_t lo = std::min<uint64_t>(sb, (uint64_t)group_begin(nblk, G, g) * R);
                const uint64_t hi = g + 1 == G ? sb : std::min<uint64_t>(sb, (uint64_t)group_begin(nblk, G, g + 1) * R);
                if (hi > lo) CUDA_TRY(cudaMemcpyAsync(kd + lo, key_host + lo, hi - lo, cudaMemcpyHostToDevice, c->copy_stream));
                CUDA_TRY(cudaEventRecord(c->copy_ev[g], c->copy_stream));
            }
            bool first = true;
            for (int g = 0; g < G; g++) {
                const uint32_t v0 = group_begin(nblk, G, g), v1 = group_begin(nblk, G, g + 1);
                CUDA_TRY(cudaStreamWaitEvent(c->stream, c->copy_ev[g], 0));
                if (v1 > v0) TRY(mmh_forward(c, key, v0, v1));
                if (v1 > v0) TRY(mmh_mac(c, v0, v1, first, G == 1));
                if (v1 > v0) first = false;
            }
            return launch_export(c, c->xsend[set], c->x_u64);
        }));
    } else
    TRY(graph_run(c, c->g_mg_pre[set], {key}, [&] {
        c->launches = 0;
        TRY(run_mmh_acc(c, key));
        return launch_export(c, c->xsend[set], c->x_u64);
    }));
    launched += c->launches;
    {
        ProfScope ps(c, "mmh_nccl_reduce");
        NCCL_TRY(nccl_api().Reduce(c->xsend[set], c->xrecv[set], total, c->x_u64 ? ncclUint64 : ncclUint32, ncclSum,
                                   root, c->comm, c->stream));
    }
    if (rank == root) {
        TRY(graph_run(c, c->g_mg_post[set], {out}, [&] {
            return mg_post_enqueue(c, c->xrecv[set], static_cast<uint32_t *>(c->xsend[set]), out);
        }));
        launched += c->launches;
    }
    c->launches = launched;
    c->launches_total += launched;
    return PA_OK;
}

// ---- P2P exchange (pa_params.p2p; exchange.cuh).  Counter words of a region (each
// kFlagWords apart): FREE(q, s) -- root q's receive buffer s may take new sums (written by q);
// READY(s, r) -- rank r's sums for this GPU's buffer s are complete (written by r);
// EXPF / EXPR -- this GPU's "expected" companions of FREE / READY (local only).
enum { P2P_FREE = 0, P2P_READY = 2 * kMaxWorld, P2P_EXPF = 4 * kMaxWorld, P2P_EXPR = 6 * kMaxWorld,
       P2P_NFLAG = 8 * kMaxWorld };
static uint32_t *p2p_flag(uint8_t *region, size_t recv_bytes, uint32_t idx) {
    return reinterpret_cast<uint32_t *>(region + 2 * recv_bytes) + (size_t)idx * kFlagWords;
}

// one key on a P2P multi-GPU context, finished on `root`, hashing buffer set `set`
static int mg_hash_p2p(pa_ctx *c, const uint8_t *key, uint8_t *out, int root, int set) {
    const int rank = c->pl.rank, world = c->pl.world;
    if (rank == root && !out) return set_err(PA_E_PARAM, "NULL output on the root rank");
    const uint32_t s = c->p2p_uses[root]++ & 1u;         // receive buffer of this use of root's
    const size_t RB = c->p2p_recv_bytes;
    uint8_t *rreg = c->p2p_peer[root];
    auto *dst64 = reinterpret_cast<unsigned long long *>(rreg + s * RB);
    uint32_t launched = 0;
    // S1-S3: transforms, then (once root has freed buffer s) the row MAC adding into it over
    // NVLink, then READY(s, rank) += 1 on the root
    TRY(graph_run(c, c->g_p2p_pre[root][s][set], {key, c->scratch}, [&] {
        c->launches = 0;
        TRY(mmh_forward(c, key, 0, c->nblk));
        p2p_wait<<<1, 64, 0, c->stream>>>(p2p_flag(c->p2p_region, RB, P2P_FREE + 2 * root + s),
                                          p2p_flag(c->p2p_region, RB, P2P_EXPF + 2 * root + s), 1);
        CUDA_TRY(cudaGetLastError());
        const size_t off = 0;
        TRY(stage_mac(c, c->smmh, c->nblk, c->scratch + off, c->ahat + off, c->acc, true, "mmh_fwd_row_mac_p2p", true,
                      false, dst64));
        PeerFlags pf{};
        pf.p[0] = p2p_flag(rreg, RB, P2P_READY + s * kMaxWorld + rank);
        p2p_signal<<<1, 64, 0, c->stream>>>(pf, 1);
        CUDA_TRY(cudaGetLastError());
        c->launches += 2;
        return PA_OK;
    }));
    launched += c->launches;
    if (rank == root) {
        // every rank's sums in: import (mod each prime; the import zeroes the buffer), S4-S7,
        // FREE(rank, s) += 1 on every rank
        TRY(graph_run(c, c->g_p2p_post[s][set], {out, c->scratch}, [&] {
            c->launches = 0;
            TRY(carry_reset(c));
            p2p_wait<<<1, 64, 0, c->stream>>>(p2p_flag(c->p2p_region, RB, P2P_READY + s * kMaxWorld),
                                              p2p_flag(c->p2p_region, RB, P2P_EXPR + s * kMaxWorld), (uint32_t)world);
            CUDA_TRY(cudaGetLastError());
            const uint64_t total = (uint64_t)c->pl.mmh.nprimes * c->smmh.L;
            const uint32_t grid = (uint32_t)std::min<uint64_t>(cdiv(total, 256), (uint64_t)g_num_sms * 8);
            {
                ProfScope ps(c, "mmh_acc_import");
                acc_import_u64<true><<<grid, 256, 0, c->stream>>>(reinterpret_cast<uint64_t *>(c->p2p_region + s * RB),
                                                                   c->pl.mmh.log2_len, total, c->smmh.pks, c->p2p_tmp[set]);
                CUDA_TRY(cudaGetLastError());
            }
            PeerFlags pf{};
            for (int r = 0; r < world; r++) pf.p[r] = p2p_flag(c->p2p_peer[r], RB, P2P_FREE + 2 * rank + s);
            p2p_signal<<<1, 64, 0, c->stream>>>(pf, (uint32_t)world);
            CUDA_TRY(cudaGetLastError());
            c->launches += 3;
            uint32_t *y = nullptr;
            TRY(mmh_tail(c, &y, c->p2p_tmp[set], 1, 0));
            return run_mh(c, y, out);
        }));
        launched += c->launches;
    }
    c->launches = launched;
    c->launches_total += launched;
    return PA_OK;
}

// P2P setup (collective, after the communicator exists): region, IPC handles all-gathered
// over NCCL, peers mapped, FREE counters primed; a final all-gather is the barrier after which
// any rank may signal any other
static int p2p_init(pa_ctx *c) {
    const int world = c->pl.world, rank = c->pl.rank;
    if (world > kMaxWorld) return set_err(PA_E_PARAM, "p2p: world %d > %d", world, kMaxWorld);
    NcclApi &api = nccl_api();
    const size_t total = (size_t)c->pl.mmh.nprimes * c->smmh.L;
    c->p2p_recv_bytes = (total * 8 + 4095) & ~(size_t)4095;
    const size_t bytes = 2 * c->p2p_recv_bytes + (size_t)P2P_NFLAG * kFlagWords * 4;
    CUDA_TRY(cudaMalloc(&c->p2p_region, bytes));
    dbg_add(c->p2p_region, bytes);
    TRY(c->da.alloc(&c->p2p_tmp[0], total));
    TRY(c->da.alloc(&c->p2p_tmp[1], total));
    CUDA_TRY(cudaMemsetAsync(c->p2p_region, 0, bytes, c->stream));
    std::vector<uint32_t> one(2 * kMaxWorld * kFlagWords, 0);
    for (int i = 0; i < 2 * kMaxWorld; i++) one[(size_t)i * kFlagWords] = 1u;   // every buffer free for use 1
    CUDA_TRY(cudaMemcpyAsync(p2p_flag(c->p2p_region, c->p2p_recv_bytes, P2P_FREE), one.data(), one.size() * 4,
                             cudaMemcpyHostToDevice, c->stream));
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, c->p2p_region));
    uint8_t *hb = nullptr;
    TRY(c->da.alloc(&hb, (size_t)world * sizeof h));
    CUDA_TRY(cudaMemcpyAsync(hb + (size_t)rank * sizeof h, &h, sizeof h, cudaMemcpyHostToDevice, c->stream));
    NCCL_TRY(api.AllGather(hb + (size_t)rank * sizeof h, hb, sizeof h, ncclUint8, c->comm, c->stream));
    std::vector<cudaIpcMemHandle_t> all(world);
    CUDA_TRY(cudaMemcpyAsync(all.data(), hb, (size_t)world * sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    for (int q = 0; q < world; q++) {
        if (q == rank) { c->p2p_peer[q] = c->p2p_region; continue; }
        void *ptr = nullptr;
        CUDA_TRY(cudaIpcOpenMemHandle(&ptr, all[q], cudaIpcMemLazyEnablePeerAccess));
        c->p2p_peer[q] = static_cast<uint8_t *>(ptr);
        dbg_add(ptr, bytes);
    }
    // barrier: every rank has primed its counters and mapped its peers
    NCCL_TRY(api.AllGather(hb + (size_t)rank * sizeof h, hb, sizeof h, ncclUint8, c->comm, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->p2p = true;
    return PA_OK;
}

// stream of keys with the root rotating (key j on rank j mod world), alternating buffer sets
// and streams so key j's reduce and tail overlap key j+1's transforms
static int mg_hash_batch(pa_ctx *c, const uint8_t *const *keys, uint8_t *const *outs, uint32_t count) {
    const int world = c->pl.world, rank = c->pl.rank;
    for (uint32_t j = 0; j < count; j++) {
        if (!keys[j]) return set_err(PA_E_PARAM, "NULL key in batch");
        if ((int)(j % world) == rank && !outs[j]) return set_err(PA_E_PARAM, "NULL output of a key this rank is root of");
    }
    if (count == 0) return PA_OK;
    TRY(alloc_alt(c));
    CUDA_TRY(cudaEventRecord(c->bev[0], c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->alt.stream, c->bev[0], 0));
    uint32_t total = 0;
    for (uint32_t j = 0; j < count; j++) {
        const int set = (int)(j & 1);
        if (set) swap_bufs(c);
        const int rc = c->p2p ? mg_hash_p2p(c, keys[j], outs[j], (int)(j % world), set)
                              : mg_hash(c, keys[j], outs[j], (int)(j % world), set);
        total += c->launches;
        if (set) swap_bufs(c);
        TRY(rc);
    }
    CUDA_TRY(cudaEventRecord(c->bev[1], c->alt.stream));
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->bev[1], 0));
    c->launches = total;
    return PA_OK;
}

// NCCL communicator and exchange buffers of a multi-GPU context (collective: blocks until
// every rank of the job has joined)
static int mg_init(pa_ctx *c, const pa_params *prm) {
    NcclApi &api = nccl_api();
    if (!api.ok) return set_err(PA_E_NCCL, "NCCL unavailable: %s", api.why);
    uint32_t qmax = 0;
    for (uint32_t i = 0; i < c->pl.mmh.nprimes; i++) qmax = std::max(qmax, c->pl.mmh.primes[i]);
    // u32 sums must stay below 4 q (the inverse row pass reduces its input from [0, 4q))
    c->x_u64 = c->pl.world > 4 || (uint64_t)c->pl.world * (qmax - 1) >= (1ull << 32);
    // test knob: take the 64-bit exchange (the world > 4 path) on any world size
    if (const char *e = getenv("PA_FORCE_X64")) c->x_u64 = c->x_u64 || atoi(e) != 0;
    const size_t total = (size_t)c->pl.mmh.nprimes * c->smmh.L;
    for (int s = 0; s < 2; s++) {
        // u64 buffers also hold the u32 conversion on the root (tmp32 = xsend)
        if (c->x_u64) {
            uint64_t *a, *b;
            TRY(c->da.alloc(&a, total));
            TRY(c->da.alloc(&b, total));
            c->xsend[s] = a;
            c->xrecv[s] = b;
        } else {
            uint32_t *a, *b;
            TRY(c->da.alloc(&a, total));
            TRY(c->da.alloc(&b, total));
            c->xsend[s] = a;
            c->xrecv[s] = b;
        }
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    ncclUniqueId id;
    static_assert(sizeof id.internal == sizeof prm->nccl_id, "ncclUniqueId size");
    memcpy(id.internal, prm->nccl_id, sizeof id.internal);
    NCCL_TRY(api.CommInitRank(&c->comm, c->pl.world, id, c->pl.rank));
    if (prm->p2p) TRY(p2p_init(c));
    return PA_OK;
}

extern "C" int pa_abi_sizes(uint64_t *params_bytes, uint64_t *info_bytes) {
    if (params_bytes) *params_bytes = sizeof(pa_params);
    if (info_bytes) *info_bytes = sizeof(pa_info);
    return PA_OK;
}

extern "C" int pa_nccl_unique_id(uint8_t *id_out) {
    if (!id_out) return set_err(PA_E_PARAM, "NULL argument");
    NcclApi &api = nccl_api();
    if (!api.ok) return set_err(PA_E_NCCL, "NCCL unavailable: %s", api.why);
    ncclUniqueId id;
    NCCL_TRY(api.GetUniqueId(&id));
    memcpy(id_out, id.internal, sizeof id.internal);
    return PA_OK;
}

// ---- transform-domain split with a caller-side exchange (include/pa.h)
extern "C" int pa_mmh_acc(pa_ctx *c, const uint8_t *key_slice, uint32_t *acc_out) {
    if (!c || !key_slice || !acc_out) return set_err(PA_E_PARAM, "NULL argument");
    DevGuard dg_(c);
    dbg_user({{key_slice, key_slice_len(c)}, {acc_out, 4ull * c->pl.mmh.nprimes * c->smmh.L}});
    if (c->pl.mh_only || c->pl.toeplitz || c->pl.paper_k) return set_err(PA_E_STATE, "r-bit MMH-MH contexts only");
    c->launches = 0;
    int rc = run_mmh_acc(c, key_slice);
    if (rc == PA_OK) rc = launch_export(c, acc_out, false);
    c->launches_total += c->launches;
    return rc;
}

extern "C" int pa_tail_merge(pa_ctx *c, const uint32_t *acc_parts, uint32_t G, uint8_t *out_bits) {
    if (!c || !acc_parts || !out_bits || G == 0) return set_err(PA_E_PARAM, "bad argument");
    DevGuard dg_(c);
    dbg_user({{acc_parts, 4ull * G * c->pl.mmh.nprimes * c->smmh.L}, {out_bits, cdiv(c->pl.m, 8)}});
    if (c->pl.mh_only || c->pl.toeplitz || c->pl.paper_k) return set_err(PA_E_STATE, "r-bit MMH-MH contexts only");
    if (G > 4096) return set_err(PA_E_PARAM, "too many parts");
    c->launches = 0;
    int rc = carry_reset(c);
    uint32_t *y = nullptr;
    if (rc == PA_OK) rc = mmh_tail(c, &y, acc_parts, G, (uint64_t)c->pl.mmh.nprimes * c->smmh.L);
    if (rc == PA_OK) rc = run_mh(c, y, out_bits);
    c->launches_total += c->launches;
    return rc;
}

static int grouped_copy_hash(pa_ctx *c, const uint8_t *key_host, uint8_t *key_dev, uint8_t *out_dev,
                             uint8_t *out_host) {
    // copy_stream is already ordered after every earlier user of key_dev
    const uint64_t nb = cdiv(c->pl.n, 8), mb = cdiv(c->pl.m, 8);
    const uint32_t nblk = c->nblk;
    const int G = (int)std::min<uint32_t>(kCopyGroups, nblk);
    const uint64_t R = c->pl.r / 8;
    for (int g = 0; g < G; g++) {
        const uint64_t lo = G == 1 ? 0 : std::min<uint64_t>(nb, (uint64_t)group_begin(nblk, G, g) * R);
        const uint64_t hi = G == 1 ? nb : std::min<uint64_t>(nb, (uint64_t)group_begin(nblk, G, g + 1) * R);
        if (hi > lo) CUDA_TRY(cudaMemcpyAsync(key_dev + lo, key_host + lo, hi - lo, cudaMemcpyHostToDevice, c->copy_stream));
        CUDA_TRY(cudaEventRecord(c->copy_ev[g], c->copy_stream));
    }
    c->launches = 0;
    TRY(carry_reset(c));
    bool first = true;
    for (int g = 0; g < G; g++) {
        const uint32_t v0 = group_begin(nblk, G, g), v1 = group_begin(nblk, G, g + 1);
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->copy_ev[g], 0));
        if (v1 > v0) TRY(mmh_forward(c, key_dev, v0, v1));
        if (v1 > v0) TRY(mmh_mac(c, v0, v1, first, G == 1));
        first = false;
    }
    uint32_t *y = nullptr;
    TRY(mmh_tail(c, &y));
    TRY(run_mh(c, y, out_dev));
    CUDA_TRY(cudaMemcpyAsync(out_host, out_dev, mb, cudaMemcpyDeviceToHost, c->stream));
    return PA_OK;
}

static int hash_host_enqueue(pa_ctx *c, const uint8_t *key_host, uint8_t *out_host) {
    const uint64_t nb = cdiv(c->pl.n, 8), mb = cdiv(c->pl.m, 8);
    // the copies may overwrite key_dev only after earlier work on the ctx stream is done
    CUDA_TRY(cudaEventRecord(c->copy_ev[kCopyGroups], c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->copy_ev[kCopyGroups], 0));
    // paper mode: the reload rule needs the whole key before any block offset is known;
    // MH-only: one product over the whole key
    const bool whole = c->pl.paper_k || c->pl.mh_only || c->pl.toeplitz;
    if (whole) {
        CUDA_TRY(cudaMemcpyAsync(c->key_dev, key_host, nb, cudaMemcpyHostToDevice, c->copy_stream));
        CUDA_TRY(cudaEventRecord(c->copy_ev[0], c->copy_stream));
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->copy_ev[0], 0));
        TRY(hash_enqueue(c, c->key_dev, c->out_dev));
        CUDA_TRY(cudaMemcpyAsync(out_host, c->out_dev, mb, cudaMemcpyDeviceToHost, c->stream));
        return PA_OK;
    }
    return grouped_copy_hash(c, key_host, c->key_dev, c->out_dev, out_host);
}

// page-locked (cudaHostAlloc / cudaHostRegister) host memory?
static bool host_pinned(const void *p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();                               // clear the sticky-free error state
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// The synchronous host-buffer calls poll rather than block, so their return does not wait on
// a thread wake-up (cudaStreamSynchronize may yield under the default scheduling heuristic).
static int stream_poll(cudaStream_t st, const char *what) {
    cudaError_t q;
    while ((q = cudaStreamQuery(st)) == cudaErrorNotReady) { }
    if (q != cudaSuccess) return set_err(PA_E_CUDA, "%s: %s", what, cudaGetErrorString(q));
    return PA_OK;
}

extern "C" int pa_hash_host(pa_ctx *c, const uint8_t *key_host, uint8_t *out_host) {
    if (!c || !key_host) return set_err(PA_E_PARAM, "NULL argument");
    DevGuard dg_(c);
    const uint64_t nb = cdiv(c->pl.n, 8), mb = cdiv(c->pl.m, 8);
    if (c->comm) {
        // multi-GPU context: every rank copies in its own key slice over its own host link,
        // the ranks' accumulators are merged as in pa_hash, the root (rank 0) copies the output back
        const uint64_t sb = key_slice_len(c);
        const bool root = c->pl.rank == 0;
        if (root && !out_host) return set_err(PA_E_PARAM, "NULL output on the root rank");
        if (!c->key_dev) TRY(c->da.alloc(&c->key_dev, std::max<uint64_t>(sb, 1)));
        if (root && !c->out_dev) TRY(c->da.alloc(&c->out_dev, mb));
        if (!c->p2p && c->nblk > 0 && host_pinned(key_host)) {
            // pinned slice, NCCL reduce: the slice is copied in block groups on the copy stream and
            // each group's transforms start as it lands (grouped_copy_hash's scheme), captured
            // with the export as one graph
            if (!c->copy_stream) {
                CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
                for (int g = 0; g < kCopyGroups + 1; g++) CUDA_TRY(cudaEventCreateWithFlags(&c->copy_ev[g], cudaEventDisableTiming));
            }
            TRY(mg_hash(c, c->key_dev, root ? c->out_dev : nullptr, 0, 0, key_host));
        } else {
            // pageable memory (its copies synchronise, so they stay outside the graphs) or the
            // peer-memory exchange: one copy, then the device path
            if (sb) CUDA_TRY(cudaMemcpyAsync(c->key_dev, key_host, sb, cudaMemcpyHostToDevice, c->stream));
            TRY(c->p2p ? mg_hash_p2p(c, c->key_dev, root ? c->out_dev : nullptr, 0, 0)
                       : mg_hash(c, c->key_dev, root ? c->out_dev : nullptr, 0, 0));
        }
        if (root) CUDA_TRY(cudaMemcpyAsync(out_host, c->out_dev, mb, cudaMemcpyDeviceToHost, c->stream));
        TRY(stream_poll(c->stream, "pa_hash_host"));
        return PA_OK;
    }
    if (!out_host) return set_err(PA_E_PARAM, "NULL argument");
    if (c->pl.b0 != 0 || c->pl.b1 != c->pl.k) return set_err(PA_E_STATE, "shard context: use pa_mmh_partial + pa_mh_merge");
    if (!c->key_dev) TRY(c->da.alloc(&c->key_dev, nb));
    if (!c->out_dev) TRY(c->da.alloc(&c->out_dev, mb));
    if (!c->copy_stream) {
        CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        for (int g = 0; g < kCopyGroups + 1; g++) CUDA_TRY(cudaEventCreateWithFlags(&c->copy_ev[g], cudaEventDisableTiming));
    }
    // copies from / to pageable host memory synchronise with the host, which stream capture
    // forbids: such buffers take the direct (uncaptured) path
    if (!host_pinned(key_host) || !host_pinned(out_host)) {
        const int rc = hash_host_enqueue(c, key_host, out_host);
        c->launches_total += c->launches;
        TRY(rc);
    } else {
        const int rc = graph_run(c, c->g_host, {key_host, out_host}, [&] { return hash_host_enqueue(c, key_host, out_host); });
        c->launches_total += c->launches;
        TRY(rc);
    }
    TRY(stream_poll(c->stream, "pa_hash_host"));
    if (c->pl.paper_k) return pa_ctx_status(c);
    return PA_OK;
}

// ---- end-to-end stream mode: host-resident keys.  Key j's H2D (copy stream, into staging
// buffer j % 2) overlaps the hash of key j - 1 (buffer set / stream (j - 1) % 2); the copy
// of key j waits for the hash of key j - 2 (same staging buffer) to finish; the output of
// key j is copied back on its hash stream.  Synchronous: returns after the last D2H.
// End-to-end stream mode on a multi-GPU context: key j's slice goes host -> device on this
// rank's copy stream (staging buffer j % 2) while key j - 1 is hashed; the root rotates as in
// pa_hash_batch (key j is merged and finished on rank j mod world, which copies its output back).
static int mg_hash_host_batch(pa_ctx *c, const uint8_t *const *keys_host, uint8_t *const *outs_host, uint32_t count) {
    const int world = c->pl.world, rank = c->pl.rank;
    for (uint32_t j = 0; j < count; j++) {
        if (!keys_host[j]) return set_err(PA_E_PARAM, "NULL key in batch");
        if ((int)(j % world) == rank && !outs_host[j]) return set_err(PA_E_PARAM, "NULL output of a key this rank is root of");
    }
    if (count == 0) return PA_OK;
    const uint64_t sb = key_slice_len(c), mb = cdiv(c->pl.m, 8);
    if (!c->key_dev) TRY(c->da.alloc(&c->key_dev, std::max<uint64_t>(sb, 1)));
    if (!c->key_dev2) TRY(c->da.alloc(&c->key_dev2, std::max<uint64_t>(sb, 1)));
    if (!c->out_dev) TRY(c->da.alloc(&c->out_dev, mb));
    if (!c->out_dev2) TRY(c->da.alloc(&c->out_dev2, mb));
    if (!c->copy_stream) {
        CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        for (int g = 0; g < kCopyGroups + 1; g++) CUDA_TRY(cudaEventCreateWithFlags(&c->copy_ev[g], cudaEventDisableTiming));
    }
    if (!c->hb_copy[0])
        for (int s = 0; s < 2; s++) {
            CUDA_TRY(cudaEventCreateWithFlags(&c->hb_copy[s], cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&c->hb_done[s], cudaEventDisableTiming));
        }
    TRY(alloc_alt(c));
    uint8_t *kbuf[2] = {c->key_dev, c->key_dev2}, *obuf[2] = {c->out_dev, c->out_dev2};
    CUDA_TRY(cudaEventRecord(c->bev[0], c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->alt.stream, c->bev[0], 0));
    CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->bev[0], 0));
    uint32_t total = 0;
    int rc = PA_OK;
    for (uint32_t j = 0; j < count && rc == PA_OK; j++) {
        const int s = (int)(j & 1), root = (int)(j % world);
        if (j >= 2 && cudaStreamWaitEvent(c->copy_stream, c->hb_done[s], 0) != cudaSuccess) rc = set_err(PA_E_CUDA, "event wait failed");
        if (rc == PA_OK && sb && cudaMemcpyAsync(kbuf[s], keys_host[j], sb, cudaMemcpyHostToDevice, c->copy_stream) != cudaSuccess)
            rc = set_err(PA_E_CUDA, "H2D copy failed");
        if (rc == PA_OK && cudaEventRecord(c->hb_copy[s], c->copy_stream) != cudaSuccess) rc = set_err(PA_E_CUDA, "event record failed");
        if (rc != PA_OK) break;
        if (s) swap_bufs(c);
        if (cudaStreamWaitEvent(c->stream, c->hb_copy[s], 0) != cudaSuccess) rc = set_err(PA_E_CUDA, "event wait failed");
        if (rc == PA_OK)
            rc = c->p2p ? mg_hash_p2p(c, kbuf[s], root == rank ? obuf[s] : nullptr, root, s)
                        : mg_hash(c, kbuf[s], root == rank ? obuf[s] : nullptr, root, s);
        total += c->launches;
        if (rc == PA_OK && root == rank &&
            cudaMemcpyAsync(outs_host[j], obuf[s], mb, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
            rc = set_err(PA_E_CUDA, "D2H copy failed");
        if (rc == PA_OK && cudaEventRecord(c->hb_done[s], c->stream) != cudaSuccess) rc = set_err(PA_E_CUDA, "event record failed");
        if (s) swap_bufs(c);
    }
    CUDA_TRY(cudaEventRecord(c->bev[1], c->alt.stream));
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->bev[1], 0));
    c->launches = total;
    TRY(rc);
    return stream_poll(c->stream, "pa_hash_host_batch");
}

extern "C" int pa_hash_host_batch(pa_ctx *c, const uint8_t *const *keys_host, uint8_t *const *outs_host,
                                  uint32_t count) {
    if (!c || (count && (!keys_host || !outs_host))) return set_err(PA_E_PARAM, "NULL argument");
    DevGuard dg_(c);
    if (c->comm) return mg_hash_host_batch(c, keys_host, outs_host, count);
    if (c->pl.b0 != 0 || c->pl.b1 != c->pl.k) return set_err(PA_E_STATE, "shard context: use pa_mmh_partial + pa_mh_merge");
    if (c->pl.paper_k || c->pl.mh_only || c->pl.toeplitz)
        return set_err(PA_E_STATE, "paper mode / comparators: use pa_hash_host per key");
    for (uint32_t j = 0; j < count; j++)
        if (!keys_host[j] || !outs_host[j]) return set_err(PA_E_PARAM, "NULL key or output in batch");
    if (count == 0) return PA_OK;
    const uint64_t nb = cdiv(c->pl.n, 8), mb = cdiv(c->pl.m, 8);
    if (!c->key_dev) TRY(c->da.alloc(&c->key_dev, nb));
    if (!c->out_dev) TRY(c->da.alloc(&c->out_dev, mb));
    if (!c->key_dev2) TRY(c->da.alloc(&c->key_dev2, nb));
    if (!c->out_dev2) TRY(c->da.alloc(&c->out_dev2, mb));
    if (!c->copy_stream) {
        CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        for (int g = 0; g < kCopyGroups + 1; g++) CUDA_TRY(cudaEventCreateWithFlags(&c->copy_ev[g], cudaEventDisableTiming));
    }
    if (!c->hb_copy[0])
        for (int s = 0; s < 2; s++) {
            CUDA_TRY(cudaEventCreateWithFlags(&c->hb_copy[s], cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&c->hb_done[s], cudaEventDisableTiming));
        }
    TRY(alloc_alt(c));
    uint8_t *kbuf[2] = {c->key_dev, c->key_dev2}, *obuf[2] = {c->out_dev, c->out_dev2};
    // fork: both hash streams and the copy stream start after prior ctx-stream work
    CUDA_TRY(cudaEventRecord(c->bev[0], c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->alt.stream, c->bev[0], 0));
    CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->bev[0], 0));
    uint32_t total = 0;
    int rc = PA_OK;
    for (uint32_t j = 0; j < count && rc == PA_OK; j++) {
        const int s = (int)(j & 1);
        if (j >= 2 && cudaStreamWaitEvent(c->copy_stream, c->hb_done[s], 0) != cudaSuccess) rc = set_err(PA_E_CUDA, "event wait failed");
        if (rc != PA_OK) break;
        if (j + 1 == count) {
            // the last key: copied in block groups, its transforms starting as groups land, so
            // only the last group's work, the tails and the D2H follow the last byte (the drain)
            if (s) swap_bufs(c);
            rc = grouped_copy_hash(c, keys_host[j], kbuf[s], obuf[s], outs_host[j]);
            total += c->launches;
            if (s) swap_bufs(c);
            break;
        }
        if (rc == PA_OK && cudaMemcpyAsync(kbuf[s], keys_host[j], nb, cudaMemcpyHostToDevice, c->copy_stream) != cudaSuccess)
            rc = set_err(PA_E_CUDA, "H2D copy failed");
        if (rc == PA_OK && cudaEventRecord(c->hb_copy[s], c->copy_stream) != cudaSuccess) rc = set_err(PA_E_CUDA, "event record failed");
        if (rc != PA_OK) break;
        if (s) swap_bufs(c);
        if (cudaStreamWaitEvent(c->stream, c->hb_copy[s], 0) != cudaSuccess) rc = set_err(PA_E_CUDA, "event wait failed");
        if (rc == PA_OK) rc = hash_enqueue(c, kbuf[s], obuf[s]);
        total += c->launches;
        if (rc == PA_OK && cudaMemcpyAsync(outs_host[j], obuf[s], mb, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
            rc = set_err(PA_E_CUDA, "D2H copy failed");
        if (rc == PA_OK && cudaEventRecord(c->hb_done[s], c->stream) != cudaSuccess) rc = set_err(PA_E_CUDA, "event record failed");
        if (s) swap_bufs(c);
    }
    // join
    CUDA_TRY(cudaEventRecord(c->bev[1], c->alt.stream));
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->bev[1], 0));
    c->launches = total;
    c->launches_total += total;
    TRY(rc);
    return stream_poll(c->stream, "pa_hash_host_batch");
}

extern "C" int pa_ctx_set_profiling(pa_ctx *c, int enable) {
    if (!c) return set_err(PA_E_PARAM, "NULL ctx");
    DevGuard dg_(c);
    c->prof = enable != 0;
    return PA_OK;
}

extern "C" int pa_ctx_stage_times(pa_ctx *c, const char **names, double *ms, uint32_t *launches, int max) {
    if (!c) return set_err(PA_E_PARAM, "NULL ctx");
    DevGuard dg_(c);
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    for (auto &r : c->recs) {
        float t = 0;
        cudaEventElapsedTime(&t, r.a, r.b);
        auto &slot = c->acc_ms[r.name];
        slot.first += t;
        slot.second += 1;
        c->evpool.push_back(r.a);
        c->evpool.push_back(r.b);
    }
    c->recs.clear();
    if (max < 0) { c->acc_ms.clear(); return 0; }
    int i = 0;
    for (auto &kv : c->acc_ms) {
        if (i >= max) break;
        if (names) names[i] = kv.first.c_str();   // map keys: stable while the ctx lives
        if (ms) ms[i] = kv.second.first;
        if (launches) launches[i] = kv.second.second;
        i++;
    }
    return i;
}

// ---------------------------------------------------------------- host helpers
extern "C" int pa_philox4x64_10(uint64_t key0, uint64_t key1, uint64_t nwords, uint64_t *out) {
    if (!out && nwords) return set_err(PA_E_PARAM, "NULL out");
    Philox4x64::words(key0, key1, 0, nwords, out);
    return PA_OK;
}

extern "C" int pa_expand_a(uint64_t seed, uint64_t i, uint64_t gamma, uint32_t *out) {
    if (!out || !gamma) return set_err(PA_E_PARAM, "bad argument");
    std::vector<uint32_t> w;
    TRY(expand_words(seed, i, gamma, w, true));
    memcpy(out, w.data(), w.size() * 4);
    return PA_OK;
}

extern "C" int pa_derive_security_coefficient(double epsilon, uint64_t *s) {
    if (!(epsilon > 0.0 && epsilon < 1.0) || !s) return set_err(PA_E_PARAM, "epsilon must be in (0, 1)");
    // smallest integer s >= 1 with 2^(-s/2 - 1) <= epsilon, i.e. s >= 2 log2(1/epsilon) - 2;
    // the 1e-9 slack keeps exact powers (epsilon = 2^-j) from rounding up
    const double x = 2.0 * std::log2(1.0 / epsilon) - 2.0;
    const double c = std::ceil(x - 1e-9);
    *s = c < 1.0 ? 1 : (uint64_t)c;
    return PA_OK;
}

extern "C" int pa_select_block_count(double ratio, uint64_t *k) {
    if (!(ratio > 0.0 && ratio < 1.0) || !k) return set_err(PA_E_PARAM, "compression ratio must be in (0, 1)");
    *k = (uint64_t)std::floor(1.0 / ratio + 1e-12);
    return PA_OK;
}

extern "C" int pa_select_gamma(uint64_t target_n, uint64_t k, uint64_t *gamma, int *exceeds) {
    if (!target_n || !k || !gamma) return set_err(PA_E_PARAM, "target_n and k must be >= 1");
    uint64_t best = 0;
    for (uint64_t e : kMersenne)
        if (e <= target_n / k) best = e;
    if (exceeds) *exceeds = best ? 0 : 1;
    *gamma = best ? best : kMersenne[0];
    return PA_OK;
}

extern "C" int pa_derive_paper_params(uint64_t target_n, double ratio, uint64_t t, double epsilon, uint64_t *gamma,
                                      uint64_t *k, uint64_t *n, uint64_t *s, uint64_t *m) {
    uint64_t kk = 0, g = 0, ss = 0;
    int ex = 0;
    TRY(pa_select_block_count(ratio, &kk));
    TRY(pa_select_gamma(target_n, kk, &g, &ex));
    TRY(pa_derive_security_coefficient(epsilon, &ss));
    const uint64_t nn = kk * g;
    if (t + ss >= nn) return set_err(PA_E_PARAM, "m = n - t - s must be > 0");
    const uint64_t mm = nn - t - ss;
    if (mm + ss > g) return set_err(PA_E_PARAM, "m + s must be <= gamma (SPEC.md:187)");
    if (gamma) *gamma = g;
    if (k) *k = kk;
    if (n) *n = nn;
    if (s) *s = ss;
    if (m) *m = mm;
    return PA_OK;
}

extern "C" int pa_expand_bc(uint64_t seed, uint64_t alpha, uint32_t *b_out, uint32_t *c_out) {
    if (!b_out || !c_out || !alpha) return set_err(PA_E_PARAM, "bad argument");
    std::vector<uint32_t> w;
    TRY(expand_words(seed, kStreamB, alpha, w, false));
    w[0] |= 1u;
    memcpy(b_out, w.data(), w.size() * 4);
    TRY(expand_words(seed, kStreamC, alpha, w, false));
    memcpy(c_out, w.data(), w.size() * 4);
    return PA_OK;
}

// ====================================================================== debug-build probes
extern "C" int pa_debug_build(void) {
#ifdef PA_DEBUG
    return 1;
#else
    return 0;
#endif
}

#ifdef PA_DEBUG
// soft-mode probe: one registered range, one address past its end, one smem index past the
// dynamic allocation -> exactly 2 violations counted
__global__ void dbg_selftest_k(const uint32_t *inside, const uint32_t *past_end) {
    extern __shared__ uint32_t dsm[];
    PA_CK(inside, 4);
    PA_CK(past_end, 4);
    PA_SMEM_CK(8);                       // launched with 32 bytes of dynamic smem: index 8 is out
    PA_SMEM_CK(7);
    if (threadIdx.x == 1024) dsm[0] = 0;  // keeps dsm referenced
}
#endif

extern "C" int pa_debug_selftest(void) {
#ifdef PA_DEBUG
    uint32_t *buf = nullptr;
    CUDA_TRY(cudaMalloc(&buf, 64));
    dbg_add(buf, 64);
    const uint32_t one = 1, zero = 0;
    CUDA_TRY(cudaMemcpyToSymbol(pa::g_dbg_soft, &one, 4));
    CUDA_TRY(cudaMemcpyToSymbol(pa::g_dbg_violations, &zero, 4));
    dbg_selftest_k<<<1, 1, 32>>>(buf + 15, buf + 16);
    CUDA_TRY(cudaDeviceSynchronize());
    uint32_t nv = 0;
    CUDA_TRY(cudaMemcpyFromSymbol(&nv, pa::g_dbg_violations, 4));
    CUDA_TRY(cudaMemcpyToSymbol(pa::g_dbg_soft, &zero, 4));
    dbg_remove(buf);
    cudaFree(buf);
    if (nv != 2) return set_err(PA_E_STATE, "debug self-test counted %u violations, expected 2", nv);
    return PA_OK;
#else
    return set_err(PA_E_STATE, "not a PA_DEBUG build");
#endif
}

#ifdef PA_TPROF
// timeline profiling build only (scripts/tprof.py; not part of include/pa.h)
extern "C" int pa_tprof_reset(void) {
    const uint32_t z = 0;
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpyToSymbol(pa::g_tn, &z, 4));
    return PA_OK;
}
extern "C" int pa_tprof_dump(void *host, uint32_t max_records) {
    uint32_t n = 0;
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpyFromSymbol(&n, pa::g_tn, 4));
    n = std::min(std::min(n, pa::kTMax), max_records);
    if (n) CUDA_TRY(cudaMemcpyFromSymbol(host, pa::g_trec, (size_t)n * sizeof(pa::TRec)));
    return (int)n;
}
#endif
