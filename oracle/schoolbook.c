/*
 * Plain C schoolbook oracle of the MMH-MH pipeline.  TEST INFRASTRUCTURE ONLY.
 *
 * Nothing in the product path may include, link or call this file.  It shares no
 * header, table or helper with the CUDA library (include/, paper_2105_13678_b200/).
 *
 * What it computes (the plain definition, no transforms, no blocking beyond
 * "split the work over threads and add the partial sums"):
 *   oracle_mmh:  y = (sum_{i in [b0,b1)} a_i * x_i) mod (2^gamma - 1)
 *                  Eq. 2; fold identity PAPER.md:130-132;
 *                  canonical residue SPEC.md:38,87 (reading A6).
 *                x_i = big-endian integer of key bytes [i*r/8, (i+1)*r/8),
 *                  bits >= n ignored, zero-extended (readings A3, A4).
 *   oracle_mh:   z = ((b*y + c) mod 2^alpha) >> (alpha - m), emitted MSB-first
 *                  into ceil(m/8) bytes (Eq. 4; readings A5, A8).
 * Multiplication is the schoolbook row-by-row method on 32-bit limbs with a 64-bit
 * accumulator.  All integers are little-endian arrays of 32-bit words.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef uint32_t u32;
typedef uint64_t u64;

static u64 words_for_bits(u64 bits) { return (bits + 31) / 32; }

/* acc[pos..] += v (single word), propagating the carry; acc has len words. */
static void add_word_at(u32 *acc, u64 len, u64 pos, u32 v) {
    u64 t = v;
    while (t && pos < len) {
        t += acc[pos];
        acc[pos] = (u32)t;
        t >>= 32;
        pos++;
    }
}

/* dst[0..len) += src[0..slen), carries propagate inside dst. */
static void add_into(u32 *dst, u64 len, const u32 *src, u64 slen) {
    u64 carry = 0, i;
    for (i = 0; i < slen && i < len; i++) {
        u64 t = (u64)dst[i] + src[i] + carry;
        dst[i] = (u32)t;
        carry = t >> 32;
    }
    for (; carry && i < len; i++) {
        u64 t = (u64)dst[i] + carry;
        dst[i] = (u32)t;
        carry = t >> 32;
    }
}

/* acc += a[ja..jb) * 2^(32*ja) * x  (schoolbook rows), acc long enough. */
static void mul_rows(u32 *acc, u64 acc_len, const u32 *a, u64 ja, u64 jb,
                     const u32 *x, u64 wx, u64 limit /* keep words < limit */) {
    for (u64 j = ja; j < jb; j++) {
        u64 aj = a[j], carry = 0;
        if (!aj) continue;
        u64 lmax = wx;
        if (j >= limit) continue;
        if (j + lmax > limit) lmax = limit - j;
        for (u64 l = 0; l < lmax; l++) {
            u64 t = (u64)acc[j + l] + aj * x[l] + carry;
            acc[j + l] = (u32)t;
            carry = t >> 32;
        }
        if (j + lmax < limit) add_word_at(acc, acc_len < limit ? acc_len : limit, j + lmax, (u32)carry);
    }
}

/* Block i of the key as little-endian words (wx = ceil(r/32) words). r % 8 == 0. */
static void load_block(const uint8_t *key, u64 n, u64 r, u64 i, u32 *xw, u64 wx) {
    u64 nbytes = (n + 7) / 8, R = r / 8, start = i * R;
    memset(xw, 0, wx * 4);
    for (u64 q = 0; q < R; q++) {           /* q-th byte from the end = bits [8q, 8q+8) */
        u64 pos = start + R - 1 - q;
        u32 v = 0;
        if (pos < nbytes) {
            v = key[pos];
            if (pos == nbytes - 1 && (n % 8)) v &= (0xFFu << (8 - n % 8)) & 0xFFu;
        }
        xw[q / 4] |= v << (8 * (q % 4));
    }
}

/* bits [start, start+len) of Y (wy words) into out (ceil(len/32) words). */
static void get_bits(const u32 *Y, u64 wy, u64 start, u64 len, u32 *out) {
    u64 wo = words_for_bits(len);
    for (u64 w = 0; w < wo; w++) {
        u64 b = start + 32 * w, q = b / 32, s = b % 32;
        u64 lo = q < wy ? Y[q] : 0, hi = (q + 1) < wy ? Y[q + 1] : 0;
        u32 v = (u32)(((hi << 32) | lo) >> s);
        if (32 * (w + 1) > len) v &= (u32)((1ull << (len - 32 * w)) - 1);
        out[w] = v;
    }
}

static int bits_above(const u32 *v, u64 wv, u64 gamma) {
    for (u64 w = gamma / 32; w < wv; w++) {
        u32 x = v[w];
        if (w == gamma / 32) x &= ~(u32)((1ull << (gamma % 32)) - 1);
        if (x) return 1;
    }
    return 0;
}

/* y (wg = ceil(gamma/32) words) = Y mod (2^gamma - 1), canonical.  Fold identity
 * PAPER.md:130-132 applied to all gamma-bit chunks at once, then repeated. */
static void reduce_mersenne_words(const u32 *Y, u64 wy, u64 gamma, u32 *y) {
    u64 wg = words_for_bits(gamma), wt = wg + 2;
    u32 *t = calloc(wt, 4), *chunk = calloc(wg, 4);
    u64 nchunks = (32 * wy + gamma - 1) / gamma;
    for (u64 c = 0; c < nchunks; c++) {            /* sum of gamma-bit chunks */
        get_bits(Y, wy, c * gamma, gamma, chunk);
        add_into(t, wt, chunk, wg);
    }
    while (bits_above(t, wt, gamma)) {              /* fold again until < 2^gamma */
        u32 *hi = calloc(wt, 4), *lo = calloc(wt, 4);
        get_bits(t, wt, gamma, 32 * wt - gamma, hi);
        get_bits(t, wt, 0, gamma, lo);
        memcpy(t, lo, wt * 4);
        add_into(t, wt, hi, wt);
        free(hi); free(lo);
    }
    /* canonical zero: p = 2^gamma - 1 maps to 0 */
    int allones = 1;
    for (u64 b = 0; b < gamma && allones; b++) allones = (t[b / 32] >> (b % 32)) & 1;
    if (allones) memset(t, 0, wt * 4);
    memcpy(y, t, wg * 4);
    free(t); free(chunk);
}

/* y = sum_{i=b0}^{b1-1} a_i x_i mod (2^gamma - 1).
 * a_words: (b1-b0) * ceil(gamma/32) words, a_i at a_words + (i-b0)*wg.
 * Returns 0, or -1 on bad arguments.  nthreads <= 0: OpenMP default. */
int oracle_mmh(const uint8_t *key, u64 n, u64 r, u64 gamma, const u32 *a_words,
               u64 b0, u64 b1, u32 *y_out, int nthreads) {
    if (r % 8 || r == 0 || gamma < r || b1 < b0) return -1;
    u64 wg = words_for_bits(gamma), wx = words_for_bits(r), wy = wg + wx + 2;
    u64 nb = b1 - b0;
    /* work items: (block, a-word range) so that small k still uses every thread */
    u64 chunk = 4096, per = (wg + chunk - 1) / chunk, items = nb * per;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
    int T = omp_get_max_threads();
#else
    int T = 1;
#endif
    u32 *accs = calloc((u64)T * wy, 4);
    if (!accs) return -2;
#pragma omp parallel
    {
#ifdef _OPENMP
        int tid = omp_get_thread_num();
#else
        int tid = 0;
#endif
        u32 *acc = accs + (u64)tid * wy;
        u32 *xw = malloc(wx * 4);
        u64 cur = (u64)-1;
#pragma omp for schedule(dynamic, 1)
        for (long long it = 0; it < (long long)items; it++) {
            u64 i = b0 + (u64)it / per, part = (u64)it % per;
            if (i != cur) { load_block(key, n, r, i, xw, wx); cur = i; }
            u64 ja = part * chunk, jb = ja + chunk < wg ? ja + chunk : wg;
            mul_rows(acc, wy, a_words + (i - b0) * wg, ja, jb, xw, wx, wy);
        }
        free(xw);
    }
    for (int t = 1; t < T; t++) add_into(accs, wy, accs + (u64)t * wy, wy);
    reduce_mersenne_words(accs, wy, gamma, y_out);
    free(accs);
    return 0;
}

/* y = sum of G residues mod p (S6). parts: G * ceil(gamma/32) words. */
int oracle_merge(const u32 *parts, u64 G, u64 gamma, u32 *y_out) {
    u64 wg = words_for_bits(gamma), wy = wg + 2;
    u32 *Y = calloc(wy, 4);
    for (u64 g = 0; g < G; g++) add_into(Y, wy, parts + g * wg, wg);
    reduce_mersenne_words(Y, wy, gamma, y_out);
    free(Y);
    return 0;
}

/* out = MSB-first bytes of ((b*y + c) mod 2^alpha) >> (alpha - m).
 * b, c: ceil(alpha/32) words; y: ceil(gamma/32) words. */
int oracle_mh(const u32 *y, u64 gamma, const u32 *b, const u32 *c, u64 alpha, u64 m,
              uint8_t *out, int nthreads) {
    if (m > alpha || m == 0) return -1;
    u64 wa = words_for_bits(alpha), wg = words_for_bits(gamma);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
    int T = omp_get_max_threads();
#else
    int T = 1;
#endif
    u32 *accs = calloc((u64)T * wa, 4);
    u64 chunk = 2048, items = (wg + chunk - 1) / chunk;
#pragma omp parallel
    {
#ifdef _OPENMP
        int tid = omp_get_thread_num();
#else
        int tid = 0;
#endif
        u32 *acc = accs + (u64)tid * wa;
#pragma omp for schedule(dynamic, 1)
        for (long long it = 0; it < (long long)items; it++) {
            u64 ja = (u64)it * chunk, jb = ja + chunk < wg ? ja + chunk : wg;
            /* rows of y times b, truncated to wa words (mod 2^(32 wa)) */
            mul_rows(acc, wa, y, ja, jb, b, wa, wa);
        }
    }
    for (int t = 1; t < T; t++) add_into(accs, wa, accs + (u64)t * wa, wa);
    add_into(accs, wa, c, wa);
    if (alpha % 32) accs[wa - 1] &= (u32)((1ull << (alpha % 32)) - 1);   /* mod 2^alpha */
    /* z = bits [alpha-m, alpha); out byte q holds z bits (m-1-8q) .. (m-8-8q) */
    u64 nbo = (m + 7) / 8;
    for (u64 q = 0; q < nbo; q++) {
        uint8_t v = 0;
        for (int s = 0; s < 8; s++) {
            u64 j = 8 * q + s;                      /* output bit j = z bit (m-1-j) */
            if (j < m) {
                u64 bit = alpha - 1 - j;            /* = (alpha-m) + (m-1-j) */
                v |= (uint8_t)(((accs[bit / 32] >> (bit % 32)) & 1u) << (7 - s));
            }
        }
        out[q] = v;
    }
    free(accs);
    return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
