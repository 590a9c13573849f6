/*
 * pa.h -- C ABI of the B200-native MMH-MH privacy-amplification hash
 *         (hybrid multilinear-modular hashing + modular arithmetic hashing,
 *          arXiv 2105.13678, Algorithm 1).
 *
 * What a context computes (readings A1-A13 are listed in DESIGN.md):
 *   key bits kappa_0..kappa_{n-1}, MSB-first within each byte
 *       (reading A4), bits >= n ignored;
 *   k = ceil(n/r) blocks x_i = big-endian integer of key bits [i r, (i+1) r),
 *       the last block zero-padded at its end (reading A3);
 *   p = 2^gamma - 1, a Mersenne prime with gamma > r (reading A2);
 *   y = sum_i a_i x_i mod p                       (MMH, Eq. 2),
 *       canonical in [0, p-1] (reading A6);
 *   z = ((b y + c) mod 2^alpha) >> (alpha - m),  alpha = max(gamma, m)
 *                                                 (MH, Eq. 4, PAPER.md:99-101;
 *                                                  readings A1, A8);
 *   out = z, MSB-first in ceil(m/8) bytes, pad bits 0 (reading A5).
 * The hash keys a_i in [0, p-1], b odd < 2^alpha, c < 2^alpha are drawn from a
 * 64-bit seed with Philox4x64-10 (reading A7), or
 * supplied explicitly through pa_ctx_create_ex.
 *
 * Error behaviour: every int-returning call returns PA_OK (0) or a negative
 * PA_E_* code; pa_ctx_create returns NULL on failure.  The code and a message of
 * the last failure on the calling thread are available from pa_last_error().
 * No call aborts the process.  CUDA failures are reported as PA_E_CUDA.
 *
 * Threading / streams: a context is not re-entrant (one pa_hash at a time);
 * distinct contexts are independent.  All device work of a
 * context is enqueued on its stream (pa_params.stream, default: the legacy
 * default stream); pa_hash / pa_mmh_partial / pa_mh_merge are asynchronous
 * with respect to the host, pa_hash_host is synchronous.
 *
 * Ownership: the context owns its precomputed transforms and scratch (device
 * memory from pa_params.dev_alloc, default cudaMallocAsync on the context stream,
 * on the device current at creation); the caller owns every key / output buffer
 * passed in.  Every call on a context runs on the context's device (the caller's
 * current device is restored on return).
 */
#ifndef PA_H_
#define PA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define PA_OK                    0
#define PA_E_PARAM              -1   /* invalid parameter */
#define PA_E_INSUFFICIENT_INPUT -2   /* reserved for reload mode */
#define PA_E_BOUND              -3   /* no transform plan covers the coefficient bound */
#define PA_E_NOMEM              -4   /* device or host allocation failed */
#define PA_E_CUDA               -5   /* a CUDA runtime call or kernel failed */
#define PA_E_STATE              -6   /* call not valid for this context (e.g. shard) */
#define PA_E_NCCL               -7   /* NCCL unavailable or an NCCL call failed (world >= 1) */

typedef struct pa_ctx pa_ctx;

/* Transform plan of one big-integer product stage (MMH or MH).  The product
 * is computed exactly as a cyclic convolution of B-bit limbs, modulo each of
 * `nprimes` 30-bit NTT primes, recombined by CRT: `bound_log2` is log2 of the
 * largest possible convolution coefficient, `modulus_log2` of the prime
 * product (bound_log2 < modulus_log2 always holds for an accepted plan). */
typedef struct {
    uint32_t limb_bits;      /* B */
    uint32_t nprimes;        /* P */
    uint32_t log2_len;       /* L = 2^log2_len */
    uint32_t n_col;          /* column (first) pass length N2 */
    uint32_t n_row;          /* row (second) pass length N1; L = N1 * N2 */
    uint32_t primes[16];
    double   bound_log2;
    double   modulus_log2;
} pa_stage_plan;

typedef struct {
    uint64_t n, r, m;
    uint64_t gamma;          /* Mersenne exponent, p = 2^gamma - 1 */
    uint64_t alpha;          /* MH modulus width, max(gamma, m) */
    uint64_t k;              /* total number of blocks ceil(n/r) */
    uint64_t block_begin;    /* this context's shard [block_begin, block_end) */
    uint64_t block_end;
    pa_stage_plan mmh;
    pa_stage_plan mh;
    uint64_t device_bytes;   /* device memory held by the context */
    uint32_t kernels_per_hash; /* kernel launches enqueued by the last pa_hash /
                                  pa_mmh_partial / pa_mh_merge call */
    uint32_t launches_total; /* kernel launches enqueued since creation (mod 2^32),
                                precompute included */
    uint32_t insecure_length; /* 1 when m >= gamma (MMH-MH contexts): alpha = m > gamma and
                                 the output is longer than the gamma bits of entropy y can
                                 carry -- a throughput configuration, security-vacuous
                                 (PAPER.md:143 requires gamma > beta; reading A1).  strict
                                 contexts reject it instead. */
    int32_t  world;          /* multi-GPU contexts: ranks sharing each key, else 0 */
    int32_t  rank;           /* this context's rank in [0, world) */
    uint64_t acc_words;      /* words of one transform-domain accumulator (pa_mmh_acc):
                                mmh.nprimes * 2^mmh.log2_len */
    uint32_t graph_captures; /* CUDA-graph captures since creation (new pointer sets) */
    uint32_t graph_updates;  /* ... of which updated an executable graph in place */
    uint32_t graph_instantiations;
    uint32_t tz_group_blocks;/* Toeplitz contexts: input blocks per accumulation group */
    uint32_t p2p;            /* multi-GPU contexts: 1 = accumulators exchanged over peer memory
                                (pa_params.p2p), 0 = ncclReduce */
} pa_info;

typedef struct {
    uint64_t n;              /* key bits, >= 1 */
    uint64_t r;              /* block bits, >= 16 and a multiple of 16 */
    uint64_t m;              /* output bits, >= 1 */
    uint64_t gamma;          /* Mersenne exponent (gamma > r), 0 = smallest table entry > r */
    uint64_t seed;           /* hash-key seed (ignored for keys given explicitly) */
    uint64_t block_begin;    /* shard: blocks [block_begin, block_end); both 0 = all */
    uint64_t block_end;
    /* Optional explicit hash keys (host pointers, little-endian 32-bit words).
     * a_words: (block_end-block_begin) * ceil(gamma/32) words, a_i < p each;
     * b_words, c_words: ceil(alpha/32) words each, b odd, both < 2^alpha.
     * NULL = expand from `seed` (reading A7). */
    const uint32_t *a_words;
    const uint32_t *b_words;
    const uint32_t *c_words;
    void *stream;            /* cudaStream_t, NULL = legacy default stream */
    int32_t limb_bits;       /* 0 = planner's choice, else force B (multiple of 8, 16..256) */
    int32_t strict;          /* nonzero: reject m >= gamma ("gamma > beta") */
    /* Paper mode (Algorithm 1 exactly): when
     * nonzero, the key is split into paper_k blocks of gamma bits (r is ignored; gamma must
     * be given), window t = key bits [t gamma, (t+1) gamma); a window equal to 2^gamma - 1
     * is cast away and the next consumed (reading A10); alpha = gamma
     * and m < gamma are required.  Needs n >= paper_k * gamma; fewer than
     * paper_k usable windows -> PA_E_INSUFFICIENT_INPUT (pa_ctx_status / pa_hash_host).
     * Not available for shard contexts. */
    uint64_t paper_k;
    /* Comparator (Table 1 "Modular Arithmetic Hashing PA",
     * SPEC.md:305-313): when nonzero the context computes MH-only PA instead of MMH-MH:
     * out = top m bits of (b x + c) mod 2^n, x = the n-bit key integer (MSB-first),
     * b odd and c drawn with alpha = n (reading A7).  r, gamma, shards and paper_k must be 0;
     * m <= n.  pa_hash / pa_hash_host only. */
    uint64_t mh_only;
    /* Comparator (Table 1 "Toeplitz Hashing PA"):
     * when nonzero the context computes Toeplitz-hashing PA over GF(2):
     * out bit j = XOR_{i<n} d[m-1-j+i] x_i (reading A14), x_i = key bit i (MSB-first), the
     * n + m - 1 diagonal bits d drawn from `seed` (reading A15).  Exact integer NTT
     * convolution mod one 30-bit prime, r x r block split (r = min(2^22, 2^ceil(log2 max(n,
     * m))), at least 512; limb_bits != 0 forces r = 2^limb_bits, 9..22).  r, gamma, shards,
     * paper_k, mh_only must be 0; m < 2^31.  Each output bit is the parity of a count <= n:
     * with n below the prime one accumulation is exact; otherwise the input blocks are summed
     * in groups of floor((prime - 1) / r) blocks (each group's counts exact) and the groups'
     * parities XORed.  Output blocks are accumulated kTzMaxOut (16) at a time.  pa_query
     * reports r, k = ceil(n/r) input blocks, alpha = ceil(m/r) output blocks, the transform in
     * `mmh` and the group size in tz_group_blocks.  pa_hash / pa_hash_host only. */
    uint64_t toeplitz;
    /* Multi-GPU (SURVEY.md §8(b,e); MMH splits over blocks, "split and separately
     * handle"): world >= 1 makes the context rank `rank` of a `world`-rank job
     * hashing every key together.  Each rank owns blocks [floor(k rank / world),
     * floor(k (rank+1) / world)) (block_begin/block_end must be 0 or exactly that range) and
     * the transforms of its own a_i; every rank plans the transform for all k blocks, so the
     * partial sums are compatible.  The ranks' transform-domain accumulators
     * sum_{i in shard} X_i (.) A_i are summed by ONE ncclReduce to the key's root, which
     * alone runs the inverse transform, CRT, carries, the Mersenne fold and MH.
     * nccl_id: the ncclUniqueId bytes from pa_nccl_unique_id() on one rank, given to all.
     * Creation is collective (every rank must call pa_ctx_create_ex; it blocks until all
     * ranks joined).  world = 1 is a one-rank communicator (the same code path).  NCCL is
     * loaded at run time (libnccl.so.2; PA_NCCL_LIB overrides); failures -> PA_E_NCCL.
     * Not available with paper_k, mh_only or toeplitz. */
    int32_t world;
    int32_t rank;
    uint8_t nccl_id[128];
    /* Device memory of the context (precomputed transforms and scratch): dev_alloc(bytes,
     * stream, alloc_user) -> 256-byte aligned pointer or NULL, dev_free(ptr, bytes, stream,
     * alloc_user) at pa_ctx_destroy -- e.g. PyTorch's caching allocator (the Python binding
     * passes torch.cuda.caching_allocator_alloc / _delete).  NULL: cudaMallocAsync /
     * cudaFreeAsync on the context stream (the device's default memory pool). */
    void *(*dev_alloc)(size_t bytes, void *stream, void *user);
    void (*dev_free)(void *ptr, size_t bytes, void *stream, void *user);
    void *alloc_user;
    /* Toeplitz comparator only: input blocks per accumulation group, at most the automatic
     * floor((prime - 1) / r) (0 = automatic).  Smaller groups exercise the grouped (parity
     * XOR) path at small n; the output does not depend on it. */
    uint64_t tz_group_blocks;
    /* Multi-GPU contexts (world >= 1): exchange the transform-domain accumulators over peer
     * memory instead of an ncclReduce.  Each rank's row multiply-accumulate adds its canonical
     * partial sums with 64-bit atomics straight into the key root's receive buffer (NVLink peer
     * stores, overlapping the transforms; the compute and the collective are one kernel), and
     * 32-bit counters in each GPU's own memory order the uses of a receive buffer (the root
     * zeroes and frees it after its import; ranks wait for that before their next atomics).
     * The buffers (cudaMalloc) are shared through CUDA IPC handles all-gathered once over the
     * context's NCCL communicator at creation.  Ranks must issue the same sequence of
     * pa_hash / pa_hash_batch calls.  Requires peer access between the GPUs (one node);
     * creation fails with PA_E_CUDA otherwise.  0: ncclReduce (default). */
    int32_t p2p;
} pa_params;

/* Create a context on the current CUDA device.  `p` is the Mersenne EXPONENT
 * gamma (p = 2^gamma - 1), or 0 for the smallest known exponent > r (reading A2).
 * Validates n >= 1; r >= 16, r % 16 == 0; gamma in the SPEC.md:33 table, gamma > r;
 * m >= 1.  Expands a_i, b, c from `seed`, precomputes the transforms of a_i and b
 * in device memory.  Returns NULL on failure (see pa_last_error). */
pa_ctx *pa_ctx_create(uint64_t n, uint64_t r, uint64_t m, uint64_t p, uint64_t seed);

/* Same with every option; *out = context.  Returns PA_OK or PA_E_*. */
int pa_ctx_create_ex(const pa_params *prm, pa_ctx **out);

/* Hash one key.  key_bits: DEVICE pointer to ceil(n/8) bytes (bits >= n ignored).
 * For a shard context it points to the shard's slice: key bytes
 * [block_begin*r/8, min(block_end*r/8, ceil(n/8))).  A shard context without world
 * (block_begin/block_end only) fails with PA_E_STATE: it hashes through pa_mmh_partial +
 * pa_mh_merge or pa_mmh_acc + pa_tail_merge (host-side exchange).  A multi-GPU context
 * (world >= 1) runs S1-S3 on its blocks, one ncclReduce of the transform-domain
 * accumulators to rank 0, and S4-S7 on rank 0: out_bits is written on rank 0 only (other
 * ranks may pass NULL); every rank must call pa_hash for every key, in the same order.
 * out_bits: DEVICE pointer to ceil(m/8) bytes (written MSB-first, pad bits 0).
 * Asynchronous on the context stream. */
int pa_hash(pa_ctx *ctx, const uint8_t *key_bits, uint8_t *out_bits);

/* Stream mode: hash `count` independent keys with this
 * context's hash function.  keys[j] / outs[j]: HOST arrays of DEVICE pointers, each as in
 * pa_hash.  Keys alternate between two buffer sets and streams (forked from and joined
 * back into the context stream), so one key's latency-bound MH / tail kernels overlap the
 * next key's MMH transforms.  The first call allocates the second buffer set (about the
 * per-hash scratch of pa_ctx_query's device_bytes minus the precomputed transforms).
 * Multi-GPU contexts (world >= 1): the root rotates -- key j is reduced to and finished on
 * rank j mod world (SPEC.md:235-243 pa_stream), so every rank
 * computes 1/world of every key's MMH and the tail + MH of every world-th key; outs[j] is
 * written on rank j mod world only (NULL allowed elsewhere).  All ranks pass the same count.
 * Asynchronous on the context stream; outputs are identical to count pa_hash calls. */
int pa_hash_batch(pa_ctx *ctx, const uint8_t *const *keys, uint8_t *const *outs, uint32_t count);

/* End-to-end variant with HOST buffers: copies the key host->device, hashes,
 * copies the output device->host and synchronizes the stream before returning.
 * Pinned host memory gives full PCIe bandwidth; the copy is split in chunks that
 * overlap the first pass of the transform.
 * Multi-GPU contexts (world >= 1): key_host is this rank's key SLICE (the bytes of its
 * blocks, as for pa_hash), copied over this rank's own host link; out_host is written on
 * rank 0 only (NULL allowed elsewhere).  Collective: every rank calls it; each rank
 * returns when its own stream has drained (rank 0: after the output has landed). */
int pa_hash_host(pa_ctx *ctx, const uint8_t *key_host, uint8_t *out_host);

/* End-to-end stream mode: `count` keys in HOST memory (keys_host[j]: ceil(n/8) bytes,
 * outs_host[j]: ceil(m/8) bytes; pinned memory for full PCIe bandwidth).  Key j's H2D
 * overlaps the hash of key j-1 (two device staging buffers, the two buffer sets of
 * pa_hash_batch).  Synchronous.  Not available in paper mode or for shards.
 * Multi-GPU contexts (world >= 1): keys_host[j] is this rank's slice of key j; the root
 * rotates as in pa_hash_batch, outs_host[j] is written on rank j mod world only (NULL
 * allowed elsewhere).  Collective: every rank passes the same count. */
int pa_hash_host_batch(pa_ctx *ctx, const uint8_t *const *keys_host, uint8_t *const *outs_host, uint32_t count);

/* Stages S1-S5 on this context's blocks: y_part = sum_{i in shard} a_i x_i mod p,
 * canonical, as ceil(gamma/32) little-endian 32-bit words at DEVICE pointer y_out.
 * key_slice: DEVICE pointer to the shard's key bytes (see pa_hash). Asynchronous. */
int pa_mmh_partial(pa_ctx *ctx, const uint8_t *key_slice, uint32_t *y_out);

/* Stages S6-S7: y = sum_{g<G} y_parts[g] mod p (each part ceil(gamma/32) words,
 * DEVICE, contiguous), then MH into out_bits (DEVICE, ceil(m/8) bytes). */
int pa_mh_merge(pa_ctx *ctx, const uint32_t *y_parts, uint32_t G, uint8_t *out_bits);

/* Transform-domain split of S1-S7 with a caller-side exchange (any transport; the
 * single-GPU validation of the multi-GPU path).
 * pa_mmh_acc: S1-S3 on this context's blocks -> acc_out (DEVICE, pa_info.acc_words
 *   32-bit words) = sum_{i in shard} NTT(x_i) (.) NTT(a_i), prime by prime, each word
 *   canonical (< its prime), in the transform's internal order.  Any context with the
 *   same (n, r, m, gamma, limb_bits) produces the same layout (shards plan for all k
 *   blocks), and the sum of the parts over a partition of the blocks is the whole key's.
 * pa_tail_merge: S4-S7 from G such accumulators (DEVICE, contiguous, G * acc_words
 *   words): their sum mod each prime is inverse-transformed, CRT-recombined, carried,
 *   folded mod p and hashed by MH into out_bits (DEVICE, ceil(m/8) bytes).  Both
 *   asynchronous on the context stream; no NCCL involved. */
int pa_mmh_acc(pa_ctx *ctx, const uint8_t *key_slice, uint32_t *acc_out);
int pa_tail_merge(pa_ctx *ctx, const uint32_t *acc_parts, uint32_t G, uint8_t *out_bits);

/* A fresh ncclUniqueId (128 bytes) for pa_params.nccl_id: call on one rank and broadcast
 * the bytes to the others (e.g. torch.distributed).  PA_E_NCCL if NCCL cannot be loaded. */
int pa_nccl_unique_id(uint8_t *id_out);

/* Fresh hash keys per job: re-draw a_i, b, c from `seed` on the
 * GPU (reading A7; bit-identical to pa_expand_a / pa_expand_bc and to a context created
 * with this seed) and recompute the transforms of the a_i and b.  Asynchronous on the
 * context stream: hashes enqueued after it use the new function. */
int pa_ctx_rekey(pa_ctx *ctx, uint64_t seed);

/* Synchronizes the context stream and returns the device-side status of the last hash:
 * PA_OK, or PA_E_INSUFFICIENT_INPUT (paper mode: fewer than paper_k usable windows; the
 * output is then undefined). */
int pa_ctx_status(pa_ctx *ctx);

/* Paper mode: consumption statistics of the last hash (SPEC.md pa_run "stats: consumed_bits,
 * rejected_blocks"; the reload rule of PAPER.md:130,147-148): *consumed_bits = key bits up to
 * the end of the k-th usable window, *rejected_windows = all-ones windows cast away before it.
 * Synchronizes the context stream.  PA_E_STATE if the context is not in paper mode,
 * PA_E_INSUFFICIENT_INPUT as pa_ctx_status.  Outputs may be NULL. */
int pa_ctx_paper_stats(pa_ctx *ctx, uint64_t *consumed_bits, uint64_t *rejected_windows);

/* Free everything the context owns; NULL is a no-op. */
void pa_ctx_destroy(pa_ctx *ctx);

/* Describe a context (plans, shard, memory). */
int pa_ctx_query(const pa_ctx *ctx, pa_info *info);

/* Change the stream later work of the context is enqueued on. */
int pa_ctx_set_stream(pa_ctx *ctx, void *stream);

/* Stage timing: when enabled, pa_hash records CUDA events around each kernel
 * on the context stream; pa_ctx_stage_times accumulates milliseconds per named
 * stage since the last reset (names are static strings).  Returns the number of
 * stages written (<= max). */
int pa_ctx_set_profiling(pa_ctx *ctx, int enable);
int pa_ctx_stage_times(pa_ctx *ctx, const char **names, double *ms, uint32_t *launches, int max);

/* ---- host-only helpers (no GPU needed) ---------------------------------- */

/* Validate parameters and compute the plan without a GPU.  Returns PA_OK and
 * fills *info (device_bytes = projected), or PA_E_*. */
int pa_plan(const pa_params *prm, pa_info *info);

/* The Philox4x64-10 generator of reading A7 (numpy's convention): writes words
 * w = 0..nwords-1 of stream key (key0, key1), word w = block(counter =
 * floor(w/4) + 1)[w mod 4]. */
int pa_philox4x64_10(uint64_t key0, uint64_t key1, uint64_t nwords, uint64_t *out);

/* Hash-key expansion of reading A7 into little-endian 32-bit words:
 * a_i (ceil(gamma/32) words), b and c (ceil(alpha/32) words each). */
int pa_expand_a(uint64_t seed, uint64_t i, uint64_t gamma, uint32_t *out);
int pa_expand_bc(uint64_t seed, uint64_t alpha, uint32_t *b_out, uint32_t *c_out);

/* Parameter derivation of the paper's shape.
 *
 * pa_derive_security_coefficient: s = ceil(2 log2(1/epsilon) - 2), at least 1 -- the
 *   smallest s with 2^(-s/2-1) <= epsilon, inverting the composition bound of PAPER.md:185-188
 *   ("secure under composition").  0 < epsilon < 1, else PA_E_PARAM.
 * pa_select_block_count: k = floor(1/ratio) for the compression ratio 0 < ratio < 1
 *   ("k <= 1/r"; Table 3: 0.2957 -> 3, 0.0972 -> 10), else PA_E_PARAM.
 * pa_select_gamma: the largest Mersenne exponent (SPEC.md:33 table) with k gamma <= target_n
 *   ("n is equal to gamma x k"); when even k * 3 > target_n, the smallest
 *   exponent with *exceeds = 1.  target_n >= 1 and k >= 1, else PA_E_PARAM.
 * pa_derive_paper_params: the composition SPEC.md:185-191, 465: k from ratio, gamma from
 *   (target_n, k), n = k gamma, s from epsilon, m = n - t - s.  PA_E_PARAM when m <= 0 or
 *   m + s > gamma (the invariant "m + s <= gamma").  Outputs may be NULL. */
int pa_derive_security_coefficient(double epsilon, uint64_t *s);
int pa_select_block_count(double ratio, uint64_t *k);
int pa_select_gamma(uint64_t target_n, uint64_t k, uint64_t *gamma, int *exceeds);
int pa_derive_paper_params(uint64_t target_n, double ratio, uint64_t t, double epsilon, uint64_t *gamma,
                           uint64_t *k, uint64_t *n, uint64_t *s, uint64_t *m);

/* Bounds-asserting debug build (built with -DPA_DEBUG into _pa_debug.so): every global
 * access site of the kernels is checked against the live device ranges (context
 * allocations + the caller's buffers of the current call) and every shared-memory index
 * against the launch's shared memory; a violation prints the site and traps.
 * pa_debug_build: 1 in that build, 0 in the release build.  pa_debug_selftest: (debug
 * build) counts, without trapping, one out-of-range global address and one out-of-range
 * shared index and returns PA_OK when exactly those two are caught; PA_E_STATE otherwise
 * or in the release build. */
int pa_debug_build(void);
int pa_debug_selftest(void);

/* Code of the last failure on this thread; copies its message into buf. */
int pa_last_error(char *buf, size_t len);

/* sizeof(pa_params) and sizeof(pa_info) as compiled into the library (host only): bindings
 * check their struct mirrors against them.  Outputs may be NULL.  Returns PA_OK. */
int pa_abi_sizes(uint64_t *params_bytes, uint64_t *info_bytes);

#ifdef __cplusplus
}
#endif
#endif /* PA_H_ */
