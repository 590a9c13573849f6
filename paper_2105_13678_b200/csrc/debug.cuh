// Bounds-asserting debug build (-DPA_DEBUG; `python paper_2105_13678_b200/build.py --debug`
// -> _pa_debug.so).  compute-sanitizer is closed on the GPU pool, so the debug build checks
// every global-memory access site of the kernels against the set of live device ranges
// (the context's allocations and the caller's key / output / exchange buffers of the current
// call), and every dynamic shared-memory index against the launch's dynamic smem size.  A
// violation prints the site and traps (or, in the self-test's soft mode, is counted).
// In the release build every macro here expands to nothing.
#pragma once
#include <cstdint>
#include <cstdio>

#ifdef PA_DEBUG
namespace pa {

constexpr int kDbgMaxRanges = 512;
struct DbgRange {
    uint64_t lo, hi;                       // [lo, hi)
};
__device__ DbgRange g_dbg_ranges[kDbgMaxRanges];
__device__ uint32_t g_dbg_n;
__device__ uint32_t g_dbg_soft;            // self-test: count instead of trapping
__device__ uint32_t g_dbg_violations;

__device__ __noinline__ void dbg_fail(const char *what, const char *file, int line, uint64_t a, uint64_t b) {
    if (g_dbg_soft) {
        atomicAdd(&g_dbg_violations, 1u);
        return;
    }
    printf("PA_DEBUG bounds violation: %s at %s:%d [%llx, %llx) block (%d,%d) thread %d\n", what, file, line,
           (unsigned long long)a, (unsigned long long)b, (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);
    __trap();
}

__device__ __forceinline__ void dbg_check(const void *p, uint64_t bytes, const char *what, const char *file, int line) {
    const uint64_t a = reinterpret_cast<uint64_t>(p), b = a + bytes;
    const uint32_t n = *(volatile uint32_t *)&g_dbg_n;
    for (uint32_t i = 0; i < n && i < kDbgMaxRanges; i++)
        if (a >= g_dbg_ranges[i].lo && b <= g_dbg_ranges[i].hi) return;
    dbg_fail(what, file, line, a, b);
}

__device__ __forceinline__ uint32_t dbg_dyn_smem_bytes() {
    uint32_t r;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}

}  // namespace pa
namespace pa {
// static shared memory lies below the dynamic array, which ends at its base + the launch's
// dynamic size: a shared access is in bounds iff it ends at or below that end
__device__ __forceinline__ void dbg_smem_check(const void *p, uint64_t bytes, const char *what, const char *file, int line) {
    extern __shared__ __align__(16) uint8_t pa_dbg_dyn_base[];
    const uint32_t end = (uint32_t)__cvta_generic_to_shared(pa_dbg_dyn_base) + dbg_dyn_smem_bytes();
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
    if ((uint64_t)a + bytes > end) dbg_fail(what, file, line, a, end);
}
__device__ __forceinline__ void dbg_idx_check(int64_t i, int64_t n, const char *what, const char *file, int line) {
    if (i < 0 || i >= n) dbg_fail(what, file, line, (uint64_t)i, (uint64_t)n);
}
__device__ __forceinline__ void dbg_dsmem_check(int64_t i, const char *what, const char *file, int line) {
    if (i < 0 || (uint64_t)(i + 1) * 4 > dbg_dyn_smem_bytes()) dbg_fail(what, file, line, (uint64_t)i, 0);
}
}  // namespace pa
#define PA_CK(p, bytes) ::pa::dbg_check((const void *)(p), (uint64_t)(bytes), #p, __FILE__, __LINE__)
// index i (in words) into the dynamic shared-memory array of the launch
#define PA_SMEM_CK(i) ::pa::dbg_dsmem_check((int64_t)(i), "dynamic smem index " #i, __FILE__, __LINE__)
// shared-memory pointer p (any window address): [p, p + bytes) inside the CTA's shared memory
#define PA_SMEM_PTR_CK(p, bytes) ::pa::dbg_smem_check((const void *)(p), (uint64_t)(bytes), "smem pointer " #p, __FILE__, __LINE__)
// index i into a static array of n elements
#define PA_IDX_CK(i, n) ::pa::dbg_idx_check((int64_t)(i), (int64_t)(n), "index " #i, __FILE__, __LINE__)
#else
#define PA_CK(p, bytes) ((void)0)
#define PA_SMEM_CK(i) ((void)0)
#define PA_SMEM_PTR_CK(p, bytes) ((void)0)
#define PA_IDX_CK(i, n) ((void)0)
#endif

// checked read-only load and checked lvalue (load or store) of *p
#ifdef PA_DEBUG
#define PA_LDG(...) (PA_CK((__VA_ARGS__), sizeof(*(__VA_ARGS__))), __ldg(__VA_ARGS__))
#define PA_AT(...) (*(PA_CK((__VA_ARGS__), sizeof(*(__VA_ARGS__))), (__VA_ARGS__)))
#else
#define PA_LDG(...) __ldg(__VA_ARGS__)
#define PA_AT(...) (*(__VA_ARGS__))
#endif

// ---- timeline profiling build (-DPA_TPROF, development only; scripts/tprof.py): thread 0
// of every CTA of the instrumented kernels appends (kernel id, CTA, phase, SM, globaltimer,
// clock64) records; pa_tprof_dump copies them out.  Nothing in the release build.
#ifdef PA_TPROF
namespace pa {
struct TRec {
    uint32_t kid, blk, phase, sm;
    uint64_t t, clk;
};
constexpr uint32_t kTMax = 1u << 20;
__device__ TRec g_trec[kTMax];
__device__ uint32_t g_tn;
__device__ __forceinline__ void tmark(uint32_t kid, uint32_t phase, uint32_t blk = 0xFFFFFFFFu) {
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        uint64_t t, clk;
        uint32_t sm;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(clk));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        const uint32_t i = atomicAdd(&g_tn, 1u);
        if (i < kTMax) g_trec[i] = TRec{kid, blk != 0xFFFFFFFFu ? blk : blockIdx.x + blockIdx.y * gridDim.x, phase, sm, t, clk};
    }
}
}  // namespace pa
#define PA_TMARK(kid, phase) ::pa::tmark((uint32_t)(kid), (uint32_t)(phase))
#define PA_TMARK_B(kid, phase, blk) ::pa::tmark((uint32_t)(kid), (uint32_t)(phase), (uint32_t)(blk))
#else
#define PA_TMARK(kid, phase) ((void)0)
#define PA_TMARK_B(kid, phase, blk) ((void)0)
#endif
