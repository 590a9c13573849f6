// Integer-pipe throughput microbenchmark for sm_100a ("microbenchmark
// it before quoting a %").  The MMH-MH hot path is modular integer arithmetic on the
// 32-bit pipes: a Shoup butterfly mod a 30-bit prime is IADD3,
// VIADDMNMX, IADD3, IMAD.HI, IMAD, IMAD.  This program measures, per SM and SM clock,
// the lane-operations per cycle each of those instruction classes sustains, and the
// butterfly mix itself, with one 1024-thread CTA per SM and 8 independent dependency
// chains per thread.  Cycles come from clock64 on each SM (so the figure does not
// depend on the clock the GPU ran at); the wall time from CUDA events gives the clock.
//
// Output: one JSON object on stdout (bench.py reads profiles/int_peak.json written from it).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int kThreads = 1024;
constexpr int kChains = 8;
constexpr int kIters = 4096;

enum Op { OP_IMAD, OP_IMAD_WIDE, OP_IMAD_HI, OP_IADD3, OP_LOP3, OP_SHF, OP_PRMT, OP_VIADDMNMX,
          OP_MIX_IMAD_IADD3, OP_BFLY, OP_COUNT };
static const char *kNames[OP_COUNT] = {"IMAD", "mad.wide.u32 chain step (IMAD.WIDE.U32 + IADD3 + IADD3.X/IMAD.X)", "IMAD.HI.U32", "IADD3", "LOP3", "SHF", "PRMT",
                                       "VIADDMNMX", "IMAD+IADD3 1:1", "shoup_butterfly"};
// lane-operations (SASS instructions x 32 lanes / 32) per chain step; the mad.wide.u32 step
// is counted as one (ptxas emits it as IMAD.WIDE.U32 with a zero addend plus a 64-bit add)
static const int kInstrPerStep[OP_COUNT] = {1, 1, 1, 1, 1, 1, 1, 1, 2, 6};

template <int OP>
__device__ __forceinline__ void step(uint32_t (&x)[kChains], uint32_t (&y)[kChains], uint32_t a, uint32_t b, uint32_t p) {
#pragma unroll
    for (int c = 0; c < kChains; c++) {
        if constexpr (OP == OP_IMAD) {
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        } else if constexpr (OP == OP_IMAD_WIDE) {
            // chain through the 64-bit addend: t = y * a + t (one IMAD.WIDE.U32 per step)
            uint64_t t = ((uint64_t)x[c] << 32) | y[c];
            asm volatile("{\n\t.reg .u32 lo, hi;\n\tmov.b64 {lo, hi}, %0;\n\tmad.wide.u32 %0, hi, %1, %0;\n\t}" : "+l"(t) : "r"(a));
            x[c] = (uint32_t)(t >> 32);
            y[c] = (uint32_t)t;
        } else if constexpr (OP == OP_IMAD_HI) {
            asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(a));
        } else if constexpr (OP == OP_IADD3) {
            asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        } else if constexpr (OP == OP_LOP3) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
        } else if constexpr (OP == OP_SHF) {
            asm volatile("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        } else if constexpr (OP == OP_PRMT) {
            asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(x[c]) : "r"(a));
        } else if constexpr (OP == OP_VIADDMNMX) {
            uint32_t t;
            asm volatile("sub.u32 %1, %0, %2;\n\tmin.u32 %0, %0, %1;" : "+r"(x[c]), "=r"(t) : "r"(p));
        } else if constexpr (OP == OP_MIX_IMAD_IADD3) {
            asm volatile("mad.lo.u32 %0, %0, %2, %3;\n\tadd.u32 %1, %1, %2;\n\tadd.u32 %1, %1, %3;"
                         : "+r"(x[c]), "+r"(y[c]) : "r"(a), "r"(b));
        } else {
            // DIF butterfly (modarith.cuh bfly_dif): s = min(u+v, u+v-2p); d = u - v + 2p;
            // v' = d w - umulhi(d, wp) p
            const uint32_t u = x[c], v = y[c];
            uint32_t s = u + v;
            s = min(s, s - 2 * p);
            const uint32_t d = u - v + 2 * p;
            const uint32_t q = __umulhi(d, b);
            y[c] = d * a - q * p;
            x[c] = s;
        }
    }
}

template <int OP>
__global__ void __launch_bounds__(kThreads, 1) kern(uint32_t a, uint32_t b, uint32_t p, uint32_t *sink,
                                                    unsigned long long *cycles) {
    uint32_t x[kChains], y[kChains];
#pragma unroll
    for (int c = 0; c < kChains; c++) { x[c] = threadIdx.x * 7 + c; y[c] = threadIdx.x * 3 + 5 * c; }
    __syncthreads();
    const unsigned long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < kIters; i++) {
#pragma unroll
        for (int u = 0; u < 8; u++) step<OP>(x, y, a, b, p);
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; c++) acc ^= x[c] ^ y[c];
    if (acc == 0x12345678u) sink[blockIdx.x] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
static int run(int nsm, uint32_t *sink, unsigned long long *dcyc, double *per_sm_clk, double *lane_ops_per_s,
               double *mhz) {
    const uint32_t p = 998244353u, a = 123456789u % p, b = (uint32_t)(((uint64_t)a << 32) / p);
    for (int rep = 0; rep < 2; rep++) kern<OP><<<nsm, kThreads>>>(a, b, p, sink, dcyc);   // warm-up
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    kern<OP><<<nsm, kThreads>>>(a, b, p, sink, dcyc);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::vector<unsigned long long> cyc(nsm);
    CK(cudaMemcpy(cyc.data(), dcyc, nsm * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    const unsigned long long cmax = *std::max_element(cyc.begin(), cyc.end());
    const double lane_ops_per_sm = (double)kThreads * kIters * 8 * kChains * kInstrPerStep[OP];
    *per_sm_clk = lane_ops_per_sm / (double)cmax;
    *lane_ops_per_s = lane_ops_per_sm * nsm / (ms * 1e-3);
    *mhz = (double)cmax / (ms * 1e-3) / 1e6;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return 0;
}

int main() {
    int dev = 0, nsm = 0, clk_khz = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    uint32_t *sink;
    unsigned long long *dcyc;
    CK(cudaMalloc(&sink, nsm * 4));
    CK(cudaMalloc(&dcyc, nsm * 8));
    double r[OP_COUNT], s[OP_COUNT], mhz[OP_COUNT];
    int rc = 0;
    rc |= run<OP_IMAD>(nsm, sink, dcyc, &r[0], &s[0], &mhz[0]);
    rc |= run<OP_IMAD_WIDE>(nsm, sink, dcyc, &r[1], &s[1], &mhz[1]);
    rc |= run<OP_IMAD_HI>(nsm, sink, dcyc, &r[2], &s[2], &mhz[2]);
    rc |= run<OP_IADD3>(nsm, sink, dcyc, &r[3], &s[3], &mhz[3]);
    rc |= run<OP_LOP3>(nsm, sink, dcyc, &r[4], &s[4], &mhz[4]);
    rc |= run<OP_SHF>(nsm, sink, dcyc, &r[5], &s[5], &mhz[5]);
    rc |= run<OP_PRMT>(nsm, sink, dcyc, &r[6], &s[6], &mhz[6]);
    rc |= run<OP_VIADDMNMX>(nsm, sink, dcyc, &r[7], &s[7], &mhz[7]);
    rc |= run<OP_MIX_IMAD_IADD3>(nsm, sink, dcyc, &r[8], &s[8], &mhz[8]);
    rc |= run<OP_BFLY>(nsm, sink, dcyc, &r[9], &s[9], &mhz[9]);
    if (rc) return 1;
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"threads_per_sm\": %d, \"chains_per_thread\": %d, "
           "\"unit\": \"lane-ops per SM per SM-clock (1 lane-op = one SASS instruction on one lane)\", \"ops\": {",
           prop.name, nsm, kThreads, kChains);
    for (int i = 0; i < OP_COUNT; i++)
        printf("%s\"%s\": {\"lane_ops_per_sm_clk\": %.2f, \"lane_ops_per_s\": %.4e, \"sm_mhz\": %.0f}",
               i ? ", " : "", kNames[i], r[i], s[i], mhz[i]);
    printf("}}\n");
    return 0;
}
