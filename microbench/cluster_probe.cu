// Cluster probe for the cluster-resident forward transform design:
//  (1) how many clusters of 2/4/8/16 CTAs the B200 keeps resident at one CTA per SM
//      (cudaOccupancyMaxActiveClusters), i.e. how many SMs a cluster launch strands;
//  (2) the cycles one four-step transpose exchange through distributed shared memory
//      takes in a cluster of 8: every thread holds 32 column outputs and stores them to the
//      CTA owning each output row (warp-contiguous 128-byte remote stores), then cluster sync.
// Output: JSON on stdout.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void dummy(uint32_t *o) { extern __shared__ uint32_t s[]; if (o) o[0] = s[threadIdx.x]; }

constexpr int kC = 8;            // cluster size
constexpr int kRowsPerCta = 32;  // 256 rows / 8
constexpr int kN1 = 512;         // row length (columns)
__device__ __forceinline__ int c_rank_off(int c) { return c * 32; }   // rank's 32-uint4 slice of a 256-uint4 row pair

__global__ void __cluster_dims__(kC, 1, 1) __launch_bounds__(512, 1)
exchange(int iters, unsigned long long *cyc, uint32_t *sink) {
    extern __shared__ uint32_t xs[];   // [32 rows][512] chunk
    cg::cluster_group cl = cg::this_cluster();
    const int c = cl.block_rank();
    const int t = threadIdx.x;
    const int j = t & 63, v = t >> 6;
    uint32_t x[32];
#pragma unroll
    for (int e = 0; e < 32; e++) x[e] = t * 32 + e;
    uint32_t *rem[kC];
#pragma unroll
    for (int k = 0; k < kC; k++) rem[k] = cl.map_shared_rank(xs, k);
    cl.sync();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int h = 0; h < 4; h++)
#pragma unroll
            for (int kk = 0; kk < 8; kk++)
                rem[kk][(v + 8 * h) * kN1 + c * 64 + j] = x[h * 8 + kk] + it;
        cl.sync();
#pragma unroll
        for (int e = 0; e < 32; e++) x[e] ^= xs[(t * 32 + e * 17) & (kRowsPerCta * kN1 - 1)];
        cl.sync();
    }
    const unsigned long long t1 = clock64();
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
    uint32_t s = 0;
#pragma unroll
    for (int e = 0; e < 32; e++) s += x[e];
    if (s == 0x12345678u) sink[0] = s;
}

// the same volume with 16-byte remote stores (a warp writes 512 contiguous bytes per store)
__global__ void __cluster_dims__(kC, 1, 1) __launch_bounds__(512, 1)
exchange_v4(int iters, unsigned long long *cyc, uint32_t *sink) {
    extern __shared__ uint4 xs4[];     // [32 rows][512] chunk as 4096 uint4
    cg::cluster_group cl = cg::this_cluster();
    const int t = threadIdx.x;
    uint4 x[8];
#pragma unroll
    for (int e = 0; e < 8; e++) x[e] = make_uint4(t, e, t + e, t ^ e);
    uint4 *rem[kC];
#pragma unroll
    for (int k = 0; k < kC; k++) rem[k] = cl.map_shared_rank(xs4, k);
    cl.sync();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int kk = 0; kk < 8; kk++) {
            uint4 v = x[kk]; v.x += it;
            rem[kk][(t >> 5) * 256 + c_rank_off(cl.block_rank()) + (t & 31)] = v;
        }
        cl.sync();
#pragma unroll
        for (int e = 0; e < 8; e++) x[e].y ^= xs4[(t * 8 + e * 17) & 4095].x;
        cl.sync();
    }
    const unsigned long long t1 = clock64();
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
    uint32_t s = 0;
#pragma unroll
    for (int e = 0; e < 8; e++) s += x[e].x + x[e].y;
    if (s == 0x12345678u) sink[0] = s;
}

__global__ void __cluster_dims__(kC, 1, 1) __launch_bounds__(512, 1)
sync_only(int iters, unsigned long long *cyc) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; it++) { cl.sync(); cl.sync(); }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int dev = 0;
    CK(cudaSetDevice(dev));
    cudaDeviceProp pr;
    CK(cudaGetDeviceProperties(&pr, dev));
    CK(cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    printf("{\"sms\": %d, \"occupancy\": [", pr.multiProcessorCount);
    const int cfg[][2] = {{512, 200 * 1024}, {256, 100 * 1024}, {1024, 200 * 1024}};
    bool first = true;
    for (auto &c : cfg) {
        for (int cs : {1, 2, 4, 8, 16}) {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(cs * 64);
            lc.blockDim = dim3(c[0]);
            lc.dynamicSmemBytes = c[1];
            cudaLaunchAttribute at;
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = cs; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
            lc.attrs = &at; lc.numAttrs = 1;
            int ncl = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void *)dummy, &lc);
            printf("%s{\"threads\": %d, \"smem\": %d, \"cluster\": %d, \"max_active_clusters\": %d, \"ctas\": %d%s}",
                   first ? "" : ", ", c[0], c[1], cs, ncl, ncl * cs, e == cudaSuccess ? "" : ", \"err\": 1");
            first = false;
            cudaGetLastError();
        }
    }
    printf("]");
    const int smem = kRowsPerCta * kN1 * 4;
    CK(cudaFuncSetAttribute(exchange, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    unsigned long long *cyc;
    uint32_t *sink;
    const int grid = 128;
    CK(cudaMalloc(&cyc, grid * sizeof(unsigned long long)));
    CK(cudaMalloc(&sink, 4));
    const int iters = 200;
    exchange<<<grid, 512, smem>>>(iters, cyc, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    exchange<<<grid, 512, smem>>>(iters, cyc, sink);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[grid];
    CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
    unsigned long long mx = 0; for (int i = 0; i < grid; i++) mx = h[i] > mx ? h[i] : mx;
    printf(", \"exchange\": {\"cluster\": %d, \"bytes_per_cta\": %d, \"cycles_per_iter\": %.1f, \"ms\": %.3f}",
           kC, smem, (double)mx / iters, ms);
    CK(cudaFuncSetAttribute(exchange_v4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    exchange_v4<<<grid, 512, smem>>>(iters, cyc, sink);
    CK(cudaDeviceSynchronize());
    exchange_v4<<<grid, 512, smem>>>(iters, cyc, sink);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
    mx = 0; for (int i = 0; i < grid; i++) mx = h[i] > mx ? h[i] : mx;
    printf(", \"exchange_v4\": {\"bytes_per_cta\": %d, \"cycles_per_iter\": %.1f}", smem, (double)mx / iters);
    sync_only<<<grid, 512>>>(iters, cyc);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
    mx = 0; for (int i = 0; i < grid; i++) mx = h[i] > mx ? h[i] : mx;
    printf(", \"two_cluster_syncs_cycles\": %.1f}\n", (double)mx / iters);
    return 0;
}
