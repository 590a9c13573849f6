// dev check of the bulk-copy ring protocol used by row_mac (not part of the product)
#include <cstdio>
#include <vector>
#include "../../paper_2105_13678_b200/csrc/bulk.cuh"
using namespace pa;
constexpr int SW = 2048, NS = 2;
__global__ void ring_sum(const uint32_t *src, uint64_t total, uint32_t *out) {
    extern __shared__ __align__(128) uint32_t smem[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + NS * SW);
    const uint64_t it0 = blockIdx.x * total / gridDim.x, it1 = (blockIdx.x + 1) * total / gridDim.x;
    if (threadIdx.x == 0) { for (int s = 0; s < NS; s++) mbar_init(&bars[s], 1); fence_mbar_init(); }
    __syncthreads();
    auto issue = [&](uint64_t it, int s) {
        mbar_arrive_expect_tx(&bars[s], SW * 4);
        bulk_g2s(smem + s * SW, src + it * SW, SW * 4, &bars[s]);
    };
    if (threadIdx.x == 0) for (int s = 0; s < NS; s++) if (it0 + s < it1) issue(it0 + s, s);
    for (uint64_t it = it0; it < it1; it++) {
        const int s = (int)((it - it0) % NS);
        mbar_wait(&bars[s], (uint32_t)(((it - it0) / NS) & 1));
        uint32_t acc = 0;
        for (int i = threadIdx.x; i < SW; i += blockDim.x) acc += smem[s * SW + i];
        atomicAdd(out + it, acc);
        __syncthreads();
        if (threadIdx.x == 0 && it + NS < it1) issue(it + NS, s);
    }
}
int main() {
    const uint64_t total = 5000;
    std::vector<uint32_t> h(total * SW);
    for (size_t i = 0; i < h.size(); i++) h[i] = (uint32_t)(i * 2654435761u);
    uint32_t *d, *o;
    cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, total * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    for (int grid : {1, 7, 148, 600}) {
        cudaMemset(o, 0, total * 4);
        size_t sm = NS * SW * 4 + 64;
        cudaFuncSetAttribute(ring_sum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        ring_sum<<<grid, 64, sm>>>(d, total, o);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint32_t> got(total);
        cudaMemcpy(got.data(), o, total * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (uint64_t it = 0; it < total; it++) {
            uint32_t want = 0;
            for (int i = 0; i < SW; i++) want += h[it * SW + i];
            if (want != got[it]) bad++;
        }
        printf("grid %d: err=%s bad=%d/%llu\n", grid, cudaGetErrorString(e), bad, (unsigned long long)total);
    }
}
