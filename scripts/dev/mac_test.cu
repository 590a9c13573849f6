// dev check + timing: row_mac variants vs old row_pass<ROW_MAC> on a real context's buffers
#include "../../paper_2105_13678_b200/csrc/pa_api.cu"
#include <cstdlib>
template <int S_LOG, int E_LOG, int DBG = 0, int PAD = mac_pad(S_LOG)>
static float run_variant(const StageDev &sd, pa_ctx *c, uint32_t *out, int reps) {
    const uint32_t P = sd.pl.nprimes;
    MacArgs M{}; M.nt = ntt_args(sd, 0, 1, E_LOG); M.src = c->scratch; M.ahat = c->ahat; M.dst = out; M.nvec = c->nblk;
    M.nunits = (sd.pl.n_col / mac_v(S_LOG)) * P;
    auto fn = row_mac<S_LOG, E_LOG, DBG, PAD>;
    const int thr = mac_threads(S_LOG, E_LOG);
    const size_t sm = mac_smem_bytes<S_LOG, PAD>();
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, thr, sm);
    const int grid = std::min<int>(3 * M.nunits, occ * 148);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9;
    for (int i = 0; i < reps; i++) {
        cudaMemset(out, 0, (size_t)P * sd.L * 4);
        cudaEventRecord(a);
        fn<<<grid, thr, sm>>>(M);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        best = std::min(best, ms);
    }
    printf("  row_mac<%d,%d,dbg%d,pad%d>: threads %d occ %d grid %d  best %.1f us\n", S_LOG, E_LOG, DBG, PAD, thr, occ, grid, best * 1e3);
    return best;
}
int main(int argc, char **argv) {
    uint64_t n = argc > 1 ? atoll(argv[1]) : 260000000ull, r = argc > 2 ? atoll(argv[2]) : (1ull << 23), m = argc > 3 ? atoll(argv[3]) : 26000000ull;
    pa_ctx *c = pa_ctx_create(n, r, m, 0, 42);
    if (!c) { char b[512]; pa_last_error(b, 512); printf("create failed %s\n", b); return 1; }
    StageDev &sd = c->smmh;
    const uint32_t P = sd.pl.nprimes, L = sd.L, nvec = c->nblk;
    std::vector<uint32_t> h((size_t)nvec * P * L);
    uint64_t st = 1;
    for (uint32_t iv = 0; iv < nvec; iv++)
        for (uint32_t pi = 0; pi < P; pi++)
            for (uint32_t j = 0; j < L; j++) { st = st * 6364136223846793005ull + 1442695040888963407ull; h[((size_t)iv * P + pi) * L + j] = (uint32_t)(st >> 33) % (2 * sd.pl.primes[pi]); }
    cudaMemcpy(c->scratch, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    const int rlog = __builtin_ctz(sd.pl.n_row);
    uint32_t *o1, *o2;
    cudaMalloc(&o1, (size_t)P * L * 4); cudaMalloc(&o2, (size_t)P * L * 4);
    RowArgs R{}; R.nt = ntt_args(sd, 0, 1); R.src = c->scratch; R.dst = o1; R.ahat = c->ahat; R.nvec = nvec;
    launch_row<ROW_MAC>(rlog, R, 0);
    cudaDeviceSynchronize();
    std::vector<uint32_t> a((size_t)P * L), b((size_t)P * L);
    cudaMemcpy(a.data(), o1, a.size() * 4, cudaMemcpyDeviceToHost);
    printf("n=%llu r=%llu rlog=%d n_col=%u nvec=%u P=%u\n", (unsigned long long)n, (unsigned long long)r, rlog, sd.pl.n_col, nvec, P);
    auto check = [&](const char *name) {
        cudaMemcpy(b.data(), o2, b.size() * 4, cudaMemcpyDeviceToHost);
        size_t bad = 0;
        for (uint32_t pi = 0; pi < P; pi++)
            for (uint32_t j = 0; j < L; j++) {
                const size_t i = (size_t)pi * L + j;
                if (a[i] % sd.pl.primes[pi] != b[i] % sd.pl.primes[pi]) bad++;
            }
        printf("  %s: bad=%zu/%zu err=%s\n", name, bad, a.size(), cudaGetErrorString(cudaGetLastError()));
    };
    const int reps = 10;
    if (rlog == 10) {
        run_variant<10, 5>(sd, c, o2, reps); check("E32");
        run_variant<10, 5, 1>(sd, c, o2, reps);
        run_variant<10, 5, 2>(sd, c, o2, reps);
        run_variant<10, 4>(sd, c, o2, reps); check("E16");
    } else if (rlog == 9) {
        run_variant<9, 5>(sd, c, o2, reps); check("E32");
        run_variant<9, 5, 0, 0>(sd, c, o2, reps); check("E32 swizzle");
        run_variant<9, 5, 1>(sd, c, o2, reps);
        run_variant<9, 5, 2>(sd, c, o2, reps);
        run_variant<9, 4>(sd, c, o2, reps); check("E16");
    } else if (rlog == 5) {
        run_variant<5, 5>(sd, c, o2, reps); check("E32");
        run_variant<5, 4>(sd, c, o2, reps); check("E16");
    }
    pa_ctx_destroy(c);
}
