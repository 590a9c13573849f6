// dev check: new row_mac vs old row_pass<ROW_MAC> on a real context's buffers
#include "../../paper_2105_13678_b200/csrc/pa_api.cu"
#include <cstdlib>
int main(int argc, char **argv) {
    uint64_t n = argc > 1 ? atoll(argv[1]) : 100000000ull, r = argc > 2 ? atoll(argv[2]) : (1ull << 22), m = argc > 3 ? atoll(argv[3]) : 10000000ull;
    pa_ctx *c = pa_ctx_create(n, r, m, 0, 42);
    if (!c) { char b[512]; pa_last_error(b, 512); printf("create failed %s\n", b); return 1; }
    StageDev &sd = c->smmh;
    const uint32_t P = sd.pl.nprimes, L = sd.L, nvec = c->nblk;
    // random scratch in [0, 2p)
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
    int rc = launch_row<ROW_MAC>(rlog, R, 0);
    cudaMemset(o2, 0, (size_t)P * L * 4);
    MacArgs M{}; M.nt = ntt_args(sd, 0, 1); M.src = c->scratch; M.ahat = c->ahat; M.dst = o2; M.nvec = nvec;
    M.nunits = (sd.pl.n_col / mac_v_rt(rlog)) * P;
    int rc2 = launch_mac(rlog, M, 0);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint32_t> a((size_t)P * L), b((size_t)P * L);
    cudaMemcpy(a.data(), o1, a.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), o2, b.size() * 4, cudaMemcpyDeviceToHost);
    size_t bad = 0, first = ~0ull;
    for (uint32_t pi = 0; pi < P; pi++)
        for (uint32_t j = 0; j < L; j++) {
            const size_t i = (size_t)pi * L + j;
            if (a[i] % sd.pl.primes[pi] != b[i] % sd.pl.primes[pi]) { bad++; if (first == ~0ull) first = i; }
        }
    printf("n=%llu r=%llu rlog=%d n_col=%u V=%u nvec=%u rc=%d/%d err=%s bad=%zu/%zu first=%zu\n", (unsigned long long)n,
           (unsigned long long)r, rlog, sd.pl.n_col, mac_v_rt(rlog), nvec, rc, rc2, cudaGetErrorString(e), bad, a.size(), first);
    if (first != ~0ull) {
        size_t i = first;
        printf("  old %u new %u (row %zu col %zu)\n", a[i], b[i], (i % L) / sd.pl.n_row, i % sd.pl.n_row);
    }
    pa_ctx_destroy(c);
}
