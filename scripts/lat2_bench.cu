// lat2_bench.cu — microbenchmark (not product code): unloaded latency of one dependent
// access by a single thread: pointer chase over a random cyclic permutation (no index
// arithmetic), for L1-, L2- and HBM-sized footprints, with plain / .cg / .ca loads and
// with atomicCAS (the chase value is the CAS return).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/lat2_bench scripts/lat2_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <algorithm>
#include <random>

template <int MODE>
__global__ void chase(uint32_t* a, int steps, uint32_t* out, long long* cyc) {
    uint32_t i = 0;
    const long long t0 = clock64();
    for (int k = 0; k < steps; k++) {
        if (MODE == 0) i = __ldcg(a + i);
        else if (MODE == 1) i = __ldca(a + i);
        else if (MODE == 2) i = atomicCAS(a + i, 0xFFFFFFFFu, 0xFFFFFFFEu);  // never matches: returns the word
        else i = atomicOr(a + i, 0u);
    }
    const long long t1 = clock64();
    out[0] = i;
    cyc[0] = t1 - t0;
}

int main() {
    const size_t sizes[] = {16 << 10, 1 << 20, 32 << 20, 256 << 20, 1ull << 30};
    uint32_t *d, *out;
    long long* cyc;
    cudaMalloc(&d, 1ull << 30);
    cudaMalloc(&out, 4);
    cudaMalloc(&cyc, 8);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("footprint, mode, cycles/access, ns/access (at the SM clock during the run)\n");
    const char* names[] = {"ld.cg", "ld.ca", "atomicCAS", "atomicOr"};
    for (size_t s : sizes) {
        // one random cycle over s/128 lines (one element per 128-byte line)
        const size_t lines = s / 128;
        std::vector<uint32_t> perm(lines);
        for (size_t i = 0; i < lines; i++) perm[i] = (uint32_t)i;
        std::mt19937_64 g(1);
        std::shuffle(perm.begin() + 1, perm.end(), g);
        std::vector<uint32_t> h(s / 4, 0);
        for (size_t i = 0; i < lines; i++) h[(size_t)perm[i] * 32] = perm[(i + 1) % lines] * 32;
        cudaMemcpy(d, h.data(), s, cudaMemcpyHostToDevice);
        for (int mode = 0; mode < 4; mode++) {
            const int steps = 4096;
            for (int rep = 0; rep < 2; rep++) {  // first pass warms the caches
                if (mode == 0) chase<0><<<1, 1>>>(d, steps, out, cyc);
                else if (mode == 1) chase<1><<<1, 1>>>(d, steps, out, cyc);
                else if (mode == 2) chase<2><<<1, 1>>>(d, steps, out, cyc);
                else chase<3><<<1, 1>>>(d, steps, out, cyc);
            }
            long long c = 0;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("%10zu KB, %-9s, %7.1f\n", s >> 10, names[mode], (double)c / steps);
        }
    }
    printf("status %s, nominal clock %d MHz\n", cudaGetErrorString(cudaGetLastError()), clk_khz / 1000);
    return 0;
}
