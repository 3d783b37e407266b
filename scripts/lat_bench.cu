// lat_bench.cu — microbenchmark (not product code): latency of dependent random 4-byte
// loads as a function of the footprint they are spread over (TLB reach), and at two
// load levels.  Each thread runs a chain: i_{k+1} = hash(a[i_k] + k) mod N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/lat_bench scripts/lat_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    return x;
}

__global__ void chase(const uint32_t* __restrict__ a, uint64_t n, int steps, uint64_t* out, int mode) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t i = mix(tid * 0x9E3779B97F4A7C15ull + 1) % n;
    uint32_t acc = 0;
    for (int k = 0; k < steps; k++) {
        uint32_t v;
        if (mode == 0) v = __ldcg(a + i);
        else v = __ldg(a + i);
        acc += v;
        i = mix(i + v + k) % n;
    }
    if (acc == 0x12345u) out[0] = i;
}

int main() {
    const uint64_t max_bytes = 16ull << 30;
    uint32_t* a;
    if (cudaMalloc(&a, max_bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(a, 0, max_bytes);
    uint64_t* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int steps = 64;
    const uint64_t sizes[] = {32ull << 20, 128ull << 20, 512ull << 20, 1ull << 30, 2ull << 30, 4ull << 30, 8ull << 30, 16ull << 30};
    const int threads[][2] = {{148, 32}, {148, 256}, {148, 1024}};
    printf("footprint_MB, ctas x threads, ns per dependent load (per thread), G loads/s\n");
    for (auto& t : threads) {
        for (uint64_t s : sizes) {
            const uint64_t n = s / 4;
            chase<<<t[0], t[1]>>>(a, n, 8, out, 0);
            cudaEventRecord(e0);
            chase<<<t[0], t[1]>>>(a, n, steps, out, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ns = ms * 1e6 / steps;
            printf("%8llu, %4d x %4d, %8.1f, %8.2f\n", (unsigned long long)(s >> 20), t[0], t[1], ns,
                   (double)t[0] * t[1] * steps / (ms * 1e-3) / 1e9);
        }
    }
    cudaError_t err = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(err));
    return 0;
}
