// bench_barrier.cu — microbenchmark (not product code): cost of one grid-wide barrier
// inside a persistent cooperative kernel on B200, for the round-loop design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bench_barrier scripts/bench_barrier.cu
//   ./scripts/bench_barrier
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdio.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int MODE>
__device__ __forceinline__ void bar(unsigned* b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned inc = (blockIdx.x == 0) ? (0x80000000u - (gridDim.x - 1)) : 1u;
        __threadfence();
        unsigned old = atomicAdd(b, inc);
        if (MODE == 0) {
            while (((old ^ ld_acquire(b)) & 0x80000000u) == 0) {
            }
        } else {
            while (((old ^ ld_acquire(b)) & 0x80000000u) == 0) __nanosleep(MODE);
        }
        __threadfence();
    }
    __syncthreads();
}

template <int MODE>
__global__ void k_bar(unsigned* b, int iters) {
    for (int i = 0; i < iters; i++) bar<MODE>(b);
}

__global__ void k_cg(int iters) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; i++) g.sync();
}

// dependent L2 loads (pointer chase) from one thread: latency per hop
__global__ void k_chase(const unsigned* next, int hops, unsigned* out) {
    unsigned x = 0;
    for (int i = 0; i < hops; i++) x = __ldcg(next + x);
    *out = x;
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    unsigned* b;
    cudaMalloc(&b, 4096);
    cudaMemset(b, 0, 4096);
    const int iters = 20000;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int threads : {256, 512, 1024}) {
        for (int per_sm : {1, 2, 3, 4}) {
            if (threads * per_sm > 2048) continue;
            int grid = sms * per_sm;
            int ok = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ok, k_bar<0>, threads, 0);
            if (ok < per_sm) continue;
            void* args[] = {&b, (void*)&iters};
            float t0 = timeit([&] { cudaLaunchCooperativeKernel((void*)k_bar<0>, grid, threads, args, 0, 0); });
            float t1 = timeit([&] { cudaLaunchCooperativeKernel((void*)k_bar<32>, grid, threads, args, 0, 0); });
            float t2 = timeit([&] { cudaLaunchCooperativeKernel((void*)k_bar<200>, grid, threads, args, 0, 0); });
            void* args2[] = {(void*)&iters};
            float t3 = timeit([&] { cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args2, 0, 0); });
            printf("grid %4d x %4d: spin %.3f us  nanosleep32 %.3f us  nanosleep200 %.3f us  cg::grid.sync %.3f us\n",
                   grid, threads, t0 * 1e3 / iters, t1 * 1e3 / iters, t2 * 1e3 / iters, t3 * 1e3 / iters);
        }
    }
    // L2-hit and DRAM pointer chase
    for (size_t n : {(size_t)1 << 16, (size_t)1 << 28}) {
        unsigned* nx;
        cudaMalloc(&nx, n * 4);
        unsigned* h = (unsigned*)malloc(n * 4);
        // random cyclic permutation with stride to defeat locality
        unsigned long long s = 88172645463325252ull;
        for (size_t i = 0; i < n; i++) h[i] = (unsigned)i;
        for (size_t i = n - 1; i > 0; i--) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            size_t j = s % i;  // Sattolo: single cycle
            unsigned t = h[i]; h[i] = h[j]; h[j] = t;
        }
        cudaMemcpy(nx, h, n * 4, cudaMemcpyHostToDevice);
        unsigned* out;
        cudaMalloc(&out, 4);
        const int hops = 20000;
        float t = timeit([&] { k_chase<<<1, 1>>>(nx, hops, out); });
        printf("pointer chase over %zu MB: %.1f ns per dependent load\n", n * 4 >> 20, t * 1e6 / hops);
        cudaFree(nx);
        free(h);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
