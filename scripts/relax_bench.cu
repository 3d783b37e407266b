// relax_bench.cu — microbenchmarks (not product code): hardware ceilings of the relax
// access pattern on a real CSR (streamed idx/w + random gathers into an 8n- or 4n-byte
// array + atomics), to tell latency limits from bandwidth limits in the round loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -shared \
//        -o scripts/librelaxbench.so scripts/relax_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>

// mode 0: stream idx+w only; 1: + gather u64 dist[v]; 2: + gather u32 key[v];
// 3: relax = gather + atomicMin(u64) when smaller (dist pre-filled so ~rate% succeed);
// 4: blind RED.MIN u64 on dist (no gather, no return); 5: blind RED.MIN u32 on key
template <int MODE, int ARCS>
__global__ void __launch_bounds__(512) k_relax(int64_t m, const int32_t* __restrict__ idx, const uint32_t* __restrict__ w,
                                               unsigned long long* dist, const uint32_t* key, unsigned long long* out) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    unsigned long long acc = 0;
    for (int64_t base = tid; base < m; base += nth * ARCS) {
        int32_t v[ARCS];
        uint32_t ww[ARCS];
#pragma unroll
        for (int t = 0; t < ARCS; t++) {
            const int64_t e = base + (int64_t)t * nth;
            v[t] = e < m ? __ldcs(idx + e) : -1;
            ww[t] = e < m ? __ldcs(w + e) : 0;
        }
        if (MODE == 0) {
#pragma unroll
            for (int t = 0; t < ARCS; t++) acc += (unsigned)v[t] + ww[t];
        } else if (MODE == 1) {
#pragma unroll
            for (int t = 0; t < ARCS; t++) acc += v[t] >= 0 ? __ldcg(dist + v[t]) + ww[t] : 0;
        } else if (MODE == 2) {
#pragma unroll
            for (int t = 0; t < ARCS; t++) acc += v[t] >= 0 ? __ldcg(key + v[t]) + ww[t] : 0;
        } else if (MODE == 4) {  // blind WriteMin: RED.MIN (no return value, nothing waits on it)
#pragma unroll
            for (int t = 0; t < ARCS; t++)
                if (v[t] >= 0) atomicMin(dist + v[t], (unsigned long long)ww[t] * 4);
        } else if (MODE == 5) {  // blind RED.MIN on a 4n-byte (L2-resident) array
#pragma unroll
            for (int t = 0; t < ARCS; t++)
                if (v[t] >= 0) atomicMin((unsigned*)key + v[t], ww[t] * 4u);
        } else {
            unsigned long long cur[ARCS];
#pragma unroll
            for (int t = 0; t < ARCS; t++) cur[t] = v[t] >= 0 ? __ldcg(dist + v[t]) : 0;
#pragma unroll
            for (int t = 0; t < ARCS; t++) {
                const unsigned long long c = (unsigned long long)ww[t] * 4;  // candidate
                if (v[t] >= 0 && c < cur[t]) acc += atomicMin(dist + v[t], c);
            }
        }
    }
    if (acc == 0x123456789ull) *out = acc;  // keep the loads alive
}

extern "C" float relax_bench(int mode, int arcs, int blocks, int64_t m, const int32_t* idx, const uint32_t* w,
                             unsigned long long* dist, const uint32_t* key, unsigned long long* out, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto launch = [&]() {
#define L(MO, AR) k_relax<MO, AR><<<blocks, 512>>>(m, idx, w, dist, key, out)
        if (arcs == 4) {
            if (mode == 0) L(0, 4); else if (mode == 1) L(1, 4); else if (mode == 2) L(2, 4); else if (mode == 3) L(3, 4); else if (mode == 4) L(4, 4); else L(5, 4);
        } else if (arcs == 8) {
            if (mode == 0) L(0, 8); else if (mode == 1) L(1, 8); else if (mode == 2) L(2, 8); else if (mode == 3) L(3, 8); else if (mode == 4) L(4, 8); else L(5, 8);
        } else {
            if (mode == 0) L(0, 16); else if (mode == 1) L(1, 16); else if (mode == 2) L(2, 16); else if (mode == 3) L(3, 16); else if (mode == 4) L(4, 16); else L(5, 16);
        }
#undef L
    };
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < reps; r++) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms / reps;
}
