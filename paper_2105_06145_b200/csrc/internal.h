// internal.h — host-side declarations shared by the library's translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sssp.h"

namespace sssp {

// Thread-local error detail (api.cu).  Returns `s` for chaining.
sssp_status set_error(sssp_status s, const char* fmt, ...);
sssp_status cuda_error(cudaError_t e, const char* what);

// Make the device owning `ptr` current for this (statically linked) runtime.
inline cudaError_t bind_device_of(const void* ptr, int* dev) {
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, ptr);
    if (e != cudaSuccess) return e;
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return cudaErrorInvalidDevicePointer;
    *dev = a.device;
    return cudaSetDevice(a.device);
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Simple bump allocator over a caller workspace; used identically for sizing
// (base == nullptr) and carving.
struct Carver {
    char* base;
    size_t off = 0;
    explicit Carver(void* b) : base((char*)b) {}
    template <typename T>
    T* take(size_t count) {
        off = align_up(off, 256);
        T* p = base ? (T*)(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};

}  // namespace sssp
