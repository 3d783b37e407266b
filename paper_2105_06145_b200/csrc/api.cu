// api.cu — status strings and the thread-local error detail of the C ABI.
#include <stdarg.h>
#include <stdio.h>

#include "internal.h"

namespace sssp {

static thread_local char g_err[512] = "";

sssp_status set_error(sssp_status s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}

sssp_status cuda_error(cudaError_t e, const char* what) {
    return set_error(SSSP_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

}  // namespace sssp

extern "C" {

const char* sssp_status_string(sssp_status s) {
    switch (s) {
        case SSSP_OK: return "SSSP_OK";
        case SSSP_ERR_INVALID: return "SSSP_ERR_INVALID";
        case SSSP_ERR_INVALID_GRAPH: return "SSSP_ERR_INVALID_GRAPH";
        case SSSP_ERR_RANGE: return "SSSP_ERR_RANGE";
        case SSSP_ERR_CAPACITY: return "SSSP_ERR_CAPACITY";
        case SSSP_ERR_CUDA: return "SSSP_ERR_CUDA";
        case SSSP_ERR_ROUNDS: return "SSSP_ERR_ROUNDS";
        case SSSP_ERR_DEVICE: return "SSSP_ERR_DEVICE";
        case SSSP_ERR_INTERNAL: return "SSSP_ERR_INTERNAL";
    }
    return "SSSP_ERR_UNKNOWN";
}

const char* sssp_last_error(void) { return sssp::g_err; }

int32_t sssp_abi_version(void) { return SSSP_ABI_VERSION; }

}  // extern "C"
