// inst.cu — explicit instantiation of the round-loop kernels for one (policy, bidirectional,
// fusion) triple (INST_POL, INST_BIDIR, INST_FUSE), compiled once per triple in parallel by
// build.py.  A unit may be compiled with its own tuning constants (build.py UNIT_DEFINES), so
// it also exports the dynamic shared memory its kernels need.
#include "loop.cuh"

#if !defined(INST_POL) || !defined(INST_BIDIR) || !defined(INST_FUSE)
#error "compile with -DINST_POL=<policy> -DINST_BIDIR=<0|1> -DINST_FUSE=<0|1>"
#endif

namespace sssp {

#define SSSP_UNIT_NAME2(X, P, B, F) X##_##P##_##B##_##F
#define SSSP_UNIT_NAME(X, P, B, F) SSSP_UNIT_NAME2(X, P, B, F)

KernelUnit SSSP_UNIT_NAME(kernel_unit, INST_POL, INST_BIDIR, INST_FUSE)() {
    constexpr bool B = INST_BIDIR != 0, F = INST_FUSE != 0;
    return KernelUnit{sssp_round_loop<INST_POL, false, F, B>, sssp_round_loop<INST_POL, true, F, B>, smem_bytes(F), kBlock};
}

}  // namespace sssp
