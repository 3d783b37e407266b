// inst.cu — explicit instantiation of the round-loop kernels for one policy and one
// bidirectional setting (INST_POL, INST_BIDIR), compiled once per pair in parallel by build.py.
#include "loop.cuh"

#ifndef INST_POL
#error "compile with -DINST_POL=<policy> -DINST_BIDIR=<0|1>"
#endif

namespace sssp {

#define SSSP_TABLE_NAME2(P, B) kernel_table_##P##_##B
#define SSSP_TABLE_NAME(P, B) SSSP_TABLE_NAME2(P, B)

KernelFn SSSP_TABLE_NAME(INST_POL, INST_BIDIR)(bool stats, bool fuse) {
    constexpr bool B = INST_BIDIR != 0;
    if (fuse) return stats ? sssp_round_loop<INST_POL, true, true, B> : sssp_round_loop<INST_POL, false, true, B>;
    return stats ? sssp_round_loop<INST_POL, true, false, B> : sssp_round_loop<INST_POL, false, false, B>;
}

}  // namespace sssp
