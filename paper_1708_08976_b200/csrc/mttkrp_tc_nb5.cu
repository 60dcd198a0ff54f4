// Instantiations of the tensor-core MTTKRP kernel for NB = 5 column groups
// of 8 (split per TU to keep nvcc parallel). See mttkrp_tc.cuh.
#include "mttkrp_tc.cuh"
#include "kernels.h"

namespace dmtkg {

template <int TAIL, bool KM>
static void launch_one(const TcPlan& p, const CUtensorMap& map, int grid, cudaStream_t s) {
    auto k = mttkrp_tc_kernel<5, TAIL, KM>;
    const int smem = TcCfg<5, TAIL>::SMEM;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<grid, kThreads, smem, s>>>(map, p);
}

bool launch_tc_nb5(const TcPlan& p, const CUtensorMap& map, int tail, bool kmajor, int grid, cudaStream_t s) {
    switch (tail * 2 + (kmajor ? 1 : 0)) {
        case 0: launch_one<0, false>(p, map, grid, s); return true;
        case 1: launch_one<0, true>(p, map, grid, s); return true;
        case 2: launch_one<1, false>(p, map, grid, s); return true;
        case 3: launch_one<1, true>(p, map, grid, s); return true;
        case 4: launch_one<2, false>(p, map, grid, s); return true;
        case 5: launch_one<2, true>(p, map, grid, s); return true;
        case 8: launch_one<4, false>(p, map, grid, s); return true;
        case 9: launch_one<4, true>(p, map, grid, s); return true;
        default: return false;
    }
}

int tc_smem_nb5(int tail) {
    switch (tail) {
        case 0: return TcCfg<5, 0>::SMEM;
        case 1: return TcCfg<5, 1>::SMEM;
        case 2: return TcCfg<5, 2>::SMEM;
        case 4: return TcCfg<5, 4>::SMEM;
        default: return -1;
    }
}

}  // namespace dmtkg
