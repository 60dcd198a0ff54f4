// Instantiations of the tensor-core MTTKRP kernel for NB = 5 column groups
// of 8 (split per TU to keep nvcc parallel). See mttkrp_tc.cuh.
#include "mttkrp_tc.cuh"
#include "kernels.h"

namespace dmtkg {

template <int TAIL, bool KM>
static void launch_one(const TcPlan& p, const CUtensorMap& map, int grid, cudaStream_t s) {
    auto k = mttkrp_tc_kernel<5, TAIL, KM>;
    static int opted = 0;  // raise the opt-in once (not a stream op: stays out of graph captures)
    if (p.smem > opted) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        opted = 227 * 1024;
    }
    k<<<grid, kThreads, p.smem, s>>>(map, p);
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

template <int TAIL>
static int smem_of(int G, int stages) {
    using Cfg = TcCfg<5, TAIL>;
    return Cfg::FIXED + stages * (Cfg::A_BYTES + G * Cfg::B_BYTES);
}

int tc_smem_nb5(int tail, int G, int stages) {
    switch (tail) {
        case 0: return smem_of<0>(G, stages);
        case 1: return smem_of<1>(G, stages);
        case 2: return smem_of<2>(G, stages);
        case 4: return smem_of<4>(G, stages);
        default: return -1;
    }
}

}  // namespace dmtkg
