// Dispatch over the per-NB instantiation TUs of the tensor-core MTTKRP.
#include "kernels.h"

namespace dmtkg {

#define DMTKG_NB(X) \
    bool launch_tc_nb##X(const TcPlan&, const CUtensorMap&, int, bool, int, cudaStream_t); \
    int tc_smem_nb##X(int, int, int);
DMTKG_NB(1) DMTKG_NB(2) DMTKG_NB(3) DMTKG_NB(4) DMTKG_NB(5) DMTKG_NB(6) DMTKG_NB(7) DMTKG_NB(8)
#undef DMTKG_NB

bool launch_mttkrp_tc(const TcPlan& p, const CUtensorMap& map, int nb, int tail, bool kmajor, int grid,
                      cudaStream_t s) {
    switch (nb) {
        case 1: return launch_tc_nb1(p, map, tail, kmajor, grid, s);
        case 2: return launch_tc_nb2(p, map, tail, kmajor, grid, s);
        case 3: return launch_tc_nb3(p, map, tail, kmajor, grid, s);
        case 4: return launch_tc_nb4(p, map, tail, kmajor, grid, s);
        case 5: return launch_tc_nb5(p, map, tail, kmajor, grid, s);
        case 6: return launch_tc_nb6(p, map, tail, kmajor, grid, s);
        case 7: return launch_tc_nb7(p, map, tail, kmajor, grid, s);
        case 8: return launch_tc_nb8(p, map, tail, kmajor, grid, s);
        default: return false;
    }
}

int tc_smem_bytes(int nb, int tail, int G, int stages) {
    switch (nb) {
        case 1: return tc_smem_nb1(tail, G, stages);
        case 2: return tc_smem_nb2(tail, G, stages);
        case 3: return tc_smem_nb3(tail, G, stages);
        case 4: return tc_smem_nb4(tail, G, stages);
        case 5: return tc_smem_nb5(tail, G, stages);
        case 6: return tc_smem_nb6(tail, G, stages);
        case 7: return tc_smem_nb7(tail, G, stages);
        case 8: return tc_smem_nb8(tail, G, stages);
        default: return -1;
    }
}

}  // namespace dmtkg
