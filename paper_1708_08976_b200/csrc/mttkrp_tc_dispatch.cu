// Dispatch over the (NB, RB) instantiation units of the tensor-core MTTKRP
// (mttkrp_tc_inst.cu). Taller tiles (RB = 3, 4) exist for NB <= 3: wider
// ranks would exceed the 168-register budget with 3-4 row blocks per warp.
#include "kernels.h"

namespace dmtkg {

#define DMTKG_UNIT(N, R)                                                                   \
    bool launch_tc_##N##_##R(const TcPlan&, const CUtensorMap&, int, bool, int, cudaStream_t); \
    int tc_smem_##N##_##R(int, int, int);
DMTKG_UNIT(1, 2) DMTKG_UNIT(2, 2) DMTKG_UNIT(3, 2) DMTKG_UNIT(4, 2)
DMTKG_UNIT(5, 2) DMTKG_UNIT(6, 2) DMTKG_UNIT(7, 2) DMTKG_UNIT(8, 2)
DMTKG_UNIT(1, 3) DMTKG_UNIT(2, 3) DMTKG_UNIT(3, 3)
DMTKG_UNIT(1, 4) DMTKG_UNIT(2, 4) DMTKG_UNIT(3, 4)
#undef DMTKG_UNIT

// Shapes that compile without local-memory spills (ptxas -v, 168 registers).
bool tc_has_tile(int nb, int tail, int rb) {
    if (rb == 2) return nb >= 1 && nb <= 8;
    if (nb < 1 || nb > 3 || tail > 2) return false;
    if (rb == 3) return true;
    return rb == 4 && (tail <= 1 || nb == 1);
}

bool launch_mttkrp_tc(const TcPlan& p, const CUtensorMap& map, int nb, int tail, bool kmajor, int grid,
                      cudaStream_t s) {
#define DMTKG_CASE(N, R) \
    if (nb == N && p.RB == R) return launch_tc_##N##_##R(p, map, tail, kmajor, grid, s);
    DMTKG_CASE(1, 2) DMTKG_CASE(2, 2) DMTKG_CASE(3, 2) DMTKG_CASE(4, 2)
    DMTKG_CASE(5, 2) DMTKG_CASE(6, 2) DMTKG_CASE(7, 2) DMTKG_CASE(8, 2)
    DMTKG_CASE(1, 3) DMTKG_CASE(2, 3) DMTKG_CASE(3, 3)
    DMTKG_CASE(1, 4) DMTKG_CASE(2, 4) DMTKG_CASE(3, 4)
#undef DMTKG_CASE
    return false;
}

int tc_smem_bytes(int nb, int tail, int G, int stages, int rb) {
#define DMTKG_CASE(N, R) \
    if (nb == N && rb == R) return tc_smem_##N##_##R(tail, G, stages);
    DMTKG_CASE(1, 2) DMTKG_CASE(2, 2) DMTKG_CASE(3, 2) DMTKG_CASE(4, 2)
    DMTKG_CASE(5, 2) DMTKG_CASE(6, 2) DMTKG_CASE(7, 2) DMTKG_CASE(8, 2)
    DMTKG_CASE(1, 3) DMTKG_CASE(2, 3) DMTKG_CASE(3, 3)
    DMTKG_CASE(1, 4) DMTKG_CASE(2, 4) DMTKG_CASE(3, 4)
#undef DMTKG_CASE
    return -1;
}

}  // namespace dmtkg
