// One instantiation unit of the tensor-core MTTKRP kernel (mttkrp_tc.cuh),
// compiled once per (NB, RB) pair by the Makefile with -DTC_NB=.. -DTC_RB=..
// (split per TU to keep nvcc parallel). Exports launch_tc_<NB>_<RB> and
// tc_smem_<NB>_<RB> for mttkrp_tc_dispatch.cu.
#include "kernels.h"
#include "mttkrp_tc.cuh"

#ifndef TC_NB
#error "compile with -DTC_NB=<column groups> -DTC_RB=<row blocks per warp>"
#endif

#define TC_CAT_(a, b, c, d) a##b##_##c##d
#define TC_CAT(a, b, c, d) TC_CAT_(a, b, c, d)
#define TC_LAUNCH TC_CAT(launch_tc_, TC_NB, , TC_RB)
#define TC_SMEM TC_CAT(tc_smem_, TC_NB, , TC_RB)

namespace dmtkg {

// DFMA tails the unit instantiates: 1 and 2 everywhere, 4 (only reachable
// with DMTK_GPU_MAX_TAIL=4) on 128-row tiles.
constexpr bool tc_has_tail(int tail) { return tail == 0 || tail == 1 || tail == 2 || (tail == 4 && TC_RB == 2); }

template <int TAIL, bool KM, int EPI = kEpiGen>
static void launch_one(const TcPlan& p, const CUtensorMap& map, int grid, cudaStream_t s) {
    if constexpr (tc_has_tail(TAIL)) {
        auto k = mttkrp_tc_kernel<TC_NB, TAIL, KM, TC_RB, EPI>;
        static std::atomic<unsigned long long> opted{0};  // per device; not a stream op (graph-safe)
        once_on_device(opted, [k] { cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024); });
        launch_pdl(k, dim3(grid), dim3(tc_threads(TC_RB)), p.smem, s, map, p);
    }
}

bool TC_LAUNCH(const TcPlan& p, const CUtensorMap& map, int tail, bool kmajor, int grid, cudaStream_t s) {
    if (p.RB != TC_RB || !tc_has_tail(tail)) return false;
    // one-flavor epilogue instantiations (tails 0-2), else the general kernel;
    // the 1-step/2-step ones only up to 3 column groups (measured 1-2% slower
    // than the general kernel at C = 32 and 50, 1-6% faster at C <= 25)
    if (p.epi != kEpiGen && tail <= 2 && (p.epi == kEpiMM) != kmajor) {
        switch (p.epi * 4 + tail) {
            case kEpiSwr * 4 + 0: launch_one<0, true, kEpiSwr>(p, map, grid, s); return true;
            case kEpiSwr * 4 + 1: launch_one<1, true, kEpiSwr>(p, map, grid, s); return true;
            case kEpiSwr * 4 + 2: launch_one<2, true, kEpiSwr>(p, map, grid, s); return true;
#if TC_NB <= 3
            case kEpiMM * 4 + 0: launch_one<0, false, kEpiMM>(p, map, grid, s); return true;
            case kEpiMM * 4 + 1: launch_one<1, false, kEpiMM>(p, map, grid, s); return true;
            case kEpiMM * 4 + 2: launch_one<2, false, kEpiMM>(p, map, grid, s); return true;
            case kEpiKJ * 4 + 0: launch_one<0, true, kEpiKJ>(p, map, grid, s); return true;
            case kEpiKJ * 4 + 1: launch_one<1, true, kEpiKJ>(p, map, grid, s); return true;
            case kEpiKJ * 4 + 2: launch_one<2, true, kEpiKJ>(p, map, grid, s); return true;
            case kEpiJK * 4 + 0: launch_one<0, true, kEpiJK>(p, map, grid, s); return true;
            case kEpiJK * 4 + 1: launch_one<1, true, kEpiJK>(p, map, grid, s); return true;
            case kEpiJK * 4 + 2: launch_one<2, true, kEpiJK>(p, map, grid, s); return true;
#endif
            default: break;
        }
    }
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
    using Cfg = TcCfg<TC_NB, TAIL, TC_RB>;
    return Cfg::FIXED + stages * (Cfg::A_BYTES + G * Cfg::B_BYTES);
}

// -1: no instantiation for this tail
int TC_SMEM(int tail, int G, int stages) {
    if (!tc_has_tail(tail)) return -1;
    switch (tail) {
        case 0: return smem_of<0>(G, stages);
        case 1: return smem_of<1>(G, stages);
        case 2: return smem_of<2>(G, stages);
        case 4: return smem_of<4>(G, stages);
        default: return -1;
    }
}

}  // namespace dmtkg
