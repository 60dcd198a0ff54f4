// mttkrp_plan.h -- the launch description shared by the host planner
// (plan.cpp) and the tensor-core MTTKRP kernel (mttkrp_tc.cuh).
//
// Every MTTKRP mode is a 3-way contraction over the collapsed view
// X(l, i, j), l in [L = left(n)) fastest, i in [I = I_n), j in [R = right(n)):
//     M(i, c) = sum_{l, j} X(l, i, j) * KL(l, c) * KR(j, c)
// with KL = KRP(U_{n-1}, ..., U_0) and KR = KRP(U_{N-1}, ..., U_{n+1})
// (reference mttkrp.cpp:55-75, 340-376). Three streaming flavors cover the
// reference algorithms:
//   kMMajor   the tensor as a column-major (L*I) x R matrix, contraction over
//             j with the B tile = KR rows built on the fly; epilogue scales
//             row (l, i) by KL(l, :) and sums over l (multi-TTV).
//             = one_step on mode 0 (L == 1) and two_step "right" order.
//   kKMajorJ  rows (i, j), contraction over l with B = KL rows on the fly;
//             epilogue scales by KR(j, :) and sums over j.
//             = one_step on the last mode (R == 1) and two_step "left" order.
//   kKMajorJK rows i, contraction over (j, l) with B = KL(l, :) * KR(j, :)
//             built per stage (KR materialised by a prologue kernel).
//             = one_step on interior modes (reference mttkrp.cpp:165-242).
// swap = 1 runs the paper's 2-step on a boundary mode, where the reference
// has none: mode 0 as kMMajor on the view (L' = I_0, I' = I_1..I_s, R' =
// the rest), output index l (rows of X stay contiguous), scale KRP over i';
// the last mode as kKMajorJ on (L' = I_0..I_{s-1}, I' = I_s..I_{N-2}, R' =
// I_{N-1}), output index j, scale KRP over i'. Small boundary extents then
// no longer set the tile height.
// Work is split stream-K style: the (tile, stage) sequence is cut into
// equal contiguous ranges, one per CTA; each tile segment a CTA finishes
// writes one BM-row slot block to the workspace, and a deterministic CSR
// reduction (reduce kernel) sums the slots of every output row.
#pragma once

#include "common.cuh"

namespace dmtkg {

constexpr int kConsumerWarps = 8;  // two per SM sub-partition
// Tile shape by RB (DMMA row blocks per consumer warp, 2..4): tile rows
// 64 * RB at G = 1; contraction indices per stage (and row group) 32 for
// RB = 2, 16 for taller tiles, so a stage stays 24-32 KB of X.
__host__ __device__ constexpr int tc_bk(int rb) { return rb == 2 ? 32 : 16; }
__host__ __device__ constexpr int tc_bm(int rb) { return kConsumerWarps * 8 * rb; }
// Warp roles: producer, three builders, eight consumers (see mttkrp_tc.cuh).
// (A setmaxnreg rebalance toward the consumers was measured to add spills,
// not remove them: ptxas keeps values live across the role split.)
#ifndef DMTK_TC_BUILDERS
#define DMTK_TC_BUILDERS 3  // (build macro; 2 builders measured 1-5% slower, and 11 warps get the same 168
                            // registers per thread as 12: the register file is allocated per four warps)
#endif
__host__ __device__ constexpr int tc_builders(int) { return DMTK_TC_BUILDERS; }
__host__ __device__ constexpr int tc_threads(int rb) { return (kConsumerWarps + tc_builders(rb) + 1) * 32; }
constexpr int kProducerWarp = 0;
constexpr int kFirstBuilderWarp = 1;

enum Flavor : int { kMMajor = 0, kKMajorJ = 1, kKMajorJK = 2 };

struct TcPlan {
    int flavor;
    int C;                    // rank
    long long L, I, R;        // collapsed view
    int RB;                   // DMMA row blocks per consumer warp (kernel template, 2..4)
    int BK;                   // contraction indices per stage and row group (tc_bk(RB))
    int G;                    // row groups: the BM = tc_bm(RB) tile rows are G groups of TR = BM/G
                              // rows, each group contracting its own BK-index slice of a stage
    int TR;                   // tile rows (BM / G)
    int stages;               // ring depth (2..6)
    int BI, BJ;               // K-major row tile: BI * BJ == TR (kKMajorJK: TR, 1)
    long long n_ti, n_tj;     // tiles along rows (M-major: n_ti = ceil(L*I/TR), n_tj = 1)
    long long stages_per_tile;  // contraction stages per tile (BK * G indices each)
    long long n_lc;           // kKMajorJK: l-chunks of BK * G per j
    long long total_stages;   // n_ti * n_tj * stages_per_tile
    long long kext;           // extent of the B generator index (R for M-major, L for K-major)
    int swap;                 // epilogue keeps the other row index (boundary-mode 2-step, see below)
    int max_seg;              // workspace slot blocks per CTA
    int debug;                // experiment switches (0 in production)
    KrpGen bgen;              // B operand rows (index j for M-major, l for K-major)
    KrpGen sgen;              // scale rows: KL over l (M-major), KR over j (K-major)
    double* ws;               // [grid][max_seg][BM][C]
    const double* htab;       // partial KRP of bgen factors 1..nf-1 (hrows x C), or null
    long long hrows;
    int smem;                 // dynamic shared memory bytes
    int u0_pitch;             // > 0: fastest B factor staged in shared memory with this row pitch
    const double* X;          // tensor base (the LDGSTS producer reads it directly)
    int ldgsts;               // 1: strides or base not 16-byte aligned for TMA; the producer warp
                              // copies the swizzled stage with 8-byte cp.async instead
    int epi;                  // epilogue instantiation (Epi): kEpiGen compiles every flavor's epilogue,
                              // the others only their own (fewer live registers in the consumer loop)
    int x_wait;               // 1: X is a scratch buffer an earlier kernel wrote (the baseline's
                              // matricised copy): the producer waits for it too (pdl_wait)
    unsigned long long* trace;  // developer timeline (DMTK_GPU_TRACE): kTraceSlots stamps per CTA, or null
    int m3;                   // M-major: the tensor map is the 3-D view (16 m, j, m / 16) and one box
                              // {16, BK, TR / 16} loads a row group's whole stage (else TR / 16 2-D boxes)
};

// Timeline stamps of the streaming kernel (%globaltimer, ns). Developer tool only.
constexpr int kTraceStages = 24;  // per-stage stamps of the first stages
constexpr int kTraceSlots = 16 + 2 * kTraceStages;
enum TraceEv : int {
    kTrEntry = 0, kTrPrologue = 1, kTrTmaFirst = 2, kTrTmaLast = 3, kTrBuildFirst = 4, kTrBuildLast = 5,
    kTrConsFirst = 6, kTrConsLoop = 7, kTrConsEpi = 8, kTrCons7Loop = 9, kTrExit = 10,
    kTrClkEntry = 11, kTrClkExit = 12,  // clock64 (SM cycles) at entry and exit: the SM clock rate
    kTrBuildStart = 13,                   // builder warp 0 enters its item loop
    kTrBuildLoaded = 14,                  // ... has issued its first item's factor / head loads
    kTrStageIssue = 16,                   // producer: stage k's loads issued
    kTrStageReady = 16 + kTraceStages,    // observer: stage k's full barrier complete
};

// Epilogue instantiations of the streaming kernel (template parameter EPI).
enum Epi : int {
    kEpiGen = 0,  // every flavor (boundary 2-step views other than kEpiSwr)
    kEpiSwr = 1,  // K-major boundary 2-step, BI >= 8 RB, one-factor scale: one output row per warp
    kEpiMM = 2,   // M-major, no swap (1-step mode 0, 2-step right)
    kEpiKJ = 3,   // K-major rows (i, j), no swap (1-step last mode, 2-step left)
    kEpiJK = 4,   // K-major interior 1-step
};

// Stage range of CTA b under the stream-K split.
__host__ __device__ inline void cta_stage_range(long long total, int grid, int b, long long& lo, long long& hi) {
    const long long a0 = total * b, a1 = total * (b + 1);
    if (a1 < 0x7fffffffLL) {  // 32-bit division when it fits (every BASELINE shape)
        lo = static_cast<unsigned>(a0) / static_cast<unsigned>(grid);
        hi = static_cast<unsigned>(a1) / static_cast<unsigned>(grid);
    } else {
        lo = a0 / grid;
        hi = a1 / grid;
    }
}

}  // namespace dmtkg
