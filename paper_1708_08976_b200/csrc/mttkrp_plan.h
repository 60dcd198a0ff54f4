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
// Work is split stream-K style: the (tile, stage) sequence is cut into
// equal contiguous ranges, one per CTA; each tile segment a CTA finishes
// writes one 128-row slot block to the workspace, and a deterministic CSR
// reduction (reduce kernel) sums the slots of every output row.
#pragma once

#include "common.cuh"

namespace dmtkg {

constexpr int kBM = 128;  // rows per CTA tile stage (8 consumer warps x 16)
constexpr int kBK = 32;   // contraction depth per pipeline stage
constexpr int kConsumerWarps = 8;   // two per SM sub-partition
constexpr int kRowsPerWarp = kBM / kConsumerWarps;  // 16
constexpr int kRB = kRowsPerWarp / 8;               // DMMA row blocks per warp
constexpr int kBuilderWarps = 3;
constexpr int kThreads = (kConsumerWarps + kBuilderWarps + 1) * 32;
constexpr int kProducerWarp = 0;
constexpr int kFirstBuilderWarp = 1;
constexpr int kFirstConsumerWarp = 1 + kBuilderWarps;

enum Flavor : int { kMMajor = 0, kKMajorJ = 1, kKMajorJK = 2 };

struct TcPlan {
    int flavor;
    int C;                    // rank
    long long L, I, R;        // collapsed view
    int G;                    // row groups: the 128 tile rows are G groups of TR = 128/G rows,
                              // each group contracting its own 32-index slice of a stage
    int TR;                   // tile rows (128 / G)
    int stages;               // ring depth (2..4)
    int BI, BJ;               // K-major row tile: BI * BJ == TR (kKMajorJK: TR, 1)
    long long n_ti, n_tj;     // tiles along rows (M-major: n_ti = ceil(L*I/TR), n_tj = 1)
    long long stages_per_tile;  // contraction stages per tile (32 * G indices each)
    long long n_lc;           // kKMajorJK: l-chunks of 32 * G per j
    long long total_stages;   // n_ti * n_tj * stages_per_tile
    long long kext;           // extent of the B generator index (R for M-major, L for K-major)
    int max_seg;              // workspace slot blocks per CTA
    int debug;                // experiment switches (0 in production)
    KrpGen bgen;              // B operand rows (index j for M-major, l for K-major)
    KrpGen sgen;              // scale rows: KL over l (M-major), KR over j (K-major)
    double* ws;               // [grid][max_seg][128][C]
    const double* htab;       // partial KRP of bgen factors 1..nf-1 (hrows x C), or null
    long long hrows;
    int smem;                 // dynamic shared memory bytes
    int u0_pitch;             // > 0: fastest B factor staged in shared memory with this row pitch
};

// Stage range of CTA b under the stream-K split.
__host__ __device__ inline void cta_stage_range(long long total, int grid, int b, long long& lo, long long& hi) {
    lo = total * b / grid;
    hi = total * (b + 1) / grid;
}

}  // namespace dmtkg
