// mttkrp_tc.cuh -- the streaming MTTKRP kernel: TMA-fed shared-memory ring,
// on-the-fly Khatri-Rao B tiles, FP64 tensor-core (DMMA 8x8x4) contraction,
// fused multi-TTV epilogue. See mttkrp_plan.h for the formulation.
//
// Warp roles (384 threads, one CTA per SM, persistent over a stream-K range):
// The consumers get the highest warp ids: the SMSP arbiter issues
// highest-wid-first, so DMMA issue wins over builder/producer bookkeeping.
//   warps 4-11 consumers (two per SM sub-partition, so one warp's loads and
//              barrier waits hide behind the other's DMMAs): RW = 8 * RB tile
//              rows each x all C columns. Columns in groups of 8 run on DMMA;
//              a C % 8 remainder of 1-2 ("tail") runs on DFMA.
//   warps 1-3  builders: write the stage's B tile (BK KRP rows x C per row
//              group) into shared memory in DMMA fragment order, one multiply
//              per entry (head-table row x fastest factor row: the paper's
//              reuse scheme, Alg. 1, krp.cpp:53-88).
//   warp 0     producer: one elected lane issues the TMA box loads.
// Per stage: full barrier (TMA bytes + one arrival per builder item), empty
// barrier (8 consumer arrivals).
//
// Tile shape (template RB): BM = 64 * RB rows x BK contraction indices per
// stage, BK = 32 for RB = 2 (128-row tiles) and 16 for RB = 3, 4 (192- and
// 256-row tiles): a stage is 24-32 KB of X either way. Taller tiles share
// one B row among more X rows (less builder work and fewer shared-memory
// B fragment reads per byte of X) and fit extents like 180 in one tile.
//
// The A tile arrives through 128-byte-swizzled TMA boxes; the k index a
// DMMA fragment lane reads is permuted (kperm) so that all fragment loads
// are 2-wavefront (bank-conflict-free) LDS.64.
#pragma once

#include "mttkrp_plan.h"

namespace dmtkg {

template <int NB, int TAIL, int RB>
struct TcCfg {
    static constexpr int CP = 8 * NB + TAIL;
    static constexpr int RW = 8 * RB;                 // rows per consumer warp
    static constexpr int BM = kConsumerWarps * RW;    // tile rows at G = 1
    static constexpr int BK = tc_bk(RB);              // contraction indices per stage (per row group)
    static constexpr int KS = BK / 4;                 // DMMA k4-steps per stage
    static constexpr int MAX_STAGES = 6;
    static constexpr int A_BYTES = BM * BK * 8;       // one stage of X: 24-32 KB
    static constexpr int BMAIN = BK * 8 * NB;         // doubles per group, DMMA fragments
    static constexpr int BTAIL = BK * TAIL;           // doubles per group, DFMA tail columns
    static constexpr int B_BYTES = ((BMAIN + BTAIL) * 8 + 1023) / 1024 * 1024;  // one row group
    static constexpr int EPI_LD = CP + 1;
    static constexpr int EPI_BYTES = ((kConsumerWarps * RW * EPI_LD * 8) + 1023) / 1024 * 1024;
    static constexpr int BAR_BYTES = 2 * MAX_STAGES * 8;
    // everything but the ring; the host adds stages * (A_BYTES + G * B_BYTES)
    static constexpr int FIXED = EPI_BYTES + BAR_BYTES + 1024;
};

// Which contraction row of a 32-row stage DMMA lane column t reads at k4-step
// s. Chosen so that each half-warp's 16 fragment loads hit 32 distinct
// banks under the 128-byte TMA swizzle (2 wavefronts per LDS.64, the
// minimum): M-major tiles are [k][16 m] boxes, K-major tiles [row][16 k].
template <bool KMAJ>
__device__ __forceinline__ int kperm(int s, int t) {
    return KMAJ ? 16 * (s >> 2) + 8 * (t >> 1) + (t & 1) + 2 * (s & 3) : 8 * (s >> 1) + 2 * t + (s & 1);
}

// (tile, stage-in-tile, ring slot, phase) walked incrementally: no 64-bit
// divisions in the pipelined loops.
struct StageCursor {
    long long tile, st;
    int slot;
    uint32_t ph;
    __device__ __forceinline__ void init(long long lo, long long spt) {
        tile = div_nn(lo, spt);
        st = lo - tile * spt;
        slot = 0;
        ph = 0;
    }
    __device__ __forceinline__ void next(long long spt, int stages) {
        if (++st == spt) {
            st = 0;
            ++tile;
        }
        if (++slot == stages) {
            slot = 0;
            ph ^= 1u;
        }
    }
};

// EPI: which epilogue is compiled (Epi, mttkrp_plan.h; TcPlan::epi).
template <int NB, int TAIL, bool KMAJ, int RB, int EPI = kEpiGen>
__global__ void __launch_bounds__(tc_threads(RB), 1)
    mttkrp_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ TcPlan p) {
    using Cfg = TcCfg<NB, TAIL, RB>;
    constexpr int RW = Cfg::RW;
    constexpr int BK = Cfg::BK;
    constexpr int KS = Cfg::KS;
    constexpr int kBuilderWarps = tc_builders(RB);
    constexpr int kFirstConsumerWarp = kFirstBuilderWarp + kBuilderWarps;
    const int STAGES = p.stages;
    const int G = p.G;
    const int GB_BYTES = G * Cfg::B_BYTES;  // B tile of one stage (all row groups)
    extern __shared__ unsigned char smem_raw[];
    // realign in the shared window (keeps the pointer in the shared state
    // space so every fragment load compiles to LDS, not a generic LD)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* sA = smem;
    unsigned char* sB = smem + STAGES * Cfg::A_BYTES;
    double* sEpi = reinterpret_cast<double*>(sB + STAGES * GB_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(sEpi) + Cfg::EPI_BYTES);
    uint64_t* empty = full + Cfg::MAX_STAGES;
    double* sU0 = reinterpret_cast<double*>(empty + Cfg::MAX_STAGES);  // optional U0 copy (u0_pitch > 0)

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // developer timeline (p.trace): %globaltimer stamps (ns; the pointer
    // stays in the parameter bank, no live registers)
    auto stamp = [&](int ev) {
        if (p.trace) {
            unsigned long long gt;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
            p.trace[static_cast<long long>(blockIdx.x) * kTraceSlots + ev] = gt;
        }
    };
    if (threadIdx.x == 0) {
        stamp(kTrEntry);
        if (p.trace) p.trace[static_cast<long long>(blockIdx.x) * kTraceSlots + kTrClkEntry] = clock64();
    }
    // shared-window addresses, computed once (no per-stage address conversion)
    const uint32_t full_a = smem_u32(full), empty_a = smem_u32(empty), sA_a = smem_u32(sA);
    long long lo, hi;
    cta_stage_range(p.total_stages, gridDim.x, blockIdx.x, lo, hi);
    const long long spt = p.stages_per_tile;

    // TMA issue of one stage (the producer lane): expect_tx + the stage's boxes
    auto issue_stage = [&](const StageCursor& cur, uint64_t pol) {
        const int slot = cur.slot;
        const long long tile = cur.tile;
        const long long st = cur.st;
        mbar_arrive_expect_tx_a(full_a + 8 * slot, Cfg::A_BYTES);
        const uint32_t dst = sA_a + slot * Cfg::A_BYTES;
        if (!KMAJ) {
            // BM / 16 boxes {16 m, BK j} of 128 * BK bytes: group gi's
            // boxes cover rows 16 bb of its TR-row tile at j0 + BK gi
            const int m0 = static_cast<int>(tile * p.TR);
            const int j0 = static_cast<int>(st * BK * G);
            const int bpg = p.TR / 16;
            uint32_t d = dst;
            if (p.m3) {
                // one 3-D box per row group: the box's 16-row blocks land
                // in the same [block][j][16 m] order as the 2-D boxes
                for (int gi = 0; gi < G; ++gi, d += bpg * 128 * BK)
                    tma_load_3d(d, &tmap, full_a + 8 * slot, 0, j0 + BK * gi, m0 >> 4, pol);
            } else {
                for (int gi = 0; gi < G; ++gi)
                    for (int bb = 0; bb < bpg; ++bb, d += 128 * BK)
                        tma_load_2d(d, &tmap, full_a + 8 * slot, m0 + 16 * bb, j0 + BK * gi, pol);
            }
        } else {
            long long ti, tj, j, l0;
            if (p.flavor == kKMajorJ) {
                tj = div_nn(tile, p.n_ti);
                ti = tile - tj * p.n_ti;
                l0 = st * BK * G;
                j = tj * p.BJ;
            } else {
                ti = tile;
                j = div_nn(st, p.n_lc);
                l0 = (st - j * p.n_lc) * BK * G;
            }
            // per group: BK / 16 boxes {16 l, BI, BJ} of TR * 128 bytes
            const int gbytes = Cfg::A_BYTES / G;
            for (int gi = 0; gi < G; ++gi) {
#pragma unroll
                for (int h = 0; h < BK / 16; ++h)
                    tma_load_3d(dst + gi * gbytes + h * (gbytes / (BK / 16)), &tmap, full_a + 8 * slot,
                                static_cast<int>(l0 + BK * gi + 16 * h), static_cast<int>(ti * p.BI),
                                static_cast<int>(j), pol);
            }
        }
    };
    // The producer lane (thread 0) initialises the barriers and issues the
    // first ring fill before the CTA barrier: the first stages' DRAM latency
    // then overlaps the other roles' start-up (their code's first fetch, PDL
    // wait, builder set-up). The ring slots are empty, so no empty-barrier
    // wait is needed for them.
    int pre = 0;  // stages issued here (the producer loop skips them)
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            // producer (one expect_tx arrival, or 32 cp.async arrivals) + one per builder item
            mbar_init(&full[s], (p.ldgsts ? 32 : 1) + p.G);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_barrier_init();
        if (!p.ldgsts) {
            tma_prefetch_desc(&tmap);
            if (!p.x_wait && !(p.debug & 2)) {
                const uint64_t pol = (p.debug & 16) ? l2_evict_normal_policy() : l2_evict_first_policy();
                StageCursor cur;
                cur.init(lo, spt);
                for (long long gs = lo; gs < hi && pre < STAGES; ++gs, ++pre, cur.next(spt, STAGES)) {
                    issue_stage(cur, pol);
                    if (pre == 0) stamp(kTrTmaFirst);
                    if (pre < kTraceStages) stamp(kTrStageIssue + pre);
                }
            }
        }
    }
    // Meanwhile the other warps stage the builders' small fastest factor in
    // shared memory (u0_pitch > 0), one batch of independent loads per
    // thread, and the builders pull the first head-table rows toward L1: the
    // first B tile is then an LDS + multiply away once the barriers are up,
    // instead of two more dependent global round trips after the CTA barrier.
    // (Factor rows may be the previous kernel's output: pdl_wait first.)
    if (warp != kProducerWarp && !(p.debug & 1)) {
        const KrpGen& Gen = p.bgen;
        const int C = p.C;
        if (p.u0_pitch > 0) {
            pdl_wait();
            const int P = p.u0_pitch;
            const int n = static_cast<int>(Gen.ext[0]) * C;
            const double* __restrict__ U0 = Gen.U[0];
            const long long ldu = Gen.ldu;
            constexpr int kStageThreads = tc_threads(RB) - 32;
            constexpr int kBatch = 8;
            for (int base = threadIdx.x - 32; base < n; base += kStageThreads * kBatch) {
                double v[kBatch];
                int so[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int e = base + u * kStageThreads;
                    const int r = static_cast<int>(static_cast<unsigned>(e < n ? e : 0) / static_cast<unsigned>(C));
                    const int cc = (e < n ? e : 0) - r * C;
                    so[u] = e < n ? r * P + cc : -1;
                    v[u] = e < n ? __ldg(U0 + static_cast<long long>(r) * ldu + cc) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u)
                    if (so[u] >= 0) sU0[so[u]] = v[u];
            }
        }
        if (warp < kFirstConsumerWarp && p.htab && Gen.ext[0] >= BK && lo < hi) {
            pdl_wait();
            const long long st0 = lo - div_nn(lo, spt) * spt;
            const long long kb0 =
                (KMAJ && p.flavor == kKMajorJK ? st0 - div_nn(st0, p.n_lc) * p.n_lc : st0) * BK * G;
            const long long q0 = div_nn(kb0, Gen.ext[0]);
            const long long nrow = p.hrows - q0 < 4 ? p.hrows - q0 : 4;  // the first ring fill's head rows
            const char* hb = reinterpret_cast<const char*>(p.htab + q0 * C);
            for (long long off = (threadIdx.x - kFirstBuilderWarp * 32) * 128LL; off < nrow * C * 8; off += kBuilderWarps * 32 * 128LL)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(hb + off));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) stamp(kTrPrologue);
    // Programmatic dependent launch: the producer streams X (never written by
    // the library's kernels) without waiting for the previous kernel unless X
    // is a buffer that kernel may have just produced (x_wait); the builders
    // (factor rows) and the consumers (workspace slots, read by the previous
    // call's reduction) wait for it.
    if (warp != kProducerWarp || p.x_wait) {
        pdl_wait();
        pdl_trigger();
    }

    // ------------------------------------------------------------ producer
    if (warp == kProducerWarp && p.ldgsts) {
        // Strides (or the base) not 16-byte aligned: TMA cannot describe the
        // view, so the whole warp copies each stage with 8-byte cp.async into
        // the same 128-byte-swizzled box layout the TMA path produces (zero
        // fill out of range), then arrives on the full barrier when its copies
        // have landed.
        StageCursor cur;
        cur.init(lo, spt);
        const double* __restrict__ X = p.X;
        for (long long gs = lo; gs < hi; ++gs, cur.next(spt, STAGES)) {
            const int slot = cur.slot;
            const long long tile = cur.tile;
            const long long st = cur.st;
            mbar_wait_a(empty_a + 8 * slot, cur.ph ^ 1u);
            const uint32_t dst = sA_a + slot * Cfg::A_BYTES;
            if (!KMAJ) {
                // lane-owned rows mm = lane + 32 q of every column: the smem row
                // offset and the global pointer advance incrementally per column
                const long long mrows = p.L * p.I;
                const long long m0 = tile * p.TR;
                const long long j0 = st * BK * G;
                const int nq = (p.TR + 31) >> 5;
                for (int q = 0; q < nq; ++q) {
                    const int mm = lane + 32 * q;
                    if (mm >= p.TR) break;
                    const long long m = m0 + mm;
                    const bool mok = m < mrows;
                    const int w16 = mm & 15;
                    const uint32_t wlo = (w16 & 1) << 3, whi = w16 >> 1;
                    for (int gi = 0; gi < G; ++gi) {
                        uint32_t d = dst + (gi * (p.TR / 16) + (mm >> 4)) * (128 * BK);
                        long long j = j0 + BK * gi;
                        const double* src = X + j * mrows + m;
#pragma unroll 8
                        for (int jj = 0; jj < BK; ++jj, d += 128, src += mrows, ++j) {
                            const bool ok = mok && j < p.R;
                            cp_async_8(d + (((whi ^ (jj & 7)) << 4) | wlo), ok ? src : X, ok ? 8u : 0u);
                        }
                    }
                }
            } else {
                long long ti, tj, j, l0;
                if (p.flavor == kKMajorJ) {
                    tj = div_nn(tile, p.n_ti);
                    ti = tile - tj * p.n_ti;
                    l0 = st * BK * G;
                    j = tj * p.BJ;
                } else {
                    ti = tile;
                    j = div_nn(st, p.n_lc);
                    l0 = (st - j * p.n_lc) * BK * G;
                }
                // lane = (row pair, l): 16 lanes per 128-byte row, two rows per pass
                const int gbytes = Cfg::A_BYTES / G;
                const int ll = lane & 15;
                const uint32_t llo = (ll & 1) << 3, lhi = ll >> 1;
                for (int rho = lane >> 4; rho < p.TR; rho += 2) {
                    const int jl = rho / p.BI;
                    const long long i = ti * p.BI + (rho - jl * p.BI);
                    const long long jj = j + jl;
                    const bool rok = i < p.I && jj < p.R;
                    const double* row = X + p.L * (i + p.I * jj);
                    const uint32_t roff = rho * 128 + ((lhi ^ (rho & 7)) << 4) + llo;
                    for (int gi = 0; gi < G; ++gi) {
#pragma unroll
                        for (int h = 0; h < BK / 16; ++h) {
                            const long long l = l0 + BK * gi + 16 * h + ll;
                            const bool ok = rok && l < p.L;
                            cp_async_8(dst + gi * gbytes + h * (gbytes / (BK / 16)) + roff, ok ? row + l : X,
                                       ok ? 8u : 0u);
                        }
                    }
                }
            }
            cp_async_mbar_arrive_noinc(full_a + 8 * slot);
        }
        return;
    }
    if (warp == kProducerWarp) {
        if (lane == 0) {
            const uint64_t pol = (p.debug & 16) ? l2_evict_normal_policy() : l2_evict_first_policy();
            StageCursor cur;
            cur.init(lo, spt);
            for (long long gs = lo; gs < hi; ++gs, cur.next(spt, STAGES)) {
                if (gs - lo < pre) continue;  // issued in the prologue
                const int slot = cur.slot;
                mbar_wait_a(empty_a + 8 * slot, cur.ph ^ 1u);
                if (p.debug & 2) {
                    mbar_arrive_a(full_a + 8 * slot);
                    continue;
                }
                issue_stage(cur, pol);
                if (gs == lo) stamp(kTrTmaFirst);
                if (gs - lo < kTraceStages) stamp(kTrStageIssue + static_cast<int>(gs - lo));
            }
            stamp(kTrTmaLast);
        } else if (lane == 1 && p.trace) {
            // timeline observer: when each of the first stages' full barrier
            // (TMA bytes + B tile) completes -- waits only, never arrives
            StageCursor cur;
            cur.init(lo, spt);
            for (long long gs = lo; gs < hi && gs - lo < kTraceStages; ++gs, cur.next(spt, STAGES)) {
                mbar_wait_a(full_a + 8 * cur.slot, cur.ph);
                stamp(kTrStageReady + static_cast<int>(gs - lo));
            }
        }
        return;
    }

    // ------------------------------------------------------------ builders
    // Work items are (stage, row group) pairs dealt round-robin to the
    // builder warps; every item arrives once on its stage's full barrier
    // (count 1 + G). Lane (g, t) produces exactly the B values DMMA lane
    // (g, t) consumes: rows kperm(s, t) for the 8 k4-steps, columns nb*8 + g,
    // stored 128-bit and lane-contiguous (conflict-free). The fastest factor
    // is read from a shared-memory copy when it is small (LDS latency instead
    // of an L2 round trip per item), the head partial from the materialised
    // head table (one row, refreshed only when the slower digits carry).
#ifdef DMTK_EXP_NO_TAIL_BUILD
    constexpr bool kExpNoTailBuild = true;  // timing experiment: builders skip the tail columns (wrong results)
#else
    constexpr bool kExpNoTailBuild = false;
#endif
    if (warp < kFirstConsumerWarp) {
        const int bw = warp - kFirstBuilderWarp;
        const int g = lane >> 2;
        const int t = lane & 3;
        // tail columns (DFMA columns 8 NB .. 8 NB + TAIL - 1): the item's
        // 4 KS TAIL entries are dealt over the lanes, entry x = (s 4 + t) TAIL
        // + column to lane x % 32 -- one load, one multiply and one store per
        // 32 entries (a DMUL costs the FP64 pipe the same with 4 lanes active
        // as with 32, and the builders share that pipe with the DMMAs)
        const int tg = TAIL > 0 ? lane % (TAIL > 0 ? TAIL : 1) : 0;  // this lane's tail column (32 % TAIL == 0)
        const KrpGen& Gen = p.bgen;
        const long long e0 = Gen.ext[0];
        const bool fast = e0 >= BK;
        const int C = p.C;
        const long long kext = p.kext;
        const double* __restrict__ U0 = Gen.U[0];
        const long long ldu = Gen.ldu;
        const int P = p.u0_pitch;  // > 0: U0 staged in shared memory with this row pitch
        // (P > 0: sU0 was staged by every non-producer warp before the CTA barrier)
        const uint32_t sU0a = smem_u32(sU0);
        double hv[2][NB];
        double ht[2];
        long long hq = -1, hj = -2;
        StageCursor cur;
        cur.init(lo, spt);
        if (bw == 0 && lane == 0) stamp(kTrBuildStart);
        int owner = 0;  // builder warp owning the next item
        for (long long gs = lo; gs < hi; ++gs, cur.next(spt, STAGES)) {
            for (int gi = 0; gi < G; ++gi, owner = (owner + 1 == kBuilderWarps ? 0 : owner + 1)) {
                if (owner != bw) continue;
                const int slot = cur.slot;
                if (p.debug & 1) {
                    mbar_wait_a(empty_a + 8 * slot, cur.ph ^ 1u);
                    __syncwarp();
                    if (lane == 0) mbar_arrive_a(full_a + 8 * slot);
                    continue;
                }
                long long kbase, jx = -1;
                if (KMAJ && p.flavor == kKMajorJK) {
                    jx = div_nn(cur.st, p.n_lc);
                    kbase = (cur.st - jx * p.n_lc) * BK * G + BK * gi;
                } else {
                    kbase = cur.st * BK * G + BK * gi;
                }
                long long q0 = 0;
                int r0 = 0;
                if (fast) {
                    q0 = div_nn(kbase, e0);
                    r0 = static_cast<int>(kbase - q0 * e0);
                    if (q0 != hq || jx != hj) {  // refresh the two head rows (q0, q0 + 1)
                        hq = q0;
                        hj = jx;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
#pragma unroll
                            for (int nb = 0; nb < NB; ++nb) hv[h][nb] = 1.0;
                            ht[h] = 1.0;
                            if (p.htab) {
                                if (q0 + h < p.hrows) {
                                    const double* row = p.htab + (q0 + h) * C;
#pragma unroll
                                    for (int nb = 0; nb < NB; ++nb)
                                        hv[h][nb] = nb * 8 + g < C ? __ldg(row + nb * 8 + g) : 0.0;
                                    if (TAIL > 0) ht[h] = (8 * NB + tg < C) ? __ldg(row + 8 * NB + tg) : 0.0;
                                }
                            } else {
                                const long long idx = (q0 + h) * e0;
                                for (int f = 1; f < Gen.nf; ++f) {
                                    const double* row = Gen.U[f] + krp_digit(Gen, f, idx) * Gen.ldu;
#pragma unroll
                                    for (int nb = 0; nb < NB; ++nb)
                                        hv[h][nb] *= nb * 8 + g < C ? __ldg(row + nb * 8 + g) : 0.0;
                                    if (TAIL > 0) ht[h] *= (8 * NB + tg < C) ? __ldg(row + 8 * NB + tg) : 0.0;
                                }
                            }
                            if (jx >= 0) {
                                const KrpGen& S = p.sgen;
                                for (int f = 0; f < S.nf; ++f) {
                                    const double* row = S.U[f] + krp_digit(S, f, jx) * S.ldu;
#pragma unroll
                                    for (int nb = 0; nb < NB; ++nb)
                                        hv[h][nb] *= nb * 8 + g < C ? __ldg(row + nb * 8 + g) : 0.0;
                                    if (TAIL > 0) ht[h] *= (8 * NB + tg < C) ? __ldg(row + 8 * NB + tg) : 0.0;
                                }
                            }
                        }
                    }
                } else {
                    hq = -1;
#pragma unroll
                    for (int nb = 0; nb < NB; ++nb) hv[0][nb] = hv[1][nb] = 1.0;
                    ht[0] = ht[1] = 1.0;
                }
                // no head partial at all (one-factor B rows, no interior-mode scale): hv == 1
                const bool unit_head = fast && Gen.nf == 1 && p.htab == nullptr && jx < 0;
                double* Bm = reinterpret_cast<double*>(sB + slot * GB_BYTES + gi * Cfg::B_BYTES);
                double* Bt = Bm + Cfg::BMAIN;
                // wide ranks build the item in two chunks of k4-steps (registers)
                constexpr int NCH = NB > 4 && KS == 8 ? 2 : 1;
                constexpr int SPC = KS / NCH;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    double u[SPC][NB];
                    bool hsel[SPC];
                    if (fast && P > 0) {
#pragma unroll
                        for (int ss = 0; ss < SPC; ++ss) {
                            const int kr = kperm<KMAJ>(ch * SPC + ss, t);
                            int r = r0 + kr;
                            hsel[ss] = r >= e0;
                            if (hsel[ss]) r -= static_cast<int>(e0);
                            const bool valid = kbase + kr < kext;
                            const uint32_t srow = sU0a + static_cast<uint32_t>(r * P) * 8u;
#pragma unroll
                            for (int nb = 0; nb < NB; ++nb)
                                u[ss][nb] = (valid && nb * 8 + g < C) ? lds_f64(srow + (nb * 8 + g) * 8) : 0.0;
                        }
                    } else if (fast) {
#pragma unroll
                        for (int ss = 0; ss < SPC; ++ss) {
                            const int kr = kperm<KMAJ>(ch * SPC + ss, t);
                            int r = r0 + kr;
                            hsel[ss] = r >= e0;
                            if (hsel[ss]) r -= static_cast<int>(e0);
                            const bool valid = kbase + kr < kext;
                            const double* row = U0 + r * ldu;
#pragma unroll
                            for (int nb = 0; nb < NB; ++nb)
                                u[ss][nb] = (valid && nb * 8 + g < C) ? __ldg(row + nb * 8 + g) : 0.0;
                        }
                    } else {
                        // small fastest radix (< 32 rows): full product per entry
#pragma unroll
                        for (int ss = 0; ss < SPC; ++ss) {
                            const int kr = kperm<KMAJ>(ch * SPC + ss, t);
                            const long long kidx = kbase + kr;
                            const bool valid = kidx < kext;
                            hsel[ss] = false;
#pragma unroll
                            for (int nb = 0; nb < NB; ++nb) {
                                const int c = nb * 8 + g;
                                double v = 0.0;
                                if (valid && c < C) {
                                    v = krp_value(Gen, kidx, c);
                                    if (jx >= 0) v *= krp_value(p.sgen, jx, c);
                                }
                                u[ss][nb] = v;
                            }
                        }
                    }
                    constexpr int TE = SPC * 4 * (TAIL > 0 ? TAIL : 1);  // tail entries of this chunk
                    constexpr int TRND = (TE + 31) / 32;
                    double tv[TRND];
                    if (TAIL > 0 && !kExpNoTailBuild) {
                        const int tcn = 8 * NB + tg;
#pragma unroll
                        for (int rd = 0; rd < TRND; ++rd) {
                            const int x = rd * 32 + lane;
                            const int xs = x / (4 * (TAIL > 0 ? TAIL : 1)), xt = (x / (TAIL > 0 ? TAIL : 1)) & 3;
                            double val = 0.0;
                            if (x < TE && tcn < C) {
                                const int kr = kperm<KMAJ>(ch * SPC + xs, xt);
                                const long long kidx = kbase + kr;
                                if (kidx < kext) {
                                    if (fast) {
                                        int r = r0 + kr;
                                        const bool hs = r >= e0;
                                        if (hs) r -= static_cast<int>(e0);
                                        const double uv = P > 0 ? lds_f64(sU0a + static_cast<uint32_t>(r * P + tcn) * 8u)
                                                                : __ldg(U0 + r * ldu + tcn);
                                        val = uv * (hs ? ht[1] : ht[0]);
                                    } else {
                                        val = krp_value(Gen, kidx, tcn);
                                        if (jx >= 0) val *= krp_value(p.sgen, jx, tcn);
                                    }
                                }
                            }
                            tv[rd] = val;
                        }
                    }
                    if (ch == 0) {
                        if (bw == 0 && lane == 0 && gs == lo) stamp(kTrBuildLoaded);
                        mbar_wait_a(empty_a + 8 * slot, cur.ph ^ 1u);
                    }
                    if (unit_head) {
                        // a single-factor B tile (no head partial): the rows as they are
#pragma unroll
                        for (int sp = 0; sp < SPC / 2; ++sp) {
                            const int s2 = ch * SPC / 2 + sp;
#pragma unroll
                            for (int nb = 0; nb < NB; ++nb) {
                                double2 v;
                                v.x = u[2 * sp][nb];
                                v.y = u[2 * sp + 1][nb];
                                *reinterpret_cast<double2*>(Bm + (((s2 * NB + nb) * 32 + lane) << 1)) = v;
                            }
                        }
                    } else {
#pragma unroll
                        for (int sp = 0; sp < SPC / 2; ++sp) {
                            const int s2 = ch * SPC / 2 + sp;
#pragma unroll
                            for (int nb = 0; nb < NB; ++nb) {
                                double2 v;
                                v.x = u[2 * sp][nb] * (hsel[2 * sp] ? hv[1][nb] : hv[0][nb]);
                                v.y = u[2 * sp + 1][nb] * (hsel[2 * sp + 1] ? hv[1][nb] : hv[0][nb]);
                                *reinterpret_cast<double2*>(Bm + (((s2 * NB + nb) * 32 + lane) << 1)) = v;
                            }
                        }
                    }
                    if (TAIL > 0 && !kExpNoTailBuild) {
#pragma unroll
                        for (int rd = 0; rd < TRND; ++rd)
                            if (rd * 32 + lane < TE) Bt[ch * TE + rd * 32 + lane] = tv[rd];
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive_a(full_a + 8 * slot);
                    if (bw == 0) stamp(gs == lo ? kTrBuildFirst : kTrBuildLast);
                }
            }
        }
        return;
    }

    // ------------------------------------------------------------ consumers
    const int w = warp - kFirstConsumerWarp;
    const int wpg = kConsumerWarps / G;  // consumer warps per row group
    const int gi = w / wpg;              // this warp's row group (its contraction slice)
    const int lw = w - gi * wpg;         // warp within the group: rows RW lw .. RW lw + RW - 1
    const int gl = lane >> 2;  // fragment row / B column
    const int tl = lane & 3;   // fragment k / D column pair
    // per-lane A fragment offsets (bytes within a stage), see kperm.
    // M-major: row block rb of this warp is stage row rho = RW w + 8 rb, in
    // box rho / 16 (128 * BK bytes each) at m = rho % 16; k = 8 (s >> 1) +
    // 2 t + (s & 1), so the box row is k & 7 = 2 t + (s & 1) of k-octet s >> 1.
    // K-major: x = s & 3; k & 15 = 8 (t >> 1) + (t & 1) + 2 (s & 3).
    uint32_t aoff[KMAJ ? 4 : 2 * RB];
    if (!KMAJ) {
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
#pragma unroll
            for (int x = 0; x < 2; ++x) {
                const uint32_t rho = RW * w + 8 * rb;
                const uint32_t kr7 = 2 * tl + x;
                const uint32_t mm = (rho & 15u) + gl;
                aoff[2 * rb + x] = (rho >> 4) * (128 * BK) + kr7 * 128 + ((mm * 8) ^ (kr7 << 4));
            }
        }
    } else {
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const uint32_t kk = 8 * (tl >> 1) + (tl & 1) + 2 * x;
            aoff[x] = (kk * 8) ^ (static_cast<uint32_t>(gl) << 4);
        }
    }

    double acc[RB][NB][2];
    // tail accumulators split by k4-step parity: two independent DFMA chains
#ifndef DMTK_TAIL_CHAINS
#define DMTK_TAIL_CHAINS 2
#endif
    constexpr int kTailChains = DMTK_TAIL_CHAINS;
    double tacc[2][RB][TAIL > 0 ? TAIL : 1];
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) {
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) acc[rb][nb][0] = acc[rb][nb][1] = 0.0;
#pragma unroll
        for (int tc = 0; tc < (TAIL > 0 ? TAIL : 1); ++tc) tacc[0][rb][tc] = tacc[1][rb][tc] = 0.0;
    }

    double* Pw = sEpi + w * RW * Cfg::EPI_LD;
    int seg = 0;

    // Fragments of one k4-step pair, double-buffered in registers: the loads
    // of the next pair (across the stage boundary too: the next stage's full
    // barrier is awaited before this stage's last DMMAs) overlap the DMMAs
    // of the current one, so the tensor pipe sees no stage-boundary bubble.
    struct Frag {
        double2 bv[NB];
        double a[2][RB];
        double bt[2][TAIL > 0 ? TAIL : 1];
    };
    const uint32_t a_warp = KMAJ ? static_cast<uint32_t>(gi * (Cfg::A_BYTES / G) + (RW * lw + gl) * 128) : 0u;
    const uint32_t a_box = KMAJ ? static_cast<uint32_t>(Cfg::A_BYTES / G / (BK / 16)) : 0u;
    // Fragment loads by 32-bit shared-window addresses (ld.shared): the
    // generic-pointer form made the compiler rebuild the CTA's shared window
    // base (S2R SR_CgaCtaId + LEA) at the top of every stage.
    const uint32_t sB_lane = smem_u32(sB) + gi * Cfg::B_BYTES + (lane << 4);
    const uint32_t sT_lane = smem_u32(sB) + gi * Cfg::B_BYTES + Cfg::BMAIN * 8 + tl * (TAIL > 0 ? TAIL : 1) * 8;
    auto load = [&](Frag& f, int sl, int s2) {
        const uint32_t As = sA_a + sl * Cfg::A_BYTES;
        const uint32_t Bl = sB_lane + sl * GB_BYTES;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) f.bv[nb] = lds_v2f64(Bl + (s2 * NB + nb) * 512);
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
            const int s = 2 * s2 + sub;
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) {
                const uint32_t off = !KMAJ ? (s >> 1) * 1024 + aoff[2 * rb + (s & 1)]
                                           : a_warp + (s >> 2) * a_box + 8 * rb * 128 + aoff[s & 3];
                f.a[sub][rb] = lds_f64(As + off);
            }
            if (TAIL > 0) {
#pragma unroll
                for (int tc = 0; tc < TAIL; ++tc)
                    f.bt[sub][tc] = lds_f64(sT_lane + sl * GB_BYTES + (s * 4 * (TAIL > 0 ? TAIL : 1) + tc) * 8);
            }
        }
    };
    auto compute = [&](const Frag& f) {
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) {
#pragma unroll
                for (int nb = 0; nb < NB; ++nb)
                    dmma_8x8x4(acc[rb][nb][0], acc[rb][nb][1], f.a[sub][rb], sub ? f.bv[nb].y : f.bv[nb].x);
            }
#ifndef DMTK_EXP_NO_TAIL_FMA
            if (TAIL > 0) {
#else
            if (TAIL > 0 && sub > 7) {  // timing experiment: tail FMAs compiled out (wrong results)
#endif
#pragma unroll
                for (int rb = 0; rb < RB; ++rb) {
#pragma unroll
                    for (int tc = 0; tc < TAIL; ++tc)
                        tacc[sub & (kTailChains - 1)][rb][tc] =
                            fma(f.a[sub][rb], f.bt[sub][tc], tacc[sub & (kTailChains - 1)][rb][tc]);
                }
            }
        }
    };

    // Cross-stage prefetch needs two fragment sets live; above 3 column
    // groups that pushes the kernel past its register budget (spills cost
    // more than the bubble), so wide ranks load per pair instead.
    constexpr bool kPrefetch = NB <= 3;
    // Segments (the stages of one tile inside this CTA's range) run as an
    // int-counted inner loop: per-stage bookkeeping is a ring-slot step only.
    int slot = 0;
    uint32_t ph = 0;
    long long tile = div_nn(lo, spt);
    long long st0 = lo - tile * spt;
    Frag f0, f1;
    if (kPrefetch && lo < hi) {
        mbar_wait_a(full_a, 0u);
        load(f0, 0, 0);
    }
    if (lane == 0 && w == 0) stamp(kTrConsFirst);
    for (long long gs = lo; gs < hi; ++tile, st0 = 0, ++seg) {
        const int nseg = static_cast<int>(spt - st0 < hi - gs ? spt - st0 : hi - gs);
        gs += nseg;
        const bool more = gs < hi;  // another segment follows
        for (int k = 0; k < nseg; ++k) {
            const int nslot = slot + 1 == STAGES ? 0 : slot + 1;
            const uint32_t nph = nslot == 0 ? ph ^ 1u : ph;
            if (kPrefetch) {
                const bool has_next = more || k + 1 < nseg;
#pragma unroll
                for (int s2 = 0; s2 < KS / 2; ++s2) {
                    Frag& cf = (s2 & 1) ? f1 : f0;
                    Frag& nf = (s2 & 1) ? f0 : f1;
                    if (s2 < KS / 2 - 1) {
                        load(nf, slot, s2 + 1);
                    } else {
                        // unconditional load keeps the fragment dataflow
                        // branch-free; past the range end it re-reads the
                        // current (still owned) slot and is discarded
                        if (has_next) mbar_wait_a(full_a + 8 * nslot, nph);
                        load(nf, has_next ? nslot : slot, 0);
                    }
                    compute(cf);
                }
            } else {
                mbar_wait_a(full_a + 8 * slot, ph);
#pragma unroll
                for (int s2 = 0; s2 < KS / 2; ++s2) {
                    load(f0, slot, s2);
                    compute(f0);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_a(empty_a + 8 * slot);
            slot = nslot;
            ph = nph;
        }
        if (lane == 0 && w == 0) stamp(kTrConsLoop);
        if (lane == 0 && w == kConsumerWarps - 1) stamp(kTrCons7Loop);
        if (p.debug & 8) {  // experiment: drop the epilogue entirely
#pragma unroll
            for (int rb = 0; rb < RB; ++rb)
#pragma unroll
                for (int nb = 0; nb < NB; ++nb) acc[rb][nb][0] = acc[rb][nb][1] = 0.0;
            continue;
        }

        // ------------------------------------------------- epilogue (warp-local)
        // Rows are finished in chunks of EC (a divisor of RW, at most 16) so
        // the scale loads in flight stay within the register budget at RW =
        // 32. The accumulators are re-zeroed only after the epilogue (dead,
        // not live zeros, meanwhile).
        constexpr int LD = Cfg::EPI_LD;
        constexpr int EC = RW % 16 == 0 ? 16 : 8;
        static_assert(RW % EC == 0, "epilogue chunk must divide the warp's rows");
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
                Pw[(8 * rb + gl) * LD + 8 * nb + 2 * tl] = acc[rb][nb][0];
                Pw[(8 * rb + gl) * LD + 8 * nb + 2 * tl + 1] = acc[rb][nb][1];
            }
            if (TAIL > 0) {
#pragma unroll
                for (int tc = 0; tc < (TAIL > 0 ? TAIL : 1); ++tc) {
                    double v = tacc[0][rb][tc] + tacc[1][rb][tc];
                    v += __shfl_xor_sync(0xffffffffu, v, 1);
                    v += __shfl_xor_sync(0xffffffffu, v, 2);
                    if (tl == 0) Pw[(8 * rb + gl) * LD + 8 * NB + tc] = v;
                }
            }
        }
        __syncwarp();
        const int C = p.C;
        double* wsb = p.ws + ((static_cast<long long>(blockIdx.x) * p.max_seg + seg) * Cfg::BM + RW * w) * C;
        if constexpr (EPI == kEpiSwr) {
            // K-major boundary 2-step, one output row j per warp (BI >= RW) and
            // one (or a materialised) scale factor: rows read from one base
            // pointer with 32-bit offsets, four independent partial sums (a
            // serial chain of FP64 FMAs costs ~100 cycles per link on B200)
            // combined pairwise in a fixed order.
            const long long tj = div_nn(tile, p.n_ti);
            const long long ti = tile - tj * p.n_ti;
            const long long j = tj * p.BJ + (RW * lw) / p.BI;
            const long long ib = ti * p.BI + (RW * lw) % p.BI;
            const int nv = p.I - ib < RW ? static_cast<int>(p.I - ib) : RW;  // valid rows
            const int ldu = static_cast<int>(p.sgen.ldu);
            const double* __restrict__ sbase = p.sgen.U[0] + ib * p.sgen.ldu;
            for (int c = lane; c < C; c += 32) {
                double part[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int r0 = 0; r0 < RW; r0 += EC) {
                    double sc[EC];
#pragma unroll
                    for (int r = 0; r < EC; ++r) sc[r] = r0 + r < nv ? __ldg(sbase + (r0 + r) * ldu + c) : 0.0;
#pragma unroll
                    for (int r = 0; r < EC; ++r) part[r % 4] = fma(Pw[(r0 + r) * LD + c], sc[r], part[r % 4]);
                }
                if (j < p.R) wsb[c] = (part[0] + part[2]) + (part[1] + part[3]);
            }
        } else {
        for (int c = lane; c < C; c += 32) {
            if (!KMAJ && EPI == kEpiGen && p.swap) {
                // boundary 2-step, mode 0: output row l = m % L, scale KRP(i = m / L)
                const long long mrows = p.L * p.I;
                const long long mbase = tile * p.TR + RW * lw;
                if (mbase < mrows) {
                    const long long ifirst = div_nn(mbase, p.L);
                    const long long l0 = mbase - ifirst * p.L;
                    if (p.L >= RW) {  // at most one wrap: two scale rows
                        const long long rw = p.L - l0;
                        const double sc0 = krp_scale(p.sgen, ifirst, c);
                        const double sc1 = (rw < RW && ifirst + 1 < p.I) ? krp_scale(p.sgen, ifirst + 1, c) : 0.0;
#pragma unroll 4
                        for (int r = 0; r < RW; ++r)
                            if (mbase + r < mrows) wsb[r * C + c] = Pw[r * LD + c] * (r < rw ? sc0 : sc1);
                    } else {
                        const int nslot = static_cast<int>(p.L);
                        for (int q = 0; q < nslot && mbase + q < mrows; ++q) {
                            double sum = 0.0;
                            for (int r = q; r < RW && mbase + r < mrows; r += nslot)
                                sum += Pw[r * LD + c] * krp_scale(p.sgen, ifirst + div_nn(l0 + r, p.L), c);
                            wsb[q * C + c] = sum;
                        }
                    }
                }
            } else if (KMAJ && EPI == kEpiGen && p.swap) {
                // boundary 2-step, last mode: output row j, scale KRP(i)
                const long long tj = div_nn(tile, p.n_ti);
                const long long ti = tile - tj * p.n_ti;
                if (p.BI >= RW) {
                    const long long j = tj * p.BJ + (RW * lw) / p.BI;
                    const long long ib = ti * p.BI + (RW * lw) % p.BI;
                    double sum = 0.0;
#pragma unroll
                    for (int r0 = 0; r0 < RW; r0 += EC) {
                        double sc[EC];
#pragma unroll
                        for (int r = 0; r < EC; ++r) sc[r] = ib + r0 + r < p.I ? krp_scale(p.sgen, ib + r0 + r, c) : 0.0;
#pragma unroll
                        for (int r = 0; r < EC; ++r) sum += Pw[(r0 + r) * LD + c] * sc[r];
                    }
                    if (j < p.R) wsb[c] = sum;
                } else {
                    const int njl = RW / p.BI;
                    const int jl0 = (RW * lw) / p.BI;
                    for (int q = 0; q < njl; ++q) {
                        const long long j = tj * p.BJ + jl0 + q;
                        double sum = 0.0;
                        for (int il = 0; il < p.BI; ++il) {
                            const long long i = ti * p.BI + il;
                            if (i < p.I) sum += Pw[(q * p.BI + il) * LD + c] * krp_scale(p.sgen, i, c);
                        }
                        if (j < p.R) wsb[q * C + c] = sum;
                    }
                }
            } else if (!KMAJ) {
                const long long mrows = p.L * p.I;
                const long long mbase = tile * p.TR + RW * lw;
                if (p.L == 1) {
                    for (int r = 0; r < RW && mbase + r < mrows; ++r) wsb[r * C + c] = Pw[r * LD + c];
                } else if (mbase + RW <= mrows && p.L >= RW && p.sgen.nf == 1) {
                    // common multi-TTV case: RW full rows, l wraps at most once,
                    // a single (materialised or one-input) scale factor
                    const long long ifirst = div_nn(mbase, p.L);
                    const int l0 = static_cast<int>(mbase - ifirst * p.L);
                    const int rw = static_cast<int>(p.L) - l0;  // first row of the next i
                    const double* sbase = p.sgen.U[0] + c;
                    const long long ldu = p.sgen.ldu;
                    // the one-flavor instantiation splits each sum into four
                    // independent chains (rows of the other output row add
                    // exact zeros); the general kernel keeps one chain (its
                    // register allocation is shared with every flavor)
                    constexpr int K4 = EPI == kEpiMM ? 4 : 1;
                    double s0[K4], s1[K4];
#pragma unroll
                    for (int q = 0; q < K4; ++q) s0[q] = s1[q] = 0.0;
#pragma unroll
                    for (int r0 = 0; r0 < RW; r0 += EC) {
                        double sc[EC];
#pragma unroll
                        for (int r = 0; r < EC; ++r) {
                            const int rr = r0 + r;
                            const int l = rr < rw ? l0 + rr : l0 + rr - static_cast<int>(p.L);
                            sc[r] = __ldg(sbase + l * ldu);
                        }
#pragma unroll
                        for (int r = 0; r < EC; ++r) {
                            const double v = Pw[(r0 + r) * LD + c] * sc[r];
                            if (K4 == 1) {
                                if (r0 + r < rw) s0[0] += v; else s1[0] += v;
                            } else {
                                const bool first = r0 + r < rw;
                                s0[r % K4] += first ? v : 0.0;
                                s1[r % K4] += first ? 0.0 : v;
                            }
                        }
                    }
                    double t0 = s0[0], t1 = s1[0];
                    if (K4 == 4) {
                        t0 = (s0[0] + s0[2]) + (s0[1] + s0[3]);
                        t1 = (s1[0] + s1[2]) + (s1[1] + s1[3]);
                    }
                    wsb[c] = t0;
                    if (rw < RW) wsb[C + c] = t1;
                } else if (mbase < mrows) {
                    // general case: partial rows, short L, multi-factor scales
                    const long long ifirst = div_nn(mbase, p.L);
                    const long long l0 = mbase - ifirst * p.L;
                    long long l = l0;
                    long long cur = ifirst;
                    double sum = 0.0;
                    for (int r0 = 0; r0 < RW && mbase + r0 < mrows; r0 += EC) {
                        double sc[EC];
#pragma unroll
                        for (int r = 0; r < EC; ++r) {
                            long long lr = l0 + r0 + r;
                            if (lr >= p.L) lr = lr - p.L * div_nn(lr, p.L);
                            sc[r] = (mbase + r0 + r < mrows) ? krp_scale(p.sgen, lr, c) : 0.0;
                        }
#pragma unroll
                        for (int r = 0; r < EC; ++r, ++l) {
                            if (mbase + r0 + r >= mrows) break;
                            if (l == p.L) {
                                wsb[(cur - ifirst) * C + c] = sum;
                                ++cur;
                                sum = 0.0;
                                l = 0;
                            }
                            sum += Pw[(r0 + r) * LD + c] * sc[r];
                        }
                    }
                    wsb[(cur - ifirst) * C + c] = sum;
                }
            } else if (EPI == kEpiKJ || (EPI == kEpiGen && p.flavor == kKMajorJ)) {
                const long long tj = div_nn(tile, p.n_ti);
                const long long ti = tile - tj * p.n_ti;
                if (p.BI >= RW) {
                    // the warp's rows (i, j) change j at most once (BI >= RW):
                    // two scale rows, one division per warp
                    const int rho0 = RW * lw;
                    const int q0 = rho0 / p.BI;
                    const int rw = p.BI - (rho0 - q0 * p.BI);  // rows before j + 1
                    const long long ib = ti * p.BI + (rho0 - q0 * p.BI);
                    const long long j0 = tj * p.BJ + q0;
                    const double sc0 = j0 < p.R ? krp_scale(p.sgen, j0, c) : 0.0;
                    const double sc1 = (rw < RW && j0 + 1 < p.R) ? krp_scale(p.sgen, j0 + 1, c) : 0.0;
#pragma unroll 8
                    for (int r = 0; r < RW; ++r) {
                        const bool first = r < rw;
                        const long long i = first ? ib + r : ti * p.BI + (r - rw);
                        const bool ok = i < p.I && (first ? j0 : j0 + 1) < p.R;
                        if (ok) wsb[r * C + c] = Pw[r * LD + c] * (first ? sc0 : sc1);
                    }
                } else {
                    const int njl = RW / p.BI;
                    const int jl0 = (RW * lw) / p.BI;
                    for (int il = 0; il < p.BI; ++il) {
                        const long long i = ti * p.BI + il;
                        if (i >= p.I) continue;
                        double sum = 0.0;
                        for (int q = 0; q < njl; ++q) {
                            const long long j = tj * p.BJ + jl0 + q;
                            if (j < p.R) sum += Pw[(q * p.BI + il) * LD + c] * krp_value(p.sgen, j, c);
                        }
                        wsb[il * C + c] = sum;
                    }
                }
            } else {
                const long long ibase = tile * p.TR + RW * lw;
                for (int r = 0; r < RW && ibase + r < p.I; ++r) wsb[r * C + c] = Pw[r * LD + c];
            }
        }
        }  // kEpiSwr
        __syncwarp();
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) acc[rb][nb][0] = acc[rb][nb][1] = 0.0;
#pragma unroll
            for (int tc = 0; tc < (TAIL > 0 ? TAIL : 1); ++tc) tacc[0][rb][tc] = tacc[1][rb][tc] = 0.0;
        }
        if (lane == 0 && w == 0) stamp(kTrConsEpi);
    }
    if (lane == 0 && w == 0) {
        stamp(kTrExit);
        if (p.trace) p.trace[static_cast<long long>(blockIdx.x) * kTraceSlots + kTrClkExit] = clock64();
    }
}

}  // namespace dmtkg
