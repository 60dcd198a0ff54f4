// mttkrp_tc.cuh -- the streaming MTTKRP kernel: TMA-fed shared-memory ring,
// on-the-fly Khatri-Rao B tiles, FP64 tensor-core (DMMA 8x8x4) contraction,
// fused multi-TTV epilogue. See mttkrp_plan.h for the formulation.
//
// Warp roles (224 threads, one CTA per SM, persistent over a stream-K range):
//   warps 0-3  consumers: 32 tile rows each x all C columns. Columns in
//              groups of 8 run on DMMA; the C % 8 remainder ("tail") runs on
//              DFMA so no tensor-core work is wasted on padding.
//   warps 4-5  builders: write the stage's B tile (32 KRP rows x C) into
//              shared memory in DMMA fragment order, one multiply per entry
//              (cached head partial x fastest factor row: the paper's
//              reuse scheme, Alg. 1, reference krp.cpp:53-88).
//   warp 6     producer: one elected lane issues the TMA box loads.
// Per stage: full barrier (TMA bytes + 2 builder arrivals), empty barrier
// (4 consumer arrivals).
//
// The A tile arrives through 128-byte-swizzled TMA boxes; the k index a
// DMMA fragment lane reads is permuted (kperm) so that all fragment loads
// are 2-wavefront (bank-conflict-free) LDS.64.
#pragma once

#include "mttkrp_plan.h"

namespace dmtkg {

template <int NB, int TAIL>
struct TcCfg {
    static constexpr int CP = 8 * NB + TAIL;
    static constexpr int STAGES = NB <= 4 ? 4 : 3;
    static constexpr int A_BYTES = kBM * kBK * 8;
    static constexpr int BMAIN = kBK * 8 * NB;  // doubles
    static constexpr int BTAIL = kBK * TAIL;    // doubles
    static constexpr int B_BYTES = ((BMAIN + BTAIL) * 8 + 1023) / 1024 * 1024;
    static constexpr int EPI_LD = CP + 1;
    static constexpr int EPI_BYTES = ((kConsumerWarps * 32 * EPI_LD * 8) + 127) / 128 * 128;
    static constexpr int HEAD_BYTES = 2 * 64 * 8;
    static constexpr int BAR_BYTES = 2 * STAGES * 8;
    static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + EPI_BYTES + HEAD_BYTES + BAR_BYTES + 1024;
};

template <int NB, int TAIL, bool KMAJ>
__global__ void __launch_bounds__(kThreads, 1)
    mttkrp_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ TcPlan p) {
    using Cfg = TcCfg<NB, TAIL>;
    constexpr int CP = Cfg::CP;
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem =
        reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sA = smem;
    double* sB = reinterpret_cast<double*>(smem + STAGES * Cfg::A_BYTES);
    double* sEpi = reinterpret_cast<double*>(smem + STAGES * (Cfg::A_BYTES + Cfg::B_BYTES));
    double* sHead = reinterpret_cast<double*>(smem + STAGES * (Cfg::A_BYTES + Cfg::B_BYTES) + Cfg::EPI_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(sHead) + Cfg::HEAD_BYTES);
    uint64_t* empty = full + STAGES;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1 + kBuilderWarps);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_barrier_init();
    }
    if (warp == kConsumerWarps + kBuilderWarps && lane == 0) tma_prefetch_desc(&tmap);
    __syncthreads();

    long long lo, hi;
    cta_stage_range(p.total_stages, gridDim.x, blockIdx.x, lo, hi);
    const long long spt = p.stages_per_tile;

    // ------------------------------------------------------------ producer
    if (warp == kConsumerWarps + kBuilderWarps) {
        if (lane == 0) {
            long long it = 0;
            for (long long gs = lo; gs < hi; ++gs, ++it) {
                const int slot = static_cast<int>(it % STAGES);
                const uint32_t ph = static_cast<uint32_t>((it / STAGES) & 1);
                mbar_wait(&empty[slot], ph ^ 1u);
                mbar_arrive_expect_tx(&full[slot], Cfg::A_BYTES);
                const long long tile = gs / spt;
                const long long st = gs - tile * spt;
                unsigned char* dst = sA + slot * Cfg::A_BYTES;
                if (!KMAJ) {
                    const int m0 = static_cast<int>(tile * kBM);
                    const int j0 = static_cast<int>(st * kBK);
#pragma unroll
                    for (int b = 0; b < 8; ++b) tma_load_2d(dst + b * 4096, &tmap, &full[slot], m0 + 16 * b, j0);
                } else if (p.flavor == kKMajorJ) {
                    const long long ti = tile % p.n_ti;
                    const long long tj = tile / p.n_ti;
                    const int l0 = static_cast<int>(st * kBK);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        tma_load_3d(dst + h * 16384, &tmap, &full[slot], l0 + 16 * h, static_cast<int>(ti * p.BI),
                                    static_cast<int>(tj * p.BJ));
                } else {
                    const long long j = st / p.n_lc;
                    const long long lc = st - j * p.n_lc;
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        tma_load_3d(dst + h * 16384, &tmap, &full[slot], static_cast<int>(lc * kBK + 16 * h),
                                    static_cast<int>(tile * kBM), static_cast<int>(j));
                }
            }
        }
        return;
    }

    // ------------------------------------------------------------ builders
    if (warp >= kConsumerWarps) {
        const int tau = threadIdx.x - kConsumerWarps * 32;  // 0..63
        const KrpGen& g = p.bgen;
        const long long e0 = g.ext[0];
        const bool fast = e0 >= kBK;
        long long it = 0;
        for (long long gs = lo; gs < hi; ++gs, ++it) {
            const int slot = static_cast<int>(it % STAGES);
            const uint32_t ph = static_cast<uint32_t>((it / STAGES) & 1);
            const long long tile = gs / spt;
            const long long st = gs - tile * spt;
            long long kbase, jx = -1;
            if (KMAJ && p.flavor == kKMajorJK) {
                jx = st / p.n_lc;
                kbase = (st - jx * p.n_lc) * kBK;
            } else {
                kbase = st * kBK;
            }
            (void)tile;
            mbar_wait(&empty[slot], ph ^ 1u);
            const long long q0 = kbase / e0;
            const int r0 = static_cast<int>(kbase - q0 * e0);
            if (fast) {
                for (int e = tau; e < 2 * CP; e += 64) {
                    const int h = e / CP;
                    const int c = e - h * CP;
                    double v = 0.0;
                    if (c < p.C) {
                        v = krp_head(g, (q0 + h) * e0, c);
                        if (jx >= 0) v *= krp_value(p.sgen, jx, c);
                    }
                    sHead[h * CP + c] = v;
                }
                named_bar_sync(1, 64);
            }
            double* Bm = sB + slot * (Cfg::B_BYTES / 8);
            double* Bt = Bm + Cfg::BMAIN;
            const double* U0 = g.U[0];
            for (int e = tau; e < kBK * CP; e += 64) {
                const int kr = e / CP;
                const int c = e - kr * CP;
                const long long kidx = kbase + kr;
                double v = 0.0;
                if (kidx < p.kext && c < p.C) {
                    if (fast) {
                        int r = r0 + kr;
                        int h = 0;
                        if (r >= e0) {
                            r -= static_cast<int>(e0);
                            h = 1;
                        }
                        v = __ldg(U0 + static_cast<long long>(r) * g.ldu + c) * sHead[h * CP + c];
                    } else {
                        v = krp_value(g, kidx, c);
                        if (jx >= 0) v *= krp_value(p.sgen, jx, c);
                    }
                }
                // inverse of kperm: row kr -> (k4 step s, fragment lane column t)
                const int rr = kr & 7;
                const int s = ((kr >> 3) << 1) | ((rr >> 1) & 1);
                const int rp = rr & ~2;
                const int t = ((rp & 1) << 1) | (rp >> 2);
                if (c < 8 * NB) {
                    const int nb = c >> 3;
                    const int gq = c & 7;
                    Bm[((((s >> 1) * NB + nb) * 32 + gq * 4 + t) << 1) | (s & 1)] = v;
                } else if (TAIL > 0) {
                    Bt[(s * 4 + t) * (TAIL > 0 ? TAIL : 1) + (c - 8 * NB)] = v;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[slot]);
            if (fast) named_bar_sync(1, 64);
        }
        return;
    }

    // ------------------------------------------------------------ consumers
    const int w = warp;
    const int gl = lane >> 2;  // fragment row / B column
    const int tl = lane & 3;   // fragment k / D column pair
    const int kt = (tl >> 1) + 4 * (tl & 1);  // kperm lane term
    // per-lane A offsets (bytes within the stage) for the two parities of s
    // (and of rb for M-major / of (s>>1) for K-major)
    uint32_t aoff[2][2];
#pragma unroll
    for (int x = 0; x < 2; ++x) {
#pragma unroll
        for (int y = 0; y < 2; ++y) {
            if (!KMAJ) {
                // x = s & 1, y = rb & 1 ; box-relative row k&7 = 2x + kt
                const uint32_t kr7 = 2 * x + kt;
                const uint32_t mm = 8 * y + gl;
                aoff[x][y] = kr7 * 128 + ((mm * 8) ^ (kr7 << 4));
            } else {
                // x = (s >> 1) & 1, y = s & 1 ; kk = 8x + 2y + kt
                const uint32_t kk = 8 * x + 2 * y + kt;
                aoff[x][y] = (kk * 8) ^ (static_cast<uint32_t>(gl) << 4);
            }
        }
    }

    double acc[4][NB][2];
    double tacc[4][TAIL > 0 ? TAIL : 1];
#pragma unroll
    for (int rb = 0; rb < 4; ++rb) {
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) acc[rb][nb][0] = acc[rb][nb][1] = 0.0;
#pragma unroll
        for (int tc = 0; tc < (TAIL > 0 ? TAIL : 1); ++tc) tacc[rb][tc] = 0.0;
    }

    double* Pw = sEpi + w * 32 * Cfg::EPI_LD;
    int seg = 0;
    long long it = 0;
    for (long long gs = lo; gs < hi; ++gs, ++it) {
        const int slot = static_cast<int>(it % STAGES);
        const uint32_t ph = static_cast<uint32_t>((it / STAGES) & 1);
        const long long tile = gs / spt;
        mbar_wait(&full[slot], ph);
        const unsigned char* As = sA + slot * Cfg::A_BYTES;
        const double* Bm = sB + slot * (Cfg::B_BYTES / 8);
        const double* Bt = Bm + Cfg::BMAIN;
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) {
            double2 bv[NB];
#pragma unroll
            for (int nb = 0; nb < NB; ++nb)
                bv[nb] = *reinterpret_cast<const double2*>(Bm + (((s2 * NB + nb) * 32 + lane) << 1));
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
                const int s = 2 * s2 + sub;
                double a[4];
#pragma unroll
                for (int rb = 0; rb < 4; ++rb) {
                    uint32_t off;
                    if (!KMAJ) {
                        off = (2 * w + (rb >> 1)) * 4096 + (s >> 1) * 1024 + aoff[s & 1][rb & 1];
                    } else {
                        off = (s >> 2) * 16384 + (32 * w + 8 * rb + gl) * 128 + aoff[(s >> 1) & 1][s & 1];
                    }
                    a[rb] = *reinterpret_cast<const double*>(As + off);
                }
#pragma unroll
                for (int rb = 0; rb < 4; ++rb) {
#pragma unroll
                    for (int nb = 0; nb < NB; ++nb)
                        dmma_8x8x4(acc[rb][nb][0], acc[rb][nb][1], a[rb], sub ? bv[nb].y : bv[nb].x);
                }
                if (TAIL > 0) {
                    double bt[TAIL > 0 ? TAIL : 1];
#pragma unroll
                    for (int tc = 0; tc < TAIL; ++tc) bt[tc] = Bt[(s * 4 + tl) * TAIL + tc];
#pragma unroll
                    for (int rb = 0; rb < 4; ++rb) {
#pragma unroll
                        for (int tc = 0; tc < TAIL; ++tc) tacc[rb][tc] = fma(a[rb], bt[tc], tacc[rb][tc]);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);

        const bool seg_end = (gs + 1 == hi) || ((gs + 1) / spt != tile);
        if (!seg_end) continue;

        // ------------------------------------------------- epilogue (warp-local)
        constexpr int LD = Cfg::EPI_LD;
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) {
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
                Pw[(8 * rb + gl) * LD + 8 * nb + 2 * tl] = acc[rb][nb][0];
                Pw[(8 * rb + gl) * LD + 8 * nb + 2 * tl + 1] = acc[rb][nb][1];
                acc[rb][nb][0] = acc[rb][nb][1] = 0.0;
            }
#pragma unroll
            for (int tc = 0; tc < (TAIL > 0 ? TAIL : 1); ++tc) {
                if (TAIL > 0) {
                    double v = tacc[rb][tc];
                    v += __shfl_xor_sync(0xffffffffu, v, 1);
                    v += __shfl_xor_sync(0xffffffffu, v, 2);
                    if (tl == 0) Pw[(8 * rb + gl) * LD + 8 * NB + tc] = v;
                }
                tacc[rb][tc] = 0.0;
            }
        }
        __syncwarp();
        const int C = p.C;
        double* wsb = p.ws + ((static_cast<long long>(blockIdx.x) * p.max_seg + seg) * kBM + 32 * w) * C;
        for (int c = lane; c < C; c += 32) {
            if (!KMAJ) {
                const long long mrows = p.L * p.I;
                const long long mbase = tile * kBM + 32 * w;
                if (p.L == 1) {
                    for (int r = 0; r < 32 && mbase + r < mrows; ++r) wsb[r * C + c] = Pw[r * LD + c];
                } else if (mbase < mrows) {
                    const long long ifirst = mbase / p.L;
                    long long cur = ifirst;
                    double sum = 0.0;
                    for (int r = 0; r < 32 && mbase + r < mrows; ++r) {
                        const long long m = mbase + r;
                        const long long i = m / p.L;
                        if (i != cur) {
                            wsb[(cur - ifirst) * C + c] = sum;
                            cur = i;
                            sum = 0.0;
                        }
                        sum += Pw[r * LD + c] * krp_value(p.sgen, m - i * p.L, c);
                    }
                    wsb[(cur - ifirst) * C + c] = sum;
                }
            } else if (p.flavor == kKMajorJ) {
                const long long ti = tile % p.n_ti;
                const long long tj = tile / p.n_ti;
                if (p.BI >= 32) {
                    for (int r = 0; r < 32; ++r) {
                        const int rho = 32 * w + r;
                        const long long i = ti * p.BI + rho % p.BI;
                        const long long j = tj * p.BJ + rho / p.BI;
                        if (i < p.I && j < p.R) wsb[r * C + c] = Pw[r * LD + c] * krp_value(p.sgen, j, c);
                    }
                } else {
                    const int njl = 32 / p.BI;
                    const int jl0 = (32 * w) / p.BI;
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
                const long long ibase = tile * kBM + 32 * w;
                for (int r = 0; r < 32 && ibase + r < p.I; ++r) wsb[r * C + c] = Pw[r * LD + c];
            }
        }
        __syncwarp();
        ++seg;
    }
}

}  // namespace dmtkg
