// mttkrp_tc.cuh -- the streaming MTTKRP kernel: TMA-fed shared-memory ring,
// on-the-fly Khatri-Rao B tiles, FP64 tensor-core (DMMA 8x8x4) contraction,
// fused multi-TTV epilogue. See mttkrp_plan.h for the formulation.
//
// Warp roles (352 threads, one CTA per SM, persistent over a stream-K range):
// The consumers get the highest warp ids: the SMSP arbiter issues
// highest-wid-first, so DMMA issue wins over builder/producer bookkeeping.
//   warps 3-10 consumers (two per SM sub-partition, so one warp's loads and
//              barrier waits hide behind the other's DMMAs): 16 tile rows
//              each x all C columns. Columns in
//              groups of 8 run on DMMA; the C % 8 remainder ("tail") runs on
//              DFMA so no tensor-core work is wasted on padding.
//   warps 1-2  builders, alternating stages: write the stage's B tile (32
//              KRP rows x C) into shared memory in DMMA fragment order, one
//              multiply per entry (cached head partial x fastest factor row:
//              the paper's reuse scheme, Alg. 1, krp.cpp:53-88).
//   warp 0     producer: one elected lane issues the TMA box loads.
// Per stage: full barrier (TMA bytes + 1 builder arrival), empty barrier
// (8 consumer arrivals).
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
    static constexpr int EPI_BYTES = ((kConsumerWarps * kRowsPerWarp * EPI_LD * 8) + 127) / 128 * 128;
    static constexpr int HEAD_BYTES = 2 * 64 * 8;
    static constexpr int BAR_BYTES = 2 * STAGES * 8;
    static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + EPI_BYTES + HEAD_BYTES + BAR_BYTES + 1024;
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
        tile = lo / spt;
        st = lo - tile * spt;
        slot = 0;
        ph = 0;
    }
    template <int STAGES>
    __device__ __forceinline__ void next(long long spt) {
        if (++st == spt) {
            st = 0;
            ++tile;
        }
        if (++slot == STAGES) {
            slot = 0;
            ph ^= 1u;
        }
    }
};

template <int NB, int TAIL, bool KMAJ>
__global__ void __launch_bounds__(kThreads, 1)
    mttkrp_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ TcPlan p) {
    using Cfg = TcCfg<NB, TAIL>;
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ unsigned char smem_raw[];
    // realign in the shared window (keeps the pointer in the shared state
    // space so every fragment load compiles to LDS, not a generic LD)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
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
            mbar_init(&full[s], 2);  // producer expect_tx + the stage's builder warp
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_barrier_init();
    }
    if (warp == kProducerWarp && lane == 0) tma_prefetch_desc(&tmap);
    __syncthreads();

    long long lo, hi;
    cta_stage_range(p.total_stages, gridDim.x, blockIdx.x, lo, hi);
    const long long spt = p.stages_per_tile;

    // ------------------------------------------------------------ producer
    if (warp == kProducerWarp) {
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            StageCursor cur;
            cur.init(lo, spt);
            for (long long gs = lo; gs < hi; ++gs, cur.next<STAGES>(spt)) {
                const int slot = cur.slot;
                const long long tile = cur.tile;
                const long long st = cur.st;
                mbar_wait(&empty[slot], cur.ph ^ 1u);
                if (p.debug & 2) {
                    mbar_arrive(&full[slot]);
                    continue;
                }
                mbar_arrive_expect_tx(&full[slot], Cfg::A_BYTES);
                unsigned char* dst = sA + slot * Cfg::A_BYTES;
                if (!KMAJ) {
                    const int m0 = static_cast<int>(tile * kBM);
                    const int j0 = static_cast<int>(st * kBK);
#pragma unroll
                    for (int b = 0; b < 8; ++b) tma_load_2d(dst + b * 4096, &tmap, &full[slot], m0 + 16 * b, j0, pol);
                } else if (p.flavor == kKMajorJ) {
                    const long long tj = div_nn(tile, p.n_ti);
                    const long long ti = tile - tj * p.n_ti;
                    const int l0 = static_cast<int>(st * kBK);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        tma_load_3d(dst + h * 16384, &tmap, &full[slot], l0 + 16 * h, static_cast<int>(ti * p.BI),
                                    static_cast<int>(tj * p.BJ), pol);
                } else {
                    const long long j = div_nn(st, p.n_lc);
                    const long long lc = st - j * p.n_lc;
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        tma_load_3d(dst + h * 16384, &tmap, &full[slot], static_cast<int>(lc * kBK + 16 * h),
                                    static_cast<int>(tile * kBM), static_cast<int>(j), pol);
                }
            }
        }
        return;
    }

    // ------------------------------------------------------------ builders
    // Builder warp bw owns the stages it % kBuilderWarps == bw. Lane (g, t)
    // produces exactly the B values DMMA lane (g, t) consumes: rows
    // kperm(s, t) for the 8 k4-steps, columns nb*8 + g. All factor loads of a
    // stage are issued before any is used (one L2 round trip per stage), and
    // the stores are 128-bit, lane-contiguous (conflict-free).
    if (warp < kFirstConsumerWarp) {
        const int bw = warp - kFirstBuilderWarp;
        const int g = lane >> 2;
        const int t = lane & 3;
        const KrpGen& G = p.bgen;
        const long long e0 = G.ext[0];
        const bool fast = e0 >= kBK;
        const int C = p.C;
        const double* __restrict__ U0 = G.U[0];
        const long long ldu = G.ldu;
        const long long kext = p.kext;
        // head partial products (all factors but the fastest, times KR(j)
        // for the one-step flavor) change only every e0 rows: cached here
        double hv[2][NB];
        double ht[2];
        long long hq = -1, hj = -2;
        StageCursor cur;
        cur.init(lo, spt);
        int mine = 0;
        for (long long gs = lo; gs < hi; ++gs, cur.next<STAGES>(spt), mine = (mine + 1 == kBuilderWarps ? 0 : mine + 1)) {
            if (mine != bw) continue;
            if (p.debug & 1) {
                mbar_wait(&empty[cur.slot], cur.ph ^ 1u);
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[cur.slot]);
                continue;
            }
            const int slot = cur.slot;
            const uint32_t ph = cur.ph;
            const long long st = cur.st;
            long long kbase, jx = -1;
            if (KMAJ && p.flavor == kKMajorJK) {
                jx = div_nn(st, p.n_lc);
                kbase = (st - jx * p.n_lc) * kBK;
            } else {
                kbase = st * kBK;
            }
            // Loads of a chunk of k4-steps are all issued before use; for wide
            // ranks the stage is built in two chunks to bound registers.
            constexpr int NCH = NB > 4 ? 2 : 1;
            constexpr int SPC = 8 / NCH;
            long long q0 = 0;
            int r0 = 0;
            if (fast) {
                q0 = div_nn(kbase, e0);
                r0 = static_cast<int>(kbase - q0 * e0);
            }
            double* Bm = sB + slot * (Cfg::B_BYTES / 8);
            double* Bt = Bm + Cfg::BMAIN;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                double u[SPC][NB];
                double ut[SPC];
                bool hsel[SPC];
                if (fast) {
#pragma unroll
                    for (int ss = 0; ss < SPC; ++ss) {
                        const int kr = kperm<KMAJ>(ch * SPC + ss, t);
                        int r = r0 + kr;
                        hsel[ss] = r >= e0;
                        if (hsel[ss]) r -= static_cast<int>(e0);
                        const bool valid = kbase + kr < kext;
                        const double* row = U0 + r * ldu;
#pragma unroll
                        for (int nb = 0; nb < NB; ++nb) {
                            const int c = nb * 8 + g;
                            u[ss][nb] = (valid && c < C) ? __ldg(row + c) : 0.0;
                        }
                        ut[ss] = 0.0;
                        if (TAIL > 0) {
                            const int c = 8 * NB + g;
                            ut[ss] = (valid && g < TAIL && c < C) ? __ldg(row + c) : 0.0;
                        }
                    }
                    if (ch == 0 && (q0 != hq || jx != hj)) {
                        hq = q0;
                        hj = jx;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const long long idx = (q0 + h) * e0;
#pragma unroll
                            for (int nb = 0; nb < NB; ++nb) hv[h][nb] = 1.0;
                            ht[h] = 1.0;
                            for (int f = 1; f < G.nf; ++f) {
                                const double* row = G.U[f] + krp_digit(G, f, idx) * G.ldu;
#pragma unroll
                                for (int nb = 0; nb < NB; ++nb) {
                                    const int c = nb * 8 + g;
                                    hv[h][nb] *= c < C ? __ldg(row + c) : 0.0;
                                }
                                if (TAIL > 0) ht[h] *= (8 * NB + g < C) ? __ldg(row + 8 * NB + g) : 0.0;
                            }
                            if (jx >= 0) {
                                const KrpGen& S = p.sgen;
                                for (int f = 0; f < S.nf; ++f) {
                                    const double* row = S.U[f] + krp_digit(S, f, jx) * S.ldu;
#pragma unroll
                                    for (int nb = 0; nb < NB; ++nb) {
                                        const int c = nb * 8 + g;
                                        hv[h][nb] *= c < C ? __ldg(row + c) : 0.0;
                                    }
                                    if (TAIL > 0) ht[h] *= (8 * NB + g < C) ? __ldg(row + 8 * NB + g) : 0.0;
                                }
                            }
                        }
                    }
                } else {
                    // small fastest radix (< 32 rows): full product per entry
                    hq = -1;
#pragma unroll
                    for (int nb = 0; nb < NB; ++nb) hv[0][nb] = hv[1][nb] = 1.0;
                    ht[0] = ht[1] = 1.0;
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
                                v = krp_value(G, kidx, c);
                                if (jx >= 0) v *= krp_value(p.sgen, jx, c);
                            }
                            u[ss][nb] = v;
                        }
                        ut[ss] = 0.0;
                        if (TAIL > 0) {
                            const int c = 8 * NB + g;
                            if (valid && g < TAIL && c < C) {
                                ut[ss] = krp_value(G, kidx, c);
                                if (jx >= 0) ut[ss] *= krp_value(p.sgen, jx, c);
                            }
                        }
                    }
                }
                if (ch == 0) mbar_wait(&empty[slot], ph ^ 1u);
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
                if (TAIL > 0 && g < TAIL) {
#pragma unroll
                    for (int ss = 0; ss < SPC; ++ss)
                        Bt[((ch * SPC + ss) * 4 + t) * TAIL + g] = ut[ss] * (hsel[ss] ? ht[1] : ht[0]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[slot]);
        }
        return;
    }

    // ------------------------------------------------------------ consumers
    const int w = warp - kFirstConsumerWarp;
    const int gl = lane >> 2;  // fragment row / B column
    const int tl = lane & 3;   // fragment k / D column pair
    // per-lane A fragment offsets (bytes within a stage), see kperm
    uint32_t aoff[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
        if (!KMAJ) {
            // x = 2 * (s & 1) + (rb & 1); box row k & 7 = 2 t + (s & 1)
            const uint32_t kr7 = 2 * tl + (x >> 1);
            const uint32_t mm = 8 * (x & 1) + gl;
            aoff[x] = kr7 * 128 + ((mm * 8) ^ (kr7 << 4));
        } else {
            // x = s & 3; k & 15 = 8 (t >> 1) + (t & 1) + 2 (s & 3)
            const uint32_t kk = 8 * (tl >> 1) + (tl & 1) + 2 * x;
            aoff[x] = (kk * 8) ^ (static_cast<uint32_t>(gl) << 4);
        }
    }

    double acc[kRB][NB][2];
    double tacc[kRB][TAIL > 0 ? TAIL : 1];
#pragma unroll
    for (int rb = 0; rb < kRB; ++rb) {
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) acc[rb][nb][0] = acc[rb][nb][1] = 0.0;
#pragma unroll
        for (int tc = 0; tc < (TAIL > 0 ? TAIL : 1); ++tc) tacc[rb][tc] = 0.0;
    }

    double* Pw = sEpi + w * kRowsPerWarp * Cfg::EPI_LD;
    int seg = 0;
    StageCursor cur;
    cur.init(lo, spt);
    for (long long gs = lo; gs < hi; ++gs, cur.next<STAGES>(spt)) {
        const int slot = cur.slot;
        const long long tile = cur.tile;
        mbar_wait(&full[slot], cur.ph);
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
                double a[kRB];
#pragma unroll
                for (int rb = 0; rb < kRB; ++rb) {
                    uint32_t off;
                    if (!KMAJ) {
                        off = (w * kRowsPerWarp / 16 + (rb >> 1)) * 4096 + (s >> 1) * 1024 + aoff[2 * (s & 1) + (rb & 1)];
                    } else {
                        off = (s >> 2) * 16384 + (kRowsPerWarp * w + 8 * rb + gl) * 128 + aoff[s & 3];
                    }
                    a[rb] = *reinterpret_cast<const double*>(As + off);
                }
#pragma unroll
                for (int rb = 0; rb < kRB; ++rb) {
#pragma unroll
                    for (int nb = 0; nb < NB; ++nb)
                        dmma_8x8x4(acc[rb][nb][0], acc[rb][nb][1], a[rb], sub ? bv[nb].y : bv[nb].x);
                }
                if (TAIL > 0) {
                    double bt[TAIL > 0 ? TAIL : 1];
#pragma unroll
                    for (int tc = 0; tc < TAIL; ++tc) bt[tc] = Bt[(s * 4 + tl) * TAIL + tc];
#pragma unroll
                    for (int rb = 0; rb < kRB; ++rb) {
#pragma unroll
                        for (int tc = 0; tc < TAIL; ++tc) tacc[rb][tc] = fma(a[rb], bt[tc], tacc[rb][tc]);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);

        const bool seg_end = (gs + 1 == hi) || (cur.st + 1 == spt);
        if (!seg_end) continue;

        // ------------------------------------------------- epilogue (warp-local)
        constexpr int LD = Cfg::EPI_LD;
#pragma unroll
        for (int rb = 0; rb < kRB; ++rb) {
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
        double* wsb = p.ws + ((static_cast<long long>(blockIdx.x) * p.max_seg + seg) * kBM + kRowsPerWarp * w) * C;
        for (int c = lane; c < C; c += 32) {
            if (!KMAJ) {
                const long long mrows = p.L * p.I;
                const long long mbase = tile * kBM + kRowsPerWarp * w;
                if (p.L == 1) {
                    for (int r = 0; r < kRowsPerWarp && mbase + r < mrows; ++r) wsb[r * C + c] = Pw[r * LD + c];
                } else if (mbase < mrows) {
                    // scale rows by KL(l, c): all loads issued before use
                    const long long ifirst = div_nn(mbase, p.L);
                    const long long l0 = mbase - ifirst * p.L;
                    double sc[kRowsPerWarp];
#pragma unroll
                    for (int r = 0; r < kRowsPerWarp; ++r) {
                        long long l = l0 + r;
                        if (l >= p.L) l -= p.L * div_nn(l, p.L);
                        sc[r] = (mbase + r < mrows) ? krp_scale(p.sgen, l, c) : 0.0;
                    }
                    long long l = l0;
                    long long cur = ifirst;
                    double sum = 0.0;
#pragma unroll
                    for (int r = 0; r < kRowsPerWarp; ++r, ++l) {
                        if (mbase + r >= mrows) break;
                        if (l == p.L) {
                            wsb[(cur - ifirst) * C + c] = sum;
                            ++cur;
                            sum = 0.0;
                            l = 0;
                        }
                        sum += Pw[r * LD + c] * sc[r];
                    }
                    wsb[(cur - ifirst) * C + c] = sum;
                }
            } else if (p.flavor == kKMajorJ) {
                const long long ti = tile % p.n_ti;
                const long long tj = tile / p.n_ti;
                if (p.BI >= kRowsPerWarp) {
                    double sc[kRowsPerWarp];
                    bool ok[kRowsPerWarp];
#pragma unroll
                    for (int r = 0; r < kRowsPerWarp; ++r) {
                        const int rho = kRowsPerWarp * w + r;
                        const long long i = ti * p.BI + rho % p.BI;
                        const long long j = tj * p.BJ + rho / p.BI;
                        ok[r] = i < p.I && j < p.R;
                        sc[r] = ok[r] ? krp_scale(p.sgen, j, c) : 0.0;
                    }
#pragma unroll
                    for (int r = 0; r < kRowsPerWarp; ++r)
                        if (ok[r]) wsb[r * C + c] = Pw[r * LD + c] * sc[r];
                } else {
                    const int njl = kRowsPerWarp / p.BI;
                    const int jl0 = (kRowsPerWarp * w) / p.BI;
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
                const long long ibase = tile * kBM + kRowsPerWarp * w;
                for (int r = 0; r < kRowsPerWarp && ibase + r < p.I; ++r) wsb[r * C + c] = Pw[r * LD + c];
            }
        }
        __syncwarp();
        ++seg;
    }
}

}  // namespace dmtkg
