// kernels.h -- host-side launchers for the dmtk B200 kernels.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <mutex>

#include "mttkrp_plan.h"

namespace dmtkg {

// Function attributes (the shared-memory opt-in) belong to the current
// device's context: raise them once per device, outside any graph capture.
// Runs f() (e.g. cudaFuncSetAttribute) once per device before any caller
// proceeds: concurrent first callers (loopback ranks) wait for it.
template <class F>
inline void once_on_device(std::atomic<unsigned long long>& mask, F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (mask.load(std::memory_order_acquire) & bit) return;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (mask.load(std::memory_order_acquire) & bit) return;
    f();
    mask.fetch_or(bit, std::memory_order_release);
}

// loopback all-reduce: out = sum of bufs[0..P-1] in rank order (P <= kLoopMax)
constexpr int kLoopMax = 16;
void launch_loop_sum(double* const* bufs, int P, long long n, double* out, cudaStream_t s);

// Fused cross-rank reduction over peer memory (xrank.cu).
// One rank's side of a launch: the local values (a plain buffer, or the CSR
// slot workspace of a streaming MTTKRP when rowptr is set), the output and
// the rank's per-block epoch counters.
struct XrankLocal {
    const double* src;
    const long long* rowptr;
    const long long* slots;
    double* out;
    unsigned long long* ctr;
};
// recv[k] / flags[k]: rank k's receive buffer [2][P][cap] and flag array
// [P][nblk_cap], mapped into this process (peer pointers, or one device's
// buffers for the emulated group). me[v]: virtual rank rank0 + v's side.
struct XrankArgs {
    int P, rank0, C;
    long long rows, cap, nblk_cap;
    double* recv[kLoopMax];
    unsigned long long* flags[kLoopMax];
    XrankLocal me[kLoopMax];
};
// grid = nblk x vranks (vranks > 1: the emulated group, all ranks in one
// cooperative launch); rows x C values, rows * C <= cap, nblk <= nblk_cap.
cudaError_t launch_xrank_reduce(const XrankArgs& a, int nblk, int vranks, cudaStream_t s);
int xrank_max_blocks();  // co-resident blocks of the kernel on the current device

void launch_krp_level(const double* P, const double* U, double* out, long long rows_out, long long J, int C,
                      cudaStream_t s);
void launch_mttkrp_generic(const double* X, long long L, long long I, long long R, int C, const KrpGen& kl,
                           const KrpGen& kr, long long jchunk, long long n_jc, double* ws, cudaStream_t s);
// Tensors symmetric in modes 0 and 1 (kernels.cu): check, pack the upper
// triangle (pairs p = j (j + 1) / 2 + i, padded to Pp), MTTKRP of mode 0/1 from
// the packed partial, pair weights of (A, B).
void launch_sym01_check(const double* X, long long I, long long pd0, long long R, int* flag, cudaStream_t s);
void launch_sym01_pack(const double* X, long long I, long long pd0, long long R, long long Pp, double* out,
                       cudaStream_t s);
void launch_sym01_mttv(const double* Q, long long I, int C, const double* V, double* M, cudaStream_t s);
void launch_sym01_pairs(const double* A, const double* B, long long I, int C, long long Pp, double* W, cudaStream_t s);
// Multi-TTV of a dimension-tree partial (see kernels.cu): M (dt x C) from P
// over rows a + A (i + dt b); ws holds multittv_ws_doubles(...) doubles.
long long multittv_ws_doubles(long long A, long long dt, long long B, int C);
void launch_multittv(const double* P, int C, long long A, long long dt, long long B, const KrpGen& kl,
                     const KrpGen& kr, double* ws, double* M, cudaStream_t s);
// nslots: total slots of the CSR map (few per row: one thread per (row, c))
void launch_slot_reduce(const double* ws, const long long* rowptr, const long long* slots, long long rows, int C,
                        double* out, cudaStream_t s, long long nslots);
void launch_matricize(const double* X, long long L, long long I, long long R, double* dst, cudaStream_t s);
void launch_gram_hadamard_accum(const double* U, long long rows, int C, double* H, bool first, cudaStream_t s);
void launch_fill(double* p, long long n, double v, cudaStream_t s);
void launch_fit_history(double* fitb, int* count, cudaStream_t s);
// scratch: >= 2*64*64 + 64 doubles; flag: 1 int
// Same contract through H^-1 = L^-T L^-1 and one dot product per output
// element (the ALS loop's fast path; rounding differs from the substitution).
void launch_solve_psd_inverse(const double* H, int n, const double* M, long long rows, double* U, double* scratch,
                              int* flag, cudaStream_t s);
void launch_solve_psd(const double* H, int n, const double* M, long long rows, double* U, double* scratch, int* flag,
                      cudaStream_t s);
void launch_normalize(double* U, long long rows, int C, double* lambda, cudaStream_t s);
void launch_fit(const double* U, const double* Mlast, long long rows, int C, const double* lambda, const double* Hlast,
                const double* normx, double* out, cudaStream_t s);
void launch_tensor_norm(const double* x, long long n, double* part, int nparts, double* out, cudaStream_t s);
void launch_dmma_peak(double* out, int blocks, int iters, cudaStream_t s);
// mt_gen.cu: gen_tensor (bench.cpp:88-97) on the device, bitwise; dst[(q / d0) * pd0 + q % d0] = draw q
size_t mt64_scratch_words(int nsm);
void mt64_generate(double* dst, long long n, long long d0, long long pd0, uint64_t seed, int nsm,
                   uint64_t* dev_scratch, cudaStream_t s);
// gen_dist.cu: value transforms of the seeded uniforms (dist 2 U[-1,1), 3 N(0,1)
// Box-Muller, 4 symmetric fMRI slices with tanh(0.3 z) off-diagonals), bitwise
// equal to the test-side restatement; u holds gen_dist_uniforms(...) draws
long long gen_dist_uniforms(int dist, long long total, long long I);
void launch_gen_dist(const double* u, long long total, int dist, long long I, long long d0, long long pd0,
                     double* dst, int nsm, cudaStream_t s);
// CP-ALS with cached Grams
void launch_gram(const double* U, long long rows, int C, double* G, cudaStream_t s);
void launch_hadamard_grams(const double* grams, int nmodes, int C, int skip, double* H, cudaStream_t s);
void launch_normalize_cols(double* U, long long rows, int C, double* lambda, cudaStream_t s);
// sharded rows (CP-ALS over last-mode shards): a shard's column sums of squares, then the
// normalisation by the sums over all shards
void launch_col_sumsq(const double* U, long long rows, int C, double* sumsq, cudaStream_t s);
void launch_normalize_cols_by(double* U, long long rows, int C, const double* sumsq, double* lambda, cudaStream_t s);
// sharded fit: a shard's <X, Y> partial, then the fit from the summed inner product
void launch_fit_inner(const double* U, const double* Mlast, long long rows, int C, const double* lambda,
                      double* inner_out, cudaStream_t s);
void launch_fit_from_inner(const double* lambda, int C, const double* Hlast, const double* Glast,
                           const double* normx, const double* inner, double* out, cudaStream_t s);
// One ALS factor update (Hadamard of cached Grams, solve through H^-1,
// normalise, new Gram). Returns the launch count.
long long als_fused_scratch_doubles();  // partial-Gram scratch after the 3 * 64 * 64 + 64 solve scratch
int launch_als_update(const double* grams, int nmodes, int C, int skip, double* H, const double* M, long long rows,
                      double* U, double* lambda, double* Gn, double* scratch, int* flag, cudaStream_t s,
                      bool solve_only = false);
void launch_fit_cached(const double* U, const double* Mlast, long long rows, int C, const double* lambda,
                       const double* Hlast, const double* Glast, const double* normx, double* out, cudaStream_t s);

// als_wide.cu: the CP-ALS update for ranks above 64 (global-memory systems)
long long wide_scratch_doubles(int C, long long max_rows);
void launch_wide_gram(const double* U, long long rows, int C, double* G, cudaStream_t s);
void launch_wide_hadamard(const double* grams, int nmodes, int C, int skip, double* H, cudaStream_t s);
int launch_wide_solve(const double* H, int C, const double* M, long long rows, double* U, double* scratch, int* flag,
                      cudaStream_t s);
void launch_wide_col_sumsq(const double* U, long long rows, int C, double* sumsq, cudaStream_t s);
void launch_wide_normalize_by(double* U, long long rows, int C, const double* sumsq, double* lambda, cudaStream_t s);
int launch_wide_als_update(const double* grams, int nmodes, int C, int skip, double* H, const double* M,
                           long long rows, double* U, double* lambda, double* Gn, double* scratch, double* sumsq,
                           int* flag, cudaStream_t s, bool solve_only);
void launch_wide_fit(const double* U, const double* Mlast, long long rows, int C, const double* lambda,
                     const double* Hlast, const double* Glast, const double* normx, double* out, const double* inner_in,
                     double* inner_out, cudaStream_t s);

// Tensor-core streaming MTTKRP (mttkrp_tc.cuh). nb in [1, 8], tail in
// {0, 1, 2, 4}, rb (row blocks per warp, p.RB) in {2, 3, 4}; returns false /
// -1 when no instantiation matches.
bool tc_has_tile(int nb, int tail, int rb);
int tc_smem_bytes(int nb, int tail, int G, int stages, int rb);
bool launch_mttkrp_tc(const TcPlan& p, const CUtensorMap& map, int nb, int tail, bool kmajor, int grid, cudaStream_t s);

}  // namespace dmtkg
