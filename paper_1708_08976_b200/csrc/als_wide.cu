// als_wide.cu -- the CP-ALS factor update for ranks above 64 (the reference
// accepts any rank >= 1, cp_als.cpp:175-177). The rank <= 64 kernels keep their
// C x C systems in shared memory and registers; these keep them in global
// memory (L1/L2-resident: a 256 x 256 system is 512 KB) and follow the
// reference's algorithms step for step:
//   Gram (linalg.cpp:210-226), Gram-Hadamard (:228-248),
//   solve_psd (:330-387): left-looking Cholesky with the 1e-12 * trace pivot
//   test (:254-276), then per-row forward and back substitution (:340-354);
//   else the cyclic-Jacobi pseudo-inverse (:281-326, 358-386),
//   normalize_mode (cp_als.cpp:101-118), the reconstruction-free fit
//   (cp_als.cpp:34-72).
// Reductions are fixed-order (deterministic). flag[0] = 1 when the Cholesky
// factorisation succeeded (the Jacobi kernels then return at once), as in the
// rank <= 64 path.
#include <cuda_runtime.h>

#include "kernels.h"

namespace dmtkg {
namespace {

constexpr int kT = 256;  // threads of the single-CTA kernels

__device__ double block_sum(double v, double* red) {
    // fixed-order: warp tree, then the warp sums by one thread in warp order
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) s += red[k];
        red[32] = s;
    }
    __syncthreads();
    return red[32];
}

// G = U^T U (rows x C), one thread per entry, rows in order
__global__ void wide_gram_kernel(const double* __restrict__ U, long long rows, int C, double* __restrict__ G) {
    pdl_wait();
    pdl_trigger();
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<long long>(C) * C) return;
    const int c1 = static_cast<int>(e / C), c2 = static_cast<int>(e % C);
    double s = 0.0;
    for (long long i = 0; i < rows; ++i) s = fma(U[i * C + c1], U[i * C + c2], s);
    G[e] = s;
}

// H = Hadamard of the cached Grams of every mode but `skip`
__global__ void wide_hadamard_kernel(const double* __restrict__ grams, int nmodes, int C, int skip,
                                     double* __restrict__ H) {
    pdl_wait();
    pdl_trigger();
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long cc = static_cast<long long>(C) * C;
    if (e >= cc) return;
    double h = 1.0;
    for (int k = 0; k < nmodes; ++k)
        if (k != skip) h *= grams[k * cc + e];
    H[e] = h;
}

// Left-looking Cholesky H = L L^T (linalg.cpp:254-276), one CTA: column j's
// entries are dot products over L's first j columns, one warp each (lanes
// split the k range, shuffle tree). flag[0] = 1 on success, 0 when a pivot
// falls to 1e-12 * trace or below.
__global__ void __launch_bounds__(kT) wide_cholesky_kernel(const double* __restrict__ H, int n, double* __restrict__ L,
                                                           int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    __shared__ double red[33];
    __shared__ double s_root;
    __shared__ int s_ok;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    double tr = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) tr += H[i * n + i];
    tr = block_sum(tr, red);
    const double tol = 1e-12 * tr;
    if (threadIdx.x == 0) s_ok = 1;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) L[e] = 0.0;
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        if (w == 0) {
            double d = 0.0;
            for (int k = l; k < j; k += 32) d = fma(L[j * n + k], L[j * n + k], d);
            for (int o = 16; o > 0; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
            if (l == 0) {
                const double piv = H[j * n + j] - d;
                if (piv <= tol) {
                    s_ok = 0;
                } else {
                    s_root = sqrt(piv);
                    L[j * n + j] = s_root;
                }
            }
        }
        __syncthreads();
        if (!s_ok) break;
        const double root = s_root;
        for (int i = j + 1 + w; i < n; i += nw) {
            double s = 0.0;
            for (int k = l; k < j; k += 32) s = fma(L[i * n + k], L[j * n + k], s);
            for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
            if (l == 0) L[i * n + j] = (H[i * n + j] - s) / root;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) flag[0] = s_ok;
}

// Per row: forward substitution L y = m, then back substitution L^T u = y
// (linalg.cpp:340-354), y kept in the output row. One thread per row.
__global__ void wide_chol_rows_kernel(const double* __restrict__ L, int n, const double* __restrict__ M, long long rows,
                                      double* __restrict__ U, const int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    if (!flag[0]) return;
    const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const double* m = M + r * n;
    double* u = U + r * n;
    for (int c = 0; c < n; ++c) {
        double s = m[c];
        for (int k = 0; k < c; ++k) s -= L[c * n + k] * u[k];
        u[c] = s / L[c * n + c];
    }
    for (int c = n - 1; c >= 0; --c) {
        double s = u[c];
        for (int k = c + 1; k < n; ++k) s -= L[k * n + c] * u[k];
        u[c] = s / L[c * n + c];
    }
}

// Cyclic Jacobi eigendecomposition of H (linalg.cpp:281-326): <= 128 sweeps,
// stop at off <= 1e-300 or <= 1e-30 diag; gain = 1/lambda above 1e-12
// lambda_max (:358-386). Only when the Cholesky factorisation failed.
__global__ void __launch_bounds__(kT) wide_jacobi_kernel(const double* __restrict__ H, int n, double* __restrict__ a,
                                                         double* __restrict__ v, double* __restrict__ gain,
                                                         const int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    if (flag[0]) return;
    __shared__ double red[33];
    __shared__ double s_cs, s_sn;
    __shared__ int s_done;
    const int tid = threadIdx.x;
    for (int e = tid; e < n * n; e += blockDim.x) {
        a[e] = H[e];
        v[e] = (e / n == e % n) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int sweep = 0; sweep < 128; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (int e = tid; e < n * n; e += blockDim.x) {
            const int p = e / n, q = e % n;
            if (q > p) off += a[e] * a[e];
            if (q == p) diag += a[e] * a[e];
        }
        off = block_sum(off, red);
        diag = block_sum(diag, red);
        if (tid == 0) s_done = (off <= 1e-300) || (off <= 1e-30 * (diag > 1e-300 ? diag : 1e-300));
        __syncthreads();
        if (s_done) break;
        for (int p = 0; p < n; ++p) {
            for (int q = p + 1; q < n; ++q) {
                if (tid == 0) {
                    const double apq = a[p * n + q];
                    if (apq == 0.0) {
                        s_cs = 1.0;
                        s_sn = 0.0;
                    } else {
                        const double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
                        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                        s_cs = 1.0 / sqrt(t * t + 1.0);
                        s_sn = t * s_cs;
                    }
                }
                __syncthreads();
                const double cs = s_cs, sn = s_sn;
                if (sn != 0.0 || cs != 1.0) {
                    for (int r = tid; r < n; r += blockDim.x) {
                        const double arp = a[r * n + p], arq = a[r * n + q];
                        a[r * n + p] = cs * arp - sn * arq;
                        a[r * n + q] = sn * arp + cs * arq;
                    }
                    __syncthreads();
                    for (int c = tid; c < n; c += blockDim.x) {
                        const double apc = a[p * n + c], aqc = a[q * n + c];
                        a[p * n + c] = cs * apc - sn * aqc;
                        a[q * n + c] = sn * apc + cs * aqc;
                    }
                    for (int r = tid; r < n; r += blockDim.x) {
                        const double vrp = v[r * n + p], vrq = v[r * n + q];
                        v[r * n + p] = cs * vrp - sn * vrq;
                        v[r * n + q] = sn * vrp + cs * vrq;
                    }
                }
                __syncthreads();
            }
        }
    }
    if (tid == 0) {
        double lam_max = 0.0;
        for (int i = 0; i < n; ++i) lam_max = a[i * n + i] > lam_max ? a[i * n + i] : lam_max;
        const double fl = 1e-12 * lam_max;
        for (int i = 0; i < n; ++i) {
            const double lam = a[i * n + i];
            gain[i] = (lam > fl && lam > 0.0) ? 1.0 / lam : 0.0;
        }
    }
}

// U = M V diag(gain) V^T per row (tmp: rows x n scratch)
__global__ void wide_jacobi_rows_kernel(const double* __restrict__ V, const double* __restrict__ gain, int n,
                                        const double* __restrict__ M, long long rows, double* __restrict__ tmp,
                                        double* __restrict__ U, const int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    if (flag[0]) return;
    const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const double* m = M + r * n;
    double* t = tmp + r * n;
    for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int c = 0; c < n; ++c) s += m[c] * V[c * n + j];
        t[j] = s * gain[j];
    }
    for (int c = 0; c < n; ++c) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += t[j] * V[c * n + j];
        U[r * n + c] = s;
    }
}

// Column sums of squares, one CTA per column (fixed order)
__global__ void __launch_bounds__(kT) wide_col_sumsq_kernel(const double* __restrict__ U, long long rows, int C,
                                                            double* __restrict__ sumsq) {
    pdl_wait();
    pdl_trigger();
    __shared__ double red[33];
    const int c = blockIdx.x;
    double sq = 0.0;
    for (long long i = threadIdx.x; i < rows; i += blockDim.x) sq = fma(U[i * C + c], U[i * C + c], sq);
    sq = block_sum(sq, red);
    if (threadIdx.x == 0) sumsq[c] = sq;
}

// lambda_c = sqrt(sumsq_c); column c scaled by 1 / lambda_c when positive
// (normalize_mode, cp_als.cpp:101-118)
__global__ void wide_normalize_by_kernel(double* __restrict__ U, long long rows, int C,
                                         const double* __restrict__ sumsq, double* __restrict__ lambda) {
    pdl_wait();
    pdl_trigger();
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long c = e % C;
    const double nrm = sqrt(sumsq[c]);
    if (e < C) lambda[e] = nrm;
    if (e < rows * C && nrm > 0.0) U[e] *= 1.0 / nrm;
}

// Reconstruction-free fit (cp_als.cpp:34-72): <X, Y> from the last mode's
// MTTKRP, ||Y||^2 from H o G_last. inner_out: write this shard's <X, Y> and
// stop; inner_in: take the summed <X, Y> from there.
__global__ void __launch_bounds__(kT) wide_fit_kernel(const double* __restrict__ U, const double* __restrict__ Mlast,
                                                      long long rows, int C, const double* __restrict__ lambda,
                                                      const double* __restrict__ Hlast,
                                                      const double* __restrict__ Glast,
                                                      const double* __restrict__ normx, double* __restrict__ out,
                                                      const double* __restrict__ inner_in,
                                                      double* __restrict__ inner_out) {
    pdl_wait();
    pdl_trigger();
    __shared__ double red[33];
    double inner = 0.0;
    if (!inner_in)
        for (long long e = threadIdx.x; e < rows * C; e += blockDim.x) inner += Mlast[e] * lambda[e % C] * U[e];
    inner = block_sum(inner, red);
    if (inner_out) {
        if (threadIdx.x == 0) inner_out[0] = inner;
        return;
    }
    if (inner_in) inner = inner_in[0];
    double ny = 0.0;
    for (long long e = threadIdx.x; e < static_cast<long long>(C) * C; e += blockDim.x)
        ny += lambda[e / C] * lambda[e % C] * Hlast[e] * Glast[e];
    ny = block_sum(ny, red);
    if (threadIdx.x == 0) {
        const double nx = normx[0];
        double res2 = nx * nx - 2.0 * inner + ny;
        if (res2 < 0.0) res2 = 0.0;
        const double ar = sqrt(res2);
        out[2] = ar;
        if (nx > 0.0) {
            out[1] = ar / nx;
            out[0] = 1.0 - out[1];
            out[3] = 1.0;
        } else {
            out[0] = 0.0;
            out[1] = 0.0;
            out[3] = 0.0;
        }
    }
}

unsigned blocks_for(long long n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

long long wide_scratch_doubles(int C, long long max_rows) {
    return 3LL * C * C + C + max_rows * C;
}

void launch_wide_gram(const double* U, long long rows, int C, double* G, cudaStream_t s) {
    launch_pdl(wide_gram_kernel, dim3(blocks_for(static_cast<long long>(C) * C, 128)), dim3(128), 0, s, U, rows, C, G);
}

void launch_wide_hadamard(const double* grams, int nmodes, int C, int skip, double* H, cudaStream_t s) {
    launch_pdl(wide_hadamard_kernel, dim3(blocks_for(static_cast<long long>(C) * C, 256)), dim3(256), 0, s, grams, nmodes, C, skip, H);
}

// solve_psd for any rank: scratch = wide_scratch_doubles(C, rows)
int launch_wide_solve(const double* H, int C, const double* M, long long rows, double* U, double* scratch, int* flag,
                      cudaStream_t s) {
    double* L = scratch;
    double* a = L + static_cast<long long>(C) * C;
    double* V = a + static_cast<long long>(C) * C;
    double* gain = V + static_cast<long long>(C) * C;
    double* tmp = gain + C;
    launch_pdl(wide_cholesky_kernel, dim3(1), dim3(kT), 0, s, H, C, L, flag);
    launch_pdl(wide_chol_rows_kernel, dim3(blocks_for(rows, 128)), dim3(128), 0, s, L, C, M, rows, U, flag);
    launch_pdl(wide_jacobi_kernel, dim3(1), dim3(kT), 0, s, H, C, a, V, gain, flag);
    launch_pdl(wide_jacobi_rows_kernel, dim3(blocks_for(rows, 128)), dim3(128), 0, s, V, gain, C, M, rows, tmp, U, flag);
    return 4;
}

void launch_wide_col_sumsq(const double* U, long long rows, int C, double* sumsq, cudaStream_t s) {
    launch_pdl(wide_col_sumsq_kernel, dim3(C), dim3(kT), 0, s, U, rows, C, sumsq);
}

void launch_wide_normalize_by(double* U, long long rows, int C, const double* sumsq, double* lambda, cudaStream_t s) {
    const long long n = rows * C > C ? rows * C : C;
    launch_pdl(wide_normalize_by_kernel, dim3(blocks_for(n, 256)), dim3(256), 0, s, U, rows, C, sumsq, lambda);
}

// One ALS factor update for any rank (the rank <= 64 launch_als_update's
// contract): Hadamard of cached Grams, solve_psd, normalise (column sums of
// squares into sumsq), new Gram. Returns the launch count.
int launch_wide_als_update(const double* grams, int nmodes, int C, int skip, double* H, const double* M,
                           long long rows, double* U, double* lambda, double* Gn, double* scratch, double* sumsq,
                           int* flag, cudaStream_t s, bool solve_only) {
    launch_wide_hadamard(grams, nmodes, C, skip, H, s);
    const int n = 1 + launch_wide_solve(H, C, M, rows, U, scratch, flag, s);
    if (solve_only) return n;
    launch_wide_col_sumsq(U, rows, C, sumsq, s);
    launch_wide_normalize_by(U, rows, C, sumsq, lambda, s);
    launch_wide_gram(U, rows, C, Gn, s);
    return n + 3;
}

void launch_wide_fit(const double* U, const double* Mlast, long long rows, int C, const double* lambda,
                     const double* Hlast, const double* Glast, const double* normx, double* out, const double* inner_in,
                     double* inner_out, cudaStream_t s) {
    launch_pdl(wide_fit_kernel, dim3(1), dim3(kT), 0, s, U, Mlast, rows, C, lambda, Hlast, Glast, normx, out, inner_in, inner_out);
}

}  // namespace dmtkg
