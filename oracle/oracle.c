/*
 * oracle.c -- plain-C restatement of the reference dmtk hot path.
 * TEST INFRASTRUCTURE ONLY (see oracle.h): the checker, never the product.
 * Citations are /root/reference/proj/<file>:<line>.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* mt19937_64, the published Matsumoto-Nishimura 64-bit Mersenne Twister    */
/* (the engine std::mt19937_64 names; used by bench.cpp:93 and cp_als.cpp:89) */
/* ------------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i) {
        const uint64_t prev = g->mt[i - 1];
        g->mt[i] = 6364136223846793005ULL * (prev ^ (prev >> 62)) + (uint64_t)i;
    }
    g->idx = MT_N;
}

static void mt_twist(orc_mt64* g) {
    for (int i = 0; i < MT_N; ++i) {
        const uint64_t y = (g->mt[i] & MT_UPPER) | (g->mt[(i + 1) % MT_N] & MT_LOWER);
        uint64_t v = g->mt[(i + MT_M) % MT_N] ^ (y >> 1);
        if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
        g->mt[i] = v;
    }
    g->idx = 0;
}

uint64_t orc_mt64_next(orc_mt64* g) {
    if (g->idx >= MT_N) mt_twist(g);
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

double orc_uniform01(orc_mt64* g) { return (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53; }

void orc_gen_uniform(uint64_t seed, int64_t n, double* out) {
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = orc_uniform01(&g);
}

uint64_t orc_mode_seed(uint64_t seed, int64_t mode) {
    return seed + 0x9e3779b97f4a7c15ULL * (uint64_t)(mode + 1);
}

void orc_gen_factors(int ndim, const int64_t* dims, int64_t rank, uint64_t seed, double* out) {
    int64_t off = 0;
    for (int n = 0; n < ndim; ++n) {
        orc_gen_uniform(orc_mode_seed(seed, n), dims[n] * rank, out + off);
        off += dims[n] * rank;
    }
}

void orc_kruskal_random(int ndim, const int64_t* dims, int64_t rank, uint64_t seed,
                        double* factors_out, double* lambda_out) {
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    int64_t total = 0;
    for (int n = 0; n < ndim; ++n) total += dims[n] * rank;
    for (int64_t i = 0; i < total; ++i) factors_out[i] = orc_uniform01(&g);
    for (int64_t c = 0; c < rank; ++c) lambda_out[c] = 1.0;
}

/* ------------------------------------------------------------------------ */
/* Khatri-Rao: iterated Kronecker per column (oracle.cpp:9-36)              */
/* ------------------------------------------------------------------------ */
int orc_krp_kron(int z, const double* const* inputs, const int64_t* rows, int64_t cols,
                 double* out) {
    if (z < 1 || cols < 0) return -1;
    int64_t total = 1;
    for (int k = 0; k < z; ++k) {
        if (!inputs[k] || rows[k] < 1) return -1;
        total *= rows[k];
    }
    double* cur = (double*)malloc(sizeof(double) * (size_t)total);
    double* nxt = (double*)malloc(sizeof(double) * (size_t)total);
    if (!cur || !nxt) {
        free(cur);
        free(nxt);
        return -1;
    }
    for (int64_t c = 0; c < cols; ++c) {
        int64_t len = rows[0];
        for (int64_t r = 0; r < len; ++r) cur[r] = inputs[0][r * cols + c];
        for (int k = 1; k < z; ++k) {
            const int64_t ur = rows[k];
            for (int64_t i = 0; i < len; ++i)
                for (int64_t t = 0; t < ur; ++t) nxt[i * ur + t] = cur[i] * inputs[k][t * cols + c];
            len *= ur;
            double* tmp = cur;
            cur = nxt;
            nxt = tmp;
        }
        for (int64_t r = 0; r < total; ++r) out[r * cols + c] = cur[r];
    }
    free(cur);
    free(nxt);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* MTTKRP by exhaustive summation (oracle.cpp:38-70)                        */
/* ------------------------------------------------------------------------ */
int orc_mttkrp_loops(int ndim, const int64_t* dims, const double* x,
                     const double* const* factors, int64_t rank, int64_t mode, double* out) {
    if (ndim < 1 || mode < 0 || mode >= ndim || rank < 1) return -1;
    int64_t total = 1;
    for (int k = 0; k < ndim; ++k) total *= dims[k];
    memset(out, 0, sizeof(double) * (size_t)(dims[mode] * rank));
    int64_t index[64];
    if (ndim > 64) return -1;
    for (int k = 0; k < ndim; ++k) index[k] = 0;
    for (int64_t off = 0; off < total; ++off) {
        const double v = x[off];
        double* mrow = out + index[mode] * rank;
        for (int64_t c = 0; c < rank; ++c) {
            double p = v;
            for (int k = 0; k < ndim; ++k) {
                if (k == mode) continue;
                p *= factors[k][index[k] * rank + c];
            }
            mrow[c] += p;
        }
        for (int k = 0; k < ndim; ++k) { /* mode 0 varies fastest */
            if (++index[k] < dims[k]) break;
            index[k] = 0;
        }
    }
    return 0;
}

int orc_reconstruct(int ndim, const int64_t* dims, const double* const* factors,
                    const double* lambda, int64_t rank, double* out) {
    if (ndim < 1 || ndim > 64) return -1;
    int64_t total = 1;
    for (int k = 0; k < ndim; ++k) total *= dims[k];
    int64_t index[64];
    for (int k = 0; k < ndim; ++k) index[k] = 0;
    for (int64_t off = 0; off < total; ++off) {
        double v = 0.0;
        for (int64_t c = 0; c < rank; ++c) {
            double p = lambda[c];
            for (int k = 0; k < ndim; ++k) p *= factors[k][index[k] * rank + c];
            v += p;
        }
        out[off] = v;
        for (int k = 0; k < ndim; ++k) {
            if (++index[k] < dims[k]) break;
            index[k] = 0;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Gram / solve (linalg.cpp:210-387)                                        */
/* ------------------------------------------------------------------------ */
void orc_gram(const double* u, int64_t rows, int64_t c, double* g) {
    memset(g, 0, sizeof(double) * (size_t)(c * c));
    for (int64_t r = 0; r < rows; ++r) {
        const double* row = u + r * c;
        for (int64_t c1 = 0; c1 < c; ++c1) {
            const double a = row[c1];
            for (int64_t c2 = c1; c2 < c; ++c2) g[c1 * c + c2] += a * row[c2];
        }
    }
    for (int64_t c1 = 0; c1 < c; ++c1)
        for (int64_t c2 = c1 + 1; c2 < c; ++c2) g[c2 * c + c1] = g[c1 * c + c2];
}

void orc_gram_hadamard(int ndim, const int64_t* dims, const double* const* factors, int64_t c,
                       int64_t skip, double* h) {
    double* g = (double*)malloc(sizeof(double) * (size_t)(c * c));
    for (int64_t i = 0; i < c * c; ++i) h[i] = 1.0;
    for (int n = 0; n < ndim; ++n) {
        if (n == skip) continue;
        orc_gram(factors[n], dims[n], c, g);
        for (int64_t i = 0; i < c * c; ++i) h[i] *= g[i];
    }
    free(g);
}

/* linalg.cpp:254-276 */
static int cholesky(const double* h, int64_t n, double* l) {
    double trace = 0.0;
    for (int64_t i = 0; i < n; ++i) trace += h[i * n + i];
    const double tol = 1e-12 * trace;
    memset(l, 0, sizeof(double) * (size_t)(n * n));
    for (int64_t j = 0; j < n; ++j) {
        double d = h[j * n + j];
        for (int64_t k = 0; k < j; ++k) d -= l[j * n + k] * l[j * n + k];
        if (d <= tol) return 0;
        const double root = sqrt(d);
        l[j * n + j] = root;
        for (int64_t i = j + 1; i < n; ++i) {
            double s = h[i * n + j];
            for (int64_t k = 0; k < j; ++k) s -= l[i * n + k] * l[j * n + k];
            l[i * n + j] = s / root;
        }
    }
    return 1;
}

/* linalg.cpp:281-326, cyclic Jacobi */
static void jacobi_eigen(double* a, double* v, int64_t n) {
    for (int64_t i = 0; i < n * n; ++i) v[i] = 0.0;
    for (int64_t i = 0; i < n; ++i) v[i * n + i] = 1.0;
    for (int sweep = 0; sweep < 128; ++sweep) {
        double off = 0.0;
        for (int64_t p = 0; p < n; ++p)
            for (int64_t q = p + 1; q < n; ++q) off += a[p * n + q] * a[p * n + q];
        if (off <= 1e-300) return;
        double diag = 0.0;
        for (int64_t p = 0; p < n; ++p) diag += a[p * n + p] * a[p * n + p];
        if (off <= 1e-30 * (diag > 1e-300 ? diag : 1e-300)) return;
        for (int64_t p = 0; p < n; ++p) {
            for (int64_t q = p + 1; q < n; ++q) {
                const double apq = a[p * n + q];
                if (apq == 0.0) continue;
                const double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double cs = 1.0 / sqrt(t * t + 1.0);
                const double sn = t * cs;
                for (int64_t r = 0; r < n; ++r) {
                    const double arp = a[r * n + p], arq = a[r * n + q];
                    a[r * n + p] = cs * arp - sn * arq;
                    a[r * n + q] = sn * arp + cs * arq;
                }
                for (int64_t cc = 0; cc < n; ++cc) {
                    const double apc = a[p * n + cc], aqc = a[q * n + cc];
                    a[p * n + cc] = cs * apc - sn * aqc;
                    a[q * n + cc] = sn * apc + cs * aqc;
                }
                for (int64_t r = 0; r < n; ++r) {
                    const double vrp = v[r * n + p], vrq = v[r * n + q];
                    v[r * n + p] = cs * vrp - sn * vrq;
                    v[r * n + q] = sn * vrp + cs * vrq;
                }
            }
        }
    }
}

int orc_solve_psd(const double* h, int64_t n, const double* m, int64_t rows, double* u) {
    double* l = (double*)malloc(sizeof(double) * (size_t)(n * n));
    if (cholesky(h, n, l)) { /* linalg.cpp:339-356 */
        double* w = (double*)malloc(sizeof(double) * (size_t)n);
        for (int64_t r = 0; r < rows; ++r) {
            const double* mrow = m + r * n;
            for (int64_t j = 0; j < n; ++j) {
                double s = mrow[j];
                for (int64_t k = 0; k < j; ++k) s -= l[j * n + k] * w[k];
                w[j] = s / l[j * n + j];
            }
            double* urow = u + r * n;
            for (int64_t j = n; j-- > 0;) {
                double s = w[j];
                for (int64_t k = j + 1; k < n; ++k) s -= l[k * n + j] * urow[k];
                urow[j] = s / l[j * n + j];
            }
        }
        free(w);
        free(l);
        return 1;
    }
    free(l);
    /* linalg.cpp:358-386: Jacobi pseudoinverse */
    double* a = (double*)malloc(sizeof(double) * (size_t)(n * n));
    double* v = (double*)malloc(sizeof(double) * (size_t)(n * n));
    double* gain = (double*)calloc((size_t)n, sizeof(double));
    double* tmp = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(a, h, sizeof(double) * (size_t)(n * n));
    jacobi_eigen(a, v, n);
    double lam_max = 0.0;
    for (int64_t i = 0; i < n; ++i)
        if (a[i * n + i] > lam_max) lam_max = a[i * n + i];
    const double floor_ = 1e-12 * lam_max;
    for (int64_t i = 0; i < n; ++i) {
        const double lam = a[i * n + i];
        if (lam > floor_ && lam > 0.0) gain[i] = 1.0 / lam;
    }
    for (int64_t r = 0; r < rows; ++r) {
        const double* mrow = m + r * n;
        for (int64_t j = 0; j < n; ++j) {
            double s = 0.0;
            for (int64_t c = 0; c < n; ++c) s += mrow[c] * v[c * n + j];
            tmp[j] = s * gain[j];
        }
        double* urow = u + r * n;
        for (int64_t c = 0; c < n; ++c) {
            double s = 0.0;
            for (int64_t j = 0; j < n; ++j) s += tmp[j] * v[c * n + j];
            urow[c] = s;
        }
    }
    free(a);
    free(v);
    free(gain);
    free(tmp);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* CP-ALS (cp_als.cpp)                                                      */
/* ------------------------------------------------------------------------ */
double orc_tensor_norm(const double* x, int64_t n) { /* cp_als.cpp:21-30,120 */
    const int64_t chunk = (int64_t)1 << 20;
    double acc = 0.0;
    for (int64_t i = 0; i < n; i += chunk) {
        const int64_t e = i + chunk < n ? i + chunk : n;
        double s = 0.0;
        for (int64_t k = i; k < e; ++k) s += x[k] * x[k];
        acc += s;
    }
    return sqrt(acc);
}

void orc_normalize_mode(double* u, int64_t rows, int64_t c, double* lambda) {
    for (int64_t col = 0; col < c; ++col) { /* cp_als.cpp:101-118 */
        double sq = 0.0;
        for (int64_t i = 0; i < rows; ++i) sq += u[i * c + col] * u[i * c + col];
        const double norm = sqrt(sq);
        lambda[col] = norm;
        if (norm > 0.0) {
            const double inv = 1.0 / norm;
            for (int64_t i = 0; i < rows; ++i) u[i * c + col] *= inv;
        }
    }
}

orc_fit_result orc_fit_from_last_mode(double norm_x, const double* u_last, int64_t rows,
                                      int64_t c, const double* lambda, const double* m_last,
                                      const double* h_skip_last) {
    double inner = 0.0; /* cp_als.cpp:40-47 */
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t k = 0; k < c; ++k) inner += m_last[i * c + k] * lambda[k] * u_last[i * c + k];
    double* g = (double*)malloc(sizeof(double) * (size_t)(c * c));
    orc_gram(u_last, rows, c, g);
    double norm_y_sq = 0.0; /* cp_als.cpp:49-57 */
    for (int64_t c1 = 0; c1 < c; ++c1)
        for (int64_t c2 = 0; c2 < c; ++c2)
            norm_y_sq += lambda[c1] * lambda[c2] * h_skip_last[c1 * c + c2] * g[c1 * c + c2];
    free(g);
    orc_fit_result out;
    double res_sq = norm_x * norm_x - 2.0 * inner + norm_y_sq;
    if (res_sq < 0.0) res_sq = 0.0;
    out.abs_residual = sqrt(res_sq);
    if (norm_x > 0.0) {
        out.rel_residual = out.abs_residual / norm_x;
        out.fit = 1.0 - out.rel_residual;
        out.defined = 1;
    } else {
        out.rel_residual = 0.0;
        out.fit = 0.0;
        out.defined = 0;
    }
    return out;
}

int orc_cp_als(int ndim, const int64_t* dims, const double* x, int64_t rank, int max_iters,
               double tol, uint64_t seed, double* factors_out, double* lambda_out,
               double* fits_out, int* zero_tensor) {
    if (rank < 1 || max_iters < 0 || ndim < 1) return -1; /* cp_als.cpp:175-177 */
    int64_t total = 1, fsize = 0, maxrows = 0;
    for (int n = 0; n < ndim; ++n) {
        total *= dims[n];
        fsize += dims[n] * rank;
        if (dims[n] > maxrows) maxrows = dims[n];
    }
    const double norm_x = orc_tensor_norm(x, total);
    orc_kruskal_random(ndim, dims, rank, seed, factors_out, lambda_out);
    *zero_tensor = 0;
    if (norm_x == 0.0) { /* cp_als.cpp:183-189 */
        memset(factors_out, 0, sizeof(double) * (size_t)fsize);
        for (int64_t c = 0; c < rank; ++c) lambda_out[c] = 0.0;
        *zero_tensor = 1;
        return 0;
    }
    const double* fptr[64];
    double* fmut[64];
    int64_t off = 0;
    for (int n = 0; n < ndim; ++n) {
        fmut[n] = factors_out + off;
        fptr[n] = fmut[n];
        off += dims[n] * rank;
    }
    double* m = (double*)malloc(sizeof(double) * (size_t)(maxrows * rank));
    double* h = (double*)malloc(sizeof(double) * (size_t)(rank * rank));
    double* unew = (double*)malloc(sizeof(double) * (size_t)(maxrows * rank));
    double prev_fit = 0.0;
    int iters = 0;
    for (int iter = 1; iter <= max_iters; ++iter) { /* cp_als.cpp:192-198 */
        for (int n = 0; n < ndim; ++n) {            /* als_iterate, cp_als.cpp:134-153 */
            orc_mttkrp_loops(ndim, dims, x, fptr, rank, n, m);
            orc_gram_hadamard(ndim, dims, fptr, rank, n, h);
            orc_solve_psd(h, rank, m, dims[n], unew);
            memcpy(fmut[n], unew, sizeof(double) * (size_t)(dims[n] * rank));
            orc_normalize_mode(fmut[n], dims[n], rank, lambda_out);
        }
        /* h and m still hold the last mode's values (cp_als.cpp:149-155) */
        const orc_fit_result f = orc_fit_from_last_mode(norm_x, fmut[ndim - 1], dims[ndim - 1],
                                                        rank, lambda_out, m, h);
        fits_out[iter - 1] = f.fit;
        iters = iter;
        if (iter > 1 && fabs(f.fit - prev_fit) < tol) break;
        prev_fit = f.fit;
    }
    free(m);
    free(h);
    free(unew);
    return iters;
}
