/*
 * oracle.h -- CPU restatement of the reference dmtk algorithms on the hot
 * path (MTTKRP, Khatri-Rao product, CP-ALS pieces) in plain C.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product path (the CUDA library,
 * its C-ABI, the Python mirror) may link, import or call this code. Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs use it, and only as the checker.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).
 *
 * Parity pinned: tests/test_oracle.py checks this restatement against the
 * reference's own known-answer tests (tests/test_krp.cpp, test_mttkrp.cpp,
 * test_cpals.cpp, test_linalg.cpp) and against golden vectors produced by
 * the real reference library compiled from /root/reference
 * (oracle/_ref/libdmtk_ref.so, see oracle/Makefile and
 * tests/golden/make_golden.py).
 *
 * Conventions (reference src/shape.cpp:8-25, include/dmtk/matrix.hpp:74-109):
 *   tensor: natural order, mode 0 fastest; offset = sum_n i_n * left(n)
 *   factor / KRP / MTTKRP matrices: row-major rows x C
 */
#ifndef DMTK_ORACLE_H
#define DMTK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- random generators (bench.cpp:22-28, 88-116; cp_als.cpp:16-19, 87-99) */
typedef struct {
    uint64_t mt[312];
    int idx;
} orc_mt64;

void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);
/* (r >> 11) * 2^-53 : bench.cpp:22-24 */
double orc_uniform01(orc_mt64* g);

/* n uniform(0,1) draws from mt19937_64(seed): bench.cpp:88-97 gen_tensor and
 * bench.cpp:99-106 gen_matrix (same stream). */
void orc_gen_uniform(uint64_t seed, int64_t n, double* out);
/* bench.cpp:26-28 */
uint64_t orc_mode_seed(uint64_t seed, int64_t mode);
/* bench.cpp:108-116: factor n from gen_matrix(I_n, rank, mode_seed(seed, n));
 * out is the concatenation U_0 | U_1 | ... (each row-major I_n x rank). */
void orc_gen_factors(int ndim, const int64_t* dims, int64_t rank, uint64_t seed, double* out);
/* cp_als.cpp:87-99 KruskalModel::random: ONE stream filling U_0..U_{N-1}. */
void orc_kruskal_random(int ndim, const int64_t* dims, int64_t rank, uint64_t seed,
                        double* factors_out, double* lambda_out);

/* ---- seeded value distributions (BASELINE configs 3-5; see oracle.c):
 * dist 0 U[0,1) (gen_tensor), 1 ones, 2 U[-1,1), 3 N(0,1) Box-Muller,
 * 4 symmetric fMRI slices (unit diagonal, tanh(0.3 z) off-diagonal).
 * Natural order, `threads` worker threads for the transform. 0 or -1. */
int orc_gen_dist(uint64_t seed, int dist, int ndim, const int64_t* dims, int threads, double* out);
/* uniform draws a distribution consumes */
int64_t orc_dist_uniforms(int dist, int ndim, const int64_t* dims);
/* gen_factors (bench.cpp:108-116) with the transform of `dist` per factor stream */
int orc_gen_factors_dist(int ndim, const int64_t* dims, int64_t rank, uint64_t seed, int dist, double* out);
double orc_box_muller(double u0, double u1, int second);
double orc_tanh_portable(double y);

/* ---- Khatri-Rao (oracle.cpp:9-36 krp_kron; krp.hpp:19-32 contract) -------
 * K = in[0] (.) in[1] (.) ... (.) in[Z-1], last input fastest, associated
 * left to right. out is (prod rows) x cols row-major. Returns 0 or -1. */
int orc_krp_kron(int z, const double* const* inputs, const int64_t* rows, int64_t cols,
                 double* out);

/* ---- MTTKRP by direct summation (oracle.cpp:38-70) ---------------------
 * factors[k] row-major I_k x rank (factors[mode] unused but required).
 * out: I_mode x rank row-major. Returns 0 or -1 on bad arguments. */
int orc_mttkrp_loops(int ndim, const int64_t* dims, const double* x,
                     const double* const* factors, int64_t rank, int64_t mode, double* out);

/* Dense reconstruction (oracle.cpp:72-101). */
int orc_reconstruct(int ndim, const int64_t* dims, const double* const* factors,
                    const double* lambda, int64_t rank, double* out);

/* ---- small dense linear algebra (linalg.cpp:210-387) -------------------- */
/* U^T U, upper triangle accumulated row by row then mirrored (linalg.cpp:210-226) */
void orc_gram(const double* u, int64_t rows, int64_t c, double* g);
/* Hadamard of Grams of all factors except skip (linalg.cpp:228-248) */
void orc_gram_hadamard(int ndim, const int64_t* dims, const double* const* factors, int64_t c,
                       int64_t skip, double* h);
/* U * H = M, Cholesky with pivot floor 1e-12*trace, else Jacobi pseudoinverse
 * clipping 1e-12*lambda_max (linalg.cpp:254-387). Returns 1 if Cholesky was
 * used, 0 for the Jacobi path. */
int orc_solve_psd(const double* h, int64_t c, const double* m, int64_t rows, double* u);

/* ---- CP-ALS (cp_als.cpp:21-200) ----------------------------------------- */
double orc_tensor_norm(const double* x, int64_t n);
/* cp_als.cpp:101-118 */
void orc_normalize_mode(double* u, int64_t rows, int64_t c, double* lambda);

typedef struct {
    double fit;
    double rel_residual;
    double abs_residual;
    int defined;
} orc_fit_result;

/* cp_als.cpp:34-72 */
orc_fit_result orc_fit_from_last_mode(double norm_x, const double* u_last, int64_t rows,
                                      int64_t c, const double* lambda, const double* m_last,
                                      const double* h_skip_last);

/* cp_als.cpp:174-200 with als_iterate (122-158). factors_out is the
 * concatenation of all U_n (row-major); fits_out gets one fit per completed
 * iteration (capacity max_iters). Returns the number of iterations run, or
 * -1 on invalid arguments; *zero_tensor set when ||X|| == 0. */
int orc_cp_als(int ndim, const int64_t* dims, const double* x, int64_t rank, int max_iters,
               double tol, uint64_t seed, double* factors_out, double* lambda_out,
               double* fits_out, int* zero_tensor);

#ifdef __cplusplus
}
#endif

#endif
