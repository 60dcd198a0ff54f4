// ref_capi.cpp -- extern "C" wrapper over the UNMODIFIED reference dmtk
// library, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libdmtk_ref.so.
//
// TEST / BASELINE INFRASTRUCTURE ONLY: used by tests/ (to pin the oracle and
// the CUDA path against the real reference), tests/golden/make_golden.py and
// bench.py's reference arm / cpu_baseline leg. The product never links it.
//
// Status codes (shared with include/dmtk_gpu.h):
//   0 ok, 1 std::invalid_argument, 2 std::out_of_range, 3 std::overflow_error,
//   4 any other exception, 5 dmtk::TensorFileError. The message is kept in a thread-local buffer.
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "dmtk/bench.hpp"
#include "dmtk/cp_als.hpp"
#include "dmtk/krp.hpp"
#include "dmtk/linalg.hpp"
#include "dmtk/mttkrp.hpp"
#include "dmtk/oracle.hpp"
#include "dmtk/tensor.hpp"
#include "dmtk/tensor_io.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::overflow_error& e) {
        g_err = e.what();
        return 3;
    } catch (const dmtk::TensorFileError& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

dmtk::Shape shape_of(int ndim, const int64_t* dims) {
    return dmtk::Shape(std::vector<std::int64_t>(dims, dims + ndim));
}

// Factors arrive as one concatenated buffer U_0 | U_1 | ... (row-major).
std::vector<dmtk::FactorMatrix> unpack(int n, const int64_t* rows, int64_t cols, const double* concat) {
    std::vector<dmtk::FactorMatrix> out;
    std::int64_t off = 0;
    for (int k = 0; k < n; ++k) {
        out.emplace_back(rows[k], cols,
                         std::vector<double>(concat + off, concat + off + rows[k] * cols));
        off += rows[k] * cols;
    }
    return out;
}

void put_times(const dmtk::TimeBreakdown& t, double* out8) {
    if (!out8) return;
    const double v[8] = {t.total, t.matmul, t.krp_full, t.krp_partial, t.matvec, t.reduce, t.reorder, t.other};
    std::memcpy(out8, v, sizeof(v));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// dmtk::write_tensor / read_tensor (tensor_io.hpp:24-25).
int ref_write_tensor(const char* path, int ndim, const int64_t* dims, const double* x) {
    return guarded([&] {
        const dmtk::Shape shape = shape_of(ndim, dims);
        const dmtk::DenseTensor t = dmtk::DenseTensor::borrow(shape, x, shape.total());
        dmtk::write_tensor(path, t);
    });
}

// values_out may be NULL (validation only); capacity in doubles.
int ref_read_tensor(const char* path, int* ndim, int64_t* dims_out64, double* values_out, int64_t capacity) {
    return guarded([&] {
        const dmtk::DenseTensor t = dmtk::read_tensor(path);
        *ndim = static_cast<int>(t.shape().ndim());
        for (int k = 0; k < *ndim; ++k) dims_out64[k] = t.shape().dim(k);
        if (values_out) {
            const auto v = t.values();
            if (static_cast<int64_t>(v.size()) > capacity) throw std::invalid_argument("capacity");
            std::memcpy(values_out, v.data(), v.size() * sizeof(double));
        }
    });
}

// dmtk::mttkrp (mttkrp.hpp:45). algo: 0 baseline, 1 one_step, 2 two_step,
// 3 automatic (mttkrp.hpp:16-21); order: 0 automatic, 1 left, 2 right.
int ref_mttkrp(int ndim, const int64_t* dims, const double* x, const double* factors,
               int64_t rank, int64_t mode, int algo, int order, int threads, double* out,
               double* times8) {
    return guarded([&] {
        const dmtk::Shape shape = shape_of(ndim, dims);
        const dmtk::DenseTensor t = dmtk::DenseTensor::borrow(shape, x, shape.total());
        const auto f = unpack(ndim, dims, rank, factors);
        dmtk::MttkrpRequest req;
        req.tensor = &t;
        req.factors = f;
        req.mode = mode;
        req.algo = static_cast<dmtk::MttkrpAlgo>(algo);
        req.order = static_cast<dmtk::TwoStepOrder>(order);
        req.threads = threads;
        const dmtk::MttkrpResult r = dmtk::mttkrp(req);
        std::memcpy(out, r.m.data(), sizeof(double) * static_cast<size_t>(r.m.rows() * r.m.cols()));
        put_times(r.time, times8);
    });
}

int ref_choose_order(int ndim, const int64_t* dims, int64_t mode) {
    return static_cast<int>(dmtk::choose_order(shape_of(ndim, dims), mode));
}

// dmtk::krp / krp_naive (krp.hpp:75-79). variant 0 = reuse, 1 = naive.
int ref_krp(int z, const int64_t* rows, int64_t cols, const double* inputs, int threads,
            int variant, double* out, uint64_t* hadamards) {
    return guarded([&] {
        const auto mats = unpack(z, rows, cols, inputs);
        dmtk::FactorList list;
        for (const auto& m : mats) list.push_back(&m);
        dmtk::KrpStats stats;
        const dmtk::FactorMatrix k =
            variant == 0 ? dmtk::krp(list, threads, &stats) : dmtk::krp_naive(list, threads, &stats);
        std::memcpy(out, k.data(), sizeof(double) * static_cast<size_t>(k.rows() * k.cols()));
        if (hadamards) *hadamards = stats.hadamard_products;
    });
}

int ref_mttkrp_oracle(int ndim, const int64_t* dims, const double* x, const double* factors,
                      int64_t rank, int64_t mode, double* out) {
    return guarded([&] {
        const dmtk::Shape shape = shape_of(ndim, dims);
        const dmtk::DenseTensor t = dmtk::DenseTensor::borrow(shape, x, shape.total());
        const auto f = unpack(ndim, dims, rank, factors);
        const dmtk::FactorMatrix m = dmtk::oracle::mttkrp_loops(t, f, mode, shape.total());
        std::memcpy(out, m.data(), sizeof(double) * static_cast<size_t>(m.rows() * m.cols()));
    });
}

// bench.cpp:88-116 generators.
int ref_gen_tensor(int ndim, const int64_t* dims, uint64_t seed, double* out) {
    return guarded([&] {
        const dmtk::DenseTensor t = dmtk::bench::gen_tensor(shape_of(ndim, dims), seed);
        std::memcpy(out, t.data(), sizeof(double) * static_cast<size_t>(t.total()));
    });
}

int ref_gen_factors(int ndim, const int64_t* dims, int64_t rank, uint64_t seed, double* out) {
    return guarded([&] {
        const auto f = dmtk::bench::gen_factors(shape_of(ndim, dims), rank, seed);
        std::int64_t off = 0;
        for (const auto& m : f) {
            std::memcpy(out + off, m.data(), sizeof(double) * static_cast<size_t>(m.rows() * m.cols()));
            off += m.rows() * m.cols();
        }
    });
}

int ref_kruskal_random(int ndim, const int64_t* dims, int64_t rank, uint64_t seed, double* factors,
                       double* lambda) {
    return guarded([&] {
        const dmtk::KruskalModel m = dmtk::KruskalModel::random(shape_of(ndim, dims), rank, seed);
        std::int64_t off = 0;
        for (const auto& u : m.factors) {
            std::memcpy(factors + off, u.data(), sizeof(double) * static_cast<size_t>(u.rows() * u.cols()));
            off += u.rows() * u.cols();
        }
        std::memcpy(lambda, m.lambda.data(), sizeof(double) * m.lambda.size());
    });
}

int ref_tensor_norm(int ndim, const int64_t* dims, const double* x, double* out) {
    return guarded([&] {
        const dmtk::Shape shape = shape_of(ndim, dims);
        *out = dmtk::tensor_norm(dmtk::DenseTensor::borrow(shape, x, shape.total()));
    });
}

int ref_gram_hadamard(int ndim, const int64_t* dims, int64_t rank, const double* factors,
                      int64_t skip, double* h) {
    return guarded([&] {
        const auto f = unpack(ndim, dims, rank, factors);
        const dmtk::GramMatrix g = dmtk::gram_hadamard(f, skip);
        std::memcpy(h, g.values.data(), sizeof(double) * g.values.size());
    });
}

int ref_solve_psd(int64_t c, const double* h, int64_t rows, const double* m, double* u) {
    return guarded([&] {
        dmtk::GramMatrix g(c);
        std::memcpy(g.values.data(), h, sizeof(double) * static_cast<size_t>(c * c));
        const dmtk::FactorMatrix mm(rows, c, std::vector<double>(m, m + rows * c));
        const dmtk::FactorMatrix r = dmtk::solve_psd(g, mm);
        std::memcpy(u, r.data(), sizeof(double) * static_cast<size_t>(rows * c));
    });
}

// dmtk::cp_als (cp_als.hpp:83). fits/iter_seconds capacity max_iters.
int ref_cp_als(int ndim, const int64_t* dims, const double* x, int64_t rank, int max_iters,
               double tol, uint64_t seed, int threads, int algo, int order, double* factors,
               double* lambda, double* fits, double* iter_seconds, int* n_iters, int* zero_tensor,
               double* norm_x) {
    return guarded([&] {
        const dmtk::Shape shape = shape_of(ndim, dims);
        const dmtk::DenseTensor t = dmtk::DenseTensor::borrow(shape, x, shape.total());
        dmtk::AlsConfig cfg;
        cfg.rank = rank;
        cfg.max_iters = max_iters;
        cfg.tol = tol;
        cfg.seed = seed;
        cfg.threads = threads;
        cfg.algo = static_cast<dmtk::MttkrpAlgo>(algo);
        cfg.order = static_cast<dmtk::TwoStepOrder>(order);
        const dmtk::AlsResult r = dmtk::cp_als(t, cfg);
        std::int64_t off = 0;
        for (const auto& u : r.model.factors) {
            std::memcpy(factors + off, u.data(), sizeof(double) * static_cast<size_t>(u.rows() * u.cols()));
            off += u.rows() * u.cols();
        }
        std::memcpy(lambda, r.model.lambda.data(), sizeof(double) * r.model.lambda.size());
        *n_iters = static_cast<int>(r.trace.iters.size());
        for (size_t i = 0; i < r.trace.iters.size(); ++i) {
            fits[i] = r.trace.iters[i].fit.fit;
            if (iter_seconds) iter_seconds[i] = r.trace.iters[i].total_seconds;
        }
        *zero_tensor = r.trace.zero_tensor ? 1 : 0;
        *norm_x = r.trace.tensor_norm;
    });
}

// dmtk::als_iterate (cp_als.hpp:74-75): one sweep of `model` in place;
// out4 = fit, rel, abs, defined; *seconds = total_seconds.
int ref_als_iterate(int ndim, const int64_t* dims, const double* x, int64_t rank, double* factors, double* lambda,
                    int threads, int algo, int order, double norm_x, int iter_index, double* out4, double* seconds) {
    return guarded([&] {
        const dmtk::Shape shape = shape_of(ndim, dims);
        const dmtk::DenseTensor t = dmtk::DenseTensor::borrow(shape, x, shape.total());
        dmtk::KruskalModel m;
        m.factors = unpack(ndim, dims, rank, factors);
        m.lambda.assign(lambda, lambda + rank);
        dmtk::AlsConfig cfg;
        cfg.rank = rank;
        cfg.threads = threads;
        cfg.algo = static_cast<dmtk::MttkrpAlgo>(algo);
        cfg.order = static_cast<dmtk::TwoStepOrder>(order);
        const dmtk::AlsIterRecord r = dmtk::als_iterate(t, m, cfg, norm_x, iter_index);
        std::int64_t off = 0;
        for (const auto& u : m.factors) {
            std::memcpy(factors + off, u.data(), sizeof(double) * static_cast<size_t>(u.rows() * u.cols()));
            off += u.rows() * u.cols();
        }
        std::memcpy(lambda, m.lambda.data(), sizeof(double) * m.lambda.size());
        out4[0] = r.fit.fit;
        out4[1] = r.fit.rel_residual;
        out4[2] = r.fit.abs_residual;
        out4[3] = r.fit.defined ? 1.0 : 0.0;
        if (seconds) *seconds = r.total_seconds;
    });
}

// dmtk::fit (cp_als.hpp:79): returns fit, rel, abs, defined.
int ref_fit(int ndim, const int64_t* dims, const double* x, int64_t rank, const double* factors,
            const double* lambda, int threads, double* out4) {
    return guarded([&] {
        const dmtk::Shape shape = shape_of(ndim, dims);
        const dmtk::DenseTensor t = dmtk::DenseTensor::borrow(shape, x, shape.total());
        dmtk::KruskalModel m;
        m.factors = unpack(ndim, dims, rank, factors);
        m.lambda.assign(lambda, lambda + rank);
        const dmtk::FitResult f = dmtk::fit(t, m, threads);
        out4[0] = f.fit;
        out4[1] = f.rel_residual;
        out4[2] = f.abs_residual;
        out4[3] = f.defined ? 1.0 : 0.0;
    });
}

}  // extern "C"
