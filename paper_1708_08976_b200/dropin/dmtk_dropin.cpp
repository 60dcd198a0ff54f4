// dmtk_dropin.cpp -- link-compatible drop-in for the reference's hot path.
//
// Defines, with the reference's own signatures (proj/include/dmtk/*.hpp), every
// symbol of the reference translation units mttkrp.cpp, krp.cpp and cp_als.cpp:
//
//   dmtk::mttkrp / mttkrp_baseline / mttkrp_one_step / mttkrp_two_step /
//         choose_order                                  (mttkrp.hpp:45-53)
//   dmtk::krp / krp_naive / krp_small, KrpState, krp_row (krp.hpp:33-83)
//   dmtk::cp_als / als_iterate / fit / tensor_norm,
//         KruskalModel::random / normalize_mode          (cp_als.hpp:16-83)
//
// so a program built against the reference relinks without source edits:
// link libdmtk_dropin.so (+ libdmtk_gpu.so) in place of those three objects
// and keep the reference's remaining objects (shape, tensor, matrix, linalg,
// parallel, kernels*, tensor_io, bench, oracle) for the data types. Calls made
// from inside those objects (bench.cpp:298 bench_mttkrp, bench.cpp:364-374
// bench_krp, the CP-ALS harness) then run on the B200 too.
//
// The compute goes through the C ABI (include/dmtk_gpu.h) via the header shim
// include/dmtk_gpu.hpp (validation, messages and exception types of the
// reference). KrpState, KruskalModel::random and normalize_mode are the
// reference's host-side data utilities (a row iterator over host factors, the
// seeded initial model, a column scaling of a host factor) and run on the host
// as their contract describes; every product of the hot path runs on the GPU.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>

#include "dmtk/cp_als.hpp"
#include "dmtk/krp.hpp"
#include "dmtk/mttkrp.hpp"
#include "dmtk_gpu.hpp"

namespace dmtk {

// ------------------------------------------------------------ mttkrp.hpp
MttkrpResult mttkrp(const MttkrpRequest& req) { return gpu::mttkrp(req); }
MttkrpResult mttkrp_baseline(const MttkrpRequest& req) { return gpu::mttkrp_baseline(req); }
MttkrpResult mttkrp_one_step(const MttkrpRequest& req) { return gpu::mttkrp_one_step(req); }
MttkrpResult mttkrp_two_step(const MttkrpRequest& req) { return gpu::mttkrp_two_step(req); }
TwoStepOrder choose_order(const Shape& shape, std::int64_t mode) { return gpu::choose_order(shape, mode); }

// --------------------------------------------------------------- krp.hpp
FactorMatrix krp(const FactorList& inputs, int threads, KrpStats* stats) { return gpu::krp(inputs, threads, stats); }
FactorMatrix krp_naive(const FactorList& inputs, int threads, KrpStats* stats) {
    return gpu::krp_naive(inputs, threads, stats);
}
FactorMatrix krp_small(const FactorList& inputs, KrpStats* stats) { return gpu::krp_small(inputs, stats); }

namespace {
// input validation shared by KrpState (krp.cpp radices_of: same order, same messages)
std::vector<std::int64_t> krp_radices(const FactorList& inputs) {
    if (inputs.empty()) throw std::invalid_argument("krp: empty input list");
    const std::int64_t cols = inputs.front() ? inputs.front()->cols() : 0;
    std::vector<std::int64_t> r;
    for (std::size_t z = 0; z < inputs.size(); ++z) {
        if (!inputs[z]) throw std::invalid_argument("krp: null input");
        if (inputs[z]->cols() != cols)
            throw std::invalid_argument("krp: input " + std::to_string(z) + " has " +
                                        std::to_string(inputs[z]->cols()) + " columns, expected " +
                                        std::to_string(cols));
        if (inputs[z]->rows() < 1) throw std::invalid_argument("krp: input " + std::to_string(z) + " has no rows");
        r.push_back(inputs[z]->rows());
    }
    return r;
}

void hadamard_into(double* out, const double* a, const double* b, std::int64_t n) {
    for (std::int64_t c = 0; c < n; ++c) out[c] = a[c] * b[c];
}
}  // namespace

// Row iterator over host factors (krp.hpp:19-66): Z-2 cached running
// products P(p) = P(p-1) (.) input_{p+1}(d_{p+1}), P(0) = input_0 (.) input_1.
KrpState::KrpState(FactorList inputs, std::int64_t start_row)
    : inputs_(std::move(inputs)), index_(krp_radices(inputs_)) {
    cols_ = inputs_.front()->cols();
    if (z() >= 3) partials_.assign(static_cast<std::size_t>((z() - 2) * cols_), 0.0);
    seek(start_row);
}

std::span<const double> KrpState::input_row(std::int64_t input) const {
    return inputs_[static_cast<std::size_t>(input)]->row(index_.digit(input));
}

void KrpState::rebuild_from(std::int64_t first_partial) {
    for (std::int64_t p = std::max<std::int64_t>(first_partial, 0); p + 3 <= z(); ++p) {
        double* dst = partials_.data() + p * cols_;
        const double* prev = p == 0 ? input_row(0).data() : dst - cols_;
        hadamard_into(dst, prev, input_row(p + 1).data(), cols_);
        ++hadamards_;
    }
}

void KrpState::seek(std::int64_t row) {
    index_.init_from_row(row);
    rebuild_from(0);
}

void KrpState::write_row(std::span<double> out) {
    if (static_cast<std::int64_t>(out.size()) != cols_)
        throw std::invalid_argument("KrpState::write_row: output span has wrong length");
    if (z() == 1) {
        std::memcpy(out.data(), input_row(0).data(), static_cast<std::size_t>(cols_) * sizeof(double));
        return;
    }
    const double* head = z() == 2 ? input_row(0).data() : partials_.data() + (z() - 3) * cols_;
    hadamard_into(out.data(), head, input_row(z() - 1).data(), cols_);
    ++hadamards_;
}

void KrpState::advance() {
    // the odometer's carry touched digits Z - carry .. Z - 1; P(p) reads digits
    // 0 .. p + 1, so the partials from p = Z - carry - 1 on are stale
    const int carry = index_.increment();
    if (carry > 1) rebuild_from(z() - carry - 1);
}

void krp_row(KrpState& state, std::span<double> out) {
    if (state.z() < 3) throw std::invalid_argument("krp_row: needs Z >= 3 inputs; use krp_small for Z in {1,2}");
    state.write_row(out);
}

// ------------------------------------------------------------ cp_als.hpp
double tensor_norm(const DenseTensor& x) { return gpu::tensor_norm(x); }

KruskalModel KruskalModel::random(const Shape& shape, std::int64_t rank, std::uint64_t seed) {
    // one mt19937_64(seed) stream, (draw >> 11) * 2^-53, factors 0..N-1 in row-major order, lambda = 1
    if (rank < 1) throw std::invalid_argument("KruskalModel::random: rank must be >= 1");
    std::mt19937_64 rng(seed);
    KruskalModel m;
    for (std::int64_t n = 0; n < shape.ndim(); ++n) {
        FactorMatrix u(shape.dim(n), rank);
        double* p = u.data();
        for (std::int64_t e = 0; e < u.rows() * rank; ++e) p[e] = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        m.factors.push_back(std::move(u));
    }
    m.lambda.assign(static_cast<std::size_t>(rank), 1.0);
    return m;
}

void KruskalModel::normalize_mode(std::int64_t n) {
    FactorMatrix& u = factors.at(static_cast<std::size_t>(n));
    lambda.assign(static_cast<std::size_t>(u.cols()), 0.0);
    for (std::int64_t c = 0; c < u.cols(); ++c) {
        double sq = 0.0;
        for (std::int64_t i = 0; i < u.rows(); ++i) sq += u(i, c) * u(i, c);
        const double nrm = std::sqrt(sq);
        lambda[static_cast<std::size_t>(c)] = nrm;
        if (nrm > 0.0) {
            const double inv = 1.0 / nrm;
            for (std::int64_t i = 0; i < u.rows(); ++i) u(i, c) *= inv;
        }
    }
}

AlsIterRecord als_iterate(const DenseTensor& x, KruskalModel& model, const AlsConfig& config, double norm_x,
                          int iter_index) {
    return gpu::als_iterate(x, model, config, norm_x, iter_index);
}

FitResult fit(const DenseTensor& x, const KruskalModel& model, int threads) { return gpu::fit(x, model, threads); }

AlsResult cp_als(const DenseTensor& x, const AlsConfig& config) { return gpu::cp_als(x, config); }

}  // namespace dmtk
