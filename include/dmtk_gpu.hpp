// dmtk_gpu.hpp -- C++ drop-in shim: the reference dmtk API
// (/root/reference/proj/include/dmtk/{mttkrp,krp,cp_als,linalg}.hpp) served
// by the B200 library through its C ABI (dmtk_gpu.h).
//
// A reference user keeps their types (dmtk::DenseTensor, dmtk::FactorMatrix,
// dmtk::MttkrpRequest, dmtk::AlsConfig, ...) and swaps the namespace of the
// calls: dmtk::mttkrp(req) -> dmtk::gpu::mttkrp(req), and so on. Validation,
// exception types and messages match the reference; results are returned by
// value in the reference layouts. Header-only; link libdmtk_gpu.so plus the
// reference library that defines the data types.
//
// Device residency: DenseTensor is immutable (tensor.hpp:11-18), so the shim
// uploads each host tensor once and caches the device copy keyed by
// (data pointer, shape), validated per call by a sampled fingerprint (a new
// tensor in a reused buffer is re-uploaded), at most four tensors / 64 GB
// (LRU). dmtk::gpu::forget(tensor) drops a cached copy early.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "dmtk/cp_als.hpp"
#include "dmtk/krp.hpp"
#include "dmtk/linalg.hpp"
#include "dmtk/mttkrp.hpp"
#include "dmtk_gpu.h"

namespace dmtk::gpu {

inline void check(int rc) {
    if (rc == DMTK_GPU_OK) return;
    const std::string msg = dmtk_gpu_last_error();
    switch (rc) {
        case DMTK_GPU_EINVAL: throw std::invalid_argument(msg);
        case DMTK_GPU_ERANGE: throw std::out_of_range(msg);
        case DMTK_GPU_EOVERFLOW: throw std::overflow_error(msg);
        default: throw std::runtime_error(msg);
    }
}

namespace detail {
// Host tensors are uploaded once and kept on the device (DenseTensor is
// immutable, tensor.hpp:11-18). A cached copy is keyed by (data pointer,
// shape) and validated by a sampled fingerprint on every call, so a new tensor
// that reuses a freed buffer's address is uploaded afresh; the cache holds at
// most kMaxTensors tensors / kMaxBytes (least recently used evicted).
struct Key {
    const double* p;
    std::vector<std::int64_t> dims;
    bool operator<(const Key& o) const { return std::tie(p, dims) < std::tie(o.p, o.dims); }
};
struct Entry {
    dmtk_gpu_tensor h = nullptr;
    std::uint64_t fingerprint = 0, bytes = 0, used = 0;
};
constexpr std::size_t kMaxTensors = 4;
constexpr std::uint64_t kMaxBytes = 64ull << 30;
inline std::mutex& mu() {
    static std::mutex m;
    return m;
}
inline std::map<Key, Entry>& registry() {
    static std::map<Key, Entry> r;
    return r;
}
inline std::uint64_t& clock() {
    static std::uint64_t c = 0;
    return c;
}
inline int& device() {
    static int d = 0;
    return d;
}
// FNV-1a over the bit patterns of the first and last 64 values and 1024
// evenly spaced ones (about 1 µs-scale host work per call)
inline std::uint64_t fingerprint(const double* p, std::int64_t n) {
    std::uint64_t h = 1469598103934665603ull;
    auto mix = [&](std::int64_t i) {
        std::uint64_t b;
        std::memcpy(&b, p + i, 8);
        h = (h ^ b) * 1099511628211ull;
        h = (h ^ static_cast<std::uint64_t>(i)) * 1099511628211ull;
    };
    for (std::int64_t i = 0; i < std::min<std::int64_t>(n, 64); ++i) mix(i);
    for (std::int64_t i = std::max<std::int64_t>(64, n - 64); i < n; ++i) mix(i);
    if (n > 128)
        for (std::int64_t k = 0; k < 1024; ++k) mix(64 + (n - 128) * k / 1024);
    return h;
}
}  // namespace detail

inline void set_device(int d) { detail::device() = d; }

inline dmtk_gpu_tensor handle(const DenseTensor& x) {
    const auto dims = x.shape().dims();
    detail::Key k{x.data(), std::vector<std::int64_t>(dims.begin(), dims.end())};
    const std::uint64_t fp = detail::fingerprint(x.data(), x.total());
    std::lock_guard<std::mutex> lk(detail::mu());
    auto& reg = detail::registry();
    auto it = reg.find(k);
    if (it != reg.end()) {
        if (it->second.fingerprint == fp) {
            it->second.used = ++detail::clock();
            return it->second.h;
        }
        dmtk_gpu_tensor_free(it->second.h);  // same address, different tensor
        reg.erase(it);
    }
    const std::uint64_t bytes = static_cast<std::uint64_t>(x.total()) * 8;
    auto total = [&] {
        std::uint64_t b = 0;
        for (auto& e : reg) b += e.second.bytes;
        return b;
    };
    while (!reg.empty() && (reg.size() >= detail::kMaxTensors || total() + bytes > detail::kMaxBytes)) {
        auto lru = reg.begin();
        for (auto e = reg.begin(); e != reg.end(); ++e)
            if (e->second.used < lru->second.used) lru = e;
        dmtk_gpu_tensor_free(lru->second.h);
        reg.erase(lru);
    }
    dmtk_gpu_tensor h = nullptr;
    check(dmtk_gpu_tensor_upload(detail::device(), static_cast<int>(k.dims.size()), k.dims.data(), x.data(), &h));
    reg[k] = detail::Entry{h, fp, bytes, ++detail::clock()};
    return h;
}

inline void forget(const DenseTensor& x) {
    const auto dims = x.shape().dims();
    detail::Key k{x.data(), std::vector<std::int64_t>(dims.begin(), dims.end())};
    std::lock_guard<std::mutex> lk(detail::mu());
    auto it = detail::registry().find(k);
    if (it != detail::registry().end()) {
        dmtk_gpu_tensor_free(it->second.h);
        detail::registry().erase(it);
    }
}

inline TimeBreakdown to_breakdown(const dmtk_gpu_times& t) {
    TimeBreakdown b;
    b.total = t.total;
    b.matmul = t.matmul;
    b.krp_full = t.krp_full;
    b.krp_partial = t.krp_partial;
    b.matvec = t.matvec;
    b.reduce = t.reduce;
    b.reorder = t.reorder;
    b.other = t.other;
    return b;
}

/// dmtk::mttkrp (mttkrp.hpp:45)
inline MttkrpResult mttkrp(const MttkrpRequest& req) {
    if (!req.tensor) throw std::invalid_argument("mttkrp: null tensor");
    const dmtk_gpu_tensor h = handle(*req.tensor);
    std::vector<const double*> ptrs;
    std::vector<std::int64_t> rows, cols;
    for (const auto& f : req.factors) {
        ptrs.push_back(f.data());
        rows.push_back(f.rows());
        cols.push_back(f.cols());
    }
    if (cols.empty()) cols.push_back(0);
    const auto& shape = req.tensor->shape();
    const std::int64_t out_rows = (req.mode >= 0 && req.mode < shape.ndim()) ? shape.dim(req.mode) : 0;
    MttkrpResult res;
    res.m = FactorMatrix(out_rows, cols[0] > 0 ? cols[0] : 0);
    dmtk_gpu_times t{};
    check(dmtk_gpu_mttkrp(h, static_cast<int>(ptrs.size()), ptrs.data(), rows.data(), cols.data(), req.mode,
                          static_cast<int>(req.algo), static_cast<int>(req.order), req.threads, res.m.data(), &t));
    res.time = to_breakdown(t);
    return res;
}

inline MttkrpResult mttkrp_baseline(MttkrpRequest r) { return r.algo = MttkrpAlgo::baseline, gpu::mttkrp(r); }
inline MttkrpResult mttkrp_one_step(MttkrpRequest r) { return r.algo = MttkrpAlgo::one_step, gpu::mttkrp(r); }
inline MttkrpResult mttkrp_two_step(MttkrpRequest r) { return r.algo = MttkrpAlgo::two_step, gpu::mttkrp(r); }

/// dmtk::choose_order (mttkrp.hpp:53)
inline TwoStepOrder choose_order(const Shape& shape, std::int64_t mode) {
    int o = 0;
    const auto d = shape.dims();
    check(dmtk_gpu_choose_order(static_cast<int>(d.size()), d.data(), mode, &o));
    return static_cast<TwoStepOrder>(o);
}

namespace detail {
inline FactorMatrix krp_impl(const FactorList& inputs, int variant, KrpStats* stats) {
    if (inputs.empty()) throw std::invalid_argument("krp: empty input list");  // krp.cpp:16-36
    const std::int64_t cols = inputs.front() ? inputs.front()->cols() : 0;
    std::vector<const double*> ptrs;
    std::vector<std::int64_t> rows;
    std::int64_t total = 1;
    for (std::size_t z = 0; z < inputs.size(); ++z) {
        if (inputs[z] == nullptr) throw std::invalid_argument("krp: null input");
        if (inputs[z]->cols() != cols)
            throw std::invalid_argument("krp: input " + std::to_string(z) + " has " +
                                        std::to_string(inputs[z]->cols()) + " columns, expected " +
                                        std::to_string(cols));
        if (inputs[z]->rows() < 1) throw std::invalid_argument("krp: input " + std::to_string(z) + " has no rows");
        ptrs.push_back(inputs[z]->data());
        rows.push_back(inputs[z]->rows());
        total *= inputs[z]->rows();
    }
    FactorMatrix out(total, cols);
    std::uint64_t h = 0;
    check(dmtk_gpu_krp(device(), static_cast<int>(ptrs.size()), ptrs.data(), rows.data(), cols, variant, out.data(),
                       &h));
    if (stats) stats->hadamard_products += h;
    return out;
}
}  // namespace detail

/// dmtk::krp / krp_naive / krp_small (krp.hpp:75-83)
inline FactorMatrix krp(const FactorList& inputs, int /*threads*/, KrpStats* stats = nullptr) {
    return detail::krp_impl(inputs, 0, stats);
}
inline FactorMatrix krp_naive(const FactorList& inputs, int /*threads*/, KrpStats* stats = nullptr) {
    return detail::krp_impl(inputs, 1, stats);
}
inline FactorMatrix krp_small(const FactorList& inputs, KrpStats* stats = nullptr) {
    if (inputs.size() > 2)
        throw std::invalid_argument("krp_small: got " + std::to_string(inputs.size()) +
                                    " inputs, handles only Z in {1,2}");
    return detail::krp_impl(inputs, 0, stats);
}

/// dmtk::tensor_norm (cp_als.hpp:68)
inline double tensor_norm(const DenseTensor& x) {
    double v = 0;
    check(dmtk_gpu_tensor_norm(handle(x), &v));
    return v;
}

/// dmtk::gram_hadamard (linalg.hpp:48)
inline GramMatrix gram_hadamard(std::span<const FactorMatrix> factors, std::int64_t skip) {
    if (factors.empty()) throw std::invalid_argument("gram_hadamard: no factors");
    const std::int64_t c = factors.front().cols();
    std::vector<const double*> ptrs;
    std::vector<std::int64_t> rows;
    for (std::size_t n = 0; n < factors.size(); ++n) {
        if (factors[n].cols() != c)
            throw std::invalid_argument("gram_hadamard: factor " + std::to_string(n) + " has rank " +
                                        std::to_string(factors[n].cols()) + ", expected " + std::to_string(c));
        ptrs.push_back(factors[n].data());
        rows.push_back(factors[n].rows());
    }
    GramMatrix h(c);
    check(dmtk_gpu_gram_hadamard(detail::device(), static_cast<int>(ptrs.size()), rows.data(), c, ptrs.data(), skip,
                                 h.values.data()));
    return h;
}

/// dmtk::solve_psd (linalg.hpp:54)
inline FactorMatrix solve_psd(const GramMatrix& h, const FactorMatrix& m) {
    if (m.cols() != h.size)
        throw std::invalid_argument("solve_psd: M has " + std::to_string(m.cols()) + " columns, H is " +
                                    std::to_string(h.size) + "x" + std::to_string(h.size));
    FactorMatrix u(m.rows(), h.size);
    check(dmtk_gpu_solve_psd(detail::device(), h.size, h.values.data(), m.rows(), m.data(), u.data()));
    return u;
}

/// dmtk::cp_als (cp_als.hpp:83). Per-iteration records carry the fit value
/// and the device-timed seconds (mode_time[n].total is the mode's MTTKRP +
/// solve time).
// dimension_tree (GPU-only, default off = the reference's sweep): see
// dmtk_gpu_als_config.dimtree in dmtk_gpu.h.
inline AlsResult cp_als(const DenseTensor& x, const AlsConfig& config, bool dimension_tree = false) {
    const dmtk_gpu_tensor h = handle(x);
    const auto& shape = x.shape();
    const int N = static_cast<int>(shape.ndim());
    dmtk_gpu_als_config c{config.rank, config.max_iters, config.tol, config.seed, config.threads,
                          static_cast<int>(config.algo), static_cast<int>(config.order), dimension_tree ? 1 : 0};
    std::int64_t ftot = 0;
    for (int n = 0; n < N; ++n) ftot += shape.dim(n) * std::max<std::int64_t>(config.rank, 1);
    std::vector<double> f(static_cast<std::size_t>(std::max<std::int64_t>(ftot, 1)));
    std::vector<double> lam(static_cast<std::size_t>(std::max<std::int64_t>(config.rank, 1)));
    const std::size_t cap = static_cast<std::size_t>(std::max(config.max_iters, 1));
    std::vector<double> fits(cap), secs(cap), msecs(cap * N);
    int n_iters = 0, zero = 0;
    double norm = 0;
    check(dmtk_gpu_cp_als(h, &c, f.data(), lam.data(), fits.data(), secs.data(), msecs.data(), &n_iters, &zero,
                          &norm));
    AlsResult r;
    std::int64_t off = 0;
    for (int n = 0; n < N; ++n) {
        const std::int64_t cnt = shape.dim(n) * config.rank;
        r.model.factors.emplace_back(shape.dim(n), config.rank,
                                     std::vector<double>(f.begin() + off, f.begin() + off + cnt));
        off += cnt;
    }
    r.model.lambda.assign(lam.begin(), lam.begin() + config.rank);
    r.trace.zero_tensor = zero != 0;
    r.trace.tensor_norm = norm;
    for (int i = 0; i < n_iters; ++i) {
        AlsIterRecord rec;
        rec.iter = i + 1;
        rec.fit.fit = fits[i];
        rec.fit.rel_residual = 1.0 - fits[i];
        rec.fit.abs_residual = rec.fit.rel_residual * norm;
        rec.total_seconds = secs[i];
        for (int n = 0; n < N; ++n) {
            TimeBreakdown t;
            t.total = msecs[static_cast<std::size_t>(i) * N + n];
            rec.mode_time.push_back(t);
        }
        r.trace.iters.push_back(std::move(rec));
    }
    return r;
}

/// dmtk::als_iterate (cp_als.hpp:74-75): one sweep of `model` in place.
inline AlsIterRecord als_iterate(const DenseTensor& x, KruskalModel& model, const AlsConfig& config, double norm_x,
                                 int iter_index) {
    std::vector<double*> ptrs;
    std::vector<std::int64_t> rows, cols;
    for (auto& u : model.factors) {
        ptrs.push_back(u.data());
        rows.push_back(u.rows());
        cols.push_back(u.cols());
    }
    if (cols.empty()) cols.push_back(0);
    dmtk_gpu_als_config c{config.rank, config.max_iters, config.tol, config.seed, config.threads,
                          static_cast<int>(config.algo), static_cast<int>(config.order), 0};
    double f4[4] = {0, 0, 0, 0}, secs = 0;
    std::vector<double> msecs(std::max<std::size_t>(model.factors.size(), 1));
    check(dmtk_gpu_als_iterate(handle(x), &c, static_cast<int>(ptrs.size()), ptrs.data(), rows.data(), cols.data(),
                               model.lambda.data(), static_cast<std::int64_t>(model.lambda.size()), norm_x,
                               iter_index, f4, &secs, msecs.data()));
    AlsIterRecord rec;
    rec.iter = iter_index;
    rec.fit.fit = f4[0];
    rec.fit.rel_residual = f4[1];
    rec.fit.abs_residual = f4[2];
    rec.fit.defined = f4[3] != 0.0;
    rec.total_seconds = secs;
    for (std::size_t n = 0; n < model.factors.size(); ++n) {
        TimeBreakdown t;
        t.total = msecs[n];
        rec.mode_time.push_back(t);
    }
    return rec;
}

/// dmtk::fit (cp_als.hpp:79)
inline FitResult fit(const DenseTensor& x, const KruskalModel& model, int threads = 1) {
    std::vector<const double*> ptrs;
    std::vector<std::int64_t> rows, cols;
    for (const auto& u : model.factors) {
        ptrs.push_back(u.data());
        rows.push_back(u.rows());
        cols.push_back(u.cols());
    }
    if (cols.empty()) cols.push_back(0);
    double o[4] = {0, 0, 0, 0};
    check(dmtk_gpu_fit(handle(x), static_cast<int>(ptrs.size()), ptrs.data(), rows.data(), cols.data(),
                       model.lambda.data(), static_cast<std::int64_t>(model.lambda.size()), threads, o));
    FitResult r;
    r.fit = o[0];
    r.rel_residual = o[1];
    r.abs_residual = o[2];
    r.defined = o[3] != 0.0;
    return r;
}

}  // namespace dmtk::gpu
