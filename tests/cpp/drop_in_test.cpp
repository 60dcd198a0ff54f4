// drop_in_test.cpp -- the reference test strategy (proj/tests/test_mttkrp.cpp,
// test_krp.cpp, test_cpals.cpp) replayed through the C++ drop-in shim
// include/dmtk_gpu.hpp: same reference types, calls moved from dmtk:: to
// dmtk::gpu::, results checked against the unmodified reference library.
// Exit code 0 = all checks passed. Needs a B200.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "dmtk/oracle.hpp"
#include "dmtk_gpu.hpp"

using namespace dmtk;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (cond) {                                                              \
            ++g_pass;                                                            \
        } else {                                                                 \
            ++g_fail;                                                            \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
        }                                                                        \
    } while (0)
template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static double frand(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

static DenseTensor random_tensor(const Shape& s, std::uint64_t seed) {
    std::mt19937_64 g(seed);
    std::vector<double> v(static_cast<std::size_t>(s.total()));
    for (auto& x : v) x = frand(g);
    return DenseTensor(s, std::move(v));
}

static std::vector<FactorMatrix> random_factors(const Shape& s, std::int64_t rank, std::uint64_t seed) {
    std::mt19937_64 g(seed);
    std::vector<FactorMatrix> out;
    for (std::int64_t n = 0; n < s.ndim(); ++n) {
        FactorMatrix m(s.dim(n), rank);
        for (auto& v : m.values()) v = frand(g);
        out.push_back(std::move(m));
    }
    return out;
}

static double rel(const FactorMatrix& a, const FactorMatrix& b) {
    double d = 0, r = 0;
    for (std::size_t i = 0; i < a.values().size(); ++i) {
        const double e = a.values()[i] - b.values()[i];
        d += e * e;
        r += b.values()[i] * b.values()[i];
    }
    return r == 0 ? std::sqrt(d) : std::sqrt(d / r);
}

static MttkrpRequest req(const DenseTensor& x, const std::vector<FactorMatrix>& f, std::int64_t mode, MttkrpAlgo a,
                         TwoStepOrder o = TwoStepOrder::automatic, int threads = 1) {
    MttkrpRequest r;
    r.tensor = &x;
    r.factors = f;
    r.mode = mode;
    r.algo = a;
    r.order = o;
    r.threads = threads;
    return r;
}

int main() {
    // test_mttkrp.cpp:120-151 -- every algorithm agrees with the exhaustive sum
    for (auto dims : std::vector<std::vector<std::int64_t>>{{3, 4, 5}, {2, 3, 4, 2}, {2, 2, 2, 2, 2}, {4, 1, 3},
                                                             {6, 7}, {9}, {40, 30, 20}, {12, 10, 8, 6}}) {
        const Shape s(dims);
        const DenseTensor x = random_tensor(s, 17);
        for (std::int64_t rank : {1, 2, 5, 25}) {
            const auto f = random_factors(s, rank, 23);
            for (std::int64_t mode = 0; mode < s.ndim(); ++mode) {
                const FactorMatrix want = oracle::mttkrp_loops(x, f, mode, s.total());
                for (MttkrpAlgo a : {MttkrpAlgo::baseline, MttkrpAlgo::one_step, MttkrpAlgo::automatic})
                    CHECK(rel(gpu::mttkrp(req(x, f, mode, a)).m, want) <= 1e-12);
                if (mode > 0 && mode + 1 < s.ndim())
                    for (TwoStepOrder o : {TwoStepOrder::left, TwoStepOrder::right})
                        CHECK(rel(gpu::mttkrp(req(x, f, mode, MttkrpAlgo::two_step, o)).m, want) <= 1e-12);
                // and the reference's own fast path on the same bytes
                CHECK(rel(gpu::mttkrp(req(x, f, mode, MttkrpAlgo::automatic)).m,
                          mttkrp(req(x, f, mode, MttkrpAlgo::automatic, TwoStepOrder::automatic, 4)).m) <= 1e-12);
            }
        }
        gpu::forget(x);  // the buffer is freed at scope exit (pointer-keyed device cache)
    }
    // frozen case, test_mttkrp.cpp:99-118
    {
        const Shape s({2, 3, 2});
        std::vector<double> v(12);
        for (int i = 0; i < 12; ++i) v[i] = i;
        const DenseTensor x(s, v);
        std::vector<FactorMatrix> f;
        f.emplace_back(2, 2);
        f.emplace_back(3, 2, std::vector<double>{1, 0, 0, 1, 0, 0});
        f.emplace_back(2, 2, std::vector<double>{1, 1, 1, 1});
        const auto m = gpu::mttkrp(req(x, f, 0, MttkrpAlgo::one_step)).m;
        CHECK(m(0, 0) == 6.0 && m(0, 1) == 10.0 && m(1, 0) == 8.0 && m(1, 1) == 12.0);
        gpu::forget(x);
    }
    // validation, test_mttkrp.cpp:160-173, 276-306
    {
        const Shape s({3, 4, 5});
        const DenseTensor x = random_tensor(s, 2);
        const auto f = random_factors(s, 2, 3);
        CHECK(throws<std::invalid_argument>([&] { gpu::mttkrp(req(x, f, 0, MttkrpAlgo::two_step)); }));
        CHECK(throws<std::out_of_range>([&] { gpu::mttkrp(req(x, f, 3, MttkrpAlgo::one_step)); }));
        MttkrpRequest r = req(x, f, 0, MttkrpAlgo::one_step);
        r.threads = 0;
        CHECK(throws<std::invalid_argument>([&] { gpu::mttkrp(r); }));
        r.tensor = nullptr;
        r.threads = 1;
        CHECK(throws<std::invalid_argument>([&] { gpu::mttkrp(r); }));
        gpu::forget(x);
    }
    // KRP bitwise vs the Kronecker oracle, test_krp.cpp:69-81, and counts :108-128
    for (auto dims : std::vector<std::vector<std::int64_t>>{{6}, {3, 4}, {2, 3, 4}, {3, 2, 2, 3}, {2, 2, 3, 2, 2},
                                                             {4, 1, 3}, {1, 1, 5}}) {
        for (std::int64_t cols : {1, 3, 25}) {
            std::vector<FactorMatrix> mats;
            for (std::size_t z = 0; z < dims.size(); ++z) {
                std::mt19937_64 g(42 + z * 1000);
                FactorMatrix m(dims[z], cols);
                for (auto& v : m.values()) v = frand(g);
                mats.push_back(std::move(m));
            }
            FactorList in;
            for (auto& m : mats) in.push_back(&m);
            CHECK(gpu::krp(in, 1) == oracle::krp_kron(in));
            CHECK(gpu::krp_naive(in, 1) == oracle::krp_kron(in));
        }
    }
    {
        std::vector<FactorMatrix> m3;
        for (int z = 0; z < 3; ++z) m3.emplace_back(2, 4, std::vector<double>(8, 1.5));
        FactorList in{&m3[0], &m3[1], &m3[2]};
        KrpStats st, nv;
        gpu::krp(in, 1, &st);
        gpu::krp_naive(in, 1, &nv);
        CHECK(st.hadamard_products == 12);
        CHECK(nv.hadamard_products == 16);
    }
    // CP-ALS: same fits as the reference after the same iterations (<= 1e-9)
    {
        const Shape s({7, 6, 5});
        const DenseTensor x = random_tensor(s, 10);
        AlsConfig c;
        c.rank = 3;
        c.max_iters = 8;
        c.tol = 0.0;
        c.seed = 42;
        const AlsResult a = gpu::cp_als(x, c);
        const AlsResult b = cp_als(x, c);
        CHECK(a.trace.iters.size() == b.trace.iters.size());
        for (std::size_t i = 0; i < a.trace.iters.size(); ++i)
            CHECK(std::fabs(a.trace.iters[i].fit.fit - b.trace.iters[i].fit.fit) <= 1e-9);
        const FitResult fa = gpu::fit(x, a.model);
        const FitResult fb = fit(x, b.model, 1);
        CHECK(std::fabs(fa.fit - fb.fit) <= 1e-9);
        CHECK(std::fabs(gpu::tensor_norm(x) - tensor_norm(x)) <= 1e-12 * tensor_norm(x));
    }
    std::printf("drop_in_test: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
