// relink_driver.cpp -- a program written against the UNMODIFIED reference API
// only (proj/include/dmtk/*.hpp: dmtk::mttkrp, krp, KrpState, cp_als,
// als_iterate, fit, the bench harness with its --check gate). It is built
// twice from this one source (tests/cpp/Makefile):
//   relink_ref  linked with the reference library (oracle/_ref/libdmtk_ref.so)
//   relink_gpu  linked with libdmtk_dropin.so (the B200 path) + the reference's
//               remaining objects (oracle/_ref/libdmtk_rest.so: shape, tensor,
//               matrix, linalg, parallel, kernels, tensor_io, bench, oracle)
// and tests/test_gpu_dropin.py compares the two outputs line by line
// (MTTKRP <= 1e-12 relative Frobenius, KRP / KrpState / generators bitwise,
// fits <= 1e-9, identical exception types and messages). Inside relink_gpu the
// reference's own bench_mttkrp / bench_krp (bench.cpp:241-394) call the GPU
// through the relinked symbols and apply their own --check against the
// exhaustive oracle.
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "dmtk/bench.hpp"
#include "dmtk/cp_als.hpp"
#include "dmtk/krp.hpp"
#include "dmtk/mttkrp.hpp"

using namespace dmtk;

static void print_mat(const char* key, const FactorMatrix& m) {
    std::printf("MAT %s %" PRId64 " %" PRId64, key, m.rows(), m.cols());
    for (double v : m.values()) std::printf(" %.17g", v);
    std::printf("\n");
}

static void print_bits(const char* key, std::span<const double> v) {
    std::printf("BITS %s", key);
    for (double x : v) {
        std::uint64_t b;
        std::memcpy(&b, &x, 8);
        std::printf(" %016" PRIx64, b);
    }
    std::printf("\n");
}

template <class F>
static void expect_error(const char* key, F&& f) {
    try {
        f();
        std::printf("ERR %s none\n", key);
    } catch (const std::out_of_range& e) {
        std::printf("ERR %s out_of_range %s\n", key, e.what());
    } catch (const std::invalid_argument& e) {
        std::printf("ERR %s invalid_argument %s\n", key, e.what());
    } catch (const std::exception& e) {
        std::printf("ERR %s exception %s\n", key, e.what());
    }
}

static const char* algo_s(MttkrpAlgo a) {
    switch (a) {
        case MttkrpAlgo::baseline: return "baseline";
        case MttkrpAlgo::one_step: return "one_step";
        case MttkrpAlgo::two_step: return "two_step";
        default: return "automatic";
    }
}

int main() {
    // ---- MTTKRP sweep (test_mttkrp.cpp:120-151 shapes), every algorithm / order / mode
    const std::vector<std::vector<std::int64_t>> shapes = {{3, 4, 5}, {2, 3, 4, 2}, {2, 2, 2, 2, 2}, {4, 1, 3},
                                                           {6, 7},    {9},          {30, 25, 20}, {12, 10, 9, 8}};
    for (std::size_t si = 0; si < shapes.size(); ++si) {
        const Shape shape(shapes[si]);
        const DenseTensor x = bench::gen_tensor(shape, 17 + si);
        for (std::int64_t rank : {1, 2, 5, 25}) {
            const auto f = bench::gen_factors(shape, rank, 23);
            for (std::int64_t mode = 0; mode < shape.ndim(); ++mode) {
                const bool boundary = mode == 0 || mode == shape.ndim() - 1;
                for (MttkrpAlgo a : {MttkrpAlgo::baseline, MttkrpAlgo::one_step, MttkrpAlgo::two_step,
                                     MttkrpAlgo::automatic}) {
                    if (a == MttkrpAlgo::two_step && boundary) continue;
                    for (TwoStepOrder o : {TwoStepOrder::automatic, TwoStepOrder::left, TwoStepOrder::right}) {
                        if (o != TwoStepOrder::automatic && a != MttkrpAlgo::two_step) continue;
                        MttkrpRequest req;
                        req.tensor = &x;
                        req.factors = f;
                        req.mode = mode;
                        req.algo = a;
                        req.order = o;
                        req.threads = 2;
                        char key[128];
                        std::snprintf(key, sizeof key, "mttkrp_s%zu_r%" PRId64 "_m%" PRId64 "_%s_o%d", si, rank, mode,
                                      algo_s(a), static_cast<int>(o));
                        print_mat(key, mttkrp(req).m);
                    }
                }
                MttkrpRequest req;
                req.tensor = &x;
                req.factors = f;
                req.mode = mode;
                char key[96];
                std::snprintf(key, sizeof key, "onestep_s%zu_r%" PRId64 "_m%" PRId64, si, rank, mode);
                print_mat(key, mttkrp_one_step(req).m);
                if (!boundary) {
                    std::snprintf(key, sizeof key, "twostep_s%zu_r%" PRId64 "_m%" PRId64, si, rank, mode);
                    print_mat(key, mttkrp_two_step(req).m);
                    std::snprintf(key, sizeof key, "baseline_s%zu_r%" PRId64 "_m%" PRId64, si, rank, mode);
                    print_mat(key, mttkrp_baseline(req).m);
                }
                std::printf("ORDER s%zu_m%" PRId64 " %d\n", si, mode, static_cast<int>(choose_order(shape, mode)));
            }
        }
    }
    // ---- validation: exception types and messages (mttkrp.cpp:20-46, 317-321)
    {
        const Shape shape({3, 4, 5});
        const DenseTensor x = bench::gen_tensor(shape, 1);
        const auto f = bench::gen_factors(shape, 3, 2);
        MttkrpRequest req;
        req.tensor = &x;
        req.factors = f;
        expect_error("null_tensor", [&] {
            MttkrpRequest r = req;
            r.tensor = nullptr;
            mttkrp(r);
        });
        expect_error("mode_range", [&] {
            MttkrpRequest r = req;
            r.mode = 3;
            mttkrp(r);
        });
        expect_error("factor_count", [&] {
            MttkrpRequest r = req;
            r.factors = std::span<const FactorMatrix>(f.data(), 2);
            mttkrp(r);
        });
        expect_error("threads", [&] {
            MttkrpRequest r = req;
            r.threads = 0;
            mttkrp(r);
        });
        expect_error("two_step_boundary", [&] {
            MttkrpRequest r = req;
            r.mode = 0;
            mttkrp_two_step(r);
        });
        expect_error("krp_empty", [&] { krp(FactorList{}, 1); });
        expect_error("krp_small_z3", [&] {
            const auto g = bench::gen_factors(Shape({2, 3, 4}), 2, 5);
            krp_small(FactorList{&g[0], &g[1], &g[2]});
        });
        expect_error("cp_rank", [&] {
            AlsConfig c;
            c.rank = 0;
            cp_als(x, c);
        });
    }
    // ---- KRP: bitwise, hadamard counts (test_krp.cpp:69-155)
    const std::vector<std::vector<std::int64_t>> kshapes = {{6}, {3, 4}, {2, 3, 4}, {3, 2, 2, 3}, {2, 2, 3, 2, 2},
                                                            {4, 1, 3}, {1, 1, 5}};
    for (std::size_t si = 0; si < kshapes.size(); ++si) {
        for (std::int64_t rank : {1, 3, 25}) {
            const auto g = bench::gen_factors(Shape(kshapes[si]), rank, 31 + si);
            FactorList in;
            for (const auto& m : g) in.push_back(&m);
            KrpStats s1, s2;
            char key[64];
            std::snprintf(key, sizeof key, "krp_s%zu_r%" PRId64, si, rank);
            print_bits(key, krp(in, 1, &s1).values());
            std::snprintf(key, sizeof key, "krpnaive_s%zu_r%" PRId64, si, rank);
            print_bits(key, krp_naive(in, 1, &s2).values());
            std::printf("COUNT krp_s%zu_r%" PRId64 " %" PRIu64 " %" PRIu64 "\n", si, rank, s1.hadamard_products,
                        s2.hadamard_products);
            if (in.size() <= 2) {
                std::snprintf(key, sizeof key, "krpsmall_s%zu_r%" PRId64, si, rank);
                print_bits(key, krp_small(in).values());
            } else {  // the row iterator: sequential, seek, counts (test_krp.cpp:93-128)
                KrpState st(in, 0);
                std::vector<double> row(static_cast<std::size_t>(rank));
                const std::int64_t rows = st.rows();
                for (std::int64_t j = 0; j < rows; ++j) {
                    krp_row(st, row);
                    std::snprintf(key, sizeof key, "state_s%zu_r%" PRId64 "_j%" PRId64, si, rank, j);
                    print_bits(key, row);
                    if (j + 1 < rows) st.advance();
                }
                std::printf("COUNT state_s%zu_r%" PRId64 " %" PRIu64 "\n", si, rank, st.hadamard_count());
                KrpState sk(in, rows / 2);
                sk.seek(rows - 1);
                sk.write_row(row);
                std::snprintf(key, sizeof key, "seek_s%zu_r%" PRId64, si, rank);
                print_bits(key, row);
                std::printf("COUNT seek_s%zu_r%" PRId64 " %" PRIu64 " %" PRId64 "\n", si, rank, sk.hadamard_count(),
                            sk.row_index());
            }
        }
    }
    // ---- CP-ALS (cp_als.cpp:87-200): random model, normalize, sweeps, fit
    {
        const Shape shape({9, 8, 7, 6});
        const DenseTensor x = bench::gen_tensor(shape, 41);
        KruskalModel m = KruskalModel::random(shape, 4, 5);
        for (std::size_t n = 0; n < m.factors.size(); ++n) {
            char key[32];
            std::snprintf(key, sizeof key, "random_f%zu", n);
            print_bits(key, m.factors[n].values());
        }
        KruskalModel mn = m;
        mn.normalize_mode(2);
        print_mat("normalized_f2", mn.factors[2]);
        std::printf("VEC lambda_norm2");
        for (double v : mn.lambda) std::printf(" %.17g", v);
        std::printf("\n");
        const double nx = tensor_norm(x);
        std::printf("SCALAR tensor_norm %.17g\n", nx);
        const FitResult f0 = fit(x, m, 2);
        std::printf("SCALAR fit_random %.17g\n", f0.fit);
        AlsConfig cfg;
        cfg.rank = 4;
        cfg.max_iters = 8;
        cfg.tol = 0.0;
        cfg.seed = 5;
        cfg.threads = 2;
        for (int it = 1; it <= 3; ++it) {
            const AlsIterRecord r = als_iterate(x, m, cfg, nx, it);
            std::printf("SCALAR als_iterate_%d %.17g\n", it, r.fit.fit);
        }
        print_mat("als_iterate_f0", m.factors[0]);
        for (MttkrpAlgo a : {MttkrpAlgo::automatic, MttkrpAlgo::one_step, MttkrpAlgo::baseline}) {
            cfg.algo = a;
            const AlsResult r = cp_als(x, cfg);
            for (std::size_t i = 0; i < r.trace.iters.size(); ++i)
                std::printf("SCALAR cp_%s_it%zu %.17g\n", algo_s(a), i, r.trace.iters[i].fit.fit);
            std::printf("SCALAR cp_%s_norm %.17g\n", algo_s(a), r.trace.tensor_norm);
            print_mat((std::string("cp_") + algo_s(a) + "_f3").c_str(), r.model.factors[3]);
        }
        cfg.algo = MttkrpAlgo::automatic;
        cfg.tol = 1e-3;
        cfg.max_iters = 50;
        std::printf("SCALAR cp_tol_iters %zu\n", cp_als(x, cfg).trace.iters.size());
        const DenseTensor z(Shape({3, 4, 2}), std::vector<double>(24, 0.0));
        const AlsResult rz = cp_als(z, cfg);
        std::printf("SCALAR cp_zero %d %zu\n", rz.trace.zero_tensor ? 1 : 0, rz.trace.iters.size());
    }
    // ---- the reference's own harness with its --check gate (bench.cpp:241-394)
    {
        bench::MttkrpBenchArgs a;
        a.shape = Shape({40, 30, 20});
        a.rank = 16;
        a.trials = 2;
        a.check = true;
        a.seed = 3;
        for (MttkrpAlgo al : {MttkrpAlgo::one_step, MttkrpAlgo::two_step, MttkrpAlgo::automatic}) {
            a.algo = al;
            const auto rows = bench::bench_mttkrp(a);
            for (const auto& r : rows)
                std::printf("HARNESS mttkrp_%s_mode%s checked=%s\n", algo_s(al), r.mode.c_str(), r.checked.c_str());
        }
        bench::KrpBenchArgs k;
        k.dims = {20, 15, 10};
        k.rank = 16;
        k.trials = 2;
        k.check = true;
        for (const auto& r : bench::bench_krp(k))
            std::printf("HARNESS krp_%s checked=%s\n", r.algo.c_str(), r.checked.c_str());
        bench::CpBenchArgs c;
        c.shape = Shape({12, 10, 8});
        c.ranks = {3};
        c.iters = 4;
        c.seed = 9;
        for (const auto& r : bench::bench_cp(c))
            if (r.mode == "all") std::printf("HARNESSFIT cp_it%d %s\n", r.iter, r.fit.c_str());
    }
    std::printf("DONE\n");
    return 0;
}
