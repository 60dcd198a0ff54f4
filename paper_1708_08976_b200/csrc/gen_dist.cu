// gen_dist.cu -- value transforms of the seeded generator for the BASELINE
// configs that are not U[0,1) (BASELINE.json configs 3-5; SURVEY.md 8d,
// BASELINE.md 3): U[-1,1), N(0,1) by Box-Muller, and the fMRI-shaped
// symmetric slices with tanh(N(0, 0.3^2)) off-diagonals. The uniforms come
// from mt64_generate (the reference's gen_tensor stream, bench.cpp:88-97).
//
// Every operation is an explicitly rounded IEEE-754 add / sub / mul / div /
// sqrt (__dadd_rn & co. are never contracted into FMAs), in the same order as
// the test-side restatement (oracle/oracle.c, compiled -ffp-contract=off), so
// host and device produce identical bytes for a seed: the reference library
// can be fed exactly what the GPU streams.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace dmtkg {
namespace {

#define FA(a, b) __dadd_rn((a), (b))
#define FS(a, b) __dsub_rn((a), (b))
#define FM(a, b) __dmul_rn((a), (b))
#define FD(a, b) __ddiv_rn((a), (b))

__constant__ double c_log[11] = {0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3,
                                 0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4,
                                 0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5, 0x1.af286bca1af28p-5,
                                 0x1.8618618618618p-5, 0x1.642c8590b2164p-5};
__constant__ double c_cos[10] = {-0x1.0000000000000p-1, 0x1.5555555555555p-5, -0x1.6c16c16c16c17p-10,
                                 0x1.a01a01a01a01ap-16, -0x1.27e4fb7789f5cp-22, 0x1.1eed8eff8d898p-29,
                                 -0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-45, -0x1.6827863b97d97p-53,
                                 0x1.e542ba4020225p-62};
__constant__ double c_sin[10] = {-0x1.5555555555555p-3, 0x1.1111111111111p-7, -0x1.a01a01a01a01ap-13,
                                 0x1.71de3a556c734p-19, -0x1.ae64567f544e4p-26, 0x1.6124613a86d09p-33,
                                 -0x1.ae7f3e733b81fp-41, 0x1.952c77030ad4ap-49, -0x1.2f49b46814157p-57,
                                 0x1.71b8ef6dcf572p-66};
__constant__ double c_exp[15] = {0x1.0000000000000p-1, 0x1.5555555555555p-3, 0x1.5555555555555p-5,
                                 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
                                 0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22,
                                 0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33,
                                 0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-41, 0x1.ae7f3e733b81fp-45};

constexpr double kLn2Hi = 0x1.62e42fee00000p-1;
constexpr double kLn2Lo = 0x1.a39ef35793c76p-33;

// log(x), x > 0 normal: x = m 2^e, m in [sqrt(1/2), sqrt(2)), log m = 2 atanh(s)
__device__ double p_log(double x) {
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    int e = static_cast<int>((b >> 52) & 0x7ff) - 1023;
    b = (b & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL;
    double m = __longlong_as_double(static_cast<long long>(b));
    if (m > 0x1.6a09e667f3bcdp+0) {
        m = FM(m, 0.5);
        e += 1;
    }
    const double s = FD(FS(m, 1.0), FA(m, 1.0));
    const double s2 = FM(s, s);
    double p = c_log[10];
#pragma unroll
    for (int k = 9; k >= 0; --k) p = FA(FM(p, s2), c_log[k]);
    p = FA(FM(p, s2), 1.0);
    const double r = FM(FM(2.0, s), p);
    const double de = static_cast<double>(e);
    return FA(FM(de, kLn2Hi), FA(FM(de, kLn2Lo), r));
}

__device__ void p_sincos_2pi(double u, double* sn, double* cs) {
    const double t = FM(4.0, u);
    const double q = floor(t);
    const double r = FS(t, q);
    const bool swap = r > 0.5;
    const double rr = swap ? FS(1.0, r) : r;
    const double x = FM(rr, 0x1.921fb54442d18p+0);
    const double x2 = FM(x, x);
    double ps = c_sin[9], pc = c_cos[9];
#pragma unroll
    for (int k = 8; k >= 0; --k) {
        ps = FA(FM(ps, x2), c_sin[k]);
        pc = FA(FM(pc, x2), c_cos[k]);
    }
    double sx = FA(x, FM(x, FM(x2, ps)));
    double cx = FA(1.0, FM(x2, pc));
    if (swap) {
        const double tmp = sx;
        sx = cx;
        cx = tmp;
    }
    switch (static_cast<int>(q)) {
        case 0: *sn = sx; *cs = cx; break;
        case 1: *sn = cx; *cs = -sx; break;
        case 2: *sn = -sx; *cs = -cx; break;
        default: *sn = -cx; *cs = sx; break;
    }
}

__device__ double p_exp(double x) {  // x <= 0, result normal
    const double k = floor(FA(FM(x, 0x1.71547652b82fep+0), 0.5));
    const double r = FS(FS(x, FM(k, kLn2Hi)), FM(k, kLn2Lo));
    double p = c_exp[14];
#pragma unroll
    for (int i = 13; i >= 0; --i) p = FA(FM(p, r), c_exp[i]);
    p = FA(FM(FA(FM(p, r), 1.0), r), 1.0);
    const double sc = __longlong_as_double(static_cast<long long>(static_cast<unsigned long long>(
                                                                     static_cast<long long>(k) + 1023)
                                                                 << 52));
    return FM(p, sc);
}

__device__ double p_tanh(double y) {
    const double a = y < 0.0 ? -y : y;
    const double e = p_exp(FM(-2.0, a));
    const double t = FD(FS(1.0, e), FA(1.0, e));
    return y < 0.0 ? -t : t;
}

__device__ double box_muller(double u0, double u1, bool second) {
    const double rad = __dsqrt_rn(FM(-2.0, p_log(FS(1.0, u0))));
    double sn, cs;
    p_sincos_2pi(u1, &sn, &cs);
    return second ? FM(rad, sn) : FM(rad, cs);
}

// dst[(e / d0) * pd0 + e % d0] = value e of `dist` (natural order)
__global__ void __launch_bounds__(256) gen_dist_kernel(const double* __restrict__ u, long long total, int dist,
                                                       long long I, long long P, long long d0, long long pd0,
                                                       double* __restrict__ dst) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
        double v;
        if (dist == 2) {
            v = FS(FM(2.0, u[e]), 1.0);
        } else if (dist == 3) {
            const long long k = e >> 1;
            v = box_muller(u[2 * k], u[2 * k + 1], (e & 1) != 0);
        } else {  // symmetric slices (I, I, rest)
            const long long i = e % I, j = (e / I) % I, q = e / (I * I);
            if (i == j) {
                v = 1.0;
            } else {
                const long long a = i < j ? i : j, b = i < j ? j : i;
                const long long m = q * P + b * (b - 1) / 2 + a;
                const long long k = m >> 1;
                v = p_tanh(FM(0x1.3333333333333p-2, box_muller(u[2 * k], u[2 * k + 1], (m & 1) != 0)));
            }
        }
        dst[(e / d0) * pd0 + e % d0] = v;
    }
}

}  // namespace

long long gen_dist_uniforms(int dist, long long total, long long I) {
    if (dist == 3) return total + (total & 1);
    if (dist == 4) {
        const long long P = I * (I - 1) / 2, R = total / (I * I);
        return P * R + ((P * R) & 1);
    }
    return total;
}

void launch_gen_dist(const double* u, long long total, int dist, long long I, long long d0, long long pd0,
                     double* dst, int nsm, cudaStream_t s) {
    if (total <= 0) return;
    const long long want = (total + 255) / 256;
    const int blocks = static_cast<int>(want < 8LL * nsm ? want : 8LL * nsm);
    gen_dist_kernel<<<blocks, 256, 0, s>>>(u, total, dist, I, I * (I - 1) / 2, d0, pd0, dst);
}

}  // namespace dmtkg
