// On-device seeded tensor generation, bitwise equal to the reference's
// gen_tensor (bench.cpp:88-97: one std::mt19937_64(seed) stream, value k =
// (draw_k >> 11) * 2^-53, bench.cpp:22-24) — SURVEY §8f-3, so the 8 GB
// BASELINE configs need no host-side generation (~8 s for 1e9 draws).
//
// The stream is split into P contiguous chunks, one CTA each. A CTA jumps
// the generator to its chunk start and then runs the twist recurrence
//   x_{k+312} = x_{k+156} ^ twist(x_k, x_{k+1})        (draw j = temper(x_{312+j}))
// 156 words per step (every word of a step depends only on the previous
// two 156-word blocks), tempering and storing each word as it retires.
//
// Jump-ahead (the characteristic-polynomial method): the raw words satisfy
// the linear recurrence of the generator's characteristic polynomial phi
// (degree 19937, found once per process by Berlekamp-Massey on one bit of the
// raw sequence). With r(x) = x^J mod phi = sum_i r_i x^i,
//   x_{k+J} = XOR_{i : r_i = 1} x_{k+i}        for every k >= 1,
// so a CTA forms its 312-word window from the first ~20 250 raw words of the
// stream (host-computed, shared by all CTAs, staged in shared memory) and its
// 312-word coefficient vector r_p (host GF(2) polynomial arithmetic).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "kernels.h"

namespace dmtkg {
namespace {

constexpr int kNN = 312, kMM = 156;
constexpr uint64_t kMatA = 0xB5026F5AA96619E9ULL;
constexpr uint64_t kUM = 0xFFFFFFFF80000000ULL, kLM = 0x7FFFFFFFULL;
constexpr int kDeg = 19937;                        // degree of phi
constexpr int kPW = (kDeg + 63) / 64;              // 312 words per reduced polynomial
constexpr int kRaw = kDeg + kNN;                    // raw words x_1 .. x_kRaw staged per CTA
using Poly = std::vector<uint64_t>;

__host__ __device__ inline uint64_t mt_twist(uint64_t x0, uint64_t x1, uint64_t xm) {
    const uint64_t y = (x0 & kUM) | (x1 & kLM);
    return xm ^ (y >> 1) ^ ((y & 1ULL) ? kMatA : 0ULL);
}

__device__ inline double mt_value(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    // (y >> 11) * 2^-53 built from integer ops (exact: m < 2^53), keeping the
    // FP64 pipe's ~100-cycle conversion and multiply latency off each step
    const uint64_t m = y >> 11;
    if (m == 0) return 0.0;
    const int e = 63 - __clzll(static_cast<long long>(m));  // 0..52
    return __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(e + 970) << 52) |
                                                       ((m << (52 - e)) & 0xFFFFFFFFFFFFFULL)));
}

// raw words x_0 .. x_{count-1} of mt19937_64(seed) (x_0..x_311 = the seeded state)
std::vector<uint64_t> raw_words(uint64_t seed, int count) {
    std::vector<uint64_t> x(static_cast<size_t>(std::max(count, kNN)));
    x[0] = seed;
    for (int i = 1; i < kNN; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
    for (int k = kNN; k < count; ++k) x[k] = mt_twist(x[k - kNN], x[k - kNN + 1], x[k - kMM]);
    x.resize(static_cast<size_t>(count));
    return x;
}

inline int bit(const Poly& p, long i) { return static_cast<int>((p[i >> 6] >> (i & 63)) & 1ULL); }

// p ^= q << sh (bits), p long enough
void xor_shifted(Poly& p, const Poly& q, long sh) {
    const long w = sh >> 6;
    const int b = static_cast<int>(sh & 63);
    for (size_t i = 0; i < q.size(); ++i) {
        if (!q[i]) continue;
        p[i + w] ^= q[i] << b;
        if (b && i + w + 1 < p.size()) p[i + w + 1] ^= q[i] >> (64 - b);
    }
}

// Characteristic polynomial of the generator: Berlekamp-Massey over bit 0 of
// the raw words x_1, x_2, ... (phi is primitive, so any nonzero bit sequence
// of the state has it as its minimal polynomial). Returns phi with bit i the
// coefficient of x^i.
Poly find_phi() {
    const int n = 2 * kDeg + 64;
    const auto x = raw_words(5489ULL, n + 1);
    std::vector<uint8_t> s(static_cast<size_t>(n));
    for (int j = 0; j < n; ++j) s[j] = static_cast<uint8_t>(x[j + 1] & 1ULL);
    // connection polynomial C (C_0 = 1): s_t = XOR_{i=1..L} C_i s_{t-i}
    const int W = (n + 64) / 64 + 1;
    Poly C(W, 0), B(W, 0), T;
    C[0] = B[0] = 1;
    int L = 0, m = 1;
    // rs = s reversed into words, so the window (s_{t-i})_{i>=0} is a bit slice
    Poly rs(W + 1, 0);
    for (int j = 0; j < n; ++j)
        if (s[j]) rs[(n - 1 - j) >> 6] |= 1ULL << ((n - 1 - j) & 63);
    for (int t = 0; t < n; ++t) {
        // d = XOR_{i=0..L} C_i s_{t-i}, with s_{t-i} = rs bit (n-1-t+i)
        const long off = n - 1 - t;
        const long ow = off >> 6;
        const int ob = static_cast<int>(off & 63);
        uint64_t acc = 0;
        for (int w = 0; w <= L / 64; ++w) {
            uint64_t win = rs[ow + w] >> ob;
            if (ob && ow + w + 1 < static_cast<long>(rs.size())) win |= rs[ow + w + 1] << (64 - ob);
            acc ^= win & C[w];
        }
        if (!(__builtin_popcountll(acc) & 1)) {
            ++m;
        } else if (2 * L <= t) {
            T = C;
            xor_shifted(C, B, m);
            L = t + 1 - L;
            B = T;
            m = 1;
        } else {
            xor_shifted(C, B, m);
            ++m;
        }
    }
    if (L != kDeg) throw std::runtime_error("mt19937_64 jump-ahead: unexpected linear complexity");
    // phi(x) = x^L C(1/x): coefficient of x^(L-i) is C_i
    Poly phi(kPW + 1, 0);
    for (int i = 0; i <= L; ++i)
        if (bit(C, i)) phi[(L - i) >> 6] |= 1ULL << ((L - i) & 63);
    return phi;
}

struct PhiTables {
    Poly phi;
    std::vector<Poly> sh;  // phi << s, s = 0..63
};

const PhiTables& phi_tables() {
    static std::once_flag once;
    static std::unique_ptr<PhiTables> t;
    std::call_once(once, [] {
        auto p = std::make_unique<PhiTables>();
        p->phi = find_phi();
        p->sh.resize(64);
        for (int s = 0; s < 64; ++s) {
            p->sh[s].assign(kPW + 2, 0);
            xor_shifted(p->sh[s], p->phi, s);
        }
        t = std::move(p);
    });
    return *t;
}

// (a * b) mod phi, deg a, b < kDeg
Poly mulmod(const Poly& a, const Poly& b) {
    const PhiTables& T = phi_tables();
    std::vector<Poly> bs(64);
    for (int s = 0; s < 64; ++s) {
        bs[s].assign(kPW + 1, 0);
        xor_shifted(bs[s], b, s);
    }
    Poly p(2 * kPW + 2, 0);
    for (int w = 0; w < kPW; ++w) {
        uint64_t a_w = a[w];
        while (a_w) {
            const int s = __builtin_ctzll(a_w);
            a_w &= a_w - 1;
            const Poly& q = bs[s];
            for (int i = 0; i <= kPW; ++i) p[w + i] ^= q[i];
        }
    }
    for (long j = 2L * kDeg - 2; j >= kDeg; --j) {
        if (!bit(p, j)) continue;
        const long sh = j - kDeg;
        const Poly& q = T.sh[sh & 63];
        const long w = sh >> 6;
        for (size_t i = 0; i < q.size() && w + static_cast<long>(i) < static_cast<long>(p.size()); ++i) p[w + i] ^= q[i];
    }
    p.resize(kPW);
    return p;
}

Poly monomial(long e) {  // x^e, e < kDeg
    Poly p(kPW, 0);
    p[e >> 6] = 1ULL << (e & 63);
    return p;
}

Poly xpow(long long e) {  // x^e mod phi
    Poly r = monomial(0), base = monomial(1);
    while (e) {
        if (e & 1) r = mulmod(r, base);
        e >>= 1;
        if (e) base = mulmod(base, base);
    }
    return r;
}

// coefficient vectors r_p = x^(311 + p * chunk) mod phi, cached per chunk
std::vector<uint64_t> jump_coeffs(long long chunk, int P) {
    static std::mutex mu;
    static std::map<long long, std::vector<Poly>> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto& v = cache[chunk];
    if (v.empty()) v.push_back(monomial(kNN - 1));
    if (static_cast<int>(v.size()) < P) {
        const Poly g = xpow(chunk);
        while (static_cast<int>(v.size()) < P) v.push_back(mulmod(v.back(), g));
    }
    std::vector<uint64_t> out(static_cast<size_t>(P) * kPW);
    for (int p = 0; p < P; ++p) std::memcpy(out.data() + static_cast<size_t>(p) * kPW, v[p].data(), kPW * 8);
    return out;
}

// One CTA per chunk: window from the staged raw words and r_p, then the
// recurrence. Output q (tensor order) goes to dst[(q / d0) * pd0 + q % d0].
__global__ void __launch_bounds__(320) mt64_generate_kernel(const uint64_t* __restrict__ raw,
                                                            const uint64_t* __restrict__ coeffs, long long n,
                                                            long long chunk, long long d0, long long pd0,
                                                            double* __restrict__ dst) {
    extern __shared__ uint64_t sm[];
    uint64_t* sraw = sm;             // x_1 .. x_kRaw
    uint64_t* sco = sm + kRaw;       // r_p
    uint64_t* ring = sco + kPW;      // four 156-word blocks
    const int tid = threadIdx.x;
    const long long start = static_cast<long long>(blockIdx.x) * chunk;
    if (start >= n) return;
    const long long end = start + chunk < n ? start + chunk : n;
    for (int i = tid; i < kRaw; i += blockDim.x) sraw[i] = raw[i + 1];
    for (int i = tid; i < kPW; i += blockDim.x) sco[i] = coeffs[static_cast<long long>(blockIdx.x) * kPW + i];
    __syncthreads();
    if (tid < kNN) {  // word tid of the window: x_{312 + start + tid} = XOR_{r_i = 1} x_{1 + i + tid}
        uint64_t acc = 0;
        for (int w = 0; w < kPW; ++w) {
            uint64_t c = sco[w];
            while (c) {
                const int b = __ffsll(static_cast<long long>(c)) - 1;
                c &= c - 1;
                acc ^= sraw[64 * w + b + tid];
            }
        }
        ring[tid] = acc;  // blocks 0 and 1
    }
    __syncthreads();
    // Warp-specialised steps over a four-block ring: warps 0-4 run the
    // recurrence (block b+2 from blocks b, b+1), warps 5-9 temper and store
    // block b-1, which stays untouched until step b+1 overwrites its slot.
    const long long nblk = (end - start + kMM - 1) / kMM;  // blocks this chunk outputs
    const bool rec = tid < kMM;
    const int u = tid - 160;
    const bool sto = u >= 0 && u < kMM;
    long long row = 0, col = 0, q = start + u;
    if (sto) {
        row = q / d0;
        col = q - row * d0;
    }
    for (long long b = 0; b <= nblk; ++b) {
        if (rec) {
            const uint64_t* old = ring + (b & 3) * kMM;
            const uint64_t* nxt = ring + ((b + 1) & 3) * kMM;
            const uint64_t x0 = old[tid];
            ring[((b + 2) & 3) * kMM + tid] = mt_twist(x0, tid + 1 < kMM ? old[tid + 1] : nxt[0], nxt[tid]);
        } else if (sto && b > 0) {
            const uint64_t y = ring[((b - 1) & 3) * kMM + u];
            if (q < end) dst[row * pd0 + col] = mt_value(y);
            q += kMM;
            col += kMM;
            while (col >= d0) {
                col -= d0;
                ++row;
            }
        }
        __syncthreads();
    }
}

}  // namespace

size_t mt64_generate_smem() { return static_cast<size_t>(kRaw + kPW + 4 * kMM) * sizeof(uint64_t); }

void mt64_generate(double* dst, long long n, long long d0, long long pd0, uint64_t seed, int nsm,
                   uint64_t* dev_scratch, cudaStream_t s) {
    if (n <= 0) return;
    const long long want = (n + 65535) / 65536;
    const int P = static_cast<int>(std::max<long long>(1, std::min<long long>(want, nsm)));
    const long long chunk = (n + P - 1) / P;
    const auto raw = raw_words(seed, kRaw + 1);
    const auto co = jump_coeffs(chunk, P);
    uint64_t* draw = dev_scratch;           // x_0 .. x_kRaw
    uint64_t* dco = dev_scratch + kRaw + 1;  // P coefficient vectors
    cudaMemcpyAsync(draw, raw.data(), raw.size() * 8, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(dco, co.data(), co.size() * 8, cudaMemcpyHostToDevice, s);
    const size_t smem = mt64_generate_smem();
    cudaFuncSetAttribute(mt64_generate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    mt64_generate_kernel<<<P, 320, smem, s>>>(draw, dco, n, chunk, d0, pd0, dst);
    // the host vectors must outlive the async copies (pageable: the copies are
    // staged synchronously before cudaMemcpyAsync returns)
}

size_t mt64_scratch_words(int nsm) { return static_cast<size_t>(kRaw + 1) + static_cast<size_t>(nsm) * kPW; }

}  // namespace dmtkg

// Host-side check of the jump-ahead (no device needed): the raw words
// x_{312+start} .. x_{623+start} of mt19937_64(seed), formed from the first
// raw words and x^(311+start) mod phi exactly as a generator CTA forms its
// window. Returns 0, or -1 on a negative start.
extern "C" int dmtk_gpu_mt64_jump(uint64_t seed, int64_t start, uint64_t* words312) {
    using namespace dmtkg;
    if (start < 0 || !words312) return -1;
    try {
        const auto raw = raw_words(seed, kRaw + 1);
        const Poly r = start == 0 ? monomial(kNN - 1) : mulmod(monomial(kNN - 1), xpow(start));
        for (int k = 0; k < kNN; ++k) {
            uint64_t acc = 0;
            for (int w = 0; w < kPW; ++w) {
                uint64_t c = r[w];
                while (c) {
                    const int b = __builtin_ctzll(c);
                    c &= c - 1;
                    acc ^= raw[1 + 64 * w + b + k];
                }
            }
            words312[k] = acc;
        }
        return 0;
    } catch (...) {
        return -1;
    }
}
