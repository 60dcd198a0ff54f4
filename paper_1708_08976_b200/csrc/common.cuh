// common.cuh -- device primitives shared by the dmtk B200 kernels:
// mbarrier + TMA (cp.async.bulk.tensor) wrappers, the FP64 tensor-core
// DMMA (mma.sync m8n8k4 f64) and the on-the-fly Khatri-Rao row generator.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cuda.h>
#include <cuda_runtime.h>

namespace dmtkg {

constexpr int kMaxFactors = 12;  // KRP inputs per generator (tensor order <= 13)

// Khatri-Rao row generator over a compound index (reference krp.hpp:19-32,
// mttkrp.cpp:55-75): value(idx, c) = prod_f U_f[((idx / stride_f) % ext_f) * ldu + c].
// Factor 0 is the fastest-varying input (stride 1). nf == 0 is the empty KRP
// (a row of ones, mttkrp.cpp:142-144).
struct KrpGen {
    int nf;
    int ldu;
    const double* U[kMaxFactors];
    long long ext[kMaxFactors];
    long long stride[kMaxFactors];
};

// 64-bit division, out of line: the software sequence is ~70 instructions,
// and inlined at every index computation it made the streaming kernels
// 14-24 K instructions long -- their one-shot code (prologue, builder set-up,
// epilogue) then ran from instruction-cache misses, tens of microseconds per
// launch once L2 had been flushed. The common (32-bit) paths stay inline.
static __device__ __noinline__ long long div64_slow(long long a, long long b) { return a / b; }

// a / b for non-negative operands, 32-bit when both fit.
__device__ __forceinline__ long long div_nn(long long a, long long b) {
    if (a < 0x7fffffffLL && b < 0x7fffffffLL) return static_cast<unsigned>(a) / static_cast<unsigned>(b);
    return div64_slow(a, b);
}

// Digit of factor f for a compound index (32-bit division when it fits).
__device__ __forceinline__ long long krp_digit(const KrpGen& g, int f, long long idx) {
    if (idx < 0x7fffffffLL && g.stride[f] < 0x7fffffffLL && g.ext[f] < 0x7fffffffLL) {
        const unsigned q = static_cast<unsigned>(idx) / static_cast<unsigned>(g.stride[f]);
        return q % static_cast<unsigned>(g.ext[f]);
    }
    const long long q = div64_slow(idx, g.stride[f]);
    return q - div64_slow(q, g.ext[f]) * g.ext[f];
}

__device__ __forceinline__ double krp_value(const KrpGen& g, long long idx, int c) {
    double v = 1.0;
#pragma unroll 1
    for (int f = 0; f < g.nf; ++f) {
        v *= __ldg(g.U[f] + krp_digit(g, f, idx) * g.ldu + c);
    }
    return v;
}

// krp_value with the single-factor case (a materialised or one-input KRP,
// the common scale operand of the multi-TTV epilogue) as one plain load.
__device__ __forceinline__ double krp_scale(const KrpGen& g, long long idx, int c) {
    if (g.nf == 1) return __ldg(g.U[0] + idx * g.ldu + c);  // idx < ext for every caller
    return krp_value(g, idx, c);
}

// Same, skipping factor 0 (the "head" partial product of the slower inputs).
__device__ __forceinline__ double krp_head(const KrpGen& g, long long idx, int c) {
    double v = 1.0;
#pragma unroll 1
    for (int f = 1; f < g.nf; ++f) {
        v *= __ldg(g.U[f] + krp_digit(g, f, idx) * g.ldu + c);
    }
    return v;
}

// ------------------------------------------- programmatic dependent launch
// Kernels launched with launch_pdl may start while the previous kernel in the
// stream finishes (its launch latency and prologue overlap that kernel's
// tail). Every such kernel calls pdl_wait() before it reads anything an
// earlier kernel wrote (and before it writes anything an earlier kernel
// reads), then pdl_trigger() -- always after the wait, so a chain of early
// launches never overtakes a kernel that is still running two launches back.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// DMTK_GPU_NO_PDL=1: plain launches (A/B switch)
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DMTK_GPU_NO_PDL");
        return !(e && *e && *e != '0');
    }();
    return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(std::forward<Args>(args))...);
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx_a(uint32_t bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(bar),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITA_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITA_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// -------------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// L2 policy for data read exactly once (the streamed tensor): evict first,
// so the factor rows the builders re-read stay L2-resident.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t l2_evict_normal_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1,
                                            uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1,
                                            int c2, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
}

// 8-byte asynchronous global->shared copy (LDGSTS); src_bytes = 0 zero-fills.
__device__ __forceinline__ void cp_async_8(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

// Arrive on an mbarrier once this thread's prior cp.async copies have landed
// (the barrier's expected count includes this arrival).
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ double2 lds_v2f64(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// ------------------------------------------------------------ FP64 DMMA
// D(8x8) += A(8x4, row) * B(4x8, col). Lane (g = lane>>2, t = lane&3) holds
// A[g][t], B[t][g] and D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// 128-byte TMA swizzle: within each 1024-byte atom the 16-byte chunk index
// (address bits 4..6) is XORed with the 128-byte row index (bits 7..9).
__device__ __forceinline__ uint32_t swz128(uint32_t off) { return off ^ ((off >> 3) & 0x70u); }

}  // namespace dmtkg
