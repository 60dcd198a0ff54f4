// xrank.cu -- the fused cross-rank reduction of the sharded CP-ALS
// (SURVEY §8f-1): one kernel that finishes a mode's MTTKRP (the CSR slot
// reduction of the streaming kernel's partial rows) AND sums the I_n x C
// partials of every last-mode shard over NVLink peer memory, replacing the
// separate slot_reduce launch + ncclAllReduce at the reference's exchange
// point (cp_als.cpp:142, every non-last mode).
//
// Protocol (one-shot push, deterministic): the reduced array is split into
// nblk row chunks, block b of every rank owns chunk b.
//   1. block b forms its chunk's local values (the slot sums, or a plain
//      buffer) and stores them into EVERY rank's receive buffer, in the
//      sender's row [parity][sender] (peer stores over NVLink);
//   2. one thread fences (system scope) and release-stores the block's epoch
//      into flag[sender][b] of every rank;
//   3. the block spins (acquire, system scope) on its OWN memory until all P
//      senders' flags for chunk b reached the epoch, then sums the P rows in
//      rank order 0..P-1 -- the same bytes on every rank (bitwise identical
//      factors on all ranks, run to run).
// Epochs are per block in device memory (ctr[b], read and advanced only by
// block b), so the kernel is graph-replayable. Receive rows alternate by
// epoch parity: a rank writes parity e & 1 at epoch e only after every peer
// flagged epoch e - 1 for that chunk, which each peer does only after its
// stream finished epoch e - 2 (all of its reads of that parity).
//
// A block waits only for the same block index of the other ranks; nblk is
// at most the co-resident capacity and the launch is cooperative, so every
// block of every rank is resident. With fewer GPUs than ranks (the loopback
// group) the P ranks run as ONE cooperative launch, gridDim.y = P virtual
// ranks over one device's buffers (never as launches that wait on each other).
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace dmtkg {

namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

constexpr int kXThreads = 256;
constexpr unsigned long long kXTimeoutNs = 30ull * 1000 * 1000 * 1000;  // 30 s

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(kXThreads) xrank_reduce_kernel(const XrankArgs a) {
    const int vr = blockIdx.y;  // virtual rank (emulated group) or 0
    const int rank = a.rank0 + vr;
    const XrankLocal& me = a.me[vr];
    const int P = a.P;
    const int b = blockIdx.x;
    const int nblk = gridDim.x;
    const int C = a.C;
    const long long rows = a.rows;
    const long long r0 = rows * b / nblk, r1 = rows * (b + 1) / nblk;
    __shared__ unsigned long long s_epoch;
    __shared__ double part[kXThreads];
    if (threadIdx.x == 0) s_epoch = me.ctr[b] + 1;
    __syncthreads();
    const unsigned long long e = s_epoch;
    const long long par = static_cast<long long>(e & 1ull);
    // this rank's row of every receive buffer
    const long long mine = (par * P + rank) * a.cap;

    // 1. local values of the chunk, pushed to every rank
    if (me.rowptr) {
        // CSR slot sums, as slot_reduce_kernel: thread (p, c) sums slots
        // k0 + p, k0 + p + Q, ... of the row, the Q partials added in order
        const int Q = kXThreads / C;
        const int p = threadIdx.x / C;
        const int c = threadIdx.x - p * C;
        for (long long i = r0; i < r1; ++i) {
            const long long k0 = me.rowptr[i], k1 = me.rowptr[i + 1];
            double s = 0.0;
            if (p < Q) {  // four independent chains, as slot_reduce_kernel
                double q[4] = {0.0, 0.0, 0.0, 0.0};
                long long k = k0 + p;
                for (; k + 3 * Q < k1; k += 4 * Q) {
                    const long long e0 = me.slots[k], e1 = me.slots[k + Q], e2 = me.slots[k + 2 * Q],
                                    e3 = me.slots[k + 3 * Q];
                    q[0] += me.src[e0 * C + c];
                    q[1] += me.src[e1 * C + c];
                    q[2] += me.src[e2 * C + c];
                    q[3] += me.src[e3 * C + c];
                }
                if (k < k1) q[0] += me.src[me.slots[k] * C + c];  // at most three left
                if (k + Q < k1) q[1] += me.src[me.slots[k + Q] * C + c];
                if (k + 2 * Q < k1) q[2] += me.src[me.slots[k + 2 * Q] * C + c];
                s = (q[0] + q[1]) + (q[2] + q[3]);
            }
            part[threadIdx.x] = s;
            __syncthreads();
            if (threadIdx.x < C) {
                double u[4] = {0.0, 0.0, 0.0, 0.0};  // the same fold as slot_reduce_kernel
                for (int q = 0; q < Q; ++q) u[q & 3] += part[q * C + threadIdx.x];
                const double t = (u[0] + u[1]) + (u[2] + u[3]);
                for (int k = 0; k < P; ++k) a.recv[k][mine + i * C + threadIdx.x] = t;
            }
            __syncthreads();
        }
    } else {
        for (long long x = r0 * C + threadIdx.x; x < r1 * C; x += kXThreads) {
            const double v = me.src[x];
            for (int k = 0; k < P; ++k) a.recv[k][mine + x] = v;
        }
    }
    __syncthreads();
    // 2. publish: every store above happens-before the flag (bar.sync + a
    //    system-scope fence by the releasing thread, cumulative)
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (int k = 0; k < P; ++k) st_release_sys(a.flags[k] + static_cast<long long>(rank) * a.nblk_cap + b, e);
    }
    // 3. wait for chunk b of every sender (flags in this rank's own memory)
    if (threadIdx.x < P) {
        const unsigned long long* f = a.flags[rank] + static_cast<long long>(threadIdx.x) * a.nblk_cap + b;
        const unsigned long long t0 = globaltimer_ns();
        int spins = 0;
        while (ld_acquire_sys(f) < e) {
            // a peer that never arrives (its process died) fails the launch
            // loudly instead of hanging the device
            if (++spins == 4096) {
                spins = 0;
                if (globaltimer_ns() - t0 > kXTimeoutNs) __trap();
            }
        }
    }
    __syncthreads();
    __threadfence();
    const double* in = a.recv[rank] + par * P * a.cap;
    for (long long x = r0 * C + threadIdx.x; x < r1 * C; x += kXThreads) {
        double s = in[x];
        for (int k = 1; k < P; ++k) s += in[k * a.cap + x];
        me.out[x] = s;
    }
    if (threadIdx.x == 0) me.ctr[b] = e;
}

}  // namespace

cudaError_t launch_xrank_reduce(const XrankArgs& a, int nblk, int vranks, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(nblk), static_cast<unsigned>(vranks));
    cfg.blockDim = dim3(kXThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every block resident: they wait on each other
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, xrank_reduce_kernel, a);
}

int xrank_max_blocks() {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, xrank_reduce_kernel, kXThreads, 0);
    return sms * per;
}

}  // namespace dmtkg
