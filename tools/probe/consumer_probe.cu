// Consumer-loop microbenchmark: DMMA 8x8x4 fed from shared memory with the
// streaming kernel's fragment pattern (no TMA, no barriers). Answers: how
// close to the FP64 tensor peak can W warps/CTA x RB row blocks x NB column
// groups (+ DFMA tail) get when every fragment comes from LDS?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o consumer_probe consumer_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); std::exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int RB, int NB, int TAIL, bool PF, int TM = 0>
__global__ void consumer(double* out, int stages) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 12288; i += blockDim.x) sm[i] = 1.0 + i * 1e-7;
  __syncthreads();
  const unsigned char* base = reinterpret_cast<const unsigned char*>(sm);
  struct Frag { double2 bv[NB]; double a[2][RB]; double bt[2][TAIL > 0 ? TAIL : 1]; };
  double acc[RB][NB][2];
  double tacc[RB][TAIL > 0 ? TAIL : 1];
  double tacc2[RB][TAIL > 0 ? TAIL : 1];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
#pragma unroll
    for (int n = 0; n < NB; ++n) acc[r][n][0] = acc[r][n][1] = 0;
#pragma unroll
    for (int t = 0; t < (TAIL > 0 ? TAIL : 1); ++t) tacc[r][t] = tacc2[r][t] = 0;
  }
  auto load = [&](Frag& f, int slot, int s2) {
    const unsigned char* A = base + (slot & 1) * 32768 + (w & 7) * 4096;
    const unsigned char* B = base + 65536 + (slot & 1) * 8192;
#pragma unroll
    for (int n = 0; n < NB; ++n) f.bv[n] = *reinterpret_cast<const double2*>(B + (((s2 * NB + n) * 32 + lane) << 4));
#pragma unroll
    for (int sub = 0; sub < 2; ++sub) {
#pragma unroll
      for (int r = 0; r < RB; ++r)
        f.a[sub][r] = *reinterpret_cast<const double*>(A + ((((2 * s2 + sub) * RB + r) & 15) << 8) + lane * 8);
      if (TAIL > 0)
#pragma unroll
        for (int t = 0; t < TAIL; ++t) f.bt[sub][t] = *reinterpret_cast<const double*>(B + 6144 + ((2 * s2 + sub) * 4 + (lane & 3)) * 8 * TAIL + t * 8);
    }
  };
  auto compute = [&](const Frag& f) {
#pragma unroll
    for (int sub = 0; sub < 2; ++sub) {
#pragma unroll
      for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int n = 0; n < NB; ++n) dmma(acc[r][n][0], acc[r][n][1], f.a[sub][r], sub ? f.bv[n].y : f.bv[n].x);
      if (TAIL > 0)
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int t = 0; t < TAIL; ++t) {
            if (TM == 1 && sub) tacc2[r][t] = fma(f.a[sub][r], f.bt[sub][t], tacc2[r][t]);
            else tacc[r][t] = fma(f.a[sub][r], f.bt[sub][t], tacc[r][t]);
          }
    }
  };
  Frag f0, f1;
  if (PF) load(f0, 0, 0);
  for (int st = 0; st < stages; ++st) {
    if (PF) {
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        Frag& cf = (s2 & 1) ? f1 : f0;
        Frag& nf = (s2 & 1) ? f0 : f1;
        if (s2 < 3) load(nf, st, s2 + 1); else load(nf, st + 1, 0);
        compute(cf);
      }
    } else {
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) { load(f0, st, s2); compute(f0); }
    }
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < RB; ++r) {
#pragma unroll
    for (int n = 0; n < NB; ++n) s += acc[r][n][0] + acc[r][n][1];
#pragma unroll
    for (int t = 0; t < (TAIL > 0 ? TAIL : 1); ++t) s += tacc[r][t] + tacc2[r][t];
  }
  if (s == 12345.678) out[0] = s;
}

template <int RB, int NB, int TAIL, bool PF, int TM = 0>
void run(const char* name, int warps, int sms, double* out) {
  const int smem = 98304;
  CK(cudaFuncSetAttribute(consumer<RB, NB, TAIL, PF, TM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int stages = 4000;
  consumer<RB, NB, TAIL, PF, TM><<<sms, warps * 32, smem>>>(out, 10);
  CK(cudaEventRecord(e0));
  consumer<RB, NB, TAIL, PF, TM><<<sms, warps * 32, smem>>>(out, stages);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  // useful flops: 8 k4-steps x (RB*8 rows) x (NB*8 + TAIL cols) x 4 k x 2
  const double fl = 2.0 * sms * warps * (double)stages * 8 * (RB * 8) * (NB * 8 + TAIL) * 4;
  cudaFuncAttributes a; CK(cudaFuncGetAttributes(&a, consumer<RB, NB, TAIL, PF, TM>));
  std::printf("%-22s warps %2d regs %3d: %.2f TFLOP/s\n", name, warps, a.numRegs, fl / ms / 1e9);
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  double* out; CK(cudaMalloc(&out, 64));
  const int sms = p.multiProcessorCount;
  for (int w : {8, 12}) {
    run<2, 3, 1, true>("RB2 NB3 T1 pf", w, sms, out);
    run<2, 3, 1, true, 1>("RB2 NB3 T1 pf split", w, sms, out);
    run<2, 3, 0, true>("RB2 NB3 T0 pf", w, sms, out);
    run<4, 3, 1, true, 1>("RB4 NB3 T1 pf split", w, sms, out);
    run<2, 6, 2, true, 1>("RB2 NB6 T2 pf split", w, sms, out);
    run<2, 6, 2, true, 0>("RB2 NB6 T2 pf", w, sms, out);
    run<2, 6, 0, true, 0>("RB2 NB6 T0 pf", w, sms, out);
  }
  return 0;
}
