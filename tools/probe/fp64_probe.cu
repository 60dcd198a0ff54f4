// B200 FP64 / HBM microbenchmark: measures the denominators the MTTKRP
// roofline needs but MEASURED_PEAKS.json does not carry (FP64 DFMA and DMMA
// throughput, read-only HBM streaming bandwidth). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); std::exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double r[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) r[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = fma(r[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += r[k];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) { acc[k][0] = 0; acc[k][1] = 0; }
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma884(acc[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
               "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

__global__ void dmma16816_kernel(double* out, int iters) {
  double acc[4][4];
  double a[8], b[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + threadIdx.x * 1e-6 + k;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = 0.5 + k;
#pragma unroll
  for (int k = 0; k < 4; ++k) for (int q = 0; q < 4; ++q) acc[k][q] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) dmma16816(acc[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) for (int q = 0; q < 4; ++q) s += acc[k][q];
  if (s == 12345.678) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ x, size_t n2, double* out) {
  double s0 = 0, s1 = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride * 4) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      size_t j = i + u * stride;
      v[u] = j < n2 ? __ldcs(x + j) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) { s0 += v[u].x; s1 += v[u].y; }
  }
  if (s0 + s1 == 12345.678) out[0] = s0;
}


__global__ void write_kernel(double2* __restrict__ x, size_t n2, double v) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride)
    __stcs(x + i, make_double2(v, v + 1.0));
}

__global__ void fill_kernel(double* x, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    x[i] = (double)(i & 1023) * 1e-3;
}

// warps [0, dmma_warps) issue DMMA, the rest DFMA: does the FP64 vector pipe
// run concurrently with the FP64 tensor pipe?
__global__ void mixed_kernel(double* out, int iters, int dmma_warps, double a0, double b0) {
  const int w = threadIdx.x >> 5;
  double s = 0;
  if (w < dmma_warps) {
    double acc[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc[k][0] = 0; acc[k][1] = 0; }
    double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) dmma884(acc[k], a, b);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1];
  } else {
    double r[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = threadIdx.x * 1e-3 + k;
    for (int it = 0; it < iters * 8; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) r[k] = fma(r[k], a0, b0);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) s += r[k];
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  std::printf("device %s sms %d l2 %d MB smem/blk optin %zu\n", p.name, sms, p.l2CacheSize >> 20,
              p.sharedMemPerBlockOptin);
  double* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms;

  for (int tpb : {256, 512}) {
    for (int per_sm : {2, 4}) {
      int iters = 20000;
      int grid = sms * per_sm;
      dfma_kernel<<<grid, tpb>>>(out, 100, 1.0000001, 1e-9);
      CK(cudaEventRecord(e0));
      dfma_kernel<<<grid, tpb>>>(out, iters, 1.0000001, 1e-9);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double flops = 2.0 * 16 * iters * (double)grid * tpb;
      std::printf("DFMA tpb %d blocks/sm %d: %.2f TFLOP/s (%.3f ms)\n", tpb, per_sm, flops / ms / 1e9, ms);
    }
  }
  for (int tpb : {128, 256, 512}) {
    for (int per_sm : {1, 2, 4}) {
      int iters = 4000;
      int grid = sms * per_sm;
      dmma_kernel<<<grid, tpb>>>(out, 100);
      CK(cudaEventRecord(e0));
      dmma_kernel<<<grid, tpb>>>(out, iters);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double flops = 2.0 * 256 * 8 * iters * (double)grid * (tpb / 32);
      std::printf("DMMA884 tpb %d blocks/sm %d: %.2f TFLOP/s (%.3f ms)\n", tpb, per_sm, flops / ms / 1e9, ms);
    }
  }
  for (int tpb : {128, 256}) {
    int iters = 1000;
    int grid = sms * 2;
    dmma16816_kernel<<<grid, tpb>>>(out, 10);
    CK(cudaEventRecord(e0));
    dmma16816_kernel<<<grid, tpb>>>(out, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 16 * 8 * 16 * 4 * iters * (double)grid * (tpb / 32);
    std::printf("DMMA16816 tpb %d: %.2f TFLOP/s (%.3f ms)\n", tpb, flops / ms / 1e9, ms);
  }
  {
    // per warp per iter: DMMA warp 8*512 flop, DFMA warp 8*16*32*2 = 8192 flop
    const int tpb = 512, grid = sms;
    for (int dw : {16, 8, 12, 4, 0}) {
      int iters = 2000;
      mixed_kernel<<<grid, tpb>>>(out, 10, dw, 1.0000001, 1e-9);
      CK(cudaEventRecord(e0));
      mixed_kernel<<<grid, tpb>>>(out, iters, dw, 1.0000001, 1e-9);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double fl = (double)grid * iters * (dw * 8.0 * 512 + (16 - dw) * 8.0 * 16 * 32 * 2);
      std::printf("MIXED dmma_warps %d/16: %.2f TFLOP/s (%.3f ms)\n", dw, fl / ms / 1e9, ms);
    }
  }
  size_t n = (size_t)1 << 30;  // 8 GiB of doubles
  double* x;
  CK(cudaMalloc(&x, n * 8));
  fill_kernel<<<sms * 8, 256>>>(x, n);
  CK(cudaDeviceSynchronize());
  for (int per_sm : {4, 8, 16}) {
    for (int tpb : {256, 512}) {
      int grid = sms * per_sm;
      read_kernel<<<grid, tpb>>>((const double2*)x, n / 2, out);
      CK(cudaEventRecord(e0));
      for (int r = 0; r < 5; ++r) read_kernel<<<grid, tpb>>>((const double2*)x, n / 2, out);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      std::printf("read-stream blocks/sm %d tpb %d: %.1f GB/s\n", per_sm, tpb, 5.0 * n * 8 / ms / 1e6);
    }
  }
  for (int per_sm : {4, 8, 16}) {
    const int tpb = 256, grid = sms * per_sm;
    write_kernel<<<grid, tpb>>>((double2*)x, n / 2, 1.0);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) write_kernel<<<grid, tpb>>>((double2*)x, n / 2, 1.0 + r);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::printf("write-stream blocks/sm %d: %.1f GB/s\n", per_sm, 5.0 * n * 8 / ms / 1e6);
  }
  for (int r = 0; r < 2; ++r) {
    CK(cudaEventRecord(e0));
    CK(cudaMemsetAsync(x, r, n * 8));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::printf("cudaMemset: %.1f GB/s\n", n * 8 / ms / 1e6);
  }
  CK(cudaFree(x));
  return 0;
}
