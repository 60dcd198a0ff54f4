// FP64 tensor-core throughput by MMA shape and warps per SM sub-partition.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_shape_probe mma_shape_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void m884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void m1684(double (&d)[4], const double (&a)[2], double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b));
}
__device__ __forceinline__ void m1688(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void m16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int SHAPE, int NACC>
__global__ void probe(double* out, int iters) {
  const double v = threadIdx.x * 1e-9 + 1.0;
  double acc[NACC][4];
  for (int k = 0; k < NACC; ++k) acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.0;
  double a[8], b[4];
  for (int k = 0; k < 8; ++k) a[k] = v + k;
  for (int k = 0; k < 4; ++k) b[k] = v - k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < NACC; ++k) {
      if (SHAPE == 0) m884(reinterpret_cast<double(&)[2]>(acc[k]), a[k & 7], b[k & 3]);
      if (SHAPE == 1) m1684(acc[k], reinterpret_cast<const double(&)[2]>(a), b[k & 3]);
      if (SHAPE == 2) m1688(acc[k], reinterpret_cast<const double(&)[4]>(a), reinterpret_cast<const double(&)[2]>(b));
      if (SHAPE == 3) m16816(acc[k], a, b);
    }
  }
  double s = 0;
  for (int k = 0; k < NACC; ++k) s += acc[k][0] + acc[k][1] + acc[k][2] + acc[k][3];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int SHAPE, int NACC>
int run(const char* name, double fma_per, int sms, double* out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int wps : {1, 2, 3, 4}) {  // warps per SM sub-partition
    const int tpb = 128 * wps;
    const int iters = SHAPE == 3 ? 2000 : (SHAPE == 0 ? 16000 : (SHAPE == 1 ? 8000 : 4000));
    probe<SHAPE, NACC><<<sms, tpb>>>(out, 10);
    CK(cudaEventRecord(e0));
    probe<SHAPE, NACC><<<sms, tpb>>>(out, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double flops = 2.0 * fma_per * NACC * iters * (double)sms * (tpb / 32);
    std::printf("%-10s nacc %d warps/SMSP %d: %6.2f TFLOP/s\n", name, NACC, wps, flops / ms / 1e9);
  }
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 4096 * 8));
  run<0, 8>("m8n8k4", 256, sms, out);
  run<0, 12>("m8n8k4", 256, sms, out);
  run<1, 8>("m16n8k4", 512, sms, out);
  run<2, 8>("m16n8k8", 1024, sms, out);
  run<3, 4>("m16n8k16", 2048, sms, out);
  run<3, 8>("m16n8k16", 2048, sms, out);
  return 0;
}
