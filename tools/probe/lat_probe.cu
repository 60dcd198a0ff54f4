// FP64 dependent-latency microbenchmark (one thread): DFMA, DADD, sqrt,
// division, shared-memory load, warp shuffle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, int iters, int kind, long long* cycles) {
    __shared__ double sm[64];
    sm[threadIdx.x] = 1.0 + threadIdx.x * 1e-9;
    __syncwarp();
    double x = 1.0000001 + threadIdx.x * 1e-12, y = 0.9999999;
    int idx = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (kind == 0) x = fma(x, y, 1e-9);
        else if (kind == 1) x = sqrt(x + 1.0);
        else if (kind == 2) x = 1.0 / (x + 1.0);
        else if (kind == 3) { x = sm[idx] + x * 1e-30; idx = (int)(x) & 31; }
        else x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * y;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) *cycles = t1 - t0;
    if (x == 12345.0) *out = x;
}

int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 8);
    cudaMalloc(&c, 8);
    const char* names[] = {"dfma", "sqrt+add", "div+add", "lds", "shfl+mul"};
    for (int k = 0; k < 5; ++k) {
        lat<<<1, 32>>>(o, 100, k, c);
        lat<<<1, 32>>>(o, 10000, k, c);
        long long h;
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        std::printf("%-10s %.1f cycles per dependent op\n", names[k], h / 10000.0);
    }
    return 0;
}
