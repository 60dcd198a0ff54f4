// Times the CP-ALS solve kernels in isolation (one 20x20 SPD matrix, n
// launches back to back): shared-memory vs register Cholesky + inverse.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../include -o chol_probe chol_probe.cu
#include "../../paper_1708_08976_b200/csrc/kernels.cu"

#include <cstdio>
#include <vector>

int main() {
    using namespace dmtkg;
    const int n = 20;
    std::vector<double> h(n * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) h[i * n + j] = (i == j ? n : 0.0) + 1.0 / (1.0 + i + j);
    double *H, *Hi;
    int* flag;
    cudaMalloc(&H, n * n * 8);
    cudaMalloc(&Hi, n * n * 8);
    cudaMalloc(&flag, 4);
    cudaMemcpy(H, h.data(), n * n * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(cholesky_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * 64 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int v = 0; v < 3; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            for (int i = 0; i < 200; ++i) {
                if (v == 0) cholesky_inverse_kernel<<<1, 32, 2 * n * n * 8>>>(H, n, Hi, flag);
                if (v == 1) cholesky_inverse_rl_kernel<<<1, 32>>>(H, n, Hi, flag);
                if (v == 2) cholesky_kernel<<<1, 32>>>(H, n, Hi, flag);
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) std::printf("variant %d: %.2f us per launch (%s)\n", v, ms * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
