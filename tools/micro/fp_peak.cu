// fp_peak.cu -- measured FP32 / FP64 arithmetic peaks of this B200 (the
// denominators of the FP-bound rooflines in bench.py): independent FMA /
// ADD chains per thread, many warps per SM, CUDA events.  Prints JSON.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp_peak fp_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, bool FMA>
__global__ void k_peak(T *out, int iters, T a, T b) {
    T x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = (T)(threadIdx.x + k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = FMA ? x[k] * a + b : x[k] + b;
    }
    T s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == (T)-1.2345) out[threadIdx.x] = s;  // keep the chains alive
}

template <typename T, bool FMA>
double run(int sms) {
    T *out;
    cudaMalloc(&out, 1024 * sizeof(T));
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_peak<T, FMA><<<blocks, threads>>>(out, 64, (T)0.999, (T)1e-3);
    cudaEventRecord(a);
    k_peak<T, FMA><<<blocks, threads>>>(out, iters, (T)0.999, (T)1e-3);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(out);
    const double instr = (double)blocks * threads * iters * 8;  // per-thread ops
    return instr / (ms * 1e-3) / 1e12;                          // T instr/s
}

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double best[4] = {0, 0, 0, 0};
    for (int r = 0; r < 5; ++r) {
        double v[4] = {run<float, true>(sms), run<float, false>(sms), run<double, true>(sms), run<double, false>(sms)};
        for (int k = 0; k < 4; ++k) best[k] = v[k] > best[k] ? v[k] : best[k];
    }
    printf("{\"fp32_fma_tinstr\": %.3f, \"fp32_add_tinstr\": %.3f, \"fp64_fma_tinstr\": %.3f, "
           "\"fp64_add_tinstr\": %.3f, \"fp32_tflops\": %.3f, \"fp64_tflops\": %.3f, \"sms\": %d, "
           "\"how\": \"tools/micro/fp_peak.cu: 8 independent FMA / ADD chains per thread, 8 x 256-thread CTAs "
           "per SM, CUDA events, best of 5\"}\n",
           best[0], best[1], best[2], best[3], 2 * best[0], 2 * best[2], sms);
    return 0;
}
