// Micro-benchmark: per-node cost of a chain of small dependent kernels in a
// CUDA graph, with and without programmatic dependent launch (PDL).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_step(int *x, int n, int pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] += 1;
    if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}

static float run(int nodes, int pdl, int ctas) {
    int *x;
    cudaMalloc(&x, sizeof(int) * ctas * 256);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < nodes; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ctas);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k_step, x, ctas * 256, pdl);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int w = 0; w < 20; ++w) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(x);
    return ms * 1000.0f / 20 / nodes;
}

int main() {
    for (int ctas : {148, 1184})
        for (int pdl : {0, 1})
            printf("ctas %4d pdl %d: %.2f us per node\n", ctas, pdl, run(40, pdl, ctas));
    return 0;
}
