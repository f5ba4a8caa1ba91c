// Launch-gap probe: a CUDA graph of N back-to-back dependent launches of an
// (almost) empty kernel, grid G x 256 threads; prints us per launch.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_nop(float* p, int n) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && n < 0) p[0] = 1.f;
}
int main() {
    float* d;
    cudaMalloc(&d, 16);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    const int grids[] = {1, 148, 256, 512, 1024};
    for (int g : grids) {
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < 400; ++i) k_nop<<<g, 256, 0, s>>>(d, i);
        cudaStreamEndCapture(s, &graph);
        cudaGraphInstantiate(&exec, graph, 0);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int w = 0; w < 3; ++w) cudaGraphLaunch(exec, s);
        cudaEventRecord(a, s);
        for (int r = 0; r < 10; ++r) cudaGraphLaunch(exec, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("grid %5d x 256: %.2f us per launch (graph of 400)\n", g, ms * 1e3 / 4000);
    }
    return 0;
}
