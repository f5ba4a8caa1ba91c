// Throughput probe: scalar FFMA vs packed FFMA2 (__ffma2_rn) on sm_100a.
// Each thread runs 8 independent accumulator chains for N iterations.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float* out, float a, float b, int n) {
    float x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
    float s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a, float b, int n) {
    float2 x[8];
    for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x * 1e-3f + k, k + 0.5f);
    const float2 aa = make_float2(a, a), bb = make_float2(b, b);
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __ffma2_rn(x[k], aa, bb);
    float s = 0;
    for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, n = 1 << 14;
    float* out;
    cudaMalloc(&out, sizeof(float) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        float ms1, ms2;
        cudaEventRecord(e0);
        k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-3f, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms1, e0, e1);
        cudaEventRecord(e0);
        k_ffma2<<<blocks, threads>>>(out, 0.999f, 1e-3f, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms2, e0, e1);
        const double fl1 = 2.0 * 8 * n * (double)blocks * threads, fl2 = 2 * fl1;
        printf("FFMA : %.3f ms  %.1f TFLOP/s\nFFMA2: %.3f ms  %.1f TFLOP/s\n", ms1, fl1 / ms1 / 1e9, ms2,
               fl2 / ms2 / 1e9);
    }
    return 0;
}
