#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lds(float* out, int iters) {
    __shared__ float4 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, i+1, i+2, i+3);
    __syncthreads();
    float4 acc = make_float4(0,0,0,0);
    int idx = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
        #pragma unroll
        for (int k = 0; k < 8; ++k) { float4 v = s[(idx + k * 32) & 2047]; acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
        idx += 1;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}
__global__ void k_shfl(float* out, int iters) {
    float a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
    float acc = 0;
    for (int it = 0; it < iters; ++it) {
        #pragma unroll
        for (int k = 0; k < 8; ++k) {
            a = __shfl_down_sync(0xffffffff, a, 1) + 1.f;
            b = __shfl_down_sync(0xffffffff, b, 2) + 1.f;
            c = __shfl_down_sync(0xffffffff, c, 3) + 1.f;
            d = __shfl_down_sync(0xffffffff, d, 4) + 1.f;
        }
        acc += a + b + c + d;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_mix(float* out, int iters) {
    __shared__ float4 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, i+1, i+2, i+3);
    __syncthreads();
    float4 acc = make_float4(0,0,0,0);
    float a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
    int idx = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
        #pragma unroll
        for (int k = 0; k < 8; ++k) {
            float4 v = s[(idx + k * 32) & 2047]; acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            a = __shfl_down_sync(0xffffffff, a, 1) + 1.f;
            b = __shfl_down_sync(0xffffffff, b, 2) + 1.f;
            c = __shfl_down_sync(0xffffffff, c, 3) + 1.f;
            d = __shfl_down_sync(0xffffffff, d, 4) + 1.f;
        }
        idx += 1;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w + a + b + c + d;
}
int main() {
    float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 4096; int blocks = 148 * 4, threads = 512;
    for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k_lds<<<blocks, threads>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)blocks * threads / 32 * iters * 8; // warp-level LDS.128
    printf("LDS.128: %.3f ms, %.2f warp-instr/clk/SM (at 1.965 GHz)\n", ms, n / (ms * 1e-3) / 148 / 1.965e9);
    cudaEventRecord(e0); k_shfl<<<blocks, threads>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    n = (double)blocks * threads / 32 * iters * 8 * 4; // warp-level SHFL
    printf("SHFL.32: %.3f ms, %.2f warp-instr/clk/SM\n", ms, n / (ms * 1e-3) / 148 / 1.965e9);
    cudaEventRecord(e0); k_mix<<<blocks, threads>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("mix (8 LDS.128 + 32 SHFL per iteration): %.3f ms (sum of the two alone would be ~8.6 ms)\n", ms);
    }
    return 0;
}
