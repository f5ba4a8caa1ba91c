// bw_probe.cu -- microbenchmark of the row-streaming pattern used by the box
// engine: how much HBM bandwidth can a TMA bulk-copy ring (one producer
// thread, S stages, row segments of SEGB bytes) sustain, versus plain
// coalesced float4 loads?  Throwaway measurement tool (not product code).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int S, int NT, int R>
__global__ void __launch_bounds__(NT + 32) k_ring(const float* in, float* out, int W, int H, int band, int segf) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = (uint64_t*)sm;
    uint64_t* empty = full + S;
    float* ring = (float*)(sm + 1024);
    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * segf;
    const int y0 = blockIdx.y * band;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(NT / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (tid >= NT) {
        if (tid == NT) {
            for (int i = 0; i < band / R; ++i) {
                const int s = i % S;
                if (i >= S) {
                    unsigned par = ((i / S) - 1) & 1;
                    asm volatile("{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}" ::"r"(su32(&empty[s])), "r"(par) : "memory");
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(segf * 4 * R) : "memory");
                for (int r = 0; r < R; ++r)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(ring + (s * R + r) * segf)), "l"(in + (size_t)(y0 + i * R + r) * W + x0), "r"(segf * 4), "r"(su32(&full[s])) : "memory");
            }
        }
        return;
    }
    float acc = 0.f;
    for (int i = 0; i < band / R; ++i) {
        const int s = i % S;
        unsigned par = (i / S) & 1;
        asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}" ::"r"(su32(&full[s])), "r"(par) : "memory");
        for (int c = tid; c < R * segf / 4; c += NT) {
            float4 v = ((float4*)(ring + s * R * segf))[c];
            acc += v.x + v.y + v.z + v.w;
        }
        __syncwarp();
        if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
    if (acc == 123.f) out[0] = acc;
}

__global__ void k_ldg(const float4* in, float* out, size_t n4) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = in[i];
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 123.f) out[0] = acc;
}

template <int S, int NT, int R = 1>
float run_ring(const float* in, float* out, int W, int H, int segf, int band) {
    dim3 grid(W / segf, H / band);
    size_t smem = 1024 + (size_t)S * R * segf * 4;
    cudaFuncSetAttribute(k_ring<S, NT, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_ring<S, NT, R><<<grid, NT + 32, smem>>>(in, out, W, H, band, segf);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k_ring<S, NT, R><<<grid, NT + 32, smem>>>(in, out, W, H, band, segf);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e) printf("err %s\n", cudaGetErrorString(e));
    return (float)W * H * 4 * 5 / (ms * 1e-3) / 1e9;
}

int main() {
    const int W = 16384, H = 16384;
    float *in, *out;
    cudaMalloc(&in, (size_t)W * H * 4);
    cudaMalloc(&out, 64);
    cudaMemset(in, 0, (size_t)W * H * 4);
    {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        k_ldg<<<148 * 8, 256>>>((float4*)in, out, (size_t)W * H / 4);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k_ldg<<<148 * 8, 256>>>((float4*)in, out, (size_t)W * H / 4);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("ldg read-only: %.0f GB/s\n", (double)W * H * 4 * 5 / (ms * 1e-3) / 1e9);
    }
#define P(S_, NT_, R_, SEG, BAND) printf("ring S=%d NT=%d R=%d seg=%d floats band=%d: %.0f GB/s\n", S_, NT_, R_, SEG, BAND, run_ring<S_, NT_, R_>(in, out, W, H, SEG, BAND))
    P(8, 128, 1, 512, 256);
    P(16, 128, 1, 512, 256);
    P(24, 128, 1, 512, 256);
    P(32, 128, 1, 512, 256);
    P(8, 128, 2, 512, 256);
    P(8, 128, 4, 512, 256);
    P(4, 128, 4, 512, 256);
    P(6, 128, 4, 512, 256);
    P(16, 128, 2, 512, 256);
    P(8, 128, 1, 1024, 256);
    P(16, 128, 1, 1024, 256);
    P(8, 256, 1, 1024, 256);
    P(8, 256, 2, 1024, 256);
    P(4, 512, 1, 4096, 256);
    P(8, 128, 1, 2048, 256);
    return 0;
}
