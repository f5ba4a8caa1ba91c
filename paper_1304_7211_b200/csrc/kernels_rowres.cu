// kernels_rowres.cu -- row-resident Richardson-Lucy for horizontal line PSFs
// (uniform 1 x M box with dy = 0: Box1dSliding / Box1dCumulated,
// convolve.hpp:217-280; configs 0 and 4b).
//
// With a single-row PSF at dy = 0 every image row evolves independently
// under RL (replicate clamping only acts along the row), so a CTA can keep
// its rows' u, f and q in shared memory for ALL iterations: HBM traffic is
// one read of f and one write of u per run (8 B/px instead of 24 B/px per
// iteration of the two-pass engines).  Per iteration and thread (8 adjacent
// columns):
//   1. window of 8+M-1 u values (clamped at the row ends) -> register prefix
//      sums (restarting per thread: fp32 cancellation ~1e-7 relative) ->
//      v = sum/M -> q = f / max(v, eps) into shared memory;      __syncthreads
//   2. window of q under the adjoint line (offsets negated) -> c ->
//      u' = max(c u, 0), max|du| and the NaN checksum;            __syncthreads
// Per-iteration max|du| / NaN are reduced per CTA in shared memory and
// published with one atomic per (CTA, iteration) only when they raise the
// running maximum.  Images are batches of rows (batch x H rows of W).
#include "common.cuh"

namespace fdg {
namespace {

constexpr int PT = 8;  // columns per thread

struct RowResArgs {
    const float* f;
    float* u;
    int pitch, W, rows_total, H;  // rows_total = batch * H
    long long bstride;
    int rows_per_cta, iters;
    int min_dx;                    // forward line offsets: [min_dx, min_dx + M - 1]
    float inv_m, eps;
    int clamp;
    unsigned* maxchange;  // [iters] float bits
    int* nanflag;         // [iters]
};

template <int M>
__device__ __forceinline__ void window_sums(const float* row, int W, int xb, int off, float (&out)[PT]) {
    // out[i] = sum_{k<M} row[clamp(xb + i + off + k)]
    constexpr int NW = PT + M - 1;
    float w[NW];
    const int lo = xb + off;
    if (lo >= 0 && lo + NW - 1 <= W - 1) {
#pragma unroll
        for (int k = 0; k < NW; ++k) w[k] = row[lo + k];
    } else {
#pragma unroll
        for (int k = 0; k < NW; ++k) w[k] = row[clampi(lo + k, 0, W - 1)];
    }
    float p[NW];
    p[0] = w[0];
#pragma unroll
    for (int k = 1; k < NW; ++k) p[k] = p[k - 1] + w[k];
    out[0] = p[M - 1];
#pragma unroll
    for (int i = 1; i < PT; ++i) out[i] = p[i + M - 1] - p[i - 1];
}

template <int M>
__global__ void __launch_bounds__(256) k_rowres(const RowResArgs a) {
    extern __shared__ __align__(16) float sm[];
    const int W = a.W;
    const int wp = (W + 3) & ~3;
    const int nthr_row = (W + PT - 1) / PT;
    const int rloc = threadIdx.x / nthr_row;  // row within the CTA
    const int chunk = threadIdx.x - rloc * nthr_row;
    const int R = a.rows_per_cta;
    float* su = sm;                 // R x wp
    float* sf = su + R * wp;        // R x wp
    float* sq = sf + R * wp;        // R x wp
    float* smax = sq + R * wp;      // iters
    int* snan = reinterpret_cast<int*>(smax + a.iters);
    const int grow = blockIdx.x * R + rloc;  // global row id (batch * H)
    const bool active = rloc < R && grow < a.rows_total;
    long long goff = 0;
    if (active) {
        const int b = grow / a.H, y = grow - b * a.H;
        goff = (long long)b * a.bstride + (long long)y * a.pitch;
    }
    for (int k = threadIdx.x; k < a.iters; k += blockDim.x) {
        smax[k] = 0.f;
        snan[k] = 0;
    }
    // load f (u0 = f)
    float* ru = su + rloc * wp;
    float* rf = sf + rloc * wp;
    float* rq = sq + rloc * wp;
    const int xb = chunk * PT;
    if (active) {
        for (int i = 0; i < PT; ++i) {
            const int x = xb + i;
            if (x < W) {
                const float v = a.f[goff + x];
                rf[x] = v;
                ru[x] = v;
            }
        }
    }
    __syncthreads();
    const int off1 = a.min_dx;               // forward window start
    const int off2 = -(a.min_dx + M - 1);    // adjoint window start (offsets negated)
    for (int it = 0; it < a.iters; ++it) {
        if (active) {
            float v[PT];
            window_sums<M>(ru, W, xb, off1, v);
#pragma unroll
            for (int i = 0; i < PT; ++i) {
                const int x = xb + i;
                if (x < W) {
                    const float d = v[i] * a.inv_m;
                    rq[x] = div_fast(rf[x], d < a.eps ? a.eps : d);
                }
            }
        }
        __syncthreads();
        float maxd = 0.f, csum = 0.f;
        if (active) {
            float c[PT];
            window_sums<M>(rq, W, xb, off2, c);
#pragma unroll
            for (int i = 0; i < PT; ++i) {
                const int x = xb + i;
                if (x < W) {
                    const float u = ru[x];
                    float value = c[i] * a.inv_m * u;
                    if (a.clamp && value < 0.f) value = 0.f;
                    maxd = fmaxf(maxd, fabsf(value - u));
                    csum += value;
                    ru[x] = value;
                }
            }
        }
        const unsigned bits = __reduce_max_sync(0xffffffffu, __float_as_uint(maxd));
        const int nan = __reduce_or_sync(0xffffffffu, (int)isnan(csum));
        if ((threadIdx.x & 31) == 0) {
            if (bits) atomicMax(reinterpret_cast<unsigned*>(smax) + it, bits);
            if (nan) snan[it] = 1;
        }
        __syncthreads();
    }
    if (active) {
        for (int i = 0; i < PT; ++i) {
            const int x = xb + i;
            if (x < W) a.u[goff + x] = ru[x];
        }
    }
    // publish per-iteration maxima: only values that raise the running maximum
    for (int k = threadIdx.x; k < a.iters; k += blockDim.x) {
        const unsigned b = reinterpret_cast<unsigned*>(smax)[k];
        if (a.maxchange && b > a.maxchange[k]) atomicMax(a.maxchange + k, b);
        if (a.nanflag && snan[k]) atomicOr(a.nanflag + k, 1);
    }
}

template <int M>
cudaError_t launch_m(const RowResArgs& a, int threads, size_t smem, int blocks, cudaStream_t st) {
    cudaError_t err = smem_attr<k_rowres<M>>();
    if (err != cudaSuccess) return err;
    k_rowres<M><<<blocks, threads, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

bool rowres_supported(int mx, int my, int min_dy, int W) {
    return my == 1 && min_dy == 0 && (mx == 15 || mx == 31 || mx == 9 || mx == 17) && W >= 1 && W <= 8192;
}

cudaError_t launch_rowres(int mx, int min_dx, float inv_m, const float* f, float* u, int pitch, int W, int H,
                          int batch, long long bstride, int iters, float eps, int clamp, unsigned* maxchange,
                          int* nanflag, cudaStream_t st) {
    RowResArgs a;
    a.f = f;
    a.u = u;
    a.pitch = pitch;
    a.W = W;
    a.H = H;
    a.rows_total = H * batch;
    a.bstride = bstride;
    a.iters = iters;
    a.min_dx = min_dx;
    a.inv_m = inv_m;
    a.eps = eps;
    a.clamp = clamp;
    a.maxchange = maxchange;
    a.nanflag = nanflag;
    const int nthr_row = (W + PT - 1) / PT;
    const int rows_per_cta = nthr_row >= 256 ? 1 : 256 / nthr_row;
    a.rows_per_cta = rows_per_cta;
    const int threads = ((rows_per_cta * nthr_row + 31) / 32) * 32;
    if (threads > 1024) return cudaErrorInvalidConfiguration;
    const int wp = (W + 3) & ~3;
    const size_t smem = sizeof(float) * (3 * (size_t)rows_per_cta * wp + iters) + sizeof(int) * iters;
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    const int blocks = (a.rows_total + rows_per_cta - 1) / rows_per_cta;
    switch (mx) {
        case 9: return launch_m<9>(a, threads, smem, blocks, st);
        case 15: return launch_m<15>(a, threads, smem, blocks, st);
        case 17: return launch_m<17>(a, threads, smem, blocks, st);
        case 31: return launch_m<31>(a, threads, smem, blocks, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace fdg
