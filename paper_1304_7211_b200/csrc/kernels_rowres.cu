// kernels_rowres.cu -- row-resident Richardson-Lucy for horizontal line PSFs
// (uniform 1 x M box with dy = 0: Box1dSliding / Box1dCumulated,
// convolve.hpp:217-280; configs 0 and 4b).
//
// With a single-row PSF at dy = 0 every image row evolves independently
// under RL (replicate clamping only acts along the row), so a CTA can keep
// its rows' u, f and q in shared memory for ALL iterations: HBM traffic is
// one read of f and one write of u per run (8 B/px instead of 24 B/px per
// iteration of the two-pass engines).  Per iteration and thread (PT = 4 or 8
// adjacent columns):
//   1. window of 8+M-1 u values (clamped at the row ends) -> register prefix
//      sums (restarting per thread: fp32 cancellation ~1e-7 relative) ->
//      v = sum/M -> q = f / max(v, eps) into shared memory;      __syncthreads
//   2. window of q under the adjoint line (offsets negated) -> c ->
//      u' = max(c u, 0), max|du| and the NaN checksum;            __syncthreads
// Per-iteration max|du| / NaN are reduced per CTA in shared memory and
// published with one atomic per (CTA, iteration) only when they raise the
// running maximum.  Images are batches of rows (batch x H rows of W).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace fdg {
namespace {


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
    unsigned long long* tend;  // [iters] %globaltimer at the end of iteration k (max over CTAs)
    unsigned long long* tbegin;  // start stamp of the run (block 0)
    unsigned long long* tdur;    // [iters] sum over CTAs of the iteration's duration (ns)
};

template <int N>
__device__ __forceinline__ float tsum(const float* v) {
    if constexpr (N == 1) {
        return v[0];
    } else {
        return tsum<N / 2>(v) + tsum<N - N / 2>(v + N / 2);
    }
}

// out[i] = sum_{k<M} row[clamp(xb + i + off + k)], i < PT (M >= PT).
// Interior threads read aligned float4 chunks (the window start sits at
// OFF4 = off & 3 inside its chunk, xb being a multiple of 4); threads at the
// row ends read clamped scalars.  Sums are formed without subtraction:
// shared middle (balanced tree) + left suffix + right prefix, dependency
// depth ~log2(M) + PT instead of a length-M chain.
template <int M, int OFF4, int PT>
__device__ __forceinline__ void window_sums(const float* row, int W, int xb, int off, float (&out)[PT]) {
    constexpr int NW = PT + M - 1;
    constexpr int NCH = (OFF4 + NW - 1) / 4 + 1;
    float v[4 * NCH];
    const int lo = xb + off;
    const int c0 = lo - OFF4;  // multiple of 4
    if (c0 >= 0 && c0 + 4 * NCH <= W) {
        const float4* p = reinterpret_cast<const float4*>(row + c0);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const float4 q = p[c];
            v[4 * c] = q.x;
            v[4 * c + 1] = q.y;
            v[4 * c + 2] = q.z;
            v[4 * c + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < NW; ++k) v[OFF4 + k] = row[clampi(lo + k, 0, W - 1)];
    }
    const float* w = v + OFF4;
    const float mid = tsum<M - PT + 1>(w + PT - 1);  // taps common to all PT windows
    float left = 0.f, right = 0.f;
    float L[PT], Rr[PT];
#pragma unroll
    for (int i = PT - 2; i >= 0; --i) {  // L[i] = sum_{k=i}^{PT-2} w[k]
        left += w[i];
        L[i] = left;
    }
    L[PT - 1] = 0.f;
    Rr[0] = 0.f;
#pragma unroll
    for (int i = 1; i < PT; ++i) {  // Rr[i] = sum_{k=M}^{M+i-1} w[k]
        right += w[M + i - 1];
        Rr[i] = right;
    }
#pragma unroll
    for (int i = 0; i < PT; ++i) out[i] = (L[i] + mid) + Rr[i];
}

// PT columns per thread: 4 (rows up to 1024 px: more threads per row) or 8
template <int M, int O1, int O2, int PT>
__global__ void __launch_bounds__(256, 2) k_rowres(const RowResArgs a) {
    constexpr int NV4 = PT / 4;  // own columns as float4 chunks
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
    unsigned long long* stime = reinterpret_cast<unsigned long long*>(snan + a.iters);  // iters
    const int grow = blockIdx.x * R + rloc;  // global row id (batch * H)
    const bool active = rloc < R && grow < a.rows_total;
    long long goff = 0;
    if (active) {
        const int b = grow / a.H, y = grow - b * a.H;
        goff = (long long)b * a.bstride + (long long)y * a.pitch;
    }
    const unsigned long long t0 = globaltimer();
    if (a.tbegin && blockIdx.x == 0 && threadIdx.x == 0) *a.tbegin = t0;
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
        // own PT columns move as float4 chunks (scalar smem accesses at a
        // PT-float lane stride would conflict PT-way)
        const bool vec = xb + PT <= W;
        if (active) {
            float v[PT];
            window_sums<M, O1, PT>(ru, W, xb, off1, v);
            float fv[PT], qv[PT];
            if (vec) {
#pragma unroll
                for (int c = 0; c < NV4; ++c) {
                    const float4 a0 = *reinterpret_cast<const float4*>(rf + xb + 4 * c);
                    fv[4 * c] = a0.x, fv[4 * c + 1] = a0.y, fv[4 * c + 2] = a0.z, fv[4 * c + 3] = a0.w;
                }
            } else {
#pragma unroll
                for (int i = 0; i < PT; ++i) fv[i] = xb + i < W ? rf[xb + i] : 1.f;
            }
#pragma unroll
            for (int i = 0; i < PT; ++i) {
                const float d = v[i] * a.inv_m;
                qv[i] = div_fast(fv[i], d < a.eps ? a.eps : d);
            }
            if (vec) {
#pragma unroll
                for (int c = 0; c < NV4; ++c)
                    *reinterpret_cast<float4*>(rq + xb + 4 * c) =
                        make_float4(qv[4 * c], qv[4 * c + 1], qv[4 * c + 2], qv[4 * c + 3]);
            } else {
#pragma unroll
                for (int i = 0; i < PT; ++i)
                    if (xb + i < W) rq[xb + i] = qv[i];
            }
        }
        __syncthreads();
        float maxd = 0.f, csum = 0.f;
        if (active) {
            float c[PT];
            window_sums<M, O2, PT>(rq, W, xb, off2, c);
            float uv[PT];
            if (vec) {
#pragma unroll
                for (int c4 = 0; c4 < NV4; ++c4) {
                    const float4 a0 = *reinterpret_cast<const float4*>(ru + xb + 4 * c4);
                    uv[4 * c4] = a0.x, uv[4 * c4 + 1] = a0.y, uv[4 * c4 + 2] = a0.z, uv[4 * c4 + 3] = a0.w;
                }
            } else {
#pragma unroll
                for (int i = 0; i < PT; ++i) uv[i] = xb + i < W ? ru[xb + i] : 0.f;
            }
#pragma unroll
            for (int i = 0; i < PT; ++i) {
                float value = c[i] * a.inv_m * uv[i];
                if (a.clamp && value < 0.f) value = 0.f;
                if (xb + i < W) {
                    maxd = fmaxf(maxd, fabsf(value - uv[i]));
                    csum += value;
                }
                uv[i] = value;
            }
            if (vec) {
#pragma unroll
                for (int c4 = 0; c4 < NV4; ++c4)
                    *reinterpret_cast<float4*>(ru + xb + 4 * c4) =
                        make_float4(uv[4 * c4], uv[4 * c4 + 1], uv[4 * c4 + 2], uv[4 * c4 + 3]);
            } else {
#pragma unroll
                for (int i = 0; i < PT; ++i)
                    if (xb + i < W) ru[xb + i] = uv[i];
            }
        }
        const unsigned bits = __reduce_max_sync(0xffffffffu, __float_as_uint(maxd));
        const int nan = __reduce_or_sync(0xffffffffu, (int)isnan(csum));
        if ((threadIdx.x & 31) == 0) {
            if (bits) atomicMax(reinterpret_cast<unsigned*>(smax) + it, bits);
            if (nan) snan[it] = 1;
        }
        __syncthreads();
        if (threadIdx.x == 0) stime[it] = globaltimer();  // this CTA's end of iteration it
    }
    if (active) {
        for (int i = 0; i < PT; ++i) {
            const int x = xb + i;
            if (x < W) a.u[goff + x] = ru[x];
        }
    }
    __syncthreads();
    // publish per-iteration maxima: only values that raise the running maximum
    for (int k = threadIdx.x; k < a.iters; k += blockDim.x) {
        const unsigned b = reinterpret_cast<unsigned*>(smax)[k];
        if (a.maxchange && b > a.maxchange[k]) atomicMax(a.maxchange + k, b);
        if (a.nanflag && snan[k]) atomicOr(a.nanflag + k, 1);
        if (a.tend) atomicMax(a.tend + k, stime[k]);
        // CTAs run their iterations out of phase (several waves): the
        // per-iteration share of the run is the summed per-CTA duration
        if (a.tdur) atomicAdd(a.tdur + k, stime[k] - (k ? stime[k - 1] : t0));
    }
}

// anchor-centred lines (makeLinePsf): forward window starts at -(M/2), the
// adjoint's at -(M - 1 - M/2)
constexpr int o1_of(int m) { return (-(m / 2)) & 3; }
constexpr int o2_of(int m) { return (-(m - 1 - m / 2)) & 3; }

template <int M, int PT>
cudaError_t launch_m(const RowResArgs& a, int threads, size_t smem, int blocks, cudaStream_t st) {
    constexpr int O1 = o1_of(M), O2 = o2_of(M);
    cudaError_t err = smem_attr<k_rowres<M, O1, O2, PT>>();
    if (err != cudaSuccess) return err;
    k_rowres<M, O1, O2, PT><<<blocks, threads, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

// anchor-centred horizontal lines of 5 .. 31 px (8 columns per thread -- rows
// wider than 1024 px -- need a window of at least 9)
bool rowres_supported(int mx, int my, int min_dx, int min_dy, int W) {
    // one row per <= 256-thread CTA: W <= 256 x 8 columns
    return my == 1 && min_dy == 0 && min_dx == -(mx / 2) && mx <= 31 && mx >= (W <= 1024 ? 5 : 9) && W >= 1 &&
           W <= 2048;
}

namespace {
// the instantiation for line length mx, M = 5 .. 31
template <int M>
cudaError_t launch_len(int mx, int PT, const RowResArgs& a, int threads, size_t smem, int blocks, cudaStream_t st) {
    if (mx == M) {
        if (PT == 4) return launch_m<M, 4>(a, threads, smem, blocks, st);
        if constexpr (M >= 9) return launch_m<M, 8>(a, threads, smem, blocks, st);
        return cudaErrorInvalidValue;
    }
    if constexpr (M < 31) return launch_len<M + 1>(mx, PT, a, threads, smem, blocks, st);
    return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t launch_rowres(int mx, int min_dx, float inv_m, const float* f, float* u, int pitch, int W, int H,
                          int batch, long long bstride, int iters, float eps, int clamp, unsigned* maxchange,
                          int* nanflag, unsigned long long* tend, unsigned long long* tbegin, unsigned long long* tdur,
                          cudaStream_t st) {
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
    a.tend = tend;
    a.tbegin = tbegin;
    a.tdur = tdur;
    // 4 columns per thread when a row fits 256 threads (more warps per row:
    // config 0 212k -> 264k Mpx*it/s), else 8
    const int PT = W <= 1024 ? 4 : 8;
    const int nthr_row = (W + PT - 1) / PT;
    // up to 256 threads per CTA, but at least ~3 CTAs per SM: small images
    // (config 0: 512 rows) otherwise leave SMs idle (4 rows/CTA = 128 CTAs on
    // 148 SMs: 201k Mpx*it/s; 1 row/CTA: 212k)
    static const int sms = [] {
        int dev = 0, n = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n;
    }();
    int rows_per_cta = nthr_row >= 256 ? 1 : 256 / nthr_row;
    rows_per_cta = std::max(1, std::min(rows_per_cta, a.rows_total / (3 * sms)));
    a.rows_per_cta = rows_per_cta;
    const int threads = ((rows_per_cta * nthr_row + 31) / 32) * 32;
    if (threads > 1024) return cudaErrorInvalidConfiguration;
    const int wp = (W + 3) & ~3;
    const size_t smem = sizeof(float) * (3 * (size_t)rows_per_cta * wp + iters) + sizeof(int) * iters +
                        sizeof(unsigned long long) * iters;
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    const int blocks = (a.rows_total + rows_per_cta - 1) / rows_per_cta;
    return launch_len<5>(mx, PT, a, threads, smem, blocks, st);
}

}  // namespace fdg
