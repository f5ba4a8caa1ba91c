// kernels_spanr.cu -- "spans" engine for ANY row-convex uniform PSF
// (GenericBox, convolve.hpp:177-212): the span table {dy, xMin, xMax}
// (asUniformConvex, psf.hpp:444-464) travels in the kernel parameter space,
// so every UniformConvexPsf with <= 64 rows and xMax - xMin extents
// (max_dx - min_dx) <= 64 runs here -- the paper's discs of any diameter,
// diagonals and oblique lines at any angle.  The two BASELINE shapes keep
// their compile-time kernels (kernels_spans.cu); anything larger falls back
// to the per-tap engine.
//
// The reference evaluates a row's window sum once at x = 0 and then slides
// it along the row, sum += p[x + xMax] - p[x - 1 + xMin] per span: 2 M_y
// operations per pixel.  A long fp32 slide drifts (SURVEY 7 hard part 1),
// so the B200 form keeps the 2-operations-per-span cost but bounds the
// accumulation length:
//
//   CTA = 8 warps over a 128 x 32 output tile: warp (gx, gy) owns columns
//   [32 gx, 32 gx + 32) x rows [16 gy, 16 gy + 16), one column and 16 rows
//   per lane.
//   1. The replicate-clamped input tile + halo (32 + NR - 1 rows x
//      128 + XL + XR columns) is staged in shared memory with 4-byte
//      cp.async copies (odd row pitch).
//   2. Each column group g gets its own exclusive row prefix table over the
//      only columns its 32 lanes ever read, [32 g - XL, 32 g + 31 + XR]:
//      T_g[t][k] = sum_{i<k} in[t][32 g - XL + i]  (<= 97 terms: the
//      prefix magnitude, hence the cancellation error of a difference, stays
//      that of a ~100-pixel sum).  One lane per (row, group) scans
//      sequentially; odd pitches keep the lanes on distinct banks.
//   3. Output (x, y) adds, for each PSF row r in dy order (one partial per
//      PSF row, as the other engines), T[y + r][x' + xMax_r + 1] -
//      T[y + r][x' + xMin_r]: two conflict-free LDS and two FADD per span,
//      the span bounds uniform parameter-space loads.  Spans of 1 or 2
//      pixels read the tile itself (no more loads, and exact for one tap).
//   4. Fused RL epilogue (quotient / update + max|du| + NaN) as every engine.
#include <algorithm>

#include "common.cuh"

namespace fdg {
namespace {

constexpr int SR_V = 16;            // output rows per lane
constexpr int SR_TH = 2 * SR_V;     // tile rows
constexpr int SR_TW = 128;          // tile columns
constexpr int SR_MAXR = 64;         // PSF rows
constexpr int SR_MAXX = 64;         // max_dx - min_dx

struct SpanTab {
    int nr, mindy, xl, xr;
    int2 lohi[SR_MAXR];  // xMin, xMax per row r = dy - mindy
};

struct SpanRArgs {
    const float* in;
    const float* aux;
    float* out;
    int pitch, W;
    int y0, y1, ylo, yhi;
    long long bstride;
    float scale, eps;
    int clamp;
    int tr, tcp, sl, slp;  // tile rows, raw pitch (odd), segment length, table pitch (odd)
    unsigned* maxchange;
    int* nanflag;
    unsigned long long* tend;
};

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int MODE>
__device__ __forceinline__ float epi_r(float v, float x, float eps, int clamp, float& maxd, float& csum) {
    if (MODE == EPI_STORE) return v;
    if (MODE == EPI_QUOT) return div_fast(x, v < eps ? eps : v);
    float value = v * x;
    if (clamp && value < 0.f) value = 0.f;
    maxd = fmaxf(maxd, fabsf(value - x));
    csum += value;
    return value;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_spanr(const SpanRArgs a, const __grid_constant__ SpanTab tb) {
    extern __shared__ __align__(16) float smr[];
    const int tr = a.tr, tcp = a.tcp, sl = a.sl, slp = a.slp;
    float* raw = smr;                     // tr x tcp
    float* tab = smr + tr * tcp;          // 4 groups x tr x slp
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = blockIdx.x * SR_TW;
    const int yt0 = a.y0 + blockIdx.y * SR_TH;
    const long long img = (long long)blockIdx.z * a.bstride;
    const float* src = a.in + img;
    const int tc = SR_TW + tb.xl + tb.xr;
    const int wm1 = a.W - 1;

    // 1. stage the clamped tile (every copy in flight, no register round trip)
    for (int t = warp; t < tr; t += 8) {
        const float* rp = src + (long long)clampi(yt0 + tb.mindy + t, a.ylo, a.yhi) * a.pitch;
        float* dst = raw + t * tcp;
        for (int c = lane; c < tc; c += 32) cp_async4(dst + c, rp + clampi(x0 - tb.xl + c, 0, wm1));
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();

    // 2. per column group exclusive row prefixes; lane = one (row, group)
    const int chunks = (tr + 31) >> 5;
    for (int j = warp; j < 4 * chunks; j += 8) {
        const int g = j / chunks;
        const int t = ((j - g * chunks) << 5) + lane;
        if (t < tr) {
            const float* rp = raw + t * tcp + 32 * g;
            float* tp = tab + (g * tr + t) * slp;
            float s = 0.f;
            tp[0] = 0.f;
#pragma unroll 4
            for (int k = 0; k < sl; ++k) {
                s += rp[k];
                tp[k + 1] = s;
            }
        }
    }
    __syncthreads();

    // 3. span differences: output (x, yo) accumulates PSF rows in dy order
    const int gx = warp & 3, gy = warp >> 2;
    float acc[SR_V];
#pragma unroll
    for (int o = 0; o < SR_V; ++o) acc[o] = 0.f;
    const float* tg = tab + (gx * tr + gy * SR_V) * slp + lane + tb.xl;
    const float* rg = raw + gy * SR_V * tcp + 32 * gx + lane + tb.xl;
    for (int r = 0; r < tb.nr; ++r) {
        const int2 s = tb.lohi[r];
        if (s.y - s.x < 2) {
            // 1- and 2-pixel spans (lines, diagonals, disc caps) straight from
            // the tile: exact for a single tap (identity PSF bit-identical)
            const float* p = rg + r * tcp + s.x;
            if (s.y == s.x) {
#pragma unroll
                for (int o = 0; o < SR_V; ++o) acc[o] += p[o * tcp];
            } else {
#pragma unroll
                for (int o = 0; o < SR_V; ++o) acc[o] += p[o * tcp] + p[o * tcp + 1];
            }
            continue;
        }
        const float* pa = tg + r * slp + s.y + 1;
        const float* pb = tg + r * slp + s.x;
#pragma unroll
        for (int o = 0; o < SR_V; ++o) acc[o] += pa[o * slp] - pb[o * slp];
    }

    // 4. fused epilogue
    const int x = x0 + 32 * gx + lane;
    float maxd = 0.f, csum = 0.f;
    if (x < a.W) {
        const int yb = yt0 + gy * SR_V;
#pragma unroll
        for (int o = 0; o < SR_V; ++o) {
            const int y = yb + o;
            if (y >= a.y1) break;
            const long long idx = img + (long long)y * a.pitch + x;
            const float xa = MODE == EPI_STORE ? 0.f : __ldg(a.aux + idx);
            a.out[idx] = epi_r<MODE>(acc[o] * a.scale, xa, a.eps, a.clamp, maxd, csum);
        }
    }
    if (MODE == EPI_UPDATE && a.maxchange) {
        const unsigned bits = __reduce_max_sync(0xffffffffu, __float_as_uint(maxd));
        const int nan = __reduce_or_sync(0xffffffffu, (int)isnan(csum));
        if (lane == 0) {
            if (bits) atomicMax(a.maxchange, bits);
            if (nan) atomicOr(a.nanflag, 1);
            stamp_end(a.tend);
        }
    }
}

template <int MODE>
cudaError_t launch_r(const SpanRArgs& a, const SpanTab& tb, dim3 grid, size_t smem, cudaStream_t st) {
    cudaError_t err = smem_attr<k_spanr<MODE>>();
    if (err != cudaSuccess) return err;
    k_spanr<MODE><<<grid, 256, smem, st>>>(a, tb);
    return cudaGetLastError();
}

}  // namespace

bool spanr_supported(const DevPsf& p) {
    if (p.nrows < 1 || p.nrows > SR_MAXR || (int)p.h_span.size() != 2 * p.nrows) return false;
    int xl = 0, xr = 0;
    for (int r = 0; r < p.nrows; ++r) {
        xl = std::max(xl, -p.h_span[2 * r]);
        xr = std::max(xr, p.h_span[2 * r + 1]);
    }
    return xl + xr <= SR_MAXX;
}

static size_t spanr_smem(const DevPsf& p, int* tr, int* tcp, int* sl, int* slp, int* xl, int* xr) {
    int l = 0, r_ = 0;
    for (int r = 0; r < p.nrows; ++r) {
        l = std::max(l, -p.h_span[2 * r]);
        r_ = std::max(r_, p.h_span[2 * r + 1]);
    }
    *xl = l;
    *xr = r_;
    *tr = SR_TH + p.nrows - 1;
    *tcp = (SR_TW + l + r_) | 1;
    *sl = 32 + l + r_;
    *slp = (*sl + 1) | 1;
    return sizeof(float) * ((size_t)*tr * *tcp + (size_t)4 * *tr * *slp);
}

cudaError_t launch_spanr(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st) {
    if (!spanr_supported(p)) return cudaErrorNotSupported;
    SpanTab tb;
    SpanRArgs a;
    const size_t smem = spanr_smem(p, &a.tr, &a.tcp, &a.sl, &a.slp, &tb.xl, &tb.xr);
    tb.nr = p.nrows;
    tb.mindy = p.min_dy;
    for (int r = 0; r < p.nrows; ++r) tb.lohi[r] = make_int2(p.h_span[2 * r], p.h_span[2 * r + 1]);
    a.in = g.in;
    a.aux = e.aux;
    a.out = g.out;
    a.pitch = g.pitch;
    a.W = g.W;
    a.y0 = g.y0;
    a.y1 = g.y1;
    a.ylo = g.ylo;
    a.yhi = g.yhi;
    a.bstride = g.bstride;
    a.scale = p.scale;
    a.eps = e.eps;
    a.clamp = e.clamp;
    a.maxchange = e.maxchange;
    a.nanflag = e.nanflag;
    a.tend = e.tend;
    const int rows = g.y1 - g.y0;
    if (rows <= 0) return cudaSuccess;
    dim3 grid((g.W + SR_TW - 1) / SR_TW, (rows + SR_TH - 1) / SR_TH, g.batch);
    switch (e.mode) {
        case EPI_STORE: return launch_r<EPI_STORE>(a, tb, grid, smem, st);
        case EPI_QUOT: return launch_r<EPI_QUOT>(a, tb, grid, smem, st);
        case EPI_UPDATE: return launch_r<EPI_UPDATE>(a, tb, grid, smem, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace fdg
