// spans_jit.cu -- runtime specialisation of the span-table tile kernel.
//
// The tile kernel k_spant (kernels_spans.cu) is fast because the span
// table is compile-time: every span bound becomes a static register index
// into the thread's window prefix.  Any other row-convex PSF runs the
// runtime-table kernel (kernels_spanr.cu, two shared loads per span per
// pixel) -- unless this module compiles the tile kernel for its table at
// plan time with NVRTC (sm_100a CUBIN, cached per table and device for the
// life of the process) and launches it through the driver API.  Both
// libraries are resolved at run time (dlopen libnvrtc.so.12;
// cudaGetDriverEntryPoint for the driver calls), so libfdgpu has no extra
// link dependency; any failure (no NVRTC, compile error) leaves the plan on
// the runtime-table kernel.  fdg_set_option("spans_jit", 0) disables it.
#include <cuda.h>
#include <dlfcn.h>

#include <atomic>
#include <cstdio>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "common.cuh"

namespace fdg {
namespace {

// ---- device source (compiled by NVRTC with a generated `struct SH` in front)
const char* kJitSource = R"JIT(
struct JitArgs {
    const float* in;
    const float* aux;
    float* out;
    int pitch, W;
    int y0, y1, ylo, yhi;
    long long bstride;
    float scale, eps;
    int clamp;
    unsigned* maxchange;
    int* nanflag;
    unsigned long long* tend;
};
template <int NT>
struct Ext {
    static constexpr int xl() {
        int m = 0;
        for (int r = 0; r < SH::NR; ++r) m = SH::LO(r) < -m ? -SH::LO(r) : m;
        return m;
    }
    static constexpr int xr() {
        int m = 0;
        for (int r = 0; r < SH::NR; ++r) m = SH::HI(r) > m ? SH::HI(r) : m;
        return m;
    }
    static constexpr int XL = xl(), XR = xr();
    static constexpr int HL = (XL + 3) / 4 * 4, HR = (XR + 3) / 4 * 4;
    static constexpr int OFF = HL - XL;
    static constexpr int NWIN = 4 + XL + XR;
    static constexpr int NCH = (OFF + NWIN - 1) / 4 + 1;
};
__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float div_fast(float f, float d) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
    const float q0 = f * r;
    const float e = fmaf(-d, q0, f);
    return fmaf(e, r, q0);
}
template <int MODE>
__device__ __forceinline__ float epi1(float v, float x, float eps, int clamp, float& maxd, float& csum) {
    if (MODE == 0) return v;
    if (MODE == 1) return div_fast(x, v < eps ? eps : v);
    float value = v * x;
    if (clamp && value < 0.f) value = 0.f;
    maxd = fmaxf(maxd, fabsf(value - x));
    csum += value;
    return value;
}
template <int MODE, int V, int NTY>
__device__ void spant(const JitArgs& a) {
    using E = Ext<32>;
    constexpr int NR = SH::NR;
    constexpr int TW = 128, TH = V * NTY, TR = TH + NR - 1, TC = TW + E::HL + E::HR, TCP = TC + 4;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* tile = reinterpret_cast<float*>(smem_raw);
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int x0 = blockIdx.x * TW;
    const int yt0 = a.y0 + blockIdx.y * TH;
    const long long img = (long long)blockIdx.z * a.bstride;
    const float* src = a.in + img;
    const int sb = x0 - E::HL;
    constexpr int NQ = TC / 4;
    const bool col_interior = sb >= 0 && sb + TC <= a.W;
    // epilogue operand of this thread's V rows, loaded before the tile so its
    // latency overlaps the tile load (the small-image launches are latency bound)
    float4 pre[V];
    {
        const int xq = x0 + 4 * tx;
#pragma unroll
        for (int o = 0; o < V; ++o) {
            pre[o] = make_float4(0.f, 0.f, 0.f, 0.f);
            const int y = min(yt0 + ty * V + o, a.y1 - 1);
            if ((MODE == 1 || MODE == 2) && xq < a.W) {
                const long long idx = img + (long long)y * a.pitch + xq;
                if (xq + 3 < a.W) {
                    pre[o] = __ldg(reinterpret_cast<const float4*>(a.aux + idx));
                } else {
                    pre[o].x = a.aux[idx];
                    if (xq + 1 < a.W) pre[o].y = a.aux[idx + 1];
                    if (xq + 2 < a.W) pre[o].z = a.aux[idx + 2];
                }
            }
        }
    }

    for (int k = threadIdx.x; k < TR * NQ; k += 32 * NTY) {
        const int t = k / NQ, q = k - t * NQ;
        const int row = clampi(yt0 + SH::MINDY + t, a.ylo, a.yhi);
        const float* rp = src + (long long)row * a.pitch;
        const int c = sb + 4 * q;
        float* dst = tile + t * TCP + 4 * q;
        if (col_interior || (c >= 0 && c + 3 < a.W)) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(rp + c) : "memory");
        } else {
            float4 v;
            v.x = __ldg(rp + clampi(c, 0, a.W - 1));
            v.y = __ldg(rp + clampi(c + 1, 0, a.W - 1));
            v.z = __ldg(rp + clampi(c + 2, 0, a.W - 1));
            v.w = __ldg(rp + clampi(c + 3, 0, a.W - 1));
            *reinterpret_cast<float4*>(dst) = v;
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    float4 acc[V];
#pragma unroll
    for (int o = 0; o < V; ++o) acc[o] = make_float4(0.f, 0.f, 0.f, 0.f);
    const float* base = tile + (ty * V) * TCP + 4 * tx;
#pragma unroll
    for (int tl = 0; tl < V + NR - 1; ++tl) {
        float v[4 * E::NCH];
        const float4* p = reinterpret_cast<const float4*>(base + tl * TCP);
#pragma unroll
        for (int c = 0; c < E::NCH; ++c) {
            const float4 q = p[c];
            v[4 * c] = q.x;
            v[4 * c + 1] = q.y;
            v[4 * c + 2] = q.z;
            v[4 * c + 3] = q.w;
        }
        float Pf[E::NWIN];
        Pf[0] = v[E::OFF];
#pragma unroll
        for (int k = 1; k < E::NWIN; ++k) Pf[k] = Pf[k - 1] + v[E::OFF + k];
#pragma unroll
        for (int o = 0; o < V; ++o) {
            const int r = tl - o;
            if (r < 0 || r >= NR) continue;
            const int lo = SH::LO(r) + E::XL, hi = SH::HI(r) + E::XL;
            if (hi - lo < 2) {  // 1- and 2-pixel spans straight from the window (exact for one tap)
                const float* w = v + E::OFF + lo;
                if (hi == lo) {
                    acc[o].x += w[0];
                    acc[o].y += w[1];
                    acc[o].z += w[2];
                    acc[o].w += w[3];
                } else {
                    acc[o].x += w[0] + w[1];
                    acc[o].y += w[1] + w[2];
                    acc[o].z += w[2] + w[3];
                    acc[o].w += w[3] + w[4];
                }
                continue;
            }
            acc[o].x += Pf[hi] - (lo > 0 ? Pf[lo - 1] : 0.f);
            acc[o].y += Pf[hi + 1] - Pf[lo];
            acc[o].z += Pf[hi + 2] - Pf[lo + 1];
            acc[o].w += Pf[hi + 3] - Pf[lo + 2];
        }
    }
    const int xc = x0 + 4 * tx;
    float maxd = 0.f, csum = 0.f;
    if (xc < a.W) {
        const bool full_store = xc + 3 < a.W;
        const int yo0 = yt0 + ty * V;
#pragma unroll
        for (int o = 0; o < V; ++o) {
            const int y = yo0 + o;
            if (y >= a.y1) break;
            const long long idx = img + (long long)y * a.pitch + xc;
            float4 x = pre[o];
            float4 vv = make_float4(acc[o].x * a.scale, acc[o].y * a.scale, acc[o].z * a.scale, acc[o].w * a.scale);
            if (!full_store) {
                if (xc + 1 >= a.W) vv.y = x.y = 0.f;
                if (xc + 2 >= a.W) vv.z = x.z = 0.f;
                vv.w = x.w = 0.f;
            }
            float4 ov;
            ov.x = epi1<MODE>(vv.x, x.x, a.eps, a.clamp, maxd, csum);
            ov.y = epi1<MODE>(vv.y, x.y, a.eps, a.clamp, maxd, csum);
            ov.z = epi1<MODE>(vv.z, x.z, a.eps, a.clamp, maxd, csum);
            ov.w = epi1<MODE>(vv.w, x.w, a.eps, a.clamp, maxd, csum);
            float* op = a.out + idx;
            if (full_store) {
                *reinterpret_cast<float4*>(op) = ov;
            } else {
                op[0] = ov.x;
                if (xc + 1 < a.W) op[1] = ov.y;
                if (xc + 2 < a.W) op[2] = ov.z;
            }
        }
    }
    if (MODE == 2 && a.maxchange) {
        const unsigned bits = __reduce_max_sync(0xffffffffu, __float_as_uint(maxd));
        const int nan = __reduce_or_sync(0xffffffffu, (int)isnan(csum));
        if (tx == 0) {
            if (bits) atomicMax(a.maxchange, bits);
            if (nan) atomicOr(a.nanflag, 1);
            if (a.tend) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                atomicMax(a.tend, t);
            }
        }
    }
}
// one entry point per program: JMODE (0 store, 1 quotient, 2 update) on
// JV x JNTY-row tiles (large images) or 2 x 4-row tiles (JSMALL: small,
// latency-bound images get many more CTAs)
#if JSMALL
extern "C" __global__ void __launch_bounds__(128) fdg_jit_entry(const JitArgs a) { spant<JMODE, 2, 4>(a); }
#else
extern "C" __global__ void __launch_bounds__(32 * JNTY, JMINB) fdg_jit_entry(const JitArgs a) { spant<JMODE, JV, JNTY>(a); }
#endif
)JIT";

// tap-list variant: struct TP {NR, MINDY, MINDX, NWX, UNI, row start / dx
// (relative to MINDX) / weight tables} generated per plan, one partial per
// PSF row in tap order (k_taps' order), wrap = the cyclic (Fourier) contract
const char* kJitTapsSource = R"JIT(
struct JitArgs {
    const float* in;
    const float* aux;
    float* out;
    int pitch, W;
    int y0, y1, ylo, yhi;
    long long bstride;
    float scale, eps;
    int clamp;
    unsigned* maxchange;
    int* nanflag;
    unsigned long long* tend;
    int wrap;
    float* out2;            // masked quotient: cachedV
    unsigned char* active;  // masked modes 3-5
    float thr;
    int may_thin;
};
__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
__device__ __forceinline__ int wrapi(int v, int n) { int r = v % n; return r < 0 ? r + n : r; }
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float div_fast(float f, float d) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
    const float q0 = f * r;
    const float e = fmaf(-d, q0, f);
    return fmaf(e, r, q0);
}
template <int MODE>
__device__ __forceinline__ float epi1(float v, float x, float eps, int clamp, float& maxd, float& csum) {
    if (MODE == 0) return v;
    if (MODE == 1) return div_fast(x, v < eps ? eps : v);
    float value = v * x;
    if (clamp && value < 0.f) value = 0.f;
    maxd = fmaxf(maxd, fabsf(value - x));
    csum += value;
    return value;
}
// compile-time loops (the tap indices must be static register indices; a
// plain #pragma unroll over V + NR - 1 rows x V outputs x taps gives up on
// larger lists and falls back to local-memory arrays)
template <int I>
struct IC {
    static constexpr int value = I;
};
template <int I, int N>
struct SFor {
    template <class F>
    __device__ __forceinline__ static void run(F&& f) {
        f(IC<I>{});
        SFor<I + 1, N>::run(f);
    }
};
template <int N>
struct SFor<N, N> {
    template <class F>
    __device__ __forceinline__ static void run(F&&) {}
};
template <int MODE, int V, int NTY>
__device__ void tapt(const JitArgs& a) {
    constexpr int NR = TP::NR;
    constexpr int TW = 128, TH = V * NTY, TR = TH + NR - 1;
    constexpr int NWIN = 4 + TP::NWX - 1;            // window values per thread per row
    constexpr int NCH = (NWIN + 3) / 4;               // float4 chunks (window starts at a chunk)
    constexpr int TCP = TW + 4 * ((TP::NWX + 2) / 4) + 8;  // tile columns (+ slack)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* tile = reinterpret_cast<float*>(smem_raw);
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int x0 = blockIdx.x * TW;
    const int yt0 = a.y0 + blockIdx.y * TH;
    const long long img = (long long)blockIdx.z * a.bstride;
    const float* src = a.in + img;
    const int cb = x0 + TP::MINDX;  // image column of tile column 0
    const int hgt = a.yhi - a.ylo + 1;
    // epilogue operand of this thread's V rows, loaded before the tile so its
    // latency overlaps the tile load (the small-image launches are latency bound)
    float4 pre[V];
    {
        const int xq = x0 + 4 * tx;
#pragma unroll
        for (int o = 0; o < V; ++o) {
            pre[o] = make_float4(0.f, 0.f, 0.f, 0.f);
            const int y = min(yt0 + ty * V + o, a.y1 - 1);
            if ((MODE == 1 || MODE == 2) && xq < a.W) {
                const long long idx = img + (long long)y * a.pitch + xq;
                if (xq + 3 < a.W) {
                    pre[o] = __ldg(reinterpret_cast<const float4*>(a.aux + idx));
                } else {
                    pre[o].x = a.aux[idx];
                    if (xq + 1 < a.W) pre[o].y = a.aux[idx + 1];
                    if (xq + 2 < a.W) pre[o].z = a.aux[idx + 2];
                }
            }
        }
    }
    if (MODE >= 3) {  // thinned pass: tiles without an active output pixel keep their fallback
        int any = 0;
        const int xq = x0 + 4 * tx;
        for (int o = 0; o < V; ++o) {
            const int y = yt0 + ty * V + o;
            if (y >= a.y1 || xq >= a.W) break;
            const unsigned char* m = a.active + img + (long long)y * a.pitch + xq;
            any |= m[0] | (xq + 1 < a.W ? m[1] : 0) | (xq + 2 < a.W ? m[2] : 0) | (xq + 3 < a.W ? m[3] : 0);
        }
        if (!__syncthreads_or(any)) return;
    }
    for (int k = threadIdx.x; k < TR * TCP; k += 32 * NTY) {
        const int t = k / TCP, c = k - t * TCP;
        int gy = yt0 + TP::MINDY + t, gx = cb + c;
        if (a.wrap) {
            gy = a.ylo + wrapi(gy - a.ylo, hgt);
            gx = wrapi(gx, a.W);
        } else {
            gy = clampi(gy, a.ylo, a.yhi);
            gx = clampi(gx, 0, a.W - 1);
        }
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(tile + k)),
                     "l"(src + (long long)gy * a.pitch + gx) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    float4 acc[V];
#pragma unroll
    for (int o = 0; o < V; ++o) acc[o] = make_float4(0.f, 0.f, 0.f, 0.f);
    const float* base = tile + (ty * V) * TCP + 4 * tx;
    SFor<0, V + NR - 1>::run([&](auto tlc) {
        constexpr int tl = decltype(tlc)::value;
        float v[4 * NCH];
        const float4* p = reinterpret_cast<const float4*>(base + tl * TCP);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const float4 q = p[c];
            v[4 * c] = q.x;
            v[4 * c + 1] = q.y;
            v[4 * c + 2] = q.z;
            v[4 * c + 3] = q.w;
        }
        SFor<0, V>::run([&](auto oc) {
            constexpr int o = decltype(oc)::value;
            constexpr int r = tl - o;
            if constexpr (r >= 0 && r < NR) {
                float4 part = make_float4(0.f, 0.f, 0.f, 0.f);
                SFor<TP::RS(r), TP::RS(r + 1)>::run([&](auto kc) {
                    constexpr int k = decltype(kc)::value;
                    constexpr int d = TP::DX(k);
                    if constexpr (TP::UNI) {
                        part.x += v[d];
                        part.y += v[d + 1];
                        part.z += v[d + 2];
                        part.w += v[d + 3];
                    } else {
                        constexpr float w = TP::WT(k);
                        part.x = fmaf(w, v[d], part.x);
                        part.y = fmaf(w, v[d + 1], part.y);
                        part.z = fmaf(w, v[d + 2], part.z);
                        part.w = fmaf(w, v[d + 3], part.w);
                    }
                });
                acc[o].x += part.x;
                acc[o].y += part.y;
                acc[o].z += part.z;
                acc[o].w += part.w;
            }
        });
    });
    const int xc = x0 + 4 * tx;
    float maxd = 0.f, csum = 0.f;
    if constexpr (MODE >= 3) if (xc < a.W) {  // masked epilogues (convolve.hpp:473-510): active pixels only
        const int yo0 = yt0 + ty * V;
#pragma unroll
        for (int o = 0; o < V; ++o) {
            const int y = yo0 + o;
            if (y >= a.y1) break;
            const long long idx = img + (long long)y * a.pitch + xc;
            const float vv[4] = {acc[o].x, acc[o].y, acc[o].z, acc[o].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (xc + j >= a.W || !a.active[idx + j]) continue;
                const float v = TP::UNI ? vv[j] * a.scale : vv[j];
                if (MODE == 3) {
                    a.out2[idx + j] = v;
                    a.out[idx + j] = div_fast(a.aux[idx + j], v < a.eps ? a.eps : v);
                } else if (MODE == 4) {
                    const float u = a.aux[idx + j];
                    float value = v * u;
                    if (a.clamp && value < 0.f) value = 0.f;
                    const float d = fabsf(value - u);
                    maxd = fmaxf(maxd, d);
                    csum += value;
                    if (a.may_thin && d < a.thr) a.active[idx + j] = 0;
                    a.out[idx + j] = value;
                } else {
                    a.out[idx + j] = v;
                }
            }
        }
    }
    if constexpr (MODE < 3) if (xc < a.W) {
        const bool full_store = xc + 3 < a.W;
        const int yo0 = yt0 + ty * V;
#pragma unroll
        for (int o = 0; o < V; ++o) {
            const int y = yo0 + o;
            if (y >= a.y1) break;
            const long long idx = img + (long long)y * a.pitch + xc;
            float4 x = pre[o];
            float4 vv = acc[o];
            if (TP::UNI) vv = make_float4(vv.x * a.scale, vv.y * a.scale, vv.z * a.scale, vv.w * a.scale);
            if (!full_store) {
                if (xc + 1 >= a.W) vv.y = x.y = 0.f;
                if (xc + 2 >= a.W) vv.z = x.z = 0.f;
                vv.w = x.w = 0.f;
            }
            float4 ov;
            ov.x = epi1<MODE>(vv.x, x.x, a.eps, a.clamp, maxd, csum);
            ov.y = epi1<MODE>(vv.y, x.y, a.eps, a.clamp, maxd, csum);
            ov.z = epi1<MODE>(vv.z, x.z, a.eps, a.clamp, maxd, csum);
            ov.w = epi1<MODE>(vv.w, x.w, a.eps, a.clamp, maxd, csum);
            float* op = a.out + idx;
            if (full_store) {
                *reinterpret_cast<float4*>(op) = ov;
            } else {
                op[0] = ov.x;
                if (xc + 1 < a.W) op[1] = ov.y;
                if (xc + 2 < a.W) op[2] = ov.z;
            }
        }
    }
    if ((MODE == 2 || MODE == 4) && a.maxchange) {
        const unsigned bits = __reduce_max_sync(0xffffffffu, __float_as_uint(maxd));
        const int nan = __reduce_or_sync(0xffffffffu, (int)isnan(csum));
        if (tx == 0) {
            if (bits) atomicMax(a.maxchange, bits);
            if (nan) atomicOr(a.nanflag, 1);
            if (a.tend) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                atomicMax(a.tend, t);
            }
        }
    }
}
#if JSMALL
extern "C" __global__ void __launch_bounds__(128) fdg_jit_entry(const JitArgs a) { tapt<JMODE, 2, 4>(a); }
#else
extern "C" __global__ void __launch_bounds__(32 * JNTY, JMINB) fdg_jit_entry(const JitArgs a) { tapt<JMODE, JV, JNTY>(a); }
#endif
)JIT";

// host mirror of JitArgs (same layout)
struct JitArgs {
    const float* in;
    const float* aux;
    float* out;
    int pitch, W;
    int y0, y1, ylo, yhi;
    long long bstride;
    float scale, eps;
    int clamp;
    unsigned* maxchange;
    int* nanflag;
    unsigned long long* tend;
    int wrap;  // tap kernels only (the span source's struct ends before it)
    float* out2;
    unsigned char* active;
    float thr;
    int may_thin;
};

// ---- NVRTC (dlopen) and the driver calls (cudaGetDriverEntryPoint)
typedef int nvrtcResult_;
typedef struct _nvrtcProgram* nvrtcProgram_;
struct Nvrtc {
    nvrtcResult_ (*create)(nvrtcProgram_*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
    nvrtcResult_ (*compile)(nvrtcProgram_, int, const char* const*) = nullptr;
    nvrtcResult_ (*cubin_size)(nvrtcProgram_, size_t*) = nullptr;
    nvrtcResult_ (*cubin)(nvrtcProgram_, char*) = nullptr;
    nvrtcResult_ (*log_size)(nvrtcProgram_, size_t*) = nullptr;
    nvrtcResult_ (*log)(nvrtcProgram_, char*) = nullptr;
    nvrtcResult_ (*destroy)(nvrtcProgram_*) = nullptr;
    CUresult (*module_load)(CUmodule*, const void*) = nullptr;
    CUresult (*get_function)(CUfunction*, CUmodule, const char*) = nullptr;
    CUresult (*func_set_attr)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                       void**, void**) = nullptr;
    bool ok = false;
};

Nvrtc& nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnvrtc.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        bool all = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            all = all && fn != nullptr;
        };
        sym(n.create, "nvrtcCreateProgram");
        sym(n.compile, "nvrtcCompileProgram");
        sym(n.cubin_size, "nvrtcGetCUBINSize");
        sym(n.cubin, "nvrtcGetCUBIN");
        sym(n.log_size, "nvrtcGetProgramLogSize");
        sym(n.log, "nvrtcGetProgramLog");
        sym(n.destroy, "nvrtcDestroyProgram");
        auto drv = [&](auto& fn, const char* name) {
            void* p = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                p = nullptr;
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
            all = all && p != nullptr;
        };
        drv(n.module_load, "cuModuleLoadData");
        drv(n.get_function, "cuModuleGetFunction");
        drv(n.func_set_attr, "cuFuncSetAttribute");
        drv(n.launch, "cuLaunchKernel");
        n.ok = all;
    });
    return n;
}

// one table / tap list: the generated header, and one module per
// (epilogue mode, tile size) built on first use (~0.1-0.8 s each)
struct JitKernel {
    bool ok = false;              // header generated (the shape qualifies)
    std::string header;
    const char* source = nullptr;
    const char* what = "";
    int V = 0, NTY = 0;
    size_t smem = 0, smem_s = 0;
    CUfunction fn[2][6] = {};     // [small][mode]: 0-2 store / quotient / update, 3-5 masked
    bool failed[2][6] = {};
};
constexpr int JIT_SMALL_PX = 512 * 1024;  // images up to this many pixels per launch: small tiles

std::atomic<int> g_jit{getenv("FDG_SPANS_JIT") ? atoi(getenv("FDG_SPANS_JIT")) : 1};
std::mutex g_jit_mu;
std::map<std::string, std::unique_ptr<JitKernel>> g_jit_cache;  // key: device + span table / tap list

// compile `header + source` with one entry point (mode, tile size); nullptr
// (logged) on any failure.  Called with g_jit_mu held.
CUfunction jit_build(JitKernel* k, int mode, int small) {
    if (k->fn[small][mode]) return k->fn[small][mode];
    if (k->failed[small][mode]) return nullptr;
    k->failed[small][mode] = true;
    Nvrtc& n = nvrtc();
    if (!n.ok) return nullptr;
    const std::string src = k->header + "#define JMODE " + std::to_string(mode) + "\n#define JSMALL " +
                            std::to_string(small) + "\n" + k->source;
    nvrtcProgram_ prog = nullptr;
    if (n.create(&prog, src.c_str(), "fdg_jit.cu", 0, nullptr, nullptr) != 0) return nullptr;
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=true", "-default-device"};
    const int rc = n.compile(prog, 4, opts);
    if (rc != 0) {
        size_t ls = 0;
        n.log_size(prog, &ls);
        std::string log(ls, '\0');
        n.log(prog, log.data());
        std::fprintf(stderr, "[fdg] %s JIT compile failed, the generic kernel is used:\n%s\n", k->what, log.c_str());
        n.destroy(&prog);
        return nullptr;
    }
    size_t cs = 0;
    n.cubin_size(prog, &cs);
    std::string cubin(cs, '\0');
    n.cubin(prog, cubin.data());
    n.destroy(&prog);
    CUmodule mod = nullptr;
    CUfunction f = nullptr;
    if (n.module_load(&mod, cubin.data()) != CUDA_SUCCESS) return nullptr;
    if (n.get_function(&f, mod, "fdg_jit_entry") != CUDA_SUCCESS) return nullptr;
    const size_t smem = small ? k->smem_s : k->smem;
    if (n.func_set_attr(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem) != CUDA_SUCCESS) return nullptr;
    k->failed[small][mode] = false;
    return k->fn[small][mode] = f;
}

std::string tile_defs(int V, int NTY, int minb) {
    return "#define JV " + std::to_string(V) + "\n#define JNTY " + std::to_string(NTY) + "\n#define JMINB " +
           std::to_string(minb) + "\n";
}

// cache lookup / insertion; `make` builds a new entry (called with the lock held)
template <class F>
JitKernel* jit_cached(const std::string& key, F make) {
    std::lock_guard<std::mutex> lk(g_jit_mu);
    auto it = g_jit_cache.find(key);
    if (it != g_jit_cache.end()) return it->second->ok ? it->second.get() : nullptr;
    auto jk = std::make_unique<JitKernel>();
    JitKernel* out = jk.get();
    g_jit_cache[key] = std::move(jk);
    make(out);
    return out->ok ? out : nullptr;
}

// span table -> tile kernel (once per table and device); nullptr when unavailable
JitKernel* jit_get(const DevPsf& p) {
    if (!g_jit.load() || p.nrows < 1 || p.nrows > 64 || (int)p.h_span.size() != 2 * p.nrows) return nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::string key = "S" + std::to_string(dev) + ":" + std::to_string(p.min_dy);
    for (int v : p.h_span) key += "," + std::to_string(v);
    return jit_cached(key, [&](JitKernel* out) {
        int xl = 0, xr = 0;
        for (int r = 0; r < p.nrows; ++r) {
            xl = std::max(xl, -p.h_span[2 * r]);
            xr = std::max(xr, p.h_span[2 * r + 1]);
        }
        if (xl + xr > 64) return;
        // tile shape as for the compile-time tables: tall PSFs 8 warps x 7 rows,
        // short ones 7 x 4; wide windows keep more registers (2 CTAs per SM)
        const int V = p.nrows > 16 ? 7 : 4, NTY = p.nrows > 16 ? 8 : 7;
        const int minb = 4 + xl + xr > 26 ? 2 : 4;
        std::string sh = "struct SH {\n  static constexpr int NR = " + std::to_string(p.nrows) +
                         ", MINDY = " + std::to_string(p.min_dy) +
                         ";\n  __device__ static constexpr int LO(int r) {\n    constexpr int t[NR] = {";
        for (int r = 0; r < p.nrows; ++r) sh += (r ? "," : "") + std::to_string(p.h_span[2 * r]);
        sh += "};\n    return t[r];\n  }\n  __device__ static constexpr int HI(int r) {\n    constexpr int t[NR] = {";
        for (int r = 0; r < p.nrows; ++r) sh += (r ? "," : "") + std::to_string(p.h_span[2 * r + 1]);
        sh += "};\n    return t[r];\n  }\n};\n" + tile_defs(V, NTY, minb);
        const int TCP = 128 + (xl + 3) / 4 * 4 + (xr + 3) / 4 * 4 + 4;
        out->header = sh;
        out->source = kJitSource;
        out->what = "span table";
        out->V = V;
        out->NTY = NTY;
        out->smem = sizeof(float) * (size_t)(V * NTY + p.nrows - 1) * TCP;
        out->smem_s = sizeof(float) * (size_t)(2 * 4 + p.nrows - 1) * TCP;
        out->ok = nvrtc().ok;
    });
}

// tap list -> tile kernel (<= 128 taps, x extent <= 32)
JitKernel* taps_get(const DevPsf& p) {
    if (!g_jit.load() || p.ntaps < 1 || p.ntaps > 128 || p.nrows < 1 || p.nrows > 64 ||
        (int)p.h_dx.size() != p.ntaps || (int)p.h_row_start.size() != p.nrows + 1)
        return nullptr;
    const int nwx = p.max_dx - p.min_dx + 1;
    if (nwx > 65) return nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    char buf[64];
    std::string key = "T" + std::to_string(dev) + ":" + std::to_string(p.min_dx) + ":" + std::to_string(p.min_dy) +
                      ":" + std::to_string(p.uniform);
    for (int r = 0; r <= p.nrows; ++r) key += "," + std::to_string(p.h_row_start[r]);
    for (int k = 0; k < p.ntaps; ++k) {
        std::snprintf(buf, sizeof buf, ";%d:%a", p.h_dx[k], p.h_w.empty() ? 0.0 : (double)p.h_w[k]);
        key += buf;
    }
    return jit_cached(key, [&](JitKernel* out) {
        const int V = p.nrows > 16 ? 7 : 4, NTY = p.nrows > 16 ? 8 : 7;
        std::string tp = "struct TP {\n  static constexpr int NR = " + std::to_string(p.nrows) +
                         ", MINDY = " + std::to_string(p.min_dy) + ", MINDX = " + std::to_string(p.min_dx) +
                         ", NWX = " + std::to_string(nwx) + ";\n  static constexpr bool UNI = " +
                         (p.uniform ? "true" : "false") +
                         ";\n  __device__ static constexpr int RS(int r) {\n    constexpr int t[NR + 1] = {";
        for (int r = 0; r <= p.nrows; ++r) tp += (r ? "," : "") + std::to_string(p.h_row_start[r]);
        tp += "};\n    return t[r];\n  }\n  __device__ static constexpr int DX(int k) {\n    constexpr int t[" +
              std::to_string(p.ntaps) + "] = {";
        for (int k = 0; k < p.ntaps; ++k) tp += (k ? "," : "") + std::to_string(p.h_dx[k] - p.min_dx);
        tp += "};\n    return t[k];\n  }\n  __device__ static constexpr float WT(int k) {\n    constexpr float t[" +
              std::to_string(p.ntaps) + "] = {";
        for (int k = 0; k < p.ntaps; ++k) {
            std::snprintf(buf, sizeof buf, "%s%.9ef", k ? "," : "", p.h_w.empty() ? 0.0 : (double)p.h_w[k]);
            tp += buf;
        }
        tp += "};\n    return t[k];\n  }\n};\n" + tile_defs(V, NTY, 2);
        const int TCP = 128 + 4 * ((nwx + 2) / 4) + 8;
        out->header = tp;
        out->source = kJitTapsSource;
        out->what = "tap list";
        out->V = V;
        out->NTY = NTY;
        out->smem = sizeof(float) * (size_t)(V * NTY + p.nrows - 1) * TCP;
        out->smem_s = sizeof(float) * (size_t)(2 * 4 + p.nrows - 1) * TCP;
        out->ok = nvrtc().ok;
    });
}

cudaError_t jit_launch(JitKernel* k, JitArgs& a, const Geom& g, const Epi& e, cudaStream_t st) {
    const int rows = g.y1 - g.y0;
    if (rows <= 0) return cudaSuccess;
    const bool small = (long long)g.W * rows * g.batch <= JIT_SMALL_PX;
    const int V = small ? 2 : k->V, NTY = small ? 4 : k->NTY, TH = V * NTY;
    int m = -1;
    if (!e.active) m = e.mode == EPI_STORE ? 0 : e.mode == EPI_QUOT ? 1 : e.mode == EPI_UPDATE ? 2 : -1;
    else m = e.mode == EPI_MQUOT ? 3 : e.mode == EPI_MUPDATE ? 4 : e.mode == EPI_STORE ? 5 : -1;
    if (m < 0) return cudaErrorInvalidValue;
    CUfunction f;
    {
        std::lock_guard<std::mutex> lk(g_jit_mu);
        f = jit_build(k, m, small ? 1 : 0);
    }
    if (!f) return cudaErrorNotSupported;
    void* args[] = {&a};
    const CUresult r = nvrtc().launch(f, (unsigned)((g.W + 127) / 128),
                                      (unsigned)((rows + TH - 1) / TH), (unsigned)g.batch, 32u * NTY, 1, 1,
                                      (unsigned)(small ? k->smem_s : k->smem), reinterpret_cast<CUstream>(st), args,
                                      nullptr);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

JitArgs jit_args(const DevPsf& p, const Geom& g, const Epi& e) {
    JitArgs a;
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
    a.wrap = g.wrap;
    a.out2 = e.out2;
    a.active = e.active;
    a.thr = e.thr;
    a.may_thin = e.may_thin;
    return a;
}

}  // namespace

void set_spans_jit(int v) { g_jit.store(v); }
int spans_jit_mode() { return g_jit.load(); }

bool spans_jit_ready(const DevPsf& p) { return jit_get(p) != nullptr; }

cudaError_t launch_spans_jit(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st) {
    JitKernel* k = jit_get(p);
    if (!k) return cudaErrorNotSupported;
    JitArgs a = jit_args(p, g, e);
    return jit_launch(k, a, g, e, st);
}

bool taps_jit_ready(const DevPsf& p) { return taps_get(p) != nullptr; }

cudaError_t launch_taps_jit(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st) {
    JitKernel* k = taps_get(p);
    if (!k) return cudaErrorNotSupported;
    JitArgs a = jit_args(p, g, e);
    return jit_launch(k, a, g, e, st);
}

}  // namespace fdg
