// ATTIC: an experimental variant of the box engine (compile-time width, register/smem
// ring variants) that measured SLOWER than kernels_rect.cu on B200 (see
// profiles/r01_box_engine_notes.md); kept for reference, not built.
// kernels_box.cu -- specialised uniform-box engine (compile-time width MX),
// the hot kernel of configs 0, 4 and 4b (Box1d*/Box2d*, convolve.hpp:217-388).
//
// One CTA marches down a 512-column strip of a row band.  A producer warp
// streams one replicate-clamped input row segment (strip + horizontal halo)
// and one epilogue-operand row per step into an S-deep shared-memory ring
// with TMA bulk copies (cp.async.bulk + mbarrier complete_tx).  Four consumer
// warps, 4 adjacent columns per thread:
//   * horizontal window sums of MX taps from float4 shared loads, as
//     left partial + (balanced-tree) shared middle + right partial -- adds
//     only, no sliding subtraction;
//   * vertical running sum over the last MY rows with the horizontal sums
//     kept in a per-thread shared-memory ring (runtime MY), rebuilt from the
//     ring every REFRESH rows so fp32 drift stays bounded (hard
//     part 1);
//   * fused RL epilogue: quotient f / max(v, eps), or update
//     max(v * u, 0) with max|du| and the reference's NaN checksum
//     (rl.hpp:164-173), then a float4 store.
// One elected lane per consumer warp arrives on the "empty" barrier (all 32
// lanes arriving serialises on the barrier word: measured 40% slower), and the
// replicate-clamped slow path is a separate instantiation taken by whole
// warps (only the warps at the image's left / right edge).
// HBM traffic per pass: read input + read epilogue operand + write = 12 B/px,
// plus (MY-1)/band re-read halo rows.
#include <cstdlib>

#include "common.cuh"

namespace fdg {
namespace {

constexpr int REFRESH = 32;

struct BoxArgs {
    const float* in;
    const float* aux;
    float* out;
    int pitch, W, Wp4;
    int y0, y1, ylo, yhi, band;
    long long bstride;
    int my, min_dx, min_dy;
    int HL, HR, seg;
    float scale, eps;
    int clamp;
    unsigned* maxchange;
    int* nanflag;
    unsigned hint;
    int pd;  // L2 prefetch distance in rows (0 = off)
};

__device__ __forceinline__ void prefetch_l2(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void wait_sleep(uint64_t* bar, unsigned parity, unsigned hint) {
    if (hint == 0) {
        mbar_wait(bar, parity);
        return;
    }
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(hint)
        : "memory");
}

template <int N>
__device__ __forceinline__ float tree_sum(const float* v) {
    if constexpr (N == 1) {
        return v[0];
    } else {
        return tree_sum<N / 2>(v) + tree_sum<N - N / 2>(v + N / 2);
    }
}

// 4 horizontal window sums of MX taps; chunk 0 holds output 0's first tap at
// position OFF.
template <int MX, int OFF>
__device__ __forceinline__ float4 hsum(const float4* p) {
    constexpr int NCH = (OFF + 3 + MX - 1) / 4 + 1;
    float v[4 * NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const float4 q = p[c];
        v[4 * c] = q.x;
        v[4 * c + 1] = q.y;
        v[4 * c + 2] = q.z;
        v[4 * c + 3] = q.w;
    }
    if constexpr (MX >= 4) {
        const float mid = tree_sum<MX - 3>(v + OFF + 3);  // taps common to all four windows
        const float l2 = v[OFF + 2], l1 = v[OFF + 1] + l2, l0 = v[OFF] + l1;
        const float r1 = v[OFF + MX], r2 = r1 + v[OFF + MX + 1], r3 = r2 + v[OFF + MX + 2];
        return make_float4(l0 + mid, (l1 + mid) + r1, (l2 + mid) + r2, mid + r3);
    } else {
        float H[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) H[j] = tree_sum<MX>(v + OFF + j);
        return make_float4(H[0], H[1], H[2], H[3]);
    }
}

template <int MX>
__device__ __forceinline__ float4 hsum_clamped(const float* seg, int xc, int min_dx, int W, int sb) {
    float H[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float s = 0.f;
#pragma unroll 4
        for (int k = 0; k < MX; ++k) s += seg[clampi(xc + j + min_dx + k, 0, W - 1) - sb];
        H[j] = s;
    }
    return make_float4(H[0], H[1], H[2], H[3]);
}

template <int MODE>
__device__ __forceinline__ float epi1(float v, float x, float eps, int clamp, float& maxd, float& csum) {
    if (MODE == EPI_STORE) return v;
    if (MODE == EPI_QUOT) return x / (v < eps ? eps : v);
    float value = v * x;  // EPI_UPDATE: x = u
    if (clamp && value < 0.f) value = 0.f;
    maxd = fmaxf(maxd, fabsf(value - x));
    csum += value;
    return value;
}

struct Ring {
    uint64_t* full;
    uint64_t* empty;
    float* in;
    float* aux;
    float4* h;
};

template <int MODE, int MX, int OFF, bool EDGE, int NT, int S, int R>
__device__ __forceinline__ void consume(const BoxArgs& a, const Ring& ring, int tid, int x0, int yb0, int steps,
                                        long long img) {
    constexpr bool HAS_AUX = MODE != EPI_STORE;
    constexpr int CW = 4 * NT;
    const int my = a.my;
    const int xc = x0 + 4 * tid;
    const int k0 = (a.HL + a.min_dx) >> 2;
    const int sb = x0 - a.HL;
    const bool full_store = xc + 3 < a.W;
    const float scale = a.scale, eps = a.eps;
    const int clamp = a.clamp;
    const int segf = a.seg;
    float maxd = 0.f, csum = 0.f;
    float4 col = make_float4(0.f, 0.f, 0.f, 0.f);
    float* outp = a.out + img + (long long)yb0 * a.pitch + xc;
    const long long pitch = a.pitch;
    float4* hslot = ring.h + tid;
    float4* const hend = ring.h + (size_t)my * NT + tid;
    int s = 0;
    unsigned phase = 0;
    for (int i0 = 0; i0 < steps; i0 += R) {
        wait_sleep(&ring.full[s], phase, a.hint);
        const float* seg0 = ring.in + (size_t)s * R * segf;
        const float* aux0 = ring.aux + (size_t)s * R * CW + 4 * tid;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int i = i0 + r;
            if (i >= steps) break;
            const float* seg = seg0 + r * segf;
            const float4 h = EDGE ? hsum_clamped<MX>(seg, xc, a.min_dx, a.W, sb)
                                  : hsum<MX, OFF>(reinterpret_cast<const float4*>(seg) + k0 + tid);
            if (my > 1) {
                if (i >= my) {
                    const float4 old = *hslot;
                    col.x -= old.x;
                    col.y -= old.y;
                    col.z -= old.z;
                    col.w -= old.w;
                }
                col.x += h.x;
                col.y += h.y;
                col.z += h.z;
                col.w += h.w;
                *hslot = h;
                if ((i & (REFRESH - 1)) == REFRESH - 1 && i >= my) {  // rebuild from the ring
                    float4 f = ring.h[tid];
                    for (int k = 1; k < my; ++k) {
                        const float4 q = ring.h[(size_t)k * NT + tid];
                        f.x += q.x;
                        f.y += q.y;
                        f.z += q.z;
                        f.w += q.w;
                    }
                    col = f;
                }
                hslot += NT;
                if (hslot == hend) hslot = ring.h + tid;
            } else {
                col = h;
            }
            if (i >= my - 1) {
                float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
                if (HAS_AUX) x = *reinterpret_cast<const float4*>(aux0 + r * CW);
                float4 v = make_float4(col.x * scale, col.y * scale, col.z * scale, col.w * scale);
                if (!full_store) {  // past the image edge: neutral values, never stored
                    if (xc >= a.W) v.x = x.x = 0.f;
                    if (xc + 1 >= a.W) v.y = x.y = 0.f;
                    if (xc + 2 >= a.W) v.z = x.z = 0.f;
                    v.w = x.w = 0.f;
                }
                float4 o;
                o.x = epi1<MODE>(v.x, x.x, eps, clamp, maxd, csum);
                o.y = epi1<MODE>(v.y, x.y, eps, clamp, maxd, csum);
                o.z = epi1<MODE>(v.z, x.z, eps, clamp, maxd, csum);
                o.w = epi1<MODE>(v.w, x.w, eps, clamp, maxd, csum);
                if (full_store) {
                    *reinterpret_cast<float4*>(outp) = o;
                } else {
                    if (xc < a.W) outp[0] = o.x;
                    if (xc + 1 < a.W) outp[1] = o.y;
                    if (xc + 2 < a.W) outp[2] = o.z;
                }
                outp += pitch;
            }
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&ring.empty[s]);  // one arrival per consumer warp
        if (++s == S) {
            s = 0;
            phase ^= 1u;
        }
    }
    if (MODE == EPI_UPDATE && a.maxchange) {
        const unsigned bits = __reduce_max_sync(0xffffffffu, __float_as_uint(maxd));
        const int nan = __reduce_or_sync(0xffffffffu, (int)isnan(csum));
        if ((tid & 31) == 0) {
            if (bits) atomicMax(a.maxchange, bits);
            if (nan) atomicOr(a.nanflag, 1);
        }
    }
}

template <int MODE, int MX, int OFF, int NT, int S, int R>
__global__ void __launch_bounds__(NT + 32) k_box(const BoxArgs a) {
    constexpr int CW = 4 * NT;
    constexpr int BAR_BYTES = (2 * S * 8 + 127) / 128 * 128;  // full[S] + empty[S]
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Ring ring;
    ring.full = reinterpret_cast<uint64_t*>(smem_raw);
    ring.empty = ring.full + S;
    ring.in = reinterpret_cast<float*>(smem_raw + BAR_BYTES);
    ring.aux = ring.in + (size_t)S * R * a.seg;
    ring.h = reinterpret_cast<float4*>(ring.aux + (size_t)S * R * CW);

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * CW;
    const int yb0 = a.y0 + blockIdx.y * a.band;
    const int yb1 = min(a.y1, yb0 + a.band);
    if (yb0 >= yb1) return;
    const long long img = (long long)blockIdx.z * a.bstride;
    const int my = a.my;
    const int steps = (yb1 - yb0) + my - 1;
    constexpr bool HAS_AUX = MODE != EPI_STORE;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&ring.full[s], 1);
            mbar_init(&ring.empty[s], NT / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (tid >= NT) {  // producer warp: one thread issues the TMA bulk copies
        if (tid == NT) {
            const int c0 = max(0, x0 - a.HL);
            const int c1 = min(a.Wp4, x0 + CW + a.HR);
            const unsigned in_bytes = (unsigned)(c1 - c0) * 4u;
            const unsigned aux_bytes = (unsigned)(min(a.Wp4, x0 + CW) - x0) * 4u;
            const float* src_in = a.in + img + c0;
            const float* src_aux = a.aux + img + x0 + (long long)(yb0 - (my - 1)) * a.pitch;
            float* dst_in = ring.in + (c0 - (x0 - a.HL));
            const long long pitch = a.pitch;
            int s = 0;
            unsigned phase = 0;
            for (int i0 = 0; i0 < steps; i0 += R) {
                if (i0 >= S * R) wait_sleep(&ring.empty[s], phase ^ 1u, a.hint);
                const int nr = min(R, steps - i0);
                const int naux = HAS_AUX ? max(0, min(nr, i0 + nr - (my - 1))) : 0;
                mbar_arrive_expect_tx(&ring.full[s], nr * in_bytes + naux * aux_bytes);
                for (int r = 0; r < nr; ++r) {
                    const int i = i0 + r;
                    const int row = clampi(yb0 + a.min_dy + i, a.ylo, a.yhi);
                    bulk_g2s(dst_in + (size_t)(s * R + r) * a.seg, src_in + row * pitch, in_bytes, &ring.full[s]);
                    if (HAS_AUX && i >= my - 1)
                        bulk_g2s(ring.aux + (size_t)(s * R + r) * CW, src_aux + i * pitch, aux_bytes, &ring.full[s]);
                }
                if (++s == S) {
                    s = 0;
                    phase ^= 1u;
                }
            }
        }
        return;
    }
    // warps touching the replicate-clamped image edges take the clamped path
    const int xw = x0 + 128 * (tid >> 5);  // first column of this warp (4 columns per lane)
    const bool edge = (xw + a.min_dx < 0) || (xw + 127 + a.min_dx + MX - 1 > a.W - 1);
    if (edge)
        consume<MODE, MX, OFF, true, NT, S, R>(a, ring, tid, x0, yb0, steps, img);
    else
        consume<MODE, MX, OFF, false, NT, S, R>(a, ring, tid, x0, yb0, steps, img);
}

template <int MODE, int MX, int OFF, int NT, int S, int R>
cudaError_t launch_one(const BoxArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
    auto k = k_box<MODE, MX, OFF, NT, S, R>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    k<<<grid, NT + 32, smem, st>>>(a);
    return cudaGetLastError();
}

template <int MX, int OFF, int NT, int S, int R>
cudaError_t launch_modes(int mode, const BoxArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
    switch (mode) {
        case EPI_STORE: return launch_one<EPI_STORE, MX, OFF, NT, S, R>(a, grid, smem, st);
        case EPI_QUOT: return launch_one<EPI_QUOT, MX, OFF, NT, S, R>(a, grid, smem, st);
        case EPI_UPDATE: return launch_one<EPI_UPDATE, MX, OFF, NT, S, R>(a, grid, smem, st);
    }
    return cudaErrorInvalidValue;
}

constexpr int off_centered(int mx) { return (-(mx / 2)) & 3; }

// specialised widths (anchor-centred, as makeLinePsf / makeBoxPsf build them):
// BASELINE's 15 and 31 plus the common odd sizes; others use k_rect
#define FDG_BOX_WIDTHS(X) X(15) X(31) X(3) X(5) X(7) X(9) X(11) X(13) X(17) X(21) X(25)

}  // namespace

bool box_specialized(int mx, int my, int min_dx) {
    if (my < 1 || my > 64) return false;
#define FDG_BOX_CASE(MX) \
    if (mx == MX && (min_dx & 3) == off_centered(MX)) return true;
    FDG_BOX_WIDTHS(FDG_BOX_CASE)
#undef FDG_BOX_CASE
    return false;
}

template <int MX, int NT, int S, int R>
cudaError_t launch_geom(BoxArgs a, const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st) {
    constexpr int CW = 4 * NT;
    a.seg = CW + a.HL + a.HR + 8;
    const int strips = (g.W + CW - 1) / CW;
    const int rows = g.y1 - g.y0;
    if (rows <= 0) return cudaSuccess;
    const long long want = (long long)148 * 6 * (128 / NT);
    int band = (int)(((long long)rows * strips * g.batch + want - 1) / want);
    band = band < 8 ? 8 : (band > 256 ? 256 : band);
    if (p.my > 1 && band < 8 * p.my) band = 8 * p.my;
    a.band = band;
    dim3 grid(strips, (rows + band - 1) / band, g.batch);
    const size_t smem = (2 * S * 8 + 127) / 128 * 128 + sizeof(float) * ((size_t)S * R * a.seg + (size_t)S * R * CW) +
                        (p.my > 1 ? sizeof(float4) * (size_t)NT * p.my : 0);
    return launch_modes<MX, off_centered(MX), NT, S, R>(e.mode, a, grid, smem, st);
}

cudaError_t launch_box(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st) {
    BoxArgs a;
    a.in = g.in;
    a.aux = e.aux;
    a.out = g.out;
    a.pitch = g.pitch;
    a.W = g.W;
    a.Wp4 = (g.W + 3) & ~3;
    a.y0 = g.y0;
    a.y1 = g.y1;
    a.ylo = g.ylo;
    a.yhi = g.yhi;
    a.bstride = g.bstride;
    a.my = p.my;
    a.min_dx = p.min_dx;
    a.min_dy = p.min_dy;
    const int max_dx = p.min_dx + p.mx - 1;
    a.HL = ((max(0, -p.min_dx) + 3) / 4) * 4;
    a.HR = ((max(0, max_dx) + 3) / 4) * 4;
    a.scale = p.scale;
    a.eps = e.eps;
    a.clamp = e.clamp;
    a.maxchange = e.maxchange;
    a.nanflag = e.nanflag;
    static const unsigned hint_env = [] {
        const char* v = getenv("FDG_WAIT_HINT");
        return v ? (unsigned)strtoul(v, nullptr, 0) : 0u;
    }();
    a.hint = hint_env;
    static const int variant = [] {
        const char* v = getenv("FDG_BOX_VARIANT");
        return v ? atoi(v) : 0;
    }();
    static const int pd_env = [] {
        const char* v = getenv("FDG_BOX_PD");
        return v ? atoi(v) : 0;
    }();
    a.pd = pd_env;
    if (p.mx == 15 || p.mx == 31) {  // tuning variants (FDG_BOX_VARIANT) for the BASELINE widths
        switch (variant) {
            case 1: return p.mx == 15 ? launch_geom<15, 128, 3, 4>(a, p, g, e, st) : launch_geom<31, 128, 3, 4>(a, p, g, e, st);
            case 2: return p.mx == 15 ? launch_geom<15, 128, 4, 2>(a, p, g, e, st) : launch_geom<31, 128, 4, 2>(a, p, g, e, st);
            case 3: return p.mx == 15 ? launch_geom<15, 128, 8, 2>(a, p, g, e, st) : launch_geom<31, 128, 8, 2>(a, p, g, e, st);
            case 4: return p.mx == 15 ? launch_geom<15, 128, 2, 4>(a, p, g, e, st) : launch_geom<31, 128, 2, 4>(a, p, g, e, st);
            default: break;
        }
    }
#define FDG_BOX_LAUNCH(MX) \
    if (p.mx == MX) return launch_geom<MX, 128, 4, 4>(a, p, g, e, st);
    FDG_BOX_WIDTHS(FDG_BOX_LAUNCH)
#undef FDG_BOX_LAUNCH
    return cudaErrorInvalidValue;
}

}  // namespace fdg
