// kernels_spans.cu -- "spans" engine: row-convex uniform PSFs (GenericBox,
// convolve.hpp:177-212) whose span table is known at compile time -- the
// BASELINE disc r<=10 (config 2, 21 rows, 317 taps) and the 21 px @ 30 deg
// oblique line (config 1, 11 rows, 29 taps).  Other row-convex PSFs use the
// generic "taps" engine.
//
// Same streaming structure as the box engine (kernels_rect.cu): a CTA
// marches down a 512-column strip; a producer warp streams R replicate-
// clamped input rows (+ halo) and R epilogue-operand rows per mbarrier stage
// with TMA bulk copies.  Consumer thread = 4 adjacent columns:
//   * per input row: float4 window loads, a 24-value register prefix sum,
//     then every span's 4 window sums as prefix differences (static indices;
//     the prefix restarts every row inside a 24-value window, so fp32
//     cancellation stays ~1e-7 relative -- SURVEY 7 hard part 1);
//   * scatter: the row's span sums are added into the NR pending output rows
//     it feeds (output o = i - r for span row r), held in a register ring --
//     the step loop is unrolled by NR so every ring slot is a static register;
//     each output thus accumulates one partial per PSF row, in dy order;
//   * when output o = i - (NR-1) is complete: scale by 1/count and apply the
//     fused quotient / update epilogue, float4 store.
#include <cstdlib>

#include "common.cuh"

namespace fdg {
namespace {

constexpr int S = 8;  // rows in flight
constexpr int R = 4;  // rows per mbarrier stage
constexpr int SS = S / R;

// ---- compile-time span tables (dy = MINDY + r)
struct DiscR10 {
    static constexpr int NR = 21, MINDY = -10;
    __host__ __device__ static constexpr int LO(int r) {
        constexpr int t[NR] = {0, -4, -6, -7, -8, -8, -9, -9, -9, -9, -10, -9, -9, -9, -9, -8, -8, -7, -6, -4, 0};
        return t[r];
    }
    __host__ __device__ static constexpr int HI(int r) { return -LO(r); }
};
struct Oblique21 {
    static constexpr int NR = 11, MINDY = -5;
    __host__ __device__ static constexpr int LO(int r) {
        constexpr int t[NR] = {8, 6, 4, 3, 1, -1, -3, -4, -6, -8, -9};
        return t[r];
    }
    __host__ __device__ static constexpr int HI(int r) {
        constexpr int t[NR] = {9, 8, 6, 4, 3, 1, -1, -3, -4, -6, -8};
        return t[r];
    }
};

template <class SH, int NT>
struct Ext {
    static constexpr int CW = 4 * NT;
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
    static constexpr int count() {
        int n = 0;
        for (int r = 0; r < SH::NR; ++r) n += SH::HI(r) - SH::LO(r) + 1;
        return n;
    }
    static constexpr int XL = xl(), XR = xr();
    static constexpr int HL = (XL + 3) / 4 * 4, HR = (XR + 3) / 4 * 4;
    static constexpr int OFF = HL - XL;                     // window start within its first chunk
    static constexpr int NWIN = 4 + XL + XR;                // window values per thread
    static constexpr int NCH = (OFF + NWIN - 1) / 4 + 1;    // float4 chunks
    static constexpr int SEG = CW + HL + HR + 8;
};

struct SpanArgs {
    const float* in;
    const float* aux;
    float* out;
    int pitch, W, Wp4;
    int y0, y1, ylo, yhi, band;
    long long bstride;
    float scale, eps;
    int clamp;
    unsigned* maxchange;
    int* nanflag;
};

template <int MODE>
__device__ __forceinline__ float epi1(float v, float x, float eps, int clamp, float& maxd, float& csum) {
    if (MODE == EPI_STORE) return v;
    if (MODE == EPI_QUOT) return div_fast(x, v < eps ? eps : v);
    float value = v * x;
    if (clamp && value < 0.f) value = 0.f;
    maxd = fmaxf(maxd, fabsf(value - x));
    csum += value;
    return value;
}

template <int MODE, class SH, int NT>
__global__ void __launch_bounds__(NT + 32, 2) k_spans(const SpanArgs a) {
    using E = Ext<SH, NT>;
    constexpr int CW = E::CW;
    constexpr int NR = SH::NR;
    constexpr bool HAS_AUX = MODE != EPI_STORE;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + SS;
    float* in_ring = reinterpret_cast<float*>(smem_raw + 128);
    float* aux_ring = in_ring + S * E::SEG;

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * CW;
    const int yb0 = a.y0 + blockIdx.y * a.band;
    const int yb1 = min(a.y1, yb0 + a.band);
    if (yb0 >= yb1) return;
    const long long img = (long long)blockIdx.z * a.bstride;
    const int rows = yb1 - yb0;
    const int steps = rows + NR - 1;

    if (tid == 0) {
        for (int s = 0; s < SS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NT / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (tid >= NT) {  // producer
        if (tid == NT) {
            const int c0 = max(0, x0 - E::HL);
            const int c1 = min(a.Wp4, x0 + CW + E::HR);
            const unsigned in_bytes = (unsigned)(c1 - c0) * 4u;
            const int dst_off = c0 - (x0 - E::HL);
            const unsigned aux_bytes = (unsigned)(min(a.Wp4, x0 + CW) - x0) * 4u;
            for (int i0 = 0, st = 0; i0 < steps; i0 += R, ++st) {
                const int s = st % SS;
                if (st >= SS) mbar_wait(&empty[s], ((st / SS) - 1) & 1);
                const int nr = min(R, steps - i0);
                const int naux = HAS_AUX ? max(0, min(nr, i0 + nr - (NR - 1))) : 0;
                mbar_arrive_expect_tx(&full[s], nr * in_bytes + naux * aux_bytes);
                for (int r = 0; r < nr; ++r) {
                    const int i = i0 + r;
                    const int row = clampi(yb0 + SH::MINDY + i, a.ylo, a.yhi);
                    bulk_g2s(in_ring + (size_t)(s * R + r) * E::SEG + dst_off,
                             a.in + img + (long long)row * a.pitch + c0, in_bytes, &full[s]);
                    if (HAS_AUX && i >= NR - 1)
                        bulk_g2s(aux_ring + (size_t)(s * R + r) * CW,
                                 a.aux + img + (long long)(yb0 + i - (NR - 1)) * a.pitch + x0, aux_bytes, &full[s]);
                }
            }
        }
        return;
    }

    const int lane = tid & 31;
    const int xc = x0 + 4 * tid;
    const bool interior = (x0 - E::XL >= 0) && (x0 + CW - 1 + E::XR <= a.W - 1);
    const int sb = x0 - E::HL;  // image column of segment position 0
    const bool full_store = xc + 3 < a.W;
    const float scale = a.scale, eps = a.eps;
    const int clamp = a.clamp;
    float maxd = 0.f, csum = 0.f;
    float4 acc[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    float* outp = a.out + img + (long long)yb0 * a.pitch + xc;
    int s = 0, rr = 0;
    unsigned phase = 0;

    for (int base = 0; base < steps; base += NR) {
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const int i = base + j;
            if (i >= steps) break;
            if (rr == 0) mbar_wait(&full[s], phase);
            const float* seg = in_ring + (size_t)(s * R + rr) * E::SEG;
            // window values w[k] = image column xc - XL + k, k < NWIN
            float w[E::NWIN];
            if (interior) {
                float v[4 * E::NCH];
                const float4* p = reinterpret_cast<const float4*>(seg + 4 * tid);
#pragma unroll
                for (int c = 0; c < E::NCH; ++c) {
                    const float4 q = p[c];
                    v[4 * c] = q.x;
                    v[4 * c + 1] = q.y;
                    v[4 * c + 2] = q.z;
                    v[4 * c + 3] = q.w;
                }
#pragma unroll
                for (int k = 0; k < E::NWIN; ++k) w[k] = v[E::OFF + k];
            } else {
#pragma unroll
                for (int k = 0; k < E::NWIN; ++k) w[k] = seg[clampi(xc - E::XL + k, 0, a.W - 1) - sb];
            }
            // inclusive prefix over the window (restarts every row)
            float P[E::NWIN];
            P[0] = w[0];
#pragma unroll
            for (int k = 1; k < E::NWIN; ++k) P[k] = P[k - 1] + w[k];
            // scatter every span row's 4 window sums into its pending output
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const int lo = SH::LO(r) + E::XL, hi = SH::HI(r) + E::XL;
                float4& t = acc[((j - r) % NR + NR) % NR];
                t.x += P[hi] - (lo > 0 ? P[lo - 1] : 0.f);
                t.y += P[hi + 1] - P[lo];
                t.z += P[hi + 2] - P[lo + 1];
                t.w += P[hi + 3] - P[lo + 2];
            }
            // output o = i - (NR-1) is complete: its accumulator is slot (j+1) % NR
            float4& done = acc[(j + 1) % NR];
            if (i >= NR - 1) {
                float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
                if (HAS_AUX) x = *reinterpret_cast<const float4*>(aux_ring + (size_t)(s * R + rr) * CW + 4 * tid);
                float4 v = make_float4(done.x * scale, done.y * scale, done.z * scale, done.w * scale);
                if (!full_store) {
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
                outp += a.pitch;
            }
            done = make_float4(0.f, 0.f, 0.f, 0.f);  // the slot starts output o + NR next step
            if (++rr == R || i == steps - 1) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                rr = 0;
                if (++s == SS) {
                    s = 0;
                    phase ^= 1u;
                }
            }
        }
    }
    if (MODE == EPI_UPDATE && a.maxchange) {
        const unsigned bits = __reduce_max_sync(0xffffffffu, __float_as_uint(maxd));
        const int nan = __reduce_or_sync(0xffffffffu, (int)isnan(csum));
        if (lane == 0) {
            if (bits) atomicMax(a.maxchange, bits);
            if (nan) atomicOr(a.nanflag, 1);
        }
    }
}

template <int MODE, class SH, int NT>
cudaError_t launch_t(const SpanArgs& a, dim3 grid, cudaStream_t st) {
    using E = Ext<SH, NT>;
    const size_t smem = 128 + sizeof(float) * ((size_t)S * E::SEG + (size_t)S * E::CW);
    cudaError_t err = smem_attr<k_spans<MODE, SH, NT>>();
    if (err != cudaSuccess) return err;
    k_spans<MODE, SH, NT><<<grid, NT + 32, smem, st>>>(a);
    return cudaGetLastError();
}

template <class SH>
bool same_shape(const DevPsf& p) {
    if (p.nrows != SH::NR || p.min_dy != SH::MINDY || (int)p.h_span.size() != 2 * SH::NR) return false;
    for (int r = 0; r < SH::NR; ++r)
        if (p.h_span[2 * r] != SH::LO(r) || p.h_span[2 * r + 1] != SH::HI(r)) return false;
    return true;
}

template <class SH, int NT>
cudaError_t launch_nt(SpanArgs a, const Geom& g, const Epi& e, cudaStream_t st) {
    constexpr int CW = 4 * NT;
    const int strips = (g.W + CW - 1) / CW;
    const int rows = g.y1 - g.y0;
    if (rows <= 0) return cudaSuccess;
    // Enough CTAs to fill the machine twice over (2 resident per SM by
    // registers); bands no shorter than 1.5 NR (the NR-1 halo rows are
    // recomputed per band).  Measured on cfg1/cfg2: profiles/r01_spans_notes.md
    static const int band_env = [] {
        const char* v = getenv("FDG_SPANS_BAND");
        return v ? atoi(v) : 0;
    }();
    const long long want = (long long)148 * 2 * 2;
    int band = (int)(((long long)rows * strips * g.batch + want - 1) / want);
    const int bmin = max(16, 3 * SH::NR / 2);
    band = band < bmin ? bmin : (band > 256 ? 256 : band);
    if (band_env > 0) band = band_env;
    a.band = band;
    dim3 grid(strips, (rows + band - 1) / band, g.batch);
    switch (e.mode) {
        case EPI_STORE: return launch_t<EPI_STORE, SH, NT>(a, grid, st);
        case EPI_QUOT: return launch_t<EPI_QUOT, SH, NT>(a, grid, st);
        case EPI_UPDATE: return launch_t<EPI_UPDATE, SH, NT>(a, grid, st);
    }
    return cudaErrorInvalidValue;
}

template <class SH>
cudaError_t launch_shape(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st) {
    SpanArgs a;
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
    a.scale = p.scale;
    a.eps = e.eps;
    a.clamp = e.clamp;
    a.maxchange = e.maxchange;
    a.nanflag = e.nanflag;
    static const int nt_env = [] {
        const char* v = getenv("FDG_SPANS_NT");
        return v ? atoi(v) : 0;
    }();
    // narrow images: 256-column strips give more CTAs for the same band
    const bool narrow = nt_env ? nt_env == 64 : (long long)g.W * (g.y1 - g.y0) * g.batch <= 8ll << 20;
    return narrow ? launch_nt<SH, 64>(a, g, e, st) : launch_nt<SH, 128>(a, g, e, st);
}

}  // namespace

bool spans_supported(const DevPsf& p) {
    if (getenv("FDG_NO_SPANS")) return false;
    return same_shape<DiscR10>(p) || same_shape<Oblique21>(p);
}

cudaError_t launch_spans(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st) {
    if (same_shape<DiscR10>(p)) return launch_shape<DiscR10>(p, g, e, st);
    if (same_shape<Oblique21>(p)) return launch_shape<Oblique21>(p, g, e, st);
    return cudaErrorNotSupported;
}

}  // namespace fdg
