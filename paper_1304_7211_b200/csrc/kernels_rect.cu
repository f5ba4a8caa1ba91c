// kernels_rect.cu -- "rows" / "box2d" engine: uniform axis-aligned boxes
// (Box1dSliding/Cumulated, Box2dSliding/Cumulated; convolve.hpp:217-388).
//
// One CTA owns a column strip of CW = 512 outputs and a band of rows and
// marches down it.  A producer warp streams one replicate-clamped input row
// segment (strip + horizontal halo) and one epilogue-operand row per step
// into an S-deep shared-memory ring with TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx); four consumer warps compute the
// horizontal box sum of 4 adjacent columns per thread from float4 shared
// loads, keep a per-column vertical running sum over the last `my` rows
// (ring of horizontal sums in shared memory, rebuilt every REFRESH rows so
// fp32 drift stays bounded -- SURVEY 7 hard part 1), and apply the fused RL
// epilogue (quotient or multiplicative update + max|du| + NaN flag) before a
// float4 store.  HBM traffic per pass: one read of the conv input, one read
// of the epilogue operand, one write (12 B/px), plus (my-1)/band halo rows.
#include <cstdlib>

#include "common.cuh"

namespace fdg {
namespace {

constexpr int NT = 128;       // consumer threads (4 columns each)
constexpr int CW = 4 * NT;    // columns per CTA
constexpr int S = 8;          // pipeline stages
constexpr int REFRESH = 16;   // vertical running-sum rebuild period
constexpr int MXMAX = 33;

struct RectArgs {
    const float* in;
    const float* aux;
    float* out;
    int pitch, W, Wp4;
    int y0, y1, ylo, yhi, band;
    long long bstride;
    int mx, my, min_dx, min_dy;
    int HL, HR, seg;
    float scale;
    Epi e;
};

// Horizontal box sums of MX taps for 4 adjacent outputs; v[] holds the
// aligned float4 chunks starting at the chunk that contains the first tap
// of output 0, which sits at position OFF within v.  Sums are formed as
// left partial + shared middle + right partial (additions only, no sliding
// subtraction), the shared middle being the MX-3 taps common to all four.
template <int MX, int OFF, int NV>
__device__ __forceinline__ void hsum4(const float (&v)[NV], float (&H)[4]) {
    if constexpr (MX >= 4) {
        float mid = 0.f;
#pragma unroll
        for (int k = 3; k < MX; ++k) mid += v[OFF + k];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float l = 0.f;
#pragma unroll
            for (int k = j; k < 3; ++k) l += v[OFF + k];
            float r = 0.f;
#pragma unroll
            for (int k = MX; k < MX + j; ++k) r += v[OFF + k];
            H[j] = (l + mid) + r;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float s = 0.f;
#pragma unroll
            for (int k = 0; k < MX; ++k) s += v[OFF + j + k];
            H[j] = s;
        }
    }
}

template <int MX, int OFF>
__device__ __forceinline__ void hsum_fast(const float* seg_row, int t, float (&H)[4]) {
    // first chunk: the one holding position HL + 4t + min_dx = 4t + OFF (+ 4*k0)
    constexpr int NCH = (OFF + 3 + MX - 1) / 4 + 1;
    float v[4 * NCH];
    const float4* p = reinterpret_cast<const float4*>(seg_row) + t;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const float4 q = p[c];
        v[4 * c] = q.x;
        v[4 * c + 1] = q.y;
        v[4 * c + 2] = q.z;
        v[4 * c + 3] = q.w;
    }
    hsum4<MX, OFF, 4 * NCH>(v, H);
}

template <int MODE, int MX, int R>
__global__ void __launch_bounds__(NT + 32) k_rect(const RectArgs a) {
    constexpr int SS = S / R;  // stages of R rows (S rows in flight)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + SS;
    float* in_ring = reinterpret_cast<float*>(smem_raw + 128);
    float* aux_ring = in_ring + S * a.seg;
    float4* hring = reinterpret_cast<float4*>(aux_ring + S * CW);

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
        for (int s = 0; s < SS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NT / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (tid >= NT) {
        // ---------------- producer warp: TMA bulk copies into the ring
        if (tid == NT) {
            const int c0 = max(0, x0 - a.HL);
            const int c1 = min(a.Wp4, x0 + CW + a.HR);
            const unsigned in_bytes = (unsigned)(c1 - c0) * 4u;
            const int dst_off = c0 - (x0 - a.HL);
            const unsigned aux_bytes = (unsigned)(min(a.Wp4, x0 + CW) - x0) * 4u;
            for (int i0 = 0, st = 0; i0 < steps; i0 += R, ++st) {
                const int s = st % SS;
                if (st >= SS) mbar_wait(&empty[s], ((st / SS) - 1) & 1);
                const int nr = min(R, steps - i0);
                const int naux = HAS_AUX ? max(0, min(nr, i0 + nr - (my - 1))) : 0;
                mbar_arrive_expect_tx(&full[s], nr * in_bytes + naux * aux_bytes);
                for (int r = 0; r < nr; ++r) {
                    const int i = i0 + r;
                    const int row = clampi(yb0 + a.min_dy + i, a.ylo, a.yhi);
                    bulk_g2s(in_ring + (size_t)(s * R + r) * a.seg + dst_off, a.in + img + (long long)row * a.pitch + c0,
                             in_bytes, &full[s]);
                    if (HAS_AUX && i >= my - 1) {
                        const int yo = yb0 + i - (my - 1);
                        bulk_g2s(aux_ring + (size_t)(s * R + r) * CW, a.aux + img + (long long)yo * a.pitch + x0,
                                 aux_bytes, &full[s]);
                    }
                }
            }
        }
        return;
    }

    // ---------------- consumers
    const int lane = tid & 31;
    const int xc = x0 + 4 * tid;  // first of this thread's 4 columns
    const bool interior = (x0 + a.min_dx >= 0) && (x0 + CW - 1 + a.min_dx + a.mx - 1 <= a.W - 1);
    const int off = a.HL + a.min_dx;  // position of output 0's first tap within the segment
    const int k0 = off >> 2, offm = off & 3;
    float4 col = make_float4(0.f, 0.f, 0.f, 0.f);
    TraceAcc tr;
    int slot = 0;

    for (int i0 = 0, st = 0; i0 < steps; i0 += R, ++st) {
      const int s = st % SS;
      mbar_wait(&full[s], (st / SS) & 1);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = i0 + r;
        if (i >= steps) break;
        const float* seg = in_ring + (size_t)(s * R + r) * a.seg;
        float H[4];
        if (interior) {
            const float* base = seg + 4 * k0;
            switch (offm) {
                case 0: hsum_fast<MX, 0>(base, tid, H); break;
                case 1: hsum_fast<MX, 1>(base, tid, H); break;
                case 2: hsum_fast<MX, 2>(base, tid, H); break;
                default: hsum_fast<MX, 3>(base, tid, H); break;
            }
        } else {
            const int sb = x0 - a.HL;  // column of seg[0]
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float acc = 0.f;
                for (int k = 0; k < MX; ++k) acc += seg[clampi(xc + j + a.min_dx + k, 0, a.W - 1) - sb];
                H[j] = acc;
            }
        }
        // vertical running sum over the last `my` horizontal sums
        float4 hv = make_float4(H[0], H[1], H[2], H[3]);
        if (my > 1) {
            float4* rs = hring + (size_t)slot * NT + tid;
            if (i >= my) {
                const float4 old = *rs;
                col.x -= old.x;
                col.y -= old.y;
                col.z -= old.z;
                col.w -= old.w;
            }
            col.x += hv.x;
            col.y += hv.y;
            col.z += hv.z;
            col.w += hv.w;
            *rs = hv;
            if (i >= my - 1 && (i % REFRESH) == 0) {
                float4 fresh = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int k = 1; k <= my; ++k) {
                    int sl = slot + k;
                    if (sl >= my) sl -= my;
                    const float4 h = hring[(size_t)sl * NT + tid];
                    fresh.x += h.x;
                    fresh.y += h.y;
                    fresh.z += h.z;
                    fresh.w += h.w;
                }
                col = fresh;
            }
            if (++slot == my) slot = 0;
        } else {
            col = hv;
        }
        if (i >= my - 1) {
            const int yo = yb0 + i - (my - 1);
            const long long rowoff = img + (long long)yo * a.pitch;
            float v[4] = {col.x * a.scale, col.y * a.scale, col.z * a.scale, col.w * a.scale};
            float res[4];
            const float* ax = aux_ring + (size_t)(s * R + r) * CW + 4 * tid;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (MODE == EPI_STORE) {
                    res[j] = v[j];
                } else if (MODE == EPI_QUOT) {
                    res[j] = div_fast(ax[j], v[j] < a.e.eps ? a.e.eps : v[j]);
                } else {  // EPI_UPDATE
                    const float u = ax[j];
                    float value = v[j] * u;
                    if (a.e.clamp && value < 0.f) value = 0.f;
                    if (xc + j < a.W) tr.add(fabsf(value - u), value);
                    res[j] = value;
                }
            }
            if (xc + 3 < a.W) {
                *reinterpret_cast<float4*>(a.out + rowoff + xc) = make_float4(res[0], res[1], res[2], res[3]);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (xc + j < a.W) a.out[rowoff + xc + j] = res[j];
            }
        }
      }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (MODE == EPI_UPDATE) trace_flush(a.e, tr);
}

template <int MODE, int MX, int R>
cudaError_t launch_r(const RectArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
    cudaError_t err = smem_attr<k_rect<MODE, MX, R>>();
    if (err != cudaSuccess) return err;
    k_rect<MODE, MX, R><<<grid, NT + 32, smem, st>>>(a);
    return cudaGetLastError();
}

template <int MODE, int MX>
cudaError_t launch_mx(const RectArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
    static const int rows_per_stage = [] {
        const char* v = getenv("FDG_RECT_R");
        return v ? atoi(v) : 4;
    }();
    if (rows_per_stage == 1) return launch_r<MODE, MX, 1>(a, grid, smem, st);
    if (rows_per_stage == 2) return launch_r<MODE, MX, 2>(a, grid, smem, st);
    return launch_r<MODE, MX, 4>(a, grid, smem, st);
}

template <int MODE, int... MXS>
cudaError_t dispatch_mx(int mx, const RectArgs& a, dim3 grid, size_t smem, cudaStream_t st,
                        std::integer_sequence<int, MXS...>) {
    cudaError_t r = cudaErrorInvalidValue;
    ((mx == MXS + 1 ? (r = launch_mx<MODE, MXS + 1>(a, grid, smem, st), true) : false) || ...);
    return r;
}

}  // namespace

bool rect_supported(int mx) { return mx >= 1 && mx <= MXMAX; }

cudaError_t launch_rect(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st) {
    if (!rect_supported(p.mx)) return cudaErrorInvalidValue;
    RectArgs a;
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
    a.mx = p.mx;
    a.my = p.my;
    a.min_dx = p.min_dx;
    a.min_dy = p.min_dy;
    const int max_dx = p.min_dx + p.mx - 1;
    a.HL = ((max(0, -p.min_dx) + 3) / 4) * 4;
    a.HR = ((max(0, max_dx) + 3) / 4) * 4;
    a.seg = CW + a.HL + a.HR + 8;  // +8: fast path may read one chunk past the window
    a.scale = p.scale;
    a.e = e;
    const int strips = (g.W + CW - 1) / CW;
    const int rows = g.y1 - g.y0;
    if (rows <= 0) return cudaSuccess;
    // band height: enough CTAs for ~6 per SM, long enough to amortise the halo
    long long want = (long long)148 * 6;
    int band = (int)(((long long)rows * strips * g.batch + want - 1) / want);
    band = band < 8 ? 8 : (band > 256 ? 256 : band);
    if (p.my > 1 && band < 4 * p.my) band = 4 * p.my;
    a.band = band;
    dim3 grid(strips, (rows + band - 1) / band, g.batch);
    const size_t smem = 128 + sizeof(float) * ((size_t)S * a.seg + (size_t)S * CW) +
                        sizeof(float4) * (size_t)NT * (p.my > 1 ? p.my : 0);
    using seq = std::make_integer_sequence<int, MXMAX>;
    switch (e.mode) {
        case EPI_STORE: return dispatch_mx<EPI_STORE>(p.mx, a, grid, smem, st, seq{});
        case EPI_QUOT: return dispatch_mx<EPI_QUOT>(p.mx, a, grid, smem, st, seq{});
        case EPI_UPDATE: return dispatch_mx<EPI_UPDATE>(p.mx, a, grid, smem, st, seq{});
    }
    return cudaErrorInvalidValue;
}

}  // namespace fdg
