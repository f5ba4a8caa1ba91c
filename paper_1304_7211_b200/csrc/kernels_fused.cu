// kernels_fused.cu -- one launch per Richardson-Lucy iteration for centred
// separable boxes (Box2d*, config 4): both convolutions, the quotient and the
// multiplicative update fused, q never leaving the SM.
//
//   u_out = max( box*( f / max(box(u_in), eps) ) * u_in, 0 )
//
// HBM traffic per iteration: read u_in (+ halo rows), read f, write u_out =
// 12 B/px instead of 24 B/px for the two-pass engines.  u ping-pongs between
// two planes (neighbouring bands read u_in halos while others write u_out).
//
// A CTA owns CW output columns of a row band and marches down u rows
// j = qr_lo - RY ... yb1 - 1 + 2 RY (qr_lo..qr_hi = the q rows the band needs,
// clamped to the readable rows).  A producer warp streams, per step, the
// replicate-clamped u row j (CW + 4 HX columns), the f row j - RY and the u
// row j - 2 RY of the output (TMA bulk copies, R rows per mbarrier stage).
// Consumers (4 columns / thread):
//   A  H1 = horizontal box sum of u row j over the q columns (CW + 2 HX);
//      vertical running sum over the last MY H1 rows (smem ring) -> v row
//      j - RY -> q = f / max(v / (MX MY), eps), clamped to the image columns,
//      into a double-buffered shared q row;              named barrier
//   B  H2 = horizontal box sum of the q row over the output columns; pushed
//      (once, or RY+1 times at the top image edge, or repeated at the bottom
//      edge -- replicate clamping of q) into a vertical ring -> c row ->
//      u_out = max(c / (MX MY) * u, 0) with max|du| and the NaN checksum.
// Window sums are formed by additions only; vertical running sums are
// rebuilt from their rings every 32 rows (fp32 drift, SURVEY 7 part 1).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace fdg {
namespace {

constexpr int REFRESH = 32;

template <int RX, int RY, int NT>
struct FG {
    static constexpr int MX = 2 * RX + 1, MY = 2 * RY + 1;
    static constexpr int CW = 4 * NT;           // output columns
    static constexpr int HX = (RX + 3) / 4 * 4; // aligned horizontal halo
    static constexpr int QW = CW + 2 * HX;      // q columns
    static constexpr int UW = CW + 4 * HX;      // u columns of a streamed row
    static constexpr int NQT = QW / 4;          // stage-A threads
    static constexpr int NCT = ((NQT + 31) / 32) * 32;  // consumer threads
    static constexpr int USEG = UW + 8, QSEG = QW + 8;
    static constexpr int OFF = HX - RX;         // window start inside its chunk
};

struct FusedArgs {
    const float* u_in;
    const float* f;
    float* u_out;
    int pitch, W, Wp4;
    int H;  // rows of the image (clamp range [0, H-1])
    int band, batch;
    long long bstride;
    float scale, eps;
    int clamp;
    unsigned* maxchange;
    int* nanflag;
};

template <int MX, int OFF>
__device__ __forceinline__ float4 hsum_fast(const float* seg, int chunk) {
    constexpr int NCH = (OFF + 3 + MX - 1) / 4 + 1;
    float v[4 * NCH];
    const float4* p = reinterpret_cast<const float4*>(seg) + chunk;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const float4 q = p[c];
        v[4 * c] = q.x;
        v[4 * c + 1] = q.y;
        v[4 * c + 2] = q.z;
        v[4 * c + 3] = q.w;
    }
    float mid = 0.f;
#pragma unroll
    for (int k = 3; k < MX; ++k) mid += v[OFF + k];
    const float l2 = v[OFF + 2], l1 = v[OFF + 1] + l2, l0 = v[OFF] + l1;
    const float r1 = v[OFF + MX], r2 = r1 + v[OFF + MX + 1], r3 = r2 + v[OFF + MX + 2];
    return make_float4(l0 + mid, (l1 + mid) + r1, (l2 + mid) + r2, mid + r3);
}

// clamped variant: column c of the window sum uses image columns
// clamp(cc, 0, W-1) where cc = clamp(c, 0, W-1) + dx  (q columns outside the
// image are replaced by the clamped column's value -- replicate semantics)
template <int MX>
__device__ __forceinline__ float4 hsum_clamped(const float* seg, int seg_col0, int c0, int rx, int W, bool clamp_out) {
    float h[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int c = clamp_out ? clampi(c0 + j, 0, W - 1) : c0 + j;
        float s = 0.f;
        for (int k = 0; k < MX; ++k) s += seg[clampi(c - rx + k, 0, W - 1) - seg_col0];
        h[j] = s;
    }
    return make_float4(h[0], h[1], h[2], h[3]);
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void add4(float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
}
__device__ __forceinline__ void sub4(float4& a, const float4& b) {
    a.x -= b.x;
    a.y -= b.y;
    a.z -= b.z;
    a.w -= b.w;
}

template <int RX, int RY, int NT, int R, int S>
__global__ void __launch_bounds__(FG<RX, RY, NT>::NCT + 32) k_fused(const FusedArgs a) {
    using G = FG<RX, RY, NT>;
    constexpr int SS = S / R;
    constexpr int MY = G::MY;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + SS;
    float* uring = reinterpret_cast<float*>(smem_raw + 256);
    float* fring = uring + S * G::USEG;
    float* aring = fring + S * G::QSEG;
    float* qbuf = aring + S * G::CW;            // 2 x QSEG
    float4* v1 = reinterpret_cast<float4*>(qbuf + 2 * G::QSEG);  // MY x NQT
    float4* v2 = v1 + MY * G::NQT;                                // MY x NT

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * G::CW;
    const int yb0 = blockIdx.y * a.band;
    const int yb1 = min(a.H, yb0 + a.band);
    if (yb0 >= yb1) return;
    const long long img = (long long)blockIdx.z * a.bstride;
    const int qr_lo = max(0, yb0 - RY), qr_hi = min(a.H - 1, yb1 - 1 + RY);
    const int j0 = qr_lo - RY;                 // first streamed u row (may be < 0: clamped)
    const int steps = (yb1 - 1 + 2 * RY) - j0 + 1;

    if (tid == 0) {
        for (int s = 0; s < SS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], G::NCT / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (tid >= G::NCT) {  // producer warp
        if (tid == G::NCT) {
            const int uc0 = max(0, x0 - 2 * G::HX), uc1 = min(a.Wp4, x0 + G::CW + 2 * G::HX);
            const unsigned ubytes = (unsigned)(uc1 - uc0) * 4u;
            const int udst = uc0 - (x0 - 2 * G::HX);
            const int fc0 = max(0, x0 - G::HX), fc1 = min(a.Wp4, x0 + G::CW + G::HX);
            const unsigned fbytes = (unsigned)(fc1 - fc0) * 4u;
            const int fdst = fc0 - (x0 - G::HX);
            const unsigned abytes = (unsigned)(min(a.Wp4, x0 + G::CW) - x0) * 4u;
            for (int i0 = 0, st = 0; i0 < steps; i0 += R, ++st) {
                const int s = st % SS;
                if (st >= SS) mbar_wait(&empty[s], ((st / SS) - 1) & 1);
                const int nr = min(R, steps - i0);
                unsigned bytes = 0;
                for (int r = 0; r < nr; ++r) {
                    const int j = j0 + i0 + r;
                    bytes += ubytes;
                    if (j - RY >= qr_lo && j - RY <= qr_hi) bytes += fbytes;
                    if (j - 2 * RY >= yb0 && j - 2 * RY < yb1) bytes += abytes;
                }
                mbar_arrive_expect_tx(&full[s], bytes);
                for (int r = 0; r < nr; ++r) {
                    const int j = j0 + i0 + r;
                    const int slot = s * R + r;
                    bulk_g2s(uring + (size_t)slot * G::USEG + udst,
                             a.u_in + img + (long long)clampi(j, 0, a.H - 1) * a.pitch + uc0, ubytes, &full[s]);
                    if (j - RY >= qr_lo && j - RY <= qr_hi)
                        bulk_g2s(fring + (size_t)slot * G::QSEG + fdst,
                                 a.f + img + (long long)(j - RY) * a.pitch + fc0, fbytes, &full[s]);
                    if (j - 2 * RY >= yb0 && j - 2 * RY < yb1)
                        bulk_g2s(aring + (size_t)slot * G::CW,
                                 a.u_in + img + (long long)(j - 2 * RY) * a.pitch + x0, abytes, &full[s]);
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------- consumers
    const int lane = tid & 31;
    const bool doA = tid < G::NQT, doB = tid < NT;
    const int qc = x0 - G::HX + 4 * tid;  // first q column of this thread (stage A)
    const int oc = x0 + 4 * tid;          // first output column (stage B)
    // warp-uniform edge decisions
    const int wfirstA = x0 - G::HX + 128 * (tid >> 5);
    const bool edgeA = (wfirstA - RX < 0) || (wfirstA + 127 + RX > a.W - 1) || (wfirstA < 0) || (wfirstA + 127 > a.W - 1);
    const int wfirstB = x0 + 128 * (tid >> 5);
    const bool edgeB = (wfirstB - RX < 0) || (wfirstB + 127 + RX > a.W - 1);
    const bool full_store = oc + 3 < a.W;
    const float scale = a.scale, eps = a.eps;
    float4 col1 = make_float4(0.f, 0.f, 0.f, 0.f), col2 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 hlast = make_float4(0.f, 0.f, 0.f, 0.f);
    int n1 = 0, n2 = 0;  // rows pushed into the vertical rings
    float maxd = 0.f, csum = 0.f;
    float* outp = a.u_out + img + (long long)yb0 * a.pitch + oc;
    int s = 0, rr = 0;
    unsigned phase = 0;

    for (int i = 0; i < steps; ++i) {
        const int j = j0 + i;
        if (rr == 0) mbar_wait(&full[s], phase);
        const int slot = s * R + rr;
        const int qrow = j - RY;
        const bool makeq = qrow >= qr_lo && qrow <= qr_hi;
        float* qb = qbuf + (i & 1) * G::QSEG;
        // ---- stage A: H1 of u row j, vertical window -> q row j - RY
        if (doA) {
            const float* useg = uring + (size_t)slot * G::USEG;
            const float4 h = edgeA ? hsum_clamped<G::MX>(useg, x0 - 2 * G::HX, qc, RX, a.W, true)
                                   : hsum_fast<G::MX, G::OFF>(useg, tid);
            float4* rs = v1 + (size_t)(n1 % MY) * G::NQT + tid;
            if (n1 >= MY) sub4(col1, *rs);
            add4(col1, h);
            *rs = h;
            ++n1;
            if (n1 > MY && (n1 & (REFRESH - 1)) == 0) {
                float4 fr = v1[tid];
                for (int k = 1; k < MY; ++k) add4(fr, v1[(size_t)k * G::NQT + tid]);
                col1 = fr;
            }
            if (makeq) {
                const float* fseg = fring + (size_t)slot * G::QSEG;
                float4 fv = *reinterpret_cast<const float4*>(fseg + 4 * tid);
                if (edgeA) {  // q columns outside the image take the clamped column's f
                    float fx[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) fx[e] = fseg[clampi(qc + e, 0, a.W - 1) - (x0 - G::HX)];
                    fv = make_float4(fx[0], fx[1], fx[2], fx[3]);
                }
                const float d0 = col1.x * scale, d1 = col1.y * scale, d2 = col1.z * scale, d3 = col1.w * scale;
                float4 q;
                q.x = div_fast(fv.x, d0 < eps ? eps : d0);
                q.y = div_fast(fv.y, d1 < eps ? eps : d1);
                q.z = div_fast(fv.z, d2 < eps ? eps : d2);
                q.w = div_fast(fv.w, d3 < eps ? eps : d3);
                *reinterpret_cast<float4*>(qb + 4 * tid) = q;
            }
        }
        named_bar(1, G::NCT);
        // ---- stage B: H2 of q row, pushed into the vertical window
        if (doB) {
            int pushes = 0;
            if (makeq) {
                hlast = edgeB ? hsum_clamped<G::MX>(qb, x0 - G::HX, oc, RX, a.W, false)
                              : hsum_fast<G::MX, G::OFF>(qb, tid);
                pushes = (qrow == qr_lo) ? qr_lo - (yb0 - RY) + 1 : 1;
            } else if (qrow > qr_hi) {
                pushes = 1;  // replicate the last q row below the image
            }
            for (int p = 0; p < pushes; ++p) {
                float4* rs = v2 + (size_t)(n2 % MY) * NT + tid;
                if (n2 >= MY) sub4(col2, *rs);
                add4(col2, hlast);
                *rs = hlast;
                ++n2;
                if (n2 > MY && (n2 & (REFRESH - 1)) == 0) {
                    float4 fr = v2[tid];
                    for (int k = 1; k < MY; ++k) add4(fr, v2[(size_t)k * NT + tid]);
                    col2 = fr;
                }
                if (n2 >= MY) {  // output row yb0 + n2 - MY complete
                    const float* ax = aring + (size_t)slot * G::CW + 4 * tid;
                    float4 u = *reinterpret_cast<const float4*>(ax);
                    float4 c = make_float4(col2.x * scale, col2.y * scale, col2.z * scale, col2.w * scale);
                    if (!full_store) {
                        if (oc >= a.W) c.x = u.x = 0.f;
                        if (oc + 1 >= a.W) c.y = u.y = 0.f;
                        if (oc + 2 >= a.W) c.z = u.z = 0.f;
                        c.w = u.w = 0.f;
                    }
                    float val[4] = {c.x * u.x, c.y * u.y, c.z * u.z, c.w * u.w};
                    const float uo[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        if (a.clamp && val[e] < 0.f) val[e] = 0.f;
                        maxd = fmaxf(maxd, fabsf(val[e] - uo[e]));
                        csum += val[e];
                    }
                    if (full_store) {
                        *reinterpret_cast<float4*>(outp) = make_float4(val[0], val[1], val[2], val[3]);
                    } else {
                        if (oc < a.W) outp[0] = val[0];
                        if (oc + 1 < a.W) outp[1] = val[1];
                        if (oc + 2 < a.W) outp[2] = val[2];
                    }
                    outp += a.pitch;
                }
            }
        }
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
    if (a.maxchange) {
        const unsigned bits = __reduce_max_sync(0xffffffffu, __float_as_uint(maxd));
        const int nan = __reduce_or_sync(0xffffffffu, (int)isnan(csum));
        if (lane == 0) {
            if (bits) atomicMax(a.maxchange, bits);
            if (nan) atomicOr(a.nanflag, 1);
        }
    }
}

template <int RX, int RY, int NT, int R, int S>
size_t smem_bytes() {
    using G = FG<RX, RY, NT>;
    return 256 + sizeof(float) * ((size_t)S * G::USEG + (size_t)S * G::QSEG + (size_t)S * G::CW + 2 * (size_t)G::QSEG) +
           sizeof(float4) * ((size_t)G::MY * G::NQT + (size_t)G::MY * NT);
}

// Band height: whole waves of resident CTAs (one CTA per band x strip x image).
template <int RX, int RY, int NT, int R, int S>
cudaError_t launch_t(FusedArgs a, cudaStream_t st) {
    using G = FG<RX, RY, NT>;
    const size_t smem = smem_bytes<RX, RY, NT, R, S>();
    cudaError_t err = smem_attr<k_fused<RX, RY, NT, R, S>>();
    if (err != cudaSuccess) return err;
    static int occ = 0;
    if (!occ) {
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused<RX, RY, NT, R, S>, G::NCT + 32, smem);
        if (err != cudaSuccess) return err;
        if (occ < 1) occ = 1;
    }
    static const int sms = [] {
        int dev = 0, n = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n;
    }();
    const int strips = (a.W + G::CW - 1) / G::CW;
    const long long cols = (long long)strips * a.batch;
    // one wave of resident CTAs, bands no shorter than 4 MY rows (halo recompute)
    const long long per_wave = std::max(1LL, (long long)sms * occ / cols);
    const long long ctas_y = std::min(per_wave, std::max(1LL, (long long)a.H / (4 * G::MY)));
    a.band = (int)((a.H + ctas_y - 1) / ctas_y);
    if (const char* e = getenv("FDG_FUSED_BAND")) a.band = std::max(1, atoi(e));
    dim3 grid(strips, (a.H + a.band - 1) / a.band, a.batch);
    k_fused<RX, RY, NT, R, S><<<grid, G::NCT + 32, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

// Engine selection: 0 = off (default until it beats the two-pass engine on
// config 4), 1 = on; FDG_FUSED=0/1 or fdg_set_option("fused", v).
static int g_fused = getenv("FDG_FUSED") ? atoi(getenv("FDG_FUSED")) : 0;

void set_fused_mode(int v) { g_fused = v; }
int fused_mode() { return g_fused; }

bool fused_supported(int mx, int my, int min_dx, int min_dy) {
    return g_fused == 1 && mx == 15 && my == 15 && min_dx == -7 && min_dy == -7;
}

cudaError_t launch_fused(const float* u_in, const float* f, float* u_out, int pitch, int W, int H, int batch,
                         long long bstride, float scale, float eps, int clamp, unsigned* maxchange, int* nanflag,
                         cudaStream_t st) {
    FusedArgs a;
    a.u_in = u_in;
    a.f = f;
    a.u_out = u_out;
    a.pitch = pitch;
    a.W = W;
    a.Wp4 = (W + 3) & ~3;
    a.H = H;
    a.batch = batch;
    a.bstride = bstride;
    a.scale = scale;
    a.eps = eps;
    a.clamp = clamp;
    a.maxchange = maxchange;
    a.nanflag = nanflag;
    static const int variant = getenv("FDG_FUSED_V") ? atoi(getenv("FDG_FUSED_V")) : 0;
    switch (variant) {
        case 1: return launch_t<7, 7, 128, 2, 4>(a, st);
        case 2: return launch_t<7, 7, 64, 4, 8>(a, st);
        case 3: return launch_t<7, 7, 64, 2, 4>(a, st);
        default: return launch_t<7, 7, 128, 4, 8>(a, st);
    }
}

}  // namespace fdg
