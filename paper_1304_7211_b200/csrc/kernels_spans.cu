// kernels_spans.cu -- "spans" engine: row-convex uniform PSFs (GenericBox,
// convolve.hpp:177-212) whose span table is known at compile time -- the
// BASELINE disc r<=10 (config 2, 21 rows, 317 taps) and the 21 px @ 30 deg
// oblique line (config 1, 11 rows, 29 taps).
//
// Any other row-convex PSF runs the runtime-table kernel (kernels_spanr.cu).
//
// Two kernels (choice by image size in launch_shape):
//
// * k_spant, the TILE kernel (images <= 4.5 Mpx per launch: configs 1, 2) --
//   see its comment further down: a CTA loads its output tile + halo into
//   shared memory and every thread computes 4 columns x V rows.
//
// * k_spans, the MARCHING kernel (larger images): same streaming structure
//   as the box engine (kernels_rect.cu) -- a CTA marches down a column
//   strip; a producer warp streams R replicate-clamped input rows (+ halo)
//   and R epilogue-operand rows per mbarrier stage with TMA bulk copies.  In
//   CTAs whose segment reaches past column 0 or W-1 the producer also writes
//   the halo columns the copy does not cover (replicate-clamped, from global
//   memory) before it arrives on the stage barrier, so every consumer runs
//   the same float4 window code.
//
// Both compute a thread's 4 adjacent output columns the same way:
//   * per input row: float4 window loads, a register prefix sum over the
//     window (restarted every row, so fp32 cancellation stays ~1e-7
//     relative -- SURVEY 7 hard part 1), every span's 4 window sums as prefix
//     differences (static indices);
//   * the row's span sums are added into the pending outputs they feed
//     (output o = i - r for PSF row r), each output accumulating one partial
//     per PSF row, in dy order -- the two kernels produce bit-identical
//     results.  The marching kernel keeps the pending outputs in a register
//     ring (step loop unrolled by the ring length: static slots).
//
// Marching-kernel option G = 2 (FDG_SPANS_G=2; measured slower on configs 1
// and 2, profiles/r01_spans_notes.md): the PSF rows are split between two
// consumer groups that stream only the input rows their rows touch; group 0
// hands its partial sum of output o to group 1 through a shared slot
// (mbarrier pair), group 1 adds it and applies the fused epilogue.
#include <cstdlib>

#include "common.cuh"

namespace fdg {
namespace {

constexpr int S = 8;  // rows in flight
constexpr int R = 4;  // rows per mbarrier stage
constexpr int SS = S / R;
constexpr int K = 16;  // partial-sum slots between the groups

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
    static constexpr int XL = xl(), XR = xr();
    static constexpr int HL = (XL + 3) / 4 * 4, HR = (XR + 3) / 4 * 4;
    static constexpr int OFF = HL - XL;                   // window start within its first chunk
    static constexpr int NWIN = 4 + XL + XR;              // window values per thread
    static constexpr int NCH = (OFF + NWIN - 1) / 4 + 1;  // float4 chunks
    static constexpr int SEG = CW + HL + HR + 8;
};

// PSF rows [RA, RB) of group GI out of G
template <class SH, int G, int GI>
struct Part {
    static constexpr int SPLIT = (SH::NR + 1) / 2;
    static constexpr int RA = G == 1 ? 0 : (GI == 0 ? 0 : SPLIT);
    static constexpr int RB = G == 1 ? SH::NR : (GI == 0 ? SPLIT : SH::NR);
    static constexpr int NRG = RB - RA;
    static constexpr bool LAST = GI == G - 1;
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
    unsigned long long* tend;
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

struct Shared {
    uint64_t* gate;   // consumers wait here (stage full)
    uint64_t* empty;  // consumers release a stage
    uint64_t* pready;
    uint64_t* pfree;
    const float* in_ring;
    const float* aux_ring;
    float4* part;  // K x NT
};

__device__ __forceinline__ void release(uint64_t* empty, int lane) {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty);
}

// One consumer group: PSF rows [P::RA, P::RB) for the 4 columns xc..xc+3.
template <int MODE, class SH, int NT, int G, int GI>
__device__ __forceinline__ void consume(const SpanArgs& a, const Shared& sh, int t, int rows, int steps, int x0,
                                        long long img, int yb0) {
    using E = Ext<SH, NT>;
    using P = Part<SH, G, GI>;
    constexpr int CW = E::CW, NRG = P::NRG, RA = P::RA, RB = P::RB;
    constexpr bool HAS_AUX = MODE != EPI_STORE;
    const int lane = t & 31;
    const int xc = x0 + 4 * t;
    const bool full_store = xc + 3 < a.W;
    const float scale = a.scale, eps = a.eps;
    const int clamp = a.clamp;
    float maxd = 0.f, csum = 0.f;

    // input steps this group uses: output o = i - r >= 0 for some r in [RA, RB)
    // and o < rows for some r  ->  i in [RA, rows - 1 + RB)
    const int i_begin = RA, i_end = rows - 1 + RB;
    const int last_stage = (steps - 1) / R;
    int st = 0;
    for (; (st + 1) * R <= i_begin; ++st) {  // stages wholly before i_begin
        mbar_wait(&sh.gate[st % SS], (st / SS) & 1);
        release(&sh.empty[st % SS], lane);
    }
    if (i_begin % R) mbar_wait(&sh.gate[st % SS], (st / SS) & 1);

    float4 acc[NRG];
#pragma unroll
    for (int k = 0; k < NRG; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    float* outp = a.out + img + (long long)yb0 * a.pitch + xc;

    for (int base = i_begin; base < i_end; base += NRG) {
#pragma unroll
        for (int j = 0; j < NRG; ++j) {
            const int i = base + j;
            if (i >= i_end) break;
            const int rr = i & (R - 1);
            const int s = (i / R) % SS;
            if (rr == 0) mbar_wait(&sh.gate[s], ((i / R) / SS) & 1);
            const float* seg = sh.in_ring + (size_t)(s * R + rr) * E::SEG;
            // window values w[k] = image column xc - XL + k, k < NWIN
            float v[4 * E::NCH];
            const float4* p = reinterpret_cast<const float4*>(seg + 4 * t);
#pragma unroll
            for (int c = 0; c < E::NCH; ++c) {
                const float4 q = p[c];
                v[4 * c] = q.x;
                v[4 * c + 1] = q.y;
                v[4 * c + 2] = q.z;
                v[4 * c + 3] = q.w;
            }
            // inclusive prefix over the window (restarts every row); then this
            // group's span rows, scattered into their pending outputs --
            // (i - r) mod NRG is static because base = RA (mod NRG)
            float Pf[E::NWIN];
            Pf[0] = v[E::OFF];
#pragma unroll
            for (int k = 1; k < E::NWIN; ++k) Pf[k] = Pf[k - 1] + v[E::OFF + k];
#pragma unroll
            for (int r = RA; r < RB; ++r) {
                const int lo = SH::LO(r) + E::XL, hi = SH::HI(r) + E::XL;
                float4& tt = acc[((RA + j - r) % NRG + NRG) % NRG];
                tt.x += Pf[hi] - (lo > 0 ? Pf[lo - 1] : 0.f);
                tt.y += Pf[hi + 1] - Pf[lo];
                tt.z += Pf[hi + 2] - Pf[lo + 1];
                tt.w += Pf[hi + 3] - Pf[lo + 2];
            }
            // output o = i - (RB - 1) has all of this group's rows: slot (j + 1) % NRG
            float4& done = acc[(j + 1) % NRG];
            const int o = i - (RB - 1);
            if (o >= 0) {
                if (!P::LAST) {
                    const int k = o & (K - 1);
                    if (o >= K) mbar_wait(&sh.pfree[k], ((o / K) - 1) & 1);
                    sh.part[k * NT + t] = done;
                    release(&sh.pready[k], lane);
                } else {
                    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (HAS_AUX)
                        x = *reinterpret_cast<const float4*>(sh.aux_ring + (size_t)(s * R + rr) * CW + 4 * t);
                    float4 c = done;
                    if (G > 1) {
                        const int k = o & (K - 1);
                        mbar_wait(&sh.pready[k], (o / K) & 1);
                        const float4 pp = sh.part[k * NT + t];
                        release(&sh.pfree[k], lane);
                        c.x = pp.x + c.x;
                        c.y = pp.y + c.y;
                        c.z = pp.z + c.z;
                        c.w = pp.w + c.w;
                    }
                    float4 vv = make_float4(c.x * scale, c.y * scale, c.z * scale, c.w * scale);
                    if (!full_store) {
                        if (xc >= a.W) vv.x = x.x = 0.f;
                        if (xc + 1 >= a.W) vv.y = x.y = 0.f;
                        if (xc + 2 >= a.W) vv.z = x.z = 0.f;
                        vv.w = x.w = 0.f;
                    }
                    float4 ov;
                    ov.x = epi1<MODE>(vv.x, x.x, eps, clamp, maxd, csum);
                    ov.y = epi1<MODE>(vv.y, x.y, eps, clamp, maxd, csum);
                    ov.z = epi1<MODE>(vv.z, x.z, eps, clamp, maxd, csum);
                    ov.w = epi1<MODE>(vv.w, x.w, eps, clamp, maxd, csum);
                    if (full_store) {
                        *reinterpret_cast<float4*>(outp) = ov;
                    } else {
                        if (xc < a.W) outp[0] = ov.x;
                        if (xc + 1 < a.W) outp[1] = ov.y;
                        if (xc + 2 < a.W) outp[2] = ov.z;
                    }
                    outp += a.pitch;
                }
            }
            done = make_float4(0.f, 0.f, 0.f, 0.f);  // the slot starts output o + NRG next step
            if (rr == R - 1 || i == steps - 1) release(&sh.empty[s], lane);
        }
    }
    // release the rest: the stage holding step i_end - 1 (if not yet) and all later ones
    {
        const int il = i_end - 1;
        st = il / R;
        if (!((il & (R - 1)) == R - 1 || il == steps - 1)) release(&sh.empty[st % SS], lane);
        for (++st; st <= last_stage; ++st) {
            mbar_wait(&sh.gate[st % SS], (st / SS) & 1);
            release(&sh.empty[st % SS], lane);
        }
    }
    if (MODE == EPI_UPDATE && P::LAST && a.maxchange) {
        const unsigned bits = __reduce_max_sync(0xffffffffu, __float_as_uint(maxd));
        const int nan = __reduce_or_sync(0xffffffffu, (int)isnan(csum));
        if (lane == 0) {
            if (bits) atomicMax(a.maxchange, bits);
            if (nan) atomicOr(a.nanflag, 1);
            stamp_end(a.tend);
        }
    }
}

template <int MODE, class SH, int NT, int G>
__global__ void __launch_bounds__(G* NT + 32) k_spans(const SpanArgs a) {
    using E = Ext<SH, NT>;
    constexpr int CW = E::CW;
    constexpr int NR = SH::NR;
    constexpr bool HAS_AUX = MODE != EPI_STORE;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + SS;
    uint64_t* pready = empty + SS;
    uint64_t* pfree = pready + K;
    float* in_ring = reinterpret_cast<float*>(smem_raw + 512);
    float* aux_ring = in_ring + S * E::SEG;
    float4* part = reinterpret_cast<float4*>(aux_ring + S * CW);

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * CW;
    const int yb0 = a.y0 + blockIdx.y * a.band;
    const int yb1 = min(a.y1, yb0 + a.band);
    if (yb0 >= yb1) return;
    const long long img = (long long)blockIdx.z * a.bstride;
    const int rows = yb1 - yb0;
    const int steps = rows + NR - 1;
    const int sb = x0 - E::HL;  // image column of segment position 0
    const bool edge_cta = sb < 0 || sb + E::SEG > a.W;

    if (tid == 0) {
        for (int s = 0; s < SS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], G * NT / 32);
        }
        for (int k = 0; k < K; ++k) {
            mbar_init(&pready[k], NT / 32);
            mbar_init(&pfree[k], NT / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (tid >= G * NT) {  // ------------------------------------ producer warp
        const int lane = tid - G * NT;
        // TMA covers image columns [c0, c1) (16-byte aligned); in edge CTAs the
        // producer itself writes the rest of the segment -- columns left of 0
        // and right of c1 -- from global memory with replicate clamping,
        // before its arrive, so no stage waits on a fix-up pass.
        const int c0 = max(0, sb);
        const int c1 = max(c0, min(a.W & ~3, x0 + CW + E::HR));
        const unsigned in_bytes = (unsigned)(c1 - c0) * 4u;
        const int dst_off = c0 - sb;
        const int fix_lo = c0 - sb, fix_hi = c1 - sb;  // segment positions [fix_lo, fix_hi) come by TMA
        const unsigned aux_bytes = (unsigned)(min(a.Wp4, x0 + CW) - x0) * 4u;
        const int nst = (steps + R - 1) / R;
        for (int st = 0; st < nst; ++st) {
            const int s = st % SS;
            if (st >= SS) mbar_wait(&empty[s], ((st / SS) - 1) & 1);
            const int i0 = st * R;
            const int nr = min(R, steps - i0);
            const int naux = HAS_AUX ? max(0, min(nr, i0 + nr - (NR - 1))) : 0;
            if (lane == 0) {
                mbar_expect_tx(&full[s], nr * in_bytes + naux * aux_bytes);
                for (int r = 0; r < nr; ++r) {
                    const int i = i0 + r;
                    const int row = clampi(yb0 + SH::MINDY + i, a.ylo, a.yhi);
                    if (in_bytes)
                        bulk_g2s(in_ring + (size_t)(s * R + r) * E::SEG + dst_off,
                                 a.in + img + (long long)row * a.pitch + c0, in_bytes, &full[s]);
                    if (HAS_AUX && i >= NR - 1)
                        bulk_g2s(aux_ring + (size_t)(s * R + r) * CW,
                                 a.aux + img + (long long)(yb0 + i - (NR - 1)) * a.pitch + x0, aux_bytes,
                                 &full[s]);
                }
            }
            if (edge_cta) {
                // per row only columns 0 and W&~3 .. W-1 are needed: lanes 0-3
                // load the tail columns (clamped to W-1), lane 4 column 0, all
                // rows of the stage in flight at once; then shuffle into place
                const int tail = a.W & ~3;
                const int col = lane < 4 ? min(tail + lane, a.W - 1) : 0;
                float v[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int row = clampi(yb0 + SH::MINDY + i0 + min(r, nr - 1), a.ylo, a.yhi);
                    v[r] = __ldg(a.in + img + (long long)row * a.pitch + col);
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float* seg = in_ring + (size_t)(s * R + r) * E::SEG;
                    for (int b = 0; b < fix_lo; b += 32) {
                        const float x = __shfl_sync(0xffffffffu, v[r], 4);
                        if (r < nr && b + lane < fix_lo) seg[b + lane] = x;
                    }
                    for (int b = fix_hi; b < E::SEG; b += 32) {
                        const int p = b + lane;
                        const float x = __shfl_sync(0xffffffffu, v[r], clampi(sb + p - tail, 0, 3));
                        if (r < nr && p < E::SEG) seg[p] = x;
                    }
                }
                __syncwarp();
            }
            if (lane == 0) mbar_arrive(&full[s]);
        }
        return;
    }

    const Shared sh{full, empty, pready, pfree, in_ring, aux_ring, part};
    if (G == 1 || tid < NT)
        consume<MODE, SH, NT, G, 0>(a, sh, tid, rows, steps, x0, img, yb0);
    else
        consume<MODE, SH, NT, G, G - 1>(a, sh, tid - NT, rows, steps, x0, img, yb0);
}

template <int MODE, class SH, int NT, int G>
cudaError_t launch_t(const SpanArgs& a, dim3 grid, cudaStream_t st) {
    using E = Ext<SH, NT>;
    const size_t smem = 512 + sizeof(float) * ((size_t)S * E::SEG + (size_t)S * E::CW) +
                        (G > 1 ? sizeof(float4) * K * NT : 0);
    cudaError_t err = smem_attr<k_spans<MODE, SH, NT, G>>();
    if (err != cudaSuccess) return err;
    k_spans<MODE, SH, NT, G><<<grid, G * NT + 32, smem, st>>>(a);
    return cudaGetLastError();
}

template <class SH>
bool same_shape(const DevPsf& p) {
    if (p.nrows != SH::NR || p.min_dy != SH::MINDY || (int)p.h_span.size() != 2 * SH::NR) return false;
    for (int r = 0; r < SH::NR; ++r)
        if (p.h_span[2 * r] != SH::LO(r) || p.h_span[2 * r + 1] != SH::HI(r)) return false;
    return true;
}

int env_int(const char* name) {
    const char* v = getenv(name);
    return v ? atoi(v) : 0;
}

template <class SH, int NT, int G>
cudaError_t launch_nt(SpanArgs a, const Geom& g, const Epi& e, cudaStream_t st) {
    constexpr int CW = 4 * NT;
    const int strips = (g.W + CW - 1) / CW;
    const int rows = g.y1 - g.y0;
    if (rows <= 0) return cudaSuccess;
    // Enough CTAs to fill the machine twice over; bands no shorter than
    // 1.5 NR (the NR-1 halo rows are streamed again per band).  Measured on
    // cfg1/cfg2: profiles/r01_spans_notes.md
    static const int band_env = env_int("FDG_SPANS_BAND");
    const long long want = (long long)148 * 4;
    int band = (int)(((long long)rows * strips * g.batch + want - 1) / want);
    const int bmin = max(16, 3 * SH::NR / 2);
    band = band < bmin ? bmin : (band > 256 ? 256 : band);
    if (band_env > 0) band = band_env;
    a.band = band;
    dim3 grid(strips, (rows + band - 1) / band, g.batch);
    switch (e.mode) {
        case EPI_STORE: return launch_t<EPI_STORE, SH, NT, G>(a, grid, st);
        case EPI_QUOT: return launch_t<EPI_QUOT, SH, NT, G>(a, grid, st);
        case EPI_UPDATE: return launch_t<EPI_UPDATE, SH, NT, G>(a, grid, st);
    }
    return cudaErrorInvalidValue;
}


// ---------------------------------------------------------------------------
// Tile variant (k_spant): no marching.  A CTA of 32 x NTY threads owns a
// 128 x (V NTY) output tile; it loads the replicate-clamped input tile + halo
// (V NTY + NR - 1 rows x 128 + HL + HR columns) into shared memory with
// coalesced float4 loads, then each thread computes 4 columns x V rows with
// the same per-row prefix sums, the V outputs held in registers (output o
// accumulates its PSF rows in dy order).  Many more independent warps per SM
// than the marching kernel: it wins on small (L2-resident) images -- configs
// 1 and 2 -- where the marching grid cannot fill 148 SMs; the marching kernel
// wins on large ones (less halo recompute).  AP: the epilogue operand is
// loaded into registers before the tile, so its latency overlaps the stencil.
template <int MODE, class SH, int V, int NTY, bool AP, int MINB>
__global__ void __launch_bounds__(32 * NTY, MINB) k_spant(const SpanArgs a) {
    using E = Ext<SH, 32>;
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
    // epilogue operand of this thread's 4 columns at row y (a valid row)
    auto ld_aux = [&](int y) {
        const int xq = x0 + 4 * tx;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (MODE == EPI_STORE || xq >= a.W) return x;
        const long long idx = img + (long long)y * a.pitch + xq;
        if (xq + 3 < a.W) {
            x = __ldg(reinterpret_cast<const float4*>(a.aux + idx));
        } else {
            x.x = a.aux[idx];
            if (xq + 1 < a.W) x.y = a.aux[idx + 1];
            if (xq + 2 < a.W) x.z = a.aux[idx + 2];
        }
        return x;
    };
    float4 pre[AP ? V : 1];
    if constexpr (AP) {
#pragma unroll
        for (int o = 0; o < V; ++o) pre[o] = ld_aux(min(yt0 + ty * V + o, a.y1 - 1));
    }
    constexpr int NQ = TC / 4;
    const bool col_interior = sb >= 0 && sb + TC <= a.W;
    // Tile load in NBAND row bands, each tracked by its own mbarrier (every
    // thread's copies of a band complete -> cp.async.mbarrier.arrive), so a
    // warp starts on its first input rows while later bands are in flight
    // (one wave of tiles: nothing else hides the load).  Interior chunks are
    // 16-byte cp.async, chunks straddling the image edge 4-byte cp.async from
    // clamped columns.
    // (measured: 4 bands +4 % on config 1's oblique line, -7 % on config 2's
    // disc, whose 8 warps x 7 rows need most of the tile at once: 1 band)
    constexpr int NBAND = SH::NR > 16 ? 1 : 4, BR = (TR + NBAND - 1) / NBAND;
    __shared__ __align__(8) uint64_t bars[NBAND];
    if constexpr (NBAND > 1) {
        if (threadIdx.x == 0) {
#pragma unroll
            for (int b = 0; b < NBAND; ++b) mbar_init(&bars[b], 32 * NTY);
            mbar_fence_init();
        }
        __syncthreads();
    }
#pragma unroll
    for (int b = 0; b < NBAND; ++b) {
        const int t0 = b * BR, t1 = min(TR, t0 + BR);
        for (int k = t0 * NQ + threadIdx.x; k < t1 * NQ; k += 32 * NTY) {
            const int t = k / NQ, q = k - t * NQ;
            const int row = clampi(yt0 + SH::MINDY + t, a.ylo, a.yhi);
            const float* rp = src + (long long)row * a.pitch;
            const int c = sb + 4 * q;
            float* dst = tile + t * TCP + 4 * q;
            if (col_interior || (c >= 0 && c + 3 < a.W)) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(rp + c) : "memory");
            } else if (NBAND > 1) {  // tracked by the band's mbarrier too
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst + j)),
                                 "l"(rp + clampi(c + j, 0, a.W - 1))
                                 : "memory");
            } else {
                float4 v;
                v.x = __ldg(rp + clampi(c, 0, a.W - 1));
                v.y = __ldg(rp + clampi(c + 1, 0, a.W - 1));
                v.z = __ldg(rp + clampi(c + 2, 0, a.W - 1));
                v.w = __ldg(rp + clampi(c + 3, 0, a.W - 1));
                *reinterpret_cast<float4*>(dst) = v;
            }
        }
        if constexpr (NBAND > 1)
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&bars[b])) : "memory");
    }
    if constexpr (NBAND == 1) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    }
    float4 acc[V];
#pragma unroll
    for (int o = 0; o < V; ++o) acc[o] = make_float4(0.f, 0.f, 0.f, 0.f);
    const float* base = tile + (ty * V) * TCP + 4 * tx;
#pragma unroll
    for (int tl = 0; tl < V + NR - 1; ++tl) {
        {
            const int row = ty * V + tl;
            if (NBAND > 1 && (tl == 0 || row % BR == 0)) mbar_wait(&bars[row / BR], 0);  // band landed
        }
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
            // packed accumulate (FADD2, same rounding per lane): +3 % on configs 1 / 2
            const float2 d01 = make_float2(Pf[hi] - (lo > 0 ? Pf[lo - 1] : 0.f), Pf[hi + 1] - Pf[lo]);
            const float2 d23 = make_float2(Pf[hi + 2] - Pf[lo + 1], Pf[hi + 3] - Pf[lo + 2]);
            const float2 a01 = __fadd2_rn(make_float2(acc[o].x, acc[o].y), d01);
            const float2 a23 = __fadd2_rn(make_float2(acc[o].z, acc[o].w), d23);
            acc[o] = make_float4(a01.x, a01.y, a23.x, a23.y);
        }
    }
    const int xc = x0 + 4 * tx;
    if (xc >= a.W) return;
    const bool full_store = xc + 3 < a.W;
    const float scale = a.scale, eps = a.eps;
    const int clamp = a.clamp;
    float maxd = 0.f, csum = 0.f;
    const int yo0 = yt0 + ty * V;
#pragma unroll
    for (int o = 0; o < V; ++o) {
        const int y = yo0 + o;
        if (y >= a.y1) break;
        const long long idx = img + (long long)y * a.pitch + xc;
        float4 x = AP ? pre[AP ? o : 0] : ld_aux(y);  // loaded after the row check: not hoisted
        float4 vv = make_float4(acc[o].x * scale, acc[o].y * scale, acc[o].z * scale, acc[o].w * scale);
        if (!full_store) {
            if (xc + 1 >= a.W) vv.y = x.y = 0.f;
            if (xc + 2 >= a.W) vv.z = x.z = 0.f;
            vv.w = x.w = 0.f;
        }
        float4 ov;
        ov.x = epi1<MODE>(vv.x, x.x, eps, clamp, maxd, csum);
        ov.y = epi1<MODE>(vv.y, x.y, eps, clamp, maxd, csum);
        ov.z = epi1<MODE>(vv.z, x.z, eps, clamp, maxd, csum);
        ov.w = epi1<MODE>(vv.w, x.w, eps, clamp, maxd, csum);
        float* op = a.out + idx;
        if (full_store) {
            *reinterpret_cast<float4*>(op) = ov;
        } else {
            op[0] = ov.x;
            if (xc + 1 < a.W) op[1] = ov.y;
            if (xc + 2 < a.W) op[2] = ov.z;
        }
    }
    if (MODE == EPI_UPDATE && a.maxchange) {
        const unsigned bits = __reduce_max_sync(__activemask(), __float_as_uint(maxd));
        const int nan = __reduce_or_sync(__activemask(), (int)isnan(csum));
        if (bits && (bits == __float_as_uint(maxd))) atomicMax(a.maxchange, bits);
        if (nan && isnan(csum)) atomicOr(a.nanflag, 1);
        if ((threadIdx.x & 31) == (unsigned)(__ffs(__activemask()) - 1)) stamp_end(a.tend);
    }
}

template <int MODE, class SH, int V, int NTY, bool AP, int MINB>
cudaError_t launch_tile_t(const SpanArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
    cudaError_t err = smem_attr<k_spant<MODE, SH, V, NTY, AP, MINB>>();
    if (err != cudaSuccess) return err;
    k_spant<MODE, SH, V, NTY, AP, MINB><<<grid, 32 * NTY, smem, st>>>(a);
    return cudaGetLastError();
}

template <class SH, int V, int NTY, bool AP, int MINB = 1>
cudaError_t launch_tile(const SpanArgs& a, const Geom& g, const Epi& e, cudaStream_t st) {
    using E = Ext<SH, 32>;
    constexpr int TH = V * NTY;
    const size_t smem = sizeof(float) * (TH + SH::NR - 1) * (128 + E::HL + E::HR + 4);
    const int rows = g.y1 - g.y0;
    if (rows <= 0) return cudaSuccess;
    dim3 grid((g.W + 127) / 128, (rows + TH - 1) / TH, g.batch);
    switch (e.mode) {
        case EPI_STORE: return launch_tile_t<EPI_STORE, SH, V, NTY, AP, MINB>(a, grid, smem, st);
        case EPI_QUOT: return launch_tile_t<EPI_QUOT, SH, V, NTY, AP, MINB>(a, grid, smem, st);
        case EPI_UPDATE: return launch_tile_t<EPI_UPDATE, SH, V, NTY, AP, MINB>(a, grid, smem, st);
    }
    return cudaErrorInvalidValue;
}

// Largest launch (pixels) the tile kernel takes before the marching kernel
// does.  Measured per RL iteration (profiles/r02_engine_probe_4096.txt): the
// disc's tiles lead at every size tried (4096^2: 140 vs 173 us, 6144^2: 280 vs
// 331), the oblique line's up to 2560^2 (43 vs 54 us; 3072^2: 67 vs 54).
template <class SH>
constexpr long long tile_limit() {
    return SH::NR > 16 ? (128ll << 20) : (7ll << 20);
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
    a.tend = e.tend;
    static const int nt_env = env_int("FDG_SPANS_NT");
    static const int g_env = env_int("FDG_SPANS_G");
    // Small images: the tile kernel -- the marching grid cannot fill the SMs
    // (profiles/r01_spans_notes.md); larger ones march (tile_limit).
    // fdg_set_option("spans", 1 | 2) forces one (tests, A/B).
    const long long px = (long long)g.W * (g.y1 - g.y0) * g.batch;
    const int mode = spans_mode();
    const bool tile = mode ? mode == 1 : px <= tile_limit<SH>();
    if (tile) {
        // disc: 128 x 56 tiles, 64 registers forced (4 CTAs = 32 warps per SM;
        // the register count of this kernel otherwise drifts between builds,
        // and 3 CTAs/SM costs a second wave).  2048^2: 37 x 16 = 592 tiles =
        // exactly one wave of 148 x 4 (128 x 64 tiles: 512 = 0.86 wave, 102k;
        // 128 x 56: 108k Mpx*it/s on config 2)
        if constexpr (SH::NR > 16) {
            return launch_tile<SH, 7, 8, false, 4>(a, g, e, st);
        } else {
            // oblique: 128 x 28 tiles (7 warps x 4 rows), aux prefetch, <= 64
            // registers; 1024^2: 37 x 8 = 296 tiles = 2 per SM (128 x 32:
            // 256 tiles, 1-2 per SM: 83.0k; 128 x 28: 85.2k Mpx*it/s)
            return launch_tile<SH, 4, 7, true, 4>(a, g, e, st);
        }
    }
    // marching: 256-column strips give more CTAs for the same band on narrow images
    const bool narrow = nt_env ? nt_env == 64 : px <= 8ll << 20;
    if (g_env == 2) return narrow ? launch_nt<SH, 64, 2>(a, g, e, st) : launch_nt<SH, 128, 2>(a, g, e, st);
    return narrow ? launch_nt<SH, 64, 1>(a, g, e, st) : launch_nt<SH, 128, 1>(a, g, e, st);
}

std::atomic<int> g_spans_mode{env_int("FDG_SPANS_TILE")};

}  // namespace

void set_spans_mode(int v) { g_spans_mode.store(v); }
int spans_mode() { return g_spans_mode.load(); }

bool spans_supported(const DevPsf& p) {
    if (getenv("FDG_NO_SPANS")) return false;
    return same_shape<DiscR10>(p) || same_shape<Oblique21>(p) || spanr_supported(p);
}

// compile-time tables first (unless spans mode 3 forces the runtime-table
// kernel, for A/B and tests), then the runtime-table kernel (kernels_spanr.cu)
cudaError_t launch_spans(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st) {
    if (spans_mode() != 3) {
        if (same_shape<DiscR10>(p)) return launch_shape<DiscR10>(p, g, e, st);
        if (same_shape<Oblique21>(p)) return launch_shape<Oblique21>(p, g, e, st);
        // any other table: the tile kernel compiled for it at plan time (NVRTC)
        if (spans_jit_mode() && spans_jit_ready(p)) {
            const cudaError_t r = launch_spans_jit(p, g, e, st);
            if (r != cudaErrorNotSupported) return r;  // else the JIT build failed: runtime-table kernel
        }
    }
    return launch_spanr(p, g, e, st);
}

const char* spans_kernel(const DevPsf& p, long long px) {
    if (spans_mode() != 3 && (same_shape<DiscR10>(p) || same_shape<Oblique21>(p))) {
        const int mode = spans_mode();
        const long long lim = same_shape<DiscR10>(p) ? tile_limit<DiscR10>() : tile_limit<Oblique21>();
        return (mode ? mode == 1 : px <= lim) ? "tile" : "marching";
    }
    if (spans_mode() != 3 && spans_jit_mode() && spans_jit_ready(p)) return "jit-tile";
    return "runtime-table";
}

}  // namespace fdg
