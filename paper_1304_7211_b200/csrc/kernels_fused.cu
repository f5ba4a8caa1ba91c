// kernels_fused.cu -- one launch per Richardson-Lucy iteration for centred odd
// boxes 3 x 3 ... 17 x 17, square or not (Box2d*, config 4 = 15 x 15): both
// convolutions, the quotient and the multiplicative update fused, q never
// leaving the SM.
//
//   u_out = max( box*( f / max(box(u_in), eps) ) * u_in, 0 )
//
// HBM traffic per iteration: read u_in (+ halo rows), read f, write u_out =
// 12 B/px instead of 24 B/px for the two-pass engines.  u ping-pongs between
// two planes (neighbouring bands read u_in halos while others write u_out).
//
// A CTA owns CW = 4 NT - 16 output columns of a range of rows and marches
// down u rows j = qr_lo - RY ... yb1 - 1 + 2 RY (qr_lo..qr_hi = the q rows the
// range needs, clamped to the image).  Warp-specialised CTA, 2 NT + 32 threads:
//   producer warp  streams the replicate-clamped u rows (CW + 32 columns) into
//                  a shared ring with TMA bulk copies (R rows per mbarrier
//                  stage; in edge CTAs it also replicates columns 0 / W-1 into
//                  the halo) and prefetches the matching f rows into L2;
//   A warps (NT)   per u row: H1 = horizontal box sum over the CW + 16 q
//                  columns -> vertical running sum over the last MY H1 rows
//                  (shared ring) -> v -> q = f / max(v / (MX MY), eps) into a
//                  QR-row shared q ring (per-slot qfull / qempty mbarriers, A
//                  runs up to QR rows ahead of B);
//   B warps (NT)   per q row: H2 = horizontal box sum over the output columns
//                  -> vertical ring (q rows above / below the image replicated
//                  by repeated pushes) -> c -> u_out = max(c / (MX MY) * u, 0),
//                  max|du| and NaN.
// Packed fp32x2 arithmetic (FADD2 / FMUL2 / FFMA2).  Window sums are formed by
// additions only; vertical running sums are rebuilt from their rings every 32
// rows (fp32 drift, SURVEY 7 part 1).
//
// Work distribution: one wave of resident CTAs (2 per SM).  For single images
// each CTA takes an equal range of the strip-major sequence of (strip, row)
// pairs -- possibly the tail of one strip and the head of the next, run as two
// segments with the barriers re-initialised in between -- so no CTA slot idles
// (config 4: 34 strips x 8 bands would fill only 272 of 296 slots).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <type_traits>

#include "common.cuh"

namespace fdg {
namespace {

constexpr int REFRESH = 32;
// haloed u planes (fused_halo_*): replicated columns left / right of each row,
// enough for every strip's u segment [x0 - 16, x0 + 512) when W >= CW and
// W % 4 == 0 (the last strip then ends exactly at W)
constexpr int FUSED_HALO_L = 16, FUSED_HALO_R = 16;
#ifndef FDG_QSLEEP
#define FDG_QSLEEP 40
#endif

template <int RX, int RY, int NT>
struct FG {
    static constexpr int MX = 2 * RX + 1, MY = 2 * RY + 1;
    static constexpr int QW = 4 * NT;       // q columns (stage A)
    static constexpr int HX = 8;            // q halo each side (>= RX, multiple of 4)
    static constexpr int CW = QW - 2 * HX;  // output columns (stage B)
    static constexpr int NB = CW / 4;       // stage-B threads
    static constexpr int UW = QW + 2 * HX;  // u columns of a streamed row
    static constexpr int USEG = UW + 8, QSEG = QW + 16;  // B reads 4 NT + 16 q columns
    static constexpr int OFF = HX - RX;  // window start inside its chunk
    static_assert(RX <= HX && RY <= 8, "box radius");
};

struct FusedArgs {
    const float* u_in;
    const float* f;
    float* u_out;
    int pitch, W, Wp4;    // pitch: f's row pitch (elements)
    int pitch_u, pitch_o;  // row pitches of u_in / u_out
    long long bs_u, bs_o;  // image strides of u_in / u_out (batches)
    int y0, y1;    // output rows
    int y2, y3;    // optional second output row range (plain grid only: both boundary bands of a
                   // row strip in one launch); nb1 = CTA rows (blockIdx.y) of the first range
    int nb1;
    int ylo, yhi;  // readable rows; replicate clamping at these (image) edges
    int band, batch;
    int lin_len, strips;  // lin_len > 0: work-balanced row ranges over the strips (batch 1)
    long long bstride;
    float scale, eps;
    int clamp;
    unsigned* maxchange;
    int* nanflag;
    unsigned long long* tend;
    unsigned long long* probe;  // diagnostics (FDG_FUSED_PROBE): per CTA {start, end, smid, rows}
    int halo_in;   // u_in carries FUSED_HALO_L / _R replicated columns left / right of every row
    int halo_out;  // write those columns of u_out too
    int ry;        // vertical radius (read by the RY = 0 instantiations: any RY <= 8 at run time)
};

// ---- packed fp32x2 arithmetic (Blackwell FADD2 / FMUL2 / FFMA2)
__device__ __forceinline__ float2 lo2(const float4 v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(const float4 v) { return make_float2(v.z, v.w); }
__device__ __forceinline__ float4 cat4(const float2 a, const float2 b) { return make_float4(a.x, a.y, b.x, b.y); }
__device__ __forceinline__ float2 add2(const float2 a, const float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(const float2 a, const float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(const float2 a, const float2 b, const float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float4 add4(const float4 a, const float4 b) {
    return cat4(add2(lo2(a), lo2(b)), add2(hi2(a), hi2(b)));
}
__device__ __forceinline__ float4 sub4(const float4 a, const float4 b) {
    return cat4(add2(lo2(a), make_float2(-b.x, -b.y)), add2(hi2(a), make_float2(-b.z, -b.w)));
}
__device__ __forceinline__ float4 mul4s(const float4 a, const float s) {
    const float2 ss = make_float2(s, s);
    return cat4(mul2(lo2(a), ss), mul2(hi2(a), ss));
}

// 15-wide window sums of 4 consecutive columns, packed: window e covers
// v[1+e .. 15+e] of the 5 float4 chunks starting at `chunk`.
__device__ __forceinline__ float4 hsum15x4(const float* seg, int chunk) {
    const float4* p = reinterpret_cast<const float4*>(seg) + chunk;
    const float4 c0 = p[0], c1 = p[1], c2 = p[2], c3 = p[3], c4 = p[4];
    // shared middle v[4..15] = chunks 1..3 as six pairs, tree-summed
    const float2 m = add2(add2(add2(lo2(c1), hi2(c1)), add2(lo2(c2), hi2(c2))), add2(lo2(c3), hi2(c3)));
    const float mid = m.x + m.y;
    const float a = c0.z + c0.w;  // v2 + v3
    const float b = c4.x + c4.y;  // v16 + v17
    const float2 mm = make_float2(mid, mid);
    const float2 o01 = add2(add2(make_float2(c0.y, c4.x), make_float2(a, a)), mm);  // v1 + a, v16 + a
    const float2 o23 = add2(add2(make_float2(c0.w, c4.z), make_float2(b, b)), mm);  // v3 + b, v18 + b
    return cat4(o01, o23);
}

// (2 RX + 1)-wide window sums of 4 consecutive columns for any radius
// RX <= 8: window e covers v[OFF + e .. OFF + e + 2 RX] of the chunks
// starting at `chunk` (OFF = 8 - RX); additions only, the shared middle
// v[OFF + 3 .. OFF + 2 RX] formed once.  RX = 7 takes hsum15x4.
template <int RX>
__device__ __forceinline__ float4 hsumx4(const float* seg, int chunk) {
    if constexpr (RX == 7) {
        return hsum15x4(seg, chunk);
    } else if constexpr (RX == 0) {  // vertical lines: the window is the column itself
        return reinterpret_cast<const float4*>(seg)[chunk + 2];
    } else {
        constexpr int OFF = 8 - RX, LAST = OFF + 3 + 2 * RX;
        constexpr int C0 = OFF / 4, C1 = LAST / 4;
        float v[4 * (C1 + 1)];
        const float4* p = reinterpret_cast<const float4*>(seg) + chunk;
#pragma unroll
        for (int c = C0; c <= C1; ++c) {
            const float4 q = p[c];
            v[4 * c] = q.x;
            v[4 * c + 1] = q.y;
            v[4 * c + 2] = q.z;
            v[4 * c + 3] = q.w;
        }
        float mid = 0.f;
#pragma unroll
        for (int k = 3; k <= 2 * RX; ++k) mid += v[OFF + k];
        const float a = v[OFF + 1] + v[OFF + 2];
        const float b = v[OFF + 2 * RX + 1] + v[OFF + 2 * RX + 2];
        return make_float4(v[OFF] + a + mid, a + mid + v[OFF + 2 * RX + 1], v[OFF + 2] + mid + b,
                           mid + b + v[OFF + 2 * RX + 3]);
    }
}

// max that propagates NaN (the reference's clamp `value < 0 ? 0 : value`
// keeps a NaN, and a NaN anywhere must reach the per-iteration check)
__device__ __forceinline__ float fmax_nan(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// vertical running sum over a ring of MY rows of float4 (one slot per thread);
// MYT = 0: the ring height is a run-time value (rectangular boxes)
template <int MYT>
struct VRing {
    float4 col = make_float4(0.f, 0.f, 0.f, 0.f);
    int n = 0, slot = 0;
    int my_rt = 0;
    __device__ __forceinline__ int my() const { return MYT ? MYT : my_rt; }
    // steady state: the ring is full
    __device__ __forceinline__ void push_full(float4* ring, int stride, int t, const float4 h) {
        float4* rs = ring + (size_t)slot * stride + t;
        const float4 o = *rs;
        col = add4(sub4(col, o), h);
        *rs = h;
        slot = slot + 1 == my() ? 0 : slot + 1;
    }
    __device__ __forceinline__ void refresh(const float4* ring, int stride, int t) {
        float4 fr = ring[t];
#pragma unroll
        for (int k = 1; k < my(); ++k) fr = add4(fr, ring[(size_t)k * stride + t]);
        col = fr;
    }
    __device__ __forceinline__ void push(float4* ring, int stride, int t, const float4 h) {
        if (n >= my()) {
            push_full(ring, stride, t, h);
        } else {
            col = add4(col, h);
            ring[(size_t)slot * stride + t] = h;
            slot = slot + 1 == my() ? 0 : slot + 1;
        }
        ++n;
        if (n > my() && (n & (REFRESH - 1)) == 0) refresh(ring, stride, t);  // fp32 drift
    }
};

// PD: rows of u the B warps keep in flight (register prefetch depth);
// HINT: u rows streamed with L2 evict_last (the B warps re-read them ~25 rows
// later) and re-read with evict_first
template <int RX, int RY, int NT, int R, int S, int QR, int PD, bool HINT>
__global__ void __launch_bounds__(2 * NT + 32, 2) k_fused(const FusedArgs a) {
    using G = FG<RX, RY, NT>;
    static_assert(R == 2, "stage logic assumes two rows per stage");
    static_assert(G::OFF == 8 - RX, "window offset inside its chunk");
    constexpr int SS = S / R;
    constexpr int LAG = SS / 2;  // edge CTAs: the producer readies stage st - LAG
    // RY = 0: the vertical radius comes with the arguments (rectangular boxes
    // share one instantiation per RX); otherwise a compile-time constant
    const int ry = RY ? RY : a.ry;
    const int my = 2 * ry + 1;
    static_assert((QR & (QR - 1)) == 0, "q ring rows between the A and B warps: power of two");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + SS;
    uint64_t* ready = empty + SS;
    uint64_t* qfull = ready + SS;
    uint64_t* qempty = qfull + QR;
    float* uring = reinterpret_cast<float*>(smem_raw + 512);
    float* qbuf = uring + S * G::USEG;                            // ring of QR q rows
    float4* v1 = reinterpret_cast<float4*>(qbuf + QR * G::QSEG);  // my x NT
    float4* v2 = v1 + my * NT;                                    // my x NT

    const int tid = threadIdx.x;
#ifdef FDG_FUSED_PROBE
    if (a.probe && tid == 0)  // diagnostics: start stamp parked in the barrier area's spare bytes
        *reinterpret_cast<unsigned long long*>(smem_raw + 504) = globaltimer();
#endif
    const long long img = (long long)blockIdx.z * a.bstride;  // f
    const long long img_u = (long long)blockIdx.z * a.bs_u, img_o = (long long)blockIdx.z * a.bs_o;
    const long long pitch = a.pitch, pitch_u = a.pitch_u, pitch_o = a.pitch_o;
    // one column strip x0, output rows [yb0, yb1): fresh barriers, every role
    // runs its pipeline to the end of the segment
    auto run_segment = [&](const int x0, const int xown, const int yb0, const int yb1) {
        const int qr_lo = max(a.ylo, yb0 - ry), qr_hi = min(a.yhi, yb1 - 1 + ry);
        const int nq = qr_hi - qr_lo + 1;  // q rows this band needs
        const int j0 = qr_lo - ry;         // first streamed u row (may be < 0: clamped)
        const int steps = nq + 2 * ry;     // u rows streamed: j0 .. qr_hi + RY
        const int useg0 = x0 - 2 * G::HX;  // image column of u-segment index 0
        // the u segment reaches outside the image: replicate columns 0 / W-1
        // there (not needed when u_in carries replicated halo columns)
        const bool edge_cta = !a.halo_in && (useg0 < 0 || x0 + G::CW + 2 * G::HX > a.W);
        const int lo_end = max(0, -useg0);       // segment indices [0, lo_end) are left of column 0
        const int hi_beg = max(0, a.W - useg0);  // [hi_beg, UW) are right of column W-1
#ifdef FDG_FUSED_NOEDGE
        const bool prod_fix = false;  // diagnostics: timing without the edge-replication path (wrong edges)
#else
        const bool prod_fix = edge_cta;
#endif

        if (tid == 0) {
            for (int s = 0; s < SS; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], NT);  // every A thread arrives
                mbar_init(&ready[s], 32);
            }
            for (int r = 0; r < QR; ++r) {
                mbar_init(&qfull[r], NT);   // A threads publish a q row
                mbar_init(&qempty[r], NT);  // B threads are done reading it
            }
            mbar_fence_init();
        }
        __syncthreads();

        if (tid >= 2 * NT) {  // ------------------------------------ producer warp
            const int lane = tid - 2 * NT;
            const int nst = (steps + R - 1) / R;
            const int uc0 = a.halo_in ? useg0 : max(0, useg0);
            const int uc1 = a.halo_in ? useg0 + G::UW : min(a.Wp4, x0 + G::CW + 2 * G::HX);
            const unsigned ubytes = (unsigned)(uc1 - uc0) * 4u;
            const int udst = uc0 - useg0;
            const int fc0 = max(0, x0 - G::HX), fc1 = min(a.Wp4, x0 + G::CW + G::HX);
            const unsigned fbytes = (unsigned)(fc1 - fc0) * 4u;
            const uint64_t pol_last = HINT ? policy_evict_last() : 0;
            auto issue = [&](int st) {
                const int s = st % SS;
                if (st >= SS) mbar_wait_sleep(&empty[s], ((st / SS) - 1) & 1, 200);
                const int nr = min(R, steps - st * R);
                mbar_arrive_expect_tx(&full[s], ubytes * nr);
                for (int r = 0; r < nr; ++r) {
                    const int j = j0 + st * R + r;
                    if (HINT)
                        bulk_g2s_hint(uring + (size_t)(s * R + r) * G::USEG + udst,
                                      a.u_in + img_u + (long long)clampi(j, a.ylo, a.yhi) * pitch_u + uc0, ubytes,
                                      &full[s], pol_last);
                    else
                        bulk_g2s(uring + (size_t)(s * R + r) * G::USEG + udst,
                                 a.u_in + img_u + (long long)clampi(j, a.ylo, a.yhi) * pitch_u + uc0, ubytes,
                                 &full[s]);
                    if (j - ry >= qr_lo && j - ry <= qr_hi)
                        l2_prefetch(a.f + img + (long long)(j - ry) * pitch + fc0, fbytes);
                }
            };
            if (!prod_fix) {
                if (lane == 0)
                    for (int st = 0; st < nst; ++st) issue(st);
                return;
            }
            const int i0c = lo_end, iWc = a.W - 1 - useg0;
            for (int st = 0; st < nst + LAG; ++st) {
                if (st < nst && lane == 0) issue(st);
                const int sd = st - LAG;
                if (sd >= 0 && sd < nst) {
                    const int s = sd % SS;
                    mbar_wait(&full[s], (sd / SS) & 1);
                    const int nr = min(R, steps - sd * R);
                    for (int r = 0; r < nr; ++r) {
                        float* seg = uring + (size_t)(s * R + r) * G::USEG;
                        const float vl = lo_end > 0 ? seg[i0c] : 0.f;
                        const float vr = hi_beg < G::UW ? seg[iWc] : 0.f;
                        __syncwarp();
                        for (int p = lane; p < lo_end; p += 32) seg[p] = vl;
                        for (int p = hi_beg + lane; p < G::UW; p += 32) seg[p] = vr;
                    }
                    __syncwarp();
                    mbar_arrive(&ready[s]);
                }
            }
            return;
        }

        auto qrow_ptr = [&](int r) { return qbuf + (size_t)(r & (QR - 1)) * G::QSEG; };
        const float scale = a.scale, eps = a.eps;

        if (tid < NT) {  // ---------------------------------- A warps: q rows
            uint64_t* gate = prod_fix ? ready : full;
            const int qc = x0 - G::HX + 4 * tid;  // first q column of this thread
            // q columns outside the image take the edge column's value (q is
            // replicate-continued for the adjoint pass): the thread owning
            // column 0 / W-1 writes those slots of the q row itself, threads
            // wholly outside the image compute throwaway values and store
            // nothing (the edge stays out of the hot path's arithmetic: a
            // per-row component select in the edge warp gated the whole
            // CTA's pipeline -- edge strips ran ~40 % slower)
            const int c0 = x0 - G::HX;  // image column of q-row index 0
            const bool outside = qc + 3 < 0 || qc > a.W - 1;
            // owner of column W-1 when the q row reaches past it (also makes its
            // own components beyond W-1 take that column's value)
            const bool ownR = qc <= a.W - 1 && a.W - 1 <= qc + 3 && (c0 + G::QW > a.W || qc + 3 > a.W - 1);
            const int tR = (a.W - 1 - c0) >> 2;  // A thread owning column W-1 (if in this strip)
            // edge warps: the threads left of column 0 take q(0) from lane 2 (the
            // owner of column 0, x0 == 0), those right of W-1 take q(W-1) from its
            // owner -- one shuffle each when the owner shares their warp (it does
            // unless the image is narrower than ~400 columns: then the owner
            // fills those slots with scalar stores)
            const int wid = tid >> 5;
            const bool wL = c0 < 0 && wid == 0;
            const bool rInStrip = tR >= 0 && tR < NT && c0 + G::QW > a.W;
            const bool wR = rInStrip && wid == NT / 32 - 1 && (tR >> 5) == wid;
            const bool slowR = ownR && !((tR >> 5) == NT / 32 - 1);
            const bool edgeW = wL || wR || (rInStrip && wid == (tR >> 5)) || outside;
            const int chunk = tid;
            const float* fcol = a.f + img + clampi(qc, 0, a.Wp4 - 4);
            // store of this thread's q chunk into q row buffer `qrow`
            auto put_q = [&](float* qrow, float4 q) {
                if (!edgeW) {  // warp-uniform for interior warps
                    *reinterpret_cast<float4*>(qrow + 4 * tid) = q;
                    return;
                }
                float vR = q.w;
                if (ownR) {
                    const int e = a.W - 1 - qc;
                    vR = e == 0 ? q.x : e == 1 ? q.y : e == 2 ? q.z : q.w;
                    if (e < 3) q.w = vR;
                    if (e < 2) q.z = vR;
                    if (e < 1) q.y = vR;
                }
                if (wL) {
                    const float qL = __shfl_sync(0xffffffffu, q.x, 2);
                    if (qc + 3 < 0) q = make_float4(qL, qL, qL, qL);
                }
                if (wR) {
                    const float qR = __shfl_sync(0xffffffffu, vR, tR & 31);
                    if (qc > a.W - 1) q = make_float4(qR, qR, qR, qR);
                }
                if (outside && !wL && !wR) return;  // filled by the owner (slowR)
                *reinterpret_cast<float4*>(qrow + 4 * tid) = q;
                if (slowR)
                    for (int c = qc + 4; c < c0 + G::QW; ++c) qrow[c - c0] = vR;
            };
            VRing<RY ? 2 * RY + 1 : 0> r1;
            r1.my_rt = my;
            int s = 0;
            unsigned phase = 0;
            // f for A(i): row j0 + i - RY (clamped: prefetches past the band are unused)
            auto load_f = [&](int i) { return ldg4(fcol + clampi(j0 + i - ry, qr_lo, qr_hi) * pitch); };
            // step i: u row j0 + i -> H1 -> vertical window -> q row i - 2 RY.
            // Steady (ST): ring full, a q row every step, the q slot was used
            // before, parity ODD known at compile time.
            // q = f / max(v, eps) with v = col / (MX MY): max.NaN keeps the
            // reference's NaN propagation; MUFU reciprocal + one Newton step (packed)
            auto quot4 = [&](const float4 col, const float4 fv) {
                const float4 v = mul4s(col, scale);
                const float4 d = make_float4(fmax_nan(v.x, eps), fmax_nan(v.y, eps), fmax_nan(v.z, eps), fmax_nan(v.w, eps));
                float4 r;
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.x) : "f"(d.x));
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.y) : "f"(d.y));
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.z) : "f"(d.z));
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.w) : "f"(d.w));
                const float2 q0l = mul2(lo2(fv), lo2(r)), q0h = mul2(hi2(fv), hi2(r));
    #ifdef FDG_FUSED_NO_NEWTON
                return cat4(q0l, q0h);
    #endif
                const float2 el = fma2(make_float2(-d.x, -d.y), q0l, lo2(fv));
                const float2 eh = fma2(make_float2(-d.z, -d.w), q0h, hi2(fv));
                return cat4(fma2(el, lo2(r), q0l), fma2(eh, hi2(r), q0h));
            };
            auto step = [&](auto steady, auto odd, const int i, float4& fx) {
                constexpr bool ST = decltype(steady)::value;
                constexpr int ODD = decltype(odd)::value;
                const bool par = ST ? ODD : (i & 1);
                if (!par) mbar_wait(&gate[s], phase);
                float4 h = hsumx4<RX>(uring + (size_t)(s * R + par) * G::USEG, chunk);
                if (par || (!ST && i == steps - 1)) {  // this thread is done with the stage's u rows
                    mbar_arrive(&empty[s]);
                    if (++s == SS) {
                        s = 0;
                        phase ^= 1u;
                    }
                }
                if (ST)
                    r1.push_full(v1, NT, tid, h);
                else
                    r1.push(v1, NT, tid, h);
                const int r = i - 2 * ry;
                if (ST || r >= 0) {
                    // f / max(v, eps): max.NaN keeps the reference's NaN propagation
                    const float4 q = quot4(r1.col, fx);
                    if (ST || r >= QR) mbar_wait(&qempty[r & (QR - 1)], ((r / QR) - 1) & 1);
                    put_q(qrow_ptr(r), q);
                    mbar_arrive(&qfull[r & (QR - 1)]);
                }
                if (!ST) fx = load_f(i + 2);
            };
            float4 F0 = load_f(0), F1 = load_f(1);
            const int i_s = 2 * ry + QR;  // ring full, q rows past the first ring turn
            // steady blocks end 2 rows before the last q row (prefetch stays in range)
            const int nblk = steps - 2 > i_s ? (steps - 2 - i_s) / REFRESH : 0;
            int i = 0;
            for (; i < (nblk ? i_s : steps); i += 2) {
                step(std::false_type(), std::integral_constant<int, 0>(), i, F0);
                if (i + 1 < steps) step(std::false_type(), std::integral_constant<int, 1>(), i + 1, F1);
            }
            if (nblk) {
                const float* fp = fcol + (long long)(j0 + i + 2 - ry) * pitch;  // f row of A(i + 2)
                for (int b = 0; b < nblk; ++b) {
    #pragma unroll 1
                    for (int t = 0; t < REFRESH; t += 2, i += 2) {
    #ifdef FDG_FUSED_STEPWISE
                        step(std::true_type(), std::integral_constant<int, 0>(), i, F0);
                        F0 = ldg4(fp);
                        step(std::true_type(), std::integral_constant<int, 1>(), i + 1, F1);
                        F1 = ldg4(fp + pitch);
    #else
                        // one stage (2 u rows) per iteration: both window sums in
                        // flight, then both q rows handed to the B warps
                        mbar_wait(&gate[s], phase);
                        const float* us = uring + (size_t)(s * R) * G::USEG;
                        float4 h0 = hsumx4<RX>(us, chunk);
                        float4 h1 = hsumx4<RX>(us + G::USEG, chunk);
                        mbar_arrive(&empty[s]);
                        if (++s == SS) {
                            s = 0;
                            phase ^= 1u;
                        }
                        r1.push_full(v1, NT, tid, h0);
                        const float4 qa = quot4(r1.col, F0);
                        r1.push_full(v1, NT, tid, h1);
                        const float4 qb = quot4(r1.col, F1);
                        F0 = ldg4(fp);
                        F1 = ldg4(fp + pitch);
                        const int r = i - 2 * ry;  // even: slots r, r + 1 in the same ring turn
                        mbar_wait(&qempty[r & (QR - 1)], ((r / QR) - 1) & 1);
                        mbar_wait(&qempty[(r + 1) & (QR - 1)], (((r + 1) / QR) - 1) & 1);
                        put_q(qrow_ptr(r), qa);
                        put_q(qrow_ptr(r + 1), qb);
                        mbar_arrive(&qfull[r & (QR - 1)]);
                        mbar_arrive(&qfull[(r + 1) & (QR - 1)]);
    #endif
                        fp += 2 * pitch;
                    }
                    r1.refresh(v1, NT, tid);  // fp32 drift
                }
                r1.n += nblk * REFRESH;
            }
            for (; i < steps; i += 2) {
                step(std::false_type(), std::integral_constant<int, 0>(), i, F0);
                if (i + 1 < steps) step(std::false_type(), std::integral_constant<int, 1>(), i + 1, F1);
            }
            return;
        }

        // ------------------------------------------------ B warps: output rows
        const int tb = tid - NT;
        const int lane = tid & 31;
        const int oc = x0 + 4 * tb;
        // lanes past the strip compute, never store; neither do the lanes of a
        // shifted last strip left of the columns it owns (xown): the neighbour's
        // CTA computes those from another segment start (its running sums round
        // differently), and two writers would make the result depend on timing
        const bool has_out = tb < G::NB && oc < a.W && oc >= xown;
        const bool full_store = oc + 3 < a.W;
        // replicated halo columns of u_out: the owners of columns 0 / W-1
        // replicated halo columns of u_out (halo mode needs W % 4 == 0): B warp 0
        // of the x0 = 0 strip writes columns -16..-1 from lanes 1..4, the warp
        // holding column W-1 writes W..W+15 from the lanes past the image
        // (values shuffled from the edge owners; one store per lane)
        const int bw = tid >> 5;
        const bool bL = a.halo_out && x0 == 0 && bw == (NT >> 5);
        const int tbR = (a.W - 4 - x0) >> 2;  // B thread holding columns W-4..W-1
        const bool bR = a.halo_out && tbR >= 0 && tbR + 4 < NT && ((NT + tbR) >> 5) == bw &&
                        ((NT + tbR + 4) >> 5) == bw;
        const int ocl = min(oc, a.Wp4 - 4);
        const float* ucol = a.u_in + img_u + ocl;
        float* ocol = a.u_out + img_o + oc;
        VRing<RY ? 2 * RY + 1 : 0> r2;
        r2.my_rt = my;
        float4 hlast = make_float4(0.f, 0.f, 0.f, 0.f);
        float maxd = 0.f;
        const uint64_t pol_first = HINT ? policy_evict_first() : 0;
        auto load_u = [&](int o) {  // u of output o (o < 0: ring not yet full, the value is unused --
                                     // clamp the row so a tiny image never reads before its plane)
            const float* p = ucol + clampi(yb0 + o, yb0, yb1 - 1) * pitch_u;
            return HINT ? ldg4_hint(p, pol_first) : ldg4(p);
        };
        auto store = [&](auto fs, const int o, const float4 c, const float4 u) {
            constexpr bool FS = decltype(fs)::value;
            const bool fst = FS || full_store;
            const float4 cu = mul4s(c, scale);
            float4 v4 = cat4(mul2(lo2(cu), lo2(u)), mul2(hi2(cu), hi2(u)));
            if (a.clamp)
                v4 = make_float4(fmax_nan(v4.x, 0.f), fmax_nan(v4.y, 0.f), fmax_nan(v4.z, 0.f), fmax_nan(v4.w, 0.f));
            const float4 dv = sub4(v4, u);
            float val[4] = {v4.x, v4.y, v4.z, v4.w};
            const float dd[4] = {dv.x, dv.y, dv.z, dv.w};
    #pragma unroll
            for (int e = 0; e < 4; ++e)
                if (has_out && (fst || oc + e < a.W)) maxd = fmax_nan(maxd, fabsf(dd[e]));
            float* outp = ocol + (yb0 + o) * pitch_o;
            if (bL | bR) {  // warp-uniform: edge warps only
                if (bL) {
                    const float v0 = __shfl_sync(0xffffffffu, val[0], 0);
                    if (tb >= 1 && tb <= FUSED_HALO_L / 4)
                        *reinterpret_cast<float4*>(outp - oc - 4 * tb) = make_float4(v0, v0, v0, v0);
                }
                if (bR) {
                    const float vR = __shfl_sync(0xffffffffu, val[3], (NT + tbR) & 31);
                    if (oc >= a.W && oc < a.W + FUSED_HALO_R)
                        *reinterpret_cast<float4*>(outp) = make_float4(vR, vR, vR, vR);
                }
            }
            if (!has_out) return;
            if (fst) {
                *reinterpret_cast<float4*>(outp) = make_float4(val[0], val[1], val[2], val[3]);
            } else {
                outp[0] = val[0];
                if (oc + 1 < a.W) outp[1] = val[1];
                if (oc + 2 < a.W) outp[2] = val[2];
            }
        };
        auto take = [&](int r) {  // H2 of q row r (waits for the A warps, frees the slot)
            mbar_wait_sleep(&qfull[r & (QR - 1)], (r / QR) & 1, FDG_QSLEEP);
            const float4 h = hsumx4<RX>(qrow_ptr(r), tb);
            mbar_arrive(&qempty[r & (QR - 1)]);
            return h;
        };
        // pushes: q rows above the image replicate row 0 (extras), rows below
        // the image replicate the last one (trailing); output o = push - 2 RY
        const int extras = qr_lo - (yb0 - ry);
        const int band = yb1 - yb0;
        auto push_out = [&](const float4 h, float4 u) {
            r2.push(v2, NT, tb, h);
            if (r2.n >= my) store(std::false_type(), r2.n - my, r2.col, u);
        };
        // warm-up: q rows 0 .. r_s-1 (ring not yet full)
        const int r_s = (max(1, 2 * ry + 1 - extras) + 1) & ~1;
        const int r_e = nq;  // steady: one push and one output per q row
        const int nblk = r_e > r_s ? (r_e - r_s) / REFRESH : 0;
        int r = 0;
        for (; r < min(r_s, nq); ++r) {
            hlast = take(r);
            if (r == 0)
                for (int p = 0; p < extras; ++p) r2.push(v2, NT, tb, hlast);
            const int o = r2.n + 1 - my;
            push_out(hlast, o >= 0 ? load_u(o) : make_float4(0.f, 0.f, 0.f, 0.f));
        }
        if (nblk) {
            // here r2 is full and output o = r + extras - 2 RY follows every push
            const int o0 = r + extras - 2 * ry;
            float4 U0 = load_u(o0), U1 = load_u(o0 + 1);
            float4 U2 = PD > 2 ? load_u(o0 + 2) : U0, U3 = PD > 2 ? load_u(o0 + 3) : U1;
            auto blocks = [&](auto fs) {
                for (int b = 0; b < nblk; ++b) {
    #pragma unroll 1
                    for (int t = 0; t < REFRESH; t += 2, r += 2) {
                        const int o = r + extras - 2 * ry;
                        const float4 g0 = take(r);
                        const float4 g1 = take(r + 1);
                        r2.push_full(v2, NT, tb, g0);
                        store(fs, o, r2.col, U0);
                        r2.push_full(v2, NT, tb, g1);
                        store(fs, o + 1, r2.col, U1);
                        if (PD > 2) {
                            U0 = U2;
                            U1 = U3;
                            U2 = load_u(o + 4);
                            U3 = load_u(o + 5);
                        } else {
                            U0 = load_u(o + 2);
                            U1 = load_u(o + 3);
                        }
                        hlast = g1;
                    }
                    r2.refresh(v2, NT, tb);  // fp32 drift
                }
            };
            if (x0 + G::CW <= a.W)
                blocks(std::true_type());  // every B lane owns 4 image columns
            else
                blocks(std::false_type());
            r2.n += nblk * REFRESH;
        }
        for (; r < nq; ++r) {
            hlast = take(r);
            push_out(hlast, load_u(r2.n + 1 - my));
        }
        while (r2.n - 2 * ry < band) push_out(hlast, load_u(r2.n + 1 - my));  // below the image

        if (a.maxchange) {
            const bool nan = isnan(maxd);
            const unsigned bits = __reduce_max_sync(0xffffffffu, nan ? 0u : __float_as_uint(maxd));
            const int anynan = __reduce_or_sync(0xffffffffu, (int)nan);
            if (lane == 0) {
                if (bits) atomicMax(a.maxchange, bits);
                if (anynan) atomicOr(a.nanflag, 1);
                stamp_end(a.tend);
            }
        }
    };
    auto reset_barriers = [&]() {  // between segments: every role is done with them
        __syncthreads();
        if (tid == 0) {
            for (int s = 0; s < 3 * SS + 2 * QR; ++s) mbar_inval(full + s);
        }
        __syncthreads();
    };
    // Work of this CTA as a range [p, end) of the strip-major sequence of
    // (strip, row) pairs.  Plain grid: strip blockIdx.x, one row band.
    // Work-balanced (lin_len > 0): rows [b L, (b + 1) L) of the sequence,
    // possibly the tail of one strip and the head of the next, so every
    // resident CTA slot gets the same work (the plain grid leaves slots idle
    // when strips x bands < SMs x occupancy).  One call site of the segment
    // body keeps it inlined.
    int ybase = a.y0, rows = a.y1 - a.y0;
    long long p, end;
    if (a.lin_len > 0) {
        p = (long long)blockIdx.x * a.lin_len;
        end = min((long long)a.strips * rows, p + a.lin_len);
    } else {
        int by = blockIdx.y;
        if (by >= a.nb1) {  // second row range
            by -= a.nb1;
            ybase = a.y2;
            rows = a.y3 - a.y2;
        }
        p = (long long)blockIdx.x * rows + (long long)by * a.band;
        end = min((long long)blockIdx.x * rows + rows, p + a.band);
    }
    for (bool first = true; p < end; first = false) {
        const int sx = (int)(p / rows), r0 = (int)(p - (long long)sx * rows);
        const int r1 = (int)min((long long)rows, r0 + (end - p));
        if (!first) reset_barriers();
        // the last strip is shifted left to end at the image edge (overlapping
        // its neighbour, whose columns it computes but does not store): a
        // strip reaching far past column W-1 makes the producer replicate
        // hundreds of columns per row and straggles the whole launch
        const int xs = a.W > G::CW ? min(sx * G::CW, (a.W - G::CW + 3) & ~3) : 0;
        run_segment(xs, a.W > G::CW ? sx * G::CW : 0, ybase + r0, ybase + r1);
        p += r1 - r0;
    }
#ifdef FDG_FUSED_PROBE
    if (a.probe) {
        __syncthreads();
        if (tid == 0) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            unsigned long long* q = a.probe + 4 * (size_t)blockIdx.x;
            q[0] = *reinterpret_cast<const unsigned long long*>(smem_raw + 504);
            q[1] = globaltimer();
            q[2] = smid;
            q[3] = (unsigned long long)(end - (a.lin_len > 0 ? (long long)blockIdx.x * a.lin_len : 0));
        }
    }
#endif
}

// dst row y = src row y with FUSED_HALO_L / _R replicated columns (dst
// points at column 0 of a haloed plane)
__global__ void k_pad_halo(const float* __restrict__ src, int pitch_src, long long bs_src, float* __restrict__ dst,
                           int pitch_dst, long long bs_dst, int W, int H) {
    const int y = blockIdx.y;
    const long long b = blockIdx.z;
    const float* sr = src + b * bs_src + (long long)y * pitch_src;
    float* dr = dst + b * bs_dst + (long long)y * pitch_dst;
    for (int x = (int)threadIdx.x + blockIdx.x * blockDim.x - FUSED_HALO_L; x < W + FUSED_HALO_R;
         x += blockDim.x * gridDim.x)
        dr[x] = sr[min(max(x, 0), W - 1)];
}

template <int RX, int RY, int NT, int R, int S, int QR, int PD, bool HINT>
size_t smem_bytes(int my) {
    using G = FG<RX, RY, NT>;
    return 512 + sizeof(float) * ((size_t)S * G::USEG + QR * (size_t)G::QSEG) + sizeof(float4) * 2 * (size_t)my * NT;
}

template <int RX, int RY, int NT, int R, int S, int QR, int PD, bool HINT>
cudaError_t launch_t(FusedArgs a, cudaStream_t st) {
    using G = FG<RX, RY, NT>;
    const int ry = RY ? RY : a.ry, my = 2 * ry + 1;  // RY = 0: the radius is a run-time argument
    if (ry < 1 || ry > 8) return cudaErrorInvalidValue;
    a.ry = ry;
    const size_t smem = smem_bytes<RX, RY, NT, R, S, QR, PD, HINT>(my);
    cudaError_t err = smem_attr<k_fused<RX, RY, NT, R, S, QR, PD, HINT>>();
    if (err != cudaSuccess) return err;
    static int occ = 0;
    if (!occ) {  // (run-time radius: 17 rows, the tallest ring, still fits two CTAs per SM)
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused<RX, RY, NT, R, S, QR, PD, HINT>, 2 * NT + 32,
                                                            smem_bytes<RX, RY, NT, R, S, QR, PD, HINT>(RY ? my : 17));
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
    const int rows = a.y1 - a.y0;
    if (rows <= 0) return cudaSuccess;
    // bands no shorter than the box (2 RY halo rows of q, 4 RY of u per band):
    // short launches -- images up to ~2048^2, the pipeline's first and last
    // strips -- need the CTAs more than the halo economy (2048^2 x 15 x 15:
    // 43 -> 31.5 us per iteration against bands >= 4 MY; FDG_FUSED_MINBAND)
    static const int minband = getenv("FDG_FUSED_MINBAND") ? std::max(1, atoi(getenv("FDG_FUSED_MINBAND"))) : 1;
    const long long ctas_y = std::min(per_wave, std::max(1LL, (long long)rows / (minband * my)));
    a.band = (int)((rows + ctas_y - 1) / ctas_y);
    if (const char* e = getenv("FDG_FUSED_BAND")) a.band = std::max(1, atoi(e));
    a.nb1 = (rows + a.band - 1) / a.band;
    const int rows2 = a.y3 - a.y2;
    if (rows2 > 0) {  // both ranges with one band height (boundary bands: one CTA row each)
        a.band = std::max(a.band, rows2);
        a.nb1 = (rows + a.band - 1) / a.band;
    }
    dim3 grid(strips, a.nb1 + (rows2 > 0 ? (rows2 + a.band - 1) / a.band : 0), a.batch);
    // single images: spread (strip, row) work evenly over every resident CTA
    // slot when the plain grid leaves slots idle (config 4: 34 strips x 8
    // bands = 272 of 296 slots)
    static const bool lin_on = !getenv("FDG_FUSED_LIN") || atoi(getenv("FDG_FUSED_LIN")) != 0;
    a.strips = strips;
    const long long slots = (long long)sms * occ;
    const bool want_lin = a.lin_len >= 0;  // caller: -1 = plain grid
    a.lin_len = 0;
    if (lin_on && want_lin && rows2 <= 0 && a.batch == 1 && grid.x * grid.y < slots) {
        const long long total = (long long)strips * rows;
        const long long L = (total + slots - 1) / slots;
        if (L >= 8 * my) {
            a.lin_len = (int)L;
            grid = dim3((unsigned)((total + L - 1) / L), 1, 1);
        }
    }
#ifdef FDG_FUSED_PROBE
    static const char* probe_path = getenv("FDG_FUSED_PROBE");
#else
    static const char* probe_path = nullptr;
#endif
    static unsigned long long* d_probe = nullptr;
    a.probe = nullptr;
    if (probe_path) {
        if (!d_probe) cudaMalloc(&d_probe, 4 * sizeof(unsigned long long) * 65536);
        a.probe = d_probe;
    }
    k_fused<RX, RY, NT, R, S, QR, PD, HINT><<<grid, 2 * NT + 32, smem, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (probe_path && e == cudaSuccess) {  // diagnostics only (eager launches): append the per-CTA record
        const size_t n = (size_t)grid.x * grid.y * grid.z;
        std::vector<unsigned long long> h(4 * n);
        cudaStreamSynchronize(st);
        cudaMemcpy(h.data(), d_probe, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        if (FILE* fp = fopen(probe_path, "a")) {
            for (size_t i = 0; i < n; ++i) fprintf(fp, "%zu %llu %llu %llu %llu\n", i, h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
            fprintf(fp, "--\n");
            fclose(fp);
        }
    }
    return e;
}

// Engine selection: 1 = on where it pays (default: launches of more than ~3
// Mpx, ~12 Mpx for boxes up to 9 px -- below that the two-pass span tiles win,
// use_fused in fdgpu.cu), 2 = whenever the box qualifies (tests), 0 = off;
// FDG_FUSED=0/1/2 or fdg_set_option("fused", v).
std::atomic<int> g_fused{getenv("FDG_FUSED") ? atoi(getenv("FDG_FUSED")) : 1};

}  // namespace

void set_fused_mode(int v) { g_fused.store(v); }
int fused_mode() { return g_fused.load(); }

// centred odd boxes 3 x 3 ... 17 x 17, square or not (config 4 = 15 x 15), and
// centred vertical lines of 3 ... 17 px
bool fused_supported(int mx, int my, int min_dx, int min_dy) {
    return g_fused.load() >= 1 && (mx & 1) && (my & 1) && mx >= 1 && mx <= 17 && my >= 3 && my <= 17 &&
           min_dx == -(mx / 2) && min_dy == -(my / 2);
}

int fused_halo_left() { return FUSED_HALO_L; }
int fused_halo_right() { return FUSED_HALO_R; }
bool fused_halo_ok(int W) { return W >= FG<7, 7, 128>::CW && W % 4 == 0; }

cudaError_t launch_pad_halo(const float* src, int pitch_src, long long bs_src, float* dst, int pitch_dst,
                            long long bs_dst, int W, int H, int batch, cudaStream_t st) {
    const int threads = 256;
    const int bx = std::max(1, std::min(8, (W + FUSED_HALO_L + FUSED_HALO_R + threads - 1) / threads));
    k_pad_halo<<<dim3(bx, H, batch), threads, 0, st>>>(src, pitch_src, bs_src, dst, pitch_dst, bs_dst, W, H);
    return cudaGetLastError();
}

cudaError_t launch_fused(const float* u_in, const float* f, float* u_out, int pitch, int W, int y0, int y1, int ylo,
                         int yhi, int batch, long long bstride, float scale, float eps, int clamp, unsigned* maxchange, int* nanflag,
                         unsigned long long* tend, cudaStream_t st, int halo_in, int halo_out, int pitch_h,
                         long long bstride_h, int y2, int y3, int balanced, int rx, int ry) {
    FusedArgs a;
    a.lin_len = balanced ? 0 : -1;
    a.y2 = y2;
    a.y3 = y3;
    a.nb1 = 1 << 30;
    a.halo_in = halo_in;
    a.halo_out = halo_out;
    a.pitch_u = halo_in ? pitch_h : pitch;  // haloed planes share one pitch
    a.pitch_o = halo_out ? pitch_h : pitch;
    a.bs_u = halo_in ? bstride_h : bstride;
    a.bs_o = halo_out ? bstride_h : bstride;
    a.u_in = u_in;
    a.f = f;
    a.u_out = u_out;
    a.pitch = pitch;
    a.W = W;
    a.Wp4 = (W + 3) & ~3;
    a.y0 = y0;
    a.y1 = y1;
    a.ylo = ylo;
    a.yhi = yhi;
    a.batch = batch;
    a.bstride = bstride;
    a.scale = scale;
    a.eps = eps;
    a.clamp = clamp;
    a.maxchange = maxchange;
    a.nanflag = nanflag;
    a.tend = tend;
    static const int variant = getenv("FDG_FUSED_V") ? atoi(getenv("FDG_FUSED_V")) : 0;
    a.ry = ry;
    if (rx != ry) {  // rectangular boxes: one instantiation per RX, the vertical radius at run time
        switch (rx) {
            case 0: return launch_t<0, 0, 128, 2, 12, 8, 2, true>(a, st);  // vertical lines
            case 1: return launch_t<1, 0, 128, 2, 12, 8, 2, true>(a, st);
            case 2: return launch_t<2, 0, 128, 2, 12, 8, 2, true>(a, st);
            case 3: return launch_t<3, 0, 128, 2, 12, 8, 2, true>(a, st);
            case 4: return launch_t<4, 0, 128, 2, 12, 8, 2, true>(a, st);
            case 5: return launch_t<5, 0, 128, 2, 12, 8, 2, true>(a, st);
            case 6: return launch_t<6, 0, 128, 2, 12, 8, 2, true>(a, st);
            case 7: return launch_t<7, 0, 128, 2, 12, 8, 2, true>(a, st);
            case 8: return launch_t<8, 0, 128, 2, 12, 8, 2, true>(a, st);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (rx) {  // every radius but config 4's: the generic window sums (hsumx4)
        case 1: return launch_t<1, 1, 128, 2, 12, 8, 2, true>(a, st);  // 3 x 3
        case 2: return launch_t<2, 2, 128, 2, 12, 8, 2, true>(a, st);
        case 3: return launch_t<3, 3, 128, 2, 12, 8, 2, true>(a, st);
        case 4: return launch_t<4, 4, 128, 2, 12, 8, 2, true>(a, st);  // 9 x 9
        case 5: return launch_t<5, 5, 128, 2, 12, 8, 2, true>(a, st);
        case 6: return launch_t<6, 6, 128, 2, 12, 8, 2, true>(a, st);
        case 8: return launch_t<8, 8, 128, 2, 12, 8, 2, true>(a, st);  // 17 x 17
        case 7: break;
        default: return cudaErrorInvalidValue;
    }
    switch (variant) {
        case 1: return launch_t<7, 7, 128, 2, 12, 8, 2, false>(a, st);  // no L2 cache hints
        default: return launch_t<7, 7, 128, 2, 12, 8, 2, true>(a, st);
    }
}

}  // namespace fdg
