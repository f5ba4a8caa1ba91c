// kernels_band.cu -- the boundary bands of a row strip for the fused
// 15x15-box RL iteration (sharded config 4, shard.cuh).
//
// The fused kernel streams rows through a deep pipeline: a CTA pays ~40 rows
// of latency (u halo + q halo + ring) before its first output, so a 14-row
// band costs as much wall time as ~200 interior rows (25 us measured at
// 16384 columns).  Here a band tile is computed in place, no streaming: one
// 128-thread CTA per 32 output columns x <= 16 output rows loads its u tile
// (+ 2 x 7 rows / columns each side, replicate-clamped into the readable
// rows [ylo, yhi] and columns [0, W)) into shared memory, forms
//   H1 = horizontal 15-sums of u,  q = f / max(vertical 15-sum(H1) / 225, eps)
//   H2 = horizontal 15-sums of q,  u_out = max(vertical 15-sum(H2) / 225 * u, 0)
// with q rows / columns outside the image replicated (the reference pads the
// second convolution's input, convolve.hpp:288-342), and the max|du| / NaN
// trace of the fused epilogue.  Each thread item forms 8 consecutive window
// sums (15 additions, then 7 slides), q rows / columns beyond the image are
// copies of the edge ones.
#include "common.cuh"

namespace fdg {
namespace {

constexpr int BT_W = 32;        // output columns per CTA
constexpr int BT_R = 16;        // output rows per CTA (max)
constexpr int BT_T = 128;       // threads
constexpr int BR_ = 7;          // box radius (15 x 15)
constexpr int BW_ = 2 * BR_ + 1;
constexpr int BT_UC = BT_W + 4 * BR_;  // u columns
constexpr int BT_QC = BT_W + 2 * BR_;  // q columns
constexpr int BT_UR = BT_R + 4 * BR_;  // u rows (max)
constexpr int BT_QR = BT_R + 2 * BR_;  // q rows (max)
constexpr int RUN = 8;                 // window sums per thread item (running sum)

struct BandArgs {
    const float* u_in;
    const float* f;
    float* u_out;
    int pitch_u, pitch_f, pitch_o;
    int W;
    int y0, y1, y2, y3;  // output row ranges
    int nb1;             // CTA rows of the first range
    int ylo, yhi;
    float scale, eps;
    int clamp;
    int halo_out, halo_l, halo_r;
    unsigned* maxchange;
    int* nanflag;
    unsigned long long* tend;
};

// RUN consecutive 15-wide window sums of src[0 .. RUN + 13] (stride st):
// the first by additions, then slid (7 steps: the fp32 drift stays ~1e-7)
__device__ __forceinline__ void window_run(const float* src, int st, float* out, int n) {
    float v[RUN + BW_ - 1];
#pragma unroll
    for (int k = 0; k < RUN + BW_ - 1; ++k) v[k] = src[k * st];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < BW_; ++k) s += v[k];
    out[0] = s;
#pragma unroll
    for (int k = 1; k < RUN; ++k) {
        s += v[k + BW_ - 1] - v[k - 1];
        if (k < n) out[k] = s;
    }
}

__global__ void __launch_bounds__(BT_T) k_band(const BandArgs a) {
    // (+1 / + RUN rows: window_run reads RUN + 14 values even for a short tail)
    __shared__ float su[BT_UR + 1][BT_UC + 1];
    __shared__ float sh[BT_UR + RUN][BT_QC + 1];  // H1, then H2 (first BT_QR rows, BT_W columns)
    __shared__ float sq[BT_QR][BT_QC + 1];        // f, then q
    const int tid = threadIdx.x;
    int by = blockIdx.y, ya = a.y0, yb = a.y1;
    if (by >= a.nb1) {
        by -= a.nb1;
        ya = a.y2;
        yb = a.y3;
    }
    const int yb0 = ya + by * BT_R;
    const int yb1 = min(yb, yb0 + BT_R);
    if (yb0 >= yb1) return;
    const int nr = yb1 - yb0;
    const int ur = nr + 4 * BR_, qr = nr + 2 * BR_;
    const int x0 = blockIdx.x * BT_W;
    const int wm1 = a.W - 1;
    // u tile: image rows clamp(yb0 - 14 + t), columns clamp(x0 - 14 + c);
    // f at the q positions (rows clamp(yb0 - 7 + r), columns clamp(x0 - 7 + j)).
    // Asynchronous 4-byte copies: every load of the CTA in flight at once.
    // (one row per warp at a time: the row pointer and clamp once per row)
    const int lane = tid & 31, wrp = tid >> 5;
    for (int t = wrp; t < ur; t += BT_T / 32) {
        const float* rp = a.u_in + (long long)clampi(yb0 - 2 * BR_ + t, a.ylo, a.yhi) * a.pitch_u;
        for (int c = lane; c < BT_UC; c += 32) {
            const float* src = rp + clampi(x0 - 2 * BR_ + c, 0, wm1);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(&su[t][c])), "l"(src) : "memory");
        }
    }
    for (int r = wrp; r < qr; r += BT_T / 32) {
        const float* rp = a.f + (long long)clampi(yb0 - BR_ + r, a.ylo, a.yhi) * a.pitch_f;
        for (int j = lane; j < BT_QC; j += 32) {
            const float* src = rp + clampi(x0 - BR_ + j, 0, wm1);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(&sq[r][j])), "l"(src) : "memory");
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    // H1[t][j] = sum of u tile columns j .. j + 14 (q column j <-> image column
    // x0 - 7 + j; columns beyond the image are fixed up below)
    constexpr int JC = (BT_QC + RUN - 1) / RUN;
    for (int i = tid; i < ur * JC; i += BT_T) {
        const int t = i / JC, j0 = (i - t * JC) * RUN;
        float o[RUN];
        window_run(&su[t][j0], 1, o, BT_QC - j0);
#pragma unroll
        for (int k = 0; k < RUN; ++k)
            if (j0 + k < BT_QC) sh[t][j0 + k] = o[k];
    }
    __syncthreads();
    // q[r][j] = f / max(sum of H1 rows r .. r + 14 / 225, eps)  (q row r <-> image row yb0 - 7 + r)
    constexpr int RC = (BT_QR + RUN - 1) / RUN;
    for (int i = tid; i < RC * BT_QC; i += BT_T) {
        const int r0 = (i / BT_QC) * RUN, j = i - (i / BT_QC) * BT_QC;
        if (r0 >= qr) continue;
        float o[RUN];
        window_run(&sh[r0][j], BT_QC + 1, o, qr - r0);
#pragma unroll
        for (int k = 0; k < RUN; ++k) {
            if (r0 + k >= qr) break;
            const float v = o[k] * a.scale;
            sq[r0 + k][j] = div_fast(sq[r0 + k][j], v < a.eps ? a.eps : v);  // f there -> q
        }
    }
    __syncthreads();
    // q rows / columns beyond the readable rows / the image replicate the edge
    // (the second convolution pads its input, convolve.hpp:288-342)
    if (yb0 - BR_ < a.ylo || yb1 - 1 + BR_ > a.yhi || x0 - BR_ < 0 || x0 + BT_QC - 1 - BR_ > wm1) {  // edge tiles only
        const int rlo = a.ylo - (yb0 - BR_), rhi = a.yhi - (yb0 - BR_);
        const int clo = -(x0 - BR_), chi = wm1 - (x0 - BR_);
        for (int i = tid; i < qr * BT_QC; i += BT_T) {
            const int r = i / BT_QC, j = i - r * BT_QC;
            const int rs = clampi(r, rlo, rhi), js = clampi(j, clo, chi);
            if (rs != r || js != j) sh[r][j] = sq[rs][js];
        }
        __syncthreads();
        for (int i = tid; i < qr * BT_QC; i += BT_T) {
            const int r = i / BT_QC, j = i - r * BT_QC;
            if (clampi(r, rlo, rhi) != r || clampi(j, clo, chi) != j) sq[r][j] = sh[r][j];
        }
        __syncthreads();
    }
    // H2[r][c] = sum of q columns c .. c + 14 (output column x0 + c)
    constexpr int CC = BT_W / RUN;
    for (int i = tid; i < qr * CC; i += BT_T) {
        const int r = i / CC, c0 = (i - r * CC) * RUN;
        float o[RUN];
        window_run(&sq[r][c0], 1, o, RUN);
#pragma unroll
        for (int k = 0; k < RUN; ++k) sh[r][c0 + k] = o[k];
    }
    __syncthreads();
    float maxd = 0.f;
    int nan = 0;
    const int OC = (nr + RUN - 1) / RUN;
    for (int i = tid; i < OC * BT_W; i += BT_T) {
        const int o0 = (i / BT_W) * RUN, c = i - (i / BT_W) * BT_W;
        const int x = x0 + c;
        if (x > wm1) continue;
        float o[RUN];
        window_run(&sh[o0][c], BT_QC + 1, o, nr - o0);
        float* orow0 = a.u_out + (long long)(yb0 + o0) * a.pitch_o;
#pragma unroll
        for (int k = 0; k < RUN; ++k) {
            if (o0 + k >= nr) break;
            const float u = su[o0 + k + 2 * BR_][c + 2 * BR_];
            float value = o[k] * a.scale * u;
            if (a.clamp && value < 0.f) value = 0.f;
            maxd = fmaxf(maxd, fabsf(value - u));
            nan |= isnan(value);
            float* orow = orow0 + (long long)k * a.pitch_o;
            orow[x] = value;
            if (a.halo_out) {  // replicated edge columns of a haloed plane
                if (x == 0)
                    for (int h = 1; h <= a.halo_l; ++h) orow[-h] = value;
                if (x == wm1)
                    for (int h = 1; h <= a.halo_r; ++h) orow[wm1 + h] = value;
            }
        }
    }
    if (a.maxchange) {
        const unsigned bits = __reduce_max_sync(0xffffffffu, __float_as_uint(maxd));
        const int anynan = __reduce_or_sync(0xffffffffu, nan);
        if ((tid & 31) == 0) {
            if (bits) atomicMax(a.maxchange, bits);
            if (anynan) atomicOr(a.nanflag, 1);
            stamp_end(a.tend);
        }
    }
}

}  // namespace

cudaError_t launch_band(const float* u_in, int pitch_u, const float* f, int pitch_f, float* u_out, int pitch_o,
                        int W, int y0, int y1, int y2, int y3, int ylo, int yhi, float scale, float eps, int clamp,
                        int halo_out, int halo_l, int halo_r, unsigned* maxchange, int* nanflag,
                        unsigned long long* tend, cudaStream_t st) {
    BandArgs a;
    a.u_in = u_in;
    a.f = f;
    a.u_out = u_out;
    a.pitch_u = pitch_u;
    a.pitch_f = pitch_f;
    a.pitch_o = pitch_o;
    a.W = W;
    a.y0 = y0;
    a.y1 = y1;
    a.y2 = y2;
    a.y3 = y3;
    a.nb1 = (std::max(0, y1 - y0) + BT_R - 1) / BT_R;
    a.ylo = ylo;
    a.yhi = yhi;
    a.scale = scale;
    a.eps = eps;
    a.clamp = clamp;
    a.halo_out = halo_out;
    a.halo_l = halo_l;
    a.halo_r = halo_r;
    a.maxchange = maxchange;
    a.nanflag = nanflag;
    a.tend = tend;
    const int nb2 = (std::max(0, y3 - y2) + BT_R - 1) / BT_R;
    if (a.nb1 + nb2 == 0) return cudaSuccess;
    k_band<<<dim3((W + BT_W - 1) / BT_W, a.nb1 + nb2), BT_T, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace fdg
