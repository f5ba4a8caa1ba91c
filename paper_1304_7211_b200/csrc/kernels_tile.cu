// kernels_tile.cu -- 2-D tiled engines.
//
// "taps":  any PSF as a tap list grouped by PSF row (List, GenericBox
//          fallback, Naive with wide grids, Fourier with wrap-around).  The
//          input tile + halo is staged in shared memory with replicate
//          (or cyclic) clamping; every output accumulates one partial per
//          PSF row and adds the partials in row order (per-row partials keep
//          fp32 within 1e-4 of the fp64 reference: SURVEY 8a-11).
// "dense": DensePsf up to 32 columns wide (Naive; config 3's 31x31
//          Gaussian).  FP32-FMA-bound (no tensor cores: 961 taps x 2 convs
//          = 3844 FLOP/px.it).  64x64 output tile, each thread a 4x4 register
//          block: one shared-memory input row (float4 loads) feeds 4 output
//          rows x 4 columns x MWP taps as packed FFMA2, two output columns
//          per instruction (the tile is also stored shifted by one column, so
//          every adjacent input pair is an aligned register pair); the
//          weights come from the kernel parameter space as uniform operands.
//          Same per-lane fmaf order as scalar FFMA: results are unchanged.
//          The masked (thinned) variant consumes the per-tile compacted list
//          of active 4x4 blocks built by k_tile_compact (kernels_mask.cu).
#include "common.cuh"

namespace fdg {
namespace {

// ------------------------------------------------------------------- taps
constexpr int TT_W = 64, TT_H = 16;  // output tile
struct TapsArgs {
    const float* in;
    float* out;
    int pitch, W;
    int y0, y1, ylo, yhi;
    long long bstride;
    int wrap;
    int min_dx, min_dy, nrows, ntaps, tw, th;
    int uniform;
    float scale;
    const int* row_start;
    const int* dx;
    const float* w;
    Epi e;
};

template <int MODE, bool MASKED>
__global__ void __launch_bounds__(256) k_taps(const TapsArgs a) {
    extern __shared__ __align__(16) float sm[];
    int* s_rs = reinterpret_cast<int*>(sm);
    int* s_dx = s_rs + a.nrows + 1;
    float* s_w = reinterpret_cast<float*>(s_dx + a.ntaps);
    float* tile = s_w + a.ntaps;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    for (int i = tid; i <= a.nrows; i += 256) s_rs[i] = a.row_start[i];
    for (int i = tid; i < a.ntaps; i += 256) {
        s_dx[i] = a.dx[i] - a.min_dx;
        s_w[i] = a.w[i];
    }
    const int ox0 = blockIdx.x * TT_W;
    const int oy0 = a.y0 + blockIdx.y * TT_H;
    const long long img = (long long)blockIdx.z * a.bstride;
    const float* in = a.in + img;
    const int hgt = a.yhi - a.ylo + 1;
    for (int i = tid; i < a.tw * a.th; i += 256) {
        const int ty = i / a.tw, tx = i - ty * a.tw;
        int gy = oy0 + a.min_dy + ty, gx = ox0 + a.min_dx + tx;
        if (a.wrap) {
            gy = a.ylo + wrapi(gy - a.ylo, hgt);
            gx = wrapi(gx, a.W);
        } else {
            gy = clampi(gy, a.ylo, a.yhi);
            gx = clampi(gx, 0, a.W - 1);
        }
        // 4-byte cp.async: every load of the thread in flight at once (the
        // dependent load -> store loop was ~5 serial global round trips)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(tile + i)),
                     "l"(in + (long long)gy * a.pitch + gx)
                     : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    // masked (thinned) evaluation: compact the tile's active pixels into a
    // shared list first, so the work scales with active pixels, not with
    // the tile (convolve.hpp:473-510 walks the active runs)
    __shared__ int s_n;
    __shared__ short s_list[TT_W * TT_H];
    if (MASKED) {
        if (tid == 0) s_n = 0;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int ly = threadIdx.y + 8 * (k >> 1), lx = threadIdx.x + 32 * (k & 1);
            const int y = oy0 + ly, x = ox0 + lx;
            if (y < a.y1 && x < a.W && a.e.active[img + (long long)y * a.pitch + x])
                s_list[atomicAdd(&s_n, 1)] = (short)(ly * TT_W + lx);
        }
    }
    __syncthreads();
    TraceAcc tr;
    const int nwork = MASKED ? s_n : 4 * 256;
    for (int w = tid; w < nwork; w += 256) {
        {
            int ly, lx;
            if (MASKED) {
                ly = s_list[w] / TT_W;
                lx = s_list[w] - ly * TT_W;
            } else {  // the fixed 2 x 2 assignment: rows ty, ty + 8, columns tx, tx + 32
                const int k = w >> 8;
                ly = threadIdx.y + 8 * (k >> 1);
                lx = threadIdx.x + 32 * (k & 1);
            }
            const int y = oy0 + ly, x = ox0 + lx;
            if (y >= a.y1 || x >= a.W) continue;
            const long long idx = img + (long long)y * a.pitch + x;
            float acc = 0.f;
            for (int r = 0; r < a.nrows; ++r) {
                const float* trow = tile + (ly + r) * a.tw + lx;
                float part = 0.f;
                const int k1 = s_rs[r + 1];
                if (a.uniform) {
                    for (int k = s_rs[r]; k < k1; ++k) part += trow[s_dx[k]];
                } else {
                    for (int k = s_rs[r]; k < k1; ++k) part = fmaf(s_w[k], trow[s_dx[k]], part);
                }
                acc += part;
            }
            if (a.uniform) acc *= a.scale;
            epilogue<MODE>(a.e, a.out, idx, acc, tr);
        }
    }
    if (MODE == EPI_UPDATE || MODE == EPI_MUPDATE) trace_flush(a.e, tr);
}

template <int MODE, bool MASKED>
cudaError_t launch_taps_t(const TapsArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
    cudaError_t err = smem_attr<k_taps<MODE, MASKED>>();
    if (err != cudaSuccess) return err;
    k_taps<MODE, MASKED><<<grid, dim3(32, 8), smem, st>>>(a);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ dense
constexpr int TD = 64;  // output tile edge
struct DenseArgs {
    const float* in;
    float* out;
    int pitch, W;
    int y0, y1, ylo, yhi;
    long long bstride;
    int min_dx, min_dy, mh, ts, th;  // ts: tile row stride (floats), th: tile rows
    const float* wts;            // mh x MWP, zero padded (device copy)
    const int* tile_blocks;      // masked: per tile up to 256 block ids
    const int* tile_count;
    int tiles_x;
    Epi e;
};
// The dense weights travel in the kernel parameter space (constant bank 0,
// 32 KB limit): the inner loop reads them with a warp-uniform index, which
// compiles to uniform constant loads (LDCU) feeding FFMA directly -- no
// shared-memory traffic for the 961 weights.
struct DenseW {
    float w[64 * 32];  // mh x MWP row-major, zero padded (8 KB of the 32 KB parameter space)
};

template <int MWP, int MW, int MODE, bool MASKED>
__global__ void __launch_bounds__(256, 2) k_dense(const DenseArgs a, const __grid_constant__ DenseW wp) {
    extern __shared__ __align__(16) float sm[];
    float* tile = sm;                  // (TD + mh - 1) rows x ts
    float* tile_s = sm + a.th * a.ts;  // the same rows shifted left by one column
    const int tid = threadIdx.x;
    const int tile_id = blockIdx.y * gridDim.x + blockIdx.x;
    int nblk = 256;
    if (MASKED) {
        nblk = a.tile_count[tile_id];
        if (nblk == 0) return;
    }
    const int ox0 = blockIdx.x * TD;
    const int oy0 = a.y0 + blockIdx.y * TD;
    const long long img = (long long)blockIdx.z * a.bstride;
    const float* in = a.in + img;
    const int th = TD + a.mh - 1;
    const int tw = TD + MWP - 1;
    // tile column t = image column ox0 + min_dx + t.  Loads go by aligned
    // float4 chunks of image columns c0 + 4q (c0 = the 16-byte boundary at or
    // below column ox0 + min_dx), clamped per element only at the image edge.
    const int cbase = ox0 + a.min_dx;
    const int c0 = cbase & ~3;  // <= cbase (also for negative cbase)
    const int sh = cbase - c0;  // tile column of chunk element k: 4 q + k - sh
    const int nq = (tw + sh + 3) / 4;
#pragma unroll 4
    for (int i = tid; i < th * nq; i += 256) {  // unrolled: 4 loads in flight per thread
        const int ty = i / nq, q = i - ty * nq;
        const int gy = clampi(oy0 + a.min_dy + ty, a.ylo, a.yhi);
        const float* rp = in + (long long)gy * a.pitch;
        const int c = c0 + 4 * q;
        float v[4];
        if (c >= 0 && c + 3 < a.W) {
            const float4 f4 = __ldg(reinterpret_cast<const float4*>(rp + c));
            v[0] = f4.x;
            v[1] = f4.y;
            v[2] = f4.z;
            v[3] = f4.w;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = __ldg(rp + clampi(c + k, 0, a.W - 1));
        }
        float* trow = tile + ty * a.ts;
        float* srow = tile_s + ty * a.ts;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int tx = 4 * q + k - sh;
            if (tx >= 0 && tx < tw) trow[tx] = v[k];
            if (tx >= 1 && tx < tw) srow[tx - 1] = v[k];
        }
    }
    __syncthreads();
    if (tid >= nblk) return;
    int blk = tid;
    if (MASKED) blk = a.tile_blocks[(long long)tile_id * 256 + tid];
    const int bx = blk & 15, by = blk >> 4;
    // packed accumulators: acc[i][0] = outputs (i, 0..1), acc[i][1] = (i, 2..3)
    float2 acc[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = make_float2(0.f, 0.f);
    constexpr int NV = MWP + 4;  // input values per row segment (float4 chunks)
    constexpr int NP = NV / 2;
    for (int ir = 0; ir < a.mh + 3; ++ir) {
        // vA[k] = (v[2k], v[2k+1]) and vB[k] = (v[2k+1], v[2k+2]): every
        // adjacent pair of the window is an aligned register pair, so each
        // weight (a scalar broadcast operand) feeds two outputs per FFMA2
        float2 vA[NP], vB[NP];
        const float4* src = reinterpret_cast<const float4*>(tile + (4 * by + ir) * a.ts + 4 * bx);
        const float4* srs = reinterpret_cast<const float4*>(tile_s + (4 * by + ir) * a.ts + 4 * bx);
#pragma unroll
        for (int c = 0; c < NV / 4; ++c) {
            const float4 q = src[c], qs = srs[c];
            vA[2 * c] = make_float2(q.x, q.y);
            vA[2 * c + 1] = make_float2(q.z, q.w);
            vB[2 * c] = make_float2(qs.x, qs.y);
            vB[2 * c + 1] = make_float2(qs.z, qs.w);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = ir - i;  // PSF row feeding output row i from input row ir
            if (r < 0 || r >= a.mh) continue;
            const float4* wr = reinterpret_cast<const float4*>(wp.w + r * MWP);
            float2 p01 = make_float2(0.f, 0.f), p23 = make_float2(0.f, 0.f);
#pragma unroll
            for (int kc = 0; kc < MWP / 4; ++kc) {
                const float4 w4 = wr[kc];
                const float wk[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int m = 4 * kc + e;  // window offset of output column 0
                    if (m >= MW) continue;     // zero padding of the grid (MW < MWP): no FMA
                    const float2 ww = make_float2(wk[e], wk[e]);
                    if ((m & 1) == 0) {
                        p01 = __ffma2_rn(ww, vA[m / 2], p01);
                        p23 = __ffma2_rn(ww, vA[m / 2 + 1], p23);
                    } else {
                        p01 = __ffma2_rn(ww, vB[m / 2], p01);
                        p23 = __ffma2_rn(ww, vB[m / 2 + 1], p23);
                    }
                }
            }
            acc[i][0] = __fadd2_rn(acc[i][0], p01);
            acc[i][1] = __fadd2_rn(acc[i][1], p23);
        }
    }
    TraceAcc tr;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int y = oy0 + 4 * by + i;
        if (y >= a.y1) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int x = ox0 + 4 * bx + j;
            if (x >= a.W) continue;
            const long long idx = img + (long long)y * a.pitch + x;
            if (MASKED && !a.e.active[idx]) continue;
            const float2 pr = acc[i][j >> 1];
            epilogue<MODE>(a.e, a.out, idx, (j & 1) ? pr.y : pr.x, tr);
        }
    }
    if (MODE == EPI_UPDATE || MODE == EPI_MUPDATE) trace_flush(a.e, tr);
}

template <int MWP, int MW, int MODE, bool MASKED>
cudaError_t launch_dense_t(const DenseArgs& a, const DenseW& w, dim3 grid, size_t smem, cudaStream_t st) {
    cudaError_t err = smem_attr<k_dense<MWP, MW, MODE, MASKED>>();
    if (err != cudaSuccess) return err;
    k_dense<MWP, MW, MODE, MASKED><<<grid, 256, smem, st>>>(a, w);
    return cudaGetLastError();
}

template <int MWP, int MW = MWP>
cudaError_t dense_mode(const DenseArgs& a, const DenseW& w, int mode, bool masked, dim3 grid, size_t smem,
                       cudaStream_t st) {
    if (!masked) {
        switch (mode) {
            case EPI_STORE: return launch_dense_t<MWP, MW, EPI_STORE, false>(a, w, grid, smem, st);
            case EPI_QUOT: return launch_dense_t<MWP, MW, EPI_QUOT, false>(a, w, grid, smem, st);
            case EPI_UPDATE: return launch_dense_t<MWP, MW, EPI_UPDATE, false>(a, w, grid, smem, st);
        }
    } else {
        switch (mode) {
            case EPI_STORE: return launch_dense_t<MWP, MW, EPI_STORE, true>(a, w, grid, smem, st);
            case EPI_MQUOT: return launch_dense_t<MWP, MW, EPI_MQUOT, true>(a, w, grid, smem, st);
            case EPI_MUPDATE: return launch_dense_t<MWP, MW, EPI_MUPDATE, true>(a, w, grid, smem, st);
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_taps(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st) {
    // unmasked passes: the tile kernel compiled for this tap list (NVRTC)
    if (spans_jit_mode() && taps_jit_ready(p)) {
        const cudaError_t r = launch_taps_jit(p, g, e, st);
        if (r != cudaErrorNotSupported) return r;  // else the JIT build failed: the generic tap kernel
    }
    TapsArgs a;
    a.in = g.in;
    a.out = g.out;
    a.pitch = g.pitch;
    a.W = g.W;
    a.y0 = g.y0;
    a.y1 = g.y1;
    a.ylo = g.ylo;
    a.yhi = g.yhi;
    a.bstride = g.bstride;
    a.wrap = g.wrap;
    a.min_dx = p.min_dx;
    a.min_dy = p.min_dy;
    a.nrows = p.nrows;
    a.ntaps = p.ntaps;
    a.tw = TT_W + (p.max_dx - p.min_dx);
    a.th = TT_H + (p.max_dy - p.min_dy);
    a.uniform = p.uniform;
    a.scale = p.scale;
    a.row_start = p.d_row_start;
    a.dx = p.d_dx;
    a.w = p.d_w;
    a.e = e;
    const int rows = g.y1 - g.y0;
    if (rows <= 0) return cudaSuccess;
    const size_t smem = sizeof(int) * (p.nrows + 1 + p.ntaps) + sizeof(float) * (p.ntaps + (size_t)a.tw * a.th);
    if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
    dim3 grid((g.W + TT_W - 1) / TT_W, (rows + TT_H - 1) / TT_H, g.batch);
    const bool masked = e.active != nullptr;
    if (!masked) {
        switch (e.mode) {
            case EPI_STORE: return launch_taps_t<EPI_STORE, false>(a, grid, smem, st);
            case EPI_QUOT: return launch_taps_t<EPI_QUOT, false>(a, grid, smem, st);
            case EPI_UPDATE: return launch_taps_t<EPI_UPDATE, false>(a, grid, smem, st);
        }
    } else {
        switch (e.mode) {
            case EPI_STORE: return launch_taps_t<EPI_STORE, true>(a, grid, smem, st);
            case EPI_MQUOT: return launch_taps_t<EPI_MQUOT, true>(a, grid, smem, st);
            case EPI_MUPDATE: return launch_taps_t<EPI_MUPDATE, true>(a, grid, smem, st);
        }
    }
    return cudaErrorInvalidValue;
}

bool dense_supported(const DevPsf& p) { return p.mw >= 1 && p.mw <= 32 && p.mh >= 1 && p.mh <= 64; }

DenseTiling dense_tiling(int W, int H) { return {(W + TD - 1) / TD, (H + TD - 1) / TD}; }

cudaError_t launch_dense(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st,
                         const int* d_tile_blocks, const int* d_tile_count) {
    DenseArgs a;
    a.in = g.in;
    a.out = g.out;
    a.pitch = g.pitch;
    a.W = g.W;
    a.y0 = g.y0;
    a.y1 = g.y1;
    a.ylo = g.ylo;
    a.yhi = g.yhi;
    a.bstride = g.bstride;
    a.min_dx = p.min_dx;
    a.min_dy = p.min_dy;
    a.mh = p.mh;
    a.wts = p.d_dense;
    a.tile_blocks = d_tile_blocks;
    a.tile_count = d_tile_count;
    a.e = e;
    const int rows = g.y1 - g.y0;
    if (rows <= 0) return cudaSuccess;
    const int mwp = p.mwp;
    a.ts = TD + mwp;       // the last thread's window ends at column TD - 4 + MWP + 3
    a.th = TD + p.mh - 1;  // rows 4 by + ir, ir < mh + 3
    const size_t smem = sizeof(float) * 2 * ((size_t)a.th * a.ts);
    if ((size_t)p.mh * mwp > 64 * 32 || p.h_dense.size() < (size_t)p.mh * mwp) return cudaErrorInvalidValue;
    DenseW w;
    for (int i = 0; i < 64 * 32; ++i) w.w[i] = i < p.mh * mwp ? p.h_dense[i] : 0.f;
    dim3 grid((g.W + TD - 1) / TD, (rows + TD - 1) / TD, g.batch);
    a.tiles_x = grid.x;
    const bool masked = d_tile_count != nullptr;
    switch (mwp) {
        case 4: return dense_mode<4>(a, w, e.mode, masked, grid, smem, st);
        case 8: return dense_mode<8>(a, w, e.mode, masked, grid, smem, st);
        case 16: return dense_mode<16>(a, w, e.mode, masked, grid, smem, st);
        case 32:  // 31-wide grids (config 3) skip the padded column's FMAs
            return p.mw == 31 ? dense_mode<32, 31>(a, w, e.mode, masked, grid, smem, st)
                              : dense_mode<32>(a, w, e.mode, masked, grid, smem, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace fdg
