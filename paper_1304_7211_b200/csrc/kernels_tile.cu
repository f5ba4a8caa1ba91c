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
//          rows x 4 columns x MWP taps; weights are float4 broadcasts.
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
        tile[i] = in[(long long)gy * a.pitch + gx];
    }
    __syncthreads();
    TraceAcc tr;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            const int ly = threadIdx.y + 8 * rr, lx = threadIdx.x + 32 * cc;
            const int y = oy0 + ly, x = ox0 + lx;
            if (y >= a.y1 || x >= a.W) continue;
            const long long idx = img + (long long)y * a.pitch + x;
            if (MASKED && !a.e.active[idx]) continue;
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
    int min_dx, min_dy, mh, ts;  // ts: tile row stride (floats)
    const float* wts;            // mh x MWP, zero padded
    const int* tile_blocks;      // masked: per tile up to 256 block ids
    const int* tile_count;
    int tiles_x;
    Epi e;
};

template <int MWP, int MODE, bool MASKED>
__global__ void __launch_bounds__(256, 2) k_dense(const DenseArgs a) {
    extern __shared__ __align__(16) float sm[];
    float* s_w = sm;                 // mh * MWP
    float* tile = sm + a.mh * MWP;   // (TD + mh - 1) rows x ts
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
    for (int i = tid; i < a.mh * MWP; i += 256) s_w[i] = a.wts[i];
    const int th = TD + a.mh - 1;
    const int tw = TD + MWP - 1;
    for (int i = tid; i < th * tw; i += 256) {
        const int ty = i / tw, tx = i - ty * tw;
        const int gy = clampi(oy0 + a.min_dy + ty, a.ylo, a.yhi);
        const int gx = clampi(ox0 + a.min_dx + tx, 0, a.W - 1);
        tile[ty * a.ts + tx] = in[(long long)gy * a.pitch + gx];
    }
    __syncthreads();
    if (tid >= nblk) return;
    int blk = tid;
    if (MASKED) blk = a.tile_blocks[(long long)tile_id * 256 + tid];
    const int bx = blk & 15, by = blk >> 4;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    constexpr int NV = MWP + 4;  // input values per row segment (float4 chunks)
    for (int ir = 0; ir < a.mh + 3; ++ir) {
        float v[NV];
        const float4* src = reinterpret_cast<const float4*>(tile + (4 * by + ir) * a.ts + 4 * bx);
#pragma unroll
        for (int c = 0; c < NV / 4; ++c) {
            const float4 q = src[c];
            v[4 * c] = q.x;
            v[4 * c + 1] = q.y;
            v[4 * c + 2] = q.z;
            v[4 * c + 3] = q.w;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = ir - i;  // PSF row feeding output row i from input row ir
            if (r < 0 || r >= a.mh) continue;
            const float4* wr = reinterpret_cast<const float4*>(s_w + r * MWP);
            float part[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int kc = 0; kc < MWP / 4; ++kc) {
                const float4 w4 = wr[kc];
                const float wk[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
#pragma unroll
                    for (int j = 0; j < 4; ++j) part[j] = fmaf(wk[e], v[4 * kc + e + j], part[j]);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] += part[j];
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
            epilogue<MODE>(a.e, a.out, idx, acc[i][j], tr);
        }
    }
    if (MODE == EPI_UPDATE || MODE == EPI_MUPDATE) trace_flush(a.e, tr);
}

template <int MWP, int MODE, bool MASKED>
cudaError_t launch_dense_t(const DenseArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
    cudaError_t err = smem_attr<k_dense<MWP, MODE, MASKED>>();
    if (err != cudaSuccess) return err;
    k_dense<MWP, MODE, MASKED><<<grid, 256, smem, st>>>(a);
    return cudaGetLastError();
}

template <int MWP>
cudaError_t dense_mode(const DenseArgs& a, int mode, bool masked, dim3 grid, size_t smem, cudaStream_t st) {
    if (!masked) {
        switch (mode) {
            case EPI_STORE: return launch_dense_t<MWP, EPI_STORE, false>(a, grid, smem, st);
            case EPI_QUOT: return launch_dense_t<MWP, EPI_QUOT, false>(a, grid, smem, st);
            case EPI_UPDATE: return launch_dense_t<MWP, EPI_UPDATE, false>(a, grid, smem, st);
        }
    } else {
        switch (mode) {
            case EPI_STORE: return launch_dense_t<MWP, EPI_STORE, true>(a, grid, smem, st);
            case EPI_MQUOT: return launch_dense_t<MWP, EPI_MQUOT, true>(a, grid, smem, st);
            case EPI_MUPDATE: return launch_dense_t<MWP, EPI_MUPDATE, true>(a, grid, smem, st);
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_taps(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st) {
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
    a.ts = ((TD + mwp - 1 + 4) + 3) & ~3;  // room for the last float4 chunk
    const int th = TD + p.mh - 1 + 3;
    const size_t smem = sizeof(float) * ((size_t)p.mh * mwp + (size_t)th * a.ts);
    dim3 grid((g.W + TD - 1) / TD, (rows + TD - 1) / TD, g.batch);
    a.tiles_x = grid.x;
    const bool masked = d_tile_count != nullptr;
    switch (mwp) {
        case 4: return dense_mode<4>(a, e.mode, masked, grid, smem, st);
        case 8: return dense_mode<8>(a, e.mode, masked, grid, smem, st);
        case 16: return dense_mode<16>(a, e.mode, masked, grid, smem, st);
        case 32: return dense_mode<32>(a, e.mode, masked, grid, smem, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace fdg
