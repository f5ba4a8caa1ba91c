// kernels_mask.cu -- stream compaction for selective (thinned) RL.
//
// k_tile_compact: one CTA per 64x64 dense tile; each thread owns a 4x4 pixel
//   block, flags it when any pixel is active, and the CTA compacts the
//   flagged block ids (warp ballots + popc prefix sums) in a bank-friendly
//   round-robin order over the block columns.  The thinned dense kernel consumes these per-tile lists
//   (tiles with no active block exit immediately).  The same pass counts the
//   inactive pixels of the iteration for RlTrace.inactiveFraction.
// k_row_count / k_row_emit: the reference's row-major run walk
//   (convolve.hpp:450-465) on the device, one thread per row, emitting the
//   ordered active index list and (y, x0, len) runs for bit-exact checks.
#include "common.cuh"

namespace fdg {
namespace {

constexpr int TD = 64;

__global__ void __launch_bounds__(256) k_tile_compact(const uint8_t* act, int W, int H, int pitch,
                                                      int* tile_blocks, int* tile_count,
                                                      unsigned long long* inactive) {
    __shared__ int warp_bn[8][8];  // per warp: active blocks per bucket
    __shared__ unsigned long long warp_inact[8];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int tile = blockIdx.y * gridDim.x + blockIdx.x;
    const int bx = t & 15, by = t >> 4;
    const int x0 = blockIdx.x * TD + 4 * bx, y0 = blockIdx.y * TD + 4 * by;
    int any = 0, nin = 0;
    for (int i = 0; i < 4; ++i) {
        const int y = y0 + i;
        if (y >= H) break;
        for (int j = 0; j < 4; ++j) {
            const int x = x0 + j;
            if (x >= W) break;
            const int a = act[(long long)y * pitch + x];
            any |= a;
            nin += !a;
        }
    }
    const unsigned ball = __ballot_sync(0xffffffffu, any);
    const int cnt_inact = __reduce_add_sync(0xffffffffu, nin);
    // List order: the dense kernel gives list entry i to thread i, and its
    // float4 tile loads are bank-conflict free only when the 8 lanes of a
    // quarter warp read 8 different 16-byte columns -- block column bx mod 8
    // (tile rows are a multiple of 32 floats apart).  A plain ascending list
    // puts arbitrary bx side by side (measured: the masked pass then runs
    // shared-memory bound and skipping blocks buys nothing), so the blocks are
    // dealt round-robin from 8 buckets j = bx mod 8: entry (r, j) = the r-th
    // active block of bucket j, entries in (r, j) order with the absent ones
    // squeezed out.  Any 8 consecutive entries then hold 8 different buckets
    // except where a bucket ran out.
    const int j = t & 7;  // = bx & 7
    const unsigned bmask = 0x01010101u << j;
    if (lane < 8) warp_bn[wid][lane] = __popc(ball & (0x01010101u << lane));
    if (lane == 0) warp_inact[wid] = (unsigned long long)cnt_inact;
    __syncthreads();
    int r = __popc(ball & bmask & ((1u << lane) - 1u));  // rank inside the bucket
    for (int w = 0; w < wid; ++w) r += warp_bn[w][j];
    int total = 0, before = 0;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
        int n = 0;
        for (int w = 0; w < 8; ++w) n += warp_bn[w][jj];
        total += n;
        before += min(n, r) + (jj < j && n > r);
    }
    if (any) tile_blocks[(long long)tile * 256 + before] = t;
    if (t == 0) {
        unsigned long long ni = 0;
        for (int w = 0; w < 8; ++w) ni += warp_inact[w];
        tile_count[tile] = total;
        if (inactive && ni) atomicAdd(inactive, ni);
    }
}

__global__ void k_fill_u8(uint8_t* p, uint8_t v, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void k_count_zero(const uint8_t* p, size_t n, unsigned long long* out) {
    unsigned long long c = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        c += p[i] == 0;
    c = __reduce_add_sync(0xffffffffu, (unsigned)c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// per row: [0] = number of active runs, [1] = number of active pixels
__global__ void k_row_count(const uint8_t* act, int W, int H, int* counts) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= H) return;
    const uint8_t* r = act + (long long)y * W;
    int runs = 0, n = 0, prev = 0;
    for (int x = 0; x < W; ++x) {
        const int a = r[x] != 0;
        runs += a && !prev;
        n += a;
        prev = a;
    }
    counts[2 * y] = runs;
    counts[2 * y + 1] = n;
}

__global__ void k_row_emit(const uint8_t* act, int W, int H, const long long* run_off, const long long* act_off,
                           int32_t* runs, int64_t* idx) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= H) return;
    const uint8_t* r = act + (long long)y * W;
    long long ro = run_off[y], ao = act_off[y];
    int x = 0;
    while (x < W) {  // the run walk of convolve.hpp:450-465
        int end = x + 1;
        if (r[x]) {
            while (end < W && r[end]) ++end;
            if (runs) {
                runs[3 * ro] = y;
                runs[3 * ro + 1] = x;
                runs[3 * ro + 2] = end - x;
            }
            ++ro;
            if (idx)
                for (int i = x; i < end; ++i) idx[ao++] = (int64_t)y * W + i;
        } else {
            while (end < W && !r[end]) ++end;
        }
        x = end;
    }
}

__global__ void k_stamp(unsigned long long* t) { *t = globaltimer(); }

}  // namespace

cudaError_t launch_stamp(unsigned long long* t, cudaStream_t st) {
    k_stamp<<<1, 1, 0, st>>>(t);
    return cudaGetLastError();
}

cudaError_t launch_tile_compact(const uint8_t* active, int W, int H, int pitch_mask, int* d_tile_blocks,
                                int* d_tile_count, unsigned long long* d_inactive, cudaStream_t st) {
    const DenseTiling t = dense_tiling(W, H);
    k_tile_compact<<<dim3(t.tiles_x, t.tiles_y), 256, 0, st>>>(active, W, H, pitch_mask, d_tile_blocks,
                                                               d_tile_count, d_inactive);
    return cudaGetLastError();
}

cudaError_t launch_fill_u8(uint8_t* p, uint8_t v, size_t n, cudaStream_t st) {
    k_fill_u8<<<1184, 256, 0, st>>>(p, v, n);
    return cudaGetLastError();
}

cudaError_t launch_count_inactive(const uint8_t* active, size_t n, unsigned long long* out, cudaStream_t st) {
    k_count_zero<<<1184, 256, 0, st>>>(active, n, out);
    return cudaGetLastError();
}

cudaError_t launch_row_runs(const uint8_t* active, int W, int H, int* d_counts, cudaStream_t st) {
    k_row_count<<<(H + 127) / 128, 128, 0, st>>>(active, W, H, d_counts);
    return cudaGetLastError();
}

cudaError_t launch_row_runs_emit(const uint8_t* active, int W, int H, const long long* d_run_off,
                                 const long long* d_act_off, int32_t* d_runs, int64_t* d_idx, cudaStream_t st) {
    k_row_emit<<<(H + 127) / 128, 128, 0, st>>>(active, W, H, d_run_off, d_act_off, d_runs, d_idx);
    return cudaGetLastError();
}

}  // namespace fdg

namespace fdg {
namespace {
// q = f / max(c, eps) over a pitched batch (selective RL start: cachedV = 0,
// so every pixel's quotient is defined before the first masked pass)
__global__ void k_quot_const(const float* f, float* q, int W, int H, int pitch, long long bstride, int batch,
                             float c, float eps) {
    const long long n = (long long)W * H * batch;
    const float d = c < eps ? eps : c;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long b = i / ((long long)W * H), r = i - b * W * H;
        const long long idx = b * bstride + (r / W) * pitch + (r % W);
        q[idx] = f[idx] / d;
    }
}
}  // namespace

cudaError_t launch_quot_const(const float* f, float* q, int W, int H, int pitch, long long bstride, int batch,
                              float c, float eps, cudaStream_t st) {
    k_quot_const<<<1184, 256, 0, st>>>(f, q, W, H, pitch, bstride, batch, c, eps);
    return cudaGetLastError();
}
}  // namespace fdg

namespace fdg {
namespace {
// first non-finite / first negative row-major index: float4 per thread
// (rows are 16-byte aligned, pitch % 4 == 0), one integer division per 4 px
__global__ void k_validate(const float* f, int W, int H, int pitch, unsigned long long* out,
                           unsigned long long first = 0) {
    unsigned long long bad_nf = ~0ull, bad_neg = ~0ull;
    const long long nq = (W + 3) / 4;
    const long long n = nq * H;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
        const long long y = t / nq;
        const int x = 4 * (int)(t - y * nq);
        const float* row = f + y * pitch;
        float v[4];
        if (x + 3 < W) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(row + x));
            v[0] = q.x;
            v[1] = q.y;
            v[2] = q.z;
            v[3] = q.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = x + e < W ? row[x + e] : 0.f;
        }
        const unsigned long long base = first + (unsigned long long)y * W + x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (!isfinite(v[e])) bad_nf = min(bad_nf, base + e);
            else if (v[e] < 0.f) bad_neg = min(bad_neg, base + e);
        }
    }
    // warp minimum of 64-bit values: two 32-bit passes
    auto wmin = [](unsigned long long v) {
        const unsigned hi = __reduce_min_sync(0xffffffffu, (unsigned)(v >> 32));
        const unsigned lo = __reduce_min_sync(0xffffffffu, (unsigned)(v >> 32) == hi ? (unsigned)v : ~0u);
        return ((unsigned long long)hi << 32) | lo;
    };
    bad_nf = wmin(bad_nf);
    bad_neg = wmin(bad_neg);
    if ((threadIdx.x & 31) == 0) {
        if (bad_nf != ~0ull) atomicMin(&out[0], bad_nf);
        if (bad_neg != ~0ull) atomicMin(&out[1], bad_neg);
    }
}
__global__ void k_fill_u64(unsigned long long* p, int n) {
    if (threadIdx.x < n) p[threadIdx.x] = ~0ull;
}
}  // namespace

cudaError_t launch_validate(const float* f, int W, int H, int pitch, unsigned long long* out, cudaStream_t st) {
    k_fill_u64<<<1, 32, 0, st>>>(out, 2);
    k_validate<<<1184, 256, 0, st>>>(f, W, H, pitch, out);
    return cudaGetLastError();
}

// rows [r0, r0 + rows) of an image whose row 0 is f (indices stay those of
// the whole image); init: reset the two slots first
cudaError_t launch_validate_rows(const float* f, int W, int r0, int rows, int pitch, unsigned long long* out, int init,
                                 cudaStream_t st) {
    if (init) k_fill_u64<<<1, 32, 0, st>>>(out, 2);
    if (rows > 0)
        k_validate<<<592, 256, 0, st>>>(f + (size_t)r0 * pitch, W, rows, pitch, out, (unsigned long long)r0 * W);
    return cudaGetLastError();
}
}  // namespace fdg
