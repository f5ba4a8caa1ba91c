// internal.h -- shared declarations of libfdgpu (host plan logic + kernel
// launchers).  Not part of the ABI; see include/fdgpu.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "fdgpu.h"

namespace fdg {

// ---------------------------------------------------------------- host PSF
struct Tap {
    int dx, dy;
    double w;
};
struct Span {
    int dy, xmin, xmax;
};

// A restated Psf variant (psf.hpp:173) built from an fdg_psf_desc.
struct HostPsf {
    int repr = FDG_PSF_DENSE;
    int w = 0, h = 0, ax = 0, ay = 0;  // DensePsf
    std::vector<double> weights;
    std::vector<Span> rows;  // UniformConvexPsf
    std::vector<Tap> taps;   // SparsePsf
};

struct LineShape {
    int length, min_dx, dy;
};
struct RectShape {
    int mx, my, min_dx, min_dy;
};

// psf.hpp restatement used by the plan builder (plan.cpp)
bool psf_from_desc(const fdg_psf_desc* d, HostPsf* out, std::string* err);
HostPsf psf_adjoint(const HostPsf& p);
std::vector<Tap> psf_taps(const HostPsf& p);  // toSparse order
bool psf_as_line(const HostPsf& p, LineShape* out);
bool psf_as_rect(const HostPsf& p, RectShape* out);
bool psf_as_convex(const HostPsf& p, std::vector<Span>* out);
bool psf_accepts(int kind, const HostPsf& p);
int psf_dispatch(const HostPsf& p, int preference, std::string* err);  // -1 on error
const char* op_name(int kind);

// ------------------------------------------------------------ device plan
enum Engine { ENG_RECT = 0, ENG_SPANS = 1, ENG_DENSE = 2, ENG_TAPS = 3, ENG_CYCLIC = 4 };

struct DevPsf {
    int engine = ENG_TAPS;
    int min_dx = 0, max_dx = 0, min_dy = 0, max_dy = 0;  // tap extents
    int mx = 1, my = 1;                                  // rect engine
    int uniform = 0;
    float scale = 1.f;  // uniform weight (1/count) or 1
    int nrows = 0, ntaps = 0;
    int* d_row_start = nullptr;  // [nrows+1], rows r = dy - min_dy
    int* d_dx = nullptr;         // [ntaps]
    float* d_w = nullptr;        // [ntaps]
    std::vector<int> h_span;     // [2*nrows] xmin,xmax per row (spans engine, host)
    std::vector<int> h_row_start, h_dx;  // taps engine, host copies (JIT tap kernels)
    std::vector<float> h_w;
    int mw = 0, mh = 0, mwp = 0;  // dense engine: grid, padded width
    float* d_dense = nullptr;     // [mh * mwp]
    std::vector<float> h_dense;   // host copy (passed as kernel parameters)
};

enum EpiMode {
    EPI_STORE = 0,    // out = v
    EPI_QUOT = 1,     // out = aux / max(v, eps)
    EPI_UPDATE = 2,   // out = clamp(v * aux); max|out-aux|, NaN
    EPI_MQUOT = 3,    // masked fwd: active: out2(cachedV) = v, out = aux / max(v, eps)
    EPI_MUPDATE = 4,  // masked adj: active: as UPDATE + deactivate when |du| < thr
};

struct Epi {
    int mode = EPI_STORE;
    const float* aux = nullptr;
    float* out2 = nullptr;
    float eps = 1e-8f;
    int clamp = 1;
    unsigned* maxchange = nullptr;  // float bits, atomicMax
    int* nanflag = nullptr;
    unsigned long long* tend = nullptr;  // %globaltimer at the end of the pass (atomicMax)
    uint8_t* active = nullptr;      // masked modes / masked store
    float thr = 0.f;
    int may_thin = 0;
};

struct Geom {
    const float* in = nullptr;
    float* out = nullptr;
    int pitch = 0;
    int W = 0;
    int y0 = 0, y1 = 0;    // output rows [y0, y1)
    int ylo = 0, yhi = 0;  // readable input rows (inclusive clamp range)
    int batch = 1;
    long long bstride = 0;  // elements between images
    int wrap = 0;           // cyclic boundary (Fourier contract)
};

// kernel launchers (return cudaError_t of the launch)
cudaError_t launch_rect(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st);
cudaError_t launch_taps(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st);
cudaError_t launch_dense(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st,
                         const int* d_tile_blocks, const int* d_tile_count);
cudaError_t launch_spans(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st);
bool spans_supported(const DevPsf& p);
// runtime span-table kernel (kernels_spanr.cu): any row-convex PSF with
// <= 64 rows and max_dx - min_dx <= 64
bool spanr_supported(const DevPsf& p);
cudaError_t launch_spanr(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st);
// span tile kernel compiled at run time for a plan's table (spans_jit.cu,
// NVRTC); ready() compiles on first use per table and device (plan build)
bool spans_jit_ready(const DevPsf& p);
// the per-tap tile kernel compiled at run time for a plan's tap list
// (List / wide Naive / Fourier passes, masked ones too; <= 128 taps, x extent <= 65)
bool taps_jit_ready(const DevPsf& p);
cudaError_t launch_taps_jit(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st);
cudaError_t launch_spans_jit(const DevPsf& p, const Geom& g, const Epi& e, cudaStream_t st);
void set_spans_jit(int v);
int spans_jit_mode();
// "tile" / "marching" (compile-time tables), "jit-tile" or "runtime-table"
const char* spans_kernel(const DevPsf& p, long long px);
// spans kernel choice: 0 = by image size (tile <= 4.5 Mpx per launch), 1 = tile, 2 = marching,
// 3 = the runtime-table kernel for every shape
void set_spans_mode(int v);
int spans_mode();
bool dense_supported(const DevPsf& p);

// compaction (kernels_mask.cu)
struct DenseTiling {
    int tiles_x, tiles_y;
};
DenseTiling dense_tiling(int W, int H);
cudaError_t launch_tile_compact(const uint8_t* active, int W, int H, int pitch_mask,
                                int* d_tile_blocks, int* d_tile_count,
                                unsigned long long* d_inactive, cudaStream_t st);
cudaError_t launch_fill_u8(uint8_t* p, uint8_t v, size_t n, cudaStream_t st);
cudaError_t launch_row_runs(const uint8_t* active, int W, int H, int* d_counts, cudaStream_t st);
cudaError_t launch_row_runs_emit(const uint8_t* active, int W, int H, const long long* d_run_off,
                                 const long long* d_act_off, int32_t* d_runs, int64_t* d_idx,
                                 cudaStream_t st);
cudaError_t launch_quot_const(const float* f, float* q, int W, int H, int pitch, long long bstride, int batch,
                              float c, float eps, cudaStream_t st);
bool rect_supported(int mx);
bool rowres_supported(int mx, int my, int min_dx, int min_dy, int W);
cudaError_t launch_rowres(int mx, int min_dx, float inv_m, const float* f, float* u, int pitch, int W, int H,
                          int batch, long long bstride, int iters, float eps, int clamp, unsigned* maxchange,
                          int* nanflag, unsigned long long* tend, unsigned long long* tbegin, unsigned long long* tdur,
                          cudaStream_t st);
// Whole RL iteration in one pass for centred 9x9 / 15x15 / 17x17 boxes (kernels_fused.cu):
// u_out = max(box*(f / max(box(u_in), eps)) * u_in, 0); u_in != u_out.
bool fused_supported(int mx, int my, int min_dx, int min_dy);
void set_fused_mode(int v);
int fused_mode();
// Output rows [y0, y1) (and [y2, y3) when y3 > y2: the two boundary bands of
// a row strip in one launch), reads clamped into [ylo, yhi] (the image edges; rows
// ... balanced = 0: the plain strip x band grid instead of work-balanced
// segments (row strips of a sharded image: 145 vs 150 us per 2048-row strip)
// between a shard's core and those edges must hold valid halo rows).
// halo_in / halo_out: u_in / u_out are haloed planes (pitch_h, bstride_h;
// fused_halo_left() / _right() replicated columns around each row; the
// pointer addresses column 0), else they use f's pitch and stride.  Halo
// input needs W >= the kernel's strip width (fused_halo_ok).
cudaError_t launch_fused(const float* u_in, const float* f, float* u_out, int pitch, int W, int y0, int y1, int ylo,
                         int yhi, int batch, long long bstride, float scale, float eps, int clamp,
                         unsigned* maxchange, int* nanflag, unsigned long long* tend, cudaStream_t st,
                         int halo_in = 0, int halo_out = 0, int pitch_h = 0, long long bstride_h = 0,
                         int y2 = 0, int y3 = 0, int balanced = 1, int rx = 7, int ry = 7);
// The boundary bands of a row strip for the fused iteration (kernels_band.cu):
// output rows [y0, y1) and [y2, y3) computed in place per 16 x 16 tile (no
// row streaming), small enough to run next to the fused interior launch.
cudaError_t launch_band(const float* u_in, int pitch_u, const float* f, int pitch_f, float* u_out, int pitch_o,
                        int W, int y0, int y1, int y2, int y3, int ylo, int yhi, float scale, float eps, int clamp,
                        int halo_out, int halo_l, int halo_r, unsigned* maxchange, int* nanflag,
                        unsigned long long* tend, cudaStream_t st);
int fused_halo_left();
int fused_halo_right();
bool fused_halo_ok(int W);
// haloed copy of src (dst addresses column 0 of the haloed plane)
cudaError_t launch_pad_halo(const float* src, int pitch_src, long long bs_src, float* dst, int pitch_dst,
                            long long bs_dst, int W, int H, int batch, cudaStream_t st);
// first non-finite / first negative row-major index (~0 if none) -> out[0..1]
cudaError_t launch_validate(const float* f, int W, int H, int pitch, unsigned long long* out, cudaStream_t st);
cudaError_t launch_validate_rows(const float* f, int W, int r0, int rows, int pitch, unsigned long long* out, int init,
                                 cudaStream_t st);
// one thread writes %globaltimer to *t (start stamp of a timed RL loop)
cudaError_t launch_stamp(unsigned long long* t, cudaStream_t st);
cudaError_t launch_count_inactive(const uint8_t* active, size_t n, unsigned long long* out,
                                  cudaStream_t st);

}  // namespace fdg
