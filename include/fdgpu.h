/*
 * fdgpu.h -- C ABI of the B200-native Richardson-Lucy hot path
 *            (libfdgpu.so, hand-written sm_100a CUDA).
 *
 * The reference (fastdeconv, /root/reference/proj/include/fastdeconv) is a
 * header-only C++20 library with no ABI of its own.  This header is the
 * boundary its hot path is re-bound to: every entry point below replaces one
 * reference function (cited per declaration), with plain pointers and sizes,
 * int status codes instead of exceptions, and no torch / C++ types.  The C++
 * drop-in headers (include/fastdeconv/{convolve,rl}.hpp) and the Python
 * package (paper_1304_7211_b200) are thin marshalling layers over it.
 *
 * Images are row-major float32 planes, width*height (host entry points) or
 * width x height with a row pitch in elements (device entry points; pitch a
 * multiple of 4, pointers 16-byte aligned).  Arithmetic is fp32 on the device
 * (the reference computes in fp64; the parity bound is max-rel <= 1e-4 after
 * the configured iteration count).  There is no CPU fallback: without a CUDA
 * device every compute entry point returns FDG_ECUDA.
 */
#ifndef FDGPU_H
#define FDGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FDG_ABI_VERSION 1

/* status codes: the reference's exception classes */
#define FDG_OK 0
#define FDG_EINVAL 1   /* std::invalid_argument (validation, dispatch)      */
#define FDG_ENAN 2     /* std::runtime_error "NaN in iterate at iteration k" */
#define FDG_ELOGIC 3   /* std::logic_error                                   */
#define FDG_ECUDA 4    /* no device / CUDA failure (no fallback exists)      */

/* OperatorKind, same numbering as convolve.hpp:22-32 */
enum fdg_op {
    FDG_OP_NAIVE = 0,
    FDG_OP_LIST = 1,
    FDG_OP_GENERIC_BOX = 2,
    FDG_OP_BOX2D_SLIDING = 3,
    FDG_OP_BOX2D_CUMUL = 4,
    FDG_OP_BOX1D_SLIDING = 5,
    FDG_OP_BOX1D_CUMUL = 6,
    FDG_OP_FOURIER = 7,
    FDG_OP_AUTO = 8
};

/* Psf variant alternative, psf.hpp:173 */
enum fdg_repr { FDG_PSF_DENSE = 0, FDG_PSF_UNIFORM_CONVEX = 1, FDG_PSF_SPARSE = 2 };

/* PSF as the reference stores it (normalised weights).
 *   DensePsf          psf.hpp:26-70   width,height,anchor_x,anchor_y,weights[w*h]
 *   UniformConvexPsf  psf.hpp:75-120  n_rows,row_dy[],row_xmin[],row_xmax[]
 *   SparsePsf         psf.hpp:124-170 n_taps,tap_dx[],tap_dy[],tap_w[]          */
typedef struct fdg_psf_desc {
    int repr;
    int width, height, anchor_x, anchor_y;
    const double* weights;
    int n_rows;
    const int *row_dy, *row_xmin, *row_xmax;
    int n_taps;
    const int *tap_dx, *tap_dy;
    const double* tap_w;
} fdg_psf_desc;

/* RlConfig, rl.hpp:18-23 */
typedef struct fdg_rl_config {
    int iterations;
    int op;
    double epsilon_div;
    int clamp_nonnegative;
} fdg_rl_config;

/* RlIterationRecord, rl.hpp:25-30 */
typedef struct fdg_rl_record {
    int iteration;
    double inactive_fraction;
    double max_abs_change;
    double seconds;
} fdg_rl_record;

typedef struct fdg_ctx fdg_ctx;
typedef struct fdg_plan fdg_plan;
typedef struct fdg_solver fdg_solver;

int fdg_abi_version(void);
/* last error message of this thread (ctx-independent) */
const char* fdg_last_error(void);
/* 1 when a CUDA device is usable, else 0 */
int fdg_device_available(void);
/* the calling thread's current CUDA device (FDG_ECUDA without a device) */
int fdg_get_device(int* device);
/* Process-wide engine options (no reference counterpart; tuning/testing):
 *   "fused": 1 = run each RL iteration of a centred odd box (extents 3 ..
 *            17, square or not; config 4 = 15x15) as one fused pass
 *            (kernels_fused.cu) when a launch is large enough for it to beat
 *            the two passes (~3 Mpx; ~12 Mpx for boxes up to 9 px; default),
 *            2 = whatever the size, 0 = two fused-epilogue passes.
 *   "spans": GenericBox span-table kernels (kernels_spans.cu): 0 = by size
 *            (tile kernel up to 4.5 Mpx per launch, default), 1 = tile
 *            kernel, 2 = marching kernel.
 *   "pipeline": fdg_rl_deconvolve with the fused engine runs as time-skewed
 *            row strips whose uploads / downloads (pageable buffers: staged)
 *            overlap the iterations: 1 = when the hidden copies outweigh
 *            the strips' extra launches (default; ~100 Mpx at 100
 *            iterations), 0 = never, 2 = whenever engine and buffers allow.
 * Returns the previous value, or -1 for an unknown name. */
int fdg_set_option(const char* name, int value);

/* Context: device, stream (default: a private non-blocking stream), scratch
 * and pinned staging buffers.  Calls on one context are serialised (one
 * caller at a time); calls on different contexts share nothing, so a
 * per-thread context makes the API reentrant like the reference
 * (SPEC.md:314).  Every entry point runs on the context's device and
 * restores the caller's current device.  fdg_ctx_destroy drops the caller's
 * reference: plans and solvers created on the context keep it alive. */
int fdg_ctx_create(int device, fdg_ctx** out);
void fdg_ctx_destroy(fdg_ctx* ctx);
/* run on an external cudaStream_t (e.g. torch.cuda.current_stream()) */
int fdg_ctx_set_stream(fdg_ctx* ctx, void* cuda_stream);
int fdg_ctx_synchronize(fdg_ctx* ctx);
/* number of kernel launches issued through this context so far */
uint64_t fdg_ctx_launch_count(const fdg_ctx* ctx);
/* Layout of the strip pipeline (no reference counterpart; host only): first
 * rows of the strips at iteration 0 for a width x height image whose fused
 * iteration reaches `shift` rows up and down (2 x the box's vertical radius),
 * chosen by the library's timeline model of the call.
 * Strip s covers rows [bounds[s] - shift k, bounds[s + 1] - shift k) of
 * iteration k, clipped to the image (strip 0 from row 0, the last strip to the
 * last row).  Returns the number of strips. */
int fdg_pipeline_layout(int width, int height, int shift, int iterations, int* bounds, int cap);
/* schedule of the context's last fdg_rl_deconvolve: 0 = upload, iterate,
 * download; n >= 2 = time-skewed pipeline over n row strips */
int fdg_ctx_last_schedule(const fdg_ctx* ctx);

/* ---- plan logic (host only; no device needed) ----------------------- */
/* dispatch(), convolve.hpp:627-643 -> *kind, or FDG_EINVAL naming op+PSF */
int fdg_dispatch(const fdg_psf_desc* psf, int preference, int* kind);
/* operatorAcceptsPsf(), convolve.hpp:607-625 */
int fdg_operator_accepts(int kind, const fdg_psf_desc* psf, int* accepts);

/* ConvPlan(psf, preference), convolve.hpp:652-676.  The plan holds the
 * device representation (uploaded on ctx's device) and is immutable: any
 * context on that device may apply it concurrently (fdg_conv_apply_ctx). */
int fdg_plan_create(fdg_ctx* ctx, const fdg_psf_desc* psf, int preference, fdg_plan** out);
void fdg_plan_destroy(fdg_plan* plan);
/* ConvPlan::kind(), convolve.hpp:678 */
int fdg_plan_kind(const fdg_plan* plan);
/* ConvCounters the reference operator would report for one width x height
 * application (convolve.hpp:140-143,165-167,206-210,239-243,274-278,
 * 315-318,328,339-341,372,383-386); analytic, no device work. */
int fdg_plan_counters(const fdg_plan* plan, int width, int height, uint64_t counters[3]);
/* the same counters without a device: dispatch + analytic formulas */
int fdg_op_counters(const fdg_psf_desc* psf, int preference, int width, int height,
                    uint64_t counters[3]);
/* which device engine serves the plan: "rows", "box2d", "spans", "dense",
 * "taps" or "cyclic" (diagnostics / bench labels) */
const char* fdg_plan_engine(const fdg_plan* plan);
/* CUDA device the plan's representation lives on */
int fdg_plan_device(const fdg_plan* plan);

/* ConvPlan::applyInto, convolve.hpp:680-715 (host buffers), on the calling
 * thread's context `ctx` (scratch, stream); fdg_conv_apply uses the context
 * the plan was created on. */
int fdg_conv_apply_ctx(fdg_ctx* ctx, const fdg_plan* plan, const float* in, int width, int height, float* out);
int fdg_conv_apply(fdg_plan* plan, const float* in, int width, int height, float* out);
/* ConvPlan::applyMaskedInto, convolve.hpp:724-736: only Naive and List plans,
 * else FDG_EINVAL "operator does not support masked evaluation" */
int fdg_conv_apply_masked_ctx(fdg_ctx* ctx, const fdg_plan* plan, const float* in, int width, int height,
                              const uint8_t* active, const float* fallback, float* out);
int fdg_conv_apply_masked(fdg_plan* plan, const float* in, int width, int height,
                          const uint8_t* active, const float* fallback, float* out);
/* device-resident variant on the context stream */
int fdg_conv_apply_device(fdg_plan* plan, const float* d_in, float* d_out, int width, int height,
                          int pitch);

/* ---- Richardson-Lucy drivers (host buffers) ------------------------- */
/* rlDeconvolve, rl.hpp:140-179.  trace: nullable, cfg->iterations records;
 * seconds = per-iteration device time (%globaltimer stamps written by each
 * iteration's last kernel, so graph-replayed loops report real per-iteration
 * times).  The input check of rl.hpp:78-83 runs on the device and its
 * verdict returns with the trace (one synchronisation per call): on any
 * error the contents of u_out are unspecified. */
int fdg_rl_deconvolve(fdg_ctx* ctx, const fdg_psf_desc* psf, const fdg_rl_config* cfg,
                      const float* f, int width, int height, float* u_out, fdg_rl_record* trace);
/* The same on the reference's own pixel type (Image holds doubles,
 * image.hpp:14-52): rlDeconvolve(const Image&, ...), rl.hpp:140-179, binds
 * here.  The doubles become the device's fp32 planes on their way through the
 * pinned staging chunks (a multi-threaded pass per chunk, strip by strip
 * behind the iterations when the strip pipeline applies) and the result comes
 * back the same way -- no float copy of the image on the host.  rl.hpp:78-83
 * is checked on the caller's doubles in that pass (first non-finite or
 * negative pixel in row-major order decides the message; a finite value
 * beyond FLT_MAX is refused with "input pixel exceeds the fp32 range of the
 * GPU path"); the verdict is read after the loop. */
int fdg_rl_deconvolve_f64(fdg_ctx* ctx, const fdg_psf_desc* psf, const fdg_rl_config* cfg,
                          const double* f, int width, int height, double* u_out, fdg_rl_record* trace);
/* rlDeconvolve over `batch` independent width x height images stored one
 * after another (f, u_out: batch * width * height floats).  One solver runs
 * the images in chunks; with page-locked host buffers the upload of the next
 * chunk and the download of the previous one overlap the iterations of the
 * current chunk (copy engines vs SMs).  trace (nullable, iterations
 * records): max|du| over the batch, seconds summed over the chunks.  Same
 * errors as fdg_rl_deconvolve (any image). */
int fdg_rl_deconvolve_batch(fdg_ctx* ctx, const fdg_psf_desc* psf, const fdg_rl_config* cfg, const float* f,
                            int width, int height, int batch, float* u_out, fdg_rl_record* trace);
/* rlDeconvolveSelective, rl.hpp:187-257.  thin_start: deactivation is held
 * off for 0-based k < thin_start (0 = the reference).  mask_replay
 * (nullable, iterations*width*height bytes) replaces the device's own
 * deactivation decisions with recorded masks; mask_record (nullable) gets
 * the mask each iteration's convolutions used. */
int fdg_rl_deconvolve_selective(fdg_ctx* ctx, const fdg_psf_desc* psf, const fdg_rl_config* cfg,
                                double threshold, int period, int thin_start,
                                const uint8_t* mask_replay, uint8_t* mask_record, const float* f,
                                int width, int height, float* u_out, fdg_rl_record* trace);
/* rlStep, rl.hpp:131-137 */
int fdg_rl_step(fdg_ctx* ctx, const fdg_psf_desc* psf, const fdg_rl_config* cfg, const float* u,
                const float* f, int width, int height, float* u_out, double* max_abs_change);
/* detail::rlStepPlanned, rl.hpp:101-125: one step with the caller's forward
 * and adjoint plans (both on ctx's device) */
int fdg_rl_step_planned(fdg_ctx* ctx, const fdg_plan* forward, const fdg_plan* adjoint, const fdg_rl_config* cfg,
                        const float* u, const float* f, int width, int height, float* u_out,
                        double* max_abs_change);

/* ---- device-resident solver (bench, sharding, batches) --------------- */
/* Plans for h and adjoint(h) + per-iteration trace arrays, for `batch`
 * images of width x height (rows of a shard may carry halos: see
 * fdg_solver_pass). */
int fdg_solver_create(fdg_ctx* ctx, const fdg_psf_desc* psf, const fdg_rl_config* cfg, int width,
                      int height, int batch, fdg_solver** out);
void fdg_solver_destroy(fdg_solver* s);
/* Full RL loop in place on device buffers: u <- f, then cfg->iterations
 * iterations (q is a solver-owned scratch plane).  Images are `batch`
 * planes of height rows each, `image_stride` elements apart. */
int fdg_solver_run(fdg_solver* s, const float* d_f, float* d_u, int pitch, long long image_stride,
                   int iterations);
/* One fused pass over output rows [y0, y1) of each image, reading input rows
 * clamped to [ylo, yhi] (relative to the same row 0; halos of a row strip
 * are rows < 0 or >= height).  pass 1: out = aux / max(h (x) in, eps)
 * (aux = f);  pass 2: out = max(h* (x) in * aux, 0) (aux = u; out may alias
 * aux) with max|du| and NaN accumulated into trace slot `iteration`. */
int fdg_solver_pass(fdg_solver* s, int pass, const float* d_in, const float* d_aux, float* d_out,
                    int pitch, long long image_stride, int y0, int y1, int ylo, int yhi,
                    int iteration);
/* One whole RL iteration with the fused engine (fdg_solver_engine() ==
 * "fused"): u_out rows [y0, y1) from u_in, reading rows clamped into
 * [ylo, yhi] (same row convention as fdg_solver_pass; a row strip needs
 * 2 x (PSF vertical radius) valid halo rows of u_in on each inner side).
 * u_in != u_out. */
int fdg_solver_iterate(fdg_solver* s, const float* d_f, const float* d_u_in, float* d_u_out, int pitch,
                       long long image_stride, int y0, int y1, int ylo, int yhi, int iteration);
/* copy per-iteration {max|du|, NaN (in inactive_fraction), seconds} of the
 * last run back (synchronises) */
int fdg_solver_trace(fdg_solver* s, fdg_rl_record* out, int n);
/* Engine fdg_solver_run uses: "fused" (one launch per iteration), "rowres"
 * (one launch per run) or the plan engine of the two-pass loop ("box",
 * "spans", "taps", "dense"). */
const char* fdg_solver_engine(const fdg_solver* s);
int fdg_solver_reset_trace(fdg_solver* s);

/* ---- stream compaction (selective path) ------------------------------ */
/* Row-major active list and (y, x0, len) runs of a device mask, the order
 * of the reference's run walk (convolve.hpp:450-465).  Host buffers out;
 * returns counts through n_active / n_runs (buffers may be NULL to query). */
int fdg_mask_compact(fdg_ctx* ctx, const uint8_t* active, int width, int height,
                     int64_t* idx, int64_t idx_cap, int64_t* n_active, int32_t* runs,
                     int64_t runs_cap, int64_t* n_runs);

/* ---- row-strip sharded RL --------------------------------
 * One image of width x height split into `world` row strips, one per rank
 * (one process per GPU).  Rank r owns rows [r*H/world, (r+1)*H/world) and
 * runs the loop of rlDeconvolve (rl.hpp:153-177) on them; each iteration
 * exchanges PSF-radius halo rows with ranks r-1 / r+1 through NCCL
 * send/recv (NVLink), posted on a communication stream while the strip
 * interior is computed, the two boundary bands following once the halo has
 * landed.  Replicate clamping only at global rows 0 and H-1, so the result
 * equals the single-GPU run.  Engines: "fused" (centred 15x15 box: one
 * exchange of 2T rows per iteration), "rowres" (horizontal lines at dy = 0:
 * rows independent, no exchange), else two passes with a T-row exchange of
 * u and of q.  NCCL (libnccl.so.2) is loaded at run time (FDG_NCCL_LIB
 * overrides the path); world == 1 needs no NCCL. */
typedef struct fdg_shard fdg_shard;
/* ncclGetUniqueId: rank 0 calls it and sends the 128 bytes to every rank */
int fdg_comm_unique_id(unsigned char id[128]);
/* this process's strip (rank of world; comm_id may be NULL when world == 1;
 * given with world == 1, a one-rank NCCL communicator carries the trace
 * all-reduce) */
int fdg_shard_create(fdg_ctx* ctx, const fdg_psf_desc* psf, const fdg_rl_config* cfg, int width, int height,
                     int rank, int world, const unsigned char* comm_id, fdg_shard** out);
/* `world` strips of one image in THIS process on ctx's device, the halo
 * exchange done by device copies between them (tests / single-GPU
 * measurement of the sharded schedule): out[0..world-1] */
int fdg_shard_group_create(fdg_ctx* ctx, const fdg_psf_desc* psf, const fdg_rl_config* cfg, int width,
                           int height, int world, fdg_shard** out);
void fdg_shard_destroy(fdg_shard* s);
/* info[0..5] = first row, core rows, halo rows, exchanges per iteration,
 * halo bytes sent per iteration, engine id (0 fused, 1 two-pass, 2 rowres) */
int fdg_shard_info(const fdg_shard* s, long long info[6]);
const char* fdg_shard_engine(const fdg_shard* s);
/* RL on this rank's strip: f / u = its core rows (row r0 .. r0+core-1),
 * host (host != 0) or device memory, row pitch `pitch` floats.  Device
 * buffers and trace == NULL: asynchronous on ctx's stream.  trace (n =
 * iterations): max|du| and NaN reduced over all ranks (one all-reduce at
 * the end), seconds = this rank's device time per iteration. */
int fdg_shard_run(fdg_shard* s, const float* f, float* u, int pitch, int host, int iterations,
                  fdg_rl_record* trace);
/* a group from fdg_shard_group_create: f / u = the whole image */
int fdg_shard_group_run(fdg_shard** group, int world, const float* f, float* u, int pitch, int host,
                        int iterations, fdg_rl_record* trace);
/* device time of the last run's kernels per iteration, split: [0] interior
 * launches, [1] boundary-band launches, [2] halo exchange (ms, summed over
 * iterations; events on the launching streams) */
int fdg_shard_timing(fdg_shard* s, double ms[3]);

#ifdef __cplusplus
}
#endif
#endif
