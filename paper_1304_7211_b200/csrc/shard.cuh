// shard.cuh -- row-strip sharded Richardson-Lucy: the
// fdg_shard_* entry points of include/fdgpu.h.  Part of fdgpu.cu's
// translation unit (it uses the plan, pass and trace internals there).
//
// Each rank runs the loop of rl.hpp:153-177 on its rows [r0, r0 + core) of
// the image, stored with `halo` extra rows above and below (planes address
// core row 0).  Per iteration, on two streams:
//
//   comm   wait(u ready) -> NCCL group {send the halo rows next to each inner
//          edge, receive the neighbours' into the halo} -> record(halo)
//   comp   interior rows [halo, core - halo)  (windows stay inside the core)
//          wait(halo) -> both boundary bands in ONE launch -> record(u ready)
//
// so the exchange is in flight while the interior -- all but 2 x halo rows
// -- is computed.  The fused engine (centred 15x15 box) needs one exchange
// of 2T = 14 rows of u per iteration (the q rows beyond the core are
// recomputed from them); the two-pass engines exchange T rows of u before
// pass 1 and T rows of q before pass 2; the row-resident engine (horizontal
// lines at dy = 0) needs none.  Replicate clamping only at global rows 0 and
// H - 1 (ylo / yhi), so strips reproduce the single-GPU result.
//
// Hazards (ping-pong u planes A/B; iteration k reads A, writes B):
//   * send(k) reads A's core edge rows, recv(k) writes A's halo rows; the
//     interior(k) reads A's core rows only and writes B's interior: no
//     conflict; the bands(k) wait for recv(k).
//   * iteration k+1 writes A again: its interior touches only A's interior
//     rows (send(k) read edge rows); its bands wait for halo(k+1), which is
//     behind send(k) on the comm stream.
// The per-iteration max|du| / NaN slots stay on each device and are reduced
// over the ranks once, after the loop (ncclAllReduce max).
//
// NCCL is resolved with dlopen at first use (libnccl.so.2, the copy torch
// already loaded when present; FDG_NCCL_LIB overrides), so the library has
// no link-time NCCL dependency and world == 1 never touches it.
// fdg_shard_group_create builds `world` strips in one process on one device
// whose exchange is a device copy between the strips' planes: the same
// schedule, row ranges and kernels, checkable against the single-image run
// (tests) and timeable on one GPU.
#include <dlfcn.h>

namespace {

// ---- the NCCL ABI subset (nccl.h, NCCL 2.x; stable) -----------------------
typedef struct {
    char internal[128];
} nccl_unique_id;
typedef void* nccl_comm;
enum { NCCL_OK = 0, NCCL_UINT32 = 3, NCCL_FLOAT32 = 7, NCCL_MAX = 2 };

struct NcclApi {
    int (*get_unique_id)(nccl_unique_id*) = nullptr;
    int (*comm_init_rank)(nccl_comm*, int, nccl_unique_id, int) = nullptr;
    int (*comm_destroy)(nccl_comm) = nullptr;
    int (*send)(const void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    int (*recv)(void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    int (*all_reduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    int (*group_start)() = nullptr;
    int (*group_end)() = nullptr;
    const char* (*error_string)(int) = nullptr;
    bool ok = false;
    std::string err;
};

NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* env = getenv("FDG_NCCL_LIB");
        void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.err = std::string("cannot load NCCL (") + (env ? env : "libnccl.so.2") + "): " + dlerror();
            return;
        }
        bool all = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            all = all && fn != nullptr;
        };
        sym(api.get_unique_id, "ncclGetUniqueId");
        sym(api.comm_init_rank, "ncclCommInitRank");
        sym(api.comm_destroy, "ncclCommDestroy");
        sym(api.send, "ncclSend");
        sym(api.recv, "ncclRecv");
        sym(api.all_reduce, "ncclAllReduce");
        sym(api.group_start, "ncclGroupStart");
        sym(api.group_end, "ncclGroupEnd");
        sym(api.error_string, "ncclGetErrorString");
        api.ok = all;
        if (!all) api.err = "NCCL library lacks a required symbol";
    });
    return api;
}

int nccl_err(int r, const char* where) {
    NcclApi& a = nccl_api();
    return set_err(FDG_ECUDA, std::string(where) + ": " + (a.error_string ? a.error_string(r) : "NCCL error"));
}

#define NK(call)                                          \
    do {                                                  \
        int _r = (call);                                  \
        if (_r != NCCL_OK) return nccl_err(_r, #call);    \
    } while (0)

enum ShardEngine { SH_FUSED = 0, SH_TWOPASS = 1, SH_ROWRES = 2 };

// fdg_set_option("shard_loopback", 1): fdg_shard_create accepts world > 1
// without a communicator and exchanges a strip's own edge rows (results are
// meaningless; the per-rank schedule and its timing are the production ones)
std::atomic<int> g_shard_loopback{0};
bool shard_loopback() { return g_shard_loopback.load() != 0; }
// fdg_set_option("shard_bands", 0 | 1): fused boundary bands after the
// interior on the compute stream (0, default) or concurrently on a
// high-priority stream (1)
std::atomic<int> g_shard_bands{getenv("FDG_SHARD_BANDS") ? atoi(getenv("FDG_SHARD_BANDS")) : 0};
bool shard_bands_concurrent() { return g_shard_bands.load() != 0; }

}  // namespace

struct fdg_shard {
    fdg_ctx* ctx = nullptr;
    std::unique_ptr<fdg_plan> fwd, adj;
    fdg_rl_config cfg{};
    int W = 0, H = 0, rank = 0, world = 1;
    int r0 = 0, core = 0, T = 0, halo = 0, engine = SH_TWOPASS;
    nccl_comm comm = nullptr;
    std::vector<fdg_shard*> group;  // emulated group (device-copy exchange), else empty
    int pitch = 0;                  // f / two-pass planes
    HaloPlanes hp;                  // fused: u planes with replicated edge columns
    DevBuf<float> fb, ub, qb;       // planes incl. halo rows
    float* f = nullptr;             // core row 0 of each plane
    float* uA = nullptr;
    float* uB = nullptr;
    float* q = nullptr;
    int upitch = 0;
    DevBuf<unsigned> mc;
    DevBuf<int> nf;
    DevBuf<unsigned long long> ts;
    int ntrace = 0;
    bool loopback = false;          // timing mode: world > 1 without peers (exchange = own rows)
    cudaStream_t comm_st = nullptr;
    cudaStream_t band_st = nullptr;  // high priority: boundary bands next to the interior launch
    cudaEvent_t ev_ready = nullptr, ev_halo = nullptr, ev_join = nullptr, ev_band = nullptr;
    // per-iteration timing events: interior begin/end, bands begin/end, exchange begin/end
    std::vector<cudaEvent_t> tev;
    int t_iters = 0;
    ~fdg_shard() {
        DevScope ds;
        if (ctx) ds.enter(ctx->device);
        if (comm_st) cudaStreamSynchronize(comm_st);
        if (comm && nccl_api().ok) nccl_api().comm_destroy(comm);
        for (cudaEvent_t e : tev) cudaEventDestroy(e);
        if (ev_ready) cudaEventDestroy(ev_ready);
        if (ev_halo) cudaEventDestroy(ev_halo);
        if (ev_join) cudaEventDestroy(ev_join);
        if (ev_band) cudaEventDestroy(ev_band);
        if (band_st) cudaStreamSynchronize(band_st), cudaStreamDestroy(band_st);
        if (comm_st) cudaStreamDestroy(comm_st);
        fwd.reset();
        adj.reset();
        ctx_release(ctx);
    }
};

namespace {

int shard_init(fdg_shard* s, fdg_ctx* ctx, const fdg_psf_desc* psf, const fdg_rl_config* cfg, int W, int H,
               int rank, int world) {
    if (!cfg) return set_err(FDG_EINVAL, "null argument");
    if (W < 1 || H < 1) return set_err(FDG_EINVAL, "sharded RL: empty input image");
    if (world < 1 || rank < 0 || rank >= world) return set_err(FDG_EINVAL, "sharded RL: bad rank / world");
    if (!(cfg->epsilon_div > 0.0)) return set_err(FDG_EINVAL, "sharded RL: epsilonDiv must be positive");
    s->ctx = ctx;
    ctx_retain(ctx);
    s->cfg = *cfg;
    s->W = W;
    s->H = H;
    s->rank = rank;
    s->world = world;
    int st = make_rl_plans(ctx, psf, cfg->op, &s->fwd, &s->adj);
    if (st) return st;
    const DevPsf& d = s->fwd->dev;
    s->T = std::max(std::max(0, -d.min_dy), std::max(0, d.max_dy));
    if (use_fused(s->fwd.get()) && fused_halo_ok(W) && d.mx == 15 && d.my == 15) {  // k_band: the 15 x 15 box
        s->engine = SH_FUSED;
        s->halo = 2 * s->T;
    } else if (use_rowres(s->fwd.get(), W)) {
        s->engine = SH_ROWRES;
        s->halo = 0;
    } else {
        s->engine = SH_TWOPASS;
        s->halo = s->T;
    }
    s->r0 = (int)((long long)rank * H / world);
    s->core = (int)((long long)(rank + 1) * H / world) - s->r0;
    if (world > 1 && s->core < std::max(1, s->halo))
        return set_err(FDG_EINVAL, "sharded RL: strip of " + std::to_string(s->core) + " rows is thinner than its " +
                                       std::to_string(s->halo) + "-row halo");
    const int rows = s->core + 2 * s->halo;
    s->pitch = pitch_for(W);
    CK(s->fb.ensure((size_t)rows * s->pitch));
    s->f = s->fb.p + (size_t)s->halo * s->pitch;
    if (s->engine == SH_FUSED) {
        s->hp.pitch = (W + fused_halo_left() + fused_halo_right() + 31) & ~31;
        s->hp.stride = (long long)s->hp.pitch * rows;
        CK(s->ub.ensure(2 * (size_t)s->hp.stride + 32));
        s->uA = s->ub.p + fused_halo_left() + (size_t)s->halo * s->hp.pitch;
        s->uB = s->uA + s->hp.stride;
        s->hp.p[0] = s->uA;
        s->hp.p[1] = s->uB;
        s->upitch = s->hp.pitch;
    } else {
        CK(s->ub.ensure((size_t)rows * s->pitch));
        s->uA = s->ub.p + (size_t)s->halo * s->pitch;
        s->upitch = s->pitch;
        if (s->engine == SH_TWOPASS) {
            CK(s->qb.ensure((size_t)rows * s->pitch));
            s->q = s->qb.p + (size_t)s->halo * s->pitch;
        }
    }
    s->ntrace = std::max(cfg->iterations, 1);
    CK(s->mc.ensure(s->ntrace));
    CK(s->nf.ensure(s->ntrace));
    CK(s->ts.ensure(s->ntrace + 1));
    // the exchange must not queue behind the interior launch's CTAs (NCCL
    // send/recv and device copies are kernels too): highest priority
    int plo = 0, phi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&plo, &phi));
    CK(cudaStreamCreateWithPriority(&s->comm_st, cudaStreamNonBlocking, phi));
    CK(cudaEventCreateWithFlags(&s->ev_ready, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s->ev_halo, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s->ev_band, cudaEventDisableTiming));
    CK(cudaStreamCreateWithPriority(&s->band_st, cudaStreamNonBlocking, phi));
    return FDG_OK;
}

int shard_ylo(const fdg_shard* s) { return s->rank > 0 ? -s->halo : 0; }
int shard_yhi(const fdg_shard* s) { return s->core - 1 + (s->rank < s->world - 1 ? s->halo : 0); }

// Halo exchange of `rows` rows of a plane (core row 0 at p, row pitch pp)
// on the comm stream.  NCCL: grouped send/recv with rank -/+ 1.  Emulated
// group: device copies from the neighbours' planes of the same role (the
// group runs its strips in lockstep on one stream).
int shard_exchange(fdg_shard* s, int role, int rows, cudaStream_t st) {
    auto plane = [](fdg_shard* x, int r) -> float* { return r == 0 ? x->uA : r == 1 ? x->uB : r == 2 ? x->q : x->f; };
    // whole rows: a haloed plane's row starts fused_halo_left() columns
    // before column 0 (the replicated edge columns travel with the row)
    const int lo = (role == 0 || role == 1) && s->engine == SH_FUSED ? fused_halo_left() : 0;
    float* p = plane(s, role) - lo;
    const int pp = role == 2 || role == 3 ? s->pitch : s->upitch;
    const size_t n = (size_t)rows * pp;
    if (s->world == 1 || rows == 0) return FDG_OK;
    static const bool noexch = getenv("FDG_SHARD_NOEXCH") != nullptr;  // diagnostics (timing only)
    if (s->loopback && noexch) return FDG_OK;
    if (s->loopback) {  // timing mode: the same copies, from this strip's own edge rows
        if (s->rank > 0)
            CK(cudaMemcpyAsync(p - n, p, n * sizeof(float), cudaMemcpyDeviceToDevice, st));
        if (s->rank < s->world - 1)
            CK(cudaMemcpyAsync(p + (size_t)s->core * pp, p + (size_t)(s->core - rows) * pp, n * sizeof(float),
                               cudaMemcpyDeviceToDevice, st));
        return FDG_OK;
    }
    if (!s->group.empty()) {
        if (s->rank > 0) {
            fdg_shard* up = s->group[s->rank - 1];
            CK(cudaMemcpyAsync(p - n, plane(up, role) - lo + (size_t)(up->core - rows) * pp, n * sizeof(float),
                               cudaMemcpyDeviceToDevice, st));
        }
        if (s->rank < s->world - 1) {
            fdg_shard* dn = s->group[s->rank + 1];
            CK(cudaMemcpyAsync(p + (size_t)s->core * pp, plane(dn, role) - lo, n * sizeof(float),
                               cudaMemcpyDeviceToDevice, st));
        }
        return FDG_OK;
    }
    NcclApi& api = nccl_api();
    NK(api.group_start());
    if (s->rank > 0) {
        NK(api.send(p, n, NCCL_FLOAT32, s->rank - 1, s->comm, st));
        NK(api.recv(p - n, n, NCCL_FLOAT32, s->rank - 1, s->comm, st));
    }
    if (s->rank < s->world - 1) {
        NK(api.send(p + (size_t)(s->core - rows) * pp, n, NCCL_FLOAT32, s->rank + 1, s->comm, st));
        NK(api.recv(p + (size_t)s->core * pp, n, NCCL_FLOAT32, s->rank + 1, s->comm, st));
    }
    NK(api.group_end());
    return FDG_OK;
}

// one fused iteration k over output rows [y0, y1) (+ [y2, y3)); strips up to
// ~3000 rows run the plain strip x band grid (measured at 16384 columns: 2048-row
// strips 145 vs 150 us, 4096-row strips 266 vs 252 us with work-balanced segments)
int shard_fused(fdg_shard* s, int k, int y0, int y1, int y2, int y3, cudaStream_t st) {
    const float* src = k == 0 ? s->f : (k & 1 ? s->uA : s->uB);
    float* dst = k & 1 ? s->uB : s->uA;
    const int slot = std::min(k, s->ntrace - 1);
    cudaError_t r = launch_fused(src, s->f, dst, s->pitch, s->W, y0, y1, shard_ylo(s), shard_yhi(s), 1, 0,
                                 s->fwd->dev.scale, (float)s->cfg.epsilon_div, s->cfg.clamp_nonnegative,
                                 s->mc.p + slot, s->nf.p + slot, s->ts.p + 1 + slot, st, k > 0, 1, s->hp.pitch,
                                 s->hp.stride, y2, y3, s->world == 1 || s->core > 3000, s->fwd->dev.mx / 2,
                                 s->fwd->dev.my / 2);
    if (r != cudaSuccess) return cuda_err(r, "fused RL iteration launch (strip)");
    s->ctx->launches += 1;
    return FDG_OK;
}

// the two boundary bands of fused iteration k (kernels_band.cu)
int shard_fused_bands(fdg_shard* s, int k, cudaStream_t st) {
    const float* src = k == 0 ? s->f : (k & 1 ? s->uA : s->uB);
    float* dst = k & 1 ? s->uB : s->uA;
    const int slot = std::min(k, s->ntrace - 1);
    cudaError_t r = launch_band(src, k == 0 ? s->pitch : s->upitch, s->f, s->pitch, dst, s->upitch, s->W, 0, s->halo,
                                s->core - s->halo, s->core, shard_ylo(s), shard_yhi(s), s->fwd->dev.scale,
                                (float)s->cfg.epsilon_div, s->cfg.clamp_nonnegative, 1, fused_halo_left(),
                                fused_halo_right(), s->mc.p + slot, s->nf.p + slot, s->ts.p + 1 + slot, st);
    if (r != cudaSuccess) return cuda_err(r, "boundary band launch (strip)");
    s->ctx->launches += 1;
    return FDG_OK;
}

// one pass of the two-pass loop over output rows [y0, y1)
int shard_pass(fdg_shard* s, int which, int k, int y0, int y1, cudaStream_t st) {
    Geom g;
    g.pitch = s->pitch;
    g.W = s->W;
    g.y0 = y0;
    g.y1 = y1;
    g.ylo = shard_ylo(s);
    g.yhi = shard_yhi(s);
    Epi e;
    if (which == 1) {
        g.in = s->uA;
        g.out = s->q;
        e.mode = EPI_QUOT;
        e.aux = s->f;
        e.eps = (float)s->cfg.epsilon_div;
        return run_pass(s->ctx, s->fwd.get(), g, e, st);
    }
    const int slot = std::min(k, s->ntrace - 1);
    g.in = s->q;
    g.out = s->uA;
    e.mode = EPI_UPDATE;
    e.aux = s->uA;
    e.clamp = s->cfg.clamp_nonnegative;
    e.maxchange = s->mc.p + slot;
    e.nanflag = s->nf.p + slot;
    e.tend = s->ts.p + 1 + slot;
    return run_pass(s->ctx, s->adj.get(), g, e, st);
}

// Timing events per iteration: [6 k + 0/1] interior, [+2/3] bands, [+4/5] exchange
int shard_timing_events(fdg_shard* s, int iters) {
    static const bool off = getenv("FDG_SHARD_NOTIMING") != nullptr;
    if (off) return FDG_OK;
    const size_t need = (size_t)6 * std::max(iters, 1);
    while (s->tev.size() < need) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        s->tev.push_back(e);
    }
    s->t_iters = iters;
    return FDG_OK;
}

// Issue the loop of one strip.  phase: -1 = everything (own streams, NCCL);
// for an emulated group the runner calls phase 0 (exchange) of every strip,
// then phase 1 (compute) of every strip, per iteration, all on one stream.
int shard_iteration(fdg_shard* s, int k, int phase, cudaStream_t comp) {
    const bool split_ok = s->world > 1 && s->halo > 0 && s->core > 2 * s->halo;
    cudaEvent_t* te = s->tev.empty() ? nullptr : &s->tev[(size_t)6 * k];
    const bool emu = !s->group.empty();
    cudaStream_t comm = emu ? comp : s->comm_st;
    auto exchange = [&](int role, int rows) -> int {
        if (s->world == 1) return FDG_OK;
        if (!emu) CK(cudaStreamWaitEvent(comm, s->ev_ready, 0));
        if (te) CK(cudaEventRecord(te[4], comm));
        int r = shard_exchange(s, role, rows, comm);
        if (r) return r;
        if (te) CK(cudaEventRecord(te[5], comm));
        if (!emu) CK(cudaEventRecord(s->ev_halo, comm));
        return FDG_OK;
    };
    if (s->engine == SH_FUSED) {
        // iteration 0 reads f, whose halo rows were exchanged before the loop
        if (phase != 1 && k > 0) {
            int r = exchange(k & 1 ? 0 : 1, s->halo);  // the plane iteration k reads
            if (r) return r;
        }
        if (phase == 0) return FDG_OK;
        if (!split_ok) {
            if (!emu && s->world > 1 && k > 0) CK(cudaStreamWaitEvent(comp, s->ev_halo, 0));
            if (te) CK(cudaEventRecord(te[0], comp));
            int r = shard_fused(s, k, 0, s->core, 0, 0, comp);
            if (r) return r;
            if (te) {
                CK(cudaEventRecord(te[1], comp));
                CK(cudaEventRecord(te[2], comp));
                CK(cudaEventRecord(te[3], comp));
            }
        } else if (emu || !shard_bands_concurrent()) {
            if (te) CK(cudaEventRecord(te[0], comp));
            int r = shard_fused(s, k, s->halo, s->core - s->halo, 0, 0, comp);
            if (r) return r;
            if (te) CK(cudaEventRecord(te[1], comp));
            if (!emu && k > 0) CK(cudaStreamWaitEvent(comp, s->ev_halo, 0));
            if (te) CK(cudaEventRecord(te[2], comp));
            if ((r = shard_fused_bands(s, k, comp))) return r;
            if (te) CK(cudaEventRecord(te[3], comp));
        } else {
            // bands on the high-priority stream once the halo has landed
            // (iteration 0: f's halo, exchanged before the loop), running
            // next to the interior launch
            cudaStream_t bs = s->band_st;
            CK(cudaStreamWaitEvent(bs, k > 0 ? s->ev_halo : s->ev_ready, 0));
            if (te) CK(cudaEventRecord(te[2], bs));
            int r = shard_fused_bands(s, k, bs);
            if (r) return r;
            if (te) CK(cudaEventRecord(te[3], bs));
            CK(cudaEventRecord(s->ev_band, bs));
            if (te) CK(cudaEventRecord(te[0], comp));
            if ((r = shard_fused(s, k, s->halo, s->core - s->halo, 0, 0, comp))) return r;
            if (te) CK(cudaEventRecord(te[1], comp));
            CK(cudaStreamWaitEvent(comp, s->ev_band, 0));
        }
        if (!emu) CK(cudaEventRecord(s->ev_ready, comp));
        return FDG_OK;
    }
    // two passes, each: exchange its input's halo, interior, bands
    for (int which = 1; which <= 2; ++which) {
        if (phase == 0 || phase == -1) {
            // u's halo before pass 1 (iteration 0: filled with f's before the loop); q's before pass 2
            if (which == 2 || k > 0) {
                int r = exchange(which == 1 ? 0 : 2, s->halo);
                if (r) return r;
            }
        }
        if (phase == 0) {
            if (which == 1) return FDG_OK;  // the group runner computes pass 1 before exchanging q
            continue;
        }
        const bool waited = !emu && s->world > 1 && (which == 2 || k > 0);
        if (!split_ok) {
            if (waited) CK(cudaStreamWaitEvent(comp, s->ev_halo, 0));
            if (te && which == 1) CK(cudaEventRecord(te[0], comp));
            int r = shard_pass(s, which, k, 0, s->core, comp);
            if (r) return r;
            if (te && which == 2) {
                CK(cudaEventRecord(te[1], comp));
                CK(cudaEventRecord(te[2], comp));
                CK(cudaEventRecord(te[3], comp));
            }
        } else {
            if (te && which == 1) CK(cudaEventRecord(te[0], comp));
            int r = shard_pass(s, which, k, s->halo, s->core - s->halo, comp);
            if (r) return r;
            if (waited) CK(cudaStreamWaitEvent(comp, s->ev_halo, 0));
            if (te && which == 2) {
                CK(cudaEventRecord(te[1], comp));
                CK(cudaEventRecord(te[2], comp));
            }
            if ((r = shard_pass(s, which, k, 0, s->halo, comp))) return r;
            if ((r = shard_pass(s, which, k, s->core - s->halo, s->core, comp))) return r;
            if (te && which == 2) CK(cudaEventRecord(te[3], comp));
        }
        if (!emu) CK(cudaEventRecord(s->ev_ready, comp));
        if (phase == 1 && which == 1) return FDG_OK;  // group runner: q exchange next
    }
    return FDG_OK;
}

// the plane holding the result after `iters` iterations
const float* shard_result(const fdg_shard* s, int iters) {
    if (s->engine == SH_FUSED) return iters == 0 ? s->f : ((iters - 1) & 1 ? s->uB : s->uA);
    return s->uA;
}
int shard_result_pitch(const fdg_shard* s, int iters) {
    return s->engine == SH_FUSED && iters > 0 ? s->upitch : (s->engine == SH_FUSED ? s->pitch : s->upitch);
}

// load f's core rows, reset the trace slots, u0 = f (two-pass / rowres)
int shard_prologue(fdg_shard* s, const float* f, int pitch, int host, cudaStream_t st) {
    if (host) {
        if (pageable(f) && pitch == s->W) {  // staged through the context's pinned chunks
            int r = h2d(s->ctx->stg, s->f, s->pitch, f, s->W, s->core, st);
            if (r) return r;
        } else {
            CK(cudaMemcpy2DAsync(s->f, (size_t)s->pitch * 4, f, (size_t)pitch * 4, (size_t)s->W * 4, s->core,
                                 cudaMemcpyHostToDevice, st));
        }
    } else {
        CK(cudaMemcpy2DAsync(s->f, (size_t)s->pitch * 4, f, (size_t)pitch * 4, (size_t)s->W * 4, s->core,
                             cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaMemsetAsync(s->mc.p, 0, sizeof(unsigned) * s->ntrace, st));
    CK(cudaMemsetAsync(s->nf.p, 0, sizeof(int) * s->ntrace, st));
    CK(cudaMemsetAsync(s->ts.p, 0, sizeof(unsigned long long) * (s->ntrace + 1), st));
    CK(launch_stamp(s->ts.p, st));
    s->ctx->launches += 1;
    return FDG_OK;
}

int shard_copy_u0(fdg_shard* s, cudaStream_t st) {
    if (s->engine == SH_FUSED) return FDG_OK;
    const int rows = s->core + 2 * s->halo;
    CK(cudaMemcpyAsync(s->uA - (size_t)s->halo * s->pitch, s->f - (size_t)s->halo * s->pitch,
                       (size_t)rows * s->pitch * sizeof(float), cudaMemcpyDeviceToDevice, st));
    return FDG_OK;
}

int shard_epilogue(fdg_shard* s, float* u, int pitch, int host, int iters, cudaStream_t st) {
    const float* res = shard_result(s, iters);
    const int rp = shard_result_pitch(s, iters);
    if (host && pageable(u) && pitch == s->W && rp == s->pitch) return d2h(s->ctx->stg, u, res, rp, s->W, s->core, st);
    if (host && pageable(u) && pitch == s->W) {  // haloed plane: compact through f's plane first (f is no longer needed)
        CK(cudaMemcpy2DAsync(s->f, (size_t)s->pitch * 4, res, (size_t)rp * 4, (size_t)s->W * 4, s->core,
                             cudaMemcpyDeviceToDevice, st));
        return d2h(s->ctx->stg, u, s->f, s->pitch, s->W, s->core, st);
    }
    CK(cudaMemcpy2DAsync(u, (size_t)pitch * 4, res, (size_t)rp * 4, (size_t)s->W * 4, s->core,
                         host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st));
    return FDG_OK;
}

int shard_trace_out(fdg_shard* s, int iters, fdg_rl_record* trace, cudaStream_t st, bool reduce) {
    if (reduce && s->comm) {
        NcclApi& api = nccl_api();
        NK(api.all_reduce(s->mc.p, s->mc.p, (size_t)iters, NCCL_UINT32, NCCL_MAX, s->comm, st));
        NK(api.all_reduce(s->nf.p, s->nf.p, (size_t)iters, NCCL_UINT32, NCCL_MAX, s->comm, st));
    }
    std::vector<unsigned> hmc(iters);
    std::vector<int> hnf(iters);
    std::vector<unsigned long long> hts(iters + 1);
    CK(cudaMemcpyAsync(hmc.data(), s->mc.p, sizeof(unsigned) * iters, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hnf.data(), s->nf.p, sizeof(int) * iters, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hts.data(), s->ts.p, sizeof(unsigned long long) * (iters + 1), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const std::vector<double> sec = trace_seconds(hts, {}, iters);
    for (int k = 0; k < iters; ++k) {
        if (hnf[k])  // rl.hpp:96-99,173
            return set_err(FDG_ENAN, "rlDeconvolve: NaN in iterate at iteration " + std::to_string(k + 1));
        float m;
        std::memcpy(&m, &hmc[k], sizeof m);
        trace[k] = {k + 1, 0.0, (double)m, sec[k]};
    }
    return FDG_OK;
}

}  // namespace

int shard_set_loopback(int v) { return g_shard_loopback.exchange(v); }
int shard_set_bands(int v) { return g_shard_bands.exchange(v); }

extern "C" {

int fdg_comm_unique_id(unsigned char id[128]) {
    if (!id) return set_err(FDG_EINVAL, "null argument");
    NcclApi& api = nccl_api();
    if (!api.ok) return set_err(FDG_ECUDA, api.err);
    nccl_unique_id u;
    NK(api.get_unique_id(&u));
    std::memcpy(id, u.internal, 128);
    return FDG_OK;
}

int fdg_shard_create(fdg_ctx* ctx, const fdg_psf_desc* psf, const fdg_rl_config* cfg, int width, int height,
                     int rank, int world, const unsigned char* comm_id, fdg_shard** out) {
    if (!out) return set_err(FDG_EINVAL, "null argument");
    *out = nullptr;
    const bool loop = world > 1 && !comm_id && shard_loopback();
    if (world > 1 && !comm_id && !loop) return set_err(FDG_EINVAL, "sharded RL: world > 1 needs a communicator id");
    Entry en;
    int st = enter(ctx, en);
    if (st) return st;
    auto s = std::make_unique<fdg_shard>();
    if ((st = shard_init(s.get(), ctx, psf, cfg, width, height, rank, world))) return st;
    s->loopback = loop;
    // a communicator whenever an id is given (world 1 too: the trace
    // all-reduce then runs through NCCL on one GPU)
    if (comm_id && !loop) {
        NcclApi& api = nccl_api();
        if (!api.ok) return set_err(FDG_ECUDA, api.err);
        nccl_unique_id u;
        std::memcpy(u.internal, comm_id, 128);
        NK(api.comm_init_rank(&s->comm, world, u, rank));
    }
    *out = s.release();
    return FDG_OK;
}

int fdg_shard_group_create(fdg_ctx* ctx, const fdg_psf_desc* psf, const fdg_rl_config* cfg, int width, int height,
                           int world, fdg_shard** out) {
    if (!out) return set_err(FDG_EINVAL, "null argument");
    if (world < 1) return set_err(FDG_EINVAL, "sharded RL: bad rank / world");
    Entry en;
    int st = enter(ctx, en);
    if (st) return st;
    std::vector<std::unique_ptr<fdg_shard>> v;
    for (int r = 0; r < world; ++r) {
        v.push_back(std::make_unique<fdg_shard>());
        if ((st = shard_init(v.back().get(), ctx, psf, cfg, width, height, r, world))) return st;
    }
    std::vector<fdg_shard*> raw;
    for (auto& p : v) raw.push_back(p.get());
    for (int r = 0; r < world; ++r) {
        v[r]->group = raw;
        out[r] = v[r].release();
    }
    return FDG_OK;
}

void fdg_shard_destroy(fdg_shard* s) { delete s; }

int fdg_shard_info(const fdg_shard* s, long long info[6]) {
    if (!s || !info) return set_err(FDG_EINVAL, "null argument");
    const int ex = s->world == 1 || s->halo == 0 ? 0 : (s->engine == SH_FUSED ? 1 : 2);
    const int nb = (s->rank > 0) + (s->rank < s->world - 1);
    const long long row = (long long)(s->engine == SH_FUSED ? s->upitch : s->pitch) * 4;
    info[0] = s->r0;
    info[1] = s->core;
    info[2] = s->halo;
    info[3] = ex;
    info[4] = (long long)ex * nb * s->halo * row;
    info[5] = s->engine;
    return FDG_OK;
}

const char* fdg_shard_engine(const fdg_shard* s) {
    if (!s) return "?";
    return s->engine == SH_FUSED ? "fused" : s->engine == SH_ROWRES ? "rowres" : engine_name(s->fwd->dev.engine);
}

int fdg_shard_run(fdg_shard* s, const float* f, float* u, int pitch, int host, int iterations,
                  fdg_rl_record* trace) {
    if (!s || !f || !u) return set_err(FDG_EINVAL, "null argument");
    if (iterations < 0 || iterations > s->ntrace) return set_err(FDG_EINVAL, "sharded RL: iterations out of range");
    if (!s->group.empty()) return set_err(FDG_EINVAL, "sharded RL: use fdg_shard_group_run for a group");
    if (pitch < s->W) return set_err(FDG_EINVAL, "pitch must be >= width");
    Entry en;
    int st = enter(s->ctx, en);
    if (st) return st;
    cudaStream_t comp = s->ctx->stream;
    if ((st = shard_prologue(s, f, pitch, host, comp))) return st;
    if ((st = shard_timing_events(s, iterations))) return st;
    // f's halo rows (also u0's), then u0 = f
    CK(cudaEventRecord(s->ev_ready, comp));
    if (s->world > 1 && s->halo > 0) {
        CK(cudaStreamWaitEvent(s->comm_st, s->ev_ready, 0));
        if ((st = shard_exchange(s, 3, s->halo, s->comm_st))) return st;
        CK(cudaEventRecord(s->ev_halo, s->comm_st));
        CK(cudaStreamWaitEvent(comp, s->ev_halo, 0));
    }
    if ((st = shard_copy_u0(s, comp))) return st;
    if (s->engine == SH_ROWRES) {
        TraceSlots tr{s->mc.p, s->nf.p, s->ts.p, nullptr};
        if (iterations > 0 && (st = run_rowres(s->ctx, s->fwd.get(), s->f, s->uA, s->pitch, s->W, s->core, 1, 0,
                                               iterations, &s->cfg, tr, comp)))
            return st;
    } else {
        CK(cudaEventRecord(s->ev_ready, comp));
        for (int k = 0; k < iterations; ++k)
            if ((st = shard_iteration(s, k, -1, comp))) return st;
    }
    // the comm stream's last work joins the caller's stream
    CK(cudaEventRecord(s->ev_join, s->comm_st));
    CK(cudaStreamWaitEvent(comp, s->ev_join, 0));
    if ((st = shard_epilogue(s, u, pitch, host, iterations, comp))) return st;
    if (trace && iterations > 0) return shard_trace_out(s, iterations, trace, comp, true);
    if (host) CK(cudaStreamSynchronize(comp));
    return FDG_OK;
}

int fdg_shard_group_run(fdg_shard** group, int world, const float* f, float* u, int pitch, int host, int iterations,
                        fdg_rl_record* trace) {
    if (!group || world < 1 || !f || !u) return set_err(FDG_EINVAL, "null argument");
    for (int r = 0; r < world; ++r)
        if (!group[r] || (int)group[r]->group.size() != world || group[r]->group[r] != group[r])
            return set_err(FDG_EINVAL, "sharded RL: not a shard group");
    fdg_shard* s0 = group[0];
    if (iterations < 0 || iterations > s0->ntrace) return set_err(FDG_EINVAL, "sharded RL: iterations out of range");
    if (pitch < s0->W) return set_err(FDG_EINVAL, "pitch must be >= width");
    Entry en;
    int st = enter(s0->ctx, en);
    if (st) return st;
    cudaStream_t comp = s0->ctx->stream;
    for (fdg_shard* s : std::vector<fdg_shard*>(group, group + world)) {
        if ((st = shard_prologue(s, f + (size_t)s->r0 * pitch, pitch, host, comp))) return st;
        if ((st = shard_timing_events(s, iterations))) return st;
    }
    for (int r = 0; r < world; ++r)
        if ((st = shard_exchange(group[r], 3, group[r]->halo, comp))) return st;
    for (int r = 0; r < world; ++r)
        if ((st = shard_copy_u0(group[r], comp))) return st;
    for (int k = 0; k < iterations; ++k) {
        if (s0->engine == SH_ROWRES) break;
        for (int r = 0; r < world; ++r)
            if ((st = shard_iteration(group[r], k, 0, comp))) return st;
        for (int r = 0; r < world; ++r)
            if ((st = shard_iteration(group[r], k, 1, comp))) return st;
        if (s0->engine == SH_TWOPASS) {  // q exchange, then pass 2 of every strip
            for (int r = 0; r < world; ++r)
                if ((st = shard_exchange(group[r], 2, group[r]->halo, comp))) return st;
            for (int r = 0; r < world; ++r) {
                fdg_shard* s = group[r];
                const bool split_ok = s->world > 1 && s->halo > 0 && s->core > 2 * s->halo;
                if (!split_ok) {
                    if ((st = shard_pass(s, 2, k, 0, s->core, comp))) return st;
                } else {
                    if ((st = shard_pass(s, 2, k, s->halo, s->core - s->halo, comp))) return st;
                    if ((st = shard_pass(s, 2, k, 0, s->halo, comp))) return st;
                    if ((st = shard_pass(s, 2, k, s->core - s->halo, s->core, comp))) return st;
                }
            }
        }
    }
    if (s0->engine == SH_ROWRES) {
        for (int r = 0; r < world; ++r) {
            fdg_shard* s = group[r];
            TraceSlots tr{s->mc.p, s->nf.p, s->ts.p, nullptr};
            if (iterations > 0 && (st = run_rowres(s->ctx, s->fwd.get(), s->f, s->uA, s->pitch, s->W, s->core, 1, 0,
                                                   iterations, &s->cfg, tr, comp)))
                return st;
        }
    }
    for (int r = 0; r < world; ++r) {
        fdg_shard* s = group[r];
        if ((st = shard_epilogue(s, u + (size_t)s->r0 * pitch, pitch, host, iterations, comp))) return st;
    }
    if (trace && iterations > 0) {
        std::vector<fdg_rl_record> tmp(iterations);
        for (int r = 0; r < world; ++r) {
            if ((st = shard_trace_out(group[r], iterations, tmp.data(), comp, false))) return st;
            for (int k = 0; k < iterations; ++k) {
                if (r == 0)
                    trace[k] = tmp[k];
                else
                    trace[k].max_abs_change = std::max(trace[k].max_abs_change, tmp[k].max_abs_change);
            }
        }
    }
    if (host) CK(cudaStreamSynchronize(comp));
    return FDG_OK;
}

int fdg_shard_timing(fdg_shard* s, double ms[3]) {
    if (!s || !ms) return set_err(FDG_EINVAL, "null argument");
    Entry en;
    int st = enter(s->ctx, en);
    if (st) return st;
    ms[0] = ms[1] = ms[2] = 0.0;
    if (s->tev.empty()) return FDG_OK;
    CK(cudaStreamSynchronize(s->ctx->stream));
    CK(cudaStreamSynchronize(s->comm_st));
    const bool fused = s->engine == SH_FUSED;
    for (int k = 0; k < s->t_iters; ++k) {
        cudaEvent_t* te = &s->tev[(size_t)6 * k];
        float a = 0.f;
        if (cudaEventElapsedTime(&a, te[0], te[1]) == cudaSuccess) ms[0] += a;
        if (cudaEventElapsedTime(&a, te[2], te[3]) == cudaSuccess) ms[1] += a;
        if ((fused ? k > 0 : true) && s->world > 1 && s->halo > 0 &&
            cudaEventElapsedTime(&a, te[4], te[5]) == cudaSuccess)
            ms[2] += a;
    }
    cudaGetLastError();  // events never recorded in this run (e.g. k = 0 exchange)
    return FDG_OK;
}

}  // extern "C"
