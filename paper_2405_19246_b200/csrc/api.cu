// api.cu -- the C ABI declared in include/mmot.h: argument validation, context workspace,
// and the device-resident Sinkhorn driver (Algorithm 4).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <vector>

#include "../../include/mmot.h"
#include "internal.h"

using mmot::Plan;

namespace {

struct ncclUniqueIdBytes {
    char internal[128];
};

struct DevScalars {
    int stop;
    int status;
    int fail_iter;
    int iters_done;
    int converged;
    int guard;          // single-walk precision guard tripped (k_sw_guard)
    int sweep;          // completed sweeps of the current solve (device counter)
    int g_done, g_n;    // device-resident loop: periods done / to do
    int flags[2 * mmot::kStMaxL];
    double resid;
    double res_acc;
    double W;
    double mass[mmot::kStMaxL];
};

char g_err[256] = "";

// ---------------------------------------------------------------------------------------
// NCCL, resolved at run time from the libnccl.so.2 already loaded in the process (PyTorch's)
// or the system one, so the library never pins an NCCL version at link time.
typedef int nccl_result;
typedef void *nccl_comm;
struct NcclApi {
    bool tried = false, ok = false;
    nccl_result (*GetUniqueId)(void *);
    nccl_result (*CommInitRank)(nccl_comm *, int, ncclUniqueIdBytes, int);
    nccl_result (*CommDestroy)(nccl_comm);
    nccl_result (*AllGather)(const void *, void *, size_t, int, nccl_comm, cudaStream_t);
    nccl_result (*AllReduce)(const void *, void *, size_t, int, int, nccl_comm, cudaStream_t);
    const char *(*GetErrorString)(nccl_result);
};
NcclApi g_nccl;
constexpr int kNcclInt32 = 2, kNcclFloat64 = 8, kNcclSum = 0, kNcclMax = 2;

bool nccl_load() {
    if (g_nccl.tried) return g_nccl.ok;
    g_nccl.tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    g_nccl.GetUniqueId = (nccl_result(*)(void *))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (nccl_result(*)(nccl_comm *, int, ncclUniqueIdBytes, int))dlsym(h, "ncclCommInitRank");
    g_nccl.CommDestroy = (nccl_result(*)(nccl_comm))dlsym(h, "ncclCommDestroy");
    g_nccl.AllGather = (nccl_result(*)(const void *, void *, size_t, int, nccl_comm, cudaStream_t))dlsym(h, "ncclAllGather");
    g_nccl.AllReduce = (nccl_result(*)(const void *, void *, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclAllReduce");
    g_nccl.GetErrorString = (const char *(*)(nccl_result))dlsym(h, "ncclGetErrorString");
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.AllGather && g_nccl.AllReduce &&
                g_nccl.GetErrorString;
    return g_nccl.ok;
}

}  // namespace

// In-process group of `world` sharded contexts on one device (virtual shards, mmot_vgroup_create):
// each context is driven by its own host thread on its own stream; a collective is a host barrier
// plus cross-stream event waits and device copies -- no kernel ever waits on another.
struct mmot_vgroup {
    int world = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    int64_t gen = 0;
    std::vector<const void *> src;
    std::vector<cudaEvent_t> ready, done;
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const int64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct mmot_ctx {
    int l = 0;
    int64_t N = 0;
    double eta = 0, h = 0;
    mmot_grid grid{0, 1};
    mmot_dtype dt = MMOT_F64;
    mmot_opts opts{0, 0, MMOT_LOG, 0, MMOT_KERNEL_AUTO};
    bool sw = false;
    void *car_bi = nullptr;
    cudaStream_t stream = nullptr;
    int device = 0;
    mmot::Weights W{};
    int64_t P = 0, nchunks = 0;
    int nlev = 0;
    int64_t nlev_n[mmot::kMaxLevels] = {0};
    void *ws = nullptr;
    void *ops_f[mmot::kMaxLevels] = {nullptr}, *ops_b[mmot::kMaxLevels] = {nullptr};
    void *car_f[mmot::kMaxLevels] = {nullptr}, *car_b[mmot::kMaxLevels] = {nullptr};
    double *partial = nullptr;
    DevScalars *dsc = nullptr;
    DevScalars *hsc = nullptr;  // pinned host mirror
    double *lin[mmot::kMaxL] = {nullptr};  // internal linear scalings (MMOT_LOG repr, or any repr when sw)
    int64_t nchp = 0;                       // sw: chains rounded up to 32 (transposed row length)
    double *mu_t[mmot::kMaxL] = {nullptr};  // sw: marginals in the chain-transposed layout
    double *out_t = nullptr;                // sw: marginal output in the chain-transposed layout
    void *sw_end = nullptr;                 // sw: walked end state per chain ([nchunks][M] Dual-sized; guard)
    mmot_ctx *fb = nullptr;                 // sw: two-walk context the guard falls back to (lazy)
    int64_t fallbacks = 0;                  // sw: calls redone on the two-walk family
    // restricted next-update scan (single-walk contexts): second carry buffer + affine elements
    bool rx = false;
    void *rx_mem = nullptr;
    void *carB_f = nullptr, *carB_bi = nullptr;
    void *rxe_f[mmot::kMaxLevels] = {nullptr}, *rxe_b[mmot::kMaxLevels] = {nullptr};
    void *rcar_f[mmot::kMaxLevels] = {nullptr}, *rcar_b[mmot::kMaxLevels] = {nullptr};
    // sharded contexts (mmot_create_sharded)
    bool sharded = false;
    int rank = 0, world = 1;
    int64_t N_global = 0, lo = 0;
    nccl_comm comm = nullptr;
    mmot_vgroup *vg = nullptr;              // virtual shards: in-process group instead of NCCL
    double *vg_tmp = nullptr;               // virtual shards: reduction result staging
    double *shard_mem = nullptr;            // agg_send [2*SZ], agg_all [world*2*SZ], rank_car [2*M] (Dual-sized)
    int exch_error = 0;
    // stabilised family (MMOT_KERNEL_STABLE, stable.cu): log-domain, one warp per instance
    bool stable = false;
    mmot::SPlan sp{};
    double *st_mem = nullptr;               // eta, g planes, scratch, wout, resid
    int *st_int = nullptr;                  // status, fail_iter, iters_done, converged, sel  ([5][batch])
    int *st_shost = nullptr;                // pinned [4][batch]
    double *st_rhost = nullptr, *st_whost = nullptr;  // pinned [batch]
    std::vector<double> eta_host;           // per-instance eta (fallback creation)
    mmot_ctx *st_fb = nullptr;              // stabilised context the plain families fall back to (lazy)
    int64_t st_fallbacks = 0;               // calls redone on the stabilised family
    double *u_save = nullptr;               // two-walk LINEAR solves: initial u (for the fallback)
    // l = 6 lane-state family (lanes.cu)
    mmot::LsWork ls{};
    double *ls_mem = nullptr;
    bool ls_on = false;
    // NEXT-1: all-marginals residual pass (MODE_ALLRES) -- its own chain layout and scan workspace
    // for the DP over all l scalings (2^l states)
    int all_state = 0;                      // 0 untried, 1 ready, -1 unavailable
    void *all_mem = nullptr;
    int64_t all_P = 0, all_nchunks = 0;
    int all_nlev = 0;
    int64_t all_nlev_n[mmot::kMaxLevels] = {0};
    void *all_ops_f[mmot::kMaxLevels] = {nullptr}, *all_ops_b[mmot::kMaxLevels] = {nullptr};
    void *all_car_f[mmot::kMaxLevels] = {nullptr}, *all_car_b[mmot::kMaxLevels] = {nullptr};
    void *all_car_bi = nullptr;
    double *all_partial = nullptr;
    int64_t allres_checks = 0;
    // 2-D grids (mmot_create_2d, grid2d.cu): l = 3 on an N1 x N2 mesh, vectors column-major
    bool g2 = false;
    int64_t g2N = 0, g2M = 0;               // rows (inner), columns (outer)
    double g2h1 = 0, g2h2 = 0;              // spacings
    double *g2_mem = nullptr;               // Fa, Fb, Ga, Gb [4][N1 N2] + transposed scalings [3][N1 N2]
    void *g2_T = nullptr;                   // Y, st, Gab (Dual-sized)
    // batched contexts (mmot_create_batched)
    bool batched = false;
    int64_t batch = 1;
    mmot::BatchArgs ba{};
    double *bat_mem = nullptr;              // eta, phit, scratch, wout (one allocation)
    // pair family (pair.cu): large batches, tol <= 0 -- its own layout, allocated on first use
    mmot::PairPlan pp{};
    void *pair_mem = nullptr;
    int pair_state = 0;                     // 0 unknown, 1 available, -1 not for this context
    int64_t pair_solves = 0;
    int64_t pair_f32_solves = 0;            // of which in fp32 arithmetic
    int64_t pair_redo = 0;                  // fp32 pair instances redone in fp64 (states left the fp32 range)
    // CTA family (cta.cu): small instances, a thread block each
    mmot::CtaPlan cp{};
    double *cta_mem = nullptr;
    int cta_state = 0;
    int64_t cta_solves = 0;
    double *pts_mem = nullptr;              // non-uniform grids: hx [ne], lambda [batch][ne]
    double *f32_mem = nullptr;              // MMOT_F32 I/O: widened marginals [l][n] + output [n] (lazy)
    float *f32_stage = nullptr;             // MMOT_F32 host calls: float staging [l][n] (lazy)
    const double *pts_lam = nullptr;        // non-uniform grid, two-walk contexts: per-edge decays
    const double *pts_hx = nullptr;         // ... and edge lengths
    int *bat_int = nullptr;                 // E, status, fail_iter
    void **bat_ptrs = nullptr;              // device array of l pointers (u[] for import/export)
    double *bat_whost = nullptr;            // pinned [batch]
    int *bat_shost = nullptr;               // pinned [4*batch]: status, fail_iter, iters_done, converged
    double *bat_rhost = nullptr;            // pinned [batch]: last residual
    double *stage_mu[mmot::kStMaxL] = {nullptr};
    double *stage_u[mmot::kStMaxL] = {nullptr};
    int *hstop = nullptr;       // pinned, async stop polling (hstop[1]: loop period count for the graph)
    cudaEvent_t poll_ev = nullptr;
    // device-resident Sinkhorn loop: cached graph (a WHILE node whose body is `period` sweeps)
    cudaGraphExec_t g_exec = nullptr;
    cudaGraph_t g_graph = nullptr;
    const void *g_key[2 * mmot::kMaxL + 4] = {nullptr};
    int64_t g_launches = 0;     // kernels per graph period (launch accounting)
    int64_t g_allres = 0;       // all-marginals residual checks per graph period
    int64_t graph_solves = 0;
    bool graph_broken = false;  // capture failed once: host loop from then on
    cudaStream_t cap_stream = nullptr;  // private stream the loop graph is captured on
    int64_t launches = 0;
    char err[256] = "";
    // profiling (mmot_profile_enable)
    bool prof = false;
    std::vector<cudaEvent_t> pool;
    std::vector<int> pool_mode;
    size_t used = 0;
};

static cudaEvent_t *prof_events(mmot_ctx *c, int mode) {
    if (!c->prof) return nullptr;
    if (c->used + 4 > c->pool.size()) {
        for (int i = 0; i < 4; ++i) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
            c->pool.push_back(e);
        }
    }
    cudaEvent_t *ev = &c->pool[c->used];
    c->pool_mode.push_back(mode);
    c->used += 4;
    return ev;
}

static void set_err(mmot_ctx *c, const char *fmt, ...) {
    char buf[256];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) snprintf(c->err, sizeof c->err, "%s", buf);
    snprintf(g_err, sizeof g_err, "%s", buf);
}

#define CK(ctx, call)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            set_err(ctx, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
            return e_ == cudaErrorMemoryAllocation ? MMOT_ENOMEM : MMOT_ECUDA;          \
        }                                                                               \
    } while (0)

extern "C" {

const char *mmot_strerror(mmot_status s) {
    switch (s) {
        case MMOT_OK: return "ok";
        case MMOT_EINVAL: return "invalid argument";
        case MMOT_ESHAPE: return "shape / pointer layout mismatch";
        case MMOT_ENONFINITE: return "non-finite input";
        case MMOT_ENEGMASS: return "negative mass in a marginal";
        case MMOT_EZEROMASS: return "marginal with zero total mass";
        case MMOT_EOVERFLOW: return "tensor-vector product left the representable range";
        case MMOT_ECUDA: return "CUDA error";
        case MMOT_ENCCL: return "NCCL error";
        case MMOT_ENOMEM: return "device allocation failed";
        case MMOT_EUNSUPPORTED: return "unsupported in this build";
        case MMOT_EPRECISION: return "single-walk precision guard tripped";
    }
    return "unknown status";
}

const char *mmot_last_error(const mmot_ctx *ctx) { return ctx ? ctx->err : g_err; }

int mmot_version(void) { return (MMOT_VERSION_MAJOR << 16) | MMOT_VERSION_MINOR; }

int64_t mmot_launch_count(const mmot_ctx *ctx) { return ctx ? ctx->launches + (ctx->fb ? ctx->fb->launches : 0) : 0; }

int64_t mmot_fallback_count(const mmot_ctx *ctx) { return ctx ? ctx->fallbacks : 0; }

int64_t mmot_allres_checks(const mmot_ctx *ctx) { return ctx ? ctx->allres_checks : 0; }

int64_t mmot_stable_fallback_count(const mmot_ctx *ctx) {
    return ctx ? ctx->st_fallbacks + (ctx->fb ? ctx->fb->st_fallbacks : 0) : 0;
}

int64_t mmot_graph_solves(const mmot_ctx *ctx) { return ctx ? ctx->graph_solves + (ctx->fb ? ctx->fb->graph_solves : 0) : 0; }
int64_t mmot_pair_solves(const mmot_ctx *ctx) { return ctx ? ctx->pair_solves : 0; }
int64_t mmot_pair_f32_solves(const mmot_ctx *ctx) { return ctx ? ctx->pair_f32_solves : 0; }
int64_t mmot_pair_redo_count(const mmot_ctx *ctx) { return ctx ? ctx->pair_redo : 0; }
int64_t mmot_cta_solves(const mmot_ctx *ctx) { return ctx ? ctx->cta_solves : 0; }

mmot_status mmot_info(const mmot_ctx *ctx, int64_t *chain_len, int64_t *nchains, int *kernel) {
    if (!ctx) { set_err(nullptr, "NULL context"); return MMOT_EINVAL; }
    if (chain_len) *chain_len = ctx->g2 ? ctx->g2N : ctx->stable ? ctx->N : ctx->batched ? ctx->ba.P : ctx->P;
    if (nchains) *nchains = ctx->g2 ? ctx->g2M : ctx->stable ? ctx->batch : ctx->batched ? 32 * ctx->batch : ctx->nchunks;
    if (kernel) *kernel = ctx->g2 ? 5 : ctx->ls_on ? 6 : ctx->stable ? MMOT_KERNEL_STABLE
                          : ctx->batched ? MMOT_KERNEL_PERSISTENT : (ctx->sw ? MMOT_KERNEL_SINGLE_WALK : MMOT_KERNEL_TWO_WALK);
    return MMOT_OK;
}

void mmot_destroy(mmot_ctx *ctx) {
    if (!ctx) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    else cudaDeviceSynchronize();
    mmot_destroy(ctx->fb);
    mmot_destroy(ctx->st_fb);
    cudaFree(ctx->st_mem);
    cudaFree(ctx->all_mem);
    cudaFree(ctx->ls_mem);
    cudaFree(ctx->g2_mem);
    cudaFree(ctx->g2_T);
    cudaFree(ctx->st_int);
    cudaFree(ctx->u_save);
    if (ctx->st_shost) cudaFreeHost(ctx->st_shost);
    if (ctx->st_rhost) cudaFreeHost(ctx->st_rhost);
    if (ctx->st_whost) cudaFreeHost(ctx->st_whost);
    cudaFree(ctx->ws);
    cudaFree(ctx->out_t);
    cudaFree(ctx->sw_end);
    cudaFree(ctx->bat_mem);
    cudaFree(ctx->pair_mem);
    cudaFree(ctx->cta_mem);
    cudaFree(ctx->pts_mem);
    cudaFree(ctx->f32_mem);
    cudaFree(ctx->f32_stage);
    cudaFree(ctx->rx_mem);
    cudaFree(ctx->shard_mem);
    cudaFree(ctx->vg_tmp);
    if (ctx->comm && g_nccl.ok) g_nccl.CommDestroy(ctx->comm);
    cudaFree(ctx->bat_int);
    cudaFree(ctx->bat_ptrs);
    if (ctx->bat_whost) cudaFreeHost(ctx->bat_whost);
    if (ctx->bat_shost) cudaFreeHost(ctx->bat_shost);
    if (ctx->bat_rhost) cudaFreeHost(ctx->bat_rhost);
    for (int q = 0; q < mmot::kMaxL; ++q) {
        cudaFree(ctx->lin[q]);
        cudaFree(ctx->mu_t[q]);
    }
    for (int q = 0; q < mmot::kStMaxL; ++q) {
        cudaFree(ctx->stage_mu[q]);
        cudaFree(ctx->stage_u[q]);
    }
    if (ctx->hsc) cudaFreeHost(ctx->hsc);
    if (ctx->hstop) cudaFreeHost(ctx->hstop);
    if (ctx->poll_ev) cudaEventDestroy(ctx->poll_ev);
    if (ctx->g_exec) cudaGraphExecDestroy(ctx->g_exec);
    if (ctx->g_graph) cudaGraphDestroy(ctx->g_graph);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    for (cudaEvent_t e : ctx->pool) cudaEventDestroy(e);
    cudaSetDevice(cur);
    delete ctx;
}

static mmot_status create_single(int l, int64_t N, double eta, mmot_grid grid, mmot_dtype dt, const mmot_opts *opts,
                                 void *cuda_stream, mmot_ctx **out, bool allow_persistent, bool exact_chains = false);
static mmot_status create_stable(int l, int64_t N, int64_t batch, const double *eta_host, mmot_grid grid, mmot_dtype dt,
                                 const mmot_opts *opts, void *cuda_stream, mmot_ctx **out);

mmot_status mmot_create(int l, int64_t N, double eta, mmot_grid grid, mmot_dtype dt, const mmot_opts *opts,
                        void *cuda_stream, mmot_ctx **out) {
    return create_single(l, N, eta, grid, dt, opts, cuda_stream, out, true);
}

// Single-walk chain length dividing N exactly (shards with a successor: padded points would add
// spurious edge weights to the carries leaving the shard): the multiple of the slab length in
// [lo, hi] closest to `want` that divides N, or 0 if there is none.
static int64_t exact_chain_len(int64_t N, int64_t want, int64_t lo, int64_t hi, int64_t slab) {
    int64_t best = 0;
    for (int64_t P = std::max<int64_t>(slab, lo / slab * slab); P <= hi; P += slab)
        if (N % P == 0 && (best == 0 || llabs(P - want) < llabs(best - want))) best = P;
    return best;
}

// allow_persistent = false (shards of a sharded context): the persistent batched kernel has no
// cross-rank exchange, so a shard always gets a scan-based kernel family.  exact_chains = true
// (shards with a successor): single-walk chains must tile the shard exactly (exact_chain_len).
static mmot_status create_single(int l, int64_t N, double eta, mmot_grid grid, mmot_dtype dt, const mmot_opts *opts,
                                 void *cuda_stream, mmot_ctx **out, bool allow_persistent, bool exact_chains) {
    if (!out) { set_err(nullptr, "out is NULL"); return MMOT_EINVAL; }
    *out = nullptr;
    if (l < 2 || l > 8) { set_err(nullptr, "l=%d outside [2,8]", l); return MMOT_EINVAL; }
    if (N < 1) { set_err(nullptr, "N=%lld < 1", (long long)N); return MMOT_EINVAL; }
    if (!(eta > 0) || !isfinite(eta)) { set_err(nullptr, "eta must be finite and > 0"); return MMOT_EINVAL; }
    if (!isfinite(grid.x_min) || !isfinite(grid.x_max) || (N > 1 && !(grid.x_max > grid.x_min))) {
        set_err(nullptr, "grid must satisfy x_max > x_min");
        return MMOT_EINVAL;
    }
    if (dt != MMOT_F64 && dt != MMOT_F32) { set_err(nullptr, "bad dtype"); return MMOT_EINVAL; }
    if (opts && (opts->check_every < 0 || opts->chunk < 0 || (opts->repr != MMOT_LOG && opts->repr != MMOT_LINEAR) ||
                 opts->kernel < MMOT_KERNEL_AUTO || opts->kernel > MMOT_KERNEL_STABLE)) {
        set_err(nullptr, "bad opts");
        return MMOT_EINVAL;
    }
    if (l > MMOT_MAX_L) { set_err(nullptr, "l=%d > MMOT_MAX_L=%d in this build", l, MMOT_MAX_L); return MMOT_EUNSUPPORTED; }
    if (l > mmot::kMaxL) {
        // l = 7, 8 (2^(l-1) = 64 / 128 subset states): the stabilised family only (stable.cu)
        const int kreq = opts ? opts->kernel : MMOT_KERNEL_AUTO;
        if (!allow_persistent || dt != MMOT_F64 || (kreq != MMOT_KERNEL_AUTO && kreq != MMOT_KERNEL_STABLE)) {
            set_err(nullptr, "l=%d > %d runs on the stabilised family only (MMOT_F64, MMOT_KERNEL_AUTO or _STABLE, not sharded)", l, mmot::kMaxL);
            return MMOT_EUNSUPPORTED;
        }
        return create_stable(l, N, 1, &eta, grid, dt, opts, cuda_stream, out);
    }
    // small instances: the persistent batched kernel with one instance (all sweeps in one launch,
    // no per-update kernel latency)
    const int kern = opts ? opts->kernel : MMOT_KERNEL_AUTO;
    const int chunk = opts ? opts->chunk : 0;
    if (kern == MMOT_KERNEL_STABLE) {
        if (!allow_persistent) { set_err(nullptr, "sharded contexts cannot use the stabilised family"); return MMOT_EUNSUPPORTED; }
        return create_stable(l, N, 1, &eta, grid, dt, opts, cuda_stream, out);
    }
    if (kern == MMOT_KERNEL_PERSISTENT && !allow_persistent) {
        set_err(nullptr, "sharded contexts cannot use the persistent kernel");
        return MMOT_EUNSUPPORTED;
    }
    if (kern == MMOT_KERNEL_PERSISTENT || (allow_persistent && kern == MMOT_KERNEL_AUTO && chunk == 0 && l <= 5 &&
                                           N <= 4096 && getenv("MMOT_NO_PERSISTENT") == nullptr)) {
        if (l > 5) { set_err(nullptr, "the persistent kernel supports l <= 5"); return MMOT_EUNSUPPORTED; }
        return mmot_create_batched(l, N, 1, &eta, grid, dt, opts, cuda_stream, out);
    }

    mmot_ctx *c = new mmot_ctx();
    c->l = l;
    c->N = N;
    c->eta = eta;
    c->grid = grid;
    c->dt = dt;
    if (opts) c->opts = *opts;
    c->stream = static_cast<cudaStream_t>(cuda_stream);
    cudaGetDevice(&c->device);
    c->h = N > 1 ? (grid.x_max - grid.x_min) / (double)(N - 1) : 1.0;
    // w_a = lambda^{a(l-a)} = exp(-a(l-a) h/eta) in fp64 (A15)
    for (int a = 0; a <= mmot::kMaxL; ++a) {
        const int e = a <= l ? a * (l - a) : 0;
        c->W.e[a] = (double)e;
        c->W.w[a] = a <= l ? exp(-(double)e * c->h / eta) : 0.0;
    }
    const int NB = l - 1;
    const int64_t pmax = mmot::chunk_max(NB);
    const int q = mmot::sub_q(NB);
    // Single-walk kernels (k_sw_apply): the suffix states are walked forward through the
    // inverse step, whose error growth over a chain is bounded by (1/w_min)^P =
    // exp(P * emax * h/eta), emax = max_a a(l-a).  Auto-selected when a chain of >= 64 points
    // keeps that exponent <= kSwBound.
    const double emax = (double)((l / 2) * ((l + 1) / 2));
    const double hoe = c->h / eta;
    const int slab = mmot::kSwSlab;
    int64_t P;
    bool sw = false;
    if (c->opts.kernel == MMOT_KERNEL_SINGLE_WALK) {
        sw = NB <= 4;
        if (!sw) { set_err(nullptr, "single-walk kernels support l <= 5"); delete c; return MMOT_EUNSUPPORTED; }
    }
    if (c->opts.chunk > 0) {
        P = sw ? ((int64_t)c->opts.chunk + mmot::kSwSlab - 1) / mmot::kSwSlab * mmot::kSwSlab
               : std::min<int64_t>(c->opts.chunk, pmax);
        if (sw && exact_chains && N % P != 0) {
            P = exact_chain_len(N, P, slab, std::max<int64_t>(4 * P, 1024), slab);
            if (P == 0) {
                set_err(nullptr, "single-walk shard: no chain length (multiple of %d) divides the shard size %lld",
                        slab, (long long)N);
                delete c;
                return MMOT_EUNSUPPORTED;
            }
        }
    } else {
        // one chain per lane, 2 waves of (SMs x resident warps x 32 lanes)
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
        const int64_t target = (NB <= 4 ? (int64_t)nsm * mmot::sw_blocks_per_sm(NB) * mmot::kWarpsPerCtaHost * 32 * 2
                                        : (int64_t)nsm * 8 * 32 * 2);
        int64_t Psw = (N + target - 1) / target;
        Psw = std::max<int64_t>(64, ((Psw + slab - 1) / slab) * slab);
        const double capd = mmot::kSwBound / (emax * hoe);
        const int64_t Pcap = capd > 1e15 ? (int64_t)1e15 : (int64_t)capd;
        if (Psw > Pcap) Psw = (Pcap / slab) * slab;
        if (c->opts.kernel == MMOT_KERNEL_AUTO && NB <= 4 && Psw >= 64 && N >= 64LL * 148 * 8 * 32) sw = true;
        if ((sw || c->opts.kernel == MMOT_KERNEL_SINGLE_WALK) && exact_chains && N % Psw != 0) {
            const int64_t Pe = exact_chain_len(N, Psw, 64, std::min<int64_t>(Pcap, 2 * Psw + 64), slab);
            if (Pe > 0) Psw = Pe;
            else if (c->opts.kernel == MMOT_KERNEL_AUTO) sw = false;
            else {
                set_err(nullptr, "single-walk shard: no chain length (multiple of %d) divides the shard size %lld",
                        slab, (long long)N);
                delete c;
                return MMOT_EUNSUPPORTED;
            }
        }
        if (sw) {
            P = std::max<int64_t>(slab, Psw);
        } else {
            const int64_t target2 = 148 * 256;
            P = (N + target2 - 1) / target2;
            if (NB >= 4) P = pmax;  // heavy operators: as few chains as the checkpoint store allows
            P = ((P + q - 1) / q) * q;
            P = std::max<int64_t>(q, std::min<int64_t>(P, pmax));
        }
    }
    c->sw = sw;
    c->P = P;
    c->nchunks = (N + P - 1) / P;
    // levels of the hierarchical operator scan
    int64_t n = c->nchunks;
    c->nlev = 0;
    const int grp = mmot::group_of(NB);
    while (true) {
        c->nlev_n[c->nlev++] = n;
        if (n <= grp || c->nlev == mmot::kMaxLevels) break;
        n = (n + grp - 1) / grp;
    }
    // workspace, sized for dual numbers (the cost) so every mode fits
    const int M = 1 << NB;
    const size_t opsz = (size_t)(NB + 1) * M * sizeof(mmot::Dual);
    const size_t carsz = (size_t)M * sizeof(mmot::Dual);
    size_t total = 0;
    size_t off_ops[mmot::kMaxLevels], off_car[mmot::kMaxLevels];
    for (int i = 0; i < c->nlev; ++i) {
        off_ops[i] = total;
        total += 2 * (size_t)c->nlev_n[i] * opsz;
        total = (total + 255) & ~(size_t)255;
        off_car[i] = total;
        total += 2 * (size_t)c->nlev_n[i] * carsz;
        total = (total + 255) & ~(size_t)255;
    }
    const size_t off_bi = total;
    total += (size_t)c->nchunks * carsz;
    total = (total + 255) & ~(size_t)255;
    const size_t off_part = total;
    total += (size_t)c->nchunks * sizeof(double);
    total = (total + 255) & ~(size_t)255;
    const size_t off_sc = total;
    total += sizeof(DevScalars);
    cudaError_t e = cudaMalloc(&c->ws, total);
    if (e != cudaSuccess) {
        set_err(c, "cudaMalloc(%zu): %s", total, cudaGetErrorString(e));
        snprintf(g_err, sizeof g_err, "%s", c->err);
        delete c;
        return MMOT_ENOMEM;
    }
    char *base = static_cast<char *>(c->ws);
    for (int i = 0; i < c->nlev; ++i) {
        c->ops_f[i] = base + off_ops[i];
        c->ops_b[i] = base + off_ops[i] + (size_t)c->nlev_n[i] * opsz;
        c->car_f[i] = base + off_car[i];
        c->car_b[i] = base + off_car[i] + (size_t)c->nlev_n[i] * carsz;
    }
    c->car_bi = base + off_bi;
    c->partial = reinterpret_cast<double *>(base + off_part);
    c->dsc = reinterpret_cast<DevScalars *>(base + off_sc);
    c->nchp = (c->nchunks + 31) / 32 * 32;
    if (c->sw) {
        // chain-transposed internal vectors; zero-filled once so the tail of the last chain
        // (points >= N) holds phi = mu = 0 for the whole life of the context
        const size_t tb = (size_t)c->nchp * (size_t)c->P * sizeof(double);
        bool ok = cudaMalloc(&c->out_t, tb) == cudaSuccess && cudaMemsetAsync(c->out_t, 0, tb, c->stream) == cudaSuccess &&
                  cudaMalloc(&c->sw_end, 2 * (size_t)c->nchunks * M * sizeof(mmot::Dual)) == cudaSuccess;
        for (int qq = 0; qq < l && ok; ++qq)
            ok = cudaMalloc(&c->lin[qq], tb) == cudaSuccess && cudaMalloc(&c->mu_t[qq], tb) == cudaSuccess &&
                 cudaMemsetAsync(c->lin[qq], 0, tb, c->stream) == cudaSuccess &&
                 cudaMemsetAsync(c->mu_t[qq], 0, tb, c->stream) == cudaSuccess;
        if (!ok) {
            set_err(c, "cudaMalloc of the transposed vectors (%zu B each) failed", tb);
            snprintf(g_err, sizeof g_err, "%s", c->err);
            mmot_destroy(c);
            return MMOT_ENOMEM;
        }
        // restricted next-update scan: a second set of level-0 carries and the affine elements
        if (l >= 3 && l <= 5) {
            const int MO = 1 << (NB - 1);
            const size_t SZE = (size_t)(NB + 1) * MO;
            size_t tot = 2 * (size_t)c->nchunks * M;  // carB_f, carB_bi
            for (int i = 0; i < c->nlev; ++i) tot += 2 * (size_t)c->nlev_n[i] * (SZE + MO);
            if (cudaMalloc(&c->rx_mem, tot * sizeof(double)) != cudaSuccess) {
                set_err(c, "cudaMalloc of the restricted-scan workspace failed");
                snprintf(g_err, sizeof g_err, "%s", c->err);
                mmot_destroy(c);
                return MMOT_ENOMEM;
            }
            double *q = static_cast<double *>(c->rx_mem);
            c->carB_f = q;
            q += (size_t)c->nchunks * M;
            c->carB_bi = q;
            q += (size_t)c->nchunks * M;
            for (int i = 0; i < c->nlev; ++i) {
                c->rxe_f[i] = q;
                q += (size_t)c->nlev_n[i] * SZE;
                c->rxe_b[i] = q;
                q += (size_t)c->nlev_n[i] * SZE;
                c->rcar_f[i] = q;
                q += (size_t)c->nlev_n[i] * MO;
                c->rcar_b[i] = q;
                q += (size_t)c->nlev_n[i] * MO;
            }
            c->rx = getenv("MMOT_NO_RX") == nullptr;  // MMOT_NO_RX=1: full operator path (A/B runs)
        }
    } else if (c->opts.repr == MMOT_LOG) {
        for (int qq = 0; qq < l; ++qq) {
            e = cudaMalloc(&c->lin[qq], (size_t)N * sizeof(double));
            if (e != cudaSuccess) {
                set_err(c, "cudaMalloc scalings: %s", cudaGetErrorString(e));
                snprintf(g_err, sizeof g_err, "%s", c->err);
                mmot_destroy(c);
                return MMOT_ENOMEM;
            }
        }
    }
    if (l == 6 && !c->sw && c->opts.chunk == 0 && c->opts.kernel == MMOT_KERNEL_AUTO && getenv("MMOT_NO_LANES") == nullptr) {
        // lane-state family: chains of 32 points (its own operator / scan workspace)
        mmot::LsWork &w = c->ls;
        w.P = 32;
        w.C = (N + 31) / 32;
        w.nlev = 0;
        const int64_t B = mmot::kLsB;
        for (int64_t n = w.C;; n = (n + B - 1) / B) {
            w.lv_n[w.nlev++] = n;
            if (n <= B || w.nlev == mmot::kLsMaxLv) break;
        }
        size_t nd = 2 * (size_t)w.C * 192;
        for (int lv = 0; lv < w.nlev; ++lv) nd += 2 * (size_t)w.lv_n[lv] * (192 + 32) + 2 * (size_t)((w.lv_n[lv] + B - 1) / B) * 192;
        if (w.lv_n[w.nlev - 1] <= B && cudaMalloc(&c->ls_mem, nd * sizeof(double)) == cudaSuccess) {
            double *q = c->ls_mem;
            w.ops_f = q; q += (size_t)w.C * 192;
            w.ops_b = q; q += (size_t)w.C * 192;
            for (int lv = 0; lv < w.nlev; ++lv)
                for (int d = 0; d < 2; ++d) {
                    w.lv_excl[lv][d] = q; q += (size_t)w.lv_n[lv] * 192;
                    w.lv_car[lv][d] = q; q += (size_t)w.lv_n[lv] * 32;
                    w.lv_agg[lv][d] = q; q += (size_t)((w.lv_n[lv] + B - 1) / B) * 192;
                }
            c->ls_on = mmot::ls_init_tables() == cudaSuccess;
        } else {
            cudaGetLastError();
        }
    }
    if (cudaMallocHost(&c->hsc, sizeof(DevScalars)) != cudaSuccess ||
        cudaMallocHost(&c->hstop, 2 * sizeof(int)) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->poll_ev, cudaEventDisableTiming) != cudaSuccess) {
        set_err(c, "host allocation failed");
        snprintf(g_err, sizeof g_err, "%s", c->err);
        mmot_destroy(c);
        return MMOT_ENOMEM;
    }
    if (cudaMemsetAsync(c->dsc, 0, sizeof(DevScalars), c->stream) != cudaSuccess) {
        set_err(c, "memset failed");
        mmot_destroy(c);
        return MMOT_ECUDA;
    }
    *out = c;
    return MMOT_OK;
}

// Stabilised family (stable.cu): `batch` instances (1 for mmot_create), log-domain scalings g.
static mmot_status create_stable(int l, int64_t N, int64_t batch, const double *eta_host, mmot_grid grid, mmot_dtype dt,
                                 const mmot_opts *opts, void *cuda_stream, mmot_ctx **out) {
    mmot_ctx *c = new mmot_ctx();
    c->l = l;
    c->N = N;
    c->eta = eta_host[0];
    c->grid = grid;
    c->dt = dt;
    if (opts) c->opts = *opts;
    c->opts.kernel = MMOT_KERNEL_STABLE;
    c->stream = static_cast<cudaStream_t>(cuda_stream);
    cudaGetDevice(&c->device);
    c->h = N > 1 ? (grid.x_max - grid.x_min) / (double)(N - 1) : 1.0;
    c->stable = true;
    c->batch = batch;
    c->eta_host.assign(eta_host, eta_host + batch);
    const int M = 1 << (l - 1);
    mmot::SPlan &sp = c->sp;
    sp.l = l;
    sp.N = N;
    sp.batch = batch;
    sp.h = c->h;
    sp.hc = c->h;
    sp.slots = std::min<int64_t>(batch, 148 * 8);
    sp.scratch_per_warp = 2 * N * M;
    const size_t nd = (size_t)batch + (size_t)l * batch * N + (size_t)sp.slots * sp.scratch_per_warp + 2 * (size_t)batch;
    bool ok = cudaMalloc(&c->st_mem, nd * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&c->st_int, 5 * (size_t)batch * sizeof(int)) == cudaSuccess &&
              cudaMallocHost(&c->st_shost, 4 * (size_t)batch * sizeof(int)) == cudaSuccess &&
              cudaMallocHost(&c->st_rhost, (size_t)batch * sizeof(double)) == cudaSuccess &&
              cudaMallocHost(&c->st_whost, (size_t)batch * sizeof(double)) == cudaSuccess &&
              cudaMallocHost(&c->hsc, sizeof(DevScalars)) == cudaSuccess &&
              cudaMallocHost(&c->hstop, 2 * sizeof(int)) == cudaSuccess &&
              cudaMalloc(&c->ws, sizeof(DevScalars)) == cudaSuccess;
    if (!ok) {
        set_err(c, "stabilised workspace allocation failed (%zu B)", nd * sizeof(double));
        snprintf(g_err, sizeof g_err, "%s", c->err);
        mmot_destroy(c);
        return MMOT_ENOMEM;
    }
    c->dsc = static_cast<DevScalars *>(c->ws);
    double *p = c->st_mem;
    sp.eta = p;
    p += batch;
    for (int q = 0; q < l; ++q) {
        sp.g[q] = p;
        p += (size_t)batch * N;
    }
    sp.scratch = p;
    p += (size_t)sp.slots * sp.scratch_per_warp;
    sp.wout = p;
    sp.resid = p + batch;
    sp.status = c->st_int;
    sp.fail_iter = c->st_int + batch;
    sp.iters_done = c->st_int + 2 * batch;
    sp.converged = c->st_int + 3 * batch;
    if (cudaMemcpyAsync(const_cast<double *>(sp.eta), eta_host, (size_t)batch * sizeof(double), cudaMemcpyHostToDevice,
                        c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->dsc, 0, sizeof(DevScalars), c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess) {
        set_err(c, "stabilised workspace init failed");
        mmot_destroy(c);
        return MMOT_ECUDA;
    }
    *out = c;
    return MMOT_OK;
}

mmot_status mmot_create_batched(int l, int64_t N, int64_t batch, const double *eta_host, mmot_grid grid,
                                mmot_dtype dt, const mmot_opts *opts, void *cuda_stream, mmot_ctx **out) {
    if (!out) { set_err(nullptr, "out is NULL"); return MMOT_EINVAL; }
    *out = nullptr;
    if (l < 2 || l > 8) { set_err(nullptr, "l=%d outside [2,8]", l); return MMOT_EINVAL; }
    if (N < 1 || batch < 1 || !eta_host) { set_err(nullptr, "N, batch must be >= 1 and eta_host non-NULL"); return MMOT_EINVAL; }
    for (int64_t b = 0; b < batch; ++b)
        if (!(eta_host[b] > 0) || !isfinite(eta_host[b])) { set_err(nullptr, "eta[%lld] must be finite and > 0", (long long)b); return MMOT_EINVAL; }
    if (!isfinite(grid.x_min) || !isfinite(grid.x_max) || (N > 1 && !(grid.x_max > grid.x_min))) {
        set_err(nullptr, "grid must satisfy x_max > x_min");
        return MMOT_EINVAL;
    }
    if (dt != MMOT_F64 && dt != MMOT_F32) { set_err(nullptr, "bad dtype"); return MMOT_EINVAL; }
    if (opts && (opts->check_every < 0 || opts->chunk < 0 || (opts->repr != MMOT_LOG && opts->repr != MMOT_LINEAR))) {
        set_err(nullptr, "bad opts");
        return MMOT_EINVAL;
    }
    if (l > mmot::kMaxL && (dt != MMOT_F64 || (opts && opts->kernel != MMOT_KERNEL_AUTO && opts->kernel != MMOT_KERNEL_STABLE))) {
        set_err(nullptr, "l=%d > %d runs on the stabilised family only (MMOT_F64, MMOT_KERNEL_AUTO or _STABLE)", l, mmot::kMaxL);
        return MMOT_EUNSUPPORTED;
    }
    if ((opts && opts->kernel == MMOT_KERNEL_STABLE) || l > mmot::kMaxL) return create_stable(l, N, batch, eta_host, grid, dt, opts, cuda_stream, out);
    if (l > 5) {
        // l = 6 batches: the stabilised family (warp per instance, lane = subset state) under AUTO
        if (dt == MMOT_F64 && (!opts || opts->kernel == MMOT_KERNEL_AUTO))
            return create_stable(l, N, batch, eta_host, grid, dt, opts, cuda_stream, out);
        set_err(nullptr, "batched contexts with l > 5 run on the stabilised family only (MMOT_F64, MMOT_KERNEL_AUTO or _STABLE)");
        return MMOT_EUNSUPPORTED;
    }
    mmot_ctx *c = new mmot_ctx();
    c->l = l;
    c->N = N;
    c->eta = eta_host[0];
    c->grid = grid;
    c->dt = dt;
    if (opts) c->opts = *opts;
    c->stream = static_cast<cudaStream_t>(cuda_stream);
    cudaGetDevice(&c->device);
    c->h = N > 1 ? (grid.x_max - grid.x_min) / (double)(N - 1) : 1.0;
    c->batched = true;
    c->batch = batch;
    c->eta_host.assign(eta_host, eta_host + batch);
    mmot::BatchArgs &a = c->ba;
    a.l = l;
    a.N = N;
    a.batch = batch;
    a.P = (int)(((N + 31) / 32 + 7) / 8 * 8);
    a.h = c->h;
    a.slots = std::min<int64_t>(mmot::bat_slots(l), (batch + 3) / 4 * 4);
    const int NB = l - 1, M = 1 << NB;
    const size_t opsz = (size_t)2 * (NB + 1) * M * 32 * sizeof(mmot::Dual);      // per slot
    const size_t cksz = (size_t)(a.P / 8) * M * 32 * sizeof(mmot::Dual);         // per slot
    const size_t nd = (size_t)batch                      // eta
                      + (size_t)l * batch * N            // phit
                      + (size_t)a.slots * (opsz + cksz) / sizeof(double)
                      + (size_t)a.slots * N                // deferred-residual save planes
                      + 2 * (size_t)batch;               // wout, resid
    const size_t ni = (size_t)batch * l * 32 + 4 * (size_t)batch;
    bool ok = cudaMalloc(&c->bat_mem, nd * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&c->bat_int, ni * sizeof(int)) == cudaSuccess &&
              cudaMalloc(&c->bat_ptrs, 2 * mmot::kMaxL * sizeof(void *)) == cudaSuccess &&
              cudaMallocHost(&c->bat_whost, (size_t)batch * sizeof(double)) == cudaSuccess &&
              cudaMallocHost(&c->bat_shost, 4 * (size_t)batch * sizeof(int)) == cudaSuccess &&
              cudaMallocHost(&c->bat_rhost, (size_t)batch * sizeof(double)) == cudaSuccess &&
              cudaMallocHost(&c->hsc, sizeof(DevScalars)) == cudaSuccess &&
              cudaMalloc(&c->ws, sizeof(DevScalars)) == cudaSuccess;
    if (!ok) {
        set_err(c, "batched workspace allocation failed (%zu B)", nd * sizeof(double));
        snprintf(g_err, sizeof g_err, "%s", c->err);
        mmot_destroy(c);
        return MMOT_ENOMEM;
    }
    c->dsc = static_cast<DevScalars *>(c->ws);
    double *p = c->bat_mem;
    a.eta = p;
    p += batch;
    for (int q = 0; q < l; ++q) {
        a.phit[q] = p;
        p += (size_t)batch * N;
    }
    a.ops = p;
    p += (size_t)a.slots * opsz / sizeof(double);
    a.ckpt = p;
    p += (size_t)a.slots * cksz / sizeof(double);
    a.rsave = p;
    p += (size_t)a.slots * N;
    a.wout = p;
    a.resid = p + batch;
    a.E = c->bat_int;
    a.status = c->bat_int + (size_t)batch * l * 32;
    a.fail_iter = a.status + batch;
    a.iters_done = a.status + 2 * batch;
    a.converged = a.status + 3 * batch;
    if (cudaMemsetAsync(c->bat_mem, 0, nd * sizeof(double), c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->bat_int, 0, ni * sizeof(int), c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->dsc, 0, sizeof(DevScalars), c->stream) != cudaSuccess ||
        cudaMemcpyAsync(c->bat_mem, eta_host, (size_t)batch * sizeof(double), cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess) {
        set_err(c, "batched workspace init failed");
        mmot_destroy(c);
        return MMOT_ECUDA;
    }
    *out = c;
    return MMOT_OK;
}

// Non-uniform grid points (paper footnote P:182): batched context as above whose edge e (between
// points e-1 and e) has its own length h_e = x[e] - x[e-1] and decay lambda_e = exp(-h_e / eta).
mmot_status mmot_create_batched_points(int l, int64_t N, int64_t batch, const double *eta_host, const double *x_host,
                                       mmot_dtype dt, const mmot_opts *opts, void *cuda_stream, mmot_ctx **out) {
    if (!out) { set_err(nullptr, "out is NULL"); return MMOT_EINVAL; }
    *out = nullptr;
    if (!x_host || N < 1) { set_err(nullptr, "x_host must hold N >= 1 grid points"); return MMOT_EINVAL; }
    for (int64_t i = 0; i < N; ++i)
        if (!isfinite(x_host[i]) || (i > 0 && !(x_host[i] > x_host[i - 1]))) {
            set_err(nullptr, "grid points must be finite and strictly increasing (index %lld)", (long long)i);
            return MMOT_EINVAL;
        }
    if (opts && opts->kernel != MMOT_KERNEL_AUTO && opts->kernel != MMOT_KERNEL_PERSISTENT) {
        set_err(nullptr, "non-uniform grids run on the persistent (batched) kernel family only");
        return MMOT_EUNSUPPORTED;
    }
    mmot_grid g{x_host[0], N > 1 ? x_host[N - 1] : x_host[0] + 1.0};
    mmot_ctx *c = nullptr;
    mmot_status st = mmot_create_batched(l, N, batch, eta_host, g, dt, opts, cuda_stream, &c);
    if (st) return st;
    mmot::BatchArgs &a = c->ba;
    const int64_t ne = 32 * (int64_t)a.P + 1;
    std::vector<double> hx((size_t)ne, 0.0);
    for (int64_t e = 1; e < N; ++e) hx[(size_t)e] = x_host[e] - x_host[e - 1];
    if (cudaMalloc(&c->pts_mem, (size_t)(1 + batch) * ne * sizeof(double)) != cudaSuccess) {
        set_err(c, "grid workspace allocation failed");
        snprintf(g_err, sizeof g_err, "%s", c->err);
        mmot_destroy(c);
        return MMOT_ENOMEM;
    }
    double *dhx = c->pts_mem, *dlam = c->pts_mem + ne;
    if (cudaMemcpyAsync(dhx, hx.data(), (size_t)ne * sizeof(double), cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
        mmot::launch_bat_lambda(dlam, dhx, a.eta, batch, ne, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess) {
        set_err(c, "grid workspace init failed");
        snprintf(g_err, sizeof g_err, "%s", c->err);
        mmot_destroy(c);
        return MMOT_ECUDA;
    }
    a.hx = dhx;
    a.lam = dlam;
    a.ne = ne;
    *out = c;
    return MMOT_OK;
}

mmot_status mmot_create_2d(int l, int64_t N1, int64_t N2, double eta, mmot_grid2d grid, mmot_dtype dt,
                           const mmot_opts *opts, void *cuda_stream, mmot_ctx **out) {
    if (!out) { set_err(nullptr, "out is NULL"); return MMOT_EINVAL; }
    *out = nullptr;
    if (l < 2 || l > 8) { set_err(nullptr, "l=%d outside [2,8]", l); return MMOT_EINVAL; }
    if (N1 < 1 || N2 < 1) { set_err(nullptr, "N1, N2 must be >= 1"); return MMOT_EINVAL; }
    if (!(eta > 0) || !isfinite(eta)) { set_err(nullptr, "eta must be finite and > 0"); return MMOT_EINVAL; }
    if (!isfinite(grid.x_min) || !isfinite(grid.x_max) || !isfinite(grid.y_min) || !isfinite(grid.y_max) ||
        (N1 > 1 && !(grid.x_max > grid.x_min)) || (N2 > 1 && !(grid.y_max > grid.y_min))) {
        set_err(nullptr, "grid must satisfy x_max > x_min, y_max > y_min");
        return MMOT_EINVAL;
    }
    if (dt != MMOT_F64 && dt != MMOT_F32) { set_err(nullptr, "bad dtype"); return MMOT_EINVAL; }
    if (opts && (opts->check_every < 0 || (opts->repr != MMOT_LOG && opts->repr != MMOT_LINEAR))) {
        set_err(nullptr, "bad opts");
        return MMOT_EINVAL;
    }
    if (l != 3) { set_err(nullptr, "2-D grids: l = 3 in this build (the paper's 2-D case, P:712-979)"); return MMOT_EUNSUPPORTED; }
    mmot_ctx *c = new mmot_ctx();
    c->l = l;
    c->N = N1 * N2;
    c->eta = eta;
    c->dt = dt;
    if (opts) c->opts = *opts;
    c->stream = static_cast<cudaStream_t>(cuda_stream);
    cudaGetDevice(&c->device);
    c->g2 = true;
    c->g2N = N1;
    c->g2M = N2;
    c->g2h1 = N1 > 1 ? (grid.x_max - grid.x_min) / (double)(N1 - 1) : 1.0;
    c->g2h2 = N2 > 1 ? (grid.y_max - grid.y_min) / (double)(N2 - 1) : 1.0;
    c->h = c->g2h1;
    c->grid = mmot_grid{grid.x_min, grid.x_max};
    const int64_t n = c->N;
    const size_t tsz = ((size_t)6 * n + (size_t)18 * n + (size_t)(std::max(N1, N2) + 1) * std::max(N1, N2) + 64) *
                       sizeof(mmot::Dual);
    bool ok = cudaMalloc(&c->g2_mem, (size_t)7 * n * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&c->g2_T, tsz) == cudaSuccess &&
              cudaMalloc(&c->ws, sizeof(DevScalars) + (size_t)(std::max(N1, N2) + 64) * sizeof(double)) == cudaSuccess &&
              cudaMallocHost(&c->hsc, sizeof(DevScalars)) == cudaSuccess &&
              cudaMallocHost(&c->hstop, 2 * sizeof(int)) == cudaSuccess &&
              cudaEventCreateWithFlags(&c->poll_ev, cudaEventDisableTiming) == cudaSuccess;
    for (int q = 0; q < l && ok; ++q) ok = cudaMalloc(&c->lin[q], (size_t)n * sizeof(double)) == cudaSuccess;
    if (!ok) {
        set_err(c, "2-D workspace allocation failed");
        snprintf(g_err, sizeof g_err, "%s", c->err);
        mmot_destroy(c);
        return MMOT_ENOMEM;
    }
    c->dsc = static_cast<DevScalars *>(c->ws);
    c->partial = reinterpret_cast<double *>(static_cast<char *>(c->ws) + ((sizeof(DevScalars) + 255) / 256) * 256);
    if (cudaMemsetAsync(c->dsc, 0, sizeof(DevScalars), c->stream) != cudaSuccess) {
        set_err(c, "memset failed");
        mmot_destroy(c);
        return MMOT_ECUDA;
    }
    *out = c;
    return MMOT_OK;
}

mmot_status mmot_create_points(int l, int64_t N, double eta, const double *x_host, mmot_dtype dt, const mmot_opts *opts,
                               void *cuda_stream, mmot_ctx **out) {
    if (!out) { set_err(nullptr, "out is NULL"); return MMOT_EINVAL; }
    *out = nullptr;
    if (!(eta > 0) || !isfinite(eta)) { set_err(nullptr, "eta must be finite and > 0"); return MMOT_EINVAL; }
    const int kern = opts ? opts->kernel : MMOT_KERNEL_AUTO;
    if (kern == MMOT_KERNEL_PERSISTENT || (kern == MMOT_KERNEL_AUTO && l <= 5 && N <= 4096))
        return mmot_create_batched_points(l, N, 1, &eta, x_host, dt, opts, cuda_stream, out);
    if (kern == MMOT_KERNEL_SINGLE_WALK) {
        set_err(nullptr, "non-uniform grids run on the two-walk or persistent kernel families");
        return MMOT_EUNSUPPORTED;
    }
    // larger instances: the two-walk family with per-edge decays
    if (!x_host || N < 1) { set_err(nullptr, "x_host must hold N >= 1 grid points"); return MMOT_EINVAL; }
    for (int64_t i = 0; i < N; ++i)
        if (!isfinite(x_host[i]) || (i > 0 && !(x_host[i] > x_host[i - 1]))) {
            set_err(nullptr, "grid points must be finite and strictly increasing (index %lld)", (long long)i);
            return MMOT_EINVAL;
        }
    mmot_opts o2 = opts ? *opts : mmot_opts{0, 0, MMOT_LOG, 0, MMOT_KERNEL_AUTO};
    o2.kernel = MMOT_KERNEL_TWO_WALK;
    mmot_grid g{x_host[0], N > 1 ? x_host[N - 1] : x_host[0] + 1.0};
    mmot_ctx *c = nullptr;
    mmot_status st = create_single(l, N, eta, g, dt, &o2, cuda_stream, &c, false);
    if (st) return st;
    const int64_t ne = c->nchunks * c->P + 1;
    std::vector<double> hv(2 * (size_t)ne, 0.0);  // [hx | lambda]
    for (int64_t e = 0; e < ne; ++e) {
        const double he = (e >= 1 && e < N) ? x_host[e] - x_host[e - 1] : 0.0;
        hv[(size_t)e] = he;
        hv[(size_t)(ne + e)] = he > 0.0 ? exp(-he / eta) : 1.0;
    }
    if (cudaMalloc(&c->pts_mem, 2 * (size_t)ne * sizeof(double)) != cudaSuccess ||
        cudaMemcpyAsync(c->pts_mem, hv.data(), 2 * (size_t)ne * sizeof(double), cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess) {
        set_err(c, "grid workspace allocation failed");
        snprintf(g_err, sizeof g_err, "%s", c->err);
        mmot_destroy(c);
        return MMOT_ENOMEM;
    }
    c->pts_hx = c->pts_mem;
    c->pts_lam = c->pts_mem + ne;
    *out = c;
    return MMOT_OK;
}

}  // extern "C"

static mmot_status reset_scalars(mmot_ctx *c);
static mmot_status sync_report(mmot_ctx *c);

// Upload an array of l device pointers (for the batched import / export kernels).
static mmot_status bat_upload_ptrs(mmot_ctx *c, const void *const *u, int slot) {
    void *h[mmot::kMaxL] = {nullptr};
    for (int q = 0; q < c->l; ++q) {
        if (!u[q]) { set_err(c, "u[%d] is NULL", q); return MMOT_EINVAL; }
        h[q] = const_cast<void *>(u[q]);
    }
    CK(c, cudaMemcpyAsync(c->bat_ptrs + slot * mmot::kMaxL, h, sizeof h, cudaMemcpyHostToDevice, c->stream));
    return MMOT_OK;
}

static mmot_status bat_import(mmot_ctx *c, const void *const *u) {
    mmot_status st = bat_upload_ptrs(c, u, 0);
    if (st) return st;
    CK(c, mmot::launch_bat_convert(c->ba, c->bat_ptrs, 1, c->opts.repr == MMOT_LOG, c->stream, &c->launches));
    return MMOT_OK;
}

// Per-instance report arrays [status | fail_iter | iters_done | converged] (ints) and residuals ->
// the batch report (max sweeps, max residual, all converged, first failing instance).
static mmot_status aggregate_report(mmot_ctx *c, int64_t B, const int *sh, const double *rh, double tol,
                                    mmot_report *rep) {
    int status = 0, fail = -1, done = 0, conv = 1;
    double res = 0.0;
    for (int64_t b = 0; b < B; ++b) {
        if (sh[b] && !status) { status = sh[b]; fail = sh[B + b]; }
        done = std::max(done, sh[2 * B + b]);
        conv &= sh[3 * B + b];
        res = std::max(res, rh[b]);  // NaN (never computed) propagates as "not a number"
        if (isnan(rh[b])) res = NAN;
    }
    if (rep) {
        rep->iters_done = done;                      // max over instances
        rep->residual = tol > 0 ? res : NAN;         // max over instances
        rep->converged = tol > 0 && conv;            // all instances
        rep->status = status;
        rep->fail_iter = status ? fail : -1;
    }
    if (status) set_err(c, "%s (an instance failed at sweep %d)", mmot_strerror((mmot_status)status), fail);
    return (mmot_status)status;
}

// ---------------------------------------------------------------------------------------
// Stabilised family (stable.cu).  u (caller layout, repr per opts) <-> g = log phi; sel: device
// mask of the instances to touch (null: all).
static mmot_status st_import(mmot_ctx *c, const void *const *u, const int *sel) {
    for (int q = 0; q < c->l; ++q) {
        if (!u[q]) { set_err(c, "u[%d] is NULL", q); return MMOT_EINVAL; }
        CK(c, mmot::launch_st_convert(static_cast<const double *>(u[q]), c->sp.g[q], c->batch, c->N, sel,
                                      c->opts.repr == MMOT_LOG ? 0 : 1, c->stream, &c->launches));
    }
    return MMOT_OK;
}
static mmot_status st_export(mmot_ctx *c, void *const *u, const int *sel) {
    for (int q = 0; q < c->l; ++q)
        CK(c, mmot::launch_st_convert(c->sp.g[q], static_cast<double *>(u[q]), c->batch, c->N, sel,
                                      c->opts.repr == MMOT_LOG ? 0 : 2, c->stream, &c->launches));
    return MMOT_OK;
}

// Sinkhorn on the stabilised family from u_in into u_out (may alias).  sel_host (optional): the
// instances to run; the per-instance results are left in st_shost / st_rhost.  report_all = false:
// the caller merges them (no aggregate, returns MMOT_OK unless the call itself failed).
static mmot_status st_sinkhorn(mmot_ctx *c, const double *const *mu, int iters, double tol, const void *const *u_in,
                               void *const *u_out, mmot_report *rep, const int *sel_host, bool report_all = true) {
    const int l = c->l;
    const int64_t B = c->batch, n = B * c->N;
    mmot_status st = reset_scalars(c);
    if (st) return st;
    for (int q = 0; q < l; ++q) {
        if (!u_in[q] || !u_out[q]) { set_err(c, "u[%d] is NULL", q); return MMOT_EINVAL; }
        CK(c, mmot::launch_check(mu[q], n, 0, &c->dsc->flags[q], nullptr, c->stream, &c->launches));
        CK(c, mmot::launch_bat_min_mass(mu[q], B, c->N, &c->dsc->mass[q], c->stream, &c->launches));
        CK(c, mmot::launch_check(static_cast<const double *>(u_in[q]), n, c->opts.repr == MMOT_LOG ? 1 : 0,
                                 &c->dsc->flags[l + q], nullptr, c->stream, &c->launches));
    }
    CK(c, mmot::launch_check_finish(c->dsc->flags, c->dsc->mass, 2 * l, l, &c->dsc->status, &c->dsc->stop,
                                    &c->dsc->fail_iter, c->stream, &c->launches));
    if ((st = sync_report(c))) return st;
    if (c->hsc->status) {
        if (rep) { rep->status = c->hsc->status; rep->fail_iter = 0; }
        set_err(c, "%s", mmot_strerror((mmot_status)c->hsc->status));
        return (mmot_status)c->hsc->status;
    }
    int *sel = nullptr;
    if (sel_host) {
        sel = c->st_int + 4 * B;
        CK(c, cudaMemcpyAsync(sel, sel_host, (size_t)B * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    }
    CK(c, cudaMemsetAsync(c->st_int, 0, 4 * (size_t)B * sizeof(int), c->stream));
    if ((st = st_import(c, u_in, sel))) return st;
    mmot::SPlan sp = c->sp;
    for (int q = 0; q < l; ++q) sp.mu[q] = mu[q];
    sp.iters = iters;
    sp.tol = tol;
    sp.check_every = c->opts.check_every > 0 ? c->opts.check_every : 1;
    sp.sel = sel;
    CK(c, mmot::launch_stable(sp, 0, c->stream, &c->launches));
    if ((st = st_export(c, u_out, sel))) return st;
    CK(c, cudaMemcpyAsync(c->st_shost, c->st_int, 4 * (size_t)B * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaMemcpyAsync(c->st_rhost, sp.resid, (size_t)B * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    if (!report_all) return MMOT_OK;
    return aggregate_report(c, B, c->st_shost, c->st_rhost, tol, rep);
}

static mmot_status st_marginal(mmot_ctx *c, int k, const void *const *u, void *out) {
    mmot_status st = st_import(c, u, nullptr);
    if (st) return st;
    CK(c, cudaMemsetAsync(c->st_int, 0, 4 * (size_t)c->batch * sizeof(int), c->stream));
    mmot::SPlan sp = c->sp;
    sp.k = k;
    sp.out = static_cast<double *>(out);
    CK(c, mmot::launch_stable(sp, 1, c->stream, &c->launches));
    return MMOT_OK;
}

static mmot_status st_cost(mmot_ctx *c, const void *const *u, double *W) {
    mmot_status st = st_import(c, u, nullptr);
    if (st) return st;
    CK(c, cudaMemsetAsync(c->st_int, 0, 4 * (size_t)c->batch * sizeof(int), c->stream));
    CK(c, mmot::launch_stable(c->sp, 2, c->stream, &c->launches));
    CK(c, cudaMemcpyAsync(c->st_whost, c->sp.wout, (size_t)c->batch * sizeof(double), cudaMemcpyDeviceToHost,
                          c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    memcpy(W, c->st_whost, (size_t)c->batch * sizeof(double));
    return MMOT_OK;
}

// The plain families fall back to the stabilised one when a product leaves the fp64 range
// (MMOT_EOVERFLOW): the call is redone from its inputs on a stabilised context of the same problem
// (created on first use).  Uniform grids only (the stabilised family has no per-edge weights).
static mmot_status ensure_stable(mmot_ctx *c) {
    if (c->st_fb) return MMOT_OK;
    if (c->eta_host.empty()) c->eta_host.assign(1, c->eta);
    mmot_opts o = c->opts;
    o.kernel = MMOT_KERNEL_STABLE;
    mmot_status st = create_stable(c->l, c->N, (int64_t)c->eta_host.size(), c->eta_host.data(), c->grid, MMOT_F64, &o,
                                   c->stream, &c->st_fb);
    if (st) set_err(c, "stabilised fallback context: %s", mmot_last_error(nullptr));
    return st;
}

static bool can_stabilise(const mmot_ctx *c) {
    return !c->sharded && !c->pts_lam && !c->ba.lam && !c->stable && getenv("MMOT_NO_STABLE") == nullptr;
}

// Pair family (pair.cu): batched contexts with uniform grids and a fixed sweep count (tol <= 0)
// whose batch fills the GPU (>= MMOT_PAIR_MIN instances, default 4096: two threads per instance,
// so smaller batches leave SMs idle and the one-warp-per-instance kernel is faster).  MMOT_NO_PAIR=1
// disables it.  The workspace (its own layout: mantissas + slab exponents, checkpoints) is
// allocated on first use.
static bool ensure_pair(mmot_ctx *c) {
    if (c->pair_state) return c->pair_state > 0;
    c->pair_state = -1;
    const char *mn = getenv("MMOT_PAIR_MIN");
    const int64_t pmin = mn ? atoll(mn) : 4096;
    if (!c->batched || c->ba.lam || c->l < 2 || c->l > 5 || c->batch < pmin || getenv("MMOT_NO_PAIR") != nullptr)
        return false;
    mmot::PairPlan &p = c->pp;
    p.l = c->l;
    p.batch = c->batch;
    p.N = c->N;
    p.nA = (int)((c->N + 1) / 2);
    p.nB = (int)(c->N / 2);
    p.nslab = (p.nA + 7) / 8;
    p.nblk = (c->batch + 15) / 16;
    p.h = c->h;
    p.eta = c->ba.eta;
    p.f32 = c->dt == MMOT_F32 ? 1 : 0;
    p.f32c = p.f32 && getenv("MMOT_PAIR_F64") == nullptr ? 1 : 0;
    p.slots = (std::min<int64_t>(p.nblk, mmot::pair_slots()) + 1) / 2 * 2;
    const size_t es = p.f32 ? sizeof(float) : sizeof(double);
    const size_t nv = (size_t)c->l * p.nblk * p.nslab * 8 * 32;
    const size_t ne = (size_t)c->l * p.nblk * p.nslab * 32;
    const size_t nck = (size_t)p.slots * p.nslab * (1u << (c->l - 1)) * 32;
    const size_t bytes = nck * sizeof(double) + 2 * nv * es + 2 * ne * sizeof(int);  // E and G records
    if (cudaMalloc(&c->pair_mem, bytes) != cudaSuccess) {
        cudaGetLastError();
        c->pair_mem = nullptr;
        return false;  // the persistent kernel runs instead
    }
    char *q = static_cast<char *>(c->pair_mem);
    p.ckpt = reinterpret_cast<double *>(q);
    q += nck * sizeof(double);
    p.phit = q;
    q += nv * es;
    p.mu = q;
    q += nv * es;
    p.E = reinterpret_cast<int *>(q);
    p.status = c->ba.status;
    p.fail_iter = c->ba.fail_iter;
    p.iters_done = c->ba.iters_done;
    p.converged = c->ba.converged;
    p.resid = c->ba.resid;
    c->pair_state = 1;
    return true;
}

// CTA family (cta.cu): batched contexts of at most one wave of instances (batch <= SM count) with
// l <= 4, N <= 4096, a uniform grid, and every instance inside kCtaRange (plain fp64 scalings).
// MMOT_NO_CTA=1 disables it.
static bool ensure_cta(mmot_ctx *c) {
    if (c->cta_state) return c->cta_state > 0;
    c->cta_state = -1;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    if (!c->batched || c->ba.lam || c->l < 2 || c->l > 4 || c->N > 4096 || c->batch > sms ||
        getenv("MMOT_NO_CTA") != nullptr)
        return false;
    const double span = c->grid.x_max - c->grid.x_min;
    for (double e : c->eta_host)
        if ((c->l - 1) * span / e > mmot::kCtaRange) return false;
    mmot::CtaPlan &p = c->cp;
    p.l = c->l;
    p.N = c->N;
    p.batch = c->batch;
    p.P = mmot::cta_chain_len(c->N);
    p.h = c->h;
    p.eta = c->ba.eta;
    for (int q = 0; q < c->l; ++q) p.phi[q] = c->ba.phit[q];
    if (cudaMalloc(&c->cta_mem, (size_t)c->batch * c->N * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        c->cta_mem = nullptr;
        return false;
    }
    p.scr = c->cta_mem;
    p.status = c->ba.status;
    p.fail_iter = c->ba.fail_iter;
    p.iters_done = c->ba.iters_done;
    p.converged = c->ba.converged;
    p.resid = c->ba.resid;
    c->cta_state = 1;
    return true;
}

static mmot_status bat_sinkhorn(mmot_ctx *c, const double *const *mu, int iters, double tol, void *const *u,
                                mmot_report *rep) {
    mmot_status st = reset_scalars(c);
    if (st) return st;
    const int64_t n = c->batch * c->N;
    for (int q = 0; q < c->l; ++q) {
        // element checks over the whole batch; zero mass per instance (the smallest instance mass)
        CK(c, mmot::launch_check(mu[q], n, 0, &c->dsc->flags[q], nullptr, c->stream, &c->launches));
        CK(c, mmot::launch_bat_min_mass(mu[q], c->batch, c->N, &c->dsc->mass[q], c->stream, &c->launches));
        CK(c, mmot::launch_check(static_cast<const double *>(u[q]), n, c->opts.repr == MMOT_LOG ? 1 : 0,
                                 &c->dsc->flags[c->l + q], nullptr, c->stream, &c->launches));
    }
    CK(c, mmot::launch_check_finish(c->dsc->flags, c->dsc->mass, 2 * c->l, c->l, &c->dsc->status, &c->dsc->stop,
                                    &c->dsc->fail_iter, c->stream, &c->launches));
    CK(c, cudaMemcpyAsync(c->hsc, c->dsc, sizeof(DevScalars), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    if (c->hsc->status) {
        if (rep) { rep->status = c->hsc->status; rep->fail_iter = 0; }
        set_err(c, "%s", mmot_strerror((mmot_status)c->hsc->status));
        return (mmot_status)c->hsc->status;
    }
    const bool pair = tol <= 0 && ensure_pair(c);
    const bool cta = !pair && ensure_cta(c);
    if (cta) {
        // CTA family: linear scalings, all sweeps (and residual checks) in one launch
        if ((st = bat_upload_ptrs(c, u, 0))) return st;
        CK(c, mmot::launch_cta_convert(c->cp, c->bat_ptrs, 0, c->opts.repr == MMOT_LOG, c->stream, &c->launches));
        mmot::CtaPlan p = c->cp;
        for (int q = 0; q < c->l; ++q) p.mu[q] = mu[q];
        p.iters = iters;
        p.tol = tol;
        p.check_every = c->opts.check_every > 0 ? c->opts.check_every : 1;
        CK(c, mmot::launch_cta_sinkhorn(p, c->stream, &c->launches));
        ++c->cta_solves;
    } else if (pair) {
        // pair family: u and mu into its layout, all sweeps in one launch
        if ((st = bat_upload_ptrs(c, u, 0))) return st;
        if ((st = bat_upload_ptrs(c, reinterpret_cast<const void *const *>(mu), 1))) return st;
        CK(c, mmot::launch_pair_convert(c->pp, c->bat_ptrs, 0, c->opts.repr == MMOT_LOG, c->stream, &c->launches));
        CK(c, mmot::launch_pair_convert(c->pp, c->bat_ptrs + mmot::kMaxL, 2, 0, c->stream, &c->launches));
        mmot::PairPlan p = c->pp;
        p.iters = iters;
        CK(c, mmot::launch_pair_sinkhorn(p, c->stream, &c->launches));
        ++c->pair_solves;
        if (p.f32c) ++c->pair_f32_solves;
    } else {
        st = bat_import(c, u);
        if (st) return st;
        mmot::BatchArgs a = c->ba;
        for (int q = 0; q < c->l; ++q) a.mu[q] = mu[q];
        a.iters = iters;
        a.tol = tol;
        a.check_every = c->opts.check_every > 0 ? c->opts.check_every : 1;
        CK(c, mmot::launch_batched(a, 0, c->stream, &c->launches));
    }
    CK(c, cudaMemcpyAsync(c->bat_shost, c->ba.status, 4 * (size_t)c->batch * sizeof(int), cudaMemcpyDeviceToHost,
                          c->stream));
    CK(c, cudaMemcpyAsync(c->bat_rhost, c->ba.resid, (size_t)c->batch * sizeof(double), cudaMemcpyDeviceToHost,
                          c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    const int64_t B = c->batch;
    // instances whose products left the fp64 range: redo them on the stabilised family, from this
    // call's u (still untouched: the export below comes after the stabilised import)
    std::vector<int> sel((size_t)B, 0);
    int64_t nfail = 0;
    for (int64_t b = 0; b < B; ++b)
        if (c->bat_shost[b] == MMOT_EOVERFLOW) { sel[(size_t)b] = 1; ++nfail; }
    if (nfail > 0 && getenv("MMOT_DEBUG_FAIL")) {  // diagnostics: which instances left the range
        std::vector<double> eh((size_t)B);
        cudaMemcpy(eh.data(), c->ba.eta, (size_t)B * sizeof(double), cudaMemcpyDeviceToHost);
        fprintf(stderr, "[mmot] %lld of %lld instances left the range (family: %s)\n", (long long)nfail, (long long)B,
                pair ? (c->pp.f32c ? "pair fp32" : "pair fp64") : cta ? "cta" : "persistent");
        int shown = 0;
        for (int64_t b = 0; b < B && shown < 64; ++b)
            if (sel[(size_t)b]) {
                fprintf(stderr, "[mmot]   instance %lld eta %.6g fail_iter %d\n", (long long)b, eh[(size_t)b],
                        c->bat_shost[B + b]);
                ++shown;
            }
    }
    // fp32 pair solves: instances whose states left the fp32 range (rare: 2 of C5's 8192, deep marginal
    // tails at moderate eta) are redone first in fp64 on a batched context of their own
    // (the one-warp-per-instance kernel: per-instance latency, not the pair family's), from this
    // call's u (still untouched: the export below comes after the gather)
    std::vector<double *> sub_u;
    std::vector<int64_t> sub_idx;
    mmot_ctx *sub = nullptr;
    if (nfail > 0 && pair && c->pp.f32c) {
        const size_t row = (size_t)c->N * sizeof(double);
        for (int64_t b = 0; b < B; ++b)
            if (sel[(size_t)b]) sub_idx.push_back(b);
        const int64_t nf = (int64_t)sub_idx.size();
        std::vector<double> eh((size_t)B), es((size_t)nf);
        CK(c, cudaMemcpy(eh.data(), c->ba.eta, (size_t)B * sizeof(double), cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < nf; ++i) es[(size_t)i] = eh[(size_t)sub_idx[(size_t)i]];
        mmot_opts so = c->opts;
        so.kernel = MMOT_KERNEL_AUTO;
        mmot_status cs = mmot_create_batched(c->l, c->N, nf, es.data(), c->grid, MMOT_F64, &so, c->stream, &sub);
        double *buf = nullptr;
        if (cs == MMOT_OK && cudaMalloc(&buf, 2 * (size_t)c->l * nf * row) == cudaSuccess) {
            std::vector<const void *> smu((size_t)c->l);
            for (int q = 0; q < c->l; ++q) {
                double *mq = buf + (size_t)q * nf * c->N, *uq = buf + (size_t)(c->l + q) * nf * c->N;
                smu[(size_t)q] = mq;
                sub_u.push_back(uq);
                for (int64_t i = 0; i < nf; ++i) {
                    const int64_t b = sub_idx[(size_t)i];
                    CK(c, cudaMemcpyAsync(mq + i * c->N, mu[q] + b * c->N, row, cudaMemcpyDeviceToDevice, c->stream));
                    CK(c, cudaMemcpyAsync(uq + i * c->N, static_cast<const double *>(u[q]) + b * c->N, row,
                                          cudaMemcpyDeviceToDevice, c->stream));
                }
            }
            mmot_report sr{};
            cs = mmot_sinkhorn(sub, smu.data(), iters, tol, reinterpret_cast<void *const *>(sub_u.data()), &sr);
            if (cs == MMOT_OK) {
                for (int64_t i = 0; i < nf; ++i) {
                    const int64_t b = sub_idx[(size_t)i];
                    sel[(size_t)b] = 0;
                    c->bat_shost[b] = 0;
                    c->bat_shost[B + b] = -1;
                    c->bat_shost[2 * B + b] = iters;
                    c->bat_shost[3 * B + b] = 0;
                }
                c->pair_redo += nf;
                nfail = 0;
            } else {
                sub_u.clear();  // the stabilised family redoes them below
            }
        } else {
            cudaGetLastError();
        }
        if (sub_u.empty()) {
            cudaFree(buf);
            mmot_destroy(sub);
            sub = nullptr;
        } else {
            sub_u.push_back(buf);  // freed after the scatter
        }
    }
    const bool redo = nfail > 0 && can_stabilise(c);
    if (redo) {
        if ((st = ensure_stable(c))) return st;
        mmot_ctx *sc = c->st_fb;
        ++c->st_fallbacks;
        // import first (reads the caller's u), then this context's export, then the stabilised solve
        int *dsel = sc->st_int + 4 * B;
        CK(c, cudaMemcpyAsync(dsel, sel.data(), (size_t)B * sizeof(int), cudaMemcpyHostToDevice, c->stream));
        if ((st = st_import(sc, const_cast<const void *const *>(u), dsel))) return st;
    }
    st = bat_upload_ptrs(c, const_cast<const void *const *>(u), 0);
    if (st) return st;
    if (cta) CK(c, mmot::launch_cta_convert(c->cp, c->bat_ptrs, 1, c->opts.repr == MMOT_LOG, c->stream, &c->launches));
    else if (pair) CK(c, mmot::launch_pair_convert(c->pp, c->bat_ptrs, 1, c->opts.repr == MMOT_LOG, c->stream, &c->launches));
    else CK(c, mmot::launch_bat_convert(c->ba, c->bat_ptrs, 0, c->opts.repr == MMOT_LOG, c->stream, &c->launches));
    if (sub) {
        // the fp64 results of the redone instances over the export
        const size_t row = (size_t)c->N * sizeof(double);
        for (int q = 0; q < c->l; ++q)
            for (size_t i = 0; i < sub_idx.size(); ++i)
                CK(c, cudaMemcpyAsync(static_cast<double *>(u[q]) + sub_idx[i] * c->N, sub_u[(size_t)q] + i * c->N, row,
                                      cudaMemcpyDeviceToDevice, c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
        cudaFree(sub_u.back());
        mmot_destroy(sub);
    }
    if (redo) {
        mmot_ctx *sc = c->st_fb;
        CK(c, cudaMemsetAsync(sc->st_int, 0, 4 * (size_t)B * sizeof(int), c->stream));
        mmot::SPlan sp = sc->sp;
        for (int q = 0; q < c->l; ++q) sp.mu[q] = mu[q];
        sp.iters = iters;
        sp.tol = tol;
        sp.check_every = c->opts.check_every > 0 ? c->opts.check_every : 1;
        sp.sel = sc->st_int + 4 * B;
        CK(c, mmot::launch_stable(sp, 0, c->stream, &sc->launches));
        if ((st = st_export(sc, u, sp.sel))) return st;
        CK(c, cudaMemcpyAsync(sc->st_shost, sc->st_int, 4 * (size_t)B * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaMemcpyAsync(sc->st_rhost, sp.resid, (size_t)B * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
        for (int64_t b = 0; b < B; ++b)
            if (sel[(size_t)b]) {
                for (int f = 0; f < 4; ++f) c->bat_shost[f * B + b] = sc->st_shost[f * B + b];
                c->bat_rhost[b] = sc->st_rhost[b];
            }
    } else {
        CK(c, cudaStreamSynchronize(c->stream));
    }
    return aggregate_report(c, B, c->bat_shost, c->bat_rhost, tol, rep);
}

// ---------------------------------------------------------------------------------------
// Collectives of sharded contexts, on the context stream: NCCL across processes, or the
// in-process virtual group (several shards on one device).  Every rank issues the same sequence.
static int coll_fail(mmot_ctx *c, const char *what, int r) {
    if (!c->exch_error) {
        c->exch_error = r ? r : -1;
        set_err(c, "%s: %s", what, c->vg ? "virtual group" : g_nccl.GetErrorString(r));
    }
    return c->exch_error;
}

// recv[r * n + i] = send_r[i] (n doubles per rank)
static int coll_allgather(mmot_ctx *c, const double *send, double *recv, size_t n, cudaStream_t s) {
    if (c->vg) {
        mmot_vgroup *g = c->vg;
        const int r = c->rank;
        g->src[r] = send;
        if (cudaEventRecord(g->ready[r], s) != cudaSuccess) return coll_fail(c, "cudaEventRecord", 0);
        g->barrier();
        for (int j = 0; j < g->world; ++j) {
            cudaStreamWaitEvent(s, g->ready[j], 0);
            cudaMemcpyAsync(recv + (size_t)j * n, g->src[j], n * sizeof(double), cudaMemcpyDeviceToDevice, s);
        }
        cudaEventRecord(g->done[r], s);
        g->barrier();  // every rank has read every send buffer before any rank overwrites its own
        for (int j = 0; j < g->world; ++j)
            if (j != r) cudaStreamWaitEvent(s, g->done[j], 0);
        if (cudaGetLastError() != cudaSuccess) return coll_fail(c, "virtual all-gather", 0);
        return 0;
    }
    const nccl_result rr = g_nccl.AllGather(send, recv, n, kNcclFloat64, c->comm, s);
    return rr ? coll_fail(c, "ncclAllGather", rr) : 0;
}

// dev[0..n) <- sum (op 0, doubles) or max (op 1, ints) over the ranks, in place
static int coll_allreduce(mmot_ctx *c, void *dev, int n, int op, cudaStream_t s) {
    if (c->vg) {
        mmot_vgroup *g = c->vg;
        const int r = c->rank;
        g->src[r] = dev;
        if (cudaEventRecord(g->ready[r], s) != cudaSuccess) return coll_fail(c, "cudaEventRecord", 0);
        g->barrier();
        mmot::VPtrs vp{};
        for (int j = 0; j < g->world; ++j) {
            vp.p[j] = g->src[j];
            cudaStreamWaitEvent(s, g->ready[j], 0);
        }
        int64_t dummy = 0;
        mmot::launch_vreduce(vp, g->world, n, op, c->vg_tmp, s, &dummy);
        c->launches += dummy;
        cudaEventRecord(g->done[r], s);
        g->barrier();
        for (int j = 0; j < g->world; ++j)
            if (j != r) cudaStreamWaitEvent(s, g->done[j], 0);
        cudaMemcpyAsync(dev, c->vg_tmp, (size_t)n * (op == 0 ? sizeof(double) : sizeof(int)), cudaMemcpyDeviceToDevice, s);
        if (cudaGetLastError() != cudaSuccess) return coll_fail(c, "virtual all-reduce", 0);
        return 0;
    }
    const nccl_result rr = g_nccl.AllReduce(dev, dev, (size_t)n, op == 0 ? kNcclFloat64 : kNcclInt32,
                                            op == 0 ? kNcclSum : kNcclMax, c->comm, s);
    return rr ? coll_fail(c, "ncclAllReduce", rr) : 0;
}

// All-gather of the whole-shard operators ([2][SZ] elements) on the context stream (called from
// inside the scan, between up-sweep and down-sweep).
static void shard_exchange(void *vctx, size_t n, cudaStream_t s) {
    mmot_ctx *c = static_cast<mmot_ctx *>(vctx);
    const size_t SZ = (size_t)c->l * (1 << (c->l - 1));
    coll_allgather(c, c->shard_mem, c->shard_mem + 2 * SZ * 2, n, s);
}

static bool multi_rank(const mmot_ctx *c) { return c->sharded && c->world > 1; }

// Sum a device double over the ranks (residual, cost) in place.
static mmot_status shard_allreduce(mmot_ctx *c, double *dev, int n = 1) {
    if (!multi_rank(c)) return MMOT_OK;
    return coll_allreduce(c, dev, n, 0, c->stream) ? MMOT_ENCCL : MMOT_OK;
}

// Max of the device ints stop, status, fail_iter (, iters_done, converged) over the ranks, so every
// rank stops, and reports, together.
static mmot_status shard_agree(mmot_ctx *c, int *first, int n) {
    if (!multi_rank(c)) return MMOT_OK;
    return coll_allreduce(c, first, n, 1, c->stream) ? MMOT_ENCCL : MMOT_OK;
}

// ---------------------------------------------------------------------------------------
static Plan make_plan(mmot_ctx *c, int k, const double *const *lin, const double *mu, double *out, int iter) {
    Plan p{};
    p.NB = c->l - 1;
    p.N = c->N;
    p.P = c->P;
    p.nchunks = c->nchunks;
    // Bound marginals in CYCLIC order k+1, k+2, ..., k+l-1 (mod l).  J_k is symmetric in its
    // bound vectors, and with this order the bound set of update k+1 is this one shifted by one
    // slot with the new phi_k appended, so the fused next-update operators need no selects.
    for (int b = 0; b < c->l - 1; ++b) p.bound[b] = lin[(k + 1 + b) % c->l];
    p.phik = lin[k];
    p.muk = mu;
    p.outk = out;
    p.W = c->W;
    p.nlev = c->nlev;
    for (int i = 0; i < c->nlev; ++i) {
        p.nlev_n[i] = c->nlev_n[i];
        p.ops_f[i] = c->ops_f[i];
        p.ops_b[i] = c->ops_b[i];
        p.car_f[i] = c->car_f[i];
        p.car_b[i] = c->car_b[i];
    }
    p.car_bi = c->car_bi;
    p.sw = c->sw ? 1 : 0;
    for (int i = 0; i < c->nlev; ++i) {
        p.rxe_f[i] = c->rxe_f[i];
        p.rxe_b[i] = c->rxe_b[i];
        p.rcar_f[i] = c->rcar_f[i];
        p.rcar_b[i] = c->rcar_b[i];
    }
    p.nchp = c->nchp;
    if (c->sw && mu) p.muk = c->mu_t[k];
    if (c->sharded) {
        const int M = 1 << (c->l - 1);
        const size_t SZ = (size_t)c->l * M;  // (NB+1) * 2^NB, in Dual units below
        p.exch = shard_exchange;
        p.exch_ctx = c;
        p.agg_send = c->shard_mem;
        p.agg_all = c->shard_mem + 2 * SZ * 2;
        p.rank_car = c->shard_mem + 2 * SZ * 2 + (size_t)c->world * 2 * SZ * 2;
        p.world = c->world;
        p.rank = c->rank;
    }
    p.lam = c->pts_lam;
    p.hx = c->pts_hx;
    p.partial = c->partial;
    p.stop = &c->dsc->stop;
    p.status = &c->dsc->status;
    p.fail_iter = &c->dsc->fail_iter;
    p.iter = iter;
    if (iter > 0) p.sweep = &c->dsc->sweep;  // inside a solve
    if (c->sw) {
        p.sw_end = c->sw_end;
        p.guard = &c->dsc->guard;
    }
    if (c->ls_on) p.ls = &c->ls;
    return p;
}

static mmot_status reset_scalars(mmot_ctx *c) {
    CK(c, cudaMemsetAsync(c->dsc, 0, sizeof(DevScalars), c->stream));
    return MMOT_OK;
}

// Resolve the linear scalings used by the kernels (convert from log if needed).
static mmot_status to_linear(mmot_ctx *c, const void *const *u, const double **lin) {
    for (int q = 0; q < c->l; ++q) {
        if (!u[q]) { set_err(c, "u[%d] is NULL", q); return MMOT_EINVAL; }
        if (c->sw) {
            CK(c, mmot::launch_to_t(static_cast<const double *>(u[q]), c->lin[q], c->N, c->P, c->nchunks, c->nchp,
                                    c->opts.repr == MMOT_LOG ? 1 : 0, c->stream, &c->launches));
            lin[q] = c->lin[q];
        } else if (c->opts.repr == MMOT_LOG) {
            CK(c, mmot::launch_exp(static_cast<const double *>(u[q]), c->lin[q], c->N, c->stream, &c->launches));
            lin[q] = c->lin[q];
        } else {
            lin[q] = static_cast<const double *>(u[q]);
        }
    }
    return MMOT_OK;
}

static mmot_status sync_report(mmot_ctx *c) {
    CK(c, cudaMemcpyAsync(c->hsc, c->dsc, sizeof(DevScalars), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    return MMOT_OK;
}

// Single-walk precision guard tripped (non-smooth scalings): the call is redone on a
// two-walk context of the same problem (created on first use; fp64 internal vectors).  Sharded
// contexts cannot switch families alone and report MMOT_EPRECISION on every rank instead.
static mmot_status ensure_fallback(mmot_ctx *c) {
    if (c->fb) return MMOT_OK;
    mmot_opts o = c->opts;
    o.kernel = MMOT_KERNEL_TWO_WALK;
    o.chunk = 0;
    mmot_status st = create_single(c->l, c->N, c->eta, c->grid, MMOT_F64, &o, c->stream, &c->fb, false);
    if (st) set_err(c, "two-walk fallback context: %s", mmot_last_error(nullptr));
    else c->fb->prof = c->prof;
    return st;
}

static mmot_status guard_tripped(mmot_ctx *c) {
    set_err(c, "single-walk precision guard: a walked suffix state lost accuracy (non-smooth scalings); "
               "use MMOT_KERNEL_TWO_WALK");
    return MMOT_EPRECISION;
}

// NEXT-1: the all-marginals residual pass is available on two-walk contexts with l <= 5 (the DP over
// all l scalings has 2^l states, NB = l <= 5 kernels), uniform grids, one process.  Lazily allocates
// its own chain layout (P from the NB = l checkpoint limits) and scan workspace.
static bool ensure_allres(mmot_ctx *c) {
    if (c->all_state) return c->all_state > 0;
    c->all_state = -1;
    if (c->sw || c->sharded || c->pts_lam || c->batched || c->stable || c->g2 || c->l < 2 || c->l > 5 ||
        getenv("MMOT_NO_ALLRES") != nullptr)
        return false;
    const int NB = c->l;
    const int64_t pmax = mmot::chunk_max(NB);
    const int64_t q = mmot::sub_q(NB);
    int64_t P = (c->N + 148 * 256 - 1) / (148 * 256);
    if (NB >= 4) P = pmax;
    P = ((P + q - 1) / q) * q;
    P = std::max<int64_t>(q, std::min<int64_t>(P, pmax));
    c->all_P = P;
    c->all_nchunks = (c->N + P - 1) / P;
    int64_t n = c->all_nchunks;
    c->all_nlev = 0;
    const int grp = mmot::group_of(NB);
    while (true) {
        c->all_nlev_n[c->all_nlev++] = n;
        if (n <= grp || c->all_nlev == mmot::kMaxLevels) break;
        n = (n + grp - 1) / grp;
    }
    const int M = 1 << NB;
    const size_t opsz = (size_t)(NB + 1) * M, carsz = M;
    size_t total = 0;
    size_t off_ops[mmot::kMaxLevels], off_car[mmot::kMaxLevels];
    for (int i = 0; i < c->all_nlev; ++i) {
        off_ops[i] = total;
        total += 2 * (size_t)c->all_nlev_n[i] * opsz;
        off_car[i] = total;
        total += 2 * (size_t)c->all_nlev_n[i] * carsz;
    }
    const size_t off_bi = total;
    total += (size_t)c->all_nchunks * carsz;
    const size_t off_part = total;
    total += (size_t)c->all_nchunks;
    if (cudaMalloc(&c->all_mem, total * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    double *base = static_cast<double *>(c->all_mem);
    for (int i = 0; i < c->all_nlev; ++i) {
        c->all_ops_f[i] = base + off_ops[i];
        c->all_ops_b[i] = base + off_ops[i] + (size_t)c->all_nlev_n[i] * opsz;
        c->all_car_f[i] = base + off_car[i];
        c->all_car_b[i] = base + off_car[i] + (size_t)c->all_nlev_n[i] * carsz;
    }
    c->all_car_bi = base + off_bi;
    c->all_partial = base + off_part;
    c->all_state = 1;
    return true;
}

static Plan make_plan_all(mmot_ctx *c, const double *const *lin, const double *const *mu, int iter) {
    Plan p{};
    p.NB = c->l;
    p.N = c->N;
    p.P = c->all_P;
    p.nchunks = c->all_nchunks;
    for (int b = 0; b < c->l; ++b) p.bound[b] = lin[b];  // the DP over ALL l scalings, index order
    for (int k = 0; k + 1 < c->l; ++k) p.mus[k] = mu[k];
    p.W = c->W;
    p.nlev = c->all_nlev;
    for (int i = 0; i < c->all_nlev; ++i) {
        p.nlev_n[i] = c->all_nlev_n[i];
        p.ops_f[i] = c->all_ops_f[i];
        p.ops_b[i] = c->all_ops_b[i];
        p.car_f[i] = c->all_car_f[i];
        p.car_b[i] = c->all_car_b[i];
    }
    p.car_bi = c->all_car_bi;
    p.nchp = (c->all_nchunks + 31) / 32 * 32;
    p.partial = c->all_partial;
    p.stop = &c->dsc->stop;
    p.status = &c->dsc->status;
    p.fail_iter = &c->dsc->fail_iter;
    p.iter = iter;
    if (iter > 0) p.sweep = &c->dsc->sweep;
    return p;
}

// Host-side state of the update sequence: which chain operators / restricted-scan elements the
// previous product left behind (they decide the launch configuration of the next update).
struct SweepState {
    int ops_for = -1;      // bound set whose chain operators are in ops level 0
    bool rx_ready = false; // the previous update wrote this update's affine elements
    int cur = 0;           // restricted scan: which carry set is current
    bool operator==(const SweepState &o) const { return ops_for == o.ops_for && rx_ready == o.rx_ready && cur == o.cur; }
};

// Enqueue sweep t (l fused updates, then the residual check or the sweep counter).
static mmot_status enqueue_sweep(mmot_ctx *c, int t, bool check, double tol, const double *const *lin,
                                 const double *const *mu, SweepState &ss) {
    const int l = c->l;
    const bool rx = c->rx && (!c->sharded || c->nlev >= 2);
    void *cf[2] = {c->car_f[0], c->carB_f}, *cb[2] = {c->car_bi, c->carB_bi};
    for (int k = 0; k < l; ++k) {
        // fused update: scan (+ operators only if not produced by the previous update),
        // apply phi_k <- mu_k / J_k and build the operators of update k+1 in the same walk
        Plan p = make_plan(c, k, lin, mu[k], const_cast<double *>(lin[k]), t);
        if (rx) {
            p.car_f[0] = cf[ss.cur];
            p.car_bi = cb[ss.cur];
            p.ncar_f = cf[1 - ss.cur];
            p.ncar_bi = cb[1 - ss.cur];
            p.nxr = 1;
            p.rx_scan = ss.rx_ready ? 1 : 0;
        }
        CK(c, mmot::launch_product(p, mmot::MODE_UPD, c->stream, &c->launches, prof_events(c, mmot::MODE_UPD),
                                   rx ? !ss.rx_ready : ss.ops_for != k, true));
        // l = 6 / non-uniform grids: next-update operators are not fused
        ss.ops_for = (l <= 5 && !c->pts_lam) ? (k + 1) % l : -1;
        if (rx) {
            ss.rx_ready = true;
            ss.cur = 1 - ss.cur;
        }
    }
    CK(c, mmot::launch_sweep_done(&c->dsc->sweep, &c->dsc->iters_done, &c->dsc->stop, c->stream, &c->launches));
    if (check && ensure_allres(c)) {
        // NEXT-1: every marginal from one pass of the 2^l-state DP (its own workspace, so this
        // update sequence's operators and carries stay valid)
        Plan p = make_plan_all(c, lin, mu, t);
        CK(c, mmot::launch_product(p, mmot::MODE_ALLRES, c->stream, &c->launches, prof_events(c, mmot::MODE_RES)));
        CK(c, mmot::launch_sum(c->all_partial, c->all_nchunks, &c->dsc->res_acc, 1.0, 0, &c->dsc->stop, c->stream,
                               &c->launches));
        ++c->allres_checks;
        mmot_status st = shard_allreduce(c, &c->dsc->res_acc);
        if (st) return st;
        CK(c, mmot::launch_resid_finish(&c->dsc->res_acc, tol, &c->dsc->sweep, &c->dsc->resid, &c->dsc->iters_done,
                                        &c->dsc->converged, &c->dsc->stop, c->stream, &c->launches));
    } else if (check) {
        for (int k = 0; k + 1 < l; ++k) {
            Plan p = make_plan(c, k, lin, mu[k], nullptr, t);
            CK(c, mmot::launch_product(p, mmot::MODE_RES, c->stream, &c->launches, prof_events(c, mmot::MODE_RES)));
            ss.ops_for = -1;      // the residual products overwrote the chain operators
            ss.rx_ready = false;  // ... and the level-0 carries: the next update starts from a full scan
            ss.cur = 0;
            // (the lane-state family leaves one partial per 32-point chain)
            CK(c, mmot::launch_sum(c->partial, c->ls_on ? c->ls.C : c->nchunks, &c->dsc->res_acc, 1.0, k > 0,
                                   &c->dsc->stop, c->stream, &c->launches));
        }
        mmot_status st = shard_allreduce(c, &c->dsc->res_acc);
        if (st) return st;
        CK(c, mmot::launch_resid_finish(&c->dsc->res_acc, tol, &c->dsc->sweep, &c->dsc->resid, &c->dsc->iters_done,
                                        &c->dsc->converged, &c->dsc->stop, c->stream, &c->launches));
    }
    return MMOT_OK;
}

// Device-resident loop: a CUDA graph whose WHILE node runs `n` periods of `period` sweeps (each
// ending with the residual check when tol > 0) until the periods are done or the device stop flag is
// set -- one graph launch, no host round trip per sweep.  The graph bakes in the context's vectors,
// so it is rebuilt when the caller's pointers (or the schedule) change.
static mmot_status run_graph_loop(mmot_ctx *c, int period, int n, bool check, double tol, const double *const *lin,
                                  const double *const *mu, const SweepState &ss0) {
    const void *key[2 * mmot::kMaxL + 4] = {nullptr};
    for (int q = 0; q < c->l; ++q) {
        key[q] = lin[q];
        key[mmot::kMaxL + q] = mu[q];
    }
    key[2 * mmot::kMaxL] = reinterpret_cast<const void *>((intptr_t)period);
    key[2 * mmot::kMaxL + 1] = reinterpret_cast<const void *>((intptr_t)(check ? 1 : 0));
    key[2 * mmot::kMaxL + 2] = reinterpret_cast<const void *>((intptr_t)(ss0.ops_for + 8 * ss0.rx_ready + 64 * ss0.cur));
    double tkey = check ? tol : 0.0;
    memcpy(&key[2 * mmot::kMaxL + 3], &tkey, sizeof(tkey) <= sizeof(void *) ? sizeof(tkey) : sizeof(void *));
    if (!c->g_exec || memcmp(key, c->g_key, sizeof key) != 0) {
        if (c->g_exec) { cudaGraphExecDestroy(c->g_exec); c->g_exec = nullptr; }
        if (c->g_graph) { cudaGraphDestroy(c->g_graph); c->g_graph = nullptr; }
        cudaGraph_t g = nullptr;
        CK(c, cudaGraphCreate(&g, 0));
        c->g_graph = g;
        cudaGraphConditionalHandle h;
        CK(c, cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams np = {};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = h;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        CK(c, cudaGraphAddNode(&node, g, nullptr, 0, &np));
        cudaGraph_t body = np.conditional.phGraph_out[0];
        const int64_t l0 = c->launches, a0 = c->allres_checks;
        // capture on a private stream (the caller's may be the legacy default stream, which cannot
        // be captured); the graph is launched on the context stream
        if (!c->cap_stream) CK(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
        cudaStream_t user = c->stream;
        c->stream = c->cap_stream;
        mmot_status st = MMOT_OK;
        cudaError_t e = cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) st = MMOT_ECUDA;
        SweepState ss = ss0;
        for (int i = 0; i < period && !st; ++i) st = enqueue_sweep(c, 1, check && i + 1 == period, tol, lin, mu, ss);
        if (!st) {
            e = mmot::launch_loop_cond(h, &c->dsc->g_done, &c->dsc->g_n, &c->dsc->stop, c->stream, &c->launches);
            if (e != cudaSuccess) st = MMOT_ECUDA;
        }
        cudaGraph_t cap = nullptr;
        e = cudaStreamEndCapture(c->stream, &cap);
        c->stream = user;
        if (st || e != cudaSuccess) {
            // capture refused something: forget the graph, clear the error, let the host loop run
            cudaGetLastError();
            c->launches = l0;
            c->graph_broken = true;
            return MMOT_EUNSUPPORTED;
        }
        if (!(ss == ss0)) { set_err(c, "internal: graph period does not return to its start state"); return MMOT_ECUDA; }
        c->g_launches = c->launches - l0;
        c->launches = l0;
        c->g_allres = c->allres_checks - a0;  // all-marginals checks per period
        c->allres_checks = a0;
        CK(c, cudaGraphInstantiate(&c->g_exec, g, 0));
        memcpy(c->g_key, key, sizeof key);
    }
    c->hstop[1] = n;
    CK(c, cudaMemsetAsync(&c->dsc->g_done, 0, sizeof(int), c->stream));
    CK(c, cudaMemcpyAsync(&c->dsc->g_n, &c->hstop[1], sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaGraphLaunch(c->g_exec, c->stream));
    c->launches += c->g_launches * n;  // upper bound: periods after a stop exit at the condition
    c->allres_checks += c->g_allres * n;
    ++c->graph_solves;
    return MMOT_OK;
}

static mmot_status sinkhorn_impl(mmot_ctx *c, const double *const *mu, int iters, double tol, void *const *u,
                                 mmot_report *rep) {
    const int l = c->l;
    mmot_status st = reset_scalars(c);
    if (st) return st;
    c->exch_error = 0;
    // data checks (P:75 marginals are probability vectors; SPEC S:77 error vocabulary); a sharded
    // context tests the mass of the whole marginal and all ranks adopt the worst status.  The
    // single-walk family fuses them into its layout conversion (one pass over each input).
    double *lin[mmot::kMaxL];
    for (int q = 0; q < l; ++q) {
        const int is_log = c->opts.repr == MMOT_LOG ? 1 : 0;
        if (c->sw) {
            CK(c, mmot::launch_to_t(static_cast<const double *>(u[q]), c->lin[q], c->N, c->P, c->nchunks, c->nchp,
                                    is_log, c->stream, &c->launches, &c->dsc->flags[l + q], nullptr, is_log));
            CK(c, mmot::launch_to_t(mu[q], c->mu_t[q], c->N, c->P, c->nchunks, c->nchp, 0, c->stream, &c->launches,
                                    &c->dsc->flags[q], &c->dsc->mass[q], 0));
            lin[q] = c->lin[q];
            continue;
        }
        CK(c, mmot::launch_check(mu[q], c->N, 0, &c->dsc->flags[q], &c->dsc->mass[q], c->stream, &c->launches));
        CK(c, mmot::launch_check(static_cast<const double *>(u[q]), c->N, is_log, &c->dsc->flags[l + q], nullptr,
                                 c->stream, &c->launches));
        if (is_log) {
            CK(c, mmot::launch_exp(static_cast<const double *>(u[q]), c->lin[q], c->N, c->stream, &c->launches));
            lin[q] = c->lin[q];
        } else {
            lin[q] = static_cast<double *>(u[q]);
        }
    }
    if ((st = shard_allreduce(c, c->dsc->mass, l))) return st;
    CK(c, mmot::launch_check_finish(c->dsc->flags, c->dsc->mass, 2 * l, l, &c->dsc->status, &c->dsc->stop,
                                    &c->dsc->fail_iter, c->stream, &c->launches));
    if ((st = shard_agree(c, &c->dsc->stop, 3))) return st;
    if (!c->sw && c->opts.repr == MMOT_LINEAR && can_stabilise(c)) {
        // the updates rewrite u in place: keep the input for a stabilised redo
        if (!c->u_save) CK(c, cudaMalloc(&c->u_save, (size_t)l * c->N * sizeof(double)));
        for (int q = 0; q < l; ++q)
            CK(c, cudaMemcpyAsync(c->u_save + (size_t)q * c->N, u[q], (size_t)c->N * sizeof(double),
                                  cudaMemcpyDeviceToDevice, c->stream));
    }
    const int check_every = c->opts.check_every > 0 ? c->opts.check_every : 1;
    const bool rx = c->rx && (!c->sharded || c->nlev >= 2);
    SweepState ss;
    // Device-resident loop (CUDA graph, WHILE node) for single-process contexts when not profiling:
    // tol > 0 -- periods of check_every sweeps ending with the residual check, from the solve's
    // start state; tol <= 0 -- after `warm` host-issued sweeps the update sequence is periodic with
    // `period` sweeps (the restricted scan alternates two carry sets, so odd l needs two sweeps).
    const bool graph = !c->sharded && !c->prof && !c->graph_broken && iters >= 4 && getenv("MMOT_NO_GRAPH") == nullptr;
    int t = 1;
    if (graph) {
        const int period = tol > 0 ? check_every : ((rx && (l & 1)) ? 2 : 1);
        // (the all-marginals check leaves the update sequence's state alone, so with it the periods
        // start after one host-issued period, like the fixed-sweep case)
        const int warm = tol > 0 && !ensure_allres(c) ? 0 : period;
        for (; t <= warm; ++t)
            if ((st = enqueue_sweep(c, t, tol > 0 && (t % check_every == 0 || t == iters), tol, lin, mu, ss))) return st;
        const int n = (iters - warm) / period;
        if (n >= 1) {
            st = run_graph_loop(c, period, n, tol > 0, tol, lin, mu, ss);
            if (st == MMOT_OK) t += n * period;
            else if (st != MMOT_EUNSUPPORTED) return st;  // EUNSUPPORTED: not capturable, host loop
        }
    }
    bool poll_pending = false;
    for (; t <= iters; ++t) {
        // asynchronous early exit: the device stop flag is polled without blocking
        if (poll_pending && cudaEventQuery(c->poll_ev) == cudaSuccess) {
            poll_pending = false;
            if (*c->hstop) break;
        }
        const bool check = tol > 0 && (t % check_every == 0 || t == iters);
        if ((st = enqueue_sweep(c, t, check, tol, lin, mu, ss))) return st;
        if (tol > 0 && multi_rank(c) && t % 8 == 0) {
            // sharded: the early exit must be collective -- agree on the stop flag, then read it
            // synchronously, so every rank leaves the loop after the same sweep and issues the
            // same collectives afterwards
            if ((st = shard_agree(c, &c->dsc->stop, 3))) return st;
            CK(c, cudaMemcpyAsync(c->hstop, &c->dsc->stop, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
            CK(c, cudaStreamSynchronize(c->stream));
            if (*c->hstop) break;
        } else if (tol > 0 && !multi_rank(c) && !poll_pending && (t % 8 == 0)) {
            CK(c, cudaMemcpyAsync(c->hstop, &c->dsc->stop, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
            CK(c, cudaEventRecord(c->poll_ev, c->stream));
            poll_pending = true;
        }
    }
    // decided before u is written, so that a redo starts from this call's input: the single-walk
    // precision guard (-> two-walk family) and products beyond the fp64 range (-> stabilised family)
    if ((st = shard_agree(c, &c->dsc->stop, 6))) return st;
    if ((st = sync_report(c))) return st;
    if (c->exch_error) return MMOT_ENCCL;
    // (an EOVERFLOW of the single walk may itself be the lost precision: redo it on two-walk first)
    if (c->sw && c->hsc->guard && (!c->hsc->status || c->hsc->status == MMOT_EOVERFLOW)) {
        if (c->sharded) return guard_tripped(c);
        ++c->fallbacks;
        if ((st = ensure_fallback(c))) return st;
        return sinkhorn_impl(c->fb, mu, iters, tol, u, rep);
    }
    if (c->hsc->status == MMOT_EOVERFLOW && can_stabilise(c)) {
        ++c->st_fallbacks;
        if ((st = ensure_stable(c))) return st;
        const void *uin[mmot::kMaxL];
        for (int q = 0; q < l; ++q) uin[q] = c->u_save ? c->u_save + (size_t)q * c->N : u[q];
        return st_sinkhorn(c->st_fb, mu, iters, tol, uin, u, rep, nullptr);
    }
    if (c->sw) {
        for (int q = 0; q < l; ++q)
            CK(c, mmot::launch_from_t(c->lin[q], static_cast<double *>(u[q]), c->N, c->P, c->nchunks, c->nchp,
                                      c->opts.repr == MMOT_LOG ? 2 : 0, c->stream, &c->launches));
    } else if (c->opts.repr == MMOT_LOG) {
        for (int q = 0; q < l; ++q)
            CK(c, mmot::launch_log(c->lin[q], static_cast<double *>(u[q]), c->N, c->stream, &c->launches));
    }
    CK(c, cudaStreamSynchronize(c->stream));
    const DevScalars &h = *c->hsc;
    if (rep) {
        rep->iters_done = h.iters_done;
        rep->residual = tol > 0 && h.iters_done > 0 ? h.resid : NAN;
        rep->converged = h.converged;
        rep->status = h.status;
        rep->fail_iter = h.status ? h.fail_iter : -1;
    }
    if (h.status) set_err(c, "%s (sweep %d)", mmot_strerror((mmot_status)h.status), h.fail_iter);
    return (mmot_status)h.status;
}

// ---------------------------------------------------------------------------------------
// 2-D grids (grid2d.cu; §4.1).  Free marginal k, bound marginals k+1, k+2 (mod 3).
static mmot::G2Plan g2_plan(mmot_ctx *c, int k, const double *const *lin, const double *mu, double *out, int iter,
                            bool transposed = false) {
    mmot::G2Plan p{};
    const int64_t N = transposed ? c->g2M : c->g2N, M = transposed ? c->g2N : c->g2M;
    const double hi = transposed ? c->g2h2 : c->g2h1, ho = transposed ? c->g2h1 : c->g2h2;
    p.N = N;
    p.M = M;
    for (int a = 0; a <= mmot::kMaxL; ++a) {
        const int e = a <= 3 ? a * (3 - a) : 0;
        p.Wi.e[a] = (double)e;
        p.Wi.w[a] = a <= 3 ? exp(-(double)e * hi / c->eta) : 0.0;
    }
    p.wo1 = exp(-2.0 * ho / c->eta);  // lambda2^{1*2}
    p.wo2 = p.wo1;                    // lambda2^{2*1}
    p.a = lin[(k + 1) % 3];
    p.b = lin[(k + 2) % 3];
    p.phik = lin[k];
    p.muk = mu;
    p.outk = out;
    const int64_t n = c->N;
    p.Fa = c->g2_mem;
    p.Fb = c->g2_mem + n;
    p.Ga = c->g2_mem + 2 * n;
    p.Gb = c->g2_mem + 3 * n;
    mmot::Dual *T = static_cast<mmot::Dual *>(c->g2_T);
    p.Y = T;
    p.st = T + 6 * n;
    p.Gab = T + 24 * n;
    p.partial = c->partial;
    p.status = &c->dsc->status;
    p.stop = &c->dsc->stop;
    p.fail_iter = &c->dsc->fail_iter;
    p.iter = iter;
    return p;
}

static mmot_status g2_linear(mmot_ctx *c, const void *const *u, const double **lin) {
    for (int q = 0; q < c->l; ++q) {
        if (!u[q]) { set_err(c, "u[%d] is NULL", q); return MMOT_EINVAL; }
        if (c->opts.repr == MMOT_LOG) {
            CK(c, mmot::launch_exp(static_cast<const double *>(u[q]), c->lin[q], c->N, c->stream, &c->launches));
            lin[q] = c->lin[q];
        } else {
            lin[q] = static_cast<const double *>(u[q]);
        }
    }
    return MMOT_OK;
}

static mmot_status g2_sinkhorn(mmot_ctx *c, const double *const *mu, int iters, double tol, void *const *u,
                               mmot_report *rep) {
    const int l = c->l;
    mmot_status st = reset_scalars(c);
    if (st) return st;
    for (int q = 0; q < l; ++q) {
        CK(c, mmot::launch_check(mu[q], c->N, 0, &c->dsc->flags[q], &c->dsc->mass[q], c->stream, &c->launches));
        CK(c, mmot::launch_check(static_cast<const double *>(u[q]), c->N, c->opts.repr == MMOT_LOG ? 1 : 0,
                                 &c->dsc->flags[l + q], nullptr, c->stream, &c->launches));
    }
    CK(c, mmot::launch_check_finish(c->dsc->flags, c->dsc->mass, 2 * l, l, &c->dsc->status, &c->dsc->stop,
                                    &c->dsc->fail_iter, c->stream, &c->launches));
    const double *lin[mmot::kMaxL];
    if ((st = g2_linear(c, const_cast<const void *const *>(u), lin))) return st;
    const int check_every = c->opts.check_every > 0 ? c->opts.check_every : 1;
    bool poll_pending = false;
    for (int t = 1; t <= iters; ++t) {
        if (poll_pending && cudaEventQuery(c->poll_ev) == cudaSuccess) {
            poll_pending = false;
            if (*c->hstop) break;
        }
        for (int k = 0; k < l; ++k) {
            mmot::G2Plan p = g2_plan(c, k, lin, mu[k], const_cast<double *>(lin[k]), t);
            CK(c, mmot::launch_g2_product(p, mmot::MODE_UPD, c->stream, &c->launches));
        }
        CK(c, mmot::launch_sweep_done(&c->dsc->sweep, &c->dsc->iters_done, &c->dsc->stop, c->stream, &c->launches));
        if (tol > 0 && (t % check_every == 0 || t == iters)) {
            for (int k = 0; k + 1 < l; ++k) {
                mmot::G2Plan p = g2_plan(c, k, lin, mu[k], nullptr, t);
                CK(c, mmot::launch_g2_product(p, mmot::MODE_RES, c->stream, &c->launches));
                CK(c, mmot::launch_sum(c->partial, c->g2N, &c->dsc->res_acc, 1.0, k > 0, &c->dsc->stop, c->stream,
                                       &c->launches));
            }
            CK(c, mmot::launch_resid_finish(&c->dsc->res_acc, tol, &c->dsc->sweep, &c->dsc->resid, &c->dsc->iters_done,
                                            &c->dsc->converged, &c->dsc->stop, c->stream, &c->launches));
            if (!poll_pending && t % 8 == 0) {
                CK(c, cudaMemcpyAsync(c->hstop, &c->dsc->stop, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
                CK(c, cudaEventRecord(c->poll_ev, c->stream));
                poll_pending = true;
            }
        }
    }
    if (c->opts.repr == MMOT_LOG)
        for (int q = 0; q < l; ++q)
            CK(c, mmot::launch_log(lin[q], static_cast<double *>(u[q]), c->N, c->stream, &c->launches));
    if ((st = sync_report(c))) return st;
    const DevScalars &h = *c->hsc;
    if (rep) {
        rep->iters_done = h.iters_done;
        rep->residual = tol > 0 && h.iters_done > 0 ? h.resid : NAN;
        rep->converged = h.converged;
        rep->status = h.status;
        rep->fail_iter = h.status ? h.fail_iter : -1;
    }
    if (h.status) set_err(c, "%s (sweep %d)", mmot_strerror((mmot_status)h.status), h.fail_iter);
    return (mmot_status)h.status;
}

static mmot_status g2_marginal(mmot_ctx *c, int k, const void *const *u, void *out) {
    mmot_status st = reset_scalars(c);
    if (st) return st;
    const double *lin[mmot::kMaxL];
    if ((st = g2_linear(c, u, lin))) return st;
    mmot::G2Plan p = g2_plan(c, k, lin, nullptr, static_cast<double *>(out), 0);
    CK(c, mmot::launch_g2_product(p, mmot::MODE_MARG, c->stream, &c->launches));
    return MMOT_OK;
}

// W = h1 <phi_3, hatJ^(1)> + h2 <phi_3, hatJ^(2)>: the lambda1 tangent on the mesh, the lambda2
// tangent on the transposed mesh (reading A21; the paper omits the 2-D cost product).
static mmot_status g2_cost(mmot_ctx *c, const void *const *u, double *W) {
    mmot_status st = reset_scalars(c);
    if (st) return st;
    const double *lin[mmot::kMaxL];
    if ((st = g2_linear(c, u, lin))) return st;
    mmot::G2Plan p = g2_plan(c, 2, lin, nullptr, nullptr, 0);
    CK(c, mmot::launch_g2_product(p, mmot::MODE_COST, c->stream, &c->launches));
    CK(c, mmot::launch_sum(c->partial, c->g2N, &c->dsc->W, c->g2h1, 0, &c->dsc->stop, c->stream, &c->launches));
    const double *tr[mmot::kMaxL];
    for (int q = 0; q < 3; ++q) {
        double *dst = c->g2_mem + (4 + q) * c->N;
        CK(c, mmot::launch_g2_transpose(lin[q], dst, c->g2N, c->g2M, c->stream, &c->launches));
        tr[q] = dst;
    }
    mmot::G2Plan pt = g2_plan(c, 2, tr, nullptr, nullptr, 0, true);
    CK(c, mmot::launch_g2_product(pt, mmot::MODE_COST, c->stream, &c->launches));
    CK(c, mmot::launch_sum(c->partial, c->g2M, &c->dsc->W, c->g2h2, 1, &c->dsc->stop, c->stream, &c->launches));
    if ((st = sync_report(c))) return st;
    *W = c->hsc->W;
    return (mmot_status)c->hsc->status;
}

// MMOT_F32 contexts take float marginals and write float marginal outputs; the scans run in fp64
// on widened copies (on B200 an fp32 scan would need per-state exponents and issue
// more instructions than the fp64 one).
static int64_t io_elems(const mmot_ctx *c) { return c->N * (c->batched || c->stable ? c->batch : 1); }
static mmot_status f32_ensure(mmot_ctx *c) {
    if (c->f32_mem) return MMOT_OK;
    CK(c, cudaMalloc(&c->f32_mem, (size_t)(c->l + 1) * io_elems(c) * sizeof(double)));
    return MMOT_OK;
}
static mmot_status f32_widen(mmot_ctx *c, const void *const *marginals, const double **mu) {
    mmot_status st = f32_ensure(c);
    if (st) return st;
    const int64_t n = io_elems(c);
    for (int q = 0; q < c->l; ++q) {
        double *dst = c->f32_mem + (size_t)q * n;
        CK(c, mmot::launch_convert(marginals[q], dst, n, 1, c->stream, &c->launches));
        mu[q] = dst;
    }
    return MMOT_OK;
}

extern "C" {

static mmot_status marginal_f64(mmot_ctx *c, int k, const void *const *u, void *out);

mmot_status mmot_marginal(mmot_ctx *c, int k, const void *const *u, void *out) {
    if (!c || !u || !out) { set_err(c, "NULL argument"); return MMOT_EINVAL; }
    if (k < 0 || k >= c->l) { set_err(c, "k=%d outside [0,%d)", k, c->l); return MMOT_EINVAL; }
    cudaSetDevice(c->device);
    if (c->dt != MMOT_F32) return marginal_f64(c, k, u, out);
    mmot_status st = f32_ensure(c);
    if (st) return st;
    double *o64 = c->f32_mem + (size_t)c->l * io_elems(c);
    st = marginal_f64(c, k, u, o64);
    if (st) return st;
    CK(c, mmot::launch_convert(o64, out, io_elems(c), 0, c->stream, &c->launches));
    return MMOT_OK;
}

static mmot_status marginal_f64(mmot_ctx *c, int k, const void *const *u, void *out) {
    if (c->g2) return g2_marginal(c, k, u, out);
    if (c->stable) return st_marginal(c, k, u, out);
    if (c->batched && c->st_fb) return st_marginal(c->st_fb, k, u, out);  // a solve of it needed the log domain
    if (c->batched) {
        mmot_status st = bat_import(c, u);
        if (st) return st;
        mmot::BatchArgs a = c->ba;
        a.k = k;
        a.out = static_cast<double *>(out);
        CK(c, mmot::launch_batched(a, 1, c->stream, &c->launches));
        return MMOT_OK;
    }
    mmot_status st = reset_scalars(c);
    if (st) return st;
    c->exch_error = 0;
    const double *lin[mmot::kMaxL];
    st = to_linear(c, u, lin);
    if (st) return st;
    Plan p = make_plan(c, k, lin, nullptr, c->sw ? c->out_t : static_cast<double *>(out), 0);
    CK(c, mmot::launch_product(p, mmot::MODE_MARG, c->stream, &c->launches, prof_events(c, mmot::MODE_MARG)));
    if (c->exch_error) return MMOT_ENCCL;
    // precision guard (single walk) and range check (synchronises once): a product that left the
    // fp64 range is redone on the stabilised family
    if ((st = shard_agree(c, &c->dsc->stop, 6))) return st;
    if ((st = sync_report(c))) return st;
    if (c->sw && c->hsc->guard) {
        if (c->sharded) return guard_tripped(c);
        ++c->fallbacks;
        if ((st = ensure_fallback(c))) return st;
        return marginal_f64(c->fb, k, u, out);
    }
    if (c->hsc->status == MMOT_EOVERFLOW && can_stabilise(c)) {
        ++c->st_fallbacks;
        if ((st = ensure_stable(c))) return st;
        return st_marginal(c->st_fb, k, u, out);
    }
    if (c->hsc->status) {
        set_err(c, "%s", mmot_strerror((mmot_status)c->hsc->status));
        return (mmot_status)c->hsc->status;
    }
    if (c->sw)
        CK(c, mmot::launch_from_t(c->out_t, static_cast<double *>(out), c->N, c->P, c->nchunks, c->nchp, 0, c->stream,
                                  &c->launches));
    return MMOT_OK;
}

mmot_status mmot_sinkhorn(mmot_ctx *c, const void *const *marginals, int iters, double tol, void *const *u,
                          mmot_report *rep) {
    if (rep) { rep->iters_done = 0; rep->residual = NAN; rep->converged = 0; rep->status = 0; rep->fail_iter = -1; }
    if (!c || !marginals || !u) { set_err(c, "NULL argument"); return MMOT_EINVAL; }
    if (iters < 0 || isnan(tol)) { set_err(c, "iters must be >= 0"); return MMOT_EINVAL; }
    const double *mu[mmot::kStMaxL];
    for (int q = 0; q < c->l; ++q) {
        if (!marginals[q] || !u[q]) { set_err(c, "marginals[%d] or u[%d] is NULL", q, q); return MMOT_EINVAL; }
        mu[q] = static_cast<const double *>(marginals[q]);
    }
    cudaSetDevice(c->device);
    if (c->dt == MMOT_F32) {
        mmot_status st = f32_widen(c, marginals, mu);
        if (st) return st;
    }
    if (c->g2) return g2_sinkhorn(c, mu, iters, tol, u, rep);
    if (c->stable) return st_sinkhorn(c, mu, iters, tol, const_cast<const void *const *>(u), u, rep, nullptr);
    if (c->batched) return bat_sinkhorn(c, mu, iters, tol, u, rep);
    return sinkhorn_impl(c, mu, iters, tol, u, rep);
}

mmot_status mmot_sinkhorn_host(mmot_ctx *c, const void *const *marginals_host, int iters, double tol,
                               void *const *u_host, mmot_report *rep) {
    if (rep) { rep->iters_done = 0; rep->residual = NAN; rep->converged = 0; rep->status = 0; rep->fail_iter = -1; }
    if (!c || !marginals_host || !u_host) { set_err(c, "NULL argument"); return MMOT_EINVAL; }
    if (iters < 0 || isnan(tol)) { set_err(c, "iters must be >= 0"); return MMOT_EINVAL; }
    cudaSetDevice(c->device);
    const size_t bytes = (size_t)io_elems(c) * sizeof(double);
    const bool f32 = c->dt == MMOT_F32;
    if (f32 && !c->f32_stage) CK(c, cudaMalloc(&c->f32_stage, (size_t)c->l * io_elems(c) * sizeof(float)));
    for (int q = 0; q < c->l; ++q) {
        if (!marginals_host[q] || !u_host[q]) { set_err(c, "NULL host pointer"); return MMOT_EINVAL; }
        if (!c->stage_mu[q]) CK(c, cudaMalloc(&c->stage_mu[q], bytes));
        if (!c->stage_u[q]) CK(c, cudaMalloc(&c->stage_u[q], bytes));
        if (f32) {
            // fp32 marginals cross PCIe as floats and are widened on the device
            float *fs = c->f32_stage + (size_t)q * io_elems(c);
            CK(c, cudaMemcpyAsync(fs, marginals_host[q], (size_t)io_elems(c) * sizeof(float), cudaMemcpyHostToDevice,
                                  c->stream));
            CK(c, mmot::launch_convert(fs, c->stage_mu[q], io_elems(c), 1, c->stream, &c->launches));
        } else {
            CK(c, cudaMemcpyAsync(c->stage_mu[q], marginals_host[q], bytes, cudaMemcpyHostToDevice, c->stream));
        }
        CK(c, cudaMemcpyAsync(c->stage_u[q], u_host[q], bytes, cudaMemcpyHostToDevice, c->stream));
    }
    const double *mu[mmot::kStMaxL];
    void *ud[mmot::kStMaxL];
    for (int q = 0; q < c->l; ++q) {
        mu[q] = c->stage_mu[q];
        ud[q] = c->stage_u[q];
    }
    mmot_status st = c->g2        ? g2_sinkhorn(c, mu, iters, tol, ud, rep)
                     : c->stable  ? st_sinkhorn(c, mu, iters, tol, const_cast<const void *const *>(ud), ud, rep, nullptr)
                     : c->batched ? bat_sinkhorn(c, mu, iters, tol, ud, rep)
                                  : sinkhorn_impl(c, mu, iters, tol, ud, rep);
    for (int q = 0; q < c->l; ++q)
        CK(c, cudaMemcpyAsync(u_host[q], c->stage_u[q], bytes, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    return st;
}

mmot_status mmot_cost(mmot_ctx *c, const void *const *u, double *W) {
    if (!c || !u || !W) { set_err(c, "NULL argument"); return MMOT_EINVAL; }
    cudaSetDevice(c->device);
    if (c->g2) return g2_cost(c, u, W);
    if (c->stable) return st_cost(c, u, W);
    if (c->batched && c->st_fb) return st_cost(c->st_fb, u, W);
    if (c->batched) {
        mmot_status st = bat_import(c, u);
        if (st) return st;
        mmot::BatchArgs a = c->ba;
        a.k = c->l - 1;
        CK(c, mmot::launch_batched(a, 2, c->stream, &c->launches));
        CK(c, cudaMemcpyAsync(c->bat_whost, c->ba.wout, (size_t)c->batch * sizeof(double), cudaMemcpyDeviceToHost,
                              c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
        memcpy(W, c->bat_whost, (size_t)c->batch * sizeof(double));
        return MMOT_OK;
    }
    mmot_status st = reset_scalars(c);
    if (st) return st;
    c->exch_error = 0;
    const double *lin[mmot::kMaxL];
    st = to_linear(c, u, lin);
    if (st) return st;
    const int k = c->l - 1;
    Plan p = make_plan(c, k, lin, nullptr, nullptr, 0);
    CK(c, mmot::launch_product(p, mmot::MODE_COST, c->stream, &c->launches, prof_events(c, mmot::MODE_COST)));
    // uniform grids: hatJ counts crossed edges (W = h <phi, hatJ>); non-uniform: the duals carry h_e
    CK(c, mmot::launch_sum(c->partial, c->nchunks, &c->dsc->W, c->pts_lam ? 1.0 : c->h, 0, &c->dsc->stop, c->stream,
                           &c->launches));
    st = shard_allreduce(c, &c->dsc->W);
    if (st) return st;
    if ((st = shard_agree(c, &c->dsc->stop, 6))) return st;
    st = sync_report(c);
    if (st) return st;
    if (c->exch_error) return MMOT_ENCCL;
    if (c->sw && c->hsc->guard && (!c->hsc->status || c->hsc->status == MMOT_EOVERFLOW)) {
        if (c->sharded) return guard_tripped(c);
        ++c->fallbacks;
        if ((st = ensure_fallback(c))) return st;
        return mmot_cost(c->fb, u, W);
    }
    if (c->hsc->status == MMOT_EOVERFLOW && can_stabilise(c)) {
        ++c->st_fallbacks;
        if ((st = ensure_stable(c))) return st;
        return st_cost(c->st_fb, u, W);
    }
    *W = c->hsc->W;
    return (mmot_status)c->hsc->status;
}

mmot_status mmot_profile_enable(mmot_ctx *c, int enable) {
    if (!c) { set_err(c, "NULL context"); return MMOT_EINVAL; }
    c->prof = enable != 0;
    return MMOT_OK;
}

mmot_status mmot_profile_read(mmot_ctx *c, double *ms, double *ms_mode, int64_t *n_mode) {
    if (!c) { set_err(c, "NULL context"); return MMOT_EINVAL; }
    CK(c, cudaStreamSynchronize(c->stream));
    double acc[4] = {0, 0, 0, 0}, accm[4] = {0, 0, 0, 0};
    int64_t nm[4] = {0, 0, 0, 0};
    for (size_t i = 0; i + 4 <= c->used; i += 4) {
        float t01 = 0, t12 = 0, t23 = 0, t03 = 0;
        CK(c, cudaEventElapsedTime(&t01, c->pool[i], c->pool[i + 1]));
        CK(c, cudaEventElapsedTime(&t12, c->pool[i + 1], c->pool[i + 2]));
        CK(c, cudaEventElapsedTime(&t23, c->pool[i + 2], c->pool[i + 3]));
        CK(c, cudaEventElapsedTime(&t03, c->pool[i], c->pool[i + 3]));
        acc[0] += t01; acc[1] += t12; acc[2] += t23; acc[3] += t03;
        const int m = c->pool_mode[i / 4];
        accm[m] += t03;
        nm[m] += 1;
    }
    c->used = 0;
    c->pool_mode.clear();
    if (ms) for (int i = 0; i < 4; ++i) ms[i] = acc[i];
    if (ms_mode) for (int i = 0; i < 4; ++i) ms_mode[i] = accm[i];
    if (n_mode) for (int i = 0; i < 4; ++i) n_mode[i] = nm[i];
    return MMOT_OK;
}

mmot_status mmot_cost_staged(mmot_ctx *c, double *W) {
    if (!c || !W) { set_err(c, "NULL argument"); return MMOT_EINVAL; }
    const void *u[mmot::kStMaxL];
    for (int q = 0; q < c->l; ++q) {
        if (!c->stage_u[q]) { set_err(c, "mmot_cost_staged before mmot_sinkhorn_host"); return MMOT_EINVAL; }
        u[q] = c->stage_u[q];
    }
    return mmot_cost(c, u, W);
}

mmot_status mmot_init_uniform(mmot_ctx *c, void *const *u) {
    if (!c || !u) { set_err(c, "NULL argument"); return MMOT_EINVAL; }
    cudaSetDevice(c->device);
    // a shard starts from the global problem's 1/N
    const double Ng = (double)(c->sharded ? c->N_global : c->N);
    const double v = c->opts.repr == MMOT_LOG ? -log(Ng) : 1.0 / Ng;
    for (int q = 0; q < c->l; ++q) {
        if (!u[q]) { set_err(c, "u[%d] is NULL", q); return MMOT_EINVAL; }
        CK(c, mmot::launch_fill(static_cast<double *>(u[q]), v, c->N * c->batch, c->stream, &c->launches));
    }
    return MMOT_OK;
}

mmot_status mmot_nccl_unique_id(void *out) {
    if (!out) { set_err(nullptr, "out is NULL"); return MMOT_EINVAL; }
    if (!nccl_load()) { set_err(nullptr, "libnccl.so.2 not found"); return MMOT_ENCCL; }
    const nccl_result r = g_nccl.GetUniqueId(out);
    if (r != 0) { set_err(nullptr, "ncclGetUniqueId: %s", g_nccl.GetErrorString(r)); return MMOT_ENCCL; }
    return MMOT_OK;
}

void mmot_shard_range(int64_t N_global, int rank, int world, int64_t *lo, int64_t *hi) {
    if (lo) *lo = world > 0 ? (int64_t)((__int128)N_global * rank / world) : 0;
    if (hi) *hi = world > 0 ? (int64_t)((__int128)N_global * (rank + 1) / world) : 0;
}

mmot_status mmot_compose_rank_carries(int l, const double *ops_all, int world, int rank, double *fin, double *bin) {
    if (!ops_all || !fin || !bin || world < 1 || rank < 0 || rank >= world) { set_err(nullptr, "bad arguments"); return MMOT_EINVAL; }
    switch (l - 1) {
        case 1: mmot::compose_rank_carries<1, double>(ops_all, world, rank, fin, bin); break;
        case 2: mmot::compose_rank_carries<2, double>(ops_all, world, rank, fin, bin); break;
        case 3: mmot::compose_rank_carries<3, double>(ops_all, world, rank, fin, bin); break;
        case 4: mmot::compose_rank_carries<4, double>(ops_all, world, rank, fin, bin); break;
        case 5: mmot::compose_rank_carries<5, double>(ops_all, world, rank, fin, bin); break;
        default: set_err(nullptr, "l=%d unsupported", l); return MMOT_EINVAL;
    }
    return MMOT_OK;
}

mmot_status mmot_compose_rank_affine(int l, const double *elems_all, int world, int rank, double *fin, double *bin) {
    if (!elems_all || !fin || !bin || world < 1 || rank < 0 || rank >= world) { set_err(nullptr, "bad arguments"); return MMOT_EINVAL; }
    switch (l - 1) {
        case 2: mmot::compose_rank_affine<2>(elems_all, world, rank, fin, bin); break;
        case 3: mmot::compose_rank_affine<3>(elems_all, world, rank, fin, bin); break;
        case 4: mmot::compose_rank_affine<4>(elems_all, world, rank, fin, bin); break;
        default: set_err(nullptr, "l=%d unsupported (3..5)", l); return MMOT_EINVAL;
    }
    return MMOT_OK;
}

static mmot_status create_sharded(int l, int64_t N_global, double eta, mmot_grid grid, mmot_dtype dt,
                                  const void *nccl_unique_id, mmot_vgroup *vg, int rank, int world,
                                  const mmot_opts *opts, void *cuda_stream, mmot_ctx **out) {
    if (!out) { set_err(nullptr, "out is NULL"); return MMOT_EINVAL; }
    *out = nullptr;
    if ((!nccl_unique_id && !vg) || world < 1 || rank < 0 || rank >= world) { set_err(nullptr, "bad rank/world/id"); return MMOT_EINVAL; }
    if (vg && world != vg->world) { set_err(nullptr, "world=%d differs from the group's %d", world, vg->world); return MMOT_EINVAL; }
    int64_t lo, hi;
    mmot_shard_range(N_global, rank, world, &lo, &hi);
    if (N_global < world) { set_err(nullptr, "N_global=%lld < world=%d", (long long)N_global, world); return MMOT_ESHAPE; }
    // the shard's grid: same spacing h as the global grid, x_min shifted to the shard start
    const double h = N_global > 1 ? (grid.x_max - grid.x_min) / (double)(N_global - 1) : 1.0;
    mmot_grid g2{grid.x_min + lo * h, grid.x_min + (hi - 1) * h};
    if (hi - lo == 1) g2.x_max = g2.x_min + h;  // a 1-point shard keeps the global h below
    mmot_ctx *c = nullptr;
    mmot_status st = create_single(l, hi - lo, eta, g2, dt, opts, cuda_stream, &c, false, rank + 1 < world);
    if (st) return st;
    c->h = h;
    for (int a = 0; a <= mmot::kMaxL; ++a) {
        const int e = a <= l ? a * (l - a) : 0;
        c->W.w[a] = a <= l ? exp(-(double)e * h / eta) : 0.0;
    }
    c->sharded = true;
    c->rank = rank;
    c->world = world;
    c->N_global = N_global;
    c->lo = lo;
    c->grid = grid;
    const size_t SZ = (size_t)l * (1 << (l - 1));
    const size_t nd = (2 * SZ + (size_t)world * 2 * SZ + 2 * (1 << (l - 1))) * 2;  // Dual-sized
    if (cudaMalloc(&c->shard_mem, nd * sizeof(double)) != cudaSuccess ||
        (vg && cudaMalloc(&c->vg_tmp, 16 * sizeof(double)) != cudaSuccess)) {
        set_err(c, "shard workspace allocation failed");
        snprintf(g_err, sizeof g_err, "%s", c->err);
        mmot_destroy(c);
        return MMOT_ENOMEM;
    }
    if (vg) {
        c->vg = vg;
    } else {
        if (!nccl_load()) {
            set_err(c, "libnccl.so.2 not found");
            snprintf(g_err, sizeof g_err, "%s", c->err);
            mmot_destroy(c);
            return MMOT_ENCCL;
        }
        ncclUniqueIdBytes id;
        memcpy(id.internal, nccl_unique_id, sizeof id.internal);
        const nccl_result r = g_nccl.CommInitRank(&c->comm, world, id, rank);
        if (r != 0) {
            set_err(c, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
            snprintf(g_err, sizeof g_err, "%s", c->err);
            c->comm = nullptr;
            mmot_destroy(c);
            return MMOT_ENCCL;
        }
    }
    // Every rank must run the same collective sequence with the same payloads: the kernel family
    // and the scan mode, chosen from the local shard size, have to agree across ranks.
    {
        const double sig = (double)((c->sw ? 4 : 0) + (c->rx ? 2 : 0) + (c->nlev >= 2 ? 1 : 0));
        std::vector<double> all((size_t)world);
        double *d = c->shard_mem;
        bool ok = cudaMemcpyAsync(d, &sig, sizeof sig, cudaMemcpyHostToDevice, c->stream) == cudaSuccess &&
                  coll_allgather(c, d, d + 1, 1, c->stream) == 0 &&
                  cudaMemcpyAsync(all.data(), d + 1, (size_t)world * sizeof(double), cudaMemcpyDeviceToHost,
                                  c->stream) == cudaSuccess &&
                  cudaStreamSynchronize(c->stream) == cudaSuccess;
        for (int r2 = 0; ok && r2 < world; ++r2) ok = all[r2] == sig;
        if (!ok) {
            set_err(c, "sharded context: ranks chose different kernel configurations (shard sizes too uneven)");
            snprintf(g_err, sizeof g_err, "%s", c->err);
            mmot_destroy(c);
            return MMOT_ESHAPE;
        }
    }
    *out = c;
    return MMOT_OK;
}

mmot_status mmot_create_sharded(int l, int64_t N_global, double eta, mmot_grid grid, mmot_dtype dt,
                                const void *nccl_unique_id, int rank, int world, const mmot_opts *opts,
                                void *cuda_stream, mmot_ctx **out) {
    if (!nccl_unique_id) {
        if (out) *out = nullptr;
        set_err(nullptr, "nccl_unique_id is NULL");
        return MMOT_EINVAL;
    }
    return create_sharded(l, N_global, eta, grid, dt, nccl_unique_id, nullptr, rank, world, opts, cuda_stream, out);
}

mmot_status mmot_vgroup_create(int world, mmot_vgroup **out) {
    if (!out) { set_err(nullptr, "out is NULL"); return MMOT_EINVAL; }
    *out = nullptr;
    if (world < 1 || world > mmot::kMaxWorld) { set_err(nullptr, "world=%d outside [1,%d]", world, mmot::kMaxWorld); return MMOT_EINVAL; }
    mmot_vgroup *g = new mmot_vgroup();
    g->world = world;
    g->src.assign((size_t)world, nullptr);
    g->ready.assign((size_t)world, nullptr);
    g->done.assign((size_t)world, nullptr);
    for (int r = 0; r < world; ++r)
        if (cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming) != cudaSuccess) {
            set_err(nullptr, "cudaEventCreate failed");
            mmot_vgroup_destroy(g);
            return MMOT_ECUDA;
        }
    *out = g;
    return MMOT_OK;
}

void mmot_vgroup_destroy(mmot_vgroup *g) {
    if (!g) return;
    for (cudaEvent_t e : g->ready) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : g->done) if (e) cudaEventDestroy(e);
    delete g;
}

mmot_status mmot_create_sharded_virtual(int l, int64_t N_global, double eta, mmot_grid grid, mmot_dtype dt,
                                        mmot_vgroup *group, int rank, const mmot_opts *opts, void *cuda_stream,
                                        mmot_ctx **out) {
    if (!group) {
        if (out) *out = nullptr;
        set_err(nullptr, "group is NULL");
        return MMOT_EINVAL;
    }
    return create_sharded(l, N_global, eta, grid, dt, nullptr, group, rank, group->world, opts, cuda_stream, out);
}

}  // extern "C"
